// Launch-overhead microbenchmark (standalone; not part of libpolar_b200):
// graph of 50 launches per variant, reports us per launch.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2505_14884_b200/csrc/common.cuh"
using namespace ps;

template <int VARIANT>
__global__ void __launch_bounds__(320, 2) kern(const uint16_t* src, int* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (VARIANT >= 2 && threadIdx.x < 32) {  // TMEM alloc/dealloc
    tmem_alloc(&slot, 128);
  }
  if (VARIANT >= 3 && threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (VARIANT >= 3 && threadIdx.x == 0) {  // one 16 KB bulk copy round trip
    mbar_arrive_expect_tx(&bar, 16384);
    bulk_g2s(smem, src + (size_t)blockIdx.x * 8192, 16384, &bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  if (VARIANT >= 2 && threadIdx.x < 32) tmem_dealloc(slot, 128);
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = smem[0];
}

template <int V>
float run(int grid, size_t smem, int cluster, const uint16_t* src, int* out) {
  cudaFuncSetAttribute(kern<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t st;
  cudaStreamCreate(&st);
  auto launch = [&]() {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern<V>, src, out);
    if (e != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(e));
  };
  for (int i = 0; i < 5; ++i) launch();
  cudaStreamSynchronize(st);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 50; ++i) launch();
  cudaStreamEndCapture(st, &g);
  if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return -1.f; }
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms * 1000.f / 50;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  printf("start\n");
  uint16_t* src;
  int* out;
  cudaMalloc(&src, 64 << 20);
  cudaMalloc(&out, 4);
  for (int cl : {1, 2, 8}) {
    printf("cluster %d: empty/0KB %.2f | empty/105KB %.2f | +TMEM %.2f | +TMEM+bulk16KB %.2f  (grid 296, us)\n", cl,
           run<0>(296, 0, cl, src, out), run<0>(296, 105 * 1024, cl, src, out),
           run<2>(296, 105 * 1024, cl, src, out), run<3>(296, 105 * 1024, cl, src, out));
  }
  fflush(stdout);
  printf("grid 148 cluster 1: empty/105KB %.2f | +TMEM+bulk %.2f\n", run<0>(148, 105 * 1024, 1, src, out),
         run<3>(148, 105 * 1024, 1, src, out));
  return 0;
}
