// Minimal programmatic-dependent-launch probe: kernel A (few CTAs) triggers
// launch_dependents and then spins ~20 us; kernel B (PDL attribute) stamps
// its CTA start times.  B starting before A ends == PDL overlap works.
// Variants: trigger by thread 0 only / by every thread; stream vs graph.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o pdl_test pdl_test.cu && ./pdl_test
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void kA(unsigned long long* st, int mode, int spin_ns) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (mode == 0 && threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (mode == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  unsigned long long t0 = gt();
  if (threadIdx.x == 0) st[blockIdx.x * 2] = t0;
  while (gt() - t0 < (unsigned long long)spin_ns) {
  }
  if (threadIdx.x == 0) st[blockIdx.x * 2 + 1] = gt();
}

__global__ void kB(unsigned long long* st) {
  if (threadIdx.x == 0) st[blockIdx.x] = gt();
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

int launch(void (*k)(unsigned long long*, int, int), dim3 g, dim3 b, size_t smem, cudaStream_t s, bool pdl,
           unsigned long long* p, int mode, int spin) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g; cfg.blockDim = b; cfg.dynamicSmemBytes = smem; cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, p, mode, spin);
}
int launchB(dim3 g, dim3 b, size_t smem, cudaStream_t s, bool pdl, unsigned long long* p, int cluster = 1) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g; cfg.blockDim = b; cfg.dynamicSmemBytes = smem; cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster; at[n].val.clusterDim.y = 1; at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at; cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kB, p);
}

int main() {
  unsigned long long *a, *b;
  cudaMalloc(&a, 4096 * 8);
  cudaMalloc(&b, 4096 * 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  unsigned long long ha[4096], hb[4096];
  const int nA = 64, nB = 148;
  cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(kB, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int variants[][3] = {{0, 0, 1}, {160, 0, 1}, {160, 108, 1}, {160, 108, 2}, {160, 108, 4}, {160, 108, 8},
                             {0, 108, 4}, {0, 0, 4}};
  for (auto& v : variants)
  for (int graph = 1; graph < 2; ++graph)
    for (int mode = 1; mode < 2; ++mode) {
      const size_t smA = v[0] * 1024, smB = v[1] * 1024;
      const int cl = v[2];
      const int nBv = (nB / cl) * cl;
      cudaMemset(a, 0, 4096 * 8);
      cudaMemset(b, 0, 4096 * 8);
      cudaDeviceSynchronize();
      cudaGraphExec_t ge = nullptr;
      if (graph) {
        cudaGraph_t gr;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        launch(kA, dim3(nA), dim3(512), smA, s, true, a, mode, 20000);
        launchB(dim3(nBv), dim3(256), smB, s, true, b, cl);
        cudaStreamEndCapture(s, &gr);
        if (cudaGraphInstantiate(&ge, gr, 0) != cudaSuccess) printf("instantiate failed\n");
        cudaGraphLaunch(ge, s);
      } else {
        int r1 = launch(kA, dim3(nA), dim3(512), 0, s, true, a, mode, 20000);
        int r2 = launchB(dim3(nB), dim3(256), 0, s, true, b);
        if (r1 || r2) printf("launch err %d %d\n", r1, r2);
      }
      cudaStreamSynchronize(s);
      cudaError_t e = cudaGetLastError();
      cudaMemcpy(ha, a, nA * 16, cudaMemcpyDeviceToHost);
      cudaMemcpy(hb, b, nB * 8, cudaMemcpyDeviceToHost);
      unsigned long long a0 = ~0ull, a1 = 0, b0 = ~0ull, b1 = 0;
      for (int i = 0; i < nA; ++i) { a0 = ha[2 * i] < a0 ? ha[2 * i] : a0; a1 = ha[2 * i + 1] > a1 ? ha[2 * i + 1] : a1; }
      for (int i = 0; i < nBv; ++i) { b0 = hb[i] < b0 ? hb[i] : b0; b1 = hb[i] > b1 ? hb[i] : b1; }
      printf("smemA %3dK smemB %3dK cluster %d: ", v[0], v[1], v[2]);
      printf("%s trigger=%s: A %.2f..%.2f us, B start %.2f..%.2f us  (%s)\n", graph ? "graph " : "stream",
             mode == 0 ? "tid0 " : (mode == 1 ? "all  " : "none "), 0.0, (a1 - a0) / 1e3, ((long long)(b0 - a0)) / 1e3,
             ((long long)(b1 - a0)) / 1e3, cudaGetErrorString(e));
    }
  return 0;
}
