// Gathered-row streaming rate vs the per-row chunk size (the access pattern of
// the selective GEMM's A operand).  148 CTAs (one per SM) x 128 loader
// threads stream R gathered 8 KB rows each through a ring of 16 KB stages with
// 16-byte cp.async; a stage holds 16384/C rows x C bytes (C = bytes of one row
// per stage: 128 = the K-block of 64 bf16 the GEMM uses, 8192 = whole rows).
// A consumer thread releases stages.  Every launch reads 8 distinct weight
// matrices (8 x 64 MB of selected rows, > L2); reports TB/s.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_2505_14884_b200/csrc/common.cuh"
namespace ps { int g_pdl = 0; }
using namespace ps;

constexpr int kLd = 128;

template <bool HINT>
__global__ void __launch_bounds__(kLd + 32, 1) gather_kernel(const uint16_t* w, const int* idx, int n_sel, int D,
                                                            int chunk, int S, int mats, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * 16384);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], kLd);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int rows_per_cta = n_sel / gridDim.x;
  const int r0 = blockIdx.x * rows_per_cta;
  const int rows_per_stage = 16384 / chunk;
  const int chunks_per_row = 8192 / chunk;
  // stage order: row groups of rows_per_stage, walking the row chunks (like the GEMM's K loop)
  const int groups = rows_per_cta / rows_per_stage;
  const int stages_total = mats * groups * chunks_per_row;
  if (tid < kLd) {
    for (int i = 0; i < stages_total; ++i) {
      const int s = i % S;
      if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
      const int mat = i / (groups * chunks_per_row);
      const int rem = i % (groups * chunks_per_row);
      const int grp = rem / chunks_per_row, ck = rem % chunks_per_row;
      const uint8_t* base = reinterpret_cast<const uint8_t*>(w) + (size_t)mat * D * 8192;
      uint8_t* dst = smem + s * 16384;
#pragma unroll 8
      for (int j = 0; j < 8; ++j) {
        const int c = j * kLd + tid;            // 16-byte unit of the stage
        const int rr = c / (chunk / 16);        // row within the stage
        const int off = (c % (chunk / 16)) * 16;
        const int row = __ldg(idx + r0 + grp * rows_per_stage + rr);
        const uint8_t* src = base + (size_t)row * 8192 + ck * chunk + off;
        if (HINT) cp_async16_l2_256(dst + c * 16, src, 16);
        else cp_async16(dst + c * 16, src, 16);
      }
      cp_async_arrive_noinc(&full[s]);
    }
  } else if (tid == kLd) {
    unsigned long long acc = 0;
    for (int i = 0; i < stages_total; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      acc += smem[s * 16384 + (i & 1023)];
      mbar_arrive(&empty[s]);
    }
    if (acc == 0x1234567) sink[0] = acc;
  }
}

int main() {
  const int D = 32768, mats = 4;
  int n_sel = 148 * 128;  // ~0.58 D per matrix, 128 rows per CTA
  std::vector<int> h(D);
  for (int i = 0; i < D; ++i) h[i] = i;
  srand(1);
  std::random_shuffle(h.begin(), h.end());
  h.resize(n_sel);
  std::sort(h.begin(), h.end());
  uint16_t* w;
  int* idx;
  unsigned long long* sink;
  cudaMalloc(&w, (size_t)mats * D * 8192);
  cudaMemset(w, 0, (size_t)mats * D * 8192);
  cudaMalloc(&idx, n_sel * 4);
  cudaMemcpy(idx, h.data(), n_sel * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&sink, 8);
  for (int hint = 0; hint < 2; ++hint) {
    for (int chunk : {128, 256, 512, 1024, 2048, 8192}) {
      for (int S : {4, 12}) {
        auto k = hint ? gather_kernel<true> : gather_kernel<false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        const size_t smem = (size_t)S * 16384 + 2 * S * 8;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
          cudaEventRecord(a);
          k<<<148, kLd + 32, smem>>>(w, idx, n_sel, D, chunk, S, mats, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep) best = std::min(best, ms);
        }
        const double bytes = (double)mats * n_sel * 8192;
        printf("hint=%d chunk %5d B  S=%2d: %7.1f us  %5.2f TB/s\n", hint, chunk, S, best * 1e3,
               bytes / (best * 1e-3) / 1e12);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
