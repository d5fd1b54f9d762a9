// Streaming-bandwidth microbenchmark for the gathered-row A operand of the
// selective GEMM (d = 4096 bf16 rows = 8 KB, ~half of 16384 rows selected):
// G CTAs each stream their rows into an S-stage ring of 16 KB stages; one
// consumer thread releases stages (no MMA).  Copy engines compared:
//   mode 0: cp.async 16 B (LDGSTS) by L loader warps
//   mode 1: LDG.128 + STS.128 by L loader warps
//   mode 2: 1-D bulk copies (TMA engine) of whole 8 KB rows, one thread
//   mode 3: 1-D bulk copies of 128-byte row chunks (the SW128 K-block shape)
// Reports aggregate GB/s (best of 7, CUDA events, includes launch).
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_2505_14884_b200/csrc/common.cuh"
namespace ps { int g_pdl = 0; }
using namespace ps;

template <int MODE, int LW>
__global__ void __launch_bounds__(32 * LW + 32) stream_kernel(const uint16_t* w, const int* idx, int rows_per_cta,
                                                             int S, unsigned long long* sink, int passes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int kLd = 32 * LW;
  constexpr int row_bytes = 8192;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * 16384);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x;
  __shared__ int s_rows[512];
  const int r0 = blockIdx.x * rows_per_cta;
  for (int r = tid; r < rows_per_cta; r += blockDim.x) s_rows[r] = __ldg(idx + r0 + r);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], (MODE == 2 || MODE == 3) ? 1 : kLd);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int stages_per_pass = rows_per_cta * row_bytes / 16384;
  const int stages_total = stages_per_pass * passes;
  if (tid < kLd) {
    if (MODE == 0 || MODE == 1) {
      for (int i = 0; i < stages_total; ++i) {
        const int s = i % S;
        if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        uint8_t* dst = smem + s * 16384;
        constexpr int per = 1024 / kLd;  // 16-byte chunks per thread per stage
        uint4 v[per];
#pragma unroll
        for (int j = 0; j < per; ++j) {
          const int c = j * kLd + tid;
          const int rr = (i % stages_per_pass) * 2 + c / 512;
          const uint8_t* src = reinterpret_cast<const uint8_t*>(w) + (size_t)s_rows[rr] * row_bytes + (c % 512) * 16;
          if (MODE == 0) cp_async16(dst + c * 16, src, 16);
          else v[j] = __ldg(reinterpret_cast<const uint4*>(src));
        }
        if (MODE == 1) {
#pragma unroll
          for (int j = 0; j < per; ++j) *reinterpret_cast<uint4*>(dst + (j * kLd + tid) * 16) = v[j];
          mbar_arrive(&full[s]);
        } else {
          cp_async_arrive_noinc(&full[s]);
        }
      }
    } else if (tid == 0) {
      for (int i = 0; i < stages_total; ++i) {
        const int s = i % S;
        if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        uint8_t* dst = smem + s * 16384;
        mbar_arrive_expect_tx(&full[s], 16384);
        if (MODE == 2) {
          for (int r = 0; r < 2; ++r)
            bulk_g2s(dst + r * 8192, reinterpret_cast<const uint8_t*>(w) + (size_t)s_rows[(i % stages_per_pass) * 2 + r] * row_bytes, 8192,
                     &full[s]);
        } else {
          // 128 rows x 128 B (K-block of 64): rows cycle over this CTA's rows
          for (int r = 0; r < 128; ++r) {
            const int rr = (i * 128 + r) % rows_per_cta;
            const int kb = ((i * 128 + r) / rows_per_cta) % 64;
            bulk_g2s(dst + r * 128, reinterpret_cast<const uint8_t*>(w) + (size_t)s_rows[rr] * row_bytes + kb * 128,
                     128, &full[s]);
          }
        }
      }
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

template <int MODE, int LW>
void run(const char* name, const uint16_t* w, const int* idx, unsigned long long* sink, int D, int d, int n_sel) {
  cudaFuncSetAttribute(stream_kernel<MODE, LW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int G : {52, 74, 104, 148, 296}) {
    for (int S : {4, 8, 13}) {
      const int rows_per_cta = (n_sel / G) & ~1;
      const size_t smem = (size_t)S * 16384 + 2 * S * 8;
      float t[2];
      for (int pi = 0; pi < 2; ++pi) {
        const int passes = pi == 0 ? 1 : 4;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
          const uint16_t* wc = w + (size_t)(rep % 4) * D * d;
          cudaEventRecord(a);
          stream_kernel<MODE, LW><<<G, 32 * LW + 32, smem>>>(wc, idx, rows_per_cta, S, sink, passes);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          if (rep > 0) best = std::min(best, ms);
        }
        t[pi] = best * 1e3f;
      }
      const double bytes = (double)rows_per_cta * G * d * 2;
      const double rate = 3 * bytes / ((t[1] - t[0]) * 1e-6) / 1e9;
      printf("%-18s G=%3d S=%d: 1 pass %6.1f us, 4 passes %6.1f us -> steady %5.0f GB/s (%4.1f GB/s/CTA), fixed %4.1f us\n",
             name, G, S, t[0], t[1], rate, rate / G, t[0] - bytes / (rate * 1e9) * 1e6);
    }
  }
}

int main() {
  const int D = 16384, d = 4096, n_sel = 8192;
  std::vector<int> h(n_sel);
  for (int i = 0; i < n_sel; ++i) h[i] = (i * 2 + (i % 3 == 0)) % D;
  std::sort(h.begin(), h.end());
  uint16_t* w; int* idx; unsigned long long* sink;
  cudaMalloc(&w, (size_t)4 * D * d * 2);
  cudaMemset(w, 0, (size_t)4 * D * d * 2);
  cudaMalloc(&idx, n_sel * 4);
  cudaMemcpy(idx, h.data(), n_sel * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&sink, 8);
  run<0, 4>("cp.async 4 warps", w, idx, sink, D, d, n_sel);
  run<3, 1>("bulk 128B chunks", w, idx, sink, D, d, n_sel);


  run<2, 1>("bulk 8KB rows", w, idx, sink, D, d, n_sel);

  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
