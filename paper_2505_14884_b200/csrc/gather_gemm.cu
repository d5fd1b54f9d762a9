// Gathered GEMMs on 5th-generation tensor cores (tcgen05 + TMEM), sm_100a.
//
// Polar Sparsity's selective MLP (Alg. 2, kernels.py:223-256 / 353-373)
// touches only the batch-union S of active neurons.  Weights are stored
// NEURON-MAJOR (W1^T, W2^T as (D, d) rows) so each selected neuron is one
// contiguous 2*d-byte row and both projections become row gathers:
//
//   rows form   (MODE_UP):   out[n, j] = act(sum_k W[idx[j], k] x[n, k] + b[idx[j]])
//   contraction (MODE_DOWN): out[n, m] = sum_j h[n, j] W[idx[j], m] + b[m] (+ res)
//
// Swap-AB mapping for decode: the MMA M dimension (128) runs over the
// weight side (neurons for UP, output features for DOWN) and N over the
// batch (16..256), so even a batch of 16 uses full 128-row UMMA tiles.
//   * 4 producer warps gather operands with 16-byte cp.async (LDGSTS) into
//     128B-swizzled shared memory: K-major rows for UP; for DOWN the gathered
//     rows are K slices, stored MN-major (tcgen05 transposes via the
//     instruction descriptor);  mbarrier full/empty ring of stages;
//   * one elected thread issues tcgen05.mma (M=128, N=batch, K=16) into a
//     TMEM accumulator and commits stages back to the producers;
//   * the 4 producer warps then drain TMEM (tcgen05.ld 32x32b) and apply the
//     epilogue (bias, ReLU, bf16/f32 store, residual add);
//   * split-K over CTAs for parallelism at small S / d; the last CTA of a
//     tile (atomic ticket, self-resetting) reduces the f32 partials in a
//     fixed order, so results are deterministic.
// The device-resident union size (*count) bounds the work: tiles/blocks
// beyond it exit without touching memory, so no host sync is needed and the
// whole MLP is CUDA-graph capturable.
#include "common.cuh"

namespace ps {
namespace {

constexpr int BM = 128;   // UMMA M
constexpr int BK = 64;    // K elements per stage (one 128-byte swizzle row)
constexpr int kEpiThreads = 128;
constexpr int kThreads = 160;  // warps 0-3 producer+epilogue, warp 4 MMA
constexpr int kMaxNB = 256;
constexpr int kTicketBytes = 65536;

enum { MODE_UP = 0, MODE_DOWN = 1 };

struct GGParams {
  const uint16_t* w;
  int64_t w_ld;
  const int32_t* idx;
  const int32_t* count;
  const uint16_t* x;  // B operand rows (N, K)
  int64_t x_ld;
  const float* bias;
  const float* residual;
  int64_t res_ld;
  int N, M, K;  // UP: M = output columns (neurons), K = d.  DOWN: M = d, K = max union size
  int act;
  int splits;
  int NB;       // batch rows per CTA tile (multiple of 16, <= 256)
  int stages;
  void* out;
  int64_t out_ld;
  int out_bf16;
  int* tickets;
  float* partials;
};

PS_DEV uint32_t sw128(int row, int unit) {  // byte offset inside a K-major SW128 atom column
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((unit ^ (row & 7)) << 4));
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) gather_gemm_kernel(const GGParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NB = p.NB;
  const uint32_t a_bytes = BM * BK * 2;          // 16 KB
  const uint32_t b_bytes = (uint32_t)NB * BK * 2;  // NB * 128
  const uint32_t stage_bytes = a_bytes + b_bytes;
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* accum = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mt = blockIdx.x, split = blockIdx.y, ntile = blockIdx.z;
  const int m0 = mt * BM;
  const int n0 = ntile * NB;
  const int count = p.count ? *p.count : (MODE == MODE_UP ? p.M : p.K);

  // work bounds (uniform across the CTA)
  if (MODE == MODE_UP && m0 >= count) return;  // beyond the union: nothing to write
  const int klimit = (MODE == MODE_UP) ? p.K : count;
  const int kbt = (klimit + BK - 1) / BK;
  const int per = (kbt + p.splits - 1) / p.splits;
  const int kb0 = split * per;
  const int nkb = max(0, min(kbt, kb0 + per) - kb0);

  const uint32_t tcols = NB <= 32 ? 32 : (NB <= 64 ? 64 : (NB <= 128 ? 128 : 256));
  if (warp == 4) {
    if (lane == 0) {
      for (int s = 0; s < S; ++s) {
        mbar_init(&full[s], kEpiThreads);
        mbar_init(&empty[s], 1);
      }
      mbar_init(accum, 1);
      fence_mbar_init();
    }
    __syncwarp();
    tmem_alloc(tmem_slot, tcols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------------------ producers
    const int t = tid;
    // UP: thread t owns A row t (one gathered weight row)
    const uint16_t* a_row = nullptr;
    if (MODE == MODE_UP) {
      const int gr = m0 + t;
      if (gr < count) a_row = p.w + (size_t)(p.idx ? p.idx[gr] : gr) * p.w_ld;
    }
    for (int i = 0; i < nkb; ++i) {
      const int s = i % S;
      if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
      uint8_t* sa = smem + s * stage_bytes;
      uint8_t* sb = sa + a_bytes;
      const int k0 = (kb0 + i) * BK;
      if (MODE == MODE_UP) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int kc = k0 + u * 8;
          const bool ok = a_row && kc < p.K;
          cp_async16(sa + sw128(t, u), ok ? (const void*)(a_row + kc) : (const void*)p.w, ok ? 16u : 0u);
        }
      } else {
        // A tile: 64 gathered K rows x 128 output features, MN-major SW128
        // atoms of 8 K x 64 MN; LBO (MN chunk) = 8192 B, SBO (8-K group) = 1024 B
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = t + j * kEpiThreads;
          const int kk = c >> 4, mu = c & 15;
          const int kg = k0 + kk;
          const int gm = m0 + mu * 8;
          const bool ok = kg < count && gm < p.M;
          const uint16_t* src = p.w;
          if (ok) src = p.w + (size_t)(p.idx ? p.idx[kg] : kg) * p.w_ld + gm;
          const uint32_t off = (uint32_t)((mu >> 3) * 8192 + (kk >> 3) * 1024 + (kk & 7) * 128 +
                                          (((mu & 7) ^ (kk & 7)) << 4));
          cp_async16(sa + off, src, ok ? 16u : 0u);
        }
      }
      // B tile: NB batch rows x 64 K, K-major SW128
      const int bchunks = NB * 8;
      for (int c = t; c < bchunks; c += kEpiThreads) {
        const int n = c >> 3, u = c & 7;
        const int gn = n0 + n, kc = k0 + u * 8;
        uint32_t bytes = 0;
        if (gn < p.N) {
          const int rem = klimit - kc;
          bytes = rem >= 8 ? 16u : (rem > 0 ? (uint32_t)rem * 2 : 0u);
        }
        const void* src = bytes ? (const void*)(p.x + (size_t)gn * p.x_ld + kc) : (const void*)p.x;
        cp_async16(sb + sw128(n, u), src, bytes);
      }
      cp_async_arrive_noinc(&full[s]);
    }
  } else {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
    const uint32_t idesc = make_idesc_bf16(BM, NB, MODE == MODE_DOWN ? 1 : 0, 0);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      fence_proxy_async();
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * stage_bytes);
      const uint32_t sb = sa + a_bytes;
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk) {
        uint64_t ad, bd;
        if (MODE == MODE_UP)
          ad = make_sdesc_sw128(sa + kk * 32, 16, 1024);
        else
          ad = make_sdesc_sw128(sa + kk * 2048, 8192, 1024);
        bd = make_sdesc_sw128(sb + kk * 32, 16, 1024);
        umma_bf16(tmem, ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
      }
      umma_commit(&empty[s]);
    }
    if (nkb > 0)
      umma_commit(accum);
    else
      mbar_arrive(accum);
    }
    __syncwarp();
  }

  if (warp < 4) {
    // ------------------------------------------------------------ epilogue
    mbar_wait(accum, 0);
    tc_fence_after();
    const int m = warp * 32 + lane;  // TMEM lane == tile row
    const int gm = m0 + m;
    const int nrows = min(NB, p.N - n0);
    const bool direct = p.splits == 1;
    float* part = p.partials +
                  ((size_t)(ntile * gridDim.x + mt) * p.splits + split) * (size_t)NB * BM;
    // per-row epilogue constants
    bool row_ok, row_live;
    float bias = 0.f;
    if (MODE == MODE_UP) {
      row_ok = gm < p.M;       // column exists in the output
      row_live = gm < count;   // selected neuron (else written as 0)
      if (row_live && p.bias) bias = p.bias[p.idx ? p.idx[gm] : gm];
    } else {
      row_ok = gm < p.M;
      row_live = row_ok;
      if (row_live && p.bias) bias = p.bias[gm];
    }
    for (int c0 = 0; c0 < NB; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = c0 + j;
        const float acc = nkb > 0 ? __uint_as_float(r[j]) : 0.f;
        if (direct) {
          if (n < nrows && row_ok) {
            float v = 0.f;
            if (row_live) {
              v = acc + bias;
              if (MODE == MODE_UP && p.act == PS_ACT_RELU) v = fmaxf(v, 0.f);
              if (p.residual) v += p.residual[(size_t)(n0 + n) * p.res_ld + gm];
            }
            const size_t o = (size_t)(n0 + n) * p.out_ld + gm;
            if (p.out_bf16)
              reinterpret_cast<uint16_t*>(p.out)[o] = f2bf(v);
            else
              reinterpret_cast<float*>(p.out)[o] = v;
          }
        } else {
          part[(size_t)n * BM + m] = acc;
        }
      }
    }
    if (!direct) {
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));
      if (tid == 0) {
        int* tk = p.tickets + ntile * gridDim.x + mt;
        const int prev = atomicAdd(tk, 1);
        *flag = prev == p.splits - 1;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));
      if (*flag) {
        __threadfence();
        const float* base = p.partials + ((size_t)(ntile * gridDim.x + mt) * p.splits) * (size_t)NB * BM;
        for (int n = 0; n < nrows; ++n) {
          float acc = 0.f;
          for (int s2 = 0; s2 < p.splits; ++s2) acc += __ldcg(base + ((size_t)s2 * NB + n) * BM + m);
          if (!row_ok) continue;
          float v = 0.f;
          if (row_live) {
            v = acc + bias;
            if (MODE == MODE_UP && p.act == PS_ACT_RELU) v = fmaxf(v, 0.f);
            if (p.residual) v += p.residual[(size_t)(n0 + n) * p.res_ld + gm];
          }
          const size_t o = (size_t)(n0 + n) * p.out_ld + gm;
          if (p.out_bf16)
            reinterpret_cast<uint16_t*>(p.out)[o] = f2bf(v);
          else
            reinterpret_cast<float*>(p.out)[o] = v;
        }
        if (tid == 0) p.tickets[ntile * gridDim.x + mt] = 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
}

int pick_nb(int N) {
  int nb = (N + 15) / 16 * 16;
  return nb > kMaxNB ? kMaxNB : nb;
}

int pick_stages(int NB) {
  const int stage = BM * BK * 2 + NB * BK * 2;
  const int budget = NB <= 128 ? 100 * 1024 : 200 * 1024;
  int s = budget / stage;
  if (s < 2) s = 2;
  if (s > 8) s = 8;
  return s;
}

size_t smem_bytes(int NB, int stages) {
  return 1024 + (size_t)stages * (BM * BK * 2 + NB * BK * 2) + (2 * stages + 1) * 8 + 16;
}

template <int MODE>
int launch(GGParams& prm, int m_tiles, int n_tiles, cudaStream_t st) {
  const size_t smem = smem_bytes(prm.NB, prm.stages);
  auto kern = gather_gemm_kernel<MODE>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      return PS_ERR_CUDA;
    configured = true;
  }
  dim3 grid(m_tiles, prm.splits, n_tiles);
  kern<<<grid, kThreads, smem, st>>>(prm);
  return launch_status();
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" size_t ps_gather_gemm_workspace_bytes(int N, int M, int K, int splits) {
  (void)K;
  if (N < 1 || M < 1) return 0;
  if (splits < 1) splits = 1;
  const int NB = pick_nb(N);
  const int n_tiles = (N + NB - 1) / NB;
  const int m_tiles = (M + BM - 1) / BM;
  return kTicketBytes + (size_t)n_tiles * m_tiles * splits * NB * BM * 4 +
         ((size_t)n_tiles * m_tiles * 4 > kTicketBytes ? (size_t)n_tiles * m_tiles * 4 : 0);
}

extern "C" int ps_gather_gemm_auto_splits(int N, int M, int K) {
  const int NB = pick_nb(N);
  const int tiles = ((N + NB - 1) / NB) * ((M + BM - 1) / BM);
  const int kbt = (K + BK - 1) / BK;
  const int target = 2 * ps_num_sms();
  int s = (target + tiles - 1) / tiles;
  int cap = kbt / 4;  // keep >= 4 K blocks per split
  if (cap < 1) cap = 1;
  if (s > cap) s = cap;
  if (s > 16) s = 16;
  return s < 1 ? 1 : s;
}

static int gg_common(GGParams& prm, const void* w_rows, const int32_t* idx, const int32_t* count_dev,
                     const void* x, int64_t x_ld, const float* bias, int N, int M, int K, int splits, void* out,
                     int64_t out_ld, int out_dtype, void* ws, size_t ws_bytes) {
  if (N < 1 || M < 1 || K < 1 || !w_rows || !x || !out || !ws) return PS_ERR_VALUE;
  if (splits < 1) return PS_ERR_VALUE;
  if (((uintptr_t)w_rows % 16) || ((uintptr_t)x % 16) || (x_ld % 8)) return PS_ERR_VALUE;
  prm.w = static_cast<const uint16_t*>(w_rows);
  prm.idx = idx;
  prm.count = count_dev;
  prm.x = static_cast<const uint16_t*>(x);
  prm.x_ld = x_ld;
  prm.bias = bias;
  prm.residual = nullptr;
  prm.res_ld = 0;
  prm.N = N;
  prm.M = M;
  prm.K = K;
  prm.act = PS_ACT_NONE;
  prm.splits = splits;
  prm.NB = pick_nb(N);
  prm.stages = pick_stages(prm.NB);
  prm.out = out;
  prm.out_ld = out_ld;
  prm.out_bf16 = out_dtype == PS_DTYPE_BF16;
  if (ws_bytes < ps_gather_gemm_workspace_bytes(N, M, K, splits)) return PS_ERR_WORKSPACE;
  prm.tickets = static_cast<int*>(ws);
  prm.partials = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kTicketBytes);
  return PS_OK;
}

extern "C" int ps_gather_gemm(const void* w_rows, const int32_t* idx, const int32_t* count_dev, const void* x,
                              int64_t x_ld, const float* bias, const float* residual, int64_t residual_ld, int N,
                              int M, int K, int act, int splits, void* out, int64_t out_ld, int out_dtype, void* ws,
                              size_t ws_bytes, void* stream) {
  if (K % 8 || x_ld < K || out_ld < M) return PS_ERR_VALUE;
  if (splits <= 0) splits = ps_gather_gemm_auto_splits(N, M, K);
  GGParams prm;
  int st = gg_common(prm, w_rows, idx, count_dev, x, x_ld, bias, N, M, K, splits, out, out_ld, out_dtype, ws,
                     ws_bytes);
  if (st != PS_OK) return st;
  prm.w_ld = K;
  prm.act = act;
  prm.residual = residual;
  prm.res_ld = residual_ld;
  const int m_tiles = (M + BM - 1) / BM;
  const int n_tiles = (N + prm.NB - 1) / prm.NB;
  if ((size_t)n_tiles * m_tiles * 4 > kTicketBytes) return PS_ERR_UNSUPPORTED;
  return launch<MODE_UP>(prm, m_tiles, n_tiles, static_cast<cudaStream_t>(stream));
}

extern "C" int ps_gather_gemm_t(const void* w_rows, const int32_t* idx, const int32_t* count_dev, const void* h,
                                int64_t h_ld, const float* bias, const float* residual, int64_t residual_ld, int N,
                                int M, int K_max, int splits, void* out, int64_t out_ld, int out_dtype, void* ws,
                                size_t ws_bytes, void* stream) {
  if (M % 8 || h_ld < K_max || out_ld < M) return PS_ERR_VALUE;
  if (splits <= 0) splits = ps_gather_gemm_auto_splits(N, M, K_max);
  GGParams prm;
  int st = gg_common(prm, w_rows, idx, count_dev, h, h_ld, bias, N, M, K_max, splits, out, out_ld, out_dtype, ws,
                     ws_bytes);
  if (st != PS_OK) return st;
  prm.w_ld = M;
  prm.residual = residual;
  prm.res_ld = residual_ld;
  const int m_tiles = (M + BM - 1) / BM;
  const int n_tiles = (N + prm.NB - 1) / prm.NB;
  if ((size_t)n_tiles * m_tiles * 4 > kTicketBytes) return PS_ERR_UNSUPPORTED;
  return launch<MODE_DOWN>(prm, m_tiles, n_tiles, static_cast<cudaStream_t>(stream));
}
