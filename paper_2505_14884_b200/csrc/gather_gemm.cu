// Gathered GEMMs on 5th-generation tensor cores (tcgen05 + TMEM), sm_100a.
//
// Polar Sparsity's selective MLP (Alg. 2, kernels.py:223-256 / 353-373)
// touches only the batch-union S of active neurons.  Weights are stored
// NEURON-MAJOR (W1^T, W2^T as (D, d) rows) so each selected neuron is one
// contiguous 2*d-byte row and both projections become row gathers:
//
//   rows form   (MODE_UP):   out[n, j] = act(sum_k W[idx[j], k] x[n, k] + b[idx[j]]) (+ res)
//   contraction (MODE_DOWN): out[n, m] = sum_j h[n, j] W[idx[j], m] + b[m] (+ res)
//
// Decode GEMMs are weight-streaming (batch N <= 256 << the ~250 flop/byte
// ridge), so the design goal is every SM streaming weights continuously:
//   * swap-AB: the UMMA M dimension (128) runs over the weight side (neurons
//     for UP, output features for DOWN), N over the batch (16..256);
//   * persistent stream-K: a fixed grid (SMs x 2) splits the total
//     (tile, 64-wide K block) iteration space evenly ON THE DEVICE, from the
//     device-resident union size (*count) -- no host sync, graph-capturable,
//     no idle waves whatever |S| is; CTAs sharing a tile add their partial
//     sums into an f32 tile accumulator with fire-and-forget global
//     reductions, and the last contributor (atomic ticket, self-resetting)
//     applies the epilogue and re-zeroes it -- no latency-serial fix-up on
//     the tail (summation order across CTAs is not fixed, so shared tiles are
//     reproducible to f32 rounding, not bitwise);
//   * warp roles: warp 0 drives the TMA engine (dense operands as 2-D tiled
//     boxes; gathered neuron rows with sm_100 `tile::gather4`, 4 rows per
//     instruction, 32 per stage), all landing 128B-swizzled (K-major rows for
//     UP; for DOWN the gathered rows are K slices stored MN-major, tcgen05
//     transposes via the instruction descriptor); warp 1 issues tcgen05.mma
//     from one thread into one of two TMEM accumulators; warps 2-5 drain the
//     other accumulator (tcgen05.ld 32x32b) and apply bias / ReLU / residual
//     / bf16-or-f32 store, so the epilogue of one tile overlaps the main loop
//     of the next.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace ps {
namespace {

constexpr int BM = 128;   // UMMA M
constexpr int BK = 64;    // K elements per stage (one 128-byte swizzle row)
constexpr int kEpiThreads = 128;
constexpr int kThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kMaxNB = 256;
constexpr int kTicketBytes = 65536;
constexpr int kMinItersPerCta = 4;
constexpr int kEpiCols = 64;  // batch rows staged per epilogue pass (32 KB of smem)
constexpr int kProdWarp = 0, kMmaWarp = 1, kEpiWarp0 = 2;

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
  int NB;       // batch rows per tile (multiple of 16, <= 256)
  int n_tiles;  // ceil(N / NB)
  int stages;
  void* out;
  int64_t out_ld;
  int out_bf16;
  int vec_ok;  // out / residual rows 16-byte aligned: vector epilogue stores
  int* tickets;
  float* partials;            // [tiles][NB][BM] f32 accumulators, zero between calls
  unsigned long long* trace;  // debug: per-CTA timestamps (ps_debug_gemm_trace), NULL normally
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Stream-K partition of T iterations over G CTAs.
struct Part {
  int64_t T;
  int G;
  PS_DEV int64_t lo(int c) const { return T * c / G; }
  // CTA whose range contains iteration `it`
  PS_DEV int owner(int64_t it) const {
    int c = (int)((it * G) / T);
    while (c + 1 < G && lo(c + 1) <= it) ++c;
    while (c > 0 && lo(c) > it) --c;
    return c;
  }
};

template <int MODE, bool GATHER>
__global__ void __launch_bounds__(kThreads, 1)
    gather_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const GGParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NB = p.NB;
  const uint32_t a_bytes = BM * BK * 2;            // 16 KB
  const uint32_t b_bytes = (uint32_t)NB * BK * 2;  // NB * 128
  const uint32_t stage_bytes = a_bytes + b_bytes;
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;  // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x;
  unsigned long long* tr = p.trace ? p.trace + 16 * (size_t)cta : nullptr;
  if (tr && tid == 0) {
    unsigned smid;
    asm("mov.u32 %0, %smid;" : "=r"(smid));
    tr[0] = gtimer();
    tr[7] = smid;
  }

  // ---- device-side work partition (identical in every role)
  const int count = p.count ? *p.count : (MODE == MODE_UP ? p.M : p.K);
  const int klimit = (MODE == MODE_UP) ? p.K : count;
  const int kbt = (klimit + BK - 1) / BK;
  const int live_m = (MODE == MODE_UP) ? (count + BM - 1) / BM : (p.M + BM - 1) / BM;
  const int tiles = live_m * p.n_tiles;
  if (tiles == 0) return;
  if (kbt == 0) {
    // DOWN with an empty union: out = bias (+ residual), one tile per CTA
    if (warp < kEpiWarp0) return;
    for (int t = cta; t < tiles; t += gridDim.x) {
      const int mt = t % live_m, nt = t / live_m;
      const int gm = mt * BM + (tid - kEpiWarp0 * 32);
      if (gm >= p.M) continue;
      for (int n = 0; n < NB && nt * NB + n < p.N; ++n) {
        const int gn = nt * NB + n;
        float v = p.bias ? p.bias[gm] : 0.f;
        if (p.residual) v += p.residual[(size_t)gn * p.res_ld + gm];
        const size_t o = (size_t)gn * p.out_ld + gm;
        if (p.out_bf16)
          reinterpret_cast<uint16_t*>(p.out)[o] = f2bf(v);
        else
          reinterpret_cast<float*>(p.out)[o] = v;
      }
    }
    return;
  }
  Part part;
  part.T = (int64_t)tiles * kbt;
  {
    int64_t g = part.T / kMinItersPerCta;
    if (g < 1) g = 1;
    if (g > (int64_t)gridDim.x) g = gridDim.x;
    part.G = (int)g;
  }
  if (cta >= part.G) return;
  const int64_t it_lo = part.lo(cta), it_hi = part.lo(cta + 1);
  if (it_lo >= it_hi) return;

  const uint32_t tcols = NB <= 16 ? 32 : (NB <= 32 ? 64 : (NB <= 64 ? 128 : (NB <= 128 ? 256 : 512)));
  if (warp == kMmaWarp) {
    if (lane == 0) {
      for (int s = 0; s < S; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], 4);  // one arrival per epilogue warp
      }
      fence_mbar_init();
    }
    __syncwarp();
    tmem_alloc(tmem_slot, tcols);
  } else if (warp == kProdWarp && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tr && tid == 0) tr[1] = gtimer();

  if (warp == kProdWarp) {
    // ------------------------------------------------------------ TMA producer
    // 4 gathered ids per lane and stage, loaded one stage ahead (int4) so
    // the TMA issue never waits on a dependent global load.
    auto load4 = [&](int base, int lim, int first) -> int4 {
      if (base + 4 <= lim) return __ldg(reinterpret_cast<const int4*>(p.idx + base));
      int r[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = base + j < lim ? __ldg(p.idx + base + j) : first;
      return make_int4(r[0], r[1], r[2], r[3]);
    };
    auto ids_for = [&](int64_t it) -> int4 {
      if (!GATHER) return make_int4(0, 0, 0, 0);
      const int t = (int)(it / kbt), kb = (int)(it - (int64_t)t * kbt);
      if (MODE == MODE_UP) {
        const int m0 = (t % live_m) * BM;
        return load4(m0 + lane * 4, count, __ldg(p.idx + m0));  // rows of the tile
      }
      return load4(kb * BK + 4 * (lane & 15), count, __ldg(p.idx));  // K rows of the stage
    };
    int i = 0;  // global stage counter
    int4 cur = ids_for(it_lo);
    for (int64_t it = it_lo; it < it_hi; ++it, ++i) {
      const int t = (int)(it / kbt), kb = (int)(it - (int64_t)t * kbt);
      const int mt = t % live_m, nt = t / live_m;
      const int m0 = mt * BM, n0 = nt * NB, k0 = kb * BK;
      const int4 nxt = (it + 1 < it_hi) ? ids_for(it + 1) : cur;
      const int s = i % S;
      if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
      uint8_t* sa = smem + s * stage_bytes;
      uint8_t* sb = sa + a_bytes;
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        tma_load_2d(sb, &tmB, k0, n0, &full[s]);  // B: NB batch rows x 64 K
      }
      if (GATHER) {
        if (MODE == MODE_UP) {
          tma_gather4(sa + lane * 512, &tmA, k0, cur.x, cur.y, cur.z, cur.w, &full[s]);
        } else {
          const int c = lane >> 4, j = lane & 15;
          tma_gather4(sa + c * 8192 + (j >> 1) * 1024 + (j & 1) * 512, &tmA, m0 + 64 * c, cur.x, cur.y, cur.z,
                      cur.w, &full[s]);
        }
      } else if (lane == 0) {
        if (MODE == MODE_UP) {
          tma_load_2d(sa, &tmA, k0, m0, &full[s]);  // 128 rows x 64 K
        } else {
          tma_load_2d(sa, &tmA, m0, k0, &full[s]);  // 64 K rows x 64 MN, two MN chunks
          tma_load_2d(sa + 8192, &tmA, m0 + 64, k0, &full[s]);
        }
      }
      cur = nxt;
      __syncwarp();
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = make_idesc_bf16(BM, NB, MODE == MODE_DOWN ? 1 : 0, 0);
      int i = 0, seg = 0;
      int64_t it = it_lo;
      while (it < it_hi) {
        const int t = (int)(it / kbt);
        const int64_t seg_end = min(it_hi, (int64_t)(t + 1) * kbt);
        const int a = seg & 1;
        if (seg >= 2) mbar_wait(&tempty[a], ((seg >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + a * NB;
        for (int64_t j = it; j < seg_end; ++j, ++i) {
          const int s = i % S;
          mbar_wait(&full[s], (i / S) & 1);
          if (tr && i == 0) tr[2] = gtimer();
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
            umma_bf16(acc, ad, bd, idesc, (j > it || kk > 0) ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[a]);
        it = seg_end;
        ++seg;
      }
      if (tr) tr[3] = gtimer();
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    // TMEM -> registers -> smem staging tile S[n][m] (f32) -> 16-byte vector
    // stores / reductions along m, 4 output columns per operation.
    const int q = warp & 3;               // TMEM lane quadrant of this warp
    const int m = q * 32 + lane;          // tile row (TMEM lane)
    const int et = tid - kEpiWarp0 * 32;  // 0..127
    float* stg = reinterpret_cast<float*>(smem + S * stage_bytes + 256);  // [kEpiCols][BM]
    int seg = 0;
    int64_t it = it_lo;
    while (it < it_hi) {
      const int t = (int)(it / kbt);
      const int64_t t_lo = (int64_t)t * kbt, t_hi = t_lo + kbt;
      const int64_t seg_end = min(it_hi, t_hi);
      const int a = seg & 1;
      const int mt = t % live_m, nt = t / live_m;
      const int m0 = mt * BM, n0 = nt * NB;
      const int nrows = min(NB, p.N - n0);
      // contributors of tile t: CTAs owning t_lo .. t_hi-1
      const int c_first = (it == t_lo) ? cta : part.owner(t_lo);
      const int c_last = (seg_end == t_hi) ? cta : part.owner(t_hi - 1);
      const bool direct = c_first == c_last;
      // shared tiles: contributors add partial sums into the tile's f32
      // accumulator with vector reductions; the last to arrive applies the
      // epilogue and re-zeroes the accumulator for the next call
      float* tacc = p.partials + (size_t)t * NB * BM;

      // epilogue for 4 consecutive output columns gm0..gm0+3 of batch row n
      auto finish4 = [&](int n, int mc, float4 v) {
        const int gm0 = m0 + mc;
        const size_t o = (size_t)(n0 + n) * p.out_ld + gm0;
        float vv[4] = {v.x, v.y, v.z, v.w};
        float res[4] = {0.f, 0.f, 0.f, 0.f};
        if (p.residual) {
          if (p.vec_ok && gm0 + 4 <= p.M) {
            const float4 r4 = *reinterpret_cast<const float4*>(p.residual + (size_t)(n0 + n) * p.res_ld + gm0);
            res[0] = r4.x; res[1] = r4.y; res[2] = r4.z; res[3] = r4.w;
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (gm0 + j < p.M) res[j] = p.residual[(size_t)(n0 + n) * p.res_ld + gm0 + j];
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int gm = gm0 + j;
          const bool live = (MODE == MODE_UP) ? gm < count : gm < p.M;
          float x = 0.f;
          if (live) {
            float bias = 0.f;
            if (p.bias) bias = __ldg(p.bias + ((MODE == MODE_UP && p.idx) ? __ldg(p.idx + gm) : gm));
            x = vv[j] + bias;
            if (MODE == MODE_UP && p.act == PS_ACT_RELU) x = fmaxf(x, 0.f);
            x += res[j];
          }
          vv[j] = x;
        }
        if (p.vec_ok && gm0 + 4 <= p.M) {
          if (p.out_bf16) {
            uint2 pk;
            pk.x = pack_bf16x2(vv[0], vv[1]);
            pk.y = pack_bf16x2(vv[2], vv[3]);
            *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(p.out) + o) = pk;
          } else {
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + o) = make_float4(vv[0], vv[1], vv[2], vv[3]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (gm0 + j >= p.M) break;
            if (p.out_bf16)
              reinterpret_cast<uint16_t*>(p.out)[o + j] = f2bf(vv[j]);
            else
              reinterpret_cast<float*>(p.out)[o + j] = vv[j];
          }
        }
      };

      mbar_wait(&tfull[a], (seg >> 1) & 1);
      if (tr && et == 0 && seg == 0) tr[8] = gtimer();
      tc_fence_after();
      for (int cb = 0; cb < NB; cb += kEpiCols) {
        const int ncb = min(kEpiCols, NB - cb);
        for (int c0 = 0; c0 < ncb; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(tmem + a * NB + ((uint32_t)(q * 32) << 16) + cb + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) stg[(c0 + j) * BM + m] = __uint_as_float(r[j]);
        }
        if (cb + kEpiCols >= NB) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[a]);  // accumulator free for the MMA warp
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));
        const int rows_here = min(ncb, nrows - cb);
        for (int v = et; v < rows_here * (BM / 4); v += kEpiThreads) {
          const int n = v / (BM / 4), mc = (v % (BM / 4)) * 4;
          const float4 val = *reinterpret_cast<const float4*>(stg + n * BM + mc);
          if (direct)
            finish4(cb + n, mc, val);
          else
            red_add_v4(tacc + (size_t)(cb + n) * BM + mc, val);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));
      }
      if (tr && et == 0 && seg == 0) tr[9] = gtimer();

      if (!direct) {
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));
        if (et == 0) {
          const int prev = atomicAdd(p.tickets + t, 1);
          *flag = prev == (c_last - c_first);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));
        const bool last = *flag;
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));
        if (last) {
          __threadfence();
          const int nv = nrows * (BM / 4);
          for (int v0 = et; v0 < nv; v0 += 4 * kEpiThreads) {
            float4 val[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int v = v0 + u * kEpiThreads;
              val[u] = v < nv ? __ldcg(reinterpret_cast<const float4*>(tacc) + v) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int v = v0 + u * kEpiThreads;
              if (v < nv) {
                finish4(v / (BM / 4), (v % (BM / 4)) * 4, val[u]);
                __stcg(reinterpret_cast<float4*>(tacc) + v, make_float4(0.f, 0.f, 0.f, 0.f));
              }
            }
          }
          if (et == 0) p.tickets[t] = 0;
        }
      }
      if (tr && et == 0 && seg == 0) tr[10] = gtimer();
      it = seg_end;
      ++seg;
    }
    if (tr && et == 0) tr[4] = gtimer();
  }
  tc_fence_before();
  __syncthreads();
  if (tr && tid == 0) {
    tr[5] = gtimer();
    tr[6] = it_hi - it_lo;
  }
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
}

int pick_nb(int N) {
  int nb = (N + 15) / 16 * 16;
  return nb > kMaxNB ? kMaxNB : nb;
}

unsigned long long* g_trace = nullptr;
int g_stages_override = 0, g_target_override = 0;

int ctas_per_sm(int NB) { return NB <= 128 ? 2 : 1; }

int pick_stages(int NB) {
  if (g_stages_override > 0) return g_stages_override;
  const int stage = BM * BK * 2 + NB * BK * 2;
  const int budget = (ctas_per_sm(NB) == 2 ? 108 : 216) * 1024 - kEpiCols * BM * 4;
  int s = budget / stage;
  if (s < 2) s = 2;
  if (s > 12) s = 12;
  return s;
}

size_t smem_bytes(int NB, int stages) {
  return 1024 + (size_t)stages * (BM * BK * 2 + NB * BK * 2) + 256 + (size_t)kEpiCols * BM * 4;
}

int grid_ctas(int NB) { return g_target_override > 0 ? g_target_override : ps_num_sms() * ctas_per_sm(NB); }

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int get_encode() {
  if (g_encode) return PS_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
    return PS_ERR_CUDA;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return PS_OK;
}

// bf16 row-major (rows, cols) matrix, row stride ld elements, SW128 boxes
int make_map(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_cols,
             uint32_t box_rows) {
  if (get_encode() != PS_OK) return PS_ERR_CUDA;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? PS_OK : PS_ERR_VALUE;
}

template <int MODE, bool GATHER>
int launch_t(const CUtensorMap& ta, const CUtensorMap& tb, GGParams& prm, cudaStream_t st) {
  const size_t smem = smem_bytes(prm.NB, prm.stages);
  auto kern = gather_gemm_kernel<MODE, GATHER>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      return PS_ERR_CUDA;
    configured = true;
  }
  kern<<<grid_ctas(prm.NB), kThreads, smem, st>>>(ta, tb, prm);
  return launch_status();
}

// w_rows: (w_rows_n, w_cols) row-major; B operand x: (N, kx) with row stride x_ld
template <int MODE>
int launch(GGParams& prm, int64_t w_rows_n, int64_t w_cols, int64_t kx, cudaStream_t st) {
  CUtensorMap ta, tb;
  int rc = make_map(&tb, prm.x, (uint64_t)kx, (uint64_t)prm.N, (uint64_t)prm.x_ld, BK, prm.NB);
  if (rc != PS_OK) return rc;
  const bool gather = prm.idx != nullptr;
  if (MODE == MODE_UP)
    rc = make_map(&ta, prm.w, (uint64_t)w_cols, (uint64_t)w_rows_n, (uint64_t)prm.w_ld, BK, gather ? 1 : BM);
  else
    rc = make_map(&ta, prm.w, (uint64_t)w_cols, (uint64_t)w_rows_n, (uint64_t)prm.w_ld, 64, gather ? 1 : BK);
  if (rc != PS_OK) return rc;
  return gather ? launch_t<MODE, true>(ta, tb, prm, st) : launch_t<MODE, false>(ta, tb, prm, st);
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" size_t ps_gather_gemm_workspace_bytes(int N, int M, int K, int splits) {
  (void)K;
  (void)splits;
  if (N < 1 || M < 1) return 0;
  const int NB = pick_nb(N);
  const size_t tiles = (size_t)((M + BM - 1) / BM) * ((N + NB - 1) / NB);
  return kTicketBytes + tiles * NB * BM * 4;
}

// Kept for ABI compatibility: the persistent stream-K kernel partitions the
// work on the device, so the split count is always chosen there.
extern "C" int ps_gather_gemm_auto_splits(int N, int M, int K) {
  (void)N; (void)M; (void)K;
  return 1;
}

static int gg_common(GGParams& prm, const void* w_rows, const int32_t* idx, const int32_t* count_dev,
                     const void* x, int64_t x_ld, const float* bias, int N, int M, int K, void* out, int64_t out_ld,
                     int out_dtype, void* ws, size_t ws_bytes) {
  if (N < 1 || M < 1 || K < 1 || !w_rows || !x || !out || !ws) return PS_ERR_VALUE;
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
  prm.NB = pick_nb(N);
  prm.n_tiles = (N + prm.NB - 1) / prm.NB;
  prm.stages = pick_stages(prm.NB);
  prm.trace = g_trace;
  prm.out = out;
  prm.out_ld = out_ld;
  prm.out_bf16 = out_dtype == PS_DTYPE_BF16;
  prm.vec_ok = (out_ld % 4 == 0) && ((uintptr_t)out % 16 == 0);
  if (ws_bytes < ps_gather_gemm_workspace_bytes(N, M, K, 1)) return PS_ERR_WORKSPACE;
  prm.tickets = static_cast<int*>(ws);
  prm.partials = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kTicketBytes);
  return PS_OK;
}

extern "C" int ps_gather_gemm(const void* w_rows, int w_height, const int32_t* idx, const int32_t* count_dev,
                              const void* x, int64_t x_ld, const float* bias, const float* residual,
                              int64_t residual_ld, int N, int M, int K, int act, int splits, void* out, int64_t out_ld,
                              int out_dtype, void* ws, size_t ws_bytes, void* stream) {
  (void)splits;
  if (K % 8 || x_ld < K || out_ld < M) return PS_ERR_VALUE;
  GGParams prm;
  int st = gg_common(prm, w_rows, idx, count_dev, x, x_ld, bias, N, M, K, out, out_ld, out_dtype, ws, ws_bytes);
  if (st != PS_OK) return st;
  prm.w_ld = K;
  prm.act = act;
  prm.residual = residual;
  prm.res_ld = residual_ld;
  if (residual && ((residual_ld % 4) || ((uintptr_t)residual % 16))) prm.vec_ok = 0;
  if ((size_t)((M + BM - 1) / BM) * prm.n_tiles * 4 > kTicketBytes) return PS_ERR_UNSUPPORTED;
  if (w_height < (idx ? 1 : M)) return PS_ERR_VALUE;
  return launch<MODE_UP>(prm, w_height, K, K, static_cast<cudaStream_t>(stream));
}

extern "C" int ps_gather_gemm_t(const void* w_rows, int w_height, const int32_t* idx, const int32_t* count_dev,
                                const void* h, int64_t h_ld, const float* bias, const float* residual,
                                int64_t residual_ld, int N, int M, int K_max, int splits, void* out, int64_t out_ld,
                                int out_dtype, void* ws, size_t ws_bytes, void* stream) {
  (void)splits;
  if (M % 8 || h_ld < K_max || out_ld < M) return PS_ERR_VALUE;
  GGParams prm;
  int st = gg_common(prm, w_rows, idx, count_dev, h, h_ld, bias, N, M, K_max, out, out_ld, out_dtype, ws, ws_bytes);
  if (st != PS_OK) return st;
  prm.w_ld = M;
  prm.residual = residual;
  prm.res_ld = residual_ld;
  if (residual && ((residual_ld % 4) || ((uintptr_t)residual % 16))) prm.vec_ok = 0;
  if ((size_t)((M + BM - 1) / BM) * prm.n_tiles * 4 > kTicketBytes) return PS_ERR_UNSUPPORTED;
  if (w_height < (idx ? 1 : K_max)) return PS_ERR_VALUE;
  return launch<MODE_DOWN>(prm, w_height, M, K_max, static_cast<cudaStream_t>(stream));
}

// Debug hooks (tools/kbench.py): trace buffer of 16 u64 per CTA (start, setup
// done, first stage landed, last MMA issued, epilogue done, end, iterations,
// smid, first accumulator ready, first drained, first segment finished), and overrides of the pipeline depth / persistent grid (0 = default).
extern "C" void ps_debug_gemm_trace(void* buf, int stages, int target_ctas) {
  g_trace = static_cast<unsigned long long*>(buf);
  g_stages_override = stages;
  g_target_override = target_ctas;
}
