// Two chained gathered GEMMs in ONE persistent stream-K launch (sm_100a,
// tcgen05 + TMEM).  Serves the selective MLP (Polar Sparsity Alg. 2,
// kernels.py:353-373: UP over the union rows of W1^T, ReLU, DOWN over the
// same union rows of W2^T) and the two-layer router MLP (routers.py:286-288:
// W_in^T rows, ReLU, W_out^T rows).
//
//   phase 0 ("rows" form):        y0[n, j] = act0(sum_k W0[id0(j), k] x[n, k] + b0[id0(j)])   j < ext0
//   phase 1 ("rows" form):        y1[n, j] = act1(sum_k W1[id1(j), k] y0[n, k] + b1[id1(j)])
//        or ("contraction" form): y1[n, m] = sum_{j < ext} y0[n, j] W1[id(j), m] + b1[m] (+ res[n, m])
//
// Why one launch: at decode batch sizes both phases stream weights (HBM
// bound), and the two-launch version paid a launch prologue, a split-K
// cluster epilogue and an UP->DOWN residency gap per phase (~25 us of fixed
// cost on ~17 us of streaming at B = 64).  Here:
//   * grid = one CTA per SM (216 KB of pipeline stages, so never two), every
//     CTA co-resident: the kernel's own cross-CTA waits are safe;
//   * each phase's (tile, K-block) units are split into equal CONTIGUOUS
//     ranges per CTA (stream-K): perfect balance whatever the union size;
//     a tile cut between CTAs is reduced by its last-arriving piece (an
//     acq_rel ticket; partials in a global f32 workspace, summed in piece
//     order so results are deterministic); tickets self-reset;
//   * phase-1 K-block kb needs phase-0 tile kb/2 only: the finisher of a
//     phase-0 tile publishes it with a release flag (= launch epoch + 1), and
//     the B-operand producer acquires it before its TMA load -- no grid
//     barrier; the A loaders keep streaming phase-1 weight rows meanwhile, so
//     the phase switch costs no HBM idle time;
//   * warp roles as in gather_gemm.cu: warp 0 TMA (B operand), warp 1
//     tcgen05.mma issuer, warps 2-5 TMEM epilogue, warps 6-9 cp.async (LDGSTS)
//     gather of the A operand (weight rows) into 128B-swizzled stages.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"

namespace ps {
namespace {

constexpr int CBM = 128;  // UMMA M (weight rows / output features per tile)
constexpr int CBK = 64;   // K elements per stage
constexpr int kCThreads = 320;
constexpr int kCMaxNB = 256;
constexpr int kCLd0 = 6;  // first A-loader warp
constexpr int kCLdThreads = 128;

enum { FORM_ROWS = 0, FORM_CONTRACT = 1 };

struct ChainPhase {
  const uint16_t* w;  // weight rows, row stride w_ld elements
  int64_t w_ld;
  const int32_t* idx;  // gather ids (NULL: identity)
  int form;
  int M;          // rows: max output columns; contraction: output features
  int K;          // rows: contraction length; contraction: max K (union bound)
  int use_count;  // extent from *count (rows: output columns; contraction: K)
  const float* bias;
  int act;
  const float* residual;
  int64_t res_ld;
  void* out;
  int64_t out_ld;
  int out_bf16;
  int out_cols;  // rows form: columns [ext, out_cols) are written as 0
  int whole;       // one whole tile per CTA (T <= grid): no split pieces
  int accumulate;  // phase 1: every piece adds into the pre-initialised f32 output (red.add)
};

struct ChainParams {
  ChainPhase ph[2];
  const int32_t* count;
  int N, NB, stages;
  float* acc0;     // phase-0 split-tile sums [cols][NB] f32, zero between launches (the finisher re-zeroes)
  uint32_t* sync;  // [0] epoch, [1] exit count, then per tile t: [2+3t] phase-0 flag, [3+3t] / [4+3t] tickets
                   // (a fixed per-tile layout: a workspace reused at another shape keeps its meaning)
  int maxT;
  unsigned long long* trace;  // debug: 16 timestamps per CTA (ps_debug_chain_trace), NULL normally
  int gate;  // debug: phase-1 weight loads wait for the first phase-0 flag they need
  int dbg;   // debug experiments (0 = normal)
};

struct Geo {
  int T, KB, ext, Ge;  // Ge: CTAs that get units (min(G, U): every one of them gets >= 1)
  int U, s, e;         // units (tile-major (tile, K block)) and this CTA's range [s, e)
  int t0, kb0;         // (tile, K block) of unit s: the role loops walk incremental cursors
};                     // (no per-unit integer division on the streaming path)

PS_DEV Geo geo_of(const ChainPhase& ph, int count, int G, int bid) {
  Geo g;
  if (ph.form == FORM_ROWS) {
    g.ext = ph.use_count ? min(count, ph.M) : ph.M;
    g.T = (g.ext + CBM - 1) / CBM;
    g.KB = (ph.K + CBK - 1) / CBK;
  } else {
    g.ext = ph.use_count ? min(count, ph.K) : ph.K;
    g.T = (ph.M + CBM - 1) / CBM;
    g.KB = (g.ext + CBK - 1) / CBK;
  }
  g.U = g.T * g.KB;
  if (ph.whole) {  // contiguous ranges of WHOLE tiles per CTA: never a split tile
    g.Ge = g.T < G ? g.T : G;
    const int ts = bid < g.Ge ? (int)((long long)bid * g.T / g.Ge) : g.T;
    const int te = bid < g.Ge ? (int)((long long)(bid + 1) * g.T / g.Ge) : g.T;
    g.s = ts * g.KB;
    g.e = te * g.KB;
    g.t0 = ts;
    g.kb0 = 0;
    return g;
  }
  g.Ge = g.U < G ? g.U : G;
  g.s = bid < g.Ge ? (int)((long long)bid * g.U / g.Ge) : g.U;
  g.e = bid < g.Ge ? (int)((long long)(bid + 1) * g.U / g.Ge) : g.U;
  g.t0 = g.KB ? g.s / g.KB : 0;
  g.kb0 = g.KB ? g.s - g.t0 * g.KB : 0;
  return g;
}

// CTA owning unit u: largest c with floor(c*U/Ge) <= u (Ge <= U: no CTA below Ge has an empty range)
PS_DEV int owner_of(int u, int U, int Ge) { return (int)(((long long)(u + 1) * Ge - 1) / U); }

// (tile, K block) cursor over a tile-major unit range
struct Cur {
  int t, kb;
  PS_DEV void next(int KB) {
    if (++kb == KB) {
      kb = 0;
      ++t;
    }
  }
};

PS_DEV uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PS_DEV void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
PS_DEV uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
  uint32_t o;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
  return o;
}
PS_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

PS_DEV uint32_t csw128(int row, int unit) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((unit ^ (row & 7)) << 4));
}

__global__ void __launch_bounds__(kCThreads, 1)
    chain_gemm_kernel(const __grid_constant__ CUtensorMap tmB0, const __grid_constant__ CUtensorMap tmB1,
                      const ChainParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NB = p.NB;
  const uint32_t a_bytes = CBM * CBK * 2;
  const uint32_t b_bytes = (uint32_t)NB * CBK * 2;
  const uint32_t stage_bytes = a_bytes + b_bytes;
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  volatile int* s_last = reinterpret_cast<volatile int*>(tmem_slot + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = (int)gridDim.x, bid = (int)blockIdx.x;
  unsigned long long* tr = p.trace ? p.trace + 16 * (size_t)blockIdx.x : nullptr;
  auto stamp = [&](int i) {
    if (tr) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tr[i] = t;
    }
  };
  if (tid == 0) stamp(0);
  const uint32_t tcols = NB <= 16 ? 32 : (NB <= 32 ? 64 : (NB <= 64 ? 128 : (NB <= 128 ? 256 : 512)));

  // ---- prologue (input independent): barriers, TMEM, tensor maps
  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < S; ++s) {
        mbar_init(&full[s], 1 + kCLdThreads);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], 4);
      }
      fence_mbar_init();
    }
    __syncwarp();
    tmem_alloc(tmem_slot, tcols);
  } else if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmB0);
    prefetch_tmap(&tmB1);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  griddep_wait();  // ids / count / x come from the preceding launches
  if (tid == 0) griddep_launch();
  const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(p.sync);
  const int count = p.count ? *reinterpret_cast<const volatile int32_t*>(p.count) : 0;
  if (tid == 0) stamp(1);
  uint32_t* tiles = p.sync + 2;  // [t][0] flag, [t][1 + ph] ticket

  if (warp == 0) {
    // ------------------------------------------------------------ B operand (TMA)
    if (lane == 0) {
      int it = 0;
      for (int ph = 0; ph < 2; ++ph) {
        const Geo g = geo_of(p.ph[ph], count, G, bid);
        int ready_tile = -1;
        Cur c{g.t0, g.kb0};
        for (int u = g.s; u < g.e; ++u, ++it, c.next(g.KB)) {
          const int kb = c.kb;
          const int s = it % S;
          if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
          if (ph == 1 && (kb >> 1) != ready_tile) {
            if (ready_tile < 0) stamp(4);
            ready_tile = kb >> 1;
            const uint32_t* f = tiles + 3 * ready_tile;
            // bounded spin: a missing producer traps (a launch error) instead of hanging the GPU
            for (uint32_t spin = 0; ld_acquire_u32(f) != epoch + 1u; ++spin) {
              if (spin > (1u << 26)) __trap();
              __nanosleep(32);
            }
            if (tr && tr[5] == 0) stamp(5);
            fence_proxy_async_global();  // generic-proxy stores of y0 -> async-proxy (TMA) reads
          }
          uint8_t* sb = smem + s * stage_bytes + a_bytes;
          mbar_arrive_expect_tx(&full[s], b_bytes);
          tma_load_2d(sb, ph == 0 ? &tmB0 : &tmB1, kb * CBK, 0, &full[s]);
          if (it == 0) stamp(15);
        }
      }
    }
  } else if (warp >= kCLd0) {
    // ------------------------------------------------------------ A operand (weight rows, cp.async)
    const int lt = tid - kCLd0 * 32;
    int it = 0;
    for (int ph = 0; ph < 2; ++ph) {
      const ChainPhase& P = p.ph[ph];
      const Geo g = geo_of(P, count, G, bid);
      // the gather ids of unit u (8 per thread) are loaded 4 units ahead: an
      // id load is an L2 round trip (~0.5-1 us) against ~0.4 us per stage
      auto ids_of = [&](const Cur& c, bool live, int* o) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int pos = P.form == FORM_ROWS ? c.t * CBM + (lt >> 3) + 16 * r : c.kb * CBK + (lt >> 4) + 8 * r;
          o[r] = (live && pos < g.ext) ? (P.idx ? __ldg(P.idx + pos) : pos) : -1;
        }
      };
      const bool rows = P.form == FORM_ROWS;
      int i0[8], i1[8], i2[8], i3[8];
      Cur c{g.t0, g.kb0}, c4{g.t0, g.kb0};  // c4: the unit 4 ahead (its ids are being fetched)
      ids_of(c4, g.s < g.e, i0);
      c4.next(g.KB);
      ids_of(c4, g.s + 1 < g.e, i1);
      c4.next(g.KB);
      ids_of(c4, g.s + 2 < g.e, i2);
      c4.next(g.KB);
      ids_of(c4, g.s + 3 < g.e, i3);
      c4.next(g.KB);
      if (ph == 1 && p.gate && g.s < g.e) {
        const uint32_t* f = tiles + 3 * (g.kb0 >> 1);
        while (ld_acquire_u32(f) != epoch + 1u) __nanosleep(64);
      }
      for (int u = g.s; u < g.e; ++u, ++it, c.next(g.KB), c4.next(g.KB)) {
        const int t = c.t, kb = c.kb;
        int nx[8];
        // rows form: the ids change only with the tile
        if (rows && c4.kb != 0) {
#pragma unroll
          for (int r = 0; r < 8; ++r) nx[r] = i3[r];
        } else {
          ids_of(c4, u + 4 < g.e, nx);
        }
        const int s = it % S;
        if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
        uint8_t* sa = smem + s * stage_bytes;
        if (P.form == FORM_ROWS) {
          const int uu = lt & 7;
          const int k0 = kb * CBK + uu * 8;
          const bool kok = k0 < P.K;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const int row = (lt >> 3) + 16 * r;
            const bool ok = kok && i0[r] >= 0;
            cp_async16_l2_256(sa + csw128(row, uu), ok ? (const void*)(P.w + (size_t)i0[r] * P.w_ld + k0)
                                                       : (const void*)P.w, ok ? 16u : 0u);
          }
        } else {
          // 64 K rows x 128 output features, MN-major SW128 atoms (8 K x 64 MN)
          const int mu = lt & 15;
          const int gm = t * CBM + mu * 8;
          const bool mok = gm < P.M;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const int kk = (lt >> 4) + 8 * r;
            const bool ok = mok && i0[r] >= 0;
            const void* sp = ok ? (const void*)(P.w + (size_t)i0[r] * P.w_ld + gm) : (const void*)P.w;
            const uint32_t off = (uint32_t)((mu >> 3) * 8192 + (kk >> 3) * 1024 + (kk & 7) * 128 +
                                            (((mu & 7) ^ (kk & 7)) << 4));
            cp_async16_l2_256(sa + off, sp, ok ? 16u : 0u);
          }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          i0[r] = i1[r];
          i1[r] = i2[r];
          i2[r] = i3[r];
          i3[r] = nx[r];
        }
        cp_async_arrive_noinc(&full[s]);
        if (it == 0 && lt == 0 && tr) stamp(14);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int it = 0, j = 0;
      for (int ph = 0; ph < 2; ++ph) {
        const Geo g = geo_of(p.ph[ph], count, G, bid);
        const bool mn = p.ph[ph].form == FORM_CONTRACT;
        const uint32_t idesc = make_idesc_bf16(CBM, NB, mn ? 1 : 0, 0);
        uint32_t acc = 0;
        bool first = true;
        Cur c{g.t0, g.kb0};
        for (int u = g.s; u < g.e; ++u, ++it, c.next(g.KB)) {
          const int kb = c.kb;
          if (u == g.s || kb == 0) {
            const int a = j & 1;
            if (j >= 2) mbar_wait(&tempty[a], ((j >> 1) - 1) & 1);
            tc_fence_after();
            acc = tmem + a * NB;
            first = true;
          }
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          if (it == 0) stamp(2);
          fence_proxy_async();  // cp.async (generic proxy) stage writes -> tcgen05 reads
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * stage_bytes);
          const uint32_t sb = sa + a_bytes;
#pragma unroll
          for (int kk = 0; kk < CBK / 16; ++kk) {
            const uint64_t ad = mn ? make_sdesc_sw128(sa + kk * 2048, 8192, 1024) : make_sdesc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t bd = make_sdesc_sw128(sb + kk * 32, 16, 1024);
            umma_bf16(acc, ad, bd, idesc, (!first || kk > 0) ? 1u : 0u);
          }
          first = false;
          umma_commit(&empty[s]);
          if (u == g.e - 1 || kb == g.KB - 1) {
            umma_commit(&tfull[j & 1]);
            if (ph == 0) stamp(3);
            ++j;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;
    const int m = q * 32 + lane;  // tile row = TMEM lane
    const int et = tid - 64;      // 0..127
    int j = 0;
    for (int ph = 0; ph < 2; ++ph) {
      const ChainPhase& P = p.ph[ph];
      const Geo g = geo_of(P, count, G, bid);
      if (ph == 1 && g.KB == 0) {
        // empty contraction (no active unit): y1 = bias (+ residual); tiles split over the CTAs
        for (int t = bid; t < g.T; t += G) {
          const int col = t * CBM + m;
          if (col >= P.M) continue;
          const float b = P.bias ? __ldg(P.bias + col) : 0.f;
          for (int n = 0; n < p.N; ++n) {
            if (P.accumulate) {
              reinterpret_cast<float*>(P.out)[(size_t)n * P.out_ld + col] += b;
              continue;
            }
            float v = b;
            if (P.residual) v += P.residual[(size_t)n * P.res_ld + col];
            if (P.out_bf16) reinterpret_cast<uint16_t*>(P.out)[(size_t)n * P.out_ld + col] = f2bf(v);
            else reinterpret_cast<float*>(P.out)[(size_t)n * P.out_ld + col] = v;
          }
        }
        continue;
      }
      int u = g.s;
      while (u < g.e) {
        const int t = u / g.KB;  // once per piece
        const int t0 = t * g.KB, t1 = t0 + g.KB;  // units of tile t
        const bool has_k0 = u == t0;              // this piece holds the tile's first K block
        u = g.e < t1 ? g.e : t1;
        const int np = P.whole ? 1 : owner_of(t1 - 1, g.U, g.Ge) - owner_of(t0, g.U, g.Ge) + 1;
        const int a = j & 1;
        const uint32_t acc = tmem + a * NB + ((uint32_t)(q * 32) << 16);
        mbar_wait(&tfull[a], (j >> 1) & 1);
        const int tb = (ph == 0 && j == 0) ? 9 : -1;  // trace slots of the first two phase-0 pieces
        if (et == 0 && tb >= 0 && j < 2) stamp(tb);
        tc_fence_after();
        const int col = t * CBM + m;
        const bool live = P.form == FORM_ROWS ? col < g.ext : col < P.M;
        float bias_v = 0.f;
        if (live && P.bias) bias_v = __ldg(P.bias + ((P.form == FORM_ROWS && P.idx) ? __ldg(P.idx + col) : col));
        auto release_acc = [&]() {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[a]);  // accumulator free for the MMA warp
        };
        auto store_out = [&](int n, float v) {  // bias / act / residual, then the output element
          float x = 0.f;
          if (live) {
            x = v + bias_v;
            if (P.act == PS_ACT_RELU) x = fmaxf(x, 0.f);
            if (P.residual) x += P.residual[(size_t)n * P.res_ld + col];
          }
          if (P.out_bf16) reinterpret_cast<uint16_t*>(P.out)[(size_t)n * P.out_ld + col] = f2bf(x);
          else reinterpret_cast<float*>(P.out)[(size_t)n * P.out_ld + col] = x;
        };
        const bool write = P.form == FORM_ROWS ? col < P.out_cols : live;
        bool finish = false;
        if (ph == 1 && P.accumulate) {
          // split contraction: every piece adds its partial into the (pre-initialised)
          // output; the piece holding K block 0 adds the bias
          float* o = reinterpret_cast<float*>(P.out) + col;
          const float bv = has_k0 ? bias_v : 0.f;
          for (int c0 = 0; c0 < NB; c0 += 16) {
            uint32_t r[16];
            tmem_ld16(acc + c0, r);
            tmem_ld_wait();
            if (live) {
#pragma unroll
              for (int uu = 0; uu < 16; ++uu)
                if (c0 + uu < p.N) red_add_f32(o + (size_t)(c0 + uu) * P.out_ld, __uint_as_float(r[uu]) + bv);
            }
          }
          release_acc();
        } else if (np == 1) {
          // the whole tile in this CTA: straight from TMEM
          for (int c0 = 0; c0 < NB; c0 += 16) {
            uint32_t r[16];
            tmem_ld16(acc + c0, r);
            tmem_ld_wait();
            if (write) {
#pragma unroll
              for (int uu = 0; uu < 16; ++uu)
                if (c0 + uu < p.N) store_out(c0 + uu, __uint_as_float(r[uu]));
            }
          }
          release_acc();
          finish = true;
        } else {
          // split tile (phase 0): f32 partial added into the tile's accumulator
          // block acc0[col][n] (fire-and-forget reductions), then the tile's ticket;
          // the last piece reads the sums back (one round trip, every load in
          // flight), re-zeroes the block and writes the activations
          float* blk = p.acc0 + (size_t)col * NB;
          for (int c0 = 0; c0 < NB; c0 += 16) {
            uint32_t r[16];
            tmem_ld16(acc + c0, r);
            tmem_ld_wait();
#pragma unroll
            for (int v4 = 0; v4 < 4; ++v4)
              red_add_v4(blk + c0 + 4 * v4, make_float4(__uint_as_float(r[4 * v4]), __uint_as_float(r[4 * v4 + 1]),
                                                        __uint_as_float(r[4 * v4 + 2]), __uint_as_float(r[4 * v4 + 3])));
          }
          release_acc();
          asm volatile("bar.sync 1, %0;" ::"n"(kCLdThreads));
          if (et == 0) {
            // release (cumulative over the barrier: every thread's reductions) + acquire
            uint32_t* tk = tiles + 3 * t + 1 + ph;
            const uint32_t old = atom_add_acq_rel(tk, 1u);
            const int last = old == (uint32_t)(np - 1);
            if (last) *tk = 0u;  // every piece arrived: self-reset for the next launch
            *s_last = last;
          }
          asm volatile("bar.sync 1, %0;" ::"n"(kCLdThreads));
          finish = *s_last != 0;
          if (et == 0 && tb >= 0 && j < 2) stamp(tb + 1);
          if (finish) {
            for (int c0 = 0; c0 < NB; c0 += 64) {
              float4 v[16];
#pragma unroll
              for (int v4 = 0; v4 < 16; ++v4)
                v[v4] = c0 + 4 * v4 < NB ? __ldcg(reinterpret_cast<const float4*>(blk + c0) + v4)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
              if (et == 0 && c0 == 0 && tb >= 0) {
                asm volatile("" ::"f"(v[0].x), "f"(v[15].w));
                stamp(13);
              }
#pragma unroll
              for (int v4 = 0; v4 < 16; ++v4)
                if (c0 + 4 * v4 < NB && !(p.dbg & 2)) reinterpret_cast<float4*>(blk + c0)[v4] = make_float4(0.f, 0.f, 0.f, 0.f);
              if (write && !(p.dbg & 1)) {
#pragma unroll
                for (int v4 = 0; v4 < 16; ++v4) {
                  const int n = c0 + 4 * v4;
                  if (n < p.N) store_out(n, v[v4].x);
                  if (n + 1 < p.N) store_out(n + 1, v[v4].y);
                  if (n + 2 < p.N) store_out(n + 2, v[v4].z);
                  if (n + 3 < p.N) store_out(n + 3, v[v4].w);
                }
              }
            }
          }
        }
        if (et == 0 && tb >= 0 && j < 2) stamp(tb + 2);
        ++j;
        if (finish && ph == 0) {
          // publish phase-0 tile t to the phase-1 B producers of every CTA
          // (the release store is cumulative over the barrier)
          asm volatile("bar.sync 1, %0;" ::"n"(kCLdThreads));
          if (et == 0) {
            fence_proxy_async_global();
            st_release_u32(tiles + 3 * t, epoch + 1u);
            if (tb == 9) stamp(12);
          }
        }
      }
    }
    if (et == 0) stamp(6);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
  if (tid == 0) {
    stamp(7);
    if (tr) {
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[8] = smid;
    }
  }
  if (tid == 0) {
    // the last CTA out advances the epoch (flags of this launch = epoch + 1)
    const uint32_t old = atom_add_acq_rel(p.sync + 1, 1u);
    if (old == (uint32_t)(G - 1)) {
      p.sync[1] = 0u;
      __threadfence();
      st_release_u32(p.sync, epoch + 1u);
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode_c = nullptr;

int make_map_b(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_rows) {
  if (!g_encode_c) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return PS_ERR_CUDA;
    g_encode_c = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)CBK, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode_c(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? PS_OK : PS_ERR_VALUE;
}

int g_chain_stages = 0;  // debug override
unsigned long long* g_chain_trace = nullptr;

int chain_stages(int NB) {
  if (g_chain_stages > 0) return g_chain_stages;
  const int stage = CBM * CBK * 2 + NB * CBK * 2;
  int s = (224 * 1024 - 2048) / stage;
  return s > 12 ? 12 : (s < 2 ? 2 : s);
}

size_t chain_smem(int NB, int S) { return 1024 + (size_t)S * (CBM * CBK * 2 + NB * CBK * 2) + 256; }

int chain_nb(int N) { return (N + 15) / 16 * 16; }

// the sync area has a fixed size (kChainMaxTiles tiles), so a workspace reused
// at another shape keeps every flag / ticket where it was
constexpr int kChainMaxTiles = 1024;
constexpr size_t kChainSyncBytes = ((size_t)(2 + 3 * kChainMaxTiles) * 4 + 255) / 256 * 256;

// sync area + the phase-0 split-tile accumulators (rows0 columns x NB batch rows, f32)
size_t chain_ws_bytes(int N, int rows0) {
  return kChainSyncBytes + (size_t)((rows0 + CBM - 1) / CBM * CBM) * chain_nb(N) * 4;
}

// y0 = phase 0 output (bf16, (N, >= K of phase 1) row-major, row stride y0_ld)
int launch_chain(ChainParams& prm, const void* x, int64_t x_ld, int K0, const void* y0, int64_t y0_ld, int K1,
                 void* ws, size_t ws_bytes, cudaStream_t st) {
  const int rows0 = prm.ph[0].M;
  const int N = prm.N;
  if (N < 1 || N > kCMaxNB) return PS_ERR_VALUE;
  if (((uintptr_t)x % 16) || (x_ld % 8) || ((uintptr_t)y0 % 16) || (y0_ld % 8)) return PS_ERR_VALUE;
  prm.NB = chain_nb(N);
  prm.trace = g_chain_trace;
  {
    static const int gate = [] { const char* e = getenv("PS_CHAIN_GATE"); return e ? atoi(e) : 0; }();
    prm.gate = gate;
    static const int dbg = [] { const char* e = getenv("PS_CHAIN_DBG"); return e ? atoi(e) : 0; }();
    prm.dbg = dbg;
  }
  prm.stages = chain_stages(prm.NB);
  if (prm.maxT > kChainMaxTiles) return PS_ERR_VALUE;
  if (!ws || ws_bytes < chain_ws_bytes(N, rows0)) return PS_ERR_VALUE;
  prm.sync = static_cast<uint32_t*>(ws);
  prm.acc0 = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kChainSyncBytes);
  CUtensorMap t0, t1;
  int rc = make_map_b(&t0, x, (uint64_t)K0, (uint64_t)N, (uint64_t)x_ld, (uint32_t)prm.NB);
  if (rc != PS_OK) return rc;
  rc = make_map_b(&t1, y0, (uint64_t)K1, (uint64_t)N, (uint64_t)y0_ld, (uint32_t)prm.NB);
  if (rc != PS_OK) return rc;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(chain_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) !=
        cudaSuccess)
      return PS_ERR_CUDA;
    configured = true;
  }
  const size_t smem = chain_smem(prm.NB, prm.stages);
  // one CTA per SM: the stages take > half of the SM's shared memory, so
  // every CTA of the grid is resident at once (the flag waits rely on it)
  return launch_ex(chain_gemm_kernel, dim3(ps_num_sms()), dim3(kCThreads), smem, st, 1, t0, t1, prm);
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" size_t ps_sparse_mlp_workspace_bytes(int N, int D, int d) {
  (void)d;
  return chain_ws_bytes(N, D);
}

// Selective MLP in one launch: hidden[:, j] = relu(x W1[:, idx[j]] + b1[idx[j]]) (bf16, j < count; columns
// [count, round_up(count, 128)) written as 0); out += hidden[:, :count] W2[:, idx[:count]]^T + b2 (f32,
// accumulated: out holds the residual on entry).
extern "C" int ps_sparse_mlp(const void* w1_rows, const float* b1, const void* w2_rows, const float* b2, int D,
                             int d, const int32_t* idx, const int32_t* count_dev, const void* x, int64_t x_ld, int N,
                             void* hidden, int64_t h_ld, float* out, int64_t out_ld, void* ws, size_t ws_bytes,
                             void* stream) {
  if (!w1_rows || !w2_rows || !x || !hidden || !out || D < 1 || d < 8 || d % 8 || N < 1) return PS_ERR_VALUE;
  const int D_pad = (D + 127) / 128 * 128;
  if (h_ld < D_pad || out_ld < d || ((uintptr_t)w1_rows % 16) || ((uintptr_t)w2_rows % 16)) return PS_ERR_VALUE;
  if ((idx == nullptr) != (count_dev == nullptr)) return PS_ERR_VALUE;
  ChainParams prm = {};
  ChainPhase& u = prm.ph[0];
  u.w = static_cast<const uint16_t*>(w1_rows);
  u.w_ld = d;
  u.idx = idx;
  u.form = FORM_ROWS;
  u.M = D;
  u.K = d;
  u.use_count = count_dev != nullptr;
  u.bias = b1;
  u.act = PS_ACT_RELU;
  u.out = hidden;
  u.out_ld = h_ld;
  u.out_bf16 = 1;
  u.out_cols = D_pad;
  ChainPhase& v = prm.ph[1];
  v.w = static_cast<const uint16_t*>(w2_rows);
  v.w_ld = d;
  v.idx = idx;
  v.form = FORM_CONTRACT;
  v.M = d;
  v.K = D;
  v.use_count = count_dev != nullptr;
  v.bias = b2;
  v.act = PS_ACT_NONE;
  v.out = out;
  v.out_ld = out_ld;
  v.accumulate = 1;
  prm.count = count_dev;
  prm.N = N;
  prm.maxT = ((D + 127) / 128 > (d + 127) / 128) ? (D + 127) / 128 : (d + 127) / 128;
  return launch_chain(prm, x, x_ld, d, hidden, h_ld, D_pad, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

extern "C" size_t ps_router_mlp_workspace_bytes(int N, int h, int D) {
  (void)D;
  return chain_ws_bytes(N, h);
}

// Two-layer router MLP in one launch (routers.py:286-288):
// hid = relu(x W_in + b_in) (bf16), logits = hid W_out + b_out (f32, b_out may be NULL).
extern "C" int ps_router_mlp(const void* w_in_rows, const float* b_in, const void* w_out_rows, const float* b_out,
                             int d, int h, int D, const void* x, int64_t x_ld, int N, void* hid, int64_t hid_ld,
                             float* logits, int64_t logits_ld, void* ws, size_t ws_bytes, void* stream) {
  if (!w_in_rows || !w_out_rows || !x || !hid || !logits || d < 8 || d % 8 || h < 8 || h % 8 || D < 1 || N < 1)
    return PS_ERR_VALUE;
  if (hid_ld < h || logits_ld < D || ((uintptr_t)w_in_rows % 16) || ((uintptr_t)w_out_rows % 16))
    return PS_ERR_VALUE;
  ChainParams prm = {};
  ChainPhase& a = prm.ph[0];
  a.w = static_cast<const uint16_t*>(w_in_rows);
  a.w_ld = d;
  a.form = FORM_ROWS;
  a.M = h;
  a.K = d;
  a.bias = b_in;
  a.act = PS_ACT_RELU;
  a.out = hid;
  a.out_ld = hid_ld;
  a.out_bf16 = 1;
  a.out_cols = h;
  ChainPhase& b = prm.ph[1];
  b.w = static_cast<const uint16_t*>(w_out_rows);
  b.w_ld = h;
  b.form = FORM_ROWS;
  b.M = D;
  b.K = h;
  b.bias = b_out;
  b.act = PS_ACT_NONE;
  b.out = logits;
  b.out_ld = logits_ld;
  b.out_bf16 = 0;
  b.out_cols = D;
  b.whole = 1;  // output tiles never split: logits are stored, not accumulated
  prm.N = N;
  prm.maxT = ((D + 127) / 128 > (h + 127) / 128) ? (D + 127) / 128 : (h + 127) / 128;
  return launch_chain(prm, x, x_ld, d, hid, hid_ld, h, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

extern "C" void ps_debug_chain_stages(int stages) { g_chain_stages = stages; }
// debug: per-CTA timestamps (16 u64 per CTA: start, after griddep wait, first
// stage at the MMA, last phase-0 accumulator, first phase-1 flag wait begins,
// first flag acquired, epilogue done, end, smid); NULL = off
extern "C" void ps_debug_chain_trace(void* buf) { g_chain_trace = static_cast<unsigned long long*>(buf); }
