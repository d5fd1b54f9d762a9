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
// Decode GEMMs stream weights (batch N <= 256 << the ~250 flop/byte ridge),
// so the design goal is every SM streaming weights continuously with short
// prologue / epilogue tails:
//   * swap-AB: the UMMA M dimension (128) runs over the weight side (neurons
//     for UP, output features for DOWN), N over the batch (16..256);
//   * persistent thread-block CLUSTERS split K: the C CTAs of a cluster work
//     on the same 128-row tile concurrently, each over 1/C of the K blocks
//     (K = the union size for DOWN, read on the device), and reduce their f32
//     partial tiles through distributed shared memory (DSMEM) with mbarrier
//     handshakes -- no global partials, no atomics, deterministic rank-order
//     sums; clusters loop over tiles (the device-resident union size bounds
//     the tile count: no host sync, CUDA-graph capturable);
//   * warp roles: warp 0 drives the TMA engine (B operand, and dense A as
//     2-D tiles / gathered A as sm_100 tile::gather4 when lsu_mode == 0);
//     warps 6-9 stream the A operand with 16-byte cp.async (LDGSTS) into the
//     same 128B-swizzled layout (the default for gathered rows: two copy
//     engines per SM, ~2x the gather4 rate); warp 1 issues tcgen05.mma from
//     one thread into one of two TMEM accumulators; warps 2-5 drain the other
//     accumulator (tcgen05.ld 32x32b) through a shared-memory staging tile and
//     apply bias / ReLU / residual with 16-byte vector stores.
#include <cuda.h>
#include <type_traits>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"

namespace ps {
namespace {

constexpr int BM = 128;   // UMMA M
constexpr int BK = 64;    // K elements per stage (one 128-byte swizzle row)
constexpr int kEpiThreads = 128;
constexpr int kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue, warps 6-9 LSU loaders
constexpr int kMaxNB = 256;
constexpr int kEpiCols = 64;   // batch rows staged per epilogue pass (32 KB of smem)
constexpr int kProdWarp = 0, kMmaWarp = 1, kEpiWarp0 = 2, kLdWarp0 = 6;
constexpr int kLdThreads = 128;
constexpr int kMaxCluster = 8;

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
  int push;     // split-K reduction: 1 = partial rows pushed to their owner CTA (st.async), 0 = pulled (DSMEM loads)
  int a_early;  // A (weights, idx, count) ready before the previous kernel ends: stream A pre-griddep_wait
  // union hand-off (PS_GG_BITMAP): the ids are derived on the device from the
  // selection bitmap (bm_words uint32 words) instead of a compacted id list
  const uint32_t* bm;
  int bm_words;
  int32_t* count_out;  // UP, bitmap mode: receives the union size
  int ids_cap;         // bitmap mode: ids expanded into shared memory up front (the rest: cursor walk)
  unsigned long long* trace;  // debug: per-CTA timestamps (ps_debug_gemm_trace), NULL normally
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

PS_DEV uint32_t sw128(int row, int unit) {  // byte offset of 16B unit `unit` of K-major row `row`
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((unit ^ (row & 7)) << 4));
}

PS_DEV uint32_t cluster_id() {
  uint32_t r;
  asm("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
PS_DEV uint32_t num_clusters() {
  uint32_t r;
  asm("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
PS_DEV void remote_arrive(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
// relaxed remote arrive: no fence (MEMBAR.GPU) -- for "done reading your
// staging tile" signals whose loads already returned their data
PS_DEV void remote_arrive_relaxed(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
PS_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
PS_DEV float4 ld_dsmem_v4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

// LSU_A: the A operand (weights, gathered or dense) is streamed by 4 loader
// warps with 16-byte cp.async (LDGSTS) while the TMA engine moves only the B
// operand.  GATHER: A rows (UP) / K rows (DOWN) are selected by idx.  BMAP
// (union hand-off, PS_GG_BITMAP): the ids come from the selection bitmap; a
// separate instantiation, so the id-list path compiles exactly as before.
template <int MODE, bool GATHER, bool LSU_A, bool BMAP = false>
__global__ void __launch_bounds__(kThreads, 2)
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
  uint64_t* rdy = tempty + 2;    // cluster: every CTA's partial tile staged
  uint64_t* fre = rdy + 1;       // cluster: every CTA done reading the staged tiles
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fre + 1);
  float* stg = reinterpret_cast<float*>(smem + S * stage_bytes + 256);  // [kEpiCols][BM] f32
  uint32_t* s_bw = reinterpret_cast<uint32_t*>(stg + kEpiCols * BM);  // bitmap mode: [bm_words] words
  int* s_bpre = reinterpret_cast<int*>(s_bw + p.bm_words);            // [bm_words + 1] prefix popcounts
  int* s_bscan = s_bpre + p.bm_words + 1;                              // [kThreads / 32] warp totals
  uint16_t* s_ids = reinterpret_cast<uint16_t*>(s_bscan + kThreads / 32);  // [ids_cap] ids of this CTA's positions

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = (int)cluster_size();
  const int rank = (int)cluster_rank();
  const int cid = (int)cluster_id(), ncl = (int)num_clusters();
  unsigned long long* tr = p.trace ? p.trace + 16 * (size_t)blockIdx.x : nullptr;
  if (tr && tid == 0) {
    unsigned smid;
    asm("mov.u32 %0, %smid;" : "=r"(smid));
    tr[0] = gtimer();
    tr[7] = smid;
  }

  // ---- input-independent prologue first (barrier init, TMEM alloc, tensor
  // map prefetch): under PDL it overlaps the previous grid's tail
  const uint32_t tcols = NB <= 16 ? 32 : (NB <= 32 ? 64 : (NB <= 64 ? 128 : (NB <= 128 ? 256 : 512)));
  if (warp == kMmaWarp) {
    if (lane == 0) {
      for (int s = 0; s < S; ++s) {
        mbar_init(&full[s], LSU_A ? 1 + kLdThreads : 1);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], 4);  // one arrival per epilogue warp
      }
      mbar_init(rdy, p.push ? 1 : C);
      mbar_init(fre, p.push ? (C > 1 ? C - 1 : 1) : C);
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
  // peers' barriers must be initialised before any remote arrive
  // (fence_mbar_init already released the inits at cluster scope: a relaxed
  //  barrier suffices and avoids a MEMBAR.GPU)
  if (C > 1) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  }
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // ---- PDL: with the A operand ready (static weights, or ids produced >= 2
  // launches earlier) only the B / epilogue roles wait for the previous grid
  if (!p.a_early) {
    griddep_wait();
    if (tid == 0) griddep_launch();
  }
  // ---- union hand-off: word-prefix popcounts of the selection bitmap, so
  // union position `pos` maps to its id with a binary search + __fns (no
  // compacted id list, no compaction on the selection kernel's tail)
  if (BMAP) {
    const int nw = p.bm_words;
    const int per = (nw + kThreads - 1) / kThreads;
    const int w0 = tid * per;
    int loc = 0;
    for (int q = 0; q < per; ++q) {
      const int w = w0 + q;
      if (w < nw) {
        const uint32_t a = __ldcg(p.bm + w);
        s_bw[w] = a;
        loc += __popc(a);
      }
    }
    int incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_bscan[warp] = incl;
    __syncthreads();
    int run = incl - loc;
    for (int i = 0; i < warp; ++i) run += s_bscan[i];
    for (int q = 0; q < per; ++q) {
      const int w = w0 + q;
      if (w < nw) {
        s_bpre[w] = run;
        run += __popc(s_bw[w]);
      }
    }
    if (tid == 0) {
      int tot = 0;
      for (int i = 0; i < kThreads / 32; ++i) tot += s_bscan[i];
      s_bpre[nw] = tot;
    }
    __syncthreads();
  }
  // bitmap mode: the word holding union position pos (< count) by binary
  // search, then ascending positions walk forward from it (a thread's
  // positions are increasing, a few words apart)
  auto bm_seek = [&](int pos) -> int {
    int lo = 0, hi = p.bm_words - 1;  // the last word whose prefix is <= pos holds it
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_bpre[mid] <= pos) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  };
  auto bm_id = [&](int pos, int& w) -> int {  // w: a word at or before pos's word
    while (s_bpre[w + 1] <= pos) ++w;
    return w * 32 + (int)__fns(s_bw[w], 0u, pos - s_bpre[w] + 1);
  };
  // ---- device-side work partition (identical in every role and CTA of a cluster)
  const int count = BMAP ? s_bpre[p.bm_words] : (p.count ? *p.count : (MODE == MODE_UP ? p.M : p.K));
  if (MODE == MODE_UP && BMAP && p.count_out && blockIdx.x == 0 && tid == 0) *p.count_out = count;
  const int klimit = (MODE == MODE_UP) ? p.K : count;
  const int kbt = (klimit + BK - 1) / BK;
  const int live_m = (MODE == MODE_UP) ? (count + BM - 1) / BM : (p.M + BM - 1) / BM;
  const int tiles = live_m * p.n_tiles;
  const int per = (kbt + C - 1) / C;
  const int kb0 = rank * per;
  const int nkb = max(0, min(kbt, kb0 + per) - kb0);  // K blocks of this CTA (same for every tile)
  const int my_tiles = cid < tiles ? (tiles - cid + ncl - 1) / ncl : 0;
  // bitmap mode: expand the ids of this CTA's union positions (DOWN: its K
  // range; UP: its first tile) into shared memory with every thread, one word
  // each, so the loaders read them with one shared load
  int ids_p0 = 0, ids_n = 0;
  if (BMAP) {
    if (MODE == MODE_DOWN) {
      ids_p0 = kb0 * BK;
      ids_n = min(count, (kb0 + nkb) * BK) - ids_p0;
    } else {
      ids_p0 = live_m > 0 ? (cid % live_m) * BM : 0;
      ids_n = min(count, ids_p0 + BM) - ids_p0;
    }
    if (my_tiles == 0 || ids_n < 0) ids_n = 0;
    if (ids_n > p.ids_cap) ids_n = p.ids_cap;
    if (ids_n > 0) {
      const int wa = bm_seek(ids_p0), wb = bm_seek(ids_p0 + ids_n - 1);
      for (int w = wa + tid; w <= wb; w += kThreads) {
        uint32_t bits = s_bw[w];
        int q = s_bpre[w] - ids_p0;
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1;
          if (q >= 0 && q < ids_n) s_ids[q] = (uint16_t)(w * 32 + b);
          ++q;
        }
      }
    }
    __syncthreads();
  }
  // every CTA of a cluster sees the same my_tiles, so whole clusters leave together
  if (my_tiles == 0) {
    if (p.a_early) {
      griddep_wait();
      if (tid == 0) griddep_launch();
    }
    if (warp == kMmaWarp) tmem_dealloc(tmem, tcols);
    return;
  }

  if (tr && tid == 0) tr[1] = gtimer();

  auto tile_of = [&](int j) { return cid + j * ncl; };

  if (warp == kProdWarp) {
    // ------------------------------------------------------------ TMA producer
    auto load4 = [&](int base, int lim, int first) -> int4 {
      if (base + 4 <= lim) return __ldg(reinterpret_cast<const int4*>(p.idx + base));
      int r[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = base + j < lim ? __ldg(p.idx + base + j) : first;
      return make_int4(r[0], r[1], r[2], r[3]);
    };
    if (p.a_early) {
      griddep_wait();
      if (lane == 0) griddep_launch();
    }
    int i = 0;
    for (int j = 0; j < my_tiles; ++j) {
      const int t = tile_of(j);
      const int mt = t % live_m, nt = t / live_m;
      const int m0 = mt * BM, n0 = nt * NB;
      int4 rid = make_int4(0, 0, 0, 0);
      if (!LSU_A && GATHER && MODE == MODE_UP) rid = load4(m0 + lane * 4, count, __ldg(p.idx + m0));
      for (int kb = kb0; kb < kb0 + nkb; ++kb, ++i) {
        const int k0 = kb * BK;
        int4 kid = make_int4(0, 0, 0, 0);
        if (!LSU_A && GATHER && MODE == MODE_DOWN) kid = load4(k0 + 4 * (lane & 15), count, __ldg(p.idx));
        const int s = i % S;
        if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        uint8_t* sa = smem + s * stage_bytes;
        uint8_t* sb = sa + a_bytes;
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[s], LSU_A ? b_bytes : stage_bytes);
          tma_load_2d(sb, &tmB, k0, n0, &full[s]);  // B: NB batch rows x 64 K
        }
        if (!LSU_A) {
          if (GATHER) {
            if (MODE == MODE_UP) {
              tma_gather4(sa + lane * 512, &tmA, k0, rid.x, rid.y, rid.z, rid.w, &full[s]);
            } else {
              const int c = lane >> 4, jj = lane & 15;
              tma_gather4(sa + c * 8192 + (jj >> 1) * 1024 + (jj & 1) * 512, &tmA, m0 + 64 * c, kid.x, kid.y,
                          kid.z, kid.w, &full[s]);
            }
          } else if (lane == 0) {
            if (MODE == MODE_UP) {
              tma_load_2d(sa, &tmA, k0, m0, &full[s]);  // 128 rows x 64 K
            } else {
              tma_load_2d(sa, &tmA, m0, k0, &full[s]);  // 64 K rows x 64 MN, two MN chunks
              tma_load_2d(sa + 8192, &tmA, m0 + 64, k0, &full[s]);
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp >= kLdWarp0) {
    // ------------------------------------------------------------ LSU A loaders (warps 6..9)
    if (LSU_A) {
      const int lt = tid - kLdWarp0 * 32;  // 0..127
      int i = 0;
      for (int j = 0; j < my_tiles; ++j) {
        const int t = tile_of(j);
        const int m0 = (t % live_m) * BM;
        const uint16_t* src[8];  // UP: this thread's 8 rows of the tile
        if (MODE == MODE_UP) {
          int bw = (BMAP && j > 0 && m0 + (lt >> 3) < count) ? bm_seek(m0 + (lt >> 3)) : 0;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const int gr = m0 + (lt >> 3) + 16 * r;
            const int id = gr < count ? (GATHER ? (BMAP ? (j == 0 && gr - ids_p0 < ids_n ? (int)s_ids[gr - ids_p0]
                                                                                         : bm_id(gr, bw))
                                                            : __ldg(p.idx + gr))
                                                : gr)
                                      : -1;
            src[r] = id >= 0 ? p.w + (size_t)id * p.w_ld + (lt & 7) * 8 : nullptr;
          }
        }
        int kid[8];  // DOWN: ids of this thread's 8 K rows of the current stage (prefetched)
        int dw = -1;   // bitmap mode: word cursor (positions ascend through the tile's K blocks)
        auto down_ids = [&](int kb, int* o) {
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const int kg = kb * BK + (lt >> 4) + 8 * r;
            if (BMAP && kg < count && kg - ids_p0 >= ids_n && dw < 0) dw = bm_seek(kg);
            o[r] = kg < count ? (GATHER ? (BMAP ? (kg - ids_p0 < ids_n ? (int)s_ids[kg - ids_p0] : bm_id(kg, dw))
                                                : __ldg(p.idx + kg))
                                       : kg)
                              : -1;
          }
        };
        if (MODE == MODE_DOWN && nkb > 0) down_ids(kb0, kid);
        for (int kb = kb0; kb < kb0 + nkb; ++kb, ++i) {
          const int k0 = kb * BK;
          int kid_next[8];
          if (MODE == MODE_DOWN && kb + 1 < kb0 + nkb) down_ids(kb + 1, kid_next);
          const int s = i % S;
          if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
          uint8_t* sa = smem + s * stage_bytes;
          if (MODE == MODE_UP) {
            const int u = lt & 7;
            const bool kok = k0 + u * 8 < p.K;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              const int row = (lt >> 3) + 16 * r;
              const bool ok = kok && src[r] != nullptr;
              cp_async16_l2_256(sa + sw128(row, u), ok ? (const void*)(src[r] + k0) : (const void*)p.w, ok ? 16u : 0u);
            }
          } else {
            // 64 K rows x 128 output features, MN-major SW128 atoms (8 K x 64 MN);
            // 16 lanes read one 256-byte K row
            const int mu = lt & 15;
            const int gm = m0 + mu * 8;
            const bool mok = gm < p.M;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              const int kk = (lt >> 4) + 8 * r;
              const bool ok = mok && kid[r] >= 0;
              const void* srcp = ok ? (const void*)(p.w + (size_t)kid[r] * p.w_ld + gm) : (const void*)p.w;
              const uint32_t off = (uint32_t)((mu >> 3) * 8192 + (kk >> 3) * 1024 + (kk & 7) * 128 +
                                              (((mu & 7) ^ (kk & 7)) << 4));
              cp_async16_l2_256(sa + off, srcp, ok ? 16u : 0u);
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) kid[r] = kid_next[r];
          }
          cp_async_arrive_noinc(&full[s]);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = make_idesc_bf16(BM, NB, MODE == MODE_DOWN ? 1 : 0, 0);
      int i = 0;
      for (int j = 0; j < my_tiles; ++j) {
        const int a = j & 1;
        if (j >= 2) mbar_wait(&tempty[a], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + a * NB;
        for (int kb = 0; kb < nkb; ++kb, ++i) {
          const int s = i % S;
          mbar_wait(&full[s], (i / S) & 1);
          if (tr && i == 0) tr[2] = gtimer();
          if (LSU_A) fence_proxy_async();  // generic-proxy cp.async writes -> async-proxy MMA reads
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
            umma_bf16(acc, ad, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        if (nkb > 0)
          umma_commit(&tfull[a]);
        else
          mbar_arrive(&tfull[a]);  // this CTA has no K blocks: its partial is zero
      }
      if (tr) tr[3] = gtimer();
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    if (p.a_early) griddep_wait();       // residual / out belong to the previous grid's stream order
    const int q = warp & 3;               // TMEM lane quadrant of this warp
    const int m = q * 32 + lane;          // tile row (TMEM lane)
    const int et = tid - kEpiWarp0 * 32;  // 0..127
    // this CTA finishes rows [rank*rows, (rank+1)*rows) of every tile; each
    // thread always owns the same 4 consecutive output rows (columns of out)
    const int rows = BM / C;
    const int vec_per_n = rows / 4;
    const int my_m = rank * rows + (et % vec_per_n) * 4;
    int use = 0;  // rdy / fre phase counter
    const uint32_t stg_s = smem_u32(stg);
    uint32_t peer_stg[kMaxCluster], peer_rdy[kMaxCluster], peer_fre[kMaxCluster];
#pragma unroll
    for (int c = 0; c < kMaxCluster; ++c) {
      if (c < C) {
        peer_stg[c] = map_peer(stg_s, c);
        peer_rdy[c] = map_peer(smem_u32(rdy), c);
        peer_fre[c] = map_peer(smem_u32(fre), c);
      }
    }
    for (int j = 0; j < my_tiles; ++j) {
      const int t = tile_of(j);
      const int a = j & 1;
      const int mt = t % live_m, nt = t / live_m;
      const int m0 = mt * BM, n0 = nt * NB;
      const int nrows = min(NB, p.N - n0);
      float my_bias[4] = {0.f, 0.f, 0.f, 0.f};
      bool my_live[4];
      int ew = (MODE == MODE_UP && BMAP && p.bias && j > 0 && m0 + my_m < count) ? bm_seek(m0 + my_m) : 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int gm = m0 + my_m + u;
        my_live[u] = (MODE == MODE_UP) ? gm < count : gm < p.M;
        if (my_live[u] && p.bias)
          my_bias[u] = __ldg(p.bias + ((MODE == MODE_UP && p.idx)
                                           ? (BMAP ? (j == 0 && gm - ids_p0 < ids_n ? (int)s_ids[gm - ids_p0]
                                                                                    : bm_id(gm, ew))
                                                   : __ldg(p.idx + gm))
                                           : gm));
      }
      auto load_res = [&](int n) -> float4 {
        float res[4] = {0.f, 0.f, 0.f, 0.f};
        const int gm0 = m0 + my_m;
        if (p.residual) {
          if (p.vec_ok && gm0 + 4 <= p.M) {
            return *reinterpret_cast<const float4*>(p.residual + (size_t)(n0 + n) * p.res_ld + gm0);
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (gm0 + u < p.M) res[u] = p.residual[(size_t)(n0 + n) * p.res_ld + gm0 + u];
          }
        }
        return make_float4(res[0], res[1], res[2], res[3]);
      };
      auto finish4r = [&](int n, float4 v, float4 r4) {
        const int gm0 = m0 + my_m;
        const size_t o = (size_t)(n0 + n) * p.out_ld + gm0;
        float vv[4] = {v.x, v.y, v.z, v.w};
        float res[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float x = 0.f;
          if (my_live[u]) {
            x = vv[u] + my_bias[u];
            if (MODE == MODE_UP && p.act == PS_ACT_RELU) x = fmaxf(x, 0.f);
            x += res[u];
          }
          vv[u] = x;
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
          for (int u = 0; u < 4; ++u) {
            if (gm0 + u >= p.M) break;
            if (p.out_bf16)
              reinterpret_cast<uint16_t*>(p.out)[o + u] = f2bf(vv[u]);
            else
              reinterpret_cast<float*>(p.out)[o + u] = vv[u];
          }
        }
      };
      auto finish4 = [&](int n, float4 v) { finish4r(n, v, load_res(n)); };

      mbar_wait(&tfull[a], (j >> 1) & 1);
      if (tr && et == 0 && j == 0) tr[8] = gtimer();
      tc_fence_after();
      for (int cb = 0; cb < NB; cb += kEpiCols) {
        const int ncb = min(kEpiCols, NB - cb);
        if (C > 1 && p.push) {
          // ---- push reduction: CTA `rank` owns rows [rank*rows, (rank+1)*rows) of
          // the tile.  Every CTA sends each row's partial straight from TMEM to
          // the owner's slot `rank` (st.async, completing bytes on the owner's
          // rdy barrier); the owner sums its C slots from local shared memory.
          // stg is viewed as slot[C][kEpiCols][rows].
          const int rows_o = rows;
          const int rows_here = min(ncb, nrows - cb);
          if (use > 0) mbar_wait_cluster(fre, (use - 1) & 1);  // every owner consumed the last chunk
          {
            const int o = m / rows_o, ml = m - o * rows_o;
            const uint32_t dst = peer_stg[o], bar_o = peer_rdy[o];
            for (int c0 = 0; c0 < ncb; c0 += 16) {
              uint32_t r[16];
              if (nkb > 0) {
                tmem_ld16(tmem + a * NB + ((uint32_t)(q * 32) << 16) + cb + c0, r);
                tmem_ld_wait();
              } else {
#pragma unroll
                for (int u = 0; u < 16; ++u) r[u] = 0u;
              }
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const int idx = (rank * kEpiCols + c0 + u) * rows_o + ml;
                if (o == rank) stg[idx] = __uint_as_float(r[u]);
                else st_async_f32(dst + (uint32_t)idx * 4u, __uint_as_float(r[u]), bar_o);
              }
            }
          }
          if (cb + kEpiCols >= NB) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[a]);  // accumulator free for the MMA warp
          }
          if (et == 0) mbar_arrive_expect_tx(rdy, (uint32_t)((C - 1) * rows_o * ncb * 4));
          auto push_reduce = [&](auto cc) {
            constexpr int CC = decltype(cc)::value;
            constexpr int NV = (kEpiCols * (BM / CC / 4)) / kEpiThreads;  // vectors per thread
            const int vpn = BM / CC / 4;
            const int mloc = (et % vpn) * 4;
            float4 res[NV];
#pragma unroll
            for (int g = 0; g < NV; ++g) {  // residual rows in flight across the wait
              const int v = et + g * kEpiThreads;
              res[g] = v < rows_here * vpn ? load_res(cb + v / vpn) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));  // my own slot written
            mbar_wait_cluster(rdy, use & 1);                      // the peers' slots landed
            if (tr && et == 0 && j == 0 && cb == 0) tr[11] = gtimer();
#pragma unroll
            for (int g = 0; g < NV; ++g) {
              const int v = et + g * kEpiThreads;
              if (v < rows_here * vpn) {
                const int n = v / vpn;
                float4 sum = *reinterpret_cast<const float4*>(stg + n * rows_o + mloc);
#pragma unroll
                for (int c = 1; c < CC; ++c) {
                  const float4 t4 = *reinterpret_cast<const float4*>(stg + (c * kEpiCols + n) * rows_o + mloc);
                  sum.x += t4.x; sum.y += t4.y; sum.z += t4.z; sum.w += t4.w;
                }
                finish4r(cb + n, sum, res[g]);
              }
            }
          };
          if (C == 2) push_reduce(std::integral_constant<int, 2>{});
          else if (C == 4) push_reduce(std::integral_constant<int, 4>{});
          else push_reduce(std::integral_constant<int, 8>{});
          asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));  // every read of my slots done
          if (tr && et == 0 && j == 0 && cb == 0) tr[12] = gtimer();
          if (et == 0 && !(j == my_tiles - 1 && cb + kEpiCols >= NB))
            for (int c = 0; c < C; ++c)
              if (c != rank) remote_arrive_relaxed(peer_fre[c]);
          ++use;
          continue;
        }
        // 1) this CTA's partial (or zero) -> staging tile stg[n][m]
        for (int c0 = 0; c0 < ncb; c0 += 16) {
          uint32_t r[16];
          if (nkb > 0) {
            tmem_ld16(tmem + a * NB + ((uint32_t)(q * 32) << 16) + cb + c0, r);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int u = 0; u < 16; ++u) r[u] = 0u;
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) stg[(c0 + u) * BM + m] = __uint_as_float(r[u]);
        }
        if (cb + kEpiCols >= NB) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[a]);  // accumulator free for the MMA warp
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));
        if (tr && et == 0 && j == 0 && cb == 0) tr[10] = gtimer();
        const int rows_here = min(ncb, nrows - cb);
        if (C == 1) {
          for (int v = et; v < rows_here * vec_per_n; v += kEpiThreads) {
            const int n = v / vec_per_n;
            finish4(cb + n, *reinterpret_cast<const float4*>(stg + n * BM + my_m));
          }
          asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));
        } else {
          // 2) every CTA staged: reduce my rows over the C partials in rank
          //    order.  A thread owns <= kVecT vectors (C >= 2); its residual
          //    rows are fetched before the wait and all C x kVecT DSMEM loads
          //    are issued before the first use.
          constexpr int kVecT = (kEpiCols * BM / 8) / kEpiThreads;  // 8
          const int nvec = rows_here * vec_per_n;
          if (et == 0)
            for (int c = 0; c < C; ++c) remote_arrive(peer_rdy[c]);
          mbar_wait_cluster(rdy, use & 1);
          if (tr && et == 0 && j == 0 && cb == 0) tr[11] = gtimer();
          auto reduce = [&](auto cc) {
            constexpr int CC = decltype(cc)::value;
            constexpr int NV = 2 * kVecT / CC;  // vectors per thread at this cluster size
            constexpr int GV = 8 / CC;          // vectors per load batch (8 DSMEM float4 in flight)
#pragma unroll
            for (int g0 = 0; g0 < NV; g0 += GV) {
              float4 buf[GV][CC], res[GV];
#pragma unroll
              for (int gi = 0; gi < GV; ++gi) {
                const int v = et + (g0 + gi) * kEpiThreads;
                const uint32_t off = (uint32_t)(((v / vec_per_n) * BM + my_m) * 4);
                res[gi] = v < nvec ? load_res(cb + v / vec_per_n) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int c = 0; c < CC; ++c)
                  buf[gi][c] = v < nvec ? ld_dsmem_v4(map_peer(stg_s, c) + off) : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int gi = 0; gi < GV; ++gi) {
                const int v = et + (g0 + gi) * kEpiThreads;
                if (v < nvec) {
                  float4 sum = buf[gi][0];
#pragma unroll
                  for (int c = 1; c < CC; ++c) {
                    sum.x += buf[gi][c].x; sum.y += buf[gi][c].y; sum.z += buf[gi][c].z; sum.w += buf[gi][c].w;
                  }
                  finish4r(cb + v / vec_per_n, sum, res[gi]);
                }
              }
            }
          };
          if (C == 2) reduce(std::integral_constant<int, 2>{});
          else if (C == 4) reduce(std::integral_constant<int, 4>{});
          else reduce(std::integral_constant<int, 8>{});
          // 3) done reading the peers' staging tiles
          asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads));
          if (et == 0)
            for (int c = 0; c < C; ++c) remote_arrive_relaxed(peer_fre[c]);
          if (tr && et == 0 && j == 0 && cb == 0) tr[12] = gtimer();
          mbar_wait_cluster(fre, use & 1);
          if (tr && et == 0 && j == 0 && cb == 0) tr[13] = gtimer();
          ++use;
        }
      }
      if (tr && et == 0 && j == 0) tr[9] = gtimer();
    }
    if (tr && et == 0) tr[4] = gtimer();
  }
  tc_fence_before();
  __syncthreads();
  if (tr && tid == 0) tr[5] = gtimer();
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
int g_push = -1;     // -1: from env PS_GG_PUSH (default 1)
int g_lsu_mode = 1;  // 0: TMA for A, 1: LSU for gathered A, 2: LSU for all A

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

int cta_slots(int NB) {
  static const int env_target = [] {  // tuning hook: PS_GG_TARGET = CTA slots per launch
    const char* e = getenv("PS_GG_TARGET");
    return e ? atoi(e) : 0;
  }();
  if (g_target_override > 0) return g_target_override;
  if (env_target > 0) return env_target;
  return ps_num_sms() * ctas_per_sm(NB);
}

// cluster size: enough CTAs per tile to fill every CTA slot, >= 2 K blocks each
int pick_cluster(int NB, int tiles_est, int kbt) {
  const int slots = cta_slots(NB);
  int c = 1;
  while (c < kMaxCluster && tiles_est * c * 2 <= slots && (kbt / (c * 2)) >= 2) c *= 2;
  return c;
}

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

template <int MODE, bool GATHER, bool LSU_A, bool BMAP = false>
int launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const GGParams& prm, int cluster, int work_ctas,
             cudaStream_t st) {
  const size_t smem = smem_bytes(prm.NB, prm.stages) +
                      (prm.bm ? 4 * (2 * (size_t)prm.bm_words + 1 + kThreads / 32) + ((size_t)prm.ids_cap * 2 + 15) / 16 * 16
                              : 0);
  auto kern = gather_gemm_kernel<MODE, GATHER, LSU_A, BMAP>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      return PS_ERR_CUDA;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      return PS_ERR_CUDA;
    configured = true;
  }
  // persistent grid: the CTA slots, but no more than the expected work (idle
  // CTAs would only occupy slots the next kernel's early (PDL) CTAs can use);
  // more live tiles than expected are picked up by the tile loop
  int grid = (cta_slots(prm.NB) / cluster) * cluster;
  if (work_ctas > 0 && work_ctas < grid) grid = work_ctas;
  return launch_ex(kern, dim3(grid), dim3(kThreads), smem, st, cluster, ta, tb, prm);
}

// w_rows: (w_rows_n, w_cols) row-major; B operand x: (N, kx) with row stride x_ld
template <int MODE>
int launch(GGParams& prm, int64_t w_rows_n, int64_t w_cols, int64_t kx, int tiles_est, int kbt_est,
           cudaStream_t st) {
  CUtensorMap ta, tb;
  int rc = make_map(&tb, prm.x, (uint64_t)kx, (uint64_t)prm.N, (uint64_t)prm.x_ld, BK, prm.NB);
  if (rc != PS_OK) return rc;
  const bool gather = prm.idx != nullptr;
  if (MODE == MODE_UP)
    rc = make_map(&ta, prm.w, (uint64_t)w_cols, (uint64_t)w_rows_n, (uint64_t)prm.w_ld, BK, gather ? 1 : BM);
  else
    rc = make_map(&ta, prm.w, (uint64_t)w_cols, (uint64_t)w_rows_n, (uint64_t)prm.w_ld, 64, gather ? 1 : BK);
  if (rc != PS_OK) return rc;
  const int cluster = pick_cluster(prm.NB, tiles_est * prm.n_tiles, kbt_est);
  const int work = tiles_est * prm.n_tiles * cluster;
  // bitmap mode: ids expanded up front (one more K block of margin for DOWN)
  prm.ids_cap = MODE == MODE_DOWN ? ((kbt_est + cluster - 1) / cluster + 1) * BK : BM;
  const bool lsu = g_lsu_mode == 2 || (g_lsu_mode == 1 && gather);
  if (prm.bm) return launch_t<MODE, true, true, true>(ta, tb, prm, cluster, work, st);  // gg_bitmap checked lsu
  if (gather)
    return lsu ? launch_t<MODE, true, true>(ta, tb, prm, cluster, work, st)
               : launch_t<MODE, true, false>(ta, tb, prm, cluster, work, st);
  return lsu ? launch_t<MODE, false, true>(ta, tb, prm, cluster, work, st)
             : launch_t<MODE, false, false>(ta, tb, prm, cluster, work, st);
}

}  // namespace
}  // namespace ps

using namespace ps;

// The cluster kernel reduces split-K partials on chip: only a token
// workspace is needed (kept in the ABI for callers that size one).
extern "C" size_t ps_gather_gemm_workspace_bytes(int N, int M, int K, int splits) {
  (void)N; (void)M; (void)K; (void)splits;
  return 256;
}

// `splits` argument of ps_gather_gemm(_t) = expected live union size (rows
// for UP, K for DOWN) used to size the K-split clusters; 0 = the maximum.
extern "C" int ps_gather_gemm_auto_splits(int N, int M, int K) {
  (void)N; (void)M; (void)K;
  return 0;
}

static int gg_common(GGParams& prm, const void* w_rows, const int32_t* idx, const int32_t* count_dev,
                     const void* x, int64_t x_ld, const float* bias, int N, int M, int K, void* out, int64_t out_ld,
                     int out_dtype) {
  if (N < 1 || M < 1 || K < 1 || !w_rows || !x || !out) return PS_ERR_VALUE;
  if (((uintptr_t)w_rows % 16) || ((uintptr_t)x % 16) || (x_ld % 8)) return PS_ERR_VALUE;
  prm.w = static_cast<const uint16_t*>(w_rows);
  prm.idx = idx;
  prm.count = count_dev;
  prm.bm = nullptr;
  prm.bm_words = 0;
  prm.count_out = nullptr;
  prm.ids_cap = 0;
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
  prm.a_early = 0;
  if (g_push < 0) {
    const char* e = getenv("PS_GG_PUSH");
    g_push = e ? atoi(e) : 1;
  }
  // push pays while a tile has <= 2 column chunks; at 4 (B = 256) the per-chunk
  // "slot free" round trips serialise it (UP 41.7 -> 48.1 us, ncu, B = 256)
  prm.push = g_push && prm.NB <= 2 * kEpiCols;
  prm.vec_ok = (out_ld % 4 == 0) && ((uintptr_t)out % 16 == 0);
  return PS_OK;
}

namespace ps {
namespace {

// ---------------------------------------------------------------------------
// Small-batch UP projection as a gathered GEMV on CUDA cores (N <= 4; at 8
// and 16 rows the per-element x unpacking makes it FMA-bound and the tcgen05
// tiles win -- measured in the decode step).  Every warp owns whole rows, so
// there is no split-K and no cross-CTA reduction -- the kernel is a pure row
// stream.  A warp issues a whole 8 KB chunk of its row (16 x 16 B per lane)
// before consuming any of it, and its first chunk before x is staged, so at
// B = 1 (|S| ~ 1.6 K rows, >= one warp per row) the entire gathered matrix is
// in flight at once: one HBM round trip instead of the four serial 4 KB
// round trips of a two-rows-per-warp unroll-4 loop (6.6 -> 5.6 us alone).
// x is staged once per CTA in shared memory (rows >= N zero).  Positions in
// [count, round_up(count, pad)) are written as zeros, like the tile path.
constexpr int kGvThreads = 256;
constexpr int kGvChunk = 16;  // 16-byte loads in flight per lane

template <int NB>
__global__ void __launch_bounds__(kGvThreads) gemv_up_kernel(const uint16_t* __restrict__ w, int64_t w_ld,
                                                             const int32_t* __restrict__ idx,
                                                             const int32_t* __restrict__ count_dev, int M,
                                                             const uint16_t* __restrict__ x, int64_t x_ld, int N,
                                                             int K, const float* __restrict__ bias, int act,
                                                             void* out, int64_t out_ld, int out_bf16, int pad) {
  extern __shared__ __align__(16) uint4 sx4[];  // [NB][K / 8]
  const int kv = K >> 3;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  griddep_wait();  // x, idx and count come from the preceding kernels
  griddep_launch();
  const int count = count_dev ? min(__ldg(count_dev), M) : M;
  const int nw = gridDim.x * (kGvThreads / 32);
  int p = blockIdx.x * (kGvThreads / 32) + warp;
  uint4 a[kGvChunk];
  const uint4* wr = nullptr;
  int id = 0;
  auto load_chunk = [&](int c0) {
#pragma unroll
    for (int u = 0; u < kGvChunk; ++u) {
      const int c = c0 + lane + 32 * u;
      a[u] = c < kv ? __ldg(wr + c) : make_uint4(0, 0, 0, 0);
    }
  };
  if (p < count) {  // the first chunk streams in while x is staged
    id = idx ? __ldg(idx + p) : p;
    wr = reinterpret_cast<const uint4*>(w + (size_t)id * w_ld);
    load_chunk(0);
  }
  for (int i = threadIdx.x; i < NB * kv; i += kGvThreads) {
    const int b = i / kv, c = i - b * kv;
    sx4[i] = b < N ? __ldg(reinterpret_cast<const uint4*>(x + (size_t)b * x_ld) + c) : make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  for (; p < count; p += nw) {
    float acc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[b] = 0.f;
    for (int c0 = 0; c0 < kv; c0 += 32 * kGvChunk) {
      if (c0 > 0) load_chunk(c0);
#pragma unroll
      for (int u = 0; u < kGvChunk; ++u) {
        const int c = c0 + lane + 32 * u;
        if (c < kv) {
          float wa[8];
          unpack8(a[u], wa);
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            float xf[8];
            unpack8(sx4[b * kv + c], xf);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[b] = fmaf(wa[e], xf[e], acc[b]);
          }
        }
      }
    }
    const int id_done = id, p_done = p;
    if (p + nw < count) {  // next row's first chunk before this row's reduction
      id = idx ? __ldg(idx + p + nw) : p + nw;
      wr = reinterpret_cast<const uint4*>(w + (size_t)id * w_ld);
      load_chunk(0);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[b] = warp_sum(acc[b]);
    float v = 0.f;  // lane b stores batch row b
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if (lane == b) v = acc[b];
    if (lane < N) {
      v += bias ? __ldg(bias + id_done) : 0.f;
      if (act == PS_ACT_RELU) v = fmaxf(v, 0.f);
      const size_t o = (size_t)lane * out_ld + p_done;
      if (out_bf16) reinterpret_cast<uint16_t*>(out)[o] = f2bf(v);
      else reinterpret_cast<float*>(out)[o] = v;
    }
  }
  // zero the padding positions the next kernel may read
  const int pend = min((count + pad - 1) / pad * pad, (int)out_ld);
  for (int i = blockIdx.x * kGvThreads + threadIdx.x; i < (pend - count) * N; i += gridDim.x * kGvThreads) {
    const int b = i / (pend - count), pp = count + (i - b * (pend - count));
    if (out_bf16) reinterpret_cast<uint16_t*>(out)[(size_t)b * out_ld + pp] = 0;
    else reinterpret_cast<float*>(out)[(size_t)b * out_ld + pp] = 0.f;
  }
}

int g_gemv = -1;  // -1: from env PS_GG_GEMV (default 1): small-batch UP on the GEMV kernel

template <int NB>
int launch_gemv_up(const void* w, int64_t w_ld, const int32_t* idx, const int32_t* count_dev, int M, const void* x,
                   int64_t x_ld, int N, int K, const float* bias, int act, void* out, int64_t out_ld, int out_bf16,
                   cudaStream_t st) {
  const size_t smem = (size_t)NB * K * 2;
  static bool configured = false;
  static int occ_k = -1, occ = 1;
  if (!configured) {
    if (cudaFuncSetAttribute(gemv_up_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
        cudaSuccess)
      return PS_ERR_CUDA;
    configured = true;
  }
  if (occ_k != K) {  // resident CTAs per SM at this x footprint (registers bound it at small K)
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gemv_up_kernel<NB>, kGvThreads, smem) != cudaSuccess)
      return PS_ERR_CUDA;
    occ = n < 1 ? 1 : n;
    occ_k = K;
  }
  return launch_ex(gemv_up_kernel<NB>, dim3(ps_num_sms() * occ), dim3(kGvThreads), smem, st, 1,
                   static_cast<const uint16_t*>(w), w_ld, idx, count_dev, M, static_cast<const uint16_t*>(x), x_ld,
                   N, K, bias, act, out, out_ld, out_bf16, BM);
}

}  // namespace
}  // namespace ps

// PS_GG_BITMAP: `idx` is the union bitmap over the w_height weight rows
// (ceil(w_height / 32) uint32 words); the tcgen05 path with the cp.async A
// loaders derives the ids from it on the device.  UP writes the union size to
// count_dev (may be NULL); DOWN ignores count_dev.
static int gg_bitmap(GGParams& prm, const int32_t* idx, int32_t* count_out, int w_height, int rows_max) {
  if (!idx || g_lsu_mode < 1) return PS_ERR_UNSUPPORTED;
  const int words = (w_height + 31) / 32;
  if ((int64_t)words * 32 > (int64_t)rows_max + 31 || words > 1024) return PS_ERR_VALUE;
  prm.bm = reinterpret_cast<const uint32_t*>(idx);
  prm.bm_words = words;
  prm.count = nullptr;
  prm.count_out = count_out;
  return PS_OK;
}

extern "C" int ps_gather_gemm(const void* w_rows, int w_height, const int32_t* idx, const int32_t* count_dev,
                              const void* x, int64_t x_ld, const float* bias, const float* residual,
                              int64_t residual_ld, int N, int M, int K, int act, int splits, int flags, void* out,
                              int64_t out_ld, int out_dtype, void* ws, size_t ws_bytes, void* stream) {
  (void)ws; (void)ws_bytes;
  if (K % 8 || x_ld < K || out_ld < M) return PS_ERR_VALUE;
  GGParams prm;
  int st = gg_common(prm, w_rows, idx, count_dev, x, x_ld, bias, N, M, K, out, out_ld, out_dtype);
  if (st != PS_OK) return st;
  prm.w_ld = K;
  prm.act = act;
  prm.a_early = (!idx && !count_dev) || (flags & PS_GG_A_READY);
  prm.residual = residual;
  prm.res_ld = residual_ld;
  if (residual && ((residual_ld % 4) || ((uintptr_t)residual % 16))) prm.vec_ok = 0;
  if (w_height < (idx ? 1 : M)) return PS_ERR_VALUE;
  if (flags & PS_GG_BITMAP) {
    const int st2 = gg_bitmap(prm, idx, const_cast<int32_t*>(count_dev), w_height, M);
    if (st2 != PS_OK) return st2;
    const int rows_est = splits > 0 ? (splits < M ? splits : M) : M;
    return launch<MODE_UP>(prm, w_height, K, K, (rows_est + BM - 1) / BM, (K + BK - 1) / BK,
                           static_cast<cudaStream_t>(stream));
  }
  if (g_gemv < 0) {
    const char* e = getenv("PS_GG_GEMV");
    g_gemv = e ? atoi(e) : 1;
  }
  if (g_gemv && N <= 4 && !residual && (size_t)16 * K * 2 <= 200 * 1024 && x_ld % 8 == 0 &&
      ((uintptr_t)x % 16) == 0 && ((uintptr_t)w_rows % 16) == 0) {
    cudaStream_t s2 = static_cast<cudaStream_t>(stream);
    const int ob = out_dtype == PS_DTYPE_BF16;
    if (N <= 1) return launch_gemv_up<1>(w_rows, K, idx, count_dev, M, x, x_ld, N, K, bias, act, out, out_ld, ob, s2);
    if (N <= 2) return launch_gemv_up<2>(w_rows, K, idx, count_dev, M, x, x_ld, N, K, bias, act, out, out_ld, ob, s2);
    return launch_gemv_up<4>(w_rows, K, idx, count_dev, M, x, x_ld, N, K, bias, act, out, out_ld, ob, s2);
  }
  const int rows_est = splits > 0 ? (splits < M ? splits : M) : M;
  return launch<MODE_UP>(prm, w_height, K, K, (rows_est + BM - 1) / BM, (K + BK - 1) / BK,
                         static_cast<cudaStream_t>(stream));
}

extern "C" int ps_gather_gemm_t(const void* w_rows, int w_height, const int32_t* idx, const int32_t* count_dev,
                                const void* h, int64_t h_ld, const float* bias, const float* residual,
                                int64_t residual_ld, int N, int M, int K_max, int splits, int flags, void* out,
                                int64_t out_ld, int out_dtype, void* ws, size_t ws_bytes, void* stream) {
  (void)ws; (void)ws_bytes;
  if (M % 8 || h_ld < K_max || out_ld < M) return PS_ERR_VALUE;
  GGParams prm;
  int st = gg_common(prm, w_rows, idx, count_dev, h, h_ld, bias, N, M, K_max, out, out_ld, out_dtype);
  if (st != PS_OK) return st;
  prm.w_ld = M;
  prm.a_early = (!idx && !count_dev) || (flags & PS_GG_A_READY);
  prm.residual = residual;
  prm.res_ld = residual_ld;
  if (residual && ((residual_ld % 4) || ((uintptr_t)residual % 16))) prm.vec_ok = 0;
  if (w_height < (idx ? 1 : K_max)) return PS_ERR_VALUE;
  if (flags & PS_GG_BITMAP) {
    const int st2 = gg_bitmap(prm, idx, nullptr, w_height, K_max);
    if (st2 != PS_OK) return st2;
  }
  // the K extent (union size) is read on the device; `splits` > 0 is its expected value
  const int k_est = splits > 0 ? (splits < K_max ? splits : K_max) : K_max;
  return launch<MODE_DOWN>(prm, w_height, M, K_max, (M + BM - 1) / BM, (k_est + BK - 1) / BK,
                           static_cast<cudaStream_t>(stream));
}

// Debug hooks (tools/kbench.py): trace buffer of 16 u64 per CTA (start, setup
// done, first stage landed, last MMA issued, epilogue done, end, -, smid,
// first accumulator ready, first tile finished), and overrides of the
// pipeline depth / CTA slots (0 = default).
extern "C" void ps_debug_gemm_trace(void* buf, int stages, int target_ctas) {
  g_trace = static_cast<unsigned long long*>(buf);
  g_stages_override = stages;
  g_target_override = target_ctas;
}

// A-operand copy engine: 0 = TMA only, 1 = LSU for gathered rows (default),
// 2 = LSU for every A operand.
extern "C" void ps_debug_gemm_lsu_mode(int mode) { g_lsu_mode = mode; }
extern "C" void ps_debug_gemm_gemv(int enable) { g_gemv = enable ? 1 : 0; }
