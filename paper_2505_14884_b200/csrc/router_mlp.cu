// The MLP router (routers.py:286-288) as ONE persistent tcgen05 launch:
//
//   hid    = relu(h W_in + b_in)     bf16 (B, r)
//   logits = hid W_out (+ b_out)     f32  (B, D)
//
// Decode routers are weight streams with tiny outputs (r = 1024 hidden units,
// B <= 128 rows), so the cost is latency: two dependent GEMMs, each with a
// launch prologue, and W_in's K = d contraction split across CTAs.  Here:
//   * grid = one CTA per W_out row tile (128 logit columns, <= #SMs), one CTA
//     per SM (> 114 KB of shared memory), every CTA co-resident;
//   * the weights are static: each CTA's W_in slice (<= 4 K-blocks of one
//     128-row hidden tile) and the first kRStages K-blocks of its W_out tile
//     are TMA-loaded BEFORE griddepcontrol.wait, overlapping the previous
//     kernel (LayerNorm);
//   * phase 1: W_in split-K over (tile, slice) CTAs; every CTA writes its f32
//     partial (TMEM -> coalesced stores) to a workspace, passes a grid barrier,
//     then reduces 4 consecutive hidden units of one row per thread (all
//     slices, bias, ReLU) into hid (bf16);
//   * second grid barrier, then phase 2: the TMA producer streams hid (the B
//     operand, from L2) behind the prefetched W_out stages and the rest of
//     W_out; the epilogue writes logits (+ b_out) straight from TMEM.
// The grid barrier is a monotonic 64-bit counter (grid_arrive / grid_wait).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace ps {
namespace {

constexpr int RBM = 128;        // UMMA M (weight rows per tile)
constexpr int RBK = 64;         // K elements per stage (one 128-byte swizzle row)
constexpr int kRThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kREpi = 128;
constexpr int kRA1 = 4;       // phase-1 A K-blocks per CTA (64 KB)
constexpr int kRStages = 12;  // phase-2 pipeline stages (at most: as many as the shared memory holds)

struct GridBar {
  unsigned long long count;  // monotonic: every barrier adds exactly kBarUnit
  unsigned long long pad[15];
};
constexpr unsigned long long kBarUnit = 1ull << 20;  // > any grid size

struct RParams {
  int B, NB, d, r, D;
  int tiles1, slices1, kb1, tiles2;
  int stages;  // phase-2 pipeline depth (<= kRStages)
  const float* b_in;
  const float* b_out;
  float* part;  // [slices1][NB][r] f32 phase-1 partials
  uint16_t* hid;
  int64_t hid_ld;
  float* logits;
  int64_t lg_ld;
  GridBar* bar;
  unsigned long long* trace;
};

PS_DEV unsigned long long r_time() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}


PS_DEV void fence_proxy_async_global_r() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Grid barrier (one thread per CTA) on a monotonic 64-bit counter: CTA 0
// adds kBarUnit - (n - 1), every other CTA adds 1, so each barrier advances
// it by exactly kBarUnit whatever the grid size, and barrier k of a launch
// whose counter started at `base` has completed once count >= base + k *
// kBarUnit.  Arrival is a fire-and-forget release reduction and the waiters
// poll the counter itself: no last-arriver atomic round trip, reset store or
// second release on the critical path (2.4 / 1.8 -> 1.8 / 1.0 us, B = 1).
// `base` = count rounded down to a kBarUnit multiple, read before the CTA's
// first arrival: until barrier 1 completes the partial sums stay below it.

PS_DEV unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

PS_DEV void grid_wait(const GridBar* bar, unsigned long long target) {
  while (ld_acquire_u64(&bar->count) < target) __nanosleep(20);
}

// Called by one thread after a CTA barrier: the release is cumulative over
// the writes the barrier ordered before it (as in a cooperative grid sync).
PS_DEV void grid_arrive(GridBar* bar, int cta, int nctas) {
  const unsigned long long add = cta == 0 ? kBarUnit - (unsigned long long)(nctas - 1) : 1ull;
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(&bar->count), "l"(add) : "memory");
}

__global__ void __launch_bounds__(kRThreads, 1)
    router_mlp_kernel(const __grid_constant__ CUtensorMap tmWin, const __grid_constant__ CUtensorMap tmH,
                      const __grid_constant__ CUtensorMap tmWout, const __grid_constant__ CUtensorMap tmHid,
                      const RParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NB = p.NB;
  const uint32_t a_bytes = RBM * RBK * 2;            // 16 KB
  const uint32_t b_bytes = (uint32_t)NB * RBK * 2;   // NB * 128 B (a multiple of 2 KB)
  const uint32_t stage_bytes = a_bytes + b_bytes;
  uint8_t* A1 = smem;
  uint8_t* B1 = A1 + kRA1 * a_bytes;
  uint8_t* ST = B1 + kRA1 * b_bytes;
  const int S2 = p.stages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ST + S2 * stage_bytes);
  uint64_t* a1full = bars;
  uint64_t* b1full = bars + 1;
  uint64_t* p1done = bars + 2;
  uint64_t* full = bars + 3;
  uint64_t* empty = full + kRStages;
  uint64_t* p2done = empty + kRStages;
  uint64_t* genbar = p2done + 1;  // the producer read this launch's barrier generation
  uint64_t* xfull = genbar + 1;   // [kRA1] phase-2 K-blocks S2 .. S2+3 in the phase-1 buffers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfull + kRA1);
  unsigned long long& s_base = reinterpret_cast<unsigned long long*>(tmem_slot)[1];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x, nctas = gridDim.x;
  unsigned long long* tr = p.trace ? p.trace + 16 * (size_t)cta : nullptr;
  if (tr && tid == 0) tr[0] = r_time();

  // phase-1 item: (hidden tile t1, K slice s1), K blocks [k1lo, k1lo + n1)
  const bool has1 = cta < p.tiles1 * p.slices1;
  const int t1 = has1 ? cta / p.slices1 : 0, s1 = has1 ? cta % p.slices1 : 0;
  const int k1lo = (int)((long long)s1 * p.kb1 / p.slices1);
  const int n1 = has1 ? (int)((long long)(s1 + 1) * p.kb1 / p.slices1) - k1lo : 0;
  const int t2 = cta;  // phase-2 tile (grid == tiles2)
  const int kb2 = p.r / RBK;
  const uint32_t tcols = NB <= 16 ? 32 : (NB <= 32 ? 64 : (NB <= 64 ? 128 : (NB <= 128 ? 256 : 512)));

  if (warp == 1) {
    if (lane == 0) {
      mbar_init(a1full, 1);
      mbar_init(b1full, 1);
      mbar_init(p1done, 1);
      for (int s = 0; s < S2; ++s) {
        mbar_init(&full[s], 2);  // A and B arrive separately (A may be prefetched)
        mbar_init(&empty[s], 1);
      }
      mbar_init(p2done, 1);
      mbar_init(genbar, 1);
      for (int i = 0; i < kRA1; ++i) mbar_init(&xfull[i], 2);
      fence_mbar_init();
    }
    __syncwarp();
    tmem_alloc(tmem_slot, tcols);
  } else if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmWin);
    prefetch_tmap(&tmH);
    prefetch_tmap(&tmWout);
    prefetch_tmap(&tmHid);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0) griddep_launch();

  if (warp == 0) {
    if (lane == 0) {
      // ---- static weights first (overlap the previous kernel)
      if (has1) {
        mbar_arrive_expect_tx(a1full, (uint32_t)n1 * a_bytes);
        for (int i = 0; i < n1; ++i) tma_load_2d(A1 + i * a_bytes, &tmWin, (k1lo + i) * RBK, t1 * RBM, a1full);
      }
      const int pre = kb2 < S2 ? kb2 : S2;
      for (int s = 0; s < pre; ++s) {
        mbar_arrive_expect_tx(&full[s], a_bytes);
        tma_load_2d(ST + s * stage_bytes, &tmWout, s * RBK, t2 * RBM, &full[s]);
      }
      if (tr) tr[1] = r_time();
      griddep_wait();  // h comes from the previous kernel
      // barrier base of this launch: read after the previous grid (possibly the
      // previous launch of this kernel on the same workspace) completed, and
      // before this CTA arrives (so barrier 1 cannot have completed)
      const unsigned long long base = ld_acquire_u64(&p.bar->count) / kBarUnit * kBarUnit;
      if (tr) tr[7] = r_time();
      s_base = base;
      mbar_arrive(genbar);
      if (has1) {
        mbar_arrive_expect_tx(b1full, (uint32_t)n1 * b_bytes);
        for (int i = 0; i < n1; ++i) tma_load_2d(B1 + i * b_bytes, &tmH, (k1lo + i) * RBK, 0, b1full);
      }
      // the phase-1 buffers become phase-2 slots S2 .. S2+3 once the phase-1
      // MMAs have read them: more of W_out in flight before hid exists
      const int nx = kb2 - S2 < kRA1 ? (kb2 - S2 > 0 ? kb2 - S2 : 0) : kRA1;
      if (has1) mbar_wait(p1done, 0);
      for (int i = 0; i < nx; ++i) {
        mbar_arrive_expect_tx(&xfull[i], a_bytes);
        tma_load_2d(A1 + i * a_bytes, &tmWout, (S2 + i) * RBK, t2 * RBM, &xfull[i]);
      }
      // ---- phase 2: hid is complete after the second grid barrier
      grid_wait(p.bar, base + 2 * kBarUnit);
      if (tr) tr[4] = r_time();
      for (int kb = 0; kb < kb2; ++kb) {
        if (kb >= S2 && kb < S2 + nx) {  // a phase-1 buffer, used once
          const int i = kb - S2;
          mbar_arrive_expect_tx(&xfull[i], b_bytes);
          tma_load_2d(B1 + i * b_bytes, &tmHid, kb * RBK, 0, &xfull[i]);
          continue;
        }
        const int j = kb < S2 ? kb : kb - nx;  // position in the stage ring
        const int s = j % S2;
        uint8_t* sa = ST + s * stage_bytes;
        if (j >= S2) {
          mbar_wait(&empty[s], ((j / S2) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], a_bytes);
          tma_load_2d(sa, &tmWout, kb * RBK, t2 * RBM, &full[s]);
        }
        mbar_arrive_expect_tx(&full[s], b_bytes);
        tma_load_2d(sa + a_bytes, &tmHid, kb * RBK, 0, &full[s]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc_bf16(RBM, NB, 0, 0);
      if (has1) {
        mbar_wait(a1full, 0);
        mbar_wait(b1full, 0);
        tc_fence_after();
        for (int i = 0; i < n1; ++i) {
          const uint32_t sa = smem_u32(A1 + i * a_bytes), sb = smem_u32(B1 + i * b_bytes);
#pragma unroll
          for (int kk = 0; kk < RBK / 16; ++kk)
            umma_bf16(tmem, make_sdesc_sw128(sa + kk * 32, 16, 1024), make_sdesc_sw128(sb + kk * 32, 16, 1024),
                      idesc, (i > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(p1done);
        if (tr) tr[12] = r_time();
      }
      const uint32_t acc2 = tmem + (uint32_t)NB;
      const int nx = kb2 - S2 < kRA1 ? (kb2 - S2 > 0 ? kb2 - S2 : 0) : kRA1;
      for (int kb = 0; kb < kb2; ++kb) {
        uint32_t sa, sb;
        int s = -1;
        if (kb >= S2 && kb < S2 + nx) {
          const int i = kb - S2;
          mbar_wait(&xfull[i], 0);
          sa = smem_u32(A1 + i * a_bytes);
          sb = smem_u32(B1 + i * b_bytes);
        } else {
          const int j = kb < S2 ? kb : kb - nx;
          s = j % S2;
          mbar_wait(&full[s], (j / S2) & 1);
          sa = smem_u32(ST + s * stage_bytes);
          sb = sa + a_bytes;
        }
        tc_fence_after();
        if (tr && kb == 0) tr[8] = r_time();
        if (tr && kb == kb2 - 1) tr[9] = r_time();
#pragma unroll
        for (int kk = 0; kk < RBK / 16; ++kk)
          umma_bf16(acc2, make_sdesc_sw128(sa + kk * 32, 16, 1024), make_sdesc_sw128(sb + kk * 32, 16, 1024), idesc,
                    (kb > 0 || kk > 0) ? 1u : 0u);
        if (s >= 0) umma_commit(&empty[s]);
      }
      umma_commit(p2done);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue warps 2..5
    const int q = warp & 3;  // TMEM lane quadrant
    const int m = q * 32 + lane;
    const int et = tid - 64;
    // phase 1: my partial tile -> part[s1][n][t1*128 + m] (lanes = consecutive hidden units)
    if (has1) {
      mbar_wait(p1done, 0);
      tc_fence_after();
      if (tr && et == 0) tr[13] = r_time();
      float* dst = p.part + (size_t)s1 * NB * p.r + t1 * RBM + m;
      const bool live = t1 * RBM + m < p.r;
      for (int c0 = 0; c0 < NB; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_ld_wait();
        if (live) {
#pragma unroll
          for (int u = 0; u < 16; ++u)
            if (c0 + u < p.B) __stcg(dst + (size_t)(c0 + u) * p.r, __uint_as_float(v[u]));
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kREpi));
    unsigned long long base = 0;
    if (et == 0) {
      if (tr) tr[2] = r_time();
      mbar_wait(genbar, 0);
      base = s_base;
      grid_arrive(p.bar, cta, nctas);
      grid_wait(p.bar, base + kBarUnit);
      if (tr) tr[3] = r_time();
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kREpi));
    if (tr && et == 0) tr[10] = r_time();
    // reduce: 4 consecutive hidden units of one row per thread, every slice
    const int quads = p.B * (p.r >> 2);
    for (int g = cta * kREpi + et; g < quads; g += nctas * kREpi) {
      const int n = g / (p.r >> 2), j = (g - n * (p.r >> 2)) * 4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4* src = reinterpret_cast<const float4*>(p.part + (size_t)n * p.r + j);
      const size_t step = (size_t)NB * p.r / 4;
      for (int s0 = 0; s0 < p.slices1; s0 += 16) {  // 16 loads in flight, then the sums (slice order)
        float4 t[16];
#pragma unroll
        for (int s = 0; s < 16; ++s)
          t[s] = s0 + s < p.slices1 ? __ldcg(src + (s0 + s) * step) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int s = 0; s < 16; ++s) {
          acc.x += t[s].x; acc.y += t[s].y; acc.z += t[s].z; acc.w += t[s].w;
        }
      }
      const float4 b = p.b_in ? __ldg(reinterpret_cast<const float4*>(p.b_in + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
      uint2 pk;
      pk.x = pack_bf16x2(fmaxf(acc.x + b.x, 0.f), fmaxf(acc.y + b.y, 0.f));
      pk.y = pack_bf16x2(fmaxf(acc.z + b.z, 0.f), fmaxf(acc.w + b.w, 0.f));
      *reinterpret_cast<uint2*>(p.hid + (size_t)n * p.hid_ld + j) = pk;
    }
    fence_proxy_async_global_r();  // generic hid stores -> the other CTAs' TMA (async proxy) loads
    if (tr && et == 0) tr[11] = r_time();
    asm volatile("bar.sync 1, %0;" ::"n"(kREpi));
    if (et == 0) grid_arrive(p.bar, cta, nctas);
    // phase 2: logits tile straight from TMEM (lanes = consecutive logit columns)
    mbar_wait(p2done, 0);
    tc_fence_after();
    if (tr && et == 0) tr[5] = r_time();
    const int col = t2 * RBM + m;
    const bool live = col < p.D;
    const float bo = (live && p.b_out) ? __ldg(p.b_out + col) : 0.f;
    for (int c0 = 0; c0 < NB; c0 += 16) {
      uint32_t v[16];
      tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)NB + c0, v);
      tmem_ld_wait();
      if (live) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (c0 + u < p.B) p.logits[(size_t)(c0 + u) * p.lg_ld + col] = __uint_as_float(v[u]) + bo;
      }
    }
    if (tr && et == 0) tr[6] = r_time();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;

int rmap(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_rows) {
  if (!g_enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return PS_ERR_CUDA;
    g_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)RBK, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? PS_OK : PS_ERR_VALUE;
}

// phase-1 split: slices per hidden tile (<= kRA1 K-blocks each, tiles1 *
// slices1 <= grid); 0 = the shape is not supported
int r_slices(int tiles1, int kb1, int grid) {
  int s = grid / tiles1;
  if (s > kb1) s = kb1;
  if (s < 1 || (kb1 + s - 1) / s > kRA1) return 0;
  return s;
}

unsigned long long* g_router_trace = nullptr;

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" size_t ps_router_mlp_fused_workspace_bytes(int B, int d, int r, int D) {
  if (B < 1 || B > 128 || d < 64 || r < 128 || D < 1) return 0;  // B > 128: phase-1 buffers exceed shared memory
  const int NB = (B + 15) / 16 * 16;
  const int tiles1 = (r + RBM - 1) / RBM, grid = (D + RBM - 1) / RBM;
  if (grid > ps_num_sms()) return 0;
  const int s = r_slices(tiles1, d / RBK, grid);
  if (!s) return 0;
  return 256 + (size_t)s * NB * r * 4;
}

// Returns PS_ERR_UNSUPPORTED for shapes outside the fused kernel (B > 128,
// D > 128 * #SMs, W_in slices of more than 4 K-blocks, d or r not a multiple of
// 64); the caller then runs the two GEMMs separately.
extern "C" int ps_router_mlp_fused(const void* w_in_t, const float* b_in, const void* w_out_t, const float* b_out,
                                   int d, int r, int D, const void* x, int64_t x_ld, int B, void* hid,
                                   int64_t hid_ld, float* logits, int64_t lg_ld, void* ws, size_t ws_bytes,
                                   void* stream) {
  if (!w_in_t || !w_out_t || !x || !hid || !logits || !ws || B < 1 || d < 1 || r < 1 || D < 1) return PS_ERR_VALUE;
  if (x_ld < d || hid_ld < r || lg_ld < D || x_ld % 8 || hid_ld % 8) return PS_ERR_VALUE;
  if (B > 128 || d % RBK || r % RBM || (D + RBM - 1) / RBM > ps_num_sms()) return PS_ERR_UNSUPPORTED;
  const size_t need = ps_router_mlp_fused_workspace_bytes(B, d, r, D);
  if (!need) return PS_ERR_UNSUPPORTED;
  if (ws_bytes < need) return PS_ERR_WORKSPACE;
  if (((uintptr_t)x | (uintptr_t)hid | (uintptr_t)w_in_t | (uintptr_t)w_out_t) % 16) return PS_ERR_VALUE;
  RParams prm{};
  prm.B = B;
  prm.NB = (B + 15) / 16 * 16;
  prm.d = d; prm.r = r; prm.D = D;
  prm.tiles1 = r / RBM;
  prm.kb1 = d / RBK;
  prm.tiles2 = (D + RBM - 1) / RBM;
  prm.slices1 = r_slices(prm.tiles1, prm.kb1, prm.tiles2);
  prm.b_in = b_in; prm.b_out = b_out;
  prm.bar = static_cast<GridBar*>(ws);
  prm.part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + 256);
  prm.hid = static_cast<uint16_t*>(hid); prm.hid_ld = hid_ld;
  prm.logits = logits; prm.lg_ld = lg_ld;
  prm.trace = g_router_trace;
  CUtensorMap tWin, tH, tWout, tHid;
  int rc;
  if ((rc = rmap(&tWin, w_in_t, d, r, d, RBM)) != PS_OK) return rc;
  if ((rc = rmap(&tH, x, d, B, x_ld, prm.NB)) != PS_OK) return rc;
  if ((rc = rmap(&tWout, w_out_t, r, D, r, RBM)) != PS_OK) return rc;
  if ((rc = rmap(&tHid, hid, r, B, hid_ld, prm.NB)) != PS_OK) return rc;
  const size_t stage = (size_t)RBM * RBK * 2 + (size_t)prm.NB * RBK * 2;
  const size_t fixed = 1024 + (size_t)kRA1 * stage + 512;  // + barriers (<= 35 x 8 B) and the TMEM slot
  prm.stages = fixed < 227 * 1024 ? (int)((227 * 1024 - fixed) / stage) : 0;
  if (prm.stages > kRStages) prm.stages = kRStages;
  if (prm.stages < 2) return PS_ERR_UNSUPPORTED;
  const size_t smem = fixed + (size_t)prm.stages * stage;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(router_mlp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) !=
        cudaSuccess)
      return PS_ERR_CUDA;
    configured = true;
  }
  // one CTA per SM: every CTA of the grid barrier is resident at once
  if (smem <= 114 * 1024) return PS_ERR_UNSUPPORTED;
  return launch_ex(router_mlp_kernel, dim3(prm.tiles2), dim3(kRThreads), smem, static_cast<cudaStream_t>(stream),
                   1, tWin, tH, tWout, tHid, prm);
}

extern "C" void ps_debug_router_trace(void* buf) { g_router_trace = static_cast<unsigned long long*>(buf); }
