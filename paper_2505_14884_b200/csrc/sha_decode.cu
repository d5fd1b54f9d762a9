// Select-Head Attention (SHA) split-KV decode for sm_100a.
//
// Semantics: sparsedecode.kernels.gqa_selective_attention_decode
// (kernels.py:513-548 -> _attention_over_units 386-444): for every sequence b
// and every selected KV group g = sel[b, j], the G = H/H_kv query heads
// g*G .. g*G+G-1 attend over K/V[b, g, :lengths[b]] with softmax scale
// `scale`; heads of non-selected groups are written as exact 0.0 and their
// cache rows are never read (NaN-poison safe).
//
// Design (B200-first, HBM-bound: ~G flop per KV byte):
//   * one CTA = one (b, g) unit x one KV split (FlashDecoding); grid sized to
//     several waves of 148 SMs x 3 resident CTAs;
//   * each selected (b, g) history is one contiguous slab of the
//     (B, H_kv, cap, d_h) cache, so K and V tiles (8 KB each) are staged into
//     shared memory by 1-D bulk async copies (TMA engine, `cp.async.bulk`)
//     behind a 4-stage mbarrier pipeline -- only valid rows are copied;
//   * 128-bit shared-memory reads: each lane owns 8 head dims of a row,
//     d_h/8 lanes per row; G query heads held in registers, pre-scaled by
//     scale*log2(e) so the softmax runs on ex2;
//   * online softmax per warp (one rescale per tile), warp/CTA merges in
//     registers/smem, per-split (m, l, o) partials merged by the last CTA of
//     the unit (atomic ticket; counters self-reset, so the call is graph-safe);
//   * B extra CTAs write the exact zeros of the non-selected heads.
#include "common.cuh"

namespace ps {
namespace {

constexpr int kThreads = 128;
constexpr int kWarps = 4;
constexpr int kStages = 4;
constexpr int kTileBytes = 8192;  // bytes of one K (or V) tile
// Fixed-size ticket region at the head of the workspace: its layout must not
// depend on the launch shape, or a previous launch's partials would alias
// another shape's tickets (they are only zero where the last CTA reset them).
constexpr int kMaxUnits = 65536;
constexpr size_t kCounterBytes = (size_t)kMaxUnits * 4;

template <int D_H>
struct ShaShape {
  static constexpr int LPR = D_H / 8;                    // lanes per row
  static constexpr int RPW = 32 / LPR;                   // rows per warp pass
  static constexpr int T = kTileBytes / (D_H * 2);       // rows per tile
  static constexpr int ROWS_PER_WARP = T / kWarps;
  static constexpr int PASSES = ROWS_PER_WARP / RPW;
  static_assert(PASSES * RPW * kWarps == T, "tile geometry");
};

struct ShaParams {
  const uint16_t* q;
  int64_t q_ld;
  const uint16_t* k;
  const uint16_t* v;
  const int32_t* lengths;
  const int32_t* sel;
  int group_base;
  int B, H, H_kv, cap, top_k;
  int NT;        // virtual tiles per unit (>= ceil(max length / T))
  int n_ctas;    // stream-K CTAs (the B zero-fill CTAs follow them)
  int max_seg;   // partial slots per unit
  float scale_log2;
  void* out;
  int64_t out_ld;
  int* counters;
  float* partials;
};

template <int D_H, int G>
constexpr size_t sha_smem_bytes() {
  return 2 * kStages * kTileBytes + 64 + (size_t)kWarps * G * (D_H + 2) * 4 + 16;
}

template <bool BF16>
PS_DEV void store_out(void* out, size_t off, float v) {
  if (BF16)
    reinterpret_cast<uint16_t*>(out)[off] = f2bf(v);
  else
    reinterpret_cast<float*>(out)[off] = v;
}

// Stream-K: the flattened (unit, tile) space F = units x NT is cut into
// n_ctas equal contiguous ranges, one per CTA, so every CTA moves the same
// number of KV bytes (no tail wave).  A CTA walks its range unit segment by
// unit segment with ONE continuous TMA pipeline; a unit covered by several
// CTAs gets per-segment partials (m, l, o) merged by the last arriving
// segment in segment order (deterministic).  Tiles beyond a sequence's
// length are empty pipeline slots (plain arrive, nothing read).
PS_DEV int cta_of(long long f, long long F, int n) { return (int)(((f + 1) * n - 1) / F); }

template <int D_H, int G, bool OUT_BF16>
__global__ void __launch_bounds__(kThreads) sha_decode_kernel(const ShaParams p) {
  using S = ShaShape<D_H>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint16_t* sK = reinterpret_cast<uint16_t*>(smem);
  uint16_t* sV = sK + kStages * S::T * D_H;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kStages * kTileBytes);
  float* red = reinterpret_cast<float*>(smem + 2 * kStages * kTileBytes + 64);
  float* red_m = red;                            // [kWarps][G]
  float* red_l = red + kWarps * G;               // [kWarps][G]
  float* red_o = red + 2 * kWarps * G;           // [kWarps][G][D_H]
  int* flag = reinterpret_cast<int*>(red + kWarps * G * (D_H + 2));

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int n_units = p.B * p.top_k;
  const int bid = blockIdx.x;
  griddep_wait();  // q / KV / sel / lengths come from the preceding launches
  // (griddep_launch only after the main loop: with several waves of CTAs, an
  // early trigger lets the next grid's CTAs park on SM slots this grid needs)

  if (bid >= p.n_ctas) {
    // ---- zero-fill CTA for sequence b: heads of non-selected groups = 0.0
    const int b = bid - p.n_ctas;
    int* sel_flag = reinterpret_cast<int*>(smem);
    for (int g = tid; g < p.H_kv; g += kThreads) sel_flag[g] = 0;
    __syncthreads();
    for (int j = tid; j < p.top_k; j += kThreads) {
      int g = p.sel[(size_t)b * p.top_k + j] - p.group_base;
      if (g >= 0 && g < p.H_kv) sel_flag[g] = 1;
    }
    __syncthreads();
    const int total = p.H * D_H;
    for (int e = tid; e < total; e += kThreads) {
      int grp = (e / D_H) / G;
      if (!sel_flag[grp]) store_out<OUT_BF16>(p.out, (size_t)b * p.out_ld + e, 0.0f);
    }
    griddep_launch();
    return;
  }

  const long long F = (long long)n_units * p.NT;
  const long long f0 = (long long)bid * F / p.n_ctas, f1 = (long long)(bid + 1) * F / p.n_ctas;
  const int n_it = (int)(f1 - f0);

  // first unit's selection / length: loaded before the barrier setup so the
  // latency overlaps it (every thread needs them for its first segment)
  const int u_first = n_it > 0 ? (int)(f0 / p.NT) : 0;
  const int sel_first = __ldg(p.sel + u_first);
  const int len_first = __ldg(p.lengths + u_first / p.top_k);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // producer (thread 0): walks the flattened tiles in order with an
  // incremental (unit, tile) cursor -- the unit's slab / length are loaded
  // once per unit; empty tiles (beyond the length, other rank's group) just
  // arrive
  struct Cursor {
    int u, t, len;
    bool live;
    const uint16_t* kb;
    const uint16_t* vb;
  } cur;
  auto load_unit = [&](int u) {
    cur.u = u;
    const int b = u / p.top_k;
    const int g = (u == u_first ? sel_first : __ldg(p.sel + u)) - p.group_base;
    cur.live = g >= 0 && g < p.H_kv;
    cur.len = u == u_first ? len_first : __ldg(p.lengths + b);
    const size_t slab = ((size_t)b * p.H_kv + (cur.live ? g : 0)) * (size_t)p.cap * D_H;
    cur.kb = p.k + slab;
    cur.vb = p.v + slab;
  };
  auto issue_next = [&](int stage) {
    const int row0 = cur.t * S::T;
    if (!cur.live || row0 >= cur.len) {
      mbar_arrive(&bars[stage]);
    } else {
      const int rows = min(S::T, cur.len - row0);
      const uint32_t bytes = (uint32_t)rows * D_H * 2;
      mbar_arrive_expect_tx(&bars[stage], 2 * bytes);
      bulk_g2s(sK + stage * S::T * D_H, cur.kb + (size_t)row0 * D_H, bytes, &bars[stage]);
      bulk_g2s(sV + stage * S::T * D_H, cur.vb + (size_t)row0 * D_H, bytes, &bars[stage]);
    }
    if (++cur.t == p.NT) {  // advance the cursor
      cur.t = 0;
      if (cur.u + 1 < n_units) load_unit(cur.u + 1);
    }
  };
  if (tid == 0 && n_it > 0) {
    const int u0 = (int)(f0 / p.NT);
    load_unit(u0);
    cur.t = (int)(f0 - (long long)u0 * p.NT);
    const int pre = min(kStages, n_it);
    for (int s2 = 0; s2 < pre; ++s2) issue_next(s2);
  }

  const int c = lane % S::LPR;   // 16-byte column chunk owned by this lane
  const int slot = lane / S::LPR;
  int it = 0;
  long long f = f0;
  while (f < f1) {
    const int u = (int)(f / p.NT);
    const long long u_end = (long long)(u + 1) * p.NT;
    const long long seg_end = f1 < u_end ? f1 : u_end;
    const int b = u / p.top_k;
    const int g = (u == u_first ? sel_first : __ldg(p.sel + u)) - p.group_base;
    const bool live = g >= 0 && g < p.H_kv;  // another rank's group (or invalid): never read
    const int len = u == u_first ? len_first : __ldg(p.lengths + b);

    // ---- queries of the group, 8 dims per lane, pre-scaled for exp2
    float qf[G][8];
    float m_run[G], l_run[G], o[G][8];
    if (live) {
      const uint16_t* qb = p.q + (size_t)b * p.q_ld + (size_t)g * G * D_H + c * 8;
#pragma unroll
      for (int h = 0; h < G; ++h) {
        uint4 raw = *reinterpret_cast<const uint4*>(qb + h * D_H);
        unpack8(raw, qf[h]);
#pragma unroll
        for (int i = 0; i < 8; ++i) qf[h][i] *= p.scale_log2;
      }
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
      m_run[h] = -INFINITY;
      l_run[h] = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) o[h][i] = 0.f;
    }

    const int nt_seg = (int)(seg_end - f);
    const int t0 = (int)(f - (long long)u * p.NT);
    f = seg_end;
    if (!live) {  // another rank's group: only keep the pipeline moving
      for (int k2 = 0; k2 < nt_seg; ++k2, ++it) {
        const int stage = it % kStages;
        mbar_wait(&bars[stage], (it / kStages) & 1);
        __syncthreads();
        if (tid == 0 && it + kStages < n_it) issue_next(stage);
      }
      continue;
    }
    // tiles of this segment that hold rows (the rest are empty pipeline slots)
    const int nt_real = max(0, min(nt_seg, (len + S::T - 1) / S::T - t0));
    for (int k2 = 0; k2 < nt_seg; ++k2, ++it) {
      const int stage = it % kStages;
      mbar_wait(&bars[stage], (it / kStages) & 1);
      if (k2 < nt_real) {
        const int row0 = (t0 + k2) * S::T;
        const int valid = min(S::T, len - row0);
        const uint16_t* tk = sK + stage * S::T * D_H;
        const uint16_t* tv = sV + stage * S::T * D_H;
        float s_[S::PASSES][G];
#pragma unroll
        for (int ps_ = 0; ps_ < S::PASSES; ++ps_) {
          const int r = warp * S::ROWS_PER_WARP + ps_ * S::RPW + slot;
          float kf[8];
          const bool ok = r < valid;
          if (ok) {
            uint4 raw = *reinterpret_cast<const uint4*>(tk + r * D_H + c * 8);
            unpack8(raw, kf);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) kf[i] = 0.f;
          }
#pragma unroll
          for (int h = 0; h < G; ++h) {
            float acc = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) acc = fmaf(qf[h][i], kf[i], acc);
#pragma unroll
            for (int off = 1; off < S::LPR; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            s_[ps_][h] = ok ? acc : -INFINITY;
          }
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
          float mx = s_[0][h];
#pragma unroll
          for (int ps_ = 1; ps_ < S::PASSES; ++ps_) mx = fmaxf(mx, s_[ps_][h]);
#pragma unroll
          for (int off = S::LPR; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
          const float m_new = fmaxf(m_run[h], mx);
          const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
          const float alpha = fast_exp2(m_run[h] - m_use);
          float lsum = 0.f;
#pragma unroll
          for (int ps_ = 0; ps_ < S::PASSES; ++ps_) {
            s_[ps_][h] = fast_exp2(s_[ps_][h] - m_use);
            lsum += s_[ps_][h];
          }
          l_run[h] = l_run[h] * alpha + lsum;
#pragma unroll
          for (int i = 0; i < 8; ++i) o[h][i] *= alpha;
          m_run[h] = m_new;
        }
#pragma unroll
        for (int ps_ = 0; ps_ < S::PASSES; ++ps_) {
          const int r = warp * S::ROWS_PER_WARP + ps_ * S::RPW + slot;
          if (r < valid) {
            float vf[8];
            uint4 raw = *reinterpret_cast<const uint4*>(tv + r * D_H + c * 8);
            unpack8(raw, vf);
#pragma unroll
            for (int h = 0; h < G; ++h)
#pragma unroll
              for (int i = 0; i < 8; ++i) o[h][i] = fmaf(s_[ps_][h], vf[i], o[h][i]);
          }
        }
      }
      __syncthreads();  // every warp is done with this stage
      if (tid == 0 && it + kStages < n_it) issue_next(stage);
    }

    // ---- merge row slots inside the warp (same m_run across the warp)
#pragma unroll
    for (int h = 0; h < G; ++h) {
#pragma unroll
      for (int off = S::LPR; off < 32; off <<= 1) {
        l_run[h] += __shfl_xor_sync(0xffffffffu, l_run[h], off);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[h][i] += __shfl_xor_sync(0xffffffffu, o[h][i], off);
      }
    }
    if (slot == 0) {
#pragma unroll
      for (int h = 0; h < G; ++h)
#pragma unroll
        for (int i = 0; i < 8; ++i) red_o[(warp * G + h) * D_H + c * 8 + i] = o[h][i];
      if (lane == 0) {
#pragma unroll
        for (int h = 0; h < G; ++h) {
          red_m[warp * G + h] = m_run[h];
          red_l[warp * G + h] = l_run[h];
        }
      }
    }
    __syncthreads();

    // ---- merge warps; a unit inside one CTA writes its output directly
    const int c_first = cta_of((long long)u * p.NT, F, p.n_ctas);
    const int c_last = cta_of(u_end - 1, F, p.n_ctas);
    const int nseg = c_last - c_first + 1, seg = bid - c_first;
    const size_t out_row = (size_t)b * p.out_ld + (size_t)g * G * D_H;
    const int stride = G * (D_H + 2);
    float* part = p.partials + ((size_t)u * p.max_seg + seg) * (size_t)stride;
    for (int e = tid; e < G * D_H; e += kThreads) {
      const int h = e / D_H;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) M = fmaxf(M, red_m[w * G + h]);
      float L = 0.f, O = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const float mw = red_m[w * G + h];
        const float wt = (mw == -INFINITY) ? 0.f : fast_exp2(mw - M);
        L += red_l[w * G + h] * wt;
        O += red_o[(w * G) * D_H + e] * wt;
      }
      if (nseg == 1) {
        store_out<OUT_BF16>(p.out, out_row + e, O / L);
      } else {
        part[2 * G + e] = O;
        if ((e % D_H) == 0) {
          part[h] = M;
          part[G + h] = L;
        }
      }
    }
    if (nseg > 1) {
      // ---- last arriving segment merges the unit's partials (segment order)
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        const int prev = atomicAdd(&p.counters[u], 1);
        *flag = (prev == nseg - 1);
      }
      __syncthreads();
      if (*flag) {
        __threadfence();
        const float* base = p.partials + (size_t)u * p.max_seg * (size_t)stride;
        for (int e = tid; e < G * D_H; e += kThreads) {
          const int h = e / D_H;
          float M = -INFINITY;
          for (int s2 = 0; s2 < nseg; ++s2) M = fmaxf(M, __ldcg(base + s2 * stride + h));
          float L = 0.f, O = 0.f;
          for (int s2 = 0; s2 < nseg; ++s2) {
            const float ms = __ldcg(base + s2 * stride + h);
            const float wt = (ms == -INFINITY) ? 0.f : fast_exp2(ms - M);
            L += __ldcg(base + s2 * stride + G + h) * wt;
            O += __ldcg(base + s2 * stride + 2 * G + e) * wt;
          }
          store_out<OUT_BF16>(p.out, out_row + e, O / L);
        }
        if (tid == 0) p.counters[u] = 0;  // self-reset for the next launch / graph replay
      }
    }
    __syncthreads();  // red_* / flag reused by the next segment
  }
  griddep_launch();
}

template <int D_H, int G, bool BF16>
int launch_sha(const ShaParams& prm, int grid, cudaStream_t st) {
  constexpr size_t smem = sha_smem_bytes<D_H, G>();
  auto kern = sha_decode_kernel<D_H, G, BF16>;
  static bool configured = false;  // per-instantiation, per-process
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return PS_ERR_CUDA;
    configured = true;
  }
  return launch_ex(kern, dim3(grid), dim3(kThreads), smem, st, 1, prm);
}

template <int D_H, int G>
int dispatch_dtype(const ShaParams& prm, int grid, bool bf16, cudaStream_t st) {
  return bf16 ? launch_sha<D_H, G, true>(prm, grid, st) : launch_sha<D_H, G, false>(prm, grid, st);
}

template <int D_H>
int dispatch_g(const ShaParams& prm, int grid, int G, bool bf16, cudaStream_t st) {
  switch (G) {
    case 1: return dispatch_dtype<D_H, 1>(prm, grid, bf16, st);
    case 2: return dispatch_dtype<D_H, 2>(prm, grid, bf16, st);
    case 4: return dispatch_dtype<D_H, 4>(prm, grid, bf16, st);
    case 8:
      if constexpr (D_H <= 128) return dispatch_dtype<D_H, 8>(prm, grid, bf16, st);
      return PS_ERR_UNSUPPORTED;
    default: return PS_ERR_UNSUPPORTED;
  }
}

int partial_floats(int G, int d_h) { return G * (d_h + 2); }

// resident SHA CTAs (64 KB of K/V stages each: 3 per SM)
int sha_slots() { return ps_num_sms() * 3; }

// stream-K CTAs: num_splits > 0 caps them at units * num_splits (the classic
// FlashDecoding split count); 0 = one resident wave (every SM streaming)
int sha_ctas(int units, int NT, int num_splits) {
  long long cap = num_splits > 0 ? (long long)units * num_splits : (long long)sha_slots();
  const long long F = (long long)units * NT;
  if (cap > F) cap = F;
  return (int)(cap < 1 ? 1 : cap);
}

// segments per unit: ranges hold >= floor(F/n) >= F/(2n) tiles (F >= n), so a
// unit of NT = F/units tiles meets at most ceil(2n/units) + 1 of them
int sha_max_seg(int units, int n_ctas) { return (2 * n_ctas + units - 1) / units + 1; }


}  // namespace
}  // namespace ps

using namespace ps;

extern "C" size_t ps_sha_workspace_bytes(int B, int H, int H_kv, int d_h, int top_k, int num_splits) {
  if (B < 1 || H_kv < 1 || top_k < 1 || H % H_kv) return 0;
  const size_t units = (size_t)B * top_k;
  const int n = num_splits > 0 ? (int)(units * num_splits) : sha_slots();  // upper bound of sha_ctas
  return kCounterBytes + units * (size_t)sha_max_seg((int)units, n) * (size_t)partial_floats(H / H_kv, d_h) * 4;
}

// 0 = stream-K over one resident wave (the default)
extern "C" int ps_sha_auto_splits(int B, int H_kv, int d_h, int top_k, int max_len) {
  (void)B; (void)H_kv; (void)d_h; (void)top_k; (void)max_len;
  return 0;
}

extern "C" int ps_sha_decode(const void* q, int64_t q_ld, const void* k_cache, const void* v_cache,
                             const int32_t* lengths, const int32_t* sel, int group_base, int B, int H, int H_kv,
                             int cap,
                             int d_h, int top_k, float scale, int num_splits, int max_len_hint, void* out,
                             int64_t out_ld, int out_dtype, void* ws, size_t ws_bytes, void* stream) {
  if (B < 1 || H < 1 || H_kv < 1 || cap < 1 || top_k < 1 || group_base < 0) return PS_ERR_VALUE;
  if (H % H_kv) return PS_ERR_VALUE;
  if ((int64_t)B * top_k > kMaxUnits) return PS_ERR_UNSUPPORTED;
  if (!(scale > 0.f)) return PS_ERR_VALUE;
  if (q_ld < (int64_t)H * d_h || out_ld < (int64_t)H * d_h) return PS_ERR_VALUE;
  if (!q || !k_cache || !v_cache || !lengths || !sel || !out || !ws) return PS_ERR_VALUE;
  if ((q_ld * 2) % 16 || ((uintptr_t)q % 16) || ((uintptr_t)k_cache % 16) || ((uintptr_t)v_cache % 16))
    return PS_ERR_VALUE;
  if (d_h < 8 || d_h > 256 || (d_h & (d_h - 1))) return PS_ERR_UNSUPPORTED;
  const int G = H / H_kv;
  if (num_splits < 0) num_splits = 0;
  if (ws_bytes < ps_sha_workspace_bytes(B, H, H_kv, d_h, top_k, num_splits)) return PS_ERR_WORKSPACE;
  // max_len_hint must bound every lengths[b]: rows beyond NT tiles are not read
  const int T = kTileBytes / (d_h * 2);
  int max_len = max_len_hint > 0 ? max_len_hint : cap;
  if (max_len > cap) max_len = cap;
  const int NT = (max_len + T - 1) / T > 0 ? (max_len + T - 1) / T : 1;
  const int units = B * top_k;
  ShaParams prm;
  prm.q = static_cast<const uint16_t*>(q);
  prm.q_ld = q_ld;
  prm.k = static_cast<const uint16_t*>(k_cache);
  prm.v = static_cast<const uint16_t*>(v_cache);
  prm.lengths = lengths;
  prm.sel = sel;
  prm.group_base = group_base;
  prm.B = B; prm.H = H; prm.H_kv = H_kv; prm.cap = cap; prm.top_k = top_k;
  prm.NT = NT;
  prm.n_ctas = sha_ctas(units, NT, num_splits);
  prm.max_seg = sha_max_seg(units, prm.n_ctas);
  prm.scale_log2 = scale * kLog2e;
  prm.out = out;
  prm.out_ld = out_ld;
  prm.counters = static_cast<int*>(ws);
  prm.partials = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kCounterBytes);
  const int grid = prm.n_ctas + B;
  const bool bf16 = out_dtype == PS_DTYPE_BF16;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (d_h) {
    case 8: return dispatch_g<8>(prm, grid, G, bf16, st);
    case 16: return dispatch_g<16>(prm, grid, G, bf16, st);
    case 32: return dispatch_g<32>(prm, grid, G, bf16, st);
    case 64: return dispatch_g<64>(prm, grid, G, bf16, st);
    case 128: return dispatch_g<128>(prm, grid, G, bf16, st);
    case 256: return dispatch_g<256>(prm, grid, G, bf16, st);
    default: return PS_ERR_UNSUPPORTED;
  }
}
