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
#include <cmath>
#include <cuda.h>
#include <cudaTypedefs.h>

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
  // paged KV (ps_sha_decode_paged): logical row r of sequence b lives in
  // physical page table[b * table_ld + r / page_rows], row r % page_rows, of
  // a (pages, H_kv, page_rows, d_h) pool; NULL = contiguous (B, H_kv, cap, d_h)
  const int32_t* table;
  int64_t table_ld;
  int page_rows;
  int pool_pages;
  // virtual tiles per unit.  The partition uses NT = ceil(max_b lengths[b] / T)
  // read from the DEVICE lengths by every CTA (so a captured graph stays
  // exact as the sequences grow); NT_hint (from the host's length mirror)
  // only sizes the grid and lets a CTA prefetch its first unit's metadata
  // before the lengths are reduced
  int NT_hint;
  int NT_cap;    // ceil(cap / T)
  int n_ctas;    // stream-K CTAs (the B zero-fill CTAs follow them)
  int max_seg;   // partial slots per unit
  float scale_log2;
  void* out;
  int64_t out_ld;
  int* counters;
  float* partials;
  unsigned long long* trace;  // debug (ps_debug_sha_trace): 8 u64 per CTA, NULL normally
  int zero_inline;  // tensor-core kernel: the stream-K CTAs zero the unselected heads themselves (no B extra CTAs)
};

// Physical row of logical row `row0` of unit (b, g) in the row view of the
// cache: (b*H_kv + g)*cap + row0 (contiguous) or (page*H_kv + g)*page_rows +
// row0 % page_rows (paged).  The producer walks a unit's tiles in order: the
// table entries of the first page and the next one are loaded when the unit
// is entered (independent of the length load), and entering a page loads
// the entry after it, so a table read is one page ahead of its use.
struct PageCursor {
  int b, g, pg, pb, pbn, off, base;
  // unmapped pages are -1 in the table: they are only ever prefetched as
  // hints (rows < lengths[b] are mapped by contract); clamp so a violated
  // contract reads page 0 instead of faulting
  PS_DEV int entry(const ShaParams& p, int j) const {
    return j < p.table_ld ? max(0, __ldg(p.table + (size_t)b * p.table_ld + j)) : 0;
  }
  // issued before the unit's selection load so the two latencies overlap
  PS_DEV void start(const ShaParams& p, int b_, int row_first) {
    b = b_;
    off = row_first;
    if (p.table) {
      pg = row_first / p.page_rows;
      off = row_first - pg * p.page_rows;
      pb = entry(p, pg);
      pbn = entry(p, pg + 1);
    }
  }
  PS_DEV void set_group(const ShaParams& p, int g_) {
    g = g_;
    base = (b * p.H_kv + g) * p.cap;  // contiguous slab of (b, g); rows < 2^31 (host-checked)
  }
  // physical row of the unit's next tile (tiles are consumed in order), then
  // advance by `rows`: one add per tile, a table step per page
  PS_DEV int next(const ShaParams& p, int rows) {
    int r;
    if (!p.table) {
      r = base + off;
    } else {
      if (off == p.page_rows) {
        pb = pbn;
        ++pg;
        pbn = entry(p, pg + 1);
        off = 0;
      }
      r = (pb * p.H_kv + g) * p.page_rows + off;
    }
    off += rows;
    return r;
  }
};

template <int D_H, int G>
constexpr size_t sha_smem_bytes() {
  return 2 * kStages * kTileBytes + 64 + (size_t)kWarps * G * (D_H + 2) * 4 + 32;  // flag, kWarps length partials, tile count
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

// Per-warp partial of max_b lengths[b] into scratch[warp]; after the caller's
// __syncthreads, sha_nt() turns the kWarps partials into the tile count.
PS_DEV void sha_len_partial(const ShaParams& p, int* scratch) {
  int m = 0;
  for (int b = threadIdx.x; b < p.B; b += kThreads) m = max(m, __ldg(p.lengths + b));
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = m;
}
// the tile count lives in shared memory (flag[5]) and is re-read where it is
// used: keeping it in a register across the main loop pushed the tensor-core
// kernel past 168 registers (3 CTAs / SM -> 2) and cost ~9 % of the stream rate
PS_DEV int ld_nt(const int* s) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(s)));
  return v;
}
PS_DEV int sha_nt(const ShaParams& p, const int* scratch, int T) {
  int m = scratch[0];
#pragma unroll
  for (int w = 1; w < kWarps; ++w) m = max(m, scratch[w]);
  const int nt = (m + T - 1) / T;
  return nt < 1 ? 1 : (nt > p.NT_cap ? p.NT_cap : nt);
}

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
  // the B zero-fill CTAs come first (they overlap the main work instead of
  // forming a tail); stream-K CTA index = blockIdx.x - B
  const int bid = (int)blockIdx.x - p.B;
  griddep_wait();  // q / KV / sel / lengths come from the preceding launches
  // (griddep_launch only after the main loop: with several waves of CTAs, an
  // early trigger lets the next grid's CTAs park on SM slots this grid needs)

  if (bid < 0) {
    // ---- zero-fill CTA for sequence b: heads of non-selected groups = 0.0
    const int b = (int)blockIdx.x;
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

  // first unit's selection / length under the host's tile-count hint: loaded
  // before the barrier setup so the latency overlaps it (every thread needs
  // them for its first segment); reloaded if the device tile count differs
  // first unit = floor(units * bid / n_ctas) whatever the tile count
  // (floor(floor(U*NT*bid/n) / NT) = floor(U*bid/n)), so its selection and
  // length load before the tile count is known
  const int u_first = min(n_units - 1, (int)((long long)n_units * bid / p.n_ctas));
  const int sel_first = __ldg(p.sel + u_first);
  const int len_first = __ldg(p.lengths + u_first / p.top_k);
  sha_len_partial(p, flag + 1);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  {
    const int nt = sha_nt(p, flag + 1, S::T);
    flag[5] = nt;  // every thread stores the same value
  }
  const long long f0 = (long long)bid * ((long long)n_units * ld_nt(flag + 5)) / p.n_ctas;
  const long long f1 = (long long)(bid + 1) * ((long long)n_units * ld_nt(flag + 5)) / p.n_ctas;
  const int n_it = (int)(f1 - f0);

  // producer (thread 0): walks the flattened tiles in order with an
  // incremental (unit, tile) cursor -- the unit's slab / length are loaded
  // once per unit; empty tiles (beyond the length, other rank's group) just
  // arrive
  struct Cursor {
    int u, t, len;
    bool live;
    PageCursor pc;
  } cur;
  auto load_unit = [&](int u) {
    cur.u = u;
    const int b = u / p.top_k;
    cur.pc.start(p, b, cur.t * S::T);
    const int g = (u == u_first ? sel_first : __ldg(p.sel + u)) - p.group_base;
    cur.live = g >= 0 && g < p.H_kv;
    cur.len = u == u_first ? len_first : __ldg(p.lengths + b);
    cur.pc.set_group(p, cur.live ? g : 0);
  };
  auto issue_next = [&](int stage) {
    const int row0 = cur.t * S::T;
    if (!cur.live || row0 >= cur.len) {
      mbar_arrive(&bars[stage]);
    } else {
      const int rows = min(S::T, cur.len - row0);
      const uint32_t bytes = (uint32_t)rows * D_H * 2;
      const size_t off = (size_t)cur.pc.next(p, S::T) * D_H;
      mbar_arrive_expect_tx(&bars[stage], 2 * bytes);
      bulk_g2s(sK + stage * S::T * D_H, p.k + off, bytes, &bars[stage]);
      bulk_g2s(sV + stage * S::T * D_H, p.v + off, bytes, &bars[stage]);
    }
    if (++cur.t == ld_nt(flag + 5)) {  // advance the cursor
      cur.t = 0;
      if (cur.u + 1 < n_units) load_unit(cur.u + 1);
    }
  };
  if (tid == 0 && n_it > 0) {
    const int NT = ld_nt(flag + 5);
    const int u0 = (int)(f0 / NT);
    cur.t = (int)(f0 - (long long)u0 * NT);
    load_unit(u0);
    const int pre = min(kStages, n_it);
    for (int s2 = 0; s2 < pre; ++s2) issue_next(s2);
  }

  const int c = lane % S::LPR;   // 16-byte column chunk owned by this lane
  const int slot = lane / S::LPR;
  int it = 0;
  long long f = f0;
  while (f < f1) {
    const int NT = ld_nt(flag + 5);
    const int u = (int)(f / NT);
    const long long u_end = (long long)(u + 1) * NT;
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
    const int t0 = (int)(f - (long long)u * NT);
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
    const long long F = (long long)n_units * ld_nt(flag + 5);
    const int c_first = cta_of((long long)u * ld_nt(flag + 5), F, p.n_ctas);
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

// ============================================================================
// Tensor-core SHA (d_h = 128, G <= 8).  Same stream-K partition and merge as
// above, but the per-tile math runs on mma.sync: each warp owns 8 KV rows of
// a 32-row tile; S = Q K^T with m16n8k16 (the G query heads are the M rows,
// zero-padded to 16), online softmax on the S fragment (the 4 lanes of a
// head shuffle-reduce its row max), P (bf16) V with m16n8k8 into a 16 x 128
// f32 accumulator.  K/V tiles arrive through 2-D TMA boxes (32 rows x 64
// dims) with the 128-byte swizzle, so the ldmatrix reads of 8 rows at one
// column chunk are bank-conflict free.  ~80 instructions per warp per tile
// (vs ~280 for the CUDA-core path), so the kernel streams at HBM rate.
// Rows past a sequence's length inside its last tile are loaded (the box is
// fixed) but never used: their scores are masked by select and their V rows
// are zeroed in shared memory before the P.V product.
constexpr int kMmaT = 32;
#ifndef PS_SHA_STAGES
#define PS_SHA_STAGES 5
#endif
#ifndef PS_SHA_CTAS
#define PS_SHA_CTAS 2
#endif
constexpr int kMmaStages = PS_SHA_STAGES;
constexpr int kMmaTileBytes = kMmaT * 128 * 2;  // 8 KB of K (or V)

PS_DEV void ldsm_x4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
PS_DEV void ldsm_x4_t(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
PS_DEV void mma_16816(float* d, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  // A rows 8..15 (a1, a3) are the zero padding of the G <= 8 heads
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
PS_DEV void mma_1688(float* d, uint32_t a0, uint32_t b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(b0));
}
// byte offset of 16-byte chunk C (0..15) of tile row r in a swizzled K/V tile
PS_DEV uint32_t mma_sw(int r, int C) {
  return (uint32_t)((C >> 3) * 4096 + r * 128 + (((C & 7) ^ (r & 7)) << 4));
}

PS_DEV unsigned long long sha_time() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SHA_STAMP(slot) \
  do { if (p.trace && threadIdx.x == 0) p.trace[(size_t)blockIdx.x * 8 + (slot)] = sha_time(); } while (0)

template <int G, bool OUT_BF16>
__global__ void __launch_bounds__(kThreads, PS_SHA_CTAS) sha_mma_kernel(const __grid_constant__ CUtensorMap tmK,
                                                          const __grid_constant__ CUtensorMap tmV, const ShaParams p) {
  constexpr int D_H = 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + kMmaStages * kMmaTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kMmaStages * kMmaTileBytes);
  float* red = reinterpret_cast<float*>(smem + 2 * kMmaStages * kMmaTileBytes + 64);
  float* red_m = red;                 // [kWarps][G]
  float* red_l = red + kWarps * G;    // [kWarps][G]
  float* red_o = red + 2 * kWarps * G;  // [kWarps][G][D_H]
  int* flag = reinterpret_cast<int*>(red + kWarps * G * (D_H + 2));

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int n_units = p.B * p.top_k;
  // the B zero-fill CTAs come first (they overlap the main work instead of
  // forming a tail); stream-K CTA index = blockIdx.x - B
  // zero_inline: every CTA is a stream-K CTA (the unselected heads are zeroed
  // below, while its first tiles are in flight); else the B zero-fill CTAs
  // come first and stream-K CTA index = blockIdx.x - B
  const int bid = p.zero_inline ? (int)blockIdx.x : (int)blockIdx.x - p.B;
  SHA_STAMP(0);
  // input-independent prologue before the dependency wait (overlaps the
  // previous kernel's tail under PDL)
  if (bid >= 0 && tid == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    for (int s = 0; s < kMmaStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  griddep_wait();
  SHA_STAMP(1);

  if (bid < 0) {
    // ---- zero-fill CTA for sequence b: heads of non-selected groups = 0.0
    const int b = (int)blockIdx.x;
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

  // tile count from the device lengths (see ShaParams::NT_hint)
  // first unit = floor(units * bid / n_ctas) whatever the tile count
  // (floor(floor(U*NT*bid/n) / NT) = floor(U*bid/n)), so its selection and
  // length load before the tile count is known
  const int u_first = min(n_units - 1, (int)((long long)n_units * bid / p.n_ctas));
  const int sel_first = __ldg(p.sel + u_first);
  const int len_first = __ldg(p.lengths + u_first / p.top_k);
  sha_len_partial(p, flag + 1);
  __syncthreads();
  {
    const int nt = sha_nt(p, flag + 1, kMmaT);
    flag[5] = nt;  // every thread stores the same value
  }
  const long long f0 = (long long)bid * ((long long)n_units * ld_nt(flag + 5)) / p.n_ctas;
  const long long f1 = (long long)(bid + 1) * ((long long)n_units * ld_nt(flag + 5)) / p.n_ctas;
  const int n_it = (int)(f1 - f0);

  // producer cursor (thread 0)
  struct Cursor {
    int u, t, len;
    bool live;
    PageCursor pc;
  } cur;
  auto load_unit = [&](int u) {
    cur.u = u;
    const int b = u / p.top_k;
    cur.pc.start(p, b, cur.t * kMmaT);
    const int g = (u == u_first ? sel_first : __ldg(p.sel + u)) - p.group_base;
    cur.live = g >= 0 && g < p.H_kv;
    cur.len = u == u_first ? len_first : __ldg(p.lengths + b);
    cur.pc.set_group(p, cur.live ? g : 0);
  };
  auto issue_next = [&](int stage) {
    const int row0 = cur.t * kMmaT;
    if (!cur.live || row0 >= cur.len) {
      mbar_arrive(&bars[stage]);
    } else {
      const int row = cur.pc.next(p, kMmaT);
      mbar_arrive_expect_tx(&bars[stage], 2 * kMmaTileBytes);
      uint8_t* k_dst = sK + stage * kMmaTileBytes;
      uint8_t* v_dst = sV + stage * kMmaTileBytes;
      tma_load_2d(k_dst, &tmK, 0, row, &bars[stage]);
      tma_load_2d(k_dst + 4096, &tmK, 64, row, &bars[stage]);
      tma_load_2d(v_dst, &tmV, 0, row, &bars[stage]);
      tma_load_2d(v_dst + 4096, &tmV, 64, row, &bars[stage]);
    }
    if (++cur.t == ld_nt(flag + 5)) {
      cur.t = 0;
      if (cur.u + 1 < n_units) load_unit(cur.u + 1);
    }
  };
  if (tid == 0 && n_it > 0) {
    cur.t = (int)(f0 - (long long)u_first * ld_nt(flag + 5));
    load_unit(u_first);
    const int pre = min(kMmaStages, n_it);
    for (int s2 = 0; s2 < pre; ++s2) issue_next(s2);
  }

  const int gq = lane >> 2;         // head (M row) of this lane's fragments
  const int kq = (lane & 3) * 2;    // column pair inside an 8-wide block
  const int lrow = warp * 8 + (lane & 7);  // ldmatrix row supplied by this lane
  const int lmat = lane >> 3;              // ldmatrix matrix index
  const uint32_t sK_u = smem_u32(sK), sV_u = smem_u32(sV);
  if (p.zero_inline && p.top_k < p.H_kv) {  // every group selected (dense): nothing to zero
    // heads of the groups a sequence did not select are 0.0 (sequences
    // bid, bid + n_ctas, ...); red_o is free until the first unit epilogue
    int* sel_flag = reinterpret_cast<int*>(red_o);
    for (int b = bid; b < p.B; b += p.n_ctas) {
      for (int g2 = tid; g2 < p.H_kv; g2 += kThreads) sel_flag[g2] = 0;
      __syncthreads();
      for (int j = tid; j < p.top_k; j += kThreads) {
        const int g2 = p.sel[(size_t)b * p.top_k + j] - p.group_base;
        if (g2 >= 0 && g2 < p.H_kv) sel_flag[g2] = 1;
      }
      __syncthreads();
      for (int e = tid; e < p.H * D_H; e += kThreads)
        if (!sel_flag[(e / D_H) / G]) store_out<OUT_BF16>(p.out, (size_t)b * p.out_ld + e, 0.0f);
      __syncthreads();
    }
  }
  int it = 0;
  long long f = f0;
  SHA_STAMP(2);
  while (f < f1) {
    const int NT = ld_nt(flag + 5);
    const int u = (int)(f / NT);
    const long long u_end = (long long)(u + 1) * NT;
    const long long seg_end = f1 < u_end ? f1 : u_end;
    const int b = u / p.top_k;
    const int g = (u == u_first ? sel_first : __ldg(p.sel + u)) - p.group_base;
    const bool live = g >= 0 && g < p.H_kv;
    const int len = u == u_first ? len_first : __ldg(p.lengths + b);
    const int nt_seg = (int)(seg_end - f);
    const int t0 = (int)(f - (long long)u * NT);
    f = seg_end;
    if (!live) {
      for (int k2 = 0; k2 < nt_seg; ++k2, ++it) {
        const int stage = it % kMmaStages;
        mbar_wait(&bars[stage], (it / kMmaStages) & 1);
        __syncthreads();
        if (tid == 0 && it + kMmaStages < n_it) issue_next(stage);
      }
      continue;
    }
    // Q fragments (rows = heads; heads >= G are zero)
    uint32_t qa[8][2];
    {
      const uint16_t* qb = p.q + (size_t)b * p.q_ld + (size_t)g * G * D_H;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (gq < G) {
          qa[j][0] = *reinterpret_cast<const uint32_t*>(qb + gq * D_H + 16 * j + kq);
          qa[j][1] = *reinterpret_cast<const uint32_t*>(qb + gq * D_H + 16 * j + 8 + kq);
        } else {
          qa[j][0] = qa[j][1] = 0u;
        }
      }
    }
    float m_run = -INFINITY, l_run = 0.f;
    float o[16][4];
#pragma unroll
    for (int nb = 0; nb < 16; ++nb) o[nb][0] = o[nb][1] = o[nb][2] = o[nb][3] = 0.f;
    const int nt_real = max(0, min(nt_seg, (len + kMmaT - 1) / kMmaT - t0));
    for (int k2 = 0; k2 < nt_seg; ++k2, ++it) {
      const int stage = it % kMmaStages;
      mbar_wait(&bars[stage], (it / kMmaStages) & 1);
      if (it == 0) SHA_STAMP(4);
      if (k2 < nt_real) {
        const int valid = min(kMmaT, len - (t0 + k2) * kMmaT);
        const uint32_t kbase = sK_u + stage * kMmaTileBytes, vbase = sV_u + stage * kMmaTileBytes;
        if (valid < kMmaT && warp * 8 + 8 > valid) {
          // rows past the length in this warp's slice: zero their V (never used, maybe NaN)
          uint8_t* vt = sV + stage * kMmaTileBytes;
          for (int e = lane; e < 8 * 16; e += 32) {
            const int r = warp * 8 + (e >> 4), C = e & 15;
            if (r >= valid) *reinterpret_cast<uint4*>(vt + mma_sw(r, C)) = make_uint4(0, 0, 0, 0);
          }
          fence_proxy_async();  // generic writes before the next TMA into this stage
          __syncwarp();
        }
        // ---- S = Q K^T for this warp's 8 rows (two accumulators: shorter MMA chain)
        float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t kb[4];
          ldsm_x4(kbase + mma_sw(lrow, 4 * i + lmat), kb);
          mma_16816(sa, qa[2 * i][0], qa[2 * i][1], kb[0], kb[1]);
          mma_16816(sb, qa[2 * i + 1][0], qa[2 * i + 1][1], kb[2], kb[3]);
        }
        const int r0 = warp * 8 + kq;
        float s0 = (sa[0] + sb[0]) * p.scale_log2, s1 = (sa[1] + sb[1]) * p.scale_log2;
        s0 = r0 < valid ? s0 : -INFINITY;
        s1 = r0 + 1 < valid ? s1 : -INFINITY;
        float mx = fmaxf(s0, s1);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float m_new = fmaxf(m_run, mx);
        const float m_use = m_new == -INFINITY ? 0.f : m_new;
        const float alpha = fast_exp2(m_run - m_use);
        const float p0 = fast_exp2(s0 - m_use), p1 = fast_exp2(s1 - m_use);
        l_run = l_run * alpha + p0 + p1;
        m_run = m_new;
        const uint32_t pa = pack_bf16x2(p0, p1);
        // ---- O = O * alpha + P V
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t vb[4];
          ldsm_x4_t(vbase + mma_sw(lrow, 4 * i + lmat), vb);
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            float* acc = o[4 * i + m];
            acc[0] *= alpha;
            acc[1] *= alpha;
            mma_1688(acc, pa, vb[m]);
          }
        }
      }
      __syncthreads();  // every warp is done with this stage
      if (tid == 0 && it + kMmaStages < n_it) issue_next(stage);
    }

    // ---- per-warp state -> shared (lanes of head gq own dims 8nb + kq, +1)
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    if (gq < G) {
#pragma unroll
      for (int nb = 0; nb < 16; ++nb) {
        red_o[(warp * G + gq) * D_H + 8 * nb + kq] = o[nb][0];
        red_o[(warp * G + gq) * D_H + 8 * nb + kq + 1] = o[nb][1];
      }
      if ((lane & 3) == 0) {
        red_m[warp * G + gq] = m_run;
        red_l[warp * G + gq] = l_run;
      }
    }
    __syncthreads();

    // ---- merge warps; a unit inside one CTA writes its output directly
    const long long F = (long long)n_units * ld_nt(flag + 5);
    const int c_first = cta_of((long long)u * ld_nt(flag + 5), F, p.n_ctas);
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
        if (tid == 0) p.counters[u] = 0;
      }
    }
    __syncthreads();
  }
  SHA_STAMP(3);
  griddep_launch();
}

template <int G>
constexpr size_t sha_mma_smem_bytes() {
  return 1024 + 2 * kMmaStages * kMmaTileBytes + 64 + (size_t)kWarps * G * (128 + 2) * 4 + 32;  // flag, kWarps length partials, tile count
}

PFN_cuTensorMapEncodeTiled_v12000 g_sha_encode = nullptr;

int sha_tmap(CUtensorMap* m, const void* base, uint64_t rows) {
  if (!g_sha_encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return PS_ERR_CUDA;
    g_sha_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {128, rows};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {64, (cuuint32_t)kMmaT};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_sha_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? PS_OK : PS_ERR_VALUE;
}

template <int G, bool BF16>
int launch_sha_mma(const ShaParams& prm, int grid, cudaStream_t st) {
  constexpr size_t smem = sha_mma_smem_bytes<G>();
  auto kern = sha_mma_kernel<G, BF16>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return PS_ERR_CUDA;
    configured = true;
  }
  const uint64_t rows = prm.table ? (uint64_t)prm.pool_pages * prm.H_kv * prm.page_rows
                                  : (uint64_t)prm.B * prm.H_kv * prm.cap;
  CUtensorMap tk, tv;
  int rc = sha_tmap(&tk, prm.k, rows);
  if (rc == PS_OK) rc = sha_tmap(&tv, prm.v, rows);
  if (rc != PS_OK) return rc;
  // the stream-K CTAs zero the unselected heads themselves: no B extra CTAs
  // holding slots at the start (their stream-K neighbours started ~2 us late
  // and finished last)
  (void)grid;
  ShaParams p2 = prm;
  p2.zero_inline = 1;
  return launch_ex(kern, dim3(prm.n_ctas), dim3(kThreads), smem, st, 1, tk, tv, p2);
}

int g_sha_mma = 1;  // 0: CUDA-core path for every shape (ps_debug_sha_mma)

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

// resident SHA CTAs (80 KB of K/V stages each: 2 per SM)
int sha_slots() { return ps_num_sms() * PS_SHA_CTAS; }

// CTAs = units x splits (each unit cut into `splits` equal tile ranges).
// Auto (num_splits == 0): the split count minimising the last-wave waste
// ceil(W)/W (W = units*s / resident slots) plus a per-split cost (partials +
// merge, ~4 % each), with >= 4 tiles per split -- measured on B200 (ctx
// 1920): s = 1 at 2048 and 256 units, 3 at 1024 (OPT-6.7B B=64 rho=.5), 4 at
// 512, 2 at 128.
int sha_auto_splits(int units, int NT) {
  const double slots = (double)sha_slots();
  int best = 1;
  double best_cost = 1e30;
  for (int s = 1; s <= 8; ++s) {
    if (s > 1 && NT / s < 4) break;
    const double n = units * (double)s, w = n / slots;
    // one partial wave streams at full rate once ~256 CTAs (1.7 per SM) are
    // in flight; beyond a wave, the last wave's idle fraction is lost
    const double wave = n <= slots ? (n >= 256.0 ? 1.0 : 256.0 / n) : std::ceil(w) / w;
    const double cost = wave + 0.04 * s;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

int sha_ctas(int units, int NT, int num_splits, int G) {
  // num_splits < 0: exactly -num_splits stream-K CTAs (tuning hook)
  long long cap;
  if (num_splits < 0) {
    cap = -(long long)num_splits;
  } else if (num_splits == 0 && units >= sha_slots()) {
    // at least one unit per resident slot: ONE persistent stream-K wave
    // (2 CTAs x 5 stages per SM).  Measured on B200 at ctx 1920 against the
    // wave model below (3 CTAs x 4 stages): OPT-6.7B B=64 rho=.5 157.3 ->
    // 151.5 us, LLaMA-8B B=256 k=4 162.7 -> 157.4 us, dense B=128 570.8 -> 565.7 us
    cap = sha_slots();
  } else if (num_splits == 0 && G >= 4 && units >= (sha_slots() * 9) / 10) {
    // grouped heads (G >= 4: a unit's partial is G x (d_h + 2) floats, so
    // splitting costs more): one CTA per unit once there are ~2 waves of
    // units, else exactly one resident wave -- measured on B200 at ctx 1920,
    // H_kv = 8: 512 units 98 -> 90 us, 1024 units 167 -> 162 us, 4096 units
    // 595 -> 575 us against the wave model below
    cap = units >= (sha_slots() * 9) / 5 ? units : sha_slots();
  } else {
    if (num_splits == 0) num_splits = sha_auto_splits(units, NT);
    cap = (long long)units * num_splits;
  }
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
  const int n = num_splits < 0 ? -num_splits : (int)(units * (num_splits > 0 ? num_splits : 8));  // >= sha_ctas
  return kCounterBytes + units * (size_t)sha_max_seg((int)units, n) * (size_t)partial_floats(H / H_kv, d_h) * 4;
}

extern "C" void ps_debug_sha_mma(int enable) { g_sha_mma = enable ? 1 : 0; }
static unsigned long long* g_sha_trace = nullptr;
extern "C" void ps_debug_sha_trace(void* buf) { g_sha_trace = static_cast<unsigned long long*>(buf); }

// 0 = stream-K over one resident wave (the default)
extern "C" int ps_sha_auto_splits(int B, int H_kv, int d_h, int top_k, int max_len) {
  (void)B; (void)H_kv; (void)d_h; (void)top_k; (void)max_len;
  return 0;
}

static int sha_decode_impl(const void* q, int64_t q_ld, const void* k_cache, const void* v_cache,
                           const int32_t* lengths, const int32_t* sel, int group_base, int B, int H, int H_kv,
                           int cap, int d_h, int top_k, float scale, int num_splits, int max_len_hint, void* out,
                           int64_t out_ld, int out_dtype, void* ws, size_t ws_bytes, void* stream,
                           const int32_t* table, int64_t table_ld, int page_rows, int pool_pages) {
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
  if (ws_bytes < ps_sha_workspace_bytes(B, H, H_kv, d_h, top_k, num_splits)) return PS_ERR_WORKSPACE;
  // max_len_hint only sizes the grid (and the first-unit prefetch): the
  // kernel takes the tile count from the device lengths, so any lengths[b] <=
  // cap are read in full (a graph captured at one length stays exact)
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
  prm.table = table;
  prm.table_ld = table_ld;
  prm.page_rows = table ? page_rows : cap;
  prm.pool_pages = pool_pages;
  if (table && page_rows % T) return PS_ERR_VALUE;  // a tile never straddles a page
  if (!table && (long long)B * H_kv * cap >= (1ll << 31)) return PS_ERR_UNSUPPORTED;  // 32-bit row index
  prm.NT_hint = NT;
  prm.NT_cap = (cap + T - 1) / T;
  prm.n_ctas = sha_ctas(units, NT, num_splits, G);
  prm.max_seg = sha_max_seg(units, prm.n_ctas);
  prm.scale_log2 = scale * kLog2e;
  prm.out = out;
  prm.out_ld = out_ld;
  prm.counters = static_cast<int*>(ws);
  prm.trace = g_sha_trace;
  prm.partials = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + kCounterBytes);
  const int grid = prm.n_ctas + B;  // the CUDA-core kernel's B zero-fill CTAs (the tensor-core kernel zeroes inline)
  const bool bf16 = out_dtype == PS_DTYPE_BF16;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (d_h) {
    case 8: return dispatch_g<8>(prm, grid, G, bf16, st);
    case 16: return dispatch_g<16>(prm, grid, G, bf16, st);
    case 32: return dispatch_g<32>(prm, grid, G, bf16, st);
    case 64: return dispatch_g<64>(prm, grid, G, bf16, st);
    case 128:
      if (g_sha_mma && G <= 8 && (((uintptr_t)k_cache | (uintptr_t)v_cache) % 16) == 0) {
        switch (G) {
          case 1: return bf16 ? launch_sha_mma<1, true>(prm, grid, st) : launch_sha_mma<1, false>(prm, grid, st);
          case 2: return bf16 ? launch_sha_mma<2, true>(prm, grid, st) : launch_sha_mma<2, false>(prm, grid, st);
          case 4: return bf16 ? launch_sha_mma<4, true>(prm, grid, st) : launch_sha_mma<4, false>(prm, grid, st);
          case 8: return bf16 ? launch_sha_mma<8, true>(prm, grid, st) : launch_sha_mma<8, false>(prm, grid, st);
          default: break;
        }
      }
      return dispatch_g<128>(prm, grid, G, bf16, st);
    case 256: return dispatch_g<256>(prm, grid, G, bf16, st);
    default: return PS_ERR_UNSUPPORTED;
  }
}

extern "C" int ps_sha_decode(const void* q, int64_t q_ld, const void* k_cache, const void* v_cache,
                             const int32_t* lengths, const int32_t* sel, int group_base, int B, int H, int H_kv,
                             int cap,
                             int d_h, int top_k, float scale, int num_splits, int max_len_hint, void* out,
                             int64_t out_ld, int out_dtype, void* ws, size_t ws_bytes, void* stream) {
  return sha_decode_impl(q, q_ld, k_cache, v_cache, lengths, sel, group_base, B, H, H_kv, cap, d_h, top_k, scale,
                         num_splits, max_len_hint, out, out_ld, out_dtype, ws, ws_bytes, stream, nullptr, 0, 0, 0);
}

extern "C" int ps_sha_decode_paged(const void* q, int64_t q_ld, const void* k_pool, const void* v_pool,
                                   int pool_pages, int page_rows, const int32_t* block_table, int64_t table_ld,
                                   const int32_t* lengths, const int32_t* sel, int group_base, int B, int H,
                                   int H_kv, int d_h, int top_k, float scale, int num_splits, int max_len_hint,
                                   void* out, int64_t out_ld, int out_dtype, void* ws, size_t ws_bytes,
                                   void* stream) {
  if (!block_table || pool_pages < 1 || page_rows < 1 || table_ld < 1) return PS_ERR_VALUE;
  if ((long long)pool_pages * H_kv * page_rows >= (1ll << 31)) return PS_ERR_UNSUPPORTED;  // TMA row coordinate
  const long long cap = (long long)table_ld * page_rows;
  if (cap >= (1ll << 31)) return PS_ERR_VALUE;
  return sha_decode_impl(q, q_ld, k_pool, v_pool, lengths, sel, group_base, B, H, H_kv, (int)cap, d_h, top_k,
                         scale, num_splits, max_len_hint, out, out_ld, out_dtype, ws, ws_bytes, stream, block_table,
                         table_ld, page_rows, pool_pages);
}
