// Selection kernels: bit-exact per-row top-k, threshold selection, batch
// union by bitmap + ascending compaction, and the head router fused with its
// top-k.  Ordering contract (tensors.py:54-73, numpy stable argsort of
// -scores): value descending, ties -> lower index, -0.0 == +0.0, NaN ranks
// below -inf (NaNs tied among themselves by index); ids written ascending.
#include <cstdlib>

#include "common.cuh"

namespace ps {
namespace {

// Order-preserving uint32 key; 0 is reserved for NaN (below -inf).
PS_DEV uint32_t order_key(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0u;  // NaN
  if (u == 0x80000000u) u = 0u;                     // -0.0 -> +0.0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Block-wide exclusive scan of one int per thread (blockDim multiple of 32).
template <int NT>
PS_DEV int block_excl_scan(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < NT / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) s_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const int before = warp ? s_warp[warp - 1] : 0;
  const int t = s_warp[NT / 32 - 1];
  __syncthreads();
  if (total) *total = t;
  return before + x - v;
}

constexpr int kTopkThreads = 512;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kTopkSmemCols = 36864;  // rows up to this width are staged in shared memory (144 KB; 220 KB total)
constexpr int kSample = 2048;         // strided sample of a row that brackets the k-th key
constexpr int kMaxCand = 3072;        // keys inside the bracket kept for the exact select
constexpr int kGroupRows = 16;        // union: rows ORed by the last CTA of each row group
constexpr int kMaxGroups = 64;        // ps_select_union: rows <= 1024
constexpr int kUnionWPT = 4;          // co-resident union: words per thread (cols <= 65536)

struct TopkParams {
  const float* logits;
  int rows, cols;
  int64_t ld;
  int k;             // > 0: top-k per row; <= 0: threshold selection (logit > thr)
  float thr;
  const float* bias;  // added to every row before selection (router output bias), or NULL
  int32_t* idx_out;  // (rows, k) ascending ids, or NULL
  uint32_t* bitmap;  // atomic-OR union bitmap, or NULL
  // fused union (ps_select_union): per-row words, per-group words, tickets
  uint32_t* row_bits;    // (rows, words) or NULL
  uint32_t* group_bits;  // (groups, words)
  int* tickets;          // [groups] + [1] + 8-byte barrier word + spare (self-resetting)
  int coresident;        // every row CTA is resident at once: grid barrier + distributed union
  int lo, hi, pad;
  int32_t* union_out;
  int32_t* count_out;
  unsigned long long* trace;  // debug phase stamps (16 per CTA) or NULL
};

PS_DEV void hist_add_agg(int* hist, bool act, uint32_t bin, int lane) {
  if (__ballot_sync(0xffffffffu, act)) {
    const uint32_t b = act ? bin : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, b);
    if (act && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&hist[b], __popc(peers));
  }
}

// Descending scan of g[0, bins): the bin holding the `remaining`-th largest
// key.  Writes s_sel = {bin, remaining within the bin, bin count}.
template <int NT>
PS_DEV void select_bin(const int* g, int bins, int remaining, int* s_warp, int* s_sel) {
  const int per = bins / NT;
  const int hi = bins - (int)threadIdx.x * per;
  int loc = 0;
  for (int j = 1; j <= per; ++j) loc += g[hi - j];
  const int above = block_excl_scan<NT>(loc, s_warp, nullptr);
  if (above < remaining && above + loc >= remaining) {
    int cum = above;
    for (int j = 1; j <= per; ++j) {
      const int c = g[hi - j];
      if (cum + c >= remaining) {
        s_sel[0] = hi - j;
        s_sel[1] = remaining - cum;
        s_sel[2] = c;
        break;
      }
      cum += c;
    }
  }
  __syncthreads();
}

// Block form of select_bin for up to two (histogram, rank) pairs at once
// (r2 <= 0: none), with two block barriers: warp w owns bins
// [BINS - (w+1)*BINS/16, BINS - w*BINS/16) (warp 0 the highest), each lane
// PER contiguous bins; warp scans, then a 16-entry scan of the warp totals
// through shared memory.  out = {bin, remaining within the bin, bin count}.
template <int BINS, int NT>
PS_DEV void bsel2(const int* g1, int r1, int* o1, const int* g2, int r2, int* o2, int* s_wt) {
  constexpr int NW = NT / 32, PER_W = BINS / NW, PER = PER_W / 32;
  static_assert(PER >= 1 && NW <= 32, "bsel2 shape");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lo = BINS - warp * PER_W - (lane + 1) * PER;
  int a1 = 0, a2 = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    a1 += g1[lo + j];
    if (r2 > 0) a2 += g2[lo + j];
  }
  int x1 = a1, x2 = a2;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y1 = __shfl_up_sync(0xffffffffu, x1, o), y2 = __shfl_up_sync(0xffffffffu, x2, o);
    if (lane >= o) { x1 += y1; x2 += y2; }
  }
  if (lane == 31) { s_wt[warp] = x1; s_wt[32 + warp] = x2; }
  __syncthreads();
  int w1 = lane < NW ? s_wt[lane] : 0, w2 = lane < NW ? s_wt[32 + lane] : 0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y1 = __shfl_up_sync(0xffffffffu, w1, o), y2 = __shfl_up_sync(0xffffffffu, w2, o);
    if (lane >= o) { w1 += y1; w2 += y2; }
  }
  // exclusive prefix of this warp = inclusive of warp-1
  const int b1 = __shfl_sync(0xffffffffu, w1, (warp + 31) & 31), b2 = __shfl_sync(0xffffffffu, w2, (warp + 31) & 31);
  auto find = [&](const int* g, int r, int base, int x, int a, int* o) {
    const int above = (warp ? base : 0) + x - a;
    if (r > 0 && above < r && above + a >= r) {
      int cum = above;
#pragma unroll
      for (int b = lo + PER - 1; b >= lo; --b) {
        const int c = g[b];
        if (cum + c >= r) {
          o[0] = b;
          o[1] = r - cum;
          o[2] = c;
          break;
        }
        cum += c;
      }
    }
  };
  find(g1, r1, b1, x1, a1, o1);
  find(g2, r2, b2, x2, a2, o2);
  __syncthreads();
}

// r-th largest (1-based) of n u32 keys in shared memory: 3 radix passes
// (12/10/10 bits).  Returns the key; *eq = how many keys equal it, *rem =
// how many of those reach rank r.  Block-wide; r in [1, n].
template <int NT>
PS_DEV uint32_t list_select(const uint32_t* keys, int n, int r, int* hA, int* hB, int* s_sel, int* s_wt, int* eq,
                            int* rem) {
  // hA [4096] serves passes 0 and 2, hB [1024] pass 1; hA is re-zeroed
  // during pass 1, so each pass costs two block barriers
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096; i += NT) hA[i] = 0;
  for (int i = threadIdx.x; i < 1024; i += NT) hB[i] = 0;
  __syncthreads();
  uint32_t prefix = 0, mask = 0;
  int remaining = r;
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    const int shift = pass == 0 ? 20 : (pass == 1 ? 10 : 0);
    const int bins = pass == 0 ? 4096 : 1024;
    int* h = pass == 1 ? hB : hA;
    for (int base = 0; base < n; base += NT) {
      const int i = base + (int)threadIdx.x;
      const uint32_t u = i < n ? keys[i] : 0u;
      hist_add_agg(h, i < n && (u & mask) == prefix, (u >> shift) & (uint32_t)(bins - 1), lane);
    }
    if (pass == 1)
      for (int i = threadIdx.x; i < 1024; i += NT) hA[i] = 0;
    __syncthreads();
    if (pass == 0) bsel2<4096, NT>(h, remaining, s_sel, h, 0, s_sel, s_wt);
    else bsel2<1024, NT>(h, remaining, s_sel, h, 0, s_sel, s_wt);
    prefix |= (uint32_t)s_sel[0] << shift;
    remaining = s_sel[1];
    mask |= (uint32_t)(bins - 1) << shift;
  }
  *eq = s_sel[2];
  *rem = remaining;
  return prefix;  // s_sel is next written only after another block barrier
}

// debug: per-CTA globaltimer stamps of the phases (ps_debug_topk_trace)
PS_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TK_STAMP(slot) \
  do { if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 16 + (slot)] = gtime(); } while (0)

// word w of the OR over `nrows` (<= MAXR) bitmaps of stride `words`: every
// load issued before the first use (one memory latency)
template <int MAXR>
PS_DEV uint32_t or_rows(const uint32_t* bits, int nrows, int words, int w) {
  uint32_t v[MAXR];
#pragma unroll
  for (int r = 0; r < MAXR; ++r) v[r] = r < nrows ? __ldcg(bits + (size_t)r * words + w) : 0u;
  uint32_t acc = 0;
#pragma unroll
  for (int r = 0; r < MAXR; ++r) acc |= v[r];
  return acc;
}

// Ascending ids - lo of the set bits of `word(w)` in [lo, hi); device count;
// idx_out padded up to a multiple of `pad` with the last id.
template <int NT, typename WordFn>
PS_DEV void compact_words(WordFn word, int lo, int hi, int pad, int32_t* out, int32_t* count, int* s_warp) {
  const int wlo = lo >> 5, whi = (hi + 31) >> 5;
  const int nw = whi - wlo;
  const int per = (nw + NT - 1) / NT;
  const int w0 = wlo + min(nw, (int)threadIdx.x * per), w1 = wlo + min(nw, (int)(threadIdx.x + 1) * per);
  auto clip = [&](int w, uint32_t bits) {
    const int top = hi - (w << 5);
    if (top < 32) bits &= (top <= 0) ? 0u : ((1u << top) - 1u);
    return bits;
  };
  uint32_t mine[4];
  int cnt = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    mine[j] = (w0 + j < w1) ? clip(w0 + j, word(w0 + j)) : 0u;
    cnt += __popc(mine[j]);
  }
  for (int w = w0 + 4; w < w1; ++w) cnt += __popc(clip(w, word(w)));
  int total;
  int pos = block_excl_scan<NT>(cnt, s_warp, &total);
  for (int w = w0; w < w1; ++w) {
    uint32_t bits = (w - w0 < 4) ? mine[w - w0] : clip(w, word(w));
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      out[pos++] = (w << 5) + b - lo;
    }
  }
  if (threadIdx.x == 0) *count = total;
  if (pad > 1) {
    __syncthreads();
    const int padded = (total + pad - 1) / pad * pad;
    const int32_t last = total > 0 ? out[total - 1] : 0;
    for (int i = total + (int)threadIdx.x; i < padded; i += NT) out[i] = last;
  }
}

// Per-row top-k (and threshold selection), bit-exact with numpy's stable
// argsort of -scores: value descending, ties -> lower index, -0.0 == +0.0,
// NaN below -inf.  One CTA (1024 threads) per row; the row (+ optional
// bias) is staged in shared memory as order-preserving u32 keys.
//   1. bracket: a strided sample of 2048 keys, taken while staging, gives
//      the sample order statistics at ranks k*S/cols -/+ (3 sigma + 2) to
//      22-bit precision (two shared radix passes, both ranks per scan);
//   2. one pass counts the keys above the bracket and appends the keys
//      inside it (~7 % of the row) to per-warp candidate lists (no shared
//      atomics), then compacted;
//   3. exact k-th key T = radix select over the candidates; ties at T go to
//      the lowest columns: the last one taken, I, is a radix select over the
//      tied candidates' inverted columns;
//   4. every key is then decided locally (key > T, or key == T and column
//      <= I): one ballot per 32 columns.
// The bracket is verified exactly (count above < k <= above + candidates);
// a miss (or a per-warp list overflow) falls back to a full 3-pass radix
// select with per-warp tie ranking.  Outputs: ids (ps_topk_rows), an
// atomic-OR bitmap, or -- ps_select_union -- this row's words stored
// plainly; the last CTA of each group of 16 rows ORs the group, and the last
// group compacts the union (ascending ids, device count, padded): no
// contended atomics.  Threshold mode keeps logit (+ bias) > thr.
constexpr int kWarpCand = kMaxCand / kTopkWarps;  // per-warp candidate capacity
constexpr int kStageVec = 4;  // float4 per thread per staging batch (loads issued together)
constexpr int kRegCols = 16384;  // rows up to this width stay in registers while the bracket is computed
constexpr int kRegVec = kRegCols / 4 / kTopkThreads;  // 8 float4 per thread

__global__ void __launch_bounds__(kTopkThreads) topk_rows_kernel(const TopkParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  int* hist = reinterpret_cast<int*>(smem);                          // [4096]
  uint32_t* samp = reinterpret_cast<uint32_t*>(hist + 4096);         // [kMaxCand] samples, then tied cols
  uint32_t* wc_key = samp + kMaxCand;                                // [kMaxCand] per-warp lists
  // [2048] second-level histograms: used by the bracket before the per-warp
  // lists are filled and by list_select after they were compacted
  int* hist2 = reinterpret_cast<int*>(wc_key);
  int* wc_idx = reinterpret_cast<int*>(wc_key + kMaxCand);           // [kMaxCand]
  uint32_t* cand_key = reinterpret_cast<uint32_t*>(wc_idx + kMaxCand);  // [kMaxCand] compacted
  int* cand_idx = reinterpret_cast<int*>(cand_key + kMaxCand);       // [kMaxCand]
  uint32_t* keys = reinterpret_cast<uint32_t*>(cand_idx + kMaxCand);  // [cols] if staged
  __shared__ int s_warp[64];
  __shared__ int s_eq[kTopkWarps], s_gt[kTopkWarps], s_wn[kTopkWarps];
  __shared__ int s_sel[6];
  __shared__ int s_na, s_ovf, s_n2, s_last;
  const int row = blockIdx.x, cols = p.cols;
  const float* x = p.logits + (size_t)row * p.ld;
  const float* bias = p.bias;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool threshold = p.k <= 0;
  const bool staged = !threshold && cols <= kTopkSmemCols;
  auto logit = [&](int i) -> float { return bias ? __ldg(x + i) + __ldg(bias + i) : __ldg(x + i); };
  auto key_at = [&](int i) -> uint32_t { return staged ? keys[i] : order_key(logit(i)); };
  const bool vec_ok = staged && (cols & 3) == 0 && (p.ld & 3) == 0 && ((uintptr_t)x & 15) == 0 &&
                      (!bias || ((uintptr_t)bias & 15) == 0);
  const bool fused = vec_ok && cols <= kRegCols;
  if (fused && bias) {
    // the bias is static: copy it into the key slots before waiting on the
    // previous kernel; each thread later reads back only its own slots
    const float4* b4 = reinterpret_cast<const float4*>(bias);
#pragma unroll
    for (int j = 0; j < kRegVec; ++j) {
      const int i = j * kTopkThreads + tid;
      if (i < (cols >> 2)) cp_async16(keys + 4 * i, b4 + i, 16);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  griddep_wait();
  griddep_launch();
  TK_STAMP(0);
  uint32_t prefix = 0;
  int remaining = 0;
  bool fast = true;          // every key decided locally
  int tie_lim = 0x7fffffff;  // fast: tied keys at column < tie_lim are taken
  if (!threshold) {
    if (tid == 0) { s_na = 0; s_ovf = 0; s_n2 = 0; }
    for (int i = tid; i < 4096; i += kTopkThreads) hist[i] = 0;
    for (int i = tid; i < 2048; i += kTopkThreads) hist2[i] = 0;
    const int S = min(cols, kSample);
    const int stride = cols / S;
    const float q = (float)p.k / (float)cols;
    const float rs = q * (float)S;
    const float dl = 3.f * sqrtf(fmaxf(rs * (1.f - q), 0.f)) + 2.f;
    const bool open_top = rs - dl < 1.f, open_bottom = rs + dl > (float)S;
    const int r_hi = max(1, min(S, (int)floorf(rs - dl)));
    const int r_lo = max(1, min(S, (int)ceilf(rs + dl)));
    // bracket (22-bit sample order statistics at ranks r_hi / r_lo) from samp[0, S)
    auto bracket = [&](uint32_t& hi22, uint32_t& lo22) {
      // hist (top 12 bits) and hist2 (next 10 bits, one half per rank) were
      // zeroed at entry; warp 0 scans, 4 block barriers in all
      for (int base = 0; base < S; base += kTopkThreads) {
        const int j = base + tid;
        const uint32_t u = j < S ? samp[j] : 0u;
        hist_add_agg(hist, j < S, u >> 20, lane);
      }
      __syncthreads();
      TK_STAMP(12);
      bsel2<4096, kTopkThreads>(hist, r_hi, s_sel, hist, r_lo, s_sel + 3, s_warp);
      TK_STAMP(13);
      const int bin_hi = s_sel[0], rem_hi = s_sel[1], bin_lo = s_sel[3], rem_lo = s_sel[4];
      for (int base = 0; base < S; base += kTopkThreads) {
        const int j = base + tid;
        const uint32_t u = j < S ? samp[j] : 0u;
        const int top = (int)(u >> 20);
        const uint32_t sub = (u >> 10) & 1023u;
        hist_add_agg(hist2, j < S && top == bin_hi, sub, lane);
        hist_add_agg(hist2 + 1024, j < S && top == bin_lo, sub, lane);
      }
      __syncthreads();
      TK_STAMP(14);
      bsel2<1024, kTopkThreads>(hist2, rem_hi, s_sel, hist2 + 1024, rem_lo, s_sel + 3, s_warp);
      hi22 = open_top ? 0x3FFFFFu : (((uint32_t)bin_hi << 10) | (uint32_t)s_sel[0]);
      lo22 = open_bottom ? 0u : (((uint32_t)bin_lo << 10) | (uint32_t)s_sel[3]);
    };
    int n_above_t = 0, wn = 0;  // this thread's count above the bracket; this warp's candidates
    uint32_t* wk = wc_key + warp * kWarpCand;
    int* wi = wc_idx + warp * kWarpCand;
    auto classify_key = [&](bool ok, uint32_t u, int i, uint32_t hi22, uint32_t lo22) {
      const uint32_t t22 = u >> 10;
      n_above_t += (ok && t22 > hi22) ? 1 : 0;
      const bool cand = ok && t22 >= lo22 && t22 <= hi22;
      const uint32_t bal = __ballot_sync(0xffffffffu, cand);
      const int slot = wn + __popc(bal & ((1u << lane) - 1u));
      if (cand && slot < kWarpCand) {
        wk[slot] = u;
        wi[slot] = i;
      }
      wn += __popc(bal);
    };
    uint32_t hi22, lo22;
    if (fused) {
      // ---- fused: the row's loads are in flight (registers) while the
      //      bracket is computed from a strided sample read directly from
      //      memory; then ONE pass converts, stages and classifies every key
      const float4* x4 = reinterpret_cast<const float4*>(x);
      const int n4 = cols >> 2;
      float4 v[kRegVec];
#pragma unroll
      for (int j = 0; j < kRegVec; ++j) {
        const int i = j * kTopkThreads + tid;
        if (i < n4) v[j] = __ldg(x4 + i);
      }
      for (int j = tid; j < S; j += kTopkThreads) samp[j] = order_key(logit(j * stride));
      __syncthreads();
      TK_STAMP(1);
      bracket(hi22, lo22);
      TK_STAMP(2);
      if (bias) asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
      for (int j = 0; j < kRegVec; ++j) {
        const int i = j * kTopkThreads + tid;
        const bool ok = i < n4;
        if (ok && bias) {
          const float4 bb = *reinterpret_cast<const float4*>(keys + 4 * i);
          v[j].x += bb.x; v[j].y += bb.y; v[j].z += bb.z; v[j].w += bb.w;
        }
        const uint4 u = ok ? make_uint4(order_key(v[j].x), order_key(v[j].y), order_key(v[j].z), order_key(v[j].w))
                           : make_uint4(0, 0, 0, 0);
        if (ok) *reinterpret_cast<uint4*>(keys + 4 * i) = u;
        classify_key(ok, u.x, 4 * i, hi22, lo22);
        classify_key(ok, u.y, 4 * i + 1, hi22, lo22);
        classify_key(ok, u.z, 4 * i + 2, hi22, lo22);
        classify_key(ok, u.w, 4 * i + 3, hi22, lo22);
      }
    } else {
      // ---- stage the keys, keep a strided sample, then bracket and classify
      if (vec_ok) {
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const float4* b4 = reinterpret_cast<const float4*>(bias);
        const int n4 = cols >> 2;
        for (int i0 = 0; i0 < n4; i0 += kStageVec * kTopkThreads) {
          float4 v[kStageVec], bb[kStageVec];
#pragma unroll
          for (int j = 0; j < kStageVec; ++j) {
            const int i = i0 + j * kTopkThreads + tid;
            if (i < n4) {
              v[j] = __ldg(x4 + i);
              if (bias) bb[j] = __ldg(b4 + i);
            }
          }
#pragma unroll
          for (int j = 0; j < kStageVec; ++j) {
            const int i = i0 + j * kTopkThreads + tid;
            if (i < n4) {
              if (bias) {
                v[j].x += bb[j].x; v[j].y += bb[j].y; v[j].z += bb[j].z; v[j].w += bb[j].w;
              }
              *reinterpret_cast<uint4*>(keys + 4 * i) =
                  make_uint4(order_key(v[j].x), order_key(v[j].y), order_key(v[j].z), order_key(v[j].w));
            }
          }
        }
      } else if (staged) {
        for (int i = tid; i < cols; i += kTopkThreads) keys[i] = order_key(logit(i));
      }
      for (int j = tid; j < S; j += kTopkThreads) samp[j] = staged ? keys[j * stride] : order_key(logit(j * stride));
      __syncthreads();
      TK_STAMP(1);
      bracket(hi22, lo22);
      TK_STAMP(2);
      for (int base = 0; base < cols; base += kTopkThreads) {
        const int i = base + tid;
        classify_key(i < cols, i < cols ? key_at(i) : 0u, i, hi22, lo22);
      }
    }
    n_above_t = warp_sum(n_above_t);
    if (lane == 0) {
      s_wn[warp] = wn;
      atomicAdd(&s_na, n_above_t);
      if (wn > kWarpCand) s_ovf = 1;
    }
    __syncthreads();
    int n_cand = 0, my_off = 0;
    for (int w = 0; w < kTopkWarps; ++w) {
      const int c = s_wn[w];
      if (w < warp) my_off += c;
      n_cand += c;
    }
    const int n_above = s_na;
    if (!s_ovf && n_above < p.k && n_above + n_cand >= p.k) {
      // compact the per-warp lists (each warp copies its own)
      const int wn = s_wn[warp];
      for (int j = lane; j < wn; j += 32) {
        cand_key[my_off + j] = wc_key[warp * kWarpCand + j];
        cand_idx[my_off + j] = wc_idx[warp * kWarpCand + j];
      }
      __syncthreads();
      TK_STAMP(3);
      // ---- 3. exact k-th key among the candidates, then the tie column
      int n_eq, rem;
      prefix = list_select<kTopkThreads>(cand_key, n_cand, p.k - n_above, hist, hist2, s_sel, s_warp, &n_eq, &rem);
      remaining = rem;
      if (rem < n_eq) {
        for (int base = 0; base < n_cand; base += kTopkThreads) {
          const int j = base + tid;
          const bool eq = j < n_cand && cand_key[j] == prefix;
          const uint32_t bal = __ballot_sync(0xffffffffu, eq);
          if (bal) {
            const int leader = __ffs(bal) - 1;
            int slot = 0;
            if (lane == leader) slot = atomicAdd(&s_n2, __popc(bal));
            slot = __shfl_sync(0xffffffffu, slot, leader) + __popc(bal & ((1u << lane) - 1u));
            if (eq) samp[slot] = ~(uint32_t)cand_idx[j];  // descending ~col == ascending col
          }
        }
        __syncthreads();
        int e2, r2;
        const uint32_t v = list_select<kTopkThreads>(samp, s_n2, rem, hist, hist2, s_sel, s_warp, &e2, &r2);
        tie_lim = (int)~v + 1;  // the highest taken tied column + 1
      }
      if (p.trace && tid == 0) p.trace[blockIdx.x * 16 + 10] = ((unsigned long long)n_cand << 32) | (unsigned)n_eq;
    } else {
      // ---- fallback: full radix select over all keys
      if (p.trace && tid == 0) p.trace[blockIdx.x * 16 + 11] = 1;
      remaining = p.k;
      uint32_t mask = 0;
#pragma unroll 1
      for (int pass = 0; pass < 3; ++pass) {
        const int shift = pass == 0 ? 20 : (pass == 1 ? 10 : 0);
        const int bins = pass == 0 ? 4096 : 1024;
        for (int i = tid; i < bins; i += kTopkThreads) hist[i] = 0;
        __syncthreads();
        for (int base = 0; base < cols; base += kTopkThreads) {
          const int i = base + tid;
          const uint32_t u = i < cols ? key_at(i) : 0u;
          hist_add_agg(hist, i < cols && (u & mask) == prefix, (u >> shift) & (uint32_t)(bins - 1), lane);
        }
        __syncthreads();
        select_bin<kTopkThreads>(hist, bins, remaining, s_warp, s_sel);
        prefix |= (uint32_t)s_sel[0] << shift;
        remaining = s_sel[1];
        mask |= (uint32_t)(bins - 1) << shift;
      }
      if (s_sel[2] != remaining) fast = false;  // rank ties with per-warp counts
    }
  }
  TK_STAMP(4);

  // ---- 4. selection
  const int words = (cols + 31) >> 5;
  if (fast && !p.idx_out && !threshold && staged) {
    // one word per thread: its 32 keys as 8 x 16-byte shared loads, the bit
    // decisions made locally, the words stored coalesced
    for (int w = tid; w < words; w += kTopkThreads) {
      uint32_t bt = 0;
      const int e0 = w << 5;
      if (e0 + 32 <= cols) {
        // the 8 quads are visited in a lane-rotated order: consecutive lanes'
        // words are 128 bytes apart, so an unrotated walk is an 8-way conflict
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c4 = (j + lane) & 7;
          const uint4 u4 = *reinterpret_cast<const uint4*>(keys + e0 + 4 * c4);
          const uint32_t uu[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
          for (int t2 = 0; t2 < 4; ++t2) {
            const int e = e0 + 4 * c4 + t2;
            const bool take = uu[t2] > prefix || (uu[t2] == prefix && e < tie_lim);
            bt |= (take ? 1u : 0u) << (4 * c4 + t2);
          }
        }
      } else {
        for (int e = e0; e < cols; ++e) {
          const uint32_t u = keys[e];
          bt |= ((u > prefix || (u == prefix && e < tie_lim)) ? 1u : 0u) << (e - e0);
        }
      }
      if (p.row_bits) p.row_bits[(size_t)row * words + w] = bt;
      else if (p.bitmap && bt) atomicOr(p.bitmap + w, bt);
    }
  } else if (fast && !p.idx_out) {
    // decide, ballot, store / OR the word
    for (int w = warp; w < words; w += kTopkWarps) {
      const int e = (w << 5) + lane;
      bool take = false;
      if (e < cols) {
        if (threshold) {
          take = logit(e) > p.thr;
        } else {
          const uint32_t u = key_at(e);
          take = u > prefix || (u == prefix && e < tie_lim);
        }
      }
      const uint32_t bt = __ballot_sync(0xffffffffu, take);
      if (lane == 0) {
        if (p.row_bits) p.row_bits[(size_t)row * words + w] = bt;
        else if (p.bitmap && bt) atomicOr(p.bitmap + w, bt);
      }
    }
  } else {
    // index-order: warp-contiguous segments (multiples of 32)
    const int seg = (cols + kTopkThreads - 1) / kTopkThreads * 32;
    const int sbeg = warp * seg, send = min(cols, sbeg + seg);
    auto classify = [&](int e, bool& gt, bool& eq) {
      gt = eq = false;
      if (e < send) {
        const uint32_t u = key_at(e);
        if (fast) {
          gt = u > prefix || (u == prefix && e < tie_lim);
        } else {
          gt = u > prefix;
          eq = u == prefix;
        }
      }
    };
    int n_eq = 0, n_gt = 0;
    for (int e0 = sbeg; e0 < send; e0 += 32) {
      bool gt, eq;
      classify(e0 + lane, gt, eq);
      n_gt += __popc(__ballot_sync(0xffffffffu, gt));
      n_eq += __popc(__ballot_sync(0xffffffffu, eq));
    }
    if (lane == 0) {
      s_eq[warp] = n_eq;
      s_gt[warp] = n_gt;
    }
    __syncthreads();
    int eq_before = 0, gt_before = 0;
    for (int w = 0; w < warp; ++w) {
      eq_before += s_eq[w];
      gt_before += s_gt[w];
    }
    int pos = gt_before + (fast ? 0 : min(eq_before, remaining));
    int eq_run = eq_before;
    const uint32_t lt = (1u << lane) - 1u;
    for (int e0 = sbeg; e0 < send; e0 += 32) {
      bool gt, eq;
      classify(e0 + lane, gt, eq);
      const uint32_t beq = __ballot_sync(0xffffffffu, eq);
      const bool take = gt || (eq && (eq_run + __popc(beq & lt)) < remaining);
      const uint32_t bt = __ballot_sync(0xffffffffu, take);
      eq_run += __popc(beq);
      if (take && p.idx_out) p.idx_out[(size_t)row * p.k + pos + __popc(bt & lt)] = e0 + lane;
      pos += __popc(bt);
      if (lane == 0) {
        if (p.row_bits) p.row_bits[(size_t)row * words + (e0 >> 5)] = bt;
        else if (p.bitmap && bt) atomicOr(p.bitmap + (e0 >> 5), bt);
      }
    }
  }
  TK_STAMP(5);

  // ---- fused union
  if (p.row_bits) {
    const int groups = (p.rows + kGroupRows - 1) / kGroupRows;
    if (p.coresident) {
      // every row CTA is resident (rows <= SMs, one CTA per SM): one grid
      // barrier, then each CTA writes the ascending ids of its own word
      // range -- no single-CTA tail
      // barrier word {gen:32 | count:32} (8-byte aligned inside the ticket
      // head): the last arriver bumps gen and clears count in ONE atomic and
      // does not wait; the others pass on count == rows or a changed gen
      unsigned long long* bar = reinterpret_cast<unsigned long long*>(p.tickets + ((groups + 2) & ~1));
      auto grid_barrier = [&]() {
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          const unsigned long long old = atomicAdd(bar, 1ull);
          const uint32_t g = (uint32_t)(old >> 32);
          if ((uint32_t)old == (uint32_t)p.rows - 1u) {
            atomicAdd(bar, (1ull << 32) - (unsigned long long)p.rows);
          } else {
            while (true) {
              const unsigned long long v = *reinterpret_cast<volatile unsigned long long*>(bar);
              if ((uint32_t)v == (uint32_t)p.rows || (uint32_t)(v >> 32) != g) break;
            }
          }
          __threadfence();
        }
        __syncthreads();
      };
      grid_barrier();
      TK_STAMP(6);
      // every CTA ORs ALL words over the rows (L2-resident, coalesced) and
      // scans their popcounts, so it knows the global prefix of its own word
      // range without a second barrier; it then writes only its range's ids
      const int wlo = p.lo >> 5, whi = (p.hi + 31) >> 5;
      const int nw = whi - wlo;
      const int w0 = wlo + (int)((long long)row * nw / p.rows), w1 = wlo + (int)((long long)(row + 1) * nw / p.rows);
      const int kw = (nw + kTopkThreads - 1) / kTopkThreads;  // contiguous words per thread (<= kUnionWPT)
      const int tw0 = wlo + tid * kw;
      // OR over the rows with 16-byte loads; when the words are few the
      // threads also split the rows (slices), ORed through shared memory
      const int q0 = wlo >> 2, nq = ((whi + 3) >> 2) - q0;
      const bool vec = (words & 3) == 0 && nq <= kTopkThreads;
      const int slices = vec ? max(1, min(kTopkThreads / nq, 8)) : 0;
      uint32_t* s_or = reinterpret_cast<uint32_t*>(hist);  // [slices][nq * 4]
      if (vec) {
        const int sl = tid / nq, qq = tid - sl * nq;
        if (sl < slices) {
          const uint4* rb = reinterpret_cast<const uint4*>(p.row_bits) + q0 + qq;
          const int wq = words >> 2;
          uint4 acc4 = make_uint4(0, 0, 0, 0);
          for (int r0 = sl; r0 < p.rows; r0 += 8 * slices) {
            uint4 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int r = r0 + j * slices;
              v[j] = r < p.rows ? __ldcg(rb + (size_t)r * wq) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              acc4.x |= v[j].x; acc4.y |= v[j].y; acc4.z |= v[j].z; acc4.w |= v[j].w;
            }
          }
          reinterpret_cast<uint4*>(s_or)[sl * nq + qq] = acc4;
        }
        __syncthreads();
      }
      TK_STAMP(8);
      uint32_t wb[kUnionWPT];
      int cnt = 0;
#pragma unroll
      for (int j = 0; j < kUnionWPT; ++j) {
        const int w = tw0 + j;
        uint32_t acc = 0;
        if (j < kw && w < whi) {
          if (vec) {
            for (int sl = 0; sl < slices; ++sl) acc |= s_or[sl * nq * 4 + (w - 4 * q0)];
          } else {
            // 32 loads in flight per batch (one L2 round trip per 32 rows)
            for (int r0 = 0; r0 < p.rows; r0 += 32) {
              uint32_t v[32];
#pragma unroll
              for (int r = 0; r < 32; ++r) v[r] = r0 + r < p.rows ? __ldcg(p.row_bits + (size_t)(r0 + r) * words + w) : 0u;
#pragma unroll
              for (int r = 0; r < 32; ++r) acc |= v[r];
            }
          }
          const int top = p.hi - (w << 5);
          if (top < 32) acc &= (top <= 0) ? 0u : ((1u << top) - 1u);
        }
        wb[j] = acc;
        cnt += __popc(acc);
      }
      int total;
      int pos = block_excl_scan<kTopkThreads>(cnt, s_warp, &total);
      TK_STAMP(9);
#pragma unroll
      for (int j = 0; j < kUnionWPT; ++j) {
        const int w = tw0 + j;
        uint32_t bits = wb[j];
        if (w >= w0 && w < w1) {
          while (bits) {
            const int b2 = __ffs(bits) - 1;
            bits &= bits - 1;
            p.union_out[pos++] = (w << 5) + b2 - p.lo;
          }
        } else {
          pos += __popc(bits);
        }
      }
      if (row == 0 && tid == 0) *p.count_out = total;
      // the CTA whose range holds the last id pads idx_out up to a multiple of pad
      __shared__ int s_range[2];
      if (tid == 0) { s_range[0] = 0x7fffffff; s_range[1] = -1; }
      __syncthreads();
      {
        // global positions covered by this CTA's words
        int lo_pos = 0x7fffffff, hi_pos = -1, p2 = pos;
        for (int j = kUnionWPT - 1; j >= 0; --j) {
          const int w = tw0 + j;
          p2 -= __popc(wb[j]);
          if (w >= w0 && w < w1 && wb[j]) {
            lo_pos = min(lo_pos, p2);
            hi_pos = max(hi_pos, p2 + __popc(wb[j]) - 1);
          }
        }
        if (hi_pos >= 0) {
          atomicMin(&s_range[0], lo_pos);
          atomicMax(&s_range[1], hi_pos);
        }
      }
      __syncthreads();
      if (p.pad > 1 && total > 0 && s_range[1] == total - 1) {
        const int padded = (total + p.pad - 1) / p.pad * p.pad;
        const int32_t last = p.union_out[total - 1];
        for (int i = total + tid; i < padded; i += kTopkThreads) p.union_out[i] = last;
      }
      TK_STAMP(7);
      return;
    }
    // rows > SMs: the last CTA of each group of 16 rows ORs the group, and
    // the last group compacts
    const int g = row / kGroupRows;
    const int g_rows = min(kGroupRows, p.rows - g * kGroupRows);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&p.tickets[g], 1) == g_rows - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const uint32_t* gb = p.row_bits + (size_t)g * kGroupRows * words;
    for (int w = tid; w < words; w += kTopkThreads)
      p.group_bits[(size_t)g * words + w] = or_rows<kGroupRows>(gb, g_rows, words, w);
    if (tid == 0) p.tickets[g] = 0;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&p.tickets[groups], 1) == groups - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const uint32_t* gbits = p.group_bits;
    if (groups <= 4)
      compact_words<kTopkThreads>([&](int w) { return or_rows<4>(gbits, groups, words, w); }, p.lo, p.hi, p.pad,
                                  p.union_out, p.count_out, s_warp);
    else
      compact_words<kTopkThreads>([&](int w) { return or_rows<kMaxGroups>(gbits, groups, words, w); }, p.lo, p.hi,
                                  p.pad, p.union_out, p.count_out, s_warp);
    if (tid == 0) p.tickets[groups] = 0;
    TK_STAMP(6);
  }
}

size_t topk_smem(int cols, bool threshold) {
  size_t b = (size_t)4096 * 4 + (size_t)kMaxCand * 4 * 5;
  if (!threshold && cols <= kTopkSmemCols) b += (size_t)cols * 4;
  return b;
}

unsigned long long* g_topk_trace = nullptr;

int launch_topk(TopkParams prm, cudaStream_t st) {
  prm.trace = g_topk_trace;
  const size_t smem = topk_smem(prm.cols, prm.k <= 0);
  static int configured = 0;
  if (!configured) {
    if (cudaFuncSetAttribute(topk_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024) !=
        cudaSuccess)
      return PS_ERR_CUDA;
    configured = 1;
  }
  if (prm.coresident) {
    // grid-barrier union: a cooperative launch guarantees co-residency
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(prm.rows);
    cfg.blockDim = dim3(kTopkThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, topk_rows_kernel, prm) != cudaSuccess) return PS_ERR_CUDA;
    return launch_status();
  }
  return launch_ex(topk_rows_kernel, dim3(prm.rows), dim3(kTopkThreads), smem, st, 1, prm);
}

__global__ void union_rows_kernel(const int32_t* __restrict__ ids, int n, int width, uint32_t* __restrict__ bitmap) {
  griddep_wait();
  griddep_launch();
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int i = ids[e];
    if (i >= 0 && i < width) atomicOr(bitmap + (i >> 5), 1u << (i & 31));
  }
}

constexpr int kCompactThreads = 1024;

// Ascending ids of the set bits; clears the bitmap; pads idx_out with the
// last id up to a multiple of `pad`; device-resident count (no host sync).
__global__ void __launch_bounds__(kCompactThreads) bitmap_compact_kernel(uint32_t* __restrict__ bitmap, int width,
                                                                         int lo, int hi, int pad,
                                                                         int32_t* __restrict__ idx_out,
                                                                         int32_t* __restrict__ count_out) {
  __shared__ int s_warp[32];
  __shared__ int s_total;
  griddep_wait();
  griddep_launch();
  const int words = (width + 31) >> 5;
  const int wlo = lo >> 5, whi = (hi + 31) >> 5;
  const int nw = whi - wlo;
  const int per = (nw + kCompactThreads - 1) / kCompactThreads;
  const int w0 = wlo + min(nw, (int)threadIdx.x * per), w1 = wlo + min(nw, (int)(threadIdx.x + 1) * per);
  auto word = [&](int w) {
    uint32_t bits = bitmap[w];
    const int top = hi - (w << 5);  // bits at or above `hi` belong to another shard
    if (top < 32) bits &= (top <= 0) ? 0u : ((1u << top) - 1u);
    return bits;
  };
  int cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(word(w));
  int total;
  int pos = block_excl_scan<kCompactThreads>(cnt, s_warp, &total);
  for (int w = w0; w < w1; ++w) {
    uint32_t bits = word(w);
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      idx_out[pos++] = (w << 5) + b - lo;
    }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < words; w += kCompactThreads) bitmap[w] = 0u;
  if (threadIdx.x == 0) {
    *count_out = total;
    s_total = total;
  }
  __syncthreads();
  if (pad > 1) {
    const int padded = (s_total + pad - 1) / pad * pad;
    __syncthreads();
    const int32_t last = s_total > 0 ? idx_out[s_total - 1] : 0;
    for (int i = s_total + threadIdx.x; i < padded; i += kCompactThreads) idx_out[i] = last;
  }
}

// Head router fused with top-k (routers.py:324-325 + tensors.py:65-73).
// One thread-block CLUSTER per group of R batch rows: CTA j of the cluster
// computes the logits of heads [j*HB, (j+1)*HB) for those rows (each warp
// one (head, d-segment) item, all of a lane's 16-byte W^T loads independent
// so they are in flight together), and stores them into CTA 0's shared
// memory through DSMEM; after one cluster barrier CTA 0 ranks every row
// (one warp per row).  The whole W^T (H x d bf16) is read once per cluster,
// from L2 after the first cluster.
constexpr int kHrThreads = 256;
constexpr int kHrWarps = kHrThreads / 32;
constexpr int kHrMaxHeads = 256;
constexpr int kHrMaxRows = 4;

// Optional fused KV append (ps_head_router_topk_append): the cluster of row
// group r0.. also writes the step's K/V rows (tensors.py:150-170) -- CTA j
// copies cache heads [j*hb, (j+1)*hb) -- and CTA 0 bumps lengths after the
// cluster barrier, saving the separate append launch.
struct AppendArgs {
  uint16_t* kc;
  uint16_t* vc;
  int32_t* lengths;
  const uint16_t* kn;
  const uint16_t* vn;
  int64_t src_ld;
  int Hc, cap, d_h;
  int32_t* err;
  // paged caches (pages, Hc, page_rows, d_h): NULL = contiguous (B, Hc, cap, d_h)
  const int32_t* table;
  int64_t table_ld;
  int page_rows;
};

template <int R>
__global__ void __launch_bounds__(kHrThreads) head_router_topk_kernel(
    const uint16_t* __restrict__ x, int64_t x_ld, const uint16_t* __restrict__ w_t, const float* __restrict__ bias,
    int B, int d, int H, int HB, int k, float* __restrict__ logits_out, int32_t* __restrict__ sel_out,
    const AppendArgs ap) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ float s_log[kHrMaxRows * kHrMaxHeads];          // CTA 0: the cluster's logits
  __shared__ float s_part[kHrWarps * 2][kHrMaxRows];         // per-item partial sums
  uint16_t* sx = reinterpret_cast<uint16_t*>(smem);          // [R][d]
  const int crank = (int)cluster_rank(), csize = (int)cluster_size();
  griddep_wait();
  griddep_launch();
  const int r0 = (blockIdx.x / csize) * R;
  const int nr = min(R, B - r0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int chunks = d >> 3;
  // CTA 0's arrival barrier for the cluster's logits (st.async complete_tx);
  // every CTA of the cluster must have started before its DSMEM is written
  __shared__ uint64_t s_bar;
  if (crank == 0 && tid == 0) {
    mbar_init(&s_bar, 1);
    fence_mbar_init();
  }
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  for (int c = tid; c < R * chunks; c += kHrThreads) {
    const int r = c / chunks, cc = c - r * chunks;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < nr) v = *reinterpret_cast<const uint4*>(x + (size_t)(r0 + r) * x_ld + cc * 8);
    *reinterpret_cast<uint4*>(sx + r * d + cc * 8) = v;
  }
  if (ap.kc) {
    const int hb = (ap.Hc + csize - 1) / csize, ha0 = crank * hb, ha1 = min(ap.Hc, ha0 + hb);
    const int vph = ap.d_h >> 3;
    for (int r = 0; r < nr; ++r) {
      const int b = r0 + r;
      const int pos = ap.lengths[b];
      if (pos >= ap.cap) {
        if (tid == 0 && crank == 0 && ap.err) *ap.err = 1;
        continue;
      }
      const int total = max(0, ha1 - ha0) * vph;
      // row of (b, head 0) at pos, heads `hs` rows apart (contiguous or paged)
      size_t rb, hs;
      if (ap.table) {
        const int pg = __ldg(ap.table + (size_t)b * ap.table_ld + pos / ap.page_rows);
        if (pg < 0) {  // unmapped page: nothing written, length kept (below)
          if (tid == 0 && crank == 0 && ap.err) *ap.err = 2;
          continue;
        }
        rb = (size_t)pg * ap.Hc * ap.page_rows + pos % ap.page_rows;
        hs = ap.page_rows;
      } else {
        rb = (size_t)b * ap.Hc * ap.cap + pos;
        hs = ap.cap;
      }
      for (int e = tid; e < total; e += kHrThreads) {
        const int h = ha0 + e / vph, c = e - (e / vph) * vph;
        const size_t src = (size_t)b * ap.src_ld + (size_t)h * ap.d_h + c * 8;
        const size_t dst = (rb + h * hs) * ap.d_h + c * 8;
        const uint4 kv = __ldg(reinterpret_cast<const uint4*>(ap.kn + src));
        const uint4 vv = __ldg(reinterpret_cast<const uint4*>(ap.vn + src));
        *reinterpret_cast<uint4*>(ap.kc + dst) = kv;
        *reinterpret_cast<uint4*>(ap.vc + dst) = vv;
      }
    }
  }
  const int h0 = crank * HB;
  const int hn = max(0, min(HB, H - h0));
  // items = (head, segment); segments per head so that every warp has work
  const int segs = hn > 0 ? max(1, kHrWarps / hn) : 1;
  const int items = hn * segs;
  const int seg_len = (chunks + segs - 1) / segs;
  __syncthreads();
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  const uint32_t s_log_base = smem_u32(s_log);
  const uint32_t leader_log = map_peer(s_log_base, 0);
  const uint32_t leader_bar = map_peer(smem_u32(&s_bar), 0);
  if (crank == 0 && tid == 0) mbar_arrive_expect_tx(&s_bar, (uint32_t)(nr * H * 4));
  for (int it0 = 0; it0 < items; it0 += kHrWarps) {
    const int it = it0 + warp;
    if (it < items) {
      const int hh = it / segs, sg = it - hh * segs;
      const int c0 = sg * seg_len, c1 = min(chunks, c0 + seg_len);
      const uint16_t* wr = w_t + (size_t)(h0 + hh) * d;
      float acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.f;
#pragma unroll 8
      for (int c = c0 + lane; c < c1; c += 32) {
        float wf[8], xf[8];
        unpack8(__ldg(reinterpret_cast<const uint4*>(wr + c * 8)), wf);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          unpack8(*reinterpret_cast<const uint4*>(sx + r * d + c * 8), xf);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[r] = fmaf(wf[i], xf[i], acc[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float v = warp_sum(acc[r]);
        if (lane == 0) s_part[warp][r] = v;
      }
    }
    __syncthreads();
    // combine the segments of each head of this round; ship to CTA 0
    const int n_round = min(kHrWarps, items - it0);
    if (tid < R * kHrWarps) {
      const int r = tid / kHrWarps, j = tid - r * kHrWarps;  // j: item slot in this round
      if (j < n_round && r < nr) {
        const int item = it0 + j, hh = item / segs, sg = item - hh * segs;
        if (sg == 0) {
          float v = 0.f;
          for (int q = 0; q < segs; ++q) v += s_part[j + q][r];  // segments of a head are adjacent slots
          const int h = h0 + hh;
          v += bias ? bias[h] : 0.f;
          st_async_f32(leader_log + (uint32_t)(r * H + h) * 4u, v, leader_bar);
        }
      }
    }
    __syncthreads();
  }
  if (crank != 0) return;
  mbar_wait(&s_bar, 0);  // every CTA's logits landed (they read lengths[] before sending)
  // every CTA of the cluster read lengths[] before its logits arrived: bump them now
  if (ap.kc && tid < nr) {
    const int b = r0 + tid, pos = ap.lengths[b];
    const bool mapped = !ap.table || __ldg(ap.table + (size_t)b * ap.table_ld + pos / ap.page_rows) >= 0;
    if (pos < ap.cap && mapped) ap.lengths[b] = pos + 1;
  }
  // top-k of each row by rank counting, one warp per row
  if (warp < nr) {
    const int r = warp;
    const float* lr = s_log + r * H;
    if (logits_out)
      for (int i = lane; i < H; i += 32) logits_out[(size_t)(r0 + r) * H + i] = lr[i];
    int base = 0;
    for (int i0 = 0; i0 < H; i0 += 32) {
      const int i = i0 + lane;
      bool take = false;
      if (i < H) {
        const uint32_t ki = order_key(lr[i]);
        int rank = 0;
        for (int j = 0; j < H; ++j) {
          const uint32_t kj = order_key(lr[j]);
          rank += (kj > ki) || (kj == ki && j < i);
        }
        take = rank < k;
      }
      const uint32_t ballot = __ballot_sync(0xffffffffu, take);
      if (take) sel_out[(size_t)(r0 + r) * k + base + __popc(ballot & ((1u << lane) - 1u))] = i;
      base += __popc(ballot);
    }
  }
}

template <int R>
int launch_head_router(const uint16_t* x, int64_t x_ld, const uint16_t* w_t, const float* bias, int B, int d,
                       int H, int k, float* logits_out, int32_t* sel_out, const AppendArgs& ap, cudaStream_t st) {
  auto kern = head_router_topk_kernel<R>;
  const size_t smem = (size_t)R * d * 2;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024) != cudaSuccess)
      return PS_ERR_CUDA;
    configured = true;
  }
  static const int cmax = [] {
    const char* e = getenv("PS_HR_CLUSTER");  // tuning hook: CTAs per row group (1..8)
    const int v = e ? atoi(e) : 4;  // 4 measured best on B200 (B=64, H_kv=32)
    return v < 2 ? 2 : (v > 8 ? 8 : v);
  }();
  // >= 2: the kernel uses cluster barriers / DSMEM, which need a cluster
  // launch (a CTA of the pair may own no head, e.g. H == 1)
  const int csize = H < 2 ? 2 : (H < cmax ? H : cmax);
  const int HB = (H + csize - 1) / csize;
  const int groups = (B + R - 1) / R;
  return launch_ex(kern, dim3(groups * csize), dim3(kHrThreads), smem, st, csize, x, x_ld, w_t, bias, B, d, H, HB, k,
                   logits_out, sel_out, ap);
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" int ps_topk_rows(const float* logits, int rows, int cols, int64_t ld, int k, int32_t* idx_out,
                            uint32_t* bitmap, void* stream) {
  if (rows < 1 || cols < 1 || ld < cols || k < 1 || k > cols || !logits) return PS_ERR_VALUE;
  if (!idx_out && !bitmap) return PS_ERR_VALUE;
  TopkParams prm{};
  prm.logits = logits; prm.rows = rows; prm.cols = cols; prm.ld = ld; prm.k = k;
  prm.idx_out = idx_out; prm.bitmap = bitmap;
  return launch_topk(prm, static_cast<cudaStream_t>(stream));
}

extern "C" int ps_threshold_rows(const float* logits, int rows, int cols, int64_t ld, float thr, uint32_t* bitmap,
                                 void* stream) {
  if (rows < 1 || cols < 1 || ld < cols || !logits || !bitmap) return PS_ERR_VALUE;
  TopkParams prm{};
  prm.logits = logits; prm.rows = rows; prm.cols = cols; prm.ld = ld; prm.k = 0; prm.thr = thr;
  prm.bitmap = bitmap;
  return launch_topk(prm, static_cast<cudaStream_t>(stream));
}

static size_t su_words(int cols) { return (size_t)(cols + 31) / 32; }
static size_t su_groups(int rows) { return (size_t)(rows + kGroupRows - 1) / kGroupRows; }

extern "C" size_t ps_select_union_workspace_bytes(int rows, int cols) {
  if (rows < 1 || cols < 1) return 0;
  const size_t tickets = (su_groups(rows) + 3 + (size_t)rows) * 4;
  const size_t head = (tickets + 255) / 256 * 256;
  // + the low-latency kernel's region: a ticket (256 B) and one union bitmap
  return head + (su_groups(rows) + (size_t)rows) * su_words(cols) * 4 + 256 + su_words(cols) * 4;
}

namespace ps {
int select_union_v2(const float* logits, const float* bias, int rows, int cols, int64_t ld, int k, float thr,
                    int* ticket, uint32_t* bitmap, int lo, int hi, int pad, int32_t* union_out, int32_t* count_out,
                    unsigned long long* trace, cudaStream_t st);
int select_union_v2_max_cols();
int select_union_v2_bitmap(const float* logits, const float* bias, int rows, int cols, int64_t ld, int k, float thr,
                           uint32_t* bitmap, uint32_t* clear, unsigned long long* trace, cudaStream_t st);
}  // namespace ps
static int g_topk_v2 = -1;  // -1: from env PS_TOPK_V2 (default 1)
static const int g_topk_coop = [] {
  const char* e = getenv("PS_TOPK_COOP");
  return e ? atoi(e) : 0;
}();
extern "C" void ps_debug_topk_v2(int enable) { g_topk_v2 = enable ? 1 : 0; }

extern "C" int ps_select_union(const float* logits, const float* bias, int rows, int cols, int64_t ld, int k,
                               float thr, void* ws, size_t ws_bytes, int lo, int hi, int pad, int32_t* union_out,
                               int32_t* count_out, void* stream) {
  if (rows < 1 || cols < 1 || ld < cols || k > cols || !logits || !ws || !union_out || !count_out)
    return PS_ERR_VALUE;
  if (rows > kGroupRows * kMaxGroups) return PS_ERR_UNSUPPORTED;
  if (lo < 0 || lo % 32 || hi > cols || hi <= lo || pad < 1) return PS_ERR_VALUE;
  if (ws_bytes < ps_select_union_workspace_bytes(rows, cols)) return PS_ERR_WORKSPACE;
  const size_t tickets = (su_groups(rows) + 3 + (size_t)rows) * 4;
  const size_t head = (tickets + 255) / 256 * 256;
  uint8_t* base = static_cast<uint8_t*>(ws);
  if (g_topk_v2 < 0) {
    const char* e = getenv("PS_TOPK_V2");
    g_topk_v2 = e ? atoi(e) : 1;
  }
  if (g_topk_v2 && cols <= select_union_v2_max_cols()) {
    uint8_t* v2 = base + head + (su_groups(rows) + (size_t)rows) * su_words(cols) * 4;
    return select_union_v2(logits, bias, rows, cols, ld, k > 0 ? k : 0, thr, reinterpret_cast<int*>(v2),
                           reinterpret_cast<uint32_t*>(v2 + 256), lo, hi, pad, union_out, count_out, g_topk_trace,
                           static_cast<cudaStream_t>(stream));
  }
  TopkParams prm{};
  prm.logits = logits; prm.rows = rows; prm.cols = cols; prm.ld = ld; prm.k = k > 0 ? k : 0; prm.thr = thr;
  prm.bias = bias;
  // one CTA per row and per SM (the kernel's shared memory): all resident
  // at once iff rows <= SMs, and every CTA owns <= 512 words
  // the grid-barrier union needs every row CTA resident at once, which a
  // plain launch does not guarantee: it is used only under a cooperative
  // launch (PS_TOPK_COOP=1); otherwise the ticketed group union (no waits)
  prm.coresident = g_topk_coop && rows <= ps_num_sms() && (cols + 31) / 32 <= (size_t)kUnionWPT * kTopkThreads;
  prm.tickets = reinterpret_cast<int*>(base);
  prm.group_bits = reinterpret_cast<uint32_t*>(base + head);
  prm.row_bits = prm.group_bits + su_groups(rows) * su_words(cols);
  prm.lo = lo; prm.hi = hi; prm.pad = pad;
  prm.union_out = union_out; prm.count_out = count_out;
  return launch_topk(prm, static_cast<cudaStream_t>(stream));
}

// Union hand-off: the rows' top-k (or threshold) sets OR-ed into `bitmap`
// (ceil(cols / 32) words, zero on entry) and nothing else -- the gathered
// GEMMs read the bitmap (PS_GG_BITMAP).  CTA 0 zeroes `clear` (may be NULL),
// the buffer the previous layer used, so two buffers alternate.
extern "C" int ps_select_union_bitmap(const float* logits, const float* bias, int rows, int cols, int64_t ld, int k,
                                      float thr, uint32_t* bitmap, uint32_t* clear, void* stream) {
  if (rows < 1 || cols < 1 || ld < cols || k > cols || !logits || !bitmap || bitmap == clear) return PS_ERR_VALUE;
  if (cols > select_union_v2_max_cols()) return PS_ERR_UNSUPPORTED;
  return select_union_v2_bitmap(logits, bias, rows, cols, ld, k > 0 ? k : 0, thr, bitmap, clear, g_topk_trace,
                                static_cast<cudaStream_t>(stream));
}

extern "C" void ps_debug_topk_trace(void* buf) { g_topk_trace = static_cast<unsigned long long*>(buf); }

extern "C" int ps_union_rows(const int32_t* rows_idx, int rows, int k, int width, uint32_t* bitmap, void* stream) {
  if (rows < 1 || k < 1 || width < 1 || !rows_idx || !bitmap) return PS_ERR_VALUE;
  const int n = rows * k;
  int grid = (n + 255) / 256;
  if (grid > 1184) grid = 1184;
  return launch_ex(union_rows_kernel, dim3(grid), dim3(256), 0, static_cast<cudaStream_t>(stream), 1, rows_idx, n,
                   width, bitmap);
}

extern "C" int ps_bitmap_compact(uint32_t* bitmap, int width, int lo, int hi, int pad, int32_t* idx_out,
                                 int32_t* count_out, void* stream) {
  if (width < 1 || !bitmap || !idx_out || !count_out || pad < 1) return PS_ERR_VALUE;
  if (lo < 0 || lo % 32 || hi > width || hi <= lo) return PS_ERR_VALUE;
  return launch_ex(bitmap_compact_kernel, dim3(1), dim3(kCompactThreads), 0, static_cast<cudaStream_t>(stream), 1,
                   bitmap, width, lo, hi, pad, idx_out, count_out);
}

static int head_router_common(const void* x, int64_t x_ld, const void* w_t, const float* bias, int B, int d, int H_kv,
                              int k, float* logits_out, int32_t* sel_out, const AppendArgs& ap, void* stream) {
  if (B < 1 || d < 8 || d % 8 || H_kv < 1 || H_kv > kHrMaxHeads || k < 1 || k > H_kv) return PS_ERR_VALUE;
  if (!x || !w_t || !sel_out || x_ld < d || x_ld % 8) return PS_ERR_VALUE;
  if ((size_t)kHrMaxRows * d * 2 > 160 * 1024) return PS_ERR_UNSUPPORTED;
  const auto* xp = static_cast<const uint16_t*>(x);
  const auto* wp = static_cast<const uint16_t*>(w_t);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // rows per cluster: keep >= ~64 clusters in flight, fewer W^T re-reads at large batch
  if (B >= 256) return launch_head_router<4>(xp, x_ld, wp, bias, B, d, H_kv, k, logits_out, sel_out, ap, st);
  if (B >= 128) return launch_head_router<2>(xp, x_ld, wp, bias, B, d, H_kv, k, logits_out, sel_out, ap, st);
  return launch_head_router<1>(xp, x_ld, wp, bias, B, d, H_kv, k, logits_out, sel_out, ap, st);
}

extern "C" int ps_head_router_topk(const void* x, int64_t x_ld, const void* w_t, const float* bias, int B, int d,
                                   int H_kv, int k, float* logits_out, int32_t* sel_out, void* stream) {
  AppendArgs ap{};
  return head_router_common(x, x_ld, w_t, bias, B, d, H_kv, k, logits_out, sel_out, ap, stream);
}

extern "C" int ps_head_router_topk_append(const void* x, int64_t x_ld, const void* w_t, const float* bias, int B,
                                          int d, int H_kv, int k, float* logits_out, int32_t* sel_out,
                                          void* k_cache, void* v_cache, int32_t* lengths, const void* k_new,
                                          const void* v_new, int64_t src_ld, int H_cache, int cap, int d_h,
                                          int32_t* err_flag, void* stream) {
  if (!k_cache || !v_cache || !lengths || !k_new || !v_new || H_cache < 1 || cap < 1 || d_h < 8 || d_h % 8 ||
      src_ld < (int64_t)H_cache * d_h || src_ld % 8)
    return PS_ERR_VALUE;
  if (((uintptr_t)k_new % 16) || ((uintptr_t)v_new % 16) || ((uintptr_t)k_cache % 16) || ((uintptr_t)v_cache % 16))
    return PS_ERR_VALUE;
  AppendArgs ap{static_cast<uint16_t*>(k_cache), static_cast<uint16_t*>(v_cache), lengths,
                static_cast<const uint16_t*>(k_new), static_cast<const uint16_t*>(v_new), src_ld, H_cache, cap, d_h,
                err_flag, nullptr, 0, 0};
  return head_router_common(x, x_ld, w_t, bias, B, d, H_kv, k, logits_out, sel_out, ap, stream);
}

extern "C" int ps_head_router_topk_append_paged(const void* x, int64_t x_ld, const void* w_t, const float* bias,
                                                int B, int d, int H_kv, int k, float* logits_out, int32_t* sel_out,
                                                void* k_pool, void* v_pool, int page_rows,
                                                const int32_t* block_table, int64_t table_ld, int32_t* lengths,
                                                const void* k_new, const void* v_new, int64_t src_ld, int H_cache,
                                                int d_h, int32_t* err_flag, void* stream) {
  if (!k_pool || !v_pool || !block_table || !lengths || !k_new || !v_new || H_cache < 1 || page_rows < 1 ||
      table_ld < 1 || d_h < 8 || d_h % 8 || src_ld < (int64_t)H_cache * d_h || src_ld % 8)
    return PS_ERR_VALUE;
  if (((uintptr_t)k_new % 16) || ((uintptr_t)v_new % 16) || ((uintptr_t)k_pool % 16) || ((uintptr_t)v_pool % 16))
    return PS_ERR_VALUE;
  const long long cap = (long long)table_ld * page_rows;
  if (cap >= (1ll << 31)) return PS_ERR_VALUE;
  AppendArgs ap{static_cast<uint16_t*>(k_pool), static_cast<uint16_t*>(v_pool), lengths,
                static_cast<const uint16_t*>(k_new), static_cast<const uint16_t*>(v_new), src_ld, H_cache, (int)cap,
                d_h, err_flag, block_table, table_ld, page_rows};
  return head_router_common(x, x_ld, w_t, bias, B, d, H_kv, k, logits_out, sel_out, ap, stream);
}
