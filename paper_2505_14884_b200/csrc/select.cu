// Selection kernels: bit-exact per-row top-k, threshold selection, batch
// union by bitmap + ascending compaction, and the head router fused with its
// top-k.  Ordering contract (tensors.py:54-73, numpy stable argsort of
// -scores): value descending, ties -> lower index, -0.0 == +0.0, NaN ranks
// below -inf (NaNs tied among themselves by index); ids written ascending.
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
constexpr int kTopkSmemCols = 49152;  // rows up to this width are staged in shared memory

struct TopkParams {
  const float* logits;
  int rows, cols;
  int64_t ld;
  int k;            // > 0: top-k per row; <= 0: threshold selection (logit > thr)
  float thr;
  int32_t* idx_out;  // (rows, k) ascending ids, or NULL
  uint32_t* bitmap;  // union bitmap (atomic OR), or NULL
  // fused union compaction by the last CTA (ticket != NULL)
  int* ticket;
  int lo, hi, pad;
  int32_t* union_out;
  int32_t* count_out;
};

// Last-CTA compaction of bitmap bits in [lo, hi) -> ascending ids - lo;
// clears the whole bitmap.  Called by every thread of one CTA.
template <int NT>
PS_DEV void compact_bitmap(uint32_t* bitmap, int width, int lo, int hi, int pad, int32_t* out, int32_t* count,
                           int* s_warp) {
  const int words = (width + 31) >> 5;
  const int wlo = lo >> 5, whi = (hi + 31) >> 5;
  const int nw = whi - wlo;
  const int per = (nw + NT - 1) / NT;
  const int w0 = wlo + min(nw, (int)threadIdx.x * per), w1 = wlo + min(nw, (int)(threadIdx.x + 1) * per);
  auto word = [&](int w) {
    uint32_t bits = __ldcg(bitmap + w);
    const int top = hi - (w << 5);
    if (top < 32) bits &= (top <= 0) ? 0u : ((1u << top) - 1u);
    return bits;
  };
  int cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(word(w));
  int total;
  int pos = block_excl_scan<NT>(cnt, s_warp, &total);
  for (int w = w0; w < w1; ++w) {
    uint32_t bits = word(w);
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      out[pos++] = (w << 5) + b - lo;
    }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < words; w += NT) bitmap[w] = 0u;
  if (threadIdx.x == 0) *count = total;
  if (pad > 1) {
    const int padded = (total + pad - 1) / pad * pad;
    __syncthreads();
    const int32_t last = total > 0 ? out[total - 1] : 0;
    for (int i = total + threadIdx.x; i < padded; i += NT) out[i] = last;
  }
}

// One CTA per row.  Top-k: 3-pass (12/10/10-bit) radix select of the k-th
// largest key over keys staged in shared memory, then ONE index-order pass in which each
// warp owns a contiguous segment and ranks its elements with ballots: keep
// every key above the k-th and the lowest-index ties up to k (exactly the
// stable-argsort rule).  Threshold mode keeps logit > thr.  Each 32-id word
// of the selection is ORed into the union bitmap once, by one lane.
__global__ void __launch_bounds__(kTopkThreads) topk_rows_kernel(const TopkParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  int* hist = reinterpret_cast<int*>(smem);                              // [4096] radix histogram
  uint32_t* keys = reinterpret_cast<uint32_t*>(hist + 4096);              // [cols] if staged
  __shared__ int s_warp[32];
  __shared__ int s_eq[kTopkWarps], s_gt[kTopkWarps];
  __shared__ uint32_t s_prefix;
  __shared__ int s_remaining, s_last;
  const int row = blockIdx.x, cols = p.cols;
  const float* x = p.logits + (size_t)row * p.ld;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool threshold = p.k <= 0;
  const bool staged = !threshold && cols <= kTopkSmemCols;
  auto key_at = [&](int i) -> uint32_t { return staged ? keys[i] : order_key(__ldg(x + i)); };

  uint32_t prefix = 0;
  int remaining = 0;
  if (!threshold) {
    if (staged)
      for (int i = tid; i < cols; i += kTopkThreads) keys[i] = order_key(__ldg(x + i));
    // three radix passes over (12, 10, 10) key bits; only keys matching the
    // prefix found so far touch the histogram, so after the first pass
    // (where the exponent clustering of real logits spreads over ~10^2
    // bins) almost no atomics are issued
    remaining = p.k;
    uint32_t mask = 0;
    const int shifts[3] = {20, 10, 0};
    const int nbins[3] = {4096, 1024, 1024};
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
      const int shift = shifts[pass], bins = nbins[pass];
      for (int i = tid; i < bins; i += kTopkThreads) hist[i] = 0;
      __syncthreads();
      for (int i = tid; i < cols; i += kTopkThreads) {
        const uint32_t u = key_at(i);
        if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & (uint32_t)(bins - 1)], 1);
      }
      __syncthreads();
      // descending scan: thread t owns bins [bins - (t+1)*per, bins - t*per)
      const int per = bins / kTopkThreads;  // 8 or 2
      const int hi = bins - tid * per;
      int loc = 0;
      for (int j = 1; j <= per; ++j) loc += hist[hi - j];
      const int above = block_excl_scan<kTopkThreads>(loc, s_warp, nullptr);
      if (above < remaining && above + loc >= remaining) {
        int cum = above;
        for (int j = 1; j <= per; ++j) {
          const int c = hist[hi - j];
          if (cum + c >= remaining) {
            s_prefix = prefix | ((uint32_t)(hi - j) << shift);
            s_remaining = remaining - cum;
            break;
          }
          cum += c;
        }
      }
      __syncthreads();
      prefix = s_prefix;
      remaining = s_remaining;
      mask |= (uint32_t)(bins - 1) << shift;
      __syncthreads();
    }
  }

  // ---- index-order selection: warp-contiguous segments (multiples of 32)
  const int seg = (cols + kTopkThreads - 1) / kTopkThreads * 32;
  const int sbeg = warp * seg, send = min(cols, sbeg + seg);
  auto classify = [&](int e, bool& gt, bool& eq) {
    gt = eq = false;
    if (e < send) {
      if (threshold) {
        gt = __ldg(x + e) > p.thr;
      } else {
        const uint32_t u = key_at(e);
        gt = u > prefix;
        eq = u == prefix;
      }
    }
  };
  int n_eq = 0, n_gt = 0;
  if (!threshold || p.idx_out) {
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
  }
  int eq_before = 0, gt_before = 0;
  if (!threshold || p.idx_out)
    for (int w = 0; w < warp; ++w) {
      eq_before += s_eq[w];
      gt_before += s_gt[w];
    }
  int pos = gt_before + (threshold ? 0 : min(eq_before, remaining));
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
    if (p.bitmap && lane == 0 && bt) atomicOr(p.bitmap + (e0 >> 5), bt);
  }

  // ---- fused union compaction by the last CTA
  if (p.ticket) {
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(p.ticket, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      compact_bitmap<kTopkThreads>(p.bitmap, cols, p.lo, p.hi, p.pad, p.union_out, p.count_out, s_warp);
      if (tid == 0) *p.ticket = 0;
    }
  }
}

size_t topk_smem(int cols, bool threshold) {
  size_t b = (size_t)4096 * 4;
  if (!threshold && cols <= kTopkSmemCols) b += (size_t)cols * 4;
  return b;
}

int launch_topk(const TopkParams& prm, cudaStream_t st) {
  const size_t smem = topk_smem(prm.cols, prm.k <= 0);
  static int configured = 0;
  if (!configured) {
    if (cudaFuncSetAttribute(topk_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024) !=
        cudaSuccess)
      return PS_ERR_CUDA;
    configured = 1;
  }
  topk_rows_kernel<<<prm.rows, kTopkThreads, smem, st>>>(prm);
  return launch_status();
}

__global__ void union_rows_kernel(const int32_t* __restrict__ ids, int n, int width, uint32_t* __restrict__ bitmap) {
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

// Head router fused with top-k.  R rows per CTA share each 16-byte W^T load.
constexpr int kHrThreads = 256;
constexpr int kHrRows = 1;
constexpr int kHrMaxHeads = 256;

__global__ void __launch_bounds__(kHrThreads) head_router_topk_kernel(
    const uint16_t* __restrict__ x, int64_t x_ld, const uint16_t* __restrict__ w_t, const float* __restrict__ bias,
    int B, int d, int H, int k, float* __restrict__ logits_out, int32_t* __restrict__ sel_out) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint16_t* sx = reinterpret_cast<uint16_t*>(smem);                       // [kHrRows][d]
  float* slog = reinterpret_cast<float*>(smem + (size_t)kHrRows * d * 2);  // [kHrRows][H]
  const int r0 = blockIdx.x * kHrRows;
  const int nr = min(kHrRows, B - r0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int chunks = d / 8;
  for (int c = tid; c < kHrRows * chunks; c += kHrThreads) {
    const int r = c / chunks, cc = c - r * chunks;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < nr) v = *reinterpret_cast<const uint4*>(x + (size_t)(r0 + r) * x_ld + cc * 8);
    *reinterpret_cast<uint4*>(sx + r * d + cc * 8) = v;
  }
  __syncthreads();
  for (int h = warp; h < H; h += kHrThreads / 32) {
    float acc[kHrRows];
#pragma unroll
    for (int r = 0; r < kHrRows; ++r) acc[r] = 0.f;
    for (int cc = lane; cc < chunks; cc += 32) {
      float wf[8], xf[8];
      unpack8(*reinterpret_cast<const uint4*>(w_t + (size_t)h * d + cc * 8), wf);
#pragma unroll
      for (int r = 0; r < kHrRows; ++r) {
        unpack8(*reinterpret_cast<const uint4*>(sx + r * d + cc * 8), xf);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[r] = fmaf(wf[i], xf[i], acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kHrRows; ++r) {
      float v = warp_sum(acc[r]);
      if (lane == 0) slog[r * H + h] = v + (bias ? bias[h] : 0.f);
    }
  }
  __syncthreads();
  // top-k of each row by rank counting (H <= kHrMaxHeads), one warp per row
  if (warp < nr) {
    const int r = warp;
    const float* lr = slog + r * H;
    for (int i = lane; i < H; i += 32) {
      if (logits_out) logits_out[(size_t)(r0 + r) * H + i] = lr[i];
    }
    // selected flags -> ascending positions
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

extern "C" int ps_select_union(const float* logits, int rows, int cols, int64_t ld, int k, float thr,
                               uint32_t* bitmap, int* ticket, int lo, int hi, int pad, int32_t* union_out,
                               int32_t* count_out, void* stream) {
  if (rows < 1 || cols < 1 || ld < cols || k > cols || !logits || !bitmap || !ticket || !union_out || !count_out)
    return PS_ERR_VALUE;
  if (lo < 0 || lo % 32 || hi > cols || hi <= lo || pad < 1) return PS_ERR_VALUE;
  TopkParams prm{};
  prm.logits = logits; prm.rows = rows; prm.cols = cols; prm.ld = ld; prm.k = k > 0 ? k : 0; prm.thr = thr;
  prm.bitmap = bitmap; prm.ticket = ticket; prm.lo = lo; prm.hi = hi; prm.pad = pad;
  prm.union_out = union_out; prm.count_out = count_out;
  return launch_topk(prm, static_cast<cudaStream_t>(stream));
}

extern "C" int ps_union_rows(const int32_t* rows_idx, int rows, int k, int width, uint32_t* bitmap, void* stream) {
  if (rows < 1 || k < 1 || width < 1 || !rows_idx || !bitmap) return PS_ERR_VALUE;
  const int n = rows * k;
  int grid = (n + 255) / 256;
  if (grid > 1184) grid = 1184;
  union_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(rows_idx, n, width, bitmap);
  return launch_status();
}

extern "C" int ps_bitmap_compact(uint32_t* bitmap, int width, int lo, int hi, int pad, int32_t* idx_out,
                                 int32_t* count_out, void* stream) {
  if (width < 1 || !bitmap || !idx_out || !count_out || pad < 1) return PS_ERR_VALUE;
  if (lo < 0 || lo % 32 || hi > width || hi <= lo) return PS_ERR_VALUE;
  bitmap_compact_kernel<<<1, kCompactThreads, 0, static_cast<cudaStream_t>(stream)>>>(bitmap, width, lo, hi, pad,
                                                                                      idx_out, count_out);
  return launch_status();
}

extern "C" int ps_head_router_topk(const void* x, int64_t x_ld, const void* w_t, const float* bias, int B, int d,
                                   int H_kv, int k, float* logits_out, int32_t* sel_out, void* stream) {
  if (B < 1 || d < 8 || d % 8 || H_kv < 1 || H_kv > kHrMaxHeads || k < 1 || k > H_kv) return PS_ERR_VALUE;
  if (!x || !w_t || !sel_out || x_ld < d || x_ld % 8) return PS_ERR_VALUE;
  const size_t smem = (size_t)kHrRows * d * 2 + (size_t)kHrRows * H_kv * 4;
  if (smem > 200 * 1024) return PS_ERR_UNSUPPORTED;
  static int configured = 0;
  if (!configured) {
    if (cudaFuncSetAttribute(head_router_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
        cudaSuccess)
      return PS_ERR_CUDA;
    configured = 1;
  }
  const int grid = (B + kHrRows - 1) / kHrRows;
  head_router_topk_kernel<<<grid, kHrThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(x), x_ld, static_cast<const uint16_t*>(w_t), bias, B, d, H_kv, k, logits_out,
      sel_out);
  return launch_status();
}
