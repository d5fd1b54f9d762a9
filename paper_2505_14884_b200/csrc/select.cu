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

// One CTA per row: 4-pass 8-bit radix select of the k-th largest key, then
// an index-order pass that keeps every key above it and the lowest-index
// ties up to k (exactly the stable-argsort rule).
__global__ void __launch_bounds__(kTopkThreads) topk_rows_kernel(const float* __restrict__ logits, int cols,
                                                                 int64_t ld, int k, int32_t* __restrict__ idx_out,
                                                                 uint32_t* __restrict__ bitmap) {
  __shared__ int hist[256];
  __shared__ int s_warp[32];
  __shared__ uint32_t s_prefix;
  __shared__ int s_remaining;
  const int row = blockIdx.x;
  const float* x = logits + (size_t)row * ld;
  const int tid = threadIdx.x;

  uint32_t prefix = 0, mask = 0;
  int remaining = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += kTopkThreads) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < cols; i += kTopkThreads) {
      const uint32_t u = order_key(__ldg(x + i));
      if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1);
    }
    __syncthreads();
    if (tid < 32) {
      int loc[8], lsum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        loc[j] = hist[tid * 8 + j];
        lsum += loc[j];
      }
      int incl = lsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += y;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      int cum = total - incl;  // count in bins above this lane's range
#pragma unroll
      for (int j = 7; j >= 0; --j) {
        if (cum < remaining && cum + loc[j] >= remaining) {
          s_prefix = prefix | ((uint32_t)(tid * 8 + j) << shift);
          s_remaining = remaining - cum;
        }
        cum += loc[j];
      }
    }
    __syncthreads();
    prefix = s_prefix;
    remaining = s_remaining;
    mask |= 255u << shift;
    __syncthreads();
  }
  // prefix = k-th largest key; take all keys > prefix and the first
  // `remaining` (lowest-index) keys == prefix.
  const int per = (cols + kTopkThreads - 1) / kTopkThreads;
  const int c0 = min(cols, tid * per), c1 = min(cols, c0 + per);
  int n_eq = 0;
  for (int i = c0; i < c1; ++i) n_eq += (order_key(__ldg(x + i)) == prefix);
  const int eq_before = block_excl_scan<kTopkThreads>(n_eq, s_warp, nullptr);
  int n_sel = 0, eq_seen = eq_before;
  for (int i = c0; i < c1; ++i) {
    const uint32_t u = order_key(__ldg(x + i));
    if (u > prefix) ++n_sel;
    else if (u == prefix) n_sel += (eq_seen++ < remaining);
  }
  int pos = block_excl_scan<kTopkThreads>(n_sel, s_warp, nullptr);
  eq_seen = eq_before;
  for (int i = c0; i < c1; ++i) {
    const uint32_t u = order_key(__ldg(x + i));
    bool take = false;
    if (u > prefix) take = true;
    else if (u == prefix) take = (eq_seen++ < remaining);
    if (take) {
      if (idx_out) idx_out[(size_t)row * k + pos] = i;
      if (bitmap) atomicOr(bitmap + (i >> 5), 1u << (i & 31));
      ++pos;
    }
  }
}

__global__ void threshold_rows_kernel(const float* __restrict__ logits, int rows, int cols, int64_t ld, float thr,
                                      uint32_t* __restrict__ bitmap) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / cols), c = (int)(e - (int64_t)r * cols);
    if (__ldg(logits + (size_t)r * ld + c) > thr) atomicOr(bitmap + (c >> 5), 1u << (c & 31));
  }
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
constexpr int kHrRows = 4;
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
  topk_rows_kernel<<<rows, kTopkThreads, 0, static_cast<cudaStream_t>(stream)>>>(logits, cols, ld, k, idx_out,
                                                                                 bitmap);
  return launch_status();
}

extern "C" int ps_threshold_rows(const float* logits, int rows, int cols, int64_t ld, float thr, uint32_t* bitmap,
                                 void* stream) {
  if (rows < 1 || cols < 1 || ld < cols || !logits || !bitmap) return PS_ERR_VALUE;
  const int64_t total = (int64_t)rows * cols;
  int grid = (int)((total + 255) / 256);
  if (grid > 4 * 148 * 8) grid = 4 * 148 * 8;
  threshold_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(logits, rows, cols, ld, thr, bitmap);
  return launch_status();
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
