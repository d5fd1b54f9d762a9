// Decode-step glue around the hot path + library metadata.
//   * ps_kv_append  -- KVCache.append_step (tensors.py:150-170)
//   * ps_layernorm  -- model.layernorm (model.py:168-175)
//   * ps_embed      -- token + position embedding (engine.py:342)
#include "common.cuh"

namespace ps {
namespace {

// one CTA per sequence: copy H_kv*d_h new keys/values to row lengths[b],
// then bump lengths[b].  Every thread issues all of its 16-byte loads before
// its stores (one memory latency per CTA).  A full sequence is left
// untouched (err_flag = 1), and so is one whose next row falls in an unmapped
// page (block-table entry < 0; err_flag = 2).
constexpr int kKvThreads = 512;
constexpr int kKvVec = 4;  // 16-byte vectors per thread per tensor (H_kv*d_h <= 16384)

__global__ void __launch_bounds__(kKvThreads) kv_append_kernel(uint16_t* __restrict__ kc, uint16_t* __restrict__ vc,
                                                               int32_t* __restrict__ lengths,
                                                               const uint16_t* __restrict__ kn,
                                                               const uint16_t* __restrict__ vn, int64_t src_ld,
                                                               int H_kv, int cap, int d_h, int32_t* err_flag,
                                                               const int32_t* __restrict__ table, int64_t table_ld,
                                                               int page_rows) {
  const int b = blockIdx.x;
  griddep_wait();
  griddep_launch();
  const int pos = lengths[b];
  if (pos >= cap) {
    if (threadIdx.x == 0 && err_flag) *err_flag = 1;
    return;
  }
  // row base of (b, head 0) at `pos`; heads are `hstride` rows apart
  size_t base;
  size_t hstride;
  if (table) {  // paged pool (pages, H_kv, page_rows, d_h)
    const int pg = __ldg(table + (size_t)b * table_ld + pos / page_rows);
    if (pg < 0) {  // the page holding `pos` was never mapped: write nothing, keep the length
      if (threadIdx.x == 0 && err_flag) *err_flag = 2;
      return;
    }
    base = (size_t)pg * H_kv * page_rows + pos % page_rows;
    hstride = page_rows;
  } else {
    base = (size_t)b * H_kv * cap + pos;
    hstride = cap;
  }
  const int vec_per_head = d_h / 8;
  const int total = H_kv * vec_per_head;
  for (int e0 = 0; e0 < total; e0 += kKvThreads * kKvVec) {
    uint4 kr[kKvVec], vr[kKvVec];
#pragma unroll
    for (int j = 0; j < kKvVec; ++j) {
      const int e = e0 + j * kKvThreads + threadIdx.x;
      if (e < total) {
        const int h = e / vec_per_head, c = e - h * vec_per_head;
        const size_t src = (size_t)b * src_ld + (size_t)h * d_h + c * 8;
        kr[j] = __ldg(reinterpret_cast<const uint4*>(kn + src));
        vr[j] = __ldg(reinterpret_cast<const uint4*>(vn + src));
      }
    }
#pragma unroll
    for (int j = 0; j < kKvVec; ++j) {
      const int e = e0 + j * kKvThreads + threadIdx.x;
      if (e < total) {
        const int h = e / vec_per_head, c = e - h * vec_per_head;
        const size_t dst = (base + h * hstride) * d_h + c * 8;
        *reinterpret_cast<uint4*>(kc + dst) = kr[j];
        *reinterpret_cast<uint4*>(vc + dst) = vr[j];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) lengths[b] = pos + 1;
}

// LayerNorm of one f32 row per CTA held in registers (float4 per slot):
// optional pending-bias add (x += add, written back -- the bias of the
// projection whose GEMM wrote x), two-pass mean / variance from registers,
// bf16 output with 8-byte stores.
constexpr int kLnThreads = 256;
constexpr int kLnSlots = 16;  // float4 per thread: d <= 16384

template <bool ADD>
__global__ void __launch_bounds__(kLnThreads) layernorm_kernel(float* __restrict__ x, int64_t x_ld,
                                                               const float* __restrict__ add,
                                                               const float* __restrict__ g,
                                                               const float* __restrict__ bta, int d,
                                                               uint16_t* __restrict__ y, int64_t y_ld) {
  __shared__ float red[2][kLnThreads / 32];
  float* xr = x + (size_t)blockIdx.x * x_ld;
  const int n4 = d >> 2;
  // gamma / beta / pending bias are static: copied to shared memory with
  // cp.async before the dependency wait (their latency overlaps the
  // previous kernel's tail)
  extern __shared__ __align__(16) float ln_smem[];
  float* sg = ln_smem;
  float* sb = ln_smem + d;
  float* sa = ln_smem + 2 * d;
  for (int i = threadIdx.x; i < n4; i += kLnThreads) {
    cp_async16(sg + 4 * i, g + 4 * i, 16);
    cp_async16(sb + 4 * i, bta + 4 * i, 16);
    if (ADD) cp_async16(sa + 4 * i, add + 4 * i, 16);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  griddep_wait();
  griddep_launch();
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  float4 v[kLnSlots];
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < kLnSlots; ++j) {
    const int i = j * kLnThreads + threadIdx.x;
    if (i < n4) {
      v[j] = *reinterpret_cast<const float4*>(xr + 4 * i);
      if (ADD) {
        const float4 a = *reinterpret_cast<const float4*>(sa + 4 * i);
        v[j].x += a.x; v[j].y += a.y; v[j].z += a.z; v[j].w += a.w;
        *reinterpret_cast<float4*>(xr + 4 * i) = v[j];
      }
      s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
    }
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[0][threadIdx.x >> 5] = s;
  __syncthreads();
  float mean = 0.f;
#pragma unroll
  for (int w = 0; w < kLnThreads / 32; ++w) mean += red[0][w];
  mean /= d;
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < kLnSlots; ++j) {
    const int i = j * kLnThreads + threadIdx.x;
    if (i < n4) {
      const float a = v[j].x - mean, b2 = v[j].y - mean, c = v[j].z - mean, e = v[j].w - mean;
      q += (a * a + b2 * b2) + (c * c + e * e);
    }
  }
  q = warp_sum(q);
  if ((threadIdx.x & 31) == 0) red[1][threadIdx.x >> 5] = q;
  __syncthreads();
  float var = 0.f;
#pragma unroll
  for (int w = 0; w < kLnThreads / 32; ++w) var += red[1][w];
  var /= d;
  const float rstd = rsqrtf(var + 1e-5f);
  uint16_t* yr = y + (size_t)blockIdx.x * y_ld;
#pragma unroll
  for (int j = 0; j < kLnSlots; ++j) {
    const int i = j * kLnThreads + threadIdx.x;
    if (i < n4) {
      const float4 gg = *reinterpret_cast<const float4*>(sg + 4 * i);
      const float4 bb = *reinterpret_cast<const float4*>(sb + 4 * i);
      uint2 o;
      o.x = pack_bf16x2((v[j].x - mean) * rstd * gg.x + bb.x, (v[j].y - mean) * rstd * gg.y + bb.y);
      o.y = pack_bf16x2((v[j].z - mean) * rstd * gg.z + bb.z, (v[j].w - mean) * rstd * gg.w + bb.w);
      *reinterpret_cast<uint2*>(yr + 4 * i) = o;
    }
  }
}

__global__ void embed_kernel(const int32_t* __restrict__ tok, const int32_t* __restrict__ len,
                             const uint16_t* __restrict__ emb, const uint16_t* __restrict__ pos, int d,
                             float* __restrict__ x) {
  const int b = blockIdx.x;
  griddep_wait();
  griddep_launch();
  const uint16_t* er = emb + (size_t)tok[b] * d;
  const uint16_t* pr = pos + (size_t)len[b] * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    x[(size_t)b * d + i] = __uint_as_float((uint32_t)er[i] << 16) + __uint_as_float((uint32_t)pr[i] << 16);
}

// h = silu(gate) * up, gate/up from one (B, 2D) bf16 row [gate | up]:
// grid (column blocks, B), 8 columns per thread with 16-byte loads/stores
__global__ void swiglu_kernel(const uint16_t* __restrict__ gu, int64_t gu_ld, int B, int D,
                              uint16_t* __restrict__ h, int64_t h_ld, int vec) {
  griddep_wait();
  griddep_launch();
  const int b = blockIdx.y;
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (j0 >= D) return;
  const uint16_t* gr = gu + (size_t)b * gu_ld;
  uint16_t* hr = h + (size_t)b * h_ld;
  if (vec && j0 + 8 <= D) {
    float g[8], u[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(gr + j0)), g);
    unpack8(__ldg(reinterpret_cast<const uint4*>(gr + D + j0)), u);
    uint4 o;
    o.x = pack_bf16x2(g[0] / (1.f + __expf(-g[0])) * u[0], g[1] / (1.f + __expf(-g[1])) * u[1]);
    o.y = pack_bf16x2(g[2] / (1.f + __expf(-g[2])) * u[2], g[3] / (1.f + __expf(-g[3])) * u[3]);
    o.z = pack_bf16x2(g[4] / (1.f + __expf(-g[4])) * u[4], g[5] / (1.f + __expf(-g[5])) * u[5]);
    o.w = pack_bf16x2(g[6] / (1.f + __expf(-g[6])) * u[6], g[7] / (1.f + __expf(-g[7])) * u[7]);
    *reinterpret_cast<uint4*>(hr + j0) = o;
  } else {
    for (int j = j0; j < min(D, j0 + 8); ++j) {
      const float g = __uint_as_float((uint32_t)gr[j] << 16), u = __uint_as_float((uint32_t)gr[D + j] << 16);
      hr[j] = f2bf(g / (1.f + __expf(-g)) * u);
    }
  }
}

}  // namespace

int g_num_sms = 0;
int g_pdl = 1;

}  // namespace ps

using namespace ps;

extern "C" int ps_version(void) { return 1; }

extern "C" void ps_set_pdl(int enable) { g_pdl = enable ? 1 : 0; }

extern "C" const char* ps_status_string(int status) {
  switch (status) {
    case PS_OK: return "ok";
    case PS_ERR_VALUE: return "invalid argument";
    case PS_ERR_INDEX: return "index out of range";
    case PS_ERR_EMPTY_CACHE: return "empty KV cache";
    case PS_ERR_CAPACITY: return "KV cache capacity exhausted";
    case PS_ERR_UNSUPPORTED: return "shape not supported by the sm_100a kernels";
    case PS_ERR_WORKSPACE: return "workspace too small";
    case PS_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

extern "C" int ps_num_sms(void) {
  if (g_num_sms == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      g_num_sms = n;
    else
      return 148;
  }
  return g_num_sms;
}

extern "C" int ps_kv_append(void* k_cache, void* v_cache, int32_t* lengths, const void* k_new, const void* v_new,
                            int64_t src_ld, int B, int H_kv, int cap, int d_h, int32_t* err_flag, void* stream) {
  if (B < 1 || H_kv < 1 || cap < 1 || d_h < 8 || d_h % 8 || src_ld < (int64_t)H_kv * d_h || src_ld % 8)
    return PS_ERR_VALUE;
  if (!k_cache || !v_cache || !lengths || !k_new || !v_new) return PS_ERR_VALUE;
  if (((uintptr_t)k_new % 16) || ((uintptr_t)v_new % 16) || ((uintptr_t)k_cache % 16) || ((uintptr_t)v_cache % 16))
    return PS_ERR_VALUE;
  return launch_ex(kv_append_kernel, dim3(B), dim3(kKvThreads), 0, static_cast<cudaStream_t>(stream), 1,
                   static_cast<uint16_t*>(k_cache), static_cast<uint16_t*>(v_cache), lengths,
                   static_cast<const uint16_t*>(k_new), static_cast<const uint16_t*>(v_new), src_ld, H_kv, cap, d_h,
                   err_flag, static_cast<const int32_t*>(nullptr), (int64_t)0, 0);
}

extern "C" int ps_kv_append_paged(void* k_pool, void* v_pool, int page_rows, const int32_t* block_table,
                                  int64_t table_ld, int32_t* lengths, const void* k_new, const void* v_new,
                                  int64_t src_ld, int B, int H_kv, int d_h, int32_t* err_flag, void* stream) {
  if (B < 1 || H_kv < 1 || page_rows < 1 || table_ld < 1 || d_h < 8 || d_h % 8 || src_ld < (int64_t)H_kv * d_h ||
      src_ld % 8)
    return PS_ERR_VALUE;
  if (!k_pool || !v_pool || !block_table || !lengths || !k_new || !v_new) return PS_ERR_VALUE;
  if (((uintptr_t)k_new % 16) || ((uintptr_t)v_new % 16) || ((uintptr_t)k_pool % 16) || ((uintptr_t)v_pool % 16))
    return PS_ERR_VALUE;
  const long long cap = (long long)table_ld * page_rows;
  if (cap >= (1ll << 31)) return PS_ERR_VALUE;
  return launch_ex(kv_append_kernel, dim3(B), dim3(kKvThreads), 0, static_cast<cudaStream_t>(stream), 1,
                   static_cast<uint16_t*>(k_pool), static_cast<uint16_t*>(v_pool), lengths,
                   static_cast<const uint16_t*>(k_new), static_cast<const uint16_t*>(v_new), src_ld, H_kv, (int)cap,
                   d_h, err_flag, block_table, table_ld, page_rows);
}

static int ln_launch(float* x, int64_t x_ld, const float* add, const float* gamma, const float* beta, int B, int d,
                     void* y, int64_t y_ld, void* stream) {
  if (B < 1 || d < 4 || d % 4 || d > 4 * kLnSlots * kLnThreads || !x || !gamma || !beta || !y || x_ld < d ||
      y_ld < d || x_ld % 4 || y_ld % 4)
    return PS_ERR_VALUE;
  if (((uintptr_t)x % 16) || ((uintptr_t)gamma % 16) || ((uintptr_t)beta % 16) || ((uintptr_t)y % 8) ||
      (add && ((uintptr_t)add % 16)))
    return PS_ERR_VALUE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t smem = (size_t)(add ? 3 : 2) * d * 4;
  {
    static bool big = false;  // opt in once (first call is eager, before any graph capture)
    if (!big) {
      if (cudaFuncSetAttribute(layernorm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
              cudaSuccess ||
          cudaFuncSetAttribute(layernorm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
              cudaSuccess)
        return PS_ERR_CUDA;
      big = true;
    }
  }
  return launch_ex(add ? layernorm_kernel<true> : layernorm_kernel<false>, dim3(B), dim3(kLnThreads), smem, st, 1, x,
                   x_ld, add, gamma, beta, d, static_cast<uint16_t*>(y), y_ld);
}

extern "C" int ps_layernorm(const float* x, int64_t x_ld, const float* gamma, const float* beta, int B, int d,
                            void* y, int64_t y_ld, void* stream) {
  return ln_launch(const_cast<float*>(x), x_ld, nullptr, gamma, beta, B, d, y, y_ld, stream);
}

extern "C" int ps_add_layernorm(float* x, int64_t x_ld, const float* add, const float* gamma, const float* beta,
                                int B, int d, void* y, int64_t y_ld, void* stream) {
  return ln_launch(x, x_ld, add, gamma, beta, B, d, y, y_ld, stream);
}

extern "C" int ps_embed(const int32_t* tokens, const int32_t* lengths, const void* embed, const void* pos_embed,
                        int B, int d, float* x, void* stream) {
  if (B < 1 || d < 1 || !tokens || !lengths || !embed || !pos_embed || !x) return PS_ERR_VALUE;
  return launch_ex(embed_kernel, dim3(B), dim3(256), 0, static_cast<cudaStream_t>(stream), 1, tokens, lengths,
                   static_cast<const uint16_t*>(embed), static_cast<const uint16_t*>(pos_embed), d, x);
}

extern "C" int ps_swiglu(const void* gu, int64_t gu_ld, int B, int D, void* h, int64_t h_ld, void* stream) {
  if (B < 1 || D < 1 || !gu || !h || gu_ld < 2 * (int64_t)D || h_ld < D) return PS_ERR_VALUE;
  // 16-byte vector path needs 8-element aligned rows and halves
  const int vec = !((gu_ld % 8) || (h_ld % 8) || (D % 8) || ((uintptr_t)gu % 16) || ((uintptr_t)h % 16));
  const int threads = 128;
  const dim3 grid((D / 8 + threads - 1) / threads, B);
  return launch_ex(swiglu_kernel, grid, dim3(threads), 0, static_cast<cudaStream_t>(stream), 1,
                   static_cast<const uint16_t*>(gu), gu_ld, B, D, static_cast<uint16_t*>(h), h_ld, vec);
}
