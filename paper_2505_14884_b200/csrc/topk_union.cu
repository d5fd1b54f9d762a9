// Low-latency per-row top-k (or threshold) selection fused with the batch
// union -- the engine's ps_select_union path (sm_100a).
//
// Semantics (tensors.py:54-73 top-k, kernels.py:376-383 union): per row, the
// k largest of logits + bias in numpy stable-argsort order of -scores (value
// descending, ties to the lower column, -0.0 == +0.0, NaN below -inf); the
// union over rows of the selected columns in [lo, hi), written ascending
// (relative to lo), padded with the last id to a multiple of `pad`, its size
// in *count.  k <= 0: threshold selection (logit + bias > thr).
//
// Design (one 1024-thread CTA per row, no grid barrier):
//   * the row lives in registers: thread t holds float4 chunks at columns
//     4t + 4096j (coalesced 16-byte loads); the static bias is loaded before
//     griddepcontrol.wait, the logits right after it;
//   * exact radix select of the k-th largest order key in three rounds of
//     (11, 11, 10) bits over a 2048-bin shared histogram; each round the
//     threads that read the bins zero them for the next round, and a round
//     whose bin holds exactly the remaining rank ends the search (all its
//     keys are taken: no tie ranking);
//   * ties at the final key are ranked by column (one block scan per chunk,
//     only when the tied keys outnumber the remaining rank);
//   * the row's selection bits are OR-ed straight into the union bitmap
//     (8 lanes -> one 32-bit word, one atomicOr per non-empty word);
//   * the last row CTA to finish (acq_rel ticket) compacts the bitmap into
//     ascending ids, pads, writes the count, and re-zeroes the bitmap and the
//     ticket (self-resetting: CUDA-graph replayable).
// Rows never wait for each other, so any number of rows is safe (no
// co-residency assumption).
#include "common.cuh"

namespace ps {
namespace {

constexpr int kTuThreads = 1024;
constexpr int kTuWarps = kTuThreads / 32;
constexpr int kTuChunk = 4 * kTuThreads;  // columns per float4 chunk of the CTA
constexpr int kTuBins = 2048;
constexpr int kTuMaxWPT = 4;  // compaction: bitmap words per thread (cols <= 131072)
constexpr int kTuCand = 4096;  // round-1 bin keys kept for rounds 2-3 (else they rescan the registers)

struct TuParams {
  const float* logits;
  int rows, cols;
  int64_t ld;
  int k;
  float thr;
  const float* bias;
  uint32_t* bitmap;  // ceil(cols / 32) words, zero between launches
  int* ticket;
  int lo, hi, pad;
  int32_t* union_out;
  int32_t* count_out;
  unsigned long long* trace;
  // union hand-off (ps_select_union_bitmap): rows only OR into `bitmap`; no
  // ticket, no compaction, no reset; CTA 0 zeroes `clear` (the other buffer)
  int no_compact;
  uint32_t* clear;
};

PS_DEV uint32_t tu_key(float f) {  // order-preserving; 0 = NaN (below -inf)
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0u;
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

PS_DEV unsigned long long tu_time() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Block exclusive scan (1024 threads); *total = block sum.  Three barriers.
PS_DEV int tu_scan(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;
  }
  __syncthreads();
  const int r = (warp ? s_warp[warp - 1] : 0) + x - v;
  if (total) *total = s_warp[kTuWarps - 1];
  __syncthreads();
  return r;
}

template <int NCH>  // float4 chunks per thread: cols <= NCH * 4096
__global__ void __launch_bounds__(kTuThreads, 1) topk_union_kernel(const TuParams p) {
  // ping-pong histograms (round r fills hist[r & 1]); bin kTuBins is a
  // dummy that absorbs non-matching keys (the increments stay unconditional)
  __shared__ __align__(16) int hist[2][kTuBins + 4];
  __shared__ uint32_t s_cand[kTuCand];  // keys in round 1's bin (rounds 2-3 run on them)
  __shared__ int s_ncand;
  __shared__ int s_warp[kTuWarps];
  __shared__ int s_sel[3];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31;
  const int row = blockIdx.x;
  const int cols = p.cols;
  const bool vec = (p.ld & 3) == 0 && (cols & 3) == 0 && ((uintptr_t)p.logits & 15) == 0 &&
                   (!p.bias || ((uintptr_t)p.bias & 15) == 0);
  // ---- static bias before the dependency wait (registers permitting)
  constexpr bool kPre = NCH <= 4;
  constexpr int NB = kPre ? NCH : 1;
  auto load_bias = [&](int j, float* b) {
    const int c0 = j * kTuChunk + 4 * tid;
    if (p.bias && vec && c0 < cols) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(p.bias + c0));
      b[0] = t.x; b[1] = t.y; b[2] = t.z; b[3] = t.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) b[e] = (p.bias && c0 + e < cols) ? __ldg(p.bias + c0 + e) : 0.f;
    }
  };
  float bv[NB][4];
  if (kPre) {
#pragma unroll
    for (int j = 0; j < NB; ++j) load_bias(j, bv[j]);
  }
  for (int i = tid; i < kTuBins + 4; i += kTuThreads) hist[0][i] = 0;
  if (tid == 0) s_ncand = 0;
  griddep_wait();
  griddep_launch();
  if (p.clear && row == 0)  // last read by the previous layer's GEMMs, which completed before this grid
    for (int w = tid; w < ((cols + 31) >> 5); w += kTuThreads) p.clear[w] = 0u;
  if (p.trace && tid == 0) {
    p.trace[row * 16 + 0] = tu_time();
    p.trace[row * 16 + 8] = clock64();
  }

  // ---- the row (+ bias) into registers
  const float* xr = p.logits + (size_t)row * p.ld;
  float v[NCH][4];
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int c0 = j * kTuChunk + 4 * tid;
    if (vec && c0 < cols) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(xr + c0));
      v[j][0] = a.x; v[j][1] = a.y; v[j][2] = a.z; v[j][3] = a.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) v[j][e] = c0 + e < cols ? __ldcg(xr + c0 + e) : 0.f;
    }
  }
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    float b[4];
    if (kPre) {
#pragma unroll
      for (int e = 0; e < 4; ++e) b[e] = bv[kPre ? j : 0][e];
    } else {
      load_bias(j, b);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) v[j][e] += b[e];
  }
  if (p.trace && tid == 0) p.trace[row * 16 + 1] = tu_time();
  uint32_t sel[NCH];  // 4 selection bits per chunk
  const bool threshold = p.k <= 0;
  if (threshold) {
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c0 = j * kTuChunk + 4 * tid;
      uint32_t s = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (c0 + e < cols && v[j][e] > p.thr) s |= 1u << e;
      sel[j] = s;
    }
  } else {
    uint32_t key[NCH][4];
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c0 = j * kTuChunk + 4 * tid;
#pragma unroll
      for (int e = 0; e < 4; ++e) key[j][e] = tu_key(v[j][e]);
      if (c0 >= cols) {
#pragma unroll
        for (int e = 0; e < 4; ++e) key[j][e] = 0u;
      }
    }
    // ---- exact radix select of the k-th largest key: rounds of 11, 11, 10 bits.
    // Round 1 histograms every key; its bin's keys are appended to s_cand
    // and rounds 2-3 histogram only those (unless the bin overflows s_cand).
    uint32_t prefix = 0, pmask = 0;
    int remaining = p.k, bin_count = 0;
    bool exact = false;  // the final bin holds exactly `remaining` keys
    const int warp = tid >> 5;
    int n_cand = 0;  // > 0: rounds 2-3 run on s_cand[0, n_cand)
#pragma unroll 1
    for (int r = 0; r < 3; ++r) {
      const int shift = r == 0 ? 21 : (r == 1 ? 10 : 0);
      const int bins = r == 2 ? 1024 : 2048;
      const uint32_t dmask = (uint32_t)bins - 1u;
      int* h = hist[r & 1];
      // the other buffer was last read before the previous round's final
      // barrier: clear it for the next round while this one fills
      reinterpret_cast<int2*>(hist[(r + 1) & 1])[tid] = make_int2(0, 0);
      if (n_cand) {
        for (int i = tid; i < n_cand; i += kTuThreads) {
          const uint32_t kk = s_cand[i];
          atomicAdd(&h[(kk & pmask) == prefix ? (kk >> shift) & dmask : kTuBins], 1);
        }
      } else {
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const int c0 = j * kTuChunk + 4 * tid;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool m = c0 + e < cols && (key[j][e] & pmask) == prefix;
            atomicAdd(&h[m ? (key[j][e] >> shift) & dmask : kTuBins], 1);
          }
        }
      }
      __syncthreads();
      if (p.trace && tid == 0 && r < 2) p.trace[row * 16 + 10 + r] = tu_time();
      // descending scan: thread t owns bins hb and hb - 1 (hb = bins - 1 - 2t)
      const int hb = bins - 1 - 2 * tid;
      int c_hi = 0, c_lo = 0;
      if (hb >= 1) {
        const int2 pr = reinterpret_cast<const int2*>(h)[hb >> 1];  // {hb - 1, hb}
        c_lo = pr.x;
        c_hi = pr.y;
      }
      const int loc = c_hi + c_lo;
      int incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_warp[warp] = incl;
      __syncthreads();
      int wt = s_warp[lane];  // every warp scans the 32 warp totals itself
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, wt, o);
        if (lane >= o) wt += y;
      }
      const int wabove = warp ? __shfl_sync(0xffffffffu, wt, warp - 1) : 0;
      const int above = wabove + incl - loc;
      if (hb >= 1 && above < remaining && above + loc >= remaining) {
        if (above + c_hi >= remaining) {
          s_sel[0] = hb; s_sel[1] = remaining - above; s_sel[2] = c_hi;
        } else {
          s_sel[0] = hb - 1; s_sel[1] = remaining - above - c_hi; s_sel[2] = c_lo;
        }
      }
      __syncthreads();
      prefix |= (uint32_t)s_sel[0] << shift;
      pmask |= dmask << shift;
      remaining = s_sel[1];
      bin_count = s_sel[2];
      if (p.trace && tid == 0) p.trace[row * 16 + 2 + r] = tu_time();
      // s_sel / s_warp are rewritten next round only after its first
      // barrier, which every thread reaches after reading them here
      if (bin_count == remaining) {
        exact = true;
        break;
      }
      if (r == 0 && bin_count <= kTuCand) {
        // append round 1's bin: per-thread counts, a warp scan, one shared
        // atomic per warp for the base
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const int c0 = j * kTuChunk + 4 * tid;
#pragma unroll
          for (int e = 0; e < 4; ++e) cnt += (c0 + e < cols && (key[j][e] & pmask) == prefix) ? 1 : 0;
        }
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        int base = 0;
        if (lane == 31 && inc) base = atomicAdd(&s_ncand, inc);
        base = __shfl_sync(0xffffffffu, base, 31) + inc - cnt;
        if (cnt) {
#pragma unroll
          for (int j = 0; j < NCH; ++j) {
            const int c0 = j * kTuChunk + 4 * tid;
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (c0 + e < cols && (key[j][e] & pmask) == prefix) s_cand[base++] = key[j][e];
          }
        }
        __syncthreads();
        n_cand = bin_count;
      }
    }
    // ---- classify: above the prefix -> in; equal -> in if exact, else by column rank
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c0 = j * kTuChunk + 4 * tid;
      uint32_t s = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t m = key[j][e] & pmask;
        if (c0 + e < cols && (m > prefix || (exact && m == prefix))) s |= 1u << e;
      }
      sel[j] = s;
    }
    if (!exact) {
      // tied keys at the k-th key: the `remaining` lowest columns win.
      // Column order is chunk-major, then thread, then element.
      int base = 0;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int c0 = j * kTuChunk + 4 * tid;
        uint32_t eqm = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (c0 + e < cols && (key[j][e] & pmask) == prefix) eqm |= 1u << e;
        int tot;
        const int before = tu_scan(__popc(eqm), s_warp, &tot);
        int rank = base + before;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (eqm & (1u << e)) {
            if (rank < remaining) sel[j] |= 1u << e;
            ++rank;
          }
        base += tot;
      }
    }
  }
  // ---- OR the row's bits into the union bitmap: 8 lanes form one word
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    uint32_t w = sel[j] << (4 * (tid & 7));
    w |= __shfl_xor_sync(0xffffffffu, w, 1);
    w |= __shfl_xor_sync(0xffffffffu, w, 2);
    w |= __shfl_xor_sync(0xffffffffu, w, 4);
    const int c0 = j * kTuChunk + 4 * tid;
    if ((tid & 7) == 0 && w && c0 < cols) atomicOr(p.bitmap + (c0 >> 5), w);
  }
  if (p.trace && tid == 0) {
    p.trace[row * 16 + 5] = tu_time();
    p.trace[row * 16 + 9] = clock64();
  }
  if (p.no_compact) return;  // the GEMMs read the bitmap (PS_GG_BITMAP)
  // ---- the last row CTA compacts
  // one acq_rel ticket (release: this CTA's bitmap ORs, ordered before it by
  // the barrier; acquire: every other CTA's, for the compacting CTA) instead
  // of a fence on each side of a relaxed atomic
  __syncthreads();
  if (tid == 0) {
    unsigned int old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(p.ticket) : "memory");
    s_last = old == (unsigned int)p.rows - 1u;
  }
  __syncthreads();
  if (!s_last) return;
  if (p.trace && tid == 0) p.trace[row * 16 + 6] = tu_time();
  const int words = (cols + 31) >> 5;
  const int wlo = p.lo >> 5, whi = (p.hi + 31) >> 5;
  const int nw = whi - wlo;
  const int kw = (nw + kTuThreads - 1) / kTuThreads;  // <= kTuMaxWPT (checked on the host)
  const int tw0 = wlo + tid * kw;
  uint32_t wb[kTuMaxWPT];
  int cnt = 0;
#pragma unroll
  for (int j = 0; j < kTuMaxWPT; ++j) {
    const int w = tw0 + j;
    uint32_t a = 0;
    if (j < kw && w < whi) {
      a = __ldcg(p.bitmap + w);
      const int top = p.hi - (w << 5);
      if (top < 32) a &= top <= 0 ? 0u : ((1u << top) - 1u);
      const int bot = p.lo - (w << 5);  // lo is a multiple of 32: always <= 0 here
      if (bot > 0) a &= ~((1u << bot) - 1u);
    }
    wb[j] = a;
    cnt += __popc(a);
  }
  int total;
  const int pos0 = tu_scan(cnt, s_warp, &total);
  // ids staged in shared memory (each thread writes its words' ids), then
  // copied out with coalesced 16-byte stores
  extern __shared__ __align__(16) int s_ids[];
  {
    int pos = pos0;
#pragma unroll
    for (int j = 0; j < kTuMaxWPT; ++j) {
      uint32_t bits = wb[j];
      const int base = ((tw0 + j) << 5) - p.lo;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        s_ids[pos++] = base + b;
      }
    }
  }
  __syncthreads();
  {
    const int n4 = ((uintptr_t)p.union_out & 15) ? 0 : total >> 2;
    int4* o4 = reinterpret_cast<int4*>(p.union_out);
    const int4* s4 = reinterpret_cast<const int4*>(s_ids);
    for (int i = tid; i < n4; i += kTuThreads) o4[i] = s4[i];
    for (int i = (n4 << 2) + tid; i < total; i += kTuThreads) p.union_out[i] = s_ids[i];
  }
  __syncthreads();  // every id written before the padding reads the last one
  if (tid == 0) *p.count_out = total;
  if (p.pad > 1 && total > 0) {
    const int padded = (total + p.pad - 1) / p.pad * p.pad;
    const int32_t last = s_ids[total - 1];
    for (int i = total + tid; i < padded; i += kTuThreads) p.union_out[i] = last;
  }
  // self-reset for the next launch
  for (int w = tid; w < words; w += kTuThreads) p.bitmap[w] = 0u;
  if (tid == 0) *p.ticket = 0;
  if (p.trace && tid == 0) p.trace[row * 16 + 7] = tu_time();
}

template <int NCH>
int launch_tu(const TuParams& prm, cudaStream_t st) {
  // dynamic shared memory: the compacting CTA's staged ids (one int per
  // column of [lo, hi) rounded to whole words)
  const size_t smem = (size_t)(((prm.hi + 31) >> 5) - (prm.lo >> 5)) * 32 * 4;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(topk_union_kernel<NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024) !=
        cudaSuccess)
      return PS_ERR_CUDA;
    configured = true;
  }
  return launch_ex(topk_union_kernel<NCH>, dim3(prm.rows), dim3(kTuThreads), smem, st, 1, prm);
}

}  // namespace

// Host entry (select.cu's ps_select_union routes here): the caller has
// validated the arguments and carved `ticket` / `bitmap` out of its
// zero-initialised workspace.
int select_union_v2(const float* logits, const float* bias, int rows, int cols, int64_t ld, int k, float thr,
                    int* ticket, uint32_t* bitmap, int lo, int hi, int pad, int32_t* union_out, int32_t* count_out,
                    unsigned long long* trace, cudaStream_t st) {
  TuParams prm{};
  prm.logits = logits; prm.rows = rows; prm.cols = cols; prm.ld = ld; prm.k = k; prm.thr = thr;
  prm.bias = bias; prm.bitmap = bitmap; prm.ticket = ticket;
  prm.lo = lo; prm.hi = hi; prm.pad = pad; prm.union_out = union_out; prm.count_out = count_out;
  prm.trace = trace;
  if (cols <= 1 * kTuChunk) return launch_tu<1>(prm, st);
  if (cols <= 2 * kTuChunk) return launch_tu<2>(prm, st);
  if (cols <= 4 * kTuChunk) return launch_tu<4>(prm, st);
  if (cols <= 8 * kTuChunk) return launch_tu<8>(prm, st);
  if (cols <= 9 * kTuChunk) return launch_tu<9>(prm, st);  // OPT-66B: D = 36864
  return PS_ERR_UNSUPPORTED;
}

int select_union_v2_max_cols() { return 9 * kTuChunk; }

int select_union_v2_bitmap(const float* logits, const float* bias, int rows, int cols, int64_t ld, int k, float thr,
                           uint32_t* bitmap, uint32_t* clear, unsigned long long* trace, cudaStream_t st) {
  TuParams prm{};
  prm.logits = logits; prm.rows = rows; prm.cols = cols; prm.ld = ld; prm.k = k; prm.thr = thr;
  prm.bias = bias; prm.bitmap = bitmap; prm.ticket = nullptr;
  prm.lo = 0; prm.hi = cols; prm.pad = 1; prm.union_out = nullptr; prm.count_out = nullptr;
  prm.trace = trace;
  prm.no_compact = 1;
  prm.clear = clear;
  if (cols <= 1 * kTuChunk) return launch_tu<1>(prm, st);
  if (cols <= 2 * kTuChunk) return launch_tu<2>(prm, st);
  if (cols <= 4 * kTuChunk) return launch_tu<4>(prm, st);
  if (cols <= 8 * kTuChunk) return launch_tu<8>(prm, st);
  if (cols <= 9 * kTuChunk) return launch_tu<9>(prm, st);
  return PS_ERR_UNSUPPORTED;
}

}  // namespace ps
