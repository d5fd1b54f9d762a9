// Tensor-parallel all-reduce of the bf16 partial residual updates FUSED with
// the residual add, over peer memory (the exchange after
// the O- and down-projections, parallel.py).
//
//   x[b, :] += sum_{r < world} part_r[b, :]        (part_r: rank r's bf16 partial)
//
// Every rank's partial buffer (two slots, alternating call to call) and a
// per-rank inbox of flags are mapped into every other rank's address space
// with CUDA IPC (NVLink peer memory on one node; the same device when the
// ranks share a GPU in tests).  One launch per all-reduce:
//   * CTA 0 signals every peer's inbox (slot `rank`) with this launch's
//     epoch (a release at system scope, after the partial is complete);
//   * every CTA waits until its own inbox holds the epoch from every rank,
//     then sums its 16-byte chunks across the ranks' buffers in f32 (one-shot:
//     each rank reads every partial) and adds them into its f32 residual x;
//   * the last CTA (ticket) advances the device epoch, so a CUDA-graph replay
//     issues fresh epochs without host involvement.
// Slot reuse is safe with two slots: a rank rewrites slot s only after its
// next all-reduce's barrier, which every peer enters after finishing its
// reads of s.  With a multicast (NVLS) mapping the chunk sum would be one
// multimem.ld_reduce per chunk; the box this is developed on exposes one
// GPU and no multicast object, so only the peer-load form is built.
#include "common.cuh"

namespace ps {
namespace {

constexpr int kArThreads = 256;
constexpr int kArMaxWorld = 8;

struct ArParams {
  const unsigned long long* bufs;   // [world] peer partial buffers (this call's slot), bf16
  const unsigned long long* flags;  // [world] peer inboxes (uint32 [kArMaxWorld] each)
  unsigned int* inbox;              // this rank's inbox
  unsigned int* state;              // [0] epoch, [1] ticket
  int rank, world;
  int B, d;
  float* x;
  int64_t x_ld;
};

PS_DEV unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PS_DEV void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kArThreads) allreduce_add_kernel(const ArParams p) {
  __shared__ unsigned int s_epoch;
  __shared__ int s_last;
  const int tid = threadIdx.x;
  griddep_wait();  // this rank's partial (the previous kernel) is complete
  if (tid == 0) s_epoch = *reinterpret_cast<volatile unsigned int*>(p.state) + 1u;
  __syncthreads();
  const unsigned int e = s_epoch;
  if (blockIdx.x == 0 && tid < p.world) {
    __threadfence_system();
    unsigned int* peer_inbox = reinterpret_cast<unsigned int*>(p.flags[tid]);
    st_release_sys(peer_inbox + p.rank, e);
  }
  if (tid < p.world) {
    while ((int)(ld_acquire_sys(p.inbox + tid) - e) < 0) {
    }
  }
  __syncthreads();
  griddep_launch();
  const uint4* src[kArMaxWorld];
#pragma unroll
  for (int r = 0; r < kArMaxWorld; ++r)
    src[r] = r < p.world ? reinterpret_cast<const uint4*>(p.bufs[r]) : nullptr;
  const int per_row = p.d >> 3;  // 16-byte chunks per row
  const int chunks = p.B * per_row;
  for (int c = blockIdx.x * kArThreads + tid; c < chunks; c += gridDim.x * kArThreads) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint4 v[kArMaxWorld];
#pragma unroll
    for (int r = 0; r < kArMaxWorld; ++r)
      if (r < p.world) v[r] = __ldcv(src[r] + c);  // volatile: peers wrote it, no stale L1 lines
#pragma unroll
    for (int r = 0; r < kArMaxWorld; ++r) {
      if (r < p.world) {
        float f[8];
        unpack8(v[r], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += f[k];
      }
    }
    const int b = c / per_row, col = (c - b * per_row) * 8;
    float4* xo = reinterpret_cast<float4*>(p.x + (size_t)b * p.x_ld + col);
    float4 a0 = xo[0], a1 = xo[1];
    a0.x += acc[0]; a0.y += acc[1]; a0.z += acc[2]; a0.w += acc[3];
    a1.x += acc[4]; a1.y += acc[5]; a1.z += acc[6]; a1.w += acc[7];
    xo[0] = a0;
    xo[1] = a1;
  }
  // the last CTA advances the epoch for the next launch
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(p.state + 1, 1u) == gridDim.x - 1;
    if (s_last) {
      p.state[1] = 0u;
      p.state[0] = e;
    }
  }
}

}  // namespace
}  // namespace ps

using namespace ps;

// bufs / flags: device arrays of `world` 64-bit addresses (this rank's own
// entries included); inbox: this rank's kArMaxWorld uint32 flags; state: 2
// uint32 (epoch, ticket), zero-initialised once.  x: f32 (B, d) residual,
// row stride x_ld; d % 8 == 0, 16-byte aligned rows.
extern "C" int ps_allreduce_add_bf16(const unsigned long long* bufs, const unsigned long long* flags,
                                     unsigned int* inbox, unsigned int* state, int rank, int world, int B, int d,
                                     float* x, int64_t x_ld, void* stream) {
  if (!bufs || !flags || !inbox || !state || !x || world < 1 || world > kArMaxWorld || rank < 0 || rank >= world ||
      B < 1 || d < 8 || d % 8 || x_ld < d || x_ld % 4 || ((uintptr_t)x % 16))
    return PS_ERR_VALUE;
  ArParams prm{};
  prm.bufs = bufs; prm.flags = flags; prm.inbox = inbox; prm.state = state;
  prm.rank = rank; prm.world = world; prm.B = B; prm.d = d; prm.x = x; prm.x_ld = x_ld;
  const int chunks = B * (d / 8);
  int grid = (chunks + kArThreads - 1) / kArThreads;
  if (grid > ps_num_sms()) grid = ps_num_sms();
  return launch_ex(allreduce_add_kernel, dim3(grid), dim3(kArThreads), 0, static_cast<cudaStream_t>(stream), 1,
                   prm);
}
