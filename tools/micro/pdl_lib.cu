// PDL probe kernels as a shared library (tools/pdl_probe2.py launches them
// from Python inside torch.cuda.graph capture).
#include <cuda_runtime.h>
__device__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void kA(unsigned long long* st, int spin_ns) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  unsigned long long t0 = gt();
  if (threadIdx.x == 0) st[blockIdx.x * 2] = t0;
  while (gt() - t0 < (unsigned long long)spin_ns) {
  }
  if (threadIdx.x == 0) st[blockIdx.x * 2 + 1] = gt();
}
__global__ void kB(unsigned long long* st) {
  if (threadIdx.x == 0) st[blockIdx.x] = gt();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
extern "C" int pdl_a(void* st, int n, int spin, void* stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n); cfg.blockDim = dim3(512); cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kA, (unsigned long long*)st, spin);
}
extern "C" int pdl_b(void* st, int n, void* stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n); cfg.blockDim = dim3(256); cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kB, (unsigned long long*)st);
}
