// Launch overhead of back-to-back kernels in a CUDA graph as a function of the
// dynamic shared memory and block size (148 CTAs, each spinning ~2 us).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__global__ void k_spin(int ns, int tmem) {
  extern __shared__ char sm[];
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) sm[0] = 1;
  if (tmem && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  uint64_t t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint64_t t = t0;
  while (t - t0 < (uint64_t)ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && sm[0] == 7) printf("x");
  asm volatile("griddepcontrol.launch_dependents;");
  __syncthreads();
  if (tmem && threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
int main() {
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int tm : {0, 1})
  for (int smem : {0, 48 * 1024, 190 * 1024})
    for (int thr : {128, 512}) for (int pdl : {0, 1}) {
      cudaFuncSetAttribute(k_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      const int n = 20;
      for (int i = 0; i < n; ++i) {
        cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(148); cfg.blockDim = dim3(thr); cfg.dynamicSmemBytes = smem; cfg.stream = st;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl; cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_spin, 2000, tm);
      }
      cudaStreamEndCapture(st, &g);
      if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed: %s\n", cudaGetErrorString(cudaGetLastError())); continue; }
      cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
      cudaEventRecord(a, st); cudaGraphLaunch(ge, st); cudaEventRecord(b, st); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("tmem %d smem %6d B, %3d threads, pdl %d: %.2f us per 2-us kernel (%s)\n", tm, smem, thr, pdl, ms * 1e3 / n,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
