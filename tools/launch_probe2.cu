// Launch gap of back-to-back kernels in a CUDA graph vs registers per thread:
// 148 CTAs x 512 threads, 190 KB smem, TMEM 512 cols, ~2 us spin, PDL on/off;
// the register count is forced with __launch_bounds__ + a live-value array.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
template <int R>
__global__ void __launch_bounds__(512, 1) k_spin(int ns, int* sink) {
  extern __shared__ char sm[];
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  uint32_t v[R];
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = threadIdx.x * (i + 1);
  uint64_t t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint64_t t = t0;
  while (t - t0 < (uint64_t)ns) {
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = v[i] * 3 + 1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) acc ^= v[i];
  if (acc == 0x12345) *sink = acc;
  asm volatile("griddepcontrol.launch_dependents;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
template <int R>
void run(cudaStream_t st, int* sink, int smem_kb) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_spin<R>);
  cudaFuncSetAttribute(k_spin<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
  for (int pdl : {0, 1}) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    const int n = 20;
    for (int i = 0; i < n; ++i) {
      cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(148); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem_kb * 1024; cfg.stream = st;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = pdl; cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_spin<R>, 2000, sink);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    cudaEventRecord(a, st); cudaGraphLaunch(ge, st); cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("smem %3d KB regs %3d pdl %d: %.2f us per 2-us kernel (%s)\n", smem_kb, fa.numRegs, pdl, ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
  }
}
int main() {
  cudaStream_t st; cudaStreamCreate(&st);
  int* sink; cudaMalloc(&sink, 4);
  for (int kb : {190, 200, 210, 220, 226}) run<90>(st, sink, kb);
  return 0;
}
