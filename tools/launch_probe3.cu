// Which feature of a kernel stretches the CTA end -> next CTA start gap on an SM?
// 148 CTAs x 512 threads, 200 KB smem, b2b in a CUDA graph (PDL on), ~2 us body.
// mode bits: 1 = TMEM alloc/dealloc, 2 = six 32 KB cp.async.bulk loads (waited),
// 4 = tcgen05.mma (one, committed + waited), 8 = prefetch.tensormap of a param map
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(512, 1) k(const __grid_constant__ CUtensorMap tm, const uint8_t* src, int ns, int mode,
                                             int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    if (mode & 8) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
  }
  if ((mode & 1) && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if ((mode & 2) && threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(6 * 32768));
    for (int i = 0; i < 6; ++i)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32768, [%2];" ::"r"(
                       su(sm + i * 32768)),
                   "l"(src + (static_cast<size_t>(blockIdx.x) * 6 + i) * 32768), "r"(su(&bar))
                   : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(su(&bar)) : "memory");
  }
  if ((mode & 16) && threadIdx.x == 0) {  // one 16 KB 2-D TMA tensor load, waited
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(16384));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(su(sm)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su(&bar)), "r"(0), "r"(int(blockIdx.x % 8) * 128)
                 : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(su(&bar)), "r"((mode & 2) ? 1 : 0) : "memory");
  }
  if ((mode & 32) && threadIdx.x == 0) {  // one 16 KB 1-D bulk copy, waited
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(16384));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(
                     su(sm)), "l"(src + (blockIdx.x % 8) * 16384), "r"(su(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(su(&bar)) : "memory");
  }
  uint64_t t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint64_t t = t0;
  while (t - t0 < (uint64_t)ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && sm[5] == 77) *sink = 1;
  asm volatile("griddepcontrol.launch_dependents;");
  __syncthreads();
  if ((mode & 1) && threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
int main() {
  cudaStream_t st; cudaStreamCreate(&st);
  int* sink; cudaMalloc(&sink, 4);
  uint8_t* src; cudaMalloc(&src, 148 * 6 * 32768); cudaMemset(src, 1, 148 * 6 * 32768);
  CUtensorMap tm{};
  cuuint64_t dims[2] = {128, 1024}; cuuint64_t str[1] = {128}; cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
  cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode : {0, 16, 32, 0, 16, 32}) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    const int n = 20;
    for (int i = 0; i < n; ++i) {
      cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(148); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 200 * 1024; cfg.stream = st;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k, tm, (const uint8_t*)src, 2000, mode, sink);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    cudaEventRecord(a, st); cudaGraphLaunch(ge, st); cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("mode %2d: %.2f us per 2-us kernel (%s)\n", mode, ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
