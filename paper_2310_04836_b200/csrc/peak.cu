// Measured dense INT8 tensor-core peak of this GPU (the INT8
// roofline denominator): every SM pair issues tcgen05.mma.cta_group::2.kind::i8
// (M = 256, N = 256, K = 32 per instruction — the shape K5p uses) back to back
// from operands resident in shared memory, accumulating into tensor memory.
// No global traffic inside the timed loop, so the figure is the tensor pipe's
// sustained issue rate at the clock the GPU runs (bench.py reports it beside
// the cuBLASLt and 2 x bf16 figures).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "ptx.cuh"

namespace dgqk {
namespace peak {

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mma2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::
          "r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

// grid: 2 * pairs CTAs in clusters of 2; 128 threads; `blocks` k-blocks of 4
// MMAs each (alternating two accumulator sets so consecutive MMAs of different
// k-blocks do not serialise on one accumulator).
__global__ void __launch_bounds__(128, 1) k_i8_peak(int blocks, unsigned long long* sink) {
  __shared__ __align__(1024) uint8_t sA[128 * 128];
  __shared__ __align__(1024) uint8_t sB[128 * 128];
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) {
    sA[i] = static_cast<uint8_t>(i * 7 + 1);
    sB[i] = static_cast<uint8_t>(i * 13 + 3);
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cooperative_groups::this_cluster().sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (cta_rank() == 0 && warp == 0) {
    constexpr uint32_t kIdesc = idesc_i8(256, 256);
    const uint64_t da = umma_desc_sw128(smem_u32(sA));
    const uint64_t db = umma_desc_sw128(smem_u32(sB));
    for (int kb = 0; kb < blocks; ++kb) {
      const uint32_t d = tmem + (kb & 1) * 256;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma2(d, da + 2 * kk, db + 2 * kk, kIdesc, kb >= 2 || kk != 0);
    }
    commit2(&done);
  }
  __syncwarp();
  mbar_wait(&done, 0);  // both CTAs: the pair's MMAs are complete
  tc_fence_after();
  if (warp == 0) {
    uint32_t v[8];
    tmem_ld8(tmem, v);
    tmem_ld_wait();
    if (threadIdx.x == 0 && v[0] == 0x7FFFFFFFu) *sink = v[1];  // keep the accumulator live
  }
  tc_fence_before();
  cooperative_groups::this_cluster().sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

}  // namespace peak
}  // namespace dgqk

cudaError_t dgq_launch_i8_peak(int pairs, int blocks, unsigned long long* sink, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, dgqk::peak::k_i8_peak, blocks, sink);
}
