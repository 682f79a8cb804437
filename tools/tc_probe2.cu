// MMA issue-rate probe: one or two issuing warps, TS kind::i8 M=128 N=8/16,
// D address rotating like the decode kernel (4 MMAs per accumulator).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "ptx.cuh"
using namespace dgqk;
__device__ __forceinline__ long long clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory"); return c; }

template <int N>
__global__ void k(long long* out, int issuers, int rot) {
  __shared__ __align__(1024) uint8_t sB[16384];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sB[i] = 1;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  const int total = 512;
  if (warp < issuers && rot == 2) {
    const uint32_t idesc = idesc_u8s8(128, N);
    const uint64_t db = umma_desc_sw128(smem_u32(sB));
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const int mine = total / issuers;
    long long t0 = clk();
    for (int it = 0; it < mine; ++it) {
      const int kk = it & 3;
      const uint32_t d = tm + 256 + warp * 128 + ((it >> 2) & 7) * N;
      mma_i8_ts_warp(d, tm + warp * 64 + kk * 8, db + 2 * kk, idesc, kk ? 1u : 0u);
    }
    long long t1 = clk();
    mma_commit_warp(&bar[warp]);
    mbar_wait(&bar[warp], 0);
    long long t2 = clk();
    if (lane == 0) {
      out[warp * 2] = t1 - t0;
      out[warp * 2 + 1] = t2 - t0;
    }
  } else if (warp < issuers && lane == 0) {
    const uint32_t idesc = idesc_u8s8(128, N);
    const uint64_t db = umma_desc_sw128(smem_u32(sB));
    const int mine = total / issuers;
    long long t0 = clk();
    for (int it = 0; it < mine; ++it) {
      const int kk = it & 3;
      const uint32_t d = rot ? tmem + 256 + warp * 128 + ((it >> 2) & 7) * N : tmem + 256 + warp * 128;
      mma_i8_ts(d, tmem + warp * 64 + kk * 8, db + 2 * kk, idesc, kk ? 1u : 0u);
    }
    long long t1 = clk();
    mma_commit(&bar[warp]);
    mbar_wait(&bar[warp], 0);
    long long t2 = clk();
    out[warp * 2] = t1 - t0;
    out[warp * 2 + 1] = t2 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int N> void run(int issuers, int rot) {
  long long* d; cudaMalloc(&d, 64); cudaMemset(d, 0, 64);
  k<N><<<1, 128>>>(d, issuers, rot); k<N><<<1, 128>>>(d, issuers, rot);
  long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("N=%d issuers=%d rot=%d: 512 MMAs: issue %lld / %lld cyc, complete %lld / %lld cyc -> %.1f cyc per MMA (%s)\n", N,
         issuers, rot, h[0], h[2], h[1], h[3], (double)(h[1] > h[3] ? h[1] : h[3]) / 512, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() {
  for (int rot = 1; rot < 3; ++rot) { run<8>(1, rot); run<8>(2, rot); run<16>(1, rot); run<16>(2, rot); }
  return 0;
}
