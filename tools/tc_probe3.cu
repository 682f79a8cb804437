// MMA (TS, kind::i8, M=128 N=8, K=32) issue rate under concurrent TMEM traffic
// from other warps: none / tcgen05.st x16 / tcgen05.ld x32 loops.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "ptx.cuh"
using namespace dgqk;
__device__ __forceinline__ long long clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory"); return c; }

__global__ void k(long long* out, int mode, int ss, int u8) {
  __shared__ __align__(1024) uint8_t sB[16384];
  __shared__ __align__(1024) uint8_t sA[16384];
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) { sB[i] = 1; sA[i] = 1; }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    if (lane == 0) {
      const uint32_t idesc = u8 ? idesc_u8s8(128, 8) : idesc_i8(128, 8);
      const uint64_t db = umma_desc_sw128(smem_u32(sB));
      const uint64_t da = umma_desc_sw128(smem_u32(sA));
      long long t0 = clk();
      for (int it = 0; it < 1024; ++it) {
        const int kk = it & 3;
        if (ss) mma_i8_ss(tmem + 256 + ((it >> 2) & 7) * 8, da + 2 * kk, db + 2 * kk, idesc, kk ? 1u : 0u);
        else mma_i8_ts(tmem + 256 + ((it >> 2) & 7) * 8, tmem + kk * 8, db + 2 * kk, idesc, kk ? 1u : 0u);
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      out[0] = clk() - t0;
      stop = 1;
    }
    __syncwarp();
  } else if (mode == 1 && warp >= 4) {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = lane * i;
    long long n = 0;
    while (!stop) {
      tmem_st16(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 64 + (warp >> 2) * 16, v);
      tmem_st_wait();
      ++n;
    }
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(out + 1), n);
  } else if (mode == 2 && warp >= 4) {
    uint32_t d[32];
    long long n = 0; uint32_t acc = 0;
    while (!stop) {
      tmem_ld32(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 320, d);
      tmem_ld_wait();
      acc += d[lane];
      ++n;
    }
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(out + 1), n + (acc == 12345));
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  const char* names[3] = {"alone", "8 warps tcgen05.st x16", "8 warps tcgen05.ld x32"};
  for (int u8 = 0; u8 < 2; ++u8)
  for (int ss = 0; ss < 2; ++ss)
    for (int mode = 0; mode < 2; ++mode) {
      cudaMemset(d, 0, 64);
      k<<<1, 384>>>(d, mode, ss, u8);
      cudaMemset(d, 0, 64);
      k<<<1, 384>>>(d, mode, ss, u8);
      long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("%s %s MMA N=8, %-24s: %.1f cycles per MMA; other-warp ops %lld (%s)\n", u8 ? "u8" : "s8", ss ? "SS" : "TS", names[mode],
             h[0] / 1024.0, h[1], cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
