// Microbenchmark of the tcgen05 primitives the decode kernel uses (one CTA):
// cycles per tcgen05.st (32x32b.x16) + wait::st, per tcgen05.mma kind::i8 with
// A in TMEM / in SMEM (M = 128, N = 8..256, K = 32) issue, and commit latency.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_04836_b200/csrc -o tc_probe tools/tc_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "ptx.cuh"

using namespace dgqk;

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %clock64;" : "=l"(c));
  return c;
}

template <int N>
__global__ void k_probe(long long* out, int iters) {
  __shared__ __align__(1024) uint8_t sB[256 * 128 - 1024];
  __shared__ __align__(1024) uint8_t sA[128 * 128];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 256 * 128; i += blockDim.x) sB[i] = 1;
  for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) sA[i] = 1;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  // (1) tcgen05.st x16 + wait, all 4 warps
  {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = i * lane;
    __syncthreads();
    long long t0 = clk();
    for (int it = 0; it < iters; ++it) {
      tmem_st16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + (it & 7) * 16, v);
      tmem_st_wait();
    }
    long long t1 = clk();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
    long long t2 = clk();
    for (int it = 0; it < iters; ++it) tmem_st16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + (it & 7) * 16, v);
    tmem_st_wait();
    long long t3 = clk();
    if (threadIdx.x == 0) out[1] = (t3 - t2) / iters;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // (2) MMA issue cost (TS and SS), one thread; then commit -> mbarrier latency
  if (threadIdx.x == 0) {
    const uint32_t idesc_ts = idesc_u8s8(128, N);
    const uint32_t idesc_ss = idesc_i8(128, N);
    const uint64_t db = umma_desc_sw128(smem_u32(sB));
    const uint64_t da = umma_desc_sw128(smem_u32(sA));
    uint32_t phase = 0;
    long long t0 = clk();
    for (int it = 0; it < iters; ++it) mma_i8_ts(tmem + 256, tmem + (it & 3) * 8, db + 2 * (it & 3), idesc_ts, 1);
    long long t1 = clk();
    mma_commit(&bar);
    mbar_wait(&bar, phase);
    phase ^= 1;
    long long t2 = clk();
    out[2] = (t1 - t0) / iters;
    out[3] = t2 - t1;
    t0 = clk();
    for (int it = 0; it < iters; ++it) mma_i8_ss(tmem + 256, da + 2 * (it & 3), db + 2 * (it & 3), idesc_ss, 1);
    t1 = clk();
    mma_commit(&bar);
    mbar_wait(&bar, phase);
    phase ^= 1;
    t2 = clk();
    out[4] = (t1 - t0) / iters;
    out[5] = t2 - t1;
    // single MMA + commit round trip
    t0 = clk();
    for (int it = 0; it < 16; ++it) {
      mma_i8_ts(tmem + 256, tmem, db, idesc_ts, 1);
      mma_commit(&bar);
      mbar_wait(&bar, phase);
      phase ^= 1;
    }
    t1 = clk();
    out[6] = (t1 - t0) / 16;
    // 4 MMAs + 3 commits (the decode unit)
    t0 = clk();
    for (int it = 0; it < 16; ++it) {
      for (int kk = 0; kk < 4; ++kk) mma_i8_ts(tmem + 256, tmem + kk * 8, db + 2 * kk, idesc_ts, kk ? 1u : 0u);
      mma_commit(&bar);
      mbar_wait(&bar, phase);
      phase ^= 1;
    }
    t1 = clk();
    out[7] = (t1 - t0) / 16;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // (3) tcgen05.ld x8 + wait
  {
    uint32_t d[8];
    long long t0 = clk();
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
      tmem_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 256 + (it & 7) * 8, d);
      tmem_ld_wait();
      acc += d[0];
    }
    long long t1 = clk();
    if (threadIdx.x == 0) out[8] = (t1 - t0) / iters;
    if (acc == 12345) out[15] = acc;
  }
  // (3b) tcgen05.st / ld latency while another warp keeps the tensor core busy
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  {
    if (threadIdx.x == 0) {
      const uint32_t idesc_ts = idesc_u8s8(128, N);
      const uint64_t db = umma_desc_sw128(smem_u32(sB));
      for (int it = 0; it < 64; ++it) mma_i8_ts(tmem + 256, tmem + (it & 3) * 8, db + 2 * (it & 3), idesc_ts, 1);
    }
    if (warp >= 1) {
      uint32_t v[16];
      for (int i = 0; i < 16; ++i) v[i] = i * lane;
      long long t0 = clk();
      for (int it = 0; it < 16; ++it) {
        tmem_st16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 128 + (it & 3) * 16, v);
        tmem_st_wait();
      }
      long long t1 = clk();
      uint32_t d[8];
      for (int it = 0; it < 16; ++it) {
        tmem_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 448 + (it & 3) * 8, d);
        tmem_ld_wait();
      }
      long long t2 = clk();
      if (threadIdx.x == 32) {
        out[10] = (t1 - t0) / 16;
        out[11] = (t2 - t1) / 16;
      }
    }
    if (threadIdx.x == 0) {
      long long t0 = clk();
      mma_commit(&bar);
      mbar_wait(&bar, 0);  // phase after the probes above: recomputed below
      out[12] = clk() - t0;
    }
  }
  // (4) clock rate reference: globaltimer vs clock64 over a spin
  if (threadIdx.x == 0) {
    uint64_t g0, g1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g0));
    long long c0 = clk();
    while (clk() - c0 < 2000000) {
    }
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g1));
    out[9] = static_cast<long long>(2000000.0 / ((g1 - g0) * 1e-9) / 1e6);  // MHz
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int N>
void run() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  cudaMemset(d, 0, 16 * sizeof(long long));
  k_probe<N><<<1, 128>>>(d, 256);
  k_probe<N><<<1, 128>>>(d, 256);
  long long h[16];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("N=%3d: sttm.x16+wait %lld cyc, sttm.x16 pipelined %lld | mma TS issue %lld cyc/instr, drain %lld | "
         "mma SS issue %lld, drain %lld | 1 mma+commit RT %lld | 4 mma+commit RT %lld | ldtm.x8+wait %lld | clk %lld MHz "
         "| under 64 busy MMAs: sttm+wait %lld ldtm+wait %lld (%s)\n",
         N, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9], h[10], h[11], cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<8>();
  run<16>();
  run<64>();
  run<256>();
  return 0;
}
