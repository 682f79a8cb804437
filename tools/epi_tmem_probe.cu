// The K5p exposed-epilogue drain in isolation, from real TMEM: one CTA per SM
// holds a 128-row x 512-column int32 accumulator (two 256-column sub-tiles),
// and W warps (W / 4 per TMEM lane quadrant, 32-column units split between
// them) turn it into FP16 rows in global memory the way csrc/prefill.cu's
// epi_direct does (16-column tcgen05.ld, (acc*rs)*s1, 64-byte swizzled staging
// rows, transposed 16-byte stores).  Reports SM cycles per drain (both
// sub-tiles), averaged over CTAs, for W = 8 / 12 / 16 and variants:
//   0 = epi_direct's structure, 1 = TMEM loads only, 2 = 32-column loads,
//   3 = the next unit's first load issued before the stores (no register cap here),
//   4 = no global stores, 6 = 256-bit global stores, 7 = no staging: each lane
//   stores its row's 16 values with one 32-byte store, 8 / 9 = .cs / .cg stores; and the W = 12 drain on
//   8 / 37 / 74 / 148 CTAs, and 128-byte staging rows
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_04836_b200/csrc -o tools/_bin/epi_tmem_probe tools/epi_tmem_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "ptx.cuh"
using namespace dgqk;

__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(dst)) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t t) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(t) : "memory");
}

template <int W, int V, int EX = 0>
__global__ void __launch_bounds__((W + EX) * 32, 1) k_drain(__half* __restrict__ out, const float* __restrict__ s1g,
                                                    unsigned long long* cyc, int reps, int ldy_ = 512) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t stop;
  __shared__ __align__(16) float s_s1[512];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, jq = warp >> 2;
  constexpr int kPerQ = W / 4, kUnits = 8;  // 32-column units per 256-column sub-tile
  const int cbeg = (jq * kUnits / kPerQ) * 32, cend = ((jq + 1) * kUnits / kPerQ) * 32;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) s_s1[i] = s1g[i & 255];
  if (threadIdx.x == 0) {
    mbar_init(&stop, W);
    fence_mbar_init();
  }
  if (warp == 0) {
    if (V == 10)
      tmem_alloc_pair(&tslot);  // as the pair kernel allocates (2-CTA cluster launch)
    else
      tmem_alloc<512>(&tslot);
  }
  tc_fence_before();
  if (V == 10) asm volatile("barrier.cluster.arrive.aligned; barrier.cluster.wait.aligned;" ::: "memory");
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp >= W) {  // EX warps waiting on an mbarrier during every drain (the kernel's idle roles)
    tc_fence_before();
    __syncthreads();  // the fill barrier
    for (int rep = 0; rep < reps; ++rep) {
      __syncthreads();
      while (!mbar_try_wait(&stop, rep & 1)) {
      }
      __syncthreads();
    }
    tc_fence_before();
    __syncthreads();
    return;
  }
  const uint32_t tl = tmem + (static_cast<uint32_t>(q * 32) << 16);
  // fill this warp's share of both sub-tiles
  for (int sub = 0; sub < 2; ++sub)
    for (int c = cbeg; c < cend; c += 16) {
      uint32_t v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = static_cast<uint32_t>(lane * 977 + (sub * 256 + c + k) * 131 - 20000);
      tmem_st16(tl + sub * 256 + c, v);
    }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint8_t* stg = smem + warp * 2048;
  uint8_t* myrow = stg + lane * 64;
  const uint32_t sw = (lane >> 1) & 3;
  const float rsm = 0.0123f + lane * 1e-4f;
  const size_t ldy = ldy_;
  unsigned long long total = 0;
  for (int rep = 0; rep < reps; ++rep) {
    __syncthreads();
    const long long t0 = clock64();
    for (int sub = 0; sub < 2; ++sub) {
      const uint32_t tb = tl + sub * 256;
      const float* sv1 = s_s1 + sub * 256;
      // rep-dependent column window when the rows are long: 20 reps touch 20x
      // the lines (more than L2 holds at row stride 28672), as a kernel streaming
      // a 117 MB output does
      const size_t cw = ldy >= 28672 ? static_cast<size_t>(rep % 28) * 1024 : 0;
      __half* orow = out + (static_cast<size_t>(blockIdx.x) * 128 + q * 32) * ldy + sub * 256 + cw;
      uint32_t r[2][16];
      if (V == 3) tmem_ld16(tb + cbeg, r[0]);
#pragma unroll 1
      for (int c0 = cbeg; c0 < cend; c0 += 32) {
        if (V == 1) {
          tmem_ld16(tb + c0, r[0]);
          tmem_ld16(tb + c0 + 16, r[1]);
          tmem_ld_wait();
          if (r[0][0] == 0x7FFFFFFFu && r[1][3] == 1u) myrow[0] = 1;
          continue;
        }
        uint32_t big[32];
        if (V == 2) {
          tmem_ld32(tb + c0, big);
          tmem_ld_wait();
        } else if (V == 0) {
          tmem_ld16(tb + c0, r[0]);
          tmem_ld_wait();
        } else {
          tmem_ld_wait();
        }
#pragma unroll
        for (int c16 = 0; c16 < 32; c16 += 16) {
          uint32_t(&cur)[16] = r[(c16 / 16) & 1];
          if (V == 2) {
#pragma unroll
            for (int k = 0; k < 16; ++k) cur[k] = big[c16 + k];
          } else if (c16 == 0) {
            tmem_ld16(tb + c0 + 16, r[1]);
          } else if (V == 3 && c0 + 32 < cend) {
            tmem_ld16(tb + c0 + 32, r[0]);
          }
          if (V == 7) {  // 16 values of this lane's row -> one 32-byte store, no staging
            uint32_t h[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float a = __fmul_rn(__fmul_rn(__int2float_rn(static_cast<int32_t>(cur[2 * k])), rsm), sv1[c0 + c16 + 2 * k]);
              const float b2 = __fmul_rn(__fmul_rn(__int2float_rn(static_cast<int32_t>(cur[2 * k + 1])), rsm),
                                         sv1[c0 + c16 + 2 * k + 1]);
              const __half2 hh = __floats2half2_rn(a, b2);
              h[k] = *reinterpret_cast<const uint32_t*>(&hh);
            }
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(orow + lane * ldy + c0 + c16),
                         "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7])
                         : "memory");
            if (c16 == 0) tmem_ld_wait();
            continue;
          }
#pragma unroll
          for (int c8 = 0; c8 < 16; c8 += 8) {
            const int c1 = c16 + c8;
            const float4 sa = *reinterpret_cast<const float4*>(sv1 + c0 + c1);
            const float4 sb = *reinterpret_cast<const float4*>(sv1 + c0 + c1 + 4);
            const float s[8] = {sa.x, sa.y, sa.z, sa.w, sb.x, sb.y, sb.z, sb.w};
            uint32_t h[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float a = __fmul_rn(__fmul_rn(__int2float_rn(static_cast<int32_t>(cur[c8 + 2 * k])), rsm), s[2 * k]);
              const float b =
                  __fmul_rn(__fmul_rn(__int2float_rn(static_cast<int32_t>(cur[c8 + 2 * k + 1])), rsm), s[2 * k + 1]);
              const __half2 hh = __floats2half2_rn(a, b);
              h[k] = *reinterpret_cast<const uint32_t*>(&hh);
            }
            *reinterpret_cast<uint4*>(myrow + (((c1 / 8) ^ sw) << 4)) = make_uint4(h[0], h[1], h[2], h[3]);
          }
          if (V != 2 && c16 == 0) tmem_ld_wait();
        }
        if (V == 7) continue;
        __syncwarp();
        const int ch = lane & 3;
        if (V == 4) {
          if (stg[lane] == 0x5A && rep < 0) orow[0] = __float2half(1.0f);
          continue;
        }
        if (V == 6) {  // 256-bit stores: two lanes per 64-byte row segment, 16 rows per instruction
          const int hf = lane & 1;
#pragma unroll
          for (int it = 0; it < 2; ++it) {
            const int row = it * 16 + (lane >> 1);
            const int rsw = (row >> 1) & 3;
            const uint4 a = *reinterpret_cast<const uint4*>(stg + row * 64 + (((2 * hf) ^ rsw) << 4));
            const uint4 b = *reinterpret_cast<const uint4*>(stg + row * 64 + (((2 * hf + 1) ^ rsw) << 4));
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(orow + row * ldy + c0 + hf * 16),
                         "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                         : "memory");
          }
          __syncwarp();
          continue;
        }
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int row = it * 8 + (lane >> 2);
          const uint4 v = *reinterpret_cast<const uint4*>(stg + row * 64 + ((ch ^ ((row >> 1) & 3)) << 4));
          if (V == 8)  // streaming store (.cs: evict-first)
            __stcs(reinterpret_cast<uint4*>(orow + row * ldy + c0 + ch * 8), v);
          else if (V == 9)  // L2-cached only (.cg)
            __stcg(reinterpret_cast<uint4*>(orow + row * ldy + c0 + ch * 8), v);
          else
            *reinterpret_cast<uint4*>(orow + row * ldy + c0 + ch * 8) = v;
        }
        __syncwarp();
      }
      if (V == 3) tmem_ld_wait();
    }
    if (lane == 0) mbar_arrive(&stop);
    __syncthreads();
    if (rep == 0 && threadIdx.x == 0) cyc[148 + blockIdx.x] = clock64() - t0;  // first (cold) drain
    total += clock64() - t0;
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = total / reps;
  tc_fence_before();
  __syncthreads();
  if (V == 10) {
    asm volatile("barrier.cluster.arrive.aligned; barrier.cluster.wait.aligned;" ::: "memory");
    if (warp == 0) tmem_dealloc_pair(tmem);
  } else if (warp == 0) {
    tmem_dealloc<512>(tmem);
  }
}

// 128-byte staging rows (64-column units, 4 KB per warp): each 16-byte store
// instruction writes four whole 128-byte row segments instead of eight 64-byte ones
template <int W>
__global__ void __launch_bounds__(W * 32, 1) k_drain128(__half* __restrict__ out, const float* __restrict__ s1g,
                                                       unsigned long long* cyc, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(16) float s_s1[512];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, jq = warp >> 2;
  constexpr int kPerQ = W / 4, kUnits = 4;  // 64-column units per 256-column sub-tile
  const int cbeg = (jq * kUnits / kPerQ) * 64, cend = ((jq + 1) * kUnits / kPerQ) * 64;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) s_s1[i] = s1g[i & 255];
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t tl = tmem + (static_cast<uint32_t>(q * 32) << 16);
  __syncthreads();
  uint8_t* stg = smem + warp * 4096;
  uint8_t* myrow = stg + lane * 128;
  const uint32_t sw = lane & 7;
  const float rsm = 0.0123f + lane * 1e-4f;
  const size_t ldy = 512;
  unsigned long long total = 0;
  for (int rep = 0; rep < reps; ++rep) {
    __syncthreads();
    const long long t0 = clock64();
    for (int sub = 0; sub < 2; ++sub) {
      const uint32_t tb = tl + sub * 256;
      const float* sv1 = s_s1 + sub * 256;
      __half* orow = out + (static_cast<size_t>(blockIdx.x) * 128 + q * 32) * ldy + sub * 256;
#pragma unroll 1
      for (int c0 = cbeg; c0 < cend; c0 += 64) {
        uint32_t r[2][16];
        tmem_ld16(tb + c0, r[0]);
        tmem_ld_wait();
#pragma unroll
        for (int c16 = 0; c16 < 64; c16 += 16) {
          uint32_t(&cur)[16] = r[(c16 / 16) & 1];
          if (c16 + 16 < 64) tmem_ld16(tb + c0 + c16 + 16, r[((c16 / 16) + 1) & 1]);
#pragma unroll
          for (int c8 = 0; c8 < 16; c8 += 8) {
            const int c1 = c16 + c8;
            const float4 sa = *reinterpret_cast<const float4*>(sv1 + c0 + c1);
            const float4 sb = *reinterpret_cast<const float4*>(sv1 + c0 + c1 + 4);
            const float sv[8] = {sa.x, sa.y, sa.z, sa.w, sb.x, sb.y, sb.z, sb.w};
            uint32_t h[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float a = __fmul_rn(__fmul_rn(__int2float_rn(static_cast<int32_t>(cur[c8 + 2 * k])), rsm), sv[2 * k]);
              const float b =
                  __fmul_rn(__fmul_rn(__int2float_rn(static_cast<int32_t>(cur[c8 + 2 * k + 1])), rsm), sv[2 * k + 1]);
              const __half2 hh = __floats2half2_rn(a, b);
              h[k] = *reinterpret_cast<const uint32_t*>(&hh);
            }
            *reinterpret_cast<uint4*>(myrow + (((c1 / 8) ^ sw) << 4)) = make_uint4(h[0], h[1], h[2], h[3]);
          }
          if (c16 + 16 < 64) tmem_ld_wait();
        }
        __syncwarp();
        const int ch = lane & 7;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int row = it * 4 + (lane >> 3);
          const uint4 v = *reinterpret_cast<const uint4*>(stg + row * 128 + ((ch ^ (row & 7)) << 4));
          *reinterpret_cast<uint4*>(orow + row * ldy + c0 + ch * 8) = v;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    total += clock64() - t0;
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = total / reps;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// L2 read stream (the main loops of the other pairs): each CTA streams a
// 24 MB buffer (L2-resident) with 16-byte loads until `stop` is set
__global__ void k_l2_stream(const uint4* __restrict__ src, size_t n, volatile int* stop, unsigned long long* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  size_t i = blockIdx.x * blockDim.x + threadIdx.x;
  int iter = 0;
  while (true) {
    const uint4 v = src[i];
    acc.x ^= v.x; acc.y += v.y;
    i += static_cast<size_t>(gridDim.x) * blockDim.x;
    if (i >= n) i -= n;
    if ((++iter & 255) == 0 && *stop) break;
  }
  if (acc.x == 0x12345678u) *sink = acc.y;
}

template <int W>
static void run128(__half* out, const float* s1, unsigned long long* cyc) {
  auto k = k_drain128<W>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, W * 4096);
  k<<<148, W * 32, W * 4096>>>(out, s1, cyc, 20);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += h[i];
  printf("W=%2d 128-byte rows: %7.0f cycles per 128x512 drain = %.2f us at 1.93 GHz\n", W, m / 148, m / 148 / 1930.0);
}

template <int W, int V, int EX = 0>
static void run(__half* out, const float* s1, unsigned long long* cyc, int ctas = 148, int ldy = 512) {
  auto k = k_drain<W, V, EX>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, W * 2048);
  cudaMemset(cyc, 0, 296 * 8);
  k<<<ctas, (W + EX) * 32, W * 2048>>>(out, s1, cyc, 20, ldy);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("W=%d V=%d error %s\n", W, V, cudaGetErrorString(e));
    return;
  }
  unsigned long long h[296];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0, mx = 0, m0 = 0;
  for (int i = 0; i < ctas; ++i) {
    m += h[i];
    m0 += h[148 + i];
    mx = h[i] > mx ? h[i] : mx;
  }
  printf("   first (cold) drain: %7.0f cycles\n", m0 / ctas);
  printf("W=%2d variant %d, %2d waiting warps, %3d CTAs, row stride %5d: %7.0f cycles per 128x512 drain (max %7.0f) = %.2f us\n",
         W, V, EX, ctas, ldy, m / ctas, mx, m / ctas / 1930.0);
}

int main() {
  __half* out;
  float* s1;
  unsigned long long* cyc;
  cudaMalloc(&out, 148ull * 128 * 28672 * 2);
  cudaMalloc(&s1, 256 * 4);
  cudaMalloc(&cyc, 296 * 8);
  float hs[256];
  for (int i = 0; i < 256; ++i) hs[i] = 0.5f + i * 1e-3f;
  cudaMemcpy(s1, hs, sizeof(hs), cudaMemcpyHostToDevice);
  run<8, 0>(out, s1, cyc);
  run<8, 1>(out, s1, cyc);
  run<12, 0>(out, s1, cyc);
  run<12, 1>(out, s1, cyc);
  run<12, 2>(out, s1, cyc);
  run<12, 3>(out, s1, cyc);
  run<16, 0>(out, s1, cyc);
  run<16, 1>(out, s1, cyc);
  run<16, 2>(out, s1, cyc);
  run<16, 3>(out, s1, cyc);
  run<32, 0>(out, s1, cyc);
  run<32, 1>(out, s1, cyc);
  run<12, 4>(out, s1, cyc);
  run<16, 4>(out, s1, cyc);
  for (int n : {8, 37, 74, 148}) run<12, 0>(out, s1, cyc, n);
  run<12, 0, 9>(out, s1, cyc, 148, 28672);  // + the kernel's 9 other warps waiting on mbarriers
  run<12, 0>(out, s1, cyc, 148, 28672);  // OPT-30B fc1 output rows
  run<12, 0>(out, s1, cyc, 148, 7168);
  {
    auto k = k_drain<12, 10, 0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 2048);
    cudaMemset(cyc, 0, 296 * 8);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(12 * 32);
    cfg.dynamicSmemBytes = 12 * 2048;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, out, (const float*)s1, cyc, 20, 28672);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    printf("W=12 drain, TMEM allocated cta_group::2 in 2-CTA clusters: %7.0f cycles = %.2f us (%s)\n", m / 148,
           m / 148 / 1930.0, cudaGetErrorString(e));
  }
  run<12, 8>(out, s1, cyc, 148, 28672);
  run<12, 9>(out, s1, cyc, 148, 28672);
  run<12, 0>(out, s1, cyc, 148, 28672);
  run<12, 7>(out, s1, cyc);
  run<12, 7>(out, s1, cyc, 148, 28672);
  run<16, 7>(out, s1, cyc);
  run<8, 7>(out, s1, cyc);
  run<12, 6>(out, s1, cyc);
  run<16, 6>(out, s1, cyc);
  run<8, 6>(out, s1, cyc);
  {
    // the drain on 74 SMs while 74 other SMs stream L2 reads
    uint4* src;
    int* stop;
    unsigned long long* sink;
    const size_t n = (24u << 20) / 16;
    cudaMalloc(&src, n * 16);
    cudaMemset(src, 1, n * 16);
    cudaMalloc(&stop, 4);
    cudaMalloc(&sink, 8);
    cudaMemset(stop, 0, 4);
    cudaStream_t sa, sb;
    cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
    k_l2_stream<<<74, 1024, 0, sb>>>(src, n, stop, sink);
    auto k = k_drain<12, 0, 0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 2048);
    cudaMemset(cyc, 0, 296 * 8);
    k<<<74, 12 * 32, 12 * 2048, sa>>>(out, s1, cyc, 20, 28672);
    cudaStreamSynchronize(sa);
    int one = 1;
    cudaMemcpy(stop, &one, 4, cudaMemcpyHostToDevice);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    int cnt = 0;
    for (int i = 0; i < 148; ++i)
      if (h[i]) { m += h[i]; ++cnt; }
    printf("W=12 drain on %d CTAs beside an L2 read stream on 74 SMs: %7.0f cycles = %.2f us\n", cnt, m / cnt,
           m / cnt / 1930.0);
  }
  run<12, 0>(out, s1, cyc, 74, 28672);
  run128<8>(out, s1, cyc);
  run128<16>(out, s1, cyc);
  return 0;
}
