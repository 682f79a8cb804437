// K1 — per-token INT8 activation quantisation after percentile-clip smoothing.
//
// Restates proj/src/kernel.cpp:14-44 (quantize_activations) for the GPU:
//   x'  = x / k[j]                                  (IEEE fp32 division)
//   s   = dynamic ? float(max(double(max|x'|)/127, double(1e-8f))) : act_scale
//   q   = clamp(rhe(double(x')/double(s)), -127, 127)
// bit-exact (see numerics.cuh).  One CTA per token row; the row stays in
// registers between the absmax reduction and the quantisation (128-bit
// loads, X is read from HBM exactly once).  Output rows are written with a
// padded stride ldq >= K and the pad columns zero-filled, which is the
// layout the GEMM's TMA expects.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include "kernels.h"
#include "numerics.cuh"
#include "ptx.cuh"

namespace cg = cooperative_groups;

namespace dgqk {

template <int T>
__device__ __forceinline__ float block_max(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < T / 32 ? red[l] : 0.0f;
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0) red[32] = v;
  }
  __syncthreads();
  float r = red[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
  return (static_cast<uint32_t>(a) & 0xFFu) | ((static_cast<uint32_t>(b) & 0xFFu) << 8) |
         ((static_cast<uint32_t>(c) & 0xFFu) << 16) | ((static_cast<uint32_t>(d) & 0xFFu) << 24);
}

// Generic path: any K / alignment.  Two passes over the row (the second hits L2).
template <int T>
__global__ void __launch_bounds__(T) k_actquant_any(const float* __restrict__ X, size_t ldx,
                                                     const float* __restrict__ kv, int K, int Kpad,
                                                     int dynamic, float act_scale, int8_t* __restrict__ Q,
                                                     size_t ldq, float* __restrict__ rs, int M) {
  __shared__ float red[33];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int row = blockIdx.x; row < M; row += gridDim.x) {
    const float* xr = X + static_cast<size_t>(row) * ldx;
    float s = act_scale;
    if (dynamic) {
      float am = 0.0f;
      for (int j = threadIdx.x; j < K; j += T) am = fmaxf(am, fabsf(__fdiv_rn(xr[j], kv[j])));
      s = dynamic_row_scale(block_max<T>(am, red));
    }
    if (threadIdx.x == 0) rs[row] = s;
    int8_t* qr = Q + static_cast<size_t>(row) * ldq;
    const bool safe = scale_is_safe(s);
    const float inv = __frcp_rn(s);
    for (int j = threadIdx.x; j < K; j += T) {
      const float x = __fdiv_rn(xr[j], kv[j]);
      qr[j] = static_cast<int8_t>(safe ? quant_code_f32(x, s, inv) : quant_code_f64(x, s));
    }
    for (int j = K + threadIdx.x; j < Kpad; j += T) qr[j] = 0;
  }
}

// FP16 input (the inter-layer activation format), optionally stored as the
// all-gather of column shards: logical element (m, j) lives at
//   X + (j / seg) * seg_stride + m * ldx + (j % seg)
// so the next layer quantises the gathered [p][M][K/p] buffer in place.
// float(x_f16) is exact, so this equals K1 on the float32 copy bit-for-bit.
// Generic FP16 path (any K / segment geometry); the vector paths are k_actquant2/3.
template <int T>
__global__ void __launch_bounds__(T) k_actquant_h_any(const __half* __restrict__ X, size_t ldx, int seg,
                                                       size_t seg_stride, const float* __restrict__ kv, int K,
                                                       int Kpad, int dynamic, float act_scale,
                                                       int8_t* __restrict__ Q, size_t ldq, float* __restrict__ rs,
                                                       int M) {
  __shared__ float red[33];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int row = blockIdx.x; row < M; row += gridDim.x) {
    auto at = [&](int j) {
      return __half2float(X[static_cast<size_t>(j / seg) * seg_stride + static_cast<size_t>(row) * ldx + (j % seg)]);
    };
    float s = act_scale;
    if (dynamic) {
      float am = 0.0f;
      for (int j = threadIdx.x; j < K; j += T) am = fmaxf(am, fabsf(__fdiv_rn(at(j), kv[j])));
      s = dynamic_row_scale(block_max<T>(am, red));
    }
    if (threadIdx.x == 0) rs[row] = s;
    int8_t* qr = Q + static_cast<size_t>(row) * ldq;
    const bool safe = scale_is_safe(s);
    const float inv = __frcp_rn(s);
    for (int j = threadIdx.x; j < K; j += T) {
      const float x = __fdiv_rn(at(j), kv[j]);
      qr[j] = static_cast<int8_t>(safe ? quant_code_f32(x, s, inv) : quant_code_f64(x, s));
    }
    for (int j = K + threadIdx.x; j < Kpad; j += T) qr[j] = 0;
  }
}

// ---- K1 v2: one row per CL-CTA cluster, 8-element chunks, loads front-loaded ----
// chunk c of a row (elements 8c..8c+7) belongs to cluster rank c / (T*V); every
// thread first issues all of its V 16-B (f16) or 32-B (f32) loads, then divides
// by k with the hoisted reciprocal (div_k), reduces the row absmax (block, then
// over the cluster through DSMEM), and quantises from registers.
// x' = x / k for one 8-channel chunk c.  kone[c] != 0 marks a chunk whose eight
// k are exactly 1 (compute_smooth, proj/src/smoothing.cpp:45-47, gives k =
// max(1, z/threshold): all but the top `percentile` channels): x / 1 == x in
// IEEE arithmetic for every finite x, so the division and the k / RN(1/k)
// loads are skipped.
template <bool kCheckX, bool kCheckK>
__device__ __forceinline__ void smooth_chunk(const float (&x)[8], const float* __restrict__ kv,
                                             const float* __restrict__ rkv, bool unit, int c, float (&q)[8]) {
  if (unit) {
#pragma unroll
    for (int t = 0; t < 8; ++t) q[t] = x[t];
    return;
  }
  const int j = c * 8;
  const float4 k0 = __ldg(reinterpret_cast<const float4*>(kv + j));
  const float4 k1 = __ldg(reinterpret_cast<const float4*>(kv + j + 4));
  const float4 r0 = __ldg(reinterpret_cast<const float4*>(rkv + j));
  const float4 r1 = __ldg(reinterpret_cast<const float4*>(rkv + j + 4));
  const float kk[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
  const float rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
  div_chunk<kCheckX, kCheckK>(x, kk, rr, q);
}

// Bit v: chunk threadIdx.x-based index cbase + v*T is a unit-k chunk.  Built
// once per kernel with all V flag loads in flight together (a flag load per
// chunk inside the row loop was a dependent L2 round trip: 34 % of K1's stall
// samples, profiles/ncu_summary_r01c.json era capture).
template <int T, int V>
__device__ __forceinline__ uint32_t unit_mask(const uint8_t* __restrict__ kone, int cbase, int C8) {
  if (!kone) return 0u;
  uint8_t f[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c = cbase + v * T;
    f[v] = c < C8 ? __ldg(kone + c) : 0;
  }
  uint32_t m = 0;
#pragma unroll
  for (int v = 0; v < V; ++v) m |= (f[v] ? 1u : 0u) << v;
  return m;
}

template <int T, int V, int CL, bool kF16, bool kCheckK>
__global__ void __launch_bounds__(T) k_actquant2(const void* __restrict__ Xv, size_t ldx, int seg, size_t seg_stride,
                                                  const float* __restrict__ kv, const float* __restrict__ rkv,
                                                  const uint8_t* __restrict__ kone, int K, int Kpad, int dynamic,
                                                  float act_scale, int8_t* __restrict__ Q, size_t ldq,
                                                  float* __restrict__ rs, int M) {
  __shared__ float red[33];
  __shared__ float cl_max;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int row = blockIdx.x / CL;
  const int part = blockIdx.x % CL;
  if (row >= M) return;  // grid is exactly M*CL; keeps the cluster barrier uniform
  const int C8 = K >> 3;
  const int cbase = part * T * V + threadIdx.x;
  const uint32_t umask = unit_mask<T, V>(kone, cbase, C8);
  uint4 raw[V][kF16 ? 1 : 2];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c = cbase + v * T;
    if (c < C8) {
      const int j = c * 8;
      if constexpr (kF16) {
        const __half* src = static_cast<const __half*>(Xv) + static_cast<size_t>(j / seg) * seg_stride +
                            static_cast<size_t>(row) * ldx + (j % seg);
        raw[v][0] = __ldcs(reinterpret_cast<const uint4*>(src));
      } else {
        const float* src = static_cast<const float*>(Xv) + static_cast<size_t>(row) * ldx + j;
        raw[v][0] = __ldcs(reinterpret_cast<const uint4*>(src));
        raw[v][1] = __ldcs(reinterpret_cast<const uint4*>(src + 4));
      }
    }
  }
  float xv[V][8];
  float am = 0.0f;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c = cbase + v * T;
    if (c < C8) {
      const int j = c * 8;
      float x[8];
      if constexpr (kF16) {
        const __half2* h2 = reinterpret_cast<const __half2*>(&raw[v][0]);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 f = __half22float2(h2[t]);
          x[2 * t] = f.x;
          x[2 * t + 1] = f.y;
        }
      } else {
        const float* f = reinterpret_cast<const float*>(&raw[v][0]);
#pragma unroll
        for (int t = 0; t < 8; ++t) x[t] = f[t];
      }
      smooth_chunk<!kF16, kCheckK>(x, kv, rkv, (umask >> v) & 1u, c, xv[v]);
#pragma unroll
      for (int t = 0; t < 8; ++t) am = fmaxf(am, fabsf(xv[v][t]));
    }
  }
  float s = act_scale;
  if (dynamic) {
    float bm = block_max<T>(am, red);
    if constexpr (CL > 1) {
      cg::cluster_group cluster = cg::this_cluster();
      if (threadIdx.x == 0) cl_max = bm;
      cluster.sync();
#pragma unroll
      for (int r = 0; r < CL; ++r) bm = fmaxf(bm, *cluster.map_shared_rank(&cl_max, r));
      cluster.sync();  // peers finished reading cl_max
    }
    s = dynamic_row_scale(bm);
  }
  if (part == 0 && threadIdx.x == 0) rs[row] = s;
  uint2* qr = reinterpret_cast<uint2*>(Q + static_cast<size_t>(row) * ldq);
  const bool safe = scale_is_safe(s);
  const float inv = __frcp_rn(s);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c = cbase + v * T;
    if (c < C8) {
      int o[8];
      if (safe) {
        if (dynamic)
          quant_chunk<false>(xv[v], s, inv, o);
        else
          quant_chunk<true>(xv[v], s, inv, o);
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) o[t] = quant_code_f64(xv[v][t], s);
      }
      qr[c] = make_uint2(pack4(o[0], o[1], o[2], o[3]), pack4(o[4], o[5], o[6], o[7]));
    }
  }
  if (part == 0)
    for (int c = C8 + threadIdx.x; c < (Kpad >> 3); c += T) qr[c] = make_uint2(0u, 0u);
}

// ---- K1 v3 (large M): persistent CTAs, whole rows staged in shared memory by
// 1-D TMA bulk copies two rows ahead (double buffer, one mbarrier each), so
// the HBM stream never waits for the divide / reduce / quantise of the
// previous row.  x' = x/k stays in registers between the absmax and the codes.
template <int T, int V, bool kF16, bool kCheckK>
__global__ void __launch_bounds__(T) k_actquant3(const void* __restrict__ Xv, size_t ldx, int seg, size_t seg_stride,
                                                  const float* __restrict__ kv, const float* __restrict__ rkv,
                                                  const uint8_t* __restrict__ kone, int K, int Kpad, int dynamic,
                                                  float act_scale, int8_t* __restrict__ Q, size_t ldq,
                                                  float* __restrict__ rs, int M) {
  extern __shared__ __align__(128) uint8_t sbuf[];
  __shared__ __align__(8) uint64_t full[2];
  __shared__ float red[33];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int kEsz = kF16 ? 2 : 4;
  const uint32_t rowbytes = static_cast<uint32_t>(K) * kEsz;
  const uint32_t bufstride = (rowbytes + 127u) & ~127u;
  const int C8 = K >> 3;
  const int nseg = K / seg;
  auto issue = [&](int r, int b) {  // thread 0 only
    dgqk::mbar_arrive_expect_tx(&full[b], rowbytes);
    for (int sg = 0; sg < nseg; ++sg) {
      const uint8_t* src = static_cast<const uint8_t*>(Xv) +
                           (static_cast<size_t>(sg) * seg_stride + static_cast<size_t>(r) * ldx) * kEsz;
      dgqk::bulk_load(sbuf + b * bufstride + static_cast<size_t>(sg) * seg * kEsz, src,
                      static_cast<uint32_t>(seg) * kEsz, &full[b]);
    }
  };
  if (threadIdx.x == 0) {
    dgqk::mbar_init(&full[0], 1);
    dgqk::mbar_init(&full[1], 1);
    dgqk::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t umask = unit_mask<T, V>(kone, static_cast<int>(threadIdx.x), C8);
  int it = 0;
  if (threadIdx.x == 0) {
    if (static_cast<int>(blockIdx.x) < M) issue(blockIdx.x, 0);
    if (static_cast<int>(blockIdx.x + gridDim.x) < M) issue(blockIdx.x + gridDim.x, 1);
  }
  for (int row = blockIdx.x; row < M; row += gridDim.x, ++it) {
    const int b = it & 1;
    dgqk::mbar_wait(&full[b], (it >> 1) & 1);
    const uint8_t* buf = sbuf + b * bufstride;
    float xv[V][8];
    float am = 0.0f;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c = threadIdx.x + v * T;
      if (c < C8) {
        const int j = c * 8;
        float x[8];
        if constexpr (kF16) {
          const uint4 raw = *reinterpret_cast<const uint4*>(buf + j * 2);
          const __half2* h2 = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 f = __half22float2(h2[t]);
            x[2 * t] = f.x;
            x[2 * t + 1] = f.y;
          }
        } else {
          const float4 a = *reinterpret_cast<const float4*>(buf + j * 4);
          const float4 bb = *reinterpret_cast<const float4*>(buf + j * 4 + 16);
          x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
          x[4] = bb.x; x[5] = bb.y; x[6] = bb.z; x[7] = bb.w;
        }
        smooth_chunk<!kF16, kCheckK>(x, kv, rkv, (umask >> v) & 1u, c, xv[v]);
#pragma unroll
        for (int t = 0; t < 8; ++t) am = fmaxf(am, fabsf(xv[v][t]));
      }
    }
    float s = act_scale;
    if (dynamic) {
      s = dynamic_row_scale(block_max<T>(am, red));  // its barriers also retire every read of buf
    } else {
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      rs[row] = s;
      const int nxt = row + 2 * gridDim.x;
      if (nxt < M) issue(nxt, b);
    }
    uint2* qr = reinterpret_cast<uint2*>(Q + static_cast<size_t>(row) * ldq);
    const bool safe = scale_is_safe(s);
    const float inv = __frcp_rn(s);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c = threadIdx.x + v * T;
      if (c < C8) {
        int o[8];
        if (safe) {
          if (dynamic)
            quant_chunk<false>(xv[v], s, inv, o);
          else
            quant_chunk<true>(xv[v], s, inv, o);
        } else {
#pragma unroll
          for (int t = 0; t < 8; ++t) o[t] = quant_code_f64(xv[v][t], s);
        }
        qr[c] = make_uint2(pack4(o[0], o[1], o[2], o[3]), pack4(o[4], o[5], o[6], o[7]));
      }
    }
    for (int c = C8 + threadIdx.x; c < (Kpad >> 3); c += T) qr[c] = make_uint2(0u, 0u);
  }
}

__global__ void k_reciprocal(const float* __restrict__ k, float* __restrict__ rk, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rk[i] = (k[i] <= 0x1p24f) ? __frcp_rn(k[i]) : 0.0f;  // 0 marks k outside div_k's fast range
}

// unit test hook: y[i] = div_k(x[i], k[i], RN(1/k[i])) next to __fdiv_rn
__global__ void k_div_check(const float* __restrict__ x, const float* __restrict__ k, float* __restrict__ fast,
                            float* __restrict__ ieee, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    fast[i] = div_k(x[i], k[i], __frcp_rn(k[i]));
    ieee[i] = __fdiv_rn(x[i], k[i]);
  }
}

}  // namespace dgqk

using namespace dgqk;

namespace {
template <int T, int V, int CL, bool F16, bool CK>
cudaError_t launch_aq2(const void* X, size_t ldx, int seg, size_t seg_stride, const float* k, const float* rk,
                       const uint8_t* kone, int K, int Kpad, int dynamic, float act_scale, int8_t* Q, size_t ldq,
                       float* rs, int M, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(M) * CL);
  cfg.blockDim = dim3(T);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = CL > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_actquant2<T, V, CL, F16, CK>, X, ldx, seg, seg_stride, k, rk, kone, K, Kpad,
                            dynamic, act_scale, Q, ldq, rs, M);
}
}  // namespace

cudaError_t dgq_launch_actquant2(const void* X, bool f16, size_t ldx, int seg, size_t seg_stride, const float* k,
                                 const float* rk, int K, int Kpad, int dynamic, float act_scale, int8_t* Q, size_t ldq,
                                 float* rs, int M, cudaStream_t st, bool k_checked, const uint8_t* kone) {
  if (M <= 0) return cudaSuccess;
  if (seg <= 0) seg = K;
  const size_t align = f16 ? 8 : 4;  // elements per 16 bytes
  const bool vec = rk && (K % 8 == 0) && (seg % 8 == 0) && (ldx % align == 0) && (seg_stride % align == 0) &&
                   (ldq % 8 == 0) && (Kpad % 8 == 0) && (reinterpret_cast<uintptr_t>(X) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(k) % 16 == 0) && (reinterpret_cast<uintptr_t>(rk) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(Q) % 8 == 0) && (f16 || seg == K);
  if (!vec) {
    if (f16)
      k_actquant_h_any<256><<<M, 256, 0, st>>>(static_cast<const __half*>(X), ldx, seg, seg_stride, k, K, Kpad,
                                                dynamic, act_scale, Q, ldq, rs, M);
    else
      k_actquant_any<256><<<M, 256, 0, st>>>(static_cast<const float*>(X), ldx, k, K, Kpad, dynamic, act_scale, Q,
                                              ldq, rs, M);
    return cudaGetLastError();
  }
  const int C8 = K / 8;
  cudaError_t e;
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t stage = 2 * ((static_cast<size_t>(K) * (f16 ? 2 : 4) + 127) & ~size_t(127));
  if (M >= n_sm && C8 <= 4096 && stage <= 220 * 1024) {
#define DGQ_AQ3(T_, V_)                                                                                         \
  {                                                                                                             \
    auto kern = f16 ? (k_checked ? k_actquant3<T_, V_, true, false> : k_actquant3<T_, V_, true, true>)          \
                    : (k_checked ? k_actquant3<T_, V_, false, false> : k_actquant3<T_, V_, false, true>);       \
    { cudaError_t e_ = dgq_allow_smem(kern, stage); if (e_ != cudaSuccess) return e_; }                       \
    int occ = 1;                                                                                                \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, T_, stage);                                       \
    const int grid = std::min(M, n_sm * std::max(occ, 1));                                                      \
    kern<<<grid, T_, stage, st>>>(X, ldx, seg, seg_stride, k, rk, kone, K, Kpad, dynamic, act_scale, Q, ldq, rs, M);  \
    return cudaGetLastError();                                                                                  \
  }
    if (C8 <= 256) DGQ_AQ3(256, 1)
    if (C8 <= 512) DGQ_AQ3(256, 2)
    if (C8 <= 1024) DGQ_AQ3(256, 4)
    if (C8 <= 2048) DGQ_AQ3(512, 4)
    // one row per CTA fills the smem (114 KB double-buffered at K = 28672 FP16):
    // 32 warps instead of 16 hide the per-row latency (fc2 input 69.7 -> 65.5 us;
    // the same widening slowed 7168-wide rows, tools/k1_time.py)
    DGQ_AQ3(1024, 4)
#undef DGQ_AQ3
  }
#define DGQ_AQ(T_, V_, CL_)                                                                                    \
  e = f16 ? (k_checked ? launch_aq2<T_, V_, CL_, true, false>(X, ldx, seg, seg_stride, k, rk, kone, K, Kpad, dynamic,    \
                                                               act_scale, Q, ldq, rs, M, st)                     \
                       : launch_aq2<T_, V_, CL_, true, true>(X, ldx, seg, seg_stride, k, rk, kone, K, Kpad, dynamic,     \
                                                              act_scale, Q, ldq, rs, M, st))                     \
          : (k_checked ? launch_aq2<T_, V_, CL_, false, false>(X, ldx, seg, seg_stride, k, rk, kone, K, Kpad, dynamic,   \
                                                                act_scale, Q, ldq, rs, M, st)                    \
                       : launch_aq2<T_, V_, CL_, false, true>(X, ldx, seg, seg_stride, k, rk, kone, K, Kpad, dynamic,    \
                                                               act_scale, Q, ldq, rs, M, st))
  if (C8 <= 128) DGQ_AQ(128, 1, 1);
  else if (C8 <= 256) DGQ_AQ(128, 2, 1);
  else if (C8 <= 512) DGQ_AQ(128, 4, 1);
  else if (C8 <= 1024) DGQ_AQ(256, 4, 1);
  else if (C8 <= 2048) DGQ_AQ(256, 4, 2);
  else if (C8 <= 4096) DGQ_AQ(256, 4, 4);
  else if (C8 <= 8192) DGQ_AQ(256, 4, 8);
  else {
    if (f16)
      k_actquant_h_any<256><<<M, 256, 0, st>>>(static_cast<const __half*>(X), ldx, seg, seg_stride, k, K, Kpad,
                                                dynamic, act_scale, Q, ldq, rs, M);
    else
      k_actquant_any<256><<<M, 256, 0, st>>>(static_cast<const float*>(X), ldx, k, K, Kpad, dynamic, act_scale, Q,
                                              ldq, rs, M);
    e = cudaSuccess;
  }
#undef DGQ_AQ
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t dgq_launch_reciprocal(const float* k, float* rk, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_reciprocal<<<(n + 255) / 256, 256, 0, st>>>(k, rk, n);
  return cudaGetLastError();
}

cudaError_t dgq_launch_div_check(const float* x, const float* k, float* fast, float* ieee, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_div_check<<<(n + 255) / 256, 256, 0, st>>>(x, k, fast, ieee, n);
  return cudaGetLastError();
}
