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
#include <cstdint>

#include "kernels.h"
#include "numerics.cuh"

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

// Vector path: K % 4 == 0, 16-B aligned rows, K <= 4*T*V.
template <int T, int V>
__global__ void __launch_bounds__(T) k_actquant_vec(const float* __restrict__ X, size_t ldx,
                                                     const float* __restrict__ kv, int K, int Kpad,
                                                     int dynamic, float act_scale, int8_t* __restrict__ Q,
                                                     size_t ldq, float* __restrict__ rs, int M) {
  __shared__ float red[33];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // let the GEMM start streaming weights
  const int K4 = K >> 2;
  for (int row = blockIdx.x; row < M; row += gridDim.x) {
    const float4* xr = reinterpret_cast<const float4*>(X + static_cast<size_t>(row) * ldx);
    const float4* k4 = reinterpret_cast<const float4*>(kv);
    float4 xv[V];
    float am = 0.0f;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int i = threadIdx.x + v * T;
      if (i < K4) {
        float4 x = __ldcs(xr + i);  // streamed once
        float4 k = __ldg(k4 + i);
        x.x = __fdiv_rn(x.x, k.x);
        x.y = __fdiv_rn(x.y, k.y);
        x.z = __fdiv_rn(x.z, k.z);
        x.w = __fdiv_rn(x.w, k.w);
        xv[v] = x;
        am = fmaxf(am, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
      }
    }
    float s = act_scale;
    if (dynamic) s = dynamic_row_scale(block_max<T>(am, red));
    if (threadIdx.x == 0) rs[row] = s;
    uint32_t* qr = reinterpret_cast<uint32_t*>(Q + static_cast<size_t>(row) * ldq);
    if (scale_is_safe(s)) {
      const float inv = __frcp_rn(s);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int i = threadIdx.x + v * T;
        if (i < K4) {
          const float4 x = xv[v];
          qr[i] = pack4(quant_code_f32(x.x, s, inv), quant_code_f32(x.y, s, inv), quant_code_f32(x.z, s, inv),
                        quant_code_f32(x.w, s, inv));
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int i = threadIdx.x + v * T;
        if (i < K4) {
          const float4 x = xv[v];
          qr[i] = pack4(quant_code_f64(x.x, s), quant_code_f64(x.y, s), quant_code_f64(x.z, s),
                        quant_code_f64(x.w, s));
        }
      }
    }
    for (int i = K4 + threadIdx.x; i < (Kpad >> 2); i += T) qr[i] = 0u;
  }
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

}  // namespace dgqk

using namespace dgqk;

cudaError_t dgq_launch_actquant(const float* X, size_t ldx, const float* k, int K, int Kpad, int dynamic,
                                float act_scale, int8_t* Q, size_t ldq, float* rs, int M, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  const int grid = M;
  const bool vec = (K % 4 == 0) && (ldx % 4 == 0) && (ldq % 4 == 0) && (Kpad % 4 == 0) &&
                   (reinterpret_cast<uintptr_t>(X) % 16 == 0) && (reinterpret_cast<uintptr_t>(k) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(Q) % 4 == 0);
  const int K4 = K / 4;
  if (vec && K4 <= 256 * 1) {
    k_actquant_vec<256, 1><<<grid, 256, 0, st>>>(X, ldx, k, K, Kpad, dynamic, act_scale, Q, ldq, rs, M);
  } else if (vec && K4 <= 256 * 2) {
    k_actquant_vec<256, 2><<<grid, 256, 0, st>>>(X, ldx, k, K, Kpad, dynamic, act_scale, Q, ldq, rs, M);
  } else if (vec && K4 <= 256 * 4) {
    k_actquant_vec<256, 4><<<grid, 256, 0, st>>>(X, ldx, k, K, Kpad, dynamic, act_scale, Q, ldq, rs, M);
  } else if (vec && K4 <= 256 * 8) {
    k_actquant_vec<256, 8><<<grid, 256, 0, st>>>(X, ldx, k, K, Kpad, dynamic, act_scale, Q, ldq, rs, M);
  } else if (vec && K4 <= 512 * 8) {
    k_actquant_vec<512, 8><<<grid, 512, 0, st>>>(X, ldx, k, K, Kpad, dynamic, act_scale, Q, ldq, rs, M);
  } else if (vec && K4 <= 512 * 16) {
    k_actquant_vec<512, 16><<<grid, 512, 0, st>>>(X, ldx, k, K, Kpad, dynamic, act_scale, Q, ldq, rs, M);
  } else {
    k_actquant_any<256><<<grid, 256, 0, st>>>(X, ldx, k, K, Kpad, dynamic, act_scale, Q, ldq, rs, M);
  }
  return cudaGetLastError();
}
