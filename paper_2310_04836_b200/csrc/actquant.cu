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
#include <cstdlib>

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

// ---- vector paths (K % 8 == 0, 16-byte aligned rows) -------------------------
// Elements are handled in 8-channel chunks.  ksm[c] (built once per layer) has
// bit t set when k[8c + t] != 1: only those channels divide (smooth_sparse).
// Chunk c of a row belongs to thread (c mod T) (plus the cluster rank for v2),
// so every warp load or store instruction touches contiguous memory.

// Bits 8v..8v+7: the k != 1 mask of the thread's v-th chunk (V <= 4).  Built
// once per kernel with all V loads in flight together.
template <int T, int V>
__device__ __forceinline__ uint32_t special_masks(const uint8_t* __restrict__ ksm, int cbase, int C8) {
  static_assert(V <= 4, "one byte per chunk in a 32-bit word");
  if (!ksm) return 0xFFFFFFFFu;  // no layer mask: every channel divides
  uint32_t m = 0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c = cbase + v * T;
    if (c < C8) m |= static_cast<uint32_t>(__ldg(ksm + c)) << (8 * v);
  }
  return m;
}

// 8 input values of chunk c from a row in registers / shared memory as FP32
template <bool kF16>
__device__ __forceinline__ void unpack8(const uint4* raw, float (&x)[8]) {
  if constexpr (kF16) {
    const __half2* h2 = reinterpret_cast<const __half2*>(raw);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float2 f = __half22float2(h2[t]);
      x[2 * t] = f.x;
      x[2 * t + 1] = f.y;
    }
  } else {
    const float* f = reinterpret_cast<const float*>(raw);
#pragma unroll
    for (int t = 0; t < 8; ++t) x[t] = f[t];
  }
}

// codes of one chunk: the fast exact path for normal scales, doubles otherwise
static __device__ __noinline__ uint2 chunk_codes_f64(float4 a, float4 b, float s) {
  return make_uint2(pack4(quant_code_f64(a.x, s), quant_code_f64(a.y, s), quant_code_f64(a.z, s), quant_code_f64(a.w, s)),
                    pack4(quant_code_f64(b.x, s), quant_code_f64(b.y, s), quant_code_f64(b.z, s), quant_code_f64(b.w, s)));
}
template <bool kStatic>
__device__ __forceinline__ uint2 chunk_codes(const float (&xp)[8], float s, float inv, bool safe) {
  if (safe) return quant_chunk<kStatic>(xp, s, inv);
  return chunk_codes_f64(make_float4(xp[0], xp[1], xp[2], xp[3]), make_float4(xp[4], xp[5], xp[6], xp[7]), s);
}

// ---- K1 v2 (small M): one row per CL-CTA cluster, loads front-loaded ---------
// every thread first issues all of its V 16-B (f16) or 32-B (f32) loads, then
// smooths, reduces the row absmax (block, then over the cluster through DSMEM)
// and quantises from registers.
template <int T, int V, int CL, bool kF16, bool kDyn>
__global__ void __launch_bounds__(T) k_actquant2(const void* __restrict__ Xv, size_t ldx, int seg, size_t seg_stride,
                                                  const float* __restrict__ kv, const float* __restrict__ rkv,
                                                  const uint8_t* __restrict__ ksm, int K, int Kpad,
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
  const uint32_t sm = special_masks<T, V>(ksm, cbase, C8);
  // launched with programmatic stream serialisation: everything above read
  // layer constants only; X, Q and rs belong to the neighbouring kernels
  asm volatile("griddepcontrol.wait;" ::: "memory");
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
      unpack8<kF16>(raw[v], xv[v]);
      smooth_sparse(xv[v], (sm >> (8 * v)) & 0xFFu, kv, rkv, c * 8);
#pragma unroll
      for (int t = 0; t < 8; ++t) am = fmaxf(am, fabsf(xv[v][t]));
    }
  }
  float s = act_scale;
  if constexpr (kDyn) {
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
    if (c < C8) qr[c] = chunk_codes<!kDyn>(xv[v], s, inv, safe);
  }
  if (part == 0)
    for (int c = C8 + threadIdx.x; c < (Kpad >> 3); c += T) qr[c] = make_uint2(0u, 0u);
}

// ---- K1 v3 (large M): persistent CTAs, whole rows staged in shared memory by
// 1-D TMA bulk copies through a ring of `depth` row buffers (one mbarrier
// each).  Both passes read the row from shared memory (nothing row-sized is
// held in registers), so a CTA of T threads covers a row in V = K / (8 T)
// chunks per thread and the per-row fixed costs (the waits, two barriers, the
// reduction) are spread over many chunks.
//
// Per row:
//   1. the channels with k != 1 (compute_smooth leaves k == 1 on all but the
//      top percentile; at most T of them — kSparse) are owned by threads of
//      their own: thread i < nspec reads x[spec[i]], forms x' = x / k with k
//      and RN(1/k) in registers, and overwrites the staged value with 0;
//   2. barrier; absmax over the row (FP16 rows in packed form: |x| of a
//      binary16 value orders like its magnitude bits, so an unsigned 16-bit max
//      of the sign-cleared halves is the exact maximum; no conversion), the
//      specials' |x'| folded in, warp maxima to a per-parity slot;
//   3. barrier; every warp reduces the slots itself; the buffer of the
//      PREVIOUS row (its second pass retired before this barrier) is refilled;
//   4. codes from the staged row (a special's lane reads 0 -> code 0); the
//      special thread's own code byte is written after the next row's barrier
//      (or the final one), which orders it after the owner's 8-byte store.
// Without kSparse (a layer with more than T channels k != 1, e.g. random-k
// tests) the masked lanes divide inline instead (ksm bit masks).
constexpr int kRing = 8;
// barrier of the T compute threads of k_actquant3 (its producer warp does not take part)
template <int T>
__device__ __forceinline__ void compute_bar(int grp) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(T) : "memory");
}
// kExact: the launcher guarantees C8 == T * V (every thread owns exactly V
// chunks), so the per-chunk `c < C8` guards and their branches compile away.
// G > 1: G independent groups of T compute threads per CTA, each taking every
// G-th row of the CTA, each with its own named barrier — one group's barrier
// waits overlap the other's passes.
template <int T, int V, bool kF16, bool kDyn, bool kSparse, bool kExact = false, int G = 1>
__global__ void __launch_bounds__(G * T + 32, G * T >= 512 ? 1 : 2) k_actquant3(const void* __restrict__ Xv, size_t ldx, int seg, size_t seg_stride,
                                                  const float* __restrict__ kv, const float* __restrict__ rkv,
                                                  const uint8_t* __restrict__ ksm, const int* __restrict__ spec,
                                                  int nspec, int K, int Kpad, float act_scale,
                                                  int8_t* __restrict__ Q, size_t ldq, float* __restrict__ rs, int M,
                                                  int depth) {
  extern __shared__ __align__(128) uint8_t sbuf[];
  __shared__ __align__(8) uint64_t full[kRing];
  __shared__ __align__(8) uint64_t empty[kRing];  // the T compute threads are done with a buffer (one arrive per warp)
  __shared__ float red_all[G][2][32];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int kEsz = kF16 ? 2 : 4;
  constexpr int kW = T / 32;
  const uint32_t rowbytes = static_cast<uint32_t>(K) * kEsz;
  const uint32_t bufstride = (rowbytes + 127u) & ~127u;
  const int C8 = K >> 3;
  const int nseg = K / seg;
  auto issue = [&](int r, int b) {  // the producer lane only
    dgqk::mbar_arrive_expect_tx(&full[b], rowbytes);
    for (int sg = 0; sg < nseg; ++sg) {
      const uint8_t* src = static_cast<const uint8_t*>(Xv) +
                           (static_cast<size_t>(sg) * seg_stride + static_cast<size_t>(r) * ldx) * kEsz;
      dgqk::bulk_load(sbuf + b * bufstride + static_cast<size_t>(sg) * seg * kEsz, src,
                      static_cast<uint32_t>(seg) * kEsz, &full[b]);
    }
  };
  // launched with programmatic stream serialisation: X, Q and rs belong to the
  // neighbouring kernels, so every thread waits for them before its first access
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int b = 0; b < depth; ++b) {
      dgqk::mbar_init(&full[b], 1);
      dgqk::mbar_init(&empty[b], kW);
    }
    dgqk::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x >= G * T) {
    // Producer warp: one bulk copy per row into the ring; a row's buffer is
    // refilled as soon as every compute warp has finished with it.  A TMA
    // issue holds its lane for ~700 cycles (tools/l2_stream.cu): issued by a
    // compute thread it delayed that warp's share of every row.
    if (threadIdx.x == G * T) {
      for (int row = blockIdx.x, i = 0; row < M; row += gridDim.x, ++i) {
        const int bb = i % depth;
        if (i >= depth) dgqk::mbar_wait(&empty[bb], ((i / depth) - 1) & 1);
        issue(row, bb);
      }
    }
    return;
  }
  const int grp = static_cast<int>(threadIdx.x) / T;  // this thread's row group
  const int tid = static_cast<int>(threadIdx.x) % T;  // index inside the group
  float(&red)[2][32] = red_all[grp];
  const bool special = kSparse && tid < nspec;
  int sj = 0;
  float sk = 1.0f, srk = 1.0f;
  if (special) {
    sj = __ldg(spec + tid);
    sk = __ldg(kv + sj);
    srk = __ldg(rkv + sj);
  }
  int8_t* pend = nullptr;  // the special's code byte of the previous row
  int pcode = 0;
  const int lane = threadIdx.x & 31, warp = tid >> 5;
  for (int row = blockIdx.x + grp * static_cast<int>(gridDim.x), it = 0, i = grp; row < M;
       row += G * static_cast<int>(gridDim.x), ++it, i += G) {
    const int b = i % depth;  // row i of this CTA sits in buffer i % depth
    const uint32_t phase = (i / depth) & 1;
    dgqk::mbar_wait(&full[b], phase);
    uint8_t* buf = sbuf + b * bufstride;
    float am = 0.0f, xs = 0.0f;
    if constexpr (kSparse) {
      if (special) {
        if constexpr (kF16) {
          __half* p = reinterpret_cast<__half*>(buf) + sj;
          xs = div_k(__half2float(*p), sk, srk);
          *p = __float2half_rn(0.0f);
        } else {
          float* p = reinterpret_cast<float*>(buf) + sj;
          xs = div_k(*p, sk, srk);
          *p = 0.0f;
        }
        am = fabsf(xs);
      }
      compute_bar<T>(grp);  // specials zeroed in the staged row
    }
    if constexpr (kDyn) {
      uint32_t am16 = 0u;
      uint4 r16[kF16 && kSparse ? V : 1];  // all of the thread's FP16 chunks loaded before any use
      if constexpr (kF16 && kSparse) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int c = tid + v * T;
          r16[v] = (kExact || c < C8) ? *reinterpret_cast<const uint4*>(buf + c * 16) : make_uint4(0u, 0u, 0u, 0u);
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int c = tid + v * T;
        if (kExact || c < C8) {
          if constexpr (kF16) {
            const uint4 raw = kSparse ? r16[kSparse ? v : 0] : *reinterpret_cast<const uint4*>(buf + c * 16);
            if (kSparse || (ksm && !__ldg(ksm + c))) {
              am16 = __vmaxu2(am16, raw.x & 0x7FFF7FFFu);
              am16 = __vmaxu2(am16, raw.y & 0x7FFF7FFFu);
              am16 = __vmaxu2(am16, raw.z & 0x7FFF7FFFu);
              am16 = __vmaxu2(am16, raw.w & 0x7FFF7FFFu);
            } else {
              float x[8];
              unpack8<true>(&raw, x);
              smooth_sparse(x, ksm ? __ldg(ksm + c) : 0xFFu, kv, rkv, c * 8);
#pragma unroll
              for (int t = 0; t < 8; ++t) am = fmaxf(am, fabsf(x[t]));
            }
          } else {
            uint4 raw[2];
            raw[0] = *reinterpret_cast<const uint4*>(buf + c * 32);
            raw[1] = *reinterpret_cast<const uint4*>(buf + c * 32 + 16);
            float x[8];
            unpack8<false>(raw, x);
            if constexpr (!kSparse) smooth_sparse(x, ksm ? __ldg(ksm + c) : 0xFFu, kv, rkv, c * 8);
#pragma unroll
            for (int t = 0; t < 8; ++t) am = fmaxf(am, fabsf(x[t]));
          }
        }
      }
      if constexpr (kF16) {
        const float2 m2 = __half22float2(*reinterpret_cast<const __half2*>(&am16));
        am = fmaxf(am, fmaxf(m2.x, m2.y));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
      if (lane == 0) red[it & 1][warp] = am;
    }
    compute_bar<T>(grp);  // warp maxima published; the previous row's stores retired
    if (kSparse && pend) *pend = static_cast<int8_t>(pcode);
    float s = act_scale;
    if constexpr (kDyn) {
      float w = lane < kW ? red[it & 1][lane] : 0.0f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) w = fmaxf(w, __shfl_xor_sync(0xffffffffu, w, o));
      s = dynamic_row_scale(w);
    }
    if (tid == 0) rs[row] = s;
    int8_t* qrow = Q + static_cast<size_t>(row) * ldq;
    uint2* qr = reinterpret_cast<uint2*>(qrow);
    const bool safe = scale_is_safe(s);
    const float inv = __frcp_rn(s);
    // pass 2 (FP16 rows in groups of 4 chunks: the group's shared-memory loads
    // are all issued before the first conversion)
    constexpr int kG = kF16 ? 4 : 1;
#pragma unroll
    for (int v0 = 0; v0 < V; v0 += kG) {
      uint4 raw[kG][kF16 ? 1 : 2];
#pragma unroll
      for (int v = v0; v < v0 + kG && v < V; ++v) {
        const int c = tid + v * T;
        if (kExact || c < C8) {
          raw[v - v0][0] = *reinterpret_cast<const uint4*>(buf + c * 8 * kEsz);
          if constexpr (!kF16) raw[v - v0][1] = *reinterpret_cast<const uint4*>(buf + c * 32 + 16);
        }
      }
#pragma unroll
      for (int v = v0; v < v0 + kG && v < V; ++v) {
        const int c = tid + v * T;
        if (kExact || c < C8) {
          float x[8];
          unpack8<kF16>(raw[v - v0], x);
          if constexpr (!kSparse) smooth_sparse(x, ksm ? __ldg(ksm + c) : 0xFFu, kv, rkv, c * 8);
          qr[c] = chunk_codes<!kDyn>(x, s, inv, safe);
        }
      }
    }
    for (int c = C8 + tid; c < (Kpad >> 3); c += T) qr[c] = make_uint2(0u, 0u);
    if (special) {
      pend = qrow + sj;
      pcode = safe ? quant_code_f32(xs, s, inv) : quant_code_f64(xs, s);
    }
    __syncwarp();
    if (lane == 0) dgqk::mbar_arrive(&empty[b]);  // this warp's reads of the staged row are done
  }
  if constexpr (kSparse) {
    compute_bar<T>(grp);
    if (pend) *pend = static_cast<int8_t>(pcode);
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
// a launch with programmatic stream serialisation (the kernel griddepcontrol.waits
// before touching X / Q / rs, so its launch and prologue overlap the previous kernel)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int threads, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(threads));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int T, int V, int CL, bool F16>
cudaError_t launch_aq2(const void* X, size_t ldx, int seg, size_t seg_stride, const float* k, const float* rk,
                       const uint8_t* ksm, int K, int Kpad, int dynamic, float act_scale, int8_t* Q, size_t ldq,
                       float* rs, int M, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(M) * CL);
  cfg.blockDim = dim3(T);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = CL;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = CL > 1 ? 2 : 1;
  if (dynamic)
    return cudaLaunchKernelEx(&cfg, k_actquant2<T, V, CL, F16, true>, X, ldx, seg, seg_stride, k, rk, ksm, K, Kpad,
                              act_scale, Q, ldq, rs, M);
  return cudaLaunchKernelEx(&cfg, k_actquant2<T, V, CL, F16, false>, X, ldx, seg, seg_stride, k, rk, ksm, K, Kpad,
                            act_scale, Q, ldq, rs, M);
}
}  // namespace

// tools: DGQ_K1_DEPTH=3..8 row buffers and DGQ_K1_T=128|256|512 threads per
// K1 v3 CTA (A/B runs; 0 = the planner's choice)
static int aq_depth() {
  static const int v = [] {
    const char* e = getenv("DGQ_K1_DEPTH");
    const int d = e ? atoi(e) : 0;
    return d <= 0 ? 0 : (d < 3 ? 3 : (d > kRing ? kRing : d));
  }();
  return v;
}
// tools: DGQ_K1_DEC=0 keeps one CTA per row for few-row calls (A/B runs)
static int aq_decode_clusters() {
  static const int v = [] {
    const char* e = getenv("DGQ_K1_DEC");
    return e ? atoi(e) : 1;
  }();
  return v;
}
// row groups per persistent K1 CTA on the exact shapes: two groups, each on
// every other row with its own barrier, overlap one group's barrier waits with
// the other's passes (tools/k1_ab.py, 2048 rows: 28672 FP16 42.4 -> 36.0 us,
// 7168 FP32 18.4 -> 15.2 us, 7168 FP16 13.0 -> 12.5 us).  DGQ_K1_G=1: one
// group (A/B)
static int aq_groups() {
  static const int v = [] {
    const char* e = getenv("DGQ_K1_G");
    return e ? atoi(e) : 2;
  }();
  return v;
}
static int aq_threads() {
  static const int v = [] {
    const char* e = getenv("DGQ_K1_T");
    const int t = e ? atoi(e) : 0;
    return (t == 128 || t == 256 || t == 512) ? t : 0;
  }();
  return v;
}

cudaError_t dgq_launch_actquant2(const void* X, bool f16, size_t ldx, int seg, size_t seg_stride, const float* k,
                                 const float* rk, int K, int Kpad, int dynamic, float act_scale, int8_t* Q, size_t ldq,
                                 float* rs, int M, cudaStream_t st, const uint8_t* ksm, const int* spec, int nspec) {
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
  const size_t bufstride = (static_cast<size_t>(K) * (f16 ? 2 : 4) + 127) & ~size_t(127);
  if (M >= n_sm && C8 <= 16 * 512 && 3 * bufstride <= 220 * 1024) {
    // persistent CTAs of T threads, V <= 16 chunks per thread, `depth` row buffers
    int T = aq_threads();
    if (!T) {
      T = C8 <= 8 * 256 ? 256 : 512;  // measured (tools/k1_ab.py): <= 8 chunks per thread
      // few special channels (the sparse path) and a row of 7 or 4 chunks per
      // thread at T = 128: the exact kernel (dense-k rows stay at T = 256)
      if ((C8 == 7 * 128 || C8 == 4 * 128) && ksm && nspec <= 128) T = 128;
    }
    while ((C8 + T - 1) / T > 16) T *= 2;
    const int need = (C8 + T - 1) / T;
    int depth = aq_depth();
    if (!depth) depth = 3;
    while (depth > 3 && depth * bufstride > 220 * 1024) --depth;
    const size_t smem = depth * bufstride;
#define DGQ_AQ3_K(T_, V_, F_, D_, S_, G_)                                                                      \
  {                                                                                                             \
    auto kern = k_actquant3<T_, (V_ < 0 ? -V_ : V_), F_, D_, S_, (V_ < 0), G_>;                                \
    { cudaError_t e_ = dgq_allow_smem(kern, smem); if (e_ != cudaSuccess) return e_; }                        \
    int occ = 1;                                                                                                \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G_ * T_ + 32, smem);                              \
    const int grid = std::min(M, n_sm * std::max(occ, 1));                                                      \
    return launch_pdl(kern, grid, G_ * T_ + 32, smem, st, X, ldx, seg, seg_stride, k, rk, ksm, spec, nspec, K,  \
                      Kpad, act_scale, Q, ldq, rs, M, depth);                                                   \
  }
#define DGQ_AQ3_S(T_, V_, F_, D_, G_)                                                                           \
  {                                                                                                             \
    if (ksm && nspec <= T_) DGQ_AQ3_K(T_, V_, F_, D_, true, G_)                                                 \
    DGQ_AQ3_K(T_, V_, F_, D_, false, G_)                                                                        \
  }
#define DGQ_AQ3(T_, V_, G_)                                                                                     \
  {                                                                                                             \
    if (f16) {                                                                                                  \
      if (dynamic) DGQ_AQ3_S(T_, V_, true, true, G_)                                                            \
      DGQ_AQ3_S(T_, V_, true, false, G_)                                                                        \
    }                                                                                                           \
    if (dynamic) DGQ_AQ3_S(T_, V_, false, true, G_)                                                             \
    DGQ_AQ3_S(T_, V_, false, false, G_)                                                                         \
  }
#define DGQ_AQ3_V(T_)                                                                                           \
  {                                                                                                             \
    if (need <= 4) DGQ_AQ3(T_, 4, 1)                                                                            \
    if (need <= 8) DGQ_AQ3(T_, 8, 1)                                                                            \
    if (need <= 12) DGQ_AQ3(T_, 12, 1)                                                                          \
    DGQ_AQ3(T_, 16, 1)                                                                                          \
  }
    // exact shapes (C8 == T * V): no per-chunk guards, no idle chunk slots
    // (tools/k1_ab.py, 2048 rows, smoothed k: K = 28672 f16 50.7 -> 43.8 us at
    // T = 512; K = 7168 f16 16.3 -> 14.4 us, f32 20.2 -> 19.6 us at T = 128)
    // and two independent row groups per CTA (aq_groups)
    const bool g2 = aq_groups() == 2;
    if (T == 128 && C8 == 7 * 128) { if (g2) DGQ_AQ3(128, -7, 2) DGQ_AQ3(128, -7, 1) }
    if (T == 128 && C8 == 4 * 128) { if (g2) DGQ_AQ3(128, -4, 2) DGQ_AQ3(128, -4, 1) }
    if (T == 256 && C8 == 4 * 256) { if (g2) DGQ_AQ3(256, -4, 2) DGQ_AQ3(256, -4, 1) }
    if (T == 512 && C8 == 7 * 512) { if (g2) DGQ_AQ3(256, -14, 2) DGQ_AQ3(512, -7, 1) }
    if (T == 128) DGQ_AQ3_V(128)
    if (T == 256) DGQ_AQ3_V(256)
    DGQ_AQ3_V(512)
#undef DGQ_AQ3_V
#undef DGQ_AQ3
#undef DGQ_AQ3_S
#undef DGQ_AQ3_K
  }
#define DGQ_AQ(T_, V_, CL_)                                                                                   \
  e = f16 ? launch_aq2<T_, V_, CL_, true>(X, ldx, seg, seg_stride, k, rk, ksm, K, Kpad, dynamic, act_scale, Q, ldq, \
                                           rs, M, st)                                                            \
          : launch_aq2<T_, V_, CL_, false>(X, ldx, seg, seg_stride, k, rk, ksm, K, Kpad, dynamic, act_scale, Q,     \
                                            ldq, rs, M, st)
  // few rows (decode): spread each row over a cluster so every thread owns one
  // or two chunks — the row's loads are all in flight at once (latency-bound)
  if (M <= 16 && aq_decode_clusters() && C8 > 256 && C8 <= 4096) {
    if (C8 <= 512) DGQ_AQ(256, 1, 2);
    else if (C8 <= 1024) DGQ_AQ(256, 1, 4);
    else if (C8 <= 2048) DGQ_AQ(256, 1, 8);
    else DGQ_AQ(256, 2, 8);
  }
  else if (C8 <= 128) DGQ_AQ(128, 1, 1);
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
