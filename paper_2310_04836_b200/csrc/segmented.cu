// Comparators and the f32 weight view that sit beside the hot path:
//  * k_segmented — the group-wise ("segmented") semantics of
//    segmented_gemm_reference (proj/src/kernel.cpp:118-142): per group an exact
//    integer partial sum of x * (code - ZP), scaled by S2 in 64-bit integer
//    arithmetic, converted to f32 and accumulated in f32 in group order; then
//    ((fsum * rs) * s1).  This is the computation DGQ's single INT8 GEMM
//    replaces, kept exact so it can serve as the reference's
//    comparator on the GPU.
//  * k_dequant_f32 — dequantize_to_f32 (proj/src/format.cpp:143-154):
//    float(double(s1[c]) * double(W_s8[i, c])).
#include <cuda_runtime.h>
#include <cstdint>

#include "kernels.h"

namespace dgqk {

// One thread per output column c of one token row r (blockIdx.y): the group
// loop runs in ascending order so the f32 accumulation matches the reference
// bit for bit.  The token row is staged in shared memory; codes are read as
// bytes of the N-packed reference layout (coalesced across the warp).
__global__ void k_segmented(const int8_t* __restrict__ Xq, size_t ldx, const float* __restrict__ rs,
                            const uint8_t* __restrict__ codes, const int8_t* __restrict__ s2,
                            const uint8_t* __restrict__ zp, const float* __restrict__ s1, int h, int o, int g,
                            float* __restrict__ y, size_t ldy) {
  extern __shared__ int8_t s_x[];
  const int r = blockIdx.y;
  for (int i = threadIdx.x; i < h; i += blockDim.x) s_x[i] = Xq[static_cast<size_t>(r) * ldx + i];
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= o) return;
  const size_t half_o = static_cast<size_t>(o) / 2;
  const int shift = (c & 1) * 4;
  const int ng = h / g;
  float fsum = 0.0f;
  for (int kg = 0; kg < ng; ++kg) {
    const int z = (zp[static_cast<size_t>(kg) * half_o + (c >> 1)] >> shift) & 0xF;
    int32_t partial = 0;  // |partial| <= g * 127 * 15 < 2^31 for any g the layer admits
    const uint8_t* crow = codes + static_cast<size_t>(kg) * g * half_o + (c >> 1);
    for (int j = 0; j < g; ++j) {
      const int code = (crow[static_cast<size_t>(j) * half_o] >> shift) & 0xF;
      partial += static_cast<int32_t>(s_x[kg * g + j]) * (code - z);
    }
    const long long scaled = static_cast<long long>(s2[static_cast<size_t>(kg) * o + c]) * partial;
    fsum = __fadd_rn(fsum, __ll2float_rn(scaled));
  }
  y[static_cast<size_t>(r) * ldy + c] = __fmul_rn(__fmul_rn(fsum, rs[r]), s1[c]);
}

__global__ void k_dequant_f32(const int8_t* __restrict__ w, const float* __restrict__ s1, int h, int o,
                              float* __restrict__ out) {
  const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<size_t>(h) * o) return;
  const int c = static_cast<int>(idx % o);
  out[idx] = __double2float_rn(__dmul_rn(static_cast<double>(s1[c]), static_cast<double>(w[idx])));
}

}  // namespace dgqk

using namespace dgqk;

cudaError_t dgq_launch_segmented(const int8_t* Xq, size_t ldx, const float* rs, const uint8_t* codes,
                                 const int8_t* s2, const uint8_t* zp, const float* s1, int M, int h, int o, int g,
                                 float* y, size_t ldy, cudaStream_t st) {
  if (M <= 0 || o <= 0) return cudaSuccess;
  if (h > 48 * 1024) {
    cudaError_t e = dgq_allow_smem(k_segmented, static_cast<size_t>(h));
    if (e != cudaSuccess) return e;
  }
  dim3 grid((o + 127) / 128, M);
  k_segmented<<<grid, 128, h, st>>>(Xq, ldx, rs, codes, s2, zp, s1, h, o, g, y, ldy);
  return cudaGetLastError();
}

cudaError_t dgq_launch_dequant_f32(const int8_t* w, const float* s1, int h, int o, float* out, cudaStream_t st) {
  const size_t total = static_cast<size_t>(h) * o;
  if (!total) return cudaSuccess;
  k_dequant_f32<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(w, s1, h, o, out);
  return cudaGetLastError();
}
