// Calibration statistics on the GPU: the two HBM-bound passes
// over the calibration activations that produce a layer's smoothing vector k
// and static activation scale (proj/src/pipeline.cpp:352-360):
//   z[c]     = max_r |X[r, c]|                      channel_maxima, proj/src/smoothing.cpp:9-24
//   absmax   = max_{r,c} |X[r, c] / k[c]|           static_act_scale over smooth_activations,
//                                                   proj/src/pipeline.cpp:96-101, smoothing.cpp:52-63
// Maxima of non-negative floats are exact in any order, so both equal the
// reference bit for bit (the IEEE division is __fdiv_rn).  The percentile
// selection of compute_smooth (an nth_element over h values) runs on the host.
#include <cuda_runtime.h>
#include <cstdint>

#include "kernels.h"

namespace dgqk {

// grid (ceil(h / 256), row slices); atomicMax on the bit patterns of
// non-negative floats orders like the floats themselves
__global__ void k_colmax(const float* __restrict__ X, size_t ldx, int rows, int h, unsigned* __restrict__ z) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= h) return;
  float m = 0.0f;
  for (int r = blockIdx.y; r < rows; r += gridDim.y) m = fmaxf(m, fabsf(X[static_cast<size_t>(r) * ldx + c]));
  atomicMax(z + c, __float_as_uint(m));
}

__global__ void k_smooth_absmax(const float* __restrict__ X, size_t ldx, int rows, int h, const float* __restrict__ k,
                                unsigned* __restrict__ out) {
  float m = 0.0f;
  const size_t n = static_cast<size_t>(rows) * h;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / h, c = i - r * h;
    m = fmaxf(m, fabsf(__fdiv_rn(X[r * ldx + c], k[c])));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

}  // namespace dgqk

cudaError_t dgq_launch_colmax(const float* X, size_t ldx, int rows, int h, unsigned* z, cudaStream_t st) {
  if (rows <= 0 || h <= 0) return cudaSuccess;
  const int slices = rows < 64 ? rows : 64;
  dgqk::k_colmax<<<dim3((h + 255) / 256, slices), 256, 0, st>>>(X, ldx, rows, h, z);
  return cudaGetLastError();
}

cudaError_t dgq_launch_smooth_absmax(const float* X, size_t ldx, int rows, int h, const float* k, unsigned* out,
                                     cudaStream_t st) {
  if (rows <= 0 || h <= 0) return cudaSuccess;
  const size_t n = static_cast<size_t>(rows) * h;
  const int blocks = static_cast<int>(n / 256 + 1 < 148 * 8 ? n / 256 + 1 : 148 * 8);
  dgqk::k_smooth_absmax<<<blocks, 256, 0, st>>>(X, ldx, rows, h, k, out);
  return cudaGetLastError();
}
