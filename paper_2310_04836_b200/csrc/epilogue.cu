// K4 standalone epilogue (drop-in for proj/src/kernel.cpp:89-116) and the
// accumulator audit behind int8_gemm's max_abs_acc (proj/src/kernel.cpp:73-77).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "kernels.h"
#include "numerics.cuh"

namespace dgqk {

__global__ void k_epilogue(const int32_t* __restrict__ acc, size_t lda, const float* __restrict__ rs,
                           const float* __restrict__ s1, const float* __restrict__ bias, int M, int N, int fp16_mode,
                           int out_f16, void* __restrict__ y, size_t ldy) {
  const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<size_t>(M) * N) return;
  const int r = static_cast<int>(idx / N), c = static_cast<int>(idx % N);
  const int32_t a = acc[static_cast<size_t>(r) * lda + c];
  float v = fp16_mode ? epilogue_f16mode(a, rs[r], s1[c]) : epilogue_f32(a, rs[r], s1[c]);
  if (bias) v = __fadd_rn(v, bias[c]);
  if (out_f16)
    static_cast<__half*>(y)[static_cast<size_t>(r) * ldy + c] = fp16_ref(v);
  else
    static_cast<float*>(y)[static_cast<size_t>(r) * ldy + c] = v;
}

// One thread per (r, c) walks k in order, exactly like the reference's scalar
// loop: the running sum (|sum| < 2^31 by the h*127^2 < 2^31 precondition) and
// its largest magnitude.  Audit only — the tensor-core GEMM is the product.
__global__ void k_audit(const int8_t* __restrict__ Xq, size_t ldx, const int8_t* __restrict__ W, size_t ldw, int M,
                        int K, int N, unsigned long long* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  int32_t best = 0;
  for (int r = blockIdx.y; r < M; r += gridDim.y) {  // any M: rows beyond grid.y loop
    if (c >= N) break;
    const int8_t* x = Xq + static_cast<size_t>(r) * ldx;
    int32_t s = 0;
    for (int i = 0; i < K; ++i) {
      s += static_cast<int32_t>(x[i]) * static_cast<int32_t>(W[static_cast<size_t>(i) * ldw + c]);
      best = max(best, abs(s));
    }
  }
  // warp max then one atomic
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(best));
}

}  // namespace dgqk

using namespace dgqk;

cudaError_t dgq_launch_epilogue(const int32_t* acc, size_t lda, const float* rs, const float* s1, const float* bias,
                                int M, int N, int fp16_mode, int out_f16, void* y, size_t ldy, cudaStream_t st) {
  const size_t total = static_cast<size_t>(M) * N;
  if (!total) return cudaSuccess;
  k_epilogue<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(acc, lda, rs, s1, bias, M, N, fp16_mode,
                                                                          out_f16, y, ldy);
  return cudaGetLastError();
}

cudaError_t dgq_launch_audit(const int8_t* Xq, size_t ldx, const int8_t* W, size_t ldw, int M, int K, int N,
                             unsigned long long* out, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  dim3 grid((N + 127) / 128, M < 65535 ? M : 65535);
  k_audit<<<grid, 128, 0, st>>>(Xq, ldx, W, ldw, M, K, N, out);
  return cudaGetLastError();
}
