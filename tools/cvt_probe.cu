// Conversion-pipe throughput probe for the K5p epilogue (int32 accumulator ->
// FP32 -> scales -> FP16).  Each variant converts 16 independent values per
// thread per iteration; reports SM cycles per value per SM at 8 warps / CTA
// (the epilogue's warp count) and 32 warps / CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_bin/cvt_probe tools/cvt_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

template <int V>
__global__ void k(const int* in, uint32_t* out, int iters, unsigned long long* cyc) {
  int x[16];
  for (int i = 0; i < 16; ++i) x[i] = in[(threadIdx.x * 16 + i) & 1023];
  uint32_t accum = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float y[16];
    if (V == 0) {  // I2F
#pragma unroll
      for (int i = 0; i < 16; ++i) y[i] = __int2float_rn(x[i]);
    } else if (V == 1) {  // exact split: fma(float(hi + 1.5*2^23), 2^16, -C) + float(lo + 2^23)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float a = __int_as_float((x[i] >> 16) + 0x4B400000);
        const float b = __int_as_float((x[i] & 0xFFFF) | 0x4B000000);
        y[i] = __fadd_rn(__fmaf_rn(a, 65536.0f, -824642109440.0f), b);
      }
    } else if (V == 2) {  // F2FP pack only (from int bits reinterpreted)
#pragma unroll
      for (int i = 0; i < 16; ++i) y[i] = __int_as_float(x[i]);
    } else if (V == 3) {  // I2F + 2 FMUL + F2FP (the current epilogue math)
#pragma unroll
      for (int i = 0; i < 16; ++i) y[i] = __fmul_rn(__fmul_rn(__int2float_rn(x[i]), 1.5f), 0.75f);
    } else {  // split + 2 FMUL + F2FP
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float a = __int_as_float((x[i] >> 16) + 0x4B400000);
        const float b = __int_as_float((x[i] & 0xFFFF) | 0x4B000000);
        y[i] = __fmul_rn(__fmul_rn(__fadd_rn(__fmaf_rn(a, 65536.0f, -824642109440.0f), b), 1.5f), 0.75f);
      }
    }
    if (V >= 2) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const __half2 h = __floats2half2_rn(y[i], y[i + 1]);
        accum ^= *reinterpret_cast<const uint32_t*>(&h);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) accum ^= __float_as_uint(y[i]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] += it;
  }
  const unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = accum;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
static void run(const char* name, int* in, uint32_t* out, unsigned long long* cyc, int threads) {
  const int iters = 2000;
  k<V><<<148, threads>>>(in, out, iters, cyc);
  k<V><<<148, threads>>>(in, out, iters, cyc);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += h[i];
  m /= 148;
  const double vals = static_cast<double>(iters) * 16 * threads;
  printf("%-28s threads %4d: %.3f cycles per value per SM (%.1f values/clk/SM)\n", name, threads, m / vals, vals / m);
}

int main() {
  int* in;
  uint32_t* out;
  unsigned long long* cyc;
  cudaMalloc(&in, 4096 * 4);
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  int h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = (i * 2654435761u) >> 4;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  // exactness of the split conversion over edge values
  for (int threads : {256, 1024}) {
    run<0>("I2F", in, out, cyc, threads);
    run<1>("split int->float", in, out, cyc, threads);
    run<2>("F2FP pack", in, out, cyc, threads);
    run<3>("I2F+2FMUL+F2FP", in, out, cyc, threads);
    run<4>("split+2FMUL+F2FP", in, out, cyc, threads);
  }
  return 0;
}
