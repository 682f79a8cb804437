// Semantics probe: mbarrier.test_wait / try_wait .parity on a fresh barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -o mbar_probe tools/mbar_probe.cu
#include <cstdint>
#include <cstdio>
__global__ void k(int* out) {
  __shared__ uint64_t bar;
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
  asm volatile("fence.mbarrier_init.release.cluster;");
  for (int par = 0; par < 2; ++par) {
    uint32_t ok1, ok2;
    asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok1) : "r"(a), "r"(par) : "memory");
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000; selp.u32 %0,1,0,p;}"
                 : "=r"(ok2) : "r"(a), "r"(par) : "memory");
    out[par * 2] = ok1;
    out[par * 2 + 1] = ok2;
  }
}
int main() {
  int* d;
  cudaMalloc(&d, 16);
  k<<<1, 1>>>(d);
  int h[4];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("fresh barrier: parity0 test=%d try=%d | parity1 test=%d try=%d\n", h[0], h[1], h[2], h[3]);
}
