// Microbenchmark: how fast can one persistent CTA per SM stream a contiguous
// HBM range into shared memory?  Variants: 1-D bulk copies (cp.async.bulk) of
// various sizes / depths, and plain LDG.128 by all warps.  Each SM reads an
// equal contiguous slice of a 1 GiB buffer (weights-like, no reuse).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench tools/stream_bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) { while (!mbar_try_wait(bar, parity)) {} }
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

// producer lane issues `per` copies of `chunk` bytes per stage; consumer warp
// touches one word per stage and releases it.
__global__ void k_bulk(const uint8_t* buf, size_t per_cta, int chunk, int stages, int per, int hint, unsigned* sink,
                       int consumers) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(stages) * chunk * per);
  uint64_t* empty = full + stages;
  const uint8_t* base = buf + blockIdx.x * per_cta;
  const int n = static_cast<int>(per_cta / (static_cast<size_t>(chunk) * per));
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], consumers); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol = 0;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      mbar_wait(&empty[s], ((i / stages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], chunk * per);
      for (int c = 0; c < per; ++c) {
        const uint8_t* src = base + (static_cast<size_t>(i) * per + c) * chunk;
        uint8_t* dst = sm + (static_cast<size_t>(s) * per + c) * chunk;
        if (hint) bulk_load_hint(dst, src, chunk, &full[s], pol); else bulk_load(dst, src, chunk, &full[s]);
      }
    }
  } else if (threadIdx.x >= 32 && threadIdx.x < 32 * (consumers + 1)) {
    unsigned acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      acc += sm[static_cast<size_t>(s) * chunk * per + threadIdx.x];
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0xFFFFFFFFu) *sink = acc;
  }
}

__global__ void k_ldg(const uint4* buf, size_t per_cta16, unsigned* sink) {
  const uint4* base = buf + blockIdx.x * per_cta16;
  uint32_t acc = 0;
  for (size_t i = threadIdx.x; i < per_cta16; i += blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (i + u * blockDim.x < per_cta16) ? __ldcs(base + i + u * blockDim.x) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = size_t(1) << 30;
  uint8_t* buf;
  unsigned* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch, size_t bytes, const char* name) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-48s %8.1f GB/s  (%s)\n", name, bytes * reps / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  struct Cfg { int chunk, stages, per, hint, ctas_per_sm, consumers; };
  std::vector<Cfg> cfgs = {{8448, 16, 1, 0, 1, 1}, {16384, 12, 1, 0, 1, 1}, {16896, 10, 1, 0, 1, 1},
                           {16896, 10, 1, 0, 1, 15}, {8448, 16, 1, 0, 1, 15}, {32768, 6, 1, 0, 1, 15},
                           {8448, 8, 1, 0, 2, 7}};
  for (auto c : cfgs) {
    const int ctas = nsm * c.ctas_per_sm;
    const size_t unit = static_cast<size_t>(c.chunk) * c.per;
    const size_t per_cta = (total / ctas) / unit * unit;
    const size_t smem = static_cast<size_t>(c.stages) * unit + 2 * c.stages * 8 + 1024;
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    char name[128];
    snprintf(name, sizeof name, "bulk chunk=%d st=%d per=%d ctas/sm=%d consumers=%d", c.chunk, c.stages, c.per, c.ctas_per_sm, c.consumers);
    timeit([&] { k_bulk<<<ctas, 32 * (c.consumers + 1), smem>>>(buf, per_cta, c.chunk, c.stages, c.per, c.hint, sink, c.consumers); }, per_cta * ctas, name);
  }
  for (int threads : {1024}) {
    for (int mult : {1}) {
      const int ctas = nsm * mult;
      const size_t per16 = total / 16 / ctas;
      char name[128];
      snprintf(name, sizeof name, "ldg.128 threads=%d ctas=%dx", threads, mult);
      timeit([&] { k_ldg<<<ctas, threads>>>(reinterpret_cast<const uint4*>(buf), per16, sink); }, per16 * 16 * ctas, name);
    }
  }
  return 0;
}
