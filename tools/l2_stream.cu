// Microbenchmark: per-SM TMA bulk-copy throughput when the source is L2-resident
// (all CTAs stream the same `wrap`-byte window), against the HBM case, with
// 1-D bulk copies of several sizes and ring depths; and a 2-D tensor-map load.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_stream tools/l2_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

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
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y) : "memory");
}

// mode 0: 1-D bulk of `chunk` bytes; mode 1: 2-D tensor box 128 rows x 128 B (16 KB)
__global__ void k_stream(const __grid_constant__ CUtensorMap tm, const uint8_t* buf, size_t wrap, int n, int chunk,
                         int stages, int mode, unsigned* sink, int producers) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(stages) * chunk);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t start = (static_cast<size_t>(blockIdx.x) * 7919 * chunk) % wrap;
  const int pw = threadIdx.x / 32;
  if (pw < producers) {
    if ((threadIdx.x & 31) == 0) {
      for (int i = pw; i < n; i += producers) {
        const int s = i % stages;
        mbar_wait(&empty[s], ((i / stages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], chunk);
        const size_t off = (start + static_cast<size_t>(i) * chunk) % wrap;
        if (mode == 0) bulk_load(sm + static_cast<size_t>(s) * chunk, buf + off, chunk, &full[s]);
        else tma2d(sm + static_cast<size_t>(s) * chunk, &tm, &full[s], 0, static_cast<int>((off / 128) % (wrap / 128 - 128)));
      }
    }
    __syncwarp();
  } else if (pw == producers) {
    unsigned acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      acc += sm[static_cast<size_t>(s) * chunk + threadIdx.x];
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0xFFFFFFFFu) *sink = acc;
  }
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
  CUtensorMap tm{};
  {
    cuuint64_t dims[2] = {128, total / 128};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("tensor map failed %d\n", (int)r);
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  struct Cfg { size_t wrap; int chunk, stages, mode; const char* name; int producers = 1; };
  Cfg cfgs[] = {{32u << 20, 8448, 8, 0, "L2 bulk 8.4KB x8"}, {32u << 20, 16384, 8, 0, "L2 bulk 16KB x8"},
                {32u << 20, 32768, 6, 0, "L2 bulk 32KB x6"}, {32u << 20, 16384, 8, 1, "L2 tensor 16KB x8"},
                {32u << 20, 16384, 12, 1, "L2 tensor 16KB x12"},
                {total, 16384, 8, 0, "HBM bulk 16KB x8"}, {total, 16384, 8, 1, "HBM tensor 16KB x8"},
                {32u << 20, 8448, 8, 0, "L2 bulk 8.4KB x8 p2", 2}, {32u << 20, 8448, 8, 0, "L2 bulk 8.4KB x8 p4", 4},
                {32u << 20, 16384, 8, 1, "L2 tensor 16KB x8 p2", 2}, {32u << 20, 16384, 8, 1, "L2 tensor 16KB x8 p4", 4},
                {32u << 20, 8448, 16, 0, "L2 bulk 8.4KB x16 p8", 8}};
  for (auto& c : cfgs) {
    const size_t smem = static_cast<size_t>(c.stages) * c.chunk + 2 * c.stages * 8 + 2048;
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const int n = static_cast<int>((total / nsm) / c.chunk);
    const int thr = 32 * (c.producers + 1);
    k_stream<<<nsm, thr, smem>>>(tm, buf, c.wrap, n, c.chunk, c.stages, c.mode, sink, c.producers);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    k_stream<<<nsm, thr, smem>>>(tm, buf, c.wrap, n, c.chunk, c.stages, c.mode, sink, c.producers);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = static_cast<double>(n) * c.chunk * nsm;
    const double gbs = bytes / (ms * 1e-3) / 1e9;
    printf("%-22s %8.1f GB/s chip, %6.1f B/clk/SM @%d MHz (%s)\n", c.name, gbs, gbs * 1e9 / nsm / (clk * 1e3), clk / 1000,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
