// K5 — the fused DGQ A8W4 linear on sm_100a (and K3, the plain int8 GEMM,
// as the same kernel with the dequant stage switched off).
//
// out[m, n] = ((float(acc[m, n]) * rs[m]) * s1[n]) (+ bias[n])
// acc[m, n] = sum_k Xq[m, k] * W_s8[k, n],  W_s8 = S2 * (code - ZP)
// (proj/src/kernel.cpp:144-153 = dequantize_to_s8 -> int8_gemm -> epilogue).
//
// Swap-AB: the tensor core's M side is the output-channel tile (128 weight
// rows), its N side the token tile (BN = 16..256), so one kernel serves decode
// (M = 1..64 tokens, weight-bandwidth bound) and prefill (tensor bound), and
// the TMEM accumulator lane == output channel makes the epilogue stores
// coalesced along n.
//
// Warp roles (256 threads, 1 CTA / SM):
//   warp 0     TMA producer: 1-D bulk copy of the packed INT4 chunk (+ group
//              scales) and a 2-D TMA of the Xq tile (SW128), one mbarrier/stage
//   warp 1     TMEM allocator + single-thread tcgen05.mma.kind::i8 issuer
//   warps 4-7  dequantisers (thread == weight row) writing the INT8 A tile in
//              the canonical SW128 K-major layout, then the epilogue
//              (tcgen05.ld -> scales -> global), or the split-K reduction.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "dequant.cuh"
#include "kernels.h"
#include "numerics.cuh"
#include "ptx.cuh"

namespace dgqk {

constexpr int kThreads = 256;
constexpr uint32_t kABytes = 128 * 128;

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void store_out(const DgqGemmParams& p, int m, int n, int32_t acc, float rsm, float s1v,
                                          float bv) {
  if (p.acc_out) p.acc_out[static_cast<size_t>(m) * p.ld_acc + n] = acc;
  if (p.out) {
    float y = p.fp16_mode ? epilogue_f16mode(acc, rsm, s1v) : epilogue_f32(acc, rsm, s1v);
    if (p.bias) y = __fadd_rn(y, bv);
    if (p.out_f16)
      static_cast<__half*>(p.out)[static_cast<size_t>(m) * p.ldy + n] = fp16_ref(y);
    else
      static_cast<float*>(p.out)[static_cast<size_t>(m) * p.ldy + n] = y;
  }
}

template <int BN, int SL, int SA, bool kFused>
__global__ void __launch_bounds__(kThreads, 1)
    k_dgq_gemm(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmA,
               const DgqGemmParams p) {
  static_assert(BN == 16 || BN == 32 || BN == 64 || BN == 128 || BN == 256, "BN");
  constexpr uint32_t kBBytes = BN * 128;
  constexpr int NA = kFused ? SA : SL;
  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
  constexpr uint32_t kIdesc = idesc_i8(128, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;
  uint8_t* sB = sA + NA * kABytes;
  uint8_t* sC = sB + SL * kBBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + (kFused ? SL * p.chunk_stride : 0));
  uint64_t* full_l = bars;
  uint64_t* empty_l = bars + SL;
  uint64_t* afull = bars + 2 * SL;
  uint64_t* aempty = afull + SA;
  uint64_t* done = aempty + SA;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  uint32_t* flag = tmem_slot + 1;

  const uint32_t warp = warp_id(), lane = lane_id();
  const int nt = blockIdx.x, mt = blockIdx.y, z = blockIdx.z;
  const int kb0 = z * p.kb_per_split;
  const int nkb = min(p.k_blocks - kb0, p.kb_per_split);

  if (threadIdx.x == 0) {
    for (int s = 0; s < SL; ++s) {
      mbar_init(&full_l[s], 1);
      mbar_init(&empty_l[s], kFused ? 129 : 1);
    }
    for (int s = 0; s < SA; ++s) {
      mbar_init(&afull[s], 128);
      mbar_init(&aempty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmB);
    if (!kFused) tma_prefetch_desc(&tmA);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      const uint32_t stage_tx = (kFused ? p.chunk_bytes : kABytes) + kBBytes;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % SL;
        const uint32_t ph = (i / SL) & 1;
        mbar_wait(&empty_l[s], ph ^ 1);
        const int kb = kb0 + i;
        mbar_arrive_expect_tx(&full_l[s], stage_tx);
        if (kFused) {
          const uint8_t* src = p.tiles + (static_cast<size_t>(nt) * p.k_blocks + kb) * p.chunk_bytes;
          bulk_load(sC + s * p.chunk_stride, src, p.chunk_bytes, &full_l[s]);
        } else {
          tma_load_2d(sA + s * kABytes, &tmA, &full_l[s], kb * 128, nt * 128);
        }
        tma_load_2d(sB + s * kBBytes, &tmB, &full_l[s], kb * 128, mt * BN);
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ----------------------------
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % SL;
        mbar_wait(&full_l[s], (i / SL) & 1);
        const int sa = kFused ? (i % SA) : s;
        if (kFused) mbar_wait(&afull[sa], (i / SA) & 1);
        tc_fence_after();
        const uint64_t da = umma_desc_sw128(smem_u32(sA + sa * kABytes));
        const uint64_t db = umma_desc_sw128(smem_u32(sB + s * kBBytes));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          // +32 bytes of K per step inside the 128-byte swizzle row
          mma_i8_ss(tmem, da + 2 * kk, db + 2 * kk, kIdesc, (i | kk) != 0);
        }
        mma_commit(&empty_l[s]);
        if (kFused) mma_commit(&aempty[sa]);
      }
      mma_commit(done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int d = threadIdx.x - 128;  // weight row / TMEM lane owned by this thread
    if (kFused) {
      // ------------------------------ dequantiser ------------------------
      const uint32_t sw = d & 7;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % SL;
        const int sa = i % SA;
        mbar_wait(&full_l[s], (i / SL) & 1);
        mbar_wait(&aempty[sa], ((i / SA) & 1) ^ 1);
        const uint8_t* chunk = sC + s * p.chunk_stride;
        const uint16_t* sc = reinterpret_cast<const uint16_t*>(chunk + 8192);
        uint8_t* arow = sA + sa * kABytes + (d >> 3) * 1024 + (d & 7) * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 w4 = *reinterpret_cast<const uint4*>(chunk + j * 2048 + d * 16);
          const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
          uint32_t o[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t sv = sc[((j * 32 + q * 8) >> p.gshift) * 128 + d];
            const uint32_t s2 = sv & 0xFFu, zp = sv >> 8;
            dq_word(wv[q], s2, dq_bias2(s2, zp), o[2 * q], o[2 * q + 1]);
          }
          *reinterpret_cast<uint4*>(arow + (((2 * j) ^ sw) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
          *reinterpret_cast<uint4*>(arow + (((2 * j + 1) ^ sw) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
        }
        fence_proxy_async_smem();
        mbar_arrive(&afull[sa]);
        mbar_arrive(&empty_l[s]);
      }
    }
    // ------------------------------ epilogue -----------------------------
    mbar_wait(done, 0);
    tc_fence_after();
    const uint32_t q = warp & 3;
    const uint32_t trow = tmem + ((q * 32) << 16);
    const int n = nt * 128 + d;
    const bool nvalid = n < p.N;
    const int m0 = mt * BN;
    const int mcount = min(BN, p.M - m0);
    const float s1v = (nvalid && p.s1) ? p.s1[n] : 0.0f;
    const float bv = (nvalid && p.bias) ? p.bias[n] : 0.0f;
    if (p.splits == 1) {
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        if (c0 >= mcount) break;
        uint32_t r[16];
        tmem_ld16(trow + c0, r);
        tmem_ld_wait();
        if (nvalid) {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int mi = c0 + t;
            if (mi < mcount) store_out(p, m0 + mi, n, static_cast<int32_t>(r[t]), p.rs ? p.rs[m0 + mi] : 0.0f, s1v, bv);
          }
        }
      }
    } else {
      // split-K: exact int32 reduction through L2, the last CTA applies the epilogue
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        if (c0 >= mcount) break;
        uint32_t r[16];
        tmem_ld16(trow + c0, r);
        tmem_ld_wait();
        if (nvalid) {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int mi = c0 + t;
            if (mi < mcount) atomicAdd(&p.ws[static_cast<size_t>(m0 + mi) * p.ldw + n], static_cast<int32_t>(r[t]));
          }
        }
      }
      __threadfence();
      named_bar_sync(1, 128);
      if (d == 0) {
        const uint32_t prev = atomicAdd(&p.counters[mt * gridDim.x + nt], 1u);
        *flag = (prev == static_cast<uint32_t>(p.splits - 1)) ? 1u : 0u;
      }
      named_bar_sync(1, 128);
      if (*flag) {
        __threadfence();
        if (nvalid) {
          for (int mi = 0; mi < mcount; ++mi) {
            int32_t* wp = &p.ws[static_cast<size_t>(m0 + mi) * p.ldw + n];
            const int32_t a = __ldcg(wp);
            __stcg(wp, 0);
            store_out(p, m0 + mi, n, a, p.rs ? p.rs[m0 + mi] : 0.0f, s1v, bv);
          }
        }
        if (d == 0) p.counters[mt * gridDim.x + nt] = 0u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

template <int BN, int SL, int SA, bool kFused>
size_t smem_bytes_for(uint32_t chunk_stride) {
  constexpr int NA = kFused ? SA : SL;
  size_t b = 1024 + static_cast<size_t>(NA) * kABytes + static_cast<size_t>(SL) * BN * 128;
  if (kFused) b += static_cast<size_t>(SL) * chunk_stride;
  b += (2 * SL + 2 * SA + 1) * 8 + 16;
  return b;
}

template <int BN, int SL, int SA, bool kFused>
cudaError_t launch_one(const DgqGemmPlan& plan, const CUtensorMap& tmB, const CUtensorMap& tmA,
                       const DgqGemmParams& p, cudaStream_t st) {
  auto kern = k_dgq_gemm<BN, SL, SA, kFused>;
  const size_t smem = smem_bytes_for<BN, SL, SA, kFused>(p.chunk_stride);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(plan.n_tiles, plan.m_tiles, plan.splits);
  kern<<<grid, kThreads, smem, st>>>(tmB, tmA, p);
  return cudaGetLastError();
}

}  // namespace dgqk

using namespace dgqk;

// Stage counts per token-tile width (~160-180 KB of smem, 1 CTA/SM).
#define DGQ_GEMM_CONFIGS(X) \
  X(16, 8, 3)               \
  X(32, 8, 3)               \
  X(64, 6, 3)               \
  X(128, 4, 3)              \
  X(256, 3, 2)

DgqGemmPlan dgq_plan_gemm(int M, int N, int K_pad, bool fused, int g, int force_bn, int force_splits) {
  DgqGemmPlan pl{};
  int bn = 256;
  if (M <= 16) bn = 16;
  else if (M <= 32) bn = 32;
  else if (M <= 64) bn = 64;
  else if (M <= 128) bn = 128;
  if (force_bn) bn = force_bn;
  pl.bn = bn;
  pl.m_tiles = (M + bn - 1) / bn;
  pl.n_tiles = (N + 127) / 128;
  const int kblocks = K_pad / 128;
  const int tiles = pl.m_tiles * pl.n_tiles;
  int splits = 1;
  if (tiles < 120) {
    splits = (148 + tiles - 1) / tiles;
    splits = splits > kblocks / 2 ? kblocks / 2 : splits;
    if (splits < 1) splits = 1;
  }
  if (force_splits) splits = force_splits;
  if (splits > kblocks) splits = kblocks;
  pl.kb_per_split = (kblocks + splits - 1) / splits;
  pl.splits = (kblocks + pl.kb_per_split - 1) / pl.kb_per_split;
  const uint32_t cs = (dgq_layout::chunk_bytes(g > 0 ? g : 128) + 1023) & ~1023u;
  size_t smem = 0;
#define DGQ_SMEM(BN_, SL_, SA_) \
  if (bn == BN_) smem = fused ? smem_bytes_for<BN_, SL_, SA_, true>(cs) : smem_bytes_for<BN_, SL_, SA_, false>(cs);
  DGQ_GEMM_CONFIGS(DGQ_SMEM)
#undef DGQ_SMEM
  pl.smem_bytes = smem;
  pl.ws_bytes = pl.splits > 1 ? static_cast<size_t>(pl.m_tiles) * bn * pl.n_tiles * 128 * sizeof(int32_t) : 0;
  pl.counter_bytes = pl.splits > 1 ? static_cast<size_t>(tiles) * sizeof(uint32_t) : 0;
  return pl;
}

cudaError_t dgq_launch_gemm(const DgqGemmPlan& plan, bool fused, const CUtensorMap& tmB, const CUtensorMap& tmA,
                            const DgqGemmParams& p, cudaStream_t st) {
#define DGQ_LAUNCH(BN_, SL_, SA_)                                                           \
  if (plan.bn == BN_)                                                                       \
    return fused ? launch_one<BN_, SL_, SA_, true>(plan, tmB, tmA, p, st)                   \
                 : launch_one<BN_, SL_, SA_, false>(plan, tmB, tmA, p, st);
  DGQ_GEMM_CONFIGS(DGQ_LAUNCH)
#undef DGQ_LAUNCH
  return cudaErrorInvalidValue;
}
