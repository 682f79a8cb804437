// K5 — the fused DGQ A8W4 linear on sm_100a (and K3, the plain int8 GEMM,
// as the same kernel with the dequant stage switched off).
//
// out[m, n] = ((float(acc[m, n]) * rs[m]) * s1[n]) (+ bias[n])
// acc[m, n] = sum_k Xq[m, k] * W_s8[k, n],  W_s8 = S2 * (code - ZP)
// (proj/src/kernel.cpp:144-153 = dequantize_to_s8 -> int8_gemm -> epilogue).
//
// Two orientations of one pipeline (tcgen05.mma.cta_group::1.kind::i8, TMEM
// int32 accumulators, SW128 K-major smem operands):
//  * decode (BN <= 64 tokens, kSwap): D^T[n, m] = W^T Xq^T — the 128 weight
//    rows are the MMA M side, the tokens the N side (N = 16..64).  The K range
//    is split over a thread-block CLUSTER (gridDim.z = splits <= 8) whose
//    partial int32 tiles are reduced through distributed shared memory.
//  * prefill (BN = 128/256 tokens): D[m, n] = Xq W — tokens on TMEM lanes, the
//    NT = 2 dequantised weight tiles (256 output channels) are one N = 256
//    operand, so each epilogue thread owns 16 consecutive output channels
//    and stores 16-byte vectors.
// Warp roles (128 + 32*DQW threads, 1 CTA / SM):
//   warp 0     TMA producer: 1-D bulk copies of the packed INT4 chunks (+ group
//              scales), 2-D TMA of the Xq tile.  With programmatic dependent
//              launch the weight loads of the first stages are issued before
//              griddepcontrol.wait, overlapping the previous kernel.
//   warp 1     TMEM allocator + single-thread MMA issuer
//   warps 4..  DQW dequantiser warps (INT4 -> INT8 into the SW128 A/B tile),
//              then the epilogue (tcgen05.ld -> scales -> global).
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "dequant.cuh"
#include "kernels.h"
#include "numerics.cuh"
#include "ptx.cuh"

namespace cg = cooperative_groups;

namespace dgqk {

constexpr uint32_t kABytes = 128 * 128;

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Debug phase timestamps (p.dbg != null): [cta][8] ns
#define DGQ_TS(slot)                                                                                        \
  do {                                                                                                      \
    if (p.dbg)                                                                                              \
      p.dbg[(static_cast<size_t>(blockIdx.z) * gridDim.y * gridDim.x + blockIdx.y * gridDim.x + blockIdx.x) * \
                8 + (slot)] = gtimer();                                                                     \
  } while (0)

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ float epi_value(const DgqGemmParams& p, int32_t acc, float rsm, float s1v, float bv) {
  float y = p.fp16_mode ? epilogue_f16mode(acc, rsm, s1v) : epilogue_f32(acc, rsm, s1v);
  if (p.bias) y = __fadd_rn(y, bv);
  return y;
}

__device__ __forceinline__ void store_out(const DgqGemmParams& p, int m, int n, int32_t acc, float rsm, float s1v,
                                          float bv) {
  if (p.acc_out) p.acc_out[static_cast<size_t>(m) * p.ld_acc + n] = acc;
  if (p.out) {
    const float y = epi_value(p, acc, rsm, s1v, bv);
    if (p.out_f16)
      static_cast<__half*>(p.out)[static_cast<size_t>(m) * p.ldy + n] = fp16_ref(y);
    else
      static_cast<float*>(p.out)[static_cast<size_t>(m) * p.ldy + n] = y;
  }
}

constexpr uint32_t tmem_cols_pow2(int c) {
  return c <= 32 ? 32 : (c <= 64 ? 64 : (c <= 128 ? 128 : (c <= 256 ? 256 : 512)));
}

template <int BN, int NT, int SL, int SA, int DQW, bool kFused>
struct Cfg {
  static constexpr bool kSwap = BN <= 64;
  static constexpr int kThreads = 128 + 32 * DQW;
  static constexpr int kDqThreads = 32 * DQW;
  static constexpr int kRows = 128 * NT;              // weight rows per CTA
  static constexpr int kJP = 4 * kRows / kDqThreads;  // 32-k slices per dequant thread
  static constexpr int kAcc = kSwap ? NT : BN / 128;  // accumulators
  static constexpr int kAccCols = kSwap ? BN : 128 * NT;
  static constexpr uint32_t kBBytes = BN * 128;
  static constexpr int NA = kFused ? SA : SL;  // A-tile slots
  static constexpr uint32_t kTmemCols = tmem_cols_pow2(kAcc * kAccCols);
  static_assert(kJP == 1 || kJP == 2 || kJP == 4, "dequant split");
  static_assert(kSwap || NT == 2, "prefill orientation uses two weight tiles (N = 256)");
  static size_t smem_bytes(uint32_t chunk_stride) {
    size_t b = 1024 + static_cast<size_t>(NA) * NT * kABytes + static_cast<size_t>(SL) * kBBytes;
    if (kFused) b += static_cast<size_t>(SL) * NT * chunk_stride;
    b += (2 * SL + 2 * SA + 1) * 8 + 16 + BN * 4 + 2 * 256 * 4;
    return b;
  }
};

// Prefill epilogue, one warp: 32 token rows x [cbeg, cend) output channels.
// Per 128-byte box column block: all TMEM loads of the block in flight before
// one wait, branch-free scale math, packed FP16 conversion (+ the reference's
// sub-2^-24 flush), 128B-swizzled smem staging and one TMA tensor store.
template <bool kF16, bool kF16Mode, bool kBias>
__device__ __forceinline__ void epi_tma(const DgqGemmParams& p, uint32_t tbase, float rsm, const float* s_s1,
                                        const float* s_bias, uint8_t* stg0, const CUtensorMap* tmY, int cbeg,
                                        int cend, int nbase, int mbox) {
  constexpr int kCB = kF16 ? 64 : 32;  // columns per 128-byte box row
  const uint32_t lane = lane_id();
  uint8_t* row0 = stg0 + lane * 128;
  const uint32_t sw = lane & 7;
  int buf = 0;
#pragma unroll 1
  for (int c0 = cbeg; c0 < cend; c0 += kCB) {
    if (nbase + c0 >= p.N) break;
    uint32_t r[kCB];
#pragma unroll
    for (int c1 = 0; c1 < kCB; c1 += 16) tmem_ld16(tbase + c0 + c1, *reinterpret_cast<uint32_t(*)[16]>(&r[c1]));
    if (lane == 0) bulk_wait_read<1>();  // this buffer's previous store has finished reading smem
    __syncwarp();
    tmem_ld_wait();
    uint8_t* row = row0 + buf * 4096;
#pragma unroll
    for (int c1 = 0; c1 < kCB; c1 += 8) {
      float y[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int32_t acc = static_cast<int32_t>(r[c1 + k]);
        const float s1v = s_s1[c0 + c1 + k];
        float v = kF16Mode ? epilogue_f16mode(acc, rsm, s1v) : epilogue_f32(acc, rsm, s1v);
        if (kBias) v = __fadd_rn(v, s_bias[c0 + c1 + k]);
        y[k] = v;
      }
      if (kF16) {
        uint32_t h[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const __half2 hh = __floats2half2_rn(y[2 * k], y[2 * k + 1]);
          uint32_t u = *reinterpret_cast<const uint32_t*>(&hh);
          // fp16_round (proj/src/quant.cpp:33-35) flushes |x| < 2^-24 to signed zero
          if (fabsf(y[2 * k]) < 0x1p-24f) u = (u & 0xFFFF0000u) | ((__float_as_uint(y[2 * k]) >> 16) & 0x8000u);
          if (fabsf(y[2 * k + 1]) < 0x1p-24f) u = (u & 0x0000FFFFu) | (__float_as_uint(y[2 * k + 1]) & 0x80000000u);
          h[k] = u;
        }
        *reinterpret_cast<uint4*>(row + (((c1 / 8) ^ sw) << 4)) = make_uint4(h[0], h[1], h[2], h[3]);
      } else {
        *reinterpret_cast<float4*>(row + (((c1 / 4) ^ sw) << 4)) = make_float4(y[0], y[1], y[2], y[3]);
        *reinterpret_cast<float4*>(row + (((c1 / 4 + 1) ^ sw) << 4)) = make_float4(y[4], y[5], y[6], y[7]);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmY, stg0 + buf * 4096, nbase + c0, mbox);
      bulk_commit();
    }
    buf ^= 1;
  }
  if (lane == 0) bulk_wait_all();
}

template <int BN, int NT, int SL, int SA, int DQW, bool kFused>
__global__ void __launch_bounds__(Cfg<BN, NT, SL, SA, DQW, kFused>::kThreads, 1)
    k_dgq_gemm(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmA,
               const __grid_constant__ CUtensorMap tmY, const DgqGemmParams p) {
  using C = Cfg<BN, NT, SL, SA, DQW, kFused>;
  static_assert(BN == 16 || BN == 32 || BN == 64 || BN == 128 || BN == 256, "BN");
  constexpr bool kSwap = C::kSwap;
  constexpr uint32_t kBBytes = C::kBBytes;
  constexpr uint32_t kIdesc = kSwap ? idesc_i8(128, BN) : idesc_i8(128, 128 * NT);

  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-B alignment for the SW128 atoms, applied as an offset so the compiler
  // keeps the shared address space (LDS/STS rather than generic LD/ST)
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = sm;                         // [NA][NT][128 x 128] weights (INT8, SW128 K-major)
  uint8_t* sB = sA + C::NA * NT * kABytes;  // [SL][BN x 128]      activation codes (SW128 K-major)
  uint8_t* sC = sB + SL * kBBytes;          // [SL][NT][chunk_stride] packed INT4 chunks
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + (kFused ? SL * NT * p.chunk_stride : 0));
  uint64_t* full_l = bars;
  uint64_t* empty_l = bars + SL;
  uint64_t* afull = bars + 2 * SL;
  uint64_t* aempty = afull + SA;
  uint64_t* done = aempty + SA;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  float* s_rs = reinterpret_cast<float*>(tmem_slot + 4);  // [BN]
  float* s_s1 = s_rs + BN;                                  // [256] (prefill orientation)
  float* s_bias = s_s1 + 256;                               // [256]

  const uint32_t warp = warp_id(), lane = lane_id();
  const int mt = blockIdx.x;   // token tile (fastest: CTAs in flight share weights in L2)
  const int ntp = blockIdx.y;  // group of NT weight tiles
  const int z = blockIdx.z;    // K split (cluster rank when splits > 1)
  const int kb0 = z * p.kb_per_split;
  const int nkb = max(0, min(p.k_blocks - kb0, p.kb_per_split));
  const int n_tiles = (p.N + 127) / 128;

  if (threadIdx.x == 0) {
    DGQ_TS(0);
    for (int s = 0; s < SL; ++s) {
      mbar_init(&full_l[s], 1);
      mbar_init(&empty_l[s], kFused ? DQW + 1 : 1);  // dequant warps + the MMA commit
    }
    for (int s = 0; s < SA; ++s) {
      mbar_init(&afull[s], DQW);
      mbar_init(&aempty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmB);
    if (!kFused) tma_prefetch_desc(&tmA);
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) DGQ_TS(1);

  if (warp == 0) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      int ntl = 0;  // weight tiles that exist in this group (the last group may hold one)
      for (int t = 0; t < NT; ++t) ntl += (ntp * NT + t) < n_tiles;
      const uint32_t stage_tx = (kFused ? p.chunk_bytes : kABytes) * ntl + kBBytes;
      auto load_w = [&](int i) {
        const int s = i % SL, kb = kb0 + i;
        for (int t = 0; t < ntl; ++t) {
          const int nt = ntp * NT + t;
          if (kFused) {
            const uint8_t* src = p.tiles + (static_cast<size_t>(nt) * p.k_blocks + kb) * p.chunk_bytes;
            bulk_load(sC + (s * NT + t) * p.chunk_stride, src, p.chunk_bytes, &full_l[s]);
          } else {
            tma_load_2d(sA + (s * NT + t) * kABytes, &tmA, &full_l[s], kb * 128, nt * 128);
          }
        }
      };
      // weights do not depend on the previous kernel: stream the first stages
      // before waiting for it (programmatic dependent launch)
      const int pre = nkb < SL ? nkb : SL;
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full_l[i], stage_tx);
        load_w(i);
      }
      griddep_wait();
      for (int i = 0; i < pre; ++i) tma_load_2d(sB + i * kBBytes, &tmB, &full_l[i], (kb0 + i) * 128, mt * BN);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % SL;
        mbar_wait(&empty_l[s], ((i / SL) & 1) ^ 1);
        mbar_arrive_expect_tx(&full_l[s], stage_tx);
        load_w(i);
        tma_load_2d(sB + s * kBBytes, &tmB, &full_l[s], (kb0 + i) * 128, mt * BN);
      }
    }
    __syncwarp();  // lanes 1-31 wait here, not at the CTA barrier (see prefill.cu)
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ----------------------------
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % SL;
        mbar_wait(&full_l[s], (i / SL) & 1);
        const int sa = kFused ? (i % SA) : s;
        if (kFused) mbar_wait(&afull[sa], (i / SA) & 1);
        tc_fence_after();
        const uint32_t b_addr = smem_u32(sB + s * kBBytes);
        const uint32_t a_addr = smem_u32(sA + sa * NT * kABytes);
        if constexpr (kSwap) {
          const uint64_t db = umma_desc_sw128(b_addr);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const uint64_t da = umma_desc_sw128(a_addr + t * kABytes);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // +32 B of K per step inside the 128-B swizzle row
              mma_i8_ss(tmem + t * BN, da + 2 * kk, db + 2 * kk, kIdesc, (i | kk) != 0);
          }
        } else {
          const uint64_t dw = umma_desc_sw128(a_addr);  // 256 weight rows = the N operand
#pragma unroll
          for (int a = 0; a < C::kAcc; ++a) {
            const uint64_t dx = umma_desc_sw128(b_addr + a * 128 * 128);  // 128 tokens = the M operand
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_i8_ss(tmem + a * 256, dx + 2 * kk, dw + 2 * kk, kIdesc, (i | kk) != 0);
          }
        }
        mma_commit(&empty_l[s]);
        if (kFused) mma_commit(&aempty[sa]);
      }
      mma_commit(done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int e = threadIdx.x - 128;  // 0 .. 32*DQW-1
    if (kFused) {
      // ------------------------------ dequantiser ------------------------
      const int rr = e % C::kRows;
      const int t = rr >> 7, d = rr & 127;
      const int j0 = (e / C::kRows) * C::kJP;
      const uint32_t sw = d & 7;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % SL;
        const int sa = i % SA;
        mbar_wait(&full_l[s], (i / SL) & 1);
        if (i == 0 && e == 0) DGQ_TS(2);
        mbar_wait(&aempty[sa], ((i / SA) & 1) ^ 1);
        const uint8_t* chunk = sC + (s * NT + t) * p.chunk_stride;
        const uint16_t* sc = reinterpret_cast<const uint16_t*>(chunk + 8192);
        uint8_t* arow = sA + (sa * NT + t) * kABytes + (d >> 3) * 1024 + (d & 7) * 128;
        uint4 w4[C::kJP];
#pragma unroll
        for (int jj = 0; jj < C::kJP; ++jj) w4[jj] = *reinterpret_cast<const uint4*>(chunk + (j0 + jj) * 2048 + d * 16);
        if (p.gshift >= 5) {
          // g >= 32: one (S2, ZP) per 32-k slice (one per k-block when g >= 128)
#pragma unroll
          for (int jj = 0; jj < C::kJP; ++jj) {
            const int j = j0 + jj;
            const uint32_t sv = sc[((j * 32) >> p.gshift) * 128 + d];
            const uint32_t s2 = sv & 0xFFu, bs = dq_bias2(s2, sv >> 8);
            const uint32_t wv[4] = {w4[jj].x, w4[jj].y, w4[jj].z, w4[jj].w};
            uint32_t o[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) dq_word(wv[q], s2, bs, o[2 * q], o[2 * q + 1]);
            *reinterpret_cast<uint4*>(arow + (((2 * j) ^ sw) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(arow + (((2 * j + 1) ^ sw) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < C::kJP; ++jj) {
            const int j = j0 + jj;
            const uint32_t wv[4] = {w4[jj].x, w4[jj].y, w4[jj].z, w4[jj].w};
            uint32_t o[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t sv = sc[((j * 32 + q * 8) >> p.gshift) * 128 + d];
              const uint32_t s2 = sv & 0xFFu;
              dq_word(wv[q], s2, dq_bias2(s2, sv >> 8), o[2 * q], o[2 * q + 1]);
            }
            *reinterpret_cast<uint4*>(arow + (((2 * j) ^ sw) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(arow + (((2 * j + 1) ^ sw) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&afull[sa]);
          mbar_arrive(&empty_l[s]);
        }
      }
    }
    // ------------------------------ epilogue -----------------------------
    if (e == 0) DGQ_TS(3);
    griddep_wait();  // row scales come from the previous kernel (K1)
    const int m0 = mt * BN;
    for (int i = e; i < BN; i += C::kDqThreads) s_rs[i] = (p.rs && m0 + i < p.M) ? p.rs[m0 + i] : 0.0f;
    if constexpr (!kSwap) {
      for (int i = e; i < 256; i += C::kDqThreads) {
        const int n = ntp * 256 + i;
        s_s1[i] = (p.s1 && n < p.N) ? p.s1[n] : 0.0f;
        s_bias[i] = (p.bias && n < p.N) ? p.bias[n] : 0.0f;
      }
    }
    named_bar_sync(1, C::kDqThreads);
    mbar_wait(done, 0);
    if (e == 0) DGQ_TS(4);
    griddep_launch();
    tc_fence_after();
    const uint32_t q = warp & 3;  // TMEM lane quadrant this warp may access
    if constexpr (kSwap) {
      if (e < 128 * NT && p.splits == 1) {
        const int t = e >> 7, d = e & 127;
        const int n = (ntp * NT + t) * 128 + d;
        const bool nvalid = n < p.N;
        const int mcount = min(BN, p.M - m0);
        const float s1v = (nvalid && p.s1) ? p.s1[n] : 0.0f;
        const float bv = (nvalid && p.bias) ? p.bias[n] : 0.0f;
        const uint32_t trow = tmem + ((q * 32) << 16) + t * BN;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          if (c0 >= mcount) break;
          uint32_t r[16];
          tmem_ld16(trow + c0, r);
          tmem_ld_wait();
          if (nvalid) {
#pragma unroll
            for (int k = 0; k < 16; ++k)
              if (c0 + k < mcount) store_out(p, m0 + c0 + k, n, static_cast<int32_t>(r[k]), s_rs[c0 + k], s1v, bv);
          }
        }
      } else if (e < 128 * NT) {
        // stage this CTA's partial tile for the cluster reduction: [col][row]
        int32_t* part = reinterpret_cast<int32_t*>(sB);
        const int t = e >> 7, d = e & 127;
        const uint32_t trow = tmem + ((q * 32) << 16) + t * BN;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(trow + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 16; ++k) part[(c0 + k) * (128 * NT) + t * 128 + d] = static_cast<int32_t>(r[k]);
        }
      }
    } else {
      // prefill orientation: lane = token, 16 consecutive output channels per load
      const int w8 = warp - 4;
      constexpr int kCSplit = 8 / (4 * C::kAcc);  // column splits per accumulator
      constexpr int kColsPerWarp = 256 / kCSplit;
      const int a = (w8 >> 2) % C::kAcc;
      const int cs = (w8 >> 2) / C::kAcc;
      const int mrow = a * 128 + q * 32 + lane;
      const int m = m0 + mrow;
      const bool mvalid = m < p.M;
      const float rsm = s_rs[mrow];
      const uint32_t tbase = tmem + ((q * 32) << 16) + a * 256;
      if (p.tma_out && !p.acc_out) {
        uint8_t* stg0 = sB + w8 * 8192;  // two 4 KB buffers per warp (pipeline smem is idle now)
        const int cbeg = cs * kColsPerWarp, cend = (cs + 1) * kColsPerWarp;
        const int mbox = m0 + a * 128 + q * 32;
#define DGQ_EPI(F16_, MODE_, BIAS_) \
  epi_tma<F16_, MODE_, BIAS_>(p, tbase, rsm, s_s1, s_bias, stg0, &tmY, cbeg, cend, ntp * 256, mbox)
        const bool b = p.bias != nullptr, f = p.fp16_mode != 0;
        if (p.out_f16) {
          if (f) { if (b) DGQ_EPI(true, true, true); else DGQ_EPI(true, true, false); }
          else   { if (b) DGQ_EPI(true, false, true); else DGQ_EPI(true, false, false); }
        } else {
          if (f) { if (b) DGQ_EPI(false, true, true); else DGQ_EPI(false, true, false); }
          else   { if (b) DGQ_EPI(false, false, true); else DGQ_EPI(false, false, false); }
        }
#undef DGQ_EPI
      } else {
#pragma unroll 1
        for (int c0 = cs * kColsPerWarp; c0 < (cs + 1) * kColsPerWarp; c0 += 16) {
          const int n0 = ntp * 256 + c0;
          if (n0 >= p.N) break;
          uint32_t r[16];
          tmem_ld16(tbase + c0, r);
          tmem_ld_wait();
          if (!mvalid) continue;
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (n0 + k < p.N) store_out(p, m, n0 + k, static_cast<int32_t>(r[k]), rsm, s_s1[c0 + k], s_bias[c0 + k]);
        }
      }
    }
  }
  if constexpr (kSwap) {
    if (p.splits > 1) {
      // ---- cluster split-K: exact int32 sum of the partial tiles over DSMEM ----
      cg::cluster_group cluster = cg::this_cluster();
      tc_fence_before();
      cluster.sync();  // every partial staged (release / acquire across the cluster)
      const int e = static_cast<int>(threadIdx.x) - 128;
      if (e >= 0 && e < 128 * NT) {
        const int t = e >> 7, d = e & 127;
        const int n = (ntp * NT + t) * 128 + d;
        const int m0 = mt * BN;
        const int mcount = min(BN, p.M - m0);
        const int per = (mcount + p.splits - 1) / p.splits;  // token columns reduced by this rank
        const int c_lo = z * per, c_hi = min(mcount, c_lo + per);
        if (n < p.N && c_lo < c_hi) {
          const float s1v = p.s1 ? p.s1[n] : 0.0f;
          const float bv = p.bias ? p.bias[n] : 0.0f;
          int32_t* part = reinterpret_cast<int32_t*>(sB);
          for (int c = c_lo; c < c_hi; ++c) {
            int32_t acc = 0;
            for (int r = 0; r < p.splits; ++r) acc += cluster.map_shared_rank(part, r)[c * (128 * NT) + t * 128 + d];
            store_out(p, m0 + c, n, acc, s_rs[c], s1v, bv);
          }
        }
      }
      cluster.sync();  // peers may still read this CTA's partial tile
    }
  }
  if (threadIdx.x == 128) DGQ_TS(6);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
  if (threadIdx.x == 32) DGQ_TS(7);
}

template <int BN, int NT, int SL, int SA, int DQW, bool kFused>
cudaError_t launch_one(const DgqGemmPlan& plan, const CUtensorMap& tmB, const CUtensorMap& tmA,
                       const CUtensorMap& tmY, const DgqGemmParams& p, cudaStream_t st) {
  using C = Cfg<BN, NT, SL, SA, DQW, kFused>;
  auto kern = k_dgq_gemm<BN, NT, SL, SA, DQW, kFused>;
  const size_t smem = C::smem_bytes(p.chunk_stride);
  cudaError_t e = dgq_allow_smem(kern, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(plan.m_tiles, (plan.n_tiles + NT - 1) / NT, plan.splits);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[na].val.programmaticStreamSerializationAllowed = plan.pdl ? 1 : 0;
  ++na;
  if (plan.splits > 1) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = 1;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = plan.splits;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  e = cudaLaunchKernelEx(&cfg, kern, tmB, tmA, tmY, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace dgqk

using namespace dgqk;

// (BN, NT, SL, SA, DQW): <= 227 KB of smem, 1 CTA / SM.  BN <= 64: decode
// orientation with cluster split-K; BN >= 128: prefill orientation.
#define DGQ_GEMM_CONFIGS(X) \
  X(16, 1, 8, 6, 8)         \
  X(32, 1, 8, 6, 8)         \
  X(64, 1, 8, 4, 8)         \
  X(128, 2, 4, 2, 8)        \
  X(256, 2, 3, 2, 8)

namespace {
constexpr size_t kMaxSmem = 232448;

// Cycle estimate for one config: per k-block the slowest of the tensor pipe
// (8192 MAC/clk/SM), the dequantiser and the L2->SM stream (~40 B/clk/SM),
// times the k-blocks a CTA runs, times the waves; cluster split-K adds a
// DSMEM reduction.
double est_cycles(int M, int N, int kblocks, int bn, int nt, int splits, bool fused) {
  const int m_tiles = (M + bn - 1) / bn;
  const int groups = ((N + 127) / 128 + nt - 1) / nt;
  const long ctas = static_cast<long>(m_tiles) * groups * splits;
  const double waves = static_cast<double>((ctas + 147) / 148);
  const double bytes = nt * (fused ? 8448.0 : 16384.0) + bn * 128.0;
  double kb = nt * bn / 2.0;
  if (fused && kb < 160.0 * nt) kb = 160.0 * nt;
  if (bytes / 40.0 > kb) kb = bytes / 40.0;
  const int kps = (kblocks + splits - 1) / splits;
  double t = waves * (kps * kb + 2500.0 + nt * bn * 6.0);
  if (splits > 1) t += 800.0 + bn * 8.0;
  return t;
}
}  // namespace

namespace {
// Test/tools override of the planner (0 = never use K5d; other bits force work
// splits).  Thread-local: an override set by one host thread never changes the
// plans of another caller of the library.
thread_local int g_decode_mode = 1;
int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}
}  // namespace

extern "C" void dgq_debug_set_decode(int mode) { g_decode_mode = mode; }
namespace {
thread_local int g_pair_cap = 0;
}
extern "C" void dgq_debug_set_pair_cap(int cap) { g_pair_cap = cap; }
int dgq_prefill2_cluster_cap() { return g_pair_cap; }
extern "C" int dgq_debug_decode_mode() { return g_decode_mode; }

DgqGemmPlan dgq_plan_gemm(int M, int N, int K_pad, bool fused, int g, int force_bn, int force_splits) {
  DgqGemmPlan pl{};
  const int kblocks = K_pad / 128;
  // K5p (CTA pairs, prefill.cu) for M >= 256: persistent pairs with a
  // stream-K split of the (256 x 256 tile, k-block) units, so every pair does
  // the same MMA work whatever the tile count (the one-CTA kernel below
  // leaves 1.51 waves of 224 tiles on OPT-30B q/k/v/out/fc2 at 2048 tokens).
  // Tools / tests: mode bit 10 forces K5p, bit 11 forces the 128-wide tile,
  // bit 12 disables K5p, bit 13 disables stream-K (round-robin whole tiles,
  // and then K5p only when its tiles fill >= 6 waves of pairs).
  const bool sk = (g_decode_mode & 0x2000) == 0;
  const uint32_t cb = static_cast<uint32_t>(dgq_layout::chunk_bytes(g > 0 ? g : 128));
  const long long t256_ = static_cast<long long>((M + 255) / 256) * ((N + 255) / 256);
  const bool pair_ok = (g_decode_mode & 0x400) != 0 || sk || t256_ >= 6LL * (sm_count() / 2);
  // K5p from 256 tokens; between 64 and 256 only for large weight matrices,
  // whose stream-K pairs outrun the one-CTA kernel (tools/decode_sweep.py:
  // OPT-30B fc2 at M = 128 / 192: 56 vs 93 / 142 us) while small ones keep
  // the one-CTA kernel (K5p has a ~30 us floor: 4096^2 at M = 64 takes 29 vs 12 us)
  const bool big_w = static_cast<double>(N) * K_pad >= 100e6;
  const int pair_min_m = (g_decode_mode & 0x400) ? 33 : (big_w ? 64 : 256);  // tools: 0x400 admits 33 <= M
  if (fused && M >= pair_min_m && pair_ok && (g_decode_mode & 0x1000) == 0 && !force_bn && !force_splits &&
      dgq_prefill2_smem_bytes(cb, 1) <= 232448) {
    const int pairs = sm_count() / 2;
    const long long mp = (M + 255) / 256;
    const long long t256 = mp * ((N + 255) / 256), t128 = mp * ((N + 127) / 128);
    const double c256 = static_cast<double>((t256 + pairs - 1) / pairs);        // waves x tile time
    const double c128 = 0.5 * static_cast<double>((t128 + pairs - 1) / pairs);
    pl.prefill2 = 1;
    pl.stream_k = sk ? 1 : 0;
    // round robin: the 128-wide tile measured ~40 % slower per tile area, so it
    // is only taken when it saves more than half of the 256-wide tail
    pl.pair_tn = ((g_decode_mode & 0x800) != 0 || (!sk && c128 * 1.6 < c256)) ? 128 : 256;
    // two token sub-tiles per CTA (512-token pair tiles) from 512 tokens, with
    // stream-K balancing the tiles; mode bit 17 keeps one (256-token tiles)
    // two sub-tiles pay an exposed epilogue per segment for a ~30 % faster
    // main loop: worth it from ~25 k-blocks of 512-token tiles per pair
    // (tools/decode_sweep.py --s2 / --s1, after the branch-free epilogue:
    // q 7168^2 at M = 1024 / 2048 45 / 84 vs 54 / 91 us, 4096^2 at 1024 30 vs 23)
    const long long t512 = ((M + 511) / 512) * static_cast<long long>((N + 255) / 256);
    const bool s2_pays = t512 * kblocks >= 25LL * pairs;
    pl.pair_sub = (sk && M >= 512 && (s2_pays || (g_decode_mode & 0x40000000)) &&
                   (g_decode_mode & 0x20000) == 0 && dgq_prefill2_smem_bytes(cb, 2) <= 232448) ? 2 : 1;
    pl.bn = 256 * pl.pair_sub;
    pl.nt = pl.pair_tn / 128;
    pl.m_tiles = static_cast<int>((M + pl.bn - 1) / pl.bn);
    pl.n_tiles = (N + 127) / 128;
    pl.splits = 1;
    pl.kb_per_split = kblocks;
    pl.ctas = 2 * dgq_prefill2_clusters(M, N, pl.pair_tn, kblocks, sk, pl.pair_sub);
    pl.smem_bytes = dgq_prefill2_smem_bytes(cb, pl.pair_sub);
    if (sk) {
      pl.ws_bytes = static_cast<size_t>(pairs) * kPrefill2SlotBytes;
      pl.counter_bytes = static_cast<size_t>(pairs) * 2 * 4;
    }
    pl.pdl = 1;
    return pl;
  }
  const int dec_bn = M <= 8 ? 8 : (M <= 16 ? 16 : (M <= 32 ? 32 : 64));
  const int dec_gpk = g >= 128 ? 1 : (g > 0 ? 128 / g : 1);
  // K5d wins up to 32 tokens; at 33..64 the weight-tile-per-CTA kernel below is faster
  // K5d streams the weights with every SM from its first cycle but pays a
  // fixed ~8 us; the one-CTA kernel is cheaper for small matrices and, as M
  // grows, for medium ones (tools/decode_sweep.py --nodec: 4096^2 7.6 vs 8.6 us
  // at M = 1, LLaMA-7B up 16.0 vs 16.8 at M = 16, OPT-30B q 19.7 vs 21.3 at
  // M = 32; fc1 / fc2 always K5d)
  const double kn = static_cast<double>(K_pad) * N;
  const int dec_max_m = (g_decode_mode & 0x10000000) ? 64  // tools: mode bit 28 admits M <= 64
                        : (g_decode_mode & 0x8000000) ? 32   // tools: mode bit 27: K5d up to 32 whatever the size
                        : kn >= 100e6 ? 32 : kn >= 48e6 ? 16 : kn >= 32e6 ? 8 : 0;
  if (fused && g >= 32 && g % 32 == 0 && M <= dec_max_m && dec_bn * dec_gpk <= 128 && g_decode_mode && !force_bn &&
      !force_splits) {
    // K5d: weight-streaming decode kernel, one persistent CTA per SM (stream-K)
    pl.decode = 1;
    pl.bn = dec_bn;
    pl.nt = 1;
    pl.m_tiles = 1;
    pl.n_tiles = (N + 127) / 128;
    pl.splits = 1;
    pl.kb_per_split = kblocks;
    const long long units = static_cast<long long>(pl.n_tiles) * kblocks;
    pl.ctas = static_cast<int>(units < sm_count() ? units : sm_count());
    const uint32_t cs = static_cast<uint32_t>(dgq_layout::chunk_bytes(g));
    pl.smem_bytes = dgq_decode_smem_bytes(pl.bn, dgq_decode_stages(pl.bn), cs);
    pl.ws_bytes = static_cast<size_t>(pl.n_tiles) * pl.bn * 128 * 4;
    pl.counter_bytes = static_cast<size_t>(pl.n_tiles) * 4;
    pl.est_cycles = 0;
    pl.pdl = (g_decode_mode & 0x100) ? 0 : 1;  // tools: mode bit 8 disables PDL
    return pl;
  }
  const uint32_t cs = (dgq_layout::chunk_bytes(g > 0 ? g : 128) + 1023) & ~1023u;
  double best = 1e30;
  int bbn = 0, bnt = 1, bsp = 1;
  size_t bsmem = 0;
  struct Cand {
    int bn, nt;
    size_t smem;
  };
  const Cand cand[] = {
#define DGQ_CAND(BN_, NT_, SL_, SA_, DQ_)                                                \
  {BN_, NT_, fused ? Cfg<BN_, NT_, SL_, SA_, DQ_, true>::smem_bytes(cs)                 \
                   : Cfg<BN_, NT_, SL_, SA_, DQ_, false>::smem_bytes(cs)},
      DGQ_GEMM_CONFIGS(DGQ_CAND)
#undef DGQ_CAND
  };
  for (const auto& c : cand) {
    const int bn = c.bn, nt = c.nt;
    if (c.smem > kMaxSmem) continue;
    if (force_bn && bn != force_bn) continue;
    if (!force_bn && bn > 16 && bn / 2 >= M) continue;  // never more than 2x token padding
    const int m_tiles = (M + bn - 1) / bn;
    const int groups = ((N + 127) / 128 + nt - 1) / nt;
    const int ctas = m_tiles * groups;
    int smax = 1;
    if (bn <= 64) {  // cluster split-K (decode orientation only), <= 8 CTAs per cluster
      smax = ctas >= 148 ? 1 : 148 / ctas;
      if (smax > 8) smax = 8;
      if (smax > kblocks) smax = kblocks;
    }
    for (int sp = 1; sp <= smax; ++sp) {
      if (force_splits && sp != force_splits) continue;
      const int kps = (kblocks + sp - 1) / sp;
      if (kps * (sp - 1) >= kblocks) continue;  // a rank would get no k-block
      const double t = est_cycles(M, N, kblocks, bn, nt, sp, fused);
      if (t < best) {
        best = t;
        bbn = bn;
        bnt = nt;
        bsp = sp;
        bsmem = c.smem;
      }
    }
  }
  if (bbn == 0) {  // forced combination outside the search space: smallest tile, no split
    bbn = 16;
    bnt = 1;
    bsp = 1;
  }
  pl.bn = bbn;
  pl.nt = bnt;
  pl.m_tiles = (M + bbn - 1) / bbn;
  pl.n_tiles = (N + 127) / 128;
  pl.kb_per_split = (kblocks + bsp - 1) / bsp;
  pl.splits = bsp;
  pl.smem_bytes = bsmem;
  pl.ws_bytes = 0;
  pl.counter_bytes = 0;
  pl.est_cycles = best;
  pl.pdl = 1;
  return pl;
}

cudaError_t dgq_launch_gemm(const DgqGemmPlan& plan, bool fused, const CUtensorMap& tmB, const CUtensorMap& tmA,
                            const CUtensorMap& tmY, const DgqGemmParams& p, cudaStream_t st) {
#define DGQ_LAUNCH(BN_, NT_, SL_, SA_, DQ_)                                          \
  if (plan.bn == BN_ && plan.nt == NT_)                                              \
    return fused ? launch_one<BN_, NT_, SL_, SA_, DQ_, true>(plan, tmB, tmA, tmY, p, st)  \
                 : launch_one<BN_, NT_, SL_, SA_, DQ_, false>(plan, tmB, tmA, tmY, p, st);
  DGQ_GEMM_CONFIGS(DGQ_LAUNCH)
#undef DGQ_LAUNCH
  return cudaErrorInvalidValue;
}
