// K5d — the decode-shaped (M <= 64 tokens) fused DGQ linear on sm_100a.
//
// acc[m, n] = sum_k Xq[m, k] * S2[g, n] * (code[k, n] - ZP[g, n])
//           = sum_g S2[g, n] * D_g[n, m],   D_g[n, m] = sum_{k in g} (code[k, n] - ZP[g, n]) * Xq[m, k]
// (proj/src/kernel.cpp:144-153; W_s8 = S2 (code - ZP), proj/src/format.cpp:129-130).
// Every term is an exact integer (int32 wrap-around is harmless: the final sum
// is inside int32 by the h * 127^2 < 2^31 precondition), so the result is
// bit-identical to int8_gemm on dequantize_to_s8.
//
// Why this shape: at M <= 64 the layer is weight-bandwidth bound, and the
// per-code INT4 -> INT8 dequantisation of the prefill kernel (13 integer
// instructions per 8 codes, plus a shared-memory round trip) caps the stream
// near 2 TB/s.  Here the tensor core consumes (code - ZP) as a signed 8-bit
// A operand staged in TENSOR MEMORY — 7 integer instructions per 8 codes
// (nibble spread and a borrow-free byte-wise subtraction) and no shared-memory
// write — and the group scale S2 is applied to the small TMEM partial D_g
// (one IMAD per (group, channel, token)) instead of to every weight.
//
// Data path, one persistent CTA per SM, units of 128 channels x 128 k,
// grouped into stages of up to 4 consecutive units of one tile:
//   warp 0     producer: ONE 1-D bulk copy of the stage's contiguous prepared
//              chunks (~34 KB; per-CTA TMA throughput grows with request size,
//              tools/stream_bench.cu) and one 3-D TMA box of its Xq tiles.
//   warps 1-2  MMA issuers (warp 1 owns TMEM): tcgen05.mma kind::i8, A from
//              TMEM, B (tokens) from shared memory; a single thread issues an
//              MMA only every ~50 cycles, so the two warps take alternate units.
//   warps 4-11 unpack, two per TMEM lane quadrant (thread = channel, 64-k half):
//              codes - ZP -> tcgen05.st into the A slot.
//   warps 12-15 epilogue, thread = channel (its TMEM lane): 32-column
//              tcgen05.ld of the stage's partials, S2-scaled into register
//              accumulators, and the segment finish.
// Rings decouple the roles: SL shared-memory stages, 2 TMEM A slots, up to 8
// TMEM partial slots.
// Work split ("stream-K"): the n_tiles x k_blocks units are cut into P equal
// contiguous ranges (P = #SMs), so every SM streams the same number of bytes
// whatever the layer shape.  A tile whose K range is split across CTAs is
// reduced exactly with int32 red.global.add into a zeroed workspace; the CTA
// that arrives last (per-tile counter) applies the FP epilogue and re-zeroes
// the workspace.  Integer addition is associative, so the result does not
// depend on the arrival order.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "kernels.h"
#include "numerics.cuh"
#include "ptx.cuh"

namespace dgqk {

namespace dec {
// TMEM (512 columns): A ring [kSA][UPS x 32] in [0, kDCol0), partial ring
// [SD][ku x gpk x BN] in [256, 512).
#ifndef DGQ_DEC_SA
#define DGQ_DEC_SA 2  // TMEM A slots (stages of UPS units x 32 columns); tools A/B
#endif
constexpr int kSA = DGQ_DEC_SA;
constexpr int kDCol0 = kSA * 128;  // A ring [0, kSA x 128), partial ring [kDCol0, 512)
constexpr int kMaxSD = 8;
constexpr int kMmaWarps = 2;     // warps 1..2: MMA issuers (warp 1 also owns TMEM)
constexpr int kUnpackWarps = 8;  // warps 4..11; epilogue warps 12..15
constexpr int kThreads = 128 + 32 * kUnpackWarps + 128;

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ int owner_of(long long u, int P, long long U) {
  return static_cast<int>(((u + 1) * P - 1) / U);
}

__device__ __forceinline__ long long clk64() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
  return c;
}

__device__ __forceinline__ void trace_stamp(const DgqDecodeParams& p, int role, int i) {
  if (p.trace && static_cast<int>(blockIdx.x) == p.trace_cta && i < 1024) {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    p.trace[role * 1024 + i] = t;
  }
}

// Walks this CTA's range of units (128 channels x 128 k each) in STAGES: up
// to `ku` consecutive units of one tile, moved by one bulk copy and consumed
// by every role as one step (per-step synchronisation costs ~100s of cycles,
// so a step carries up to ku x 8.4 KB of weights).  Tile / k-block are kept
// incrementally (no 64-bit division in the loops); every role walks the same
// sequence.
struct StageWalk {
  int kb, tile, cnt, left, idx;
  __device__ __forceinline__ void init(long long u0, int nu, int KB, int ku) {
    tile = static_cast<int>(u0 / KB);
    kb = static_cast<int>(u0 - static_cast<long long>(tile) * KB);
    left = nu;
    idx = 0;
    cnt = min(min(ku, KB - kb), left);
  }
  __device__ __forceinline__ bool valid() const { return left > 0; }
  __device__ __forceinline__ void next(int KB, int ku) {
    left -= cnt;
    kb += cnt;
    if (kb == KB) {
      kb = 0;
      ++tile;
    }
    ++idx;
    cnt = min(min(ku, KB - kb), left);
  }
  // this stage ends the CTA's range or its tile: a segment of accumulation ends
  __device__ __forceinline__ bool ends_segment(int KB) const { return left == cnt || kb + cnt == KB; }
};

template <int BN>
__device__ __forceinline__ void store_final(const DgqDecodeParams& p, int t, int e, const int32_t (&acc)[BN]) {
  int li = 0;  // which layer the global tile t belongs to
#pragma unroll
  for (int i = 1; i < kDecodeMaxSub; ++i)
    if (i < p.nsub && t >= p.sub[i].tile_begin) li = i;
  const DgqDecodeSub& sb = p.sub[li];
  const int n = (t - sb.tile_begin) * 128 + e;
  if (n >= sb.N) return;
  const float s1v = sb.s1 ? sb.s1[n] : 0.0f;
  const float bv = sb.bias ? sb.bias[n] : 0.0f;
#pragma unroll
  for (int m = 0; m < BN; ++m) {
    if (m >= p.M) break;
    if (p.acc_out) p.acc_out[static_cast<size_t>(m) * p.ld_acc + n] = acc[m];
    if (sb.out) {
      const float rsm = p.rs[m];
      float y = p.fp16_mode ? epilogue_f16mode(acc[m], rsm, s1v) : epilogue_f32(acc[m], rsm, s1v);
      if (sb.bias) y = __fadd_rn(y, bv);
      if (p.out_f16)
        static_cast<__half*>(sb.out)[static_cast<size_t>(m) * sb.ldy + n] = fp16_ref(y);
      else
        static_cast<float*>(sb.out)[static_cast<size_t>(m) * sb.ldy + n] = y;
    }
  }
}

// global address of the prepared chunk of (global tile t, k-block kb)
__device__ __forceinline__ const uint8_t* chunk_addr(const DgqDecodeParams& p, int t, int kb) {
  int li = 0;
#pragma unroll
  for (int i = 1; i < kDecodeMaxSub; ++i)
    if (i < p.nsub && t >= p.sub[i].tile_begin) li = i;
  return p.sub[li].tiles +
         (static_cast<size_t>(t - p.sub[li].tile_begin) * p.k_blocks + kb) * static_cast<size_t>(p.chunk_bytes);
}

}  // namespace dec

template <int BN, int SL, int UPS>
__global__ void __launch_bounds__(dec::kThreads, 1)
    k_dgq_decode(const __grid_constant__ CUtensorMap tmB, const DgqDecodeParams p) {
  using namespace dec;
  constexpr uint32_t kBBytes = BN * 128;
  constexpr uint32_t kIdesc = idesc_i8(128, BN);  // A = code - ZP (s8), B = Xq (s8)
  const int KB = p.k_blocks;
  const int ku = p.ku;                   // units per stage (<= UPS)
  const int gpk = p.gpk;                 // groups per k-block (1, 2 or 4)
  const int gpk_log2 = gpk >> 1;         // 1 -> 0, 2 -> 1, 4 -> 2
  const int dslot = ku * gpk * BN;       // TMEM columns of one stage's partials
  const int sdl = p.sd_log2;             // partial slots = 1 << sdl
  const long long U = static_cast<long long>(p.n_tiles) * KB;
  const int P = gridDim.x;
  const long long u0 = static_cast<long long>(blockIdx.x) * U / P;
  const long long u1 = static_cast<long long>(blockIdx.x + 1) * U / P;
  const int nu = static_cast<int>(u1 - u0);

  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = sm;                       // [SL][UPS][BN x 128] Xq tiles (SW128 K-major)
  uint8_t* sC = sB + SL * UPS * kBBytes;  // [SL][UPS x chunk_bytes] prepared weight chunks (one bulk copy)
  const uint32_t stage_cb = UPS * p.chunk_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + SL * stage_cb);
  uint64_t* full = bars;                  // [SL] chunks + Xq tiles landed
  uint64_t* empty = full + SL;            // [SL] stage consumed by every role
  uint64_t* afull = empty + SL;           // [kSA] A slot written (unpack warps)
  uint64_t* aempty = afull + kSA;         // [kSA] A slot read by the MMA
  uint64_t* dfull = aempty + kSA;         // [kMaxSD] partials ready (MMA commit)
  uint64_t* dempty = dfull + kMaxSD;      // [kMaxSD] partials read (epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + kMaxSD);
  uint32_t* s_flag = tmem_slot + 1;

  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0 && p.trace && blockIdx.x < 1024) {  // tools only: CTA start stamp
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    p.trace[14 * 1024 + blockIdx.x] = static_cast<long long>(t);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < SL; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kUnpackWarps + kMmaWarps + 4);
    }
    for (int s = 0; s < kSA; ++s) {
      mbar_init(&afull[s], kUnpackWarps);
      mbar_init(&aempty[s], kMmaWarps);
    }
    for (int s = 0; s < kMaxSD; ++s) {
      mbar_init(&dfull[s], kMmaWarps);
      mbar_init(&dempty[s], 4);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (p.dbg & 1024) {
    // tools/dec_gap.py: the weight stream alone (one producer lane, every other
    // role idle) — separates the copy engine from the pipeline's cost at the
    // kernel boundary
    if (threadIdx.x == 0 && nu > 0) {
      StageWalk w;
      w.init(u0, nu, KB, ku);
      for (; w.valid(); w.next(KB, ku)) {
        const int sl = w.idx % SL;
        if (w.idx >= SL) mbar_wait(&full[sl], ((w.idx / SL) - 1) & 1);
        mbar_arrive_expect_tx(&full[sl], w.cnt * p.chunk_bytes);
        bulk_load(sC + sl * stage_cb, dec::chunk_addr(p, w.tile, w.kb), w.cnt * p.chunk_bytes, &full[sl]);
      }
      for (int i = (w.idx > SL ? w.idx - SL : 0); i < w.idx; ++i) mbar_wait(&full[i % SL], (i / SL) & 1);
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    if ((p.dbg & 2048) && threadIdx.x == 32) asm volatile("griddepcontrol.wait;" ::: "memory");  // tools
  } else if (warp == 0) {
    // ------------------------------ producer ------------------------------
    // one bulk copy of the stage's contiguous chunks + one 3-D TMA box of its
    // Xq tiles (large requests keep the per-CTA TMA queue streaming)
    if (lane == 0 && nu > 0) {
      auto issue = [&](const StageWalk& w, bool weights, bool btile) {
        const int sl = w.idx % SL;
        if (weights) {
          mbar_wait(&empty[sl], ((w.idx / SL) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[sl], w.cnt * p.chunk_bytes + ((p.dbg & 8) ? 0u : ku * kBBytes));
          bulk_load(sC + sl * stage_cb, dec::chunk_addr(p, w.tile, w.kb), w.cnt * p.chunk_bytes, &full[sl]);
          dec::trace_stamp(p, 0, w.idx);
        }
        if (btile && !(p.dbg & 8)) tma_load_3d(sB + sl * UPS * kBBytes, &tmB, &full[sl], 0, 0, w.kb);  // tools: bit 3
      };
      // the first stages' weights do not depend on the previous kernel (PDL);
      // their Xq tiles do.  Each bulk request occupies the TMA engine for
      // ~bytes / 32 B per clock, so only p.pre_stages stages go ahead of the wait.
      StageWalk w;
      w.init(u0, nu, KB, ku);
      const int pre = p.pre_stages < 1 ? 1 : (p.pre_stages > SL ? SL : p.pre_stages);
      StageWalk w2 = w;
      int last = 0;  // the last stage whose weights went ahead
      issue(w2, true, false);
      for (int i = 1; i < pre; ++i) {
        w2.next(KB, ku);
        if (!w2.valid()) break;
        issue(w2, true, false);
        last = w2.idx;
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      // those stages get their Xq tiles; then weights and Xq together
      for (;;) {
        issue(w, false, true);
        if (w.idx == last) break;
        w.next(KB, ku);
      }
      for (w.next(KB, ku); w.valid(); w.next(KB, ku)) issue(w, true, true);
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    __syncwarp();  // lanes 1-31 wait here, not at the CTA barrier (see prefill.cu)
  } else if (warp <= kMmaWarps) {
    // ------------------------------ MMA issuers ----------------------------
    // A single thread issues a tcgen05.mma only every ~50 cycles (issue
    // latency, not tensor-core throughput: tools/tc_probe2.cu), so two warps
    // issue alternate units of each stage.  The unpack warps arrive on afull
    // only after they waited for the stage's TMA (full), so afull also orders
    // the Xq tile before the MMA reads it.
    // The whole warp runs the loop converged and one lane is elected inside
    // the MMA/commit asm: the operands stay in uniform registers, which takes
    // the issue cost from ~50 to ~24 cycles per MMA (tools/tc_probe2.cu).
    {
      const int mw = warp - 1;
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      uint32_t qoff[4], acc_in[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int q = p.gshift >= 7 ? 0 : ((kk * 32) >> p.gshift);
        qoff[kk] = static_cast<uint32_t>(q * BN);
        acc_in[kk] = (p.gshift >= 7 ? kk == 0 : ((kk * 32) & ((1 << p.gshift) - 1)) == 0) ? 0u : 1u;
      }
      const uint32_t unit_dcols = static_cast<uint32_t>(gpk * BN);
      StageWalk w;
      for (w.init(u0, nu, KB, ku); w.valid(); w.next(KB, ku)) {
        const int i = w.idx, s = i % SL, sa = i % kSA, sd = i & ((1 << sdl) - 1);
        mbar_wait(&afull[sa], (i / kSA) & 1);
        mbar_wait(&dempty[sd], ((i >> sdl) & 1) ^ 1);
        tc_fence_after();
        for (int c = mw; c < w.cnt && !(p.dbg & 1); c += kMmaWarps) {  // tools: bit 0 skips the MMAs
          const uint64_t db = umma_desc_sw128(smem_u32(sB + (s * UPS + c) * kBBytes));
          const uint32_t a0 = tm + (sa * UPS + c) * 32;
          const uint32_t d0 = tm + kDCol0 + sd * dslot + c * unit_dcols;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // K = 32 per MMA: +8 TMEM columns of A, +32 B of the B row
            mma_i8_ts_warp(d0 + qoff[kk], a0 + kk * 8, db + 2 * kk, kIdesc, acc_in[kk]);
        }
        if (p.dbg & 1) {  // tools: no tcgen05 at all -> plain arrives
          if (lane == 0) {
            mbar_arrive(&empty[s]);
            mbar_arrive(&aempty[sa]);
            mbar_arrive(&dfull[sd]);
          }
        } else {
          mma_commit_warp(&empty[s]);
          mma_commit_warp(&aempty[sa]);
          mma_commit_warp(&dfull[sd]);
        }
        if (mw == 0 && lane == 0) dec::trace_stamp(p, 1, i);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 4 + kUnpackWarps) {
    // -------- unpack: codes - ZP -> s8 A tile in TMEM (two warps per lane quadrant) ---------
    // byte-wise (c - z) without borrows: ((c | 0x80) - z) ^ 0x80 with c, z in [0, 15]
    const int row = (warp & 3) * 32 + lane;     // output channel inside the tile == TMEM lane
    const int half = (warp - 4) >> 2;           // which 64-k half of the row
    const uint32_t taddr_lane = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int q0h = p.gshift >= 7 ? 0 : ((half * 64) >> p.gshift);       // group of k [64h, 64h+32)
    const int q1h = p.gshift >= 7 ? 0 : ((half * 64 + 32) >> p.gshift);  // group of k [64h+32, 64h+64)
    StageWalk w;
    for (w.init(u0, nu, KB, ku); w.valid(); w.next(KB, ku)) {
      const int i = w.idx, s = i % SL, sa = i % kSA;
      mbar_wait(&full[s], (i / SL) & 1);
      mbar_wait(&aempty[sa], ((i / kSA) & 1) ^ 1);
      // all of the stage's loads first (one shared-memory round trip), then the
      // byte arithmetic and one tcgen05.st per unit
      const uint8_t* stage_c = sC + s * stage_cb;
      uint4 cw[UPS][2];
      uint32_t zz[UPS][2];
#pragma unroll
      for (int c = 0; c < UPS; ++c) {
        if (c < w.cnt) {
          // 64 codes of channel `row`: [j][row][16 B]; byte b of word w = k(8w+b) | k(8w+b+4) << 4
          const uint8_t* chunk = stage_c + c * p.chunk_bytes;
          const uint16_t* sc = reinterpret_cast<const uint16_t*>(chunk + 8192);
          cw[c][0] = *reinterpret_cast<const uint4*>(chunk + (half * 2) * 2048 + row * 16);
          cw[c][1] = *reinterpret_cast<const uint4*>(chunk + (half * 2 + 1) * 2048 + row * 16);
          // zero points of the (up to two) groups of this 64-k half
          zz[c][0] = sc[q0h * 128 + row] >> 8;
          zz[c][1] = sc[q1h * 128 + row] >> 8;
        }
      }
#pragma unroll
      for (int c = 0; c < UPS; ++c) {
        if (c < w.cnt) {
          const uint32_t z0 = zz[c][0] * 0x01010101u, z1 = zz[c][1] * 0x01010101u;
          const uint32_t wv[8] = {cw[c][0].x, cw[c][0].y, cw[c][0].z, cw[c][0].w,
                                  cw[c][1].x, cw[c][1].y, cw[c][1].z, cw[c][1].w};
          uint32_t a[16];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t z = k < 4 ? z0 : z1;
            a[2 * k] = (((wv[k] & 0x0F0F0F0Fu) | 0x80808080u) - z) ^ 0x80808080u;
            a[2 * k + 1] = ((((wv[k] >> 4) & 0x0F0F0F0Fu) | 0x80808080u) - z) ^ 0x80808080u;
          }
          if (!(p.dbg & 2)) tmem_st16(tmem + taddr_lane + (sa * UPS + c) * 32 + half * 16, a);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&afull[sa]);
        mbar_arrive(&empty[s]);
        if (warp == 4) dec::trace_stamp(p, 2, i);
      }
    }
  } else if (warp >= 4 + kUnpackWarps) {
    // ------------------------- group epilogue ----------------------------------
    const int e = (warp & 3) * 32 + lane;  // output channel inside the tile == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // rs / workspace of earlier kernels
    int32_t acc[BN];
#pragma unroll
    for (int m = 0; m < BN; ++m) acc[m] = 0;
    StageWalk w;
    w.init(u0, nu, KB, ku);
    bool seg_from_tile_start = w.kb == 0;
    for (; w.valid(); w.next(KB, ku)) {
      const int i = w.idx, s = i % SL, sd = i & ((1 << sdl) - 1);
      mbar_wait(&dfull[sd], (i >> sdl) & 1);
      tc_fence_after();
      // group scales of the stage's (unit, group) partials, then the partials
      // themselves in 32-column TMEM loads (column j = (unit * gpk + group) * BN + token)
      int32_t s2v[UPS * 4];
      const int ncq = w.cnt * gpk;
      const uint16_t* sc0 = reinterpret_cast<const uint16_t*>(sC + s * stage_cb + 8192) + e;
      const int cstride = static_cast<int>(p.chunk_bytes >> 1);  // u16 stride between the stage's chunks
#pragma unroll
      for (int cq = 0; cq < UPS * 4; ++cq) {
        s2v[cq] = 0;
        if (cq < ncq) {
          const int c = cq >> gpk_log2, q = cq & (gpk - 1);
          s2v[cq] = static_cast<int32_t>(sc0[c * cstride + q * 128] & 0xFFu);
        }
      }
      const uint32_t dcol = tmem + lane_base + kDCol0 + sd * dslot;
      const int ncols = ncq * BN;
#pragma unroll
      for (int j0 = 0; j0 < UPS * 4 * BN && j0 < 128; j0 += 32) {
        if (j0 < ncols) {
          uint32_t d[32];
          if (p.dbg & 4) {
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) d[jj] = 0;
          } else {
            tmem_ld32(dcol + j0, d);
            tmem_ld_wait();
          }
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int j = j0 + jj;
            if (j < ncols) acc[j % BN] += s2v[j / BN] * static_cast<int32_t>(d[jj]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&dempty[sd]);
        mbar_arrive(&empty[s]);
        if (warp == 12) dec::trace_stamp(p, 3, i);
      }
      if (w.ends_segment(KB)) {
        const int t = w.tile;
        const long long tb = static_cast<long long>(t) * KB, te = tb + KB;
        if (seg_from_tile_start && w.kb + w.cnt == KB) {
          if (!(p.dbg & 4096)) dec::store_final<BN>(p, t, e, acc);
        } else {
          int32_t* ws = p.ws + static_cast<size_t>(t) * BN * 128 + e;
#pragma unroll
          for (int m = 0; m < BN; ++m)
            if (m < p.M) atomicAdd(ws + m * 128, acc[m]);
          __threadfence();
          named_bar(2, 128);
          if (e == 0) {
            const int contrib = owner_of(te - 1, P, U) - owner_of(tb, P, U) + 1;
            const unsigned old = atomicAdd(p.counters + t, 1u);
            *s_flag = (old == static_cast<unsigned>(contrib - 1)) ? 1u : 0u;
          }
          named_bar(2, 128);
          if (*s_flag) {
            __threadfence();
#pragma unroll
            for (int m = 0; m < BN; ++m) {
              if (m < p.M) {
                acc[m] = __ldcg(ws + m * 128);
                ws[m * 128] = 0;
              }
            }
            if (!(p.dbg & 4096)) dec::store_final<BN>(p, t, e, acc);
            if (e == 0) p.counters[t] = 0u;
          }
          named_bar(2, 128);  // s_flag is rewritten by the next segment
        }
#pragma unroll
        for (int m = 0; m < BN; ++m) acc[m] = 0;
        seg_from_tile_start = true;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0 && p.trace && blockIdx.x < 1024) {  // tools only: CTA end stamp
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    p.trace[15 * 1024 + blockIdx.x] = static_cast<long long>(t);
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int BN, int SL, int UPS>
static cudaError_t launch_dec(const CUtensorMap& tmB, const DgqDecodeParams& p, int grid, bool pdl,
                              cudaStream_t st) {
  auto kern = k_dgq_decode<BN, SL, UPS>;
  const size_t smem = dgq_decode_smem_bytes(BN, SL * UPS, p.chunk_bytes);
  cudaError_t e = dgq_allow_smem(kern, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(dec::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, tmB, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace dgqk

using namespace dgqk;

int dgq_decode_partial_cols() { return 512 - dec::kDCol0; }

size_t dgq_decode_smem_bytes(int bn, int sl, uint32_t chunk_stride) {
  return 1024 + static_cast<size_t>(sl) * (bn * 128 + chunk_stride) +
         (2 * sl + 2 * dec::kSA + 2 * dec::kMaxSD) * 8 + 16;
}

// (token tile) -> stages x units per stage; <= 227 KB of shared memory at g = 32
#define DGQ_DEC_CFG(X) X(8, 5, 4) X(16, 5, 4) X(32, 4, 4) X(64, 3, 4)

int dgq_decode_stages(int bn) {
#define DGQ_DEC_ST(BN_, SL_, UPS_) \
  if (bn == BN_) return SL_ * UPS_;
  DGQ_DEC_CFG(DGQ_DEC_ST)
#undef DGQ_DEC_ST
  return 0;
}

int dgq_decode_units_per_stage(int bn) {
#define DGQ_DEC_U(BN_, SL_, UPS_) \
  if (bn == BN_) return UPS_;
  DGQ_DEC_CFG(DGQ_DEC_U)
#undef DGQ_DEC_U
  return 1;
}

cudaError_t dgq_launch_decode(int bn, const CUtensorMap& tmB, const DgqDecodeParams& p, int grid, bool pdl,
                              cudaStream_t st) {
#define DGQ_DEC_L(BN_, SL_, UPS_) \
  if (bn == BN_) return launch_dec<BN_, SL_, UPS_>(tmB, p, grid, pdl, st);
  DGQ_DEC_CFG(DGQ_DEC_L)
#undef DGQ_DEC_L
  return cudaErrorInvalidValue;
}
