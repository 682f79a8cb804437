// K5p — the prefill-shaped (many tokens) fused DGQ linear on sm_100a: a
// persistent, CTA-PAIR kernel (tcgen05.mma.cta_group::2, M = 256, N = 256).
//
// out[m, n] = ((float(acc[m, n]) * rs[m]) * s1[n]) (+ bias[n]),
// acc[m, n] = sum_k Xq[m, k] * W_s8[k, n],  W_s8 = S2 * (code - ZP)
// (proj/src/kernel.cpp:144-153; proj/src/format.cpp:129-130).
//
// Why a CTA pair: the INT4 -> INT8 dequantisation of the weight operand costs
// ~13 integer instructions per 8 codes and must keep pace with the tensor
// pipe.  With cta_group::2 the pair computes a 256-token x 256-channel tile
// per MMA while each CTA stages only ITS half of each operand: 128 token rows
// of Xq (TMA) and 128 dequantised channel rows of W_s8 — half the dequant per
// MMA cycle compared with one CTA doing the same tile.  Each CTA's TMEM holds
// its 128 tokens x 256 channels, so two accumulators fit in 512 columns and
// the epilogue of tile t overlaps the main loop of tile t + 1.
//
// Per CTA (512 threads), both CTAs of the pair run the same tile sequence:
//   warp 0      producer: 2-D TMA of its 128 x 128 Xq tile + 1-D bulk copy of
//               its 128-channel prepared weight chunk per k-block (SL ring).
//   warp 1      TMEM (cta_group::2 alloc, both CTAs); in the leader CTA the
//               converged MMA issuer: waits until BOTH CTAs' dequantised
//               stages are ready, 4 x tcgen05.mma.cta_group::2.kind::i8 per
//               k-block, commits multicast to both CTAs' barriers.
//   warps 4-11  dequantisers: channel row x 64-k half, INT4 -> INT8 into the
//               canonical SW128 K-major B tile, then (one thread) a
//               release.cluster arrive on the leader's `ready` barrier.
//   warps 12-15 epilogue: tcgen05.ld (thread = token row) -> scales -> FP16
//               -> 128B-swizzled staging -> TMA tensor store; releases the
//               accumulator with arrives on the leader's `tempty`.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <mutex>
#include <map>
#include <cstdlib>
#include <algorithm>

#include "dequant.cuh"
#include "kernels.h"
#include "numerics.cuh"
#include "ptx.cuh"

namespace dgqk {
namespace pf {

// Three rings, sized from the measured chain (tools/pf_trace.py): a bulk copy
// lands ~0.5-0.8 us after issue and a group dequantises a k-block in ~0.8 us,
// against a 0.26 us MMA step, so the packed chunks are fetched kLag k-blocks
// ahead of the Xq tiles and released by the dequantisers (not the MMA).
// S = token sub-tiles per CTA: each dequantised weight tile feeds S MMAs
// (pair tile = 256*S tokens x TN channels), so the INT4 -> INT8 work per MMA
// cycle falls by S.  S = 2 fills TMEM with one accumulator set (2 x 256
// columns): the epilogue of a tile no longer overlaps the next tile's main
// loop, but the dequantisers (now two groups) have twice the time per k-block.
template <int S, int TN = 256>
struct Cfg {
  static constexpr int kSA = S == 1 ? 5 : 3;        // Xq stages (S tiles each, released by the MMA)
#ifndef DGQ_PF_EPIW2
#define DGQ_PF_EPIW2 12  // epilogue warps at S = 2 (8: two per TMEM lane quadrant, 4 KB staging each)
#endif
  // S == 2 exposes the epilogue (one accumulator set): three warps per TMEM
  // lane quadrant split the channels, with 2 KB staging buffers (64-byte row
  // segments) and one packed-chunk stage fewer to fit
  static constexpr int kEpiWarps = S == 1 ? 4 : DGQ_PF_EPIW2;
  static constexpr uint32_t kStagingPerWarp = (S == 2 && kEpiWarps > 8) ? 2048 : 4096;
  static constexpr int kSC = S == 1 ? 7 : (kEpiWarps > 8 ? 4 : 5);  // packed-chunk stages (released by the dequantisers)
  static constexpr int kSB = S == 1 ? 4 : 3;        // dequantised weight-tile slots (> dequant groups)
  static constexpr int kDqGroups = S == 1 ? 3 : 2;  // groups of four dequant warps, alternate k-blocks
  static constexpr int kEpiWarp0 = 4 + 4 * kDqGroups;  // first epilogue warp
  static constexpr int kXWarp = kEpiWarp0 + kEpiWarps;  // second Xq-tile producer warp
  static constexpr int kThreads = 32 * (kXWarp + 1);
  // accumulator sets in TMEM (TN * S columns each): two whenever they fit, so a
  // tile's epilogue overlaps the next tile's main loop
  static constexpr int kNAcc = TN * S <= 256 ? 2 : 1;
};
constexpr uint32_t kATile = 128 * 128;   // 128 token rows x 128 k (bytes)
constexpr uint32_t kBTile = 128 * 128;   // 128 channel rows x 128 k

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Per-k-block "stage dequantised" signal to the leader: a relaxed arrive
// preceded by a cluster-scope release fence restricted to shared::cta (a
// release pattern; see the dequantiser).
// The dequant threads' st.shared are made visible to the async proxy by
// fence.proxy.async and ordered before the fence by the group's named barrier;
// the leader's tcgen05.mma reads them after its acquire.cluster wait.
__device__ __forceinline__ void arrive_remote_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
#ifndef DGQ_PF_TEMPTY_RELAXED
#define DGQ_PF_TEMPTY_RELAXED 1  // tools: 0 = release.cluster arrive on tempty (A/B)
#endif
// "This warp has drained its accumulator rows" to the leader's tempty: the
// TMEM reads are ordered by tcgen05.fence::before_thread_sync (issued by the
// caller, after tcgen05.wait::ld), the MMA issuer's acquire wait and its
// tcgen05.fence::after_thread_sync.  A release arrive at cluster scope would
// also wait for this warp's ~10 KB of output stores to be performed cluster-
// wide (~0.8 us of the tile-boundary stop, tools/pf_trace.py): the release
// here is restricted to shared::cta (nothing in shared memory is published)
// and the arrive is relaxed, so the stores drain while the next tile's MMAs run.
__device__ __forceinline__ void arrive_tmem_drained(uint32_t cluster_addr) {
#if DGQ_PF_TEMPTY_RELAXED
  asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#else
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#endif
}
// Barriers completed by arrivals from the PEER CTA are polled with test_wait:
// a suspended try_wait is not woken promptly by a remote (DSMEM) arrival and
// sleeps out its time limit (~1000 cycles per k-block, measured).
__device__ __forceinline__ bool try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
#ifndef DGQ_PF_LATE_TRIGGER
#define DGQ_PF_LATE_TRIGGER 0  // tools: 1 triggers dependents at the end of the epilogue (A/B)
#endif
#ifndef DGQ_PF_RELAXED_READY
#define DGQ_PF_RELAXED_READY 0  // tools: 1 drops the release fence before the ready arrive (A/B of its cost)
#endif
#ifndef DGQ_PF_TSLEEP
#define DGQ_PF_TSLEEP 128  // ns the MMA issuer sleeps between polls of tempty (tools: A/B)
#endif
#ifndef DGQ_PF_BACKOFF
#define DGQ_PF_BACKOFF 0
#endif
#ifndef DGQ_PF_WATCHDOG
#define DGQ_PF_WATCHDOG 0
#endif
__device__ __forceinline__ void watchdog(long long& n, int id, uint32_t parity) {
#if DGQ_PF_WATCHDOG
  if (++n == (1ll << 24)) {
    printf("prefill2 stuck: cta %d warp %d lane %d wait %d parity %u\n", blockIdx.x, threadIdx.x / 32, threadIdx.x % 32,
           id, parity);
  }
  if (n > (1ll << 25)) __trap();
#endif
}
// non-blocking probe of a local barrier phase
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// 2-D TMA load into this CTA's smem whose completion is signalled on an
// mbarrier of either CTA of the pair (here: the leader's), so the leader's
// MMA issuer learns directly that both halves of the Xq tile have landed.
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity, int id = 0) {
  long long n = 0;
  while (!try_wait_cluster(bar, parity)) watchdog(n, id, parity);
}
__device__ __forceinline__ void wait_local(uint64_t* bar, uint32_t parity, int id) {
  long long n = 0;
  while (!mbar_try_wait(bar, parity)) {
#if DGQ_PF_BACKOFF
    __nanosleep(DGQ_PF_BACKOFF);
#endif
    watchdog(n, id, parity);
  }
}
// converged-warp issue (one lane elected inside the asm)
__device__ __forceinline__ void mma2_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::
          "r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(kCols) : "memory");
}
__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Work decomposition.  Round robin: pair c runs whole tiles c, c + ncl, ...
// Stream-K (p.stream_k): the tiles x k-blocks units are cut into ncl equal
// contiguous ranges, one per pair, so every pair does the same MMA work
// whatever the tile count (e.g. 224 tiles of OPT-30B q_proj at 2048 tokens
// over 74 pairs = 3.03 tiles each instead of 4 waves).  A range is a sequence
// of segments (tile t, k-blocks [lo, hi)); only the FIRST segment of a range
// can start inside a tile (lo > 0, a "contributor": its int32 partial goes to
// the pair's workspace slot) and only the LAST can end inside one (lo == 0,
// hi < KB, the "owner": it adds the contributors' partials — exact integer
// sums — before the epilogue).  Owners run at the end of their range and
// contributors at the start of theirs, so the owner's wait is normally over
// before it begins; all pairs are co-resident (grid <= active clusters).
struct SegIter {
  long long u, uend;  // stream-K: current / end unit
  int t, total, step, KB, sk;
  __device__ SegIter(const DgqGemmParams& p, int cid, int ncl, int total_, int KB_)
      : t(cid), total(total_), step(ncl), KB(KB_), sk(p.stream_k) {
    const long long U = static_cast<long long>(total_) * KB_;
    if (p.sk_b[0] >= 0) {  // the launcher's balanced split (see sk_bounds)
      u = p.sk_b[cid];
      uend = p.sk_b[cid + 1];
    } else {
      u = U * cid / ncl;
      uend = U * (cid + 1) / ncl;
    }
  }
  // units of this pair and the (tile, k-block) of its i-th unit
  __device__ int count() const {
    if (sk) return static_cast<int>(uend - u);  // valid before the first next()
    const int mine = t < total ? (total - 1 - t) / step + 1 : 0;
    return mine * KB;
  }
  // A division-free cursor over the pair's units: the producer and the
  // dequantisers step through units one (or kDqGroups) at a time, and a 64-bit
  // division per unit costs a lone producer thread ~0.5 us (tools/pf_trace.py).
  struct Cursor {
    int t, kb;
  };
  __device__ Cursor first() const {
    Cursor c;
    if (sk) {
      c.t = static_cast<int>(u / KB);
      c.kb = static_cast<int>(u - static_cast<long long>(c.t) * KB);
    } else {
      c.t = t;
      c.kb = 0;
    }
    return c;
  }
  __device__ void advance(Cursor& c) const {
    if (++c.kb == KB) {
      c.kb = 0;
      c.t += sk ? 1 : step;
    }
  }
  __device__ bool next(int& tile, int& lo, int& hi) {
    if (sk) {
      if (u >= uend) return false;
      tile = static_cast<int>(u / KB);
      lo = static_cast<int>(u - static_cast<long long>(tile) * KB);
      const long long tend = static_cast<long long>(tile + 1) * KB;
      hi = static_cast<int>((uend < tend ? uend : tend) - static_cast<long long>(tile) * KB);
      u = static_cast<long long>(tile) * KB + hi;
      return true;
    }
    if (t >= total) return false;
    tile = t;
    lo = 0;
    hi = KB;
    t += step;
    return true;
  }
};
// tools/pf_trace.py: globaltimer stamps of CTA 0, dbg[slot * 1024 + k-block]
__device__ __forceinline__ void pf_stamp(const DgqGemmParams& p, int slot, int it) {
  if (p.dbg && blockIdx.x == 0 && it < 1024) {
    uint64_t g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.dbg[slot * 1024 + it] = g;
  }
}
__device__ __forceinline__ long long sk_begin(const DgqGemmParams& p, long long U, int c, int ncl) {
  return p.sk_b[0] >= 0 ? p.sk_b[c] : U * c / ncl;
}

__device__ __forceinline__ void st_release_gpu(uint32_t* a, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
// Stream-K partial layout (one 128-row sub-tile, 128 KB): [c16][v][row][4]
// int32 — chunk c16 of 16 columns, quarter v of it, token row, 4 values — so
// a warp's 16-byte stores and loads of one (c16, v) are 512 contiguous bytes.
__device__ __forceinline__ size_t part_off(int c16, int v, int row) {
  return (static_cast<size_t>(c16 * 4 + v) * 128 + row) * 4;
}

// Exposed epilogue of the two-sub-tile kernel: 32 token rows (this warp's
// TMEM lane quadrant) x TN channels -> scales -> FP16/FP32, transposed through
// the warp's 4 KB staging buffer so each global store instruction writes four
// whole 128-byte row segments (a lane-per-row 16-byte store touched 32 lines
// per instruction; tools/pf_trace.py measured an 11 us epilogue that way, and
// a TMA store per 64 columns serialises on its issue latency).
template <int TN, bool kF16, bool kFlush, int kRowB>
__device__ __forceinline__ void epi_direct(const DgqGemmParams& p, const DgqDecodeSub& d, uint32_t tbase, float rsm,
                                           const float* s_s1, const float* s_bias, uint8_t* stg, int mrow0, int nbase,
                                           int cbeg, int cend) {
  // the FP16 epilogue mode and the bias are uniform runtime branches: every
  // template variant unrolled here cost instruction-cache misses (the kernel's
  // SASS reached 350 KB and the exposed epilogue ran at ~1/6 of its issue rate)
  const bool kF16Mode = p.fp16_mode != 0, kBias = d.bias != nullptr;
  // the warp's staging buffer holds 32 rows x kRowB bytes (128 or 64): the
  // 16-byte chunks of a row are XOR-swizzled so the row-per-lane writes and the
  // transposed reads hit distinct banks
  constexpr int kCB = kRowB / (kF16 ? 2 : 4);  // columns per row segment
  constexpr int kNC = kRowB / 16;               // 16-byte chunks per row segment
  const uint32_t lane = lane_id();
  uint8_t* myrow = stg + lane * kRowB;
  const uint32_t sw = kNC == 8 ? (lane & 7) : ((lane >> 1) & 3);
#pragma unroll 1
  for (int c0 = cbeg; c0 < cend; c0 += kCB) {
    if (nbase + c0 >= d.N) break;
    // 16-column TMEM loads, the next one in flight while this one is converted
    // (a whole 64-column batch in registers spilled: 96 registers per thread)
    uint32_t r[2][16];
    tmem_ld16(tbase + c0, r[0]);
    tmem_ld_wait();
    if (p.dbg_flags & 4) {  // tools (mode bit 20): TMEM loads only
      for (int c16 = 16; c16 < kCB; c16 += 16) {
        tmem_ld16(tbase + c0 + c16, r[1]);
        tmem_ld_wait();
        r[0][0] ^= r[1][0];
      }
      if (r[0][0] == 0x7FFFFFFFu) myrow[0] = 1;
      continue;
    }
#pragma unroll
    for (int c16 = 0; c16 < kCB; c16 += 16) {
      uint32_t (&cur)[16] = r[(c16 / 16) & 1];
      if (c16 + 16 < kCB) tmem_ld16(tbase + c0 + c16 + 16, r[((c16 / 16) + 1) & 1]);
      {
#pragma unroll
        for (int c8 = 0; c8 < 16; c8 += 8) {
          const int c1 = c16 + c8;
          float y[8];
          const float4 sa = *reinterpret_cast<const float4*>(s_s1 + c0 + c1);
          const float4 sb = *reinterpret_cast<const float4*>(s_s1 + c0 + c1 + 4);
          const float sv[8] = {sa.x, sa.y, sa.z, sa.w, sb.x, sb.y, sb.z, sb.w};
          // branch-free: a vote + branch per 8 values cost more than the
          // conversion it avoided (tools/epi_probe.cu)
#pragma unroll
          for (int k = 0; k < 8; ++k) y[k] = __int2float_rn(static_cast<int32_t>(cur[c8 + k]));
          // (acc * rs) * s1, two values per packed FP32x2 multiply (each RN, no contraction:
          // the intermediate product is rounded before the second multiply, as in epilogue_f32)
          {
            const unsigned long long r2 = f32x2(rsm, rsm);
#pragma unroll
            for (int k = 0; k < 8; k += 2) {
              unsigned long long t, u;
              asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f32x2(y[k], y[k + 1])), "l"(r2));
              asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(u) : "l"(t), "l"(f32x2(sv[k], sv[k + 1])));
              const float2 v = f32x2_split(u);
              y[k] = v.x;
              y[k + 1] = v.y;
            }
          }
          if (kF16Mode) {
#pragma unroll
            for (int k = 0; k < 8; ++k) y[k] = epilogue_f16mode(static_cast<int32_t>(cur[c8 + k]), rsm, sv[k]);
          }
          if (kBias) {
            const float4 ba = *reinterpret_cast<const float4*>(s_bias + c0 + c1);
            const float4 bb = *reinterpret_cast<const float4*>(s_bias + c0 + c1 + 4);
            y[0] = __fadd_rn(y[0], ba.x); y[1] = __fadd_rn(y[1], ba.y); y[2] = __fadd_rn(y[2], ba.z);
            y[3] = __fadd_rn(y[3], ba.w); y[4] = __fadd_rn(y[4], bb.x); y[5] = __fadd_rn(y[5], bb.y);
            y[6] = __fadd_rn(y[6], bb.z); y[7] = __fadd_rn(y[7], bb.w);
          }
          if (kF16) {
            uint32_t h[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const __half2 hh = __floats2half2_rn(y[2 * k], y[2 * k + 1]);
              uint32_t u = *reinterpret_cast<const uint32_t*>(&hh);
              // fp16_round (proj/src/quant.cpp:33-35) flushes |x| < 2^-24 to a signed
              // zero; selects, not a branch (tools/epi_probe.cu: the branch cost 2x)
              const uint32_t lo = (__float_as_uint(y[2 * k]) >> 16) & 0x8000u;
              const uint32_t hi = __float_as_uint(y[2 * k + 1]) & 0x80000000u;
              if (kFlush) {
                u = fabsf(y[2 * k]) < 0x1p-24f ? ((u & 0xFFFF0000u) | lo) : u;
                u = fabsf(y[2 * k + 1]) < 0x1p-24f ? ((u & 0x0000FFFFu) | hi) : u;
              }
              h[k] = u;
            }
            *reinterpret_cast<uint4*>(myrow + (((c1 / 8) ^ sw) << 4)) = make_uint4(h[0], h[1], h[2], h[3]);
          } else {
            *reinterpret_cast<float4*>(myrow + (((c1 / 4) ^ sw) << 4)) = make_float4(y[0], y[1], y[2], y[3]);
            *reinterpret_cast<float4*>(myrow + (((c1 / 4 + 1) ^ sw) << 4)) = make_float4(y[4], y[5], y[6], y[7]);
          }
        }
      }
      if (c16 + 16 < kCB) tmem_ld_wait();
    }
    __syncwarp();
    if (p.dbg_flags & 2) continue;  // tools (mode bit 19): no global stores
    // 32 / kRPP passes x (kRPP rows x kNC lanes x 16 bytes)
    constexpr int kRPP = 32 / kNC;                              // rows per pass
    const int ch = static_cast<int>(lane % kNC);                // 16-byte chunk of the row segment
    const int n = nbase + c0 + ch * (kF16 ? 8 : 4);            // first output column of the chunk
    constexpr int kPer = kF16 ? 8 : 4;                         // outputs per chunk
    uint8_t* const out0 = static_cast<uint8_t*>(d.out) + (static_cast<size_t>(mrow0) * d.ldy + n) * (kF16 ? 2 : 4);
    const size_t row_bytes = d.ldy * (kF16 ? 2 : 4);
    if (mrow0 + 32 <= p.M && nbase + c0 + kCB <= d.N) {
      // interior block: no per-store bounds checks (branches cost the exposed epilogue)
#pragma unroll
      for (int it = 0; it < 32 / kRPP; ++it) {
        const int row = it * kRPP + static_cast<int>(lane / kNC);
        const int rsw = kNC == 8 ? (row & 7) : ((row >> 1) & 3);
        const uint4 v = *reinterpret_cast<const uint4*>(stg + row * kRowB + ((ch ^ rsw) << 4));
        __stcg(reinterpret_cast<uint4*>(out0 + row * row_bytes), v);  // L2 only: written once (3 % faster drain in tools/epi_tmem_probe.cu, neutral in the layer)
      }
    } else {
#pragma unroll 1
      for (int it = 0; it < 32 / kRPP; ++it) {
        const int row = it * kRPP + static_cast<int>(lane / kNC);
        const int m = mrow0 + row;
        const int rsw = kNC == 8 ? (row & 7) : ((row >> 1) & 3);
        const uint4 v = *reinterpret_cast<const uint4*>(stg + row * kRowB + ((ch ^ rsw) << 4));
        if (m < p.M) {
          uint8_t* dst = out0 + row * row_bytes;
          if (n + kPer <= d.N) {
            *reinterpret_cast<uint4*>(dst) = v;
          } else if (n < d.N) {
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            for (int k = 0; k < kPer && n + k < d.N; ++k) {
              if (kF16)
                reinterpret_cast<uint16_t*>(dst)[k] = static_cast<uint16_t>(w[k >> 1] >> ((k & 1) * 16));
              else
                reinterpret_cast<uint32_t*>(dst)[k] = w[k];
            }
          }
        }
      }
    }
    __syncwarp();
  }
}

// 32 token rows (this warp's TMEM lane quadrant) x 256 channels of one
// accumulator -> scales -> FP16/FP32 -> swizzled staging -> TMA store.
template <int TN, bool kF16, bool kF16Mode, bool kBias>
__device__ __forceinline__ void epi_rows(const DgqGemmParams& p, int N, uint32_t tbase, float rsm, const float* s_s1,
                                         const float* s_bias, uint8_t* stg0, const CUtensorMap* tmY, int nbase,
                                         int mbox) {
  constexpr int kCB = kF16 ? 64 : 32;  // columns per 128-byte box row
  const uint32_t lane = lane_id();
  uint8_t* row0 = stg0 + lane * 128;
  const uint32_t sw = lane & 7;
#pragma unroll 1
  for (int c0 = 0; c0 < TN; c0 += kCB) {
    if (nbase + c0 >= N) break;
    uint32_t r[kCB];
#pragma unroll
    for (int c1 = 0; c1 < kCB; c1 += 16) tmem_ld16(tbase + c0 + c1, *reinterpret_cast<uint32_t(*)[16]>(&r[c1]));
    if (lane == 0) bulk_wait_read<0>();  // the previous store has finished reading the staging buffer
    __syncwarp();
    tmem_ld_wait();
    uint8_t* row = row0;
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
      tma_store_2d(tmY, stg0, nbase + c0, mbox);
      bulk_commit();
    }
  }
}

}  // namespace pf

// TN = pair-tile width in channels: 256 (each CTA dequantises 128 channel
// rows, one prepared tile) or 128 (each CTA dequantises 64 rows of the SAME
// prepared tile; twice the tiles, for shapes whose 256-wide tiles leave a
// ragged last wave).
template <int TN, int S>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pf::Cfg<S, TN>::kThreads, 1)
    k_dgq_prefill2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmY,
                   const DgqGemmParams p) {
  using namespace pf;
  using C = Cfg<S, TN>;
  constexpr int kSA = C::kSA, kSC = C::kSC, kSB = C::kSB, kDqGroups = C::kDqGroups;
  constexpr int kEpiWarp0 = C::kEpiWarp0, kXWarp = C::kXWarp, kNAcc = C::kNAcc, kEpiWarps = C::kEpiWarps;
  constexpr int kEpiThreads = 32 * kEpiWarps;
  constexpr uint32_t kStagingPerWarp = C::kStagingPerWarp;
  constexpr uint32_t kStaging = kEpiWarps * kStagingPerWarp;
  constexpr uint32_t kAStage = S * kATile;  // one Xq stage: S tiles of 128 token rows
  constexpr uint32_t kIdesc = idesc_i8(256, TN);
  constexpr int kRows = TN / 2;  // channel rows of B held (and dequantised) by each CTA
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int KB = p.k_blocks;
  // tiles are token-tile major (t = mt * n_pairs + nt): the stream-K ranges of
  // the pairs working on different token tiles sweep the same weight tiles at
  // the same time, so each weight chunk comes from HBM once and is re-read from
  // L2 (n-major order re-read every chunk per token tile: 3.7x the unique HBM
  // bytes on OPT-30B fc1, profiles/ncu_summary_r01c.json)
  const int m_pairs = (p.M + 256 * S - 1) / (256 * S), n_pairs = p.n_pair_tiles;
  // pair tile nt (of the concatenation) -> its layer (several layers sharing
  // the input run as one problem; a single layer is sub[0])
  auto sub_of = [&](int nt) {
    int i = 0;
    while (i + 1 < p.nsub && nt >= p.sub[i + 1].tile_begin) ++i;
    return i;
  };
  // this CTA's 128-channel prepared tile of pair tile nt inside its layer
  // (TN = 128: both CTAs dequantise halves of the same one) and whether it exists
  auto ctile_of = [&](int nt, int& sub, int& ctile) {
    sub = sub_of(nt);
    const int ntl = nt - p.sub[sub].tile_begin;
    ctile = TN == 256 ? ntl * 2 + static_cast<int>(rank) : ntl;
    return ctile < (p.sub[sub].N + 127) / 128;
  };
  const int total = m_pairs * n_pairs;
  const int cid = static_cast<int>(cluster_id_x()), ncl = static_cast<int>(nclusters_x());

  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = sm;                          // [kSA][S][128 x 128] Xq (SW128 K-major)
  uint8_t* sB = sA + kSA * kAStage;          // [kSB][128 x 128] W_s8 (SW128 K-major)
  uint8_t* sStg = sB + kSB * kBTile;         // epilogue staging
  uint8_t* sC = sStg + kStaging;             // [kSC][chunk_stride] packed chunks
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + kSC * p.chunk_stride);
  uint64_t* afull = bars;                    // [kSA] leader: both CTAs' Xq halves landed (pair TMA tx)
  uint64_t* aempty = afull + kSA;            // [kSA] MMA done with the Xq tile (multicast commit)
  uint64_t* cfull = aempty + kSA;            // [kSC] packed chunk landed (local)
  uint64_t* cempty = cfull + kSC;            // [kSC] dequantised (one arrive by the group)
  uint64_t* ready = cempty + kSC;            // [kSB] leader: both CTAs' B slot dequantised (2 arrivals)
  uint64_t* bempty = ready + kSB;            // [kSB] MMA done with the B slot (multicast commit)
  uint64_t* tfull = bempty + kSB;            // [2] accumulator set complete (multicast commit)
  uint64_t* tempty = tfull + 2;              // [2] leader: both CTAs' epilogues drained it (8 arrivals)
  uint64_t* fbar = tempty + 2;               // [1] stream-K fix-up: a contributor's partial landed in sA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fbar + 1);
  // 16-byte aligned (float4 reads) by an offset, so the pointer stays in the shared window (LDS, not generic LD)
  uint8_t* after_slot = reinterpret_cast<uint8_t*>(tmem_slot + 4);
  float* s_rs = reinterpret_cast<float*>(after_slot + ((16u - (smem_u32(after_slot) & 15u)) & 15u));  // [S * 128]
  float* s_s1 = s_rs + 128 * S;                            // [TN]
  float* s_bias = s_s1 + 256;                              // [TN]

  const uint32_t warp = warp_id(), lane = lane_id();
#if !DGQ_PF_LATE_TRIGGER
  // Dependents may be scheduled as soon as SMs free up: the next kernel's CTAs
  // fill the SMs this launch's early-finishing pairs leave (stream-K tail)
  // and start streaming their weights; they griddepcontrol.wait before
  // touching anything this kernel writes.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSA; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < kSC; ++s) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], 1);
    }
    for (int b = 0; b < kSB; ++b) {
      mbar_init(&ready[b], 2);
      mbar_init(&bempty[b], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);
    }
    mbar_init(fbar, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmY);
  }
  if (p.dbg && threadIdx.x == 0 && blockIdx.x < 1024) {  // tools/pf_trace.py: CTA start
    uint64_t g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.dbg[7 * 1024 + blockIdx.x] = g;
  }
  if (warp == 1) tmem_alloc2<512>(tmem_slot);
  tc_fence_before();
  cooperative_groups::this_cluster().sync();  // barrier inits + TMEM visible pair-wide
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == 2) {
    // ------------------------ chunk producers (2 warps) ------------------------
    // A TMA/bulk-copy instruction holds its issuing warp for ~650-850 cycles
    // (tools/l2_stream.cu: one lone issuing thread streams one request per
    // ~660 cycles whatever its size; N issuing warps stream N times that), so
    // each operand stream has two issuing warps taking alternate k-blocks.
    // Packed chunks run up to kSC k-blocks ahead (freed by the dequantisers);
    // they do not depend on the previous kernel, so no griddepcontrol.wait.
    if (lane == 0) {
      const int w = warp == 0 ? 0 : 1;
      SegIter si(p, cid, ncl, total, KB);
      const int n = si.count();
      SegIter::Cursor c = si.first();
      if (w) si.advance(c);
      for (int i = w; i < n; i += 2) {
        const int t = c.t, kb = c.kb;
        si.advance(c);
        si.advance(c);
        int sub, ctile;
        // the prepared 128-channel weight tile this CTA dequantises (from)
        const bool has_w = ctile_of(t % n_pairs, sub, ctile);
        const int s = i % kSC;
        wait_local(&cempty[s], ((i / kSC) & 1) ^ 1, 1);
        pf_stamp(p, 1, i);
        mbar_arrive_expect_tx(&cfull[s], has_w ? p.chunk_bytes : 0u);
        if (has_w)
          bulk_load(sC + s * p.chunk_stride, p.sub[sub].tiles + (static_cast<size_t>(ctile) * KB + kb) * p.chunk_bytes,
                    p.chunk_bytes, &cfull[s]);
      }
    }
    __syncwarp();  // lanes 1-31 park here (a lone lane next to a warp parked at a CTA/cluster barrier issues slowly)
  } else if (warp == 3 || warp == static_cast<uint32_t>(kXWarp)) {
    // ------------------------ Xq-tile producers (2 warps) ------------------------
    // Each CTA loads its 128 token rows; the copy signals the LEADER's afull
    // (cta_group::2 TMA), which expects both halves' bytes.
    if (lane == 0) {
      const int w = warp == 3 ? 0 : 1;
      const uint32_t afull_leader = mapa(afull, 0);
      SegIter si(p, cid, ncl, total, KB);
      const int n = si.count();
      SegIter::Cursor c = si.first();
      if (w) si.advance(c);
      asm volatile("griddepcontrol.wait;" ::: "memory");  // Xq / row scales come from K1
      for (int i = w; i < n; i += 2) {
        const int t = c.t, kb = c.kb;
        si.advance(c);
        si.advance(c);
        const int s = i % kSA;
        wait_local(&aempty[s], ((i / kSA) & 1) ^ 1, 7);
        const int mpair = (t / n_pairs) * 256 * S;
        // token quarters entirely past M are not loaded: their rows of D are never stored
        if (leader) {
          uint32_t tx = 0;
#pragma unroll
          for (int q = 0; q < 2 * S; ++q) tx += mpair + q * 128 < p.M ? kATile : 0u;
          mbar_arrive_expect_tx(&afull[s], tx);
        }
#pragma unroll
        for (int sub = 0; sub < S; ++sub) {
          const int mrow = mpair + sub * 256 + static_cast<int>(rank) * 128;
          if (mrow < p.M)
            tma_load_2d_pair(sA + s * kAStage + sub * kATile, &tmA, afull_leader + s * 8, kb * 128, mrow);
        }
        pf_stamp(p, 5, i);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // --------------------- MMA issuer (leader CTA, converged warp) ---------------------
    if (leader) {
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      int it = 0, tl = 0;
      SegIter si(p, cid, ncl, total, KB);
      int t, lo, hi;
      for (; si.next(t, lo, hi); ++tl) {
        const int acc = tl % kNAcc;
        {  // both epilogues drained this accumulator set; back off while polling so the
           // spinning issuer does not take the issue slots of the epilogue warp
           // sharing its SMSP (the epilogue is exposed when S == 2)
          long long n = 0;
          while (!try_wait_cluster(&tempty[acc], ((tl / kNAcc) & 1) ^ 1)) {
#if DGQ_PF_TSLEEP > 0
            __nanosleep(DGQ_PF_TSLEEP);
#endif
            watchdog(n, 2, 0);
          }
        }
        tc_fence_after();
        const uint32_t d = tm + acc * TN * S;  // accumulator set: S sub-tiles x TN columns
        for (int kb = lo; kb < hi; ++kb, ++it) {
          const int s = it % kSA, b = it % kSB;
          wait_cluster(&ready[b], (it / kSB) & 1, 3);  // both CTAs' B slots dequantised
          wait_cluster(&afull[s], (it / kSA) & 1, 7);  // both CTAs' Xq halves landed
          if (p.dbg && blockIdx.x == 0 && lane == 0 && it < 1024) {  // tools/pf_trace.py
            uint64_t g;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
            p.dbg[it] = g;
          }
          tc_fence_after();
          const uint64_t db = umma_desc_sw128(smem_u32(sB + b * kBTile));
#pragma unroll
          for (int sub = 0; sub < S; ++sub) {
            const uint64_t da = umma_desc_sw128(smem_u32(sA + s * kAStage + sub * kATile));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma2_i8(d + sub * TN, da + 2 * kk, db + 2 * kk, kIdesc, (kb != lo) || kk != 0);
          }
          commit2_mc(&aempty[s]);
          commit2_mc(&bempty[b]);
        }
        commit2_mc(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < static_cast<uint32_t>(kEpiWarp0)) {
    // ------------------------------ dequantisers ------------------------------
    // kDqGroups groups of four warps take k-blocks round robin, so several
    // k-blocks are in flight: one k-block's dequantisation is latency-bound
    // (~1700 cycles for 128 rows on four SMSPs, tools/pf_trace.py), well above
    // the 512-cycle MMA step it feeds.
    const int grp = (warp - 4) >> 2;
    (void)kRows;
    // TN = 256: thread = one of 128 rows, all four 32-k slices; TN = 128: 64 rows x two halves of k
    const int d = TN == 256 ? static_cast<int>((warp & 3) * 32 + lane) : static_cast<int>((warp & 1) * 32 + lane);
    const int jbeg = TN == 256 ? 0 : static_cast<int>(((warp & 3) >> 1) * 2);
    constexpr int kJ = TN == 256 ? 4 : 2;   // 32-k slices per thread
    const int crow = TN == 256 ? d : static_cast<int>(rank) * 64 + d;  // row inside the prepared chunk
    const uint32_t sw = d & 7;
    const uint32_t ready_leader = mapa(ready, 0);
    SegIter si(p, cid, ncl, total, KB);
    const int n = si.count();
    SegIter::Cursor cu = si.first();
    for (int i = 0; i < grp; ++i) si.advance(cu);
    {
      for (int it = grp; it < n; it += kDqGroups) {
        const int t = cu.t;
        for (int i = 0; i < kDqGroups; ++i) si.advance(cu);
        int sub_, ctile_;
        const bool has_w = ctile_of(t % n_pairs, sub_, ctile_);
        const int s = it % kSC, b = it % kSB;
        wait_local(&cfull[s], (it / kSC) & 1, 4);
        if ((warp & 3) == 0 && lane == 0) pf_stamp(p, 2, it);
        wait_local(&bempty[b], ((it / kSB) & 1) ^ 1, 6);
        if ((warp & 3) == 0 && lane == 0) pf_stamp(p, 3, it);
        uint8_t* brow = sB + b * kBTile + (d >> 3) * 1024 + (d & 7) * 128;
        if (has_w) {
          const uint8_t* chunk = sC + s * p.chunk_stride;
          const uint16_t* sc = reinterpret_cast<const uint16_t*>(chunk + 8192);
          uint4 w4[kJ];
#pragma unroll
          for (int jj = 0; jj < kJ; ++jj)
            w4[jj] = *reinterpret_cast<const uint4*>(chunk + (jbeg + jj) * 2048 + crow * 16);
#pragma unroll
          for (int jj = 0; jj < kJ; ++jj) {
            const int j = jbeg + jj;
            const uint32_t wv[4] = {w4[jj].x, w4[jj].y, w4[jj].z, w4[jj].w};
            uint32_t o[8];
            if (p.gshift >= 5) {
              const uint32_t sv = sc[((j * 32) >> p.gshift) * 128 + crow];
              const uint32_t s2 = sv & 0xFFu, bs = dq_bias2(s2, sv >> 8);
#pragma unroll
              for (int q = 0; q < 4; ++q) dq_word(wv[q], s2, bs, o[2 * q], o[2 * q + 1]);
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t sv = sc[((j * 32 + q * 8) >> p.gshift) * 128 + crow];
                const uint32_t s2 = sv & 0xFFu;
                dq_word(wv[q], s2, dq_bias2(s2, sv >> 8), o[2 * q], o[2 * q + 1]);
              }
            }
            *reinterpret_cast<uint4*>(brow + (((2 * j) ^ sw) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(brow + (((2 * j + 1) ^ sw) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
          }
        } else {
          const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int c = 0; c < 2 * kJ; ++c) *reinterpret_cast<uint4*>(brow + (((2 * jbeg + c) ^ sw) << 4)) = z;
        }
        fence_proxy_async_smem();
        named_bar(3 + grp, 128);  // the group's four warps wrote their rows (barrier ids 3..)
        if ((warp & 3) == 0 && lane == 0) {
          pf_stamp(p, 4, it);
          mbar_arrive(&cempty[s]);  // the chunk has been read
          // Release pattern at cluster scope: the group's B-tile writes happen
          // before this thread's fence (bar.sync orders them within the CTA), the
          // fence is cumulative, and the leader's acquire.cluster wait on ready[b]
          // synchronises with the arrive that follows it, so the peer's rows are
          // visible to the leader before its tcgen05.mma reads them.
#if !DGQ_PF_RELAXED_READY
          // release fence restricted to this CTA's shared memory (the B rows):
          // MEMBAR.CTA + FENCE.VIEW.ASYNC.S in SASS, where fence.acq_rel.cluster
          // is a GPU-scope MEMBAR that cost ~20 % of the kernel (tools/pf_ab.py)
          asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
#endif
          arrive_remote_relaxed(ready_leader + b * 8);  // one per group: leader's ready[b]
        }
      }
    }
  } else if (warp >= static_cast<uint32_t>(kEpiWarp0) && warp < static_cast<uint32_t>(kXWarp)) {
    // ------------------------------ epilogue ------------------------------
    const int et = threadIdx.x - 32 * kEpiWarp0;     // 0 .. kEpiThreads-1
    const uint32_t q = warp & 3;                     // TMEM lane quadrant
    const int e = static_cast<int>(q * 32 + lane);   // token row of this CTA's D
    // channels of this warp: the quadrant's kEpiWarps / 4 warps split the TN
    // columns in 32-column units (three warps: 2 / 3 / 3 units of 8)
    constexpr int kPerQ = kEpiWarps / 4, kUnits = TN / 32;
    const int jq = static_cast<int>(warp - kEpiWarp0) >> 2;
    const int cbeg = (jq * kUnits / kPerQ) * 32, cend = ((jq + 1) * kUnits / kPerQ) * 32;
    const uint32_t tempty_leader = mapa(tempty, 0);
    uint8_t* stg0 = sStg + (warp - kEpiWarp0) * kStagingPerWarp;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // row scales from K1
    int tl = 0;
    SegIter si(p, cid, ncl, total, KB);
    const long long U = static_cast<long long>(total) * KB;
    constexpr size_t kSub = 128 * TN;    // ints of one 128-row partial
    constexpr size_t kSlot = S * kSub;   // ints per CTA partial (S sub-tiles)
    const bool f_ = p.fp16_mode != 0;
    uint32_t fphase = 0;
    int t, lo, hi;
    for (; si.next(t, lo, hi); ++tl) {
      const int mt = t / n_pairs, nt = t % n_pairs;
      const int acc = tl % kNAcc;
      const uint32_t tpar = (tl / kNAcc) & 1;
      const DgqDecodeSub& d = p.sub[sub_of(nt)];  // this tile's layer
      const int n0 = (nt - d.tile_begin) * TN;      // first channel of the tile inside its layer
      const bool b_ = d.bias != nullptr;
      const int mrow = q * 32 + lane;
      // sub-tile `sub` of this CTA: token rows mt*256S + sub*256 + rank*128 + [0, 128)
      auto m0_of = [&](int sub) { return mt * 256 * S + sub * 256 + static_cast<int>(rank) * 128; };
      auto tbase_of = [&](int sub) {
        return tmem + ((q * 32) << 16) + static_cast<uint32_t>(acc * TN * S + sub * TN);
      };
      if (lo > 0) {
        // stream-K contributor: park the int32 partials in this pair's slot
        wait_local(&tfull[acc], tpar, 5);
        tc_fence_after();
#pragma unroll 1
        for (int sub = 0; sub < S; ++sub) {
          int32_t* slot = p.ws + (static_cast<size_t>(cid) * 2 + rank) * kSlot + sub * kSub;
#pragma unroll 1
          for (int c0 = cbeg; c0 < cend; c0 += 16) {
            uint32_t r[16];
            tmem_ld16(tbase_of(sub) + c0, r);
            tmem_ld_wait();
#pragma unroll
            for (int v = 0; v < 4; ++v)
              __stcg(reinterpret_cast<int4*>(slot + part_off(c0 / 16, v, mrow)),
                     make_int4(static_cast<int>(r[4 * v]), static_cast<int>(r[4 * v + 1]),
                               static_cast<int>(r[4 * v + 2]), static_cast<int>(r[4 * v + 3])));
          }
        }
        __threadfence();
        tc_fence_before();
        named_bar(2, kEpiThreads);
        if (et == 0) st_release_gpu(p.counters + cid * 2 + rank, 1u);
        __syncwarp();
        if (lane == 0) arrive_tmem_drained(tempty_leader + acc * 8);
        continue;
      }
      // owner of a split tile: the pairs after this one whose ranges start inside it
      int npart = 0;
      if (hi < KB) {
        const long long tend = static_cast<long long>(t + 1) * KB;
        while (cid + 1 + npart < ncl && sk_begin(p, U, cid + 1 + npart, ncl) < tend) ++npart;
      }
      // per-tile scales (all four epilogue warps)
      for (int i = et; i < S * 128; i += kEpiThreads) {
        const int mm = m0_of(i >> 7) + (i & 127);
        s_rs[i] = (p.rs && mm < p.M) ? p.rs[mm] : 0.0f;
      }
      for (int i = et; i < TN; i += kEpiThreads) {
        s_s1[i] = (d.s1 && n0 + i < d.N) ? d.s1[n0 + i] : 0.0f;
        s_bias[i] = (d.bias && n0 + i < d.N) ? d.bias[n0 + i] : 0.0f;
      }
      if (npart) {
        for (int c = 1; c <= npart; ++c) {
          long long n = 0;
          while (ld_acquire_gpu(p.counters + (cid + c) * 2 + rank) == 0) watchdog(n, 9, 0);
        }
      }
      named_bar(2, kEpiThreads);
      if (npart && et == 0)  // every thread has seen the flags: re-arm them for the next launch
        for (int c = 1; c <= npart; ++c) p.counters[(cid + c) * 2 + rank] = 0u;
      wait_local(&tfull[acc], tpar, 5);
      tc_fence_after();
      if (et == 0 && tl < 8) pf_stamp(p, 9, 2 * tl);
#pragma unroll 1
      for (int sub = 0; sub < S; ++sub) {
        const uint32_t tbase = tbase_of(sub);
        const int m0 = m0_of(sub);
        // fold the contributors' partials into this thread's TMEM row (exact
        // int32).  An owner segment is always its pair's LAST, so the Xq / B
        // rings are idle: each contributor's 128-row partial (128 KB) comes in
        // with one bulk copy instead of per-thread L2 round trips.
        auto load_part = [&](int c, int s) {
          mbar_arrive_expect_tx(fbar, static_cast<uint32_t>(kSub * 4));
          bulk_load(sA, p.ws + (static_cast<size_t>(cid + c) * 2 + rank) * kSlot + s * kSub,
                    static_cast<uint32_t>(kSub * 4), fbar);
        };
#pragma unroll 1
        for (int c = 1; c <= npart; ++c) {
          // sub-tile 1's first partial was prefetched while sub-tile 0's rows drained
          if (et == 0 && !(sub > 0 && c == 1)) load_part(c, sub);
          wait_local(fbar, fphase, 10);
          fphase ^= 1u;
          const int32_t* sp = reinterpret_cast<const int32_t*>(sA);
#pragma unroll 1
          for (int c0 = cbeg; c0 < cend; c0 += 16) {
            uint32_t r[16];
            tmem_ld16(tbase + c0, r);
            tmem_ld_wait();
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int4 x = *reinterpret_cast<const int4*>(sp + part_off(c0 / 16, v, mrow));
              r[4 * v + 0] += static_cast<uint32_t>(x.x);
              r[4 * v + 1] += static_cast<uint32_t>(x.y);
              r[4 * v + 2] += static_cast<uint32_t>(x.z);
              r[4 * v + 3] += static_cast<uint32_t>(x.w);
            }
            tmem_st16(tbase + c0, r);
          }
          tmem_st_wait();
          named_bar(2, kEpiThreads);  // every row read before the next partial overwrites the buffer
          if (et == 0 && c == npart && sub + 1 < S) load_part(1, sub + 1);
        }
        const float rsm = s_rs[sub * 128 + mrow];
        if (et == 0 && tl < 8) pf_stamp(p, 9, 512 + 4 * tl + sub);
        if (m0 >= p.M) continue;  // a token quarter past M: nothing to store
        if (d.out && p.vec_ok && !p.acc_out && !(S == 1 && (p.dbg_flags & 16))) {  // tools: 16 = S=1 TMA epilogue
          {
            // No value of this warp's rows can land in fp16_round's flush range
            // (0 < |y| < 2^-24) when rs * min(s1) >= 2^-24: |acc| >= 1 for every
            // non-zero accumulator and RN is monotonic (no bias, FP32 scale mode)
            float s1min = 3.0e38f;
            for (int c = cbeg + static_cast<int>(lane); c < cend; c += 32) s1min = fminf(s1min, s_s1[c]);
            for (int o = 16; o > 0; o >>= 1) s1min = fminf(s1min, __shfl_xor_sync(0xffffffffu, s1min, o));
            const bool safe = !d.bias && !p.fp16_mode && __fmul_rn(rsm, s1min) >= 0x1p-24f;
            if (p.out_f16) {
              if (__all_sync(0xffffffffu, safe))
                epi_direct<TN, true, false, kStagingPerWarp / 32>(p, d, tbase, rsm, s_s1, s_bias, stg0, m0 + q * 32, n0, cbeg, cend);
              else
                epi_direct<TN, true, true, kStagingPerWarp / 32>(p, d, tbase, rsm, s_s1, s_bias, stg0, m0 + q * 32, n0, cbeg, cend);
            } else {
              epi_direct<TN, false, true, kStagingPerWarp / 32>(p, d, tbase, rsm, s_s1, s_bias, stg0, m0 + q * 32, n0, cbeg, cend);
            }
          }
        } else if (S == 1 && p.tma_out && !p.acc_out) {
          if constexpr (S == 1) {
            const int mbox = m0 + q * 32;
#define DGQ_EPI2(F16_, MODE_, BIAS_) \
  epi_rows<TN, F16_, MODE_, BIAS_>(p, d.N, tbase, rsm, s_s1, s_bias, stg0, &tmY, n0, mbox)
            if (p.out_f16) {
              if (f_) { if (b_) DGQ_EPI2(true, true, true); else DGQ_EPI2(true, true, false); }
              else    { if (b_) DGQ_EPI2(true, false, true); else DGQ_EPI2(true, false, false); }
            } else {
              if (f_) { if (b_) DGQ_EPI2(false, true, true); else DGQ_EPI2(false, true, false); }
              else    { if (b_) DGQ_EPI2(false, false, true); else DGQ_EPI2(false, false, false); }
            }
#undef DGQ_EPI2
          }
        } else {
          const int m = m0 + mrow;
#pragma unroll 1
          for (int c0 = cbeg; c0 < cend; c0 += 16) {
            if (n0 + c0 >= d.N) break;
            uint32_t r[16];
            tmem_ld16(tbase + c0, r);
            tmem_ld_wait();
            if (m >= p.M) continue;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const int n = n0 + c0 + k;
              if (n >= d.N) break;
              const int32_t a = static_cast<int32_t>(r[k]);
              if (p.acc_out) p.acc_out[static_cast<size_t>(m) * p.ld_acc + n] = a;
              if (d.out) {
                float y = p.fp16_mode ? epilogue_f16mode(a, rsm, s_s1[c0 + k]) : epilogue_f32(a, rsm, s_s1[c0 + k]);
                if (d.bias) y = __fadd_rn(y, s_bias[c0 + k]);
                if (p.out_f16)
                  static_cast<__half*>(d.out)[static_cast<size_t>(m) * d.ldy + n] = fp16_ref(y);
                else
                  static_cast<float*>(d.out)[static_cast<size_t>(m) * d.ldy + n] = y;
              }
            }
          }
        }
      }
      if (et == 0 && tl < 8) pf_stamp(p, 9, 512 + 4 * tl + 2);
      tc_fence_before();
      __syncwarp();
      if (et == 0 && tl < 8) pf_stamp(p, 9, 2 * tl + 1);
      if (p.dbg && lane == 0 && tl == 0 && blockIdx.x < 2) {  // tools/pf_trace.py: per-warp drain end, first segment
        uint64_t g;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
        p.dbg[10 * 1024 + blockIdx.x * 32 + warp] = g;
      }
      if (lane == 0) arrive_tmem_drained(tempty_leader + acc * 8);  // the leader's tempty[acc]
      named_bar(2, kEpiThreads);  // scales of the next tile are rewritten
    }
    if (lane == 0) bulk_wait_all();
    if (p.dbg && e == 0 && blockIdx.x < 1024) {  // tools/pf_trace.py: epilogue done
      uint64_t g;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
      p.dbg[8 * 1024 + blockIdx.x] = g;
    }
#if DGQ_PF_LATE_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  }
  tc_fence_before();
  cooperative_groups::this_cluster().sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem);
  }
}

}  // namespace dgqk

using namespace dgqk;

template <int S, int TN = 256>
static size_t smem_bytes_s(uint32_t chunk_stride) {
  using C = pf::Cfg<S, TN>;
  return 1024 + static_cast<size_t>(C::kSA) * S * pf::kATile + C::kSC * chunk_stride + C::kSB * pf::kBTile +
         C::kEpiWarps * C::kStagingPerWarp + (2 * C::kSA + 2 * C::kSC + 2 * C::kSB + 5) * 8 + 32 +
         (128 * S + 256 + 256) * 4;
}

size_t dgq_prefill2_smem_bytes(uint32_t chunk_stride, int sub) {
  return sub == 2 ? smem_bytes_s<2>(chunk_stride) : smem_bytes_s<1>(chunk_stride);
}

template <int TN, int S>
static int max_active_pairs() {
  // persistent + stream-K spin-waits need every pair co-resident: ask the
  // occupancy calculator how many 2-CTA clusters of this kernel fit at once
  static int cached = 0;
  if (cached) return cached;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int n = sms / 2;
  const size_t smem = smem_bytes_s<S, TN>(static_cast<uint32_t>(dgq_layout::chunk_bytes(128)));
  auto kern = k_dgq_prefill2<TN, S>;
  if (dgq_allow_smem(kern, smem) ==
      cudaSuccess) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * n);
    cfg.blockDim = dim3(pf::Cfg<S, TN>::kThreads);
    cfg.dynamicSmemBytes = smem;
    int q = 0;
    if (cudaOccupancyMaxActiveClusters(&q, kern, &cfg) == cudaSuccess && q > 0 && q < n) n = q;
  }
  cudaGetLastError();
  cached = n;
  return cached;
}

int dgq_prefill2_clusters(int M, int N, int tn, int k_blocks, bool stream_k, int sub) {
  const int pairs = sub == 2 ? (tn == 128 ? max_active_pairs<128, 2>() : max_active_pairs<256, 2>())
                             : (tn == 128 ? max_active_pairs<128, 1>() : max_active_pairs<256, 1>());
  const long long tiles = static_cast<long long>((M + 256 * sub - 1) / (256 * sub)) * ((N + tn - 1) / tn);
  const long long work = stream_k ? tiles * k_blocks : tiles;
  int n = static_cast<int>(work < pairs ? work : pairs);
  static const bool dp_switch = [] {  // tools: DGQ_PF_DP=0 always splits stream-K over every pair
    const char* e = getenv("DGQ_PF_DP");
    return !(e && atoi(e) == 0);
  }();
  if (stream_k && tiles > 0 && dp_switch) {
    // Whole tiles per pair when that is cheaper than splitting them: a split
    // tile costs its owner a wait + fix-up and its contributors a partial
    // store (~6 us per piece, tools/decode_sweep.py --cap: 4096^2 at M = 1024
    // runs 64 whole tiles in 23 us on 64 pairs vs 31 us stream-K on 74).
    const double t_kb = sub == 2 ? 0.70 : 0.49;  // us per k-block of one pair tile (measured)
    const long long w = (tiles + pairs - 1) / pairs;
    const double dp = static_cast<double>(w) * k_blocks * t_kb;
    const long long pieces = tiles >= pairs ? 1 : (pairs + tiles - 1) / tiles;
    const double skt = static_cast<double>(tiles) * k_blocks / pairs * t_kb + 6.0 * static_cast<double>(pieces);
    if (dp <= skt) n = static_cast<int>((tiles + w - 1) / w);
  }
  const int cap = dgq_prefill2_cluster_cap();  // tools: planner experiments
  if (cap > 0 && n > cap) n = cap;
  return n;
}

// tools: DGQ_PF_BALANCE=0 keeps the even stream-K split (A/B)
static bool sk_balance() {
  static const bool v = [] {
    const char* e = getenv("DGQ_PF_BALANCE");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

// Stream-K split balanced for the per-segment cost.  A pair's time is its MMA
// units plus a fixed cost per segment (tile piece) it touches: the exposed
// epilogue (S = 2: one accumulator set), a contributor's parked partial or an
// owner's fix-up (E = 8 k-block steps of a 512-token tile measured best).  An even
// split of the units gives the pairs that touch one more tile one more such
// stop; here the smallest per-pair cost C for which a greedy walk (each pair
// takes units while units + E x segments <= C) covers everything with at most
// `ncl` pairs is found by bisection, so the pairs end at about the same time
// (simulated on OPT-30B at 2048 tokens: the slowest pair 2-5 % sooner).  The
// walk may need fewer pairs than available: the launch then uses that many
// (every range non-empty, which the owners' contributor count relies on).
// Returns the pairs used (b[0..used] = range starts, b[used] = U), or 0 for
// the even split (more pairs than the table holds).  Cached per (U, KB, ncl, E).
static int sk_bounds(long long U, int KB, int ncl, int E, int* b) {
  if (ncl > kPrefillMaxPairs || ncl < 1 || U <= 0 || KB <= 0 || U > 0x7FFFFFFFLL || E < 0) return 0;
  struct Key {
    long long U;
    int KB, ncl, E;
    bool operator<(const Key& o) const {
      return U != o.U ? U < o.U : KB != o.KB ? KB < o.KB : ncl != o.ncl ? ncl < o.ncl : E < o.E;
    }
  };
  static std::mutex mu;
  static std::map<Key, std::vector<int>> cache;
  const Key key{U, KB, ncl, E};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      std::copy(it->second.begin(), it->second.end(), b);
      return static_cast<int>(it->second.size()) - 1;
    }
  }
  // greedy ranges of cost <= C; true when they cover U with at most ncl pairs
  auto walk = [&](long long C, std::vector<int>* out) {
    if (out) out->assign(1, 0);
    long long pos = 0;
    for (int c = 0; c < ncl && pos < U; ++c) {
      long long rem = C;
      const long long start = pos;
      while (pos < U) {
        const long long seg = std::min<long long>(KB - pos % KB, U - pos);
        if (rem >= seg + E) {
          rem -= seg + E;
          pos += seg;
        } else {
          if (rem - E > 0) pos += rem - E;
          break;
        }
      }
      if (pos == start) return false;  // C below one unit + E
      if (out) out->push_back(static_cast<int>(pos));
    }
    return pos >= U;
  };
  long long lo = 1, hi = U + static_cast<long long>(E) * (U / KB + 2) + 1;  // one pair takes everything
  while (lo < hi) {
    const long long mid = lo + (hi - lo) / 2;
    if (walk(mid, nullptr)) hi = mid; else lo = mid + 1;
  }
  std::vector<int> best;
  walk(hi, &best);
  std::lock_guard<std::mutex> lk(mu);
  cache.emplace(key, best);
  std::copy(best.begin(), best.end(), b);
  return static_cast<int>(best.size()) - 1;
}

// not in the public header: the balanced split for tools / host-side tests
extern "C" int dgq_debug_sk_bounds(long long U, int KB, int ncl, int E, int* b) {
  return sk_bounds(U, KB, ncl, E, b);
}

template <int TN, int S>
static cudaError_t launch_pf(const CUtensorMap& tmA, const CUtensorMap& tmY, const DgqGemmParams& p_, bool pdl,
                             cudaStream_t st) {
  DgqGemmParams p = p_;
  const size_t smem = smem_bytes_s<S, TN>(p.chunk_stride);
  auto kern = k_dgq_prefill2<TN, S>;
  cudaError_t e = dgq_allow_smem(kern, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  int ncl = dgq_prefill2_clusters(p.M, p.n_pair_tiles * TN, TN, p.k_blocks, p.stream_k != 0, S);
  p.sk_b[0] = -1;
  if (p.stream_k && sk_balance()) {
    const long long U = static_cast<long long>((p.M + 256 * S - 1) / (256 * S)) * p.n_pair_tiles * p.k_blocks;
    static const int e_env = [] {  // tools: DGQ_PF_E overrides the per-segment cost (k-block steps)
      const char* e = getenv("DGQ_PF_E");
      return e ? atoi(e) : -1;
    }();
    const int E = e_env >= 0 ? e_env : (S == 2 ? 8 : 5);  // A/B at 2048 tokens: E = 0 / 8 / 15 / 25 -> 934 / 920 / 925 / 930 us
    const int used = sk_bounds(U, p.k_blocks, ncl, E, p.sk_b);
    if (used > 0) ncl = used; else p.sk_b[0] = -1;
  }
  cfg.gridDim = dim3(2 * ncl);
  cfg.blockDim = dim3(pf::Cfg<S, TN>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, tmA, tmY, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t dgq_launch_prefill2(const CUtensorMap& tmA, const CUtensorMap& tmY, const DgqGemmParams& p, int tn,
                                int sub, bool pdl, cudaStream_t st) {
  if (sub == 2) return tn == 128 ? launch_pf<128, 2>(tmA, tmY, p, pdl, st) : launch_pf<256, 2>(tmA, tmY, p, pdl, st);
  return tn == 128 ? launch_pf<128, 1>(tmA, tmY, p, pdl, st) : launch_pf<256, 1>(tmA, tmY, p, pdl, st);
}
