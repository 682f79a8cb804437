// Internal launch interface between the C-ABI layer (capi.cu) and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

// ---- prepared ("B200-tiled") weight layout ---------------------------------
// Output channels are cut into 128-row tiles, the reduction axis into 128-wide
// k-blocks.  Every (n-tile, k-block) owns one contiguous chunk in HBM:
//   [0, 8192)            packed INT4 codes: for j in 0..3 (32-k slice), for n in
//                        0..127: 16 B = 4 words of 8 k each.  Inside a word the
//                        k-offset t sits in nibble kNibblePos[t]: byte j holds
//                        k = j (low nibble) and k = j + 4 (high nibble), so
//                        `w & 0x0F0F0F0F` / `(w >> 4) & 0x0F0F0F0F` are the
//                        raw codes of k 0..3 / 4..7 in order (decode kernel),
//                        and the IMAD/PRMT dequantiser (dequant.cuh) pairs
//                        16-bit lanes (k0,k2)+(k1,k3) and (k4,k6)+(k5,k7).
//   [8192, 8192+256*gpk) per-group scales: for each group overlapping the
//                        k-block, 128 x u16 (S2 | ZP << 8).
// Chunks are ordered n-tile major so one CTA streams a contiguous range.
namespace dgq_layout {
constexpr int kTileN = 128;
constexpr int kBlockK = 128;
constexpr int kCodeBytes = 8192;
constexpr int kNibblePos[8] = {0, 2, 4, 6, 1, 3, 5, 7};
inline int groups_per_kblock(int g) { return g >= kBlockK ? 1 : kBlockK / g; }
inline int chunk_bytes(int g) { return kCodeBytes + 256 * groups_per_kblock(g); }
// The fused path needs every 8-k word inside one group and whole groups per
// k-block (or whole k-blocks per group).
inline bool fused_ok(int g) {
  return g > 0 && g % 8 == 0 && ((kBlockK % g == 0) || (g % kBlockK == 0));
}
}  // namespace dgq_layout

// Layers that share one input (e.g. q / k / v) and run as ONE stream-K
// problem over the concatenation of their weight tiles: K5d (decode.cu, up to
// kDecodeMaxSub layers) and K5p (prefill.cu).  tile_begin = the layer's first
// tile of the concatenation (K5d: 128-channel tiles; K5p: pair tiles).
constexpr int kDecodeMaxSub = 4;
constexpr int kPrefillMaxPairs = 128;  // K5p pairs with a launcher-balanced stream-K split
struct DgqDecodeSub {
  const uint8_t* tiles;
  const float* s1;
  const float* bias;
  void* out;
  size_t ldy;
  int N;
  int tile_begin;  // first global tile of this layer
};

struct DgqGemmParams {
  // A side (weights): prepared INT4 tiles (fused) or via tensor map (plain int8)
  const uint8_t* tiles;
  uint32_t chunk_bytes;
  uint32_t chunk_stride;  // smem bytes per staged chunk
  uint32_t gshift;        // k-offset >> gshift = group index inside a k-block
  int M, N, k_blocks, kb_per_split, splits;
  // epilogue
  const float* rs;    // [M] per-token scales
  const float* s1;    // [N] per-channel scales (may be null when out == null)
  const float* bias;  // [N] or null
  void* out;          // [M x ldy] f32 or f16, or null
  size_t ldy;
  int out_f16;
  int fp16_mode;
  int vec_ok;  // 16-byte aligned rows: vector epilogue stores allowed
  int tma_out; // prefill orientation: output written by TMA tensor stores (tmY)
  int32_t* acc_out;  // optional raw int32 accumulators [M x ld_acc]
  size_t ld_acc;
  // split-K workspace (zero on entry, left zero on exit)
  int32_t* ws;
  size_t ldw;
  uint32_t* counters;
  unsigned long long* dbg;  // optional phase timestamps [cta][8] (debug builds of tools/)
  int stream_k;             // K5p: stream-K over (tile, k-block) units (ws / counters = pair slots / flags)
  int dbg_flags;            // tools only (K5p): 16 = 256-token tiles keep the TMA-store epilogue
  // K5p: the layers of the launch (nsub >= 1; a single layer is sub[0]) and
  // the total number of TN-wide pair tiles over all of them
  int nsub;
  int n_pair_tiles;
  DgqDecodeSub sub[kDecodeMaxSub];
  // K5p stream-K: first unit of each pair's range (sk_b[ncl] = total units),
  // balanced by the launcher for the per-segment cost; sk_b[0] < 0: even split
  int sk_b[kPrefillMaxPairs + 1];
};

struct DgqDecodeParams {
  int nsub;  // number of layers (1 = the single-layer fields below are mirrored in sub[0])
  DgqDecodeSub sub[kDecodeMaxSub];
  const uint8_t* tiles;
  uint32_t chunk_bytes;
  uint32_t chunk_stride;
  int gpk;     // groups per k-block: 1 (g >= 128), 2 (g = 64), 4 (g = 32)
  int gshift;  // log2(g) for g < 128, else 7
  int sd_log2; // log2 of the TMEM partial slots (<= 8 slots)
  int ku;      // units (k-blocks of one tile) per pipeline stage, <= dgq_decode_units_per_stage
  int M, N, n_tiles, k_blocks;
  const float* rs;
  const float* s1;
  const float* bias;
  void* out;
  size_t ldy;
  int out_f16;
  int fp16_mode;
  int32_t* acc_out;
  size_t ld_acc;
  int32_t* ws;         // [n_tiles][bn][128] int32, zero on entry and exit
  uint32_t* counters;  // [n_tiles], zero on entry and exit
  int dbg;             // tools only: bit0 skip MMA, bit1 skip unpack, bit2 skip epilogue math
  unsigned long long* trace;  // tools only: [4 roles][1024 units] globaltimer stamps of CTA `trace_cta`
  int trace_cta;
  int pre_stages;  // stages whose weights are requested before griddepcontrol.wait (>= 1)
};
int dgq_decode_partial_cols();  // TMEM columns K5d keeps for its partial ring
size_t dgq_decode_smem_bytes(int bn, int sl, uint32_t chunk_stride);
int dgq_decode_stages(int bn);            // units of shared-memory ring (stages x units per stage)
int dgq_decode_units_per_stage(int bn);   // box depth of the 3-D Xq tensor map
cudaError_t dgq_launch_decode(int bn, const CUtensorMap& tmB, const DgqDecodeParams& p, int grid, bool pdl,
                              cudaStream_t st);

struct DgqGemmPlan {
  int decode;    // 1: K5d (decode.cu) with token tile bn, `ctas` persistent CTAs
  int prefill2;  // 1: K5p (prefill.cu), persistent CTA pairs, 256 x `pair_tn` tiles
  int pair_tn;   // 256 or 128 channels per pair tile
  int stream_k;  // K5p: stream-K work split (workspace = ws_bytes + counter_bytes)
  int pair_sub;  // K5p: token sub-tiles per CTA (pair tile = 256 * pair_sub tokens)
  int ctas;
  int bn;
  int nt;  // 128-row weight tiles per CTA
  int m_tiles, n_tiles, splits, kb_per_split;
  size_t smem_bytes;
  size_t ws_bytes;       // split-K accumulator bytes needed (0 if splits == 1)
  size_t counter_bytes;  // split-K tile counters
  double est_cycles;     // planner's cost-model estimate
  int pdl;               // launch with programmatic stream serialisation
};

DgqGemmPlan dgq_plan_gemm(int M, int N, int K_pad, bool fused, int g, int force_bn = 0, int force_splits = 0);

// K5p (prefill.cu): persistent CTA-pair kernel; tmA = Xq with 128-row boxes.
// sub = token sub-tiles per CTA (1: 256-token pair tiles, 2: 512-token pair tiles)
size_t dgq_prefill2_smem_bytes(uint32_t chunk_stride, int sub);
int dgq_prefill2_clusters(int M, int N, int tn, int k_blocks, bool stream_k, int sub);
int dgq_prefill2_cluster_cap();  // tools: debug cap on K5p pairs (0 = none)
// stream-K workspace: per pair two CTA partials of up to 2 x 128 x 256 int32, + flags
constexpr size_t kPrefill2SlotBytes = 2 * 2 * 128 * 256 * 4;
cudaError_t dgq_launch_prefill2(const CUtensorMap& tmA, const CUtensorMap& tmY, const DgqGemmParams& p, int tn,
                                int sub, bool pdl, cudaStream_t st);

cudaError_t dgq_launch_gemm(const DgqGemmPlan& plan, bool fused, const CUtensorMap& tmB, const CUtensorMap& tmA,
                            const CUtensorMap& tmY, const DgqGemmParams& p, cudaStream_t st);

// K1 v2 (f32 or f16 input; f16 may be the all-gathered [p][M][seg] layout);
// rk = RN(1/k) per input channel (dgq_launch_reciprocal).
cudaError_t dgq_launch_actquant2(const void* X, bool f16, size_t ldx, int seg, size_t seg_stride, const float* k,
                                 const float* rk, int K, int Kpad, int dynamic, float act_scale, int8_t* Q, size_t ldq,
                                 float* rs, int M, cudaStream_t st,
                                 const uint8_t* ksm = nullptr,  // ksm[c] bit t: k[8c + t] != 1
                                 const int* spec = nullptr,     // the channels with k != 1, ascending
                                 int nspec = 0);
cudaError_t dgq_launch_reciprocal(const float* k, float* rk, int n, cudaStream_t st);
cudaError_t dgq_launch_div_check(const float* x, const float* k, float* fast, float* ieee, int n, cudaStream_t st);

// Two-phase grid search (csrc/search.cu).  Scratch: mn/mx [n_g x o] floats,
// ref [n_g x o x b] doubles, err [n_g x o x n_alpha] doubles (phase 1);
// absmax [o] floats, ref [o x b], err [o x n_alpha] doubles (phase 2).
cudaError_t dgq_launch_phase1(const float* W, const float* X, const float* Xhat, int h, int o, int b, int g,
                              int levels, const float* alpha, int n_alpha, float* mn, float* mx, double* ref,
                              double* err, float* sp, int32_t* zp, float* err_out, float* alpha_out,
                              cudaStream_t st);
cudaError_t dgq_launch_phase2(const float* W, const float* X, const float* Xhat, int h, int o, int b, int g,
                              const float* sp, const int32_t* zp, const float* alpha, int n_alpha, float* absmax,
                              double* ref, double* err, float* s1, int8_t* s2, int32_t* codes, double* col_err,
                              float* col_alpha, cudaStream_t st);

// Dense INT8 tensor peak microbenchmark (csrc/peak.cu): `pairs` SM pairs, each
// issuing `blocks` x 4 tcgen05.mma.cta_group::2.kind::i8 of 256 x 256 x 32.
cudaError_t dgq_launch_i8_peak(int pairs, int blocks, unsigned long long* sink, cudaStream_t st);

// NVTX range around a C-ABI entry point (visible in Nsight Systems / ncu
// --nvtx; a few tens of ns per call when no tool is attached).
#include <nvtx3/nvToolsExt.h>
struct DgqNvtxRange {
  explicit DgqNvtxRange(const char* name) { nvtxRangePushA(name); }
  ~DgqNvtxRange() { nvtxRangePop(); }
};
#define DGQ_NVTX(name) DgqNvtxRange dgq_nvtx_range_(name)

// Raise a kernel's dynamic shared-memory limit to the device's opt-in maximum,
// once per (kernel, device) under a lock, so concurrent launches of one
// instantiation with different sizes never shrink each other's limit.
// cudaErrorInvalidValue when `bytes` exceeds the opt-in maximum.
cudaError_t dgq_allow_smem(const void* kernel, size_t bytes);
template <typename F>
inline cudaError_t dgq_allow_smem(F* kernel, size_t bytes) {
  return dgq_allow_smem(reinterpret_cast<const void*>(kernel), bytes);
}

// Reference layout (codes u4 [h x o_full] packed along o, s2 i8, zp u4) column
// slice [c0, c0+n) -> prepared tiles.
cudaError_t dgq_launch_repack(const uint8_t* codes, const int8_t* s2, const uint8_t* zp, int h, int o_full, int g,
                              int c0, int n, int n_tiles, int k_blocks, uint8_t* tiles, cudaStream_t st);
// streaming loader: rows [r0, r0 + rows) (k-block aligned r0) of a shard's codes
// (dense [rows x n/2]) with the shard's full S2 / ZP ([n_g x n]) -> those k-blocks
cudaError_t dgq_launch_repack_slab(const uint8_t* codes, const int8_t* s2, const uint8_t* zp, int h, int r0, int rows,
                                   int g, int n, int n_tiles, int k_blocks, uint8_t* tiles, cudaStream_t st);
// validate_layer's S2 range (first_s2 may be null) and clip-interval checks on
// a shard / slab, first violation in the reference's loop order (atomicMin keys)
cudaError_t dgq_launch_validate(const uint8_t* codes, const int8_t* s2, const uint8_t* zp, int r0, int rows, int g,
                                int n_g, int n, int c0, int o_full, unsigned long long* first_s2,
                                unsigned long long* first_code, cudaStream_t st);
// prepared tiles -> W_s8 row-major [h x n] (same dequantiser as the fused GEMM)
cudaError_t dgq_launch_dequant_tiles(const uint8_t* tiles, int g, int h, int n, int n_tiles, int k_blocks,
                                     int8_t* w, size_t ldw, cudaStream_t st);
// Reference layout -> W_s8 row-major [h x o]; flags any value outside [-127,127]
// (first offending linear index in *bad, initialised to UINT64_MAX).
cudaError_t dgq_launch_dequant_ref(const uint8_t* codes, const int8_t* s2, const uint8_t* zp, int h, int o, int g,
                                   int8_t* w, unsigned long long* bad, cudaStream_t st);
// W [K x N] row-major -> WT [Npad x Kpad] K-major, zero padded.
cudaError_t dgq_launch_transpose_pad(const int8_t* W, int K, int N, int8_t* WT, int Kpad, int Npad, cudaStream_t st);
// Standalone epilogue over an int32 accumulator [M x N] (ld = N).
cudaError_t dgq_launch_epilogue(const int32_t* acc, size_t lda, const float* rs, const float* s1, const float* bias,
                                int M, int N, int fp16_mode, int out_f16, void* y, size_t ldy, cudaStream_t st);
// max over (r, c, i) of |prefix sum| (proj/src/kernel.cpp:73-77); *out must be 0.
cudaError_t dgq_launch_audit(const int8_t* Xq, size_t ldx, const int8_t* W, size_t ldw, int M, int K, int N,
                             unsigned long long* out, cudaStream_t st);
// segmented_gemm_reference comparator (proj/src/kernel.cpp:118-142) over the
// reference layout; y [M x o] f32.
cudaError_t dgq_launch_segmented(const int8_t* Xq, size_t ldx, const float* rs, const uint8_t* codes,
                                 const int8_t* s2, const uint8_t* zp, const float* s1, int M, int h, int o, int g,
                                 float* y, size_t ldy, cudaStream_t st);
// dequantize_to_f32 (proj/src/format.cpp:143-154) from W_s8 [h x o].
cudaError_t dgq_launch_dequant_f32(const int8_t* w, const float* s1, int h, int o, float* out, cudaStream_t st);

// calibration statistics (calib.cu): z (uint bits of non-negative floats) must
// be zero on entry; out likewise
cudaError_t dgq_launch_colmax(const float* X, size_t ldx, int rows, int h, unsigned* z, cudaStream_t st);
cudaError_t dgq_launch_smooth_absmax(const float* X, size_t ldx, int rows, int h, const float* k, unsigned* out,
                                     cudaStream_t st);
