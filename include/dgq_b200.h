/*
 * dgq_b200.h — C ABI of the B200-native DGQ A8W4 linear-layer hot path.
 *
 * Plain pointers, sizes and status codes only (no CUDA, torch or C++ types),
 * so a cgo / JNI / ctypes binding is a direct transcription.  Device pointers
 * are prefixed d; `stream` is a cudaStream_t passed as void* (NULL = legacy
 * default stream).  Every function returns dgq_status; on failure
 * dgq_last_error() holds a thread-local message and dgq_last_error_field() the
 * offending DgqLayer field for DGQ_EVALIDATION (mirrors dgq::validation_error).
 *
 * The C++ operator API of the reference (proj/include/dgq/kernel.hpp,
 * proj/include/dgq/format.hpp) is implemented on top of the host-buffer entry
 * points below by paper_2310_04836_b200/dropin/dgq_kernel_b200.cpp, compiled
 * against the reference's own, unchanged headers.  Status codes map back to
 * the reference's exception taxonomy:
 *   DGQ_EINVAL      -> std::invalid_argument   (proj/src/kernel.cpp:15-19,47-54,92-98)
 *   DGQ_EVALIDATION -> dgq::validation_error   (proj/src/format.cpp:18-20,131-136)
 *   DGQ_EOVERFLOW   -> std::runtime_error      (proj/src/kernel.cpp:83-85)
 *   DGQ_EFORMAT     -> dgq::format_error       (proj/src/format.cpp:214-250)
 *   DGQ_EIO         -> dgq::io_error           (proj/src/format.cpp:268-290)
 */
#ifndef DGQ_B200_H
#define DGQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DGQ_B200_ABI_VERSION 1

typedef enum dgq_status {
  DGQ_OK = 0,
  DGQ_EINVAL = 1,
  DGQ_EVALIDATION = 2,
  DGQ_EOVERFLOW = 3,
  DGQ_ECUDA = 4,
  DGQ_ENOMEM = 5,
  DGQ_EFORMAT = 6,
  DGQ_EIO = 7
} dgq_status;

enum { DGQ_MODE_STATIC = 0, DGQ_MODE_DYNAMIC = 1 };      /* proj/include/dgq/format.hpp:32 ActMode */
enum { DGQ_OUT_F32 = 0, DGQ_OUT_F16 = 1 };

/* Opaque device-resident prepared layer: the DgqLayer of
 * proj/include/dgq/format.hpp:36-49, validated on the host, uploaded once and
 * repacked into the B200 tile layout (optionally one column shard of it).
 * Immutable after creation; safe to share across host threads and streams
 * (split-K workspaces are per call, see dgq_linear). */
typedef struct dgq_layer dgq_layer;

typedef struct dgq_layer_info {
  size_t h;          /* input channels (K) */
  size_t o_full;     /* output channels of the unsharded layer */
  size_t o;          /* output channels held by this shard */
  size_t col_begin;  /* first output channel of this shard */
  size_t g;          /* group size */
  size_t k_pad;      /* activation-code row stride the GEMM expects (h rounded up to 128) */
  size_t n_pad;      /* o rounded up to 128 */
  int mode;          /* DGQ_MODE_* */
  float act_scale;
  int fused;         /* 1: INT4 tiles + in-kernel dequant; 0: materialised INT8 (exotic g) */
  size_t device_bytes;
} dgq_layer_info;

int dgq_abi_version(void);
const char* dgq_last_error(void);
const char* dgq_last_error_field(void);

/* ---- host-side numerics / invariants (no GPU) ------------------------------ */
/* replaces dgq::validate_layer, proj/src/format.cpp:24-75 (host arrays, reference layout) */
dgq_status dgq_validate_layer(size_t h, size_t o, size_t g, int mode, float act_scale, const uint8_t* codes_u4,
                              const int8_t* s2, const uint8_t* zp_u4, const float* s1, const float* k);
/* replaces dgq::clip_interval, proj/src/search.cpp:190-201 */
dgq_status dgq_clip_interval(int s2, int zp, int* lo, int* hi);
/* replaces dgq::fp16_round, proj/src/quant.cpp:9-58 */
float dgq_fp16_round(float x);

/* ---- prepared layer ---------------------------------------------------------
 * Host arrays in the reference layout (codes u4 [h x o] packed along o, even
 * column in the low nibble; s2 int8 [h/g x o]; zp u4 [h/g x o]; s1 f32[o];
 * k f32[h]).  Output channels [col_begin, col_end) are kept (col_end == 0
 * means o): the column-parallel shard of SURVEY.md §8e.  validate != 0 runs
 * the reference invariants first (DGQ_EVALIDATION + field on failure). */
dgq_status dgq_layer_create(int device, size_t h, size_t o, size_t g, int mode, float act_scale,
                            const uint8_t* codes_u4, const int8_t* s2, const uint8_t* zp_u4, const float* s1,
                            const float* k, size_t col_begin, size_t col_end, int validate, void* stream,
                            dgq_layer** out);
/* DGQ1 artifact bytes (proj/include/dgq/format.hpp:6-21, dgq_from_bytes
 * proj/src/format.cpp:214-266) straight to a prepared (sharded) layer. */
dgq_status dgq_layer_create_from_dgq1(int device, const uint8_t* bytes, size_t nbytes, size_t col_begin,
                                      size_t col_end, void* stream, dgq_layer** out);
/* The same from a DGQ1 FILE, streamed: S2 / ZP / s1 / k are read first, then
 * the code rows in ~32 MB slabs through pinned buffers, validated on the GPU
 * and repacked (only the shard's columns are uploaded).  DGQ_EIO (dgq::io_error)
 * when the file cannot be opened or read. */
dgq_status dgq_layer_create_from_dgq1_file(int device, const char* path, size_t col_begin, size_t col_end,
                                           void* stream, dgq_layer** out);
void dgq_layer_destroy(dgq_layer* layer);
dgq_status dgq_layer_get_info(const dgq_layer* layer, dgq_layer_info* info);

/* Bytes of zero-initialised scratch dgq_linear may need for M tokens (split-K
 * partial sums + tile counters; 0 when the call does not split K).  The
 * workspace is left zeroed on return, so it can be reused call after call. */
size_t dgq_linear_workspace_bytes(const dgq_layer* layer, size_t M);

/* The launch plan dgq_linear uses for M tokens: token-tile width, weight tiles
 * per CTA, K splits (a thread-block cluster when > 1) and the CTA count. */
dgq_status dgq_linear_plan(const dgq_layer* layer, size_t M, int* token_tile, int* weight_tiles, int* k_splits,
                           int* ctas);

/* ---- K1: per-token INT8 activation quantisation ----------------------------
 * replaces dgq::quantize_activations, proj/src/kernel.cpp:14-44.
 * dXq rows use stride ldq >= h (pass info.k_pad for dgq_linear); pad columns
 * are zero-filled. */
dgq_status dgq_quantize_act(const dgq_layer* layer, const float* dX, size_t M, size_t ldx, int8_t* dXq, size_t ldq,
                            float* dRowScale, void* stream);
/* FP16 activations (the inter-layer format; float(x_f16) is exact, so the codes
 * equal dgq_quantize_act on the float32 copy).  seg_cols > 0 reads the
 * all-gather of column shards: element (m, j) at
 * dX[(j / seg_cols) * seg_stride + m * ldx + j % seg_cols]. */
dgq_status dgq_quantize_act_f16(const dgq_layer* layer, const void* dX, size_t M, size_t ldx, size_t seg_cols,
                                size_t seg_stride, int8_t* dXq, size_t ldq, float* dRowScale, void* stream);
dgq_status dgq_quantize_act_raw(const float* dX, size_t M, size_t K, size_t ldx, const float* dK, int mode,
                                float act_scale, int8_t* dXq, size_t ldq, float* dRowScale, void* stream);

/* ---- K5: fused DGQ linear (INT4 dequant prologue + tcgen05 kind::i8 + epilogue)
 * replaces int8_gemm + epilogue of dgq::dgq_forward, proj/src/kernel.cpp:144-153.
 * dXq: [M x ldq] codes from K1 (ldq must equal info.k_pad, 16-B aligned).
 * dY:  [M x ldy] f32 or f16 (out_dtype); fp16_mode selects the reference's
 *      binary16 epilogue (proj/src/kernel.cpp:105-108).  dY may be NULL.
 * dAcc: optional raw int32 accumulators [M x ld_acc].
 * dWorkspace: dgq_linear_workspace_bytes(layer, M) zeroed bytes, or NULL to use
 *      the layer's internal workspace (then calls on the same layer must be
 *      stream-ordered). */
dgq_status dgq_linear(const dgq_layer* layer, const int8_t* dXq, size_t ldq, const float* dRowScale, size_t M,
                      const float* dBias, int out_dtype, int fp16_mode, void* dY, size_t ldy, int32_t* dAcc,
                      size_t ld_acc, void* dWorkspace, size_t ws_bytes, void* stream);
/* Several layers that share the input (q / k / v of a decoder layer, gate / up
 * of an MLP): `count` (1..4) outputs from one activation-code buffer.  Decode-
 * shaped calls (M <= 32) run as ONE K5d launch over the concatenation of the
 * layers' weight tiles, prefill-shaped calls (the pair kernel's M range) as ONE
 * K5p launch over their pair tiles (one stream-K problem: fewer launches, one
 * tail, better balance); other shapes fall back to one dgq_linear per layer.
 * Layers must share h, g.
 * dBias may be NULL or hold NULL entries; dY[i] is [M x ldy[i]].  dWorkspace:
 * dgq_linear_multi_workspace_bytes zeroed bytes, or NULL for layers[0]'s own. */
dgq_status dgq_linear_multi(const dgq_layer* const* layers, int count, const int8_t* dXq, size_t ldq,
                            const float* dRowScale, size_t M, const float* const* dBias, int out_dtype,
                            void* const* dY, const size_t* ldy, void* dWorkspace, size_t ws_bytes, void* stream);
size_t dgq_linear_multi_workspace_bytes(const dgq_layer* const* layers, int count, size_t M);
/* K1 + K5 in one call; dXq [M x k_pad] and dRowScale [M] are caller scratch. */
dgq_status dgq_forward_device(const dgq_layer* layer, const float* dX, size_t M, size_t ldx, const float* dBias,
                              int out_dtype, void* dY, size_t ldy, int8_t* dXq, float* dRowScale, void* dWorkspace,
                              size_t ws_bytes, void* stream);

/* ---- K2s: INT4 -> INT8 dequantisation ---------------------------------------
 * replaces dgq::dequantize_to_s8, proj/src/format.cpp:122-141.
 * From a prepared layer (same dequantiser as K5) into dW [h x ldw]: */
dgq_status dgq_layer_dequant_s8(const dgq_layer* layer, int8_t* dW, size_t ldw, void* stream);
/* From reference-layout device arrays, with the reference's range check
 * (synchronises the stream; DGQ_EVALIDATION field "codes" on corruption): */
dgq_status dgq_dequantize_to_s8(size_t h, size_t o, size_t g, const uint8_t* d_codes_u4, const int8_t* d_s2,
                                const uint8_t* d_zp_u4, int8_t* dW, void* stream);

/* ---- K3: exact INT8 GEMM (tcgen05 kind::i8) ---------------------------------
 * replaces dgq::int8_gemm, proj/src/kernel.cpp:46-87.  dXq [M x ldx], dW [K x ldw]
 * row-major, dAcc [M x ld_acc] int32.  max_abs_acc (HOST pointer, may be NULL)
 * runs the running-sum audit and synchronises the stream. */
dgq_status dgq_int8_gemm(const int8_t* dXq, size_t ldx, const int8_t* dW, size_t ldw, size_t M, size_t K, size_t N,
                         int32_t* dAcc, size_t ld_acc, int64_t* max_abs_acc, void* stream);

/* ---- K4: standalone epilogue -------------------------------------------------
 * replaces dgq::epilogue, proj/src/kernel.cpp:89-116. */
dgq_status dgq_epilogue(const int32_t* dAcc, size_t lda, const float* dRowScale, const float* dS1, const float* dBias,
                        size_t M, size_t N, int fp16_mode, int out_dtype, void* dY, size_t ldy, void* stream);

/* ---- audit: max over (r,c,i) of |running sum| (proj/src/kernel.cpp:73-77) --- */
dgq_status dgq_audit_max_abs_acc(const int8_t* dXq, size_t ldx, const int8_t* dW, size_t ldw, size_t M, size_t K,
                                 size_t N, int64_t* max_abs_acc, void* stream);

/* ---- calibration statistics --------------------------------
 * The step before the path: from calibration activations dX [rows x h]
 * (row-major f32, device) computes the smoothing vector and the static
 * activation scale exactly as the reference's quantize_layer does
 * (proj/src/pipeline.cpp:352-360): z = channel_maxima (proj/src/smoothing.cpp:9-24),
 * k = compute_smooth(z, percentile) (proj/src/smoothing.cpp:26-49; with
 * fp16_scales, k = max(1, fp16_round(k))), act_scale = static_act_scale of the
 * smoothed rows (proj/src/pipeline.cpp:96-101; fp16_round'ed with fp16_scales).
 * k_out [h], threshold_out and act_scale_out are HOST pointers; the call
 * synchronises the stream.  DGQ_EINVAL for a percentile outside (0, 1) or a
 * non-positive threshold (all-zero calibration), as the reference throws. */
dgq_status dgq_calibrate(const float* dX, size_t rows, size_t h, size_t ldx, float percentile, int fp16_scales,
                         float* k_out, float* threshold_out, float* act_scale_out, void* stream);

/* ---- offline quantiser: two-phase grid search -----------
 * The step that produces a layer's S2 / ZP / s1 / codes from FP32 weights,
 * bit-exact with the reference (FP64 objectives accumulated in the
 * reference's fixed order, smallest-alpha tie-break).  Device arrays:
 * dW [h x o] f32 row-major; dX, dXhat [b x h] f32 = the smoothed calibration
 * rows and their quantise-dequantise (SearchConfig::calib_X and X_hat).
 * alpha_grid is a HOST array searched in the given order.  Stream-ordered
 * (scratch from the device's stream-ordered pool: phase 1 needs
 * (h/g)*o*(8*b + 8*n_alpha + 8) bytes); evals (host, may be NULL) =
 * objective evaluations.  Errors mirror SearchConfig::validate. */
/* replaces dgq::phase1_search, proj/src/search.cpp:83-163: per (group, column)
 * S' [h/g x o] f32, ZP int32, winning objective f32 and alpha f32 */
dgq_status dgq_phase1_search(const float* dW, size_t h, size_t o, const float* dX, const float* dXhat, size_t b,
                             size_t g, int n_bits, const float* alpha_grid, size_t n_alpha, float* dSprime,
                             int32_t* dZp, float* dErr, float* dAlpha, uint64_t* evals, void* stream);
/* replaces dgq::phase2_search, proj/src/search.cpp:252-326: from phase 1's S'
 * and ZP, per column s1 [o] f32, S2 [h/g x o] int8, codes [h x o] int32,
 * objective [o] f64 and winning alpha [o] f32 */
dgq_status dgq_phase2_search(const float* dW, size_t h, size_t o, const float* dX, const float* dXhat, size_t b,
                             size_t g, const float* dSprime, const int32_t* dZp, const float* alpha_grid,
                             size_t n_alpha, float* dS1, int8_t* dS2, int32_t* dCodes, double* dColErr,
                             float* dColAlpha, uint64_t* evals, void* stream);

/* ---- column-parallel linear + all-gather --------------------
 * Rank r holds the column shard [r N/p, (r+1) N/p) of a layer
 * (dgq_layer_create col_begin / col_end).  NCCL is resolved at run time
 * (libnccl.so.2, preferring the copy already loaded in the process); `comm`
 * is an ncclComm_t passed as void*, ours (dgq_comm_create) or the caller's. */
#define DGQ_COMM_ID_BYTES 128
dgq_status dgq_comm_unique_id(uint8_t* id /* [DGQ_COMM_ID_BYTES] */);
dgq_status dgq_comm_create(int nranks, int rank, const uint8_t* id, int device, void** comm);
void dgq_comm_destroy(void* comm);
/* dgq_linear of this rank's shard into dY_local [M x o_shard] (dense), then an
 * NCCL all-gather into dY_all [nranks][M][o_shard] on `stream`: the layout the
 * next layer's K1 reads in place (dgq_quantize_act_f16, seg_cols = o_shard). */
dgq_status dgq_linear_allgather(const dgq_layer* layer, const int8_t* dXq, size_t ldq, const float* dRowScale,
                                size_t M, const float* dBias, int out_dtype, void* dY_local, void* dY_all, void* comm,
                                void* stream);

/* ---- measured dense INT8 tensor peak ----------------------------------------
 * The INT8 roofline denominator: every SM pair issues
 * tcgen05.mma.cta_group::2.kind::i8 (256 x 256 x 32, K5p's shape) back to back
 * from shared-memory operands; best of `reps` launches (CUDA events), TOPS out
 * (the burst rate).  reps < 0: -reps launches back to back timed as one span —
 * the sustained rate at the clock the GPU holds under continuous tensor load
 * (the denominator for kernels timed inside a long step).  reps = 0: 10.
 * Synchronises; runs on the current device. */
dgq_status dgq_measure_i8_peak(int reps, double* tops, double* best_ms);

/* ---- host-buffer API: the reference's calling convention --------------------
 * Host arrays in (reference layouts), host arrays out; each call uploads,
 * runs the CUDA kernels on a per-thread stream of the CURRENT device and
 * synchronises.  These are what the C++ drop-in for proj/include/dgq/kernel.hpp
 * (paper_2310_04836_b200/dropin/) and FFI bindings call.  Row-major, dense. */
/* quantize_activations, proj/src/kernel.cpp:14-44: X [M x K] -> codes [M x K], row_scales [M] */
dgq_status dgq_host_quantize_activations(const float* X, size_t M, size_t K, const float* k, int mode,
                                         float act_scale, int8_t* codes, float* row_scales);
/* dequantize_to_s8, proj/src/format.cpp:122-141 (DGQ_EVALIDATION field "codes" on corruption) */
dgq_status dgq_host_dequantize_to_s8(size_t h, size_t o, size_t g, const uint8_t* codes_u4, const int8_t* s2,
                                     const uint8_t* zp_u4, int8_t* w_s8);
/* dequantize_to_f32, proj/src/format.cpp:143-154 */
dgq_status dgq_host_dequantize_to_f32(size_t h, size_t o, size_t g, const uint8_t* codes_u4, const int8_t* s2,
                                      const uint8_t* zp_u4, const float* s1, float* w);
/* int8_gemm, proj/src/kernel.cpp:46-87: Xq [M x K] x W [K x N] -> acc [M x N];
 * max_abs_acc (may be NULL) = the reference's running-sum audit */
dgq_status dgq_host_int8_gemm(const int8_t* Xq, const int8_t* W, size_t M, size_t K, size_t N, int32_t* acc,
                              int64_t* max_abs_acc);
/* epilogue, proj/src/kernel.cpp:89-116 (bias may be NULL) -> y f32 [M x N] */
dgq_status dgq_host_epilogue(const int32_t* acc, const float* row_scales, const float* s1, const float* bias,
                             size_t M, size_t N, int fp16_mode, float* y);
/* segmented_gemm_reference, proj/src/kernel.cpp:118-142 (group-wise comparator) */
dgq_status dgq_host_segmented_gemm(const int8_t* Xq, const float* row_scales, size_t M, size_t h, size_t o, size_t g,
                                   const uint8_t* codes_u4, const int8_t* s2, const uint8_t* zp_u4, const float* s1,
                                   float* y);
/* dgq_forward, proj/src/kernel.cpp:144-153: the whole path per call (dequant with
 * range check, K1, fused K5 with FP32 out, audit).  w_s8, act_codes,
 * row_scales, max_abs_acc may be NULL (not returned). */
dgq_status dgq_host_forward(size_t M, size_t h, size_t o, size_t g, int mode, float act_scale,
                            const uint8_t* codes_u4, const int8_t* s2, const uint8_t* zp_u4, const float* s1,
                            const float* k, const float* X, const float* bias, float* out, int8_t* w_s8,
                            int8_t* act_codes, float* row_scales, int64_t* max_abs_acc);
/* Prepared-layer forward with HOST buffers (the serving call): X host f32
 * [M x h] -> Y host [M x o] (out_dtype); dBias is a DEVICE pointer or NULL.
 * stream NULL = the per-thread stream.  Synchronises before returning. */
dgq_status dgq_layer_forward_host(const dgq_layer* layer, const float* X, size_t M, const float* dBias,
                                  int out_dtype, void* Y, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DGQ_B200_H */
