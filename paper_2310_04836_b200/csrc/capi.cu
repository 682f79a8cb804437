// C-ABI entry points (include/dgq_b200.h): argument checks with the reference's
// error semantics, prepared-layer lifetime, TMA descriptor construction and
// kernel dispatch.  No CPU compute path exists: every numeric result comes
// from a CUDA kernel in this library.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/dgq_b200.h"
#include "kernels.h"

extern "C" int dgq_debug_decode_mode();

cudaError_t dgq_allow_smem(const void* kernel, size_t bytes) {
  // The limit only ever grows (to the largest size requested so far, per kernel
  // and device), so a concurrent launch needing less can never shrink it under
  // a launch needing more; it stays at what the calls need rather than the
  // opt-in maximum, which keeps the driver's L1 / shared-memory carveout as
  // large as the kernel allows.
  static std::mutex mu;
  static std::unordered_map<const void*, std::vector<size_t>> done;  // per device: limit set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  std::vector<size_t>& v = done[kernel];
  if (v.size() <= static_cast<size_t>(dev)) v.resize(dev + 1, 0);
  if (bytes <= v[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) v[dev] = bytes;
  return e;
}

namespace {

thread_local std::string t_msg;
thread_local std::string t_field;

dgq_status fail(dgq_status st, const std::string& msg, const std::string& field = "") {
  t_msg = msg;
  t_field = field;
  return st;
}

#define DGQ_CUDA(expr)                                                                           \
  do {                                                                                           \
    cudaError_t e_ = (expr);                                                                     \
    if (e_ != cudaSuccess)                                                                       \
      return fail(e_ == cudaErrorMemoryAllocation ? DGQ_ENOMEM : DGQ_ECUDA,                      \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                           \
  } while (0)

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2-D uint8 tensor map: rows x cols (cols contiguous, row stride `ld` bytes),
// box = box_rows x 128 bytes, 128-byte swizzle, zero fill out of bounds.
dgq_status make_tmap(CUtensorMap* m, const void* base, size_t rows, size_t cols, size_t ld, uint32_t box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(DGQ_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld)};
  cuuint32_t box[2] = {128u, box_rows};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DGQ_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return DGQ_OK;
}

// 3-D view of the activation codes for the decode kernel: (128 k, rows, k-block)
// with strides (1, ld, 128) bytes; box = 128 B x box_rows x depth, 128-byte
// swizzle: one request stages `depth` consecutive k-blocks' [rows x 128] tiles.
dgq_status make_tmap_kblocks(CUtensorMap* m, const void* base, size_t rows, size_t cols, size_t ld, uint32_t box_rows,
                             uint32_t depth) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(DGQ_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {128u, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols / 128)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld), 128u};
  cuuint32_t box[3] = {128u, box_rows, depth};
  cuuint32_t es[3] = {1u, 1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DGQ_ECUDA, "cuTensorMapEncodeTiled (3-D) failed (" + std::to_string(r) + ")");
  return DGQ_OK;
}

unsigned long long* g_dbg_ts = nullptr;  // tools only: per-CTA phase timestamps

// Output tensor map for the prefill epilogue: rows x cols elements of `dt`,
// box = 32 rows x 128 bytes, 128-byte swizzle (matches the smem staging).
dgq_status make_out_tmap(CUtensorMap* m, void* base, size_t rows, size_t cols, size_t ld, bool f16) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(DGQ_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const size_t esz = f16 ? 2 : 4;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * esz)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esz), 32u};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = enc(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DGQ_ECUDA, "cuTensorMapEncodeTiled (output) failed (" + std::to_string(r) + ")");
  return DGQ_OK;
}

size_t round_up(size_t v, size_t m) { return (v + m - 1) / m * m; }

inline int nib(const uint8_t* p, size_t idx) { return (idx & 1) ? (p[idx >> 1] >> 4) : (p[idx >> 1] & 0x0F); }

}  // namespace

struct dgq_layer {
  int device = 0;
  size_t h = 0, o_full = 0, o = 0, c0 = 0, g = 0;
  int mode = 1;
  float act_scale = 0.0f;
  size_t k_pad = 0, n_pad = 0;
  int n_tiles = 0, k_blocks = 0;
  bool fused = true;
  uint8_t* tiles = nullptr;  // fused: prepared INT4 tiles
  int8_t* wt = nullptr;      // non-fused: W_s8^T [n_pad x k_pad]
  float* s1 = nullptr;       // [o] (this shard)
  float* k = nullptr;        // [h]
  float* rk = nullptr;       // [h] RN(1/k): hoisted reciprocals for K1
  uint8_t* ksm = nullptr;    // [h/8] bit t of chunk c: k[8c + t] != 1 (only those channels divide in K1)
  int* spec = nullptr;       // [nspec] the channels with k != 1, ascending
  int nspec = 0;
  size_t device_bytes = 0;
  CUtensorMap tmA{};  // non-fused A operand
  // Internal split-K workspaces for callers that pass none, one per stream:
  // the stream-K partials and tile flags of a launch must not be shared with a
  // launch on another stream (the kernels run after the host call returns).
  // `ev` marks the last launch that used the slot, so a destroyed stream whose
  // handle is reused while its work is pending cannot overlap it either.
  struct StreamWs {
    void* p = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool used = false;
  };
  std::mutex ws_mu;
  std::unordered_map<cudaStream_t, StreamWs> ws;
};

// The layer's internal workspace for stream `st` (caller holds L->ws_mu),
// grown to `need` zeroed bytes.  Outside stream capture the launch that uses it
// is ordered after the previous user of the slot (ws_release records it).
static dgq_status ws_acquire(dgq_layer* L, cudaStream_t st, size_t need, void** out, size_t* cap) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  DGQ_CUDA(cudaStreamIsCapturing(st, &cs));
  auto& w = L->ws[st];
  if (w.cap < need) {
    if (cs != cudaStreamCaptureStatusNone)
      return fail(DGQ_EINVAL, "internal workspace must grow during stream capture: call once before capturing or "
                              "pass dWorkspace");
    if (w.p) {
      DGQ_CUDA(cudaEventSynchronize(w.ev));
      cudaFree(w.p);
      w.p = nullptr;
      w.cap = 0;
    }
    DGQ_CUDA(cudaMalloc(&w.p, need));
    DGQ_CUDA(cudaMemsetAsync(w.p, 0, need, st));
    w.cap = need;
  }
  if (!w.ev) DGQ_CUDA(cudaEventCreateWithFlags(&w.ev, cudaEventDisableTiming));
  if (w.used && cs == cudaStreamCaptureStatusNone) DGQ_CUDA(cudaStreamWaitEvent(st, w.ev, 0));
  *out = w.p;
  *cap = w.cap;
  return DGQ_OK;
}

// Argument checks shared by dgq_linear and every layer of dgq_linear_multi
// (the reference's preconditions of int8_gemm, proj/src/kernel.cpp:47-54).
static dgq_status check_linear_args(const dgq_layer* L, const int8_t* dXq, size_t ldq, const float* dRs, size_t M,
                                    const void* dY, size_t ldy, const int32_t* dAcc, size_t ld_acc) {
  if (!dXq || !dRs) return fail(DGQ_EINVAL, "null activation codes or row scales");
  if (ldq != L->k_pad) return fail(DGQ_EINVAL, "ldq must equal the layer's k_pad (" + std::to_string(L->k_pad) + ")");
  if (reinterpret_cast<uintptr_t>(dXq) % 16) return fail(DGQ_EINVAL, "activation codes must be 16-byte aligned");
  if (dY && ldy < L->o) return fail(DGQ_EINVAL, "ldy smaller than the output width");
  if (dAcc && ld_acc < L->o) return fail(DGQ_EINVAL, "ld_acc smaller than the output width");
  if (M > 0x7FFFFFFF) return fail(DGQ_EINVAL, "too many rows");
  if (static_cast<double>(L->h) * 127.0 * 127.0 >= 2147483648.0)
    return fail(DGQ_EINVAL, "h too large for 32-bit accumulation");
  return DGQ_OK;
}

static void ws_release(dgq_layer* L, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
  auto& w = L->ws[st];
  if (cudaEventRecord(w.ev, st) == cudaSuccess) w.used = true;
}

extern "C" {

int dgq_abi_version(void) { return DGQ_B200_ABI_VERSION; }
/* not in the public header: profiling hook for tools/ (device buffer of [cta][8] u64, or NULL) */
void dgq_debug_set_timestamps(void* d_buf) { g_dbg_ts = static_cast<unsigned long long*>(d_buf); }
const char* dgq_last_error(void) { return t_msg.c_str(); }
/* not in the public header: lets the other translation units of the library set the thread-local error */
dgq_status dgq_internal_fail(dgq_status st, const char* msg, const char* field) {
  return fail(st, msg ? msg : "", field ? field : "");
}
const char* dgq_last_error_field(void) { return t_field.c_str(); }

dgq_status dgq_clip_interval(int s2, int zp, int* lo, int* hi) {
  if (s2 < 1) return fail(DGQ_EINVAL, "clip_interval requires S2 >= 1");
  const int a = (-127) / s2 + zp, b = 127 / s2 + zp;  // C++ truncating division
  const int l = a > 0 ? a : 0, u = b < 15 ? b : 15;
  if (l > u)
    return fail(DGQ_EOVERFLOW, "empty clip interval for S2=" + std::to_string(s2) + " ZP=" + std::to_string(zp));
  *lo = l;
  *hi = u;
  return DGQ_OK;
}

float dgq_fp16_round(float x) {
  uint32_t b;
  std::memcpy(&b, &x, 4);
  const uint32_t sign = b & 0x80000000u, mag = b & 0x7FFFFFFFu;
  if (mag >= 0x7F800000u) return x;
  const int e = static_cast<int>(mag >> 23) - 127;
  uint32_t h;
  if (e > 15) {
    h = 0x7C00u;
  } else if (e >= -14) {
    const uint32_t m = mag & 0x7FFFFFu, rem = m & 0x1FFFu;
    h = (static_cast<uint32_t>(e + 15) << 10) | (m >> 13);
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
  } else if (e >= -24) {
    const uint32_t m = (mag & 0x7FFFFFu) | 0x800000u;
    const int sh = -e - 1;
    const uint32_t rem = m & ((1u << sh) - 1u), half = 1u << (sh - 1);
    h = m >> sh;
    if (rem > half || (rem == half && (h & 1u))) ++h;
  } else {
    h = 0;
  }
  const uint32_t he = (h >> 10) & 0x1Fu;
  uint32_t hm = h & 0x3FFu, out;
  if (he == 0x1Fu) {
    out = sign | 0x7F800000u;
  } else if (he) {
    out = sign | ((he + 112u) << 23) | (hm << 13);
  } else if (!hm) {
    out = sign;
  } else {
    int sh = 0;
    while (!(hm & 0x400u)) {
      hm <<= 1;
      --sh;
    }
    out = sign | (static_cast<uint32_t>(113 + sh) << 23) | ((hm & 0x3FFu) << 13);
  }
  float r;
  std::memcpy(&r, &out, 4);
  return r;
}

dgq_status dgq_validate_layer(size_t h, size_t o, size_t g, int mode, float act_scale, const uint8_t* codes,
                              const int8_t* s2, const uint8_t* zp, const float* s1, const float* k) {
  auto bad = [](const char* field, const std::string& m) {
    return fail(DGQ_EVALIDATION, std::string("invalid DgqLayer field '") + field + "': " + m, field);
  };
  if (h == 0 || o == 0) return bad("shape", "h and o must be positive");
  if (o % 2) return bad("shape", "o must be even for packed 4-bit storage");
  if (g == 0 || h % g) return bad("g", "group size must divide h");
  if (!codes || !s2 || !zp || !s1 || !k) return fail(DGQ_EINVAL, "null layer array");
  const size_t ng = h / g;
  for (size_t i = 0; i < ng * o; ++i)
    if (s2[i] < 1) return bad("s2", "value " + std::to_string(int(s2[i])) + " outside [1, 127]");
  for (size_t c = 0; c < o; ++c)
    if (!(s1[c] > 0.0f) || !std::isfinite(s1[c])) return bad("s1", "scales must be positive and finite");
  for (size_t j = 0; j < h; ++j)
    if (!(k[j] >= 1.0f) || !std::isfinite(k[j])) return bad("k", "smoothing scales must be >= 1");
  if (mode == DGQ_MODE_STATIC && !(act_scale > 0.0f))
    return bad("act_scale", "static mode requires a positive activation scale");
  if (!(act_scale >= 0.0f) || !std::isfinite(act_scale)) return bad("act_scale", "must be finite and non-negative");
  for (size_t kk = 0; kk < ng; ++kk)
    for (size_t c = 0; c < o; ++c) {
      const int sv = s2[kk * o + c], z = nib(zp, kk * o + c);
      const int q = 127 / sv;
      const int lo = std::max(0, z - q), hi = std::min(15, z + q);
      for (size_t j = 0; j < g; ++j) {
        const size_t i = kk * g + j;
        const int code = nib(codes, i * o + c);
        if (code < lo || code > hi)
          return bad("codes", "code " + std::to_string(code) + " at (" + std::to_string(i) + ", " +
                                  std::to_string(c) + ") outside clip interval [" + std::to_string(lo) + ", " +
                                  std::to_string(hi) + "]");
      }
    }
  return DGQ_OK;
}

void dgq_layer_destroy(dgq_layer* L) {
  if (!L) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(L->device);
  cudaFree(L->tiles);
  cudaFree(L->wt);
  cudaFree(L->s1);
  cudaFree(L->k);
  cudaFree(L->rk);
  cudaFree(L->ksm);
  cudaFree(L->spec);
  for (auto& kv : L->ws) {
    cudaFree(kv.second.p);
    if (kv.second.ev) cudaEventDestroy(kv.second.ev);
  }
  cudaSetDevice(prev);
  delete L;
}

// validate_layer's O(h + o) checks (proj/src/format.cpp:48-59), in the
// reference's order; the O(h o) ones run on the GPU (create_layer).
static dgq_status validate_scalars(size_t h, size_t o, int mode, float act_scale, const float* s1, const float* k,
                                   std::string* field, std::string* msg) {
  for (size_t c = 0; c < o; ++c)
    if (!(s1[c] > 0.0f) || !std::isfinite(s1[c])) {
      *field = "s1";
      *msg = "scales must be positive and finite";
      return DGQ_EVALIDATION;
    }
  for (size_t j = 0; j < h; ++j)
    if (!(k[j] >= 1.0f) || !std::isfinite(k[j])) {
      *field = "k";
      *msg = "smoothing scales must be >= 1";
      return DGQ_EVALIDATION;
    }
  if (mode == DGQ_MODE_STATIC && !(act_scale > 0.0f)) {
    *field = "act_scale";
    *msg = "static mode requires a positive activation scale";
    return DGQ_EVALIDATION;
  }
  if (!(act_scale >= 0.0f) || !std::isfinite(act_scale)) {
    *field = "act_scale";
    *msg = "must be finite and non-negative";
    return DGQ_EVALIDATION;
  }
  return DGQ_OK;
}

// Source of the packed code rows (reference layout, o/2 bytes per row):
// returns a host pointer to rows [r0, r0 + rows) (row pitch o/2), valid until
// the next call with the same buffer index.
using RowFetch = std::function<const uint8_t*(size_t r0, size_t rows, int buf)>;

// The prepared layer.  Fused group sizes take the streaming path: the shard's
// S2 / ZP columns are uploaded once, the codes in k-block-aligned slabs of
// ~32 MB (only the shard's columns), each slab validated on the GPU (S2 range
// and clip intervals, first violation in the reference's loop order) and
// repacked into its k-blocks, so neither host nor device ever holds a second
// full copy of the weights.  validate != 0 reports failures exactly as
// dgq::validate_layer (proj/src/format.cpp:24-75) would, restricted to the
// shard's columns for S2 and codes.
static dgq_status create_layer(int device, size_t h, size_t o, size_t g, int mode, float act_scale,
                               const RowFetch& fetch, const uint8_t* codes_full, const int8_t* s2, const uint8_t* zp,
                               const float* s1, const float* k, size_t col_begin, size_t col_end, int validate,
                               void* stream, dgq_layer** out, cudaEvent_t* copy_done = nullptr) {
  DGQ_NVTX("dgq_layer_create");
  if (!out) return fail(DGQ_EINVAL, "out is null");
  *out = nullptr;
  auto bad = [](const std::string& field, const std::string& m) {
    return fail(DGQ_EVALIDATION, "invalid DgqLayer field '" + field + "': " + m, field);
  };
  if (validate) {
    if (h == 0 || o == 0) return bad("shape", "h and o must be positive");
    if (o % 2) return bad("shape", "o must be even for packed 4-bit storage");
    if (g == 0 || h % g) return bad("g", "group size must divide h");
  } else if (h == 0 || o == 0 || o % 2 || g == 0 || h % g) {
    return fail(DGQ_EINVAL, "inconsistent layer shape");
  }
  if (!s2 || !zp || !s1 || !k) return fail(DGQ_EINVAL, "null layer array");
  if (col_end == 0) col_end = o;
  if (col_begin >= col_end || col_end > o) return fail(DGQ_EINVAL, "bad column shard range");
  if (col_begin % 2 || col_end % 2) return fail(DGQ_EINVAL, "column shard bounds must be even (packed 4-bit storage)");
  if (h > (1u << 30) || o > (1u << 30)) return fail(DGQ_EINVAL, "layer too large");
  const bool fused = dgq_layout::fused_ok(static_cast<int>(g));
  if (!fused) {
    // exotic group sizes keep the host validation and a full upload (below)
    if (!codes_full) return fail(DGQ_EINVAL, "this group size needs the codes in memory");
    if (validate) {
      dgq_status st = dgq_validate_layer(h, o, g, mode, act_scale, codes_full, s2, zp, s1, k);
      if (st != DGQ_OK) return st;
    }
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int prev_dev = 0;
  DGQ_CUDA(cudaGetDevice(&prev_dev));
  DGQ_CUDA(cudaSetDevice(device));
  struct RestoreDevice {
    int d;
    ~RestoreDevice() { cudaSetDevice(d); }
  } restore_dev{prev_dev};

  auto* L = new dgq_layer();
  L->device = device;
  L->h = h;
  L->o_full = o;
  L->c0 = col_begin;
  L->o = col_end - col_begin;
  L->g = g;
  L->mode = mode ? DGQ_MODE_DYNAMIC : DGQ_MODE_STATIC;
  L->act_scale = act_scale;
  L->k_pad = round_up(h, 128);
  L->n_pad = round_up(L->o, 128);
  L->n_tiles = static_cast<int>(L->n_pad / 128);
  L->k_blocks = static_cast<int>(L->k_pad / 128);
  L->fused = fused;

  const size_t ng = h / g, w = L->o, c0 = col_begin;
  uint8_t *d_codes = nullptr, *d_zp = nullptr;
  int8_t* d_s2 = nullptr;
  unsigned long long* d_first = nullptr;
  auto cleanup_tmp = [&] {
    cudaFree(d_codes);
    cudaFree(d_s2);
    cudaFree(d_zp);
    cudaFree(d_first);
  };
#define DGQ_CUDA_L(expr)                        \
  do {                                          \
    cudaError_t e_ = (expr);                    \
    if (e_ != cudaSuccess) {                    \
      cleanup_tmp();                            \
      dgq_layer_destroy(L);                     \
      return fail(e_ == cudaErrorMemoryAllocation ? DGQ_ENOMEM : DGQ_ECUDA, \
                  std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    }                                           \
  } while (0)
  DGQ_CUDA_L(cudaMalloc(&L->s1, L->o * sizeof(float)));
  DGQ_CUDA_L(cudaMalloc(&L->k, h * sizeof(float)));
  DGQ_CUDA_L(cudaMemcpyAsync(L->s1, s1 + col_begin, L->o * sizeof(float), cudaMemcpyHostToDevice, st));
  DGQ_CUDA_L(cudaMemcpyAsync(L->k, k, h * sizeof(float), cudaMemcpyHostToDevice, st));
  DGQ_CUDA_L(cudaMalloc(&L->rk, h * sizeof(float)));
  DGQ_CUDA_L(dgq_launch_reciprocal(L->k, L->rk, static_cast<int>(h), st));
  if (h % 8 == 0) {
    std::vector<uint8_t> ksm(h / 8);
    for (size_t c = 0; c < h / 8; ++c) {
      uint8_t m = 0;
      for (size_t t = 0; t < 8; ++t) m |= (k[c * 8 + t] != 1.0f ? 1u : 0u) << t;
      ksm[c] = m;
    }
    DGQ_CUDA_L(cudaMalloc(&L->ksm, h / 8));
    DGQ_CUDA_L(cudaMemcpy(L->ksm, ksm.data(), h / 8, cudaMemcpyHostToDevice));
    std::vector<int> spec;
    for (size_t j = 0; j < h; ++j)
      if (k[j] != 1.0f) spec.push_back(static_cast<int>(j));
    L->nspec = static_cast<int>(spec.size());
    if (!spec.empty()) {
      DGQ_CUDA_L(cudaMalloc(&L->spec, spec.size() * sizeof(int)));
      DGQ_CUDA_L(cudaMemcpy(L->spec, spec.data(), spec.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
  }
  L->device_bytes = (L->o + h) * sizeof(float);
  if (fused) {
    const size_t tb = static_cast<size_t>(L->n_tiles) * L->k_blocks * dgq_layout::chunk_bytes(static_cast<int>(g));
    DGQ_CUDA_L(cudaMalloc(&L->tiles, tb));
    L->device_bytes += tb;
    // the shard's S2 / ZP columns, dense [n_g x w] / [n_g x w/2]
    DGQ_CUDA_L(cudaMalloc(&d_s2, ng * w));
    DGQ_CUDA_L(cudaMalloc(&d_zp, ng * w / 2));
    DGQ_CUDA_L(cudaMemcpy2DAsync(d_s2, w, s2 + c0, o, w, ng, cudaMemcpyHostToDevice, st));
    DGQ_CUDA_L(cudaMemcpy2DAsync(d_zp, w / 2, zp + c0 / 2, o / 2, w / 2, ng, cudaMemcpyHostToDevice, st));
    DGQ_CUDA_L(cudaMalloc(&d_first, 2 * sizeof(unsigned long long)));
    DGQ_CUDA_L(cudaMemsetAsync(d_first, 0xFF, 2 * sizeof(unsigned long long), st));
    // slabs: k-block and group aligned, ~32 MB of the shard's codes
    const size_t unit = g > 128 ? g : 128;
    size_t rows = std::max(unit, ((32u << 20) / std::max<size_t>(w / 2, 1)) / unit * unit);
    if (rows > h) rows = round_up(h, unit);
    DGQ_CUDA_L(cudaMalloc(&d_codes, rows * (w / 2)));
    int buf = 0;
    for (size_t r0 = 0; r0 < h; r0 += rows, buf ^= 1) {
      const size_t n = std::min(rows, h - r0);
      const uint8_t* src = fetch(r0, n, buf);
      if (!src) {
        cleanup_tmp();
        dgq_layer_destroy(L);
        return fail(DGQ_EFORMAT, "could not read the code rows of the artifact", "truncated");
      }
      DGQ_CUDA_L(cudaMemcpy2DAsync(d_codes, w / 2, src + c0 / 2, o / 2, w / 2, n, cudaMemcpyHostToDevice, st));
      if (copy_done) DGQ_CUDA_L(cudaEventRecord(copy_done[buf], st));  // the host buffer may be refilled after this
      if (validate)
        DGQ_CUDA_L(dgq_launch_validate(d_codes, d_s2, d_zp, static_cast<int>(r0), static_cast<int>(n),
                                       static_cast<int>(g), static_cast<int>(ng), static_cast<int>(w),
                                       static_cast<int>(c0), static_cast<int>(o), r0 == 0 ? d_first : nullptr,
                                       d_first + 1, st));
      DGQ_CUDA_L(dgq_launch_repack_slab(d_codes, d_s2, d_zp, static_cast<int>(h), static_cast<int>(r0),
                                        static_cast<int>(n), static_cast<int>(g), static_cast<int>(w), L->n_tiles,
                                        L->k_blocks, L->tiles, st));
    }
    if (validate) {
      unsigned long long first[2];
      DGQ_CUDA_L(cudaMemcpyAsync(first, d_first, sizeof first, cudaMemcpyDeviceToHost, st));
      DGQ_CUDA_L(cudaStreamSynchronize(st));
      std::string field, msg;
      dgq_status vs = DGQ_OK;
      if (first[0] != ~0ull) {  // S2 outside [1, 127] (proj/src/format.cpp:44-47)
        const size_t kg = first[0] / o, c = first[0] % o;
        int8_t v = 0;
        std::memcpy(&v, s2 + kg * o + c, 1);
        field = "s2";
        msg = "value " + std::to_string(int(v)) + " outside [1, 127]";
        vs = DGQ_EVALIDATION;
      } else {
        vs = validate_scalars(h, o, mode, act_scale, s1, k, &field, &msg);
        if (vs == DGQ_OK && first[1] != ~0ull) {  // clip intervals (proj/src/format.cpp:60-74)
          const size_t j = first[1] % g, kc = first[1] / g, kg = kc / o, c = kc % o, i = kg * g + j;
          const int sv = s2[kg * o + c], z = nib(zp, kg * o + c), q = 127 / sv;
          const int lo = std::max(0, z - q), hi = std::min(15, z + q);
          int code = -1;
          const uint8_t* row = fetch(i, 1, 0);
          if (row) code = nib(row, c);
          field = "codes";
          msg = "code " + std::to_string(code) + " at (" + std::to_string(i) + ", " + std::to_string(c) +
                ") outside clip interval [" + std::to_string(lo) + ", " + std::to_string(hi) + "]";
          vs = DGQ_EVALIDATION;
        }
      }
      if (vs != DGQ_OK) {
        cleanup_tmp();
        dgq_layer_destroy(L);
        return bad(field, msg);
      }
    }
  } else {
    // exotic group sizes: materialise W_s8 once, transpose to K-major
    const size_t codes_b = h * o / 2, s2_b = ng * o, zp_b = ng * o / 2;
    DGQ_CUDA_L(cudaMalloc(&d_codes, codes_b));
    DGQ_CUDA_L(cudaMalloc(&d_s2, s2_b));
    DGQ_CUDA_L(cudaMalloc(&d_zp, zp_b));
    DGQ_CUDA_L(cudaMemcpyAsync(d_codes, codes_full, codes_b, cudaMemcpyHostToDevice, st));
    DGQ_CUDA_L(cudaMemcpyAsync(d_s2, s2, s2_b, cudaMemcpyHostToDevice, st));
    DGQ_CUDA_L(cudaMemcpyAsync(d_zp, zp, zp_b, cudaMemcpyHostToDevice, st));
    int8_t* w_full = nullptr;
    unsigned long long* d_bad = nullptr;
    DGQ_CUDA_L(cudaMalloc(&w_full, h * o));
    DGQ_CUDA_L(cudaMalloc(&d_bad, sizeof(unsigned long long)));
    DGQ_CUDA_L(cudaMemsetAsync(d_bad, 0xFF, sizeof(unsigned long long), st));
    DGQ_CUDA_L(dgq_launch_dequant_ref(d_codes, d_s2, d_zp, static_cast<int>(h), static_cast<int>(o),
                                      static_cast<int>(g), w_full, d_bad, st));
    // transpose the shard's columns
    DGQ_CUDA_L(cudaMalloc(&L->wt, L->n_pad * L->k_pad));
    L->device_bytes += L->n_pad * L->k_pad;
    int8_t* w_shard = w_full;
    if (L->o != o) {
      DGQ_CUDA_L(cudaMalloc(&w_shard, h * L->o));
      DGQ_CUDA_L(cudaMemcpy2DAsync(w_shard, L->o, w_full + col_begin, o, L->o, h, cudaMemcpyDeviceToDevice, st));
    }
    DGQ_CUDA_L(dgq_launch_transpose_pad(w_shard, static_cast<int>(h), static_cast<int>(L->o), L->wt,
                                        static_cast<int>(L->k_pad), static_cast<int>(L->n_pad), st));
    DGQ_CUDA_L(cudaStreamSynchronize(st));
    if (w_shard != w_full) cudaFree(w_shard);
    cudaFree(w_full);
    cudaFree(d_bad);
    dgq_status ms = make_tmap(&L->tmA, L->wt, L->n_pad, L->k_pad, L->k_pad, 128);
    if (ms != DGQ_OK) {
      cleanup_tmp();
      dgq_layer_destroy(L);
      return ms;
    }
  }
  DGQ_CUDA_L(cudaStreamSynchronize(st));
  cleanup_tmp();
#undef DGQ_CUDA_L
  *out = L;
  return DGQ_OK;
}

dgq_status dgq_layer_create(int device, size_t h, size_t o, size_t g, int mode, float act_scale,
                            const uint8_t* codes, const int8_t* s2, const uint8_t* zp, const float* s1,
                            const float* k, size_t col_begin, size_t col_end, int validate, void* stream,
                            dgq_layer** out) {
  if (!codes) return fail(DGQ_EINVAL, "null layer array");
  const size_t pitch = o / 2;
  RowFetch fetch = [codes, pitch](size_t r0, size_t, int) { return codes + r0 * pitch; };
  return create_layer(device, h, o, g, mode, act_scale, fetch, codes, s2, zp, s1, k, col_begin, col_end, validate,
                      stream, out);
}

dgq_status dgq_layer_create_from_dgq1(int device, const uint8_t* bytes, size_t nbytes, size_t col_begin,
                                      size_t col_end, void* stream, dgq_layer** out) {
  // DGQ1 layout, proj/include/dgq/format.hpp:6-21; checks of proj/src/format.cpp:214-250
  constexpr size_t kHeader = 29;
  if (!bytes || nbytes < kHeader) return fail(DGQ_EFORMAT, "truncated: DGQ file shorter than the header", "truncated");
  if (std::memcmp(bytes, "DGQ1", 4) != 0) return fail(DGQ_EFORMAT, "bad magic, expected \"DGQ1\"", "bad_magic");
  auto u64 = [&](size_t off) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(bytes[off + i]) << (8 * i);
    return v;
  };
  const uint64_t h = u64(4), o = u64(12), g = u64(20);
  const uint8_t mode = bytes[28];
  if (mode > 1) return fail(DGQ_EFORMAT, "unknown mode byte " + std::to_string(int(mode)), "bad_header");
  if (h == 0 || o == 0 || o % 2 || g == 0 || h % g)
    return fail(DGQ_EFORMAT, "inconsistent dimensions in header", "bad_header");
  if (h > (1ull << 30) || o > (1ull << 30)) return fail(DGQ_EFORMAT, "dimensions too large", "bad_header");
  const uint64_t ng = h / g;
  const uint64_t need = kHeader + h * o / 2 + ng * o + ng * o / 2 + 4 * o + 4 * h + 4;
  if (nbytes < need)
    return fail(DGQ_EFORMAT,
                "truncated payload: have " + std::to_string(nbytes) + " bytes, header implies " + std::to_string(need),
                "truncated");
  if (nbytes > need) return fail(DGQ_EFORMAT, "payload longer than the header implies", "size_mismatch");
  const uint8_t* p = bytes + kHeader;
  const uint8_t* codes = p;
  p += h * o / 2;
  const int8_t* s2 = reinterpret_cast<const int8_t*>(p);
  p += ng * o;
  const uint8_t* zp = p;
  p += ng * o / 2;
  std::vector<float> s1(o), k(h);
  std::memcpy(s1.data(), p, 4 * o);
  p += 4 * o;
  std::memcpy(k.data(), p, 4 * h);
  p += 4 * h;
  float act_scale;
  std::memcpy(&act_scale, p, 4);
  return dgq_layer_create(device, h, o, g, mode, act_scale, codes, s2, zp, s1.data(), k.data(), col_begin, col_end,
                          1, stream, out);
}

// DGQ1 file -> prepared (sharded) layer without holding the artifact in host
// memory: header, S2 / ZP / s1 / k / act_scale are read first (small), then the
// code rows stream through two pinned slabs into the GPU validator + repack.
dgq_status dgq_layer_create_from_dgq1_file(int device, const char* path, size_t col_begin, size_t col_end,
                                           void* stream, dgq_layer** out) {
  constexpr size_t kHeader = 29;
  if (!path || !out) return fail(DGQ_EINVAL, "null argument");
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return fail(DGQ_EIO, std::string("cannot open: ") + path, "io");  // read_dgq, proj/src/format.cpp:276-278
  struct Closer {
    std::FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  fseeko(f, 0, SEEK_END);
  const long long nbytes = static_cast<long long>(ftello(f));
  fseeko(f, 0, SEEK_SET);
  uint8_t hdr[kHeader];
  if (nbytes < static_cast<long long>(kHeader) || std::fread(hdr, 1, kHeader, f) != kHeader)
    return fail(DGQ_EFORMAT, "truncated: DGQ file shorter than the header", "truncated");
  if (std::memcmp(hdr, "DGQ1", 4) != 0) return fail(DGQ_EFORMAT, "bad magic, expected \"DGQ1\"", "bad_magic");
  auto u64 = [&](size_t off) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(hdr[off + i]) << (8 * i);
    return v;
  };
  const uint64_t h = u64(4), o = u64(12), g = u64(20);
  const uint8_t mode = hdr[28];
  if (mode > 1) return fail(DGQ_EFORMAT, "unknown mode byte " + std::to_string(int(mode)), "bad_header");
  if (h == 0 || o == 0 || o % 2 || g == 0 || h % g)
    return fail(DGQ_EFORMAT, "inconsistent dimensions in header", "bad_header");
  if (h > (1ull << 30) || o > (1ull << 30)) return fail(DGQ_EFORMAT, "dimensions too large", "bad_header");
  const uint64_t ng = h / g;
  const uint64_t need = kHeader + h * o / 2 + ng * o + ng * o / 2 + 4 * o + 4 * h + 4;
  if (static_cast<uint64_t>(nbytes) < need)
    return fail(DGQ_EFORMAT,
                "truncated payload: have " + std::to_string(nbytes) + " bytes, header implies " + std::to_string(need),
                "truncated");
  if (static_cast<uint64_t>(nbytes) > need)
    return fail(DGQ_EFORMAT, "payload longer than the header implies", "size_mismatch");
  const long long off_s2 = kHeader + h * o / 2;
  std::vector<int8_t> s2(ng * o);
  std::vector<uint8_t> zp(ng * o / 2);
  std::vector<float> s1(o), k(h);
  float act_scale = 0.0f;
  fseeko(f, static_cast<off_t>(off_s2), SEEK_SET);
  if (std::fread(s2.data(), 1, s2.size(), f) != s2.size() || std::fread(zp.data(), 1, zp.size(), f) != zp.size() ||
      std::fread(s1.data(), 4, o, f) != o || std::fread(k.data(), 4, h, f) != h ||
      std::fread(&act_scale, 4, 1, f) != 1)
    return fail(DGQ_EIO, std::string("read failed: ") + path, "io");
  // two pinned row slabs (the loader's slab is <= 32 MB of the shard; full rows are read)
  const size_t pitch = o / 2;
  uint8_t* pinned[2] = {nullptr, nullptr};
  size_t cap = 0;
  cudaEvent_t done[2] = {nullptr, nullptr};
  int prev_dev = 0;
  DGQ_CUDA(cudaGetDevice(&prev_dev));
  DGQ_CUDA(cudaSetDevice(device));
  for (auto& e : done) DGQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaSetDevice(prev_dev);
  bool used[2] = {false, false};
  RowFetch fetch = [&](size_t r0, size_t rows, int b) -> const uint8_t* {
    const size_t bytes = rows * pitch;
    if (used[b]) cudaEventSynchronize(done[b]);  // the previous copy out of this slab finished
    if (bytes > cap) {
      for (auto& p : pinned) {
        cudaFreeHost(p);
        p = nullptr;
      }
      if (cudaHostAlloc(&pinned[0], bytes, cudaHostAllocDefault) != cudaSuccess ||
          cudaHostAlloc(&pinned[1], bytes, cudaHostAllocDefault) != cudaSuccess)
        return nullptr;
      cap = bytes;
    }
    fseeko(f, static_cast<off_t>(kHeader + r0 * pitch), SEEK_SET);
    if (std::fread(pinned[b], 1, bytes, f) != bytes) return nullptr;
    used[b] = true;
    return pinned[b];
  };
  dgq_status st = create_layer(device, h, o, g, mode, act_scale, fetch, nullptr, s2.data(), zp.data(), s1.data(),
                               k.data(), col_begin, col_end, 1, stream, out, done);
  if (st == DGQ_EINVAL && !dgq_layout::fused_ok(static_cast<int>(g))) {
    // exotic group sizes need the codes in memory: read them whole
    std::vector<uint8_t> codes(h * o / 2);
    fseeko(f, static_cast<off_t>(kHeader), SEEK_SET);
    if (std::fread(codes.data(), 1, codes.size(), f) != codes.size())
      st = fail(DGQ_EIO, std::string("read failed: ") + path, "io");
    else
      st = dgq_layer_create(device, h, o, g, mode, act_scale, codes.data(), s2.data(), zp.data(), s1.data(),
                            k.data(), col_begin, col_end, 1, stream, out);
  }
  for (auto& p : pinned) cudaFreeHost(p);
  for (auto& e : done) cudaEventDestroy(e);
  return st;
}

dgq_status dgq_layer_get_info(const dgq_layer* L, dgq_layer_info* info) {
  if (!L || !info) return fail(DGQ_EINVAL, "null argument");
  info->h = L->h;
  info->o_full = L->o_full;
  info->o = L->o;
  info->col_begin = L->c0;
  info->g = L->g;
  info->k_pad = L->k_pad;
  info->n_pad = L->n_pad;
  info->mode = L->mode;
  info->act_scale = L->act_scale;
  info->fused = L->fused ? 1 : 0;
  info->device_bytes = L->device_bytes;
  return DGQ_OK;
}

size_t dgq_linear_workspace_bytes(const dgq_layer* L, size_t M) {
  if (!L || M == 0) return 0;
  DgqGemmPlan pl = dgq_plan_gemm(static_cast<int>(M), static_cast<int>(L->o), static_cast<int>(L->k_pad), L->fused,
                                 static_cast<int>(L->g));
  return pl.ws_bytes + pl.counter_bytes;
}

dgq_status dgq_linear_plan(const dgq_layer* L, size_t M, int* token_tile, int* weight_tiles, int* k_splits,
                           int* ctas) {
  if (!L || M == 0) return fail(DGQ_EINVAL, "null layer or M == 0");
  DgqGemmPlan pl = dgq_plan_gemm(static_cast<int>(M), static_cast<int>(L->o), static_cast<int>(L->k_pad), L->fused,
                                 static_cast<int>(L->g));
  if (token_tile) *token_tile = pl.bn;
  if (weight_tiles) *weight_tiles = pl.nt;
  if (k_splits) *k_splits = pl.splits;
  if (ctas) *ctas = (pl.decode || pl.prefill2) ? pl.ctas : pl.m_tiles * ((pl.n_tiles + pl.nt - 1) / pl.nt) * pl.splits;
  return DGQ_OK;
}

dgq_status dgq_quantize_act_raw(const float* dX, size_t M, size_t K, size_t ldx, const float* dK, int mode,
                                float act_scale, int8_t* dXq, size_t ldq, float* dRowScale, void* stream) {
  DGQ_NVTX("dgq_quantize_act_raw");
  if (M == 0) return DGQ_OK;
  if (!dX || !dK || !dXq || !dRowScale) return fail(DGQ_EINVAL, "null argument");
  if (ldx < K || ldq < K) return fail(DGQ_EINVAL, "leading dimension smaller than the row length");
  if (M > 0x7FFFFFFF || K > 0x7FFFFFFF) return fail(DGQ_EINVAL, "too large");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* rk = nullptr;
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rk), (K ? K : 1) * sizeof(float), st));
  DGQ_CUDA(dgq_launch_reciprocal(dK, rk, static_cast<int>(K), st));
  cudaError_t e = dgq_launch_actquant2(dX, false, ldx, static_cast<int>(K), 0, dK, rk, static_cast<int>(K),
                                       static_cast<int>(ldq), mode != 0, act_scale, dXq, ldq, dRowScale,
                                       static_cast<int>(M), st);
  cudaFreeAsync(rk, st);
  DGQ_CUDA(e);
  return DGQ_OK;
}

/* not in the public header: test hook pinning the hoisted-reciprocal division to IEEE div.rn */
dgq_status dgq_debug_div_check(const float* dx, const float* dk, float* dfast, float* dieee, size_t n, void* stream) {
  DGQ_CUDA(dgq_launch_div_check(dx, dk, dfast, dieee, static_cast<int>(n), static_cast<cudaStream_t>(stream)));
  return DGQ_OK;
}

dgq_status dgq_quantize_act_f16(const dgq_layer* L, const void* dX, size_t M, size_t ldx, size_t seg_cols,
                                size_t seg_stride, int8_t* dXq, size_t ldq, float* dRowScale, void* stream) {
  DGQ_NVTX("dgq_quantize_act_f16");
  if (!L) return fail(DGQ_EINVAL, "null layer");
  if (M == 0) return DGQ_OK;
  if (!dX || !dXq || !dRowScale) return fail(DGQ_EINVAL, "null argument");
  const size_t seg = seg_cols ? seg_cols : L->h;
  if (L->h % seg) return fail(DGQ_EINVAL, "seg_cols must divide h");
  if (ldx < seg || ldq < L->h) return fail(DGQ_EINVAL, "leading dimension smaller than the row length");
  if (seg_cols && seg_stride < M * ldx) return fail(DGQ_EINVAL, "seg_stride smaller than one shard");
  DGQ_CUDA(dgq_launch_actquant2(dX, true, ldx, static_cast<int>(seg), seg_stride, L->k, L->rk,
                                static_cast<int>(L->h), static_cast<int>(ldq), L->mode, L->act_scale, dXq, ldq,
                                dRowScale, static_cast<int>(M), static_cast<cudaStream_t>(stream), L->ksm, L->spec, L->nspec));
  return DGQ_OK;
}

dgq_status dgq_quantize_act(const dgq_layer* L, const float* dX, size_t M, size_t ldx, int8_t* dXq, size_t ldq,
                            float* dRowScale, void* stream) {
  DGQ_NVTX("dgq_quantize_act");
  if (!L) return fail(DGQ_EINVAL, "null layer");
  if (M == 0) return DGQ_OK;
  if (!dX || !dXq || !dRowScale) return fail(DGQ_EINVAL, "null argument");
  if (ldx < L->h || ldq < L->h) return fail(DGQ_EINVAL, "leading dimension smaller than the row length");
  if (M > 0x7FFFFFFF) return fail(DGQ_EINVAL, "too many rows");
  DGQ_CUDA(dgq_launch_actquant2(dX, false, ldx, static_cast<int>(L->h), 0, L->k, L->rk, static_cast<int>(L->h),
                                static_cast<int>(ldq), L->mode, L->act_scale, dXq, ldq, dRowScale,
                                static_cast<int>(M), static_cast<cudaStream_t>(stream), L->ksm, L->spec, L->nspec));
  return DGQ_OK;
}

struct DecodeSub {
  const uint8_t* tiles;
  const float* s1;
  const float* bias;
  void* out;
  size_t ldy;
  int N;
};

// K5d stages whose weight chunks are requested before the kernel waits for its
// predecessor (PDL): the weights stream while the previous kernel drains.
// tools/dec_step.py (OPT-30B decode layer, graph replay, L2 flushed): 1 / 2 /
// 3 / 4 stages -> 115.6 / 112.9 / 112.2 / 112.9 us at M = 1, 138.0 / 136.5 /
// 135.1 / 135.4 us at M = 16.  DGQ_DEC_PRE overrides it (tools).
static int decode_pre_stages() {
  static const int v = [] {
    const char* e = getenv("DGQ_DEC_PRE");
    return e ? atoi(e) : 3;
  }();
  return v;
}

// K5d over `count` layers that share the input (one stream-K problem over the
// concatenation of their weight tiles).  ws: dgq_decode_workspace(total tiles).
static dgq_status run_decode(const DecodeSub* subs, int count, int g, size_t k_pad, const int8_t* dXq, size_t ldq,
                             size_t M, const float* dRs, int out_dtype, int fp16_mode, int32_t* dAcc, size_t ld_acc,
                             void* ws, cudaStream_t st) {
  int total_tiles = 0;
  for (int i = 0; i < count; ++i) total_tiles += (subs[i].N + 127) / 128;
  DgqGemmPlan pl = dgq_plan_gemm(static_cast<int>(M), total_tiles * 128, static_cast<int>(k_pad), true, g);
  if (!pl.decode) return fail(DGQ_EINVAL, "not a decode-shaped call");
  DgqDecodeParams d{};
  d.nsub = count;
  int tb = 0;
  for (int i = 0; i < count; ++i) {
    d.sub[i] = DgqDecodeSub{subs[i].tiles, subs[i].s1, subs[i].bias, subs[i].out, subs[i].ldy, subs[i].N, tb};
    tb += (subs[i].N + 127) / 128;
  }
  d.chunk_bytes = static_cast<uint32_t>(dgq_layout::chunk_bytes(g));
  d.chunk_stride = d.chunk_bytes;
  d.gpk = g >= 128 ? 1 : 128 / g;
  d.gshift = 7;
  if (g < 128) {
    d.gshift = 0;
    while ((1 << d.gshift) < g) ++d.gshift;
  }
  {
    // units per stage: as many as the TMEM partial ring allows with >= 2 slots
    const int per = d.gpk * pl.bn;
    const int ku = dgq_decode_partial_cols() / 2 / per;
    const int ups = dgq_decode_units_per_stage(pl.bn);
    d.ku = ku < 1 ? 1 : (ku > ups ? ups : ku);
    const int room = dgq_decode_partial_cols() / (d.ku * per);  // TMEM columns of the partial ring
    d.sd_log2 = room >= 8 ? 3 : (room >= 4 ? 2 : (room >= 2 ? 1 : 0));
  }
  CUtensorMap tmB;
  dgq_status ms =
      make_tmap_kblocks(&tmB, dXq, M, k_pad, ldq, static_cast<uint32_t>(pl.bn), static_cast<uint32_t>(d.ku));
  if (ms != DGQ_OK) return ms;
  d.M = static_cast<int>(M);
  d.n_tiles = total_tiles;
  d.k_blocks = static_cast<int>(k_pad / 128);
  d.rs = dRs;
  d.out_f16 = out_dtype == DGQ_OUT_F16;
  d.fp16_mode = fp16_mode;
  d.acc_out = count == 1 ? dAcc : nullptr;
  d.ld_acc = ld_acc;
  d.ws = static_cast<int32_t*>(ws);
  d.counters = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + pl.ws_bytes);
  d.dbg = ((dgq_debug_decode_mode() >> 1) & 0x7F) | ((dgq_debug_decode_mode() >> 12) & 0x1C00) | ((dgq_debug_decode_mode() >> 7) & 0x380);  // tools: mode bits 14-16, 22-24 -> dbg bits 7-9, 10-12
  d.trace = g_dbg_ts;
  d.trace_cta = 0;
  d.pre_stages = decode_pre_stages();
  DGQ_CUDA(dgq_launch_decode(pl.bn, tmB, d, pl.ctas, pl.pdl != 0, st));
  return DGQ_OK;
}

// One fused linear launch.  `count` > 1: layers sharing the input run as one
// K5p stream-K problem over the concatenation of their pair tiles (prefill-
// shaped calls of dgq_linear_multi; the caller checked the plan is K5p).
static dgq_status run_gemm(bool fused, const DecodeSub* subs, int count, const CUtensorMap& tmA, int g, size_t k_pad,
                           const int8_t* dXq, size_t ldq, size_t M, const float* dRs, int out_dtype, int fp16_mode,
                           int32_t* dAcc, size_t ld_acc, void* ws, size_t ws_bytes, cudaStream_t st) {
  const uint8_t* tiles = subs[0].tiles;
  const float *dS1 = subs[0].s1, *dBias = subs[0].bias;
  void* dY = subs[0].out;
  const size_t ldy = subs[0].ldy;
  size_t N = static_cast<size_t>(subs[0].N);
  if (count > 1) {  // plan on the concatenation (128-channel tiles)
    N = 0;
    for (int i = 0; i < count; ++i) N += static_cast<size_t>((subs[i].N + 127) / 128) * 128;
  }
  DgqGemmPlan pl = dgq_plan_gemm(static_cast<int>(M), static_cast<int>(N), static_cast<int>(k_pad), fused, g);
  if (count > 1 && !pl.prefill2) return fail(DGQ_EINVAL, "multi-layer launch is only planned for the pair kernel");
  if (pl.ws_bytes + pl.counter_bytes > ws_bytes)
    return fail(DGQ_EINVAL, "workspace too small: need " + std::to_string(pl.ws_bytes + pl.counter_bytes));
  CUtensorMap tmB{};
  dgq_status ms = DGQ_OK;
  if (!pl.prefill2) {  // K5p builds its own 128-row map below
    ms = make_tmap(&tmB, dXq, M, k_pad, ldq, static_cast<uint32_t>(pl.bn));
    if (ms != DGQ_OK) return ms;
  }
  if (pl.decode) {
    if (!ws) return fail(DGQ_EINVAL, "decode kernel needs a workspace");
    DecodeSub one{tiles, dS1, dBias, dY, ldy, static_cast<int>(N)};
    return run_decode(&one, 1, g, k_pad, dXq, ldq, M, dRs, out_dtype, fp16_mode, dAcc, ld_acc, ws, st);
  }
  DgqGemmParams p{};
  p.tiles = tiles;
  p.chunk_bytes = static_cast<uint32_t>(dgq_layout::chunk_bytes(g > 0 ? g : 128));
  p.chunk_stride = (p.chunk_bytes + 1023u) & ~1023u;
  p.gshift = 7;
  if (g > 0 && g < 128) {
    p.gshift = 0;
    while ((1 << p.gshift) < g) ++p.gshift;
  }
  p.M = static_cast<int>(M);
  p.N = static_cast<int>(N);
  p.k_blocks = static_cast<int>(k_pad / 128);
  p.kb_per_split = pl.kb_per_split;
  p.splits = pl.splits;
  p.rs = dRs;
  p.s1 = dS1;
  p.bias = dBias;
  p.out = dY;
  p.ldy = ldy;
  p.out_f16 = out_dtype == DGQ_OUT_F16;
  p.fp16_mode = fp16_mode;
  p.acc_out = dAcc;
  p.ld_acc = ld_acc;
  {
    const size_t esz = out_dtype == DGQ_OUT_F16 ? 2 : 4;
    bool ok = true;
    for (int i = 0; i < count; ++i)
      if (subs[i].out)
        ok = ok && (reinterpret_cast<uintptr_t>(subs[i].out) % 16 == 0) && ((subs[i].ldy * esz) % 16 == 0);
    if (dAcc) ok = ok && (reinterpret_cast<uintptr_t>(dAcc) % 16 == 0) && ((ld_acc * 4) % 16 == 0);
    p.vec_ok = ok ? 1 : 0;
  }
  CUtensorMap tmY{};
  if (pl.bn >= 128 && dY && p.vec_ok && count == 1) {
    dgq_status ys = make_out_tmap(&tmY, dY, M, N, ldy, out_dtype == DGQ_OUT_F16);
    if (ys != DGQ_OK) return ys;
    p.tma_out = 1;
  }
  p.dbg = g_dbg_ts;
  if (pl.prefill2) {
    CUtensorMap tmX;
    ms = make_tmap(&tmX, dXq, M, k_pad, ldq, 128u);
    if (ms != DGQ_OK) return ms;
    p.chunk_stride = p.chunk_bytes;
    p.dbg_flags = (dgq_debug_decode_mode() >> 18) & 31;  // tools: mode bits 18-22
    p.nsub = count;
    int tb = 0;
    for (int i = 0; i < count; ++i) {
      p.sub[i] = DgqDecodeSub{subs[i].tiles, subs[i].s1, subs[i].bias, subs[i].out, subs[i].ldy, subs[i].N, tb};
      tb += (subs[i].N + pl.pair_tn - 1) / pl.pair_tn;
    }
    p.n_pair_tiles = tb;
    if (pl.stream_k) {
      if (!ws) return fail(DGQ_EINVAL, "stream-K prefill kernel needs a workspace");
      p.stream_k = 1;
      p.ws = static_cast<int32_t*>(ws);
      p.counters = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + pl.ws_bytes);
    }
    DGQ_CUDA(dgq_launch_prefill2(tmX, tmY, p, pl.pair_tn, pl.pair_sub, pl.pdl != 0, st));
    return DGQ_OK;
  }
  DGQ_CUDA(dgq_launch_gemm(pl, fused, tmB, tmA, tmY, p, st));
  return DGQ_OK;
}

dgq_status dgq_linear(const dgq_layer* Lc, const int8_t* dXq, size_t ldq, const float* dRs, size_t M,
                      const float* dBias, int out_dtype, int fp16_mode, void* dY, size_t ldy, int32_t* dAcc,
                      size_t ld_acc, void* dWorkspace, size_t ws_bytes, void* stream) {
  DGQ_NVTX("dgq_linear");
  auto* L = const_cast<dgq_layer*>(Lc);
  if (!L) return fail(DGQ_EINVAL, "null layer");
  if (M == 0) return DGQ_OK;
  {
    dgq_status s = check_linear_args(L, dXq, ldq, dRs, M, dY, ldy, dAcc, ld_acc);
    if (s != DGQ_OK) return s;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const DecodeSub one{L->tiles, L->s1, dBias, dY, ldy, static_cast<int>(L->o)};
  const size_t need = dgq_linear_workspace_bytes(L, M);
  void* ws = dWorkspace;
  if (need && !ws) {
    std::lock_guard<std::mutex> lk(L->ws_mu);
    dgq_status s = ws_acquire(L, st, need, &ws, &ws_bytes);
    if (s != DGQ_OK) return s;
    s = run_gemm(L->fused, &one, 1, L->tmA, static_cast<int>(L->g), L->k_pad, dXq, ldq, M, dRs, out_dtype, fp16_mode,
                 dAcc, ld_acc, ws, ws_bytes, st);
    ws_release(L, st);
    return s;
  }
  return run_gemm(L->fused, &one, 1, L->tmA, static_cast<int>(L->g), L->k_pad, dXq, ldq, M, dRs, out_dtype, fp16_mode,
                  dAcc, ld_acc, ws, ws_bytes, st);
}

dgq_status dgq_forward_device(const dgq_layer* L, const float* dX, size_t M, size_t ldx, const float* dBias,
                              int out_dtype, void* dY, size_t ldy, int8_t* dXq, float* dRs, void* dWorkspace,
                              size_t ws_bytes, void* stream) {
  DGQ_NVTX("dgq_forward_device");
  if (!L) return fail(DGQ_EINVAL, "null layer");
  dgq_status s = dgq_quantize_act(L, dX, M, ldx, dXq, L->k_pad, dRs, stream);
  if (s != DGQ_OK) return s;
  return dgq_linear(L, dXq, L->k_pad, dRs, M, dBias, out_dtype, 0, dY, ldy, nullptr, 0, dWorkspace, ws_bytes,
                    stream);
}

dgq_status dgq_calibrate(const float* dX, size_t rows, size_t h, size_t ldx, float percentile, int fp16_scales,
                         float* k_out, float* threshold_out, float* act_scale_out, void* stream) {
  DGQ_NVTX("dgq_calibrate");
  if (!dX || !k_out) return fail(DGQ_EINVAL, "null argument");
  if (rows == 0 || h == 0) return fail(DGQ_EINVAL, "empty calibration set");
  if (ldx < h) return fail(DGQ_EINVAL, "leading dimension smaller than the row length");
  if (rows > 0x7FFFFFFF || h > 0x7FFFFFFF) return fail(DGQ_EINVAL, "too large");
  if (!(percentile > 0.0f && percentile < 1.0f)) return fail(DGQ_EINVAL, "percentile must be in (0, 1)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned* dz = nullptr;
  float* dk = nullptr;
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dz), (h + 1) * sizeof(unsigned), st));
  DGQ_CUDA(cudaMemsetAsync(dz, 0, (h + 1) * sizeof(unsigned), st));
  DGQ_CUDA(dgq_launch_colmax(dX, ldx, static_cast<int>(rows), static_cast<int>(h), dz, st));
  std::vector<float> z(h);
  DGQ_CUDA(cudaMemcpyAsync(z.data(), dz, h * sizeof(float), cudaMemcpyDeviceToHost, st));
  DGQ_CUDA(cudaStreamSynchronize(st));
  // compute_smooth (proj/src/smoothing.cpp:26-49): rank-th largest channel maximum
  size_t rank = static_cast<size_t>(std::ceil(static_cast<double>(percentile) * static_cast<double>(h)));
  rank = std::max<size_t>(rank, 1);
  std::vector<float> sorted = z;
  std::nth_element(sorted.begin(), sorted.begin() + (rank - 1), sorted.end(), std::greater<float>());
  const float threshold = sorted[rank - 1];
  if (!(threshold > 0.0f)) {
    cudaFreeAsync(dz, st);
    return fail(DGQ_EINVAL, "smoothing undefined: percentile threshold is not positive (all-zero calibration?)");
  }
  for (size_t j = 0; j < h; ++j) {
    float v = std::max(1.0f, z[j] / threshold);
    if (fp16_scales) v = std::max(1.0f, dgq_fp16_round(v));  // proj/src/pipeline.cpp:354-356
    k_out[j] = v;
  }
  if (threshold_out) *threshold_out = threshold;
  if (act_scale_out) {
    DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dk), h * sizeof(float), st));
    DGQ_CUDA(cudaMemcpyAsync(dk, k_out, h * sizeof(float), cudaMemcpyHostToDevice, st));
    DGQ_CUDA(dgq_launch_smooth_absmax(dX, ldx, static_cast<int>(rows), static_cast<int>(h), dk, dz + h, st));
    unsigned bits = 0;
    DGQ_CUDA(cudaMemcpyAsync(&bits, dz + h, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    DGQ_CUDA(cudaStreamSynchronize(st));
    float absmax;
    std::memcpy(&absmax, &bits, sizeof(float));
    // static_act_scale (proj/src/pipeline.cpp:96-101), kScaleFloor = 1e-8f
    float s = static_cast<float>(std::max(static_cast<double>(absmax) / 127.0, static_cast<double>(1e-8f)));
    if (fp16_scales) s = dgq_fp16_round(s);  // proj/src/pipeline.cpp:361
    *act_scale_out = s;
    cudaFreeAsync(dk, st);
  }
  cudaFreeAsync(dz, st);
  return DGQ_OK;
}

dgq_status dgq_layer_dequant_s8(const dgq_layer* L, int8_t* dW, size_t ldw, void* stream) {
  DGQ_NVTX("dgq_layer_dequant_s8");
  if (!L || !dW) return fail(DGQ_EINVAL, "null argument");
  if (ldw < L->o) return fail(DGQ_EINVAL, "ldw smaller than the shard width");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (L->fused) {
    DGQ_CUDA(dgq_launch_dequant_tiles(L->tiles, static_cast<int>(L->g), static_cast<int>(L->h),
                                      static_cast<int>(L->o), L->n_tiles, L->k_blocks, dW, ldw, st));
  } else {
    // transpose back from the K-major copy
    DGQ_CUDA(dgq_launch_transpose_pad(L->wt, static_cast<int>(L->n_pad), static_cast<int>(L->k_pad), dW,
                                      static_cast<int>(L->o), static_cast<int>(L->h), st));
  }
  return DGQ_OK;
}

dgq_status dgq_dequantize_to_s8(size_t h, size_t o, size_t g, const uint8_t* d_codes, const int8_t* d_s2,
                                const uint8_t* d_zp, int8_t* dW, void* stream) {
  if (h == 0 || o == 0 || o % 2 || g == 0 || h % g) return fail(DGQ_EINVAL, "inconsistent layer shape");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* d_bad = nullptr;
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_bad), sizeof(unsigned long long), st));
  DGQ_CUDA(cudaMemsetAsync(d_bad, 0xFF, sizeof(unsigned long long), st));
  DGQ_CUDA(dgq_launch_dequant_ref(d_codes, d_s2, d_zp, static_cast<int>(h), static_cast<int>(o), static_cast<int>(g),
                                  dW, d_bad, st));
  unsigned long long bad = 0;
  DGQ_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
  DGQ_CUDA(cudaFreeAsync(d_bad, st));
  DGQ_CUDA(cudaStreamSynchronize(st));
  if (bad != ~0ull) {
    const size_t i = bad / o, c = bad % o;
    return fail(DGQ_EVALIDATION,
                "dequantized 8-bit weight at (" + std::to_string(i) + ", " + std::to_string(c) +
                    ") outside [-127, 127]; artifact is corrupted",
                "codes");
  }
  return DGQ_OK;
}

dgq_status dgq_audit_max_abs_acc(const int8_t* dXq, size_t ldx, const int8_t* dW, size_t ldw, size_t M, size_t K,
                                 size_t N, int64_t* max_abs_acc, void* stream) {
  if (!max_abs_acc) return fail(DGQ_EINVAL, "null output");
  *max_abs_acc = 0;
  if (M == 0 || N == 0 || K == 0) return DGQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* d = nullptr;
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned long long), st));
  DGQ_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), st));
  DGQ_CUDA(dgq_launch_audit(dXq, ldx, dW, ldw, static_cast<int>(M), static_cast<int>(K), static_cast<int>(N), d, st));
  unsigned long long v = 0;
  DGQ_CUDA(cudaMemcpyAsync(&v, d, sizeof(v), cudaMemcpyDeviceToHost, st));
  DGQ_CUDA(cudaFreeAsync(d, st));
  DGQ_CUDA(cudaStreamSynchronize(st));
  *max_abs_acc = static_cast<int64_t>(v);
  return DGQ_OK;
}

dgq_status dgq_int8_gemm(const int8_t* dXq, size_t ldx, const int8_t* dW, size_t ldw, size_t M, size_t K, size_t N,
                         int32_t* dAcc, size_t ld_acc, int64_t* max_abs_acc, void* stream) {
  DGQ_NVTX("dgq_int8_gemm");
  if (static_cast<double>(K) * 127.0 * 127.0 >= 2147483648.0)
    return fail(DGQ_EINVAL, "h too large for 32-bit accumulation");
  if (max_abs_acc) *max_abs_acc = 0;
  if (M == 0 || N == 0) return DGQ_OK;
  if (!dXq || !dW || !dAcc) return fail(DGQ_EINVAL, "null argument");
  if (ldx < K || ldw < N || ld_acc < N) return fail(DGQ_EINVAL, "leading dimension too small");
  if (M > 0x7FFFFFFF || N > (1u << 30)) return fail(DGQ_EINVAL, "too large");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t k_pad = round_up(K ? K : 1, 128), n_pad = round_up(N, 128);
  int8_t *wt = nullptr, *xq = nullptr;
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&wt), n_pad * k_pad, st));
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&xq), M * k_pad, st));
  // W [K x N] (ld = ldw) -> WT [n_pad x k_pad]
  const int8_t* wsrc = dW;
  int8_t* wdense = nullptr;
  if (ldw != N) {
    DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&wdense), K * N ? K * N : 1, st));
    DGQ_CUDA(cudaMemcpy2DAsync(wdense, N, dW, ldw, N, K, cudaMemcpyDeviceToDevice, st));
    wsrc = wdense;
  }
  DGQ_CUDA(dgq_launch_transpose_pad(wsrc, static_cast<int>(K), static_cast<int>(N), wt, static_cast<int>(k_pad),
                                    static_cast<int>(n_pad), st));
  DGQ_CUDA(cudaMemsetAsync(xq, 0, M * k_pad, st));
  if (K) DGQ_CUDA(cudaMemcpy2DAsync(xq, k_pad, dXq, ldx, K, M, cudaMemcpyDeviceToDevice, st));
  CUtensorMap tmA;
  dgq_status s = make_tmap(&tmA, wt, n_pad, k_pad, k_pad, 128);
  void* ws = nullptr;
  DgqGemmPlan pl = dgq_plan_gemm(static_cast<int>(M), static_cast<int>(N), static_cast<int>(k_pad), false, 128);
  const size_t need = pl.ws_bytes + pl.counter_bytes;
  if (s == DGQ_OK && need) {
    DGQ_CUDA(cudaMallocAsync(&ws, need, st));
    DGQ_CUDA(cudaMemsetAsync(ws, 0, need, st));
  }
  if (s == DGQ_OK) {
    const DecodeSub plain{nullptr, nullptr, nullptr, nullptr, 0, static_cast<int>(N)};
    s = run_gemm(false, &plain, 1, tmA, 128, k_pad, xq, k_pad, M, nullptr, DGQ_OUT_F32, 0, dAcc, ld_acc, ws, need, st);
  }
  if (s == DGQ_OK && max_abs_acc) s = dgq_audit_max_abs_acc(dXq, ldx, dW, ldw, M, K, N, max_abs_acc, stream);
  if (ws) cudaFreeAsync(ws, st);
  if (wdense) cudaFreeAsync(wdense, st);
  cudaFreeAsync(wt, st);
  cudaFreeAsync(xq, st);
  if (s == DGQ_OK && max_abs_acc && *max_abs_acc > 2147483647LL)
    return fail(DGQ_EOVERFLOW, "int8_gemm accumulator overflow despite precondition");
  return s;
}

dgq_status dgq_epilogue(const int32_t* dAcc, size_t lda, const float* dRs, const float* dS1, const float* dBias,
                        size_t M, size_t N, int fp16_mode, int out_dtype, void* dY, size_t ldy, void* stream) {
  if (M == 0 || N == 0) return DGQ_OK;
  if (!dAcc || !dRs || !dS1 || !dY) return fail(DGQ_EINVAL, "null argument");
  if (lda < N || ldy < N) return fail(DGQ_EINVAL, "leading dimension too small");
  DGQ_CUDA(dgq_launch_epilogue(dAcc, lda, dRs, dS1, dBias, static_cast<int>(M), static_cast<int>(N), fp16_mode,
                               out_dtype == DGQ_OUT_F16, dY, ldy, static_cast<cudaStream_t>(stream)));
  return DGQ_OK;
}

dgq_status dgq_linear_multi(const dgq_layer* const* layers, int count, const int8_t* dXq, size_t ldq,
                            const float* dRowScale, size_t M, const float* const* dBias, int out_dtype,
                            void* const* dY, const size_t* ldy, void* dWorkspace, size_t ws_bytes, void* stream) {
  DGQ_NVTX("dgq_linear_multi");
  if (!layers || count < 1 || count > kDecodeMaxSub || !dY || !ldy)
    return fail(DGQ_EINVAL, "dgq_linear_multi: 1..4 layers with outputs");
  const dgq_layer* L0 = layers[0];
  for (int i = 0; i < count; ++i) {
    if (!layers[i] || !dY[i]) return fail(DGQ_EINVAL, "null layer or output");
    if (layers[i]->h != L0->h || layers[i]->g != L0->g || layers[i]->fused != L0->fused)
      return fail(DGQ_EINVAL, "dgq_linear_multi: layers must share h, g and the prepared layout");
    if (layers[i]->device != L0->device) return fail(DGQ_EINVAL, "dgq_linear_multi: layers on different devices");
  }
  if (M == 0) return DGQ_OK;
  for (int i = 0; i < count; ++i) {
    dgq_status s = check_linear_args(layers[i], dXq, ldq, dRowScale, M, dY[i], ldy[i], nullptr, 0);
    if (s != DGQ_OK) return s;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int total_tiles = 0;
  for (int i = 0; i < count; ++i) total_tiles += layers[i]->n_tiles;
  DgqGemmPlan pl = dgq_plan_gemm(static_cast<int>(M), total_tiles * 128, static_cast<int>(L0->k_pad), L0->fused,
                                 static_cast<int>(L0->g));
  if (pl.prefill2 && L0->fused) {
    // prefill-shaped: one K5p stream-K problem over the layers' pair tiles
    // (one launch, one tail, instead of one per layer)
    DecodeSub subs[kDecodeMaxSub];
    for (int i = 0; i < count; ++i)
      subs[i] = DecodeSub{layers[i]->tiles, layers[i]->s1, dBias ? dBias[i] : nullptr, dY[i], ldy[i],
                          static_cast<int>(layers[i]->o)};
    const size_t need = pl.ws_bytes + pl.counter_bytes;
    if (dWorkspace) {
      if (ws_bytes < need) return fail(DGQ_EINVAL, "workspace too small: need " + std::to_string(need));
      return run_gemm(true, subs, count, L0->tmA, static_cast<int>(L0->g), L0->k_pad, dXq, ldq, M, dRowScale,
                      out_dtype, 0, nullptr, 0, dWorkspace, ws_bytes, st);
    }
    auto* L = const_cast<dgq_layer*>(L0);
    std::lock_guard<std::mutex> lk(L->ws_mu);
    void* ws = nullptr;
    size_t cap = 0;
    dgq_status s = ws_acquire(L, st, need, &ws, &cap);
    if (s != DGQ_OK) return s;
    s = run_gemm(true, subs, count, L0->tmA, static_cast<int>(L0->g), L0->k_pad, dXq, ldq, M, dRowScale, out_dtype, 0,
                 nullptr, 0, ws, cap, st);
    ws_release(L, st);
    return s;
  }
  if (!pl.decode) {  // neither decode- nor pair-kernel-shaped: one launch per layer
    for (int i = 0; i < count; ++i) {
      dgq_status s = dgq_linear(layers[i], dXq, ldq, dRowScale, M, dBias ? dBias[i] : nullptr, out_dtype, 0, dY[i],
                                ldy[i], nullptr, 0, nullptr, 0, stream);
      if (s != DGQ_OK) return s;
    }
    return DGQ_OK;
  }
  const size_t need = pl.ws_bytes + pl.counter_bytes;
  void* ws = dWorkspace;
  DecodeSub subs[kDecodeMaxSub];
  for (int i = 0; i < count; ++i)
    subs[i] = DecodeSub{layers[i]->tiles, layers[i]->s1, dBias ? dBias[i] : nullptr, dY[i], ldy[i],
                        static_cast<int>(layers[i]->o)};
  if (!ws) {  // the first layer's internal workspace for this stream, grown to the combined problem
    auto* L = const_cast<dgq_layer*>(L0);
    std::lock_guard<std::mutex> lk(L->ws_mu);
    size_t cap = 0;
    dgq_status s = ws_acquire(L, st, need, &ws, &cap);
    if (s != DGQ_OK) return s;
    s = run_decode(subs, count, static_cast<int>(L0->g), L0->k_pad, dXq, ldq, M, dRowScale, out_dtype, 0, nullptr, 0,
                   ws, st);
    ws_release(L, st);
    return s;
  }
  if (ws_bytes < need) return fail(DGQ_EINVAL, "workspace too small: need " + std::to_string(need));
  return run_decode(subs, count, static_cast<int>(L0->g), L0->k_pad, dXq, ldq, M, dRowScale, out_dtype, 0, nullptr, 0,
                    ws, st);
}

size_t dgq_linear_multi_workspace_bytes(const dgq_layer* const* layers, int count, size_t M) {
  if (!layers || count < 1 || M == 0) return 0;
  int total_tiles = 0;
  for (int i = 0; i < count; ++i) total_tiles += layers[i] ? layers[i]->n_tiles : 0;
  DgqGemmPlan pl = dgq_plan_gemm(static_cast<int>(M), total_tiles * 128, static_cast<int>(layers[0]->k_pad),
                                 layers[0]->fused, static_cast<int>(layers[0]->g));
  return pl.ws_bytes + pl.counter_bytes;
}

// ---- offline quantiser: two-phase grid search -------------
static dgq_status upload_grid(const float* grid, size_t n, float** d, cudaStream_t st) {
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(d), n * sizeof(float), st));
  DGQ_CUDA(cudaMemcpyAsync(*d, grid, n * sizeof(float), cudaMemcpyHostToDevice, st));
  return DGQ_OK;
}

dgq_status dgq_phase1_search(const float* dW, size_t h, size_t o, const float* dX, const float* dXhat, size_t b,
                             size_t g, int n_bits, const float* alpha_grid, size_t n_alpha, float* dSprime,
                             int32_t* dZp, float* dErr, float* dAlpha, uint64_t* evals, void* stream) {
  DGQ_NVTX("dgq_phase1_search");
  // SearchConfig::validate (proj/src/search.cpp:24-45)
  if (g < 1 || h % g != 0)
    return fail(DGQ_EINVAL, "group size " + std::to_string(g) + " must divide h = " + std::to_string(h));
  if (n_bits < 2 || n_bits > 8) return fail(DGQ_EINVAL, "n_bits_w must be in [2, 8]");
  if (!alpha_grid || n_alpha == 0) return fail(DGQ_EINVAL, "alpha_grid_phase1 is empty");
  for (size_t i = 0; i < n_alpha; ++i)
    if (!(alpha_grid[i] > 0.0f && alpha_grid[i] <= 1.0f))
      return fail(DGQ_EINVAL, "alpha_grid_phase1 values must be in (0, 1]");
  if (evals) *evals = static_cast<uint64_t>(h / g) * o * n_alpha;
  if (o == 0 || h == 0) return DGQ_OK;
  if (!dW || (b && (!dX || !dXhat)) || !dSprime || !dZp || !dErr || !dAlpha) return fail(DGQ_EINVAL, "null argument");
  const size_t n_g = h / g;
  if (h > 0x7FFFFFFF || o * n_alpha > 0x7FFFFFFF || b > 0x7FFFFFFF || n_g > 65535)
    return fail(DGQ_EINVAL, "search problem too large");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float *da = nullptr, *mn = nullptr, *mx = nullptr;
  double *ref = nullptr, *err = nullptr;
  dgq_status s = upload_grid(alpha_grid, n_alpha, &da, st);
  if (s != DGQ_OK) return s;
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&mn), n_g * o * sizeof(float), st));
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&mx), n_g * o * sizeof(float), st));
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ref), (n_g * o * b + 1) * sizeof(double), st));
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&err), n_g * o * n_alpha * sizeof(double), st));
  cudaError_t e = dgq_launch_phase1(dW, dX, dXhat, static_cast<int>(h), static_cast<int>(o), static_cast<int>(b),
                                    static_cast<int>(g), (1 << n_bits) - 1, da, static_cast<int>(n_alpha), mn, mx,
                                    ref, err, dSprime, dZp, dErr, dAlpha, st);
  cudaFreeAsync(da, st);
  cudaFreeAsync(mn, st);
  cudaFreeAsync(mx, st);
  cudaFreeAsync(ref, st);
  cudaFreeAsync(err, st);
  DGQ_CUDA(e);
  return DGQ_OK;
}

dgq_status dgq_phase2_search(const float* dW, size_t h, size_t o, const float* dX, const float* dXhat, size_t b,
                             size_t g, const float* dSprime, const int32_t* dZp, const float* alpha_grid,
                             size_t n_alpha, float* dS1, int8_t* dS2, int32_t* dCodes, double* dColErr,
                             float* dColAlpha, uint64_t* evals, void* stream) {
  DGQ_NVTX("dgq_phase2_search");
  if (g == 0 || h % g != 0) return fail(DGQ_EINVAL, "GroupParams shape does not match weights");
  if (!alpha_grid || n_alpha == 0) return fail(DGQ_EINVAL, "alpha_grid_phase2 is empty");
  if (evals) *evals = static_cast<uint64_t>(o) * n_alpha;
  if (o == 0 || h == 0) return DGQ_OK;
  if (!dW || (b && (!dX || !dXhat)) || !dSprime || !dZp || !dS1 || !dS2 || !dCodes || !dColErr || !dColAlpha)
    return fail(DGQ_EINVAL, "null argument");
  const size_t n_g = h / g;
  if (h > 0x7FFFFFFF || o * n_alpha > 0x7FFFFFFF || b > 0x7FFFFFFF || n_g > 65535)
    return fail(DGQ_EINVAL, "search problem too large");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float *da = nullptr, *am = nullptr;
  double *ref = nullptr, *err = nullptr;
  dgq_status s = upload_grid(alpha_grid, n_alpha, &da, st);
  if (s != DGQ_OK) return s;
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&am), o * sizeof(float), st));
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ref), (o * b + 1) * sizeof(double), st));
  DGQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&err), o * n_alpha * sizeof(double), st));
  cudaError_t e = dgq_launch_phase2(dW, dX, dXhat, static_cast<int>(h), static_cast<int>(o), static_cast<int>(b),
                                    static_cast<int>(g), dSprime, dZp, da, static_cast<int>(n_alpha), am, ref, err,
                                    dS1, dS2, dCodes, dColErr, dColAlpha, st);
  cudaFreeAsync(da, st);
  cudaFreeAsync(am, st);
  cudaFreeAsync(ref, st);
  cudaFreeAsync(err, st);
  DGQ_CUDA(e);
  return DGQ_OK;
}

// ---- measured INT8 tensor peak (the roofline denominator) ----
dgq_status dgq_measure_i8_peak(int reps, double* tops, double* best_ms) {
  if (!tops) return fail(DGQ_EINVAL, "null argument");
  int dev = 0, sms = 148;
  DGQ_CUDA(cudaGetDevice(&dev));
  DGQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int pairs = sms / 2, blocks = 4096;
  unsigned long long* sink = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  DGQ_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  DGQ_CUDA(cudaMalloc(&sink, sizeof(unsigned long long)));
  DGQ_CUDA(cudaEventCreate(&e0));
  DGQ_CUDA(cudaEventCreate(&e1));
  float best = 1e30f;
  if (reps == 0) reps = 10;
  cudaError_t e = dgq_launch_i8_peak(pairs, blocks, sink, st);  // warm-up
  if (reps < 0) {
    // sustained: -reps launches back to back, timed as one span (the clock
    // the tensor pipe holds under continuous load, e.g. inside a long step)
    cudaEventRecord(e0, st);
    for (int i = 0; e == cudaSuccess && i < -reps; ++i) e = dgq_launch_i8_peak(pairs, blocks, sink, st);
    cudaEventRecord(e1, st);
    if (e == cudaSuccess) e = cudaEventSynchronize(e1);
    float ms = 0.0f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
    best = ms / static_cast<float>(-reps);
    reps = 0;
  }
  for (int i = 0; e == cudaSuccess && i < reps; ++i) {
    cudaEventRecord(e0, st);
    e = dgq_launch_i8_peak(pairs, blocks, sink, st);
    cudaEventRecord(e1, st);
    if (e == cudaSuccess) e = cudaEventSynchronize(e1);
    float ms = 0.0f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
    if (e == cudaSuccess && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  cudaStreamDestroy(st);
  DGQ_CUDA(e);
  const double ops = 2.0 * 256 * 256 * 32 * 4.0 * blocks * pairs;
  *tops = ops / (best * 1e-3) / 1e12;
  if (best_ms) *best_ms = best;
  return DGQ_OK;
}

}  // extern "C"
