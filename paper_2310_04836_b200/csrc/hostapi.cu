// Host-buffer entry points (include/dgq_b200.h, "host-buffer API"): the
// reference's own calling convention — host arrays in, host arrays out, every
// call self-contained — over the device entry points of capi.cu.  This is the
// layer the C++ drop-in (paper_2310_04836_b200/dropin/) and any FFI binding of
// proj/include/dgq/kernel.hpp call.  Each function uploads its inputs, runs
// the CUDA kernels on a per-thread stream of the current device, downloads the
// results and synchronises; scratch comes from the device's stream-ordered
// memory pool (kept cached between calls).  There is no CPU compute here.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dgq_b200.h"
#include "kernels.h"

extern "C" dgq_status dgq_internal_fail(dgq_status st, const char* msg, const char* field);

namespace {

dgq_status cuda_fail(cudaError_t e, const char* what) {
  const std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return dgq_internal_fail(e == cudaErrorMemoryAllocation ? DGQ_ENOMEM : DGQ_ECUDA, m.c_str(), "");
}

#define DGQ_H_CUDA(expr)                                \
  do {                                                  \
    cudaError_t e_ = (expr);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
  } while (0)
#define DGQ_H_TRY(expr)                 \
  do {                                  \
    dgq_status s_ = (expr);             \
    if (s_ != DGQ_OK) return s_;        \
  } while (0)

// Per-thread, per-device stream; the device's default pool keeps freed blocks.
struct ThreadStream {
  int dev = -1;
  cudaStream_t st = nullptr;
  ~ThreadStream() {
    if (st) cudaStreamDestroy(st);
  }
};
thread_local ThreadStream t_stream;

dgq_status host_stream(cudaStream_t* out) {
  int dev = 0;
  DGQ_H_CUDA(cudaGetDevice(&dev));
  if (t_stream.dev != dev || !t_stream.st) {
    if (t_stream.st) cudaStreamDestroy(t_stream.st);
    t_stream.st = nullptr;
    DGQ_H_CUDA(cudaStreamCreateWithFlags(&t_stream.st, cudaStreamNonBlocking));
    t_stream.dev = dev;
    static std::mutex mu;
    static bool pool_set[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 64 && !pool_set[dev]) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      pool_set[dev] = true;
    }
  }
  *out = t_stream.st;
  return DGQ_OK;
}

// Stream-ordered device scratch, freed (back to the pool) on scope exit.
struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  cudaError_t alloc(size_t n, cudaStream_t s) {
    st = s;
    return cudaMallocAsync(&p, n ? n : 16, s);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

dgq_status upload(DevBuf& b, const void* host, size_t n, cudaStream_t st) {
  DGQ_H_CUDA(b.alloc(n, st));
  if (n) DGQ_H_CUDA(cudaMemcpyAsync(b.p, host, n, cudaMemcpyHostToDevice, st));
  return DGQ_OK;
}

dgq_status download(void* host, const DevBuf& b, size_t n, cudaStream_t st) {
  if (n && host) DGQ_H_CUDA(cudaMemcpyAsync(host, b.p, n, cudaMemcpyDeviceToHost, st));
  return DGQ_OK;
}

size_t round_up(size_t v, size_t m) { return (v + m - 1) / m * m; }

// Per-thread copy streams and events of the serving call's pipeline (one set
// per host thread and device).
struct CopyLanes {
  int dev = -1;
  cudaStream_t in = nullptr, out = nullptr;
  static constexpr int kEv = 16;
  cudaEvent_t ev_in[kEv] = {}, ev_c[kEv] = {};
  ~CopyLanes() { release(); }
  void release() {
    if (in) cudaStreamDestroy(in);
    if (out) cudaStreamDestroy(out);
    for (int i = 0; i < kEv; ++i) {
      if (ev_in[i]) cudaEventDestroy(ev_in[i]);
      if (ev_c[i]) cudaEventDestroy(ev_c[i]);
      ev_in[i] = ev_c[i] = nullptr;
    }
    in = out = nullptr;
  }
};
thread_local CopyLanes t_lanes;

dgq_status copy_lanes(CopyLanes** out) {
  int dev = 0;
  DGQ_H_CUDA(cudaGetDevice(&dev));
  if (t_lanes.dev != dev || !t_lanes.in) {
    t_lanes.release();
    DGQ_H_CUDA(cudaStreamCreateWithFlags(&t_lanes.in, cudaStreamNonBlocking));
    DGQ_H_CUDA(cudaStreamCreateWithFlags(&t_lanes.out, cudaStreamNonBlocking));
    for (int i = 0; i < CopyLanes::kEv; ++i) {
      DGQ_H_CUDA(cudaEventCreateWithFlags(&t_lanes.ev_in[i], cudaEventDisableTiming));
      DGQ_H_CUDA(cudaEventCreateWithFlags(&t_lanes.ev_c[i], cudaEventDisableTiming));
    }
    t_lanes.dev = dev;
  }
  *out = &t_lanes;
  return DGQ_OK;
}

bool shape_ok(size_t h, size_t o, size_t g) { return h && o && o % 2 == 0 && g && h % g == 0; }

}  // namespace

extern "C" {

dgq_status dgq_host_quantize_activations(const float* X, size_t M, size_t K, const float* k, int mode,
                                         float act_scale, int8_t* codes, float* row_scales) {
  if (M == 0) return DGQ_OK;
  if (!X || !k || !codes || !row_scales) return dgq_internal_fail(DGQ_EINVAL, "null argument", "");
  cudaStream_t st;
  DGQ_H_TRY(host_stream(&st));
  DevBuf dx, dk, dq, drs;
  DGQ_H_TRY(upload(dx, X, M * K * sizeof(float), st));
  DGQ_H_TRY(upload(dk, k, K * sizeof(float), st));
  DGQ_H_CUDA(dq.alloc(M * K, st));
  DGQ_H_CUDA(drs.alloc(M * sizeof(float), st));
  if (K) DGQ_H_TRY(dgq_quantize_act_raw(dx.as<float>(), M, K, K, dk.as<float>(), mode, act_scale, dq.as<int8_t>(), K,
                                        drs.as<float>(), st));
  else DGQ_H_CUDA(cudaMemsetAsync(drs.p, 0, M * sizeof(float), st));  // unreachable for valid layers
  DGQ_H_TRY(download(codes, dq, M * K, st));
  DGQ_H_TRY(download(row_scales, drs, M * sizeof(float), st));
  DGQ_H_CUDA(cudaStreamSynchronize(st));
  return DGQ_OK;
}

dgq_status dgq_host_dequantize_to_s8(size_t h, size_t o, size_t g, const uint8_t* codes_u4, const int8_t* s2,
                                     const uint8_t* zp_u4, int8_t* w_s8) {
  if (!shape_ok(h, o, g)) return dgq_internal_fail(DGQ_EINVAL, "inconsistent layer shape", "");
  if (!codes_u4 || !s2 || !zp_u4 || !w_s8) return dgq_internal_fail(DGQ_EINVAL, "null argument", "");
  cudaStream_t st;
  DGQ_H_TRY(host_stream(&st));
  const size_t ng = h / g;
  DevBuf dc, ds, dz, dw;
  DGQ_H_TRY(upload(dc, codes_u4, h * o / 2, st));
  DGQ_H_TRY(upload(ds, s2, ng * o, st));
  DGQ_H_TRY(upload(dz, zp_u4, ng * o / 2, st));
  DGQ_H_CUDA(dw.alloc(h * o, st));
  DGQ_H_TRY(dgq_dequantize_to_s8(h, o, g, dc.as<uint8_t>(), ds.as<int8_t>(), dz.as<uint8_t>(), dw.as<int8_t>(), st));
  DGQ_H_TRY(download(w_s8, dw, h * o, st));
  DGQ_H_CUDA(cudaStreamSynchronize(st));
  return DGQ_OK;
}

dgq_status dgq_host_dequantize_to_f32(size_t h, size_t o, size_t g, const uint8_t* codes_u4, const int8_t* s2,
                                      const uint8_t* zp_u4, const float* s1, float* w) {
  if (!shape_ok(h, o, g)) return dgq_internal_fail(DGQ_EINVAL, "inconsistent layer shape", "");
  if (!codes_u4 || !s2 || !zp_u4 || !s1 || !w) return dgq_internal_fail(DGQ_EINVAL, "null argument", "");
  cudaStream_t st;
  DGQ_H_TRY(host_stream(&st));
  const size_t ng = h / g;
  DevBuf dc, ds, dz, dw, d1, df;
  DGQ_H_TRY(upload(dc, codes_u4, h * o / 2, st));
  DGQ_H_TRY(upload(ds, s2, ng * o, st));
  DGQ_H_TRY(upload(dz, zp_u4, ng * o / 2, st));
  DGQ_H_TRY(upload(d1, s1, o * sizeof(float), st));
  DGQ_H_CUDA(dw.alloc(h * o, st));
  DGQ_H_CUDA(df.alloc(h * o * sizeof(float), st));
  DGQ_H_TRY(dgq_dequantize_to_s8(h, o, g, dc.as<uint8_t>(), ds.as<int8_t>(), dz.as<uint8_t>(), dw.as<int8_t>(), st));
  DGQ_H_CUDA(dgq_launch_dequant_f32(dw.as<int8_t>(), d1.as<float>(), static_cast<int>(h), static_cast<int>(o),
                                    df.as<float>(), st));
  DGQ_H_TRY(download(w, df, h * o * sizeof(float), st));
  DGQ_H_CUDA(cudaStreamSynchronize(st));
  return DGQ_OK;
}

dgq_status dgq_host_int8_gemm(const int8_t* Xq, const int8_t* W, size_t M, size_t K, size_t N, int32_t* acc,
                              int64_t* max_abs_acc) {
  if (static_cast<double>(K) * 127.0 * 127.0 >= 2147483648.0)
    return dgq_internal_fail(DGQ_EINVAL, "h too large for 32-bit accumulation", "");
  if (max_abs_acc) *max_abs_acc = 0;
  if (M == 0 || N == 0) return DGQ_OK;
  if (!Xq || !W || !acc) return dgq_internal_fail(DGQ_EINVAL, "null argument", "");
  cudaStream_t st;
  DGQ_H_TRY(host_stream(&st));
  DevBuf dx, dw, da;
  DGQ_H_TRY(upload(dx, Xq, M * K, st));
  DGQ_H_TRY(upload(dw, W, K * N, st));
  DGQ_H_CUDA(da.alloc(M * N * sizeof(int32_t), st));
  if (K == 0) {
    DGQ_H_CUDA(cudaMemsetAsync(da.p, 0, M * N * sizeof(int32_t), st));
  } else {
    DGQ_H_TRY(dgq_int8_gemm(dx.as<int8_t>(), K, dw.as<int8_t>(), N, M, K, N, da.as<int32_t>(), N, max_abs_acc, st));
  }
  DGQ_H_TRY(download(acc, da, M * N * sizeof(int32_t), st));
  DGQ_H_CUDA(cudaStreamSynchronize(st));
  return DGQ_OK;
}

dgq_status dgq_host_epilogue(const int32_t* acc, const float* row_scales, const float* s1, const float* bias,
                             size_t M, size_t N, int fp16_mode, float* y) {
  if (M == 0 || N == 0) return DGQ_OK;
  if (!acc || !row_scales || !s1 || !y) return dgq_internal_fail(DGQ_EINVAL, "null argument", "");
  cudaStream_t st;
  DGQ_H_TRY(host_stream(&st));
  DevBuf da, dr, d1, db, dy;
  DGQ_H_TRY(upload(da, acc, M * N * sizeof(int32_t), st));
  DGQ_H_TRY(upload(dr, row_scales, M * sizeof(float), st));
  DGQ_H_TRY(upload(d1, s1, N * sizeof(float), st));
  if (bias) DGQ_H_TRY(upload(db, bias, N * sizeof(float), st));
  DGQ_H_CUDA(dy.alloc(M * N * sizeof(float), st));
  DGQ_H_TRY(dgq_epilogue(da.as<int32_t>(), N, dr.as<float>(), d1.as<float>(), bias ? db.as<float>() : nullptr, M, N,
                         fp16_mode, DGQ_OUT_F32, dy.p, N, st));
  DGQ_H_TRY(download(y, dy, M * N * sizeof(float), st));
  DGQ_H_CUDA(cudaStreamSynchronize(st));
  return DGQ_OK;
}

dgq_status dgq_host_segmented_gemm(const int8_t* Xq, const float* row_scales, size_t M, size_t h, size_t o, size_t g,
                                   const uint8_t* codes_u4, const int8_t* s2, const uint8_t* zp_u4, const float* s1,
                                   float* y) {
  if (!shape_ok(h, o, g)) return dgq_internal_fail(DGQ_EINVAL, "inconsistent layer shape", "");
  if (M == 0) return DGQ_OK;
  if (!Xq || !row_scales || !codes_u4 || !s2 || !zp_u4 || !s1 || !y)
    return dgq_internal_fail(DGQ_EINVAL, "null argument", "");
  if (M > 65535 || h > 200000) return dgq_internal_fail(DGQ_EINVAL, "segmented comparator: shape too large", "");
  cudaStream_t st;
  DGQ_H_TRY(host_stream(&st));
  const size_t ng = h / g;
  DevBuf dx, dr, dc, ds, dz, d1, dy;
  DGQ_H_TRY(upload(dx, Xq, M * h, st));
  DGQ_H_TRY(upload(dr, row_scales, M * sizeof(float), st));
  DGQ_H_TRY(upload(dc, codes_u4, h * o / 2, st));
  DGQ_H_TRY(upload(ds, s2, ng * o, st));
  DGQ_H_TRY(upload(dz, zp_u4, ng * o / 2, st));
  DGQ_H_TRY(upload(d1, s1, o * sizeof(float), st));
  DGQ_H_CUDA(dy.alloc(M * o * sizeof(float), st));
  DGQ_H_CUDA(dgq_launch_segmented(dx.as<int8_t>(), h, dr.as<float>(), dc.as<uint8_t>(), ds.as<int8_t>(),
                                  dz.as<uint8_t>(), d1.as<float>(), static_cast<int>(M), static_cast<int>(h),
                                  static_cast<int>(o), static_cast<int>(g), dy.as<float>(), o, st));
  DGQ_H_TRY(download(y, dy, M * o * sizeof(float), st));
  DGQ_H_CUDA(cudaStreamSynchronize(st));
  return DGQ_OK;
}

dgq_status dgq_host_forward(size_t M, size_t h, size_t o, size_t g, int mode, float act_scale,
                            const uint8_t* codes_u4, const int8_t* s2, const uint8_t* zp_u4, const float* s1,
                            const float* k, const float* X, const float* bias, float* out, int8_t* w_s8,
                            int8_t* act_codes, float* row_scales, int64_t* max_abs_acc) {
  if (!shape_ok(h, o, g)) return dgq_internal_fail(DGQ_EINVAL, "inconsistent layer shape", "");
  if (!codes_u4 || !s2 || !zp_u4 || !s1 || !k || (M && !X) || (M && !out))
    return dgq_internal_fail(DGQ_EINVAL, "null argument", "");
  if (max_abs_acc) *max_abs_acc = 0;
  cudaStream_t st;
  DGQ_H_TRY(host_stream(&st));
  int dev = 0;
  DGQ_H_CUDA(cudaGetDevice(&dev));
  const size_t ng = h / g;
  // 1. dequantize_to_s8 (proj/src/kernel.cpp:146): range check first, as the reference
  DevBuf dc, ds, dz, dw;
  DGQ_H_TRY(upload(dc, codes_u4, h * o / 2, st));
  DGQ_H_TRY(upload(ds, s2, ng * o, st));
  DGQ_H_TRY(upload(dz, zp_u4, ng * o / 2, st));
  DGQ_H_CUDA(dw.alloc(h * o, st));
  DGQ_H_TRY(dgq_dequantize_to_s8(h, o, g, dc.as<uint8_t>(), ds.as<int8_t>(), dz.as<uint8_t>(), dw.as<int8_t>(), st));
  DGQ_H_TRY(download(w_s8, dw, h * o, st));
  if (static_cast<double>(h) * 127.0 * 127.0 >= 2147483648.0)
    return dgq_internal_fail(DGQ_EINVAL, "h too large for 32-bit accumulation", "");
  if (M == 0) {
    DGQ_H_CUDA(cudaStreamSynchronize(st));
    return DGQ_OK;
  }
  // 2. the prepared layer (fused INT4 tiles), unvalidated like the reference's dgq_forward
  dgq_layer* L = nullptr;
  DGQ_H_TRY(dgq_layer_create(dev, h, o, g, mode, act_scale, codes_u4, s2, zp_u4, s1, k, 0, 0, 0, st, &L));
  struct LayerGuard {
    dgq_layer* l;
    ~LayerGuard() { dgq_layer_destroy(l); }
  } guard{L};
  dgq_layer_info info;
  DGQ_H_TRY(dgq_layer_get_info(L, &info));
  // 3. quantize_activations (K1) -> 4. int8_gemm + epilogue (K5, FP32 out)
  DevBuf dx, dq, dr, db, dy;
  DGQ_H_TRY(upload(dx, X, M * h * sizeof(float), st));
  if (bias) DGQ_H_TRY(upload(db, bias, o * sizeof(float), st));
  DGQ_H_CUDA(dq.alloc(M * info.k_pad, st));
  DGQ_H_CUDA(dr.alloc(M * sizeof(float), st));
  DGQ_H_CUDA(dy.alloc(M * o * sizeof(float), st));
  DGQ_H_TRY(dgq_quantize_act(L, dx.as<float>(), M, h, dq.as<int8_t>(), info.k_pad, dr.as<float>(), st));
  DGQ_H_TRY(dgq_linear(L, dq.as<int8_t>(), info.k_pad, dr.as<float>(), M, bias ? db.as<float>() : nullptr,
                       DGQ_OUT_F32, 0, dy.p, o, nullptr, 0, nullptr, 0, st));
  if (act_codes) DGQ_H_CUDA(cudaMemcpy2DAsync(act_codes, h, dq.p, info.k_pad, h, M, cudaMemcpyDeviceToHost, st));
  DGQ_H_TRY(download(row_scales, dr, M * sizeof(float), st));
  DGQ_H_TRY(download(out, dy, M * o * sizeof(float), st));
  // 5. the running-sum audit behind max_abs_acc (proj/src/kernel.cpp:73-77)
  if (max_abs_acc) DGQ_H_TRY(dgq_audit_max_abs_acc(dq.as<int8_t>(), info.k_pad, dw.as<int8_t>(), o, M, h, o,
                                                   max_abs_acc, st));
  DGQ_H_CUDA(cudaStreamSynchronize(st));
  if (max_abs_acc && *max_abs_acc > 2147483647LL)
    return dgq_internal_fail(DGQ_EOVERFLOW, "int8_gemm accumulator overflow despite precondition", "");
  return DGQ_OK;
}

dgq_status dgq_layer_forward_host(const dgq_layer* layer, const float* X, size_t M, const float* dBias,
                                  int out_dtype, void* Y, void* stream) {
  DGQ_NVTX("dgq_layer_forward_host");
  if (!layer) return dgq_internal_fail(DGQ_EINVAL, "null layer", "");
  if (M == 0) return DGQ_OK;
  if (!X || !Y) return dgq_internal_fail(DGQ_EINVAL, "null argument", "");
  dgq_layer_info info;
  DGQ_H_TRY(dgq_layer_get_info(layer, &info));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!st) DGQ_H_TRY(host_stream(&st));
  CopyLanes* ln = nullptr;
  DGQ_H_TRY(copy_lanes(&ln));
  const size_t esz = out_dtype == DGQ_OUT_F16 ? 2 : 4;
  // Token chunks: chunk c's input copy (lane `in`), K1 + K5 (the caller's stream)
  // and output copy (lane `out`) are ordered by events, so copies of one chunk
  // run under the kernels of its neighbours (PCIe is full duplex).  Small
  // calls are one chunk.  Scratch comes from the stream-ordered pool.
  size_t chunk = M <= 256 ? M : round_up((M + 3) / 4, 128);
  const int nch = static_cast<int>((M + chunk - 1) / chunk);
  if (nch > CopyLanes::kEv) chunk = round_up((M + CopyLanes::kEv - 1) / CopyLanes::kEv, 128);
  DevBuf dx, dq, dr, dy;
  DGQ_H_CUDA(dx.alloc(M * info.h * sizeof(float), st));
  DGQ_H_CUDA(dq.alloc(M * info.k_pad, st));
  DGQ_H_CUDA(dr.alloc(M * sizeof(float), st));
  DGQ_H_CUDA(dy.alloc(M * info.o * esz, st));
  // the copy lanes must not run ahead of the pool allocations made on `st`
  DGQ_H_CUDA(cudaEventRecord(ln->ev_c[0], st));
  DGQ_H_CUDA(cudaStreamWaitEvent(ln->in, ln->ev_c[0], 0));
  DGQ_H_CUDA(cudaStreamWaitEvent(ln->out, ln->ev_c[0], 0));
  int c = 0;
  for (size_t r0 = 0; r0 < M; r0 += chunk, ++c) {
    const size_t m = std::min(chunk, M - r0);
    DGQ_H_CUDA(cudaMemcpyAsync(dx.as<float>() + r0 * info.h, X + r0 * info.h, m * info.h * sizeof(float),
                               cudaMemcpyHostToDevice, ln->in));
    DGQ_H_CUDA(cudaEventRecord(ln->ev_in[c], ln->in));
    DGQ_H_CUDA(cudaStreamWaitEvent(st, ln->ev_in[c], 0));
    DGQ_H_TRY(dgq_forward_device(layer, dx.as<float>() + r0 * info.h, m, info.h, dBias, out_dtype,
                                 static_cast<uint8_t*>(dy.p) + r0 * info.o * esz, info.o,
                                 dq.as<int8_t>() + r0 * info.k_pad, dr.as<float>() + r0, nullptr, 0, st));
    DGQ_H_CUDA(cudaEventRecord(ln->ev_c[c], st));
    DGQ_H_CUDA(cudaStreamWaitEvent(ln->out, ln->ev_c[c], 0));
    DGQ_H_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(Y) + r0 * info.o * esz,
                               static_cast<uint8_t*>(dy.p) + r0 * info.o * esz, m * info.o * esz,
                               cudaMemcpyDeviceToHost, ln->out));
  }
  // the scratch is released on `st` once the output copies are done
  DGQ_H_CUDA(cudaEventRecord(ln->ev_in[0], ln->out));
  DGQ_H_CUDA(cudaStreamWaitEvent(st, ln->ev_in[0], 0));
  DGQ_H_CUDA(cudaStreamSynchronize(st));
  return DGQ_OK;
}

}  // extern "C"
