// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the reference's own CPU library, compiled from the
// unmodified sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libdgq_ref.so.  Python (oracle/__init__.py) binds it with ctypes
// so tests, the golden-vector generator and bench.py's reference arm can call
// the reference itself on plain buffers.
//
// Every entry point returns 0 on success, 1 for std::invalid_argument,
// 2 for dgq::validation_error, 3 for std::runtime_error / other exceptions;
// the message (and the validation field) are kept in thread-local storage.

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "dgq/format.hpp"
#include "dgq/kernel.hpp"
#include "dgq/quant.hpp"
#include "dgq/search.hpp"
#include "dgq/smoothing.hpp"
#include "dgq/tensor.hpp"

namespace {

thread_local std::string g_msg;
thread_local std::string g_field;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const dgq::validation_error& e) {
    g_msg = e.what();
    g_field = e.field();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_msg = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 3;
  }
}

dgq::Tensor tensor_from(dgq::Dtype dt, size_t rows, size_t cols, const void* p) {
  dgq::Tensor t;
  t.dtype = dt;
  t.rows = rows;
  t.cols = cols;
  size_t nb = dgq::payload_bytes(dt, rows, cols);
  t.data.resize(nb);
  if (nb) std::memcpy(t.data.data(), p, nb);
  return t;
}

dgq::DgqLayer layer_from(size_t h, size_t o, size_t g, int mode, float act_scale,
                         const uint8_t* codes, const int8_t* s2, const uint8_t* zp,
                         const float* s1, const float* k) {
  dgq::DgqLayer L;
  L.h = h;
  L.o = o;
  L.g = g;
  const size_t ng = g ? h / g : 0;
  L.codes = tensor_from(dgq::Dtype::kU4, h, o, codes);
  L.s2 = tensor_from(dgq::Dtype::kI8, ng, o, s2);
  L.zp = tensor_from(dgq::Dtype::kU4, ng, o, zp);
  L.s1.assign(s1, s1 + o);
  L.k.assign(k, k + h);
  L.act_scale = act_scale;
  L.mode = mode ? dgq::ActMode::kDynamic : dgq::ActMode::kStatic;
  return L;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_msg.c_str(); }
const char* ref_last_field(void) { return g_field.c_str(); }

float ref_fp16_round(float x) { return dgq::fp16_round(x); }
double ref_round_half_even(double x) { return dgq::round_half_even(x); }

int ref_clip_interval(int s2, int zp, int* lo, int* hi) {
  return guarded([&] {
    dgq::ClipInterval ci = dgq::clip_interval(s2, zp);
    *lo = ci.lo;
    *hi = ci.hi;
  });
}

int ref_gen_synthetic(size_t rows, size_t cols, uint64_t seed, size_t count, float magnitude,
                      int has_column_seed, uint64_t column_seed, float* out) {
  return guarded([&] {
    dgq::OutlierSpec spec;
    spec.count = count;
    spec.magnitude = magnitude;
    if (has_column_seed) spec.column_seed = column_seed;
    dgq::Tensor t = dgq::gen_synthetic(rows, cols, seed, spec);
    std::memcpy(out, t.data.data(), t.data.size());
  });
}

// k = compute_smooth(channel_maxima({X}), percentile).k
int ref_smooth_from_calib(const float* X, size_t rows, size_t cols, float percentile,
                          float* k_out, float* threshold) {
  return guarded([&] {
    std::vector<dgq::Tensor> calib{tensor_from(dgq::Dtype::kF32, rows, cols, X)};
    dgq::SmoothScale s = dgq::compute_smooth(dgq::channel_maxima(calib), percentile);
    std::memcpy(k_out, s.k.data(), 4 * s.k.size());
    *threshold = s.threshold;
  });
}

int ref_validate_layer(size_t h, size_t o, size_t g, int mode, float act_scale,
                       const uint8_t* codes, const int8_t* s2, const uint8_t* zp,
                       const float* s1, const float* k) {
  return guarded([&] {
    dgq::validate_layer(layer_from(h, o, g, mode, act_scale, codes, s2, zp, s1, k));
  });
}

int ref_quantize_activations(const float* X, size_t M, size_t K, const float* k, int mode,
                             float act_scale, int8_t* codes, float* row_scales) {
  return guarded([&] {
    dgq::DgqLayer L;
    L.h = K;
    L.k.assign(k, k + K);
    L.mode = mode ? dgq::ActMode::kDynamic : dgq::ActMode::kStatic;
    L.act_scale = act_scale;
    dgq::ActQuant aq = dgq::quantize_activations(tensor_from(dgq::Dtype::kF32, M, K, X), L);
    std::memcpy(codes, aq.codes.data.data(), aq.codes.data.size());
    std::memcpy(row_scales, aq.row_scales.data(), 4 * M);
  });
}

int ref_dequantize_to_s8(size_t h, size_t o, size_t g, const uint8_t* codes, const int8_t* s2,
                         const uint8_t* zp, int8_t* w_s8) {
  return guarded([&] {
    std::vector<float> s1(o, 1.0f), k(h, 1.0f);
    dgq::DgqLayer L = layer_from(h, o, g, 1, 0.0f, codes, s2, zp, s1.data(), k.data());
    dgq::Tensor w = dgq::dequantize_to_s8(L);
    std::memcpy(w_s8, w.data.data(), w.data.size());
  });
}

int ref_int8_gemm(const int8_t* Xq, const int8_t* Wq, size_t M, size_t K, size_t N, int threads,
                  int32_t* acc, int64_t* max_abs_acc) {
  return guarded([&] {
    dgq::IntGemmResult r = dgq::int8_gemm(tensor_from(dgq::Dtype::kI8, M, K, Xq),
                                          tensor_from(dgq::Dtype::kI8, K, N, Wq), threads);
    std::memcpy(acc, r.acc.data.data(), r.acc.data.size());
    *max_abs_acc = r.max_abs_acc;
  });
}

int ref_epilogue(const int32_t* acc, size_t M, size_t N, const float* row_scales,
                 const float* s1, const float* bias, int fp16_mode, float* out) {
  return guarded([&] {
    std::vector<float> rs(row_scales, row_scales + M), s(s1, s1 + N), b;
    if (bias) b.assign(bias, bias + N);
    dgq::Tensor y = dgq::epilogue(tensor_from(dgq::Dtype::kI32, M, N, acc), rs, s, b,
                                  fp16_mode != 0);
    std::memcpy(out, y.data.data(), y.data.size());
  });
}

int ref_segmented_gemm(const int8_t* Xq, const float* row_scales, size_t M, size_t h, size_t o,
                       size_t g, const uint8_t* codes, const int8_t* s2, const uint8_t* zp,
                       const float* s1, float* out) {
  return guarded([&] {
    std::vector<float> k(h, 1.0f);
    dgq::DgqLayer L = layer_from(h, o, g, 1, 0.0f, codes, s2, zp, s1, k.data());
    dgq::ActQuant aq;
    aq.codes = tensor_from(dgq::Dtype::kI8, M, h, Xq);
    aq.row_scales.assign(row_scales, row_scales + M);
    dgq::Tensor y = dgq::segmented_gemm_reference(aq, L);
    std::memcpy(out, y.data.data(), y.data.size());
  });
}

// The full reference hot path (kernel.cpp:144-153). Any of the optional
// outputs may be NULL.
int ref_dgq_forward(const float* X, size_t M, size_t h, size_t o, size_t g, int mode,
                    float act_scale, const uint8_t* codes, const int8_t* s2, const uint8_t* zp,
                    const float* s1, const float* k, const float* bias, int threads, float* out,
                    int8_t* w_s8, int8_t* act_codes, float* row_scales, int64_t* max_abs_acc) {
  return guarded([&] {
    dgq::DgqLayer L = layer_from(h, o, g, mode, act_scale, codes, s2, zp, s1, k);
    std::vector<float> b;
    if (bias) b.assign(bias, bias + o);
    dgq::ForwardResult r =
        dgq::dgq_forward(tensor_from(dgq::Dtype::kF32, M, h, X), L, b, threads);
    std::memcpy(out, r.out.data.data(), r.out.data.size());
    if (w_s8) std::memcpy(w_s8, r.w_s8.data.data(), r.w_s8.data.size());
    if (act_codes) std::memcpy(act_codes, r.act.codes.data.data(), r.act.codes.data.size());
    if (row_scales) std::memcpy(row_scales, r.act.row_scales.data(), 4 * M);
    if (max_abs_acc) *max_abs_acc = r.max_abs_acc;
  });
}

// DGQ1 serialisation round trip through the reference (format.cpp:195-266).
// Returns the byte count in *nbytes; call with out == NULL first to size.
int ref_dgq_to_bytes(size_t h, size_t o, size_t g, int mode, float act_scale,
                     const uint8_t* codes, const int8_t* s2, const uint8_t* zp, const float* s1,
                     const float* k, uint8_t* out, size_t* nbytes) {
  return guarded([&] {
    auto bytes = dgq::dgq_to_bytes(layer_from(h, o, g, mode, act_scale, codes, s2, zp, s1, k));
    if (out) std::memcpy(out, bytes.data(), bytes.size());
    *nbytes = bytes.size();
  });
}

// Two-phase grid search (search.cpp:83-163, 252-326) on plain buffers.
// W [h x o] f32, X / X_hat [b x h] f32 (smoothed calibration rows and their
// quantise-dequantise), grids in the caller's order.
int ref_phase1_search(const float* W, size_t h, size_t o, const float* X, const float* Xhat, size_t b,
                      size_t g, int n_bits, const float* grid1, size_t n1, int threads, float* s_prime,
                      int32_t* zp, float* err, float* alpha, uint64_t* evals) {
  return guarded([&] {
    dgq::SearchConfig cfg;
    cfg.group_size = g;
    cfg.n_bits_w = n_bits;
    cfg.alpha_grid_phase1.assign(grid1, grid1 + n1);
    cfg.calib_X = tensor_from(dgq::Dtype::kF32, b, h, X);
    cfg.threads = threads;
    dgq::GroupParams gp =
        dgq::phase1_search(tensor_from(dgq::Dtype::kF32, h, o, W), cfg, tensor_from(dgq::Dtype::kF32, b, h, Xhat));
    const size_t n = gp.s_prime.size();
    std::memcpy(s_prime, gp.s_prime.f32_data(), 4 * n);
    std::memcpy(zp, gp.zp.i32_data(), 4 * n);
    std::memcpy(err, gp.err.f32_data(), 4 * n);
    std::memcpy(alpha, gp.alpha.f32_data(), 4 * n);
    *evals = gp.objective_evals;
  });
}

int ref_phase2_search(const float* W, size_t h, size_t o, const float* X, const float* Xhat, size_t b,
                      size_t g, int n_bits, const float* s_prime, const int32_t* zp, const float* grid2,
                      size_t n2, int threads, float* s1, int8_t* s2, int32_t* codes, double* col_err,
                      float* col_alpha, uint64_t* evals) {
  return guarded([&] {
    dgq::SearchConfig cfg;
    cfg.group_size = g;
    cfg.n_bits_w = n_bits;
    cfg.alpha_grid_phase2.assign(grid2, grid2 + n2);
    cfg.calib_X = tensor_from(dgq::Dtype::kF32, b, h, X);
    cfg.threads = threads;
    dgq::GroupParams gp;
    gp.group_size = g;
    gp.n_bits = n_bits;
    gp.s_prime = tensor_from(dgq::Dtype::kF32, h / g, o, s_prime);
    gp.zp = tensor_from(dgq::Dtype::kI32, h / g, o, zp);
    dgq::DualSearchResult r = dgq::phase2_search(tensor_from(dgq::Dtype::kF32, h, o, W), gp, cfg,
                                                 tensor_from(dgq::Dtype::kF32, b, h, Xhat));
    std::memcpy(s1, r.params.s1.data(), 4 * o);
    std::memcpy(s2, r.params.s2.i8_data(), r.params.s2.size());
    std::memcpy(codes, r.codes.i32_data(), 4 * r.codes.size());
    std::memcpy(col_err, r.col_err.data(), 8 * o);
    std::memcpy(col_alpha, r.col_alpha.data(), 4 * o);
    *evals = r.objective_evals;
  });
}

}  // extern "C"
