/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the DGQ A8W4 hot path.
 *
 * A plain-C restatement of the reference algorithm (arxiv 2310.04836, DGQ),
 * written from the reference's CPU code under /root/reference/proj and pinned
 * against it: tests/test_oracle.py checks every function here bit-for-bit
 * against oracle/_ref/libdgq_ref.so (the reference's own sources, built by
 * oracle/Makefile) and against the committed golden vectors in tests/golden/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product (paper_2310_04836_b200) never does.
 *
 * Build: oracle/Makefile → oracle/_build/libdgq_oracle.so (gcc -O2
 * -ffp-contract=off, so float expressions round exactly like the reference's).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- numerics primitives ------------------------------------------------ */

/* proj/include/dgq/quant.hpp:24-30 — round half to even in double. */
double orc_rhe(double v) {
  double fl = floor(v);
  double diff = v - fl;
  if (diff > 0.5) return fl + 1.0;
  if (diff < 0.5) return fl;
  return (fmod(fl, 2.0) == 0.0) ? fl : fl + 1.0;
}

/* proj/src/quant.cpp:9-58 — binary16 round trip (RNE), except that
 * |x| < 2^-24 flushes to signed zero (the reference's exp < -24 branch). */
float orc_fp16_round(float x) {
  uint32_t bits;
  memcpy(&bits, &x, 4);
  uint32_t sign = bits & 0x80000000u, mag = bits & 0x7FFFFFFFu;
  if (mag >= 0x7F800000u) return x;
  int e = (int)(mag >> 23) - 127;
  uint32_t h;
  if (e > 15) {
    h = 0x7C00u;
  } else if (e >= -14) {
    uint32_t m = mag & 0x7FFFFFu, keep = m >> 13, rem = m & 0x1FFFu;
    h = ((uint32_t)(e + 15) << 10) | keep;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;
  } else if (e >= -24) {
    uint32_t m = (mag & 0x7FFFFFu) | 0x800000u;
    int sh = -e - 1;
    uint32_t keep = m >> sh, rem = m & ((1u << sh) - 1u), half = 1u << (sh - 1);
    h = keep;
    if (rem > half || (rem == half && (h & 1u))) h++;
  } else {
    h = 0;
  }
  uint32_t he = (h >> 10) & 0x1Fu, hm = h & 0x3FFu, out;
  if (he == 0x1Fu) {
    out = sign | 0x7F800000u;
  } else if (he) {
    out = sign | ((he + 112u) << 23) | (hm << 13);
  } else if (!hm) {
    out = sign;
  } else {
    int sh = 0;
    while (!(hm & 0x400u)) { hm <<= 1; sh--; }
    out = sign | ((uint32_t)(113 + sh) << 23) | ((hm & 0x3FFu) << 13);
  }
  float r;
  memcpy(&r, &out, 4);
  return r;
}

/* proj/src/search.cpp:190-201 — fused code interval, C truncating division. */
int orc_clip_interval(int s2, int zp, int* lo, int* hi) {
  if (s2 < 1) return 1;
  int a = (-127) / s2 + zp, b = 127 / s2 + zp;
  *lo = a > 0 ? a : 0;
  *hi = b < 15 ? b : 15;
  return *lo > *hi ? 3 : 0;
}

/* ---- nibble access: proj/src/tensor.cpp:100-105 (even index = low nibble) */
static inline int u4_at(const uint8_t* p, size_t r, size_t c, size_t cols) {
  size_t i = r * cols + c;
  uint8_t b = p[i >> 1];
  return (i & 1) ? (b >> 4) : (b & 0x0F);
}

/* ---- synthetic data: proj/include/dgq/tensor.hpp:101-131,
 *      proj/src/tensor.cpp:222-257 (SplitMix64 + Box-Muller) -------------- */
static inline uint64_t sm64_next(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline double sm64_unit(uint64_t* s) {
  return (double)((sm64_next(s) >> 11) + 1) * 0x1.0p-53;
}
static int cmp_size(const void* a, const void* b) {
  size_t x = *(const size_t*)a, y = *(const size_t*)b;
  return x < y ? -1 : x > y;
}
int orc_outlier_columns(size_t cols, uint64_t column_seed, size_t count, size_t* out) {
  if (count > cols) return 1;
  size_t* idx = (size_t*)malloc(sizeof(size_t) * (cols ? cols : 1));
  uint64_t st = column_seed ^ 0xD1B54A32D192ED03ULL;
  for (size_t i = 0; i < cols; ++i) idx[i] = i;
  for (size_t i = 0; i < count; ++i) {
    size_t j = i + (size_t)(sm64_next(&st) % (uint64_t)(cols - i));
    size_t t = idx[i]; idx[i] = idx[j]; idx[j] = t;
  }
  qsort(idx, count, sizeof(size_t), cmp_size);
  memcpy(out, idx, count * sizeof(size_t));
  free(idx);
  return 0;
}
int orc_gen_synthetic(size_t rows, size_t cols, uint64_t seed, size_t count, float magnitude,
                      int has_column_seed, uint64_t column_seed, float* v) {
  if (count > cols) return 1;
  const double two_pi = 2.0 * 3.14159265358979323846;
  uint64_t st = seed;
  size_t n = rows * cols;
  for (size_t i = 0; i < n; i += 2) {
    double u1 = sm64_unit(&st), u2 = sm64_unit(&st);
    double r = sqrt(-2.0 * log(u1));
    v[i] = (float)(r * cos(two_pi * u2));
    if (i + 1 < n) v[i + 1] = (float)(r * sin(two_pi * u2));
  }
  if (count) {
    size_t* oc = (size_t*)malloc(sizeof(size_t) * count);
    orc_outlier_columns(cols, has_column_seed ? column_seed : seed, count, oc);
    for (size_t t = 0; t < count; ++t)
      for (size_t r = 0; r < rows; ++r) v[r * cols + oc[t]] *= magnitude;
    free(oc);
  }
  return 0;
}

/* ---- calibration: proj/src/smoothing.cpp:9-49 ------------------------- */
static int cmp_desc_f(const void* a, const void* b) {
  float x = *(const float*)a, y = *(const float*)b;
  return x > y ? -1 : x < y;
}
int orc_smooth_from_calib(const float* X, size_t rows, size_t cols, float percentile,
                          float* k, float* threshold) {
  if (!cols) return 1;
  if (!(percentile > 0.0f && percentile < 1.0f)) return 1;
  float* z = (float*)calloc(cols, sizeof(float));
  for (size_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < cols; ++c) {
      float a = fabsf(X[r * cols + c]);
      if (z[c] < a) z[c] = a;
    }
  size_t rank = (size_t)ceil((double)percentile * (double)cols);
  if (rank < 1) rank = 1;
  float* s = (float*)malloc(sizeof(float) * cols);
  memcpy(s, z, sizeof(float) * cols);
  qsort(s, cols, sizeof(float), cmp_desc_f);
  float th = s[rank - 1];
  free(s);
  if (!(th > 0.0f)) { free(z); return 1; }
  for (size_t j = 0; j < cols; ++j) {
    float q = z[j] / th;
    k[j] = (1.0f < q) ? q : 1.0f;
  }
  *threshold = th;
  free(z);
  return 0;
}

/* ---- layer invariants: proj/src/format.cpp:24-75.  Returns 0 or 2 and the
 *      offending field name (static string) in *field. ------------------- */
int orc_validate_layer(size_t h, size_t o, size_t g, int mode, float act_scale,
                       const uint8_t* codes, const int8_t* s2, const uint8_t* zp,
                       const float* s1, const float* k, const char** field) {
#define FAIL(f) do { *field = f; return 2; } while (0)
  if (h == 0 || o == 0) FAIL("shape");
  if (o % 2) FAIL("shape");
  if (g == 0 || h % g) FAIL("g");
  size_t ng = h / g;
  for (size_t i = 0; i < ng * o; ++i)
    if (s2[i] < 1) FAIL("s2");  /* int8 cannot exceed 127 */
  for (size_t c = 0; c < o; ++c)
    if (!(s1[c] > 0.0f) || !isfinite(s1[c])) FAIL("s1");
  for (size_t j = 0; j < h; ++j)
    if (!(k[j] >= 1.0f) || !isfinite(k[j])) FAIL("k");
  if (mode == 0 && !(act_scale > 0.0f)) FAIL("act_scale");
  if (!(act_scale >= 0.0f) || !isfinite(act_scale)) FAIL("act_scale");
  for (size_t kk = 0; kk < ng; ++kk)
    for (size_t c = 0; c < o; ++c) {
      int lo, hi;
      orc_clip_interval(s2[kk * o + c], u4_at(zp, kk, c, o), &lo, &hi);
      for (size_t j = 0; j < g; ++j) {
        int code = u4_at(codes, kk * g + j, c, o);
        if (code < lo || code > hi) FAIL("codes");
      }
    }
  *field = "";
  return 0;
#undef FAIL
}

/* ---- the hot path ------------------------------------------------------ */

/* proj/src/kernel.cpp:14-44 — per-token INT8 after dividing by k. */
int orc_quantize_activations(const float* X, size_t M, size_t K, const float* k, int mode,
                             float act_scale, int8_t* q, float* rs) {
  float* row = (float*)malloc(sizeof(float) * (K ? K : 1));
  for (size_t r = 0; r < M; ++r) {
    for (size_t j = 0; j < K; ++j) row[j] = X[r * K + j] / k[j];
    float s;
    if (mode) {
      float am = 0.0f;
      for (size_t j = 0; j < K; ++j) {
        float a = fabsf(row[j]);
        if (am < a) am = a;
      }
      double d = (double)am / 127.0, fl = (double)1e-8f;
      s = (float)(d < fl ? fl : d);
    } else {
      s = act_scale;
    }
    rs[r] = s;
    for (size_t j = 0; j < K; ++j) {
      double c = orc_rhe((double)row[j] / (double)s);
      if (c < -127.0) c = -127.0;
      if (c > 127.0) c = 127.0;
      q[r * K + j] = (int8_t)c;
    }
  }
  free(row);
  return 0;
}

/* proj/src/format.cpp:122-141 — W_s8 = S2 * (code - ZP); 2 if out of range. */
int orc_dequantize_to_s8(size_t h, size_t o, size_t g, const uint8_t* codes, const int8_t* s2,
                         const uint8_t* zp, int8_t* w) {
  for (size_t i = 0; i < h; ++i) {
    size_t kk = i / g;
    for (size_t c = 0; c < o; ++c) {
      int v = (int)s2[kk * o + c] * (u4_at(codes, i, c, o) - u4_at(zp, kk, c, o));
      if (v < -127 || v > 127) return 2;
      w[i * o + c] = (int8_t)v;
    }
  }
  return 0;
}

/* proj/src/kernel.cpp:46-87 — exact INT8 GEMM plus the running-|sum| audit.
 * Row-parallel under OpenMP exactly like the reference's parallel_for (rows
 * are independent, so the result does not depend on the thread count). */
int orc_int8_gemm(const int8_t* Xq, const int8_t* Wq, size_t M, size_t K, size_t N,
                  int32_t* acc, int64_t* max_abs_acc) {
  if ((double)K * 127.0 * 127.0 >= 2147483648.0) return 1;
  int8_t* wt = (int8_t*)malloc(K * N ? K * N : 1);
  for (size_t i = 0; i < K; ++i)
    for (size_t c = 0; c < N; ++c) wt[c * K + i] = Wq[i * N + c];
  int64_t best = 0;
#pragma omp parallel for schedule(static) reduction(max : best)
  for (size_t r = 0; r < M; ++r) {
    const int8_t* x = Xq + r * K;
    for (size_t c = 0; c < N; ++c) {
      const int8_t* w = wt + c * K;
      int64_t s = 0;
      for (size_t i = 0; i < K; ++i) {
        s += (int64_t)x[i] * (int64_t)w[i];
        int64_t a = s < 0 ? -s : s;
        if (a > best) best = a;
      }
      acc[r * N + c] = (int32_t)s;
    }
  }
  free(wt);
  *max_abs_acc = best;
  return best > 2147483647LL ? 3 : 0;
}

/* proj/src/kernel.cpp:89-116 — FP32 (or the binary16 mode) epilogue. */
int orc_epilogue(const int32_t* acc, size_t M, size_t N, const float* rs, const float* s1,
                 const float* bias, int fp16_mode, float* y) {
  for (size_t r = 0; r < M; ++r)
    for (size_t c = 0; c < N; ++c) {
      float v;
      if (fp16_mode) {
        float s = orc_fp16_round(orc_fp16_round(rs[r]) * orc_fp16_round(s1[c]));
        v = orc_fp16_round((float)acc[r * N + c] * s);
      } else {
        v = (float)acc[r * N + c] * rs[r] * s1[c];
      }
      if (bias) v += bias[c];
      y[r * N + c] = v;
    }
  return 0;
}

/* proj/src/kernel.cpp:118-142 — group-wise (segmented) baseline. */
int orc_segmented_gemm(const int8_t* Xq, const float* rs, size_t M, size_t h, size_t o,
                       size_t g, const uint8_t* codes, const int8_t* s2, const uint8_t* zp,
                       const float* s1, float* y) {
  size_t ng = h / g;
  for (size_t r = 0; r < M; ++r)
    for (size_t c = 0; c < o; ++c) {
      float f = 0.0f;
      for (size_t kk = 0; kk < ng; ++kk) {
        int64_t part = 0;
        int z = u4_at(zp, kk, c, o);
        for (size_t j = 0; j < g; ++j) {
          size_t i = kk * g + j;
          part += (int64_t)Xq[r * h + i] * (int64_t)(u4_at(codes, i, c, o) - z);
        }
        f += (float)((int64_t)s2[kk * o + c] * part);
      }
      y[r * o + c] = f * rs[r] * s1[c];
    }
  return 0;
}

/* proj/src/kernel.cpp:144-153 — dequant → act quant → GEMM → epilogue. */
int orc_dgq_forward(const float* X, size_t M, size_t h, size_t o, size_t g, int mode,
                    float act_scale, const uint8_t* codes, const int8_t* s2, const uint8_t* zp,
                    const float* s1, const float* k, const float* bias, float* out,
                    int8_t* w_s8, int8_t* q, float* rs, int64_t* max_abs_acc) {
  int8_t* w = w_s8 ? w_s8 : (int8_t*)malloc(h * o);
  int8_t* qq = q ? q : (int8_t*)malloc(M * h ? M * h : 1);
  float* rr = rs ? rs : (float*)malloc(sizeof(float) * (M ? M : 1));
  int32_t* acc = (int32_t*)malloc(sizeof(int32_t) * (M * o ? M * o : 1));
  int64_t mx = 0;
  int st = orc_dequantize_to_s8(h, o, g, codes, s2, zp, w);
  if (!st) st = orc_quantize_activations(X, M, h, k, mode, act_scale, qq, rr);
  if (!st) st = orc_int8_gemm(qq, w, M, h, o, acc, &mx);
  if (!st) st = orc_epilogue(acc, M, o, rr, s1, bias, 0, out);
  if (max_abs_acc) *max_abs_acc = mx;
  free(acc);
  if (!w_s8) free(w);
  if (!q) free(qq);
  if (!rs) free(rr);
  return st;
}
