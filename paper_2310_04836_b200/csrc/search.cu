// Two-phase grid search of the DGQ weight quantiser on the GPU (SURVEY.md
// §8f(4)): phase1_search (proj/src/search.cpp:83-163) and phase2_search
// (proj/src/search.cpp:252-326), bit-exact with the reference.
//
// Both phases score candidates with the same objective
//   err(q) = sum_r ( ref[r] - sum_j xh[r, j] * w_hat_q[j] )^2
// where the inner sum runs over j in ascending order and the outer over r in
// ascending order, each a plain double accumulation (search.cpp:64-79, :296-304).
// Floating-point addition is not associative, so each (candidate, row) dot is
// ONE sequential chain on ONE thread — never split across lanes or tensor-core
// tiles.  Parallelism comes from the number of chains: a block owns 128
// candidates; lane l of every warp holds candidates 4l..4l+3 and warp w rows
// 8w..8w+7 of a 64-row block, i.e. 32 independent FP64 chains per thread.
// Per k-step a thread loads its 4 candidate weights (one LDS.128) and the 8
// rows' activations (four broadcast LDS.128 of doubles) and issues 32 DFMAs.
// x * w of two floats is exact in double, so fma(x, w, dot) == dot + x * w of
// the reference.  The squared error of each row lands in shared memory and one
// thread per candidate adds the 64 rows in order, block after block.
//
// The quantise-dequantise of every candidate weight (a double division, RHE,
// clamp) is recomputed per 64-row block inside the kernel instead of being
// materialised (phase 2 would need o * 21 * h floats).  The translation unit is
// compiled with -fmad=false; every other double operation is an explicit
// _rn intrinsic, so no contraction changes a rounding.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace dgqk {
namespace search {

constexpr int kThreads = 256;
constexpr int kCands = 128;      // candidates per block (4 per lane)
constexpr int kRowsPerWarp = 8;
constexpr int kRowBlock = 64;    // 8 warps x 8 rows
constexpr int kJ = 32;           // reduction elements staged per step
constexpr float kScaleFloor = 1e-8f;  // proj/include/dgq/quant.hpp:21

// proj/include/dgq/quant.hpp:24-30: v - floor(v) is exact, so this equals rint
__device__ __forceinline__ double rhe(double v) { return rint(v); }
__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

// Phase-1 candidate (k, c, alpha): asym_params (search.cpp:55-63) and the
// quantise-dequantise of one weight (search.cpp:139-143).
struct P1 {
  float s;
  int zp;
};
__device__ __forceinline__ P1 asym_params(float mn, float mx, double alpha, int levels) {
  const double dmn = static_cast<double>(mn), dmx = static_cast<double>(mx);
  const double lo = 0.0 < dmn ? 0.0 : dmn;  // std::min(double(mn), 0.0)
  const double hi = dmx < 0.0 ? 0.0 : dmx;  // std::max(double(mx), 0.0)
  const double s = __ddiv_rn(__dmul_rn(alpha, __dsub_rn(hi, lo)), static_cast<double>(levels));
  const double fl = static_cast<double>(kScaleFloor);
  const float sf = __double2float_rn(s < fl ? fl : s);  // std::max(s, floor)
  const double zp = rhe(__ddiv_rn(__dmul_rn(-alpha, lo), static_cast<double>(sf)));
  return {sf, static_cast<int>(clampd(zp, 0.0, static_cast<double>(levels)))};
}
__device__ __forceinline__ float p1_what(float w, P1 p, int levels) {
  const double code = __dadd_rn(rhe(__ddiv_rn(static_cast<double>(w), static_cast<double>(p.s))),
                                static_cast<double>(p.zp));
  const int q = static_cast<int>(clampd(code, 0.0, static_cast<double>(levels)));
  return __double2float_rn(__dmul_rn(static_cast<double>(q - p.zp), static_cast<double>(p.s)));
}

// Phase-2 candidate (c, alpha) on group k: build_column_candidate
// (search.cpp:222-247) — s1 from the column absmax, S2 = clamp(rhe(S'/s1)),
// the clip interval of (S2, ZP), the re-quantised code and its dequantisation.
struct P2 {
  double s1;   // float value widened
  int s2, zp, lo, hi;
  double eff;  // s1 * s2 (exact)
};
__device__ __forceinline__ float p2_s1(float absmax, float alpha) {
  const double v = __ddiv_rn(__dmul_rn(static_cast<double>(alpha), static_cast<double>(absmax)), 127.0);
  const double fl = static_cast<double>(kScaleFloor);
  return __double2float_rn(v < fl ? fl : v);  // std::max(v, floor)
}
__device__ __forceinline__ P2 p2_group(float s1, float sp, int zp) {
  P2 p;
  p.s1 = static_cast<double>(s1);
  p.s2 = static_cast<int>(clampd(rhe(__ddiv_rn(static_cast<double>(sp), p.s1)), 1.0, 127.0));
  p.zp = zp;
  const int a = (-127) / p.s2 + zp, b = 127 / p.s2 + zp;  // clip_interval, search.cpp:190-201
  p.lo = a > 0 ? a : 0;
  p.hi = b < 15 ? b : 15;
  p.eff = __dmul_rn(p.s1, static_cast<double>(p.s2));
  return p;
}
__device__ __forceinline__ int p2_code(float w, const P2& p) {
  const double code = __dadd_rn(rhe(__ddiv_rn(static_cast<double>(w), p.eff)), static_cast<double>(p.zp));
  return static_cast<int>(clampd(code, static_cast<double>(p.lo), static_cast<double>(p.hi)));
}
__device__ __forceinline__ float p2_what(float w, const P2& p) {
  const int q = p2_code(w, p);
  return __double2float_rn(__dmul_rn(p.s1, static_cast<double>(p.s2 * (q - p.zp))));
}

// Column min / max of each group (phase 1, search.cpp:122-127, std::min/max
// order) and column absmax (phase 2, search.cpp:226-227): one thread per
// (group, column), sequential like the reference.
__global__ void k_group_minmax(const float* __restrict__ W, int h, int o, int g, float* __restrict__ mn,
                               float* __restrict__ mx) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (c >= o) return;
  const size_t base = static_cast<size_t>(k) * g;
  float lo = W[base * o + c], hi = lo;
  for (int j = 0; j < g; ++j) {
    const float v = W[(base + j) * o + c];
    lo = v < lo ? v : lo;  // std::min(lo, v)
    hi = hi < v ? v : hi;  // std::max(hi, v)
  }
  mn[static_cast<size_t>(k) * o + c] = lo;
  mx[static_cast<size_t>(k) * o + c] = hi;
}

__global__ void k_col_absmax(const float* __restrict__ W, int h, int o, float* __restrict__ am) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= o) return;
  float a = 0.0f;
  for (int i = 0; i < h; ++i) {
    const float v = fabsf(W[static_cast<size_t>(i) * o + c]);
    a = a < v ? v : a;  // std::max(absmax, fabs(v))
  }
  am[c] = a;
}

// What a block evaluates.  kind 0: reference dots (candidate = column, weight =
// W itself, output the dot); 1: phase-1 objective; 2: phase-2 objective.
struct EvalArgs {
  const float* W;      // [h x o]
  const float* X;      // [b x h] (X for refs, X_hat for objectives)
  int h, o, b, g;
  int n_alpha;         // alphas per column (kind 1/2)
  const float* alpha;  // [n_alpha]
  int levels;          // 2^n_bits - 1
  const float* mn;     // [n_g x o] phase 1
  const float* mx;
  const float* absmax; // [o] phase 2
  const float* sp;     // [n_g x o] phase 2: S'
  const int32_t* zp;   // [n_g x o] phase 2: ZP
  const double* ref;   // kind 1: [n_g][o][b]; kind 2: [o][b]
  double* out;         // kind 0: refs (layout as `ref`); kind 1/2: err [seg][q]
  int seg_len;         // reduction length of one segment (g for phase 1 / phase-1 refs, h for phase 2)
};

// Candidate weights w_hat for elements [jabs, jabs + len) of one group into
// ws rows [0, len) (the caller syncs before use; it syncs once itself so the
// per-group phase-2 parameters are visible).
template <int kKind>
__device__ void fill_weights(const EvalArgs& a, float (*ws)[128], int jabs, int len, int seg_pos, const int* cols,
                             const P1* p1s, P2* p2s, const float* s1s) {
  const int tid = threadIdx.x;
  if (kKind == 2) {
    if (tid < 128) {
      const int c = cols[tid] < 0 ? 0 : cols[tid];
      const size_t kc = static_cast<size_t>(jabs / a.g) * a.o + c;
      p2s[tid] = p2_group(s1s[tid], a.sp[kc], a.zp[kc]);
    }
    __syncthreads();
  }
  for (int e = tid; e < len * 128; e += blockDim.x) {
    const int jj = e / 128, qq = e % 128;
    float w = 0.0f;
    const int c = cols[qq];
    if (c >= 0) {
      const float wr = a.W[static_cast<size_t>(jabs + jj) * a.o + c];
      if (kKind == 0) w = wr;
      if (kKind == 1) w = p1_what(wr, p1s[qq], a.levels);
      if (kKind == 2) w = p2_what(wr, p2s[qq]);
    }
    ws[jj][qq] = w;
  }
  (void)seg_pos;
}

// Dynamic shared memory: xs [kJ][kRowBlock] doubles (staged activations),
// ds [kRowBlock][kCands] doubles (per-row squared errors / dots), ws
// [ws_rows][kCands] floats (candidate weights).  A segment of at most kSegCache
// elements (phase 1: one group) keeps all of its candidate weights in ws for
// every row block; longer ones (phase 2: the whole column) recompute each
// chunk's weights per row block.
constexpr int kSegCache = 128;
inline size_t eval_smem_bytes(int seg_len) {
  const int ws_rows = seg_len <= kSegCache ? (seg_len > kJ ? seg_len : kJ) : kJ;
  return sizeof(double) * kJ * kRowBlock + sizeof(double) * kRowBlock * kCands + sizeof(float) * ws_rows * kCands;
}

template <int kKind>
__global__ void __launch_bounds__(kThreads, 1) k_eval(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  auto xs = reinterpret_cast<double(*)[kRowBlock]>(smem);
  auto ds = reinterpret_cast<double(*)[kCands]>(smem + sizeof(double) * kJ * kRowBlock);
  auto ws = reinterpret_cast<float(*)[kCands]>(smem + sizeof(double) * kJ * kRowBlock +
                                               sizeof(double) * kRowBlock * kCands);
  const bool cached = kKind != 2 && a.seg_len <= kSegCache;  // phase-2 weights depend on the group
  __shared__ P1 p1s[kCands];
  __shared__ P2 p2s[kCands];
  __shared__ int cols[kCands];
  __shared__ float s1s[kCands];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int seg = blockIdx.y;                       // group k (kind 0 with seg_len == g, kind 1) or 0
  const int seg_base = seg * a.seg_len;
  const int per_col = kKind == 0 ? 1 : a.n_alpha;
  const long long q_count = static_cast<long long>(a.o) * per_col;
  const long long q0 = static_cast<long long>(blockIdx.x) * kCands;

  if (tid < kCands) {
    const long long q = q0 + tid;
    const bool ok = q < q_count;
    const int c = ok ? static_cast<int>(q / per_col) : 0;
    const int al = ok ? static_cast<int>(q % per_col) : 0;
    cols[tid] = ok ? c : -1;
    if (kKind == 1) {
      const size_t kc = static_cast<size_t>(seg) * a.o + c;
      p1s[tid] = ok ? asym_params(a.mn[kc], a.mx[kc], static_cast<double>(a.alpha[al]), a.levels) : P1{1.0f, 0};
    }
    if (kKind == 2) s1s[tid] = ok ? p2_s1(a.absmax[c], a.alpha[al]) : 1.0f;
  }
  double err = 0.0;  // threads < kCands: the objective of candidate q0 + tid
  __syncthreads();
  if (cached) fill_weights<kKind>(a, ws, seg_base, a.seg_len, seg_base, cols, p1s, p2s, s1s);

  for (int r0 = 0; r0 < a.b; r0 += kRowBlock) {
    double acc[4][kRowsPerWarp];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int r = 0; r < kRowsPerWarp; ++r) acc[i][r] = 0.0;

    for (int j0 = 0; j0 < a.seg_len;) {
      // chunks never straddle a group boundary (phase-2 parameters are per group)
      const int gj = (seg_base + j0) % a.g;
      int len = a.seg_len - j0;
      if (len > kJ) len = kJ;
      if (len > a.g - gj) len = a.g - gj;
      const int jabs = seg_base + j0;
      // stage activations: rows r0.., elements jabs..jabs+len (zero beyond the ends)
      for (int e = tid; e < kJ * kRowBlock; e += kThreads) {
        const int r = e / kJ, jj = e % kJ;
        double v = 0.0;
        if (jj < len && r0 + r < a.b) v = static_cast<double>(a.X[static_cast<size_t>(r0 + r) * a.h + jabs + jj]);
        xs[jj][r] = v;
      }
      if (!cached) fill_weights<kKind>(a, ws, jabs, len, jabs, cols, p1s, p2s, s1s);
      __syncthreads();
      const int wbase = cached ? j0 : 0;
      for (int jj = 0; jj < len; ++jj) {
        const float4 w4 = *reinterpret_cast<const float4*>(&ws[wbase + jj][lane * 4]);
        const double wv[4] = {static_cast<double>(w4.x), static_cast<double>(w4.y), static_cast<double>(w4.z),
                              static_cast<double>(w4.w)};
        double xv[kRowsPerWarp];
#pragma unroll
        for (int r = 0; r < kRowsPerWarp; r += 2) {
          const double2 x2 = *reinterpret_cast<const double2*>(&xs[jj][warp * kRowsPerWarp + r]);
          xv[r] = x2.x;
          xv[r + 1] = x2.y;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int r = 0; r < kRowsPerWarp; ++r) acc[i][r] = __fma_rn(xv[r], wv[i], acc[i][r]);  // exact product
      }
      __syncthreads();
      j0 += len;
    }
    // per-row results of this row block
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int qq = lane * 4 + i;
#pragma unroll
      for (int r = 0; r < kRowsPerWarp; ++r) {
        const int rl = warp * kRowsPerWarp + r, row = r0 + rl;
        double v = acc[i][r];
        if (kKind != 0 && row < a.b && cols[qq] >= 0) {
          const int c = cols[qq];
          const size_t ri = (kKind == 1 ? (static_cast<size_t>(seg) * a.o + c) : static_cast<size_t>(c)) * a.b + row;
          const double d = __dsub_rn(a.ref[ri], v);
          v = __dmul_rn(d, d);
        }
        ds[rl][qq] = v;
      }
    }
    __syncthreads();
    if (tid < kCands && cols[tid] >= 0) {
      const int c = cols[tid];
      if (kKind == 0) {
        double* o = a.out + (static_cast<size_t>(seg) * a.o + c) * a.b + r0;
        for (int r = 0; r < kRowBlock && r0 + r < a.b; ++r) o[r] = ds[r][tid];
      } else {
        for (int r = 0; r < kRowBlock && r0 + r < a.b; ++r) err = __dadd_rn(err, ds[r][tid]);  // rows in order
      }
    }
    __syncthreads();
  }
  if (kKind != 0 && tid < kCands && q0 + tid < q_count) a.out[static_cast<size_t>(seg) * q_count + q0 + tid] = err;
}

// argmin over the grid in grid order with the reference's predicate
// (search.cpp:147, :310): first || err < best || (err == best && alpha < best_alpha)
__device__ __forceinline__ int pick(const double* e, const float* alpha, int n, double* best_err) {
  int best = 0;
  double be = 0.0;
  float ba = 0.0f;
  for (int i = 0; i < n; ++i) {
    const double v = e[i];
    if (i == 0 || v < be || (v == be && alpha[i] < ba)) {
      best = i;
      be = v;
      ba = alpha[i];
    }
  }
  *best_err = be;
  return best;
}

__global__ void k_phase1_pick(const double* __restrict__ err, const float* __restrict__ alpha, int n_alpha,
                              const float* __restrict__ mn, const float* __restrict__ mx, int n_g, int o, int levels,
                              float* __restrict__ sp, int32_t* __restrict__ zp, float* __restrict__ err_out,
                              float* __restrict__ alpha_out) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;  // k * o + c
  if (i >= static_cast<size_t>(n_g) * o) return;
  double be;
  const int a = pick(err + i * n_alpha, alpha, n_alpha, &be);
  const P1 p = asym_params(mn[i], mx[i], static_cast<double>(alpha[a]), levels);
  sp[i] = p.s;
  zp[i] = p.zp;
  err_out[i] = __double2float_rn(be);
  alpha_out[i] = alpha[a];
}

__global__ void k_phase2_pick(const double* __restrict__ err, const float* __restrict__ alpha, int n_alpha,
                              const float* __restrict__ absmax, int o, float* __restrict__ s1,
                              double* __restrict__ col_err, float* __restrict__ col_alpha) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= o) return;
  double be;
  const int a = pick(err + static_cast<size_t>(c) * n_alpha, alpha, n_alpha, &be);
  s1[c] = p2_s1(absmax[c], alpha[a]);
  col_err[c] = be;
  col_alpha[c] = alpha[a];
}

// The winning candidate's S2 and codes (search.cpp:316-317)
__global__ void k_phase2_emit(const float* __restrict__ W, int h, int o, int g, const float* __restrict__ s1,
                              const float* __restrict__ sp, const int32_t* __restrict__ zp, int8_t* __restrict__ s2,
                              int32_t* __restrict__ codes) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (c >= o) return;
  const size_t kc = static_cast<size_t>(k) * o + c;
  const P2 p = p2_group(s1[c], sp[kc], zp[kc]);
  s2[kc] = static_cast<int8_t>(p.s2);
  for (int j = 0; j < g; ++j) {
    const size_t i = static_cast<size_t>(k) * g + j;
    codes[i * o + c] = p2_code(W[i * o + c], p);
  }
}

}  // namespace search
}  // namespace dgqk

using namespace dgqk::search;

static cudaError_t launch_eval(int kind, const EvalArgs& a, int segs, cudaStream_t st) {
  const long long q = static_cast<long long>(a.o) * (kind == 0 ? 1 : a.n_alpha);
  const dim3 grid(static_cast<unsigned>((q + kCands - 1) / kCands), static_cast<unsigned>(segs));
  const size_t smem = eval_smem_bytes(a.seg_len);
  cudaError_t e = cudaSuccess;
  if (kind == 0 && (e = dgq_allow_smem(k_eval<0>, smem)) == cudaSuccess) k_eval<0><<<grid, kThreads, smem, st>>>(a);
  if (kind == 1 && (e = dgq_allow_smem(k_eval<1>, smem)) == cudaSuccess) k_eval<1><<<grid, kThreads, smem, st>>>(a);
  if (kind == 2 && (e = dgq_allow_smem(k_eval<2>, smem)) == cudaSuccess) k_eval<2><<<grid, kThreads, smem, st>>>(a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t dgq_launch_phase1(const float* W, const float* X, const float* Xhat, int h, int o, int b, int g,
                              int levels, const float* alpha, int n_alpha, float* mn, float* mx, double* ref,
                              double* err, float* sp, int32_t* zp, float* err_out, float* alpha_out,
                              cudaStream_t st) {
  const int n_g = h / g;
  k_group_minmax<<<dim3((o + 127) / 128, n_g), 128, 0, st>>>(W, h, o, g, mn, mx);
  EvalArgs a{};
  a.W = W;
  a.h = h;
  a.o = o;
  a.b = b;
  a.g = g;
  a.n_alpha = n_alpha;
  a.alpha = alpha;
  a.levels = levels;
  a.mn = mn;
  a.mx = mx;
  a.seg_len = g;
  a.X = X;  // refs: the full-precision partial products (search.cpp:128-132)
  a.out = ref;
  cudaError_t e = launch_eval(0, a, n_g, st);
  if (e != cudaSuccess) return e;
  a.X = Xhat;
  a.ref = ref;
  a.out = err;
  e = launch_eval(1, a, n_g, st);
  if (e != cudaSuccess) return e;
  const size_t n = static_cast<size_t>(n_g) * o;
  k_phase1_pick<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(err, alpha, n_alpha, mn, mx, n_g, o, levels,
                                                                         sp, zp, err_out, alpha_out);
  return cudaGetLastError();
}

cudaError_t dgq_launch_phase2(const float* W, const float* X, const float* Xhat, int h, int o, int b, int g,
                              const float* sp, const int32_t* zp, const float* alpha, int n_alpha, float* absmax,
                              double* ref, double* err, float* s1, int8_t* s2, int32_t* codes, double* col_err,
                              float* col_alpha, cudaStream_t st) {
  k_col_absmax<<<(o + 127) / 128, 128, 0, st>>>(W, h, o, absmax);
  EvalArgs a{};
  a.W = W;
  a.h = h;
  a.o = o;
  a.b = b;
  a.g = g;
  a.n_alpha = n_alpha;
  a.alpha = alpha;
  a.absmax = absmax;
  a.sp = sp;
  a.zp = zp;
  a.seg_len = h;
  a.X = X;  // refs: full-column products (search.cpp:286-292)
  a.out = ref;
  cudaError_t e = launch_eval(0, a, 1, st);
  if (e != cudaSuccess) return e;
  a.X = Xhat;
  a.ref = ref;
  a.out = err;
  e = launch_eval(2, a, 1, st);
  if (e != cudaSuccess) return e;
  k_phase2_pick<<<(o + 127) / 128, 128, 0, st>>>(err, alpha, n_alpha, absmax, o, s1, col_err, col_alpha);
  k_phase2_emit<<<dim3((o + 127) / 128, h / g), 128, 0, st>>>(W, h, o, g, s1, sp, zp, s2, codes);
  return cudaGetLastError();
}
