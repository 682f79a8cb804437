// Weight-side kernels: the one-time repack of a reference-layout DGQ layer into
// the prepared tile layout (kernels.h), and the standalone INT4 -> INT8
// dequantisers (K2s) behind the drop-in dequantize_to_s8
// (proj/src/format.cpp:122-141).
#include <cuda_runtime.h>
#include <cstdint>

#include "dequant.cuh"
#include "kernels.h"

namespace dgqk {

__device__ __forceinline__ uint32_t ref_nibble(const uint8_t* p, size_t idx) {
  const uint8_t b = p[idx >> 1];
  return (idx & 1) ? (b >> 4) : (b & 0x0Fu);
}

__constant__ int c_nib_pos[8] = {0, 2, 4, 6, 1, 3, 5, 7};

// one thread per (n-tile, k-block, j, n): 32 codes -> 16 bytes (+ scales when j == 0)
__global__ void k_repack(const uint8_t* __restrict__ codes, const int8_t* __restrict__ s2,
                         const uint8_t* __restrict__ zp, int h, int o_full, int g, int c0, int n_cols,
                         int n_tiles, int k_blocks, int chunk_bytes, int gpk, uint8_t* __restrict__ tiles) {
  const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const size_t total = static_cast<size_t>(n_tiles) * k_blocks * 4 * 128;
  if (tid >= total) return;
  const int n = static_cast<int>(tid % 128);
  const int j = static_cast<int>((tid / 128) % 4);
  const size_t blk = tid / 512;  // nt * k_blocks + kb
  const int kb = static_cast<int>(blk % k_blocks);
  const int nt = static_cast<int>(blk / k_blocks);
  const int col = nt * 128 + n;
  const bool cvalid = col < n_cols;
  const size_t gcol = static_cast<size_t>(c0) + col;
  uint8_t* chunk = tiles + blk * static_cast<size_t>(chunk_bytes);
  uint32_t words[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t word = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int k = kb * 128 + j * 32 + w * 8 + t;
      uint32_t c = 0;
      if (cvalid && k < h) c = ref_nibble(codes, static_cast<size_t>(k) * o_full + gcol);
      word |= c << (4 * c_nib_pos[t]);
    }
    words[w] = word;
  }
  *reinterpret_cast<uint4*>(chunk + j * 2048 + n * 16) = make_uint4(words[0], words[1], words[2], words[3]);
  if (j == 0) {
    uint16_t* sc = reinterpret_cast<uint16_t*>(chunk + 8192);
    for (int gi = 0; gi < gpk; ++gi) {
      const int kstart = kb * 128 + (g >= 128 ? 0 : gi * g);
      uint32_t sv = 1u;  // S2 = 1, ZP = 0 for padding
      if (cvalid && kstart < h) {
        const size_t grp = static_cast<size_t>(kstart / g);
        const uint32_t s = static_cast<uint8_t>(s2[grp * o_full + gcol]);
        const uint32_t z = ref_nibble(zp, grp * o_full + gcol);
        sv = s | (z << 8);
      }
      sc[gi * 128 + n] = static_cast<uint16_t>(sv);
    }
  }
}

// Slab form of the repack for the streaming loader: rows [r0, r0 + rows) of
// the shard's codes (dense [rows x n_cols/2], k-block aligned r0) plus the
// shard's full S2 / ZP ([n_g x n_cols]) -> k-blocks [r0/128, ...) of the tiles.
__global__ void k_repack_slab(const uint8_t* __restrict__ codes, const int8_t* __restrict__ s2,
                              const uint8_t* __restrict__ zp, int h, int r0, int rows, int g, int n_cols, int n_tiles,
                              int k_blocks, int chunk_bytes, int gpk, uint8_t* __restrict__ tiles) {
  const int kb_slab = (rows + 127) / 128, kb0 = r0 / 128;
  const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const size_t total = static_cast<size_t>(n_tiles) * kb_slab * 4 * 128;
  if (tid >= total) return;
  const int n = static_cast<int>(tid % 128);
  const int j = static_cast<int>((tid / 128) % 4);
  const size_t b = tid / 512;
  const int kb = kb0 + static_cast<int>(b % kb_slab);
  const int nt = static_cast<int>(b / kb_slab);
  const int col = nt * 128 + n;
  const bool cvalid = col < n_cols;
  uint8_t* chunk = tiles + (static_cast<size_t>(nt) * k_blocks + kb) * static_cast<size_t>(chunk_bytes);
  uint32_t words[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t word = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int k = kb * 128 + j * 32 + w * 8 + t;  // global row
      uint32_t c = 0;
      if (cvalid && k < h) c = ref_nibble(codes, static_cast<size_t>(k - r0) * n_cols + col);
      word |= c << (4 * c_nib_pos[t]);
    }
    words[w] = word;
  }
  *reinterpret_cast<uint4*>(chunk + j * 2048 + n * 16) = make_uint4(words[0], words[1], words[2], words[3]);
  if (j == 0) {
    uint16_t* sc = reinterpret_cast<uint16_t*>(chunk + 8192);
    for (int gi = 0; gi < gpk; ++gi) {
      const int kstart = kb * 128 + (g >= 128 ? 0 : gi * g);
      uint32_t sv = 1u;  // S2 = 1, ZP = 0 for padding
      if (cvalid && kstart < h) {
        const size_t grp = static_cast<size_t>(kstart / g);
        sv = static_cast<uint32_t>(static_cast<uint8_t>(s2[grp * n_cols + col])) |
             (ref_nibble(zp, grp * n_cols + col) << 8);
      }
      sc[gi * 128 + n] = static_cast<uint16_t>(sv);
    }
  }
}

// validate_layer's O(h o) checks on the GPU (proj/src/format.cpp:44-47, 60-74),
// over a column shard [c0, c0 + n_cols) of an o_full-wide layer.  The first
// violation in the reference's loop order wins: S2 by flat (group, column)
// index, codes by (group, column, row within the group).  ~0 = none.
__global__ void k_validate_s2(const int8_t* __restrict__ s2, int n_g, int n_cols, int c0, int o_full,
                              unsigned long long* first) {
  const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<size_t>(n_g) * n_cols) return;
  const size_t kg = idx / n_cols, c = idx % n_cols;
  if (s2[idx] < 1) atomicMin(first, static_cast<unsigned long long>(kg * o_full + c0 + c));
}
__global__ void k_validate_codes(const uint8_t* __restrict__ codes, const int8_t* __restrict__ s2,
                                 const uint8_t* __restrict__ zp, int r0, int rows, int g, int n_cols, int c0,
                                 int o_full, unsigned long long* first) {
  const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<size_t>(rows) * n_cols) return;
  const size_t il = idx / n_cols, c = idx % n_cols;
  const size_t i = r0 + il, kg = i / g;
  const int sv = s2[kg * n_cols + c];
  if (sv < 1) return;  // reported by k_validate_s2 first
  const int z = static_cast<int>(ref_nibble(zp, kg * n_cols + c));
  const int q = 127 / sv;
  const int lo = z - q > 0 ? z - q : 0, hi = z + q < 15 ? z + q : 15;
  const int code = static_cast<int>(ref_nibble(codes, idx));
  if (code < lo || code > hi)
    atomicMin(first, static_cast<unsigned long long>((kg * o_full + c0 + c) * g + (i - kg * g)));
}

// prepared tiles -> row-major W_s8 via the fused kernel's dequantiser
__global__ void k_dequant_tiles(const uint8_t* __restrict__ tiles, int chunk_bytes, int gshift, int h, int n_cols,
                                int n_tiles, int k_blocks, int8_t* __restrict__ w, size_t ldw) {
  const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const size_t total = static_cast<size_t>(n_tiles) * k_blocks * 4 * 128;
  if (tid >= total) return;
  const int n = static_cast<int>(tid % 128);
  const int j = static_cast<int>((tid / 128) % 4);
  const size_t blk = tid / 512;
  const int kb = static_cast<int>(blk % k_blocks);
  const int nt = static_cast<int>(blk / k_blocks);
  const int col = nt * 128 + n;
  if (col >= n_cols) return;
  const uint8_t* chunk = tiles + blk * static_cast<size_t>(chunk_bytes);
  const uint4 w4 = *reinterpret_cast<const uint4*>(chunk + j * 2048 + n * 16);
  const uint16_t* sc = reinterpret_cast<const uint16_t*>(chunk + 8192);
  const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int koff = j * 32 + q * 8;
    const uint32_t sv = sc[(koff >> gshift) * 128 + n];
    const uint32_t s = sv & 0xFFu, z = sv >> 8;
    uint32_t lo, hi;
    dq_word(ws[q], s, dq_bias2(s, z), lo, hi);
    const uint32_t b[2] = {lo, hi};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int k = kb * 128 + koff + t;
      if (k < h) w[static_cast<size_t>(k) * ldw + col] = static_cast<int8_t>((b[t >> 2] >> (8 * (t & 3))) & 0xFFu);
    }
  }
}

// reference layout -> W_s8, exact integer arithmetic with the range check
__global__ void k_dequant_ref(const uint8_t* __restrict__ codes, const int8_t* __restrict__ s2,
                              const uint8_t* __restrict__ zp, int h, int o, int g, int8_t* __restrict__ w,
                              unsigned long long* bad) {
  const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const size_t total = static_cast<size_t>(h) * o;
  if (idx >= total) return;
  const size_t i = idx / o, c = idx % o;
  const size_t grp = (i / g) * o + c;
  const int v = static_cast<int>(s2[grp]) * (static_cast<int>(ref_nibble(codes, idx)) -
                                             static_cast<int>(ref_nibble(zp, grp)));
  if (v < -127 || v > 127) atomicMin(bad, static_cast<unsigned long long>(idx));
  w[idx] = static_cast<int8_t>(v);
}

// W [K x N] -> WT [Npad x Kpad], 32x32 tiles through smem, zero padding
__global__ void k_transpose_pad(const int8_t* __restrict__ W, int K, int N, int8_t* __restrict__ WT, int Kpad,
                                int Npad) {
  __shared__ int8_t t[32][33];
  const int k0 = blockIdx.x * 32, n0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int k = k0 + r, n = n0 + threadIdx.x;
    t[r][threadIdx.x] = (k < K && n < N) ? W[static_cast<size_t>(k) * N + n] : static_cast<int8_t>(0);
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int n = n0 + r, k = k0 + threadIdx.x;
    if (n < Npad && k < Kpad) WT[static_cast<size_t>(n) * Kpad + k] = t[threadIdx.x][r];
  }
}

}  // namespace dgqk

using namespace dgqk;

cudaError_t dgq_launch_repack(const uint8_t* codes, const int8_t* s2, const uint8_t* zp, int h, int o_full, int g,
                              int c0, int n, int n_tiles, int k_blocks, uint8_t* tiles, cudaStream_t st) {
  const size_t total = static_cast<size_t>(n_tiles) * k_blocks * 512;
  const int cb = dgq_layout::chunk_bytes(g), gpk = dgq_layout::groups_per_kblock(g);
  k_repack<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(codes, s2, zp, h, o_full, g, c0, n, n_tiles,
                                                                        k_blocks, cb, gpk, tiles);
  return cudaGetLastError();
}

cudaError_t dgq_launch_repack_slab(const uint8_t* codes, const int8_t* s2, const uint8_t* zp, int h, int r0, int rows,
                                   int g, int n_cols, int n_tiles, int k_blocks, uint8_t* tiles, cudaStream_t st) {
  const size_t total = static_cast<size_t>(n_tiles) * ((rows + 127) / 128) * 512;
  if (!total) return cudaSuccess;
  const int cb = dgq_layout::chunk_bytes(g), gpk = dgq_layout::groups_per_kblock(g);
  k_repack_slab<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(codes, s2, zp, h, r0, rows, g, n_cols,
                                                                             n_tiles, k_blocks, cb, gpk, tiles);
  return cudaGetLastError();
}

cudaError_t dgq_launch_validate(const uint8_t* codes, const int8_t* s2, const uint8_t* zp, int r0, int rows, int g,
                                int n_g, int n_cols, int c0, int o_full, unsigned long long* first_s2,
                                unsigned long long* first_code, cudaStream_t st) {
  if (first_s2) {
    const size_t n = static_cast<size_t>(n_g) * n_cols;
    if (n) k_validate_s2<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(s2, n_g, n_cols, c0, o_full, first_s2);
  }
  const size_t n = static_cast<size_t>(rows) * n_cols;
  if (n)
    k_validate_codes<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(codes, s2, zp, r0, rows, g, n_cols, c0,
                                                                              o_full, first_code);
  return cudaGetLastError();
}

static int gshift_of(int g) {
  if (g >= 128) return 7;
  int s = 0;
  while ((1 << s) < g) ++s;
  return s;
}

cudaError_t dgq_launch_dequant_tiles(const uint8_t* tiles, int g, int h, int n, int n_tiles, int k_blocks,
                                     int8_t* w, size_t ldw, cudaStream_t st) {
  const size_t total = static_cast<size_t>(n_tiles) * k_blocks * 512;
  k_dequant_tiles<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
      tiles, dgq_layout::chunk_bytes(g), gshift_of(g), h, n, n_tiles, k_blocks, w, ldw);
  return cudaGetLastError();
}

cudaError_t dgq_launch_dequant_ref(const uint8_t* codes, const int8_t* s2, const uint8_t* zp, int h, int o, int g,
                                   int8_t* w, unsigned long long* bad, cudaStream_t st) {
  const size_t total = static_cast<size_t>(h) * o;
  if (!total) return cudaSuccess;
  k_dequant_ref<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(codes, s2, zp, h, o, g, w, bad);
  return cudaGetLastError();
}

cudaError_t dgq_launch_transpose_pad(const int8_t* W, int K, int N, int8_t* WT, int Kpad, int Npad, cudaStream_t st) {
  dim3 grid((Kpad + 31) / 32, (Npad + 31) / 32);
  k_transpose_pad<<<grid, dim3(32, 8), 0, st>>>(W, K, N, WT, Kpad, Npad);
  return cudaGetLastError();
}
