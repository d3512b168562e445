// Device-side building blocks shared by the ABCS kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dct_gen.cuh"

namespace abcs_b200 {

// ---- block transforms -------------------------------------------------------
// Dct<B>::fwd(x, y): y[k] = sum_n C[k][n] x[n]; inv: x[n] = sum_k C[k][n] y[k]
// (orthonormal DCT-II, reference basis dct.cpp:9-21, fp32, generated butterflies).
template <int B> struct Dct;
template <> struct Dct<8> {
  static __device__ __forceinline__ void fwd(const float* x, float* y) { abcs_gen::dct8_fwd(x, y); }
  static __device__ __forceinline__ void inv(const float* y, float* x) { abcs_gen::dct8_inv(y, x); }
};
template <> struct Dct<16> {
  static __device__ __forceinline__ void fwd(const float* x, float* y) { abcs_gen::dct16_fwd(x, y); }
  static __device__ __forceinline__ void inv(const float* y, float* x) { abcs_gen::dct16_inv(y, x); }
};
template <> struct Dct<32> {
  static __device__ __forceinline__ void fwd(const float* x, float* y) { abcs_gen::dct32_fwd(x, y); }
  static __device__ __forceinline__ void inv(const float* y, float* x) { abcs_gen::dct32_inv(y, x); }
};

// A "group" = B consecutive lanes of one warp that own one B x B block
// (lane r of the group holds row r / column r).
template <int B>
__device__ __forceinline__ unsigned group_mask() {
  if (B >= 32) return 0xffffffffu;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned base = lane & ~(unsigned)(B - 1);
  return ((1u << B) - 1u) << base;
}

template <int B>
__device__ __forceinline__ int group_sum(int v) {
#pragma unroll
  for (int o = B / 2; o > 0; o >>= 1) v += __shfl_xor_sync(group_mask<B>(), v, o, B);
  return v;
}

// Padded B x (B+1) float tile in shared memory: conflict-free row and column access.
template <int B>
struct Tile {
  static constexpr int kPitch = B + 1;
  static constexpr int kFloats = B * kPitch;
  float* p;
  __device__ __forceinline__ float& at(int r, int c) { return p[r * kPitch + c]; }
  __device__ __forceinline__ float& zz(int flat) { return p[(flat / B) * kPitch + (flat % B)]; }
};

// Load row r (B pixels) of a u8 block into floats.
template <int B>
__device__ __forceinline__ void load_row_u8(const uint8_t* __restrict__ src, float* x, bool aligned) {
  if (aligned) {
    if constexpr (B == 8) {
      const uint2 v = *reinterpret_cast<const uint2*>(src);
      const uint32_t w[2] = {v.x, v.y};
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = (float)((w[i >> 2] >> (8 * (i & 3))) & 0xffu);
    } else {
#pragma unroll
      for (int q = 0; q < B / 16; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(src + 16 * q);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 16; ++i) x[16 * q + i] = (float)((w[i >> 2] >> (8 * (i & 3))) & 0xffu);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < B; ++i) x[i] = (float)src[i];
  }
}

template <int B>
__device__ __forceinline__ void load_row_f32(const float* __restrict__ src, float* x, bool aligned) {
  if (aligned) {
#pragma unroll
    for (int q = 0; q < B / 4; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(src + 4 * q);
      x[4 * q + 0] = v.x;
      x[4 * q + 1] = v.y;
      x[4 * q + 2] = v.z;
      x[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < B; ++i) x[i] = src[i];
  }
}

template <int B>
__device__ __forceinline__ void store_row_f32(float* __restrict__ dst, const float* x, bool aligned) {
  if (aligned) {
#pragma unroll
    for (int q = 0; q < B / 4; ++q)
      *reinterpret_cast<float4*>(dst + 4 * q) = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < B; ++i) dst[i] = x[i];
  }
}

// Exact unsigned division by a runtime-constant divisor for n, d < 2^31
// (Granlund-Montgomery round-up multiplier): q = (umulhi(m, n) + n) >> l.
struct FastDiv {
  uint32_t d = 1, m = 0, l = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    l = 0;
    while ((1ull << l) < div) ++l;
    m = (uint32_t)((((1ull << 32) * ((1ull << l) - div)) / div) + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((uint64_t)__umulhi(m, n) + n) >> l);
  }
};

// zigzag_order (zigzag.cpp:8-26) and the fp64 reference basis as device tables.
template <int B> __device__ __forceinline__ const unsigned short* zigzag_dev();
template <> __device__ __forceinline__ const unsigned short* zigzag_dev<8>() { return abcs_gen::kZigzagDev8; }
template <> __device__ __forceinline__ const unsigned short* zigzag_dev<16>() { return abcs_gen::kZigzagDev16; }
template <> __device__ __forceinline__ const unsigned short* zigzag_dev<32>() { return abcs_gen::kZigzagDev32; }
template <int B> __device__ __forceinline__ const unsigned short* zigzag_rank_dev();
template <> __device__ __forceinline__ const unsigned short* zigzag_rank_dev<8>() { return abcs_gen::kZigzagRankDev8; }
template <> __device__ __forceinline__ const unsigned short* zigzag_rank_dev<16>() { return abcs_gen::kZigzagRankDev16; }
template <> __device__ __forceinline__ const unsigned short* zigzag_rank_dev<32>() { return abcs_gen::kZigzagRankDev32; }
template <int B> __device__ __forceinline__ const double* basis_dev();
template <> __device__ __forceinline__ const double* basis_dev<8>() { return abcs_gen::kBasisDev8; }
template <> __device__ __forceinline__ const double* basis_dev<16>() { return abcs_gen::kBasisDev16; }
template <> __device__ __forceinline__ const double* basis_dev<32>() { return abcs_gen::kBasisDev32; }

// Copy the zigzag table into shared memory (called by the whole CTA).
template <int B>
__device__ __forceinline__ void load_zigzag(unsigned short* s_zz) {
  const unsigned short* g = zigzag_dev<B>();
  for (int i = threadIdx.x; i < B * B; i += blockDim.x) s_zz[i] = g[i];
}

}  // namespace abcs_b200
