// 8-point orthonormal DCT-II / its inverse on packed fp32 pairs (sm_100 FFMA2 / FADD2 / FMUL2):
// each float2 lane carries one element of two independent vectors, so one instruction advances
// both transforms. Same factorisation and operation order as abcs_gen::dct8_fwd / dct8_inv
// (dct_gen.cuh, generated from the reference basis, dct.cpp:9-21): even/odd butterflies,
// 36 packed operations per transform pair, constants as instruction immediates.
#pragma once
#include <cuda_runtime.h>

namespace abcs_b200 {

__device__ __forceinline__ float2 p_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 p_sub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 p_mul(float k, float2 a) { return __fmul2_rn(make_float2(k, k), a); }
__device__ __forceinline__ float2 p_fma(float k, float2 a, float2 c) { return __ffma2_rn(make_float2(k, k), a, c); }

// y[k] = sum_n C8[k][n] x[n]
__device__ __forceinline__ void dct8_fwd_pair(const float2 (&x)[8], float2 (&y)[8]) {
  const float2 e1 = p_add(x[0], x[7]), o2 = p_sub(x[0], x[7]);
  const float2 e3 = p_add(x[1], x[6]), o4 = p_sub(x[1], x[6]);
  const float2 e5 = p_add(x[2], x[5]), o6 = p_sub(x[2], x[5]);
  const float2 e7 = p_add(x[3], x[4]), o8 = p_sub(x[3], x[4]);
  y[1] = p_fma(9.754516184e-02f, o8, p_fma(2.777851224e-01f, o6, p_fma(4.157347977e-01f, o4, p_mul(4.903926253e-01f, o2))));
  y[3] = p_fma(-2.777851224e-01f, o8, p_fma(-4.903926253e-01f, o6, p_fma(-9.754516184e-02f, o4, p_mul(4.157347977e-01f, o2))));
  y[5] = p_fma(4.157347977e-01f, o8, p_fma(9.754516184e-02f, o6, p_fma(-4.903926253e-01f, o4, p_mul(2.777851224e-01f, o2))));
  y[7] = p_fma(-4.903926253e-01f, o8, p_fma(4.157347977e-01f, o6, p_fma(-2.777851224e-01f, o4, p_mul(9.754516184e-02f, o2))));
  const float2 e9 = p_add(e1, e7), o10 = p_sub(e1, e7);
  const float2 e11 = p_add(e3, e5), o12 = p_sub(e3, e5);
  y[2] = p_fma(1.913417131e-01f, o12, p_mul(4.619397521e-01f, o10));
  y[6] = p_fma(-4.619397521e-01f, o12, p_mul(1.913417131e-01f, o10));
  y[4] = p_mul(3.535533845e-01f, p_sub(e9, e11));
  y[0] = p_mul(3.535533845e-01f, p_add(e9, e11));
}

// x[n] = sum_k C8[k][n] y[k]
__device__ __forceinline__ void dct8_inv_pair(const float2 (&y)[8], float2 (&x)[8]) {
  const float2 s1 = p_mul(3.535533845e-01f, y[0]), q2 = p_mul(3.535533845e-01f, y[4]);
  const float2 s3 = p_add(s1, q2), s4 = p_sub(s1, q2);
  const float2 q5 = p_fma(1.913417131e-01f, y[6], p_mul(4.619397521e-01f, y[2]));
  const float2 q6 = p_fma(-4.619397521e-01f, y[6], p_mul(1.913417131e-01f, y[2]));
  const float2 s7 = p_add(s3, q5), s8 = p_sub(s3, q5), s9 = p_add(s4, q6), s10 = p_sub(s4, q6);
  const float2 q11 = p_fma(9.754516184e-02f, y[7], p_fma(2.777851224e-01f, y[5], p_fma(4.157347977e-01f, y[3], p_mul(4.903926253e-01f, y[1]))));
  const float2 q12 = p_fma(-2.777851224e-01f, y[7], p_fma(-4.903926253e-01f, y[5], p_fma(-9.754516184e-02f, y[3], p_mul(4.157347977e-01f, y[1]))));
  const float2 q13 = p_fma(4.157347977e-01f, y[7], p_fma(9.754516184e-02f, y[5], p_fma(-4.903926253e-01f, y[3], p_mul(2.777851224e-01f, y[1]))));
  const float2 q14 = p_fma(-4.903926253e-01f, y[7], p_fma(4.157347977e-01f, y[5], p_fma(-2.777851224e-01f, y[3], p_mul(9.754516184e-02f, y[1]))));
  x[0] = p_add(s7, q11);
  x[7] = p_sub(s7, q11);
  x[1] = p_add(s9, q12);
  x[6] = p_sub(s9, q12);
  x[2] = p_add(s10, q13);
  x[5] = p_sub(s10, q13);
  x[3] = p_add(s8, q14);
  x[4] = p_sub(s8, q14);
}

// Soft threshold sign(c) max(|c| - t, 0) per lane as c - clamp(c, -t, t) (bit-identical for finite
// c, see ida_mma.cu soft()); t = 0 passes c through (the DC), t = +inf gives 0 (a tile whose
// origin is not on the image's tile grid contributes nothing).
__device__ __forceinline__ float2 p_soft(float2 c, float t0, float t1) {
  const float2 k = make_float2(fminf(fmaxf(c.x, -t0), t0), fminf(fmaxf(c.y, -t1), t1));
  return p_sub(c, k);
}

// clamp(c, -t, t) for t >= 0 in ONE instruction per lane: min.xorsign.abs gives min(|c|, |t|) with
// the sign of c (t's sign bit is clear), SASS FMNMX.XORSIGN. c - clamp(c, -t, t) is the soft
// threshold above, so the IDA denoiser can sum clamps instead (linearity, see ida_mma.cu).
__device__ __forceinline__ float clamp_abs(float c, float t) {
  float r;
  asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(r) : "f"(c), "f"(t));
  return r;
}
__device__ __forceinline__ float2 p_clamp(float2 c, float t0, float t1) {
  return make_float2(clamp_abs(c.x, t0), clamp_abs(c.y, t1));
}

}  // namespace abcs_b200
