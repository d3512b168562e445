// Exact integer emulation of the reference's x87 ranking in
// largest_remainder_allocate (/root/reference/proj/core/src/sensing.cpp:133-158).
//
// The reference computes, per active block,
//     share = (long double)remaining * w / total          (sensing.cpp:144)
//     whole = (long long)share,  frac = share - whole       (:145-148)
// in 80-bit x87 arithmetic (64-bit significand, round-to-nearest-even), then
// hands the leftover units to the largest `frac` (ties -> lower block index,
// :150-158). For integer weights, P = remaining*w and T = sum(w) are exact
// integers (< 2^64), so share = RN64(P / T) exactly. We reproduce RN64(P / T)
// with u128 long division and derive an order-preserving 65-bit key
// (floor(frac * 2^64), frac*2^64-not-integer) that ranks blocks exactly as the
// reference's long-double `frac` does. A plain rational floor/remainder port
// disagrees with the reference on ~0.3% of adversarial vectors;
// this one is checked against the reference on adversarial and realistic
// vectors by tests/native/alloc_keys_check.c (host build of this same header, run from
// tests/test_host_logic.py).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define AK_HD __host__ __device__ __forceinline__
#else
#define AK_HD static inline
#endif

typedef unsigned __int128 ak_u128;

AK_HD int ak_bitlen64(uint64_t v) {
#if defined(__CUDA_ARCH__)
  return v ? 64 - __clzll((long long)v) : 0;
#else
  return v ? 64 - __builtin_clzll(v) : 0;
#endif
}

AK_HD int ak_bitlen128(ak_u128 v) {
  const uint64_t hi = (uint64_t)(v >> 64);
  return hi ? 64 + ak_bitlen64(hi) : ak_bitlen64((uint64_t)v);
}

typedef struct {
  uint64_t whole;  // trunc(share)
  uint64_t key;    // floor(frac * 2^64)
  uint32_t flag;   // frac * 2^64 has a nonzero fractional part
} ak_share;

// floor(R * 2^64 / T) and whether the division leaves a remainder; requires R < T.
AK_HD uint64_t ak_frac64(uint64_t R, uint64_t T, int* sticky) {
  if (T < (1ull << 32)) {  // two 32-bit digits with 64-bit divisions (R < T < 2^32)
    const uint64_t n1 = R << 32;
    const uint64_t q1 = n1 / T;
    const uint64_t n2 = (n1 - q1 * T) << 32;
    const uint64_t q2 = n2 / T;
    *sticky = (n2 - q2 * T) != 0;
    return (q1 << 32) | q2;
  }
  const ak_u128 num = (ak_u128)R << 64;
  const ak_u128 q = num / T;
  const ak_u128 rem = num - q * T;
  *sticky = rem != 0;
  return (uint64_t)q;
}

// share = RN64(P / T) split into whole part and an exact ordering key for its
// fractional part. P = remaining * w (exact), T = total weight > 0.
AK_HD ak_share ak_compute(ak_u128 P, uint64_t T) {
  ak_share s;
  ak_u128 I128;
  uint64_t R;
  if ((uint64_t)(P >> 64) == 0) {  // common case: 64-bit division
    const uint64_t p = (uint64_t)P;
    const uint64_t q = p / T;
    I128 = q;
    R = p - q * T;
  } else {
    I128 = P / T;
    R = (uint64_t)(P - I128 * T);
  }
  s.flag = 0;
  if (R == 0) {  // exact
    s.whole = (uint64_t)I128;
    s.key = 0;
    return s;
  }
  if (I128 != 0) {
    // value in [2^e, 2^(e+1)), 64-bit significand -> f = 63 - e fraction bits kept
    const uint64_t I = (uint64_t)I128;  // I < 2^64 (the reference's share fits long long)
    const int e = ak_bitlen64(I) - 1;
    const int f = 63 - e;
    int sticky;
    const uint64_t X = ak_frac64(R, T, &sticky);
    uint64_t F, rbit;
    int stk;
    if (f == 0) {
      F = 0;
      rbit = X >> 63;
      stk = sticky || (X & 0x7FFFFFFFFFFFFFFFull) != 0;
    } else {
      F = X >> (64 - f);
      rbit = (X >> (63 - f)) & 1u;
      const uint64_t below = (63 - f) > 0 ? (X & ((1ull << (63 - f)) - 1)) : 0;
      stk = sticky || below != 0;
    }
    const ak_u128 N = ((ak_u128)I << f) + F;  // < 2^64
    const uint64_t up = rbit && (stk || (N & 1));
    const ak_u128 N2 = N + up;  // may reach 2^64: then share = 2^(e+1), an integer
    s.whole = (uint64_t)(N2 >> f);
    const uint64_t fb = f ? (uint64_t)(N2 & ((((ak_u128)1) << f) - 1)) : 0;
    s.key = f ? (fb << (64 - f)) : 0;
    return s;
  }
  // I == 0: R/T in [2^-j, 2^(1-j)), significand N = 2^63 + floor(R1/T * 2^63)
  int j = ak_bitlen64(T) - ak_bitlen64(R);
  if ((((ak_u128)R) << j) < (ak_u128)T) ++j;
  const uint64_t R1 = (uint64_t)((((ak_u128)R) << j) - T);  // < T
  int sticky;
  const uint64_t X = ak_frac64(R1, T, &sticky);
  const ak_u128 N = ((ak_u128)1 << 63) + (X >> 1);
  const uint64_t rbit = X & 1u;
  const uint64_t up = rbit && (sticky || (N & 1));
  const ak_u128 N2 = N + up;
  // share = N2 * 2^(-j-63);  share * 2^64 = N2 * 2^(1-j)
  if (N2 >> 64) {  // rounded up to 2^(1-j)
    if (j == 1) {
      s.whole = 1;
      s.key = 0;
    } else {
      s.whole = 0;
      s.key = 1ull << (65 - j);
    }
    return s;
  }
  s.whole = 0;
  if (j == 1) {
    s.key = (uint64_t)N2;
  } else if (j - 1 < 64) {
    s.key = (uint64_t)(N2 >> (j - 1));
    s.flag = (uint64_t)(N2 & ((((ak_u128)1) << (j - 1)) - 1)) != 0;
  } else {
    s.key = 0;
    s.flag = 1;
  }
  return s;
}

// Strict "a ranks before b" in the reference's sort (frac desc, index asc).
AK_HD int ak_before(uint64_t ka, uint32_t fa, uint32_t ia, uint64_t kb, uint32_t fb, uint32_t ib) {
  if (ka != kb) return ka > kb;
  if (fa != fb) return fa > fb;
  return ia < ib;
}
