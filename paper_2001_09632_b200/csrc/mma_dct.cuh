// Tensor-core 16x16 block DCTs (warp per block) with an fp16 hi/lo split that
// keeps fp32-level accuracy.
//
// Y = C X C^T (forward) and X = C^T Y C (inverse) are two 16x16x16 products
// each. With mma.sync.m16n8k16 (fp16 in, fp32 accumulate) the accumulator of
// stage 1 is, register for register, the A fragment of stage 2, so no
// transpose or shared-memory round trip sits between the stages. fp32 operands
// are split v = hi + lo (two fp16, 22 significant bits) and products are
// accumulated as lo-terms first, then hi*hi; u8 pixels are exact in fp16 and
// need no split. Accuracy ~1e-4 absolute on 8-bit blocks (DESIGN.md
// "Precision"), the same order as the fp32 CUDA-core transform.
//
// Fragment layout (PTX ISA, m16n8k16, lane = 4g + t):
//   A (16x16 row-major): a0={A[g][2t],A[g][2t+1]} a1={A[g+8][2t],..} a2={A[g][2t+8],..} a3={A[g+8][2t+8],..}
//   B (16x8):            b0={B[2t][g],B[2t+1][g]} b1={B[2t+8][g],B[2t+9][g]}
//   D (16x8 fp32):       d0=D[g][2t] d1=D[g][2t+1] d2=D[g+8][2t] d3=D[g+8][2t+1]
// For a 16x16 operand split in two n-tiles j (columns 8j..8j+7).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "common.cuh"

namespace abcs_b200 {

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// {a, b} - {c, d} in one packed FADD2 (sm_100: two fp32 lanes per instruction, each RN as FADD)
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n sub.rn.f32x2 rd, ra, rb;\n"
      " mov.b64 {%0,%1}, rd;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

// {a, b} -> hi = fp16(a,b), lo = fp16(a - hi, b - hi)
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 hf = __half22float2(h);
  hi = h2u(h);
  const float2 r = fsub2(make_float2(a, b), hf);
  lo = h2u(__floats2half2_rn(r.x, r.y));
}

// two u8 values (zero-extended) -> exact fp16 pair {lo, hi}
__device__ __forceinline__ uint32_t u8pair_to_h2(uint32_t lo, uint32_t hi) {
  const uint32_t v = __byte_perm(lo, hi, 0x5410) | 0x64006400u;  // 1024 + value
  __half2 h = *reinterpret_cast<const __half2*>(&v);
  h = __hsub2(h, __floats2half2_rn(1024.f, 1024.f));
  return h2u(h);
}

// Per-lane fragments of the B=16 reference basis (dct.cpp:9-21), hi/lo split.
//   c*: C as the A operand (forward stage 1) == C^T as the B operand (forward stage 2)
//   t*: C^T as the A operand (inverse stage 1) == C as the B operand (inverse stage 2)
struct Frag16 {
  uint32_t ch[4], cl[4], th[4], tl[4];
  // the same values regrouped as stage-2 B operands (adjacent registers per n-tile):
  // cb*[j] = {c*[j], c*[j+2]} (C^T as B), tb*[j] = {t*[j], t*[j+2]} (C as B)
  uint32_t cbh[2][2], cbl[2][2], tbh[2][2], tbl[2][2];
};

__device__ __forceinline__ void load_frag16(Frag16& f) {
  const double* Cd = basis_dev<16>();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  auto C = [&](int r, int c) { return (float)Cd[r * 16 + c]; };
  const int rows[4] = {g, g + 8, g, g + 8};
  const int cols[4] = {2 * t, 2 * t, 2 * t + 8, 2 * t + 8};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    split2(C(rows[i], cols[i]), C(rows[i], cols[i] + 1), f.ch[i], f.cl[i]);       // C[r][c], C[r][c+1]
    split2(C(cols[i], rows[i]), C(cols[i] + 1, rows[i]), f.th[i], f.tl[i]);       // C^T[r][c] = C[c][r]
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    f.cbh[j][0] = f.ch[j];
    f.cbh[j][1] = f.ch[j + 2];
    f.cbl[j][0] = f.cl[j];
    f.cbl[j][1] = f.cl[j + 2];
    f.tbh[j][0] = f.th[j];
    f.tbh[j][1] = f.th[j + 2];
    f.tbl[j][0] = f.tl[j];
    f.tbl[j][1] = f.tl[j + 2];
  }
}

// D fragments of a 16x16 result: v[j][0..3] for n-tile j.
struct Acc16 {
  float v[2][4];
};

// Stage-2 helper: A = S (from accumulator frags, split hi/lo), B = M given per n-tile
// as adjacent register pairs bh[j], bl[j]. Returns S * M.
__device__ __forceinline__ Acc16 stage2(const Acc16& S, const uint32_t (&bh)[2][2], const uint32_t (&bl)[2][2]) {
  uint32_t ah[4], al[4];
  split2(S.v[0][0], S.v[0][1], ah[0], al[0]);
  split2(S.v[0][2], S.v[0][3], ah[1], al[1]);
  split2(S.v[1][0], S.v[1][1], ah[2], al[2]);
  split2(S.v[1][2], S.v[1][3], ah[3], al[3]);
  Acc16 R;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    R.v[j][0] = R.v[j][1] = R.v[j][2] = R.v[j][3] = 0.f;
    mma16816(R.v[j], al, bh[j][0], bh[j][1]);
    mma16816(R.v[j], ah, bl[j][0], bl[j][1]);
    mma16816(R.v[j], ah, bh[j][0], bh[j][1]);
  }
  return R;
}

// Stage 2 with the basis B pairs read from a shared table (lane-minor, conflict-free LDS.64):
// tab[(2j + {0 hi, 1 lo}) * 32 + lane]. Saves the register moves that pair non-adjacent A-quad
// registers into B operands.
__device__ __forceinline__ Acc16 stage2_tab(const Acc16& S, const uint2* tab) {
  const int lane = threadIdx.x & 31;
  uint32_t ah[4], al[4];
  split2(S.v[0][0], S.v[0][1], ah[0], al[0]);
  split2(S.v[0][2], S.v[0][3], ah[1], al[1]);
  split2(S.v[1][0], S.v[1][1], ah[2], al[2]);
  split2(S.v[1][2], S.v[1][3], ah[3], al[3]);
  Acc16 R;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const uint2 bh = tab[(2 * j) * 32 + lane], bl = tab[(2 * j + 1) * 32 + lane];
    R.v[j][0] = R.v[j][1] = R.v[j][2] = R.v[j][3] = 0.f;
    mma16816(R.v[j], al, bh.x, bh.y);
    mma16816(R.v[j], ah, bl.x, bl.y);
    mma16816(R.v[j], ah, bh.x, bh.y);
  }
  return R;
}

// Fill a 8 x 32 uint2 table: rows 0-3 forward stage-2 pairs (C^T as B), rows 4-7 inverse (C as B).
__device__ __forceinline__ void fill_btab16(const Frag16& f, uint2* tab) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    tab[(2 * j) * 32 + lane] = make_uint2(f.cbh[j][0], f.cbh[j][1]);
    tab[(2 * j + 1) * 32 + lane] = make_uint2(f.cbl[j][0], f.cbl[j][1]);
    tab[(4 + 2 * j) * 32 + lane] = make_uint2(f.tbh[j][0], f.tbh[j][1]);
    tab[(4 + 2 * j + 1) * 32 + lane] = make_uint2(f.tbl[j][0], f.tbl[j][1]);
  }
}

// Forward DCT of an exact-fp16 block given as B fragments bx[j][0..1] (n-tile j):
//   T = C X (stage 1), Y = T C^T (stage 2). Returns Y in D-fragment layout.
__device__ __forceinline__ Acc16 dct16_fwd_exact(const Frag16& f, const uint32_t (&bx)[2][2]) {
  Acc16 T;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    T.v[j][0] = T.v[j][1] = T.v[j][2] = T.v[j][3] = 0.f;
    mma16816(T.v[j], f.cl, bx[j][0], bx[j][1]);
    mma16816(T.v[j], f.ch, bx[j][0], bx[j][1]);
  }
  return stage2(T, f.cbh, f.cbl);
}

// Two exact-fp16 blocks at once (independent MMA chains interleave).
__device__ __forceinline__ void dct16_fwd_exact_x2(const Frag16& f, const uint32_t (&bx)[2][2][2], Acc16 (&Y)[2]) {
  Acc16 T[2];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int j = 0; j < 2; ++j) T[q].v[j][0] = T[q].v[j][1] = T[q].v[j][2] = T[q].v[j][3] = 0.f;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int q = 0; q < 2; ++q) mma16816(T[q].v[j], f.cl, bx[q][j][0], bx[q][j][1]);
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int q = 0; q < 2; ++q) mma16816(T[q].v[j], f.ch, bx[q][j][0], bx[q][j][1]);
#pragma unroll
  for (int q = 0; q < 2; ++q) Y[q] = stage2(T[q], f.cbh, f.cbl);
}

// dct16_fwd_exact_x2 with stage-2 B pairs from the shared table (fill_btab16)
__device__ __forceinline__ void dct16_fwd_exact_x2_tab(const Frag16& f, const uint2* tab, const uint32_t (&bx)[2][2][2],
                                                       Acc16 (&Y)[2]) {
  Acc16 T[2];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int j = 0; j < 2; ++j) T[q].v[j][0] = T[q].v[j][1] = T[q].v[j][2] = T[q].v[j][3] = 0.f;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int q = 0; q < 2; ++q) mma16816(T[q].v[j], f.cl, bx[q][j][0], bx[q][j][1]);
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int q = 0; q < 2; ++q) mma16816(T[q].v[j], f.ch, bx[q][j][0], bx[q][j][1]);
#pragma unroll
  for (int q = 0; q < 2; ++q) Y[q] = stage2_tab(T[q], tab);
}

// Same, computing only rows 0..7 and columns 0..7 of Y^T (n-tile 0, A rows g): enough when
// every wanted coefficient has u, v <= 7 (DD phase 1 with a zigzag prefix of <= 36 entries).
__device__ __forceinline__ void dct16_fwd_exact_x2_lo(const Frag16& f, const uint32_t (&bx)[2][2][2], Acc16 (&Y)[2]) {
  Acc16 T[2];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int j = 0; j < 2; ++j) T[q].v[j][0] = T[q].v[j][1] = T[q].v[j][2] = T[q].v[j][3] = 0.f;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int q = 0; q < 2; ++q) mma16816(T[q].v[j], f.cl, bx[q][j][0], bx[q][j][1]);
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int q = 0; q < 2; ++q) mma16816(T[q].v[j], f.ch, bx[q][j][0], bx[q][j][1]);
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    // output rows 8..15 (v >= 8) are not wanted: their A rows (a1, a3) stay zero
    uint32_t ah[4], al[4];
    split2(T[q].v[0][0], T[q].v[0][1], ah[0], al[0]);
    split2(T[q].v[1][0], T[q].v[1][1], ah[2], al[2]);
    ah[1] = al[1] = ah[3] = al[3] = 0u;
    Y[q].v[0][0] = Y[q].v[0][1] = Y[q].v[0][2] = Y[q].v[0][3] = 0.f;
    Y[q].v[1][0] = Y[q].v[1][1] = Y[q].v[1][2] = Y[q].v[1][3] = 0.f;
    mma16816(Y[q].v[0], al, f.cbh[0][0], f.cbh[0][1]);
    mma16816(Y[q].v[0], ah, f.cbl[0][0], f.cbl[0][1]);
    mma16816(Y[q].v[0], ah, f.cbh[0][0], f.cbh[0][1]);
  }
}

// Forward DCT of an fp32 block given as B-fragment values xv[j][0..3] =
// {X[2t][8j+g], X[2t+1][8j+g], X[2t+8][8j+g], X[2t+9][8j+g]}.
__device__ __forceinline__ Acc16 dct16_fwd_f32(const Frag16& f, const float (&xv)[2][4]) {
  Acc16 T;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    uint32_t h0, l0, h1, l1;
    split2(xv[j][0], xv[j][1], h0, l0);
    split2(xv[j][2], xv[j][3], h1, l1);
    T.v[j][0] = T.v[j][1] = T.v[j][2] = T.v[j][3] = 0.f;
    mma16816(T.v[j], f.ch, l0, l1);
    mma16816(T.v[j], f.cl, h0, h1);
    mma16816(T.v[j], f.ch, h0, h1);
  }
  return stage2(T, f.cbh, f.cbl);
}

// Inverse DCT of an fp32 coefficient block given as B-fragment values yv[j][0..3]
// (same positions as dct16_fwd_f32). Returns X in D-fragment layout.
__device__ __forceinline__ Acc16 dct16_inv_f32(const Frag16& f, const float (&yv)[2][4]) {
  Acc16 T;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    uint32_t h0, l0, h1, l1;
    split2(yv[j][0], yv[j][1], h0, l0);
    split2(yv[j][2], yv[j][3], h1, l1);
    T.v[j][0] = T.v[j][1] = T.v[j][2] = T.v[j][3] = 0.f;
    mma16816(T.v[j], f.th, l0, l1);
    mma16816(T.v[j], f.tl, h0, h1);
    mma16816(T.v[j], f.th, h0, h1);
  }
  return stage2(T, f.tbh, f.tbl);
}

// Inverse DCT X = C^T Y C where Y is given TRANSPOSED in D-fragment layout, i.e. the
// output of a forward transform computed as Y^T = C X^T C^T: the accumulator pairs of
// Y^T are exactly the stage-1 B fragments of Y (tile 0: {D0.d0,d1},{D1.d0,d1};
// tile 1: {D0.d2,d3},{D1.d2,d3}), so the fused decode needs no shuffle or smem.
__device__ __forceinline__ Acc16 dct16_inv_from_yt(const Frag16& f, const Acc16& Yt) {
  uint32_t bh[2][2], bl[2][2];
  split2(Yt.v[0][0], Yt.v[0][1], bh[0][0], bl[0][0]);
  split2(Yt.v[1][0], Yt.v[1][1], bh[0][1], bl[0][1]);
  split2(Yt.v[0][2], Yt.v[0][3], bh[1][0], bl[1][0]);
  split2(Yt.v[1][2], Yt.v[1][3], bh[1][1], bl[1][1]);
  Acc16 T;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    T.v[j][0] = T.v[j][1] = T.v[j][2] = T.v[j][3] = 0.f;
    mma16816(T.v[j], f.th, bl[j][0], bl[j][1]);
    mma16816(T.v[j], f.tl, bh[j][0], bh[j][1]);
    mma16816(T.v[j], f.th, bh[j][0], bh[j][1]);
  }
  return stage2(T, f.tbh, f.tbl);
}

// A 16-byte block row with its bytes reordered to [0,1,8,9 | 2,3,10,11 | 4,5,12,13 | 6,7,14,15]:
// word t then holds exactly the two byte pairs lane (g, t) needs (see u8_bfragT_il).
// The B = 16 fragments as a shared table (register-lean kernels): per lane the A quads
// ch, cl, th, tl and the stage-2 B pairs of fill_btab16. Filled by one warp.
struct Frag16Tab {
  uint4 a[4][32];
  uint2 b[8][32];
};
__device__ __forceinline__ void fill_frag16_tab(Frag16Tab& T) {
  const int lane = threadIdx.x & 31;
  Frag16 f;
  load_frag16(f);
  T.a[0][lane] = make_uint4(f.ch[0], f.ch[1], f.ch[2], f.ch[3]);
  T.a[1][lane] = make_uint4(f.cl[0], f.cl[1], f.cl[2], f.cl[3]);
  T.a[2][lane] = make_uint4(f.th[0], f.th[1], f.th[2], f.th[3]);
  T.a[3][lane] = make_uint4(f.tl[0], f.tl[1], f.tl[2], f.tl[3]);
  fill_btab16(f, &T.b[0][0]);
}
__device__ __forceinline__ void quad(uint4 q, uint32_t (&a)[4]) {
  a[0] = q.x;
  a[1] = q.y;
  a[2] = q.z;
  a[3] = q.w;
}
// dct16_fwd_f32 with the fragments read from the table at the point of use.
__device__ __forceinline__ Acc16 dct16_fwd_f32_t(const Frag16Tab& F, const float (&xv)[2][4]) {
  const int lane = threadIdx.x & 31;
  uint32_t ch[4], cl[4];
  quad(F.a[0][lane], ch);
  quad(F.a[1][lane], cl);
  Acc16 T;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    uint32_t h0, l0, h1, l1;
    split2(xv[j][0], xv[j][1], h0, l0);
    split2(xv[j][2], xv[j][3], h1, l1);
    T.v[j][0] = T.v[j][1] = T.v[j][2] = T.v[j][3] = 0.f;
    mma16816(T.v[j], ch, l0, l1);
    mma16816(T.v[j], cl, h0, h1);
    mma16816(T.v[j], ch, h0, h1);
  }
  return stage2_tab(T, &F.b[0][0]);
}
// dct16_inv_from_yt with the fragments read from the table at the point of use.
__device__ __forceinline__ Acc16 dct16_inv_from_yt_t(const Frag16Tab& F, const Acc16& Yt) {
  const int lane = threadIdx.x & 31;
  uint32_t bh[2][2], bl[2][2];
  split2(Yt.v[0][0], Yt.v[0][1], bh[0][0], bl[0][0]);
  split2(Yt.v[1][0], Yt.v[1][1], bh[0][1], bl[0][1]);
  split2(Yt.v[0][2], Yt.v[0][3], bh[1][0], bl[1][0]);
  split2(Yt.v[1][2], Yt.v[1][3], bh[1][1], bl[1][1]);
  uint32_t th[4], tl[4];
  quad(F.a[2][lane], th);
  quad(F.a[3][lane], tl);
  Acc16 T;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    T.v[j][0] = T.v[j][1] = T.v[j][2] = T.v[j][3] = 0.f;
    mma16816(T.v[j], th, bl[j][0], bl[j][1]);
    mma16816(T.v[j], tl, bh[j][0], bh[j][1]);
    mma16816(T.v[j], th, bh[j][0], bh[j][1]);
  }
  return stage2_tab(T, &F.b[4][0]);
}

// dct16_inv_from_yt for a Y^T supported on its top-left 8x8 (slots 0/1 only: zigzag ranks
// < 36): stage 1's second n-tile is zero and stage 2's k-range 8..15 is zero, so 9 of the 12
// MMAs and 4 of the 8 splits remain. Bit-identical to dct16_inv_from_yt on such input (the
// skipped terms are exact zeros).
__device__ __forceinline__ Acc16 dct16_inv_from_yt_lo(const Frag16& f, const Acc16& Yt) {
  uint32_t bh0, bl0;
  split2(Yt.v[0][0], Yt.v[0][1], bh0, bl0);
  Acc16 T;
  T.v[0][0] = T.v[0][1] = T.v[0][2] = T.v[0][3] = 0.f;
  mma16816(T.v[0], f.th, bl0, 0u);
  mma16816(T.v[0], f.tl, bh0, 0u);
  mma16816(T.v[0], f.th, bh0, 0u);
  uint32_t ah[4], al[4];
  split2(T.v[0][0], T.v[0][1], ah[0], al[0]);
  split2(T.v[0][2], T.v[0][3], ah[1], al[1]);
  ah[2] = al[2] = ah[3] = al[3] = 0u;
  Acc16 R;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    R.v[j][0] = R.v[j][1] = R.v[j][2] = R.v[j][3] = 0.f;
    mma16816(R.v[j], al, f.tbh[j][0], f.tbh[j][1]);
    mma16816(R.v[j], ah, f.tbl[j][0], f.tbl[j][1]);
    mma16816(R.v[j], ah, f.tbh[j][0], f.tbh[j][1]);
  }
  return R;
}

// Y^T split once into the stage-1 B operands of the inverse (dct16_inv_from_yt's pairs:
// slots {0,1}, {4,5}, {2,3}, {6,7}); plans then mask the split halves instead of re-splitting.
struct YtSplit {
  uint32_t h[2][2], l[2][2];
};
__device__ __forceinline__ YtSplit split_yt(const Acc16& Yt) {
  YtSplit r;
  split2(Yt.v[0][0], Yt.v[0][1], r.h[0][0], r.l[0][0]);
  split2(Yt.v[1][0], Yt.v[1][1], r.h[0][1], r.l[0][1]);
  split2(Yt.v[0][2], Yt.v[0][3], r.h[1][0], r.l[1][0]);
  split2(Yt.v[1][2], Yt.v[1][3], r.h[1][1], r.l[1][1]);
  return r;
}
// per-half 0xffff where rank < count (ranks and count as exact fp16 pairs)
__device__ __forceinline__ uint32_t h2_lt_mask(uint32_t ranks, uint32_t count) {
  uint32_t m;
  asm("set.lt.u32.f16x2 %0, %1, %2;" : "=r"(m) : "r"(ranks), "r"(count));
  return m;
}
// The zigzag-prefix mask of a plan applied to the split halves: bit-identical to splitting the
// masked Y^T (a masked value splits to +0 / +0). rk[j][i]: the slot pair's ranks as fp16x2.
__device__ __forceinline__ YtSplit mask_yt(const YtSplit& S, const uint32_t (&rk)[2][2], uint32_t count_h2) {
  YtSplit r;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const uint32_t m = h2_lt_mask(rk[j][i], count_h2);
      r.h[j][i] = S.h[j][i] & m;
      r.l[j][i] = S.l[j][i] & m;
    }
  return r;
}
// dct16_inv_from_yt from pre-split (masked) operands
__device__ __forceinline__ Acc16 dct16_inv_from_split(const Frag16& f, const YtSplit& S) {
  Acc16 T;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    T.v[j][0] = T.v[j][1] = T.v[j][2] = T.v[j][3] = 0.f;
    mma16816(T.v[j], f.th, S.l[j][0], S.l[j][1]);
    mma16816(T.v[j], f.tl, S.h[j][0], S.h[j][1]);
    mma16816(T.v[j], f.th, S.h[j][0], S.h[j][1]);
  }
  return stage2(T, f.tbh, f.tbl);
}
// dct16_inv_from_yt_lo from pre-split (masked) operands: only slots {0,1} (S.h/l[0][0])
__device__ __forceinline__ Acc16 dct16_inv_from_split_lo(const Frag16& f, const YtSplit& S) {
  Acc16 T;
  T.v[0][0] = T.v[0][1] = T.v[0][2] = T.v[0][3] = 0.f;
  mma16816(T.v[0], f.th, S.l[0][0], 0u);
  mma16816(T.v[0], f.tl, S.h[0][0], 0u);
  mma16816(T.v[0], f.th, S.h[0][0], 0u);
  uint32_t ah[4], al[4];
  split2(T.v[0][0], T.v[0][1], ah[0], al[0]);
  split2(T.v[0][2], T.v[0][3], ah[1], al[1]);
  ah[2] = al[2] = ah[3] = al[3] = 0u;
  Acc16 R;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    R.v[j][0] = R.v[j][1] = R.v[j][2] = R.v[j][3] = 0.f;
    mma16816(R.v[j], al, f.tbh[j][0], f.tbh[j][1]);
    mma16816(R.v[j], ah, f.tbl[j][0], f.tbl[j][1]);
    mma16816(R.v[j], ah, f.tbh[j][0], f.tbh[j][1]);
  }
  return R;
}

__device__ __forceinline__ uint4 interleave_row16(uint4 v) {
  return make_uint4(__byte_perm(v.x, v.z, 0x5410), __byte_perm(v.x, v.z, 0x7632), __byte_perm(v.y, v.w, 0x5410),
                    __byte_perm(v.y, v.w, 0x7632));
}

// bytes 0,1 (sel 0x4140) or 2,3 (sel 0x4342) of w -> exact fp16 pair: 0x64 high bytes make 1024 + v
__device__ __forceinline__ uint32_t u8sel_to_h2(uint32_t w, uint32_t sel) {
  const uint32_t v = __byte_perm(w, 0x64646464u, sel);
  __half2 h = *reinterpret_cast<const __half2*>(&v);
  h = __hadd2(h, __floats2half2_rn(-1024.f, -1024.f));
  return h2u(h);
}

// B fragments of X^T from a block staged with interleave_row16 rows (16-byte pitch): one
// 32-bit load per n-tile gives {X[8j+g][2t], X[8j+g][2t+1]} and {X[8j+g][2t+8], X[8j+g][2t+9]}.
__device__ __forceinline__ void u8_bfragT_il(const uint8_t* blk, uint32_t (&bx)[2][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(blk + (8 * j + g) * 16 + 4 * t);
    bx[j][0] = u8sel_to_h2(w, 0x4140);
    bx[j][1] = u8sel_to_h2(w, 0x4342);
  }
}

// dct16_inv_from_yt with stage-2 B pairs from the shared table (rows 4-7)
__device__ __forceinline__ Acc16 dct16_inv_from_yt_tab(const Frag16& f, const uint2* tab, const Acc16& Yt) {
  uint32_t bh[2][2], bl[2][2];
  split2(Yt.v[0][0], Yt.v[0][1], bh[0][0], bl[0][0]);
  split2(Yt.v[1][0], Yt.v[1][1], bh[0][1], bl[0][1]);
  split2(Yt.v[0][2], Yt.v[0][3], bh[1][0], bl[1][0]);
  split2(Yt.v[1][2], Yt.v[1][3], bh[1][1], bl[1][1]);
  Acc16 T;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    T.v[j][0] = T.v[j][1] = T.v[j][2] = T.v[j][3] = 0.f;
    mma16816(T.v[j], f.th, bl[j][0], bl[j][1]);
    mma16816(T.v[j], f.tl, bh[j][0], bh[j][1]);
    mma16816(T.v[j], f.th, bh[j][0], bh[j][1]);
  }
  return stage2_tab(T, tab + 4 * 32);
}

// B fragments of X^T (for the transposed forward) from a u8 block in smem with a
// 16-byte row pitch: tile j: {X[8j+g][2t], X[8j+g][2t+1]}, {X[8j+g][2t+8], X[8j+g][2t+9]}
// -- contiguous byte pairs, one 16-bit load each.
__device__ __forceinline__ void u8_bfragT(const uint8_t* blk, uint32_t (&bx)[2][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const uint8_t* row = blk + (8 * j + g) * 16 + 2 * t;
    const uint32_t p0 = *reinterpret_cast<const uint16_t*>(row);
    const uint32_t p1 = *reinterpret_cast<const uint16_t*>(row + 8);
    bx[j][0] = u8pair_to_h2(p0 & 0xffu, p0 >> 8);
    bx[j][1] = u8pair_to_h2(p1 & 0xffu, p1 >> 8);
  }
}

// ---------------------------------------------------------------------------
// 8x8 transforms, two blocks per warp step. The forward runs transposed
// (Y^T = C8 P^T C8^T, as for B = 16) so its accumulator pairs are the inverse's
// stage-1 B fragments. Slot layout of the 16x8 results: rows g / g+8 = row g of
// block 0 / block 1, columns 2t, 2t+1.
//
// Stage 1 (per block, no block-diagonal padding): one m16n8k16 with
//   A = [Mh Mh; Ml Ml] (the basis hi/lo split over the two row halves),
//   B = [Ph^T; Pl^T]   (the operand's hi/lo split over the two k halves),
// so rows g and g+8 of D are Mh*P and Ml*P; their sum (one FADD2) is M*P to ~fp32
// accuracy, and the two blocks' MMAs are independent. For exact (u8) operands
// one m16n8k8 with A = [Mh; Ml] suffices. Stage 2 uses m16n8k8 whose A fragment
// is the stage-1 result of both blocks (rows g: block 0, g+8: block 1).
__device__ __forceinline__ void mma1688(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(b0));
}

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n add.rn.f32x2 rd, ra, rb;\n"
      " mov.b64 {%0,%1}, rd;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

struct Frag8 {
  uint32_t ch, cl;  // {C8[g][2t], C8[g][2t+1]} hi/lo: C8 rows as A (forward stage 1) == C8^T as B (stage 2)
  uint32_t th, tl;  // {C8[2t][g], C8[2t+1][g]} hi/lo: C8^T rows as A (inverse stage 1) == C8 as B
};

__device__ __forceinline__ void load_frag8(Frag8& f) {
  const double* C = basis_dev<8>();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  split2((float)C[g * 8 + 2 * t], (float)C[g * 8 + 2 * t + 1], f.ch, f.cl);
  split2((float)C[(2 * t) * 8 + g], (float)C[(2 * t + 1) * 8 + g], f.th, f.tl);
}

// M * P^T for one block: A = [Mh Mh; Ml Ml], B = {hi pair, lo pair} of the lane's P[g][2t..2t+1].
__device__ __forceinline__ float2 stage1_8(uint32_t mh, uint32_t ml, uint32_t bh, uint32_t bl) {
  float d[4] = {0.f, 0.f, 0.f, 0.f};
  const uint32_t a[4] = {mh, ml, mh, ml};
  mma16816(d, a, bh, bl);
  return fadd2(make_float2(d[0], d[1]), make_float2(d[2], d[3]));
}

// The same for an exact fp16 operand pair (u8 pixels).
__device__ __forceinline__ float2 stage1_8_exact(uint32_t mh, uint32_t ml, uint32_t b) {
  float d[4] = {0.f, 0.f, 0.f, 0.f};
  mma1688(d, mh, ml, b);
  return fadd2(make_float2(d[0], d[1]), make_float2(d[2], d[3]));
}

// Stage 2 of both blocks: S (rows g: block 0 pair s0, g+8: block 1 pair s1) times the
// basis given as the B operand pair (bh, bl).
__device__ __forceinline__ void stage2_8(float2 s0, float2 s1, uint32_t bh, uint32_t bl, float (&R)[4]) {
  uint32_t h0, l0, h1, l1;
  split2(s0.x, s0.y, h0, l0);
  split2(s1.x, s1.y, h1, l1);
  R[0] = R[1] = R[2] = R[3] = 0.f;
  mma1688(R, l0, l1, bh);
  mma1688(R, h0, h1, bl);
  mma1688(R, h0, h1, bh);
}

// Y^T of two fp32 blocks; lane (g, t) holds p0 = P0[g][2t..2t+1], p1 = P1[g][2t..2t+1].
__device__ __forceinline__ void dct8x2_fwdT(const Frag8& f, float2 p0, float2 p1, float (&Y)[4]) {
  uint32_t h0, l0, h1, l1;
  split2(p0.x, p0.y, h0, l0);
  split2(p1.x, p1.y, h1, l1);
  const float2 q0 = stage1_8(f.ch, f.cl, h0, l0);
  const float2 q1 = stage1_8(f.ch, f.cl, h1, l1);
  stage2_8(q0, q1, f.ch, f.cl, Y);
}

// Y^T of two u8 blocks given as exact fp16 pairs b0 (block 0) and b1 (block 1).
__device__ __forceinline__ void dct8x2_fwdT_exact(const Frag8& f, uint32_t b0, uint32_t b1, float (&Y)[4]) {
  const float2 q0 = stage1_8_exact(f.ch, f.cl, b0);
  const float2 q1 = stage1_8_exact(f.ch, f.cl, b1);
  stage2_8(q0, q1, f.ch, f.cl, Y);
}

// X = C8^T Y C8 of two blocks given as Y^T in the slot layout (output of dct8x2_fwdT).
__device__ __forceinline__ void dct8x2_inv_from_yt(const Frag8& f, const float (&Yt)[4], float (&X)[4]) {
  uint32_t h0, l0, h1, l1;
  split2(Yt[0], Yt[1], h0, l0);
  split2(Yt[2], Yt[3], h1, l1);
  const float2 r0 = stage1_8(f.th, f.tl, h0, l0);
  const float2 r1 = stage1_8(f.th, f.tl, h1, l1);
  stage2_8(r0, r1, f.th, f.tl, X);
}

// Positions of the D-fragment slots: slot s = 4j + i -> (row, col)
__device__ __forceinline__ int dslot_row(int s) { return ((threadIdx.x & 31) >> 2) + ((s & 3) >= 2 ? 8 : 0); }
__device__ __forceinline__ int dslot_col(int s) { return 8 * (s >> 2) + 2 * (threadIdx.x & 3) + (s & 1); }
// Positions of the B-fragment value slots xv[j][i]: (row, col)
__device__ __forceinline__ int bslot_row(int s) {
  return 2 * (threadIdx.x & 3) + (s & 1) + ((s & 3) >= 2 ? 8 : 0);
}
__device__ __forceinline__ int bslot_col(int s) { return 8 * (s >> 2) + ((threadIdx.x & 31) >> 2); }

}  // namespace abcs_b200
