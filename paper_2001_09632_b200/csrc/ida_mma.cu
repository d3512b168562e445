// Tensor-core IDA iteration and dct_threshold denoiser for B = 8 and 16
// (recon.cpp:199-259, denoise.cpp:52-92; the CUDA-core kernels in ida.cu keep B = 32).
//
// One CTA owns a 64x64 output region of one image and runs, per launch:
//   1. the 72x72 field window (4-px halo) HBM -> smem (float4);
//   2. the denoiser: the 17x17 grid of 8x8 tiles at stride 4 touching the region
//      is processed in the 4 parity phases (tiles of one phase never overlap, and
//      the phase order fixes each pixel's summation order). A warp transforms two
//      horizontally adjacent tiles per step on the tensor cores: Y^T = C8 P^T C8^T
//      (m16n8k16 with diag(C8, C8), then m16n8k8), soft threshold in registers
//      (DC kept, denoise.cpp:76), X = C8^T Y C8 straight from the Y^T accumulators,
//      and overlap-add into the smem accumulator; then / weight (denoise.cpp:90);
//   3. the block phase per sensing block (B = 16: one block per warp step with the
//      m16n8k16 transforms of mma_dct.cuh; B = 8: two blocks per step):
//        z_new = (y - A x) + z_old / D_F, pseudo = x + A* z_new  (recon.cpp:81-93, 75-79)
//      with y / z prefixes staged through smem by coalesced loads and the
//      transposed forward's slots indexing them by zigzag rank;
//   4. per-image reductions folded by the last CTA (finish_image).
// fp32 operands are split into fp16 hi/lo pairs (mma_dct.cuh), ~fp32 accuracy.
#include <cfloat>
#include <cstring>
#include <type_traits>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ida_common.cuh"
#include "internal.h"
#include "dct_pair.cuh"
#include "mma_dct.cuh"

namespace abcs_b200 {

constexpr int kMR = 64;          // output region side
constexpr int kMIn = kMR + 8;    // 72: region + 4-px halo each side
constexpr int kWinBytes = 76 * kMIn * 4;  // the fused kernel's TMA window box (kWP x kMIn floats)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// 16-byte async copy global -> shared; src_bytes = 0 zero-fills (out-of-image window parts)
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// The 76 x 72 window (4-px halo, 4 spare columns) of image `img` by one TMA tile copy: the 3-D
// tensor map (Wc, Hc, n) of the pseudo field fills out-of-image elements with zeros, which is the
// denoiser's boundary (tiles there are off the grid and weigh nothing).
__device__ __forceinline__ void tma_window(float* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
  const uint32_t b = smem_u32(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(kWinBytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
      ::"r"(smem_u32(dst)), "l"(tm), "r"(x), "r"(y), "r"(z), "r"(b)
      : "memory");
}
__device__ __forceinline__ void tma_window_wait(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred p;\nWIN_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      "@!p bra WIN_WAIT_%=;\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}


// field[R0-4 .. R0+68) x [C0-4 .. C0+68) -> s.in (zeros outside the image). The vector path
// only issues async copies; the caller waits (cp_async_wait_all + barrier) before reading.
template <bool kVec, int WP>
__device__ __forceinline__ void load_window(const float* __restrict__ f, int64_t pitch, int R0, int C0, int H, int W,
                                            float* in) {
  if (kVec) {  // W % 4 == 0, 16-byte aligned rows: every float4 is wholly inside or outside
    constexpr int Q = WP / 4;  // float4 per window row
    const int step = blockDim.x, dr = step / Q, dc = step % Q;
    int r = threadIdx.x / Q, c4 = threadIdx.x % Q;  // (r, c4) advanced incrementally
    const float* fb = f + (int64_t)(R0 - 4) * pitch + (C0 - 4);
    for (; r < kMIn;) {
      const int gr = R0 - 4 + r, gc = C0 - 4 + 4 * c4;
      const bool ok = (unsigned)gr < (unsigned)H && (unsigned)gc < (unsigned)W && c4 < kMIn / 4;
      cp_async16(in + r * WP + 4 * c4, ok ? fb + (int64_t)r * pitch + 4 * c4 : f, ok ? 16 : 0);
      c4 += dc;
      r += dr;
      if (c4 >= Q) {
        c4 -= Q;
        ++r;
      }
    }
  } else {
    for (int i = threadIdx.x; i < kMIn * WP; i += blockDim.x) {
      const int r = i / WP, c = i % WP;
      const int gr = R0 - 4 + r, gc = C0 - 4 + c;
      in[r * WP + c] = (gr >= 0 && gr < H && gc >= 0 && gc < W && c < kMIn) ? __ldg(f + (int64_t)gr * pitch + gc) : 0.f;
    }
  }
}

// ---- fp32 denoiser of the IDA step (dct_soft_threshold, denoise.cpp:52-92) ------------------
// The 17 x 17 tiles (8 x 8, stride 4) over the 72 x 72 window are transformed separably on the
// CUDA cores with packed-pair butterflies (dct_pair.cuh), and the separability is used twice:
//   A. row DCT of every (window row, 8-px segment tj): shared by the two tiles that contain that
//      row segment (tiles ti and ti - 1), so each row transform is done once, not twice;
//   B. per tile, column DCT -> soft threshold -> inverse column DCT, summed into S over the two
//      tiles covering each row (even tile rows store, odd tile rows add: a fixed order);
//   C. inverse row DCT of S (linearity: the two tiles' contributions to a row segment are summed
//      before the inverse, halving those transforms), then the two segments covering each pixel
//      are summed and scaled by 1 / weight (denoise.cpp:90), straight into acc.
// Vectors are paired across adjacent segments (tj = 2 tp, 2 tp + 1), so every transform is one
// FFMA2 / FADD2 stream with no transposes. Tiles whose origin is off the image's tile grid get an
// infinite threshold, so they contribute zero (denoise.cpp:57-62).
constexpr int kWP = 76;            // window pitch: 72 + 4 zero columns (A reads 12 px from col 8 tp)
constexpr int kTP = 9;             // segment pairs per row (tj = 17 is a zero dummy)
constexpr int kRP = kTP * 16 + 4;  // R / S row pitch: [tp][v][2] + 4 (148 = 20 mod 32: conflict-free)
#ifndef IDA_MINB
#define IDA_MINB 3
#endif
constexpr int kFThreads = 32 * kTP;  // fused kernel: warp w owns segment pair tp = w through stages A-C

// The denoiser's output x replaces the window in place (same layout), so acc is the window: region
// pixel (0, 0) at kAOff, pitch kWP (76 = 12 mod 32: the block phase's float4 row loads are
// conflict-free per quarter warp).
constexpr int kAOff = 4 * kWP + 4;
struct IdaF32Smem {
  union {
    float in[kMIn * kWP];   // field window (pitch kWP), the TMA destination (128-B aligned)
    float acc[kMIn * kWP];  // then x over the region (at kAOff, pitch kWP) for the block phase
  };
  union {
    float RS[kMIn * kRP];     // stage A output R[y][tp][v][tj parity], overwritten in place by stage B's S
    float stage[kMIn * kRP];  // y / z staging in the block phase
  };
  int meta_cnt[64];
  int meta_off[64];
  double red[4][16];
  unsigned int bad[2];
  double mine[4];
  uint64_t win_bar;          // TMA window load (one phase per CTA)
  unsigned short zslot[256];  // B = 16: rank k's slot in a block's transpose tile, (v, u) -> v * 20 + u
};
static_assert(kFThreads / 32 * 512 <= kMIn * kRP, "staging buffers fit");

__device__ __forceinline__ bool tile_on_grid(int R0, int C0, int H, int W, int ti, int tj) {
  return tj <= 16 && (unsigned)(R0 - 4 + 4 * ti) <= (unsigned)(H - 8) && (unsigned)(C0 - 4 + 4 * tj) <= (unsigned)(W - 8);
}

__device__ __forceinline__ void sts2(float* p, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};\n" ::"r"(smem_u32(p)), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ float2 lds2(const float* p) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(v.x), "=f"(v.y) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ float2 shfl2(float2 v, int src) {
  return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// dct_soft_threshold of the window s.in into s.acc (the 64 x 64 region, pitch kWP at kAOff;
// acc aliases the window, which is dead once every warp is past stage A).
// Warp w owns segment pair tp = w (tj = 2w, 2w + 1) through stages A-C, so the stages are
// ordered by __syncwarp; only stage C's quads shared with the neighbouring pair need the CTA.
// Expects the window's async copies issued; ends with __syncthreads.
// The region's y / z prefixes (one run per block row) into L1 while the denoiser runs: the block
// phase's rank-order accesses to them then hit L1 instead of waiting on L2.
__device__ __forceinline__ void l1_prefetch_region_yz(const IdaParams& P, int img, const IdaF32Smem& s) {
  if (!P.y) return;
  const int t = threadIdx.x;
  const int j = (t >> 5) & 3, line = t & 31;  // warps 0-3 -> block rows 0-3 of y, warps 4-7 of z
  if (t >= 256) return;
  int first = -1, n = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = s.meta_cnt[4 * j + i];
    if (c >= 0) {
      if (first < 0) first = s.meta_off[4 * j + i];
      n += c;
    }
  }
  if (first < 0) return;
  const float* base = ((t >> 7) ? P.z : P.y) + (int64_t)img * P.y_stride + first;
  for (int o = line * 32; o < n; o += 32 * 32)
    asm volatile("prefetch.global.L1 [%0];\n" ::"l"(base + o));
}

// Linearity form of the soft threshold: soft(Y) = Y - clamp(Y, -t, t) (t = 0 at the DC, which
// passes, and for tiles off the image's tile grid, which weigh nothing), and the on-grid tiles
// covering a pixel sum to w p, so
//   dct_soft_threshold(p) = (sum_tiles IDCT(soft(Y))) / w = p - (sum_tiles IDCT(clamp(Y))) / w.
// The clamp is one FMNMX.XORSIGN per coefficient (the soft threshold took two FMNMX and half an
// FADD2), and the transformed corrections are bounded by the threshold, not by the field.
// 1 / (on-grid tile origins covering the 4-px band starting at b) along one axis: 1 or 1/2 (the
// weight is separable, w = w_row w_col, so 1 / w is the product of the two axis factors)
__device__ __forceinline__ float axis_scale(int b, int extent) {
  return (b >= 4 && b <= extent - 8) ? 0.5f : 1.f;
}

__device__ void denoise_region_f32(IdaF32Smem& s, int R0, int C0, int H, int W, float thr) {
  const int lane = threadIdx.x & 31, tp = threadIdx.x >> 5;
  // The forward transforms run on the field centred on a per-region constant cen (the AC
  // coefficients are those of p; the DC is never used, its clamp is 0): smaller magnitudes, less
  // fp32 rounding in every butterfly stage (DAMP's Monte-Carlo divergence differences two
  // denoiser calls and feels that rounding).
  const float cen = 0.25f * (s.in[35 * kWP + 35] + s.in[35 * kWP + 36] + s.in[36 * kWP + 35] + s.in[36 * kWP + 36]);
  const float2 mc = make_float2(-cen, -cen);
  // A: row DCTs of the window rows y = lane + 32 j (lanes along rows: conflict-free)
#pragma unroll 1
  for (int y = lane; y < kMIn; y += 32) {
    const float* src = s.in + y * kWP + 8 * tp;
    const float4 a = *reinterpret_cast<const float4*>(src), b = *reinterpret_cast<const float4*>(src + 4),
                 c = *reinterpret_cast<const float4*>(src + 8);
    float2 x[8] = {make_float2(a.x, b.x), make_float2(a.y, b.y), make_float2(a.z, b.z), make_float2(a.w, b.w),
                   make_float2(b.x, c.x), make_float2(b.y, c.y), make_float2(b.z, c.z), make_float2(b.w, c.w)};
#pragma unroll
    for (int n = 0; n < 8; ++n) x[n] = p_add(x[n], mc);
    float2 Y[8];
    dct8_fwd_pair(x, Y);
    float4* d = reinterpret_cast<float4*>(s.RS + y * kRP + 16 * tp);
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = make_float4(Y[2 * q].x, Y[2 * q].y, Y[2 * q + 1].x, Y[2 * q + 1].y);
  }
  __syncwarp();
  // B: lanes = (coefficient column v, run tq). Run tq walks the tile rows [first, end) = 0..4, 5..8,
  // 9..12, 13..16 top to bottom; per tile: column DCT, clamp, inverse column DCT. The window of 8
  // rows slides by 4 in registers (4 new rows per tile), and a tile's top half plus the bottom half
  // of the tile above (carried in registers) completes those S rows, written in place over R: the
  // rows a store replaces were last read by the same lane. A run's first tile keeps its top half
  // until every run is done: the previous run's last tile still reads those R rows.
  {
    const int v = lane & 7, tq = lane >> 3;
    const bool gc0 = (unsigned)(C0 - 4 + 8 * tp) <= (unsigned)(W - 8);
    const bool gc1 = tp < 8 && (unsigned)(C0 + 8 * tp) <= (unsigned)(W - 8);
    const int t_first = tq == 0 ? 0 : 4 * tq + 1, t_end = 4 * tq + 5;
    float* col = s.RS + 16 * tp + 2 * v;
    float2 x[8], first[4], carry[4];
#pragma unroll
    for (int r = 0; r < 8; ++r) x[r] = lds2(col + (4 * t_first + r) * kRP);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const int ti = t_first + i;
      const bool act = ti < t_end;  // warp-uniform except the 5th tile (run 0 only)
      if (i > 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) x[r] = x[4 + r];
        if (act) {
#pragma unroll
          for (int r = 0; r < 4; ++r) x[4 + r] = lds2(col + (4 * ti + 4 + r) * kRP);
        }
      }
      float2 Y[8], X[8];
      dct8_fwd_pair(x, Y);
      const bool gr = (unsigned)(R0 - 4 + 4 * ti) <= (unsigned)(H - 8);
      const float t0 = gr && gc0 ? thr : 0.f, t1 = gr && gc1 ? thr : 0.f;
      Y[0] = p_clamp(Y[0], v == 0 ? 0.f : t0, v == 0 ? 0.f : t1);  // the DC passes (denoise.cpp:76)
#pragma unroll
      for (int u = 1; u < 8; ++u) Y[u] = p_clamp(Y[u], t0, t1);
      dct8_inv_pair(Y, X);
      if (i == 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) first[r] = X[r];
      } else if (act) {
#pragma unroll
        for (int r = 0; r < 4; ++r) sts2(col + (4 * ti + r) * kRP, p_add(X[r], carry[r]));
      }
      if (act) {
#pragma unroll
        for (int r = 0; r < 4; ++r) carry[r] = X[4 + r];
      }
    }
    __syncwarp();  // every run past its loads
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float2 above = shfl2(carry[r], (lane + 24) & 31);  // the previous run's last tile
      if (tq > 0) sts2(col + (4 * t_first + r) * kRP, p_add(first[r], above));
    }
  }
  __syncthreads();  // stage C writes window quads the neighbouring pairs' stage A read
  // C: inverse row DCTs of S over the region rows yr = lane + 32 j, and x = p - correction / w in
  // place over the window. Output quads (window cols): Q0 = 8tp..+3 (tj0 only), Q1 = 8tp+4..+7
  // (tj0 + tj1, complete), Q2 = 8tp+8..+11 (tj1 only). Q0 of pair tp+1 and Q2 of pair tp are the
  // same quad: Q0 is applied first, Q2 after a barrier (a fixed order).
  float4 q2[2];
  const float fc0 = axis_scale(C0 + 8 * tp - 4, W), fc1 = axis_scale(C0 + 8 * tp, W);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int yr = lane + 32 * j;
    const float4* src = reinterpret_cast<const float4*>(s.RS + (yr + 4) * kRP + 16 * tp);
    float2 y[8], X[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 v = src[q];
      y[2 * q] = make_float2(v.x, v.y);
      y[2 * q + 1] = make_float2(v.z, v.w);
    }
    dct8_inv_pair(y, X);
    float* row = s.in + (yr + 4) * kWP;  // indexed by window column
    const float fr = axis_scale((R0 + yr) & ~3, H);  // weights: on-grid tile origins per axis (1 or 2)
    if (tp >= 1) {
      const float sc = fr * fc0;
      float4* d = reinterpret_cast<float4*>(row + 8 * tp);
      const float4 p = *d;
      *d = make_float4(fmaf(-X[0].x, sc, p.x), fmaf(-X[1].x, sc, p.y), fmaf(-X[2].x, sc, p.z), fmaf(-X[3].x, sc, p.w));
    }
    if (tp <= 7) {
      const float sc = fr * fc1;
      float4* d = reinterpret_cast<float4*>(row + 8 * tp + 4);
      const float4 p = *d;
      *d = make_float4(fmaf(-(X[4].x + X[0].y), sc, p.x), fmaf(-(X[5].x + X[1].y), sc, p.y),
                       fmaf(-(X[6].x + X[2].y), sc, p.z), fmaf(-(X[7].x + X[3].y), sc, p.w));
    }
    q2[j] = make_float4(X[4].y, X[5].y, X[6].y, X[7].y);
  }
  __syncthreads();
  if (tp <= 7) {
    const float fc2 = axis_scale(C0 + 8 * tp + 4, W);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int yr = lane + 32 * j;
      const float sc = axis_scale((R0 + yr) & ~3, H) * fc2;
      float4* d = reinterpret_cast<float4*>(s.in + (yr + 4) * kWP + 8 * tp + 8);
      const float4 a = *d;
      *d = make_float4(fmaf(-q2[j].x, sc, a.x), fmaf(-q2[j].y, sc, a.y), fmaf(-q2[j].z, sc, a.z),
                       fmaf(-q2[j].w, sc, a.w));
    }
  }
  __syncthreads();
}

struct IdaLaneSums {
  double z = 0.0, sse = 0.0, y = 0.0;
  int cnt = 0;
  unsigned int badx = ~0u, badz = ~0u;  // first offending index (x: index << 1 | kind), < 2^32 per image
};

// check_finite on x (recon.cpp:56-65) and the trace SSE for one float2 of x at (gr, gc).
__device__ __forceinline__ void x_checks(const IdaParams& P, int img, int gr, int gc, float2 x, IdaLaneSums& S) {
  const float xs[2] = {x.x, x.y};
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const float xv = xs[e];
    if (!isfinite(xv) || fabsf(xv) > 1e6f) {
      const unsigned long long gi =
          ((unsigned long long)((int64_t)gr * P.Wc + gc + e) << 1) | (isfinite(xv) ? 1ull : 0ull);
      const unsigned g32 = (unsigned)min(gi, 0xfffffffeull) | (unsigned)(gi & 1ull);  // kind bit kept
      S.badx = g32 < S.badx ? g32 : S.badx;
    }
  }
  if (P.ref) {
    const uint8_t* rp = P.ref + (int64_t)img * P.ref_stride + (int64_t)gr * P.ref_pitch + gc;
    const double d0 = (double)rp[0] - (double)x.x, d1 = (double)rp[1] - (double)x.y;
    S.sse += d0 * d0 + d1 * d1;
  }
}

__device__ __forceinline__ void store_out(const IdaParams& P, int img, int gr, int gc, float2 x, float2 az) {
  if (P.pseudo_out) {
    float2 o = make_float2(x.x + az.x, x.y + az.y);
    *reinterpret_cast<float2*>(P.pseudo_out + (int64_t)img * P.Hc * P.Wc + (int64_t)gr * P.Wc + gc) = o;
  } else {  // last iteration: clamp (recon.cpp:255-257), or the raw state x for damp_step
    float* d = P.x_out + (int64_t)img * P.out_stride + (int64_t)gr * P.out_pitch + gc;
    const float o0 = P.clamp_out ? fminf(fmaxf(x.x, 0.f), 255.f) : x.x;
    const float o1 = P.clamp_out ? fminf(fmaxf(x.y, 0.f), 255.f) : x.y;
    if (((P.out_pitch | P.out_stride) & 1) == 0) {
      *reinterpret_cast<float2*>(d) = make_float2(o0, o1);
    } else {
      d[0] = o0;
      d[1] = o1;
    }
  }
}

// Issue the async staging of cnt values of y (and z) of one block into smem (per warp).
__device__ __forceinline__ void stage_yz_async(const IdaParams& P, int64_t off, int cnt, float* yb, float* zb,
                                              bool need_z) {
  for (int k = threadIdx.x & 31; k < cnt; k += 32) {
    cp_async4(yb + k, P.y + off + k);
    if (need_z) cp_async4(zb + k, P.z + off + k);
  }
}
// Wait for the warp's staging; ||y||^2 for the init step (recon.cpp:128) from the staged copy.
__device__ __forceinline__ void stage_yz_wait(const IdaParams& P, int cnt, const float* yb, IdaLaneSums& S) {
  cp_async_wait_all();
  __syncwarp();
  if (P.is_init)
    for (int k = threadIdx.x & 31; k < cnt; k += 32) S.y += (double)yb[k] * (double)yb[k];
}

// The region's sensing blocks (kMR / B)^2, row-major: count (-1 outside the grid) and offset.
template <int B, class Sm>
__device__ __forceinline__ void fetch_meta(const IdaParams& P, int img, int R0, int C0, Sm& s) {
  constexpr int PB = kMR / B;
  for (int bi = threadIdx.x; bi < PB * PB; bi += blockDim.x) {
    const int gbr = R0 / B + bi / PB, gbc = C0 / B + bi % PB;
    int cnt = -1, off = 0;
    if (gbr < P.rows && gbc < P.cols) {
      const int64_t bidx = (int64_t)img * P.rows * P.cols + (int64_t)gbr * P.cols + gbc;
      cnt = P.counts[bidx];
      off = P.offsets[bidx];
    }
    s.meta_cnt[bi] = cnt;
    s.meta_off[bi] = off;
  }
}

__device__ __forceinline__ float z_update(const IdaParams& P, float yv, float ax, float zo, unsigned long long gi,
                                          IdaLaneSums& S, float onsager) {
  const float zn = (yv - ax) + onsager * zo;  // finish_step (recon.cpp:86-88)
  S.z += (double)zn * (double)zn;
  if (!isfinite(zn)) S.badz = (unsigned)gi < S.badz ? (unsigned)gi : S.badz;
  return zn;
}



// Power-of-two rescale keeping the fp16 hi/lo operand split of the B = 8 tensor-core transforms in
// range (as decode16_kernel): when any of the warp's values exceeds kIdaSafeMax, scale them all by
// 2^-e (exact) and return 2^e for the result. Warp-uniform; the common case is one compare per value.
constexpr float kIdaSafeMax = 8192.f;
__device__ __forceinline__ float fp16_range_scale(float (&v)[4]) {
  bool big = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) big |= !(fabsf(v[i]) <= kIdaSafeMax);
  if (!__any_sync(0xffffffffu, big)) return 1.f;
  float mx = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) mx = fmaxf(mx, fabsf(v[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (!isfinite(mx) || mx <= kIdaSafeMax) return 1.f;  // non-finite: check_finite reports it
  int e;
  frexpf(mx / kIdaSafeMax, &e);
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = ldexpf(v[i], -e);
  return ldexpf(1.f, e);
}

// ---- B = 16 block phase on the CUDA cores (recon.cpp:81-93, 75-79; operators.cpp:50-76) ------
// Thread (b, r) / (b, v) of the region's 16 sensing blocks (threads 0..255):
//   1. rows:    T[r][.] = DCT16(x[r][.])                 check_finite, trace SSE, last step: x out
//   2. columns: Y[.][v] = DCT16(T[.][v]); in the zigzag prefix z <- (y - Y) + z / D_F and
//               W = Y + z, else W = Y;                    V[.][v] = IDCT16(W[.][v])
//   3. rows:    pseudo[r][.] = IDCT16(V[r][.])  =  x + A* z  (IDCT16 o DCT16 = identity: the full
//               transform of x is already at hand, so pseudo needs one inverse, not x + a second one)
// The transposes go through the window buffer (x is dead once every thread holds its row). y and z
// are read where they lie (a block's prefix is one short run, so the column threads' rank-order
// accesses stay in L1) and z is written back in place.
constexpr int kTB = 336;  // per-block transpose tile: 16 rows x pitch 20 (+16: conflict-free between blocks)
static_assert(16 * kTB <= kMIn * kRP, "transpose tiles fit in RS");

// check_finite (recon.cpp:56-65) over a thread's 16 x values: the common case is one compare per
// value; the first offending index (x-major, kind bit as in x_checks) only on the rare path.
__device__ __forceinline__ void row_checks(const IdaParams& P, int img, int gr, int gc, const float (&x)[16],
                                           IdaLaneSums& S) {
  bool bad = false;
#pragma unroll
  for (int c = 0; c < 16; ++c) bad |= !(fabsf(x[c]) <= 1e6f);
  if (bad) {
#pragma unroll
    for (int c = 0; c < 16; c += 2) x_checks(P, img, gr, gc + c, make_float2(x[c], x[c + 1]), S);
  } else if (P.ref) {
    const uint8_t* rp = P.ref + (int64_t)img * P.ref_stride + (int64_t)gr * P.ref_pitch + gc;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const double d = (double)rp[c] - (double)x[c];
      S.sse += d * d;
    }
  }
}

__device__ __forceinline__ void load_row16(const float* p, float (&v)[16]) {
  const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 a = q[i];
    v[4 * i] = a.x;
    v[4 * i + 1] = a.y;
    v[4 * i + 2] = a.z;
    v[4 * i + 3] = a.w;
  }
}

template <class Sm>
__device__ void block_phase16_f32(const IdaParams& P, int img, int R0, int C0, Sm& s, IdaLaneSums& S) {
  const int t = threadIdx.x;
  const int b = (t >> 4) & 15, lr = t & 15;  // block of the region (row-major) and row / column
  const int br = b >> 2, bc = b & 3;
  const int cnt = s.meta_cnt[b];
  const bool valid = t < 256 && cnt >= 0;
  const bool last = P.pseudo_out == nullptr;
  const float ons = P.onsager_img ? (float)P.onsager_img[img] : P.onsager;
  const int gr = R0 + 16 * br + lr, gc = C0 + 16 * bc;  // this thread's image row (stages 1, 3)
  // 1. rows of x. Each block is centred on its centre pixel cb before the transforms (the transform
  // of x - cb is that of x less 16 cb at the DC; pseudo gets cb back): smaller magnitudes, less
  // fp32 rounding in every butterfly stage.
  float T[16], cb = 0.f;
  if (valid) {
    float xr[16];
    load_row16(s.acc + kAOff + (16 * br + lr) * kWP + 16 * bc, xr);
    cb = s.acc[kAOff + (16 * br + 8) * kWP + 16 * bc + 8];
    row_checks(P, img, gr, gc, xr, S);
    if (last) {  // the estimate itself (recon.cpp:255-257 clamp on reconstruct's final step)
#pragma unroll
      for (int c = 0; c < 16; c += 2) store_out(P, img, gr, gc + c, make_float2(xr[c], xr[c + 1]), make_float2(0.f, 0.f));
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) xr[c] -= cb;
    abcs_gen::dct16_fwd(xr, T);
  }
  // Warp w owns blocks 2w and 2w + 1 through all stages, and each block's transpose tile lives in
  // RS (free after the denoiser): the stages synchronise per warp, not per CTA.
  float* tb = s.RS + b * kTB;
  if (valid) {
#pragma unroll
    for (int v = 0; v < 16; ++v) tb[v * 20 + lr] = T[v];
  }
  __syncwarp();
  // 2. columns: v = lr. The column DCT lands in the tile as Y[u] at (row v, col u); the z update
  // then walks the warp's two blocks' prefixes in zigzag order (they are consecutive in the
  // payload: coalesced y / z loads, all in flight at once, and coalesced z stores), reading Y at
  // each rank's (u, v) and leaving W = Y + z in its place; the column threads reload W.
  float Y[16];
  if (valid) {
    float Tc[16];
    load_row16(tb + lr * 20, Tc);
    abcs_gen::dct16_fwd(Tc, Y);
    if (lr == 0) Y[0] += 16.f * cb;  // the tile holds the true DC: the centred one lacks 16 cb (exact)
  }
  __syncwarp();  // every lane holds its column: the tile takes Y
  if (valid) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<float4*>(tb + lr * 20 + 4 * q) = make_float4(Y[4 * q], Y[4 * q + 1], Y[4 * q + 2], Y[4 * q + 3]);
  }
  __syncwarp();
  if (t < 256) {
    const int lane = t & 31, b0 = b & ~1;
    const int c0 = max(s.meta_cnt[b0], 0), c1 = max(s.meta_cnt[b0 + 1], 0), kw = c0 + c1;
    const int64_t pb = (int64_t)img * P.y_stride + s.meta_off[b0];  // the pair's run in y / z
    const float* yrun = P.y + pb;
    float* zrun = P.z + pb;
    float* tile0 = s.RS + b0 * kTB;
    float zsq = 0.f, ysq = 0.f;
    bool bad = false;
    // NS elements per lane in flight per round; NS from the pair's run length (warp-uniform), so
    // short runs (cfg4: ~130) do not pay for 8 predicated slots per lane
    auto rounds = [&](auto ns) {
      constexpr int NS = decltype(ns)::value;
#pragma unroll 1
      for (int e0 = lane; e0 < kw; e0 += 32 * NS) {
        float yv[NS], zo[NS];
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const int e = e0 + 32 * i;
          yv[i] = e < kw ? __ldg(yrun + e) : 0.f;
          zo[i] = (e < kw && !P.is_init) ? zrun[e] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const int e = e0 + 32 * i;
          if (e < kw) {
            const bool q = e >= c0;
            float* slot = tile0 + (q ? kTB : 0) + s.zslot[q ? e - c0 : e];
            const float yc = *slot;
            const float zn = (yv[i] - yc) + ons * zo[i];  // finish_step (recon.cpp:86-88)
            zrun[e] = zn;
            *slot = yc + zn;  // W = Y + z
            zsq = fmaf(zn, zn, zsq);
            ysq = fmaf(yv[i], yv[i], ysq);
            bad |= !(fabsf(zn) <= FLT_MAX);
          }
        }
      }
    };
    if (kw <= 128) rounds(std::integral_constant<int, 4>{});
    else if (kw <= 160) rounds(std::integral_constant<int, 5>{});
    else rounds(std::integral_constant<int, 8>{});
    S.z += (double)zsq;
    if (P.is_init) S.y += (double)ysq;  // ||y||^2 (recon.cpp:128)
    if (bad) {  // rare: the first non-finite residual of this lane's elements (its own stores)
      for (int e = lane; e < kw; e += 32)
        if (!isfinite(zrun[e])) {
          const unsigned int gi = (unsigned)(s.meta_off[b0] + e);
          S.badz = gi < S.badz ? gi : S.badz;
          break;
        }
    }
    if ((t & 15) == 0 && cnt >= 0) S.cnt += cnt;
  }
  __syncwarp();
  if (valid) {
    load_row16(tb + lr * 20, Y);  // W of column lr
    if (lr == 0) Y[0] -= 16.f * cb;  // centred again for the inverse
  }
  if (last) return;
  __syncwarp();  // all column loads of the warp's tiles done: they take V
  if (valid) {
    float V[16];
    abcs_gen::dct16_inv(Y, V);
#pragma unroll
    for (int r = 0; r < 16; ++r) tb[r * 20 + lr] = V[r];
  }
  __syncwarp();
  // 3. rows: pseudo = IDCT16 of row r of V
  if (valid) {
    float Vr[16], O[16];
    load_row16(tb + lr * 20, Vr);
    abcs_gen::dct16_inv(Vr, O);
    float4* dst = reinterpret_cast<float4*>(P.pseudo_out + (int64_t)img * P.Hc * P.Wc + (int64_t)gr * P.Wc + gc);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = make_float4(O[4 * q] + cb, O[4 * q + 1] + cb, O[4 * q + 2] + cb, O[4 * q + 3] + cb);
  }
}

// init, warm start: acc <- x0 = A* y (recon.cpp:119-131), the inverse of each block's y prefix
// (columns then rows through the transpose tiles). Called before block_phase16_f32.
template <class Sm>
__device__ void init_x16_f32(const IdaParams& P, int img, int R0, int C0, Sm& s, float& ysq, float (&xo)[16]) {
  const int t = threadIdx.x;
  const int b = (t >> 4) & 15, lr = t & 15, br = b >> 2, bc = b & 3;
  const int cnt = s.meta_cnt[b];
  const bool valid = t < 256 && cnt >= 0;
  float* tb = s.RS + b * kTB;  // per-block transpose tile; warp w owns blocks 2w, 2w + 1
  float cb = 0.f;
  // embed each block's y prefix: zero the tile, then the warp scatters its two blocks' run (one
  // coalesced read) to each rank's (u, v) slot (tile row v, column u)
  if (t < 256) {
#pragma unroll
    for (int q = 0; q < 4; ++q) *reinterpret_cast<float4*>(tb + lr * 20 + 4 * q) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncwarp();
  if (t < 256) {  // the pair's payload run: up to 8 loads per lane in flight; z0 = 0 and ||y||^2 on the way
    const int lane = t & 31, b0 = b & ~1;
    const int c0 = max(s.meta_cnt[b0], 0), kw = c0 + max(s.meta_cnt[b0 + 1], 0);
    const int64_t pb = (int64_t)img * P.y_stride + s.meta_off[b0];
#pragma unroll 1
    for (int e0 = 0; e0 < kw; e0 += 256) {
      float yv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = e0 + lane + 32 * i;
        yv[i] = e < kw ? __ldg(P.y + pb + e) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = e0 + lane + 32 * i;
        if (e < kw) {
          const int q = e < c0 ? 0 : 1, k = e - (q ? c0 : 0);
          s.RS[(b0 + q) * kTB + s.zslot[k]] = yv[i];
          P.z[pb + e] = 0.f;
          ysq = fmaf(yv[i], yv[i], ysq);
        }
      }
    }
  }
  __syncwarp();
  float V[16];
  if (valid) {
    float Wc[16];
    load_row16(tb + lr * 20, Wc);
    if (lr == 0) {  // centre on the block mean y00 / 16: out of the transform, added back after
      cb = Wc[0] * 0.0625f;
      Wc[0] = 0.f;
    }
    abcs_gen::dct16_inv(Wc, V);
  }
  __syncwarp();  // every column loaded: the tile takes V
  if (valid) {
#pragma unroll
    for (int r = 0; r < 16; ++r) tb[r * 20 + lr] = V[r];
  }
  cb = __shfl_sync(0xffffffffu, cb, threadIdx.x & 16);  // from the block's column-0 thread
  __syncwarp();
  float O[16];
  if (valid) {
    float Vr[16];
    load_row16(tb + lr * 20, Vr);
    abcs_gen::dct16_inv(Vr, O);
  }
#pragma unroll
  for (int c = 0; c < 16; ++c) xo[c] = O[c] + cb;  // row lr of block b: the thread that checks / stores it
}

// Warm start, the rest of init_state (recon.cpp:119-131): x0 = A* y is in acc; z0 = y - A x0 is 0
// (the prefix of DCT(IDCT(embed y)) is y: the reference's own z0 is rounding residue, ~1e-13),
// so pseudo0 = x0 + A* z0 = x0 and the block phase's transforms are skipped. sigma0 = ||y|| / sqrt(M)
// needs ||y||^2, summed over each warp's payload run; the trace's PSNR of x0 needs the SSE.
template <class Sm>
__device__ void init_finish16(const IdaParams& P, int img, int R0, int C0, Sm& s, IdaLaneSums& S, float ysq,
                              const float (&xr)[16]) {
  const int t = threadIdx.x;
  const int b = (t >> 4) & 15, lr = t & 15, br = b >> 2, bc = b & 3;
  const int cnt = s.meta_cnt[b];
  if (t < 256 && cnt >= 0) {
    const int gr = R0 + 16 * br + lr, gc = C0 + 16 * bc;
    row_checks(P, img, gr, gc, xr, S);
    if (P.pseudo_out) {  // pseudo0 = x0 (internal buffer: Wc % 16 == 0, 16-B aligned rows)
      float4* dst = reinterpret_cast<float4*>(P.pseudo_out + (int64_t)img * P.Hc * P.Wc + (int64_t)gr * P.Wc + gc);
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = make_float4(xr[4 * q], xr[4 * q + 1], xr[4 * q + 2], xr[4 * q + 3]);
    } else {
#pragma unroll
      for (int c = 0; c < 16; c += 2) store_out(P, img, gr, gc + c, make_float2(xr[c], xr[c + 1]), make_float2(0.f, 0.f));
    }
    if (lr == 0) S.cnt += cnt;
  }
  if (t < 256) S.y += (double)ysq;  // ||y||^2 (recon.cpp:128), summed while init_x16_f32 embedded y
}

// ---- B = 8: two horizontally adjacent sensing blocks per warp step ------------------------
template <class Sm>
__device__ void init_x8(const IdaParams& P, int img, int R0, int C0, Sm& s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  Frag8 f;
  load_frag8(f);
  uint32_t rank[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) rank[e] = zigzag_rank_dev<8>()[(2 * t + e) * 8 + g];  // Y^T[g][2t+e] = Y[2t+e][g]
  float* yb = s.stage + warp * 512;
  for (int pi = warp; pi < 32; pi += (int)(blockDim.x >> 5)) {
    const int br = pi / 4, bc = 2 * (pi % 4);
    const int gbr = R0 / 8 + br;
    int cnt[2] = {0, 0};
    int64_t off[2] = {0, 0};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int gbc = C0 / 8 + bc + q;
      if (gbr < P.rows && gbc < P.cols) {
        const int64_t bidx = (int64_t)img * P.rows * P.cols + (int64_t)gbr * P.cols + gbc;
        cnt[q] = P.counts[bidx];
        off[q] = (int64_t)img * P.y_stride + P.offsets[bidx];
      }
    }
    for (int k = lane; k < cnt[0]; k += 32) yb[k] = __ldg(P.y + off[0] + k);
    for (int k = lane; k < cnt[1]; k += 32) yb[64 + k] = __ldg(P.y + off[1] + k);
    __syncwarp();
    float Yt[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = i >> 1, r = (int)rank[i & 1];
      Yt[i] = r < cnt[q] ? yb[64 * q + r] : 0.f;
    }
    float X[4];
    const float ysc = fp16_range_scale(Yt);
    dct8x2_inv_from_yt(f, Yt, X);
#pragma unroll
    for (int i = 0; i < 4; ++i) X[i] *= ysc;
    const int lr = 8 * br + g, lc = 8 * bc + 2 * t;
    *reinterpret_cast<float2*>(s.acc + kAOff + lr * kWP + lc) = make_float2(X[0], X[1]);
    *reinterpret_cast<float2*>(s.acc + kAOff + lr * kWP + lc + 8) = make_float2(X[2], X[3]);
    __syncwarp();
  }
}

template <class Sm>
__device__ void block_phase8(const IdaParams& P, int img, int R0, int C0, Sm& s, IdaLaneSums& S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float ons = P.onsager_img ? (float)P.onsager_img[img] : P.onsager;
  Frag8 f;
  load_frag8(f);
  uint32_t rank[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) rank[e] = zigzag_rank_dev<8>()[(2 * t + e) * 8 + g];
  float* yb = s.stage + warp * 512;  // [q][64] y, then [q][64] z at +128
  float* zb = yb + 128;
  const bool last = P.pseudo_out == nullptr;
  for (int pi = warp; pi < 32; pi += (int)(blockDim.x >> 5)) {
    const int br = pi / 4, bc = 2 * (pi % 4);
    const int bi0 = br * 8 + bc;
    if (s.meta_cnt[bi0] < 0) continue;  // outside the block grid (warp-uniform)
    const bool has1 = s.meta_cnt[bi0 + 1] >= 0;
    const int cnt[2] = {s.meta_cnt[bi0], has1 ? s.meta_cnt[bi0 + 1] : 0};
    const int32_t boff[2] = {s.meta_off[bi0], has1 ? s.meta_off[bi0 + 1] : 0};
    const int64_t ibase = (int64_t)img * P.y_stride;
    stage_yz_async(P, ibase + boff[0], cnt[0], yb, zb, !P.is_init);
    stage_yz_async(P, ibase + boff[1], cnt[1], yb + 64, zb + 64, !P.is_init);
    if (lane == 0) S.cnt += cnt[0] + cnt[1];
    const int lr = 8 * br + g, lc = 8 * bc + 2 * t;
    const float2 x0 = *reinterpret_cast<const float2*>(s.acc + kAOff + lr * kWP + lc);
    const float2 x1 = *reinterpret_cast<const float2*>(s.acc + kAOff + lr * kWP + lc + 8);
    float Yt[4], xs[4] = {x0.x, x0.y, x1.x, x1.y};
    const float xsc = fp16_range_scale(xs);
    dct8x2_fwdT(f, make_float2(xs[0], xs[1]), make_float2(xs[2], xs[3]), Yt);
#pragma unroll
    for (int i = 0; i < 4; ++i) Yt[i] *= xsc;
    cp_async_wait_all();
    __syncwarp();
    if (P.is_init)  // ||y||^2 (recon.cpp:128), block 0 then block 1 as staged
      for (int q = 0; q < 2; ++q)
        for (int k = lane; k < cnt[q]; k += 32) S.y += (double)yb[64 * q + k] * (double)yb[64 * q + k];
    float Zm[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = i >> 1, r = (int)rank[i & 1];
      float zn = 0.f;
      if (r < cnt[q]) {
        zn = z_update(P, yb[64 * q + r], Yt[i], P.is_init ? 0.f : zb[64 * q + r], (unsigned long long)(boff[q] + r), S,
                      ons);
        zb[64 * q + r] = zn;
      }
      Zm[i] = zn;
    }
    __syncwarp();
    for (int k = lane; k < cnt[0]; k += 32) P.z[ibase + boff[0] + k] = zb[k];
    for (int k = lane; k < cnt[1]; k += 32) P.z[ibase + boff[1] + k] = zb[64 + k];
    float Az[4] = {0.f, 0.f, 0.f, 0.f};
    if (!last) {
      const float zsc = fp16_range_scale(Zm);
      dct8x2_inv_from_yt(f, Zm, Az);
#pragma unroll
      for (int i = 0; i < 4; ++i) Az[i] *= zsc;
    }
    x_checks(P, img, R0 + lr, C0 + lc, x0, S);
    store_out(P, img, R0 + lr, C0 + lc, x0, make_float2(Az[0], Az[1]));
    if (has1) {
      x_checks(P, img, R0 + lr, C0 + lc + 8, x1, S);
      store_out(P, img, R0 + lr, C0 + lc + 8, x1, make_float2(Az[2], Az[3]));
    }
    __syncwarp();
  }
}

// CTA reduction of the lane sums -> mine[4] (+ bad indices) and the per-image fold.
template <class Sm>
__device__ void reduce_and_finish(const IdaParams& P, int img, int region, Sm& s, IdaLaneSums& S) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    s.bad[0] = ~0u;
    s.bad[1] = ~0u;
  }
  const bool has_sse = P.ref != nullptr, has_y = P.is_init != 0;  // otherwise those sums are 0
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    S.z += __shfl_xor_sync(0xffffffffu, S.z, o);
    if (has_sse) S.sse += __shfl_xor_sync(0xffffffffu, S.sse, o);
    if (has_y) S.y += __shfl_xor_sync(0xffffffffu, S.y, o);
    S.cnt += __shfl_xor_sync(0xffffffffu, S.cnt, o);
  }
  __syncthreads();
  if ((tid & 31) == 0) {
    s.red[0][tid >> 5] = S.z;
    s.red[1][tid >> 5] = S.sse;
    s.red[2][tid >> 5] = S.y;
    s.red[3][tid >> 5] = (double)S.cnt;
  }
  if (S.badx != ~0u) atomicMin(&s.bad[0], S.badx);
  if (S.badz != ~0u) atomicMin(&s.bad[1], S.badz);
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < 4; ++q) {
      double a = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += s.red[q][w];
      s.mine[q] = a;
    }
    if (s.bad[0] != ~0u) atomicMin(P.badx + img, (unsigned long long)s.bad[0]);
    if (s.bad[1] != ~0u) atomicMin(P.badz + img, (unsigned long long)s.bad[1]);
  }
  finish_image(P, img, region, s.mine);
}

template <int B>
__global__ void __launch_bounds__(kFThreads, IDA_MINB) ida_mma_kernel(IdaParams P, const __grid_constant__ CUtensorMap win_map) {
  extern __shared__ __align__(128) unsigned char ida_smem_raw[];
  IdaF32Smem& s = *reinterpret_cast<IdaF32Smem*>(ida_smem_raw + ((128 - (smem_u32(ida_smem_raw) & 127)) & 127));
  const int img = blockIdx.y, region = blockIdx.x;
  const int R0 = (region / P.regions_x) * kMR, C0 = (region % P.regions_x) * kMR;
  const bool denoise = !P.is_init && !P.x_in;
  if (denoise && threadIdx.x == 0)  // window first: its latency overlaps the metadata set-up
    tma_window(s.in, &win_map, C0 - 4, R0 - 4, img, &s.win_bar);
  const double sigma = denoise ? P.sigma_in[img] : 0.0;
  fetch_meta<B>(P, img, R0, C0, s);  // visible to the block phase after the next barrier
  if (B == 16 && threadIdx.x < 256) {  // rank k's (u, v) = f / 16, f % 16 -> tile slot v * 20 + u
    const int f = zigzag_dev<16>()[threadIdx.x];
    s.zslot[threadIdx.x] = (unsigned short)((f & 15) * 20 + (f >> 4));
  }
  if (P.is_init && P.warm) __syncthreads();  // the warm start reads the region's metadata right away
  if (P.is_init) {
    if (!P.warm) {  // cold start: x0 = 0, so z0 = y (recon.cpp:119-131)
      for (int i = threadIdx.x; i < kMIn * kWP / 4; i += blockDim.x)
        reinterpret_cast<float4*>(s.acc)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {  // B = 16 warm starts run ida_init16_kernel
      init_x8(P, img, R0, C0, s);
    }
    __syncthreads();
  } else if (P.x_in) {  // x from another denoiser: load the region
    const float* xs = P.x_in + (int64_t)img * P.Hc * P.Wc;
    for (int i = threadIdx.x; i < kMR * kMR / 4; i += blockDim.x) {
      const int r = i / (kMR / 4), c = 4 * (i % (kMR / 4));
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (R0 + r < P.Hc && C0 + c < P.Wc) v = __ldg(reinterpret_cast<const float4*>(xs + (int64_t)(R0 + r) * P.Wc + C0 + c));
      *reinterpret_cast<float4*>(s.acc + kAOff + r * kWP + c) = v;
    }
    __syncthreads();
  } else {
    __syncthreads();  // the window's mbarrier is initialised (thread 0) before anyone waits on it
    l1_prefetch_region_yz(P, img, s);
    tma_window_wait(&s.win_bar);
    denoise_region_f32(s, R0, C0, P.Hc, P.Wc, (float)(P.k * sigma));
  }
  IdaLaneSums S;
  if (B == 16) block_phase16_f32(P, img, R0, C0, s, S);
  else block_phase8(P, img, R0, C0, s, S);
  reduce_and_finish(P, img, region, s, S);
}

// Warm-start init for B = 16 (init_state, recon.cpp:119-131): x0 = A* y per sensing block, straight
// from the transpose tiles to pseudo0 (or x) in registers. No window and no denoiser, so only the
// tiles and the metadata live in shared memory: 8 warps and ~24 KB per CTA, several CTAs per SM.
struct IdaInitSmem {
  float RS[16 * kTB];  // the region's 16 per-block transpose tiles
  int meta_cnt[64];
  int meta_off[64];
  double red[4][16];
  unsigned int bad[2];
  double mine[4];
  unsigned short zslot[256];
};

__global__ void __launch_bounds__(256, 6) ida_init16_kernel(IdaParams P) {
  __shared__ __align__(16) IdaInitSmem s;
  const int img = blockIdx.y, region = blockIdx.x;
  const int R0 = (region / P.regions_x) * kMR, C0 = (region % P.regions_x) * kMR;
  fetch_meta<16>(P, img, R0, C0, s);
  {
    const int f = zigzag_dev<16>()[threadIdx.x];
    s.zslot[threadIdx.x] = (unsigned short)((f & 15) * 20 + (f >> 4));
  }
  __syncthreads();
  float ysq = 0.f, xr[16];
  init_x16_f32(P, img, R0, C0, s, ysq, xr);
  IdaLaneSums S;
  init_finish16(P, img, R0, C0, s, S, ysq, xr);
  reduce_and_finish(P, img, region, s, S);
}

// Standalone denoise(dct_threshold) on f32 fields (denoise.cpp:96-109): the IDA step's fp32
// denoiser (denoise_region_f32) over 64 x 64 regions, the window by cp.async (any field stride).
template <bool kVec>
__global__ void __launch_bounds__(kFThreads, 3)
denoise_f32_kernel(const float* __restrict__ field, int H, int W, int64_t stride, const double* __restrict__ thr,
                   float* __restrict__ out, int regions_x) {
  extern __shared__ __align__(128) unsigned char den_smem_raw[];
  IdaF32Smem& s = *reinterpret_cast<IdaF32Smem*>(den_smem_raw + ((128 - (smem_u32(den_smem_raw) & 127)) & 127));
  const int img = blockIdx.y, region = blockIdx.x;
  const int R0 = (region / regions_x) * kMR, C0 = (region % regions_x) * kMR;
  load_window<kVec, kWP>(field + (int64_t)img * stride, W, R0, C0, H, W, s.in);
  cp_async_wait_all();
  __syncthreads();
  denoise_region_f32(s, R0, C0, H, W, (float)thr[img]);
  for (int i = threadIdx.x; i < kMR * kMR; i += blockDim.x) {
    const int r = i / kMR, c = i % kMR;
    if (R0 + r < H && C0 + c < W) out[(int64_t)img * stride + (int64_t)(R0 + r) * W + C0 + c] = s.acc[kAOff + r * kWP + c];
  }
}

int launch_denoise(Ctx* ctx, const float* field, int32_t h, int32_t w, int64_t stride, int32_t n,
                   const double* thresholds_dev, float* out, cudaStream_t s) {
  const int rx = (w + kMR - 1) / kMR, ry = (h + kMR - 1) / kMR;
  const bool vec = (w % 4 == 0) && (stride % 4 == 0) && (reinterpret_cast<uintptr_t>(field) % 16 == 0);
  const int bytes = (int)sizeof(IdaF32Smem) + 128;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(denoise_f32_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(denoise_f32_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    attr = true;
  }
  for (int done = 0; done < n;) {
    const int cnt = std::min(n - done, 65535);
    const dim3 grid(rx * ry, cnt);
    const int kt = ktimer_begin(ctx, s, "denoise");
    if (vec)
      denoise_f32_kernel<true><<<grid, kFThreads, bytes, s>>>(field + (int64_t)done * stride, h, w, stride,
                                                               thresholds_dev + done, out + (int64_t)done * stride, rx);
    else
      denoise_f32_kernel<false><<<grid, kFThreads, bytes, s>>>(field + (int64_t)done * stride, h, w, stride,
                                                                thresholds_dev + done, out + (int64_t)done * stride, rx);
    ktimer_end(ctx, s, kt);
    ctx->launches++;
    done += cnt;
  }
  return cuda_status(cudaGetLastError(), "denoise launch");
}

int ida_mma_region() { return kMR; }

// 3-D tiled tensor map over the pseudo field (Wc, Hc, n) with the window box (kWP x kMIn x 1).
static int encode_window_map(CUtensorMap* tm, const float* field, int Wc, int Hc, int n) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode)
      return set_error(ABCS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  }
  const cuuint64_t dims[3] = {(cuuint64_t)Wc, (cuuint64_t)Hc, (cuuint64_t)n};
  const cuuint64_t strides[2] = {(cuuint64_t)Wc * 4, (cuuint64_t)Wc * Hc * 4};
  const cuuint32_t box[3] = {(cuuint32_t)kWP, (cuuint32_t)kMIn, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(field), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? ABCS_OK : set_error(ABCS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
}

template <int B>
static void launch_ida_b(const IdaParams& P, dim3 grid, cudaStream_t s) {
  static bool attr = false;  // > 48 KB of dynamic shared memory: opt in once per instantiation
  const int bytes = (int)sizeof(IdaF32Smem) + 128;  // + alignment slack (TMA destination: 128 B)
  if (!attr) {
    cudaFuncSetAttribute(ida_mma_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    attr = true;
  }
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  if (B == 16 && P.is_init && P.warm) {
    ida_init16_kernel<<<grid, 256, 0, s>>>(P);
    return;
  }
  if (!P.is_init && !P.x_in && P.pseudo_in && encode_window_map(&tm, P.pseudo_in, P.Wc, P.Hc, P.n) != ABCS_OK) return;
  ida_mma_kernel<B><<<grid, kFThreads, bytes, s>>>(P, tm);
}

void launch_ida_mma_kernel(int block, const IdaParams& P, dim3 grid, cudaStream_t s) {
  // pseudo buffers are internal (256-B aligned, Wc % 8 == 0): always the vector window
  if (block == 16) launch_ida_b<16>(P, grid, s);
  else launch_ida_b<8>(P, grid, s);
}


}  // namespace abcs_b200
