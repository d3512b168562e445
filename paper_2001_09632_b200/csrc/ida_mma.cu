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

#include "common.cuh"
#include "ida_common.cuh"
#include "internal.h"
#include "mma_dct.cuh"

namespace abcs_b200 {

constexpr int kMThreads = 256;
constexpr int kMWarps = kMThreads / 32;
constexpr int kMR = 64;          // output region side
constexpr int kMIn = kMR + 8;    // 72: region + 4-px halo each side
constexpr int kMP = 72;          // smem row pitch (floats): 72 = 8 mod 32 -> conflict-free float2 fragments

struct IdaMmaSmem {
  float in[kMIn * kMP];   // field window; reused as per-warp y/z staging in the block phase
  float acc[kMIn * kMP];  // denoiser accumulator over the window (region at +4, +4), then x
  double red[4][kMWarps];
  unsigned long long bad[2];
  double mine[4];
};
static_assert(kMWarps * 512 <= kMIn * kMP, "staging buffers fit in the window");
constexpr int kMOff = 4 * kMP + 4;  // region pixel (0, 0) inside acc

// field[R0-4 .. R0+68) x [C0-4 .. C0+68) -> s.in (zeros outside the image).
template <bool kVec>
__device__ __forceinline__ void load_window(const float* __restrict__ f, int64_t pitch, int R0, int C0, int H, int W,
                                            float* in) {
  if (kVec) {  // W % 4 == 0, 16-byte aligned rows: every float4 is wholly inside or outside
    for (int i = threadIdx.x; i < kMIn * (kMIn / 4); i += kMThreads) {
      const int r = i / (kMIn / 4), c4 = i % (kMIn / 4);
      const int gr = R0 - 4 + r, gc = C0 - 4 + 4 * c4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr >= 0 && gr < H && gc >= 0 && gc < W) v = __ldg(reinterpret_cast<const float4*>(f + (int64_t)gr * pitch + gc));
      *reinterpret_cast<float4*>(in + r * kMP + 4 * c4) = v;
    }
  } else {
    for (int i = threadIdx.x; i < kMIn * kMIn; i += kMThreads) {
      const int r = i / kMIn, c = i % kMIn;
      const int gr = R0 - 4 + r, gc = C0 - 4 + c;
      in[r * kMP + c] = (gr >= 0 && gr < H && gc >= 0 && gc < W) ? __ldg(f + (int64_t)gr * pitch + gc) : 0.f;
    }
  }
}

// Soft threshold sign(c) * max(|c| - t, 0) as c - clamp(c, -t, t): the same fp32
// result for every finite c (c -/+ t is exactly |c| - t with c's sign), and t = 0
// is the identity (the DC pass-through, denoise.cpp:76).
__device__ __forceinline__ float soft(float c, float t) { return c - fminf(fmaxf(c, -t), t); }

// One parity phase of the tile grid: tiles (PA + 2a, PB + 2b) are disjoint; the
// phase's tiles are taken two at a time (consecutive in row-major order) per MMA.
template <int PA, int PB, bool kInterior, int NP>
__device__ __forceinline__ void denoise_pairs(const float* in, float* acc, const Frag8& f, int R0, int C0, int H, int W,
                                              float thr, float thr_dc, const int (&p)[NP]) {
  constexpr int NA = PA ? 8 : 9, NB = PB ? 8 : 9, NT = NA * NB;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  int o1[NP], o2[NP];
  bool v1[NP], v2[NP];
  float Y[NP][4], X[NP][4];
#pragma unroll
  for (int u = 0; u < NP; ++u) {
    const int k1 = 2 * p[u], k2 = (2 * p[u] + 1 < NT) ? 2 * p[u] + 1 : 2 * p[u];  // odd count: last tile alone
    const int ti1 = PA + 2 * (k1 / NB), tj1 = PB + 2 * (k1 % NB);
    const int ti2 = PA + 2 * (k2 / NB), tj2 = PB + 2 * (k2 % NB);
    o1[u] = (4 * ti1 + g) * kMP + 4 * tj1 + 2 * t;
    o2[u] = (4 * ti2 + g) * kMP + 4 * tj2 + 2 * t;
    v1[u] = true;
    v2[u] = k2 != k1;
    if (!kInterior) {  // tile origins must lie on the image's origin grid (denoise.cpp:57-62)
      v1[u] = (unsigned)(R0 - 4 + 4 * ti1) <= (unsigned)(H - 8) && (unsigned)(C0 - 4 + 4 * tj1) <= (unsigned)(W - 8);
      v2[u] = v2[u] && (unsigned)(R0 - 4 + 4 * ti2) <= (unsigned)(H - 8) && (unsigned)(C0 - 4 + 4 * tj2) <= (unsigned)(W - 8);
    }
    const float2 p0 = *reinterpret_cast<const float2*>(in + o1[u]);
    const float2 p1 = *reinterpret_cast<const float2*>(in + o2[u]);
    dct8x2_fwdT(f, p0, p1, Y[u]);
  }
#pragma unroll
  for (int u = 0; u < NP; ++u) {
    // Y^T slots: 0/1 -> tile 1 (row g, cols 2t, 2t+1), 2/3 -> tile 2; DC = slots 0/2 of lane 0
    Y[u][0] = soft(Y[u][0], thr_dc);
    Y[u][1] = soft(Y[u][1], thr);
    Y[u][2] = soft(Y[u][2], thr_dc);
    Y[u][3] = soft(Y[u][3], thr);
    dct8x2_inv_from_yt(f, Y[u], X[u]);
  }
#pragma unroll
  for (int u = 0; u < NP; ++u) {
    if (v1[u]) {
      float2* d = reinterpret_cast<float2*>(acc + o1[u]);
      float2 v = *d;
      v.x += X[u][0];
      v.y += X[u][1];
      *d = v;
    }
    if (v2[u]) {
      float2* d = reinterpret_cast<float2*>(acc + o2[u]);
      float2 v = *d;
      v.x += X[u][2];
      v.y += X[u][3];
      *d = v;
    }
  }
}

template <int PA, int PB, bool kInterior>
__device__ __forceinline__ void denoise_phase(const float* in, float* acc, const Frag8& f, int R0, int C0, int H, int W,
                                              float thr, float thr_dc) {
  constexpr int NA = PA ? 8 : 9, NB = PB ? 8 : 9, NPAIR = (NA * NB + 1) / 2;
  const int warp = threadIdx.x >> 5;
#pragma unroll 1
  for (int p = warp; p < NPAIR; p += kMWarps) {  // (two pairs per warp in flight measured slower: registers)
    const int pp[1] = {p};
    denoise_pairs<PA, PB, kInterior, 1>(in, acc, f, R0, C0, H, W, thr, thr_dc, pp);
  }
  __syncthreads();
}

template <bool kInterior>
__device__ __forceinline__ void denoise_phases(const float* in, float* acc, const Frag8& f, int R0, int C0, int H,
                                               int W, float thr, float thr_dc) {
  denoise_phase<0, 0, kInterior>(in, acc, f, R0, C0, H, W, thr, thr_dc);
  denoise_phase<0, 1, kInterior>(in, acc, f, R0, C0, H, W, thr, thr_dc);
  denoise_phase<1, 0, kInterior>(in, acc, f, R0, C0, H, W, thr, thr_dc);
  denoise_phase<1, 1, kInterior>(in, acc, f, R0, C0, H, W, thr, thr_dc);
}

// dct_soft_threshold of the window into acc, normalised on the region (denoise.cpp:90).
// Expects the window loaded; ends with __syncthreads.
__device__ void denoise_region_mma(const float* in, float* acc, int R0, int C0, int H, int W, float thr) {
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < kMIn * kMP / 4; i += kMThreads) reinterpret_cast<float4*>(acc)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  Frag8 f;
  load_frag8(f);
  const float thr_dc = lane == 0 ? 0.f : thr;
  __syncthreads();
  if (R0 >= 4 && C0 >= 4 && R0 + kMR + 4 <= H && C0 + kMR + 4 <= W) denoise_phases<true>(in, acc, f, R0, C0, H, W, thr, thr_dc);
  else denoise_phases<false>(in, acc, f, R0, C0, H, W, thr, thr_dc);
  // weights: valid tile origins covering the pixel per axis (1 or 2 each) -> exact power-of-two scale;
  // the 4 pixels of a float4 share their 4-aligned column group
  for (int i = tid; i < kMR * kMR / 4; i += kMThreads) {
    const int r = i / (kMR / 4), c = 4 * (i % (kMR / 4));
    const int br = (R0 + r) & ~3, bc = C0 + c;
    const int wr = (br >= 4 ? 1 : 0) + (br <= H - 8 ? 1 : 0);
    const int wc = (bc >= 4 ? 1 : 0) + (bc <= W - 8 ? 1 : 0);
    const int w = wr * wc;
    const float sc = w == 4 ? 0.25f : (w == 2 ? 0.5f : 1.f);
    float4* d = reinterpret_cast<float4*>(acc + kMOff + r * kMP + c);
    float4 v = *d;
    v.x *= sc;
    v.y *= sc;
    v.z *= sc;
    v.w *= sc;
    *d = v;
  }
  __syncthreads();
}

struct IdaLaneSums {
  double z = 0.0, sse = 0.0, y = 0.0, cnt = 0.0;
  unsigned long long badx = ~0ull, badz = ~0ull;
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
      S.badx = gi < S.badx ? gi : S.badx;
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

// Stage cnt values of y (and z) of one block into smem; returns after __syncwarp.
__device__ __forceinline__ void stage_yz(const IdaParams& P, int64_t off, int cnt, float* yb, float* zb, bool need_z,
                                        IdaLaneSums& S) {
  const int lane = threadIdx.x & 31;
  for (int k = lane; k < cnt; k += 32) {
    const float yv = __ldg(P.y + off + k);
    yb[k] = yv;
    if (P.is_init) S.y += (double)yv * (double)yv;
    if (need_z) zb[k] = P.z[off + k];
  }
  __syncwarp();
}

__device__ __forceinline__ float z_update(const IdaParams& P, float yv, float ax, float zo, unsigned long long gi,
                                          IdaLaneSums& S, float onsager) {
  const float zn = (yv - ax) + onsager * zo;  // finish_step (recon.cpp:86-88)
  S.z += (double)zn * (double)zn;
  if (!isfinite(zn)) S.badz = gi < S.badz ? gi : S.badz;
  return zn;
}

// ---- B = 16: one sensing block per warp step ---------------------------------------------
// init: acc <- A* y (the warm start x0, recon.cpp:119-131)
__device__ void init_x16(const IdaParams& P, int img, int R0, int C0, IdaMmaSmem& s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  Frag16 f;
  load_frag16(f);
  uint32_t rank[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) rank[q] = zigzag_rank_dev<16>()[dslot_col(q) * 16 + dslot_row(q)];
  float* yb = s.in + warp * 512;
  for (int bi = warp; bi < 16; bi += kMWarps) {
    const int gbr = R0 / 16 + bi / 4, gbc = C0 / 16 + bi % 4;
    const int lr0 = (bi / 4) * 16, lc0 = (bi % 4) * 16;
    int cnt = 0;
    int64_t off = 0;
    if (gbr < P.rows && gbc < P.cols) {
      const int64_t bidx = (int64_t)img * P.rows * P.cols + (int64_t)gbr * P.cols + gbc;
      cnt = P.counts[bidx];
      off = (int64_t)img * P.y_stride + P.offsets[bidx];
    }
    for (int k = lane; k < cnt; k += 32) yb[k] = __ldg(P.y + off + k);
    __syncwarp();
    Acc16 Yt;
#pragma unroll
    for (int q = 0; q < 8; ++q) Yt.v[q >> 2][q & 3] = (int)rank[q] < cnt ? yb[rank[q]] : 0.f;
    const Acc16 X = dct16_inv_from_yt(f, Yt);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        *reinterpret_cast<float2*>(s.acc + kMOff + (lr0 + g + 8 * h) * kMP + lc0 + 8 * j + 2 * t) =
            make_float2(X.v[j][2 * h], X.v[j][2 * h + 1]);
    __syncwarp();
  }
}

__device__ void block_phase16(const IdaParams& P, int img, int R0, int C0, IdaMmaSmem& s, IdaLaneSums& S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float ons = P.onsager_img ? (float)P.onsager_img[img] : P.onsager;
  Frag16 f;
  load_frag16(f);
  uint32_t rank[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) rank[q] = zigzag_rank_dev<16>()[dslot_col(q) * 16 + dslot_row(q)];
  float* yb = s.in + warp * 512;
  float* zb = yb + 256;
  const bool last = P.pseudo_out == nullptr;
  for (int bi = warp; bi < 16; bi += kMWarps) {
    const int gbr = R0 / 16 + bi / 4, gbc = C0 / 16 + bi % 4;
    if (gbr >= P.rows || gbc >= P.cols) continue;  // warp-uniform
    const int lr0 = (bi / 4) * 16, lc0 = (bi % 4) * 16;
    const int64_t bidx = (int64_t)img * P.rows * P.cols + (int64_t)gbr * P.cols + gbc;
    const int cnt = P.counts[bidx];
    const int32_t boff = P.offsets[bidx];
    const int64_t off = (int64_t)img * P.y_stride + boff;
    if (lane == 0) S.cnt += (double)cnt;
    float xv[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float* r = s.acc + kMOff + (lr0 + 8 * j + g) * kMP + lc0 + 2 * t;
      const float2 a = *reinterpret_cast<const float2*>(r);
      const float2 b = *reinterpret_cast<const float2*>(r + 8);
      xv[j][0] = a.x;
      xv[j][1] = a.y;
      xv[j][2] = b.x;
      xv[j][3] = b.y;
    }
    const Acc16 Yt = dct16_fwd_f32(f, xv);  // (A x)^T in slot layout
    stage_yz(P, off, cnt, yb, zb, !P.is_init, S);
    Acc16 Zm;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = (int)rank[q];
      float zn = 0.f;
      if (r < cnt) {
        zn = z_update(P, yb[r], Yt.v[q >> 2][q & 3], P.is_init ? 0.f : zb[r], (unsigned long long)(boff + r), S,
                      ons);
        zb[r] = zn;
      }
      Zm.v[q >> 2][q & 3] = zn;
    }
    __syncwarp();
    for (int k = lane; k < cnt; k += 32) P.z[off + k] = zb[k];
    Acc16 Az;
    if (!last) Az = dct16_inv_from_yt(f, Zm);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lr = lr0 + g + 8 * h, lc = lc0 + 8 * j + 2 * t;
        const float2 x = *reinterpret_cast<const float2*>(s.acc + kMOff + lr * kMP + lc);
        x_checks(P, img, R0 + lr, C0 + lc, x, S);
        store_out(P, img, R0 + lr, C0 + lc, x, last ? make_float2(0.f, 0.f) : make_float2(Az.v[j][2 * h], Az.v[j][2 * h + 1]));
      }
    __syncwarp();
  }
}

// ---- B = 8: two horizontally adjacent sensing blocks per warp step ------------------------
__device__ void init_x8(const IdaParams& P, int img, int R0, int C0, IdaMmaSmem& s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  Frag8 f;
  load_frag8(f);
  uint32_t rank[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) rank[e] = zigzag_rank_dev<8>()[(2 * t + e) * 8 + g];  // Y^T[g][2t+e] = Y[2t+e][g]
  float* yb = s.in + warp * 512;
  for (int pi = warp; pi < 32; pi += kMWarps) {
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
    dct8x2_inv_from_yt(f, Yt, X);
    const int lr = 8 * br + g, lc = 8 * bc + 2 * t;
    *reinterpret_cast<float2*>(s.acc + kMOff + lr * kMP + lc) = make_float2(X[0], X[1]);
    *reinterpret_cast<float2*>(s.acc + kMOff + lr * kMP + lc + 8) = make_float2(X[2], X[3]);
    __syncwarp();
  }
}

__device__ void block_phase8(const IdaParams& P, int img, int R0, int C0, IdaMmaSmem& s, IdaLaneSums& S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float ons = P.onsager_img ? (float)P.onsager_img[img] : P.onsager;
  Frag8 f;
  load_frag8(f);
  uint32_t rank[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) rank[e] = zigzag_rank_dev<8>()[(2 * t + e) * 8 + g];
  float* yb = s.in + warp * 512;  // [q][64] y, then [q][64] z at +128
  float* zb = yb + 128;
  const bool last = P.pseudo_out == nullptr;
  for (int pi = warp; pi < 32; pi += kMWarps) {
    const int br = pi / 4, bc = 2 * (pi % 4);
    const int gbr = R0 / 8 + br, gbc0 = C0 / 8 + bc;
    if (gbr >= P.rows || gbc0 >= P.cols) continue;  // warp-uniform
    const bool has1 = gbc0 + 1 < P.cols;
    int cnt[2] = {0, 0};
    int32_t boff[2] = {0, 0};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (q == 1 && !has1) break;
      const int64_t bidx = (int64_t)img * P.rows * P.cols + (int64_t)gbr * P.cols + gbc0 + q;
      cnt[q] = P.counts[bidx];
      boff[q] = P.offsets[bidx];
    }
    if (lane == 0) S.cnt += (double)(cnt[0] + cnt[1]);
    const int lr = 8 * br + g, lc = 8 * bc + 2 * t;
    const float2 x0 = *reinterpret_cast<const float2*>(s.acc + kMOff + lr * kMP + lc);
    const float2 x1 = *reinterpret_cast<const float2*>(s.acc + kMOff + lr * kMP + lc + 8);
    float Yt[4];
    dct8x2_fwdT(f, x0, x1, Yt);
    const int64_t ibase = (int64_t)img * P.y_stride;
    stage_yz(P, ibase + boff[0], cnt[0], yb, zb, !P.is_init, S);
    stage_yz(P, ibase + boff[1], cnt[1], yb + 64, zb + 64, !P.is_init, S);
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
    if (!last) dct8x2_inv_from_yt(f, Zm, Az);
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
__device__ void reduce_and_finish(const IdaParams& P, int img, int region, IdaMmaSmem& s, IdaLaneSums& S) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    s.bad[0] = ~0ull;
    s.bad[1] = ~0ull;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    S.z += __shfl_xor_sync(0xffffffffu, S.z, o);
    S.sse += __shfl_xor_sync(0xffffffffu, S.sse, o);
    S.y += __shfl_xor_sync(0xffffffffu, S.y, o);
    S.cnt += __shfl_xor_sync(0xffffffffu, S.cnt, o);
  }
  __syncthreads();
  if ((tid & 31) == 0) {
    s.red[0][tid >> 5] = S.z;
    s.red[1][tid >> 5] = S.sse;
    s.red[2][tid >> 5] = S.y;
    s.red[3][tid >> 5] = S.cnt;
  }
  if (S.badx != ~0ull) atomicMin(&s.bad[0], S.badx);
  if (S.badz != ~0ull) atomicMin(&s.bad[1], S.badz);
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < 4; ++q) {
      double a = 0.0;
      for (int w = 0; w < kMWarps; ++w) a += s.red[q][w];
      s.mine[q] = a;
    }
    if (s.bad[0] != ~0ull) atomicMin(P.badx + img, s.bad[0]);
    if (s.bad[1] != ~0ull) atomicMin(P.badz + img, s.bad[1]);
  }
  finish_image(P, img, region, s.mine);
}

template <int B, bool kVec>
__global__ void __launch_bounds__(kMThreads, 4) ida_mma_kernel(IdaParams P) {
  __shared__ __align__(16) IdaMmaSmem s;
  const int img = blockIdx.y, region = blockIdx.x;
  const int R0 = (region / P.regions_x) * kMR, C0 = (region % P.regions_x) * kMR;
  if (P.is_init) {
    if (!P.warm) {  // cold start: x0 = 0, so z0 = y (recon.cpp:119-131)
      for (int i = threadIdx.x; i < kMIn * kMP / 4; i += kMThreads)
        reinterpret_cast<float4*>(s.acc)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else if (B == 16) {
      init_x16(P, img, R0, C0, s);
    } else {
      init_x8(P, img, R0, C0, s);
    }
    __syncthreads();
  } else if (P.x_in) {  // x from another denoiser: load the region
    const float* xs = P.x_in + (int64_t)img * P.Hc * P.Wc;
    for (int i = threadIdx.x; i < kMR * kMR / 4; i += kMThreads) {
      const int r = i / (kMR / 4), c = 4 * (i % (kMR / 4));
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (R0 + r < P.Hc && C0 + c < P.Wc) v = __ldg(reinterpret_cast<const float4*>(xs + (int64_t)(R0 + r) * P.Wc + C0 + c));
      *reinterpret_cast<float4*>(s.acc + kMOff + r * kMP + c) = v;
    }
    __syncthreads();
  } else {
    const float thr = (float)(P.k * P.sigma_in[img]);
    load_window<kVec>(P.pseudo_in + (int64_t)img * P.Hc * P.Wc, P.Wc, R0, C0, P.Hc, P.Wc, s.in);
    denoise_region_mma(s.in, s.acc, R0, C0, P.Hc, P.Wc, thr);
  }
  IdaLaneSums S;
  if (B == 16) block_phase16(P, img, R0, C0, s, S);
  else block_phase8(P, img, R0, C0, s, S);
  reduce_and_finish(P, img, region, s, S);
}

// Standalone denoise(dct_threshold) on f32 fields (denoise.cpp:96-109).
template <bool kVec>
__global__ void __launch_bounds__(kMThreads, 3)
denoise_mma_kernel(const float* __restrict__ field, int H, int W, int64_t stride, const double* __restrict__ thr,
                   float* __restrict__ out, int regions_x) {
  __shared__ __align__(16) IdaMmaSmem s;
  const int img = blockIdx.y, region = blockIdx.x;
  const int R0 = (region / regions_x) * kMR, C0 = (region % regions_x) * kMR;
  load_window<kVec>(field + (int64_t)img * stride, W, R0, C0, H, W, s.in);
  denoise_region_mma(s.in, s.acc, R0, C0, H, W, (float)thr[img]);
  for (int i = threadIdx.x; i < kMR * kMR; i += kMThreads) {
    const int r = i / kMR, c = i % kMR;
    if (R0 + r < H && C0 + c < W) out[(int64_t)img * stride + (int64_t)(R0 + r) * W + C0 + c] = s.acc[kMOff + r * kMP + c];
  }
}

int launch_denoise(Ctx* ctx, const float* field, int32_t h, int32_t w, int64_t stride, int32_t n,
                   const double* thresholds_dev, float* out, cudaStream_t s) {
  const int rx = (w + kMR - 1) / kMR, ry = (h + kMR - 1) / kMR;
  const bool vec = (w % 4 == 0) && (stride % 4 == 0) && (reinterpret_cast<uintptr_t>(field) % 16 == 0);
  for (int done = 0; done < n;) {
    const int cnt = std::min(n - done, 65535);
    const dim3 grid(rx * ry, cnt);
    const int kt = ktimer_begin(ctx, s, "denoise");
    if (vec)
      denoise_mma_kernel<true><<<grid, kMThreads, 0, s>>>(field + (int64_t)done * stride, h, w, stride,
                                                           thresholds_dev + done, out + (int64_t)done * stride, rx);
    else
      denoise_mma_kernel<false><<<grid, kMThreads, 0, s>>>(field + (int64_t)done * stride, h, w, stride,
                                                            thresholds_dev + done, out + (int64_t)done * stride, rx);
    ktimer_end(ctx, s, kt);
    ctx->launches++;
    done += cnt;
  }
  return cuda_status(cudaGetLastError(), "denoise launch");
}

int ida_mma_region() { return kMR; }

void launch_ida_mma_kernel(int block, const IdaParams& P, dim3 grid, cudaStream_t s) {
  // pseudo buffers are internal (256-B aligned, Wc % 8 == 0): always the vector window
  if (block == 16) ida_mma_kernel<16, true><<<grid, kMThreads, 0, s>>>(P);
  else ida_mma_kernel<8, true><<<grid, kMThreads, 0, s>>>(P);
}

}  // namespace abcs_b200
