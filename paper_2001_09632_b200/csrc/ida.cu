// IDA refinement for B = 32 on CUDA cores (B = 8/16: ida_mma.cu) -- reconstruct() with
// ReconMethod::Ida, recon.cpp:199-259 -- and
// the dct_threshold denoiser (denoise.cpp:52-92).
//
// State carried between launches is pseudo_t = x_t + A* z_t (recon.cpp:75-79)
// plus z_t, so one launch per iteration does everything blockwise-local:
//   x_{t+1} = D_{sigma_t}(pseudo_t)          (8x8 tiles, stride 4, 4-px halo)
//   z_{t+1} = y - A x_{t+1} + z_t / D_F      (finish_step, recon.cpp:81-93)
//   pseudo_{t+1} = x_{t+1} + A* z_{t+1}      (next iteration's pseudo_data)
// and reduces ||z_{t+1}||^2, the trace PSNR error and the divergence checks
// (check_finite, recon.cpp:53-73) per image; the last CTA of each image turns
// the partials into sigma_{t+1} = ||z||/sqrt(M) for the next launch (the only
// cross-block dependency, hence the kernel boundary). The warm start
// (init_state, recon.cpp:119-131: x0 = A*y, z0 = y - A x0, sigma0 = ||y||/sqrt(M))
// is the same block phase fed by a decode. The last iteration writes the
// clamped estimate instead of pseudo (recon.cpp:255-257).
#include <cfloat>

#include "common.cuh"
#include "ida_common.cuh"
#include "internal.h"

namespace abcs_b200 {

constexpr int kIdaThreads = 256;
constexpr int kRegion = 32;             // output pixels per CTA side
constexpr int kHalo = 4;                // denoiser tile overlap
constexpr int kIn = kRegion + 2 * kHalo;  // 40
constexpr int kInPitch = kIn + 1;
constexpr int kAccPitch = kRegion + 1;
constexpr int kTileSlots = kIdaThreads / 8;  // 32 concurrent 8x8 tiles
constexpr int kTileFloats = 8 * 9;



// ---------------------------------------------------------------------------
// dct_soft_threshold over one 32x32 output region: s_in holds the field on
// [R0-4, R0+36) x [C0-4, C0+36) (zeros outside the image). Tiles with origins
// in {R0-4, ..., R0+28} intersected with the valid origin set {0,4,..,H-8} are
// processed in 4 parity phases so overlapping tiles never race, which also
// fixes the summation order. s_acc receives sum/weight (denoise.cpp:90).
__device__ void denoise_region(const float* s_in, float* s_acc, float* s_tile, int R0, int C0, int H, int W,
                               float thr) {
  const int tid = threadIdx.x;
  for (int i = tid; i < kRegion * kAccPitch; i += kIdaThreads) s_acc[i] = 0.f;
  __syncthreads();
  const int slot = tid / 8, t = tid % 8;
  const unsigned gmask = 0xffu << ((tid & 31) & ~7);
  float* T = s_tile + slot * kTileFloats;
  for (int phase = 0; phase < 4; ++phase) {
    const int pa = phase >> 1, pb = phase & 1;
    // tiles of this phase: ti in {pa, pa+2, ..}, tj in {pb, pb+2, ..} (ti,tj in 0..8)
    const int nti = (9 - pa + 1) / 2, ntj = (9 - pb + 1) / 2;
    const int ntiles = nti * ntj;
    for (int base = 0; base < ntiles; base += kTileSlots) {
      const int idx = base + slot;
      bool active = idx < ntiles;
      int orr = 0, oc = 0;
      if (active) {
        const int ti = pa + 2 * (idx / ntj), tj = pb + 2 * (idx % ntj);
        orr = R0 - kHalo + 4 * ti;
        oc = C0 - kHalo + 4 * tj;
        active = orr >= 0 && orr <= H - 8 && oc >= 0 && oc <= W - 8;
      }
      if (active) {
        const int lr = orr - (R0 - kHalo), lc = oc - (C0 - kHalo);
        float x[8], y[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = s_in[(lr + t) * kInPitch + lc + c];
        Dct<8>::fwd(x, y);
#pragma unroll
        for (int v = 0; v < 8; ++v) T[t * 9 + v] = y[v];
        __syncwarp(gmask);
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = T[u * 9 + t];
        Dct<8>::fwd(x, y);  // y[u] = coefficient (u, t)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (u == 0 && t == 0) continue;  // DC passes through (denoise.cpp:76)
          const float c = y[u];
          const float mag = fabsf(c) - thr;
          y[u] = mag > 0.f ? copysignf(mag, c) : 0.f;
        }
        Dct<8>::inv(y, x);  // x[r] = column t of C^T Y
#pragma unroll
        for (int r = 0; r < 8; ++r) T[r * 9 + t] = x[r];
        __syncwarp(gmask);
#pragma unroll
        for (int v = 0; v < 8; ++v) y[v] = T[t * 9 + v];
        Dct<8>::inv(y, x);  // row t of the tile
        const int ar = orr + t - R0;
        if (ar >= 0 && ar < kRegion) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int ac = oc + c - C0;
            if (ac >= 0 && ac < kRegion) s_acc[ar * kAccPitch + ac] += x[c];
          }
        }
      }
      __syncthreads();
    }
  }
  // weights: number of valid tile origins covering the pixel, per axis
  for (int i = tid; i < kRegion * kRegion; i += kIdaThreads) {
    const int r = i / kRegion, c = i % kRegion;
    const int gr = R0 + r, gc = C0 + c;
    if (gr >= H || gc >= W) continue;
    const int br = 4 * (gr / 4), bc = 4 * (gc / 4);
    const int wr = (br - 4 >= 0 ? 1 : 0) + (br <= H - 8 ? 1 : 0);
    const int wc = (bc - 4 >= 0 ? 1 : 0) + (bc <= W - 8 ? 1 : 0);
    s_acc[r * kAccPitch + c] = s_acc[r * kAccPitch + c] / (float)(wr * wc);
  }
  __syncthreads();
}

// Load field[R0-4 .. R0+36) x [C0-4 .. C0+36) into s_in (zeros outside).
__device__ void load_halo(const float* __restrict__ f, int64_t pitch, int R0, int C0, int H, int W, float* s_in) {
  for (int i = threadIdx.x; i < kIn * kIn; i += kIdaThreads) {
    const int r = i / kIn, c = i % kIn;
    const int gr = R0 - kHalo + r, gc = C0 - kHalo + c;
    float v = 0.f;
    if (gr >= 0 && gr < H && gc >= 0 && gc < W) v = __ldg(f + (int64_t)gr * pitch + gc);
    s_in[r * kInPitch + c] = v;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Block phase over the sensing blocks of the region, with x in s_x:
//   z_new = (y - A x) + onsager * z_old   (init: z_old = 0)
//   out   = x + A* z_new                  (last step: clamp(x) instead)
// red[0] = sum z_new^2, red[1] = sum (ref - x)^2, red[2] = sum y^2, red[3] = sum counts.
template <int B>
__device__ void block_phase(const IdaParams& P, int img, int R0, int C0, const float* s_x, float* s_tile,
                            const unsigned short* s_zz, double* red) {
  constexpr int BPR = kRegion / B;  // blocks per region side
  constexpr int NG = BPR * BPR;     // groups needed
  constexpr int TF = Tile<B>::kFloats;
  __shared__ double s_red[4][kIdaThreads / 32];
  __shared__ unsigned long long s_bad[2];
  const int tid = threadIdx.x;
  const int g = tid / B, lane = tid % B;
  double zsum = 0.0, sse = 0.0, ysum = 0.0, csum = 0.0;
  unsigned long long badx = ~0ull, badz = ~0ull;
  if (tid == 0) {
    s_bad[0] = ~0ull;
    s_bad[1] = ~0ull;
  }
  if (g < NG) {
    const int gbr = R0 / B + g / BPR, gbc = C0 / B + g % BPR;
    if (gbr < P.rows && gbc < P.cols) {
      const int64_t nb = (int64_t)P.rows * P.cols;
      const int64_t bidx = (int64_t)img * nb + (int64_t)gbr * P.cols + gbc;
      const int cnt = P.counts[bidx];
      const int64_t off = (int64_t)img * P.y_stride + P.offsets[bidx];
      if (lane == 0) csum = (double)cnt;
      Tile<B> ta{s_tile + g * 2 * TF}, tb{s_tile + g * 2 * TF + TF};
      const int lr = (g / BPR) * B + lane, lc0 = (g % BPR) * B;
      float xr[B], y[B];
#pragma unroll
      for (int c = 0; c < B; ++c) xr[c] = s_x[lr * kAccPitch + lc0 + c];
      // A x (operators.cpp:23-48): forward DCT of the block, rows then columns
      Dct<B>::fwd(xr, y);
#pragma unroll
      for (int v = 0; v < B; ++v) ta.at(lane, v) = y[v];
#pragma unroll
      for (int v = 0; v < B; ++v) tb.at(lane, v) = 0.f;
      __syncwarp(group_mask<B>());
      {
        float col[B], cy[B];
#pragma unroll
        for (int u = 0; u < B; ++u) col[u] = ta.at(u, lane);
        Dct<B>::fwd(col, cy);
#pragma unroll
        for (int u = 0; u < B; ++u) ta.at(u, lane) = cy[u];
      }
      __syncwarp(group_mask<B>());
      // finish_step z update (recon.cpp:86-88)
      for (int k = lane; k < cnt; k += B) {
        const int flat = s_zz[k];
        const float ax = ta.zz(flat);
        const float yv = P.y[off + k];
        const float zo = P.is_init ? 0.f : P.z[off + k];
        const float zn = (yv - ax) + (P.onsager_img ? (float)P.onsager_img[img] : P.onsager) * zo;
        P.z[off + k] = zn;
        tb.zz(flat) = zn;
        zsum += (double)zn * (double)zn;
        ysum += (double)yv * (double)yv;
        if (!isfinite(zn)) {
          const unsigned long long gi = (unsigned long long)(P.offsets[bidx] + k);
          badz = gi < badz ? gi : badz;
        }
      }
      __syncwarp(group_mask<B>());
      // A* z_new (operators.cpp:50-76): columns then rows
      {
        float col[B], cx[B];
#pragma unroll
        for (int u = 0; u < B; ++u) col[u] = tb.at(u, lane);
        Dct<B>::inv(col, cx);
#pragma unroll
        for (int r = 0; r < B; ++r) tb.at(r, lane) = cx[r];
      }
      __syncwarp(group_mask<B>());
      float az[B];
      {
        float rw[B];
#pragma unroll
        for (int v = 0; v < B; ++v) rw[v] = tb.at(lane, v);
        Dct<B>::inv(rw, az);
      }
      const int gr = gbr * B + lane, gc0 = gbc * B;
      const uint8_t* refrow =
          P.ref ? P.ref + (int64_t)img * P.ref_stride + (int64_t)gr * P.ref_pitch + gc0 : nullptr;
#pragma unroll
      for (int c = 0; c < B; ++c) {
        const float xv = xr[c];
        if (!isfinite(xv) || fabsf(xv) > 1e6f) {  // check_finite (recon.cpp:56-65)
          const unsigned long long gi =
              ((unsigned long long)((int64_t)gr * P.Wc + gc0 + c) << 1) | (isfinite(xv) ? 1ull : 0ull);
          badx = gi < badx ? gi : badx;
        }
        if (refrow) {
          const double d = (double)refrow[c] - (double)xv;
          sse += d * d;
        }
      }
      float o[B];
      float* dst;
      if (P.pseudo_out) {
        dst = P.pseudo_out + (int64_t)img * P.Hc * P.Wc + (int64_t)gr * P.Wc + gc0;
#pragma unroll
        for (int c = 0; c < B; ++c) o[c] = xr[c] + az[c];
        store_row_f32<B>(dst, o, true);
      } else {
        dst = P.x_out + (int64_t)img * P.out_stride + (int64_t)gr * P.out_pitch + gc0;
#pragma unroll
        for (int c = 0; c < B; ++c) o[c] = P.clamp_out ? fminf(fmaxf(xr[c], 0.f), 255.f) : xr[c];  // recon.cpp:255-257
        store_row_f32<B>(dst, o, (P.out_pitch % 4 == 0) && (P.out_stride % 4 == 0));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    zsum += __shfl_xor_sync(0xffffffffu, zsum, o);
    sse += __shfl_xor_sync(0xffffffffu, sse, o);
    ysum += __shfl_xor_sync(0xffffffffu, ysum, o);
    csum += __shfl_xor_sync(0xffffffffu, csum, o);
  }
  __syncthreads();
  if ((tid & 31) == 0) {
    s_red[0][tid >> 5] = zsum;
    s_red[1][tid >> 5] = sse;
    s_red[2][tid >> 5] = ysum;
    s_red[3][tid >> 5] = csum;
  }
  if (badx != ~0ull) atomicMin(&s_bad[0], badx);
  if (badz != ~0ull) atomicMin(&s_bad[1], badz);
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < 4; ++q) {
      double a = 0.0;
      for (int w = 0; w < kIdaThreads / 32; ++w) a += s_red[q][w];
      red[q] = a;
    }
    if (s_bad[0] != ~0ull) atomicMin(P.badx + img, s_bad[0]);
    if (s_bad[1] != ~0ull) atomicMin(P.badz + img, s_bad[1]);
  }
}

// Warm start: x0 = A* y (decode into smem), then the block phase with onsager 0.
template <int B>
__global__ void __launch_bounds__(kIdaThreads) ida_init_kernel(IdaParams P) {
  __shared__ float s_x[kRegion * kAccPitch];
  __shared__ float s_tile[2 * (kRegion / B) * (kRegion / B) * Tile<B>::kFloats];
  __shared__ unsigned short s_zz[B * B];
  __shared__ double s_mine[4];
  load_zigzag<B>(s_zz);
  const int img = blockIdx.y;
  const int region = blockIdx.x;
  const int R0 = (region / P.regions_x) * kRegion, C0 = (region % P.regions_x) * kRegion;
  __syncthreads();
  constexpr int BPR = kRegion / B;
  const int g = threadIdx.x / B, lane = threadIdx.x % B;
  if (g < BPR * BPR) {
    const int gbr = R0 / B + g / BPR, gbc = C0 / B + g % BPR;
    if (gbr < P.rows && gbc < P.cols) {
      const int64_t bidx = (int64_t)img * P.rows * P.cols + (int64_t)gbr * P.cols + gbc;
      const int cnt = P.counts[bidx];
      const float* src = P.y + (int64_t)img * P.y_stride + P.offsets[bidx];
      Tile<B> t{s_tile + g * Tile<B>::kFloats};
#pragma unroll
      for (int v = 0; v < B; ++v) t.at(lane, v) = 0.f;
      __syncwarp(group_mask<B>());
      for (int k = lane; k < cnt; k += B) t.zz(s_zz[k]) = src[k];
      __syncwarp(group_mask<B>());
      float col[B], cx[B];
#pragma unroll
      for (int u = 0; u < B; ++u) col[u] = t.at(u, lane);
      Dct<B>::inv(col, cx);
#pragma unroll
      for (int r = 0; r < B; ++r) t.at(r, lane) = cx[r];
      __syncwarp(group_mask<B>());
#pragma unroll
      for (int v = 0; v < B; ++v) col[v] = t.at(lane, v);
      Dct<B>::inv(col, cx);
      const int lr = (g / BPR) * B + lane, lc0 = (g % BPR) * B;
#pragma unroll
      for (int c = 0; c < B; ++c) s_x[lr * kAccPitch + lc0 + c] = (cnt && P.warm) ? cx[c] : 0.f;
    }
  }
  __syncthreads();
  block_phase<B>(P, img, R0, C0, s_x, s_tile, s_zz, s_mine);
  finish_image(P, img, region, s_mine);
}

// One IDA iteration: denoise pseudo_t over the region (+4 px halo), then the block phase.
template <int B>
__global__ void __launch_bounds__(kIdaThreads) ida_step_kernel(IdaParams P) {
  __shared__ float s_in[kIn * kInPitch];
  __shared__ float s_x[kRegion * kAccPitch];
  __shared__ float s_tile[kTileSlots * kTileFloats];
  __shared__ unsigned short s_zz[B * B];
  __shared__ double s_mine[4];
  static_assert(2 * (kRegion / B) * (kRegion / B) * Tile<B>::kFloats <= kTileSlots * kTileFloats, "tile smem");
  load_zigzag<B>(s_zz);
  const int img = blockIdx.y;
  const int region = blockIdx.x;
  const int R0 = (region / P.regions_x) * kRegion, C0 = (region % P.regions_x) * kRegion;
  if (P.x_in) {  // x from another denoiser
    for (int i = threadIdx.x; i < kRegion * kRegion; i += kIdaThreads) {
      const int r = i / kRegion, c = i % kRegion;
      s_x[r * kAccPitch + c] = (R0 + r < P.Hc && C0 + c < P.Wc)
                                   ? P.x_in[(int64_t)img * P.Hc * P.Wc + (int64_t)(R0 + r) * P.Wc + C0 + c]
                                   : 0.f;
    }
    __syncthreads();
  } else {
    const float thr = (float)(P.k * P.sigma_in[img]);
    load_halo(P.pseudo_in + (int64_t)img * P.Hc * P.Wc, P.Wc, R0, C0, P.Hc, P.Wc, s_in);
    denoise_region(s_in, s_x, s_tile, R0, C0, P.Hc, P.Wc, thr);
  }
  block_phase<B>(P, img, R0, C0, s_x, s_tile, s_zz, s_mine);
  finish_image(P, img, region, s_mine);
}

static size_t align256(size_t v) { return (v + 255) / 256 * 256; }

size_t ida_scratch_bytes(int32_t rows, int32_t cols, int32_t block, int64_t y_stride, int32_t n,
                         const abcs_ida_config& cfg) {
  const int64_t Hc = (int64_t)rows * block, Wc = (int64_t)cols * block;
  const int64_t regions = ((Hc + kRegion - 1) / kRegion) * ((Wc + kRegion - 1) / kRegion);  // >= the 64x64 grid
  size_t b = 0;
  b += 2 * align256((size_t)n * Hc * Wc * 4);               // pseudo ping-pong
  b += align256((size_t)n * y_stride * 4);                  // z
  b += align256((size_t)n * (cfg.iterations + 1) * 8);      // sigma per step
  b += align256((size_t)n * 8);                             // M
  b += align256((size_t)n * regions * 4 * 8);               // partials
  b += align256((size_t)n * 4);                             // counters
  b += 2 * align256((size_t)n * 8);                         // badx, badz
  return b;
}

namespace {

struct IdaLayout {
  float* pseudo[2];
  float* z;
  double* sigma;
  double* msize;
  double* partials;
  unsigned int* counters;
  unsigned long long* badx;
  unsigned long long* badz;
};

IdaLayout carve(void* scratch, int64_t Hc, int64_t Wc, int64_t y_stride, int n, int iterations, int64_t regions) {
  IdaLayout L;
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += align256(bytes);
    return r;
  };
  L.pseudo[0] = reinterpret_cast<float*>(take((size_t)n * Hc * Wc * 4));
  L.pseudo[1] = reinterpret_cast<float*>(take((size_t)n * Hc * Wc * 4));
  L.z = reinterpret_cast<float*>(take((size_t)n * y_stride * 4));
  L.sigma = reinterpret_cast<double*>(take((size_t)n * (iterations + 1) * 8));
  L.msize = reinterpret_cast<double*>(take((size_t)n * 8));
  L.partials = reinterpret_cast<double*>(take((size_t)n * regions * 4 * 8));
  L.counters = reinterpret_cast<unsigned int*>(take((size_t)n * 4));
  L.badx = reinterpret_cast<unsigned long long*>(take((size_t)n * 8));
  L.badz = reinterpret_cast<unsigned long long*>(take((size_t)n * 8));
  return L;
}

struct IdaGeometry {
  bool mma;
  int rx, ry;
  int64_t Hc, Wc, regions;
};

IdaGeometry geometry(int rows, int cols, int block) {
  IdaGeometry G;
  G.Hc = (int64_t)rows * block;
  G.Wc = (int64_t)cols * block;
  G.mma = (block == 8 || block == 16);  // tensor-core kernels (ida_mma.cu), 64x64 regions
  const int side = G.mma ? ida_mma_region() : kRegion;
  G.rx = (int)((G.Wc + side - 1) / side);
  G.ry = (int)((G.Hc + side - 1) / side);
  G.regions = (int64_t)G.rx * G.ry;
  return G;
}

cudaError_t reset_reductions(const IdaLayout& L, int n, int32_t* diverged, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(L.counters, 0, (size_t)n * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(L.badx, 0xff, (size_t)n * 8, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(L.badz, 0xff, (size_t)n * 8, s);
  if (e == cudaSuccess && diverged) e = cudaMemsetAsync(diverged, 0, (size_t)n * 2 * 4, s);
  return e;
}

IdaParams base_params(const IdaGeometry& G, const IdaLayout& L, int rows, int cols, int n, const uint16_t* counts,
                      const int32_t* offsets, const float* y, int64_t y_stride, double k) {
  IdaParams P{};
  P.rows = rows;
  P.cols = cols;
  P.n = n;
  P.Hc = (int)G.Hc;
  P.Wc = (int)G.Wc;
  P.regions_x = G.rx;
  P.regions_y = G.ry;
  P.regions_per_img = (int)G.regions;
  P.counts = counts;
  P.offsets = offsets;
  P.y = y;
  P.y_stride = y_stride;
  P.z = L.z;
  P.k = k;
  P.msize = L.msize;
  P.partials = L.partials;
  P.counters = L.counters;
  P.badx = L.badx;
  P.badz = L.badz;
  P.warm = 1;
  P.clamp_out = 1;
  return P;
}

void launch_one(Ctx* ctx, int block, const IdaGeometry& G, const IdaParams& P, cudaStream_t s) {
  const dim3 grid((unsigned)G.regions, (unsigned)P.n);
  const int kt = ktimer_begin(ctx, s, P.is_init ? "ida_init" : "ida_step");
  if (G.mma) launch_ida_mma_kernel(block, P, grid, s);
  else if (P.is_init) ida_init_kernel<32><<<grid, kIdaThreads, 0, s>>>(P);
  else ida_step_kernel<32><<<grid, kIdaThreads, 0, s>>>(P);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
}

}  // namespace

int launch_ida(Ctx* ctx, int32_t rows, int32_t cols, int32_t block, const uint16_t* counts, const int32_t* offsets,
               const float* y, int64_t y_stride, int32_t n, const abcs_ida_config& cfg, const uint8_t* ref,
               int64_t ref_stride, int32_t ref_pitch, float* out, int64_t out_stride, int32_t out_pitch,
               double* trace, int32_t* diverged, void* scratch, cudaStream_t s) {
  if (block != 8 && block != 16 && block != 32)
    return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  if (n > 65535) return set_error(ABCS_ERR_UNSUPPORTED, "IDA batch limited to 65535 images per call");
  const IdaGeometry G = geometry(rows, cols, block);
  const IdaLayout L = carve(scratch, G.Hc, G.Wc, y_stride, n, cfg.iterations, G.regions);
  cudaError_t e = reset_reductions(L, n, diverged, s);
  if (e != cudaSuccess) return cuda_status(e, "ida scratch init");
  IdaParams P = base_params(G, L, rows, cols, n, counts, offsets, y, y_stride, cfg.k);
  P.out_stride = out_stride;
  P.out_pitch = out_pitch;
  P.ref = ref;
  P.ref_stride = ref_stride;
  P.ref_pitch = ref_pitch;
  P.trace = trace;
  P.trace_rows = cfg.iterations + 1;
  P.diverged = diverged;
  // warm start (init_state, recon.cpp:119-131) -> pseudo_0
  P.is_init = 1;
  P.onsager = 0.f;
  P.pseudo_out = L.pseudo[0];
  P.sigma_out = L.sigma;
  P.trace_row = 0;
  P.iteration = 0;
  launch_one(ctx, block, G, P, s);
  for (int t = 0; t < cfg.iterations; ++t) {  // damp_step(Ida) x iterations (recon.cpp:236-253)
    ABCS_NVTX("ida_iteration");
    P.is_init = 0;
    P.onsager = (float)(1.0 / cfg.damping);  // IDA: onsager = 1/D_F (recon.cpp:183-184)
    P.pseudo_in = L.pseudo[t & 1];
    const bool last = (t + 1 == cfg.iterations);
    P.pseudo_out = last ? nullptr : L.pseudo[(t + 1) & 1];
    P.x_out = last ? out : nullptr;
    P.sigma_in = L.sigma + (int64_t)t * n;
    P.sigma_out = L.sigma + (int64_t)(t + 1) * n;
    P.trace_row = t + 1;
    P.iteration = t + 1;
    launch_one(ctx, block, G, P, s);
  }
  return cuda_status(cudaGetLastError(), "ida launch");
}

// ---- explicit solver state (init_state / damp_step with variant Ida) -----------------------
__global__ void add_field_kernel(float* __restrict__ dst, const float* __restrict__ src, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

size_t ida_state_scratch_bytes(int32_t rows, int32_t cols, int32_t block, int64_t y_stride, int32_t n) {
  abcs_ida_config one{};
  one.iterations = 1;
  return ida_scratch_bytes(rows, cols, block, y_stride, n, one);
}

int launch_ida_state(Ctx* ctx, bool init, int32_t rows, int32_t cols, int32_t block, const uint16_t* counts,
                     const int32_t* offsets, const float* y, int64_t y_stride, int32_t n, int warm, double damping,
                     double k, float* x, float* z, double* sigma, int32_t iteration, int32_t* diverged, void* scratch,
                     cudaStream_t s) {
  if (block != 8 && block != 16 && block != 32)
    return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  if (n > 65535) return set_error(ABCS_ERR_UNSUPPORTED, "IDA batch limited to 65535 images per call");
  const IdaGeometry G = geometry(rows, cols, block);
  const IdaLayout L = carve(scratch, G.Hc, G.Wc, y_stride, n, 1, G.regions);
  cudaError_t e = reset_reductions(L, n, diverged, s);
  if (e != cudaSuccess) return cuda_status(e, "ida scratch init");
  IdaParams P = base_params(G, L, rows, cols, n, counts, offsets, y, y_stride, k);
  P.z = z;  // the caller's residual, updated in place
  P.x_out = x;
  P.out_stride = G.Hc * G.Wc;
  P.out_pitch = (int)G.Wc;
  P.clamp_out = 0;
  P.diverged = diverged;
  P.pseudo_out = nullptr;  // write x, not pseudo
  P.sigma_out = L.sigma + n;
  P.iteration = iteration;
  if (init) {
    P.is_init = 1;
    P.warm = warm;
    P.onsager = 0.f;
  } else {
    // pseudo = A* z + x (pseudo_data, recon.cpp:75-79) into the scratch field
    int st = launch_decode(ctx, rows, cols, block, counts, offsets, z, y_stride, n, L.pseudo[0], G.Hc * G.Wc,
                           (int)G.Wc, s);
    if (st) return st;
    const int64_t cnt = (int64_t)n * G.Hc * G.Wc;
    add_field_kernel<<<(unsigned)std::min<int64_t>((cnt + 255) / 256, (int64_t)ctx->sm_count * 8), 256, 0, s>>>(
        L.pseudo[0], x, cnt);
    ctx->launches++;
    P.is_init = 0;
    P.onsager = (float)(1.0 / damping);
    P.pseudo_in = L.pseudo[0];
    P.sigma_in = sigma;
  }
  launch_one(ctx, block, G, P, s);
  e = cudaMemcpyAsync(sigma, L.sigma + n, (size_t)n * 8, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return cuda_status(e, "ida sigma copy");
  return cuda_status(cudaGetLastError(), "ida state launch");
}

// ---- every iterative method (recon.cpp:133-259) -------------------------------------------
namespace {

struct ReconScratch {
  IdaLayout L;          // block-phase reductions; L.pseudo[0] = pseudo field, L.pseudo[1] = new estimate
  float* perturbed;     // DAMP: pseudo + eps * probe
  float* moved;         // DAMP: D(perturbed)
  float* tmp;           // blur intermediate
  float* probe;         // Rademacher probe (one field, shared by the batch)
  float* x;             // reconstruct(): state x
  float* z;             // reconstruct(): state z
  double* sigma;        // reconstruct(): state sigma
  double* thr;          // k * sigma
  double* eps;
  double* onsager;
  double* partials;
  unsigned* maxbits;
  unsigned long long* active;
  int32_t* offsets;     // computed when the caller passes none
};

}  // namespace

// Denoise `in` -> `out` with the configured denoiser at sigma (device, per image) (denoise.cpp:96-109).
int run_denoiser(Ctx* ctx, const abcs_recon_config& cfg, const float* in, float* out, float* tmp,
                        int H, int W, int n, const double* sigma, double* thr, cudaStream_t s) {
  const int64_t N = (int64_t)H * W;
  if (cfg.denoiser == ABCS_DENOISER_IDENTITY) {
    return cuda_status(cudaMemcpyAsync(out, in, (size_t)n * N * 4, cudaMemcpyDeviceToDevice, s), "identity denoiser");
  }
  if (cfg.denoiser == ABCS_DENOISER_DCT_THRESHOLD) {
    int st = launch_scale(ctx, sigma, cfg.k, n, thr, s);
    if (st) return st;
    return launch_denoise(ctx, in, H, W, N, n, thr, out, s);
  }
  // blur: the radius depends on sigma (device) -> read the batch's largest sigma first
  std::vector<double> h(n);
  cudaError_t e = cudaMemcpyAsync(h.data(), sigma, (size_t)n * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e, "blur sigma readback");
  double smax = 0.0;
  for (double v : h) smax = std::max(smax, v);
  const int rmax = std::max(1, (int)std::ceil(3.0 * smax / cfg.sigma_scale));
  void* wbuf = nullptr;
  e = cudaMallocAsync(&wbuf, (size_t)n * (2 * rmax + 1) * 8 + (size_t)n * 4, s);
  if (e != cudaSuccess) return cuda_status(e, "blur weights alloc");
  double* w = static_cast<double*>(wbuf);
  int* r = reinterpret_cast<int*>(w + (size_t)n * (2 * rmax + 1));
  int st = launch_blur(ctx, in, tmp, out, H, W, n, sigma, cfg.sigma_scale, rmax, w, r, s);
  cudaFreeAsync(wbuf, s);
  return st;
}

int launch_recon(Ctx* ctx, bool one_step, int32_t rows, int32_t cols, int32_t block, const uint16_t* counts,
                 const int32_t* offsets_in, const float* y, int64_t y_stride, int32_t n, const abcs_recon_config& cfg,
                 const uint8_t* ref, int64_t ref_stride, int32_t ref_pitch, float* x_state, float* z_state,
                 double* sigma_state, int32_t iteration0, float* out, int64_t out_stride, int32_t out_pitch,
                 double* trace, int32_t* diverged, cudaStream_t s) {
  if (block != 8 && block != 16 && block != 32)
    return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  if (n > 65535) return set_error(ABCS_ERR_UNSUPPORTED, "reconstruction batch limited to 65535 images per call");
  const IdaGeometry G = geometry(rows, cols, block);
  const int64_t N = G.Hc * G.Wc;
  const bool damp = cfg.method == ABCS_RECON_DAMP || cfg.method == ABCS_RECON_DAMPD;
  // one ctx scratch request for everything
  abcs_ida_config one{};
  one.iterations = 1;
  const size_t base = ida_scratch_bytes(rows, cols, block, y_stride, n, one);
  auto al = [](size_t v) { return (v + 255) / 256 * 256; };
  const size_t fld = al((size_t)n * N * 4);
  const size_t parts = divergence_partials(ctx, N, n);
  const int steps = one_step ? 1 : cfg.iterations;
  const size_t probe_bytes = al((size_t)N * 4 * (damp ? steps : 1));  // every iteration's probe
  size_t need = base + 3 * fld + probe_bytes + 6 * al((size_t)n * 8) + al(parts * 8) + al((size_t)n * 4) +
                al((size_t)n * rows * cols * 4);
  if (!one_step) need += fld + al((size_t)n * y_stride * 4) + al((size_t)n * 8);
  int st;
  char* p = static_cast<char*>(ctx_scratch(ctx, need, s, &st));
  if (st) return st;
  ReconScratch R{};
  R.L = carve(p, G.Hc, G.Wc, y_stride, n, 1, G.regions);
  p += base;
  auto take = [&](size_t b) {
    char* r = p;
    p += b;
    return r;
  };
  R.perturbed = reinterpret_cast<float*>(take(fld));
  R.moved = reinterpret_cast<float*>(take(fld));
  R.tmp = reinterpret_cast<float*>(take(fld));
  R.probe = reinterpret_cast<float*>(take(probe_bytes));
  R.thr = reinterpret_cast<double*>(take(al((size_t)n * 8)));
  R.eps = reinterpret_cast<double*>(take(al((size_t)n * 8)));
  R.onsager = reinterpret_cast<double*>(take(al((size_t)n * 8)));
  R.active = reinterpret_cast<unsigned long long*>(take(al((size_t)n * 8)));
  double* sigma_next = reinterpret_cast<double*>(take(al((size_t)n * 8)));
  double* Mimg = reinterpret_cast<double*>(take(al((size_t)n * 8)));  // op.measurements() per image
  R.partials = reinterpret_cast<double*>(take(al(parts * 8)));
  R.maxbits = reinterpret_cast<unsigned*>(take(al((size_t)n * 4)));
  R.offsets = reinterpret_cast<int32_t*>(take(al((size_t)n * rows * cols * 4)));
  if (!one_step) {
    R.x = reinterpret_cast<float*>(take(fld));
    R.z = reinterpret_cast<float*>(take(al((size_t)n * y_stride * 4)));
    R.sigma = reinterpret_cast<double*>(take(al((size_t)n * 8)));
  } else {
    R.x = x_state;
    R.z = z_state;
    R.sigma = sigma_state;
  }
  const int32_t* offsets = offsets_in;
  if (!offsets) {
    st = launch_offsets(ctx, rows * cols, n, block, counts, R.offsets, nullptr, nullptr, s);
    if (st) return st;
    offsets = R.offsets;
  }
  cudaError_t e = reset_reductions(R.L, n, diverged, s);
  if (e != cudaSuccess) return cuda_status(e, "recon scratch init");
  IdaParams P = base_params(G, R.L, rows, cols, n, counts, offsets, y, y_stride, cfg.k);
  P.z = R.z;
  P.ref = ref;
  P.ref_stride = ref_stride;
  P.ref_pitch = ref_pitch;
  P.trace = trace;
  P.trace_rows = cfg.iterations + 1;
  P.diverged = diverged;
  st = launch_measurements(ctx, counts, offsets, rows * cols, n, Mimg, s);
  if (st) return st;
  int it = iteration0;
  if (!one_step) {  // warm start (init_state, recon.cpp:119-131): x0 = A* y, z0 = y - A x0, sigma0
    P.is_init = 1;
    P.warm = 1;
    P.onsager = 0.f;
    P.pseudo_out = nullptr;
    P.x_out = R.x;
    P.out_stride = N;
    P.out_pitch = (int)G.Wc;
    P.clamp_out = 0;
    P.sigma_out = R.sigma;
    P.trace_row = 0;
    P.iteration = 0;
    launch_one(ctx, block, G, P, s);
    it = 0;
  }
  if (damp) {  // the probes depend only on (seed, iteration): all of them in one launch up front
    st = launch_probes(ctx, cfg.seed, it, steps, N, R.probe, s);
    if (st) return st;
  }
  for (int t = 0; t < steps; ++t) {
    // pseudo_data (recon.cpp:75-79): P = A* z + x
    float* pseudo = R.L.pseudo[0];
    float* xn = R.L.pseudo[1];
    st = launch_decode(ctx, rows, cols, block, counts, offsets, R.z, y_stride, n, pseudo, N, (int)G.Wc, s);
    if (st) return st;
    add_field_kernel<<<(unsigned)std::min<int64_t>((n * N + 255) / 256, (int64_t)ctx->sm_count * 8), 256, 0, s>>>(
        pseudo, R.x, n * N);
    ctx->launches++;
    float onsager_scalar = 0.f;
    const double* onsager_img = nullptr;
    if (cfg.method == ABCS_RECON_ISTA || cfg.method == ABCS_RECON_AMP) {
      st = launch_soft_threshold(ctx, pseudo, xn, N, n, R.sigma, cfg.lambda, R.active, s);
      if (st) return st;
      if (cfg.method == ABCS_RECON_AMP) {
        st = launch_amp_onsager(ctx, R.active, n, Mimg, (double)N, it == 0, R.onsager, s);
        if (st) return st;
        onsager_img = R.onsager;
      }
    } else {
      st = run_denoiser(ctx, cfg, pseudo, xn, R.tmp, (int)G.Hc, (int)G.Wc, n, R.sigma, R.thr, s);
      if (st) return st;
      if (damp) {
        const float* probe = R.probe + (int64_t)t * N;
        st = launch_divergence_prep(ctx, pseudo, probe, N, n, R.maxbits, R.perturbed, R.eps, s);
        if (!st) st = run_denoiser(ctx, cfg, R.perturbed, R.moved, R.tmp, (int)G.Hc, (int)G.Wc, n, R.sigma, R.thr, s);
        if (!st)
          st = launch_damp_onsager(ctx, probe, R.moved, xn, N, n, R.eps, Mimg,
                                   cfg.method == ABCS_RECON_DAMPD ? cfg.damping : 1.0, R.partials, R.onsager, s);
        if (st) return st;
        onsager_img = R.onsager;
      } else {
        onsager_scalar = (float)(1.0 / cfg.damping);  // Ida (recon.cpp:183-184)
      }
    }
    // finish_step (recon.cpp:81-93) in the block phase with the new estimate precomputed
    const bool last = !one_step && t + 1 == steps;
    P.is_init = 0;
    P.x_in = xn;
    P.onsager = onsager_scalar;
    P.onsager_img = onsager_img;
    P.pseudo_in = nullptr;
    P.pseudo_out = nullptr;
    P.x_out = last ? out : R.x;
    P.out_stride = last ? out_stride : N;
    P.out_pitch = last ? out_pitch : (int)G.Wc;
    P.clamp_out = last ? 1 : 0;
    P.sigma_in = R.sigma;
    P.sigma_out = sigma_next;
    P.trace_row = it + 1;
    P.iteration = it + 1;
    launch_one(ctx, block, G, P, s);
    e = cudaMemcpyAsync(R.sigma, sigma_next, (size_t)n * 8, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "sigma copy");
    ++it;
  }
  return cuda_status(cudaGetLastError(), "recon launch");
}

}  // namespace abcs_b200
