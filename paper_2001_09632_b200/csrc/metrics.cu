// psnr / mse (metrics.cpp:63-77) between u8 references and f32 images, per image:
// mse accumulated in fp64 over the h x w pixels, psnr = 10 log10(255^2 / mse), +inf
// when mse == 0. Row slabs -> per-CTA fp64 partials -> fixed-order fold per image
// (deterministic). Used for the Idct branch of reconstruct()'s trace (recon.cpp:217-221).
#include <algorithm>
#include <cmath>

#include "internal.h"

namespace abcs_b200 {

constexpr int kMetricThreads = 256;
constexpr int kMetricRowsPerCta = 16;

__global__ void __launch_bounds__(kMetricThreads)
sse_partials_kernel(const uint8_t* __restrict__ ref, int64_t ref_stride, int ref_pitch, const float* __restrict__ img,
                    int64_t img_stride, int img_pitch, int h, int w, double* __restrict__ partials) {
  __shared__ double s_red[kMetricThreads / 32];
  const int img_i = blockIdx.y;
  const int r0 = blockIdx.x * kMetricRowsPerCta, r1 = min(h, r0 + kMetricRowsPerCta);
  const uint8_t* R = ref + img_i * ref_stride;
  const float* X = img + img_i * img_stride;
  double acc = 0.0;
  for (int r = r0; r < r1; ++r)
    for (int c = threadIdx.x; c < w; c += kMetricThreads) {
      const double d = (double)R[(int64_t)r * ref_pitch + c] - (double)X[(int64_t)r * img_pitch + c];
      acc += d * d;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int q = 0; q < kMetricThreads / 32; ++q) a += s_red[q];
    partials[(int64_t)img_i * gridDim.x + blockIdx.x] = a;
  }
}

__global__ void psnr_fold_kernel(const double* __restrict__ partials, int parts, int n, double pixels,
                                 double* __restrict__ psnr, double* __restrict__ mse_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double sse = 0.0;
  for (int p = 0; p < parts; ++p) sse += partials[(int64_t)i * parts + p];
  const double mse = sse / pixels;
  if (mse_out) mse_out[i] = mse;
  if (psnr) psnr[i] = mse == 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 10.0 * log10(255.0 * 255.0 / mse);
}

// ---------------------------------------------------------------------------
// ssim (metrics.cpp:79-116): 11x11 Gaussian window (sigma 1.5, normalised), means over
// every fully interior window position, fp64 statistics. The separable passes run in
// the reference's order (horizontal then vertical, taps ascending) with fused multiply-add
// accumulation (the reference rounds the product first), so window means agree with the
// reference's to ~1e-16 relative and the map average within the 1e-12 the tests hold; the
// average is folded per image from per-tile fp64 partials in a fixed order.
constexpr int kSsimWin = 11;
constexpr int kSsimTR = 32, kSsimTC = 32;        // output (window) positions per tile: rows x cols
constexpr int kSsimInR = kSsimTR + kSsimWin - 1, kSsimInC = kSsimTC + kSsimWin - 1;  // 42 x 42
constexpr int kSsimThreads = 256;
constexpr int kSsimRun = 4;  // outputs per thread in each pass (register blocking)
static_assert(kSsimTC % kSsimRun == 0 && kSsimTR % kSsimRun == 0, "ssim tile");
static_assert((kSsimTR / kSsimRun) * kSsimTC == kSsimThreads, "one vertical run per thread");

struct SsimKernel {
  double k[kSsimWin];
};

static SsimKernel ssim_kernel_weights() {
  SsimKernel w;
  double sum = 0.0;
  for (int i = 0; i < kSsimWin; ++i) {
    const double d = i - (kSsimWin - 1) / 2.0;
    w.k[i] = std::exp(-0.5 * d * d / (1.5 * 1.5));
    sum += w.k[i];
  }
  for (double& v : w.k) v /= sum;
  return w;
}

struct SsimSmem {
  float x[kSsimInR][kSsimInC + 1], y[kSsimInR][kSsimInC + 1];
  double h[5][kSsimInR][kSsimTC];  // horizontal pass: x, y, xx, yy, xy
  double red[kSsimThreads / 32];
};

// Each thread keeps a run of 4 outputs in registers in both passes, so every input value is
// read (and squared) once per run instead of once per tap: the products x*x, y*y, x*y are the
// reference's xx/yy/xy arrays (metrics.cpp:96-100) and each window sum still adds its taps in
// ascending order. 80 registers (a few bytes spilled) for 3 CTAs per SM: the kernel is
// FP64-latency-bound, and 2 CTAs per SM (106 registers, no spills) measured 6.6 ms against
// 5.4 ms per 1024 images.
__global__ void __launch_bounds__(kSsimThreads, 3)
ssim_tiles_kernel(const uint8_t* __restrict__ ref, int64_t ref_stride, int ref_pitch, const float* __restrict__ img,
                  int64_t img_stride, int img_pitch, int H, int W, int tiles_x, SsimKernel kw,
                  double* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char ssim_smem_raw[];
  SsimSmem& S = *reinterpret_cast<SsimSmem*>(ssim_smem_raw);
  const int image = blockIdx.y, tile = blockIdx.x;
  const int r0 = (tile / tiles_x) * kSsimTR, c0 = (tile % tiles_x) * kSsimTC;
  const int Hv = H - kSsimWin + 1, Wv = W - kSsimWin + 1;
  const uint8_t* R = ref + image * ref_stride;
  const float* X = img + image * img_stride;
  for (int i = threadIdx.x; i < kSsimInR * kSsimInC; i += kSsimThreads) {
    const int r = i / kSsimInC, c = i % kSsimInC;
    const int gr = r0 + r, gc = c0 + c;
    const bool in = gr < H && gc < W;
    S.x[r][c] = in ? (float)R[(int64_t)gr * ref_pitch + gc] : 0.f;
    S.y[r][c] = in ? X[(int64_t)gr * img_pitch + gc] : 0.f;
  }
  __syncthreads();
  constexpr int kGroups = kSsimTC / kSsimRun;
  for (int i = threadIdx.x; i < kSsimInR * kGroups; i += kSsimThreads) {
    const int r = i / kGroups, c = (i % kGroups) * kSsimRun;
    double a[kSsimRun][5];
#pragma unroll
    for (int o = 0; o < kSsimRun; ++o)
#pragma unroll
      for (int q = 0; q < 5; ++q) a[o][q] = 0.0;
#pragma unroll
    for (int u = 0; u < kSsimRun + kSsimWin - 1; ++u) {
      const double x = S.x[r][c + u], y = S.y[r][c + u];
      const double xx = __dmul_rn(x, x), yy = __dmul_rn(y, y), xy = __dmul_rn(x, y);
#pragma unroll
      for (int o = 0; o < kSsimRun; ++o) {
        const int t = u - o;  // tap of output o that reads input u
        if (t < 0 || t >= kSsimWin) continue;
        const double kt = kw.k[t];
        a[o][0] = __fma_rn(kt, x, a[o][0]);
        a[o][1] = __fma_rn(kt, y, a[o][1]);
        a[o][2] = __fma_rn(kt, xx, a[o][2]);
        a[o][3] = __fma_rn(kt, yy, a[o][3]);
        a[o][4] = __fma_rn(kt, xy, a[o][4]);
      }
    }
#pragma unroll
    for (int o = 0; o < kSsimRun; ++o)
#pragma unroll
      for (int q = 0; q < 5; ++q) S.h[q][r][c + o] = a[o][q];
  }
  __syncthreads();
  const double C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
  double acc = 0.0;
  {
    const int c = threadIdx.x % kSsimTC, rr = (threadIdx.x / kSsimTC) * kSsimRun;
    double m[kSsimRun][5];
#pragma unroll
    for (int o = 0; o < kSsimRun; ++o)
#pragma unroll
      for (int q = 0; q < 5; ++q) m[o][q] = 0.0;
#pragma unroll
    for (int u = 0; u < kSsimRun + kSsimWin - 1; ++u) {
      double v[5];
#pragma unroll
      for (int q = 0; q < 5; ++q) v[q] = S.h[q][rr + u][c];
#pragma unroll
      for (int o = 0; o < kSsimRun; ++o) {
        const int t = u - o;
        if (t < 0 || t >= kSsimWin) continue;
        const double kt = kw.k[t];
#pragma unroll
        for (int q = 0; q < 5; ++q) m[o][q] = __fma_rn(kt, v[q], m[o][q]);
      }
    }
#pragma unroll
    for (int o = 0; o < kSsimRun; ++o) {
      if (r0 + rr + o >= Hv || c0 + c >= Wv) continue;
      const double mx = m[o][0], my = m[o][1];
      const double var_x = __dadd_rn(m[o][2], -__dmul_rn(mx, mx));
      const double var_y = __dadd_rn(m[o][3], -__dmul_rn(my, my));
      const double cov = __dadd_rn(m[o][4], -__dmul_rn(mx, my));
      const double num =
          __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mx), my), C1), __dadd_rn(__dmul_rn(2.0, cov), C2));
      const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mx, mx), __dmul_rn(my, my)), C1),
                                   __dadd_rn(__dadd_rn(var_x, var_y), C2));
      acc += __ddiv_rn(num, den);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kSsimThreads / 32; ++w) t += S.red[w];
    partials[(int64_t)image * gridDim.x + tile] = t;
  }
}

__global__ void ssim_fold_kernel(const double* __restrict__ partials, int tiles, int n, double windows,
                                 double* __restrict__ ssim) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int t = 0; t < tiles; ++t) s += partials[(int64_t)i * tiles + t];
  ssim[i] = s / windows;
}

size_t ssim_scratch_bytes(int h, int w, int n) {
  const int Hv = h - kSsimWin + 1, Wv = w - kSsimWin + 1;
  const int tx = (Wv + kSsimTC - 1) / kSsimTC, ty = (Hv + kSsimTR - 1) / kSsimTR;
  return (size_t)n * tx * ty * 8;
}

size_t psnr_scratch_bytes(int h, int n) { return (size_t)n * ((h + kMetricRowsPerCta - 1) / kMetricRowsPerCta) * 8; }

int launch_ssim(Ctx* ctx, const uint8_t* ref, int64_t ref_stride, int ref_pitch, const float* img, int64_t img_stride,
                int img_pitch, int h, int w, int n, double* ssim, cudaStream_t s, void* scratch) {
  const int Hv = h - kSsimWin + 1, Wv = w - kSsimWin + 1;
  const int tx = (Wv + kSsimTC - 1) / kSsimTC, ty = (Hv + kSsimTR - 1) / kSsimTR;
  int st = ABCS_OK;
  // concurrent callers (the host pipeline's slots) pass their own scratch
  double* partials = static_cast<double*>(scratch ? scratch : ctx_scratch(ctx, ssim_scratch_bytes(h, w, n), s, &st));
  if (st) return st;
  const SsimKernel kw = ssim_kernel_weights();
  cudaFuncSetAttribute(ssim_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SsimSmem));
  const int kt = ktimer_begin(ctx, s, "ssim");
  for (int done = 0; done < n;) {
    const int cnt = std::min(n - done, 65535);
    ssim_tiles_kernel<<<dim3(tx * ty, cnt), kSsimThreads, sizeof(SsimSmem), s>>>(ref + done * ref_stride, ref_stride, ref_pitch,
                                                                  img + done * img_stride, img_stride, img_pitch, h,
                                                                  w, tx, kw, partials + (int64_t)done * tx * ty);
    ctx->launches++;
    done += cnt;
  }
  ssim_fold_kernel<<<(n + 127) / 128, 128, 0, s>>>(partials, tx * ty, n, (double)Hv * (double)Wv, ssim);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "ssim launch");
}

int launch_psnr(Ctx* ctx, const uint8_t* ref, int64_t ref_stride, int ref_pitch, const float* img, int64_t img_stride,
                int img_pitch, int h, int w, int n, double* psnr, cudaStream_t s, double* mse, void* scratch) {
  const int parts = (h + kMetricRowsPerCta - 1) / kMetricRowsPerCta;
  int st = ABCS_OK;
  double* partials = static_cast<double*>(scratch ? scratch : ctx_scratch(ctx, psnr_scratch_bytes(h, n), s, &st));
  if (st) return st;
  for (int done = 0; done < n;) {
    const int cnt = std::min(n - done, 65535);
    sse_partials_kernel<<<dim3(parts, cnt), kMetricThreads, 0, s>>>(ref + done * ref_stride, ref_stride, ref_pitch,
                                                                    img + done * img_stride, img_stride, img_pitch, h,
                                                                    w, partials + (int64_t)done * parts);
    ctx->launches++;
    done += cnt;
  }
  psnr_fold_kernel<<<(n + 127) / 128, 128, 0, s>>>(partials, parts, n, (double)h * (double)w, psnr, mse);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "psnr launch");
}

}  // namespace abcs_b200
