// psnr / mse (metrics.cpp:63-77) between u8 references and f32 images, per image:
// mse accumulated in fp64 over the h x w pixels, psnr = 10 log10(255^2 / mse), +inf
// when mse == 0. Row slabs -> per-CTA fp64 partials -> fixed-order fold per image
// (deterministic). Used for the Idct branch of reconstruct()'s trace (recon.cpp:217-221).
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
                                 double* __restrict__ psnr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double sse = 0.0;
  for (int p = 0; p < parts; ++p) sse += partials[(int64_t)i * parts + p];
  const double mse = sse / pixels;
  psnr[i] = mse == 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 10.0 * log10(255.0 * 255.0 / mse);
}

int launch_psnr(Ctx* ctx, const uint8_t* ref, int64_t ref_stride, int ref_pitch, const float* img, int64_t img_stride,
                int img_pitch, int h, int w, int n, double* psnr, cudaStream_t s) {
  const int parts = (h + kMetricRowsPerCta - 1) / kMetricRowsPerCta;
  int st;
  double* partials = static_cast<double*>(ctx_scratch(ctx, (size_t)n * parts * 8, s, &st));
  if (st) return st;
  for (int done = 0; done < n;) {
    const int cnt = std::min(n - done, 65535);
    sse_partials_kernel<<<dim3(parts, cnt), kMetricThreads, 0, s>>>(ref + done * ref_stride, ref_stride, ref_pitch,
                                                                    img + done * img_stride, img_stride, img_pitch, h,
                                                                    w, partials + (int64_t)done * parts);
    ctx->launches++;
    done += cnt;
  }
  psnr_fold_kernel<<<(n + 127) / 128, 128, 0, s>>>(partials, parts, n, (double)h * (double)w, psnr);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "psnr launch");
}

}  // namespace abcs_b200
