// The rest of the reconstruction family on the device:
//   ista_step / amp_step (recon.cpp:133-168): pixel-domain soft threshold at lambda*sigma,
//     AMP's Onsager term (active/N)/delta from a per-image active count;
//   damp_step with variants Damp / DampD (recon.cpp:170-197): any denoiser, Onsager term
//     from the Monte-Carlo divergence (denoise.cpp:111-128): a Rademacher probe drawn from
//     std::mt19937_64 seeded by splitmix(seed, iteration) (recon.cpp:95-105), generated here
//     with the standard twist split into its two data-parallel halves;
//   the blur denoiser (denoise.cpp:14-48): separable Gaussian, clamp-to-edge, radius
//     ceil(3 sigma_s), sigma_s = sigma / sigma_scale.
// Every method then runs the fused finish_step block phase of the IDA kernels with the new
// estimate precomputed (IdaParams::x_in) and a per-image Onsager coefficient.
#include <cmath>

#include "internal.h"

namespace abcs_b200 {

constexpr int kRThreads = 256;

// ---- ISTA / AMP soft threshold ---------------------------------------------------------
// x = sign(p) max(|p| - lambda*sigma, 0); active[img] += #{|p| > thr} (recon.cpp:136-157)
__global__ void soft_threshold_kernel(const float* __restrict__ pseudo, float* __restrict__ x, int64_t N,
                                      const double* __restrict__ sigma, double lambda,
                                      unsigned long long* __restrict__ active) {
  const int img = blockIdx.y;
  const float thr = (float)(lambda * sigma[img]);
  const float* p = pseudo + (int64_t)img * N;
  float* o = x + (int64_t)img * N;
  unsigned cnt = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = p[i];
    const float mag = fabsf(v) - thr;
    const bool on = mag > 0.f;
    o[i] = on ? copysignf(mag, v) : 0.f;
    cnt += on ? 1u : 0u;
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(active + img, (unsigned long long)cnt);
}

// AMP: onsager = mean_derivative / delta = (active / N) / (M / N) in the reference's operation
// order (recon.cpp:158-165); 0 on the first step
__global__ void amp_onsager_kernel(const unsigned long long* __restrict__ active, int n, const double* __restrict__ M,
                                   double N, int first, double* __restrict__ onsager) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) onsager[i] = first ? 0.0 : ((double)active[i] / N) / (M[i] / N);
}

// op.measurements() per image = sum of counts = last offset + last count
__global__ void measurements_kernel(const uint16_t* __restrict__ counts, const int32_t* __restrict__ offsets, int nb,
                                    int n, double* __restrict__ M) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) M[i] = (double)offsets[(int64_t)i * nb + nb - 1] + (double)counts[(int64_t)i * nb + nb - 1];
}

// ---- DAMP divergence ---------------------------------------------------------------------
// epsilon = max|p| * 1e-3 + 1e-6 per image (recon.cpp:186-188); |p| >= 0 so its float bits order as u32
__global__ void absmax_kernel(const float* __restrict__ p, int64_t N, unsigned* __restrict__ maxbits) {
  const int img = blockIdx.y;
  unsigned m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, __float_as_uint(fabsf(p[(int64_t)img * N + i])));
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits + img, m);
}

// splitmix-style probe seed of an iteration (recon.cpp:95-105)
__device__ __forceinline__ uint64_t probe_seed_dev(uint64_t seed, int iteration) {
  uint64_t v = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(iteration + 1);
  v ^= v >> 30;
  v *= 0xBF58476D1CE4E5B9ull;
  v ^= v >> 27;
  v *= 0x94D049BB133111EBull;
  v ^= v >> 31;
  return v;
}

// std::mt19937_64 (seed) -> probe[i] = (out_i & 1) ? +1 : -1 for i < N. One CTA of 320 threads
// per probe: with it0 >= 0, CTA b writes the probe of iteration it0 + b (seed derived from
// `seed` as the reference does per damp_step) at probe + b * N, so a whole reconstruction's
// probes come from one launch; with it0 < 0 one CTA uses `seed` itself.
__global__ void __launch_bounds__(320)
mt19937_64_probe_kernel(uint64_t seed, int it0, int64_t N, float* __restrict__ probe) {
  constexpr int kN = 312, kM = 156;
  constexpr uint64_t kA = 0xB5026F5AA96619E9ull, kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;
  __shared__ uint64_t mt[kN];
  const int t = threadIdx.x;
  if (it0 >= 0) {
    seed = probe_seed_dev(seed, it0 + (int)blockIdx.x);
    probe += (int64_t)blockIdx.x * N;
  }
  if (t == 0) {  // seeding is sequential (mt[i] depends on mt[i-1])
    mt[0] = seed;
    for (int i = 1; i < kN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
  }
  __syncthreads();
  auto mix = [](uint64_t a, uint64_t b) {
    const uint64_t x = (a & kUpper) | (b & kLower);
    return (x >> 1) ^ ((x & 1ull) ? kA : 0ull);
  };
  for (int64_t base = 0; base < N; base += kN) {
    // twist (libstdc++ _M_gen_rand). Phase 1: i < 156 reads only old words.
    uint64_t v = 0;
    if (t < kM) v = mt[t + kM] ^ mix(mt[t], mt[t + 1]);
    __syncthreads();
    if (t < kM) mt[t] = v;
    __syncthreads();
    // Phase 2: 156 <= i < 312 reads new[i - 156] and old[i], old[i + 1] (new[0] for i = 311).
    const int i2 = t + kM;
    if (t < kM) v = mt[i2 - kM] ^ mix(mt[i2], (i2 + 1 < kN) ? mt[i2 + 1] : mt[0]);
    __syncthreads();
    if (t < kM) mt[i2] = v;
    __syncthreads();
    // temper and emit
    if (t < kN && base + t < N) {
      uint64_t y = mt[t];
      y ^= (y >> 29) & 0x5555555555555555ull;
      y ^= (y << 17) & 0x71D67FFFEDA60000ull;
      y ^= (y << 37) & 0xFFF7EEE000000000ull;
      y ^= y >> 43;
      probe[base + t] = (y & 1ull) ? 1.f : -1.f;
    }
    __syncthreads();
  }
}

// perturbed = p + eps[img] * probe (denoise.cpp:119-120)
__global__ void perturb_kernel(const float* __restrict__ p, const float* __restrict__ probe, int64_t N,
                               const unsigned* __restrict__ maxbits, float* __restrict__ out, double* __restrict__ eps) {
  const int img = blockIdx.y;
  const double e = (double)__uint_as_float(maxbits[img]) * 1e-3 + 1e-6;
  if (blockIdx.x == 0 && threadIdx.x == 0) eps[img] = e;
  const float ef = (float)e;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    out[(int64_t)img * N + i] = p[(int64_t)img * N + i] + ef * probe[i];
}

// per-CTA partial of sum probe * (moved - base) (denoise.cpp:124-127), folded in a fixed order
__global__ void div_partials_kernel(const float* __restrict__ probe, const float* __restrict__ moved,
                                    const float* __restrict__ base, int64_t N, double* __restrict__ partials) {
  __shared__ double s_red[kRThreads / 32];
  const int img = blockIdx.y;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    acc += (double)probe[i] * ((double)moved[(int64_t)img * N + i] - (double)base[(int64_t)img * N + i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRThreads / 32; ++w) t += s_red[w];
    partials[(int64_t)img * gridDim.x + blockIdx.x] = t;
  }
}

// onsager = (div / eps) / (delta * M) with delta = M / N, / D_F for DampD (recon.cpp:189-194)
__global__ void damp_onsager_kernel(const double* __restrict__ partials, int parts, const double* __restrict__ eps,
                                    int n, const double* __restrict__ Mv, double N, double divisor,
                                    double* __restrict__ onsager) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int p = 0; p < parts; ++p) s += partials[(int64_t)i * parts + p];
  const double div = s / eps[i];
  const double M = Mv[i];
  double o = div / ((M / N) * M);
  if (divisor != 1.0) o /= divisor;  // DampD: onsager /= D_F
  onsager[i] = o;
}

// dct_threshold's threshold k * sigma per image (denoise.cpp:105-106)
__global__ void scale_kernel(const double* __restrict__ sigma, double k, int n, double* __restrict__ thr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) thr[i] = k * sigma[i];
}

// ---- blur denoiser -----------------------------------------------------------------------
// per-image normalised Gaussian taps (denoise.cpp:15-24): radius = ceil(3 s), s = sigma / scale
__global__ void blur_weights_kernel(const double* __restrict__ sigma, double scale, int n, int rmax,
                                    double* __restrict__ w, int* __restrict__ radius) {
  const int img = blockIdx.x;
  if (threadIdx.x != 0) return;
  const double s = sigma[img] / scale;
  double* k = w + (int64_t)img * (2 * rmax + 1);
  if (s <= 0.0) {  // gaussian_blur returns the input unchanged
    radius[img] = -1;
    return;
  }
  const int r = (int)ceil(3.0 * s);
  radius[img] = r;
  double sum = 0.0;
  for (int i = -r; i <= r; ++i) {
    k[i + r] = exp(-0.5 * (double)(i * i) / (s * s));
    sum += k[i + r];
  }
  for (int i = 0; i <= 2 * r; ++i) k[i] /= sum;
}

template <bool kRows>
__global__ void blur_pass_kernel(const float* __restrict__ in, float* __restrict__ out, int H, int W,
                                 const double* __restrict__ w, const int* __restrict__ radius, int rmax) {
  const int img = blockIdx.y;
  const int r = radius[img];
  const int64_t N = (int64_t)H * W;
  const float* src = in + img * N;
  float* dst = out + img * N;
  const double* k = w + (int64_t)img * (2 * rmax + 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if (r < 0) {
      dst[i] = src[i];
      continue;
    }
    const int row = (int)(i / W), col = (int)(i % W);
    double acc = 0.0;
    for (int t = -r; t <= r; ++t) {
      const int rr = kRows ? row : min(max(row + t, 0), H - 1);
      const int cc = kRows ? min(max(col + t, 0), W - 1) : col;
      acc += k[t + r] * (double)src[(int64_t)rr * W + cc];
    }
    dst[i] = (float)acc;
  }
}

static unsigned grid_x(Ctx* ctx, int64_t N, int n) {
  const int64_t want = (N + kRThreads - 1) / kRThreads;
  const int64_t cap = std::max<int64_t>(1, (int64_t)ctx->sm_count * 8 / std::max(n, 1));
  return (unsigned)std::max<int64_t>(1, std::min(want, std::max<int64_t>(cap, 4)));
}

int launch_soft_threshold(Ctx* ctx, const float* pseudo, float* x, int64_t N, int n, const double* sigma,
                          double lambda, unsigned long long* active, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(active, 0, (size_t)n * 8, s);
  if (e != cudaSuccess) return cuda_status(e, "active reset");
  const int kt = ktimer_begin(ctx, s, "soft_threshold");
  soft_threshold_kernel<<<dim3(grid_x(ctx, N, n), n), kRThreads, 0, s>>>(pseudo, x, N, sigma, lambda, active);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "soft threshold launch");
}

int launch_measurements(Ctx* ctx, const uint16_t* counts, const int32_t* offsets, int nb, int n, double* M,
                        cudaStream_t s) {
  measurements_kernel<<<(n + 127) / 128, 128, 0, s>>>(counts, offsets, nb, n, M);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "measurements launch");
}

int launch_amp_onsager(Ctx* ctx, const unsigned long long* active, int n, const double* M, double N, bool first,
                       double* onsager, cudaStream_t s) {
  amp_onsager_kernel<<<(n + 127) / 128, 128, 0, s>>>(active, n, M, N, first ? 1 : 0, onsager);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "amp onsager launch");
}

int launch_blur(Ctx* ctx, const float* in, float* tmp, float* out, int H, int W, int n, const double* sigma_dev,
                double scale, int rmax, double* wscratch, int* rscratch, cudaStream_t s) {
  blur_weights_kernel<<<n, 32, 0, s>>>(sigma_dev, scale, n, rmax, wscratch, rscratch);
  ctx->launches++;
  const int64_t N = (int64_t)H * W;
  const dim3 grid(grid_x(ctx, N, n), n);
  const int kt = ktimer_begin(ctx, s, "blur");
  blur_pass_kernel<true><<<grid, kRThreads, 0, s>>>(in, tmp, H, W, wscratch, rscratch, rmax);
  blur_pass_kernel<false><<<grid, kRThreads, 0, s>>>(tmp, out, H, W, wscratch, rscratch, rmax);
  ktimer_end(ctx, s, kt);
  ctx->launches += 2;
  return cuda_status(cudaGetLastError(), "blur launch");
}

int launch_probe(Ctx* ctx, uint64_t seed, int64_t N, float* probe, cudaStream_t s) {
  const int kt = ktimer_begin(ctx, s, "mt19937_64_probe");
  mt19937_64_probe_kernel<<<1, 320, 0, s>>>(seed, -1, N, probe);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "probe launch");
}

int launch_probes(Ctx* ctx, uint64_t seed, int it0, int count, int64_t N, float* probes, cudaStream_t s) {
  const int kt = ktimer_begin(ctx, s, "mt19937_64_probe");
  mt19937_64_probe_kernel<<<(unsigned)count, 320, 0, s>>>(seed, it0, N, probes);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "probe launch");
}

int launch_divergence_prep(Ctx* ctx, const float* pseudo, const float* probe, int64_t N, int n, unsigned* maxbits,
                           float* perturbed, double* eps, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(maxbits, 0, (size_t)n * 4, s);
  if (e != cudaSuccess) return cuda_status(e, "absmax reset");
  const dim3 grid(grid_x(ctx, N, n), n);
  absmax_kernel<<<grid, kRThreads, 0, s>>>(pseudo, N, maxbits);
  perturb_kernel<<<grid, kRThreads, 0, s>>>(pseudo, probe, N, maxbits, perturbed, eps);
  ctx->launches += 2;
  return cuda_status(cudaGetLastError(), "divergence prep launch");
}

int launch_damp_onsager(Ctx* ctx, const float* probe, const float* moved, const float* base, int64_t N, int n,
                        const double* eps, const double* M, double divisor, double* partials, double* onsager,
                        cudaStream_t s) {
  const unsigned gx = grid_x(ctx, N, n);
  div_partials_kernel<<<dim3(gx, n), kRThreads, 0, s>>>(probe, moved, base, N, partials);
  damp_onsager_kernel<<<(n + 127) / 128, 128, 0, s>>>(partials, (int)gx, eps, n, M, (double)N, divisor, onsager);
  ctx->launches += 2;
  return cuda_status(cudaGetLastError(), "damp onsager launch");
}

size_t divergence_partials(Ctx* ctx, int64_t N, int n) { return (size_t)grid_x(ctx, N, n) * n; }

__global__ void perturb_given_kernel(const float* __restrict__ p, const float* __restrict__ probe, int64_t N,
                                     const double* __restrict__ eps, float* __restrict__ out) {
  const int img = blockIdx.y;
  const float ef = (float)eps[img];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    out[(int64_t)img * N + i] = p[(int64_t)img * N + i] + ef * probe[i];
}

__global__ void div_fold_kernel(const double* __restrict__ partials, int parts, const double* __restrict__ eps, int n,
                                double* __restrict__ div) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int p = 0; p < parts; ++p) s += partials[(int64_t)i * parts + p];
  div[i] = s / eps[i];
}

// divergence() with given epsilons: perturbed = field + eps * probe, then (probe . (D(pert) - D(field))) / eps
int launch_divergence_given(Ctx* ctx, const float* field, const float* probe, const float* base, int64_t N, int n,
                            const double* eps, float* perturbed, const float* moved, double* partials,
                            double* div, bool perturb_only, cudaStream_t s) {
  const unsigned gx = grid_x(ctx, N, n);
  if (perturb_only) {
    perturb_given_kernel<<<dim3(gx, n), kRThreads, 0, s>>>(field, probe, N, eps, perturbed);
    ctx->launches++;
    return cuda_status(cudaGetLastError(), "perturb launch");
  }
  div_partials_kernel<<<dim3(gx, n), kRThreads, 0, s>>>(probe, moved, base, N, partials);
  div_fold_kernel<<<(n + 127) / 128, 128, 0, s>>>(partials, (int)gx, eps, n, div);
  ctx->launches += 2;
  return cuda_status(cudaGetLastError(), "divergence launch");
}

int launch_scale(Ctx* ctx, const double* sigma, double k, int n, double* thr, cudaStream_t s) {
  scale_kernel<<<(n + 127) / 128, 128, 0, s>>>(sigma, k, n, thr);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "scale launch");
}

}  // namespace abcs_b200
