// State shared by the IDA kernels (ida.cu: CUDA-core path for B = 32; ida_mma.cu:
// tensor-core path for B = 8, 16): launch parameters and the per-image fold of the
// region partials into sigma / trace / divergence (recon.cpp:81-93, 53-73).
#pragma once
#include <cstdint>

#include "common.cuh"

namespace abcs_b200 {

struct IdaParams {
  int rows, cols, n;
  int Hc, Wc;
  int regions_x, regions_y, regions_per_img;
  const uint16_t* counts;
  const int32_t* offsets;
  const float* y;
  int64_t y_stride;
  float* z;                // in place
  const float* pseudo_in;  // step: pseudo_t
  float* pseudo_out;       // pseudo_{t+1} (nullptr on the last step)
  float* x_out;            // estimate x on the last step (clamped when clamp_out)
  int64_t out_stride;
  int out_pitch;
  const uint8_t* ref;
  int64_t ref_stride;
  int ref_pitch;
  float onsager;           // 1/D_F (0 for the warm start)
  double k;                // threshold multiplier
  const double* sigma_in;  // sigma_t per image (step); unused for init
  double* sigma_out;       // sigma_{t+1} per image
  double* msize;           // M per image (written by init, read by steps)
  double* partials;        // [n][regions_per_img][4]
  unsigned int* counters;  // [n]
  double* trace;           // [n][iters+1][4] or nullptr
  int trace_row;
  int trace_rows;
  int32_t* diverged;       // [n][2] or nullptr
  unsigned long long* badx;  // [n] min (index*2 + kind) for x, ~0 = none
  unsigned long long* badz;  // [n] min index for z
  int iteration;           // iteration number after this launch (0 for init)
  int is_init;
  int warm;                // init: x0 = A* y (1) or x0 = 0 (0) (init_state, recon.cpp:119-131)
  int clamp_out;           // x_out gets clamp(x, 0, 255) (reconstruct's final estimate) or raw x (damp_step state)
  const float* x_in;       // step: the new estimate precomputed by another denoiser (ISTA/AMP/DAMP, blur), pitch Wc;
                           // nullptr = denoise pseudo_in with the fused dct_threshold
  const double* onsager_img;  // per-image Onsager coefficient (AMP/DAMP), else the scalar `onsager`
};

// Last CTA of an image folds the region partials (fixed order, so the result
// is deterministic) into sigma, the trace row and the divergence record.
// Called by every thread with `mine` written by thread 0: the partial is published with a
// release RMW on the image's counter, and the CTA whose RMW completes the count acquires every
// other CTA's partial and folds them with all its threads. No sequentially consistent fence.
static __device__ void finish_image(const IdaParams& P, int img, int region, const double* mine) {
  __shared__ unsigned int s_last;
  __shared__ double s_fold[32][4];
  if (threadIdx.x == 0) {
    double* part = P.partials + ((int64_t)img * P.regions_per_img + region) * 4;
    for (int q = 0; q < 4; ++q) part[q] = mine[q];
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;\n" : "=r"(prev) : "l"(P.counters + img) : "memory");
    s_last = prev == (unsigned)P.regions_per_img - 1 ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  // The last CTA of the image folds every region's partial with all its threads (a 4096-region
  // image is 4096 L2 round trips for one thread): thread t sums regions t, t + nt, ... in order,
  // then a fixed shuffle tree and the warps in order -- deterministic for a given block size.
  __threadfence();  // the other threads' side of thread 0's acquire
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  const double2* pp = reinterpret_cast<const double2*>(P.partials + (int64_t)img * P.regions_per_img * 4);
  for (int r = threadIdx.x; r < P.regions_per_img; r += blockDim.x) {
    const double2 v0 = __ldcg(pp + 2 * r), v1 = __ldcg(pp + 2 * r + 1);  // L2, never a stale L1 line
    a[0] += v0.x;
    a[1] += v0.y;
    a[2] += v1.x;
    a[3] += v1.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int q = 0; q < 4; ++q) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
  if ((threadIdx.x & 31) == 0)
    for (int q = 0; q < 4; ++q) s_fold[threadIdx.x >> 5][q] = a[q];
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int q = 0; q < 4; ++q) {
    a[q] = 0.0;
    for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) a[q] += s_fold[w][q];
  }
  P.counters[img] = 0;  // ready for the next launch
  const double M = a[3];  // op.measurements() = sum of counts, re-summed every launch (exact in fp64)
  if (P.is_init && P.msize) P.msize[img] = M;
  const double znorm = sqrt(a[0]);
  // init_state: sigma0 = ||y|| / sqrt(M) (recon.cpp:129); finish_step: ||z|| / sqrt(M) (:91)
  const double sigma = (P.is_init ? sqrt(a[2]) : znorm) / sqrt(M);
  P.sigma_out[img] = sigma;
  if (P.trace) {
    double* row = P.trace + ((int64_t)img * P.trace_rows + P.trace_row) * 4;
    row[0] = (double)P.iteration;
    row[1] = znorm;
    row[2] = sigma;
    double psnr = __longlong_as_double(0x7ff8000000000000ll);  // NaN without a reference
    if (P.ref) {
      const double mse = a[1] / ((double)P.Hc * (double)P.Wc);  // metrics.cpp:63-77
      psnr = (mse == 0.0) ? __longlong_as_double(0x7ff0000000000000ll) : 10.0 * log10(255.0 * 255.0 / mse);
    }
    row[3] = psnr;
  }
  if (!P.is_init) {
    const unsigned long long bx = P.badx[img], bz = P.badz[img];
    if ((bx != ~0ull || bz != ~0ull) && P.diverged && P.diverged[2 * img] == 0) {
      P.diverged[2 * img] = P.iteration;
      P.diverged[2 * img + 1] = (bx != ~0ull) ? ((bx & 1ull) ? 2 : 1) : 3;
    }
  }
  P.badx[img] = ~0ull;
  P.badz[img] = ~0ull;
}


}  // namespace abcs_b200
