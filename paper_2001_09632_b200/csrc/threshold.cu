// THB / THI full-sensing oracle decodes (metrics.cpp:126-225, metrics.hpp:27-38) on the
// device, bit-exact: keep the largest-|coefficient| entries per block (THB, balanced counts)
// or across the whole image (THI), ties to the lower zigzag index then the lower block
// index, and invert.
//
// These are quality baselines, so the transforms run in fp64 in the reference's exact
// operation order (dct.cpp:23-79: multiply then add, no fused multiply-add, the host glibc
// basis): every coefficient equals the reference's bit for bit, the selection is exact
// without guard bands, and so is the decoded image. B200's FP64 rate makes this cheap
// (~16 K fp64 operations per 16x16 block each way).
//   fwd64_kernel<B>:       u8 blocks -> fp64 coefficients (one thread per (u,c) then (u,v))
//   thb_select_kernel<B>:  per block, rank of each |c| among the block's B^2 -> zero the rest
//   thi_select_kernel<B>:  per image, radix select on the 64-bit |c| bits (8 x 8-bit digits),
//                          then on (zigzag rank * n_B + block) among exact ties; zero the rest
//   inv64_kernel<B>:       fp64 inverse, per block, in the reference order
#include <cfloat>

#include "common.cuh"
#include "internal.h"

namespace abcs_b200 {

template <int B>
struct Tb {
  static constexpr int kArea = B * B;
  static constexpr int kPerCta = B == 8 ? 4 : 1;  // 256 threads for B = 8 / 16, 1024 for B = 32
  static constexpr int kThreads = kArea * kPerCta;
};

// tmp[u][c] = sum_r C[u][r] x[r][c];  Y[u][v] = sum_c tmp[u][c] C[v][c]   (dct.cpp:30-49)
template <int B>
__global__ void __launch_bounds__(Tb<B>::kThreads)
fwd64_kernel(const uint8_t* __restrict__ imgs, int64_t img_stride, int pitch, int rows, int cols, int64_t nblocks_total,
             double* __restrict__ Y) {
  constexpr int A = Tb<B>::kArea;
  __shared__ double s_x[Tb<B>::kPerCta][A], s_t[Tb<B>::kPerCta][A];
  const double* C = basis_dev<B>();
  const int g = threadIdx.x / A, e = threadIdx.x % A;
  const int64_t blk = (int64_t)blockIdx.x * Tb<B>::kPerCta + g;
  const bool on = blk < nblocks_total;
  const int64_t nb = (int64_t)rows * cols;
  if (on) {
    const int64_t img = blk / nb, b = blk % nb;
    const int br = (int)(b / cols), bc = (int)(b % cols);
    const int r = e / B, c = e % B;
    s_x[g][e] = (double)imgs[img * img_stride + (int64_t)(br * B + r) * pitch + bc * B + c];
  }
  __syncthreads();
  if (on) {
    const int u = e / B, c = e % B;
    double t = 0.0;
    for (int r = 0; r < B; ++r) t = __dadd_rn(t, __dmul_rn(C[u * B + r], s_x[g][r * B + c]));
    s_t[g][e] = t;
  }
  __syncthreads();
  if (on) {
    const int u = e / B, v = e % B;
    double acc = 0.0;
    for (int c = 0; c < B; ++c) acc = __dadd_rn(acc, __dmul_rn(s_t[g][u * B + c], C[v * B + c]));
    Y[blk * A + e] = acc;
  }
}

// tmp[r][v] = sum_u C[u][r] Y[u][v];  X[r][c] = sum_v tmp[r][v] C[v][c]   (dct.cpp:52-79)
template <int B>
__global__ void __launch_bounds__(Tb<B>::kThreads)
inv64_kernel(const double* __restrict__ Y, int rows, int cols, int64_t nblocks_total, double* __restrict__ out,
             int64_t out_stride, int out_pitch) {
  constexpr int A = Tb<B>::kArea;
  __shared__ double s_y[Tb<B>::kPerCta][A], s_t[Tb<B>::kPerCta][A];
  const double* C = basis_dev<B>();
  const int g = threadIdx.x / A, e = threadIdx.x % A;
  const int64_t blk = (int64_t)blockIdx.x * Tb<B>::kPerCta + g;
  const bool on = blk < nblocks_total;
  if (on) s_y[g][e] = Y[blk * A + e];
  __syncthreads();
  if (on) {
    const int r = e / B, v = e % B;
    double t = 0.0;
    for (int u = 0; u < B; ++u) t = __dadd_rn(t, __dmul_rn(C[u * B + r], s_y[g][u * B + v]));
    s_t[g][e] = t;
  }
  __syncthreads();
  if (on) {
    const int64_t nb = (int64_t)rows * cols;
    const int64_t img = blk / nb, b = blk % nb;
    const int br = (int)(b / cols), bc = (int)(b % cols);
    const int r = e / B, c = e % B;
    double x = 0.0;
    for (int v = 0; v < B; ++v) x = __dadd_rn(x, __dmul_rn(s_t[g][r * B + v], C[v * B + c]));
    out[img * out_stride + (int64_t)(br * B + r) * out_pitch + bc * B + c] = x;
  }
}

// THB: keep the m = counts[b] best of each block: better(a, b) = |a| > |b|, ties -> lower zigzag rank
template <int B>
__global__ void __launch_bounds__(Tb<B>::kThreads)
thb_select_kernel(double* __restrict__ Y, int64_t nblocks_total, int64_t nb, int64_t m_target, int cap) {
  constexpr int A = Tb<B>::kArea;
  __shared__ double s_m[Tb<B>::kPerCta][A];
  const unsigned short* rank = zigzag_rank_dev<B>();
  const int g = threadIdx.x / A, e = threadIdx.x % A;
  const int64_t blk = (int64_t)blockIdx.x * Tb<B>::kPerCta + g;
  const bool on = blk < nblocks_total;
  double me = 0.0;
  if (on) {
    me = fabs(Y[blk * A + e]);
    s_m[g][e] = me;
  }
  __syncthreads();
  if (!on) return;
  const int b = (int)(blk % nb);
  // balanced_counts (metrics.cpp:50-59)
  const int64_t per = m_target / nb, extra = m_target % nb;
  const int64_t mm = per + (b < extra ? 1 : 0);
  const int m = (int)(mm < cap ? mm : cap);
  const int rk = rank[e];
  int pos = 0;
  for (int j = 0; j < A; ++j) {
    const double o = s_m[g][j];
    pos += (o > me || (o == me && rank[j] < rk)) ? 1 : 0;
  }
  if (pos >= m) Y[blk * A + e] = 0.0;
}

// ---- THI: per image top-M over all coefficients -----------------------------------------
constexpr int kThiThreads = 1024;

__device__ __forceinline__ unsigned long long mag_key(double v) {  // |v| >= 0: its bits order as u64
  return (unsigned long long)__double_as_longlong(fabs(v));
}

// CTA-wide: find the digit bin (scanning from the top for kDesc, from 0 otherwise) where the
// running count reaches `need`; returns the digit, sets `before` = count strictly beyond it.
template <bool kDesc>
__device__ int pick_bin(const unsigned int* hist, long long need, long long& before, int* s_pick, long long* s_before) {
  if (threadIdx.x == 0) {
    long long cum = 0;
    int pick = 0;
    for (int i = 0; i < 256; ++i) {
      const int d = kDesc ? 255 - i : i;
      if (cum + hist[d] >= need) {
        pick = d;
        break;
      }
      cum += hist[d];
    }
    *s_pick = pick;
    *s_before = cum;
  }
  __syncthreads();
  before = *s_before;
  return *s_pick;
}

// One CTA per image. better(a, b): |a| > |b|, then lower zigzag rank, then lower block
// (metrics.cpp:163-170): select the top M, zero the rest, count the kept ones per block.
template <int B>
__global__ void __launch_bounds__(kThiThreads)
thi_select_kernel(double* __restrict__ Yall, int64_t nb, int64_t m_target, int* __restrict__ counts_all) {
  constexpr int A = Tb<B>::kArea;
  __shared__ unsigned int hist[256];
  __shared__ int s_pick;
  __shared__ long long s_before;
  const int64_t E = nb * A;
  double* Y = Yall + (int64_t)blockIdx.x * E;
  int* counts = counts_all + (int64_t)blockIdx.x * nb;
  const unsigned short* rank = zigzag_rank_dev<B>();
  const long long M = (long long)(m_target < E ? m_target : E);
  for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) counts[b] = 0;
  // 1) the M-th largest |c| (exact bits), 8 digits of 8 bits from the top
  unsigned long long prefix = 0;
  long long need = M;
  for (int pass = 0; pass < 8 && M > 0 && M < E; ++pass) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const int sh = 56 - 8 * pass;
    for (int64_t i = threadIdx.x; i < E; i += blockDim.x) {
      const unsigned long long k = mag_key(Y[i]);
      if (pass == 0 || (k >> (sh + 8)) == prefix) atomicAdd(&hist[(k >> sh) & 0xffu], 1u);
    }
    __syncthreads();
    long long above;
    const int d = pick_bin<true>(hist, need, above, &s_pick, &s_before);
    need -= above;
    prefix = (prefix << 8) | (unsigned long long)d;
    __syncthreads();
  }
  const unsigned long long t = prefix;  // threshold magnitude bits (when 0 < M < E)
  // 2) among |c| == t take the `need` smallest tie keys (rank * nb + block), 4 digits of 8 bits
  unsigned int tprefix = 0;
  long long need2 = need;
  long long ties = 0;
  if (M > 0 && M < E) {
    for (int pass = 0; pass < 4; ++pass) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      const int sh = 24 - 8 * pass;
      for (int64_t i = threadIdx.x; i < E; i += blockDim.x) {
        if (mag_key(Y[i]) != t) continue;
        const unsigned int k2 = (unsigned int)rank[i % A] * (unsigned int)nb + (unsigned int)(i / A);
        if (pass == 0 || (k2 >> (sh + 8)) == tprefix) atomicAdd(&hist[(k2 >> sh) & 0xffu], 1u);
      }
      __syncthreads();
      if (pass == 0 && threadIdx.x == 0) {
        long long tot = 0;
        for (int i = 0; i < 256; ++i) tot += hist[i];
        s_before = tot;
      }
      __syncthreads();
      if (pass == 0) ties = s_before;
      __syncthreads();
      long long below;
      const int d = pick_bin<false>(hist, need2, below, &s_pick, &s_before);
      need2 -= below;
      tprefix = (tprefix << 8) | (unsigned int)d;
      __syncthreads();
    }
  }
  (void)ties;
  // 3) keep: |c| > t, or |c| == t with tie key <= the selected one; zero the rest, count per block
  for (int64_t i = threadIdx.x; i < E; i += blockDim.x) {
    bool keep;
    if (M >= E) {
      keep = true;
    } else if (M == 0) {
      keep = false;
    } else {
      const unsigned long long k = mag_key(Y[i]);
      const unsigned int k2 = (unsigned int)rank[i % A] * (unsigned int)nb + (unsigned int)(i / A);
      keep = k > t || (k == t && k2 <= tprefix);
    }
    if (keep) atomicAdd(counts + i / A, 1);
    else Y[i] = 0.0;
  }
}

template <int B>
static int threshold_decode(Ctx* ctx, const uint8_t* imgs, int64_t img_stride, int pitch, int rows, int cols, int n,
                            int64_t m_target, bool global, int* counts, double* out, int64_t out_stride, int out_pitch,
                            double* Y, int chunk, cudaStream_t s) {
  const int64_t nb = (int64_t)rows * cols;
  for (int done = 0; done < n; done += chunk) {
    const int cnt = std::min(chunk, n - done);
    const int64_t tot = (int64_t)cnt * nb;
    const unsigned grid = (unsigned)((tot + Tb<B>::kPerCta - 1) / Tb<B>::kPerCta);
    fwd64_kernel<B><<<grid, Tb<B>::kThreads, 0, s>>>(imgs + (int64_t)done * img_stride, img_stride, pitch, rows, cols,
                                                     tot, Y);
    if (global) {
      thi_select_kernel<B><<<cnt, kThiThreads, 0, s>>>(Y, nb, m_target, counts + (int64_t)done * nb);
    } else {
      thb_select_kernel<B><<<grid, Tb<B>::kThreads, 0, s>>>(Y, tot, nb, m_target, B * B);
    }
    inv64_kernel<B><<<grid, Tb<B>::kThreads, 0, s>>>(Y, rows, cols, tot, out + (int64_t)done * out_stride, out_stride,
                                                     out_pitch);
    ctx->launches += 3;
  }
  if (!global) {  // THB counts are balanced_counts (metrics.cpp:178-193)
    std::vector<int> h(nb);
    const int64_t per = m_target / nb, extra = m_target % nb;
    for (int64_t b = 0; b < nb; ++b) h[b] = (int)std::min<int64_t>(per + (b < extra ? 1 : 0), (int64_t)B * B);
    for (int i = 0; i < n; ++i) {
      cudaError_t e = cudaMemcpyAsync(counts + (int64_t)i * nb, h.data(), nb * 4, cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return cuda_status(e, "thb counts");
    }
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "thb counts");
  }
  return cuda_status(cudaGetLastError(), "threshold decode launch");
}

int launch_threshold_decode(Ctx* ctx, int block, const uint8_t* imgs, int64_t img_stride, int pitch, int rows, int cols,
                            int n, int64_t m_target, bool global, int* counts, double* out, int64_t out_stride,
                            int out_pitch, cudaStream_t s) {
  const int64_t per_img = (int64_t)rows * cols * block * block * 8;
  const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(n, ((int64_t)512 << 20) / std::max<int64_t>(per_img, 1)));
  int st;
  double* Y = static_cast<double*>(ctx_scratch(ctx, (size_t)chunk * per_img, s, &st));
  if (st) return st;
  const int kt = ktimer_begin(ctx, s, global ? "thi" : "thb");
  if (block == 8)
    st = threshold_decode<8>(ctx, imgs, img_stride, pitch, rows, cols, n, m_target, global, counts, out, out_stride,
                             out_pitch, Y, chunk, s);
  else if (block == 16)
    st = threshold_decode<16>(ctx, imgs, img_stride, pitch, rows, cols, n, m_target, global, counts, out, out_stride,
                              out_pitch, Y, chunk, s);
  else if (block == 32)
    st = threshold_decode<32>(ctx, imgs, img_stride, pitch, rows, cols, n, m_target, global, counts, out, out_stride,
                              out_pitch, Y, chunk, s);
  else
    st = set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  ktimer_end(ctx, s, kt);
  return st;
}

}  // namespace abcs_b200

using namespace abcs_b200;

extern "C" int abcs_threshold_decode_batch(abcs_ctx* c, const abcs_sensing_config* cfg, const uint8_t* d_images,
                                           int64_t image_stride, int32_t pitch, int32_t height, int32_t width,
                                           int32_t n, int32_t global, int32_t* d_counts, double* d_out,
                                           int64_t out_stride, int32_t out_pitch, void* stream) {
  if (!c) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null context");
  if (!cfg || n < 0 || height < 1 || width < 1 || (n > 0 && (!d_images || !d_counts || !d_out)))
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  // SensingConfig::validate + make_grid (sensing.cpp:32-39, image.cpp:106-116)
  if (cfg->block < 2 || cfg->block > 255) return set_error(ABCS_ERR_INVALID_ARGUMENT, "block size must be in [2, 255]");
  if (cfg->cr_num == 0 || cfg->cr_den == 0) return set_error(ABCS_ERR_INVALID_ARGUMENT, "C_R must be positive");
  if (cfg->cr_num > cfg->cr_den) return set_error(ABCS_ERR_INVALID_ARGUMENT, "C_R must be in (0, 1]");
  if (cfg->block > height || cfg->block > width)
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "block size exceeds image dimensions");
  if (cfg->block != 8 && cfg->block != 16 && cfg->block != 32)
    return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  const int rows = height / cfg->block, cols = width / cfg->block;
  if (out_pitch < cols * cfg->block) return set_error(ABCS_ERR_INVALID_ARGUMENT, "output pitch smaller than the image");
  if (n == 0) return ABCS_OK;
  const unsigned long long N = (unsigned long long)rows * cols * cfg->block * cfg->block;
  const int64_t m_target = (int64_t)((unsigned long long)cfg->cr_num * N / cfg->cr_den);  // sensing.cpp:41-44
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  return launch_threshold_decode(ctx, cfg->block, d_images, image_stride, pitch, rows, cols, n, m_target, global != 0,
                                 d_counts, d_out, out_stride, out_pitch, reinterpret_cast<cudaStream_t>(stream));
}
