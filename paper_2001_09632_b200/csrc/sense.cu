// Sensing kernels: phase-1 pre-measurements (BBV boundary probes, DD
// significance counts), ZZ balanced counts, and the per-block DCT +
// zigzag-prefix gather that produces the packed payload.
#include <cstdio>

#include "common.cuh"
#include "internal.h"

namespace abcs_b200 {

constexpr int kGatherThreads = 256;

// ---------------------------------------------------------------------------
// Per-block 2D DCT into a padded smem tile (group of B lanes, lane r = row r).
// Y = C X C^T: rows first (lane r transforms row r), then columns (lane v
// transforms column v). Leaves Y[u][v] at tile(u, v).
template <int B, typename InT>
__device__ __forceinline__ void block_dct(const InT* __restrict__ row_src, bool aligned, Tile<B> t) {
  float x[B], y[B];
  const int lane = threadIdx.x % B;
  if constexpr (sizeof(InT) == 1) {
    load_row_u8<B>(reinterpret_cast<const uint8_t*>(row_src), x, aligned);
  } else {
    load_row_f32<B>(reinterpret_cast<const float*>(row_src), x, aligned);
  }
  Dct<B>::fwd(x, y);
#pragma unroll
  for (int v = 0; v < B; ++v) t.at(lane, v) = y[v];
  __syncwarp(group_mask<B>());
#pragma unroll
  for (int u = 0; u < B; ++u) x[u] = t.at(u, lane);
  Dct<B>::fwd(x, y);
#pragma unroll
  for (int u = 0; u < B; ++u) t.at(u, lane) = y[u];
  __syncwarp(group_mask<B>());
}

// Exact fp64 coefficient Y[u][v] in the reference's operation order
// (dct.cpp:30-49: tmp[u][c] accumulated over r ascending from 0.0, then
// Y[u][v] accumulated over c ascending), no FMA contraction, reference basis.
template <int B>
__device__ __forceinline__ double exact_coef(const uint8_t* __restrict__ blk, int pitch, int flat) {
  const double* C = basis_dev<B>();
  const int u = flat / B, v = flat % B;
  double y = 0.0;
  for (int c = 0; c < B; ++c) {
    double t = 0.0;
    for (int r = 0; r < B; ++r) t = __dadd_rn(t, __dmul_rn(C[u * B + r], (double)blk[(size_t)r * pitch + c]));
    y = __dadd_rn(y, __dmul_rn(t, C[v * B + c]));
  }
  return y;
}

// Guard band for the fp32 significance test |c| > T: fp32 errors of the
// butterfly DCT on 8-bit blocks stay below 2e-3 (B<=16) / 1.2e-2 (B=32)
// (DESIGN.md "DD exactness"); comparisons closer than this are redone in fp64.
template <int B> struct GuardBand { static constexpr double v = (B >= 32) ? 6e-2 : 2e-2; };

// ---------------------------------------------------------------------------
// DD phase 1 (sense_dd, sensing.cpp:341-358): n_i = #{k < phase1 : |c_zz[k]| > T}.
template <int B>
__global__ void __launch_bounds__(kGatherThreads)
dd_weights_kernel(const uint8_t* __restrict__ imgs, int64_t img_stride, int pitch, int rows, int cols,
                  int n, bool aligned, int phase1, double T, uint32_t* __restrict__ weights) {
  constexpr int GPB = kGatherThreads / B;
  __shared__ float s_tile[GPB * Tile<B>::kFloats];
  __shared__ unsigned short s_zz[B * B];
  load_zigzag<B>(s_zz);
  __syncthreads();
  const int g = threadIdx.x / B, lane = threadIdx.x % B;
  const int64_t nb = (int64_t)rows * cols;
  const int64_t gid = (int64_t)blockIdx.x * GPB + g;
  if (gid >= (int64_t)n * nb) return;
  const int64_t img = gid / nb;
  const int bi = (int)(gid % nb), br = bi / cols, bc = bi % cols;
  const uint8_t* blk = imgs + img * img_stride + (int64_t)br * B * pitch + (int64_t)bc * B;
  Tile<B> t{s_tile + g * Tile<B>::kFloats};
  block_dct<B, uint8_t>(blk + (int64_t)lane * pitch, aligned, t);
  int sig = 0;
  for (int k = lane; k < phase1; k += B) {
    const int flat = s_zz[k];
    const double c = (double)t.zz(flat);
    const double d = fabs(c) - T;
    bool s;
    if (fabs(d) < GuardBand<B>::v) {
      s = fabs(exact_coef<B>(blk, pitch, flat)) > T;  // sensing.cpp:354, strict
    } else {
      s = d > 0.0;
    }
    sig += s ? 1 : 0;
  }
  sig = group_sum<B>(sig);
  if (lane == 0) weights[gid] = (uint32_t)sig;
}

// ---------------------------------------------------------------------------
// BBV phase 1 (bbv_measure, sensing.cpp:266-294): per block the sum of 4*n_S
// boundary |differences| (integer valued), and the unique probes as side data
// in block-major order: per probe j top, left, [bottom on the last block
// row], [right on the last block column].
__global__ void __launch_bounds__(256)
bbv_weights_kernel(const uint8_t* __restrict__ imgs, int64_t img_stride, int pitch, int rows, int cols,
                   int n, int B, int L, int offset, int per_side, int valid, uint32_t* __restrict__ weights,
                   float* __restrict__ side, int64_t side_stride, bool below) {
  // below: the block rows continue under this field (a shard strip whose buffer holds the next
  // strip's first pixel row after its last block row), so its last block row is not the image's
  const int64_t nb = (int64_t)rows * cols;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)n * nb) return;
  const int64_t img = gid / nb;
  const int bi = (int)(gid % nb), br = bi / cols, bc = bi % cols;
  const uint8_t* im = imgs + img * img_stride;
  const int r0 = br * B, c0 = bc * B;
  const bool last_row = (br + 1 == rows) && !below, last_col = (bc + 1 == cols);
  const int bottom = last_row ? r0 + B - 1 : r0 + B;
  const int right = (bc + 1 < cols) ? c0 + B : c0 + B - 1;
  float* out = nullptr;
  if (side) {
    out = side + img * side_stride +
          (int64_t)valid * (2LL * bi + (last_row ? bc : 0) + br);
  }
  uint32_t sum = 0;
  for (int j = 0; j < per_side; ++j) {
    const long long p = offset + (long long)j * L;  // 1-based (sensing.cpp:260-264)
    if (p < 1 || p + 1 > B) continue;
    const int a = (int)(p - 1), b = (int)p;
    const int top = abs((int)im[(int64_t)r0 * pitch + c0 + b] - (int)im[(int64_t)r0 * pitch + c0 + a]);
    const int left = abs((int)im[(int64_t)(r0 + b) * pitch + c0] - (int)im[(int64_t)(r0 + a) * pitch + c0]);
    const int bot = abs((int)im[(int64_t)bottom * pitch + c0 + b] - (int)im[(int64_t)bottom * pitch + c0 + a]);
    const int rgt = abs((int)im[(int64_t)(r0 + b) * pitch + right] - (int)im[(int64_t)(r0 + a) * pitch + right]);
    sum += (uint32_t)(top + left + bot + rgt);
    if (out) {
      *out++ = (float)top;
      *out++ = (float)left;
      if (last_row) *out++ = (float)bot;
      if (last_col) *out++ = (float)rgt;
    }
  }
  weights[gid] = sum;
}

// ---------------------------------------------------------------------------
// balanced_counts (sensing.cpp:181-190) + closed-form offsets.
__global__ void zz_counts_kernel(int64_t nb, int n, int64_t per, int64_t extra, int64_t cap,
                                 uint16_t* __restrict__ counts, int32_t* __restrict__ offsets) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)n * nb) return;
  const int64_t i = gid % nb;
  int64_t c = per + (i < extra ? 1 : 0);
  if (c > cap) c = cap;
  counts[gid] = (uint16_t)c;
  if (offsets) {
    const int64_t off = (per >= cap) ? i * cap : i * per + (i < extra ? i : extra);
    offsets[gid] = (int32_t)off;
  }
}

// ---------------------------------------------------------------------------
// gather_prefixes (sensing.cpp:192-227) / SensingOperator::forward
// (operators.cpp:23-48): DCT each block, write its first counts[i] zigzag
// coefficients at payload[offsets[i] ..]. InT = uint8_t (sense) or float (A x).
template <int B, typename InT>
__global__ void __launch_bounds__(kGatherThreads)
gather_kernel(const InT* __restrict__ imgs, int64_t img_stride, int pitch, int rows, int cols, int n,
              bool aligned, const uint16_t* __restrict__ counts, const int32_t* __restrict__ offsets,
              float* __restrict__ payload, int64_t payload_stride) {
  constexpr int GPB = kGatherThreads / B;
  __shared__ float s_tile[GPB * Tile<B>::kFloats];
  __shared__ unsigned short s_zz[B * B];
  load_zigzag<B>(s_zz);
  __syncthreads();
  const int g = threadIdx.x / B, lane = threadIdx.x % B;
  const int64_t nb = (int64_t)rows * cols;
  const int64_t gid = (int64_t)blockIdx.x * GPB + g;
  if (gid >= (int64_t)n * nb) return;
  const int cnt = counts[gid];
  if (cnt == 0) return;  // whole group agrees; nothing to emit (operators.cpp:36)
  const int64_t img = gid / nb;
  const int bi = (int)(gid % nb), br = bi / cols, bc = bi % cols;
  const InT* blk = imgs + img * img_stride + (int64_t)br * B * pitch + (int64_t)bc * B;
  Tile<B> t{s_tile + g * Tile<B>::kFloats};
  block_dct<B, InT>(blk + (int64_t)lane * pitch, aligned, t);
  float* dst = payload + img * payload_stride + offsets[gid];
  for (int k = lane; k < cnt; k += B) dst[k] = t.zz(s_zz[k]);
}

// ---------------------------------------------------------------------------
static bool aligned_rows(const void* base, int64_t img_stride_bytes, int64_t pitch_bytes, int row_bytes) {
  const int a = row_bytes >= 16 ? 16 : row_bytes;
  return ((uintptr_t)base % a) == 0 && (img_stride_bytes % a) == 0 && (pitch_bytes % a) == 0;
}

int launch_sense_weights(Ctx* ctx, const abcs_sense_plan& p, const uint8_t* imgs, int64_t img_stride,
                         int32_t pitch, int32_t n, uint32_t* weights, float* side, cudaStream_t s,
                         uint32_t* fix_scratch, bool bbv_below) {
  const int64_t total = (int64_t)n * p.n_blocks;
  if (total == 0) return ABCS_OK;
  if (p.algorithm_used == ABCS_ALGO_BBV) {
    const int threads = 256;
    const int64_t grid = (total + threads - 1) / threads;
    const int kt = ktimer_begin(ctx, s, "bbv_weights");
    bbv_weights_kernel<<<(unsigned)grid, threads, 0, s>>>(imgs, img_stride, pitch, p.rows, p.cols, n, p.block,
                                                          (int)p.bbv_stride, p.bbv_offset, p.bbv_per_side,
                                                          p.bbv_valid_probes, weights, side, p.side_per_image,
                                                          bbv_below);
    ktimer_end(ctx, s, kt);
  } else if (p.algorithm_used == ABCS_ALGO_DD && p.block == 16 && mma16_supported(p.rows, p.cols, n)) {
    return launch_sense16(ctx, 1, p.rows, p.cols, n, imgs, img_stride, pitch, p.dd_phase1, p.threshold, weights,
                          nullptr, nullptr, nullptr, 0, nullptr, 0, 0, s, fix_scratch);
  } else if (p.algorithm_used == ABCS_ALGO_DD) {
    const bool al = aligned_rows(imgs, img_stride, pitch, p.block);
    const int B = p.block;
    const int64_t groups_per_cta = kGatherThreads / B;
    const int64_t grid = (total + groups_per_cta - 1) / groups_per_cta;
    const int kt = ktimer_begin(ctx, s, "dd_weights");
    if (B == 8)
      dd_weights_kernel<8><<<(unsigned)grid, kGatherThreads, 0, s>>>(imgs, img_stride, pitch, p.rows, p.cols, n, al,
                                                                     p.dd_phase1, p.threshold, weights);
    else if (B == 16)
      dd_weights_kernel<16><<<(unsigned)grid, kGatherThreads, 0, s>>>(imgs, img_stride, pitch, p.rows, p.cols, n, al,
                                                                       p.dd_phase1, p.threshold, weights);
    else if (B == 32)
      dd_weights_kernel<32><<<(unsigned)grid, kGatherThreads, 0, s>>>(imgs, img_stride, pitch, p.rows, p.cols, n, al,
                                                                       p.dd_phase1, p.threshold, weights);
    else
      return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
    ktimer_end(ctx, s, kt);
  } else {
    return set_error(ABCS_ERR_INVALID_ARGUMENT, "zz sensing has no phase-1 weights");
  }
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "sense weights launch");
}

int launch_zz_counts(Ctx* ctx, const abcs_sense_plan& p, int32_t n, uint16_t* counts, int32_t* offsets,
                     cudaStream_t s) {
  const int64_t total = (int64_t)n * p.n_blocks;
  if (total == 0) return ABCS_OK;
  const int threads = 256;
  zz_counts_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(
      p.n_blocks, n, p.zz_per_block, p.zz_extra, (int64_t)p.block * p.block, counts, offsets);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "zz counts launch");
}

int launch_gather(Ctx* ctx, int32_t rows, int32_t cols, int32_t B, const uint8_t* imgs, const float* fimgs,
                  int64_t img_stride, int32_t pitch, int32_t n, const uint16_t* counts, const int32_t* offsets,
                  float* payload, int64_t payload_stride, cudaStream_t s) {
  const int64_t total = (int64_t)n * rows * cols;
  if (total == 0) return ABCS_OK;
  const int64_t gpc = kGatherThreads / B;
  const unsigned grid = (unsigned)((total + gpc - 1) / gpc);
  if (imgs && B == 8 && mma16_supported(rows, cols, n)) {
    return launch_sense8(ctx, true, false, rows, cols, n, imgs, img_stride, pitch, counts, offsets, payload,
                         payload_stride, nullptr, 0, 0, s);
  } else if (imgs && B == 16 && mma16_supported(rows, cols, n)) {
    return launch_sense16(ctx, 2, rows, cols, n, imgs, img_stride, pitch, 0, 0.0, nullptr, counts, offsets, payload,
                          payload_stride, nullptr, 0, 0, s);
  }
  const int kt = ktimer_begin(ctx, s, "gather");
  if (imgs) {
    const bool al = aligned_rows(imgs, img_stride, pitch, B);
    if (B == 8)
      gather_kernel<8, uint8_t><<<grid, kGatherThreads, 0, s>>>(imgs, img_stride, pitch, rows, cols, n, al, counts,
                                                                offsets, payload, payload_stride);
    else if (B == 16)
      gather_kernel<16, uint8_t><<<grid, kGatherThreads, 0, s>>>(imgs, img_stride, pitch, rows, cols, n, al, counts,
                                                                 offsets, payload, payload_stride);
    else if (B == 32)
      gather_kernel<32, uint8_t><<<grid, kGatherThreads, 0, s>>>(imgs, img_stride, pitch, rows, cols, n, al, counts,
                                                                 offsets, payload, payload_stride);
    else
      return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  } else {
    const bool al = aligned_rows(fimgs, img_stride * 4, (int64_t)pitch * 4, B * 4);
    if (B == 8)
      gather_kernel<8, float><<<grid, kGatherThreads, 0, s>>>(fimgs, img_stride, pitch, rows, cols, n, al, counts,
                                                              offsets, payload, payload_stride);
    else if (B == 16)
      gather_kernel<16, float><<<grid, kGatherThreads, 0, s>>>(fimgs, img_stride, pitch, rows, cols, n, al, counts,
                                                               offsets, payload, payload_stride);
    else if (B == 32)
      gather_kernel<32, float><<<grid, kGatherThreads, 0, s>>>(fimgs, img_stride, pitch, rows, cols, n, al, counts,
                                                               offsets, payload, payload_stride);
    else
      return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  }
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "gather launch");
}

}  // namespace abcs_b200
