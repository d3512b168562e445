// decode_idct (recon.cpp:109-117) == SensingOperator::adjoint
// (operators.cpp:50-76): per block, scatter the zigzag prefix into a zero
// B x B coefficient tile, inverse DCT, write the pixels. Count-0 blocks decode
// to zeros. Plus the per-image offsets scan (SensingOperator ctor,
// operators.cpp:8-21) with the payload-length / count validation.
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "internal.h"

namespace abcs_b200 {

constexpr int kDecodeThreads = 256;
constexpr int kScanThreads = 1024;

__global__ void __launch_bounds__(kScanThreads)
offsets_kernel(int nb, int block_area, const uint16_t* __restrict__ counts, int32_t* __restrict__ offsets,
               const int64_t* __restrict__ payload_len, int32_t* __restrict__ error) {
  using Scan = cub::BlockScan<int, kScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int bad;
  const int v = blockIdx.x, tid = threadIdx.x;
  if (tid == 0) bad = 0;
  __syncthreads();
  int running = 0;
  for (int start = 0; start < nb; start += kScanThreads) {
    const int i = start + tid;
    const int c = i < nb ? counts[(int64_t)v * nb + i] : 0;
    if (c > block_area) bad = 1;  // "SensingOperator: count exceeds B^2"
    int ex, total;
    Scan(tmp).ExclusiveSum(c, ex, total);
    __syncthreads();
    if (i < nb && offsets) offsets[(int64_t)v * nb + i] = (int32_t)(running + ex);
    running += total;
  }
  __syncthreads();
  if (tid == 0 && error) {
    int st = ABCS_OK;
    if (bad) st = ABCS_ERR_INVALID_ARGUMENT;
    else if (payload_len && payload_len[v] != (int64_t)running) st = ABCS_ERR_FORMAT;  // recon.cpp:111-113
    error[v] = st;
  }
}

template <int B>
__global__ void __launch_bounds__(kDecodeThreads)
decode_kernel(int rows, int cols, int n, const uint16_t* __restrict__ counts, const int32_t* __restrict__ offsets,
              const float* __restrict__ payload, int64_t payload_stride, float* __restrict__ out,
              int64_t out_stride, int out_pitch, bool aligned) {
  constexpr int GPB = kDecodeThreads / B;
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
  Tile<B> t{s_tile + g * Tile<B>::kFloats};
  const int cnt = counts[gid];
  float x[B], y[B];
  float* dst = out + img * out_stride + (int64_t)(br * B + lane) * out_pitch + (int64_t)bc * B;
  if (cnt == 0) {  // operators.cpp:63: block stays zero
#pragma unroll
    for (int i = 0; i < B; ++i) x[i] = 0.f;
    store_row_f32<B>(dst, x, aligned);
    return;
  }
#pragma unroll
  for (int v = 0; v < B; ++v) t.at(lane, v) = 0.f;
  __syncwarp(group_mask<B>());
  const float* src = payload + img * payload_stride + offsets[gid];
  for (int k = lane; k < cnt; k += B) t.zz(s_zz[k]) = src[k];
  __syncwarp(group_mask<B>());
  // X = C^T Y C: columns first (lane v inverts column v over u), then rows.
#pragma unroll
  for (int u = 0; u < B; ++u) y[u] = t.at(u, lane);
  Dct<B>::inv(y, x);
#pragma unroll
  for (int r = 0; r < B; ++r) t.at(r, lane) = x[r];
  __syncwarp(group_mask<B>());
#pragma unroll
  for (int v = 0; v < B; ++v) y[v] = t.at(lane, v);
  Dct<B>::inv(y, x);
  store_row_f32<B>(dst, x, aligned);
}

int launch_offsets(Ctx* ctx, int32_t n_blocks, int32_t n, int32_t block, const uint16_t* counts, int32_t* offsets,
                   const int64_t* payload_len, int32_t* error, cudaStream_t s) {
  if (n == 0) return ABCS_OK;
  offsets_kernel<<<n, kScanThreads, 0, s>>>(n_blocks, block * block, counts, offsets, payload_len, error);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "offsets launch");
}

int launch_decode(Ctx* ctx, int32_t rows, int32_t cols, int32_t B, const uint16_t* counts, const int32_t* offsets,
                  const float* payload, int64_t payload_stride, int32_t n, float* out, int64_t out_stride,
                  int32_t out_pitch, cudaStream_t s) {
  const int64_t total = (int64_t)n * rows * cols;
  if (total == 0) return ABCS_OK;
  const int64_t gpc = kDecodeThreads / B;
  const unsigned grid = (unsigned)((total + gpc - 1) / gpc);
  const bool al = ((uintptr_t)out % 16 == 0) && (out_stride % 4 == 0) && (out_pitch % 4 == 0);
  if (B == 16 && out_pitch % 2 == 0 && out_stride % 2 == 0 && ((uintptr_t)out % 8) == 0 &&
      mma16_supported(rows, cols, n)) {
    return launch_decode16(ctx, rows, cols, n, counts, offsets, payload, payload_stride, out, out_stride, out_pitch, s);
  }
  if (B == 8 && out_pitch % 2 == 0 && out_stride % 2 == 0 && ((uintptr_t)out % 8) == 0 &&
      mma16_supported(rows, cols, n)) {
    return launch_sense8(ctx, false, true, rows, cols, n, nullptr, 0, 0, counts, offsets, const_cast<float*>(payload),
                         payload_stride, out, out_stride, out_pitch, s);
  }
  const int kt = ktimer_begin(ctx, s, "decode");
  if (B == 8)
    decode_kernel<8><<<grid, kDecodeThreads, 0, s>>>(rows, cols, n, counts, offsets, payload, payload_stride, out,
                                                     out_stride, out_pitch, al);
  else if (B == 16)
    decode_kernel<16><<<grid, kDecodeThreads, 0, s>>>(rows, cols, n, counts, offsets, payload, payload_stride, out,
                                                      out_stride, out_pitch, al);
  else if (B == 32)
    decode_kernel<32><<<grid, kDecodeThreads, 0, s>>>(rows, cols, n, counts, offsets, payload, payload_stride, out,
                                                      out_stride, out_pitch, al);
  else
    return set_error(ABCS_ERR_UNSUPPORTED, "device path supports block sizes 8, 16, 32");
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "decode launch");
}

}  // namespace abcs_b200
