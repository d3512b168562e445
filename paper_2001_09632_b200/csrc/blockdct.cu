// BlockDct::forward / inverse (dct.cpp:9-79) as a batched C-ABI entry: any block size >= 1, fp64,
// bit-identical to the reference. The basis is built on the host with the reference's expression
// (glibc cos, dct.cpp:12-19) and every sum runs in the reference's order with separate rounded
// multiply and add (no FMA contraction), so each coefficient / pixel equals the reference's bits.
// Two launches per call: stage 1 (thread per (block, u, c) / (block, r, v)) into scratch, stage 2
// (thread per output). This is the drop-in's dct.hpp; the hot path uses the fused fp32 kernels.
#include <cmath>
#include <vector>

#include "internal.h"

namespace abcs_b200 {

// forward: tmp[u][c] = sum_r C[u][r] X[r][c]   (r ascending from 0.0, dct.cpp:30-36)
// inverse: tmp[r][v] = sum_u C[u][r] Y[u][v]   (u ascending, dct.cpp:58-64)
__global__ void blockdct_stage1(int B, int inverse, const double* __restrict__ C, const double* __restrict__ in,
                                double* __restrict__ tmp, int64_t total) {
  const int64_t n2 = (int64_t)B * B;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = i / n2;
    const int e = (int)(i - blk * n2), a = e / B, col = e % B;  // (u, c) forward, (r, v) inverse
    const double* x = in + blk * n2;
    double t = 0.0;
    if (!inverse) {
      for (int r = 0; r < B; ++r) t = __dadd_rn(t, __dmul_rn(C[a * B + r], x[r * B + col]));
    } else {
      for (int u = 0; u < B; ++u) t = __dadd_rn(t, __dmul_rn(C[u * B + a], x[u * B + col]));
    }
    tmp[i] = t;
  }
}

// forward: Y[u][v] = sum_c tmp[u][c] C[v][c]   (c ascending, dct.cpp:38-48)
// inverse: X[r][c] = sum_v tmp[r][v] C[v][c]   (v ascending, dct.cpp:66-76)
__global__ void blockdct_stage2(int B, int inverse, const double* __restrict__ C, const double* __restrict__ tmp,
                                double* __restrict__ out, int64_t total) {
  const int64_t n2 = (int64_t)B * B;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = i / n2;
    const int e = (int)(i - blk * n2), a = e / B, b = e % B;
    const double* t = tmp + blk * n2 + (int64_t)a * B;
    double acc = 0.0;
    if (!inverse) {
      for (int c = 0; c < B; ++c) acc = __dadd_rn(acc, __dmul_rn(t[c], C[b * B + c]));
    } else {
      for (int v = 0; v < B; ++v) acc = __dadd_rn(acc, __dmul_rn(t[v], C[v * B + b]));
    }
    out[i] = acc;
  }
}

}  // namespace abcs_b200

using namespace abcs_b200;

extern "C" int abcs_block_dct_f64(abcs_ctx* c, int32_t size, int32_t inverse, const double* d_in, double* d_out,
                                  int64_t n_blocks, void* stream) {
  if (!c) return set_error(ABCS_ERR_INVALID_ARGUMENT, "null context");
  if (size < 1) return set_error(ABCS_ERR_INVALID_ARGUMENT, "BlockDct: size must be >= 1");
  if (n_blocks < 0 || (n_blocks > 0 && (!d_in || !d_out))) return set_error(ABCS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n_blocks == 0) return ABCS_OK;
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int B = size;
  const int64_t n2 = (int64_t)B * B, total = n2 * n_blocks;
  constexpr double kPi = 3.14159265358979323846;  // == std::numbers::pi (the same double)
  // basis_[k*B+n] = scale * cos(pi * (2n + 1) * k / (2B)), the reference's expression and order
  std::vector<double> basis((size_t)n2);
  const double n0 = std::sqrt(1.0 / B), nk = std::sqrt(2.0 / B);
  for (int k = 0; k < B; ++k) {
    const double scale = (k == 0) ? n0 : nk;
    for (int n = 0; n < B; ++n)
      basis[(size_t)k * B + n] = scale * std::cos(kPi * (2.0 * n + 1.0) * k / (2.0 * B));
  }
  int st = ABCS_OK;
  char* scratch = static_cast<char*>(ctx_scratch(ctx, (size_t)(n2 + total) * sizeof(double), s, &st));
  if (st) return st;
  double* d_basis = reinterpret_cast<double*>(scratch);
  double* d_tmp = d_basis + n2;
  cudaError_t e = cudaMemcpyAsync(d_basis, basis.data(), (size_t)n2 * sizeof(double), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_status(e, "block dct basis upload");
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)ctx->sm_count * 16);
  blockdct_stage1<<<grid, 256, 0, s>>>(B, inverse ? 1 : 0, d_basis, d_in, d_tmp, total);
  blockdct_stage2<<<grid, 256, 0, s>>>(B, inverse ? 1 : 0, d_basis, d_tmp, d_out, total);
  ctx->launches += 2;
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "block dct launch");
  // the host basis vector is released on return: the upload must have completed
  return cuda_status(cudaStreamSynchronize(s), "block dct sync");
}
