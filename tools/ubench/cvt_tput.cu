// Issue-throughput microbenchmark of the ops in the fp16 hi/lo split on sm_100a:
// cycles per warp-instruction per SMSP with 8 independent chains per thread, 16 warps/SM.
#include <cstdio>
#include <cuda_fp16.h>

#define CHAINS 8
#define ITERS 4096

__global__ void k_f2fp(unsigned* out, float seed, long long* cyc) {
  float a[CHAINS];
  unsigned r[CHAINS];
  for (int i = 0; i < CHAINS; ++i) { a[i] = seed + threadIdx.x + i; r[i] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      unsigned h;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(a[i]), "f"(a[i]));
      r[i] ^= h;
      a[i] = __int_as_float(__float_as_int(a[i]) ^ (h & 1));
    }
  }
  long long t1 = clock64();
  unsigned x = 0;
  for (int i = 0; i < CHAINS; ++i) x ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_h2f(unsigned* out, float seed, long long* cyc) {
  unsigned h[CHAINS];
  float acc[CHAINS];
  for (int i = 0; i < CHAINS; ++i) { h[i] = 0x3c003c00u + threadIdx.x + i; acc[i] = 0.f; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      float lo, hi;
      asm volatile("{.reg .f16 l, u;\n mov.b32 {l, u}, %2;\n cvt.f32.f16 %0, l;\n cvt.f32.f16 %1, u;}"
                   : "=f"(lo), "=f"(hi) : "r"(h[i]));
      acc[i] += lo;
      h[i] ^= __float_as_uint(hi) & 1u;
    }
  }
  long long t1 = clock64();
  unsigned x = 0;
  for (int i = 0; i < CHAINS; ++i) x ^= __float_as_uint(acc[i]) ^ h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_lop(unsigned* out, float seed, long long* cyc) {
  unsigned v[CHAINS];
  for (int i = 0; i < CHAINS; ++i) v[i] = threadIdx.x * 7 + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[i]) : "r"(it), "r"(i));
  }
  long long t1 = clock64();
  unsigned x = 0;
  for (int i = 0; i < CHAINS; ++i) x ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_hmma(unsigned* out, float seed, long long* cyc) {
  float d[CHAINS / 2][4];
  unsigned a0 = 0x3c003c00u + threadIdx.x, b0 = 0x3c003c00u;
  for (int i = 0; i < CHAINS / 2; ++i) d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS / 2; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                   : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3]) : "r"(a0), "r"(b0));
  }
  long long t1 = clock64();
  unsigned x = 0;
  for (int i = 0; i < CHAINS / 2; ++i) x ^= __float_as_uint(d[i][0] + d[i][3]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <class K>
void run(const char* name, K kern, int ops_per_iter_per_thread) {
  unsigned* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 8);
  kern<<<148, 512>>>(out, 1.f, cyc);
  cudaDeviceSynchronize();
  kern<<<148, 512>>>(out, 1.f, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // 512 threads = 16 warps per SM = 4 warps per SMSP
  const double warp_instr_per_smsp = 4.0 * ITERS * ops_per_iter_per_thread;
  printf("%-26s %8.3f cycles per warp-instruction per SMSP\n", name, (double)c / warp_instr_per_smsp);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run("F2FP (cvt.rn.f16x2.f32)", k_f2fp, CHAINS);
  run("cvt.f32.f16 x2 (HADD2.F32)", k_h2f, 2 * CHAINS);
  run("LOP3", k_lop, CHAINS);
  run("HMMA.16816.F32", k_hmma, CHAINS / 2);
  return 0;
}
