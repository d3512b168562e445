// FP32 issue rates on sm_100a for the CUDA-core transform design: scalar FADD/FFMA (register and
// immediate forms), packed f32x2 add/fma, FMNMX, and mixes. 8 independent chains per thread,
// 32 warps per SM. Prints cycles per warp-instruction per SMSP (1.0 = one issue per clock).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ void op(int kind, float& a, float& b, float c, float d) {
  switch (kind) {
    case 0: asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a) : "f"(c)); break;
    case 1: asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a) : "f"(c), "f"(d)); break;
    case 2: asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFF0, %1;" : "+f"(a) : "f"(c)); break;
    case 3: asm volatile("mul.rn.f32 %0, %0, 0f3F7FFFF0;" : "+f"(a)); break;
    case 4: asm volatile("{.reg .b64 x, y; mov.b64 x, {%0,%1}; mov.b64 y, {%2,%3}; add.rn.f32x2 x, x, y; mov.b64 {%0,%1}, x;}"
                         : "+f"(a), "+f"(b) : "f"(c), "f"(d)); break;
    case 5: asm volatile("{.reg .b64 x, y; mov.b64 x, {%0,%1}; mov.b64 y, {%2,%3}; fma.rn.f32x2 x, x, y, y; mov.b64 {%0,%1}, x;}"
                         : "+f"(a), "+f"(b) : "f"(c), "f"(d)); break;
    case 6: asm volatile("min.f32 %0, %0, %1;" : "+f"(a) : "f"(c)); break;
    case 7: asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFF0, %1;" : "+f"(a) : "f"(c));
            asm volatile("min.f32 %0, %0, %1;" : "+f"(b) : "f"(d)); break;
    case 8: asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a) : "f"(c));
            asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFF0, %1;" : "+f"(b) : "f"(d)); break;
    case 9: asm volatile("{.reg .b64 x, y; mov.b64 x, {%0,%1}; mov.b64 y, {%2,%3}; add.rn.f32x2 x, x, y; mov.b64 {%0,%1}, x;}"
                         : "+f"(a), "+f"(b) : "f"(c), "f"(d));
            asm volatile("min.f32 %0, %0, %1;" : "+f"(c) : "f"(d)); break;
    case 10: asm volatile("{.reg .b64 x, y; mov.b64 x, {%0,%1}; mov.b64 y, {%2,%3}; mul.rn.f32x2 x, x, y; mov.b64 {%0,%1}, x;}"
                         : "+f"(a), "+f"(b) : "f"(c), "f"(d)); break;
  }
}

template <int KIND>
__global__ void k(float* out, int iters, float seed) {
  float a[8], b[8];
  float c = seed * 1e-9f, d = seed * 2e-9f;
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = seed + i; b[i] = seed - i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) op(KIND, a[i], b[i], c, d);
  }
  float s = c + d;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + b[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND>
void run(const char* name, int instrs_per_op, float* out, int sms) {
  const int iters = 8192, blocks = sms * 4, threads = 256;
  k<KIND><<<blocks, threads>>>(out, 16, 1.f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<KIND><<<blocks, threads>>>(out, iters, 1.f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double clk_ghz = 1.965;
  const double winstr_per_smsp = (double)iters * 8 * instrs_per_op * (blocks * threads / 32) / (sms * 4.0);
  printf("%-28s %.3f ms  %.2f cycles per warp-instruction per SMSP (at %.3f GHz)\n", name, ms,
         ms * 1e-3 * clk_ghz * 1e9 / winstr_per_smsp, clk_ghz);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sms * 4 * 256 * sizeof(float));
  run<0>("FADD reg", 1, out, sms);
  run<1>("FFMA reg", 1, out, sms);
  run<2>("FFMA imm", 1, out, sms);
  run<3>("FMUL imm", 1, out, sms);
  run<4>("FADD2 (add.f32x2)", 1, out, sms);
  run<5>("FFMA2 (fma.f32x2)", 1, out, sms);
  run<10>("FMUL2 (mul.f32x2)", 1, out, sms);
  run<6>("FMNMX", 1, out, sms);
  run<7>("FFMA imm + FMNMX", 2, out, sms);
  run<8>("FADD + FFMA imm", 2, out, sms);
  run<9>("FADD2 + FMNMX", 2, out, sms);
  return 0;
}
