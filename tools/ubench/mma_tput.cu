// Legacy mma.sync issue cost on sm_100a: f16 m16n8k16 / m16n8k8 vs tf32 m16n8k8 (independent chains).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

template <int KIND>
__global__ void k(float* out, int iters, uint32_t seed) {
  float d[8][4];
  uint32_t a[4] = {seed, seed ^ 1u, seed ^ 2u, seed ^ 3u}, b0 = seed * 3u, b1 = seed * 5u;
  for (int c = 0; c < 8; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
      else if (KIND == 1)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                     : "r"(a[0]), "r"(a[1]), "r"(b0));
      else
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
  }
  float s = 0.f;
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND>
void run(const char* name, float* out, int sms) {
  const int iters = 4096, blocks = sms * 4, threads = 256;
  k<KIND><<<blocks, threads>>>(out, 16, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<KIND><<<blocks, threads>>>(out, iters, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double mma_per_smsp = (double)iters * 8 * (blocks * threads / 32) / (sms * 4.0);
  printf("%s: %.3f ms, %.2f cycles/mma/SMSP at %d MHz (nominal)\n", name, ms, ms * 1e-3 * clk * 1e3 / mma_per_smsp, clk / 1000);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sms * 4 * 256 * sizeof(float));
  run<0>("f16 m16n8k16", out, sms);
  run<1>("f16 m16n8k8 ", out, sms);
  run<2>("tf32 m16n8k8", out, sms);
  return 0;
}
