// tcgen05 (UMMA, accumulators in TMEM) forward 16x16 block DCT of 8 blocks (one 16 x 128 u8
// strip) with the fp16 hi/lo split, checked against an fp64 host DCT. A feasibility probe for
// moving the block transforms off legacy mma.sync.
//
//   stage 1: D1[(b,c)][u | 16+u] = sum_r X_b[r][c] * {Ch, Cl}[u][r]      M=128 N=32 K=16
//   stage 2: D2[(b,u)][v | 16+v] = sum_c {Qh, Ql}_b[u][c] * {Ch, Cl}[v][c] M=128 N=32 K=32
// Operands K-major, SWIZZLE_NONE: element (m, k) at (m%8)*16 + (m/8)*SBO + (k/8)*LBO + (k%8)*2.
#include <cuda_fp16.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(const void* base, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(base) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// kind::f16 instruction descriptor: D f32, A/B f16, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, int accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n" ::"l"((uint64_t)smem_u32(mbar)));
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, unsigned phase) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(mbar)),
      "r"(phase));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t kmaj(int m, int k, int sbo) { return (m & 7) * 16 + (m >> 3) * sbo + (k >> 3) * 128 + (k & 7) * 2; }

struct Smem {
  alignas(128) __half a1[128 * 16];  // 4 KB: m = (b, c), k = r;   SBO 256
  alignas(128) __half b1[32 * 16];   // 1 KB: n = u | 16+u, k = r;  SBO 256
  alignas(128) __half a2[128 * 32];  // 8 KB: m = (b, u), k = c | 16+c; SBO 512
  alignas(128) __half b2[32 * 32];   // 2 KB: n = v | 16+v, k = c | 16+c; SBO 512
  uint64_t mbar;
  uint32_t tmem_base;
};

// basis hi/lo from the host (fp32 basis split)
__global__ void __launch_bounds__(128) umma_dct_kernel(const uint8_t* __restrict__ img, int pitch, int n_strips,
                                                       const float* __restrict__ basis, float* __restrict__ out,
                                                       int reps) {
  extern __shared__ __align__(1024) unsigned char raw[];
  Smem& s = *reinterpret_cast<Smem*>(raw);
  const int t = threadIdx.x, warp = t >> 5;
  // B operands (constant): hi/lo split of the fp32 basis
  for (int i = t; i < 32 * 16; i += 128) {
    const int n = i / 16, k = i % 16;
    const float c = basis[(n & 15) * 16 + k];
    const __half h = __float2half_rn(c);
    const __half l = __float2half_rn(c - __half2float(h));
    *reinterpret_cast<__half*>(reinterpret_cast<char*>(s.b1) + kmaj(n, k, 256)) = n < 16 ? h : l;
  }
  for (int i = t; i < 32 * 32; i += 128) {
    const int n = i / 32, k = i % 32;
    const float c = basis[(n & 15) * 16 + (k & 15)];
    const __half h = __float2half_rn(c);
    const __half l = __float2half_rn(c - __half2float(h));
    *reinterpret_cast<__half*>(reinterpret_cast<char*>(s.b2) + kmaj(n, k, 512)) = n < 16 ? h : l;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(smem_u32(&s.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (t == 0) mbar_init(&s.mbar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = s.tmem_base;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  constexpr uint32_t kIdesc = idesc_f16(128, 32);
  unsigned phase = 0;
  for (int it = 0; it < reps; ++it)
    for (int strip = blockIdx.x; strip < n_strips; strip += gridDim.x) {
      const uint8_t* src = img + (int64_t)strip * 16 * pitch;
      // stage-1 A: thread t = (b, c) writes column c of block b (exact in fp16)
      {
        const int b = t >> 4, c = t & 15;
#pragma unroll
        for (int r = 0; r < 16; ++r)
          *reinterpret_cast<__half*>(reinterpret_cast<char*>(s.a1) + kmaj(t, r, 256)) =
              __ushort2half_rn(src[r * pitch + b * 16 + c]);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (t == 0) {
        umma_f16(tmem, sdesc(s.a1, 128, 256), sdesc(s.b1, 128, 256), kIdesc, 0);
        umma_commit(&s.mbar);
      }
      mbar_wait(&s.mbar, phase);
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      // D1 row (b, c): Q_b[u][c] = hi + lo halves; split and scatter into stage-2 A (m = (b, u), k = c | 16+c)
      {
        float v[32];
        tmem_ld32(tmem + lane_base, v);
        const int b = t >> 4, c = t & 15;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const float q = v[u] + v[16 + u];
          const __half h = __float2half_rn(q);
          const __half l = __float2half_rn(q - __half2float(h));
          char* base = reinterpret_cast<char*>(s.a2);
          *reinterpret_cast<__half*>(base + kmaj(b * 16 + u, c, 512)) = h;
          *reinterpret_cast<__half*>(base + kmaj(b * 16 + u, 16 + c, 512)) = l;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (t == 0) {
        umma_f16(tmem + 32, sdesc(s.a2, 128, 512), sdesc(s.b2, 128, 512), kIdesc, 0);
        umma_f16(tmem + 32, sdesc(reinterpret_cast<char*>(s.a2) + 256, 128, 512),
                 sdesc(reinterpret_cast<char*>(s.b2) + 256, 128, 512), kIdesc, 1);
        umma_commit(&s.mbar);
      }
      mbar_wait(&s.mbar, phase);
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      {
        float v[32];
        tmem_ld32(tmem + lane_base + 32, v);
        const int b = t >> 4, u = t & 15;
        if (it == reps - 1) {
          float* o = out + ((int64_t)strip * 8 + b) * 256 + u * 16;
#pragma unroll
          for (int w = 0; w < 16; ++w) o[w] = v[w] + v[16 + w];  // Y_b[u][v]
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tmem));
}

int main(int argc, char** argv) {
  const int n_strips = argc > 1 ? atoi(argv[1]) : 4096, reps = argc > 2 ? atoi(argv[2]) : 1;
  const int W = 128, H = 16 * n_strips;
  std::vector<uint8_t> img((size_t)W * H);
  srand(1);
  for (auto& p : img) p = (uint8_t)(rand() & 255);
  std::vector<float> basis(256);
  std::vector<double> Cd(256);
  for (int k = 0; k < 16; ++k)
    for (int n = 0; n < 16; ++n) {
      Cd[k * 16 + n] = (k ? std::sqrt(2.0 / 16) : std::sqrt(1.0 / 16)) * std::cos(M_PI * (2 * n + 1) * k / 32.0);
      basis[k * 16 + n] = (float)Cd[k * 16 + n];
    }
  uint8_t* d_img;
  float *d_basis, *d_out;
  cudaMalloc(&d_img, img.size());
  cudaMalloc(&d_basis, 256 * 4);
  cudaMalloc(&d_out, (size_t)n_strips * 8 * 256 * 4);
  cudaMemcpy(d_img, img.data(), img.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(d_basis, basis.data(), 256 * 4, cudaMemcpyHostToDevice);
  const int smem = (int)sizeof(Smem) + 1024;
  cudaFuncSetAttribute(umma_dct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int per_sm = argc > 3 ? atoi(argv[3]) : 8;  // CTAs per SM (1: the chain latency alone)
  const int grid = std::min(n_strips, sms * per_sm);
  umma_dct_kernel<<<grid, 128, smem>>>(d_img, W, n_strips, d_basis, d_out, 1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> out((size_t)n_strips * 8 * 256);
  cudaMemcpy(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int sI = 0; sI < std::min(n_strips, 64); ++sI)
    for (int b = 0; b < 8; ++b)
      for (int u = 0; u < 16; ++u)
        for (int v = 0; v < 16; ++v) {
          double y = 0;
          for (int r = 0; r < 16; ++r)
            for (int c = 0; c < 16; ++c)
              y += Cd[u * 16 + r] * (double)img[(size_t)(sI * 16 + r) * W + b * 16 + c] * Cd[v * 16 + c];
          maxerr = std::max(maxerr, std::fabs(y - out[((size_t)sI * 8 + b) * 256 + u * 16 + v]));
        }
  printf("max |Y - Y_fp64| over %d strips: %.3g\n", std::min(n_strips, 64), maxerr);
  cudaEvent_t a, z;
  cudaEventCreate(&a);
  cudaEventCreate(&z);
  cudaEventRecord(a);
  umma_dct_kernel<<<grid, 128, smem>>>(d_img, W, n_strips, d_basis, d_out, reps);
  cudaEventRecord(z);
  cudaEventSynchronize(z);
  float ms;
  cudaEventElapsedTime(&ms, a, z);
  printf("%d strips x %d reps, %d CTAs/SM: %.3f ms -> %.1f M blocks/s, %.2f us per strip per CTA (%s)\n", n_strips,
         reps, per_sm, ms, (double)n_strips * 8 * reps / ms / 1e3, ms * 1e3 * grid / ((double)n_strips * reps),
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
