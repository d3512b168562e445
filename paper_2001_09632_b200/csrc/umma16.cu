// B = 16 gather (+ decode) on the 5th-generation tensor cores: tcgen05.mma (UMMA) with
// accumulators in tensor memory (sensing.cpp:192-227 apply_plan, recon.cpp:109-117 decode_idct).
//
// A CTA (4 warps) walks strips of 8 consecutive blocks of a block row (a 16 x 128 pixel
// tile). Per strip, four M=128 x N=32 UMMAs with fp16 hi/lo operands (fp32-level accuracy,
// fp32 accumulation in TMEM); TMEM lane m is thread m, so each thread reads back one row:
//   1. D1[(b,c)][u|16+u] = sum_r X_b[r][c] {Ch,Cl}[u][r]       A = u8 pixels (exact), K = 16
//   2. D2[(b,u)][v|16+v] = sum_c {Qh,Ql}_b[u][c] {Ch,Cl}[v][c]  Y_b[u][v] = hi + lo halves
//      -> the zigzag prefix of each block (rank < count) -> payload
//   3. D3[(b,u)][c|16+c] = sum_v {Ymh,Yml}_b[u][v] {Ch,Cl}[v][c] (Ym = Y masked to the prefix)
//   4. D4[(b,c)][r|16+r] = sum_u {Wh,Wl}_b[u][c] {Ch,Cl}[u][r]  X_b[r][c]
// The decode-only variant (payload -> pixels) runs steps 3-4 from the payload, so the fused
// decode equals decode_idct of the written payload bit for bit.
//
// Shared-memory operands use the SWIZZLE_NONE canonical layouts: K-major element (m, k) at
// (m%8)*16 + (m/8)*SBO + (k/8)*LBO + (k%8)*2 bytes, MN-major at (m%8)*2 + (m/8)*SBO +
// (k%8)*16 + (k/8)*LBO; LBO = 128 B (next 8 k), SBO = 128 B * K/8 (next 8 m).
#include <cuda_fp16.h>

#include "common.cuh"
#include "internal.h"
#include "mma_dct.cuh"

namespace abcs_b200 {

constexpr int kUThreads = 128;
constexpr int kUBlocks = 8;  // blocks per strip (M = 8 x 16 = 128 rows)

struct UmmaSmem {
  __half a1[16 * 128];  // stage-1 A: MN-major, K = 16 (SBO 256)
  __half ax[32 * 128];  // stage-2/4 A (MN-major) and stage-3 A (K-major), K = 32 (SBO 512)
  __half b1[32 * 16];   // basis {Ch; Cl}[u][r]: K-major, N = 32, K = 16 (SBO 256)
  __half b2[32 * 32];   // basis {Ch; Cl}[v][c] over k = c | 16 + c: K-major, K = 32 (SBO 512)
  __half b3[32 * 32];   // transposed basis {Ch; Cl}[k][n]: B of stages 3 and 4
  float zb[kUBlocks * 256];  // the strip's zigzag-ordered prefixes
  int cnt[kUBlocks];
  int off[kUBlocks];
  int pre[kUBlocks + 1];  // exclusive prefix of the strip's counts (zb is packed: block b at pre[b])
  uint64_t mbar;
  uint32_t tmem;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_sdesc(const void* base, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((su32(base) >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1, SWIZZLE_NONE
}

// kind::f16: D f32, A/B f16, M = 128, N = 32, A major as given, B K-major
__host__ __device__ constexpr uint32_t umma_idesc(bool a_mn_major) {
  return (1u << 4) | ((a_mn_major ? 1u : 0u) << 15) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
}

__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n" ::"l"((uint64_t)su32(mbar)));
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t& phase) {
  asm volatile(
      "{\n.reg .pred p;\nUWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      "@!p bra UWAIT_%=;\n}\n" ::"r"(su32(mbar)),
      "r"(phase)
      : "memory");
  phase ^= 1u;
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// thread-written smem operands -> visible to the tensor core, then a CTA barrier
__device__ __forceinline__ void operands_ready() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// this thread's TMEM lane, 32 consecutive columns from col
__device__ __forceinline__ void tmem_row32(uint32_t tmem, int col, float (&v)[32]) {
  const uint32_t addr = tmem + ((uint32_t)((threadIdx.x >> 5) * 32) << 16) + (uint32_t)col;
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 values of this thread -> hi/lo fp16 halves: h[0..3] = values 0-7, h[4..7] = 8-15 (pairs)
__device__ __forceinline__ void split16(const float (&x)[16], uint32_t (&h)[8], uint32_t (&l)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) split2(x[2 * i], x[2 * i + 1], h[i], l[i]);
}

// MN-major K = 32 operand: this thread's 16 values at m = 16 b + i (i = 0..15), k = kk (hi) and
// 16 + kk (lo)
__device__ __forceinline__ void store_mn32(__half* a, int b, int kk, const uint32_t (&h)[8], const uint32_t (&l)[8]) {
  char* base = reinterpret_cast<char*>(a);
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int mg = 2 * b + half;
    *reinterpret_cast<uint4*>(base + mg * 512 + (kk & 7) * 16 + (kk >> 3) * 128) =
        make_uint4(h[4 * half], h[4 * half + 1], h[4 * half + 2], h[4 * half + 3]);
    const int kl = 16 + kk;
    *reinterpret_cast<uint4*>(base + mg * 512 + (kl & 7) * 16 + (kl >> 3) * 128) =
        make_uint4(l[4 * half], l[4 * half + 1], l[4 * half + 2], l[4 * half + 3]);
  }
}

// K-major K = 32 operand row m: k = 0..15 hi, 16..31 lo
__device__ __forceinline__ void store_k32(__half* a, int m, const uint32_t (&h)[8], const uint32_t (&l)[8]) {
  char* base = reinterpret_cast<char*>(a) + (m & 7) * 16 + (m >> 3) * 512;
  *reinterpret_cast<uint4*>(base + 0 * 128) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(base + 1 * 128) = make_uint4(h[4], h[5], h[6], h[7]);
  *reinterpret_cast<uint4*>(base + 2 * 128) = make_uint4(l[0], l[1], l[2], l[3]);
  *reinterpret_cast<uint4*>(base + 3 * 128) = make_uint4(l[4], l[5], l[6], l[7]);
}

__device__ __forceinline__ void put_half(__half* a, uint32_t byte_off, __half v) {
  *reinterpret_cast<__half*>(reinterpret_cast<char*>(a) + byte_off) = v;
}

struct UmmaArgs {
  const uint8_t* imgs;
  int64_t img_stride;
  int pitch;
  const uint16_t* counts;
  const int32_t* offsets;
  float* payload;  // written (from image) or read (decode only)
  int64_t payload_stride;
  float* out;
  int64_t out_stride;
  int out_pitch;
  bool aligned;               // image rows 8-byte aligned
  int rows, cols, spr;        // block grid, strips per block row
  uint32_t nb, total_strips;
  FastDiv div_img, div_row;   // strips per image, strips per row
};

// This thread's 2 x 8 bytes of a strip (row r = i / 16, pixels 8 (i % 16) ..), zeros past the
// block row's last block. Rows are 8-byte aligned (A.aligned), else bytewise.
__device__ __forceinline__ void load_strip_u8(const UmmaArgs& A, uint32_t strip, uint2 (&w)[2]) {
  const uint32_t img = A.div_img.div(strip);
  const uint32_t rem = strip - img * A.div_img.d;
  const uint32_t br = A.div_row.div(rem);
  const int bc0 = (int)(rem - br * A.div_row.d) * kUBlocks;
  const int width = min(kUBlocks, A.cols - bc0) * 16;
  const uint8_t* src = A.imgs + (int64_t)img * A.img_stride + (int64_t)(br * 16) * A.pitch + bc0 * 16;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int i = threadIdx.x + j * kUThreads, r = i >> 4, g = i & 15;
    w[j] = make_uint2(0u, 0u);
    if (8 * g < width) {
      const uint8_t* p = src + (int64_t)r * A.pitch + 8 * g;
      if (A.aligned) {
        w[j] = __ldg(reinterpret_cast<const uint2*>(p));
      } else {
        w[j].x = (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24;
        w[j].y = (uint32_t)p[4] | (uint32_t)p[5] << 8 | (uint32_t)p[6] << 16 | (uint32_t)p[7] << 24;
      }
    }
  }
}

template <bool kFromImage, bool kDecode>
__global__ void __launch_bounds__(kUThreads, 8) sense16_umma_kernel(UmmaArgs A) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  UmmaSmem& s = *reinterpret_cast<UmmaSmem*>(smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023));
  const int t = threadIdx.x, warp = t >> 5;
  // constant B operands: the reference basis (dct.cpp:9-21) split into fp16 hi/lo
  {
    const double* C = basis_dev<16>();
    for (int i = t; i < 32 * 16; i += kUThreads) {  // b1[n][k = r] = C?[u = n%16][r]
      const int n = i >> 4, k = i & 15;
      const float c = (float)C[(n & 15) * 16 + k];
      const __half h = __float2half_rn(c);
      put_half(s.b1, (n & 7) * 16 + (n >> 3) * 256 + (k >> 3) * 128 + (k & 7) * 2,
               n < 16 ? h : __float2half_rn(c - __half2float(h)));
    }
    for (int i = t; i < 32 * 32; i += kUThreads) {
      const int n = i >> 5, k = i & 31;
      const uint32_t o = (n & 7) * 16 + (n >> 3) * 512 + (k >> 3) * 128 + (k & 7) * 2;
      const float c2 = (float)C[(n & 15) * 16 + (k & 15)];  // b2[n = v][k = c]: C[v][c]
      const float c3 = (float)C[(k & 15) * 16 + (n & 15)];  // b3[n][k]: C[k][n]
      const __half h2 = __float2half_rn(c2), h3 = __float2half_rn(c3);
      put_half(s.b2, o, n < 16 ? h2 : __float2half_rn(c2 - __half2float(h2)));
      put_half(s.b3, o, n < 16 ? h3 : __float2half_rn(c3 - __half2float(h3)));
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(su32(&s.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(su32(&s.mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  operands_ready();
  const uint32_t tmem = s.tmem;
  uint32_t phase = 0;
  const unsigned short* zr = zigzag_rank_dev<16>();
  constexpr uint32_t kIdMN = umma_idesc(true), kIdK = umma_idesc(false);
  uint2 pre_w[2] = {make_uint2(0u, 0u), make_uint2(0u, 0u)};
  if (kFromImage && blockIdx.x < A.total_strips) load_strip_u8(A, blockIdx.x, pre_w);

  for (uint32_t strip = blockIdx.x; strip < A.total_strips; strip += gridDim.x) {
    const uint32_t img = A.div_img.div(strip);
    const uint32_t rem = strip - img * A.div_img.d;
    const uint32_t br = A.div_row.div(rem);
    const int bc0 = (int)(rem - br * A.div_row.d) * kUBlocks;
    const int nblk = min(kUBlocks, A.cols - bc0);
    const uint32_t bidx0 = img * A.nb + br * (uint32_t)A.cols + (uint32_t)bc0;
    if (t < 32) {  // counts, offsets and their in-strip prefix (warp 0)
      const int c = t < nblk ? A.counts[bidx0 + t] : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < kUBlocks; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (t >= o) incl += x;
      }
      if (t < kUBlocks) {
        s.cnt[t] = c;
        s.off[t] = t < nblk ? A.offsets[bidx0 + t] : 0;
        s.pre[t] = incl - c;
        if (t == kUBlocks - 1) s.pre[kUBlocks] = incl;
      }
    }
    float* pay = A.payload + (int64_t)img * A.payload_stride;
    if constexpr (kFromImage) {
      // stage 1 A: row r, 8-pixel group g of the strip -> MN-major (m = pixel column, k = r);
      // the bytes were loaded one strip ahead
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int i = t + j * kUThreads, r = i >> 4, g = i & 15;
        const uint4 v = make_uint4(u8sel_to_h2(pre_w[j].x, 0x4140), u8sel_to_h2(pre_w[j].x, 0x4342),
                                   u8sel_to_h2(pre_w[j].y, 0x4140), u8sel_to_h2(pre_w[j].y, 0x4342));
        *reinterpret_cast<uint4*>(reinterpret_cast<char*>(s.a1) + g * 256 + (r & 7) * 16 + (r >> 3) * 128) = v;
      }
      if (strip + gridDim.x < A.total_strips) load_strip_u8(A, strip + gridDim.x, pre_w);
      operands_ready();
      if (t == 0) {
        umma(tmem, umma_sdesc(s.a1, 128, 256), umma_sdesc(s.b1, 128, 256), kIdMN, 0);
        umma_commit(&s.mbar);
      }
      mbar_wait(&s.mbar, phase);
      {  // D1 row (b, c): Q_b[u][c] = hi + lo -> stage 2 A at m = (b, u), k = c
        float v[32], q[16];
        tmem_row32(tmem, 0, v);
#pragma unroll
        for (int u = 0; u < 16; ++u) q[u] = v[u] + v[16 + u];
        uint32_t h[8], l[8];
        split16(q, h, l);
        store_mn32(s.ax, t >> 4, t & 15, h, l);
      }
      operands_ready();
      if (t == 0) {
        umma(tmem + 32, umma_sdesc(s.ax, 128, 512), umma_sdesc(s.b2, 128, 512), kIdMN, 0);
        umma(tmem + 32, umma_sdesc(reinterpret_cast<char*>(s.ax) + 256, 128, 512),
             umma_sdesc(reinterpret_cast<char*>(s.b2) + 256, 128, 512), kIdMN, 1);
        umma_commit(&s.mbar);
      }
      mbar_wait(&s.mbar, phase);
      {  // D2 row (b, u): Y_b[u][v]; zigzag prefix -> zb, masked row -> stage 3 A (K-major)
        float v[32], ym[16];
        tmem_row32(tmem, 32, v);
        const int b = t >> 4, u = t & 15, cnt = s.cnt[b];
        float* zbb = s.zb + s.pre[b];
#pragma unroll
        for (int w = 0; w < 16; ++w) {
          const float y = v[w] + v[16 + w];
          const int rk = zr[u * 16 + w];
          const bool in = rk < cnt;
          if (in) zbb[rk] = y;
          ym[w] = in ? y : 0.f;
        }
        if constexpr (kDecode) {
          uint32_t h[8], l[8];
          split16(ym, h, l);
          store_k32(s.ax, t, h, l);
        }
      }
      if constexpr (!kDecode) {  // gather only: the strip's payload, then the next strip
        __syncthreads();
        float* dst = pay + s.off[0];
        const int total = s.pre[kUBlocks];
        for (int k = t; k < total; k += kUThreads) dst[k] = s.zb[k];
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        continue;
      }
    } else {
      __syncthreads();  // cnt / off / pre
      // the strip's prefixes (contiguous in the payload) -> zb, then each row gathers its masked Y
      {
        const float* src = pay + s.off[0];
        const int total = s.pre[kUBlocks];
        for (int k = t; k < total; k += kUThreads) s.zb[k] = __ldg(src + k);
      }
      __syncthreads();
      const int b = t >> 4, u = t & 15, cnt = s.cnt[b];
      const float* zbb = s.zb + s.pre[b];
      float ym[16];
#pragma unroll
      for (int w = 0; w < 16; ++w) {
        const int rk = zr[u * 16 + w];
        ym[w] = rk < cnt ? zbb[rk] : 0.f;
      }
      uint32_t h[8], l[8];
      split16(ym, h, l);
      store_k32(s.ax, t, h, l);
    }
    operands_ready();
    if (t == 0) {
      umma(tmem, umma_sdesc(s.ax, 128, 512), umma_sdesc(s.b3, 128, 512), kIdK, 0);
      umma(tmem, umma_sdesc(reinterpret_cast<char*>(s.ax) + 256, 128, 512),
           umma_sdesc(reinterpret_cast<char*>(s.b3) + 256, 128, 512), kIdK, 1);
      umma_commit(&s.mbar);
    }
    if constexpr (kFromImage) {  // the payload copy (contiguous over the strip) overlaps stage 3
      float* dst = pay + s.off[0];
      const int total = s.pre[kUBlocks];
      for (int k = t; k < total; k += kUThreads) dst[k] = s.zb[k];
    }
    mbar_wait(&s.mbar, phase);
    {  // D3 row (b, u): W_b[u][c] -> stage 4 A at m = (b, c), k = u (MN-major)
      float v[32], w16[16];
      tmem_row32(tmem, 0, v);
#pragma unroll
      for (int c = 0; c < 16; ++c) w16[c] = v[c] + v[16 + c];
      uint32_t h[8], l[8];
      split16(w16, h, l);
      store_mn32(s.ax, t >> 4, t & 15, h, l);
    }
    operands_ready();
    if (t == 0) {
      umma(tmem + 32, umma_sdesc(s.ax, 128, 512), umma_sdesc(s.b3, 128, 512), kIdMN, 0);
      umma(tmem + 32, umma_sdesc(reinterpret_cast<char*>(s.ax) + 256, 128, 512),
           umma_sdesc(reinterpret_cast<char*>(s.b3) + 256, 128, 512), kIdMN, 1);
      umma_commit(&s.mbar);
    }
    mbar_wait(&s.mbar, phase);
    {  // D4 row (b, c): X_b[r][c] -> pixels (a warp writes 32 consecutive columns per row)
      float v[32];
      tmem_row32(tmem, 32, v);
      const int b = t >> 4, c = t & 15;
      if (b < nblk) {
        float* o = A.out + (int64_t)img * A.out_stride + (int64_t)(br * 16) * A.out_pitch + (bc0 + b) * 16 + c;
#pragma unroll
        for (int r = 0; r < 16; ++r) o[(int64_t)r * A.out_pitch] = v[r] + v[16 + r];
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();  // smem operands, zb and cnt are reused by the next strip
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tmem));
}

// Opt-in (ABCS_UMMA=1, read per launch): measured slower than the mma.sync kernels so far
// ("tcgen05 path"), so not the default.
bool umma16_enabled() {
  const char* e = getenv("ABCS_UMMA");
  return e && e[0] == '1';
}

int launch_sense16_umma(Ctx* ctx, int mode, int rows, int cols, int n, const uint8_t* imgs, int64_t img_stride,
                        int pitch, const uint16_t* counts, const int32_t* offsets, float* payload,
                        int64_t payload_stride, float* out, int64_t out_stride, int out_pitch, cudaStream_t s) {
  UmmaArgs A{};
  A.imgs = imgs;
  A.img_stride = img_stride;
  A.pitch = pitch;
  A.aligned = ((uintptr_t)imgs % 8 == 0) && (img_stride % 8 == 0) && (pitch % 8 == 0);
  A.counts = counts;
  A.offsets = offsets;
  A.payload = payload;
  A.payload_stride = payload_stride;
  A.out = out;
  A.out_stride = out_stride;
  A.out_pitch = out_pitch;
  A.rows = rows;
  A.cols = cols;
  A.spr = (cols + kUBlocks - 1) / kUBlocks;
  A.nb = (uint32_t)rows * cols;
  A.total_strips = (uint32_t)A.spr * rows * n;
  A.div_img = FastDiv((uint32_t)A.spr * rows);
  A.div_row = FastDiv((uint32_t)A.spr);
  if (A.total_strips == 0) return ABCS_OK;
  const int smem = (int)sizeof(UmmaSmem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sense16_umma_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sense16_umma_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sense16_umma_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const unsigned grid = (unsigned)std::min<int64_t>(A.total_strips, (int64_t)ctx->sm_count * 8);
  // mode 2: gather (payload only), 3: gather + decode, 4: decode from the payload
  const int kt = ktimer_begin(ctx, s, mode == 2 ? "sense16_gather" : mode == 3 ? "sense16_gather_decode" : "decode16");
  if (mode == 2) sense16_umma_kernel<true, false><<<grid, kUThreads, smem, s>>>(A);
  else if (mode == 3) sense16_umma_kernel<true, true><<<grid, kUThreads, smem, s>>>(A);
  else sense16_umma_kernel<false, true><<<grid, kUThreads, smem, s>>>(A);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "sense16 umma launch");
}

}  // namespace abcs_b200
