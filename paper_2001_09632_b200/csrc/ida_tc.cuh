// IDA step for B = 16 with the dct_threshold denoiser on the 5th-generation tensor cores
// (damp_step(Ida), recon.cpp:170-197; dct_soft_threshold, denoise.cpp:52-92). Included once by
// ida_mma.cu, whose fp32 block phase (block_phase16_f32) and per-image fold it shares.
//
// A persistent CTA (2 per SM, 8 warps) walks 64 x 64 output regions. Per region:
//   1. The 72 x 76 pseudo window (4-px halo) arrives by TMA, prefetched one region ahead.
//   2. Quad operand Q: the window as 18 x 18 quads of 4 x 4 pixels, one quad per operand row
//      (row m = qy * 18 + qx, K = the quad's 16 pixels), centred on a region constant and split
//      into fp16 hi + lo planes. Rows are 16 B apart within each 8-pixel k-group (SWIZZLE_NONE,
//      SBO = 16 B x 8), so a descriptor moved by s rows reads the raster shifted by s rows.
//   3. Forward DCT of every 8 x 8 tile at stride 4 as a GEMM: tile t = ty * 18 + tx covers quads
//      t, t + 1, t + 18, t + 19, so D[t][k] = sum_j Q[t + s_j] F_j with the four shifted
//      descriptors and F_j[p][k] = C[u][4dy + p/4] C[v][4dx + p%4] (k = 8u + v; dct.cpp:23-50
//      separable basis as a Kronecker product). M = 128 tiles, N = 64 coefficients, fp32 in TMEM;
//      hi*hi + lo*hi + hi*lo per shift (~fp32 accuracy).
//   4. Soft threshold of the AC coefficients at k * sigma (DC kept, denoise.cpp:70-78) from
//      tcgen05.ld rows, split again and stored as the inverse's A operand, one quarter of the 64
//      coefficients (K = 16) at a time.
//   5. Inverse DCT with the overlap-add folded into the GEMM: output quad q sits at quad position
//      (a, b) of tile q - 18a - b, so X[q][p] = sum_{a,b} Ythr[q - 18a - b] G_ab[k][p] with
//      G_ab[k][p] = C[u][4a + p/4] C[v][4b + p%4]: the tensor core sums the four covering tiles
//      (M = 128 quads, N = 16 pixels, K = 4 x 64), and x = cen + X / weight (denoise.cpp:84-90).
//   6. The fp32 block phase (z update, pseudo = x + A* z) and the region partials, as in
//      ida_mma_kernel.
// Tiles off the image's tile grid (and the raster's wrap-around column tx = 17) get an infinite
// threshold, which zeroes them (denoise.cpp:57-62). Fields whose centred magnitude exceeds
// kTcSafe are scaled by a power of two first (exact), so the fp16 halves never overflow.
#pragma once  // included inside namespace abcs_b200 (ida_mma.cu)

constexpr int kTcThreads = 256;
constexpr int kTQ = 18;                      // window quads per row (16 region quads + 1 halo each side)
constexpr int kTRows = 408;                  // rows per operand plane (the shifted descriptors read up to 402)
constexpr int kTKg = kTRows * 16;            // one k-group of a plane: 6528 B (the descriptors' LBO)
constexpr int kTOp = 4 * kTKg;               // hi k-groups 0, 1 then lo k-groups 0, 1: 26112 B
constexpr int kTTiles = 17 * kTQ;            // raster rows holding the region's 17 x 17 tiles (+ wrap column)
constexpr int kTOut0 = kTQ + 1;              // first output quad row: window quad (1, 1)
constexpr int kTOutEnd = 16 * kTQ + 17;      // one past the last output quad row: (16, 16)
constexpr uint32_t kTmemCols = 256;          // forward D: 3 x 64 columns; inverse X: 192 + 3 x 16
constexpr int kTXCol = 192;
constexpr float kTcSafe = 4096.f;            // |centred field| bound: every fp16 operand stays < 2^15
#ifndef IDA_TC_MINB
#define IDA_TC_MINB 2
#endif

struct IdaTcSmem {
  float win[kMIn * kWP];  // TMA window of the next region (128-B aligned: offset 0)
  union {
    unsigned char ythr[kTOp];  // thresholded coefficients, one quarter (K = 16) of each tile
    float RS[16 * kTB];        // then the block phase's transpose tiles
  };
  union {
    unsigned char q[kTOp];    // quad operand of the window
    float acc[kMIn * kMP];    // then x over the region (kMOff, pitch kMP) for the block phase
  };
  unsigned char fb[4 * 2 * 2048];     // F_j hi / lo: B operand [64 coefficients][16 pixels]
  unsigned char gb[4 * 4 * 2 * 512];  // G_{c,j} hi / lo: B operand [16 pixels][16 coefficients of quarter c]
  int meta_cnt[64];
  int meta_off[64];
  double red[4][16];
  unsigned int bad[2];
  double mine[4];
  uint64_t win_bar, mma_bar;
  uint32_t tmem;
  unsigned int cmax;  // float bits of the region's largest centred magnitude (rare rescale path)
  unsigned short zidx[256];
};
static_assert(kMIn * kMP * 4 <= kTOp, "acc fits in the quad operand's space");
static_assert(16 * kTB * 4 <= kTOp, "transpose tiles fit in the coefficient operand's space");

__device__ __forceinline__ uint64_t tc_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1, SWIZZLE_NONE
}
// kind::f16: D f32, A / B f16, both K-major, M = 128, N as given
__host__ __device__ constexpr uint32_t tc_idesc(int N) { return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24); }

// Issued by a whole warp (warp-uniform descriptors stay in uniform registers); one elected lane
// issues the MMA / commit.
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n}\n" ::"l"((uint64_t)smem_u32(bar)));
}
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t& phase) {
  asm volatile(
      "{\n.reg .pred p;\nTCW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      "@!p bra TCW_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
  phase ^= 1u;
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// thread-written operands -> the tensor core's proxy, then a CTA barrier
__device__ __forceinline__ void tc_operands_ready() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_ld8(uint32_t addr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
}
__device__ __forceinline__ void tc_ld16(uint32_t addr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
}
__device__ __forceinline__ void tc_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

// The basis operands (B, K-major, SWIZZLE_NONE: element (n, k) at (n%8)*16 + (n/8)*256 + (k/8)*128
// + (k%8)*2): F_j hi / lo (16 KB) then G_{c,j} hi / lo (16 KB), built once on the host from the
// reference's fp64 basis (dct.cpp:9-21; ida_tc_upload_bases) and copied into each CTA.
__device__ __align__(16) unsigned char g_tc_bases[32768];

__device__ __forceinline__ void tc_load_bases(IdaTcSmem& s) {
  const uint4* src = reinterpret_cast<const uint4*>(g_tc_bases);
  uint4* f = reinterpret_cast<uint4*>(s.fb);
  uint4* g = reinterpret_cast<uint4*>(s.gb);
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) {
    const uint4 v = __ldg(src + i);
    if (i < 1024) f[i] = v;
    else g[i - 1024] = v;
  }
}

// Window -> quad operand (hi / lo planes) at scale sc; returns this thread's largest |centred value|.
__device__ __forceinline__ float tc_build_q(IdaTcSmem& s, float cen, float sc) {
  const uint32_t qa = smem_u32(s.q);
  float mx = 0.f;
  for (int qi = threadIdx.x; qi < kTQ * kTQ; qi += kTcThreads) {
    const int qy = qi / kTQ, qx = qi - kTQ * qy;
    const float* src = s.win + 4 * qy * kWP + 4 * qx;
    uint32_t h[8], l[8];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float4 a = *reinterpret_cast<const float4*>(src + r * kWP);
      const float v0 = (a.x - cen) * sc, v1 = (a.y - cen) * sc, v2 = (a.z - cen) * sc, v3 = (a.w - cen) * sc;
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v0), fabsf(v1)), fmaxf(fabsf(v2), fabsf(v3))));
      split2(v0, v1, h[2 * r], l[2 * r]);
      split2(v2, v3, h[2 * r + 1], l[2 * r + 1]);
    }
    const uint32_t a = qa + qi * 16;
    sts128(a, h[0], h[1], h[2], h[3]);
    sts128(a + kTKg, h[4], h[5], h[6], h[7]);
    sts128(a + 2 * kTKg, l[0], l[1], l[2], l[3]);
    sts128(a + 3 * kTKg, l[4], l[5], l[6], l[7]);
  }
  return mx;
}

template <class Sm>
__device__ __forceinline__ void l1_prefetch_yz(const IdaParams& P, int img, const Sm& s) {
  if (!P.y) return;
  const int t = threadIdx.x;
  const int j = (t >> 5) & 3, line = t & 31;  // warps 0-3 -> block rows 0-3 of y, warps 4-7 of z
  if (t >= 256) return;
  int first = -1, n = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = s.meta_cnt[4 * j + i];
    if (c >= 0) {
      if (first < 0) first = s.meta_off[4 * j + i];
      n += c;
    }
  }
  if (first < 0) return;
  const float* base = ((t >> 7) ? P.z : P.y) + (int64_t)img * P.y_stride + first;
  for (int o = line * 32; o < n; o += 32 * 32) asm volatile("prefetch.global.L1 [%0];\n" ::"l"(base + o));
}

__device__ __forceinline__ void tc_window_issue(IdaTcSmem& s, const CUtensorMap* tm, int w, const IdaParams& P) {
  const int img = w / P.regions_per_img, region = w - img * P.regions_per_img;
  const int R0 = (region / P.regions_x) * kMR, C0 = (region % P.regions_x) * kMR;
  const uint32_t b = smem_u32(&s.win_bar);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // the window's generic reads precede the overwrite
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(kWinBytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
      ::"r"(smem_u32(s.win)), "l"(tm), "r"(C0 - 4), "r"(R0 - 4), "r"(img), "r"(b)
      : "memory");
}

__global__ void __launch_bounds__(kTcThreads, IDA_TC_MINB) ida_tc_kernel(IdaParams P, const __grid_constant__ CUtensorMap win_map) {
  extern __shared__ __align__(128) unsigned char tc_smem_raw[];
  IdaTcSmem& s = *reinterpret_cast<IdaTcSmem*>(tc_smem_raw + ((128 - (smem_u32(tc_smem_raw) & 127)) & 127));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int total = P.n * P.regions_per_img;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&s.tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&s.win_bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&s.mma_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  s.zidx[tid] = zigzag_dev<16>()[tid];
  tc_load_bases(s);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = s.tmem;
  if (tid == 0 && (int)blockIdx.x < total) tc_window_issue(s, &win_map, blockIdx.x, P);
  uint32_t win_phase = 0, mma_phase = 0;
  const uint32_t qa = smem_u32(s.q), ya = smem_u32(s.ythr), fa = smem_u32(s.fb), ga = smem_u32(s.gb);
  // base descriptors (CTA-uniform); a row shift of r adds r to the start-address field (16-B units)
  const uint64_t dq_hi = tc_sdesc(qa, kTKg, 128), dq_lo = tc_sdesc(qa + 2 * kTKg, kTKg, 128);
  const uint64_t dy_hi = tc_sdesc(ya, kTKg, 128), dy_lo = tc_sdesc(ya + 2 * kTKg, kTKg, 128);
  const uint64_t dg = tc_sdesc(ga, 128, 256);
  uint64_t df[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) df[i] = tc_sdesc(fa + i * 2048, 128, 256);
  const float kInf = __int_as_float(0x7f800000);
  const int wq = warp & 3, half = warp >> 2;
  const uint32_t lane_base = (uint32_t)(32 * wq) << 16;

  for (int w = blockIdx.x; w < total; w += gridDim.x) {
    const int img = w / P.regions_per_img, region = w - img * P.regions_per_img;
    const int R0 = (region / P.regions_x) * kMR, C0 = (region % P.regions_x) * kMR;
    fetch_meta<16>(P, img, R0, C0, s);  // visible after the next barrier
    if (tid == 0) s.cmax = 0u;
    // 1-2. window -> quad operand (the window's TMA was issued a region ahead)
    asm volatile(
        "{\n.reg .pred p;\nTCWIN_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
        "@!p bra TCWIN_%=;\n}\n" ::"r"(smem_u32(&s.win_bar)),
        "r"(win_phase)
        : "memory");
    win_phase ^= 1u;
    const float cen = 0.25f * (s.win[35 * kWP + 35] + s.win[35 * kWP + 36] + s.win[36 * kWP + 35] + s.win[36 * kWP + 36]);
    float mx = tc_build_q(s, cen, 1.f);
    float up = 1.f, thr = (float)(P.k * P.sigma_in[img]);
    if (__syncthreads_or(!(mx <= kTcSafe))) {  // rare: rescale by 2^-e (exact) so every fp16 half is finite
      if (mx > 0.f) atomicMax(&s.cmax, __float_as_uint(fminf(mx, FLT_MAX)));
      __syncthreads();
      const float m = __uint_as_float(s.cmax);
      int e = 0;
      if (m > kTcSafe) frexpf(m / kTcSafe, &e);
      tc_build_q(s, cen, ldexpf(1.f, -e));
      up = ldexpf(1.f, e);
      thr = ldexpf(thr, -e);
      __syncthreads();
    }
    // the raster's tail rows (read by the wrap-around tiles' shifted descriptors): zeros
    for (int i = tid; i < (kTRows - kTQ * kTQ) * 4; i += kTcThreads) {
      const int row = kTQ * kTQ + (i >> 2), g = i & 3;
      sts128(qa + g * kTKg + row * 16, 0u, 0u, 0u, 0u);
    }
    tc_operands_ready();  // Q complete; the window is consumed
    const int wn = w + gridDim.x;
    if (tid == 0 && wn < total) tc_window_issue(s, &win_map, wn, P);
    // 3. forward transforms of the 3 x 128 raster tiles (warp 0 issues)
    if (warp == 0) {
#pragma unroll
      for (int mb = 0; mb < 3; ++mb) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t ro = (uint32_t)(128 * mb + kTQ * (j >> 1) + (j & 1));  // row shift (16-B units)
          const uint32_t d = tmem + 64 * mb;
          tc_mma(d, dq_hi + ro, df[2 * j], tc_idesc(64), j > 0);
          tc_mma(d, dq_lo + ro, df[2 * j], tc_idesc(64), 1);
          tc_mma(d, dq_hi + ro, df[2 * j + 1], tc_idesc(64), 1);
        }
      }
      tc_commit(&s.mma_bar);
    }
    l1_prefetch_yz(P, img, s);
    // tile on-grid flags of this thread's raster rows (t = 128 mb + 32 wq + lane)
    bool on[3];
#pragma unroll
    for (int mb = 0; mb < 3; ++mb) {
      const int t = 128 * mb + 32 * wq + lane, ty = t / kTQ, tx = t - kTQ * ty;
      on[mb] = tx <= 16 && ty <= 16 && (unsigned)(R0 - 4 + 4 * ty) <= (unsigned)(P.Hc - 8) &&
               (unsigned)(C0 - 4 + 4 * tx) <= (unsigned)(P.Wc - 8);
    }
    // 4-5. per quarter of the coefficients: threshold + split -> Ythr, then the folded inverse
#pragma unroll 1
    for (int c4 = 0; c4 < 4; ++c4) {
      tc_wait(&s.mma_bar, mma_phase);  // forward done (c4 = 0) / previous quarter's inverse done (Ythr free)
      uint32_t y[3][8];
#pragma unroll
      for (int mb = 0; mb < 3; ++mb)
        if (128 * mb + 32 * wq < kTTiles) tc_ld8(tmem + lane_base + 64 * mb + 16 * c4 + 8 * half, y[mb]);
      tc_ld_wait();
#pragma unroll
      for (int mb = 0; mb < 3; ++mb) {
        if (128 * mb + 32 * wq >= kTTiles) continue;  // warp-uniform: raster rows past the tiles
        const int t = 128 * mb + 32 * wq + lane;
        const float T = on[mb] ? thr : kInf;
        float sv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float yv = __uint_as_float(y[mb][i]);
          const float ti = (i == 0 && c4 == 0 && half == 0) ? (on[mb] ? 0.f : kInf) : T;  // the DC passes
          sv[i] = yv - fminf(fmaxf(yv, -ti), ti);
        }
        uint32_t h[4], l[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) split2(sv[2 * i], sv[2 * i + 1], h[i], l[i]);
        const uint32_t a = ya + half * kTKg + t * 16;
        sts128(a, h[0], h[1], h[2], h[3]);
        sts128(a + 2 * kTKg, l[0], l[1], l[2], l[3]);
      }
      tc_operands_ready();
      if (warp == 0) {
#pragma unroll
        for (int mb = 0; mb < 3; ++mb) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t ro = (uint32_t)(kTOut0 + 128 * mb - kTQ * (j >> 1) - (j & 1));
            const uint64_t bh = dg + (uint32_t)(((c4 * 4 + j) * 2) * 512 / 16), bl = bh + 512 / 16;
            const uint32_t d = tmem + kTXCol + 16 * mb;
            tc_mma(d, dy_hi + ro, bh, tc_idesc(16), (c4 | j) != 0);
            tc_mma(d, dy_lo + ro, bh, tc_idesc(16), 1);
            tc_mma(d, dy_hi + ro, bl, tc_idesc(16), 1);
          }
        }
        tc_commit(&s.mma_bar);
      }
    }
    tc_wait(&s.mma_bar, mma_phase);  // the last quarter's inverse
    // 5. x over the region: X / weight + cen (the four covering tiles' sum, denoise.cpp:84-90)
#pragma unroll
    for (int mb = 0; mb < 3; ++mb) {
      if ((mb & 1) != (warp >= 4 ? 1 : 0)) continue;  // warps 0-3: mb 0, 2; warps 4-7: mb 1
      const int q0 = kTOut0 + 128 * mb + 32 * wq;
      if (q0 >= kTOutEnd) continue;
      uint32_t X[16];
      tc_ld16(tmem + lane_base + kTXCol + 16 * mb, X);
      tc_ld_wait();
      const int qq = q0 + lane, qy = qq / kTQ, qx = qq - kTQ * qy;
      if (qx >= 1 && qx <= 16 && qy <= 16) {
        const int r0 = 4 * (qy - 1), c0 = 4 * (qx - 1);
        const int br = R0 + r0, bc = C0 + c0;  // tile origins covering the quad per axis: 1 or 2
        const int wgt = max(((br >= 4 ? 1 : 0) + (br <= P.Hc - 8 ? 1 : 0)) * ((bc >= 4 ? 1 : 0) + (bc <= P.Wc - 8 ? 1 : 0)), 1);
        const float sc = (wgt == 4 ? 0.25f : (wgt == 2 ? 0.5f : 1.f)) * up;
#pragma unroll
        for (int r = 0; r < 4; ++r)
          *reinterpret_cast<float4*>(s.acc + kMOff + (r0 + r) * kMP + c0) =
              make_float4(fmaf(__uint_as_float(X[4 * r]), sc, cen), fmaf(__uint_as_float(X[4 * r + 1]), sc, cen),
                          fmaf(__uint_as_float(X[4 * r + 2]), sc, cen), fmaf(__uint_as_float(X[4 * r + 3]), sc, cen));
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();  // x complete; Ythr (now the transpose tiles) is no longer read by the tensor core
    // 6. block phase and the region's partials
    IdaLaneSums S;
    block_phase16_f32(P, img, R0, C0, s, S);
    reduce_and_finish(P, img, region, s, S);
    __syncthreads();  // acc / meta / red reused by the next region
  }
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
  }
}

