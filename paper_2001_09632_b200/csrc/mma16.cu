// B = 16 hot path on tensor cores (mma.sync, fp16 hi/lo split; mma_dct.cuh).
//
//  * sense16_kernel<kWeights, kPayload, kDecode>: u8 image blocks ->
//      kWeights: DD phase-1 significance counts n_i (sensing.cpp:341-358)
//      kPayload: zigzag-prefix payload (gather_prefixes, sensing.cpp:192-227)
//      kDecode:  decode_idct of that payload (recon.cpp:109-117), fused: the
//                inverse transform consumes the same fp32 values that were
//                written to the payload, so the pixels equal decode(payload)
//                bit for bit without re-reading the payload from HBM.
//  * decode16_kernel: decode_idct from a packed payload.
//
// A warp owns a pair of horizontally adjacent blocks per step (lane L loads row
// L%16 of block L/16 with one 16-B load; the pair's rows share a 32-B sector),
// stages them in shared memory and gathers its B-fragment bytes from there; the
// next pair is prefetched into registers meanwhile. Coefficients travel through
// a per-warp zigzag-ordered buffer: prefix writes to the payload are coalesced
// and the inverse transform reads buf[rank] for rank < count (zeros above),
// so no tile has to be cleared between blocks.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "internal.h"
#include "mma_dct.cuh"
#include "zz_banks.cuh"
#include "cta_alloc.cuh"
#include "warp_alloc.cuh"

namespace abcs_b200 {

constexpr int kM16Threads = 256;
constexpr int kM16Warps = kM16Threads / 32;

struct Grid16 {
  int rows, cols;
  uint32_t nb;                // rows * cols
  uint32_t pairs_per_row;     // ceil(cols / 2)
  uint32_t units_per_img;     // rows * pairs_per_row
  uint32_t total_units;
  int run_len;                // blocks per warp run: 32, or 16 / 8 when a small batch would underfill the GPU
  uint32_t runs_per_row;      // ceil(cols / run_len): a run = up to run_len consecutive blocks of a block-row
  uint32_t total_runs;
  FastDiv div_units, div_pairs, div_nb, div_cols, div_runs_img, div_runs_row;
};

static Grid16 make_grid16(int rows, int cols, int n) {
  Grid16 g;
  g.rows = rows;
  g.cols = cols;
  g.nb = (uint32_t)rows * cols;
  g.pairs_per_row = (uint32_t)(cols + 1) / 2;
  g.units_per_img = (uint32_t)rows * g.pairs_per_row;
  g.total_units = g.units_per_img * (uint32_t)n;
  // one warp per run: shorter runs for small batches (cfg1, cfg4) so the warps still fill the
  // 148 SMs (>= 1024 runs; cfg4 measured slower at 16), 32-block runs otherwise (fewer per-run set-ups)
  g.run_len = 32;
  while (g.run_len > 8 && (uint64_t)((cols + g.run_len - 1) / g.run_len) * rows * n < 1024) g.run_len /= 2;
  g.runs_per_row = (uint32_t)((cols + g.run_len - 1) / g.run_len);
  g.total_runs = g.runs_per_row * (uint32_t)rows * (uint32_t)n;
  g.div_runs_img = FastDiv(g.runs_per_row * (uint32_t)rows);
  g.div_runs_row = FastDiv(g.runs_per_row);
  g.div_units = FastDiv(g.units_per_img);
  g.div_pairs = FastDiv(g.pairs_per_row);
  g.div_nb = FastDiv(g.nb);
  g.div_cols = FastDiv((uint32_t)cols);
  return g;
}

__device__ __forceinline__ void unit_pos(const Grid16& G, uint32_t u, uint32_t& img, int& br, int& bc0) {
  img = G.div_units.div(u);
  const uint32_t rem = u - img * G.units_per_img;
  const uint32_t r = G.div_pairs.div(rem);
  br = (int)r;
  bc0 = 2 * (int)(rem - r * G.pairs_per_row);
}

// Lane L reads row L % 16 of block L / 16 of a pair: the run's row pointer, advanced 32 B per pair.
__device__ __forceinline__ const uint8_t* run_row_ptr(const uint8_t* __restrict__ imgs, int64_t img_stride, int pitch,
                                                      uint32_t img, int br, int bcf) {
  const int lane = threadIdx.x & 31;
  return imgs + (int64_t)img * img_stride + (int64_t)(br * 16 + (lane & 15)) * pitch + (bcf + (lane >> 4)) * 16;
}

__device__ __forceinline__ uint4 load_row16_at(const uint8_t* p, bool valid, bool aligned) {
  uint4 v = make_uint4(0, 0, 0, 0);
  if (valid) {
    if (aligned) {
      v = __ldg(reinterpret_cast<const uint4*>(p));
    } else {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        w[q] = (uint32_t)p[4 * q] | ((uint32_t)p[4 * q + 1] << 8) | ((uint32_t)p[4 * q + 2] << 16) |
               ((uint32_t)p[4 * q + 3] << 24);
      v = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  return v;
}

// exact-fp16 B fragments of block b of the staged pair
__device__ __forceinline__ void staged_bfrag(const uint8_t* st, int b, uint32_t (&bx)[2][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const uint8_t* base = st + b * 256;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int c = 8 * j + g;
    bx[j][0] = u8pair_to_h2(base[(2 * t) * 16 + c], base[(2 * t + 1) * 16 + c]);
    bx[j][1] = u8pair_to_h2(base[(2 * t + 8) * 16 + c], base[(2 * t + 9) * 16 + c]);
  }
}

// fp64 |c| for the DD guard band, reference operation order (dct.cpp:30-49)
[[maybe_unused]] __device__ __forceinline__ double exact_coef16(const uint8_t* __restrict__ blk, int pitch, int flat) {
  const double* C = basis_dev<16>();
  const int u = flat >> 4, v = flat & 15;
  double y = 0.0;
  for (int c = 0; c < 16; ++c) {
    double t = 0.0;
    for (int r = 0; r < 16; ++r) t = __dadd_rn(t, __dmul_rn(C[u * 16 + r], (double)blk[(size_t)r * pitch + c]));
    y = __dadd_rn(y, __dmul_rn(t, C[v * 16 + c]));
  }
  return y;
}

__device__ __forceinline__ void store_dfrag(float* __restrict__ blk_out, int pitch, const Acc16& X) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  float* p0 = blk_out + g * pitch + 2 * t;
  float* p1 = p0 + 8 * pitch;
  *reinterpret_cast<float2*>(p0) = make_float2(X.v[0][0], X.v[0][1]);
  *reinterpret_cast<float2*>(p1) = make_float2(X.v[0][2], X.v[0][3]);
  *reinterpret_cast<float2*>(p0 + 8) = make_float2(X.v[1][0], X.v[1][1]);
  *reinterpret_cast<float2*>(p1 + 8) = make_float2(X.v[1][2], X.v[1][3]);
}

struct Sense16Args {
  const uint8_t* imgs;
  int64_t img_stride;
  int pitch;
  bool aligned;
  // weights (DD phase 1)
  int phase1;
  double T;
  float Tf, band;
  uint32_t* weights;
  uint32_t* fix_list;   // (block, coefficient) pairs for the fp64 decision
  uint32_t* fix_count;
  uint32_t fix_cap;
  uint8_t* fix_flag;    // per block: had a near-threshold coefficient (overflow fallback)
  // payload
  const uint16_t* counts;
  const int32_t* offsets;
  float* payload;
  int64_t payload_stride;
  // decode
  float* out;
  int64_t out_stride;
  int out_pitch;
  // subrate sweep (kSweep): DD phase 1 of up to kMaxSweep plans from one transform
  int n_sw;
  int sw_phase1[4];
  float sw_hi[4], sw_lo[4];
  uint32_t* sw_weights[4];
  uint32_t* sw_fix_list[4];
  uint32_t* sw_fix_count[4];
  uint8_t* sw_fix_flag[4];
};
constexpr int kMaxSweep = 4;

__device__ __forceinline__ void run_pos(const Grid16& G, uint32_t r, uint32_t& img, int& br, int& bc_first,
                                        int& nblk) {
  img = G.div_runs_img.div(r);
  const uint32_t rem = r - img * (G.runs_per_row * (uint32_t)G.rows);
  const uint32_t row = G.div_runs_row.div(rem);
  br = (int)row;
  bc_first = G.run_len * (int)(rem - row * G.runs_per_row);
  nblk = min(G.run_len, G.cols - bc_first);
}

template <bool kWeights, bool kPayload, bool kDecode, bool kLowCols = false, int kSweep = 0>
__global__ void __launch_bounds__(kM16Threads, 3)
sense16_kernel(Grid16 G, Sense16Args A) {
  __shared__ __align__(16) uint8_t s_stage[kM16Warps][512];
  constexpr int kWbuf = kSweep > 0 ? 272 : 256;  // sweep: the second block's buffer 16 banks over
  __shared__ float s_buf[kM16Warps][2][kWbuf];
  __shared__ uint2 s_btab[kWeights ? 8 * 32 : 1];  // stage-2 basis B pairs (fill_btab16), weights pass only
  // sweep: per rank e = 16 i + kl each plan's band edge hi (s_thr[e]) and lo (s_thr[128 + e]), +inf
  // where the rank lies outside that plan's phase-1 prefix (membership folded into the threshold)
  __shared__ float4 s_thr[kSweep > 0 ? 8 * 16 * 2 : 1];
  Frag16 f;
  load_frag16(f);
  if constexpr (kWeights) {  // (measured: a win for the weights pass, a loss for the fused decode pass)
    if (threadIdx.x < 32) fill_btab16(f, s_btab);
    if constexpr (kSweep > 0) {
      for (int e = threadIdx.x; e < 8 * 16; e += blockDim.x) {
        float h[4], l[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const bool in = j < kSweep && e < A.sw_phase1[j];  // e = 16 i + kl = the rank
          h[j] = in ? A.sw_hi[j] : INFINITY;
          l[j] = in ? A.sw_lo[j] : INFINITY;
        }
        s_thr[e] = make_float4(h[0], h[1], h[2], h[3]);
        s_thr[8 * 16 + e] = make_float4(l[0], l[1], l[2], l[3]);
      }
    }
    __syncthreads();
  }
  // The forward runs transposed (Y^T = C X^T C^T): D slot s holds Y[dslot_col(s)][dslot_row(s)].
  uint32_t rank_d[8];
  float thr_hi[kWeights ? 8 : 1], thr_lo[kWeights ? 8 : 1];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    rank_d[s] = zigzag_rank_dev<16>()[dslot_col(s) * 16 + dslot_row(s)];
    if constexpr (kSweep > 0) rank_d[s] = (rank_d[s] & ~31u) | kZzBank16[rank_d[s]];  // store address
    if constexpr (kWeights && !kSweep) {
      const bool in = (int)rank_d[s] < A.phase1;
      thr_hi[s] = in ? A.Tf + A.band : INFINITY;
      thr_lo[s] = in ? A.Tf - A.band : INFINITY;
    }
  }
  // sweep: plan j's phase-1 prefix and band, hoisted; P = the widest prefix
  int sw_ph1[kSweep > 0 ? kSweep : 1];
  float sw_hi[kSweep > 0 ? kSweep : 1], sw_lo[kSweep > 0 ? kSweep : 1];
  int sw_P = 0;
  uint32_t sw_addr[2] = {0u, 0u};  // read address of test group i (8 bits each): rank 16 i + kl
  if constexpr (kSweep > 0) {
#pragma unroll
    for (int j = 0; j < kSweep; ++j) {
      sw_ph1[j] = A.sw_phase1[j];
      sw_hi[j] = A.sw_hi[j];
      sw_lo[j] = A.sw_lo[j];
      sw_P = max(sw_P, sw_ph1[j]);
    }
    const int kl = threadIdx.x & 15;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int k = 16 * i + kl;
      sw_addr[i >> 2] |= ((uint32_t)(k & ~31) | kZzBank16[k]) << (8 * (i & 3));
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* st = s_stage[warp];
  float* zb0 = &s_buf[warp][0][0];
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < G.total_runs; r += nwarps) {
    uint32_t img;
    int br, bcf, nblk;
    run_pos(G, r, img, br, bcf, nblk);
    const uint32_t bidx_first = img * G.nb + (uint32_t)(br * G.cols + bcf);
    // lane i <-> block bcf + i of the run: counts/offsets in one coalesced load each
    int my_cnt = 0;
    int32_t my_off = 0;
    if constexpr (kPayload || kDecode) {
      if (lane < nblk) {
        my_cnt = A.counts[bidx_first + lane];
        if constexpr (kPayload) my_off = A.offsets[bidx_first + lane];
      }
    }
    const uint8_t* rowp = run_row_ptr(A.imgs, A.img_stride, A.pitch, img, br, bcf);
    uint4 nxt = load_row16_at(rowp, (lane >> 4) < nblk, A.aligned);
    for (int p = 0; 2 * p < nblk; ++p) {
      const int bc0 = bcf + 2 * p;
      const bool two = 2 * p + 1 < nblk;
      __syncwarp();
      reinterpret_cast<uint4*>(st)[lane] = interleave_row16(nxt);
      __syncwarp();
      if (2 * p + 2 < nblk) nxt = load_row16_at(rowp + 32 * (p + 1), 2 * p + 2 + (lane >> 4) < nblk, A.aligned);
      uint32_t bx[2][2][2];
      u8_bfragT_il(st, bx[0]);
      u8_bfragT_il(st + 256, bx[1]);
      Acc16 Y[2];  // Y^T of each block
      // payload pass: when both blocks keep <= 36 coefficients their zigzag prefixes lie in the
      // top-left 8x8 (slots 0/1), so the low-quadrant transforms suffice (warp-uniform choice)
      bool lo_pair = false;
      if constexpr (kPayload && !kWeights) {
        const int c0 = __shfl_sync(0xffffffffu, my_cnt, 2 * p);
        const int c1 = two ? __shfl_sync(0xffffffffu, my_cnt, (2 * p + 1) & 31) : 0;
        lo_pair = c0 <= 36 && c1 <= 36;
      }
      if constexpr (kLowCols) dct16_fwd_exact_x2_lo(f, bx, Y);
      else if constexpr (kWeights) dct16_fwd_exact_x2_tab(f, s_btab, bx, Y);
      else if (lo_pair) dct16_fwd_exact_x2_lo(f, bx, Y);
      else dct16_fwd_exact_x2(f, bx, Y);
      const uint32_t bidx0 = bidx_first + 2 * p;
      if constexpr (kSweep > 0) {
        // DD phase 1 of kSweep plans by zigzag compaction: the pair's coefficients of rank < P go to
        // the warp's rank-ordered buffer and lane L tests ranks (L & 15) + 16 i of
        // block L >> 4 against each plan (prefix phase1_j, band around T_j): 2P / 32 coefficients
        // per lane instead of 8 slots per plan, most of them outside every prefix. A zigzag prefix
        // of <= 136 entries lies in slots 0-5 (u + v <= 15), so slots 6-7 are stored only beyond.
        // Bank-permuted rows (kZzBank16) with the second block 16 banks over: every store slot and
        // every test read is one wavefront.
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int s = 0; s < 8; ++s)
            if (s < 6 || sw_P > 136) zb0[kWbuf * q + rank_d[s]] = Y[q].v[s >> 2][s & 3];
        __syncwarp();
        const int qb = lane >> 4, kl = lane & 15;
        const float* zq = zb0 + kWbuf * qb;
        // per plan j (byte j): coefficients at or above T_j + band (counted) and above T_j - band;
        // the two words differ iff some coefficient is near T_j (inside the band)
        uint32_t packed = 0, above_lo = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (16 * i >= sw_P) break;
          const float a = fabsf(zq[(sw_addr[i >> 2] >> (8 * (i & 3))) & 255u]);
          const float4 th = s_thr[16 * i + kl], tl = s_thr[8 * 16 + 16 * i + kl];  // conflict-free
          const float hv[4] = {th.x, th.y, th.z, th.w}, lv[4] = {tl.x, tl.y, tl.z, tl.w};
#pragma unroll
          for (int j = 0; j < kSweep; ++j)
            asm("{\n .reg .pred ph, pl;\n setp.ge.f32 ph, %2, %4;\n setp.gt.f32 pl, %2, %5;\n"
                " @ph add.u32 %0, %0, %3;\n @pl add.u32 %1, %1, %3;\n}"
                : "+r"(packed), "+r"(above_lo)
                : "f"(a), "r"(1u << (8 * j)), "f"(hv[j]), "f"(lv[j]));
        }
        bool nr = packed != above_lo;
        if (qb == 1 && !two) {
          packed = 0;
          nr = false;
        }
        const uint32_t sig0 = __reduce_add_sync(0xffffffffu, qb == 0 ? packed : 0u);
        const uint32_t sig1 = __reduce_add_sync(0xffffffffu, qb == 1 ? packed : 0u);
        if (__any_sync(0xffffffffu, nr)) {  // rare: record each plan's near-threshold coefficients
          if (nr) {
#pragma unroll 1
            for (int j = 0; j < kSweep; ++j) {
              bool mine = false;
#pragma unroll 1
              for (int i = 0; 16 * i < sw_P; ++i) {
                const int k = kl + 16 * i;
                const float a = fabsf(zq[(k & ~31) | kZzBank16[k]]);
                if (k < sw_ph1[j] && !(a >= sw_hi[j]) && a > sw_lo[j]) {
                  mine = true;
                  const uint32_t e = atomicAdd(A.sw_fix_count[j], 1u);
                  if (e < A.fix_cap) {
                    A.sw_fix_list[j][2 * e] = bidx0 + qb;
                    A.sw_fix_list[j][2 * e + 1] = zigzag_dev<16>()[k];  // flat u * 16 + v
                  }
                }
              }
              if (mine) A.sw_fix_flag[j][bidx0 + qb] = 1;
            }
          }
        }
        if (lane < kSweep) {
          uint32_t* w = A.sw_weights[lane];
          w[bidx0] = (sig0 >> (8 * lane)) & 255u;
          if (two) w[bidx0 + 1] = (sig1 >> (8 * lane)) & 255u;
        }
      } else if constexpr (kWeights) {
        // phase-1 test in registers: slot s is in the prefix iff rank_d[s] < phase1 (thresholds
        // pre-masked to +inf outside it); counts reduce across the warp. A coefficient within the
        // MMA error band of T is neither counted nor dropped: dd_fixup16_kernel decides it in fp64.
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (q == 1 && !two) break;
          int cnt = 0;
          bool nr = false;
#pragma unroll
          for (int s = 0; s < (kLowCols ? 2 : 8); ++s) {
            const float a = fabsf(Y[q].v[s >> 2][s & 3]);
            const bool hi = a >= thr_hi[s];
            cnt += hi ? 1 : 0;
            nr |= !hi && a > thr_lo[s];
          }
          const int sig = (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt);
          if (__any_sync(0xffffffffu, nr)) {  // rare: record the near-threshold coefficients
            if (nr) {
              A.fix_flag[bidx0 + q] = 1;
#pragma unroll
              for (int s = 0; s < (kLowCols ? 2 : 8); ++s) {
                const float a = fabsf(Y[q].v[s >> 2][s & 3]);
                if (!(a >= thr_hi[s]) && a > thr_lo[s]) {
                  const uint32_t e = atomicAdd(A.fix_count, 1u);
                  if (e < A.fix_cap) {
                    A.fix_list[2 * e] = bidx0 + q;
                    A.fix_list[2 * e + 1] = (uint32_t)(dslot_col(s) * 16 + dslot_row(s));  // flat u*16+v
                  }
                }
              }
            }
          }
          if (lane == 0) A.weights[bidx0 + q] = (uint32_t)sig;
        }
      }
      if constexpr (kPayload || kDecode) {
        int cnt[2];
        cnt[0] = __shfl_sync(0xffffffffu, my_cnt, 2 * p);
        cnt[1] = two ? __shfl_sync(0xffffffffu, my_cnt, (2 * p + 1) & 31) : 0;
        if constexpr (kPayload) {
          // zigzag-ordered copy in smem -> coalesced prefix writes
#pragma unroll
          for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int s = 0; s < 8; ++s)
              if (s < 2 || !lo_pair) zb0[kWbuf * q + rank_d[s]] = Y[q].v[s >> 2][s & 3];
          __syncwarp();
          // the pair's prefixes are adjacent in the payload (offset1 = offset0 + cnt0): one
          // coalesced copy of cnt0 + cnt1 values, two loads in flight per iteration
          const int32_t o0 = __shfl_sync(0xffffffffu, my_off, 2 * p);
          float* dst = A.payload + (int64_t)img * A.payload_stride + o0;
          const int total = cnt[0] + cnt[1], skip = kWbuf - cnt[0];
#pragma unroll 1
          for (int k = lane; k < total; k += 64) {
            const int k2 = k + 32;
            const float v0 = zb0[k < cnt[0] ? k : k + skip];
            float v1 = 0.f;
            if (k2 < total) v1 = zb0[k2 < cnt[0] ? k2 : k2 + skip];
            dst[k] = v0;
            if (k2 < total) dst[k2] = v1;
          }
          __syncwarp();
        }
        if constexpr (kDecode) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (q == 1 && !two) break;
            Acc16 Ym;  // zero the coefficients outside the block's zigzag prefix
#pragma unroll
            for (int s = 0; s < 8; ++s) Ym.v[s >> 2][s & 3] = (int)rank_d[s] < cnt[q] ? Y[q].v[s >> 2][s & 3] : 0.f;
            const Acc16 X = lo_pair ? dct16_inv_from_yt_lo(f, Ym) : dct16_inv_from_yt(f, Ym);
            store_dfrag(A.out + (int64_t)img * A.out_stride + (int64_t)(br * 16) * A.out_pitch + (bc0 + q) * 16,
                        A.out_pitch, X);
          }
        }
      }
    }
  }
}

constexpr float kMmaSafeMax = 8192.f;  // |coef| bound keeping the fp16 split in range

// decode_idct from a packed payload. A warp walks a run of up to 32 consecutive
// blocks of a block-row: counts/offsets arrive in one coalesced load (lane i <->
// block i) and each block's prefix (8 values per lane at most) is prefetched
// one block ahead while the current block is transformed.
__global__ void __launch_bounds__(kM16Threads, 3)
decode16_kernel(Grid16 G, uint32_t total_blocks, const uint16_t* __restrict__ counts,
                const int32_t* __restrict__ offsets, const float* __restrict__ payload, int64_t payload_stride,
                float* __restrict__ out, int64_t out_stride, int out_pitch) {
  __shared__ float s_buf[kM16Warps][256];
  Frag16 f;
  load_frag16(f);
  uint32_t rank_b[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) rank_b[s] = zigzag_rank_dev<16>()[bslot_row(s) * 16 + bslot_col(s)];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* zb = s_buf[warp];
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < G.total_runs; r += nwarps) {
    uint32_t img;
    int br, bcf, nblk;
    run_pos(G, r, img, br, bcf, nblk);
    const uint32_t bidx_first = img * G.nb + (uint32_t)(br * G.cols + bcf);
    const int my_cnt = lane < nblk ? counts[bidx_first + lane] : 0;
    const int32_t my_off = lane < nblk ? offsets[bidx_first + lane] : 0;
    const float* base = payload + (int64_t)img * payload_stride;
    float* obase = out + (int64_t)img * out_stride + (int64_t)(br * 16) * out_pitch;
    int c0 = __shfl_sync(0xffffffffu, my_cnt, 0);
    const float* s0 = base + __shfl_sync(0xffffffffu, my_off, 0);
    float pv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) pv[q] = lane + 32 * q < c0 ? __ldg(s0 + lane + 32 * q) : 0.f;
    for (int i = 0; i < nblk; ++i) {
      // prefetch block i+1
      float pn[8];
      const int c1 = __shfl_sync(0xffffffffu, my_cnt, (i + 1) & 31);
      const float* s1 = base + __shfl_sync(0xffffffffu, my_off, (i + 1) & 31);
      const bool more = i + 1 < nblk;
#pragma unroll
      for (int q = 0; q < 8; ++q) pn[q] = (more && lane + 32 * q < c1) ? __ldg(s1 + lane + 32 * q) : 0.f;
      bool big = false;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (lane + 32 * q < c0) zb[lane + 32 * q] = pv[q];
        big |= !(fabsf(pv[q]) <= kMmaSafeMax);
      }
      __syncwarp();
      float yv[2][4];
#pragma unroll
      for (int s = 0; s < 8; ++s) yv[s >> 2][s & 3] = (int)rank_b[s] < c0 ? zb[rank_b[s]] : 0.f;
      __syncwarp();
      float scale = 1.f;
      if (__any_sync(0xffffffffu, big)) {
        // rare: rescale by a power of two so the fp16 split stays in range (exact)
        float mx = 0.f;
#pragma unroll
        for (int s = 0; s < 8; ++s) mx = fmaxf(mx, fabsf(yv[s >> 2][s & 3]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (isfinite(mx) && mx > kMmaSafeMax) {
          int e;
          frexpf(mx / kMmaSafeMax, &e);
          scale = ldexpf(1.f, e);
#pragma unroll
          for (int s = 0; s < 8; ++s) yv[s >> 2][s & 3] = ldexpf(yv[s >> 2][s & 3], -e);
        }
      }
      Acc16 X = dct16_inv_f32(f, yv);
      if (scale != 1.f) {
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k) X.v[j][k] *= scale;
      }
      store_dfrag(obase + (bcf + i) * 16, out_pitch, X);
      c0 = c1;
#pragma unroll
      for (int q = 0; q < 8; ++q) pv[q] = pn[q];
    }
  }
}

// fp64 decision for the (rare) phase-1 coefficients whose MMA value came within
// the error band of T: one thread per listed (block, coefficient), computed in the
// reference's exact operation order (dct.cpp:30-49) with no FMA contraction and
// the reference basis, |c| > T strict (sensing.cpp:354). Should the list overflow
// (only adversarial inputs: capacity is 2 entries per block), every flagged block
// is recounted in full in fp64 instead.
struct FixPlans {  // plan j = blockIdx.y
  int phase1[4];
  double T[4];
  const uint32_t* list[4];
  const uint32_t* count[4];
  const uint8_t* flags[4];
  uint32_t* weights[4];
};
__global__ void __launch_bounds__(256)
dd_fixup16_kernel(const uint8_t* __restrict__ imgs, int64_t img_stride, int pitch, Grid16 G, FixPlans F, uint32_t cap,
                  uint32_t total_blocks) {
  const int j = blockIdx.y;
  const int phase1 = F.phase1[j];
  const double T = F.T[j];
  const uint32_t* __restrict__ list = F.list[j];
  const uint8_t* __restrict__ flags = F.flags[j];
  uint32_t* __restrict__ weights = F.weights[j];
  const uint32_t n = *F.count[j];
  const double* C = basis_dev<16>();
  const int lane = threadIdx.x & 31, c = lane & 15;
  const unsigned half = 0xffffu << (lane & 16);
  if (n <= cap) {
    // 16 lanes per entry: lane c forms tmp[u][c] = sum_r C[u][r] x[r][c] (r ascending), then the
    // group's first lane accumulates y = sum_c tmp[u][c] C[v][c] in c order -- the reference's order.
    const uint32_t groups = (gridDim.x * blockDim.x) >> 4;
    for (uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 4; e < ((n + 1) & ~1u); e += groups) {
      const bool valid = e < n;
      const uint32_t bidx = valid ? list[2 * e] : 0;
      const int flat = valid ? (int)list[2 * e + 1] : 0;
      const int u = flat >> 4, v = flat & 15;
      const uint32_t img = G.div_nb.div(bidx);
      const uint32_t bi = bidx - img * G.nb;
      const uint32_t br = G.div_cols.div(bi), bc = bi - br * (uint32_t)G.cols;
      const uint8_t* col = imgs + (int64_t)img * img_stride + (int64_t)(br * 16) * pitch + bc * 16 + c;
      double x[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) x[r] = valid ? (double)col[(size_t)r * pitch] : 0.0;
      double t = 0.0;
#pragma unroll
      for (int r = 0; r < 16; ++r) t = __dadd_rn(t, __dmul_rn(C[u * 16 + r], x[r]));
      double y = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) y = __dadd_rn(y, __dmul_rn(__shfl_sync(half, t, k, 16), C[v * 16 + k]));
      if (valid && c == 0 && fabs(y) > T) atomicAdd(weights + bidx, 1u);
    }
    return;
  }
  const unsigned short* zz = zigzag_dev<16>();
  for (uint32_t bidx = blockIdx.x * blockDim.x + threadIdx.x; bidx < total_blocks; bidx += gridDim.x * blockDim.x) {
    if (!flags[bidx]) continue;
    const uint32_t img = G.div_nb.div(bidx);
    const uint32_t bi = bidx - img * G.nb;
    const uint32_t br = G.div_cols.div(bi), bc = bi - br * (uint32_t)G.cols;
    const uint8_t* blk = imgs + (int64_t)img * img_stride + (int64_t)(br * 16) * pitch + bc * 16;
    uint32_t sig = 0;
    for (int k = 0; k < phase1; ++k) sig += fabs(exact_coef16(blk, pitch, zz[k])) > T ? 1u : 0u;
    weights[bidx] = sig;
  }
}

// Allocation of DD plans from computed weights: one warp per image (warp_alloc.cuh), four
// images per CTA; ABCS_ALLOC_CTA=1 selects the 256-thread CTA allocator (cta_alloc.cuh).
constexpr int kWarpAllocWarps = 4;
static bool alloc_use_cta() {
  static const int v = [] {
    const char* e = getenv("ABCS_ALLOC_CTA");
    return e && e[0] == '1' ? 1 : 0;
  }();
  return v != 0;
}
static int warp_alloc_smem(int nb) { return kWarpAllocWarps * warp_alloc_bytes(nb); }
static void warp_alloc_attr(const void* k) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, warp_alloc_smem(kCtaAllocMaxBlocks));
}

__global__ void __launch_bounds__(32 * kWarpAllocWarps)
alloc_warp_kernel(const uint32_t* __restrict__ weights, int nb, int n, int wmax, long long budget, int cap, int base,
                  uint16_t* __restrict__ counts, int32_t* __restrict__ offsets, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char wsm[];
  const int warp = threadIdx.x >> 5, img = blockIdx.x * kWarpAllocWarps + warp;
  if (img >= n) return;
  const int st = warp_allocate(wsm + warp * warp_alloc_bytes(nb), weights + (int64_t)img * nb, nb, wmax, budget, cap,
                               base, counts + (int64_t)img * nb, offsets + (int64_t)img * nb);
  if ((threadIdx.x & 31) == 0 && status) status[img] = st;
}

// Allocation for the fused DD path: one CTA per image (cta_alloc.cuh).
__global__ void __launch_bounds__(kCtaAllocThreads, 7)
alloc_cta_kernel(const uint32_t* __restrict__ weights, int nb, int wmax, long long budget, int cap, int base,
                 uint16_t* __restrict__ counts, int32_t* __restrict__ offsets, int32_t* __restrict__ status) {
  __shared__ CtaAllocSmem S;
  const int img = blockIdx.x;
  const int st = cta_allocate(S, weights + (int64_t)img * nb, nb, wmax, budget, cap, base, counts + (int64_t)img * nb,
                              offsets + (int64_t)img * nb);
  if (threadIdx.x == 0 && status) status[img] = st;
}

// ---------------------------------------------------------------------------
// Grid-stride CTAs: two full waves of `per_sm` resident CTAs per SM (equal work per CTA).
static unsigned grid_for(Ctx* ctx, uint32_t warps_needed, uint32_t per_sm = 3, uint32_t dflt_waves = 2) {
  const uint32_t ctas = (warps_needed + kM16Warps - 1) / kM16Warps;
  static const int env_waves = [] {
    const char* e = getenv("ABCS_GRID_WAVES");  // 0 = one run per warp (no grid-stride)
    return e ? atoi(e) : -1;
  }();
  const uint32_t waves = env_waves >= 0 ? (uint32_t)env_waves : dflt_waves;
  if (waves == 0) return ctas ? ctas : 1;
  const uint32_t cap = (uint32_t)ctx->sm_count * per_sm * waves;
  return ctas < cap ? (ctas ? ctas : 1) : cap;
}


// ---------------------------------------------------------------------------
// B = 8 on the tensor cores (mma_dct.cuh Frag8: two 8x8 blocks per warp-MMA).
//  * kFromImage: u8 blocks -> Y (forward, exact u8 operands) -> zigzag prefix payload
//    (gather_prefixes, sensing.cpp:192-227); kDecode additionally inverts the masked Y
//    straight from the accumulators (decode_idct, recon.cpp:109-117).
//  * !kFromImage: decode_idct from a packed payload.
// A warp walks a run of <= 32 consecutive blocks of a block-row in quads of 8 blocks: lane
// L stages row L%8 of the block pair L/8 (16 bytes, rows interleaved so each lane's
// fragment bytes are one 32-bit word); the quad's 8 prefixes are contiguous in the payload
// and go through a per-warp smem buffer for one coalesced copy.
constexpr int kQuadFloats = 8 * 64;

template <bool kFromImage, bool kDecode>
__global__ void __launch_bounds__(kM16Threads, 4)
sense8_kernel(Grid16 G, Sense16Args A) {
  __shared__ __align__(16) uint8_t s_stage[kM16Warps][512];
  __shared__ float s_buf[kM16Warps][kQuadFloats];
  Frag8 f;
  load_frag8(f);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  uint32_t rank[2];  // Y^T slot e of a block: row g, col 2t+e -> Y[2t+e][g]
#pragma unroll
  for (int e = 0; e < 2; ++e) rank[e] = zigzag_rank_dev<8>()[(2 * t + e) * 8 + g];
  uint8_t* st = s_stage[warp];
  float* zb = s_buf[warp];
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < G.total_runs; r += nwarps) {
    uint32_t img;
    int br, bcf, nblk;
    run_pos(G, r, img, br, bcf, nblk);
    const uint32_t bidx_first = img * G.nb + (uint32_t)(br * G.cols + bcf);
    const int my_cnt = lane < nblk ? A.counts[bidx_first + lane] : 0;
    const int32_t my_off = lane < nblk ? A.offsets[bidx_first + lane] : 0;
    int tot;
    const int my_pre = warp_excl_scan(my_cnt, tot);  // prefix of the run's counts (lane = block)
    // the quad's image rows: lane -> pair L/8, row L%8 (16 bytes = blocks 2p, 2p+1 of the quad);
    // the next quad's row is loaded while the current one is transformed (its latency hidden)
    auto quad_row = [&](int qb) {
      const int pp = lane >> 3, row = lane & 7;
      const int b = qb + 2 * pp;  // run-relative block
      uint4 v = make_uint4(0, 0, 0, 0);
      if (b < nblk) {
        const uint8_t* src = A.imgs + (int64_t)img * A.img_stride + (int64_t)(br * 8 + row) * A.pitch + (bcf + b) * 8;
        const bool both = b + 1 < nblk;
        if (A.aligned && both) {
          v = __ldg(reinterpret_cast<const uint4*>(src));
        } else {
          uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (q < 8 || both) w[q >> 2] |= (uint32_t)src[q] << (8 * (q & 3));
          v = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      return v;
    };
    uint4 vnext = make_uint4(0, 0, 0, 0);
    if constexpr (kFromImage) vnext = quad_row(0);
    for (int qb = 0; qb < nblk; qb += 8) {
      const int pre0 = __shfl_sync(0xffffffffu, my_pre, qb);
      const int32_t off0 = __shfl_sync(0xffffffffu, my_off, qb);
      const int qend = min(qb + 8, nblk);
      const int qtot = (qend < 32 ? __shfl_sync(0xffffffffu, my_pre, qend & 31) : tot) - pre0;
      if constexpr (kFromImage) {
        __syncwarp();
        reinterpret_cast<uint4*>(st)[lane] = interleave_row16(vnext);
        __syncwarp();
        if (qb + 8 < nblk) vnext = quad_row(qb + 8);
      } else {
        // the quad's prefixes (contiguous in the payload) -> smem, coalesced
        const float* src = A.payload + (int64_t)img * A.payload_stride + off0;
        __syncwarp();
        for (int k = lane; k < qtot; k += 32) zb[k] = __ldg(src + k);
        __syncwarp();
      }
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) {
        const int b = qb + 2 * pp;
        if (b >= nblk) break;
        const bool two = b + 1 < nblk;
        const int c0 = __shfl_sync(0xffffffffu, my_cnt, b & 31);
        const int c1 = two ? __shfl_sync(0xffffffffu, my_cnt, (b + 1) & 31) : 0;
        const int p0 = __shfl_sync(0xffffffffu, my_pre, b & 31) - pre0;
        const int p1 = p0 + c0;
        float Y[4];
        if constexpr (kFromImage) {
          const uint32_t w = *reinterpret_cast<const uint32_t*>(st + pp * 128 + g * 16 + 4 * t);
          dct8x2_fwdT_exact(f, u8sel_to_h2(w, 0x4140), u8sel_to_h2(w, 0x4342), Y);
          // zigzag-ordered prefix of each block -> the quad buffer
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if ((int)rank[e] < c0) zb[p0 + rank[e]] = Y[e];
            if ((int)rank[e] < c1) zb[p1 + rank[e]] = Y[2 + e];
          }
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            Y[e] = (int)rank[e] < c0 ? zb[p0 + rank[e]] : 0.f;
            Y[2 + e] = (int)rank[e] < c1 ? zb[p1 + rank[e]] : 0.f;
          }
        }
        if constexpr (kDecode) {
          float Ym[4];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            Ym[e] = (int)rank[e] < c0 ? Y[e] : 0.f;
            Ym[2 + e] = (int)rank[e] < c1 ? Y[2 + e] : 0.f;
          }
          float X[4];
          dct8x2_inv_from_yt(f, Ym, X);
          float* o = A.out + (int64_t)img * A.out_stride + (int64_t)(br * 8 + g) * A.out_pitch + (bcf + b) * 8 + 2 * t;
          *reinterpret_cast<float2*>(o) = make_float2(X[0], X[1]);
          if (two) *reinterpret_cast<float2*>(o + 8) = make_float2(X[2], X[3]);
        }
      }
      if constexpr (kFromImage) {
        __syncwarp();
        float* dst = A.payload + (int64_t)img * A.payload_stride + off0;
        for (int k = lane; k < qtot; k += 32) dst[k] = zb[k];
      }
      __syncwarp();
    }
  }
}

int launch_sense8(Ctx* ctx, bool from_image, bool decode, int rows, int cols, int n, const uint8_t* imgs,
                  int64_t img_stride, int pitch, const uint16_t* counts, const int32_t* offsets, float* payload,
                  int64_t payload_stride, float* out, int64_t out_stride, int out_pitch, cudaStream_t s) {
  const Grid16 G = make_grid16(rows, cols, n);
  if (G.total_runs == 0) return ABCS_OK;
  Sense16Args A{};
  A.imgs = imgs;
  A.img_stride = img_stride;
  A.pitch = pitch;
  A.aligned = imgs && ((uintptr_t)imgs % 16 == 0) && (img_stride % 16 == 0) && (pitch % 16 == 0);
  A.counts = counts;
  A.offsets = offsets;
  A.payload = payload;
  A.payload_stride = payload_stride;
  A.out = out;
  A.out_stride = out_stride;
  A.out_pitch = out_pitch;
  const unsigned grid = grid_for(ctx, G.total_runs, 4, 4);  // cfg3: 1.100 ms at 2 rounds, 1.080 at 4
  const char* name = from_image ? (decode ? "sense8_gather_decode" : "sense8_gather") : "decode8";
  const int kt = ktimer_begin(ctx, s, name);
  if (from_image && decode) sense8_kernel<true, true><<<grid, kM16Threads, 0, s>>>(G, A);
  else if (from_image) sense8_kernel<true, false><<<grid, kM16Threads, 0, s>>>(G, A);
  else sense8_kernel<false, true><<<grid, kM16Threads, 0, s>>>(G, A);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "sense8 launch");
}

bool mma16_supported(int rows, int cols, int n) {
  const uint64_t blocks = (uint64_t)rows * cols * (uint64_t)n;
  return blocks < (1ull << 31);
}

bool fused_alloc_supported(Ctx* ctx, int rows, int cols, int n, int wmax) {
  (void)ctx;
  return (int64_t)rows * cols <= kCtaAllocMaxBlocks && wmax <= kCtaAllocMaxW &&
         mma16_supported(rows, cols, n);
}

int launch_sense16(Ctx* ctx, int mode, int rows, int cols, int n, const uint8_t* imgs, int64_t img_stride, int pitch,
                   int phase1, double T, uint32_t* weights, const uint16_t* counts, const int32_t* offsets,
                   float* payload, int64_t payload_stride, float* out, int64_t out_stride, int out_pitch,
                   cudaStream_t s, uint32_t* fix_scratch, const FusedAlloc* fa) {
  const Grid16 G = make_grid16(rows, cols, n);
  if (G.total_units == 0) return ABCS_OK;
  Sense16Args A{};
  A.imgs = imgs;
  A.img_stride = img_stride;
  A.pitch = pitch;
  A.aligned = ((uintptr_t)imgs % 16 == 0) && (img_stride % 16 == 0) && (pitch % 16 == 0);
  A.phase1 = phase1;
  A.T = T;
  A.Tf = (float)T;
  A.band = (float)(1e-2 + fabs(T - (double)A.Tf));  // >= worst-case MMA transform error + rounding of T
  A.weights = weights;
  if (mode == 1) {
    if (!fix_scratch) return set_error(ABCS_ERR_LOGIC, "sense16: missing fixup scratch");
    const int64_t nbt = (int64_t)G.nb * n;
    A.fix_count = fix_scratch;
    A.fix_list = fix_scratch + 4;
    A.fix_cap = (uint32_t)(nbt * 2);
    A.fix_flag = reinterpret_cast<uint8_t*>(fix_scratch + 4 + 2 * (int64_t)A.fix_cap);
    cudaError_t e = cudaMemsetAsync(A.fix_count, 0, 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(A.fix_flag, 0, (size_t)nbt, s);
    if (e != cudaSuccess) return cuda_status(e, "fixup reset");
  }
  A.counts = counts;
  A.offsets = offsets;
  A.payload = payload;
  A.payload_stride = payload_stride;
  A.out = out;
  A.out_stride = out_stride;
  A.out_pitch = out_pitch;
  const unsigned grid = grid_for(ctx, G.total_runs);
  int kt;
  switch (mode) {
    case 1:
      kt = ktimer_begin(ctx, s, "sense16_weights");
      if (phase1 <= 36)  // zigzag prefix of <= 36 entries lives in columns 0..7
        sense16_kernel<true, false, false, true><<<grid, kM16Threads, 0, s>>>(G, A);
      else
        sense16_kernel<true, false, false><<<grid, kM16Threads, 0, s>>>(G, A);
      ktimer_end(ctx, s, kt);
      ctx->launches++;
      kt = ktimer_begin(ctx, s, "dd_fixup16");
      {
      FixPlans F{};
      F.phase1[0] = phase1;
      F.T[0] = T;
      F.list[0] = A.fix_list;
      F.count[0] = A.fix_count;
      F.flags[0] = A.fix_flag;
      F.weights[0] = weights;
      dd_fixup16_kernel<<<(unsigned)ctx->sm_count, 256, 0, s>>>(imgs, img_stride, pitch, G, F, A.fix_cap,
                                                               G.nb * (uint32_t)n);
      }
      ktimer_end(ctx, s, kt);
      if (fa) {  // allocation: one CTA per image (cta_alloc.cuh)
        ctx->launches++;
        kt = ktimer_begin(ctx, s, "alloc_cta");
        if (alloc_use_cta()) {
          alloc_cta_kernel<<<(unsigned)n, kCtaAllocThreads, 0, s>>>(weights, (int)G.nb, fa->wmax, fa->budget, fa->cap,
                                                                     fa->base, fa->counts, fa->offsets, fa->status);
        } else {
          static bool attr = false;
          if (!attr) {
            warp_alloc_attr((const void*)alloc_warp_kernel);
            attr = true;
          }
          alloc_warp_kernel<<<(unsigned)((n + kWarpAllocWarps - 1) / kWarpAllocWarps), 32 * kWarpAllocWarps,
                              warp_alloc_smem((int)G.nb), s>>>(weights, (int)G.nb, n, fa->wmax, fa->budget, fa->cap,
                                                               fa->base, fa->counts, fa->offsets, fa->status);
        }
        ktimer_end(ctx, s, kt);
      }
      break;
    case 2:
      if (umma16_enabled())
        return launch_sense16_umma(ctx, 2, rows, cols, n, imgs, img_stride, pitch, counts, offsets, payload,
                                   payload_stride, nullptr, 0, 0, s);
      kt = ktimer_begin(ctx, s, "sense16_gather");
      sense16_kernel<false, true, false><<<grid, kM16Threads, 0, s>>>(G, A);
      ktimer_end(ctx, s, kt);
      break;
    case 3:
      if (umma16_enabled())
        return launch_sense16_umma(ctx, 3, rows, cols, n, imgs, img_stride, pitch, counts, offsets, payload,
                                   payload_stride, out, out_stride, out_pitch, s);
      kt = ktimer_begin(ctx, s, "sense16_gather_decode");
      sense16_kernel<false, true, true><<<grid, kM16Threads, 0, s>>>(G, A);
      ktimer_end(ctx, s, kt);
      break;
    default: return set_error(ABCS_ERR_LOGIC, "bad sense16 mode");
  }
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "sense16 launch");
}

// The sweep's payload passes in one: each block's forward transform (and its u8 read) is
// computed once and serves every plan (its zigzag prefix to that plan's payload, its masked
// inverse to that plan's decoded image). Per plan the arithmetic is sense16_kernel<0,1,1>'s, so
// the outputs are bit-identical to the per-plan launches.
struct MultiArgs {
  const uint8_t* imgs;
  int64_t img_stride;
  int pitch;
  bool aligned;
  int np;
  const uint16_t* counts[kMaxSweep];
  const int32_t* offsets[kMaxSweep];
  float* payload[kMaxSweep];
  int64_t payload_stride[kMaxSweep];
  float* out[kMaxSweep];
  int64_t out_stride;
  int out_pitch;
};

__device__ __forceinline__ int pick4(const int (&a)[kMaxSweep], int j) {
  return j == 0 ? a[0] : j == 1 ? a[1] : j == 2 ? a[2] : a[3];
}

// Decoded pixels of a block pair (16 x 32 fp32) leave through shared memory by one TMA tensor store
// per plan (cp.async.bulk.tensor, 3-D map of that plan's decoded batch): the warp moves on while
// the copy engine drains it, so bytes in flight no longer scale with the warps' own stores. The
// 2-KB staging tile uses the 128-B swizzle (16-B chunk ^ row), which makes the fragment writes
// bank-conflict free. Two tiles per warp alternate; a tile is rewritten only after its store has
// finished reading it (wait_group.read).
struct MultiMaps {
  CUtensorMap m[kMaxSweep];
};
__device__ __forceinline__ void stage_dfrag_sw(unsigned char* tile, int col0, const Acc16& X) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = g + 8 * h, col = col0 + 8 * j + 2 * t;
      const int off = row * 128 + (((col >> 2) ^ (row & 7)) << 4) + ((col & 3) << 2);
      *reinterpret_cast<float2*>(tile + off) = make_float2(X.v[j][2 * h], X.v[j][2 * h + 1]);
    }
}
__device__ __forceinline__ void tma_store_tile(const CUtensorMap* m, int x, int y, int z, const void* tile) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(m), "r"(x), "r"(y),
      "r"(z), "r"((uint32_t)__cvta_generic_to_shared(tile))
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

template <bool kBulk>
__global__ void __launch_bounds__(kM16Threads, 2)
sense16_multi_kernel(Grid16 G, MultiArgs A, const __grid_constant__ MultiMaps maps) {
  __shared__ __align__(16) uint8_t s_stage[kM16Warps][512];
  constexpr int kWbuf = 256;
  __shared__ float s_buf[kM16Warps][2][kWbuf];
  extern __shared__ __align__(1024) unsigned char s_out_raw[];  // kBulk: [warp][2] 2-KB swizzled tiles
  unsigned char* s_out = s_out_raw + ((1024 - ((uint32_t)__cvta_generic_to_shared(s_out_raw) & 1023)) & 1023);
  int tile_sel = 0;
  Frag16 f;
  load_frag16(f);
  uint32_t rank_d[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) rank_d[s] = zigzag_rank_dev<16>()[dslot_col(s) * 16 + dslot_row(s)];
  uint32_t rk[2][2];  // the ranks of YtSplit's slot pairs {0,1}, {4,5} / {2,3}, {6,7} as fp16x2
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 2; ++i)
      rk[j][i] = h2u(__floats2half2_rn((float)rank_d[2 * j + 4 * i], (float)rank_d[2 * j + 4 * i + 1]));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* st = s_stage[warp];
  float* zb0 = &s_buf[warp][0][0];
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < G.total_runs; r += nwarps) {
    uint32_t img;
    int br, bcf, nblk;
    run_pos(G, r, img, br, bcf, nblk);
    const uint32_t bidx_first = img * G.nb + (uint32_t)(br * G.cols + bcf);
    int my_cnt[kMaxSweep], my_off[kMaxSweep];
#pragma unroll
    for (int j = 0; j < kMaxSweep; ++j) {
      my_cnt[j] = 0;
      my_off[j] = 0;
      if (j < A.np && lane < nblk) {
        my_cnt[j] = A.counts[j][bidx_first + lane];
        my_off[j] = A.offsets[j][bidx_first + lane];
      }
    }
    const uint8_t* rowp = run_row_ptr(A.imgs, A.img_stride, A.pitch, img, br, bcf);
    uint4 nxt = load_row16_at(rowp, (lane >> 4) < nblk, A.aligned);
    for (int p = 0; 2 * p < nblk; ++p) {
      const int bc0 = bcf + 2 * p;
      const bool two = 2 * p + 1 < nblk;
      __syncwarp();
      reinterpret_cast<uint4*>(st)[lane] = interleave_row16(nxt);
      __syncwarp();
      if (2 * p + 2 < nblk) nxt = load_row16_at(rowp + 32 * (p + 1), 2 * p + 2 + (lane >> 4) < nblk, A.aligned);
      uint32_t bx[2][2][2];
      u8_bfragT_il(st, bx[0]);
      u8_bfragT_il(st + 256, bx[1]);
      int cnt0[kMaxSweep], cnt1[kMaxSweep];
      bool lo_all = true;
#pragma unroll
      for (int j = 0; j < kMaxSweep; ++j) {
        cnt0[j] = __shfl_sync(0xffffffffu, my_cnt[j], 2 * p);
        cnt1[j] = two ? __shfl_sync(0xffffffffu, my_cnt[j], (2 * p + 1) & 31) : 0;
        if (j < A.np) lo_all = lo_all && cnt0[j] <= 36 && cnt1[j] <= 36;
      }
      Acc16 Y[2];
      if (lo_all) dct16_fwd_exact_x2_lo(f, bx, Y);
      else dct16_fwd_exact_x2(f, bx, Y);
      // zigzag-ordered copy of both blocks (every plan's prefix is a prefix of it)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s < 2 || !lo_all) zb0[kWbuf * q + rank_d[s]] = Y[q].v[s >> 2][s & 3];
      // each block's Y^T split once into fp16 hi/lo; every plan masks the split halves
      YtSplit ys[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (lo_all) {
          split2(Y[q].v[0][0], Y[q].v[0][1], ys[q].h[0][0], ys[q].l[0][0]);
        } else {
          ys[q] = split_yt(Y[q]);
        }
      }
      __syncwarp();
#pragma unroll 1
      for (int j = 0; j < A.np; ++j) {
        // register arrays picked by a select chain: a dynamic index would put them in local memory
        const int32_t o0 = __shfl_sync(0xffffffffu, pick4(my_off, j), 2 * p);
        float* dst = A.payload[j] + (int64_t)img * A.payload_stride[j] + o0;
        const int c0 = pick4(cnt0, j), c1 = pick4(cnt1, j);
        // the pair's prefixes are adjacent in the payload: block 0's, then block 1's
#pragma unroll 2
        for (int k = lane; k < c0; k += 32) dst[k] = zb0[k];
        float* dst1 = dst + c0;
#pragma unroll 2
        for (int k = lane; k < c1; k += 32) dst1[k] = zb0[kWbuf + k];
        const bool lo_j = c0 <= 36 && c1 <= 36;
        // both blocks' inverses back to back (two independent MMA chains interleave); a lone last
        // block's partner is a zero block, clipped by the tensor map or skipped below
        const uint32_t ch0 = h2u(__floats2half2_rn((float)c0, (float)c0));
        const uint32_t ch1 = h2u(__floats2half2_rn((float)c1, (float)c1));
        Acc16 X[2];
        if (lo_j) {
          YtSplit m0, m1;
          const uint32_t k0 = h2_lt_mask(rk[0][0], ch0), k1 = h2_lt_mask(rk[0][0], ch1);
          m0.h[0][0] = ys[0].h[0][0] & k0;
          m0.l[0][0] = ys[0].l[0][0] & k0;
          m1.h[0][0] = ys[1].h[0][0] & k1;
          m1.l[0][0] = ys[1].l[0][0] & k1;
          X[0] = dct16_inv_from_split_lo(f, m0);
          X[1] = dct16_inv_from_split_lo(f, m1);
        } else {
          X[0] = dct16_inv_from_split(f, mask_yt(ys[0], rk, ch0));
          X[1] = dct16_inv_from_split(f, mask_yt(ys[1], rk, ch1));
        }
        if (kBulk) {
          if (lane == 0) bulk_wait_read1();  // this tile's store from two rounds ago
          __syncwarp();
          stage_dfrag_sw(s_out + (warp * 2 + tile_sel) * 2048, 0, X[0]);
          stage_dfrag_sw(s_out + (warp * 2 + tile_sel) * 2048, 16, X[1]);
        } else {
          float* o = A.out[j] + (int64_t)img * A.out_stride + (int64_t)(br * 16) * A.out_pitch + bc0 * 16;
          store_dfrag(o, A.out_pitch, X[0]);
          if (two) store_dfrag(o + 16, A.out_pitch, X[1]);
        }
        if (kBulk) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // st.shared -> async proxy
          __syncwarp();
          if (lane == 0) {  // a lone last block: the map clips the pair's second half (past the image)
            tma_store_tile(&maps.m[j], bc0 * 16, br * 16, (int)img, s_out + (warp * 2 + tile_sel) * 2048);
            bulk_commit();
          }
          tile_sel ^= 1;
        }
      }
      __syncwarp();
    }
  }
  if (kBulk && (threadIdx.x & 31) == 0) bulk_wait_all();  // smem must outlive the copies
}

// The payload pass's grid: one warp per run when ABCS_MULTI_WAVES=0 (no grid-stride tail),
// else grid_for's cap of `waves` rounds of 2 resident CTAs per SM.
static unsigned multi_grid(Ctx* ctx, uint32_t runs) {
  static const int waves = [] {
    const char* e = getenv("ABCS_MULTI_WAVES");
    return e ? atoi(e) : 3;  // the 3-chunk pipelined cfg2 step: 1.325 ms at 3, 1.341 at 2, 1.334 at 0
  }();
  const uint32_t ctas = (runs + kM16Warps - 1) / kM16Warps;
  if (waves <= 0) return ctas ? ctas : 1;
  const uint32_t cap = (uint32_t)ctx->sm_count * 2u * (uint32_t)waves;
  return ctas < cap ? (ctas ? ctas : 1) : cap;
}

int launch_sense16_multi(Ctx* ctx, int np, int rows, int cols, int n, const uint8_t* imgs, int64_t img_stride,
                         int pitch, const uint16_t* const* counts, const int32_t* const* offsets,
                         float* const* payload, const int64_t* payload_stride, float* const* out, int64_t out_stride,
                         int out_pitch, cudaStream_t s) {
  if (np < 1 || np > kMaxSweep) return set_error(ABCS_ERR_LOGIC, "sense16 multi: 1..4 plans");
  const Grid16 G = make_grid16(rows, cols, n);
  if (G.total_units == 0) return ABCS_OK;
  MultiArgs A{};
  A.imgs = imgs;
  A.img_stride = img_stride;
  A.pitch = pitch;
  A.aligned = ((uintptr_t)imgs % 16 == 0) && (img_stride % 16 == 0) && (pitch % 16 == 0);
  A.np = np;
  for (int j = 0; j < np; ++j) {
    A.counts[j] = counts[j];
    A.offsets[j] = offsets[j];
    A.payload[j] = payload[j];
    A.payload_stride[j] = payload_stride[j];
    A.out[j] = out[j];
  }
  A.out_stride = out_stride;
  A.out_pitch = out_pitch;
  bool bulk = (out_pitch % 4 == 0) && (out_stride % 4 == 0) && out_pitch >= cols * 16;  // 16-B aligned rows
  for (int j = 0; j < np; ++j) bulk = bulk && ((uintptr_t)out[j] % 16 == 0);
  if (const char* e = getenv("ABCS_MULTI_BULK")) bulk = bulk && e[0] != '0';
  MultiMaps maps;
  memset(&maps, 0, sizeof(maps));
  if (bulk) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                  &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        encode = nullptr;
    }
    for (int j = 0; j < np && bulk; ++j) {
      const cuuint64_t dims[3] = {(cuuint64_t)cols * 16, (cuuint64_t)rows * 16, (cuuint64_t)n};
      const cuuint64_t strides[2] = {(cuuint64_t)out_pitch * 4, (cuuint64_t)out_stride * 4};
      const cuuint32_t box[3] = {32, 16, 1}, estr[3] = {1, 1, 1};
      bulk = encode && encode(&maps.m[j], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out[j], dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  constexpr int kOutBytes = kM16Warps * 2 * 2048 + 1024;  // + alignment slack (swizzled tiles: 1024 B)
  static bool attr = false;
  if (bulk && !attr) {
    cudaFuncSetAttribute(sense16_multi_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kOutBytes);
    attr = true;
  }
  const int kt = ktimer_begin(ctx, s, "sense16_gather_decode");
  if (bulk)
    sense16_multi_kernel<true><<<multi_grid(ctx, G.total_runs), kM16Threads, kOutBytes, s>>>(G, A, maps);
  else
    sense16_multi_kernel<false><<<multi_grid(ctx, G.total_runs), kM16Threads, 0, s>>>(G, A, maps);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "sense16 multi launch");
}

// DD phase 1 of n_sw plans (same geometry, prefixes phase1[j], thresholds T[j]) from one
// forward transform per block; then the fp64 fixup of each plan's near-threshold list.
int launch_sense16_sweep(Ctx* ctx, int n_sw, int rows, int cols, int n, const uint8_t* imgs, int64_t img_stride,
                         int pitch, const int* phase1, const double* T, uint32_t* const* weights,
                         uint32_t* const* fix_scratch, cudaStream_t s) {
  if (n_sw < 1 || n_sw > kMaxSweep) return set_error(ABCS_ERR_LOGIC, "sense16 sweep: 1..4 plans");
  const Grid16 G = make_grid16(rows, cols, n);
  if (G.total_units == 0) return ABCS_OK;
  Sense16Args A{};
  A.imgs = imgs;
  A.img_stride = img_stride;
  A.pitch = pitch;
  A.aligned = ((uintptr_t)imgs % 16 == 0) && (img_stride % 16 == 0) && (pitch % 16 == 0);
  const int64_t nbt = (int64_t)G.nb * n;
  A.fix_cap = (uint32_t)(nbt * 2);
  A.n_sw = n_sw;
  for (int j = 0; j < n_sw; ++j) {
    if (phase1[j] < 0 || phase1[j] > 128) return set_error(ABCS_ERR_LOGIC, "sense16 sweep: phase-1 prefix above 128");
    const float Tf = (float)T[j];
    const float band = (float)(1e-2 + fabs(T[j] - (double)Tf));  // as launch_sense16
    A.sw_phase1[j] = phase1[j];
    A.sw_hi[j] = Tf + band;
    A.sw_lo[j] = Tf - band;
    A.sw_weights[j] = weights[j];
    A.sw_fix_count[j] = fix_scratch[j];
    A.sw_fix_list[j] = fix_scratch[j] + 4;
    A.sw_fix_flag[j] = reinterpret_cast<uint8_t*>(fix_scratch[j] + 4 + 2 * (int64_t)A.fix_cap);
    cudaError_t e = cudaMemsetAsync(A.sw_fix_count[j], 0, 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(A.sw_fix_flag[j], 0, (size_t)nbt, s);
    if (e != cudaSuccess) return cuda_status(e, "fixup reset");
  }
  int kt = ktimer_begin(ctx, s, "sense16_weights_sweep");
  const unsigned grid = grid_for(ctx, G.total_runs);
  switch (n_sw) {  // the plan count is a template argument: the per-coefficient tests fully unroll
    case 1: sense16_kernel<true, false, false, false, 1><<<grid, kM16Threads, 0, s>>>(G, A); break;
    case 2: sense16_kernel<true, false, false, false, 2><<<grid, kM16Threads, 0, s>>>(G, A); break;
    case 3: sense16_kernel<true, false, false, false, 3><<<grid, kM16Threads, 0, s>>>(G, A); break;
    default: sense16_kernel<true, false, false, false, 4><<<grid, kM16Threads, 0, s>>>(G, A); break;
  }
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "sense16 sweep launch");
  // every plan's fp64 fixup in one launch (plan j = blockIdx.y)
  FixPlans F{};
  for (int j = 0; j < n_sw; ++j) {
    F.phase1[j] = phase1[j];
    F.T[j] = T[j];
    F.list[j] = A.sw_fix_list[j];
    F.count[j] = A.sw_fix_count[j];
    F.flags[j] = A.sw_fix_flag[j];
    F.weights[j] = weights[j];
  }
  kt = ktimer_begin(ctx, s, "dd_fixup16");
  dd_fixup16_kernel<<<dim3((unsigned)(ctx->sm_count + n_sw - 1) / n_sw, (unsigned)n_sw), 256, 0, s>>>(
      imgs, img_stride, pitch, G, F, A.fix_cap, G.nb * (uint32_t)n);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "dd fixup launch");
}

// Several plans' allocations in one launch (plan j = blockIdx.y, image = blockIdx.x).
struct AllocPlans {
  const uint32_t* weights[4];
  FusedAlloc fa[4];
};
__global__ void __launch_bounds__(kCtaAllocThreads, 7)
alloc_cta_plans_kernel(AllocPlans P, int nb) {
  __shared__ CtaAllocSmem S;
  const int img = blockIdx.x, j = blockIdx.y;
  const FusedAlloc& fa = P.fa[j];
  const int st = cta_allocate(S, P.weights[j] + (int64_t)img * nb, nb, fa.wmax, fa.budget, fa.cap, fa.base,
                              fa.counts + (int64_t)img * nb, fa.offsets + (int64_t)img * nb);
  if (threadIdx.x == 0 && fa.status) fa.status[img] = st;
}

__global__ void __launch_bounds__(32 * kWarpAllocWarps)
alloc_warp_plans_kernel(AllocPlans P, int nb, int n) {
  extern __shared__ __align__(16) unsigned char wsm[];
  const int warp = threadIdx.x >> 5, img = blockIdx.x * kWarpAllocWarps + warp, j = blockIdx.y;
  if (img >= n) return;
  const FusedAlloc& fa = P.fa[j];
  const int st = warp_allocate(wsm + warp * warp_alloc_bytes(nb), P.weights[j] + (int64_t)img * nb, nb, fa.wmax,
                               fa.budget, fa.cap, fa.base, fa.counts + (int64_t)img * nb, fa.offsets + (int64_t)img * nb);
  if ((threadIdx.x & 31) == 0 && fa.status) fa.status[img] = st;
}

int launch_alloc_cta_plans(Ctx* ctx, int np, int rows, int cols, int n, uint32_t* const* weights,
                           const FusedAlloc* fa, cudaStream_t s) {
  if (np < 1 || np > 4) return set_error(ABCS_ERR_LOGIC, "alloc plans: 1..4 plans");
  const Grid16 G = make_grid16(rows, cols, n);
  if (G.total_units == 0) return ABCS_OK;
  AllocPlans P{};
  for (int j = 0; j < np; ++j) {
    P.weights[j] = weights[j];
    P.fa[j] = fa[j];
  }
  const int kt = ktimer_begin(ctx, s, "alloc_cta");
  if (alloc_use_cta()) {
    alloc_cta_plans_kernel<<<dim3((unsigned)n, (unsigned)np), kCtaAllocThreads, 0, s>>>(P, (int)G.nb);
  } else {
    static bool attr = false;
    if (!attr) {
      warp_alloc_attr((const void*)alloc_warp_plans_kernel);
      attr = true;
    }
    alloc_warp_plans_kernel<<<dim3((unsigned)((n + kWarpAllocWarps - 1) / kWarpAllocWarps), (unsigned)np),
                              32 * kWarpAllocWarps, warp_alloc_smem((int)G.nb), s>>>(P, (int)G.nb, n);
  }
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "alloc_cta launch");
}

int launch_alloc_small(Ctx* ctx, int n_blocks, int n, const uint32_t* weights, const FusedAlloc& fa, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    warp_alloc_attr((const void*)alloc_warp_kernel);
    attr = true;
  }
  const int kt = ktimer_begin(ctx, s, "alloc_small");
  alloc_warp_kernel<<<(unsigned)((n + kWarpAllocWarps - 1) / kWarpAllocWarps), 32 * kWarpAllocWarps,
                      warp_alloc_smem(n_blocks), s>>>(weights, n_blocks, n, fa.wmax, fa.budget, fa.cap, fa.base,
                                                      fa.counts, fa.offsets, fa.status);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "alloc_small launch");
}

// The per-image allocation of a DD plan (alloc_cta_kernel) from weights already computed.
int launch_alloc_cta(Ctx* ctx, int rows, int cols, int n, const uint32_t* weights, const FusedAlloc& fa,
                     cudaStream_t s) {
  const Grid16 G = make_grid16(rows, cols, n);
  if (G.total_units == 0) return ABCS_OK;
  const int kt = ktimer_begin(ctx, s, "alloc_cta");
  if (alloc_use_cta()) {
    alloc_cta_kernel<<<(unsigned)n, kCtaAllocThreads, 0, s>>>(weights, (int)G.nb, fa.wmax, fa.budget, fa.cap, fa.base,
                                                               fa.counts, fa.offsets, fa.status);
  } else {
    static bool attr = false;
    if (!attr) {
      warp_alloc_attr((const void*)alloc_warp_kernel);
      attr = true;
    }
    alloc_warp_kernel<<<(unsigned)((n + kWarpAllocWarps - 1) / kWarpAllocWarps), 32 * kWarpAllocWarps,
                        warp_alloc_smem((int)G.nb), s>>>(weights, (int)G.nb, n, fa.wmax, fa.budget, fa.cap, fa.base,
                                                         fa.counts, fa.offsets, fa.status);
  }
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "alloc_cta launch");
}

int launch_decode16(Ctx* ctx, int rows, int cols, int n, const uint16_t* counts, const int32_t* offsets,
                    const float* payload, int64_t payload_stride, float* out, int64_t out_stride, int out_pitch,
                    cudaStream_t s) {
  const Grid16 G = make_grid16(rows, cols, n);
  const uint32_t total = G.nb * (uint32_t)n;
  if (total == 0) return ABCS_OK;
  if (umma16_enabled())
    return launch_sense16_umma(ctx, 4, rows, cols, n, nullptr, 0, 0, counts, offsets, const_cast<float*>(payload),
                               payload_stride, out, out_stride, out_pitch, s);
  const int kt = ktimer_begin(ctx, s, "decode16");
  decode16_kernel<<<grid_for(ctx, G.total_runs), kM16Threads, 0, s>>>(G, total, counts, offsets, payload,
                                                                      payload_stride, out, out_stride, out_pitch);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "decode16 launch");
}

}  // namespace abcs_b200
