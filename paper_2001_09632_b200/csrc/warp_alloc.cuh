// Warp-level largest_remainder_allocate (sensing.cpp:110-177) for one image's small weight
// alphabet (DD phase-1 counts: weights in [0, wmax], wmax <= kCtaAllocMaxW), bit-exact with
// cta_allocate (cta_alloc.cuh) and the reference.
//
// One warp per image: the rounds synchronise with __syncwarp and shuffles instead of CTA
// barriers, so a batch of images runs as independent warps (many per SM) rather than as
// latency-bound 256-thread CTAs. Lane L owns the contiguous block range [L per, (L + 1) per), so
// "ties -> lower index" is one warp exclusive scan; per-block state is lane-strided in shared
// memory (block b0 + k of lane L at k * 32 + L: conflict-free). The class histogram is built once
// and updated as blocks reach their cap; each round computes one exact RN64 share per class
// (alloc_keys.h), the threshold class, then a per-class give table, so the per-block passes are
// a table lookup.
#pragma once
#include "cta_alloc.cuh"

namespace abcs_b200 {

struct WarpAllocTables {
  uint64_t key[kCtaAllocMaxW + 1];
  uint32_t hist[kCtaAllocMaxW + 1];
  uint32_t give[kCtaAllocMaxW + 1];  // whole (+1 above the threshold); bit 31: the exact-tie group
  uint8_t flag[kCtaAllocMaxW + 1];
  uint32_t bucket[256];  // the round's weighted histogram of the keys' top 8 bits
  uint8_t cand[32];      // classes in the threshold's bucket
};

// bytes of one warp's shared state for nb blocks (tables, u8 weights, u16 allocations)
__host__ __device__ __forceinline__ int warp_alloc_bytes(int nb) {
  const int per = (nb + 31) / 32;
  return ((int)sizeof(WarpAllocTables) + 32 * per * 3 + 15) & ~15;
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// weights: nb u32 (global); counts[nb] = base + alloc, offsets[nb] = exclusive scan.
// Returns an abcs_status, identical in every lane.
__device__ int warp_allocate(unsigned char* sm, const uint32_t* __restrict__ weights, int nb, int wmax,
                             long long budget, int cap, int base, uint16_t* __restrict__ counts,
                             int32_t* __restrict__ offsets) {
  const int lane = threadIdx.x & 31;
  const int per = (nb + 31) / 32;
  const int b0 = min(nb, lane * per), nmine = min(nb, b0 + per) - b0;
  WarpAllocTables& S = *reinterpret_cast<WarpAllocTables*>(sm);
  uint8_t* wv = sm + sizeof(WarpAllocTables);  // [k * 32 + lane]
  uint16_t* av = reinterpret_cast<uint16_t*>(wv + 32 * per + ((32 * per) & 1));
  for (int c = lane; c <= wmax; c += 32) S.hist[c] = 0;
  __syncwarp();
  bool bad = false;
  int tw = 0, na = 0;  // per-image totals < 2^31 (<= 4096 blocks x 127)
  {  // each lane loads its own contiguous range (16-byte loads where aligned)
    const uint32_t* wl = weights + b0;
    int k = 0;
    if (((uintptr_t)wl & 15) == 0)
      for (; k + 4 <= nmine; k += 4) {
        const uint4 q = __ldcg(reinterpret_cast<const uint4*>(wl + k));
        const uint32_t wq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          bad |= wq[e] > (uint32_t)wmax;
          wv[(k + e) * 32 + lane] = (uint8_t)min(wq[e], (uint32_t)wmax);
        }
      }
    for (; k < nmine; ++k) {
      const uint32_t wi = __ldcg(wl + k);
      bad |= wi > (uint32_t)wmax;
      wv[k * 32 + lane] = (uint8_t)min(wi, (uint32_t)wmax);
    }
  }
  if (__any_sync(0xffffffffu, bad) || budget > (long long)cap * nb || budget < 0) return ABCS_ERR_LOGIC;
  __syncwarp();
  for (int k = 0; k < per; ++k) {  // the initial histogram of active blocks (all, when cap > 0)
    const bool act = k < nmine && cap > 0;
    const int wi = act ? (int)wv[k * 32 + lane] : -1;
    if (k < nmine) av[k * 32 + lane] = 0;
    const unsigned peers = __match_any_sync(0xffffffffu, wi);
    if (act && (__ffs(peers) - 1) == lane) atomicAdd(&S.hist[wi], (unsigned)__popc(peers));
    if (act) {
      tw += wi;
      na += 1;
    }
  }
  tw = warp_sum_i(tw);
  na = warp_sum_i(na);
  long long remaining = budget;
  int round = 0;
  while (remaining > 0) {
    if (++round > nb + 1) return ABCS_ERR_LOGIC;
    __syncwarp();  // histogram updates of the previous round visible
    // total <= 0 -> uniform weights over the active blocks (sensing.cpp:137-141)
    const bool uniform = tw == 0;
    const uint64_t T = uniform ? (uint64_t)na : (uint64_t)tw;
    long long handed = 0;
    for (int c = lane; c <= wmax; c += 32) {
      const uint32_t h = S.hist[c];
      uint32_t whole = 0;
      if (h) {
        const ak_share sh = ak_compute((ak_u128)(uint64_t)remaining * (uniform ? 1u : (uint32_t)c), T);
        whole = (uint32_t)sh.whole;
        S.key[c] = sh.key;
        S.flag[c] = (uint8_t)sh.flag;
        handed += (long long)h * sh.whole;
      }
      S.give[c] = whole;
    }
    handed = warp_sum_ll(handed);
    __syncwarp();
    const int leftover = (int)(remaining - handed);  // < number of active blocks (each frac < 1)
    const bool sel_all = leftover > 0 && leftover >= na;
    const bool none = leftover <= 0;
    int need = leftover;
    bool all_taken = false, any_tie = false;
    if (sel_all) {
      for (int c = lane; c <= wmax; c += 32) S.give[c] += 1u;
    } else if (!none) {
      // the threshold class: blocks strictly above it < need <= above + tied (classes with hist 0
      // contribute 0: stale keys). Lane c ranks class c against every class.
      int thr_above = -1, thr_eq = 0;
      uint64_t thr_key = 0;
      int thr_flag = 0;
      // 1. the bucket (top 8 key bits) where the blocks ranking above first reach `need`: a
      //    weighted 256-bucket histogram scanned from the top, lane L owning buckets 255-8L..-7
      for (int b = lane; b < 256; b += 32) S.bucket[b] = 0;
      __syncwarp();
      for (int c = lane; c <= wmax; c += 32)
        if (S.hist[c]) atomicAdd(&S.bucket[(unsigned)(S.key[c] >> 56)], S.hist[c]);
      __syncwarp();
      int bk[8], loc = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        bk[i] = (int)S.bucket[255 - (8 * lane + i)];
        loc += bk[i];
      }
      int incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      int bstar = -1, above_b = 0;
      {
        int cum = incl - loc;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (bstar < 0 && cum < need && need <= cum + bk[i]) {
            bstar = 255 - (8 * lane + i);
            above_b = cum;
          }
          cum += bk[i];
        }
        const unsigned ball = __ballot_sync(0xffffffffu, bstar >= 0);
        const int src = ball ? __ffs(ball) - 1 : 0;
        bstar = __shfl_sync(0xffffffffu, bstar, src);
        above_b = __shfl_sync(0xffffffffu, above_b, src);
      }
      // 2. the classes in that bucket: compacted into the warp's candidate list (class order)
      int m = 0;
      for (int c0 = 0; c0 <= wmax; c0 += 32) {
        const int c = c0 + lane;
        const bool in = c <= wmax && S.hist[c] && (int)(S.key[c] >> 56) == bstar;
        const unsigned ball = __ballot_sync(0xffffffffu, in);
        if (in && m + __popc(ball & ((1u << lane) - 1)) < 32) S.cand[m + __popc(ball & ((1u << lane) - 1))] = (uint8_t)c;
        m += __popc(ball);
      }
      __syncwarp();
      if (bstar >= 0 && m <= 32) {
        // 3. lane j ranks candidate j among the candidates (blocks above it = higher buckets plus
        //    the candidates ranking above it)
        int above = above_b, eqc = 0;
        uint64_t kk = 0;
        int fk = 0;
        if (lane < m) {
          const int c = S.cand[lane];
          kk = S.key[c];
          fk = S.flag[c];
          for (int j = 0; j < m; ++j) {
            const int d = S.cand[j];
            const uint64_t kd = S.key[d];
            const int fd = S.flag[d];
            const int hd = (int)S.hist[d];
            above += (kd > kk || (kd == kk && fd > fk)) ? hd : 0;
            eqc += (kd == kk && fd == fk) ? hd : 0;
          }
        }
        const bool hit = lane < m && above < need && need <= above + eqc;  // tied classes agree
        const unsigned ball = __ballot_sync(0xffffffffu, hit);
        if (ball) {
          const int src = __ffs(ball) - 1;
          thr_above = __shfl_sync(0xffffffffu, above, src);
          thr_eq = __shfl_sync(0xffffffffu, eqc, src);
          thr_key = __shfl_sync(0xffffffffu, kk, src);
          thr_flag = __shfl_sync(0xffffffffu, fk, src);
        }
      } else {  // crowded bucket (tiny shares): every class ranks against every class
      for (int c0 = 0; c0 <= wmax; c0 += 32) {
        const int c = c0 + lane;
        const uint32_t h = c <= wmax ? S.hist[c] : 0u;
        int above = 0, eqc = 0;
        uint64_t kk = 0;
        int fk = 0;
        if (h) {
          kk = S.key[c];
          fk = S.flag[c];
#pragma unroll 4
          for (int d = 0; d <= wmax; ++d) {
            const int hd = (int)S.hist[d];
            const uint64_t kd = S.key[d];
            const int fd = S.flag[d];
            const bool gt = kd > kk || (kd == kk && fd > fk), eq = kd == kk && fd == fk;
            above += gt ? hd : 0;
            eqc += eq ? hd : 0;
          }
        }
        const bool hit = h && above < need && need <= above + eqc;  // tied classes agree
        const unsigned ball = __ballot_sync(0xffffffffu, hit);
        if (ball) {
          const int src = __ffs(ball) - 1;
          thr_above = __shfl_sync(0xffffffffu, above, src);
          thr_eq = __shfl_sync(0xffffffffu, eqc, src);
          thr_key = __shfl_sync(0xffffffffu, kk, src);
          thr_flag = __shfl_sync(0xffffffffu, fk, src);
        }
      }
      }
      if (thr_above < 0) return ABCS_ERR_LOGIC;
      need -= thr_above;
      all_taken = need == thr_eq;
      any_tie = !all_taken;
      for (int c = lane; c <= wmax; c += 32) {
        if (!S.hist[c]) continue;
        const uint64_t kk = S.key[c];
        const int fk = S.flag[c];
        const int rel = kk != thr_key ? (kk > thr_key ? 1 : 0) : (fk > thr_flag ? 1 : (fk == thr_flag ? 2 : 0));
        if (rel == 1 || (rel == 2 && all_taken)) S.give[c] += 1u;
        else if (rel == 2) S.give[c] |= 0x80000000u;
      }
    }
    __syncwarp();
    int tie_base = 0;
    if (any_tie) {  // the tied blocks in index order: lane order, then position within the lane
      int ties = 0;
      for (int k0 = 0; k0 < nmine; k0 += 8) {  // 8 blocks' loads in flight per batch
        int a[8], c[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const bool in = k0 + e < nmine;
          a[e] = in ? (int)av[(k0 + e) * 32 + lane] : cap;
          c[e] = in ? (int)wv[(k0 + e) * 32 + lane] : 0;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) ties += (a[e] < cap && (S.give[c[e]] >> 31)) ? 1 : 0;
      }
      int incl = ties;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      tie_base = incl - ties;
    }
    int taken_sum = 0, dtw = 0, dna = 0;
    for (int k0 = 0; k0 < nmine; k0 += 8) {  // 8 blocks per batch: loads first, then the updates
      int a[8], c[8];
      uint32_t g[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool in = k0 + e < nmine;
        a[e] = in ? (int)av[(k0 + e) * 32 + lane] : cap;
        c[e] = in ? (int)wv[(k0 + e) * 32 + lane] : 0;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) g[e] = S.give[c[e]];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (a[e] >= cap) continue;  // capped (or past the lane's range)
        int give = (int)(g[e] & 0x7fffffffu);
        if (g[e] >> 31) give += (tie_base++ < need) ? 1 : 0;
        const int room = cap - a[e];
        const int taken = give < room ? give : room;  // sensing.cpp:162-171
        av[(k0 + e) * 32 + lane] = (uint16_t)(a[e] + taken);
        taken_sum += taken;
        if (a[e] + taken >= cap) {  // capped: the block leaves the active pool
          atomicSub(&S.hist[c[e]], 1u);
          dtw += c[e];
          dna += 1;
        }
      }
    }
    taken_sum = warp_sum_i(taken_sum);
    tw -= warp_sum_i(dtw);
    na -= warp_sum_i(dna);
    remaining -= taken_sum;
    if (remaining > 0 && na == 0) return ABCS_ERR_LOGIC;  // capacity exhausted
  }
  // counts = base + allocation, offsets = exclusive scan (lane order, then position)
  int mine = 0;
  for (int k = 0; k < nmine; ++k) mine += base + (int)av[k * 32 + lane];
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  int ex = incl - mine;
  uint16_t* cnt = counts + b0;
  int32_t* off = offsets + b0;
  int k = 0;
  if (((uintptr_t)cnt & 15) == 0 && ((uintptr_t)off & 15) == 0)  // lane-contiguous 16-byte stores
    for (; k + 8 <= nmine; k += 8) {
      int c[8], o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        c[e] = base + (int)av[(k + e) * 32 + lane];
        o[e] = ex;
        ex += c[e];
      }
      *reinterpret_cast<uint4*>(cnt + k) =
          make_uint4((uint32_t)c[0] | (uint32_t)c[1] << 16, (uint32_t)c[2] | (uint32_t)c[3] << 16,
                     (uint32_t)c[4] | (uint32_t)c[5] << 16, (uint32_t)c[6] | (uint32_t)c[7] << 16);
      *reinterpret_cast<int4*>(off + k) = make_int4(o[0], o[1], o[2], o[3]);
      *reinterpret_cast<int4*>(off + k + 4) = make_int4(o[4], o[5], o[6], o[7]);
    }
  for (; k < nmine; ++k) {
    const int c = base + (int)av[k * 32 + lane];
    cnt[k] = (uint16_t)c;
    off[k] = ex;
    ex += c;
  }
  return ABCS_OK;
}

}  // namespace abcs_b200
