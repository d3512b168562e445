// CTA-level largest_remainder_allocate (sensing.cpp:110-177) for one image's small
// weight alphabet (DD phase-1 counts: weights in [0, wmax], wmax <= kCtaAllocMaxW).
//
// One 256-thread CTA per image. Thread t owns a contiguous slice of blocks, so block
// index order is (thread, position) order and the reference's "ties -> lower index"
// rule becomes a CTA exclusive scan. Bit-exact via alloc_keys.h: blocks with equal
// weights share one exact RN64 share/fraction key, so each round computes <= wmax+1
// keys (one thread per class), ranks the classes (2-4 threads per class), and hands
// the leftover units to the classes above the threshold key plus the first `need`
// tied blocks in index order. Cap rounds repeat while capped blocks release budget.
#pragma once
#include "alloc_keys.h"

namespace abcs_b200 {

constexpr int kCtaAllocThreads = 256;
constexpr int kCtaAllocWarps = kCtaAllocThreads / 32;
constexpr int kCtaAllocMaxW = 127;  // weight alphabet (phase1 <= 127)
constexpr int kCtaAllocMaxBlocks = 4096;

struct CtaAllocSmem {
  uint16_t w[kCtaAllocMaxBlocks];  // weights
  uint16_t a[kCtaAllocMaxBlocks];  // allocation so far
  uint32_t hist[kCtaAllocMaxW + 1];
  uint64_t key[kCtaAllocMaxW + 1];
  uint32_t whole[kCtaAllocMaxW + 1];
  uint8_t flag[kCtaAllocMaxW + 1];
  int red[kCtaAllocWarps][2];
  int scan[kCtaAllocWarps];
  long long thr_above, thr_eq;
  uint64_t thr_key;
  int thr_flag;
};


__device__ __forceinline__ int warp_excl_scan(int v, int& total) {
  const int lane = threadIdx.x & 31;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  total = __shfl_sync(0xffffffffu, incl, 31);
  return incl - v;
}

// CTA-wide sums of (x, y), returned to every thread. Starts and ends with a barrier.
// (Every per-image total here is < 2^31: <= 4096 blocks x 256 coefficients.)
__device__ __forceinline__ void cta_sum2(int& x, int& y, CtaAllocSmem& S) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    x += __shfl_xor_sync(0xffffffffu, x, o);
    y += __shfl_xor_sync(0xffffffffu, y, o);
  }
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    S.red[w][0] = x;
    S.red[w][1] = y;
  }
  __syncthreads();
  x = 0;
  y = 0;
#pragma unroll
  for (int i = 0; i < kCtaAllocWarps; ++i) {
    x += S.red[i][0];
    y += S.red[i][1];
  }
}

// CTA-wide exclusive scan in thread order.
__device__ __forceinline__ int cta_excl_scan(int v, int& total, CtaAllocSmem& S) {
  int wt;
  const int ex = warp_excl_scan(v, wt);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) S.scan[w] = wt;
  __syncthreads();
  int before = 0;
  total = 0;
#pragma unroll
  for (int i = 0; i < kCtaAllocWarps; ++i) {
    before += i < w ? S.scan[i] : 0;
    total += S.scan[i];
  }
  return before + ex;
}

// weights: nb u32 (global, written by an earlier kernel); writes counts[nb] = base + alloc
// and offsets[nb] (exclusive scan). Returns an abcs_status, identical in every thread.
__device__ int cta_allocate(CtaAllocSmem& S, const uint32_t* __restrict__ weights, int nb, int wmax, long long budget,
                            int cap, int base, uint16_t* __restrict__ counts, int32_t* __restrict__ offsets) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int per = (nb + kCtaAllocThreads - 1) / kCtaAllocThreads;
  const int b0 = min(nb, tid * per), b1 = min(nb, b0 + per);
  bool bad = false;
  for (int i = b0; i < b1; ++i) {
    const uint32_t wi = __ldcg(weights + i);
    bad |= wi > (uint32_t)wmax;
    S.w[i] = (uint16_t)min(wi, (uint32_t)wmax);
    S.a[i] = 0;
  }
  if (__syncthreads_or(bad) || budget > (long long)cap * nb || budget < 0) return ABCS_ERR_LOGIC;
  long long remaining = budget;
  int round = 0;
  while (remaining > 0) {
    if (++round > nb + 1) return ABCS_ERR_LOGIC;
    for (int c = tid; c <= wmax; c += kCtaAllocThreads) S.hist[c] = 0;
    __syncthreads();
    // active blocks: warp-aggregated class histogram (DD weights cluster on few values)
    int tw = 0, na = 0;
    for (int k = 0; k < per; ++k) {
      const int i = b0 + k;
      const bool act = i < b1 && (int)S.a[i] < cap;
      const int wi = act ? (int)S.w[i] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, wi);
      if (act && (__ffs(peers) - 1) == lane) atomicAdd(&S.hist[wi], (unsigned)__popc(peers));
      if (act) {
        tw += wi;
        na += 1;
      }
    }
    cta_sum2(tw, na, S);
    // total <= 0 -> uniform weights over the active blocks (sensing.cpp:137-141)
    const bool uniform = tw == 0;
    const uint64_t T = uniform ? (uint64_t)na : (uint64_t)tw;
    int handed = 0, unused = 0;
    for (int c = tid; c <= wmax; c += kCtaAllocThreads) {
      const uint32_t h = S.hist[c];
      if (!h) continue;
      const ak_share sh = ak_compute((ak_u128)(uint64_t)remaining * (uniform ? 1u : (uint32_t)c), T);
      S.whole[c] = (uint32_t)sh.whole;
      S.key[c] = sh.key;
      S.flag[c] = (uint8_t)sh.flag;
      handed += (int)h * (int)sh.whole;
    }
    cta_sum2(handed, unused, S);
    const long long leftover = remaining - (long long)handed;
    const bool sel_all = leftover > 0 && leftover >= na;
    const bool none = leftover <= 0;
    long long need = leftover;
    uint64_t thr_key = 0;
    int thr_flag = 0;
    bool all_taken = false;
    if (!sel_all && !none) {
      // threshold class: blocks strictly above it < need <= above + tied. `tpc` threads per class
      // walk the class table branch-free (classes with hist 0 contribute 0 whatever their stale key).
      const int tpc = wmax < 64 ? 4 : 2;
      const int sub = tid & (tpc - 1);
      for (int c0 = 0; c0 <= wmax; c0 += kCtaAllocThreads / tpc) {
        const int c = c0 + tid / tpc;
        const uint32_t h = c <= wmax ? S.hist[c] : 0u;
        int above = 0, eqc = 0;
        uint64_t kk = 0;
        int fk = 0;
        if (h) {
          kk = S.key[c];
          fk = S.flag[c];
#pragma unroll 4
          for (int d = sub; d <= wmax; d += tpc) {
            const int hd = (int)S.hist[d];
            const uint64_t kd = S.key[d];
            const int fd = S.flag[d];
            above += (kd > kk || (kd == kk && fd > fk)) ? hd : 0;
            eqc += (kd == kk && fd == fk) ? hd : 0;
          }
        }
        for (int o = 1; o < tpc; o <<= 1) {
          above += __shfl_xor_sync(0xffffffffu, above, o);
          eqc += __shfl_xor_sync(0xffffffffu, eqc, o);
        }
        if (h && sub == 0 && above < need && need <= (long long)above + eqc) {  // tied classes write the same
          S.thr_above = above;
          S.thr_eq = eqc;
          S.thr_key = kk;
          S.thr_flag = fk;
        }
      }
      __syncthreads();
      thr_key = S.thr_key;
      thr_flag = S.thr_flag;
      need -= S.thr_above;
      all_taken = need == S.thr_eq;
    }
    auto rel = [&](int c) -> int {  // 1: above the threshold, 2: tied with it
      if (sel_all) return 1;
      if (none) return 0;
      const uint64_t kk = S.key[c];
      if (kk != thr_key) return kk > thr_key ? 1 : 0;
      const int fk = S.flag[c];
      return fk > thr_flag ? 1 : (fk == thr_flag ? 2 : 0);
    };
    int tie_base = 0;
    if (!sel_all && !none && !all_taken) {
      int ties = 0;
      for (int i = b0; i < b1; ++i)
        if ((int)S.a[i] < cap && rel(S.w[i]) == 2) ++ties;
      int tot;
      tie_base = cta_excl_scan(ties, tot, S);
    }
    int taken_sum = 0, still = 0;
    for (int i = b0; i < b1; ++i) {
      if ((int)S.a[i] >= cap) continue;
      const int c = S.w[i];
      const int r = rel(c);
      bool sel = r == 1;
      if (r == 2) sel = all_taken || (long long)(tie_base++) < need;
      const long long give = (long long)S.whole[c] + (sel ? 1 : 0);
      const long long room = (long long)cap - S.a[i];
      const long long taken = give < room ? give : room;  // sensing.cpp:162-171
      S.a[i] = (uint16_t)(S.a[i] + taken);
      taken_sum += (int)taken;
      if ((int)S.a[i] < cap) ++still;
    }
    cta_sum2(taken_sum, still, S);
    remaining -= taken_sum;
    if (remaining > 0 && still == 0) return ABCS_ERR_LOGIC;  // capacity exhausted
  }
  int mine = 0;
  for (int i = b0; i < b1; ++i) mine += base + (int)S.a[i];
  int total;
  int ex = cta_excl_scan(mine, total, S);
  for (int i = b0; i < b1; ++i) {
    const int c = base + (int)S.a[i];
    counts[i] = (uint16_t)c;
    offsets[i] = ex;
    ex += c;
  }
  return ABCS_OK;
}

}  // namespace abcs_b200
