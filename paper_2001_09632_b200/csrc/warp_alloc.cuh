// Warp-level largest_remainder_allocate (sensing.cpp:110-177) for small weight
// alphabets (DD phase-1 counts: weights in [0, wmax], wmax <= kWarpAllocMaxW).
//
// Run by ONE warp -- the last warp to finish an image's phase-1 runs -- so the
// allocation needs neither a separate launch nor CTA barriers. Bit-exact with
// the reference via alloc_keys.h: blocks with equal weights share one exact
// RN64 share/fraction key, so each round computes <= wmax+1 keys, ranks the
// classes (O(classes^2), lanes stride over classes), and resolves exact ties by
// block index with a warp prefix scan (lanes own contiguous block ranges).
#pragma once
#include "alloc_keys.h"

namespace abcs_b200 {

constexpr int kWarpAllocMaxW = 127;     // weight alphabet (phase1 <= 127)
constexpr int kWarpAllocMaxBlocks = 4096;

struct WarpAllocSmem {
  uint16_t w[kWarpAllocMaxBlocks];   // weights
  uint16_t a[kWarpAllocMaxBlocks];   // allocation so far
  uint32_t hist[kWarpAllocMaxW + 1];
  uint64_t key[kWarpAllocMaxW + 1];
  uint32_t whole[kWarpAllocMaxW + 1];
  uint8_t flag[kWarpAllocMaxW + 1];
};

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

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

// weights: nb u32 (global, produced by this kernel); writes counts[nb] = base + alloc and
// offsets[nb] (exclusive scan). Returns an abcs_status (same for every lane).
__device__ __forceinline__ int warp_allocate(WarpAllocSmem& S, const uint32_t* weights, int nb, int wmax, long long budget, int cap,
                             int base, uint16_t* counts, int32_t* offsets) {
  const int lane = threadIdx.x & 31;
  const int per = (nb + 31) / 32;
  const int b0 = min(nb, lane * per), b1 = min(nb, b0 + per);
  bool bad = false;
  for (int i = b0; i < b1; ++i) {
    const uint32_t wi = __ldcg(weights + i);  // written by other warps: bypass L1
    bad |= wi > (uint32_t)wmax;
    S.w[i] = (uint16_t)min(wi, (uint32_t)wmax);
    S.a[i] = 0;
  }
  if (__any_sync(0xffffffffu, bad) || budget > (long long)cap * nb || budget < 0) return ABCS_ERR_LOGIC;
  long long remaining = budget;
  int round = 0;
  while (remaining > 0) {
    if (++round > nb + 1) return ABCS_ERR_LOGIC;
    for (int c = lane; c <= wmax; c += 32) S.hist[c] = 0;
    __syncwarp();
    long long tw = 0, na = 0;
    for (int k = 0; k < per; ++k) {  // warp-aggregated histogram (DD weights cluster on few values)
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
    tw = warp_sum_ll(tw);
    na = warp_sum_ll(na);
    __syncwarp();
    const bool uniform = tw == 0;
    const uint64_t T = uniform ? (uint64_t)na : (uint64_t)tw;
    long long handed = 0;
    for (int c = lane; c <= wmax; c += 32) {
      const uint32_t h = S.hist[c];
      if (!h) continue;
      const ak_share sh = ak_compute((ak_u128)(uint64_t)remaining * (uniform ? 1u : (uint32_t)c), T);
      S.whole[c] = (uint32_t)sh.whole;
      S.key[c] = sh.key;
      S.flag[c] = (uint8_t)sh.flag;
      handed += (long long)h * (long long)sh.whole;
    }
    handed = warp_sum_ll(handed);
    __syncwarp();
    const long long leftover = remaining - handed;
    const bool sel_all = leftover > 0 && leftover >= na;
    const bool none = leftover <= 0;
    long long need = leftover;
    uint64_t thr_key = 0;
    int thr_flag = 0;
    bool all_taken = false;
    if (!sel_all && !none) {
      // class ranks: blocks strictly above, blocks tied (equal key and flag)
      long long my_above = -1, my_eq = 0;
      uint64_t my_key = 0;
      int my_flag = 0;
      for (int c = lane; c <= wmax; c += 32) {
        if (!S.hist[c]) continue;
        const uint64_t kk = S.key[c];
        const int fk = S.flag[c];
        long long above = 0, eqc = 0;
        for (int d = 0; d <= wmax; ++d) {
          const uint32_t hd = S.hist[d];
          if (!hd) continue;
          const uint64_t kd = S.key[d];
          const int fd = S.flag[d];
          if (kd > kk || (kd == kk && fd > fk)) above += hd;
          else if (kd == kk && fd == fk) eqc += hd;
        }
        if (above < need && need <= above + eqc) {
          my_above = above;
          my_eq = eqc;
          my_key = kk;
          my_flag = fk;
        }
      }
      const unsigned who = __ballot_sync(0xffffffffu, my_above >= 0);
      const int src = __ffs(who) - 1;
      const long long above = __shfl_sync(0xffffffffu, my_above, src);
      const long long eqc = __shfl_sync(0xffffffffu, my_eq, src);
      thr_key = __shfl_sync(0xffffffffu, my_key, src);
      thr_flag = __shfl_sync(0xffffffffu, my_flag, src);
      need -= above;
      all_taken = need == eqc;
    }
    auto rel = [&](int c) -> int {  // 1 above the threshold, 2 tied with it
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
      tie_base = warp_excl_scan(ties, tot);
    }
    long long taken_sum = 0, still = 0;
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
      taken_sum += taken;
      if ((int)S.a[i] < cap) ++still;
    }
    taken_sum = warp_sum_ll(taken_sum);
    still = warp_sum_ll(still);
    __syncwarp();
    remaining -= taken_sum;
    if (remaining > 0 && still == 0) return ABCS_ERR_LOGIC;  // capacity exhausted
  }
  int mine = 0;
  for (int i = b0; i < b1; ++i) mine += base + (int)S.a[i];
  int total;
  int ex = warp_excl_scan(mine, total);
  for (int i = b0; i < b1; ++i) {
    const int c = base + (int)S.a[i];
    counts[i] = (uint16_t)c;
    offsets[i] = ex;
    ex += c;
  }
  return ABCS_OK;
}

}  // namespace abcs_b200
