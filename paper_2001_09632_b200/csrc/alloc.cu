// largest_remainder_allocate (/root/reference/proj/core/src/sensing.cpp:110-177)
// on the device: one CTA per weight vector (image), bit-exact with the
// reference's x87 ranking via alloc_keys.h.
//
// Per round (sensing.cpp:133-175):
//   T = sum of active weights (uniform weights when T == 0),
//   share_i = RN64(remaining * w_i / T) -> whole_i + exact 65-bit frac key,
//   leftover = remaining - sum(whole) units go to the largest fracs (ties ->
//   lower index) via an MSB-first radix select over the keys plus an ordered
//   block scan for exact ties, then clamp to caps; capped blocks leave.
// Finally counts = base + alloc and offsets = exclusive scan of counts.
#include <cub/block/block_reduce.cuh>
#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>
#include <cstdlib>
#include <type_traits>

#include "alloc_keys.h"
#include "common.cuh"
#include "internal.h"

namespace abcs_b200 {
namespace cg = cooperative_groups;

constexpr int kAllocThreads = 1024;

struct AllocScratch {
  uint64_t* key;
  uint32_t* give;
  uint32_t* alloc;
  uint8_t* flag;
};

size_t allocate_scratch_bytes(int32_t n_blocks, int32_t n_vectors) {
  // radix kernel: 17 B per block; class kernel: 2 u16 per block, each cluster CTA's range padded
  // to 1024-thread spans (up to 16 CTAs per image)
  const size_t per = std::max((size_t)n_blocks * (8 + 4 + 4 + 1), ((size_t)n_blocks + 16 * 1024) * 4);
  return per * (size_t)n_vectors + 256;
}

__device__ __forceinline__ int cap_of(const int32_t* caps, int cap_u, int i) { return caps ? caps[i] : cap_u; }

__global__ void __launch_bounds__(kAllocThreads)
alloc_kernel(const uint32_t* __restrict__ weights, int nb, int64_t budget, const int32_t* __restrict__ caps_all,
             int cap_u, int base, uint16_t* __restrict__ counts, int32_t* __restrict__ offsets,
             int32_t* __restrict__ status, AllocScratch scr) {
  using Reduce64 = cub::BlockReduce<unsigned long long, kAllocThreads>;
  using ScanI = cub::BlockScan<int, kAllocThreads>;
  __shared__ union {
    typename Reduce64::TempStorage r;
    typename ScanI::TempStorage s;
  } tmp;
  __shared__ unsigned int hist[256];
  __shared__ long long sh_ll[4];
  __shared__ int sh_int[4];

  const int v = blockIdx.x, tid = threadIdx.x;
  const uint32_t* w = weights + (int64_t)v * nb;
  const int32_t* caps = caps_all ? caps_all + (int64_t)v * nb : nullptr;
  uint64_t* key = scr.key + (int64_t)v * nb;
  uint32_t* give = scr.give + (int64_t)v * nb;
  uint32_t* alloc = scr.alloc + (int64_t)v * nb;
  uint8_t* flag = scr.flag + (int64_t)v * nb;

  // preconditions (sensing.cpp:114-124)
  {
    unsigned long long cap_sum = 0, neg = 0;
    for (int i = tid; i < nb; i += kAllocThreads) {
      const int c = cap_of(caps, cap_u, i);
      if (c < 0) neg = 1;
      else cap_sum += (unsigned long long)c;
      alloc[i] = 0;
    }
    const unsigned long long tot = Reduce64(tmp.r).Sum(cap_sum);
    __syncthreads();
    const unsigned long long nneg = Reduce64(tmp.r).Sum(neg);
    if (tid == 0) {
      int st = ABCS_OK;
      if (budget < 0 || nneg) st = ABCS_ERR_INVALID_ARGUMENT;
      else if ((unsigned long long)budget > tot) st = ABCS_ERR_INVALID_ARGUMENT;
      sh_int[0] = st;
    }
    __syncthreads();
    if (sh_int[0] != ABCS_OK) {
      if (tid == 0 && status) status[v] = sh_int[0];
      return;
    }
  }

  long long remaining = budget;
  int st = ABCS_OK;
  int round = 0;
  while (remaining > 0) {
    // every round places all units or caps >= 1 block, so nb + 1 rounds always suffice
    if (++round > nb + 1) {
      st = ABCS_ERR_LOGIC;
      break;
    }
    // ---- total weight and active count (sensing.cpp:134-137)
    unsigned long long tw = 0, na = 0;
    for (int i = tid; i < nb; i += kAllocThreads) {
      if ((int)alloc[i] < cap_of(caps, cap_u, i)) {
        tw += w[i];
        na += 1;
      }
    }
    const unsigned long long T0 = Reduce64(tmp.r).Sum(tw);
    __syncthreads();
    const unsigned long long n_active = Reduce64(tmp.r).Sum(na);
    if (tid == 0) {
      sh_ll[0] = (long long)T0;
      sh_ll[1] = (long long)n_active;
    }
    __syncthreads();
    const bool uniform = sh_ll[0] == 0;
    const uint64_t T = uniform ? (uint64_t)sh_ll[1] : (uint64_t)sh_ll[0];
    const long long n_act = sh_ll[1];

    // ---- shares (sensing.cpp:142-149)
    unsigned long long handed = 0;
    for (int i = tid; i < nb; i += kAllocThreads) {
      if ((int)alloc[i] < cap_of(caps, cap_u, i)) {
        const ak_u128 P = (ak_u128)(uint64_t)remaining * (uniform ? 1u : w[i]);
        const ak_share s = ak_compute(P, T);
        give[i] = (uint32_t)s.whole;
        key[i] = s.key;
        flag[i] = (uint8_t)s.flag;
        handed += s.whole;
      }
    }
    const unsigned long long h = Reduce64(tmp.r).Sum(handed);
    if (tid == 0) sh_ll[2] = (long long)h;
    __syncthreads();
    const long long leftover = remaining - sh_ll[2];

    // ---- hand out leftovers by largest fraction, ties -> lower index (:150-158)
    if (leftover > 0 && leftover >= n_act) {
      for (int i = tid; i < nb; i += kAllocThreads)
        if ((int)alloc[i] < cap_of(caps, cap_u, i)) give[i] += 1;
    } else if (leftover > 0) {
      long long need = leftover;
      unsigned long long prefix = 0;
      int passes = 0;         // digit passes resolved (8 bits each over key, then the flag)
      int flag_sel = -1;      // selected flag value if the flag pass ran
      bool all_equal_taken = false;
      for (int pass = 0; pass < 9; ++pass) {
        const int nbins = pass < 8 ? 256 : 2;
        for (int b = tid; b < 256; b += kAllocThreads) hist[b] = 0;
        __syncthreads();
        const int shift_hi = 64 - 8 * pass;  // bits already fixed: key >> shift_hi == prefix
        for (int i = tid; i < nb; i += kAllocThreads) {
          if ((int)alloc[i] >= cap_of(caps, cap_u, i)) continue;
          const uint64_t k = key[i];
          const bool match = (pass == 0) ? true : (pass < 8 ? ((k >> shift_hi) == prefix) : (k == prefix));
          if (!match) continue;
          const unsigned d = pass < 8 ? (unsigned)((k >> (56 - 8 * pass)) & 0xffu) : (unsigned)flag[i];
          atomicAdd(&hist[d], 1u);
        }
        __syncthreads();
        if (tid < 32) {
          // descending digit order: lane l owns digits [nbins-1-8l .. nbins-8-8l]
          const int lane = tid;
          const int per = (nbins + 31) / 32;
          unsigned local = 0;
          for (int q = 0; q < per; ++q) {
            const int d = nbins - 1 - (lane * per + q);
            if (d >= 0) local += hist[d];
          }
          unsigned incl = local;
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
          }
          const unsigned excl = incl - local;
          const bool hit = (excl < (unsigned long long)need) && ((unsigned long long)incl >= (unsigned long long)need);
          const unsigned ball = __ballot_sync(0xffffffffu, hit);
          const int src = __ffs(ball) - 1;
          if (lane == src) {
            unsigned cum = excl;
            for (int q = 0; q < per; ++q) {
              const int d = nbins - 1 - (lane * per + q);
              if (d < 0) break;
              if ((unsigned long long)cum + hist[d] >= (unsigned long long)need) {
                sh_int[1] = d;
                sh_int[2] = (int)hist[d];
                sh_ll[3] = (long long)cum;
                break;
              }
              cum += hist[d];
            }
          }
        }
        __syncthreads();
        const int g = sh_int[1];
        const long long above = sh_ll[3];
        const int eq = sh_int[2];
        need -= above;
        if (pass < 8) prefix = (prefix << 8) | (unsigned long long)g;
        else flag_sel = g;
        passes = pass + 1;
        __syncthreads();
        if (eq == need) {
          all_equal_taken = true;
          break;
        }
      }
      // mark selections; exact ties (all 65 bits equal) resolved by ascending index
      int base_rank = 0;
      for (int start = 0; start < nb; start += kAllocThreads) {
        const int i = start + tid;
        int gt = 0, eqv = 0;
        if (i < nb && (int)alloc[i] < cap_of(caps, cap_u, i)) {
          const uint64_t k = key[i];
          if (passes <= 8) {
            const int sh = 64 - 8 * passes;
            const unsigned long long top = sh >= 64 ? 0ull : (k >> sh);
            if (top > prefix) gt = 1;
            else if (top == prefix) eqv = 1;
          } else {
            if (k > prefix) gt = 1;
            else if (k == prefix) {
              if ((int)flag[i] > flag_sel) gt = 1;
              else if ((int)flag[i] == flag_sel) eqv = 1;
            }
          }
        }
        int rank, total;
        ScanI(tmp.s).ExclusiveSum(eqv, rank, total);
        __syncthreads();
        if (i < nb && (gt || (eqv && (all_equal_taken || (long long)(base_rank + rank) < need)))) give[i] += 1;
        base_rank += total;
      }
    }
    __syncthreads();

    // ---- clamp to caps, capped blocks leave the pool (sensing.cpp:162-174)
    unsigned long long taken_sum = 0, still = 0;
    for (int i = tid; i < nb; i += kAllocThreads) {
      const int c = cap_of(caps, cap_u, i);
      if ((int)alloc[i] < c) {
        const long long room = (long long)c - alloc[i];
        const long long taken = (long long)give[i] < room ? (long long)give[i] : room;
        alloc[i] += (uint32_t)taken;
        taken_sum += (unsigned long long)taken;
        if ((int)alloc[i] < c) still += 1;
      }
    }
    const unsigned long long tk = Reduce64(tmp.r).Sum(taken_sum);
    __syncthreads();
    const unsigned long long st_open = Reduce64(tmp.r).Sum(still);
    if (tid == 0) {
      sh_ll[0] = (long long)tk;
      sh_ll[1] = (long long)st_open;
    }
    __syncthreads();
    remaining -= sh_ll[0];
    if (remaining > 0 && sh_ll[1] == 0) {
      st = ABCS_ERR_LOGIC;  // "allocate: capacity exhausted before budget placed"
      break;
    }
    __syncthreads();
  }

  // ---- counts and offsets
  int running = 0;
  for (int start = 0; start < nb; start += kAllocThreads) {
    const int i = start + tid;
    const int c = i < nb ? base + (int)alloc[i] : 0;
    int ex, total;
    ScanI(tmp.s).ExclusiveSum(c, ex, total);
    __syncthreads();
    if (i < nb) {
      counts[(int64_t)v * nb + i] = (uint16_t)c;
      if (offsets) offsets[(int64_t)v * nb + i] = running + ex;
    }
    running += total;
  }
  if (tid == 0 && status) status[v] = st;
}

// ---------------------------------------------------------------------------
// Weight-class allocator (the production path for sense). Blocks with equal
// weights get equal shares and equal fraction keys, so each round needs one
// exact RN64 key per DISTINCT weight (DD: <= phase1 + 1 classes; BBV: the
// distinct boundary variations) instead of one per block. Per round:
// histogram of active weights -> compacted class table (count, whole, key) ->
// threshold of the leftover units over the classes weighted by their counts
// (rank mode for few classes, else an MSB radix select) -> exact ties resolved
// by block index (ordered scan) -> clamp. Results are identical to alloc_kernel
// / the reference.
//
// A weight vector (image) is owned by a thread-block CLUSTER of cs CTAs
// (cs = 1 .. 16, chosen by the launcher so small batches of large images still
// fill the GPU). CTA r of the cluster owns the contiguous block range
// [nb r / cs, nb (r + 1) / cs); within a CTA each thread owns a contiguous
// sub-range, so "ties to the lower index" is one ordered scan: thread order
// inside the CTA, rank order across the cluster. The round's cross-CTA terms go
// through distributed shared memory: the active-weight histogram and (T,
// active) after barrier A, the tie counts of lower ranks after barrier C, and
// (taken, still open) after barrier D; the class table and the threshold are
// recomputed identically in every CTA from the cluster-wide histogram.
// ---- one round's class table and leftover threshold (shared by the cluster and the
// distributed allocators; every thread of the CTA calls it and gets the same result) ------
constexpr int kClassThreads = 1024;
using Reduce64C = cub::BlockReduce<unsigned long long, kClassThreads>;
using ScanIC = cub::BlockScan<int, kClassThreads>;
constexpr int kBucketBits = 11;  // threshold search: classes bucketed by their key's top 11 bits
constexpr int kBuckets = 1 << kBucketBits;
constexpr int kMaxCand = 256;    // classes sharing the threshold's bucket ranked pairwise
struct ClassShared {
  union {
    typename Reduce64C::TempStorage r;
    typename ScanIC::TempStorage s;
  } tmp;
  unsigned int hist8[256];
  long long sh_ll[4];
  int sh_int[4];
  unsigned int bucket[kBuckets];  // weighted (blocks per class) histogram of the key's top bits
  int cand[kMaxCand];
  int ncand;
};
struct ClassSel {  // the round's selection: units by class rank, exact ties by block index
  long long need;  // tie-group units still to hand out (to the lowest indices)
  unsigned long long prefix;
  uint64_t thr_key;
  int ncls, passes, flag_sel, thr_flag;
  int sel_all, none, rank_mode, all_equal_taken;
};

// gh[c] (c in this thread's weight range [c0, c1)) = active blocks of weight c in the whole
// vector; on return gh[c] = the class index of weight c, and ccnt/cwhole/ckey/cflag hold the
// class table (ordered by weight).
__device__ ClassSel class_round_select(ClassShared& sm, uint32_t* gh, int c0, int c1, long long remaining,
                                       uint64_t T, bool uniform, long long n_act, uint32_t* ccnt, uint32_t* cwhole,
                                       uint64_t* ckey, uint8_t* cflag) {
  using Reduce64 = Reduce64C;
  using ScanI = ScanIC;
  const int tid = threadIdx.x, lane = tid & 31;
  // compact the nonempty classes (ordered by weight) and compute their shares
  int mine = 0;
  for (int c = c0; c < c1; ++c) mine += gh[c] ? 1 : 0;
  int id, ncls;
  ScanI(sm.tmp.s).ExclusiveSum(mine, id, ncls);
  unsigned long long handed = 0;
  for (int c = c0; c < c1; ++c) {
    const uint32_t h = gh[c];
    if (!h) continue;
    const int k = id++;
    ccnt[k] = h;
    const ak_u128 P = (ak_u128)(uint64_t)remaining * (uniform ? 1u : (uint32_t)c);
    const ak_share sh = ak_compute(P, T);  // sensing.cpp:144-148
    cwhole[k] = (uint32_t)sh.whole;
    ckey[k] = sh.key;
    cflag[k] = (uint8_t)sh.flag;
    gh[c] = (uint32_t)k;
    handed += (unsigned long long)h * sh.whole;
  }
  __syncthreads();
  const unsigned long long hsum = Reduce64(sm.tmp.r).Sum(handed);
  if (tid == 0) sm.sh_ll[2] = (long long)hsum;
  __syncthreads();
  const long long leftover = remaining - sm.sh_ll[2];
  // leftover units -> largest fractions, ties to the lower index (sensing.cpp:150-158)
  const bool sel_all = leftover > 0 && leftover >= n_act;
  const bool none = leftover <= 0;
  unsigned long long prefix = 0;
  int passes = 0, flag_sel = -1;
  bool all_equal_taken = false;
  long long need = leftover;
  bool rank_mode = false;
  uint64_t thr_key = 0;
  int thr_flag = 0;
  bool bucketed = false;
  if (!sel_all && !none && ncls > 64) {  // (a few dozen classes: the pairwise ranking below is cheaper)
    // threshold by bucket: a weighted histogram of the keys' top kBucketBits bits, a descending
    // scan for the bucket where the count of blocks ranking above first reaches `need`, then the
    // classes inside that bucket (usually one or two) ranked pairwise by (key, flag)
    for (int b = tid; b < kBuckets; b += kClassThreads) sm.bucket[b] = 0;
    if (tid == 0) sm.ncand = 0;
    __syncthreads();
    for (int k = tid; k < ncls; k += kClassThreads)
      atomicAdd(&sm.bucket[(unsigned)(ckey[k] >> (64 - kBucketBits))], ccnt[k]);
    __syncthreads();
    constexpr int kPer = kBuckets / kClassThreads;  // buckets per thread, descending
    unsigned int loc = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) loc += sm.bucket[kBuckets - 1 - (tid * kPer + i)];
    unsigned int before, total_b;
    {
      int ex, tot;
      ScanI(sm.tmp.s).ExclusiveSum((int)loc, ex, tot);
      before = (unsigned)ex;
      total_b = (unsigned)tot;
    }
    (void)total_b;
    if ((long long)before < need && need <= (long long)before + loc) {
      unsigned int cum = before;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int b = kBuckets - 1 - (tid * kPer + i);
        const unsigned int h = sm.bucket[b];
        if ((long long)cum < need && need <= (long long)cum + h) {
          sm.sh_int[0] = b;
          sm.sh_ll[0] = (long long)cum;  // blocks in higher buckets
        }
        cum += h;
      }
    }
    __syncthreads();
    const int bstar = sm.sh_int[0];
    const long long above_b = sm.sh_ll[0];
    for (int k = tid; k < ncls; k += kClassThreads)
      if ((int)(ckey[k] >> (64 - kBucketBits)) == bstar) {
        const int slot = atomicAdd(&sm.ncand, 1);
        if (slot < kMaxCand) sm.cand[slot] = k;
      }
    __syncthreads();
    const int m = sm.ncand;
    if (m <= kMaxCand) {
      bucketed = true;
      rank_mode = true;
      if (tid < m) {
        const int c = sm.cand[tid];
        const uint64_t kk = ckey[c];
        const int fk = cflag[c];
        long long above = above_b, eqc = 0;
        for (int j = 0; j < m; ++j) {
          const int d = sm.cand[j];
          const uint64_t kd = ckey[d];
          const int fd = cflag[d];
          const long long cd = ccnt[d];
          above += (kd > kk || (kd == kk && fd > fk)) ? cd : 0;
          eqc += (kd == kk && fd == fk) ? cd : 0;
        }
        if (above < need && need <= above + eqc) {  // the threshold tie group (tied classes agree)
          sm.sh_ll[3] = above;
          sm.sh_int[2] = (int)eqc;
          sm.sh_int[1] = fk;
          sm.sh_ll[2] = (long long)kk;
        }
      }
      __syncthreads();
      need -= sm.sh_ll[3];
      all_equal_taken = need == (long long)sm.sh_int[2];
      thr_key = (uint64_t)sm.sh_ll[2];
      thr_flag = sm.sh_int[1];
      __syncthreads();
    }
  }
  if (bucketed) {
  } else if (!sel_all && !none && ncls <= 512) {
    // few classes: each class counts the blocks ranking strictly above it and tied with it
    // (a power-of-two group of tpc threads per class splits the scan; shuffle-reduced)
    rank_mode = true;
    int tpc = 1;
    while (tpc < 32 && 2 * tpc * ncls <= kClassThreads) tpc *= 2;
    const int cls = tid / tpc, sub = tid & (tpc - 1);
    int above = 0, eqc = 0;
    uint64_t kk = 0;
    int fk = 0;
    if (cls < ncls) {
      kk = ckey[cls];
      fk = cflag[cls];
#pragma unroll 4
      for (int j = sub; j < ncls; j += tpc) {
        const uint64_t kj = ckey[j];
        const int fj = cflag[j];
        const int cj = (int)ccnt[j];
        above += (kj > kk || (kj == kk && fj > fk)) ? cj : 0;
        eqc += (kj == kk && fj == fk) ? cj : 0;
      }
    }
    for (int o = 1; o < tpc; o <<= 1) {
      above += __shfl_xor_sync(0xffffffffu, above, o);
      eqc += __shfl_xor_sync(0xffffffffu, eqc, o);
    }
    if (cls < ncls && sub == 0 && above < need && need <= (long long)above + eqc) {  // the threshold tie group
      sm.sh_ll[3] = above;
      sm.sh_int[2] = eqc;
      sm.sh_int[1] = fk;
      sm.sh_ll[2] = (long long)kk;
    }
    __syncthreads();
    need -= sm.sh_ll[3];
    all_equal_taken = need == (long long)sm.sh_int[2];
    thr_key = (uint64_t)sm.sh_ll[2];
    thr_flag = sm.sh_int[1];
    __syncthreads();
  } else if (!sel_all && !none) {
    for (int pass = 0; pass < 9; ++pass) {
      const int nbins = pass < 8 ? 256 : 2;
      if (tid < 256) sm.hist8[tid] = 0;
      __syncthreads();
      const int shift_hi = 64 - 8 * pass;
      for (int k = tid; k < ncls; k += kClassThreads) {
        const uint64_t kk = ckey[k];
        const bool match = (pass == 0) ? true : (pass < 8 ? ((kk >> shift_hi) == prefix) : (kk == prefix));
        if (!match) continue;
        const unsigned d = pass < 8 ? (unsigned)((kk >> (56 - 8 * pass)) & 0xffu) : (unsigned)cflag[k];
        atomicAdd(&sm.hist8[d], ccnt[k]);
      }
      __syncthreads();
      if (tid < 32) {
        const int per = (nbins + 31) / 32;
        unsigned local = 0;
        for (int q = 0; q < per; ++q) {
          const int d = nbins - 1 - (lane * per + q);
          if (d >= 0) local += sm.hist8[d];
        }
        unsigned incl = local;
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const unsigned excl = incl - local;
        const bool hit = ((long long)excl < need) && ((long long)incl >= need);
        const unsigned ball = __ballot_sync(0xffffffffu, hit);
        const int src = __ffs(ball) - 1;
        if (lane == src) {
          unsigned cum = excl;
          for (int q = 0; q < per; ++q) {
            const int d = nbins - 1 - (lane * per + q);
            if (d < 0) break;
            if ((long long)cum + sm.hist8[d] >= need) {
              sm.sh_int[1] = d;
              sm.sh_int[2] = (int)sm.hist8[d];
              sm.sh_ll[3] = (long long)cum;
              break;
            }
            cum += sm.hist8[d];
          }
        }
      }
      __syncthreads();
      const int g = sm.sh_int[1];
      const int eq = sm.sh_int[2];
      need -= sm.sh_ll[3];
      if (pass < 8) prefix = (prefix << 8) | (unsigned long long)g;
      else flag_sel = g;
      passes = pass + 1;
      __syncthreads();
      if (eq == need) {
        all_equal_taken = true;
        break;
      }
    }
  }
  ClassSel S;
  S.need = need;
  S.prefix = prefix;
  S.thr_key = thr_key;
  S.ncls = ncls;
  S.passes = passes;
  S.flag_sel = flag_sel;
  S.thr_flag = thr_flag;
  S.sel_all = sel_all;
  S.none = none;
  S.rank_mode = rank_mode;
  S.all_equal_taken = all_equal_taken;
  return S;
}

// Class k's relation to the threshold: 1 = above it, 2 = in the exact-tie group, 0 = below.
__device__ __forceinline__ int class_rel(const ClassSel& S, int k, const uint64_t* ckey, const uint8_t* cflag) {
  if (S.sel_all) return 1;
  if (S.none) return 0;
  const uint64_t kk = ckey[k];
  if (S.rank_mode) {
    if (kk != S.thr_key) return kk > S.thr_key ? 1 : 0;
    return (int)cflag[k] > S.thr_flag ? 1 : ((int)cflag[k] == S.thr_flag ? 2 : 0);
  }
  if (S.passes <= 8) {
    const int sh = 64 - 8 * S.passes;
    const unsigned long long top = sh >= 64 ? 0ull : (kk >> sh);
    return top > S.prefix ? 1 : (top == S.prefix ? 2 : 0);
  }
  if (kk != S.prefix) return kk > S.prefix ? 1 : 0;
  return (int)cflag[k] > S.flag_sel ? 1 : ((int)cflag[k] == S.flag_sel ? 2 : 0);
}

constexpr int kMaxCluster = 16;
static_assert(kClassThreads <= 1024, "allocate_scratch_bytes pads spans by 1024");

template <typename T>
struct Arr {
  T* p;
  __device__ __forceinline__ T& operator[](int i) const { return p[i]; }
};

// entries per per-block array of a CTA owning nbl blocks (thread-strided layout)
__host__ __device__ __forceinline__ int class_span(int nbl) {
  return (nbl + kClassThreads - 1) / kClassThreads * kClassThreads;
}
__host__ __device__ __forceinline__ int cluster_lo(int nb, int cs, int r) { return (int)((int64_t)nb * r / cs); }

size_t class_smem_bytes(int wmax, int n_blocks, int cs, bool arrays_in_smem) {
  const size_t ncls = (size_t)std::min(n_blocks, wmax + 1);
  size_t b = 8 * (size_t)(wmax + 1) + ncls * (8 + 4 + 4 + 1) + 64;
  if (arrays_in_smem) b += (size_t)class_span((n_blocks + cs - 1) / cs) * 4 + 16;
  return b;
}

// kSmemArrays: weights and allocations in shared memory; else weights in global scratch and
// allocations in shared memory as u8 (kAv8, caps <= 255) or in global scratch as u16.
// Weight ranges at least this wide take plain shared-memory atomics for the per-round histogram
// (collisions are rare); narrower ones (DD: phase-1 counts, <= 256 classes) aggregate equal
// weights in the warp first (__match_any_sync).
constexpr int kAggregateBelow = 256;

template <bool kSmemArrays, bool kAv8 = false>
__global__ void __launch_bounds__(kClassThreads)
alloc_class_kernel(const uint32_t* __restrict__ weights, int nb, int wmax, int64_t budget, int cap, int base,
                   uint16_t* __restrict__ counts, int32_t* __restrict__ offsets, int32_t* __restrict__ status,
                   uint32_t* __restrict__ gscratch) {
  using Reduce64 = Reduce64C;
  using ScanI = ScanIC;
  __shared__ ClassShared sm;
  auto& tmp = sm.tmp;
  auto& sh_int = sm.sh_int;
  __shared__ long long pub[6];  // published to the cluster: 0/1 (T, active) | 2 ties | 3/4 (taken, open) | 5 misc
  __shared__ long long agg[2];  // cluster aggregates read back by warp 0
  extern __shared__ __align__(16) unsigned char dyn[];
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks(), rk = (int)cluster.block_rank();
  const int ncls_cap = min(nb, wmax + 1);
  unsigned char* p = dyn;
  uint64_t* ckey = reinterpret_cast<uint64_t*>(p);
  p += 8 * (size_t)ncls_cap;
  uint32_t* hist = reinterpret_cast<uint32_t*>(p);  // this CTA's active-weight histogram (read cluster-wide)
  p += 4 * (size_t)(wmax + 1);
  // the cluster's histogram, then weight -> class index (a cluster of one uses hist in place)
  uint32_t* ghist = cs == 1 ? hist : reinterpret_cast<uint32_t*>(p);
  p += 4 * (size_t)(wmax + 1);
  uint32_t* ccnt = reinterpret_cast<uint32_t*>(p);
  p += 4 * (size_t)ncls_cap;
  uint32_t* cwhole = reinterpret_cast<uint32_t*>(p);
  p += 4 * (size_t)ncls_cap;
  uint8_t* cflag = p;
  p += ncls_cap;
  const int v = blockIdx.x / cs, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lo = cluster_lo(nb, cs, rk), nbl = cluster_lo(nb, cs, rk + 1) - lo;
  using AvT = typename std::conditional<kAv8, uint8_t, uint16_t>::type;
  Arr<uint16_t> wv;  // weight and allocation per block
  Arr<AvT> av;
  // per-block state laid out thread-strided (thread t's k-th block at k * kClassThreads + t) so
  // the warps' accesses coalesce while each thread still walks its blocks in index order
  const int span = class_span(nbl);
  if constexpr (kSmemArrays) {
    uint16_t* q = reinterpret_cast<uint16_t*>(dyn + ((p - dyn + 15) & ~15));
    wv.p = q;
    av.p = reinterpret_cast<AvT*>(q + span);
  } else {
    const int span_max = class_span((nb + cs - 1) / cs);
    wv.p = reinterpret_cast<uint16_t*>(gscratch) + (int64_t)blockIdx.x * 2 * span_max;
    if constexpr (kAv8) av.p = reinterpret_cast<AvT*>(dyn + ((p - dyn + 15) & ~15));
    else av.p = reinterpret_cast<AvT*>(wv.p + span);
  }
  const uint32_t* w = weights + (int64_t)v * nb + lo;
  const int per_b = (nbl + kClassThreads - 1) / kClassThreads;  // contiguous block range per thread
  const int b0 = min(nbl, tid * per_b), b1 = min(nbl, b0 + per_b);
  const int per_c = (wmax + 1 + kClassThreads - 1) / kClassThreads;
  const int c0 = min(wmax + 1, tid * per_c), c1 = min(wmax + 1, c0 + per_c);
  if (budget < 0 || (unsigned long long)budget > (unsigned long long)cap * (unsigned long long)nb || cap < 0 ||
      cap > 65535) {  // the same decision in every CTA of the cluster (before any cluster barrier)
    if (rk == 0 && tid == 0 && status) status[v] = ABCS_ERR_INVALID_ARGUMENT;
    return;
  }
  // cluster barrier (a CTA barrier for a cluster of one)
  auto csync = [&]() {
    if (cs == 1) __syncthreads();
    else cluster.sync();
  };
  // sum over the cluster's ranks < upto of pub[slot0] (and pub[slot1]) -> agg[0..1]; after csync
  auto cluster_sum2 = [&](int slot0, int slot1, int upto) {
    if (warp == 0) {
      long long a = 0, b = 0;
      if (lane < upto) {
        a = cs == 1 ? pub[slot0] : *cluster.map_shared_rank(&pub[slot0], lane);
        if (slot1 >= 0) b = cs == 1 ? pub[slot1] : *cluster.map_shared_rank(&pub[slot1], lane);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      if (lane == 0) {
        agg[0] = a;
        agg[1] = b;
      }
    }
    __syncthreads();
  };
  // weights: coalesced loads, scattered into the owners' thread-strided slots
  if (tid == 0) sh_int[3] = 0;
  __syncthreads();
  if constexpr (kSmemArrays) {
    for (int j = tid; j < nbl; j += kClassThreads) {
      const uint32_t wi = w[j];
      if (wi > (uint32_t)wmax) sh_int[3] = 1;  // caller's weight bound violated
      const int owner = j / per_b, ph = (j - owner * per_b) * kClassThreads + owner;
      wv[ph] = (uint16_t)min(wi, (uint32_t)wmax);
      av[ph] = 0;
    }
  } else {  // global state: keep its accesses coalesced, read the weights per thread range
    int i = b0, ph = tid;
    if (((uintptr_t)(w + b0) & 15) == 0)  // 16-byte loads of 4 weights
      for (; i + 4 <= b1; i += 4, ph += 4 * kClassThreads) {
        const uint4 q = *reinterpret_cast<const uint4*>(w + i);
        const uint32_t wq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (wq[e] > (uint32_t)wmax) sh_int[3] = 1;
          wv[ph + e * kClassThreads] = (uint16_t)min(wq[e], (uint32_t)wmax);
          av[ph + e * kClassThreads] = 0;
        }
      }
    for (; i < b1; ++i, ph += kClassThreads) {
      const uint32_t wi = w[i];
      if (wi > (uint32_t)wmax) sh_int[3] = 1;
      wv[ph] = (uint16_t)min(wi, (uint32_t)wmax);
      av[ph] = 0;
    }
  }
  __syncthreads();
  if (tid == 0) pub[5] = sh_int[3];
  csync();
  cluster_sum2(5, -1, cs);
  long long remaining = budget;
  int st = agg[0] ? ABCS_ERR_LOGIC : ABCS_OK;
  int round = 0;
  while (remaining > 0 && st == ABCS_OK) {
    if (++round > nb + 1) {
      st = ABCS_ERR_LOGIC;
      break;
    }
    for (int c = c0; c < c1; ++c) hist[c] = 0;
    __syncthreads();
    unsigned long long tw = 0, na = 0;
    if (wmax >= kAggregateBelow) {  // many distinct weights (BBV): plain shared atomics rarely collide
      for (int k = 0; k < per_b; ++k) {
        const int i = b0 + k, ph = k * kClassThreads + tid;
        if (i < b1 && (int)av[ph] < cap) {
          const int wi = (int)wv[ph];
          atomicAdd(&hist[wi], 1u);
          tw += (unsigned)wi;
          na += 1;
        }
      }
    } else {
      for (int k = 0; k < per_b; ++k) {  // warp-aggregated histogram (uniform trip count for match_any)
        const int i = b0 + k, ph = k * kClassThreads + tid;
        const bool act = i < b1 && (int)av[ph] < cap;
        const int wi = act ? (int)wv[ph] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, wi);
        if (act && (__ffs(peers) - 1) == lane) atomicAdd(&hist[wi], (unsigned)__popc(peers));
        if (act) {
          tw += (unsigned)wi;
          na += 1;
        }
      }
    }
    const unsigned long long T0l = Reduce64(tmp.r).Sum(tw);
    __syncthreads();
    const unsigned long long nal = Reduce64(tmp.r).Sum(na);
    if (tid == 0) {
      pub[0] = (long long)T0l;
      pub[1] = (long long)nal;
    }
    csync();  // A: pub[0..1] and every CTA's hist complete
    if (cs > 1)
      for (int c = c0; c < c1; ++c) {
        uint32_t h = 0;
        for (int q = 0; q < cs; ++q) h += cluster.map_shared_rank(hist, q)[c];
        ghist[c] = h;
      }
    cluster_sum2(0, 1, cs);  // (ends with __syncthreads: ghist complete)
    const bool uniform = agg[0] == 0;
    const uint64_t T = uniform ? (uint64_t)agg[1] : (uint64_t)agg[0];
    const long long n_act = agg[1];
    const ClassSel S = class_round_select(sm, ghist, c0, c1, remaining, T, uniform, n_act, ccnt, cwhole, ckey, cflag);
    auto cls_rel = [&](int k) -> int { return class_rel(S, k, ckey, cflag); };
    const bool sel_all = S.sel_all, none = S.none, all_equal_taken = S.all_equal_taken;
    long long need = S.need;
    long long tie_base = 0;
    if (!sel_all && !none && !all_equal_taken) {  // the same decision in every CTA
      int ties = 0;
      for (int i = b0, ph = tid; i < b1; ++i, ph += kClassThreads)
        if ((int)av[ph] < cap && cls_rel((int)ghist[wv[ph]]) == 2) ++ties;
      int tb, tot;
      ScanI(tmp.s).ExclusiveSum(ties, tb, tot);
      if (tid == 0) pub[2] = tot;
      csync();                 // C: tie counts of every rank published
      cluster_sum2(2, -1, rk);  // ties of the lower ranks (lower block indices)
      tie_base = tb + agg[0];
    }
    unsigned long long taken_sum = 0, still = 0;
    for (int i = b0, ph = tid; i < b1; ++i, ph += kClassThreads) {
      if ((int)av[ph] >= cap) continue;
      const int k = (int)ghist[wv[ph]];
      const int rel = cls_rel(k);
      bool sel = rel == 1;
      if (rel == 2) sel = all_equal_taken || (tie_base++) < need;
      const long long give = (long long)cwhole[k] + (sel ? 1 : 0);
      const long long room = (long long)cap - av[ph];
      const long long taken = give < room ? give : room;  // sensing.cpp:162-171
      av[ph] = (AvT)(av[ph] + taken);
      taken_sum += (unsigned long long)taken;
      if ((int)av[ph] < cap) still += 1;
    }
    const unsigned long long tk = Reduce64(tmp.r).Sum(taken_sum);
    __syncthreads();
    const unsigned long long st_open = Reduce64(tmp.r).Sum(still);
    if (tid == 0) {
      pub[3] = (long long)tk;
      pub[4] = (long long)st_open;
    }
    csync();  // D
    cluster_sum2(3, 4, cs);
    remaining -= agg[0];
    if (remaining > 0 && agg[1] == 0) st = ABCS_ERR_LOGIC;  // capacity exhausted
    __syncthreads();
  }
  // counts = base + allocation, offsets = exclusive scan over the image (this CTA's range
  // after the lower ranks'); written coalesced: warp w walks its threads' contiguous ranges
  // in index order with a running warp scan
  int mine = 0;
  for (int i = b0, ph = tid; i < b1; ++i, ph += kClassThreads) mine += base + (int)av[ph];
  int ex, total;
  ScanI(tmp.s).ExclusiveSum(mine, ex, total);
  if (tid == 0) pub[5] = total;
  csync();  // E
  cluster_sum2(5, -1, rk);
  uint16_t* cnt_out = counts + (int64_t)v * nb + lo;
  int32_t* off_out = offsets ? offsets + (int64_t)v * nb + lo : nullptr;
  if constexpr (!kSmemArrays) {  // global state: per thread range, 16-byte stores where aligned
    ex += (int)agg[0];
    int i = b0, ph = tid;
    if (((uintptr_t)(cnt_out + b0) & 15) == 0 && (!off_out || ((uintptr_t)(off_out + b0) & 15) == 0))
      for (; i + 8 <= b1; i += 8, ph += 8 * kClassThreads) {
        int c[8], o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          c[e] = base + (int)av[ph + e * kClassThreads];
          o[e] = ex;
          ex += c[e];
        }
        *reinterpret_cast<uint4*>(cnt_out + i) =
            make_uint4((uint32_t)c[0] | (uint32_t)c[1] << 16, (uint32_t)c[2] | (uint32_t)c[3] << 16,
                       (uint32_t)c[4] | (uint32_t)c[5] << 16, (uint32_t)c[6] | (uint32_t)c[7] << 16);
        if (off_out) {
          *reinterpret_cast<int4*>(off_out + i) = make_int4(o[0], o[1], o[2], o[3]);
          *reinterpret_cast<int4*>(off_out + i + 4) = make_int4(o[4], o[5], o[6], o[7]);
        }
      }
    for (; i < b1; ++i, ph += kClassThreads) {
      const int c = base + (int)av[ph];
      cnt_out[i] = (uint16_t)c;
      if (off_out) off_out[i] = ex;
      ex += c;
    }
  }
  int run = __shfl_sync(0xffffffffu, ex, 0) + (int)agg[0];  // prefix at block warp * 32 * per_b
  const int wbase = warp * 32 * per_b;
  for (int j = 0; j < (kSmemArrays ? per_b : 0); ++j) {
    const int idx = wbase + j * 32 + lane;
    int c = 0;
    if (idx < nbl) {
      const int owner = idx / per_b;
      c = base + (int)av[(idx - owner * per_b) * kClassThreads + owner];
    }
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (idx < nbl) {
      cnt_out[idx] = (uint16_t)c;
      if (off_out) off_out[idx] = run + incl - c;
    }
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (rk == 0 && tid == 0 && status) status[v] = st;
  if (cs > 1) cluster.sync();  // F: no CTA leaves while a peer may still read its shared memory
}

// Cluster size for n_vectors images of n_blocks: split an image over more CTAs only while the
// batch stays within half the SMs (cluster barriers cost more than they save beyond that; cfg5
// measured 0.45 / 0.27 / 0.09 / 0.12 / 0.14 ms at 1 / 2 / 4 / 8 / 16) and CTAs keep >= 2048 blocks.
static int class_cluster_size(const Ctx* ctx, int32_t n_blocks, int32_t n_vectors) {
  int cs = 1;
  while (2 * cs <= kMaxCluster && (int64_t)n_vectors * cs * 2 <= ctx->sm_count / 2 && n_blocks / (cs * 2) >= 2048)
    cs *= 2;
  return cs;
}

int launch_allocate(Ctx* ctx, const uint32_t* weights, int32_t n_blocks, int32_t n_vectors, int64_t budget,
                    const int32_t* caps, int32_t cap, int32_t base, uint16_t* counts, int32_t* offsets,
                    int32_t* status, void* scratch, cudaStream_t s, int32_t wmax) {
  if (n_vectors == 0 || n_blocks == 0) return ABCS_OK;
  if (!caps && wmax >= 0 && wmax < 65536 && cap <= 65535) {
    static bool attr_set = false;
    if (!attr_set) {
      for (auto k : {alloc_class_kernel<true>, alloc_class_kernel<false>, alloc_class_kernel<false, true>}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      }
      attr_set = true;
    }
    const char* env = getenv("ABCS_ALLOC_CLUSTER");  // tuning override (power of two <= 16)
    const int cs = env ? std::max(1, std::min(kMaxCluster, atoi(env))) : class_cluster_size(ctx, n_blocks, n_vectors);
    uint32_t* gscr = reinterpret_cast<uint32_t*>(scratch);  // n_vectors * n_blocks * 2 u16 (+ padding)
    const size_t smem_in = class_smem_bytes(wmax, n_blocks, cs, true);
    const size_t smem_out = class_smem_bytes(wmax, n_blocks, cs, false);
    // u8 allocations in shared memory beside global weights (caps <= 255)
    const size_t smem_av8 = smem_out + (size_t)class_span((n_blocks + cs - 1) / cs) + 16;
    bool in_smem, av8 = false;
    if (smem_in <= 100 * 1024) in_smem = true;  // keep 2 CTAs (2048 threads) per SM
    else if (smem_out <= 200 * 1024) {
      in_smem = false;
      av8 = cap <= 255 && smem_av8 <= 100 * 1024;
    } else goto generic;
    {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3((unsigned)(n_vectors * cs));
      lc.blockDim = dim3(kClassThreads);
      lc.dynamicSmemBytes = in_smem ? smem_in : av8 ? smem_av8 : smem_out;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      const int kt = ktimer_begin(ctx, s, "alloc_class");
      const cudaError_t e =
          in_smem ? cudaLaunchKernelEx(&lc, alloc_class_kernel<true>, weights, (int)n_blocks, (int)wmax, budget,
                                       (int)cap, (int)base, counts, offsets, status, gscr)
          : av8   ? cudaLaunchKernelEx(&lc, alloc_class_kernel<false, true>, weights, (int)n_blocks, (int)wmax,
                                       budget, (int)cap, (int)base, counts, offsets, status, gscr)
                  : cudaLaunchKernelEx(&lc, alloc_class_kernel<false>, weights, (int)n_blocks, (int)wmax, budget,
                                       (int)cap, (int)base, counts, offsets, status, gscr);
      ktimer_end(ctx, s, kt);
      ctx->launches++;
      if (e != cudaSuccess) return cuda_status(e, "allocate(class) launch");
      return cuda_status(cudaGetLastError(), "allocate(class) launch");
    }
  }
generic:
  AllocScratch scr;
  char* p = reinterpret_cast<char*>(scratch);
  const size_t n = (size_t)n_blocks * n_vectors;
  scr.key = reinterpret_cast<uint64_t*>(p);
  p += n * 8;
  scr.give = reinterpret_cast<uint32_t*>(p);
  p += n * 4;
  scr.alloc = reinterpret_cast<uint32_t*>(p);
  p += n * 4;
  scr.flag = reinterpret_cast<uint8_t*>(p);
  const int kt = ktimer_begin(ctx, s, "alloc_radix");
  alloc_kernel<<<n_vectors, kAllocThreads, 0, s>>>(weights, n_blocks, budget, caps, cap, base, counts, offsets,
                                                   status, scr);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "allocate launch");
}

// ---------------------------------------------------------------------------
// Sharded allocation: one weight vector (image) split over shards held by different
// GPUs / processes (intra-image sharding). Shard s owns the contiguous
// block range its caller assigns (shards in block order). The round structure is the
// cluster allocator's, with each exchange point turned into a kernel boundary and a
// host collective: (1) active-weight histogram + (sum w, active) -> all-reduce,
// (2) class table + threshold from the global histogram (identical on every shard) and
// the shard's tie-group count -> exclusive prefix over shards, (3) apply + clamp ->
// all-reduce of (taken, still open), (4) counts and offsets with the shard's global
// offset prefix. One 1024-thread CTA per shard; state persists in global scratch.
struct ShardState {
  ClassSel sel;
  long long remaining;
};

struct ShardArgs {
  const uint32_t* weights;  // the shard's weights (nbl)
  int nbl, wmax, cap, base;
  uint16_t* wv;  // thread-strided per-block state, class_span(nbl) entries each
  uint16_t* av;
  uint32_t* gh;  // wmax + 1: global histogram -> class index
  uint32_t* ccnt;
  uint32_t* cwhole;
  uint64_t* ckey;
  uint8_t* cflag;
  ShardState* state;
  long long* out;        // phase outputs (phase 1: wmax + 3 values)
  const long long* in;   // phase 2: the all-reduced phase-1 output
  long long remaining;   // phase 2
  long long prefix;      // phase 3: tie-group blocks in lower shards; phase 4: offset of the shard
  uint16_t* counts;      // phase 4
  int32_t* offsets;      // phase 4 (nullable)
};

size_t shard_scratch_bytes(int32_t n_blocks, int32_t wmax) {
  const size_t span = (size_t)class_span(n_blocks);
  const size_t nc = (size_t)wmax + 1;
  return 256 + sizeof(ShardState) + 2 * span * 2 + nc * (4 + 4 + 4 + 8 + 1) + 8 * (nc + 3) + 64;
}

__global__ void __launch_bounds__(kClassThreads) alloc_shard_kernel(int phase, ShardArgs A) {
  using Reduce64 = Reduce64C;
  using ScanI = ScanIC;
  __shared__ ClassShared sm;
  extern __shared__ __align__(16) unsigned int shist[];  // phase 1: wmax + 1 bins
  const int tid = threadIdx.x, lane = tid & 31;
  const int per_b = (A.nbl + kClassThreads - 1) / kClassThreads;
  const int b0 = min(A.nbl, tid * per_b), b1 = min(A.nbl, b0 + per_b);
  const int per_c = (A.wmax + 1 + kClassThreads - 1) / kClassThreads;
  const int c0 = min(A.wmax + 1, tid * per_c), c1 = min(A.wmax + 1, c0 + per_c);
  Arr<uint16_t> wv{A.wv}, av{A.av};
  if (phase == 0) {  // load: weights -> state; out[0] = weight bound violated
    unsigned bad = 0;
    for (int i = b0, ph = tid; i < b1; ++i, ph += kClassThreads) {
      const uint32_t wi = A.weights[i];
      bad |= wi > (uint32_t)A.wmax ? 1u : 0u;
      wv[ph] = (uint16_t)min(wi, (uint32_t)A.wmax);
      av[ph] = 0;
    }
    const unsigned long long b = Reduce64(sm.tmp.r).Sum(bad);
    if (tid == 0) A.out[0] = (long long)b;
  } else if (phase == 1) {  // local histogram of active weights, sum of weights, active count
    for (int c = tid; c <= A.wmax; c += kClassThreads) shist[c] = 0;
    __syncthreads();
    unsigned long long tw = 0, na = 0;
    for (int k = 0; k < per_b; ++k) {
      const int i = b0 + k, ph = k * kClassThreads + tid;
      const bool act = i < b1 && (int)av[ph] < A.cap;
      const int wi = act ? (int)wv[ph] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, wi);
      if (act && (__ffs(peers) - 1) == lane) atomicAdd(&shist[wi], (unsigned)__popc(peers));
      if (act) {
        tw += (unsigned)wi;
        na += 1;
      }
    }
    const unsigned long long T0 = Reduce64(sm.tmp.r).Sum(tw);
    __syncthreads();
    const unsigned long long n_act = Reduce64(sm.tmp.r).Sum(na);
    for (int c = tid; c <= A.wmax; c += kClassThreads) A.out[c] = shist[c];
    if (tid == 0) {
      A.out[A.wmax + 1] = (long long)T0;
      A.out[A.wmax + 2] = (long long)n_act;
    }
  } else if (phase == 2) {  // class table + threshold from the global histogram; local tie count
    for (int c = c0; c < c1; ++c) A.gh[c] = (uint32_t)A.in[c];
    const long long T0 = A.in[A.wmax + 1], n_act = A.in[A.wmax + 2];
    const bool uniform = T0 == 0;
    const uint64_t T = uniform ? (uint64_t)n_act : (uint64_t)T0;
    __syncthreads();
    const ClassSel S =
        class_round_select(sm, A.gh, c0, c1, A.remaining, T, uniform, n_act, A.ccnt, A.cwhole, A.ckey, A.cflag);
    __syncthreads();  // the class table and gh map complete
    int ties = 0;
    if (!S.sel_all && !S.none && !S.all_equal_taken)
      for (int i = b0, ph = tid; i < b1; ++i, ph += kClassThreads)
        if ((int)av[ph] < A.cap && class_rel(S, (int)A.gh[wv[ph]], A.ckey, A.cflag) == 2) ++ties;
    const unsigned long long tt = Reduce64(sm.tmp.r).Sum((unsigned long long)ties);
    if (tid == 0) {
      A.state->sel = S;
      A.state->remaining = A.remaining;
      A.out[0] = (long long)tt;
    }
  } else if (phase == 3) {  // apply with the tie ranks of the lower shards; out = (taken, still open)
    const ClassSel S = A.state->sel;
    long long tie_base = 0;
    if (!S.sel_all && !S.none && !S.all_equal_taken) {
      int ties = 0;
      for (int i = b0, ph = tid; i < b1; ++i, ph += kClassThreads)
        if ((int)av[ph] < A.cap && class_rel(S, (int)A.gh[wv[ph]], A.ckey, A.cflag) == 2) ++ties;
      int tb, tot;
      ScanI(sm.tmp.s).ExclusiveSum(ties, tb, tot);
      __syncthreads();
      tie_base = tb + A.prefix;
    }
    unsigned long long taken_sum = 0, still = 0;
    for (int i = b0, ph = tid; i < b1; ++i, ph += kClassThreads) {
      if ((int)av[ph] >= A.cap) continue;
      const int k = (int)A.gh[wv[ph]];
      const int rel = class_rel(S, k, A.ckey, A.cflag);
      bool sel = rel == 1;
      if (rel == 2) sel = S.all_equal_taken || (tie_base++) < S.need;
      const long long give = (long long)A.cwhole[k] + (sel ? 1 : 0);
      const long long room = (long long)A.cap - av[ph];
      const long long taken = give < room ? give : room;  // sensing.cpp:162-171
      av[ph] = (uint16_t)(av[ph] + taken);
      taken_sum += (unsigned long long)taken;
      if ((int)av[ph] < A.cap) still += 1;
    }
    const unsigned long long tk = Reduce64(sm.tmp.r).Sum(taken_sum);
    __syncthreads();
    const unsigned long long st_open = Reduce64(sm.tmp.r).Sum(still);
    if (tid == 0) {
      A.out[0] = (long long)tk;
      A.out[1] = (long long)st_open;
    }
  } else {  // phase 4: counts = base + allocation; offsets from the shard's global offset
    int mine = 0;
    for (int i = b0, ph = tid; i < b1; ++i, ph += kClassThreads) mine += A.base + (int)av[ph];
    int ex, total;
    ScanI(sm.tmp.s).ExclusiveSum(mine, ex, total);
    long long run = ex + A.prefix;
    for (int i = b0, ph = tid; i < b1; ++i, ph += kClassThreads) {
      const int c = A.base + (int)av[ph];
      A.counts[i] = (uint16_t)c;
      if (A.offsets) A.offsets[i] = (int32_t)run;
      run += c;
    }
    if (tid == 0) A.out[0] = total;
  }
}

int launch_alloc_shard(Ctx* ctx, int phase, const uint32_t* weights, int32_t n_blocks, int32_t wmax, int32_t cap,
                       int32_t base, void* scratch, long long* out, const long long* in, long long remaining,
                       long long prefix, uint16_t* counts, int32_t* offsets, cudaStream_t s) {
  ShardArgs A{};
  char* p = reinterpret_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* q = p;
    p += (bytes + 15) & ~size_t(15);
    return q;
  };
  const size_t span = (size_t)class_span(n_blocks), nc = (size_t)wmax + 1;
  A.state = reinterpret_cast<ShardState*>(take(sizeof(ShardState)));
  A.wv = reinterpret_cast<uint16_t*>(take(span * 2));
  A.av = reinterpret_cast<uint16_t*>(take(span * 2));
  A.ckey = reinterpret_cast<uint64_t*>(take(nc * 8));
  A.gh = reinterpret_cast<uint32_t*>(take(nc * 4));
  A.ccnt = reinterpret_cast<uint32_t*>(take(nc * 4));
  A.cwhole = reinterpret_cast<uint32_t*>(take(nc * 4));
  A.cflag = reinterpret_cast<uint8_t*>(take(nc));
  A.weights = weights;
  A.nbl = n_blocks;
  A.wmax = wmax;
  A.cap = cap;
  A.base = base;
  A.out = out;
  A.in = in;
  A.remaining = remaining;
  A.prefix = prefix;
  A.counts = counts;
  A.offsets = offsets;
  const size_t dyn = phase == 1 ? nc * 4 : 0;
  // the opt-in covers static + dynamic shared memory above 48 KB (ClassShared is ~14 KB static)
  if (dyn > 16 * 1024) cudaFuncSetAttribute(alloc_shard_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  const int kt = ktimer_begin(ctx, s, "alloc_shard");
  alloc_shard_kernel<<<1, kClassThreads, dyn, s>>>(phase, A);
  ktimer_end(ctx, s, kt);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "alloc_shard launch");
}

}  // namespace abcs_b200
