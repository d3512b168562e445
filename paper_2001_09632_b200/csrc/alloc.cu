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
#include <cub/block/block_scan.cuh>

#include "alloc_keys.h"
#include "common.cuh"
#include "internal.h"

namespace abcs_b200 {

constexpr int kAllocThreads = 1024;

struct AllocScratch {
  uint64_t* key;
  uint32_t* give;
  uint32_t* alloc;
  uint8_t* flag;
};

size_t allocate_scratch_bytes(int32_t n_blocks, int32_t n_vectors) {
  const size_t per = (size_t)n_blocks * (8 + 4 + 4 + 1);
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
  __shared__ unsigned long long sh_prefix;
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

int launch_allocate(Ctx* ctx, const uint32_t* weights, int32_t n_blocks, int32_t n_vectors, int64_t budget,
                    const int32_t* caps, int32_t cap, int32_t base, uint16_t* counts, int32_t* offsets,
                    int32_t* status, void* scratch, cudaStream_t s) {
  if (n_vectors == 0 || n_blocks == 0) return ABCS_OK;
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
  alloc_kernel<<<n_vectors, kAllocThreads, 0, s>>>(weights, n_blocks, budget, caps, cap, base, counts, offsets,
                                                   status, scr);
  ctx->launches++;
  return cuda_status(cudaGetLastError(), "allocate launch");
}

}  // namespace abcs_b200
