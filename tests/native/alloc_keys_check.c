/* Host build of the product's alloc_keys.h checked against x87 long double —
 * the arithmetic the reference's largest_remainder_allocate ranks with
 * (sensing.cpp:134-149). Prints "ok <n>" or the first mismatch. */
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include "alloc_keys.h"

static uint64_t s = 0x9E3779B97F4A7C15ull;
static uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 200000;
  for (long i = 0; i < n; ++i) {
    uint64_t rem, w, T;
    switch (i % 4) {
      case 0: rem = 1 + rnd() % 5000000; w = rnd() % 20000; T = 1 + rnd() % 2000000000ull; break;
      case 1: rem = 1 + rnd() % 100; w = rnd() % 100; T = 1 + rnd() % 100; break;        /* adversarial small */
      case 2: rem = 1 + rnd() % (1ull << 30); w = rnd() % (1ull << 30); T = 1 + rnd() % (1ull << 40); break;
      default: rem = 1 + rnd() % 70000; w = 1; T = 1 + rnd() % 70000; break;            /* uniform mode */
    }
    long double share = (long double)rem * (long double)w / (long double)T;
    long long whole = (long long)share;
    long double frac = share - (long double)whole;
    long double scaled = frac * 18446744073709551616.0L;
    long double fl = __builtin_floorl(scaled);
    uint64_t key = (uint64_t)fl;
    uint32_t flag = scaled != fl;
    ak_share a = ak_compute((ak_u128)rem * w, T);
    if ((uint64_t)whole != a.whole || key != a.key || flag != a.flag) {
      printf("mismatch rem=%llu w=%llu T=%llu: ref whole=%lld key=%llu flag=%u ; emu whole=%llu key=%llu flag=%u\n",
             (unsigned long long)rem, (unsigned long long)w, (unsigned long long)T, whole,
             (unsigned long long)key, flag, (unsigned long long)a.whole, (unsigned long long)a.key, a.flag);
      return 1;
    }
  }
  printf("ok %ld\n", n);
  return 0;
}
