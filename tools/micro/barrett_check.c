// Check of the device draw's r % b (lp_device.cuh mod64_small: three lazy
// Barrett reductions, then min(x, x - b)) against the 64-bit % operator:
// every b <= 46340 (kMaxN = 16384 is the largest bound the draws use), 2000
// random 64-bit r each plus edge values; and the lazy reduction's range
// a - umulhi(a, m) b in [0, 2b) on the same samples.
//   gcc -O2 -o barrett_check barrett_check.c && ./barrett_check   -> bad=0
#include <stdio.h>
#include <stdint.h>
static uint64_t s = 0x12345;
static uint64_t rnd() {
  s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static uint32_t umulhi(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }
static uint32_t lazy(uint32_t a, uint32_t m, uint32_t negb) { return a + umulhi(a, m) * negb; }
int main() {
  long bad = 0;
  for (uint32_t b = 1; b <= 46340; ++b) {
    const uint32_t m = b == 1 ? 0xffffffffu : (uint32_t)((1ull << 32) / b);
    const uint32_t c32 = (uint32_t)((1ull << 32) % b), negb = 0u - b;
    for (int t = 0; t < 2000; ++t) {
      uint64_t r = rnd();
      if (t < 4) r = t == 0 ? 0 : t == 1 ? ~0ull : t == 2 ? ((uint64_t)b << 32) - 1 : (uint64_t)-1 - b;
      const uint32_t h = lazy((uint32_t)(r >> 32), m, negb), l = lazy((uint32_t)r, m, negb);
      if (h >= 2 * b || l >= 2 * b) ++bad;
      const uint32_t x = lazy(h * c32 + l, m, negb);
      const uint32_t xs = x + negb;
      const uint32_t got = x < xs ? x : xs;
      if (got != r % b) {
        if (bad < 5) printf("bad b=%u r=%llu got %u want %llu\n", b, (unsigned long long)r, got, (unsigned long long)(r % b));
        ++bad;
      }
    }
  }
  printf("bad=%ld\n", bad);
  return 0;
}
