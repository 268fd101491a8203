// lp_device.cuh — device building blocks of the liveput hot path (sm_100a).
//
//   * splitmix64 counter streams, bit-exact with the reference Rng
//     (rng.hpp:11-55): draw i of Rng(s) is fmix64(s + (i+1)*gamma).
//   * Rng::below without 64-bit division: r % b via three lazy Barrett
//     reductions of the 32-bit halves (b <= kMaxN), rejection limit
//     precomputed per bound.
//   * sample_distinct (rng.cpp:8-19) as a sparse partial Fisher-Yates: only
//     displaced pool positions are recorded, so a trial needs O(k) state
//     instead of an n-int pool.
//   * lexicographic k-subset unranking for the exact branch
//     (enumerate_vectors, preemption.cpp:23-45).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "lp_layout.h"

namespace lp {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Lazy Barrett reduction with m = floor(2^32 / d) (2^32 - 1 for d = 1):
// q = umulhi(a, m) is floor(a / d) or one less, so a - q d is congruent to a
// mod d and lies in [0, 2d).  negd = 2^32 - d makes it one IMAD after the
// IMAD.HI.
__device__ __forceinline__ uint32_t mod32_lazy(uint32_t a, uint32_t m, uint32_t negd) {
  return a + __umulhi(a, m) * negd;
}

// r % b for 64-bit r and b <= kMaxN: the halves are reduced lazily to [0, 2b),
// so h (2^32 mod b) + l < 2b(b + 1) < 2^32 for b < 46341; one more lazy
// reduction and min(x, x - b) (unsigned: x - b wraps when x < b) finish.
// Nine instructions (tools/micro/barrett_check.c checks b <= 46340).
__device__ __forceinline__ uint32_t mod64_small(uint64_t r, const DrawConst& c) {
  const uint32_t h = mod32_lazy(static_cast<uint32_t>(r >> 32), c.m32, c.negb);
  const uint32_t l = mod32_lazy(static_cast<uint32_t>(r), c.m32, c.negb);
  const uint32_t x = mod32_lazy(h * c.c32 + l, c.m32, c.negb);
  return min(x, x + c.negb);
}

// One Rng::below(b) draw from a splitmix state (rng.hpp:23-30).
__device__ __forceinline__ uint32_t draw_below(uint64_t& state, const DrawConst& c) {
  uint64_t r;
  do {
    state += kGamma;
    r = fmix64(state);
  } while (r >= c.lim);
  return mod64_small(r, c);
}

// Initial state of trial t: Rng(mix_seed(seed, t)) (preemption.cpp:53).
__device__ __forceinline__ uint64_t trial_state(uint64_t seed, uint64_t t) {
  return fmix64(seed + kGamma * (t + 1));
}

// Sorting network (bitonic) over a register array; KMAX a power of two.
template <int KMAX>
__device__ __forceinline__ void sort_regs(uint32_t (&s)[KMAX]) {
#pragma unroll
  for (int k2 = 2; k2 <= KMAX; k2 <<= 1) {
#pragma unroll
    for (int j2 = k2 >> 1; j2 > 0; j2 >>= 1) {
#pragma unroll
      for (int i = 0; i < KMAX; ++i) {
        const int l = i ^ j2;
        if (l > i) {
          const uint32_t a = s[i], b = s[l];
          const bool up = (i & k2) == 0;
          s[i] = up ? min(a, b) : max(a, b);
          s[l] = up ? max(a, b) : min(a, b);
        }
      }
    }
  }
}

// Monte-Carlo scenario of trial t in registers, sorted ascending; slots
// i >= k hold 0xffffffff.  dc[i] are the constants of below(n - i).
template <int KMAX>
__device__ __forceinline__ void gen_mc_regs(uint64_t seed, uint64_t t, int k, const DrawConst* dc,
                                            uint32_t (&s)[KMAX]) {
  uint64_t st = trial_state(seed, t);
  uint32_t tgt[KMAX], mov[KMAX];
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    s[i] = 0xffffffffu;
    if (i < k) {
      const uint32_t j = static_cast<uint32_t>(i) + draw_below(st, dc[i]);
      // pool[i] and pool[j] before the swap: the last displacement wins
      uint32_t vi = static_cast<uint32_t>(i), vj = j;
#pragma unroll
      for (int q = 0; q < i; ++q) {
        vi = (tgt[q] == static_cast<uint32_t>(i)) ? mov[q] : vi;
        vj = (tgt[q] == j) ? mov[q] : vj;
      }
      s[i] = (j == static_cast<uint32_t>(i)) ? vi : vj;
      tgt[i] = j;   // position j now holds the old pool[i]
      mov[i] = vi;
    }
  }
  sort_regs<KMAX>(s);
}

// Same draw, but only the selected set is kept: each slot is OR-ed into the
// thread's bitmap column BMc[w * T] (zeroed by the caller) and the smallest
// slot is returned.  The displacement map is packed (target << 16 | value)
// in KMAX registers, so k up to 64 stays out of shared memory.
template <int KMAX>
__device__ __forceinline__ uint32_t gen_mc_bitmap(uint64_t seed, uint64_t t, int k,
                                                  const DrawConst* dc, uint32_t* BMc, int T) {
  uint64_t st = trial_state(seed, t);
  uint32_t map[KMAX];
  uint32_t smin = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    if (i < k) {
      const uint32_t j = static_cast<uint32_t>(i) + draw_below(st, dc[i]);
      uint32_t vi = static_cast<uint32_t>(i), vj = j;
#pragma unroll
      for (int q = 0; q < i; ++q) {
        const uint32_t tg = map[q] >> 16;
        vi = (tg == static_cast<uint32_t>(i)) ? (map[q] & 0xffffu) : vi;
        vj = (tg == j) ? (map[q] & 0xffffu) : vj;
      }
      const uint32_t sel = (j == static_cast<uint32_t>(i)) ? vi : vj;
      map[i] = (j << 16) | vi;
      BMc[(sel >> 5) * T] |= 1u << (sel & 31);
      smin = min(smin, sel);
    }
  }
  return smin;
}

// gen_mc_bitmap with the displacement map in a strided shared-memory column
// (map[i * ms], any k): a compact loop instead of an unrolled one.
__device__ __forceinline__ uint32_t gen_mc_bitmap_smem(uint64_t seed, uint64_t t, int k,
                                                       const DrawConst* dc, uint32_t* map, int ms,
                                                       uint32_t* BMc, int T) {
  uint64_t st = trial_state(seed, t);
  uint32_t smin = 0xffffffffu;
  for (int i = 0; i < k; ++i) {
    const uint32_t j = static_cast<uint32_t>(i) + draw_below(st, dc[i]);
    uint32_t vi = static_cast<uint32_t>(i), vj = j;
    for (int q = 0; q < i; ++q) {
      const uint32_t e = map[q * ms];
      const uint32_t tg = e >> 16;
      vi = (tg == static_cast<uint32_t>(i)) ? (e & 0xffffu) : vi;
      vj = (tg == j) ? (e & 0xffffu) : vj;
    }
    const uint32_t sel = (j == static_cast<uint32_t>(i)) ? vi : vj;
    map[i * ms] = (j << 16) | vi;
    atomicOr(BMc + (sel >> 5) * T, 1u << (sel & 31));
    smin = min(smin, sel);
  }
  return smin;
}

// gen_mc_bitmap with the displaced pool positions held in a per-thread byte
// table (n <= 256, so positions and values fit a byte): TAB[p] is valid when
// bit p of the thread's displaced bitmap DISc[w * T] is set (the caller
// zeroes it).  O(1) per draw instead of a scan of the earlier draws.  TAB is
// this thread's byte column: position p lives in word (p >> 2) * T, byte
// p & 3, so every lane of a warp stays in its own bank.
__device__ __forceinline__ uint32_t tab_off(uint32_t p, int T) {
  return (p & ~3u) * static_cast<uint32_t>(T) + (p & 3u);
}

__device__ __forceinline__ uint32_t gen_mc_bitmap_tab(uint64_t seed, uint64_t t, int k,
                                                      const DrawConst* dc, uint8_t* TAB,
                                                      uint32_t* DISc, uint32_t* BMc, int T) {
  uint64_t st = trial_state(seed, t);
  uint32_t smin = 0xffffffffu;
  for (int i = 0; i < k; ++i) {
    const uint32_t ui = static_cast<uint32_t>(i);
    const uint32_t j = ui + draw_below(st, dc[i]);
    const uint32_t di = DISc[(ui >> 5) * T];
    uint32_t vi = ui;
    if ((di >> (ui & 31u)) & 1u) vi = TAB[tab_off(ui, T)];
    uint32_t* dw = DISc + (j >> 5) * T;
    const uint32_t dj = *dw;
    uint32_t vj = j;
    const uint32_t oj = tab_off(j, T);
    if ((dj >> (j & 31u)) & 1u) vj = TAB[oj];
    const uint32_t sel = (j == ui) ? vi : vj;
    TAB[oj] = static_cast<uint8_t>(vi);  // position j now holds the old pool[i]
    *dw = dj | (1u << (j & 31u));
    // fire-and-forget OR: the column is this thread's, but a shared-memory
    // atomic has no result to wait for, so the next draw does not stall on it
    atomicOr(BMc + (sel >> 5) * T, 1u << (sel & 31u));
    smin = min(smin, sel);
  }
  return smin;
}

// Saturated binomial C(a, b) from the exact pair's table, indexed by
// (a, min(b, a-b)); callers guarantee a - b <= n - k and b <= k.
__device__ __forceinline__ uint64_t binom_at(const uint64_t* tab, int stride, int a, int b) {
  if (b < 0 || a < b) return 0;
  const int s = min(b, a - b);
  return tab[a * stride + s];
}

// rank-th k-subset of [0, n) in lexicographic order (the order of
// enumerate_vectors), sorted ascending.
template <int KMAX>
__device__ __forceinline__ void gen_exact_regs(uint64_t rank, int n, int k, const uint64_t* binom,
                                               int stride, uint32_t (&s)[KMAX]) {
  int c = 0;
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    s[i] = 0xffffffffu;
    if (i < k) {
      const int rem = k - i - 1;
      while (true) {
        const uint64_t num = binom_at(binom, stride, n - c - 1, rem);
        if (rank < num) break;
        rank -= num;
        ++c;
      }
      s[i] = static_cast<uint32_t>(c);
      ++c;
    }
  }
}

// Generic-k versions writing to strided scratch (shared or global memory).
// map[i * ms] holds (target << 16) | moved value of draw i; bm[w * bs] is a
// per-trial bitmap of the selected set; out[j * os] receives the sorted set.
__device__ __forceinline__ int gen_mc_generic(uint64_t seed, uint64_t t, int n, int k,
                                              const DrawConst* dc, uint32_t* map, int ms,
                                              uint32_t* bm, int bs, uint16_t* out, int os) {
  uint64_t st = trial_state(seed, t);
  const int nw = (n + 31) >> 5;
  for (int w = 0; w < nw; ++w) bm[w * bs] = 0u;
  for (int i = 0; i < k; ++i) {
    const uint32_t j = static_cast<uint32_t>(i) + draw_below(st, dc[i]);
    uint32_t vi = static_cast<uint32_t>(i), vj = j;
    for (int q = 0; q < i; ++q) {
      const uint32_t e = map[q * ms];
      const uint32_t tg = e >> 16, mv = e & 0xffffu;
      vi = (tg == static_cast<uint32_t>(i)) ? mv : vi;
      vj = (tg == j) ? mv : vj;
    }
    const uint32_t sel = (j == static_cast<uint32_t>(i)) ? vi : vj;
    map[i * ms] = (j << 16) | vi;
    bm[(sel >> 5) * bs] |= 1u << (sel & 31);
  }
  int c = 0;
  for (int w = 0; w < nw; ++w) {
    uint32_t bits = bm[w * bs];
    while (bits) {
      const int b = __ffs(bits) - 1;
      out[(c++) * os] = static_cast<uint16_t>(w * 32 + b);
      bits &= bits - 1;
    }
  }
  return c;
}

__device__ __forceinline__ void gen_exact_generic(uint64_t rank, int n, int k, const uint64_t* binom,
                                                  int stride, uint16_t* out, int os) {
  int c = 0;
  for (int i = 0; i < k; ++i) {
    const int rem = k - i - 1;
    while (true) {
      const uint64_t num = binom_at(binom, stride, n - c - 1, rem);
      if (rank < num) break;
      rank -= num;
      ++c;
    }
    out[i * os] = static_cast<uint16_t>(c);
    ++c;
  }
}

// floor(s / P) for s < 2^20 with magic = floor(2^32/P)+1 (P >= 2).
__device__ __forceinline__ uint32_t div_p(uint32_t s, uint32_t magic) { return __umulhi(s, magic); }

}  // namespace lp
