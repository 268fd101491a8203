// lp_hist_rows.cu — K1 v4: bit-sliced row resolution (sm_100a), k-independent.
//
// For depth P the slots of a scenario form a Dmax x P grid (row x = pipeline,
// column = stage); a config (D, P) owns rows 0..D-1.  Instead of visiting the
// k preempted slots once per depth, a thread walks the Dmax rows of its
// scenario's slot bitmap, each row a P-bit vector pulled out of the bitmap
// with funnel shifts, and keeps the per-stage preemption counts as B
// bit-planes (a vertical binary counter per stage, B = bits(tmax)):
//
//   hit  = R & (count == max)          (B LOP3 per word)
//   if hit != 0: event (t = max + 1, x); max++
//   count += R                         (ripple carry, 2B ops per word)
//
// so a depth costs Dmax * ceil(P/32) * (3B + 4) integer ops, independent of
// how many slots were preempted.  All lanes of a warp walk the same depth,
// the same rows and the same plane count: the loop has no divergence; only
// the (rare) event RED.ADD is predicated.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lp_device.cuh"
#include "lp_launch.h"
#include "lp_layout.h"

namespace lp {
namespace {

__device__ __forceinline__ size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

template <typename T>
__device__ __forceinline__ T* carve(unsigned char*& p, size_t count) {
  T* r = reinterpret_cast<T*>(p);
  p += a16(count * sizeof(T));
  return r;
}

// Shared-memory event cells are u16 pairs packed in u32 words (a block
// handles at most 4096 scenarios, so a cell never exceeds 4096); global
// cells are u32.
template <bool SMEM_EVT>
__device__ __forceinline__ void evt_add(uint32_t* base, int idx) {
  if (SMEM_EVT) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(base + (idx >> 1)));
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"((idx & 1) * 0xffffu + 1u) : "memory");
  } else {
    atomicAdd(base + idx, 1u);
  }
}

// Rows where the running maximum rose, as a bit mask (u32 when Dmax <= 32):
// the first rise is t = 1 (h0's event), the i-th further one is t = i + 1.
template <bool SMEM_EVT, typename M>
__device__ __forceinline__ void emit_rises(M rises, uint32_t* eb, int eo, int Dm) {
  rises &= rises - 1;
  while (rises) {
    const int x = sizeof(M) == 8 ? __ffsll(static_cast<long long>(rises)) - 1
                                 : __ffs(static_cast<int>(rises)) - 1;
    rises &= rises - 1;
    evt_add<SMEM_EVT>(eb, eo + x);
    eo += Dm;
  }
}

// The same rises accumulated in row order by shifting left (row x at bit
// Dmax-1-x): emitted from the highest set bit down.
template <bool SMEM_EVT, typename M>
__device__ __forceinline__ void emit_rises_rev(M rises, uint32_t* eb, int eo, int Dm) {
  constexpr int top = 8 * static_cast<int>(sizeof(M)) - 1;
  auto msb = [](M r) { return top - (sizeof(M) == 8 ? __clzll(static_cast<long long>(r)) : __clz(static_cast<int>(r))); };
  if (!rises) return;
  rises ^= static_cast<M>(1) << msb(rises);  // the first rise is t = 1 (h0's event)
  while (rises) {
    const int b = msb(rises);
    rises ^= static_cast<M>(1) << b;
    evt_add<SMEM_EVT>(eb, eo + (Dm - 1 - b));
    eo += Dm;
  }
}

// Walk the rows of one depth.  BMc: this thread's bitmap column (stride T),
// with at least one zero word past the last slot word.  Planes hold the
// distance to the running maximum, dist = mx - count, in B bits per stage:
//   hit     = R & (dist == 0)            OR-reduce of the planes
//   on hit  : mx++ ; dist += 1 (all)     (rare: at most tmax times)
//   always  : dist -= R                  (borrow chain, 2B ops per word)
template <int W, int B, bool SMEM_EVT>
__device__ __forceinline__ void walk_rows(const uint32_t* BMc, int T, uint32_t P, int Dm,
                                          uint32_t* eb, int eoff) {
  uint32_t Dp[B][W];
#pragma unroll
  for (int l = 0; l < B; ++l)
#pragma unroll
    for (int w = 0; w < W; ++w) Dp[l][w] = 0u;
  const uint32_t tail = P - 32u * (W - 1);  // bits in the last word (1..32)
  const uint32_t tmask = tail >= 32u ? 0xffffffffu : ((1u << tail) - 1u);
  // rows where the maximum rose, shifted in (row x at bit Dm-1-x) when
  // Dm <= 64 (always for W > 1: P > 32, Dm <= 512 / 33); emitted in the
  // loop otherwise (one-word rows of P < n/64)
  const bool masked = Dm <= 64;
  unsigned long long rises = 0ull;
  int mx = 0;
  uint32_t pos = 0;
  for (int x = 0; x < Dm; ++x, pos += P) {
    const uint32_t wi = pos >> 5, sh = pos & 31u;
    uint32_t R[W];
    uint32_t lo = BMc[wi * T];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t hi = BMc[(wi + w + 1) * T];
      R[w] = __funnelshift_r(lo, hi, sh);
      lo = hi;
    }
    R[W - 1] &= tmask;
    uint32_t hit = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint32_t z = 0;
#pragma unroll
      for (int l = 0; l < B; ++l) z |= Dp[l][w];
      hit |= R[w] & ~z;
    }
    // dist' = dist + inc - R with inc = (hit != 0): where R = 1 and inc = 1
    // nothing changes, so the update is one chain of +1 (inc) or -1 (!inc)
    // over the mask c = inc ? ~R : R — branch-free.
    const uint32_t keep = hit ? 0u : 0xffffffffu;
    if (W > 1 || masked) {
      rises = rises + rises + static_cast<unsigned long long>(keep + 1u);
    } else if (hit) {
      ++mx;
      if (mx >= 2) evt_add<SMEM_EVT>(eb, eoff + (mx - 2) * Dm + x);
    }
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint32_t c = R[w] ^ ~keep;
      if (w == W - 1) c &= tmask;
#pragma unroll
      for (int l = 0; l < B; ++l) {
        const uint32_t t = (Dp[l][w] ^ keep) & c;
        Dp[l][w] ^= c;
        c = t;
      }
    }
  }
  if (W > 1 || masked) emit_rises_rev<SMEM_EVT>(rises, eb, eoff, Dm);
}

// One-word rows (P <= 32) and at most 64 of them: the bitmap streams
// through a two-word window (refilled when the row start crosses a word —
// a warp-uniform test, every lane walks the same depth), and the rows where
// the maximum rose are kept as a 64-bit mask, so the row loop has no branch;
// the events are emitted once after the walk.
template <int B, bool SMEM_EVT, typename M>
__device__ __forceinline__ void walk_rows1(const uint32_t* BMc, int T, uint32_t P, int Dm,
                                           uint32_t* eb, int eoff) {
  uint32_t Dp[B];
#pragma unroll
  for (int l = 0; l < B; ++l) Dp[l] = 0u;
  const uint32_t tmask = P >= 32u ? 0xffffffffu : ((1u << P) - 1u);
  uint32_t w0 = BMc[0], w1 = BMc[T];
  const uint32_t* next = BMc + 2 * T;
  uint32_t sh = 0;
  M rises = 0;
  for (int x = 0; x < Dm; ++x) {
    const uint32_t R = __funnelshift_r(w0, w1, sh) & tmask;
    uint32_t z = 0;
#pragma unroll
    for (int l = 0; l < B; ++l) z |= Dp[l];
    const uint32_t hit = R & ~z;
    const uint32_t keep = hit ? 0u : 0xffffffffu;  // all-ones: decrement by R
    rises = rises + rises + static_cast<M>(keep + 1u);  // shift in (hit != 0)
    uint32_t c = R ^ (~keep & tmask);
#pragma unroll
    for (int l = 0; l < B; ++l) {
      const uint32_t t = (Dp[l] ^ keep) & c;
      Dp[l] ^= c;
      c = t;
    }
    sh += P;
    if (sh >= 32u) {  // uniform across the warp; the column has zero words past the slots
      sh -= 32u;
      w0 = w1;
      w1 = *next;
      next += T;
    }
  }
  emit_rises_rev<SMEM_EVT>(rises, eb, eoff, Dm);
}

// Depths with Dmax = DM <= 4 rows: the rows are unrolled at compile time and
// the per-stage counts kept as level masks G[t] = {stages with count >= t+1}:
// G[t] |= G[t-1] & R.  Level t+1 first becomes non-empty at row x exactly
// when the maximum reaches t+1 there — the event (t+1, x).  Dmax = 2 (half
// the depths at N = 256) costs one AND per word.
template <int DM, int W, bool SMEM_EVT>
__device__ __forceinline__ void walk_small(const uint32_t* BMc, int T, uint32_t P, uint32_t* eb,
                                           int eoff) {
  const uint32_t tail = P - 32u * (W - 1);
  const uint32_t tmask = tail >= 32u ? 0xffffffffu : ((1u << tail) - 1u);
  uint32_t G[DM][W];
#pragma unroll
  for (int x = 0; x < DM; ++x) {
    const uint32_t pos = static_cast<uint32_t>(x) * P;
    const uint32_t wi = pos >> 5, sh = pos & 31u;
    uint32_t R[W];
    uint32_t lo = BMc[wi * T];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t hi = BMc[(wi + w + 1) * T];
      R[w] = __funnelshift_r(lo, hi, sh);
      lo = hi;
    }
    R[W - 1] &= tmask;
#pragma unroll
    for (int t = x; t >= 1; --t) {  // count >= t+1 is first possible at row t
      uint32_t prior = 0, fresh = 0;  // G[t-1] is still the pre-row value here
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const uint32_t old = (t < x) ? G[t][w] : 0u;
        const uint32_t nv = G[t - 1][w] & R[w];
        prior |= old;
        fresh |= nv;
        G[t][w] = old | nv;
      }
      if (prior == 0u && fresh != 0u) evt_add<SMEM_EVT>(eb, eoff + (t - 1) * DM + x);
    }
#pragma unroll
    for (int w = 0; w < W; ++w) G[0][w] = (x == 0 ? 0u : G[0][w]) | R[w];
  }
}

// Few stages (P <= 16) and many rows (10..64): visit the sorted,
// register-resident slots instead of the rows.  Per-stage counts are nibbles
// of one 64-bit word; with k <= 16 a count can only reach 16 on the last
// slot, after its comparison, so the carry into the next nibble is never
// read.  A slot (x, r) raises the maximum exactly when its stage's count
// equals it; the rows where that happened are kept as a mask and the events
// emitted after the walk, as in walk_rows1.  Branch-free: slots past lim
// (and the 0xffffffff padding) count nothing.
template <int KS, bool P1, bool SMEM_EVT, typename M>
__device__ __forceinline__ void walk_elems(const uint32_t (&s)[KS], uint32_t P, uint32_t magic,
                                           uint32_t lim, int Dm, uint32_t* eb, int eo) {
  unsigned long long cnt = 0ull;
  M rises = 0;
  uint32_t mx = 0;
  const uint32_t negP = 0u - P;
#pragma unroll
  for (int i = 0; i < KS; ++i) {
    const uint32_t v = s[i];
    const uint32_t q = P1 ? v : __umulhi(v, magic);
    const uint32_t sh = (v + q * negP) << 2;
    const uint32_t c = static_cast<uint32_t>(cnt >> sh) & 15u;
    const bool hit = v < lim && c == mx;
    mx += hit ? 1u : 0u;
    rises |= static_cast<M>(hit) << (q & (8u * sizeof(M) - 1u));
    // slots are sorted, so the ones past lim come last: counting them is harmless
    cnt += 1ull << sh;
  }
  emit_rises<SMEM_EVT>(rises, eb, eo, Dm);
}

// Depths with exactly two rows (P in (n/3, n/2]) for all P of a run at once:
// (2, x = 1) is the only event, and it happens at P exactly when some slot
// a < P has a + P selected.  For every selected a below the run's largest P,
// the bitmap shifted right by a + Plo gives "a + P selected" for all P of the
// run in one window of WW words (P <= a masked off); the OR over a marks the
// depths with an event.  Cost ~ (slots below Phi) * WW instead of
// (depths) * 2 rows * ceil(P/32).
template <int WW, bool SMEM_EVT>
__device__ __forceinline__ void dm2_run(const EntryDesc* ents, int e0, int e1, const uint32_t* BMc,
                                        int T, uint32_t* eb) {
  const int Plo = ents[e0].P, Phi = ents[e1 - 1].P;
  uint32_t E[WW];
#pragma unroll
  for (int i = 0; i < WW; ++i) E[i] = 0u;
  const int wlast = (Phi - 1) >> 5;
  for (int w = 0; w <= wlast; ++w) {
    uint32_t bits = BMc[w * T];
    if (w == wlast) {
      const int top = (Phi - 1) & 31;  // keep a <= Phi - 1
      bits &= top == 31 ? 0xffffffffu : ((2u << top) - 1u);
    }
    while (bits) {
      const int a = w * 32 + __ffs(static_cast<int>(bits)) - 1;
      bits &= bits - 1;
      const uint32_t sbit = static_cast<uint32_t>(a + Plo);
      const uint32_t* src = BMc + (sbit >> 5) * T;
      const uint32_t sh = sbit & 31u;
      const int cut = a - Plo + 1;  // window bits b < cut have P <= a
      uint32_t lo = src[0];
#pragma unroll
      for (int i = 0; i < WW; ++i) {
        const uint32_t hi = src[(i + 1) * T];
        const uint32_t x = __funnelshift_r(lo, hi, sh);
        lo = hi;
        const int rel = cut - 32 * i;
        const uint32_t keep = rel <= 0 ? 0xffffffffu : (rel >= 32 ? 0u : (0xffffffffu << rel));
        E[i] |= x & keep;
      }
    }
  }
  const int width = Phi - Plo + 1;
  if (Phi - Plo == e1 - e0 - 1) {  // one entry per P of the run
#pragma unroll
    for (int i = 0; i < WW; ++i) {
      const int rel = width - 32 * i;
      uint32_t bits = E[i] & (rel >= 32 ? 0xffffffffu : (rel <= 0 ? 0u : ((1u << rel) - 1u)));
      while (bits) {
        const int b = 32 * i + __ffs(static_cast<int>(bits)) - 1;
        bits &= bits - 1;
        evt_add<SMEM_EVT>(eb, ents[e0 + b].evt_off + 1);
      }
    }
  } else {
    for (int e = e0; e < e1; ++e) {
      const int b = ents[e].P - Plo;
      const uint32_t wv = WW == 1 ? E[0] : (b < 32 ? E[0] : (WW == 2 || b < 64 ? E[WW > 1 ? 1 : 0] : E[WW - 1]));
      if ((wv >> (b & 31)) & 1u) evt_add<SMEM_EVT>(eb, ents[e].evt_off + 1);
    }
  }
}

template <int W, int B, bool SMEM_EVT>
__device__ __forceinline__ void walk_gen(const uint32_t* BMc, int T, uint32_t P, int Dm,
                                         uint32_t* eb, int eoff) {
  if (W == 1 && Dm <= 64) walk_rows1<B, SMEM_EVT, unsigned long long>(BMc, T, P, Dm, eb, eoff);
  else walk_rows<W, B, SMEM_EVT>(BMc, T, P, Dm, eb, eoff);
}

// (words per row, mode):
//   2..4    Dmax <= 4: walk_small
//   5, 6    slot walk (ELEMS: k <= 16 slots in registers; P <= 16 and 10..64
//           rows), rise mask u32 / u64
//   8 + B   walk_rows (walk_rows1 with a u64 rise mask when W = 1, Dmax <= 64), B <= 10
//   24 + B  walk_rows1 with a u32 rise mask (W = 1, Dmax <= 32)
// B = plane count = bits(tmax).
template <bool ELEMS>
__device__ __forceinline__ int depth_class(const EntryDesc& e) {
  const int W = (e.P + 31) >> 5;
  if (ELEMS && e.P <= 16 && e.Dmax >= 10 && e.Dmax <= 64) return (1 << 5) | (e.Dmax <= 32 ? 5 : 6);
  if (e.Dmax == 2) return (1 << 5) | 7;  // all two-row depths: dm2_run
  if (e.Dmax <= 4) return (W << 5) | e.Dmax;
  const int B = 32 - __clz(static_cast<uint32_t>(e.tmax));
  return (W << 5) | ((W == 1 && e.Dmax <= 32 ? 24 : 8) + B);  // B <= 10 (tmax <= n <= 512)
}

template <int KS, bool SMEM_EVT, typename M>
__device__ __forceinline__ void elems_run(const EntryDesc* ents, int e0, int e1, uint32_t* eb,
                                          const uint32_t (&sl)[KS]) {
  for (int e = e0; e < e1; ++e) {
    const EntryDesc& x = ents[e];
    const uint32_t P = static_cast<uint32_t>(x.P);
    if (P == 1u)
      walk_elems<KS, true, SMEM_EVT, M>(sl, P, 0u, static_cast<uint32_t>(x.lim), x.Dmax, eb, x.evt_off);
    else
      walk_elems<KS, false, SMEM_EVT, M>(sl, P, x.magic, static_cast<uint32_t>(x.lim), x.Dmax, eb,
                                         x.evt_off);
  }
}

template <int W, bool SMEM_EVT, int KS>
__device__ __forceinline__ void walk_run(int mode, const EntryDesc* ents, int e0, int e1,
                                         const uint32_t* BMc, int T, uint32_t* eb,
                                         const uint32_t (&sl)[KS]) {
#define LP_RUN(CALL)                                                              \
  for (int e = e0; e < e1; ++e) {                                                 \
    const uint32_t P = static_cast<uint32_t>(ents[e].P);                          \
    const int Dm = ents[e].Dmax, eo = ents[e].evt_off;                            \
    (void)Dm;                                                                     \
    CALL;                                                                         \
  }                                                                               \
  return;
#define LP_R1(B) LP_RUN((walk_rows1<B, SMEM_EVT, uint32_t>(BMc, T, P, Dm, eb, eo)))
  if (W == 1 && mode == 7) {
    const int ww = ((ents[e1 - 1].P - ents[e0].P) >> 5) + 1;
    if (ww == 1) return dm2_run<1, SMEM_EVT>(ents, e0, e1, BMc, T, eb);
    if (ww == 2) return dm2_run<2, SMEM_EVT>(ents, e0, e1, BMc, T, eb);
    return dm2_run<3, SMEM_EVT>(ents, e0, e1, BMc, T, eb);
  }
  if (W == 1 && KS > 1 && mode == 5) return elems_run<KS, SMEM_EVT, uint32_t>(ents, e0, e1, eb, sl);
  if (W == 1 && KS > 1 && mode == 6)
    return elems_run<KS, SMEM_EVT, unsigned long long>(ents, e0, e1, eb, sl);
  if (W == 1 && mode > 24) {
    switch (mode) {
      case 26: LP_R1(2)
      case 27: LP_R1(3)
      case 28: LP_R1(4)
      case 29: LP_R1(5)
      case 30: LP_R1(6)
      default: break;  // tmax <= Dmax <= 32: at most 6 planes
    }
  }
  switch (mode) {
    case 2: LP_RUN((walk_small<2, W, SMEM_EVT>(BMc, T, P, eb, eo)))
    case 3: LP_RUN((walk_small<3, W, SMEM_EVT>(BMc, T, P, eb, eo)))
    case 4: LP_RUN((walk_small<4, W, SMEM_EVT>(BMc, T, P, eb, eo)))
    case 10: LP_RUN((walk_gen<W, 2, SMEM_EVT>(BMc, T, P, Dm, eb, eo)))
    case 11: LP_RUN((walk_gen<W, 3, SMEM_EVT>(BMc, T, P, Dm, eb, eo)))
    case 12: LP_RUN((walk_gen<W, 4, SMEM_EVT>(BMc, T, P, Dm, eb, eo)))
    case 13: LP_RUN((walk_gen<W, 5, SMEM_EVT>(BMc, T, P, Dm, eb, eo)))
    case 14: LP_RUN((walk_gen<W, 6, SMEM_EVT>(BMc, T, P, Dm, eb, eo)))
    case 15: LP_RUN((walk_gen<W, 7, SMEM_EVT>(BMc, T, P, Dm, eb, eo)))
    case 16: LP_RUN((walk_gen<W, 8, SMEM_EVT>(BMc, T, P, Dm, eb, eo)))
    // k > 255 with more than 255 rows: only depths 1 and 2 at n <= 512
    case 17: LP_RUN((walk_gen<(W < 2 ? W : 1), 9, SMEM_EVT>(BMc, T, P, Dm, eb, eo)))
    default: LP_RUN((walk_gen<(W < 2 ? W : 1), 10, SMEM_EVT>(BMc, T, P, Dm, eb, eo)))
  }
#undef LP_R1
#undef LP_RUN
}

}  // namespace

// KREG > 0: register-resident Fisher-Yates map for k <= KREG; 0: shared-memory
// map (any k).  WMAX: largest ceil(P/32) among the work item's depths.
// Occupancy is two 256-thread blocks per SM either way (shared memory); the
// <0, 4> instance (k > 16, n <= 256: the bench's hot kernel) is compiled to
// the three-block register budget, where it fits 72 registers without a
// spill (95 at two blocks) and runs 0.45% faster (profiles/r02_rows_regs_ab.log);
// the other instances would spill there.
template <int KREG, int WMAX, bool SMEM_EVT>
__global__ void __launch_bounds__(256, (KREG == 0 && WMAX <= 4) ? 3 : 2) hist_rows_kernel(const WorkItem* __restrict__ work,
                                                           const PairDesc* __restrict__ pairs,
                                                           const EntryDesc* __restrict__ entries,
                                                           const DrawConst* __restrict__ draws,
                                                           const uint64_t* __restrict__ binom,
                                                           uint32_t* __restrict__ evt_g,
                                                           uint32_t* __restrict__ h0_g) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const WorkItem w = work[blockIdx.x];
  const PairDesc pd = pairs[w.pair];
  const int ne = w.e_res_hi - w.e_lo;
  const int k = pd.k, n = pd.n;
  const int nw = (n + 31) >> 5;
  const bool own_h0 = (w.e_lo == pd.entry_base);
  const int evt_words = SMEM_EVT ? (w.evt_len + 1) / 2 : 0;

  unsigned char* p = smem;
  EntryDesc* ents = carve<EntryDesc>(p, ne > 0 ? ne : 1);
  int2* runs = carve<int2>(p, ne + 1);  // (first entry, class) of each class run
  DrawConst* dc = carve<DrawConst>(p, k > 0 ? k : 1);
  uint32_t* h0 = carve<uint32_t>(p, n);
  uint32_t* evt = SMEM_EVT ? carve<uint32_t>(p, evt_words) : nullptr;
  uint32_t* BM = carve<uint32_t>(p, static_cast<size_t>(nw + 3) * T);  // +3 zero words (dm2_run window)
  // KREG = 0 generator scratch (sized as smem_rows in lp_api.cpp): the
  // displacement list MAP[i * T], or for n <= 256 the displaced bitmap
  // DIS[w * T] followed by the byte position table.
  const bool use_tab = KREG == 0 && !pd.exact && n <= 256;
  uint32_t* MAP = nullptr;
  uint32_t* DIS = nullptr;
  uint8_t* TAB = nullptr;
  if (KREG == 0) {
    const size_t kk = k > 0 ? k : 1;
    size_t gen = 4 * kk * T;
    if (use_tab) gen = max(gen, 4 * static_cast<size_t>(nw) * T + static_cast<size_t>((n + 3) & ~3) * T);
    unsigned char* g = carve<unsigned char>(p, gen);
    MAP = reinterpret_cast<uint32_t*>(g);
    DIS = reinterpret_cast<uint32_t*>(g);
    TAB = g + 4 * static_cast<size_t>(nw) * T;
  }

  for (int i = tid; i < ne; i += T) {
    EntryDesc e = entries[w.e_lo + i];
    e.evt_off -= w.evt_lo;  // cell index relative to the work item's range
    ents[i] = e;
  }
  if (!pd.exact)
    for (int i = tid; i < k; i += T) dc[i] = draws[pd.draw_off + i];
  for (int i = tid; i < n; i += T) h0[i] = 0u;
  for (int i = tid; i < evt_words; i += T) evt[i] = 0u;
  __syncthreads();
  // Depths come in ascending P, so (words per row, walk mode) classes form
  // contiguous runs: one warp lists them once per block, and every scenario
  // dispatches once per run.
  __shared__ int nruns_s;
  if (tid < 32) {
    int cnt = 0;
    for (int b = 0; b < ne; b += 32) {
      const int i = b + tid;
      const int c = i < ne ? depth_class<(KREG > 0)>(ents[i]) : -1;
      const bool start = i < ne && (i == 0 || depth_class<(KREG > 0)>(ents[i - 1]) != c);
      const unsigned m = __ballot_sync(0xffffffffu, start);
      if (start) runs[cnt + __popc(m & ((1u << tid) - 1u))] = make_int2(i, c);
      cnt += __popc(m);
    }
    if (tid == 0) {
      runs[cnt] = make_int2(ne, 0);
      nruns_s = cnt;
    }
  }
  __syncthreads();
  const int nruns = nruns_s;
  uint32_t* evt_base = SMEM_EVT ? evt : evt_g + w.evt_lo;
  uint32_t* BMc = BM + tid;

  constexpr int KS = KREG > 0 ? KREG : 1;
  for (uint64_t t = w.t0 + tid; t < w.t1; t += T) {
    uint32_t s0 = 0;
    uint32_t sl[KS];  // KREG > 0: the sorted slots (padding 0xffffffff)
    for (int i = 0; i < nw + 3; ++i) BMc[i * T] = 0u;
    if (KREG > 0) {
      if (pd.exact) gen_exact_regs<KS>(t, n, k, binom + pd.binom_off, pd.binom_stride, sl);
      else gen_mc_regs<KS>(pd.seed, t, k, dc, sl);
#pragma unroll
      for (int i = 0; i < KS; ++i)
        if (sl[i] != 0xffffffffu) atomicOr(BMc + (sl[i] >> 5) * T, 1u << (sl[i] & 31));
      s0 = sl[0];
    } else if (pd.exact) {
      uint64_t rank = t;
      int c = 0;
      for (int i = 0; i < k; ++i) {
        const int rem = k - i - 1;
        while (true) {
          const uint64_t num = binom_at(binom + pd.binom_off, pd.binom_stride, n - c - 1, rem);
          if (rank < num) break;
          rank -= num;
          ++c;
        }
        if (i == 0) s0 = static_cast<uint32_t>(c);
        BMc[(c >> 5) * T] |= 1u << (c & 31);
        ++c;
      }
    } else if (use_tab) {
      for (int i = 0; i < nw; ++i) DIS[i * T + tid] = 0u;
      s0 = gen_mc_bitmap_tab(pd.seed, t, k, dc, TAB + 4 * tid, DIS + tid, BMc, T);
    } else {
      s0 = gen_mc_bitmap_smem(pd.seed, t, k, dc, MAP + tid, T, BMc, T);
    }
    if (own_h0 && k > 0) atomicAdd(&h0[s0], 1u);

    for (int ri = 0; ri < nruns; ++ri) {
      const int2 r0 = runs[ri];
      const int ei = r0.x, ej = runs[ri + 1].x, cls = r0.y;
      const int W = cls >> 5, mode = cls & 31;
      switch (W) {
        case 1: walk_run<1, SMEM_EVT>(mode, ents, ei, ej, BMc, T, evt_base, sl); break;
        case 2: walk_run<2, SMEM_EVT>(mode, ents, ei, ej, BMc, T, evt_base, sl); break;
        case 3: walk_run<3, SMEM_EVT>(mode, ents, ei, ej, BMc, T, evt_base, sl); break;
        case 4: walk_run<4, SMEM_EVT>(mode, ents, ei, ej, BMc, T, evt_base, sl); break;
        default:
          if (WMAX > 4) {
            switch (W) {
              case 5: walk_run<5, SMEM_EVT>(mode, ents, ei, ej, BMc, T, evt_base, sl); break;
              case 6: walk_run<6, SMEM_EVT>(mode, ents, ei, ej, BMc, T, evt_base, sl); break;
              case 7: walk_run<7, SMEM_EVT>(mode, ents, ei, ej, BMc, T, evt_base, sl); break;
              default: walk_run<8, SMEM_EVT>(mode, ents, ei, ej, BMc, T, evt_base, sl); break;
            }
          }
          break;
      }
    }
  }
  __syncthreads();
  if (own_h0)
    for (int i = tid; i < n; i += T)
      if (h0[i]) atomicAdd(&h0_g[pd.h0_off + i], h0[i]);
  for (int i = tid; i < evt_words; i += T) {
    const uint32_t v = evt[i];
    if (v & 0xffffu) atomicAdd(&evt_g[w.evt_lo + 2 * i], v & 0xffffu);
    if (v >> 16) atomicAdd(&evt_g[w.evt_lo + 2 * i + 1], v >> 16);
  }
}

template <int KREG, int WMAX, bool SM>
static cudaError_t launch_rows_t(int blocks, int threads, size_t smem, cudaStream_t st,
                                 const WorkItem* w, const PairDesc* pairs, const EntryDesc* ents,
                                 const DrawConst* dr, const uint64_t* binom, uint32_t* evt,
                                 uint32_t* h0) {
  auto fn = hist_rows_kernel<KREG, WMAX, SM>;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(fn), smem);
  if (e != cudaSuccess) return e;
  fn<<<blocks, threads, smem, st>>>(w, pairs, ents, dr, binom, evt, h0);
  return cudaGetLastError();
}

// kreg in {0, 16, 32, 64}; wmax in {4, 8}
cudaError_t launch_hist_rows(int kreg, int wmax, bool smem_evt, int blocks, int threads,
                             size_t smem, cudaStream_t st, const WorkItem* w,
                             const PairDesc* pairs, const EntryDesc* ents, const DrawConst* dr,
                             const uint64_t* binom, uint32_t* evt, uint32_t* h0) {
  if (blocks <= 0) return cudaSuccess;
#define LP_W(K, WM)                                                                              \
  if (kreg == K && wmax == WM)                                                                   \
    return smem_evt ? launch_rows_t<K, WM, true>(blocks, threads, smem, st, w, pairs, ents, dr,  \
                                                 binom, evt, h0)                                 \
                    : launch_rows_t<K, WM, false>(blocks, threads, smem, st, w, pairs, ents, dr, \
                                                  binom, evt, h0);
  LP_W(0, 4)
  LP_W(0, 8)
  LP_W(16, 4)
  LP_W(16, 8)
#undef LP_W
  return cudaErrorInvalidValue;
}

// Load the row kernels' code now (lazy module loading would otherwise load
// each on its first launch, inside the first re-plan that uses it).
void preload_rows() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, hist_rows_kernel<0, 4, true>);
  cudaFuncGetAttributes(&a, hist_rows_kernel<0, 4, false>);
  cudaFuncGetAttributes(&a, hist_rows_kernel<16, 4, true>);
  cudaFuncGetAttributes(&a, hist_rows_kernel<0, 8, true>);
}

}  // namespace lp
