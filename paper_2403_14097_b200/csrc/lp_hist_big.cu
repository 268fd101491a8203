// lp_hist_big.cu — K1 for very large availability counts (2048 < n <= 16384).
//
// The shared-memory kernels keep per-thread scenario state in on-chip
// columns sized by n and k; past n = 2048 those columns no longer fit.  This
// kernel is the same threshold-event resolution with every per-thread array
// in a global scratch slice (L2-resident): the rare huge-cluster case stays
// exact instead of being refused.
//
//   * sample_distinct (rng.cpp:8-19) as a partial Fisher-Yates over a u16
//     position table TAB[n] plus a displaced-position bitmap, O(1) per draw;
//     the selected set lands in a slot bitmap, read back in ascending order;
//   * enumerate_vectors' lexicographic unranking for the exact branch;
//   * per depth P: stamped class counters (stamp << 16 | count, count <=
//     Dmax <= n / 2 < 2^16); when the count of slot s_j's class first
//     exceeds the running maximum, event (t, x = floor(s_j / P)) — the
//     deficit of (D, P) reaches t at D = x + 1;
//   * events and the smallest-slot histogram h0 go straight to global
//     atomics.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lp_device.cuh"
#include "lp_launch.h"
#include "lp_layout.h"

namespace lp {

// Scratch words per thread: TAB (n u16), displaced bitmap and slot bitmap
// (nw each), sorted slots (k u16), class counters (pmax u32).
size_t big_scratch_words(int n, int k, int pmax) {
  const size_t nw = (static_cast<size_t>(n) + 31) / 32;
  return (static_cast<size_t>(n) + 1) / 2 + 2 * nw + (static_cast<size_t>(k) + 1) / 2 + static_cast<size_t>(pmax) + 4;
}

__global__ void __launch_bounds__(64) hist_big_kernel(const WorkItem* __restrict__ work, int n_items,
                                                      const PairDesc* __restrict__ pairs,
                                                      const EntryDesc* __restrict__ entries,
                                                      const DrawConst* __restrict__ draws,
                                                      const uint64_t* __restrict__ binom,
                                                      uint32_t* __restrict__ evt_g, uint32_t* __restrict__ h0_g,
                                                      uint32_t* __restrict__ scratch, size_t per_thread) {
  uint32_t* my = scratch + (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * per_thread;
  for (int wi = blockIdx.x; wi < n_items; wi += gridDim.x) {
    const WorkItem w = work[wi];
    const PairDesc pd = pairs[w.pair];
    const int n = pd.n, k = pd.k;
    const int nw = (n + 31) >> 5;
    const bool own_h0 = (w.e_lo == pd.entry_base);
    uint16_t* TAB = reinterpret_cast<uint16_t*>(my);
    uint32_t* DIS = my + (n + 1) / 2;
    uint32_t* BM = DIS + nw;
    uint16_t* S = reinterpret_cast<uint16_t*>(BM + nw);
    uint32_t* CNT = BM + nw + (k + 1) / 2;
    uint32_t stamp = 0x10000u;  // forces a clear before first use
    int pmax = 1;
    for (int e = w.e_lo; e < w.e_res_hi; ++e) pmax = max(pmax, entries[e].P);
    for (uint64_t t = w.t0 + threadIdx.x; t < w.t1; t += blockDim.x) {
      if (pd.exact) {
        gen_exact_generic(t, n, k, binom + pd.binom_off, pd.binom_stride, S, 1);
      } else {
        for (int i = 0; i < nw; ++i) DIS[i] = BM[i] = 0u;
        uint64_t st = trial_state(pd.seed, t);
        for (int i = 0; i < k; ++i) {
          const uint32_t ui = static_cast<uint32_t>(i);
          const uint32_t j = ui + draw_below(st, draws[pd.draw_off + i]);
          const uint32_t vi = ((DIS[ui >> 5] >> (ui & 31u)) & 1u) ? TAB[ui] : ui;
          const uint32_t vj = ((DIS[j >> 5] >> (j & 31u)) & 1u) ? TAB[j] : j;
          const uint32_t sel = (j == ui) ? vi : vj;
          TAB[j] = static_cast<uint16_t>(vi);  // position j now holds the old pool[i]
          DIS[j >> 5] |= 1u << (j & 31u);
          BM[sel >> 5] |= 1u << (sel & 31u);
        }
        int c = 0;
        for (int i = 0; i < nw; ++i) {
          uint32_t b = BM[i];
          while (b) {
            S[c++] = static_cast<uint16_t>(i * 32 + __ffs(static_cast<int>(b)) - 1);
            b &= b - 1;
          }
        }
      }
      if (own_h0 && k > 0) atomicAdd(&h0_g[pd.h0_off + S[0]], 1u);
      for (int e = w.e_lo; e < w.e_res_hi; ++e) {
        const EntryDesc E = entries[e];
        const uint32_t P = static_cast<uint32_t>(E.P), lim = static_cast<uint32_t>(E.lim);
        uint32_t* eb = evt_g + E.evt_off;
        if (P == 1u) {  // one class: the (j+1)-th slot is its (j+1)-th member
          for (int j = 1; j < k; ++j) {
            const uint32_t sv = S[j];
            if (sv >= lim) break;
            atomicAdd(eb + (j - 1) * E.Dmax + static_cast<int>(sv), 1u);
          }
          continue;
        }
        if (++stamp > 0xffffu) {
          for (int i = 0; i < pmax; ++i) CNT[i] = 0u;
          stamp = 1u;
        }
        uint32_t mx = 1u;
        for (int j = 0; j < k; ++j) {
          const uint32_t sv = S[j];
          if (sv >= lim) break;
          const uint32_t q = div_p(sv, E.magic);
          const uint32_t r = sv - q * P;
          const uint32_t v = CNT[r];
          const uint32_t cnt = ((v >> 16) == stamp) ? (v & 0xffffu) + 1u : 1u;
          CNT[r] = (stamp << 16) | cnt;
          if (cnt > mx) {
            mx = cnt;
            atomicAdd(eb + static_cast<int>(cnt - 2) * E.Dmax + static_cast<int>(q), 1u);
          }
        }
      }
    }
  }
}

cudaError_t launch_hist_big(int n_items, int grid, cudaStream_t st, const WorkItem* w, const PairDesc* pairs,
                            const EntryDesc* ents, const DrawConst* dr, const uint64_t* binom, uint32_t* evt,
                            uint32_t* h0, uint32_t* scratch, size_t per_thread) {
  if (n_items <= 0) return cudaSuccess;
  hist_big_kernel<<<grid, kBigThreads, 0, st>>>(w, n_items, pairs, ents, dr, binom, evt, h0, scratch, per_thread);
  return cudaGetLastError();
}

}  // namespace lp
