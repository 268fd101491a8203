// lp_hist_scn.cu — K1 v2: scenario-major survivor-deficit histograms (sm_100a).
//
// Same threshold-event algorithm as lp_hist.cu (see the header there), laid
// out so that no block-wide barrier sits inside the trial loop:
//
//   * a thread owns one scenario at a time: it draws it (sample_distinct,
//     rng.cpp:8-19, or lexicographic unranking for the exact branch) into its
//     private shared-memory columns — the sorted slot list S and the slot
//     bitmap BM — and then walks every depth P of its work item;
//   * all lanes of a warp walk the same depth at the same time, so the depth's
//     constants are shared-memory broadcasts;
//   * per-thread columns are laid out [row][thread] so every lane hits its own
//     bank (no conflicts);
//   * depths whose configs hold at most one pipeline per class (Dmax == 1)
//     can never lose two slots of one stage: they are skipped entirely (their
//     histogram comes from h0 alone);
//   * depths with Dmax <= kComb count class members with a "comb" of bitmap
//     tests c_j = 1 + sum_{y=1..q_j} BM[s_j - y*P] (no per-class state);
//   * the other (small) depths count classes in stamped u16 counters,
//     (stamp << 8) | count (12-bit counts when k > 255), so nothing is
//     cleared between scenarios.
//
// Events (t >= 2) go to a per-block shared-memory table with RED.ADD and are
// flushed to HBM once per block; t = 1 events are the per-scenario minimum
// slot (h0).
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

template <bool SMEM_EVT>
__device__ __forceinline__ void evt_add(uint32_t* a) {
  if (SMEM_EVT) {
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(a)))
                 : "memory");
  } else {
    atomicAdd(a, 1u);
  }
}

}  // namespace

template <int KREG, bool SMEM_EVT>
__global__ void __launch_bounds__(256, 2) hist_scn_kernel(const WorkItem* __restrict__ work,
                                                       const PairDesc* __restrict__ pairs,
                                                       const EntryDesc* __restrict__ entries,
                                                       const DrawConst* __restrict__ draws,
                                                       const uint64_t* __restrict__ binom,
                                                       uint32_t* __restrict__ evt_g,
                                                       uint32_t* __restrict__ h0_g, int uw) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const WorkItem w = work[blockIdx.x];
  const PairDesc pd = pairs[w.pair];
  const int ne = w.e_res_hi - w.e_lo;  // depths that can produce t >= 2 events
  const int k = pd.k, n = pd.n;
  const int nw = (n + 31) >> 5;
  const bool own_h0 = (w.e_lo == pd.entry_base);

  unsigned char* p = smem;
  EntryDesc* ents = carve<EntryDesc>(p, ne > 0 ? ne : 1);
  DrawConst* dc = carve<DrawConst>(p, k > 0 ? k : 1);
  uint32_t* h0 = carve<uint32_t>(p, n);
  uint32_t* evt = SMEM_EVT ? carve<uint32_t>(p, w.evt_len) : nullptr;
  uint16_t* S = carve<uint16_t>(p, static_cast<size_t>(k > 0 ? k : 1) * T);  // S[j*T + tid]
  uint32_t* BM = carve<uint32_t>(p, static_cast<size_t>(nw) * T);            // BM[w*T + tid]
  uint32_t* U = carve<uint32_t>(p, static_cast<size_t>(uw > 0 ? uw : 1) * T); // map | counters

  for (int i = tid; i < ne; i += T) {
    EntryDesc e = entries[w.e_lo + i];
    if (SMEM_EVT) e.evt_off -= w.evt_lo;
    ents[i] = e;
  }
  if (!pd.exact)
    for (int i = tid; i < k; i += T) dc[i] = draws[pd.draw_off + i];
  for (int i = tid; i < n; i += T) h0[i] = 0u;
  if (SMEM_EVT)
    for (int i = tid; i < w.evt_len; i += T) evt[i] = 0u;
  __syncthreads();
  uint32_t* evt_base = SMEM_EVT ? evt : evt_g;

  uint16_t* Sc = S + tid;
  uint32_t* BMc = BM + tid;
  uint32_t* Uc = U + tid;
  unsigned char* ctr = reinterpret_cast<unsigned char*>(U) + 4 * tid;  // u16 counters, swizzled
  // (stamp << cb) | count: 8-bit counts, or 12-bit when a class can hold
  // more than 255 slots (k > 255; Dmax <= n / 2 <= 1024 then)
  const uint32_t cb = k > 255 ? 12u : 8u, cmask = (1u << cb) - 1u, smax = (1u << (16u - cb)) - 1u;
  uint32_t stamp = smax + 1u;  // forces a clear before first use

  for (uint64_t t = w.t0 + tid; t < w.t1; t += T) {
    // ---- draw scenario t: sorted slots into Sc[j*T], bitmap into BMc[w*T]
    if (KREG > 0 && !pd.exact) {
      uint32_t s[KREG > 0 ? KREG : 1];
      gen_mc_regs<(KREG > 0 ? KREG : 1)>(pd.seed, t, k, dc, s);
      for (int i = 0; i < nw; ++i) BMc[i * T] = 0u;
#pragma unroll
      for (int j = 0; j < (KREG > 0 ? KREG : 1); ++j)
        if (j < k) {
          Sc[j * T] = static_cast<uint16_t>(s[j]);
          BMc[(s[j] >> 5) * T] |= 1u << (s[j] & 31);
        }
    } else if (pd.exact) {
      gen_exact_generic(t, n, k, binom + pd.binom_off, pd.binom_stride, Sc, T);
      for (int i = 0; i < nw; ++i) BMc[i * T] = 0u;
      for (int j = 0; j < k; ++j) {
        const uint32_t v = Sc[j * T];
        BMc[(v >> 5) * T] |= 1u << (v & 31);
      }
    } else {
      gen_mc_generic(pd.seed, t, n, k, dc, Uc, T, BMc, T, Sc, T);
      stamp = smax + 1u;  // the map overwrote the counters
    }
    if (own_h0 && k > 0) atomicAdd(&h0[Sc[0]], 1u);

    // ---- resolve against every depth
    for (int ei = 0; ei < ne; ++ei) {
      const EntryDesc e = ents[ei];
      const uint32_t P = static_cast<uint32_t>(e.P);
      const uint32_t lim = static_cast<uint32_t>(e.lim);
      const int Dm = e.Dmax;
      uint32_t* eb = evt_base + e.evt_off;
      if (P == 1) {  // one class: the (j+1)-th slot is the (j+1)-th member
        for (int j = 1; j < k; ++j) {
          const uint32_t sv = Sc[j * T];
          if (sv >= lim) break;
          evt_add<SMEM_EVT>(eb + (j - 1) * Dm + static_cast<int>(sv));
        }
        continue;
      }
      int mx = 1;
      if (Dm <= kComb) {
        for (int j = 1; j < k; ++j) {
          const uint32_t sv = Sc[j * T];
          if (sv >= lim) break;
          const uint32_t q = div_p(sv, e.magic);
          int c = 1;
          uint32_t x = sv;
          for (uint32_t y = 0; y < q; ++y) {
            x -= P;
            c += (BMc[(x >> 5) * T] >> (x & 31)) & 1u;
          }
          if (c > mx) {
            mx = c;
            evt_add<SMEM_EVT>(eb + (c - 2) * Dm + static_cast<int>(q));
          }
        }
      } else {
        if (++stamp > smax) {
          for (int i = 0; i < uw; ++i) Uc[i * T] = 0u;
          stamp = 1;
        }
        for (int j = 0; j < k; ++j) {
          const uint32_t sv = Sc[j * T];
          if (sv >= lim) break;
          const uint32_t q = div_p(sv, e.magic);
          const uint32_t r = sv - q * P;
          uint16_t* a = reinterpret_cast<uint16_t*>(ctr + ((r >> 1) * T << 2) + ((r & 1) << 1));
          const uint32_t h = *a;
          const uint32_t c = ((h >> cb) == stamp) ? (h & cmask) + 1u : 1u;
          *a = static_cast<uint16_t>((stamp << cb) | c);
          if (static_cast<int>(c) > mx) {
            mx = static_cast<int>(c);
            evt_add<SMEM_EVT>(eb + (mx - 2) * Dm + static_cast<int>(q));
          }
        }
      }
    }
  }
  __syncthreads();
  if (own_h0)
    for (int i = tid; i < n; i += T)
      if (h0[i]) atomicAdd(&h0_g[pd.h0_off + i], h0[i]);
  if (SMEM_EVT)
    for (int i = tid; i < w.evt_len; i += T)
      if (evt[i]) atomicAdd(&evt_g[w.evt_lo + i], evt[i]);
}

template <int KREG, bool SM>
static cudaError_t launch_scn_t(int blocks, int threads, size_t smem, int uw, cudaStream_t st,
                                const WorkItem* w, const PairDesc* pairs, const EntryDesc* ents,
                                const DrawConst* dr, const uint64_t* binom, uint32_t* evt,
                                uint32_t* h0) {
  auto fn = hist_scn_kernel<KREG, SM>;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(fn), smem);
  if (e != cudaSuccess) return e;
  fn<<<blocks, threads, smem, st>>>(w, pairs, ents, dr, binom, evt, h0, uw);
  return cudaGetLastError();
}

cudaError_t launch_hist_scn(int kreg, bool smem_evt, int blocks, int threads, size_t smem, int uw,
                            cudaStream_t st, const WorkItem* w, const PairDesc* pairs,
                            const EntryDesc* ents, const DrawConst* dr, const uint64_t* binom,
                            uint32_t* evt, uint32_t* h0) {
  if (blocks <= 0) return cudaSuccess;
#define LP_S(K)                                                                                   \
  if (kreg == K)                                                                                  \
    return smem_evt ? launch_scn_t<K, true>(blocks, threads, smem, uw, st, w, pairs, ents, dr,   \
                                            binom, evt, h0)                                       \
                    : launch_scn_t<K, false>(blocks, threads, smem, uw, st, w, pairs, ents, dr,  \
                                             binom, evt, h0);
  LP_S(0)
  LP_S(8)
  LP_S(16)
#undef LP_S
  return cudaErrorInvalidValue;
}

}  // namespace lp
