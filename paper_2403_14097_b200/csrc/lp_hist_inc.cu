// lp_hist_inc.cu — K1 v3 for k <= 16: sparse "incidence" resolution (sm_100a).
//
// Two preempted slots s_i < s_j sit in the same stage of every config of
// depth P exactly when P divides d = s_j - s_i.  Instead of visiting every
// (slot, depth) pair, each thread enumerates its scenario's k(k-1)/2
// differences and reads the depths dividing d from a per-ensemble divisor
// table (CSR in shared memory).  Only those (j, P) "incidences" can raise a
// residue-class count above 1, so they carry all t >= 2 threshold events.
//
// Per (thread, depth) a 16-bit state tracks the scan in slot order:
//   [0:4) M-1   running maximum class count before the current row
//   [4:8) cnt   incidences of depth P seen in row j (= earlier class members)
//   [8:12) row  the row j cnt belongs to
//   [12:16) stamp  scenario tag (lazy reset; the column is cleared every 15)
// Row j of depth P has c_j = 1 + #{i < j : P | s_j - s_i}; the count crosses
// the running maximum at most once per row, which is exactly the event
// (t = c_j, x = floor(s_j / P)) of the dense algorithm (lp_hist.cu).
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

template <int KMAX, bool SMEM_EVT>
__global__ void __launch_bounds__(256, 2) hist_inc_kernel(const WorkItem* __restrict__ work,
                                                          const PairDesc* __restrict__ pairs,
                                                          const EntryDesc* __restrict__ entries,
                                                          const DrawConst* __restrict__ draws,
                                                          const uint64_t* __restrict__ binom,
                                                          const uint16_t* __restrict__ divtab,
                                                          uint32_t* __restrict__ evt_g,
                                                          uint32_t* __restrict__ h0_g) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const WorkItem w = work[blockIdx.x];
  const PairDesc pd = pairs[w.pair];
  const int ne = w.e_res_hi - w.e_lo;
  const int k = pd.k, n = pd.n;
  const bool own_h0 = (w.e_lo == pd.entry_base);

  unsigned char* p = smem;
  EntryDesc* ents = carve<EntryDesc>(p, ne > 0 ? ne : 1);
  DrawConst* dc = carve<DrawConst>(p, KMAX);
  uint32_t* h0 = carve<uint32_t>(p, n);
  uint32_t* evt = SMEM_EVT ? carve<uint32_t>(p, w.evt_len) : nullptr;
  uint16_t* dt = carve<uint16_t>(p, w.dtab_len > 0 ? w.dtab_len : 1);  // [n+1 offsets][list]
  uint32_t* st32 = carve<uint32_t>(p, static_cast<size_t>((ne + 1) / 2) * T);

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
  for (int i = tid; i < w.dtab_len; i += T) dt[i] = divtab[w.dtab_off + i];
  __syncthreads();
  uint32_t* evt_base = SMEM_EVT ? evt : evt_g;
  const uint16_t* doff = dt;
  const uint16_t* dlist = dt + (n + 1);
  const bool has_p1 = ne > 0 && ents[0].P == 1;
  // state column: u16 per depth, two depths per 32-bit word [e/2][T]
  unsigned char* stc = reinterpret_cast<unsigned char*>(st32) + 4 * tid;
  const int sw = (ne + 1) / 2;
  uint32_t stamp = 16;

  for (uint64_t t = w.t0 + tid; t < w.t1; t += T) {
    uint32_t s[KMAX];
    if (pd.exact)
      gen_exact_regs<KMAX>(t, n, k, binom + pd.binom_off, pd.binom_stride, s);
    else
      gen_mc_regs<KMAX>(pd.seed, t, k, dc, s);
    if (own_h0 && k > 0) atomicAdd(&h0[s[0]], 1u);
    if (++stamp > 15u) {
      for (int i = 0; i < sw; ++i) st32[i * T + tid] = 0u;
      stamp = 1;
    }
    if (has_p1) {  // depth 1: every slot is in the single class
      const EntryDesc& e = ents[0];
#pragma unroll
      for (int j = 1; j < KMAX; ++j)
        if (j < k && s[j] < static_cast<uint32_t>(e.lim))
          evt_add<SMEM_EVT>(evt_base + e.evt_off + (j - 1) * e.Dmax + static_cast<int>(s[j]));
    }
#pragma unroll
    for (int j = 1; j < KMAX; ++j) {
      if (j >= k) break;
      const uint32_t sj = s[j];
#pragma unroll
      for (int i = 0; i < j; ++i) {
        const uint32_t d = sj - s[i];
        const int a = doff[d], b = doff[d + 1];
        for (int q = a; q < b; ++q) {
          const int e = dlist[q];
          uint16_t* sp = reinterpret_cast<uint16_t*>(stc + ((e >> 1) * T << 2) + ((e & 1) << 1));
          uint32_t v = *sp;
          if ((v >> 12) != stamp) v = stamp << 12;
          const uint32_t mm1 = v & 15u;
          const uint32_t cnt = (((v >> 8) & 15u) == static_cast<uint32_t>(j) ? ((v >> 4) & 15u) : 0u) + 1u;
          uint32_t nm = mm1;
          if (cnt > mm1) {  // c = cnt + 1 exceeds the running maximum M = mm1 + 1
            nm = cnt;
            const EntryDesc& E = ents[e];
            if (sj < static_cast<uint32_t>(E.lim)) {
              const uint32_t x = div_p(sj, E.magic);
              evt_add<SMEM_EVT>(evt_base + E.evt_off + (cnt - 1) * E.Dmax + static_cast<int>(x));
            }
          }
          *sp = static_cast<uint16_t>((stamp << 12) | (static_cast<uint32_t>(j) << 8) | (cnt << 4) | nm);
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

template <int KMAX, bool SM>
static cudaError_t launch_inc_t(int blocks, int threads, size_t smem, cudaStream_t st,
                                const WorkItem* w, const PairDesc* pairs, const EntryDesc* ents,
                                const DrawConst* dr, const uint64_t* binom, const uint16_t* divtab,
                                uint32_t* evt, uint32_t* h0) {
  auto fn = hist_inc_kernel<KMAX, SM>;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(fn), smem);
  if (e != cudaSuccess) return e;
  fn<<<blocks, threads, smem, st>>>(w, pairs, ents, dr, binom, divtab, evt, h0);
  return cudaGetLastError();
}

cudaError_t launch_hist_inc(int kmax, bool smem_evt, int blocks, int threads, size_t smem,
                            cudaStream_t st, const WorkItem* w, const PairDesc* pairs,
                            const EntryDesc* ents, const DrawConst* dr, const uint64_t* binom,
                            const uint16_t* divtab, uint32_t* evt, uint32_t* h0) {
  if (blocks <= 0) return cudaSuccess;
#define LP_I(K)                                                                                     \
  if (kmax == K)                                                                                    \
    return smem_evt ? launch_inc_t<K, true>(blocks, threads, smem, st, w, pairs, ents, dr, binom,   \
                                            divtab, evt, h0)                                        \
                    : launch_inc_t<K, false>(blocks, threads, smem, st, w, pairs, ents, dr, binom,  \
                                             divtab, evt, h0);
  LP_I(4)
  LP_I(8)
  LP_I(16)
#undef LP_I
  return cudaErrorInvalidValue;
}

}  // namespace lp
