// lp_hist_bits.cu — K1 v5 for k <= 8: bit-parallel incidence resolution (sm_100a).
//
// Two preempted slots s_i < s_j share a stage of every depth-P config exactly
// when P divides d = s_j - s_i.  A host table gives, for every difference d,
// the 32-bit masks of the resolution depths dividing it (NG groups of 32
// depths per pass, one LDS.32/.64/.128 per slot pair).  Row j of the sorted
// scenario then has, for all 32*NG depths at once,
//
//   R_j = #{i < j : P | s_j - s_i} = c_j - 1      (bit-sliced adds, 4 LOP3 each)
//
// and the reference's stage_survivors / min (optimizer.cpp:76-82) reduce to
// threshold events: depth P emits (t = c_j, x = floor(s_j / P)) whenever c_j
// exceeds the running maximum of the earlier rows (bit-sliced compare with
// the planes Mx = max c - 1), because the deficit of (D, P) reaches t at
// D = x + 1.  Every lane runs the same rows, pairs and
// plane operations — no data-dependent loop but the event emission itself —
// and there is no per-(thread, depth) state in shared memory, so four
// 256-thread blocks fit an SM (the incidence kernel of lp_hist_inc.cu kept a
// u16 per thread and depth, ran 12 of 32 lanes and 3.7 warps per scheduler).
//
// Groups of 32 depths are resolved one after the other (9 live planes), and
// the t = 2 events — the first collision of each depth, 90% of all events —
// are emitted after the last row from three planes J holding the row of the
// first collision: one data-dependent loop per group instead of one per row
// and group (measured: 0.77 against 0.87 ms for the forecast-like re-plan).
#include <cuda_runtime.h>
#include <stdint.h>

#include "lp_device.cuh"
#include "lp_launch.h"
#include "lp_layout.h"

namespace lp {
namespace {

constexpr int kT = 256;  // threads per block (the host launches exactly this)

__device__ __forceinline__ size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

template <typename T>
__device__ __forceinline__ T* carve(unsigned char*& p, size_t count) {
  T* r = reinterpret_cast<T*>(p);
  p += a16(count * sizeof(T));
  return r;
}

// Event of depth info {magic, (evt_off << 12) | Dmax} at slot s_j, level t:
// cell evt_off + (t - 2) * Dmax + floor(s_j / P) when floor(s_j / P) < Dmax
// (s_j below lim = P * Dmax); otherwise the add goes to the block's spare
// cell `sink` (never flushed), so the emission loop has no branch.
template <bool SMEM_EVT>
__device__ __forceinline__ void emit(uint2 inf, uint32_t tm2, uint32_t sj, uint32_t* eb, uint32_t sink) {
  const uint32_t x = __umulhi(sj, inf.x);
  const uint32_t dmax = inf.y & 0xfffu;
  const uint32_t cell = (inf.y >> 12) + tm2 * dmax + x;
  if (SMEM_EVT) {
    atomicAdd(eb + (x < dmax ? cell : sink), 1u);
  } else if (x < dmax) {
    atomicAdd(eb + cell, 1u);
  }
}

}  // namespace

// KMAX: register scenario size (4, 8 or 16); NG: depth groups per divisor-table
// word (1: the table is [group][d]).  R and Mx need bits(KMAX - 1) planes.
template <int KMAX, int NG, bool SMEM_EVT>
__global__ void __launch_bounds__(kT, (KMAX > 8 ? 3 : 4)) hist_bits_kernel(const WorkItem* __restrict__ work,
                                                          const PairDesc* __restrict__ pairs,
                                                          const EntryDesc* __restrict__ entries,
                                                          const DrawConst* __restrict__ draws,
                                                          const uint64_t* __restrict__ binom,
                                                          const uint32_t* __restrict__ dmask,
                                                          uint32_t* __restrict__ evt_g,
                                                          uint32_t* __restrict__ h0_g) {
  constexpr int B = KMAX <= 4 ? 2 : (KMAX <= 8 ? 3 : 4);  // bits of KMAX - 1
  constexpr int TD = KMAX <= 4 ? 2 : 3;  // levels t <= TD emitted after the rows
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x;
  const WorkItem w = work[blockIdx.x];
  const PairDesc pd = pairs[w.pair];
  const int k = pd.k, n = pd.n;
  const bool own_h0 = (w.e_lo == pd.entry_base);
  // entries [e_lo, e_res_hi) emit t >= 2 events; a depth-1 entry sorts first
  // and is resolved by rule (every slot is in its single class)
  const bool has_p1 = w.e_res_hi > w.e_lo && entries[w.e_lo].P == 1;
  const int eb0 = w.e_lo + (has_p1 ? 1 : 0);
  const int ne = w.e_res_hi - eb0;
  const int npass = w.dtab_len;
  const int nbits = npass * 32 * NG;

  unsigned char* p = smem;
  uint2* info = carve<uint2>(p, nbits > 0 ? nbits : 1);
  DrawConst* dc = carve<DrawConst>(p, KMAX);
  uint32_t* h0 = carve<uint32_t>(p, n);
  uint32_t* evt = SMEM_EVT ? carve<uint32_t>(p, w.evt_len + 1) : nullptr;  // + sink
  uint32_t* dm = carve<uint32_t>(p, static_cast<size_t>(npass) * n * NG);
  uint32_t* scol = carve<uint32_t>(p, static_cast<size_t>(KMAX) * kT) + tid;  // sorted slots

  for (int i = tid; i < nbits; i += kT) {
    uint2 v = make_uint2(0u, 0u);
    if (i < ne) {
      const EntryDesc e = entries[eb0 + i];
      v = make_uint2(e.magic, (static_cast<uint32_t>(e.evt_off - w.evt_lo) << 12) | static_cast<uint32_t>(e.Dmax));
    }
    info[i] = v;
  }
  if (!pd.exact)
    for (int i = tid; i < k; i += kT) dc[i] = draws[pd.draw_off + i];
  for (int i = tid; i < n; i += kT) h0[i] = 0u;
  if (SMEM_EVT)
    for (int i = tid; i < w.evt_len; i += kT) evt[i] = 0u;
  {
    const uint4* src = reinterpret_cast<const uint4*>(dmask + w.dtab_off);
    uint4* dst = reinterpret_cast<uint4*>(dm);
    const int nv = (npass * n * NG + 3) / 4;
    for (int i = tid; i < nv; i += kT) dst[i] = src[i];
  }
  int p1_off = 0, p1_dmax = 0;
  if (has_p1) {
    const EntryDesc e = entries[w.e_lo];
    p1_off = e.evt_off - w.evt_lo;
    p1_dmax = e.Dmax;
  }
  __syncthreads();
  uint32_t* eb = SMEM_EVT ? evt : evt_g + w.evt_lo;
  const uint32_t sink = static_cast<uint32_t>(w.evt_len);

  for (uint64_t t = w.t0 + tid; t < w.t1; t += kT) {
    uint32_t s[KMAX];
    if (pd.exact)
      gen_exact_regs<KMAX>(t, n, k, binom + pd.binom_off, pd.binom_stride, s);
    else
      gen_mc_regs<KMAX>(pd.seed, t, k, dc, s);
    if (own_h0 && k > 0) atomicAdd(&h0[s[0]], 1u);
    if (has_p1) {  // depth 1: slot j is the (j+1)-th member of the one class
#pragma unroll
      for (int j = 1; j < KMAX; ++j)
        if (j < k && s[j] < static_cast<uint32_t>(p1_dmax))
          atomicAdd(eb + p1_off + (j - 1) * p1_dmax + static_cast<int>(s[j]), 1u);
    }
#pragma unroll
    for (int j = 0; j < KMAX; ++j) scol[j * kT] = s[j];
    for (int ps = 0; ps < npass; ++ps) {
      const uint32_t* D = dm + static_cast<size_t>(ps) * n * NG;
#pragma unroll 1
      for (int g = 0; g < NG; ++g) {
        const uint2* I = info + (ps * NG + g) * 32;
        // J[t-2]: the row at which each depth reached level t (t = 2 .. TD),
        // emitted after the last row; levels above TD (rare) inline
        uint32_t M[B], J[TD - 1][B];
#pragma unroll
        for (int q = 0; q < B; ++q) {
          M[q] = 0u;
#pragma unroll
          for (int l = 0; l < TD - 1; ++l) J[l][q] = 0u;
        }
#pragma unroll
        for (int j = 1; j < KMAX; ++j) {
          if (j >= k) break;
          const uint32_t sj = s[j];
          uint32_t R[B];
#pragma unroll
          for (int q = 0; q < B; ++q) R[q] = 0u;
#pragma unroll
          for (int i = 0; i < j; ++i) {  // R += divisor mask of s_j - s_i, bit-sliced
            uint32_t c = D[(sj - s[i]) * NG + g];
#pragma unroll
            for (int q = 0; q < B - 1; ++q) {
              const uint32_t nc = R[q] & c;
              R[q] ^= c;
              c = nc;
            }
            R[B - 1] |= c;  // R <= j <= KMAX - 1 never overflows B bits
          }
          // gt = R > M (per bit, most significant plane first), M = max(M, R)
          uint32_t gt = 0u, eq = ~0u;
#pragma unroll
          for (int q = B - 1; q >= 0; --q) {
            gt |= eq & R[q] & ~M[q];
            eq &= ~(R[q] ^ M[q]);
          }
#pragma unroll
          for (int q = 0; q < B; ++q) M[q] = (gt & R[q]) | (~gt & M[q]);
          // an event has R = M_old + 1 = t - 1: record its row per level
          uint32_t rest = gt;
#pragma unroll
          for (int l = 0; l < TD - 1; ++l) {
            uint32_t at = rest;  // R == l + 1
#pragma unroll
            for (int q = 0; q < B; ++q) at &= (((l + 1) >> q) & 1) ? R[q] : ~R[q];
            rest &= ~at;
#pragma unroll
            for (int q = 0; q < B; ++q)
              if ((j >> q) & 1) J[l][q] |= at;
          }
          while (rest) {  // t = R + 1 > TD
            const int b = __ffs(static_cast<int>(rest)) - 1;
            rest &= rest - 1;
            uint32_t r = 0u;
#pragma unroll
            for (int q = 0; q < B; ++q) r |= ((R[q] >> b) & 1u) << q;
            emit<SMEM_EVT>(I[b], r - 1u, sj, eb, sink);
          }
        }
        // depths that reached level t: final M >= t - 1
#pragma unroll
        for (int l = 0; l < TD - 1; ++l) {
          uint32_t reached = 0u, eqv = ~0u;  // M > l  (M >= l + 1)
#pragma unroll
          for (int q = B - 1; q >= 0; --q) {
            const uint32_t lb = ((l >> q) & 1) ? ~0u : 0u;
            reached |= eqv & M[q] & ~lb;
            eqv &= ~(M[q] ^ lb);
          }
          while (reached) {
            const int b = __ffs(static_cast<int>(reached)) - 1;
            reached &= reached - 1;
            uint32_t jj = 0u;
#pragma unroll
            for (int q = 0; q < B; ++q) jj |= ((J[l][q] >> b) & 1u) << q;
            emit<SMEM_EVT>(I[b], static_cast<uint32_t>(l), scol[jj * kT], eb, sink);
          }
        }
      }
    }
  }
  __syncthreads();
  if (own_h0)
    for (int i = tid; i < n; i += kT)
      if (h0[i]) atomicAdd(&h0_g[pd.h0_off + i], h0[i]);
  if (SMEM_EVT)
    for (int i = tid; i < w.evt_len; i += kT)
      if (evt[i]) atomicAdd(&evt_g[w.evt_lo + i], evt[i]);
}

template <int KMAX, int NG, bool SM>
static cudaError_t launch_bits_t(int blocks, size_t smem, cudaStream_t st, const WorkItem* w,
                                 const PairDesc* pairs, const EntryDesc* ents, const DrawConst* dr,
                                 const uint64_t* binom, const uint32_t* dmask, uint32_t* evt,
                                 uint32_t* h0) {
  auto fn = hist_bits_kernel<KMAX, NG, SM>;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(fn), smem);
  if (e != cudaSuccess) return e;
  fn<<<blocks, kT, smem, st>>>(w, pairs, ents, dr, binom, dmask, evt, h0);
  return cudaGetLastError();
}

cudaError_t launch_hist_bits(int kmax, bool smem_evt, int blocks, int threads, size_t smem,
                             cudaStream_t st, const WorkItem* w, const PairDesc* pairs,
                             const EntryDesc* ents, const DrawConst* dr, const uint64_t* binom,
                             const uint32_t* dmask, uint32_t* evt, uint32_t* h0) {
  if (blocks <= 0) return cudaSuccess;
  if (threads != kT) return cudaErrorInvalidValue;
#define LP_B(K)                                                                                   \
  if (kmax == K)                                                                                  \
    return smem_evt ? launch_bits_t<K, 1, true>(blocks, smem, st, w, pairs, ents, dr, binom, dmask, \
                                                evt, h0)                                          \
                    : launch_bits_t<K, 1, false>(blocks, smem, st, w, pairs, ents, dr, binom,     \
                                                 dmask, evt, h0);
  LP_B(4)
  LP_B(8)
  LP_B(16)
#undef LP_B
  return cudaErrorInvalidValue;
}

void preload_bits() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, hist_bits_kernel<16, 1, true>);
  cudaFuncGetAttributes(&a, hist_bits_kernel<8, 1, true>);
  cudaFuncGetAttributes(&a, hist_bits_kernel<4, 1, true>);
  cudaFuncGetAttributes(&a, hist_bits_kernel<16, 1, false>);
  cudaFuncGetAttributes(&a, hist_bits_kernel<8, 1, false>);
  cudaFuncGetAttributes(&a, hist_bits_kernel<4, 1, false>);
}

}  // namespace lp
