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

// Shared-memory event cells are u16 pairs in u32 words (a block handles at
// most 4096 scenarios); global cells are u32.
template <bool SMEM_EVT>
__device__ __forceinline__ void evt_add(uint32_t* base, int idx) {
  if (SMEM_EVT) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(base + (idx >> 1)));
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"((idx & 1) * 0xffffu + 1u) : "memory");
  } else {
    atomicAdd(base + idx, 1u);
  }
}

template <int NG>
struct Masks;
template <>
struct Masks<1> {
  __device__ static void load(const uint32_t* p, uint32_t (&m)[1]) { m[0] = *p; }
};
template <>
struct Masks<2> {
  __device__ static void load(const uint32_t* p, uint32_t (&m)[2]) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    m[0] = v.x;
    m[1] = v.y;
  }
};
template <>
struct Masks<4> {
  __device__ static void load(const uint32_t* p, uint32_t (&m)[4]) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    m[0] = v.x;
    m[1] = v.y;
    m[2] = v.z;
    m[3] = v.w;
  }
};

// Depth info for the event address: {magic, evt_off, Dmax, -}.
template <bool SMEM_EVT>
__device__ __forceinline__ void emit(const uint4& inf, uint32_t tm2, uint32_t sj, uint32_t* eb) {
  const uint32_t x = __umulhi(sj, inf.x);  // floor(s_j / P)
  if (x < inf.z)                           // s_j < lim = P * Dmax
    evt_add<SMEM_EVT>(eb, static_cast<int>(inf.y + tm2 * inf.z + x));
}

}  // namespace

// KMAX: register scenario size (4 or 8); NG: 32-depth groups per pass.
// R and Mx need bits(KMAX - 1) planes.
// Four blocks per SM fit 64 registers; the widest instantiation needs more
// (k <= 8 over 128 depths per pass holds 2 x 12 bit planes and 8 slots).
template <int KMAX, int NG>
constexpr int bits_min_blocks(bool gseq) { return (!gseq && KMAX > 4 && NG >= 2) ? 3 : 4; }

template <int KMAX, int NG, bool SMEM_EVT, bool GSEQ>
__global__ void __launch_bounds__(256, (bits_min_blocks<KMAX, NG>(GSEQ))) hist_bits_kernel(const WorkItem* __restrict__ work,
                                                           const PairDesc* __restrict__ pairs,
                                                           const EntryDesc* __restrict__ entries,
                                                           const DrawConst* __restrict__ draws,
                                                           const uint64_t* __restrict__ binom,
                                                           const uint32_t* __restrict__ dmask,
                                                           uint32_t* __restrict__ evt_g,
                                                           uint32_t* __restrict__ h0_g) {
  constexpr int B = KMAX <= 4 ? 2 : 3;
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = blockDim.x;
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
  uint4* info = carve<uint4>(p, nbits > 0 ? nbits : 1);
  DrawConst* dc = carve<DrawConst>(p, KMAX);
  uint32_t* h0 = carve<uint32_t>(p, n);
  uint32_t* evt = SMEM_EVT ? carve<uint32_t>(p, (w.evt_len + 1) / 2) : nullptr;
  uint32_t* dm = carve<uint32_t>(p, static_cast<size_t>(npass) * n * NG);
  uint32_t* scol = GSEQ ? carve<uint32_t>(p, static_cast<size_t>(KMAX) * T) + tid : nullptr;  // sorted slots

  const int evt_rel = SMEM_EVT ? w.evt_lo : 0;
  for (int i = tid; i < nbits; i += T) {
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (i < ne) {
      const EntryDesc e = entries[eb0 + i];
      v = make_uint4(e.magic, static_cast<uint32_t>(e.evt_off - evt_rel), static_cast<uint32_t>(e.Dmax), 0u);
    }
    info[i] = v;
  }
  if (!pd.exact)
    for (int i = tid; i < k; i += T) dc[i] = draws[pd.draw_off + i];
  for (int i = tid; i < n; i += T) h0[i] = 0u;
  if (SMEM_EVT)
    for (int i = tid; i < (w.evt_len + 1) / 2; i += T) evt[i] = 0u;
  {
    const uint4* src = reinterpret_cast<const uint4*>(dmask + w.dtab_off);
    uint4* dst = reinterpret_cast<uint4*>(dm);
    const int nv = (npass * n * NG + 3) / 4;
    for (int i = tid; i < nv; i += T) dst[i] = src[i];
  }
  int p1_off = 0, p1_dmax = 0;
  if (has_p1) {
    const EntryDesc e = entries[w.e_lo];
    p1_off = e.evt_off - evt_rel;
    p1_dmax = e.Dmax;
  }
  __syncthreads();
  uint32_t* eb = SMEM_EVT ? evt : evt_g;

  for (uint64_t t = w.t0 + tid; t < w.t1; t += T) {
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
          evt_add<SMEM_EVT>(eb, p1_off + (j - 1) * p1_dmax + static_cast<int>(s[j]));
    }
    if (GSEQ) {
      // group-sequential: one 32-depth group at a time (9 live planes), the
      // t = 2 events of the whole scenario emitted after the last row from
      // the row-of-first-collision planes J (one loop per group instead of
      // one per row and group); t >= 3 events (rare) are emitted per row.
#pragma unroll
      for (int j = 0; j < KMAX; ++j) scol[j * T] = s[j];
      for (int ps = 0; ps < npass; ++ps) {
        const uint32_t* D = dm + static_cast<size_t>(ps) * n * NG;
        const uint4* I = info + ps * 32 * NG;
#pragma unroll 1
        for (int g = 0; g < NG; ++g) {
          uint32_t M[B], J[3];
#pragma unroll
          for (int b = 0; b < B; ++b) M[b] = 0u;
          J[0] = J[1] = J[2] = 0u;
#pragma unroll
          for (int j = 1; j < KMAX; ++j) {
            if (j >= k) break;
            const uint32_t sj = s[j];
            uint32_t R[B];
#pragma unroll
            for (int b = 0; b < B; ++b) R[b] = 0u;
#pragma unroll
            for (int i = 0; i < j; ++i) {
              const uint32_t m = D[(sj - s[i]) * NG + g];
              const uint32_t c0 = R[0] & m;
              R[0] ^= m;
              if (B == 3) R[2] |= R[1] & c0;
              R[1] ^= c0;
            }
            uint32_t gt, eq;
            if (B == 3) {
              gt = R[2] & ~M[2];
              eq = ~(R[2] ^ M[2]);
              gt |= eq & R[1] & ~M[1];
              eq &= ~(R[1] ^ M[1]);
            } else {
              gt = R[1] & ~M[1];
              eq = ~(R[1] ^ M[1]);
            }
            gt |= eq & R[0] & ~M[0];
#pragma unroll
            for (int b = 0; b < B; ++b) M[b] = (gt & R[b]) | (~gt & M[b]);
            uint32_t hi = R[1];
            if (B == 3) hi |= R[2];
            const uint32_t e2 = gt & ~hi;  // first collision: t = 2 at row j
            if (j & 1) J[0] |= e2;
            if (j & 2) J[1] |= e2;
            if (j & 4) J[2] |= e2;
            uint32_t e3 = gt & hi;
            while (e3) {
              const int b = __ffs(static_cast<int>(e3)) - 1;
              e3 &= e3 - 1;
              uint32_t r = ((R[0] >> b) & 1u) | (((R[1] >> b) & 1u) << 1);
              if (B == 3) r |= ((R[2] >> b) & 1u) << 2;
              emit<SMEM_EVT>(I[g * 32 + b], r - 1u, sj, eb);
            }
          }
          uint32_t seen = M[0] | M[1];
          if (B == 3) seen |= M[2];
          while (seen) {
            const int b = __ffs(static_cast<int>(seen)) - 1;
            seen &= seen - 1;
            const uint32_t jj = ((J[0] >> b) & 1u) | (((J[1] >> b) & 1u) << 1) | (((J[2] >> b) & 1u) << 2);
            emit<SMEM_EVT>(I[g * 32 + b], 0u, scol[jj * T], eb);
          }
        }
      }
      continue;
    }
    for (int ps = 0; ps < npass; ++ps) {
      const uint32_t* D = dm + static_cast<size_t>(ps) * n * NG;
      const uint4* I = info + ps * 32 * NG;
      uint32_t M[B][NG];  // running maximum of R over the rows so far
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int g = 0; g < NG; ++g) M[b][g] = 0u;
#pragma unroll
      for (int j = 1; j < KMAX; ++j) {
        if (j >= k) break;
        const uint32_t sj = s[j];
        uint32_t R[B][NG];
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
          for (int g = 0; g < NG; ++g) R[b][g] = 0u;
#pragma unroll
        for (int i = 0; i < j; ++i) {
          uint32_t m[NG];
          Masks<NG>::load(D + (sj - s[i]) * NG, m);
#pragma unroll
          for (int g = 0; g < NG; ++g) {  // R += m, bit-sliced (R <= j <= KMAX - 1)
            const uint32_t c0 = R[0][g] & m[g];
            R[0][g] ^= m[g];
            if (B == 3) R[2][g] |= R[1][g] & c0;
            R[1][g] ^= c0;
          }
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          // gt = R > M (per bit), then M = max(M, R)
          uint32_t gt, eq;
          if (B == 3) {
            gt = R[2][g] & ~M[2][g];
            eq = ~(R[2][g] ^ M[2][g]);
            gt |= eq & R[1][g] & ~M[1][g];
            eq &= ~(R[1][g] ^ M[1][g]);
          } else {
            gt = R[1][g] & ~M[1][g];
            eq = ~(R[1][g] ^ M[1][g]);
          }
          gt |= eq & R[0][g] & ~M[0][g];
#pragma unroll
          for (int b = 0; b < B; ++b) M[b][g] = (gt & R[b][g]) | (~gt & M[b][g]);
          // t = R + 1: t == 2 is the common case (first collision of the depth)
          uint32_t hi = R[1][g];
          if (B == 3) hi |= R[2][g];
          uint32_t e2 = gt & ~hi;
          uint32_t e3 = gt & hi;
          while (e2) {
            const int b = __ffs(static_cast<int>(e2)) - 1;
            e2 &= e2 - 1;
            emit<SMEM_EVT>(I[g * 32 + b], 0u, sj, eb);
          }
          while (e3) {
            const int b = __ffs(static_cast<int>(e3)) - 1;
            e3 &= e3 - 1;
            uint32_t r = ((R[0][g] >> b) & 1u) | (((R[1][g] >> b) & 1u) << 1);
            if (B == 3) r |= ((R[2][g] >> b) & 1u) << 2;
            emit<SMEM_EVT>(I[g * 32 + b], r - 1u, sj, eb);
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
    for (int i = tid; i < (w.evt_len + 1) / 2; i += T) {
      const uint32_t v = evt[i];
      if (v & 0xffffu) atomicAdd(&evt_g[w.evt_lo + 2 * i], v & 0xffffu);
      if (v >> 16) atomicAdd(&evt_g[w.evt_lo + 2 * i + 1], v >> 16);
    }
}

template <int KMAX, int NG, bool SM, bool GSEQ>
static cudaError_t launch_bits_t(int blocks, int threads, size_t smem, cudaStream_t st,
                                 const WorkItem* w, const PairDesc* pairs, const EntryDesc* ents,
                                 const DrawConst* dr, const uint64_t* binom, const uint32_t* dmask,
                                 uint32_t* evt, uint32_t* h0) {
  auto fn = hist_bits_kernel<KMAX, NG, SM, GSEQ>;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(fn), smem);
  if (e != cudaSuccess) return e;
  fn<<<blocks, threads, smem, st>>>(w, pairs, ents, dr, binom, dmask, evt, h0);
  return cudaGetLastError();
}

cudaError_t launch_hist_bits(int kmax, int ng, bool smem_evt, bool gseq, int blocks, int threads,
                             size_t smem, cudaStream_t st, const WorkItem* w, const PairDesc* pairs,
                             const EntryDesc* ents, const DrawConst* dr, const uint64_t* binom,
                             const uint32_t* dmask, uint32_t* evt, uint32_t* h0) {
  if (blocks <= 0) return cudaSuccess;
#define LP_B(K, G)                                                                                   \
  if (kmax == K && ng == G) {                                                                        \
    if (gseq)                                                                                        \
      return smem_evt ? launch_bits_t<K, G, true, true>(blocks, threads, smem, st, w, pairs, ents, dr, \
                                                        binom, dmask, evt, h0)                       \
                      : launch_bits_t<K, G, false, true>(blocks, threads, smem, st, w, pairs, ents,  \
                                                         dr, binom, dmask, evt, h0);                 \
    return smem_evt ? launch_bits_t<K, G, true, false>(blocks, threads, smem, st, w, pairs, ents, dr,  \
                                                       binom, dmask, evt, h0)                        \
                    : launch_bits_t<K, G, false, false>(blocks, threads, smem, st, w, pairs, ents, dr, \
                                                        binom, dmask, evt, h0);                      \
  }
  LP_B(4, 1)
  LP_B(4, 2)
  LP_B(4, 4)
  LP_B(8, 1)
  LP_B(8, 2)
  LP_B(8, 4)
#undef LP_B
  return cudaErrorInvalidValue;
}

}  // namespace lp
