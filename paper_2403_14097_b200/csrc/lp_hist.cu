// lp_hist.cu — K1/K1e: survivor-deficit histograms of every (n, k) scenario
// ensemble against every prev config (D, P), on sm_100a.
//
// Replaces Planner::survivor_histogram (optimizer.cpp:64-94) with its callees
// sample_vectors / enumerate_vectors / sample_distinct / stage_survivors
// (preemption.cpp:23-66, rng.cpp:8-19).
//
// Resolution algorithm (threshold events).  For a sorted scenario S and depth
// P, config (D, P) loses d(D) = max_r #{s in S : s % P == r, s < D*P}
// pipelines (m = D - d).  d(D) is a non-decreasing step function of D; it
// reaches t at D = floor(e_t / P) + 1, where e_t is the first element of S
// (in sorted order) that is the t-th member of its residue class.  So per
// (scenario, P) we emit at most one event per t >= 2 into evt[P][t][x =
// floor(e_t/P)], and one event per scenario for t = 1 into h0[min S]
// (e_1 = min S for every P).  Prefix sums over x (finalize kernel) turn
// events into histograms for all D at once: the per-(scenario, config) bin
// update of the reference disappears and the work per scenario is
// O(S(k) + |P| * R(k)) instead of O(|C| * n).
//
// Variant R (k <= 16): a thread owns one scenario in registers and walks all
//   depths of its work item; residue collisions by pairwise compares.
// Variant C (k > 16): a block stages a batch of scenarios in shared memory,
//   a thread owns one depth and counts residue classes in u8 counters.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lp_device.cuh"
#include "lp_launch.h"
#include "lp_layout.h"

namespace lp {

// ---------------------------------------------------------------------------
// shared-memory carve-up helpers
__device__ __forceinline__ size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <typename T>
__device__ __forceinline__ T* carve(unsigned char*& p, size_t count) {
  T* r = reinterpret_cast<T*>(p);
  p += align16(count * sizeof(T));
  return r;
}

// One threshold event.  Shared-memory tables use a fire-and-forget RED.
template <bool SMEM_EVT>
__device__ __forceinline__ void evt_add(uint32_t* a) {
  if (SMEM_EVT) {
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(a)))
                 : "memory");
  } else {
    atomicAdd(a, 1u);
  }
}

// Events of one (scenario, depth) — register variant.
template <int KMAX, bool SMEM_EVT>
__device__ __forceinline__ void resolve_regs(const uint32_t (&s)[KMAX], int k, const EntryDesc& e,
                                             uint32_t* evt) {
  const uint32_t P = static_cast<uint32_t>(e.P);
  const uint32_t lim = static_cast<uint32_t>(e.lim);
  const int Dm = e.Dmax;
  const int off = e.evt_off;
  if (P == 1) {  // one residue class: element j is the (j+1)-th member
#pragma unroll
    for (int j = 1; j < KMAX; ++j) {
      if (j < k && s[j] < lim) {
        evt_add<SMEM_EVT>(evt + off + (j - 1) * Dm + s[j]);
      }
    }
    return;
  }
  uint32_t r[KMAX], q[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    q[j] = div_p(s[j], e.magic);
    r[j] = s[j] - q[j] * P;
  }
  int mx = 1;
#pragma unroll
  for (int j = 1; j < KMAX; ++j) {
    if (j < k && s[j] < lim) {
      int c = 1;
#pragma unroll
      for (int i = 0; i < j; ++i) c += (r[i] == r[j]) ? 1 : 0;
      if (c > mx) {
        mx = c;
        evt_add<SMEM_EVT>(evt + off + (c - 2) * Dm + static_cast<int>(q[j]));
      }
    }
  }
}

template <int KMAX, bool SMEM_EVT>
__global__ void __launch_bounds__(256) hist_regs_kernel(const WorkItem* __restrict__ work,
                                                        const PairDesc* __restrict__ pairs,
                                                        const EntryDesc* __restrict__ entries,
                                                        const DrawConst* __restrict__ draws,
                                                        const uint64_t* __restrict__ binom,
                                                        uint32_t* __restrict__ evt_g,
                                                        uint32_t* __restrict__ h0_g) {
  extern __shared__ __align__(16) unsigned char smem[];
  const WorkItem w = work[blockIdx.x];
  const PairDesc pd = pairs[w.pair];
  const int ne = w.e_res_hi - w.e_lo;  // depths with Dmax >= 2
  const int k = pd.k;
  const bool own_h0 = (w.e_lo == pd.entry_base);

  unsigned char* p = smem;
  EntryDesc* ents = carve<EntryDesc>(p, ne > 0 ? ne : 1);
  DrawConst* dc = carve<DrawConst>(p, KMAX);
  uint32_t* h0 = carve<uint32_t>(p, pd.n);
  uint32_t* evt = SMEM_EVT ? carve<uint32_t>(p, w.evt_len) : nullptr;

  for (int i = threadIdx.x; i < ne; i += blockDim.x) {
    EntryDesc e = entries[w.e_lo + i];
    if (SMEM_EVT) e.evt_off -= w.evt_lo;
    ents[i] = e;
  }
  if (!pd.exact)
    for (int i = threadIdx.x; i < k; i += blockDim.x) dc[i] = draws[pd.draw_off + i];
  for (int i = threadIdx.x; i < pd.n; i += blockDim.x) h0[i] = 0u;
  if (SMEM_EVT)
    for (int i = threadIdx.x; i < w.evt_len; i += blockDim.x) evt[i] = 0u;
  __syncthreads();
  uint32_t* evt_base = SMEM_EVT ? evt : evt_g;

  for (uint64_t t = w.t0 + threadIdx.x; t < w.t1; t += blockDim.x) {
    uint32_t s[KMAX];
    if (pd.exact)
      gen_exact_regs<KMAX>(t, pd.n, k, binom + pd.binom_off, pd.binom_stride, s);
    else
      gen_mc_regs<KMAX>(pd.seed, t, k, dc, s);
    if (own_h0 && k > 0) atomicAdd(&h0[s[0]], 1u);
    for (int ei = 0; ei < ne; ++ei) {
      const EntryDesc e = ents[ei];
      resolve_regs<KMAX, SMEM_EVT>(s, k, e, evt_base);
    }
  }
  __syncthreads();
  if (own_h0)
    for (int i = threadIdx.x; i < pd.n; i += blockDim.x)
      if (h0[i]) atomicAdd(&h0_g[pd.h0_off + i], h0[i]);
  if (SMEM_EVT)
    for (int i = threadIdx.x; i < w.evt_len; i += blockDim.x)
      if (evt[i]) atomicAdd(&evt_g[w.evt_lo + i], evt[i]);
}

// ---------------------------------------------------------------------------
// Variant C: batch of blockDim scenarios in shared memory, depth-major
// resolution with per-thread u8 residue counters (bank-swizzled so the 32
// lanes of a warp always hit 32 distinct banks).
__device__ __forceinline__ uint8_t* ctr_addr(unsigned char* base, int T, int col, uint32_t r) {
  return base + ((((r >> 2) * T) + col) << 2) + (r & 3);
}

template <bool SMEM_EVT>
__global__ void __launch_bounds__(128) hist_ctr_kernel(const WorkItem* __restrict__ work,
                                                       const PairDesc* __restrict__ pairs,
                                                       const EntryDesc* __restrict__ entries,
                                                       const DrawConst* __restrict__ draws,
                                                       const uint64_t* __restrict__ binom,
                                                       uint32_t* __restrict__ evt_g,
                                                       uint32_t* __restrict__ h0_g, int pmax_cap) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const WorkItem w = work[blockIdx.x];
  const PairDesc pd = pairs[w.pair];
  const int ne = w.e_hi - w.e_lo;
  const int k = pd.k, n = pd.n;
  const bool own_h0 = (w.e_lo == pd.entry_base);

  unsigned char* p = smem;
  EntryDesc* ents = carve<EntryDesc>(p, ne);
  DrawConst* dc = carve<DrawConst>(p, k);
  uint32_t* h0 = carve<uint32_t>(p, n);
  uint32_t* evt = SMEM_EVT ? carve<uint32_t>(p, w.evt_len) : nullptr;
  uint16_t* S = carve<uint16_t>(p, static_cast<size_t>(k) * T);  // S[j * T + b]
  // scratch: generation (map [k][T] u32 + bitmap [nw][T] u32) or counters
  unsigned char* scratch = p;
  uint32_t* gmap = reinterpret_cast<uint32_t*>(scratch);
  uint32_t* gbm = gmap + static_cast<size_t>(k) * T;
  unsigned char* ctr = scratch;

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

  // thread -> (entry lane, scenario group)
  const int E2 = ne <= T ? ((ne + 31) & ~31) : T;
  const int G = T / E2;
  const int lane_e = tid % E2;
  const int grp = tid / E2;
  const int ctr_words = (pmax_cap + 3) >> 2;

  for (uint64_t base = w.t0; base < w.t1; base += T) {
    const uint64_t left = w.t1 - base;
    const int nb = left < static_cast<uint64_t>(T) ? static_cast<int>(left) : T;
    // ---- generate one scenario per thread into S[.][tid]
    if (tid < nb) {
      const uint64_t t = base + tid;
      if (pd.exact)
        gen_exact_generic(t, n, k, binom + pd.binom_off, pd.binom_stride, S + tid, T);
      else
        gen_mc_generic(pd.seed, t, n, k, dc, gmap + tid, T, gbm + tid, T, S + tid, T);
      if (own_h0 && k > 0) atomicAdd(&h0[S[tid]], 1u);
    }
    __syncthreads();
    // ---- zero counters (the generation scratch is reused)
    {
      uint32_t* c32 = reinterpret_cast<uint32_t*>(ctr);
      for (int i = tid; i < ctr_words * T; i += T) c32[i] = 0u;
    }
    __syncthreads();
    // ---- resolve: thread owns depth lane_e (+ multiples of T when ne > T)
    for (int ei = lane_e; ei < ne; ei += E2) {
      const EntryDesc e = ents[ei];
      const uint32_t P = static_cast<uint32_t>(e.P);
      const uint32_t lim = static_cast<uint32_t>(e.lim);
      for (int b = grp; b < nb; b += G) {
        int mx = 1, jend = 0;
        for (int j = 0; j < k; ++j) {
          const uint32_t sv = S[j * T + b];
          if (sv >= lim) break;
          const uint32_t q = (P == 1) ? sv : div_p(sv, e.magic);
          const uint32_t r = sv - q * P;
          uint8_t* a = ctr_addr(ctr, T, tid, r);
          const int c = *a + 1;
          *a = static_cast<uint8_t>(c);
          if (c > mx) {
            mx = c;
            evt_add<SMEM_EVT>(evt_base + e.evt_off + (c - 2) * e.Dmax + static_cast<int>(q));
          }
          jend = j + 1;
        }
        for (int j = 0; j < jend; ++j) {  // reset the touched counters
          const uint32_t sv = S[j * T + b];
          const uint32_t q = (P == 1) ? sv : div_p(sv, e.magic);
          *ctr_addr(ctr, T, tid, sv - q * P) = 0;
        }
      }
    }
    __syncthreads();
  }
  if (own_h0)
    for (int i = tid; i < n; i += T)
      if (h0[i]) atomicAdd(&h0_g[pd.h0_off + i], h0[i]);
  if (SMEM_EVT)
    for (int i = tid; i < w.evt_len; i += T)
      if (evt[i]) atomicAdd(&evt_g[w.evt_lo + i], evt[i]);
}

// ---------------------------------------------------------------------------
// h0 -> inclusive prefix (one block per pair), then events -> histograms.
__global__ void h0_scan_kernel(const PairDesc* __restrict__ pairs, uint32_t* __restrict__ h0) {
  const PairDesc pd = pairs[blockIdx.x];
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    uint32_t* h = h0 + pd.h0_off;
    for (int i = 0; i < pd.n; ++i) {
      acc += h[i];
      h[i] = acc;
    }
  }
}

// One block per entry: evt rows -> in-place inclusive prefix over x, then
// hist[D][d] = N_d(D) - N_{d+1}(D) with N_0 = local ensemble size,
// N_1(D) = h0prefix[D*P - 1], N_t(D) = evt_prefix[t][D-1].
__global__ void finalize_kernel(const PairDesc* __restrict__ pairs,
                                const EntryDesc* __restrict__ entries, uint32_t* __restrict__ evt,
                                const uint32_t* __restrict__ h0p, uint32_t* __restrict__ hist) {
  const EntryDesc e = entries[blockIdx.x];
  const PairDesc pd = pairs[e.pair];
  const int k = pd.k;
  const int Dm = e.Dmax;
  uint32_t* ev = evt + e.evt_off;
  for (int t = 2 + threadIdx.x; t <= e.tmax; t += blockDim.x) {
    uint32_t* row = ev + (t - 2) * Dm;
    uint32_t acc = 0;
    for (int x = 0; x < Dm; ++x) {
      acc += row[x];
      row[x] = acc;
    }
  }
  __syncthreads();
  const uint32_t n0 = static_cast<uint32_t>(pd.t_hi - pd.t_lo);
  const uint32_t* h = h0p + pd.h0_off;
  for (int D = 1 + threadIdx.x; D <= Dm; D += blockDim.x) {
    uint32_t* out = hist + e.hist_off + hist_row(D, k);
    const int dmax = min(k, D);
    uint32_t prev = n0;  // N_0
    for (int d = 0; d <= dmax; ++d) {
      uint32_t nxt;  // N_{d+1}(D)
      const int t = d + 1;
      if (t > dmax) nxt = 0;
      else if (t == 1) nxt = h[D * e.P - 1];
      else nxt = (t <= e.tmax) ? ev[(t - 2) * Dm + (D - 1)] : 0u;
      out[d] = prev - nxt;
      prev = nxt;
    }
  }
}

// ---------------------------------------------------------------------------
// Parity dumps (lp_dump_scenarios / lp_dump_survivors): one thread per trial,
// the same generators as the histogram kernels; scratch in global memory.
__global__ void dump_kernel(int n, int k, int exact, int trials, uint64_t seed,
                            const DrawConst* __restrict__ dc, const uint64_t* __restrict__ binom,
                            int binom_stride, uint32_t* __restrict__ gscratch,
                            uint16_t* __restrict__ sorted_out, const int2* __restrict__ cfgs,
                            int n_cfg, uint16_t* __restrict__ m_out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= trials) return;
  const int nw = (n + 31) >> 5;
  uint16_t* srt = sorted_out + static_cast<size_t>(t) * (k > 0 ? k : 1);
  if (k <= 16) {
    uint32_t s[16];
    if (exact) gen_exact_regs<16>(static_cast<uint64_t>(t), n, k, binom, binom_stride, s);
    else gen_mc_regs<16>(seed, static_cast<uint64_t>(t), k, dc, s);
    for (int j = 0; j < k; ++j) srt[j] = static_cast<uint16_t>(s[j]);
  } else {
    uint32_t* map = gscratch + static_cast<size_t>(t) * (k + nw);
    if (exact) gen_exact_generic(static_cast<uint64_t>(t), n, k, binom, binom_stride, srt, 1);
    else gen_mc_generic(seed, static_cast<uint64_t>(t), n, k, dc, map, 1, map + k, 1, srt, 1);
  }
  if (!m_out) return;
  // survivor minimum per config, directly: m = D - max_p #{s < D*P, s % P == p}
  for (int c = 0; c < n_cfg; ++c) {
    const int D = cfgs[c].x, P = cfgs[c].y;
    const int lim = D * P;
    int mx = 0;
    for (int j = 0; j < k; ++j) {
      const int sj = srt[j];
      if (sj >= lim) break;
      int cnt = 1;
      for (int i = 0; i < j; ++i) cnt += (srt[i] % P == sj % P) ? 1 : 0;
      mx = max(mx, cnt);
    }
    m_out[static_cast<size_t>(t) * n_cfg + c] = static_cast<uint16_t>(D - mx);
  }
}

// ---------------------------------------------------------------------------
// launch wrappers (host)
template <int KMAX, bool SM>
static cudaError_t launch_regs(int blocks, size_t smem, cudaStream_t st, const WorkItem* w,
                               const PairDesc* pairs, const EntryDesc* ents, const DrawConst* dr,
                               const uint64_t* binom, uint32_t* evt, uint32_t* h0) {
  auto fn = hist_regs_kernel<KMAX, SM>;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(fn), smem);
  if (e != cudaSuccess) return e;
  fn<<<blocks, 256, smem, st>>>(w, pairs, ents, dr, binom, evt, h0);
  return cudaGetLastError();
}

cudaError_t launch_hist_regs(int kmax, bool smem_evt, int blocks, size_t smem, cudaStream_t st,
                             const WorkItem* w, const PairDesc* pairs, const EntryDesc* ents,
                             const DrawConst* dr, const uint64_t* binom, uint32_t* evt,
                             uint32_t* h0) {
  if (blocks <= 0) return cudaSuccess;
#define LP_R(K)                                                                                  \
  if (kmax == K)                                                                                 \
    return smem_evt ? launch_regs<K, true>(blocks, smem, st, w, pairs, ents, dr, binom, evt, h0) \
                    : launch_regs<K, false>(blocks, smem, st, w, pairs, ents, dr, binom, evt, h0);
  LP_R(4)
  LP_R(8)
  LP_R(16)
#undef LP_R
  return cudaErrorInvalidValue;
}

cudaError_t launch_hist_ctr(bool smem_evt, int blocks, int threads, size_t smem, int pmax_cap,
                            cudaStream_t st, const WorkItem* w, const PairDesc* pairs,
                            const EntryDesc* ents, const DrawConst* dr, const uint64_t* binom,
                            uint32_t* evt, uint32_t* h0) {
  if (blocks <= 0) return cudaSuccess;
  auto fn = smem_evt ? hist_ctr_kernel<true> : hist_ctr_kernel<false>;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(fn), smem);
  if (e != cudaSuccess) return e;
  fn<<<blocks, threads, smem, st>>>(w, pairs, ents, dr, binom, evt, h0, pmax_cap);
  return cudaGetLastError();
}

// Finalize of a stage: pairs [p0, p0 + n_pairs), entries [e0, e0 + n_entries).
// One thread per block of the histogram launches: its WorkItem from the
// span holding it (binary search over the spans' first blocks).
__global__ void expand_work_kernel(const WorkSpan* __restrict__ spans, int n_spans, int n_work,
                                   WorkItem* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_work) return;
  int lo = 0, hi = n_spans - 1;  // last span with first <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (spans[mid].first <= b) lo = mid;
    else hi = mid - 1;
  }
  const WorkSpan sp = spans[lo];
  WorkItem w = sp.w;
  w.t0 = sp.w.t0 + static_cast<uint64_t>(b - sp.first) * sp.chunk;
  w.t1 = min(sp.w.t1, w.t0 + sp.chunk);
  out[b] = w;
}

cudaError_t launch_expand_work(const WorkSpan* spans, int n_spans, int n_work, WorkItem* out, cudaStream_t st) {
  if (n_work <= 0) return cudaSuccess;
  expand_work_kernel<<<(n_work + 255) / 256, 256, 0, st>>>(spans, n_spans, n_work, out);
  return cudaGetLastError();
}

cudaError_t launch_finalize_range(int p0, int n_pairs, int e0, int n_entries, cudaStream_t st,
                                  const PairDesc* pairs, const EntryDesc* ents, uint32_t* evt,
                                  uint32_t* h0, uint32_t* hist) {
  if (n_pairs > 0) {
    h0_scan_kernel<<<n_pairs, 32, 0, st>>>(pairs + p0, h0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (n_entries <= 0) return cudaSuccess;
  finalize_kernel<<<n_entries, 128, 0, st>>>(pairs, ents + e0, evt, h0, hist);
  return cudaGetLastError();
}

cudaError_t launch_finalize(int n_pairs, int n_entries, cudaStream_t st, const PairDesc* pairs,
                            const EntryDesc* ents, uint32_t* evt, uint32_t* h0, uint32_t* hist) {
  if (n_pairs <= 0) return cudaSuccess;
  h0_scan_kernel<<<n_pairs, 32, 0, st>>>(pairs, h0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  finalize_kernel<<<n_entries, 128, 0, st>>>(pairs, ents, evt, h0, hist);
  return cudaGetLastError();
}

cudaError_t launch_dump(int n, int k, int exact, int trials, uint64_t seed, const DrawConst* dc,
                        const uint64_t* binom, int binom_stride, uint32_t* gscratch,
                        uint16_t* sorted_out, const int2* cfgs, int n_cfg, uint16_t* m_out,
                        cudaStream_t st) {
  const int threads = 128;
  const int blocks = (trials + threads - 1) / threads;
  if (blocks <= 0) return cudaSuccess;
  dump_kernel<<<blocks, threads, 0, st>>>(n, k, exact, trials, seed, dc, binom, binom_stride,
                                          gscratch, sorted_out, cfgs, n_cfg, m_out);
  return cudaGetLastError();
}

void preload_hist() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, h0_scan_kernel);
  cudaFuncGetAttributes(&a, finalize_kernel);
  cudaFuncGetAttributes(&a, expand_work_kernel);
}

}  // namespace lp
