// lp_dp.cu — K2/K3/K4: transition value phi, the lookahead max-plus DP and
// the on-device traceback (sm_100a, FP64).
//
// Replaces Planner::phi_uncached (optimizer.cpp:96-138) with
// transition_outcome_min / resume_cost (migration.cpp:49-104), the level loop
// of Planner::dp_optimize (optimizer.cpp:157-183), the final pick
// (:185-195) and the traceback (:197-204).
//
// Bit-exactness: every FP64 operation is an explicit __d*_rn intrinsic in the
// reference's operand order, so nothing is contracted into an FMA (the
// reference's x86-64 build has no FMA).  Probabilities are
// count_m / count exactly as the reference's normalised histogram.
//
// Layout: one block per next-level node; threads stride over prev nodes; the
// (value desc, mig asc, first index) argmax is a warp-shuffle + cross-warp
// reduction.  The winning value, migration total, back-pointer and step terms
// of every node stay in HBM for the traceback.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "liveput.h"
#include "lp_launch.h"
#include "lp_layout.h"

namespace lp {

struct PhiOut {
  double committed;
  double mig;
};

__device__ __forceinline__ int replication_rounds(int sources, int transfers) {
  int rounds = 0;
  long long have = sources;
  const long long need = static_cast<long long>(sources) + transfers;
  while (have < need) {
    have *= 2;
    ++rounds;
  }
  return rounds;
}

// transition_outcome_min (migration.cpp:49-89) + rollback penalty
// (optimizer.cpp:123).  fixed = fresh > 0 ? fresh_fixed : 0.0.
__device__ __forceinline__ double transition_cost(int m, int sd, int sp, int td, int tp,
                                                  double fixed, const NodeCost& nc,
                                                  const DpScalars& S, bool* rollback) {
  *rollback = false;
  const double base = __dadd_rn(__dadd_rn(fixed, S.build), S.update);
  if (m == 0) {
    *rollback = true;
    return __dadd_rn(base, nc.pipe);
  }
  if (tp != sp) return __dadd_rn(base, nc.pipe);
  const int transfers = td - m > 0 ? td - m : 0;
  const int rounds = replication_rounds(m, transfers);
  const bool assigned_dead = m < sd;
  if (rounds == 0 && !assigned_dead && td == sd) return 0.0;
  if (rounds == 0) return base;
  const double a = __dmul_rn(static_cast<double>(rounds), nc.unit);
  const double inter = (nc.pipe < a) ? nc.pipe : a;  // std::min(a, pipe)
  return __dadd_rn(base, inter);
}

// phi(prev, next, n_now, n_next) from the prev config's deficit histogram
// (rows d = 0..min(k, D), m = D - d).  prob(d) returns hist[m] of the
// reference, count_m / count (0.0 for an empty bin).  thr_tab/thr_row:
// throughput(D, P).
// Bin accessors: probability of bin d, and eight bins d0, d0-1, ... d0-7
// (0.0 below d = 0) fetched together.
// Eight bins that are all +0.0 (probabilities are never -0.0) add nothing:
// adding +0.0 to a non-negative sum is exact, so a zero chunk is skipped.
__device__ __forceinline__ bool zero8(const double (&pr)[8]) {
  unsigned long long o = 0ull;
#pragma unroll
  for (int u = 0; u < 8; ++u) o |= static_cast<unsigned long long>(__double_as_longlong(pr[u]));
  return o == 0ull;
}

struct ProbPtr {
  const double* hp;
  __device__ __forceinline__ double operator()(int d) const { return hp[d]; }
  __device__ __forceinline__ void chunk(int d0, double (&pr)[8]) const {
    const double* q = hp + d0;
#pragma unroll
    for (int u = 0; u < 8; ++u) pr[u] = (u <= d0) ? q[-u] : 0.0;
  }
};

struct ProbCounts {  // count_m / count straight from the u32 histogram
  const uint32_t* h;
  double total;
  __device__ __forceinline__ double operator()(int d) const {
    return h[d] ? __ddiv_rn(static_cast<double>(h[d]), total) : 0.0;
  }
  __device__ __forceinline__ void chunk(int d0, double (&pr)[8]) const {
#pragma unroll
    for (int u = 0; u < 8; ++u) pr[u] = (u <= d0) ? (*this)(d0 - u) : 0.0;
  }
};

// Terms of phi that depend only on the level and the next config, in the
// reference's order: the repartition cost (rollback when m == 0, or any
// depth change) is ((fixed + build) + update) + pipe (+ rollback penalty).
struct PhiConst {
  double base, c_pipe, c_rb, teff_pipe, teff_rb;
};

__device__ __forceinline__ PhiConst phi_const(const LevelDesc& L, const DpScalars& S, const NodeCost& nc) {
  PhiConst c;
  c.base = __dadd_rn(__dadd_rn(L.fixed, S.build), S.update);
  c.c_pipe = __dadd_rn(c.base, nc.pipe);
  c.c_rb = __dadd_rn(c.c_pipe, S.rollback);
  const double te_pipe = __dsub_rn(S.T, c.c_pipe), te_rb = __dsub_rn(S.T, c.c_rb);
  c.teff_pipe = (0.0 < te_pipe) ? te_pipe : 0.0;
  c.teff_rb = (0.0 < te_rb) ? te_rb : 0.0;
  return c;
}

template <class Prob>
__device__ __forceinline__ PhiOut phi_dev(const NodeCfg& pv, const NodeCfg& nx, const NodeCost& nc,
                                          const LevelDesc& L, const DpScalars& S, Prob prob,
                                          const double* __restrict__ thr_tab,
                                          const int32_t* __restrict__ thr_row, const PhiConst& K) {
  PhiOut o{0.0, 0.0};
  if (nx.d <= 0) return o;  // suspended next: nothing committed, nothing moved
  if (pv.d <= 0) {          // resume from suspension (optimizer.cpp:108-115)
    const double te = __dsub_rn(S.T, nc.resume);
    o.mig = nc.resume;
    o.committed = __dmul_rn(nc.thr, (0.0 < te) ? te : 0.0);
    return o;
  }
  const int dmax = min(L.k, pv.d);
  const double base = K.base, c_pipe = K.c_pipe, c_rb = K.c_rb;
  const double teff_pipe = K.teff_pipe, teff_rb = K.teff_rb;
  const bool same_depth = nx.p == pv.p;
  double committed = 0.0, cost_sum = 0.0;
  if (!same_depth && !S.strict) {
    // Depth change (most pairs): every bin but m = 0 costs c_pipe at the
    // next config's own rate.  Empty bins add +0.0 to non-negative sums,
    // which is exact, so the loop needs no per-bin branch; bins are fetched
    // eight at a time ahead of the order-fixed accumulation.
    const double rate = nc.thr;
    int d = dmax;
    if (dmax == pv.d) {  // m = 0: rollback
      const double p = prob(d);
      committed = __dadd_rn(committed, __dmul_rn(__dmul_rn(p, rate), teff_rb));
      cost_sum = __dadd_rn(cost_sum, __dmul_rn(p, c_rb));
      --d;
    }
    for (int d0 = d; d0 >= 0; d0 -= 8) {
      double pr[8];
      prob.chunk(d0, pr);
      if (zero8(pr)) continue;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        committed = __dadd_rn(committed, __dmul_rn(__dmul_rn(pr[u], rate), teff_pipe));
        cost_sum = __dadd_rn(cost_sum, __dmul_rn(pr[u], c_pipe));
      }
    }
    o.committed = committed;
    o.mig = cost_sum;
    return o;
  }
  if (!S.strict) {
    // Same depth: transition_cost per bin, branch-free.  rounds = the least
    // r with m * 2^r >= max(td, m) (replication_rounds) from the bit lengths;
    // every FP64 value is computed as the branchy code would and selected.
    const int sd = pv.d, td = nx.d;
    const double rate = nc.thr;
    for (int d0 = dmax; d0 >= 0; d0 -= 8) {
      double pr[8];
      prob.chunk(d0, pr);
      if (zero8(pr)) continue;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int m = sd - (d0 - u);  // bins past d = 0 carry p = 0
        const int mm = m > 0 ? m : 1;
        int r = 0;
        if (td > mm) {
          r = __clz(mm) - __clz(td);
          r += ((mm << r) < td) ? 1 : 0;
        }
        const double inter_a = __dmul_rn(static_cast<double>(r), nc.unit);
        const double inter = (nc.pipe < inter_a) ? nc.pipe : inter_a;
        const double c_rep = __dadd_rn(base, inter);
        double cost = (r == 0) ? ((m >= sd && td == sd) ? 0.0 : base) : c_rep;
        cost = (m == 0) ? c_rb : cost;
        const double te = __dsub_rn(S.T, cost);
        double t_eff = (0.0 < te) ? te : 0.0;
        t_eff = (m == 0) ? teff_rb : t_eff;
        committed = __dadd_rn(committed, __dmul_rn(__dmul_rn(pr[u], rate), t_eff));
        cost_sum = __dadd_rn(cost_sum, __dmul_rn(pr[u], cost));
      }
    }
    o.committed = committed;
    o.mig = cost_sum;
    return o;
  }
  for (int d0 = dmax; d0 >= 0; d0 -= 8) {  // m = D - d ascending
    double pr[8];
    prob.chunk(d0, pr);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int d = d0 - u;
      if (d < 0) break;
      const double p = pr[u];
      if (p == 0.0) continue;
      const int m = pv.d - d;
      double cost, t_eff;
      if (m == 0) {
        cost = c_rb;
        t_eff = teff_rb;
      } else if (!same_depth) {
        cost = c_pipe;
        t_eff = teff_pipe;
      } else {
        bool rb;
        cost = transition_cost(m, pv.d, pv.p, nx.d, nx.p, L.fixed, nc, S, &rb);
        const double te = __dsub_rn(S.T, cost);
        t_eff = (0.0 < te) ? te : 0.0;
      }
      double rate = nc.thr;
      if (S.strict) {
        const int alive = min(nx.d, m);
        rate = alive > 0 ? thr_tab[thr_row[nx.p] + alive] : 0.0;
      }
      committed = __dadd_rn(committed, __dmul_rn(__dmul_rn(p, rate), t_eff));
      cost_sum = __dadd_rn(cost_sum, __dmul_rn(p, cost));
    }
  }
  o.committed = committed;
  o.mig = cost_sum;
  return o;
}

// phi of two depth-changing pairs (prev a, prev b -> the same next,
// non-strict) with their bin loops interleaved: two independent FP64 chains
// per step instead of one.  Each pair's operation sequence is exactly
// phi_dev's fast path (bins d = dmax .. 0 in order, +0.0 past d = 0).
__device__ __forceinline__ void phi_fast2(const NodeCfg& a, const NodeCfg& b, const double* ha,
                                          const double* hb, int k, double rate, const PhiConst& K,
                                          PhiOut& oa, PhiOut& ob) {
  const int da = min(k, a.d), db = min(k, b.d);
  double ca, ma, cb, mb;
  {  // bin d = dmax: the rollback bin (m = 0) when every assigned slot can be lost
    const double pa = ha[da], pb = hb[db];
    const bool ra = da == a.d, rb = db == b.d;
    ca = __dadd_rn(0.0, __dmul_rn(__dmul_rn(pa, rate), ra ? K.teff_rb : K.teff_pipe));
    ma = __dadd_rn(0.0, __dmul_rn(pa, ra ? K.c_rb : K.c_pipe));
    cb = __dadd_rn(0.0, __dmul_rn(__dmul_rn(pb, rate), rb ? K.teff_rb : K.teff_pipe));
    mb = __dadd_rn(0.0, __dmul_rn(pb, rb ? K.c_rb : K.c_pipe));
  }
  const int nb = max(da, db);  // bins i = 1 .. nb (d = dmax - i)
  for (int i0 = 1; i0 <= nb; i0 += 8) {
    double pa[8], pb[8];
    const double* qa = ha + (da - i0);
    const double* qb = hb + (db - i0);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      pa[u] = (i0 + u <= da) ? qa[-u] : 0.0;
      pb[u] = (i0 + u <= db) ? qb[-u] : 0.0;
    }
    if (zero8(pa) && zero8(pb)) continue;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      ca = __dadd_rn(ca, __dmul_rn(__dmul_rn(pa[u], rate), K.teff_pipe));
      cb = __dadd_rn(cb, __dmul_rn(__dmul_rn(pb[u], rate), K.teff_pipe));
      ma = __dadd_rn(ma, __dmul_rn(pa[u], K.c_pipe));
      mb = __dadd_rn(mb, __dmul_rn(pb[u], K.c_pipe));
    }
  }
  oa = PhiOut{ca, ma};
  ob = PhiOut{cb, mb};
}

// hist[m] = count_m / count, once per re-plan (after the cross-rank reduce),
// so the DP's inner loop has no FP64 division.  One block per depth entry.
__global__ void normalize_kernel(const PairDesc* __restrict__ pairs,
                                 const EntryDesc* __restrict__ entries,
                                 const uint32_t* __restrict__ hist,
                                 const int32_t* __restrict__ store_off, double* __restrict__ store) {
  const EntryDesc e = entries[blockIdx.x];
  const PairDesc pd = pairs[e.pair];
  const int len = hist_row(e.Dmax + 1, pd.k);
  const double total = static_cast<double>(pd.count);
  double* out = store + store_off[blockIdx.x];
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    const uint32_t c = hist[e.hist_off + i];
    out[i] = c ? __ddiv_rn(static_cast<double>(c), total) : 0.0;
  }
}

struct Cand {
  double value, mig, stc, stm;
  int idx;
};

// a better than b in the DP's take order: value desc, mig asc, index asc.
__device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) {
  if (a.idx < 0) return false;
  if (b.idx < 0) return true;
  if (a.value > b.value) return true;
  if (a.value < b.value) return false;
  if (a.mig < b.mig) return true;
  if (a.mig > b.mig) return false;
  return a.idx < b.idx;
}

__device__ __forceinline__ Cand shfl_cand(const Cand& c, int src) {
  Cand o;
  o.value = __shfl_sync(0xffffffffu, c.value, src);
  o.mig = __shfl_sync(0xffffffffu, c.mig, src);
  o.stc = __shfl_sync(0xffffffffu, c.stc, src);
  o.stm = __shfl_sync(0xffffffffu, c.stm, src);
  o.idx = __shfl_sync(0xffffffffu, c.idx, src);
  return o;
}

// F_{j+1}[c'] = max_c F_j[c] + phi(c, c') with the reference's tie rules.
// One block per next-level node; threads stride over the prev nodes (each
// keeps the first best in its own ascending order), then a warp-shuffle and a
// cross-warp reduction pick (value desc, mig asc, index asc).
__global__ void __launch_bounds__(512) dp_step_kernel(int j, const LevelDesc* __restrict__ levels,
                                                      const NodeCfg* __restrict__ cfg,
                                                      const double4* __restrict__ pcost,
                                                      const double* __restrict__ histp,
                                                      const double* __restrict__ thr_tab,
                                                      const int32_t* __restrict__ thr_row,
                                                      DpScalars S, double* __restrict__ val,
                                                      double* __restrict__ mig,
                                                      int32_t* __restrict__ parent,
                                                      double* __restrict__ stc,
                                                      double* __restrict__ stm) {
  __shared__ Cand s_best[16];
  // Programmatic dependent launch: level j+1 may start once every block of
  // level j runs; its prologue (tables only) then overlaps this level, and
  // griddepcontrol.wait below holds it until level j's values are visible.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const LevelDesc L = levels[j];
  if (static_cast<int>(blockIdx.x) >= L.next_count) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ni = L.next_base + blockIdx.x;
  const NodeCfg nx = cfg[ni];
  NodeCost nc{0.0, 0.0, 0.0, 0.0};
  if (nx.d > 0) {  // per-depth cost terms + throughput(next) from the tables
    const double4 pc = pcost[nx.p];
    nc.thr = thr_tab[thr_row[nx.p] + nx.d];
    nc.pipe = pc.x;
    nc.unit = pc.y;
    nc.resume = pc.z;
  }
  const PhiConst K = phi_const(L, S, nc);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // level j-1's val / mig
  Cand best{0.0, 0.0, 0.0, 0.0, -1};
  // full take-order key (value desc, mig asc, index asc): prevs may be
  // folded out of index order below
  auto take = [&](int pi, int gi, const PhiOut& ph) {
    const double v = __dadd_rn(val[gi], ph.committed);
    const double mg = __dadd_rn(mig[gi], ph.mig);
    if (best.idx < 0 || v > best.value ||
        (v == best.value && (mg < best.mig || (mg == best.mig && pi < best.idx)))) {
      best.value = v;
      best.mig = mg;
      best.stc = ph.committed;
      best.stm = ph.mig;
      best.idx = pi;
    }
  };
  // depth-changing prevs (most of them) are evaluated two at a time
  const bool fast_ok = nx.d > 0 && !S.strict;
  int held = -1;  // an eligible prev waiting for a partner
  NodeCfg held_cfg{};
  for (int pi = threadIdx.x; pi < L.prev_count; pi += blockDim.x) {
    const int gi = L.prev_base + pi;
    const NodeCfg pv = cfg[gi];
    if (fast_ok && pv.d > 0 && pv.p != nx.p) {
      if (held < 0) {
        held = pi;
        held_cfg = pv;
        continue;
      }
      PhiOut oa, ob;
      phi_fast2(held_cfg, pv, histp + held_cfg.hist_off, histp + pv.hist_off, L.k, nc.thr, K, oa, ob);
      take(held, L.prev_base + held, oa);
      take(pi, gi, ob);
      held = -1;
      continue;
    }
    const PhiOut ph = phi_dev(pv, nx, nc, L, S, ProbPtr{histp + pv.hist_off}, thr_tab, thr_row, K);
    take(pi, gi, ph);
  }
  if (held >= 0) {
    const PhiOut ph = phi_dev(held_cfg, nx, nc, L, S, ProbPtr{histp + held_cfg.hist_off}, thr_tab, thr_row, K);
    take(held, L.prev_base + held, ph);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const Cand o = shfl_cand(best, lane ^ off);
    if (cand_better(o, best)) best = o;
  }
  if (lane == 0) s_best[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (cand_better(s_best[w], best)) best = s_best[w];
    val[ni] = best.value;
    mig[ni] = best.mig;
    parent[ni] = best.idx;
    stc[ni] = best.stc;
    stm[ni] = best.stm;
  }
}

// Materialised phi for the pipelined re-plan.  phi(prev, next) of level j
// depends only on the level's histograms and the two configs, never on the
// DP values, so it is taken off the level chain: once a pipeline stage's
// probabilities are in the store, throughput launches evaluate every
// (prev, next) pair of the levels that stage released into
// phi[L.phi_off + prev * next_count + next] = (committed, mig).
// One block per (level, kPhiG consecutive prevs): each prev's nonzero bins
// are compacted in shared memory in summation order (d = dmax .. 0, i.e.
// m ascending); each thread then takes next nodes, loads the next node's
// constants once and sums the kPhiG prevs against them.  Skipping a zero bin
// is exact (it adds +0.0 to non-negative sums), and every other operation
// is phi_dev's, in its order, so the values are phi_dev's bit for bit.
// blockIdx.y indexes the launch's level list.
constexpr int kPhiG = 4;        // prevs per block
constexpr int kPhiBins = 512;   // longer rows take phi_dev on the store directly

__global__ void __launch_bounds__(256) phi_matrix_kernel(const int32_t* __restrict__ lv_list,
                                                         const LevelDesc* __restrict__ levels,
                                                         const NodeCfg* __restrict__ cfg,
                                                         const double4* __restrict__ pcost,
                                                         const double* __restrict__ histp,
                                                         const double* __restrict__ thr_tab,
                                                         const int32_t* __restrict__ thr_row,
                                                         DpScalars S, double2* __restrict__ phi) {
  __shared__ double s_p[kPhiG][kPhiBins];  // nonzero bins in summation order
  __shared__ int s_m[kPhiG][kPhiBins];     // ... their m = D - d
  __shared__ int s_nnz[kPhiG];
  const LevelDesc L = levels[lv_list[blockIdx.y]];
  const int p0 = blockIdx.x * kPhiG;
  if (p0 >= L.prev_count) return;
  const int ng = min(kPhiG, L.prev_count - p0);
  const int ncnt = L.next_count;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < ng) {  // warp g compacts prev p0 + g's nonzero bins, d descending
    const NodeCfg pv = cfg[L.prev_base + p0 + warp];
    const int dmax = pv.d > 0 ? min(L.k, pv.d) : -1;
    int cnt = -1;  // -1: not staged (suspended prev, or a row past kPhiBins)
    if (dmax >= 0 && dmax < kPhiBins) {
      const double* hp = histp + pv.hist_off;
      cnt = 0;
      for (int c0 = dmax; c0 >= 0; c0 -= 32) {
        const int d = c0 - lane;
        const double v = d >= 0 ? hp[d] : 0.0;
        const unsigned nz = __ballot_sync(0xffffffffu, v != 0.0);
        if (v != 0.0) {
          const int at = cnt + __popc(nz & ((1u << lane) - 1u));
          s_p[warp][at] = v;
          s_m[warp][at] = pv.d - d;
        }
        cnt += __popc(nz);
      }
    }
    if (lane == 0) s_nnz[warp] = cnt;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ncnt; i += blockDim.x) {
    const NodeCfg nx = cfg[L.next_base + i];
    NodeCost nc{0.0, 0.0, 0.0, 0.0};
    if (nx.d > 0) {
      const double4 c = pcost[nx.p];
      nc.thr = thr_tab[thr_row[nx.p] + nx.d];
      nc.pipe = c.x;
      nc.unit = c.y;
      nc.resume = c.z;
    }
    const PhiConst K = phi_const(L, S, nc);
    const double rate = nc.thr;
    for (int g = 0; g < ng; ++g) {
      const NodeCfg pv = cfg[L.prev_base + p0 + g];
      const int nnz = s_nnz[g];
      PhiOut o{0.0, 0.0};
      if (nx.d <= 0 || pv.d <= 0 || S.strict || nnz < 0) {
        o = phi_dev(pv, nx, nc, L, S, ProbPtr{histp + pv.hist_off}, thr_tab, thr_row, K);
      } else if (nx.p != pv.p) {  // depth change: c_pipe for m >= 1, rollback for m = 0
        double committed = 0.0, cost_sum = 0.0;
        for (int q = 0; q < nnz; ++q) {
          const double pr = s_p[g][q];
          const bool rb = s_m[g][q] == 0;
          committed = __dadd_rn(committed, __dmul_rn(__dmul_rn(pr, rate), rb ? K.teff_rb : K.teff_pipe));
          cost_sum = __dadd_rn(cost_sum, __dmul_rn(pr, rb ? K.c_rb : K.c_pipe));
        }
        o = PhiOut{committed, cost_sum};
      } else {  // same depth: phi_dev's branch-free per-bin transition cost
        const int sd = pv.d, td = nx.d;
        double committed = 0.0, cost_sum = 0.0;
        for (int q = 0; q < nnz; ++q) {
          const double pr = s_p[g][q];
          const int m = s_m[g][q];
          const int mm = m > 0 ? m : 1;
          int r = 0;
          if (td > mm) {
            r = __clz(mm) - __clz(td);
            r += ((mm << r) < td) ? 1 : 0;
          }
          const double inter_a = __dmul_rn(static_cast<double>(r), nc.unit);
          const double inter = (nc.pipe < inter_a) ? nc.pipe : inter_a;
          const double c_rep = __dadd_rn(K.base, inter);
          double cost = (r == 0) ? ((m >= sd && td == sd) ? 0.0 : K.base) : c_rep;
          cost = (m == 0) ? K.c_rb : cost;
          const double te = __dsub_rn(S.T, cost);
          double t_eff = (0.0 < te) ? te : 0.0;
          t_eff = (m == 0) ? K.teff_rb : t_eff;
          committed = __dadd_rn(committed, __dmul_rn(__dmul_rn(pr, rate), t_eff));
          cost_sum = __dadd_rn(cost_sum, __dmul_rn(pr, cost));
        }
        o = PhiOut{committed, cost_sum};
      }
      phi[static_cast<int64_t>(L.phi_off) + static_cast<int64_t>(p0 + g) * ncnt + i] =
          make_double2(o.committed, o.mig);
    }
  }
}

// The level step over materialised phi: F_{j+1}[c'] = max_c F_j[c] +
// phi(c, c'), a max-plus pass with the reference's take order.  A warp per
// next node (eight per block, so a level needs few SM slots while the
// sampling still runs), lanes over the prevs (a column of the prev-major phi
// block) with four loads in flight per lane, then a shuffle arg-max.  phi is
// fetched before griddepcontrol.wait (it was complete before this level's
// event wait), the previous level's values after it.
__global__ void __launch_bounds__(256) dp_maxplus_kernel(int j, const LevelDesc* __restrict__ levels,
                                                         const double2* __restrict__ phi,
                                                         double* __restrict__ val, double* __restrict__ mig,
                                                         int32_t* __restrict__ parent,
                                                         double* __restrict__ stc, double* __restrict__ stm) {
  constexpr int kU = 4;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const LevelDesc L = levels[j];
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const bool live = i < L.next_count;
  const int pc = L.prev_count;
  const int64_t ncnt = L.next_count;
  const double2* col = phi + static_cast<int64_t>(L.phi_off) + i;
  double2 f[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int pi = lane + 32 * u;
    f[u] = live && pi < pc ? col[pi * ncnt] : make_double2(0.0, 0.0);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // level j-1's val / mig
  if (!live) return;
  const double* pval = val + L.prev_base;
  const double* pmig = mig + L.prev_base;
  Cand best{0.0, 0.0, 0.0, 0.0, -1};
  auto take = [&](int pi, double v0, double m0, const double2& ph) {
    const double v = __dadd_rn(v0, ph.x);
    const double mg = __dadd_rn(m0, ph.y);
    if (best.idx < 0 || v > best.value || (v == best.value && mg < best.mig)) {
      best.value = v;
      best.mig = mg;
      best.stc = ph.x;
      best.stm = ph.y;
      best.idx = pi;
    }
  };
  for (int p0 = 0; p0 < pc; p0 += 32 * kU) {
    double v[kU], m[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int pi = p0 + lane + 32 * u;
      if (p0 > 0) f[u] = pi < pc ? col[pi * ncnt] : make_double2(0.0, 0.0);
      v[u] = pi < pc ? pval[pi] : 0.0;
      m[u] = pi < pc ? pmig[pi] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int pi = p0 + lane + 32 * u;
      if (pi < pc) take(pi, v[u], m[u], f[u]);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const Cand o = shfl_cand(best, lane ^ off);
    if (cand_better(o, best)) best = o;
  }
  if (lane == 0) {
    const int ni = L.next_base + i;
    val[ni] = best.value;
    mig[ni] = best.mig;
    parent[ni] = best.idx;
    stc[ni] = best.stc;
    stm[ni] = best.stm;
  }
}

// Final pick (rank = (value, -mig, D, -P), suspended = (-1, 0), first index
// wins) and traceback into PlanStep[horizon], by one block of 256 threads.
// With s_dyn (n_nodes +
// 2 * horizon ints of shared memory) every back-pointer is staged first, so
// the serial walk costs a shared-memory load per level instead of an L2
// round trip, and the plan rows are then written in parallel.
__device__ void final_pick_traceback(const LevelDesc* __restrict__ levels, int horizon,
                                     const NodeCfg* __restrict__ cfg, const double* val, const double* mig,
                                     const int32_t* parent, const double* stc, const double* stm,
                                     lp_plan_step* __restrict__ plan, double* __restrict__ final_value,
                                     int* s_idx, int* s_dyn, int n_nodes) {
  const LevelDesc last = levels[horizon - 1];
  const int base = last.next_base, cnt = last.next_count;
  // rank = (value, -mig, D, -P), suspended (-1, 0); the first index wins
  // ties.  Each thread scans its nodes in ascending order (strict > keeps
  // the first), then the keys are reduced in registers: warp shuffles, then
  // one slot per warp in shared memory.
  struct Key {
    double v, nm;
    int d, np, idx;
  };
  auto better = [](const Key& a, const Key& b) -> bool {  // a ranks above b (b.idx < 0: empty)
    if (a.idx < 0) return false;
    if (b.idx < 0) return true;
    if (a.v != b.v) return b.v < a.v;
    if (a.nm != b.nm) return b.nm < a.nm;
    if (a.d != b.d) return b.d < a.d;
    if (a.np != b.np) return b.np < a.np;
    return a.idx < b.idx;
  };
  Key mine{0.0, 0.0, 0, 0, -1};
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const NodeCfg c = cfg[base + i];
    const Key k{__ldcg(val + base + i), -__ldcg(mig + base + i), c.d > 0 ? c.d : -1, c.d > 0 ? -c.p : 0, i};
    if (better(k, mine)) mine = k;
  }
  if (s_dyn) {
    for (int i = threadIdx.x; i < n_nodes; i += blockDim.x) s_dyn[i] = __ldcg(parent + i);
    for (int jj = threadIdx.x; jj < horizon; jj += blockDim.x) s_dyn[n_nodes + jj] = levels[jj].next_base;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Key o;
    o.v = __shfl_xor_sync(0xffffffffu, mine.v, off);
    o.nm = __shfl_xor_sync(0xffffffffu, mine.nm, off);
    o.d = __shfl_xor_sync(0xffffffffu, mine.d, off);
    o.np = __shfl_xor_sync(0xffffffffu, mine.np, off);
    o.idx = __shfl_xor_sync(0xffffffffu, mine.idx, off);
    if (better(o, mine)) mine = o;
  }
  __shared__ Key s_key[32];
  if ((threadIdx.x & 31) == 0) s_key[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (better(s_key[w], mine)) mine = s_key[w];
    s_idx[0] = mine.idx;
  }
  __syncthreads();
  auto row = [&](int jj, int gi) {  // plan step of interval jj (1-based)
    const NodeCfg c = cfg[gi];
    lp_plan_step st;
    st.interval_index = jj;
    st.config.pipelines = c.d > 0 ? c.d : 0;
    st.config.stages = c.d > 0 ? c.p : 0;
    st.expected_committed = __ldcg(stc + gi);
    st.expected_mig_cost_s = __ldcg(stm + gi);
    plan[jj - 1] = st;
  };
  if (s_dyn) {
    const int* s_nb = s_dyn + n_nodes;
    int* s_gi = s_dyn + n_nodes + horizon;
    if (threadIdx.x == 0) {
      int idx = s_idx[0];
      if (final_value) *final_value = __ldcg(val + base + idx);
      for (int jj = horizon; jj >= 1; --jj) {
        const int gi = s_nb[jj - 1] + idx;
        s_gi[jj - 1] = gi;
        idx = s_dyn[gi];
      }
    }
    __syncthreads();
    for (int jj = threadIdx.x; jj < horizon; jj += blockDim.x) row(jj + 1, s_gi[jj]);
    return;
  }
  if (threadIdx.x == 0) {
    int idx = s_idx[0];
    if (final_value) *final_value = __ldcg(val + base + idx);
    for (int jj = horizon; jj >= 1; --jj) {
      const int gi = levels[jj - 1].next_base + idx;
      row(jj, gi);
      idx = __ldcg(parent + gi);
    }
  }
}

__global__ void __launch_bounds__(256) dp_final_kernel(const LevelDesc* __restrict__ levels, int horizon,
                                                       const NodeCfg* __restrict__ cfg, const double* val,
                                                       const double* mig, const int32_t* parent,
                                                       const double* stc, const double* stm,
                                                       lp_plan_step* __restrict__ plan,
                                                       double* __restrict__ final_value, int n_nodes) {
  __shared__ int s_idx[256];
  extern __shared__ int s_dyn[];
  final_pick_traceback(levels, horizon, cfg, val, mig, parent, stc, stm, plan, final_value, s_idx,
                       n_nodes > 0 ? s_dyn : nullptr, n_nodes);
}

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Monotone arrival counter (zeroed before the launch): a barrier completes
// when the counter reaches `target`, the running total of the blocks taking
// part in every barrier so far (all blocks for the first, the level blocks
// after it).
__device__ __forceinline__ void grid_barrier(uint32_t* ctr, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (ld_relaxed_u32(ctr) < target) __nanosleep(32);
    __threadfence();  // acquire: orders the block's later reads after the arrivals
  }
  __syncthreads();
}



// Liveput table: for each (level with histogram, prev config) row,
// sum_m count_m * throughput(m, P) / count (expected_liveput semantics,
// preemption.cpp:87-112, intra-stage recovery).
__global__ void liveput_kernel(const int4* __restrict__ rows /* level, node, out_row, - */,
                               int n_rows, const LevelDesc* __restrict__ levels,
                               const NodeCfg* __restrict__ cfg, const uint32_t* __restrict__ hist,
                               const double* __restrict__ probs,
                               const double* __restrict__ thr_tab,
                               const int32_t* __restrict__ thr_row,
                               lp_liveput_row* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const int4 rw = rows[r];
  const LevelDesc L = levels[rw.x];
  const NodeCfg c = cfg[rw.y];
  const int dmax = min(L.k, c.d);
  double acc = 0.0;
  if (probs) {  // store path: sum_m p_m * thr(m, P)
    const double* p = probs + c.hist_off;
    for (int d = dmax; d >= 0; --d) {
      const int m = c.d - d;
      if (m < 1 || p[d] == 0.0) continue;
      acc = __dadd_rn(acc, __dmul_rn(p[d], thr_tab[thr_row[c.p] + m]));
    }
  } else {  // counts path: sum_m count_m * thr(m, P) / count
    const uint32_t* h = hist + c.hist_off;
    for (int d = dmax; d >= 0; --d) {
      const int m = c.d - d;
      if (m < 1 || h[d] == 0u) continue;
      acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(h[d]), thr_tab[thr_row[c.p] + m]));
    }
    acc = __ddiv_rn(acc, static_cast<double>(L.total));
  }
  lp_liveput_row o;
  o.interval = rw.x;
  o.config.pipelines = c.d;
  o.config.stages = c.p;
  o.liveput = acc;
  out[rw.z] = o;
}

// Single phi evaluation (lp_phi): one thread.
__global__ void phi_single_kernel(NodeCfg pv, NodeCfg nx, NodeCost nc, LevelDesc L, DpScalars S,
                                  const uint32_t* __restrict__ hist,
                                  const double* __restrict__ thr_tab,
                                  const int32_t* __restrict__ thr_row, double* __restrict__ out2) {
  const double total = static_cast<double>(L.total);
  const uint32_t* h = hist + pv.hist_off;
  const PhiOut o = phi_dev(pv, nx, nc, L, S, ProbCounts{h, total}, thr_tab, thr_row, phi_const(L, S, nc));
  out2[0] = o.committed;
  out2[1] = o.mig;
}

// ---------------------------------------------------------------------------
cudaError_t launch_dp_step(int j, int next_count, int prev_count, bool pdl, cudaStream_t st,
                           const LevelDesc* levels, const NodeCfg* cfg, const double4* pcost,
                           const double* histp, const double* thr_tab, const int32_t* thr_row,
                           const DpScalars& S, double* val, double* mig, int32_t* parent,
                           double* stc, double* stm) {
  const int blocks = next_count;
  if (blocks <= 0) return cudaSuccess;
  // 128 threads per next node measured fastest (more threads per node cost
  // more in the cross-warp reduction than the shorter phi chains save)
  static const int cap = [] {
    const char* e = getenv("LIVEPUT_DP_THREADS");
    const int v = e ? atoi(e) : 0;
    return (v >= 32 && v <= 512) ? v : 128;
  }();
  const int threads = std::min(cap, std::max(32, (prev_count + 31) / 32 * 32));
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(blocks);
  lc.blockDim = dim3(threads);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&lc, dp_step_kernel, j, levels, cfg, pcost, histp, thr_tab, thr_row, S, val, mig,
                            parent, stc, stm);
}

cudaError_t launch_phi_matrix(int n_levels, int64_t max_pairs, cudaStream_t st, const int32_t* lv_list,
                              const LevelDesc* levels, const NodeCfg* cfg, const double4* pcost,
                              const double* histp, const double* thr_tab, const int32_t* thr_row,
                              const DpScalars& S, double2* phi) {
  if (n_levels <= 0 || max_pairs <= 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((max_pairs + kPhiG - 1) / kPhiG), static_cast<unsigned>(n_levels));  // max_pairs: largest prev count
  phi_matrix_kernel<<<grid, 256, 0, st>>>(lv_list, levels, cfg, pcost, histp, thr_tab, thr_row, S, phi);
  return cudaGetLastError();
}

cudaError_t launch_dp_maxplus(int j, int next_count, bool pdl, cudaStream_t st, const LevelDesc* levels,
                              const double2* phi, double* val, double* mig, int32_t* parent, double* stc,
                              double* stm) {
  if (next_count <= 0) return cudaSuccess;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((next_count + 7) / 8);
  lc.blockDim = dim3(256);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&lc, dp_maxplus_kernel, j, levels, phi, val, mig, parent, stc, stm);
}

cudaError_t launch_normalize(int n_entries, cudaStream_t st, const PairDesc* pairs,
                             const EntryDesc* ents, const uint32_t* hist, const int32_t* store_off,
                             double* store) {
  if (n_entries <= 0) return cudaSuccess;
  normalize_kernel<<<n_entries, 128, 0, st>>>(pairs, ents, hist, store_off, store);
  return cudaGetLastError();
}

// dynamic shared memory of the staged traceback (0: the walk reads L2)
static size_t trace_smem(int n_nodes, int horizon) {
  const size_t b = static_cast<size_t>(n_nodes + 2 * horizon) * sizeof(int);
  return b <= 160 * 1024 ? b : 0;
}

cudaError_t launch_dp_final(int horizon, cudaStream_t st, const LevelDesc* levels,
                            const NodeCfg* cfg, const double* val, const double* mig,
                            const int32_t* parent, const double* stc, const double* stm,
                            lp_plan_step* plan, double* final_value, int n_nodes) {
  const size_t smem = n_nodes > 0 ? trace_smem(n_nodes, horizon) : 0;
  if (smem > 48 * 1024) {
    const cudaError_t e = smem_optin(reinterpret_cast<const void*>(dp_final_kernel), smem);
    if (e != cudaSuccess) return e;
  }
  dp_final_kernel<<<1, 256, smem, st>>>(levels, horizon, cfg, val, mig, parent, stc, stm, plan,
                                        final_value, smem ? n_nodes : 0);
  return cudaGetLastError();
}

cudaError_t launch_liveput(int n_rows, cudaStream_t st, const int4* rows, const LevelDesc* levels,
                           const NodeCfg* cfg, const uint32_t* hist, const double* probs,
                           const double* thr_tab, const int32_t* thr_row, lp_liveput_row* out) {
  if (n_rows <= 0) return cudaSuccess;
  liveput_kernel<<<(n_rows + 127) / 128, 128, 0, st>>>(rows, n_rows, levels, cfg, hist, probs,
                                                       thr_tab, thr_row, out);
  return cudaGetLastError();
}

cudaError_t launch_phi_single(const NodeCfg& pv, const NodeCfg& nx, const NodeCost& nc,
                              const LevelDesc& L, const DpScalars& S, const uint32_t* hist,
                              const double* thr_tab, const int32_t* thr_row, double* out2,
                              cudaStream_t st) {
  phi_single_kernel<<<1, 1, 0, st>>>(pv, nx, nc, L, S, hist, thr_tab, thr_row, out2);
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// Persistent DP: normalisation, the H level steps, the final pick and the
// traceback in ONE cooperative launch, separated by a grid barrier instead of
// H + 2 kernel boundaries.  Values written inside the launch (probabilities,
// val/mig/parent/step terms) are read back through L2 (ld.cg) or after a
// barrier that follows their only writes, never through the read-only path.

// STAGED (small re-plans, N ~ 16..48): every block copies the node list, its
// own next nodes' cost terms for every level, and all prev probability rows
// into shared memory up front, with all the loads in flight at once.  A level
// then reads only the previous level's values from L2; the dependent
// level -> node -> cost -> row load chain (~2 us of a ~5 us level at N=32)
// is gone.  Dynamic shared layout: cfg [n_nodes] | levels [H] | cost [H] |
// row bases [H + 1] | probabilities; level j's prev rows sit at
// base_j + i * (min(k_j, n_now_j) + 1).
struct StagedLayout {
  int n_nodes, horizon, n_prob;
  __host__ __device__ size_t cfg_off() const { return 0; }
  __host__ __device__ size_t lv_off() const { return (size_t)n_nodes * sizeof(NodeCfg); }
  __host__ __device__ size_t nc_off() const { return lv_off() + (size_t)horizon * sizeof(LevelDesc); }
  __host__ __device__ size_t base_off() const { return nc_off() + (size_t)horizon * sizeof(NodeCost); }
  __host__ __device__ size_t prob_off() const {
    return (base_off() + (size_t)(horizon + 1) * sizeof(int) + 15) & ~static_cast<size_t>(15);
  }
  __host__ __device__ size_t bytes() const { return prob_off() + (size_t)n_prob * sizeof(double); }
};

template <bool STAGED>
__global__ void __launch_bounds__(256, STAGED ? 2 : 4) dp_persistent_kernel(DpArgs a, DpScalars S, StagedLayout G) {
  __shared__ Cand s_best[8];
  __shared__ int s_idx[256];
  __shared__ int s_path[kMaxHorizon + 1];
  extern __shared__ __align__(16) unsigned char sm_raw[];
  NodeCfg* s_cfg = reinterpret_cast<NodeCfg*>(sm_raw + G.cfg_off());
  LevelDesc* s_lv = reinterpret_cast<LevelDesc*>(sm_raw + G.lv_off());
  NodeCost* s_nc = reinterpret_cast<NodeCost*>(sm_raw + G.nc_off());
  int* s_base = reinterpret_cast<int*>(sm_raw + G.base_off());
  double* s_prob = reinterpret_cast<double*>(sm_raw + G.prob_off());
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto next_cost = [&](const NodeCfg& nx) {
    NodeCost nc{0.0, 0.0, 0.0, 0.0};
    if (nx.d > 0) {
      const double4 pc = a.pcost[nx.p];
      nc.thr = a.thr_tab[a.thr_row[nx.p] + nx.d];
      nc.pipe = pc.x;
      nc.unit = pc.y;
      nc.resume = pc.z;
    }
    return nc;
  };
  if (STAGED) {  // tables (independent of phase 0's output)
    for (int i = threadIdx.x; i < G.n_nodes; i += blockDim.x) s_cfg[i] = a.cfg[i];
    for (int j = threadIdx.x; j < G.horizon; j += blockDim.x) {
      const LevelDesc L = a.levels[j];
      s_lv[j] = L;
      NodeCost nc{0.0, 0.0, 0.0, 0.0};
      if (static_cast<int>(blockIdx.x) < L.next_count) nc = next_cost(a.cfg[L.next_base + blockIdx.x]);
      s_nc[j] = nc;
    }
  }
  auto stamp = [&](int slot) {  // LIVEPUT_DP_TRACE: per-block globaltimer stamps
    if (a.trace && threadIdx.x == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      a.trace[(size_t)blockIdx.x * (2 * kTraceLevels + 2) + slot] = t;
    }
  };
  stamp(0);

  // phase 0: probabilities of the fresh entries
  for (int e = blockIdx.x; e < a.n_entries; e += gridDim.x) {
    const EntryDesc en = a.entries[e];
    const PairDesc pd = a.pairs[en.pair];
    const int len = hist_row(en.Dmax + 1, pd.k);
    const double total = static_cast<double>(pd.count);
    double* out = a.store + a.store_off[e];
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      const uint32_t c = a.hist[en.hist_off + i];
      out[i] = c ? __ddiv_rn(static_cast<double>(c), total) : 0.0;
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    a.val[0] = 0.0;  // level 0: value 0, migration 0
    a.mig[0] = 0.0;
  }
  stamp(1);
  uint32_t target = gridDim.x;
  grid_barrier(a.barrier, target);
  // only the blocks that own a next node at some level take part from here;
  // the others were there for the normalisation
  const uint32_t active = min(gridDim.x, static_cast<uint32_t>(a.max_next));
  if (blockIdx.x >= active) return;
  if (STAGED) {  // every prev row the DP reads, from the store (now complete)
    if (threadIdx.x == 0) {
      int b = 0;
      for (int j = 0; j < G.horizon; ++j) {
        s_base[j] = b;
        const LevelDesc& L = s_lv[j];
        if (L.has_hist) b += L.prev_count * (min(L.k, L.n_now) + 1);
      }
      s_base[G.horizon] = b;
    }
    __syncthreads();
    const int n_prev = s_lv[G.horizon - 1].next_base;
    for (int gi = threadIdx.x; gi < n_prev; gi += blockDim.x) {
      int j = 0;
      while (j + 1 < G.horizon && s_lv[j + 1].prev_base <= gi) ++j;
      const LevelDesc& L = s_lv[j];
      const NodeCfg pv = s_cfg[gi];
      if (!L.has_hist || pv.d <= 0 || pv.hist_off < 0) continue;
      const int stride = min(L.k, L.n_now) + 1, len = min(L.k, pv.d) + 1;
      const double* src = a.store + pv.hist_off;
      double* dst = s_prob + s_base[j] + (gi - L.prev_base) * stride;
      for (int d = 0; d < len; ++d) dst[d] = src[d];
    }
    __syncthreads();
  }

  // phases 1..H: F_{j+1}[c'] = max_c F_j[c] + phi(c, c'), one block per next node
  const double* histp = a.store;
  for (int j = 0; j < a.horizon; ++j) {
    const LevelDesc L = STAGED ? s_lv[j] : a.levels[j];
    const int stride = min(L.k, L.n_now) + 1;
    for (int nb = blockIdx.x; nb < L.next_count; nb += gridDim.x) {
      const int ni = L.next_base + nb;
      const NodeCfg nx = STAGED ? s_cfg[ni] : a.cfg[ni];
      const NodeCost nc = (STAGED && nb == static_cast<int>(blockIdx.x)) ? s_nc[j] : next_cost(nx);
      const PhiConst K = phi_const(L, S, nc);
      Cand best{0.0, 0.0, 0.0, 0.0, -1};
      // Prev nodes come in ascending P, descending D, so their bin counts
      // fall along the list: threads take them in snake order (t, 2T-1-t,
      // 2T+t, ...) to even out the per-thread work; ties are broken on the
      // index explicitly, so the visiting order does not matter.
      const int T2 = 2 * static_cast<int>(blockDim.x);
      for (int r = 0;; ++r) {
        const int pi = (r & 1) ? (r + 1) * static_cast<int>(blockDim.x) - 1 - static_cast<int>(threadIdx.x)
                               : r * static_cast<int>(blockDim.x) + static_cast<int>(threadIdx.x);
        if (r * static_cast<int>(blockDim.x) >= L.prev_count) break;
        if (pi >= L.prev_count) continue;
        (void)T2;
        const int gi = L.prev_base + pi;
        const NodeCfg pv = STAGED ? s_cfg[gi] : a.cfg[gi];
        const double* hp = STAGED ? s_prob + s_base[j] + pi * stride : histp + pv.hist_off;
        const PhiOut ph = phi_dev(pv, nx, nc, L, S, ProbPtr{hp}, a.thr_tab, a.thr_row, K);
        const double v = __dadd_rn(__ldcg(a.val + gi), ph.committed);
        const double mg = __dadd_rn(__ldcg(a.mig + gi), ph.mig);
        if (best.idx < 0 || v > best.value ||
            (v == best.value && (mg < best.mig || (mg == best.mig && pi < best.idx)))) {
          best.value = v;
          best.mig = mg;
          best.stc = ph.committed;
          best.stm = ph.mig;
          best.idx = pi;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const Cand o = shfl_cand(best, lane ^ off);
        if (cand_better(o, best)) best = o;
      }
      if (lane == 0) s_best[warp] = best;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
          if (cand_better(s_best[w], best)) best = s_best[w];
        __stcg(a.val + ni, best.value);
        __stcg(a.mig + ni, best.mig);
        __stcg(a.parent + ni, best.idx);
        __stcg(a.stc + ni, best.stc);
        __stcg(a.stm + ni, best.stm);
      }
      __syncthreads();
    }
    if (j < kTraceLevels) stamp(2 + 2 * j);
    target += active;
    grid_barrier(a.barrier, target);
    if (j < kTraceLevels) stamp(3 + 2 * j);
  }

  // final pick (rank = (value, -mig, D, -P), suspended as (-1, 0), first
  // index wins) and traceback, by block 0
  if (blockIdx.x != 0) return;
  const LevelDesc last = a.levels[a.horizon - 1];
  const int base = last.next_base, cnt = last.next_count;
  auto gt = [&](int x, int y) -> bool {  // rank(x) > rank(y)
    if (y < 0) return x >= 0;
    if (x < 0) return false;
    const double va = __ldcg(a.val + base + x), vb = __ldcg(a.val + base + y);
    if (vb < va) return true;
    if (va < vb) return false;
    const double ma = -__ldcg(a.mig + base + x), mb = -__ldcg(a.mig + base + y);
    if (mb < ma) return true;
    if (ma < mb) return false;
    const NodeCfg ca = a.cfg[base + x], cb = a.cfg[base + y];
    const int da = ca.d > 0 ? ca.d : -1, db = cb.d > 0 ? cb.d : -1;
    if (db < da) return true;
    if (da < db) return false;
    const int pa = ca.d > 0 ? -ca.p : 0, pb = cb.d > 0 ? -cb.p : 0;
    return pb < pa;
  };
  int mine = -1;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x)
    if (gt(i, mine)) mine = i;  // ascending i: strict > keeps the first
  s_idx[threadIdx.x] = mine;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      const int x = s_idx[threadIdx.x], y = s_idx[threadIdx.x + st];
      if (gt(y, x) || (y >= 0 && x >= 0 && !gt(x, y) && y < x)) s_idx[threadIdx.x] = y;
    }
    __syncthreads();
  }
  // back-pointer chase: only the parent loads are serial; the plan rows are
  // then written by one thread per interval
  if (threadIdx.x == 0) {
    int idx = s_idx[0];
    if (a.final_value) *a.final_value = __ldcg(a.val + base + idx);
    for (int jj = a.horizon; jj >= 1; --jj) {
      const int gi = a.levels[jj - 1].next_base + idx;
      s_path[jj] = gi;
      idx = __ldcg(a.parent + gi);
    }
  }
  __syncthreads();
  for (int jj = 1 + threadIdx.x; jj <= a.horizon; jj += blockDim.x) {
    const int gi = s_path[jj];
    const NodeCfg c = a.cfg[gi];
    lp_plan_step st;
    st.interval_index = jj;
    st.config.pipelines = c.d > 0 ? c.d : 0;
    st.config.stages = c.d > 0 ? c.p : 0;
    st.expected_committed = __ldcg(a.stc + gi);
    st.expected_mig_cost_s = __ldcg(a.stm + gi);
    a.plan[jj - 1] = st;
  }
}

size_t dp_staged_smem(int n_nodes, int horizon, int n_prob) {
  return StagedLayout{n_nodes, horizon, n_prob}.bytes();
}

cudaError_t launch_dp_persistent(int device, int num_sms, int max_next, cudaStream_t st,
                                 const DpArgs& a, const DpScalars& S, int n_nodes, int n_prob) {
  if (a.horizon > kMaxHorizon) return cudaErrorInvalidValue;
  const bool staged = n_prob >= 0;
  const StagedLayout G{staged ? n_nodes : 0, staged ? a.horizon : 0, staged ? n_prob : 0};
  const size_t smem = staged ? G.bytes() : 0;
  void* fn = staged ? reinterpret_cast<void*>(dp_persistent_kernel<true>)
                    : reinterpret_cast<void*>(dp_persistent_kernel<false>);
  // occupancy per (device, variant, shared size): the grid must be co-resident.
  // The staged variant's shared size changes with every re-plan, so the
  // opt-in above 48 KB (static + dynamic) is set once at the largest size and
  // the occupancy answers are memoised per 1 KB bucket.
  struct Occ {
    int device = -1;
    std::vector<int> per_sm;  // by ceil(smem / 1 KB); 0: unknown
  };
  static thread_local Occ occ[2];
  Occ& o = occ[staged ? 1 : 0];
  cudaError_t e;
  if (o.device != device) {
    if (staged) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) return e;
    }
    o.device = device;
    o.per_sm.assign(201, 0);
  }
  const size_t bucket = (smem + 1023) / 1024;
  if (bucket > 200) return launch_dp_persistent(device, num_sms, max_next, st, a, S, 0, -1);
  int& per_sm = o.per_sm[bucket];
  if (per_sm == 0) {
    int v = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, 256, bucket * 1024);
    if (e != cudaSuccess) return e;
    per_sm = v > 0 ? v : -1;
  }
  if (per_sm < 1)  // does not fit: the unstaged kernel needs no dynamic shared memory
    return staged ? launch_dp_persistent(device, num_sms, max_next, st, a, S, 0, -1) : cudaErrorInvalidConfiguration;
  const int cap = per_sm * num_sms;
  const int grid = std::max(1, std::min(cap, std::max(max_next, a.n_entries)));
  static const bool debug = getenv("LIVEPUT_DP_DEBUG") != nullptr;
  if (debug)
    fprintf(stderr, "[dp] staged %d smem %zu per_sm %d grid %d max_next %d entries %d\n", (int)staged, smem,
            per_sm, grid, max_next, a.n_entries);
  e = cudaMemsetAsync(a.barrier, 0, sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  DpArgs aa = a;
  DpScalars ss = S;
  StagedLayout gg = G;
  void* params[] = {&aa, &ss, &gg};
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(256), params, smem, st);
}


// ---------------------------------------------------------------------------
// Cluster DP for small re-plans (round 2).  One thread-block cluster of
// kClusterCtas CTAs runs normalisation, every level, the final pick and the
// traceback.  Levels are separated by barrier.cluster (release/acquire at
// cluster scope) instead of a grid barrier through global atomics, and the
// level values travel through distributed shared memory: the warp that
// decides node c' stores (F, M) of c' into every CTA's table, so the next
// level reads them from its own shared memory.  One warp per next node: its
// lanes stride over the prev nodes and reduce the take-order key with
// shuffles, with no block barrier inside a level.  Every CTA stages the node
// list, the per-node cost terms and every prev probability row up front, so
// a level touches no global memory except the back-pointer writes.
namespace cg = cooperative_groups;

struct ClusterLayout {
  int n_nodes, horizon, n_prob;
  int n_pcost, n_throw, n_thr;  // per-depth cost terms, throughput rows and values
  __host__ __device__ size_t cfg_off() const { return 0; }
  __host__ __device__ size_t lv_off() const { return (size_t)n_nodes * sizeof(NodeCfg); }
  __host__ __device__ size_t nc_off() const {
    return (lv_off() + (size_t)horizon * sizeof(LevelDesc) + 15) & ~static_cast<size_t>(15);
  }
  __host__ __device__ size_t vm_off() const { return nc_off() + (size_t)n_nodes * sizeof(NodeCost); }
  __host__ __device__ size_t base_off() const { return vm_off() + (size_t)n_nodes * sizeof(double2); }
  __host__ __device__ size_t prob_off() const {
    return (base_off() + (size_t)(horizon + 1) * sizeof(int) + 15) & ~static_cast<size_t>(15);
  }
  __host__ __device__ size_t pc_off() const {
    return (prob_off() + (size_t)n_prob * sizeof(double) + 15) & ~static_cast<size_t>(15);
  }
  __host__ __device__ size_t tt_off() const { return pc_off() + (size_t)n_pcost * sizeof(double4); }
  __host__ __device__ size_t tr_off() const { return tt_off() + (size_t)n_thr * sizeof(double); }
  __host__ __device__ size_t bytes() const { return tr_off() + (size_t)n_throw * sizeof(int); }
};

constexpr int kClusterCtas = 8;
constexpr int kClusterThreads = 256;

__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(kClusterThreads, 1)
    dp_cluster_kernel(DpArgs a, DpScalars S, ClusterLayout G) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  __shared__ int s_idx[kClusterThreads];
  __shared__ int s_path[kMaxHorizon + 1];
  extern __shared__ __align__(16) unsigned char sm_raw[];
  NodeCfg* s_cfg = reinterpret_cast<NodeCfg*>(sm_raw + G.cfg_off());
  LevelDesc* s_lv = reinterpret_cast<LevelDesc*>(sm_raw + G.lv_off());
  NodeCost* s_nc = reinterpret_cast<NodeCost*>(sm_raw + G.nc_off());
  double2* s_vm = reinterpret_cast<double2*>(sm_raw + G.vm_off());
  int* s_base = reinterpret_cast<int*>(sm_raw + G.base_off());
  double* s_prob = reinterpret_cast<double*>(sm_raw + G.prob_off());
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = kClusterThreads / 32;
  auto stamp = [&](int slot) {  // LIVEPUT_DP_TRACE: per-CTA globaltimer stamps
    if (a.trace && threadIdx.x == 0 && slot < 2 * kTraceLevels + 2) {
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      a.trace[(size_t)rank * (2 * kTraceLevels + 2) + slot] = t;
    }
  };
  stamp(0);

  // tables, in one pass of independent loads: node list, level descriptors,
  // per-depth cost terms and the throughput table; then every next-role
  // node's cost terms from shared memory (level 0's `current` is never a
  // next node, and its depth may have no throughput or cost row)
  double4* s_pc = reinterpret_cast<double4*>(sm_raw + G.pc_off());
  double* s_tt = reinterpret_cast<double*>(sm_raw + G.tt_off());
  int* s_tr = reinterpret_cast<int*>(sm_raw + G.tr_off());
  // every prev row the DP reads, gathered by the host-built offset list in
  // the same pass of independent loads when no histogram of this re-plan is
  // fresh (a warm re-plan), else after the normalisation below
  auto stage_rows = [&]() {
    for (int e = threadIdx.x; e < G.n_prob; e += blockDim.x) {
      const int src = a.gather[e];
      s_prob[e] = src >= 0 ? __ldcg(a.store + src) : 0.0;
    }
  };
  if (a.n_entries == 0) stage_rows();
  for (int j = threadIdx.x; j <= G.horizon; j += blockDim.x) s_base[j] = a.pbase[j];
  for (int i = threadIdx.x; i < G.n_nodes; i += blockDim.x) s_cfg[i] = a.cfg[i];
  for (int j = threadIdx.x; j < G.horizon; j += blockDim.x) s_lv[j] = a.levels[j];
  for (int i = threadIdx.x; i < G.n_pcost; i += blockDim.x) s_pc[i] = a.pcost[i];
  for (int i = threadIdx.x; i < G.n_thr; i += blockDim.x) s_tt[i] = a.thr_tab[i];
  for (int i = threadIdx.x; i < G.n_throw; i += blockDim.x) s_tr[i] = a.thr_row[i];
  __syncthreads();
  const int first_next = s_lv[0].next_base;
  for (int i = threadIdx.x; i < G.n_nodes; i += blockDim.x) {
    const NodeCfg nx = s_cfg[i];
    NodeCost nc{0.0, 0.0, 0.0, 0.0};
    if (nx.d > 0 && i >= first_next) {
      const double4 pc = s_pc[nx.p];
      nc.thr = s_tt[s_tr[nx.p] + nx.d];
      nc.pipe = pc.x;
      nc.unit = pc.y;
      nc.resume = pc.z;
    }
    s_nc[i] = nc;
  }
  if (threadIdx.x == 0) s_vm[0] = make_double2(0.0, 0.0);  // level 0: value 0, migration 0
  // phase 0: probabilities of the fresh entries, split over the cluster
  for (int e = rank; e < a.n_entries; e += kClusterCtas) {
    const EntryDesc en = a.entries[e];
    const PairDesc pd = a.pairs[en.pair];
    const int len = hist_row(en.Dmax + 1, pd.k);
    const double total = static_cast<double>(pd.count);
    double* out = a.store + a.store_off[e];
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      const uint32_t c = a.hist[en.hist_off + i];
      out[i] = c ? __ddiv_rn(static_cast<double>(c), total) : 0.0;
    }
  }
  if (a.n_entries > 0) {
    __threadfence();
    cluster.sync();  // the store is complete (every CTA's normalisation)
    stage_rows();
    __syncthreads();
  } else {
    cluster.sync();  // every CTA runs before any DSMEM store reaches it
  }

  // levels: one warp per next node
  stamp(1);
  for (int j = 0; j < G.horizon; ++j) {
    const LevelDesc L = s_lv[j];
    const int stride = min(L.k, L.n_now) + 1;
    for (int nb = rank * nwarps + warp; nb < L.next_count; nb += kClusterCtas * nwarps) {
      const int ni = L.next_base + nb;
      const NodeCfg nx = s_cfg[ni];
      const NodeCost nc = s_nc[ni];
      const PhiConst K = phi_const(L, S, nc);
      Cand best{0.0, 0.0, 0.0, 0.0, -1};
      for (int pi = lane; pi < L.prev_count; pi += 32) {
        const int gi = L.prev_base + pi;
        const NodeCfg pv = s_cfg[gi];
        const PhiOut ph = phi_dev(pv, nx, nc, L, S, ProbPtr{s_prob + s_base[j] + pi * stride}, s_tt, s_tr, K);
        const double2 vm = s_vm[gi];
        const double v = __dadd_rn(vm.x, ph.committed);
        const double mg = __dadd_rn(vm.y, ph.mig);
        if (best.idx < 0 || v > best.value ||
            (v == best.value && (mg < best.mig || (mg == best.mig && pi < best.idx)))) {
          best.value = v;
          best.mig = mg;
          best.stc = ph.committed;
          best.stm = ph.mig;
          best.idx = pi;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const Cand o = shfl_cand(best, lane ^ off);
        if (cand_better(o, best)) best = o;
      }
      // every lane holds the winner: lanes 0..kClusterCtas-1 store (F, M)
      // into their CTA's table; lane 0 also writes the traceback terms
      if (lane < kClusterCtas) {
        double2* dst = cluster.map_shared_rank(s_vm, lane);
        dst[ni] = make_double2(best.value, best.mig);
      }
      if (lane == 0) {
        __stcg(a.val + ni, best.value);
        __stcg(a.mig + ni, best.mig);
        __stcg(a.parent + ni, best.idx);
        __stcg(a.stc + ni, best.stc);
        __stcg(a.stm + ni, best.stm);
      }
    }
    // barrier.cluster arrive.release / wait.acquire orders the DSMEM stores;
    // the global back-pointers are fenced once, before the last barrier
    if (j + 1 == G.horizon) __threadfence();
    stamp(2 + 2 * j);
    cluster.sync();
    stamp(3 + 2 * j);
  }

  // final pick (rank = (value, -mig, D, -P), suspended as (-1, 0), first
  // index wins) and traceback, by CTA 0
  if (rank != 0) return;
  const LevelDesc last = s_lv[G.horizon - 1];
  const int base = last.next_base, cnt = last.next_count;
  auto gt = [&](int x, int y) -> bool {  // rank(x) > rank(y)
    if (y < 0) return x >= 0;
    if (x < 0) return false;
    const double va = s_vm[base + x].x, vb = s_vm[base + y].x;
    if (vb < va) return true;
    if (va < vb) return false;
    const double ma = -s_vm[base + x].y, mb = -s_vm[base + y].y;
    if (mb < ma) return true;
    if (ma < mb) return false;
    const NodeCfg ca = s_cfg[base + x], cb = s_cfg[base + y];
    const int da = ca.d > 0 ? ca.d : -1, db = cb.d > 0 ? cb.d : -1;
    if (db < da) return true;
    if (da < db) return false;
    const int pa = ca.d > 0 ? -ca.p : 0, pb = cb.d > 0 ? -cb.p : 0;
    return pb < pa;
  };
  int mine = -1;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x)
    if (gt(i, mine)) mine = i;  // ascending i: strict > keeps the first
  s_idx[threadIdx.x] = mine;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      const int x = s_idx[threadIdx.x], y = s_idx[threadIdx.x + st];
      if (gt(y, x) || (y >= 0 && x >= 0 && !gt(x, y) && y < x)) s_idx[threadIdx.x] = y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int idx = s_idx[0];
    if (a.final_value) *a.final_value = s_vm[base + idx].x;
    for (int jj = G.horizon; jj >= 1; --jj) {
      const int gi = s_lv[jj - 1].next_base + idx;
      s_path[jj] = gi;
      idx = __ldcg(a.parent + gi);
    }
  }
  __syncthreads();
  for (int jj = 1 + threadIdx.x; jj <= G.horizon; jj += blockDim.x) {
    const int gi = s_path[jj];
    const NodeCfg c = s_cfg[gi];
    lp_plan_step st;
    st.interval_index = jj;
    st.config.pipelines = c.d > 0 ? c.d : 0;
    st.config.stages = c.d > 0 ? c.p : 0;
    st.expected_committed = __ldcg(a.stc + gi);
    st.expected_mig_cost_s = __ldcg(a.stm + gi);
    a.plan[jj - 1] = st;
  }
}

size_t dp_cluster_smem(int n_nodes, int horizon, int n_prob, int n_pcost, int n_throw, int n_thr) {
  return ClusterLayout{n_nodes, horizon, n_prob, n_pcost, n_throw, n_thr}.bytes();
}

cudaError_t launch_dp_cluster(cudaStream_t st, const DpArgs& a, const DpScalars& S, int n_nodes, int n_prob,
                              int n_pcost, int n_throw, int n_thr) {
  if (a.horizon > kMaxHorizon) return cudaErrorInvalidValue;
  const ClusterLayout G{n_nodes, a.horizon, n_prob, n_pcost, n_throw, n_thr};
  const size_t smem = G.bytes();
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(dp_cluster_kernel), smem);
  if (e != cudaSuccess) return e;
  dp_cluster_kernel<<<kClusterCtas, kClusterThreads, smem, st>>>(a, S, G);
  return cudaGetLastError();
}

void preload_dp() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, normalize_kernel);
  cudaFuncGetAttributes(&a, dp_step_kernel);
  cudaFuncGetAttributes(&a, dp_final_kernel);
  cudaFuncGetAttributes(&a, liveput_kernel);
  cudaFuncGetAttributes(&a, dp_persistent_kernel<true>);
  cudaFuncGetAttributes(&a, dp_persistent_kernel<false>);
  cudaFuncGetAttributes(&a, dp_cluster_kernel);
}

}  // namespace lp
