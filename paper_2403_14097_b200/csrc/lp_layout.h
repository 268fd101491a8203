// lp_layout.h — POD tables shared by the host planner and the sm_100a kernels.
//
// HBM layout of one re-plan (all offsets are element indices into the
// handle's flat device buffers):
//
//   pairs[]    one PairDesc per distinct (n, k) scenario ensemble
//   entries[]  one EntryDesc per (pair, pipeline depth P): the configs
//              (1..Dmax, P) whose survivor histograms the ensemble feeds
//   draws[]    per (pair, draw i) constants of Rng::below(n - i)
//   evt[]      u32 threshold-event counters  evt[e][t-2][x]
//   h0[]       u32 histogram of the smallest preempted slot, per pair
//   hist[]     u32 final survivor-deficit histograms hist[e][D][d]
//   levels     DP node tables (config, throughput, costs) and the
//              value / migration / back-pointer arrays the DP writes
#pragma once

#include <stdint.h>

namespace lp {

constexpr int kMaxN = 16384;    // instances per availability count (u16 slot ids; > 2048: lp_hist_big.cu)
constexpr int kMaxKReg = 16;    // register-resident scenarios (variant R)
constexpr int kMaxK = 255;      // u8 class counters (variant C)
constexpr int kComb = 4;        // scenario-major kernel: Dmax <= kComb uses the bitmap comb

struct PairDesc {
  int32_t n, k;
  int32_t exact;        // 1: lexicographic enumeration, 0: Monte-Carlo
  int32_t n_entries;
  int32_t entry_base;   // first EntryDesc of this pair
  int32_t h0_off;       // n counters
  int32_t draw_off;     // k DrawConst (MC)
  int32_t binom_off;    // exact: (n+1) x binom_stride saturated binomials
  int32_t binom_stride; // min(k, n-k) + 1
  int32_t variant;      // 0: register kernel (k <= 16), 1: counter kernel
  uint64_t seed;        // mix_seed(mix_seed(mc_seed, n), k)
  uint64_t count;       // ensemble size over all ranks
  uint64_t t_lo, t_hi;  // this rank's slice of the ensemble
};

struct EntryDesc {
  int32_t P;
  int32_t Dmax;
  int32_t lim;          // P * Dmax: slots beyond are spares for every config of this depth
  uint32_t magic;       // floor(2^32 / P) + 1 (P >= 2); exact floor(s / P) for s < 2^20
  int32_t evt_off;      // evt[evt_off + (t-2)*Dmax + x], t = 2..tmax
  int32_t tmax;         // min(k, Dmax)
  int32_t hist_off;     // hist row of D = 1
  int32_t pair;
};

// Rng::below(b) for b = n - i (rng.hpp:23-30): reject r >= lim, return r % b.
struct DrawConst {
  uint64_t lim;         // UINT64_MAX - UINT64_MAX % b
  uint32_t m32;         // Barrett multiplier floor(2^32 / b) (2^32 - 1 for b = 1)
  uint32_t negb;        // 2^32 - b
  uint32_t c32;         // 2^32 mod b
  uint32_t b;
};

// One block's share of the histogram work.
struct WorkItem {
  int32_t pair;
  int32_t e_lo, e_hi;   // entry range [e_lo, e_hi) (absolute indices)
  int32_t evt_lo;       // evt offset of e_lo
  int32_t evt_len;      // evt counters of the range (staged in shared memory)
  int32_t smem_evt;     // 1: stage evt in shared memory, 0: global atomics
  int32_t e_res_hi;     // entries [e_lo, e_res_hi) can emit t >= 2 events (Dmax >= 2)
  int32_t dtab_off;     // incidence kernel: divisor table (u16) of this entry range
  int32_t dtab_len;     //   [n+1 CSR offsets][local depth indices]
  int32_t pad;
  uint64_t t0, t1;      // scenario range
};

// A run of consecutive blocks over one scenario range: block first + b
// takes scenarios [w.t0 + b * chunk, min(w.t1, w.t0 + (b + 1) * chunk)).
// The host uploads the spans (a few per ensemble) and one kernel expands
// them into per-block WorkItems on the device.
struct WorkSpan {
  WorkItem w;           // t0 / t1: the whole range
  uint64_t chunk;
  int32_t first;        // first block
  int32_t pad;
};

// Row offset of D inside an entry's histogram block: rows hold
// d = 0..min(k, D) (m = D - d).
__host__ __device__ inline int32_t hist_row(int32_t D, int32_t k) {
  const int32_t a = D - 1;  // rows before D
  if (a <= k) return a * (a + 1) / 2 + a;
  return k * (k + 1) / 2 + k + (a - k) * (k + 1);
}

// DP node (one config at one level).  d == 0 -> suspended.
struct NodeCfg {
  int32_t d, p;
  int32_t hist_off;     // prev role: histogram row (absolute), -1 if none
  int32_t pad;
};

struct NodeCost {       // next role: FP64 constants of phi (optimizer.cpp:96-138)
  double thr;           // throughput(next)
  double pipe;          // pipeline_transfer_s(next.P)
  double unit;          // inter_transfer unit for next.P
  double resume;        // resume_cost(next)
};

struct LevelDesc {
  int32_t n_now, n_next, k;
  int32_t prev_base, prev_count;   // node range of level j (prev)
  int32_t next_base, next_count;   // node range of level j+1
  int32_t fresh;                   // n_next > n_now
  int32_t has_hist;
  int32_t phi_off;                 // materialised phi: first (next, prev) pair, in double2
  uint64_t total;                  // ensemble size of the level's pair
  double fixed;                    // fresh > 0 ? fresh_fixed : 0.0
};

constexpr int kMaxHorizon = 1024;  // persistent DP's traceback buffer

struct DpScalars {
  double T;
  double build, update;
  double rollback;
  double fresh_fixed;
  int32_t strict;
  int32_t horizon;
};

}  // namespace lp
