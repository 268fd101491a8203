// lp_launch.h — host-callable launch wrappers of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include "liveput.h"
#include "lp_layout.h"

namespace lp {

// Raise a kernel's dynamic shared-memory opt-in once per (device, kernel).
cudaError_t smem_optin(const void* fn, size_t smem);

// Load the default path's kernels on the current device (once per process
// and device, from lp_create): lazy module loading would otherwise load each
// inside the first re-plan that launches it.
void preload_kernels();
void preload_rows();
void preload_bits();
void preload_hist();
void preload_dp();

cudaError_t launch_hist_regs(int kmax, bool smem_evt, int blocks, size_t smem, cudaStream_t st,
                             const WorkItem* w, const PairDesc* pairs, const EntryDesc* ents,
                             const DrawConst* dr, const uint64_t* binom, uint32_t* evt,
                             uint32_t* h0);
cudaError_t launch_hist_ctr(bool smem_evt, int blocks, int threads, size_t smem, int pmax_cap,
                            cudaStream_t st, const WorkItem* w, const PairDesc* pairs,
                            const EntryDesc* ents, const DrawConst* dr, const uint64_t* binom,
                            uint32_t* evt, uint32_t* h0);
cudaError_t launch_hist_scn(int kreg, bool smem_evt, int blocks, int threads, size_t smem, int uw,
                            cudaStream_t st, const WorkItem* w, const PairDesc* pairs,
                            const EntryDesc* ents, const DrawConst* dr, const uint64_t* binom,
                            uint32_t* evt, uint32_t* h0);
cudaError_t launch_hist_inc(int kmax, bool smem_evt, int blocks, int threads, size_t smem,
                            cudaStream_t st, const WorkItem* w, const PairDesc* pairs,
                            const EntryDesc* ents, const DrawConst* dr, const uint64_t* binom,
                            const uint16_t* divtab, uint32_t* evt, uint32_t* h0);
// n > kBigN: every per-thread array in a global scratch slice (lp_hist_big.cu)
constexpr int kBigN = 2048;
constexpr int kBigThreads = 64;
size_t big_scratch_words(int n, int k, int pmax);
cudaError_t launch_hist_big(int n_items, int grid, cudaStream_t st, const WorkItem* w, const PairDesc* pairs,
                            const EntryDesc* ents, const DrawConst* dr, const uint64_t* binom, uint32_t* evt,
                            uint32_t* h0, uint32_t* scratch, size_t per_thread);
cudaError_t launch_hist_bits(int kmax, bool smem_evt, int blocks, int threads, size_t smem,
                             cudaStream_t st, const WorkItem* w, const PairDesc* pairs,
                             const EntryDesc* ents, const DrawConst* dr, const uint64_t* binom,
                             const uint32_t* dmask, uint32_t* evt, uint32_t* h0);
cudaError_t launch_hist_rows(int kreg, int wmax, bool smem_evt, int blocks, int threads,
                             size_t smem, cudaStream_t st, const WorkItem* w,
                             const PairDesc* pairs, const EntryDesc* ents, const DrawConst* dr,
                             const uint64_t* binom, uint32_t* evt, uint32_t* h0);
// per-block WorkItems of the histogram launches from the uploaded spans
cudaError_t launch_expand_work(const WorkSpan* spans, int n_spans, int n_work, WorkItem* out, cudaStream_t st);
cudaError_t launch_finalize_range(int p0, int n_pairs, int e0, int n_entries, cudaStream_t st,
                                  const PairDesc* pairs, const EntryDesc* ents, uint32_t* evt,
                                  uint32_t* h0, uint32_t* hist);
cudaError_t launch_finalize(int n_pairs, int n_entries, cudaStream_t st, const PairDesc* pairs,
                            const EntryDesc* ents, uint32_t* evt, uint32_t* h0, uint32_t* hist);
cudaError_t launch_dump(int n, int k, int exact, int trials, uint64_t seed, const DrawConst* dc,
                        const uint64_t* binom, int binom_stride, uint32_t* gscratch,
                        uint16_t* sorted_out, const int2* cfgs, int n_cfg, uint16_t* m_out,
                        cudaStream_t st);

// pdl: programmatic dependent launch on the previous level's kernel
cudaError_t launch_dp_step(int j, int next_count, int prev_count, bool pdl, cudaStream_t st,
                           const LevelDesc* levels,
                           const NodeCfg* cfg, const double4* pcost, const double* histp,
                           const double* thr_tab, const int32_t* thr_row, const DpScalars& S,
                           double* val, double* mig, int32_t* parent, double* stc, double* stm);
// Materialised phi (pipelined re-plans): every (next, prev) pair of the
// levels in lv_list[0..n_levels), then the per-level max-plus pass over it.
cudaError_t launch_phi_matrix(int n_levels, int64_t max_pairs, cudaStream_t st, const int32_t* lv_list,
                              const LevelDesc* levels, const NodeCfg* cfg, const double4* pcost,
                              const double* histp, const double* thr_tab, const int32_t* thr_row,
                              const DpScalars& S, double2* phi);
cudaError_t launch_dp_maxplus(int j, int next_count, bool pdl, cudaStream_t st, const LevelDesc* levels,
                              const double2* phi, double* val, double* mig, int32_t* parent, double* stc,
                              double* stm);
cudaError_t launch_normalize(int n_entries, cudaStream_t st, const PairDesc* pairs,
                             const EntryDesc* ents, const uint32_t* hist, const int32_t* store_off,
                             double* store);
// n_nodes > 0: stage every back-pointer in shared memory for the walk
cudaError_t launch_dp_final(int horizon, cudaStream_t st, const LevelDesc* levels,
                            const NodeCfg* cfg, const double* val, const double* mig,
                            const int32_t* parent, const double* stc, const double* stm,
                            lp_plan_step* plan, double* final_value, int n_nodes = 0);
cudaError_t launch_liveput(int n_rows, cudaStream_t st, const int4* rows, const LevelDesc* levels,
                           const NodeCfg* cfg, const uint32_t* hist, const double* probs,
                           const double* thr_tab, const int32_t* thr_row, lp_liveput_row* out);
cudaError_t launch_phi_single(const NodeCfg& pv, const NodeCfg& nx, const NodeCost& nc,
                              const LevelDesc& L, const DpScalars& S, const uint32_t* hist,
                              const double* thr_tab, const int32_t* thr_row, double* out2,
                              cudaStream_t st);

// Persistent DP (lp_dp.cu): normalisation, every level step, the final pick
// and the traceback in one cooperative launch.
struct DpArgs {
  const LevelDesc* levels;
  const NodeCfg* cfg;
  const double4* pcost;
  const double* thr_tab;
  const int32_t* thr_row;
  // normalisation (count / total into the probability store)
  const PairDesc* pairs;
  const EntryDesc* entries;
  const uint32_t* hist;
  const int32_t* store_off;
  int n_entries;
  double* store;
  // DP state
  double* val;
  double* mig;
  int32_t* parent;
  double* stc;
  double* stm;
  lp_plan_step* plan;
  double* final_value;
  uint32_t* barrier;
  int horizon;
  int max_next;     // largest next-level node count: the blocks that run the levels
  uint64_t* trace;  // optional: per block, 2 * kTraceLevels + 2 globaltimer stamps
  // cluster DP: per staged probability element its store offset (-1: +0.0),
  // and each level's first element (horizon + 1), both built on the host
  const int32_t* gather;
  const int32_t* pbase;
};
constexpr int kTraceLevels = 32;

// n_prob >= 0: the shared-memory staged variant (small re-plans); n_prob =
// sum over hist levels of prev_count * (min(k, n_now) + 1), n_nodes = all DP nodes.
cudaError_t launch_dp_persistent(int device, int num_sms, int max_next, cudaStream_t st,
                                 const DpArgs& a, const DpScalars& S, int n_nodes = 0, int n_prob = -1);
size_t dp_staged_smem(int n_nodes, int horizon, int n_prob);

// Cluster DP (lp_dp.cu): one 8-CTA thread-block cluster, levels separated by
// barrier.cluster, level values exchanged through distributed shared memory;
// small re-plans whose whole DP input fits one CTA's shared memory.
cudaError_t launch_dp_cluster(cudaStream_t st, const DpArgs& a, const DpScalars& S, int n_nodes, int n_prob,
                              int n_pcost, int n_throw, int n_thr);
size_t dp_cluster_smem(int n_nodes, int horizon, int n_prob, int n_pcost, int n_throw, int n_thr);

}  // namespace lp
