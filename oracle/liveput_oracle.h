/*
 * liveput_oracle.h — CPU ORACLE (test infrastructure; the checker, never the
 * product).  A plain-C restatement of the reference's planning hot path:
 *
 *   splitmix64 Rng / mix_seed / below     rng.hpp:11-55
 *   sample_distinct                       rng.cpp:8-19
 *   scenario_count / enumerate_vectors /
 *   sample_vectors / stage_survivors      preemption.cpp:10-66
 *   depth_feasible / throughput /
 *   enumerate_configs                     perf_model.cpp:5-52
 *   transition_outcome_min / resume_cost  migration.cpp:22-104
 *   survivor_histogram / phi / dp_optimize /
 *   sequence_value / reactive_plan        optimizer.cpp:11-219
 *
 * Differences from the reference, on purpose: no phi/histogram caches (so
 * no key aliasing at D or P >= 257, optimizer.cpp:39-50), histograms are
 * computed scenario-major (each sampled vector is generated once and tallied
 * against every config), and the MC trial loop runs on `threads` pthreads
 * (integer counts, so the split is exact).
 *
 * Pinned against the compiled reference (oracle/_ref) and the golden vectors
 * in tests/golden/ by tests/test_oracle.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load liboracle.so.
 */
#ifndef LIVEPUT_ORACLE_H_
#define LIVEPUT_ORACLE_H_

#include <stdint.h>

#include "../include/liveput.h"

#ifdef __cplusplus
extern "C" {
#endif

uint64_t or_splitmix_next(uint64_t* state);
uint64_t or_mix_seed(uint64_t a, uint64_t b);
uint64_t or_below(uint64_t* state, uint64_t bound);
void or_sample_distinct(int n, int k, uint64_t seed, int* out);
uint64_t or_scenario_count(int n, int k);

int or_depth_feasible(const lp_profile* w, int stages);
double or_throughput(const lp_profile* w, int d, int p);
int or_enumerate_configs(const lp_profile* w, int n, int* out_dp, int cap);
int or_reactive_plan(const lp_profile* w, int n, int* out_dp);

/* returns cost; *rollback set; return kind via *kind (0 none,1 intra,2 inter,3 pipeline) */
double or_transition_cost(int m, int sd, int sp, int td, int tp, int fresh, const lp_profile* w,
                          const lp_costs* c, int* rollback, int* kind);
double or_resume_cost(int tp, const lp_profile* w, const lp_costs* c);

/* Sampled (or enumerated, exact != 0) scenarios as sorted index lists,
 * trials x k ints.  For exact, trials must equal C(n, k). */
int or_scenarios(int n, int k, int exact, int trials, uint64_t seed, int* out_sorted);

/* Survivor-minimum counts for each of n_cfg configs over one ensemble.
 * counts is n_cfg x (max_d + 1) uint64 with row stride `stride` (>= D+1),
 * indexed by m.  *total = ensemble size.  Returns 0, or -1 on bad input. */
int or_ensemble_counts(int n, int k, int exact, int trials, uint64_t seed, const int* cfg_dp,
                       int n_cfg, uint64_t* counts, int stride, uint64_t* total, int threads);

int or_ensemble_counts_range(int n, int k, int exact, int trials, uint64_t seed, const int* cfg_dp,
                             int n_cfg, uint64_t* counts, int stride, uint64_t* total, int threads,
                             long long r0, long long r1);

/* Planner-equivalent entry points (PlannerOptions semantics, exact_cap
 * switch and seed derivation of optimizer.cpp:64-94). */
typedef struct or_planner or_planner;
or_planner* or_planner_new(const lp_profile* w, const lp_costs* c, const lp_options* o,
                           int threads);
void or_planner_free(or_planner* pl);
/* opt-in memo of full-level ensembles per (n_now, k) for long replays (the
 * reference's hist_cache_); results are identical with it on or off */
void or_planner_set_cache(or_planner* pl, int on);
const char* or_last_error(void);
int or_survivor_counts(or_planner* pl, int d, int p, int n_now, int n_minus, uint64_t* counts,
                       uint64_t* total);
int or_phi(or_planner* pl, int pd, int pp, int nd, int np, int n_now, int n_next, double* out2);
int or_dp_optimize(or_planner* pl, int cd, int cp, const int* n_seq, int len, int* cfg_out,
                   double* val_out, double* final_value);
int or_sequence_value(or_planner* pl, int cd, int cp, const int* seq_dp, const int* n_seq,
                      int len, double* out);
int or_liveput(or_planner* pl, int d, int p, int n_now, int n_minus, double* out);

#ifdef __cplusplus
}
#endif
#endif
