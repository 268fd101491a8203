/*
 * liveput.h — C ABI of the B200-native liveput planner (Parcae, arxiv 2403.14097).
 *
 * Drop-in boundary for the reference's planning hot path, `spotsim::Planner`
 * (/root/reference/proj/core/include/spotsim/optimizer.hpp:41-92) and the free
 * functions it sits on.  Every entry point below names the reference symbol it
 * replaces.  Plain C types only: no torch, no C++ in the signatures.
 *
 * Conventions
 *   - Every call returns an lp_status; LP_OK == 0.  Failures store a message
 *     retrievable with lp_last_error(handle) (or lp_last_global_error() for
 *     calls that have no handle).  The C++/Python facades map LP_EINVAL to
 *     std::invalid_argument / ValueError, matching the reference's exceptions.
 *   - A config with pipelines == 0 is the suspended state (the reference's
 *     std::nullopt, optimizer.hpp:25).
 *   - All buffers are caller-owned host memory unless the name says "_dev".
 *   - One handle = one CUDA device, one stream, one host thread at a time
 *     (the reference Planner is not thread-safe either, optimizer.hpp:38-40).
 */
#ifndef LIVEPUT_H_
#define LIVEPUT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LP_OK = 0,
  LP_EINVAL = 1,       /* bad argument; reference throws std::invalid_argument */
  LP_ECUDA = 2,        /* CUDA runtime failure */
  LP_ENOMEM = 3,       /* device or host allocation failed */
  LP_EUNSUPPORTED = 4, /* outside the sizes this build supports */
  LP_ENCCL = 5,        /* NCCL failure */
  LP_EROLLBACK = 6     /* plan_migration: a stage lost every replica (RollbackRequired,
                          migration.hpp:49-51) */
} lp_status;

/* ParallelConfig (perf_model.hpp:10-16). pipelines == 0 -> suspended. */
typedef struct {
  int32_t pipelines; /* D */
  int32_t stages;    /* P */
} lp_config;

/* WorkloadProfile (perf_model.hpp:26-49).  pipeline_rates is passed as two
 * parallel arrays (depth, samples/s); n_rates may be 0. */
typedef struct {
  double compute_per_microbatch_s;
  double param_bytes;
  double activation_bytes;
  int32_t minibatch_size;
  int32_t microbatch_size;
  double device_memory_bytes;
  double memory_fixed_bytes;     /* MemoryModel::fixed_bytes */
  double memory_per_stage_bytes; /* MemoryModel::per_stage_bytes */
  double alpha_s;
  double beta_s_per_byte;
  int32_t n_rates;
  const int32_t* rate_depths;
  const double* rate_values;
} lp_profile;

/* CostTable (migration.hpp:16-27). */
typedef struct {
  double start_process_s;
  double rendezvous_s;
  double cuda_context_s;
  double load_data_s;
  double build_model_s;
  double update_comm_groups_s;
} lp_costs;

/* PlannerOptions (optimizer.hpp:13-23). */
typedef struct {
  double interval_s;
  int32_t lookahead;
  int32_t mc_trials;
  uint64_t exact_cap;
  uint64_t mc_seed;
  double rollback_penalty_s;
  int32_t strict_conditional;
} lp_options;

/* PlanStep (optimizer.hpp:26-31). */
typedef struct {
  int32_t interval_index;
  lp_config config;
  double expected_committed;
  double expected_mig_cost_s;
} lp_plan_step;

/* One row of the liveput table produced by a re-plan: the expected surviving
 * throughput of `config` over interval `interval` (n_now -> n_next), i.e. the
 * reference's expected_liveput (preemption.cpp:94-112) evaluated on the
 * planner's scenario ensemble. */
typedef struct {
  int32_t interval; /* j: the transition n_seq[j] -> n_seq[j+1] */
  lp_config config;
  double liveput;
} lp_liveput_row;

/* Counters of the last lp_replan / lp_execute on this handle. */
typedef struct {
  uint64_t resolutions;      /* (scenario, prev-config) resolutions = reference tally() calls */
  uint64_t scenarios;        /* distinct sampled/enumerated scenarios (all ranks) */
  uint64_t local_scenarios;  /* scenarios this rank generated */
  int32_t mc_pairs;          /* distinct (n, k) Monte-Carlo pairs */
  int32_t exact_pairs;       /* distinct (n, k) exactly-enumerated pairs */
  int32_t kernel_launches;   /* kernels launched by the last execute */
  int32_t horizon;
  double hist_ms;            /* device time of histogram kernels (CUDA events) */
  double reduce_ms;          /* device time of the cross-rank histogram reduce */
  double dp_ms;              /* device time of the DP kernels */
  double total_ms;           /* device time of the whole execute */
  uint64_t hist_alg_ops;     /* int32-equivalent ops of the resolution algorithms as run:
                                scenario generation 20 + 35k, the bits kernel's slot-pair
                                lookups / bit-sliced adds / row compares, the row kernel's
                                Dmax x ceil(P/32) x (3B+4) per depth */
  uint64_t h2d_bytes;        /* bytes copied host->device by the last prepare */
  uint64_t d2h_bytes;        /* bytes copied device->host by the last fetch */
  double prepare_ms;         /* host wall time of the last lp_prepare (tables + H2D issue) */
  uint64_t cached_pairs;     /* (n, k) ensembles served from the histogram cache */
  uint64_t hist_survey_ops;  /* SURVEY.md §8d's reference-equivalent model: per scenario
                                S(k) = 20 + 35k plus R(k) = 6k per depth */
} lp_stats;

typedef struct lp_handle lp_handle;

/* ---- handle lifecycle: Planner(WorkloadProfile, CostTable, PlannerOptions)
 *      optimizer.hpp:43 / optimizer.cpp:27-28 ---------------------------- */
lp_status lp_create(const lp_profile* profile, const lp_costs* costs, const lp_options* options,
                    int32_t device, lp_handle** out);
void lp_destroy(lp_handle* h);
const char* lp_last_error(const lp_handle* h);
const char* lp_last_global_error(void);
lp_status lp_get_options(const lp_handle* h, lp_options* out);

/* ---- the hot path: Planner::dp_optimize (optimizer.hpp:64-65,
 *      optimizer.cpp:140-205).  n_seq has len >= 2 entries; out has len-1
 *      steps.  liveput_out (nullable) receives up to liveput_cap rows; the row
 *      count is written to *liveput_rows (nullable). ----------------------- */
lp_status lp_replan(lp_handle* h, lp_config current, const int32_t* n_seq, int32_t len,
                    lp_plan_step* out, lp_liveput_row* liveput_out, int32_t liveput_cap,
                    int32_t* liveput_rows);

/* lp_replan split in three so that device-resident throughput can be timed:
 * prepare = host tables + one H2D upload, execute = kernels only (cold:
 * recomputes every histogram), fetch = one D2H of the plan. */
lp_status lp_prepare(lp_handle* h, lp_config current, const int32_t* n_seq, int32_t len);
lp_status lp_execute(lp_handle* h);
lp_status lp_fetch(lp_handle* h, lp_plan_step* out, lp_liveput_row* liveput_out,
                   int32_t liveput_cap, int32_t* liveput_rows);
lp_status lp_get_stats(const lp_handle* h, lp_stats* out);
/* The CUDA stream every kernel of this handle runs on (cudaStream_t as void*). */
void* lp_stream(lp_handle* h);

/* ---- device-resident histogram cache across re-plans: the reference's
 *      hist_cache_ (optimizer.hpp:88, optimizer.cpp:64-71).  Off by default,
 *      so every lp_execute is a cold re-plan that recomputes every ensemble.
 *      When on, an (n, k) ensemble computed by an earlier re-plan of this
 *      handle is reused (results are identical: they depend only on the key).
 *      max_bytes bounds the device store; when full it is dropped and refilled. */
lp_status lp_set_hist_cache(lp_handle* h, int32_t enable, uint64_t max_bytes);

/* ---- offline liveput tables ("sampling can be done
 *      offline").  lp_precompute samples every config of n at
 *      each (n[i], k[i]) into the device cache (turning the cache on), so a
 *      later re-plan over those availability steps is DP-only.  The cache can
 *      be serialised (lp_cache_export: call with buf = NULL for the size) and
 *      restored into another handle with the same sampling options
 *      (mc_trials, exact_cap, mc_seed); histograms do not depend on the
 *      profile or the cost table. */
lp_status lp_precompute(lp_handle* h, const int32_t* n, const int32_t* k, int32_t count);
lp_status lp_cache_export(lp_handle* h, void* buf, uint64_t cap, uint64_t* len);
lp_status lp_cache_import(lp_handle* h, const void* buf, uint64_t len);

/* ---- Planner::phi (optimizer.hpp:57-58, optimizer.cpp:52-62, 96-138) ---- */
lp_status lp_phi(lp_handle* h, lp_config prev, lp_config next, int32_t n_now, int32_t n_next,
                 double* committed, double* mig_cost_s);

/* ---- Planner::sequence_value (optimizer.hpp:69-71, optimizer.cpp:207-219) */
lp_status lp_sequence_value(lp_handle* h, lp_config current, const lp_config* sequence,
                            const int32_t* n_seq, int32_t len, double* out);

/* ---- Planner::survivor_histogram (optimizer.cpp:64-94), un-normalised:
 *      counts[m] for m = 0..D (D+1 entries), *total = scenario count.  ---- */
lp_status lp_survivor_hist(lp_handle* h, lp_config prev, int32_t n_now, int32_t n_minus,
                           uint64_t* counts, uint64_t* total);

/* ---- expected_liveput with EvalMode (preemption.hpp:53-65,
 *      preemption.cpp:94-112).  exact != 0 -> enumerate_vectors, else
 *      sample_vectors(n, n_minus, trials, seed).  FP64; agrees with the
 *      reference to ~1e-15 relative (summation order differs). ---------- */
lp_status lp_expected_liveput(lp_handle* h, lp_config cfg, int32_t n, int32_t n_minus,
                              int32_t exact, int32_t trials, uint64_t seed, double* out);

/* ---- parity mode: per-(trial, config) survivor minimum m of
 *      sample_vectors/enumerate_vectors + stage_survivors
 *      (preemption.cpp:23-66).  out is trials x n_cfg, row-major (trial-major),
 *      uint16 m.  exact != 0 -> trials must equal C(n, n_minus) and trial t is
 *      the t-th vector of enumerate_vectors (lexicographic).  ------------- */
lp_status lp_dump_survivors(lp_handle* h, int32_t n, int32_t n_minus, int32_t exact,
                            int32_t trials, uint64_t seed, const lp_config* cfgs, int32_t n_cfg,
                            uint16_t* out);

/* ---- parity mode: the sampled preemption sets themselves, sorted ascending,
 *      trials x n_minus uint16 (sample_vectors, preemption.cpp:47-59). ---- */
lp_status lp_dump_scenarios(lp_handle* h, int32_t n, int32_t n_minus, int32_t trials,
                            uint64_t seed, uint16_t* out);

/* ---- multi-GPU: trials of every (n, k) pair are split across ranks and the
 *      integer histograms are summed with one ncclAllReduce over NVLink. ---- */
#define LP_NCCL_ID_BYTES 128
lp_status lp_nccl_unique_id(uint8_t out[LP_NCCL_ID_BYTES]);
lp_status lp_comm_init(lp_handle* h, const uint8_t id[LP_NCCL_ID_BYTES], int32_t nranks,
                       int32_t rank);
/* Parity mode of the split: lp_survivor_hist then counts only trial slice
 * [count*rank/nranks, count*(rank+1)/nranks) of the ensemble (the slice rank
 * `rank` of an nranks-GPU re-plan generates) and *total is the slice size.
 * Summing the slices of every rank reproduces the single-GPU counts.  The
 * re-plan path is unaffected (it follows lp_comm_init). */
lp_status lp_set_shard(lp_handle* h, int32_t rank, int32_t nranks);

/* ---- host table producers (perf_model stays on the host):
 *      throughput perf_model.cpp:14-42, enumerate_configs :44-52,
 *      depth_feasible :5-8, reactive_plan optimizer.cpp:11-25,
 *      scenario_count preemption.cpp:10-21, mix_seed rng.hpp:46-55. ------- */
double lp_throughput(const lp_profile* profile, lp_config cfg);
int32_t lp_depth_feasible(const lp_profile* profile, int32_t stages);
/* Writes min(count, cap) configs in reference order; returns the full count. */
int32_t lp_enumerate_configs(const lp_profile* profile, int32_t n, lp_config* out, int32_t cap);
/* Writes the reactive choice; returns 1 if one exists, 0 if suspended. */
int32_t lp_reactive_plan(const lp_profile* profile, int32_t n_now, lp_config* out);
uint64_t lp_scenario_count(int32_t n, int32_t k);
uint64_t lp_mix_seed(uint64_t a, uint64_t b);

/* ---- migration planning for a realised scenario:
 *      plan_migration migration.cpp:106-217, migration_cost :219-236,
 *      transition_outcome_min :49-89, resume_cost :100-104.  Host code: the
 *      concrete moves of the one transition the DP chose, not a hot path. -- */
typedef enum {
  LP_MIG_NONE = 0, /* MigrationKind (migration.hpp:11) */
  LP_MIG_INTRA_STAGE = 1,
  LP_MIG_INTER_STAGE = 2,
  LP_MIG_PIPELINE = 3
} lp_migration_kind;

/* Move (migration.hpp:29-34).  from_pipeline = from_stage = -1 for a spare. */
typedef struct {
  int32_t instance;
  int32_t from_pipeline, from_stage;
  int32_t to_pipeline, to_stage;
  int32_t transfers_params; /* 0 / 1 */
} lp_move;

/* MigrationPlan (migration.hpp:36-43) without the move vector. */
typedef struct {
  int32_t kind; /* lp_migration_kind */
  int32_t transfer_rounds;
  lp_config source;
  lp_config target;
  double est_cost_s;
  int32_t n_moves; /* moves in the plan (may exceed the caller's cap) */
  int32_t pad;
} lp_migration;

/* Plans the transition from `source` (+ `spares` trailing spare instances)
 * to `target` under the preemption vector v[0 .. source.D*source.P+spares)
 * (v[k] = 1: instance k preempted).  Writes min(n_moves, cap) moves in the
 * reference's order.  LP_EROLLBACK when a stage has no survivor and the
 * target keeps a pipeline; LP_EINVAL on a size mismatch or too few bodies. */
lp_status lp_plan_migration(const lp_profile* profile, const lp_costs* costs, lp_config source,
                            int32_t spares, const uint8_t* v, int32_t v_len, lp_config target,
                            lp_migration* out, lp_move* moves, int32_t cap);
/* T_mig of a plan (migration_cost); fresh_instances > 0 adds process startup. */
double lp_migration_cost(const lp_profile* profile, const lp_costs* costs, const lp_migration* plan,
                         int32_t fresh_instances);
/* Stats-level costing from the per-stage survivor minimum. */
lp_status lp_transition_outcome(const lp_profile* profile, const lp_costs* costs,
                                int32_t min_survivor, lp_config source, lp_config target,
                                int32_t fresh_instances, double* cost_s, int32_t* kind,
                                int32_t* rollback);
double lp_resume_cost(const lp_profile* profile, const lp_costs* costs, lp_config target);

/* ---- availability forecasts, the DP's n_seq producer:
 *      predict predictor.cpp:239-274 (preprocess :29-77, ARIMA(2,1,2) two-
 *      stage least squares :81-188, postprocess :190-237), eval_l1 :276-286,
 *      and the sliding-window evaluation of `spotsim predict`
 *      (tools/commands.cpp:267-299).  One device thread per (window, method);
 *      FP64 without contraction, so forecasts are bit-identical. ---------- */
typedef enum {
  LP_PREDICT_ARIMA = 0, /* PredictMethod (predictor.hpp:25) */
  LP_PREDICT_MOVING_AVG = 1,
  LP_PREDICT_EXP_SMOOTH = 2,
  LP_PREDICT_LAST_VALUE = 3
} lp_predict_method;

/* ForecastConfig (predictor.hpp:8-18). */
typedef struct {
  int32_t history_len;
  int32_t lookahead;
  int32_t capacity;
  int32_t floor;
  int32_t max_step;
  int32_t reset_threshold;
  int32_t moving_avg_window;
  int32_t pad;
  double exp_smooth_factor;
  double steep_decay;
} lp_forecast_config;

/* The reference's defaults (history 12, lookahead 12, max_step 8, ...). */
lp_forecast_config lp_forecast_defaults(int32_t capacity);
/* predict(): forecast of the next cfg->lookahead counts from the last
 * cfg->history_len entries of history[0 .. len).  out: lookahead ints.
 * LP_EINVAL when len < history_len or lookahead < 1. */
lp_status lp_predict(const int32_t* history, int32_t len, const lp_forecast_config* cfg,
                     int32_t method, int32_t device, int32_t* out);
/* Every window t = H .. len-I of counts (history counts[t-H, t), actual
 * counts[t, t+I)) for each method: preds[(w*n_methods + m)*I + j] and, when
 * l1 is not null, l1[w*n_methods + m] = eval_l1.  *n_windows receives the
 * window count (0 when len < H + I). */
lp_status lp_predict_windows(const int32_t* counts, int32_t len, const lp_forecast_config* cfg,
                             const int32_t* methods, int32_t n_methods, int32_t device,
                             int32_t* preds, double* l1, int32_t* n_windows);
/* (sum |pred - actual|) / (sum actual); 0 for an exact all-zero match, +inf
 * when actual sums to zero and pred does not. */
double lp_eval_l1(const int32_t* pred, const int32_t* actual, int32_t len);

/* ---- the replay driver: the reference simulator's run()
 *      (simulator.cpp:119-340) over an availability trace, with this
 *      library's planner (its device histogram store persists across the
 *      re-plans) and forecasts.  Host bookkeeping (placements, rollbacks,
 *      sample accounting, the ledger) restates the reference exactly. ---- */
typedef enum {
  LP_POLICY_PROACTIVE = 0, /* PolicyKind (simulator.hpp:16-22) */
  LP_POLICY_IDEAL = 1,
  LP_POLICY_REACTIVE = 2,
  LP_POLICY_CHECKPOINT = 3,
  LP_POLICY_REDUNDANCY = 4
} lp_policy_kind;

/* Policy (simulator.hpp:38-75) with CheckpointParams / RedundancyParams. */
typedef struct {
  int32_t kind;
  int32_t lookahead;       /* proactive / ideal */
  int32_t method;          /* proactive: lp_predict_method */
  int32_t history;         /* proactive */
  int32_t ckpt_period_intervals;
  int32_t redundancy_fixed_stages;
  double ckpt_save_cost_s;
  double ckpt_restore_cost_s;
  double ckpt_restart_cost_s;
  double redundancy_slowdown;
} lp_policy;

/* Ledger (simulator.hpp:85-97): instance-seconds by category. */
typedef struct {
  double effective_s, migration_s, checkpoint_s, wasted_rollback_s, idle_s;
} lp_ledger;

/* IntervalLog (simulator.hpp:99-109). */
typedef struct {
  int32_t interval, available, pipelines, stages;
  double throughput;
  int64_t committed, rolled_back;
  int32_t migration; /* lp_migration_kind */
  int32_t pad;
  lp_ledger ledger;
} lp_interval_log;

/* SimReport (simulator.hpp:111-127) without the per-interval vector. */
typedef struct {
  uint64_t seed;
  int64_t committed_samples;
  double wall_time_s;
  lp_ledger ledger;
  double instance_seconds, instance_hours, spot_cost, ondemand_cost;
  double cost_per_sample; /* valid when has_cost_per_sample */
  int32_t has_cost_per_sample;
  int32_t epochs_completed, rollback_events, suspended_intervals, sample_accounting_ok;
  int32_t pad;
} lp_sim_report;

/* The reference's defaults: Policy::Proactive(12, arima, 12),
 * CheckpointParams{5, 10, 30, 30}, RedundancyParams{4, 0.75}. */
lp_policy lp_policy_defaults(int32_t kind);
/* run(series, w, policy, seed, {epoch_samples, planner, costs}, shared):
 * counts[0 .. len) at interval_s seconds, capacity for the forecasts.
 * shared != NULL: plan with that handle as is (the reference's injected
 * Planner); else a private planner from (profile, costs, planner options)
 * with interval_s = interval_s and rollback = the policy's restore cost, on
 * `device`.  logs: len entries.  spot / on-demand prices per instance-hour
 * (WorkloadProfile::spot_price_per_hour etc.). */
lp_status lp_simulate(lp_handle* shared, const lp_profile* profile, const lp_costs* costs,
                      const lp_options* planner_options, int32_t device, const int32_t* counts,
                      int32_t len, double interval_s, int32_t capacity, const lp_policy* policy,
                      uint64_t seed, int32_t epoch_samples, double spot_price_per_hour,
                      double ondemand_price_per_hour, lp_sim_report* report, lp_interval_log* logs);

/* The same for many seeds at once: the configuration sequence (and so every
 * re-plan) does not depend on the seed — only the placements and sample
 * shuffles do — so the trace is planned once and each seed replays the
 * bookkeeping.  reports: n_seeds; logs: n_seeds x len (seed-major). */
lp_status lp_simulate_batch(lp_handle* shared, const lp_profile* profile, const lp_costs* costs,
                            const lp_options* planner_options, int32_t device, const int32_t* counts,
                            int32_t len, double interval_s, int32_t capacity, const lp_policy* policy,
                            const uint64_t* seeds, int32_t n_seeds, int32_t epoch_samples,
                            double spot_price_per_hour, double ondemand_price_per_hour,
                            lp_sim_report* reports, lp_interval_log* logs);

/* Build information (sm arch, sizes supported). */
int32_t lp_max_instances(void);
const char* lp_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* LIVEPUT_H_ */
