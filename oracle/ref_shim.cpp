// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" layer over the UNMODIFIED reference library (spotsim,
// /root/reference/proj/core) so that Python tests, the golden-fixture script
// and bench.py's CPU arm can call the reference's own code.  Built by
// oracle/Makefile from the reference sources where they lie; output goes to
// oracle/_ref/libspotsim_ref.so only.  Nothing here is copied from the
// reference: it only includes its headers and calls its public API (plus the
// private Planner::survivor_histogram, reached with the access trick below so
// the un-normalised histogram can be compared directly).
//
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
// legs may load this library.

#include <atomic>
#include <chrono>
#include <cstring>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#define private public  // reach Planner::survivor_histogram (optimizer.hpp:81-82)
#include "spotsim/optimizer.hpp"
#undef private
#include "spotsim/migration.hpp"
#include "spotsim/perf_model.hpp"
#include "spotsim/preemption.hpp"
#include "spotsim/rng.hpp"
#include "spotsim/trace.hpp"
#include "spotsim/predictor.hpp"
#include "spotsim/simulator.hpp"

#include "liveput.h"

using namespace spotsim;

namespace {

thread_local std::string g_err;

WorkloadProfile to_profile(const lp_profile* p) {
  WorkloadProfile w;
  w.name = "ffi";
  w.compute_per_microbatch_s = p->compute_per_microbatch_s;
  w.param_bytes = p->param_bytes;
  w.activation_bytes = p->activation_bytes;
  w.minibatch_size = p->minibatch_size;
  w.microbatch_size = p->microbatch_size;
  w.device_memory_bytes = p->device_memory_bytes;
  w.memory = {p->memory_fixed_bytes, p->memory_per_stage_bytes};
  w.alpha_s = p->alpha_s;
  w.beta_s_per_byte = p->beta_s_per_byte;
  for (int i = 0; i < p->n_rates; ++i) w.pipeline_rates[p->rate_depths[i]] = p->rate_values[i];
  return w;
}

CostTable to_costs(const lp_costs* c) {
  CostTable t;
  t.start_process_s = c->start_process_s;
  t.rendezvous_s = c->rendezvous_s;
  t.cuda_context_s = c->cuda_context_s;
  t.load_data_s = c->load_data_s;
  t.build_model_s = c->build_model_s;
  t.update_comm_groups_s = c->update_comm_groups_s;
  return t;
}

PlannerOptions to_options(const lp_options* o) {
  PlannerOptions t;
  t.interval_s = o->interval_s;
  t.lookahead = o->lookahead;
  t.mc_trials = o->mc_trials;
  t.exact_cap = o->exact_cap;
  t.mc_seed = o->mc_seed;
  t.rollback_penalty_s = o->rollback_penalty_s;
  t.strict_conditional = o->strict_conditional != 0;
  return t;
}

std::optional<ParallelConfig> opt_cfg(int d, int p) {
  if (d <= 0) return std::nullopt;
  return ParallelConfig{d, p};
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_planner_new(const lp_profile* p, const lp_costs* c, const lp_options* o) {
  return new Planner(to_profile(p), to_costs(c), to_options(o));
}

void ref_planner_free(void* pl) { delete static_cast<Planner*>(pl); }

size_t ref_planner_cache_size(void* pl) { return static_cast<Planner*>(pl)->cache_size(); }

int ref_phi(void* pl, int pd, int pp, int nd, int np, int n_now, int n_next, double* out2) {
  try {
    auto v = static_cast<Planner*>(pl)->phi(opt_cfg(pd, pp), opt_cfg(nd, np), n_now, n_next);
    out2[0] = v.committed;
    out2[1] = v.mig_cost_s;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// steps_out: per step {D, P} in cfg_out[2*j], values in val_out[2*j].
int ref_dp_optimize(void* pl, int cd, int cp, const int* n_seq, int len, int* cfg_out,
                    double* val_out) {
  try {
    std::vector<int> ns(n_seq, n_seq + len);
    auto plan = static_cast<Planner*>(pl)->dp_optimize(opt_cfg(cd, cp), ns);
    for (size_t j = 0; j < plan.size(); ++j) {
      cfg_out[2 * j] = plan[j].config ? plan[j].config->pipelines : 0;
      cfg_out[2 * j + 1] = plan[j].config ? plan[j].config->stages : 0;
      val_out[2 * j] = plan[j].expected_committed;
      val_out[2 * j + 1] = plan[j].expected_mig_cost_s;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_sequence_value(void* pl, int cd, int cp, const int* seq_cfg, const int* n_seq, int len,
                       double* out) {
  try {
    std::vector<int> ns(n_seq, n_seq + len);
    std::vector<std::optional<ParallelConfig>> seq;
    for (int j = 0; j + 1 < len; ++j) seq.push_back(opt_cfg(seq_cfg[2 * j], seq_cfg[2 * j + 1]));
    *out = static_cast<Planner*>(pl)->sequence_value(opt_cfg(cd, cp), seq, ns);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Normalised histogram exactly as the Planner caches it (D+1 doubles).
int ref_survivor_hist(void* pl, int d, int p, int n_now, int n_minus, double* out) {
  try {
    const auto& h = static_cast<Planner*>(pl)->survivor_histogram({d, p}, n_now, n_minus);
    for (size_t i = 0; i < h.size(); ++i) out[i] = h[i];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

uint64_t ref_scenario_count(int n, int k) { return scenario_count(n, k); }
uint64_t ref_mix_seed(uint64_t a, uint64_t b) { return mix_seed(a, b); }

void ref_rng_draws(uint64_t seed, int count, uint64_t* out) {
  Rng r(seed);
  for (int i = 0; i < count; ++i) out[i] = r.next();
}

int ref_sample_distinct(int n, int k, uint64_t seed, int* out) {
  try {
    Rng r(seed);
    auto v = sample_distinct(n, k, r);
    for (int i = 0; i < k; ++i) out[i] = v[i];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// trials x n bytes.
int ref_sample_vectors(int n, int k, int trials, uint64_t seed, uint8_t* out) {
  try {
    auto vs = sample_vectors(n, k, trials, seed);
    for (int t = 0; t < trials; ++t) std::memcpy(out + (size_t)t * n, vs[t].data(), n);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Returns the count written (capped); -1 on error.
long long ref_enumerate_vectors(int n, int k, uint8_t* out, long long cap) {
  try {
    auto vs = enumerate_vectors(n, k);
    long long w = 0;
    for (auto& v : vs) {
      if (w >= cap) break;
      std::memcpy(out + (size_t)w * n, v.data(), n);
      ++w;
    }
    return (long long)vs.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Per-vector survivor minimum for config (d, p) using stage_survivors
// (preemption.cpp:61-66) and the min of optimizer.cpp:76-82.
void ref_tally(const uint8_t* vecs, int count, int n, int d, int p, uint16_t* out_m) {
  const Topology topo{d, p, n - d * p};
  for (int t = 0; t < count; ++t) {
    PreemptionVector v(vecs + (size_t)t * n, vecs + (size_t)(t + 1) * n);
    int m = d;
    for (int s : stage_survivors(topo, v)) m = std::min(m, s);
    out_m[t] = (uint16_t)m;
  }
}

int ref_surviving_pipelines(const uint8_t* v, int n, int d, int p, int intra) {
  const Topology topo{d, p, n - d * p};
  PreemptionVector vec(v, v + n);
  return surviving_pipelines(topo, vec, intra != 0);
}

double ref_throughput(const lp_profile* p, int d, int s) {
  return throughput({d, s}, to_profile(p));
}

int ref_depth_feasible(const lp_profile* p, int s) { return depth_feasible(s, to_profile(p)); }

int ref_enumerate_configs(const lp_profile* p, int n, int* out, int cap) {
  auto cs = enumerate_configs(n, to_profile(p));
  for (int i = 0; i < (int)cs.size() && i < cap; ++i) {
    out[2 * i] = cs[i].pipelines;
    out[2 * i + 1] = cs[i].stages;
  }
  return (int)cs.size();
}

int ref_reactive_plan(const lp_profile* p, int n, int* out2) {
  auto r = reactive_plan(n, to_profile(p));
  if (!r) return 0;
  out2[0] = r->pipelines;
  out2[1] = r->stages;
  return 1;
}

int ref_expected_liveput(const lp_profile* p, int d, int s, int n, int k, int exact, int trials,
                         uint64_t seed, double* out) {
  try {
    const EvalMode mode = exact ? EvalMode::Exact() : EvalMode::MC(trials, seed);
    *out = expected_liveput({d, s}, n, k, to_profile(p), mode);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// transition_outcome_min (migration.cpp:49-89): out2 = {cost, rollback}; returns kind.
int ref_transition_outcome_min(int m, int sd, int sp, int td, int tp, int fresh,
                               const lp_profile* p, const lp_costs* c, double* out2) {
  TransitionOutcome t = transition_outcome_min(m, {sd, sp}, {td, tp}, fresh, to_profile(p),
                                               to_costs(c));
  out2[0] = t.cost_s;
  out2[1] = t.rollback ? 1.0 : 0.0;
  return (int)t.kind;
}

double ref_resume_cost(int td, int tp, const lp_profile* p, const lp_costs* c) {
  return resume_cost({td, tp}, to_profile(p), to_costs(c));
}

// plan_migration (migration.cpp:106-217) + migration_cost (:219-236).
// moves_out: 6 ints per move (instance, from_pipeline, from_stage,
// to_pipeline, to_stage, transfers_params).  info_out: {kind, transfer_rounds,
// n_moves}.  cost_out: {est_cost_s, migration_cost(fresh = 1)}.  Returns 0,
// 1 for RollbackRequired, 2 for std::invalid_argument.
int ref_plan_migration(int sd, int sp, int spares, const uint8_t* v, int v_len, int td, int tp,
                       const lp_profile* p, const lp_costs* c, int* info_out, int* moves_out,
                       int cap, double* cost_out) {
  try {
    const Topology topo{sd, sp, spares};
    PreemptionVector vec(v, v + v_len);
    const WorkloadProfile w = to_profile(p);
    const CostTable costs = to_costs(c);
    MigrationPlan plan = plan_migration(topo, vec, {td, tp}, w, costs);
    info_out[0] = (int)plan.kind;
    info_out[1] = plan.transfer_rounds;
    info_out[2] = (int)plan.moves.size();
    for (int i = 0; i < (int)plan.moves.size() && i < cap; ++i) {
      const Move& m = plan.moves[i];
      int* o = moves_out + 6 * i;
      o[0] = m.instance;
      o[1] = m.from_pipeline;
      o[2] = m.from_stage;
      o[3] = m.to_pipeline;
      o[4] = m.to_stage;
      o[5] = m.transfers_params ? 1 : 0;
    }
    cost_out[0] = plan.est_cost_s;
    cost_out[1] = migration_cost(plan, w, costs, 1);
    return 0;
  } catch (const RollbackRequired& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// predict (predictor.cpp:239-274): cfg9 = {history_len, lookahead, capacity,
// floor, max_step, reset_threshold, moving_avg_window} ints + {exp_smooth,
// steep_decay} doubles.  Returns 0, or 2 on std::invalid_argument.
int ref_predict(const int* history, int len, const int* cfg_i, const double* cfg_d, int method,
                int* out) {
  try {
    ForecastConfig fc;
    fc.history_len = cfg_i[0];
    fc.lookahead = cfg_i[1];
    fc.capacity = cfg_i[2];
    fc.floor = cfg_i[3];
    fc.max_step = cfg_i[4];
    fc.reset_threshold = cfg_i[5];
    fc.moving_avg_window = cfg_i[6];
    fc.exp_smooth_factor = cfg_d[0];
    fc.steep_decay = cfg_d[1];
    const Forecast f = predict(std::vector<int>(history, history + len), fc, (PredictMethod)method);
    for (size_t i = 0; i < f.values.size(); ++i) out[i] = f.values[i];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

double ref_eval_l1(const int* pred, const int* actual, int len) {
  Forecast f;
  f.values.assign(pred, pred + len);
  return eval_l1(f, std::vector<int>(actual, actual + len));
}

// run() (simulator.cpp:119-340).  pol_i = {kind, lookahead, method, history,
// ckpt_period, redundancy_stages}, pol_d = {save, restore, restart,
// slowdown}.  rep_d = {committed_samples, wall_time_s, ledger x5,
// instance_seconds, instance_hours, spot_cost, ondemand_cost,
// cost_per_sample (NaN if none)}, rep_i = {epochs_completed,
// rollback_events, suspended_intervals, sample_accounting_ok}.
// log_i: 7 per interval {interval, available, pipelines, stages, committed,
// rolled_back, migration}; log_d: 6 per interval {throughput, ledger x5}.
int ref_simulate(const int* counts, int len, double interval_s, int capacity, const lp_profile* p,
                 double spot, double ondemand, const lp_costs* c, const lp_options* o, const int* pol_i,
                 const double* pol_d, uint64_t seed, int epoch_samples, double* rep_d, int* rep_i,
                 long long* log_i, double* log_d) {
  try {
    IntervalSeries series;
    series.interval_seconds = interval_s;
    series.capacity = capacity;
    series.counts.assign(counts, counts + len);
    WorkloadProfile w = to_profile(p);
    w.spot_price_per_hour = spot;
    w.ondemand_price_per_hour = ondemand;
    Policy pol;
    pol.kind = (PolicyKind)pol_i[0];
    pol.lookahead = pol_i[1];
    pol.method = (PredictMethod)pol_i[2];
    pol.history = pol_i[3];
    pol.checkpoint.period_intervals = pol_i[4];
    pol.redundancy.fixed_stages = pol_i[5];
    pol.checkpoint.save_cost_s = pol_d[0];
    pol.checkpoint.restore_cost_s = pol_d[1];
    pol.checkpoint.restart_cost_s = pol_d[2];
    pol.redundancy.slowdown_factor = pol_d[3];
    SimOptions so;
    so.epoch_samples = epoch_samples;
    so.planner = to_options(o);
    so.costs = to_costs(c);
    SimReport r = run(series, w, pol, seed, so, nullptr);
    rep_d[0] = (double)r.committed_samples;
    rep_d[1] = r.wall_time_s;
    rep_d[2] = r.ledger.effective_s;
    rep_d[3] = r.ledger.migration_s;
    rep_d[4] = r.ledger.checkpoint_s;
    rep_d[5] = r.ledger.wasted_rollback_s;
    rep_d[6] = r.ledger.idle_s;
    rep_d[7] = r.instance_seconds;
    rep_d[8] = r.instance_hours;
    rep_d[9] = r.spot_cost;
    rep_d[10] = r.ondemand_cost;
    rep_d[11] = r.cost_per_sample ? *r.cost_per_sample : std::numeric_limits<double>::quiet_NaN();
    rep_i[0] = r.epochs_completed;
    rep_i[1] = r.rollback_events;
    rep_i[2] = r.suspended_intervals;
    rep_i[3] = r.sample_accounting_ok ? 1 : 0;
    for (int i = 0; i < len; ++i) {
      const IntervalLog& L = r.intervals[i];
      long long* li = log_i + 7 * i;
      li[0] = L.interval;
      li[1] = L.available;
      li[2] = L.pipelines;
      li[3] = L.stages;
      li[4] = L.committed;
      li[5] = L.rolled_back;
      li[6] = (long long)L.migration;
      double* ld = log_d + 6 * i;
      ld[0] = L.throughput;
      ld[1] = L.ledger.effective_s;
      ld[2] = L.ledger.migration_s;
      ld[3] = L.ledger.checkpoint_s;
      ld[4] = L.ledger.wasted_rollback_s;
      ld[5] = L.ledger.idle_s;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// gen_synthetic (trace.cpp:80-180): writes up to cap counts, returns length.
int ref_gen_synthetic(uint64_t seed, int cap, int length, int loss_events, int gain_events,
                      int min_step, int max_step, int* out, int out_cap) {
  try {
    IntervalSeries s = gen_synthetic(seed, cap, length, loss_events, gain_events, min_step,
                                     max_step);
    for (int i = 0; i < (int)s.counts.size() && i < out_cap; ++i) out[i] = s.counts[i];
    return (int)s.counts.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ---------------------------------------------------------------------------
// CPU arm for bench.py: the reference's own survivor-histogram path
// (Planner::phi -> survivor_histogram, optimizer.cpp:52-94) on `threads`
// host threads.  Each thread owns a fresh (cold) Planner and takes every
// threads-th prev config of each (n, k) pair.  Returns wall seconds; writes
// the number of (scenario, prev-config) resolutions performed.
double ref_bench_histograms(const lp_profile* p, const lp_costs* c, const lp_options* o,
                            const int* pair_n, const int* pair_k, int n_pairs, int threads,
                            unsigned long long* resolutions) {
  const WorkloadProfile w = to_profile(p);
  const CostTable costs = to_costs(c);
  const PlannerOptions opt = to_options(o);
  struct Job {
    ParallelConfig cfg;
    int n, k;
    unsigned long long res;
  };
  std::vector<Job> jobs;
  for (int i = 0; i < n_pairs; ++i) {
    const uint64_t count = scenario_count(pair_n[i], pair_k[i]);
    const unsigned long long per =
        count <= opt.exact_cap ? count : (unsigned long long)opt.mc_trials;
    for (const ParallelConfig& cfg : enumerate_configs(pair_n[i], w))
      jobs.push_back({cfg, pair_n[i], pair_k[i], per});
  }
  std::atomic<size_t> next{0};
  std::atomic<unsigned long long> done{0};
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&] {
      Planner planner(w, costs, opt);
      unsigned long long local = 0;
      for (size_t i = next++; i < jobs.size(); i = next++) {
        const Job& j = jobs[i];
        planner.survivor_histogram(j.cfg, j.n, j.k);
        local += j.res;
      }
      done += local;
    });
  }
  for (auto& th : pool) th.join();
  auto t1 = std::chrono::steady_clock::now();
  *resolutions = done.load();
  return std::chrono::duration<double>(t1 - t0).count();
}

// One cold Planner::dp_optimize (single thread, as the reference runs it).
double ref_bench_replan(const lp_profile* p, const lp_costs* c, const lp_options* o, int cd,
                        int cp, const int* n_seq, int len) {
  Planner planner(to_profile(p), to_costs(c), to_options(o));
  std::vector<int> ns(n_seq, n_seq + len);
  auto t0 = std::chrono::steady_clock::now();
  auto plan = planner.dp_optimize(opt_cfg(cd, cp), ns);
  auto t1 = std::chrono::steady_clock::now();
  (void)plan;
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
