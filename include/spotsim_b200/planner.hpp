// spotsim_b200/planner.hpp — header-only C++ facade over liveput.h.
//
// Mirrors the reference's planning interface (proj/core/include/spotsim/
// optimizer.hpp:13-92, perf_model.hpp:10-60, migration.hpp:16-27): same type
// and member names, std::optional<ParallelConfig> for the suspended state,
// std::invalid_argument for bad arguments.  Every call goes through the C ABI
// to the sm_100a kernels in libliveput.so; nothing is computed here except
// argument marshalling.  Link with -lliveput (paper_2403_14097_b200/lib).
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "liveput.h"

namespace spotsim_b200 {

struct ParallelConfig {
  int pipelines = 1;  // D
  int stages = 1;     // P
  int instances() const { return pipelines * stages; }
  bool operator==(const ParallelConfig&) const = default;
};

struct MemoryModel {
  double fixed_bytes = 0.0;
  double per_stage_bytes = 0.0;
};

struct WorkloadProfile {
  std::string name;
  double compute_per_microbatch_s = 0.0;
  double param_bytes = 0.0;
  double activation_bytes = 0.0;
  int minibatch_size = 1;
  int microbatch_size = 1;
  double device_memory_bytes = 0.0;
  MemoryModel memory;
  double alpha_s = 0.0;
  double beta_s_per_byte = 0.0;
  std::map<int, double> pipeline_rates;
  double spot_price_per_hour = 0.0;      // simulator costs only
  double ondemand_price_per_hour = 0.0;
};

struct CostTable {
  double start_process_s = 1.0;
  double rendezvous_s = 5.0;
  double cuda_context_s = 5.0;
  double load_data_s = 5.0;
  double build_model_s = 5.0;
  double update_comm_groups_s = 10.0;
};

struct PlannerOptions {
  double interval_s = 60.0;
  int lookahead = 12;
  int mc_trials = 200;
  uint64_t exact_cap = 2000;
  uint64_t mc_seed = 0x5eedULL;
  double rollback_penalty_s = 30.0;
  bool strict_conditional = false;
};

struct PlanStep {
  int interval_index = 0;
  std::optional<ParallelConfig> config;
  double expected_committed = 0.0;
  double expected_mig_cost_s = 0.0;
};

class LiveputError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {

// Keeps the rate arrays alive while an lp_profile points into them.
struct ProfileC {
  lp_profile p{};
  std::vector<int32_t> depths;
  std::vector<double> rates;
  explicit ProfileC(const WorkloadProfile& w) {
    for (const auto& [d, r] : w.pipeline_rates) {
      depths.push_back(d);
      rates.push_back(r);
    }
    p.compute_per_microbatch_s = w.compute_per_microbatch_s;
    p.param_bytes = w.param_bytes;
    p.activation_bytes = w.activation_bytes;
    p.minibatch_size = w.minibatch_size;
    p.microbatch_size = w.microbatch_size;
    p.device_memory_bytes = w.device_memory_bytes;
    p.memory_fixed_bytes = w.memory.fixed_bytes;
    p.memory_per_stage_bytes = w.memory.per_stage_bytes;
    p.alpha_s = w.alpha_s;
    p.beta_s_per_byte = w.beta_s_per_byte;
    p.n_rates = static_cast<int32_t>(depths.size());
    p.rate_depths = depths.empty() ? nullptr : depths.data();
    p.rate_values = rates.empty() ? nullptr : rates.data();
  }
};

inline lp_costs to_c(const CostTable& c) {
  return {c.start_process_s, c.rendezvous_s, c.cuda_context_s, c.load_data_s, c.build_model_s,
          c.update_comm_groups_s};
}

inline lp_options to_c(const PlannerOptions& o) {
  return {o.interval_s, o.lookahead, o.mc_trials, o.exact_cap, o.mc_seed, o.rollback_penalty_s,
          o.strict_conditional ? 1 : 0};
}

inline lp_config to_c(const std::optional<ParallelConfig>& c) {
  return c ? lp_config{c->pipelines, c->stages} : lp_config{0, 0};
}

inline std::optional<ParallelConfig> from_c(const lp_config& c) {
  if (c.pipelines <= 0) return std::nullopt;
  return ParallelConfig{c.pipelines, c.stages};
}

inline void check(lp_status s, const lp_handle* h) {
  if (s == LP_OK) return;
  const char* m = h ? lp_last_error(h) : lp_last_global_error();
  if (s == LP_EINVAL) throw std::invalid_argument(m ? m : "liveput: invalid argument");
  throw LiveputError(std::string("liveput: ") + (m ? m : "error"));
}

}  // namespace detail

// perf_model.hpp:52-60 / optimizer.hpp:36 — host table producers.
inline double throughput(const ParallelConfig& cfg, const WorkloadProfile& w) {
  detail::ProfileC p(w);
  return lp_throughput(&p.p, {cfg.pipelines, cfg.stages});
}

inline bool depth_feasible(int stages, const WorkloadProfile& w) {
  detail::ProfileC p(w);
  return lp_depth_feasible(&p.p, stages) != 0;
}

inline std::vector<ParallelConfig> enumerate_configs(int n, const WorkloadProfile& w) {
  detail::ProfileC p(w);
  const int cnt = lp_enumerate_configs(&p.p, n, nullptr, 0);
  std::vector<lp_config> buf(cnt > 0 ? cnt : 1);
  lp_enumerate_configs(&p.p, n, buf.data(), cnt);
  std::vector<ParallelConfig> out;
  for (int i = 0; i < cnt; ++i) out.push_back({buf[i].pipelines, buf[i].stages});
  return out;
}

inline std::optional<ParallelConfig> reactive_plan(int n_now, const WorkloadProfile& w) {
  detail::ProfileC p(w);
  lp_config c{};
  if (!lp_reactive_plan(&p.p, n_now, &c)) return std::nullopt;
  return ParallelConfig{c.pipelines, c.stages};
}

inline uint64_t scenario_count(int n, int k) { return lp_scenario_count(n, k); }
inline uint64_t mix_seed(uint64_t a, uint64_t b) { return lp_mix_seed(a, b); }

// optimizer.hpp:41-92
class Planner {
 public:
  Planner(WorkloadProfile w, CostTable costs, PlannerOptions opt = {}, int device = 0)
      : workload_(std::move(w)), costs_(costs), options_(opt) {
    detail::ProfileC p(workload_);
    const lp_costs c = detail::to_c(costs_);
    const lp_options o = detail::to_c(options_);
    detail::check(lp_create(&p.p, &c, &o, device, &h_), nullptr);
  }
  ~Planner() { lp_destroy(h_); }
  Planner(const Planner&) = delete;
  Planner& operator=(const Planner&) = delete;

  const WorkloadProfile& workload() const { return workload_; }
  const CostTable& costs() const { return costs_; }
  const PlannerOptions& options() const { return options_; }

  struct PhiValue {
    double committed = 0.0;
    double mig_cost_s = 0.0;
  };

  PhiValue phi(const std::optional<ParallelConfig>& prev, const std::optional<ParallelConfig>& next,
               int n_now, int n_next) {
    PhiValue v;
    detail::check(lp_phi(h_, detail::to_c(prev), detail::to_c(next), n_now, n_next, &v.committed,
                         &v.mig_cost_s),
                  h_);
    return v;
  }

  std::vector<PlanStep> dp_optimize(const std::optional<ParallelConfig>& current,
                                    const std::vector<int>& n_seq) {
    if (n_seq.size() < 2) throw std::invalid_argument("dp_optimize: need at least N_i and N_{i+1}");
    std::vector<int32_t> ns(n_seq.begin(), n_seq.end());
    std::vector<lp_plan_step> out(n_seq.size() - 1);
    detail::check(lp_replan(h_, detail::to_c(current), ns.data(), static_cast<int32_t>(ns.size()),
                            out.data(), nullptr, 0, nullptr),
                  h_);
    std::vector<PlanStep> plan;
    for (const lp_plan_step& s : out)
      plan.push_back({s.interval_index, detail::from_c(s.config), s.expected_committed,
                      s.expected_mig_cost_s});
    return plan;
  }

  double sequence_value(const std::optional<ParallelConfig>& current,
                        const std::vector<std::optional<ParallelConfig>>& sequence,
                        const std::vector<int>& n_seq) {
    if (sequence.size() + 1 != n_seq.size())
      throw std::invalid_argument("sequence_value: sequence/N length mismatch");
    std::vector<lp_config> seq;
    for (const auto& c : sequence) seq.push_back(detail::to_c(c));
    std::vector<int32_t> ns(n_seq.begin(), n_seq.end());
    double v = 0.0;
    detail::check(lp_sequence_value(h_, detail::to_c(current), seq.data(), ns.data(),
                                    static_cast<int32_t>(ns.size()), &v),
                  h_);
    return v;
  }

  // Un-normalised survivor histogram (counts[m], m = 0..D) and its ensemble size.
  std::vector<uint64_t> survivor_counts(const ParallelConfig& prev, int n_now, int n_minus,
                                        uint64_t* total) {
    std::vector<uint64_t> c(prev.pipelines + 1, 0);
    detail::check(lp_survivor_hist(h_, {prev.pipelines, prev.stages}, n_now, n_minus, c.data(), total),
                  h_);
    return c;
  }

  lp_handle* handle() { return h_; }

 private:
  WorkloadProfile workload_;
  CostTable costs_;
  PlannerOptions options_;
  lp_handle* h_ = nullptr;
};

// preemption.hpp:53-65
struct EvalMode {
  bool exact = true;
  int trials = 1000;
  uint64_t seed = 0;
  static EvalMode Exact() { return {true, 0, 0}; }
  static EvalMode MC(int trials, uint64_t seed) { return {false, trials, seed}; }
};

inline double expected_liveput(Planner& planner, const ParallelConfig& cfg, int n, int n_minus,
                               const EvalMode& mode) {
  double v = 0.0;
  detail::check(lp_expected_liveput(planner.handle(), {cfg.pipelines, cfg.stages}, n, n_minus,
                                    mode.exact ? 1 : 0, mode.trials, mode.seed, &v),
                planner.handle());
  return v;
}

// ---- migration.hpp:11-101 — concrete moves for a realised scenario ------
enum class MigrationKind { none, intra_stage, inter_stage, pipeline };

struct Topology {  // preemption.hpp:13-20
  int pipelines = 0;
  int stages = 0;
  int spares = 0;
  int assigned() const { return pipelines * stages; }
  int total() const { return assigned() + spares; }
};

using PreemptionVector = std::vector<uint8_t>;

struct Move {
  int instance = 0;
  int from_pipeline = 0, from_stage = 0;
  int to_pipeline = 0, to_stage = 0;
  bool transfers_params = false;
};

struct MigrationPlan {
  MigrationKind kind = MigrationKind::none;
  std::vector<Move> moves;
  ParallelConfig source;
  ParallelConfig target;
  int transfer_rounds = 0;
  double est_cost_s = 0.0;
};

struct RollbackRequired : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct TransitionOutcome {
  double cost_s = 0.0;
  MigrationKind kind = MigrationKind::none;
  bool rollback = false;
};

inline MigrationPlan plan_migration(const Topology& topo, const PreemptionVector& v,
                                    const ParallelConfig& target, const WorkloadProfile& w,
                                    const CostTable& costs) {
  detail::ProfileC p(w);
  const lp_costs c = detail::to_c(costs);
  lp_migration out{};
  std::vector<lp_move> mv(v.size() + 1);
  const lp_status s = lp_plan_migration(&p.p, &c, {topo.pipelines, topo.stages}, topo.spares, v.data(),
                                        static_cast<int32_t>(v.size()), {target.pipelines, target.stages},
                                        &out, mv.data(), static_cast<int32_t>(mv.size()));
  if (s == LP_EROLLBACK) throw RollbackRequired(lp_last_global_error());
  detail::check(s, nullptr);
  MigrationPlan plan;
  plan.kind = static_cast<MigrationKind>(out.kind);
  plan.source = {out.source.pipelines, out.source.stages};
  plan.target = {out.target.pipelines, out.target.stages};
  plan.transfer_rounds = out.transfer_rounds;
  plan.est_cost_s = out.est_cost_s;
  for (int i = 0; i < out.n_moves; ++i)
    plan.moves.push_back({mv[i].instance, mv[i].from_pipeline, mv[i].from_stage, mv[i].to_pipeline,
                          mv[i].to_stage, mv[i].transfers_params != 0});
  return plan;
}

inline double migration_cost(const MigrationPlan& plan, const WorkloadProfile& w,
                             const CostTable& costs, int fresh_instances) {
  detail::ProfileC p(w);
  const lp_costs c = detail::to_c(costs);
  lp_migration m{};
  m.kind = static_cast<int32_t>(plan.kind);
  m.transfer_rounds = plan.transfer_rounds;
  m.source = {plan.source.pipelines, plan.source.stages};
  m.target = {plan.target.pipelines, plan.target.stages};
  return lp_migration_cost(&p.p, &c, &m, fresh_instances);
}

inline TransitionOutcome transition_outcome_min(int min_survivor, const ParallelConfig& source,
                                                const ParallelConfig& target, int fresh_instances,
                                                const WorkloadProfile& w, const CostTable& costs) {
  detail::ProfileC p(w);
  const lp_costs c = detail::to_c(costs);
  TransitionOutcome o;
  int32_t kind = 0, rb = 0;
  detail::check(lp_transition_outcome(&p.p, &c, min_survivor, {source.pipelines, source.stages},
                                      {target.pipelines, target.stages}, fresh_instances, &o.cost_s,
                                      &kind, &rb),
                nullptr);
  o.kind = static_cast<MigrationKind>(kind);
  o.rollback = rb != 0;
  return o;
}

inline double resume_cost(const ParallelConfig& target, const WorkloadProfile& w,
                          const CostTable& costs) {
  detail::ProfileC p(w);
  const lp_costs c = detail::to_c(costs);
  return lp_resume_cost(&p.p, &c, {target.pipelines, target.stages});
}

// ---- simulator.hpp:14-140 — the replay driver over this planner ---------
struct IntervalSeries {  // trace.hpp:17-24
  double interval_seconds = 60.0;
  int capacity = 0;
  std::vector<int> counts;
};

enum class PolicyKind { proactive, ideal, reactive, checkpoint, redundancy };
enum class PredictMethod { arima, moving_avg, exp_smooth, last_value };

struct CheckpointParams {
  int period_intervals = 5;
  double save_cost_s = 10.0, restore_cost_s = 30.0, restart_cost_s = 30.0;
};
struct RedundancyParams {
  int fixed_stages = 4;
  double slowdown_factor = 0.75;
};
struct Policy {
  PolicyKind kind = PolicyKind::reactive;
  int lookahead = 12;
  PredictMethod method = PredictMethod::arima;
  int history = 12;
  CheckpointParams checkpoint;
  RedundancyParams redundancy;
  static Policy Proactive(int lookahead = 12, PredictMethod m = PredictMethod::arima, int history = 12) {
    Policy p;
    p.kind = PolicyKind::proactive;
    p.lookahead = lookahead;
    p.method = m;
    p.history = history;
    return p;
  }
  static Policy Ideal(int lookahead = 12) {
    Policy p;
    p.kind = PolicyKind::ideal;
    p.lookahead = lookahead;
    return p;
  }
  static Policy Reactive() { return Policy{}; }
  static Policy Checkpoint(CheckpointParams c = {}) {
    Policy p;
    p.kind = PolicyKind::checkpoint;
    p.checkpoint = c;
    return p;
  }
  static Policy Redundancy(int fixed_stages, double slowdown = 0.75) {
    Policy p;
    p.kind = PolicyKind::redundancy;
    p.redundancy = {fixed_stages, slowdown};
    return p;
  }
};

struct SimOptions {
  int epoch_samples = 0;
  PlannerOptions planner;
  CostTable costs;
};

struct Ledger {
  double effective_s = 0.0, migration_s = 0.0, checkpoint_s = 0.0, wasted_rollback_s = 0.0, idle_s = 0.0;
  double total() const { return effective_s + migration_s + checkpoint_s + wasted_rollback_s + idle_s; }
};

struct IntervalLog {
  int interval = 0, available = 0, pipelines = 0, stages = 0;
  double throughput = 0.0;
  long long committed = 0, rolled_back = 0;
  MigrationKind migration = MigrationKind::none;
  Ledger ledger;
};

struct SimReport {
  std::string policy;
  uint64_t seed = 0;
  std::vector<IntervalLog> intervals;
  long long committed_samples = 0;
  double wall_time_s = 0.0;
  Ledger ledger;
  double instance_seconds = 0.0, instance_hours = 0.0, spot_cost = 0.0, ondemand_cost = 0.0;
  std::optional<double> cost_per_sample;
  int epochs_completed = 0, rollback_events = 0, suspended_intervals = 0;
  bool sample_accounting_ok = true;
};

// run (simulator.cpp:119-340); the planner is `shared` when given, else a
// private one on `device`.
inline SimReport run(const IntervalSeries& series, const WorkloadProfile& w, const Policy& policy,
                     uint64_t seed, const SimOptions& options = {}, Planner* shared = nullptr,
                     int device = 0) {
  detail::ProfileC p(w);
  const lp_costs c = detail::to_c(options.costs);
  const lp_options o = detail::to_c(options.planner);
  lp_policy pol = lp_policy_defaults(static_cast<int32_t>(policy.kind));
  pol.lookahead = policy.lookahead;
  pol.method = static_cast<int32_t>(policy.method);
  pol.history = policy.history;
  pol.ckpt_period_intervals = policy.checkpoint.period_intervals;
  pol.ckpt_save_cost_s = policy.checkpoint.save_cost_s;
  pol.ckpt_restore_cost_s = policy.checkpoint.restore_cost_s;
  pol.ckpt_restart_cost_s = policy.checkpoint.restart_cost_s;
  pol.redundancy_fixed_stages = policy.redundancy.fixed_stages;
  pol.redundancy_slowdown = policy.redundancy.slowdown_factor;
  std::vector<lp_interval_log> logs(series.counts.size() + 1);
  lp_sim_report r{};
  std::vector<int32_t> counts(series.counts.begin(), series.counts.end());
  detail::check(lp_simulate(shared ? shared->handle() : nullptr, &p.p, &c, &o, device, counts.data(),
                            static_cast<int32_t>(counts.size()), series.interval_seconds, series.capacity,
                            &pol, seed, options.epoch_samples, w.spot_price_per_hour,
                            w.ondemand_price_per_hour, &r, logs.data()),
                nullptr);
  static const char* kNames[] = {"proactive", "ideal", "reactive", "checkpoint", "redundancy"};
  SimReport rep;
  rep.policy = kNames[static_cast<int>(policy.kind)];
  rep.seed = r.seed;
  rep.committed_samples = r.committed_samples;
  rep.wall_time_s = r.wall_time_s;
  auto led = [](const lp_ledger& l) {
    return Ledger{l.effective_s, l.migration_s, l.checkpoint_s, l.wasted_rollback_s, l.idle_s};
  };
  rep.ledger = led(r.ledger);
  rep.instance_seconds = r.instance_seconds;
  rep.instance_hours = r.instance_hours;
  rep.spot_cost = r.spot_cost;
  rep.ondemand_cost = r.ondemand_cost;
  if (r.has_cost_per_sample) rep.cost_per_sample = r.cost_per_sample;
  rep.epochs_completed = r.epochs_completed;
  rep.rollback_events = r.rollback_events;
  rep.suspended_intervals = r.suspended_intervals;
  rep.sample_accounting_ok = r.sample_accounting_ok != 0;
  for (size_t i = 0; i < series.counts.size(); ++i) {
    const lp_interval_log& L = logs[i];
    rep.intervals.push_back({L.interval, L.available, L.pipelines, L.stages, L.throughput, L.committed,
                             L.rolled_back, static_cast<MigrationKind>(L.migration), led(L.ledger)});
  }
  return rep;
}

}  // namespace spotsim_b200
