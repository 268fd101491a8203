// adapter/optimizer.cpp — spotsim::Planner over the liveput C ABI.
//
// Replaces the reference's optimizer.cpp (/root/reference/proj/core/src/
// optimizer.cpp:11-219) behind its unchanged public header interface
// (adapter/include/spotsim/optimizer.hpp).  Every planning computation runs
// in libliveput.so on the B200:
//   reactive_plan   optimizer.cpp:11-25    -> lp_reactive_plan
//   Planner::phi    optimizer.cpp:52-62    -> lp_phi (+ a host memo, as the reference's phi_cache_)
//   dp_optimize     optimizer.cpp:140-205  -> lp_replan
//   sequence_value  optimizer.cpp:207-219  -> sum of phi, same loop
// Error behaviour follows the reference: std::invalid_argument with its
// messages for bad arguments (LP_EINVAL); anything else is a runtime_error.
#include "spotsim/optimizer.hpp"

#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

#include "liveput.h"

namespace spotsim {
namespace {

lp_config to_c(const std::optional<ParallelConfig>& c) {
  return c ? lp_config{c->pipelines, c->stages} : lp_config{0, 0};
}

std::optional<ParallelConfig> from_c(lp_config c) {
  if (c.pipelines <= 0) return std::nullopt;
  return ParallelConfig{c.pipelines, c.stages};
}

struct Profile {
  lp_profile p{};
  std::vector<int32_t> depths;
  std::vector<double> rates;
};

// WorkloadProfile (perf_model.hpp:26-49) -> lp_profile; pipeline_rates as
// parallel arrays owned by the caller.
lp_profile profile_c(const WorkloadProfile& w, std::vector<int32_t>& depths, std::vector<double>& rates) {
  depths.clear();
  rates.clear();
  for (const auto& [d, r] : w.pipeline_rates) {
    depths.push_back(d);
    rates.push_back(r);
  }
  lp_profile p{};
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
  return p;
}

lp_costs costs_c(const CostTable& c) {
  return lp_costs{c.start_process_s, c.rendezvous_s,  c.cuda_context_s,
                  c.load_data_s,     c.build_model_s, c.update_comm_groups_s};
}

lp_options options_c(const PlannerOptions& o) {
  lp_options r{};
  r.interval_s = o.interval_s;
  r.lookahead = o.lookahead;
  r.mc_trials = o.mc_trials;
  r.exact_cap = o.exact_cap;
  r.mc_seed = o.mc_seed;
  r.rollback_penalty_s = o.rollback_penalty_s;
  r.strict_conditional = o.strict_conditional ? 1 : 0;
  return r;
}

[[noreturn]] void raise(lp_status s, const lp_handle* h) {
  const char* m = h ? lp_last_error(h) : lp_last_global_error();
  const std::string msg = m ? m : "liveput error";
  if (s == LP_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("liveput status " + std::to_string(static_cast<int>(s)) + ": " + msg);
}

int device_ordinal() {
  const char* e = std::getenv("LIVEPUT_DEVICE");
  return e ? std::atoi(e) : 0;
}

int n_configs(const WorkloadProfile& w, int n) {
  std::vector<int32_t> d;
  std::vector<double> r;
  const lp_profile p = profile_c(w, d, r);
  return lp_enumerate_configs(&p, n, nullptr, 0);
}

uint64_t level_key(int n_now, int n_next) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(n_now)) << 32) | static_cast<uint32_t>(n_next);
}

}  // namespace

std::optional<ParallelConfig> reactive_plan(int n_now, const WorkloadProfile& w) {
  std::vector<int32_t> d;
  std::vector<double> r;
  const lp_profile p = profile_c(w, d, r);
  lp_config out{0, 0};
  return lp_reactive_plan(&p, n_now, &out) ? from_c(out) : std::nullopt;
}

size_t Planner::KeyHash::operator()(const Key& k) const {
  uint64_t x = static_cast<uint64_t>(k.pd) * 0x9e3779b97f4a7c15ull;
  for (int v : {k.pp, k.nd, k.np, k.n_now, k.n_next}) x = (x ^ static_cast<uint64_t>(v)) * 0xbf58476d1ce4e5b9ull;
  return static_cast<size_t>(x ^ (x >> 31));
}

Planner::Planner(WorkloadProfile w, CostTable costs, PlannerOptions opt)
    : workload_(std::move(w)), costs_(costs), options_(opt) {
  const lp_profile p = profile_c(workload_, rate_depths_, rate_values_);
  const lp_costs c = costs_c(costs_);
  const lp_options o = options_c(options_);
  lp_handle* h = nullptr;
  const lp_status s = lp_create(&p, &c, &o, device_ordinal(), &h);
  if (s != LP_OK) raise(s, nullptr);
  h_ = h;
}

Planner::~Planner() {
  if (h_) lp_destroy(h_);
}

Planner::Planner(Planner&& o) noexcept
    : workload_(std::move(o.workload_)),
      costs_(o.costs_),
      options_(o.options_),
      rate_depths_(std::move(o.rate_depths_)),
      rate_values_(std::move(o.rate_values_)),
      h_(std::exchange(o.h_, nullptr)),
      phi_memo_(std::move(o.phi_memo_)),
      dp_levels_(std::move(o.dp_levels_)),
      dp_singles_(std::move(o.dp_singles_)) {}

Planner& Planner::operator=(Planner&& o) noexcept {
  if (this != &o) {
    if (h_) lp_destroy(h_);
    workload_ = std::move(o.workload_);
    costs_ = o.costs_;
    options_ = o.options_;
    rate_depths_ = std::move(o.rate_depths_);
    rate_values_ = std::move(o.rate_values_);
    h_ = std::exchange(o.h_, nullptr);
    phi_memo_ = std::move(o.phi_memo_);
    dp_levels_ = std::move(o.dp_levels_);
    dp_singles_ = std::move(o.dp_singles_);
  }
  return *this;
}

Planner::PhiValue Planner::phi(const std::optional<ParallelConfig>& prev,
                               const std::optional<ParallelConfig>& next, int n_now, int n_next) {
  const lp_config a = to_c(prev), b = to_c(next);
  const Key key{a.pipelines, a.stages, b.pipelines, b.stages, n_now, n_next};
  auto it = phi_memo_.find(key);
  if (it != phi_memo_.end()) return it->second;
  PhiValue v;
  const lp_status s = lp_phi(h_, a, b, n_now, n_next, &v.committed, &v.mig_cost_s);
  if (s != LP_OK) raise(s, h_);
  phi_memo_.emplace(key, v);
  return v;
}

void Planner::note_level(const std::optional<ParallelConfig>& prev, bool full_level, int n_now, int n_next) {
  if (full_level) {
    dp_levels_.insert(level_key(n_now, n_next));
  } else {
    const lp_config a = to_c(prev);
    dp_singles_.insert(Key{a.pipelines, a.stages, -1, -1, n_now, n_next});  // every next of n_next
  }
}

std::vector<PlanStep> Planner::dp_optimize(const std::optional<ParallelConfig>& current,
                                           const std::vector<int>& n_seq) {
  if (n_seq.size() < 2) throw std::invalid_argument("dp_optimize: need at least N_i and N_{i+1}");
  const int len = static_cast<int>(n_seq.size());
  std::vector<int32_t> ns(n_seq.begin(), n_seq.end());
  std::vector<lp_plan_step> out(len - 1);
  const lp_status s = lp_replan(h_, to_c(current), ns.data(), len, out.data(), nullptr, 0, nullptr);
  if (s != LP_OK) raise(s, h_);
  for (int j = 0; j + 1 < len; ++j) note_level(current, j > 0, n_seq[j], n_seq[j + 1]);
  std::vector<PlanStep> plan(len - 1);
  for (int j = 0; j + 1 < len; ++j)
    plan[j] = PlanStep{out[j].interval_index, from_c(out[j].config), out[j].expected_committed,
                       out[j].expected_mig_cost_s};
  return plan;
}

double Planner::sequence_value(const std::optional<ParallelConfig>& current,
                               const std::vector<std::optional<ParallelConfig>>& sequence,
                               const std::vector<int>& n_seq) {
  if (sequence.size() + 1 != n_seq.size())
    throw std::invalid_argument("sequence_value: sequence/N length mismatch");
  double value = 0.0;
  std::optional<ParallelConfig> prev = current;
  for (size_t j = 0; j < sequence.size(); ++j) {
    value += phi(prev, sequence[j], n_seq[j], n_seq[j + 1]).committed;
    prev = sequence[j];
  }
  return value;
}

size_t Planner::cache_size() const {
  // full DP levels: (|C(n_now)| + 1) x (|C(n_next)| + 1) keys each
  std::unordered_map<int, int> nc;
  auto count = [&](int n) {
    auto it = nc.find(n);
    if (it == nc.end()) it = nc.emplace(n, n_configs(workload_, n) + 1).first;
    return it->second;
  };
  size_t total = 0;
  for (uint64_t lk : dp_levels_)
    total += static_cast<size_t>(count(static_cast<int>(lk >> 32))) * count(static_cast<int>(lk & 0xffffffffu));
  // single-prev levels and phi calls not covered by a full level
  std::vector<int32_t> d;
  std::vector<double> r;
  const lp_profile p = profile_c(workload_, d, r);
  auto in_level = [&](int pd, int pp, int n_now) {  // prev is a node of a full level of n_now
    return pd <= 0 || (lp_depth_feasible(&p, pp) && static_cast<long long>(pd) * pp <= n_now);
  };
  std::unordered_set<Key, KeyHash> extra;
  for (const Key& s : dp_singles_) {
    if (dp_levels_.count(level_key(s.n_now, s.n_next)) && in_level(s.pd, s.pp, s.n_now)) continue;
    const int m = count(s.n_next) - 1;
    std::vector<lp_config> nx(m);
    if (m > 0) lp_enumerate_configs(&p, s.n_next, nx.data(), m);
    nx.push_back(lp_config{0, 0});
    for (const lp_config& c : nx) extra.insert(Key{s.pd, s.pp, c.pipelines, c.stages, s.n_now, s.n_next});
  }
  for (const auto& [k, v] : phi_memo_) {
    const bool next_node = k.nd <= 0 || (lp_depth_feasible(&p, k.np) && static_cast<long long>(k.nd) * k.np <= k.n_next);
    if (dp_levels_.count(level_key(k.n_now, k.n_next)) && in_level(k.pd, k.pp, k.n_now) && next_node) continue;
    extra.insert(k);
  }
  return total + extra.size();
}

}  // namespace spotsim
