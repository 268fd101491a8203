// lp_model.cpp — host table producers (see lp_model.hpp).  Compiled by g++
// with -ffp-contract=off and no -march, like the reference's Release build,
// so every FP64 table entry is bit-identical to the reference's value.
#include "lp_model.hpp"

#include <algorithm>

namespace lp {

Model::Model(const lp_profile& prof) : prof_(prof) {
  for (int i = 0; i < prof.n_rates; ++i) {
    depths_.push_back(prof.rate_depths[i]);
    rates_.push_back(prof.rate_values[i]);
  }
  prof_.rate_depths = depths_.empty() ? nullptr : depths_.data();
  prof_.rate_values = rates_.empty() ? nullptr : rates_.data();
}

bool Model::depth_ok(int stages) const {
  if (stages < 1) return false;
  const double per_stage = prof_.memory_fixed_bytes + prof_.memory_per_stage_bytes / stages;
  return per_stage <= prof_.device_memory_bytes;
}

bool Model::lookup_rate(int p, double* r) const {
  for (size_t i = 0; i < depths_.size(); ++i)
    if (depths_[i] == p) {
      *r = rates_[i];
      return true;
    }
  return false;
}

double Model::rate(int d, int p) const {
  if (d < 1 || !depth_ok(p)) return 0.0;
  const long long batch = prof_.minibatch_size;
  const long long ub = prof_.microbatch_size;
  // microbatches per pipeline: ceil(B / (D*u)), at least 1 (returned as int)
  const long long per_pipe = static_cast<long long>(d) * prof_.microbatch_size;
  const long long mb_raw = (prof_.minibatch_size + per_pipe - 1) / per_pipe;
  const long long mb = static_cast<int>(mb_raw < 1 ? 1 : mb_raw);

  double grad_sync = 0.0;
  if (d > 1) {
    // ring all-reduce of each stage's gradient shard across D replicas
    grad_sync = 2.0 * (d - 1) / d * (prof_.param_bytes / p) * prof_.beta_s_per_byte +
                2.0 * (d - 1) * prof_.alpha_s;
  }
  double profiled;
  if (lookup_rate(p, &profiled)) {
    if (grad_sync == 0.0) return profiled * static_cast<double>(batch) / static_cast<double>(mb * ub);
    const double pipe_s = static_cast<double>(mb * ub) / profiled;
    return static_cast<double>(batch) / (pipe_s + grad_sync);
  }
  const double stage_s = prof_.compute_per_microbatch_s / p;
  const double pipe_s =
      static_cast<double>(mb + p - 1) * stage_s +
      2.0 * (p - 1) * (prof_.alpha_s + prof_.activation_bytes * prof_.beta_s_per_byte);
  return static_cast<double>(batch) / (pipe_s + grad_sync);
}

double Model::rate_cached(int d, int p) {
  if (p < 1 || d < 1) return rate(d, p);
  if (static_cast<int>(rate_cache_.size()) <= p) rate_cache_.resize(p + 1);
  std::vector<double>& row = rate_cache_[p];
  while (static_cast<int>(row.size()) <= d) row.push_back(rate(static_cast<int>(row.size()), p));
  return row[d];
}

const std::vector<Cfg>& Model::configs(int n) {
  static const std::vector<Cfg> kEmpty;
  if (n <= 0) return kEmpty;
  if (static_cast<int>(cfg_cache_.size()) <= n) {
    cfg_cache_.resize(n + 1);
    cfg_have_.resize(n + 1, 0);
  }
  if (!cfg_have_[n]) {
    std::vector<Cfg>& out = cfg_cache_[n];
    for (int p = 1; p <= n; ++p) {
      if (!depth_ok(p)) continue;
      for (int d = n / p; d >= 1; --d) out.push_back({d, p});
    }
    cfg_have_[n] = 1;
  }
  return cfg_cache_[n];
}

bool Model::reactive(int n, Cfg* out) {
  bool have = false;
  Cfg best;
  double best_rate = 0.0;
  for (const Cfg& c : configs(n)) {
    const double r = rate(c.d, c.p);
    if (r <= 0.0) continue;
    const bool better = !have || r > best_rate ||
                        (r == best_rate && (c.d > best.d || (c.d == best.d && c.p < best.p)));
    if (better) {
      have = true;
      best = c;
      best_rate = r;
    }
  }
  if (have && out) *out = best;
  return have;
}

double Model::pipe_transfer(int stages) const {
  return prof_.param_bytes * prof_.beta_s_per_byte + stages * prof_.alpha_s;
}

double Model::inter_unit(int stages) const {
  return (prof_.param_bytes / stages) * prof_.beta_s_per_byte + prof_.alpha_s;
}

uint64_t scenario_count(int n, int k) {
  if (k < 0 || k > n) return 0;
  k = std::min(k, n - k);
  long double c = 1.0L;
  const long double sat = 9.22e18L;
  for (int i = 1; i <= k; ++i) {
    c = c * (n - k + i) / i;
    if (c > sat) return static_cast<uint64_t>(sat);
  }
  return static_cast<uint64_t>(c + 0.5L);
}

uint64_t mix_seed(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

CostScalars cost_scalars(const lp_costs& c) {
  CostScalars s;
  s.fresh_fixed = c.start_process_s + c.rendezvous_s + c.cuda_context_s + c.load_data_s;
  s.build = c.build_model_s;
  s.update = c.update_comm_groups_s;
  return s;
}

}  // namespace lp
