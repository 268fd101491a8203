// lp_simulate.cpp — the replay driver, host C++.
//
// Restates the reference simulator's run() (simulator.cpp:119-340: the
// per-interval placement draw, rollback detection, migration costing,
// commit/revoke accounting through the sample manager, the ledger and the
// totals) around this library's planner.  Proactive / Ideal policies re-plan
// every interval through lp_replan on one handle, so the device histogram
// store persists across the replay like the reference's hist_cache_; every
// Proactive forecast of the trace comes from one lp_predict_windows launch
// (the history never depends on the decisions).  Compiled with
// -ffp-contract=off: every double is the reference's.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <optional>
#include <string>
#include <vector>

#include "liveput.h"
#include "lp_model.hpp"

namespace lp {
std::string& global_error();  // lp_api.cpp
}

namespace {

lp_status sim_fail(lp_status s, const char* fmt, ...) {
  char buf[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  lp::global_error() = buf;
  return s;
}

constexpr uint64_t kPlacementStream = 0xD00D;  // simulator.cpp:47-48
constexpr uint64_t kShuffleStream = 0x5AFE;

// splitmix64 (rng.hpp:11-41)
struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  uint64_t below(uint64_t b) {
    const uint64_t lim = UINT64_MAX - UINT64_MAX % b;
    uint64_t r;
    do r = next();
    while (r >= lim);
    return r % b;
  }
};

uint64_t mix3(uint64_t a, uint64_t b, uint64_t c) { return lp::mix_seed(lp::mix_seed(a, b), c); }

// sample_distinct (rng.cpp:8-19): the first k of a partial Fisher-Yates.
std::vector<int> distinct(int n, int k, Rng& r) {
  std::vector<int> pool(n);
  for (int i = 0; i < n; ++i) pool[i] = i;
  for (int i = 0; i < k; ++i) std::swap(pool[i], pool[i + static_cast<int>(r.below(n - i))]);
  pool.resize(k);
  return pool;
}

// Which samples of the current epoch are committed (simulator.cpp:51-105):
// commits draw from a shuffled pending pool, revokes put samples back.
class Samples {
 public:
  Samples(int epoch, uint64_t seed) : epoch_(epoch), seed_(seed), seen_(epoch, 0) { refill(); }
  void commit(long long count, std::vector<int>& out, int& ok) {
    for (long long c = 0; c < count; ++c) {
      if (pending_.empty()) refill();
      const int idx = pending_.back();
      pending_.pop_back();
      if (seen_[idx]) ok = 0;
      seen_[idx] = 1;
      ++in_epoch_;
      out.push_back(idx);
      if (in_epoch_ == epoch_) close_epoch(ok);
    }
  }
  void revoke(const std::vector<int>& idxs) {
    for (int idx : idxs) {
      if (!seen_[idx]) continue;  // its epoch already closed: only time is wasted
      seen_[idx] = 0;
      --in_epoch_;
      pending_.push_back(idx);
    }
  }
  int epochs() const { return done_; }

 private:
  void refill() {
    pending_.resize(epoch_);
    for (int i = 0; i < epoch_; ++i) pending_[i] = i;
    Rng r(mix3(seed_, kShuffleStream, static_cast<uint64_t>(done_)));
    for (size_t i = pending_.size(); i > 1; --i) std::swap(pending_[i - 1], pending_[r.below(i)]);
  }
  void close_epoch(int& ok) {
    for (uint8_t s : seen_)
      if (s != 1) ok = 0;
    std::fill(seen_.begin(), seen_.end(), 0);
    in_epoch_ = 0;
    ++done_;
    refill();
  }
  int epoch_;
  uint64_t seed_;
  std::vector<uint8_t> seen_;
  std::vector<int> pending_;
  int in_epoch_ = 0, done_ = 0;
};

using Config = std::optional<lp_config>;

int instances(const lp_config& c) { return c.pipelines * c.stages; }

// adjust_config (simulator.cpp:31-43)
Config adjust(const Config& planned, int n, lp::Model& m) {
  if (planned) {
    if (n >= instances(*planned)) return planned;
    const int d = n / planned->stages;
    if (d >= 1) return lp_config{d, planned->stages};
  }
  for (int p = n; p >= 1; --p)
    if (m.depth_ok(p)) return lp_config{1, p};
  return std::nullopt;
}

Config reactive(int n, lp::Model& m) {
  lp::Cfg c;
  if (!m.reactive(n, &c)) return std::nullopt;
  return lp_config{c.d, c.p};
}

// Pass 1, seed-independent: the configuration of every interval.  Under the
// planning policies it is adjust_config of the previous plan's first step
// (simulator.cpp:196-199), and the plan only sees the trace and that
// configuration — never the placements — so one planning pass serves every
// seed of a batch.
lp_status targets_of(lp_handle* shared, const lp_profile* profile, const lp_costs* costs,
                     const lp_options* planner_options, int32_t device, const int32_t* counts, int32_t len,
                     double T, int32_t capacity, const lp_policy* policy, lp::Model& model,
                     std::vector<Config>& targets) {
  const int kind = policy->kind;
  const bool needs_plan = kind == LP_POLICY_PROACTIVE || kind == LP_POLICY_IDEAL;
  targets.assign(len, std::nullopt);
  if (!needs_plan) {
    for (int i = 0; i < len; ++i) {
      const int n = counts[i];
      if (kind == LP_POLICY_REDUNDANCY) {
        const int fs = policy->redundancy_fixed_stages;
        const int d = fs > 0 ? n / fs : 0;
        if (d >= 1 && model.depth_ok(fs)) targets[i] = lp_config{d, fs};
      } else {
        targets[i] = reactive(n, model);
      }
    }
    return LP_OK;
  }
  // the planner: the injected handle, or a private one with this run's T and
  // rollback penalty (simulator.cpp:126-130)
  lp_handle* h = shared;
  lp_handle* own = nullptr;
  if (!h) {
    lp_options o = *planner_options;
    o.interval_s = T;
    o.rollback_penalty_s = policy->ckpt_restore_cost_s;
    lp_status s = lp_create(profile, costs, &o, device, &own);
    if (s != LP_OK) return s;
    lp_set_hist_cache(own, 1, 0);
    h = own;
  }
  struct Guard {
    lp_handle* h;
    ~Guard() {
      if (h) lp_destroy(h);
    }
  } guard{own};
  // Proactive forecasts of every interval in one launch: window i of
  // [c0]*(H-1) + counts + I pad values is the history at interval i, padded
  // as simulator.cpp:311-313 does.
  const int I = std::max(1, policy->lookahead);
  std::vector<int32_t> fc_all;
  if (kind == LP_POLICY_PROACTIVE) {
    lp_forecast_config fc = lp_forecast_defaults(capacity);
    fc.history_len = std::max(3, policy->history);
    fc.lookahead = I;
    const int H = fc.history_len;
    std::vector<int32_t> series(H - 1, counts[0]);
    series.insert(series.end(), counts, counts + len);
    series.insert(series.end(), I, 0);
    fc_all.assign(static_cast<size_t>(len) * I, 0);
    int32_t nw = 0;
    const int32_t m = policy->method;
    lp_status s = lp_predict_windows(series.data(), (int32_t)series.size(), &fc, &m, 1, device, fc_all.data(),
                                     nullptr, &nw);
    if (s != LP_OK) return s;
    if (nw < len) return sim_fail(LP_ECUDA, "simulate: forecast windows %d < %d", nw, len);
  }
  Config planned;
  std::vector<int32_t> ns;
  std::vector<lp_plan_step> steps;
  for (int i = 0; i < len; ++i) {
    const int n = counts[i];
    const Config target = (i == 0) ? reactive(n, model) : adjust(planned, n, model);
    targets[i] = target;
    ns.assign(1, n);
    if (kind == LP_POLICY_IDEAL) {
      for (int j = 1; j <= I; ++j) ns.push_back(i + j < len ? counts[i + j] : counts[len - 1]);
    } else {
      ns.insert(ns.end(), fc_all.begin() + static_cast<size_t>(i) * I, fc_all.begin() + static_cast<size_t>(i + 1) * I);
    }
    steps.resize(ns.size() - 1);
    const lp_config cur = target ? *target : lp_config{0, 0};
    lp_status s = lp_replan(h, cur, ns.data(), (int32_t)ns.size(), steps.data(), nullptr, 0, nullptr);
    if (s != LP_OK) return sim_fail(s, "simulate: re-plan at interval %d: %s", i, lp_last_error(h));
    planned = steps[0].config.pipelines > 0 ? Config(steps[0].config) : std::nullopt;
  }
  return LP_OK;
}

// Pass 2, per seed: placements, rollbacks, migration costs, commits and the
// ledger (simulator.cpp:152-340) for the given configuration sequence.
void run_seed(const std::vector<Config>& targets, const lp_profile* profile, const lp_costs* costs,
              const int32_t* counts, int32_t len, double T, const lp_policy* policy, uint64_t seed, int epoch,
              double spot_price_per_hour, double ondemand_price_per_hour, lp::Model& model,
              lp_sim_report* report, lp_interval_log* logs) {
  const int B = profile->minibatch_size;
  const int kind = policy->kind;
  lp_sim_report rep{};
  rep.seed = seed;
  rep.sample_accounting_ok = 1;
  Samples samples(epoch, seed);
  struct Commit {
    std::vector<int> samples;
    double seconds = 0.0;
  };
  std::vector<Commit> commits(len);
  Config cfg;
  int alive = 0, last_save = 0;
  auto revoke = [&](int j) {
    Commit& c = commits[j];
    if (c.samples.empty()) return;
    lp_interval_log& lj = logs[j];
    samples.revoke(c.samples);
    lj.rolled_back += static_cast<long long>(c.samples.size());
    lj.committed -= static_cast<long long>(c.samples.size());
    const double moved = std::min(c.seconds, lj.ledger.effective_s);
    lj.ledger.effective_s -= moved;
    lj.ledger.wasted_rollback_s += moved;
    c.samples.clear();
    c.seconds = 0.0;
  };
  for (int i = 0; i < len; ++i) {
    const int n = counts[i];
    const int k_dead = std::max(0, alive - n);
    const int fresh = std::max(0, n - alive);
    std::vector<int> dead;  // which allocated instances die: a per-interval stream
    if (k_dead > 0) {
      Rng r(mix3(seed, kPlacementStream, static_cast<uint64_t>(i)));
      dead = distinct(alive, k_dead, r);
    }
    std::vector<int> surv;  // per stage of the outgoing config
    bool wiped = false;
    if (cfg) {
      surv.assign(cfg->stages, cfg->pipelines);
      for (int idx : dead)
        if (idx < instances(*cfg)) --surv[idx % cfg->stages];
      for (int s : surv) wiped |= s == 0;
    }

    const Config target = targets[i];

    lp_interval_log log{};
    log.interval = i;
    log.available = n;

    bool rollback = false;
    double restore_due = 0.0;
    if (kind == LP_POLICY_CHECKPOINT) {
      if (k_dead > 0 && i > 0) {  // back to the last periodic save
        rollback = true;
        for (int j = last_save; j < i; ++j) revoke(j);
      }
    } else if (kind != LP_POLICY_REDUNDANCY) {
      if (cfg && wiped && i > 0) {  // the one-interval-old in-memory checkpoint
        rollback = true;
        revoke(i - 1);
        restore_due = policy->ckpt_restore_cost_s;
      }
    }
    if (rollback) ++rep.rollback_events;

    double mig_due = 0.0;
    int mig_kind = LP_MIG_NONE;
    if (i > 0 && target && kind != LP_POLICY_REDUNDANCY && kind != LP_POLICY_CHECKPOINT) {
      if (!cfg || wiped) {
        mig_due = lp_resume_cost(profile, costs, *target);
        mig_kind = LP_MIG_PIPELINE;
      } else {
        int mn = cfg->pipelines;  // transition_outcome (migration.cpp:91-98)
        for (int s : surv) mn = std::min(mn, s);
        int32_t rb = 0;
        lp_transition_outcome(profile, costs, mn, *cfg, *target, fresh, &mig_due, &mig_kind, &rb);  // args valid
      }
    }

    double save_due = 0.0, restart_due = 0.0;
    if (kind == LP_POLICY_CHECKPOINT && target && i > 0) {
      if (rollback) restart_due = policy->ckpt_restart_cost_s;
      if (i - last_save >= policy->ckpt_period_intervals) {
        save_due = policy->ckpt_save_cost_s;
        last_save = i;
      }
    }
    if (kind == LP_POLICY_CHECKPOINT && rollback) last_save = i;  // resume point after restart

    if (target) {
      double avail = T;
      const double mig_s = std::min(avail, mig_due);
      avail -= mig_s;
      const double restore_s = std::min(avail, restore_due);
      avail -= restore_s;
      const double restart_s = std::min(avail, restart_due);
      avail -= restart_s;
      const double save_s = std::min(avail, save_due);
      avail -= save_s;
      const double t_eff = avail;
      double rate = model.rate(target->pipelines, target->stages);
      if (kind == LP_POLICY_REDUNDANCY) rate *= policy->redundancy_slowdown;
      const long long mb = rate > 0 ? static_cast<long long>(std::floor(rate * t_eff / B)) : 0;
      const long long committed = mb * B;
      Commit& c = commits[i];
      samples.commit(committed, c.samples, rep.sample_accounting_ok);
      const int active = instances(*target);
      c.seconds = rate > 0 ? static_cast<double>(committed) / rate * active : 0.0;
      log.pipelines = target->pipelines;
      log.stages = target->stages;
      log.throughput = rate;
      log.committed = committed;
      log.migration = mig_kind;
      log.ledger.effective_s = t_eff * active;
      log.ledger.migration_s = mig_s * active;
      log.ledger.checkpoint_s = (save_s + restart_s) * active;
      log.ledger.wasted_rollback_s = restore_s * active;
      log.ledger.idle_s = (n - active) * T;
    } else {
      ++rep.suspended_intervals;
      log.ledger.idle_s = static_cast<double>(n) * T;
    }
    logs[i] = log;
    cfg = target;
    alive = n;

  }

  for (int i = 0; i < len; ++i) {  // totals (simulator.cpp:321-329)
    rep.committed_samples += logs[i].committed;
    rep.ledger.effective_s += logs[i].ledger.effective_s;
    rep.ledger.migration_s += logs[i].ledger.migration_s;
    rep.ledger.checkpoint_s += logs[i].ledger.checkpoint_s;
    rep.ledger.wasted_rollback_s += logs[i].ledger.wasted_rollback_s;
    rep.ledger.idle_s += logs[i].ledger.idle_s;
  }
  rep.wall_time_s = static_cast<double>(len) * T;
  double inst = 0.0;  // integrate_instance_seconds (trace.cpp:210-214)
  for (int i = 0; i < len; ++i) inst += static_cast<double>(counts[i]) * T;
  rep.instance_seconds = inst;
  rep.instance_hours = rep.instance_seconds / 3600.0;
  rep.spot_cost = spot_price_per_hour * rep.instance_hours;
  rep.ondemand_cost = ondemand_price_per_hour * rep.instance_hours;
  if (rep.committed_samples > 0) {
    rep.has_cost_per_sample = 1;
    rep.cost_per_sample = rep.spot_cost / static_cast<double>(rep.committed_samples);
  }
  rep.epochs_completed = samples.epochs();
  (void)model;
  *report = rep;
}

}  // namespace

extern "C" {

lp_policy lp_policy_defaults(int32_t kind) {
  lp_policy p{};
  p.kind = kind;
  p.lookahead = 12;
  p.method = LP_PREDICT_ARIMA;
  p.history = 12;
  p.ckpt_period_intervals = 5;
  p.ckpt_save_cost_s = 10.0;
  p.ckpt_restore_cost_s = 30.0;
  p.ckpt_restart_cost_s = 30.0;
  p.redundancy_fixed_stages = 4;
  p.redundancy_slowdown = 0.75;
  return p;
}

lp_status lp_simulate_batch(lp_handle* shared, const lp_profile* profile, const lp_costs* costs,
                            const lp_options* planner_options, int32_t device, const int32_t* counts,
                            int32_t len, double interval_s, int32_t capacity, const lp_policy* policy,
                            const uint64_t* seeds, int32_t n_seeds, int32_t epoch_samples,
                            double spot_price_per_hour, double ondemand_price_per_hour,
                            lp_sim_report* reports, lp_interval_log* logs) {
  if (!profile || !costs || !planner_options || !policy || !reports || !logs || !seeds || n_seeds < 1 ||
      (!counts && len > 0))
    return sim_fail(LP_EINVAL, "simulate: null argument");
  if (len <= 0) return sim_fail(LP_EINVAL, "run: empty series");
  if (policy->kind < LP_POLICY_PROACTIVE || policy->kind > LP_POLICY_REDUNDANCY)
    return sim_fail(LP_EINVAL, "simulate: unknown policy");
  lp::Model model(*profile);
  std::vector<Config> targets;
  lp_status s = targets_of(shared, profile, costs, planner_options, device, counts, len, interval_s, capacity,
                           policy, model, targets);
  if (s != LP_OK) return s;
  const int epoch = epoch_samples > 0 ? epoch_samples : 64 * profile->minibatch_size;
  for (int q = 0; q < n_seeds; ++q)
    run_seed(targets, profile, costs, counts, len, interval_s, policy, seeds[q], epoch, spot_price_per_hour,
             ondemand_price_per_hour, model, reports + q, logs + static_cast<size_t>(q) * len);
  return LP_OK;
}

lp_status lp_simulate(lp_handle* shared, const lp_profile* profile, const lp_costs* costs,
                      const lp_options* planner_options, int32_t device, const int32_t* counts,
                      int32_t len, double interval_s, int32_t capacity, const lp_policy* policy,
                      uint64_t seed, int32_t epoch_samples, double spot_price_per_hour,
                      double ondemand_price_per_hour, lp_sim_report* report, lp_interval_log* logs) {
  return lp_simulate_batch(shared, profile, costs, planner_options, device, counts, len, interval_s, capacity,
                           policy, &seed, 1, epoch_samples, spot_price_per_hour, ondemand_price_per_hour,
                           report, logs);
}

}  // extern "C"
