// spotsim/optimizer.hpp — drop-in replacement header for the reference's
// Planner (/root/reference/proj/core/include/spotsim/optimizer.hpp:13-92).
//
// Placed ahead of the reference's include directory, it gives every caller
// (simulator.cpp:119-340, commands.cpp, proj/tests/*) the same public
// interface — PlannerOptions, PlanStep, reactive_plan, Planner's ctor,
// accessors, phi, dp_optimize, sequence_value, cache_size — while the
// implementation (adapter/optimizer.cpp) runs the histograms, phi and the
// DP on the B200 through the C ABI in include/liveput.h.  Only the private
// section differs: a liveput handle instead of the host caches.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "spotsim/migration.hpp"
#include "spotsim/perf_model.hpp"
#include "spotsim/preemption.hpp"

struct lp_handle;

namespace spotsim {

// optimizer.hpp:13-23 (same members, same defaults)
struct PlannerOptions {
  double interval_s = 60.0;
  int lookahead = 12;
  int mc_trials = 200;
  uint64_t exact_cap = 2000;
  uint64_t mc_seed = 0x5eedULL;
  double rollback_penalty_s = 30.0;
  bool strict_conditional = false;
};

// optimizer.hpp:26-31; config == nullopt is the suspended state.
struct PlanStep {
  int interval_index = 0;
  std::optional<ParallelConfig> config;
  double expected_committed = 0.0;
  double expected_mig_cost_s = 0.0;
};

// optimizer.hpp:36 — lp_reactive_plan.
std::optional<ParallelConfig> reactive_plan(int n_now, const WorkloadProfile& w);

class Planner {
 public:
  // optimizer.hpp:43.  Creates the device handle on the calling thread's
  // current CUDA device (LIVEPUT_DEVICE overrides); throws std::runtime_error
  // when no B200 is available — there is no CPU fallback.
  Planner(WorkloadProfile w, CostTable costs, PlannerOptions opt = {});
  ~Planner();
  Planner(Planner&&) noexcept;
  Planner& operator=(Planner&&) noexcept;
  Planner(const Planner&) = delete;
  Planner& operator=(const Planner&) = delete;

  const WorkloadProfile& workload() const { return workload_; }
  const CostTable& costs() const { return costs_; }
  const PlannerOptions& options() const { return options_; }

  struct PhiValue {
    double committed = 0.0;
    double mig_cost_s = 0.0;
  };

  // optimizer.hpp:57-58 — lp_phi, memoised per key like the reference.
  PhiValue phi(const std::optional<ParallelConfig>& prev, const std::optional<ParallelConfig>& next,
               int n_now, int n_next);

  // optimizer.hpp:64-65 — lp_replan (histograms + max-plus DP + traceback on
  // the device).  Throws std::invalid_argument with the reference's messages.
  std::vector<PlanStep> dp_optimize(const std::optional<ParallelConfig>& current,
                                    const std::vector<int>& n_seq);

  // optimizer.hpp:69-71 — sum of phi over the sequence.
  double sequence_value(const std::optional<ParallelConfig>& current,
                        const std::vector<std::optional<ParallelConfig>>& sequence,
                        const std::vector<int>& n_seq);

  // optimizer.hpp:73 — number of distinct transition values (prev, next,
  // n_now, n_next) this planner has evaluated, through phi or a DP.
  size_t cache_size() const;

 private:
  struct Key {
    int pd, pp, nd, np, n_now, n_next;
    bool operator==(const Key& o) const {
      return pd == o.pd && pp == o.pp && nd == o.nd && np == o.np && n_now == o.n_now && n_next == o.n_next;
    }
  };
  struct KeyHash {
    size_t operator()(const Key& k) const;
  };
  void note_level(const std::optional<ParallelConfig>& prev, bool full_level, int n_now, int n_next);

  WorkloadProfile workload_;
  CostTable costs_;
  PlannerOptions options_;
  std::vector<int32_t> rate_depths_;
  std::vector<double> rate_values_;
  lp_handle* h_ = nullptr;
  std::unordered_map<Key, PhiValue, KeyHash> phi_memo_;
  // transition keys a DP evaluated: whole (n_now, n_next) levels, and the
  // single-prev level 0 of each re-plan
  std::unordered_set<uint64_t> dp_levels_;
  std::unordered_set<Key, KeyHash> dp_singles_;
};

}  // namespace spotsim
