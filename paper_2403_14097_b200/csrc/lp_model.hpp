// lp_model.hpp — host-side table producers for the liveput planner.
//
// The reference keeps throughput/feasibility/config enumeration on the host
// (perf_model.cpp) and so do we: the device never evaluates a profile, it
// reads tables built here.  Every formula keeps the reference's operand order
// so the FP64 tables are bit-identical (compiled with -ffp-contract=off).
#pragma once

#include <cstdint>
#include <vector>

#include "liveput.h"

namespace lp {

struct Cfg {
  int d = 0;  // pipelines (0 = suspended)
  int p = 0;  // stages
};

class Model {
 public:
  Model() = default;
  explicit Model(const lp_profile& prof);

  // perf_model.cpp:5-8
  bool depth_ok(int stages) const;
  // perf_model.cpp:14-42 (+ microbatches_per_pipeline, perf_model.hpp:44-48)
  double rate(int d, int p) const;
  // memoised rate(d, p): the profile is fixed for the life of a handle
  double rate_cached(int d, int p);
  // perf_model.cpp:44-52 — ascending P, descending D (fixes DP tie order)
  const std::vector<Cfg>& configs(int n);
  // optimizer.cpp:11-25
  bool reactive(int n, Cfg* out);

  // migration.cpp:32-34 and :39-42 (per target depth)
  double pipe_transfer(int stages) const;
  double inter_unit(int stages) const;

  const lp_profile& profile() const { return prof_; }

 private:
  lp_profile prof_{};
  std::vector<int32_t> depths_;
  std::vector<double> rates_;
  std::vector<std::vector<Cfg>> cfg_cache_;
  std::vector<std::vector<double>> rate_cache_;  // [p][d]
  std::vector<char> cfg_have_;
  bool lookup_rate(int p, double* r) const;
};

// preemption.cpp:10-21 (long double, saturating at 9.22e18)
uint64_t scenario_count(int n, int k);
// rng.hpp:46-55
uint64_t mix_seed(uint64_t a, uint64_t b);

// CostTable scalars pre-combined in the reference's addition order
// (migration.cpp:49-104).
struct CostScalars {
  double fresh_fixed;  // ((start + rendezvous) + cuda_context) + load_data
  double build;
  double update;
};
CostScalars cost_scalars(const lp_costs& c);

}  // namespace lp
