// C++ parity tests through the header-only facade (include/spotsim_b200/planner.hpp)
// -> C ABI -> sm_100a kernels.  They restate the behaviours the reference's
// own optimizer/preemption tests pin (proj/tests/test_optimizer.cpp,
// test_preemption.cpp), plus the SURVEY §8c known answers.  Built and run by
// tests/test_cpp_facade.py; exits non-zero on any failure.
#include <cmath>
#include <cstdio>
#include <functional>
#include <optional>
#include <vector>

#include "spotsim_b200/planner.hpp"

using namespace spotsim_b200;

static int g_fail = 0, g_pass = 0;
#define EXPECT(cond)                                                        \
  do {                                                                      \
    if (cond) ++g_pass;                                                     \
    else {                                                                  \
      ++g_fail;                                                             \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);  \
    }                                                                       \
  } while (0)

// small deterministic generator for random instances (splitmix64 stream)
struct Gen {
  uint64_t s;
  explicit Gen(uint64_t seed) : s(seed) {}
  uint64_t next() { return mix_seed(s++, 0x1234); }
  int below(int b) { return static_cast<int>(next() % static_cast<uint64_t>(b)); }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

static WorkloadProfile six_instance() {  // two rate-table depths, P >= 2
  WorkloadProfile w;
  w.compute_per_microbatch_s = 1.0;
  w.minibatch_size = 6;
  w.microbatch_size = 1;
  w.device_memory_bytes = 1.0;
  w.memory = {0.0, 2.0};
  w.pipeline_rates = {{2, 30.0}, {3, 50.0}};
  return w;
}

static WorkloadProfile lm_1p5b() {
  WorkloadProfile w;
  w.compute_per_microbatch_s = 1.0;
  w.param_bytes = 3.0e9;
  w.activation_bytes = 4.0e7;
  w.minibatch_size = 128;
  w.microbatch_size = 1;
  w.device_memory_bytes = 16.0e9;
  w.memory = {1.5e9, 88.0e9};
  w.alpha_s = 5e-3;
  w.beta_s_per_byte = 2.5e-9;
  return w;
}

static WorkloadProfile random_profile(Gen& g) {
  WorkloadProfile w;
  w.compute_per_microbatch_s = 0.05 + g.unit() * 2.0;
  w.param_bytes = g.unit() * 4e9;
  w.activation_bytes = g.unit() * 1e7;
  w.microbatch_size = 1 + g.below(4);
  w.minibatch_size = w.microbatch_size * (1 + g.below(32));
  w.device_memory_bytes = 16.0;
  w.memory = {0.0, 16.0 * (1 + g.below(3))};
  w.alpha_s = g.unit() * 0.01;
  w.beta_s_per_byte = g.unit() * 2e-9;
  return w;
}

static CostTable random_costs(Gen& g) {
  return {g.unit(), g.unit() * 10, g.unit() * 10, g.unit() * 10, g.unit() * 10, g.unit() * 20};
}

static PlannerOptions exact_opts() {
  PlannerOptions o;
  o.exact_cap = 100000;
  return o;
}

// brute force over every configuration sequence, using the planner's phi
static double exhaustive(Planner& pl, const std::optional<ParallelConfig>& cur,
                         const std::vector<int>& ns) {
  const int H = static_cast<int>(ns.size()) - 1;
  double best = -1.0;
  std::function<void(int, double, std::optional<ParallelConfig>)> rec =
      [&](int j, double acc, std::optional<ParallelConfig> prev) {
        if (j == H) {
          best = std::max(best, acc);
          return;
        }
        std::vector<std::optional<ParallelConfig>> ch;
        for (const auto& c : enumerate_configs(ns[j + 1], pl.workload())) ch.emplace_back(c);
        ch.emplace_back(std::nullopt);
        for (const auto& c : ch) rec(j + 1, acc + pl.phi(prev, c, ns[j], ns[j + 1]).committed, c);
      };
  rec(0, 0.0, cur);
  return best;
}

int main() {
  // ---- phi basics (test_optimizer.cpp:19-68 behaviours)
  {
    Planner pl(six_instance(), CostTable{}, exact_opts());
    auto v = pl.phi(ParallelConfig{2, 3}, ParallelConfig{2, 3}, 6, 6);
    EXPECT(std::abs(v.committed - 100.0 * 60.0) < 1e-9);
    EXPECT(v.mig_cost_s == 0.0);
    EXPECT(pl.phi(ParallelConfig{2, 3}, ParallelConfig{1, 1}, 6, 6).committed == 0.0);
    EXPECT(pl.phi(ParallelConfig{2, 3}, ParallelConfig{4, 2}, 6, 6).committed == 0.0);
    EXPECT(pl.phi(ParallelConfig{2, 3}, std::nullopt, 6, 0).committed == 0.0);
    // growth 4 -> 6 keeps the depth and adds one pipeline: inter-stage transfer
    auto g = pl.phi(ParallelConfig{2, 2}, ParallelConfig{3, 2}, 4, 6);
    const CostTable c;
    const double base = c.start_process_s + c.rendezvous_s + c.cuda_context_s + c.load_data_s +
                        c.build_model_s + c.update_comm_groups_s;
    EXPECT(std::abs(g.mig_cost_s - base) < 1e-9);  // fresh fixed terms; this profile moves no bytes
    EXPECT(std::abs(g.committed - 90.0 * (60.0 - g.mig_cost_s)) < 1e-9);
  }
  {
    Gen g(5150);
    for (int trial = 0; trial < 40; ++trial) {
      WorkloadProfile w = random_profile(g);
      CostTable costs = random_costs(g);
      PlannerOptions o = exact_opts();
      o.interval_s = 10.0;
      Planner pl(w, costs, o);
      const int a = 1 + g.below(8), b = 1 + g.below(8);
      auto pc = enumerate_configs(a, w), nc = enumerate_configs(b, w);
      if (pc.empty() || nc.empty()) continue;
      const auto& p = pc[g.below(static_cast<int>(pc.size()))];
      const auto& q = nc[g.below(static_cast<int>(nc.size()))];
      auto v = pl.phi(p, q, a, b);
      EXPECT(v.committed >= 0.0);
      EXPECT(v.committed <= throughput(q, w) * o.interval_s + 1e-9);
    }
  }
  // ---- reactive / one-step / greedy (test_optimizer.cpp:70-105 behaviours)
  {
    const WorkloadProfile w = six_instance();
    auto r = reactive_plan(6, w);
    EXPECT(r && *r == (ParallelConfig{2, 3}));
    EXPECT(!reactive_plan(0, w) && !reactive_plan(1, w));
    Planner zero(w, CostTable{0, 0, 0, 0, 0, 0}, exact_opts());
    auto plan = zero.dp_optimize(ParallelConfig{2, 3}, {6, 6});
    EXPECT(plan.size() == 1 && plan[0].config && *plan[0].config == *reactive_plan(6, w));
    Planner pl(w, CostTable{}, exact_opts());
    const std::vector<int> ns{6, 6, 4, 4};
    auto dp = pl.dp_optimize(ParallelConfig{2, 3}, ns);
    std::vector<std::optional<ParallelConfig>> seq, greedy;
    for (const auto& s : dp) seq.push_back(s.config);
    for (size_t j = 1; j < ns.size(); ++j) greedy.push_back(reactive_plan(ns[j], w));
    EXPECT(pl.sequence_value(ParallelConfig{2, 3}, seq, ns) >=
           pl.sequence_value(ParallelConfig{2, 3}, greedy, ns));
    auto susp = pl.dp_optimize(ParallelConfig{2, 2}, {4, 1, 4});
    EXPECT(susp.size() == 2 && !susp[0].config && susp[0].expected_committed == 0.0 && susp[1].config);
  }
  // ---- DP value == exhaustive search (test_optimizer.cpp:107-131 behaviour)
  {
    Gen g(161803);
    int checked = 0;
    for (int trial = 0; trial < 60; ++trial) {
      WorkloadProfile w = random_profile(g);
      CostTable costs = random_costs(g);
      Planner pl(w, costs, exact_opts());
      const int H = 1 + g.below(3);
      std::vector<int> ns(H + 1);
      for (int& x : ns) x = g.below(9);
      auto sc = enumerate_configs(ns[0], w);
      std::optional<ParallelConfig> cur;
      if (!sc.empty()) cur = sc[g.below(static_cast<int>(sc.size()))];
      auto plan = pl.dp_optimize(cur, ns);
      std::vector<std::optional<ParallelConfig>> seq;
      for (const auto& s : plan) seq.push_back(s.config);
      EXPECT(pl.sequence_value(cur, seq, ns) == exhaustive(pl, cur, ns));
      ++checked;
    }
    EXPECT(checked == 60);
  }
  // ---- six-instance expectations (test_preemption.cpp:97-120 behaviours)
  {
    Planner pl(six_instance(), CostTable{}, exact_opts());
    EXPECT(expected_liveput(pl, {2, 3}, 6, 1, EvalMode::Exact()) == 50.0);
    EXPECT(expected_liveput(pl, {3, 2}, 6, 1, EvalMode::Exact()) == 60.0);
    EXPECT(expected_liveput(pl, {2, 3}, 6, 2, EvalMode::Exact()) == 40.0);
    EXPECT(expected_liveput(pl, {3, 2}, 6, 2, EvalMode::Exact()) == 48.0);
    EXPECT(expected_liveput(pl, {2, 3}, 6, 0, EvalMode::Exact()) == 100.0);
    EXPECT(expected_liveput(pl, {2, 3}, 6, 6, EvalMode::Exact()) == 0.0);
    const double mc = expected_liveput(pl, {3, 2}, 6, 2, EvalMode::MC(10000, 9));
    EXPECT(std::abs(mc - 48.0) / 48.0 < 0.02);
  }
  // ---- SURVEY §8c known answers (GPT-2 profile, 1e4 MC trials)
  {
    PlannerOptions o;
    o.mc_trials = 10000;
    Planner pl(lm_1p5b(), CostTable{}, o);
    uint64_t tot = 0;
    auto cnt = pl.survivor_counts({4, 7}, 32, 3, &tot);
    EXPECT(tot == 10000 && cnt == (std::vector<uint64_t>{0, 46, 2412, 7535, 7}));
    auto a = pl.phi(ParallelConfig{4, 7}, ParallelConfig{4, 7}, 32, 29);
    EXPECT(a.committed == 675.38034536719283 && a.mig_cost_s == 16.070126642857144);
    auto b = pl.phi(ParallelConfig{4, 7}, ParallelConfig{3, 8}, 32, 29);
    EXPECT(b.committed == 533.35706340378192 && b.mig_cost_s == 22.539999999999999);
    const std::vector<int> ns{32, 28, 28, 26, 29, 26, 26, 21, 23, 23, 21, 25, 22};
    auto cur = reactive_plan(32, lm_1p5b());
    EXPECT(cur && *cur == (ParallelConfig{4, 8}));
    auto plan = pl.dp_optimize(cur, ns);
    std::vector<std::optional<ParallelConfig>> seq;
    for (size_t j = 0; j < plan.size(); ++j) {
      seq.push_back(plan[j].config);
      EXPECT(plan[j].config && *plan[j].config == (j < 6 ? ParallelConfig{3, 8} : ParallelConfig{3, 7}));
    }
    EXPECT(pl.sequence_value(cur, seq, ns) == 8460.1874990222786);
  }
  // ---- errors map to std::invalid_argument
  {
    Planner pl(lm_1p5b(), CostTable{}, PlannerOptions{});
    bool thrown = false;
    try {
      pl.dp_optimize(ParallelConfig{4, 8}, {32});
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    EXPECT(thrown);
  }
  // ---- migration planning (test_migration.cpp:8-75 behaviours)
  {
    const WorkloadProfile w = lm_1p5b();
    const CostTable costs;
    PreemptionVector none(12, 0);
    MigrationPlan keep = plan_migration(Topology{3, 4, 0}, none, {3, 4}, w, costs);
    EXPECT(keep.kind == MigrationKind::none && keep.moves.empty() && keep.est_cost_s == 0.0);
    PreemptionVector two(12, 0);
    two[0] = 1;
    two[5] = 1;
    MigrationPlan intra = plan_migration(Topology{3, 4, 0}, two, {2, 4}, w, costs);
    EXPECT(intra.kind == MigrationKind::intra_stage && intra.moves.size() == 1 &&
           !intra.moves[0].transfers_params);
    PreemptionVector lost(6, 0);
    lost[1] = 1;
    lost[4] = 1;
    bool rolled = false;
    try {
      plan_migration(Topology{2, 3, 0}, lost, {1, 3}, w, costs);
    } catch (const RollbackRequired&) {
      rolled = true;
    }
    EXPECT(rolled);
    PreemptionVector hole(17, 0);
    hole[3] = 1;
    MigrationPlan inter = plan_migration(Topology{2, 8, 1}, hole, {2, 8}, w, costs);
    EXPECT(inter.kind == MigrationKind::inter_stage && inter.transfer_rounds == 1);
    EXPECT(migration_cost(inter, w, costs, 0) == inter.est_cost_s);
    const TransitionOutcome t = transition_outcome_min(0, {4, 8}, {3, 8}, 0, w, costs);
    EXPECT(t.rollback && t.kind == MigrationKind::pipeline);
    EXPECT(resume_cost({3, 8}, w, costs) > t.cost_s);
  }
  // ---- the replay driver (simulator.cpp:119-340)
  {
    IntervalSeries series;
    series.capacity = 32;
    series.counts = {32, 30, 30, 28, 31, 27, 27, 24, 26, 26, 22, 25, 25, 25, 20, 28, 32, 32, 29, 30};
    SimOptions so;
    so.planner.mc_trials = 1000;
    for (Policy pol : {Policy::Reactive(), Policy::Checkpoint(), Policy::Ideal(), Policy::Proactive()}) {
      SimReport r = run(series, lm_1p5b(), pol, 11, so);
      EXPECT(r.intervals.size() == series.counts.size() && r.sample_accounting_ok);
      double total = 0.0;
      for (const IntervalLog& l : r.intervals) total += l.ledger.total();
      EXPECT(std::abs(total - r.ledger.total()) < 1e-6 * (1.0 + total));
      EXPECT(std::abs(r.ledger.total() - r.instance_seconds) < 1e-6 * r.instance_seconds);
    }
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
