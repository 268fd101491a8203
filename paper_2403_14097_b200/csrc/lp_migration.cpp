// lp_migration.cpp — concrete migration plans for a realised preemption
// scenario, host C++.
//
// Restates plan_migration / migration_cost / transition_outcome_min /
// resume_cost (reference migration.cpp:49-236).  The planner's hot path only
// needs the costs (lp_dp.cu transition_cost); this is what a caller executes
// once the DP has picked the next configuration and the scenario is known.
// Compiled with -ffp-contract=off like lp_model.cpp, so every cost is the
// reference's double.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "liveput.h"
#include "lp_model.hpp"

namespace lp {
std::string& global_error();  // lp_api.cpp
}

namespace {

using lp::Model;

lp_status mig_fail(lp_status s, const char* fmt, ...) {
  char buf[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  lp::global_error() = buf;
  return s;
}

// migration.cpp:22-30: source-doubling rounds until `sources` copies cover
// sources + transfers holders.
int doubling_rounds(int sources, int transfers) {
  int r = 0;
  for (long long have = sources; have < static_cast<long long>(sources) + transfers; have *= 2) ++r;
  return r;
}

// inter_transfer_s (migration.cpp:39-42): never worse than a repartition.
double inter_transfer(const Model& m, int rounds, int stages) {
  const double serial = rounds * m.inter_unit(stages);
  const double repartition = m.pipe_transfer(stages);
  return std::min(serial, repartition);
}

double fresh_fixed(const lp_costs& c) {
  return c.start_process_s + c.rendezvous_s + c.cuda_context_s + c.load_data_s;
}

double plan_cost(const Model& m, const lp_costs& c, int kind, int rounds, int target_stages,
                 int fresh) {
  if (kind == LP_MIG_NONE) return 0.0;
  double cost = c.build_model_s + c.update_comm_groups_s;
  if (fresh > 0) cost += fresh_fixed(c);
  if (kind == LP_MIG_INTER_STAGE) cost += inter_transfer(m, std::max(1, rounds), target_stages);
  if (kind == LP_MIG_PIPELINE) cost += m.pipe_transfer(target_stages);
  return cost;
}

}  // namespace

extern "C" {

lp_status lp_plan_migration(const lp_profile* profile, const lp_costs* costs, lp_config source,
                            int32_t spares, const uint8_t* v, int32_t v_len, lp_config target,
                            lp_migration* out, lp_move* moves, int32_t cap) {
  if (!profile || !costs || !out || (!v && v_len > 0) || (!moves && cap > 0))
    return mig_fail(LP_EINVAL, "plan_migration: null argument");
  const int D = source.pipelines, P = source.stages;
  if (D < 0 || P < 1 || spares < 0 || target.pipelines < 0 || target.stages < 1)
    return mig_fail(LP_EINVAL, "plan_migration: bad topology or target");
  const int assigned = D * P;
  if (v_len != assigned + spares)
    return mig_fail(LP_EINVAL, "plan_migration: vector/topology size mismatch");
  const Model model(*profile);
  auto dead = [&](int k) { return v[k] != 0; };

  // stage_survivors (preemption.cpp:61-66)
  std::vector<int> alive_in_stage(P, 0);
  for (int d = 0; d < D; ++d)
    for (int p = 0; p < P; ++p) alive_in_stage[p] += dead(d * P + p) ? 0 : 1;
  if (target.pipelines >= 1)
    for (int p = 0; p < P; ++p)
      if (alive_in_stage[p] == 0)
        return mig_fail(LP_EROLLBACK, "stage fully preempted, no parameter source survives");

  std::vector<lp_move> mv;
  lp_migration plan{};
  plan.source = source;
  plan.target = target;
  int rounds = 0;
  bool transfers_any = false;

  if (target.stages != P) {
    plan.kind = LP_MIG_PIPELINE;  // a depth change repartitions everything
  } else {
    // Pipelines ranked by surviving slots (stable: ties keep index order);
    // the first min(target.D, D) stay as the bases of the new layout.
    std::vector<int> alive_in_pipe(D, 0);
    for (int d = 0; d < D; ++d)
      for (int p = 0; p < P; ++p) alive_in_pipe[d] += dead(d * P + p) ? 0 : 1;
    std::vector<int> rank(D);
    for (int d = 0; d < D; ++d) rank[d] = d;
    std::stable_sort(rank.begin(), rank.end(),
                     [&](int a, int b) { return alive_in_pipe[a] > alive_in_pipe[b]; });
    const int bases = std::min(target.pipelines, D);
    std::vector<char> is_base(D, 0);
    for (int i = 0; i < bases; ++i) is_base[rank[i]] = 1;

    std::vector<int> spare_pool;  // live spares, taken from the back
    for (int k = assigned; k < assigned + spares; ++k)
      if (!dead(k)) spare_pool.push_back(k);
    std::vector<std::vector<int>> stage_donors(P);  // live slots of non-base pipelines
    for (int d = 0; d < D; ++d)
      if (!is_base[d])
        for (int p = 0; p < P; ++p)
          if (!dead(d * P + p)) stage_donors[p].push_back(d * P + p);

    std::vector<int> leftover;                 // donors not needed in their stage
    std::vector<std::pair<int, int>> needs;    // (row, stage) filled by a transfer
    for (int p = 0; p < P; ++p) {
      int have = 0;
      for (int i = 0; i < bases; ++i) have += dead(rank[i] * P + p) ? 0 : 1;
      int holes = target.pipelines - have;
      // Hole rows of stage p: bases whose slot p is dead (in rank order),
      // then the rows appended past the old pipelines.
      int cur = 0;
      auto hole_row = [&]() {
        while (cur < bases && !dead(rank[cur] * P + p)) ++cur;
        const int row = cur < bases ? rank[cur] : D + (cur - bases);
        ++cur;
        return row;
      };
      size_t used = 0;
      for (; holes > 0 && used < stage_donors[p].size(); ++used, --holes) {
        const int inst = stage_donors[p][used];  // same stage: reroute only
        mv.push_back({inst, inst / P, p, hole_row(), p, 0});
      }
      leftover.insert(leftover.end(), stage_donors[p].begin() + used, stage_donors[p].end());
      const int fills = std::max(0, holes);
      for (int f = 0; f < fills; ++f) needs.push_back({hole_row(), p});
      if (fills > 0) rounds = std::max(rounds, doubling_rounds(alive_in_stage[p], fills));
    }
    for (const auto& [row, p] : needs) {
      if (!spare_pool.empty()) {
        const int body = spare_pool.back();
        spare_pool.pop_back();
        mv.push_back({body, -1, -1, row, p, 1});
      } else if (!leftover.empty()) {
        const int body = leftover.back();
        leftover.pop_back();
        mv.push_back({body, body / P, body % P, row, p, 1});
      } else {
        return mig_fail(LP_EINVAL, "plan_migration: not enough instances for target");
      }
    }
    transfers_any = !needs.empty();
    if (transfers_any) plan.kind = LP_MIG_INTER_STAGE;
    else if (!mv.empty() || target.pipelines != D) plan.kind = LP_MIG_INTRA_STAGE;
    else plan.kind = LP_MIG_NONE;
  }
  plan.transfer_rounds = rounds;
  plan.n_moves = static_cast<int32_t>(mv.size());
  plan.est_cost_s = plan_cost(model, *costs, plan.kind, rounds, target.stages, 0);
  const int n = std::min<int>(plan.n_moves, std::max(cap, 0));
  for (int i = 0; i < n; ++i) moves[i] = mv[i];
  *out = plan;
  return LP_OK;
}

double lp_migration_cost(const lp_profile* profile, const lp_costs* costs, const lp_migration* plan,
                         int32_t fresh_instances) {
  if (!profile || !costs || !plan) return 0.0;
  const Model model(*profile);
  return plan_cost(model, *costs, plan->kind, plan->transfer_rounds, plan->target.stages,
                   fresh_instances);
}

lp_status lp_transition_outcome(const lp_profile* profile, const lp_costs* costs,
                                int32_t min_survivor, lp_config source, lp_config target,
                                int32_t fresh_instances, double* cost_s, int32_t* kind,
                                int32_t* rollback) {
  if (!profile || !costs || !cost_s || !kind || !rollback)
    return mig_fail(LP_EINVAL, "transition_outcome: null argument");
  const Model model(*profile);
  const lp_costs& c = *costs;
  const double fixed = fresh_instances > 0 ? fresh_fixed(c) : 0.0;
  *rollback = 0;
  if (min_survivor == 0 || target.stages != source.stages) {
    *rollback = min_survivor == 0 ? 1 : 0;
    *kind = LP_MIG_PIPELINE;
    *cost_s = fixed + c.build_model_s + c.update_comm_groups_s + model.pipe_transfer(target.stages);
    return LP_OK;
  }
  const int rounds = doubling_rounds(min_survivor, std::max(0, target.pipelines - min_survivor));
  const bool lost_assigned = min_survivor < source.pipelines;
  const bool same = target.pipelines == source.pipelines && target.stages == source.stages;
  if (rounds == 0 && !lost_assigned && same) {
    *kind = LP_MIG_NONE;
    *cost_s = 0.0;
    return LP_OK;
  }
  const double base = fixed + c.build_model_s + c.update_comm_groups_s;
  if (rounds == 0) {
    *kind = LP_MIG_INTRA_STAGE;
    *cost_s = base;
  } else {
    *kind = LP_MIG_INTER_STAGE;
    *cost_s = base + inter_transfer(model, rounds, target.stages);
  }
  return LP_OK;
}

double lp_resume_cost(const lp_profile* profile, const lp_costs* costs, lp_config target) {
  if (!profile || !costs) return 0.0;
  const Model model(*profile);
  return fresh_fixed(*costs) + costs->build_model_s + costs->update_comm_groups_s +
         model.pipe_transfer(target.stages);
}

}  // extern "C"
