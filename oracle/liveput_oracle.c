/*
 * liveput_oracle.c — CPU ORACLE (test infrastructure; the checker, never the
 * product).  See liveput_oracle.h for the reference functions restated here
 * and how they are pinned.  Every function cites the reference file:line it
 * follows; floating-point expressions keep the reference's operand order and
 * are compiled with -ffp-contract=off, like the reference's x86-64 build.
 */
#define _GNU_SOURCE
#include "liveput_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9e3779b97f4a7c15ULL
#define ENUM_CAP 1000000ULL /* kEnumerationCap, preemption.hpp:26 */

static __thread char g_err[256];
static void set_err(const char* m) { snprintf(g_err, sizeof g_err, "%s", m); }
const char* or_last_error(void) { return g_err; }

/* ---- rng.hpp:15-20 ------------------------------------------------------ */
static uint64_t fmix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
uint64_t or_splitmix_next(uint64_t* state) { return fmix(*state += GAMMA); }

/* rng.hpp:46-55 */
uint64_t or_mix_seed(uint64_t a, uint64_t b) { return fmix(a + GAMMA * (b + 1)); }

/* rng.hpp:23-30: rejection without modulo bias */
uint64_t or_below(uint64_t* state, uint64_t bound) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t r;
  do r = or_splitmix_next(state);
  while (r >= limit);
  return r % bound;
}

/* rng.cpp:8-19: partial Fisher-Yates over pool[0..n) */
static void sample_distinct_buf(int n, int k, uint64_t seed, int* pool, int* out) {
  uint64_t st = seed;
  for (int i = 0; i < n; ++i) pool[i] = i;
  for (int i = 0; i < k; ++i) {
    int j = i + (int)or_below(&st, (uint64_t)(n - i));
    int t = pool[i];
    pool[i] = pool[j];
    pool[j] = t;
  }
  for (int i = 0; i < k; ++i) out[i] = pool[i];
}

void or_sample_distinct(int n, int k, uint64_t seed, int* out) {
  int* pool = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
  sample_distinct_buf(n, k, seed, pool, out);
  free(pool);
}

/* preemption.cpp:10-21 */
uint64_t or_scenario_count(int n, int k) {
  if (k < 0 || k > n) return 0;
  if (n - k < k) k = n - k;
  long double c = 1.0L;
  const long double cap = 9.22e18L;
  for (int i = 1; i <= k; ++i) {
    c = c * (n - k + i) / i;
    if (c > cap) return (uint64_t)cap;
  }
  return (uint64_t)(c + 0.5L);
}

/* ---- perf_model.cpp:5-8 ------------------------------------------------- */
int or_depth_feasible(const lp_profile* w, int stages) {
  if (stages < 1) return 0;
  return w->memory_fixed_bytes + w->memory_per_stage_bytes / stages <= w->device_memory_bytes;
}

static int rate_for(const lp_profile* w, int p, double* r) {
  for (int i = 0; i < w->n_rates; ++i)
    if (w->rate_depths[i] == p) {
      *r = w->rate_values[i];
      return 1;
    }
  return 0;
}

/* perf_model.cpp:14-42 and microbatches_per_pipeline, perf_model.hpp:44-48 */
double or_throughput(const lp_profile* w, int d, int p) {
  if (!(d >= 1 && or_depth_feasible(w, p))) return 0.0;
  const long long B = w->minibatch_size;
  const long long per = (long long)d * w->microbatch_size;
  long long mm = (w->minibatch_size + per - 1) / per;
  const long long M = (int)(mm < 1 ? 1 : mm);
  const long long u = w->microbatch_size;
  double sync = 0.0;
  if (d > 1)
    sync = 2.0 * (d - 1) / d * (w->param_bytes / p) * w->beta_s_per_byte +
           2.0 * (d - 1) * w->alpha_s;
  double rate;
  if (rate_for(w, p, &rate)) {
    if (sync == 0.0) return rate * (double)B / (double)(M * u);
    const double t_pipe = (double)(M * u) / rate;
    return (double)B / (t_pipe + sync);
  }
  const double t_stage = w->compute_per_microbatch_s / p;
  const double t_pipe = (double)(M + p - 1) * t_stage +
                        2.0 * (p - 1) * (w->alpha_s + w->activation_bytes * w->beta_s_per_byte);
  return (double)B / (t_pipe + sync);
}

/* perf_model.cpp:44-52: ascending P, descending D */
int or_enumerate_configs(const lp_profile* w, int n, int* out, int cap) {
  int c = 0;
  if (n <= 0) return 0;
  for (int p = 1; p <= n; ++p) {
    if (!or_depth_feasible(w, p)) continue;
    for (int d = n / p; d >= 1; --d) {
      if (c < cap) {
        out[2 * c] = d;
        out[2 * c + 1] = p;
      }
      ++c;
    }
  }
  return c;
}

/* optimizer.cpp:11-25 */
int or_reactive_plan(const lp_profile* w, int n, int* out) {
  int cnt = or_enumerate_configs(w, n, NULL, 0);
  if (cnt <= 0) return 0;
  int* cf = (int*)malloc(sizeof(int) * 2 * cnt);
  or_enumerate_configs(w, n, cf, cnt);
  int have = 0, bd = 0, bp = 0;
  double bt = 0.0;
  for (int i = 0; i < cnt; ++i) {
    const int d = cf[2 * i], p = cf[2 * i + 1];
    const double t = or_throughput(w, d, p);
    if (t <= 0.0) continue;
    if (!have || t > bt || (t == bt && (d > bd || (d == bd && p < bp)))) {
      have = 1;
      bd = d;
      bp = p;
      bt = t;
    }
  }
  free(cf);
  if (have) {
    out[0] = bd;
    out[1] = bp;
  }
  return have;
}

/* ---- migration.cpp ------------------------------------------------------ */
static double fresh_fixed(const lp_costs* c) { /* migration.hpp:24-26 */
  return c->start_process_s + c->rendezvous_s + c->cuda_context_s + c->load_data_s;
}
static double pipeline_transfer(int stages, const lp_profile* w) { /* :32-34 */
  return w->param_bytes * w->beta_s_per_byte + stages * w->alpha_s;
}
static int replication_rounds(int sources, int transfers) { /* :22-30 */
  int rounds = 0;
  long long have = sources;
  while (have < (long long)sources + transfers) {
    have *= 2;
    ++rounds;
  }
  return rounds;
}
static double inter_transfer(int rounds, int stages, const lp_profile* w) { /* :39-42 */
  const double unit = (w->param_bytes / stages) * w->beta_s_per_byte + w->alpha_s;
  const double a = rounds * unit, b = pipeline_transfer(stages, w);
  return (b < a) ? b : a; /* std::min */
}

/* :49-89 */
double or_transition_cost(int m, int sd, int sp, int td, int tp, int fresh, const lp_profile* w,
                          const lp_costs* c, int* rollback, int* kind) {
  *rollback = 0;
  if (m == 0) {
    *rollback = 1;
    *kind = 3;
    return (fresh > 0 ? fresh_fixed(c) : 0.0) + c->build_model_s + c->update_comm_groups_s +
           pipeline_transfer(tp, w);
  }
  if (tp != sp) {
    *kind = 3;
    return (fresh > 0 ? fresh_fixed(c) : 0.0) + c->build_model_s + c->update_comm_groups_s +
           pipeline_transfer(tp, w);
  }
  const int transfers = td - m > 0 ? td - m : 0;
  const int rounds = replication_rounds(m, transfers);
  const int assigned_dead = m < sd;
  if (rounds == 0 && !assigned_dead && td == sd && tp == sp) {
    *kind = 0;
    return 0.0;
  }
  const double base = (fresh > 0 ? fresh_fixed(c) : 0.0) + c->build_model_s + c->update_comm_groups_s;
  if (rounds == 0) {
    *kind = 1;
    return base;
  }
  *kind = 2;
  return base + inter_transfer(rounds, tp, w);
}

/* :100-104 */
double or_resume_cost(int tp, const lp_profile* w, const lp_costs* c) {
  return fresh_fixed(c) + c->build_model_s + c->update_comm_groups_s + pipeline_transfer(tp, w);
}

/* ---- scenarios ---------------------------------------------------------- */
static int cmp_int(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

/* preemption.cpp:23-45 (lexicographic) and :47-59 (trial t uses Rng(mix_seed(seed,t))) */
int or_scenarios(int n, int k, int exact, int trials, uint64_t seed, int* out) {
  if (k < 0 || k > n) {
    set_err("bad n_minus");
    return -1;
  }
  if (exact) {
    uint64_t cnt = or_scenario_count(n, k);
    if (cnt > ENUM_CAP || (uint64_t)trials != cnt) {
      set_err("enumerate: bad count");
      return -1;
    }
    int* idx = (int*)malloc(sizeof(int) * (k > 0 ? k : 1));
    for (int i = 0; i < k; ++i) idx[i] = i;
    for (long long t = 0;; ++t) {
      for (int i = 0; i < k; ++i) out[t * k + i] = idx[i];
      if (k == 0) break;
      int i = k - 1;
      while (i >= 0 && idx[i] == n - k + i) --i;
      if (i < 0) break;
      ++idx[i];
      for (int j = i + 1; j < k; ++j) idx[j] = idx[j - 1] + 1;
    }
    free(idx);
    return 0;
  }
  int* pool = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int t = 0; t < trials; ++t) {
    sample_distinct_buf(n, k, or_mix_seed(seed, (uint64_t)t), pool, out + (size_t)t * k);
    qsort(out + (size_t)t * k, k, sizeof(int), cmp_int);
  }
  free(pool);
  return 0;
}

/* survivor minimum of one sorted scenario for (d, p): stage_survivors
 * (preemption.cpp:61-66) followed by the min of optimizer.cpp:76-82,
 * written as D - max_p #{preempted s < D*P : s % P == p}. */
static int survivor_min(const int* s, int k, int d, int p, int* cnt /* >= p */) {
  const int lim = d * p;
  int mx = 0;
  for (int i = 0; i < k; ++i) {
    if (s[i] >= lim) break;
    int c = ++cnt[s[i] % p];
    if (c > mx) mx = c;
  }
  for (int i = 0; i < k; ++i) {
    if (s[i] >= lim) break;
    cnt[s[i] % p] = 0;
  }
  return d - mx;
}

typedef struct {
  int n, k, exact;
  long long t0, t1;
  uint64_t seed;
  const int* cfg;
  int n_cfg;
  int stride;
  uint64_t* counts;
} ens_job;

static void* ens_worker(void* arg) {
  ens_job* jb = (ens_job*)arg;
  const int n = jb->n, k = jb->k;
  int* pool = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
  int* s = (int*)malloc(sizeof(int) * (k > 0 ? k : 1));
  int* cnt = (int*)calloc((size_t)(n > 0 ? n : 1), sizeof(int));
  int* idx = (int*)malloc(sizeof(int) * (k > 0 ? k : 1));
  for (int i = 0; i < k; ++i) idx[i] = i;
  if (jb->exact && k > 0)
    for (long long t = 0; t < jb->t0; ++t) { /* walk to the first rank of the range */
      int i = k - 1;
      while (i >= 0 && idx[i] == n - k + i) --i;
      if (i < 0) break;
      ++idx[i];
      for (int j = i + 1; j < k; ++j) idx[j] = idx[j - 1] + 1;
    }
  for (long long t = jb->t0; t < jb->t1; ++t) {
    if (jb->exact) {
      for (int i = 0; i < k; ++i) s[i] = idx[i];
    } else {
      sample_distinct_buf(n, k, or_mix_seed(jb->seed, (uint64_t)t), pool, s);
      qsort(s, k, sizeof(int), cmp_int);
    }
    for (int c = 0; c < jb->n_cfg; ++c) {
      const int m = survivor_min(s, k, jb->cfg[2 * c], jb->cfg[2 * c + 1], cnt);
      jb->counts[(size_t)c * jb->stride + m] += 1;
    }
    if (jb->exact && k > 0) {
      int i = k - 1;
      while (i >= 0 && idx[i] == n - k + i) --i;
      if (i < 0) break;
      ++idx[i];
      for (int j = i + 1; j < k; ++j) idx[j] = idx[j - 1] + 1;
    }
  }
  free(pool);
  free(s);
  free(cnt);
  free(idx);
  return NULL;
}

static int ensemble_range(int n, int k, int exact, int trials, uint64_t seed, const int* cfg,
                          int n_cfg, uint64_t* counts, int stride, uint64_t* total, int threads,
                          long long r0, long long r1);

int or_ensemble_counts(int n, int k, int exact, int trials, uint64_t seed, const int* cfg,
                       int n_cfg, uint64_t* counts, int stride, uint64_t* total, int threads) {
  return ensemble_range(n, k, exact, trials, seed, cfg, n_cfg, counts, stride, total, threads, 0,
                        -1);
}

/* Partial ensemble over scenario ranks [r0, r1) — the multi-rank split. */
int or_ensemble_counts_range(int n, int k, int exact, int trials, uint64_t seed, const int* cfg,
                             int n_cfg, uint64_t* counts, int stride, uint64_t* total, int threads,
                             long long r0, long long r1) {
  return ensemble_range(n, k, exact, trials, seed, cfg, n_cfg, counts, stride, total, threads, r0,
                        r1);
}

static int ensemble_range(int n, int k, int exact, int trials, uint64_t seed, const int* cfg,
                          int n_cfg, uint64_t* counts, int stride, uint64_t* total, int threads,
                          long long r0, long long r1) {
  if (k < 0 || k > n) {
    set_err("bad n_minus");
    return -1;
  }
  for (int c = 0; c < n_cfg; ++c)
    if (cfg[2 * c] * cfg[2 * c + 1] > n || cfg[2 * c] + 1 > stride) {
      set_err("config exceeds n");
      return -1;
    }
  long long T = trials;
  if (exact) {
    uint64_t cnt = or_scenario_count(n, k);
    if (cnt > ENUM_CAP) {
      set_err("enumerate_vectors: scenario space too large, sample instead");
      return -1;
    }
    T = (long long)cnt;
    threads = 1; /* lexicographic walk is sequential; counts are tiny */
  } else if (trials < 1) {
    set_err("sample_vectors: trials must be >= 1");
    return -1;
  }
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  if (r1 < 0 || r1 > T) r1 = T;
  if (r0 < 0) r0 = 0;
  if (r0 > r1) r0 = r1;
  memset(counts, 0, sizeof(uint64_t) * (size_t)n_cfg * stride);
  pthread_t th[64];
  ens_job jobs[64];
  uint64_t* part[64];
  for (int i = 0; i < threads; ++i) {
    part[i] = (uint64_t*)calloc((size_t)n_cfg * stride, sizeof(uint64_t));
    jobs[i] = (ens_job){n, k, exact, r0 + (r1 - r0) * i / threads, r0 + (r1 - r0) * (i + 1) / threads,
                        seed, cfg, n_cfg, stride, part[i]};
    if (threads == 1)
      ens_worker(&jobs[i]);
    else
      pthread_create(&th[i], NULL, ens_worker, &jobs[i]);
  }
  for (int i = 0; i < threads; ++i) {
    if (threads > 1) pthread_join(th[i], NULL);
    for (size_t e = 0; e < (size_t)n_cfg * stride; ++e) counts[e] += part[i][e];
    free(part[i]);
  }
  *total = (uint64_t)(r1 - r0);
  return 0;
}

/* ---- Planner ------------------------------------------------------------ */
/* Optional memo of full-level ensembles (or_planner_set_cache): the
 * reference's hist_cache_ (optimizer.hpp:88) for long replays.  Keyed by
 * (n_now, k); holds the counts of every config of n_now (enumerate_configs
 * order), so a re-plan's levels j >= 1 — whose prev nodes are exactly those
 * configs — reuse them.  Values are identical with the memo on or off. */
typedef struct {
  int n, k, nc, stride;
  int* cfg; /* nc (D, P) pairs */
  uint64_t* counts;
  uint64_t total;
} or_memo;

struct or_planner {
  lp_profile w;
  int32_t* depths;
  double* rates;
  lp_costs c;
  lp_options o;
  int threads;
  int cache_on;
  or_memo* memo;
  int n_memo, cap_memo;
};

or_planner* or_planner_new(const lp_profile* w, const lp_costs* c, const lp_options* o,
                           int threads) {
  or_planner* pl = (or_planner*)calloc(1, sizeof(or_planner));
  pl->w = *w;
  if (w->n_rates > 0) {
    pl->depths = (int32_t*)malloc(sizeof(int32_t) * w->n_rates);
    pl->rates = (double*)malloc(sizeof(double) * w->n_rates);
    memcpy(pl->depths, w->rate_depths, sizeof(int32_t) * w->n_rates);
    memcpy(pl->rates, w->rate_values, sizeof(double) * w->n_rates);
  }
  pl->w.rate_depths = pl->depths;
  pl->w.rate_values = pl->rates;
  pl->c = *c;
  pl->o = *o;
  pl->threads = threads;
  return pl;
}

void or_planner_set_cache(or_planner* pl, int on) { pl->cache_on = on; }

void or_planner_free(or_planner* pl) {
  if (!pl) return;
  for (int i = 0; i < pl->n_memo; ++i) {
    free(pl->memo[i].cfg);
    free(pl->memo[i].counts);
  }
  free(pl->memo);
  free(pl->depths);
  free(pl->rates);
  free(pl);
}

/* optimizer.cpp:64-94: exact when C(n,k) <= exact_cap, else mc_trials samples
 * with seed mix_seed(mix_seed(mc_seed, n), k). */
static int planner_counts(or_planner* pl, const int* cfg, int n_cfg, int n_now, int n_minus,
                          uint64_t* counts, int stride, uint64_t* total) {
  const int exact = or_scenario_count(n_now, n_minus) <= pl->o.exact_cap;
  const uint64_t seed = or_mix_seed(or_mix_seed(pl->o.mc_seed, (uint64_t)n_now), (uint64_t)n_minus);
  return or_ensemble_counts(n_now, n_minus, exact, pl->o.mc_trials, seed, cfg, n_cfg, counts,
                            stride, total, pl->threads);
}

int or_survivor_counts(or_planner* pl, int d, int p, int n_now, int n_minus, uint64_t* counts,
                       uint64_t* total) {
  int cfg[2] = {d, p};
  return planner_counts(pl, cfg, 1, n_now, n_minus, counts, d + 1, total);
}

/* optimizer.cpp:96-138, with the histogram supplied as counts (d+1 entries) */
static void phi_counts(const or_planner* pl, int pd, int pp, int nd, int np, int n_now, int n_next,
                       const uint64_t* counts, uint64_t total, double* out) {
  out[0] = 0.0;
  out[1] = 0.0;
  if (nd <= 0) return;
  if (!(nd >= 1 && or_depth_feasible(&pl->w, np)) || nd * np > n_next) return;
  const double T = pl->o.interval_s;
  const double tput = or_throughput(&pl->w, nd, np);
  const int fresh = n_next - n_now > 0 ? n_next - n_now : 0;
  if (pd <= 0) {
    const double cost = or_resume_cost(np, &pl->w, &pl->c);
    out[1] = cost;
    const double te = T - cost;
    out[0] = tput * ((0.0 < te) ? te : 0.0);
    return;
  }
  double committed = 0.0, cost_sum = 0.0;
  for (int m = 0; m <= pd; ++m) {
    const double p = (double)counts[m] / (double)total;
    if (p == 0.0) continue;
    int rb, kind;
    double cost = or_transition_cost(m, pd, pp, nd, np, fresh, &pl->w, &pl->c, &rb, &kind);
    if (rb) cost += pl->o.rollback_penalty_s;
    const double te = T - cost;
    const double t_eff = (0.0 < te) ? te : 0.0;
    double rate = tput;
    if (pl->o.strict_conditional) {
      const int alive = nd < m ? nd : m;
      rate = alive > 0 ? or_throughput(&pl->w, alive, np) : 0.0;
    }
    committed += p * rate * t_eff;
    cost_sum += p * cost;
  }
  out[0] = committed;
  out[1] = cost_sum;
}

int or_phi(or_planner* pl, int pd, int pp, int nd, int np, int n_now, int n_next, double* out) {
  if (nd <= 0 || !or_depth_feasible(&pl->w, np) || nd * np > n_next || pd <= 0) {
    phi_counts(pl, pd, pp, nd, np, n_now, n_next, NULL, 0, out);
    return 0;
  }
  const int k = n_now - n_next > 0 ? n_now - n_next : 0;
  uint64_t* counts = (uint64_t*)calloc((size_t)pd + 1, sizeof(uint64_t));
  uint64_t total = 0;
  int cfg[2] = {pd, pp};
  if (planner_counts(pl, cfg, 1, n_now, k, counts, pd + 1, &total) != 0) {
    free(counts);
    return -1;
  }
  phi_counts(pl, pd, pp, nd, np, n_now, n_next, counts, total, out);
  free(counts);
  return 0;
}

/* expected_liveput semantics (preemption.cpp:87-112) on the planner ensemble:
 * sum over m of count_m * throughput(m, P), divided by the count. */
int or_liveput(or_planner* pl, int d, int p, int n_now, int n_minus, double* out) {
  uint64_t* counts = (uint64_t*)calloc((size_t)d + 1, sizeof(uint64_t));
  uint64_t total = 0;
  int cfg[2] = {d, p};
  if (planner_counts(pl, cfg, 1, n_now, n_minus, counts, d + 1, &total) != 0) {
    free(counts);
    return -1;
  }
  double acc = 0.0;
  for (int m = 1; m <= d; ++m)
    if (counts[m]) acc += (double)counts[m] * or_throughput(&pl->w, m, p);
  *out = acc / (double)total;
  free(counts);
  return 0;
}

/* Counts of the configs pc[0..nc) at (n_now, k) from the memo of the full
 * config list of n_now (computed on first use); 0 on success, -1 when some
 * config is not a config of n_now (e.g. an infeasible `current`). */
static int memo_counts(or_planner* pl, const int* pc, int nc, int n_now, int k, uint64_t* counts,
                       int stride, uint64_t* total) {
  or_memo* m = NULL;
  for (int i = 0; i < pl->n_memo; ++i)
    if (pl->memo[i].n == n_now && pl->memo[i].k == k) m = &pl->memo[i];
  if (!m) {
    const int cnt = or_enumerate_configs(&pl->w, n_now, NULL, 0);
    if (cnt <= 0) return -1;
    if (pl->n_memo == pl->cap_memo) {
      pl->cap_memo = pl->cap_memo ? 2 * pl->cap_memo : 16;
      pl->memo = (or_memo*)realloc(pl->memo, sizeof(or_memo) * pl->cap_memo);
    }
    m = &pl->memo[pl->n_memo];
    m->n = n_now;
    m->k = k;
    m->nc = cnt;
    m->cfg = (int*)malloc(sizeof(int) * 2 * cnt);
    or_enumerate_configs(&pl->w, n_now, m->cfg, cnt);
    int md = 0;
    for (int i = 0; i < cnt; ++i) md = m->cfg[2 * i] > md ? m->cfg[2 * i] : md;
    m->stride = md + 1;
    m->counts = (uint64_t*)calloc((size_t)cnt * m->stride, sizeof(uint64_t));
    if (planner_counts(pl, m->cfg, cnt, n_now, k, m->counts, m->stride, &m->total) != 0) {
      free(m->cfg);
      free(m->counts);
      return -1;
    }
    ++pl->n_memo;
  }
  for (int c = 0; c < nc; ++c) {
    int row = -1;
    for (int i = 0; i < m->nc; ++i)
      if (m->cfg[2 * i] == pc[2 * c] && m->cfg[2 * i + 1] == pc[2 * c + 1]) {
        row = i;
        break;
      }
    if (row < 0) return -1;
    for (int d = 0; d < stride; ++d) counts[(size_t)c * stride + d] = d <= pc[2 * c] ? m->counts[(size_t)row * m->stride + d] : 0;
  }
  *total = m->total;
  return 0;
}

typedef struct {
  int d, p;
  double value, mig;
  int parent;
  double step_c, step_m;
} node_t;

/* optimizer.cpp:140-205 */
int or_dp_optimize(or_planner* pl, int cd, int cp, const int* n_seq, int len, int* cfg_out,
                   double* val_out, double* final_value) {
  if (len < 2) {
    set_err("dp_optimize: need at least N_i and N_{i+1}");
    return -1;
  }
  if (cd > 0 && cd * cp > n_seq[0]) {
    set_err("dp_optimize: current config exceeds n_seq[0]");
    return -1;
  }
  const int H = len - 1;
  node_t** lv = (node_t**)calloc((size_t)H + 1, sizeof(node_t*));
  int* lsz = (int*)calloc((size_t)H + 1, sizeof(int));
  lv[0] = (node_t*)malloc(sizeof(node_t));
  lv[0][0] = (node_t){cd > 0 ? cd : 0, cd > 0 ? cp : 0, 0.0, 0.0, -1, 0.0, 0.0};
  lsz[0] = 1;
  for (int j = 0; j < H; ++j) {
    const int n_now = n_seq[j], n_next = n_seq[j + 1];
    const int k = n_now - n_next > 0 ? n_now - n_next : 0;
    /* histograms of every non-suspended prev node, one ensemble pass */
    const int np_ = lsz[j];
    int* pc = (int*)malloc(sizeof(int) * 2 * (np_ > 0 ? np_ : 1));
    int* map = (int*)malloc(sizeof(int) * (np_ > 0 ? np_ : 1));
    int nc = 0, maxd = 0;
    for (int i = 0; i < np_; ++i) {
      map[i] = -1;
      if (lv[j][i].d > 0) {
        pc[2 * nc] = lv[j][i].d;
        pc[2 * nc + 1] = lv[j][i].p;
        if (lv[j][i].d > maxd) maxd = lv[j][i].d;
        map[i] = nc++;
      }
    }
    const int stride = maxd + 1;
    uint64_t* counts = (uint64_t*)calloc((size_t)(nc > 0 ? nc : 1) * stride, sizeof(uint64_t));
    uint64_t total = 0;
    if (nc > 0 && pl->cache_on && memo_counts(pl, pc, nc, n_now, k, counts, stride, &total) == 0) {
      /* served from the memo */
    } else if (nc > 0 && planner_counts(pl, pc, nc, n_now, k, counts, stride, &total) != 0) {
      free(pc);
      free(map);
      free(counts);
      for (int q = 0; q <= j; ++q) free(lv[q]);
      free(lv);
      free(lsz);
      return -1;
    }
    const int ncand = or_enumerate_configs(&pl->w, n_next, NULL, 0);
    int* cand = (int*)malloc(sizeof(int) * 2 * (ncand + 1));
    or_enumerate_configs(&pl->w, n_next, cand, ncand);
    cand[2 * ncand] = 0;
    cand[2 * ncand + 1] = 0;
    lv[j + 1] = (node_t*)malloc(sizeof(node_t) * (ncand + 1));
    int out_n = 0;
    for (int ci = 0; ci <= ncand; ++ci) {
      node_t best = {cand[2 * ci], cand[2 * ci + 1], -INFINITY, 0.0, -1, 0.0, 0.0};
      for (int pi = 0; pi < np_; ++pi) {
        const node_t* p = &lv[j][pi];
        if (!isfinite(p->value)) continue;
        double st[2];
        const uint64_t* h = map[pi] >= 0 ? counts + (size_t)map[pi] * stride : NULL;
        phi_counts(pl, p->d, p->p, best.d, best.p, n_now, n_next, h, total, st);
        const double value = p->value + st[0];
        const double mig = p->mig + st[1];
        if (best.parent < 0 || value > best.value || (value == best.value && mig < best.mig)) {
          best.value = value;
          best.mig = mig;
          best.parent = pi;
          best.step_c = st[0];
          best.step_m = st[1];
        }
      }
      if (best.parent >= 0) lv[j + 1][out_n++] = best;
    }
    lsz[j + 1] = out_n;
    free(pc);
    free(map);
    free(counts);
    free(cand);
  }
  /* optimizer.cpp:185-195: rank (value, -mig, D, -P); suspended -> (-1, 0) */
  const node_t* last = lv[H];
  int bi = 0;
  for (int i = 1; i < lsz[H]; ++i) {
    const node_t* a = &last[i];
    const node_t* b = &last[bi];
    const double am = -a->mig, bm = -b->mig;
    const int ad = a->d > 0 ? a->d : -1, bd = b->d > 0 ? b->d : -1;
    const int ap = a->d > 0 ? -a->p : 0, bp = b->d > 0 ? -b->p : 0;
    int gt;
    if (b->value < a->value) gt = 1;
    else if (a->value < b->value) gt = 0;
    else if (bm < am) gt = 1;
    else if (am < bm) gt = 0;
    else if (bd < ad) gt = 1;
    else if (ad < bd) gt = 0;
    else gt = bp < ap;
    if (gt) bi = i;
  }
  if (final_value) *final_value = last[bi].value;
  int idx = bi;
  for (int j = H; j >= 1; --j) {
    const node_t* nd = &lv[j][idx];
    cfg_out[2 * (j - 1)] = nd->d;
    cfg_out[2 * (j - 1) + 1] = nd->d > 0 ? nd->p : 0;
    val_out[2 * (j - 1)] = nd->step_c;
    val_out[2 * (j - 1) + 1] = nd->step_m;
    idx = nd->parent;
  }
  for (int j = 0; j <= H; ++j) free(lv[j]);
  free(lv);
  free(lsz);
  return 0;
}

/* optimizer.cpp:207-219 */
int or_sequence_value(or_planner* pl, int cd, int cp, const int* seq, const int* n_seq, int len,
                      double* out) {
  double value = 0.0;
  int pd = cd, pp = cp;
  for (int j = 0; j + 1 < len; ++j) {
    double st[2];
    if (or_phi(pl, pd, pp, seq[2 * j], seq[2 * j + 1], n_seq[j], n_seq[j + 1], st) != 0) return -1;
    value += st[0];
    pd = seq[2 * j];
    pp = seq[2 * j + 1];
  }
  *out = value;
  return 0;
}
