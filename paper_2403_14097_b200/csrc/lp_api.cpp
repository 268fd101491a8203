// lp_api.cpp — the C ABI of include/liveput.h: host planner over the sm_100a
// kernels.  The host side only builds tables (configs, throughput, costs,
// ensemble descriptors) and launches; every histogram, phi, DP step and the
// traceback run on the device.  There is no CPU fallback.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "liveput.h"
#include "lp_launch.h"
#include "lp_layout.h"
#include "lp_model.hpp"

namespace lp {
namespace {

thread_local std::string g_global_err;
}  // namespace

// lp_migration.cpp reports through the same per-thread message
std::string& global_error() { return g_global_err; }

namespace {

constexpr uint64_t kEnumerationCap = 1000000ULL;  // preemption.hpp:26
constexpr size_t kSmemBudgetR = 72 * 1024;
constexpr size_t kSmemBudgetC = 110 * 1024;
constexpr uint64_t kChunkR = 256 * 8;
constexpr size_t kScnFixedBudget = 64 * 1024;   // entries + event table per block
constexpr size_t kSmemBudgetScn = 112 * 1024;   // two blocks per SM
constexpr size_t kSmemBudgetInc = 75 * 1024;    // three blocks per SM
constexpr int kIncMaxK = 8;                     // incidence kernel up to k = 8, rows above
constexpr size_t kSmemBudgetBits8 = 48 * 1024;  // bits kernel, k <= 8: four 256-thread blocks per SM
constexpr size_t kSmemBudgetBits16 = 64 * 1024; // bits kernel, k <= 16: three blocks per SM

// Largest k resolved by the bits kernel (rows kernel above); LIVEPUT_BITS_MAXK
// = 8 restores the row kernel for 9 <= k <= 16 (A/B).
int bits_max_k() {
  static const int v = [] {
    const char* e = getenv("LIVEPUT_BITS_MAXK");
    return e ? std::max(8, std::min(16, atoi(e))) : 16;
  }();
  return v;
}

size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

// LIVEPUT_TIMELINE=1: lp_get_stats prints, relative to the start of the
// execute, when each stage's histogram kernels and normalisation finished
// and when each DP level finished (per-level launches only).
bool timeline() {
  static const bool on = getenv("LIVEPUT_TIMELINE") != nullptr;
  return on;
}

// Row-kernel block shape: threads per block cap, shared-memory budget per
// block and the entries + event-table share of it. LIVEPUT_ROWS_SHAPE =
// "T,smem_kb,fixed_kb" overrides the defaults (256, 112, 64) for A/B runs.
struct RowsShape {
  int tmax = 256;
  size_t smem = kSmemBudgetScn;
  size_t fixed = kScnFixedBudget;
  int kreg_max = kMaxKReg;  // LIVEPUT_ROWS_KREG=0: byte-table draws for every k
};
const RowsShape& rows_shape() {
  static const RowsShape s = [] {
    RowsShape r;
    if (const char* e = getenv("LIVEPUT_ROWS_SHAPE")) {
      int t = 0, sk = 0, fk = 0;
      if (sscanf(e, "%d,%d,%d", &t, &sk, &fk) == 3 && t >= 32 && t <= 256 && sk > 0 && fk > 0 && fk <= sk) {
        r.tmax = t & ~31;
        r.smem = (size_t)sk * 1024;
        r.fixed = (size_t)fk * 1024;
      }
    }
    if (const char* e = getenv("LIVEPUT_ROWS_KREG")) r.kreg_max = atoi(e) == 0 ? 0 : kMaxKReg;
    return r;
  }();
  return s;
}

// ---------------------------------------------------------------------------
// growable device / pinned host buffers
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 1 << 16);
    want = want + want / 4;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct PinBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 1 << 16);
    want = want + want / 4;
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  ~PinBuf() {
    if (p) cudaFreeHost(p);
  }
};

// Sections appended to one host image and uploaded with a single copy.
struct Packer {
  std::vector<unsigned char> bytes;
  Packer() { bytes.reserve(1 << 21); }
  size_t add(const void* src, size_t n) {
    size_t off = (bytes.size() + 255) & ~size_t(255);
    bytes.resize(off + std::max<size_t>(n, 1));
    if (n && src) std::memcpy(bytes.data() + off, src, n);
    else if (n) std::memset(bytes.data() + off, 0, n);
    return off;
  }
  template <typename T>
  size_t add(const std::vector<T>& v) {
    return add(v.data(), v.size() * sizeof(T));
  }
};

// Small-integer-keyed map (keys are depths P <= n): a dense vector with
// presence flags, iterated in ascending key order like std::map, without a
// node allocation per depth on the re-plan path.
template <class V>
class DenseMap {
 public:
  struct iterator {
    const DenseMap* m;
    int k;
    std::pair<int, const V&> operator*() const { return {k, m->val_[k]}; }
    iterator& operator++() {
      ++k;
      skip();
      return *this;
    }
    void skip() {
      while (k < (int)m->has_.size() && !m->has_[k]) ++k;
    }
    bool operator!=(const iterator& o) const { return k != o.k; }
  };
  V& operator[](int k) {
    if (k >= (int)val_.size()) {
      val_.resize(k + 1);
      has_.resize(k + 1, 0);
    }
    if (!has_[k]) {
      has_[k] = 1;
      ++cnt_;
      val_[k] = V{};
    }
    return val_[k];
  }
  const V* find(int k) const { return (k >= 0 && k < (int)has_.size() && has_[k]) ? &val_[k] : nullptr; }
  void erase(int k) {
    if (find(k)) {
      has_[k] = 0;
      --cnt_;
    }
  }
  size_t size() const { return (size_t)cnt_; }
  iterator begin() const {
    iterator it{this, 0};
    it.skip();
    return it;
  }
  iterator end() const { return iterator{this, (int)has_.size()}; }

 private:
  std::vector<V> val_;
  std::vector<uint8_t> has_;
  int cnt_ = 0;
};

// ---------------------------------------------------------------------------
// histogram plan: ensembles -> pairs / entries / work items / launch groups
struct EnsembleSpec {
  int n = 0, k = 0;
  bool exact = false;
  uint64_t count = 0;  // ensemble size (all ranks)
  uint64_t seed = 0;
  DenseMap<int> dmax_by_p;       // depth -> largest D needed
  uint64_t ref_keys = 0;         // distinct (D,P) keys the reference would tally
  int stage = 0;                 // pipeline stage (pairs ordered by first DP level)
};

struct Group {
  int stage = 0;
  int kind = 0;  // 0: register variant, 1: counter variant
  int kmax = 0;
  int threads = 256;
  bool smem_evt = true;
  size_t smem = 0;
  int pmax_cap = 0;
  int first = 0, count = 0;
};

struct HistPlan {
  std::vector<PairDesc> pairs;
  std::vector<EntryDesc> entries;
  std::vector<DrawConst> draws;
  std::vector<uint64_t> binom;
  std::vector<WorkSpan> spans;  // per-block WorkItems are expanded on the device
  int64_t n_work = 0;           // blocks over all groups
  std::vector<WorkItem> items;  // small plans (<= kHostItems blocks): expanded here, no expand launch
  std::vector<uint16_t> divtab;
  std::vector<uint32_t> dmask;  // bits kernel: per (range, pass, d) depth-divisor masks
  size_t big_words = 0;         // n > kBigN: scratch words per thread of the big kernel
  std::vector<Group> groups;
  // Pipeline stages: pairs (and so entries, hist rows) are contiguous per
  // stage, in the order the DP first reads them.
  struct Stage {
    int p0 = 0, p1 = 0;      // pairs
    int e0 = 0, e1 = 0;      // entries
    int64_t h0 = 0, h1 = 0;  // hist cells
  };
  std::vector<Stage> stages;
  int64_t evt_len = 0, h0_len = 0, hist_len = 0;
  uint64_t scenarios = 0, local_scenarios = 0, resolutions = 0, alg_ops = 0;
  uint64_t model_ops = 0;  // int ops of the algorithms actually run (op_model_*)
  int mc_pairs = 0, exact_pairs = 0;
};

constexpr int64_t kHostItems = 256;

int kmax_for(int k) { return k <= 4 ? 4 : (k <= 8 ? 8 : 16); }

size_t smem_regs(int ne, int kmax, int n, int64_t evt_len, bool smem_evt) {
  return a16(sizeof(EntryDesc) * ne) + a16(sizeof(DrawConst) * kmax) + a16(4 * (size_t)n) +
         (smem_evt ? a16(4 * (size_t)evt_len) : 0);
}

size_t smem_ctr(int ne, int k, int n, int64_t evt_len, bool smem_evt, int T, int pmax) {
  const size_t nw = (n + 31) / 32;
  const size_t gen = 4 * (size_t)(k + nw) * T;
  const size_t ctr = 4 * (size_t)((pmax + 3) / 4) * T;
  return a16(sizeof(EntryDesc) * ne) + a16(sizeof(DrawConst) * k) + a16(4 * (size_t)n) +
         (smem_evt ? a16(4 * (size_t)evt_len) : 0) + a16(2 * (size_t)k * T) + a16(std::max(gen, ctr));
}

size_t smem_inc(int ne_res, int kmax, int n, int64_t evt_len, bool smem_evt, int dtab_len, int T) {
  return a16(sizeof(EntryDesc) * std::max(ne_res, 1)) + a16(sizeof(DrawConst) * kmax) +
         a16(4 * (size_t)n) + (smem_evt ? a16(4 * (size_t)evt_len) : 0) +
         a16(2 * (size_t)std::max(dtab_len, 1)) + a16(4 * (size_t)((ne_res + 1) / 2) * T);
}

// CSR table: for every difference d in [1, n) the local indices of the
// resolution depths P >= 2 that divide d (incidence kernel).
void build_divtab(const std::vector<EntryDesc>& ents, int e_lo, int e_res, int n,
                  std::vector<uint16_t>& out) {
  std::vector<int> cnt(n + 1, 0);
  for (int e = e_lo; e < e_res; ++e)
    if (ents[e].P >= 2)
      for (int d = ents[e].P; d < n; d += ents[e].P) cnt[d]++;
  const size_t base = out.size();
  out.resize(base + n + 1);
  int acc = 0;
  for (int d = 0; d <= n; ++d) {
    out[base + d] = (uint16_t)acc;
    if (d < n) acc += cnt[d];
  }
  out.resize(base + n + 1 + acc);
  std::vector<int> fill(n + 1, 0);
  for (int e = e_lo; e < e_res; ++e)
    if (ents[e].P >= 2)
      for (int d = ents[e].P; d < n; d += ents[e].P)
        out[base + n + 1 + out[base + d] + fill[d]++] = (uint16_t)(e - e_lo);
}

// Must match the carve in hist_bits_kernel (lp_hist_bits.cu).
size_t smem_bits(int nbits, int kmax, int n, int64_t evt_len, bool smem_evt, int ngroups) {
  return a16(8 * (size_t)std::max(nbits, 1)) + a16(sizeof(DrawConst) * kmax) + a16(4 * (size_t)n) +
         (smem_evt ? a16(4 * (size_t)(evt_len + 1)) : 0) + a16(4 * (size_t)ngroups * n) + a16(4 * (size_t)kmax * 256);
}

// Divisor masks of the bits kernel: word (pass, d, g) has bit b set when
// the resolution depth pass*32*ng + g*32 + b divides d (d >= 1).  Appended to
// `out` at a 4-word boundary; returns the offset.
int build_dmask(const std::vector<EntryDesc>& ents, int eb0, int nres, int n, int ng, int npass,
                std::vector<uint32_t>& out) {
  while (out.size() % 4) out.push_back(0u);
  const int off = (int)out.size();
  out.resize(out.size() + (size_t)npass * n * ng, 0u);
  for (int i = 0; i < nres; ++i) {
    const int P = ents[eb0 + i].P;
    const int ps = i / (32 * ng), g = (i / 32) % ng, b = i % 32;
    uint32_t* tab = out.data() + off + (size_t)ps * n * ng;
    for (int d = P; d < n; d += P) tab[(size_t)d * ng + g] |= 1u << b;
  }
  return off;
}

// Must match the carve in hist_rows_kernel (lp_hist_rows.cu).
size_t smem_rows(int ne_res, int k, int n, int64_t evt_len, bool smem_evt, int T, int kreg, bool exact) {
  const size_t nw = (n + 31) / 32;
  const size_t kk = std::max(k, 1);
  size_t gen = 0;  // KREG = 0: displacement list, or position table + displaced bitmap (n <= 256)
  if (kreg == 0) {
    gen = 4 * kk * T;
    if (!exact && n <= 256) gen = std::max(gen, 4 * nw * T + (size_t)((n + 3) & ~3) * T);
  }
  return a16(sizeof(EntryDesc) * std::max(ne_res, 1)) + a16(8 * (size_t)(ne_res + 1)) +
         a16(sizeof(DrawConst) * kk) + a16(4 * (size_t)n) +
         (smem_evt ? a16(4 * (size_t)((evt_len + 1) / 2)) : 0) + a16(4 * (nw + 3) * T) + a16(gen);
}

size_t smem_scn(int ne_res, int k, int n, int64_t evt_len, bool smem_evt, int T, int uw) {
  const size_t nw = (n + 31) / 32;
  const size_t kk = std::max(k, 1);
  return a16(sizeof(EntryDesc) * std::max(ne_res, 1)) + a16(sizeof(DrawConst) * kk) +
         a16(4 * (size_t)n) + (smem_evt ? a16(4 * (size_t)evt_len) : 0) + a16(2 * kk * T) +
         a16(4 * nw * T) + a16(4 * (size_t)std::max(uw, 1) * T);
}

// Algorithmic int32-equivalent ops (restated for the
// threshold-event resolution): S(k) = 20 + 35k per scenario,
// R(k) = 6k per (scenario, depth); no per-(scenario, config) term.
uint64_t alg_ops(uint64_t scen, int k, int depths) {
  return scen * (20ull + 35ull * k + 6ull * k * (uint64_t)depths);
}

// Int32-equivalent ops per scenario of the resolution algorithms as run
// (the "model" roofline).  Event emission is not counted.
int planes_of(int v) {  // bits needed for 0..v
  int b = 1;
  while ((1 << b) <= v) ++b;
  return b;
}
// bits kernel, per 32-depth group: k(k-1)/2 slot pairs x (table lookup 2 +
// bit-sliced add 2B-1) and k-1 rows x (compare 3B + max B + J/event masks B+3)
uint64_t op_model_bits(int k, int km, int groups) {
  const uint64_t B = planes_of(km - 1), kp = (uint64_t)k * (k - 1) / 2;
  return (uint64_t)groups * (kp * (2 * B + 1) + (uint64_t)std::max(k - 1, 0) * (5 * B + 3));
}
// row kernel, per depth: Dmax rows x ceil(P/32) words x (3B + 4), B = bits(tmax)
uint64_t op_model_rows(const EntryDesc& e) {
  if (e.tmax < 2) return 0;
  return (uint64_t)e.Dmax * ((e.P + 31) / 32) * (3ull * planes_of(e.tmax) + 4ull);
}

// Rng::below(b) constants (rng.hpp:23-30) for b = 1 .. kMaxN, computed once
// (two 64-bit divisions each).
const DrawConst& draw_const(uint32_t b) {
  static const std::vector<DrawConst> table = [] {
    std::vector<DrawConst> t(kMaxN + 1);
    for (uint32_t v = 1; v <= (uint32_t)kMaxN; ++v) {
      DrawConst d{};
      d.b = v;
      d.lim = UINT64_MAX - UINT64_MAX % v;
      d.m32 = v == 1 ? 0xffffffffu : (uint32_t)((1ull << 32) / v);
      d.c32 = (uint32_t)((1ull << 32) % v);
      d.negb = 0u - v;
      t[v] = d;
    }
    return t;
  }();
  return table[b];
}

lp_status build_hist_plan(const std::vector<EnsembleSpec>& specs, int rank, int nranks,
                          HistPlan& hp, std::string& err, int num_sms = 148) {
  static const bool trace = getenv("LIVEPUT_TRACE_PREPARE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (trace)
      fprintf(stderr, "[histplan] %-10s %8.3f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  };
  hp = HistPlan();
  for (const EnsembleSpec& sp : specs) {
    const int n = sp.n, k = sp.k;
    if (n > kMaxN) {
      err = "liveput: n exceeds the supported maximum of " + std::to_string(kMaxN);
      return LP_EUNSUPPORTED;
    }
    PairDesc pd{};
    pd.n = n;
    pd.k = k;
    pd.exact = sp.exact ? 1 : 0;
    pd.entry_base = (int)hp.entries.size();
    pd.n_entries = (int)sp.dmax_by_p.size();
    pd.h0_off = (int)hp.h0_len;
    hp.h0_len += std::max(n, 1);
    pd.seed = sp.seed;
    pd.count = sp.count;
    pd.t_lo = sp.count * (uint64_t)rank / (uint64_t)nranks;
    pd.t_hi = sp.count * (uint64_t)(rank + 1) / (uint64_t)nranks;
    pd.variant = k <= kMaxKReg ? 0 : 1;
    const int pair_idx = (int)hp.pairs.size();
    int max_dm = 0;
    for (const auto& [P, Dm] : sp.dmax_by_p) {
      EntryDesc e{};
      e.P = P;
      e.Dmax = Dm;
      e.lim = P * Dm;
      static const std::vector<uint32_t> magic = [] {  // floor(2^32 / P) + 1, P <= kMaxN
        std::vector<uint32_t> m(kMaxN + 1, 0u);
        for (int q = 2; q <= kMaxN; ++q) m[q] = (uint32_t)((1ull << 32) / (uint64_t)q + 1ull);
        return m;
      }();
      e.magic = P >= 2 ? magic[P] : 0u;
      e.tmax = std::min(k, Dm);
      e.evt_off = (int)hp.evt_len;
      hp.evt_len += (int64_t)std::max(0, e.tmax - 1) * Dm;
      e.hist_off = (int)hp.hist_len;
      hp.hist_len += hist_row(Dm + 1, k);
      e.pair = pair_idx;
      max_dm = std::max(max_dm, Dm);
      hp.entries.push_back(e);
    }
    // only the first-generation counter kernel (LIVEPUT_HIST_KERNEL=legacy)
    // keeps u8 class counts; the row (B <= 10 planes) and scenario-major
    // (12-bit counts) kernels resolve any k
    static const bool legacy_env = [] {
      const char* e = getenv("LIVEPUT_HIST_KERNEL");
      return e && std::string(e) == "legacy";
    }();
    if (legacy_env && pd.variant == 1 && k > kMaxK && max_dm > kMaxK) {
      err = "liveput: n_minus > 255 with more than 255 pipelines per depth needs the default kernels "
            "(LIVEPUT_HIST_KERNEL=legacy keeps u8 counters)";
      return LP_EUNSUPPORTED;
    }
    if (sp.exact) {
      const int stride = std::min(k, n - k) + 1;
      pd.binom_off = (int)hp.binom.size();
      pd.binom_stride = stride;
      const uint64_t sat = 1ull << 62;
      std::vector<uint64_t> tab((size_t)(n + 1) * stride, 0);
      for (int a = 0; a <= n; ++a)
        for (int s = 0; s < stride && s <= a; ++s) {
          uint64_t v;
          if (s == 0 || s == a) v = 1;
          else {
            // C(a, s) = C(a-1, s-1) + C(a-1, s); indices stay within the
            // small side since s <= stride - 1
            const uint64_t x = tab[(size_t)(a - 1) * stride + (s - 1)];
            const uint64_t y = (s <= a - 1) ? tab[(size_t)(a - 1) * stride + s] : 0;
            v = std::min(sat, x + y);
          }
          tab[(size_t)a * stride + s] = v;
        }
      hp.binom.insert(hp.binom.end(), tab.begin(), tab.end());
      hp.exact_pairs++;
    } else {
      pd.draw_off = (int)hp.draws.size();
      for (int i = 0; i < k; ++i) hp.draws.push_back(draw_const((uint32_t)(n - i)));
      hp.mc_pairs++;
    }
    hp.pairs.push_back(pd);
    const uint64_t local = pd.t_hi - pd.t_lo;
    hp.scenarios += sp.count;
    hp.local_scenarios += local;
    hp.resolutions += sp.count * sp.ref_keys;
    hp.alg_ops += alg_ops(local, k, pd.n_entries);
    hp.model_ops += local * (20ull + 35ull * k);  // scenario generation, once per scenario
  }

  mark("pairs");
  // scenarios per block: enough blocks for ~24 per SM over all ensembles
  // (short blocks keep the last wave short; trial-sharded ranks keep every SM
  // busy), at most 4 per 256-thread block (measured with the prioritised stage
  // streams, bench re-plan: 1024 6.32-6.35 ms, 1536 6.38, 2048 6.49)
  uint64_t local_total = 0;
  for (const PairDesc& pd : hp.pairs) local_total += pd.t_hi - pd.t_lo;
  const uint64_t want_blocks = (uint64_t)std::max(num_sms, 1) * 24;
  uint64_t per_block = std::min<uint64_t>(1024, std::max<uint64_t>(256, ((local_total / want_blocks) + 255) & ~255ull));
  if (const char* pb = getenv("LIVEPUT_PER_BLOCK")) per_block = std::max<uint64_t>(256, strtoull(pb, nullptr, 10));

  // work items, grouped by launch configuration
  // one record per (pair, entry range): its work items are the chunks of
  // the pair's trial range, one WorkSpan per range (blocks expanded on the device)
  struct Range {
    WorkItem w;  // t0 / t1 set per chunk
    uint64_t t_lo, t_hi, chunk;
    size_t smem;
    int aux;
  };
  std::map<std::tuple<int, int, int, int, int>, std::vector<Range>> groups;
  const char* kenv = getenv("LIVEPUT_HIST_KERNEL");
  const bool legacy = kenv && std::string(kenv) == "legacy";
  const bool inc_off = kenv && std::string(kenv) == "noinc";
  const bool rows_off = kenv && std::string(kenv) == "norows";
  const bool bits_off = kenv && (std::string(kenv) == "inc" || std::string(kenv) == "noinc");
  for (int pi = 0; pi < (int)hp.pairs.size(); ++pi) {
    const PairDesc& pd = hp.pairs[pi];
    const uint64_t local = pd.t_hi - pd.t_lo;
    if (local == 0 || pd.n_entries == 0) continue;
    const int e_end = pd.entry_base + pd.n_entries;
    if (pd.n > kBigN) {
      // global-scratch kernel (lp_hist_big.cu): one range with every depth
      int e_res = pd.entry_base, pmax = 1;
      while (e_res < e_end && hp.entries[e_res].tmax >= 2) pmax = std::max(pmax, hp.entries[e_res++].P);
      hp.big_words = std::max(hp.big_words, big_scratch_words(pd.n, pd.k, pmax));
      hp.model_ops += local * 6ull * pd.k * (uint64_t)(e_res - pd.entry_base);
      WorkItem w{};
      w.pair = pi;
      w.e_lo = pd.entry_base;
      w.e_hi = e_end;
      w.e_res_hi = e_res;
      w.evt_lo = hp.entries[pd.entry_base].evt_off;
      groups[{specs[pi].stage, 6, 0, kBigThreads, 0}].push_back(
          {w, pd.t_lo, pd.t_hi, std::min<uint64_t>(per_block, 4096), 0, 0});
      continue;
    }
    if (!legacy && !rows_off && pd.k > kIncMaxK && pd.n <= 512 && (bits_off || pd.k > bits_max_k())) {
      // bit-sliced row kernel (lp_hist_rows.cu)
      const RowsShape& rs = rows_shape();
      const int kreg = pd.k <= rs.kreg_max ? 16 : 0;
      int e = pd.entry_base;
      while (e < e_end) {
        int e2 = e;
        int64_t ev = 0;
        while (e2 < e_end) {
          const EntryDesc& x = hp.entries[e2];
          const int64_t ev2 = ev + (int64_t)std::max(0, x.tmax - 1) * x.Dmax;
          if (e2 > e && a16(sizeof(EntryDesc) * (e2 - e + 1)) + a16(2 * (size_t)ev2) > rs.fixed)
            break;
          ev = ev2;
          ++e2;
        }
        int e_res = e;
        int pmax_res = 0;
        while (e_res < e2 && hp.entries[e_res].tmax >= 2) pmax_res = std::max(pmax_res, hp.entries[e_res++].P);
        const int wmax = pmax_res <= 128 ? 4 : 8;
        const bool sm = a16(sizeof(EntryDesc) * (e2 - e)) + a16(2 * (size_t)ev) <= rs.fixed;
        int T = rs.tmax;
        while (T > 32 && smem_rows(e_res - e, pd.k, pd.n, ev, sm, T, kreg, pd.exact) > rs.smem)
          T -= 32;
        const size_t smem = smem_rows(e_res - e, pd.k, pd.n, ev, sm, T, kreg, pd.exact);
        for (int q = e; q < e_res; ++q) hp.model_ops += local * op_model_rows(hp.entries[q]);
        const uint64_t chunk = std::min<uint64_t>((uint64_t)T * 16, per_block);
        auto& gv1 = groups[{specs[pi].stage, 4, kreg * 16 + wmax, T, sm ? 1 : 0}];
        {
          WorkItem w{};
          w.pair = pi;
          w.e_lo = e;
          w.e_hi = e2;
          w.e_res_hi = e_res;
          w.evt_lo = hp.entries[e].evt_off;
          w.evt_len = (int)ev;
          w.smem_evt = sm ? 1 : 0;
          gv1.push_back({w, pd.t_lo, pd.t_hi, (uint64_t)chunk, smem, 0});
        }
        e = e2;
      }
      continue;
    }
    if (!legacy && !bits_off && pd.k <= bits_max_k()) {
      // bit-parallel incidence kernel (lp_hist_bits.cu)
      const int km = pd.k <= 4 ? 4 : (pd.k <= 8 ? 8 : 16);
      const size_t kSmemBudgetBits = km > 8 ? kSmemBudgetBits16 : kSmemBudgetBits8;
      int e = pd.entry_base;
      // groups of 32 resolution depths; a range is a run of entries whose
      // divisor table, depth info and u32 event cells fit the budget (event
      // offsets are packed in 20 bits)
      auto shape = [&](int e0, int e1, int64_t ev, bool sm, int* nres_o, int* ng_o) {
        const int eb0 = (e0 < e1 && hp.entries[e0].P == 1) ? e0 + 1 : e0;
        int nres = 0;
        while (eb0 + nres < e1 && hp.entries[eb0 + nres].tmax >= 2) ++nres;
        const int ng = (nres + 31) / 32;
        *nres_o = nres;
        *ng_o = ng;
        return smem_bits(ng * 32, km, pd.n, ev, sm, ng);
      };
      while (e < e_end) {
        int e2 = e;
        int64_t ev = 0;
        int nres, ng;
        while (e2 < e_end) {
          const EntryDesc& x = hp.entries[e2];
          const int64_t ev2 = ev + (int64_t)std::max(0, x.tmax - 1) * x.Dmax;
          if (e2 > e && x.tmax >= 2 &&
              (shape(e, e2 + 1, ev2, true, &nres, &ng) > kSmemBudgetBits || ev2 >= (1 << 20)))
            break;
          ev = ev2;
          ++e2;
        }
        const size_t sm_need = shape(e, e2, ev, true, &nres, &ng);
        if (nres == 0 && e != pd.entry_base && !(hp.entries[e].P == 1 && hp.entries[e].tmax >= 2)) {
          e = e2;  // nothing to resolve and not the h0 owner
          continue;
        }
        const bool sm = sm_need <= kSmemBudgetBits;
        const size_t smem = shape(e, e2, ev, sm, &nres, &ng);
        const int eb0 = (hp.entries[e].P == 1) ? e + 1 : e;
        const int doff = build_dmask(hp.entries, eb0, nres, pd.n, 1, ng, hp.dmask);
        hp.model_ops += local * op_model_bits(pd.k, km, ng);
        const int T = 256;
        const uint64_t chunk = std::min<uint64_t>((uint64_t)T * 16, per_block);
        auto& gv5 = groups[{specs[pi].stage, 5, km, T, sm ? 1 : 0}];
        {
          WorkItem w{};
          w.pair = pi;
          w.e_lo = e;
          w.e_hi = e2;
          w.e_res_hi = eb0 + nres;
          w.evt_lo = hp.entries[e].evt_off;
          w.evt_len = (int)ev;
          w.smem_evt = sm ? 1 : 0;
          w.dtab_off = doff;
          w.dtab_len = ng;
          gv5.push_back({w, pd.t_lo, pd.t_hi, (uint64_t)chunk, smem, 0});
        }
        e = e2;
      }
      continue;
    }
    if (!legacy && pd.k <= kIncMaxK && !inc_off) {
      // sparse incidence kernel (lp_hist_inc.cu)
      const int km = kmax_for(pd.k);
      int e = pd.entry_base;
      while (e < e_end) {
        int e2 = e;
        int64_t ev = 0;
        while (e2 < e_end) {
          const EntryDesc& x = hp.entries[e2];
          const int64_t ev2 = ev + (int64_t)std::max(0, x.tmax - 1) * x.Dmax;
          if (e2 > e && a16(sizeof(EntryDesc) * (e2 - e + 1)) + a16(4 * (size_t)ev2) > kScnFixedBudget)
            break;
          ev = ev2;
          ++e2;
        }
        int e_res = e;
        while (e_res < e2 && hp.entries[e_res].tmax >= 2) ++e_res;
        const int doff = (int)hp.divtab.size();
        build_divtab(hp.entries, e, e_res, pd.n, hp.divtab);
        hp.model_ops += local * 6ull * pd.k * (uint64_t)(e_res - e);
        const int dlen = (int)hp.divtab.size() - doff;
        const bool sm = a16(sizeof(EntryDesc) * (e2 - e)) + a16(4 * (size_t)ev) <= kScnFixedBudget;
        int T = 128;
        while (T > 32 && smem_inc(e_res - e, km, pd.n, ev, sm, dlen, T) > kSmemBudgetInc) T >>= 1;
        const size_t smem = smem_inc(e_res - e, km, pd.n, ev, sm, dlen, T);
        const uint64_t chunk = std::min<uint64_t>((uint64_t)T * 16, per_block);
        auto& gv2 = groups[{specs[pi].stage, 3, km, T, sm ? 1 : 0}];
        {
          WorkItem w{};
          w.pair = pi;
          w.e_lo = e;
          w.e_hi = e2;
          w.e_res_hi = e_res;
          w.evt_lo = hp.entries[e].evt_off;
          w.evt_len = (int)ev;
          w.smem_evt = sm ? 1 : 0;
          w.dtab_off = doff;
          w.dtab_len = dlen;
          gv2.push_back({w, pd.t_lo, pd.t_hi, (uint64_t)chunk, smem, 0});
        }
        e = e2;
      }
      continue;
    }
    if (!legacy && pd.k > kMaxKReg) {
      // scenario-major kernel (lp_hist_scn.cu)
      const int kreg = (pd.k <= 8) ? 8 : (pd.k <= kMaxKReg ? 16 : 0);
      int e = pd.entry_base;
      while (e < e_end) {
        int e2 = e;
        int64_t ev = 0;
        while (e2 < e_end) {
          const EntryDesc& x = hp.entries[e2];
          const int64_t ev2 = ev + (int64_t)std::max(0, x.tmax - 1) * x.Dmax;
          if (e2 > e && a16(sizeof(EntryDesc) * (e2 - e + 1)) + a16(4 * (size_t)ev2) > kScnFixedBudget)
            break;
          ev = ev2;
          ++e2;
        }
        int e_res = e;
        int pc = 0;
        while (e_res < e2 && hp.entries[e_res].tmax >= 2) {
          if (hp.entries[e_res].Dmax > kComb && hp.entries[e_res].P >= 2)
            pc = std::max(pc, hp.entries[e_res].P);
          ++e_res;
        }
        const int uw = std::max(kreg == 0 ? pd.k : 0, (pc + 1) / 2);
        const bool sm = a16(sizeof(EntryDesc) * (e2 - e)) + a16(4 * (size_t)ev) <= kScnFixedBudget;
        int T = 256;
        while (T > 32 && smem_scn(e_res - e, pd.k, pd.n, ev, sm, T, uw) > kSmemBudgetScn) T >>= 1;
        const size_t smem = smem_scn(e_res - e, pd.k, pd.n, ev, sm, T, uw);
        const uint64_t chunk = std::min<uint64_t>((uint64_t)T * 16, per_block);
        hp.model_ops += local * 6ull * pd.k * (uint64_t)(e_res - e);
        auto& gv3 = groups[{specs[pi].stage, 2, kreg, T, sm ? 1 : 0}];
        {
          WorkItem w{};
          w.pair = pi;
          w.e_lo = e;
          w.e_hi = e2;
          w.e_res_hi = e_res;
          w.evt_lo = hp.entries[e].evt_off;
          w.evt_len = (int)ev;
          w.smem_evt = sm ? 1 : 0;
          gv3.push_back({w, pd.t_lo, pd.t_hi, (uint64_t)chunk, smem, uw});
        }
        e = e2;
      }
      continue;
    }
    if (pd.variant == 0) {
      const int km = kmax_for(pd.k);
      int e = pd.entry_base;
      while (e < e_end) {
        int e2 = e;
        int64_t ev = 0;
        // grow the range while it fits the shared-memory budget
        while (e2 < e_end) {
          const EntryDesc& x = hp.entries[e2];
          const int64_t ev2 = ev + (int64_t)std::max(0, x.tmax - 1) * x.Dmax;
          if (e2 > e && smem_regs(e2 - e + 1, km, pd.n, ev2, true) > kSmemBudgetR) break;
          ev = ev2;
          ++e2;
        }
        int e_res = e;  // depths with Dmax >= 2 (others emit no t >= 2 event)
        while (e_res < e2 && hp.entries[e_res].tmax >= 2) ++e_res;
        const bool sm = smem_regs(e2 - e, km, pd.n, ev, true) <= kSmemBudgetR;
        const size_t smem = smem_regs(e2 - e, km, pd.n, ev, sm);
        {
          WorkItem w{};
          w.pair = pi;
          w.e_lo = e;
          w.e_hi = e2;
          w.evt_lo = hp.entries[e].evt_off;
          w.evt_len = (int)ev;
          w.smem_evt = sm ? 1 : 0;
          w.e_res_hi = e_res;
          groups[{specs[pi].stage, 0, km, 256, sm ? 1 : 0}].push_back({w, pd.t_lo, pd.t_hi, (uint64_t)kChunkR, smem, 0});
        }
        e = e2;
      }
    } else {
      // counter variant: pick the widest block whose single-depth range fits
      int pmax_all = 0;
      for (int e = pd.entry_base; e < e_end; ++e) pmax_all = std::max(pmax_all, hp.entries[e].P);
      int T = 128;
      while (T > 32 && smem_ctr(1, pd.k, pd.n, 0, false, T, pmax_all) > kSmemBudgetC) T >>= 1;
      int e = pd.entry_base;
      while (e < e_end) {
        int e2 = e;
        int64_t ev = 0;
        while (e2 < e_end) {
          const EntryDesc& x = hp.entries[e2];
          const int64_t ev2 = ev + (int64_t)std::max(0, x.tmax - 1) * x.Dmax;
          if (e2 > e && smem_ctr(e2 - e + 1, pd.k, pd.n, ev2, true, T, x.P) > kSmemBudgetC) break;
          ev = ev2;
          ++e2;
        }
        const int pmax = hp.entries[e2 - 1].P;  // entries ascend in P
        const bool sm = smem_ctr(e2 - e, pd.k, pd.n, ev, true, T, pmax) <= kSmemBudgetC;
        const size_t smem = smem_ctr(e2 - e, pd.k, pd.n, ev, sm, T, pmax);
        const uint64_t chunk = (uint64_t)T * 8;
        auto& gv4 = groups[{specs[pi].stage, 1, 0, T, sm ? 1 : 0}];
        {
          WorkItem w{};
          w.pair = pi;
          w.e_lo = e;
          w.e_hi = e2;
          w.evt_lo = hp.entries[e].evt_off;
          w.evt_len = (int)ev;
          w.smem_evt = sm ? 1 : 0;
          gv4.push_back({w, pd.t_lo, pd.t_hi, (uint64_t)chunk, smem, pmax});
        }
        e = e2;
      }
    }
  }
  mark("items");
  int64_t nblk = 0;
  for (auto& [key, items] : groups) {
    Group g;
    g.stage = std::get<0>(key);
    g.kind = std::get<1>(key);
    g.kmax = std::get<2>(key);
    g.threads = std::get<3>(key);
    g.smem_evt = std::get<4>(key) != 0;
    g.first = (int)nblk;
    for (const Range& r : items) g.pmax_cap = std::max(g.pmax_cap, r.aux);
    for (const Range& r : items) {
      size_t sm = r.smem;
      const PairDesc& pd = hp.pairs[r.w.pair];
      if (g.kind == 2)
        sm = smem_scn(r.w.e_res_hi - r.w.e_lo, pd.k, pd.n, r.w.evt_len, g.smem_evt, g.threads, g.pmax_cap);
      if (g.kind == 1)
        sm = smem_ctr(r.w.e_hi - r.w.e_lo, pd.k, pd.n, r.w.evt_len, g.smem_evt, g.threads, g.pmax_cap);
      g.smem = std::max(g.smem, sm);
      if (r.t_hi <= r.t_lo) continue;
      WorkSpan sp{};
      sp.w = r.w;
      sp.w.t0 = r.t_lo;
      sp.w.t1 = r.t_hi;
      sp.chunk = r.chunk;
      sp.first = (int32_t)nblk;
      hp.spans.push_back(sp);
      nblk += (int64_t)((r.t_hi - r.t_lo + r.chunk - 1) / r.chunk);
    }
    g.count = (int)(nblk - g.first);
    hp.groups.push_back(g);
  }
  hp.n_work = nblk;
  if (nblk > INT32_MAX) return LP_EUNSUPPORTED;
  if (nblk <= kHostItems)  // latency-bound small re-plans: one launch fewer
    for (const WorkSpan& sp : hp.spans)
      for (uint64_t t0 = sp.w.t0; t0 < sp.w.t1; t0 += sp.chunk) {
        WorkItem w = sp.w;
        w.t0 = t0;
        w.t1 = std::min(sp.w.t1, t0 + sp.chunk);
        hp.items.push_back(w);
      }
  mark("groups");
  // stage ranges (specs come with non-decreasing stages)
  int nst = 0;
  for (const EnsembleSpec& sp : specs) nst = std::max(nst, sp.stage + 1);
  hp.stages.assign(std::max(nst, 1), HistPlan::Stage{});
  for (int st = 0, pi = 0; st < (int)hp.stages.size(); ++st) {
    HistPlan::Stage& S = hp.stages[st];
    S.p0 = pi;
    while (pi < (int)specs.size() && specs[pi].stage == st) ++pi;
    S.p1 = pi;
    S.e0 = S.p0 < (int)hp.pairs.size() ? hp.pairs[S.p0].entry_base : (int)hp.entries.size();
    S.e1 = S.p1 < (int)hp.pairs.size() ? hp.pairs[S.p1].entry_base : (int)hp.entries.size();
    S.h0 = S.e0 < (int)hp.entries.size() ? hp.entries[S.e0].hist_off : hp.hist_len;
    S.h1 = S.e1 < (int)hp.entries.size() ? hp.entries[S.e1].hist_off : hp.hist_len;
  }
  return LP_OK;
}

struct HistDev {
  const uint16_t* divtab;
  const uint32_t* dmask;
  uint32_t* big_scratch;  // n > kBigN: per stage, grid x kBigThreads x big_words
  size_t big_words;
  int big_grid;
  const PairDesc* pairs;
  const EntryDesc* entries;
  const DrawConst* draws;
  const uint64_t* binom;
  const WorkSpan* spans;
  WorkItem* work;  // expanded from spans by the first launch of an execute
  uint32_t* evt;
  uint32_t* h0;
  uint32_t* hist;
};

cudaError_t run_hist(const HistPlan& hp, const HistDev& d, cudaStream_t st, int* launches) {
  cudaError_t e = launch_expand_work(d.spans, (int)hp.spans.size(), (int)hp.n_work, d.work, st);
  if (e != cudaSuccess) return e;
  if (hp.n_work > 0) ++*launches;
  if (hp.evt_len > 0) {
    e = cudaMemsetAsync(d.evt, 0, sizeof(uint32_t) * hp.evt_len, st);
    if (e != cudaSuccess) return e;
  }
  e = cudaMemsetAsync(d.h0, 0, sizeof(uint32_t) * std::max<int64_t>(hp.h0_len, 1), st);
  if (e != cudaSuccess) return e;
  for (const Group& g : hp.groups) {
    const WorkItem* w = d.work + g.first;
    if (g.kind == 6)
      e = launch_hist_big(g.count, d.big_grid, st, w, d.pairs, d.entries, d.draws, d.binom, d.evt, d.h0,
                          d.big_scratch + (size_t)g.stage * d.big_grid * kBigThreads * d.big_words,
                          d.big_words);
    else if (g.kind == 5)
      e = launch_hist_bits(g.kmax, g.smem_evt, g.count, g.threads, g.smem, st, w,
                           d.pairs, d.entries, d.draws, d.binom, d.dmask, d.evt, d.h0);
    else if (g.kind == 4)
      e = launch_hist_rows(g.kmax / 16, g.kmax % 16, g.smem_evt, g.count, g.threads, g.smem, st, w,
                           d.pairs, d.entries, d.draws, d.binom, d.evt, d.h0);
    else if (g.kind == 3)
      e = launch_hist_inc(g.kmax, g.smem_evt, g.count, g.threads, g.smem, st, w, d.pairs, d.entries,
                          d.draws, d.binom, d.divtab, d.evt, d.h0);
    else if (g.kind == 2)
      e = launch_hist_scn(g.kmax, g.smem_evt, g.count, g.threads, g.smem, g.pmax_cap, st, w, d.pairs,
                          d.entries, d.draws, d.binom, d.evt, d.h0);
    else if (g.kind == 0)
      e = launch_hist_regs(g.kmax, g.smem_evt, g.count, g.smem, st, w, d.pairs, d.entries, d.draws,
                           d.binom, d.evt, d.h0);
    else
      e = launch_hist_ctr(g.smem_evt, g.count, g.threads, g.smem, g.pmax_cap, st, w, d.pairs,
                          d.entries, d.draws, d.binom, d.evt, d.h0);
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  e = launch_finalize((int)hp.pairs.size(), (int)hp.entries.size(), st, d.pairs, d.entries, d.evt,
                      d.h0, d.hist);
  if (!hp.pairs.empty()) *launches += 2;
  return e;
}

// The histogram launches of one pipeline stage and its finalize.
cudaError_t run_hist_stage(const HistPlan& hp, const HistDev& d, cudaStream_t st, int stage,
                           int* launches) {
  cudaError_t e = cudaSuccess;
  for (const Group& g : hp.groups) {
    if (g.stage != stage) continue;
    const WorkItem* w = d.work + g.first;
    if (g.kind == 6)
      e = launch_hist_big(g.count, d.big_grid, st, w, d.pairs, d.entries, d.draws, d.binom, d.evt, d.h0,
                          d.big_scratch + (size_t)g.stage * d.big_grid * kBigThreads * d.big_words,
                          d.big_words);
    else if (g.kind == 5)
      e = launch_hist_bits(g.kmax, g.smem_evt, g.count, g.threads, g.smem, st, w,
                           d.pairs, d.entries, d.draws, d.binom, d.dmask, d.evt, d.h0);
    else if (g.kind == 4)
      e = launch_hist_rows(g.kmax / 16, g.kmax % 16, g.smem_evt, g.count, g.threads, g.smem, st, w,
                           d.pairs, d.entries, d.draws, d.binom, d.evt, d.h0);
    else if (g.kind == 3)
      e = launch_hist_inc(g.kmax, g.smem_evt, g.count, g.threads, g.smem, st, w, d.pairs, d.entries,
                          d.draws, d.binom, d.divtab, d.evt, d.h0);
    else if (g.kind == 2)
      e = launch_hist_scn(g.kmax, g.smem_evt, g.count, g.threads, g.smem, g.pmax_cap, st, w, d.pairs,
                          d.entries, d.draws, d.binom, d.evt, d.h0);
    else if (g.kind == 0)
      e = launch_hist_regs(g.kmax, g.smem_evt, g.count, g.smem, st, w, d.pairs, d.entries, d.draws,
                           d.binom, d.evt, d.h0);
    else
      e = launch_hist_ctr(g.smem_evt, g.count, g.threads, g.smem, g.pmax_cap, st, w, d.pairs,
                          d.entries, d.draws, d.binom, d.evt, d.h0);
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  return e;
}

// thr(D, P) rows for the depths a plan touches
struct ThrTable {
  std::vector<int32_t> row;   // by P: offset, -1 if absent
  std::vector<double> vals;
};

void build_thr(Model& m, const std::map<int, int>& need, int pmax, ThrTable& t) {
  t.row.assign(pmax + 2, -1);
  t.vals.clear();
  for (const auto& [P, Dm] : need) {
    t.row[P] = (int32_t)t.vals.size();
    for (int D = 0; D <= Dm; ++D) t.vals.push_back(D == 0 ? 0.0 : m.rate_cached(D, P));
  }
}


// ---------------------------------------------------------------------------
// NCCL is bound at run time (dlopen) so this library never drags a second
// libnccl.so.2 into a process that also loads torch's bundled NCCL.
// LIVEPUT_NCCL_LIB may name the library; default "libnccl.so.2" (which
// resolves to the already-loaded copy when torch was imported first).
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    const char* env = getenv("LIVEPUT_NCCL_LIB");
    void* so = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!so) return a;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(so, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(so, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(so, "ncclCommDestroy");
    a.AllReduce = (decltype(a.AllReduce))dlsym(so, "ncclAllReduce");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(so, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.GetErrorString;
    return a;
  }();
  return api;
}

}  // namespace
}  // namespace lp

using namespace lp;

// ---------------------------------------------------------------------------
struct lp_handle {
  Model model;
  lp_costs costs{};
  lp_options opt{};
  CostScalars cs{};
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;     // histograms, collectives, fetch (lp_stream)
  cudaStream_t stream_dp = nullptr;  // DP tables and DP kernels, joined back into `stream`
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  static constexpr int kMaxStages = 16;
  cudaEvent_t ev_stage[kMaxStages] = {};  // probabilities of stage s are in the store
  cudaStream_t stream_hist[kMaxStages] = {};  // histogram kernels of stage s
  cudaEvent_t ev_hist[kMaxStages] = {};       // ... done
  cudaEvent_t ev_start = nullptr;             // scratch cleared for this execute
  cudaEvent_t ev_join = nullptr;
  // materialised phi (pipelined re-plans): the phi launches of stage s run on
  // their own stream and release the max-plus levels with ev_phi[s]
  cudaStream_t stream_phi = nullptr;
  cudaEvent_t ev_phi[kMaxStages] = {};
  std::vector<cudaEvent_t> ev_lvl;        // last stage: phi of level j done
  bool phi_on = false;
  DevBuf phi;
  std::vector<int32_t> phi_list;          // levels ordered by the stage that releases them
  std::vector<int> phi_range;             // per stage: [phi_range[s], phi_range[s+1]) of phi_list
  std::vector<int64_t> phi_maxpairs;      // per stage: largest prev count (the phi grid)
  size_t off_phi_list = 0;
  std::vector<cudaEvent_t> tl_ev;  // LIVEPUT_TIMELINE: one event per DP level (diagnostics)
  std::vector<int> level_need;  // per DP level: the last stage it must wait for (-1: none)
  std::string err;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  int shard_rank = 0, shard_n = 1;  // lp_set_shard: survivor_hist on one trial slice

  // re-plan state
  bool prepared = false;
  int horizon = 0;
  HistPlan hp;
  std::vector<LevelDesc> levels;
  std::vector<NodeCfg> cfg;
  std::vector<double4> pcost;  // per depth: pipe transfer, inter unit, resume cost
  std::vector<int4> lrows;
  // per availability n: the level's nodes (configs of n + suspension) and
  // the largest D per depth (n / P), built once — the profile is fixed
  std::vector<std::vector<NodeCfg>> level_nodes;
  std::vector<DenseMap<int>> level_depths;
  ThrTable thr;
  DpScalars S{};
  size_t off_divtab = 0, off_dmask = 0;
  size_t off_pairs = 0, off_entries = 0, off_draws = 0, off_binom = 0, off_work = 0,
         off_levels = 0, off_cfg = 0, off_cost = 0, off_lrows = 0, off_thr = 0, off_throw = 0,
         off_gather = 0, off_pbase = 0;
  std::vector<int32_t> dp_gather, dp_pbase;  // cluster DP staging lists
  size_t w_items = 0;  // the expanded WorkItems of the histogram launches
  size_t off_items = 0;  // ... or the host-expanded ones of a small plan
  size_t w_evt = 0, w_h0 = 0, w_hist = 0, w_val = 0, w_mig = 0, w_par = 0, w_stc = 0, w_stm = 0,
         w_plan = 0, w_live = 0, w_final = 0, w_bar = 0;
  int max_next = 0;         // largest level (next role), for the persistent DP grid
  bool live_pending = false;  // liveput rows of the last execute not yet computed
  bool dp_launches = false;  // LIVEPUT_DP=launches: one kernel per level (A/B)
  bool dp_staged = true;     // LIVEPUT_DP_STAGED=0: never stage the DP in shared memory (A/B)
  int dp_staged_nprob = -1;  // >= 0: this re-plan's persistent DP runs staged
  bool dp_cluster = false;   // ... as the 8-CTA cluster kernel (small re-plans)
  int dp_staged_kb = 100;    // shared-memory budget of the staged DP (LIVEPUT_DP_STAGED_KB)
  DevBuf tables, work;
  DevBuf big_scratch;  // lp_hist_big.cu scratch (n > kBigN only)
  PinBuf pin_up, pin_down;
  size_t up_bytes = 0;
  lp_stats stats{};
  // DP tables: a second image, so lp_replan can build and upload them while
  // the histogram kernels run
  DevBuf tables2;
  DevBuf dp_trace;  // LIVEPUT_DP_TRACE
  PinBuf pin_up2;
  cudaEvent_t ev_up[2] = {nullptr, nullptr};  // last upload out of pin_up / pin_up2
  struct PrepState {
    int len = 0;
    std::vector<int32_t> n_seq;
    std::vector<int> lbase, lcount, level_spec;
    std::vector<EnsembleSpec> specs;
    size_t fresh = 0;
    double host_ms = 0.0;
  } ps;

  // ensemble calls (phi / survivor_hist / liveput) and their cache
  DevBuf e_tables, e_work;
  std::map<std::tuple<int, int, int>, std::pair<int, std::vector<uint32_t>>> hist_cache;

  // device histogram store (FP64 probabilities, see lp_prepare)
  struct StoreSlot {
    uint64_t count = 0;                         // ensemble size
    DenseMap<std::pair<int, int>> ents;         // P -> (Dmax, store offset of D = 1)
  };
  bool cache_on = false;
  uint64_t cache_max = 4ull << 30;              // bytes
  std::map<std::pair<int, int>, StoreSlot> store_idx;
  DevBuf store;
  size_t store_used = 0;                        // doubles
  std::vector<int32_t> store_off;               // per fresh entry
  size_t off_store_off = 0;
};

namespace {

lp_status fail(lp_handle* h, lp_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  else g_global_err = buf;
  return s;
}

#define LP_CUDA(h, call)                                                               \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      return fail((h), LP_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, \
                  __LINE__);                                                           \
  } while (0)

template <typename T>
T* dptr(DevBuf& b, size_t off) {
  return reinterpret_cast<T*>(static_cast<unsigned char*>(b.p) + off);
}

// Builds and uploads a hist plan into (tables, work); returns device ptrs.
// Scratch of the big-n kernel: one slice per (stage, thread of its grid).
lp_status bind_big_scratch(lp_handle* h, const HistPlan& hp, HistDev& d) {
  d.big_words = hp.big_words;
  d.big_grid = std::max(1, h->num_sms);
  d.big_scratch = nullptr;
  if (hp.big_words == 0) return LP_OK;
  const size_t bytes = 4 * hp.big_words * (size_t)d.big_grid * kBigThreads * std::max<size_t>(hp.stages.size(), 1);
  LP_CUDA(h, h->big_scratch.ensure(bytes));
  d.big_scratch = static_cast<uint32_t*>(h->big_scratch.p);
  return LP_OK;
}

lp_status upload_hist(lp_handle* h, const HistPlan& hp, DevBuf& tables, DevBuf& work, HistDev& d,
                      Packer& pk, std::vector<size_t>& extra_offs) {
  (void)extra_offs;
  const size_t op = pk.add(hp.pairs), oe = pk.add(hp.entries), od = pk.add(hp.draws),
               ob = pk.add(hp.binom), ow = pk.add(hp.spans), odt = pk.add(hp.divtab),
               odm = pk.add(hp.dmask);
  LP_CUDA(h, tables.ensure(pk.bytes.size()));
  LP_CUDA(h, h->pin_up.ensure(pk.bytes.size()));
  std::memcpy(h->pin_up.p, pk.bytes.data(), pk.bytes.size());
  LP_CUDA(h, cudaMemcpyAsync(tables.p, h->pin_up.p, pk.bytes.size(), cudaMemcpyHostToDevice,
                             h->stream));
  const size_t wb0 = a16(4 * std::max<int64_t>(hp.evt_len, 1)) + a16(4 * std::max<int64_t>(hp.h0_len, 1)) +
                     a16(4 * std::max<int64_t>(hp.hist_len, 1));
  const size_t wb = wb0 + a16(sizeof(WorkItem) * std::max<int64_t>(hp.n_work, 1));
  LP_CUDA(h, work.ensure(wb));
  d.pairs = dptr<PairDesc>(tables, op);
  d.entries = dptr<EntryDesc>(tables, oe);
  d.draws = dptr<DrawConst>(tables, od);
  d.binom = dptr<uint64_t>(tables, ob);
  d.spans = dptr<WorkSpan>(tables, ow);
  d.work = dptr<WorkItem>(work, wb0);
  d.divtab = dptr<uint16_t>(tables, odt);
  d.dmask = dptr<uint32_t>(tables, odm);
  {
    lp_status bs = bind_big_scratch(h, hp, d);
    if (bs != LP_OK) return bs;
  }
  d.evt = dptr<uint32_t>(work, 0);
  d.h0 = dptr<uint32_t>(work, a16(4 * std::max<int64_t>(hp.evt_len, 1)));
  d.hist = dptr<uint32_t>(work, a16(4 * std::max<int64_t>(hp.evt_len, 1)) +
                                    a16(4 * std::max<int64_t>(hp.h0_len, 1)));
  return LP_OK;
}

// Planner ensemble semantics (optimizer.cpp:64-94).
lp_status planner_spec(lp_handle* h, int n, int k, EnsembleSpec& sp) {
  if (k < 0 || k > n) return fail(h, LP_EINVAL, "sample_vectors: bad n_minus");
  sp.n = n;
  sp.k = k;
  const uint64_t cnt = scenario_count(n, k);
  sp.exact = cnt <= h->opt.exact_cap;
  if (sp.exact) {
    if (cnt > kEnumerationCap)
      return fail(h, LP_EINVAL, "enumerate_vectors: scenario space too large, sample instead");
    sp.count = cnt;
  } else {
    if (h->opt.mc_trials < 1) return fail(h, LP_EINVAL, "sample_vectors: trials must be >= 1");
    sp.count = (uint64_t)h->opt.mc_trials;
  }
  sp.seed = mix_seed(mix_seed(h->opt.mc_seed, (uint64_t)n), (uint64_t)k);
  return LP_OK;
}

// Runs one ensemble (single GPU) for the entries of `sp` and returns the
// u32 histogram rows of (D, P) in `rows` (d = 0..min(k, D)).
lp_status ensemble_rows(lp_handle* h, const EnsembleSpec& sp, int D, int P,
                        std::vector<uint32_t>& rows) {
  HistPlan hp;
  std::string err;
  lp_status s = build_hist_plan({sp}, 0, 1, hp, err);
  if (s != LP_OK) return fail(h, s, "%s", err.c_str());
  Packer pk;
  HistDev d{};
  std::vector<size_t> extra;
  s = upload_hist(h, hp, h->e_tables, h->e_work, d, pk, extra);
  if (s != LP_OK) return s;
  int launches = 0;
  LP_CUDA(h, run_hist(hp, d, h->stream, &launches));
  // locate (D, P)
  int e = -1;
  for (size_t i = 0; i < hp.entries.size(); ++i)
    if (hp.entries[i].P == P) e = (int)i;
  if (e < 0 || D > hp.entries[e].Dmax) return fail(h, LP_EINVAL, "internal: entry missing");
  const int off = hp.entries[e].hist_off + hist_row(D, sp.k);
  const int len = std::min(sp.k, D) + 1;
  rows.assign(len, 0);
  LP_CUDA(h, h->pin_down.ensure(sizeof(uint32_t) * len));
  LP_CUDA(h, cudaMemcpyAsync(h->pin_down.p, d.hist + off, sizeof(uint32_t) * len,
                             cudaMemcpyDeviceToHost, h->stream));
  LP_CUDA(h, cudaStreamSynchronize(h->stream));
  std::memcpy(rows.data(), h->pin_down.p, sizeof(uint32_t) * len);
  return LP_OK;
}

// Cached planner histogram of (D, P) at (n, k): the reference's hist_cache_
// (optimizer.hpp:88) keyed by (n, k, P) with the largest D computed.
lp_status planner_rows(lp_handle* h, int D, int P, int n, int k, std::vector<uint32_t>& rows,
                       uint64_t* total) {
  EnsembleSpec sp;
  lp_status s = planner_spec(h, n, k, sp);
  if (s != LP_OK) return s;
  const uint64_t t_lo = sp.count * (uint64_t)h->shard_rank / (uint64_t)h->shard_n;
  const uint64_t t_hi = sp.count * (uint64_t)(h->shard_rank + 1) / (uint64_t)h->shard_n;
  *total = t_hi - t_lo;
  auto key = std::make_tuple(n, k, P);
  auto it = h->hist_cache.find(key);
  if (it == h->hist_cache.end() || it->second.first < D) {
    const int Dm = n / P;  // every D of this depth at once
    sp.dmax_by_p[P] = std::max(Dm, D);
    std::vector<uint32_t> all;
    // fetch all rows of the entry: run and copy D = 1..Dm.  With a shard
    // set this is the rank's slice of the multi-GPU split (build_hist_plan's
    // t_lo / t_hi, finalize with the local ensemble size).
    HistPlan hp;
    std::string err;
    s = build_hist_plan({sp}, h->shard_rank, h->shard_n, hp, err);
    if (s != LP_OK) return fail(h, s, "%s", err.c_str());
    Packer pk;
    HistDev d{};
    std::vector<size_t> extra;
    s = upload_hist(h, hp, h->e_tables, h->e_work, d, pk, extra);
    if (s != LP_OK) return s;
    int launches = 0;
    LP_CUDA(h, run_hist(hp, d, h->stream, &launches));
    const size_t len = (size_t)hp.hist_len;
    LP_CUDA(h, h->pin_down.ensure(sizeof(uint32_t) * len));
    LP_CUDA(h, cudaMemcpyAsync(h->pin_down.p, d.hist, sizeof(uint32_t) * len,
                               cudaMemcpyDeviceToHost, h->stream));
    LP_CUDA(h, cudaStreamSynchronize(h->stream));
    all.assign(static_cast<uint32_t*>(h->pin_down.p), static_cast<uint32_t*>(h->pin_down.p) + len);
    h->hist_cache[key] = {sp.dmax_by_p[P], std::move(all)};
    it = h->hist_cache.find(key);
  }
  const int off = hist_row(D, k);
  const int len = std::min(k, D) + 1;
  rows.assign(it->second.second.begin() + off, it->second.second.begin() + off + len);
  return LP_OK;
}

// Grows the histogram store to `doubles` entries, keeping the cached content.
lp_status grow_store(lp_handle* h, size_t doubles) {
  const size_t bytes = std::max<size_t>(doubles, 1) * sizeof(double);
  if (bytes <= h->store.cap) return LP_OK;
  void* np = nullptr;
  size_t want = std::max<size_t>(bytes + bytes / 2, 1 << 20);
  cudaError_t e = cudaMalloc(&np, want);
  if (e != cudaSuccess) return fail(h, LP_ENOMEM, "histogram store: %s", cudaGetErrorString(e));
  if (h->store.p) {
    LP_CUDA(h, cudaMemcpyAsync(np, h->store.p, h->store.cap, cudaMemcpyDeviceToDevice, h->stream));
    LP_CUDA(h, cudaStreamSynchronize(h->stream));
    cudaFree(h->store.p);
  }
  h->store.p = np;
  h->store.cap = want;
  return LP_OK;
}

NodeCost node_cost(lp_handle* h, int d, int p) {
  NodeCost c{};
  if (d <= 0) return c;
  c.thr = h->model.rate_cached(d, p);
  c.pipe = h->model.pipe_transfer(p);
  c.unit = h->model.inter_unit(p);
  // resume_cost (migration.cpp:100-104)
  c.resume = h->cs.fresh_fixed + h->cs.build + h->cs.update + c.pipe;
  return c;
}

DpScalars dp_scalars(lp_handle* h, int horizon) {
  DpScalars S{};
  S.T = h->opt.interval_s;
  S.build = h->cs.build;
  S.update = h->cs.update;
  S.rollback = h->opt.rollback_penalty_s;
  S.fresh_fixed = h->cs.fresh_fixed;
  S.strict = h->opt.strict_conditional;
  S.horizon = horizon;
  return S;
}

}  // namespace

// ===========================================================================
extern "C" {

const char* lp_last_global_error(void) { return g_global_err.c_str(); }
const char* lp_last_error(const lp_handle* h) { return h ? h->err.c_str() : g_global_err.c_str(); }

int32_t lp_max_instances(void) { return kMaxN; }

const char* lp_build_info(void) {
  return "liveput sm_100a (tcgen05-free integer/FP64 path); kMaxN=16384 (global-scratch kernel past 2048); any k";
}

lp_status lp_create(const lp_profile* profile, const lp_costs* costs, const lp_options* options,
                    int32_t device, lp_handle** out) {
  if (!profile || !costs || !options || !out)
    return fail(nullptr, LP_EINVAL, "lp_create: null argument");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, LP_ECUDA, "lp_create: no CUDA device (%s)", cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(nullptr, LP_EINVAL, "lp_create: bad device %d", device);
  lp_handle* h = new lp_handle();
  h->model = Model(*profile);
  h->costs = *costs;
  h->opt = *options;
  h->cs = cost_scalars(*costs);
  h->device = device;
  // Stream priorities (LIVEPUT_PRIO, default 3): the stage-s histogram
  // streams one step below each other so that stage 0's blocks are dispatched
  // first and it finishes first (with equal priorities the scheduler
  // interleaves the three stages and they finish in reverse order, so no DP
  // level can start early), the library stream highest, and the DP stream
  // lowest, so DP blocks only take slots the sampling leaves free.  Measured
  // on B200: 4 GPUs 1.87 ms against 1.95 ms with equal priorities, 1 GPU
  // 6.44-6.50 against 6.53 ms.  0: all equal; 1: DP highest; 2: DP at stage 0's.
  static const int prio = [] {
    const char* pe = getenv("LIVEPUT_PRIO");
    return pe ? atoi(pe) : 3;
  }();
  int least = 0, greatest = 0;
  if (prio) cudaDeviceGetStreamPriorityRange(&least, &greatest);
  const int dp_prio = prio == 2 ? std::min(least, greatest + 1) : (prio == 3 ? least : greatest);
  if ((e = cudaSetDevice(device)) != cudaSuccess ||
      (e = cudaStreamCreateWithPriority(&h->stream, cudaStreamNonBlocking, greatest)) != cudaSuccess ||
      (e = cudaStreamCreateWithPriority(&h->stream_dp, cudaStreamNonBlocking, dp_prio)) != cudaSuccess) {
    delete h;
    return fail(nullptr, LP_ECUDA, "lp_create: %s", cudaGetErrorString(e));
  }
  const unsigned tflag = timeline() ? cudaEventDefault : cudaEventDisableTiming;
  for (auto& ev : h->ev) cudaEventCreate(&ev);
  for (auto& ev : h->ev_up) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  for (auto& ev : h->ev_stage) cudaEventCreateWithFlags(&ev, tflag);
  for (auto& ev : h->ev_hist) cudaEventCreateWithFlags(&ev, tflag);
  for (int q = 0; q < lp_handle::kMaxStages; ++q)
    cudaStreamCreateWithPriority(&h->stream_hist[q], cudaStreamNonBlocking,
                                 prio ? std::min(least, greatest + 1 + q) : 0);
  cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming);
  for (auto& ev : h->ev_phi) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  {
    // LIVEPUT_PHI_PRIO: phi launches at the highest priority (default), 1:
    // at stage 0's, 2: the lowest (A/B)
    static const int pp = [] {
      const char* e = getenv("LIVEPUT_PHI_PRIO");
      return e ? atoi(e) : 0;
    }();
    const int phi_prio = pp == 1 ? std::min(least, greatest + 1) : (pp == 2 ? least : greatest);
    cudaStreamCreateWithPriority(&h->stream_phi, cudaStreamNonBlocking, phi_prio);
  }
  {
    const char* e = getenv("LIVEPUT_DP");
    h->dp_launches = (e && std::string(e) == "launches");
    const char* es = getenv("LIVEPUT_DP_STAGED");
    h->dp_staged = !(es && es[0] == '0');
    if (const char* ek = getenv("LIVEPUT_DP_STAGED_KB")) h->dp_staged_kb = std::max(0, std::min(200, atoi(ek)));
  }
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  {
    const auto t0 = std::chrono::steady_clock::now();
    preload_kernels();
    if (getenv("LIVEPUT_TRACE_PREPARE"))
      fprintf(stderr, "[create] preload %8.3f ms\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  // The staging and table buffers at their minimum sizes (what a small
  // re-plan needs): cudaMallocHost / cudaMalloc inside the first re-plan
  // cost it 2-3 ms (profiles/r02_cold_replan.log).  They grow on demand;
  // larger sizes up front made every lp_create 5-18 ms.
  if ((e = h->pin_up.ensure(1 << 16)) != cudaSuccess || (e = h->pin_up2.ensure(1 << 16)) != cudaSuccess ||
      (e = h->pin_down.ensure(1 << 16)) != cudaSuccess || (e = h->tables.ensure(1 << 16)) != cudaSuccess ||
      (e = h->tables2.ensure(1 << 16)) != cudaSuccess || (e = h->work.ensure(1 << 18)) != cudaSuccess) {
    lp_destroy(h);
    return fail(nullptr, LP_ECUDA, "lp_create: %s", cudaGetErrorString(e));
  }
  if (grow_store(h, size_t(1) << 16) != LP_OK) {
    const std::string msg = h->err;
    lp_destroy(h);
    return fail(nullptr, LP_ENOMEM, "lp_create: %s", msg.c_str());
  }
  *out = h;
  return LP_OK;
}

void lp_destroy(lp_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->comm) nccl().CommDestroy(h->comm);
  for (auto& ev : h->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : h->ev_up)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : h->ev_stage)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : h->ev_hist)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : h->tl_ev) cudaEventDestroy(ev);
  for (auto& sh : h->stream_hist)
    if (sh) {
      cudaStreamSynchronize(sh);
      cudaStreamDestroy(sh);
    }
  if (h->ev_start) cudaEventDestroy(h->ev_start);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  for (auto& ev : h->ev_phi)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : h->ev_lvl) cudaEventDestroy(ev);
  if (h->stream_phi) {
    cudaStreamSynchronize(h->stream_phi);
    cudaStreamDestroy(h->stream_phi);
  }
  if (h->stream_dp) {
    cudaStreamSynchronize(h->stream_dp);
    cudaStreamDestroy(h->stream_dp);
  }
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

lp_status lp_get_options(const lp_handle* h, lp_options* out) {
  if (!h || !out) return fail(nullptr, LP_EINVAL, "null argument");
  *out = h->opt;
  return LP_OK;
}

void* lp_stream(lp_handle* h) { return h ? (void*)h->stream : nullptr; }

}  // extern "C"

// ---------------------------------------------------------------------------
namespace {

struct Section {
  const void* src;
  size_t bytes;
  size_t* off;  // receives the section's offset in the image
};

template <typename T>
Section sec(const std::vector<T>& v, size_t* off) {
  return {v.data(), v.size() * sizeof(T), off};
}

// Lays the sections out (256-byte aligned) straight into the pinned staging
// buffer and uploads them with one copy on the handle's stream.  `done`
// marks the previous upload out of `pin`, which must finish before the
// staging memory is rewritten.
lp_status upload_image(lp_handle* h, std::initializer_list<Section> secs, DevBuf& dst, PinBuf& pin,
                       cudaEvent_t done, size_t* total, cudaStream_t st) {
  size_t o = 0;
  for (const Section& x : secs) {
    *x.off = o;
    o += (std::max<size_t>(x.bytes, 1) + 255) & ~size_t(255);
  }
  LP_CUDA(h, cudaEventSynchronize(done));
  LP_CUDA(h, pin.ensure(o));
  LP_CUDA(h, dst.ensure(o));
  unsigned char* base = static_cast<unsigned char*>(pin.p);
  for (const Section& x : secs)
    if (x.bytes) std::memcpy(base + *x.off, x.src, x.bytes);
  LP_CUDA(h, cudaMemcpyAsync(dst.p, pin.p, o, cudaMemcpyHostToDevice, st));
  LP_CUDA(h, cudaEventRecord(done, st));
  *total = o;
  return LP_OK;
}

double ms_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}

bool trace_prepare() {
  static const bool on = getenv("LIVEPUT_TRACE_PREPARE") != nullptr;
  return on;
}

// prepare, part 1: levels (optimizer.cpp:148-183), ensembles and the
// histogram plan; uploads the histogram image and sizes the work arena.
lp_status prepare_hist(lp_handle* h, lp_config current, const int32_t* n_seq, int32_t len) {
  if (!h) return fail(nullptr, LP_EINVAL, "null handle");
  const auto t_start = std::chrono::steady_clock::now();
  const bool trace = trace_prepare();
  auto mark = [&](const char* what) {
    if (trace) fprintf(stderr, "[prepare] %-10s %8.3f ms\n", what, ms_since(t_start));
  };
  h->prepared = false;  // until prepare_dp has run
  if (!n_seq || len < 2) return fail(h, LP_EINVAL, "dp_optimize: need at least N_i and N_{i+1}");
  cudaSetDevice(h->device);
  mark("setdev");
  for (int i = 0; i < len; ++i) {
    if (n_seq[i] < 0) return fail(h, LP_EINVAL, "dp_optimize: negative availability");
    if (n_seq[i] > kMaxN)
      return fail(h, LP_EUNSUPPORTED, "dp_optimize: n=%d exceeds supported maximum %d", n_seq[i], kMaxN);
  }
  const bool cur_on = current.pipelines > 0;
  if (cur_on) {
    if (current.stages < 1) return fail(h, LP_EINVAL, "dp_optimize: current config has no stages");
    if ((long long)current.pipelines * current.stages > n_seq[0])
      // the reference reads past the preemption vector here (preemption.cpp:63)
      return fail(h, LP_EINVAL, "dp_optimize: current config exceeds n_seq[0]");
  }
  const int H = len - 1;
  h->horizon = H;
  h->levels.assign(H, LevelDesc{});
  h->cfg.clear();
  {
    size_t total = 1;
    for (int j = 1; j <= H; ++j) total += h->model.configs(n_seq[j]).size() + 1;
    h->cfg.reserve(total);
  }
  std::vector<int> lbase(H + 1), lcount(H + 1);
  mark("reserve");
  // level 0: current
  lbase[0] = 0;
  lcount[0] = 1;
  h->cfg.push_back({cur_on ? current.pipelines : 0, cur_on ? current.stages : 0, -1, 0});
  auto nodes_of = [&](int n) -> const std::vector<NodeCfg>& {
    if ((int)h->level_nodes.size() <= n) {
      h->level_nodes.resize(n + 1);
      h->level_depths.resize(n + 1);
    }
    std::vector<NodeCfg>& v = h->level_nodes[n];
    if (v.empty()) {
      for (const Cfg& c : h->model.configs(n)) {
        v.push_back({c.d, c.p, -1, 0});
        int& dm = h->level_depths[n][c.p];  // ascending P, the first D of a P is n / P
        dm = std::max(dm, c.d);
      }
      v.push_back({0, 0, -1, 0});  // suspension is always reachable
    }
    return v;
  };
  for (int j = 1; j <= H; ++j) {
    lbase[j] = (int)h->cfg.size();
    const std::vector<NodeCfg>& v = nodes_of(n_seq[j]);
    h->cfg.insert(h->cfg.end(), v.begin(), v.end());
    lcount[j] = (int)h->cfg.size() - lbase[j];
  }
  mark("levels");
  // ensembles: one per distinct (n_now, k) whose histograms phi will read.
  // Level j >= 1 needs every config of n_now (all D <= n/P of each feasible
  // P); level 0 needs only `current`.
  std::map<std::pair<int, int>, int> spec_of;
  std::vector<EnsembleSpec> specs;
  std::vector<char> spec_full;             // some level j >= 1 uses the spec
  std::vector<std::pair<int, int>> spec_cur;  // (D, P) of current when level 0 uses it
  std::vector<int> level_spec(H, -1);
  for (int j = 0; j < H; ++j) {
    const int n_now = n_seq[j], n_next = n_seq[j + 1];
    const int k = std::max(0, n_now - n_next);
    const bool any_prev = (j == 0) ? cur_on : !h->model.configs(n_now).empty();
    const bool any_next = !h->model.configs(n_next).empty();
    if (!any_prev || !any_next) continue;
    auto key = std::make_pair(n_now, k);
    auto it = spec_of.find(key);
    if (it == spec_of.end()) {
      EnsembleSpec sp;
      lp_status s = planner_spec(h, n_now, k, sp);
      if (s != LP_OK) return s;
      it = spec_of.emplace(key, (int)specs.size()).first;
      specs.push_back(sp);
      spec_full.push_back(0);
      spec_cur.push_back({0, 0});
    }
    const int si = it->second;
    EnsembleSpec& sp = specs[si];
    if (j == 0) {
      // Dmax = floor(n / P) like every full-level entry (not current.pipelines):
      // the kernels resolve t >= 2 events only over the prefix of entries with
      // tmax >= 2, so Dmax must stay non-increasing in P even when current's
      // depth is infeasible and sorts below every feasible one.
      int& dm = sp.dmax_by_p[current.stages];
      dm = std::max(dm, std::max(current.pipelines, n_now / current.stages));
      spec_cur[si] = {current.pipelines, current.stages};
    } else if (!spec_full[si]) {
      spec_full[si] = 1;
      nodes_of(n_now);
      const DenseMap<int>& full = h->level_depths[n_now];
      if (sp.dmax_by_p.size() == 0) {
        sp.dmax_by_p = full;
      } else {
        for (const auto& [P, D] : full) {
          int& dm = sp.dmax_by_p[P];
          dm = std::max(dm, D);
        }
      }
    }
    level_spec[j] = si;
  }
  // distinct (D, P, n, k) histogram keys the reference would tally
  for (size_t si = 0; si < specs.size(); ++si) {
    uint64_t keys = spec_full[si] ? h->model.configs(specs[si].n).size() : 0;
    const auto [cd, cp] = spec_cur[si];
    if (cd > 0) {
      const bool covered = spec_full[si] && h->model.depth_ok(cp) && cd <= specs[si].n / cp;
      if (!covered) keys += 1;
    }
    specs[si].ref_keys = keys;
  }
  // Device histogram store: probabilities of every ensemble live in one HBM
  // array keyed by (n, k).  With the cache on, ensembles already in the store
  // (covering the depths this re-plan reads) are not recomputed — the
  // reference's hist_cache_ (optimizer.hpp:88); the cache is valid for the
  // handle's lifetime because options and profile are fixed.
  std::vector<EnsembleSpec> fresh;
  std::vector<int> fresh_of(specs.size(), -1);
  for (int pass = 0; pass < 2; ++pass) {
    if (!h->cache_on || pass == 1) {
      h->store_idx.clear();
      h->store_used = 0;
    }
    fresh.clear();
    std::fill(fresh_of.begin(), fresh_of.end(), -1);
    size_t need = 0;
    for (size_t si = 0; si < specs.size(); ++si) {
      auto it = h->store_idx.find({specs[si].n, specs[si].k});
      bool covered = it != h->store_idx.end();
      if (covered)
        for (const auto& [P, Dm] : specs[si].dmax_by_p) {
          const auto* e = it->second.ents.find(P);
          if (!e || e->first < Dm) covered = false;
        }
      if (covered) continue;
      EnsembleSpec sp = specs[si];
      if (it != h->store_idx.end())  // keep what the old slot covered
        for (const auto& [P, v] : it->second.ents) {
          int& dm = sp.dmax_by_p[P];
          dm = std::max(dm, v.first);
        }
      for (const auto& [P, Dm] : sp.dmax_by_p) need += hist_row(Dm + 1, sp.k);
      fresh_of[si] = (int)fresh.size();
      fresh.push_back(sp);
    }
    if (h->store_used + need <= h->cache_max / 8 || pass == 1) break;  // else evict all, retry
  }
  // Pipeline stages: the fresh ensembles, in the order the DP first reads
  // them, are cut into up to kMaxStages groups of similar work, so the DP
  // of the early intervals runs on its own stream while the later
  // histograms are still being sampled.
  {
    // LIVEPUT_STAGES = 1..4: shrinking cost cuts; 0: one stage per ensemble
    static const int want_env = [] {
      const char* e = getenv("LIVEPUT_STAGES");
      return e ? atoi(e) : 3;
    }();
    const int want = want_env == 0 ? std::min((int)fresh.size(), (int)lp_handle::kMaxStages)
                                   : std::max(1, std::min(want_env, 4));
    uint64_t total = 0, scen = 0;
    std::vector<uint64_t> cost(fresh.size());
    for (size_t i = 0; i < fresh.size(); ++i) {
      const uint64_t local = fresh[i].count / (uint64_t)std::max(h->nranks, 1);
      cost[i] = alg_ops(local, fresh[i].k, (int)fresh[i].dmax_by_p.size());
      total += cost[i];
      scen += local;
    }
    const bool staged = want > 1 && fresh.size() >= 2 && scen >= (1u << 18);
    // shrinking stages: the DP left to run after the last one is short
    static const double kCuts[5][4] = {{1.0}, {0.75, 1.0}, {0.5, 0.85, 1.0}, {0.4, 0.7, 0.9, 1.0}, {}};
    static const std::vector<double> env_cuts = [] {  // LIVEPUT_STAGE_CUTS=0.5,0.8,0.95 (A/B)
      std::vector<double> c;
      if (const char* e = getenv("LIVEPUT_STAGE_CUTS")) {
        std::string v(e);
        size_t pos = 0;
        while (pos < v.size()) {
          const size_t q = v.find(',', pos);
          c.push_back(atof(v.substr(pos, q == std::string::npos ? std::string::npos : q - pos).c_str()));
          if (q == std::string::npos) break;
          pos = q + 1;
        }
      }
      return c;
    }();
    uint64_t cum = 0;
    int last = 0;
    for (size_t i = 0; i < fresh.size(); ++i) {
      int st = 0;
      if (staged && total > 0) {
        if (want_env == 0) {
          st = (int)std::min<size_t>(i, want - 1);
        } else {
          const double mid = (static_cast<double>(cum) + 0.5 * static_cast<double>(cost[i])) / static_cast<double>(total);
          if (!env_cuts.empty()) {
            while (st < (int)env_cuts.size() && st < (int)lp_handle::kMaxStages - 1 && mid > env_cuts[st]) ++st;
          } else {
            while (st < want - 1 && mid > kCuts[want - 1][st]) ++st;
          }
        }
      }
      st = std::max(st, last);
      fresh[i].stage = st;
      last = st;
      cum += cost[i];
    }
    int next_id = -1, prev_raw = -1;  // renumber consecutively
    for (auto& f : fresh) {
      if (f.stage != prev_raw) {
        prev_raw = f.stage;
        ++next_id;
      }
      f.stage = next_id;
    }
    h->level_need.assign(H, -1);
    int need = -1;
    for (int j = 0; j < H; ++j) {
      const int si = level_spec[j];
      if (si >= 0 && fresh_of[si] >= 0) need = std::max(need, fresh[fresh_of[si]].stage);
      h->level_need[j] = need;
    }
    if (trace) {
      fprintf(stderr, "[prepare] stages:");
      for (size_t i = 0; i < fresh.size(); ++i)
        fprintf(stderr, " (%d,%d)s%d:%.0f%%", fresh[i].n, fresh[i].k, fresh[i].stage, 100.0 * cost[i] / std::max<uint64_t>(total, 1));
      fprintf(stderr, "\n[prepare] level need:");
      for (int j = 0; j < H; ++j) fprintf(stderr, " %d", h->level_need[j]);
      fprintf(stderr, "\n");
    }
  }
  mark("specs");
  std::string err;
  lp_status s = build_hist_plan(fresh, h->rank, h->nranks, h->hp, err, h->num_sms);
  if (s != LP_OK) return fail(h, s, "%s", err.c_str());
  mark("histplan");
  // store slots of the fresh entries (appended; old slots of recomputed
  // ensembles are abandoned until the next eviction)
  h->store_off.assign(h->hp.entries.size(), 0);
  for (const PairDesc& pd : h->hp.pairs) {
    auto& slot = h->store_idx[{pd.n, pd.k}];  // one lookup per pair
    slot.count = pd.count;
    const int e0 = pd.entry_base, e1 = pd.entry_base + pd.n_entries;
    if (slot.ents.size() > 0) {  // a cached slot: drop the depths this plan does not refresh
      std::vector<uint8_t> fresh_p(pd.n + 2, 0);
      for (int e = e0; e < e1; ++e) fresh_p[h->hp.entries[e].P] = 1;
      std::vector<int> stale;
      for (const auto& [P, v] : slot.ents)
        if (P >= (int)fresh_p.size() || !fresh_p[P]) stale.push_back(P);
      for (int P : stale) slot.ents.erase(P);
    }
    for (int e = e0; e < e1; ++e) {
      const EntryDesc& E = h->hp.entries[e];
      h->store_off[e] = (int32_t)h->store_used;
      slot.ents[E.P] = {E.Dmax, (int)h->store_used};
      h->store_used += hist_row(E.Dmax + 1, pd.k);
    }
  }
  if (h->store_used > (size_t)INT32_MAX)
    return fail(h, LP_EUNSUPPORTED, "histogram store exceeds 2^31 probabilities");
  {
    lp_status gs = grow_store(h, h->store_used);
    if (gs != LP_OK) return gs;
  }
  mark("store");
  {
    size_t bytes = 0;
    lp_status us = upload_image(h,
                                {sec(h->hp.pairs, &h->off_pairs), sec(h->hp.entries, &h->off_entries),
                                 sec(h->hp.draws, &h->off_draws), sec(h->hp.binom, &h->off_binom),
                                 sec(h->hp.spans, &h->off_work), sec(h->hp.items, &h->off_items),
                                 sec(h->hp.divtab, &h->off_divtab),
                                 sec(h->hp.dmask, &h->off_dmask),
                                 sec(h->store_off, &h->off_store_off)},
                                h->tables, h->pin_up, h->ev_up[0], &bytes, h->stream);
    if (us != LP_OK) return us;
    h->up_bytes = bytes;
  }
  // work arena: histogram scratch and the DP state of every node
  const size_t nn = h->cfg.size();
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 255) & ~size_t(255);
    return r;
  };
  h->w_evt = take(4 * std::max<int64_t>(h->hp.evt_len, 1));
  h->w_h0 = take(4 * std::max<int64_t>(h->hp.h0_len, 1));
  h->w_hist = take(4 * std::max<int64_t>(h->hp.hist_len, 1));
  h->w_items = take(sizeof(WorkItem) * std::max<int64_t>(h->hp.n_work, 1));
  h->w_val = take(8 * nn);
  h->w_mig = take(8 * nn);
  h->w_par = take(4 * nn);
  h->w_stc = take(8 * nn);
  h->w_stm = take(8 * nn);
  h->w_plan = take(sizeof(lp_plan_step) * H);
  h->w_live = take(sizeof(lp_liveput_row) * std::max<size_t>(nn, 1));  // >= liveput rows
  h->w_final = take(8);
  h->w_bar = take(4);
  LP_CUDA(h, h->work.ensure(o));
  mark("upload1");
  std::memset(&h->stats, 0, sizeof h->stats);
  h->stats.resolutions = h->hp.resolutions;
  h->stats.scenarios = h->hp.scenarios;
  h->stats.local_scenarios = h->hp.local_scenarios;
  h->stats.mc_pairs = h->hp.mc_pairs;
  h->stats.exact_pairs = h->hp.exact_pairs;
  h->stats.horizon = H;
  h->stats.hist_alg_ops = h->hp.model_ops;
  h->stats.hist_survey_ops = h->hp.alg_ops;
  h->stats.cached_pairs = specs.size() - fresh.size();
  auto& ps = h->ps;
  ps.len = len;
  ps.n_seq.assign(n_seq, n_seq + len);
  ps.lbase = std::move(lbase);
  ps.lcount = std::move(lcount);
  ps.level_spec = std::move(level_spec);
  ps.specs = std::move(specs);
  ps.fresh = fresh.size();
  ps.host_ms = ms_since(t_start);
  return LP_OK;
}

// prepare, part 2: node rows, throughput / cost tables, liveput rows and the
// DP scalars; uploads the DP image.
lp_status prepare_dp(lp_handle* h) {
  const auto t_start = std::chrono::steady_clock::now();
  const bool trace = trace_prepare();
  auto mark = [&](const char* what) {
    if (trace) fprintf(stderr, "[prepare] %-10s %8.3f ms\n", what, ms_since(t_start));
  };
  const int H = h->horizon;
  const int32_t* n_seq = h->ps.n_seq.data();
  const std::vector<int>& lbase = h->ps.lbase;
  const std::vector<int>& lcount = h->ps.lcount;
  const std::vector<int>& level_spec = h->ps.level_spec;
  const std::vector<EnsembleSpec>& specs = h->ps.specs;
  // node histogram rows + levels
  std::map<int, int> thr_need;
  int pmax = 1;
  std::vector<int> entry_of_p;  // per pair: depth -> entry index
  std::vector<int> need_d;      // per depth: largest D read from the throughput table
  for (int j = 0; j < H; ++j) {
    LevelDesc& L = h->levels[j];
    L.n_now = n_seq[j];
    L.n_next = n_seq[j + 1];
    L.k = std::max(0, L.n_now - L.n_next);
    L.prev_base = lbase[j];
    L.prev_count = lcount[j];
    L.next_base = lbase[j + 1];
    L.next_count = lcount[j + 1];
    L.fresh = L.n_next > L.n_now ? 1 : 0;
    L.fixed = L.fresh ? h->cs.fresh_fixed : 0.0;
    L.has_hist = level_spec[j] >= 0;
    if (!L.has_hist) continue;
    const EnsembleSpec& spj = specs[level_spec[j]];
    const auto& slot = h->store_idx.at({spj.n, spj.k});
    L.total = slot.count;
    entry_of_p.assign(spj.n + 2, -1);
    for (const auto& [P, v] : slot.ents) entry_of_p[P] = v.second;  // store offset of D = 1
    for (int i = 0; i < lcount[j]; ++i) {
      NodeCfg& c = h->cfg[lbase[j] + i];
      if (c.d <= 0) continue;
      const int so = entry_of_p[c.p];
      if (so >= 0) c.hist_off = so + hist_row(c.d, L.k);
      if ((int)need_d.size() <= c.p) need_d.resize(c.p + 1, 0);
      need_d[c.p] = std::max(need_d[c.p], c.d);
    }
  }
  // next-role nodes: throughput(next) (and thr(alive, P) when strict) and
  // the per-depth cost terms
  for (int j = 1; j <= H; ++j)
    for (int i = 0; i < lcount[j]; ++i) {
      const NodeCfg& c = h->cfg[lbase[j] + i];
      if (c.d <= 0) continue;
      if ((int)need_d.size() <= c.p) need_d.resize(c.p + 1, 0);
      need_d[c.p] = std::max(need_d[c.p], c.d);
    }
  h->pcost.assign(need_d.size() + 1, make_double4(0.0, 0.0, 0.0, 0.0));
  for (int p = 1; p < (int)need_d.size(); ++p)
    if (need_d[p] > 0) {
      const NodeCost nc = node_cost(h, 1, p);
      h->pcost[p] = make_double4(nc.pipe, nc.unit, nc.resume, 0.0);
    }
  for (int p = 1; p < (int)need_d.size(); ++p)
    if (need_d[p] > 0) {
      thr_need[p] = need_d[p];
      pmax = std::max(pmax, p);
    }
  mark("nodes");
  build_thr(h->model, thr_need, pmax, h->thr);
  mark("thr");
  // liveput rows
  h->lrows.clear();
  for (int j = 0; j < H; ++j) {
    if (!h->levels[j].has_hist) continue;
    for (int i = 0; i < lcount[j]; ++i) {
      const int gi = lbase[j] + i;
      if (h->cfg[gi].d > 0 && h->cfg[gi].hist_off >= 0)
        h->lrows.push_back(make_int4(j, gi, (int)h->lrows.size(), 0));
    }
  }
  h->S = dp_scalars(h, H);
  mark("lrows");
  h->max_next = 0;
  for (const LevelDesc& L : h->levels) h->max_next = std::max(h->max_next, L.next_count);
  // shared-memory staged persistent DP (lp_dp.cu) when the whole DP input
  // fits in a block's shared memory next to 3 more blocks per SM
  h->dp_staged_nprob = -1;
  h->dp_cluster = false;
  if (h->dp_staged && H <= 64) {
    long long nprob = 0;
    for (int j = 0; j < H; ++j) {
      const LevelDesc& L = h->levels[j];
      if (L.has_hist) nprob += (long long)L.prev_count * (std::min(L.k, L.n_now) + 1);
    }
    const int n_nodes = h->levels[H - 1].next_base + h->levels[H - 1].next_count;
    if (nprob < (1 << 20) && dp_staged_smem(n_nodes, H, (int)nprob) <= (size_t)h->dp_staged_kb * 1024)
      h->dp_staged_nprob = (int)nprob;
    // the cluster DP (one 8-CTA cluster, DSMEM level values) for the smallest
    // re-plans; LIVEPUT_DP_CLUSTER=0 disables, LIVEPUT_DP_CLUSTER_MAXNEXT caps
    static const int cluster_max_next = [] {
      const char* e = getenv("LIVEPUT_DP_CLUSTER");
      if (e && e[0] == '0') return 0;
      const char* m = getenv("LIVEPUT_DP_CLUSTER_MAXNEXT");
      return m ? atoi(m) : 128;
    }();
    h->dp_cluster = h->dp_staged_nprob >= 0 && h->max_next <= cluster_max_next &&
                    dp_cluster_smem(n_nodes, H, (int)nprob, (int)h->pcost.size(), (int)h->thr.row.size(),
                                    (int)h->thr.vals.size()) <= 200 * 1024;
  }
  // cluster DP: the staged probability layout is built here, so the kernel
  // gathers its rows in one pass of independent loads
  h->dp_gather.clear();
  h->dp_pbase.clear();
  if (h->dp_cluster) {
    h->dp_gather.assign(std::max(h->dp_staged_nprob, 1), -1);
    h->dp_pbase.assign(H + 1, 0);
    int b = 0;
    for (int j = 0; j < H; ++j) {
      h->dp_pbase[j] = b;
      const LevelDesc& L = h->levels[j];
      if (!L.has_hist) continue;
      const int stride = std::min(L.k, L.n_now) + 1;
      for (int i = 0; i < L.prev_count; ++i) {
        const NodeCfg& c = h->cfg[L.prev_base + i];
        if (c.d > 0 && c.hist_off >= 0) {
          const int len = std::min(L.k, c.d) + 1;
          for (int d = 0; d < len; ++d) h->dp_gather[b + i * stride + d] = c.hist_off + d;
        }
      }
      b += L.prev_count * stride;
    }
    h->dp_pbase[H] = b;
  }
  // Materialised phi: a pipelined re-plan evaluates level j's pairs in the
  // phi launch of the stage that releases it, so the level chain left after
  // the sampling is max-plus passes only.  It pays when the sampling is
  // short against the DP: measured on one B200 -7% on the
  // forecast-like re-plan (sampling ops / DP pairs = 815), -5.5% and -1.6% on
  // the bench re-plan at 125K and 250K samples (1500, 3000), +0.6% at 1e6
  // (12000); under torchrun on 4 GPUs +0.3 to +1.3% in every stream-priority
  // variant, so multi-rank re-plans keep phi inside the levels.  Default:
  // one rank and ops / pairs < 4000.  LIVEPUT_PHI=0: never; 1: every
  // pipelined re-plan; <n> > 1: per-rank ensemble share <= n samples.
  // LIVEPUT_PHI_MAX_MB bounds the phi buffer (default 1024).
  {
    static const int64_t phi_max = [] {
      const char* e = getenv("LIVEPUT_PHI_MAX_MB");
      return (e ? atoll(e) : 1024LL) << 20;
    }();
    static const int64_t phi_mode = [] {  // -1: auto
      const char* e = getenv("LIVEPUT_PHI");
      return e ? (int64_t)strtoll(e, nullptr, 10) : (int64_t)-1;
    }();
    const int nst = (int)h->hp.stages.size();
    const bool persistent = nst <= 1 && !h->dp_launches && H <= kMaxHorizon;
    uint64_t local = 0;
    for (const PairDesc& pd : h->hp.pairs) local = std::max<uint64_t>(local, pd.t_hi - pd.t_lo);
    int64_t pairs = 0;
    for (int j = 0; j < H; ++j) pairs += (int64_t)h->levels[j].prev_count * h->levels[j].next_count;
    bool want;
    if (phi_mode < 0) want = h->nranks == 1 && (double)h->hp.model_ops < 4000.0 * (double)pairs;
    else if (phi_mode == 0) want = false;
    else if (phi_mode == 1) want = true;
    else want = local <= (uint64_t)phi_mode;
    h->phi_on = !persistent && want && pairs > 0 && pairs * 16 <= phi_max && pairs < (int64_t(1) << 31);
    h->phi_list.clear();
    const int ns = std::max(nst, 1);
    h->phi_range.assign(ns + 1, 0);
    h->phi_maxpairs.assign(ns, 0);
    if (h->phi_on) {
      int64_t o = 0;
      std::vector<std::vector<int32_t>> by_stage(ns);
      for (int j = 0; j < H; ++j) {
        LevelDesc& L = h->levels[j];
        L.phi_off = (int32_t)o;
        const int64_t np = (int64_t)L.prev_count * L.next_count;
        o += np;
        if (np == 0) continue;
        const int s = j < (int)h->level_need.size() ? std::max(0, std::min(h->level_need[j], ns - 1)) : ns - 1;
        by_stage[s].push_back(j);
        h->phi_maxpairs[s] = std::max<int64_t>(h->phi_maxpairs[s], L.prev_count);
      }
      for (int s = 0; s < ns; ++s) {
        h->phi_range[s] = (int)h->phi_list.size();
        h->phi_list.insert(h->phi_list.end(), by_stage[s].begin(), by_stage[s].end());
      }
      h->phi_range[ns] = (int)h->phi_list.size();
      LP_CUDA(h, h->phi.ensure((size_t)o * 16));
    }
  }
  size_t bytes = 0;
  lp_status us = upload_image(h,
                              {sec(h->levels, &h->off_levels), sec(h->cfg, &h->off_cfg),
                               sec(h->pcost, &h->off_cost), sec(h->lrows, &h->off_lrows),
                               sec(h->thr.vals, &h->off_thr), sec(h->thr.row, &h->off_throw),
                               sec(h->dp_gather, &h->off_gather), sec(h->dp_pbase, &h->off_pbase),
                               sec(h->phi_list, &h->off_phi_list)},
                              h->tables2, h->pin_up2, h->ev_up[1], &bytes, h->stream_dp);
  if (us != LP_OK) return us;
  mark("upload2");
  h->up_bytes += bytes;
  h->prepared = true;
  h->stats.h2d_bytes = h->up_bytes + sizeof(int32_t) * h->ps.len;
  h->ps.host_ms += ms_since(t_start);
  h->stats.prepare_ms = h->ps.host_ms;
  return LP_OK;
}

// execute, part 1: histogram kernels, the cross-rank sum, normalisation
// into the probability store.  Needs only prepare_hist's image.
bool hp_small(const lp_handle* h) { return !h->hp.items.empty(); }

lp_status exec_hist(lp_handle* h) {
  cudaStream_t st = h->stream;
  HistDev d{};
  d.pairs = dptr<PairDesc>(h->tables, h->off_pairs);
  d.entries = dptr<EntryDesc>(h->tables, h->off_entries);
  d.draws = dptr<DrawConst>(h->tables, h->off_draws);
  d.binom = dptr<uint64_t>(h->tables, h->off_binom);
  d.spans = dptr<WorkSpan>(h->tables, h->off_work);
  d.work = hp_small(h) ? dptr<WorkItem>(h->tables, h->off_items) : dptr<WorkItem>(h->work, h->w_items);
  d.divtab = dptr<uint16_t>(h->tables, h->off_divtab);
  d.dmask = dptr<uint32_t>(h->tables, h->off_dmask);
  {
    lp_status bs = bind_big_scratch(h, h->hp, d);
    if (bs != LP_OK) return bs;
  }
  d.evt = dptr<uint32_t>(h->work, h->w_evt);
  d.h0 = dptr<uint32_t>(h->work, h->w_h0);
  d.hist = dptr<uint32_t>(h->work, h->w_hist);
  const HistPlan& hp = h->hp;
  const int nst = (int)hp.stages.size();
  // one stage + persistent DP: the DP kernel normalises; otherwise each
  // stage is normalised here and its event releases the DP levels reading it
  const bool norm_here = nst > 1 || h->dp_launches || h->horizon > kMaxHorizon;
  int launches = 0;
  LP_CUDA(h, cudaEventRecord(h->ev[0], st));
  if (!hp_small(h)) {
    LP_CUDA(h, launch_expand_work(d.spans, (int)hp.spans.size(), (int)hp.n_work, d.work, st));
    if (hp.n_work > 0) ++launches;
  }
  if (hp.evt_len > 0) LP_CUDA(h, cudaMemsetAsync(d.evt, 0, sizeof(uint32_t) * hp.evt_len, st));
  LP_CUDA(h, cudaMemsetAsync(d.h0, 0, sizeof(uint32_t) * std::max<int64_t>(hp.h0_len, 1), st));
  // The stages' histogram kernels go out at once, each on its own stream,
  // so a stage's tail is filled by the next stage's blocks (the scheduler
  // favours the earlier launch); finalise / reduce / normalise follow in
  // stage order on the handle's stream.
  if (nst > 1) {
    LP_CUDA(h, cudaEventRecord(h->ev_start, st));
    for (int s = 0; s < nst; ++s) {
      LP_CUDA(h, cudaStreamWaitEvent(h->stream_hist[s], h->ev_start, 0));
      LP_CUDA(h, run_hist_stage(hp, d, h->stream_hist[s], s, &launches));
      LP_CUDA(h, cudaEventRecord(h->ev_hist[s], h->stream_hist[s]));
    }
  }
  for (int s = 0; s < nst; ++s) {
    const HistPlan::Stage& S = hp.stages[s];
    if (nst > 1) LP_CUDA(h, cudaStreamWaitEvent(st, h->ev_hist[s], 0));
    else LP_CUDA(h, run_hist_stage(hp, d, st, s, &launches));
    LP_CUDA(h, launch_finalize_range(S.p0, S.p1 - S.p0, S.e0, S.e1 - S.e0, st, d.pairs, d.entries, d.evt,
                                     d.h0, d.hist));
    if (S.p1 > S.p0) launches += 2;
    if (s == nst - 1) LP_CUDA(h, cudaEventRecord(h->ev[1], st));
    if (h->nranks > 1 && S.h1 > S.h0) {
      ncclResult_t r = nccl().AllReduce(d.hist + S.h0, d.hist + S.h0, (size_t)(S.h1 - S.h0), ncclUint32,
                                        ncclSum, h->comm, st);
      if (r != ncclSuccess) return fail(h, LP_ENCCL, "ncclAllReduce: %s", nccl().GetErrorString(r));
    }
    if (norm_here && S.e1 > S.e0) {
      LP_CUDA(h, launch_normalize(S.e1 - S.e0, st, d.pairs, d.entries + S.e0, d.hist,
                                  dptr<int32_t>(h->tables, h->off_store_off) + S.e0,
                                  static_cast<double*>(h->store.p)));
      ++launches;
    }
    LP_CUDA(h, cudaEventRecord(h->ev_stage[s], st));
  }
  if (nst == 0) LP_CUDA(h, cudaEventRecord(h->ev[1], st));
  LP_CUDA(h, cudaEventRecord(h->ev[2], st));
  h->stats.kernel_launches = launches;
  return LP_OK;
}

// execute, part 2: the lookahead DP and traceback, on the DP stream.  Level
// j waits only for the stage holding the histograms it reads, so the DP of
// the early intervals overlaps the sampling of the later ones; the DP
// stream is joined back into the handle's stream at the end.

lp_status exec_dp(lp_handle* h) {
  cudaStream_t st = h->stream_dp;
  int launches = 0;
  const LevelDesc* lv = dptr<LevelDesc>(h->tables2, h->off_levels);
  const NodeCfg* cfg = dptr<NodeCfg>(h->tables2, h->off_cfg);
  const double4* pcost = dptr<double4>(h->tables2, h->off_cost);
  const double* thr = dptr<double>(h->tables2, h->off_thr);
  const int32_t* throw_ = dptr<int32_t>(h->tables2, h->off_throw);
  double* val = dptr<double>(h->work, h->w_val);
  double* mig = dptr<double>(h->work, h->w_mig);
  int32_t* par = dptr<int32_t>(h->work, h->w_par);
  double* stc = dptr<double>(h->work, h->w_stc);
  double* stm = dptr<double>(h->work, h->w_stm);
  double* histp = static_cast<double*>(h->store.p);
  const int nst = (int)h->hp.stages.size();
  const bool persistent = nst <= 1 && !h->dp_launches && h->horizon <= kMaxHorizon;
  if (persistent) {
    if (nst == 1) LP_CUDA(h, cudaStreamWaitEvent(st, h->ev_stage[0], 0));
    DpArgs a{};
    a.levels = lv;
    a.cfg = cfg;
    a.pcost = pcost;
    a.thr_tab = thr;
    a.thr_row = throw_;
    a.pairs = dptr<PairDesc>(h->tables, h->off_pairs);
    a.entries = dptr<EntryDesc>(h->tables, h->off_entries);
    a.hist = dptr<uint32_t>(h->work, h->w_hist);
    a.store_off = dptr<int32_t>(h->tables, h->off_store_off);
    a.n_entries = (int)h->hp.entries.size();
    a.store = histp;
    a.val = val;
    a.mig = mig;
    a.parent = par;
    a.stc = stc;
    a.stm = stm;
    a.plan = dptr<lp_plan_step>(h->work, h->w_plan);
    a.final_value = dptr<double>(h->work, h->w_final);
    a.barrier = dptr<uint32_t>(h->work, h->w_bar);
    a.horizon = h->horizon;
    a.max_next = std::max(1, h->max_next);
    a.gather = h->dp_cluster ? dptr<int32_t>(h->tables2, h->off_gather) : nullptr;
    a.pbase = h->dp_cluster ? dptr<int32_t>(h->tables2, h->off_pbase) : nullptr;
    static const bool trace = getenv("LIVEPUT_DP_TRACE") != nullptr;
    if (trace) {
      const size_t nb = (size_t)h->num_sms * 8 * (2 * kTraceLevels + 2);
      LP_CUDA(h, h->dp_trace.ensure(nb * 8));
      LP_CUDA(h, cudaMemsetAsync(h->dp_trace.p, 0, nb * 8, st));
      a.trace = static_cast<uint64_t*>(h->dp_trace.p);
    }
    const LevelDesc& last = h->levels[h->horizon - 1];
    if (h->dp_cluster)
      LP_CUDA(h, launch_dp_cluster(st, a, h->S, last.next_base + last.next_count, h->dp_staged_nprob,
                                   (int)h->pcost.size(), (int)h->thr.row.size(), (int)h->thr.vals.size()));
    else
      LP_CUDA(h, launch_dp_persistent(h->device, h->num_sms, h->max_next, st, a, h->S,
                                      last.next_base + last.next_count, h->dp_staged_nprob));
    ++launches;
  } else {
    LP_CUDA(h, cudaMemsetAsync(val, 0, 8, st));  // level 0: value 0, migration 0
    LP_CUDA(h, cudaMemsetAsync(mig, 0, 8, st));
    if (h->phi_on) {
      // phi of the levels each stage releases, on the phi stream (highest
      // priority), as soon as that stage's probabilities are in the store
      double2* phi = static_cast<double2*>(h->phi.p);
      const int32_t* lv_list = dptr<int32_t>(h->tables2, h->off_phi_list);
      const int ns = (int)h->phi_maxpairs.size();
      LP_CUDA(h, cudaStreamWaitEvent(h->stream_phi, h->ev_up[1], 0));  // the DP image
      // one phi launch per stage, except that the last stage's levels get a
      // launch and an event each, so the chain left after the sampling starts
      // on its first level's pairs.  LIVEPUT_PHI_LEVELS=1: per-level launches
      // and events for every stage (measured slower: a cross-stream wait per
      // level costs more than the earlier start saves)
      static const bool phi_per_level = [] {
        const char* e = getenv("LIVEPUT_PHI_LEVELS");
        return e && e[0] == '1';
      }();
      while ((int)h->ev_lvl.size() < h->horizon) {
        cudaEvent_t e;
        LP_CUDA(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->ev_lvl.push_back(e);
      }
      for (int s = 0; s < ns; ++s) {
        if (s < nst) LP_CUDA(h, cudaStreamWaitEvent(h->stream_phi, h->ev_stage[s], 0));
        const int a = h->phi_range[s], b = h->phi_range[s + 1];
        if (!phi_per_level && s < ns - 1) {
          LP_CUDA(h, launch_phi_matrix(b - a, h->phi_maxpairs[s], h->stream_phi, lv_list + a, lv, cfg, pcost, histp,
                                       thr, throw_, h->S, phi));
          if (b > a) ++launches;
          LP_CUDA(h, cudaEventRecord(h->ev_phi[s], h->stream_phi));
          continue;
        }
        for (int q = a; q < b; ++q) {
          const int j = h->phi_list[q];
          LP_CUDA(h, launch_phi_matrix(1, h->levels[j].prev_count, h->stream_phi, lv_list + q, lv, cfg, pcost, histp,
                                       thr, throw_, h->S, phi));
          ++launches;
          LP_CUDA(h, cudaEventRecord(h->ev_lvl[j], h->stream_phi));
        }
        LP_CUDA(h, cudaEventRecord(h->ev_phi[s], h->stream_phi));
      }
      static const bool pdl_on = [] {
        const char* e = getenv("LIVEPUT_PDL");
        return !(e && e[0] == '0');
      }();
      // the max-plus levels, PDL-chained while they follow a stage event;
      // the last stage's levels each wait for their own phi launch
      int waited = -1;
      for (int j = 0; j < h->horizon; ++j) {
        int need = j < (int)h->level_need.size() ? h->level_need[j] : ns - 1;
        need = std::max(0, std::min(need, ns - 1));
        bool pdl = pdl_on && j > 0;
        if ((phi_per_level || need == ns - 1) && h->levels[j].prev_count > 0 && h->levels[j].next_count > 0) {
          LP_CUDA(h, cudaStreamWaitEvent(st, h->ev_lvl[j], 0));
          pdl = false;
        } else if (need > waited) {
          LP_CUDA(h, cudaStreamWaitEvent(st, h->ev_phi[need], 0));
          waited = need;
          pdl = false;
        }
        LP_CUDA(h, launch_dp_maxplus(j, h->levels[j].next_count, pdl, st, lv, phi, val, mig, par, stc, stm));
        ++launches;
        if (timeline()) {
          while ((int)h->tl_ev.size() <= j) {
            cudaEvent_t e;
            LP_CUDA(h, cudaEventCreate(&e));
            h->tl_ev.push_back(e);
          }
          LP_CUDA(h, cudaEventRecord(h->tl_ev[j], st));
        }
      }
      LP_CUDA(h, cudaStreamWaitEvent(st, h->ev_phi[ns - 1], 0));
      const LevelDesc& last = h->levels[h->horizon - 1];
      LP_CUDA(h, launch_dp_final(h->horizon, st, lv, cfg, val, mig, par, stc, stm,
                                 dptr<lp_plan_step>(h->work, h->w_plan), dptr<double>(h->work, h->w_final),
                                 last.next_base + last.next_count));
      ++launches;
    } else {
      int waited = -1;
      static const bool pdl_on = [] {  // LIVEPUT_PDL=0: plain stream order between levels (A/B)
        const char* e = getenv("LIVEPUT_PDL");
        return !(e && e[0] == '0');
      }();
      for (int j = 0; j < h->horizon; ++j) {
        const int need = j < (int)h->level_need.size() ? h->level_need[j] : nst - 1;
        bool pdl = pdl_on && j > 0;  // right after a cross-stream wait: plain order
        if (need > waited) {
          LP_CUDA(h, cudaStreamWaitEvent(st, h->ev_stage[need], 0));
          waited = need;
          pdl = false;
        }
        LP_CUDA(h, launch_dp_step(j, h->levels[j].next_count, h->levels[j].prev_count, pdl, st, lv, cfg, pcost,
                                  histp, thr, throw_, h->S, val, mig, par, stc, stm));
        ++launches;
        if (timeline()) {
          while ((int)h->tl_ev.size() <= j) {
            cudaEvent_t e;
            LP_CUDA(h, cudaEventCreate(&e));
            h->tl_ev.push_back(e);
          }
          LP_CUDA(h, cudaEventRecord(h->tl_ev[j], st));
        }
      }
      const LevelDesc& last = h->levels[h->horizon - 1];
      LP_CUDA(h, launch_dp_final(h->horizon, st, lv, cfg, val, mig, par, stc, stm,
                                 dptr<lp_plan_step>(h->work, h->w_plan), dptr<double>(h->work, h->w_final),
                                 last.next_base + last.next_count));
      ++launches;
    }
  }
  // every stage has landed in the store before the handle's stream moves on
  if (nst > 0) LP_CUDA(h, cudaStreamWaitEvent(st, h->ev_stage[nst - 1], 0));
  LP_CUDA(h, cudaEventRecord(h->ev[3], st));
  LP_CUDA(h, cudaEventRecord(h->ev_join, st));
  LP_CUDA(h, cudaStreamWaitEvent(h->stream, h->ev_join, 0));
  h->live_pending = !h->lrows.empty();  // the liveput table is built on demand (lp_fetch)
  h->stats.kernel_launches += launches;
  return LP_OK;
}

// Liveput table rows of the last execute, Σ_m p_m·thr(m, P) per (interval,
// prev config); launched only when a caller asks for them.
lp_status exec_liveput(lp_handle* h) {
  if (!h->live_pending) return LP_OK;
  LP_CUDA(h, launch_liveput((int)h->lrows.size(), h->stream, dptr<int4>(h->tables2, h->off_lrows),
                            dptr<LevelDesc>(h->tables2, h->off_levels),
                            dptr<NodeCfg>(h->tables2, h->off_cfg), nullptr,
                            static_cast<double*>(h->store.p), dptr<double>(h->tables2, h->off_thr),
                            dptr<int32_t>(h->tables2, h->off_throw),
                            dptr<lp_liveput_row>(h->work, h->w_live)));
  h->live_pending = false;
  ++h->stats.kernel_launches;
  return LP_OK;
}

}  // namespace

extern "C" {

lp_status lp_prepare(lp_handle* h, lp_config current, const int32_t* n_seq, int32_t len) {
  lp_status s = prepare_hist(h, current, n_seq, len);
  return s != LP_OK ? s : prepare_dp(h);
}

lp_status lp_execute(lp_handle* h) {
  if (!h) return fail(nullptr, LP_EINVAL, "null handle");
  if (!h->prepared) return fail(h, LP_EINVAL, "lp_execute: call lp_prepare first");
  cudaSetDevice(h->device);
  lp_status s = exec_hist(h);
  return s != LP_OK ? s : exec_dp(h);
}

lp_status lp_fetch(lp_handle* h, lp_plan_step* out, lp_liveput_row* live, int32_t cap,
                   int32_t* rows) {
  if (!h || !out) return fail(h, LP_EINVAL, "lp_fetch: null argument");
  if (!h->prepared) return fail(h, LP_EINVAL, "lp_fetch: nothing prepared");
  cudaSetDevice(h->device);
  const size_t plan_b = sizeof(lp_plan_step) * h->horizon;
  const size_t nl = live ? std::min<size_t>(h->lrows.size(), (size_t)std::max(cap, 0)) : 0;
  const size_t live_b = sizeof(lp_liveput_row) * nl;
  if (live_b) {
    lp_status ls = exec_liveput(h);
    if (ls != LP_OK) return ls;
  }
  LP_CUDA(h, h->pin_down.ensure(plan_b + live_b + 64));
  unsigned char* pd = static_cast<unsigned char*>(h->pin_down.p);
  LP_CUDA(h, cudaMemcpyAsync(pd, dptr<void>(h->work, h->w_plan), plan_b, cudaMemcpyDeviceToHost,
                             h->stream));
  if (live_b)
    LP_CUDA(h, cudaMemcpyAsync(pd + plan_b, dptr<void>(h->work, h->w_live), live_b,
                               cudaMemcpyDeviceToHost, h->stream));
  LP_CUDA(h, cudaStreamSynchronize(h->stream));
  if (h->dp_trace.p && getenv("LIVEPUT_DP_TRACE")) {  // debug: per-level block timing
    const int per = 2 * kTraceLevels + 2;
    const size_t nb = (size_t)h->num_sms * 8;
    std::vector<uint64_t> tr(nb * per);
    cudaMemcpy(tr.data(), h->dp_trace.p, tr.size() * 8, cudaMemcpyDeviceToHost);
    int used = 0;
    while ((size_t)used < nb && tr[(size_t)used * per] != 0) ++used;
    if (used > 0 && tr[1] && tr[0])
      fprintf(stderr, "[dp] block 0: start -> first level %.2f us, kernel span %.2f us\n",
              (double)(tr[1] - tr[0]) * 1e-3,
              (double)(tr[3 + 2 * (std::min(h->horizon, kTraceLevels) - 1)] - tr[0]) * 1e-3);
    for (int j = 1; j < std::min(h->horizon, kTraceLevels); ++j) {
      uint64_t smin = UINT64_MAX, emax = 0;
      std::vector<double> comp;
      for (int b = 0; b < used; ++b) {
        const uint64_t s0 = tr[(size_t)b * per + 3 + 2 * (j - 1)], c = tr[(size_t)b * per + 2 + 2 * j],
                       e = tr[(size_t)b * per + 3 + 2 * j];
        if (s0 == 0 || e == 0) {  // left after the normalisation barrier
          comp.push_back(0.0);
          continue;
        }
        smin = std::min(smin, s0);
        emax = std::max(emax, e);
        comp.push_back((double)(c - s0) * 1e-3);
      }
      std::vector<std::pair<double, int>> bycomp;
      for (int b = 0; b < used; ++b) bycomp.push_back({comp[b], b});
      std::sort(comp.begin(), comp.end());
      std::sort(bycomp.rbegin(), bycomp.rend());
      fprintf(stderr, "[dp] level %2d: %7.2f us; block compute median %6.2f max %6.2f us (%d blocks) slowest:", j,
              (double)(emax - smin) * 1e-3, comp[comp.size() / 2], comp.back(), used);
      const LevelDesc& L = h->levels[j];
      for (int q = 0; q < 6 && q < (int)bycomp.size(); ++q) {
        const int b = bycomp[q].second;
        if (b < L.next_count) {
          const NodeCfg& c = h->cfg[L.next_base + b];
          fprintf(stderr, " (%d,%d)%.1f", c.d, c.p, bycomp[q].first);
        }
      }
      fprintf(stderr, "  fastest: (%d)%.1f\n", bycomp.back().second, bycomp.back().first);
    }
  }
  std::memcpy(out, pd, plan_b);
  if (live_b) std::memcpy(live, pd + plan_b, live_b);
  if (rows) *rows = (int32_t)h->lrows.size();
  h->stats.d2h_bytes = plan_b + live_b;
  return LP_OK;
}

lp_status lp_replan(lp_handle* h, lp_config current, const int32_t* n_seq, int32_t len,
                    lp_plan_step* out, lp_liveput_row* live, int32_t cap, int32_t* rows) {
  // The histogram kernels are launched before the DP tables are built, so
  // the host half of the preparation runs under the device's histogram time.
  lp_status s = prepare_hist(h, current, n_seq, len);
  if (s == LP_OK) s = exec_hist(h);
  if (s == LP_OK) s = prepare_dp(h);
  if (s == LP_OK) s = exec_dp(h);
  if (s != LP_OK) return s;
  return lp_fetch(h, out, live, cap, rows);
}

lp_status lp_set_hist_cache(lp_handle* h, int32_t enable, uint64_t max_bytes) {
  if (!h) return fail(nullptr, LP_EINVAL, "null handle");
  h->cache_on = enable != 0;
  // store offsets are int32 element indices (EntryDesc / store_off)
  h->cache_max = std::min<uint64_t>(max_bytes ? max_bytes : (4ull << 30), (uint64_t)INT32_MAX * 8ull);
  h->store_idx.clear();
  h->store_used = 0;
  h->prepared = false;
  return LP_OK;
}

// Offline tables: each (n, k) is staged through a one-interval re-plan
// [n, n, n - k] from suspension, whose level 1 needs every config of n at k.
lp_status lp_precompute(lp_handle* h, const int32_t* ns, const int32_t* ks, int32_t count) {
  if (!h || (count > 0 && (!ns || !ks))) return fail(h, LP_EINVAL, "lp_precompute: bad argument");
  if (!h->cache_on) {
    h->cache_on = true;
    h->store_idx.clear();
    h->store_used = 0;
  }
  for (int i = 0; i < count; ++i) {
    if (ns[i] < 0 || ks[i] < 0 || ks[i] > ns[i])
      return fail(h, LP_EINVAL, "lp_precompute: need 0 <= k <= n (got n=%d k=%d)", ns[i], ks[i]);
    const int32_t seq[3] = {ns[i], ns[i], ns[i] - ks[i]};
    lp_status s = lp_prepare(h, lp_config{0, 0}, seq, 3);
    if (s != LP_OK) return s;
    s = lp_execute(h);
    if (s != LP_OK) return s;
  }
  LP_CUDA(h, cudaStreamSynchronize(h->stream));
  h->prepared = false;
  return LP_OK;
}

namespace {
constexpr uint32_t kCacheMagic = 0x3143504cu;  // "LPC1"
struct CacheHeader {
  uint32_t magic;
  int32_t mc_trials;
  uint64_t exact_cap;
  uint64_t mc_seed;
  uint64_t slots;
};
struct SlotHeader {
  int32_t n, k;
  uint64_t count;
  int32_t entries, pad;
};
struct EntryHeader {
  int32_t P, Dmax;
  int64_t len;
};
}  // namespace

// Serialises the device histogram store: probabilities depend only on
// (n, k) and the sampling options, never on the profile or costs.
lp_status lp_cache_export(lp_handle* h, void* buf, uint64_t cap, uint64_t* len) {
  if (!h || !len) return fail(h, LP_EINVAL, "lp_cache_export: bad argument");
  uint64_t need = sizeof(CacheHeader);
  for (const auto& [key, slot] : h->store_idx) {
    need += sizeof(SlotHeader);
    for (const auto& [P, v] : slot.ents)
      need += sizeof(EntryHeader) + sizeof(double) * hist_row(v.first + 1, key.second);
  }
  *len = need;
  if (!buf) return LP_OK;
  if (cap < need) return fail(h, LP_EINVAL, "lp_cache_export: buffer of %llu bytes, need %llu",
                              (unsigned long long)cap, (unsigned long long)need);
  cudaSetDevice(h->device);
  LP_CUDA(h, cudaStreamSynchronize(h->stream));
  unsigned char* o = static_cast<unsigned char*>(buf);
  CacheHeader ch{kCacheMagic, h->opt.mc_trials, h->opt.exact_cap, h->opt.mc_seed,
                 (uint64_t)h->store_idx.size()};
  std::memcpy(o, &ch, sizeof ch);
  o += sizeof ch;
  for (const auto& [key, slot] : h->store_idx) {
    SlotHeader sh{key.first, key.second, slot.count, (int32_t)slot.ents.size(), 0};
    std::memcpy(o, &sh, sizeof sh);
    o += sizeof sh;
    for (const auto& [P, v] : slot.ents) {
      const int64_t rows = hist_row(v.first + 1, key.second);
      EntryHeader eh{P, v.first, rows};
      std::memcpy(o, &eh, sizeof eh);
      o += sizeof eh;
      LP_CUDA(h, cudaMemcpy(o, static_cast<double*>(h->store.p) + v.second, sizeof(double) * rows,
                            cudaMemcpyDeviceToHost));
      o += sizeof(double) * rows;
    }
  }
  return LP_OK;
}

lp_status lp_cache_import(lp_handle* h, const void* buf, uint64_t len) {
  if (!h || !buf || len < sizeof(CacheHeader)) return fail(h, LP_EINVAL, "lp_cache_import: bad buffer");
  const unsigned char* p = static_cast<const unsigned char*>(buf);
  const unsigned char* end = p + len;
  CacheHeader ch;
  std::memcpy(&ch, p, sizeof ch);
  p += sizeof ch;
  if (ch.magic != kCacheMagic) return fail(h, LP_EINVAL, "lp_cache_import: not a liveput table");
  if (ch.mc_trials != h->opt.mc_trials || ch.exact_cap != h->opt.exact_cap ||
      ch.mc_seed != h->opt.mc_seed)
    return fail(h, LP_EINVAL, "lp_cache_import: table was sampled with different PlannerOptions "
                              "(mc_trials/exact_cap/mc_seed)");
  cudaSetDevice(h->device);
  h->cache_on = true;
  for (uint64_t s = 0; s < ch.slots; ++s) {
    if (p + sizeof(SlotHeader) > end) return fail(h, LP_EINVAL, "lp_cache_import: truncated");
    SlotHeader sh;
    std::memcpy(&sh, p, sizeof sh);
    p += sizeof sh;
    auto& slot = h->store_idx[{sh.n, sh.k}];
    slot.count = sh.count;
    for (int e = 0; e < sh.entries; ++e) {
      if (p + sizeof(EntryHeader) > end) return fail(h, LP_EINVAL, "lp_cache_import: truncated");
      EntryHeader eh;
      std::memcpy(&eh, p, sizeof eh);
      p += sizeof eh;
      if (eh.len != hist_row(eh.Dmax + 1, sh.k) || p + sizeof(double) * eh.len > end)
        return fail(h, LP_EINVAL, "lp_cache_import: corrupt entry");
      if (h->store_used + eh.len > (size_t)INT32_MAX)
        return fail(h, LP_EUNSUPPORTED, "lp_cache_import: table exceeds 2^31 probabilities");
      lp_status gs = grow_store(h, h->store_used + eh.len);
      if (gs != LP_OK) return gs;
      LP_CUDA(h, cudaMemcpy(static_cast<double*>(h->store.p) + h->store_used, p,
                            sizeof(double) * eh.len, cudaMemcpyHostToDevice));
      slot.ents[eh.P] = {eh.Dmax, (int)h->store_used};
      h->store_used += eh.len;
      p += sizeof(double) * eh.len;
    }
  }
  h->prepared = false;
  return LP_OK;
}

lp_status lp_get_stats(const lp_handle* hc, lp_stats* out) {
  lp_handle* h = const_cast<lp_handle*>(hc);
  if (!h || !out) return fail(h, LP_EINVAL, "null argument");
  if (h->prepared && h->stats.kernel_launches > 0) {
    cudaSetDevice(h->device);
    LP_CUDA(h, cudaStreamSynchronize(h->stream));
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, h->ev[0], h->ev[1]);
    cudaEventElapsedTime(&b, h->ev[1], h->ev[2]);
    cudaEventElapsedTime(&c, h->ev[2], h->ev[3]);
    h->stats.hist_ms = a;
    h->stats.reduce_ms = b;
    h->stats.dp_ms = c;
    h->stats.total_ms = (double)a + b + c;
    if (timeline()) {
      auto rel = [&](cudaEvent_t e) {
        float t = -1.f;
        cudaEventElapsedTime(&t, h->ev[0], e);
        return t;
      };
      const int nst = (int)h->hp.stages.size();
      fprintf(stderr, "[timeline] rank %d:", h->rank);
      for (int q = 0; q < nst && nst > 1; ++q)
        fprintf(stderr, " s%d hist %.3f norm %.3f |", q, rel(h->ev_hist[q]), rel(h->ev_stage[q]));
      for (int j = 0; j < (int)h->tl_ev.size() && j < h->horizon; ++j)
        fprintf(stderr, " L%d(%d) %.3f", j, j < (int)h->level_need.size() ? h->level_need[j] : -1, rel(h->tl_ev[j]));
      fprintf(stderr, " | end %.3f\n", rel(h->ev[3]));
    }
  }
  *out = h->stats;
  return LP_OK;
}

// ---------------------------------------------------------------------------
lp_status lp_phi(lp_handle* h, lp_config prev, lp_config next, int32_t n_now, int32_t n_next,
                 double* committed, double* mig) {
  if (!h || !committed || !mig) return fail(h, LP_EINVAL, "lp_phi: null argument");
  cudaSetDevice(h->device);
  NodeCfg pv{prev.pipelines > 0 ? prev.pipelines : 0, prev.pipelines > 0 ? prev.stages : 0, 0, 0};
  NodeCfg nx{next.pipelines > 0 ? next.pipelines : 0, next.pipelines > 0 ? next.stages : 0, 0, 0};
  // optimizer.cpp:99-101: suspended / infeasible / oversized next -> {0, 0}
  if (nx.d <= 0 || !h->model.depth_ok(nx.p) || (long long)nx.d * nx.p > n_next) {
    *committed = 0.0;
    *mig = 0.0;
    return LP_OK;
  }
  LevelDesc L{};
  L.n_now = n_now;
  L.n_next = n_next;
  L.k = std::max(0, n_now - n_next);
  L.fresh = n_next > n_now;
  L.fixed = L.fresh ? h->cs.fresh_fixed : 0.0;
  std::vector<uint32_t> rows(1, 0);
  if (pv.d > 0) {
    if (pv.p < 1 || (long long)pv.d * pv.p > n_now)
      return fail(h, LP_EINVAL, "phi: prev config exceeds n_now");
    uint64_t total = 0;
    lp_status s = planner_rows(h, pv.d, pv.p, n_now, L.k, rows, &total);
    if (s != LP_OK) return s;
    L.total = total;
  }
  std::map<int, int> need;
  need[nx.p] = nx.d;
  ThrTable t;
  build_thr(h->model, need, nx.p, t);
  Packer pk;
  const size_t oh = pk.add(rows), ot = pk.add(t.vals), orow = pk.add(t.row);
  const size_t oout = pk.add(nullptr, 16);
  LP_CUDA(h, h->e_tables.ensure(pk.bytes.size()));
  LP_CUDA(h, h->pin_up.ensure(pk.bytes.size()));
  std::memcpy(h->pin_up.p, pk.bytes.data(), pk.bytes.size());
  LP_CUDA(h, cudaMemcpyAsync(h->e_tables.p, h->pin_up.p, pk.bytes.size(), cudaMemcpyHostToDevice,
                             h->stream));
  pv.hist_off = 0;
  const NodeCost nc = node_cost(h, nx.d, nx.p);
  const DpScalars S = dp_scalars(h, 1);
  LP_CUDA(h, launch_phi_single(pv, nx, nc, L, S, dptr<uint32_t>(h->e_tables, oh),
                               dptr<double>(h->e_tables, ot), dptr<int32_t>(h->e_tables, orow),
                               dptr<double>(h->e_tables, oout), h->stream));
  LP_CUDA(h, h->pin_down.ensure(16));
  LP_CUDA(h, cudaMemcpyAsync(h->pin_down.p, dptr<double>(h->e_tables, oout), 16,
                             cudaMemcpyDeviceToHost, h->stream));
  LP_CUDA(h, cudaStreamSynchronize(h->stream));
  const double* r = static_cast<const double*>(h->pin_down.p);
  *committed = r[0];
  *mig = r[1];
  return LP_OK;
}

lp_status lp_sequence_value(lp_handle* h, lp_config current, const lp_config* seq,
                            const int32_t* n_seq, int32_t len, double* out) {
  if (!h || !out || !n_seq) return fail(h, LP_EINVAL, "null argument");
  if (len < 1 || (len > 1 && !seq))
    return fail(h, LP_EINVAL, "sequence_value: sequence/N length mismatch");
  double value = 0.0;
  lp_config prev = current;
  for (int j = 0; j + 1 < len; ++j) {
    double c = 0, m = 0;
    lp_status s = lp_phi(h, prev, seq[j], n_seq[j], n_seq[j + 1], &c, &m);
    if (s != LP_OK) return s;
    value += c;
    prev = seq[j];
  }
  *out = value;
  return LP_OK;
}

lp_status lp_survivor_hist(lp_handle* h, lp_config prev, int32_t n_now, int32_t n_minus,
                           uint64_t* counts, uint64_t* total) {
  if (!h || !counts || !total) return fail(h, LP_EINVAL, "null argument");
  if (prev.pipelines < 1 || prev.stages < 1 || (long long)prev.pipelines * prev.stages > n_now)
    return fail(h, LP_EINVAL, "survivor_hist: config exceeds n_now");
  cudaSetDevice(h->device);
  std::vector<uint32_t> rows;
  lp_status s = planner_rows(h, prev.pipelines, prev.stages, n_now, n_minus, rows, total);
  if (s != LP_OK) return s;
  for (int m = 0; m <= prev.pipelines; ++m) counts[m] = 0;
  for (size_t d = 0; d < rows.size(); ++d) counts[prev.pipelines - (int)d] = rows[d];
  return LP_OK;
}

lp_status lp_expected_liveput(lp_handle* h, lp_config cfg, int32_t n, int32_t n_minus,
                              int32_t exact, int32_t trials, uint64_t seed, double* out) {
  if (!h || !out) return fail(h, LP_EINVAL, "null argument");
  if ((long long)cfg.pipelines * cfg.stages > n)
    return fail(h, LP_EINVAL, "expected_liveput: config exceeds n");
  if (n_minus < 0 || n_minus > n) return fail(h, LP_EINVAL, "sample_vectors: bad n_minus");
  if (cfg.pipelines < 1 || cfg.stages < 1) return fail(h, LP_EINVAL, "expected_liveput: empty config");
  cudaSetDevice(h->device);
  EnsembleSpec sp;
  sp.n = n;
  sp.k = n_minus;
  sp.exact = exact != 0;
  if (sp.exact) {
    sp.count = scenario_count(n, n_minus);
    if (sp.count > kEnumerationCap)
      return fail(h, LP_EINVAL, "enumerate_vectors: scenario space too large, sample instead");
  } else {
    if (trials < 1) return fail(h, LP_EINVAL, "sample_vectors: trials must be >= 1");
    sp.count = (uint64_t)trials;
  }
  sp.seed = seed;
  sp.dmax_by_p[cfg.stages] = cfg.pipelines;
  std::vector<uint32_t> rows;
  lp_status s = ensemble_rows(h, sp, cfg.pipelines, cfg.stages, rows);
  if (s != LP_OK) return s;
  // device liveput of the single row
  std::map<int, int> need;
  need[cfg.stages] = cfg.pipelines;
  ThrTable t;
  build_thr(h->model, need, cfg.stages, t);
  LevelDesc L{};
  L.k = n_minus;
  L.total = sp.count;
  NodeCfg c{cfg.pipelines, cfg.stages, 0, 0};
  int4 row = make_int4(0, 0, 0, 0);
  Packer pk;
  const size_t oh = pk.add(rows), ot = pk.add(t.vals), orow = pk.add(t.row);
  const size_t ol = pk.add(&L, sizeof L), oc = pk.add(&c, sizeof c), orw = pk.add(&row, sizeof row);
  const size_t oout = pk.add(nullptr, sizeof(lp_liveput_row));
  LP_CUDA(h, h->e_tables.ensure(pk.bytes.size()));
  LP_CUDA(h, h->pin_up.ensure(pk.bytes.size()));
  std::memcpy(h->pin_up.p, pk.bytes.data(), pk.bytes.size());
  LP_CUDA(h, cudaMemcpyAsync(h->e_tables.p, h->pin_up.p, pk.bytes.size(), cudaMemcpyHostToDevice,
                             h->stream));
  LP_CUDA(h, launch_liveput(1, h->stream, dptr<int4>(h->e_tables, orw),
                            dptr<LevelDesc>(h->e_tables, ol), dptr<NodeCfg>(h->e_tables, oc),
                            dptr<uint32_t>(h->e_tables, oh), nullptr, dptr<double>(h->e_tables, ot),
                            dptr<int32_t>(h->e_tables, orow),
                            dptr<lp_liveput_row>(h->e_tables, oout)));
  LP_CUDA(h, h->pin_down.ensure(sizeof(lp_liveput_row)));
  LP_CUDA(h, cudaMemcpyAsync(h->pin_down.p, dptr<void>(h->e_tables, oout), sizeof(lp_liveput_row),
                             cudaMemcpyDeviceToHost, h->stream));
  LP_CUDA(h, cudaStreamSynchronize(h->stream));
  *out = static_cast<lp_liveput_row*>(h->pin_down.p)->liveput;
  return LP_OK;
}

static lp_status dump_common(lp_handle* h, int32_t n, int32_t k, int32_t exact, int32_t trials,
                             uint64_t seed, const lp_config* cfgs, int32_t n_cfg,
                             uint16_t* sorted_out, uint16_t* m_out) {
  if (!h) return fail(nullptr, LP_EINVAL, "null handle");
  if (k < 0 || k > n) return fail(h, LP_EINVAL, "sample_vectors: bad n_minus");
  if (n > kMaxN) return fail(h, LP_EUNSUPPORTED, "n exceeds supported maximum");
  if (trials < 1) return fail(h, LP_EINVAL, "sample_vectors: trials must be >= 1");
  if (exact && (uint64_t)trials != scenario_count(n, k))
    return fail(h, LP_EINVAL, "dump: exact mode needs trials == C(n, k)");
  for (int c = 0; c < n_cfg; ++c)
    if (cfgs[c].pipelines < 1 || cfgs[c].stages < 1 ||
        (long long)cfgs[c].pipelines * cfgs[c].stages > n)
      return fail(h, LP_EINVAL, "dump: config exceeds n");
  cudaSetDevice(h->device);
  EnsembleSpec sp;
  sp.n = n;
  sp.k = k;
  sp.exact = exact != 0;
  sp.count = (uint64_t)trials;
  sp.seed = seed;
  HistPlan hp;
  std::string err;
  lp_status s = build_hist_plan({sp}, 0, 1, hp, err);
  if (s != LP_OK) return fail(h, s, "%s", err.c_str());
  std::vector<int2> cv(std::max(n_cfg, 1));
  for (int c = 0; c < n_cfg; ++c) cv[c] = make_int2(cfgs[c].pipelines, cfgs[c].stages);
  Packer pk;
  const size_t od = pk.add(hp.draws), ob = pk.add(hp.binom), oc = pk.add(cv);
  LP_CUDA(h, h->e_tables.ensure(pk.bytes.size()));
  LP_CUDA(h, h->pin_up.ensure(pk.bytes.size()));
  std::memcpy(h->pin_up.p, pk.bytes.data(), pk.bytes.size());
  LP_CUDA(h, cudaMemcpyAsync(h->e_tables.p, h->pin_up.p, pk.bytes.size(), cudaMemcpyHostToDevice,
                             h->stream));
  const size_t kk = std::max(k, 1);
  const size_t nw = (n + 31) / 32;
  const size_t srt_b = 2 * kk * trials, m_b = m_out ? 2 * (size_t)trials * std::max(n_cfg, 1) : 0;
  const size_t scr_b = k > 16 ? 4 * (size_t)(k + nw) * trials : 4;
  const size_t o1 = 0, o2 = (srt_b + 255) & ~size_t(255), o3 = o2 + ((m_b + 255) & ~size_t(255));
  LP_CUDA(h, h->e_work.ensure(o3 + scr_b));
  const int stride = hp.pairs.empty() ? 1 : hp.pairs[0].binom_stride;
  LP_CUDA(h, launch_dump(n, k, exact, trials, seed, dptr<DrawConst>(h->e_tables, od),
                         dptr<uint64_t>(h->e_tables, ob), stride, dptr<uint32_t>(h->e_work, o3),
                         dptr<uint16_t>(h->e_work, o1), dptr<int2>(h->e_tables, oc), n_cfg,
                         m_out ? dptr<uint16_t>(h->e_work, o2) : nullptr, h->stream));
  if (sorted_out)
    LP_CUDA(h, cudaMemcpyAsync(sorted_out, dptr<uint16_t>(h->e_work, o1), 2 * (size_t)k * trials,
                               cudaMemcpyDeviceToHost, h->stream));
  if (m_out)
    LP_CUDA(h, cudaMemcpyAsync(m_out, dptr<uint16_t>(h->e_work, o2), 2 * (size_t)trials * n_cfg,
                               cudaMemcpyDeviceToHost, h->stream));
  LP_CUDA(h, cudaStreamSynchronize(h->stream));
  return LP_OK;
}

lp_status lp_dump_survivors(lp_handle* h, int32_t n, int32_t n_minus, int32_t exact, int32_t trials,
                            uint64_t seed, const lp_config* cfgs, int32_t n_cfg, uint16_t* out) {
  if (!out || !cfgs || n_cfg < 1) return fail(h, LP_EINVAL, "lp_dump_survivors: bad output");
  return dump_common(h, n, n_minus, exact, trials, seed, cfgs, n_cfg, nullptr, out);
}

lp_status lp_dump_scenarios(lp_handle* h, int32_t n, int32_t n_minus, int32_t trials, uint64_t seed,
                            uint16_t* out) {
  if (!out) return fail(h, LP_EINVAL, "lp_dump_scenarios: null output");
  if (n_minus == 0) return dump_common(h, n, 0, 0, trials, seed, nullptr, 0, nullptr, nullptr);
  return dump_common(h, n, n_minus, 0, trials, seed, nullptr, 0, out, nullptr);
}

// ---------------------------------------------------------------------------
lp_status lp_nccl_unique_id(uint8_t out[LP_NCCL_ID_BYTES]) {
  static_assert(sizeof(ncclUniqueId) == LP_NCCL_ID_BYTES, "nccl id size");
  if (!nccl().ok) return fail(nullptr, LP_ENCCL, "NCCL library could not be loaded");
  ncclUniqueId id;
  ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess)
    return fail(nullptr, LP_ENCCL, "ncclGetUniqueId: %s", nccl().GetErrorString(r));
  std::memcpy(out, &id, sizeof id);
  return LP_OK;
}

lp_status lp_set_shard(lp_handle* h, int32_t rank, int32_t nranks) {
  if (!h || nranks < 1 || rank < 0 || rank >= nranks) return fail(h, LP_EINVAL, "lp_set_shard: bad argument");
  h->shard_rank = rank;
  h->shard_n = nranks;
  h->hist_cache.clear();
  return LP_OK;
}

lp_status lp_comm_init(lp_handle* h, const uint8_t id[LP_NCCL_ID_BYTES], int32_t nranks,
                       int32_t rank) {
  if (!h || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(h, LP_EINVAL, "lp_comm_init: bad argument");
  cudaSetDevice(h->device);
  if (h->comm) {
    nccl().CommDestroy(h->comm);
    h->comm = nullptr;
  }
  if (nranks > 1) {
    if (!nccl().ok) return fail(h, LP_ENCCL, "NCCL library could not be loaded");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclResult_t r = nccl().CommInitRank(&h->comm, nranks, uid, rank);
    if (r != ncclSuccess)
      return fail(h, LP_ENCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r));
    // NCCL connects its channels lazily on the first collective (0.4-0.75 s
    // measured on B200); pay that here, not inside the first re-plan.
    LP_CUDA(h, h->work.ensure(256));
    r = nccl().AllReduce(h->work.p, h->work.p, 1, ncclUint32, ncclSum, h->comm, h->stream);
    if (r != ncclSuccess)
      return fail(h, LP_ENCCL, "ncclAllReduce (warm-up): %s", nccl().GetErrorString(r));
    LP_CUDA(h, cudaStreamSynchronize(h->stream));
  }
  h->nranks = nranks;
  h->rank = rank;
  h->prepared = false;
  return LP_OK;
}

// ---------------------------------------------------------------------------
double lp_throughput(const lp_profile* p, lp_config c) { return Model(*p).rate(c.pipelines, c.stages); }

int32_t lp_depth_feasible(const lp_profile* p, int32_t s) { return Model(*p).depth_ok(s) ? 1 : 0; }

int32_t lp_enumerate_configs(const lp_profile* p, int32_t n, lp_config* out, int32_t cap) {
  Model m(*p);
  const auto& cs = m.configs(n);
  for (int i = 0; i < (int)cs.size() && i < cap; ++i) out[i] = {cs[i].d, cs[i].p};
  return (int32_t)cs.size();
}

int32_t lp_reactive_plan(const lp_profile* p, int32_t n, lp_config* out) {
  Model m(*p);
  Cfg c;
  if (!m.reactive(n, &c)) return 0;
  if (out) *out = {c.d, c.p};
  return 1;
}

uint64_t lp_scenario_count(int32_t n, int32_t k) { return scenario_count(n, k); }
uint64_t lp_mix_seed(uint64_t a, uint64_t b) { return mix_seed(a, b); }

}  // extern "C"
