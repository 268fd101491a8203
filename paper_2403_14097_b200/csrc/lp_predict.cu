// lp_predict.cu — availability forecasts for the DP's n_seq.
//
// Restates predict / preprocess / arima_forecast / least_squares /
// postprocess / eval_l1 (reference predictor.cpp:29-286) as device code:
// one thread per (sliding window, method) of a trace, the batch the
// reference's `spotsim predict` command walks serially (commands.cpp:267-299).
//
// Compiled with -fmad=false (Makefile): every FP64 multiply and add rounds
// separately, as in the reference's x86-64 build, so the forecasts are the
// reference's.  Also built at NVVM -O1: at -O2+ the ARIMA fit disagrees with
// the host build of this same code (see the Makefile note).  std::pow(steep_decay, e) comes in as a host-computed table
// for the same reason.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>
#include <vector>

#include "liveput.h"

namespace lp {
std::string& global_error();  // lp_api.cpp

namespace {

// history_len / lookahead up to these use per-thread local arrays; longer
// windows use a per-thread slice of a global scratch buffer (same code).
constexpr int kMaxHist = 64;
constexpr int kMaxAhead = 64;

// Per-window work arrays: h, y (H ints), raw (I), z and e (H + I), and the
// least-squares design matrix A (5 (H - 3) rows-by-columns).
struct Scratch {
  int* h;
  int* y;
  double* raw;
  double* z;
  double* e;
  double* A;
};
__host__ __device__ inline size_t scratch_doubles(int H, int I) {
  return static_cast<size_t>(I) + 2 * static_cast<size_t>(H + I) + 5 * static_cast<size_t>(H) +
         static_cast<size_t>(H);  // the last H doubles hold the 2H ints
}
__host__ __device__ inline Scratch scratch_at(double* base, int H, int I) {
  Scratch sc;
  sc.raw = base;
  sc.z = sc.raw + I;
  sc.e = sc.z + (H + I);
  sc.A = sc.e + (H + I);
  sc.h = reinterpret_cast<int*>(sc.A + 5 * static_cast<size_t>(H));
  sc.y = sc.h + H;
  return sc;
}

#define LP_HD __host__ __device__
LP_HD __forceinline__ int iabs(int x) { return x < 0 ? -x : x; }
LP_HD __forceinline__ int iclamp(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }
LP_HD __forceinline__ double dclamp(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}

// preprocess (predictor.cpp:29-77) with hop_min_jump = 3, plateau_tol = 2.
LP_HD void preprocess(int* y, int n) {
  for (int i = 1; i + 1 < n; ++i) {  // flatten 1-2 interval excursions
    if (y[i] == y[i - 1]) continue;
    const int jend = i + 2 < n - 1 ? i + 2 : n - 1;
    for (int j = i + 1; j <= jend; ++j)
      if (y[j] == y[i - 1]) {
        for (int k = i; k < j; ++k) y[k] = y[i - 1];
        break;
      }
  }
  int last_shift = 0;  // last large level shift
  for (int i = 1; i < n; ++i)
    if (iabs(y[i] - y[i - 1]) >= 3) last_shift = i;
  if (last_shift > 0 && n - last_shift >= 3) {
    int mn = y[last_shift], mx = y[last_shift];
    for (int i = last_shift + 1; i < n; ++i) {
      mn = y[i] < mn ? y[i] : mn;
      mx = y[i] > mx ? y[i] : mx;
    }
    if (mx - mn <= 2) {
      for (int i = 0; i < last_shift; ++i) y[i] = y[last_shift];
      return;
    }
  }
  int turn = 0, prev_sign = 0;  // last change of direction
  for (int i = 1; i < n; ++i) {
    const int d = y[i] - y[i - 1];
    if (d == 0) continue;
    const int sign = d > 0 ? 1 : -1;
    if (prev_sign != 0 && sign != prev_sign) turn = i - 1;
    prev_sign = sign;
  }
  if (turn > 0 && n - turn >= 3)
    for (int i = 0; i < turn; ++i) y[i] = y[turn];
}

// least_squares (predictor.cpp:81-114): (A^T A + 1e-8 I) x = A^T b by
// Gauss-Jordan elimination with partial pivoting; A is m x P, row-major.
template <int P>
LP_HD bool least_squares(int m, const double* A, const double* b, double* x) {
  if (m == 0) return false;
  double ata[P][P], atb[P];
  for (int i = 0; i < P; ++i) {
    atb[i] = 0.0;
    for (int j = 0; j < P; ++j) ata[i][j] = 0.0;
  }
  for (int r = 0; r < m; ++r) {
    const double* a = A + r * P;
    for (int i = 0; i < P; ++i) {
      atb[i] += a[i] * b[r];
      for (int j = 0; j < P; ++j) ata[i][j] += a[i] * a[j];
    }
  }
  for (int i = 0; i < P; ++i) ata[i][i] += 1e-8;
  for (int col = 0; col < P; ++col) {
    int piv = col;
    for (int r = col + 1; r < P; ++r)
      if (fabs(ata[r][col]) > fabs(ata[piv][col])) piv = r;
    if (fabs(ata[piv][col]) < 1e-12) return false;
    for (int c = 0; c < P; ++c) {
      const double t = ata[col][c];
      ata[col][c] = ata[piv][c];
      ata[piv][c] = t;
    }
    const double tb = atb[col];
    atb[col] = atb[piv];
    atb[piv] = tb;
    for (int r = 0; r < P; ++r) {
      if (r == col) continue;
      const double f = ata[r][col] / ata[col][col];
      for (int c = col; c < P; ++c) ata[r][c] -= f * ata[col][c];
      atb[r] -= f * atb[col];
    }
  }
  for (int i = 0; i < P; ++i) {
    x[i] = atb[i] / ata[i][i];
    if (!isfinite(x[i])) return false;
  }
  return true;
}

// arima_forecast (predictor.cpp:120-188): ARIMA(2,1,2) by two-stage least
// squares on the differenced series; levels are damped cumulative sums.
LP_HD bool arima(const int* h, int n, int ahead, double* out, double* z, double* e, double* A) {
  if (n < 5) return false;
  const int m = n - 1;
  bool any = false;
  for (int i = 1; i < n; ++i) {
    z[i - 1] = static_cast<double>(h[i] - h[i - 1]);
    any |= z[i - 1] != 0.0;
  }
  if (!any) return false;
  const int rows = m - 2;  // t = 2 .. m-1
  for (int r = 0; r < rows; ++r) {
    const int t = r + 2;
    A[r * 3 + 0] = 1.0;
    A[r * 3 + 1] = z[t - 1];
    A[r * 3 + 2] = z[t - 2];
  }
  double ar[3];
  if (!least_squares<3>(rows, A, z + 2, ar)) return false;
  double sse_ar = 0.0;
  for (int t = 0; t < m; ++t) e[t] = 0.0;
  for (int t = 2; t < m; ++t) {
    e[t] = z[t] - (ar[0] + ar[1] * z[t - 1] + ar[2] * z[t - 2]);
    sse_ar += e[t] * e[t];
  }
  double c[5] = {ar[0], ar[1], ar[2], 0.0, 0.0};
  if (rows >= 8) {  // residual correction, kept only if it fits better
    for (int r = 0; r < rows; ++r) {
      const int t = r + 2;
      double* a = A + r * 5;
      a[0] = 1.0;
      a[1] = z[t - 1];
      a[2] = z[t - 2];
      a[3] = e[t - 1];
      a[4] = e[t - 2];
    }
    double full[5];
    if (least_squares<5>(rows, A, z + 2, full)) {
      double sse_full = 0.0;
      for (int r = 0; r < rows; ++r) {
        const double* a = A + r * 5;
        double pred = 0.0;
        for (int k = 0; k < 5; ++k) pred += full[k] * a[k];
        const double d = z[r + 2] - pred;
        sse_full += d * d;
      }
      if (sse_full < sse_ar)
        for (int k = 0; k < 5; ++k) c[k] = full[k];
    }
  }
  const double spectral = fabs(c[1]) + fabs(c[2]);  // stationarity guard
  if (spectral > 0.95) {
    c[1] *= 0.95 / spectral;
    c[2] *= 0.95 / spectral;
  }
  c[3] = dclamp(c[3], -0.95, 0.95);
  c[4] = dclamp(c[4], -0.95, 0.95);
  double level = static_cast<double>(h[n - 1]), damp = 1.0;
  int t = m;
  for (int k = 0; k < ahead; ++k, ++t) {
    const double zhat = c[0] + c[1] * z[t - 1] + c[2] * z[t - 2] + c[3] * e[t - 1] + c[4] * e[t - 2];
    if (!isfinite(zhat)) return false;
    z[t] = zhat;
    e[t] = 0.0;
    level += zhat * damp;
    damp *= 0.85;
    out[k] = level;
  }
  return true;
}

// postprocess (predictor.cpp:190-237); pw[e] = pow(steep_decay, e).
LP_HD void postprocess(const double* raw, int ahead, const lp_forecast_config& cf, int last,
                            const double* pw, int32_t* out) {
  const int lo = cf.floor, hi = cf.capacity;
  const int anchor = iclamp(last, lo, hi);
  if (ahead > 0 && llabs(llround(raw[0]) - anchor) > cf.reset_threshold) {
    for (int k = 0; k < ahead; ++k) out[k] = anchor;
    return;
  }
  int prev = anchor, steep = 0;
  double prev_raw = static_cast<double>(anchor);
  for (int k = 0; k < ahead; ++k) {
    double inc = raw[k] - prev_raw;
    prev_raw = raw[k];
    if (fabs(inc) > 0.5 * cf.max_step) {
      ++steep;
      if (steep > 1) inc *= pw[steep - 1];
    } else {
      steep = 0;
    }
    inc = dclamp(inc, -static_cast<double>(cf.max_step), static_cast<double>(cf.max_step));
    int v = static_cast<int>(llround(prev + inc));
    v = iclamp(v, lo, hi);
    v = iclamp(v, prev - cf.max_step, prev + cf.max_step);
    out[k] = v;
    prev = v;
  }
}

// predict (predictor.cpp:239-274) for the history ending at counts[t].
LP_HD void predict_one(const int32_t* counts, int t, const lp_forecast_config& cf, int method,
                            const double* pw, int32_t* out, const Scratch& sc) {
  const int H = cf.history_len, I = cf.lookahead;
  int* h = sc.h;
  for (int i = 0; i < H; ++i) h[i] = counts[t - H + i];
  const int last = h[H - 1];
  double* raw = sc.raw;
  switch (method) {
    case LP_PREDICT_MOVING_AVG: {
      const int w = cf.moving_avg_window < H ? cf.moving_avg_window : H;
      double s = 0.0;
      for (int i = H - w; i < H; ++i) s += h[i];
      const double mean = s / w;
      for (int k = 0; k < I; ++k) raw[k] = mean;
      break;
    }
    case LP_PREDICT_EXP_SMOOTH: {
      double s = h[0];
      for (int i = 1; i < H; ++i) s = cf.exp_smooth_factor * h[i] + (1.0 - cf.exp_smooth_factor) * s;
      for (int k = 0; k < I; ++k) raw[k] = s;
      break;
    }
    case LP_PREDICT_ARIMA: {
      int* y = sc.y;
      for (int i = 0; i < H; ++i) y[i] = h[i];
      preprocess(y, H);
      if (!arima(y, H, I, raw, sc.z, sc.e, sc.A))
        for (int k = 0; k < I; ++k) raw[k] = static_cast<double>(last);
      break;
    }
    default:  // last_value
      for (int k = 0; k < I; ++k) raw[k] = static_cast<double>(last);
  }
  postprocess(raw, I, cf, last, pw, out);
}

__device__ double l1_of(const int32_t* pred, const int32_t* actual, int len) {
  double num = 0.0, den = 0.0;
  for (int i = 0; i < len; ++i) {
    num += fabs(static_cast<double>(pred[i]) - actual[i]);
    den += actual[i];
  }
  if (den == 0.0) return num == 0.0 ? 0.0 : __longlong_as_double(0x7ff0000000000000LL);
  return num / den;
}

__global__ void predict_kernel(const int32_t* __restrict__ counts, int t_first, int n_windows,
                               lp_forecast_config cf, const int32_t* __restrict__ methods,
                               int n_methods, const double* __restrict__ pw, int32_t* __restrict__ preds,
                               double* __restrict__ l1, double* __restrict__ gscratch) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_windows * n_methods) return;
  const int w = g / n_methods, mi = g % n_methods;
  const int t = t_first + w;
  int32_t* out = preds + static_cast<size_t>(g) * cf.lookahead;
  if (gscratch) {  // long windows: a slice of the global scratch buffer
    const size_t per = scratch_doubles(cf.history_len, cf.lookahead);
    predict_one(counts, t, cf, methods[mi], pw, out,
                scratch_at(gscratch + static_cast<size_t>(g) * per, cf.history_len, cf.lookahead));
  } else {
    double local[kMaxAhead + 2 * (kMaxHist + kMaxAhead) + 5 * kMaxHist + kMaxHist];
    predict_one(counts, t, cf, methods[mi], pw, out, scratch_at(local, cf.history_len, cf.lookahead));
  }
  if (l1) l1[g] = l1_of(out, counts + t, cf.lookahead);
}

lp_status pfail(lp_status s, const char* m) {
  global_error() = m;  // lp_last_global_error()
  return s;
}

lp_status run_windows(const int32_t* counts, int32_t len, int t_first, int n_windows,
                      const lp_forecast_config& cf, const int32_t* methods, int n_methods, int device,
                      int32_t* preds, double* l1) {
  if (n_windows <= 0 || n_methods <= 0) return LP_OK;
  for (int m = 0; m < n_methods; ++m)
    if (methods[m] < LP_PREDICT_ARIMA || methods[m] > LP_PREDICT_LAST_VALUE)
      return pfail(LP_EINVAL, "unknown predict method");
  std::vector<double> pw(cf.lookahead + 1);
  for (int e = 0; e <= cf.lookahead; ++e) pw[e] = std::pow(cf.steep_decay, e);  // std::pow, as the reference
  if (cudaSetDevice(device) != cudaSuccess) return pfail(LP_ECUDA, "predict: cudaSetDevice failed");
  const size_t nout = static_cast<size_t>(n_windows) * n_methods;
  size_t off = 0;
  auto take = [&](size_t b) {
    const size_t r = off;
    off += (b + 255) & ~size_t(255);
    return r;
  };
  const bool big = cf.history_len > kMaxHist || cf.lookahead > kMaxAhead;
  const size_t o_c = take(4 * static_cast<size_t>(len)), o_m = take(4 * n_methods),
               o_pw = take(8 * pw.size()), o_p = take(4 * nout * cf.lookahead), o_l = take(8 * nout),
               o_s = take(big ? 8 * nout * scratch_doubles(cf.history_len, cf.lookahead) : 0);
  unsigned char* d = nullptr;
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
    return pfail(LP_ECUDA, "predict: stream");
  lp_status rs = LP_OK;
  if (cudaMallocAsync(&d, off, st) != cudaSuccess) {
    cudaStreamDestroy(st);
    return pfail(LP_ENOMEM, "predict: device allocation failed");
  }
  cudaMemcpyAsync(d + o_c, counts, 4 * static_cast<size_t>(len), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d + o_m, methods, 4 * n_methods, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d + o_pw, pw.data(), 8 * pw.size(), cudaMemcpyHostToDevice, st);
  const int threads = 128, blocks = static_cast<int>((nout + threads - 1) / threads);
  predict_kernel<<<blocks, threads, 0, st>>>(
      reinterpret_cast<int32_t*>(d + o_c), t_first, n_windows, cf, reinterpret_cast<int32_t*>(d + o_m),
      n_methods, reinterpret_cast<double*>(d + o_pw), reinterpret_cast<int32_t*>(d + o_p),
      l1 ? reinterpret_cast<double*>(d + o_l) : nullptr, big ? reinterpret_cast<double*>(d + o_s) : nullptr);
  cudaMemcpyAsync(preds, d + o_p, 4 * nout * cf.lookahead, cudaMemcpyDeviceToHost, st);
  if (l1) cudaMemcpyAsync(l1, d + o_l, 8 * nout, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) rs = pfail(LP_ECUDA, cudaGetErrorString(e));
  cudaStreamDestroy(st);
  return rs;
}

lp_status check_cfg(const lp_forecast_config* cf) {
  if (!cf) return pfail(LP_EINVAL, "predict: null config");
  if (cf->lookahead < 1) return pfail(LP_EINVAL, "predict: lookahead must be >= 1");
  if (cf->history_len < 1) return pfail(LP_EINVAL, "predict: history_len must be >= 1");
  return LP_OK;
}

}  // namespace

// Host evaluation of the same code (tests/debugging): one window.
void predict_host(const int32_t* counts, int t, const lp_forecast_config& cf, int method, int32_t* out) {
  std::vector<double> pw(cf.lookahead + 1);
  for (int e = 0; e <= cf.lookahead; ++e) pw[e] = std::pow(cf.steep_decay, e);
  std::vector<double> sc(scratch_doubles(cf.history_len, cf.lookahead));
  predict_one(counts, t, cf, method, pw.data(), out, scratch_at(sc.data(), cf.history_len, cf.lookahead));
}
}  // namespace lp

using namespace lp;

extern "C" {

lp_forecast_config lp_forecast_defaults(int32_t capacity) {
  lp_forecast_config c{};
  c.history_len = 12;
  c.lookahead = 12;
  c.capacity = capacity;
  c.floor = 0;
  c.max_step = 8;
  c.reset_threshold = 10;
  c.moving_avg_window = 4;
  c.exp_smooth_factor = 0.5;
  c.steep_decay = 0.7;
  return c;
}

lp_status lp_predict(const int32_t* history, int32_t len, const lp_forecast_config* cfg,
                     int32_t method, int32_t device, int32_t* out) {
  lp_status s = check_cfg(cfg);
  if (s != LP_OK) return s;
  if (!history || !out) return pfail(LP_EINVAL, "predict: null argument");
  if (len < cfg->history_len) return pfail(LP_EINVAL, "predict: history shorter than history_len");
  return run_windows(history, len, len, 1, *cfg, &method, 1, device, out, nullptr);
}

lp_status lp_predict_windows(const int32_t* counts, int32_t len, const lp_forecast_config* cfg,
                             const int32_t* methods, int32_t n_methods, int32_t device,
                             int32_t* preds, double* l1, int32_t* n_windows) {
  lp_status s = check_cfg(cfg);
  if (s != LP_OK) return s;
  if (!counts || !methods || !preds || !n_windows || n_methods < 1)
    return pfail(LP_EINVAL, "predict_windows: null argument");
  const int nw = len - cfg->history_len - cfg->lookahead + 1;
  *n_windows = nw > 0 ? nw : 0;
  return run_windows(counts, len, cfg->history_len, *n_windows, *cfg, methods, n_methods, device, preds,
                     l1);
}

double lp_eval_l1(const int32_t* pred, const int32_t* actual, int32_t len) {
  double num = 0.0, den = 0.0;
  for (int i = 0; i < len; ++i) {
    num += std::fabs(static_cast<double>(pred[i]) - actual[i]);
    den += actual[i];
  }
  if (den == 0.0) return num == 0.0 ? 0.0 : INFINITY;
  return num / den;
}

}  // extern "C"
