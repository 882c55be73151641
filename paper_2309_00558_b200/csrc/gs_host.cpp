// Host-side report rendering: metrics.csv straight from the
// device row records, byte-identical to the reference's MetricsReport.to_csv()
// (pkg/src/gshare_sim/metrics.py:62-91) -- without building one Python object
// per row, and on all host cores for a batch.
//
// Number rendering follows the reference exactly:
//   * util.py:4-10 fmt_num(x): integral and |x| < 1e15 -> "%d", else repr(x);
//   * metrics.py:47-48 / :88-89: utilisation, occupancy and fragmentation as
//     fmt_num(round(x, 9)), memory as fmt_num(round(x, 6)).
// round(x, n) is CPython's float.__round__ (correctly rounded decimal string
// with n fractional digits, ties-to-even on the exact binary value, parsed
// back correctly rounded) == std::to_chars(fixed, n) + std::from_chars.
// repr(x) is CPython's 'r' format: the shortest digit string that round-trips
// (std::to_chars without precision gives the same digits), printed in fixed
// notation when the decimal exponent is in (-4, 16], else as d.ddde+XX.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "gshare_b200.h"

namespace {

// CPython float.__round__(x, nd) for finite x and small nd.
double py_round(double x, int nd) {
  if (!std::isfinite(x)) return x;
  char buf[400];
  auto r = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::fixed, nd);
  double y = 0.0;
  std::from_chars(buf, r.ptr, y);
  return y;
}

// CPython repr(float) into o; returns the length.
int py_repr(double x, char* o) {
  if (std::isnan(x)) { std::memcpy(o, "nan", 3); return 3; }
  if (std::isinf(x)) {
    if (x < 0) { std::memcpy(o, "-inf", 4); return 4; }
    std::memcpy(o, "inf", 3); return 3;
  }
  char* p = o;
  if (x == 0.0) {
    if (std::signbit(x)) *p++ = '-';
    std::memcpy(p, "0.0", 3);
    return int(p - o) + 3;
  }
  char s[64];
  auto r = std::to_chars(s, s + sizeof s, x, std::chars_format::scientific);
  const char* q = s;
  if (*q == '-') { *p++ = '-'; ++q; }
  char dig[32];
  int nd = 0;
  for (; q < r.ptr && *q != 'e'; ++q)
    if (*q != '.') dig[nd++] = *q;
  int e = 0;
  std::from_chars(q + 1 + (q[1] == '+'), r.ptr, e);
  const int decpt = e + 1;                 // value = 0.DIGITS x 10^decpt
  if (decpt > -4 && decpt <= 16) {
    if (decpt <= 0) {
      *p++ = '0'; *p++ = '.';
      for (int i = 0; i < -decpt; ++i) *p++ = '0';
      std::memcpy(p, dig, nd); p += nd;
    } else if (decpt >= nd) {
      std::memcpy(p, dig, nd); p += nd;
      for (int i = nd; i < decpt; ++i) *p++ = '0';
      *p++ = '.'; *p++ = '0';
    } else {
      std::memcpy(p, dig, decpt); p += decpt;
      *p++ = '.';
      std::memcpy(p, dig + decpt, nd - decpt); p += nd - decpt;
    }
  } else {
    *p++ = dig[0];
    if (nd > 1) { *p++ = '.'; std::memcpy(p, dig + 1, nd - 1); p += nd - 1; }
    *p++ = 'e';
    int ex = decpt - 1;
    *p++ = ex < 0 ? '-' : '+';
    if (ex < 0) ex = -ex;
    if (ex < 10) *p++ = '0';
    auto t = std::to_chars(p, p + 8, ex);
    p = t.ptr;
  }
  return int(p - o);
}

// util.py fmt_num
int fmt_num(double x, char* o) {
  if (std::isfinite(x) && x == std::floor(x) && std::fabs(x) < 1e15) {
    auto t = std::to_chars(o, o + 24, (long long)x);
    return int(t.ptr - o);
  }
  return py_repr(x, o);
}

struct Writer {
  char* p;
  void put(const char* s, size_t n) { std::memcpy(p, s, n); p += n; }
  void lit(const char* s) { put(s, std::strlen(s)); }
  void i(long long v) { p = std::to_chars(p, p + 24, v).ptr; }
  void num(double x, int nd) { p += fmt_num(py_round(x, nd), p); }
};

const char kHeader[] =
    "window,kind,entity,arrivals,completions,slo_violations,dropped,queue_depth,"
    "utilization,sm_occupancy,memory_mb,gpus_in_use,placement_failures,fragmentation_index\n";

// upper bound of run r's CSV length
int64_t csv_bound(const gs_batch_t* in, int r, const int64_t* fid_off) {
  const gs_scenario_t& s = in->runs[r];
  const int64_t names = fid_off[s.func_off + s.n_funcs] - fid_off[s.func_off];
  // global row <= 12 + 11 commas + 2*11 + 32; function row <= 12 + 5*11 + 14 + fid;
  // gpu row <= 12 + 4 + 2*32 + 40 + 14  (repr <= 24 chars, fixed <= ~40)
  const int64_t per_w = 96 + int64_t(s.n_funcs) * 96 + names + int64_t(s.n_nodes) * 160;
  return int64_t(sizeof kHeader) + int64_t(s.windows) * per_w;
}

int64_t render(const gs_batch_t* in, const gs_out_t* out, int r, const char* fid_csv,
               const int64_t* fid_off, char* buf) {
  const gs_scenario_t& s = in->runs[r];
  const int W = s.windows, F = s.n_funcs, G = s.n_nodes;
  const gs_fn_row_t* fn = out->fn_rows + s.fn_row_off;
  const gs_gpu_row_t* gp = out->gpu_rows + s.gpu_row_off;
  const gs_glob_row_t* gl = out->glob_rows + s.glob_row_off;
  Writer w{buf};
  w.put(kHeader, sizeof kHeader - 1);
  for (int k = 0; k < W; ++k) {
    w.i(k); w.lit(",global,,,,,,,,,,");
    w.i(gl[k].gpus_in_use); *w.p++ = ',';
    w.i(gl[k].placement_failures); *w.p++ = ',';
    w.num(gl[k].fragmentation_index, 9); *w.p++ = '\n';
    for (int f = 0; f < F; ++f) {
      const gs_fn_row_t& x = fn[(int64_t)k * F + f];
      const int fi = s.func_off + f;
      w.i(k); w.lit(",function,");
      w.put(fid_csv + fid_off[fi], size_t(fid_off[fi + 1] - fid_off[fi]));
      *w.p++ = ','; w.i(x.arrivals); *w.p++ = ','; w.i(x.completions);
      *w.p++ = ','; w.i(x.slo_violations); *w.p++ = ','; w.i(x.dropped);
      *w.p++ = ','; w.i(x.queue_depth); w.lit(",,,,,,\n");
    }
    for (int g = 0; g < G; ++g) {
      const gs_gpu_row_t& x = gp[(int64_t)k * G + g];
      if (!x.present) continue;
      w.i(k); w.lit(",gpu,"); w.i(g); w.lit(",,,,,,");
      w.num(x.utilization, 9); *w.p++ = ',';
      w.num(x.sm_occupancy, 9); *w.p++ = ',';
      w.num(x.memory_mb, 6); w.lit(",,,\n");
    }
  }
  return int64_t(w.p - buf);
}

bool rows_ok(const gs_batch_t* in, const gs_out_t* out) {
  return in && out && in->runs && out->fn_rows && out->gpu_rows && out->glob_rows;
}

}  // namespace

extern "C" int64_t gs_format_csv(const gs_batch_t* in, const gs_out_t* out, int run,
                                 const char* fid_csv, const int64_t* fid_off,
                                 char* buf, int64_t cap) {
  if (!rows_ok(in, out) || run < 0 || run >= in->n_runs || !fid_csv || !fid_off) return -1;
  const int64_t bound = csv_bound(in, run, fid_off);
  if (!buf || cap < bound) return bound;   // caller retries with >= bound bytes
  return render(in, out, run, fid_csv, fid_off, buf);
}

extern "C" int64_t gs_format_csv_batch(const gs_batch_t* in, const gs_out_t* out, int r0,
                                       int r1, const char* fid_csv, const int64_t* fid_off,
                                       char* buf, int64_t cap, int64_t* offs, int64_t* lens,
                                       int n_threads) {
  if (!rows_ok(in, out) || r0 < 0 || r1 > in->n_runs || r0 > r1 || !fid_csv || !fid_off)
    return -1;
  const int n = r1 - r0;
  std::vector<int64_t> start(n + 1, 0);
  for (int k = 0; k < n; ++k) start[k + 1] = start[k] + csv_bound(in, r0 + k, fid_off);
  if (!buf || !offs || !lens || cap < start[n]) return start[n];
  for (int k = 0; k < n; ++k) offs[k] = start[k];
  const int T = std::max(1, std::min(n_threads > 0 ? n_threads
                                                  : int(std::thread::hardware_concurrency()),
                                     std::max(n, 1)));
  auto work = [&](int t) {
    for (int k = t; k < n; k += T)
      lens[k] = render(in, out, r0 + k, fid_csv, fid_off, buf + start[k]);
  };
  if (T == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  return 0;
}

// fmt_num(round(x, nd)) of each value (the reference's number rendering; also
// lets the tests pin py_round / py_repr against the interpreter).
extern "C" int gs_format_numbers(const double* x, int64_t n, int nd, char* buf, int64_t stride) {
  if (!x || !buf || stride < 48) return -1;
  for (int64_t k = 0; k < n; ++k) {
    char* o = buf + k * stride;
    const double v = nd >= 0 ? py_round(x[k], nd) : x[k];
    const int len = fmt_num(v, o);
    o[len] = '\0';
  }
  return 0;
}

// Per-function totals of runs [r0, r1) for summary() (metrics.py:94-113):
// for every function of every run, (arrivals, completions, slo_violations,
// dropped) summed over the windows and the last window's queue depth --
// written at totals[5 * (funcs[func_off + f] - funcs[runs[r0].func_off]) ...],
// i.e. in batch function order.  Multithreaded over runs.
extern "C" int gs_fn_totals(const gs_batch_t* in, const gs_out_t* out, int r0, int r1,
                            int64_t* totals, int n_threads) {
  if (!in || !out || !out->fn_rows || !totals || r0 < 0 || r1 > in->n_runs || r0 > r1)
    return -1;
  const int n = r1 - r0;
  if (n == 0) return 0;
  const int base = in->runs[r0].func_off;
  const int T = std::max(1, std::min(n_threads > 0 ? n_threads
                                                  : int(std::thread::hardware_concurrency()), n));
  auto work = [&](int t) {
    for (int k = t; k < n; k += T) {
      const gs_scenario_t& s = in->runs[r0 + k];
      const int W = s.windows, F = s.n_funcs;
      const gs_fn_row_t* fn = out->fn_rows + s.fn_row_off;
      int64_t* o = totals + 5 * (int64_t)(s.func_off - base);
      for (int f = 0; f < F; ++f) {
        int64_t a = 0, c = 0, v = 0, d = 0;
        for (int w = 0; w < W; ++w) {
          const gs_fn_row_t& x = fn[(int64_t)w * F + f];
          a += x.arrivals; c += x.completions; v += x.slo_violations; d += x.dropped;
        }
        o[5 * f + 0] = a; o[5 * f + 1] = c; o[5 * f + 2] = v; o[5 * f + 3] = d;
        o[5 * f + 4] = W ? fn[(int64_t)(W - 1) * F + f].queue_depth : 0;
      }
    }
  };
  if (T == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  return 0;
}
