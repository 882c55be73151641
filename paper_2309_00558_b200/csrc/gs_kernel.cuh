// gs_kernel.cuh -- run state, epoch / packer / window code of the scenario
// kernels (sm_100a).
//
// One warp owns one (scenario, policy) run from the initial placement to the
// last window (persistent warps pull runs from an atomic work counter, longest
// first); the XL class gives a run a whole CTA (gs_xl.cuh).  This header holds
// the per-run arena view (Ctx, CtxTab), the warp-level epoch and window code
// and the arena-based per-request helpers the XL steps use:
//
//   epoch (sim_engine.py:409-430)   grouping by function (match_any counting
//                                   sort), running sets sorted in registers,
//                                   rps_gap / scale_up / scale_down on lanes
//                                   with lane-0 side effects, p_ideal argmin
//     best_match (packer.py:169-193)  warp argmin over (node, rect)
//     carve/prune (packer.py:196-242) warp ballot compaction
//   window begin (sim_engine.py:446-449)  warm-up, registered list sorted by
//                                   (node, pod_id), per-function lists
//   admit / serve (sim_engine.py:472-552) per request, arena based (XL steps)
//
// The quantum steps of the per-warp classes run on a shared-memory working set
// (gs_hot.cuh).  Exactness: every floating-point expression is the
// reference's, in Python's evaluation order, compiled with -fmad=false (no FMA
// contraction) and IEEE division; Python 3.12's compensated sum() is
// reproduced where the reference calls sum() (PySum).  Geometry is exact
// int64 on the compiler's scaled grid.
#pragma once
#include <stdint.h>

#include "../../include/gshare_b200.h"
#include "gs_state.cuh"

namespace gs {

constexpr double TIME_EPS = 1e-12;   // sim_engine.py:75
constexpr double QUOTA_EPS = 1e-9;   // token_backend.py:25
constexpr double SM_EPS = 1e-9;      // token_backend.py:26
constexpr double SM_LIMIT = 100.0;   // token_backend.py:18
constexpr unsigned FULL = 0xffffffffu;
constexpr unsigned long long POW11_10 = 25937424601ull;  // 11^10

// ----------------------------------------------------------------------------
// small helpers
// ----------------------------------------------------------------------------
struct PySum {  // Python 3.12 builtin sum() over floats (see oracle/gs_oracle.c)
  double f, c;
  int n;
  __device__ void reset() { f = 0.0; c = 0.0; n = 0; }
  __device__ void add(double x) {
    if (n++ == 0) { f = 0.0 + x; c = 0.0; return; }
    // CPython adds Neumaier's term: (f - t) + x if |f| >= |x| else (x - t) + f,
    // i.e. the exact rounding error of t = f + x (Fast2Sum with the larger
    // operand first).  Knuth's branch-free TwoSum yields that same exact
    // error for any finite operands, so c is bit-identical without the
    // data-dependent branch (-fmad=false keeps every step rounded as written).
    const double t = f + x;
    const double bp = t - f;
    c += (f - (t - bp)) + (x - bp);
    f = t;
  }
  __device__ double value() const {
    if (n == 0) return 0.0;
    double r = f;
    if (c != 0.0 && isfinite(c)) r += c;
    return r;
  }
};

// monotone map double -> u64 (non-NaN); -0.0 canonicalised to +0.0 so equal
// doubles (Python ==) get equal keys.
__device__ __forceinline__ unsigned long long ord_key(double x) {
  x = x + 0.0;
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

// Order-preserving integer of the text f"{counter:04d}" (<= 10 digits):
// base-11 digits with 0 as the "string ended" sentinel, so shorter strings
// that are prefixes sort first -- exactly Python's str comparison.  Digits
// are taken least significant first; digit j (from the right) of an n-digit
// text sits at base-11 position 10 - n + j.
__device__ __forceinline__ unsigned long long digits_key(int counter) {
  unsigned v = (unsigned)counter;
  int n = 1;
  #pragma unroll 1
  for (unsigned t = v / 10u; t && n < 10; t /= 10u) n++;
  if (n < 4) n = 4;
  unsigned long long w = 1, key = 0;
  #pragma unroll 1
  for (int i = n; i < 10; i++) w *= 11ull;
  #pragma unroll 1
  for (int j = 0; j < n; j++) { key += (unsigned long long)(v % 10u + 1u) * w; v /= 10u; w *= 11ull; }
  return key;
}

// A pod's string-order key (include/gshare_b200.h gs_id_split_t): the
// function's slot for this counter text, then the text itself.
__device__ __forceinline__ unsigned long long pod_okey(const gs_function_t& fs,
                                                       const gs_id_split_t* splits, int ctr) {
  const unsigned long long dk = digits_key(ctr);
  int slot = fs.id_rank;
  #pragma unroll 1
  for (int k = 0; k < fs.n_id_splits; k++) {
    const gs_id_split_t sp = splits[fs.id_split_off + k];
    if (dk > sp.threshold) slot = sp.slot;
  }
  return (unsigned long long)slot * POW11_10 + dk;
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll 1
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll 1
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ long long warp_max_ll(long long v) {
#pragma unroll 1
  for (int o = 16; o > 0; o >>= 1) {
    long long y = __shfl_xor_sync(FULL, v, o);
    v = y > v ? y : v;
  }
  return v;
}

// ----------------------------------------------------------------------------
// per-warp scalars (shared memory) and the run context (registers)
// ----------------------------------------------------------------------------
// Arena pointers of a run, kept in the warp's shared memory: the window and
// epoch code reads them with one LDS each instead of holding ~60 pointers in
// registers (or recomputing the layout chain when they are evicted).
struct CtxTab {
  // pods
  int *p_fn, *p_pt, *p_node, *p_flags, *p_warm, *p_ctr, *p_x, *p_y, *p_w, *p_h, *p_cw, *p_ci;
  unsigned long long* p_okey;
  double *p_sm, *p_qreq, *p_qlim, *p_qused, *p_busy, *p_invr, *p_crem, *p_carr, *p_dur;
  // functions
  int *f_qlen, *f_pinned, *f_fw, *f_fi, *f_fn, *f_nsn, *f_nsw, *f_nsi, *f_rhead, *f_retn;
  int *f_pctr, *f_warr, *f_wcomp, *f_wviol, *f_wdrop, *f_hn, *f_ringoff, *f_loff;
  double* f_hist;
  long long* f_ret;
  long long* f_ring;
  // nodes
  double *n_sr, *n_cov, *n_occ, *n_fp;
  int *n_nfree, *n_nres, *n_nplaced, *n_seg;
  int4* n_rect;
  int2* n_res;
  int* n_cnt;
  int *n_reqsm, *n_cut, *n_ngr;
  unsigned long long* n_covb;
  // scratch
  int *s_rl, *s_fl, *s_free, *s_batch, *s_list;
  unsigned long long *s_ka, *s_kd;
  int* s_ki;
  int4 *s_carve, *s_rs;
  int2* s_pos;
  int* s_fcur;
};

struct WarpShared {
  int n_reg, free_top, win_failures, n_batch;
  int err, err_detail, err_a0, err_a1;
  int n_list;
  int next_warm;          // earliest warm_at among placed, unregistered pods
  long long grants, decisions, attempts, pod_steps, rect_scans;
  // the sort scratch's arena slices while it is redirected into the warp's
  // idle working-set bytes (window rebuilds, gs_kernel.cu scratch_to_shared)
  unsigned long long *ka_arena, *kd_arena;
  int* ki_arena;
  int min_free;
  double frag;
  CtxTab tab;
};

struct Ctx {
  // inputs
  const gs_scenario_t* sc;
  const gs_function_t* fs;
  const gs_point_t* points;
  const int32_t* counts;
  const gs_init_t* inits;
  const gs_id_split_t* splits;
  int G, F, P, R, RET, W, T, flags, Q;
  double ws, qs, quantum, cap_mb;
  int lane;
  WarpShared* sh;
  CtxTab* t;         // arena pointers (shared memory)

  __device__ const gs_point_t& pt(int f, int k) const { return points[fs[f].point_off + k]; }
  __device__ int count(int f, int w) const { return counts[fs[f].count_off + w]; }
  __device__ bool integral() const { return (flags & GS_FLAG_SM_INTEGRAL) != 0; }
};

template <typename T>
__device__ __forceinline__ T* carve_ptr(char* base, size_t off) {
  return reinterpret_cast<T*>(base + off);
}

__device__ void ctx_bind(Ctx& c, char* base, const Layout& L) {  // lane 0 writes the table
  CtxTab& t = *c.t;
  if (c.lane == 0) {
  t.p_fn = carve_ptr<int>(base, L.p_fn); t.p_pt = carve_ptr<int>(base, L.p_pt);
  t.p_node = carve_ptr<int>(base, L.p_node); t.p_flags = carve_ptr<int>(base, L.p_flags);
  t.p_warm = carve_ptr<int>(base, L.p_warm); t.p_ctr = carve_ptr<int>(base, L.p_ctr);
  t.p_x = carve_ptr<int>(base, L.p_x); t.p_y = carve_ptr<int>(base, L.p_y);
  t.p_w = carve_ptr<int>(base, L.p_w); t.p_h = carve_ptr<int>(base, L.p_h);
  t.p_cw = carve_ptr<int>(base, L.p_cw); t.p_ci = carve_ptr<int>(base, L.p_ci);
  t.p_okey = carve_ptr<unsigned long long>(base, L.p_okey);
  t.p_sm = carve_ptr<double>(base, L.p_sm); t.p_qreq = carve_ptr<double>(base, L.p_qreq);
  t.p_qlim = carve_ptr<double>(base, L.p_qlim); t.p_qused = carve_ptr<double>(base, L.p_qused);
  t.p_busy = carve_ptr<double>(base, L.p_busy); t.p_invr = carve_ptr<double>(base, L.p_invr);
  t.p_crem = carve_ptr<double>(base, L.p_crem); t.p_carr = carve_ptr<double>(base, L.p_carr);
  t.p_dur = carve_ptr<double>(base, L.p_dur);
  t.f_qlen = carve_ptr<int>(base, L.f_qlen); t.f_pinned = carve_ptr<int>(base, L.f_pinned);
  t.f_fw = carve_ptr<int>(base, L.f_fw); t.f_fi = carve_ptr<int>(base, L.f_fi);
  t.f_fn = carve_ptr<int>(base, L.f_fn); t.f_nsn = carve_ptr<int>(base, L.f_nsn);
  t.f_nsw = carve_ptr<int>(base, L.f_nsw); t.f_nsi = carve_ptr<int>(base, L.f_nsi);
  t.f_rhead = carve_ptr<int>(base, L.f_rhead); t.f_retn = carve_ptr<int>(base, L.f_retn);
  t.f_pctr = carve_ptr<int>(base, L.f_pctr); t.f_warr = carve_ptr<int>(base, L.f_warr);
  t.f_wcomp = carve_ptr<int>(base, L.f_wcomp); t.f_wviol = carve_ptr<int>(base, L.f_wviol);
  t.f_wdrop = carve_ptr<int>(base, L.f_wdrop); t.f_hn = carve_ptr<int>(base, L.f_hn);
  t.f_ringoff = carve_ptr<int>(base, L.f_ringoff); t.f_loff = carve_ptr<int>(base, L.f_loff);
  t.f_hist = carve_ptr<double>(base, L.f_hist);
  t.f_ret = carve_ptr<long long>(base, L.f_ret);
  t.f_ring = carve_ptr<long long>(base, L.f_ring);
  t.n_sr = carve_ptr<double>(base, L.n_sr); t.n_cov = carve_ptr<double>(base, L.n_cov);
  t.n_occ = carve_ptr<double>(base, L.n_occ); t.n_fp = carve_ptr<double>(base, L.n_fp);
  t.n_nfree = carve_ptr<int>(base, L.n_nfree); t.n_nres = carve_ptr<int>(base, L.n_nres);
  t.n_nplaced = carve_ptr<int>(base, L.n_nplaced); t.n_seg = carve_ptr<int>(base, L.n_seg);
  t.n_rect = carve_ptr<int4>(base, L.n_rect);
  t.n_res = carve_ptr<int2>(base, L.n_res);
  t.n_cnt = carve_ptr<int>(base, L.n_cnt);
  t.n_reqsm = carve_ptr<int>(base, L.n_reqsm); t.n_cut = carve_ptr<int>(base, L.n_cut);
  t.n_ngr = carve_ptr<int>(base, L.n_ngr);
  t.n_covb = carve_ptr<unsigned long long>(base, L.n_covb);
  t.s_rl = carve_ptr<int>(base, L.s_rl); t.s_fl = carve_ptr<int>(base, L.s_fl);
  t.s_free = carve_ptr<int>(base, L.s_free); t.s_batch = carve_ptr<int>(base, L.s_batch);
  t.s_list = carve_ptr<int>(base, L.s_list);
  t.s_ka = carve_ptr<unsigned long long>(base, L.s_ka);
  t.s_kd = carve_ptr<unsigned long long>(base, L.s_kd);
  t.s_ki = carve_ptr<int>(base, L.s_ki);
  t.s_carve = carve_ptr<int4>(base, L.s_carve);
  t.s_rs = carve_ptr<int4>(base, L.s_rs);
  t.s_pos = carve_ptr<int2>(base, L.s_pos);
  t.s_fcur = carve_ptr<int>(base, L.s_fcur);
  }
  __syncwarp();
  c.Q = L.Q;
}

// Pod slots ever allocated are exactly [0, P - min_free): the free stack hands
// out fresh slots in increasing order and reuses freed ones first, so every
// scan over pods can stop at this high-water mark instead of the capacity.
__device__ __forceinline__ int pod_high(const Ctx& c) { return c.P - c.sh->min_free; }

__device__ __forceinline__ void set_error(Ctx& c, int code, int detail, int a0, int a1) {
  // lane-agnostic: first error wins
  if (c.sh->err == 0) {
    c.sh->err = code; c.sh->err_detail = detail; c.sh->err_a0 = a0; c.sh->err_a1 = a1;
  }
}
__device__ __forceinline__ bool failed(const Ctx& c) {
  __syncwarp();
  return c.sh->err != 0;
}

// ----------------------------------------------------------------------------
// warp bitonic sort of (ka, kb, v) triples held in scratch, ascending
// ----------------------------------------------------------------------------
__device__ __forceinline__ bool trip_less(unsigned long long a1, unsigned long long b1, int v1,
                                          unsigned long long a2, unsigned long long b2, int v2) {
  return a1 < a2 || (a1 == a2 && (b1 < b2 || (b1 == b2 && v1 < v2)));
}

__device__ __noinline__ void warp_sort(Ctx& c, int n) {
  unsigned long long* A = c.t->s_ka;
  unsigned long long* B = c.t->s_kd;
  int* V = c.t->s_ki;
  int q = 1;
  #pragma unroll 1
  while (q < n) q <<= 1;
  if (q < 2) { __syncwarp(); return; }
  #pragma unroll 1
  for (int i = n + c.lane; i < q; i += 32) { A[i] = ~0ull; B[i] = ~0ull; V[i] = 0x7fffffff; }
  __syncwarp();
  if (q <= 32) {
    // register path: one element per lane
    unsigned long long a = c.lane < q ? A[c.lane] : ~0ull;
    unsigned long long b = c.lane < q ? B[c.lane] : ~0ull;
    int v = c.lane < q ? V[c.lane] : 0x7fffffff;
    #pragma unroll 1
    for (int k = 2; k <= q; k <<= 1) {
      #pragma unroll 1
      for (int j = k >> 1; j > 0; j >>= 1) {
        unsigned long long oa = __shfl_xor_sync(FULL, a, j);
        unsigned long long ob = __shfl_xor_sync(FULL, b, j);
        int ov = __shfl_xor_sync(FULL, v, j);
        bool up = (c.lane & k) == 0;
        bool lower = (c.lane & j) == 0;
        bool other_less = trip_less(oa, ob, ov, a, b, v);
        // lower element keeps the min when sorting up
        bool take = lower == up ? other_less : !other_less && !(oa == a && ob == b && ov == v);
        if (take) { a = oa; b = ob; v = ov; }
      }
    }
    if (c.lane < q) { A[c.lane] = a; B[c.lane] = b; V[c.lane] = v; }
    __syncwarp();
    return;
  }
  #pragma unroll 1
  for (int k = 2; k <= q; k <<= 1) {
    #pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      #pragma unroll 1
      for (int t = c.lane; t < (q >> 1); t += 32) {
        int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        int l = i | j;
        bool up = (i & k) == 0;
        unsigned long long ai = A[i], bi = B[i], al = A[l], bl = B[l];
        int vi = V[i], vl = V[l];
        bool l_less = trip_less(al, bl, vl, ai, bi, vi);
        if (l_less == up) {
          A[i] = al; B[i] = bl; V[i] = vl;
          A[l] = ai; B[l] = bi; V[l] = vi;
        }
      }
      __syncwarp();
    }
  }
}

// ----------------------------------------------------------------------------
// request ids and arrival times (sim_engine.py:462-470)
// ----------------------------------------------------------------------------
__device__ __forceinline__ long long pack_id(int w, int i) { return ((long long)w << 32) | (unsigned)i; }
__device__ __forceinline__ int id_w(long long id) { return (int)(id >> 32); }
__device__ __forceinline__ int id_i(long long id) { return (int)(id & 0xffffffffll); }

__device__ __forceinline__ double arrival_time(const Ctx& c, int f, int w, int i) {
  // start + i * window_s / n, start = window * window_s
  double n = (double)c.count(f, w);
  return (double)w * c.ws + ((double)i * c.ws) / n;
}

// advance (w, i) to the next generated request; caller guarantees one exists
__device__ __forceinline__ void advance_id(const Ctx& c, int f, int& w, int& i) {
  i++;
  #pragma unroll 1
  while (w < c.W && i >= c.count(f, w)) { w++; i = 0; }
}

// ----------------------------------------------------------------------------
// memory model (memory_model.py:36-88)
// ----------------------------------------------------------------------------
__device__ void refresh_footprint(Ctx& c, int g) {  // lane-agnostic, single lane
  double total = 0.0;
  int nres = c.t->n_nres[g];
  const bool sharing = (c.flags & GS_FLAG_SHARING) != 0;
  #pragma unroll 1
  for (int i = 0; i < nres; i++) {
    int2 e = c.t->n_res[g * c.F + i];
    if (e.y <= 0) continue;
    const gs_function_t& f = c.fs[e.x];
    if (sharing) total += f.mem_server_mb + (double)e.y * f.mem_runtime_mb;
    else total += (double)e.y * f.mem_noshare_mb;
  }
  c.t->n_fp[g] = total;
}

__device__ __forceinline__ bool admit(const Ctx& c, int g, int f) {
  const gs_function_t& fs = c.fs[f];
  double delta;
  if (c.flags & GS_FLAG_SHARING) {
    delta = fs.mem_runtime_mb;
    if (c.t->n_cnt[g * c.F + f] <= 0) delta += fs.mem_server_mb;
  } else {
    delta = fs.mem_noshare_mb;
  }
  return c.t->n_fp[g] + delta <= c.cap_mb;
}

__device__ void mem_add(Ctx& c, int g, int f) {  // single lane
  int* cnt = &c.t->n_cnt[g * c.F + f];
  int2* res = &c.t->n_res[g * c.F];
  if (*cnt > 0) {
    int n = c.t->n_nres[g];
    #pragma unroll 1
    for (int i = 0; i < n; i++) if (res[i].x == f) { res[i].y++; break; }
  } else {
    res[c.t->n_nres[g]++] = make_int2(f, 1);
  }
  (*cnt)++;
  refresh_footprint(c, g);
}

__device__ void mem_remove(Ctx& c, int g, int f) {  // single lane
  int* cnt = &c.t->n_cnt[g * c.F + f];
  int2* res = &c.t->n_res[g * c.F];
  int n = c.t->n_nres[g];
  #pragma unroll 1
  for (int i = 0; i < n; i++) {
    if (res[i].x != f) continue;
    if (res[i].y == 1) {            // del resident[fid]: keep the order of the rest
      #pragma unroll 1
      for (int j = i; j + 1 < n; j++) res[j] = res[j + 1];
      c.t->n_nres[g] = n - 1;
    } else {
      res[i].y--;
    }
    break;
  }
  (*cnt)--;
  refresh_footprint(c, g);
}

// ----------------------------------------------------------------------------
// packer (packer.py:169-320), int64 geometry on the scaled grid
// ----------------------------------------------------------------------------
__device__ __forceinline__ bool r_intersects(int4 a, int4 b) {
  return a.x < b.x + b.z && b.x < a.x + a.z && a.y < b.y + b.w && b.y < a.y + a.w;
}
__device__ __forceinline__ bool r_contains(int4 a, int4 b) {
  return b.x >= a.x && b.y >= a.y && b.x + b.z <= a.x + a.z && b.y + b.w <= a.y + a.w;
}
__device__ __forceinline__ bool r_eq(int4 a, int4 b) {
  return a.x == b.x && a.y == b.y && a.z == b.z && a.w == b.w;
}
__device__ __forceinline__ long long r_area(int4 r) { return (long long)r.z * (long long)r.w; }

// _carve + _subdivide + _prune_contained (packer.py:196-242) on `list[0..*n)`,
// warp-cooperative, stable.  Returns false (and leaves the list untouched)
// when the pruned result would exceed `cap`.
__device__ __noinline__ bool carve(Ctx& c, int4* list, int* n_ptr, int4 placed, int cap) {
  int n = *n_ptr;
  int4* tmp = c.t->s_carve;
  int base = 0;
  #pragma unroll 1
  for (int s = 0; s < n; s += 32) {
    int j = s + c.lane;
    int4 parts[4];
    int np = 0;
    if (j < n) {
      int4 r = list[j];
      if (!r_intersects(r, placed)) {
        parts[np++] = r;
      } else {
        int ix = max(r.x, placed.x), iy = max(r.y, placed.y);
        int ix2 = min(r.x + r.z, placed.x + placed.z), iy2 = min(r.y + r.w, placed.y + placed.w);
        if (ix > r.x) parts[np++] = make_int4(r.x, r.y, ix - r.x, r.w);
        if (ix2 < r.x + r.z) parts[np++] = make_int4(ix2, r.y, r.x + r.z - ix2, r.w);
        if (iy > r.y) parts[np++] = make_int4(r.x, r.y, r.z, iy - r.y);
        if (iy2 < r.y + r.w) parts[np++] = make_int4(r.x, iy2, r.z, r.y + r.w - iy2);
      }
    }
    int incl = warp_incl_scan(np, c.lane);
    int off = base + incl - np;
    #pragma unroll 1
    for (int k = 0; k < np; k++) tmp[off + k] = parts[k];
    base += __shfl_sync(FULL, incl, 31);
  }
  __syncwarp();
  int m = base;
  // prune: drop rects contained in another; exact duplicates keep the first
  int kept_base = 0;
  #pragma unroll 1
  for (int s = 0; s < m; s += 32) {
    int i = s + c.lane;
    bool keep = false;
    if (i < m) {
      int4 r = tmp[i];
      keep = true;
      #pragma unroll 1
      for (int j = 0; j < m; j++) {
        if (j == i) continue;
        int4 o = tmp[j];
        if (!r_contains(o, r)) continue;
        if (r_eq(r, o) && i < j) continue;
        keep = false;
        break;
      }
    }
    unsigned bal = __ballot_sync(FULL, keep);
    kept_base += __popc(bal);
  }
  if (kept_base > cap) return false;
  // second pass writes (list may alias nothing in tmp)
  int outp = 0;
  #pragma unroll 1
  for (int s = 0; s < m; s += 32) {
    int i = s + c.lane;
    bool keep = false;
    int4 r = make_int4(0, 0, 0, 0);
    if (i < m) {
      r = tmp[i];
      keep = true;
      #pragma unroll 1
      for (int j = 0; j < m; j++) {
        if (j == i) continue;
        int4 o = tmp[j];
        if (!r_contains(o, r)) continue;
        if (r_eq(r, o) && i < j) continue;
        keep = false;
        break;
      }
    }
    unsigned bal = __ballot_sync(FULL, keep);
    if (keep) list[outp + __popc(bal & ((1u << c.lane) - 1u))] = r;
    outp += __popc(bal);
  }
  __syncwarp();
  if (c.lane == 0) *n_ptr = outp;
  __syncwarp();
  return true;
}

// warp argmin over candidate keys (k0, a, b, c2, idx); returns the winning idx
// (or -1) in every lane.
struct BestKey {
  long long k0;
  int a, b, d, idx;
};
__device__ __forceinline__ bool bk_less(const BestKey& x, const BestKey& y) {
  if (x.idx < 0) return false;
  if (y.idx < 0) return true;
  if (x.k0 != y.k0) return x.k0 < y.k0;
  if (x.a != y.a) return x.a < y.a;
  if (x.b != y.b) return x.b < y.b;
  if (x.d != y.d) return x.d < y.d;
  return x.idx < y.idx;
}
__device__ BestKey warp_argmin(BestKey k) {
#pragma unroll 1
  for (int o = 16; o > 0; o >>= 1) {
    BestKey y;
    y.k0 = __shfl_xor_sync(FULL, k.k0, o);
    y.a = __shfl_xor_sync(FULL, k.a, o);
    y.b = __shfl_xor_sync(FULL, k.b, o);
    y.d = __shfl_xor_sync(FULL, k.d, o);
    y.idx = __shfl_xor_sync(FULL, k.idx, o);
    if (bk_less(y, k)) k = y;
  }
  return k;
}

// best_match (packer.py:169-193): key (r.area - req.area, gpu, y, x), first
// in (gpu, list) order on full ties.  Returns node (or -1) and the rect.
__device__ __noinline__ int best_match(Ctx& c, int slot, int4* chosen) {
  int f = c.t->p_fn[slot];
  int rw = c.t->p_w[slot], rh = c.t->p_h[slot];
  long long rarea = (long long)rw * rh;
  BestKey best;
  best.idx = -1; best.k0 = 0; best.a = best.b = best.d = 0;
  long long scans = 0;
  if (c.G >= 16) {
    // large fleets: lanes = nodes, so the per-node memory admission checks
    // (dependent loads) run in parallel; each lane scans its node's list
    #pragma unroll 1
    for (int g = c.lane; g < c.G; g += 32) {
      if (!admit(c, g, f)) continue;
      const int nf = c.t->n_nfree[g];
      scans += nf;
      #pragma unroll 1
      for (int j = 0; j < nf; j++) {
        const int4 r = c.t->n_rect[g * c.R + j];
        if (rw <= r.z && rh <= r.w) {
          BestKey k;
          k.k0 = r_area(r) - rarea; k.a = g; k.b = r.y; k.d = r.x; k.idx = g * c.R + j;
          if (bk_less(k, best)) best = k;
        }
      }
    }
    scans = warp_sum_ll(scans);
  } else {
    #pragma unroll 1
    for (int g = 0; g < c.G; g++) {
      if (!admit(c, g, f)) continue;
      int nf = c.t->n_nfree[g];
      scans += nf;
      #pragma unroll 1
      for (int j = c.lane; j < nf; j += 32) {
        int4 r = c.t->n_rect[g * c.R + j];
        if (rw <= r.z && rh <= r.w) {
          BestKey k;
          k.k0 = r_area(r) - rarea; k.a = g; k.b = r.y; k.d = r.x; k.idx = g * c.R + j;
          if (bk_less(k, best)) best = k;
        }
      }
    }
  }
  best = warp_argmin(best);
  if (c.lane == 0) c.sh->rect_scans += scans;
  if (best.idx < 0) return -1;
  *chosen = c.t->n_rect[best.idx];
  return best.a;
}

// _best_fit_in_node (packer.py:278-287) on an arbitrary list
__device__ __noinline__ int best_fit_in_list(Ctx& c, const int4* list, int n, int w, int h) {
  long long area = (long long)w * h;
  BestKey best;
  best.idx = -1; best.k0 = 0; best.a = best.b = best.d = 0;
  #pragma unroll 1
  for (int j = c.lane; j < n; j += 32) {
    int4 r = list[j];
    if (w <= r.z && h <= r.w) {
      BestKey k;
      k.k0 = r_area(r) - area; k.a = r.y; k.b = r.x; k.d = 0; k.idx = j;
      if (bk_less(k, best)) best = k;
    }
  }
  best = warp_argmin(best);
  return best.idx;
}

// ----------------------------------------------------------------------------
// pods (sim_engine.py:337-407)
// ----------------------------------------------------------------------------
__device__ int make_pod(Ctx& c, int f, int k, int has_qreq, double qreq, int warm) {  // lane 0
  const gs_point_t& p = c.pt(f, k);
  if (!p.rate_ok) {  // _service_rate: zero serving rate -> ValidationError
    set_error(c, GS_ERR_VALIDATION, 0, f, k);
    return -1;
  }
  if (c.sh->free_top <= 0) {
    set_error(c, GS_ERR_CAPACITY, GS_CAP_PODS, c.P, 0);
    return -1;
  }
  int slot = c.t->s_free[--c.sh->free_top];
  if (c.sh->free_top < c.sh->min_free) c.sh->min_free = c.sh->free_top;
  int ctr = c.t->f_pctr[f]++;
  c.t->p_fn[slot] = f; c.t->p_pt[slot] = k; c.t->p_node[slot] = -1; c.t->p_flags[slot] = PF_ALIVE;
  c.t->p_warm[slot] = warm; c.t->p_ctr[slot] = ctr; c.t->p_x[slot] = 0; c.t->p_y[slot] = 0;
  c.t->p_w[slot] = p.rect_w; c.t->p_h[slot] = p.rect_h; c.t->p_cw[slot] = 0; c.t->p_ci[slot] = 0;
  c.t->p_okey[slot] = pod_okey(c.fs[f], c.splits, ctr);
  c.t->p_sm[slot] = p.sm_eff;
  c.t->p_qlim[slot] = p.quota;
  c.t->p_qreq[slot] = has_qreq ? qreq : p.quota;
  c.t->p_qused[slot] = 0.0; c.t->p_busy[slot] = 0.0; c.t->p_invr[slot] = p.inv_rate;
  c.t->p_crem[slot] = 0.0; c.t->p_carr[slot] = 0.0; c.t->p_dur[slot] = 0.0;
  return slot;
}

__device__ void free_slot(Ctx& c, int slot) {  // lane 0
  c.t->p_flags[slot] = 0;
  c.t->s_free[c.sh->free_top++] = slot;
}

// sorted insert of a returned request id (queue order == id order)
__device__ void return_request(Ctx& c, int f, long long id) {  // lane 0
  int n = c.t->f_retn[f];
  if (n >= c.RET) { set_error(c, GS_ERR_CAPACITY, GS_CAP_RETURNED, f, 0); return; }
  long long* r = &c.t->f_ret[(size_t)f * c.RET];
  int i = n;
  #pragma unroll 1
  while (i > 0 && r[i - 1] > id) { r[i] = r[i - 1]; i--; }
  r[i] = id;
  c.t->f_retn[f] = n + 1;
}

// _remove_pod: sim_engine.py:377-392 (lane 0)
__device__ void remove_pod(Ctx& c, int slot) {
  int fl = c.t->p_flags[slot];
  if (fl & PF_RETRY) { free_slot(c, slot); return; }
  int f = c.t->p_fn[slot];
  if (fl & PF_CUR) {  // in-flight request restarts from scratch on another pod
    return_request(c, f, pack_id(c.t->p_cw[slot], c.t->p_ci[slot]));
    c.t->f_pinned[f]--;
  }
  int g = c.t->p_node[slot];
  int n = c.t->n_nfree[g];
  if (n >= c.R) { set_error(c, GS_ERR_CAPACITY, GS_CAP_RECTS, g, 0); return; }
  c.t->n_rect[g * c.R + n] = make_int4(c.t->p_x[slot], c.t->p_y[slot], c.t->p_w[slot], c.t->p_h[slot]);
  c.t->n_nfree[g] = n + 1;
  mem_remove(c, g, f);
  c.t->n_nplaced[g]--;
  free_slot(c, slot);
}

// place() (packer.py:245-261) after best_match chose (g, rect)
__device__ bool place_pod(Ctx& c, int slot, int g, int4 chosen) {
  int4 placed = make_int4(chosen.x, chosen.y, c.t->p_w[slot], c.t->p_h[slot]);
  int n = c.t->n_nfree[g];
  int nn = n;
  bool ok = carve(c, &c.t->n_rect[g * c.R], &nn, placed, c.R);
  if (!ok) {
    if (c.lane == 0) set_error(c, GS_ERR_CAPACITY, GS_CAP_RECTS, g, 0);
    __syncwarp();
    return false;
  }
  if (c.lane == 0) {
    c.t->n_nfree[g] = nn;
    mem_add(c, g, c.t->p_fn[slot]);
    c.t->n_nplaced[g]++;
    c.t->p_node[slot] = g;
    c.t->p_x[slot] = chosen.x;
    c.t->p_y[slot] = chosen.y;
    c.t->p_flags[slot] = (c.t->p_flags[slot] | PF_PLACED) & ~PF_RETRY;
  }
  __syncwarp();
  return true;
}

#ifdef GS_XL_TIMING
__device__ unsigned long long gs_xl_t[64];   // -DGS_XL_TIMING split (tools/xl_timing.py)
#define GS_EPOCH_TIC(v) const long long v = clock64()
#define GS_EPOCH_ADD(k, d) atomicAdd(&gs_xl_t[k], (unsigned long long)(d))
#else
#define GS_EPOCH_TIC(v)
#define GS_EPOCH_ADD(k, d)
#endif
// _place_batch: sim_engine.py:394-407.  Batch = every alive, unplaced pod
// (the retry list plus this epoch's additions); order (-area, pod_id).
__device__ void place_batch(Ctx& c) {
  int nb = 0;
  const int phi = pod_high(c);
  #pragma unroll 1
  for (int s = 0; s < phi; s += 32) {
    int slot = s + c.lane;
    bool take = slot < phi && (c.t->p_flags[slot] & (PF_ALIVE | PF_PLACED)) == PF_ALIVE;
    unsigned bal = __ballot_sync(FULL, take);
    if (take) {
      int i = nb + __popc(bal & ((1u << c.lane) - 1u));
      long long area = (long long)c.t->p_w[slot] * c.t->p_h[slot];
      c.t->s_ka[i] = ~(unsigned long long)area;   // descending area
      c.t->s_kd[i] = c.t->p_okey[slot];
      c.t->s_ki[i] = slot;
      c.t->p_flags[slot] &= ~PF_RETRY;
    }
    nb += __popc(bal);
  }
  __syncwarp();
  warp_sort(c, nb);
  // batch order + each entry's best_match inputs (function, w, h)
  #pragma unroll 1
  for (int i = c.lane; i < nb; i += 32) {
    const int slot = c.t->s_ki[i];
    c.t->s_batch[i] = slot;
    c.t->s_ka[i] = ((unsigned long long)(unsigned)c.t->p_w[slot] << 32) | (unsigned)c.t->p_h[slot];
    c.t->s_ki[i] = c.t->p_fn[slot];
  }
  __syncwarp();
  // best_match is a pure function of (node state, function, w, h): once a
  // request fails, the identical requests that follow it in the batch fail
  // too (nothing changes in between), so a whole run of them is settled at
  // once with the same counters (attempts, failures, rect scans, retry flag).
  int i = 0;
  #pragma unroll 1
  while (i < nb) {
    const int slot = c.t->s_batch[i];
    int4 chosen;
    const long long before = c.sh->rect_scans;
    GS_EPOCH_TIC(b0_);
    const int g = best_match(c, slot, &chosen);
    __syncwarp();
    GS_EPOCH_TIC(b1_);
    if (c.lane == 0) { GS_EPOCH_ADD(7, b1_ - b0_); }
    if (g >= 0) {
      if (c.lane == 0) c.sh->attempts++;
      if (!place_pod(c, slot, g, chosen)) return;
      i++;
      continue;
    }
    const long long scans = c.sh->rect_scans - before;
    const unsigned long long key_a = c.t->s_ka[i];
    const int key_f = c.t->s_ki[i];
    int j = nb;                                  // first later entry with another key
    #pragma unroll 1
    for (int k0 = i + 1; k0 < nb; k0 += 32) {
      const int k = k0 + c.lane;
      const bool differs = k < nb && (c.t->s_ka[k] != key_a || c.t->s_ki[k] != key_f);
      const unsigned bal = __ballot_sync(FULL, differs);
      if (bal) { j = k0 + __ffs(bal) - 1; break; }
    }
    #pragma unroll 1
    for (int k = i + c.lane; k < j; k += 32) c.t->p_flags[c.t->s_batch[k]] |= PF_RETRY;
    if (c.lane == 0) {
      const int len = j - i;
      c.sh->attempts += len;
      c.sh->win_failures += len;
      c.sh->rect_scans += scans * (len - 1);
    }
    __syncwarp();
    i = j;
  }
  __syncwarp();
}

// restructure: packer.py:290-320
__device__ void restructure(Ctx& c, int g) {
  if (c.t->n_nfree[g] <= c.sc->restructure_threshold) return;
  int np = 0;
  const int phi = pod_high(c);
  #pragma unroll 1
  for (int s = 0; s < phi; s += 32) {
    int slot = s + c.lane;
    bool take = slot < phi && (c.t->p_flags[slot] & PF_PLACED) && c.t->p_node[slot] == g;
    unsigned bal = __ballot_sync(FULL, take);
    if (take) {
      int i = np + __popc(bal & ((1u << c.lane) - 1u));
      long long area = (long long)c.t->p_w[slot] * c.t->p_h[slot];
      c.t->s_ka[i] = ~(unsigned long long)area;
      c.t->s_kd[i] = c.t->p_okey[slot];
      c.t->s_ki[i] = slot;
    }
    np += __popc(bal);
  }
  __syncwarp();
  warp_sort(c, np);
  #pragma unroll 1
  for (int i = c.lane; i < np; i += 32) c.t->s_list[i] = c.t->s_ki[i];
  int4* fr = c.t->s_rs;
  int* nfr = &c.sh->n_list;
  if (c.lane == 0) { fr[0] = make_int4(0, 0, c.sc->side_x, c.sc->side_y); *nfr = 1; }
  __syncwarp();
  #pragma unroll 1
  for (int i = 0; i < np; i++) {
    int slot = c.t->s_list[i];
    int w = c.t->p_w[slot], h = c.t->p_h[slot];
    int j = best_fit_in_list(c, fr, *nfr, w, h);
    if (j < 0) return;   // abort: node unchanged (packer.py:309-313)
    int4 t = fr[j];
    if (c.lane == 0) c.t->s_pos[i] = make_int2(t.x, t.y);
    __syncwarp();
    int nn = *nfr;
    if (!carve(c, fr, &nn, make_int4(t.x, t.y, w, h), c.R)) {
      if (c.lane == 0) set_error(c, GS_ERR_CAPACITY, GS_CAP_RECTS, g, 1);
      __syncwarp();
      return;
    }
    if (c.lane == 0) *nfr = nn;
    __syncwarp();
  }
  int nn = *nfr;
  #pragma unroll 1
  for (int j = c.lane; j < nn; j += 32) c.t->n_rect[g * c.R + j] = fr[j];
  #pragma unroll 1
  for (int i = c.lane; i < np; i += 32) {
    int slot = c.t->s_list[i];
    c.t->p_x[slot] = c.t->s_pos[i].x;
    c.t->p_y[slot] = c.t->s_pos[i].y;
  }
  if (c.lane == 0) c.t->n_nfree[g] = nn;
  __syncwarp();
}

// fragmentation index over all nodes' free rects (sim_engine.py:580-583)
__device__ void refresh_frag(Ctx& c) {
  long long total = 0, largest = -1;
  #pragma unroll 1
  for (int g = 0; g < c.G; g++) {
    int nf = c.t->n_nfree[g];
    #pragma unroll 1
    for (int j = c.lane; j < nf; j += 32) {
      long long a = r_area(c.t->n_rect[g * c.R + j]);
      total += a;
      largest = a > largest ? a : largest;
    }
  }
  total = warp_sum_ll(total);
  largest = warp_max_ll(largest);
  if (c.lane == 0)
    c.sh->frag = (total == 0 || largest < 0) ? 0.0 : (double)(total - largest) / (double)total;
  __syncwarp();
}

// ----------------------------------------------------------------------------
// epoch: _run_epoch (sim_engine.py:409-430), autoscaler.py:81-160
// ----------------------------------------------------------------------------
// register bitonic sort of one (a, b, v) triple per lane, ascending over the
// first n lanes (n <= 32); lanes >= n must hold (~0, ~0, INT_MAX)
__device__ __forceinline__ void warp_sort_regs(unsigned long long& a, unsigned long long& b,
                                               int& v, int n, int lane) {
  int q = 1;
  #pragma unroll 1
  while (q < n) q <<= 1;
  #pragma unroll 1
  for (int k = 2; k <= q; k <<= 1) {
    #pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      const unsigned long long oa = __shfl_xor_sync(FULL, a, j);
      const unsigned long long ob = __shfl_xor_sync(FULL, b, j);
      const int ov = __shfl_xor_sync(FULL, v, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      const bool other_less = trip_less(oa, ob, ov, a, b, v);
      const bool take = lower == up ? other_less : !other_less && !(oa == a && ob == b && ov == v);
      if (take) { a = oa; b = ob; v = ov; }
    }
  }
}

// alive pods grouped by function, slot order inside a group:
// s_list[f_loff[f] .. f_loff[f+1]).  (f_loff is scratch until window_begin.)
__device__ void group_alive_by_fn(Ctx& c) {
  const int phi = pod_high(c);
  int* off = c.t->f_loff;
  int* cur = c.t->s_fcur;
  #pragma unroll 1
  for (int f = c.lane; f <= c.F; f += 32) cur[f] = 0;
  __syncwarp();
  #pragma unroll 1
  for (int s0 = 0; s0 < phi; s0 += 32) {
    const int slot = s0 + c.lane;
    const int fn = (slot < phi && (c.t->p_flags[slot] & PF_ALIVE)) ? c.t->p_fn[slot] : -1;
    const unsigned m = __match_any_sync(FULL, fn);
    if (fn >= 0 && c.lane == __ffs(m) - 1) atomicAdd(&cur[fn], __popc(m));
  }
  __syncwarp();
  if (c.lane == 0) {                       // exclusive scan (F is small)
    int acc = 0;
    #pragma unroll 1
    for (int f = 0; f < c.F; f++) { off[f] = acc; const int n = cur[f]; cur[f] = acc; acc += n; }
    off[c.F] = acc;
  }
  __syncwarp();
  #pragma unroll 1
  for (int s0 = 0; s0 < phi; s0 += 32) {
    const int slot = s0 + c.lane;
    const int fn = (slot < phi && (c.t->p_flags[slot] & PF_ALIVE)) ? c.t->p_fn[slot] : -1;
    const unsigned m = __match_any_sync(FULL, fn);
    if (fn >= 0) {
      const int pos = cur[fn] + __popc(m & ((1u << c.lane) - 1u));
      c.t->s_list[pos] = slot;
    }
    __syncwarp();
    if (fn >= 0 && c.lane == __ffs(m) - 1) cur[fn] += __popc(m);
    __syncwarp();
  }
}

// scale_up's p_ideal (autoscaler.py:120-126): argmin over points with T > r of
// (T - r, area, sm, quota); points are distinct in (sm, quota), so the
// reference's first-strict-minimum is the unique lexicographic minimum.
__device__ int ideal_point(const Ctx& c, int f, double residual) {
  const gs_function_t& fs = c.fs[f];
  double k0 = 0, k1 = 0, k2 = 0, k3 = 0;
  int idx = -1;
  #pragma unroll 1
  for (int k = c.lane; k < fs.n_points; k += 32) {
    const gs_point_t& p = c.pt(f, k);
    if (!(p.thr > residual)) continue;
    const double d = p.thr - residual;
    if (idx < 0 || d < k0 || (d == k0 && (p.area < k1 || (p.area == k1 &&
        (p.sm < k2 || (p.sm == k2 && p.quota < k3)))))) {
      k0 = d; k1 = p.area; k2 = p.sm; k3 = p.quota; idx = k;
    }
  }
#pragma unroll 1
  for (int o = 16; o > 0; o >>= 1) {
    const double y0 = __shfl_xor_sync(FULL, k0, o), y1 = __shfl_xor_sync(FULL, k1, o);
    const double y2 = __shfl_xor_sync(FULL, k2, o), y3 = __shfl_xor_sync(FULL, k3, o);
    const int yi = __shfl_xor_sync(FULL, idx, o);
    bool take;
    if (yi < 0) take = false;
    else if (idx < 0) take = true;
    else take = y0 < k0 || (y0 == k0 && (y1 < k1 || (y1 == k1 && (y2 < k2 || (y2 == k2 &&
                (y3 < k3 || (y3 == k3 && yi < idx)))))));
    if (take) { k0 = y0; k1 = y1; k2 = y2; k3 = y3; idx = yi; }
  }
  return idx;
}

// ----------------------------------------------------------------------------
// epoch: _run_epoch (sim_engine.py:409-430), autoscaler.py:81-160
// ----------------------------------------------------------------------------
__device__ void run_epoch(Ctx& c, int w) {
  GS_EPOCH_TIC(e0_);
  group_alive_by_fn(c);
  #pragma unroll 1
  for (int f = 0; f < c.F; f++) {
    // running set of f: placed pods + retry pods (sim_engine.py:370-375),
    // ordered by (efficiency, pod_id) (autoscaler.py:50-51); T in that order
    const int start = c.t->f_loff[f];
    const int n = c.t->f_loff[f + 1] - start;
    double thr = 0.0;                       // lane i: T of the i-th running pod (n <= 32)
    PySum sup;
    sup.reset();
    if (n <= 32) {
      unsigned long long a = ~0ull, b = ~0ull;
      int v = 0x7fffffff;
      if (c.lane < n) {
        const int slot = c.t->s_list[start + c.lane];
        a = ord_key(c.pt(f, c.t->p_pt[slot]).rpr);
        b = c.t->p_okey[slot];
        v = slot;
      }
      warp_sort_regs(a, b, v, n, c.lane);
      if (c.lane < n) {
        thr = c.pt(f, c.t->p_pt[v]).thr;
        c.t->s_ki[c.lane] = v;
      }
      #pragma unroll 1
      for (int i = 0; i < n; i++) sup.add(__shfl_sync(FULL, thr, i));   // same in every lane
      __syncwarp();
    } else {
      #pragma unroll 1
      for (int i = c.lane; i < n; i += 32) {
        const int slot = c.t->s_list[start + i];
        c.t->s_ka[i] = ord_key(c.pt(f, c.t->p_pt[slot]).rpr);
        c.t->s_kd[i] = c.t->p_okey[slot];
        c.t->s_ki[i] = slot;
      }
      __syncwarp();
      warp_sort(c, n);
      #pragma unroll 1
      for (int i = 0; i < n; i++) sup.add(c.pt(f, c.t->p_pt[c.t->s_ki[i]]).thr);
    }
    const int hn = c.t->f_hn[f];
    const double* h = &c.t->f_hist[3 * f];
    double pred = h[(hn - 1) % 3];            // max(history[-3:])
    #pragma unroll 1
    for (int k = 2; k <= 3 && k <= hn; k++) {
      const double x = h[(hn - k) % 3];
      if (x > pred) pred = x;
    }
    const double gap = pred - sup.value();    // rps_gap
    if (gap > 0) {                            // scale_up: autoscaler.py:103-131
      const gs_function_t& fs = c.fs[f];
      const int pe = fs.p_eff;
      const double t_eff = c.pt(f, pe).thr;
      if (!(t_eff > 0)) {                     // autoscaler.py:115-117
        if (c.lane == 0) set_error(c, GS_ERR_VALIDATION, GS_VAL_NO_THROUGHPUT, f, pe);
        return;
      }
      const double nd = floor(gap / t_eff);
      const double residual = gap - nd * t_eff;
      const long long cnt = (long long)nd;
      int ideal = -1;
      if (residual > 0) {
        ideal = ideal_point(c, f, residual);
        if (ideal < 0) ideal = pe;
      }
      if (c.lane == 0) {
        const long long total = cnt + (ideal >= 0 ? 1 : 0);
        c.sh->decisions += total;
        if (total > c.P) {
          set_error(c, GS_ERR_CAPACITY, GS_CAP_PODS, c.P, 1);
        } else {
          #pragma unroll 1
          for (long long i = 0; i < total; i++) {
            const int k = i < cnt ? pe : ideal;
            if (make_pod(c, f, k, 0, 0.0, w + c.sc->cold_start_windows) < 0) break;
          }
        }
      }
    } else if (gap < 0) {                     // scale_down: autoscaler.py:134-149
      double delta = gap;
      #pragma unroll 1
      for (int i = 0; i < n && delta < 0; i++) {
        const double t = n <= 32 ? __shfl_sync(FULL, thr, i)
                                 : c.pt(f, c.t->p_pt[c.t->s_ki[i]]).thr;
        if (delta + t > 0) break;
        delta += t;
        if (c.lane == 0) {
          c.sh->decisions++;
          remove_pod(c, c.t->s_ki[i]);
        }
        if (failed(c)) break;
      }
    }
    if (failed(c)) return;
  }
  GS_EPOCH_TIC(e1_);
  place_batch(c);
  GS_EPOCH_TIC(e2_);
  if (failed(c)) return;
  #pragma unroll 1
  for (int g = 0; g < c.G; g++) {
    restructure(c, g);
    if (failed(c)) return;
  }
  refresh_frag(c);
  GS_EPOCH_TIC(e3_);
  if (c.lane == 0) { GS_EPOCH_ADD(4, e1_ - e0_); GS_EPOCH_ADD(5, e2_ - e1_); GS_EPOCH_ADD(6, e3_ - e2_); }
}

// ----------------------------------------------------------------------------
// window begin: _warm_up, reset_window, _generate_arrivals (sim_engine.py:446-449)
// and the per-window pod lists
// ----------------------------------------------------------------------------
__device__ void window_begin(Ctx& c, int w) {
  int next_warm = 0x7fffffff;
  const int phi = pod_high(c);
  #pragma unroll 1
  for (int slot = c.lane; slot < phi; slot += 32) {
    int fl = c.t->p_flags[slot];
    if ((fl & PF_PLACED) && !(fl & PF_REG)) {
      if (c.t->p_warm[slot] <= w) fl |= PF_REG;
      else next_warm = min(next_warm, c.t->p_warm[slot]);
    }
    if (fl & PF_REG) { c.t->p_qused[slot] = 0.0; fl &= ~PF_GRANT; }
    c.t->p_flags[slot] = fl;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) next_warm = min(next_warm, __shfl_xor_sync(FULL, next_warm, o));
  if (c.lane == 0) c.sh->next_warm = next_warm;
  #pragma unroll 1
  for (int f = c.lane; f < c.F; f += 32) {
    int n = c.count(f, w);
    c.t->f_warr[f] = n;
    if (n > 0) {
      if (c.t->f_fn[f] == 0) { c.t->f_fw[f] = w; c.t->f_fi[f] = 0; }
      c.t->f_fn[f] += n;
    }
  }
  __syncwarp();
  // registered pods ordered by (node, pod_id)
  int nr = 0;
  #pragma unroll 1
  for (int s = 0; s < phi; s += 32) {
    int slot = s + c.lane;
    bool take = slot < phi && (c.t->p_flags[slot] & PF_REG);
    unsigned bal = __ballot_sync(FULL, take);
    if (take) {
      int i = nr + __popc(bal & ((1u << c.lane) - 1u));
      c.t->s_ka[i] = (unsigned long long)c.t->p_node[slot];
      c.t->s_kd[i] = c.t->p_okey[slot];
      c.t->s_ki[i] = slot;
    }
    nr += __popc(bal);
  }
  __syncwarp();
  warp_sort(c, nr);
  #pragma unroll 1
  for (int i = c.lane; i < nr; i += 32) c.t->s_rl[i] = c.t->s_ki[i];
  // node segments
  #pragma unroll 1
  for (int g = c.lane; g <= c.G; g += 32) {
    // lower bound of node g in the sorted keys
    int lo = 0, hi = nr;
    #pragma unroll 1
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if ((int)c.t->s_ka[mid] < g) lo = mid + 1; else hi = mid;
    }
    c.t->n_seg[g] = lo;
  }
  __syncwarp();
  // per-function lists in (node, pod_id) order: stable counting sort,
  // warp-parallel (match_any groups lanes of one function)
  int* cur = c.t->s_fcur;
  #pragma unroll 1
  for (int f = c.lane; f <= c.F; f += 32) cur[f] = 0;
  if (c.lane == 0) {
    c.sh->n_reg = nr;
    c.sh->pod_steps += (long long)nr * c.T;
  }
  __syncwarp();
  #pragma unroll 1
  for (int i0 = 0; i0 < nr; i0 += 32) {
    const int i = i0 + c.lane;
    const int fn = i < nr ? c.t->p_fn[c.t->s_rl[i]] : -1;
    const unsigned m = __match_any_sync(FULL, fn);
    if (fn >= 0 && c.lane == __ffs(m) - 1) atomicAdd(&cur[fn], __popc(m));
  }
  __syncwarp();
  if (c.lane == 0) {
    int acc = 0;
    #pragma unroll 1
    for (int f = 0; f < c.F; f++) { c.t->f_loff[f] = acc; const int k = cur[f]; cur[f] = acc; acc += k; }
    c.t->f_loff[c.F] = acc;
  }
  __syncwarp();
  #pragma unroll 1
  for (int i0 = 0; i0 < nr; i0 += 32) {
    const int i = i0 + c.lane;
    const int slot = i < nr ? c.t->s_rl[i] : -1;
    const int fn = slot >= 0 ? c.t->p_fn[slot] : -1;
    const unsigned m = __match_any_sync(FULL, fn);
    if (fn >= 0) c.t->s_fl[cur[fn] + __popc(m & ((1u << c.lane) - 1u))] = slot;
    __syncwarp();
    if (fn >= 0 && c.lane == __ffs(m) - 1) cur[fn] += __popc(m);
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------
// per-request helpers on the arena (the XL class's quantum steps, gs_xl.cuh)
// ----------------------------------------------------------------------------
__device__ void admit_arrivals(Ctx& c, int f, double t0) {  // sim_engine.py:472-480
  int fn = c.t->f_fn[f];
  if (fn == 0) return;
  int w = c.t->f_fw[f], i = c.t->f_fi[f];
  int limit = c.fs[f].max_queue;
  int qlen = c.t->f_qlen[f], nsn = c.t->f_nsn[f];
  int drop = 0;
  double now = t0 + TIME_EPS;
  #pragma unroll 1
  while (fn > 0 && arrival_time(c, f, w, i) <= now) {
    int aw = w, ai = i;
    fn--;
    if (fn > 0) advance_id(c, f, w, i);
    if (limit >= 0 && qlen >= limit) { drop++; continue; }
    qlen++;
    if (limit < 0) {
      if (nsn == 0) { c.t->f_nsw[f] = aw; c.t->f_nsi[f] = ai; }
    } else {
      int cap = limit;
      c.t->f_ring[c.t->f_ringoff[f] + (c.t->f_rhead[f] + nsn) % cap] = pack_id(aw, ai);
    }
    nsn++;
  }
  c.t->f_fn[f] = fn; c.t->f_fw[f] = w; c.t->f_fi[f] = i;
  c.t->f_qlen[f] = qlen; c.t->f_nsn[f] = nsn;
  c.t->f_wdrop[f] += drop;
}

// _serve: sim_engine.py:525-552
__device__ void serve(Ctx& c, int slot, double t_start, double t_end) {
  int f = c.t->p_fn[slot];
  int fl = c.t->p_flags[slot];
  double busy = c.t->p_busy[slot];
  double t = busy > t_start ? busy : t_start;
  if (!(t < t_end - TIME_EPS)) { c.t->p_busy[slot] = t; return; }
  double rem = c.t->p_crem[slot], arr = c.t->p_carr[slot];
  double slo = c.fs[f].slo_ms;
  int comp = 0, viol = 0;
  #pragma unroll 1
  while (t < t_end - TIME_EPS) {
    if (!(fl & PF_CUR)) {
      long long id;
      int retn = c.t->f_retn[f];
      int nsn = c.t->f_nsn[f];
      if (retn > 0) {
        long long* r = &c.t->f_ret[(size_t)f * c.RET];
        id = r[0];
        #pragma unroll 1
        for (int k = 1; k < retn; k++) r[k - 1] = r[k];
        c.t->f_retn[f] = retn - 1;
      } else if (nsn > 0) {
        int limit = c.fs[f].max_queue;
        if (limit < 0) {
          int nw = c.t->f_nsw[f], ni = c.t->f_nsi[f];
          id = pack_id(nw, ni);
          if (nsn > 1) { advance_id(c, f, nw, ni); c.t->f_nsw[f] = nw; c.t->f_nsi[f] = ni; }
        } else {
          int h = c.t->f_rhead[f];
          id = c.t->f_ring[c.t->f_ringoff[f] + h];
          c.t->f_rhead[f] = (h + 1) % limit;
        }
        c.t->f_nsn[f] = nsn - 1;
      } else {
        break;
      }
      c.t->f_pinned[f]++;
      fl |= PF_CUR;
      rem = c.t->p_invr[slot];
      arr = arrival_time(c, f, id_w(id), id_i(id));
      c.t->p_cw[slot] = id_w(id);
      c.t->p_ci[slot] = id_i(id);
    }
    double left = t_end - t;
    double span = rem < left ? rem : left;
    rem -= span;
    t += span;
    if (rem <= TIME_EPS) {
      c.t->f_qlen[f]--;
      c.t->f_pinned[f]--;
      fl &= ~PF_CUR;
      comp++;
      if ((t - arr) * 1000.0 > slo) viol++;
    }
  }
  c.t->p_busy[slot] = t;
  c.t->p_crem[slot] = rem;
  c.t->p_carr[slot] = arr;
  c.t->p_flags[slot] = fl;
  c.t->f_wcomp[f] += comp;
  c.t->f_wviol[f] += viol;
}

// ----------------------------------------------------------------------------
// warp-level quantum step on the arena: the fallback for a window whose
// registered set outgrows the run's shared-memory class (sim_engine.py:493-520)
// ----------------------------------------------------------------------------
__device__ void complete_tokens(Ctx& c) {  // _complete_live_tokens (sim_engine.py:482-486)
  int n = c.sh->n_reg;
  if (!c.integral()) {
    // sm_running -= sm in token order per node, with the float-dust clamp
    #pragma unroll 1
    for (int g = c.lane; g < c.G; g += 32) {
      double sr = c.t->n_sr[g];
      #pragma unroll 1
      for (int j = c.t->n_seg[g]; j < c.t->n_seg[g + 1]; j++) {
        int slot = c.t->s_rl[c.t->s_ki[j]];
        if (!(c.t->p_flags[slot] & PF_GRANT)) break;
        sr -= c.t->p_sm[slot];
        if (sr < 0 && sr > -SM_EPS) sr = 0.0;
      }
      c.t->n_sr[g] = sr;
    }
    __syncwarp();
  }
  #pragma unroll 1
  for (int i = c.lane; i < n; i += 32) {
    int slot = c.t->s_rl[i];
    int fl = c.t->p_flags[slot];
    if (fl & PF_GRANT) {
      c.t->p_qused[slot] += c.t->p_dur[slot];
      c.t->p_flags[slot] = fl & ~PF_GRANT;
    }
  }
  __syncwarp();
}

__device__ void run_step(Ctx& c, int w, int s) {
  const double t0 = (double)w * c.ws + (double)s * c.qs;
  if (s > 0) complete_tokens(c);   // step 0: window_begin already reset the ledger
  #pragma unroll 1
  for (int f = c.lane; f < c.F; f += 32) admit_arrivals(c, f, t0);
  __syncwarp();
  // filter_pods + requesting + build_queue keys
  const int n = c.sh->n_reg;
  #pragma unroll 1
  for (int i = c.lane; i < n; i += 32) {
    int slot = c.t->s_rl[i];
    int fl = c.t->p_flags[slot];
    double qused = c.t->p_qused[slot];
    bool cand = !(c.t->p_qlim[slot] - qused <= QUOTA_EPS);
    int f = c.t->p_fn[slot];
    bool req = cand && ((fl & PF_CUR) || (c.t->f_qlen[f] - c.t->f_pinned[f] > 0));
    c.t->s_ka[i] = ((unsigned long long)c.t->p_node[slot] << 1) | (req ? 0ull : 1ull);
    c.t->s_kd[i] = req ? ord_key(-(c.t->p_qreq[slot] - qused)) : 0ull;
    c.t->s_ki[i] = i;
  }
  __syncwarp();
  warp_sort(c, n);
  // dispatch (head-blocking) + coverage/occupancy, one lane per node
  int grants = 0;
  #pragma unroll 1
  for (int g = c.lane; g < c.G; g += 32) {
    double sr = c.integral() ? 0.0 : c.t->n_sr[g];
    double mx = 0.0;
    PySum occ;
    occ.reset();
    int ng = 0;
    #pragma unroll 1
    for (int j = c.t->n_seg[g]; j < c.t->n_seg[g + 1]; j++) {
      if (c.t->s_ka[j] & 1ull) break;           // rest of the node is not requesting
      int slot = c.t->s_rl[c.t->s_ki[j]];
      double sm = c.t->p_sm[slot];
      if (sm + sr > SM_LIMIT + SM_EPS) break;
      double rem = c.t->p_qlim[slot] - c.t->p_qused[slot];
      double dur = rem < c.quantum ? rem : c.quantum;
      c.t->p_dur[slot] = dur;
      c.t->p_flags[slot] |= PF_GRANT;
      sr += sm;
      if (ng == 0 || dur > mx) mx = dur;
      occ.add(sm * dur);
      ng++;
    }
    if (!c.integral()) c.t->n_sr[g] = sr;
    if (ng) {
      c.t->n_cov[g] += mx;
      c.t->n_occ[g] += occ.value() / 100.0;
    }
    grants += ng;
  }
  grants = warp_sum_i(grants);
  if (c.lane == 0) c.sh->grants += grants;
  __syncwarp();
  // serve, per function in (node, pod_id) order
  #pragma unroll 1
  for (int f = c.lane; f < c.F; f += 32) {
    #pragma unroll 1
    for (int j = c.t->f_loff[f]; j < c.t->f_loff[f + 1]; j++) {
      int slot = c.t->s_fl[j];
      if (c.t->p_flags[slot] & PF_GRANT) serve(c, slot, t0, t0 + c.t->p_dur[slot] * c.ws);
    }
  }
  __syncwarp();
}


}  // namespace gs
