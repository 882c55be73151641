/*
 * gs_oracle.c -- CPU ORACLE for the FaST-GShare simulator hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline -- never as the product path.
 *
 * A deliberately literal C restatement of the reference's pure-Python engine
 * (pkg/src/gshare_sim, commit mounted at /root/reference):
 *   - explicit request objects and FIFO lists, exactly as sim_engine.py keeps
 *     them (no closed-form arrival cursors, unlike the CUDA kernel);
 *   - real pod-id strings "fid-%04d" compared with strcmp (no rank tricks);
 *   - Python's evaluation order for every floating-point expression, built
 *     with -ffp-contract=off so no FMA can change a rounding.
 * Each function cites the reference lines it restates.  It consumes the same
 * gs_batch_t as the CUDA library, so GPU-vs-oracle parity compares identical
 * inputs; the oracle itself is pinned to the real reference through the
 * golden fixtures in tests/golden/ (make_golden.py imports the reference).
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/gshare_b200.h"

#define TIME_EPS 1e-12  /* sim_engine.py:75 */
#define QUOTA_EPS 1e-9  /* token_backend.py:25 */
#define SM_EPS 1e-9     /* token_backend.py:26 */
#define SM_LIMIT 100.0  /* token_backend.py:18 */

typedef struct { double arrival; int server; } Req; /* server: pod slot or -1 */

typedef struct {
  Req* q; int qhead, qn, qcap;          /* fn.queue  (sim_engine.py:281) */
  double* fut; int fhead, fn_, fcap;    /* fn.future (sim_engine.py:282) */
  int pinned;
  double* hist; int nhist;
  int pod_counter;
  int win_arr, win_comp, win_viol, win_drop;
} Fn;

typedef struct {
  int alive, fn, point, counter;
  char id[160];
  double sm, q_req, q_lim;              /* ResourceConfig */
  long long rw, rh;                      /* PodRequest w,h (scaled) */
  double inv_rate;
  int gpu, warm_at, registered, in_retry;
  double q_used, busy_until;
  int has_cur; double cur_rem, cur_arr;
  long long x, y;                        /* placement rect origin */
} Pod;

typedef struct { long long x, y, w, h; } Rect;
typedef struct { int pod; double sm, dur; } Token;

typedef struct {
  Rect* fr; int nfr, cfr;                /* free_rects list, Python order */
  int* res_fn; int* res_cnt; int nres;   /* GpuMemoryState.resident (insertion order) */
  int nplaced;
  double sm_running;
  Token* live; int nlive, clive;
  double cov, occ;
} Node;

typedef struct {
  const gs_batch_t* in;
  const gs_scenario_t* sc;
  const gs_function_t* fs;
  int G, F;
  Fn* fn;
  Pod* pods; int npods, cpods;
  Node* nodes;
  int* retry; int nretry, cretry;
  int win_failures;
  long long grants, decisions, attempts, pod_steps, rect_scans, peak_pods;
  int err_code, err_detail, err_fn, err_pt;
} Eng;

/* ------------------------------------------------------------------ utils */
static void* xrealloc(void* p, size_t n) {
  void* r = realloc(p, n ? n : 1);
  if (!r) { fprintf(stderr, "gs_oracle: out of memory\n"); abort(); }
  return r;
}
#define GROW(ptr, n, cap, extra) do { if ((n) + (extra) > (cap)) { \
  (cap) = ((n) + (extra)) * 2 + 8; (ptr) = xrealloc((ptr), sizeof(*(ptr)) * (size_t)(cap)); } } while (0)

static const gs_point_t* PT(const Eng* e, int f, int k) {
  return &e->in->points[e->fs[f].point_off + k];
}

/* Python 3.12's builtin sum() over floats (this image's interpreter): the
 * start value int 0 is absorbed by the first item, every further item goes
 * through Neumaier's compensated update, and the compensation is added once
 * at the end (CPython Python/bltinmodule.c builtin_sum_impl).  The reference
 * calls sum() in rps_gap (autoscaler.py:87) and for SM occupancy
 * (sim_engine.py:516-517); a plain loop would round differently. */
typedef struct { double f, c; int n; } PySum;
static void pysum_add(PySum* s, double x) {
  if (s->n++ == 0) { s->f = 0.0 + x; s->c = 0.0; return; }
  double t = s->f + x;
  if (fabs(s->f) >= fabs(x)) s->c += (s->f - t) + x;
  else s->c += (x - t) + s->f;
  s->f = t;
}
static double pysum_value(const PySum* s) {
  if (s->n == 0) return 0.0;
  double f = s->f;
  if (s->c != 0.0 && isfinite(s->c)) f += s->c;
  return f;
}

/* ---------------------------------------------------------- memory model */
/* footprint(): memory_model.py:61-74 -- sum in resident insertion order */
static double footprint(const Eng* e, const Node* n) {
  double total = 0.0;
  for (int i = 0; i < n->nres; i++) {
    int c = n->res_cnt[i];
    if (c <= 0) continue;
    const gs_function_t* f = &e->fs[n->res_fn[i]];
    if (e->sc->flags & GS_FLAG_SHARING) total += f->mem_server_mb + (double)c * f->mem_runtime_mb;
    else total += (double)c * f->mem_noshare_mb;
  }
  return total;
}
static int resident_count(const Node* n, int fn) {
  for (int i = 0; i < n->nres; i++) if (n->res_fn[i] == fn) return n->res_cnt[i];
  return 0;
}
/* admit(): memory_model.py:77-88 */
static int admit(const Eng* e, const Node* n, int fn) {
  const gs_function_t* f = &e->fs[fn];
  double delta;
  if (e->sc->flags & GS_FLAG_SHARING) {
    delta = f->mem_runtime_mb;
    if (resident_count(n, fn) <= 0) delta += f->mem_server_mb;
  } else {
    delta = f->mem_noshare_mb;
  }
  return footprint(e, n) + delta <= e->sc->capacity_mb;
}
static void mem_add(Node* n, int fn) {          /* memory_model.py:48-49 */
  for (int i = 0; i < n->nres; i++) if (n->res_fn[i] == fn) { n->res_cnt[i]++; return; }
  n->res_fn[n->nres] = fn; n->res_cnt[n->nres] = 1; n->nres++;
}
static void mem_remove(Node* n, int fn) {       /* memory_model.py:51-58 */
  for (int i = 0; i < n->nres; i++) if (n->res_fn[i] == fn) {
    if (n->res_cnt[i] == 1) {                   /* del resident[fid]: order of the rest kept */
      memmove(&n->res_fn[i], &n->res_fn[i + 1], sizeof(int) * (size_t)(n->nres - i - 1));
      memmove(&n->res_cnt[i], &n->res_cnt[i + 1], sizeof(int) * (size_t)(n->nres - i - 1));
      n->nres--;
    } else {
      n->res_cnt[i]--;
    }
    return;
  }
}

/* ------------------------------------------------------------------ packer */
static int r_contains(Rect a, Rect b) {          /* packer.py:77-79 */
  return b.x >= a.x && b.y >= a.y && b.x + b.w <= a.x + a.w && b.y + b.h <= a.y + a.h;
}
static int r_intersects(Rect a, Rect b) {        /* packer.py:81-84 */
  return a.x < b.x + b.w && b.x < a.x + a.w && a.y < b.y + b.h && b.y < a.y + a.h;
}
static int r_eq(Rect a, Rect b) { return a.x == b.x && a.y == b.y && a.w == b.w && a.h == b.h; }

/* _subdivide + _carve + _prune_contained: packer.py:196-242 */
static void carve(Rect** list, int* n, int* cap, Rect placed) {
  int m = 0, mc = *n * 4 + 4;
  Rect* out = xrealloc(NULL, sizeof(Rect) * (size_t)mc);
  for (int i = 0; i < *n; i++) {
    Rect r = (*list)[i];
    if (!r_intersects(r, placed)) { out[m++] = r; continue; }
    long long ix = r.x > placed.x ? r.x : placed.x;
    long long iy = r.y > placed.y ? r.y : placed.y;
    long long ix2 = (r.x + r.w) < (placed.x + placed.w) ? (r.x + r.w) : (placed.x + placed.w);
    long long iy2 = (r.y + r.h) < (placed.y + placed.h) ? (r.y + r.h) : (placed.y + placed.h);
    if (ix > r.x) out[m++] = (Rect){r.x, r.y, ix - r.x, r.h};
    if (ix2 < r.x + r.w) out[m++] = (Rect){ix2, r.y, r.x + r.w - ix2, r.h};
    if (iy > r.y) out[m++] = (Rect){r.x, r.y, r.w, iy - r.y};
    if (iy2 < r.y + r.h) out[m++] = (Rect){r.x, iy2, r.w, r.y + r.h - iy2};
  }
  int k = 0;
  GROW(*list, 0, *cap, m);
  for (int i = 0; i < m; i++) {
    int redundant = 0;
    for (int j = 0; j < m; j++) {
      if (i == j || !r_contains(out[j], out[i])) continue;
      if (r_eq(out[i], out[j]) && i < j) continue;
      redundant = 1;
      break;
    }
    if (!redundant) (*list)[k++] = out[i];
  }
  *n = k;
  free(out);
}

/* best_match: packer.py:169-193 (nodes are already in gpu_id order) */
static int best_match(const Eng* e, const Pod* p, int* out_node, Rect* out_rect) {
  int found = 0;
  long long bk0 = 0, bk2 = 0, bk3 = 0; int bk1 = 0;
  long long rarea = p->rw * p->rh;
  for (int g = 0; g < e->G; g++) {
    const Node* n = &e->nodes[g];
    if (!admit(e, n, p->fn)) continue;
    ((Eng*)e)->rect_scans += n->nfr;
    for (int i = 0; i < n->nfr; i++) {
      Rect r = n->fr[i];
      if (p->rw <= r.w && p->rh <= r.h) {
        long long k0 = r.w * r.h - rarea;
        int lt = !found || k0 < bk0 || (k0 == bk0 && (g < bk1 || (g == bk1 &&
                 (r.y < bk2 || (r.y == bk2 && r.x < bk3)))));
        if (lt) { found = 1; bk0 = k0; bk1 = g; bk2 = r.y; bk3 = r.x; *out_node = g; *out_rect = r; }
      }
    }
  }
  return found;
}

/* _best_fit_in_node: packer.py:278-287 */
static int best_fit_in_node(const Rect* fr, int n, long long w, long long h, Rect* out) {
  int found = 0; long long b0 = 0, b1 = 0, b2 = 0;
  for (int i = 0; i < n; i++) {
    Rect r = fr[i];
    if (w <= r.w && h <= r.h) {
      long long k0 = r.w * r.h - w * h;
      if (!found || k0 < b0 || (k0 == b0 && (r.y < b1 || (r.y == b1 && r.x < b2)))) {
        found = 1; b0 = k0; b1 = r.y; b2 = r.x; *out = r;
      }
    }
  }
  return found;
}

static _Thread_local const Eng* g_sort_eng;
static int cmp_restructure(const void* a, const void* b) {  /* (-area, pod_id): packer.py:302-303 */
  const Pod* pa = &g_sort_eng->pods[*(const int*)a];
  const Pod* pb = &g_sort_eng->pods[*(const int*)b];
  long long aa = pa->rw * pa->rh, ab = pb->rw * pb->rh;
  if (aa != ab) return aa > ab ? -1 : 1;
  return strcmp(pa->id, pb->id);
}

/* restructure: packer.py:290-320 */
static void restructure(Eng* e, int g) {
  Node* n = &e->nodes[g];
  if (n->nfr <= e->sc->restructure_threshold) return;
  int* order = xrealloc(NULL, sizeof(int) * (size_t)(n->nplaced + 1));
  int k = 0;
  for (int i = 0; i < e->npods; i++)
    if (e->pods[i].alive && !e->pods[i].in_retry && e->pods[i].gpu == g) order[k++] = i;
  g_sort_eng = e;
  qsort(order, (size_t)k, sizeof(int), cmp_restructure);
  int cap = 8, nf = 1;
  Rect* fr = xrealloc(NULL, sizeof(Rect) * (size_t)cap);
  fr[0] = (Rect){0, 0, e->sc->side_x, e->sc->side_y};
  long long* nx = xrealloc(NULL, sizeof(long long) * (size_t)(k + 1));
  long long* ny = xrealloc(NULL, sizeof(long long) * (size_t)(k + 1));
  for (int i = 0; i < k; i++) {
    Pod* p = &e->pods[order[i]];
    Rect t;
    if (!best_fit_in_node(fr, nf, p->rw, p->rh, &t)) {   /* abort: node unchanged */
      free(fr); free(order); free(nx); free(ny);
      return;
    }
    nx[i] = t.x; ny[i] = t.y;
    carve(&fr, &nf, &cap, (Rect){t.x, t.y, p->rw, p->rh});
  }
  for (int i = 0; i < k; i++) { e->pods[order[i]].x = nx[i]; e->pods[order[i]].y = ny[i]; }
  free(n->fr);
  n->fr = fr; n->nfr = nf; n->cfr = cap;
  free(order); free(nx); free(ny);
}

/* ---------------------------------------------------------------- pods */
/* _make_pod: sim_engine.py:352-366 */
static int make_pod(Eng* e, int f, int k, int has_qreq, double q_req, int warm_at) {
  const gs_point_t* pt = PT(e, f, k);
  if (!pt->rate_ok) {               /* _service_rate raises ValidationError, :346-349 */
    if (!e->err_code) { e->err_code = GS_ERR_VALIDATION; e->err_fn = f; e->err_pt = k; }
    return -1;
  }
  int slot = -1;
  for (int i = 0; i < e->npods; i++) if (!e->pods[i].alive) { slot = i; break; }
  if (slot < 0) { GROW(e->pods, e->npods, e->cpods, 1); slot = e->npods++; }
  Pod* p = &e->pods[slot];
  memset(p, 0, sizeof(*p));
  Fn* fn = &e->fn[f];
  const gs_function_t* fs = &e->fs[f];
  p->alive = 1; p->fn = f; p->point = k; p->counter = fn->pod_counter++;
  snprintf(p->id, sizeof(p->id), "%.*s-%04d", fs->name_len, e->in->names + fs->name_off, p->counter);
  p->sm = pt->sm_eff;
  p->q_lim = pt->quota;
  p->q_req = has_qreq ? q_req : pt->quota;
  p->rw = pt->rect_w; p->rh = pt->rect_h;
  p->inv_rate = pt->inv_rate;
  p->gpu = -1; p->warm_at = warm_at;
  {
    long long alive = 0;
    for (int i = 0; i < e->npods; i++) alive += e->pods[i].alive;
    if (alive > e->peak_pods) e->peak_pods = alive;
  }
  return slot;
}

static int cmp_place_batch(const void* a, const void* b) { /* (-area, pod_id): sim_engine.py:395 */
  return cmp_restructure(a, b);
}

/* _place_batch: sim_engine.py:394-407 */
static void place_batch(Eng* e, int* batch, int nb) {
  g_sort_eng = e;
  qsort(batch, (size_t)nb, sizeof(int), cmp_place_batch);
  for (int i = 0; i < nb; i++) {
    Pod* p = &e->pods[batch[i]];
    int g; Rect r;
    e->attempts++;
    if (getenv("GS_ORACLE_DEBUG")) fprintf(stderr, "place %s\n", p->id);
    if (!best_match(e, p, &g, &r)) {
      if (getenv("GS_ORACLE_DEBUG")) fprintf(stderr, "  no placement for %s\n", p->id);
      e->win_failures++;
      p->in_retry = 1;
      GROW(e->retry, e->nretry, e->cretry, 1);
      e->retry[e->nretry++] = batch[i];
      continue;
    }
    Node* n = &e->nodes[g];
    Rect placed = {r.x, r.y, p->rw, p->rh};           /* place(): packer.py:245-261 */
    carve(&n->fr, &n->nfr, &n->cfr, placed);
    mem_add(n, p->fn);
    n->nplaced++;
    p->x = r.x; p->y = r.y; p->gpu = g; p->in_retry = 0;
  }
}

/* _remove_pod: sim_engine.py:377-392 */
static void remove_pod(Eng* e, int slot) {
  Pod* p = &e->pods[slot];
  for (int i = 0; i < e->nretry; i++) if (e->retry[i] == slot) {
    memmove(&e->retry[i], &e->retry[i + 1], sizeof(int) * (size_t)(e->nretry - i - 1));
    e->nretry--;
    p->alive = 0;
    return;
  }
  Fn* fn = &e->fn[p->fn];
  if (p->has_cur) {                 /* the in-flight request restarts from scratch */
    for (int i = 0; i < fn->qn; i++) {
      Req* r = &fn->q[fn->qhead + i];
      if (r->server == slot) { r->server = -1; break; }
    }
    p->has_cur = 0;
    fn->pinned--;
  }
  p->registered = 0;                /* unregister_pod: token_backend.py:111-116 */
  Node* n = &e->nodes[p->gpu];      /* release(): packer.py:264-275 (append verbatim) */
  GROW(n->fr, n->nfr, n->cfr, 1);
  n->fr[n->nfr++] = (Rect){p->x, p->y, p->rw, p->rh};
  mem_remove(n, p->fn);
  n->nplaced--;
  p->alive = 0;
}

/* ------------------------------------------------------------ autoscaler */
typedef struct { int slot; double eff, thr; } RunPod;
static int cmp_runset(const void* a, const void* b) {  /* (efficiency, pod_id): autoscaler.py:50-51 */
  const RunPod* x = a; const RunPod* y = b;
  if (x->eff < y->eff) return -1;
  if (x->eff > y->eff) return 1;
  return strcmp(g_sort_eng->pods[x->slot].id, g_sort_eng->pods[y->slot].id);
}

/* _run_epoch: sim_engine.py:409-430 */
static void run_epoch(Eng* e, int window) {
  int nadd = 0, cadd = 0; int* adds = NULL;
  RunPod* rs = xrealloc(NULL, sizeof(RunPod) * (size_t)(e->npods + 1));
  for (int f = 0; f < e->F; f++) {
    Fn* fn = &e->fn[f];
    /* predict_demand: max(history[-3:]), autoscaler.py:152-160 */
    double pred = fn->hist[fn->nhist - 1];
    for (int i = fn->nhist - 2; i >= 0 && i >= fn->nhist - 3; i--) if (fn->hist[i] > pred) pred = fn->hist[i];
    /* _running_pods (placed + retry), RunningSet order: sim_engine.py:370-375 */
    int n = 0;
    for (int i = 0; i < e->npods; i++) {
      Pod* p = &e->pods[i];
      if (!p->alive || p->fn != f) continue;
      const gs_point_t* pt = PT(e, f, p->point);
      rs[n].slot = i; rs[n].eff = pt->thr / pt->area; rs[n].thr = pt->thr; n++;
    }
    g_sort_eng = e;
    qsort(rs, (size_t)n, sizeof(RunPod), cmp_runset);
    PySum sup = {0, 0, 0};                         /* rps_gap: autoscaler.py:81-88 */
    for (int i = 0; i < n; i++) pysum_add(&sup, rs[i].thr);
    double gap = pred - pysum_value(&sup);
    if (getenv("GS_ORACLE_DEBUG")) fprintf(stderr, "window %d: fn %d demand=%.3f gap=%.3f pods=%d\n", window, f, pred, gap, n);
    if (gap > 0) {                                /* scale_up: autoscaler.py:103-131 */
      const gs_function_t* fs = &e->fs[f];
      int pe = fs->p_eff;
      double t_eff = PT(e, f, pe)->thr;
      if (t_eff <= 0) {                           /* autoscaler.py:115-117 */
        if (!e->err_code) { e->err_code = GS_ERR_VALIDATION; e->err_detail = GS_VAL_NO_THROUGHPUT;
                            e->err_fn = f; e->err_pt = pe; }
        free(rs); free(adds); return;
      }
      double nd = floor(gap / t_eff);
      double residual = gap - nd * t_eff;
      long long cnt = (long long)nd;
      int ideal = -1;
      if (residual > 0) {
        ideal = pe;
        int found = 0; double b0 = 0, b1 = 0, b2 = 0, b3 = 0;
        for (int k = 0; k < fs->n_points; k++) {
          const gs_point_t* pt = PT(e, f, k);
          if (!(pt->thr > residual)) continue;
          double k0 = pt->thr - residual;
          if (!found || k0 < b0 || (k0 == b0 && (pt->area < b1 || (pt->area == b1 &&
              (pt->sm < b2 || (pt->sm == b2 && pt->quota < b3)))))) {
            found = 1; b0 = k0; b1 = pt->area; b2 = pt->sm; b3 = pt->quota; ideal = k;
          }
        }
      }
      long long total = cnt + (ideal >= 0 ? 1 : 0);
      e->decisions += total;
      for (long long i = 0; i < total; i++) {
        int k = i < cnt ? pe : ideal;
        int slot = make_pod(e, f, k, 0, 0.0, window + e->sc->cold_start_windows);
        if (slot < 0) { free(rs); free(adds); return; }
        GROW(adds, nadd, cadd, 1);
        adds[nadd++] = slot;
      }
    } else if (gap < 0) {                         /* scale_down: autoscaler.py:134-149 */
      double delta = gap;
      int front = 0;
      if (getenv("GS_ORACLE_DEBUG")) for (int i = 0; i < n; i++) fprintf(stderr, "  rs %s eff=%.17g thr=%.17g\n", e->pods[rs[i].slot].id, rs[i].eff, rs[i].thr);
      while (delta < 0 && front < n) {
        if (delta + rs[front].thr > 0) break;
        delta += rs[front].thr;
        e->decisions++;
        remove_pod(e, rs[front].slot);
        front++;
      }
    }
  }
  free(rs);
  /* retry, self.retry = self.retry, []; _place_batch(retry + additions) */
  int nb = e->nretry + nadd;
  int* batch = xrealloc(NULL, sizeof(int) * (size_t)(nb + 1));
  memcpy(batch, e->retry, sizeof(int) * (size_t)e->nretry);
  memcpy(batch + e->nretry, adds, sizeof(int) * (size_t)nadd);
  for (int i = 0; i < e->nretry; i++) e->pods[e->retry[i]].in_retry = 0;
  e->nretry = 0;
  place_batch(e, batch, nb);
  free(batch); free(adds);
  for (int g = 0; g < e->G; g++) restructure(e, g);
}

/* ------------------------------------------------------------ window loop */
static void complete_live_tokens(Eng* e) {    /* sim_engine.py:482-486 + complete_token :190-210 */
  for (int g = 0; g < e->G; g++) {
    Node* n = &e->nodes[g];
    for (int i = 0; i < n->nlive; i++) {
      Token t = n->live[i];
      n->sm_running -= t.sm;
      if (n->sm_running < 0 && n->sm_running > -SM_EPS) n->sm_running = 0.0;
      Pod* p = &e->pods[t.pod];
      if (p->registered) p->q_used += t.dur;
    }
    n->nlive = 0;
  }
}

static void admit_arrivals(Eng* e, int f, double now) {   /* sim_engine.py:472-480 */
  Fn* fn = &e->fn[f];
  int limit = e->fs[f].max_queue;
  while (fn->fn_ > 0 && fn->fut[fn->fhead] <= now + TIME_EPS) {
    double a = fn->fut[fn->fhead++]; fn->fn_--;
    if (limit >= 0 && fn->qn >= limit) { fn->win_drop++; continue; }
    if (fn->qhead + fn->qn + 1 > fn->qcap) {
      if (fn->qhead > 0) { memmove(fn->q, fn->q + fn->qhead, sizeof(Req) * (size_t)fn->qn); fn->qhead = 0; }
      GROW(fn->q, fn->qn, fn->qcap, 1);
    }
    fn->q[fn->qhead + fn->qn] = (Req){a, -1};
    fn->qn++;
  }
}

/* _serve: sim_engine.py:525-552 */
static void serve(Eng* e, int slot, double t_start, double t_end) {
  Pod* p = &e->pods[slot];
  Fn* fn = &e->fn[p->fn];
  double slo = e->fs[p->fn].slo_ms;
  double t = p->busy_until > t_start ? p->busy_until : t_start;
  while (t < t_end - TIME_EPS) {
    if (!p->has_cur) {
      int idx = -1;
      for (int i = 0; i < fn->qn; i++) if (fn->q[fn->qhead + i].server < 0) { idx = i; break; }
      if (idx < 0) break;
      fn->q[fn->qhead + idx].server = slot;
      p->has_cur = 1; p->cur_rem = p->inv_rate; p->cur_arr = fn->q[fn->qhead + idx].arrival;
      fn->pinned++;
    }
    double span = (t_end - t) < p->cur_rem ? (t_end - t) : p->cur_rem;
    p->cur_rem -= span;
    t += span;
    if (p->cur_rem <= TIME_EPS) {
      int idx = -1;
      for (int i = 0; i < fn->qn; i++) if (fn->q[fn->qhead + i].server == slot) { idx = i; break; }
      /* fn.queue.remove(req): shift the (short) prefix right by one */
      memmove(&fn->q[fn->qhead + 1], &fn->q[fn->qhead], sizeof(Req) * (size_t)idx);
      fn->qhead++; fn->qn--;
      fn->pinned--;
      p->has_cur = 0;
      fn->win_comp++;
      if ((t - p->cur_arr) * 1000.0 > slo) fn->win_viol++;
    }
  }
  p->busy_until = t;
}

typedef struct { int slot; double neg_deficit; } QEnt;
static int cmp_queue(const void* a, const void* b) {   /* build_queue: token_backend.py:157 */
  const QEnt* x = a; const QEnt* y = b;
  if (x->neg_deficit < y->neg_deficit) return -1;
  if (x->neg_deficit > y->neg_deficit) return 1;
  return strcmp(g_sort_eng->pods[x->slot].id, g_sort_eng->pods[y->slot].id);
}
static int cmp_token_pod(const void* a, const void* b) {
  const Token* x = a; const Token* y = b;
  return strcmp(g_sort_eng->pods[x->pod].id, g_sort_eng->pods[y->pod].id);
}

/* _run_window_steps: sim_engine.py:488-523 */
static void run_window_steps(Eng* e, int window) {
  const gs_scenario_t* sc = e->sc;
  for (int g = 0; g < e->G; g++) { e->nodes[g].cov = 0.0; e->nodes[g].occ = 0.0; }
  QEnt* qe = xrealloc(NULL, sizeof(QEnt) * (size_t)(e->npods + 1));
  Token* sorted = xrealloc(NULL, sizeof(Token) * (size_t)(e->npods + 1));
  for (int step = 0; step < sc->steps; step++) {
    double t0 = (double)window * sc->window_s + (double)step * sc->quantum_s;
    complete_live_tokens(e);
    for (int f = 0; f < e->F; f++) admit_arrivals(e, f, t0);
    for (int g = 0; g < e->G; g++) {
      Node* n = &e->nodes[g];
      int nq = 0;
      for (int i = 0; i < e->npods; i++) {
        Pod* p = &e->pods[i];
        if (!p->alive || !p->registered || p->gpu != g) continue;
        if (p->q_lim - p->q_used <= QUOTA_EPS) continue;           /* filter_pods */
        Fn* fn = &e->fn[p->fn];
        if (!(p->has_cur || fn->qn - fn->pinned > 0)) continue;   /* requesting */
        qe[nq].slot = i; qe[nq].neg_deficit = -(p->q_req - p->q_used); nq++;
      }
      g_sort_eng = e;
      qsort(qe, (size_t)nq, sizeof(QEnt), cmp_queue);
      for (int i = 0; i < nq; i++) {                               /* dispatch: :160-187 */
        Pod* p = &e->pods[qe[i].slot];
        if (p->sm + n->sm_running > SM_LIMIT + SM_EPS) break;
        double rem = p->q_lim - p->q_used;
        double dur = rem < sc->quantum ? rem : sc->quantum;
        GROW(n->live, n->nlive, n->clive, 1);
        n->live[n->nlive++] = (Token){qe[i].slot, p->sm, dur};
        n->sm_running += p->sm;
        e->grants++;
      }
    }
    for (int g = 0; g < e->G; g++) {
      Node* n = &e->nodes[g];
      if (n->nlive == 0) continue;
      double mx = n->live[0].dur;
      PySum occ = {0, 0, 0};
      for (int i = 0; i < n->nlive; i++) {
        if (n->live[i].dur > mx) mx = n->live[i].dur;
        pysum_add(&occ, n->live[i].sm * n->live[i].dur);
      }
      n->cov += mx;
      n->occ += pysum_value(&occ) / 100.0;
      memcpy(sorted, n->live, sizeof(Token) * (size_t)n->nlive);
      g_sort_eng = e;
      qsort(sorted, (size_t)n->nlive, sizeof(Token), cmp_token_pod);
      for (int i = 0; i < n->nlive; i++)
        serve(e, sorted[i].pod, t0, t0 + sorted[i].dur * sc->window_s);
    }
  }
  complete_live_tokens(e);
  free(qe); free(sorted);
}

static void init_engine(Eng* e, const gs_batch_t* in, int run) {
  memset(e, 0, sizeof(*e));
  e->in = in;
  e->sc = &in->runs[run];
  e->fs = &in->funcs[e->sc->func_off];
  e->G = e->sc->n_nodes;
  e->F = e->sc->n_funcs;
  e->fn = xrealloc(NULL, sizeof(Fn) * (size_t)e->F);
  memset(e->fn, 0, sizeof(Fn) * (size_t)e->F);
  for (int f = 0; f < e->F; f++) e->fn[f].hist = xrealloc(NULL, sizeof(double) * (size_t)(e->sc->windows + 1));
  e->nodes = xrealloc(NULL, sizeof(Node) * (size_t)e->G);
  memset(e->nodes, 0, sizeof(Node) * (size_t)e->G);
  for (int g = 0; g < e->G; g++) {
    Node* n = &e->nodes[g];
    n->cfr = 8; n->fr = xrealloc(NULL, sizeof(Rect) * 8);
    n->fr[0] = (Rect){0, 0, e->sc->side_x, e->sc->side_y}; n->nfr = 1;
    n->res_fn = xrealloc(NULL, sizeof(int) * (size_t)(e->F + 1));
    n->res_cnt = xrealloc(NULL, sizeof(int) * (size_t)(e->F + 1));
  }
}

static void free_engine(Eng* e) {
  for (int f = 0; f < e->F; f++) { free(e->fn[f].q); free(e->fn[f].fut); free(e->fn[f].hist); }
  for (int g = 0; g < e->G; g++) { free(e->nodes[g].fr); free(e->nodes[g].res_fn); free(e->nodes[g].res_cnt); free(e->nodes[g].live); }
  free(e->fn); free(e->nodes); free(e->pods); free(e->retry);
}

/* _Engine.run: sim_engine.py:434-452, _close_window :554-594 */
static int run_one(const gs_batch_t* in, int run, const gs_out_t* out) {
  Eng E, *e = &E;
  init_engine(e, in, run);
  const gs_scenario_t* sc = e->sc;
  gs_status_t* st = &out->status[run];
  memset(st, 0, sizeof(*st));
  gs_summary_t sum; memset(&sum, 0, sizeof(sum));
  PySum su = {0, 0, 0}, so = {0, 0, 0};
  int nb = 0, cb = 0; int* batch = NULL;
  for (int f = 0; f < e->F; f++)
    if (e->fs[f].name_len > 140) { e->err_code = GS_ERR_ARG; goto done; }
  for (int f = 0; f < e->F; f++) {
    for (int i = 0; i < e->fs[f].n_init; i++) {
      const gs_init_t* ip = &in->inits[e->fs[f].init_off + i];
      int slot = make_pod(e, f, ip->point, ip->has_q_req, ip->q_req, 0);
      if (slot < 0) goto done;
      GROW(batch, nb, cb, 1);
      batch[nb++] = slot;
    }
  }
  place_batch(e, batch, nb);
  free(batch); batch = NULL;

  for (int w = 0; w < sc->windows; w++) {
    if (w > 0 && w % sc->epoch_windows == 0) {
      run_epoch(e, w);
      if (e->err_code) goto done;
    }
    for (int i = 0; i < e->npods; i++) {                /* _warm_up: :454-460 */
      Pod* p = &e->pods[i];
      if (p->alive && !p->in_retry && p->gpu >= 0 && !p->registered && p->warm_at <= w) {
        p->registered = 1; p->q_used = 0.0;
      }
    }
    for (int i = 0; i < e->npods; i++) if (e->pods[i].registered) e->pods[i].q_used = 0.0;  /* reset_window */
    double start = (double)w * sc->window_s;          /* _generate_arrivals: :462-470 */
    for (int f = 0; f < e->F; f++) {
      Fn* fn = &e->fn[f];
      int n = in->counts[e->fs[f].count_off + w];
      fn->win_arr = n;
      if (fn->fhead + fn->fn_ + n > fn->fcap) {
        if (fn->fhead > 0) { memmove(fn->fut, fn->fut + fn->fhead, sizeof(double) * (size_t)fn->fn_); fn->fhead = 0; }
        GROW(fn->fut, fn->fn_, fn->fcap, n);
      }
      for (int i = 0; i < n; i++) fn->fut[fn->fhead + fn->fn_ + i] = start + ((double)i * sc->window_s) / (double)n;
      fn->fn_ += n;
    }
    {
      long long nreg = 0;
      for (int i = 0; i < e->npods; i++) nreg += e->pods[i].alive && e->pods[i].registered;
      e->pod_steps += nreg * sc->steps;
    }
    run_window_steps(e, w);
    /* _close_window */
    for (int f = 0; f < e->F; f++) {
      Fn* fn = &e->fn[f];
      fn->hist[fn->nhist++] = (double)fn->win_arr / sc->window_s;
      int depth = fn->qn + fn->fn_;
      if (out->fn_rows) {
        gs_fn_row_t* r = &out->fn_rows[sc->fn_row_off + (long long)w * e->F + f];
        r->arrivals = fn->win_arr; r->completions = fn->win_comp;
        r->slo_violations = fn->win_viol; r->dropped = fn->win_drop; r->queue_depth = depth;
      }
      sum.arrivals += fn->win_arr; sum.completions += fn->win_comp;
      sum.slo_violations += fn->win_viol; sum.dropped += fn->win_drop;
      if (w == sc->windows - 1) sum.final_queue_depth += depth;
      fn->win_arr = fn->win_comp = fn->win_viol = fn->win_drop = 0;
    }
    int in_use = 0;
    for (int g = 0; g < e->G; g++) {
      Node* n = &e->nodes[g];
      gs_gpu_row_t row; memset(&row, 0, sizeof(row));
      if (n->nplaced > 0) {
        in_use++;
        row.present = 1;
        row.utilization = n->cov < 1.0 ? n->cov : 1.0;
        row.sm_occupancy = n->occ < 1.0 ? n->occ : 1.0;
        row.memory_mb = footprint(e, n);
        sum.n_gpu_rows++;
        pysum_add(&su, row.utilization);
        pysum_add(&so, row.sm_occupancy);
      }
      if (out->gpu_rows) out->gpu_rows[sc->gpu_row_off + (long long)w * e->G + g] = row;
    }
    long long total = 0, largest = -1;
    for (int g = 0; g < e->G; g++)
      for (int i = 0; i < e->nodes[g].nfr; i++) {
        Rect r = e->nodes[g].fr[i];
        total += r.w * r.h;
        if (r.w * r.h > largest) largest = r.w * r.h;
      }
    double frag = (total == 0 || largest < 0) ? 0.0 : (double)(total - largest) / (double)total;
    if (out->glob_rows) {
      gs_glob_row_t* gr = &out->glob_rows[sc->glob_row_off + w];
      gr->gpus_in_use = in_use; gr->placement_failures = e->win_failures; gr->fragmentation_index = frag;
    }
    if (in_use > sum.gpus_used_peak) sum.gpus_used_peak = in_use;
    sum.placement_failures += e->win_failures;
    e->win_failures = 0;
  }
  sum.windows = sc->windows;
  sum.sum_utilization = pysum_value(&su);
  sum.sum_sm_occupancy = pysum_value(&so);
  {
    int k = 0;
    for (int i = 0; i < e->npods; i++) {
      Pod* p = &e->pods[i];
      if (!p->alive || p->in_retry || p->gpu < 0) continue;
      if (out->placements && k < sc->cap_pods) {
        gs_placement_t* pl = &out->placements[sc->place_off + k];
        pl->node = p->gpu; pl->func = p->fn; pl->counter = p->counter;
        pl->x = (int)p->x; pl->y = (int)p->y; pl->w = (int)p->rw; pl->h = (int)p->rh; pl->pad = 0;
      }
      k++;
    }
    st->n_placements = k;
  }
done:
  free(batch);
  st->code = e->err_code;
  st->detail = e->err_detail;
  st->arg0 = e->err_fn;
  st->arg1 = e->err_pt;
  st->token_grants = e->grants;
  st->scale_decisions = e->decisions;
  st->placement_attempts = e->attempts;
  st->pod_steps = e->pod_steps;
  st->rect_scans = e->rect_scans;
  st->peak_pods = e->peak_pods;
  if (out->summary) out->summary[run] = sum;
  free_engine(e);
  return st->code;
}

/* --------------------------------------------------------------- batching */
typedef struct { const gs_batch_t* in; const gs_out_t* out; atomic_int next; atomic_int worst; } Work;

static void* worker(void* arg) {
  Work* w = arg;
  for (;;) {
    int r = atomic_fetch_add(&w->next, 1);
    if (r >= w->in->n_runs) break;
    int code = run_one(w->in, r, w->out);
    int cur = atomic_load(&w->worst);
    while (code > cur && !atomic_compare_exchange_weak(&w->worst, &cur, code)) {}
  }
  return NULL;
}

int gs_oracle_abi_version(void) { return GS_ABI_VERSION; }

/* Runs every (scenario, policy) of the batch on n_threads host threads. */
int gs_oracle_run_batch(const gs_batch_t* in, const gs_out_t* out, int n_threads) {
  if (!in || !out || !out->status) return GS_ERR_ARG;
  if (n_threads < 1) n_threads = 1;
  if (n_threads > in->n_runs) n_threads = in->n_runs > 0 ? in->n_runs : 1;
  Work w = {in, out, 0, 0};
  if (n_threads == 1) { worker(&w); return atomic_load(&w.worst); }
  pthread_t* th = xrealloc(NULL, sizeof(pthread_t) * (size_t)n_threads);
  for (int i = 0; i < n_threads; i++) pthread_create(&th[i], NULL, worker, &w);
  for (int i = 0; i < n_threads; i++) pthread_join(th[i], NULL);
  free(th);
  return atomic_load(&w.worst);
}

/* Struct sizes, for the host layout self-check. */
int gs_oracle_sizeof(const char* name) {
  if (!strcmp(name, "gs_scenario_t")) return (int)sizeof(gs_scenario_t);
  if (!strcmp(name, "gs_function_t")) return (int)sizeof(gs_function_t);
  if (!strcmp(name, "gs_point_t")) return (int)sizeof(gs_point_t);
  if (!strcmp(name, "gs_init_t")) return (int)sizeof(gs_init_t);
  if (!strcmp(name, "gs_fn_row_t")) return (int)sizeof(gs_fn_row_t);
  if (!strcmp(name, "gs_gpu_row_t")) return (int)sizeof(gs_gpu_row_t);
  if (!strcmp(name, "gs_glob_row_t")) return (int)sizeof(gs_glob_row_t);
  if (!strcmp(name, "gs_placement_t")) return (int)sizeof(gs_placement_t);
  if (!strcmp(name, "gs_status_t")) return (int)sizeof(gs_status_t);
  if (!strcmp(name, "gs_summary_t")) return (int)sizeof(gs_summary_t);
  if (!strcmp(name, "gs_batch_t")) return (int)sizeof(gs_batch_t);
  if (!strcmp(name, "gs_out_t")) return (int)sizeof(gs_out_t);
  if (!strcmp(name, "gs_id_split_t")) return (int)sizeof(gs_id_split_t);
  return -1;
}
