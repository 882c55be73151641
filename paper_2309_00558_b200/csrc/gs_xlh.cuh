// gs_xlh.cuh -- the XL class's quantum steps on a CTA-wide shared-memory
// working set.
//
// Same idea as the per-warp classes (gs_hot.cuh), at CTA scale: while the
// registered set does not change, a run's registered pods (in (node, pod_id)
// order), functions and nodes live in the CTA's dynamic shared memory (up to
// ~200 KB: C4's ~10^3 registered pods, 200 functions and 64 nodes take about
// 140 KB), and all XL_THREADS threads run the steps there with block barriers
// between phases.  The layout is carved at run time for the run's (F, G) and
// the largest pod count that fits; a window whose registered set does not fit
// falls back to the arena-based steps (gs_xl.cuh).  The per-element helpers
// (hot_admit, hot_serve, hot_close, arrival arithmetic) are the per-warp
// classes' own, instantiated on this runtime-sized view.
#pragma once
#include "gs_hot.cuh"
#include "gs_xl.cuh"

namespace gs {

__device__ int xl_block_exscan(int v, int* warp_tot, int* total);   // below

// runtime-sized view of the working set (same member names as Hot<>)
struct HotX {
  // pods [PC]
  double *qused, *qreq, *qlim, *sm, *busy, *crem, *carr, *invr, *key;
  long long* cur;
  int* fnode;
  short *order, *flist, *rank, *gl;   // gl: granted pods in (function, node, pod_id) order
  int* gpick;                          // request starts of gl[k] (dry run), then its base
  unsigned char* flags;
  // functions [FC]
  double *farr, *slo;
  int *qlen, *pinned, *fw, *fi, *fcnt, *nsn, *nsw, *nsi, *rhead, *retn, *wcomp, *wviol, *wdrop;
  int *maxq, *ringoff, *fwn, *nswn, *warr, *hn, *loff, *coff;
  int *fbase, *fpicks, *fcomp, *fviol;                 // serve scratch
  // nodes [GC]
  double *sr, *cov, *occ, *fp;
  int *seg, *cut, *reqsm, *ngr, *nplaced, *fullq;   // fullq: a full-quantum token this step
  unsigned long long* covbits;
  // run constants
  const int32_t* counts;
  long long* f_ret;
  long long* f_ring;
  double ws, qs, quantum;
  int n, F, G, T, W, RET, integral, bounded, PC;

  __device__ __forceinline__ int count(int f, int w) const { return counts[coff[f] + w]; }
  __device__ __forceinline__ double dur(int i) const {
    const double rem = qlim[i] - qused[i];
    return rem < quantum ? rem : quantum;
  }
  __device__ __forceinline__ double arrival(int f, int w, int i) const {
    return (double)w * ws + ((double)i * ws) / (double)count(f, w);
  }
  __device__ __forceinline__ double arrival_n(int w, int i, int n_) const {
    return (double)w * ws + ((double)i * ws) / (double)n_;
  }
  __device__ __forceinline__ void advance(int f, int& w, int& i, int& n_) const {
    if (++i < n_) return;
    i = 0;
    do { w++; n_ = w < W ? count(f, w) : 1; } while (n_ == 0);
  }
};

template <>
struct HotCap<HotX> {
  static constexpr int PC = 1 << 30, FC = 1 << 30, GC = 1 << 30;
};

constexpr size_t XLH_DYN_BYTES = 224 * 1024;   // dynamic shared memory per XL CTA (+ ~2 KB static)
constexpr size_t XLH_POD_BYTES = 9 * 8 + 8 + 4 + 4 * 2 + 4 + 1;   // per registered pod
constexpr size_t XLH_FN_BYTES = 2 * 8 + 25 * 4 + 4;           // per function (+ loff)
constexpr size_t XLH_NODE_BYTES = 4 * 8 + 6 * 4 + 8 + 4;      // per node (+ seg)

// upper bound of the carved size (each of the ~50 arrays may pad by < 16 B)
__host__ __device__ inline size_t xlh_bytes(int PC, int F, int G) {
  return (size_t)PC * XLH_POD_BYTES + (size_t)(F + 1) * XLH_FN_BYTES
       + (size_t)(G + 1) * XLH_NODE_BYTES + 64 * 16;
}

// carve the view over `base` (thread 0 only); PC = largest pod count that fits
__device__ void xlh_carve(HotX* h, char* base, size_t bytes, int F, int G) {
  const size_t fixed = xlh_bytes(0, F, G);
  int PC = bytes > fixed ? (int)((bytes - fixed) / XLH_POD_BYTES) : 0;
  PC &= ~7;
  size_t o = 0;
  auto take = [&](size_t n, size_t elem) { char* p = base + o; o = gs_align16(o + n * elem); return p; };
  const size_t P = (size_t)PC, Fn = (size_t)F + 1, Gn = (size_t)G + 1;
  h->qused = (double*)take(P, 8); h->qreq = (double*)take(P, 8); h->qlim = (double*)take(P, 8);
  h->sm = (double*)take(P, 8); h->busy = (double*)take(P, 8); h->crem = (double*)take(P, 8);
  h->carr = (double*)take(P, 8); h->invr = (double*)take(P, 8); h->key = (double*)take(P, 8);
  h->cur = (long long*)take(P, 8); h->fnode = (int*)take(P, 4);
  h->order = (short*)take(P, 2); h->flist = (short*)take(P, 2); h->rank = (short*)take(P, 2);
  h->flags = (unsigned char*)take(P, 1);
  h->gl = (short*)take(P, 2); h->gpick = (int*)take(P, 4);
  h->farr = (double*)take(Fn, 8); h->slo = (double*)take(Fn, 8);
  int** fi[] = {&h->qlen, &h->pinned, &h->fw, &h->fi, &h->fcnt, &h->nsn, &h->nsw, &h->nsi,
                &h->rhead, &h->retn, &h->wcomp, &h->wviol, &h->wdrop, &h->maxq, &h->ringoff,
                &h->fwn, &h->nswn, &h->warr, &h->hn, &h->loff, &h->coff,
                &h->fbase, &h->fpicks, &h->fcomp, &h->fviol};
  for (int k = 0; k < 25; k++) *fi[k] = (int*)take(Fn, 4);
  h->sr = (double*)take(Gn, 8); h->cov = (double*)take(Gn, 8); h->occ = (double*)take(Gn, 8);
  h->fp = (double*)take(Gn, 8); h->covbits = (unsigned long long*)take(Gn, 8);
  h->seg = (int*)take(Gn, 4); h->cut = (int*)take(Gn, 4); h->reqsm = (int*)take(Gn, 4);
  h->ngr = (int*)take(Gn, 4); h->nplaced = (int*)take(Gn, 4); h->fullq = (int*)take(Gn, 4);
  h->PC = o <= bytes ? PC : 0;
}

// arena -> working set (all threads); false if the registered set does not fit
__device__ bool xlh_load(Ctx& c, HotX* h) {
  const int n = c.sh->n_reg;
  if (n > h->PC) return false;
  const int tid = threadIdx.x, NT = blockDim.x;
  const int* rl = c.t->s_rl;
#pragma unroll 1
  for (int i = tid; i < n; i += NT) {
    const int s = rl[i];
    h->qused[i] = c.t->p_qused[s]; h->qreq[i] = c.t->p_qreq[s]; h->qlim[i] = c.t->p_qlim[s];
    h->sm[i] = c.t->p_sm[s]; h->busy[i] = c.t->p_busy[s]; h->crem[i] = c.t->p_crem[s];
    h->carr[i] = c.t->p_carr[s]; h->invr[i] = c.t->p_invr[s];
    h->cur[i] = pack_id(c.t->p_cw[s], c.t->p_ci[s]);
    h->fnode[i] = c.t->p_fn[s] | (c.t->p_node[s] << 16);
    h->flags[i] = (unsigned char)(c.t->p_flags[s] & PF_CUR);
    h->order[i] = (short)i;
    c.t->s_list[s] = i;                 // slot -> registered index (for flist)
  }
#pragma unroll 1
  for (int f = tid; f < c.F; f += NT) {
    h->qlen[f] = c.t->f_qlen[f]; h->pinned[f] = c.t->f_pinned[f];
    h->fw[f] = c.t->f_fw[f]; h->fi[f] = c.t->f_fi[f]; h->fcnt[f] = c.t->f_fn[f];
    h->nsn[f] = c.t->f_nsn[f]; h->nsw[f] = c.t->f_nsw[f]; h->nsi[f] = c.t->f_nsi[f];
    h->rhead[f] = c.t->f_rhead[f]; h->retn[f] = c.t->f_retn[f];
    h->wcomp[f] = 0; h->wviol[f] = 0; h->wdrop[f] = 0;
    h->warr[f] = c.t->f_warr[f]; h->hn[f] = c.t->f_hn[f];
    h->maxq[f] = c.fs[f].max_queue;
    h->ringoff[f] = c.t->f_ringoff[f];
    h->slo[f] = c.fs[f].slo_ms;
    h->coff[f] = c.fs[f].count_off;
    h->farr[f] = h->fcnt[f] > 0 ? arrival_time(c, f, h->fw[f], h->fi[f]) : 0.0;
    h->fwn[f] = h->fcnt[f] > 0 ? c.count(f, h->fw[f]) : 1;
    h->nswn[f] = (h->nsn[f] > 0 && c.fs[f].max_queue < 0) ? c.count(f, h->nsw[f]) : 1;
  }
#pragma unroll 1
  for (int f = tid; f <= c.F; f += NT) h->loff[f] = c.t->f_loff[f];
#pragma unroll 1
  for (int g = tid; g < c.G; g += NT) {
    h->sr[g] = c.t->n_sr[g]; h->cov[g] = 0.0; h->occ[g] = 0.0;
    h->nplaced[g] = c.t->n_nplaced[g]; h->fp[g] = c.t->n_fp[g];
  }
#pragma unroll 1
  for (int g = tid; g <= c.G; g += NT) h->seg[g] = c.t->n_seg[g];
  if (tid == 0) {
    h->n = n;
    h->counts = c.counts; h->f_ret = c.t->f_ret; h->f_ring = c.t->f_ring;
    h->ws = c.ws; h->qs = c.qs; h->quantum = c.quantum;
    h->F = c.F; h->G = c.G; h->T = c.T; h->W = c.W; h->RET = c.RET;
    // see hot_load: order-free occupancy sums need durations > QUOTA_EPS
    h->integral = (c.integral() && c.quantum >= QUOTA_EPS) ? 1 : 0;
  }
  __syncthreads();
#pragma unroll 1
  for (int j = tid; j < n; j += NT) h->flist[j] = (short)c.t->s_list[c.t->s_fl[j]];
  __syncthreads();
  return true;
}

// working set -> arena (all threads)
__device__ void xlh_store(Ctx& c, HotX* h) {
  const int n = h->n, tid = threadIdx.x, NT = blockDim.x;
#pragma unroll 1
  for (int i = tid; i < n; i += NT) {
    const int s = c.t->s_rl[i];
    c.t->p_qused[s] = h->qused[i]; c.t->p_busy[s] = h->busy[i];
    c.t->p_crem[s] = h->crem[i]; c.t->p_carr[s] = h->carr[i];
    c.t->p_cw[s] = id_w(h->cur[i]); c.t->p_ci[s] = id_i(h->cur[i]);
    c.t->p_flags[s] = (c.t->p_flags[s] & ~(PF_CUR | PF_GRANT)) | (h->flags[i] & PF_CUR);
  }
#pragma unroll 1
  for (int f = tid; f < c.F; f += NT) {
    c.t->f_qlen[f] = h->qlen[f]; c.t->f_pinned[f] = h->pinned[f];
    c.t->f_fw[f] = h->fw[f]; c.t->f_fi[f] = h->fi[f]; c.t->f_fn[f] = h->fcnt[f];
    c.t->f_nsn[f] = h->nsn[f]; c.t->f_nsw[f] = h->nsw[f]; c.t->f_nsi[f] = h->nsi[f];
    c.t->f_rhead[f] = h->rhead[f]; c.t->f_retn[f] = h->retn[f];
    c.t->f_hn[f] = h->hn[f];
  }
#pragma unroll 1
  for (int g = tid; g < c.G; g += NT) c.t->n_sr[g] = h->sr[g];
  __syncthreads();
}

// window start without a registration change (cf. hot_begin_light), all threads
__device__ void xlh_begin_light(HotX* h, int w) {
  const int tid = threadIdx.x, NT = blockDim.x;
#pragma unroll 1
  for (int i = tid; i < h->n; i += NT) h->qused[i] = 0.0;
#pragma unroll 1
  for (int f = tid; f < h->F; f += NT) {
    const int k = h->count(f, w);
    h->warr[f] = k;
    if (k > 0) {
      if (h->fcnt[f] == 0) {
        h->fw[f] = w; h->fi[f] = 0; h->fwn[f] = k;
        h->farr[f] = h->arrival_n(w, 0, k);
      }
      h->fcnt[f] += k;
    }
  }
#pragma unroll 1
  for (int g = tid; g < h->G; g += NT) { h->cov[g] = 0.0; h->occ[g] = 0.0; }
  __syncthreads();
}

// complete live tokens (sim_engine.py:482-486), all threads
__device__ void xlh_complete(HotX* h) {
  const int tid = threadIdx.x, NT = blockDim.x;
  if (!h->integral) {
#pragma unroll 1
    for (int g = tid; g < h->G; g += NT) {
      double sr = h->sr[g];
      const int lo = h->seg[g], e = lo + h->ngr[g];      // the granted prefix
#pragma unroll 1
      for (int j = lo; j < e; j++) {
        sr -= h->sm[h->order[j]];
        if (sr < 0 && sr > -SM_EPS) sr = 0.0;
      }
      h->sr[g] = sr;
    }
    __syncthreads();
  }
#pragma unroll 1
  for (int i = tid; i < h->n; i += NT) {
    const int fl = h->flags[i];
    if (fl & PF_GRANT) {
      h->qused[i] += h->dur(i);
      h->flags[i] = (unsigned char)(fl & ~PF_GRANT);
    }
  }
  __syncthreads();
}

template <bool BND>
__device__ __forceinline__ void xlh_books(HotX* h, int f, int want, int comp);   // below

// one quantum step (sim_engine.py:493-520) on the CTA-wide working set
template <bool BND>
#ifdef GS_XL_TIMING
#define GS_PH_INIT() long long ph_t_ = clock64()
#define GS_PH(k) { const long long now_ = clock64(); \
    if (threadIdx.x == 0) atomicAdd(&gs_xl_t[k], (unsigned long long)(now_ - ph_t_)); ph_t_ = now_; }
// each warp's busy cycles of phase k (its arrival at the barrier): with the
// phase time above, the average over warps shows the phase's imbalance
#define GS_PW(k) { const long long now_ = clock64(); \
    if ((threadIdx.x & 31) == 0) atomicAdd(&gs_xl_t[32 + (k)], (unsigned long long)(now_ - ph_t_)); }
#else
#define GS_PH_INIT()
#define GS_PH(k)
#define GS_PW(k)
#endif
__device__ void xlh_step(HotX* h, int w, int s, XlShared* xs) {
  const double t0 = (double)w * h->ws + (double)s * h->qs;
  const int n = h->n, F = h->F, G = h->G;
  const int tid = threadIdx.x, NT = blockDim.x;
  const bool integral = h->integral != 0;
  GS_PH_INIT();
  if (threadIdx.x == 0) { GS_EPOCH_ADD(25, 1); GS_EPOCH_ADD(26, n); }
#ifdef GS_XL_TIMING
  if (threadIdx.x == 0) {
    int mx = 0;
    for (int g = 0; g < G; g++) mx = max(mx, h->seg[g + 1] - h->seg[g]);
    GS_EPOCH_ADD(28, mx);
    atomicMax(&gs_xl_t[29], (unsigned long long)mx);
  }
#endif
  // per-function and per-node work share one index space so they run on
  // different threads: functions on [0, F), nodes on [FP, FP + G)
  const int FP = (F + 31) & ~31;
  if (tid == 0) xs->grants = 0;
#pragma unroll 1
  for (int x = tid; x < FP + G; x += NT) {
    if (x < F) {
      if (s == 0) hot_admit<HotX, BND>(h, x, t0);   // later steps: admitted at the
                                                    // end of the previous step
    } else if (x >= FP) {
      const int g = x - FP;
      if (s > 0 && !integral) {
        // sm_running -= sm in the last dispatch order, with the float-dust clamp
        double sr = h->sr[g];
        const int lo = h->seg[g], e = lo + h->ngr[g];    // the granted prefix
#pragma unroll 1
        for (int j = lo; j < e; j++) {
          sr -= h->sm[h->order[j]];
          if (sr < 0 && sr > -SM_EPS) sr = 0.0;
        }
        h->sr[g] = sr;
      }
      h->cut[g] = 0x7fffffff; h->covbits[g] = 0ull; h->reqsm[g] = 0; h->ngr[g] = 0;
      h->fullq[g] = 0;
    }
  }
  GS_PW(16);
  __syncthreads();
  GS_PH(16);
  // complete live tokens + filter_pods + requesting -> key
#pragma unroll 1
  for (int i = tid; i < n; i += NT) {
    const int f = h->fnode[i] & 0xffff;
    int fl = h->flags[i];
    double qused = h->qused[i];
    if (fl & PF_GRANT) {
      qused += h->dur(i);
      h->qused[i] = qused;
      fl &= ~PF_GRANT;
      h->flags[i] = (unsigned char)fl;
    }
    const bool cand = !(h->qlim[i] - qused <= QUOTA_EPS);
    const bool req = cand && ((fl & PF_CUR) || (h->qlen[f] - h->pinned[f] > 0));
    h->key[i] = req ? -(h->qreq[i] - qused) : NOT_REQ;
    // integral: requesting SM per node; otherwise: requesting pods per node
    if (req) atomicAdd(&h->reqsm[h->fnode[i] >> 16], integral ? (int)h->sm[i] : 1);
  }
  GS_PW(17);
  __syncthreads();
  GS_PH(17);
  // build_queue order per node by counting (key, pod index): pods before i
  // in the node count on <=, pods after it on <.  Only requesting pods get a
  // position (non-requesting keys are +inf, never ahead of one): the node's
  // requesting prefix of `order` is all dispatch reads.  One trip count per node
  // keeps the lanes of a warp (mostly one node) converged; four independent
  // accumulators keep the shared-memory loads in flight.  In the integral
  // path the SM ahead of i is a sum of integer-valued doubles, exact in any
  // order, and only nodes whose requesting SM exceeds 100 need ranks at all
  // (the others grant every requesting pod; occupancy sums are order-free,
  // see hot_step).
#pragma unroll 1
  for (int i = tid; i < n; i += NT) {
    const double k = h->key[i];
    if (k == NOT_REQ) continue;                // never dispatched: no position needed
    const int g = h->fnode[i] >> 16;
    if (integral && h->reqsm[g] <= (int)SM_LIMIT) { h->rank[i] = 0; continue; }
    const int lo = h->seg[g], hi = h->seg[g + 1];
    const double* key = h->key;
    int r0 = 0, r1 = 0, r2 = 0, r3 = 0;
    int j = lo;
    if (integral && h->reqsm[g] > (int)SM_LIMIT) {
      const double* sm = h->sm;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 1
      for (; j + 3 < hi; j += 4) {
        const bool l0 = j < i ? key[j] <= k : key[j] < k;
        const bool l1 = j + 1 < i ? key[j + 1] <= k : key[j + 1] < k;
        const bool l2 = j + 2 < i ? key[j + 2] <= k : key[j + 2] < k;
        const bool l3 = j + 3 < i ? key[j + 3] <= k : key[j + 3] < k;
        r0 += l0; r1 += l1; r2 += l2; r3 += l3;
        a0 += l0 ? sm[j] : 0.0; a1 += l1 ? sm[j + 1] : 0.0;
        a2 += l2 ? sm[j + 2] : 0.0; a3 += l3 ? sm[j + 3] : 0.0;
      }
#pragma unroll 1
      for (; j < hi; j++) {
        const bool l = j < i ? key[j] <= k : key[j] < k;
        r0 += l; a0 += l ? sm[j] : 0.0;
      }
      const double ahead = (a0 + a1) + (a2 + a3);
      if (sm[i] + ahead > SM_LIMIT + SM_EPS) atomicMin(&h->cut[g], (r0 + r1) + (r2 + r3));
    } else {
#pragma unroll 1
      for (; j + 3 < hi; j += 4) {
        r0 += j < i ? key[j] <= k : key[j] < k;
        r1 += j + 1 < i ? key[j + 1] <= k : key[j + 1] < k;
        r2 += j + 2 < i ? key[j + 2] <= k : key[j + 2] < k;
        r3 += j + 3 < i ? key[j + 3] <= k : key[j + 3] < k;
      }
#pragma unroll 1
      for (; j < hi; j++) r0 += j < i ? key[j] <= k : key[j] < k;
    }
    const int r = (r0 + r1) + (r2 + r3);
    if (!integral) h->order[lo + r] = (short)i;
    h->rank[i] = (short)r;
  }
  GS_PW(18);
  __syncthreads();
  GS_PH(18);
  const double quantum = h->quantum;
  int grants = 0;
  if (integral) {
#pragma unroll 1
    for (int i = tid; i < n; i += NT) {
      const int g = h->fnode[i] >> 16;
      if (h->key[i] != NOT_REQ && h->rank[i] < h->cut[g]) {
        const double rem = h->qlim[i] - h->qused[i];
        h->flags[i] |= PF_GRANT;
        // the node's tokens in grant-slot order (the occupancy sum is
        // order-free, see hot_step); a full quantum is the max duration,
        // only partial tokens need the (CAS-loop) 64-bit max
        h->order[h->seg[g] + atomicAdd(&h->ngr[g], 1)] = (short)i;
        if (rem < quantum) atomicMax(&h->covbits[g], (unsigned long long)__double_as_longlong(rem));
        else atomicOr(&h->fullq[g], 1);
        grants++;
      }
    }
    GS_PW(19);
    GS_PH(19);
  } else {
#pragma unroll 1
    for (int g = tid; g < G; g += NT) {
      double sr = h->sr[g];
      double mx = 0.0;
      int ng = 0;
      const int lo = h->seg[g], e = lo + h->reqsm[g];   // the requesting prefix
#pragma unroll 1
      for (int j = lo; j < e; j++) {
        const int i = h->order[j];
        const double sm = h->sm[i];
        if (sm + sr > SM_LIMIT + SM_EPS) break;
        const double rem = h->qlim[i] - h->qused[i];
        const double dur = rem < quantum ? rem : quantum;
        h->flags[i] |= PF_GRANT;
        sr += sm;
        if (ng == 0 || dur > mx) mx = dur;
        ng++;
      }
      h->sr[g] = sr;
      h->ngr[g] = ng;
      h->covbits[g] = (unsigned long long)__double_as_longlong(mx);
      grants += ng;
    }
  }
  if (grants) atomicAdd(&xs->grants, grants);
  GS_PW(20);
  __syncthreads();
  GS_PH(20);
  // serve (sim_engine.py:514-552), pod-parallel as in the per-warp classes:
  // granted pods in (function, node, pod_id) order, a dry run counts each
  // pod's request starts, a block scan turns them into per-function FIFO
  // positions, and a replay serves exactly the requests the sequential drain
  // would hand out.  1. compact the granted pods (chunk per thread, flist order)
  const double ws = h->ws;
  const int per = (n + NT - 1) / NT;
  const int j0 = tid * per, j1 = min(n, j0 + per);
  int mine = 0;
#pragma unroll 1
  for (int j = j0; j < j1; j++) mine += (h->flags[h->flist[j]] & PF_GRANT) ? 1 : 0;
  int ngl = 0;
  int k = xl_block_exscan(mine, xs->warp_tot, &ngl);
  if (threadIdx.x == 0) { GS_EPOCH_ADD(27, ngl); }
#pragma unroll 1
  for (int j = j0; j < j1; j++) {
    const int i = h->flist[j];
    if (h->flags[i] & PF_GRANT) h->gl[k++] = (short)i;
  }
#pragma unroll 1
  for (int f = tid; f < F; f += NT) { h->fcomp[f] = 0; h->fviol[f] = 0; h->fpicks[f] = 0; }
  GS_PW(21);
  __syncthreads();
  GS_PH(21);
  // 2. dry runs (chunk per thread so the block scan below runs in gl order)
  const int pk = (ngl + NT - 1) / NT;
  const int k0 = tid * pk, k1 = min(ngl, k0 + pk);
  int picks = 0;
#pragma unroll 1
  for (int kk = k0; kk < k1; kk++) {
    const int i = h->gl[kk];
    const int p = serve_dry_run(h, i, t0, t0 + h->dur(i) * ws);
    h->gpick[kk] = p;
    picks += p;
  }
  int total = 0;
  int run = xl_block_exscan(picks, xs->warp_tot, &total);
  // 3. global exclusive prefix of picks per granted pod; each function's
  //    first granted pod records the prefix where the function starts
#pragma unroll 1
  for (int kk = k0; kk < k1; kk++) {
    const int i = h->gl[kk];
    const int f = h->fnode[i] & 0xffff;
    const int p = h->gpick[kk];
    h->gpick[kk] = run;                       // now: prefix before this pod
    if (kk == 0 || (h->fnode[h->gl[kk - 1]] & 0xffff) != f) h->fbase[f] = run;
    atomicAdd(&h->fpicks[f], p);
    run += p;
  }
  GS_PW(22);
  __syncthreads();
  GS_PH(22);
  // 4. replay with the pod's FIFO position inside its function
#pragma unroll 1
  for (int kk = tid; kk < ngl; kk += NT) {
    const int i = h->gl[kk];
    const int f = h->fnode[i] & 0xffff;
    const double t_end = t0 + h->dur(i) * ws;
    const int base = h->gpick[kk] - h->fbase[f];
    const int mypicks = (kk + 1 < ngl ? h->gpick[kk + 1] : total) - h->gpick[kk];
    int avail = h->retn[f] + h->nsn[f] - base;
    avail = avail < 0 ? 0 : (avail > mypicks ? mypicks : avail);
    int comp = 0, viol = 0;
    serve_replay<HotX, BND>(h, i, f, t0, t_end, base, avail, comp, viol);
    if (comp) atomicAdd(&h->fcomp[f], comp);
    if (viol) atomicAdd(&h->fviol[f], viol);
  }
  GS_PW(23);
  __syncthreads();
  GS_PH(23);
  // 5. each function's queue bookkeeping once; on other threads, each node's
  //    coverage (max duration) and occupancy (Python sum of sm * duration in
  //    dispatch order, sim_engine.py:514-517)
#pragma unroll 1
  for (int x = tid; x < FP + G; x += NT) {
    if (x >= FP) {
      const int g = x - FP;
      const int ng = h->ngr[g];
      if (ng == 0) continue;
      // dispatch order (float path) or grant-slot order (integral: order-free)
      h->cov[g] += h->fullq[g] ? quantum : __longlong_as_double((long long)h->covbits[g]);
      h->occ[g] += token_occupancy(h, h->seg[g], ng) / 100.0;
      continue;
    }
    if (x >= F) continue;
    const int f = x;
    const int want = h->fpicks[f];
    const int comp = h->fcomp[f];
    if (want != 0 || comp != 0) xlh_books<BND>(h, f, want, comp);
    // the next step's _admit_arrivals (sim_engine.py:472-480) on the same
    // thread, behind the node threads' occupancy sums instead of on the next
    // step's critical path
    if (s + 1 < h->T) hot_admit<HotX, BND>(h, f, (double)w * h->ws + (double)(s + 1) * h->qs);
  }
  GS_PW(24);
  __syncthreads();
  GS_PH(24);
}

// per-function queue bookkeeping after the replay (step phase 5)
template <bool BND>
__device__ __forceinline__ void xlh_books(HotX* h, int f, int want, int comp) {
  {
    const int avail = h->retn[f] + h->nsn[f];
    const int taken = want < avail ? want : avail;
    const int retn = h->retn[f];
    const int from_ret = taken < retn ? taken : retn;
    const int from_ns = taken - from_ret;
    if (from_ret) {
      long long* r = &h->f_ret[(size_t)f * h->RET];
      for (int q = from_ret; q < retn; q++) r[q - from_ret] = r[q];
      h->retn[f] = retn - from_ret;
    }
    if (from_ns) {
      const int nsn = h->nsn[f] - from_ns;
      h->nsn[f] = nsn;
      const int limit = BND ? h->maxq[f] : -1;
      if (limit >= 0) {
        h->rhead[f] = (h->rhead[f] + from_ns) % limit;
      } else if (nsn > 0) {
        int w2 = h->nsw[f], i2 = h->nsi[f] + from_ns, n2 = h->nswn[f];
        while (i2 >= n2) {
          i2 -= n2;
          do { w2++; n2 = h->count(f, w2); } while (n2 == 0);
        }
        h->nsw[f] = w2; h->nsi[f] = i2; h->nswn[f] = n2;
      }
    }
    h->pinned[f] += taken - comp;
    h->qlen[f] -= comp;
    h->wcomp[f] += comp;
    h->wviol[f] += h->fviol[f];
  }
}

}  // namespace gs

namespace gs {

// ---------------------------------------------------------------------------
// CTA-wide window begin for the XL class (same results as window_begin):
// warm-up registration + ledger reset, arrivals, the registered list sorted by
// (node, pod_id), node segments, per-function lists -- with block sorts in the
// idle shared-memory block instead of one warp's sort in HBM.
// ---------------------------------------------------------------------------

// exclusive block scan of one int per thread; returns the total in *total
__device__ int xl_block_exscan(int v, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;      // inclusive warp prefix
  }
  __syncthreads();
  const int before = wid > 0 ? warp_tot[wid - 1] : 0;
  *total = warp_tot[nw - 1];
  __syncthreads();
  return before + x - v;
}

// block bitonic sort of q (power of two) (a, b, v) triples in shared memory
__device__ void xl_block_sort(unsigned long long* A, unsigned long long* B, int* V, int q) {
#pragma unroll 1
  for (int k = 2; k <= q; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll 1
      for (int t = threadIdx.x; t < (q >> 1); t += blockDim.x) {
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int l = i | j;
        const bool up = (i & k) == 0;
        const unsigned long long ai = A[i], bi = B[i], al = A[l], bl = B[l];
        const int vi = V[i], vl = V[l];
        if (trip_less(al, bl, vl, ai, bi, vi) == up) {
          A[i] = al; B[i] = bl; V[i] = vl;
          A[l] = ai; B[l] = bi; V[l] = vi;
        }
      }
      __syncthreads();
    }
  }
}

// all threads; `scr` = shared scratch of `bytes`.  Returns false when the
// registered set is too large for the scratch (caller then uses window_begin).
__device__ bool xl_window_begin(Ctx& c, int w, char* scr, size_t bytes, int* warp_tot) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int phi = pod_high(c);
  int q = 1;
  while (q < phi) q <<= 1;
  if ((size_t)q * 20 > bytes) return false;
  unsigned long long* A = reinterpret_cast<unsigned long long*>(scr);
  unsigned long long* B = A + q;
  int* V = reinterpret_cast<int*>(B + q);
  __shared__ int next_warm_s;
  if (tid == 0) next_warm_s = 0x7fffffff;
  __syncthreads();
  // warm-up + ledger reset (sim_engine.py:454-460, token_backend.py:213-218);
  // each thread owns a contiguous chunk of slots so the registered list can be
  // compacted in slot order
  const int per = (phi + NT - 1) / NT;
  const int s0 = tid * per, s1 = min(phi, s0 + per);
  int nreg = 0, nw = 0x7fffffff;
#pragma unroll 1
  for (int slot = s0; slot < s1; slot++) {
    int fl = c.t->p_flags[slot];
    if ((fl & PF_PLACED) && !(fl & PF_REG)) {
      if (c.t->p_warm[slot] <= w) fl |= PF_REG;
      else nw = min(nw, c.t->p_warm[slot]);
    }
    if (fl & PF_REG) { c.t->p_qused[slot] = 0.0; fl &= ~PF_GRANT; nreg++; }
    c.t->p_flags[slot] = fl;
  }
  if (nw != 0x7fffffff) atomicMin(&next_warm_s, nw);
#pragma unroll 1
  for (int f = tid; f < c.F; f += NT) {            // _generate_arrivals (:462-470)
    const int n = c.count(f, w);
    c.t->f_warr[f] = n;
    if (n > 0) {
      if (c.t->f_fn[f] == 0) { c.t->f_fw[f] = w; c.t->f_fi[f] = 0; }
      c.t->f_fn[f] += n;
    }
  }
  int nr = 0;
  int pos = xl_block_exscan(nreg, warp_tot, &nr);
  // registered pods keyed (node, pod_id); padding sorts last
#pragma unroll 1
  for (int slot = s0; slot < s1; slot++) {
    if (!(c.t->p_flags[slot] & PF_REG)) continue;
    A[pos] = (unsigned long long)c.t->p_node[slot];
    B[pos] = c.t->p_okey[slot];
    V[pos] = slot;
    pos++;
  }
#pragma unroll 1
  for (int i = nr + tid; i < q; i += NT) { A[i] = ~0ull; B[i] = ~0ull; V[i] = 0x7fffffff; }
  __syncthreads();
  xl_block_sort(A, B, V, q);
#pragma unroll 1
  for (int i = tid; i < nr; i += NT) c.t->s_rl[i] = V[i];
#pragma unroll 1
  for (int g = tid; g <= c.G; g += NT) {           // lower bound of node g
    int lo = 0, hi = nr;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int)A[mid] < g) lo = mid + 1; else hi = mid;
    }
    c.t->n_seg[g] = lo;
  }
  __syncthreads();
  // per-function lists in (node, pod_id) order: sort (function, list index)
#pragma unroll 1
  for (int i = tid; i < q; i += NT) {
    if (i < nr) {
      const int slot = V[i];
      A[i] = (unsigned long long)c.t->p_fn[slot];
      B[i] = (unsigned long long)i;
    } else {
      A[i] = ~0ull; B[i] = ~0ull; V[i] = 0x7fffffff;
    }
  }
  __syncthreads();
  xl_block_sort(A, B, V, q);
#pragma unroll 1
  for (int i = tid; i < nr; i += NT) c.t->s_fl[i] = V[i];
#pragma unroll 1
  for (int f = tid; f <= c.F; f += NT) {
    int lo = 0, hi = nr;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int)A[mid] < f) lo = mid + 1; else hi = mid;
    }
    c.t->f_loff[f] = lo;
  }
  if (tid == 0) {
    c.sh->next_warm = next_warm_s;
    c.sh->n_reg = nr;
    c.sh->pod_steps += (long long)nr * c.T;
  }
  __syncthreads();
  return true;
}

// ---------------------------------------------------------------------------
// XL epoch (sim_engine.py:409-430, autoscaler.py:81-160) on the whole CTA.
//
// A function's scaling decision reads only its own running set, its request
// history and its profile, so the decisions are independent: every warp
// decides functions wid, wid + 16, ... (sort of the running set by
// (efficiency, pod_id), Python sum of the throughputs, scale-up count + ideal
// point, or the scale-down prefix length) into a per-function record, and
// warp 0 then applies the records in function order -- the make_pod /
// remove_pod sequence, slot reuse, decision counter and first error are
// exactly the sequential loop's.  place_batch / restructure stay on warp 0.
// ---------------------------------------------------------------------------

// ascending bitonic sort of n (a, b, v) triples in (warp-private) memory
__device__ void xl_warp_sort_mem(unsigned long long* A, unsigned long long* B, int* V, int n,
                                 int lane) {
  int q = 1;
  while (q < n) q <<= 1;
#pragma unroll 1
  for (int i = n + lane; i < q; i += 32) { A[i] = ~0ull; B[i] = ~0ull; V[i] = 0x7fffffff; }
  __syncwarp();
#pragma unroll 1
  for (int k = 2; k <= q; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll 1
      for (int t = lane; t < (q >> 1); t += 32) {
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int l = i | j;
        const bool up = (i & k) == 0;
        const unsigned long long ai = A[i], bi = B[i], al = A[l], bl = B[l];
        const int vi = V[i], vl = V[l];
        if (trip_less(al, bl, vl, ai, bi, vi) == up) {
          A[i] = al; B[i] = bl; V[i] = vl;
          A[l] = ai; B[l] = bi; V[l] = vi;
        }
      }
      __syncwarp();
    }
  }
}

// decision of function f by one warp; the running set s_list[f_loff[f] ..)
// is left sorted in place.  kind: 0 none, 1 up (cnt, ideal), 2 down (nrem).
__device__ void xl_decide(Ctx& c, int f, int* kind, int* ideal_o, int* nrem_o, long long* cnt_o,
                          unsigned long long* A, unsigned long long* B, int* V) {
  const int lane = c.lane;
  const int start = c.t->f_loff[f];
  const int n = c.t->f_loff[f + 1] - start;
  int* lst = c.t->s_list + start;
  double thr = 0.0;
  PySum sup;
  sup.reset();
  if (n <= 32) {
    unsigned long long a = ~0ull, b = ~0ull;
    int v = 0x7fffffff;
    if (lane < n) {
      const int slot = lst[lane];
      a = ord_key(c.pt(f, c.t->p_pt[slot]).rpr);
      b = c.t->p_okey[slot];
      v = slot;
    }
    warp_sort_regs(a, b, v, n, lane);
    __syncwarp();
    if (lane < n) {
      thr = c.pt(f, c.t->p_pt[v]).thr;
      lst[lane] = v;
    }
#pragma unroll 1
    for (int i = 0; i < n; i++) sup.add(__shfl_sync(FULL, thr, i));
  } else {
#pragma unroll 1
    for (int i = lane; i < n; i += 32) {
      const int slot = lst[i];
      A[i] = ord_key(c.pt(f, c.t->p_pt[slot]).rpr);
      B[i] = c.t->p_okey[slot];
      V[i] = slot;
    }
    __syncwarp();
    xl_warp_sort_mem(A, B, V, n, lane);
#pragma unroll 1
    for (int i = lane; i < n; i += 32) lst[i] = V[i];
#pragma unroll 1
    for (int i = 0; i < n; i++) sup.add(c.pt(f, c.t->p_pt[V[i]]).thr);
  }
  const int hn = c.t->f_hn[f];
  const double* h = &c.t->f_hist[3 * f];
  double pred = h[(hn - 1) % 3];              // max(history[-3:])
#pragma unroll 1
  for (int k = 2; k <= 3 && k <= hn; k++) {
    const double x = h[(hn - k) % 3];
    if (x > pred) pred = x;
  }
  const double gap = pred - sup.value();      // rps_gap
  int kd = 0, idl = -1, nrem = 0;
  long long cnt = 0;
  if (gap > 0) {                              // scale_up: autoscaler.py:103-131
    const int pe = c.fs[f].p_eff;
    const double t_eff = c.pt(f, pe).thr;
    if (!(t_eff > 0)) {                       // autoscaler.py:115-117
      kd = 3;
    } else {
      const double nd = floor(gap / t_eff);
      const double residual = gap - nd * t_eff;
      cnt = (long long)nd;
      if (residual > 0) {
        idl = ideal_point(c, f, residual);
        if (idl < 0) idl = pe;
      }
      kd = 1;
    }
  } else if (gap < 0) {                       // scale_down: autoscaler.py:134-149
    double delta = gap;
#pragma unroll 1
    for (int i = 0; i < n && delta < 0; i++) {
      const double t = n <= 32 ? __shfl_sync(FULL, thr, i) : c.pt(f, c.t->p_pt[V[i]]).thr;
      if (delta + t > 0) break;
      delta += t;
      nrem++;
    }
    kd = 2;
  }
  if (lane == 0) { kind[f] = kd; ideal_o[f] = idl; nrem_o[f] = nrem; cnt_o[f] = cnt; }
  __syncwarp();
}

// _carve + _subdivide + _prune_contained (packer.py:196-242) on the whole
// CTA: the split parts are compacted in (rect, part) order into shared `tmp`,
// each warp decides containment for its rects (lanes over the others), and
// the survivors are written back to `list` in order.  Returns the new count,
// or -1 (list untouched) when it would exceed `cap` -- carve()'s contract.
__device__ int xl_carve(int4* list, int n, int4 placed, int cap, int4* tmp, int* kpos,
                        int* warp_tot) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int nw = NT >> 5;
  int m = 0;
#pragma unroll 1
  for (int s0 = 0; s0 < n; s0 += NT) {
    const int j = s0 + tid;
    int4 parts[4];
    int np = 0;
    if (j < n) {
      const int4 r = list[j];
      if (!r_intersects(r, placed)) {
        parts[np++] = r;
      } else {
        const int ix = max(r.x, placed.x), iy = max(r.y, placed.y);
        const int ix2 = min(r.x + r.z, placed.x + placed.z);
        const int iy2 = min(r.y + r.w, placed.y + placed.w);
        if (ix > r.x) parts[np++] = make_int4(r.x, r.y, ix - r.x, r.w);
        if (ix2 < r.x + r.z) parts[np++] = make_int4(ix2, r.y, r.x + r.z - ix2, r.w);
        if (iy > r.y) parts[np++] = make_int4(r.x, r.y, r.z, iy - r.y);
        if (iy2 < r.y + r.w) parts[np++] = make_int4(r.x, iy2, r.z, r.y + r.w - iy2);
      }
    }
    int tot;
    const int off = m + xl_block_exscan(np, warp_tot, &tot);
#pragma unroll 1
    for (int k = 0; k < np; k++) tmp[off + k] = parts[k];
    m += tot;
  }
  __syncthreads();
  // prune: drop rects contained in another; exact duplicates keep the first
#pragma unroll 1
  for (int i = wid; i < m; i += nw) {
    const int4 r = tmp[i];
    bool kill = false;
#pragma unroll 1
    for (int j0 = 0; j0 < m && !kill; j0 += 32) {
      const int j = j0 + lane;
      bool k = false;
      if (j < m && j != i) {
        const int4 o = tmp[j];
        k = r_contains(o, r) && !(r_eq(r, o) && i < j);
      }
      kill = __any_sync(FULL, k);
    }
    if (lane == 0) kpos[i] = kill ? 0 : 1;
  }
  __syncthreads();
  int kept = 0;
#pragma unroll 1
  for (int s0 = 0; s0 < m; s0 += NT) {
    const int i = s0 + tid;
    const int kf = i < m ? kpos[i] : 0;
    int tot;
    const int off = kept + xl_block_exscan(kf, warp_tot, &tot);
    if (kf) kpos[i] = (off << 1) | 1;
    kept += tot;
  }
  if (kept > cap) return -1;                   // uniform: kept is the block total
  __syncthreads();
#pragma unroll 1
  for (int i = tid; i < m; i += NT) {
    const int kp = kpos[i];
    if (kp & 1) list[kp >> 1] = tmp[i];
  }
  return kept;
}

// footprint (memory_model.py:60-72) of node g on one warp: the terms are
// formed lane-parallel and added in resident (dict insertion) order, so the
// double equals refresh_footprint's sequential loop.
__device__ double xl_footprint(Ctx& c, int g) {
  const int lane = c.lane;
  const int2* res = &c.t->n_res[g * c.F];
  const int nres = c.t->n_nres[g];
  const bool sharing = (c.flags & GS_FLAG_SHARING) != 0;
  double total = 0.0;
#pragma unroll 1
  for (int i0 = 0; i0 < nres; i0 += 32) {
    const int i = i0 + lane;
    double term = 0.0;
    bool use = false;
    if (i < nres) {
      const int2 e = res[i];
      if (e.y > 0) {
        const gs_function_t& fs = c.fs[e.x];
        term = sharing ? fs.mem_server_mb + (double)e.y * fs.mem_runtime_mb
                       : (double)e.y * fs.mem_noshare_mb;
        use = true;
      }
    }
    const unsigned m = __ballot_sync(FULL, use);
    const int lim = min(32, nres - i0);
#pragma unroll 1
    for (int k = 0; k < lim; k++) {
      const double t = __shfl_sync(FULL, term, k);
      if ((m >> k) & 1u) total += t;
    }
  }
  if (lane == 0) c.t->n_fp[g] = total;
  __syncwarp();
  return total;
}

// memory_model.add_pod (memory_model.py:49-50) + footprint, one warp
__device__ double xl_mem_add(Ctx& c, int g, int f) {
  const int lane = c.lane;
  int* cnt = &c.t->n_cnt[g * c.F + f];
  int2* res = &c.t->n_res[g * c.F];
  const int nres = c.t->n_nres[g];
  const int had = *cnt;
  if (had > 0) {
#pragma unroll 1
    for (int i0 = 0; i0 < nres; i0 += 32) {
      const int i = i0 + lane;
      const unsigned m = __ballot_sync(FULL, i < nres && res[i].x == f);
      if (m) {
        if (lane == __ffs(m) - 1) res[i].y++;
        break;
      }
    }
  } else if (lane == 0) {
    res[nres] = make_int2(f, 1);
    c.t->n_nres[g] = nres + 1;
  }
  if (lane == 0) *cnt = had + 1;
  __syncwarp();
  return xl_footprint(c, g);
}

// memory_model.remove_pod (memory_model.py:52-58) + footprint, one warp:
// `del resident[f]` keeps the order of the others
__device__ void xl_mem_remove(Ctx& c, int g, int f) {
  const int lane = c.lane;
  int* cnt = &c.t->n_cnt[g * c.F + f];
  int2* res = &c.t->n_res[g * c.F];
  const int nres = c.t->n_nres[g];
  int at = -1;
#pragma unroll 1
  for (int i0 = 0; i0 < nres; i0 += 32) {
    const int i = i0 + lane;
    const unsigned m = __ballot_sync(FULL, i < nres && res[i].x == f);
    if (m) { at = i0 + __ffs(m) - 1; break; }
  }
  if (at >= 0) {
    const int2 e = res[at];
    if (e.y == 1) {
#pragma unroll 1
      for (int j0 = at; j0 + 1 < nres; j0 += 32) {   // shift left, chunk by chunk
        const int j = j0 + lane;
        int2 nx = make_int2(0, 0);
        if (j + 1 < nres) nx = res[j + 1];
        __syncwarp();
        if (j + 1 < nres) res[j] = nx;
        __syncwarp();
      }
      if (lane == 0) c.t->n_nres[g] = nres - 1;
    } else if (lane == 0) {
      res[at].y = e.y - 1;
    }
  }
  if (lane == 0) (*cnt)--;
  __syncwarp();
  xl_footprint(c, g);
}

// _remove_pod (sim_engine.py:377-392), one warp; same effects and error
// order as remove_pod
__device__ void xl_remove_pod(Ctx& c, int slot) {
  const int fl = c.t->p_flags[slot];
  if (fl & PF_RETRY) {
    if (c.lane == 0) free_slot(c, slot);
    __syncwarp();
    return;
  }
  const int f = c.t->p_fn[slot];
  const int g = c.t->p_node[slot];
  int ok = 1;
  if (c.lane == 0) {
    if (fl & PF_CUR) {
      return_request(c, f, pack_id(c.t->p_cw[slot], c.t->p_ci[slot]));
      c.t->f_pinned[f]--;
    }
    const int n = c.t->n_nfree[g];
    if (n >= c.R) {
      set_error(c, GS_ERR_CAPACITY, GS_CAP_RECTS, g, 0);
      ok = 0;
    } else {
      c.t->n_rect[g * c.R + n] =
          make_int4(c.t->p_x[slot], c.t->p_y[slot], c.t->p_w[slot], c.t->p_h[slot]);
      c.t->n_nfree[g] = n + 1;
    }
  }
  ok = __shfl_sync(FULL, ok, 0);
  if (!ok) return;
  xl_mem_remove(c, g, f);
  if (c.lane == 0) {
    c.t->n_nplaced[g]--;
    free_slot(c, slot);
  }
  __syncwarp();
}

// scale_up's pod creations for one function (autoscaler.py:103-131 ->
// _make_pod, sim_engine.py:337-368), one warp: pod i takes the i-th slot off
// the free stack and pod counter pctr + i, exactly as `total` sequential
// make_pod calls; the first failing call (zero-rate point, empty stack) stops
// the sequence with make_pod's error.
__device__ void xl_make_pods(Ctx& c, int f, long long n_eff, int ideal, int warm) {
  const int lane = c.lane;
  const gs_function_t& fs = c.fs[f];
  const int pe = fs.p_eff;
  const long long total = n_eff + (ideal >= 0 ? 1 : 0);
  const int top = c.sh->free_top;
  const bool pe_ok = c.pt(f, pe).rate_ok != 0;
  const bool id_ok = ideal < 0 || c.pt(f, ideal).rate_ok != 0;
  // first failing index and its error
  long long stop = total;
  int code = 0, detail = 0, a0 = 0, a1 = 0;
  if (n_eff > 0 && !pe_ok) { stop = 0; code = GS_ERR_VALIDATION; a0 = f; a1 = pe; }
  else if (ideal >= 0 && !id_ok) { stop = n_eff; code = GS_ERR_VALIDATION; a0 = f; a1 = ideal; }
  if (top < stop) { stop = top; code = GS_ERR_CAPACITY; detail = GS_CAP_PODS; a0 = c.P; a1 = 0; }
  const int made = (int)stop;
  const int ctr0 = c.t->f_pctr[f];
#pragma unroll 1
  for (int i = lane; i < made; i += 32) {
    const int k = i < n_eff ? pe : ideal;
    const gs_point_t& p = c.pt(f, k);
    const int slot = c.t->s_free[top - 1 - i];
    const int ctr = ctr0 + i;
    c.t->p_fn[slot] = f; c.t->p_pt[slot] = k; c.t->p_node[slot] = -1; c.t->p_flags[slot] = PF_ALIVE;
    c.t->p_warm[slot] = warm; c.t->p_ctr[slot] = ctr; c.t->p_x[slot] = 0; c.t->p_y[slot] = 0;
    c.t->p_w[slot] = p.rect_w; c.t->p_h[slot] = p.rect_h; c.t->p_cw[slot] = 0; c.t->p_ci[slot] = 0;
    c.t->p_okey[slot] = pod_okey(fs, c.splits, ctr);
    c.t->p_sm[slot] = p.sm_eff;
    c.t->p_qlim[slot] = p.quota;
    c.t->p_qreq[slot] = p.quota;
    c.t->p_qused[slot] = 0.0; c.t->p_busy[slot] = 0.0; c.t->p_invr[slot] = p.inv_rate;
    c.t->p_crem[slot] = 0.0; c.t->p_carr[slot] = 0.0; c.t->p_dur[slot] = 0.0;
  }
  __syncwarp();
  if (lane == 0) {
    c.sh->free_top = top - made;
    if (c.sh->free_top < c.sh->min_free) c.sh->min_free = c.sh->free_top;
    c.t->f_pctr[f] = ctr0 + made;
    if (code) set_error(c, code, detail, a0, a1);
  }
  __syncwarp();
}

// _place_batch (sim_engine.py:394-407) on the whole CTA: the batch is
// compacted and sorted (-area, pod_id) in shared memory by every thread, and
// each request's best_match (packer.py:169-193) scans the fleet's free rects
// with all threads -- tpn threads per node, a block argmin over the same
// (area gap, node, y, x, list index) key, so the choice is the warp
// version's; every warp reduces the per-warp winners itself, so the whole CTA
// follows the same sequence of decisions.  The carve runs CTA-wide
// (xl_carve); the memory ledger and the pod's fields are one thread's.
// When they fit, the fleet's free-rect lists, free counts, footprints and
// resident bits are staged in shared memory for the batch (written back at
// the end), so a placement touches HBM only for the memory ledger.
// Returns false when the batch does not fit the scratch (caller runs
// place_batch).
__device__ bool xl_place_batch(Ctx& c, char* scr, size_t bytes, int* warp_tot) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int nw = NT >> 5;
  const int phi = pod_high(c);
  int q = 1;
  while (q < phi) q <<= 1;
  const size_t carve_n = 4 * (size_t)c.R + 8;
  const size_t base_bytes = (size_t)q * 36 + carve_n * 20;
  if (base_bytes > bytes) return false;
  unsigned long long* A = reinterpret_cast<unsigned long long*>(scr);
  unsigned long long* B = A + q;
  double* dres = reinterpret_cast<double*>(B + q);      // admit delta if resident / not
  double* dnew = dres + q;
  int4* tmp = reinterpret_cast<int4*>(dnew + q);
  int* V = reinterpret_cast<int*>(tmp + carve_n);
  int* kpos = V + q;
  // staged fleet state (rects [G*R], footprints, free counts, resident bits)
  const int fwords = (c.F + 31) >> 5;
  const size_t stage_bytes = (size_t)c.G * c.R * 16 + (size_t)c.G * 8 + (size_t)c.G * 4 +
                             (size_t)c.G * fwords * 4;
  const bool staged = base_bytes + stage_bytes + 64 <= bytes;
  int4* rects = c.t->n_rect;
  int* nfree = c.t->n_nfree;
  double* fp = c.t->n_fp;
  unsigned* rbits = nullptr;
  if (staged) {
    int4* st = reinterpret_cast<int4*>((reinterpret_cast<size_t>(kpos + carve_n) + 15) & ~(size_t)15);
    rects = st;
    fp = reinterpret_cast<double*>(st + (size_t)c.G * c.R);
    nfree = reinterpret_cast<int*>(fp + c.G);
    rbits = reinterpret_cast<unsigned*>(nfree + c.G);
#pragma unroll 1
    for (int g = wid; g < c.G; g += nw) {
      const int nf = c.t->n_nfree[g];
#pragma unroll 1
      for (int j = lane; j < nf; j += 32) rects[g * c.R + j] = c.t->n_rect[g * c.R + j];
      if (lane == 0) { nfree[g] = nf; fp[g] = c.t->n_fp[g]; }
#pragma unroll 1
      for (int k = lane; k < fwords; k += 32) {
        unsigned wbits = 0;
#pragma unroll 1
        for (int b = 0; b < 32 && (k << 5) + b < c.F; b++)
          if (c.t->n_cnt[g * c.F + (k << 5) + b] > 0) wbits |= 1u << b;
        rbits[g * fwords + k] = wbits;
      }
    }
  }
  __shared__ BestKey wbest[32];
  __shared__ long long wscan[32];
  // batch = alive, unplaced pods, compacted in slot order
  const int per = (phi + NT - 1) / NT;
  const int s0 = tid * per, s1 = min(phi, s0 + per);
  int mine = 0;
#pragma unroll 1
  for (int slot = s0; slot < s1; slot++)
    mine += (c.t->p_flags[slot] & (PF_ALIVE | PF_PLACED)) == PF_ALIVE;
  int nb = 0;
  int pos = xl_block_exscan(mine, warp_tot, &nb);
#pragma unroll 1
  for (int slot = s0; slot < s1; slot++) {
    const int fl = c.t->p_flags[slot];
    if ((fl & (PF_ALIVE | PF_PLACED)) != PF_ALIVE) continue;
    A[pos] = ~(unsigned long long)((long long)c.t->p_w[slot] * c.t->p_h[slot]);   // descending area
    B[pos] = c.t->p_okey[slot];
    V[pos] = slot;
    c.t->p_flags[slot] = fl & ~PF_RETRY;
    pos++;
  }
  int qb = 1;
  while (qb < nb) qb <<= 1;
#pragma unroll 1
  for (int i = nb + tid; i < qb; i += NT) { A[i] = ~0ull; B[i] = ~0ull; V[i] = 0x7fffffff; }
  __syncthreads();
  GS_EPOCH_TIC(p0_);
  xl_block_sort(A, B, V, qb);
  // entry i's best_match inputs: A = (w, h), B = function, admit deltas
  const bool sharing = (c.flags & GS_FLAG_SHARING) != 0;
#pragma unroll 1
  for (int i = tid; i < nb; i += NT) {
    const int slot = V[i];
    const int f = c.t->p_fn[slot];
    A[i] = ((unsigned long long)(unsigned)c.t->p_w[slot] << 32) | (unsigned)c.t->p_h[slot];
    B[i] = (unsigned long long)f;
    const gs_function_t& fs = c.fs[f];
    dres[i] = sharing ? fs.mem_runtime_mb : fs.mem_noshare_mb;
    dnew[i] = sharing ? fs.mem_runtime_mb + fs.mem_server_mb : fs.mem_noshare_mb;
  }
  const double cap_mb = c.cap_mb;
  int tpn = 1;                                 // threads per node (power of two)
  while (tpn * 2 * c.G <= NT && tpn < 32) tpn <<= 1;
  const int sub = tid & (tpn - 1);
  const int gstride = NT / tpn;
  __syncthreads();
  GS_EPOCH_TIC(p1_);
  if (tid == 0) { GS_EPOCH_ADD(8, p1_ - p0_); }
  int i = 0;
#pragma unroll 1
  while (i < nb) {
    GS_EPOCH_TIC(p2_);
    const unsigned long long wh = A[i];
    const int f = (int)B[i];
    const double d_res = dres[i], d_new = dnew[i];
    const int rw = (int)(wh >> 32), rh = (int)(wh & 0xffffffffu);
    const long long rarea = (long long)rw * rh;
    BestKey best;
    best.idx = -1; best.k0 = 0; best.a = best.b = best.d = 0;
    long long scans = 0;
#pragma unroll 1
    for (int g = tid / tpn; g < c.G; g += gstride) {
      const bool res = staged ? ((rbits[g * fwords + (f >> 5)] >> (f & 31)) & 1u) != 0
                              : c.t->n_cnt[g * c.F + f] > 0;
      if (!(fp[g] + (res ? d_res : d_new) <= cap_mb)) continue;   // memory_model.admit
      const int nf = nfree[g];
      if (sub == 0) scans += nf;
      const int4* rl = &rects[g * c.R];
#pragma unroll 1
      for (int j = sub; j < nf; j += tpn) {
        const int4 r = rl[j];
        if (rw <= r.z && rh <= r.w) {
          BestKey k;
          k.k0 = r_area(r) - rarea; k.a = g; k.b = r.y; k.d = r.x; k.idx = g * c.R + j;
          if (bk_less(k, best)) best = k;
        }
      }
    }
    best = warp_argmin(best);
    scans = warp_sum_ll(scans);
    if (lane == 0) { wbest[wid] = best; wscan[wid] = scans; }
    __syncthreads();
    GS_EPOCH_TIC(p3_);
    if (tid == 0) { GS_EPOCH_ADD(11, p3_ - p2_); GS_EPOCH_ADD(10, 1); }
    BestKey k;                                 // every warp: the block winner
    k.idx = -1; k.k0 = 0; k.a = k.b = k.d = 0;
    long long sc = 0;
    if (lane < nw) { k = wbest[lane]; sc = wscan[lane]; }
    k = warp_argmin(k);
    sc = warp_sum_ll(sc);
    if (k.idx >= 0) {
      const int g = k.a;
      const int4 chosen = rects[k.idx];
      const int n = nfree[g];
      if (tid == 0) { c.sh->rect_scans += sc; c.sh->attempts++; }
      const int nn = xl_carve(&rects[g * c.R], n, make_int4(chosen.x, chosen.y, rw, rh),
                              c.R, tmp, kpos, warp_tot);
      if (wid == 0 && nn >= 0) {
        const double tot = xl_mem_add(c, g, f);
        if (lane == 0 && staged) {
          fp[g] = tot;
          rbits[g * fwords + (f >> 5)] |= 1u << (f & 31);
        }
      }
      if (tid == 0) {
        if (nn < 0) {
          set_error(c, GS_ERR_CAPACITY, GS_CAP_RECTS, g, 0);
        } else {                               // place() bookkeeping (packer.py:245-261)
          const int slot = V[i];
          nfree[g] = nn;
          c.t->n_nfree[g] = nn;
          c.t->n_nplaced[g]++;
          c.t->p_node[slot] = g;
          c.t->p_x[slot] = chosen.x;
          c.t->p_y[slot] = chosen.y;
          c.t->p_flags[slot] = (c.t->p_flags[slot] | PF_PLACED) & ~PF_RETRY;
        }
      }
      i = nn < 0 ? nb : i + 1;
      GS_EPOCH_TIC(p5_);
      if (tid == 0) { GS_EPOCH_ADD(9, p5_ - p3_); }
    } else {
      // identical requests that follow fail too (nothing changed in between)
      int j = nb;
#pragma unroll 1
      for (int k0 = i + 1; k0 < nb; k0 += 32) {
        const int kk = k0 + lane;
        const bool differs = kk < nb && (A[kk] != wh || (int)B[kk] != f);
        const unsigned bal = __ballot_sync(FULL, differs);
        if (bal) { j = k0 + __ffs(bal) - 1; break; }
      }
#pragma unroll 1
      for (int kk = i + tid; kk < j; kk += NT) c.t->p_flags[V[kk]] |= PF_RETRY;
      if (tid == 0) {
        const int len = j - i;
        c.sh->attempts += len;
        c.sh->win_failures += len;
        c.sh->rect_scans += sc * len;
      }
      i = j;
    }
    __syncthreads();
  }
  if (staged) {                                // write the free-rect lists back
#pragma unroll 1
    for (int g = wid; g < c.G; g += nw) {
      const int nf = nfree[g];
#pragma unroll 1
      for (int j = lane; j < nf; j += 32) c.t->n_rect[g * c.R + j] = rects[g * c.R + j];
    }
    __syncthreads();
  }
  return true;
}

// all threads; `scr` = idle shared scratch of `bytes`.  Returns false when a
// running set is too large for a warp's slice (caller runs run_epoch).
__device__ bool xl_run_epoch(Ctx& c, int w, char* scr, size_t bytes, XlShared* xs) {
  const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool w0 = wid == 0;
  GS_EPOCH_TIC(e0_);
  if (w0) group_alive_by_fn(c);
  GS_EPOCH_TIC(eg_);
  if (threadIdx.x == 0) { GS_EPOCH_ADD(12, eg_ - e0_); }
  long long* cnt = reinterpret_cast<long long*>(scr);
  int* kind = reinterpret_cast<int*>(cnt + c.F);
  int* ideal = kind + c.F;
  int* nrem = ideal + c.F;
  const size_t rec = ((size_t)c.F * 20 + 15) & ~(size_t)15;
  if (rec > bytes) return false;
  const size_t slice = ((bytes - rec) / nw) & ~(size_t)15;
  const int cap = (int)(slice / 20);
  char* mine = scr + rec + slice * wid;
  unsigned long long* A = reinterpret_cast<unsigned long long*>(mine);
  int q = 1;
  while (q * 2 <= cap) q <<= 1;                // largest power of two that fits
  unsigned long long* B = A + q;
  int* V = reinterpret_cast<int*>(B + q);
  if (threadIdx.x == 0) xs->stop = 0;
  __syncthreads();
#pragma unroll 1
  for (int f = wid; f < c.F; f += nw) {
    if (c.t->f_loff[f + 1] - c.t->f_loff[f] > q) {   // does not fit: sequential epoch
      if (c.lane == 0) xs->stop = 1;
      break;
    }
    xl_decide(c, f, kind, ideal, nrem, cnt, A, B, V);
  }
  __syncthreads();
  if (xs->stop) return false;                  // nothing applied yet
  GS_EPOCH_TIC(ed_);
  if (threadIdx.x == 0) { GS_EPOCH_ADD(13, ed_ - e0_); }
  if (w0) {
#pragma unroll 1
    for (int f = 0; f < c.F; f++) {
      const int kd = kind[f];
      if (kd == 1) {
        const long long n_new = cnt[f];
        const int idl = ideal[f];
        const long long total = n_new + (idl >= 0 ? 1 : 0);
        if (c.lane == 0) c.sh->decisions += total;
        if (total > c.P) {
          if (c.lane == 0) set_error(c, GS_ERR_CAPACITY, GS_CAP_PODS, c.P, 1);
        } else if (total > 0) {
          xl_make_pods(c, f, n_new, idl, w + c.sc->cold_start_windows);
        }
      } else if (kd == 3) {
        if (c.lane == 0) set_error(c, GS_ERR_VALIDATION, GS_VAL_NO_THROUGHPUT, f, c.fs[f].p_eff);
      } else if (kd == 2) {
        const int* lst = c.t->s_list + c.t->f_loff[f];
        const int m = nrem[f];
#pragma unroll 1
        for (int i = 0; i < m; i++) {
          if (c.lane == 0) c.sh->decisions++;
          xl_remove_pod(c, lst[i]);
          if (failed(c)) break;
        }
      }
      if (failed(c)) break;
    }
  }
  __syncthreads();
  GS_EPOCH_TIC(e2_);
  if (threadIdx.x == 0) { GS_EPOCH_ADD(14, e2_ - ed_); }
  if (c.sh->err) return true;
  if (!xl_place_batch(c, scr, bytes, xs->warp_tot)) {
    if (w0) place_batch(c);
    __syncthreads();
  }
  GS_EPOCH_TIC(e3_);
  if (w0 && !failed(c)) {
#pragma unroll 1
    for (int g = 0; g < c.G; g++) {
      restructure(c, g);
      if (failed(c)) break;
    }
    if (!failed(c)) refresh_frag(c);
  }
  GS_EPOCH_TIC(e4_);
  if (threadIdx.x == 0) {
    GS_EPOCH_ADD(4, e2_ - e0_); GS_EPOCH_ADD(5, e3_ - e2_); GS_EPOCH_ADD(6, e4_ - e3_);
  }
  __syncthreads();
  return true;
}

}  // namespace gs
