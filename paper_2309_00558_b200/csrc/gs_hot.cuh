// gs_hot.cuh -- the quantum-step loop on a shared-memory working set.
//
// For the ~50 quantum steps of a window, a run's registered pods, functions
// and nodes never change membership (registration changes only at window
// boundaries, sim_engine.py:443-451), so the warp copies exactly that working
// set from its HBM arena into a per-warp shared-memory block (structure of
// arrays, compile-time capacities PC/FC/GC), runs all steps there, and writes
// the persistent fields back once per window.  HBM then only sees per-window
// traffic; the per-step state touches are LDS/STS.
//
// Per step (sim_engine.py:493-520):
//   complete  lanes = pods    q_used += duration (token_backend.py:190-210)
//   admit     lanes = fns     arrivals <= t0 + 1e-12 (sim_engine.py:472-480),
//                             head arrival time cached, one IEEE division per
//                             admitted request
//   queue     lanes = pods    build_queue key (-(q_req-q_used), pod_id) and its
//                             rank inside the node by counting (no sort network)
//   dispatch  lanes = nodes   head-blocking walk in rank order (token_backend.py:160-187)
//                             + coverage max + occupancy (Python sum, in order)
//   serve     lanes = fns     FIFO drain over the function's granted pods in
//                             (node, pod_id) order (sim_engine.py:514-552)
#pragma once
#include "gs_kernel.cuh"

namespace gs {

enum : int { GS_CAP_HOT = 5 };   // status detail: working set exceeds the size class
constexpr double NOT_REQ = __builtin_huge_val();   // key of a pod that requests no token

template <int PC_, int FC_, int GC_>
struct Hot {
  static constexpr int PC = PC_, FC = FC_, GC = GC_;
  static_assert(PC <= 256, "pod indices are stored in bytes");
  // registered pods of this window, in (node, pod_id) order
  // (a granted pod's duration min(quantum, q_lim - q_used) is recomputed where
  // needed: q_used does not change between dispatch and completion)
  double qused[PC], qreq[PC], qlim[PC], sm[PC], busy[PC], crem[PC], carr[PC], invr[PC];
  // build_queue key -(q_req - q_used) as a double (+inf: not requesting);
  // double compares tie -0.0 with 0.0 exactly like Python's tuple order
  double key[PC];
  long long cur[PC];
  int fnode[PC];
  // pod indices (PC <= 256) and flag bits (PF_CUR | PF_GRANT) fit in a byte
  unsigned char flags[PC];
  unsigned char order[PC], flist[PC], rank[PC];   // rank doubles as the serve phase's granted list
  // functions
  double farr[FC], slo[FC];
  int qlen[FC], pinned[FC], fw[FC], fi[FC], fcnt[FC], nsn[FC], nsw[FC], nsi[FC];
  int rhead[FC], retn[FC], wcomp[FC], wviol[FC], wdrop[FC], maxq[FC], ringoff[FC];
  int fwn[FC], nswn[FC];   // arrival counts of the cursor windows fw / nsw (cached)
  int favail[FC], fcarry[FC], fcomp[FC], fviol[FC];   // parallel-serve scratch
  int warr[FC], hn[FC];
  int loff[FC + 1];
  int coff[FC];
  // nodes
  double sr[GC], cov[GC], occ[GC];
  int seg[GC + 1];
  int cut[GC];
  unsigned long long covbits[GC];
  // per step: requesting SM (integral), grants, 2 = a partial token / 4 = a
  // full-quantum token; occupancy-sum cache of the last all-quantum step
  // (count occn, value occv; valid while the node's bits of the granted-pod
  // words gw are those of the previous non-idle step, gwp)
  int reqsm[GC], ngr[GC], ostate[GC], occn[GC];
  unsigned gw[(PC + 31) / 32], gwp[(PC + 31) / 32];
  int maycut[GC];                  // registered SM on the node can exceed 100 (per hot set)
  double occv[GC];
  int nplaced[GC];
  double fp[GC];
  // run constants (so the step loop needs no Ctx registers)
  const int32_t* counts;
  long long* f_ret;
  long long* f_ring;
  double ws, qs, quantum;
  int n, F, G, T, W, RET, integral, bounded;

  __device__ __forceinline__ int count(int f, int w) const { return counts[coff[f] + w]; }
  // token duration of a granted pod: min(quantum, q_limit - q_used) (token_backend.py:178)
  __device__ __forceinline__ double dur(int i) const {
    const double rem = qlim[i] - qused[i];
    return rem < quantum ? rem : quantum;
  }
  __device__ __forceinline__ double arrival(int f, int w, int i) const {
    // start + i * window_s / n, start = window * window_s (sim_engine.py:463,470)
    return (double)w * ws + ((double)i * ws) / (double)count(f, w);
  }
  __device__ __forceinline__ double arrival_n(int w, int i, int n) const {
    return (double)w * ws + ((double)i * ws) / (double)n;
  }
  // next generated request after (w, i); n = count(f, w) is kept in sync
  __device__ __forceinline__ void advance(int f, int& w, int& i, int& n) const {
    if (++i < n) return;
    i = 0;
    do { w++; n = w < W ? count(f, w) : 1; } while (n == 0);
  }
};

// size classes: (pods, functions, nodes).  XS (tiny fleets such as C1 / C5:
// <= 4 functions, <= 2 nodes) is small enough to run 8 CTAs of 4 warps per SM.
typedef Hot<32, 4, 2> HotXS;
typedef Hot<64, 12, 4> HotS;
typedef Hot<128, 32, 16> HotM;
typedef Hot<256, 64, 32> HotL;

template <class H>
__host__ __device__ constexpr bool fits(int n_reg, int F, int G) {
  return n_reg <= H::PC && F <= H::FC && G <= H::GC;
}

// compile-time capacities of a working-set type (HotX, the XL class's
// runtime-sized view, specialises this with "unbounded")
template <class H>
struct HotCap {
  static constexpr int PC = H::PC, FC = H::FC, GC = H::GC;
};

// loop bound of a warp-uniform 32-wide sweep over n <= CAP items: with
// CAP <= 32 at most one trip, known at compile time
template <int CAP>
__device__ __forceinline__ int trips32(int n) { return CAP <= 32 ? (n > 0 ? 1 : 0) : n; }

// fn(x) for x = lane, lane + 32, ... < n; a class whose capacity CAP fits one
// warp needs no loop (one predicated call, no back edge)
template <int CAP, class Fn>
__device__ __forceinline__ void lane_for(int lane, int n, Fn&& fn) {
  if constexpr (CAP <= 32) {
    if (lane < n) fn(lane);
  } else {
#pragma unroll 1
    for (int x = lane; x < n; x += 32) fn(x);
  }
}

// ---------------------------------------------------------------- load/store
template <class H>
__device__ bool hot_load(Ctx& c, H* h) {
  const int n = c.sh->n_reg;
  if (n > H::PC || c.F > H::FC || c.G > H::GC) return false;   // window runs on the arena
  lane_for<H::PC>(c.lane, n, [&](int i) {
    int s = c.t->s_rl[i];
    h->qused[i] = c.t->p_qused[s];
    h->qreq[i] = c.t->p_qreq[s];
    h->qlim[i] = c.t->p_qlim[s];
    h->sm[i] = c.t->p_sm[s];
    h->busy[i] = c.t->p_busy[s];
    h->crem[i] = c.t->p_crem[s];
    h->carr[i] = c.t->p_carr[s];
    h->invr[i] = c.t->p_invr[s];
    h->cur[i] = pack_id(c.t->p_cw[s], c.t->p_ci[s]);
    h->fnode[i] = c.t->p_fn[s] | (c.t->p_node[s] << 16);
    h->flags[i] = (unsigned char)(c.t->p_flags[s] & PF_CUR);
    h->order[i] = (unsigned char)i;
  });
  lane_for<H::FC>(c.lane, c.F, [&](int f) {
    h->qlen[f] = c.t->f_qlen[f]; h->pinned[f] = c.t->f_pinned[f];
    h->fw[f] = c.t->f_fw[f]; h->fi[f] = c.t->f_fi[f]; h->fcnt[f] = c.t->f_fn[f];
    h->nsn[f] = c.t->f_nsn[f]; h->nsw[f] = c.t->f_nsw[f]; h->nsi[f] = c.t->f_nsi[f];
    h->rhead[f] = c.t->f_rhead[f]; h->retn[f] = c.t->f_retn[f];
    h->wcomp[f] = 0; h->wviol[f] = 0; h->wdrop[f] = 0;
    h->warr[f] = c.t->f_warr[f]; h->hn[f] = c.t->f_hn[f];
    h->maxq[f] = c.fs[f].max_queue;
    h->ringoff[f] = c.t->f_ringoff[f];
    h->slo[f] = c.fs[f].slo_ms;
    h->farr[f] = h->fcnt[f] > 0 ? arrival_time(c, f, h->fw[f], h->fi[f]) : 0.0;
    h->fwn[f] = h->fcnt[f] > 0 ? c.count(f, h->fw[f]) : 1;
    h->nswn[f] = (h->nsn[f] > 0 && c.fs[f].max_queue < 0) ? c.count(f, h->nsw[f]) : 1;
  });
  for (int f = c.lane; f <= c.F; f += 32) h->loff[f] = c.t->f_loff[f];
  for (int g = c.lane; g < c.G; g += 32) {
    h->sr[g] = c.t->n_sr[g]; h->cov[g] = 0.0; h->occ[g] = 0.0; h->occn[g] = -1;
    int tot = 0;                     // the node's requesting SM is at most this
    for (int j = c.t->n_seg[g]; j < c.t->n_seg[g + 1]; j++) tot += (int)c.t->p_sm[c.t->s_rl[j]];
    h->maycut[g] = tot > (int)SM_LIMIT ? 1 : 0;
    h->nplaced[g] = c.t->n_nplaced[g]; h->fp[g] = c.t->n_fp[g];
  }
  for (int g = c.lane; g <= c.G; g += 32) h->seg[g] = c.t->n_seg[g];
  for (int f = c.lane; f < c.F; f += 32) h->coff[f] = c.fs[f].count_off;
  if (c.lane == 0) {
    h->n = n;
    h->counts = c.counts; h->f_ret = c.t->f_ret; h->f_ring = c.t->f_ring;
    h->ws = c.ws; h->qs = c.qs; h->quantum = c.quantum;
    h->F = c.F; h->G = c.G; h->T = c.T; h->W = c.W; h->RET = c.RET;
    // integral SM partitions (>= 1) and token durations > QUOTA_EPS keep every
    // occupancy sum exact in any term order (see hot_step); a quantum below
    // QUOTA_EPS would void that bound, so it takes the sequential float walk
    h->integral = (c.integral() && c.quantum >= QUOTA_EPS) ? 1 : 0;
    int bnd = 0;
    for (int f = 0; f < c.F; f++) bnd |= c.fs[f].max_queue >= 0;
    h->bounded = bnd;
  }
  __syncwarp();
  // s_fl holds arena slots in (node, pod_id) order per function; the hot
  // index of an arena slot is its position in s_rl (slot -> index via s_list).
  for (int i = c.lane; i < n; i += 32) c.t->s_list[c.t->s_rl[i]] = i;
  __syncwarp();
  for (int j = c.lane; j < n; j += 32) h->flist[j] = (unsigned char)c.t->s_list[c.t->s_fl[j]];
  __syncwarp();
  return true;
}

template <class H>
__device__ void hot_store(Ctx& c, H* h) {
  const int n = h->n;
  lane_for<H::PC>(c.lane, n, [&](int i) {
    int s = c.t->s_rl[i];
    c.t->p_qused[s] = h->qused[i];
    c.t->p_busy[s] = h->busy[i];
    c.t->p_crem[s] = h->crem[i];
    c.t->p_carr[s] = h->carr[i];
    c.t->p_cw[s] = id_w(h->cur[i]);
    c.t->p_ci[s] = id_i(h->cur[i]);
    c.t->p_flags[s] = (c.t->p_flags[s] & ~(PF_CUR | PF_GRANT)) | (h->flags[i] & PF_CUR);
  });
  lane_for<H::FC>(c.lane, c.F, [&](int f) {
    c.t->f_qlen[f] = h->qlen[f]; c.t->f_pinned[f] = h->pinned[f];
    c.t->f_fw[f] = h->fw[f]; c.t->f_fi[f] = h->fi[f]; c.t->f_fn[f] = h->fcnt[f];
    c.t->f_nsn[f] = h->nsn[f]; c.t->f_nsw[f] = h->nsw[f]; c.t->f_nsi[f] = h->nsi[f];
    c.t->f_rhead[f] = h->rhead[f]; c.t->f_retn[f] = h->retn[f];
    c.t->f_hn[f] = h->hn[f];
  });
  for (int g = c.lane; g < c.G; g += 32) c.t->n_sr[g] = h->sr[g];
  __syncwarp();
}

// ------------------------------------------------------------------- phases
// The step loop reads everything through `h` (shared memory): no Ctx, so the
// whole window stays in a handful of registers.
template <class H>
__device__ __noinline__ void hot_complete_sm(H* h, int lane) {
  // sm_running -= sm in token (dispatch) order, with the float-dust clamp;
  // only needed when SM partitions are not integers (else it is exactly 0)
  #pragma unroll 1
  for (int g = lane; g < h->G; g += 32) {
    double sr = h->sr[g];
    const int lo = h->seg[g];
    #pragma unroll 1
    for (int j = lo; j < lo + h->ngr[g]; j++) {       // the granted prefix of the order
      const int i = h->order[j];
      sr -= h->sm[i];
      if (sr < 0 && sr > -SM_EPS) sr = 0.0;
    }
    h->sr[g] = sr;
  }
}

template <class H>
__device__ __forceinline__ void hot_complete(H* h, int lane) {
  const int n = h->n;
  if (!h->integral) {
    hot_complete_sm(h, lane);
    __syncwarp();
  }
  lane_for<H::PC>(lane, n, [&](int i) {
    const int fl = h->flags[i];
    if (fl & PF_GRANT) {
      h->qused[i] += h->dur(i);
      h->flags[i] = (unsigned char)(fl & ~PF_GRANT);
    }
  });
}

template <class H, bool BND>
__device__ __forceinline__ void hot_admit(H* h, int f, double t0) {
  int cnt = h->fcnt[f];
  if (cnt == 0) return;
  double a = h->farr[f];
  const double now = t0 + TIME_EPS;
  if (!(a <= now)) return;
  int w = h->fw[f], i = h->fi[f], wn = h->fwn[f];
  const int limit = BND ? h->maxq[f] : -1;
  int qlen = h->qlen[f], nsn = h->nsn[f], drop = 0;
  #pragma unroll 1
  while (true) {
    const int aw = w, ai = i, an = wn;
    cnt--;
    if (cnt > 0) h->advance(f, w, i, wn);
    if (limit >= 0 && qlen >= limit) {
      drop++;
    } else {
      qlen++;
      if (limit < 0) {
        if (nsn == 0) { h->nsw[f] = aw; h->nsi[f] = ai; h->nswn[f] = an; }
      } else {
        h->f_ring[h->ringoff[f] + (h->rhead[f] + nsn) % limit] = pack_id(aw, ai);
      }
      nsn++;
    }
    if (cnt == 0) break;
    a = h->arrival_n(w, i, wn);
    if (!(a <= now)) break;
  }
  h->farr[f] = a;
  h->fcnt[f] = cnt; h->fw[f] = w; h->fi[f] = i; h->fwn[f] = wn;
  h->qlen[f] = qlen; h->nsn[f] = nsn;
  h->wdrop[f] += drop;
}

// _serve (sim_engine.py:525-552) for hot pod i of function f, sequentially
// (the XL working set serves per function; the per-warp classes use the
// dry-run / scan / replay form below)
template <class H>
__device__ __forceinline__ void hot_serve(H* h, int i, int f, double t_start, double t_end) {
  const double busy = h->busy[i];
  double t = busy > t_start ? busy : t_start;
  if (!(t < t_end - TIME_EPS)) { h->busy[i] = t; return; }
  int fl = h->flags[i];
  double rem = h->crem[i], arr = h->carr[i];
  int comp = 0, viol = 0;
  #pragma unroll 1
  while (t < t_end - TIME_EPS) {
    if (!(fl & PF_CUR)) {
      long long id;
      const int retn = h->retn[f];
      const int nsn = h->nsn[f];
      if (retn > 0) {               // restarted requests precede never-started ones
        long long* r = &h->f_ret[(size_t)f * h->RET];
        id = r[0];
        #pragma unroll 1
        for (int k = 1; k < retn; k++) r[k - 1] = r[k];
        h->retn[f] = retn - 1;
      } else if (nsn > 0) {
        const int limit = h->maxq[f];
        if (limit < 0) {
          int nw = h->nsw[f], ni = h->nsi[f], nn = h->nswn[f];
          id = pack_id(nw, ni);
          arr = h->arrival_n(nw, ni, nn);
          if (nsn > 1) {
            h->advance(f, nw, ni, nn);
            h->nsw[f] = nw; h->nsi[f] = ni; h->nswn[f] = nn;
          }
        } else {
          const int hd = h->rhead[f];
          id = h->f_ring[h->ringoff[f] + hd];
          h->rhead[f] = (hd + 1) % limit;
          arr = h->arrival(f, id_w(id), id_i(id));
        }
        h->nsn[f] = nsn - 1;
      } else {
        break;
      }
      if (retn > 0) arr = h->arrival(f, id_w(id), id_i(id));
      h->pinned[f]++;
      fl |= PF_CUR;
      rem = h->invr[i];
      h->cur[i] = id;
    }
    const double left = t_end - t;
    const double span = rem < left ? rem : left;
    rem -= span;
    t += span;
    if (rem <= TIME_EPS) {
      h->qlen[f]--;
      h->pinned[f]--;
      fl &= ~PF_CUR;
      comp++;
      if ((t - arr) * 1000.0 > h->slo[f]) viol++;
    }
  }
  h->busy[i] = t;
  h->crem[i] = rem;
  h->carr[i] = arr;
  h->flags[i] = (unsigned char)fl;
  h->wcomp[f] += comp;
  h->wviol[f] += viol;
}

// id of the `pos`-th unpinned request of function f at the start of the serve
// phase: restarted (returned) requests first, then never-started ones in
// queue order (sim_engine.py:531 takes the first request with server None).
template <class H, bool BND>
__device__ __forceinline__ double unpinned_at(const H* h, int f, int pos, long long* id_out) {
  const int retn = h->retn[f];
  if (pos < retn) {
    const long long id = h->f_ret[(size_t)f * h->RET + pos];
    *id_out = id;
    return h->arrival(f, id_w(id), id_i(id));
  }
  const int q = pos - retn;
  const int limit = BND ? h->maxq[f] : -1;
  if (limit >= 0) {
    const long long id = h->f_ring[h->ringoff[f] + (h->rhead[f] + q) % limit];
    *id_out = id;
    return h->arrival(f, id_w(id), id_i(id));
  }
  int w = h->nsw[f], i = h->nsi[f] + q, n = h->nswn[f];
  while (i >= n) {
    i -= n;
    do { w++; n = h->count(f, w); } while (n == 0);
  }
  *id_out = pack_id(w, i);
  return h->arrival_n(w, i, n);
}

// How many requests pod i would start in [t_start, t_end) if the queue never
// ran dry (the serve loop's timing does not depend on which request it gets).
template <class H>
__device__ __forceinline__ int serve_dry_run(const H* h, int i, double t_start, double t_end) {
  const double busy = h->busy[i];
  double t = busy > t_start ? busy : t_start;
  bool cur = (h->flags[i] & PF_CUR) != 0;
  double rem = h->crem[i];
  const double inv = h->invr[i];
  int picks = 0;
#pragma unroll 1
  while (t < t_end - TIME_EPS) {
    if (!cur) { picks++; cur = true; rem = inv; }
    const double left = t_end - t;
    const double span = rem < left ? rem : left;
    rem -= span;
    t += span;
    if (rem <= TIME_EPS) cur = false;
  }
  return picks;
}

// _serve (sim_engine.py:525-552) for pod i whose k-th new request is the
// (base+k)-th unpinned one and which may start at most `avail` requests.
template <class H, bool BND>
__device__ __forceinline__ int serve_replay(H* h, int i, int f, double t_start, double t_end,
                                            int base, int avail, int& comp, int& viol) {
  const double busy = h->busy[i];
  double t = busy > t_start ? busy : t_start;
  if (!(t < t_end - TIME_EPS)) { h->busy[i] = t; return 0; }
  int fl = h->flags[i];
  double rem = h->crem[i], arr = h->carr[i];
  const double slo = h->slo[f];
  int taken = 0;
#pragma unroll 1
  while (t < t_end - TIME_EPS) {
    if (!(fl & PF_CUR)) {
      if (taken == avail) break;                 // queue ran dry
      long long id;
      arr = unpinned_at<H, BND>(h, f, base + taken, &id);
      taken++;
      h->cur[i] = id;
      rem = h->invr[i];
      fl |= PF_CUR;
    }
    const double left = t_end - t;
    const double span = rem < left ? rem : left;
    rem -= span;
    t += span;
    if (rem <= TIME_EPS) {
      fl &= ~PF_CUR;
      comp++;
      if ((t - arr) * 1000.0 > slo) viol++;
    }
  }
  h->busy[i] = t;
  h->crem[i] = rem;
  h->carr[i] = arr;
  h->flags[i] = (unsigned char)fl;
  return taken;                                   // requests started
}

// Python sum() of sm * duration over the tokens order[lo, lo + ng) (ng >= 1).
// One term: 0 + x = x.  Two terms: Neumaier's compensation is the exact
// rounding error of x1 + x2, so sum() returns fl(x1 + x2) itself; longer
// sums take the compensated loop.  (Terms are positive: no -0.0 cases.)
template <class H>
__device__ __forceinline__ double token_occupancy(const H* h, int lo, int ng) {
  const int i0 = h->order[lo];
  const double x0 = h->sm[i0] * h->dur(i0);
  if (ng == 1) return x0;
  const int i1 = h->order[lo + 1];
  const double x1 = h->sm[i1] * h->dur(i1);
  if (ng == 2) return x0 + x1;
  PySum occ;
  occ.reset();
  occ.add(x0);
  occ.add(x1);
#pragma unroll 1
  for (int j = lo + 2; j < lo + ng; j++) {
    const int i = h->order[j];
    occ.add(h->sm[i] * h->dur(i));
  }
  return occ.value();
}

// dispatch for non-integral SM partitions: the sequential head-blocking walk
// with the float sm_running dust (token_backend.py:169-187); returns this
// lane's grants
template <class H>
__device__ __noinline__ int hot_dispatch_float(H* h, int lane) {
  const double quantum = h->quantum;
  const int G = h->G;
  int grants = 0;
#pragma unroll 1
    for (int g = lane; g < G; g += 32) {
      double sr = h->sr[g];
      double mx = 0.0;
      PySum occ;
      occ.reset();
      int ng = 0;
      const int e = h->seg[g] + h->reqsm[g];      // the requesting prefix of the order
#pragma unroll 1
      for (int j = h->seg[g]; j < e; j++) {
        const int i = h->order[j];
        const double sm = h->sm[i];
        if (sm + sr > SM_LIMIT + SM_EPS) break;
        const double rem = h->qlim[i] - h->qused[i];
        const double dur = rem < quantum ? rem : quantum;
        h->flags[i] |= PF_GRANT;
        sr += sm;
        if (ng == 0 || dur > mx) mx = dur;
        occ.add(sm * dur);
        ng++;
      }
      h->sr[g] = sr;
      h->ngr[g] = ng;
      if (ng) {
        h->cov[g] += mx;
        h->occ[g] += occ.value() / 100.0;
      }
      grants += ng;
    }
  return grants;
}

// returns this lane's token grants of the step (hot_steps_t sums the warp once a window)
template <class H, bool INTEG, bool BND>
__device__ int hot_step(H* h, int lane, int w, int s) {
  const double t0 = (double)w * h->ws + (double)s * h->qs;
  const int n = h->n;
  const int F = h->F, G = h->G;
  constexpr bool integral = INTEG;
  // _admit_arrivals touches only queues and _complete_live_tokens only the
  // ledger, so admission runs first and completion fuses with the key pass.
  lane_for<H::FC>(lane, F, [&](int f) { hot_admit<H, BND>(h, f, t0); });
  if (s > 0 && !integral) hot_complete_sm(h, lane);
  lane_for<H::GC>(lane, G, [&](int g) {
    h->cut[g] = 0x7fffffff; h->covbits[g] = 0ull;
    h->reqsm[g] = 0; h->ngr[g] = 0; h->ostate[g] = 0;
  });
  __syncwarp();
  // complete live tokens + filter_pods + requesting:
  // key = -(q_req - q_used) for requesting pods, ~0 otherwise
  bool any_req = false;
  lane_for<H::PC>(lane, n, [&](int i) {
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
    // integral: requesting SM per node (only where it can exceed 100);
    // otherwise: requesting pods per node (the float dispatch walk's bound)
    if (req && (!integral || h->maycut[h->fnode[i] >> 16]))
      atomicAdd(&h->reqsm[h->fnode[i] >> 16], integral ? (int)h->sm[i] : 1);
    any_req |= req;
  });
  // No pod requests a token: dispatch grants nothing, so coverage, occupancy,
  // sm_running and every queue stay as they are (token_backend.py:160-187,
  // sim_engine.py:514-520 iterate over no tokens).
  if (!__any_sync(FULL, any_req)) return 0;
  __syncwarp();
  // build_queue order inside each node by rank counting on (key, pod_id)
  // (pod_id order == hot index order within a node).  With integral SM
  // partitions the running SM sum is exact in any order, so dispatch's
  // head-blocking cut is decided here too: a requesting pod misfits iff
  // sm + (SM of the requesting pods ahead of it) > 100 + 1e-9, and the node's
  // cut is the smallest misfit rank (token_backend.py:169-177).
  // In the integral path the order matters for nothing else: a node whose
  // requesting SM is <= 100 grants every requesting pod, and the occupancy
  // sum is order-free (below) -- such nodes need no ranks at all.
  lane_for<H::PC>(lane, n, [&](int i) {
    const double k = h->key[i];
    // non-requesting pods are never dispatched: no position needed (the
    // dispatch walks stop at the requesting / granted prefix of the order)
    if (k == NOT_REQ) return;
    const int g = h->fnode[i] >> 16;
    const int lo = h->seg[g], hi = h->seg[g + 1];
    int r = 0;
    // the SM sum ahead is only needed when the node's requesting SM can
    // exceed 100 (otherwise no requesting pod misfits)
    const bool need_ahead = integral && h->maycut[g] && h->reqsm[g] > (int)SM_LIMIT;
    if (integral && !need_ahead) { h->rank[i] = 0; return; }   // granted, cut stays open
    if (need_ahead) {
      double ahead = 0.0;
#pragma unroll 1
      for (int j = lo; j < hi; j++) {
        const double kj = h->key[j];
        const bool less = (kj < k) || (kj == k && j < i);
        r += less;
        if (less) ahead += h->sm[j];
      }
      if (h->sm[i] + ahead > SM_LIMIT + SM_EPS) atomicMin(&h->cut[g], r);
    } else {
      // (key, pod index) order: pods before i count when key <= k, the rest
      // when key < k; one convergent loop over the node for all its lanes
      int j = lo;
#pragma unroll 1
      for (; j + 1 < hi; j += 2) {
        const double a = h->key[j], b = h->key[j + 1];
        r += (int)(j < i ? a <= k : a < k) + (int)(j + 1 < i ? b <= k : b < k);
      }
      if (j < hi) {
        const double a = h->key[j];
        r += (int)(j < i ? a <= k : a < k);
      }
    }
    // (each order position is written only by the lane whose pod lands there;
    // the integral path keeps no order)
    if (!integral) h->order[lo + r] = (unsigned char)i;
    h->rank[i] = (unsigned char)r;
  });
  __syncwarp();
  const double quantum = h->quantum;
  int grants = 0;
  if (integral) {
    // grant: the node's tokens go to order[seg, seg + ngr) in any order (the
    // occupancy sum below is order-free); a ballot per 32 pods records the
    // granted set for the occupancy cache
#pragma unroll 1
    for (int j0 = 0; j0 < trips32<H::PC>(n); j0 += 32) {
      const int i = j0 + lane;
      bool gr = false;
      if (i < n) {
        const int g = h->fnode[i] >> 16;
        if (h->key[i] != NOT_REQ && h->rank[i] < h->cut[g]) {
          const double rem = h->qlim[i] - h->qused[i];
          h->flags[i] |= PF_GRANT;
          h->order[h->seg[g] + atomicAdd(&h->ngr[g], 1)] = (unsigned char)i;
          if (rem < quantum) {             // partial token: it may set the max duration
            atomicOr(&h->ostate[g], 2);
            atomicMax(&h->covbits[g], (unsigned long long)__double_as_longlong(rem));
          } else {
            atomicOr(&h->ostate[g], 4);    // a full quantum is the max
          }
          gr = true;
          grants++;
        }
      }
      const unsigned b = __ballot_sync(FULL, gr);
      if (lane == 0) { h->gwp[j0 >> 5] = h->gw[j0 >> 5]; h->gw[j0 >> 5] = b; }
    }
    __syncwarp();
    // occupancy: Python sum() of sm*duration over the node's tokens
    // (sim_engine.py:516-517).  The reference adds them in dispatch order;
    // here they are added in grant-slot order, with the same result: every
    // term is sm * dur with an integer sm in [1, 100] and dur in (1e-9, 1],
    // so the terms and partial sums lie within 2^7 .. 2^-30 and there are at
    // most 100 of them.  Each Neumaier error term (f - t) + x is then exact
    // and a multiple of 2^-82, their running sum c stays below 2^-40 and is
    // exact too, so f + c is the exact real sum S of the terms and sum()
    // returns fl(S) -- a function of the multiset of terms alone, not of
    // their order.
    lane_for<H::GC>(lane, G, [&](int g) {
      const int ng = h->ngr[g];
      if (ng == 0) { h->occn[g] = -1; return; }
      const int st = h->ostate[g];
      const int lo = h->seg[g], hi = h->seg[g + 1];
      bool same = !(st & 2) && ng == h->occn[g];
#pragma unroll 1
      for (int w = lo >> 5; same && w <= ((hi - 1) >> 5); w++) {
        const int a = lo - 32 * w, b = hi - 32 * w;
        const unsigned m = (b >= 32 ? FULL : ((1u << b) - 1u)) & (a > 0 ? ~((1u << a) - 1u) : FULL);
        same = ((h->gw[w] ^ h->gwp[w]) & m) == 0u;
      }
      double v;
      if (same) {
        v = h->occv[g];   // same granted pods, all full-quantum tokens: same terms
      } else {
        v = token_occupancy(h, lo, ng) / 100.0;
        h->occv[g] = v;
        h->occn[g] = (st & 2) ? -1 : ng;
      }
      h->cov[g] += (st & 4) ? quantum : __longlong_as_double((long long)h->covbits[g]);
      h->occ[g] += v;
    });
  } else {
    grants = hot_dispatch_float(h, lane);
  }
  // serve (sim_engine.py:514-520), pod-parallel.  Granted pods in (function,
  // node, pod_id) order; a dry run counts each pod's request starts, a
  // segmented scan per function turns them into FIFO positions, and a replay
  // serves exactly the requests the sequential drain would have handed out.
  lane_for<H::FC>(lane, F, [&](int f) {
    h->favail[f] = h->retn[f] + h->nsn[f];
    h->fcarry[f] = 0; h->fcomp[f] = 0; h->fviol[f] = 0;
  });
  __syncwarp();
  int ngl = 0;
#pragma unroll 1
  for (int j0 = 0; j0 < trips32<H::PC>(n); j0 += 32) {
    const int j = j0 + lane;
    const int i = j < n ? h->flist[j] : 0;
    const bool gr = j < n && (h->flags[i] & PF_GRANT);
    const unsigned bal = __ballot_sync(FULL, gr);
    if (gr) h->rank[ngl + __popc(bal & ((1u << lane) - 1u))] = (unsigned char)i;
    ngl += __popc(bal);
  }
  __syncwarp();
  const double ws = h->ws;
#pragma unroll 1
  for (int k0 = 0; k0 < trips32<H::PC>(ngl); k0 += 32) {
    const int k = k0 + lane;
    const bool act = k < ngl;
    const int i = act ? h->rank[k] : 0;
    const int f = act ? (h->fnode[i] & 0xffff) : -1 - lane;
    const double t_end = t0 + h->dur(i) * ws;
    // the only granted pod of its function in a single-trip step needs no
    // dry run: its FIFO base is 0, and the replay itself stops when the
    // token's time runs out (after exactly the dry run's request starts) or
    // the queue runs dry, so the requests it took are the function's "want"
    // (measured: a gain for the classes with many pods per function, a loss
    // for class XS, whose dry runs are short)
    const int fnext = __shfl_down_sync(FULL, f, 1);
    bool single = false;
    if constexpr (H::PC > 32) {
      const int fprev = __shfl_up_sync(FULL, f, 1);
      single = act && ngl <= 32 && (lane == 0 || fprev != f) &&
               (lane == 31 || k + 1 >= ngl || fnext != f);
    }
    const int picks = (act && !single) ? serve_dry_run(h, i, t0, t_end) : 0;
    int v = picks;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, v, o);
      const int fo = __shfl_up_sync(FULL, f, o);
      if (lane >= o && fo == f) v += y;
    }
    const bool seg_end = act && (lane == 31 || k + 1 >= ngl || fnext != f);
    if (act) {
      const int base = h->fcarry[f] + v - picks;
      int avail = h->favail[f] - base;
      avail = avail < 0 ? 0 : ((!single && avail > picks) ? picks : avail);
      int comp = 0, viol = 0;
      const int took = serve_replay<H, BND>(h, i, f, t0, t_end, base, avail, comp, viol);
      if (single) v = took;
      if (comp) atomicAdd(&h->fcomp[f], comp);
      if (viol) atomicAdd(&h->fviol[f], viol);
    }
    __syncwarp();
    if (seg_end) h->fcarry[f] += v;
    __syncwarp();
  }
  // apply each function's queue bookkeeping once
  lane_for<H::FC>(lane, F, [&](int f) {
    const int want = h->fcarry[f];
    if (want == 0 && h->fcomp[f] == 0) return;
    const int avail = h->favail[f];
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
    const int comp = h->fcomp[f];
    h->pinned[f] += taken - comp;
    h->qlen[f] -= comp;
    h->wcomp[f] += comp;
    h->wviol[f] += h->fviol[f];
  });
  __syncwarp();
  return grants;
}

// One instantiation per (integral SM partitions, any bounded queue): the
// common case (integral, unbounded) carries neither the float dispatch nor
// the bounded-queue ring code in its instruction stream.
template <class H, bool INTEG, bool BND>
__device__ __noinline__ long long hot_steps_t(H* h, int lane, int w) {
  const int T = h->T;
  int grants = 0;              // this lane's grants of the window (< 2^31)
  #pragma unroll 1
  for (int s = 0; s < T; s++) grants += hot_step<H, INTEG, BND>(h, lane, w, s);
  hot_complete(h, lane);
  __syncwarp();
  return warp_sum_i(grants);
}

template <class H>
__device__ long long hot_steps(H* h, int lane, int w) {
  if (h->integral) {
    return h->bounded ? hot_steps_t<H, true, true>(h, lane, w)
                      : hot_steps_t<H, true, false>(h, lane, w);
  }
  return h->bounded ? hot_steps_t<H, false, true>(h, lane, w)
                    : hot_steps_t<H, false, false>(h, lane, w);
}

// Window start when registration did not change (no epoch, nobody warmed
// up): reset_window + _generate_arrivals directly on the shared-memory set.
template <class H>
__device__ void hot_begin_light(H* h, int lane, int w) {
  lane_for<H::PC>(lane, h->n, [&](int i) { h->qused[i] = 0.0; });
  lane_for<H::FC>(lane, h->F, [&](int f) {
    const int n = h->count(f, w);
    h->warr[f] = n;
    if (n > 0) {
      if (h->fcnt[f] == 0) {
        h->fw[f] = w; h->fi[f] = 0; h->fwn[f] = n;
        h->farr[f] = h->arrival_n(w, 0, n);
      }
      h->fcnt[f] += n;
    }
  });
  lane_for<H::GC>(lane, h->G, [&](int g) { h->cov[g] = 0.0; h->occ[g] = 0.0; });
  __syncwarp();
}

}  // namespace gs
