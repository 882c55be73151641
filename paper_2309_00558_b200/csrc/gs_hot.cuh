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

template <int PC_, int FC_, int GC_>
struct Hot {
  static constexpr int PC = PC_, FC = FC_, GC = GC_;
  // registered pods of this window, in (node, pod_id) order
  double qused[PC], qreq[PC], qlim[PC], sm[PC], busy[PC], crem[PC], carr[PC], invr[PC],
      dur[PC];
  unsigned long long key[PC];
  long long cur[PC];
  int slot[PC], fnode[PC], flags[PC];
  short order[PC], flist[PC];
  // functions
  double farr[FC], slo[FC];
  int qlen[FC], pinned[FC], fw[FC], fi[FC], fcnt[FC], nsn[FC], nsw[FC], nsi[FC];
  int rhead[FC], retn[FC], wcomp[FC], wviol[FC], wdrop[FC], maxq[FC], ringoff[FC];
  int loff[FC + 1];
  // nodes
  double sr[GC], cov[GC], occ[GC];
  int seg[GC + 1];
  int n;
  long long grants;
};

// size classes: (pods, functions, nodes)
typedef Hot<64, 16, 8> HotS;
typedef Hot<128, 32, 16> HotM;
typedef Hot<256, 64, 32> HotL;

template <class H>
__host__ __device__ constexpr bool fits(int n_reg, int F, int G) {
  return n_reg <= H::PC && F <= H::FC && G <= H::GC;
}

// ---------------------------------------------------------------- load/store
template <class H>
__device__ bool hot_load(Ctx& c, H* h) {
  const int n = c.sh->n_reg;
  if (n > H::PC || c.F > H::FC || c.G > H::GC) {
    if (c.lane == 0) set_error(c, GS_ERR_CAPACITY, GS_CAP_HOT, n, 0);
    __syncwarp();
    return false;
  }
  for (int i = c.lane; i < n; i += 32) {
    int s = c.s_rl[i];
    h->slot[i] = s;
    h->qused[i] = c.p_qused[s];
    h->qreq[i] = c.p_qreq[s];
    h->qlim[i] = c.p_qlim[s];
    h->sm[i] = c.p_sm[s];
    h->busy[i] = c.p_busy[s];
    h->crem[i] = c.p_crem[s];
    h->carr[i] = c.p_carr[s];
    h->invr[i] = c.p_invr[s];
    h->dur[i] = 0.0;
    h->cur[i] = pack_id(c.p_cw[s], c.p_ci[s]);
    h->fnode[i] = c.p_fn[s] | (c.p_node[s] << 16);
    h->flags[i] = c.p_flags[s] & PF_CUR;
    h->order[i] = (short)i;
  }
  for (int f = c.lane; f < c.F; f += 32) {
    h->qlen[f] = c.f_qlen[f]; h->pinned[f] = c.f_pinned[f];
    h->fw[f] = c.f_fw[f]; h->fi[f] = c.f_fi[f]; h->fcnt[f] = c.f_fn[f];
    h->nsn[f] = c.f_nsn[f]; h->nsw[f] = c.f_nsw[f]; h->nsi[f] = c.f_nsi[f];
    h->rhead[f] = c.f_rhead[f]; h->retn[f] = c.f_retn[f];
    h->wcomp[f] = 0; h->wviol[f] = 0; h->wdrop[f] = 0;
    h->maxq[f] = c.fs[f].max_queue;
    h->ringoff[f] = c.f_ringoff[f];
    h->slo[f] = c.fs[f].slo_ms;
    h->farr[f] = h->fcnt[f] > 0 ? arrival_time(c, f, h->fw[f], h->fi[f]) : 0.0;
  }
  for (int f = c.lane; f <= c.F; f += 32) h->loff[f] = c.f_loff[f];
  for (int g = c.lane; g < c.G; g += 32) {
    h->sr[g] = c.n_sr[g]; h->cov[g] = 0.0; h->occ[g] = 0.0;
  }
  for (int g = c.lane; g <= c.G; g += 32) h->seg[g] = c.n_seg[g];
  if (c.lane == 0) { h->n = n; h->grants = 0; }
  __syncwarp();
  // s_fl holds arena slots in (node, pod_id) order per function; the hot
  // index of an arena slot is its position in s_rl (slot -> index via s_list).
  for (int i = c.lane; i < n; i += 32) c.s_list[c.s_rl[i]] = i;
  __syncwarp();
  for (int j = c.lane; j < n; j += 32) h->flist[j] = (short)c.s_list[c.s_fl[j]];
  __syncwarp();
  return true;
}

template <class H>
__device__ void hot_store(Ctx& c, H* h) {
  const int n = h->n;
  for (int i = c.lane; i < n; i += 32) {
    int s = h->slot[i];
    c.p_qused[s] = h->qused[i];
    c.p_busy[s] = h->busy[i];
    c.p_crem[s] = h->crem[i];
    c.p_carr[s] = h->carr[i];
    c.p_cw[s] = id_w(h->cur[i]);
    c.p_ci[s] = id_i(h->cur[i]);
    c.p_flags[s] = (c.p_flags[s] & ~(PF_CUR | PF_GRANT)) | (h->flags[i] & PF_CUR);
  }
  for (int f = c.lane; f < c.F; f += 32) {
    c.f_qlen[f] = h->qlen[f]; c.f_pinned[f] = h->pinned[f];
    c.f_fw[f] = h->fw[f]; c.f_fi[f] = h->fi[f]; c.f_fn[f] = h->fcnt[f];
    c.f_nsn[f] = h->nsn[f]; c.f_nsw[f] = h->nsw[f]; c.f_nsi[f] = h->nsi[f];
    c.f_rhead[f] = h->rhead[f]; c.f_retn[f] = h->retn[f];
    c.f_wcomp[f] += h->wcomp[f]; c.f_wviol[f] += h->wviol[f]; c.f_wdrop[f] += h->wdrop[f];
  }
  for (int g = c.lane; g < c.G; g += 32) {
    c.n_sr[g] = h->sr[g]; c.n_cov[g] = h->cov[g]; c.n_occ[g] = h->occ[g];
  }
  if (c.lane == 0) c.sh->grants += h->grants;
  __syncwarp();
}

// ------------------------------------------------------------------- phases
template <class H>
__device__ __forceinline__ void hot_complete(const Ctx& c, H* h) {
  const int n = h->n;
  if (!c.integral()) {
    // sm_running -= sm in token (dispatch) order, with the float-dust clamp
    for (int g = c.lane; g < c.G; g += 32) {
      double sr = h->sr[g];
      for (int j = h->seg[g]; j < h->seg[g + 1]; j++) {
        int i = h->order[j];
        if (!(h->flags[i] & PF_GRANT)) break;
        sr -= h->sm[i];
        if (sr < 0 && sr > -SM_EPS) sr = 0.0;
      }
      h->sr[g] = sr;
    }
    __syncwarp();
  }
  for (int i = c.lane; i < n; i += 32) {
    int fl = h->flags[i];
    if (fl & PF_GRANT) {
      h->qused[i] += h->dur[i];
      h->flags[i] = fl & ~PF_GRANT;
    }
  }
}

template <class H>
__device__ __forceinline__ void hot_admit(const Ctx& c, H* h, int f, double t0) {
  int cnt = h->fcnt[f];
  if (cnt == 0) return;
  double a = h->farr[f];
  const double now = t0 + TIME_EPS;
  if (!(a <= now)) return;
  int w = h->fw[f], i = h->fi[f];
  const int limit = h->maxq[f];
  int qlen = h->qlen[f], nsn = h->nsn[f], drop = 0;
  while (true) {
    const int aw = w, ai = i;
    cnt--;
    if (cnt > 0) advance_id(c, f, w, i);
    if (limit >= 0 && qlen >= limit) {
      drop++;
    } else {
      qlen++;
      if (limit < 0) {
        if (nsn == 0) { h->nsw[f] = aw; h->nsi[f] = ai; }
      } else {
        c.f_ring[h->ringoff[f] + (h->rhead[f] + nsn) % limit] = pack_id(aw, ai);
      }
      nsn++;
    }
    if (cnt == 0) break;
    a = arrival_time(c, f, w, i);
    if (!(a <= now)) break;
  }
  h->farr[f] = a;
  h->fcnt[f] = cnt; h->fw[f] = w; h->fi[f] = i;
  h->qlen[f] = qlen; h->nsn[f] = nsn;
  h->wdrop[f] += drop;
}

// _serve (sim_engine.py:525-552) for hot pod i
template <class H>
__device__ __forceinline__ void hot_serve(const Ctx& c, H* h, int i, int f, double t_start,
                                          double t_end) {
  double busy = h->busy[i];
  double t = busy > t_start ? busy : t_start;
  if (!(t < t_end - TIME_EPS)) { h->busy[i] = t; return; }
  int fl = h->flags[i];
  double rem = h->crem[i], arr = h->carr[i];
  const double slo = h->slo[f];
  int comp = 0, viol = 0;
  while (t < t_end - TIME_EPS) {
    if (!(fl & PF_CUR)) {
      long long id;
      const int retn = h->retn[f];
      const int nsn = h->nsn[f];
      if (retn > 0) {               // restarted requests precede never-started ones
        long long* r = &c.f_ret[(size_t)f * c.RET];
        id = r[0];
        for (int k = 1; k < retn; k++) r[k - 1] = r[k];
        h->retn[f] = retn - 1;
      } else if (nsn > 0) {
        const int limit = h->maxq[f];
        if (limit < 0) {
          int nw = h->nsw[f], ni = h->nsi[f];
          id = pack_id(nw, ni);
          if (nsn > 1) { advance_id(c, f, nw, ni); h->nsw[f] = nw; h->nsi[f] = ni; }
        } else {
          const int hd = h->rhead[f];
          id = c.f_ring[h->ringoff[f] + hd];
          h->rhead[f] = (hd + 1) % limit;
        }
        h->nsn[f] = nsn - 1;
      } else {
        break;
      }
      h->pinned[f]++;
      fl |= PF_CUR;
      rem = h->invr[i];
      arr = arrival_time(c, f, id_w(id), id_i(id));
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
      if ((t - arr) * 1000.0 > slo) viol++;
    }
  }
  h->busy[i] = t;
  h->crem[i] = rem;
  h->carr[i] = arr;
  h->flags[i] = fl;
  h->wcomp[f] += comp;
  h->wviol[f] += viol;
}

template <class H>
__device__ void hot_step(const Ctx& c, H* h, int w, int s) {
  const double t0 = (double)w * c.ws + (double)s * c.qs;
  const int n = h->n;
  if (s > 0) hot_complete(c, h);
  for (int f = c.lane; f < c.F; f += 32) hot_admit(c, h, f, t0);
  __syncwarp();
  // filter_pods + requesting: key = -(q_req - q_used) for requesting pods, ~0 otherwise
  for (int i = c.lane; i < n; i += 32) {
    const int f = h->fnode[i] & 0xffff;
    const double qused = h->qused[i];
    const bool cand = !(h->qlim[i] - qused <= QUOTA_EPS);
    const bool req = cand && ((h->flags[i] & PF_CUR) || (h->qlen[f] - h->pinned[f] > 0));
    h->key[i] = req ? ord_key(-(h->qreq[i] - qused)) : ~0ull;
  }
  __syncwarp();
  // build_queue order inside each node by rank counting: (key, pod_id), and
  // pod_id order == hot index order within a node
  for (int i = c.lane; i < n; i += 32) {
    const int g = h->fnode[i] >> 16;
    const unsigned long long k = h->key[i];
    const int lo = h->seg[g], hi = h->seg[g + 1];
    int r = 0;
    for (int j = lo; j < hi; j++) {
      const unsigned long long kj = h->key[j];
      r += (kj < k) || (kj == k && j < i);
    }
    h->order[lo + r] = (short)i;
  }
  __syncwarp();
  // dispatch (head-blocking) + coverage/occupancy, one lane per node
  int grants = 0;
  for (int g = c.lane; g < c.G; g += 32) {
    double sr = c.integral() ? 0.0 : h->sr[g];
    double mx = 0.0;
    PySum occ;
    occ.reset();
    int ng = 0;
    for (int j = h->seg[g]; j < h->seg[g + 1]; j++) {
      const int i = h->order[j];
      if (h->key[i] == ~0ull) break;          // rest of the node is not requesting
      const double sm = h->sm[i];
      if (sm + sr > SM_LIMIT + SM_EPS) break;
      const double rem = h->qlim[i] - h->qused[i];
      const double dur = rem < c.quantum ? rem : c.quantum;
      h->dur[i] = dur;
      h->flags[i] |= PF_GRANT;
      sr += sm;
      if (ng == 0 || dur > mx) mx = dur;
      occ.add(sm * dur);
      ng++;
    }
    if (!c.integral()) h->sr[g] = sr;
    if (ng) {
      h->cov[g] += mx;
      h->occ[g] += occ.value() / 100.0;
    }
    grants += ng;
  }
  grants = warp_sum_i(grants);
  if (c.lane == 0) h->grants += grants;
  __syncwarp();
  // serve, per function in (node, pod_id) order
  for (int f = c.lane; f < c.F; f += 32) {
    const int e = h->loff[f + 1];
    for (int j = h->loff[f]; j < e; j++) {
      const int i = h->flist[j];
      if (h->flags[i] & PF_GRANT) hot_serve(c, h, i, f, t0, t0 + h->dur[i] * c.ws);
    }
  }
  __syncwarp();
}

template <class H>
__device__ bool hot_window(Ctx& c, H* h, int w) {
  if (!hot_load(c, h)) return false;
  for (int s = 0; s < c.T; s++) hot_step(c, h, w, s);
  hot_complete(c, h);
  __syncwarp();
  hot_store(c, h);
  return true;
}

}  // namespace gs
