// gs_xl.cuh -- the XL class: runs too large for a per-warp shared-memory
// working set (e.g. BASELINE configs[3], 64 nodes x 200 functions, ~10^3
// registered pods) get a whole CTA (XL_THREADS threads) each.
//
// Warp 0 owns the run's control code exactly as in the per-warp classes
// (initial placement, epochs, window begin / close -- all warp-level code on
// the HBM arena).  The quantum steps, which are >90% of the work and whose
// phases are independent per pod / function / node, run on every thread of
// the CTA with block barriers between phases (sim_engine.py:493-520):
//
//   complete    threads = pods      q_used += duration (token_backend.py:190-210)
//   admit       threads = functions (sim_engine.py:472-480)
//   key         threads = pods      filter_pods + requesting -> -(q_req - q_used)
//   rank        threads = pods      rank in the node's build_queue by counting
//                                   (key, pod_id) over the node's pods
//   dispatch    integral SM: threads = pods (grant iff rank < the node's cut),
//               then threads = nodes for coverage / occupancy in rank order;
//               otherwise threads = nodes, the sequential head-blocking walk
//   serve       threads = functions, FIFO drain over the function's granted
//               pods in (node, pod_id) order (sim_engine.py:514-552)
#pragma once
#include "gs_kernel.cuh"

namespace gs {

constexpr int XL_THREADS = 512;

struct XlShared {
  int run;
  int stop;
  int grants;
  int warp_tot[32];
};

__device__ __forceinline__ double xl_dur(const Ctx& c, int slot) {
  const double rem = c.t->p_qlim[slot] - c.t->p_qused[slot];
  return rem < c.quantum ? rem : c.quantum;
}

// _complete_live_tokens (sim_engine.py:482-486), CTA-wide.
__device__ void xl_complete(Ctx& c) {
  const int n = c.sh->n_reg;
  const int* rl = c.t->s_rl;
  if (!c.integral()) {
    // sm_running -= sm in the last dispatch order, with the float-dust clamp
    const int* ord = c.t->s_ki;
    const int* nq = c.t->n_ngr;
#pragma unroll 1
    for (int g = threadIdx.x; g < c.G; g += blockDim.x) {
      double sr = c.t->n_sr[g];
      const int lo = c.t->n_seg[g];
#pragma unroll 1
      for (int j = lo; j < lo + nq[g]; j++) {
        const int slot = rl[ord[j]];
        sr -= c.t->p_sm[slot];
        if (sr < 0 && sr > -SM_EPS) sr = 0.0;
      }
      c.t->n_sr[g] = sr;
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int slot = rl[i];
    const int fl = c.t->p_flags[slot];
    if (fl & PF_GRANT) {
      c.t->p_qused[slot] += c.t->p_dur[slot];
      c.t->p_flags[slot] = fl & ~PF_GRANT;
    }
  }
  __syncthreads();
}

// window start with an unchanged registered set (no epoch, no warm-up):
// reset_window + _generate_arrivals, CTA-wide (sim_engine.py:446-449)
__device__ void xl_begin_light(Ctx& c, int w) {
  const int n = c.sh->n_reg;
  const int* rl = c.t->s_rl;
#pragma unroll 1
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int slot = rl[i];
    c.t->p_qused[slot] = 0.0;
    c.t->p_flags[slot] &= ~PF_GRANT;
  }
#pragma unroll 1
  for (int f = threadIdx.x; f < c.F; f += blockDim.x) {
    const int k = c.count(f, w);
    c.t->f_warr[f] = k;
    if (k > 0) {
      if (c.t->f_fn[f] == 0) { c.t->f_fw[f] = w; c.t->f_fi[f] = 0; }
      c.t->f_fn[f] += k;
    }
  }
  if (threadIdx.x == 0) c.sh->pod_steps += (long long)n * c.T;
}

// one quantum step (sim_engine.py:493-520) on every thread of the CTA
__device__ void xl_step(Ctx& c, int w, int s, XlShared* xs) {
  const double t0 = (double)w * c.ws + (double)s * c.qs;
  const int n = c.sh->n_reg;
  const int tid = threadIdx.x, NT = blockDim.x;
  const bool integral = c.integral();
  const int* rl = c.t->s_rl;
  const int* seg = c.t->n_seg;
  double* key = reinterpret_cast<double*>(c.t->s_kd);   // by registered index
  int* ord = c.t->s_ki;                                   // dispatch order per node
  int* rank = c.t->s_list;                                // rank by registered index
  int* reqsm = c.t->n_reqsm;
  int* cut = c.t->n_cut;
  int* ngr = c.t->n_ngr;
  unsigned long long* covb = c.t->n_covb;
  if (s > 0) xl_complete(c);       // step 0: window_begin already reset the ledger
  if (tid == 0) xs->grants = 0;
#pragma unroll 1
  for (int f = tid; f < c.F; f += NT) admit_arrivals(c, f, t0);
#pragma unroll 1
  for (int g = tid; g < c.G; g += NT) {
    reqsm[g] = 0; cut[g] = 0x7fffffff; ngr[g] = 0; covb[g] = 0ull;
  }
  __syncthreads();
  // complete was done above; filter_pods + requesting + key
#pragma unroll 1
  for (int i = tid; i < n; i += NT) {
    const int slot = rl[i];
    const int fl = c.t->p_flags[slot];
    const double qused = c.t->p_qused[slot];
    const bool cand = !(c.t->p_qlim[slot] - qused <= QUOTA_EPS);
    const int f = c.t->p_fn[slot];
    const bool req = cand && ((fl & PF_CUR) || (c.t->f_qlen[f] - c.t->f_pinned[f] > 0));
    key[i] = req ? -(c.t->p_qreq[slot] - qused) : NOT_REQ;
    if (req && integral) atomicAdd(&reqsm[c.t->p_node[slot]], (int)c.t->p_sm[slot]);
  }
  __syncthreads();
  // build_queue order per node: rank by counting (key, pod_id); pod_id order
  // == registered-index order inside a node (window_begin sorts (node, pod_id))
#pragma unroll 1
  for (int i = tid; i < n; i += NT) {
    const int g = c.t->p_node[rl[i]];
    const double k = key[i];
    const int lo = seg[g], hi = seg[g + 1];
    int r = 0;
    if (integral && k != NOT_REQ && reqsm[g] > (int)SM_LIMIT) {
      double ahead = 0.0;
#pragma unroll 1
      for (int j = lo; j < hi; j++) {
        const double kj = key[j];
        const bool less = (kj < k) || (kj == k && j < i);
        r += less;
        if (less) ahead += c.t->p_sm[rl[j]];
      }
      if (c.t->p_sm[rl[i]] + ahead > SM_LIMIT + SM_EPS) atomicMin(&cut[g], r);
    } else {
      int j = lo;
#pragma unroll 1
      for (; j + 1 < hi; j += 2) {
        const double a = key[j], b = key[j + 1];
        r += (int)(j < i ? a <= k : a < k) + (int)(j + 1 < i ? b <= k : b < k);
      }
      if (j < hi) {
        const double a = key[j];
        r += (int)(j < i ? a <= k : a < k);
      }
    }
    ord[lo + r] = i;
    rank[i] = r;
  }
  __syncthreads();
  const double quantum = c.quantum;
  int grants = 0;
  if (integral) {
#pragma unroll 1
    for (int i = tid; i < n; i += NT) {
      const int slot = rl[i];
      const int g = c.t->p_node[slot];
      if (key[i] != NOT_REQ && rank[i] < cut[g]) {
        const double rem = c.t->p_qlim[slot] - c.t->p_qused[slot];
        const double dur = rem < quantum ? rem : quantum;
        c.t->p_dur[slot] = dur;
        c.t->p_flags[slot] |= PF_GRANT;
        atomicMax(&covb[g], (unsigned long long)__double_as_longlong(dur));
        atomicAdd(&ngr[g], 1);
        grants++;
      }
    }
    __syncthreads();
    // coverage / occupancy: Python sum() of sm*duration in dispatch order
#pragma unroll 1
    for (int g = tid; g < c.G; g += NT) {
      const int ng = ngr[g];
      if (ng == 0) continue;
      PySum occ;
      occ.reset();
      const int lo = seg[g];
#pragma unroll 1
      for (int j = lo; j < lo + ng; j++) {
        const int slot = rl[ord[j]];
        occ.add(c.t->p_sm[slot] * c.t->p_dur[slot]);
      }
      c.t->n_cov[g] += __longlong_as_double((long long)covb[g]);
      c.t->n_occ[g] += occ.value() / 100.0;
    }
  } else {
    // head-blocking walk with the float sm_running (token_backend.py:169-187)
#pragma unroll 1
    for (int g = tid; g < c.G; g += NT) {
      double sr = c.t->n_sr[g];
      double mx = 0.0;
      PySum occ;
      occ.reset();
      int ng = 0;
      const int lo = seg[g], hi = seg[g + 1];
#pragma unroll 1
      for (int j = lo; j < hi; j++) {
        const int i = ord[j];
        if (key[i] == NOT_REQ) break;          // rest of the node is not requesting
        const int slot = rl[i];
        const double sm = c.t->p_sm[slot];
        if (sm + sr > SM_LIMIT + SM_EPS) break;
        const double rem = c.t->p_qlim[slot] - c.t->p_qused[slot];
        const double dur = rem < quantum ? rem : quantum;
        c.t->p_dur[slot] = dur;
        c.t->p_flags[slot] |= PF_GRANT;
        sr += sm;
        if (ng == 0 || dur > mx) mx = dur;
        occ.add(sm * dur);
        ng++;
      }
      c.t->n_sr[g] = sr;
      ngr[g] = ng;
      if (ng) {
        c.t->n_cov[g] += mx;
        c.t->n_occ[g] += occ.value() / 100.0;
      }
      grants += ng;
    }
  }
  if (grants) atomicAdd(&xs->grants, grants);
  __syncthreads();
  // serve: per function, its granted pods in (node, pod_id) order
#pragma unroll 1
  for (int f = tid; f < c.F; f += NT) {
    const int e = c.t->f_loff[f + 1];
#pragma unroll 1
    for (int j = c.t->f_loff[f]; j < e; j++) {
      const int slot = c.t->s_fl[j];
      if (c.t->p_flags[slot] & PF_GRANT) serve(c, slot, t0, t0 + c.t->p_dur[slot] * c.ws);
    }
  }
  __syncthreads();
  if (tid == 0) c.sh->grants += xs->grants;
}

}  // namespace gs
