// gs_state.cuh -- per-run device state layout of the B200 FaST-GShare kernel.
//
// One warp simulates one (scenario, policy) run.  Its whole mutable state is
// one contiguous arena (structure-of-arrays, 16-byte aligned slices) whose
// layout is a pure function of the run's capacities, computed identically on
// host (to size the workspace) and device (to carve it).
// "Data layout in HBM" for the field-by-field map to the reference objects
// (_Pod sim_engine.py:262-274, _FunctionState :277-299, GpuNode packer.py:147-152,
// BackendTable token_backend.py:78-93, GpuMemoryState memory_model.py:36-58).
#pragma once
#include <stdint.h>
#include <stddef.h>

namespace gs {

// pod flag bits
enum : int {
  PF_ALIVE = 1,    // slot holds a pod (placed, retrying or pending placement)
  PF_PLACED = 2,   // in fn.pods and node.placements
  PF_REG = 4,      // registered in its node's BackendTable
  PF_RETRY = 8,    // in _Engine.retry
  PF_CUR = 16,     // pod.current is not None
  PF_GRANT = 32,   // holds a live token this quantum step
};

struct Layout {
  // pods [P]
  size_t p_fn, p_pt, p_node, p_flags, p_warm, p_ctr, p_x, p_y, p_w, p_h, p_cw, p_ci;
  size_t p_okey;                                       // u64 pod-id order key
  size_t p_sm, p_qreq, p_qlim, p_qused, p_busy, p_invr, p_crem, p_carr, p_dur;  // f64
  // functions [F]
  size_t f_qlen, f_pinned, f_fw, f_fi, f_fn, f_nsn, f_nsw, f_nsi, f_rhead, f_retn;
  size_t f_pctr, f_warr, f_wcomp, f_wviol, f_wdrop, f_hn, f_ringoff, f_loff;  // f_loff [F+1]
  size_t f_hist;                                       // f64 [3F]
  size_t f_ret;                                        // i64 [F*RET]
  size_t f_ring;                                       // i64 [ring_total]
  // nodes [G]
  size_t n_sr, n_cov, n_occ, n_fp;                     // f64
  size_t n_nfree, n_nres, n_nplaced, n_seg;            // i32 (n_seg [G+1])
  size_t n_rect;                                       // int4 [G*R]
  size_t n_res;                                        // int2 [G*F] resident (fn,count), insertion order
  size_t n_cnt;                                        // i32 [G*F] dense resident counts
  size_t n_reqsm, n_cut, n_ngr;                        // i32 [G] XL step scratch
  size_t n_covb;                                       // u64 [G] XL step scratch
  // scratch
  size_t s_rl, s_fl, s_free, s_batch, s_list;         // i32 [P]
  size_t s_ka;                                         // u64 [Q]  Q = pow2 >= P
  size_t s_kd;                                         // u64 [Q]
  size_t s_ki;                                         // i32 [Q]
  size_t s_carve;                                      // int4 [4R+8]
  size_t s_rs;                                         // int4 [4R+8] restructure list
  size_t s_pos;                                        // int2 [P] restructure positions
  size_t s_fcur;                                       // i32 [F+1] per-function cursors (epoch)
  size_t bytes;
  int Q;
};

__host__ __device__ inline size_t gs_align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline int gs_pow2_at_least(int n) {
  int q = 1;
  while (q < n) q <<= 1;
  return q;
}

__host__ __device__ inline Layout gs_make_layout(int G, int F, int P, int R, int RET,
                                                 long long ring_total) {
  Layout L;
  size_t o = 0;
  auto take = [&](size_t& field, size_t n, size_t elem) {
    field = o;
    o = gs_align16(o + n * elem);
  };
  const size_t I = 4, D = 8;
  take(L.p_fn, P, I); take(L.p_pt, P, I); take(L.p_node, P, I); take(L.p_flags, P, I);
  take(L.p_warm, P, I); take(L.p_ctr, P, I); take(L.p_x, P, I); take(L.p_y, P, I);
  take(L.p_w, P, I); take(L.p_h, P, I); take(L.p_cw, P, I); take(L.p_ci, P, I);
  take(L.p_okey, P, D);
  take(L.p_sm, P, D); take(L.p_qreq, P, D); take(L.p_qlim, P, D); take(L.p_qused, P, D);
  take(L.p_busy, P, D); take(L.p_invr, P, D); take(L.p_crem, P, D); take(L.p_carr, P, D);
  take(L.p_dur, P, D);
  take(L.f_qlen, F, I); take(L.f_pinned, F, I); take(L.f_fw, F, I); take(L.f_fi, F, I);
  take(L.f_fn, F, I); take(L.f_nsn, F, I); take(L.f_nsw, F, I); take(L.f_nsi, F, I);
  take(L.f_rhead, F, I); take(L.f_retn, F, I); take(L.f_pctr, F, I); take(L.f_warr, F, I);
  take(L.f_wcomp, F, I); take(L.f_wviol, F, I); take(L.f_wdrop, F, I); take(L.f_hn, F, I);
  take(L.f_ringoff, F, I); take(L.f_loff, F + 1, I);
  take(L.f_hist, 3 * (size_t)F, D);
  take(L.f_ret, (size_t)F * RET, D);
  take(L.f_ring, (size_t)(ring_total > 0 ? ring_total : 1), D);
  take(L.n_sr, G, D); take(L.n_cov, G, D); take(L.n_occ, G, D); take(L.n_fp, G, D);
  take(L.n_nfree, G, I); take(L.n_nres, G, I); take(L.n_nplaced, G, I);
  take(L.n_seg, G + 1, I);
  take(L.n_rect, (size_t)G * R, 16);
  take(L.n_res, (size_t)G * F, 8);
  take(L.n_cnt, (size_t)G * F, I);
  take(L.n_reqsm, G, I); take(L.n_cut, G, I); take(L.n_ngr, G, I);
  take(L.n_covb, G, D);
  int Q = gs_pow2_at_least(P > 32 ? P : 32);
  L.Q = Q;
  take(L.s_rl, P, I); take(L.s_fl, P, I); take(L.s_free, P, I);
  take(L.s_batch, P, I); take(L.s_list, P, I);
  take(L.s_ka, Q, D); take(L.s_kd, Q, D); take(L.s_ki, Q, I);
  take(L.s_carve, 4 * (size_t)R + 8, 16);
  take(L.s_rs, 4 * (size_t)R + 8, 16);
  take(L.s_pos, P, 8);
  take(L.s_fcur, (size_t)F + 1, I);
  L.bytes = o;
  return L;
}

}  // namespace gs
