// gs_kernel.cu -- run driver, kernel entry and the C ABI (include/gshare_b200.h).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -lineinfo
//        -Xcompiler -fPIC -shared  (see paper_2309_00558_b200/build.py)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <new>
#include <numeric>
#include <type_traits>
#include <vector>

#include "gs_kernel.cuh"
#include "gs_hot.cuh"
#include "gs_audit.cuh"
#include "gs_xl.cuh"
#include "gs_xlh.cuh"

namespace gs {

constexpr int MAX_WARPS_PER_BLOCK = 4;   // launch bounds: 128 threads x 6 blocks/SM

struct Accum {            // per-lane run totals (reduced at the end)
  long long arrivals, completions, violations, dropped, final_depth;
};

// ring capacity of bounded queues (sum of max_queue over bounded functions)
__host__ __device__ inline long long run_ring_total(const gs_scenario_t& sc, const gs_function_t* fs) {
  long long t = 0;
  for (int f = 0; f < sc.n_funcs; f++) if (fs[f].max_queue > 0) t += fs[f].max_queue;
  return t;
}

__host__ __device__ inline Layout run_layout(const gs_scenario_t& sc, const gs_function_t* fs) {
  return gs_make_layout(sc.n_nodes, sc.n_funcs, sc.cap_pods, sc.cap_rects, sc.cap_returned,
                        run_ring_total(sc, fs));
}

__device__ void init_run(Ctx& c) {
  #pragma unroll 1
  for (int i = c.lane; i < c.P; i += 32) {
    c.t->p_flags[i] = 0;
    c.t->s_free[i] = c.P - 1 - i;  // slot 0 is allocated first
  }
  #pragma unroll 1
  for (int f = c.lane; f < c.F; f += 32) {
    c.t->f_qlen[f] = 0; c.t->f_pinned[f] = 0; c.t->f_fw[f] = 0; c.t->f_fi[f] = 0; c.t->f_fn[f] = 0;
    c.t->f_nsn[f] = 0; c.t->f_nsw[f] = 0; c.t->f_nsi[f] = 0; c.t->f_rhead[f] = 0; c.t->f_retn[f] = 0;
    c.t->f_pctr[f] = 0; c.t->f_warr[f] = 0; c.t->f_wcomp[f] = 0; c.t->f_wviol[f] = 0; c.t->f_wdrop[f] = 0;
    c.t->f_hn[f] = 0;
  }
  #pragma unroll 1
  for (int g = c.lane; g < c.G; g += 32) {
    c.t->n_sr[g] = 0.0; c.t->n_cov[g] = 0.0; c.t->n_occ[g] = 0.0; c.t->n_fp[g] = 0.0;
    c.t->n_nfree[g] = 1; c.t->n_nres[g] = 0; c.t->n_nplaced[g] = 0;
    c.t->n_rect[g * c.R] = make_int4(0, 0, c.sc->side_x, c.sc->side_y);
  }
  #pragma unroll 1
  for (int i = c.lane; i < c.G * c.F; i += 32) c.t->n_cnt[i] = 0;
  if (c.lane == 0) {
    int off = 0;
    #pragma unroll 1
    for (int f = 0; f < c.F; f++) {
      c.t->f_ringoff[f] = off;
      if (c.fs[f].max_queue > 0) off += c.fs[f].max_queue;
    }
    WarpShared* s = c.sh;
    s->n_reg = 0; s->free_top = c.P; s->win_failures = 0; s->n_batch = 0;
    s->err = 0; s->err_detail = 0; s->err_a0 = 0; s->err_a1 = 0; s->n_list = 0;
    s->grants = 0; s->decisions = 0; s->attempts = 0; s->frag = 0.0;
    s->pod_steps = 0; s->rect_scans = 0; s->min_free = c.P;
    s->ka_arena = nullptr; s->kd_arena = nullptr; s->ki_arena = nullptr;
  }
  __syncwarp();
}

__device__ void window_close(Ctx& c, int w, const gs_out_t& out, Accum& acc, PySum& su,
                             PySum& so, int& peak, int& fail_total) {
  const gs_scenario_t& sc = *c.sc;
  #pragma unroll 1
  for (int f = c.lane; f < c.F; f += 32) {
    int hn = c.t->f_hn[f];
    c.t->f_hist[3 * f + hn % 3] = (double)c.t->f_warr[f] / c.ws;   // history.append(n / W)
    c.t->f_hn[f] = hn + 1;
    int depth = c.t->f_qlen[f] + c.t->f_fn[f];                      // len(queue) + len(future)
    if (out.fn_rows) {
      gs_fn_row_t r;
      r.arrivals = c.t->f_warr[f]; r.completions = c.t->f_wcomp[f]; r.slo_violations = c.t->f_wviol[f];
      r.dropped = c.t->f_wdrop[f]; r.queue_depth = depth;
      out.fn_rows[sc.fn_row_off + (long long)w * c.F + f] = r;
    }
    acc.arrivals += c.t->f_warr[f]; acc.completions += c.t->f_wcomp[f];
    acc.violations += c.t->f_wviol[f]; acc.dropped += c.t->f_wdrop[f];
    if (w == c.W - 1) acc.final_depth += depth;
    c.t->f_wcomp[f] = 0; c.t->f_wviol[f] = 0; c.t->f_wdrop[f] = 0;
  }
  int in_use = 0;
  #pragma unroll 1
  for (int g = c.lane; g < c.G; g += 32) {
    gs_gpu_row_t r;
    r.present = c.t->n_nplaced[g] > 0 ? 1 : 0;
    r.pad = 0;
    double cov = c.t->n_cov[g], occ = c.t->n_occ[g];
    r.utilization = r.present ? (cov < 1.0 ? cov : 1.0) : 0.0;
    r.sm_occupancy = r.present ? (occ < 1.0 ? occ : 1.0) : 0.0;
    r.memory_mb = r.present ? c.t->n_fp[g] : 0.0;
    if (out.gpu_rows) out.gpu_rows[sc.gpu_row_off + (long long)w * c.G + g] = r;
    in_use += r.present;
  }
  in_use = warp_sum_i(in_use);
  __syncwarp();
  if (c.lane == 0) {
    #pragma unroll 1
    for (int g = 0; g < c.G; g++) {           // summary sums in CSV row order
      if (c.t->n_nplaced[g] <= 0) continue;
      double cov = c.t->n_cov[g], occ = c.t->n_occ[g];
      su.add(cov < 1.0 ? cov : 1.0);
      so.add(occ < 1.0 ? occ : 1.0);
    }
    if (out.glob_rows) {
      gs_glob_row_t r;
      r.gpus_in_use = in_use;
      r.placement_failures = c.sh->win_failures;
      r.fragmentation_index = c.sh->frag;
      out.glob_rows[sc.glob_row_off + w] = r;
    }
    peak = in_use > peak ? in_use : peak;
    fail_total += c.sh->win_failures;
    c.sh->win_failures = 0;
  }
  __syncwarp();
}

// _close_window (sim_engine.py:554-594) from the shared-memory working set
template <class H>
__device__ void hot_close(Ctx& c, H* h, int w, const gs_out_t& out, Accum& acc, PySum& su,
                          PySum& so, int& peak, int& fail_total) {
  const gs_scenario_t& sc = *c.sc;
  lane_for<HotCap<H>::FC>(c.lane, c.F, [&](int f) {
    const int hn = h->hn[f];
    c.t->f_hist[3 * f + hn % 3] = (double)h->warr[f] / c.ws;   // history.append(n / W)
    h->hn[f] = hn + 1;
    const int depth = h->qlen[f] + h->fcnt[f];              // len(queue) + len(future)
    if (out.fn_rows) {
      gs_fn_row_t r;
      r.arrivals = h->warr[f]; r.completions = h->wcomp[f]; r.slo_violations = h->wviol[f];
      r.dropped = h->wdrop[f]; r.queue_depth = depth;
      out.fn_rows[sc.fn_row_off + (long long)w * c.F + f] = r;
    }
    acc.arrivals += h->warr[f]; acc.completions += h->wcomp[f];
    acc.violations += h->wviol[f]; acc.dropped += h->wdrop[f];
    if (w == c.W - 1) acc.final_depth += depth;
    h->wcomp[f] = 0; h->wviol[f] = 0; h->wdrop[f] = 0;
  });
  int in_use = 0;
  lane_for<HotCap<H>::GC>(c.lane, c.G, [&](int g) {
    gs_gpu_row_t r;
    r.present = h->nplaced[g] > 0 ? 1 : 0;
    r.pad = 0;
    const double cov = h->cov[g], occ = h->occ[g];
    r.utilization = r.present ? (cov < 1.0 ? cov : 1.0) : 0.0;
    r.sm_occupancy = r.present ? (occ < 1.0 ? occ : 1.0) : 0.0;
    r.memory_mb = r.present ? h->fp[g] : 0.0;
    if (out.gpu_rows) out.gpu_rows[sc.gpu_row_off + (long long)w * c.G + g] = r;
    in_use += r.present;
  });
  in_use = warp_sum_i(in_use);
  __syncwarp();
  if (c.lane == 0) {
    #pragma unroll 1
    for (int g = 0; g < c.G; g++) {           // summary sums in CSV row order
      if (h->nplaced[g] <= 0) continue;
      const double cov = h->cov[g], occ = h->occ[g];
      su.add(cov < 1.0 ? cov : 1.0);
      so.add(occ < 1.0 ? occ : 1.0);
    }
    if (out.glob_rows) {
      gs_glob_row_t r;
      r.gpus_in_use = in_use;
      r.placement_failures = c.sh->win_failures;
      r.fragmentation_index = c.sh->frag;
      out.glob_rows[sc.glob_row_off + w] = r;
    }
    peak = in_use > peak ? in_use : peak;
    fail_total += c.sh->win_failures;
    c.sh->win_failures = 0;
  }
  __syncwarp();
}

template <class H> __host__ __device__ constexpr int class_id() {
  if constexpr (std::is_same<H, HotXS>::value) return 1;
  else if constexpr (std::is_same<H, HotS>::value) return 2;
  else if constexpr (std::is_same<H, HotM>::value) return 3;
  else if constexpr (std::is_same<H, HotL>::value) return 4;
  else return 5;
}
template <class H> __host__ __device__ constexpr size_t hot_bytes() {
  if constexpr (std::is_void<H>::value) return 0;
  else return sizeof(H);
}

// Coalesced 4-byte word copy of one run's output rows from HBM to mapped,
// page-locked host memory (zero-copy): each warp store is one contiguous
// 128-byte line on PCIe/C2C, and the copy overlaps the other runs' compute.
__device__ void copy_words(void* dst, const void* src, size_t bytes, int lane) {
  const unsigned* s = reinterpret_cast<const unsigned*>(src);
  unsigned* d = reinterpret_cast<unsigned*>(dst);
  const size_t n = bytes / 4;
#pragma unroll 4
  for (size_t k = lane; k < n; k += 32) d[k] = __ldcs(s + k);
}

__device__ void copy_out_run(const gs_scenario_t& sc, const gs_out_t& out, const gs_out_t& host,
                             int nplaced, int lane) {
  const long long W = sc.windows;
  if (host.fn_rows && out.fn_rows)
    copy_words(host.fn_rows + sc.fn_row_off, out.fn_rows + sc.fn_row_off,
               sizeof(gs_fn_row_t) * (size_t)(W * sc.n_funcs), lane);
  if (host.gpu_rows && out.gpu_rows)
    copy_words(host.gpu_rows + sc.gpu_row_off, out.gpu_rows + sc.gpu_row_off,
               sizeof(gs_gpu_row_t) * (size_t)(W * sc.n_nodes), lane);
  if (host.glob_rows && out.glob_rows)
    copy_words(host.glob_rows + sc.glob_row_off, out.glob_rows + sc.glob_row_off,
               sizeof(gs_glob_row_t) * (size_t)W, lane);
  if (host.placements && out.placements)
    copy_words(host.placements + sc.place_off, out.placements + sc.place_off,
               sizeof(gs_placement_t) * (size_t)nplaced, lane);
}

// one window stepped on the HBM arena (warp-level; out of line -- it only runs
// when a run's registered set outgrows its shared-memory class)
__device__ __noinline__ void arena_window(Ctx& c, int w, const gs_out_t& out, Accum& acc,
                                          PySum& su, PySum& so, int& peak, int& fail_total) {
  #pragma unroll 1
  for (int g = c.lane; g < c.G; g += 32) { c.t->n_cov[g] = 0.0; c.t->n_occ[g] = 0.0; }
  __syncwarp();
  #pragma unroll 1
  for (int s = 0; s < c.T; s++) run_step(c, w, s);
  complete_tokens(c);
  window_close(c, w, out, acc, su, so, peak, fail_total);
}

// status, summary, final placements and the zero-copy row copy-out of a
// finished run (warp-level; lane 0 writes the records)
__device__ void finish_run(Ctx& c, const gs_out_t& out, const gs_out_t& host, int run,
                           Accum& acc, PySum& su, PySum& so, int peak, int fail_total,
                           long long hot_grants, long long hot_pod_steps, int cls,
                           bool hot_counters) {
  // outputs
  gs_status_t st;
  memset(&st, 0, sizeof(st));
  int nplaced = 0;
  if (!c.sh->err) {
    const int phi = pod_high(c);
    #pragma unroll 1
    for (int s0 = 0; s0 < phi; s0 += 32) {
      int slot = s0 + c.lane;
      bool take = slot < phi && (c.t->p_flags[slot] & PF_PLACED);
      unsigned bal = __ballot_sync(FULL, take);
      if (take && out.placements) {
        int k = nplaced + __popc(bal & ((1u << c.lane) - 1u));
        gs_placement_t p;
        p.node = c.t->p_node[slot]; p.func = c.t->p_fn[slot]; p.counter = c.t->p_ctr[slot];
        p.x = c.t->p_x[slot]; p.y = c.t->p_y[slot]; p.w = c.t->p_w[slot]; p.h = c.t->p_h[slot]; p.pad = 0;
        out.placements[c.sc->place_off + k] = p;
      }
      nplaced += __popc(bal);
    }
  }
  acc.arrivals = warp_sum_ll(acc.arrivals);
  acc.completions = warp_sum_ll(acc.completions);
  acc.violations = warp_sum_ll(acc.violations);
  acc.dropped = warp_sum_ll(acc.dropped);
  acc.final_depth = warp_sum_ll(acc.final_depth);
  __syncwarp();
  if (c.lane == 0) {
    st.code = c.sh->err; st.detail = c.sh->err_detail;
    st.arg0 = c.sh->err_a0; st.arg1 = c.sh->err_a1;
    st.n_placements = nplaced;
    st.hot_class = cls;
    st.token_grants = c.sh->grants + hot_grants;
    st.scale_decisions = c.sh->decisions;
    st.placement_attempts = c.sh->attempts;
    st.pod_steps = hot_counters ? hot_pod_steps : c.sh->pod_steps;
    st.rect_scans = c.sh->rect_scans;
    st.peak_pods = c.P - c.sh->min_free;
    out.status[run] = st;
    if (out.summary) {
      gs_summary_t sm;
      sm.windows = c.W; sm.gpus_used_peak = peak; sm.placement_failures = fail_total;
      sm.n_gpu_rows = su.n;
      sm.arrivals = acc.arrivals; sm.completions = acc.completions;
      sm.slo_violations = acc.violations; sm.dropped = acc.dropped;
      sm.final_queue_depth = acc.final_depth;
      sm.sum_utilization = su.value(); sm.sum_sm_occupancy = so.value();
      out.summary[run] = sm;
    }
  }
  __syncwarp();
  if (!c.sh->err) copy_out_run(*c.sc, out, host, nplaced, c.lane);
}

// While the registered set is rebuilt (initial placement, epochs, window
// begin) the warp's shared-memory working set is idle: the sort scratch
// (s_ka / s_kd / s_ki, Q entries each) moves there when it fits, so the
// bitonic sorts of the rebuild hit shared memory instead of the HBM arena.
template <class H>
__device__ __forceinline__ void scratch_to_shared(Ctx& c, H* h) {
  if (20u * (unsigned)c.Q > sizeof(H)) return;
  if (c.lane == 0) {
    char* b = reinterpret_cast<char*>(h);
    c.sh->ka_arena = c.t->s_ka; c.sh->kd_arena = c.t->s_kd; c.sh->ki_arena = c.t->s_ki;
    c.t->s_ka = reinterpret_cast<unsigned long long*>(b);
    c.t->s_kd = reinterpret_cast<unsigned long long*>(b + 8 * (size_t)c.Q);
    c.t->s_ki = reinterpret_cast<int*>(b + 16 * (size_t)c.Q);
  }
  __syncwarp();
}

__device__ __forceinline__ void scratch_to_arena(Ctx& c) {
  if (c.lane == 0 && c.sh->ka_arena) {
    c.t->s_ka = c.sh->ka_arena; c.t->s_kd = c.sh->kd_arena; c.t->s_ki = c.sh->ki_arena;
    c.sh->ka_arena = nullptr;
  }
  __syncwarp();
}

template <class H>
__device__ void simulate_run(Ctx& c, const gs_out_t& out, const gs_out_t& host, int run, H* h) {
  init_run(c);
  scratch_to_shared(c, h);
  // initial pods: sorted fid order, spec order (sim_engine.py:436-441)
  if (c.lane == 0) {
    #pragma unroll 1
    for (int f = 0; f < c.F && !c.sh->err; f++) {
      const gs_function_t& fs = c.fs[f];
      #pragma unroll 1
      for (int i = 0; i < fs.n_init; i++) {
        const gs_init_t& ip = c.inits[fs.init_off + i];
        if (make_pod(c, f, ip.point, ip.has_q_req, ip.q_req, 0) < 0) break;
      }
    }
  }
  __syncwarp();
  Accum acc = {0, 0, 0, 0, 0};
  PySum su, so;
  su.reset();
  so.reset();
  int peak = 0, fail_total = 0;
  if (!failed(c)) place_batch(c);
  if (!failed(c)) refresh_frag(c);
  scratch_to_arena(c);
  bool hot_valid = false;
  long long pod_steps = 0, hot_grants = 0;   // hot-path counters kept in registers
  #pragma unroll 1
  for (int w = 0; w < c.W && !failed(c); w++) {
    const bool epoch = w > 0 && w % c.sc->epoch_windows == 0;
    {
      // Registration changes only at epochs and when a placed pod warms up;
      // otherwise the shared-memory working set carries over to the next window.
      const bool rebuild = !hot_valid || epoch || w >= c.sh->next_warm;
      if (rebuild) {
        if (hot_valid) hot_store(c, h);
        scratch_to_shared(c, h);
        if (epoch) {
          run_epoch(c, w);
          if (failed(c)) { scratch_to_arena(c); break; }
        }
        window_begin(c, w);
        scratch_to_arena(c);
        hot_valid = hot_load(c, h);
      } else {
        hot_begin_light(h, c.lane, w);
      }
#ifdef GS_XL_TIMING
      if (c.lane == 0) atomicAdd(&gs_xl_t[hot_valid ? 30 : 31], 1ull);
#endif
      if (hot_valid) {
        pod_steps += (long long)h->n * c.T;
        hot_grants += hot_steps(h, c.lane, w);
        hot_close(c, h, w, out, acc, su, so, peak, fail_total);
      } else {
        // the registered set outgrew the class: this window steps on the arena
        pod_steps += (long long)c.sh->n_reg * c.T;
        arena_window(c, w, out, acc, su, so, peak, fail_total);
      }
    }
  }
  if (hot_valid && !c.sh->err) hot_store(c, h);   // flush the last windows' counters
  finish_run(c, out, host, run, acc, su, so, peak, fail_total, hot_grants, pod_steps,
             class_id<H>(), !std::is_void<H>::value);
}


// XL class driver: warp 0 runs the control code (as simulate_run<void>), all
// XL_THREADS threads run the quantum steps (gs_xl.cuh).  Every thread calls
// this with its own Ctx view of the same run.
// -DGS_XL_TIMING: warp-0 cycle split of the XL driver (tools/xl_timing.py)
#ifdef GS_XL_TIMING
extern "C" int gs_xl_timing(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, gs_xl_t, sizeof(gs_xl_t));
}
#define GS_XL_TIC(v) const long long v = clock64()
#define GS_XL_ADD(k, d) atomicAdd(&gs_xl_t[k], (unsigned long long)(d))
#else
#define GS_XL_TIC(v)
#define GS_XL_ADD(k, d)
#endif
__device__ void simulate_run_xl(Ctx& c, const gs_out_t& out, const gs_out_t& host, int run,
                                XlShared* xs, HotX* hx, char* xdyn, size_t xbytes) {
  const bool w0 = threadIdx.x < 32;
  Accum acc = {0, 0, 0, 0, 0};
  PySum su, so;
  su.reset();
  so.reset();
  int peak = 0, fail_total = 0;
  if (w0) {
    init_run(c);
    if (c.lane == 0) {
      #pragma unroll 1
      for (int f = 0; f < c.F && !c.sh->err; f++) {
        const gs_function_t& fs = c.fs[f];
        #pragma unroll 1
        for (int i = 0; i < fs.n_init; i++) {
          const gs_init_t& ip = c.inits[fs.init_off + i];
          if (make_pod(c, f, ip.point, ip.has_q_req, ip.q_req, 0) < 0) break;
        }
      }
    }
    __syncwarp();
    if (!failed(c)) place_batch(c);
    if (!failed(c)) refresh_frag(c);
  }
  if (threadIdx.x == 0) {
    xlh_carve(hx, xdyn, xbytes, c.F, c.G);
    int bnd = 0;
    for (int f = 0; f < c.F; f++) bnd |= c.fs[f].max_queue >= 0;
    hx->bounded = bnd;
  }
  __syncthreads();
  bool lists_valid = false;            // s_rl / n_seg / s_fl match the registered set
  bool hot = false;                    // the shared-memory working set holds the run
  #pragma unroll 1
  for (int w = 0; w < c.W; w++) {
    // registration changes only at epochs and warm-ups; otherwise the sorted
    // registered list and the per-function lists carry over (cf. hot_begin_light)
    const bool epoch = w > 0 && w % c.sc->epoch_windows == 0;
    const bool rebuild = !lists_valid || epoch || w >= c.sh->next_warm;
    __syncthreads();                   // everyone read next_warm before warp 0 moves on
    if (rebuild) {
      if (hot) {                       // write the working set back before the epoch
        xlh_store(c, hx);
        hot = false;
      }
      GS_XL_TIC(t0_);
      if (epoch && !c.sh->err) {       // decisions on every warp, applied by warp 0
        if (!xl_run_epoch(c, w, xdyn, xbytes, xs)) {
          if (w0) run_epoch(c, w);
        }
      }
      if (w0) {
        const bool stop = failed(c);
        GS_XL_TIC(t1_);
        if (c.lane == 0) { GS_XL_ADD(0, t1_ - t0_); }
        if (c.lane == 0) xs->stop = stop ? 1 : 0;
      }
      lists_valid = true;
      __syncthreads();
      if (xs->stop) break;
      GS_XL_TIC(t2_);
      if (!xl_window_begin(c, w, xdyn, xbytes, xs->warp_tot)) {
        if (w0) window_begin(c, w);
        __syncthreads();
      }
      if (threadIdx.x == 0) { GS_XL_ADD(1, clock64() - t2_); }
      hot = xlh_load(c, hx);           // false: the registered set does not fit
    } else if (hot) {
      xlh_begin_light(hx, w);
      if (threadIdx.x == 0) { xs->stop = 0; c.sh->pod_steps += (long long)hx->n * c.T; }
    } else {
      xl_begin_light(c, w);
      if (threadIdx.x == 0) xs->stop = 0;
    }
    if (!hot) {
      #pragma unroll 1
      for (int g = threadIdx.x; g < c.G; g += blockDim.x) { c.t->n_cov[g] = 0.0; c.t->n_occ[g] = 0.0; }
    }
    __syncthreads();
    if (xs->stop) break;
    GS_XL_TIC(t3_);
    if (threadIdx.x == 0) { GS_XL_ADD(15, hot ? 0 : 1); }
    if (hot) {
      #pragma unroll 1
      for (int s = 0; s < c.T; s++) {
        if (hx->bounded) xlh_step<true>(hx, w, s, xs);
        else xlh_step<false>(hx, w, s, xs);
        if (threadIdx.x == 0) c.sh->grants += xs->grants;
      }
      xlh_complete(hx);
    } else {
      #pragma unroll 1
      for (int s = 0; s < c.T; s++) xl_step(c, w, s, xs);
      xl_complete(c);
    }
    GS_XL_TIC(t4_);
    if (w0) {
      if (hot) hot_close(c, hx, w, out, acc, su, so, peak, fail_total);
      else window_close(c, w, out, acc, su, so, peak, fail_total);
    }
    if (threadIdx.x == 0) { GS_XL_ADD(2, t4_ - t3_); GS_XL_ADD(3, clock64() - t4_); }
    __syncthreads();
  }
  __syncthreads();
  if (hot && !c.sh->err) xlh_store(c, hx);     // flush the last windows' state
  if (w0) finish_run(c, out, host, run, acc, su, so, peak, fail_total, 0, 0, 5, false);
  __syncthreads();
}

struct KArgs {
  gs_batch_t in;              // device pointers
  gs_out_t out;               // device pointers
  gs_out_t host;              // mapped host mirrors of out's rows (zero-copy), or NULL
  char* arena;
  const long long* ws_off;
  const int* order;           // runs of this size class, longest first
  int n_order;
  int* counter;
  int xl_bytes;               // XL class: dynamic shared memory of the working set
};

#ifndef GS_MIN_BLOCKS
#define GS_MIN_BLOCKS 6   // 128-thread CTAs per SM the register budget must allow
#endif
// class XS trades a few spilled registers (64 instead of 80) for 32 resident
// warps per SM: its runs are short and latency-bound (C1 +40%, C5 +8%)
template <class H> struct MinBlocks { static constexpr int value = GS_MIN_BLOCKS; };
template <> struct MinBlocks<HotXS> { static constexpr int value = 8; };

template <class H>
__global__ void __launch_bounds__(128, MinBlocks<H>::value)
gs_sim_kernel(KArgs a) {
  __shared__ WarpShared shs[MAX_WARPS_PER_BLOCK];
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  WarpShared* sh = &shs[wib];
  H* hot = reinterpret_cast<H*>(dyn_smem + (size_t)wib * hot_bytes<H>());
  for (;;) {
    int r = 0;
    if (lane == 0) r = atomicAdd(a.counter, 1);
    r = __shfl_sync(FULL, r, 0);
    if (r >= a.n_order) break;
    const int run = a.order[r];
    Ctx c;
    c.sc = &a.in.runs[run];
    c.fs = &a.in.funcs[c.sc->func_off];
    c.points = a.in.points;
    c.counts = a.in.counts;
    c.inits = a.in.inits;
    c.splits = a.in.id_splits;
    c.G = c.sc->n_nodes; c.F = c.sc->n_funcs; c.P = c.sc->cap_pods; c.R = c.sc->cap_rects;
    c.RET = c.sc->cap_returned; c.W = c.sc->windows; c.T = c.sc->steps; c.flags = c.sc->flags;
    c.ws = c.sc->window_s; c.qs = c.sc->quantum_s; c.quantum = c.sc->quantum;
    c.cap_mb = c.sc->capacity_mb;
    c.lane = lane;
    c.sh = sh;
    c.t = &sh->tab;
    Layout L = run_layout(*c.sc, c.fs);
    ctx_bind(c, a.arena + a.ws_off[run], L);
    simulate_run<H>(c, a.out, a.host, run, hot);
  }
}


// XL class: one run per CTA of XL_THREADS threads, runs pulled from the work
// counter longest first.
__global__ void __launch_bounds__(XL_THREADS, 1) gs_sim_kernel_xl(KArgs a) {
  __shared__ WarpShared sh;
  __shared__ XlShared xs;
  __shared__ HotX hx;
  extern __shared__ __align__(16) unsigned char xl_dyn[];
  for (;;) {
    if (threadIdx.x == 0) xs.run = atomicAdd(a.counter, 1);
    __syncthreads();
    const int r = xs.run;
    __syncthreads();
    if (r >= a.n_order) break;
    const int run = a.order[r];
    Ctx c;
    c.sc = &a.in.runs[run];
    c.fs = &a.in.funcs[c.sc->func_off];
    c.points = a.in.points;
    c.counts = a.in.counts;
    c.inits = a.in.inits;
    c.splits = a.in.id_splits;
    c.G = c.sc->n_nodes; c.F = c.sc->n_funcs; c.P = c.sc->cap_pods; c.R = c.sc->cap_rects;
    c.RET = c.sc->cap_returned; c.W = c.sc->windows; c.T = c.sc->steps; c.flags = c.sc->flags;
    c.ws = c.sc->window_s; c.qs = c.sc->quantum_s; c.quantum = c.sc->quantum;
    c.cap_mb = c.sc->capacity_mb;
    c.lane = threadIdx.x & 31;
    c.sh = &sh;
    c.t = &sh.tab;
    if (threadIdx.x < 32) {
      Layout L = run_layout(*c.sc, c.fs);
      ctx_bind(c, a.arena + a.ws_off[run], L);
    } else {
      c.Q = 0;
    }
    __syncthreads();
    simulate_run_xl(c, a.out, a.host, run, &xs, &hx, reinterpret_cast<char*>(xl_dyn), (size_t)a.xl_bytes);
  }
}

}  // namespace gs

// ============================================================================
// C ABI
// ============================================================================
using namespace gs;

namespace {

// Process-wide launch-shape DEFAULTS (tuning knobs, gs_set_launch /
// gs_set_xl_smem).  They are copied into a session when it is created and
// never read by a launch, so concurrent sessions (several devices, streams or
// threads) each run with the shape they were created with.
std::atomic<int> g_warps_per_block{4};
std::atomic<int> g_blocks_per_sm{0};
std::atomic<int> g_xl_bytes{(int)XLH_DYN_BYTES};

void put_err(char* err, size_t n, const char* msg) {
  if (err && n) { std::snprintf(err, n, "%s", msg); }
}

#define CK(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      char b_[256];                                                            \
      std::snprintf(b_, sizeof b_, "%s: %s", #call, cudaGetErrorString(e_));   \
      put_err(err, err_len, b_);                                               \
      return GS_ERR_CUDA;                                                      \
    }                                                                          \
  } while (0)

template <typename T>
size_t nbytes(long long n) { return sizeof(T) * (size_t)(n > 0 ? n : 1); }

}  // namespace

// smallest shared-memory size class whose capacities hold F functions and G
// nodes (registered pods are checked per window on the device)
static int run_class(const gs_scenario_t& sc) {
  int k = 5;
  if (sc.n_funcs <= HotXS::FC && sc.n_nodes <= HotXS::GC) k = 1;
  else if (sc.n_funcs <= HotS::FC && sc.n_nodes <= HotS::GC) k = 2;
  else if (sc.n_funcs <= HotM::FC && sc.n_nodes <= HotM::GC) k = 3;
  else if (sc.n_funcs <= HotL::FC && sc.n_nodes <= HotL::GC) k = 4;
  if (sc.hot_class > k) k = sc.hot_class > 5 ? 5 : sc.hot_class;
  return k;
}

struct gs_session {
  int device = 0;
  gs_batch_t dev_in{};        // device pointers
  gs_out_t dev_out{};
  char* blob = nullptr;       // one allocation for inputs+outputs+arena
  size_t blob_bytes = 0;
  long long* ws_off = nullptr;
  int* order = nullptr;
  int* counter = nullptr;        // one work counter per size class
  int class_off[7] = {0, 0, 0, 0, 0, 0, 0};  // order[] slice of class k: [off[k-1], off[k])
  char* arena = nullptr;
  int n_runs = 0;
  int64_t n_fn_rows = 0, n_gpu_rows = 0, n_glob_rows = 0, n_place = 0;
  gs_out_t host_map{};         // device-visible pointers of mapped host row buffers
  gs_out_t host_ptr{};         // the same buffers' host addresses (download skips them)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int last_launches = 0;
  double last_ms = 0.0;
  int warps_per_block = 4;     // launch shape, fixed at creation
  int blocks_per_sm = 0;
  int xl_bytes = (int)XLH_DYN_BYTES;
  size_t input_bytes = 0;
  bool async_alloc = false;    // blob from cudaMallocAsync on `ord` (one-shot calls)
  cudaStream_t ord = nullptr;
};

extern "C" int gs_abi_version(void) { return GS_ABI_VERSION; }

extern "C" int gs_set_xl_smem(int bytes) {
  const int v = bytes <= 0 ? (int)XLH_DYN_BYTES
                           : std::max(16 * 1024, std::min(bytes, (int)XLH_DYN_BYTES)) & ~15;
  g_xl_bytes.store(v);
  return v;
}

extern "C" int gs_set_launch(int warps_per_block, int blocks_per_sm) {
  if (warps_per_block > 0) g_warps_per_block.store(std::min(warps_per_block, MAX_WARPS_PER_BLOCK));
  if (blocks_per_sm >= 0) g_blocks_per_sm.store(blocks_per_sm);
  return 0;
}

// `ord`: a stream for stream-ordered allocation and input copies (the one-shot
// path: no device-wide synchronisation, so one-shot calls from several host
// threads overlap on the GPU); nullptr = cudaMalloc + synchronous copies.
static int session_create(const gs_batch_t* in, int device, cudaStream_t ord, bool async_alloc,
                          gs_session_t** sess_out, char* err, size_t err_len) {
  if (!in || !sess_out || in->n_runs < 0) { put_err(err, err_len, "bad arguments"); return GS_ERR_ARG; }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device) {
    put_err(err, err_len, "no CUDA device visible");
    return GS_ERR_CUDA;
  }
  CK(cudaSetDevice(device));
  gs_session* s = new (std::nothrow) gs_session();
  if (!s) { put_err(err, err_len, "out of host memory"); return GS_ERR_ARG; }
  s->device = device;
  s->warps_per_block = g_warps_per_block.load();
  s->blocks_per_sm = g_blocks_per_sm.load();
  s->xl_bytes = g_xl_bytes.load();
  s->n_runs = in->n_runs;
  s->n_fn_rows = in->n_fn_rows; s->n_gpu_rows = in->n_gpu_rows;
  s->n_glob_rows = in->n_glob_rows; s->n_place = in->n_placements;

  // per-run workspace offsets + longest-first order (host copies available)
  const int R = in->n_runs;
  std::vector<long long> ws_off(R > 0 ? R : 1, 0);
  std::vector<int> order(R > 0 ? R : 1, 0);
  std::vector<double> cost(R > 0 ? R : 1, 0.0);
  std::vector<int> cls(R > 0 ? R : 1, 5);
  long long arena_bytes = 0;
  for (int r = 0; r < R; r++) {
    const gs_scenario_t& sc = in->runs[r];
    if (sc.func_off < 0 || sc.func_off + sc.n_funcs > in->n_funcs || sc.n_nodes < 1 ||
        sc.cap_pods < 1 || sc.cap_rects < 4 || sc.cap_returned < 1) {
      put_err(err, err_len, "malformed run record");
      delete s;
      return GS_ERR_ARG;
    }
    Layout L = run_layout(sc, in->funcs + sc.func_off);
    ws_off[r] = arena_bytes;
    arena_bytes += (long long)gs_align16(L.bytes);
    cost[r] = (double)sc.windows * sc.steps * (sc.n_funcs + sc.n_nodes + 0.25 * sc.cap_pods);
    cls[r] = run_class(sc);
    order[r] = r;
  }
  for (int f = 0; f < in->n_funcs; f++) {
    const gs_function_t& fn = in->funcs[f];
    if (fn.n_id_splits < 0 || (fn.n_id_splits > 0 &&
        (!in->id_splits || fn.id_split_off < 0 ||
         (long long)fn.id_split_off + fn.n_id_splits > in->n_id_splits))) {
      put_err(err, err_len, "malformed function record (pod-id order splits)");
      delete s;
      return GS_ERR_ARG;
    }
  }
  std::stable_sort(order.begin(), order.begin() + R, [&](int a, int b) {
    return cls[a] != cls[b] ? cls[a] < cls[b] : cost[a] > cost[b];
  });
  for (int k = 1; k <= 5; k++) {
    int cnt = 0;
    for (int r = 0; r < R; r++) cnt += cls[r] <= k;
    s->class_off[k] = cnt;
  }

  // one blob: inputs | outputs | ws_off | order | counter | arena
  size_t off = 0;
  auto slot = [&](size_t n) { size_t o = off; off = gs_align16(off + n); return o; };
  size_t o_runs = slot(nbytes<gs_scenario_t>(in->n_runs));
  size_t o_funcs = slot(nbytes<gs_function_t>(in->n_funcs));
  size_t o_points = slot(nbytes<gs_point_t>(in->n_points));
  size_t o_inits = slot(nbytes<gs_init_t>(in->n_inits));
  size_t o_counts = slot(nbytes<int32_t>(in->n_counts));
  size_t o_names = slot(nbytes<char>(in->n_names));
  size_t o_splits = slot(nbytes<gs_id_split_t>(in->n_id_splits));
  size_t in_end = off;
  size_t o_fn = slot(nbytes<gs_fn_row_t>(in->n_fn_rows));
  size_t o_gpu = slot(nbytes<gs_gpu_row_t>(in->n_gpu_rows));
  size_t o_glob = slot(nbytes<gs_glob_row_t>(in->n_glob_rows));
  size_t o_place = slot(nbytes<gs_placement_t>(in->n_placements));
  size_t o_status = slot(nbytes<gs_status_t>(in->n_runs));
  size_t o_summary = slot(nbytes<gs_summary_t>(in->n_runs));
  size_t o_wsoff = slot(nbytes<long long>(R));
  size_t o_order = slot(nbytes<int>(R));
  size_t o_counter = slot(8 * sizeof(int));
  size_t o_arena = slot((size_t)(arena_bytes > 0 ? arena_bytes : 16));
  s->blob_bytes = off;
  s->async_alloc = async_alloc;
  s->ord = ord;
  cudaError_t e = async_alloc ? cudaMallocAsync(&s->blob, s->blob_bytes, ord)
                              : cudaMalloc(&s->blob, s->blob_bytes);
  if (e != cudaSuccess) {
    char b[256];
    std::snprintf(b, sizeof b, "cudaMalloc(%zu bytes): %s", s->blob_bytes, cudaGetErrorString(e));
    put_err(err, err_len, b);
    delete s;
    return GS_ERR_CUDA;
  }
  char* B = s->blob;
  auto up = [&](size_t o, const void* src, size_t n) -> cudaError_t {
    if (!src || !n) return cudaSuccess;
    // pageable sources are staged before cudaMemcpyAsync returns; page-locked
    // ones are read on `ord`, which the one-shot caller synchronises
    return async_alloc ? cudaMemcpyAsync(B + o, src, n, cudaMemcpyHostToDevice, ord)
                       : cudaMemcpy(B + o, src, n, cudaMemcpyHostToDevice);
  };
  cudaError_t ce = cudaSuccess;
  if (ce == cudaSuccess) ce = up(o_runs, in->runs, sizeof(gs_scenario_t) * (size_t)in->n_runs);
  if (ce == cudaSuccess) ce = up(o_funcs, in->funcs, sizeof(gs_function_t) * (size_t)in->n_funcs);
  if (ce == cudaSuccess) ce = up(o_points, in->points, sizeof(gs_point_t) * (size_t)in->n_points);
  if (ce == cudaSuccess) ce = up(o_inits, in->inits, sizeof(gs_init_t) * (size_t)in->n_inits);
  if (ce == cudaSuccess) ce = up(o_counts, in->counts, sizeof(int32_t) * (size_t)in->n_counts);
  if (ce == cudaSuccess) ce = up(o_names, in->names, (size_t)in->n_names);
  if (ce == cudaSuccess)
    ce = up(o_splits, in->id_splits, sizeof(gs_id_split_t) * (size_t)in->n_id_splits);
  if (ce == cudaSuccess) ce = up(o_wsoff, ws_off.data(), sizeof(long long) * (size_t)R);
  if (ce == cudaSuccess) ce = up(o_order, order.data(), sizeof(int) * (size_t)R);
  if (ce != cudaSuccess) {
    put_err(err, err_len, cudaGetErrorString(ce));
    if (async_alloc) { cudaFreeAsync(s->blob, ord); cudaStreamSynchronize(ord); }
    else cudaFree(s->blob);
    delete s;
    return GS_ERR_CUDA;
  }
  s->input_bytes = in_end;
  s->dev_in = *in;
  s->dev_in.runs = reinterpret_cast<const gs_scenario_t*>(B + o_runs);
  s->dev_in.funcs = reinterpret_cast<const gs_function_t*>(B + o_funcs);
  s->dev_in.points = reinterpret_cast<const gs_point_t*>(B + o_points);
  s->dev_in.inits = reinterpret_cast<const gs_init_t*>(B + o_inits);
  s->dev_in.counts = reinterpret_cast<const int32_t*>(B + o_counts);
  s->dev_in.names = reinterpret_cast<const char*>(B + o_names);
  s->dev_in.id_splits = reinterpret_cast<const gs_id_split_t*>(B + o_splits);
  s->dev_out.fn_rows = reinterpret_cast<gs_fn_row_t*>(B + o_fn);
  s->dev_out.gpu_rows = reinterpret_cast<gs_gpu_row_t*>(B + o_gpu);
  s->dev_out.glob_rows = reinterpret_cast<gs_glob_row_t*>(B + o_glob);
  s->dev_out.placements = reinterpret_cast<gs_placement_t*>(B + o_place);
  s->dev_out.status = reinterpret_cast<gs_status_t*>(B + o_status);
  s->dev_out.summary = reinterpret_cast<gs_summary_t*>(B + o_summary);
  s->ws_off = reinterpret_cast<long long*>(B + o_wsoff);
  s->order = reinterpret_cast<int*>(B + o_order);
  s->counter = reinterpret_cast<int*>(B + o_counter);
  s->arena = B + o_arena;
  cudaEventCreate(&s->ev0);
  cudaEventCreate(&s->ev1);
  *sess_out = s;
  return GS_OK;
}

extern "C" int gs_session_create(const gs_batch_t* in, int device, gs_session_t** sess_out,
                                 char* err, size_t err_len) {
  return session_create(in, device, nullptr, false, sess_out, err, err_len);
}

// The dynamic shared-memory opt-in is a per-(device, kernel) attribute whose
// value depends on the session's launch shape: set it before every launch (a
// cheap host call) instead of caching it per process.
template <class H>
static int launch_class(const gs_session* s, const KArgs& a, int sms, cudaStream_t st,
                        char* err, size_t err_len) {
  const int wpb = s->warps_per_block;
  const int threads = wpb * 32;
  const size_t dyn = hot_bytes<H>() * (size_t)wpb;
  CK(cudaFuncSetAttribute(gs_sim_kernel<H>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)std::max<size_t>(dyn, 48 * 1024)));
  int per_sm = s->blocks_per_sm;
  if (per_sm <= 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gs_sim_kernel<H>, threads, dyn));
    if (per_sm < 1) per_sm = 1;
  }
  long long blocks = (long long)sms * per_sm;
  long long need = ((long long)a.n_order + wpb - 1) / wpb;
  if (need < blocks) blocks = need > 0 ? need : 1;
  gs_sim_kernel<H><<<(unsigned)blocks, threads, dyn, st>>>(a);
  CK(cudaGetLastError());
  return GS_OK;
}

static int launch_xl(const KArgs& a, int sms, cudaStream_t st, char* err, size_t err_len) {
  CK(cudaFuncSetAttribute(gs_sim_kernel_xl, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)XLH_DYN_BYTES));
  long long blocks = sms;
  if (a.n_order < blocks) blocks = a.n_order > 0 ? a.n_order : 1;
  gs_sim_kernel_xl<<<(unsigned)blocks, XL_THREADS, (size_t)a.xl_bytes, st>>>(a);
  CK(cudaGetLastError());
  return GS_OK;
}

extern "C" int gs_session_run(gs_session_t* s, void* stream_ptr, char* err, size_t err_len) {
  if (!s) { put_err(err, err_len, "null session"); return GS_ERR_ARG; }
  CK(cudaSetDevice(s->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_ptr);
  CK(cudaMemsetAsync(s->counter, 0, 8 * sizeof(int), st));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device));
  CK(cudaEventRecord(s->ev0, st));
  s->last_launches = 0;
  for (int k = 1; k <= 5; k++) {
    const int lo = s->class_off[k - 1], hi = s->class_off[k];
    if (hi <= lo) continue;
    KArgs a;
    a.in = s->dev_in;
    a.out = s->dev_out;
    a.host = s->host_map;
    a.arena = s->arena;
    a.ws_off = s->ws_off;
    a.order = s->order + lo;
    a.n_order = hi - lo;
    a.counter = s->counter + k;
    a.xl_bytes = s->xl_bytes;
    int rc = GS_OK;
    switch (k) {
      case 1: rc = launch_class<HotXS>(s, a, sms, st, err, err_len); break;
      case 2: rc = launch_class<HotS>(s, a, sms, st, err, err_len); break;
      case 3: rc = launch_class<HotM>(s, a, sms, st, err, err_len); break;
      case 4: rc = launch_class<HotL>(s, a, sms, st, err, err_len); break;
      default: rc = launch_xl(a, sms, st, err, err_len); break;
    }
    if (rc != GS_OK) return rc;
    s->last_launches++;
  }
  CK(cudaEventRecord(s->ev1, st));
  CK(cudaEventSynchronize(s->ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
  s->last_ms = ms;
  return GS_OK;
}

// Re-upload a batch of the same shape (same runs, offsets and sizes) into the
// session's device buffers: the per-step H2D of a resident session.
extern "C" int gs_session_upload(gs_session_t* s, const gs_batch_t* in, void* stream_ptr,
                                 char* err, size_t err_len) {
  if (!s || !in) { put_err(err, err_len, "bad arguments"); return GS_ERR_ARG; }
  const gs_batch_t& d = s->dev_in;
  if (in->n_runs != d.n_runs || in->n_funcs != d.n_funcs || in->n_points != d.n_points ||
      in->n_inits != d.n_inits || in->n_counts != d.n_counts || in->n_names != d.n_names ||
      in->n_fn_rows != d.n_fn_rows || in->n_gpu_rows != d.n_gpu_rows ||
      in->n_glob_rows != d.n_glob_rows || in->n_placements != d.n_placements ||
      in->n_id_splits != d.n_id_splits) {
    put_err(err, err_len, "gs_session_upload: batch shape differs from the session's");
    return GS_ERR_ARG;
  }
  CK(cudaSetDevice(s->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_ptr);
  auto up = [&](const void* dst, const void* src, size_t n) -> cudaError_t {
    if (!src || !n) return cudaSuccess;
    return cudaMemcpyAsync(const_cast<void*>(dst), src, n, cudaMemcpyHostToDevice, st);
  };
  CK(up(d.runs, in->runs, sizeof(gs_scenario_t) * (size_t)in->n_runs));
  CK(up(d.funcs, in->funcs, sizeof(gs_function_t) * (size_t)in->n_funcs));
  CK(up(d.points, in->points, sizeof(gs_point_t) * (size_t)in->n_points));
  CK(up(d.inits, in->inits, sizeof(gs_init_t) * (size_t)in->n_inits));
  CK(up(d.counts, in->counts, sizeof(int32_t) * (size_t)in->n_counts));
  CK(up(d.names, in->names, (size_t)in->n_names));
  CK(up(d.id_splits, in->id_splits, sizeof(gs_id_split_t) * (size_t)in->n_id_splits));
  return GS_OK;
}

extern "C" int gs_session_download(gs_session_t* s, const gs_out_t* out, void* stream_ptr,
                                   char* err, size_t err_len) {
  if (!s || !out || !out->status) { put_err(err, err_len, "bad arguments"); return GS_ERR_ARG; }
  CK(cudaSetDevice(s->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_ptr);
  auto down = [&](void* dst, const void* src, size_t n, const void* mapped) -> cudaError_t {
    if (!dst || !n || dst == mapped) return cudaSuccess;   // already written by the kernel
    return cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st);
  };
  const gs_out_t& hp = s->host_ptr;
  CK(down(out->fn_rows, s->dev_out.fn_rows, sizeof(gs_fn_row_t) * (size_t)s->n_fn_rows,
          hp.fn_rows));
  CK(down(out->gpu_rows, s->dev_out.gpu_rows, sizeof(gs_gpu_row_t) * (size_t)s->n_gpu_rows,
          hp.gpu_rows));
  CK(down(out->glob_rows, s->dev_out.glob_rows, sizeof(gs_glob_row_t) * (size_t)s->n_glob_rows,
          hp.glob_rows));
  CK(down(out->placements, s->dev_out.placements, sizeof(gs_placement_t) * (size_t)s->n_place,
          hp.placements));
  CK(down(out->status, s->dev_out.status, sizeof(gs_status_t) * (size_t)s->n_runs, nullptr));
  CK(down(out->summary, s->dev_out.summary, sizeof(gs_summary_t) * (size_t)s->n_runs, nullptr));
  CK(cudaStreamSynchronize(st));
  int worst = GS_OK;
  for (int r = 0; r < s->n_runs; r++) worst = std::max(worst, (int)out->status[r].code);
  return worst;
}

// Packer audit of every run's final node geometry: breach
// bits (GS_AUDIT_*) OR-ed over the run's nodes, one uint32 per run.
extern "C" int gs_session_audit(gs_session_t* s, uint32_t* breaches, void* stream_ptr,
                                char* err, size_t err_len) {
  if (!s || !breaches) { put_err(err, err_len, "bad arguments"); return GS_ERR_ARG; }
  CK(cudaSetDevice(s->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_ptr);
  const int R = s->n_runs;
  if (R == 0) return GS_OK;
  const int blocks = (R + 3) / 4;
  gs_batch_t* d_in = nullptr;
  int4* scratch = nullptr;
  unsigned* d_out = nullptr;
  CK(cudaMalloc(&d_in, sizeof(gs_batch_t)));
  CK(cudaMalloc(&scratch, sizeof(int4) * (size_t)blocks * 4 * AUD_MAX_RECTS));
  CK(cudaMalloc(&d_out, sizeof(unsigned) * (size_t)R));
  CK(cudaMemcpyAsync(d_in, &s->dev_in, sizeof(gs_batch_t), cudaMemcpyHostToDevice, st));
  AuditArgs a{};
  a.in = d_in; a.arena = s->arena; a.ws_off = s->ws_off; a.n_runs = R;
  a.scratch = scratch; a.out = d_out;
  gs_audit_session_kernel<<<blocks, 128, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(breaches, d_out, sizeof(unsigned) * (size_t)R,
                                            cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d_in); cudaFree(scratch); cudaFree(d_out);
  CK(e);
  return GS_OK;
}

// The same auditor on caller-supplied geometry (host buffers): node k has
// n_free[k] free rects then n_placed[k] placed rects at rects[k*cap*4 ...]
// as (x, y, w, h) int32 quadruples on a side_x x side_y plane.
extern "C" int gs_audit_geometry(const int32_t* rects, const int32_t* n_free,
                                 const int32_t* n_placed, int n_nodes, int cap, int side_x,
                                 int side_y, uint32_t* breaches, int device, char* err,
                                 size_t err_len) {
  if (!rects || !n_free || !n_placed || !breaches || n_nodes < 0 || cap < 1) {
    put_err(err, err_len, "bad arguments");
    return GS_ERR_ARG;
  }
  if (n_nodes == 0) return GS_OK;
  CK(cudaSetDevice(device));
  int4* d_r = nullptr;
  int *d_f = nullptr, *d_p = nullptr;
  unsigned* d_o = nullptr;
  const size_t nr = (size_t)n_nodes * cap;
  CK(cudaMalloc(&d_r, sizeof(int4) * nr));
  CK(cudaMalloc(&d_f, sizeof(int) * (size_t)n_nodes));
  CK(cudaMalloc(&d_p, sizeof(int) * (size_t)n_nodes));
  CK(cudaMalloc(&d_o, sizeof(unsigned) * (size_t)n_nodes));
  cudaError_t e = cudaMemcpy(d_r, rects, sizeof(int4) * nr, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_f, n_free, sizeof(int) * n_nodes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_p, n_placed, sizeof(int) * n_nodes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    AuditArgs a{};
    a.rects = d_r; a.nfree = d_f; a.nplaced = d_p; a.cap = cap; a.n_nodes = n_nodes;
    a.side_x = side_x; a.side_y = side_y; a.out = d_o;
    gs_audit_geometry_kernel<<<(n_nodes + 3) / 4, 128>>>(a);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(breaches, d_o, sizeof(unsigned) * n_nodes,
                                       cudaMemcpyDeviceToHost);
  cudaFree(d_r); cudaFree(d_f); cudaFree(d_p); cudaFree(d_o);
  CK(e);
  return GS_OK;
}

extern "C" int gs_session_device_out(gs_session_t* s, gs_out_t* dev_out) {
  if (!s || !dev_out) return GS_ERR_ARG;
  *dev_out = s->dev_out;
  return GS_OK;
}

extern "C" int gs_session_last_launches(gs_session_t* s) { return s ? s->last_launches : 0; }
extern "C" double gs_session_last_kernel_ms(gs_session_t* s) { return s ? s->last_ms : 0.0; }

extern "C" void gs_session_destroy(gs_session_t* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  if (s->blob) {
    if (s->async_alloc) cudaFreeAsync(s->blob, s->ord);
    else cudaFree(s->blob);
  }
  delete s;
}

// device-visible alias of a page-locked, mapped host pointer (else NULL)
static void* mapped_alias(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
  return at.devicePointer;
}

extern "C" int gs_session_map_host(gs_session_t* s, const gs_out_t* host) {
  if (!s) return GS_ERR_ARG;
  if (cudaSetDevice(s->device) != cudaSuccess) return GS_ERR_CUDA;
  s->host_map = gs_out_t{};
  s->host_ptr = gs_out_t{};
  if (!host) return GS_OK;
#define GS_MAP(field, T)                                                       \
  if (void* d_ = mapped_alias(host->field)) {                                  \
    s->host_map.field = reinterpret_cast<T*>(d_);                              \
    s->host_ptr.field = host->field;                                           \
  }
  GS_MAP(fn_rows, gs_fn_row_t)
  GS_MAP(gpu_rows, gs_gpu_row_t)
  GS_MAP(glob_rows, gs_glob_row_t)
  GS_MAP(placements, gs_placement_t)
#undef GS_MAP
  return GS_OK;
}

extern "C" int gs_host_alloc(size_t bytes, void** ptr) {
  if (!ptr) return GS_ERR_ARG;
  *ptr = nullptr;
  if (cudaHostAlloc(ptr, bytes ? bytes : 1, cudaHostAllocPortable | cudaHostAllocMapped) !=
      cudaSuccess) {
    cudaGetLastError();
    *ptr = nullptr;
    return GS_ERR_CUDA;
  }
  return GS_OK;
}

extern "C" void gs_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}

// The one-shot call is stream-ordered end to end: allocation (cudaMallocAsync
// from the device's memory pool, which keeps its blocks between calls), input
// copies, the launches, the downloads and the free all go on one stream, and
// with stream == NULL that stream is a private non-blocking one.  Nothing in it
// synchronises the device, so concurrent one-shot calls (the drop-in API's
// pipelined batches, engine.simulate_records) overlap on the GPU.
extern "C" int gs_run_batch(const gs_batch_t* in, const gs_out_t* out, int device, void* stream,
                            char* err, size_t err_len) {
  if (!in || !out) { put_err(err, err_len, "bad arguments"); return GS_ERR_ARG; }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device) {
    put_err(err, err_len, "no CUDA device visible");
    return GS_ERR_CUDA;
  }
  CK(cudaSetDevice(device));
  static std::atomic<unsigned> pool_ready{0};      // bit per device (first 32)
  if (device < 32 && !(pool_ready.load() & (1u << device))) {
    cudaMemPool_t mp;
    if (cudaDeviceGetDefaultMemPool(&mp, device) == cudaSuccess) {
      unsigned long long keep = 32ull << 30;       // keep up to 32 GB cached between calls
      cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool_ready.fetch_or(1u << device);
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool own = st == nullptr;
  if (own) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  gs_session_t* s = nullptr;
  int rc = session_create(in, device, st, true, &s, err, err_len);
  if (rc == GS_OK) {
    gs_session_map_host(s, out);     // page-locked row buffers are written in place
    rc = gs_session_run(s, st, err, err_len);
    if (rc == GS_OK) rc = gs_session_download(s, out, st, err, err_len);
    gs_session_destroy(s);           // cudaFreeAsync on st
    cudaStreamSynchronize(st);
  }
  if (own) cudaStreamDestroy(st);
  return rc;
}
