/*
 * gshare_b200.h -- C ABI of the B200 batched FaST-GShare simulator.
 *
 * The reference (pkg/src/gshare_sim) is pure Python and has no FFI; its
 * drop-in boundary is the Python call
 *
 *     run(scenario, policy="fast") -> MetricsReport        sim_engine.py:601-603
 *     compare_policies(scenario)   -> {policy: report}     sim_engine.py:606-612
 *
 * This header is what a binding of that boundary sees: a BATCH of independent
 * (scenario, policy) runs, lowered on the host to flat structure-of-structs
 * arrays (paper_2309_00558_b200/compiler.py builds them with numpy structured
 * dtypes that mirror these structs byte for byte), and fixed-size output
 * records from which the host rebuilds the reference's MetricsReport rows
 * (metrics.py:27-60).  Plain pointers and sizes only; no torch types.
 *
 * Ownership: the caller owns every in/out buffer; nothing is retained after a
 * one-shot call returns.  Sessions own their device copies until destroyed.
 * Threading: calls are reentrant per (device, stream).  The only process
 * state is the launch-shape DEFAULTS of gs_set_launch / gs_set_xl_smem
 * (atomic; copied into a session at gs_session_create, never read by a
 * launch), so concurrent sessions keep the shape they were created with.
 *
 * Return codes (also per-run in gs_status_t.code):
 *   GS_OK (0)            success
 *   GS_ERR_VALIDATION(1) a run hit a reference ValidationError mid-run
 *                        (detail GS_VAL_*: sim_engine.py:346-349 zero serving
 *                        rate, autoscaler.py:115-117 no positive throughput)
 *   GS_ERR_CAPACITY  (3) a run outgrew a static capacity (pods, free rects,
 *                        returned requests); the host retries it with larger
 *                        capacities -- results are never silently truncated
 *   GS_ERR_INVARIANT (2) corrupt state (maps to InvariantError, cli.py:42-44)
 *   GS_ERR_CUDA      (4) CUDA runtime failure / no device
 *   GS_ERR_ARG       (5) malformed batch
 */
#ifndef GSHARE_B200_H
#define GSHARE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 2

enum {
  GS_OK = 0,
  GS_ERR_VALIDATION = 1,
  GS_ERR_INVARIANT = 2,
  GS_ERR_CAPACITY = 3,
  GS_ERR_CUDA = 4,
  GS_ERR_ARG = 5
};

/* gs_status_t.detail for GS_ERR_VALIDATION (arg0 = function, arg1 = point) */
enum { GS_VAL_ZERO_RATE = 0,      /* _make_pod: T(sm_eff, 1.0) <= 0   sim_engine.py:346-349 */
       GS_VAL_NO_THROUGHPUT = 1   /* scale_up: t_eff <= 0             autoscaler.py:115-117 */ };

/* gs_status_t.detail for GS_ERR_CAPACITY */
enum { GS_CAP_PODS = 1, GS_CAP_RECTS = 2, GS_CAP_RETURNED = 3, GS_CAP_NAMES = 4,
       GS_CAP_HOT = 5 /* per-window working set outgrew its shared-memory class */ };

/* gs_scenario_t.flags */
#define GS_FLAG_TIMESHARE   1  /* policy "timeshare": sm_eff = 100 (sim_engine.py:337-338) */
#define GS_FLAG_SHARING     2  /* model_sharing memory accounting (memory_model.py:70-73) */
#define GS_FLAG_SM_INTEGRAL 4  /* every sm_eff is an integer: SM sums are exact in any order */

/* One (scenario, policy) run.  Mirrors Scenario (sim_engine.py:118-130) after
 * _Engine.__init__ derived its constants (sim_engine.py:309-311). */
typedef struct gs_scenario {
  int32_t n_nodes;               /* fleet_size                                   */
  int32_t n_funcs;               /* functions, indexed in sorted(function_id)    */
  int32_t windows;
  int32_t steps;                 /* round(1/quantum)                             */
  int32_t epoch_windows;
  int32_t cold_start_windows;
  int32_t restructure_threshold;
  int32_t flags;                 /* GS_FLAG_*                                    */
  int32_t func_off;              /* first gs_function_t of this run              */
  int32_t side_x, side_y;        /* 100x100 plane in scaled integer units        */
  int32_t cap_pods;              /* pod slots (placed + retry + warming)         */
  int32_t cap_rects;             /* free rectangles per node                     */
  int32_t cap_returned;          /* un-pinned-by-removal requests per function   */
  int32_t hot_class;             /* 0 = auto; else minimum shared-memory size class */
  int64_t fn_row_off;            /* windows*n_funcs gs_fn_row_t                  */
  int64_t gpu_row_off;           /* windows*n_nodes gs_gpu_row_t                 */
  int64_t glob_row_off;          /* windows gs_glob_row_t                        */
  int64_t place_off;             /* cap_pods gs_placement_t                      */
  double window_s;               /* window_ms / 1000.0                           */
  double quantum_s;              /* window_s * quantum                           */
  double quantum;                /* token length, window fraction                */
  double capacity_mb;            /* gpu_capacity_mb                              */
} gs_scenario_t;

/* One function of a run (FunctionSpec + FunctionProfile, sim_engine.py:106-115). */
typedef struct gs_function {
  int32_t n_points, point_off;   /* profile points, sorted by (sm, quota)        */
  int32_t n_init, init_off;      /* initial pods in spec order                   */
  int32_t count_off;             /* counts[windows], zero padded past the trace  */
  int32_t max_queue;             /* -1 = unbounded                               */
  int32_t p_eff;                 /* most_efficient_point index (autoscaler.py:98)*/
  int32_t id_rank;               /* rank of fid+"-" : pod-id string order        */
  int32_t name_off, name_len;    /* UTF-8 function id in gs_batch_t.names        */
  int32_t n_id_splits;           /* pod-id order segments beyond the first       */
  int32_t id_split_off;          /* first gs_id_split_t of this function         */
  double slo_ms;
  double mem_server_mb, mem_runtime_mb, mem_noshare_mb;
} gs_function_t;

/* One profiled operating point (profiles.py:48-75 + policy-applied pod shape). */
typedef struct gs_point {
  double sm, quota;              /* profiled point                               */
  double thr;                    /* throughput_at(point)                         */
  double area;                   /* (sm/100.0)*quota                             */
  double rpr;                    /* thr/area                                     */
  double sm_eff;                 /* 100.0 under timeshare, else sm               */
  double inv_rate;               /* 1.0/T(sm_eff,1.0); 0 if that rate <= 0       */
  int32_t rect_w, rect_h;        /* as_frac(quota)*100, as_frac(sm_eff), scaled  */
  int32_t rate_ok, pad;          /* T(sm_eff,1.0) > 0                            */
} gs_point_t;

/* Pod-id string order (pod ids are f"{fid}-{counter:04d}", sim_engine.py:354;
 * many tie-breaks compare them as strings).  A pod's 64-bit order key is
 * slot * 11^10 + digits_key(counter), digits_key = the counter's decimal text
 * in base 11 (0 = end of text), so keys compare exactly as the strings do.
 * slot = id_rank unless the function id is extended by other ids with "-"
 * (e.g. "x" and "x-1"): then the pods of "x" interleave with the pods of the
 * extending ids at thresholds of the counter text, and slot = the slot of the
 * last split whose threshold is below digits_key(counter). */
typedef struct gs_id_split {
  uint64_t threshold;            /* digits_key space                             */
  int32_t slot;
  int32_t pad;
} gs_id_split_t;

typedef struct gs_init {
  int32_t point;                 /* index into the function's points             */
  int32_t has_q_req;             /* InitialPod.quota_request is not None         */
  double q_req;
} gs_init_t;

typedef struct gs_batch {
  int32_t n_runs;
  int32_t n_funcs, n_points, n_inits;
  int64_t n_counts, n_names;
  int64_t n_fn_rows, n_gpu_rows, n_glob_rows, n_placements;
  int64_t n_id_splits;
  const gs_scenario_t* runs;
  const gs_function_t* funcs;
  const gs_point_t* points;
  const gs_init_t* inits;
  const int32_t* counts;
  const char* names;
  const gs_id_split_t* id_splits;  /* may be NULL when n_id_splits == 0          */
} gs_batch_t;

/* ---- outputs (metrics.py:27-52) ---------------------------------------- */
typedef struct gs_fn_row {
  int32_t arrivals, completions, slo_violations, dropped, queue_depth;
} gs_fn_row_t;

typedef struct gs_gpu_row {
  double utilization, sm_occupancy, memory_mb;
  int32_t present;               /* node had placements (sim_engine.py:571)      */
  int32_t pad;
} gs_gpu_row_t;

typedef struct gs_glob_row {
  int32_t gpus_in_use, placement_failures;
  double fragmentation_index;
} gs_glob_row_t;

/* Final packer state, so tests can inspect _Engine.nodes[i].placements. */
typedef struct gs_placement {
  int32_t node, func, counter;   /* pod id = names[func] + "-%04d" % counter    */
  int32_t x, y, w, h;            /* scaled rectangle                             */
  int32_t pad;
} gs_placement_t;

typedef struct gs_status {
  int32_t code, detail, arg0, arg1;
  int32_t n_placements;
  int32_t hot_class;             /* size class the run executed in (1=XS .. 5=XL) */
  int64_t token_grants;          /* dispatch() outputs, token_backend.py:186     */
  int64_t scale_decisions;       /* len(scale_up)+len(scale_down)                */
  int64_t placement_attempts;    /* best_match calls, sim_engine.py:397          */
  int64_t pod_steps;             /* sum over quantum steps of registered pods    */
  int64_t rect_scans;            /* free rects examined by best_match            */
  int64_t peak_pods;             /* most pods alive at once (capacity sizing)    */
} gs_status_t;

/* Fixed-size per-run record all-gathered across GPUs (metrics.py:94-131). */
typedef struct gs_summary {
  int32_t windows, gpus_used_peak, placement_failures, n_gpu_rows;
  int64_t arrivals, completions, slo_violations, dropped, final_queue_depth;
  double sum_utilization, sum_sm_occupancy;   /* sequential, row order */
} gs_summary_t;

typedef struct gs_out {
  gs_fn_row_t* fn_rows;          /* any row pointer may be NULL: not written     */
  gs_gpu_row_t* gpu_rows;
  gs_glob_row_t* glob_rows;
  gs_placement_t* placements;
  gs_status_t* status;           /* required                                     */
  gs_summary_t* summary;
} gs_out_t;

typedef struct gs_session gs_session_t;

int gs_abi_version(void);

/* One-shot: host in -> H2D -> simulate -> D2H -> host out.  `stream` may be
 * NULL (a private non-blocking stream is used).  Stream-ordered: device memory
 * comes from the device's default memory pool (cudaMallocAsync; the pool keeps
 * up to 32 GB cached between calls), so concurrent calls from several host
 * threads overlap on the GPU.  Returns the worst per-run code. */
int gs_run_batch(const gs_batch_t* in, const gs_out_t* out, int device, void* stream,
                 char* err, size_t err_len);

/* Sessions keep inputs, workspace and outputs resident in HBM. */
int gs_session_create(const gs_batch_t* in, int device, gs_session_t** sess,
                      char* err, size_t err_len);
int gs_session_run(gs_session_t* sess, void* stream, char* err, size_t err_len);
/* Re-upload inputs of the same batch shape (per-step H2D of a resident session;
 * ordered on `stream` before the next gs_session_run on it). */
int gs_session_upload(gs_session_t* sess, const gs_batch_t* in, void* stream,
                      char* err, size_t err_len);
int gs_session_download(gs_session_t* sess, const gs_out_t* out, void* stream,
                        char* err, size_t err_len);
/* Zero-copy outputs: row buffers of `host` that are page-locked and mapped
 * (gs_host_alloc / cudaHostAlloc) are filled by the kernel itself -- each run
 * copies its rows out when it finishes, overlapping the other runs -- and
 * gs_session_download skips them.  Other pointers are ignored (copied by
 * download as usual).  gs_run_batch does this automatically. */
int gs_session_map_host(gs_session_t* sess, const gs_out_t* host);
/* Page-locked, device-mapped host memory for batch inputs and outputs. */
int gs_host_alloc(size_t bytes, void** ptr);
void gs_host_free(void* ptr);
/* Device pointers of the session's outputs (for device-side collectives). */
int gs_session_device_out(gs_session_t* sess, gs_out_t* dev_out);
/* Kernel launches issued by the last gs_session_run / its device time (ms). */
int gs_session_last_launches(gs_session_t* sess);
double gs_session_last_kernel_ms(gs_session_t* sess);
void gs_session_destroy(gs_session_t* sess);

/* Packer auditor (the reference's check_node, packer.py:327-388, decided
 * exactly on the scaled integer grid compressed to the rectangle edges): per
 * run, the OR over its nodes of GS_AUDIT_* bits for the final geometry. */
#define GS_AUDIT_PLACED_OVERLAP 1u   /* two placements intersect            */
#define GS_AUDIT_FREE_PLACED    2u   /* a free rect intersects a placement  */
#define GS_AUDIT_FREE_CONTAINED 4u   /* a free rect inside another          */
#define GS_AUDIT_GAP            8u   /* area neither free nor placed        */
#define GS_AUDIT_DOUBLE        16u   /* area both free and placed           */
#define GS_AUDIT_TOO_BIG       32u   /* > 256 rects on a node: not audited  */
int gs_session_audit(gs_session_t* sess, uint32_t* breaches /* [n_runs] */, void* stream,
                     char* err, size_t err_len);
/* The same audit on caller geometry: node k holds n_free[k] free then
 * n_placed[k] placed (x, y, w, h) int32 rects at rects[4*cap*k ...]. */
int gs_audit_geometry(const int32_t* rects, const int32_t* n_free, const int32_t* n_placed,
                      int n_nodes, int cap, int side_x, int side_y, uint32_t* breaches,
                      int device, char* err, size_t err_len);

/* Launch-shape default for sessions created afterwards (0 = built-in
 * default).  warps_per_block: scenario warps per CTA. */
int gs_set_launch(int warps_per_block, int blocks_per_sm);

/* XL class (one CTA per run): dynamic shared memory for the run's working set
 * (0 = default 224 KB; clamped to [16 KB, 224 KB]).  Smaller values force the
 * arena-stepping and warp-0 fallbacks -- a test / debugging knob; returns the
 * value in effect. */
int gs_set_xl_smem(int bytes);

/* ---- host-side report rendering ---------------------
 * metrics.csv of device rows, byte-identical to the reference's
 * MetricsReport.to_csv() (metrics.py:62-91, numbers as util.py:4-10 fmt_num
 * of round(x, 9) / round(x, 6)).  `fid_csv` holds, for every gs_function_t of
 * the batch in batch order, the function id as csv.writer renders it (UTF-8,
 * QUOTE_MINIMAL), function k at [fid_off[k], fid_off[k+1]).  No GPU needed. */
/* Run `run` into buf.  Returns the text length, or -- when buf is NULL or cap
 * is below the run's size bound -- the bound to allocate; -1 on bad args. */
int64_t gs_format_csv(const gs_batch_t* in, const gs_out_t* out, int run,
                      const char* fid_csv, const int64_t* fid_off, char* buf, int64_t cap);
/* Runs [r0, r1) on n_threads host threads (0 = all): run r0+k at
 * buf + offs[k], length lens[k].  Returns 0, or the bytes needed when buf is
 * NULL / cap is too small, -1 on bad args. */
int64_t gs_format_csv_batch(const gs_batch_t* in, const gs_out_t* out, int r0, int r1,
                            const char* fid_csv, const int64_t* fid_off, char* buf,
                            int64_t cap, int64_t* offs, int64_t* lens, int n_threads);
/* summary() inputs of runs [r0, r1): per function (batch order from the
 * first run's func_off) arrivals, completions, slo_violations, dropped summed
 * over the windows, and the final queue depth -- 5 int64 per function. */
int gs_fn_totals(const gs_batch_t* in, const gs_out_t* out, int r0, int r1, int64_t* totals,
                 int n_threads);
/* fmt_num(round(x[k], nd)) (nd < 0: fmt_num(x[k])) as NUL-terminated text
 * at buf + k*stride (stride >= 48). */
int gs_format_numbers(const double* x, int64_t n, int nd, char* buf, int64_t stride);

#ifdef __cplusplus
}
#endif
#endif /* GSHARE_B200_H */
