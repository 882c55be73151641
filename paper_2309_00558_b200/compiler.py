"""Scenario compiler: (Scenario, policy) -> flat device-ready arrays.

This is the host half of the boundary.  It performs every precondition check
the reference performs before its first window (sim_engine.py:132-170,
_Engine.__init__ :303-333, the initial ``_make_pod`` calls :437-440 with their
ResourceConfig / serving-rate checks) so errors surface as the same
``ValidationError`` with the same text, then lowers the run to the structs of
include/gshare_b200.h:

* profile points sorted by (sm, quota) with T, area, rpr, 1/rate precomputed
  by the *same Python float expressions* the reference evaluates
  (profiles.py:70-75,183; sim_engine.py:340-350,535), so the device reads
  bit-identical doubles;
* ``most_efficient_point`` per function (autoscaler.py:91-100), a static
  property of the profile;
* pod rectangles as integers: the packer's exact rationals
  (packer.py:39-53,129-133) are scaled by the lcm of their denominators so
  every coordinate, area and comparison is exact int64 arithmetic;
* a pod-id order rank per function: pod ids are ``f"{fid}-{n:04d}"``
  (sim_engine.py:354) and string order decides many tie-breaks; ranking
  ``fid + "-"`` reproduces string order whenever no function id extends
  another id followed by ``-`` (validated here).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache, reduce

import numpy as np

from .errors import ValidationError
from .scenario import POLICIES, steps_per_window, validate_scenario

# ---------------------------------------------------------------------------
# numpy mirrors of the C structs (aligned=True == natural C layout)
# ---------------------------------------------------------------------------
GS_FLAG_TIMESHARE = 1
GS_FLAG_SHARING = 2
GS_FLAG_SM_INTEGRAL = 4

GS_OK, GS_ERR_VALIDATION, GS_ERR_INVARIANT, GS_ERR_CAPACITY, GS_ERR_CUDA, GS_ERR_ARG = range(6)
GS_CAP_PODS, GS_CAP_RECTS, GS_CAP_RETURNED, GS_CAP_NAMES, GS_CAP_HOT = 1, 2, 3, 4, 5
GS_VAL_ZERO_RATE, GS_VAL_NO_THROUGHPUT = 0, 1

SCENARIO_DT = np.dtype([
    ("n_nodes", "<i4"), ("n_funcs", "<i4"), ("windows", "<i4"), ("steps", "<i4"),
    ("epoch_windows", "<i4"), ("cold_start_windows", "<i4"),
    ("restructure_threshold", "<i4"), ("flags", "<i4"), ("func_off", "<i4"),
    ("side_x", "<i4"), ("side_y", "<i4"), ("cap_pods", "<i4"), ("cap_rects", "<i4"),
    ("cap_returned", "<i4"), ("hot_class", "<i4"),
    ("fn_row_off", "<i8"), ("gpu_row_off", "<i8"), ("glob_row_off", "<i8"),
    ("place_off", "<i8"),
    ("window_s", "<f8"), ("quantum_s", "<f8"), ("quantum", "<f8"), ("capacity_mb", "<f8"),
], align=True)

FUNCTION_DT = np.dtype([
    ("n_points", "<i4"), ("point_off", "<i4"), ("n_init", "<i4"), ("init_off", "<i4"),
    ("count_off", "<i4"), ("max_queue", "<i4"), ("p_eff", "<i4"), ("id_rank", "<i4"),
    ("name_off", "<i4"), ("name_len", "<i4"),
    ("slo_ms", "<f8"), ("mem_server_mb", "<f8"), ("mem_runtime_mb", "<f8"),
    ("mem_noshare_mb", "<f8"),
], align=True)

POINT_DT = np.dtype([
    ("sm", "<f8"), ("quota", "<f8"), ("thr", "<f8"), ("area", "<f8"), ("rpr", "<f8"),
    ("sm_eff", "<f8"), ("inv_rate", "<f8"), ("rect_w", "<i4"), ("rect_h", "<i4"),
    ("rate_ok", "<i4"), ("pad", "<i4"),
], align=True)

INIT_DT = np.dtype([("point", "<i4"), ("has_q_req", "<i4"), ("q_req", "<f8")], align=True)

FN_ROW_DT = np.dtype([("arrivals", "<i4"), ("completions", "<i4"),
                      ("slo_violations", "<i4"), ("dropped", "<i4"),
                      ("queue_depth", "<i4")], align=True)
GPU_ROW_DT = np.dtype([("utilization", "<f8"), ("sm_occupancy", "<f8"),
                       ("memory_mb", "<f8"), ("present", "<i4"), ("pad", "<i4")],
                      align=True)
GLOB_ROW_DT = np.dtype([("gpus_in_use", "<i4"), ("placement_failures", "<i4"),
                        ("fragmentation_index", "<f8")], align=True)
PLACEMENT_DT = np.dtype([("node", "<i4"), ("func", "<i4"), ("counter", "<i4"),
                         ("x", "<i4"), ("y", "<i4"), ("w", "<i4"), ("h", "<i4"),
                         ("pad", "<i4")], align=True)
STATUS_DT = np.dtype([("code", "<i4"), ("detail", "<i4"), ("arg0", "<i4"), ("arg1", "<i4"),
                      ("n_placements", "<i4"), ("hot_class", "<i4"),
                      ("token_grants", "<i8"), ("scale_decisions", "<i8"),
                      ("placement_attempts", "<i8"), ("pod_steps", "<i8"),
                      ("rect_scans", "<i8"), ("peak_pods", "<i8")], align=True)
SUMMARY_DT = np.dtype([("windows", "<i4"), ("gpus_used_peak", "<i4"),
                       ("placement_failures", "<i4"), ("n_gpu_rows", "<i4"),
                       ("arrivals", "<i8"), ("completions", "<i8"),
                       ("slo_violations", "<i8"), ("dropped", "<i8"),
                       ("final_queue_depth", "<i8"),
                       ("sum_utilization", "<f8"), ("sum_sm_occupancy", "<f8")], align=True)

STRUCT_SIZES = {  # checked against sizeof() of the C structs by the tests
    "gs_scenario_t": SCENARIO_DT.itemsize, "gs_function_t": FUNCTION_DT.itemsize,
    "gs_point_t": POINT_DT.itemsize, "gs_init_t": INIT_DT.itemsize,
    "gs_fn_row_t": FN_ROW_DT.itemsize, "gs_gpu_row_t": GPU_ROW_DT.itemsize,
    "gs_glob_row_t": GLOB_ROW_DT.itemsize, "gs_placement_t": PLACEMENT_DT.itemsize,
    "gs_status_t": STATUS_DT.itemsize, "gs_summary_t": SUMMARY_DT.itemsize,
}

# exactness limits of the device geometry
_MAX_SIDE = 1 << 28
_FRAG_LIMIT = 1 << 53
_MAX_RECTS_CAP = 4096


@dataclass(frozen=True)
class Caps:
    pods: int
    rects: int
    returned: int
    hot_class: int = 0        # 0 = smallest shared-memory class that fits F and G

    def grown(self, detail: int, hot_class_used: int = 0) -> "Caps":
        if detail == GS_CAP_PODS:
            return Caps(self.pods * 4, self.rects, self.returned, self.hot_class)
        if detail == GS_CAP_RECTS:
            return Caps(self.pods, min(self.rects * 4, _MAX_RECTS_CAP), self.returned,
                        self.hot_class)
        if detail == GS_CAP_HOT:
            return Caps(self.pods, self.rects, self.returned, max(self.hot_class, hot_class_used) + 1)
        return Caps(self.pods, self.rects, self.returned * 4, self.hot_class)


@lru_cache(maxsize=65536)
def as_frac(value) -> Fraction:
    """The reference's coordinate snapping (packer.py:39-53)."""
    if isinstance(value, Fraction):
        return value
    if isinstance(value, int):
        return Fraction(value)
    if not math.isfinite(value):
        raise ValidationError(f"coordinate must be finite, got {value!r}")
    return Fraction(value).limit_denominator(10 ** 6)


def _lcm(a: int, b: int) -> int:
    return a * b // math.gcd(a, b)


def _ordered_functions(scenario):
    fns = {fn.function_id: fn for fn in scenario.functions}
    return [fns[fid] for fid in sorted(fns)]


def _check_pod_id_order(fids) -> dict:
    """Rank of each fid such that pod-id string order == (rank, counter digits)."""
    keyed = sorted(fids, key=lambda f: f + "-")
    for a in fids:
        for b in fids:
            if a != b and b.startswith(a + "-"):
                raise ValidationError(
                    f"function ids {a!r} and {b!r}: an id that extends another id "
                    f"with '-' makes pod-id order counter dependent; not supported "
                    f"by the CUDA backend")
    return {f: i for i, f in enumerate(keyed)}


def _digits_key(counter: int) -> int:
    """Order-preserving integer for the text of f"{counter:04d}" (host twin of
    the device's ``digits_key``)."""
    s = "%04d" % counter
    key = 0
    for i in range(10):
        key = key * 11 + ((ord(s[i]) - 47) if i < len(s) else 0)
    return key


def _resource_config_check(sm, q_req, q_lim):
    """ResourceConfig.__post_init__ (token_backend.py:38-49), same messages."""
    if not (math.isfinite(sm) and 0 < sm <= 100.0):
        raise ValidationError(f"sm_partition must be in (0, 100], got {sm!r}")
    for name, v in (("quota_request", q_req), ("quota_limit", q_lim)):
        if not (math.isfinite(v) and 0 < v <= 1):
            raise ValidationError(f"{name} must be in (0, 1], got {v!r}")
    if q_req > q_lim + 1e-9:
        raise ValidationError(f"quota_request {q_req!r} exceeds quota_limit {q_lim!r}")


def _profile_memo(profile, memo: dict | None) -> dict:
    """Compile-time derived data of one profile object, cached for the
    duration of ONE compile call (``memo`` is created per call): profiles are
    mutable dataclasses and the reference re-reads ``entries`` on every run,
    so nothing derived from a profile object may outlive the call."""
    if memo is None:
        return {}
    key = id(profile)
    hit = memo.get(key)
    if hit is None or hit[0] is not profile:
        hit = memo[key] = (profile, {})
    return hit[1]


def _t_eff(lo: "_LoweredProfile") -> float:
    """Throughput of most_efficient_point (autoscaler.py:98-100)."""
    return float(lo.rows["thr"][lo.p_eff])


def _default_caps(scenario, fns, lowered) -> Caps:
    """Static device capacities, sized from the trace peaks so that overflow
    (a device rerun with larger capacities) stays rare: pods for the whole
    fleet, and returned requests per function -- a scale-down can hand back
    one in-flight request per removed pod of the function."""
    window_s = scenario.window_ms / 1000.0
    pods = 8
    per_fn = 0
    for fn, lo in zip(fns, lowered):
        t_eff = _t_eff(lo)
        counts = fn.trace.counts[:scenario.windows]
        peak = max(counts, default=0) / window_s
        # t_eff <= 0: the first scale-up raises (autoscaler.py:115-117), so
        # the function never adds pods beyond its initial ones
        grow = int(math.ceil(1.5 * peak / t_eff)) if t_eff > 0 else 0
        k = len(fn.initial_pods) + grow + 4
        pods += k
        per_fn = max(per_fn, k)
    pods = min(max(32, -(-pods // 32) * 32), 1 << 20)
    returned = min(max(32, -(-per_fn // 32) * 32), 4096)
    return Caps(pods=pods, rects=64, returned=returned)


@dataclass(frozen=True)
class _LoweredProfile:
    keys: list            # [(sm, quota)] sorted
    index: dict
    rows: np.ndarray      # POINT_DT without rect_w/rect_h
    w_num: tuple
    w_den: tuple
    h_num: tuple
    h_den: tuple
    p_eff: int
    sm_integral: bool
    lx: int                 # lcm of the width / height denominators
    ly: int


_LOWER_CACHE: dict = {}


def _lower_profile(profile, timeshare: bool, memo: dict | None = None) -> _LoweredProfile:
    """Policy-specific dense point table of one profile (cached per compile
    call by object, then by content: sweeps reuse a handful of profiles across
    thousands of scenarios)."""
    memo = _profile_memo(profile, memo)
    hit = memo.get(("lower", timeshare))
    if hit is not None:
        return hit
    lo = _lower_profile_content(profile, timeshare)
    memo[("lower", timeshare)] = lo
    return lo


def _lower_profile_content(profile, timeshare: bool) -> _LoweredProfile:
    pts = sorted(profile.entries)
    ckey = (timeshare, tuple((p.sm_partition, p.quota, profile.entries[p].throughput_rps)
                             for p in pts))
    hit = _LOWER_CACHE.get(ckey)
    if hit is not None:
        return hit
    tab = {(p.sm_partition, p.quota): e.throughput_rps for p, e in profile.entries.items()}
    keys = [(p.sm_partition, p.quota) for p in pts]
    rows = np.zeros(len(pts), POINT_DT)
    w_num, w_den, h_num, h_den = [], [], [], []
    best = None
    integral = True
    for i, p in enumerate(pts):
        thr = profile.entries[p].throughput_rps
        area = p.resource_area
        rpr = thr / area
        sm_eff = 100.0 if timeshare else p.sm_partition
        rate = tab[(sm_eff, 1.0)]
        w = as_frac(p.quota) * 100
        h = as_frac(sm_eff)
        w_num.append(w.numerator); w_den.append(w.denominator)
        h_num.append(h.numerator); h_den.append(h.denominator)
        if float(sm_eff) != math.floor(float(sm_eff)):
            integral = False
        rows[i] = (float(p.sm_partition), float(p.quota), float(thr), area, rpr, float(sm_eff),
                   (1.0 / rate) if rate > 0 else 0.0, 0, 0, 1 if rate > 0 else 0, 0)
        key = (-rpr, area, p.sm_partition, p.quota)       # autoscaler.py:94-95
        if best is None or key < best[0]:
            best = (key, i)
    lo = _LoweredProfile(keys, {k: i for i, k in enumerate(keys)}, rows, tuple(w_num),
                         tuple(w_den), tuple(h_num), tuple(h_den), best[1], integral,
                         reduce(_lcm, w_den, 1), reduce(_lcm, h_den, 1))
    if len(_LOWER_CACHE) > 4096:
        _LOWER_CACHE.clear()
    _LOWER_CACHE[ckey] = lo
    return lo


@dataclass
class RunImage:
    """One compiled (scenario, policy) run, before batching."""

    policy: str
    fids: list
    scen: np.ndarray
    funcs: np.ndarray
    points: np.ndarray
    inits: np.ndarray
    counts: np.ndarray
    names: bytes
    scale_x: int
    scale_y: int
    point_keys: list          # per function: [(sm, quota)] in point order


def compile_run(scenario, policy: str = "fast", caps: Caps | None = None,
                memo: dict | None = None) -> RunImage:
    """Lower one (scenario, policy) run.  ``memo``: a dict shared by the runs of
    ONE batch compile (per-profile-object cache; never reuse it across calls)."""
    if policy not in POLICIES:
        raise ValidationError(f"policy must be one of {POLICIES}, got {policy!r}")
    validate_scenario(scenario)
    fns = _ordered_functions(scenario)
    fids = [fn.function_id for fn in fns]
    timeshare = policy == "timeshare"
    tables = []
    for fn in fns:
        tables.append({(p.sm_partition, p.quota): e for p, e in fn.profile.entries.items()})
    if timeshare:
        for fid, tab in zip(fids, tables):
            if (100.0, 1.0) not in tab:
                raise ValidationError(
                    f"{fid}: timeshare policy needs the (100, 1.0) profile point")

    # initial pods, in the order run() creates them (sorted fid, spec order)
    for fn, tab in zip(fns, tables):
        for init in fn.initial_pods:
            p = init.point
            sm_eff = 100.0 if timeshare else p.sm_partition
            q_req = p.quota if init.quota_request is None else init.quota_request
            _resource_config_check(sm_eff, q_req, p.quota)
            rate = tab[(sm_eff, 1.0)].throughput_rps
            if rate <= 0:
                raise ValidationError(
                    f"{fn.function_id}: zero serving rate at ({sm_eff:g}, 1.0)")

    rank = _check_pod_id_order(fids)
    lowered = [_lower_profile(fn.profile, timeshare, memo) for fn in fns]
    caps = caps or _default_caps(scenario, fns, lowered)

    # geometry scale: every as_frac(quota)*100 / as_frac(sm_eff) becomes integral
    lx = reduce(_lcm, (lo.lx for lo in lowered), 1)
    ly = reduce(_lcm, (lo.ly for lo in lowered), 1)
    side_x, side_y = 100 * lx, 100 * ly
    n_nodes = int(scenario.fleet_size)
    if (side_x > _MAX_SIDE or side_y > _MAX_SIDE
            or n_nodes * _MAX_RECTS_CAP * side_x * side_y >= _FRAG_LIMIT):
        raise ValidationError(
            f"profile grid needs a {side_x}x{side_y} exact raster; too fine for the "
            f"CUDA backend's int64 geometry")

    windows = int(scenario.windows)
    n_f = len(fns)
    funcs = np.zeros(n_f, FUNCTION_DT)
    point_blocks, init_rows, point_keys = [], [], []
    n_points = 0
    counts = np.zeros(n_f * windows, np.int32)
    names = b""
    sm_integral = all(lo.sm_integral for lo in lowered)
    for fi, (fn, lo) in enumerate(zip(fns, lowered)):
        block = lo.rows.copy()
        block["rect_w"] = [n * (lx // d) for n, d in zip(lo.w_num, lo.w_den)]
        block["rect_h"] = [n * (ly // d) for n, d in zip(lo.h_num, lo.h_den)]
        point_blocks.append(block)
        point_keys.append(lo.keys)
        for init in fn.initial_pods:
            k = (init.point.sm_partition, init.point.quota)
            has = init.quota_request is not None
            init_rows.append((lo.index[k], 1 if has else 0,
                              float(init.quota_request) if has else 0.0))
        trace = list(fn.trace.counts[:windows])
        counts[fi * windows: fi * windows + len(trace)] = trace
        raw = fn.function_id.encode("utf-8")
        f = funcs[fi]
        f["n_points"] = len(lo.keys)
        f["point_off"] = n_points
        n_points += len(lo.keys)
        f["n_init"] = len(fn.initial_pods)
        f["init_off"] = len(init_rows) - len(fn.initial_pods)
        f["count_off"] = fi * windows
        # None = unbounded (-1 on the device).  A negative limit makes the
        # reference's `len(fn.queue) >= limit` (sim_engine.py:476) always true,
        # exactly like 0: every arrival is dropped.
        f["max_queue"] = -1 if fn.max_queue is None else max(0, int(fn.max_queue))
        f["p_eff"] = lo.p_eff
        f["id_rank"] = rank[fn.function_id]
        f["name_off"] = len(names)
        f["name_len"] = len(raw)
        f["slo_ms"] = fn.profile.slo_latency_ms
        mem = fn.profile.mem
        f["mem_server_mb"] = mem.mem_server_mb
        f["mem_runtime_mb"] = mem.mem_runtime_mb
        f["mem_noshare_mb"] = mem.mem_noshare_mb
        names += raw

    scen = np.zeros(1, SCENARIO_DT)
    s = scen[0]
    window_s = scenario.window_ms / 1000.0
    s["n_nodes"] = n_nodes
    s["n_funcs"] = n_f
    s["windows"] = windows
    s["steps"] = steps_per_window(scenario.quantum)
    s["epoch_windows"] = scenario.epoch_windows
    s["cold_start_windows"] = scenario.cold_start_windows
    s["restructure_threshold"] = scenario.restructure_threshold
    s["flags"] = ((GS_FLAG_TIMESHARE if timeshare else 0)
                  | (GS_FLAG_SHARING if scenario.model_sharing else 0)
                  | (GS_FLAG_SM_INTEGRAL if sm_integral else 0))
    s["side_x"], s["side_y"] = side_x, side_y
    s["cap_pods"], s["cap_rects"], s["cap_returned"] = caps.pods, caps.rects, caps.returned
    s["hot_class"] = caps.hot_class
    s["window_s"] = window_s
    s["quantum_s"] = window_s * scenario.quantum
    s["quantum"] = scenario.quantum
    s["capacity_mb"] = scenario.gpu_capacity_mb
    points = np.concatenate(point_blocks) if point_blocks else np.zeros(0, POINT_DT)
    return RunImage(policy, fids, scen, funcs, points,
                    np.array(init_rows, INIT_DT), counts, names, lx, ly, point_keys)


class Batch:
    """Concatenated RunImages + the ctypes ``gs_batch_t`` pointing at them."""

    def __init__(self, images: list):
        self.images = images
        n = len(images)
        self.runs = np.zeros(n, SCENARIO_DT)
        f_off = p_off = i_off = c_off = n_off = 0
        fn_rows = gpu_rows = glob_rows = places = 0
        funcs, points, inits, counts, names = [], [], [], [], []
        for r, im in enumerate(images):
            s = im.scen.copy()
            s["func_off"] = f_off
            s["fn_row_off"] = fn_rows
            s["gpu_row_off"] = gpu_rows
            s["glob_row_off"] = glob_rows
            s["place_off"] = places
            W = int(s["windows"][0])
            fn_rows += W * int(s["n_funcs"][0])
            gpu_rows += W * int(s["n_nodes"][0])
            glob_rows += W
            places += int(s["cap_pods"][0])
            self.runs[r] = s[0]
            fc = im.funcs.copy()
            fc["point_off"] += p_off
            fc["init_off"] += i_off
            fc["count_off"] += c_off
            fc["name_off"] += n_off
            funcs.append(fc)
            points.append(im.points)
            inits.append(im.inits)
            counts.append(im.counts)
            names.append(im.names)
            f_off += len(fc)
            p_off += len(im.points)
            i_off += len(im.inits)
            c_off += len(im.counts)
            n_off += len(im.names)
        self.funcs = np.concatenate(funcs) if funcs else np.zeros(0, FUNCTION_DT)
        self.points = np.concatenate(points) if points else np.zeros(0, POINT_DT)
        self.inits = (np.concatenate(inits) if inits else np.zeros(0, INIT_DT)).astype(INIT_DT)
        self.counts = np.ascontiguousarray(np.concatenate(counts) if counts
                                           else np.zeros(0, np.int32), np.int32)
        self.names = np.frombuffer(b"".join(names) + b"\0", np.uint8).copy()
        self.n_fn_rows, self.n_gpu_rows = fn_rows, gpu_rows
        self.n_glob_rows, self.n_placements = glob_rows, places
        # keep at least one element so every pointer is valid
        if len(self.inits) == 0:
            self.inits = np.zeros(1, INIT_DT)
        self.n_inits = sum(len(im.inits) for im in images)

    def __len__(self):
        return len(self.images)

    def alloc_outputs(self, rows: bool = True, pinned: bool = False):
        """Output arrays.  ``pinned=True`` places the row arrays in page-locked,
        device-mapped host memory, which the kernel fills in place (zero-copy,
        overlapped with the simulation); the contents start uninitialised."""
        if pinned:
            from .backend import host_empty as alloc
        else:
            def alloc(n, dt):
                return np.zeros(max(n, 1), dt)
        return {
            "fn_rows": alloc(self.n_fn_rows, FN_ROW_DT) if rows else None,
            "gpu_rows": alloc(self.n_gpu_rows, GPU_ROW_DT) if rows else None,
            "glob_rows": alloc(self.n_glob_rows, GLOB_ROW_DT) if rows else None,
            "placements": alloc(self.n_placements, PLACEMENT_DT) if rows else None,
            "status": np.zeros(len(self), STATUS_DT),
            "summary": np.zeros(len(self), SUMMARY_DT),
        }

    def pin(self) -> "Batch":
        """Move the input arrays to page-locked host memory (fast H2D)."""
        from .backend import host_empty
        for name in ("runs", "funcs", "points", "inits", "counts", "names"):
            a = getattr(self, name)
            p = host_empty(len(a), a.dtype)
            p[:len(a)] = a
            setattr(self, name, p[:len(a)] if len(a) else p)
        return self

    def input_bytes(self) -> int:
        return sum(a.nbytes for a in (self.runs, self.funcs, self.points, self.inits,
                                      self.counts, self.names))
