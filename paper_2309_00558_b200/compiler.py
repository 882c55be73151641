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
* a pod-id order per function: pod ids are ``f"{fid}-{n:04d}"``
  (sim_engine.py:354) and string order decides many tie-breaks; each pod's
  64-bit key is (slot, counter text), with the slots handed out over the
  prefix forest of the ``fid + "-"`` strings so that ids extending other ids
  ("x" and "x-1") interleave exactly as the strings do (``_pod_id_order``).
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
    ("name_off", "<i4"), ("name_len", "<i4"), ("n_id_splits", "<i4"), ("id_split_off", "<i4"),
    ("slo_ms", "<f8"), ("mem_server_mb", "<f8"), ("mem_runtime_mb", "<f8"),
    ("mem_noshare_mb", "<f8"),
], align=True)

POINT_DT = np.dtype([
    ("sm", "<f8"), ("quota", "<f8"), ("thr", "<f8"), ("area", "<f8"), ("rpr", "<f8"),
    ("sm_eff", "<f8"), ("inv_rate", "<f8"), ("rect_w", "<i4"), ("rect_h", "<i4"),
    ("rate_ok", "<i4"), ("pad", "<i4"),
], align=True)

ID_SPLIT_DT = np.dtype([("threshold", "<u8"), ("slot", "<i4"), ("pad", "<i4")], align=True)

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
    "gs_id_split_t": ID_SPLIT_DT.itemsize,
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


def _digits_key_text(text: str) -> int:
    """Order-preserving integer of a digit string of <= 10 characters: base 11,
    digit d -> d + 1, 0 = end of text (so a prefix sorts first) -- the host
    twin of the device's ``digits_key``."""
    key = 0
    for i in range(10):
        key = key * 11 + ((ord(text[i]) - 47) if i < len(text) else 0)
    return key


def _digits_key(counter: int) -> int:
    return _digits_key_text("%04d" % counter)


def _split_threshold(rest: str) -> int:
    """Pods "<fid>-<digits>" of a function vs the pods of an id that extends
    it as "<fid>-<rest>": comparing <digits> with "<rest>-..." is decided
    within the leading digit run d of "<rest>-" and the character c after
    it (the digits can never reach the '-').  Returns T such that the pods
    whose digits_key is <= T sort before the extending id's pods."""
    t = rest + "-"
    k = 0
    while t[k] in "0123456789":
        k += 1
    d, c = t[:k], t[k]
    if len(d) >= 10 or c < "0":
        return _digits_key_text(d[:10])       # only counters <= d sort first
    return _digits_key_text(d + "9" * (10 - len(d)))  # every counter starting with d too


def _pod_id_order(fids):
    """``_pod_id_order_of`` of a function-id list (a pure function of the
    strings, cached: the runs of a sweep share their function ids)."""
    return _pod_id_order_of(tuple(fids))


@lru_cache(maxsize=1024)
def _pod_id_order_of(fids):
    """Pod-id string order as (first slot, [(threshold, slot)]) per function id.

    Pod ids are f"{fid}-{n:04d}" (sim_engine.py:354).  Ids whose "fid-"
    strings are not prefixes of one another order by that string alone: one
    slot each, in sorted order.  When "a-" is a prefix of "b-" ("a" and
    "a-1"), every pod of "b" lies in one contiguous block between pods of "a"
    whose position depends only on the counter text of a's pod
    (``_split_threshold``).  A depth-first walk of the prefix forest hands
    out slots: a function's segments interleave with its extenders' blocks."""
    keyed = sorted(fids, key=lambda f: f + "-")
    children: dict = {f: [] for f in fids}
    roots, stack = [], []
    for g in keyed:
        while stack and not (g + "-").startswith(stack[-1] + "-"):
            stack.pop()
        (children[stack[-1]] if stack else roots).append(g)
        stack.append(g)
    order: dict = {}
    nxt = 0

    def visit(f):
        nonlocal nxt
        first = nxt
        nxt += 1
        splits = []
        for g in children[f]:
            visit(g)
            splits.append((_split_threshold(g[len(f) + 1:]), nxt))
            nxt += 1
        order[f] = (first, splits)

    for r in roots:
        visit(r)
    return order


def pod_order_key(order, fid: str, counter: int) -> int:
    """The device's 64-bit pod order key (tests compare it with str order)."""
    first, splits = order[fid]
    dk = _digits_key(counter)
    slot = first
    for thr, s in splits:
        if dk > thr:
            slot = s
    return slot * 11 ** 10 + dk


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


def _counts_array(trace) -> np.ndarray:
    """int32 counts of a trace (this package's traces cache the array; the
    reference's WorkloadTrace only has the tuple)."""
    arr = getattr(trace, "array", None)
    return arr() if arr is not None else np.array(trace.counts, np.int32)


def _point_table(profile, memo: dict | None) -> dict:
    """{(sm, quota): ProfileEntry} of a profile (per-call memo)."""
    m = _profile_memo(profile, memo)
    tab = m.get("table")
    if tab is None:
        tab = m["table"] = {(p.sm_partition, p.quota): e for p, e in profile.entries.items()}
    return tab


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
        pk = getattr(fn.trace, "peak", None)
        if pk is not None:
            peak = pk(int(scenario.windows)) / window_s
        else:
            counts = _counts_array(fn.trace)[:scenario.windows]
            peak = (int(counts.max()) if len(counts) else 0) / window_s
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
    funcs: np.ndarray           # point_off: offset into ``points`` (this run)
    point_blocks: list          # per function, read-only, shared between runs
    inits: np.ndarray
    counts: np.ndarray
    names: bytes
    scale_x: int
    scale_y: int
    point_keys: list          # per function: [(sm, quota)] in point order
    id_splits: np.ndarray     # ID_SPLIT_DT, function-relative (id_split_off)

    @property
    def points(self) -> np.ndarray:
        """This run's point table (the functions' blocks, concatenated)."""
        if not self.point_blocks:
            return np.zeros(0, POINT_DT)
        return np.concatenate(self.point_blocks)


def _point_block(lo: "_LoweredProfile", lx: int, ly: int, memo: dict | None) -> np.ndarray:
    """Device point rows of one lowered profile on a run's (lx, ly) grid.  The
    block is read-only and shared by every function / run of the call with
    the same profile and grid, so a batch uploads it once."""
    key = ("block", id(lo), lx, ly)
    hit = memo.get(key) if memo is not None else None
    if hit is not None and hit[0] is lo:
        return hit[1]
    block = lo.rows.copy()
    block["rect_w"] = [n * (lx // d) for n, d in zip(lo.w_num, lo.w_den)]
    block["rect_h"] = [n * (ly // d) for n, d in zip(lo.h_num, lo.h_den)]
    block.flags.writeable = False
    if memo is not None:
        memo[key] = (lo, block)
    return block


def compile_run(scenario, policy: str = "fast", caps: Caps | None = None,
                memo: dict | None = None) -> RunImage:
    """Lower one (scenario, policy) run.  ``memo``: a dict shared by the runs of
    ONE batch compile (per-profile-object cache; never reuse it across calls)."""
    if policy not in POLICIES:
        raise ValidationError(f"policy must be one of {POLICIES}, got {policy!r}")
    validate_scenario(scenario, memo)
    fns = _ordered_functions(scenario)
    fids = [fn.function_id for fn in fns]
    timeshare = policy == "timeshare"
    tables = [_point_table(fn.profile, memo) for fn in fns]
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

    order = _pod_id_order(fids)
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
    point_blocks, init_rows, point_keys, frows, traces, id_splits = [], [], [], [], [], []
    n_points = 0
    names = []
    name_off = 0
    sm_integral = all(lo.sm_integral for lo in lowered)
    for fi, (fn, lo) in enumerate(zip(fns, lowered)):
        point_blocks.append(_point_block(lo, lx, ly, memo))
        point_keys.append(lo.keys)
        n_init = len(fn.initial_pods)
        for init in fn.initial_pods:
            k = (init.point.sm_partition, init.point.quota)
            has = init.quota_request is not None
            init_rows.append((lo.index[k], 1 if has else 0,
                              float(init.quota_request) if has else 0.0))
        tc = _counts_array(fn.trace)
        traces.append(tc if len(tc) <= windows else tc[:windows])
        raw = fn.function_id.encode("utf-8")
        mem = fn.profile.mem
        # None = unbounded (-1 on the device).  A negative limit makes the
        # reference's `len(fn.queue) >= limit` (sim_engine.py:476) always true,
        # exactly like 0: every arrival is dropped.
        mq = -1 if fn.max_queue is None else max(0, int(fn.max_queue))
        first, splits = order[fn.function_id]
        frows.append((len(lo.keys), n_points, n_init, len(init_rows) - n_init, fi * windows,
                      mq, lo.p_eff, first, name_off, len(raw), len(splits), len(id_splits),
                      fn.profile.slo_latency_ms, mem.mem_server_mb, mem.mem_runtime_mb,
                      mem.mem_noshare_mb))
        n_points += len(lo.keys)
        name_off += len(raw)
        names.append(raw)
        id_splits.extend((thr, slot, 0) for thr, slot in splits)
    funcs = np.array(frows, FUNCTION_DT) if frows else np.zeros(0, FUNCTION_DT)
    if all(len(t) == windows for t in traces):
        counts = np.concatenate(traces) if traces else np.zeros(0, np.int32)
    else:
        counts = np.zeros(n_f * windows, np.int32)
        for fi, t in enumerate(traces):
            counts[fi * windows: fi * windows + len(t)] = t
    names = b"".join(names)

    window_s = scenario.window_ms / 1000.0
    scen = np.array([(
        n_nodes, n_f, windows, steps_per_window(scenario.quantum), scenario.epoch_windows,
        scenario.cold_start_windows, scenario.restructure_threshold,
        ((GS_FLAG_TIMESHARE if timeshare else 0)
         | (GS_FLAG_SHARING if scenario.model_sharing else 0)
         | (GS_FLAG_SM_INTEGRAL if sm_integral else 0)),
        0, side_x, side_y, caps.pods, caps.rects, caps.returned, caps.hot_class,
        0, 0, 0, 0, window_s, window_s * scenario.quantum, scenario.quantum,
        scenario.gpu_capacity_mb)], SCENARIO_DT)
    return RunImage(policy, fids, scen, funcs, point_blocks,
                    np.array(init_rows, INIT_DT), counts, names, lx, ly, point_keys,
                    np.array(id_splits, ID_SPLIT_DT))


_POOL_MIN_RUNS = 256          # below this a fork pool costs more than it saves


def _compile_span(scenarios, policies, caps, lo, hi):
    """compile_run over inputs [lo, hi) with one shared memo (== one call)."""
    memo: dict = {}
    out = []
    for i in range(lo, hi):
        try:
            out.append(compile_run(scenarios[i], policies[i], caps, memo))
        except Exception as exc:           # shipped back, raised in input order
            out.append(exc)
    return out


_FORK_STATE = None


def _forked_part(span):
    """Worker body: compile a span and pack it into one Batch part; only the
    packed arrays and the per-run metadata (no count arrays) travel back."""
    sc, pol, caps = _FORK_STATE
    res = _compile_span(sc, pol, caps, span[0], span[1])
    ok = [k for k, r in enumerate(res) if isinstance(r, RunImage)]
    part = Batch([res[k] for k in ok]) if ok else None
    for k in ok:
        res[k].counts = None              # the part holds them
    return part, res


def compile_batch(scenarios, policies, caps: Caps | None = None, *,
                  workers: int | None = None):
    """Lower a batch of (scenario, policy) runs on all host cores.

    Returns ``(batch, index, errors)``: ``batch`` holds the runs that compiled,
    in input order, ``index[j]`` is the input position of batch run ``j`` and
    ``errors`` maps the other input positions to the exception
    ``compile_run`` raised for them.  Large batches are lowered by a fork pool:
    the scenario objects reach the workers copy-on-write, each worker packs
    its span into a ``Batch`` part, and the parts are concatenated here.
    Profile-derived data is shared by the runs of one span only (see
    ``_profile_memo``)."""
    import os
    global _FORK_STATE
    if not (hasattr(scenarios, "__getitem__") and hasattr(scenarios, "__len__")):
        scenarios = list(scenarios)       # a lazy sequence stays lazy (built in the workers)
    policies = list(policies)
    n = len(scenarios)
    workers = workers if workers is not None else (os.cpu_count() or 1)
    if n < _POOL_MIN_RUNS or workers <= 1:
        res = _compile_span(scenarios, policies, caps, 0, n)
        index = [i for i, r in enumerate(res) if isinstance(r, RunImage)]
        errors = {i: r for i, r in enumerate(res) if not isinstance(r, RunImage)}
        return Batch([res[i] for i in index]), index, errors
    import multiprocessing as mp
    chunks = workers * 2
    bounds = [(n * k // chunks, n * (k + 1) // chunks) for k in range(chunks)]
    _FORK_STATE = (scenarios, policies, caps)
    # freeze the heap before forking: a child's collector would otherwise walk
    # (and so copy-on-write fault) every object of the parent
    import gc
    gc.freeze()
    import warnings
    try:
        with warnings.catch_warnings():
            # the workers only run Python/numpy lowering (no CUDA, no threads)
            warnings.filterwarnings("ignore", message=".*use of fork\\(\\) may lead to deadlocks.*",
                                    category=DeprecationWarning)
            with mp.get_context("fork").Pool(workers) as pool:
                got = pool.map(_forked_part, bounds, chunksize=1)
    finally:
        _FORK_STATE = None
        gc.unfreeze()
    index, errors, parts = [], {}, []
    for (lo, _hi), (part, res) in zip(bounds, got):
        for k, r in enumerate(res):
            if isinstance(r, RunImage):
                index.append(lo + k)
            else:
                errors[lo + k] = r
        if part is not None:
            parts.append(part)
    return Batch.concat(parts), index, errors


def compile_stream(scenarios, policies, caps: Caps | None = None, *,
                   workers: int | None = None, parts: int | None = None):
    """``compile_batch`` as a stream: yields ``(batch, index, errors)`` per
    consecutive block of the inputs, in input order, as soon as the block is
    lowered -- so a caller can start the GPU on the first blocks while the
    host cores still lower the rest (``engine.simulate_records``).  ``index``
    holds absolute input positions.  ``parts`` = number of blocks (default:
    about 8, never below 64 runs per block)."""
    import os
    global _FORK_STATE
    if not (hasattr(scenarios, "__getitem__") and hasattr(scenarios, "__len__")):
        scenarios = list(scenarios)
    policies = list(policies)
    n = len(scenarios)
    workers = workers if workers is not None else (os.cpu_count() or 1)
    n_parts = parts if parts is not None else max(1, min(8, n // 64))
    blocks = [(n * k // n_parts, n * (k + 1) // n_parts) for k in range(n_parts)]
    if n < _POOL_MIN_RUNS or workers <= 1:
        for lo, hi in blocks:
            res = _compile_span(scenarios, policies, caps, lo, hi)
            idx = [k for k, r in enumerate(res) if isinstance(r, RunImage)]
            yield (Batch([res[k] for k in idx]), [lo + k for k in idx],
                   {lo + k: r for k, r in enumerate(res) if not isinstance(r, RunImage)})
        return
    # every block is split across all workers (spans of >= 32 runs), so the
    # blocks complete one after another (block 0 first) instead of all at the end
    spans, owner = [], []
    for b, (lo, hi) in enumerate(blocks):
        m = max(1, min(workers, (hi - lo) // 32))
        for k in range(m):
            spans.append((lo + (hi - lo) * k // m, lo + (hi - lo) * (k + 1) // m))
            owner.append(b)
    import multiprocessing as mp
    import gc
    import warnings
    _FORK_STATE = (scenarios, policies, caps)
    gc.freeze()
    try:
        with warnings.catch_warnings():
            warnings.filterwarnings("ignore", message=".*use of fork\\(\\) may lead to deadlocks.*",
                                    category=DeprecationWarning)
            pool = mp.get_context("fork").Pool(workers)
    finally:
        _FORK_STATE = None
        gc.unfreeze()
    try:
        got = pool.imap(_forked_part, spans, chunksize=1)
        cur, acc_parts, acc_index, acc_err = 0, [], [], {}
        for (lo, _hi), b, (part, res) in zip(spans, owner, got):
            if b != cur:
                yield Batch.concat(acc_parts), acc_index, acc_err
                cur, acc_parts, acc_index, acc_err = b, [], [], {}
            for k, r in enumerate(res):
                if isinstance(r, RunImage):
                    acc_index.append(lo + k)
                else:
                    acc_err[lo + k] = r
            if part is not None:
                acc_parts.append(part)
        yield Batch.concat(acc_parts), acc_index, acc_err
    finally:
        pool.terminate()
        pool.join()


def _cat(arrs, dt) -> np.ndarray:
    """Concatenate many small structured arrays of dtype ``dt`` by their bytes
    (np.concatenate re-derives the structured dtype promotion per input)."""
    dt = np.dtype(dt)
    raw = b"".join((a if a.dtype == dt else a.astype(dt)).tobytes() for a in arrs)
    return np.frombuffer(raw, dtype=dt).copy()


class Batch:
    """Concatenated RunImages + the ctypes ``gs_batch_t`` pointing at them."""

    def __init__(self, images: list):
        self.images = images
        for im in images:
            if im.counts is None:
                raise ValueError("this RunImage was packed by compile_batch; "
                                 "use Batch.prefix() / the batch it came with")
        if not images:
            self.runs = np.zeros(0, SCENARIO_DT)
            self.funcs = np.zeros(0, FUNCTION_DT)
            self.points = np.zeros(0, POINT_DT)
            self.inits = np.zeros(1, INIT_DT)
            self.counts = np.zeros(0, np.int32)
            self.names = np.zeros(1, np.uint8)
            self.id_splits = np.zeros(0, ID_SPLIT_DT)
            self.n_fn_rows = self.n_gpu_rows = self.n_glob_rows = self.n_placements = 0
            self.n_inits = 0
            return
        # per-run records and the run-level offsets, vectorised
        runs = _cat([im.scen for im in images], SCENARIO_DT)
        W = runs["windows"].astype(np.int64)
        nf = runs["n_funcs"].astype(np.int64)

        def excl(x):
            c = np.cumsum(x)
            return c - x, int(c[-1])

        runs["func_off"], n_funcs_all = excl(nf)
        runs["fn_row_off"], self.n_fn_rows = excl(W * nf)
        runs["gpu_row_off"], self.n_gpu_rows = excl(W * runs["n_nodes"].astype(np.int64))
        runs["glob_row_off"], self.n_glob_rows = excl(W)
        runs["place_off"], self.n_placements = excl(runs["cap_pods"].astype(np.int64))
        self.runs = runs
        # function records: per-run offsets into inits / counts / names /
        # id_splits repeated over the run's functions
        funcs = _cat([im.funcs for im in images], FUNCTION_DT)
        for field, arrs in (("init_off", [im.inits for im in images]),
                            ("count_off", [im.counts for im in images]),
                            ("name_off", [im.names for im in images]),
                            ("id_split_off", [im.id_splits for im in images])):
            lens = np.fromiter((len(a) for a in arrs), np.int64, len(arrs))
            funcs[field] += np.repeat(np.cumsum(lens) - lens, nf)
        # point blocks are deduplicated: by object, then by content
        seen: dict = {}
        by_content: dict = {}
        keep: list = []           # holds the blocks so ids in `seen` stay unique
        points, offs = [], []
        p_off = 0
        for im in images:
            for block in im.point_blocks:
                off = seen.get(id(block))
                if off is None:
                    ck = block.tobytes()
                    off = by_content.get(ck)
                    if off is None:
                        off = by_content[ck] = p_off
                        points.append(block)
                        p_off += len(block)
                    seen[id(block)] = off
                    keep.append(block)
                offs.append(off)
        funcs["point_off"] = np.asarray(offs, np.int64)
        self.funcs = funcs
        self.points = np.concatenate(points) if points else np.zeros(0, POINT_DT)
        inits = [im.inits for im in images]
        self.n_inits = sum(len(a) for a in inits)
        # keep at least one element so every pointer is valid
        self.inits = _cat(inits, INIT_DT) if self.n_inits else np.zeros(1, INIT_DT)
        self.counts = np.ascontiguousarray(np.concatenate([im.counts for im in images]), np.int32)
        self.names = np.frombuffer(b"".join(im.names for im in images) + b"\0", np.uint8).copy()
        self.id_splits = _cat([im.id_splits for im in images], ID_SPLIT_DT)

    def __len__(self):
        return len(self.images)

    @classmethod
    def concat(cls, parts: list) -> "Batch":
        """One batch from consecutive parts (offsets rebased, arrays joined)."""
        b = cls([])
        if not parts:
            return b
        runs, funcs, points = [], [], []
        by_content: dict = {}                     # point blocks, deduplicated across parts
        f_off = p_off = i_off = c_off = n_off = s_off = 0
        fn_rows = gpu_rows = glob_rows = places = 0
        for part in parts:
            r = part.runs.copy()
            r["func_off"] += f_off
            r["fn_row_off"] += fn_rows
            r["gpu_row_off"] += gpu_rows
            r["glob_row_off"] += glob_rows
            r["place_off"] += places
            fc = part.funcs.copy()
            starts, first, inv = np.unique(fc["point_off"], return_index=True,
                                           return_inverse=True)
            remap = np.empty(len(starts), np.int64)
            for u, (st, k) in enumerate(zip(starts.tolist(), first.tolist())):
                block = part.points[st: st + int(fc["n_points"][k])]
                key = block.tobytes()
                off = by_content.get(key)
                if off is None:
                    off = by_content[key] = p_off
                    points.append(block)
                    p_off += len(block)
                remap[u] = off
            fc["point_off"] = remap[inv.reshape(-1)]
            fc["init_off"] += i_off
            fc["count_off"] += c_off
            fc["name_off"] += n_off
            fc["id_split_off"] += s_off
            s_off += len(part.id_splits)
            runs.append(r)
            funcs.append(fc)
            f_off += len(fc)
            i_off += part.n_inits
            c_off += len(part.counts)
            n_off += len(part.names) - 1          # each part ends with one NUL
            fn_rows += part.n_fn_rows
            gpu_rows += part.n_gpu_rows
            glob_rows += part.n_glob_rows
            places += part.n_placements
        b.images = [im for part in parts for im in part.images]
        b.runs = np.concatenate(runs)
        b.funcs = np.concatenate(funcs)
        b.points = np.concatenate(points) if points else np.zeros(0, POINT_DT)
        b.inits = np.concatenate([p.inits[:p.n_inits] for p in parts] + [np.zeros(1, INIT_DT)])
        b.counts = np.ascontiguousarray(np.concatenate([p.counts for p in parts]), np.int32)
        b.names = np.concatenate([p.names[:-1] for p in parts] + [np.zeros(1, np.uint8)])
        b.id_splits = np.concatenate([p.id_splits for p in parts])
        b.n_fn_rows, b.n_gpu_rows, b.n_glob_rows = fn_rows, gpu_rows, glob_rows
        b.n_placements = places
        b.n_inits = i_off
        return b

    def prefix(self, n: int) -> "Batch":
        """The first ``n`` runs as a batch with the identical layout (row and
        placement offsets unchanged), e.g. a CPU-sample of a device batch."""
        b = Batch([])
        b.images = self.images[:n]
        b.runs = self.runs[:n].copy()
        nf = int(self.runs["func_off"][n]) if n < len(self) else len(self.funcs)
        b.funcs = self.funcs[:nf].copy()
        b.points, b.inits, b.counts, b.names = self.points, self.inits, self.counts, self.names
        b.id_splits = self.id_splits
        b.n_inits = self.n_inits
        last = self.runs[n - 1] if n else None
        if last is None:
            b.n_fn_rows = b.n_gpu_rows = b.n_glob_rows = b.n_placements = 0
        else:
            W = int(last["windows"])
            b.n_fn_rows = int(last["fn_row_off"]) + W * int(last["n_funcs"])
            b.n_gpu_rows = int(last["gpu_row_off"]) + W * int(last["n_nodes"])
            b.n_glob_rows = int(last["glob_row_off"]) + W
            b.n_placements = int(last["place_off"]) + int(last["cap_pods"])
        return b

    def alloc_outputs(self, rows: bool = True, pinned: bool | str = False):
        """Output arrays.  ``pinned=True`` places the row arrays in page-locked,
        device-mapped host memory, which the kernel fills in place (zero-copy,
        overlapped with the simulation); the contents start uninitialised.
        ``pinned="pool"``: the same, from the recycled page-locked pool."""
        if pinned:
            from .backend import host_empty

            def alloc(n, dt):
                return host_empty(n, dt, recycle=(pinned == "pool"))
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
        for name in ("runs", "funcs", "points", "inits", "counts", "names", "id_splits"):
            a = getattr(self, name)
            p = host_empty(len(a), a.dtype)
            p[:len(a)] = a
            # an empty id_splits must stay empty (its length is part of the
            # batch shape); the other arrays are never empty
            setattr(self, name, p[:len(a)] if (len(a) or name == "id_splits") else p)
        return self

    def input_bytes(self) -> int:
        return sum(a.nbytes for a in (self.runs, self.funcs, self.points, self.inits,
                                      self.counts, self.names, self.id_splits))
