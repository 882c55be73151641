"""Fast host path from device output records to the reference's report files.

SURVEY §8(f)2.  ``engine.decode_run`` rebuilds one ``MetricsReport`` per run
(one dataclass per window row) so callers get the reference's objects; for
sweeps of thousands of runs that object layer dominates host time.  The
functions here render ``metrics.csv`` and ``summary.json`` straight from the
fixed-size row records of a ``compiler.Batch`` output dict, byte-identical to
``MetricsReport.to_csv()`` / ``summary()`` (reference metrics.py:62-131):

* rows per window in the reference's order: the global row, function rows in
  function-id order (the compiler indexes functions in sorted-id order), GPU
  rows of nodes with placements in gpu-id order (sim_engine.py:569-589);
* numbers through the same ``fmt_num(round(x, 9))`` rendering (util.py:4-10),
  with a per-value cache (utilisations repeat heavily);
* summary means with Python's own ``sum`` in row order (CPython 3.12's sum is
  compensated -- the same function the reference calls).
"""
from __future__ import annotations

import csv
import io
import json
import os

import numpy as np

from .metrics import (CSV_COLUMNS, SCHEMA_VERSION, FunctionWindowRow, GlobalWindowRow,
                      GpuWindowRow, MetricsReport)
from .util import fmt_num

_HEADER = ",".join(CSV_COLUMNS) + "\n"


def _slices(batch, out: dict, r: int):
    s = batch.runs[r]
    W, F, G = int(s["windows"]), int(s["n_funcs"]), int(s["n_nodes"])
    fo, go, lo = int(s["fn_row_off"]), int(s["gpu_row_off"]), int(s["glob_row_off"])
    fn = out["fn_rows"][fo: fo + W * F].reshape(W, F) if F else np.zeros((W, 0), out["fn_rows"].dtype)
    gp = out["gpu_rows"][go: go + W * G].reshape(W, G)
    gl = out["glob_rows"][lo: lo + W]
    return W, F, G, fn, gp, gl


def _csv_field(text: str) -> str:
    """A function id as csv.writer renders it (QUOTE_MINIMAL, same dialect as
    MetricsReport.to_csv)."""
    buf = io.StringIO()
    csv.writer(buf, lineterminator="\n").writerow([text, ""])
    return buf.getvalue()[:-2]


def run_csv(batch, out: dict, r: int) -> str:
    """``metrics.csv`` of run ``r`` (== decode_run(...).report.to_csv())."""
    W, F, G, fn, gp, gl = _slices(batch, out, r)
    fids = [_csv_field(f) for f in batch.images[r].fids]
    cache: dict = {}

    def num9(x):
        v = cache.get(x)
        if v is None:
            v = cache[x] = fmt_num(round(x, 9))
        return v

    mem_cache: dict = {}

    def num6(x):
        v = mem_cache.get(x)
        if v is None:
            v = mem_cache[x] = fmt_num(round(x, 6))
        return v

    fn_cols = [fn[name].tolist() for name in
               ("arrivals", "completions", "slo_violations", "dropped", "queue_depth")]
    present = gp["present"].tolist()
    util, occ, mem = gp["utilization"].tolist(), gp["sm_occupancy"].tolist(), gp["memory_mb"].tolist()
    g_use, g_fail, g_frag = (gl["gpus_in_use"].tolist(), gl["placement_failures"].tolist(),
                            gl["fragmentation_index"].tolist())
    parts = [_HEADER]
    app = parts.append
    for w in range(W):
        app(f"{w},global,,,,,,,,,,{g_use[w]},{g_fail[w]},{num9(g_frag[w])}\n")
        a, c, v, d, q = (col[w] for col in fn_cols)
        for f in range(F):
            app(f"{w},function,{fids[f]},{a[f]},{c[f]},{v[f]},{d[f]},{q[f]},,,,,,\n")
        pw = present[w]
        for g in range(G):
            if pw[g]:
                app(f"{w},gpu,{g},,,,,,{num9(util[w][g])},{num9(occ[w][g])},{num6(mem[w][g])},,,\n")
    return "".join(parts)


def run_summary(batch, out: dict, r: int) -> dict:
    """``summary()`` of run ``r`` (== decode_run(...).report.summary())."""
    W, F, G, fn, gp, gl = _slices(batch, out, r)
    im = batch.images[r]
    per_function = {}
    comp_all = viol_all = 0
    for f in sorted(range(F), key=lambda k: im.fids[k]):
        col = fn[:, f]
        arr, comp = int(col["arrivals"].sum()), int(col["completions"].sum())
        viol, drop = int(col["slo_violations"].sum()), int(col["dropped"].sum())
        depth = int(col["queue_depth"][-1]) if W else 0
        comp_all += comp
        viol_all += viol
        per_function[im.fids[f]] = {
            "arrivals": arr, "completions": comp, "slo_violations": viol, "dropped": drop,
            "final_queue_depth": depth,
            "slo_violation_pct": round(100.0 * viol / comp, 6) if comp else 0.0,
        }
    mask = gp["present"].astype(bool)
    n_gpu = int(mask.sum())

    def mean(name):
        if not n_gpu:
            return 0.0
        return round(sum(gp[name][mask].tolist()) / n_gpu, 9)     # row (window, gpu) order

    return {
        "schema_version": SCHEMA_VERSION,
        "policy": im.policy,
        "windows": W,
        "gpus_used_peak": int(gl["gpus_in_use"].max()) if W else 0,
        "placement_failures": int(gl["placement_failures"].sum()),
        "mean_utilization": mean("utilization"),
        "mean_sm_occupancy": mean("sm_occupancy"),
        "slo_violation_pct": round(100.0 * viol_all / comp_all, 6) if comp_all else 0.0,
        "per_function": per_function,
    }


def write_run(batch, out: dict, r: int, out_dir) -> tuple:
    """``MetricsReport.write`` of run ``r``: metrics.csv + summary.json."""
    os.makedirs(out_dir, exist_ok=True)
    csv_path = os.path.join(out_dir, "metrics.csv")
    json_path = os.path.join(out_dir, "summary.json")
    with open(csv_path, "w", encoding="utf-8", newline="") as fh:
        fh.write(run_csv(batch, out, r))
    with open(json_path, "w", encoding="utf-8") as fh:
        json.dump(run_summary(batch, out, r), fh, indent=2, sort_keys=True)
        fh.write("\n")
    return csv_path, json_path


# ---------------------------------------------------------------------------
# Native rendering (csrc/gs_host.cpp) and batch summaries
# ---------------------------------------------------------------------------

def fid_csv_table(batch):
    """(UTF-8 bytes, int64 offsets) of every batch function's id as csv.writer
    renders it, in gs_function_t order -- the ``fid_csv`` input of
    gs_format_csv*.  Cached on the batch."""
    hit = getattr(batch, "_fid_csv", None)
    if hit is not None:
        return hit
    names = batch.names.tobytes()
    cache: dict = {}
    parts, offs, pos = [], [0], 0
    for off, ln in zip(batch.funcs["name_off"].tolist(), batch.funcs["name_len"].tolist()):
        raw = names[off: off + ln]
        enc = cache.get(raw)
        if enc is None:
            enc = cache[raw] = _csv_field(raw.decode("utf-8")).encode("utf-8")
        parts.append(enc)
        pos += len(enc)
        offs.append(pos)
    table = (np.frombuffer(b"".join(parts) + b"\0", np.uint8).copy(), np.array(offs, np.int64))
    batch._fid_csv = table
    return table


def csv_texts(batch, out: dict, runs=None, n_threads: int = 0) -> list:
    """``metrics.csv`` of many runs at once, rendered by the native formatter
    on ``n_threads`` host threads (0 = all cores); byte-identical to
    ``run_csv`` / ``MetricsReport.to_csv()``."""
    import ctypes as C
    from .abi import make_batch_struct, make_out_struct
    from .backend import lib
    L = lib()
    runs = range(len(batch)) if runs is None else runs
    r0, r1 = (runs.start, runs.stop) if isinstance(runs, range) and runs.step == 1 else (None, None)
    if r0 is None:
        return [csv_texts(batch, out, range(r, r + 1), n_threads)[0] for r in runs]
    b, o = make_batch_struct(batch), make_out_struct(out)
    text, offs = fid_csv_table(batch)
    need = L.gs_format_csv_batch(C.byref(b), C.byref(o), r0, r1, text.ctypes.data,
                                 offs.ctypes.data, None, 0, None, None, 0)
    if need < 0:
        raise ValueError("gs_format_csv_batch: bad arguments (rows missing?)")
    buf = np.empty(max(need, 1), np.uint8)
    starts = np.zeros(max(r1 - r0, 1), np.int64)
    lens = np.zeros(max(r1 - r0, 1), np.int64)
    rc = L.gs_format_csv_batch(C.byref(b), C.byref(o), r0, r1, text.ctypes.data,
                               offs.ctypes.data, buf.ctypes.data, len(buf), starts.ctypes.data,
                               lens.ctypes.data, int(n_threads))
    if rc != 0:
        raise ValueError(f"gs_format_csv_batch failed ({rc})")
    mv = memoryview(buf)
    return [str(mv[s: s + n], "utf-8") for s, n in zip(starts[:r1 - r0].tolist(),
                                                       lens[:r1 - r0].tolist())]


def format_numbers(values, ndigits: int) -> list:
    """fmt_num(round(x, ndigits)) by the native renderer (ndigits < 0: no
    rounding) -- exposed so the tests can pin it against the interpreter."""
    from .backend import lib
    x = np.ascontiguousarray(values, np.float64)
    stride = 48
    buf = np.zeros(len(x) * stride + 1, np.uint8)
    if lib().gs_format_numbers(x.ctypes.data, len(x), int(ndigits), buf.ctypes.data, stride):
        raise ValueError("gs_format_numbers failed")
    raw = buf[:len(x) * stride].reshape(len(x), stride) if len(x) else buf[:0].reshape(0, stride)
    return [bytes(row).split(b"\0", 1)[0].decode() for row in raw]


def summaries(batch, out: dict, runs=None) -> list:
    """``summary()`` of many runs (== MetricsReport.summary(), metrics.py:94-131):
    per-function totals as one vectorised reduction per (windows, functions)
    shape, GPU means from the device's summary record (Python ``sum`` of the
    GPU rows in row order, computed on the device), everything else from the
    global rows."""
    runs = list(range(len(batch))) if runs is None else list(runs)
    res: list = [None] * len(runs)
    R = batch.runs
    totals = None
    if runs and runs == list(range(runs[0], runs[-1] + 1)):
        # per-function totals of the whole range by the native reducer
        import ctypes as C
        from .abi import make_batch_struct, make_out_struct
        from .backend import lib
        f0 = int(R["func_off"][runs[0]])
        f1 = int(R["func_off"][runs[-1]]) + int(R["n_funcs"][runs[-1]])
        totals = np.zeros((max(f1 - f0, 1), 5), np.int64)
        b, o = make_batch_struct(batch), make_out_struct(out)
        if lib().gs_fn_totals(C.byref(b), C.byref(o), runs[0], runs[-1] + 1,
                              totals.ctypes.data, 0) != 0:
            raise ValueError("gs_fn_totals: bad arguments")
    groups: dict = {}
    for k, r in enumerate(runs):
        groups.setdefault((int(R["windows"][r]), int(R["n_funcs"][r])), []).append(k)
    fn_all, gl_all, sm_all = out["fn_rows"], out["glob_rows"], out["summary"]
    def rows_of(arr, off, per):
        """(runs, per) records: a zero-copy view when the runs' blocks are
        consecutive (the usual batch layout), else a gather."""
        if len(off) and per and np.all(np.diff(off) == per):
            return arr[int(off[0]): int(off[0]) + len(off) * per].reshape(len(off), per)
        return arr[off[:, None] + np.arange(per)[None, :]]

    for (W, F), ks in groups.items():
        rr = np.array([runs[k] for k in ks])
        if totals is not None:
            fo = R["func_off"][rr] - f0
            sums = totals[fo[:, None] + np.arange(F)[None, :]]      # (runs, F, 5)
            depth = sums[:, :, 4].tolist()
        else:
            fn = rows_of(fn_all, R["fn_row_off"][rr], W * F).reshape(len(rr), W, F)
            # the five int32 columns as one contiguous matrix: one reduction pass
            cols = np.ascontiguousarray(fn).view(np.int32).reshape(len(rr), W, F, 5)
            sums = cols.sum(axis=1, dtype=np.int64)                 # (runs, F, 5)
            depth = (cols[:, -1, :, 4] if W else np.zeros((len(rr), F), np.int32)).tolist()
        tot = {name: sums[:, :, k].tolist() for k, name in
               enumerate(("arrivals", "completions", "slo_violations", "dropped"))}
        gl = rows_of(gl_all, R["glob_row_off"][rr], W)
        peak = (gl["gpus_in_use"].max(axis=1) if W else np.zeros(len(rr), np.int32)).tolist()
        fails = gl["placement_failures"].sum(axis=1).tolist()
        sm = sm_all[rr]
        n_gpu = sm["n_gpu_rows"].tolist()
        su, so = sm["sum_utilization"].tolist(), sm["sum_sm_occupancy"].tolist()
        images = batch.images
        for j, k in enumerate(ks):
            im = images[runs[k]]
            a_, c_, v_, d_, q_ = (tot["arrivals"][j], tot["completions"][j],
                                  tot["slo_violations"][j], tot["dropped"][j], depth[j])
            per_function = {
                fid: {"arrivals": a, "completions": c, "slo_violations": v, "dropped": d,
                      "final_queue_depth": q,
                      "slo_violation_pct": round(100.0 * v / c, 6) if c else 0.0}
                for fid, a, c, v, d, q in zip(im.fids, a_, c_, v_, d_, q_)}
            comp_all, viol_all = sum(c_), sum(v_)
            n = n_gpu[j]
            res[k] = {
                "schema_version": SCHEMA_VERSION,
                "policy": im.policy,
                "windows": W,
                "gpus_used_peak": peak[j],
                "placement_failures": fails[j],
                "mean_utilization": round(su[j] / n, 9) if n else 0.0,
                "mean_sm_occupancy": round(so[j] / n, 9) if n else 0.0,
                "slo_violation_pct": round(100.0 * viol_all / comp_all, 6) if comp_all else 0.0,
                "per_function": per_function,
            }
    return res


def decode_rows(batch, out: dict, r: int) -> tuple:
    """The reference's row objects of run ``r`` (metrics.py:27-52), in its append
    order (sim_engine.py:555-589): (function_rows, gpu_rows, global_rows)."""
    W, F, G, fn, gp, gl = _slices(batch, out, r)
    fids = batch.images[r].fids
    fn_l, gp_l, gl_l = fn.reshape(-1).tolist(), gp.reshape(-1).tolist(), gl.tolist()
    frows, grows, lrows = [], [], []
    for w in range(W):
        for f in range(F):
            a, c, v, d, q = fn_l[w * F + f]
            frows.append(FunctionWindowRow(w, fids[f], a, c, v, d, q))
        for g in range(G):
            u, o, m, present, _ = gp_l[w * G + g]
            if present:
                grows.append(GpuWindowRow(w, g, u, o, m))
        n_use, fails, frag = gl_l[w]
        lrows.append(GlobalWindowRow(w, n_use, fails, frag))
    return frows, grows, lrows


class SharedOutputs:
    """One batch's output records, shared by its runs' DeviceReports; the
    summaries of all runs are computed together on first request."""

    def __init__(self, batch, out: dict):
        self.batch, self.out = batch, out
        self._summaries = None

    def prepare(self) -> None:
        """Compute every run's summary now (the API does this per block while
        the next blocks are still on the GPU)."""
        if self._summaries is None:
            self._summaries = summaries(self.batch, self.out)

    def take_summary(self, r: int) -> dict:
        if self._summaries is None:
            self._summaries = summaries(self.batch, self.out)
        s = self._summaries[r]
        if s is None:                       # handed out before: build a fresh one
            return summaries(self.batch, self.out, [r])[0]
        self._summaries[r] = None
        return s


class DeviceReport(MetricsReport):
    """A ``MetricsReport`` backed by the device's row records.

    The row lists (``function_rows`` / ``gpu_rows`` / ``global_rows``) are
    built on first access; until then ``to_csv()`` renders natively
    (csrc/gs_host.cpp) and ``summary()`` comes from the vectorised batch
    reduction -- both byte-identical to ``MetricsReport``.  Once the rows are
    materialised (and possibly edited by the caller) the inherited methods
    are used.  Compares equal to a ``MetricsReport`` with the same policy and
    rows; pickles as a plain ``MetricsReport``."""

    def __init__(self, shared: SharedOutputs, r: int):
        self.policy = shared.batch.images[r].policy
        self._shared, self._r = shared, r
        self._rows = None

    def _materialise(self):
        if self._rows is None:
            self._rows = list(decode_rows(self._shared.batch, self._shared.out, self._r))
        return self._rows

    def _set(k):
        def setter(self, value):
            self._materialise()[k] = value
        return setter

    function_rows = property(lambda self: self._materialise()[0], _set(0))
    gpu_rows = property(lambda self: self._materialise()[1], _set(1))
    global_rows = property(lambda self: self._materialise()[2], _set(2))
    del _set

    def to_csv(self) -> str:
        if self._rows is not None:
            return super().to_csv()
        sh, r = self._shared, self._r
        return csv_texts(sh.batch, sh.out, range(r, r + 1), n_threads=1)[0]

    def summary(self) -> dict:
        if self._rows is not None:
            return super().summary()
        return self._shared.take_summary(self._r)

    def __eq__(self, other):
        if not isinstance(other, MetricsReport):
            return NotImplemented
        return (self.policy, self.function_rows, self.gpu_rows, self.global_rows) == (
            other.policy, other.function_rows, other.gpu_rows, other.global_rows)

    __hash__ = None

    def __repr__(self):
        return (f"MetricsReport(policy={self.policy!r}, function_rows={self.function_rows!r}, "
                f"gpu_rows={self.gpu_rows!r}, global_rows={self.global_rows!r})")

    def __reduce__(self):
        return (MetricsReport, (self.policy, self.function_rows, self.gpu_rows,
                                self.global_rows))
