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

from .metrics import CSV_COLUMNS, SCHEMA_VERSION
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
