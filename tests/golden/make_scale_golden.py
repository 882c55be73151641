"""Reference-generated goldens at BASELINE scale (BASELINE.json configs C1-C5).

make_golden.py pins the oracle on small, branch-covering scenarios; this
script pins the GPU (and the oracle) on the shapes the benchmark actually
runs: C2 at its 300 windows, C3 seeds under both policies, C4's 64-node x
200-function fleet, and points of the C5 (SM%, quantum, SLO) grid.  It runs
the REAL reference (imported read-only from /root/reference/pkg/src) on the
scenario dicts of paper_2309_00558_b200/workloads.py and stores, per
(config, args, policy):

  * sha256 of the scenario dict (so a drifting generator is caught),
  * sha256 + length of the metrics CSV (the full CSVs would be ~20 MB),
  * the summary dict and the final placements (exact rationals as text).

Build container only (the reference does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_scale_golden.py

Output: tests/golden/golden_scale.json.gz (committed).
"""
from __future__ import annotations

import gzip
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
OUT = os.path.join(HERE, "golden_scale.json.gz")


def cases():
    """(config, generator kwargs, policy) triples."""
    out = [("c1", {}, p) for p in ("fast", "timeshare")]
    out += [("c2", {"seed": s, "windows": 300}, "fast") for s in range(16)]
    out += [("c2", {"seed": s, "windows": 300}, "timeshare") for s in range(4)]
    out += [("c3", {"seed": s}, p) for s in range(32) for p in ("fast", "timeshare")]
    out += [("c4", {"seed": s, "windows": 30}, "fast") for s in range(3)]
    out += [("c4", {"seed": 3, "windows": 60}, "timeshare")]
    out += [("c4", {"seed": 4, "windows": 150}, "fast")]
    out += [("c5", {"index": i}, "fast") for i in range(0, 100000, 1563)]
    return out


def scenario_dict(config, kw):
    sys.path.insert(0, ROOT)
    from paper_2309_00558_b200 import workloads as wl
    return getattr(wl, config)(**kw)


def dict_sha(d) -> str:
    return hashlib.sha256(json.dumps(d, sort_keys=True).encode()).hexdigest()


def run_one(case):
    config, kw, policy = case
    sys.path.insert(0, REF)
    import gshare_sim as ref
    from gshare_sim.sim_engine import _Engine
    d = scenario_dict(config, kw)
    t0 = time.time()
    rec = {"config": config, "args": kw, "policy": policy, "scenario_sha256": dict_sha(d)}
    try:
        eng = _Engine(ref.Scenario.from_dict(json.loads(json.dumps(d))), policy)
        report = eng.run()
    except ref.GShareError as exc:
        rec["expect"] = {"error": type(exc).__name__, "message": str(exc)}
        return rec
    csv = report.to_csv()
    placements = []
    for node in eng.nodes:
        for pid, p in sorted(node.placements.items()):
            r = p.rect
            placements.append([node.gpu_id, pid] + [f"{v.numerator}/{v.denominator}"
                                                    for v in (r.x, r.y, r.w, r.h)])
    rec["expect"] = {"csv_sha256": hashlib.sha256(csv.encode()).hexdigest(),
                     "csv_len": len(csv), "summary": report.summary(),
                     "placements": placements}
    rec["ref_seconds"] = round(time.time() - t0, 3)
    return rec


def main():
    todo = cases()
    # longest first so the pool drains evenly
    weight = {"c4": 3, "c2": 2, "c1": 1, "c3": 0, "c5": 0}
    order = sorted(range(len(todo)), key=lambda i: (-weight[todo[i][0]],
                                                    -todo[i][1].get("windows", 0)))
    with mp.Pool(os.cpu_count()) as pool:
        got = pool.map(run_one, [todo[i] for i in order], chunksize=1)
    recs = [None] * len(todo)
    for i, r in zip(order, got):
        recs[i] = r
    with gzip.open(OUT, "wt", encoding="utf-8") as fh:
        json.dump({"generator": "tests/golden/make_scale_golden.py",
                   "reference": "pkg/src/gshare_sim 0.1.0",
                   "python": sys.version.split()[0], "records": recs}, fh)
    cpu = sum(r.get("ref_seconds", 0.0) for r in recs)
    print(f"wrote {len(recs)} records to {OUT} ({cpu:.0f} s of reference CPU)")


if __name__ == "__main__":
    main()
