"""Generate the golden fixtures that pin the oracle (and the GPU path).

Runs the REAL reference package (imported read-only from
/root/reference/pkg/src) on

  * the three bundled scenarios (pkg/scenarios/*.json) x both policies,
  * the constructed scenarios of the reference's own engine tests
    (pkg/tests/test_sim_engine.py make_scenario variants, :22-195),
  * a seeded random sweep that exercises every engine branch: epochs,
    scale-up/down with in-flight requests, retry, memory-gated placement,
    restructure, max_queue drops, fractional quotas / SM partitions, CSV
    profiles with zero-throughput points, timeshare validation errors,

and records for each (scenario, policy) the metrics CSV (or the exception
text), the summary, and the final packer placements.  Usage (in the build
container only -- the reference does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Output: tests/golden/golden_runs.json.gz (committed).
"""
from __future__ import annotations

import gzip
import json
import os
import random
import sys
import tempfile

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "golden_runs.json.gz")

FID_POOL = ["resnet_v1", "rnnt_asr", "bert_qa", "bert", "bert2", "vit", "A", "a_b",
            "gpt.small", "z9", "Resnet", "yolo", "m"]
SM_POOL = [6, 12, 24, 50, 60, 80, 100, 12.5, 33, 40, 75]
Q_POOL = [0.2, 0.4, 0.6, 0.8, 0.1, 0.25, 0.5, 0.75, 0.3, 0.35]


def _synth(rng, with_100):
    sms = sorted(set(rng.sample(SM_POOL, rng.randint(1, 5)) + ([100] if with_100 else [])))
    qs = sorted(set(rng.sample(Q_POOL, rng.randint(0, 4)) + [1.0]))
    return {
        "t_max": round(rng.uniform(4, 120), rng.choice([0, 1, 3])),
        "sm_knee": rng.choice([6.0, 12.0, 24.0, 50.0, 100.0, 37.5]),
        "grid_sm": sms, "grid_quota": qs,
        "slo_ms": rng.choice([50.0, 100.0, 250.0, 500.0, 1000.0, 2000.0]),
        "mem": {"mem_noshare_mb": rng.choice([1200.0, 1600.0, 2500.0, 700.5]),
                "mem_runtime_mb": rng.choice([900.0, 1100.0, 400.0, 333.3]),
                "mem_server_mb": rng.choice([600.0, 800.0, 1500.0, 250.25])},
    }, sms, qs


def _csv_profile(rng, fid, with_100):
    sms = sorted(set(rng.sample(SM_POOL, rng.randint(1, 4)) + ([100] if with_100 else [])))
    qs = sorted(set(rng.sample(Q_POOL, rng.randint(0, 3)) + [1.0]))
    lines = ["function_id,sm_partition,quota,throughput_rps,p99_ms,slo_ms,"
             "mem_noshare_mb,mem_runtime_mb,mem_server_mb"]
    slo = rng.choice([100.0, 400.0, 1000.0])
    for sm in sms:
        for q in qs:
            t = round(rng.uniform(0.5, 60.0) * q, 3)
            if rng.random() < 0.06:
                t = 0.0
            lines.append(f"{fid},{sm},{q},{t},{round(1000.0 / max(t, 1e-3), 3)},{slo},"
                         f"1300,950,650")
    return "\n".join(lines) + "\n", sms, qs


def _trace(rng, windows):
    kind = rng.choice(["constant", "constant", "step", "sinusoid", "explicit", "explicit"])
    pois = rng.random() < 0.4
    if kind == "constant":
        t = {"kind": "constant", "rps": round(rng.uniform(0, 70), rng.choice([0, 2]))}
    elif kind == "step":
        t = {"kind": "step", "base_rps": round(rng.uniform(0, 40), 1),
             "step_rps": round(rng.uniform(0, 90), 1), "step_window": rng.randint(0, windows)}
    elif kind == "sinusoid":
        t = {"kind": "sinusoid", "base_rps": round(rng.uniform(0, 50), 1),
             "amplitude_rps": round(rng.uniform(0, 40), 1),
             "period_windows": rng.randint(1, max(1, windows))}
    else:
        n = rng.randint(0, windows + 3)
        t = {"kind": "explicit", "counts": [
            rng.choice([0, 0, rng.randint(0, 15), rng.randint(10, 120)]) for _ in range(n)]}
        pois = False
    if pois:
        t["poisson"] = True
        if rng.random() < 0.7:
            t["seed"] = rng.randint(0, 10 ** 6)
    return t


def random_case(rng, idx):
    windows = rng.randint(2, 22)
    files = {}
    fns = []
    fids = rng.sample(FID_POOL, rng.randint(1, 5))
    with_100 = rng.random() < 0.8
    for fid in fids:
        if rng.random() < 0.18:
            text, sms, qs = _csv_profile(rng, fid, with_100)
            files[f"{fid}.csv"] = text
            prof = {"csv": f"{fid}.csv"}
        else:
            synth, sms, qs = _synth(rng, with_100)
            prof = {"synth": synth}
        inits = []
        for _ in range(rng.choice([0, 1, 1, 2, 3, 5])):
            p = {"sm": rng.choice(sms), "quota": rng.choice(qs)}
            if rng.random() < 0.2:
                p["quota_request"] = round(p["quota"] * rng.choice([0.5, 0.9, 1.0]), 3)
            inits.append(p)
        fn = {"function_id": fid, "profile": prof, "trace": _trace(rng, windows),
              "initial_pods": inits}
        if rng.random() < 0.15:
            fn["max_queue"] = rng.randint(0, 25)
        fns.append(fn)
    sc = {
        "fleet_size": rng.choice([1, 1, 2, 2, 3, 4]),
        "windows": windows,
        "epoch_windows": rng.randint(1, 6),
        "quantum": rng.choice([0.02, 0.02, 0.05, 0.1, 0.25, 0.5, 1.0, 0.04, 0.125, 0.01]),
        "cold_start_windows": rng.randint(0, 3),
        "seed": rng.randint(0, 1000),
        "functions": fns,
    }
    if rng.random() < 0.3:
        sc["window_ms"] = rng.choice([500.0, 250.0, 2000.0, 100.0, 333.0, 1500.0])
    if rng.random() < 0.3:
        sc["model_sharing"] = False
    if rng.random() < 0.35:
        sc["gpu_capacity_mb"] = rng.choice([3000.0, 4000.0, 8000.0, 81920.0, 5500.5])
    if rng.random() < 0.35:
        sc["restructure_threshold"] = rng.choice([0, 1, 2, 3, 4, 8])
    return {"name": f"random-{idx:04d}", "scenario": sc, "files": files}


def engine_test_cases():
    """The constructed scenarios of pkg/tests/test_sim_engine.py:22-195 as dicts."""
    def mk(name, t_max=10.0, knee=24.0, rps=10.0, windows=8, fleet_size=1, epoch_windows=5,
           cold=2, initial=((24, 1.0),), slo=250.0, grid_sm=(6, 12, 24, 50, 100),
           grid_quota=(0.2, 0.4, 0.6, 0.8, 1.0), max_queue=None):
        fn = {"function_id": "fn",
              "profile": {"synth": {"t_max": t_max, "sm_knee": knee, "grid_sm": list(grid_sm),
                                    "grid_quota": list(grid_quota), "slo_ms": slo}},
              "trace": {"kind": "constant", "rps": rps},
              "initial_pods": [{"sm": s, "quota": q} for s, q in initial]}
        if max_queue is not None:
            fn["max_queue"] = max_queue
        return {"name": name, "files": {}, "scenario": {
            "fleet_size": fleet_size, "windows": windows, "epoch_windows": epoch_windows,
            "cold_start_windows": cold, "functions": [fn]}}
    return [
        mk("engine-steady"),
        mk("engine-zero-arrivals", rps=0.0, windows=6, epoch_windows=2),
        mk("engine-overload", rps=100.0, epoch_windows=2, cold=0, grid_sm=(24,),
           grid_quota=(1.0,), slo=10000.0),
        mk("engine-cold-start", rps=5.0, windows=6, epoch_windows=1, cold=2, initial=(),
           slo=100.0),
        mk("engine-empty", rps=0.0, windows=4, epoch_windows=2, initial=()),
        mk("engine-full-gpu", rps=5.0, windows=4, initial=((100, 1.0),)),
        mk("engine-dropped", rps=50.0, windows=3, grid_sm=(24,), grid_quota=(1.0,),
           slo=10000.0, max_queue=5, epoch_windows=10),
    ]


def bundled_cases():
    out = []
    sdir = "/root/reference/pkg/scenarios"
    for name in sorted(os.listdir(sdir)):
        with open(os.path.join(sdir, name)) as fh:
            out.append({"name": "bundled-" + name[:-5], "files": {}, "scenario": json.load(fh)})
    # the survey's C1: consolidation at 1 node, 60 windows
    with open(os.path.join(sdir, "consolidation.json")) as fh:
        c1 = json.load(fh)
    c1.update({"fleet_size": 1, "windows": 60, "epoch_windows": 5, "cold_start_windows": 2})
    out.append({"name": "survey-C1", "files": {}, "scenario": c1})
    return out


def _flat_csv(fid, sms, qs, thr, slo=500.0):
    """A CSV profile whose throughput is thr(sm, q) (0 allowed: ProfileEntry
    only requires >= 0, profiles.py:48-66)."""
    lines = ["function_id,sm_partition,quota,throughput_rps,p99_ms,slo_ms,"
             "mem_noshare_mb,mem_runtime_mb,mem_server_mb"]
    for sm in sms:
        for q in qs:
            t = thr(sm, q)
            lines.append(f"{fid},{sm},{q},{t},{round(1000.0 / max(t, 1e-3), 3)},{slo},"
                         f"1300,950,650")
    return "\n".join(lines) + "\n"


def error_branch_cases():
    """Every ValidationError reachable from _Engine.run after validation
    (sim_engine.py:434-452): the scale_up guard t_eff <= 0
    (autoscaler.py:115-117) and the zero serving rate of a scaled-up pod's
    (sm_eff, 1.0) point (sim_engine.py:346-349) -- on the per-warp fleet
    sizes and on an XL fleet (F > 64 functions), with demand arriving before
    and after the first epoch, and the zero-throughput function sorted first,
    in the middle and last among the function ids."""
    out = []
    sms, qs = [12, 50, 100], [0.5, 1.0]
    zero = _flat_csv("z", sms, qs, lambda sm, q: 0.0)

    def synth_fn(fid, rps, inits=()):
        return {"function_id": fid, "trace": {"kind": "constant", "rps": rps},
                "profile": {"synth": {"t_max": 40.0, "sm_knee": 50.0, "grid_sm": sms,
                                      "grid_quota": qs, "slo_ms": 500.0}},
                "initial_pods": [{"sm": s, "quota": q} for s, q in inits]}

    for tag, fid_list, zpos in (("first", ["z", "zz_a", "zz_b"], 0),
                                ("middle", ["a", "z", "zz"], 1),
                                ("last", ["a", "b", "z"], 2)):
        for rps, epoch, w in ((5.0, 2, 6), (0.0, 2, 6), (12.0, 3, 4)):
            files, fns = {}, []
            for k, fid in enumerate(fid_list):
                if k == zpos:
                    files["z.csv"] = _flat_csv(fid, sms, qs, lambda sm, q: 0.0)
                    fns.append({"function_id": fid, "profile": {"csv": "z.csv"},
                                "trace": {"kind": "constant", "rps": rps}})
                else:
                    fns.append(synth_fn(fid, 20.0, [(50, 0.5)]))
            out.append({"name": f"err-no-throughput-{tag}-{rps:g}-{epoch}-{w}", "files": files,
                        "scenario": {"fleet_size": 2, "windows": w, "epoch_windows": epoch,
                                     "cold_start_windows": 1, "functions": fns}})
    # demand only in a late window: the error fires at the first epoch after it
    out.append({"name": "err-no-throughput-late-burst", "files": {"z.csv": zero},
                "scenario": {"fleet_size": 1, "windows": 9, "epoch_windows": 2,
                             "functions": [{"function_id": "z", "profile": {"csv": "z.csv"},
                                            "trace": {"kind": "explicit",
                                                      "counts": [0, 0, 0, 0, 0, 7, 0]}}]}})
    # a zero-throughput function that never sees demand runs to completion
    out.append({"name": "ok-zero-throughput-no-demand", "files": {"z.csv": zero},
                "scenario": {"fleet_size": 1, "windows": 8, "epoch_windows": 2,
                             "functions": [{"function_id": "z", "profile": {"csv": "z.csv"},
                                            "trace": {"kind": "constant", "rps": 0.0}},
                                           synth_fn("y", 30.0, [(12, 1.0)])]}})
    # zero serving rate of the scaled-up point: (50, 1.0) serves nothing but
    # (50, 0.5) is the most efficient point (fast) -- timeshare serves at (100, 1.0)
    zr = _flat_csv("zr", sms, qs, lambda sm, q: 0.0 if (sm == 50 and q == 1.0) else
                   (30.0 * q if sm == 50 else 2.0 * q))
    out.append({"name": "err-zero-rate-scaled-point", "files": {"zr.csv": zr},
                "scenario": {"fleet_size": 2, "windows": 7, "epoch_windows": 2,
                             "functions": [{"function_id": "zr", "profile": {"csv": "zr.csv"},
                                            "trace": {"kind": "constant", "rps": 25.0}},
                                           synth_fn("a", 10.0, [(12, 0.5)])]}})
    # XL fleet: 70 functions (> class L's 64) on 40 nodes, one zero-throughput
    for zfid in ("f000", "f041", "f069"):
        files, fns = {"z.csv": None}, []
        for i in range(70):
            fid = f"f{i:03d}"
            if fid == zfid:
                files["z.csv"] = _flat_csv(fid, sms, qs, lambda sm, q: 0.0)
                fns.append({"function_id": fid, "profile": {"csv": "z.csv"},
                            "trace": {"kind": "constant", "rps": 3.0}})
            else:
                fns.append(synth_fn(fid, 6.0 + (i % 7), [(12, 0.5)]))
        out.append({"name": f"err-no-throughput-xl-{zfid}", "files": files,
                    "scenario": {"fleet_size": 40, "windows": 4, "epoch_windows": 2,
                                 "cold_start_windows": 1, "gpu_capacity_mb": 81920.0,
                                 "functions": fns}})
    # negative max_queue: the reference's `len(queue) >= limit` drops everything
    for mq in (-1, -7, 0):
        out.append({"name": f"max-queue-{mq}", "files": {},
                    "scenario": {"fleet_size": 1, "windows": 5, "epoch_windows": 2,
                                 "functions": [dict(synth_fn("q", 15.0, [(50, 1.0)]),
                                                    max_queue=mq),
                                               synth_fn("r", 9.0, [(12, 1.0)])]}})
    return out


PREFIX_FAMILIES = [
    ["x", "x-005", "x-01a", "x-0", "x-a"],
    ["m", "m-", "m-005", "m-005-1", "m-1"],
    ["1", "1-0", "1-007", "1-007-0", "10"],
    ["bert", "bert-01", "bert-01-a", "bert-015", "bert2"],
    ["f", "f-0099", "f-0100x", "f-00x"],
]


def prefix_cases(n: int = 40, seed: int = 8675309):
    """Function ids that extend other ids with "-" (pod-id string order then
    interleaves the families' pods by counter text, sim_engine.py:354): long,
    scaling-heavy runs so pod counters cross the thresholds ("x-005" splits
    the pods of "x" at counter 50, "x-01a" at 200, ...)."""
    rng = random.Random(seed)
    out = []
    for k in range(n):
        fam = PREFIX_FAMILIES[k % len(PREFIX_FAMILIES)]
        fids = rng.sample(fam, rng.randint(2, len(fam)))
        windows = rng.randint(40, 140)
        fns = []
        for fid in fids:
            synth, sms, qs = _synth(rng, True)
            synth["t_max"] = round(rng.uniform(4, 25), 1)   # small pods: many of them
            kind = rng.choice(["sinusoid", "step", "constant"])
            if kind == "sinusoid":
                tr = {"kind": "sinusoid", "base_rps": round(rng.uniform(10, 60), 1),
                      "amplitude_rps": round(rng.uniform(10, 50), 1),
                      "period_windows": rng.randint(4, 30), "poisson": True,
                      "seed": rng.randint(0, 10 ** 6)}
            elif kind == "step":
                tr = {"kind": "step", "base_rps": round(rng.uniform(0, 20), 1),
                      "step_rps": round(rng.uniform(30, 120), 1),
                      "step_window": rng.randint(1, windows)}
            else:
                tr = {"kind": "constant", "rps": round(rng.uniform(5, 80), 1), "poisson": True}
            fns.append({"function_id": fid, "profile": {"synth": synth}, "trace": tr,
                        "initial_pods": [{"sm": rng.choice(sms), "quota": 1.0}]})
        sc = {"fleet_size": rng.randint(2, 5), "windows": windows,
              "epoch_windows": rng.randint(1, 3), "cold_start_windows": rng.randint(0, 2),
              "seed": rng.randint(0, 1000), "gpu_capacity_mb": 81920.0,
              "restructure_threshold": rng.choice([2, 4, 16]), "functions": fns}
        out.append({"name": f"prefix-ids-{k:03d}", "scenario": sc, "files": {}})
    return out


def run_reference(case, policy):
    sys.path.insert(0, REF)
    import gshare_sim as ref
    from gshare_sim.sim_engine import _Engine
    with tempfile.TemporaryDirectory() as tmp:
        for fname, text in case["files"].items():
            with open(os.path.join(tmp, fname), "w") as fh:
                fh.write(text)
        try:
            sc = ref.Scenario.from_dict(json.loads(json.dumps(case["scenario"])), base_dir=tmp)
            eng = _Engine(sc, policy)
            report = eng.run()
        except ref.GShareError as exc:
            return {"error": type(exc).__name__, "message": str(exc)}
    placements = []
    for node in eng.nodes:
        for pid, p in sorted(node.placements.items()):
            r = p.rect
            placements.append([node.gpu_id, pid] + [f"{v.numerator}/{v.denominator}"
                                                    for v in (r.x, r.y, r.w, r.h)])
    return {"csv": report.to_csv(), "summary": report.summary(), "placements": placements}


def main(n_random: int = 360, seed: int = 20261017):
    rng = random.Random(seed)
    cases = bundled_cases() + engine_test_cases() + [random_case(rng, i) for i in range(n_random)]
    cases += error_branch_cases()
    cases += prefix_cases()
    records = []
    for case in cases:
        for policy in ("fast", "timeshare"):
            rec = dict(case)
            rec["policy"] = policy
            rec["expect"] = run_reference(case, policy)
            records.append(rec)
    with gzip.open(OUT, "wt", encoding="utf-8") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "seed": seed,
                   "reference": "pkg/src/gshare_sim 0.1.0", "records": records}, fh)
    n_err = sum(1 for r in records if "error" in r["expect"])
    print(f"wrote {len(records)} records ({n_err} reference errors) to {OUT}")


if __name__ == "__main__":
    main()
