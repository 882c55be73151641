"""``gshare-b200``: the reference CLI's simulation commands on the CUDA backend.

SURVEY §8(f)3.  ``run`` and ``compare`` mirror ``gshare run|compare``
(reference cli.py:84-122, 162-212): same arguments, same stdout (the summary
JSON / the policy table), same files (``metrics.csv`` + ``summary.json``), same
exit codes (0 ok, 1 ``GShareError``/``OSError``, 2 ``InvariantError``;
cli.py:42-44, 213-227).  ``sweep`` is the batched form the GPU is for: one
scenario file, many seeds (and/or both policies) simulated in one launch,
per-run reports written through the fast path (report.py) and an aggregate
table printed.  ``--backend`` accepts only ``cuda``: there is no CPU fallback.

``profile-check`` and ``pack-trace`` are host-side tools of the reference that
sit outside the simulated hot path (out of scope).

Usage: ``python -m paper_2309_00558_b200.cli run --scenario s.json [--policy P] [--out D]``
"""
from __future__ import annotations

import argparse
import json
import logging
import os
import sys
import time

from .errors import GShareError, InvariantError
from .scenario import POLICIES, Scenario

EXIT_OK = 0
EXIT_ERROR = 1
EXIT_INVARIANT = 2


def _load_scenario(path: str, seed: int | None = None) -> Scenario:
    if seed is None:
        return Scenario.from_json(path)
    with open(path, encoding="utf-8") as fh:
        data = json.load(fh)
    data["seed"] = seed
    return Scenario.from_dict(data, base_dir=os.path.dirname(os.path.abspath(path)))


def _summary_table(summaries: dict) -> str:
    """The reference's comparison table (cli.py:97-110)."""
    fields = ("gpus_used_peak", "mean_utilization", "mean_sm_occupancy",
              "slo_violation_pct", "placement_failures")
    names = sorted(summaries)
    width = max(len(f) for f in fields)
    lines = [" " * width + "  " + "  ".join(f"{n:>12}" for n in names)]
    for f in fields:
        cells = []
        for n in names:
            value = summaries[n][f]
            cells.append(f"{value:>12.4f}" if isinstance(value, float) else f"{value:>12}")
        lines.append(f"{f:<{width}}  " + "  ".join(cells))
    return "\n".join(lines)


def cmd_run(args) -> int:
    from .engine import run
    scenario = _load_scenario(args.scenario, args.seed)
    report = run(scenario, policy=args.policy)
    summary = report.summary()
    if args.out:
        report.write(args.out)
        print(f"wrote {os.path.join(args.out, 'metrics.csv')}")
        print(f"wrote {os.path.join(args.out, 'summary.json')}")
    print(json.dumps(summary, indent=2, sort_keys=True))
    return EXIT_OK


def cmd_compare(args) -> int:
    from .engine import compare_policies
    scenario = Scenario.from_json(args.scenario)
    reports = compare_policies(scenario)
    summaries = {policy: report.summary() for policy, report in reports.items()}
    print(_summary_table(summaries))
    if args.out:
        for policy, report in sorted(reports.items()):
            out_dir = os.path.join(args.out, policy)
            report.write(out_dir)
            print(f"wrote {os.path.join(out_dir, 'metrics.csv')}")
    return EXIT_OK


def _parse_seeds(text: str) -> list:
    seeds = []
    for part in text.split(","):
        if ":" in part:
            lo, hi = part.split(":")
            seeds.extend(range(int(lo), int(hi)))
        elif part:
            seeds.append(int(part))
    if not seeds:
        raise GShareError("--seeds selects no seed")
    return seeds


def cmd_sweep(args) -> int:
    """Many seeds x policies of one scenario file in one GPU batch."""
    from . import engine, report as fast
    seeds = _parse_seeds(args.seeds)
    policies = list(POLICIES) if args.policy == "both" else [args.policy]
    with open(args.scenario, encoding="utf-8") as fh:
        data = json.load(fh)
    base = os.path.dirname(os.path.abspath(args.scenario))
    t0 = time.perf_counter()
    scen, pols, keys = [], [], []
    for s in seeds:
        d = dict(data)
        d["seed"] = s
        sc = Scenario.from_dict(d, base_dir=base)
        for p in policies:
            scen.append(sc)
            pols.append(p)
            keys.append((s, p))
    t1 = time.perf_counter()
    results = engine.simulate_records(scen, pols, device=args.device, errors="return")
    t2 = time.perf_counter()
    agg: dict = {p: {"runs": 0, "errors": 0, "gpus_used_peak": 0, "mean_utilization": 0.0,
                     "mean_sm_occupancy": 0.0, "slo_violation_pct": 0.0,
                     "placement_failures": 0} for p in policies}
    lines = []
    for (s, p), res in zip(keys, results):
        a = agg[p]
        if isinstance(res, Exception):
            a["errors"] += 1
            lines.append({"seed": s, "policy": p, "error": f"{type(res).__name__}: {res}"})
            continue
        summ = fast.run_summary(*res)
        a["runs"] += 1
        a["gpus_used_peak"] = max(a["gpus_used_peak"], summ["gpus_used_peak"])
        a["placement_failures"] += summ["placement_failures"]
        for k in ("mean_utilization", "mean_sm_occupancy", "slo_violation_pct"):
            a[k] += summ[k]
        lines.append({"seed": s, "policy": p, "summary": summ})
        if args.out:
            fast.write_run(*res, os.path.join(args.out, p, f"seed-{s}"))
    for p, a in agg.items():
        for k in ("mean_utilization", "mean_sm_occupancy", "slo_violation_pct"):
            a[k] = a[k] / a["runs"] if a["runs"] else 0.0
    print(_summary_table(agg))
    sim_s = sum(sc.windows * sc.window_ms / 1000.0 for sc in scen)
    print(f"{len(scen)} runs, {sim_s:.0f} simulated scenario-seconds: build {t1 - t0:.2f} s, "
          f"simulate+decode {t2 - t1:.2f} s", file=sys.stderr)
    if args.out:
        os.makedirs(args.out, exist_ok=True)
        path = os.path.join(args.out, "sweep.jsonl")
        with open(path, "w", encoding="utf-8") as fh:
            for rec in lines:
                fh.write(json.dumps(rec, sort_keys=True) + "\n")
        print(f"wrote {path}")
    bad = sum(a["errors"] for a in agg.values())
    return EXIT_ERROR if bad and args.strict else EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="gshare-b200",
                                     description="GPU-sharing scheduler simulator (B200 backend)")
    parser.add_argument("--verbose", action="store_true", help="debug logging")
    parser.add_argument("--backend", choices=("cuda",), default="cuda",
                        help="execution backend (the CUDA library; no CPU fallback)")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("run", help="simulate one scenario")
    p.add_argument("--scenario", required=True, help="scenario JSON file")
    p.add_argument("--policy", choices=POLICIES, default="fast")
    p.add_argument("--out", help="directory for metrics.csv / summary.json")
    p.add_argument("--seed", type=int, default=None, help="override the scenario's RNG seed")
    p.set_defaults(func=cmd_run)

    p = sub.add_parser("compare", help="run a scenario under both policies")
    p.add_argument("--scenario", required=True, help="scenario JSON file")
    p.add_argument("--out", help="directory for per-policy metrics")
    p.set_defaults(func=cmd_compare)

    p = sub.add_parser("sweep", help="many seeds of one scenario in one GPU batch")
    p.add_argument("--scenario", required=True, help="scenario JSON file")
    p.add_argument("--seeds", default="0:64", help="seed list / ranges, e.g. 0:1000,2000")
    p.add_argument("--policy", choices=POLICIES + ("both",), default="fast")
    p.add_argument("--out", help="directory for per-run reports + sweep.jsonl")
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--strict", action="store_true", help="exit 1 if any run failed")
    p.set_defaults(func=cmd_sweep)
    return parser


def main(argv: list | None = None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    logging.basicConfig(level=logging.DEBUG if args.verbose else logging.WARNING,
                        format="%(levelname)s %(name)s: %(message)s")
    try:
        return args.func(args)
    except InvariantError as exc:
        print(f"invariant breach: {exc}", file=sys.stderr)
        return EXIT_INVARIANT
    except GShareError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_ERROR
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_ERROR


if __name__ == "__main__":
    sys.exit(main())
