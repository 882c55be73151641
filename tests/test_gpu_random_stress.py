"""Randomised GPU-vs-oracle stress at sizes beyond the golden set.

The oracle is pinned to the real reference on 742 golden records
(test_oracle_golden.py); here it checks the CUDA path on fresh random
scenarios drawn from the same generator as the golden set (every engine
branch: CSV profiles with zero-throughput points, fractional SM partitions,
bounded queues, restructure, memory-gated placement, both policies), but with
longer horizons and larger fleets, so the shared-memory size classes, the
class-overflow retry and the XL path all see them.
"""
import json
import os
import random
import sys
import tempfile

import pytest

from parity import diff_results, oracle_results
from paper_2309_00558_b200 import compiler as cc, engine
from paper_2309_00558_b200.scenario import Scenario

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import make_golden  # noqa: E402  (scenario generator only; the reference is not imported)

pytestmark = pytest.mark.gpu


def _scaled_case(rng, idx):
    case = make_golden.random_case(rng, idx)
    sc = case["scenario"]
    sc["windows"] = rng.randint(20, 90)
    sc["fleet_size"] = rng.choice([1, 2, 4, 6, 8])
    for fn in sc["functions"]:
        t = fn["trace"]
        if t["kind"] == "explicit":
            t["counts"] = [rng.choice([0, rng.randint(0, 20), rng.randint(10, 90)])
                           for _ in range(sc["windows"])]
        if t["kind"] == "sinusoid":
            t["period_windows"] = rng.randint(1, sc["windows"])
    return case


def _load(case):
    with tempfile.TemporaryDirectory() as tmp:
        for fname, text in case["files"].items():
            with open(os.path.join(tmp, fname), "w") as fh:
                fh.write(text)
        return Scenario.from_dict(json.loads(json.dumps(case["scenario"])), base_dir=tmp)


@pytest.mark.parametrize("block", range(4))
def test_gpu_matches_oracle_on_random_scenarios(block):
    rng = random.Random(1000 + block)
    scen, pols = [], []
    for k in range(80):
        sc = _load(_scaled_case(rng, k))
        for pol in ("fast", "timeshare"):
            try:
                cc.compile_run(sc, pol)          # the reference rejects some up front
            except Exception:
                continue
            scen.append(sc)
            pols.append(pol)
    got = engine.simulate(scen, pols, errors="return")
    want = oracle_results(scen, pols)
    bad = [(i, d) for i, d in enumerate(diff_results(x, y) for x, y in zip(got, want)) if d]
    assert not bad, f"{len(bad)} of {len(got)} runs differ; first: run {bad[0][0]}: {bad[0][1]}"
