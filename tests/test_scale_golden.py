"""Parity at BASELINE scale, pinned to the REAL reference.

tests/golden/golden_scale.json.gz (made by tests/golden/make_scale_golden.py,
which runs pkg/src/gshare_sim) holds the reference's metrics-CSV digest,
summary and final placements for the benchmark's own shapes: C1 (both
policies), C2 at 300 windows (16 seeds fast + 4 timeshare), C3 (32 seeds x
both policies), C4 (64 nodes x 200 functions at 30/60/150 windows, fast and
timeshare) and 64 points of the C5 (SM%, quantum, SLO) grid.

The CPU test pins the oracle to them; the GPU test runs all of them in one
batch through the C ABI (every size class the launcher dispatches) and
requires byte-identical CSVs, summaries and placements.
"""
import pytest

import golden
import oracle
from paper_2309_00558_b200 import compiler as cc, engine
from paper_2309_00558_b200.engine import decode_run, run_error


def _oracle_outcomes(recs):
    scen = [golden.scale_scenario(r) for r in recs]
    batch = cc.Batch([cc.compile_run(s, r["policy"]) for s, r in zip(scen, recs)])
    out = oracle.run_batch(batch, n_threads=8)
    res = []
    for j in range(len(batch)):
        err = run_error(batch.images[j], out["status"][j])
        res.append(err if err is not None else decode_run(batch, j, out))
    return res


def test_scale_goldens_cover_every_config():
    recs = golden.scale_records()
    by = {}
    for r in recs:
        by.setdefault((r["config"], r["policy"]), 0)
        by[(r["config"], r["policy"])] += 1
    assert by[("c2", "fast")] >= 8 and by[("c3", "fast")] >= 16 and by[("c3", "timeshare")] >= 16
    assert by[("c4", "fast")] >= 2 and by[("c4", "timeshare")] >= 1 and by[("c5", "fast")] >= 32
    assert all(r["args"].get("windows", 300) == 300 for r in recs if r["config"] == "c2")


@pytest.mark.parametrize("config", ["c1", "c2", "c3", "c4", "c5"])
def test_oracle_matches_reference_at_scale(config):
    recs = [r for r in golden.scale_records() if r["config"] == config]
    bad = []
    for rec, out in zip(recs, _oracle_outcomes(recs)):
        errs = golden.scale_compare(rec, out)
        if errs:
            bad.append(f"{rec['config']}{rec['args']}/{rec['policy']}: {errs}")
    assert not bad, "\n".join(bad[:5])


@pytest.mark.gpu
def test_gpu_matches_reference_at_scale():
    recs = golden.scale_records()
    scen = [golden.scale_scenario(r) for r in recs]
    got = engine.simulate(scen, [r["policy"] for r in recs], errors="return")
    bad = []
    for rec, out in zip(recs, got):
        errs = golden.scale_compare(rec, out)
        if errs:
            bad.append(f"{rec['config']}{rec['args']}/{rec['policy']}: {errs}")
    assert not bad, f"{len(bad)} of {len(recs)} differ:\n" + "\n".join(bad[:5])
