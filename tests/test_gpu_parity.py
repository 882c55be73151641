"""GPU parity: the sm_100a kernel, called through the C ABI, against
(1) the reference's own golden outputs and (2) the CPU oracle at full sizes.

Bit-exact on every record: per-window function rows (arrivals, completions,
SLO violations, drops, queue depth), GPU rows (utilisation, occupancy,
memory -- bitwise doubles, i.e. a 0 ulp tolerance, tighter than north_star's
1e-6 relative), global rows (GPUs in use, placement failures, fragmentation),
final placements, decision counters and the all-gather summary records.
"""
import numpy as np
import pytest

import golden
import oracle
from parity import assert_gpu_matches_oracle, diff_results, oracle_results
from paper_2309_00558_b200 import backend, compiler as cc, engine, workloads as wl
from paper_2309_00558_b200.scenario import Scenario

pytestmark = pytest.mark.gpu


def _outcomes_on_gpu(recs):
    scen, pols, pre = [], [], {}
    for k, rec in enumerate(recs):
        try:
            scen.append(golden.load_scenario(rec))
            pols.append(rec["policy"])
        except Exception as exc:
            pre[k] = exc
    res = engine.simulate(scen, pols, errors="return")
    it = iter(res)
    return [pre[k] if k in pre else next(it) for k in range(len(recs))]


def test_gpu_matches_reference_golden_runs():
    recs = golden.records()
    outcomes = _outcomes_on_gpu(recs)
    bad = []
    for rec, out in zip(recs, outcomes):
        errs = golden.compare(rec, out)
        if errs:
            bad.append(f"{rec['name']}/{rec['policy']}: {errs[0][:400]}")
    assert not bad, f"{len(bad)} of {len(recs)} differ:\n" + "\n".join(bad[:5])


@pytest.mark.parametrize("policy", ["fast", "timeshare"])
def test_gpu_matches_oracle_c2(policy):
    scen = [Scenario.from_dict(wl.c2(s, windows=120)) for s in range(48)]
    assert_gpu_matches_oracle(scen, [policy] * len(scen))


def test_gpu_matches_oracle_c3_both_policies():
    scen = [Scenario.from_dict(wl.c3(s)) for s in range(96)]
    assert_gpu_matches_oracle([x for x in scen for _ in (0, 1)], ["fast", "timeshare"] * 96)


def test_gpu_matches_oracle_c5_sweep_sample():
    scen = [Scenario.from_dict(wl.c5(i)) for i in range(0, 3500, 7)]
    assert_gpu_matches_oracle(scen, ["fast"] * len(scen))


def test_gpu_c1_full_length():
    sc = Scenario.from_dict(wl.c1())
    assert_gpu_matches_oracle([sc, sc], ["fast", "timeshare"])


def test_capacity_overflow_is_retried_not_truncated():
    sc = Scenario.from_dict(wl.c2(3, windows=40))
    tiny = cc.Caps(pods=8, rects=4, returned=1)
    image = cc.compile_run(sc, "fast", tiny)
    batch = cc.Batch([image])
    out = backend.run_batch(batch)
    assert int(out["status"][0]["code"]) == cc.GS_ERR_CAPACITY
    # the public API grows the capacities on the device until the run fits
    res = engine.simulate([sc], ["fast"], caps=tiny)[0]
    ref_batch = cc.Batch([cc.compile_run(sc, "fast")])
    want = engine.decode_run(ref_batch, 0, oracle.run_batch(ref_batch))
    assert diff_results(res, want) == ""


def test_gpu_matches_oracle_c4_large_fleet():
    # 64 nodes x 200 functions (BASELINE configs[3]): the HBM-arena (XL) path
    scen = [Scenario.from_dict(wl.c4(s, windows=40)) for s in range(3)]
    assert_gpu_matches_oracle(scen, ["fast"] * len(scen))


def test_gpu_matches_oracle_c4_full_day():
    # C4 at its full horizon (one compressed day, W=3600; sinusoid period = W):
    # many epochs on the CTA-wide epoch / placement path, plus a timeshare run
    scen = [Scenario.from_dict(wl.c4(s, windows=3600)) for s in range(2)]
    scen += [Scenario.from_dict(wl.c4(7, windows=60))]
    assert_gpu_matches_oracle(scen, ["fast", "fast", "timeshare"])


def test_gpu_matches_oracle_c2_timeshare_and_mixed_classes():
    # one batch mixing every size class the launcher dispatches (XS/S/M/L/XL)
    scen = [Scenario.from_dict(wl.c2(s, windows=30, n_funcs=3, fleet=2)) for s in range(2)]
    scen += [Scenario.from_dict(wl.c2(s, windows=30)) for s in range(6)]
    scen += [Scenario.from_dict(wl.c2(s, windows=30, n_funcs=20, fleet=8)) for s in range(4)]
    scen += [Scenario.from_dict(wl.c2(s, windows=20, n_funcs=48, fleet=24)) for s in range(2)]
    scen += [Scenario.from_dict(wl.c4(s, windows=12, n_funcs=80, fleet=40)) for s in range(2)]
    pols = ["fast", "timeshare"] * 8
    assert_gpu_matches_oracle(scen, pols)


def test_pipelined_run_batch_matches_oracle_reports():
    """The drop-in batch API lowers and simulates in overlapping blocks
    (engine.simulate_records: compile_stream + concurrent stream-ordered
    one-shot calls): every MetricsReport's CSV and summary equal the oracle's,
    and a run with a mid-run ValidationError (a zero-throughput CSV profile,
    autoscaler.py:115-117) comes back as that error in its input position."""
    from paper_2309_00558_b200.metrics import MetricsReport
    scen = ([Scenario.from_dict(wl.c2(s, windows=40)) for s in range(300)]
            + [Scenario.from_dict(wl.c3(s, windows=30)) for s in range(150)]
            + [Scenario.from_dict(wl.c5(i)) for i in range(0, 1500, 7)])
    pols = ["fast"] * 300 + ["fast", "timeshare"] * 75 + ["fast"] * (len(scen) - 450)
    bad = [r for r in golden.records() if "no profiled point has positive throughput"
           in str(r["expect"].get("message", ""))]
    assert bad, "golden set lost its zero-throughput error records"
    scen.insert(333, golden.load_scenario(bad[0]))
    pols.insert(333, bad[0]["policy"])
    reps = engine.run_batch(scen, pols, errors="return")
    want = oracle_results(scen, pols)
    assert len(reps) == len(want) == len(scen)
    for k, (got, ref) in enumerate(zip(reps, want)):
        if isinstance(ref, Exception):
            assert type(got) is type(ref) and str(got) == str(ref), k
            continue
        assert isinstance(got, MetricsReport), (k, got)
        assert got.to_csv() == ref.report.to_csv(), k
        assert got.summary() == ref.report.summary(), k
