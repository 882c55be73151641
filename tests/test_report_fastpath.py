"""the vectorised report writer (report.py) renders the same
bytes as the reference-shaped MetricsReport path, on the oracle's output
records for the golden scenarios and a mixed synthetic batch (CPU only)."""
import json

import pytest

import golden
import oracle
from paper_2309_00558_b200 import compiler as cc, engine, report, workloads as wl
from paper_2309_00558_b200.scenario import Scenario


def _batch_and_out(scen, pols):
    images = []
    for s, p in zip(scen, pols):
        try:
            images.append(cc.compile_run(s, p))
        except Exception:         # runs the reference rejects up front
            continue
    batch = cc.Batch(images)
    return batch, oracle.run_batch(batch)


def _check(batch, out):
    for r in range(len(batch)):
        if int(out["status"][r]["code"]) != cc.GS_OK:
            continue
        rep = engine.decode_run(batch, r, out).report
        assert report.run_csv(batch, out, r) == rep.to_csv(), r
        assert json.dumps(report.run_summary(batch, out, r), sort_keys=True) == \
            json.dumps(rep.summary(), sort_keys=True), r


def test_fast_report_matches_metrics_report_on_golden_scenarios():
    recs = [r for r in golden.records()[:120]]
    scen, pols = [], []
    for rec in recs:
        try:
            scen.append(golden.load_scenario(rec))
            pols.append(rec["policy"])
        except Exception:
            continue
    _check(*_batch_and_out(scen, pols))


def test_fast_report_matches_on_synthetic_workloads():
    scen = [Scenario.from_dict(wl.c3(s, windows=20)) for s in range(4)]
    scen += [Scenario.from_dict(wl.c2(s, windows=15)) for s in range(3)]
    scen += [Scenario.from_dict(wl.c1())]
    pols = ["fast", "timeshare"] * 4
    _check(*_batch_and_out(scen, pols))


def test_write_run_files(tmp_path):
    scen = [Scenario.from_dict(wl.c3(1, windows=10))]
    batch, out = _batch_and_out(scen, ["fast"])
    csv_path, json_path = report.write_run(batch, out, 0, tmp_path / "run0")
    rep = engine.decode_run(batch, 0, out).report
    rep.write(tmp_path / "ref")
    assert open(csv_path).read() == open(tmp_path / "ref" / "metrics.csv").read()
    assert open(json_path).read() == open(tmp_path / "ref" / "summary.json").read()
