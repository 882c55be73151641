"""The CPU oracle is pinned to the real reference.

tests/golden/golden_runs.json.gz holds the reference's own outputs (made by
tests/golden/make_golden.py, which imports pkg/src/gshare_sim) for the
bundled scenarios, the engine-test scenarios and a 360-scenario random sweep,
under both policies.  Every record must match byte for byte: metrics CSV,
summary, final placements, or the exact exception text.
"""
import numpy as np
import pytest

import golden
import oracle
from paper_2309_00558_b200 import compiler as cc
from paper_2309_00558_b200.engine import decode_run, run_error


def oracle_outcome(rec, n_threads=1):
    try:
        sc = golden.load_scenario(rec)
        batch = cc.Batch([cc.compile_run(sc, rec["policy"])])
    except Exception as exc:          # host-side validation, same as the reference
        return exc
    out = oracle.run_batch(batch, n_threads=n_threads)
    err = run_error(batch.images[0], out["status"][0])
    return err if err is not None else decode_run(batch, 0, out)


@pytest.mark.parametrize("idx", range(0, len(golden.records())))
def test_oracle_matches_reference(idx):
    rec = golden.records()[idx]
    assert golden.compare(rec, oracle_outcome(rec)) == []


def test_golden_covers_the_engine_branches():
    recs = golden.records()
    names = {r["name"] for r in recs}
    assert {"bundled-steady", "bundled-step", "bundled-consolidation"} <= names
    errors = [r for r in recs if "error" in r["expect"]]
    assert any("timeshare policy needs" in r["expect"]["message"] for r in errors)
    assert any("zero serving rate" in r["expect"]["message"] for r in errors)
    ok = [r for r in recs if "error" not in r["expect"]]
    assert sum(1 for r in ok if r["expect"]["summary"]["placement_failures"] > 0) > 20
    assert any(f["dropped"] > 0 for r in ok for f in r["expect"]["summary"]["per_function"].values())


def test_struct_layout_matches_c_header():
    for name, size in cc.STRUCT_SIZES.items():
        assert oracle.sizeof(name) == size, name


def test_threaded_oracle_is_deterministic():
    recs = [r for r in golden.records() if "error" not in r["expect"]][:40]
    images = [cc.compile_run(golden.load_scenario(r), r["policy"]) for r in recs]
    batch = cc.Batch(images)
    a = oracle.run_batch(batch, n_threads=1)
    b = oracle.run_batch(batch, n_threads=4)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    for i, rec in enumerate(recs):
        assert golden.compare(rec, decode_run(batch, i, a)) == []
