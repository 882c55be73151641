"""Host fast path, CPU only: the parallel batch compiler,
the native CSV / number renderer (csrc/gs_host.cpp, called through the C
ABI without a GPU) and the lazy DeviceReport, each against the plain Python
path it replaces.  Device outputs are produced by the oracle here."""
import pickle
import random
import struct

import numpy as np
import pytest

import golden
import oracle
from paper_2309_00558_b200 import compiler as cc, engine, report, workloads as wl
from paper_2309_00558_b200.errors import ValidationError
from paper_2309_00558_b200.metrics import MetricsReport
from paper_2309_00558_b200.scenario import Scenario
from paper_2309_00558_b200.util import fmt_num


def _values():
    rng = random.Random(7)
    v = [rng.random() for _ in range(4000)]
    v += [rng.random() * 10 ** rng.randint(-25, 25) for _ in range(4000)]
    v += [struct.unpack("d", struct.pack("Q", rng.getrandbits(64)))[0] for _ in range(4000)]
    v += [2.0 ** k for k in range(-1074, 1024, 3)] + [-(2.0 ** k) for k in range(-60, 60)]
    v += [k / 1e9 + 5e-10 for k in range(2000)] + [k / 1e6 + 5e-7 for k in range(2000)]
    v += [0.0, -0.0, 1e15, 1e16, 999999999999999.9, 1e-4, 1e-5, 0.5, 2.5, 1.0 / 3,
          float("inf"), -float("inf"), float("nan"), 5e-324, 1.7976931348623157e308]
    return v


@pytest.mark.parametrize("nd", [9, 6, -1])
def test_native_numbers_match_the_interpreter(nd):
    vals = _values()
    got = report.format_numbers(vals, nd)
    want = [fmt_num(round(x, nd) if nd >= 0 else x) for x in vals]
    bad = [(x, g, w) for x, g, w in zip(vals, got, want) if g != w]
    assert not bad, bad[:5]


def _oracle_batch(scen, pols):
    batch, index, errors = cc.compile_batch(scen, pols)
    assert not errors
    return batch, oracle.run_batch(batch, n_threads=4)


def test_native_csv_matches_metrics_report_on_goldens():
    recs = [r for r in golden.records() if "error" not in r["expect"]][:200]
    scen = [golden.load_scenario(r) for r in recs]
    batch, out = _oracle_batch(scen, [r["policy"] for r in recs])
    texts = report.csv_texts(batch, out)
    sums = report.summaries(batch, out)
    for j, rec in enumerate(recs):
        assert texts[j] == rec["expect"]["csv"], rec["name"]
        assert sums[j] == rec["expect"]["summary"], rec["name"]


def test_native_csv_quotes_function_ids_like_csv_writer():
    d = wl.c2(3, windows=12, n_funcs=3, fleet=2)
    for fn, fid in zip(d["functions"], ['a,b', 'q"x', 'café']):
        fn["function_id"] = fid
    sc = Scenario.from_dict(d)
    batch, out = _oracle_batch([sc, sc], ["fast", "timeshare"])
    for j in range(2):
        want = engine.decode_run(batch, j, out).report
        assert report.csv_texts(batch, out, range(j, j + 1))[0] == want.to_csv()


def test_device_report_is_a_lazy_metrics_report():
    scen = [Scenario.from_dict(wl.c3(s, windows=30)) for s in range(6)]
    pols = ["fast", "timeshare"] * 3
    batch, out = _oracle_batch(scen, pols)
    sh = report.SharedOutputs(batch, out)
    for j in range(len(batch)):
        want = engine.decode_run(batch, j, out).report
        lazy = report.DeviceReport(sh, j)
        assert isinstance(lazy, MetricsReport) and lazy._rows is None
        assert lazy.to_csv() == want.to_csv()
        s1 = lazy.summary()
        s1["policy"] = "mutated"                       # callers own the dict
        assert lazy.summary() == want.summary()
        assert lazy._rows is None                      # nothing materialised so far
        assert lazy == want and want == lazy
        assert lazy.function_rows == want.function_rows
        plain = pickle.loads(pickle.dumps(lazy))
        assert type(plain) is MetricsReport and plain == want
        # editing materialised rows is honoured by the inherited renderers
        lazy.function_rows.pop()
        assert lazy.to_csv() == MetricsReport(lazy.policy, lazy.function_rows,
                                              lazy.gpu_rows, lazy.global_rows).to_csv()
        assert lazy != want


def test_compile_batch_pool_matches_serial_compile():
    seq = wl.ScenarioSeq(lambda i: wl.c5(i * 37), 600)
    pols = ["fast"] * 600
    pooled, idx, err = cc.compile_batch(seq, pols, workers=4)
    serial = cc.Batch([cc.compile_run(seq[i], "fast") for i in range(600)])
    assert idx == list(range(600)) and not err
    for name in cc.SCENARIO_DT.names:
        assert np.array_equal(pooled.runs[name], serial.runs[name]), name
    assert np.array_equal(pooled.counts, serial.counts)
    for f in range(len(serial.funcs)):                 # point blocks are deduplicated
        a, b = pooled.funcs[f], serial.funcs[f]
        n = int(b["n_points"])
        assert pooled.points[a["point_off"]: a["point_off"] + n].tobytes() == \
            serial.points[b["point_off"]: b["point_off"] + n].tobytes()
    assert len(pooled.points) == len(serial.points)       # deduplicated across parts too
    assert pooled.names.tobytes() == serial.names.tobytes()
    o1 = oracle.run_batch(pooled.prefix(60), n_threads=4)
    o2 = oracle.run_batch(serial.prefix(60), n_threads=4)
    for k in ("fn_rows", "gpu_rows", "glob_rows", "summary"):
        n = len(o2[k]) if k == "summary" else None
        assert o1[k][:n].tobytes() == o2[k][:n].tobytes(), k


def test_compile_batch_reports_errors_in_input_order():
    good = Scenario.from_dict(wl.c1())
    bad = Scenario.from_dict(wl.c1())
    bad.functions[0].initial_pods.append(type(bad.functions[0].initial_pods[0])(
        type(bad.functions[0].initial_pods[0].point)(13.0, 0.4), None))
    seq = [good] * 300 + [bad] + [good] * 50
    batch, idx, err = cc.compile_batch(seq, ["fast"] * len(seq), workers=3)
    assert list(err) == [300] and isinstance(err[300], ValidationError)
    assert "is not profiled" in str(err[300])
    assert len(batch) == 350 and idx == list(range(300)) + list(range(301, 351))
    with pytest.raises(ValueError):
        cc.Batch([batch.images[0]])                    # packed images carry no counts


def test_pod_order_keys_follow_pod_id_string_order():
    """Pod ids f"{fid}-{n:04d}" with ids extending other ids with '-': the
    device's (slot, digits) key must sort exactly like the strings."""
    rng = random.Random(11)
    fams = [["x", "x-1", "x-1-2", "x-10", "x-0100", "x-a", "x-", "x--1", "x-1a", "x-005",
             "x-01a", "x-0", "x-00", "y", "x-99999999999", "x-1234567890a"],
            ["1", "1-0", "1-007", "1-007-0", "10", "1-", "1-+", "1- "],
            ["a", "a+", "a-b", "a-b-c", "a-bc", "é", "a-é", "a-9z"]]
    for fam in fams:
        for _ in range(30):
            fids = rng.sample(fam, rng.randint(1, len(fam)))
            order = cc._pod_id_order(fids)
            pods = [(f, n) for f in fids for n in rng.sample(range(0, 200000), 60)
                    + list(range(0, 120, 7)) + [999, 1000, 1999, 9999, 10000, 99999]]
            by_str = sorted(pods, key=lambda p: f"{p[0]}-{p[1]:04d}")
            by_key = sorted(pods, key=lambda p: cc.pod_order_key(order, p[0], p[1]))
            assert by_str == by_key, fids


def test_vector_poisson_draw_equals_the_scalar_loop():
    """traces.py draws a trace's Poisson counts as one vector; the reference
    draws one scalar per window (traces.py:40-42 of pkg/src).  Same stream."""
    from paper_2309_00558_b200.traces import _rates_to_counts
    rng = random.Random(5)
    for _ in range(200):
        seed = rng.randint(0, 10 ** 9)
        rates = [max(0.0, rng.uniform(-5, 200)) if rng.random() < 0.9 else 0.0
                 for _ in range(rng.randint(0, 400))]
        ws = rng.choice([1.0, 0.5, 0.25, 2.0, 0.1])
        gen = np.random.default_rng(seed)
        want = [int(gen.poisson(max(r, 0.0) * ws)) for r in rates]
        got = _rates_to_counts(rates, ws, True, seed)
        assert [int(x) for x in got] == want


def test_constant_rate_poisson_draw_equals_the_scalar_loop():
    """A constant-rate trace is drawn as poisson(lam, size=W): the same stream
    as the reference's one scalar draw per window (traces.py:40-42 of pkg/src)."""
    from paper_2309_00558_b200.traces import _rates_to_counts, constant_trace
    rng = random.Random(11)
    for _ in range(300):
        seed = rng.randint(0, 10 ** 9)
        r = rng.choice([0.0, -0.0, rng.uniform(0, 1), rng.uniform(0, 300), 1e-12])
        n = rng.randint(0, 400)
        ws = rng.choice([1.0, 0.5, 0.25, 2.0, 0.1])
        gen = np.random.default_rng(seed)
        want = [int(gen.poisson(max(r, 0.0) * ws)) for _ in range(n)]
        assert [int(x) for x in _rates_to_counts([r] * n, ws, True, seed)] == want
        if n:
            assert list(constant_trace(abs(r), n, ws, True, seed).counts) == \
                [int(gen2) for gen2 in np.random.default_rng(seed).poisson(
                    [max(abs(r), 0.0) * ws] * n)]


@pytest.mark.parametrize("parts,workers", [(1, 4), (3, 2), (8, 4), (5, 1)])
def test_compile_stream_blocks_concatenate_to_compile_batch(parts, workers):
    """engine.simulate_records streams the batch in blocks (compiler.compile_stream):
    the blocks are consecutive, carry absolute input positions, report the same
    errors as compile_batch and hold byte-identical run images."""
    good = [wl.ScenarioSeq(lambda i: wl.c5(i * 11), 400)[i] for i in range(400)]
    bad = Scenario.from_dict(wl.c1())
    bad.functions[0].initial_pods.append(type(bad.functions[0].initial_pods[0])(
        type(bad.functions[0].initial_pods[0].point)(13.0, 0.4), None))
    seq = good[:150] + [bad] + good[150:]
    pols = ["fast"] * len(seq)
    ref, ref_idx, ref_err = cc.compile_batch(seq, pols, workers=workers)
    blocks = list(cc.compile_stream(seq, pols, workers=workers, parts=parts))
    assert len(blocks) == parts
    idx = [i for _, ix, _ in blocks for i in ix]
    err = {k: v for _, _, e in blocks for k, v in e.items()}
    assert idx == ref_idx and list(err) == list(ref_err) == [150]
    assert str(err[150]) == str(ref_err[150])
    joined = cc.Batch.concat([b for b, _, _ in blocks])
    for name in ("runs", "funcs", "counts", "inits", "names", "id_splits"):
        got, want = getattr(joined, name), getattr(ref, name)
        if name == "inits":                        # a trailing pad record is optional
            got, want = got[:joined.n_inits], want[:ref.n_inits]
        assert len(got) == len(want), name
        if got.dtype.names is None:
            assert np.array_equal(got, want), name
            continue
        for field in got.dtype.names:              # field by field (struct padding is undefined)
            if name == "funcs" and field == "point_off":
                continue                           # deduplicated point blocks: offsets may differ
            assert np.array_equal(got[field], want[field]), (name, field)
