"""Device packer auditor: the reference's check_node
(packer.py:327-388) as a kernel, exact on the scaled integer grid.

Handcrafted geometries pin each breach class; the session audit checks that
every run of real batches ends with a consistent packer state."""
import gzip
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                      "golden_audit.json.gz")

S = 100
FULL = (0, 0, S, S)
PLACED_OVERLAP, FREE_PLACED, FREE_CONTAINED, GAP, DOUBLE = 1, 2, 4, 8, 16


def _golden():
    with gzip.open(GOLDEN, "rt") as fh:
        return json.load(fh)["records"]


def _scaled(rec):
    """A golden geometry on its exact integer grid: (free, placed, side)."""
    rects = [[Fraction(v) for v in r] for r in rec["free"] + rec["placed"]]
    scale = 1
    for r in rects:
        for v in r:
            scale = scale * v.denominator // math.gcd(scale, v.denominator)
    ints = [tuple(int(v * scale) for v in r) for r in rects]
    nf = len(rec["free"])
    return ints[:nf], ints[nf:], 100 * scale


def _exact_audit(free, placed, side):
    """check_node's five breach classes decided exactly on the grid compressed
    to the rectangle edges (the device auditor's method, restated in Python)."""
    def inter(a, b):
        return a[0] < b[0] + b[2] and b[0] < a[0] + a[2] and a[1] < b[1] + b[3] and b[1] < a[1] + a[3]

    def contains(a, b):
        return a[0] <= b[0] and a[1] <= b[1] and b[0] + b[2] <= a[0] + a[2] and b[1] + b[3] <= a[1] + a[3]
    bits = 0
    if any(inter(a, b) for i, a in enumerate(placed) for b in placed[i + 1:]):
        bits |= PLACED_OVERLAP
    if any(inter(r, p) for r in free for p in placed):
        bits |= FREE_PLACED
    if any(i != j and contains(o, r) and not (r == o and i < j)
           for i, r in enumerate(free) for j, o in enumerate(free)):
        bits |= FREE_CONTAINED
    xs = sorted({0, side} | {v for r in free + placed for v in (r[0], r[0] + r[2])})
    ys = sorted({0, side} | {v for r in free + placed for v in (r[1], r[1] + r[3])})
    for x0, x1 in zip(xs, xs[1:]):
        for y0, y1 in zip(ys, ys[1:]):
            cell = (x0, y0, x1 - x0, y1 - y0)
            f = any(contains(r, cell) for r in free)
            p = any(contains(r, cell) for r in placed)
            if not f and not p:
                bits |= GAP
            if f and p:
                bits |= DOUBLE
    return bits


def test_golden_audit_fixtures_agree_with_an_exact_restatement():
    recs = _golden()
    assert len(recs) > 5000 and {r["bits"] for r in recs} >= {0, 1, 4, 8, 18}
    for rec in recs[::7]:
        free, placed, side = _scaled(rec)
        mask = 7 if rec["coverage_skipped"] else 31
        assert _exact_audit(free, placed, side) & mask == rec["bits"] & mask, rec["tag"]


@pytest.mark.gpu
def test_device_auditor_matches_check_node_on_reference_geometries():
    recs = _golden()
    by_side: dict = {}
    for k, rec in enumerate(recs):
        free, placed, side = _scaled(rec)
        by_side.setdefault(side, []).append((k, free, placed))
    bad = []
    for side, items in by_side.items():
        got = backend.audit_geometry([(f, p) for _, f, p in items], side, side)
        for (k, _, _), bits in zip(items, got.tolist()):
            rec = recs[k]
            mask = 7 if rec["coverage_skipped"] else 31
            if bits & mask != rec["bits"] & mask:
                bad.append(f"{rec['tag']}: device {bits} vs check_node {rec['bits']}")
    assert not bad, f"{len(bad)} of {len(recs)} differ: {bad[:5]}"


@pytest.mark.gpu
def test_geometry_cases():
    cases = [
        (([FULL], []), 0),                                        # empty node
        (([], []), GAP),                                          # nothing covers the plane
        (([(40, 0, 60, 100), (0, 30, 100, 70)], [(0, 0, 40, 30)]), 0),   # maximal split
        (([(40, 0, 60, 100)], [(0, 0, 40, 30)]), GAP),            # lost the top-left region
        (([(40, 0, 60, 100), (0, 30, 100, 70)], [(0, 0, 40, 30), (10, 10, 5, 5)]),
         PLACED_OVERLAP),
        (([FULL], [(0, 0, 40, 30)]), FREE_PLACED | DOUBLE),
        (([FULL, (0, 0, 10, 10)], []), FREE_CONTAINED),
        (([FULL, FULL], []), FREE_CONTAINED),                     # duplicate: later one
        (([(0, 0, 50, 100), (50, 0, 50, 100)], []), 0),           # two halves tile
        (([(0, 0, 60, 100), (40, 0, 60, 100)], []), 0),           # overlapping free: allowed
    ]
    got = backend.audit_geometry([c for c, _ in cases], S, S)
    want = np.array([w for _, w in cases], np.uint32)
    assert got.tolist() == want.tolist()


@pytest.mark.gpu
def test_geometry_on_a_fine_grid():
    # exact at any scale (the reference's raster gives up beyond 20x)
    side = 100 * 7919
    free = [(0, 1, side, side - 1)]
    placed = [(0, 0, side, 1)]
    assert backend.audit_geometry([(free, placed)], side, side).tolist() == [0]
    assert backend.audit_geometry([(free, [])], side, side).tolist() == [GAP]


@pytest.mark.gpu
def test_session_audit_is_clean_on_real_batches():
    scen = [Scenario.from_dict(wl.c2(s, windows=60)) for s in range(24)]
    scen += [Scenario.from_dict(wl.c3(s)) for s in range(24)]
    pols = ["fast"] * 24 + ["fast", "timeshare"] * 12
    images = [cc.compile_run(s, p) for s, p in zip(scen, pols)]
    audited = 0
    for _attempt in range(8):                 # regrow over-capacity runs, audit every run
        batch = cc.Batch(images)
        sess = backend.Session(batch)
        sess.run()
        st = sess.download(rows=False)["status"]
        ok = st["code"] == 0
        assert set(st["code"][~ok].tolist()) <= {cc.GS_ERR_CAPACITY}
        assert sess.audit()[ok].tolist() == [0] * int(ok.sum())
        sess.close()
        audited += int(ok.sum())
        retry = []
        for j in np.nonzero(~ok)[0]:
            rr = batch.runs[j]
            caps = cc.Caps(int(rr["cap_pods"]), int(rr["cap_rects"]), int(rr["cap_returned"]),
                           int(rr["hot_class"])).grown(int(st["detail"][j]),
                                                       int(st["hot_class"][j]))
            retry.append(cc.compile_run(scen[j], pols[j], caps))
        if not retry:
            break
        scen = [scen[j] for j in np.nonzero(~ok)[0]]
        pols = [pols[j] for j in np.nonzero(~ok)[0]]
        images = retry
    assert audited == 48
