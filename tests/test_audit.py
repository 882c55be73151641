"""Device packer auditor: the reference's check_node
(packer.py:327-388) as a kernel, exact on the scaled integer grid.

Handcrafted geometries pin each breach class; the session audit checks that
every run of real batches ends with a consistent packer state."""
import numpy as np
import pytest

from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario

pytestmark = pytest.mark.gpu

S = 100
FULL = (0, 0, S, S)
PLACED_OVERLAP, FREE_PLACED, FREE_CONTAINED, GAP, DOUBLE = 1, 2, 4, 8, 16


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


def test_geometry_on_a_fine_grid():
    # exact at any scale (the reference's raster gives up beyond 20x)
    side = 100 * 7919
    free = [(0, 1, side, side - 1)]
    placed = [(0, 0, side, 1)]
    assert backend.audit_geometry([(free, placed)], side, side).tolist() == [0]
    assert backend.audit_geometry([(free, [])], side, side).tolist() == [GAP]


def test_session_audit_is_clean_on_real_batches():
    scen = [Scenario.from_dict(wl.c2(s, windows=60)) for s in range(24)]
    scen += [Scenario.from_dict(wl.c3(s)) for s in range(24)]
    pols = ["fast"] * 24 + ["fast", "timeshare"] * 12
    batch = cc.Batch([cc.compile_run(s, p) for s, p in zip(scen, pols)])
    sess = backend.Session(batch)
    sess.run()
    st = sess.download(rows=False)["status"]
    ok = st["code"] == 0              # (capacity overflows are retried by the engine)
    assert ok.sum() >= len(batch) - 4
    assert sess.audit()[ok].tolist() == [0] * int(ok.sum())
    sess.close()
