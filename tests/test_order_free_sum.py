"""The integral dispatch path adds a node's occupancy terms in grant-slot
order instead of the reference's dispatch order (csrc/gs_hot.cuh, hot_step;
csrc/gs_xlh.cuh, xlh_step).  That is exact because, for terms sm * dur with an
integer sm in [1, 100], dur in (1e-9, 1] and at most 100 terms (sum of sm <=
100), CPython 3.12's compensated sum() returns the correctly rounded exact sum
of the multiset, independent of order (sim_engine.py:516-517 sums in dispatch
order).  This checks the claim against the interpreter's own sum()."""
import random
import sys

import pytest

pytestmark = pytest.mark.skipif(sys.version_info < (3, 12),
                                reason="sum() is compensated from CPython 3.12 on")


def _terms(rng):
    left, out = 100, []
    quantum = rng.choice([1.0, 0.1, 0.05, 0.04, 0.02, 0.01, 1e-3, 1e-6])
    while left > 0 and len(out) < 100:
        sm = rng.randint(1, min(left, rng.choice([1, 3, 10, 25, 50, 100])))
        left -= sm
        r = rng.random()
        if r < 0.6:
            dur = quantum
        elif r < 0.9:
            dur = rng.uniform(1e-9, quantum) * (1 + 1e-15)
        else:
            dur = max(1e-9 * (1 + rng.random()), rng.random() * 1e-6)
        dur = min(dur, quantum) if dur > 1e-9 else 1.0000001e-9
        out.append(float(sm) * dur)
    return out


@pytest.mark.parametrize("seed", range(40))
def test_sum_is_order_free_on_occupancy_terms(seed):
    rng = random.Random(seed)
    for _ in range(250):
        xs = _terms(rng)
        want = sum(xs)
        for _ in range(6):
            ys = xs[:]
            rng.shuffle(ys)
            assert sum(ys) == want, (xs, ys)
