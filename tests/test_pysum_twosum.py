"""The kernel's PySum (csrc/gs_kernel.cuh) adds Knuth's branch-free TwoSum
error where CPython 3.12's sum() adds Neumaier's branchy Fast2Sum term
((f - t) + x if |f| >= |x| else (x - t) + f).  Both are the exact rounding
error of t = f + x for finite operands, so the compensation c -- and the
value -- are bit-identical.  Checked here in Python floats (IEEE doubles,
every operation rounded as written, like the -fmad=false build) and against
the interpreter's own sum()."""
import math
import random
import struct
import sys

import pytest


def _neumaier(xs):
    f = c = 0.0
    for k, x in enumerate(xs):
        if k == 0:
            f, c = 0.0 + x, 0.0
            continue
        t = f + x
        c += (f - t) + x if abs(f) >= abs(x) else (x - t) + f
        f = t
    return f, c


def _twosum(xs):
    f = c = 0.0
    for k, x in enumerate(xs):
        if k == 0:
            f, c = 0.0 + x, 0.0
            continue
        t = f + x
        bp = t - f
        c += (f - (t - bp)) + (x - bp)
        f = t
    return f, c


def _bits(x):
    return struct.pack("<d", x)


def _draw(rng):
    kind = rng.random()
    if kind < 0.3:
        return rng.uniform(-1e3, 1e3)
    if kind < 0.5:
        return rng.choice([1, -1]) * 10.0 ** rng.uniform(-20, 20)
    if kind < 0.7:
        return float(rng.randint(-100, 100)) * rng.choice([0.02, 0.1, 0.01, 1e-9, 1.0])
    if kind < 0.8:
        return rng.choice([0.0, -0.0, 1e-300, -1e-300, 5e-324])
    return rng.uniform(0, 1) * rng.choice([1.0, 1e-16, 1e16])


@pytest.mark.parametrize("seed", range(20))
def test_twosum_compensation_is_bit_identical(seed):
    rng = random.Random(seed)
    for _ in range(3000):
        xs = [_draw(rng) for _ in range(rng.randint(1, 40))]
        fa, ca = _neumaier(xs)
        fb, cb = _twosum(xs)
        assert _bits(fa) == _bits(fb) and _bits(ca) == _bits(cb), xs
        if sys.version_info >= (3, 12) and math.isfinite(ca):
            want = sum(xs)
            got = fb + cb if cb != 0.0 else fb
            assert _bits(got) == _bits(want) or (got == want == 0.0), xs
