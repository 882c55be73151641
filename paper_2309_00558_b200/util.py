"""Number rendering shared by the CSV/summary writers.

Same contract as the reference's ``fmt_num`` (pkg/src/gshare_sim/util.py:4-10):
integral values below 1e15 print without a decimal point, all others as the
shortest round-tripping ``repr``.
"""
import math


def fmt_num(value) -> str:
    x = float(value)
    integral = math.isfinite(x) and x == math.floor(x)
    if integral and abs(x) < 1e15:
        return str(int(x))
    return repr(x)
