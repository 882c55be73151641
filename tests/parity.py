"""GPU-vs-oracle comparison helpers (test infrastructure)."""
import numpy as np

import oracle
from paper_2309_00558_b200 import compiler as cc, engine


def oracle_results(scenarios, policies):
    images = [cc.compile_run(s, p) for s, p in zip(scenarios, policies)]
    batch = cc.Batch(images)
    out = oracle.run_batch(batch, n_threads=8)
    res = []
    for r in range(len(batch)):
        err = engine.run_error(batch.images[r], out["status"][r])
        res.append(err if err is not None else engine.decode_run(batch, r, out))
    return res


def diff_results(a, b):
    """Exact comparison of two RunResults (or exceptions); '' when equal."""
    if isinstance(a, Exception) or isinstance(b, Exception):
        if type(a) is type(b) and str(a) == str(b):
            return ""
        return f"outcome {a!r} vs {b!r}"
    ra, rb = a.report, b.report
    if ra.function_rows != rb.function_rows:
        for x, y in zip(ra.function_rows, rb.function_rows):
            if x != y:
                return f"function row {x} != {y}"
        return "function rows differ in length"
    if ra.gpu_rows != rb.gpu_rows:
        for x, y in zip(ra.gpu_rows, rb.gpu_rows):
            if x != y:
                return f"gpu row {x} != {y}"
        return "gpu rows differ in length"
    if ra.global_rows != rb.global_rows:
        for x, y in zip(ra.global_rows, rb.global_rows):
            if x != y:
                return f"global row {x} != {y}"
        return "global rows differ in length"
    if a.placements != b.placements:
        return "final placements differ"
    for f in ("token_grants", "scale_decisions", "placement_attempts", "pod_steps",
              "rect_scans", "peak_pods"):
        if getattr(a, f) != getattr(b, f):
            return f"{f} {getattr(a, f)} != {getattr(b, f)}"
    if a.summary.tobytes() != b.summary.tobytes():
        return f"summary {a.summary} != {b.summary}"
    return ""


def assert_gpu_matches_oracle(scenarios, policies):
    got = engine.simulate(scenarios, policies, errors="return")
    want = oracle_results(scenarios, policies)
    bad = [(i, d) for i, d in enumerate(diff_results(x, y) for x, y in zip(got, want)) if d]
    assert not bad, f"{len(bad)} of {len(got)} runs differ; first: run {bad[0][0]}: {bad[0][1]}"
    return got
