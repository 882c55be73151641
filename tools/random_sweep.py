"""Large randomised GPU-vs-oracle sweep (the generator of tests/test_gpu_random_stress.py,
i.e. of the reference-pinned golden set, at longer horizons and larger fleets): every
record of every run compared.  usage: python tools/random_sweep.py [blocks] [seed0]"""
import collections
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)
from parity import diff_results, oracle_results          # noqa: E402
from paper_2309_00558_b200 import compiler as cc, engine  # noqa: E402
import test_gpu_random_stress as T                          # noqa: E402

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 20
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
scen, pols = [], []
for b in range(blocks):
    rng = random.Random(seed0 + b)
    for k in range(80):
        sc = T._load(T._scaled_case(rng, k))
        for pol in ("fast", "timeshare"):
            try:
                cc.compile_run(sc, pol)
            except Exception:
                continue
            scen.append(sc)
            pols.append(pol)
t0 = time.perf_counter()
got = engine.simulate(scen, pols, errors="return")
t1 = time.perf_counter()
want = oracle_results(scen, pols)
t2 = time.perf_counter()
bad = [(i, d) for i, d in enumerate(diff_results(x, y) for x, y in zip(got, want)) if d]
kinds = collections.Counter(type(x).__name__ if isinstance(x, Exception) else "ok" for x in want)
classes = collections.Counter()
print(json.dumps({"runs": len(scen), "blocks": blocks, "seed0": seed0, "outcomes": dict(kinds),
                  "mismatched": len(bad), "first": bad[0] if bad else None,
                  "gpu_s": round(t1 - t0, 2), "oracle_s": round(t2 - t1, 2)}))
sys.exit(1 if bad else 0)
