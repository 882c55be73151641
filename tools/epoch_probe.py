"""Probe: cost of the epoch/window code in isolation -- C2 with one quantum
step per window (quantum=1.0) vs the default 50.  usage: python tools/epoch_probe.py [runs]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 9472
qs = [float(x) for x in sys.argv[2:]] or [0.02, 0.1, 0.5, 1.0]
for q in qs:
    sc = []
    for s in range(runs):
        d = wl.c2(s, windows=100)
        d["quantum"] = q
        sc.append(Scenario.from_dict(d))
    batch = cc.Batch([cc.compile_run(x, "fast") for x in sc])
    sess = backend.Session(batch)
    sess.run()
    ms = min(sess.run() for _ in range(3))
    st = sess.download(rows=False)["status"]
    slots = 24 * 148
    cyc_per_run = ms * 1e-3 * 1.965e9 * slots / runs
    print(f"quantum {q}: {ms:8.2f} ms  steps/window {int(round(1/q))}  pod-steps {st['pod_steps'].sum():.3g}"
          f"  scale {st['scale_decisions'].mean():.0f}  attempts {st['placement_attempts'].mean():.0f}"
          f"  cycles/run {cyc_per_run:.3g}  bad {(st['code'] != 0).sum()}")
    sess.close()
