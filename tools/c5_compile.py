"""Host lowering time of the 100k-run C5 sweep (BASELINE configs[4]) on this
host's cores: from scenario dicts (generated in the workers) and from prebuilt
Scenario objects.  usage: python tools/c5_compile.py [runs]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_00558_b200 import compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
seq = wl.ScenarioSeq(wl.c5, n)
cc.compile_batch(wl.ScenarioSeq(wl.c5, 2000), ["fast"] * 2000)      # warm the pool path
t = time.perf_counter()
b, _, err = cc.compile_batch(seq, ["fast"] * n)
t_dicts = time.perf_counter() - t
objs = [Scenario.from_dict(wl.c5(i)) for i in range(n)]
t = time.perf_counter()
b2, _, err2 = cc.compile_batch(objs, ["fast"] * n)
t_objs = time.perf_counter() - t
print({"runs": n, "cores": os.cpu_count(), "from_dicts_s": round(t_dicts, 3),
       "from_scenarios_s": round(t_objs, 3), "errors": len(err) + len(err2),
       "same": bool((b.counts == b2.counts).all() and (b.runs == b2.runs).all())})
