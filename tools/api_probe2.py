"""Drop-in API timing as bench.py's e2e_api measures it (same-size warm-up
call first), with a per-stage timeline of the pipelined simulate_records:
when each compiled block arrives and when its GPU call returns.
usage: python tools/api_probe2.py [runs]"""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_00558_b200 import compiler as cc, engine, workloads as wl

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3552
scen = wl.c2_scenarios(range(n), windows=300)
EV = []
T0 = [0.0]
_stream, _run = cc.compile_stream, engine._run_part


def stream(*a, **k):
    for x in _stream(*a, **k):
        EV.append(("block", len(x[0]), round(time.perf_counter() - T0[0], 4)))
        yield x


def run_part(batch, device):
    t = time.perf_counter() - T0[0]
    out = _run(batch, device)
    EV.append(("gpu", len(batch), round(t, 4), round(time.perf_counter() - T0[0], 4)))
    return out


cc.compile_stream, engine._run_part = stream, run_part
for rep in range(3):
    EV.clear()
    gc.collect()
    T0[0] = time.perf_counter()
    reps = engine.run_batch(scen)
    t1 = time.perf_counter() - T0[0]
    sums = [r.summary() for r in reps]
    t2 = time.perf_counter() - T0[0]
    del reps, sums
    print({"rep": rep, "run_batch_s": round(t1, 4), "total_s": round(t2, 4),
           "value": round(n * 300 / t2), "events": EV[:]}, flush=True)
