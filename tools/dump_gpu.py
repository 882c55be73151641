"""Debug helper: run a workload batch on the GPU and save raw outputs (npz)."""
import sys, os, pickle
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario

def make(kind):
    if kind == 'c2': return [cc.compile_run(Scenario.from_dict(wl.c2(s, windows=120)), 'fast') for s in range(48)]
    if kind == 'c3': return [cc.compile_run(Scenario.from_dict(wl.c3(s, windows=20)), p) for s in range(4) for p in ('fast','timeshare')]
    raise SystemExit(kind)

if __name__ == '__main__':
    kind = sys.argv[1]
    batch = cc.Batch(make(kind))
    out = backend.run_batch(batch)
    np.savez(f'gpurun_out/dump_{kind}.npz', **{k: v for k, v in out.items() if v is not None})
    print('saved', kind)
