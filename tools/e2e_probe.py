"""Break down the end-to-end C-ABI call (GPU box): host compile, pinned vs
pageable buffers, zero-copy rows.  usage: python tools/e2e_probe.py [runs] [windows]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 9472
windows = int(sys.argv[2]) if len(sys.argv) > 2 else 300
t = time.perf_counter()
batch = cc.Batch([cc.compile_run(s, "fast") for s in wl.c2_scenarios(range(runs), windows=windows)])
print(f"compile {time.perf_counter() - t:.2f}s  inputs {batch.input_bytes()/1e6:.1f} MB")
sess = backend.Session(batch)
sess.run()
print(f"kernel {sess.run():.1f} ms")
ref = sess.download()
sess.close()

def timed(label, fn, reps=3):
    ts = []
    for _ in range(reps):
        t = time.perf_counter(); r = fn(); ts.append(time.perf_counter() - t)
    print(f"{label:44s} best {min(ts)*1e3:8.1f} ms  all {[round(x*1e3) for x in ts]}")
    return r

timed("pageable in, fresh pageable out", lambda: backend.run_batch(batch))
out_pg = batch.alloc_outputs()
timed("pageable in, reused pageable out", lambda: backend.run_batch(batch, out=out_pg))
t = time.perf_counter(); out_pin = batch.alloc_outputs(pinned=True)
print(f"alloc pinned outputs {(time.perf_counter()-t)*1e3:.1f} ms")
r = timed("pageable in, pinned out (zero-copy rows)", lambda: backend.run_batch(batch, out=out_pin))
for k in ("fn_rows", "gpu_rows", "glob_rows", "status", "summary"):
    assert np.array_equal(r[k], ref[k]), k
t = time.perf_counter(); batch.pin(); print(f"pin inputs {(time.perf_counter()-t)*1e3:.1f} ms")
r = timed("pinned in, pinned out (zero-copy rows)", lambda: backend.run_batch(batch, out=out_pin))
for k in ("fn_rows", "gpu_rows", "glob_rows", "status", "summary"):
    assert np.array_equal(r[k], ref[k]), k
n = ref["status"]["n_placements"]
print("placements equal:", all(np.array_equal(r["placements"][o:o+c], ref["placements"][o:o+c])
      for o, c in zip(batch.runs["place_off"], n)))
timed("pinned in, reused pageable out", lambda: backend.run_batch(batch, out=out_pg))
