"""A/B timing of several builds of libgshare_b200.so on one batch (GPU box).
usage: python tools/ab.py --runs 9472 --windows 100 variants/a.so variants/b.so ...
Each variant: 1 warm-up + `--reps` timed launches, interleaved across variants."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--runs", type=int, default=9472)
ap.add_argument("--windows", type=int, default=100)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--policy", default="fast")
a = ap.parse_args()
batch = cc.Batch([cc.compile_run(s, a.policy) for s in wl.c2_scenarios(range(a.runs), windows=a.windows)])
simsec = float((batch.runs["windows"] * batch.runs["window_s"]).sum())
sess = {}
ref = None
for path in a.libs:
    backend._lib = None
    backend.LIB_PATH = os.path.abspath(path)
    s = backend.Session(batch)
    s.run()
    out = s.download(rows=False)
    if ref is None:
        ref = out
    st_fields = [f for f in out["status"].dtype.names if f != "hot_class"]   # class ids may differ
    same = (np.array_equal(out["summary"], ref["summary"])
            and all(np.array_equal(out["status"][f], ref["status"][f]) for f in st_fields))
    sess[path] = (s, [], same)
for _ in range(a.reps):
    for path, (s, times, _) in sess.items():
        times.append(s.run())
for path, (s, times, same) in sess.items():
    ms = min(times)
    print(f"{os.path.basename(path):24s} best {ms:8.2f} ms  {simsec / ms * 1e3 / 1e6:6.3f} M sim-s/s  same_as_first={same}  all={['%.1f' % t for t in times]}")
