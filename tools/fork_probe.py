import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import multiprocessing as mp, gc
import numpy as np
from paper_2309_00558_b200 import backend, workloads as wl, engine
def f(x): return x
def pool_time(tag):
    gc.freeze()
    t=time.perf_counter(); p=mp.get_context("fork").Pool(16); t1=time.perf_counter()
    r=p.map(f, range(16), chunksize=1); t2=time.perf_counter()
    p.terminate(); p.join(); t3=time.perf_counter(); gc.unfreeze()
    print(tag, "create", round(t1-t,4), "first map", round(t2-t1,4), "terminate", round(t3-t2,4), flush=True)
pool_time("bare")
scen = wl.c2_scenarios(range(21312), windows=300)
pool_time("with scenarios")
engine.run_batch(scen[:64])
pool_time("after cuda init")
reps = engine.run_batch(scen)
pool_time("after big run_batch (pinned pool populated, reports alive)")
del reps; gc.collect()
pool_time("after freeing reports")
