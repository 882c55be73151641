"""Windows stepped in the shared-memory working set vs on the HBM arena, per
config (needs a -DGS_XL_TIMING build): python tools/arena_probe.py variants/xlt.so"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GS_LIB"] = sys.argv[1]
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario
backend.LIB_PATH = sys.argv[1]
sets = {
    "C1": ([Scenario.from_dict(wl.c1())] * 512, ["fast", "timeshare"] * 256),
    "C2": (wl.c2_scenarios(range(1024), windows=300), ["fast"] * 1024),
    "C3": ([Scenario.from_dict(wl.c3(s)) for s in range(256) for _ in (0, 1)], ["fast", "timeshare"] * 256),
    "C5": ([Scenario.from_dict(wl.c5(i)) for i in range(2048)], ["fast"] * 2048),
}
for k, (scen, pols) in sets.items():
    b = cc.Batch([cc.compile_run(s, p) for s, p in zip(scen, pols)])
    t = (C.c_ulonglong * 32)()
    backend.lib().gs_xl_timing(t)
    h0, a0 = t[30], t[31]
    s = backend.Session(b); ms = s.run()
    backend.lib().gs_xl_timing(t)
    print(f"{k}: {ms:.1f} ms  windows in shared memory {t[30] - h0}  on the arena {t[31] - a0}", flush=True)
    s.close()
