"""XL driver time split (warp 0): build with `bash tools/build_variant.sh wt xlt -DGS_XL_TIMING`,
then `python tools/xl_timing.py variants/xlt.so` on the GPU box."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GS_LIB"] = sys.argv[1]
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario
backend.LIB_PATH = sys.argv[1]
b = cc.Batch([cc.compile_run(Scenario.from_dict(wl.c4(s, windows=int(os.environ.get("XLT_WINDOWS", "100")))), "fast") for s in range(16)])
s = backend.Session(b); ms = s.run()
t = (C.c_ulonglong * 64)()
backend.lib().gs_xl_timing(t)
tot = sum(t[:4])
print(f"{ms:.1f} ms; warp-0 cycles: epoch {t[0]/tot:.2%} window_begin {t[1]/tot:.2%} steps {t[2]/tot:.2%} window_close {t[3]/tot:.2%}")
ep = max(t[0], 1)
print(f"  epoch split: scaling {t[4]/ep:.1%}  place_batch {t[5]/ep:.1%} (best_match {t[7]/ep:.1%})  restructure+frag {t[6]/ep:.1%}")
print(f"  xl_place_batch: sort {t[8]/ep:.1%}  scan+barrier {t[11]/ep:.1%}  place_pod {t[9]/ep:.1%}  iterations {t[10]} ({t[11]/max(t[10],1):.0f} cyc scan, {t[9]/max(t[10],1):.0f} cyc place per iter)")
print(f"  scaling: group {t[12]/ep:.1%}  group+decide {t[13]/ep:.1%}  apply {t[14]/ep:.1%}")
print(f"  windows on the arena path (registered set did not fit shared memory): {t[15]} of {sum(int(r['windows']) for r in b.runs)}")
st = sum(t[16:25])
names = ["admit+reset", "complete+key", "rank", "grant", "cov/occ|dispatch", "compact", "dry run+scan", "replay", "queue books"]
print("  xlh_step phases: " + "  ".join(f"{nm} {t[16+i]/max(st,1):.1%}" for i, nm in enumerate(names)))
print(f"  steps {t[25]}  cycles/step {st/max(t[25],1):.0f}  pods/step {t[26]/max(t[25],1):.0f}  granted/step {t[27]/max(t[25],1):.0f}")
print(f"  max pods on one node: mean over steps {t[28]/max(t[25],1):.0f}, overall max {t[29]}")
nw = 16   # warps per XL CTA
print("  per-phase warp efficiency (mean warp busy / phase time; 1 = balanced): " + "  ".join(
    f"{nm} {t[48 + i] / nw / max(t[16 + i], 1):.2f}" for i, nm in enumerate(names)))
