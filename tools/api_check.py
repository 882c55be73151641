"""The pipelined drop-in API on a mixed batch (fork-pool lowering, 8 blocks,
concurrent stream-ordered one-shot calls), every report compared with the
oracle -- a compute-sanitizer target for the host-threaded C-ABI path.
usage: python tools/api_check.py [runs]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from parity import oracle_results
from paper_2309_00558_b200 import engine, workloads as wl
from paper_2309_00558_b200.scenario import Scenario

n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
scen = [Scenario.from_dict(wl.c2(s, windows=20) if s % 3 else wl.c5(s)) for s in range(n)]
pols = ["fast" if s % 2 else "timeshare" for s in range(n)]
reps = engine.run_batch(scen, pols, errors="return")
want = oracle_results(scen, pols)
bad = sum(1 for g, r in zip(reps, want)
          if (isinstance(r, Exception) and str(g) != str(r))
          or (not isinstance(r, Exception) and (g.to_csv() != r.report.to_csv()
                                               or g.summary() != r.report.summary())))
print({"runs": n, "mismatched": bad})
sys.exit(1 if bad else 0)
