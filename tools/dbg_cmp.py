import sys, os; sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'oracle')); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import oracle, parity
from paper_2309_00558_b200 import engine, compiler as cc, workloads as wl
from paper_2309_00558_b200.scenario import Scenario
sc = Scenario.from_dict(wl.c2(0, windows=120))
g = engine.simulate([sc], ['fast'])[0]
o = parity.oracle_results([sc], ['fast'])[0]
print('diff:', parity.diff_results(g, o))
a, b = g.report.to_csv().splitlines(), o.report.to_csv().splitlines()
print('csv equal', a == b, len(a), len(b))
for x, y in zip(a, b):
    if x != y: print('GPU', x); print('ORA', y); break
print(g.token_grants, o.token_grants, g.pod_steps, o.pod_steps)
