import sys, os
sys.path.insert(0, "/root/repo")
from paper_2309_00558_b200 import backend, compiler as cc, workloads as wl
import dataclasses
sc = wl.c2_scenarios(range(9472), windows=100)
for ret in (32, 64):
    imgs = []
    for s in sc:
        caps = cc._default_caps(s, cc._ordered_functions(s))
        imgs.append(cc.compile_run(s, "fast", dataclasses.replace(caps, returned=ret)))
    b = cc.Batch(imgs)
    S = backend.Session(b); S.run()
    print("returned", ret, min(S.run() for _ in range(3)), "ms")
