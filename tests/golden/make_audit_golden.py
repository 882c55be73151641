"""Golden verdicts of the reference's packer auditor ``check_node``
(pkg/src/gshare_sim/packer.py:327-388) on node geometries, for the device
auditor (csrc/gs_audit.cuh).

Geometries come from the reference packer itself, driven the way its own
tests drive it (test_packer.py:224-250 TestRandomSequencesAgainstRaster,
test_acceptance.py:156-181 -- seeded place/release streams over 1-2 nodes,
best_match choosing the rectangle, plus restructure), with integral and
fractional pod shapes (quota 0.125 / SM 12.5 style coordinates).  Every valid
snapshot is then also corrupted in each way check_node detects -- a dropped
or shrunk free rectangle (gap), a duplicated or nested free rectangle
(containment), an overlapping or grown placement, a free rectangle over a
placement -- and check_node's messages are classified into the device's
GS_AUDIT_* bits.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_audit_golden.py

Output: tests/golden/golden_audit.json.gz (committed).
"""
from __future__ import annotations

import dataclasses
import gzip
import json
import os
import random
import sys
from fractions import Fraction

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "golden_audit.json.gz")

PLACED_OVERLAP, FREE_PLACED, FREE_CONTAINED, GAP, DOUBLE = 1, 2, 4, 8, 16


def classify(msgs):
    bits, skipped = 0, False
    for m in msgs:
        if m.startswith("placements "):
            bits |= PLACED_OVERLAP
        elif m.startswith("free rect ") and "overlaps placement" in m:
            bits |= FREE_PLACED
        elif "is contained in" in m:
            bits |= FREE_CONTAINED
        elif m.startswith("coverage gap"):
            bits |= GAP
        elif m.startswith("coverage overlap"):
            bits |= DOUBLE
        elif m.startswith("coverage check skipped"):
            skipped = True
        else:
            raise ValueError(m)
    return bits, skipped


def fr(v: Fraction) -> str:
    return f"{v.numerator}/{v.denominator}"


def snapshot(node):
    return {"free": [[fr(x) for x in r.as_tuple()] for r in node.free_rects],
            "placed": [[fr(x) for x in p.rect.as_tuple()] for p in node.placements.values()]}


def main(seed: int = 20261017):
    sys.path.insert(0, REF)
    from gshare_sim import packer as pk
    rng = random.Random(seed)
    shapes_frac = [Fraction(1, 2), Fraction(1, 4), Fraction(1, 8), Fraction(1, 5), Fraction(1, 1)]
    records = []

    def record(node, tag):
        snap = snapshot(node)
        bits, skipped = classify(pk.check_node(node))
        records.append({"tag": tag, **snap, "bits": bits, "coverage_skipped": skipped})

    def corrupt(node, tag):
        free = list(node.free_rects)
        placed = list(node.placements.items())
        muts = []
        if free:
            k = rng.randrange(len(free))
            muts.append(("drop-free", free[:k] + free[k + 1:], None))
            r = free[k]
            if r.w > 1 and r.h > 1:
                muts.append(("shrink-free", free[:k] + [pk.rect(r.x, r.y, r.w - 1, r.h)]
                             + free[k + 1:], None))
            muts.append(("dup-free", free + [free[k]], None))
            if r.w >= 2 and r.h >= 2:
                muts.append(("nested-free", free + [pk.rect(r.x, r.y, r.w / 2, r.h / 2)], None))
        if placed:
            pid, p = placed[rng.randrange(len(placed))]
            muts.append(("free-over-placed", free + [p.rect], None))
            grown = pk.rect(p.rect.x, p.rect.y, min(p.rect.w + 3, 100 - p.rect.x),
                            min(p.rect.h + 3, 100 - p.rect.y))
            muts.append(("grow-placed", free, (pid, grown)))
            muts.append(("extra-placed", free, ("zz-extra", pk.rect(p.rect.x, p.rect.y, 1, 1))))
        for name, new_free, extra in muts:
            bak_free, bak_pl = node.free_rects, dict(node.placements)
            node.free_rects = list(new_free)
            if extra is not None:
                pid, rr = extra
                proto = node.placements.get(pid) or next(iter(node.placements.values()))
                node.placements[pid] = dataclasses.replace(proto, pod_id=pid, rect=rr)
            record(node, f"{tag}/{name}")
            node.free_rects, node.placements = bak_free, bak_pl

    for seq in range(220):
        frac = seq % 3 == 2
        nodes = [pk.new_node(g) for g in range(rng.randint(1, 2))]
        by_id = {n.gpu_id: n for n in nodes}
        live = []
        for event in range(25):
            if live and rng.random() < 0.4:
                pod_id, node = live.pop(rng.randrange(len(live)))
                pk.release(node, pod_id)
            else:
                if frac:
                    w = rng.randint(1, 7) * 100 * rng.choice(shapes_frac) / 8
                    h = rng.randint(1, 14) * rng.choice(shapes_frac) * 5
                    w, h = min(w, 100), min(h, 100)
                else:
                    w, h = rng.randint(1, 70), rng.randint(1, 70)
                request = pk.PodRequest(f"s{seq}e{event}", f"f{event % 3}", pk.as_frac(w),
                                        pk.as_frac(h))
                found = pk.best_match(nodes, request)
                if found is None:
                    continue
                gpu_id, chosen = found
                pk.place(by_id[gpu_id], chosen, request)
                live.append((request.pod_id, by_id[gpu_id]))
            if event % 6 == 5:
                for node in nodes:
                    if rng.random() < 0.3:
                        pk.restructure(node, threshold=rng.choice([0, 2, 4]))
                    record(node, f"seq{seq}e{event}")
                    corrupt(node, f"seq{seq}e{event}")
    with gzip.open(OUT, "wt", encoding="utf-8") as fh:
        json.dump({"generator": "tests/golden/make_audit_golden.py", "seed": seed,
                   "bits": {"placed_overlap": 1, "free_placed": 2, "free_contained": 4,
                            "gap": 8, "double": 16},
                   "records": records}, fh)
    valid = sum(1 for r in records if r["bits"] == 0)
    print(f"wrote {len(records)} geometries ({valid} valid, "
          f"{sum(r['coverage_skipped'] for r in records)} coverage-skipped) to {OUT}")


if __name__ == "__main__":
    main()
