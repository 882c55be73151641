"""Golden outputs of the reference's profile ingestion and serialization
(pkg/src/gshare_sim/profiles.py:228-380).

Runs the REAL reference ``ingest_profiles`` / ``ingest_profile`` /
``serialize_profiles`` on

  * the reference's own test fixtures (pkg/tests/data/*.csv: resnet_grid,
    monotone_dip, model_memory_profiles),
  * the streams of its ingestion tests (test_profiles.py:128-201:
    duplicate point, empty stream, malformed record, CSV/JSONL agreement),
  * a seeded sweep of CSV and JSONL streams, clean and broken (bad header,
    wrong field counts, missing / empty / non-numeric columns, out-of-range
    points and SLOs, invalid JSON, non-object JSON, conflicting slo/memory
    columns, duplicate points, blank lines, several functions per stream),

and records, per stream, the canonical serialization + warnings of every
function, or the exception class and text (with its line number).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_profile_golden.py

Output: tests/golden/golden_profiles.json.gz (committed).
"""
from __future__ import annotations

import gzip
import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
DATA = "/root/reference/pkg/tests/data"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "golden_profiles.json.gz")

COLS = ["function_id", "sm_partition", "quota", "throughput_rps", "p99_ms", "slo_ms",
        "mem_noshare_mb", "mem_runtime_mb", "mem_server_mb"]


def _row(rng, fid, sm, q, slo=500.0, mem=(1000.0, 800.0, 400.0)):
    t = round(rng.uniform(0.0, 90.0), rng.choice([0, 1, 3, 7]))
    return {"function_id": fid, "sm_partition": sm, "quota": q, "throughput_rps": t,
            "p99_ms": round(rng.uniform(5, 900), 2), "slo_ms": slo,
            "mem_noshare_mb": mem[0], "mem_runtime_mb": mem[1], "mem_server_mb": mem[2]}


def _csv(rows, header=COLS):
    out = [",".join(header)]
    for r in rows:
        out.append(",".join(str(r.get(c, "")) for c in header))
    return out


def _jsonl(rows):
    return [json.dumps(r) for r in rows]


def random_stream(rng, k):
    fids = rng.sample(["m", "resnet", "bert_qa", "a,b", "v.2", "Z"], rng.randint(1, 3))
    rows = []
    for fid in fids:
        slo = rng.choice([100.0, 500.0, 250.5])
        mem = rng.choice([(1000.0, 800.0, 400.0), (1200.5, 900.0, 600.0)])
        sms = rng.sample([6, 12, 24, 50, 100, 12.5, 33.3], rng.randint(1, 4))
        qs = rng.sample([0.2, 0.4, 1.0, 0.125, 0.75], rng.randint(1, 3))
        for sm in sms:
            for q in qs:
                rows.append(_row(rng, fid, sm, q, slo, mem))
    rng.shuffle(rows)
    fmt = rng.choice(["csv", "jsonl"])
    breaks = rng.random() < 0.55
    kind = "clean"
    if breaks and rows:
        kind = rng.choice(["nonnum", "missing", "empty", "sm_range", "q_range", "slo",
                           "conflict", "dup", "fields", "header", "badjson", "nonobj",
                           "blank"])
        j = rng.randrange(len(rows))
        r = dict(rows[j])
        if kind == "nonnum":
            r[rng.choice(COLS[1:])] = "n/a"
        elif kind == "missing" and fmt == "jsonl":
            del r[rng.choice(COLS)]
        elif kind in ("missing", "empty"):
            r[rng.choice(COLS)] = ""
        elif kind == "sm_range":
            r["sm_partition"] = rng.choice([0, 101, -5])
        elif kind == "q_range":
            r["quota"] = rng.choice([0, 1.5])
        elif kind == "slo":
            r["slo_ms"] = rng.choice([0, -1, "inf"])
        elif kind == "conflict":
            r["mem_server_mb"] = 123.0
        elif kind == "dup":
            rows.append(dict(r))
        rows[j] = r
    lines = _csv(rows) if fmt == "csv" else _jsonl(rows)
    if kind == "fields" and fmt == "csv" and len(lines) > 1:
        j = rng.randrange(1, len(lines))
        lines[j] += ",9"
    if kind == "header" and fmt == "csv":
        lines[0] = lines[0].replace("p99_ms", "p99")
    if kind == "badjson" and fmt == "jsonl" and lines:
        j = rng.randrange(len(lines))
        lines[j] = lines[j][:-3]
    if kind == "nonobj" and fmt == "jsonl" and lines:
        lines[rng.randrange(len(lines))] = "[1, 2]"
    if kind == "blank":
        for _ in range(3):
            lines.insert(rng.randrange(len(lines) + 1), rng.choice(["", "   "]))
    return {"name": f"random-{k:03d}-{fmt}-{kind}", "lines": lines}


def fixed_streams():
    hdr = ",".join(COLS)
    out = []
    for name in ("resnet_grid.csv", "monotone_dip.csv", "model_memory_profiles.csv"):
        with open(os.path.join(DATA, name)) as fh:
            out.append({"name": f"data/{name}", "lines": fh.read().splitlines()})
    out += [
        {"name": "test-duplicate-point", "lines": [hdr, "m,12,0.4,10,100,500,1000,800,400",
                                                   "m,12,0.4,11,100,500,1000,800,400"]},
        {"name": "test-empty-stream", "lines": [hdr]},
        {"name": "test-malformed-record", "lines": [hdr, "m,12,0.4,10,100,500,1000,800,400",
                                                    "m,24,not_a_number,12,100,500,1000,800,400"]},
        {"name": "test-csv-agree", "lines": [hdr, "m,12,0.4,10,100,500,1000,800,400"]},
        {"name": "test-jsonl-agree", "lines": [
            '{"function_id": "m", "sm_partition": 12, "quota": 0.4, "throughput_rps": 10, '
            '"p99_ms": 100, "slo_ms": 500, "mem_noshare_mb": 1000, "mem_runtime_mb": 800, '
            '"mem_server_mb": 400}']},
        {"name": "nothing", "lines": []},
        {"name": "invalid-json", "lines": [
            '{"function_id": "m", "sm_partition": 12, "quota": 0.4, "throughput_rps": 10, '
            '"p99_ms": 100, "slo_ms": 500, "mem_noshare_mb": 1000, "mem_runtime_mb": 800, '
            '"mem_server_mb": 400}', '{"function_id": "m", "sm_partition": 24,']},
        {"name": "json-not-object", "lines": [
            '{"function_id": "m", "sm_partition": 12, "quota": 0.4, "throughput_rps": 10, '
            '"p99_ms": 100, "slo_ms": 500, "mem_noshare_mb": 1000, "mem_runtime_mb": 800, '
            '"mem_server_mb": 400}', '[1, 2, 3]']},
        {"name": "json-missing-column", "lines": [
            '{"function_id": "m", "sm_partition": 12, "quota": 0.4, "throughput_rps": 10}']},
        {"name": "reordered-header", "lines": [
            "quota,function_id,sm_partition,throughput_rps,p99_ms,slo_ms,mem_noshare_mb,"
            "mem_runtime_mb,mem_server_mb", "0.4,m,12,10,100,500,1000,800,400"]},
    ]
    return out


def run_reference(stream, single):
    sys.path.insert(0, REF)
    import gshare_sim as ref
    from gshare_sim import profiles as rp
    try:
        if single:
            p = rp.ingest_profile(list(stream["lines"]))
            profs = {p.function_id: p}
        else:
            profs = rp.ingest_profiles(list(stream["lines"]))
    except ref.GShareError as exc:
        return {"error": type(exc).__name__, "message": str(exc)}
    return {"serialized": rp.serialize_profiles(profs),
            "functions": sorted(profs),
            "warnings": {k: list(v.warnings) for k, v in profs.items()},
            "slo_ms": {k: v.slo_latency_ms for k, v in profs.items()}}


def main(seed: int = 20261017):
    rng = random.Random(seed)
    streams = fixed_streams() + [random_stream(rng, k) for k in range(240)]
    recs = []
    for s in streams:
        for single in (False, True):
            recs.append(dict(s, single=single, expect=run_reference(s, single)))
    with gzip.open(OUT, "wt", encoding="utf-8") as fh:
        json.dump({"generator": "tests/golden/make_profile_golden.py", "seed": seed,
                   "records": recs}, fh)
    n_err = sum(1 for r in recs if "error" in r["expect"])
    print(f"wrote {len(recs)} records ({n_err} reference errors) to {OUT}")


if __name__ == "__main__":
    main()
