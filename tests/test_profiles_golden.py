"""Profile ingestion / serialization pinned to the reference.

tests/golden/golden_profiles.json.gz (tests/golden/make_profile_golden.py,
which runs pkg/src/gshare_sim/profiles.py) holds, for the reference's own
fixtures (pkg/tests/data), the streams of its ingestion tests
(test_profiles.py:128-201) and 240 seeded CSV / JSONL streams -- clean and
broken in every way the parser checks -- the canonical serialization and
warnings of each function, or the exception class and text (line-numbered
ParseErrors).  This package's profiles.py must reproduce every record.
"""
import gzip
import io
import json
import os

import pytest

from paper_2309_00558_b200 import errors, profiles as pp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                      "golden_profiles.json.gz")
with gzip.open(GOLDEN, "rt") as _fh:
    RECORDS = json.load(_fh)["records"]


def _outcome(lines, single):
    try:
        if single:
            p = pp.ingest_profile(list(lines))
            profs = {p.function_id: p}
        else:
            profs = pp.ingest_profiles(list(lines))
    except errors.GShareError as exc:
        return {"error": type(exc).__name__, "message": str(exc)}
    return {"serialized": pp.serialize_profiles(profs), "functions": sorted(profs),
            "warnings": {k: list(v.warnings) for k, v in profs.items()},
            "slo_ms": {k: v.slo_latency_ms for k, v in profs.items()}}


@pytest.mark.parametrize("k", range(len(RECORDS)))
def test_ingestion_matches_reference(k):
    rec = RECORDS[k]
    assert _outcome(rec["lines"], rec["single"]) == rec["expect"], rec["name"]


def test_fixture_covers_every_error_kind():
    kinds = {r["expect"].get("error") for r in RECORDS}
    assert {"ParseError", "ValidationError", "ConflictError", None} <= kinds
    msgs = " ".join(r["expect"].get("message", "") for r in RECORDS)
    for needle in ("invalid JSON", "must be an object", "is not a number", "missing column",
                   "expected 9 fields", "CSV header must contain", "slo/memory columns disagree",
                   "no records", "line "):
        assert needle in msgs, needle


def test_serialize_ingest_round_trip_on_reference_fixtures():
    for rec in RECORDS:
        exp = rec["expect"]
        if "serialized" in exp and not rec["single"]:
            again = pp.ingest_profiles(io.StringIO(exp["serialized"]))
            assert pp.serialize_profiles(again) == exp["serialized"], rec["name"]
