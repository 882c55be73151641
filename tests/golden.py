"""Helpers over tests/golden/golden_runs.json.gz (made by make_golden.py from
the real reference).  Test infrastructure only."""
from __future__ import annotations

import functools
import gzip
import json
import os
import tempfile
from fractions import Fraction

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "golden_runs.json.gz")


@functools.lru_cache(maxsize=1)
def records():
    with gzip.open(GOLDEN, "rt", encoding="utf-8") as fh:
        return json.load(fh)["records"]


def load_scenario(rec):
    """Build this package's Scenario for a golden record (CSV profiles are
    written to a temp dir because the schema references them by path)."""
    from paper_2309_00558_b200.scenario import Scenario
    with tempfile.TemporaryDirectory() as tmp:
        for fname, text in rec["files"].items():
            with open(os.path.join(tmp, fname), "w") as fh:
                fh.write(text)
        return Scenario.from_dict(json.loads(json.dumps(rec["scenario"])), base_dir=tmp)


def expected_placements(rec):
    out = {}
    for node, pid, x, y, w, h in rec["expect"]["placements"]:
        out.setdefault(node, {})[pid] = tuple(Fraction(v) for v in (x, y, w, h))
    return out


def got_placements(result):
    return {n: dict(p) for n, p in result.placements.items() if p}


def compare(rec, outcome):
    """outcome: RunResult or Exception.  Returns a list of mismatch strings."""
    from paper_2309_00558_b200.engine import RunResult
    exp = rec["expect"]
    errs = []
    if "error" in exp:
        if isinstance(outcome, RunResult):
            errs.append(f"expected {exp['error']}: {exp['message']}, got a report")
        elif type(outcome).__name__ != exp["error"] and not (
                exp["error"] == "ValidationError" and isinstance(outcome, Exception)
                and "ValidationError" in [c.__name__ for c in type(outcome).__mro__]):
            errs.append(f"expected {exp['error']}, got {type(outcome).__name__}: {outcome}")
        elif str(outcome) != exp["message"]:
            errs.append(f"message {str(outcome)!r} != {exp['message']!r}")
        return errs
    if not isinstance(outcome, RunResult):
        return [f"unexpected error {type(outcome).__name__}: {outcome}"]
    csv = outcome.report.to_csv()
    if csv != exp["csv"]:
        import difflib
        diff = list(difflib.unified_diff(exp["csv"].splitlines(), csv.splitlines(),
                                         lineterm="", n=0))
        errs.append("csv differs:\n" + "\n".join(diff[:12]))
    if outcome.report.summary() != exp["summary"]:
        errs.append("summary differs")
    if got_placements(outcome) != expected_placements(rec):
        errs.append("placements differ")
    return errs
