"""Throughput profiles over the (SM partition, window quota) grid.

Host-side model of the FaST-Profiler tables (reference:
pkg/src/gshare_sim/profiles.py).  Profiles are immutable inputs: the scenario
compiler (``compiler.py``) lowers each one to a dense, (sm, quota)-sorted
point table that the device reads with plain indexed loads -- the B200 form of
``throughput_at`` (profiles.py:167-174).  Lookups are exact; an unprofiled
point is an error, never an interpolation.
"""
from __future__ import annotations

import csv
import io
import json
import math
import os
from dataclasses import dataclass, field
from typing import Iterable, Mapping, Sequence

from .errors import ConflictError, MissingConfigurationError, ParseError, ValidationError
from .memory import DEFAULT_MEMORY_SPEC, MemorySpec
from .util import fmt_num

PROFILE_COLUMNS = ("function_id", "sm_partition", "quota", "throughput_rps", "p99_ms",
                   "slo_ms", "mem_noshare_mb", "mem_runtime_mb", "mem_server_mb")

DEFAULT_SM_GRID = (6.0, 12.0, 24.0, 50.0, 60.0, 80.0, 100.0)
DEFAULT_QUOTA_GRID = (0.2, 0.4, 0.6, 0.8, 1.0)

_DIP_EPS = 1e-9


@dataclass(frozen=True, order=True)
class ConfigPoint:
    """(sm_partition %, quota fraction); ordered lexicographically."""

    sm_partition: float
    quota: float

    def __post_init__(self):
        sm, q = self.sm_partition, self.quota
        if not (math.isfinite(sm) and 0 < sm <= 100):
            raise ValidationError(f"sm_partition must be in (0, 100], got {sm!r}")
        if not (math.isfinite(q) and 0 < q <= 1):
            raise ValidationError(f"quota must be in (0, 1], got {q!r}")

    @property
    def sm_fraction(self) -> float:
        return self.sm_partition / 100.0

    @property
    def resource_area(self) -> float:
        # (sm / 100.0) * quota, evaluated exactly as profiles.py:70,75
        return self.sm_fraction * self.quota


@dataclass(frozen=True)
class ProfileEntry:
    point: ConfigPoint
    throughput_rps: float
    p99_latency_ms: float

    def __post_init__(self):
        t, p = self.throughput_rps, self.p99_latency_ms
        if not (math.isfinite(t) and t >= 0):
            raise ValidationError(f"throughput_rps must be finite and >= 0, got {t!r}")
        if not (math.isfinite(p) and p > 0):
            raise ValidationError(f"p99_latency_ms must be positive, got {p!r}")


@dataclass
class FunctionProfile:
    function_id: str
    entries: dict
    slo_latency_ms: float
    mem: MemorySpec
    warnings: tuple = ()

    def __post_init__(self):
        if not self.function_id:
            raise ValidationError("function_id must be non-empty")
        slo = self.slo_latency_ms
        if not (math.isfinite(slo) and slo > 0):
            raise ValidationError(f"slo_latency_ms must be positive, got {slo!r}")

    @classmethod
    def from_entries(cls, function_id: str, entries: Iterable[ProfileEntry],
                     slo_latency_ms: float = 1000.0,
                     mem: MemorySpec | None = None) -> "FunctionProfile":
        table: dict = {}
        for e in entries:
            if e.point in table:
                raise ConflictError(
                    f"{function_id}: duplicate profile point "
                    f"({fmt_num(e.point.sm_partition)}, {fmt_num(e.point.quota)})")
            table[e.point] = e
        if not table:
            raise ValidationError(f"{function_id}: profile has no entries")
        return cls(function_id, table, slo_latency_ms, mem or DEFAULT_MEMORY_SPEC,
                   tuple(_dip_warnings(function_id, table)))

    def points(self) -> list:
        return sorted(self.entries)


def _dip_warnings(fid: str, table: Mapping) -> list:
    """Throughput dips along either grid axis (informational only)."""
    out = []
    axes = (("quota", lambda p: p.sm_partition, lambda p: p.quota, "sm"),
            ("sm", lambda p: p.quota, lambda p: p.sm_partition, "quota"))
    for grows, fixed_of, moving_of, fixed_name in axes:
        groups: dict = {}
        for e in table.values():
            groups.setdefault(fixed_of(e.point), []).append(e)
        for fixed in sorted(groups):
            line = sorted(groups[fixed], key=lambda e: moving_of(e.point))
            for a, b in zip(line, line[1:]):
                if b.throughput_rps < a.throughput_rps - _DIP_EPS:
                    out.append(
                        f"{fid}: throughput dips from {fmt_num(a.throughput_rps)} to "
                        f"{fmt_num(b.throughput_rps)} rps as {grows} grows "
                        f"{fmt_num(moving_of(a.point))} -> {fmt_num(moving_of(b.point))} "
                        f"at {fixed_name}={fmt_num(fixed)}")
    return out


def throughput_at(profile: FunctionProfile, point: ConfigPoint) -> float:
    entry = profile.entries.get(point)
    if entry is None:
        raise MissingConfigurationError(
            f"{profile.function_id}: no profile entry at "
            f"({fmt_num(point.sm_partition)}, {fmt_num(point.quota)})")
    return entry.throughput_rps


def rps_per_resource(profile: FunctionProfile, point: ConfigPoint) -> float:
    return throughput_at(profile, point) / point.resource_area


def grid_points(sm_values: Sequence[float], quota_values: Sequence[float]) -> list:
    return [ConfigPoint(s, q) for s in sm_values for q in quota_values]


def synth_profile(function_id: str, t_max: float, sm_knee: float,
                  grid: Sequence[ConfigPoint], *, slo_latency_ms: float = 1000.0,
                  mem: MemorySpec | None = None) -> FunctionProfile:
    """T(sm, q) = q * t_max * min(sm, knee) / knee, left to right
    (reference profiles.py:199-213)."""
    if not (math.isfinite(t_max) and t_max > 0):
        raise ValidationError(f"t_max must be positive, got {t_max!r}")
    if not (math.isfinite(sm_knee) and 0 < sm_knee <= 100):
        raise ValidationError(f"sm_knee must be in (0, 100], got {sm_knee!r}")
    if not grid:
        raise ValidationError("synth_profile requires a non-empty grid")
    entries = []
    for p in grid:
        rate = p.quota * t_max * min(p.sm_partition, sm_knee) / sm_knee
        entries.append(ProfileEntry(p, rate, 1000.0 / max(rate, 1e-3)))
    return FunctionProfile.from_entries(function_id, entries, slo_latency_ms, mem)


# ---------------------------------------------------------------------------
# ingestion (host file I/O; same formats as profiles.py:228-380)
# ---------------------------------------------------------------------------

def _lines_of(source) -> list:
    if isinstance(source, (str, os.PathLike)):
        try:
            with open(source, "r", encoding="utf-8") as fh:
                return fh.read().splitlines()
        except OSError as exc:
            raise ValidationError(f"cannot read profile file {source!r}: {exc}") from exc
    if hasattr(source, "read"):
        return source.read().splitlines()
    return [str(s).rstrip("\n") for s in source]


def _coerce(line_no: int, raw: Mapping) -> dict:
    rec = {}
    for col in PROFILE_COLUMNS:
        val = raw.get(col)
        if val is None or val == "":
            raise ParseError(f"missing column {col!r}", line_no)
        rec[col] = val
    rec["function_id"] = str(rec["function_id"])
    for col in PROFILE_COLUMNS[1:]:
        try:
            rec[col] = float(rec[col])
        except (TypeError, ValueError):
            raise ParseError(f"column {col!r} is not a number: {rec[col]!r}", line_no)
    try:
        ConfigPoint(rec["sm_partition"], rec["quota"])
        slo = rec["slo_ms"]
        if not (math.isfinite(slo) and slo > 0):
            raise ValidationError(f"slo_ms must be positive, got {slo!r}")
    except ValidationError as exc:
        raise ParseError(str(exc), line_no)
    return rec


def _records(lines: list) -> list:
    numbered = [(i + 1, s.strip()) for i, s in enumerate(lines) if s.strip()]
    if not numbered:
        return []
    if numbered[0][1].startswith("{"):
        out = []
        for n, s in numbered:
            try:
                raw = json.loads(s)
            except json.JSONDecodeError as exc:
                raise ParseError(f"invalid JSON: {exc.msg}", n)
            if not isinstance(raw, dict):
                raise ParseError("JSON record must be an object", n)
            out.append((n, _coerce(n, raw)))
        return out
    head_no, head = numbered[0]
    header = [h.strip() for h in next(csv.reader([head]))]
    if set(header) != set(PROFILE_COLUMNS):
        raise ParseError(f"CSV header must contain exactly {', '.join(PROFILE_COLUMNS)}",
                         head_no)
    out = []
    for n, s in numbered[1:]:
        vals = next(csv.reader([s]))
        if len(vals) != len(header):
            raise ParseError(f"expected {len(header)} fields, found {len(vals)}", n)
        out.append((n, _coerce(n, dict(zip(header, vals)))))
    return out


def ingest_profiles(source) -> dict:
    recs = _records(_lines_of(source))
    if not recs:
        raise ValidationError("profile stream contains no records")
    by_fn: dict = {}
    for n, r in recs:
        by_fn.setdefault(r["function_id"], []).append((n, r))
    result = {}
    for fid, rows in by_fn.items():
        n0, r0 = rows[0]
        mem = MemorySpec(r0["mem_noshare_mb"], r0["mem_runtime_mb"], r0["mem_server_mb"])
        entries = []
        for n, r in rows:
            same = (r["slo_ms"] == r0["slo_ms"]
                    and r["mem_noshare_mb"] == mem.mem_noshare_mb
                    and r["mem_runtime_mb"] == mem.mem_runtime_mb
                    and r["mem_server_mb"] == mem.mem_server_mb)
            if not same:
                raise ConflictError(
                    f"line {n}: {fid}: slo/memory columns disagree with line {n0}")
            entries.append(ProfileEntry(ConfigPoint(r["sm_partition"], r["quota"]),
                                        r["throughput_rps"], r["p99_ms"]))
        result[fid] = FunctionProfile.from_entries(fid, entries, r0["slo_ms"], mem)
    return result


def ingest_profile(source) -> FunctionProfile:
    profs = ingest_profiles(source)
    if len(profs) != 1:
        raise ValidationError(f"expected exactly one function in stream, found {sorted(profs)}")
    return next(iter(profs.values()))


def serialize_profiles(profiles) -> str:
    items = ([profiles[k] for k in sorted(profiles)] if isinstance(profiles, Mapping)
             else sorted(profiles, key=lambda p: p.function_id))
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(PROFILE_COLUMNS)
    for prof in items:
        for p in prof.points():
            e = prof.entries[p]
            w.writerow([prof.function_id] + [fmt_num(v) for v in (
                p.sm_partition, p.quota, e.throughput_rps, e.p99_latency_ms,
                prof.slo_latency_ms, prof.mem.mem_noshare_mb, prof.mem.mem_runtime_mb,
                prof.mem.mem_server_mb)])
    return buf.getvalue()


def serialize_profile(profile: FunctionProfile) -> str:
    return serialize_profiles([profile])
