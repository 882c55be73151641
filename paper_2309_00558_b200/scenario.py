"""Scenario description: the input half of the drop-in boundary.

Field names, defaults, JSON schema and validation messages follow the
reference (pkg/src/gshare_sim/sim_engine.py:100-255) so a scenario built for
``gshare_sim`` can be handed to this package unchanged -- the compiler also
accepts the reference's own ``Scenario`` objects by duck typing.
"""
from __future__ import annotations

import functools

import json
import math
import os
from dataclasses import dataclass, field

from .errors import ValidationError
from .memory import DEFAULT_GPU_MEMORY_MB, MemorySpec
from .profiles import (DEFAULT_QUOTA_GRID, DEFAULT_SM_GRID, ConfigPoint, FunctionProfile,
                       grid_points, ingest_profiles, synth_profile)
from .traces import WorkloadTrace, trace_from_spec

POLICIES = ("fast", "timeshare")

#: Free-list length past which a node is re-packed (reference packer.py:34).
DEFAULT_RESTRUCTURE_THRESHOLD = 16


@dataclass(eq=False)
class Request:
    """One request (host-side helper type; the device never materialises these)."""

    arrival_s: float
    server: str | None = None
    remaining_s: float | None = None
    started_s: float | None = None
    completed_s: float | None = None


def latency_of(request: Request) -> float:
    if request.completed_s is None:
        raise ValidationError("request has not completed")
    return (request.completed_s - request.arrival_s) * 1000.0


def violates_slo(request: Request, slo_latency_ms: float) -> bool:
    return latency_of(request) > slo_latency_ms


@dataclass
class InitialPod:
    point: ConfigPoint
    quota_request: float | None = None


@dataclass
class FunctionSpec:
    profile: FunctionProfile
    trace: WorkloadTrace
    initial_pods: list = field(default_factory=list)
    max_queue: int | None = None

    @property
    def function_id(self) -> str:
        return self.profile.function_id


@dataclass
class Scenario:
    fleet_size: int
    windows: int
    functions: list
    window_ms: float = 1000.0
    epoch_windows: int = 5
    quantum: float = 0.02
    cold_start_windows: int = 2
    seed: int = 0
    model_sharing: bool = True
    gpu_capacity_mb: float = DEFAULT_GPU_MEMORY_MB
    restructure_threshold: int = DEFAULT_RESTRUCTURE_THRESHOLD

    def validate(self) -> None:
        validate_scenario(self)

    @classmethod
    def from_dict(cls, data: dict, base_dir: str | None = None) -> "Scenario":
        if not isinstance(data, dict):
            raise ValidationError("scenario must be a JSON object")
        try:
            fns = [_function_from_dict(f, data, base_dir) for f in data.get("functions", [])]
            sc = cls(
                fleet_size=int(data["fleet_size"]),
                windows=int(data["windows"]),
                functions=fns,
                window_ms=float(data.get("window_ms", 1000.0)),
                epoch_windows=int(data.get("epoch_windows", 5)),
                quantum=float(data.get("quantum", 0.02)),
                cold_start_windows=int(data.get("cold_start_windows", 2)),
                seed=int(data.get("seed", 0)),
                model_sharing=bool(data.get("model_sharing", True)),
                gpu_capacity_mb=float(data.get("gpu_capacity_mb", DEFAULT_GPU_MEMORY_MB)),
                restructure_threshold=int(data.get("restructure_threshold",
                                                   DEFAULT_RESTRUCTURE_THRESHOLD)),
            )
        except KeyError as exc:
            raise ValidationError(f"scenario is missing required field {exc.args[0]!r}")
        except (TypeError, ValueError) as exc:
            raise ValidationError(f"scenario field has wrong type: {exc}")
        sc.validate()
        return sc

    @classmethod
    def from_json(cls, path) -> "Scenario":
        try:
            with open(path, "r", encoding="utf-8") as fh:
                data = json.load(fh)
        except OSError as exc:
            raise ValidationError(f"cannot read scenario {path!r}: {exc}") from exc
        except json.JSONDecodeError as exc:
            raise ValidationError(f"scenario {path!r} is not valid JSON: {exc}") from exc
        return cls.from_dict(data, base_dir=os.path.dirname(os.path.abspath(path)))


def steps_per_window(quantum: float) -> int:
    return round(1.0 / quantum)


def validate_scenario(sc, memo: dict | None = None) -> None:
    """Scenario preconditions, in the reference's order (sim_engine.py:132-170).

    Works on this package's ``Scenario`` and on the reference's (duck typed).
    ``memo``: the compiler's per-call dict; a profile object whose full-quota
    points were checked earlier in the same call is not re-checked.
    """
    def need(ok, msg):
        if not ok:
            raise ValidationError(msg)

    need(sc.fleet_size >= 1, f"fleet_size must be >= 1, got {sc.fleet_size!r}")
    need(sc.windows >= 1, f"windows must be >= 1, got {sc.windows!r}")
    need(sc.epoch_windows >= 1, f"epoch_windows must be >= 1, got {sc.epoch_windows!r}")
    need(math.isfinite(sc.window_ms) and sc.window_ms > 0,
         f"window_ms must be positive, got {sc.window_ms!r}")
    need(0 < sc.quantum <= 1, f"quantum must be in (0, 1], got {sc.quantum!r}")
    steps = steps_per_window(sc.quantum)
    need(steps >= 1 and abs(steps * sc.quantum - 1.0) <= 1e-9,
         f"quantum {sc.quantum!r} must divide the window evenly")
    need(sc.cold_start_windows >= 0,
         f"cold_start_windows must be >= 0, got {sc.cold_start_windows!r}")
    need(sc.gpu_capacity_mb > 0, f"gpu_capacity_mb must be positive, got {sc.gpu_capacity_mb!r}")
    need(sc.restructure_threshold >= 0, "restructure_threshold must be >= 0")
    seen = set()
    for fn in sc.functions:
        fid = fn.function_id
        need(fid not in seen, f"duplicate function id {fid!r}")
        seen.add(fid)
        entries = fn.profile.entries
        done = memo is not None and memo.get(("full-quota", id(fn.profile))) is fn.profile
        if not done:
            # (sm, 1.0) in entries, by field values (ConfigPoint equality is
            # field-tuple equality; no point objects are built)
            keys = {(p.sm_partition, p.quota) for p in entries}
            for sm in sorted({k[0] for k in keys}):
                need((sm, 1.0) in keys,
                     f"{fid}: profile needs the full-quota point ({sm:g}, 1.0) "
                     f"to derive the serving rate")
            if memo is not None:
                memo[("full-quota", id(fn.profile))] = fn.profile
        for init in fn.initial_pods:
            need(init.point in entries,
                 f"{fid}: initial pod point ({init.point.sm_partition:g}, "
                 f"{init.point.quota:g}) is not profiled")


@functools.lru_cache(maxsize=4096)
def _synth_cached(fid, t_max, knee, grid_sm, grid_q, slo_ms, mem_items):
    """One FunctionProfile object per distinct synth spec: profiles are
    immutable inputs, and sharing the object lets the compiler reuse its
    lowered point table across the scenarios of a sweep."""
    mem = MemorySpec(**dict(mem_items)) if mem_items else None
    return synth_profile(fid, t_max, knee, grid_points(list(grid_sm), list(grid_q)),
                         slo_latency_ms=slo_ms, mem=mem)


def _function_from_dict(data: dict, scenario: dict, base_dir: str | None) -> FunctionSpec:
    fid = data.get("function_id")
    if not fid:
        raise ValidationError("function entry needs a function_id")
    prof = data.get("profile")
    if not isinstance(prof, dict):
        raise ValidationError(f"{fid}: function entry needs a profile object")
    if "synth" in prof:
        s = prof["synth"]
        profile = _synth_cached(fid, float(s["t_max"]), float(s["sm_knee"]),
                                tuple(s.get("grid_sm", DEFAULT_SM_GRID)),
                                tuple(s.get("grid_quota", DEFAULT_QUOTA_GRID)),
                                float(s.get("slo_ms", 1000.0)),
                                tuple(sorted(s["mem"].items())) if s.get("mem") else None)
    elif "csv" in prof:
        path = prof["csv"]
        if base_dir is not None and not os.path.isabs(path):
            path = os.path.join(base_dir, path)
        table = ingest_profiles(path)
        if fid not in table:
            raise ValidationError(f"{fid}: not found in profile file {path!r}")
        profile = table[fid]
    else:
        raise ValidationError(f"{fid}: profile must have a 'synth' or 'csv' key")
    windows = int(scenario["windows"])
    window_s = float(scenario.get("window_ms", 1000.0)) / 1000.0
    seed = int(scenario.get("seed", 0))
    trace = trace_from_spec(data.get("trace", {"kind": "constant", "rps": 0.0}),
                            windows, window_s, seed, base_dir)
    inits = []
    for p in data.get("initial_pods", []):
        q_req = p.get("quota_request")
        inits.append(InitialPod(ConfigPoint(float(p["sm"]), float(p["quota"])),
                                None if q_req is None else float(q_req)))
    mq = data.get("max_queue")
    return FunctionSpec(profile, trace, initial_pods=inits,
                        max_queue=None if mq is None else int(mq))
