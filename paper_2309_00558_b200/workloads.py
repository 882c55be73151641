"""Synthetic MLPerf-shaped workloads C1-C5.

Every builder returns scenario *dicts* in the reference's JSON schema, so the
same inputs can be fed to ``Scenario.from_dict`` of this package or of the
reference.  Profiles are the three MLPerf-shaped synth profiles of
pkg/scenarios/consolidation.json:12-58 (ResNet-50, RNN-T, BERT).
"""
from __future__ import annotations

import random

import numpy as np

KINDS = {
    "resnet": {"t_max": 100.0, "sm_knee": 24.0,
               "mem": {"mem_noshare_mb": 1200.0, "mem_runtime_mb": 900.0, "mem_server_mb": 600.0}},
    "rnnt": {"t_max": 48.0, "sm_knee": 24.0,
             "mem": {"mem_noshare_mb": 1400.0, "mem_runtime_mb": 1000.0, "mem_server_mb": 700.0}},
    "bert": {"t_max": 30.0, "sm_knee": 50.0,
             "mem": {"mem_noshare_mb": 1600.0, "mem_runtime_mb": 1100.0, "mem_server_mb": 800.0}},
}
KIND_ORDER = ("resnet", "rnnt", "bert")
DEFAULT_GRID_SM = [6, 12, 24, 50, 60, 80, 100]
DEFAULT_GRID_Q = [0.2, 0.4, 0.6, 0.8, 1.0]


def _synth(kind, slo_ms, grid_sm=None, grid_q=None):
    k = KINDS[kind]
    return {"synth": {"t_max": k["t_max"], "sm_knee": k["sm_knee"],
                      "grid_sm": list(grid_sm or DEFAULT_GRID_SM),
                      "grid_quota": list(grid_q or DEFAULT_GRID_Q),
                      "slo_ms": float(slo_ms), "mem": dict(k["mem"])}}


def c1() -> dict:
    """consolidation.json at 1 node, 60 windows, epoch 5, cold 2 (runs on the CPU ref)."""
    grid = [12, 24, 50, 100]
    fns = []
    for fid, kind, rps, pods in (("resnet_v1", "resnet", 96.0, [(12, 0.4)] * 4),
                                 ("rnnt_asr", "rnnt", 46.0, [(24, 0.4)] * 2),
                                 ("bert_qa", "bert", 43.0, [(50, 0.6)] * 2)):
        fns.append({"function_id": fid, "profile": _synth(kind, 1000.0, grid_sm=grid),
                    "trace": {"kind": "constant", "rps": rps},
                    "initial_pods": [{"sm": s, "quota": q} for s, q in pods]})
    return {"schema_version": 1, "fleet_size": 1, "windows": 60, "epoch_windows": 5,
            "quantum": 0.02, "cold_start_windows": 2, "seed": 0, "functions": fns}


def c2(seed: int, windows: int = 300, n_funcs: int = 10, fleet: int = 4) -> dict:
    """4 nodes, 10 functions, Poisson constant rps ~U(5,60), autoscaling, sharing."""
    rng = random.Random(seed)
    fns = []
    for i in range(n_funcs):
        kind = KIND_ORDER[i % 3]
        fns.append({"function_id": f"{kind}{i:02d}", "profile": _synth(kind, 500.0),
                    "trace": {"kind": "constant", "rps": rng.uniform(5.0, 60.0),
                              "poisson": True, "seed": 100 * seed + i}})
    return {"schema_version": 1, "fleet_size": fleet, "windows": windows, "epoch_windows": 5,
            "quantum": 0.02, "cold_start_windows": 2, "seed": seed, "model_sharing": True,
            "functions": fns}


def bursty_counts(seed: int, i: int, windows: int) -> list:
    """On/off bursty Poisson counts."""
    rng = random.Random(seed * 7919 + i)
    base, burst = rng.uniform(5.0, 30.0), rng.uniform(40.0, 120.0)
    on = False
    rates = []
    for _ in range(windows):
        on = (rng.random() < 0.1) if not on else not (rng.random() < 0.3)
        rates.append(burst if on else base)
    gen = np.random.default_rng(seed * 1000 + i)
    return [int(gen.poisson(r)) for r in rates]


def c3(seed: int, windows: int = 60) -> dict:
    """4 nodes, 6 functions, explicit bursty on/off traces; run under both policies."""
    fns = []
    for i in range(6):
        kind = KIND_ORDER[i % 3]
        fns.append({"function_id": f"{kind}{i:02d}", "profile": _synth(kind, 500.0),
                    "trace": {"kind": "explicit", "counts": bursty_counts(seed, i, windows)},
                    "initial_pods": [{"sm": 24, "quota": 0.4}]})
    return {"schema_version": 1, "fleet_size": 4, "windows": windows, "epoch_windows": 5,
            "quantum": 0.02, "cold_start_windows": 2, "seed": seed, "functions": fns}


def c4(seed: int = 0, windows: int = 3600, n_funcs: int = 200, fleet: int = 64) -> dict:
    """64 nodes, 200 functions, one compressed diurnal day (sinusoid, Poisson)."""
    rng = random.Random(seed)
    fns = []
    for i in range(n_funcs):
        kind = KIND_ORDER[i % 3]
        fns.append({"function_id": f"{kind}{i:03d}",
                    "profile": _synth(kind, rng.choice([200.0, 500.0, 1000.0])),
                    "trace": {"kind": "sinusoid", "base_rps": rng.uniform(5.0, 40.0),
                              "amplitude_rps": rng.uniform(2.0, 30.0),
                              "period_windows": windows, "poisson": True,
                              "seed": 1000 * seed + i},
                    "initial_pods": [{"sm": 24, "quota": 0.6}]})
    return {"schema_version": 1, "fleet_size": fleet, "windows": windows, "epoch_windows": 5,
            "quantum": 0.02, "cold_start_windows": 2, "seed": seed, "gpu_capacity_mb": 81920.0,
            "functions": fns}


C5_SM = (6, 12, 24, 50, 60, 80, 100)
C5_QUANTUM = (0.01, 0.02, 0.04, 0.05, 0.1)
C5_SLO = (50.0, 100.0, 200.0, 500.0, 1000.0)


def c5(index: int, windows: int = 60) -> dict:
    """Run `index` of the 100k parameter sweep: (SM%, quantum, SLO) grid x seeds."""
    sm = C5_SM[index % 7]
    quantum = C5_QUANTUM[(index // 7) % 5]
    slo = C5_SLO[(index // 35) % 5]
    seed = index // 175
    rng = random.Random(index)
    fns = []
    for i in range(3):
        kind = KIND_ORDER[i]
        fns.append({"function_id": f"{kind}{i}", "profile": _synth(kind, slo),
                    "trace": {"kind": "constant", "rps": rng.uniform(5.0, 60.0),
                              "poisson": True, "seed": 100000 * seed + 10 * (index % 175) + i},
                    "initial_pods": [{"sm": sm, "quota": 0.4}]})
    return {"schema_version": 1, "fleet_size": 2, "windows": windows, "epoch_windows": 5,
            "quantum": quantum, "cold_start_windows": 2, "seed": seed, "functions": fns}


def scenarios(dicts):
    from .scenario import Scenario
    return [Scenario.from_dict(d) for d in dicts]


def c2_scenarios(seeds, windows: int = 300):
    """C2 as Scenario objects, built fast: the three MLPerf-shaped profiles are
    immutable and shared across runs (identical to Scenario.from_dict(c2(s)))."""
    from .profiles import grid_points, synth_profile
    from .scenario import FunctionSpec, Scenario
    from .traces import constant_trace
    from .memory import MemorySpec
    prof = {}
    out = []
    for seed in seeds:
        rng = random.Random(seed)
        fns = []
        for i in range(10):
            kind = KIND_ORDER[i % 3]
            k = KINDS[kind]
            key = (kind, f"{kind}{i:02d}")
            p = prof.get(key)
            if p is None:
                p = synth_profile(key[1], k["t_max"], k["sm_knee"],
                                  grid_points(DEFAULT_GRID_SM, DEFAULT_GRID_Q),
                                  slo_latency_ms=500.0, mem=MemorySpec(**k["mem"]))
                prof[key] = p
            rps = rng.uniform(5.0, 60.0)
            fns.append(FunctionSpec(p, constant_trace(rps, windows, 1.0, True, 100 * seed + i)))
        out.append(Scenario(fleet_size=4, windows=windows, functions=fns, epoch_windows=5,
                            quantum=0.02, cold_start_windows=2, seed=seed, model_sharing=True))
    return out


class ScenarioSeq:
    """A sequence of ``n`` scenarios built on first access by ``make(i)`` (a
    Scenario, or a scenario dict).  ``compiler.compile_batch`` indexes it
    inside its worker processes, so large sweeps are also *generated* on all
    host cores."""

    def __init__(self, make, n: int):
        self.make, self.n = make, n

    def __len__(self) -> int:
        return self.n

    def __getitem__(self, i: int):
        if not 0 <= i < self.n:
            raise IndexError(i)
        x = self.make(i)
        if isinstance(x, dict):
            from .scenario import Scenario
            x = Scenario.from_dict(x)
        return x
