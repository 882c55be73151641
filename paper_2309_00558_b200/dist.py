"""Multi-GPU execution: scenario sharding + one all-gather of summaries.

Runs share nothing mutable (the reference's concurrency model: "multiple
scenario runs may execute in parallel, sharing only immutable profiles",
SPEC.md:489-490), so a batch is split into contiguous per-rank blocks, each
rank simulates its block end to end on its own GPU with no data-path
collective, and the fixed-size per-run summary records (``gs_summary_t``,
72 bytes) are all-gathered once at the end -- NCCL over NVLink/NVSwitch on a
GPU box, gloo in the CPU tests.  Within one scenario nodes cannot be sharded
(the per-function FIFO is drained across nodes every quantum step,
sim_engine.py:514-531, and best_match is a fleet-wide argmin,
packer.py:184-192), so a single run never spans GPUs.
"""
from __future__ import annotations

import numpy as np

from .compiler import SUMMARY_DT


def shard(n_total: int, rank: int, world: int) -> range:
    """Contiguous, balanced block of run indices owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def _gather_padded(arr: np.ndarray, n_total: int, group, device) -> np.ndarray:
    """All-gather one fixed-size record per run (any structured dtype) into
    run order.  Blocks differ in length by at most one run, so each rank pads
    to the largest block; the padding is dropped after the gather."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    per = max(len(shard(n_total, r, world)) for r in range(world))
    item = arr.dtype.itemsize
    buf = np.zeros(per, arr.dtype)
    buf[:len(arr)] = arr
    send = torch.from_numpy(buf.view(np.uint8).copy())
    if device is not None:
        send = send.to(device)
    recv = torch.empty(per * item * world, dtype=torch.uint8, device=send.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    raw = recv.cpu().numpy().view(arr.dtype).reshape(world, per)
    parts = [raw[r, :len(shard(n_total, r, world))] for r in range(world)]
    out = np.concatenate(parts) if parts else np.zeros(0, arr.dtype)
    assert len(out) == n_total
    return out


def all_gather_summaries(summary: np.ndarray, n_total: int, group=None, device=None) -> np.ndarray:
    """All-gather every rank's gs_summary_t records into run order.

    ``device`` selects where the payload lives (a CUDA device for NCCL,
    None/CPU for gloo).
    """
    return _gather_padded(np.asarray(summary, SUMMARY_DT), n_total, group, device)


STATUS_REC_DT = np.dtype([("code", "<i4"), ("pad", "<i4")])


def gather_outcomes(local, n_total: int, group=None, device=None):
    """Gather the summaries AND a status code per run.

    ``local`` holds this rank's RunResults or exceptions (simulate(...,
    errors="return")).  A failed run contributes a zeroed summary and a
    non-zero code, so one bad scenario never leaves the other ranks blocked
    in the collective: every rank takes part in both gathers and sees the same
    global code array.
    """
    summ = np.zeros(len(local), SUMMARY_DT)
    codes = np.zeros(len(local), STATUS_REC_DT)
    for i, r in enumerate(local):
        if isinstance(r, Exception):
            codes[i]["code"] = 1
        else:
            summ[i] = r.summary
    return (all_gather_summaries(summ, n_total, group=group, device=device),
            _gather_padded(codes, n_total, group, device)["code"])


def run_sharded(scenarios, policies="fast", *, device=None, group=None, errors: str = "raise"):
    """Simulate this rank's shard on its GPU and all-gather the summaries.

    Returns (local RunResults, global summary array in input order).  Errors
    are collected first and raised only after the gathers, on EVERY rank
    (``errors="raise"``), so a failing scenario cannot hang the collective;
    with ``errors="return"`` failed runs come back as exceptions (local) and
    zeroed summaries (global).
    """
    import torch
    import torch.distributed as dist
    from .engine import simulate
    scenarios = list(scenarios)
    if isinstance(policies, str):
        policies = [policies] * len(scenarios)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = shard(len(scenarios), rank, world)
    if device is None and torch.cuda.is_available():
        device = torch.cuda.current_device()
    try:
        local = simulate([scenarios[i] for i in mine], [policies[i] for i in mine],
                         device=device or 0, errors="return")
    except Exception as exc:              # whole-shard failure (no device, ...)
        local = [exc] * len(mine)
    where = torch.device("cuda", device) if device is not None else None
    summ, codes = gather_outcomes(local, len(scenarios), group=group, device=where)
    if errors == "raise":
        bad = np.flatnonzero(codes)
        if len(bad):
            first = int(bad[0])
            if first in mine:
                raise local[first - mine.start]
            from .errors import GShareError
            raise GShareError(f"scenario {first} failed on another rank "
                              f"({len(bad)} failed runs in total)")
    return local, summ


def summary_totals(summary: np.ndarray) -> dict:
    """Fleet-level aggregates of a gathered summary array (host side)."""
    comp = int(summary["completions"].sum())
    viol = int(summary["slo_violations"].sum())
    rows = int(summary["n_gpu_rows"].sum())
    return {
        "runs": int(len(summary)),
        "arrivals": int(summary["arrivals"].sum()),
        "completions": comp,
        "slo_violation_pct": round(100.0 * viol / comp, 6) if comp else 0.0,
        "dropped": int(summary["dropped"].sum()),
        "placement_failures": int(summary["placement_failures"].sum()),
        "mean_utilization": float(summary["sum_utilization"].sum() / rows) if rows else 0.0,
        "mean_sm_occupancy": float(summary["sum_sm_occupancy"].sum() / rows) if rows else 0.0,
    }
