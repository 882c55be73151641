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


def all_gather_summaries(summary: np.ndarray, n_total: int, group=None, device=None) -> np.ndarray:
    """All-gather every rank's gs_summary_t records into run order.

    Blocks may differ in length by one run, so each rank pads to the largest
    block; the padding is dropped after the gather.  ``device`` selects where
    the payload lives (a CUDA device for NCCL, None/CPU for gloo).
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = max(len(shard(n_total, r, world)) for r in range(world))
    item = SUMMARY_DT.itemsize
    buf = np.zeros(per, SUMMARY_DT)
    buf[:len(summary)] = summary
    send = torch.from_numpy(buf.view(np.uint8).copy())
    if device is not None:
        send = send.to(device)
    recv = torch.empty(per * item * world, dtype=torch.uint8, device=send.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    raw = recv.cpu().numpy().view(SUMMARY_DT).reshape(world, per)
    parts = [raw[r, :len(shard(n_total, r, world))] for r in range(world)]
    out = np.concatenate(parts) if parts else np.zeros(0, SUMMARY_DT)
    assert len(out) == n_total and rank < world
    return out


def run_sharded(scenarios, policies="fast", *, device=None, group=None):
    """Simulate this rank's shard on its GPU and all-gather the summaries.

    Returns (local RunResults, global summary array in input order).
    """
    import torch
    import torch.distributed as dist
    from .engine import simulate
    scenarios = list(scenarios)
    if isinstance(policies, str):
        policies = [policies] * len(scenarios)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = shard(len(scenarios), rank, world)
    dev = torch.cuda.current_device() if device is None else device
    local = simulate([scenarios[i] for i in mine], [policies[i] for i in mine], device=dev)
    summ = np.array([r.summary for r in local], SUMMARY_DT) if local else np.zeros(0, SUMMARY_DT)
    return local, all_gather_summaries(summ, len(scenarios), group=group,
                                       device=torch.device("cuda", dev))


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
