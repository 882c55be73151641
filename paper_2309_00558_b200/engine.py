"""Public entry points: ``run`` / ``compare_policies`` / ``run_batch``.

Drop-in for sim_engine.py:601-612.  A call compiles each (scenario, policy)
on the host (``compiler.py``), executes the whole batch in the sm_100a kernel
through the C ABI (``backend.py``), and decodes the fixed-size device records
into the reference's ``MetricsReport`` rows, in the reference's append order
(sim_engine.py:555-589), so ``to_csv()`` / ``summary()`` are byte-identical.

There is no CPU fallback: without the CUDA library or a GPU every call raises
``BackendUnavailableError``.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import compiler as cc
from .errors import CapacityError, InvariantError, ValidationError
from .metrics import FunctionWindowRow, GlobalWindowRow, GpuWindowRow, MetricsReport
from .scenario import POLICIES

_MAX_CAP_RETRIES = 16


@dataclass
class RunResult:
    """Everything one device run reports."""

    report: MetricsReport
    # final packer state: node -> {pod_id: (x, y, w, h) as exact Fractions}
    placements: dict = field(default_factory=dict)
    token_grants: int = 0
    scale_decisions: int = 0
    placement_attempts: int = 0
    summary: object = None          # gs_summary_t record (all-gather payload)
    pod_steps: int = 0              # registered-pod x quantum-step updates
    rect_scans: int = 0             # free rectangles examined by best_match
    peak_pods: int = 0              # most pods alive at once

    @property
    def decisions(self) -> int:
        return self.token_grants + self.scale_decisions + self.placement_attempts


def run_error(image: cc.RunImage, status) -> Exception | None:
    """Map a device status record to the exception the reference would raise."""
    code = int(status["code"])
    if code == cc.GS_OK:
        return None
    if code == cc.GS_ERR_VALIDATION:
        f, k = int(status["arg0"]), int(status["arg1"])
        if int(status["detail"]) == cc.GS_VAL_NO_THROUGHPUT:
            # autoscaler.py:115-117
            return ValidationError(f"{image.fids[f]}: no profiled point has positive throughput")
        sm_eff = float(image.points[k + int(image.funcs[f]["point_off"])]["sm_eff"])
        # sim_engine.py:346-349
        return ValidationError(f"{image.fids[f]}: zero serving rate at ({sm_eff:g}, 1.0)")
    if code == cc.GS_ERR_CAPACITY:
        return CapacityError(f"device capacity exceeded (detail {int(status['detail'])})")
    if code == cc.GS_ERR_INVARIANT:
        return InvariantError(f"device reported an invariant breach (detail "
                              f"{int(status['detail'])}, {int(status['arg0'])}, "
                              f"{int(status['arg1'])})")
    return InvariantError(f"device returned code {code}")


def decode_run(batch: cc.Batch, r: int, out: dict) -> RunResult:
    """Rebuild the reference's report rows for run ``r`` from device records."""
    from .report import decode_rows
    im = batch.images[r]
    s = batch.runs[r]
    G = int(s["n_nodes"])
    rep = MetricsReport(im.policy, *decode_rows(batch, out, r))
    st = out["status"][r]
    res = RunResult(rep, token_grants=int(st["token_grants"]),
                    scale_decisions=int(st["scale_decisions"]),
                    placement_attempts=int(st["placement_attempts"]),
                    summary=out["summary"][r].copy(),
                    pod_steps=int(st["pod_steps"]), rect_scans=int(st["rect_scans"]),
                    peak_pods=int(st["peak_pods"]))
    pl = out["placements"][int(s["place_off"]): int(s["place_off"]) + int(st["n_placements"])]
    fids = im.fids
    nodes: dict = {g: {} for g in range(G)}
    for node, func, counter, x, y, w_, h, _ in pl.tolist():
        pod_id = f"{fids[func]}-{counter:04d}"
        nodes[node][pod_id] = (Fraction(x, im.scale_x), Fraction(y, im.scale_y),
                               Fraction(w_, im.scale_x), Fraction(h, im.scale_y))
    res.placements = nodes
    return res


def _normalise(scenarios, policies):
    # an indexable sequence (e.g. workloads.ScenarioSeq) stays lazy: the
    # lowering workers build its scenarios themselves
    if not (hasattr(scenarios, "__getitem__") and hasattr(scenarios, "__len__")):
        scenarios = list(scenarios)
    if isinstance(policies, str):
        policies = [policies] * len(scenarios)
    policies = list(policies)
    if len(policies) != len(scenarios):
        raise ValidationError("need one policy per scenario")
    return scenarios, policies


def _pinned_mode(batch):
    # row buffers in recycled page-locked memory: the kernel writes them in
    # place while it runs (zero-copy), no pageable D2H afterwards
    return "pool" if batch.n_fn_rows * 20 + batch.n_gpu_rows * 32 < (6 << 30) else False


def _api_workers():
    """Lowering processes of the pipelined API: the GPU, not the host, bounds
    a large batch once the first block is on the device, and every forked
    worker costs ~9 ms of page-table copying before the first block can start
    (GS_API_WORKERS overrides)."""
    import os
    env = os.environ.get("GS_API_WORKERS")
    if env:
        return max(1, int(env))
    return max(1, min(8, (os.cpu_count() or 1) // 2))


def _api_parts(n):
    import os
    env = os.environ.get("GS_API_PARTS")
    if env:
        return max(1, int(env))
    return None                   # compile_stream's default


def _run_part(batch, device):
    from . import backend
    return backend.run_batch(batch, device=device, rows=True,
                             out=batch.alloc_outputs(rows=True, pinned=_pinned_mode(batch)))


def simulate_records(scenarios, policies="fast", *, device: int = 0, errors: str = "raise",
                     caps: cc.Caps | None = None, on_block=None) -> list:
    """Run a batch of (scenario, policy) pairs on the GPU; raw device records.

    Returns one ``(batch, out, r)`` handle per input -- run ``r`` of the
    compiled ``batch`` whose output arrays are ``out`` -- or the exception
    (``errors="return"``).  Runs that outgrow a static device capacity are
    re-executed on the device with enlarged capacities; nothing is truncated.
    ``decode_run`` / ``report.run_csv`` turn a handle into report rows.

    Host lowering and the GPU are pipelined: ``compiler.compile_stream``
    yields the batch in consecutive blocks as the host cores finish them, and
    each block goes to the GPU at once as its own stream-ordered one-shot call
    (``gs_run_batch`` on a private stream, issued from a host thread, GIL
    released), so the GPU simulates block k while the host lowers block k+1
    and the blocks' kernels overlap on the device.  ``on_block(batch, out)``
    (optional) runs on the calling thread as each block's results arrive,
    while later blocks are still on the GPU.
    """
    from concurrent.futures import ThreadPoolExecutor
    scenarios, policies = _normalise(scenarios, policies)
    results: list = [None] * len(scenarios)
    images: list = [None] * len(scenarios)
    failed: dict = {}
    jobs = []
    with ThreadPoolExecutor(max_workers=16, thread_name_prefix="gs-gpu") as pool:
        for batch, index, errs in cc.compile_stream(scenarios, policies, caps,
                                                    workers=_api_workers(), parts=_api_parts(len(scenarios))):
            failed.update(errs)
            if any(errors == "raise" or not isinstance(e, ValidationError)
                   for e in errs.values()):
                break          # it will be raised: lower and simulate no further blocks
            if len(batch):
                jobs.append((pool.submit(_run_part, batch, device), batch, index))
        outs = []
        for fut, batch, index in jobs:
            outs.append(fut.result())          # re-raises a backend failure
            if on_block is not None:
                on_block(batch, outs[-1])
    for i, exc in sorted(failed.items()):
        if errors == "raise" or not isinstance(exc, ValidationError):
            raise exc
        results[i] = exc
    retry: list = []
    for (_fut, batch, index), out in zip(jobs, outs):
        retry += _settle(batch, out, index, scenarios, policies, images, results, errors)
    pending = retry
    for _attempt in range(_MAX_CAP_RETRIES - 1):
        if not pending:
            break
        batch = cc.Batch([images[i] for i in pending])
        out = _run_part(batch, device)
        pending = _settle(batch, out, pending, scenarios, policies, images, results, errors)
    for i in pending:
        err = CapacityError("run still exceeds device capacities after "
                            f"{_MAX_CAP_RETRIES} enlargements")
        if errors == "raise":
            raise err
        results[i] = err
    return results


def _settle(batch, out, index, scenarios, policies, images, results, errors) -> list:
    """Record each run of a finished block; returns the input positions to
    re-run with grown capacities (recompiled into ``images``)."""
    codes = out["status"]["code"]
    retry = []
    for j in np.flatnonzero(codes != 0).tolist():
        i = index[j]
        st = out["status"][j]
        if int(st["code"]) == cc.GS_ERR_CAPACITY:
            rr = batch.runs[j]
            caps_j = cc.Caps(int(rr["cap_pods"]), int(rr["cap_rects"]),
                             int(rr["cap_returned"]), int(rr["hot_class"])
                             ).grown(int(st["detail"]), int(st["hot_class"]))
            images[i] = cc.compile_run(scenarios[i], policies[i], caps_j)
            retry.append(i)
            continue
        err = run_error(batch.images[j], st)
        if err is not None:
            if errors == "raise":
                raise err
            results[i] = err
    again = set(retry)
    for j, i in enumerate(index):
        if results[i] is None and i not in again:
            results[i] = (batch, out, j)
    return retry


def simulate(scenarios, policies="fast", *, device: int = 0, errors: str = "raise",
             rows: bool = True, caps: cc.Caps | None = None) -> list:
    """Run a batch of (scenario, policy) pairs on the GPU.

    Returns one ``RunResult`` per input (or the exception, when
    ``errors="return"``).  Runs that outgrow a static device capacity are
    re-executed on the device with doubled capacities; nothing is truncated.
    """
    recs = simulate_records(scenarios, policies, device=device, errors=errors, caps=caps)
    return [r if isinstance(r, Exception) else decode_run(r[0], r[2], r[1]) for r in recs]


def run_batch(scenarios, policies="fast", *, device: int = 0, errors: str = "raise") -> list:
    """Batch form of ``run``: one ``MetricsReport`` (or exception) per input.

    The reports are ``report.DeviceReport``s: rows stay in the device records
    until touched, ``to_csv()`` renders natively and ``summary()`` comes from
    one vectorised reduction over the whole batch -- same values, same bytes."""
    from .report import DeviceReport, SharedOutputs
    shared: dict = {}

    def ready(batch, out):
        # summaries of a finished block, computed while later blocks simulate
        sh = shared[id(out)] = SharedOutputs(batch, out)
        sh.prepare()

    recs = simulate_records(scenarios, policies, device=device, errors=errors, on_block=ready)
    reps = []
    for r in recs:
        if isinstance(r, Exception):
            reps.append(r)
            continue
        batch, out, j = r
        sh = shared.get(id(out))
        if sh is None:
            sh = shared[id(out)] = SharedOutputs(batch, out)
        reps.append(DeviceReport(sh, j))
    return reps


def run(scenario, policy: str = "fast") -> MetricsReport:
    """Simulate one scenario under one policy (sim_engine.py:601-603)."""
    return run_batch([scenario], [policy])[0]


def compare_policies(scenario, policies=POLICIES) -> dict:
    """Each policy on the same scenario, fresh state (sim_engine.py:606-612)."""
    for p in policies:
        if p not in POLICIES:
            raise ValidationError(f"unknown policy {p!r}")
    res = run_batch([scenario] * len(policies), list(policies))
    return dict(zip(policies, res))
