"""Benchmark: simulated scenario-seconds/s of the batched FaST-GShare engine.

Workload (BASELINE.json configs[1]): 4-node cluster,
10 MLPerf-shaped functions (ResNet-50 / RNN-T / BERT profiles), Poisson
constant-rate traces, heuristic auto-scaling with model sharing, 300 one-second
windows, policy "fast"; ``--runs`` independent seeds per GPU (weak scaling:
each rank simulates its own seed block, no data-path collective; one NCCL
all-gather of the per-run summary records at the end).

A "step" = one launch of the scenario megakernel over the GPU's whole batch.
``value``  = total simulated scenario-seconds / device time of the K timed
             launches (CUDA events on the launching stream, max over ranks),
             inputs already resident in HBM, L2 flushed between launches.
``e2e``    = same metric through the C ABI with host buffers, every step:
             H2D of the compiled batch from page-locked memory
             (gs_session_upload), the kernel, and every output row back in
             host memory (written in place by the kernel into page-locked
             buffers) plus the status/summary D2H -- host wall clock, max
             over ranks.
``--impl reference`` times the CPU oracle port (oracle/, a literal C
restatement of pkg/src/gshare_sim, pinned to the reference by golden
fixtures) on all host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

def workload(windows: int) -> str:
    return ("C2: 4-node cluster, 10 functions (ResNet-50/RNN-T/BERT-shaped), Poisson "
            f"arrivals, heuristic auto-scaling, model sharing, {windows} x 1 s windows, policy fast")
METRIC = "simulated scenario-seconds/sec"
UNIT = "scenario-s/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_c2_summary.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("cuda", "reference"), default="cuda")
    ap.add_argument("--runs", type=int, default=21312,
                    help="scenario runs per GPU (6 waves of 24 resident runs x 148 SMs)")
    ap.add_argument("--windows", type=int, default=300)
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="runs in the CPU baseline sample (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def build_batch(seeds, windows):
    from paper_2309_00558_b200 import compiler as cc, workloads as wl
    scen = wl.c2_scenarios(seeds, windows=windows)
    return cc.Batch([cc.compile_run(s, "fast") for s in scen])


def sim_seconds(batch) -> float:
    r = batch.runs
    return float((r["windows"].astype("f8") * r["window_s"]).sum())


def algorithmic_bytes(batch, status, summary) -> float:
    """SURVEY.md §8(d) state-touch model, per launch:
    88 B per registered pod per quantum step, 32 B per function and 48 B per
    node per step, per window 24 B/function + 24 B/used GPU + 16 B, per
    best_match 16 B per free rect scanned, per epoch 40 B per profile point."""
    r = batch.runs
    steps_total = (r["windows"].astype("f8") * r["steps"])
    per_step = 32.0 * r["n_funcs"] + 48.0 * r["n_nodes"]
    epochs = (r["windows"] - 1) // r["epoch_windows"]
    k_points = 35.0
    b = (88.0 * status["pod_steps"].astype("f8") + steps_total * per_step
         + r["windows"] * (24.0 * r["n_funcs"] + 16.0) + 24.0 * summary["n_gpu_rows"]
         + 16.0 * status["rect_scans"] + 40.0 * k_points * r["n_funcs"] * epochs)
    return float(b.sum())


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in getattr(self, "lines", []):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        loaded = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference(batch, sample_runs: int, threads: int):
    """Time the oracle port on `sample_runs` runs of the workload."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    from paper_2309_00558_b200 import compiler as cc
    sub = cc.Batch(batch.images[:sample_runs])
    oracle.build()
    t0 = time.perf_counter()
    oracle.run_batch(sub, n_threads=threads, rows=True)
    dt = time.perf_counter() - t0
    return sim_seconds(sub) / dt, dt, sub


def cpu_sample_size(batch, threads: int, target_s: float) -> int:
    """Runs of `batch` the oracle finishes in about `target_s` seconds on
    `threads` host threads (calibrated on a small prefix)."""
    n0 = min(len(batch), max(4 * threads, 64))
    _, dt, _ = cpu_reference(batch, n0, threads)
    return int(min(len(batch), max(n0, n0 * target_s / max(dt, 1e-3))))


def fleet_totals(summary):
    from paper_2309_00558_b200.dist import summary_totals
    return summary_totals(summary)


def load_peak():
    try:
        with open(PEAKS) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic():
    try:
        with open(NCU_SUMMARY) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def measure_e2e(args, batch, sess, device, dist, compile_s):
    """The same metric through the C ABI with host buffers: every step uploads
    the batch from page-locked host memory (gs_session_upload), runs the kernel,
    and reads every result back (rows written in place into page-locked host
    memory by the kernel, status + summary by D2H).  Host wall clock around the
    steps, max over ranks."""
    import torch
    batch.pin()
    out = batch.alloc_outputs(rows=True, pinned=True)
    sess.map_host(out)

    def step():
        sess.upload()
        sess.run()
        sess.download_into(out)

    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    world = dist.get_world_size() if dist is not None else 1
    out_bytes = sum(v.nbytes for v in out.values() if v is not None)
    sess.map_host(None)
    return {"value": sim_seconds(batch) * world * args.steps / dt, "unit": UNIT,
            "h2d_bytes_per_step": int(batch.input_bytes()),
            "d2h_bytes_per_step": int(out_bytes),
            "ms_per_step": 1000.0 * dt / args.steps,
            "api": "C ABI session: gs_session_upload (pinned H2D) + gs_session_run + "
                   "gs_session_download; rows written in place into pinned host memory",
            "host_compile_s": round(compile_s, 3)}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    # each step is a bounded sample (~8 s of CPU work) of the same workload
    pool = build_batch(range(args.cpu_sample or 4096), args.windows)
    sample = args.cpu_sample or cpu_sample_size(pool, threads, 8.0)
    batch = build_batch(range(sample), args.windows) if sample > len(pool) else pool
    for _ in range(args.warmup):
        cpu_reference(batch, min(sample, 2 * threads), threads)
    times, simsec = [], []
    for _ in range(args.steps):
        _, dt, sub = cpu_reference(batch, sample, threads)
        simsec.append(sim_seconds(sub))           # the sample actually simulated
        times.append(dt)
    value = sum(simsec) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(args.windows), "runs_per_step": sample, "windows": args.windows},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} C2 runs x {args.windows} windows per step "
                                   f"(oracle/gs_oracle.c, {threads} host threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
        rc = run_reference_arm(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return rc

    import numpy as np
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2309_00558_b200 import backend

    seeds = range(rank * args.runs, (rank + 1) * args.runs)
    t_c = time.perf_counter()
    batch = build_batch(seeds, args.windows)
    compile_s = time.perf_counter() - t_c
    sess = backend.Session(batch, device=local)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        flush.zero_()
        torch.cuda.synchronize()
        sess.run()
    kernel_ms = []
    launches = 0
    with ClockSampler(local) as clk:
        barrier()
        for _ in range(args.steps):
            flush.zero_()                      # L2 flush, outside the timed kernel
            torch.cuda.synchronize()
            kernel_ms.append(sess.run())        # CUDA events around the launch
            launches += sess.launches()
        barrier()
    total_ms = sum(kernel_ms)
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    out = sess.download(rows=False)
    bad = int((out["status"]["code"] != 0).sum())

    # NCCL all-gather of the fixed-size per-run summary records
    summ = out["summary"]
    fleet = summ
    if dist is not None:
        from paper_2309_00558_b200 import dist as gdist
        fleet = gdist.all_gather_summaries(summ, args.runs * world,
                                           device=torch.device("cuda", local))
    gathered_runs = len(fleet)
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(args, batch, sess, local, dist, compile_s)
    sim_s = sim_seconds(batch) * world
    value = sim_s / (total_ms / 1000.0 / args.steps)
    st = out["status"]
    decisions = float((st["token_grants"] + st["scale_decisions"] + st["placement_attempts"]).sum())
    dec_per_s = decisions * world / (total_ms / 1000.0 / args.steps)

    line = None
    if rank == 0:
        peak, peak_src = load_peak()
        bytes_launch = algorithmic_bytes(batch, st, summ)
        achieved = bytes_launch / (total_ms / args.steps / 1000.0) / 1e9
        traffic = load_traffic()
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            threads = os.cpu_count() or 1
            sample = args.cpu_sample or cpu_sample_size(batch, threads, 15.0)
            v, dt, _ = cpu_reference(batch, sample, threads)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                   "sample": f"first {sample} of the {len(batch)} C2 runs, {dt:.2f} s wall "
                             f"on {threads} host threads (oracle/gs_oracle.c)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args.windows), "runs_per_gpu": args.runs, "windows": args.windows,
                       "policy": "fast", "l2": "flushed between launches (256 MiB write)",
                       "failed_runs": bad, "summaries_all_gathered": gathered_runs},
            "fleet_summary": fleet_totals(fleet),
            "decisions_per_sec": dec_per_s,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_src,
                         "model": "SURVEY §8d state-touch bytes per launch",
                         "bytes_per_launch": bytes_launch},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    sess.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
