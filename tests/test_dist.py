"""Multi-process host logic on CPU: world_size-2 gloo.

The scenario shard of each rank plus one all-gather of the per-run summary
records must reassemble exactly the single-process result.  The summaries
are produced by the CPU oracle here (no GPU in this container); on a GPU box
the same code path runs with NCCL on device buffers (bench.py, dist.py).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2309_00558_b200 import compiler as cc, dist as gd, workloads as wl


def test_shard_is_a_balanced_partition():
    for n in (0, 1, 7, 64, 4737):
        for world in (1, 2, 3, 8):
            parts = [gd.shard(n, r, world) for r in range(world)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_runs, out_dir):
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scen = wl.c2_scenarios(range(n_runs), windows=40)
    mine = gd.shard(n_runs, rank, world)
    batch = cc.Batch([cc.compile_run(scen[i], "fast") for i in mine])
    local = oracle.run_batch(batch, rows=False)["summary"]
    gathered = gd.all_gather_summaries(local, n_runs)
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), gathered)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_all_gather_reassembles_the_batch(tmp_path):
    import oracle
    n_runs = 13
    mp.spawn(_worker, args=(2, _free_port(), n_runs, str(tmp_path)), nprocs=2, join=True)
    gathered = np.load(tmp_path / "gathered.npy")
    scen = wl.c2_scenarios(range(n_runs), windows=40)
    whole = oracle.run_batch(cc.Batch([cc.compile_run(s, "fast") for s in scen]),
                             rows=False)["summary"]
    assert gathered.tobytes() == whole.tobytes()
    tot = gd.summary_totals(gathered)
    assert tot["runs"] == n_runs and tot["arrivals"] > 0


def _worker_errors(rank, world, port, out_dir):
    """run_sharded with one failing scenario on rank 1: every rank must leave
    the collectives and raise (no rank blocks in the all-gather)."""
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    import parity
    from paper_2309_00558_b200 import engine
    # the CPU oracle stands in for the device here (no GPU in this container)
    engine.simulate = lambda sc, pol, device=0, errors="raise": parity.oracle_results(sc, pol)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scen = wl.c2_scenarios(range(5), windows=12)
    import golden
    # an all-zero CSV profile with demand: ValidationError at the first scale-up
    rec = next(r for r in golden.records() if r["name"] == "err-no-throughput-first-5-2-6")
    scen.append(golden.load_scenario(rec))         # run 5 -> rank 1's shard
    try:
        gd.run_sharded(scen, "fast", device=None)
        outcome = "ok"
    except Exception as exc:                        # noqa: BLE001
        outcome = f"{type(exc).__name__}: {exc}"
    local, summ = gd.run_sharded(scen, "fast", device=None, errors="return")
    with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as fh:
        fh.write(outcome + "\n" + str(int((summ["windows"] == 0).sum())) + "\n")
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_failure_on_one_rank_raises_everywhere(tmp_path):
    mp.spawn(_worker_errors, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r0 = (tmp_path / "r0.txt").read_text().splitlines()
    r1 = (tmp_path / "r1.txt").read_text().splitlines()
    assert r0[0].startswith("GShareError: scenario 5 failed on another rank"), r0
    assert r1[0].startswith("ValidationError"), r1
    assert r0[1] == r1[1] == "1"        # one zeroed summary in the gathered array


def _worker_nccl(rank, world, port, out_dir):
    """dist.run_sharded on the GPU with NCCL (world 1: the box has one GPU):
    the device path, the device-buffer all-gather and the summary records."""
    import torch
    import torch.distributed as dist
    from paper_2309_00558_b200 import engine
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0))
    scen = wl.c2_scenarios(range(40), windows=60)
    local, summ = gd.run_sharded(scen, "fast")
    ref = engine.simulate(scen, "fast")
    same = all(a.report == b.report for a, b in zip(local, ref))
    recs = np.stack([r.summary for r in ref])
    with open(os.path.join(out_dir, "nccl.txt"), "w") as fh:
        fh.write(f"{same} {summ.tobytes() == recs.tobytes()} {len(summ)}\n")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_run_sharded_on_the_gpu_with_nccl(tmp_path):
    mp.spawn(_worker_nccl, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True)
    assert (tmp_path / "nccl.txt").read_text().split() == ["True", "True", "40"]
