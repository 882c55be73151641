"""CLI front end: argument surface and exit codes of the
reference's ``gshare run|compare`` (cli.py:162-227) on the CUDA backend, plus
the batched ``sweep``.  Simulation itself needs a GPU (marked); argument and
error handling run on the CPU."""
import json
import os

import pytest

from paper_2309_00558_b200 import cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _scenario_file(tmp_path, windows=8):
    from paper_2309_00558_b200 import workloads as wl
    p = tmp_path / "c3.json"
    p.write_text(json.dumps(wl.c3(3, windows=windows)))
    return str(p)


def test_parser_mirrors_reference_commands():
    p = cli.build_parser()
    a = p.parse_args(["run", "--scenario", "x.json", "--policy", "timeshare", "--out", "d",
                      "--seed", "7"])
    assert (a.command, a.policy, a.out, a.seed) == ("run", "timeshare", "d", 7)
    a = p.parse_args(["compare", "--scenario", "x.json"])
    assert a.command == "compare"
    a = p.parse_args(["--backend", "cuda", "sweep", "--scenario", "x.json", "--seeds", "0:4,9",
                      "--policy", "both"])
    assert cli._parse_seeds(a.seeds) == [0, 1, 2, 3, 9]
    with pytest.raises(SystemExit):
        p.parse_args(["--backend", "cpu", "run", "--scenario", "x.json"])


def test_missing_file_exits_1(capsys):
    assert cli.main(["run", "--scenario", "/nonexistent/s.json"]) == cli.EXIT_ERROR
    assert "error:" in capsys.readouterr().err


def test_validation_error_exits_1(tmp_path, capsys):
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"schema_version": 1, "fleet_size": 0, "windows": 3,
                               "functions": []}))
    assert cli.main(["run", "--scenario", str(bad)]) == cli.EXIT_ERROR


def test_no_gpu_is_an_error_not_a_fallback(tmp_path, capsys):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert cli.main(["run", "--scenario", _scenario_file(tmp_path)]) == cli.EXIT_ERROR
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_run_compare_and_sweep_on_gpu(tmp_path, capsys):
    import oracle
    from paper_2309_00558_b200 import compiler as cc, engine
    from paper_2309_00558_b200.scenario import Scenario
    path = _scenario_file(tmp_path, windows=12)
    assert cli.main(["run", "--scenario", path, "--out", str(tmp_path / "r")]) == 0
    sc = Scenario.from_json(path)
    batch = cc.Batch([cc.compile_run(sc, "fast")])
    want = engine.decode_run(batch, 0, oracle.run_batch(batch)).report
    assert (tmp_path / "r" / "metrics.csv").read_text() == want.to_csv()
    assert cli.main(["compare", "--scenario", path, "--out", str(tmp_path / "c")]) == 0
    assert (tmp_path / "c" / "timeshare" / "metrics.csv").exists()
    capsys.readouterr()
    assert cli.main(["sweep", "--scenario", path, "--seeds", "0:6", "--policy", "both",
                     "--out", str(tmp_path / "s")]) == 0
    recs = [json.loads(l) for l in (tmp_path / "s" / "sweep.jsonl").read_text().splitlines()]
    assert len(recs) == 12 and all("summary" in r for r in recs)
    d = json.loads(open(path).read())
    d["seed"] = 4
    sc4 = Scenario.from_dict(d)
    b4 = cc.Batch([cc.compile_run(sc4, "timeshare")])
    want4 = engine.decode_run(b4, 0, oracle.run_batch(b4)).report
    assert (tmp_path / "s" / "timeshare" / "seed-4" / "metrics.csv").read_text() == want4.to_csv()
