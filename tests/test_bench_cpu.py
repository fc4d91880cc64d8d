"""CPU tests of bench.py's host logic: the N-rank self-launcher, the
repetition statistics (bench.cpp:13-45) and the reference arm's rank gating.
No GPU and no process launch: subprocess.run is replaced."""
import json
import subprocess
import sys

import pytest

import bench


def test_defaults_are_the_driver_contract():
    a = bench.parse([])
    assert a.gpus == 1 and a.steps == 20 and a.warmup >= 3
    assert a.field == "gem+E" and a.e2e_steps >= 5 and a.refresh == 1


def test_harmonic_mean_of_equal_work_reps_is_aggregate_rate():
    step_ms = [1.0] * 10 + [2.0] * 10 + [1.5] * 5
    r = bench.harmonic_reps(step_ms, 1_000_000)
    assert r["cycles_per_rep"] == 10 and len(r["mpas"]) == 3
    assert r["mpas"][0] == pytest.approx(1000.0)
    # the harmonic mean of equal-work rates is total work / total time
    full = [r["mpas"][0], r["mpas"][1]]
    hm2 = 2 / sum(1 / m for m in full)
    assert hm2 == pytest.approx(1_000_000 * 20 / (30e-3) / 1e6)


def test_gpus_n_outside_torchrun_self_launches(monkeypatch, capsys):
    seen = {}

    def fake_run(cmd, env=None, stdout=None, text=None):
        seen["cmd"], seen["env"] = cmd, env
        out = ("NCCL INFO comm 0x1 rank 0 nranks 4\n"
               + json.dumps({"metric": "MPA/s in mover", "n_gpus": 4}) + "\n")
        return subprocess.CompletedProcess(cmd, 0, stdout=out)

    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.delenv("NCCL_DEBUG", raising=False)
    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    rc = bench.main(["--gpus", "4", "--steps", "3", "--warmup", "3"])
    assert rc == 0
    cmd = seen["cmd"]
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "3", "--warmup", "3"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"
    out, err = capsys.readouterr()
    lines = [ln for ln in out.splitlines() if ln.strip()]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 4   # one JSON line
    assert "NCCL INFO" in err                                      # the rest to stderr


def test_under_torchrun_no_relaunch(monkeypatch):
    called = {}
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(bench, "run_world", lambda a: (called.__setitem__("world", a.gpus), 0)[1])
    monkeypatch.setattr(bench.subprocess, "run", lambda *a, **k: pytest.fail("relaunched"))
    assert bench.main(["--gpus", "2"]) == 0 and called["world"] == 2


def test_reference_arm_only_on_rank_zero(monkeypatch, capsys):
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setattr(bench, "cpu_reference_measure", lambda *a, **k: pytest.fail("rank 1 ran"))
    monkeypatch.setattr(bench, "reference_simulation_measure",
                        lambda *a, **k: pytest.fail("rank 1 ran"))
    assert bench.main(["--impl", "reference", "--gpus", "2"]) == 0
    assert capsys.readouterr().out == ""


def test_reference_arm_line(monkeypatch, capsys):
    monkeypatch.setenv("RANK", "0")
    fake = {"value": 80.0, "unit": "MPA/s", "cores": 16, "kind": "reference", "cpu_model": "x",
            "ms_per_step": 400.0, "steps": 20, "particles_total": 61046784,
            "sampled": 61046784, "sample": "s"}
    monkeypatch.setattr(bench, "cpu_reference_measure", lambda *a, **k: dict(fake))
    monkeypatch.setattr(bench, "reference_simulation_measure",
                        lambda *a, **k: {"value": 60.0, "unit": "MPA/s", "workers": 16})
    assert bench.main(["--impl", "reference", "--gpus", "8"]) == 0
    line = json.loads(capsys.readouterr().out)
    assert line["impl"] == "reference" and line["n_gpus"] == 8 and line["value"] == 80.0
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["config"]["same_config"] is True  # the whole C2 state was moved
    assert line["reference_simulation"]["workers"] == 16
    assert line["e2e"] == {"value": 80.0, "unit": "MPA/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_one_rank_world_path_on_request(monkeypatch):
    """B2M_BENCH_WORLD=1 under a one-rank torchrun runs the N > 1 code path
    (the slab world over a one-rank NCCL communicator); without it, N = 1 is
    the plain single-GPU path."""
    called = {}
    monkeypatch.setenv("WORLD_SIZE", "1")
    monkeypatch.setattr(bench, "run_world", lambda a: (called.__setitem__("path", "world"), 0)[1])
    monkeypatch.setattr(bench, "run_ours", lambda a: (called.__setitem__("path", "ours"), 0)[1])
    monkeypatch.delenv("B2M_BENCH_WORLD", raising=False)
    assert bench.main([]) == 0 and called["path"] == "ours"
    monkeypatch.setenv("B2M_BENCH_WORLD", "1")
    assert bench.main([]) == 0 and called["path"] == "world"
