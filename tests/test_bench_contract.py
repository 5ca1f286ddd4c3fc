"""bench.py plumbing that runs without a GPU: the N-GPU self-launch, the shared config object of
both arms, and the algorithmic-byte model of the per-stage roofline."""

import json
import subprocess
import sys

import pytest

import bench


def _args(*extra):
    old = sys.argv
    sys.argv = ["bench.py", *extra]
    try:
        return bench.parse()
    finally:
        sys.argv = old


def test_gpus_n_self_launches_n_ranks(monkeypatch):
    calls = []

    def fake_run(cmd, *a, **k):
        calls.append(cmd)
        return subprocess.CompletedProcess(cmd, 0)

    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    assert bench.main() == 0
    (cmd,) = calls
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


def test_both_arms_report_the_same_config():
    a = _args("--config", "C3")
    assert bench.config_dict(a, 1) == bench.config_dict(a, a.gpus)
    assert bench.config_dict(a, 1)["workload"].startswith("C3:")


def test_reference_arm_line(monkeypatch, capsys):
    a = _args("--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.5")
    bench.run_reference(a)
    line = json.loads(capsys.readouterr().out.strip())
    assert line["impl"] == "reference" and line["config"] == bench.config_dict(a, 1)
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["value"] > 0 and line["unit"] == "paths/s"


def test_stage_byte_model():
    prof = {"ext_rays": 1000, "shadow_rays": 500, "paths": 400, "waves": 8, "pool_slots": 1024}
    work = {"ext_nodes_per_ray": 3.0, "ext_tris_per_ray": 2.0, "sh_nodes_per_ray": 4.0, "sh_tris_per_ray": 1.0,
            "lit_frac": 0.5}
    b, smem = bench.stage_bytes(prof, work, smem_bvh=True, nprev_bytes=0)
    assert b["trace_ext"] == 1000 * 84 and smem["trace_ext"] == (128 * 3 + 80 * 2) * 1000
    b2, smem2 = bench.stage_bytes(prof, work, smem_bvh=False, nprev_bytes=0)
    assert b2["trace_ext"] == 1000 * 84 + (128 * 3 + 80 * 2) * 1000 and not smem2["trace_ext"]
    assert b["shade"] == 1000 * 269 and b["trace_shadow"] == 500 * 68 + 250 * 80
    assert b["generate"] == 8 * 1024 + 400 * 84 + 400 * 121 + 1000 * 4
