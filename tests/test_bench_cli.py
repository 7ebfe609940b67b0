"""bench.py's contract on the host side (CPU): the N-GPU launch logic, the
reference arm's JSON line, and the profiler guard of the live traffic
measurement."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_world_size_must_match_gpus(monkeypatch, capsys):
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "0")
    monkeypatch.setenv("LOCAL_RANK", "0")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "1"])
    assert bench.main() == 2
    assert "WORLD_SIZE=2" in capsys.readouterr().err


def test_gpus_without_launcher_spawns_torchrun(monkeypatch):
    """`python bench.py --gpus 8` re-runs the same command line as 8 ranks
    under torchrun on 127.0.0.1."""
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8", "--steps", "7", "--warmup", "4"])
    assert bench.main() == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "8", "--steps", "7", "--warmup", "4"]


def test_profiler_guard(monkeypatch):
    monkeypatch.delenv("CUDA_INJECTION64_PATH", raising=False)
    monkeypatch.setenv("LD_PRELOAD", "")
    assert not bench._under_profiler()
    monkeypatch.setenv("LD_PRELOAD", "/opt/nvidia/nsight-compute/x/libTreeLauncherTargetInjection.so")
    assert bench._under_profiler()
    t, src = bench.live_traffic("asum", "asum_k0")
    assert "profiler" in src


@pytest.mark.skipif(bench.ref_lib() is None, reason="oracle/_ref not built")
def test_reference_arm_line():
    """`--impl reference`: one JSON line, the reference's CPU path on the
    bench workload, with what it actually runs in config.strategy."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--workload", "dot", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert "dot.dpia" in line["config"]["strategy"]
    assert line["config"]["workload"] == bench.WORKLOADS["dot"][0]
