"""bench.py's launch path (VERDICT r1 "Next round" 1): `--gpus N` without WORLD_SIZE spawns N
ranks itself (torch.distributed.run on 127.0.0.1), and a process group whose size is not --gpus
is refused. CPU only: the launch check runs the same spawn with a gloo all-gather."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _env(**kw):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(kw)
    return env


@pytest.mark.parametrize("n", [1, 2, 3])
def test_spawn_n_ranks(n):
    r = subprocess.run([sys.executable, BENCH, "--gpus", str(n), "--launch-check"], env=_env(),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout          # rank 0 alone prints
    out = json.loads(lines[0])
    assert out["n_gpus"] == n and out["ranks"] == list(range(n)) and out["pids"] == n


def test_world_mismatch_refused():
    # a process group of 1 rank (WORLD_SIZE set: no spawn) with --gpus 2 must not run
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--launch-check"],
                       env=_env(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"),
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
    assert "--gpus 2 but the process group has 1" in (r.stderr + r.stdout)


def test_spawn_cmd_shape():
    sys.path.insert(0, ROOT)
    import bench
    cmd = bench.spawn_cmd(8, ["--gpus", "8", "--config", "c5"], port=29511)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--config", "c5"]


def test_bench_without_gpu_fails_loudly():
    # the real arm on a box without enough CUDA devices exits non-zero (never a CPU fallback)
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--config", "c1", "--steps", "1"],
                       env=_env(), capture_output=True, text=True, timeout=300)
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this box has 2 GPUs: tests/test_gpu_bench.py runs the real thing")
    assert r.returncode != 0
    assert "CUDA device" in (r.stderr + r.stdout)
