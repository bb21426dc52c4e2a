"""bench.py's N > 1 launcher on CPU: ``--gpus 2 --dry-run`` re-launches the
script under torch.distributed.run (2 ranks, gloo, 127.0.0.1), shards the
rows with split_workload, all-reduces once per step and prints ONE line from
rank 0 with n_gpus = 2 and dp2 parallelism (the GPU arm's plumbing, no
kernels)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


@pytest.mark.timeout(600)
def test_bench_launcher_world_2_dry_run():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run", "--steps", "3", "--warmup", "3"],
                         capture_output=True, text=True, env=env, timeout=500, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"].startswith("dp2")
    assert d["check"]["rows"] == d["config"]["batch"] == 16384
    assert abs(d["check"]["sum"] - d["check"]["expected_sum"]) < 1e-9
    assert d["steps"] == 3 and d["ms_per_step"] > 0
