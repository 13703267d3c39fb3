"""bench.py's multi-GPU control path on CPU (gloo, no GPU, no compute):
`--gpus N` launches N ranks by itself (torch.distributed.run on 127.0.0.1),
the default is strong scaling of the config's batch (BASELINE config 3: 16
requests over 1/2/4/8 GPUs), every rank's selection reaches rank 0 through
the one all-gather, and a --gpus / WORLD_SIZE mismatch fails loudly."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=300):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    r = subprocess.run([sys.executable, "bench.py", *args, "--plumbing-check"], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=timeout)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return r, (json.loads(lines[-1]) if lines else None)


def test_self_launch_strong_default():
    r, line = _run(["--gpus", "2"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["global_batch"] == 16 and line["config"]["B_per_rank"] == 8
    assert line["gathered_requests"] == 16 and line["ranks_seen"] == [0, 1]


def test_self_launch_four_ranks_long_config():
    r, line = _run(["--gpus", "4", "--config", "long"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert line["config"]["global_batch"] == 64 and line["config"]["B_per_rank"] == 16
    assert line["ranks_seen"] == [0, 1, 2, 3]


def test_weak_scaling_option():
    r, line = _run(["--gpus", "2", "--per-rank-batch", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert line["scaling"] == "weak" and line["config"]["global_batch"] == 6


def test_gpus_world_size_mismatch_fails():
    r, line = _run(["--gpus", "4"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and line is None
    assert "WORLD_SIZE" in (r.stderr + r.stdout)
