"""The experimental 2-SM (cta_group::2) attention kernel (PARSE_2SM=1, see
DESIGN §6.1): the bf16 head_dim-128 parity cases of test_gpu_attn.py run
through it in a subprocess (the switch is read once per process), against
the same fp64 oracle and tolerance."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_2sm_kernel_parity():
    env = dict(os.environ, PARSE_2SM="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_attn.py", "-q", "-x", "-p", "no:cacheprovider",
                        "-k", "bf16 and (mha_d128 or gqa4 or gqa16 or delta40 or random_b or k1_full)"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "6 passed" in r.stdout


def test_2sm_kernel_varlen_and_sharded_views():
    """Packed-row (ragged) batches and head-group shard views through the 2-SM kernel."""
    env = dict(os.environ, PARSE_2SM="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_varlen.py", "tests/test_gpu_shards.py", "-q",
                        "-x", "-p", "no:cacheprovider", "-k",
                        "(bf16 and (ragged_packed or ragged_gqa16)) or shards"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "5 passed" in r.stdout
