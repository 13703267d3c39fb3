"""The experimental 2-SM (cta_group::2) attention kernel.  It is
not part of libparse.so: it is built here as the variant libparse_2sm.so
(-DPARSE_WITH_2SM), and the bf16 head_dim-128 parity cases of
test_gpu_attn.py / test_gpu_varlen.py / test_gpu_shards.py run through it in a
subprocess (PARSE_LIB selects the variant), against the same fp64 oracle and
tolerance."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANT = os.path.join(ROOT, "paper_2605_04263_b200", "libparse_2sm.so")


@pytest.fixture(scope="module")
def variant_env():
    from paper_2605_04263_b200 import build
    build.build(out=VARIANT, defines=["PARSE_WITH_2SM=1"])
    return dict(os.environ, PARSE_LIB=VARIANT)


def test_2sm_kernel_parity(variant_env):
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_attn.py", "-q", "-x", "-p", "no:cacheprovider",
                        "-k", "bf16 and (mha_d128 or gqa4 or gqa16 or delta40 or random_b or k1_full)"],
                       cwd=ROOT, env=variant_env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "6 passed" in r.stdout


def test_2sm_kernel_varlen_and_sharded_views(variant_env):
    """Packed-row (ragged) batches and head-group shard views through the 2-SM kernel."""
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_varlen.py", "tests/test_gpu_shards.py", "-q",
                        "-x", "-p", "no:cacheprovider", "-k",
                        "(bf16 and (ragged_packed or ragged_gqa16)) or shards"],
                       cwd=ROOT, env=variant_env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "5 passed" in r.stdout
