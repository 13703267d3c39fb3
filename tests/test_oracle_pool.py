"""tests/oracle_pool.py distributes oracle.verify_attn over (request, head)
units; it must return exactly what the single-process oracle returns (same
function per unit, no arithmetic of its own), here with 3 worker processes."""

import numpy as np

import oracle
import workloads
from tests.oracle_pool import verify_attn_parallel


def test_pool_equals_oracle_bitwise():
    cfg = workloads.Config("pool", 801, 2, 4, 2, 64, 150, 5, 8)
    q, k, v = workloads.make_qkv(cfg)
    bnd = np.array([[0, 30, 60, 60, 150], [10, 20, 90, 140, 150]], np.int32)
    want_o, want_l = oracle.verify_attn(q, k, v, cfg.N, cfg.K, cfg.S, bnd)
    got_o, got_l = verify_attn_parallel(q, k, v, cfg.N, cfg.K, cfg.S, bnd, workers=3)
    assert np.array_equal(got_o, want_o) and np.array_equal(got_l, want_l)
    tree = workloads.make_tree_parent(8, seed=3)
    want_o, _ = oracle.verify_attn(q, k, v, cfg.N, cfg.K, cfg.S, bnd, tree_parent=tree, heads=[1, 3])
    got_o, _ = verify_attn_parallel(q, k, v, cfg.N, cfg.K, cfg.S, bnd, tree_parent=tree, heads=[1, 3], workers=2)
    assert np.array_equal(got_o, want_o)
