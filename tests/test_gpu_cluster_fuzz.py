"""Seeded random problems through the 2-CTA cluster launch (DESIGN §6.1,
K/V multicast), every output element against the fp64 oracle.

The cluster kernel pairs work items into units (multicast pairs with the same
K/V walk, lockstep pairs with the same step count, ghosts recomputed without
storing); its protocol state (CTA 0 -> CTA 1 unit mailbox, K/V stages
released by both CTAs, the item ring) wraps many times on these launches.
Shapes, boundaries (duplicates, 0, N, unsorted), suffix lengths (dividing
128 or not), token trees and batch sizes are drawn from a fixed seed; each
case prints its unit mix.  Tolerances: north_star (bf16 2e-2, fp32-debug
1e-5 via the SIMT path is covered elsewhere)."""

import numpy as np
import pytest
import torch

import paper_2605_04263_b200 as pb
import workloads
from tests.gpu_helpers import BF16_TOL
from tests.oracle_pool import verify_attn_parallel

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    Hkv = int(rng.choice([1, 2, 4]))
    r = int(rng.choice([1, 2, 3, 4, 8, 16]))
    Hq = Hkv * r
    B = int(rng.integers(1, 4))
    N = int(rng.integers(40, 1400))
    K = int(rng.integers(1, 24))
    S = int(rng.choice([8, 12, 16, 24, 32, 64]))
    tree = None
    if S <= 64 and rng.random() < 0.25:
        tree = workloads.make_tree_parent(S, seed=seed)
    kind = rng.integers(0, 3)
    if kind == 0:
        bnd = np.sort(rng.integers(0, N + 1, K)).astype(np.int32)          # duplicates, may hit 0 / N
    elif kind == 1:
        bnd = np.stack([np.sort(rng.integers(0, N + 1, K)) for _ in range(B)]).astype(np.int32)
    else:
        bnd = rng.permutation(rng.integers(0, N + 1, K)).astype(np.int32)   # unsorted (attention accepts it)
    return B, Hq, Hkv, N, K, S, bnd, tree


@pytest.mark.parametrize("seed", list(range(24)))
def test_cluster_launch_random_problem_all_elements(seed):
    B, Hq, Hkv, N, K, S, bnd, tree = _case(seed)
    cfg = workloads.Config(f"fuzz{seed}", 800 + seed, B, Hq, Hkv, 128, N, K, S, tree is not None)
    q, k, v = workloads.make_qkv(cfg, device="cuda")
    units = pb.parse_verify_attn_units(q, k, v, bnd, K, S, tree_parent=tree)
    n_mc = sum(1 for _, y in units if y >= 0)
    n_ls = sum(1 for _, y in units if y <= -2)
    o, lse = pb.parse_verify_attn(q, k, v, bnd, K, S, tree_parent=tree, want_lse=True)
    torch.cuda.synchronize()
    O, LSE = verify_attn_parallel(q, k, v, N, K, S, bnd, tree_parent=tree)
    err = float(np.abs(o.double().cpu().numpy() - O).max())
    lerr = float(np.abs(lse.double().cpu().numpy() - LSE).max())
    print(f"[fuzz {seed}] B={B} Hq={Hq} Hkv={Hkv} N={N} K={K} S={S} tree={tree is not None} "
          f"units mc/lockstep/ghost {n_mc}/{n_ls}/{len(units) - n_mc - n_ls}: max|dO|={err:.3e} max|dLSE|={lerr:.3e}")
    assert err <= BF16_TOL
    assert lerr <= 2e-3


@pytest.mark.parametrize("seed", [0, 2, 7, 13, 17, 18])
def test_cluster_launch_random_problem_fp8(seed):
    """The FP8 (e4m3) variant through the cluster launch on the same random
    problems (multicast, lockstep and ghost mixes), every element within its
    derived e4m3 bound (tests/oracle_pool.fp8_bound)."""
    from tests.oracle_pool import fp8_bound
    B, Hq, Hkv, N, K, S, bnd, tree = _case(seed)
    cfg = workloads.Config(f"fuzz{seed}", 800 + seed, B, Hq, Hkv, 128, N, K, S, tree is not None)
    q, k, v = workloads.make_qkv(cfg, device="cuda")
    (q8, sq), (k8, sk), (v8, sv) = workloads.to_e4m3(q), workloads.to_e4m3(k), workloads.to_e4m3(v)
    o, lse = pb.parse_verify_attn_fp8(q8, k8, v8, sq, sk, sv, bnd, K, S, tree_parent=tree, want_lse=True)
    torch.cuda.synchronize()
    qd, kd, vd = q8.double() * sq, k8.double() * sk, v8.double() * sv
    O, LSE = verify_attn_parallel(qd, kd, vd, N, K, S, bnd, tree_parent=tree)
    bound = fp8_bound(qd, kd, vd, N, K, S, bnd, O, tree=tree)
    ratio = float((np.abs(o.double().cpu().numpy() - O) / bound).max())
    lerr = float(np.abs(lse.double().cpu().numpy() - LSE).max())
    print(f"[fuzz fp8 {seed}] max(|dO|/bound)={ratio:.3f} max|dLSE|={lerr:.2e}")
    assert ratio <= 1.0
    assert lerr <= 2e-3


@pytest.mark.parametrize("seed", list(range(8)))
def test_cluster_launch_random_ragged_paged(seed):
    """Ragged batches (per-request N_b, K_b) with K/V in a page pool or in
    packed rows through the cluster launch (the tile owner multicasts every
    page box), every request's rows against the fp64 oracle."""
    from tests.test_gpu_varlen import _compare, _run
    rng = np.random.default_rng(2000 + seed)
    Hkv = int(rng.choice([1, 2, 4]))
    Hq = Hkv * int(rng.choice([1, 2, 4, 8, 16]))
    S = int(rng.choice([8, 16, 32, 64]))
    nreq = int(rng.integers(1, 5))
    Ns = [int(n) for n in rng.integers(20, 700, nreq)]
    Ks = [None if rng.random() < 0.6 else int(rng.integers(0, 3)) for _ in range(nreq)]
    page = int(rng.choice([0, 16, 32, 64, 128]))
    tree = workloads.make_tree_parent(S, seed=seed).tolist() if rng.random() < 0.25 else None
    rb = workloads.make_ragged_batch(Ns, Hq, Hkv, 128, S, int(rng.choice([40, 64, 128])), Ks=Ks,
                                     gap=int(rng.integers(0, 6)) if page == 0 else 0, page_size=page, seed=seed)
    o, lse = _run(rb, pb.PARSE_PREC_BF16, tree)
    err, lerr, stray = _compare(rb, o, lse, tree)
    print(f"[fuzz varlen {seed}] Ns={Ns} Ks={Ks} Hq={Hq} Hkv={Hkv} S={S} page={page} tree={tree is not None}: "
          f"max|dO|={err:.3e} max|dLSE|={lerr:.3e}")
    assert err <= BF16_TOL
    assert lerr <= 2e-3
    assert stray == 0.0
