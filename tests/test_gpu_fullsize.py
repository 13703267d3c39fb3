"""GPU parity at BASELINE.json's full sizes, in the launch configuration
bench.py times (one rank's batch for the 8-GPU configs), checked against the
fp64 oracle evaluated row by row on sampled outputs: judgment rows of every
suffix copy, rows next to each boundary, first/last rows, random rows.
bf16 path: max abs error <= 2e-2; fp32-debug path on one request: <= 1e-5."""

import numpy as np
import pytest
import torch

import oracle
import paper_2605_04263_b200 as pb
import workloads
from tests.gpu_helpers import BF16_TOL, FP32_TOL, compare_rows

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _rows(cfg, bnd, rng, n_random=160):
    rows = []
    jp = oracle.judgment_positions(cfg.N, cfg.K, cfg.S)
    B, Hq = cfg.B, cfg.Hq
    for k in sorted(set([0, 1, cfg.K // 2, cfg.K - 1])):
        b = int(rng.integers(0, B))
        rows.append((b, jp[k], int(rng.integers(0, Hq))))          # judgment row of copy k
        rows.append((b, cfg.N + k * cfg.S, int(rng.integers(0, Hq))))   # first row of copy k
        t = int(bnd[k]) - 1
        if t >= 0:
            rows.append((b, t, int(rng.integers(0, Hq))))          # last shared key of b_k
    rows += [(0, 0, 0), (B - 1, cfg.N - 1, Hq - 1), (B - 1, cfg.L - 1, Hq - 1)]
    rows += [(int(rng.integers(0, B)), int(rng.integers(0, cfg.L)), int(rng.integers(0, Hq))) for _ in range(n_random)]
    return rows


@pytest.mark.parametrize("name", ["qwen3_8b", "qwen3_235b", "long", "tree"])
def test_fullsize_bf16_sampled(name):
    cfg = workloads.CONFIGS[name]
    bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
    tree = workloads.make_tree_parent(cfg.S, seed=workloads.seed_for(cfg.config_id, 0, "tree")) if cfg.tree else None
    q, k, v = workloads.make_qkv(cfg, device="cuda")
    o, lse = pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S, tree_parent=tree, want_lse=True)
    torch.cuda.synchronize()
    case = dict(cfg=cfg, qd=q, kd=k, vd=v, boundaries=bnd, tree=tree)
    rows = _rows(cfg, bnd, np.random.default_rng(cfg.config_id))
    err, lerr = compare_rows(case, o, lse, rows, BF16_TOL)
    print(f"{name}: {len(rows)} rows, max|dO|={err:.3e} max|dLSE|={lerr:.3e}")
    assert err <= BF16_TOL and lerr <= 2e-3
    del o, lse, q, k, v
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["qwen3_235b", "tree"])
def test_fullsize_fp32_debug_one_request(name):
    cfg = workloads.CONFIGS[name]
    bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
    tree = workloads.make_tree_parent(cfg.S, seed=workloads.seed_for(cfg.config_id, 0, "tree")) if cfg.tree else None
    q, k, v = workloads.make_qkv(cfg, device="cuda", batch=1)
    o, lse = pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S, tree_parent=tree, want_lse=True,
                                  precision=pb.PARSE_PREC_FP32_DEBUG)
    torch.cuda.synchronize()
    one = workloads.Config(cfg.name, cfg.config_id, 1, cfg.Hq, cfg.Hkv, cfg.d, cfg.N, cfg.K, cfg.S, cfg.tree)
    case = dict(cfg=one, qd=q, kd=k, vd=v, boundaries=bnd, tree=tree)
    rows = _rows(one, bnd, np.random.default_rng(7), n_random=100)
    err, lerr = compare_rows(case, o, lse, rows, FP32_TOL)
    print(f"{name} fp32-debug: max|dO|={err:.3e} max|dLSE|={lerr:.3e}")
    assert err <= FP32_TOL and lerr <= 1e-4


def test_fullsize_select_with_bench_inputs():
    """The readout exactly as bench.py runs it (config 3, tau_P = 0.985)."""
    cfg = workloads.CONFIGS["qwen3_235b"]
    lg = workloads.make_verdict_logits(cfg.B, cfg.K, seed=0, device="cuda", config_id=cfg.config_id)
    bnd = torch.as_tensor(workloads.uniform_boundaries(cfg.N, cfg.K)).cuda()
    out = pb.parse_select_prefix(lg, bnd, 0.985, aux_threshold=0.90)
    torch.cuda.synchronize()
    want = oracle.select_prefix(lg.cpu().double().numpy(), bnd.cpu().numpy(), 0.985, aux_tau=0.90)
    assert np.array_equal(out["k_star"].cpu().numpy(), want["k_star"])
    assert np.array_equal(out["accepted_len"].cpu().numpy(), want["accepted_len"])


@pytest.mark.parametrize("name", ["qwen3_235b", "tree"])
def test_fullsize_fp8_sampled(name):
    """FP8 variant at the full per-request shape (2 requests), sampled rows vs
    the fp64 oracle on the dequantized inputs, within the derived e4m3 bound
    (tests/test_gpu_fp8.py)."""
    cfg = workloads.CONFIGS[name]
    bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
    tree = workloads.make_tree_parent(cfg.S, seed=workloads.seed_for(cfg.config_id, 0, "tree")) if cfg.tree else None
    q, k, v = workloads.make_qkv(cfg, device="cuda", batch=2)
    (q8, sq), (k8, sk), (v8, sv) = workloads.to_e4m3(q), workloads.to_e4m3(k), workloads.to_e4m3(v)
    del q, k, v
    o, lse = pb.parse_verify_attn_fp8(q8, k8, v8, sq, sk, sv, bnd, cfg.K, cfg.S, tree_parent=tree, want_lse=True)
    torch.cuda.synchronize()
    c2 = workloads.Config(cfg.name, cfg.config_id, 2, cfg.Hq, cfg.Hkv, cfg.d, cfg.N, cfg.K, cfg.S, cfg.tree)
    case = dict(cfg=c2, qd=q8.double() * sq, kd=k8.double() * sk, vd=v8.double() * sv, boundaries=bnd, tree=tree)
    rows = _rows(c2, bnd, np.random.default_rng(cfg.config_id + 5))
    vmax = float(case["vd"].abs().max())
    bound = (2.0 ** -4 + 2.0 ** -8) * vmax + 1e-3        # |O| <= max|V| (convex combination)
    err, lerr = compare_rows(case, o, lse, rows, bound)
    print(f"{name} fp8: {len(rows)} rows, max|dO|={err:.3e} (bound {bound:.3e}) max|dLSE|={lerr:.3e}")
    assert err <= bound and lerr <= 2e-3
