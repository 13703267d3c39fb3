"""GPU parity: parse_verify_attn (through the C ABI) vs the fp64 oracle on the
same seeded bf16 inputs.  Tolerances from north_star: bf16 <= 2e-2, fp32
debug <= 1e-5 (max abs error over every compared element)."""

import numpy as np
import pytest
import torch

import oracle
import paper_2605_04263_b200 as pb
import workloads
from tests.gpu_helpers import (BF16_TOL, FP32_TOL, compare_dense, compare_rows, make_case, oracle_dense, run_gpu,
                               sample_rows)

pytestmark = pytest.mark.gpu

LSE_TOL_BF16 = 2e-3
LSE_TOL_FP32 = 1e-4

# (name, B, Hq, Hkv, d, N, K, S, boundaries-kind)
SMALL_CASES = [
    ("tiny", 1, 1, 1, 64, 128, 4, 8, "uniform"),            # BASELINE config 0
    ("mha_d128", 2, 2, 2, 128, 256, 4, 16, "uniform"),
    ("gqa4_packed", 1, 8, 2, 128, 384, 6, 32, "uniform"),   # head-packed suffix tiles
    ("gqa16_packed", 1, 16, 1, 128, 256, 4, 32, "uniform"),
    ("delta40", 2, 4, 1, 128, 300, 8, 16, "delta40"),       # P:573 Delta=40, unaligned
    ("prompt_offset", 1, 4, 2, 64, 200, 5, 8, "prompt"),    # shared prompt + draft (R4)
    ("random_b", 2, 4, 4, 128, 200, 7, 12, "random"),       # b_k = 0 and b_k = N included
    ("ragged_N", 1, 2, 1, 64, 77, 3, 5, "random"),          # N not a tile multiple, S odd
    ("k1_full", 1, 4, 1, 128, 190, 1, 32, "full"),          # K=1, b=N (causal prefill)
]


def _boundaries(kind, N, K, seed):
    if kind == "uniform":
        return workloads.uniform_boundaries(N, K)
    if kind == "delta40":
        b = workloads.delta_boundaries(min(N, 40 * K), 40)
        return np.concatenate([b, np.full(K - len(b), b[-1], np.int32)])[:K]
    if kind == "prompt":
        P = N - 40 * (K - 1) - 17
        return workloads.delta_boundaries(N - P, 40, prompt_len=P)[:K]
    if kind == "full":
        return np.array([N] * K, np.int32)
    b = workloads.random_boundaries(N, K, seed)
    b[0], b[-1] = 0, N
    return np.sort(b)


@pytest.mark.parametrize("case_def", SMALL_CASES, ids=[c[0] for c in SMALL_CASES])
@pytest.mark.parametrize("precision", [pb.PARSE_PREC_BF16, pb.PARSE_PREC_FP32_DEBUG], ids=["bf16", "fp32dbg"])
def test_small_dense(case_def, precision):
    name, B, Hq, Hkv, d, N, K, S, kind = case_def
    bnd = _boundaries(kind, N, K, seed=len(name))
    assert len(bnd) == K
    case = make_case(B, Hq, Hkv, d, N, K, S, bnd, seed=len(name))
    o, lse = run_gpu(case, precision)
    err, lerr = compare_dense(case, o, lse, None)
    tol = BF16_TOL if precision == pb.PARSE_PREC_BF16 else FP32_TOL
    ltol = LSE_TOL_BF16 if precision == pb.PARSE_PREC_BF16 else LSE_TOL_FP32
    print(f"{name} prec={precision}: max|dO|={err:.3e} max|dLSE|={lerr:.3e}")
    assert err <= tol
    assert lerr <= ltol


@pytest.mark.parametrize("precision", [pb.PARSE_PREC_BF16, pb.PARSE_PREC_FP32_DEBUG], ids=["bf16", "fp32dbg"])
def test_tree_mask(precision):
    S = 64
    parent = workloads.make_tree_parent(S, seed=5)
    case = make_case(1, 8, 2, 128, 256, 4, S, workloads.uniform_boundaries(256, 4), seed=11,
                     tree_parent=parent)
    o, lse = run_gpu(case, precision)
    err, lerr = compare_dense(case, o, lse, None)
    tol = BF16_TOL if precision == pb.PARSE_PREC_BF16 else FP32_TOL
    print(f"tree prec={precision}: {err:.3e} {lerr:.3e}")
    assert err <= tol


def test_peaky_data_rescale_paths():
    """Attention-sink keys + larger logits stress the online max / lazy rescale."""
    case = make_case(1, 8, 2, 128, 512, 8, 32, workloads.uniform_boundaries(512, 8), seed=21, data="peaky")
    for prec, tol in ((pb.PARSE_PREC_BF16, BF16_TOL), (pb.PARSE_PREC_FP32_DEBUG, FP32_TOL)):
        o, lse = run_gpu(case, prec)
        err, _ = compare_dense(case, o, lse, None)
        print(f"peaky prec={prec}: {err:.3e}")
        assert err <= tol


def test_negative_control_off_by_one_boundary():
    """A boundary shifted by one token must fail parity (the test can see
    mask bugs)."""
    N, K, S = 256, 4, 16
    bnd = workloads.uniform_boundaries(N, K)
    case = make_case(1, 2, 1, 128, N, K, S, bnd, seed=31)
    bad = dict(case)
    bad["boundaries"] = bnd - 1
    o, _ = run_gpu(bad, pb.PARSE_PREC_FP32_DEBUG)
    err, _ = compare_dense(case, o, None, None)
    assert err > 1e-3


def test_bf16_matches_fp32_debug_on_qwen3_8b_sample():
    """Config 1 shape at full size; oracle on sampled rows (incl. judgment rows)."""
    cfg = workloads.CONFIGS["qwen3_8b"]
    bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
    q, k, v = workloads.make_qkv(cfg, device="cuda")
    case = dict(cfg=cfg, qd=q, kd=k, vd=v, boundaries=bnd, tree=None)
    o, lse = run_gpu(case, pb.PARSE_PREC_BF16)
    jp = [(b, t, h) for b in (0, cfg.B - 1) for t in oracle.judgment_positions(cfg.N, cfg.K, cfg.S)[::5]
          for h in (0, cfg.Hq - 1)]
    rows = sample_rows(case, 200, seed=1, include=jp + [(0, 0, 0), (1, cfg.N - 1, 5), (2, cfg.N, 7)])
    err, lerr = compare_rows(case, o, lse, rows, BF16_TOL)
    print(f"qwen3_8b sampled: {err:.3e} {lerr:.3e}")
    assert err <= BF16_TOL and lerr <= LSE_TOL_BF16


def test_error_paths_gpu():
    case = make_case(1, 2, 1, 128, 64, 2, 8, [32, 64], seed=41)
    with pytest.raises(pb.ParseError) as ei:
        pb.parse_verify_attn(case["qd"], case["kd"], case["vd"], [32, 65], 2, 8)
    assert ei.value.status == pb.PARSE_ERR_INVALID
    q96 = torch.zeros((1, 80, 2, 96), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(pb.ParseError) as ei:
        pb.parse_verify_attn(q96, q96[:, :, :1], q96[:, :, :1], [32, 64], 2, 8)
    assert ei.value.status == pb.PARSE_ERR_UNSUPPORTED


def test_output_16byte_aligned_fallback():
    """O at a 16- but not 32-byte aligned address takes the 128-bit store path
    (the 256-bit epilogue stores need 32-byte alignment); same results."""
    bnd = workloads.uniform_boundaries(256, 4)
    case = make_case(1, 4, 1, 128, 256, 4, 16, bnd, seed=77)
    c = case["cfg"]
    q = case["qd"]
    raw = torch.empty(q.numel() + 8, dtype=torch.bfloat16, device="cuda")
    out = raw[8:].view(q.shape)
    assert out.data_ptr() % 32 == 16
    o, _ = pb.parse_verify_attn(q, case["kd"], case["vd"], bnd, c.K, c.S, out=out)
    torch.cuda.synchronize()
    O, _ = oracle_dense(case)
    err = float(np.abs(o.float().cpu().numpy() - O).max())
    assert err <= BF16_TOL, err
