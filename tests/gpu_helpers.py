"""Shared helpers for the GPU parity tests (inputs from ``workloads``,
expected values from ``oracle`` only)."""

from __future__ import annotations

import numpy as np
import torch

import oracle
import paper_2605_04263_b200 as pb
import workloads

BF16_TOL = 2e-2   # north_star: max abs error <= 2e-2 in bf16
FP32_TOL = 1e-5   # north_star: <= 1e-5 for the fp32-accumulate debug mode


def make_case(B, Hq, Hkv, d, N, K, S, boundaries, seed=0, data="base", tree_parent=None, device="cuda"):
    cfg = workloads.Config(f"case{seed}", 900 + seed, B, Hq, Hkv, d, N, K, S)
    q, k, v = workloads.make_qkv(cfg, device="cpu", data=data)
    return dict(cfg=cfg, q=q, k=k, v=v, qd=q.to(device), kd=k.to(device), vd=v.to(device),
                boundaries=np.asarray(boundaries, dtype=np.int32), tree=tree_parent)


def run_gpu(case, precision=pb.PARSE_PREC_BF16, want_lse=True):
    c = case["cfg"]
    o, lse = pb.parse_verify_attn(case["qd"], case["kd"], case["vd"], case["boundaries"], c.K, c.S,
                                  tree_parent=case["tree"], precision=precision, want_lse=want_lse)
    torch.cuda.synchronize()
    return o, lse


def oracle_dense(case, batches=None, heads=None):
    c = case["cfg"]
    return oracle.verify_attn(case["q"], case["k"], case["v"], c.N, c.K, c.S, case["boundaries"],
                              tree_parent=case["tree"], batches=batches, heads=heads)


def compare_dense(case, o, lse, tol, batches=None, heads=None):
    c = case["cfg"]
    O, LSE = oracle_dense(case, batches, heads)
    bs = list(range(c.B)) if batches is None else list(batches)
    hs = list(range(c.Hq)) if heads is None else list(heads)
    got = o.float().cpu().numpy()[np.ix_(bs, range(c.L), hs, range(c.d))]
    err = np.abs(got - O).max()
    lerr = 0.0
    if lse is not None:
        gl = lse.cpu().numpy()[np.ix_(bs, hs, range(c.L))]
        lerr = np.abs(gl - LSE).max()
    return float(err), float(lerr)


def sample_rows(case, n, seed=0, include=()):
    c = case["cfg"]
    rng = np.random.default_rng(seed)
    rows = [(int(rng.integers(0, c.B)), int(rng.integers(0, c.L)), int(rng.integers(0, c.Hq))) for _ in range(n)]
    return list(include) + rows


def compare_rows(case, o, lse, rows, tol):
    c = case["cfg"]
    O, LSE = oracle.verify_attn_rows(case["qd"], case["kd"], case["vd"], c.N, c.K, c.S, case["boundaries"],
                                     rows, tree_parent=case["tree"])
    oc = o.float()
    got = np.stack([oc[b, t, h].cpu().numpy() for (b, t, h) in rows])
    err = float(np.abs(got - O).max())
    lerr = 0.0
    if lse is not None:
        gl = np.array([float(lse[b, h, t]) for (b, t, h) in rows])
        lerr = float(np.abs(gl - LSE).max())
    return err, lerr
