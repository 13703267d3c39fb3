"""GPU parity for ragged and paged batches:
parse_verify_attn_varlen through the C ABI vs the fp64 oracle, request by
request, on the same seeded bf16 inputs (``workloads.make_ragged_batch``).
Tolerances as the dense path (north_star): bf16 <= 2e-2, fp32 debug <= 1e-5."""

import numpy as np
import pytest
import torch

import oracle
import paper_2605_04263_b200 as pb
import workloads
from tests.gpu_helpers import BF16_TOL, FP32_TOL

pytestmark = pytest.mark.gpu

LSE_TOL = {pb.PARSE_PREC_BF16: 2e-3, pb.PARSE_PREC_FP32_DEBUG: 1e-4}
TOL = {pb.PARSE_PREC_BF16: BF16_TOL, pb.PARSE_PREC_FP32_DEBUG: FP32_TOL}


def _run(rb, precision, tree=None, kv_row_offsets=None):
    dev = "cuda"
    bt = rb.block_table.to(dev) if rb.block_table is not None else None
    o, lse = pb.parse_verify_attn_varlen(rb.q.to(dev), rb.k.to(dev), rb.v.to(dev), rb.Ns, rb.Ks, rb.boundaries,
                                         rb.S, row_offsets=rb.row_offsets, kv_row_offsets=kv_row_offsets,
                                         block_table=bt, page_size=rb.page_size, tree_parent=tree,
                                         precision=precision, want_lse=True)
    torch.cuda.synchronize()
    return o.float().cpu().numpy(), lse.cpu().numpy()


def _compare(rb, o, lse, tree=None):
    """Max |dO| and |dLSE| over every request's rows, plus the max |O| on rows
    that belong to no request (must stay untouched = 0)."""
    err = lerr = 0.0
    owned = np.zeros(o.shape[0], bool)
    for b in range(len(rb.Ns)):
        L, r0 = rb.Ls[b], rb.row_offsets[b]
        O, LSE = oracle.verify_attn(rb.q_list[b][None], rb.k_list[b][None], rb.v_list[b][None], rb.Ns[b], rb.Ks[b],
                                    rb.S, rb.boundaries[b], tree_parent=tree)
        err = max(err, float(np.abs(o[r0:r0 + L] - O[0]).max()))
        lerr = max(lerr, float(np.abs(lse[:, r0:r0 + L] - LSE[0]).max()))
        owned[r0:r0 + L] = True
    stray = float(np.abs(o[~owned]).max()) if (~owned).any() else 0.0
    return err, lerr, stray


# (name, Ns, Ks, Hq, Hkv, d, S, delta, page_size, gap, tree)
CASES = [
    ("ragged_packed", [300, 77, 129, 260], [None, 1, 0, None], 8, 2, 128, 32, 40, 0, 5, False),
    ("ragged_tokmajor", [200, 33, 150], [None, 1, None], 4, 4, 64, 5, 40, 0, 0, False),
    ("ragged_gqa16", [384, 130], [None, 1], 16, 1, 128, 32, 64, 0, 3, False),
    ("paged16", [300, 77, 129, 260], [None, 1, 0, None], 8, 2, 128, 32, 40, 16, 0, False),
    ("paged64_tokmajor", [200, 33, 150], [None, 1, None], 4, 4, 64, 5, 40, 64, 2, False),
    ("paged128", [384, 130, 70], [None, 1, None], 16, 1, 128, 32, 64, 128, 0, False),
    ("paged256_tree", [256, 100], [None, None], 8, 2, 128, 64, 128, 256, 0, True),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("precision", [pb.PARSE_PREC_BF16, pb.PARSE_PREC_FP32_DEBUG], ids=["bf16", "fp32dbg"])
def test_varlen_parity(case, precision):
    name, Ns, Ks, Hq, Hkv, d, S, delta, page, gap, tree = case
    tp = workloads.make_tree_parent(S, seed=7).tolist() if tree else None
    rb = workloads.make_ragged_batch(Ns, Hq, Hkv, d, S, delta, Ks=Ks, gap=gap, page_size=page, seed=len(name))
    o, lse = _run(rb, precision, tp)
    err, lerr, stray = _compare(rb, o, lse, tp)
    print(f"{name}: max|dO| {err:.3e}  max|dLSE| {lerr:.3e}")
    assert err <= TOL[precision], err
    assert lerr <= LSE_TOL[precision], lerr
    assert stray == 0.0, "rows outside every request were written"


def test_varlen_uniform_equals_dense_bitwise():
    """Same requests through the dense and the varlen entry points: the
    schedule is identical, so O must match bit for bit."""
    Hq, Hkv, d, S, N = 8, 2, 128, 32, 512
    rb = workloads.make_ragged_batch([N, N, N], Hq, Hkv, d, S, 128)
    o_v, _ = _run(rb, pb.PARSE_PREC_BF16)
    q = torch.stack(rb.q_list).cuda()
    k = torch.stack(rb.k_list).cuda()
    v = torch.stack(rb.v_list).cuda()
    o_d, _ = pb.parse_verify_attn(q, k, v, np.stack(rb.boundaries), rb.Ks[0], S)
    torch.cuda.synchronize()
    o_d = o_d.float().cpu().numpy().reshape(-1, Hq, d)
    assert np.array_equal(o_v, o_d)


def test_paged_equals_contiguous():
    """Paged K/V (random page permutation, stale noise in unused pool rows)
    gives the contiguous result within bf16 rounding of a different
    self-tile alignment (both checked against the oracle above); here:
    page-size independence at a tight bound."""
    Ns, Ks = [500, 260, 90], [None, 1, None]
    outs = []
    for page in (16, 32, 128, 512):
        rb = workloads.make_ragged_batch(Ns, 8, 2, 128, 32, 40, Ks=Ks, page_size=page)
        outs.append(_run(rb, pb.PARSE_PREC_BF16)[0])
    for o in outs[1:]:
        # same 128-aligned KV tiles for every page size -> identical arithmetic
        assert np.array_equal(o, outs[0])


def test_varlen_full_verify_k1_is_causal_prefill():
    """K_b = 1, b = N_b (pi_F, P:180 / P:693) and K_b = 0 through varlen
    equal causal attention over the request's rows (oracle fp64)."""
    rb = workloads.make_ragged_batch([333, 129, 64], 4, 1, 128, 32, 40, Ks=[1, 1, 0], page_size=64)
    o, lse = _run(rb, pb.PARSE_PREC_BF16)
    err, lerr, _ = _compare(rb, o, lse)
    assert err <= BF16_TOL and lerr <= LSE_TOL[pb.PARSE_PREC_BF16]


def test_varlen_fullsize_qwen3_235b_ragged_paged():
    """A ragged Qwen3-235B-shaped batch at full size (16 requests, N_b from
    1024 to 8192, Delta = 128, S = 32, 64 q / 4 kv heads, paged K/V with
    64-token pages): sampled rows vs the oracle row by row."""
    cfg = workloads.CONFIGS["qwen3_235b"]
    rng = np.random.default_rng(11)
    Ns = sorted(int(x) for x in rng.integers(1024, cfg.N + 1, 16))
    Ns[-1] = cfg.N
    rb = workloads.make_ragged_batch(Ns, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, 128, page_size=64)
    o, lse = _run(rb, pb.PARSE_PREC_BF16)
    err = lerr = 0.0
    for b in range(len(Ns)):
        L, N, r0 = rb.Ls[b], rb.Ns[b], rb.row_offsets[b]
        rows = [(0, t, int(rng.integers(0, cfg.Hq))) for t in
                list(rng.integers(0, L, 6)) + [N - 1, N, L - 1]]      # incl. last draft row, first/last suffix row
        O, LSE = oracle.verify_attn_rows(rb.q_list[b][None], rb.k_list[b][None], rb.v_list[b][None], N, rb.Ks[b],
                                         rb.S, rb.boundaries[b], rows)
        got = np.stack([o[r0 + t, h] for (_, t, h) in rows])
        err = max(err, float(np.abs(got - O).max()))
        lerr = max(lerr, float(np.abs(np.array([lse[h, r0 + t] for (_, t, h) in rows]) - LSE).max()))
    print(f"ragged 235B paged: max|dO| {err:.3e} max|dLSE| {lerr:.3e}")
    assert err <= BF16_TOL and lerr <= LSE_TOL[pb.PARSE_PREC_BF16]
