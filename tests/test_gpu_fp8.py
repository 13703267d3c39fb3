"""GPU parity of the FP8 variant (SURVEY §8 f4 ii): parse_verify_attn_fp8
(e4m3 Q/K/V, P rounded to e4m3, tcgen05 kind::f8f6f4) through the C ABI vs
the fp64 oracle evaluated on the dequantized inputs (x8 * descale), i.e. the
exact masked attention of the values the kernel receives.

Tolerance (derived, tests/oracle_pool.fp8_bound): the only rounding beyond
fp32 accumulation is P -> e4m3 (relative 2^-4 per normal probability,
2^-10 absolute in the subnormal range, the normaliser l summed from the
unrounded values) and O -> bf16, so EVERY element is checked against its own
bound (2^-4 + 5e-4) sum_j pi_j |v_j| + 2^-14/Z sum_{subnormal j} |v_j| +
2^-8 |O| + 1e-5 max|V| computed in fp64 from the same inputs (round 1 used
the row-independent 2^-4 max|V|, ~0.3, a few times looser than needed)."""

import numpy as np
import pytest
import torch

import oracle
import paper_2605_04263_b200 as pb
import workloads
from tests.oracle_pool import fp8_bound

pytestmark = pytest.mark.gpu

# (name, B, Hq, Hkv, N, K, S, boundaries-kind, data)
CASES = [
    ("mha", 2, 2, 2, 256, 4, 16, "uniform", "base"),
    ("gqa4_packed", 1, 8, 2, 384, 6, 32, "uniform", "base"),      # head-packed suffix tiles
    ("gqa16_packed", 1, 16, 1, 256, 4, 32, "uniform", "base"),
    ("delta40_ragged", 2, 4, 1, 300, 8, 16, "delta40", "base"),   # P:573, N not a tile multiple
    ("random_b", 2, 4, 4, 200, 7, 12, "random", "base"),          # b_k = 0 and b_k = N
    ("k1_full", 1, 4, 1, 190, 1, 32, "full", "base"),             # K=1, b=N
    ("peaky", 1, 8, 2, 640, 8, 32, "uniform", "peaky"),           # attention sink, online-max rescales
]


def _boundaries(kind, N, K, seed):
    if kind == "uniform":
        return workloads.uniform_boundaries(N, K)
    if kind == "delta40":
        b = workloads.delta_boundaries(min(N, 40 * K), 40)
        return np.concatenate([b, np.full(K - len(b), b[-1], np.int32)])[:K]
    if kind == "full":
        return np.array([N] * K, np.int32)
    b = workloads.random_boundaries(N, K, seed)
    b[0], b[-1] = 0, N
    return np.sort(b)


def _run(B, Hq, Hkv, N, K, S, bnd, seed, data, tree=None):
    cfg = workloads.Config(f"fp8_{seed}", 950 + seed, B, Hq, Hkv, 128, N, K, S)
    q, k, v = workloads.make_qkv(cfg, device="cpu", data=data)
    (q8, sq), (k8, sk), (v8, sv) = workloads.to_e4m3(q), workloads.to_e4m3(k), workloads.to_e4m3(v)
    o, lse = pb.parse_verify_attn_fp8(q8.cuda(), k8.cuda(), v8.cuda(), sq, sk, sv, bnd, K, S,
                                      tree_parent=tree, want_lse=True)
    torch.cuda.synchronize()
    deq = lambda x8, s: x8.double() * s  # noqa: E731  (the values the kernel is given)
    qd, kd, vd = deq(q8, sq), deq(k8, sk), deq(v8, sv)
    O, LSE = oracle.verify_attn(qd, kd, vd, N, K, S, bnd, tree_parent=tree)
    err = np.abs(o.double().cpu().numpy() - O)
    bound = fp8_bound(qd, kd, vd, N, K, S, bnd, O, tree=tree)      # per element
    lerr = float(np.abs(lse.double().cpu().numpy() - LSE).max())
    return err, bound, lerr


@pytest.mark.parametrize("case_def", CASES, ids=[c[0] for c in CASES])
def test_fp8_parity(case_def):
    name, B, Hq, Hkv, N, K, S, kind, data = case_def
    bnd = _boundaries(kind, N, K, seed=len(name))
    err, bound, lerr = _run(B, Hq, Hkv, N, K, S, bnd, len(name), data)
    ratio = float((err / bound).max())
    print(f"{name}: max|dO| {err.max():.3e} max(|dO|/bound) {ratio:.3f} mean {err.mean():.2e} max|dLSE| {lerr:.2e}")
    assert ratio <= 1.0, f"{name}: an element exceeds its derived e4m3 bound ({ratio})"
    assert err.mean() <= 1e-2, f"{name}: mean |dO| {err.mean()}"
    assert lerr <= 2e-3, f"{name}: max |dLSE| {lerr}"


def test_fp8_tree_suffix():
    S = 64
    tree = workloads.make_tree_parent(S, seed=11)
    bnd = workloads.uniform_boundaries(256, 4)
    err, bound, lerr = _run(1, 8, 2, 256, 4, S, bnd, 31, "base", tree=tree)
    assert (err <= bound).all() and err.mean() <= 1e-2 and lerr <= 2e-3


def test_fp8_rejects_head_dim_64_and_wrong_entry():
    q8 = torch.zeros((1, 160, 1, 64), dtype=torch.float8_e4m3fn, device="cuda")
    with pytest.raises(pb.ParseError) as e:
        pb.parse_verify_attn_fp8(q8, q8, q8, 1.0, 1.0, 1.0, [32, 64, 96, 128], 4, 8)
    assert e.value.status == pb.PARSE_ERR_UNSUPPORTED


# ragged / paged batches through parse_verify_attn_varlen_fp8 (e4m3 page pool)
VARLEN_CASES = [
    ("ragged_packed", [300, 77, 129, 260], [None, 1, 0, None], 8, 2, 32, 40, 0, 5),
    ("paged16", [300, 77, 129, 260], [None, 1, 0, None], 8, 2, 32, 40, 16, 0),
    ("paged128_gqa16", [384, 130, 70], [None, 1, None], 16, 1, 32, 64, 128, 0),
]


@pytest.mark.parametrize("case", VARLEN_CASES, ids=[c[0] for c in VARLEN_CASES])
def test_fp8_varlen_parity(case):
    name, Ns, Ks, Hq, Hkv, S, delta, page, gap = case
    rb = workloads.make_ragged_batch(Ns, Hq, Hkv, 128, S, delta, Ks=Ks, gap=gap, page_size=page, seed=len(name))
    (q8, sq), (k8, sk), (v8, sv) = workloads.to_e4m3(rb.q), workloads.to_e4m3(rb.k), workloads.to_e4m3(rb.v)
    bt = rb.block_table.cuda() if rb.block_table is not None else None
    o, lse = pb.parse_verify_attn_varlen_fp8(q8.cuda(), k8.cuda(), v8.cuda(), sq, sk, sv, rb.Ns, rb.Ks,
                                             rb.boundaries, S, row_offsets=rb.row_offsets, block_table=bt,
                                             page_size=page, want_lse=True)
    torch.cuda.synchronize()
    o, lse = o.double().cpu().numpy(), lse.double().cpu().numpy()
    # the same per-tensor e4m3 encoding of every request's rows (elementwise, same descales)
    deq = lambda x, s: (x.float() / s).clamp(-448, 448).to(torch.float8_e4m3fn).double() * s  # noqa: E731
    ratio = err = lerr = 0.0
    for b in range(len(rb.Ns)):
        L, r0 = rb.Ns[b] + rb.Ks[b] * S, rb.row_offsets[b]
        qd, kd, vd = deq(rb.q_list[b], sq)[None], deq(rb.k_list[b], sk)[None], deq(rb.v_list[b], sv)[None]
        O, LSE = oracle.verify_attn(qd, kd, vd, rb.Ns[b], rb.Ks[b], S, rb.boundaries[b])
        e = np.abs(o[r0:r0 + L] - O[0])
        if rb.Ks[b] > 0:
            bound = fp8_bound(qd, kd, vd, rb.Ns[b], rb.Ks[b], S, rb.boundaries[b], O)[0]
        else:   # K = 0: a causal prefill, same bound with no suffix rows (one dummy boundary-free copy)
            bound = (2.0 ** -4 + 5e-4) * float(vd.abs().max()) + 2.0 ** -8 * np.abs(O[0]) + 1e-5
        ratio = max(ratio, float((e / bound).max()))
        err = max(err, float(e.max()))
        lerr = max(lerr, float(np.abs(lse[:, r0:r0 + L] - LSE[0]).max()))
    print(f"{name}: max|dO| {err:.3e} max(|dO|/bound) {ratio:.3f} max|dLSE| {lerr:.2e}")
    assert ratio <= 1.0 and lerr <= 2e-3
