"""GPU parity of the FP8 variant (SURVEY §8 f4 ii): parse_verify_attn_fp8
(e4m3 Q/K/V, P rounded to e4m3, tcgen05 kind::f8f6f4) through the C ABI vs
the fp64 oracle evaluated on the dequantized inputs (x8 * descale), i.e. the
exact masked attention of the values the kernel receives.

Tolerance (derived, include/parse.h): the only rounding beyond fp32
accumulation is P -> e4m3 (relative 2^-4 per probability, the normaliser l
is summed from the unrounded values) and O -> bf16 (2^-8 relative), so per
row |dO| <= 2^-4 * max_j |V_j| + 2^-8 |O| (+ fp32 noise).  The errors of
independent probabilities have random signs, so the mean over all elements
is far smaller; it is checked against 1e-2 (= 2^-4/sqrt(3) * max|V| /
sqrt(n) for rows of n >= ~100 keys, the bulk of every case here)."""

import numpy as np
import pytest
import torch

import oracle
import paper_2605_04263_b200 as pb
import workloads

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
    vq = deq(v8, sv)
    O, LSE = oracle.verify_attn(deq(q8, sq), deq(k8, sk), vq, N, K, S, bnd, tree_parent=tree)
    err = np.abs(o.double().cpu().numpy() - O)
    bound = 2.0 ** -4 * float(vq.abs().max()) + 2.0 ** -8 * float(np.abs(O).max()) + 1e-3
    lerr = float(np.abs(lse.double().cpu().numpy() - LSE).max())
    return err, bound, lerr


@pytest.mark.parametrize("case_def", CASES, ids=[c[0] for c in CASES])
def test_fp8_parity(case_def):
    name, B, Hq, Hkv, N, K, S, kind, data = case_def
    bnd = _boundaries(kind, N, K, seed=len(name))
    err, bound, lerr = _run(B, Hq, Hkv, N, K, S, bnd, len(name), data)
    print(f"{name}: max|dO| {err.max():.3e} (bound {bound:.3e}) mean {err.mean():.2e} max|dLSE| {lerr:.2e}")
    assert err.max() <= bound, f"{name}: max |dO| {err.max()} > {bound}"
    assert err.mean() <= 1e-2, f"{name}: mean |dO| {err.mean()}"
    assert lerr <= 2e-3, f"{name}: max |dLSE| {lerr}"


def test_fp8_tree_suffix():
    S = 64
    tree = workloads.make_tree_parent(S, seed=11)
    bnd = workloads.uniform_boundaries(256, 4)
    err, bound, lerr = _run(1, 8, 2, 256, 4, S, bnd, 31, "base", tree=tree)
    assert err.max() <= bound and err.mean() <= 1e-2 and lerr <= 2e-3


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
    err = lerr = 0.0
    vmax = float(v8.double().abs().max()) * sv
    for b in range(len(rb.Ns)):
        L, r0 = rb.Ns[b] + rb.Ks[b] * S, rb.row_offsets[b]
        O, LSE = oracle.verify_attn(deq(rb.q_list[b], sq)[None], deq(rb.k_list[b], sk)[None],
                                    deq(rb.v_list[b], sv)[None], rb.Ns[b], rb.Ks[b], S, rb.boundaries[b])
        err = max(err, float(np.abs(o[r0:r0 + L] - O[0]).max()))
        lerr = max(lerr, float(np.abs(lse[:, r0:r0 + L] - LSE[0]).max()))
    bound = (2.0 ** -4 + 2.0 ** -8) * vmax + 1e-3
    print(f"{name}: max|dO| {err:.3e} (bound {bound:.3e}) max|dLSE| {lerr:.2e}")
    assert err <= bound and lerr <= 2e-3
