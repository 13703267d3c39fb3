"""GPU parity of the f1 readout kernels (through the C ABI) vs oracle.readout,
and the end-to-end chain hidden states -> verdict logits -> selection."""

import numpy as np
import pytest
import torch

import oracle
from oracle import readout
from oracle import select as oracle_select
import paper_2605_04263_b200 as pb
import workloads

pytestmark = pytest.mark.gpu


def _head_inputs(B, K, H, seed, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    h = (torch.randn((B, K, H), generator=g) * scale).to(torch.bfloat16)
    gamma = (1.0 + 0.1 * torch.randn(H, generator=g)).to(torch.bfloat16)
    w = (torch.randn((2, H), generator=g) / H ** 0.5).to(torch.bfloat16)
    return h, gamma, w


@pytest.mark.parametrize("B,K,H", [(1, 1, 8), (3, 5, 64), (16, 64, 4096), (2, 7, 4104)])
def test_verdict_head(B, K, H):
    h, gamma, w = _head_inputs(B, K, H, seed=H)
    out = pb.parse_verdict_logits(h.cuda(), gamma.cuda(), w.cuda(), eps=1e-6)
    torch.cuda.synchronize()
    want = readout.verdict_logits(h, gamma, w, 1e-6)
    err = np.abs(out.cpu().numpy() - want)
    # fp32 accumulation over H products: |err| <= 1e-5 * (1 + |l|) is ~100x the fp32 bound
    assert (err <= 1e-5 * (1 + np.abs(want)) * max(1.0, H / 512)).all(), err.max()


def test_verdict_head_strided_judgment_rows():
    """Read the judgment rows in place from a [B, L, H] hidden-state tensor."""
    B, N, K, S, H = 2, 64, 4, 8, 256
    L = N + K * S
    hs, gamma, w = _head_inputs(B, L, H, seed=3)
    hsd = hs.cuda()
    jp = oracle.judgment_positions(N, K, S)
    view = hsd[:, jp[0]::S, :]                        # rows N+S-1, N+2S-1, ...
    assert view.shape == (B, K, H)
    out = pb.parse_verdict_logits(view, gamma.cuda(), w.cuda(), eps=1e-6)
    torch.cuda.synchronize()
    want = readout.verdict_logits(hs[:, jp], gamma, w, 1e-6)
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("B,K,V", [(1, 1, 8), (2, 3, 1000), (16, 64, 151936)])
def test_vocab_readout(dtype, B, K, V):
    g = torch.Generator().manual_seed(V)
    z = (torch.randn((B, K, V), generator=g) * 4).to(dtype)
    idc, idi = 3 % V, (V - 5) % V
    out = pb.parse_vocab_readout(z.cuda(), idc, idi)
    torch.cuda.synchronize()
    want = readout.vocab_readout(z, idc, idi)
    np.testing.assert_array_equal(out["pair_logits"].cpu().numpy(), want["pair_logits"].astype(np.float32))
    np.testing.assert_allclose(out["lse"].cpu().numpy(), want["lse"], rtol=2e-6, atol=2e-5)
    np.testing.assert_allclose(out["verdict_mass"].cpu().numpy(), want["verdict_mass"], rtol=5e-5, atol=1e-9)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_vocab_readout_masked_entries(dtype):
    """Constrained decoding masks vocabulary entries with -inf.  Rows whose
    first vectors (every thread's first 16-byte load) are all -inf must still
    give the finite LSE / verdict mass of the unmasked entries."""
    B, K, V = 2, 3, 151936
    g = torch.Generator().manual_seed(99)
    z = (torch.randn((B, K, V), generator=g) * 4).to(dtype)
    z[0, 0, :V // 2] = float("-inf")                   # first half masked
    z[0, 1, :] = float("-inf")
    z[0, 1, 5::97] = 1.5                              # sparse survivors
    z[1, 2, 8 * 256:] = float("-inf")                 # only each thread's first vector finite
    idc, idi = V - 3, V - 7
    z[0, 0, idc], z[0, 0, idi] = 2.0, -1.0
    z[0, 1, idc], z[0, 1, idi] = 0.5, 0.25
    out = pb.parse_vocab_readout(z.cuda(), idc, idi)
    torch.cuda.synchronize()
    want = readout.vocab_readout(z, idc, idi)
    assert np.isfinite(want["lse"]).all()
    np.testing.assert_allclose(out["lse"].cpu().numpy(), want["lse"], rtol=2e-6, atol=2e-5)
    np.testing.assert_allclose(out["verdict_mass"].cpu().numpy(), want["verdict_mass"], rtol=5e-5, atol=1e-9)


def test_hidden_to_selection_chain():
    """hidden states -> parse_verdict_logits -> parse_select_prefix equals the
    oracle's selection on the same (GPU-produced) logits, and the logits agree
    with the oracle's fp64 logits within the head tolerance."""
    cfg = workloads.CONFIGS["qwen3_235b"]
    h, gamma, w = _head_inputs(cfg.B, cfg.K, 4096, seed=11, scale=1.0)
    lg = pb.parse_verdict_logits(h.cuda(), gamma.cuda(), w.cuda(), eps=1e-6)
    bnd = torch.as_tensor(workloads.uniform_boundaries(cfg.N, cfg.K)).cuda()
    sel = pb.parse_select_prefix(lg, bnd, 0.6)
    torch.cuda.synchronize()
    want = oracle.select_prefix(lg.cpu().double().numpy(), bnd.cpu().numpy(), 0.6)
    assert np.array_equal(sel["k_star"].cpu().numpy(), want["k_star"])
    assert np.array_equal(sel["accepted_len"].cpu().numpy(), want["accepted_len"])
    np.testing.assert_allclose(lg.cpu().numpy(), readout.verdict_logits(h, gamma, w, 1e-6), rtol=1e-4, atol=1e-4)


def _stats_tuple(st):
    return st.cpu().numpy().copy()


@pytest.mark.parametrize("B,K,H,rule,thr", [
    (16, 64, 4096, pb.PARSE_RULE_LEADING_RUN, 0.6),     # config 3's judgment rows
    (3, 37, 512, pb.PARSE_RULE_MAX_CORRECT, 0.5),        # K not a multiple of 32, max rule
    (1, 1, 8, pb.PARSE_RULE_LEADING_RUN, 0.9),           # one row
    (5, 70, 1032, pb.PARSE_RULE_LEADING_RUN, 0.0),       # threshold 0, three ballot words
])
def test_verdict_select_fused_equals_two_calls(B, K, H, rule, thr):
    """parse_verdict_select (one launch) equals parse_verdict_logits +
    parse_select_prefix bit for bit (logits, k*, L*, scores, stats), and its
    selection equals the fp64 oracle's on those logits; two calls reuse the
    same per-request counters (left zero by every call)."""
    h, gamma, w = _head_inputs(B, K, H, seed=B * 1000 + K)
    h, gamma, w = h.cuda(), gamma.cuda(), w.cuda()
    rng = np.random.default_rng(K)
    bnd = torch.as_tensor(np.sort(rng.integers(0, 4 * K + 1, (B, K))).astype(np.int32)).cuda()
    counters = torch.zeros(B, dtype=torch.int32, device="cuda")
    lg = pb.parse_verdict_logits(h, gamma, w, eps=1e-6)
    ref = pb.parse_select_prefix(lg, bnd, thr, rule=rule, eta=1.0)
    for _ in range(2):
        fused = pb.parse_verdict_select(h, gamma, w, bnd, thr, eps=1e-6, rule=rule, eta=1.0, counters=counters)
        torch.cuda.synchronize()
        assert torch.equal(fused["logits"], lg)
        for key in ("k_star", "accepted_len", "scores", "stats", "status"):
            assert torch.equal(fused[key], ref[key]), key
        assert int(counters.abs().sum()) == 0
    want = oracle.select_prefix(lg.cpu().double().numpy(), bnd.cpu().numpy(), thr, eta=1.0,
                                rule=oracle_select.RULE_LEADING_RUN if rule == pb.PARSE_RULE_LEADING_RUN
                                else oracle_select.RULE_MAX_CORRECT)
    assert np.array_equal(fused["k_star"].cpu().numpy(), want["k_star"])
    assert np.array_equal(fused["accepted_len"].cpu().numpy(), want["accepted_len"])


def test_verdict_select_strided_judgment_rows():
    """The fused call reads the judgment rows in place from [B, L, H]."""
    B, N, K, S, H = 2, 64, 4, 8, 256
    hs, gamma, w = _head_inputs(B, N + K * S, H, seed=5)
    hsd = hs.cuda()
    jp = oracle.judgment_positions(N, K, S)
    view = hsd[:, jp[0]::S, :]
    bnd = torch.as_tensor(workloads.uniform_boundaries(N, K)).cuda()
    fused = pb.parse_verdict_select(view, gamma.cuda(), w.cuda(), bnd, 0.55)
    lg = pb.parse_verdict_logits(view, gamma.cuda(), w.cuda())
    ref = pb.parse_select_prefix(lg, bnd, 0.55)
    torch.cuda.synchronize()
    assert torch.equal(fused["logits"], lg)
    assert torch.equal(fused["k_star"], ref["k_star"]) and torch.equal(fused["accepted_len"], ref["accepted_len"])
