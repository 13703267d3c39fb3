"""Model-level equivalence (north-star invariant 1 lifted to a
whole decoder; "packed == K independent passes within 1e-5"):
the judgment-row logits of one packed verification pass, with suffix copy k
rotated at positions b_k .. b_k+S-1, equal the logits of K standalone passes
on draft[0:b_k] ++ suffix.

CPU (not gpu): the packed pass uses the oracle's masked attention (fp64).
GPU: the packed pass runs every attention layer through libparse (fp32-debug
and bf16 paths) and is compared with standalone fp64 SDPA passes."""

import numpy as np
import pytest
import torch

import oracle
from tests.tiny_decoder import TinyDecoder, packed_inputs, sdpa_causal_bf16_inputs, standalone_judgment_logits


def _case(seed, B=2, N=37, S=5, delta=10, P=0):
    g = torch.Generator().manual_seed(seed)
    draft = torch.randint(0, 64, (B, N), generator=g)
    suffix = torch.randint(0, 64, (B, S), generator=g)
    bnd = oracle.place_boundaries(N - P, delta, prompt_len=P)
    return draft, suffix, bnd


@pytest.mark.parametrize("seed,N,S,delta,P", [(0, 37, 5, 10, 0), (1, 64, 8, 16, 7), (2, 20, 3, 40, 0)])
def test_packed_equals_standalone_oracle_fp64(seed, N, S, delta, P):
    model = TinyDecoder(seed=seed)
    draft, suffix, bnd = _case(seed, N=N, S=S, delta=delta, P=P)
    K = len(bnd)
    toks, pos = packed_inputs(draft, suffix, bnd)

    def attend(q, k, v):
        O, _ = oracle.verify_attn(q, k, v, N, K, S, bnd)
        return torch.from_numpy(O)
    logits = model.forward(toks, pos, attend)
    jp = oracle.judgment_positions(N, K, S)
    packed = logits[:, jp]
    want = standalone_judgment_logits(model, draft, suffix, bnd)
    np.testing.assert_allclose(packed.numpy(), want.numpy(), rtol=0, atol=1e-10)


def test_wrong_positions_break_equivalence():
    """Negative control for reading R3: natural (packed-order) position ids
    for the suffix copies do NOT reproduce the standalone passes."""
    model = TinyDecoder(seed=5)
    draft, suffix, bnd = _case(5, N=40, S=4, delta=10)
    K, N, S = len(bnd), 40, 4
    toks, _ = packed_inputs(draft, suffix, bnd)
    pos = torch.arange(toks.shape[1]).expand(toks.shape[0], -1)

    def attend(q, k, v):
        return torch.from_numpy(oracle.verify_attn(q, k, v, N, K, S, bnd)[0])
    got = model.forward(toks, pos, attend)[:, oracle.judgment_positions(N, K, S)]
    want = standalone_judgment_logits(model, draft, suffix, bnd)
    assert np.abs(got.numpy() - want.numpy()).max() > 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("precision,tol", [(1, 1e-4), (0, 5e-2)], ids=["fp32dbg", "bf16"])
def test_packed_equals_standalone_libparse(precision, tol):
    import paper_2605_04263_b200 as pb
    model = TinyDecoder(seed=9, n_q=4, n_kv=2, head_dim=64, d_model=256)
    N, S = 300, 8
    draft, suffix, bnd = _case(9, B=2, N=N, S=S, delta=40)
    K = len(bnd)
    toks, pos = packed_inputs(draft, suffix, bnd)

    def attend(q, k, v):
        o, _ = pb.parse_verify_attn(q.to(torch.bfloat16).cuda().contiguous(), k.to(torch.bfloat16).cuda().contiguous(),
                                    v.to(torch.bfloat16).cuda().contiguous(), bnd, K, S, precision=precision)
        torch.cuda.synchronize()
        return o.double().cpu()
    packed = model.forward(toks, pos, attend)[:, oracle.judgment_positions(N, K, S)]
    # standalone passes see the same bf16-rounded q/k/v as libparse
    want = standalone_judgment_logits(model, draft, suffix, bnd, attend=sdpa_causal_bf16_inputs)
    err = (packed - want).abs().max().item()
    scale = want.abs().max().item()
    print(f"precision={precision}: max |d logits| = {err:.3e} (max |logit| {scale:.2f})")
    # fp32-debug: fp32 arithmetic only, but two layers: the second layer's q/k/v
    # are rounded to bf16 from values that differ in their last fp32 bits between
    # the two sides, and a flipped bf16 rounding moves a logit by ~1e-5; the 1e-5
    # contract is checked on one-layer models by the 100-case test below.
    # bf16 path: P and O rounded to bf16 in every layer.
    assert err <= tol * max(1.0, scale)


def _random_case(i):
    """Randomised geometry of case i (>= 100 random cases)."""
    rng = np.random.default_rng(1000 + i)
    n_q, n_kv = [(2, 1), (4, 2), (4, 4), (8, 2), (2, 2)][i % 5]
    hd = 64 if i % 3 else 128
    N = int(rng.integers(8, 121))
    S = int(rng.integers(1, 17))
    delta = int(rng.integers(4, 65))
    P = int(rng.integers(0, N // 4 + 1))
    B = 1 + i % 2
    return dict(seed=i, n_q=n_q, n_kv=n_kv, hd=hd, N=N, S=S, delta=delta, P=P, B=B)


def test_packed_equals_standalone_oracle_fp64_random_100():
    """100 randomised tiny decoders / geometries (2 layers): the packed pass
    through the oracle equals K standalone passes to 1e-10 (fp64)."""
    worst = 0.0
    for i in range(100):
        c = _random_case(i)
        model = TinyDecoder(seed=c["seed"], n_q=c["n_q"], n_kv=c["n_kv"], head_dim=c["hd"], d_model=64, vocab=64)
        draft, suffix, bnd = _case(c["seed"], B=c["B"], N=c["N"], S=c["S"], delta=c["delta"], P=c["P"])
        K, N, S = len(bnd), c["N"], c["S"]
        toks, pos = packed_inputs(draft, suffix, bnd)

        def attend(q, k, v):
            return torch.from_numpy(oracle.verify_attn(q, k, v, N, K, S, bnd)[0])
        packed = model.forward(toks, pos, attend)[:, oracle.judgment_positions(N, K, S)]
        want = standalone_judgment_logits(model, draft, suffix, bnd)
        err = (packed - want).abs().max().item()
        worst = max(worst, err)
        assert err <= 1e-10, (i, c, err)
    print(f"100 random cases: max |d logits| = {worst:.2e}")


@pytest.mark.gpu
def test_packed_equals_standalone_libparse_random_100():
    """S:157 on the GPU path: 100 randomised one-layer tiny decoders, the
    packed pass's attention through libparse, vs K standalone fp64 passes on
    the same bf16-rounded q/k/v.  fp32-debug: every judgment-row logit within
    1e-5 (absolute).  One layer, because with two the second layer's q/k/v
    are rounded to bf16 from values that differ in the last fp32 bits between
    the two sides, and a flipped bf16 rounding (2^-9 relative) is not an error
    of the pass.  bf16 path: P and O rounded to bf16, checked at 2e-2 of the
    logit scale."""
    import paper_2605_04263_b200 as pb
    worst = {1: 0.0, 0: 0.0}
    for i in range(100):
        c = _random_case(i)
        model = TinyDecoder(seed=c["seed"], n_q=c["n_q"], n_kv=c["n_kv"], head_dim=c["hd"], d_model=64, vocab=64,
                            n_layers=1)
        draft, suffix, bnd = _case(c["seed"], B=c["B"], N=c["N"], S=c["S"], delta=c["delta"], P=c["P"])
        K, N, S = len(bnd), c["N"], c["S"]
        toks, pos = packed_inputs(draft, suffix, bnd)
        want = standalone_judgment_logits(model, draft, suffix, bnd, attend=sdpa_causal_bf16_inputs)
        scale = max(1.0, want.abs().max().item())
        for precision in (1, 0):
            def attend(q, k, v):
                o, _ = pb.parse_verify_attn(q.to(torch.bfloat16).cuda().contiguous(),
                                            k.to(torch.bfloat16).cuda().contiguous(),
                                            v.to(torch.bfloat16).cuda().contiguous(), bnd, K, S, precision=precision)
                torch.cuda.synchronize()
                return o.double().cpu()
            packed = model.forward(toks, pos, attend)[:, oracle.judgment_positions(N, K, S)]
            err = (packed - want).abs().max().item()
            worst[precision] = max(worst[precision], err / (1.0 if precision == 1 else scale))
            if precision == 1:
                assert err <= 1e-5, (i, c, err)
            else:
                assert err <= 2e-2 * scale, (i, c, err, scale)
    print(f"100 random cases: fp32-debug max |d logits| = {worst[1]:.2e}; bf16 max |d logits| / scale = {worst[0]:.2e}")
