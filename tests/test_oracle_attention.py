"""Pins for oracle.attention: brute-force per-suffix causal attention (P:208's
"exactly the input it would have seen" claim), library SDPA special cases,
closed forms and mask soundness (CPU only)."""

import math

import numpy as np
import pytest
import torch

import oracle


def _brute_causal(q, k, v, scale, allowed=None):
    """Textbook attention with a pure-Python triple loop; allowed(i, j) -> bool
    (default causal j <= i)."""
    n = len(q)
    out = []
    for i in range(n):
        js = [j for j in range(n) if (allowed(i, j) if allowed else j <= i)]
        s = [scale * sum(q[i][c] * k[j][c] for c in range(len(q[i]))) for j in js]
        m = max(s)
        w = [math.exp(x - m) for x in s]
        z = sum(w)
        out.append([sum(w[a] * v[j][c] for a, j in enumerate(js)) / z for c in range(len(v[0]))])
    return np.array(out)


def _instance(rng, N, K, S, d, Hq=1, Hkv=1, B=1, b=None):
    L = N + K * S
    q = rng.standard_normal((B, L, Hq, d))
    k = rng.standard_normal((B, L, Hkv, d))
    v = rng.standard_normal((B, L, Hkv, d))
    if b is None:
        b = np.sort(rng.integers(0, N + 1, size=K))
    return q, k, v, [int(x) for x in b]


def test_suffix_rows_equal_standalone_prefix_plus_suffix():
    """North-star invariant 1 / S:157: suffix k's rows equal ordinary causal
    attention run separately on draft[0:b_k] ++ suffix_k (brute force)."""
    rng = np.random.default_rng(0)
    for trial in range(60):
        N = int(rng.integers(1, 24))
        K = int(rng.integers(1, 5))
        S = int(rng.integers(1, 5))
        d = int(rng.integers(1, 5))
        q, k, v, b = _instance(rng, N, K, S, d)
        b[0] = 0 if trial % 5 == 0 else b[0]                 # cover b_k = 0
        b[-1] = N if trial % 3 == 0 else b[-1]               # and b_k = N
        scale = 1 / math.sqrt(d)
        O, _ = oracle.verify_attn(q, k, v, N, K, S, b)
        for kk in range(K):
            rows = list(range(b[kk])) + list(range(N + kk * S, N + (kk + 1) * S))
            want = _brute_causal(q[0, rows, 0].tolist(), k[0, rows, 0].tolist(),
                                 v[0, rows, 0].tolist(), scale)
            np.testing.assert_allclose(O[0, N + kk * S: N + (kk + 1) * S, 0], want[b[kk]:],
                                       rtol=0, atol=1e-12)


def test_draft_rows_equal_causal_prefill_sdpa():
    """Draft purity: draft rows equal causal attention over the draft
    alone, whatever K, S, b are (torch SDPA in fp64 as the library routine)."""
    rng = np.random.default_rng(1)
    for _ in range(10):
        N, K, S, d = int(rng.integers(2, 60)), int(rng.integers(1, 6)), int(rng.integers(1, 6)), 8
        q, k, v, b = _instance(rng, N, K, S, d, Hq=2, Hkv=2)
        O, _ = oracle.verify_attn(q, k, v, N, K, S, b)
        tq = torch.from_numpy(q[0, :N]).permute(1, 0, 2)
        tk = torch.from_numpy(k[0, :N]).permute(1, 0, 2)
        tv = torch.from_numpy(v[0, :N]).permute(1, 0, 2)
        ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=True)
        np.testing.assert_allclose(O[0, :N], ref.permute(1, 0, 2).numpy(), rtol=0, atol=1e-12)


def test_k1_full_boundary_is_causal_prefill():
    """North-star invariant 2: K=1, b=N reduces to standard causal prefill of
    length N+S (SDPA is_causal, fp64)."""
    rng = np.random.default_rng(2)
    for N, S, d in [(5, 3, 4), (33, 7, 16), (100, 32, 64)]:
        q, k, v, _ = _instance(rng, N, 1, S, d, Hq=4, Hkv=2)
        O, LSE = oracle.verify_attn(q, k, v, N, 1, S, [N])
        tq = torch.from_numpy(q[0]).permute(1, 0, 2)
        tk = torch.from_numpy(k[0]).permute(1, 0, 2).repeat_interleave(2, dim=0)
        tv = torch.from_numpy(v[0]).permute(1, 0, 2).repeat_interleave(2, dim=0)
        ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=True)
        np.testing.assert_allclose(O[0], ref.permute(1, 0, 2).numpy(), rtol=0, atol=1e-12)
        # LSE: log-sum-exp of the causal scores, via torch.logsumexp
        s = (tq @ tk.transpose(1, 2)) / math.sqrt(d)
        s = s.masked_fill(torch.ones_like(s, dtype=torch.bool).triu(1), -math.inf)
        np.testing.assert_allclose(LSE[0], torch.logsumexp(s, -1).numpy(), rtol=0, atol=1e-12)


def test_k0_is_causal_prefill():
    """Reading R18: K = 0 (no suffix copies) is plain causal attention over
    the shared region (SDPA is_causal, fp64)."""
    rng = np.random.default_rng(4)
    for N, d in [(1, 4), (37, 8)]:
        q, k, v, _ = _instance(rng, N, 1, 1, d, Hq=2, Hkv=1)
        q, k, v = q[:, :N], k[:, :N], v[:, :N]
        O, _ = oracle.verify_attn(q, k, v, N, 0, 3, [])
        tq = torch.from_numpy(q[0]).permute(1, 0, 2)
        tk = torch.from_numpy(k[0]).permute(1, 0, 2).repeat_interleave(2, dim=0)
        tv = torch.from_numpy(v[0]).permute(1, 0, 2).repeat_interleave(2, dim=0)
        ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=True)
        np.testing.assert_allclose(O[0], ref.permute(1, 0, 2).numpy(), rtol=0, atol=1e-12)


def test_gqa_head_mapping():
    """q head h reads kv head h // (Hq/Hkv): compare with explicitly expanded
    K/V run as MHA."""
    rng = np.random.default_rng(3)
    N, K, S, d, Hq, Hkv = 20, 3, 4, 8, 6, 2
    q, k, v, b = _instance(rng, N, K, S, d, Hq=Hq, Hkv=Hkv)
    O, L1 = oracle.verify_attn(q, k, v, N, K, S, b)
    O2, L2 = oracle.verify_attn(q, np.repeat(k, 3, axis=2), np.repeat(v, 3, axis=2), N, K, S, b)
    assert np.array_equal(O, O2) and np.array_equal(L1, L2)


def test_mask_soundness_bitwise():
    """Perturbing K/V rows a query cannot see leaves its output bitwise equal
    (S:152): other suffix copies, and draft keys >= b_k."""
    rng = np.random.default_rng(4)
    N, K, S, d = 30, 4, 5, 8
    q, k, v, b = _instance(rng, N, K, S, d, b=[0, 9, 17, 30])
    O, _ = oracle.verify_attn(q, k, v, N, K, S, b)
    for j in range(K):                                   # perturb copy j
        lo, hi = N + j * S, N + (j + 1) * S
        k2, v2 = k.copy(), v.copy()
        k2[:, lo:hi] += 3.0
        v2[:, lo:hi] -= 5.0
        O2, _ = oracle.verify_attn(q, k2, v2, N, K, S, b)
        keep = np.ones(N + K * S, bool)
        keep[lo:hi] = False
        assert np.array_equal(O[:, keep], O2[:, keep])
        assert not np.array_equal(O[:, lo:hi], O2[:, lo:hi])
    kk = 1                                               # perturb draft >= b_1
    k2, v2 = k.copy(), v.copy()
    k2[:, b[kk]:N] *= -2.0
    v2[:, b[kk]:N] += 1.0
    O2, _ = oracle.verify_attn(q, k2, v2, N, K, S, b)
    lo, hi = N + kk * S, N + (kk + 1) * S
    assert np.array_equal(O[:, lo:hi], O2[:, lo:hi])
    assert np.array_equal(O[:, :b[kk]], O2[:, :b[kk]])


def test_uniform_v_closed_form():
    """V rows all equal c => every output row equals c (weights sum to 1)."""
    rng = np.random.default_rng(5)
    N, K, S, d = 25, 3, 4, 6
    q, k, v, b = _instance(rng, N, K, S, d)
    c = rng.standard_normal(d)
    v[:] = c
    O, _ = oracle.verify_attn(q, k, v, N, K, S, b)
    np.testing.assert_allclose(O[0, :, 0], np.broadcast_to(c, O[0, :, 0].shape), rtol=0, atol=1e-14)


def test_singleton_row_closed_form():
    """b_k = 0 => suffix row s=0 sees only itself: output == V exactly, LSE ==
    its own score."""
    rng = np.random.default_rng(6)
    N, K, S, d = 12, 3, 4, 8
    q, k, v, _ = _instance(rng, N, K, S, d, b=[0, 0, 5])
    O, LSE = oracle.verify_attn(q, k, v, N, K, S, [0, 0, 5])
    for kk in (0, 1):
        i = N + kk * S
        assert np.array_equal(O[0, i, 0], v[0, i, 0])
        assert LSE[0, 0, i] == pytest.approx(float(q[0, i, 0] @ k[0, i, 0]) / math.sqrt(d), abs=1e-12)
    assert np.array_equal(O[0, 0, 0], v[0, 0, 0])          # first draft row too


def test_tree_suffix_equals_standalone_tree_attention():
    """Tree variant (R11): suffix k's rows equal standalone attention over
    draft[0:b_k] ++ suffix_k where token s sees the prefix and its ancestors."""
    rng = np.random.default_rng(7)
    parent = [-1, 0, 0, 1, 2, 2, 4, -1]
    anc = oracle.ancestor_sets(parent)
    N, K, S, d = 14, 3, len(parent), 4
    q, k, v, b = _instance(rng, N, K, S, d, b=[0, 6, 14])
    O, _ = oracle.verify_attn(q, k, v, N, K, S, b, tree_parent=parent)
    for kk in range(K):
        rows = list(range(b[kk])) + list(range(N + kk * S, N + (kk + 1) * S))
        P = b[kk]

        def allowed(i, j, P=P):
            if j < P:
                return j <= i
            return i >= P and (j - P) in anc[i - P]
        want = _brute_causal(q[0, rows, 0].tolist(), k[0, rows, 0].tolist(),
                             v[0, rows, 0].tolist(), 1 / math.sqrt(d), allowed)
        np.testing.assert_allclose(O[0, N + kk * S: N + (kk + 1) * S, 0], want[P:], rtol=0, atol=1e-12)


def test_rows_api_matches_dense():
    rng = np.random.default_rng(8)
    N, K, S, d, Hq, Hkv, B = 40, 4, 6, 16, 4, 2, 2
    q, k, v, _ = _instance(rng, N, K, S, d, Hq=Hq, Hkv=Hkv, B=B)
    bnd = np.array([[0, 10, 30, 40], [5, 5, 20, 33]])
    O, LSE = oracle.verify_attn(q, k, v, N, K, S, bnd)
    rows = [(int(rng.integers(0, B)), int(rng.integers(0, N + K * S)), int(rng.integers(0, Hq)))
            for _ in range(50)]
    o, l = oracle.verify_attn_rows(q, k, v, N, K, S, bnd, rows)
    for n, (b, t, h) in enumerate(rows):
        np.testing.assert_allclose(o[n], O[b, t, h], rtol=0, atol=1e-13)
        assert l[n] == pytest.approx(LSE[b, h, t], abs=1e-13)


def test_bf16_inputs_are_upcast_exactly():
    """The oracle consumes the same bf16 tensors as the GPU, upcast exactly."""
    rng = np.random.default_rng(9)
    q, k, v, b = _instance(rng, 10, 2, 3, 8)
    tq, tk, tv = (torch.from_numpy(x).to(torch.bfloat16) for x in (q, k, v))
    O1, _ = oracle.verify_attn(tq, tk, tv, 10, 2, 3, b)
    O2, _ = oracle.verify_attn(tq.double().numpy(), tk.double().numpy(), tv.double().numpy(), 10, 2, 3, b)
    assert np.array_equal(O1, O2)
