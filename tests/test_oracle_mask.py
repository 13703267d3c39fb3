"""Pins for oracle.mask against the paper's worked layout, invariants and an
independent construction of App. A.3's interleaved layout (CPU only)."""

import itertools

import numpy as np
import pytest

import oracle
from oracle.mask import visible_row


def test_place_boundaries_worked(golden):
    for ex in golden["place_boundaries"]:
        assert oracle.place_boundaries(ex["T"], ex["delta"]) == ex["expect"], ex["cite"]


def test_place_boundaries_chunk_definition():
    # App. A.1: C_k = y_{(k-1)D+1 .. min(kD, T)}, K = ceil(T/D).
    # Rebuild the chunks token by token and read their right edges.
    for T in range(1, 60):
        for D in range(1, 20):
            chunks = {}
            for t in range(1, T + 1):                      # 1-indexed tokens
                chunks.setdefault((t - 1) // D + 1, []).append(t)
            edges = [max(c) for _, c in sorted(chunks.items())]
            assert oracle.place_boundaries(T, D) == edges
            assert oracle.place_boundaries(T, D, prompt_len=7) == [7 + e for e in edges]


def test_packed_layout_worked(golden):
    for ex in golden["packed_layout"]:
        K = len(ex["boundaries"])
        assert oracle.packed_length(ex["T"], K, ex["S"]) == ex["length"], ex["cite"]
        assert oracle.judgment_positions(ex["T"], K, ex["S"]) == ex["judgment_positions"]


def test_mask_visible_worked(golden):
    ex = golden["mask_visible"]
    M = oracle.visible_mask(ex["T"], len(ex["boundaries"]), ex["S"], ex["boundaries"])
    for q, k, want in ex["entries"]:
        assert bool(M[q, k]) == want, (q, k, ex["cite"])


def _random_instances(n, seed=0, maxN=40, maxK=5, maxS=5):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        N = int(rng.integers(1, maxN))
        K = int(rng.integers(1, maxK + 1))
        S = int(rng.integers(1, maxS + 1))
        b = np.sort(rng.integers(0, N + 1, size=K))
        yield N, K, S, [int(x) for x in b]


def test_mask_invariants():
    """block structure, cross-copy isolation, draft purity; and
    every visible key is at or before its query (subset of causal)."""
    for N, K, S, b in _random_instances(200):
        M = oracle.visible_mask(N, K, S, b)
        L = N + K * S
        assert M.shape == (L, L)
        assert not np.triu(M, 1).any()                      # subset of causal
        assert not M[:N, N:].any()                          # draft purity
        for i in range(N):
            assert M[i, : i + 1].all()                      # causal among draft
        spans = oracle.suffix_spans(N, K, S)
        for k, (lo, hi) in enumerate(spans):
            for j, (lo2, hi2) in enumerate(spans):
                if j != k:
                    assert not M[lo:hi, lo2:hi2].any()      # isolation
            jp = oracle.judgment_positions(N, K, S)[k]
            want = set(range(b[k])) | set(range(lo, hi))    # block structure
            assert set(np.nonzero(M[jp])[0]) == want


def test_chain_tree_equals_causal():
    for N, K, S, b in _random_instances(50, seed=1):
        chain = [-1] + list(range(S - 1))
        assert np.array_equal(oracle.visible_mask(N, K, S, b),
                              oracle.visible_mask(N, K, S, b, tree_parent=chain))


def test_tree_rows_see_exactly_ancestors():
    parent = [-1, 0, 0, 1, 1, 2, -1, 6]
    # hand-derived ancestor-or-self sets
    want = [{0}, {0, 1}, {0, 2}, {0, 1, 3}, {0, 1, 4}, {0, 2, 5}, {6}, {6, 7}]
    assert oracle.ancestor_sets(parent) == want
    N, K, S, b = 10, 2, 8, [3, 10]
    M = oracle.visible_mask(N, K, S, b, tree_parent=parent)
    for k in range(K):
        for s in range(S):
            i = N + k * S + s
            got = set(np.nonzero(M[i])[0])
            assert got == set(range(b[k])) | {N + k * S + a for a in want[s]}
    with pytest.raises(ValueError):
        oracle.ancestor_sets([-1, 2, 0])


def _interleaved_mask(P, T, delta, S):
    """App. A.3 layout built directly from its text:
    pi_P = prompt || (C_k || End)_{k=1..K}; the End slot of k attends "only to
    the question prefix plus its own prefix C_{1:k}" (+ itself causally);
    chunk tokens attend causally to the prompt and earlier chunk tokens.
    Returns (mask, kinds) with kinds[i] = ('d', draft_index) or ('s', k, s)."""
    K = -(-T // delta)
    kinds = [("d", i) for i in range(P)]
    for k in range(K):
        for t in range(k * delta, min((k + 1) * delta, T)):
            kinds.append(("d", P + t))
        for s in range(S):
            kinds.append(("s", k, s))
    L = len(kinds)
    M = np.zeros((L, L), dtype=bool)
    for i, a in enumerate(kinds):
        for j, c in enumerate(kinds[: i + 1]):
            if a[0] == "d":
                M[i, j] = c[0] == "d"
            else:
                k = a[1]
                if c[0] == "d":
                    M[i, j] = c[1] < P + min((k + 1) * delta, T)
                else:
                    M[i, j] = c[1] == k and c[2] <= a[2]
    return M, kinds


def test_interleaved_equals_appended_under_permutation():
    """Reading R1: the App. A.3 interleaved layout is a permutation of the
    §3.2 appended one with the same visibility."""
    for P, T, delta, S in itertools.product([0, 3], [1, 7, 12, 20], [4, 5, 40], [1, 3]):
        Mi, kinds = _interleaved_mask(P, T, delta, S)
        N = P + T
        b = oracle.place_boundaries(T, delta, prompt_len=P)
        K = len(b)
        Ma = oracle.visible_mask(N, K, S, b)
        perm = [c[1] if c[0] == "d" else N + c[1] * S + c[2] for c in kinds]
        assert sorted(perm) == list(range(N + K * S))
        assert np.array_equal(Mi, Ma[np.ix_(perm, perm)])


def test_visible_keys_matches_mask():
    for N, K, S, b in _random_instances(30, seed=3):
        M = oracle.visible_mask(N, K, S, b)
        for i in range(N + K * S):
            assert np.array_equal(oracle.visible_keys(i, N, K, S, b), np.nonzero(M[i])[0])


def test_suffix_positions():
    p = oracle.suffix_positions([2, 4], 3)
    assert p.tolist() == [[2, 3, 4], [4, 5, 6]]


def test_validation():
    with pytest.raises(ValueError):
        oracle.visible_mask(4, 2, 1, [2, 5])      # boundary > N
    with pytest.raises(ValueError):
        oracle.visible_mask(4, 2, 0, [2, 4])      # S = 0
    with pytest.raises(ValueError):
        oracle.place_boundaries(0, 40)
