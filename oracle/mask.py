"""Packed layout and prefix-boundary visibility (ORACLE — test infrastructure).

The paper's construction (§3.2 "Parallel Prefix Verification"):

    "We keep the draft tokens y_{1:T} as is and append n copies of the
     chat-template suffix, one per candidate boundary, into the same
     sequence. ... the draft tokens attend causally among themselves ...
     each suffix copy i attends causally to the draft tokens up through its
     assigned boundary y_{1:t_i} and to nothing else --- in particular,
     suffix copies do not see each other."

Readings taken here (DESIGN.md §3 lists all of them):
  * R1 appended layout rather than App. A.3's interleaved one
    (P:620-626); the two are a row/column permutation of each other
    (pinned in tests/test_oracle_mask.py).
  * R2 boundaries are 0-indexed half-open: suffix k sees draft keys
    [0, b_k), the same set as the paper's 1-indexed y_{1:t_k}.
  * R4 the question/system prompt is part of the shared region (P:630-632:
    each End slot sees "the question prefix plus its own prefix"), so the
    shared region length N = P + T and b_k = P + min((k+1)Delta, T).
  * R11 tree variant (not in the paper): within its own copy, suffix row s
    sees its ancestors-or-self instead of s' <= s.  parent[s] < s or -1.

Nothing here is shared with the CUDA path.
"""

from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np


def place_boundaries(T: int, delta: int, prompt_len: int = 0) -> list[int]:
    """Chunk boundaries t_k, k = 1..K (App. A.1).

    C_k = y_{(k-1)Delta+1 .. min(k Delta, T)}, K = ceil(T / Delta); the last
    chunk may be shorter, so t_K = T.  Boundaries are "uniformly every Delta
    tokens".  ``prompt_len`` shifts them into packed coordinates
    (reading R4).
    """
    if T < 1 or delta < 1 or prompt_len < 0:
        raise ValueError("need T >= 1, delta >= 1, prompt_len >= 0")
    K = math.ceil(T / delta)
    return [prompt_len + min(k * delta, T) for k in range(1, K + 1)]


def packed_length(N: int, K: int, S: int) -> int:
    """Total packed length "T + n*|suffix|" (§3.2), N = shared region."""
    return N + K * S


def suffix_spans(N: int, K: int, S: int) -> list[tuple[int, int]]:
    """Half-open packed-row span of each appended suffix copy."""
    return [(N + k * S, N + (k + 1) * S) for k in range(K)]


def judgment_positions(N: int, K: int, S: int) -> list[int]:
    """Classification position = last token of each suffix copy (P:208:
    "The classification position at the end of suffix i")."""
    return [hi - 1 for (_, hi) in suffix_spans(N, K, S)]


def suffix_positions(boundaries: Sequence[int], S: int) -> np.ndarray:
    """Position ids for suffix copy k: b_k, b_k+1, ..., b_k+S-1 (reading R3).

    P:208 requires the judgment position to see "exactly the input it would
    have seen had we run the single (y_{1:t_i}, suffix) pair on its own";
    with rotary embeddings that means the copy is positioned right after its
    boundary.  The attention op itself takes already-rotated Q/K.
    """
    b = np.asarray(boundaries, dtype=np.int64)
    return b[:, None] + np.arange(S, dtype=np.int64)[None, :]


def ancestor_sets(tree_parent: Sequence[int]) -> list[set[int]]:
    """Ancestor-or-self sets of a token tree given parent[s] (< s, or -1)."""
    S = len(tree_parent)
    out: list[set[int]] = []
    for s in range(S):
        p = int(tree_parent[s])
        if not (p == -1 or 0 <= p < s):
            raise ValueError(f"tree_parent[{s}]={p} must be -1 or in [0, {s})")
        anc = {s}
        if p >= 0:
            anc |= out[p]
        out.append(anc)
    return out


def _check(N: int, K: int, S: int, boundaries: Sequence[int]) -> None:
    # K = 0 (reading R18): no suffix copies, the packed sequence is the shared
    # region alone and the mask is plain causal.
    if N < 1 or K < 0 or S < 1:
        raise ValueError("need N, S >= 1 and K >= 0")
    if len(boundaries) != K:
        raise ValueError("need exactly K boundaries")
    for b in boundaries:
        if not (0 <= int(b) <= N):
            raise ValueError(f"boundary {b} outside [0, N={N}]")


def visible_row(i: int, N: int, K: int, S: int, boundaries: Sequence[int],
                tree_parent: Optional[Sequence[int]] = None,
                _anc: Optional[list[set[int]]] = None) -> np.ndarray:
    """Row i of the visibility relation, as a dense bool vector of length L.

    P:208: draft rows "attend causally among themselves"; suffix copy k
    "attends causally to the draft tokens up through its assigned boundary
    y_{1:t_k} and to nothing else" (plus, causally, itself); "suffix copies
    do not see each other".
    """
    L = packed_length(N, K, S)
    row = np.zeros(L, dtype=bool)
    if i < N:                                   # draft row: causal among the draft
        row[: i + 1] = True
        return row
    k, s = divmod(i - N, S)                     # suffix copy k, offset s
    base = N + k * S
    row[: int(boundaries[k])] = True            # draft prefix y_{1:t_k}
    if tree_parent is None:
        row[base: base + s + 1] = True          # causal within its own copy
    else:
        anc = _anc if _anc is not None else ancestor_sets(tree_parent)
        for s2 in anc[s]:
            row[base + s2] = True
    return row


def visible_mask(N: int, K: int, S: int, boundaries: Sequence[int],
                 tree_parent: Optional[Sequence[int]] = None) -> np.ndarray:
    """Dense bool mask M[i, j] = "query i may attend key j" over the packed
    sequence of length L = N + K*S."""
    _check(N, K, S, boundaries)
    anc = ancestor_sets(tree_parent) if tree_parent is not None else None
    if tree_parent is not None and len(tree_parent) != S:
        raise ValueError("tree_parent must have length S")
    L = packed_length(N, K, S)
    M = np.zeros((L, L), dtype=bool)
    for i in range(L):
        M[i] = visible_row(i, N, K, S, boundaries, tree_parent, anc)
    return M


def visible_keys(i: int, N: int, K: int, S: int, boundaries: Sequence[int],
                 tree_parent: Optional[Sequence[int]] = None) -> np.ndarray:
    """Sorted key indices visible from packed row i (row i of visible_mask)."""
    _check(N, K, S, boundaries)
    return np.nonzero(visible_row(i, N, K, S, boundaries, tree_parent))[0]
