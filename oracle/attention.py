"""Masked attention over the packed verification sequence (ORACLE).

What the hot path computes (§3.2): one attention layer of the single
target prefill over the packed sequence, under the prefix-boundary mask of
``oracle.mask``.  For query row i of head h (KV head g = h // (Hq/Hkv)):

    O[i] = sum_{j visible from i} softmax_j(scale * q_i . k_j) * v_j
    LSE[i] = log sum_{j visible} exp(scale * q_i . k_j)          (natural log)

This is the plain definition, evaluated in fp64 with an explicit dense
mask; rows are processed in chunks only to bound memory (a chunk is a set of
independent rows, so no arithmetic is reordered).  scale = 1/sqrt(d) unless
given (reading R10: the paper leaves it to the model).

Inputs are the SAME (bf16) tensors the GPU receives, upcast to fp64 here.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .mask import packed_length, visible_mask, visible_row, ancestor_sets


def _f64(x) -> np.ndarray:
    if hasattr(x, "detach"):                    # torch tensor (CPU or GPU)
        x = x.detach().to("cpu").double().numpy()
    return np.asarray(x, dtype=np.float64)


def masked_attention(q, k, v, mask, scale: float):
    """softmax(scale * q k^T, masked) v in fp64; returns (O, LSE).

    q [Lq, d], k [Lk, d], v [Lk, dv], mask bool [Lq, Lk].  Every row must have
    at least one visible key (true for the PARSE mask: each row sees itself).
    """
    q, k, v = _f64(q), _f64(k), _f64(v)
    mask = np.asarray(mask, dtype=bool)
    if not mask.any(axis=1).all():
        raise ValueError("a query row has no visible key")
    s = (q @ k.T) * scale
    s = np.where(mask, s, -np.inf)
    m = s.max(axis=1, keepdims=True)
    p = np.exp(s - m)
    l = p.sum(axis=1, keepdims=True)
    o = (p @ v) / l
    lse = (m + np.log(l))[:, 0]
    return o, lse


def _boundaries_2d(boundaries, B: int, K: int) -> np.ndarray:
    b = np.asarray(boundaries, dtype=np.int64)
    if b.ndim == 1:
        b = np.broadcast_to(b, (B, K))
    if b.shape != (B, K):
        raise ValueError(f"boundaries must be [K] or [B, K]; got {b.shape}")
    return b


def verify_attn(q, k, v, N: int, K: int, S: int, boundaries,
                tree_parent: Optional[Sequence[int]] = None,
                scale: Optional[float] = None,
                batches: Optional[Sequence[int]] = None,
                heads: Optional[Sequence[int]] = None,
                row_chunk: int = 2048):
    """Full packed verification attention, BSHD layout.

    q [B, L, Hq, d]; k, v [B, L, Hkv, d]; boundaries [K] (shared) or [B, K].
    Returns (O [nb, L, nh, d] fp64, LSE [nb, nh, L] fp64) for the requested
    batch entries / q heads (default all).
    """
    q, k, v = _f64(q), _f64(k), _f64(v)
    B, L, Hq, d = q.shape
    Hkv = k.shape[2]
    if L != packed_length(N, K, S) or Hq % Hkv:
        raise ValueError("shape mismatch")
    r = Hq // Hkv
    sc = 1.0 / np.sqrt(d) if not scale else float(scale)
    bnd = _boundaries_2d(boundaries, B, K)
    batches = list(range(B)) if batches is None else list(batches)
    heads = list(range(Hq)) if heads is None else list(heads)
    O = np.zeros((len(batches), L, len(heads), v.shape[3]))
    LSE = np.zeros((len(batches), len(heads), L))
    for bi, b in enumerate(batches):
        M = visible_mask(N, K, S, bnd[b], tree_parent)
        for hi, h in enumerate(heads):
            g = h // r
            for r0 in range(0, L, row_chunk):
                r1 = min(L, r0 + row_chunk)
                o, lse = masked_attention(q[b, r0:r1, h], k[b, :, g], v[b, :, g],
                                          M[r0:r1], sc)
                O[bi, r0:r1, hi] = o
                LSE[bi, hi, r0:r1] = lse
    return O, LSE


def verify_attn_rows(q, k, v, N: int, K: int, S: int, boundaries,
                     rows: Sequence[tuple[int, int, int]],
                     tree_parent: Optional[Sequence[int]] = None,
                     scale: Optional[float] = None):
    """The same definition evaluated one output row at a time.

    ``rows`` lists (b, t, h) = (request, packed row, q head).  Used for parity
    at full BASELINE sizes, where the dense oracle would not finish: each row
    is computed from its own visible key set (row t of visible_mask).
    q/k/v may be torch tensors on any device; only the needed slices are
    copied to host.  Returns (O [n, d], LSE [n]).
    """
    B, L, Hq, d = q.shape
    Hkv = k.shape[2]
    r = Hq // Hkv
    sc = 1.0 / np.sqrt(d) if not scale else float(scale)
    bnd = _boundaries_2d(boundaries, B, K)
    anc = ancestor_sets(tree_parent) if tree_parent is not None else None
    outs, lses = [], []
    cache: dict = {}
    for (b, t, h) in rows:
        g = h // r
        key = (b, g)
        if key not in cache:
            cache = {key: (_f64(k[b, :, g]), _f64(v[b, :, g]))}
        kb, vb = cache[key]
        vis = visible_row(t, N, K, S, bnd[b], tree_parent, anc)
        o, lse = masked_attention(_f64(q[b, t, h])[None, :], kb, vb, vis[None, :], sc)
        outs.append(o[0])
        lses.append(lse[0])
    return np.stack(outs), np.asarray(lses)
