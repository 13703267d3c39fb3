"""Test-side helpers on top of oracle.pool (the parallel fp64 oracle):
re-exports, plus the per-element bound terms of the FP8 parity test."""

import numpy as np

from oracle.pool import _G, available_workers, host_f32, pool_map, verify_attn_parallel  # noqa: F401
from oracle.mask import visible_mask


def fp8_bound_unit(unit):
    """Per-element e4m3 bound terms of one (request, head) unit, see
    tests/test_gpu_parity_full.fp8_bound: (2^-4 + 5e-4) sum_j pi_j |v_j| +
    2^-14 / Z sum_{x_j < m - 10} |v_j| in fp64 (x = log2-domain scores)."""
    b, h = unit
    q, k, v = _G["q"], _G["k"], _G["v"]
    r = q.shape[2] // k.shape[2]
    g = h // r
    vis = visible_mask(_G["N"], _G["K"], _G["S"], _G["bnd"][b], _G.get("tree"))
    x = (q[b, :, h].astype(np.float64) @ k[b, :, g].astype(np.float64).T) / np.sqrt(q.shape[3]) / np.log(2.0)
    x = np.where(vis, x, -np.inf)
    m = x.max(axis=1, keepdims=True)
    e = np.exp2(x - m)
    Z = e.sum(axis=1, keepdims=True)                                 # >= 1
    va = np.abs(v[b, :, g].astype(np.float64))
    normal = (e / Z) @ va                                            # sum_j pi_j |v_j|
    sub = ((x < m - 9.99) & vis).astype(np.float64) @ va             # keys that can round as subnormals
    return b, h, (2.0 ** -4 + 5e-4) * normal + 2.0 ** -14 / Z * sub


def fp8_bound(q, k, v, N, K, S, bnd, O, tree=None):
    """Per-element bound of the FP8 variant against the fp64 oracle on the
    dequantised inputs (include/parse.h, parse_verify_attn_fp8).

    The kernel biases each probability by 2^4 relative to a running max
    m_used in [m - 4, m] (log2 units; the lazy-rescale threshold is 4), rounds
    it to e4m3 and divides by the sum of the unrounded values, l >= 16 Z with
    Z = sum_j 2^(x_j - m) >= 1.  A normal e4m3 rounding is within 2^-4
    relative; below 2^-6 (subnormal) within 2^-10 absolute, which needs
    x_j < m_used - 10 <= m - 10.  So per element
      |dO_c| <= (2^-4 + 5e-4) sum_j pi_j |v_jc| + 2^-14 / Z sum_{x_j < m-10} |v_jc|
                + 2^-8 |O_c| + 1e-5 max|V|
    with pi the exact softmax; 5e-4 covers the exp2 approximation (rel.
    7.5e-5, twice) and the fp32 score / normaliser sums, 2^-8 the bf16
    rounding of O.  The sums are computed in fp64 per (request, head)."""
    qn, kn, vn = host_f32(q), host_f32(k), host_f32(v)
    B, L, Hq, d = qn.shape
    bnd2 = np.asarray(bnd, dtype=np.int64)
    if bnd2.ndim == 1:
        bnd2 = np.broadcast_to(bnd2, (B, K))
    out = np.zeros_like(O)
    units = [(b, h) for b in range(B) for h in range(Hq)]
    shared = dict(q=qn, k=kn, v=vn, bnd=bnd2, N=N, K=K, S=S, tree=tree)
    for b, h, t in pool_map(fp8_bound_unit, units, shared, per_worker_gb=6 * L * L * 8 / 1e9):
        out[b, :, h] = t
    return out + 2.0 ** -8 * np.abs(O) + 1e-5 * float(np.abs(vn).max())
