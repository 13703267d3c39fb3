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
    vis = visible_mask(_G["N"], _G["K"], _G["S"], _G["bnd"][b])
    x = (q[b, :, h].astype(np.float64) @ k[b, :, g].astype(np.float64).T) / np.sqrt(q.shape[3]) / np.log(2.0)
    x = np.where(vis, x, -np.inf)
    m = x.max(axis=1, keepdims=True)
    e = np.exp2(x - m)
    Z = e.sum(axis=1, keepdims=True)                                 # >= 1
    va = np.abs(v[b, :, g].astype(np.float64))
    normal = (e / Z) @ va                                            # sum_j pi_j |v_j|
    sub = ((x < m - 9.99) & vis).astype(np.float64) @ va             # keys that can round as subnormals
    return b, h, (2.0 ** -4 + 5e-4) * normal + 2.0 ** -14 / Z * sub
