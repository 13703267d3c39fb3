"""Verdict logits from the judge's last layer (ORACLE — test infrastructure).

P:527-529 (App. A.1): "We never sample: instead we read the verifier logits
l_C, l_I at the judgment position".  The paper does not spell out the final
layer; reading R17 takes the standard final norm + LM head of its judges
(Qwen3 / GLM: RMSNorm then a linear vocabulary projection):

    y   = h / sqrt(mean(h^2) + eps) * gamma
    z_v = y . W_U[v]                 (l_C = z_C, l_I = z_I)

Full-vocabulary readout (the "format mismatch": at an arbitrary
boundary the judge puts its mass on chat-template tokens, not on the
verdict): lse = log sum_v exp(z_v), P(C) + P(I) = exp(z_C - lse) + exp(z_I - lse).

Plain fp64 definitions, inputs upcast from the tensors the GPU receives.
"""

from __future__ import annotations

import numpy as np


def _f64(x) -> np.ndarray:
    if hasattr(x, "detach"):
        x = x.detach().to("cpu").double().numpy()
    return np.asarray(x, dtype=np.float64)


def rms_norm(h, gamma, eps: float) -> np.ndarray:
    """y = h / sqrt(mean(h^2, -1) + eps) * gamma (fp64)."""
    h, g = _f64(h), _f64(gamma)
    return h / np.sqrt(np.mean(h * h, axis=-1, keepdims=True) + eps) * g


def verdict_logits(hidden, gamma, verdict_rows, eps: float) -> np.ndarray:
    """(l_C, l_I) for hidden [..., H], verdict_rows [2, H] -> [..., 2]."""
    return rms_norm(hidden, gamma, eps) @ _f64(verdict_rows).T


def vocab_readout(vocab_logits, id_c: int, id_i: int) -> dict:
    """Per row of [..., V]: pair (z_C, z_I), lse, verdict mass P(C)+P(I)."""
    z = _f64(vocab_logits)
    m = z.max(axis=-1, keepdims=True)
    lse = (m + np.log(np.exp(z - m).sum(axis=-1, keepdims=True)))[..., 0]
    zc, zi = z[..., id_c], z[..., id_i]
    return {"pair_logits": np.stack([zc, zi], axis=-1), "lse": lse,
            "verdict_mass": np.exp(zc - lse) + np.exp(zi - lse)}
