"""Pins for oracle.readout (CPU): torch's own RMSNorm / logsumexp / softmax in
fp64 as library routines, and closed forms."""

import math

import numpy as np
import torch

from oracle import readout


def test_rms_norm_matches_torch():
    rng = np.random.default_rng(0)
    h = rng.standard_normal((3, 5, 64))
    g = rng.standard_normal(64)
    want = torch.nn.functional.rms_norm(torch.from_numpy(h), (64,), torch.from_numpy(g), eps=1e-6).numpy()
    np.testing.assert_allclose(readout.rms_norm(h, g, 1e-6), want, rtol=1e-13, atol=1e-13)


def test_rms_norm_closed_form():
    # h = c * ones -> mean(h^2) = c^2 -> y = sign(c) * gamma (eps -> 0)
    g = np.arange(1.0, 9.0)
    y = readout.rms_norm(np.full(8, -3.0), g, 1e-300)
    np.testing.assert_allclose(y, -g, rtol=1e-15)


def test_verdict_logits_scale_invariance():
    """RMSNorm makes the logits invariant to scaling h (eps -> 0)."""
    rng = np.random.default_rng(1)
    h, g, w = rng.standard_normal(32), rng.standard_normal(32), rng.standard_normal((2, 32))
    a = readout.verdict_logits(h, g, w, 1e-300)
    b = readout.verdict_logits(7.5 * h, g, w, 1e-300)
    np.testing.assert_allclose(a, b, rtol=1e-13)
    manual = [(h / math.sqrt(np.mean(h * h)) * g) @ w[0], (h / math.sqrt(np.mean(h * h)) * g) @ w[1]]
    np.testing.assert_allclose(a, manual, rtol=1e-13)


def test_vocab_readout_matches_torch_and_closed_form():
    rng = np.random.default_rng(2)
    z = rng.normal(0, 3, (2, 3, 1000))
    out = readout.vocab_readout(z, 7, 911)
    tz = torch.from_numpy(z)
    np.testing.assert_allclose(out["lse"], torch.logsumexp(tz, -1).numpy(), rtol=1e-14)
    sm = torch.softmax(tz, -1).numpy()
    np.testing.assert_allclose(out["verdict_mass"], sm[..., 7] + sm[..., 911], rtol=1e-12)
    # uniform logits: lse = c + log V, mass = 2 / V
    u = readout.vocab_readout(np.full((1, 1, 512), 2.5), 0, 1)
    assert abs(u["lse"][0, 0] - (2.5 + math.log(512))) < 1e-12
    assert abs(u["verdict_mass"][0, 0] - 2 / 512) < 1e-15
