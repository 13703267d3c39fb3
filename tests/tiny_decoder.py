"""A tiny seeded decoder used only by the model-level equivalence tests
(SPEC's "refdecoder" idea): pre-RMSNorm attention + MLP blocks
with rotary position embeddings.  The attention step is pluggable so the same
model runs (a) the packed verification sequence through libparse or the
oracle, and (b) K standalone causal passes through torch SDPA."""

from __future__ import annotations

import math

import torch


class TinyDecoder:
    def __init__(self, vocab=64, d_model=128, n_q=2, n_kv=1, head_dim=64, n_layers=2, seed=0,
                 dtype=torch.float64, device="cpu"):
        g = torch.Generator().manual_seed(seed)
        r = lambda *s: torch.randn(*s, generator=g, dtype=torch.float64)  # noqa: E731
        self.n_q, self.n_kv, self.hd, self.dm = n_q, n_kv, head_dim, d_model
        self.emb = r(vocab, d_model) * 0.5
        self.layers = []
        for _ in range(n_layers):
            self.layers.append({
                "wq": r(d_model, n_q * head_dim) / math.sqrt(d_model),
                "wk": r(d_model, n_kv * head_dim) / math.sqrt(d_model),
                "wv": r(d_model, n_kv * head_dim) / math.sqrt(d_model),
                "wo": r(n_q * head_dim, d_model) / math.sqrt(n_q * head_dim),
                "w1": r(d_model, 2 * d_model) / math.sqrt(d_model),
                "w2": r(2 * d_model, d_model) / math.sqrt(2 * d_model),
                "g1": 1 + 0.1 * r(d_model), "g2": 1 + 0.1 * r(d_model)})
        self.gf = 1 + 0.1 * r(d_model)
        self.unembed = r(d_model, vocab) / math.sqrt(d_model)
        self.dtype, self.device = dtype, device
        for lay in self.layers:
            for kk in lay:
                lay[kk] = lay[kk].to(device=device, dtype=dtype)
        self.emb, self.gf, self.unembed = (t.to(device=device, dtype=dtype) for t in (self.emb, self.gf, self.unembed))

    @staticmethod
    def _rms(x, g):
        return x / torch.sqrt((x * x).mean(-1, keepdim=True) + 1e-6) * g

    def _rope(self, x, pos):
        # x [B, L, H, d], pos [B, L] (int) -> rotated x
        d = x.shape[-1]
        inv = 1.0 / (10000 ** (torch.arange(0, d, 2, dtype=torch.float64, device=x.device) / d))
        ang = pos.to(torch.float64)[..., None] * inv                      # [B, L, d/2]
        cos, sin = torch.cos(ang)[:, :, None, :].to(x.dtype), torch.sin(ang)[:, :, None, :].to(x.dtype)
        x1, x2 = x[..., 0::2], x[..., 1::2]
        out = torch.empty_like(x)
        out[..., 0::2] = x1 * cos - x2 * sin
        out[..., 1::2] = x1 * sin + x2 * cos
        return out

    def forward(self, tokens, pos, attend):
        """tokens, pos [B, L]; attend(q, k, v) -> o with q [B, L, Hq, d],
        k/v [B, L, Hkv, d] (already rotated).  Returns logits [B, L, vocab]."""
        x = self.emb[tokens]
        B, L = tokens.shape
        for lay in self.layers:
            hN = self._rms(x, lay["g1"])
            q = (hN @ lay["wq"]).view(B, L, self.n_q, self.hd)
            k = (hN @ lay["wk"]).view(B, L, self.n_kv, self.hd)
            v = (hN @ lay["wv"]).view(B, L, self.n_kv, self.hd)
            q, k = self._rope(q, pos), self._rope(k, pos)
            o = attend(q, k, v).to(x.dtype).reshape(B, L, self.n_q * self.hd)
            x = x + o @ lay["wo"]
            hN = self._rms(x, lay["g2"])
            x = x + torch.nn.functional.silu(hN @ lay["w1"]) @ lay["w2"]
        return self._rms(x, self.gf) @ self.unembed


def sdpa_causal(q, k, v):
    """Standalone causal attention (torch SDPA), GQA by repeating K/V."""
    rep = q.shape[2] // k.shape[2]
    qt, kt, vt = q.transpose(1, 2), k.repeat_interleave(rep, 2).transpose(1, 2), v.repeat_interleave(rep, 2).transpose(1, 2)
    return torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True).transpose(1, 2)


def packed_inputs(draft, suffix, boundaries):
    """Token ids and position ids of the packed sequence (P:208 appended
    layout): draft at positions 0..N-1, copy k at b_k .. b_k+S-1 (R3)."""
    B, N = draft.shape
    K, S = len(boundaries), suffix.shape[-1]
    toks = torch.cat([draft] + [suffix] * K, dim=1)
    pos = torch.cat([torch.arange(N)] + [b + torch.arange(S) for b in boundaries]).expand(B, -1)
    return toks, pos


def sdpa_causal_bf16_inputs(q, k, v):
    """Standalone causal attention on q/k/v rounded to bf16 (what libparse
    receives), evaluated in the input precision."""
    r = lambda t: t.to(torch.bfloat16).to(t.dtype)  # noqa: E731
    return sdpa_causal(r(q), r(k), r(v))


def standalone_judgment_logits(model, draft, suffix, boundaries, attend=sdpa_causal):
    """K separate causal passes on draft[0:b_k] ++ suffix; logits at the last row."""
    out = []
    for b in boundaries:
        toks = torch.cat([draft[:, :b], suffix], dim=1)
        pos = torch.arange(toks.shape[1]).expand(toks.shape[0], -1)
        out.append(model.forward(toks, pos, attend)[:, -1])
    return torch.stack(out, dim=1)        # [B, K, vocab]
