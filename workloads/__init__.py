"""Seeded synthetic inputs shared by the oracle-side tests and the GPU path.

This module holds the INPUT RECIPE only (shapes, value distributions,
boundary placement for the BASELINE configs, token-tree shapes, verdict-logit
distributions) and none of the method's arithmetic: no masking, attention,
confidence, threshold or selection code lives here.  Both ``oracle`` users
(tests) and the product path's callers (tests, bench) draw from it.

Recipe (DESIGN.md §4 restates it):
  * Q, K, V ~ N(0, 1) -> bf16 ("base"); "peaky" adds Q ~ N(0, 2^2) and an
    attention-sink key row 0 per KV head (strength 4*sqrt(d)/2 along the
    group's mean-query direction) to stress online-max rescaling.
  * boundaries b_k = (k+1) * N / K (uniform Delta = N/K; "uniformly
    every Delta tokens"); fuzz adds Delta = 40 with a prompt offset.
  * tree: EAGLE-like parent array (depth <= 8, branching <= 4), shared by all
    suffixes (reading R11; not in the paper).
  * verdict logits: first-error index e ~ U{0..K}; d ~ N(8, 2^2) before it,
    N(-1, 3^2) from it on; l_I ~ N(0,1); l_C = l_I + d.
  * seeds: per-request seed = 1000*config_id + request; per tensor offsets
    Q=1, K=2, V=3, logits=4, tree=5 (x 1_000_003 stride), so every GPU count
    sees identical per-request data.
"""

from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np
import torch


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    config_id: int
    B: int
    Hq: int
    Hkv: int
    d: int
    N: int
    K: int
    S: int
    tree: bool = False
    gpus: tuple = (1,)

    @property
    def L(self) -> int:
        return self.N + self.K * self.S

    @property
    def delta(self) -> int:
        return self.N // self.K


# BASELINE.json "configs", in order.
CONFIGS = {
    "tiny": Config("tiny", 0, 1, 1, 1, 64, 128, 4, 8),
    "qwen3_8b": Config("qwen3_8b", 1, 8, 32, 8, 128, 2048, 16, 32),
    "qwen3_235b": Config("qwen3_235b", 2, 16, 64, 4, 128, 8192, 64, 32, gpus=(1, 2, 4, 8)),
    "long": Config("long", 3, 64, 64, 4, 128, 32768, 256, 32, gpus=(8,)),
    "tree": Config("tree", 4, 32, 64, 4, 128, 4096, 32, 64, tree=True, gpus=(8,)),
}

_TENSOR_OFFSET = {"q": 1, "k": 2, "v": 3, "logits": 4, "tree": 5}


def seed_for(config_id: int, request: int, tensor: str) -> int:
    return (1000 * config_id + request) * 1_000_003 + _TENSOR_OFFSET[tensor]


def uniform_boundaries(N: int, K: int) -> np.ndarray:
    """b_k = (k+1) * N / K, k = 0..K-1 (integer division; last one = N)."""
    return np.array([((k + 1) * N) // K for k in range(K)], dtype=np.int32)


def delta_boundaries(T: int, delta: int, prompt_len: int = 0) -> np.ndarray:
    """b_k = P + min((k+1)*Delta, T) (chunking every Delta draft tokens)."""
    K = -(-T // delta)
    return np.array([prompt_len + min((k + 1) * delta, T) for k in range(K)], dtype=np.int32)


def random_boundaries(N: int, K: int, seed: int, allow_zero: bool = True) -> np.ndarray:
    """Sorted random boundaries in [0, N] (fuzz), always including edge values."""
    rng = np.random.default_rng(seed)
    lo = 0 if allow_zero else 1
    b = np.sort(rng.integers(lo, N + 1, size=K)).astype(np.int32)
    return b


def make_tree_parent(S: int, seed: int, max_depth: int = 8, max_branch: int = 4) -> np.ndarray:
    """EAGLE-like token tree: node s>0 picks a parent among earlier nodes whose
    depth < max_depth and child count < max_branch; node 0 is the root."""
    rng = np.random.default_rng(seed)
    parent = np.full(S, -1, dtype=np.int16)
    depth = np.zeros(S, dtype=np.int32)
    children = np.zeros(S, dtype=np.int32)
    for s in range(1, S):
        cand = [p for p in range(s) if depth[p] < max_depth - 1 and children[p] < max_branch]
        # prefer recent nodes (deeper, EAGLE-like chains)
        w = np.array([1.0 + p for p in cand])
        p = int(rng.choice(cand, p=w / w.sum()))
        parent[s] = p
        depth[s] = depth[p] + 1
        children[p] += 1
    return parent


def _randn(shape, seed: int, device, std: float = 1.0) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    if std != 1.0:
        x.mul_(std)
    return x


def make_qkv(cfg: Config, device="cpu", data: str = "base", batch_offset: int = 0,
             batch: Optional[int] = None, N: Optional[int] = None, K: Optional[int] = None,
             S: Optional[int] = None):
    """Q [B, L, Hq, d], K/V [B, L, Hkv, d] bf16, generated per request.

    ``batch_offset``/``batch`` select global request indices
    [batch_offset, batch_offset+batch) so that a rank's shard is identical to
    the same requests generated on one GPU.
    """
    N = cfg.N if N is None else N
    K = cfg.K if K is None else K
    S = cfg.S if S is None else S
    L = N + K * S
    B = cfg.B if batch is None else batch
    q = torch.empty((B, L, cfg.Hq, cfg.d), dtype=torch.bfloat16, device=device)
    k = torch.empty((B, L, cfg.Hkv, cfg.d), dtype=torch.bfloat16, device=device)
    v = torch.empty((B, L, cfg.Hkv, cfg.d), dtype=torch.bfloat16, device=device)
    for i in range(B):
        r = batch_offset + i
        qstd = 2.0 if data == "peaky" else 1.0
        qi = _randn((L, cfg.Hq, cfg.d), seed_for(cfg.config_id, r, "q"), device, qstd)
        ki = _randn((L, cfg.Hkv, cfg.d), seed_for(cfg.config_id, r, "k"), device)
        vi = _randn((L, cfg.Hkv, cfg.d), seed_for(cfg.config_id, r, "v"), device)
        if data == "peaky":
            rr = cfg.Hq // cfg.Hkv
            for g in range(cfg.Hkv):
                u = qi[:, g * rr:(g + 1) * rr, :].mean(dim=(0, 1))
                u = u / u.norm().clamp_min(1e-6)
                ki[0, g] = (4.0 * math.sqrt(cfg.d) / 2.0) * u
        q[i].copy_(qi)
        k[i].copy_(ki)
        v[i].copy_(vi)
    return q, k, v


E4M3_MAX = 448.0


def to_e4m3(x: torch.Tensor):
    """Per-tensor e4m3 encoding of an input tensor for the FP8 variant (the
    form an FP8 checkpoint's activations / KV cache take): returns (x8, descale)
    with x8 = round_e4m3(x / descale), descale = amax(|x|) / 448.  The value the
    method sees is x8 * descale; both the GPU path and the oracle get exactly
    that (the oracle via ``x8.double() * descale``)."""
    # chunked along dim 0 so a large (e.g. 40 GB bf16) input never needs a
    # full fp32 copy; amax of bf16 / fp32 values is exact in either type
    n0 = x.shape[0] if x.dim() > 0 else 1
    xs = [x] if x.dim() == 0 else [x[i:i + 1] for i in range(n0)]
    amax = max(float(c.abs().max()) for c in xs)
    descale = amax / E4M3_MAX if amax > 0 else 1.0
    x8 = torch.empty(x.shape, dtype=torch.float8_e4m3fn, device=x.device)
    if x.dim() == 0:
        x8.copy_((x.float() / descale).clamp(-E4M3_MAX, E4M3_MAX).to(torch.float8_e4m3fn))
    else:
        for i in range(n0):
            x8[i:i + 1].copy_((x[i:i + 1].float() / descale).clamp(-E4M3_MAX, E4M3_MAX).to(torch.float8_e4m3fn))
    return x8, descale


def make_verdict_logits(B: int, K: int, seed: int, device="cpu",
                        batch_offset: int = 0, config_id: int = 0) -> torch.Tensor:
    """[B, K, 2] fp32 (l_C, l_I) per the recipe in the module docstring."""
    out = torch.empty((B, K, 2), dtype=torch.float32)
    for i in range(B):
        rng = np.random.default_rng(seed_for(config_id, batch_offset + i, "logits") + seed)
        e = int(rng.integers(0, K + 1))
        d = np.where(np.arange(K) < e, rng.normal(8.0, 2.0, K), rng.normal(-1.0, 3.0, K))
        li = rng.normal(0.0, 1.0, K)
        out[i, :, 0] = torch.from_numpy((li + d).astype(np.float32))
        out[i, :, 1] = torch.from_numpy(li.astype(np.float32))
    return out.to(device)


@dataclasses.dataclass
class RaggedBatch:
    """A heterogeneous serving batch: per-request shared length
    N_b, chunking every ``delta`` tokens (K_b = ceil(N_b / delta), b_k =
    min((k+1) delta, N_b)), one suffix length S.  Per-request tensors are
    [L_b, H, d] bf16 (CPU); ``q`` / ``k`` / ``v`` hold them packed as the
    varlen call takes them (rows at ``row_offsets``; K/V either packed the same
    way or scattered into a page pool through ``block_table``)."""
    Ns: list
    Ks: list
    S: int
    boundaries: list
    q_list: list
    k_list: list
    v_list: list
    row_offsets: list
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    page_size: int = 0
    block_table: Optional[torch.Tensor] = None

    @property
    def Ls(self) -> list:
        return [n + kk * self.S for n, kk in zip(self.Ns, self.Ks)]


def make_ragged_batch(Ns, Hq: int, Hkv: int, d: int, S: int, delta: int, config_id: int = 50,
                      Ks=None, gap: int = 0, page_size: int = 0, extra_pages: int = 3, data: str = "base",
                      seed: int = 0, device="cpu", keep_lists: bool = True) -> RaggedBatch:
    """Seeded ragged batch.  ``Ks`` overrides K_b (with K_b = 1 -> b_0 = N_b,
    the full-verify pass; K_b = 0 -> no suffix).  ``gap`` inserts unused rows
    between requests.  ``page_size`` > 0 scatters K/V into a pool whose pages
    are a seeded random permutation; unused pool rows hold N(0,1) noise (stale
    cache content), unused block-table entries are -1.  ``device`` = where
    the data is generated and packed (the CPU and CUDA generators draw
    different numbers from the same seed)."""
    B = len(Ns)
    Ks_, bnds = [], []
    for i, N in enumerate(Ns):
        if Ks is not None and Ks[i] in (0, 1):
            K = Ks[i]
            bnds.append(np.array([N] * K, np.int32))
        else:
            b = delta_boundaries(N, delta)
            bnds.append(b)
            K = len(b)
        Ks_.append(K)
    Ls = [n + kk * S for n, kk in zip(Ns, Ks_)]
    cfg = Config("ragged", config_id, 1, Hq, Hkv, d, 1, 1, S)
    ql, kl, vl = [], [], []
    for i in range(B):
        qi, ki, vi = make_qkv(cfg, device=device, data=data, batch_offset=i + seed * 1000, batch=1, N=Ns[i],
                              K=Ks_[i], S=S)
        ql.append(qi[0]); kl.append(ki[0]); vl.append(vi[0])
    offs, r = [], 0
    for L in Ls:
        offs.append(r)
        r += L + gap
    T = r
    q = torch.zeros((T, Hq, d), dtype=torch.bfloat16, device=device)
    for i in range(B):
        q[offs[i]:offs[i] + Ls[i]] = ql[i]
    bt = None
    if page_size == 0:
        k = torch.zeros((T, Hkv, d), dtype=torch.bfloat16, device=device)
        v = torch.zeros((T, Hkv, d), dtype=torch.bfloat16, device=device)
        for i in range(B):
            k[offs[i]:offs[i] + Ls[i]] = kl[i]
            v[offs[i]:offs[i] + Ls[i]] = vl[i]
    else:
        npg = [-(-L // page_size) for L in Ls]
        P = sum(npg) + extra_pages
        g = torch.Generator().manual_seed(seed_for(config_id, 999, "k") + seed)
        perm = torch.randperm(P, generator=g)
        k = _randn((P, page_size, Hkv, d), seed_for(config_id, 998, "k") + seed, device).to(torch.bfloat16)
        v = _randn((P, page_size, Hkv, d), seed_for(config_id, 998, "v") + seed, device).to(torch.bfloat16)
        bt = torch.full((B, max(npg)), -1, dtype=torch.int32)
        c = 0
        for i in range(B):
            for j in range(npg[i]):
                pg = int(perm[c]); c += 1
                bt[i, j] = pg
                lo, hi = j * page_size, min((j + 1) * page_size, Ls[i])
                k[pg, :hi - lo] = kl[i][lo:hi]
                v[pg, :hi - lo] = vl[i][lo:hi]
    if not keep_lists:
        ql = kl = vl = None
    return RaggedBatch(list(Ns), Ks_, S, bnds, ql, kl, vl, offs, q, k, v, page_size, bt)
