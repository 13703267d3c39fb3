"""CPU tests of the C ABI's host side (no GPU): the library loads and exports
every symbol include/parse.h declares; argument validation; and the tile
schedule checked against the oracle's dense mask — every
visible (row, key) pair is covered exactly once by the KV tiles of the one
item that owns the row, and no emitted KV tile is fully masked for all of
its item's rows."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

import oracle
import paper_2605_04263_b200 as pb
import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built_library():
    from paper_2605_04263_b200 import build
    build.build()
    pb.load_library()


def test_exports_match_header():
    with open(os.path.join(ROOT, "include", "parse.h")) as f:
        header = f.read()
    declared = set(re.findall(r"PARSE_API\s+[\w\s\*]+?\b(parse_\w+)\s*\(", header))
    assert declared == set(pb.EXPORTED_SYMBOLS)
    lib = pb.load_library()
    for name in declared:
        assert hasattr(lib, name), name
    assert pb.parse_version() == 100


def _meta(B, L, Hq, Hkv, d):
    q = torch.empty((B, L, Hq, d), dtype=torch.bfloat16, device="meta")
    k = torch.empty((B, L, Hkv, d), dtype=torch.bfloat16, device="meta")
    return q, k, k


def test_workspace_size_and_validation():
    q, k, v = _meta(2, 100 + 4 * 8, 4, 2, 128)
    n = pb.parse_verify_attn_workspace_size(q, k, v, [25, 50, 75, 100], 4, 8)
    assert n > 0
    bad = [
        (dict(boundaries=[25, 50, 75, 101]), pb.PARSE_ERR_INVALID),     # b > N
        (dict(boundaries=[-1, 50, 75, 100]), pb.PARSE_ERR_INVALID),     # b < 0
        (dict(tree_parent=[-1, 0, 5, 1, 2, 3, 4, 5]), pb.PARSE_ERR_INVALID),  # parent >= s
    ]
    for kw, status in bad:
        args = dict(boundaries=[25, 50, 75, 100], tree_parent=None)
        args.update(kw)
        with pytest.raises(pb.ParseError) as ei:
            pb.parse_verify_attn_workspace_size(q, k, v, args["boundaries"], 4, 8, tree_parent=args["tree_parent"])
        assert ei.value.status == status
        assert pb.parse_last_error()
    q96, k96, _ = _meta(1, 132, 2, 1, 96)
    with pytest.raises(pb.ParseError) as ei:
        pb.parse_verify_attn_workspace_size(q96, k96, k96, [25, 50, 75, 100], 4, 8)
    assert ei.value.status == pb.PARSE_ERR_UNSUPPORTED
    qg, kg, _ = _meta(1, 132, 3, 2, 128)                  # Hq % Hkv != 0
    with pytest.raises(pb.ParseError):
        pb.parse_verify_attn_workspace_size(qg, kg, kg, [25, 50, 75, 100], 4, 8)
    qt, kt, _ = _meta(1, 100 + 4 * 80, 2, 1, 128)         # tree needs S <= 64
    with pytest.raises(pb.ParseError) as ei:
        pb.parse_verify_attn_workspace_size(qt, kt, kt, [25, 50, 75, 100], 4, 80, tree_parent=[-1] * 80)
    assert ei.value.status == pb.PARSE_ERR_UNSUPPORTED


def test_gpu_calls_fail_loudly_without_gpu():
    """No CPU fallback: CPU tensors are rejected, never computed."""
    q = torch.zeros((1, 40, 1, 64), dtype=torch.bfloat16)
    with pytest.raises(pb.ParseError):
        pb.parse_verify_attn(q, q, q, [16, 32], 2, 4)


def test_suffix_positions_match_oracle():
    b = [3, 17, 40]
    assert np.array_equal(pb.parse_suffix_positions(b, 5).numpy(), oracle.suffix_positions(b, 5))


def _check_items(items, Ns, Ks, bnds, Hq, Hkv, S, tree=None):
    """Every (request, row, head) is computed by exactly one item, whose KV
    tiles cover exactly the oracle's visible keys of that row; no emitted
    draft tile is fully masked for all rows of its item."""
    owner = {}
    r = Hq // Hkv
    masks = {b: oracle.visible_mask(Ns[b], Ks[b], S, bnds[b], tree) for b in range(len(Ns))}
    for idx, it in enumerate(items):
        N = Ns[it["b"]]
        hpt = it["flags"] & 0xFF
        nq = 2 if (it["flags"] >> 8) & 1 else 1
        keys = [j * 128 + c for j in range(it["n_draft"]) for c in range(128)]
        self_keys = [it["self_lo"] + j * 128 + c for j in range(it["n_self"]) for c in range(128)]
        seg_draft = set(keys)
        rows_in_item = []
        copy_pair = (it["flags"] >> 9) & 1        # tile 1 = next suffix copy, same heads
        for i in range(nq):
            for row in range(128):
                t = it["t0"] + (i * S if copy_pair else 0) + row // hpt
                h = it["h0"] + (0 if copy_pair else i * hpt) + row % hpt
                assert h // r == it["h0"] // r, "tiles of an item share a KV group"
                if t >= it["t_end"]:
                    continue
                assert (it["b"], t, h) not in owner, "row computed twice"
                owner[(it["b"], t, h)] = idx
                rows_in_item.append(t)
                vis = set(np.nonzero(masks[it["b"]][t])[0].tolist())
                # the kernel's two segments: shared keys < lim (draft seg), own copy (self seg)
                covered = {j for j in seg_draft if j in vis and j < N} | {j for j in self_keys if j in vis and j >= N}
                assert covered == vis, f"row {t} of item {it}: missing {sorted(vis - covered)[:5]}"
        # skip property: every emitted KV tile has a visible key for some row of the item
        for j in range(it["n_draft"]):
            tile = set(range(j * 128, j * 128 + 128))
            assert any(tile & set(np.nonzero(masks[it["b"]][t][:N])[0].tolist()) for t in rows_in_item), \
                f"fully masked draft tile {j} emitted for item {it}"
    total = sum((n + kk * S) for n, kk in zip(Ns, Ks)) * Hq
    assert len(owner) == total, "every (request, row, head) is computed exactly once"


def _check_schedule(B, Hq, Hkv, N, K, S, bnd, tree=None):
    L = N + K * S
    q, k, v = _meta(B, L, Hq, Hkv, 128)
    items = pb.parse_verify_attn_schedule(q, k, v, bnd, K, S, tree_parent=tree)
    bnd2 = np.broadcast_to(np.asarray(bnd), (B, K))
    _check_items(items, [N] * B, [K] * B, [bnd2[b] for b in range(B)], Hq, Hkv, S, tree)
    return items


@pytest.mark.parametrize("case", [
    (1, 1, 1, 128, 4, 8, "uniform"),        # tiny: token-major suffix tiles
    (2, 8, 2, 384, 6, 32, "uniform"),       # head-packed suffix tiles, 2 per item
    (1, 16, 1, 300, 8, 16, "delta40"),      # unaligned boundaries
    (2, 4, 4, 77, 3, 5, "random"),          # ragged N, S not dividing 128
    (1, 8, 2, 256, 4, 64, "tree"),
    (1, 12, 4, 200, 5, 32, "random"),       # r = 3: odd head count per group
])
def test_schedule_covers_mask_exactly(case):
    B, Hq, Hkv, N, K, S, kind = case
    tree = None
    if kind == "uniform":
        bnd = workloads.uniform_boundaries(N, K)
    elif kind == "delta40":
        bnd = np.minimum(np.arange(1, K + 1) * 40, N).astype(np.int32)
    elif kind == "tree":
        bnd = workloads.uniform_boundaries(N, K)
        tree = workloads.make_tree_parent(S, seed=3)
    else:
        rng = np.random.default_rng(N)
        bnd = np.sort(rng.integers(0, N + 1, (B, K)), axis=1).astype(np.int32)
        bnd[:, 0] = 0
    _check_schedule(B, Hq, Hkv, N, K, S, bnd, tree)


def test_schedule_issued_vs_algorithmic_flops_qwen3_235b():
    """Config 3: tile-granular issued work within 1.5% of the visible pairs
    (1.018x: the SELF tile is computed 128 keys wide), and the order is group-major, largest first."""
    cfg = workloads.CONFIGS["qwen3_235b"]
    q, k, v = _meta(cfg.B, cfg.L, cfg.Hq, cfg.Hkv, cfg.d)
    bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
    items = pb.parse_verify_attn_schedule(q, k, v, bnd, cfg.K, cfg.S)
    issued = sum((it["n_draft"] + it["n_self"]) * (2 if it["flags"] >> 8 & 1 else 1) for it in items) * 128 * 128
    pairs = cfg.N * (cfg.N + 1) // 2 + cfg.S * int(bnd.sum()) + cfg.K * cfg.S * (cfg.S + 1) // 2
    algorithmic = pairs * cfg.Hq * cfg.B
    ratio = issued / algorithmic
    assert 1.0 <= ratio < 1.02, ratio          # measured 1.0178 (self tiles are 128 keys wide)
    groups = [it["b"] * cfg.Hkv + it["h0"] // (cfg.Hq // cfg.Hkv) for it in items]
    assert groups == sorted(groups)            # config 3: the 592-item tail lies inside the last group


def test_schedule_tail_is_largest_first_across_groups():
    """Config 2 shape: group-major order, except the last 592 items (4 per
    B200 SM), which are sorted largest first across groups so the launch ends
    on the smallest items."""
    cfg = workloads.CONFIGS["qwen3_8b"]
    q, k, v = _meta(cfg.B, cfg.L, cfg.Hq, cfg.Hkv, cfg.d)
    bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
    items = pb.parse_verify_attn_schedule(q, k, v, bnd, cfg.K, cfg.S)
    cost = [(it["n_draft"] + it["n_self"]) * (2 if it["flags"] >> 8 & 1 else 1) for it in items]
    r = cfg.Hq // cfg.Hkv
    groups = [it["b"] * cfg.Hkv + it["h0"] // r for it in items]
    head, tail = slice(0, len(items) - 592), slice(len(items) - 592, None)
    assert len(items) > 592
    assert groups[head] == sorted(groups[head])
    assert cost[tail] == sorted(cost[tail], reverse=True)
    assert len(set(groups[tail])) > 1          # the window spans several groups
    assert min(cost) == cost[-1]


def test_copy_pair_items_for_single_pack_groups():
    """Qwen3-8B shape (r=4, S=32 -> one head-pack per group): suffix copies
    are paired two per item so both Q tiles of the CTA are busy."""
    items = _check_schedule(1, 8, 2, 256, 5, 32, workloads.uniform_boundaries(256, 5))
    pairs = [it for it in items if (it["flags"] >> 9) & 1]
    assert len(pairs) == 2 * 2                    # copies (0,1), (2,3) x 2 groups; copy 4 alone
    assert all(it["t_end"] - it["t0"] == 64 for it in pairs)


def _varlen_meta(rb, Hq, Hkv, d=128):
    T = sum(rb.Ls)
    q = torch.empty((T, Hq, d), dtype=torch.bfloat16, device="meta")
    if rb.page_size:
        k = torch.empty((8, rb.page_size, Hkv, d), dtype=torch.bfloat16, device="meta")
    else:
        k = torch.empty((T, Hkv, d), dtype=torch.bfloat16, device="meta")
    return q, k


class _FakeTable:
    """Shape/stride stand-in for the DEVICE block table (host-only schedule calls never read it)."""

    def __init__(self, stride):
        self._s = stride

    def data_ptr(self):
        return 256          # never dereferenced by the host-only call

    def stride(self, i):
        return self._s


@pytest.mark.parametrize("page_size", [0, 16, 256])
@pytest.mark.parametrize("Hq,Hkv,S", [(8, 2, 32), (16, 1, 32), (4, 4, 5)])
def test_varlen_schedule_covers_mask_exactly(page_size, Hq, Hkv, S):
    """Ragged batch: per-request N_b / K_b, incl. a K=1 full
    verify (b = N_b) and a K=0 plain prefill; paged K/V aligns self tiles to
    128-key (page) boundaries."""
    Ns, Ks = [300, 77, 129, 260], [None, 1, 0, None]
    rb = workloads.make_ragged_batch(Ns, Hq, Hkv, 8, S, 40, Ks=Ks, page_size=0)
    rb.page_size = page_size
    q, k = _varlen_meta(rb, Hq, Hkv)
    bt = _FakeTable(64) if page_size else None
    items = pb.parse_verify_attn_varlen_schedule(q, k, k, rb.Ns, rb.Ks, rb.boundaries, S, page_size=page_size,
                                                 block_table=bt)
    _check_items(items, rb.Ns, rb.Ks, rb.boundaries, Hq, Hkv, S)
    if page_size:
        assert all(it["self_lo"] % 128 == 0 for it in items if it["n_self"])


def test_varlen_uniform_batch_matches_dense_schedule():
    """A ragged batch whose requests all have the same N and K yields the
    dense call's schedule item for item."""
    Hq, Hkv, S, N = 8, 2, 32, 384
    rb = workloads.make_ragged_batch([N, N], Hq, Hkv, 8, S, 64)
    q, k = _varlen_meta(rb, Hq, Hkv)
    got = pb.parse_verify_attn_varlen_schedule(q, k, k, rb.Ns, rb.Ks, rb.boundaries, S)
    qd, kd, _ = _meta(2, rb.Ls[0], Hq, Hkv, 128)
    want = pb.parse_verify_attn_schedule(qd, kd, kd, np.stack(rb.boundaries), rb.Ks[0], S)
    assert got == want


def test_varlen_validation():
    Hq, Hkv, S = 4, 2, 8
    rb = workloads.make_ragged_batch([100, 60], Hq, Hkv, 8, S, 40)
    q, k = _varlen_meta(rb, Hq, Hkv)
    ok = dict(row_offsets=None)
    pb.parse_verify_attn_varlen_schedule(q, k, k, rb.Ns, rb.Ks, rb.boundaries, S, **ok)
    bad_bnd = [list(rb.boundaries[0]), [61] + list(rb.boundaries[1][1:])]          # b > N_b
    cases = [
        dict(boundaries=bad_bnd),
        dict(row_offsets=[0, sum(rb.Ls)]),                  # request 1 past total_rows
        dict(num_suffixes=[rb.Ks[0], -1]),                  # K_b < 0
        dict(page_size=24, block_table=_FakeTable(16)),     # not a power of two
        dict(page_size=16, block_table=_FakeTable(2)),      # table stride < pages needed
        dict(page_size=16, block_table=None),               # paged without a table
    ]
    for kw in cases:
        args = dict(draft_lens=rb.Ns, num_suffixes=rb.Ks, boundaries=rb.boundaries, row_offsets=None,
                    page_size=0, block_table=None)
        args.update(kw)
        kk = k
        if args["page_size"]:
            kk = torch.empty((8, args["page_size"], Hkv, 128), dtype=torch.bfloat16, device="meta")
        with pytest.raises(pb.ParseError) as ei:
            pb.parse_verify_attn_varlen_schedule(q, kk, kk, args["draft_lens"], args["num_suffixes"],
                                                 args["boundaries"], S, row_offsets=args["row_offsets"],
                                                 page_size=args["page_size"], block_table=args["block_table"])
        assert ei.value.status == pb.PARSE_ERR_INVALID, kw


def test_fp8_entry_validation_without_gpu():
    """FP8 variant (f4): argument errors are reported before any device work;
    CPU tensors are rejected, never computed."""
    lib = pb.load_library()
    from paper_2605_04263_b200.binding import _HostArrays, make_attn_desc
    q = torch.empty((1, 100 + 4 * 8, 2, 128), dtype=torch.float8_e4m3fn, device="meta")
    k = torch.empty((1, 100 + 4 * 8, 1, 128), dtype=torch.float8_e4m3fn, device="meta")
    host = _HostArrays([25, 50, 75, 100], None)
    d = make_attn_desc(q, k, k, None, 4, 8, host, None, pb.PARSE_PREC_FP8_E4M3)
    fake = 1 << 20                                        # never dereferenced: validation fails first
    # FP8 precision through the bf16 entry point
    st = lib.parse_verify_attn(ctypes.byref(d), fake, fake, fake, fake, None, fake, 1 << 30, None)
    assert st == pb.PARSE_ERR_INVALID and "parse_verify_attn_fp8" in pb.parse_last_error()
    # non-positive descale
    st = lib.parse_verify_attn_fp8(ctypes.byref(d), fake, fake, fake, 0.0, 1.0, 1.0, fake, None, fake, 1 << 30, None)
    assert st == pb.PARSE_ERR_INVALID
    # q/k/v strides must be multiples of 16 bytes
    d.q_strides[2] = 136
    st = lib.parse_verify_attn_fp8(ctypes.byref(d), fake, fake, fake, 1.0, 1.0, 1.0, fake, None, fake, 1 << 30, None)
    assert st == pb.PARSE_ERR_INVALID
    with pytest.raises(pb.ParseError):
        qc = torch.zeros((1, 40, 1, 128), dtype=torch.float8_e4m3fn)
        pb.parse_verify_attn_fp8(qc, qc, qc, 1.0, 1.0, 1.0, [16, 32], 2, 4)


def test_plan_create_fails_loudly_without_gpu():
    """Plans validate the descriptor, then need the B200: no CPU fallback."""
    q = torch.zeros((1, 40, 1, 64), dtype=torch.bfloat16)
    with pytest.raises(pb.ParseError):
        pb.VerifyAttnPlan(q, q, q, [16, 32], 2, 4)
    qm, km, _ = _meta(1, 132, 2, 1, 128)
    with pytest.raises(pb.ParseError) as ei:                      # b > N rejected before any device work
        pb.VerifyAttnPlan(qm, km, km, [25, 50, 75, 101], 4, 8)
    assert ei.value.status == pb.PARSE_ERR_INVALID


def _kv_walk(it):
    """The K/V tile keys an item reads, in order (include/parse.h)."""
    return [128 * j for j in range(it["n_draft"])] + [it["self_lo"] + 128 * j for j in range(it["n_self"])]


@pytest.mark.parametrize("config", ["tiny", "qwen3_8b", "qwen3_235b", "tree"])
def test_cluster_units_partition_the_schedule(config):
    """2-CTA cluster units (K/V multicast): every schedule item
    runs exactly once; a multicast pair reads the same request, KV group and
    K/V tile sequence; a lockstep pair has the same step and Q-tile counts;
    a ghost (y = -1) only where no other item could partner it; units keep
    the schedule's order (each at its first item)."""
    cfg = workloads.CONFIGS[config]
    q, k, v = _meta(cfg.B, cfg.L, cfg.Hq, cfg.Hkv, cfg.d)
    bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
    tree = workloads.make_tree_parent(cfg.S, seed=1) if cfg.tree else None
    items = pb.parse_verify_attn_schedule(q, k, v, bnd, cfg.K, cfg.S, tree_parent=tree)
    units = pb.parse_verify_attn_units(q, k, v, bnd, cfg.K, cfg.S, tree_parent=tree)
    r = cfg.Hq // cfg.Hkv
    nq = lambda it: 2 if (it["flags"] >> 8) & 1 else 1            # noqa: E731
    steps = lambda it: it["n_draft"] + it["n_self"]                # noqa: E731
    seen = []
    ghosts = []
    for x, y in units:
        a = items[x]
        seen.append(x)
        if y >= 0:
            b = items[y]
            seen.append(y)
            assert (a["b"], a["h0"] // r) == (b["b"], b["h0"] // r)
            assert _kv_walk(a) == _kv_walk(b) and nq(a) == nq(b)
        elif y <= -2:
            b = items[-y - 2]
            seen.append(-y - 2)
            assert steps(a) == steps(b) and nq(a) == nq(b)
        else:
            ghosts.append(a)
    assert sorted(seen) == list(range(len(items)))
    keys = [(steps(a), nq(a)) for a in ghosts]
    assert len(keys) == len(set(keys)), "two ghosts could have been a lockstep pair"
    firsts = [min(x, y if y >= 0 else (-y - 2 if y <= -2 else x)) for x, y in units]
    assert firsts == sorted(firsts)
    if config in ("qwen3_235b", "tree"):
        assert all(y >= 0 for _, y in units)   # every K/V tile multicast to a pair


def test_parity_cases_cover_every_cluster_unit_kind():
    """The all-element GPU parity shapes (tests/test_gpu_parity_full.py and
    the dense small cases of tests/test_gpu_attn.py) exercise all three 2-CTA
    unit kinds: multicast pairs, lockstep pairs and ghosts (the second CTA
    recomputing an item without storing it)."""
    shapes = [  # (B, Hq, Hkv, N, K, S, boundaries kind, tree)
        (1, 1, 1, 128, 4, 8, "uniform", False),        # tiny (test_gpu_attn small_dense)
        (8, 32, 8, 2048, 16, 32, "uniform", False),    # config 1 at full batch
        (2, 32, 8, 1024, 32, 32, "random", False),     # copy-paired fuzz
        (4, 4, 4, 1536, 16, 64, "random", True),       # token-major tree
        (3, 32, 8, 1024, 31, 32, "random", False),     # odd number of copy-paired suffixes
        (4, 12, 4, 1024, 15, 32, "random", False),     # mixed one / two-tile items
    ]
    kinds = set()
    for B, Hq, Hkv, N, K, S, kind, tree in shapes:
        q, k, v = _meta(B, N + K * S, Hq, Hkv, 128)
        if kind == "uniform":
            bnd = workloads.uniform_boundaries(N, K)
        else:
            rng = np.random.default_rng(N + K)
            bnd = np.sort(rng.integers(0, N + 1, K)).astype(np.int32)
        parent = workloads.make_tree_parent(S, seed=17) if tree else None
        for _, y in pb.parse_verify_attn_units(q, k, v, bnd, K, S, tree_parent=parent):
            kinds.add("multicast" if y >= 0 else "lockstep" if y <= -2 else "ghost")
    assert kinds == {"multicast", "lockstep", "ghost"}, kinds
