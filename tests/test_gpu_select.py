"""GPU parity: parse_select_prefix vs oracle.select_prefix.  k* and
accepted_len bit-exact; scores within 2 fp32 ulp; stats exact."""

import itertools

import numpy as np
import pytest
import torch

import oracle
import paper_2605_04263_b200 as pb
import workloads

pytestmark = pytest.mark.gpu


def _run(lg, bnd, tau, eta=0.0, rule=0, tie=True, aux=-1.0):
    lg_d = torch.as_tensor(lg).to("cuda")
    b_d = torch.as_tensor(np.asarray(bnd, np.int32)).to("cuda")
    out = pb.parse_select_prefix(lg_d, b_d, tau, eta=eta, rule=rule, tie_is_correct=tie, aux_threshold=aux)
    torch.cuda.synchronize()
    got = {k: v.cpu() for k, v in out.items() if v is not None}
    got.update(pb.unpack_stats(out["stats"]))
    want = oracle.select_prefix(lg_d.cpu().double().numpy(), bnd, tau, eta=eta, rule=rule,
                                tie_is_correct=tie, aux_tau=aux if aux >= 0 else None)
    return got, want


def _assert_equal(got, want):
    np.testing.assert_array_equal(got["k_star"].numpy(), want["k_star"])
    np.testing.assert_array_equal(got["accepted_len"].numpy(), want["accepted_len"])
    for key in ("n_incorrect", "trailing_incorrect_run", "n_below_aux"):
        np.testing.assert_array_equal(got[key].numpy(), want[key])
    gs, ws = got["scores"].numpy(), want["scores"]
    both_nan = np.isnan(gs) & np.isnan(ws)
    ulp = np.abs(gs.view(np.int32).astype(np.int64) - ws.view(np.int32).astype(np.int64))
    assert (both_nan | (ulp <= 2)).all()
    gm, wm = got["min_score"].numpy(), want["min_score"]
    assert ((np.isnan(gm) & np.isnan(wm)) | (np.abs(gm.view(np.int32).astype(np.int64) -
                                                      wm.view(np.int32).astype(np.int64)) <= 2)).all()
    assert bool(got["status"][0] & 1) == bool(want["nonfinite"].any())


@pytest.mark.parametrize("name", list(workloads.CONFIGS))
@pytest.mark.parametrize("tau", [0.985, 0.88])
@pytest.mark.parametrize("rule", [0, 1])
def test_configs(name, tau, rule):
    cfg = workloads.CONFIGS[name]
    lg = workloads.make_verdict_logits(cfg.B, cfg.K, seed=0, config_id=cfg.config_id)
    bnd = np.broadcast_to(workloads.uniform_boundaries(cfg.N, cfg.K), (cfg.B, cfg.K)).copy()
    got, want = _run(lg, bnd, tau, rule=rule, aux=0.90)
    _assert_equal(got, want)


def test_exhaustive_patterns():
    """Every pass/fail pattern for K <= 12, both rules, several eta."""
    for K in (1, 2, 5, 12):
        pats = np.array(list(itertools.product([0, 1], repeat=K)), dtype=np.float32)
        B = pats.shape[0]
        lg = np.zeros((B, K, 2), np.float32)
        lg[:, :, 0] = np.where(pats > 0, 9.0, -4.0)
        bnd = np.broadcast_to(np.arange(1, K + 1, dtype=np.int32) * 40, (B, K)).copy()
        for rule, eta in itertools.product([0, 1], [0.0, 1.0, 2.5]):
            got, want = _run(lg, bnd, 0.985, eta=eta, rule=rule)
            _assert_equal(got, want)


def test_large_k_multiword():
    rng = np.random.default_rng(0)
    for K in (31, 32, 33, 64, 100, 1000, 4097):
        B = 9
        d = rng.normal(5, 4, (B, K)).astype(np.float32)
        d[1, :] = 9.0                                # all pass
        d[2, :] = -9.0                               # none pass
        d[3, : K - 1] = 9.0                          # only the last fails
        li = rng.normal(0, 1, (B, K)).astype(np.float32)
        lg = np.stack([li + d, li], -1)
        bnd = np.sort(rng.integers(0, 5000, (B, K)), axis=1).astype(np.int32)
        for rule in (0, 1):
            got, want = _run(lg, bnd, 0.985, rule=rule, aux=0.9)
            _assert_equal(got, want)


def test_edge_values():
    th = oracle.logit_threshold(0.985)
    lg = np.array([
        [[0.0, 0.0], [1.0, 1.0], [2.0, 2.0]],                   # ties
        [[np.float32(th), 0.0], [5.0, 0.0], [5.0, 0.0]],        # d near theta
        [[np.nan, 0.0], [5.0, 0.0], [5.0, 0.0]],                # NaN
        [[np.inf, 0.0], [5.0, -np.inf], [-np.inf, 0.0]],        # infinities
    ], dtype=np.float32)
    bnd = np.array([[40, 80, 100]] * 4, np.int32)
    for tau, tie in ((0.5, True), (0.5, False), (0.985, True), (0.0, True), (1.0, True)):
        got, want = _run(lg, bnd, tau, tie=tie, aux=0.9)
        _assert_equal(got, want)


def test_bf16_and_strided_vocab_view():
    """l_C / l_I read out of full-vocab rows through strides (pair stride =
    id_I - id_C), in bf16."""
    B, K, V = 3, 17, 50
    rng = np.random.default_rng(2)
    full = torch.from_numpy(rng.normal(0, 4, (B, K, V)).astype(np.float32)).to(torch.bfloat16).cuda()
    idc, idi = 7, 31
    view = full[:, :, idc:]                      # l_C at [...,0], l_I at [..., idi-idc]
    bnd = torch.arange(1, K + 1, dtype=torch.int32, device="cuda") * 40
    out = pb.parse_select_prefix(view, bnd, 0.6, pair_stride=idi - idc)
    torch.cuda.synchronize()
    pair = torch.stack([full[:, :, idc], full[:, :, idi]], -1).float().cpu().numpy()
    want = oracle.select_prefix(pair, bnd.cpu().numpy(), 0.6)
    np.testing.assert_array_equal(out["k_star"].cpu().numpy(), want["k_star"])
    np.testing.assert_array_equal(out["accepted_len"].cpu().numpy(), want["accepted_len"])
