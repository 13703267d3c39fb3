"""Pins for oracle.select: closed forms (decimal, 50 digits), the paper's
thresholds, worked examples, exhaustive rule enumeration, invariants."""

import itertools
import math
from decimal import Decimal, getcontext

import numpy as np
import pytest

import oracle

getcontext().prec = 50


def _sigma_dec(l_c, l_i):
    """Eq. (p2way) exp(l_C)/(exp(l_C)+exp(l_I)) in 50-digit decimal."""
    a, b = Decimal(l_c).exp(), Decimal(l_i).exp()
    return a / (a + b)


def _theta_dec(tau):
    t = Decimal(tau)
    return (t / (1 - t)).ln()


def test_two_way_confidence_worked_and_closed_form(golden):
    for ex in golden["two_way_confidence"]:
        p = oracle.two_way_confidence(ex["l_c"], ex["l_i"])
        assert f"{p:.10f}".startswith(ex["p_prefix"]), ex["cite"]
        assert p == pytest.approx(float(_sigma_dec(ex["l_c"], ex["l_i"])), rel=4e-16, abs=0)


def test_two_way_confidence_random_vs_decimal():
    rng = np.random.default_rng(0)
    for _ in range(2000):
        l_c, l_i = (float(x) for x in rng.normal(0, 10, 2))
        assert oracle.two_way_confidence(l_c, l_i) == pytest.approx(
            float(_sigma_dec(l_c, l_i)), rel=1e-14, abs=1e-300)
    # extreme logits do not overflow
    assert oracle.two_way_confidence(1000.0, -1000.0) == 1.0
    assert oracle.two_way_confidence(-1000.0, 1000.0) == 0.0


def test_confidence_invariants():
    """complement to one, monotone in l_C, shift invariance (1e-12)."""
    rng = np.random.default_rng(1)
    for _ in range(10_000):
        l_c, l_i, c = (float(x) for x in rng.normal(0, 5, 3))
        p = oracle.two_way_confidence(l_c, l_i)
        assert abs(p + oracle.two_way_confidence(l_i, l_c) - 1) <= 1e-12
        assert abs(oracle.two_way_confidence(l_c + c, l_i + c) - p) <= 1e-12
        assert oracle.two_way_confidence(l_c + abs(c), l_i) >= p


def test_logit_threshold_paper_values(golden):
    for tau in golden["paper_thresholds"]["values"]:
        th = oracle.logit_threshold(tau)
        assert th == pytest.approx(float(_theta_dec(tau)), rel=1e-14)
        assert oracle.two_way_confidence(th, 0.0) == pytest.approx(tau, abs=1e-15)
    # SURVEY §8c values for tau_P = 0.985 and tau_F = 0.998
    assert oracle.logit_threshold(0.985) == pytest.approx(4.184591440070, abs=1e-11)
    assert oracle.logit_threshold(0.998) == pytest.approx(6.212606095752, abs=1e-11)
    assert oracle.logit_threshold(0.0) == -math.inf and oracle.logit_threshold(1.0) == math.inf


def test_thresholded_verdict_worked(golden):
    for ex in golden["thresholded_verdict"]:
        got = oracle.final_verdict(ex["l_c"], ex["l_i"], ex["tau"], ex["tie_is_correct"])
        assert got == ex["final"], ex["cite"]
        assert oracle.final_verdict_literal(ex["l_c"], ex["l_i"], ex["tau"], ex["tie_is_correct"]) == ex["final"]


def test_logit_form_equals_literal_form_off_boundary(golden):
    """Reading R7: d >= theta(tau) decides the same as p >= tau except within
    rounding distance of the boundary."""
    rng = np.random.default_rng(2)
    taus = golden["paper_thresholds"]["values"] + [0.5, 0.1]
    n = 0
    for _ in range(20_000):
        tau = float(rng.choice(taus))
        th = oracle.logit_threshold(tau)
        l_i = float(rng.normal())
        d = th + float(rng.normal(0, 2))
        l_c = l_i + d
        if abs((l_c - l_i) - th) < 1e-9:
            continue
        n += 1
        assert oracle.final_verdict(l_c, l_i, tau) == oracle.final_verdict_literal(l_c, l_i, tau)
    assert n > 19_000


def test_threshold_monotone():
    """raising tau never turns Incorrect into Correct."""
    rng = np.random.default_rng(3)
    for _ in range(3000):
        l_c, l_i = (float(x) for x in rng.normal(0, 4, 2))
        t1, t2 = sorted(float(x) for x in rng.uniform(0, 1, 2))
        if oracle.final_verdict(l_c, l_i, t2):
            assert oracle.final_verdict(l_c, l_i, t1)


def _passes(s):
    return [c == "C" for c in s]


def test_k_star_worked(golden):
    for ex in golden["k_star"]:
        p = _passes(ex["verdicts"])
        assert oracle.k_star_leading_run(p) == ex["leading_run"], ex["cite"]
        assert oracle.k_star_max_correct(p) == ex["max_correct"], ex["cite"]


def test_k_star_exhaustive():
    """All 2^K verdict patterns, K <= 12, against the rules stated as
    quantified sets: leading-run = max{k : v_0..v_k all Correct};
    max = max{k : v_k Correct}; -1 for the empty set."""
    for K in range(1, 13):
        for bits in itertools.product([False, True], repeat=K):
            lead = max([k for k in range(K) if all(bits[: k + 1])], default=-1)
            mx = max([k for k in range(K) if bits[k]], default=-1)
            assert oracle.k_star_leading_run(bits) == lead
            assert oracle.k_star_max_correct(bits) == mx


def test_k_star_insert_incorrect_lowers():
    """inserting Incorrect at j <= k* strictly lowers k* (leading run)."""
    for K in range(1, 9):
        for bits in itertools.product([False, True], repeat=K):
            ks = oracle.k_star_leading_run(bits)
            for j in range(0, ks + 1):
                b2 = list(bits)
                b2[j] = False
                assert oracle.k_star_leading_run(b2) < ks


def test_adopted_prefix_len_worked(golden):
    for ex in golden["adopted_prefix_len"]:
        assert oracle.adopted_prefix_len(ex["k_star"], ex["delta"], ex["eta"], ex["T"]) == ex["expect"], ex["cite"]


def test_accepted_len_via_boundaries_equals_eq_adopted():
    """select_prefix returns L* = t_m; with the App. A.1 boundaries this must
    equal Eq. (adopted) min(T, Delta*floor(max(0, k*+1-eta))) for every k*, eta."""
    rng = np.random.default_rng(4)
    for _ in range(400):
        T = int(rng.integers(1, 400))
        delta = int(rng.choice([1, 7, 40, 128]))
        b = oracle.place_boundaries(T, delta)
        K = len(b)
        eta = float(rng.choice([0.0, 0.5, 1.0, 2.0, 3.7]))
        e = int(rng.integers(0, K + 1))                    # first failing chunk
        lg = np.zeros((1, K, 2))
        lg[0, :e, 0] = 10.0
        lg[0, e:, 0] = -10.0
        out = oracle.select_prefix(lg, b, tau=0.985, eta=eta)
        ks = e - 1
        assert out["k_star"][0] == ks
        assert out["accepted_len"][0] == oracle.adopted_prefix_len(ks, delta, eta, T)


def test_select_prefix_stats_worked(golden):
    for ex in golden["reject_rule_stats"]:
        p = _passes(ex["verdicts"])
        K = len(p)
        lg = np.zeros((1, K, 2))
        lg[0, :, 0] = [9.0 if ok else -3.0 for ok in p]
        out = oracle.select_prefix(lg, list(range(1, K + 1)), tau=0.985)
        assert out["n_incorrect"][0] == ex["n_incorrect"], ex["cite"]
        assert out["trailing_incorrect_run"][0] == ex["trailing_incorrect_run"]
        reject = (ex["n_incorrect"] / K > ex["rho"]) or (ex["trailing_incorrect_run"] >= ex["kappa"])
        assert reject == ex["reject"]


def test_select_prefix_scores_min_and_aux():
    lg = np.array([[[3.0, 0.0], [1.0, 0.0], [0.0, 0.0], [-2.0, 0.0]]])
    out = oracle.select_prefix(lg, [1, 2, 3, 4], tau=0.5, aux_tau=0.7)
    want = [float(_sigma_dec(x, 0.0)) for x in (3.0, 1.0, 0.0, -2.0)]
    np.testing.assert_array_equal(out["scores"][0], np.float32(want))
    assert out["min_score"][0] == np.float32(want[3])
    # p < 0.7 for sigma(1)=0.731? no; sigma(0)=0.5 yes; sigma(-2) yes -> 2
    assert out["n_below_aux"][0] == 2
    assert out["k_star"][0] == 2 and out["accepted_len"][0] == 3   # tie passes at tau=0.5


def test_select_prefix_nonfinite():
    lg = np.array([[[5.0, 0.0], [np.nan, 0.0], [5.0, 0.0]],
                   [[np.inf, 0.0], [5.0, 0.0], [5.0, -np.inf]]])
    out = oracle.select_prefix(lg, [1, 2, 3], tau=0.9)
    assert out["nonfinite"].tolist() == [True, True]
    assert out["k_star"].tolist() == [0, -1]
    assert out["k_star"][0] == 0
    assert math.isnan(out["scores"][0, 1])
    assert out["scores"][1, 0] == 1.0 and out["scores"][1, 2] == 1.0
    out2 = oracle.select_prefix(lg, [1, 2, 3], tau=0.9, rule=oracle.RULE_MAX_CORRECT)
    assert out2["k_star"].tolist() == [2, 1]
