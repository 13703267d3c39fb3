"""Alg. 2 host policy against the SPEC's worked examples
(derived from the paper's Alg. 2 and App. A.2 table) and
monotonicity invariants; the partial-verify results come from the oracle's
select (the GPU select is parity-tested bit-exact against it)."""

import numpy as np

import oracle
from paper_2605_04263_b200 import policy


def test_short_draft_threshold_worked():
    assert policy.short_draft_threshold(1, 0.95, 0.95) == 0.95
    assert policy.short_draft_threshold(2, 0.95, 0.95) == 0.95          # S:214 (clamped)
    assert abs(policy.short_draft_threshold(3, 0.90, 0.95) - 0.94) < 1e-12


def test_relaxed_accept_worked():
    q = policy.PolicyConfig.qwen()
    assert policy.relaxed_accept(0.96, 0.92, q)
    assert not policy.relaxed_accept(0.96, 0.85, q)
    assert not policy.relaxed_accept(0.0, 0.0, q)


def test_premature_abort_worked():
    q = policy.PolicyConfig.qwen()                                        # rho_p = 0.20, kappa = 2
    assert not policy.premature_abort(0, 7, 0, 0, q)                      # S:229 clean prefix
    assert policy.premature_abort(2, 7, 0, 0, q)                          # S:230 2/7 = 0.286 > 0.20
    assert policy.premature_abort(0, 7, 0, 3, q)                          # S:231 three chunks p < 0.90


def test_reject_rules_worked(golden):
    for ex in golden["reject_rule_stats"]:
        K = len(ex["verdicts"])
        assert policy.reject_rules(ex["n_incorrect"], K, ex["trailing_incorrect_run"], ex["rho"],
                                   ex["kappa"]) == ex["reject"], ex["cite"]


def _partial(verdicts, delta=40, T=None):
    K = len(verdicts)
    T = T or K * delta
    lg = np.zeros((1, K, 2))
    lg[0, :, 0] = [9.0 if v == "C" else -4.0 for v in verdicts]
    b = oracle.place_boundaries(T, delta)
    out = oracle.select_prefix(lg, b, 0.985, aux_tau=0.90)
    return lambda: {k: v[0] for k, v in out.items() if k != "scores"}


def test_decide_worked():
    q = policy.PolicyConfig.qwen()
    lc_999 = float(np.log(0.999 / 0.001))          # p_F = 0.999 >= tau_F = 0.998
    d = policy.decide(160, (lc_999, 0.0), q, partial=None)
    assert (d.label, d.stage, d.partial_verify) == ("Sm", 2, False)     # S:237 strict accept
    d = policy.decide(160, (0.0, 0.0), q, partial=_partial("CCII"))
    assert (d.label, d.adopted_len) == ("Sm+Lg", 80)                    # S:238 SmLg, 2*Delta
    d = policy.decide(120, (-2.2, 0.0), q, partial=_partial("III"))
    assert d.label == "Lg" and d.adopted_len == 0                       # S:239 nothing adoptable


def test_strict_threshold_monotone():
    """Raising tau_F never turns a non-Sm outcome into Sm."""
    rng = np.random.default_rng(0)
    for _ in range(200):
        lc = float(rng.normal(4, 3))
        part = _partial("".join(rng.choice(["C", "I"], 5)))
        lo = policy.decide(200, (lc, 0.0), policy.PolicyConfig(tau_F=0.9), partial=part)
        hi = policy.decide(200, (lc, 0.0), policy.PolicyConfig(tau_F=0.999), partial=part)
        if lo.label != "Sm":
            assert hi.label != "Sm" or hi.stage != 2
