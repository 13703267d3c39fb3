"""Verdict readout and prefix selection (ORACLE — test infrastructure).

Definitions followed, in the paper's order:

* Two-way confidence, Eq. (p2way) (App. A.1):
      p = exp(l_C) / (exp(l_C) + exp(l_I))
* Thresholded verdict: raw = argmax(l_C, l_I); a raw Correct is
  "downgraded to Incorrect whenever p < tau".  Alg. 2 writes the full-verify
  form as "l_C >= l_I and p >= tau", so a tie counts as Correct
  there; App. A.1 leaves ties undefined.  Reading R6: ``tie_is_correct``
  selects, default True (Alg. 2).
* Decision rounding, reading R7: "p >= tau" is decided in logit space,
  d = l_C - l_I >= theta(tau) = log(tau) - log1p(-tau), both in fp64.  This
  is the same set as p >= tau in exact arithmetic (sigma is monotone); the
  literal form is kept (``final_verdict_literal``) and the two are compared
  in tests away from the rounding boundary.
* k* (App. A.3): "the largest k such that v_k is Correct and no
  Incorrect appears earlier" -> leading run of Correct verdicts, minus one
  (0-indexed; -1 if v_0 is Incorrect).  Variant (§3.2):
  t* = max{t_i | y_{1:t_i} Correct} -> the last Correct index.
* Adopted prefix, Eq. (adopted):
      L* = min(T, Delta * floor(max(0, k* + 1 - eta)))
  Expressed through the boundaries t_k = min(k Delta, T) this is
  L* = t_m with m = floor(max(0, k*+1-eta)), and 0 when m = 0.
* Stats feeding the App. A.3 / Alg. 2 rules:
  number of Incorrect chunks, trailing Incorrect run, number of chunks with
  p < tau_aux, and min_k p_k.

Non-finite logits (reading R15): the pair's verdict is Incorrect and the
request's ``nonfinite`` flag is set.
"""

from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np

RULE_LEADING_RUN = 0     # App. A.3 — the rule "we actually run"
RULE_MAX_CORRECT = 1     # §3.2


def two_way_confidence(l_c: float, l_i: float) -> float:
    """Eq. (p2way): exp(l_C)/(exp(l_C)+exp(l_I)) in fp64.

    Evaluated after dividing numerator and denominator by exp(max(l_C, l_I))
    so nothing overflows: with x = l_I - l_C, p = 1/(1+e^x) for x < 0 and
    e^-x/(1+e^-x) for x >= 0.
    """
    x = float(l_i) - float(l_c)
    if math.isnan(x):
        return math.nan
    if x < 0:
        return 1.0 / (1.0 + math.exp(x))
    e = math.exp(-x)
    return e / (1.0 + e)


def logit_threshold(tau: float) -> float:
    """theta(tau) with sigma(theta) = tau: log(tau) - log1p(-tau) (fp64)."""
    tau = float(tau)
    if not (0.0 <= tau <= 1.0):
        raise ValueError("tau must lie in [0, 1]")
    if tau == 0.0:
        return -math.inf
    if tau == 1.0:
        return math.inf
    return math.log(tau) - math.log1p(-tau)


def raw_verdict(l_c: float, l_i: float, tie_is_correct: bool = True) -> bool:
    """argmax(l_C, l_I); a tie is Correct iff tie_is_correct (R6)."""
    return (l_c > l_i) or (l_c == l_i and bool(tie_is_correct))


def final_verdict(l_c: float, l_i: float, tau: float, tie_is_correct: bool = True) -> bool:
    """Correct iff raw Correct and p >= tau, decided as d >= theta(tau) (R7)."""
    l_c, l_i = float(l_c), float(l_i)
    if not (math.isfinite(l_c) and math.isfinite(l_i)):
        return False
    d = l_c - l_i
    return raw_verdict(l_c, l_i, tie_is_correct) and d >= logit_threshold(tau)


def final_verdict_literal(l_c: float, l_i: float, tau: float, tie_is_correct: bool = True) -> bool:
    """The literal P:537-539 reading: raw Correct and p_2w >= tau (fp64 p)."""
    l_c, l_i = float(l_c), float(l_i)
    if not (math.isfinite(l_c) and math.isfinite(l_i)):
        return False
    return raw_verdict(l_c, l_i, tie_is_correct) and two_way_confidence(l_c, l_i) >= float(tau)


def k_star_leading_run(passes: Sequence[bool]) -> int:
    """Largest k with v_k Correct and no Incorrect earlier; -1 if none."""
    k_star = -1
    for k, ok in enumerate(passes):
        if not ok:
            break
        k_star = k
    return k_star


def k_star_max_correct(passes: Sequence[bool]) -> int:
    """t* = max{t_i | y_{1:t_i} Correct}, as a chunk index; -1 if none."""
    k_star = -1
    for k, ok in enumerate(passes):
        if ok:
            k_star = k
    return k_star


def adopted_prefix_len(k_star: int, delta: int, eta: float, T: int) -> int:
    """Eq. (adopted): min(T, Delta * floor(max(0, k*+1-eta)))."""
    return min(int(T), int(delta) * int(math.floor(max(0.0, k_star + 1 - float(eta)))))


def select_prefix(logits, boundaries, tau: float, eta: float = 0.0,
                  rule: int = RULE_LEADING_RUN, tie_is_correct: bool = True,
                  aux_tau: Optional[float] = None) -> dict:
    """Per-request readout + selection over verdict logits [B, K, 2] = (l_C, l_I).

    ``boundaries`` [K] (shared) or [B, K]: t_k in draft coordinates, used for
    the adopted length L* = t_m (m = floor(max(0, k*+1-eta))), 0 if m = 0.
    Returns numpy arrays: accepted_len, k_star (int32 [B]); scores (float32
    [B, K], p_2w rounded from fp64); n_incorrect, trailing_incorrect_run,
    n_below_aux (int32 [B]); min_score (float32 [B]); nonfinite (bool [B]).
    """
    if hasattr(logits, "detach"):
        logits = logits.detach().to("cpu").double().numpy()
    lg = np.asarray(logits, dtype=np.float64)
    B, K, two = lg.shape
    assert two == 2
    bnd = np.asarray(boundaries, dtype=np.int64)
    if bnd.ndim == 1:
        bnd = np.broadcast_to(bnd, (B, K))
    if eta < 0:
        raise ValueError("eta must be >= 0")
    theta_aux = logit_threshold(aux_tau) if (aux_tau is not None and aux_tau >= 0) else None
    out = {name: np.zeros(B, dtype=np.int32) for name in
           ("accepted_len", "k_star", "n_incorrect", "trailing_incorrect_run", "n_below_aux")}
    out["scores"] = np.zeros((B, K), dtype=np.float32)
    out["min_score"] = np.zeros(B, dtype=np.float32)
    out["nonfinite"] = np.zeros(B, dtype=bool)
    for b in range(B):
        passes = []
        for k in range(K):
            l_c, l_i = float(lg[b, k, 0]), float(lg[b, k, 1])
            if not (math.isfinite(l_c) and math.isfinite(l_i)):
                out["nonfinite"][b] = True
            p = two_way_confidence(l_c, l_i)
            out["scores"][b, k] = np.float32(p)
            ok = final_verdict(l_c, l_i, tau, tie_is_correct)
            passes.append(ok)
            if theta_aux is not None:
                finite = math.isfinite(l_c) and math.isfinite(l_i)
                if not (finite and (l_c - l_i) >= theta_aux):
                    out["n_below_aux"][b] += 1
        ks = k_star_leading_run(passes) if rule == RULE_LEADING_RUN else k_star_max_correct(passes)
        m = int(math.floor(max(0.0, ks + 1 - float(eta))))
        out["k_star"][b] = ks
        out["accepted_len"][b] = int(bnd[b, m - 1]) if m >= 1 else 0
        out["n_incorrect"][b] = sum(1 for ok in passes if not ok)
        run = 0
        for ok in reversed(passes):
            if ok:
                break
            run += 1
        out["trailing_incorrect_run"][b] = run
        sc = out["scores"][b]
        finite_sc = sc[~np.isnan(sc)]
        out["min_score"][b] = finite_sc.min() if finite_sc.size else np.float32(np.nan)
    return out
