"""PARSE's per-request decision logic (Alg. 2) over the outputs of
the verify pass.  Host control logic only — every number it
compares comes from libparse (parse_select_prefix's scores / k* / accepted
length / stats, and the full-verify pair logits); it runs no compute of the
hot path.

Stages implemented (the LLM calls themselves are out of scope):
  1 premature PV abort: V_p Incorrect under (rho_p, kappa) or
                          >= 3 chunks with p < tau_C^rx
  2 strict full accept: l_C >= l_I and p_F >= tau_F -> Sm
  3 short-draft accept: K <= K_sd and p_F >= min(tau_sd + 0.02(K-1), tau_F^rx) -> Sm
  4 chunk-run rejection: fraction Incorrect > rho or trailing run >= kappa
  5 relaxed accept: p_F >= tau_F^rx and min_k p_k >= tau_C^rx -> Sm
  6 continue / restart: L* > 0 -> Sm+Lg (continue from y_{1:L*}) else Lg
"""

from __future__ import annotations

import dataclasses
import math


@dataclasses.dataclass(frozen=True)
class PolicyConfig:
    """App. A.2 hyper-parameter table."""
    delta: int = 40
    tau_F: float = 0.998
    tau_F_rx: float = 0.95
    tau_C_rx: float = 0.90
    tau_P: float = 0.985
    rho: float = 0.30
    kappa: int = 2
    eta: float = 0.0
    K_sd: int = 2
    tau_sd: float = 0.95          # = tau_F^rx in both configurations
    T_p: int = 300
    rho_p: float = 0.20

    @staticmethod
    def qwen() -> "PolicyConfig":
        return PolicyConfig()

    @staticmethod
    def glm() -> "PolicyConfig":
        return PolicyConfig(tau_F=0.95, tau_F_rx=0.90, tau_C_rx=0.83, tau_P=0.88, rho=0.20, rho_p=0.30, tau_sd=0.90)


def reject_rules(n_incorrect: int, K: int, trailing_incorrect_run: int, rho: float, kappa: int) -> bool:
    """True = the chunk run rejects the draft: "the fraction of
    Incorrect chunks exceeds rho" or "the trailing run of Incorrect chunks
    reaches kappa" (reading R13: strict >, >=)."""
    return (n_incorrect / K > rho) or (trailing_incorrect_run >= kappa)


def short_draft_threshold(K: int, tau_sd: float, tau_F_rx: float) -> float:
    """tau_sd^(K) = min(tau_sd + 0.02 (K - 1), tau_F^rx) (Alg. 2 Stage 3)."""
    return min(tau_sd + 0.02 * (K - 1), tau_F_rx)


def relaxed_accept(full_conf: float, min_chunk_conf: float, cfg: PolicyConfig) -> bool:
    """Alg. 2 Stage 5: p_F >= tau_F^rx and min_k p_k >= tau_C^rx."""
    return full_conf >= cfg.tau_F_rx and min_chunk_conf >= cfg.tau_C_rx


def premature_abort(n_incorrect: int, K: int, trailing_incorrect_run: int, n_below_aux: int,
                    cfg: PolicyConfig) -> bool:
    """Alg. 2 Stage 1: abort drafting iff V_p = Incorrect under
    (rho_p, kappa) or #{k : p_k < tau_C^rx} >= 3 (n_below_aux computed by
    parse_select_prefix with aux_threshold = tau_C^rx)."""
    return reject_rules(n_incorrect, K, trailing_incorrect_run, cfg.rho_p, cfg.kappa) or n_below_aux >= 3


def full_verdict(l_c: float, l_i: float, tau_F: float) -> tuple[bool, float]:
    """Alg. 2 Stage 2: V_F Correct iff l_C >= l_I and p_F >= tau_F."""
    x = l_i - l_c
    p = 1.0 / (1.0 + math.exp(x)) if x < 0 else math.exp(-x) / (1.0 + math.exp(-x))
    return (l_c >= l_i and p >= tau_F), p


@dataclasses.dataclass
class Decision:
    label: str             # "Sm" | "Sm+Lg" | "Lg"
    adopted_len: int       # L*: draft tokens kept (T for Sm)
    stage: int             # Alg. 2 stage that decided
    partial_verify: bool   # whether the packed verify pass was needed


def decide(T: int, full_logits: tuple[float, float], cfg: PolicyConfig, partial=None) -> Decision:
    """Stages 2-6 for one request with a T-token draft.  `partial` is a
    callable returning this request's parse_select_prefix results (dict with
    accepted_len, n_incorrect, trailing_incorrect_run, min_score) — invoked
    only when Alg. 2 reaches Stage 4, mirroring the one packed pass."""
    K = -(-T // cfg.delta)
    strict, p_full = full_verdict(full_logits[0], full_logits[1], cfg.tau_F)
    if strict:
        return Decision("Sm", T, 2, False)
    if K <= cfg.K_sd and p_full >= short_draft_threshold(K, cfg.tau_sd, cfg.tau_F_rx):
        return Decision("Sm", T, 3, False)
    r = partial()
    if relaxed_accept(p_full, float(r["min_score"]), cfg):
        return Decision("Sm", T, 5, True)
    L_star = int(r["accepted_len"])
    return Decision("Sm+Lg" if L_star > 0 else "Lg", L_star, 6, True)
