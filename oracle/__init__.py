"""PARSE parallel-prefix-verification ORACLE — test infrastructure, not product.

This package is the plain, slow, obviously-correct CPU reference for the hot
path built in ``paper_2605_04263_b200`` (arxiv 2605.04263, "PARSE").  It is
written from PAPER.md alone, in fp64 NumPy, with an explicit dense boolean
mask and no blocking, fusion or reordering beyond what the paper states.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product
path (``paper_2605_04263_b200``) never imports it and shares no code with
it; the only shared module is ``workloads`` (seeded input generators, which
hold none of the method's arithmetic).

Citations: ``P:<line>`` = /root/reference/PAPER.md line, with its section.

Modules
-------
mask       packed layout + prefix-boundary visibility (§3.2,
           P:519-525 App. A.1, App. A.3)
attention  masked attention over the packed sequence (§3.2)
select     two-way confidence, thresholded verdict, k*, adopted length
           (P:530-539 Eq. p2way, App. A.3, §3.2)
readout    verdict logits from hidden states (final RMSNorm + two LM-head
           rows) and the full-vocabulary readout
pool       verify_attn over independent (request, head) units on all host
           cores (no arithmetic of its own; GPU parity tests, bench.py's
           cpu_baseline and --impl reference)

Pins: every function is checked in ``tests/test_oracle_*.py`` against things
other than itself (brute force per-suffix causal attention, library SDPA,
closed forms, invariants, worked examples under ``tests/golden/``).  No
function here is "parity unpinned".
"""

from .mask import (
    place_boundaries,
    packed_length,
    suffix_spans,
    judgment_positions,
    suffix_positions,
    ancestor_sets,
    visible_mask,
    visible_keys,
)
from .attention import masked_attention, verify_attn, verify_attn_rows
from .select import (
    two_way_confidence,
    logit_threshold,
    raw_verdict,
    final_verdict,
    final_verdict_literal,
    k_star_leading_run,
    k_star_max_correct,
    adopted_prefix_len,
    select_prefix,
    RULE_LEADING_RUN,
    RULE_MAX_CORRECT,
)

__all__ = [
    "place_boundaries", "packed_length", "suffix_spans", "judgment_positions",
    "suffix_positions", "ancestor_sets", "visible_mask", "visible_keys",
    "masked_attention", "verify_attn", "verify_attn_rows",
    "two_way_confidence", "logit_threshold", "raw_verdict", "final_verdict",
    "final_verdict_literal", "k_star_leading_run", "k_star_max_correct",
    "adopted_prefix_len", "select_prefix", "RULE_LEADING_RUN", "RULE_MAX_CORRECT",
]
