"""paper_2605_04263_b200 — B200-native hot path of PARSE's parallel prefix
verification (arxiv 2605.04263, §3.2 + App. A.3).

The product is ``libparse.so`` (C ABI, ``include/parse.h``), built from
``csrc/`` for sm_100a.  This package is the thin Python binding: the same
names as the C entry points, argument marshalling only.  It never imports
``oracle`` and has no CPU compute path.
"""

from .binding import (  # noqa: F401
    EXPORTED_SYMBOLS,
    PARSE_ERR_CUDA,
    PARSE_ERR_INVALID,
    PARSE_ERR_UNSUPPORTED,
    PARSE_ERR_WORKSPACE,
    PARSE_OK,
    PARSE_PREC_BF16,
    PARSE_PREC_FP32_DEBUG,
    PARSE_PREC_FP8_E4M3,
    PARSE_RULE_LEADING_RUN,
    PARSE_RULE_MAX_CORRECT,
    ParseError,
    VerifyAttnPlan,
    load_library,
    parse_last_error,
    parse_peer_buffer_bytes,
    parse_peer_close,
    parse_peer_export,
    parse_peer_import,
    parse_select_prefix,
    parse_select_prefix_allgather,
    parse_suffix_positions,
    parse_verdict_logits,
    parse_verdict_select,
    parse_vocab_readout,
    parse_verify_attn,
    parse_verify_attn_fp8,
    parse_verify_attn_schedule,
    parse_verify_attn_units,
    parse_verify_attn_varlen,
    parse_verify_attn_varlen_fp8,
    parse_verify_attn_varlen_schedule,
    parse_verify_attn_workspace_size,
    parse_version,
    unpack_stats,
)
