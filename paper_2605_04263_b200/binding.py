"""Thin ctypes binding over libparse's C ABI (include/parse.h).

Argument marshalling only: every step of the path runs in libparse's CUDA
kernels.  Functions carry the C names.  Tensors are torch tensors on the
current CUDA device; the stream is torch's current stream unless given.
If libparse.so is missing or fails to load, every call raises — there is no
CPU fallback.
"""

from __future__ import annotations

import ctypes
import math
import os
from typing import Optional

import numpy as np
import torch

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libparse.so")

PARSE_OK, PARSE_ERR_INVALID, PARSE_ERR_UNSUPPORTED, PARSE_ERR_CUDA, PARSE_ERR_WORKSPACE = range(5)
PARSE_PREC_BF16, PARSE_PREC_FP32_DEBUG, PARSE_PREC_FP8_E4M3 = 0, 1, 2
PARSE_RULE_LEADING_RUN, PARSE_RULE_MAX_CORRECT = 0, 1

EXPORTED_SYMBOLS = (
    "parse_verify_attn_workspace_size",
    "parse_verify_attn_schedule",
    "parse_verify_attn_units",
    "parse_verify_attn",
    "parse_verify_attn_fp8",
    "parse_verify_attn_plan_create",
    "parse_verify_attn_plan_run",
    "parse_verify_attn_plan_destroy",
    "parse_verify_attn_varlen_workspace_size",
    "parse_verify_attn_varlen_schedule",
    "parse_verify_attn_varlen",
    "parse_verify_attn_varlen_fp8",
    "parse_select_prefix",
    "parse_select_prefix_allgather",
    "parse_peer_buffer_bytes",
    "parse_peer_export",
    "parse_peer_import",
    "parse_peer_close",
    "parse_verdict_logits",
    "parse_verdict_select",
    "parse_vocab_readout",
    "parse_suffix_positions",
    "parse_last_error",
    "parse_version",
)


class ParseError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libparse status {status}: {msg}")
        self.status = status


class AttnDesc(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32), ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32), ("draft_len", ctypes.c_int32), ("num_suffixes", ctypes.c_int32),
        ("suffix_len", ctypes.c_int32), ("boundaries", ctypes.POINTER(ctypes.c_int32)),
        ("boundary_batch_stride", ctypes.c_int64), ("tree_parent", ctypes.POINTER(ctypes.c_int16)),
        ("softmax_scale", ctypes.c_float), ("precision", ctypes.c_int32),
        ("q_strides", ctypes.c_int64 * 3), ("k_strides", ctypes.c_int64 * 3),
        ("v_strides", ctypes.c_int64 * 3), ("o_strides", ctypes.c_int64 * 3),
    ]


class VarlenDesc(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32), ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32), ("suffix_len", ctypes.c_int32),
        ("draft_lens", ctypes.POINTER(ctypes.c_int32)), ("num_suffixes", ctypes.POINTER(ctypes.c_int32)),
        ("boundaries", ctypes.POINTER(ctypes.c_int32)), ("tree_parent", ctypes.POINTER(ctypes.c_int16)),
        ("softmax_scale", ctypes.c_float), ("precision", ctypes.c_int32),
        ("row_offsets", ctypes.POINTER(ctypes.c_int64)), ("total_rows", ctypes.c_int64),
        ("kv_row_offsets", ctypes.POINTER(ctypes.c_int64)), ("kv_total_rows", ctypes.c_int64),
        ("page_size", ctypes.c_int32), ("num_pages", ctypes.c_int32),
        ("block_table", ctypes.c_void_p), ("block_table_stride", ctypes.c_int32),
        ("q_strides", ctypes.c_int64 * 2), ("k_strides", ctypes.c_int64 * 3),
        ("v_strides", ctypes.c_int64 * 3), ("o_strides", ctypes.c_int64 * 2),
    ]


class WorkItem(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("b", "h0", "t0", "t_end", "self_lo", "n_draft", "n_self", "flags")]


class VerdictHeadDesc(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("num_prefixes", ctypes.c_int32), ("hidden", ctypes.c_int32),
                ("hidden_states", ctypes.c_void_p), ("hs_batch_stride", ctypes.c_int64),
                ("hs_prefix_stride", ctypes.c_int64), ("norm_weight", ctypes.c_void_p),
                ("verdict_rows", ctypes.c_void_p), ("eps", ctypes.c_float)]


class VocabReadoutDesc(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("num_prefixes", ctypes.c_int32), ("vocab", ctypes.c_int32),
                ("vocab_logits", ctypes.c_void_p), ("logits_bf16", ctypes.c_int32),
                ("batch_stride", ctypes.c_int64), ("prefix_stride", ctypes.c_int64),
                ("id_correct", ctypes.c_int32), ("id_incorrect", ctypes.c_int32)]


class PrefixStats(ctypes.Structure):
    _fields_ = [("n_incorrect", ctypes.c_int32), ("trailing_incorrect_run", ctypes.c_int32),
                ("n_below_aux", ctypes.c_int32), ("min_score", ctypes.c_float)]


class SelectDesc(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32), ("num_prefixes", ctypes.c_int32), ("verdict_logits", ctypes.c_void_p),
        ("logits_bf16", ctypes.c_int32), ("logits_batch_stride", ctypes.c_int64),
        ("logits_prefix_stride", ctypes.c_int64), ("logits_pair_stride", ctypes.c_int64),
        ("boundaries", ctypes.c_void_p), ("boundary_batch_stride", ctypes.c_int64),
        ("threshold", ctypes.c_double), ("aux_threshold", ctypes.c_double), ("eta", ctypes.c_double),
        ("rule", ctypes.c_int32), ("tie_is_correct", ctypes.c_int32),
    ]


_lib = None


def load_library(path: str = None) -> ctypes.CDLL:
    """Load libparse.so (raises if it is missing — build it with
    ``python -m paper_2605_04263_b200.build``).  ``PARSE_LIB`` overrides the
    path (used to A/B kernel variants)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("PARSE_LIB") or _LIB_PATH
    if not os.path.exists(path):
        raise ParseError(PARSE_ERR_UNSUPPORTED, f"{path} not built; run python -m paper_2605_04263_b200.build")
    lib = ctypes.CDLL(path)
    lib.parse_verify_attn_workspace_size.argtypes = [ctypes.POINTER(AttnDesc), ctypes.POINTER(ctypes.c_size_t)]
    lib.parse_verify_attn.argtypes = [ctypes.POINTER(AttnDesc)] + [ctypes.c_void_p] * 4 + \
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    if hasattr(lib, "parse_verify_attn_fp8"):        # absent only in older A/B builds (PARSE_LIB)
        lib.parse_verify_attn_fp8.argtypes = [ctypes.POINTER(AttnDesc)] + [ctypes.c_void_p] * 3 + \
            [ctypes.c_float] * 3 + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    if hasattr(lib, "parse_verify_attn_varlen"):     # absent only in older A/B builds (PARSE_LIB)
        lib.parse_verify_attn_varlen_workspace_size.argtypes = [ctypes.POINTER(VarlenDesc),
                                                                ctypes.POINTER(ctypes.c_size_t)]
        lib.parse_verify_attn_varlen.argtypes = [ctypes.POINTER(VarlenDesc)] + [ctypes.c_void_p] * 4 + \
            [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
        lib.parse_verify_attn_varlen_schedule.argtypes = [ctypes.POINTER(VarlenDesc), ctypes.c_void_p,
                                                          ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    lib.parse_select_prefix.argtypes = [ctypes.POINTER(SelectDesc)] + [ctypes.c_void_p] * 6
    if hasattr(lib, "parse_verify_attn_varlen_fp8"):
        lib.parse_verify_attn_varlen_fp8.argtypes = [ctypes.POINTER(VarlenDesc)] + [ctypes.c_void_p] * 3 + \
            [ctypes.c_float] * 3 + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
        lib.parse_verify_attn_varlen_fp8.restype = ctypes.c_int
    if hasattr(lib, "parse_verify_attn_plan_create"):   # absent only in older A/B builds (PARSE_LIB)
        lib.parse_verify_attn_plan_create.argtypes = [ctypes.POINTER(AttnDesc), ctypes.c_void_p, ctypes.c_size_t,
                                                      ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
        lib.parse_verify_attn_plan_run.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 6
        lib.parse_verify_attn_plan_destroy.argtypes = [ctypes.c_void_p]
    if hasattr(lib, "parse_select_prefix_allgather"):   # absent only in older A/B builds (PARSE_LIB)
        lib.parse_select_prefix_allgather.argtypes = [ctypes.POINTER(SelectDesc), ctypes.c_void_p, ctypes.c_int32,
                                                      ctypes.c_int32, ctypes.c_uint32, ctypes.c_void_p,
                                                      ctypes.c_void_p, ctypes.c_void_p]
        lib.parse_peer_buffer_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                ctypes.POINTER(ctypes.c_size_t)]
        lib.parse_peer_export.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]
        lib.parse_peer_import.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]
        lib.parse_peer_close.argtypes = [ctypes.c_void_p]
    lib.parse_verdict_logits.argtypes = [ctypes.POINTER(VerdictHeadDesc), ctypes.c_void_p, ctypes.c_void_p]
    if hasattr(lib, "parse_verdict_select"):          # absent only in older A/B builds (PARSE_LIB)
        lib.parse_verdict_select.argtypes = [ctypes.POINTER(VerdictHeadDesc), ctypes.POINTER(SelectDesc)] + \
            [ctypes.c_void_p] * 8
        lib.parse_verdict_select.restype = ctypes.c_int
    lib.parse_vocab_readout.argtypes = [ctypes.POINTER(VocabReadoutDesc)] + [ctypes.c_void_p] * 4
    lib.parse_verify_attn_schedule.argtypes = [ctypes.POINTER(AttnDesc), ctypes.c_void_p, ctypes.c_size_t,
                                               ctypes.POINTER(ctypes.c_size_t)]
    if hasattr(lib, "parse_verify_attn_units"):       # absent only in older A/B builds (PARSE_LIB)
        lib.parse_verify_attn_units.argtypes = [ctypes.POINTER(AttnDesc), ctypes.c_void_p, ctypes.c_size_t,
                                                ctypes.POINTER(ctypes.c_size_t)]
    lib.parse_suffix_positions.argtypes = [ctypes.POINTER(ctypes.c_int32), ctypes.c_int32, ctypes.c_int32,
                                           ctypes.POINTER(ctypes.c_int32)]
    lib.parse_last_error.restype = ctypes.c_char_p
    lib.parse_version.restype = ctypes.c_int
    for name in ("parse_verify_attn_workspace_size", "parse_verify_attn", "parse_select_prefix",
                 "parse_suffix_positions", "parse_verify_attn_schedule", "parse_verify_attn_units",
                 "parse_verdict_logits",
                 "parse_vocab_readout", "parse_verify_attn_varlen_workspace_size", "parse_verify_attn_varlen",
                 "parse_verify_attn_varlen_schedule", "parse_verify_attn_fp8", "parse_select_prefix_allgather",
                 "parse_peer_buffer_bytes", "parse_peer_export", "parse_peer_import", "parse_peer_close",
                 "parse_verify_attn_plan_create", "parse_verify_attn_plan_run", "parse_verify_attn_plan_destroy"):
        if hasattr(lib, name):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(status: int) -> None:
    if status != PARSE_OK:
        raise ParseError(status, load_library().parse_last_error().decode())


def parse_version() -> int:
    return load_library().parse_version()


def parse_last_error() -> str:
    return load_library().parse_last_error().decode()


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _strides3(t: torch.Tensor):
    s = t.stride()
    if s[3] != 1:
        raise ParseError(PARSE_ERR_INVALID, "head_dim must be contiguous")
    return (ctypes.c_int64 * 3)(s[0], s[1], s[2])


class _HostArrays:
    """Keeps ctypes host buffers alive for the duration of a call."""

    def __init__(self, boundaries, tree_parent):
        b = torch.as_tensor(boundaries, dtype=torch.int32).cpu().contiguous()
        if b.dim() == 1:
            b = b[None, :]
        self.b = b
        self.bptr = ctypes.cast(b.data_ptr(), ctypes.POINTER(ctypes.c_int32))
        self.bstride = 0 if b.shape[0] == 1 else b.stride(0)
        if tree_parent is not None:
            self.t = torch.as_tensor(tree_parent, dtype=torch.int16).cpu().contiguous()
            self.tptr = ctypes.cast(self.t.data_ptr(), ctypes.POINTER(ctypes.c_int16))
        else:
            self.t, self.tptr = None, None


def make_attn_desc(q, k, v, o, num_suffixes: int, suffix_len: int, host: _HostArrays,
                   softmax_scale: Optional[float], precision: int) -> AttnDesc:
    B, L, Hq, D = q.shape
    N = L - num_suffixes * suffix_len
    d = AttnDesc()
    d.batch, d.num_q_heads, d.num_kv_heads, d.head_dim = B, Hq, k.shape[2], D
    d.draft_len, d.num_suffixes, d.suffix_len = N, num_suffixes, suffix_len
    d.boundaries, d.boundary_batch_stride = host.bptr, host.bstride
    d.tree_parent = host.tptr
    d.softmax_scale = float(softmax_scale) if softmax_scale else 0.0
    d.precision = precision
    d.q_strides, d.k_strides, d.v_strides = _strides3(q), _strides3(k), _strides3(v)
    d.o_strides = _strides3(o) if o is not None else (ctypes.c_int64 * 3)(*_strides3(q))
    return d


def parse_verify_attn_workspace_size(q, k, v, boundaries, num_suffixes: int, suffix_len: int,
                                     tree_parent=None, precision: int = PARSE_PREC_BF16) -> int:
    host = _HostArrays(boundaries, tree_parent)
    d = make_attn_desc(q, k, v, None, num_suffixes, suffix_len, host, None, precision)
    n = ctypes.c_size_t(0)
    _check(load_library().parse_verify_attn_workspace_size(ctypes.byref(d), ctypes.byref(n)))
    return int(n.value)


def parse_verify_attn_schedule(q, k, v, boundaries, num_suffixes: int, suffix_len: int, tree_parent=None) -> list:
    """Host-only: the work items the bf16 kernel would run (list of dicts)."""
    host = _HostArrays(boundaries, tree_parent)
    d = make_attn_desc(q, k, v, None, num_suffixes, suffix_len, host, None, PARSE_PREC_BF16)
    n = ctypes.c_size_t(0)
    lib = load_library()
    _check(lib.parse_verify_attn_schedule(ctypes.byref(d), None, 0, ctypes.byref(n)))
    arr = (WorkItem * max(1, n.value))()
    _check(lib.parse_verify_attn_schedule(ctypes.byref(d), ctypes.cast(arr, ctypes.c_void_p), n.value,
                                          ctypes.byref(n)))
    return [{f: getattr(arr[i], f) for f, _ in WorkItem._fields_} for i in range(n.value)]


def parse_verify_attn_units(q, k, v, boundaries, num_suffixes: int, suffix_len: int, tree_parent=None) -> list:
    """Host-only: the 2-CTA cluster launch's work units, (x, y) pairs of
    indices into parse_verify_attn_schedule (include/parse.h)."""
    host = _HostArrays(boundaries, tree_parent)
    d = make_attn_desc(q, k, v, None, num_suffixes, suffix_len, host, None, PARSE_PREC_BF16)
    n = ctypes.c_size_t(0)
    lib = load_library()
    _check(lib.parse_verify_attn_units(ctypes.byref(d), None, 0, ctypes.byref(n)))
    arr = (ctypes.c_int32 * max(2, 2 * n.value))()
    _check(lib.parse_verify_attn_units(ctypes.byref(d), ctypes.cast(arr, ctypes.c_void_p), n.value,
                                       ctypes.byref(n)))
    return [(arr[2 * i], arr[2 * i + 1]) for i in range(n.value)]


def parse_verify_attn(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, boundaries, num_suffixes: int,
                      suffix_len: int, tree_parent=None, softmax_scale: Optional[float] = None,
                      precision: int = PARSE_PREC_BF16, out: Optional[torch.Tensor] = None,
                      lse: Optional[torch.Tensor] = None, want_lse: bool = False,
                      workspace: Optional[torch.Tensor] = None, stream=None):
    """Masked packed-verification attention.  q [B,L,Hq,D], k/v
    [B,L,Hkv,D] bf16 CUDA tensors; boundaries [K] or [B,K] (host ints).
    Returns (O, LSE or None); O is bf16 (or fp32 for PARSE_PREC_FP32_DEBUG)."""
    lib = load_library()
    for t in (q, k, v):
        if t.dtype != torch.bfloat16 or not t.is_cuda:
            raise ParseError(PARSE_ERR_INVALID, "q, k, v must be bf16 CUDA tensors")
    if out is None:
        odt = torch.bfloat16 if precision == PARSE_PREC_BF16 else torch.float32
        out = torch.empty(q.shape, dtype=odt, device=q.device)
    if lse is None and want_lse:
        lse = torch.empty((q.shape[0], q.shape[2], q.shape[1]), dtype=torch.float32, device=q.device)
    host = _HostArrays(boundaries, tree_parent)
    d = make_attn_desc(q, k, v, out, num_suffixes, suffix_len, host, softmax_scale, precision)
    n = ctypes.c_size_t(0)
    _check(lib.parse_verify_attn_workspace_size(ctypes.byref(d), ctypes.byref(n)))
    if workspace is None or workspace.numel() < n.value:
        workspace = torch.empty(max(int(n.value), 16), dtype=torch.uint8, device=q.device)
    _check(lib.parse_verify_attn(ctypes.byref(d), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                 lse.data_ptr() if lse is not None else None, workspace.data_ptr(),
                                 workspace.numel(), _stream_ptr(stream)))
    return out, lse


def parse_verify_attn_fp8(q8: torch.Tensor, k8: torch.Tensor, v8: torch.Tensor, descale_q: float, descale_k: float,
                          descale_v: float, boundaries, num_suffixes: int, suffix_len: int, tree_parent=None,
                          softmax_scale: Optional[float] = None, out: Optional[torch.Tensor] = None,
                          lse: Optional[torch.Tensor] = None, want_lse: bool = False,
                          workspace: Optional[torch.Tensor] = None, stream=None):
    """FP8 variant: q8 [B,L,Hq,128], k8/v8 [B,L,Hkv,128]
    float8_e4m3fn CUDA tensors holding Q/descale_q, K/descale_k, V/descale_v.
    Returns (O bf16, LSE or None)."""
    lib = load_library()
    for t in (q8, k8, v8):
        if t.dtype != torch.float8_e4m3fn or not t.is_cuda:
            raise ParseError(PARSE_ERR_INVALID, "q8, k8, v8 must be float8_e4m3fn CUDA tensors")
    if out is None:
        out = torch.empty(q8.shape, dtype=torch.bfloat16, device=q8.device)
    if lse is None and want_lse:
        lse = torch.empty((q8.shape[0], q8.shape[2], q8.shape[1]), dtype=torch.float32, device=q8.device)
    host = _HostArrays(boundaries, tree_parent)
    d = make_attn_desc(q8, k8, v8, out, num_suffixes, suffix_len, host, softmax_scale, PARSE_PREC_FP8_E4M3)
    n = ctypes.c_size_t(0)
    _check(lib.parse_verify_attn_workspace_size(ctypes.byref(d), ctypes.byref(n)))
    if workspace is None or workspace.numel() < n.value:
        workspace = torch.empty(max(int(n.value), 16), dtype=torch.uint8, device=q8.device)
    _check(lib.parse_verify_attn_fp8(ctypes.byref(d), q8.data_ptr(), k8.data_ptr(), v8.data_ptr(), float(descale_q),
                                     float(descale_k), float(descale_v), out.data_ptr(),
                                     lse.data_ptr() if lse is not None else None, workspace.data_ptr(),
                                     workspace.numel(), _stream_ptr(stream)))
    return out, lse


def parse_verify_attn_varlen_fp8(q8: torch.Tensor, k8: torch.Tensor, v8: torch.Tensor, descale_q: float,
                                 descale_k: float, descale_v: float, draft_lens, num_suffixes, boundaries,
                                 suffix_len: int, row_offsets=None, kv_row_offsets=None,
                                 block_table: Optional[torch.Tensor] = None, page_size: int = 0, tree_parent=None,
                                 softmax_scale: Optional[float] = None, out: Optional[torch.Tensor] = None,
                                 lse: Optional[torch.Tensor] = None, want_lse: bool = False,
                                 workspace: Optional[torch.Tensor] = None, stream=None):
    """FP8 variant of parse_verify_attn_varlen: float8_e4m3fn q8 [T,Hq,128] and
    k8/v8 (packed rows or an e4m3 page pool) holding X / descale_X.
    Returns (O bf16 [T,Hq,128], LSE [Hq,T] or None)."""
    lib = load_library()
    for t in (q8, k8, v8):
        if t.dtype != torch.float8_e4m3fn or not t.is_cuda or t.stride(-1) != 1:
            raise ParseError(PARSE_ERR_INVALID, "q8, k8, v8 must be float8_e4m3fn CUDA tensors, head_dim contiguous")
    if page_size and (block_table is None or not block_table.is_cuda or block_table.dtype != torch.int32):
        raise ParseError(PARSE_ERR_INVALID, "paged K/V needs an int32 CUDA block_table")
    if out is None:
        out = torch.zeros(q8.shape, dtype=torch.bfloat16, device=q8.device)
    if lse is None and want_lse:
        lse = torch.zeros((q8.shape[1], q8.shape[0]), dtype=torch.float32, device=q8.device)
    host = _VarlenHost(draft_lens, num_suffixes, boundaries, suffix_len, row_offsets, kv_row_offsets, tree_parent)
    d = make_varlen_desc(q8, k8, v8, out, host, suffix_len, block_table, page_size, softmax_scale,
                         PARSE_PREC_FP8_E4M3)
    n = ctypes.c_size_t(0)
    _check(lib.parse_verify_attn_varlen_workspace_size(ctypes.byref(d), ctypes.byref(n)))
    if workspace is None or workspace.numel() < n.value:
        workspace = torch.empty(max(int(n.value), 16), dtype=torch.uint8, device=q8.device)
    _check(lib.parse_verify_attn_varlen_fp8(ctypes.byref(d), q8.data_ptr(), k8.data_ptr(), v8.data_ptr(),
                                            float(descale_q), float(descale_k), float(descale_v), out.data_ptr(),
                                            lse.data_ptr() if lse is not None else None, workspace.data_ptr(),
                                            workspace.numel(), _stream_ptr(stream)))
    return out, lse


class VerifyAttnPlan:
    """parse_verify_attn with the schedule built and uploaded once
    (parse_verify_attn_plan_*): `run` only launches, so it can be captured
    into a CUDA graph and reused by every layer with the same geometry.
    q/k/v/out passed to `run` must have the strides of the tensors given here."""

    def __init__(self, q, k, v, boundaries, num_suffixes: int, suffix_len: int, tree_parent=None,
                 softmax_scale: Optional[float] = None, precision: int = PARSE_PREC_BF16,
                 out: Optional[torch.Tensor] = None, stream=None):
        self.lib = load_library()
        host = _HostArrays(boundaries, tree_parent)
        d = make_attn_desc(q, k, v, out, num_suffixes, suffix_len, host, softmax_scale, precision)
        n = ctypes.c_size_t(0)
        self.handle = ctypes.c_void_p(0)
        _check(self.lib.parse_verify_attn_workspace_size(ctypes.byref(d), ctypes.byref(n)))   # validates desc
        if not all(t.is_cuda for t in (q, k, v)):
            raise ParseError(PARSE_ERR_INVALID, "q, k, v must be CUDA tensors")
        self.workspace = torch.empty(max(int(n.value), 16), dtype=torch.uint8, device=q.device)
        _check(self.lib.parse_verify_attn_plan_create(ctypes.byref(d), self.workspace.data_ptr(),
                                                      self.workspace.numel(), _stream_ptr(stream),
                                                      ctypes.byref(self.handle)))
        self.precision = precision

    def run(self, q, k, v, out: torch.Tensor, lse: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        _check(self.lib.parse_verify_attn_plan_run(self.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                   out.data_ptr(), lse.data_ptr() if lse is not None else None,
                                                   _stream_ptr(stream)))
        return out

    def close(self) -> None:
        if self.handle:
            self.lib.parse_verify_attn_plan_destroy(self.handle)
            self.handle = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass


class _VarlenHost:
    """Host arrays of a ragged batch, kept alive for the duration of a call."""

    def __init__(self, draft_lens, num_suffixes, boundaries, suffix_len, row_offsets, kv_row_offsets, tree_parent):
        i32 = lambda x: torch.as_tensor(x, dtype=torch.int32).cpu().contiguous().reshape(-1)  # noqa: E731
        i64 = lambda x: torch.as_tensor(x, dtype=torch.int64).cpu().contiguous().reshape(-1)  # noqa: E731
        self.N, self.K = i32(draft_lens), i32(num_suffixes)
        if isinstance(boundaries, (list, tuple)) and len(boundaries) and not isinstance(boundaries[0], (int, np.integer)):
            boundaries = [int(x) for row in boundaries for x in np.asarray(row).reshape(-1)]
        self.bnd = i32(boundaries) if len(boundaries) else torch.zeros(1, dtype=torch.int32)
        self.L = self.N.to(torch.int64) + self.K.to(torch.int64) * int(suffix_len)
        if row_offsets is None:       # requests packed back to back
            row_offsets = torch.cumsum(self.L, 0) - self.L
        self.rows = i64(row_offsets)
        self.kv_rows = i64(kv_row_offsets) if kv_row_offsets is not None else None
        self.tree = torch.as_tensor(tree_parent, dtype=torch.int16).cpu().contiguous() if tree_parent is not None else None
        p32 = lambda t: ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_int32))  # noqa: E731
        p64 = lambda t: ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_int64))  # noqa: E731
        self.p_N, self.p_K, self.p_bnd, self.p_rows = p32(self.N), p32(self.K), p32(self.bnd), p64(self.rows)
        self.p_kv = p64(self.kv_rows) if self.kv_rows is not None else None
        self.p_tree = ctypes.cast(self.tree.data_ptr(), ctypes.POINTER(ctypes.c_int16)) if self.tree is not None else None


def make_varlen_desc(q, k, v, o, host: _VarlenHost, suffix_len: int, block_table=None, page_size: int = 0,
                     softmax_scale: Optional[float] = None, precision: int = PARSE_PREC_BF16) -> VarlenDesc:
    """q [T,Hq,D]; k/v [Tk,Hkv,D] (contiguous) or [pages,page_size,Hkv,D] (paged)."""
    d = VarlenDesc()
    T, Hq, D = q.shape
    paged = page_size > 0
    Hkv = k.shape[2] if paged else k.shape[1]
    d.batch, d.num_q_heads, d.num_kv_heads, d.head_dim, d.suffix_len = len(host.N), Hq, Hkv, D, suffix_len
    d.draft_lens, d.num_suffixes, d.boundaries, d.tree_parent = host.p_N, host.p_K, host.p_bnd, host.p_tree
    d.softmax_scale = float(softmax_scale) if softmax_scale else 0.0
    d.precision = precision
    d.row_offsets, d.total_rows = host.p_rows, T
    d.kv_row_offsets = host.p_kv
    d.kv_total_rows = 0 if paged else k.shape[0]
    d.page_size = page_size
    if paged:
        d.num_pages = k.shape[0]
        d.block_table = block_table.data_ptr() if block_table is not None else None
        d.block_table_stride = block_table.stride(0) if block_table is not None else 0
        d.k_strides = (ctypes.c_int64 * 3)(*k.stride()[:3])
        d.v_strides = (ctypes.c_int64 * 3)(*v.stride()[:3])
    else:
        d.k_strides = (ctypes.c_int64 * 3)(k.stride(0), k.stride(1), 0)
        d.v_strides = (ctypes.c_int64 * 3)(v.stride(0), v.stride(1), 0)
    d.q_strides = (ctypes.c_int64 * 2)(q.stride(0), q.stride(1))
    oo = o if o is not None else q
    d.o_strides = (ctypes.c_int64 * 2)(oo.stride(0), oo.stride(1))
    return d


def parse_verify_attn_varlen_schedule(q, k, v, draft_lens, num_suffixes, boundaries, suffix_len: int,
                                      row_offsets=None, page_size: int = 0, block_table=None,
                                      tree_parent=None) -> list:
    """Host-only: the work items of a ragged (optionally paged) batch."""
    host = _VarlenHost(draft_lens, num_suffixes, boundaries, suffix_len, row_offsets, None, tree_parent)
    d = make_varlen_desc(q, k, v, None, host, suffix_len, block_table, page_size)
    n = ctypes.c_size_t(0)
    lib = load_library()
    _check(lib.parse_verify_attn_varlen_schedule(ctypes.byref(d), None, 0, ctypes.byref(n)))
    arr = (WorkItem * max(1, n.value))()
    _check(lib.parse_verify_attn_varlen_schedule(ctypes.byref(d), ctypes.cast(arr, ctypes.c_void_p), n.value,
                                                 ctypes.byref(n)))
    return [{f: getattr(arr[i], f) for f, _ in WorkItem._fields_} for i in range(n.value)]


def parse_verify_attn_varlen(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, draft_lens, num_suffixes,
                             boundaries, suffix_len: int, row_offsets=None, kv_row_offsets=None,
                             block_table: Optional[torch.Tensor] = None, page_size: int = 0, tree_parent=None,
                             softmax_scale: Optional[float] = None, precision: int = PARSE_PREC_BF16,
                             out: Optional[torch.Tensor] = None, lse: Optional[torch.Tensor] = None,
                             want_lse: bool = False, workspace: Optional[torch.Tensor] = None, stream=None):
    """Ragged / paged packed verification attention.
    q [T,Hq,D] packed rows (request b at row_offsets[b], default back to
    back); k/v [Tk,Hkv,D] or, with page_size > 0, a page pool
    [pages,page_size,Hkv,D] addressed through block_table (int32 CUDA
    [B, max_pages]).  boundaries: per-request lists or a flat list.
    Returns (O [T,Hq,D], LSE [Hq,T] or None)."""
    lib = load_library()
    for t in (q, k, v):
        if t.dtype != torch.bfloat16 or not t.is_cuda or t.stride(-1) != 1:
            raise ParseError(PARSE_ERR_INVALID, "q, k, v must be bf16 CUDA tensors with head_dim contiguous")
    if page_size and (block_table is None or not block_table.is_cuda or block_table.dtype != torch.int32):
        raise ParseError(PARSE_ERR_INVALID, "paged K/V needs an int32 CUDA block_table")
    if out is None:
        odt = torch.bfloat16 if precision == PARSE_PREC_BF16 else torch.float32
        out = torch.zeros(q.shape, dtype=odt, device=q.device)
    if lse is None and want_lse:
        lse = torch.zeros((q.shape[1], q.shape[0]), dtype=torch.float32, device=q.device)
    host = _VarlenHost(draft_lens, num_suffixes, boundaries, suffix_len, row_offsets, kv_row_offsets, tree_parent)
    d = make_varlen_desc(q, k, v, out, host, suffix_len, block_table, page_size, softmax_scale, precision)
    n = ctypes.c_size_t(0)
    _check(lib.parse_verify_attn_varlen_workspace_size(ctypes.byref(d), ctypes.byref(n)))
    if workspace is None or workspace.numel() < n.value:
        workspace = torch.empty(max(int(n.value), 16), dtype=torch.uint8, device=q.device)
    _check(lib.parse_verify_attn_varlen(ctypes.byref(d), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                        lse.data_ptr() if lse is not None else None, workspace.data_ptr(),
                                        workspace.numel(), _stream_ptr(stream)))
    return out, lse


def _select_desc(lg, bnd, threshold, eta, rule, tie_is_correct, aux_threshold, pair_stride) -> SelectDesc:
    d = SelectDesc()
    d.batch, d.num_prefixes = lg.shape[0], lg.shape[1]
    d.verdict_logits = lg.data_ptr()
    d.logits_bf16 = 1 if lg.dtype == torch.bfloat16 else 0
    d.logits_batch_stride, d.logits_prefix_stride = lg.stride(0), lg.stride(1)
    d.logits_pair_stride = pair_stride * (lg.stride(2) if lg.dim() > 2 else 1)
    d.boundaries = bnd.data_ptr()
    d.boundary_batch_stride = 0 if bnd.dim() == 1 else bnd.stride(0)
    d.threshold, d.aux_threshold, d.eta = float(threshold), float(aux_threshold), float(eta)
    d.rule, d.tie_is_correct = int(rule), 1 if tie_is_correct else 0
    return d


def parse_peer_buffer_bytes(batch: int, num_prefixes: int, world: int) -> int:
    n = ctypes.c_size_t(0)
    _check(load_library().parse_peer_buffer_bytes(batch, num_prefixes, world, ctypes.byref(n)))
    return int(n.value)


def parse_peer_export(ptr: int):
    """(64-byte IPC handle, byte offset) of a device pointer (e.g. a torch CUDA tensor's data_ptr())."""
    h = (ctypes.c_ubyte * 64)()
    off = ctypes.c_uint64(0)
    _check(load_library().parse_peer_export(ptr, h, ctypes.byref(off)))
    return bytes(h), int(off.value)


def parse_peer_import(handle: bytes, offset: int) -> int:
    h = (ctypes.c_ubyte * 64).from_buffer_copy(handle)
    p = ctypes.c_void_p(0)
    _check(load_library().parse_peer_import(h, offset, ctypes.byref(p)))
    return int(p.value)


def parse_peer_close(ptr: int) -> None:
    _check(load_library().parse_peer_close(ptr))


def parse_select_prefix_allgather(verdict_logits: torch.Tensor, boundaries: torch.Tensor, threshold: float,
                                  peer_buffers: torch.Tensor, rank: int, world: int, epoch: int,
                                  eta: float = 0.0, rule: int = PARSE_RULE_LEADING_RUN, tie_is_correct: bool = True,
                                  aux_threshold: float = -1.0, pair_stride: int = 1, stats=None, status=None,
                                  stream=None) -> None:
    """Select fused with the all-gather over peer memory (see include/parse.h).
    peer_buffers: int64 CUDA tensor [world] of every rank's gather buffer as
    mapped in this process.  Results land in every rank's buffer, set epoch % 3."""
    lib = load_library()
    lg = verdict_logits
    if not lg.is_cuda or lg.dtype not in (torch.float32, torch.bfloat16):
        raise ParseError(PARSE_ERR_INVALID, "verdict_logits must be a fp32/bf16 CUDA tensor")
    if not boundaries.is_cuda or boundaries.dtype != torch.int32:
        raise ParseError(PARSE_ERR_INVALID, "boundaries must be an int32 CUDA tensor")
    if not peer_buffers.is_cuda or peer_buffers.dtype != torch.int64:
        raise ParseError(PARSE_ERR_INVALID, "peer_buffers must be an int64 CUDA tensor")
    d = _select_desc(lg, boundaries, threshold, eta, rule, tie_is_correct, aux_threshold, pair_stride)
    _check(lib.parse_select_prefix_allgather(ctypes.byref(d), peer_buffers.data_ptr(), rank, world, epoch,
                                             stats.data_ptr() if stats is not None else None,
                                             status.data_ptr() if status is not None else None, _stream_ptr(stream)))


def parse_select_prefix(verdict_logits: torch.Tensor, boundaries: torch.Tensor, threshold: float,
                        eta: float = 0.0, rule: int = PARSE_RULE_LEADING_RUN, tie_is_correct: bool = True,
                        aux_threshold: float = -1.0, pair_stride: int = 1, want_stats: bool = True,
                        out=None, stream=None) -> dict:
    """Verdict readout + prefix selection.  verdict_logits [B,K,>=2] (fp32 or
    bf16, CUDA; l_C at [..., 0], l_I at [..., pair_stride]); boundaries [K] or
    [B,K] int32 CUDA (t_k in draft coordinates).  Returns a dict of CUDA
    tensors: accepted_len, k_star, scores, stats (int32 [B,3] + min_score),
    status."""
    lib = load_library()
    lg = verdict_logits
    if not lg.is_cuda or lg.dtype not in (torch.float32, torch.bfloat16):
        raise ParseError(PARSE_ERR_INVALID, "verdict_logits must be a fp32/bf16 CUDA tensor")
    B, K = lg.shape[0], lg.shape[1]
    bnd = boundaries
    if not bnd.is_cuda or bnd.dtype != torch.int32:
        raise ParseError(PARSE_ERR_INVALID, "boundaries must be an int32 CUDA tensor")
    dev = lg.device
    if out is None:
        out = {
            "accepted_len": torch.empty(B, dtype=torch.int32, device=dev),
            "k_star": torch.empty(B, dtype=torch.int32, device=dev),
            "scores": torch.empty((B, K), dtype=torch.float32, device=dev),
            "stats": torch.empty((B, 4), dtype=torch.int32, device=dev) if want_stats else None,
            "status": torch.zeros(1, dtype=torch.int32, device=dev),
        }
    d = _select_desc(lg, bnd, threshold, eta, rule, tie_is_correct, aux_threshold, pair_stride)
    st = out["stats"]
    _check(lib.parse_select_prefix(ctypes.byref(d), out["accepted_len"].data_ptr(), out["k_star"].data_ptr(),
                                   out["scores"].data_ptr(), st.data_ptr() if st is not None else None,
                                   out["status"].data_ptr() if out["status"] is not None else None,
                                   _stream_ptr(stream)))
    return out


def parse_verdict_logits(hidden_states: torch.Tensor, norm_weight: torch.Tensor, verdict_rows: torch.Tensor,
                         eps: float = 1e-6, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """(l_C, l_I) = RMSNorm(h) . W_U[{C, I}] for hidden_states [B, K, H] (bf16
    CUDA, may be a strided view of the judgment rows), gamma [H], W_U rows
    [2, H].  Returns fp32 [B, K, 2]."""
    h = hidden_states
    if h.dtype != torch.bfloat16 or h.stride(-1) != 1:
        raise ParseError(PARSE_ERR_INVALID, "hidden_states must be bf16 with a contiguous last dim")
    B, K, H = h.shape
    for name, t, shape in (("norm_weight", norm_weight, (H,)), ("verdict_rows", verdict_rows, (2, H))):
        # required as given: a temporary contiguous copy could be freed and its
        # memory reused before the asynchronous kernel reads it
        if not t.is_cuda or t.device != h.device or t.dtype != torch.bfloat16 or not t.is_contiguous() \
                or tuple(t.shape) != shape:
            raise ParseError(PARSE_ERR_INVALID, f"{name} must be a contiguous bf16 tensor of shape {shape} "
                                                f"on {h.device}")
    if not h.is_cuda:
        raise ParseError(PARSE_ERR_INVALID, "hidden_states must be a CUDA tensor")
    if out is None:
        out = torch.empty((B, K, 2), dtype=torch.float32, device=h.device)
    d = VerdictHeadDesc(B, K, H, h.data_ptr(), h.stride(0), h.stride(1), norm_weight.data_ptr(),
                        verdict_rows.data_ptr(), float(eps))
    _check(load_library().parse_verdict_logits(ctypes.byref(d), out.data_ptr(), _stream_ptr(stream)))
    return out


def parse_verdict_select(hidden_states: torch.Tensor, norm_weight: torch.Tensor, verdict_rows: torch.Tensor,
                         boundaries: torch.Tensor, threshold: float, eps: float = 1e-6, eta: float = 0.0,
                         rule: int = PARSE_RULE_LEADING_RUN, tie_is_correct: bool = True, aux_threshold: float = -1.0,
                         want_stats: bool = True, counters: Optional[torch.Tensor] = None, out=None,
                         stream=None) -> dict:
    """parse_verdict_logits + parse_select_prefix in one launch: hidden_states
    [B, K, H] (bf16 CUDA, may be a strided view of the judgment rows), gamma
    [H], W_U rows [2, H], boundaries [K] or [B, K] int32 CUDA.  counters: int32
    CUDA [B], zero on entry (left zero; pass the same tensor every call to keep
    the call a single launch — if None, a zeroed one is allocated).  Returns
    the parse_select_prefix dict plus 'logits' (fp32 [B, K, 2])."""
    lib = load_library()
    h = hidden_states
    if h.dtype != torch.bfloat16 or h.stride(-1) != 1 or not h.is_cuda:
        raise ParseError(PARSE_ERR_INVALID, "hidden_states must be a bf16 CUDA tensor with a contiguous last dim")
    B, K, H = h.shape
    for name, t, shape in (("norm_weight", norm_weight, (H,)), ("verdict_rows", verdict_rows, (2, H))):
        if not t.is_cuda or t.device != h.device or t.dtype != torch.bfloat16 or not t.is_contiguous() \
                or tuple(t.shape) != shape:
            raise ParseError(PARSE_ERR_INVALID, f"{name} must be a contiguous bf16 tensor of shape {shape} "
                                                f"on {h.device}")
    bnd = boundaries
    if not bnd.is_cuda or bnd.dtype != torch.int32:
        raise ParseError(PARSE_ERR_INVALID, "boundaries must be an int32 CUDA tensor")
    dev = h.device
    if counters is None:
        counters = torch.zeros(B, dtype=torch.int32, device=dev)
    elif not counters.is_cuda or counters.dtype != torch.int32 or counters.numel() < B or not counters.is_contiguous():
        raise ParseError(PARSE_ERR_INVALID, "counters must be a contiguous int32 CUDA tensor of >= batch elements")
    if out is None:
        out = {
            "logits": torch.empty((B, K, 2), dtype=torch.float32, device=dev),
            "accepted_len": torch.empty(B, dtype=torch.int32, device=dev),
            "k_star": torch.empty(B, dtype=torch.int32, device=dev),
            "scores": torch.empty((B, K), dtype=torch.float32, device=dev),
            "stats": torch.empty((B, 4), dtype=torch.int32, device=dev) if want_stats else None,
            "status": torch.zeros(1, dtype=torch.int32, device=dev),
        }
    hd = VerdictHeadDesc(B, K, H, h.data_ptr(), h.stride(0), h.stride(1), norm_weight.data_ptr(),
                         verdict_rows.data_ptr(), float(eps))
    sd = _select_desc(out["logits"], bnd, threshold, eta, rule, tie_is_correct, aux_threshold, 1)
    st = out["stats"]
    _check(lib.parse_verdict_select(ctypes.byref(hd), ctypes.byref(sd), out["logits"].data_ptr(), counters.data_ptr(),
                                    out["accepted_len"].data_ptr(), out["k_star"].data_ptr(), out["scores"].data_ptr(),
                                    st.data_ptr() if st is not None else None,
                                    out["status"].data_ptr() if out["status"] is not None else None,
                                    _stream_ptr(stream)))
    return out


def parse_vocab_readout(vocab_logits: torch.Tensor, id_correct: int, id_incorrect: int, stream=None) -> dict:
    """Full-vocabulary readout of judgment rows [B, K, V] (bf16/fp32 CUDA):
    pair logits [B, K, 2], lse [B, K], verdict mass P(C)+P(I) [B, K]."""
    z = vocab_logits
    if z.dtype not in (torch.bfloat16, torch.float32) or z.stride(-1) != 1:
        raise ParseError(PARSE_ERR_INVALID, "vocab_logits must be bf16/fp32 with contiguous rows")
    B, K, V = z.shape
    dev = z.device
    out = {"pair_logits": torch.empty((B, K, 2), dtype=torch.float32, device=dev),
           "lse": torch.empty((B, K), dtype=torch.float32, device=dev),
           "verdict_mass": torch.empty((B, K), dtype=torch.float32, device=dev)}
    d = VocabReadoutDesc(B, K, V, z.data_ptr(), 1 if z.dtype == torch.bfloat16 else 0, z.stride(0), z.stride(1),
                         int(id_correct), int(id_incorrect))
    _check(load_library().parse_vocab_readout(ctypes.byref(d), out["pair_logits"].data_ptr(), out["lse"].data_ptr(),
                                              out["verdict_mass"].data_ptr(), _stream_ptr(stream)))
    return out


def unpack_stats(stats: torch.Tensor) -> dict:
    """stats int32 [B,4] (parse_prefix_stats_t) -> dict of host tensors."""
    s = stats.cpu()
    return {"n_incorrect": s[:, 0].clone(), "trailing_incorrect_run": s[:, 1].clone(),
            "n_below_aux": s[:, 2].clone(), "min_score": s[:, 3].clone().view(torch.float32)}


def parse_suffix_positions(boundaries, suffix_len: int) -> torch.Tensor:
    b = torch.as_tensor(boundaries, dtype=torch.int32).cpu().contiguous()
    out = torch.empty((b.numel(), suffix_len), dtype=torch.int32)
    _check(load_library().parse_suffix_positions(
        ctypes.cast(b.data_ptr(), ctypes.POINTER(ctypes.c_int32)), b.numel(), suffix_len,
        ctypes.cast(out.data_ptr(), ctypes.POINTER(ctypes.c_int32))))
    return out
