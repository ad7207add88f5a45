"""ctypes binding of lib/libkvtier_b200.so (the C ABI declared in include/kvtier_b200.h).

There is no fallback: if the library is missing this module raises ImportError, and
every compute entry point requires a CUDA device.  Status codes from the ABI map onto the
reference's exception types (ValueError / RuntimeError, chunk_tree.py:251-252,275-279,
importance.py:31-32).
"""

from __future__ import annotations

import ctypes
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "lib" / "libkvtier_b200.so"
HEADER = _PKG.parent / "include" / "kvtier_b200.h"

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a extension first "
        "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_2506_20187_b200/csrc). "
        "This package has no CPU fallback."
    )

_L = ctypes.CDLL(str(LIB_PATH))

# status codes (kvt_status)
OK, ERR_SHAPE, ERR_K, ERR_COLD, ERR_OOM, ERR_CUDA, ERR_DTYPE, ERR_ARG = 0, -1, -2, -3, -4, -5, -6, -7
# dtype codes (kvt_dtype)
F32, F64, BF16, F16, I4 = 0, 1, 2, 3, 4

_i64, _i32, _vp, _dp, _fp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p
_sz = ctypes.c_size_t


class KvtLayerArgs(ctypes.Structure):
    """Mirror of kvt_layer_args (include/kvtier_b200.h)."""

    _fields_ = [
        ("n_lanes", _i64), ("n", _i64), ("k", _i64),
        ("d", _i32), ("C", _i32),
        ("key_dtype", _i32), ("v_dtype", _i32), ("q_dtype", _i32), ("abs_dtype", _i32),
        ("q", _vp), ("keys", _vp), ("values", _vp), ("lane_stride", _i64),
        ("amax", _vp), ("amin", _vp), ("abs_lane_stride", _i64),
        ("leaf_start", _vp), ("n_leaves", _vp), ("leaf_stride", _i64),
        ("sel_tok", _vp), ("sel_score", _vp), ("n_sel", _vp),
        ("run_start", _vp), ("run_len", _vp), ("n_runs", _vp),
        ("out", _vp), ("evals", _vp),
        ("attn_splits", _i32), ("score_blocks", _i32), ("exact_scores", _i32),
        ("abs_mag", _vp), ("kv_group", _i32), ("sel_hint", _vp),
    ]


class KvtTierArgs(ctypes.Structure):
    """Mirror of kvt_tier_args (include/kvtier_b200.h)."""

    _fields_ = [
        ("n_lanes", _i64), ("kv_group", _i32), ("d", _i32), ("crec", _i32), ("step", _vp),
        ("run_start", _vp), ("run_len", _vp), ("n_runs", _vp), ("run_stride", _i64),
        ("table", _vp), ("table_base", _i64), ("table_stride", _i64), ("n_lk", _i64),
        ("stamp", _vp), ("owner", _vp), ("n_slots", _i64),
        ("free_stack", _vp), ("free_top", _vp), ("victims", _vp), ("slot_of_miss", _vp),
        ("miss", _vp), ("miss_cap", _i64), ("ctl", _vp), ("pool", _vp),
        ("host_i4", _vp), ("host_raw", _vp), ("host_lane_tokens", _i64), ("n_tok", _i64),
        ("theta", _vp), ("ledger_rec_bytes", ctypes.c_longlong), ("ledger_row", _vp),
    ]


def _sig(name, restype, *argtypes):
    f = getattr(_L, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


kvt_version = _sig("kvt_version", ctypes.c_int)
kvt_status_string = _sig("kvt_status_string", ctypes.c_char_p, ctypes.c_int)
kvt_last_error = _sig("kvt_last_error", ctypes.c_char_p)
kvt_abstract_build = _sig("kvt_abstract_build", ctypes.c_int, _vp, _i32, _i64, _i64, _i64, _i32, _i32, _i64, _i64,
                          _vp, _vp, _i32, _i64, _vp)
kvt_abstract_spans = _sig("kvt_abstract_spans", ctypes.c_int, _vp, _i32, _i64, _i32, _i64, _vp, _vp, _vp, _vp, _vp,
                          _vp)
kvt_chunk_bounds = _sig("kvt_chunk_bounds", ctypes.c_int, _vp, _i32, _i64, _i32, _i64, _i32, _vp, _vp, _i64, _vp,
                        _vp, _i32, _i64, _vp, _vp, _vp, _i64, _i32, _vp)
kvt_chunk_bounds_fast = _sig("kvt_chunk_bounds_fast", ctypes.c_int, _vp, _i64, _i32, _i64, _i32, _vp, _vp, _i64,
                             _vp, _vp, _vp, _vp, _i64, _vp)
kvt_select_plan2 = _sig("kvt_select_plan2", ctypes.c_int, _i64, _i64, _i32, _vp, _vp, _i64, _vp, _vp, _i64, _i64, _vp,
                        _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp)
kvt_select_plan_group = _sig("kvt_select_plan_group", ctypes.c_int, _i64, _i64, _i32, _vp, _vp, _i64, _vp, _vp, _i64,
                             _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp)
kvt_cand_score_f32 = _sig("kvt_cand_score_f32", ctypes.c_int, _vp, _i32, _vp, _i32, _i64, _i64, _i32, _vp, _i64, _vp,
                          _vp, _vp, _i64, _vp)
kvt_i4_qprep_bytes = _sig("kvt_i4_qprep_bytes", _sz, _i64, _i32)
kvt_i4_qprep = _sig("kvt_i4_qprep", ctypes.c_int, _vp, _i32, _i64, _i32, _vp, _vp)
kvt_cand_score_i4mma = _sig("kvt_cand_score_i4mma", ctypes.c_int, _vp, _i32, _vp, _i64, _i64, _i32, _vp, _i64, _vp,
                            _vp, _vp, _i64, _vp, _vp, _vp)
kvt_topk_select_band = _sig("kvt_topk_select_band", ctypes.c_int, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _vp, _i32,
                            _vp, _i32, _i64, _i32, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp)
kvt_token_scores = _sig("kvt_token_scores", ctypes.c_int, _vp, _i32, _vp, _i32, _i64, _i64, _i64, _i32, _vp, _i64,
                        _vp)
kvt_select_plan = _sig("kvt_select_plan", ctypes.c_int, _i64, _i64, _i32, _vp, _vp, _i64, _vp, _vp, _i64, _i64, _vp,
                       _i64, _vp, _vp, _vp, _vp, _vp)
kvt_cand_score = _sig("kvt_cand_score", ctypes.c_int, _vp, _i32, _vp, _i32, _i64, _i64, _i32, _vp, _i64, _vp, _vp,
                      _vp, _i64, _i32, _vp)
kvt_topk_select = _sig("kvt_topk_select", ctypes.c_int, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp)
kvt_topk_select_runs = _sig("kvt_topk_select_runs", ctypes.c_int, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64,
                            _vp, _vp, _vp, _i64, _vp, _vp)
kvt_runs_scan = _sig("kvt_runs_scan", ctypes.c_int, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _i64,
                     _vp, _vp)
kvt_attn_workspace_bytes = _sig("kvt_attn_workspace_bytes", _sz, _i64, _i32, _i32)
kvt_sparse_decode_attn = _sig("kvt_sparse_decode_attn", ctypes.c_int, _vp, _i32, _i64, _i64, _i32, _vp, _vp, _vp,
                              _i64, ctypes.c_double, _i32, _vp, _vp, _vp, _vp)
kvt_set_kv_group = _sig("kvt_set_kv_group", ctypes.c_int, _i32)
kvt_set_cand_group = _sig("kvt_set_cand_group", ctypes.c_int, _i32)
kvt_abstract_merge = _sig("kvt_abstract_merge", ctypes.c_int, _vp, _vp, _i32, _i64, _i32, _i64, _vp, _vp, _vp,
                          _i32, _i64, _i64, _vp, _vp, _i64, _vp)
kvt_kv_append = _sig("kvt_kv_append", ctypes.c_int, _vp, _vp, _i32, _i64, _i64, _i64, _i64, _i32, _i64, _vp, _vp, _i64,
                     _i64, _vp, _i32, _vp, _vp)
kvt_nccl_available = _sig("kvt_nccl_available", ctypes.c_int)
kvt_nccl_unique_id = _sig("kvt_nccl_unique_id", ctypes.c_int, _vp)
kvt_nccl_comm_init = _sig("kvt_nccl_comm_init", ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), _i32, _i32, _vp)
kvt_nccl_comm_destroy = _sig("kvt_nccl_comm_destroy", ctypes.c_int, _vp)
kvt_lse_allgather_merge = _sig("kvt_lse_allgather_merge", ctypes.c_int, _vp, _i32, _vp, _i64, _i32, ctypes.c_double,
                               _vp, _vp, _vp, _vp)
kvt_live_chunks = _sig("kvt_live_chunks", ctypes.c_int, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp)
kvt_attn_gqa_scratch_bytes = _sig("kvt_attn_gqa_scratch_bytes", _sz, _i64, _i32, _i64)
kvt_sparse_decode_attn_gqa = _sig("kvt_sparse_decode_attn_gqa", ctypes.c_int, _vp, _i64, _i64, _i32, _i32, _i64, _vp,
                                  _vp, _vp, _i64, ctypes.c_double, _vp, _vp, _sz, _vp, _vp, _vp)
kvt_tier_ctl_bytes = _sig("kvt_tier_ctl_bytes", _sz)
kvt_tier_layer = _sig("kvt_tier_layer", ctypes.c_int, ctypes.POINTER(KvtTierArgs), _vp)
kvt_tier_read_ctl = _sig("kvt_tier_read_ctl", ctypes.c_int, _vp, _vp, _vp)
kvt_sparse_decode_attn_paged = _sig("kvt_sparse_decode_attn_paged", ctypes.c_int, _vp, _vp, _i64, _i32, _i64, _i32,
                                    _vp, _vp, _vp, _i64, ctypes.c_double, _i32, _vp, _vp, _vp, _vp)
kvt_debug_select_phases = _sig("kvt_debug_select_phases", ctypes.c_int, _vp)
kvt_attn_lse = _sig("kvt_attn_lse", ctypes.c_int, _vp, _i64, _vp, _vp)
kvt_lse_merge = _sig("kvt_lse_merge", ctypes.c_int, _vp, _i32, _i64, _i32, ctypes.c_double, _vp, _vp, _vp)
kvt_kv_quant = _sig("kvt_kv_quant", ctypes.c_int, _vp, _i32, _i64, _i64, _i64, _i64, _i32, _vp, _i64, _vp)
kvt_i4_row_bytes = _sig("kvt_i4_row_bytes", ctypes.c_int, _i32)
kvt_i4_recip_check = _sig("kvt_i4_recip_check", ctypes.c_int, _vp, _vp)
kvt_kv_dequant = _sig("kvt_kv_dequant", ctypes.c_int, _vp, _i64, _i64, _i64, _i64, _i32, _vp, _i32, _i64, _vp)
kvt_layer_workspace_bytes = _sig("kvt_layer_workspace_bytes", _sz, _i64, _i64, _i64, _i32)
kvt_select_attend = _sig("kvt_select_attend", ctypes.c_int, ctypes.POINTER(KvtLayerArgs), _vp, _sz, _vp)
_f32 = ctypes.c_float
kvt_synth_layer = _sig("kvt_synth_layer", ctypes.c_int, _vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _i32, _f32,
                       _f32, _f32, _f32, _f32, _i32, _vp)

EXPORTED = [
    "kvt_version", "kvt_status_string", "kvt_last_error", "kvt_abstract_build", "kvt_abstract_spans",
    "kvt_chunk_bounds", "kvt_token_scores", "kvt_select_plan", "kvt_cand_score", "kvt_topk_select",
    "kvt_topk_select_runs",
    "kvt_runs_scan", "kvt_attn_workspace_bytes", "kvt_sparse_decode_attn", "kvt_layer_workspace_bytes",
    "kvt_select_attend", "kvt_kv_quant", "kvt_i4_row_bytes", "kvt_i4_recip_check", "kvt_select_plan2", "kvt_cand_score_f32",
    "kvt_topk_select_band", "kvt_kv_dequant", "kvt_chunk_bounds_fast", "kvt_attn_lse", "kvt_lse_merge", "kvt_set_kv_group", "kvt_i4_qprep_bytes", "kvt_i4_qprep", "kvt_cand_score_i4mma",
    "kvt_synth_layer", "kvt_select_plan_group", "kvt_set_cand_group", "kvt_debug_select_phases",
    "kvt_abstract_merge", "kvt_live_chunks", "kvt_kv_append", "kvt_nccl_available", "kvt_nccl_unique_id", "kvt_nccl_comm_init",
    "kvt_nccl_comm_destroy", "kvt_lse_allgather_merge", "kvt_attn_gqa_scratch_bytes", "kvt_sparse_decode_attn_gqa", "kvt_tier_ctl_bytes", "kvt_tier_layer", "kvt_tier_read_ctl", "kvt_sparse_decode_attn_paged",
]


class KvtCudaError(RuntimeError):
    pass


def check(status: int, what: str = "") -> None:
    """Map a kvt_status onto the reference's exception types."""
    if status == OK:
        return
    msg = f"{what}: {kvt_status_string(status).decode()}"
    if status == ERR_CUDA:
        raise KvtCudaError(f"{msg} ({kvt_last_error().decode()})")
    if status == ERR_COLD:
        raise RuntimeError(msg)
    if status in (ERR_SHAPE, ERR_K, ERR_ARG, ERR_DTYPE):
        raise ValueError(msg)
    raise RuntimeError(msg)


def handle() -> ctypes.CDLL:
    return _L
