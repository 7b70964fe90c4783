"""ctypes binding of the C-ABI in ``include/alaya.h`` (``libalaya_b200.so``).

The library is built in-tree (``paper_2504_10326_b200/csrc/Makefile``) and
loaded from this package directory. There is no fallback: if the library is
missing or no CUDA device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_NAME = "libalaya_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME
if os.environ.get("ALAYA_LIB_VARIANT"):  # diagnostics: an in-tree build variant (tools/variants.sh)
    LIB_PATH = Path(__file__).resolve().parent / "variants" / os.environ["ALAYA_LIB_VARIANT"] / LIB_NAME

ALAYA_OK = 0
ALAYA_ERR_ARG = 1
ALAYA_ERR_SHAPE = 2
ALAYA_ERR_NONFINITE = 3
ALAYA_ERR_CUDA = 4
ALAYA_ERR_WORKSPACE = 5
ALAYA_ERR_UNSUPPORTED = 6

ALAYA_F32 = 0
ALAYA_BF16 = 1

SCAN_AUTO = 0
SCAN_CUDA_CORE = 1
SCAN_TCGEN05 = 2

MAX_BATCH = 32  # include/alaya.h ALAYA_MAX_BATCH (kernel-parameter space: small batches launch fast)

# every symbol include/alaya.h declares (checked by tests/test_boundary.py)
EXPORTS = (
    "alaya_last_error", "alaya_version", "alaya_workspace_bytes", "alaya_dipr_attention",
    "alaya_dipr_attention_update",
    "alaya_scan", "alaya_attend", "alaya_sharded_step", "alaya_merge_exchanged", "alaya_merge_partials", "alaya_merge_states", "alaya_selected",
    "alaya_ws_status", "alaya_window_append", "alaya_block_bounds", "alaya_ws_block_stats",
    "alaya_ws_candidate_counts", "alaya_topk", "alaya_block_reps", "alaya_block_topk",
    "alaya_sparse_attention", "alaya_avdb_stat", "alaya_avdb_write", "alaya_avdb_staging_bytes",
    "alaya_avdb_load", "alaya_avdb_graph", "alaya_diprs", "alaya_diprs_workspace_bytes",
    "alaya_exch_bytes", "alaya_exch_alloc", "alaya_exch_open", "alaya_exch_close", "alaya_exch_free",
    "alaya_exch", "alaya_exch_slots", "alaya_debug_trace",
)


class AlayaSeq(ctypes.Structure):
    """``alaya_seq`` (include/alaya.h)."""

    _fields_ = [
        ("k", ctypes.c_void_p), ("v", ctypes.c_void_p),
        ("wk", ctypes.c_void_p), ("wv", ctypes.c_void_p),
        ("head_stride", ctypes.c_int64), ("w_head_stride", ctypes.c_int64),
        ("token_offset", ctypes.c_int64), ("prefix_len", ctypes.c_int64),
        ("n", ctypes.c_int32), ("w", ctypes.c_int32),
        ("bounds", ctypes.c_void_p), ("bounds_head_stride", ctypes.c_int64),
        ("d_w", ctypes.c_void_p),
    ]


class AlayaParams(ctypes.Structure):
    """``alaya_params`` (include/alaya.h)."""

    _fields_ = [
        ("n_query_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
        ("dim", ctypes.c_int32), ("dtype", ctypes.c_int32), ("beta", ctypes.c_float),
        ("win_initial", ctypes.c_int32), ("win_last", ctypes.c_int32),
        ("chunk", ctypes.c_int32), ("scan_kind", ctypes.c_int32),
        ("block_filter", ctypes.c_int32),
        ("d_call_seq", ctypes.c_void_p),
    ]


class AlayaBlockIndex(ctypes.Structure):
    """``alaya_block_index`` (include/alaya.h)."""

    _fields_ = [
        ("reps", ctypes.c_void_p), ("head_stride", ctypes.c_int64),
        ("n_tokens", ctypes.c_int64), ("n_blocks", ctypes.c_int32), ("r", ctypes.c_int32),
    ]


class AlayaAvdbInfo(ctypes.Structure):
    """``alaya_avdb_info`` (include/alaya.h)."""

    _fields_ = [
        ("dim", ctypes.c_uint32), ("element_width", ctypes.c_uint32),
        ("n_vectors", ctypes.c_uint64), ("n_data_blocks", ctypes.c_uint32),
        ("n_index_blocks", ctypes.c_uint32), ("n_tombstones", ctypes.c_uint32),
        ("pad_", ctypes.c_uint32), ("file_bytes", ctypes.c_uint64),
        ("directory_offset", ctypes.c_uint64), ("index_head", ctypes.c_uint64),
    ]


class AlayaGraph(ctypes.Structure):
    """``alaya_graph`` (include/alaya.h)."""

    _fields_ = [
        ("offsets", ctypes.c_void_p), ("nbrs", ctypes.c_void_p), ("entry", ctypes.c_void_p),
        ("offsets_head_stride", ctypes.c_int64), ("nbrs_head_stride", ctypes.c_int64),
        ("n_nodes", ctypes.c_int32), ("pad_", ctypes.c_int32),
    ]


class AlayaError(RuntimeError):
    pass


_lib = None


def load() -> ctypes.CDLL:
    """Load the library (no device calls). Raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise AlayaError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (or `make -C paper_2504_10326_b200/csrc -j`). There is no CPU fallback.")
    lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL | getattr(os, "RTLD_NOW", 2))
    P, S = ctypes.POINTER(AlayaParams), ctypes.POINTER(AlayaSeq)
    vp, i32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    lib.alaya_last_error.restype = ctypes.c_char_p
    lib.alaya_last_error.argtypes = []
    lib.alaya_version.restype = i32
    if hasattr(lib, "alaya_debug_trace"):  # (absent from older diagnostic build variants)
        lib.alaya_debug_trace.restype = i32
        lib.alaya_debug_trace.argtypes = [vp, ctypes.c_int64]
    lib.alaya_workspace_bytes.restype = sz
    lib.alaya_workspace_bytes.argtypes = [P, S, i32]
    lib.alaya_dipr_attention.restype = i32
    lib.alaya_dipr_attention.argtypes = [P, S, i32, vp, vp, vp, sz, vp]
    lib.alaya_dipr_attention_update.restype = i32
    lib.alaya_dipr_attention_update.argtypes = [P, S, i32, vp, vp, vp, vp, vp, sz, vp]
    lib.alaya_scan.restype = i32
    lib.alaya_scan.argtypes = [P, S, i32, vp, vp, vp, sz, vp]
    lib.alaya_sharded_step.restype = i32
    lib.alaya_sharded_step.argtypes = [P, S, i32, vp, vp, i32, i32, ctypes.c_int64, ctypes.c_uint64,
                                       ctypes.c_uint64, vp, vp, vp, sz, vp]
    lib.alaya_merge_exchanged.restype = i32
    lib.alaya_merge_exchanged.argtypes = [vp, i32, ctypes.c_int64, ctypes.c_uint64, i32, i32, vp, vp, vp,
                                          vp]
    lib.alaya_attend.restype = i32
    lib.alaya_attend.argtypes = [P, S, i32, vp, vp, vp, i32, vp, sz, vp]
    lib.alaya_merge_partials.restype = i32
    lib.alaya_merge_partials.argtypes = [vp, i32, i32, i32, vp, vp, vp]
    lib.alaya_merge_states.restype = i32
    lib.alaya_merge_states.argtypes = [vp, i32, i32, i32, vp, vp]
    lib.alaya_selected.restype = i32
    lib.alaya_selected.argtypes = [P, S, i32, vp, ctypes.c_int64, vp, vp, vp, sz, vp]
    lib.alaya_window_append.restype = i32
    lib.alaya_window_append.argtypes = [P, S, i32, vp, vp, vp]
    lib.alaya_block_bounds.restype = i32
    lib.alaya_block_bounds.argtypes = [vp, i32, i32, ctypes.c_int64, i32, i32, vp, ctypes.c_int64, vp]
    lib.alaya_ws_candidate_counts.restype = vp
    lib.alaya_ws_candidate_counts.argtypes = [P, S, i32, vp]
    lib.alaya_ws_block_stats.restype = vp
    lib.alaya_ws_block_stats.argtypes = [P, S, i32, vp]
    i64 = ctypes.c_int64
    lib.alaya_topk.restype = i32
    lib.alaya_topk.argtypes = [P, S, i32, vp, i32, vp, vp, i64, vp, vp, sz, vp]
    lib.alaya_block_reps.restype = i32
    lib.alaya_block_reps.argtypes = [vp, i32, i32, i64, i32, i32, i32, i32, vp, i64, vp]
    lib.alaya_block_topk.restype = i32
    lib.alaya_block_topk.argtypes = [P, S, ctypes.POINTER(AlayaBlockIndex), i32, i32, i32, vp, vp,
                                     i64, vp, vp, vp, vp]
    lib.alaya_sparse_attention.restype = i32
    lib.alaya_sparse_attention.argtypes = [P, S, i32, vp, vp, i64, vp, vp, vp, vp, vp]
    cp, cpp = ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p)
    lib.alaya_avdb_stat.restype = i32
    lib.alaya_avdb_stat.argtypes = [cp, ctypes.POINTER(AlayaAvdbInfo)]
    lib.alaya_avdb_write.restype = i32
    lib.alaya_avdb_write.argtypes = [cp, vp, i64, i32, i32]
    lib.alaya_avdb_staging_bytes.restype = sz
    lib.alaya_avdb_staging_bytes.argtypes = [cpp, i32]
    lib.alaya_avdb_load.restype = i32
    lib.alaya_avdb_load.argtypes = [cpp, i32, i64, i32, i32, vp, i64, vp, sz, vp]
    G = ctypes.POINTER(AlayaGraph)
    lib.alaya_avdb_graph.restype = i32
    lib.alaya_avdb_graph.argtypes = [cp, vp, vp, vp, vp, vp, vp]
    lib.alaya_diprs_workspace_bytes.restype = sz
    lib.alaya_diprs_workspace_bytes.argtypes = [P, S, G, i32]
    lib.alaya_diprs.restype = i32
    lib.alaya_diprs.argtypes = [P, S, G, i32, vp, i32, i32, vp, vp, i64, vp, vp, vp, sz, vp]
    lib.alaya_exch_bytes.restype = sz
    lib.alaya_exch_bytes.argtypes = [i32, i64]
    lib.alaya_exch_alloc.restype = i32
    lib.alaya_exch_alloc.argtypes = [sz, ctypes.POINTER(vp), vp]
    lib.alaya_exch_open.restype = i32
    lib.alaya_exch_open.argtypes = [vp, ctypes.POINTER(vp)]
    lib.alaya_exch_close.restype = i32
    lib.alaya_exch_close.argtypes = [vp]
    lib.alaya_exch_free.restype = i32
    lib.alaya_exch_free.argtypes = [vp]
    lib.alaya_exch.restype = i32
    lib.alaya_exch.argtypes = [ctypes.POINTER(vp), i32, i32, i64, i32, vp, i64, ctypes.c_uint64, vp, vp,
                               vp]
    lib.alaya_exch_slots.restype = vp
    lib.alaya_exch_slots.argtypes = [vp, i32, i64, i32, ctypes.c_uint64]
    lib.alaya_ws_status.restype = vp
    lib.alaya_ws_status.argtypes = [vp]
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == ALAYA_OK:
        return
    msg = load().alaya_last_error().decode(errors="replace")
    if rc in (ALAYA_ERR_ARG, ALAYA_ERR_SHAPE):
        raise ValueError(msg)
    if rc == ALAYA_ERR_NONFINITE:
        raise FloatingPointError(msg or "attention output is non-finite")
    if rc == ALAYA_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise AlayaError(f"alaya status {rc}: {msg}")
