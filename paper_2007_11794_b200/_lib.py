"""ctypes binding of ``libotflm_b200.so`` (the C-ABI in include/otflm_b200.h).

The library is built in-tree (``paper_2007_11794_b200/libotflm_b200.so``,
``make -C paper_2007_11794_b200/csrc``).  There is no fallback: if the
library or a CUDA device is missing, every product entry point raises.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libotflm_b200.so"
CSRC = _PKG / "csrc"

OK = 0
ERR_VALUE, ERR_UNKNOWN_INDEX, ERR_TABLE_FULL, ERR_NO_PATH, ERR_KEY = -1, -2, -3, -4, -5
ERR_NOMEM, ERR_CYCLE, ERR_PACK, ERR_CUDA, ERR_HASH = -6, -7, -8, -9, -10

PREC = {"fp64": 0, "tf32x3": 1, "bf16": 2, "tf32": 3, "exact": 4}
PROFILE_CATEGORIES = ("expand", "hs", "advance", "assign", "final", "misc", "stream")
SCHED = {"level": 0, "stream": 1, "stream1": 2}


class UnknownIndexError(KeyError):
    """Index was never assigned (reference context_table.py:36-37)."""


class TableFullError(RuntimeError):
    """Index space exhausted (reference context_table.py:40-41)."""


class PackOverflowError(ValueError):
    """An index does not fit its bit budget (reference codec.py:31-32)."""


class LatticeCycleError(ValueError):
    pass


class NativeError(RuntimeError):
    pass


_EXC = {
    ERR_VALUE: ValueError, ERR_UNKNOWN_INDEX: UnknownIndexError, ERR_TABLE_FULL: TableFullError,
    ERR_NO_PATH: ValueError, ERR_KEY: KeyError, ERR_NOMEM: MemoryError, ERR_CYCLE: LatticeCycleError,
    ERR_PACK: PackOverflowError, ERR_CUDA: NativeError, ERR_HASH: NativeError,
}


class ModelDesc(C.Structure):
    _fields_ = [("hidden_size", C.c_int32), ("vocab_size", C.c_int32), ("maxent_order", C.c_int32),
                ("maxent_size", C.c_uint64), ("hash_seed", C.c_uint64),
                ("input_weights", C.c_void_p), ("recurrent_weights", C.c_void_p),
                ("node_vectors", C.c_void_p), ("maxent_table", C.c_void_p),
                ("path_nodes", C.c_void_p), ("path_signs", C.c_void_p),
                ("path_offsets", C.c_void_p), ("n_path", C.c_int64)]


class NgramDesc(C.Structure):
    _fields_ = [("order", C.c_int32), ("vocab_size", C.c_int32), ("bos_id", C.c_int32),
                ("n_probs", C.c_int64), ("prob_keys", C.c_void_p), ("prob_lens", C.c_void_p),
                ("prob_vals", C.c_void_p), ("n_backoffs", C.c_int64), ("bow_keys", C.c_void_p),
                ("bow_lens", C.c_void_p), ("bow_vals", C.c_void_p)]


class StreamConfig(C.Structure):
    _fields_ = [("n_streams", C.c_int32), ("cache_enabled", C.c_int32),
                ("max_contexts", C.c_int64), ("cache_slots", C.c_int64),
                ("arena_rows", C.c_int64)]


class LatticeBatch(C.Structure):
    _fields_ = [("n_utt", C.c_int32), ("n_nodes", C.c_void_p), ("start", C.c_void_p),
                ("arc_off", C.c_void_p), ("arc_src", C.c_void_p), ("arc_dst", C.c_void_p),
                ("arc_word", C.c_void_p), ("arc_ac", C.c_void_p), ("arc_slm", C.c_void_p),
                ("final_off", C.c_void_p), ("finals", C.c_void_p), ("stream_ids", C.c_void_p)]


class HypBatch(C.Structure):
    _fields_ = [("n_lists", C.c_int32), ("list_off", C.c_void_p), ("hyp_off", C.c_void_p),
                ("words", C.c_void_p), ("acoustic", C.c_void_p)]


class DecodeResult(C.Structure):
    _fields_ = [("path_len", C.c_void_p), ("path_arcs", C.c_void_p), ("max_path", C.c_int32),
                ("combined", C.c_void_p), ("acoustic", C.c_void_p), ("lm", C.c_void_p),
                ("end_ctx", C.c_void_p), ("expansions", C.c_void_p), ("status", C.c_void_p)]


# function name -> (restype, argtypes)
_P = C.c_void_p
_SIGS = {
    "otflm_model_create": (C.c_int, [C.POINTER(ModelDesc), C.c_int32, C.POINTER(C.c_void_p)]),
    "otflm_model_destroy": (C.c_int, [_P]),
    "otflm_model_info": (C.c_int, [_P, _P]),
    "otflm_ngram_create": (C.c_int, [C.POINTER(NgramDesc), _P, C.POINTER(C.c_void_p)]),
    "otflm_ngram_destroy": (C.c_int, [_P]),
    "otflm_ngram_logprob_batch": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P]),
    "otflm_feature_index_batch": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, _P, _P, _P, _P, _P]),
    "otflm_word_logprob_batch": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, _P, _P]),
    "otflm_word_logprob_batch2": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, _P, C.c_int32, _P]),
    "otflm_word_logprob_paths": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "otflm_advance_hidden_batch": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, C.c_int32, _P]),
    "otflm_advance_hidden_rows": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, C.c_int32, _P]),
    "otflm_all_word_logprobs": (C.c_int, [_P, _P, _P, C.c_int32, _P, _P]),
    "otflm_all_word_logprobs_batch": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, C.c_int32, _P]),
    "otflm_streams_create": (C.c_int, [_P, C.POINTER(StreamConfig), C.POINTER(C.c_void_p)]),
    "otflm_streams_destroy": (C.c_int, [_P]),
    "otflm_streams_reset": (C.c_int, [_P, C.c_int32, _P]),
    "otflm_streams_stats": (C.c_int, [_P, _P, _P]),
    "otflm_streams_context": (C.c_int, [_P, C.c_int32, C.c_uint32, _P, _P, _P, _P]),
    "otflm_streams_encode": (C.c_int, [_P, C.c_int32, C.c_int64, _P, _P, _P, _P, _P]),
    "otflm_streams_cache_get": (C.c_int, [_P, C.c_int32, C.c_int64, _P, _P, _P, _P, _P, _P]),
    "otflm_streams_cache_put": (C.c_int, [_P, C.c_int32, C.c_int64, _P, _P, _P, _P, _P]),
    "otflm_streams_roll_stats": (C.c_int, [_P, C.c_int32, _P]),
    "otflm_streams_cache_clear": (C.c_int, [_P, C.c_int32, _P]),
    "otflm_streams_set_capacity": (C.c_int, [_P, C.c_int64, _P]),
    "otflm_streams_cache_stats": (C.c_int, [_P, _P, _P]),
    "otflm_rnnlm_prob_batch": (C.c_int, [_P, C.c_int64, _P, _P, _P, C.c_int32, _P, _P, _P, _P]),
    "otflm_plan_create": (C.c_int, [_P, C.POINTER(LatticeBatch), C.c_int64, C.POINTER(C.c_void_p), _P]),
    "otflm_plan_destroy": (C.c_int, [_P]),
    "otflm_plan_refresh": (C.c_int, [_P, C.POINTER(LatticeBatch), C.POINTER(C.c_int32), _P]),
    "otflm_plan_info": (C.c_int, [_P, _P]),
    "otflm_decode_run": (C.c_int, [_P, _P, C.c_double, C.c_int32, C.c_int32, _P]),
    "otflm_decode_fetch": (C.c_int, [_P, C.POINTER(DecodeResult), _P]),
    "otflm_decode": (C.c_int, [_P, _P, C.POINTER(LatticeBatch), C.c_double, C.c_int64, C.c_int32,
                               C.POINTER(DecodeResult), _P]),
    "otflm_plan_counters": (C.c_int, [_P, _P, _P]),
    "otflm_decode_profile": (C.c_int, [_P, _P, C.c_double, C.c_int32, _P, _P, _P]),
    "otflm_plan_set_arena": (C.c_int, [_P, C.c_uint32, C.c_uint32]),
    "otflm_plan_set_lattice_out": (C.c_int, [_P, C.c_int32]),
    "otflm_decode_lattice_fetch": (C.c_int, [_P, _P, _P, C.c_int64, _P]),
    "otflm_plan_set_schedule": (C.c_int, [_P, C.c_int32]),
    "otflm_plan_phase_ns": (C.c_int, [_P, _P, _P]),
    "otflm_plan_wide": (C.c_int, [_P, C.POINTER(C.c_int32)]),
    "otflm_schedule_supported": (C.c_int, [_P, C.c_int32, C.c_int32]),
    "otflm_group_create": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_void_p)]),
    "otflm_group_destroy": (C.c_int, [_P]),
    "otflm_group_run": (C.c_int, [_P, _P, C.c_double, C.c_int32, _P]),
    "otflm_group_profile": (C.c_int, [_P, _P, C.c_double, C.c_int32, _P, _P, _P]),
    "otflm_last_launch_count": (C.c_int64, []),
    "otflm_nbest_create": (C.c_int, [C.POINTER(LatticeBatch), C.c_int32, C.c_double, C.c_int32,
                                     C.POINTER(C.c_void_p)]),
    "otflm_nbest_sizes": (C.c_int, [_P, _P, _P]),
    "otflm_nbest_copy": (C.c_int, [_P, _P, _P, _P, _P]),
    "otflm_nbest_destroy": (C.c_int, [_P]),
    "otflm_twopass_create": (C.c_int, [_P, _P, C.POINTER(HypBatch), C.c_int32,
                                       C.POINTER(C.c_void_p), _P]),
    "otflm_twopass_info": (C.c_int, [_P, _P]),
    "otflm_twopass_run": (C.c_int, [_P, C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_int32,
                                    _P]),
    "otflm_twopass_fetch": (C.c_int, [_P, _P, _P, _P, _P]),
    "otflm_twopass_destroy": (C.c_int, [_P]),
    "otflm_error_string": (C.c_char_p, [C.c_int32]),
    "otflm_last_error_detail": (C.c_char_p, []),
}

EXPORTS = tuple(_SIGS)

_lib = None


def build(force: bool = False) -> Path:
    """Compile libotflm_b200.so for sm_100a with the committed Makefile."""
    if force or not LIB_PATH.exists() or any(
            p.stat().st_mtime > LIB_PATH.stat().st_mtime
            for p in list(CSRC.glob("*.cu*")) + [_PKG.parent / "include" / "otflm_b200.h"]):
        subprocess.run(["make", "-s", "-C", str(CSRC)], check=True)
    return LIB_PATH


def load(allow_build: bool = False):
    """Load (never silently replace) the native library."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            if allow_build:
                build()
            else:
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `make -C {CSRC}` "
                    "(there is no CPU fallback for the product path)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != OK:
        L = load()
        msg = L.otflm_error_string(rc).decode()
        detail = L.otflm_last_error_detail().decode()
        raise _EXC.get(rc, NativeError)(f"{what}: {msg}" + (f" ({detail})" if detail else ""))
