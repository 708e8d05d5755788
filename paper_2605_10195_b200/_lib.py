"""ctypes binding of the C-ABI in include/spex.h.

The product library is ``paper_2605_10195_b200/lib/libspex_b200.so`` (built
in-tree for sm_100a by ``__graft_entry__.build()``). There is no CPU fallback:
loading fails loudly when the library is missing, and every run fails loudly
when no sm_100 device is present.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("SPEX_LIB_PATH", PKG_DIR / "lib" / "libspex_b200.so"))

MAX_TRACKED = 8


class Totals(ctypes.Structure):
    """spex_totals (RunTotals, executor.hpp:20-33)."""

    _fields_ = [
        ("makespan", ctypes.c_double),
        ("generated_tokens", ctypes.c_longlong),
        ("committed_tokens", ctypes.c_longlong),
        ("reused_tokens", ctypes.c_longlong),
        ("wasted_tokens", ctypes.c_longlong),
        ("hits", ctypes.c_longlong * (MAX_TRACKED + 1)),
        ("misses", ctypes.c_longlong * (MAX_TRACKED + 1)),
        ("queries", ctypes.c_int),
        ("correct_votes", ctypes.c_int),
        ("early_terminated", ctypes.c_int),
        ("pad_", ctypes.c_int),
    ]

    def as_dict(self) -> dict:
        return {
            "makespan": self.makespan,
            "generated_tokens": self.generated_tokens,
            "committed_tokens": self.committed_tokens,
            "reused_tokens": self.reused_tokens,
            "wasted_tokens": self.wasted_tokens,
            "hits": list(self.hits),
            "misses": list(self.misses),
            "queries": self.queries,
            "correct_votes": self.correct_votes,
            "early_terminated": self.early_terminated,
        }


class Stats(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_longlong),
        ("epochs", ctypes.c_longlong),
        ("reward_events", ctypes.c_longlong),
        ("decode_steps", ctypes.c_longlong),
        ("decode_rows", ctypes.c_longlong),
        ("log_records", ctypes.c_longlong),
        ("nodes", ctypes.c_longlong),
        ("device_ms", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class ModelStats(ctypes.Structure):
    _fields_ = [
        ("model_ms", ctypes.c_double),
        ("attn_ms", ctypes.c_double),
        ("attn_launches", ctypes.c_longlong),
        ("attn_alg_bytes", ctypes.c_double),
        ("decode_rows", ctypes.c_longlong),
        ("decode_steps", ctypes.c_longlong),
        ("prefill_rows", ctypes.c_longlong),
        ("prm_rows", ctypes.c_longlong),
        ("prm_thoughts", ctypes.c_longlong),
        ("policy_flops", ctypes.c_double),
        ("prm_flops", ctypes.c_double),
        ("launches", ctypes.c_longlong),
        ("gemm_calls", ctypes.c_longlong),
        ("control_ms", ctypes.c_double),
        ("step_ms", ctypes.c_double),
        ("streamed", ctypes.c_int),
        ("pad_", ctypes.c_int),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class DecodeOut(ctypes.Structure):
    _fields_ = [("q", ctypes.c_int), ("node", ctypes.c_uint32), ("pos", ctypes.c_int),
                ("argmax", ctypes.c_int), ("lse", ctypes.c_float), ("logit_sum", ctypes.c_float)]


class PrmOut(ctypes.Structure):
    _fields_ = [("q", ctypes.c_int), ("node", ctypes.c_uint32), ("score", ctypes.c_float), ("pad_", ctypes.c_int)]


class KvStats(ctypes.Structure):
    """spex_kv_stats (the paged tree-KV store of the last run)."""

    _fields_ = [(n, ctypes.c_longlong) for n in (
        "pages", "page_tokens", "root_pages", "peak_pages", "freed_pages", "live_pages_end", "allocated_pages",
        "fresh_pages", "page_table_entries")]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}


_EXPORTS = {
    "spex_last_error": ([], ctypes.c_char_p),
    "spex_free": ([ctypes.c_void_p], None),
    "spex_device_ok": ([], ctypes.c_int),
    "spex_canonical_config": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "spex_executor_create": (
        [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)],
        ctypes.c_int,
    ),
    "spex_executor_run": ([ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(Totals)], ctypes.c_int),
    "spex_executor_log": (
        [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)],
        ctypes.c_int,
    ),
    "spex_executor_stats": ([ctypes.c_void_p, ctypes.POINTER(Stats)], ctypes.c_int),
    "spex_frontier_step": (
        [ctypes.c_void_p, ctypes.c_longlong, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_void_p),
         ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "spex_executor_destroy": ([ctypes.c_void_p], None),
    "spex_run_batch": (
        [ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int, ctypes.c_char_p, ctypes.c_int,
         ctypes.POINTER(Totals), ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "spex_executor_query_finish": (
        [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "spex_executor_set_model": (
        [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int], ctypes.c_int),
    "spex_executor_set_shard": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "spex_split_outbox_bytes": ([ctypes.c_int, ctypes.c_int], ctypes.c_longlong),
    "spex_split_outbox_alloc": (
        [ctypes.c_int, ctypes.c_longlong, ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p], ctypes.c_int),
    "spex_split_outbox_open": ([ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "spex_split_outbox_close": ([ctypes.c_void_p], ctypes.c_int),
    "spex_split_outbox_free": ([ctypes.c_void_p], ctypes.c_int),
    "spex_executor_set_split": (
        [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), ctypes.c_longlong],
        ctypes.c_int),
    "spex_split_run": (
        [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
         ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "spex_executor_emulate_split": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "spex_executor_split_stats": (
        [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "spex_executor_model_stats": ([ctypes.c_void_p, ctypes.POINTER(ModelStats)], ctypes.c_int),
    "spex_executor_set_kv_pages": ([ctypes.c_void_p, ctypes.c_longlong], ctypes.c_int),
    "spex_policy_ucb_score": (
        [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), ctypes.c_int,
         ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "spex_policy_ucb_select": (
        [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
         ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_double,
         ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "spex_policy_rebase_widths": (
        [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), ctypes.c_int,
         ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "spex_content_token_len": (
        [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "spex_content_eval": (
        [ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
         ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double),
         ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "spex_engine_advance": (
        [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int),
         ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
         ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)],
        ctypes.c_int),
    "spex_engine_create": ([ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "spex_engine_destroy": ([ctypes.c_void_p], None),
    "spex_engine_add_stream": (
        [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_int, ctypes.c_double,
         ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_int), ctypes.c_int], ctypes.c_int),
    "spex_engine_cancel": ([ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "spex_engine_drop": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "spex_engine_step": (
        [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
         ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "spex_engine_done_tokens": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "spex_engine_stream_count": ([ctypes.c_void_p], ctypes.c_int),
    "spex_engine_active_count": ([ctypes.c_void_p], ctypes.c_int),
    "spex_engine_next_ready": ([ctypes.c_void_p], ctypes.c_double),
    "spex_termination_should_terminate": (
        [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int),
         ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_int)],
        ctypes.c_int),
    "spex_score_batch": (
        [ctypes.c_char_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64),
         ctypes.c_int, ctypes.POINTER(ctypes.c_float), ctypes.c_int], ctypes.c_int),
    "spex_budget_k_total": (
        [ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_int)],
        ctypes.c_int),
    "spex_budget_allocate": (
        [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), ctypes.c_int,
         ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "spex_executor_set_reward_source": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "spex_executor_query_wall_ms": (
        [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.POINTER(ctypes.c_int),
         ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "spex_executor_kv_stats": ([ctypes.c_void_p, ctypes.POINTER(KvStats)], ctypes.c_int),
    "spex_executor_decode_outputs": (
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.POINTER(ctypes.c_longlong)], ctypes.c_int),
    "spex_executor_prm_outputs": (
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.POINTER(ctypes.c_longlong)], ctypes.c_int),
    "spex_run_once": (
        [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.POINTER(Totals), ctypes.POINTER(ctypes.c_void_p)],
        ctypes.c_int,
    ),
}

TRACE_CB = ctypes.CFUNCTYPE(None, ctypes.c_char_p, ctypes.c_size_t, ctypes.c_void_p)
_EXPORTS["spex_run"] = ([ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p, TRACE_CB, ctypes.c_void_p,
                         ctypes.c_longlong, ctypes.POINTER(Totals)], ctypes.c_int)

_lib = None


def bind(path: str | os.PathLike) -> ctypes.CDLL:
    lib = ctypes.CDLL(str(path))
    for name, (args, res) in _EXPORTS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


def lib() -> ctypes.CDLL:
    """The product library. Raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        _lib = bind(LIB_PATH)
    return _lib
