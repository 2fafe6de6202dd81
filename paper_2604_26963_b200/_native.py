"""ctypes binding of ``libmars_b200.so`` (include/mars_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()``.  There is
no fallback: if the library or a CUDA device is missing, every entry point
raises -- the product path never silently runs on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmars_b200.so")

MARS_OK, MARS_ERR_CONTRACT, MARS_ERR_CUDA, MARS_ERR_CAPACITY, MARS_ERR_ARG = 0, 1, 2, 3, 4

i32, i64, u8, u32, f64 = C.c_int32, C.c_int64, C.c_uint8, C.c_uint32, C.c_double
P = C.POINTER


class MarsConfig(C.Structure):
    _fields_ = [
        ("block_size", i32), ("token_budget", i32), ("tick_duration_s", f64),
        ("num_levels", i32), ("max_promotions", i32), ("max_decode_slots", i32),
        ("window_size", i32), ("level_bounds", i64 * 4), ("level_quotas", i64 * 4),
        ("promotion_wait_s", f64), ("deadline_slack", f64), ("max_pin_horizon_s", f64),
        ("pressure_weight_clip", f64), ("cpu_high_fraction", f64), ("cpu_low_fraction", f64),
        ("kv_high_watermark", f64), ("kv_low_watermark", f64), ("hysteresis_window", i32),
        ("ema_smoothing", f64), ("initial_tool_estimate_s", f64), ("w_min", i32),
        ("aimd_increase", f64), ("aimd_decrease", f64), ("control_interval_s", f64),
        ("initial_window", f64), ("cpu_oversubscription", f64), ("reserve_fraction", f64),
        ("long_session_fraction", f64), ("enable_coordinator", i32), ("enable_coscheduler", i32),
        ("policy", i32), ("ttl_seconds", f64), ("ttl_multiplier", f64),
    ]


# mars_config.policy (POLICY_KINDS, baselines.py:48)
POLICY_CODES = {"mars": 0, "fcfs": 1, "program_priority": 2, "static_ttl": 3, "dynamic_ttl": 4}


class MarsCols(C.Structure):
    _fields_ = [
        ("phase", P(u8)), ("flags", P(u8)), ("level", P(u8)), ("promos", P(u8)),
        ("plevel", P(u8)), ("ready_since", P(f64)), ("wait_since", P(f64)),
        ("deadline", P(f64)), ("arrival", P(f64)), ("context", P(i32)), ("kv", P(i32)),
        ("rem_decode", P(i32)), ("pinned_blocks", P(i32)), ("req_blocks", P(i32)),
        ("r0_prefill", P(i32)), ("r0_decode", P(i32)), ("preempt", P(i32)),
        ("served", P(i64)), ("rank", P(u32)), ("rounds_left", P(i32)),
    ]


# snapshot column name -> MarsCols field
COL_FIELDS = {
    "phase": "phase", "flags": "flags", "level": "level", "promos": "promos",
    "plevel": "plevel", "ready_since": "ready_since", "wait_since": "wait_since",
    "deadline": "deadline", "arrival": "arrival", "context": "context", "kv": "kv",
    "rem_decode": "rem_decode", "pinned_blocks": "pinned_blocks", "req_blocks": "req_blocks",
    "r0_prefill": "r0_prefill", "r0_decode": "r0_decode", "preempt": "preempt",
    "served": "served", "rank": "rank", "rounds_left": "rounds_left",
}


class MarsScalars(C.Structure):
    _fields_ = [
        ("total_blocks", i64), ("free_blocks", i64), ("w_adm", f64), ("last_update", f64),
        ("cpu_overloaded", i32), ("kv_overloaded", i32), ("cpu_high_streak", i32),
        ("cpu_low_streak", i32), ("kv_high_streak", i32), ("kv_low_streak", i32),
        ("has_ema_tool", i32), ("has_ema_blocks", i32), ("has_blocks_seed", i32),
        ("ema_tool", f64), ("ema_blocks", f64), ("blocks_seed", f64), ("last_w_adm", f64),
        ("last_window_update", f64), ("has_last_w_adm", i32), ("available_kv", i64),
        ("kv_usage_ratio", f64), ("active_sessions", i64), ("active_tools", i32),
        ("queued_tools", i32), ("queue_len", i64),
    ]


class MarsKvConfig(C.Structure):
    _fields_ = [("total_blocks", i64), ("max_blocks_per_row", i32), ("block_bytes", i64),
                ("layers", i32), ("host_blocks", i64)]


KV_ALLOC, KV_FREE, KV_PIN, KV_UNPIN = 1, 2, 3, 4


class MarsStepIn(C.Structure):
    _fields_ = [("now", f64), ("control_due", i32), ("active_tools", i32),
                ("queued_tools", i32), ("worker_slots", i32), ("mode", i32)]


MODE_SKIP_EXPIRY, MODE_SKIP_PROBE, MODE_SKIP_REFRESH, MODE_NO_ROWS = 1, 2, 4, 8
MODE_SERVICE, MODE_FINISH_RETENTION, MODE_RANK_ORDERED, MODE_SHARDED = 16, 32, 64, 128
MODE_ADVANCE = 256
XC_N = 8


class MarsStepOut(C.Structure):
    _fields_ = [
        ("status", i32), ("n_expired", i32), ("n_admitted", i32), ("n_window", i32),
        ("n_decode", i32), ("n_prefill", i32), ("n_evict", i32), ("n_journal", i32),
        ("n_retention", i32), ("n_ready", i32), ("n_promoted", i32), ("pack_mode", i32),
        ("total_tokens", i64), ("free_after_expiry", i64), ("free_blocks", i64),
        ("limit", i64), ("slots", i64),
        ("expired_rows", P(u32)), ("expired_blocks", P(i32)), ("admitted_rows", P(u32)),
        ("window_rows", P(u32)), ("decode_rows", P(u32)), ("prefill_rows", P(u32)),
        ("prefill_grants", P(i32)), ("evict_rows", P(u32)), ("evict_kind", P(u8)),
        ("evict_blocks", P(i32)), ("journal_op", P(u8)), ("journal_row", P(u32)),
        ("journal_n", P(i32)), ("ret_rows", P(u32)), ("ret_pin", P(u8)),
        ("ret_benefit", P(f64)), ("ret_cost", P(f64)), ("ret_deadline", P(f64)),
        ("decode_level", P(u8)), ("prefill_level", P(u8)), ("n_finish", i32),
        ("fin_rows", P(u32)), ("fin_pin", P(u8)), ("fin_benefit", P(f64)),
        ("fin_cost", P(f64)), ("fin_deadline", P(f64)),
        ("n_window_cand", i32), ("n_victim_cand", i32), ("walk_slow", i32),
        ("sort_path", i32), ("n_round_end", i32), ("n_done", i32),
        ("end_rows", P(u32)), ("end_kind", P(u8)),
        ("end_blocks", P(i32)), ("end_pin", P(u8)), ("end_benefit", P(f64)),
        ("end_cost", P(f64)), ("end_deadline", P(f64)), ("prefill_done", P(u8)),
        ("n_fullscan", i32), ("ref_flags", i32), ("ref_rounds", i32),
        ("n_window_ref", i32), ("n_victim_ref", i32), ("plan_pre_charge", P(i64)),
    ]


_SIGS = {
    "mars_abi_version": (i32, []),
    "mars_config_default": (None, [P(MarsConfig)]),
    "mars_create": (i32, [P(MarsConfig), C.c_int, i64, i64, P(C.c_void_p)]),
    "mars_destroy": (i32, [C.c_void_p]),
    "mars_last_error": (C.c_char_p, [C.c_void_p]),
    "mars_set_stream": (i32, [C.c_void_p, C.c_void_p]),
    "mars_set_rows": (i32, [C.c_void_p, i64]),
    "mars_upsert_rows": (i32, [C.c_void_p, i64, C.c_void_p, P(MarsCols)]),
    "mars_input_arena": (i32, [C.c_void_p, P(C.c_void_p), P(i64), P(MarsCols)]),
    "mars_upsert_arena": (i32, [C.c_void_p, i64, C.c_uint64]),
    "mars_read_rows": (i32, [C.c_void_p, i64, C.c_void_p, P(MarsCols)]),
    "mars_set_queue": (i32, [C.c_void_p, i64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mars_get_queue": (i32, [C.c_void_p, i64, C.c_void_p, P(i64)]),
    "mars_queue_append": (i32, [C.c_void_p, i64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mars_on_admit": (i32, [C.c_void_p, i64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mars_expired_pins": (i32, [C.c_void_p, f64, i64, C.c_void_p, P(i64)]),
    "mars_on_service": (i32, [C.c_void_p, i64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mars_set_scalars": (i32, [C.c_void_p, P(MarsScalars)]),
    "mars_get_scalars": (i32, [C.c_void_p, P(MarsScalars)]),
    "mars_step": (i32, [C.c_void_p, P(MarsStepIn), P(MarsStepOut)]),
    "mars_step_enqueue": (i32, [C.c_void_p, P(MarsStepIn)]),
    "mars_step_fetch": (i32, [C.c_void_p, P(MarsStepOut)]),
    "mars_set_graph": (i32, [C.c_void_p, C.c_int]),
    "mars_set_config": (i32, [C.c_void_p, C.c_void_p]),
    "mars_sync": (i32, [C.c_void_p]),
    "mars_shard_init": (i32, [C.c_void_p, C.c_int, C.c_int]),
    "mars_shard_buffers": (i32, [C.c_void_p, P(C.c_void_p), P(C.c_void_p), P(C.c_void_p),
                                 P(i64)]),
    "mars_set_queue_gpos": (i32, [C.c_void_p, i64, C.c_void_p]),
    "mars_get_queue_gpos": (i32, [C.c_void_p, i64, C.c_void_p, P(i64)]),
    "mars_step_phase": (i32, [C.c_void_p, P(MarsStepIn), C.c_int]),
    "mars_kv_init": (i32, [C.c_void_p, C.c_void_p]),
    "mars_kv_apply": (i32, [C.c_void_p, i64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mars_kv_table": (i32, [C.c_void_p, u32, i64, C.c_void_p, P(i64)]),
    "mars_kv_bulk_alloc": (i32, [C.c_void_p, i64, C.c_void_p, C.c_void_p]),
    "mars_kv_state": (i32, [C.c_void_p, i64, C.c_void_p, P(i64), P(i64), P(i32)]),
    "mars_kv_evict": (i32, [C.c_void_p, i64, C.c_void_p, i64, C.c_int]),
    "mars_kv_restore": (i32, [C.c_void_p, i64, C.c_void_p, i64, C.c_int]),
    "mars_kv_host_ptr": (i32, [C.c_void_p, P(C.c_void_p), P(C.c_void_p)]),
    "mars_kv_capture": (i32, [C.c_void_p, C.c_int]),
    "mars_kv_offload_captured": (i32, [C.c_void_p, P(i64), P(i64), C.c_void_p, i64]),
    "mars_kv_offload_rows": (i32, [C.c_void_p, i64, C.c_void_p, C.c_void_p, P(i64)]),
    "mars_kv_restore_rows": (i32, [C.c_void_p, i64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mars_host_link_peak": (i32, [C.c_void_p, i64, C.c_int, P(f64), P(f64), P(f64)]),
    "mars_resume": (i32, [C.c_void_p, i64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                          C.c_void_p, f64, C.c_void_p]),
    "mars_output_arena": (i32, [C.c_void_p, P(C.c_void_p), P(i64)]),
    "mars_resume_rows": (i32, [C.c_void_p, i64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p]),
    "mars_retention_batch": (i32, [C.c_void_p, i64, C.c_void_p, C.c_void_p, i64, f64, f64, f64,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mars_checkpoint": (i32, [C.c_void_p]),
    "mars_restore": (i32, [C.c_void_p]),
    "mars_flush_l2": (i32, [C.c_void_p, i64]),
    "mars_last_launch_count": (i32, [C.c_void_p]),
    "mars_set_profiling": (i32, [C.c_void_p, C.c_int]),
    "mars_kernel_times": (i32, [C.c_void_p, P(C.c_float), C.c_int]),
}

KTIME_NAMES = ("k_scan", "k_expired_sort", "k_control", "k_walk", "k_pack", "k_kv_exp_free",
               "k_kv_apply_step")

EXPORTS = tuple(_SIGS)

_lib: Optional[C.CDLL] = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Loads the library (no GPU needed to load).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class ContractViolation(Exception):
    """A caller broke a documented precondition (agentsched/engine.py:30)."""


def check(rc: int, ctx=None) -> None:
    if rc == MARS_OK:
        return
    msg = ""
    if ctx is not None and _lib is not None:
        raw = _lib.mars_last_error(ctx)
        msg = raw.decode() if raw else ""
    if rc == MARS_ERR_CONTRACT:
        raise ContractViolation(msg)
    raise RuntimeError(f"libmars_b200 error {rc}: {msg}")
