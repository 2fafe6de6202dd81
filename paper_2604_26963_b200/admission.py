"""``balance_and_admit``: drop-in for ``agentsched.control.balance_and_admit``.

Same signature and mutation contract as the reference (control.py:166-208):
packs the queue (pack_queue, control.py:101-122), steps the AIMD window and
the triple clamp (control.py:130-163), admits the packed prefix, leaves the
residual in packed order in ``queue`` (mutated in place), emits one
``window_update`` event and folds it into the telemetry.  The packing,
median seed, window arithmetic and the admit/residual split run on the
device in one ``k_control`` launch (MARS_MODE_NO_ROWS: the one-CTA pack of a
small list or the grid LSD sort of a big one, update_window + the triple
clamp, the packed prefix and the residual list); the reference's sim binds
the function by import (sim.py:29), so the drop-in swaps
``agentsched.sim.balance_and_admit``.
"""

from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np

from . import _native as N
from .engine import MarsEngine
from .policy import config_from

_ADMIT_MODE = N.MODE_SKIP_EXPIRY | N.MODE_SKIP_PROBE | N.MODE_SKIP_REFRESH | N.MODE_NO_ROWS
_engines: Dict[tuple, MarsEngine] = {}


def _engine(controller, pressure, n: int, device: int = 0) -> MarsEngine:
    key = (device, tuple(getattr(controller, f) for f in (
        "w_min", "aimd_increase", "aimd_decrease", "control_interval_s", "initial_window",
        "cpu_oversubscription", "reserve_fraction", "long_session_fraction")),
        float(pressure.kv_low_watermark))
    eng = _engines.get(key)
    if eng is None or eng.max_queue < n:
        if eng is not None:
            eng.close()
        cap = max(1024, 1 << max(0, int(n - 1).bit_length()))
        eng = MarsEngine(max_rows=1, max_queue=cap, device=device,
                         config=config_from(pressure=pressure, controller=controller))
        eng._check(eng.lib.mars_set_rows(eng.ctx, 0))
        _engines[key] = eng
    return eng


def balance_and_admit(queue: List, state, telemetry, worker_slots: int, pressure, clock,
                      log=None, device: int = 0) -> List:
    """control.py:166-208 on the B200."""
    now = clock.now
    cfg = getattr(state, "config", state)
    n = len(queue)
    eng = _engine(cfg, pressure, n, device)
    req = np.fromiter((e.req_blocks for e in queue), np.int32, n)
    lng = np.fromiter((bool(e.is_long_session) for e in queue), np.uint8, n)
    if n and int(req.min()) < 1:
        raise N.ContractViolation("queue entry needs req_blocks >= 1")
    eng.set_queue(np.arange(n, dtype=np.uint32), req, lng)
    s = N.MarsScalars()
    s.total_blocks = max(1, int(telemetry.total_blocks))
    s.free_blocks = 0
    s.available_kv = int(telemetry.available_kv)
    s.kv_usage_ratio = float(telemetry.kv_usage_ratio)
    s.active_sessions = int(telemetry.active_sessions)
    s.queued_tools = int(telemetry.queued_tools)
    s.active_tools = int(telemetry.active_tools)
    s.cpu_overloaded = int(bool(telemetry.cpu_overloaded))
    s.kv_overloaded = int(bool(telemetry.kv_overloaded))
    eb = telemetry.ema_blocks_per_session
    s.has_ema_blocks = int(eb is not None)
    s.ema_blocks = float(eb) if eb is not None else 0.0
    seed = telemetry.blocks_seed
    s.has_blocks_seed = int(seed is not None)
    s.blocks_seed = float(seed) if seed is not None else 0.0
    s.w_adm = float(state.w_adm)
    s.last_update = float(state.last_update)
    s.queue_len = n
    eng.set_scalars(s)
    si = eng.step_in(now, True, 0, 0, worker_slots, _ADMIT_MODE)
    res = eng.step(si)
    if res.status:
        raise RuntimeError(f"device admission status {res.status}")
    out = eng.get_scalars()
    admitted_pos = res.admitted_rows.tolist()
    residual_pos = eng.get_queue().tolist()
    if telemetry.ema_blocks_per_session is None and telemetry.blocks_seed is None and queue:
        telemetry.blocks_seed = _median_value(out.blocks_seed, req)
    state.w_adm = float(out.w_adm)
    state.last_update = float(out.last_update)
    admitted = [queue[p] for p in admitted_pos]
    queue[:] = [queue[p] for p in residual_pos]
    if log is not None:
        log.emit(now, "window_update", None, w_adm=state.w_adm, limit=int(res.limit),
                 slots=int(res.slots), admitted=[e.call.session_id for e in admitted],
                 cpu_overloaded=telemetry.cpu_overloaded, kv_overloaded=telemetry.kv_overloaded)
        telemetry.record("window_update", {"w_adm": state.w_adm},
                         smoothing=pressure.ema_smoothing)
        telemetry.last_window_update = now
    return admitted


def _median_value(dev_value: float, req: np.ndarray):
    """statistics.median's return type: the element itself (int) for odd-length
    data, the float mean of the two middles otherwise.  The value is the
    device's; only the Python type is restored."""
    return int(dev_value) if len(req) % 2 == 1 else float(dev_value)
