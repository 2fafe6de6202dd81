"""Canonical (JSON-comparable) form of one scheduling-step result."""

import hashlib
import json

import numpy as np

STATE_DTYPES = dict(phase=np.uint8, flags=np.uint8, level=np.uint8, promos=np.uint8,
                    wait_since=np.float64, ready_since=np.float64, context=np.int32,
                    kv=np.int32, rem_decode=np.int32, preempt=np.int32, served=np.int64)


def state_sha(state):
    return {k: hashlib.sha256(np.asarray(state[k], dtype=t).tobytes()).hexdigest()
            for k, t in STATE_DTYPES.items()}


def canon(out):
    """Oracle/device step output -> the golden JSON layout."""
    d = {k: v for k, v in out.items() if k != "state"}
    if "state" in out:
        d["state_sha256"] = state_sha(out["state"])
    return json.loads(json.dumps(d, default=_conv))


def _conv(o):
    if isinstance(o, (np.integer,)):
        return int(o)
    if isinstance(o, (np.floating,)):
        return float(o)
    if isinstance(o, (np.bool_,)):
        return bool(o)
    if isinstance(o, np.ndarray):
        return o.tolist()
    raise TypeError(type(o))


def digest(obj, limit=2048):
    """Canonical form with every list longer than `limit` replaced by its
    length and the SHA-256 of its compact JSON (large frozen fixtures)."""
    if isinstance(obj, dict):
        return {k: digest(v, limit) for k, v in obj.items()}
    if isinstance(obj, list):
        if len(obj) > limit:
            h = hashlib.sha256(json.dumps(obj, separators=(",", ":")).encode()).hexdigest()
            return {"len": len(obj), "sha256": h}
        return [digest(v, limit) for v in obj]
    return obj
