"""S5 on the B200: paged KV block manager + HBM <-> pinned-host KV tier.

The reference ``KvPool`` (agentsched/engine.py:116-221) counts blocks; this
gives every block a concrete ID (policy: oracle/block_ids.py) and moves the
bytes.  ``KvBlockManager`` attaches to an existing ``MarsEngine`` context:
once initialised, every engine step applies its own journal (expired pins in
rank order, then the plan's alloc/evict ops) to the block tables on the
device, and ``apply`` replays any other pool op stream in order (the
``KvPool.observer`` callbacks, engine.py:129-143).

Llama-3-8B geometry (the sweep of BASELINE configs[3]): 32 layers x {K, V} x
8 KV heads x 128 dims x bf16 = 128 KiB per token, 2 MiB per 16-token block,
stored layer-major on the device (32 pieces of 64 KiB per block, vLLM style)
and block-contiguous in the host tier.
"""

from __future__ import annotations

import ctypes as C
from typing import Iterable, List, Optional, Tuple

import numpy as np

from . import _native as N

LLAMA3_8B_BLOCK_BYTES = 32 * 2 * 8 * 128 * 2 * 16   # 2 MiB
LLAMA3_8B_LAYERS = 32

METHOD_COPY_ENGINE, METHOD_SM = 0, 1


class KvBlockManager:
    def __init__(self, engine, total_blocks: int, max_blocks_per_row: int = 16384,
                 block_bytes: int = 0, layers: int = 1, host_blocks: int = 0) -> None:
        self.eng = engine
        self.lib = engine.lib
        kc = N.MarsKvConfig(total_blocks=int(total_blocks),
                            max_blocks_per_row=int(max_blocks_per_row),
                            block_bytes=int(block_bytes), layers=int(layers),
                            host_blocks=int(host_blocks))
        self._check(self.lib.mars_kv_init(engine.ctx, C.byref(kc)))
        self.total_blocks = int(total_blocks)
        self.block_bytes = int(block_bytes)
        self.layers = int(layers)
        self.host_blocks = int(host_blocks)

    def _check(self, rc: int) -> None:
        N.check(rc, self.eng.ctx)

    def apply(self, ops: Iterable[Tuple[int, int, int]]) -> None:
        """Ordered (op, row, n) stream; op in KV_ALLOC / KV_FREE (n = -1: all) / PIN / UNPIN."""
        ops = list(ops)
        if not ops:
            return
        op = np.array([o for o, _, _ in ops], np.uint8)
        row = np.array([r for _, r, _ in ops], np.uint32)
        n = np.array([k for _, _, k in ops], np.int32)
        self._check(self.lib.mars_kv_apply(self.eng.ctx, len(ops), op.ctypes.data_as(C.c_void_p),
                                           row.ctypes.data_as(C.c_void_p),
                                           n.ctypes.data_as(C.c_void_p)))

    def bulk_alloc(self, rows, counts) -> None:
        """Initial tables from a fresh pool: rows[i] (distinct) gets the next
        counts[i] never-used IDs, as sequential allocs in list order would."""
        r = np.ascontiguousarray(rows, np.uint32)
        c = np.ascontiguousarray(counts, np.int32)
        self._check(self.lib.mars_kv_bulk_alloc(self.eng.ctx, len(r), r.ctypes.data_as(C.c_void_p),
                                                c.ctypes.data_as(C.c_void_p)))

    def load_snapshot_tables(self, snap) -> int:
        """Tables for every session of a snapshot that holds KV (a running
        session's held blocks, a pin's pinned blocks), rows in session-id
        (rank) order; returns the blocks handed out."""
        from .snapshot import F_PINNED
        c = snap.cols
        held = -(-c["kv"].astype(np.int64) // 16)
        blocks = np.where((c["flags"] & F_PINNED) != 0, c["pinned_blocks"], held)
        rows = np.nonzero(blocks > 0)[0]
        rows = rows[np.argsort(c["rank"][rows], kind="stable")]
        self.bulk_alloc(rows, blocks[rows])
        return int(blocks[rows].sum())

    def table(self, row: int) -> np.ndarray:
        n = C.c_int64()
        self._check(self.lib.mars_kv_table(self.eng.ctx, row, 0, None, C.byref(n)))
        out = np.zeros(n.value, np.uint32)
        if n.value:
            self._check(self.lib.mars_kv_table(self.eng.ctx, row, n.value,
                                               out.ctypes.data_as(C.c_void_p), C.byref(n)))
        return out

    def state(self, k: int = 0):
        top = np.zeros(max(k, 1), np.uint32)
        depth, fresh, status = C.c_int64(), C.c_int64(), C.c_int32()
        self._check(self.lib.mars_kv_state(self.eng.ctx, k, top.ctypes.data_as(C.c_void_p),
                                           C.byref(depth), C.byref(fresh), C.byref(status)))
        top = top[:k]
        return top[top != 0xFFFFFFFF], depth.value, fresh.value, status.value

    def free_count(self) -> int:
        _, depth, fresh, _ = self.state(0)
        return depth + (self.total_blocks - fresh)

    def evict(self, block_ids, slot0: int = 0, method: int = METHOD_COPY_ENGINE) -> None:
        ids = np.ascontiguousarray(block_ids, np.uint32)
        self._check(self.lib.mars_kv_evict(self.eng.ctx, len(ids), ids.ctypes.data_as(C.c_void_p),
                                           int(slot0), int(method)))

    def restore(self, block_ids, slot0: int = 0, method: int = METHOD_COPY_ENGINE) -> None:
        ids = np.ascontiguousarray(block_ids, np.uint32)
        self._check(self.lib.mars_kv_restore(self.eng.ctx, len(ids),
                                             ids.ctypes.data_as(C.c_void_p), int(slot0),
                                             int(method)))

    # -- the host tier driven by the step's decisions (mars_kv_capture ...) ----

    def capture(self, on: bool = True) -> None:
        """Record the IDs that running-session evictions and unpinned tool
        boundaries free during the engine's steps (for offload_captured)."""
        self._check(self.lib.mars_kv_capture(self.eng.ctx, int(bool(on))))

    def offload_captured(self, want_ids: bool = False):
        """Copies the captured blocks to the next host-ring slots:
        (n_blocks, first slot or -1, the IDs in slot order or None)."""
        n, s0 = C.c_int64(), C.c_int64()
        ids = np.zeros(self.total_blocks if want_ids else 1, np.uint32)
        self._check(self.lib.mars_kv_offload_captured(
            self.eng.ctx, C.byref(n), C.byref(s0), ids.ctypes.data_as(C.c_void_p) if want_ids
            else None, len(ids) if want_ids else 0))
        return n.value, s0.value, (ids[:n.value].copy() if want_ids else None)

    def offload_rows(self, rows, counts) -> int:
        """Whole tables of `rows` (counts[i] = row i's table length) to the
        host ring; row i lands at the returned slot + sum(counts[:i])."""
        r = np.ascontiguousarray(rows, np.int64)
        c = np.ascontiguousarray(counts, np.int32)
        s0 = C.c_int64()
        self._check(self.lib.mars_kv_offload_rows(self.eng.ctx, len(r), r.ctypes.data_as(C.c_void_p),
                                                  c.ctypes.data_as(C.c_void_p), C.byref(s0)))
        return s0.value

    def restore_rows(self, rows, counts, slots) -> None:
        """The rows' tables back from their host slots (slots[i] = row i's first)."""
        r = np.ascontiguousarray(rows, np.int64)
        c = np.ascontiguousarray(counts, np.int32)
        s = np.ascontiguousarray(slots, np.int64)
        self._check(self.lib.mars_kv_restore_rows(self.eng.ctx, len(r), r.ctypes.data_as(C.c_void_p),
                                                  c.ctypes.data_as(C.c_void_p),
                                                  s.ctypes.data_as(C.c_void_p)))

    def host_view(self) -> np.ndarray:
        """The pinned host tier as a uint8 array [host_blocks, block_bytes]."""
        h, d = C.c_void_p(), C.c_void_p()
        self._check(self.lib.mars_kv_host_ptr(self.eng.ctx, C.byref(h), C.byref(d)))
        n = self.host_blocks * self.block_bytes
        buf = (C.c_uint8 * n).from_address(h.value)
        return np.frombuffer(buf, np.uint8).reshape(self.host_blocks, self.block_bytes)

    def device_ptr(self) -> int:
        h, d = C.c_void_p(), C.c_void_p()
        self._check(self.lib.mars_kv_host_ptr(self.eng.ctx, C.byref(h), C.byref(d)))
        return d.value


def host_link_peak(engine, nbytes: int = 1 << 30, reps: int = 10):
    """Pinned cudaMemcpyAsync peak: (d2h, h2d, bidirectional) GB/s, best of reps."""
    d2h, h2d, bi = C.c_double(), C.c_double(), C.c_double()
    N.check(engine.lib.mars_host_link_peak(engine.ctx, int(nbytes), int(reps), C.byref(d2h),
                                           C.byref(h2d), C.byref(bi)), engine.ctx)
    return d2h.value, h2d.value, bi.value


# pool op names (KvPool.observer) -> block-manager ops
OBSERVER_OPS = {"alloc": N.KV_ALLOC, "free": N.KV_FREE, "pin": N.KV_PIN, "unpin": N.KV_UNPIN}
