"""Sharded MARS engine: one replica per GPU, global admission over NCCL.

Sessions are partitioned across GPUs as data-parallel engine replicas
(SURVEY.md §8(e)); each replica owns its rows, KV pool, token budget and
window, so S1, S2, S4 and S5 never leave the GPU.  The control plane is the
only exchange, once per step:

1. ``mars_step_phase(1)`` -- the replica's table scan; it leaves its probe
   counters ``[available_kv, total_blocks, active_sessions, queue_len]`` in
   the device buffer ``xc`` and its admission entries (wire format below) in
   ``xsend``;
2. ``all_reduce(sum)`` of ``xc`` and ``all_gather`` of ``xsend`` over NCCL
   (NVLink/NVSwitch), on the replica's stream;
3. ``mars_step_phase(2)`` -- pooled telemetry, refresh_pressure, one
   balance_and_admit over the union list (identical on every replica), the
   replica admits its own winners and keeps its own residual (new dense global
   positions), then the replica-local plan.

Wire format of one admission entry: ONE uint64, ``gpos << 32 | req << 1 |
is_long``; ``xsend[0]`` is the entry count.  The row stays home: only its
owner needs it, and entry k of the owner's list is word k of its block.
Semantics and oracle: ``oracle/multi.py``.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import numpy as np

from . import _native as N

COUNTERS = ("available_kv", "total_blocks", "active_sessions", "queue_len")


def interleaved_gpos(lengths):
    """Dense global list positions for per-replica lists merged round-robin
    (entry k of replica g precedes entry k of replica g+1 and entry k+1 of
    every replica): the arrival order of independently filled shards."""
    keys = sorted((k, g) for g, n in enumerate(lengths) for k in range(n))
    pos = {kg: i for i, kg in enumerate(keys)}
    return [[pos[(k, g)] for k in range(n)] for g, n in enumerate(lengths)]


XQ_NONE = 0xFFFFFFFF  # another replica's entry: its row is not sent


def encode_queue(gpos, req, is_long, cap: int) -> np.ndarray:
    """Host restatement of k_export_queue's wire format (1 + cap uint64)."""
    n = len(gpos)
    if n > cap:
        raise ValueError("queue larger than the exchange capacity")
    buf = np.zeros(1 + cap, np.uint64)
    buf[0] = n
    buf[1:1 + n] = (np.asarray(gpos, np.uint64) << np.uint64(32)) | \
        (np.asarray(req, np.uint64) << np.uint64(1)) | (np.asarray(is_long, np.uint64) & np.uint64(1))
    return buf


def decode_gathered(recv: np.ndarray, world: int, cap: int, rank: int, own_rows):
    """Host restatement of k_build_global_queue: the union list by global
    position -> (req, is_long, owner, row) arrays of length sum(counts); row
    is this rank's local row for its own entries (``own_rows[k]`` for its
    k-th entry) and XQ_NONE for the others'."""
    words = 1 + cap
    recv = np.asarray(recv, np.uint64).reshape(world, words)
    counts = recv[:, 0].astype(np.int64)
    q = int(counts.sum())
    req = np.zeros(q, np.int64)
    lng = np.zeros(q, np.uint8)
    owner = np.zeros(q, np.int64)
    row = np.full(q, XQ_NONE, np.int64)
    for g in range(world):
        n = int(counts[g])
        key = recv[g, 1:1 + n]
        gp = (key >> np.uint64(32)).astype(np.int64)
        req[gp] = ((key >> np.uint64(1)) & np.uint64(0x7FFFFFFF)).astype(np.int64)
        lng[gp] = (key & np.uint64(1)).astype(np.uint8)
        owner[gp] = g
        if g == rank:
            row[gp] = np.asarray(own_rows, np.int64)[:n]
    return req, lng, owner, row


def exchange(xc, xsend, xrecv, group=None) -> None:
    """The step's only collectives (torch.distributed; NCCL on GPUs, gloo in
    the CPU tests): counters summed, admission entries gathered rank-major."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(xc, op=dist.ReduceOp.SUM, group=group)
        dist.all_gather_into_tensor(xrecv, xsend, group=group)
    else:
        xrecv.copy_(xsend)


class _CudaArray:
    """Zero-copy view of a device buffer owned by libmars_b200 (for torch)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<i8") -> None:
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


class ShardedEngine:
    """One replica (this rank's GPU) of a sharded engine."""

    def __init__(self, engine, group=None, world: Optional[int] = None,
                 rank: Optional[int] = None) -> None:
        import torch
        import torch.distributed as dist

        self.eng = engine
        self.group = group
        init = dist.is_available() and dist.is_initialized()
        self.world = world if world is not None else (dist.get_world_size(group) if init else 1)
        self.rank = rank if rank is not None else (dist.get_rank(group) if init else 0)
        lib = engine.lib
        N.check(lib.mars_shard_init(engine.ctx, self.world, self.rank), engine.ctx)
        xc, xs, xr = C.c_void_p(), C.c_void_p(), C.c_void_p()
        words = C.c_int64()
        N.check(lib.mars_shard_buffers(engine.ctx, C.byref(xc), C.byref(xs), C.byref(xr),
                                       C.byref(words)), engine.ctx)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.words = words.value
        self.xc = torch.as_tensor(_CudaArray(xc.value, N.XC_N), device=dev)
        self.xsend = torch.as_tensor(_CudaArray(xs.value, self.words), device=dev)
        self.xrecv = torch.as_tensor(_CudaArray(xr.value, self.words * self.world), device=dev)
        # collectives and kernels on one stream
        self.stream = torch.cuda.Stream(device=dev)
        N.check(lib.mars_set_stream(engine.ctx, self.stream.cuda_stream), engine.ctx)

    def set_queue(self, rows, req, is_long, gpos) -> None:
        self.eng.set_queue(rows, req, is_long)
        g = np.ascontiguousarray(gpos, np.uint32)
        N.check(self.eng.lib.mars_set_queue_gpos(self.eng.ctx, len(g),
                                                 g.ctypes.data_as(C.c_void_p)), self.eng.ctx)

    def get_queue(self) -> Tuple[np.ndarray, np.ndarray]:
        rows = self.eng.get_queue()
        n = C.c_int64()
        g = np.zeros(len(rows), np.uint32)
        N.check(self.eng.lib.mars_get_queue_gpos(self.eng.ctx, len(g),
                                                 g.ctypes.data_as(C.c_void_p), C.byref(n)),
                self.eng.ctx)
        return rows, g

    def phase(self, si, k: int) -> None:
        import torch

        si.mode |= N.MODE_SHARDED
        with torch.cuda.stream(self.stream):
            N.check(self.eng.lib.mars_step_phase(self.eng.ctx, C.byref(si), k), self.eng.ctx)

    def step(self, si):
        import torch

        self.phase(si, 1)
        with torch.cuda.stream(self.stream):
            exchange(self.xc[:len(COUNTERS)], self.xsend, self.xrecv, self.group)
        self.phase(si, 2)
        return self.eng.fetch()

    def capture(self, si) -> None:
        """The whole sharded step -- phase 1, the NCCL all-reduce and
        all-gather, phase 2 -- as ONE CUDA graph on the replica's stream
        (torch.cuda.graph captures the collectives; the library's kernels are
        stream-ordered launches with no host synchronisation).  ``replay``
        then launches it; ``si`` is the step the graph repeats (the step
        input is a by-value parameter of the graph's head kernel, fixed at
        capture: capture again for another input)."""
        import torch

        si.mode |= N.MODE_SHARDED
        self._si = si
        lib, ctx = self.eng.lib, self.eng.ctx
        # one eager step first: NCCL communicators and every kernel exist
        self.step(si)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            N.check(lib.mars_step_phase(ctx, C.byref(si), 1), ctx)
            exchange(self.xc[:len(COUNTERS)], self.xsend, self.xrecv, self.group)
            N.check(lib.mars_step_phase(ctx, C.byref(si), 2), ctx)

    def replay(self) -> None:
        import torch

        # (a graph replays on the current stream: the replica's, so it is
        # ordered with the library's own copies and the fetch)
        with torch.cuda.stream(self.stream):
            self.graph.replay()
