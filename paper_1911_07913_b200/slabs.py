"""Multi-GPU slabs: transports for the slab-sharded step and the slab planner.

The reference is one process (hotmpm has no distributed path; its only parallelism is the
``parallel_for`` thread pool, common.hpp:77-83).  Here every GPU runs one process with one
context, all ranks upload the same particles, and the solve cuts the level-0 rows into slabs
of lattice planes along axis 0 (include/hot_c_api.h).  Two transports:

* ``attach_nccl(sim)`` — NCCL inside the library, stream-ordered on the context's stream
  (the production path; one GPU per rank).  The unique id travels over the caller's
  ``torch.distributed`` process group.
* ``HostComm`` / ``attach_host(sim)`` — the library stages each range through pinned host
  memory and calls back into Python, which runs the collective on CPU tensors over any
  ``torch.distributed`` backend (gloo).  Used by the multi-process tests, which can place two
  ranks on one GPU because no kernel ever waits on another rank.  With ``device_buffers = 1``
  the callbacks receive the device buffers instead (tools/slab_emulate.py).
"""
from __future__ import annotations

import ctypes as C
import traceback

import numpy as np

from . import capi


def plan_slabs(plane_lo: int, weights, size: int, align: int = 2, min_width: int = 2):
    """hot_plan_slabs: cut planes [plane_lo, plane_lo + len(weights)) into ``size`` slabs.

    Returns the ``size + 1`` absolute plane cuts; raises InvalidArgument when no cut exists."""
    w = np.ascontiguousarray(weights, dtype=np.int64)
    bounds = np.zeros(size + 1, dtype=np.int32)
    code = capi.lib().hot_plan_slabs(int(plane_lo), int(w.size), w.ctypes.data_as(C.POINTER(C.c_longlong)),
                                     int(size), int(align), int(min_width), capi.iptr(bounds))
    capi.raise_for(code, "hot_plan_slabs: no admissible cut (too few planes for the slab count)")
    return [int(b) for b in bounds]


def _bytes_at(addr: int, lo: int, hi: int) -> np.ndarray:
    """A numpy view of host bytes [addr + lo, addr + hi)."""
    n = hi - lo
    if n <= 0:
        return np.zeros(0, dtype=np.uint8)
    return np.ctypeslib.as_array((C.c_ubyte * n).from_address(addr + lo))


class HostComm:
    """The collectives of hot_comm_host over a torch.distributed process group (CPU tensors).

    The three methods operate on host memory addresses exactly as the library calls them, so
    they are testable without a GPU (tests/test_slabs_cpu.py)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.calls = {"allgather_ranges": 0, "halo": 0, "allreduce_max": 0}

    def _all_gather_padded(self, payload: np.ndarray):
        import torch

        n = torch.tensor([payload.size], dtype=torch.int64)
        ns = [torch.zeros(1, dtype=torch.int64) for _ in range(self.size)]
        self.dist.all_gather(ns, n, group=self.group)
        mx = max(int(t.item()) for t in ns)
        t = torch.zeros(max(mx, 1), dtype=torch.uint8)
        if payload.size:
            t[:payload.size] = torch.from_numpy(payload.copy())
        outs = [torch.zeros(max(mx, 1), dtype=torch.uint8) for _ in range(self.size)]
        self.dist.all_gather(outs, t, group=self.group)
        return [o.numpy()[:int(k.item())] for o, k in zip(outs, ns)]

    def allgather_ranges(self, addr: int, off) -> None:
        """Rank r's bytes [off[r], off[r+1]) of the buffer at ``addr`` to every rank."""
        self.calls["allgather_ranges"] += 1
        off = [int(off[i]) for i in range(self.size + 1)]
        parts = self._all_gather_padded(_bytes_at(addr, off[self.rank], off[self.rank + 1]))
        for r in range(self.size):
            if r != self.rank:
                _bytes_at(addr, off[r], off[r + 1])[:] = parts[r]

    def halo(self, addr: int, edges) -> None:
        """Rank r receives rank r-1's last-planes range and rank r+1's first-planes range."""
        self.calls["halo"] += 1
        e = [int(edges[i]) for i in range(4 * self.size)]
        me = self.rank
        lo = _bytes_at(addr, e[4 * me], e[4 * me + 1])
        hi = _bytes_at(addr, e[4 * me + 2], e[4 * me + 3])
        parts = self._all_gather_padded(np.concatenate([lo, hi]))
        if me > 0:
            a, b, c, d = e[4 * (me - 1):4 * me]
            _bytes_at(addr, c, d)[:] = parts[me - 1][b - a:]
        if me + 1 < self.size:
            a, b = e[4 * (me + 1)], e[4 * (me + 1) + 1]
            _bytes_at(addr, a, b)[:] = parts[me + 1][:b - a]

    def allreduce_max(self, vals) -> list:
        import torch

        self.calls["allreduce_max"] += 1
        t = torch.tensor([int(v) for v in vals], dtype=torch.int64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return [int(v) for v in t.tolist()]

    # ------------------------------------------------------------------ C callbacks
    def c_struct(self) -> capi.hot_comm_host:
        def ag(user, buf, off):
            try:
                self.allgather_ranges(buf, off)
                return 0
            except Exception:  # an exception must not unwind through C frames
                traceback.print_exc()
                return 1

        def halo(user, buf, edges):
            try:
                self.halo(buf, edges)
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        def mx(user, v, n):
            try:
                out = self.allreduce_max([v[i] for i in range(n)])
                for i in range(n):
                    v[i] = out[i]
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        # the CFUNCTYPE objects must outlive the context: keep them on self
        self._cb = (capi.ALLGATHER_FN(ag), capi.HALO_FN(halo), capi.MAXI32_FN(mx))
        return capi.hot_comm_host(None, self.rank, self.size, *self._cb, int(getattr(self, "device_buffers", 0)))


def attach_host(sim, group=None) -> HostComm:
    """Host-staged collectives over ``group`` (any torch.distributed backend, CPU tensors)."""
    hc = HostComm(group)
    ops = hc.c_struct()
    sim._check(sim._lib.hot_set_comm_host(sim.handle, C.byref(ops)))
    sim._comm_keepalive = (hc, ops)
    return hc


def attach_nccl(sim, group=None) -> None:
    """NCCL collectives inside the library: rank 0 makes the unique id, the group broadcasts it."""
    import torch.distributed as dist

    import os

    if "HOT_NCCL_LIB" not in os.environ:  # prefer the NCCL torch itself loads (nvidia-nccl wheel)
        try:
            import nvidia.nccl

            cand = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["HOT_NCCL_LIB"] = cand
        except ImportError:
            pass
    rank, size = dist.get_rank(group), dist.get_world_size(group)
    uid = (C.c_ubyte * 128)()
    err = None
    if rank == 0:  # never raise before the broadcast: the other ranks would wait in it forever
        rc = capi.lib().hot_nccl_unique_id(uid)
        if rc != 0:
            err = f"hot_nccl_unique_id failed (libnccl.so.2), status {rc}"
    box = [bytes(uid), err]
    dist.broadcast_object_list(box, src=0, group=group)
    if box[1] is not None:  # every rank raises together
        raise RuntimeError(box[1])
    uid = (C.c_ubyte * 128).from_buffer_copy(box[0])
    sim._check(sim._lib.hot_set_comm_nccl(sim.handle, uid, rank, size))


def detach(sim) -> None:
    sim._check(sim._lib.hot_set_comm_host(sim.handle, None))
    sim._comm_keepalive = None


def shard_info(sim) -> dict:
    out = capi.hot_shard_info_t()
    sim._check(sim._lib.hot_shard_info(sim.handle, C.byref(out)))
    return {k: getattr(out, k) for k, _ in capi.hot_shard_info_t._fields_}
