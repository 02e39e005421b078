"""Host logic of the multi-GPU slabs, on the CPU: the slab planner (hot_plan_slabs, pure host
code in the library) and the host-staged collectives over a real 2- and 3-rank gloo group,
driven exactly as the library drives them (through the C callback structs, on raw host
addresses).  The device half is tests/test_gpu_slabs.py."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

from paper_1911_07913_b200 import InvalidArgument, capi
from paper_1911_07913_b200.slabs import HostComm, plan_slabs


def _check_cut(b, lo, n, size, align, min_width):
    assert len(b) == size + 1 and b[0] == lo and b[-1] == lo + n
    for r in range(size):
        assert b[r + 1] - b[r] >= min_width
    for c in b[1:-1]:
        assert c % align == 0


def test_plan_slabs_uniform_is_balanced():
    b = plan_slabs(0, np.ones(128, np.int64), 8)
    assert b == list(range(0, 129, 16))


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("size", [1, 2, 3, 5, 8])
def test_plan_slabs_constraints_and_balance(seed, size):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(size * 4, 200))
    lo = int(rng.integers(-50, 50))
    w = rng.integers(0, 1000, n)
    w[rng.random(n) < 0.2] = 0  # empty planes (gaps between objects)
    b = plan_slabs(lo, w, size, align=2, min_width=2)
    _check_cut(b, lo, n, size, 2, 2)
    # every interior cut is within one aligned step (2 planes) of the ideal prefix weight,
    # unless a neighbour constraint pinned it
    pre = np.concatenate([[0], np.cumsum(w)])
    for r in range(1, size):
        k = b[r] - lo
        target = pre[-1] * r / size
        slack = w[max(k - 2, 0):k + 2].sum()
        pinned = b[r] - b[r - 1] == 2 or b[r + 1] - b[r] <= 3
        assert pinned or abs(pre[k] - target) <= slack


def test_plan_slabs_negative_origin_alignment():
    b = plan_slabs(-7, np.ones(20, np.int64), 3, align=4, min_width=3)
    _check_cut(b, -7, 20, 3, 4, 3)


def test_plan_slabs_infeasible():
    with pytest.raises(InvalidArgument):
        plan_slabs(0, np.ones(7, np.int64), 4, align=2, min_width=2)
    with pytest.raises(InvalidArgument):
        plan_slabs(0, np.ones(0, np.int64), 2)


# ------------------------------------------------------------------ collectives over gloo
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, size, port, results):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=size)
    try:
        hc = HostComm()
        ops = hc.c_struct()  # call through the C function pointers, as libhotb200 does
        # a "node vector" of 3 doubles per row; rank r owns rows [8r, 8r + 8) (+ rank-specific size)
        counts = [8 + r for r in range(size)]
        rows = np.concatenate([[0], np.cumsum(counts)])
        buf = np.full(3 * rows[-1], -1.0)
        buf[3 * rows[rank]:3 * rows[rank + 1]] = rank + np.arange(3 * counts[rank]) / 1000.0
        off = (C.c_longlong * (size + 1))(*[24 * int(x) for x in rows])
        assert ops.allgather_ranges(None, buf.ctypes.data, off) == 0
        want = np.concatenate([r + np.arange(3 * counts[r]) / 1000.0 for r in range(size)])
        ok_gather = bool(np.array_equal(buf, want))
        # halo: first 2 rows / last 2 rows of each slab; the neighbours' edges land in place
        buf2 = np.full(3 * rows[-1], -1.0)
        buf2[3 * rows[rank]:3 * rows[rank + 1]] = 100 + rank
        edges = []
        for r in range(size):
            edges += [24 * int(rows[r]), 24 * int(rows[r] + 2), 24 * int(rows[r + 1] - 2), 24 * int(rows[r + 1])]
        e = (C.c_longlong * (4 * size))(*edges)
        assert ops.halo(None, buf2.ctypes.data, e) == 0
        exp = np.full(3 * rows[-1], -1.0)
        exp[3 * rows[rank]:3 * rows[rank + 1]] = 100 + rank
        if rank > 0:
            exp[3 * (rows[rank] - 2):3 * rows[rank]] = 100 + rank - 1
        if rank + 1 < size:
            exp[3 * rows[rank + 1]:3 * (rows[rank + 1] + 2)] = 100 + rank + 1
        ok_halo = bool(np.array_equal(buf2, exp))
        v = (C.c_int * 3)(rank, -rank, 7 if rank == size - 1 else 0)
        assert ops.allreduce_max_i32(None, v, 3) == 0
        ok_max = list(v) == [size - 1, 0, 7]
        results[rank] = (ok_gather, ok_halo, ok_max, dict(hc.calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("size", [2, 3])
def test_host_collectives_gloo(size):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, size, port, results)) for r in range(size)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for r in range(size):
        ok_gather, ok_halo, ok_max, calls = results[r]
        assert ok_gather and ok_halo and ok_max, (r, results[r])
        assert calls == {"allgather_ranges": 1, "halo": 1, "allreduce_max": 1}


def test_abi_exports_slab_symbols():
    L = capi.lib()
    for sym in ("hot_set_comm_host", "hot_set_comm_nccl", "hot_nccl_unique_id", "hot_shard_info", "hot_plan_slabs"):
        assert hasattr(L, sym)
    assert os.path.exists(capi.LIB_PATH)
