#!/usr/bin/env python
"""Per-rank critical path of the slab-sharded step, measured on ONE GPU.

    python tools/slab_emulate.py [--scene S] [--ranks 1,2,4,8] [--steps K] [--warmup W]

R ranks run in-process as R threads, each with its own context (scene copy) on the same GPU,
joined by caller-owned collectives on the device buffers (hot_set_comm_host with
device_buffers = 1) that copy the ranges device-to-device between the rank contexts.  A
baton serialises them: a rank holds it from the end of one collective to the start of the
next, and the library synchronises the rank's stream before every collective, so the GPU runs
one rank's segment at a time and each segment's wall time is that rank's own work (kernels +
launch overhead), with no contention.  No kernel waits on another rank.

Ranks call the same collectives in the same order, so segment k of every rank ends at the
same collective.  On R GPUs a segment ends when its slowest rank arrives:

    critical path = sum_k max_r segment[r][k]

The transport is NOT measured here (one GPU has no NVLink peer).  It is added as a model:
`lat` seconds per collective plus the bytes each rank receives over `bw` GB/s (NCCL on
NVLink 5 / NVSwitch); both are printed, and the JSON separates compute from the model.
"""
import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1911_07913_b200 import Simulation, capi, load_scene_file, sample_scene_particles  # noqa: E402
from paper_1911_07913_b200 import slabs  # noqa: E402


class Group:
    def __init__(self, R):
        self.R = R
        self.barrier = threading.Barrier(R)
        self.baton = threading.Lock()
        self.slots = [None] * R


class _DevBytes:
    """A raw device byte range as a torch tensor (zero copy)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def dev_bytes(ptr, lo, hi):
    import torch

    return torch.as_tensor(_DevBytes(ptr + lo, hi - lo), device="cuda")


class ThreadComm(slabs.HostComm):
    """hot_comm_host over an in-process exchange with the baton protocol, on the DEVICE buffers
    (device_buffers = 1): the ranges move by device-to-device copies between the rank
    contexts, outside every rank's timed segments."""

    device_buffers = 1

    def __init__(self, grp, rank):
        self.grp, self.rank, self.size = grp, rank, grp.R
        self.calls = {"allgather_ranges": 0, "halo": 0, "allreduce_max": 0}
        self.segments = []    # wall seconds of each segment this rank ran holding the baton
        self.recv_bytes = []  # bytes this rank receives at each collective
        self.t0 = None

    def start(self):
        self.grp.baton.acquire()
        self.t0 = time.perf_counter()

    def stop(self):
        self.segments.append(time.perf_counter() - self.t0)
        self.grp.baton.release()

    def _exchange(self, payload, between=None):
        self.segments.append(time.perf_counter() - self.t0)
        g = self.grp
        g.slots[self.rank] = payload
        g.baton.release()
        g.barrier.wait()
        parts = list(g.slots)
        if between:
            between(parts)
        g.barrier.wait()
        g.baton.acquire()
        self.t0 = time.perf_counter()
        return parts

    def allgather_ranges(self, addr, off):
        import torch

        self.calls["allgather_ranges"] += 1
        off = [int(off[i]) for i in range(self.size + 1)]

        def copy(ptrs):
            for r in range(self.size):
                if r != self.rank and off[r + 1] > off[r]:
                    dev_bytes(addr, off[r], off[r + 1]).copy_(dev_bytes(ptrs[r], off[r], off[r + 1]))
            torch.cuda.synchronize()

        self._exchange(addr, copy)
        self.recv_bytes.append(off[-1] - (off[self.rank + 1] - off[self.rank]))

    def halo(self, addr, edges):
        import torch

        self.calls["halo"] += 1
        e = [int(edges[i]) for i in range(4 * self.size)]
        me = self.rank
        got = [0]

        def copy(ptrs):
            if me > 0 and e[4 * (me - 1) + 3] > e[4 * (me - 1) + 2]:
                a, b = e[4 * (me - 1) + 2], e[4 * (me - 1) + 3]
                dev_bytes(addr, a, b).copy_(dev_bytes(ptrs[me - 1], a, b))
                got[0] += b - a
            if me + 1 < self.size and e[4 * (me + 1) + 1] > e[4 * (me + 1)]:
                a, b = e[4 * (me + 1)], e[4 * (me + 1) + 1]
                dev_bytes(addr, a, b).copy_(dev_bytes(ptrs[me + 1], a, b))
                got[0] += b - a
            torch.cuda.synchronize()

        self._exchange(addr, copy)
        self.recv_bytes.append(got[0])

    def allreduce_max(self, vals):
        self.calls["allreduce_max"] += 1
        parts = self._exchange(list(vals))
        self.recv_bytes.append(8 * len(vals) * (self.size - 1))
        return [max(p[i] for p in parts) for i in range(len(vals))]


def run(sc, particles, R, steps, warmup):
    grp = Group(R)
    sims, comms = [], []
    for r in range(R):
        sim = Simulation(sc, device=0)
        sim.set_particles(**particles)
        sims.append(sim)
        if R > 1:
            comm = ThreadComm(grp, r)
            ops = comm.c_struct()
            sim._check(sim._lib.hot_set_comm_host(sim.handle, C.byref(ops)))
            sim._comm_keepalive = (comm, ops)
            comms.append(comm)
    results = [None] * R
    marks = [None] * R
    ends = [None] * R

    def body(r):
        sim = sims[r]
        comm = comms[r] if R > 1 else None
        if comm:
            comm.start()
        for k in range(warmup):
            sim.advance_step((k + 1) / sc.fps)
        if comm:  # a segment boundary at the same logical point on every rank (no exchange)
            comm.segments.append(time.perf_counter() - comm.t0)
            comm.t0 = time.perf_counter()
            marks[r] = (len(comm.segments), len(comm.recv_bytes))
        sim.profile(True)
        t = time.perf_counter()
        outer = []
        for k in range(warmup, warmup + steps):
            outer.append(sim.advance_step((k + 1) / sc.fps)["outer_iterations"])
        wall = time.perf_counter() - t
        if comm:  # the timed segments end at the same logical point on every rank
            comm.segments.append(time.perf_counter() - comm.t0)
            comm.t0 = time.perf_counter()
            ends[r] = (len(comm.segments), len(comm.recv_bytes))
        prof = sim.profile_read()
        # the download is a collective when the particles are partitioned
        state = sim.particles()
        info = slabs.shard_info(sim)
        if comm:
            comm.stop()
        results[r] = dict(outer=outer, wall=wall, state=state, info=info,
                          phases={k: round(v["ms"] / steps, 3) for k, v in prof.items() if v["ms"] > 0})

    threads = [threading.Thread(target=body, args=(r,)) for r in range(R)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    out = dict(ranks=R, outer=results[0]["outer"], rank0_phase_ms_per_step=results[0]["phases"])
    if R == 1:
        out["compute_ms_per_step"] = 1000 * results[0]["wall"] / steps
        out["collectives_per_step"] = 0
        out["recv_mb_per_step"] = 0.0
    else:
        s0, b0 = marks[0]
        s1, b1 = ends[0]
        segs = np.array([c.segments[s0:s1] for c in comms])  # [R, nseg]
        recv = np.array([c.recv_bytes[b0:b1] for c in comms])
        out["compute_ms_per_step"] = 1000 * segs.max(axis=0).sum() / steps
        out["rank_busy_ms_per_step"] = [round(1000 * x / steps, 3) for x in segs.sum(axis=1)]
        slow = int(np.argmax(segs.sum(axis=1)))
        out["slowest_rank"] = slow
        out["slowest_rank_phase_ms_per_step"] = results[slow]["phases"]
        big = np.argsort(-segs[slow])[:5]
        out["slowest_rank_top_segments_ms"] = [[int(k), round(1000 * segs[slow][k], 3)] for k in big]
        out["collectives_per_step"] = recv.shape[1] / steps
        out["recv_mb_per_step"] = float(recv.max(axis=0).sum()) / 1e6 / steps
        out["rows"] = [[res["info"]["row_lo"], res["info"]["row_hi"]] for res in results]
        out["particles_local"] = [res["info"]["particles_local"] for res in results]
        out["particles_total"] = results[0]["info"]["particles_total"]
        for r in range(1, R):
            assert results[r]["outer"] == results[0]["outer"]
    out["_state"] = results[0]["state"]
    out["ranks_bitwise_equal"] = all(
        all(np.array_equal(results[r]["state"][k], results[0]["state"][k]) for k in ("x", "v", "F", "C"))
        for r in range(R))
    for s in sims:
        s.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scene", default=os.path.join(ROOT, "scenes", "cfg2_twisting_bars.json"))
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sweep", type=int, default=0, help="BASELINE config 5 particle set on an N^3 grid "
                    "(tools/kernel_sweep.py) instead of --scene")
    ap.add_argument("--repeat", type=int, default=2, help="runs per rank count; the fastest critical path is kept "
                    "(host-side hiccups of the in-process emulation only ever add time)")
    ap.add_argument("--lat-us", type=float, default=15.0, help="model: seconds per collective (NCCL, NVLink)")
    ap.add_argument("--bw-gbs", type=float, default=350.0, help="model: received GB/s per rank (NCCL, NVLink 5)")
    args = ap.parse_args()
    if args.sweep:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from kernel_sweep import particles_for, scene_for

        sc, particles = scene_for(args.sweep), particles_for(args.sweep)
    else:
        sc = load_scene_file(args.scene)
        particles = sample_scene_particles(sc)
    base = None
    ref_state = None
    for R in [int(x) for x in args.ranks.split(",")]:
        runs = [run(sc, particles, R, args.steps, args.warmup) for _ in range(max(1, args.repeat))]
        o = min(runs, key=lambda d: d["compute_ms_per_step"])
        o["compute_ms_per_step_runs"] = [round(d["compute_ms_per_step"], 3) for d in runs]
        state = o.pop("_state")
        for d in runs:
            d.pop("_state", None)
        if R == 1:
            ref_state = state
        elif ref_state is not None:  # every rank's particles vs the single-GPU run, bit for bit
            o["bitwise_equal_to_1_gpu"] = bool(o["ranks_bitwise_equal"]) and all(
                np.array_equal(state[k], ref_state[k]) for k in ("x", "v", "F", "C"))
        comm_ms = o["collectives_per_step"] * args.lat_us / 1000 + o["recv_mb_per_step"] / args.bw_gbs
        o["comm_model_ms_per_step"] = comm_ms
        o["projected_ms_per_step"] = o["compute_ms_per_step"] + comm_ms
        if base is None:
            base = o["projected_ms_per_step"]
        o["projected_speedup"] = base / o["projected_ms_per_step"]
        o["particles"] = particles["x"].shape[0]
        o["model"] = {"lat_us": args.lat_us, "bw_gbs": args.bw_gbs}
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
