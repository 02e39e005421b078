"""One rank of a slab-sharded run (tests/test_gpu_slabs.py launches `size` of these).

    python tests/slab_worker.py RANK SIZE PORT SCENE STEPS OUT.npz [transport] [levels]

Every rank uploads the same particles, attaches the host-staged transport over a gloo group
(several ranks may share one GPU: no kernel waits on another rank), advances STEPS steps and
writes its final particles, per-step stats and the shard report to OUT.npz.  SIZE = 1 runs
the single-GPU step with no transport (the reference the sharded ranks must equal bitwise).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    rank, size, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    scene_path, steps, out = sys.argv[4], int(sys.argv[5]), sys.argv[6]
    transport = sys.argv[7] if len(sys.argv) > 7 else "host"
    levels = int(sys.argv[8]) if len(sys.argv) > 8 else None
    from paper_1911_07913_b200 import Simulation, load_scene_file, sample_scene_particles
    from paper_1911_07913_b200 import slabs

    sc = load_scene_file(scene_path)
    sim = Simulation(sc, device=int(os.environ.get("SLAB_DEVICE", "0")))
    if levels is not None:
        sim.set_solver(levels=levels)
    sim.set_particles(**sample_scene_particles(sc))
    if size > 1 or transport == "nccl":
        import torch.distributed as dist

        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=size)
        if transport == "nccl":
            slabs.attach_nccl(sim)
        else:
            slabs.attach_host(sim)
    stats, infos = [], []
    for k in range(steps):
        st = sim.advance_step((k + 1) / sc.fps)
        stats.append([st["dt"], st["outer_iterations"], st["inner_total"], st["node_count"]])
        infos.append(slabs.shard_info(sim))
    p = sim.particles()
    diag = sim.diagnostics()
    # after a sharded solve level 0 holds only this rank's rows: the matrix taps must refuse
    from paper_1911_07913_b200 import LogicError

    try:
        sim.level_shape(0)
        tap_blocked = 0
    except LogicError:
        tap_blocked = 1
    np.savez(out, x=p["x"], v=p["v"], F=p["F"], C=p["C"], stats=np.array(stats),
             sharded=np.array([i["sharded"] for i in infos]),
             rows=np.array([[i["row_lo"], i["row_hi"], i["crow_lo"], i["crow_hi"], i["plane_lo"], i["plane_hi"]]
                            for i in infos]),
             halos=np.array(infos[-1]["halo_exchanges"] if infos else 0),
             particles_local=np.array([i["particles_local"] for i in infos]),
             particles_total=np.array([i["particles_total"] for i in infos]),
             partitioned=np.array([i["partitioned"] for i in infos]),
             gathers=np.array(infos[-1]["gathers"] if infos else 0),
             energy=diag["energy"], residual=diag["scaled_residual"], tap_blocked=np.array(tap_blocked))
    if size > 1 or transport == "nccl":
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    sim.close()


if __name__ == "__main__":
    main()
