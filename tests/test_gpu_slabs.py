"""Slab-sharded step on the GPU: `size` ranks, each a process with
its own context, joined by the host-staged transport over gloo.  The ranks share the one GPU
of the test box; no kernel waits on another rank (every exchange is a host-side collective
between launches), so the ranks need not be co-scheduled.

The bar is stronger than the oracle's 1e-6: every row is computed with the single-GPU
arithmetic in the single-GPU order and the replicated scalars are reduced identically, so the
sharded step must equal the single-GPU step BITWISE, and therefore the oracle as closely as the
single-GPU step does (tests/test_gpu_parity.py)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "slab_worker.py")
SCENES = os.path.join(ROOT, "scenes")

pytestmark = pytest.mark.gpu

# Every level-0 smoother schedule (dataflow on small grids, streaming on large ones, per-wave
# launches or streamed residue groups in a slab) sums a row in the same order, so sharded and
# single-GPU steps agree bit for bit under the default settings.
ENV = dict(os.environ)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_ranks(tmp_path, scene, size, steps, levels=None, tag="r"):
    port = _free_port()
    procs, outs = [], []
    for r in range(size):
        out = str(tmp_path / f"{tag}{size}_{r}.npz")
        args = [sys.executable, WORKER, str(r), str(size), str(port), os.path.join(SCENES, scene), str(steps), out,
                "host"] + ([str(levels)] if levels is not None else [])
        procs.append(subprocess.Popen(args, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, env=ENV))
        outs.append(out)
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(o)
    for p, o in zip(procs, logs):
        assert p.returncode == 0, o[-4000:]
    return [dict(np.load(o)) for o in outs]


@pytest.mark.parametrize("scene,steps", [("cfg1_stretched.json", 3), ("cfg1_drop.json", 3)])
@pytest.mark.parametrize("size", [2, 3])
def test_sharded_steps_equal_single_gpu_bitwise(tmp_path, scene, steps, size):
    ref = run_ranks(tmp_path, scene, 1, steps, tag="single")[0]
    ranks = run_ranks(tmp_path, scene, size, steps)
    iters = ref["stats"][:, 1]
    assert iters.sum() > 0, "the scene must exercise the solve"
    for r, res in enumerate(ranks):
        solved = iters > 0
        assert (res["sharded"][solved] == 1).all(), (r, res["sharded"])
        assert res["halos"] > 0 and res["gathers"] > 0
        if res["sharded"][-1]:
            assert res["tap_blocked"] == 1  # level 0 is split: no tap reads it
        # after the first sharded step the particles are partitioned: each rank stores its band
        # (on these small cubes the 8 + 1 ghost planes still cover most of the scene)
        first = int(np.argmax(res["sharded"] == 1))
        assert (res["partitioned"][first:] == 1).all(), res["partitioned"]
        assert (res["particles_local"][first:] <= res["particles_total"][first:]).all()
        np.testing.assert_array_equal(res["stats"], ref["stats"])
        for k in ("x", "v", "F", "C", "energy", "residual"):
            np.testing.assert_array_equal(res[k], ref[k], err_msg=f"rank {r} {k}")
    # the slabs tile the rows: contiguous, disjoint, covering [0, n)
    last = ranks[0]["rows"][-1]
    for r in range(1, size):
        cur = ranks[r]["rows"][-1]
        assert cur[0] == last[1] and cur[2] == last[3] and cur[4] == last[5]
        last = cur
    assert ranks[0]["rows"][-1][0] == 0 and ranks[-1]["rows"][-1][1] == ref["stats"][-1][3]


def test_sharded_two_level_hierarchy(tmp_path):
    """levels = 2: the coarse level that is replicated is also the coarsest (PCG) level."""
    ref = run_ranks(tmp_path, "cfg1_stretched.json", 1, 2, levels=2, tag="single")[0]
    ranks = run_ranks(tmp_path, "cfg1_stretched.json", 2, 2, levels=2)
    for res in ranks:
        assert res["sharded"].any()
        for k in ("x", "v", "F", "C"):
            np.testing.assert_array_equal(res[k], ref[k])


def test_sharded_benchmark_scene_two_steps(tmp_path):
    """The benchmark workload (cfg2, 1.19M particles): 2 ranks equal 1 GPU bitwise."""
    scene = "cfg2_twisting_bars.json"
    ref = run_ranks(tmp_path, scene, 1, 2, tag="single")[0]
    ranks = run_ranks(tmp_path, scene, 2, 2)
    assert ref["stats"][:, 1].sum() > 0
    for res in ranks:
        assert res["sharded"].any()
        np.testing.assert_array_equal(res["stats"], ref["stats"])
        for k in ("x", "v", "F", "C"):
            np.testing.assert_array_equal(res[k], ref[k])
        # partitioned after the first step: a rank stores its half plus 9 planes of ghosts
        assert res["partitioned"][-1] == 1
        assert res["particles_local"][-1] < 0.75 * res["particles_total"][-1], res["particles_local"]


def test_sharded_four_ranks_partition_memory(tmp_path):
    """4 ranks on the benchmark workload: bitwise equal to 1 GPU, and each rank stores only its
    slab plus the 8 + 1 ghost planes the assembly and the node passes read (cfg2's bars span
    ~130 planes along axis 0)."""
    scene = "cfg2_twisting_bars.json"
    ref = run_ranks(tmp_path, scene, 1, 3, tag="single")[0]
    four = run_ranks(tmp_path, scene, 4, 3)
    for res in four:
        np.testing.assert_array_equal(res["stats"], ref["stats"])
        for k in ("x", "v", "F", "C", "energy", "residual"):
            np.testing.assert_array_equal(res[k], ref[k])
    total = four[0]["particles_total"][-1]
    assert sum(r["partitioned"][-1] for r in four) == 4
    assert max(r["particles_local"][-1] for r in four) < 0.4 * total, [r["particles_local"] for r in four]


def test_nccl_transport_single_rank(tmp_path):
    """The NCCL transport's own calls on the one GPU of the test box: libnccl.so.2 loaded at run
    time, communicator init, the row gathers (in-place broadcasts) and the flag allreduce, with
    the sharded path forced at one rank (HOT_SHARD_FORCE).  NCCL refuses two ranks on one GPU,
    so the send/recv halo pair cannot run here."""
    ref = run_ranks(tmp_path, "cfg1_stretched.json", 1, 2, tag="single")[0]
    port = _free_port()
    out = str(tmp_path / "nccl1.npz")
    env = dict(ENV, HOT_SHARD_FORCE="1")
    p = subprocess.run([sys.executable, WORKER, "0", "1", str(port), os.path.join(SCENES, "cfg1_stretched.json"), "2",
                        out, "nccl"], capture_output=True, text=True, env=env, timeout=600)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    res = dict(np.load(out))
    assert res["sharded"].any() and res["gathers"] > 0
    for k in ("x", "v", "F", "C"):
        np.testing.assert_array_equal(res[k], ref[k])


def _gpu_count():
    from paper_1911_07913_b200 import capi

    return capi.lib().hot_device_count()


@pytest.mark.skipif(_gpu_count() < 2, reason="needs two GPUs: NCCL refuses two ranks on one device")
def test_nccl_transport_two_gpus(tmp_path):
    """Two ranks on two GPUs over the library's NCCL transport: the send/recv halo
    pairs and the grouped in-place broadcasts at size 2; every rank bitwise equal to one GPU."""
    ref = run_ranks(tmp_path, "cfg1_stretched.json", 1, 3, tag="single")[0]
    port = _free_port()
    procs, outs = [], []
    for r in range(2):
        out = str(tmp_path / f"nccl2_{r}.npz")
        env = dict(ENV, SLAB_DEVICE=str(r))
        procs.append(subprocess.Popen([sys.executable, WORKER, str(r), "2", str(port),
                                       os.path.join(SCENES, "cfg1_stretched.json"), "3", out, "nccl"],
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, env=env))
        outs.append(out)
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(o)
    for p, o in zip(procs, logs):
        assert p.returncode == 0, o[-4000:]
    for out in outs:
        res = dict(np.load(out))
        assert res["sharded"].any()
        for k in ("x", "v", "F", "C"):
            np.testing.assert_array_equal(res[k], ref[k])


def _scene_file(tmp_path, name, objects, materials=None):
    d = {"dim": 3, "dx": 1.0 / 64, "gravity": [0.0, -9.8, 0.0], "fps": 500, "frames": 4, "epsilon": 1e-05, "seed": 7,
         "ppc": 8, "domain": {"min": [0.0, 0.0, 0.0], "max": [1.0, 1.0, 1.0]},
         "materials": materials or [{"density": 1000.0, "youngs": 1e5, "poisson": 0.3}],
         "objects": objects,
         "colliders": [{"shape": {"kind": "half_space", "point": [0.0, 0.05, 0.0], "normal": [0.0, 1.0, 0.0]},
                        "motion": {"kind": "static"}}]}
    path = tmp_path / f"{name}.json"
    path.write_text(json.dumps(d))
    return str(path)


def _stretched_box(lo, hi):
    return {"shape": {"kind": "box", "min": lo, "max": hi}, "material": 0,
            "initial_deformation": {"kind": "random_diagonal", "lo": 0.7, "hi": 1.3}}


def test_sharded_gap_between_objects(tmp_path):
    """Two boxes with empty lattice planes between them along axis 0: slabs whose rows are
    unevenly spread, planes without rows inside a slab."""
    scene = _scene_file(tmp_path, "gap", [_stretched_box([0.20, 0.3, 0.3], [0.30, 0.4, 0.4]),
                                          _stretched_box([0.55, 0.3, 0.3], [0.70, 0.45, 0.45])])
    ref = run_ranks(tmp_path, scene, 1, 2, tag="single")[0]
    for size in (2, 3):
        ranks = run_ranks(tmp_path, scene, size, 2, tag=f"gap{size}_")
        for res in ranks:
            assert res["sharded"].any()
            for k in ("x", "v", "F", "C"):
                np.testing.assert_array_equal(res[k], ref[k])


def test_too_few_planes_runs_replicated(tmp_path):
    """A sliver one cell thick along axis 0 has too few planes for 3 slabs of >= 2 planes at
    even cuts: the planner declines, every rank runs the whole solve, results unchanged."""
    scene = _scene_file(tmp_path, "sliver", [_stretched_box([0.40, 0.3, 0.3], [0.42, 0.5, 0.5])])
    ref = run_ranks(tmp_path, scene, 1, 2, tag="single")[0]
    assert ref["stats"][:, 1].sum() > 0
    ranks = run_ranks(tmp_path, scene, 3, 2, tag="sliver")
    for res in ranks:
        assert not res["sharded"].any()
        for k in ("x", "v", "F", "C"):
            np.testing.assert_array_equal(res[k], ref[k])


@pytest.mark.parametrize("plasticity", [{"kind": "von_mises", "yield_stress": 3e3},
                                        {"kind": "snow_clamp", "lo": 0.975, "hi": 1.0075}])
def test_sharded_plastic_materials(tmp_path, plasticity):
    """Plastic materials (von Mises, the snow clamp) on stretched boxes that yield at once: the
    return maps run in the replicated G2P; energy, gradient and assembly are split.  2 ranks
    equal 1 GPU bitwise over 3 steps."""
    mat = [{"density": 1000.0, "youngs": 1e5, "poisson": 0.3, "plasticity": plasticity}]
    scene = _scene_file(tmp_path, "plastic", [_stretched_box([0.35, 0.35, 0.35], [0.6, 0.6, 0.6])], mat)
    ref = run_ranks(tmp_path, scene, 1, 3, tag="single")[0]
    assert ref["stats"][:, 1].sum() > 0
    ranks = run_ranks(tmp_path, scene, 2, 3)
    for res in ranks:
        assert res["sharded"].any()
        np.testing.assert_array_equal(res["stats"], ref["stats"])
        for k in ("x", "v", "F", "C"):
            np.testing.assert_array_equal(res[k], ref[k])
