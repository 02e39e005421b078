#!/usr/bin/env python
"""Benchmark of the B200 HOT implicit-MPM step (BASELINE.json metric: implicit MPM
particle-steps/s, fp64, fixed tolerance; plus the dominant kernel's roofline).

Headline workload: BASELINE configs[1], stiffness-contrast twisting bars
(scenes/cfg2_twisting_bars.json: four 0.6 x 0.08 x 0.08 bars, dx = 0.6/128, 8 ppc jittered,
1,193,126 particles, soft/stiff segments E = 1e5 / 1e9, ends driven by rotating kinematic
colliders at +-1 rad/s, fixed-corotated (the reference's only model), eps = 1e-5, dt = CFL 0.6
under a 1/24 s frame cap).  One step = one advance_step (simulation.hpp:286-323): activation +
binning + P2G, the HOT solve, G2P + strain + advect.  The other single-GPU BASELINE configs
(cfg4 colliding snow, 4.0M particles; cfg3 metal impact) are timed in the same run and reported
under "other_configs".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference CPU path on the box's host cores: the oracle port of
hotmpm::advance_step (oracle/, a line-by-line restatement; the reference itself needs Eigen,
which no box has), all host threads, on the SAME full scene, sampled by the oracle's own
restatement of sample_scene_particles, for the same warm-up and timed steps.  That arm never
loads the product library.  Under torchrun (N > 1) the ranks share ONE copy of the workload and
the solve is cut into slabs of lattice planes along axis 0 (NCCL inside the library;
DESIGN.md §6): scaling "strong", value = the scene's particle-steps / the max over ranks of the
device time.  --mode replicas runs N independent copies instead ("weak").
"""
import argparse
import atexit
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

SCENE = os.path.join(ROOT, "scenes", "cfg2_twisting_bars.json")
METRIC = "implicit MPM particle-steps/sec (fp64, fixed tol)"
FP64_PEAK_TFLOPS = 37.06  # fp64 peak measured on this pool's B200: DMMA m8n8k4 37.06, DFMA 34.79 (profiles/r01_fp64_peak.json)
# dram__bytes_read.sum + dram__bytes_write.sum per launch from `ncu --set full` (profiles/), or None
# per launch, from profiles/r02_final4_ncu_full_summary.txt
TRAFFIC = {"k_bin_pairs": 5.72e9, "k_row_gather": 7.48e9, "k_assemble_tiles": 3.467671e9, "sgs_level0": 4.086369e9}
UNIT = "particle-steps/s"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


STEP_TIMES = bool(os.environ.get("BENCH_STEP_TIMES"))  # diagnosis: per-step times of the timed region on stderr
CLOCK_PERIOD_MS = int(os.environ.get("BENCH_CLOCK_MS", "50"))  # nvidia-smi sampling period; 0: no sampler (diagnosis)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.lo, self.hi = 0, None

    def begin_timed(self, wait_s=3.0):
        """Call after warm-up: nvidia-smi's start-up (NVML attach, ~0.1 s, stalls the CUDA process it
        watches: measured 1 run in 4 losing 130 ms of a 300 ms timed region) is over once it has
        printed a row; only rows from here to end_timed() are reported."""
        t0 = time.time()
        while self.proc and not self.rows and time.time() - t0 < wait_s:
            time.sleep(0.01)
        self.lo = len(self.rows)

    def end_timed(self):
        time.sleep(0.06)  # one more sampling period: a region shorter than 50 ms still gets a row
        self.hi = len(self.rows)

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        if CLOCK_PERIOD_MS <= 0:
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", str(CLOCK_PERIOD_MS)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc and self.proc.poll() is None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = self.rows[self.lo:self.hi]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if "Active" in r[3 + k] and "Not" not in r[3 + k]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


WORKLOADS = {
    "cfg2_twisting_bars.json": "cfg2 twisting bars (BASELINE configs[1]), FCR, dt = CFL 0.6 (1/24 s frame cap), eps=1e-5",
    "cfg4_snow.json": "cfg4 colliding snow boxes (BASELINE configs[3]), snow clamp, dt = CFL 0.6, eps=1e-5",
    "cfg3_metal_impact.json": "cfg3 von Mises metal sphere on plate (BASELINE configs[2]), dt = CFL 0.6, eps=1e-5",
    "cfg2_twisting_bars_nh.json": "cfg2 twisting bars with Neo-Hookean (as BASELINE configs[1] specifies; extension)",
    "cfg4_snow_hardening.json": "cfg4 colliding snow boxes with hardening 10 (as BASELINE configs[3] specifies; extension)",
    "sand_column_dp.json": "sand column collapse, Drucker-Prager 30 deg (north star; extension)",
}
# (scene, solver overrides): the other single-GPU BASELINE configs, the extension variants the
# configs name, and the paper's default tolerance eps = 1e-7 (scene.hpp:68) on the headline scene
OTHER_SCENES = [("cfg4_snow.json", {}), ("cfg3_metal_impact.json", {}), ("cfg2_twisting_bars.json", {"epsilon": 1e-7}),
                ("cfg2_twisting_bars_nh.json", {}), ("cfg4_snow_hardening.json", {}), ("sand_column_dp.json", {})]


def workload_config(scene, scene_path, n_particles):
    """The workload description, identical in both arms (built from the scene JSON alone)."""
    name = os.path.basename(scene_path)
    return {"workload": WORKLOADS.get(name, name), "scene": name, "particles": int(n_particles),
            "dx": scene["dx"], "ppc": scene.get("ppc", 0), "fps_cap": scene.get("fps", 24),
            "levels": scene.get("levels", 3), "window": scene.get("window", 8), "epsilon": scene.get("epsilon", 1e-7),
            "l2": "inputs larger than L2 (level-0 matrix > 126 MB)"}


def frame_end(scene, k):
    """frame_end of the k-th step (0-based) in both arms: step k may advance at most to (k+1)/fps."""
    return (k + 1) / scene.get("fps", 24)


def oracle_run(scene, steps, warmup, threads, keep=None):
    """The reference CPU path: the oracle port of hotmpm::advance_step on the oracle's own sampled
    particles (sample_scene_particles restated, simulation.hpp:221-254).  keep(x) -> bool mask
    selects a bounded sample (cpu_baseline); None = the full scene.  Imports only oracle/."""
    from oracle import oracle as O

    O.set_threads(threads)
    orc = O.Oracle(int(scene.get("dim", 3)))
    orc.set_scene(scene)
    orc.sample_scene()
    if keep is not None:
        p = orc.get_particles()
        m = keep(p["x"])
        orc.set_particles(p["x"][m], p["v"][m], p["mass"][m], p["volume"][m], p["F"][m].reshape(-1),
                          p["C"][m].reshape(-1), p["material"][m])
    n = orc.particle_count()
    t_all, outer = 0.0, []
    for k in range(warmup + steps):
        t0 = time.perf_counter()
        st = orc.advance_step(frame_end(scene, k))
        dt = time.perf_counter() - t0
        if k >= warmup:
            t_all += dt
            outer.append(st["outer_iterations"])
    return dict(value=n * steps / t_all, particles=n, steps=steps, seconds=t_all, outer=outer,
                ms_per_step=1000 * t_all / max(steps, 1))


def reference_arm(args):
    """--impl reference: rank 0 alone, all host threads, the full scene, the same W + K steps."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    with open(args.scene) as f:
        scene = json.load(f)
    threads = os.cpu_count() or 1
    r = oracle_run(scene, max(args.steps, 1), args.warmup, threads)
    config = workload_config(scene, args.scene, r["particles"])
    sample = (f"the full scene ({r['particles']} particles), {args.warmup} warm-up + {r['steps']} timed steps from "
              f"t=0 (the GPU arm's step sequence), oracle port of hotmpm::advance_step, {threads} threads; "
              f"outer iterations {r['outer']}")
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": r["steps"], "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded scene sampling)",
            "config": config, "outer_iterations": r["outer"],
            "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def gpu_other_config(name, device, overrides=None, steps=5, warmup=2):
    """Device-resident particle-steps/s of another BASELINE scene on this GPU (no reference arm)."""
    import torch

    from paper_1911_07913_b200 import Simulation, load_scene_file, sample_scene_particles

    path = os.path.join(ROOT, "scenes", name)
    sc = load_scene_file(path)
    p = sample_scene_particles(sc)
    sim = Simulation(sc, device=device)
    if overrides:
        sim.set_solver(**overrides)
    sim.set_particles(**p)
    stream = torch.cuda.ExternalStream(sim.stream(), device=device)
    for k in range(warmup):
        sim.advance_step(frame_end(sc.source, k))
    torch.cuda.synchronize(device)
    sim.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    outer = []
    e0.record(stream)
    for k in range(warmup, warmup + steps):
        outer.append(sim.advance_step(frame_end(sc.source, k))["outer_iterations"])
    e1.record(stream)
    torch.cuda.synchronize(device)
    ms = e0.elapsed_time(e1)
    prof = sim.profile_read()
    sim.close()
    n = p["x"].shape[0]
    cfg = workload_config(sc.source, path, n)
    cfg.update(overrides or {})
    return {"config": cfg, "value": n * steps / (ms / 1000.0), "unit": UNIT,
            "ms_per_step": ms / steps, "steps": steps, "warmup": warmup, "outer_iterations": outer,
            "phase_ms_per_step": {k: round(v["ms"] / steps, 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])
                                  if v["ms"] > 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scene", default=SCENE)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--mode", default="slabs", choices=["slabs", "replicas"], help="N > 1: slab-sharded or replicas")
    args = ap.parse_args()

    if args.impl == "reference":
        reference_arm(args)
        return

    rank, world, local_rank = dist_env()
    from paper_1911_07913_b200 import load_scene_file, sample_scene_particles

    sc = load_scene_file(args.scene)
    particles = sample_scene_particles(sc)
    n_particles = particles["x"].shape[0]
    config = workload_config(sc.source, args.scene, n_particles)

    import torch

    force_slabs = bool(os.environ.get("HOT_SHARD_FORCE")) and args.mode == "slabs"
    if world > 1 or force_slabs:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if "MASTER_ADDR" in os.environ:
            dist.init_process_group("nccl")
        else:  # HOT_SHARD_FORCE without a launcher: a one-rank group
            dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1)
    device = local_rank
    torch.cuda.set_device(device)
    from paper_1911_07913_b200 import Simulation

    sim = Simulation(sc, device=device)
    sim.set_particles(**particles)
    stream = torch.cuda.ExternalStream(sim.stream(), device=device)
    # HOT_SHARD_FORCE=1 (test hook): the slab path at one rank too (transport calls on one GPU)
    slabbed = (world > 1 or force_slabs) and args.mode == "slabs"
    slab_error = None
    if slabbed:
        from paper_1911_07913_b200 import slabs

        try:
            slabs.attach_nccl(sim)
        except Exception as e:  # no NCCL transport: say so in the line and run replicas
            slab_error = f"{type(e).__name__}: {e}"
            slabbed = False
    copies = 1 if slabbed else world  # scene copies processed per step by the whole job

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(device)

    # the clock sampler starts before the warm-up so that its start-up is over when timing begins
    clocks = ClockSampler(device)
    clocks.__enter__()
    atexit.register(clocks.__exit__)  # never leave nvidia-smi looping if a step raises
    step_no = 0
    for _ in range(args.warmup):
        sim.advance_step(frame_end(sc.source, step_no))
        step_no += 1
    sim.clear_diagnostics()

    # ---- device-resident timed region: K steps, nothing but the steps between the two events.
    # The per-phase profile is taken over the NEXT K steps of the same run (CUDA-event pairs on the
    # context stream, no extra kernel, no host synchronisation): with the profile inside the timed
    # region, about one run in eight lost 50-150 ms of a 300 ms region between phases (event
    # creation on the host; the phase sums were unchanged), so the headline carries no
    # instrumentation and the rooflines are measured live right after it.
    clocks.begin_timed()
    barrier()
    launches0 = sim.kernel_launches()
    outer = []
    try:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        marks = []
        for _ in range(args.steps):
            st = sim.advance_step(frame_end(sc.source, step_no))
            step_no += 1
            outer.append(st["outer_iterations"])
            if STEP_TIMES:
                marks.append(torch.cuda.Event(enable_timing=True))
                marks[-1].record(stream)
        ev1.record(stream)
        barrier()
        clocks.end_timed()
        if STEP_TIMES:
            ts = [ev0.elapsed_time(m) for m in marks]
            print("step_ms", [round(b - a, 2) for a, b in zip([0.0] + ts[:-1], ts)], file=sys.stderr)
    finally:
        clocks.__exit__()
    ms = ev0.elapsed_time(ev1)
    launches = sim.kernel_launches() - launches0
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{device}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = n_particles * copies * args.steps / (ms / 1000.0)
    shard = None
    if slabbed:
        si = slabs.shard_info(sim)
        shard = {"rows": [si["row_lo"], si["row_hi"]], "planes": [si["plane_lo"], si["plane_hi"]],
                 "halo_exchanges": si["halo_exchanges"], "row_gathers": si["gathers"]}

    # ---- end-to-end through the public API with host buffers (pinned)
    host = sim.particles()
    pinned = {}
    for k, v in list(host.items()):
        t = torch.empty(v.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = v
        pinned[k] = t.numpy()
    static = {}
    for k in ("mass", "volume", "material"):
        a = particles[k]
        t = torch.empty(a.shape, dtype=torch.int32 if k == "material" else torch.float64, pin_memory=True)
        t.numpy()[...] = a
        static[k] = t.numpy()
    h2d = sum(pinned[k].nbytes for k in ("x", "v", "F", "C")) + sum(a.nbytes for a in static.values())
    d2h = sum(pinned[k].nbytes for k in ("x", "v", "F", "C"))
    e2e_steps = max(1, args.steps)  # the same number of steps as the device-resident region (same step mix)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_outer = []
    for _ in range(e2e_steps):
        sim.set_particles(pinned["x"], pinned["v"], static["mass"], static["volume"], pinned["F"], pinned["C"],
                          static["material"])
        e2e_outer.append(sim.advance_step(frame_end(sc.source, step_no))["outer_iterations"])
        step_no += 1
        sim.particles(out=pinned)
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=f"cuda:{device}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = n_particles * copies * e2e_steps / (e2e_ms / 1000.0)

    # ---- profiled pass: the same number of steps, continuing the simulation (after the e2e steps,
    # which therefore follow the timed ones directly, as in every earlier round)
    sim.profile(True)
    pv0, pv1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pv0.record(stream)
    outer_prof = []
    for _ in range(args.steps):
        st = sim.advance_step(frame_end(sc.source, step_no))
        step_no += 1
        outer_prof.append(st["outer_iterations"])
    pv1.record(stream)
    barrier()
    ms_prof = pv0.elapsed_time(pv1)
    prof = sim.profile_read()
    sim.profile(False)

    # ---- rooflines (algorithmic bytes or flops / CUDA-event duration on the context stream)
    # `roofline` is the dominant kernel of the step: the level-0 assembly, bound by fp64 FMA
    # throughput (its algorithmic flops / the measured fp64 peak).  `roofline_hbm` is the
    # largest HBM-bound phase (the level-0 smoother in practice).
    peaks, peak_kind = measured_peaks()
    # The level-0 assembly is two kernels (by bins): k_bin_pairs, bound by the fp64 tensor pipe
    # (phase "assemble_pairs": all of the assembly's algorithmic flops), and k_row_gather, bound
    # by HBM (phase "assemble_rows": the pair sums read once, the rows and their column ids).
    # `roofline` is the one with the longer launch; both are reported, and `assembly` is the two
    # together against the fp64 peak.  (HOT_ASM=tiles: one kernel, phase "assemble_rows" in flops.)
    def tensor_line(ph, kernel):
        ach = ph["flops"] / (ph["ms"] / 1000.0) / 1e12
        return {"bound": "tensor", "pipe": "fp64 DMMA m8n8k4", "kernel": kernel, "achieved": ach,
                "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": ach / FP64_PEAK_TFLOPS,
                "traffic": TRAFFIC.get(kernel), "share_of_step": ph["ms"] / ms_prof, "launches": ph["launches"],
                "ms_per_launch": ph["ms"] / max(ph["launches"], 1),
                "flops_per_launch": ph["flops"] / max(ph["launches"], 1),
                "peak_kind": "measured fp64 tensor (DMMA) peak, the higher of DMMA/DFMA (profiles/r01_fp64_peak.json, tools/microbench/dmma.cu)"}

    def hbm_line(ph, kernel):
        ach = ph["bytes"] / (ph["ms"] / 1000.0) / 1e9
        return {"bound": "hbm", "kernel": kernel, "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "traffic": TRAFFIC.get(kernel), "peak_kind": peak_kind,
                "share_of_step": ph["ms"] / ms_prof, "launches": ph["launches"],
                "ms_per_launch": ph["ms"] / max(ph["launches"], 1),
                "bytes_per_launch": ph["bytes"] / max(ph["launches"], 1)}

    roofline = roofline_pairs = roofline_rows = assembly = None
    pa, ro = prof.get("assemble_pairs"), prof.get("assemble_rows")
    if pa and pa["ms"] > 0 and ro and ro["ms"] > 0 and ro["bytes"] > 0:
        roofline_pairs = tensor_line(pa, "k_bin_pairs")
        roofline_rows = hbm_line(ro, "k_row_gather")
        roofline = roofline_rows if roofline_rows["ms_per_launch"] >= roofline_pairs["ms_per_launch"] else roofline_pairs
        tot_ms = pa["ms"] + ro["ms"]
        ach = pa["flops"] / (tot_ms / 1000.0) / 1e12
        assembly = {"kernels": ["k_bin_pairs", "k_row_gather"], "ms_per_step": tot_ms / args.steps, "achieved": ach,
                    "unit": "TFLOP/s", "peak": FP64_PEAK_TFLOPS, "frac": ach / FP64_PEAK_TFLOPS,
                    "share_of_step": tot_ms / ms_prof}
    elif ro and ro["ms"] > 0 and ro["flops"] > 0:
        roofline = tensor_line(ro, "k_assemble_tiles")
    hbm_phases = {k: v for k, v in prof.items() if v["bytes"] > 0 and v["ms"] > 0 and
                  k in ("sgs_level0", "spmv_level0", "residual_restrict", "p2g_bc", "node_gradient", "g2p_strain_advect", "prolong",
                        "lbfgs_vectors", "assemble_rows")}
    smoothers = {k: v for k, v in hbm_phases.items() if k != "assemble_rows"}  # roofline_hbm: outside the assembly
    top = max(smoothers, key=lambda k: smoothers[k]["ms"]) if smoothers else None
    # every HBM-class phase of the step: algorithmic GB/s and fraction of the measured peak
    hbm_all = {k: {"GBps": round(v["bytes"] / (v["ms"] / 1000.0) / 1e9, 1),
                   "frac": round(v["bytes"] / (v["ms"] / 1000.0) / 1e9 / peaks["hbm_gbs"], 3),
                   "ms_per_step": round(v["ms"] / args.steps, 3)} for k, v in hbm_phases.items()}
    roofline_hbm = None
    if top:
        ph = hbm_phases[top]
        achieved = ph["bytes"] / (ph["ms"] / 1000.0) / 1e9
        roofline_hbm = {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": achieved / peaks["hbm_gbs"], "traffic": TRAFFIC.get(top), "peak_kind": peak_kind,
                        "share_of_step": ph["ms"] / ms_prof, "launches": ph["launches"],
                        "bytes_per_launch": ph["bytes"] / max(ph["launches"], 1)}

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # 1 thread (the reference default, cli.cpp:26) on a bounded sample: the first 0.05 m of
        # all four bars (driven end + free material), the oracle's own sampling, 1 step from t=0
        x_cut = 0.05
        r = oracle_run(sc.source, 1, 0, 1, keep=lambda x: x[:, 0] < x_cut)
        cpu_baseline = {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "port",
                        "sample": f"{r['particles']} particles (x < {x_cut} m slab of all four bars), 1 step from t=0, "
                                  f"oracle port of hotmpm::advance_step, 1 thread (reference default), "
                                  f"{r['seconds']:.1f} s, outer iterations {r['outer']}"}

    other = None
    if rank == 0 and world == 1 and not args.no_other_configs:
        sim.close()
        other = {}
        for name, ov in OTHER_SCENES:
            key = name + "".join(f"@{k}={v}" for k, v in ov.items())
            try:
                other[key] = gpu_other_config(name, device, ov)
            except Exception as e:  # reported, never fatal to the headline
                other[key] = {"error": f"{type(e).__name__}: {e}"}

    if rank == 0:
        phases = {k: round(v["ms"] / args.steps, 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])
                  if v["ms"] > 0}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if slabbed else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded scene sampling, reference schema)",
                "config": config,
                "parallelism": (f"slabs x{world} (axis-0 lattice planes, NCCL)" if slabbed else
                                f"replicas x{world}" + (f" (slab transport failed: {slab_error})" if slab_error else "")
                                if world > 1 else "single GPU"),
                "outer_iterations": outer, "phase_ms_per_step": phases,
                "profiled_pass": {"steps": args.steps, "ms_per_step": ms_prof / args.steps, "outer_iterations": outer_prof,
                                  "note": "phase_ms_per_step, the rooflines and hbm_phases: K more steps after the timed and the e2e steps"},
                "rank0_shard": shard,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                        "steps": e2e_steps, "outer_iterations": e2e_outer},
                "gpu_launches": int(launches), "roofline": roofline, "roofline_assembly_pairs": roofline_pairs,
                "roofline_assembly_rows": roofline_rows, "assembly": assembly, "roofline_hbm": roofline_hbm,
                "hbm_phases": hbm_all,
                "cpu_baseline": cpu_baseline, "other_configs": other,
                "clocks": clocks.summary()}
        print(json.dumps(line))
    sim.close()
    if world > 1 or force_slabs:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
