"""Output formats (io.cpp:47-123) restated in paper_1911_07913_b200.io: byte layout, text
formatting, round trips.  CPU only."""
import struct

import numpy as np
import pytest

from paper_1911_07913_b200 import io


def test_snapshot_layout_and_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    pos = rng.standard_normal((5, 3))
    vel = rng.standard_normal((5, 3))
    p = tmp_path / "f.bin"
    io.write_snapshot(p, 3, pos, vel)
    buf = p.read_bytes()
    assert buf[:4] == b"HOTP"
    assert struct.unpack_from("<IIQ", buf, 4) == (1, 3, 5)  # version, dim, count (io.hpp:11-20)
    assert len(buf) == 20 + 16 * 15
    assert np.array_equal(np.frombuffer(buf, "<f8", 15, 20), pos.reshape(-1))  # positions, then velocities
    assert np.array_equal(np.frombuffer(buf, "<f8", 15, 20 + 8 * 15), vel.reshape(-1))
    s = io.read_snapshot(p)
    assert (s["version"], s["dim"], s["count"]) == (1, 3, 5)
    assert np.array_equal(s["positions"], pos.reshape(-1)) and np.array_equal(s["velocities"], vel.reshape(-1))


def test_snapshot_errors(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"XXXX" + bytes(16))
    with pytest.raises(RuntimeError, match="bad header"):
        io.read_snapshot(p)
    p.write_bytes(b"HOTP" + struct.pack("<IIQ", 1, 3, 10) + bytes(8))
    with pytest.raises(RuntimeError, match="truncated"):
        io.read_snapshot(p)
    with pytest.raises(RuntimeError, match="cannot open"):
        io.read_snapshot(tmp_path / "missing.bin")
    with pytest.raises(ValueError):
        io.write_snapshot(tmp_path / "x.bin", 3, np.zeros(4), np.zeros(4))


def test_positions_text_is_precision_17(tmp_path):
    # C++ ostream precision(17), default float field == %.17g
    pos = np.array([[0.1, 100.0, -0.0], [1e-5, 2.5e300, 1.0 / 3.0]])
    p = tmp_path / "f.txt"
    io.write_positions_text(p, 3, pos)
    assert p.read_text() == ("0.10000000000000001 100 -0\n"
                             "1.0000000000000001e-05 2.5000000000000001e+300 0.33333333333333331\n")


def test_diagnostics_csv(tmp_path):
    rec = dict(frame=np.array([1, 1]), step=np.array([0, 0]), outer_iteration=np.array([1, 2]),
               scaled_residual=np.array([0.5, 1e-6]), energy=np.array([-1.25, -1.5]),
               step_length=np.array([1.0, 0.5]), inner_iterations=np.array([3, 4]), work_units=np.array([3, 7]),
               wall_ms=np.array([12.5, 20.25]))
    p = tmp_path / "d.csv"
    io.write_diagnostics_csv(p, rec, zero_wall_time=True)
    assert p.read_text() == (io.DIAG_HEADER + "1,0,1,0.5,-1.25,1,3,3,0\n"
                             "1,0,2,9.9999999999999995e-07,-1.5,0.5,4,7,0\n")
    io.write_diagnostics_csv(p, rec, zero_wall_time=False)
    assert p.read_text().splitlines()[1].endswith(",12.5")


@pytest.mark.skipif(__import__("shutil").which("g++") is None, reason="needs g++")
def test_text_formatting_matches_cpp_ostream(tmp_path):
    """The reference writes with std::ostringstream precision(17) (io.cpp:89-90, 108-109):
    compare the Python formatting with that stream on random and edge-case values."""
    import subprocess

    src = tmp_path / "fmt.cpp"
    src.write_text("#include <iostream>\n#include <sstream>\n#include <cstdio>\n"
                   "int main(){ std::ostringstream o; o.precision(17); double v;"
                   " while (std::fread(&v, 8, 1, stdin) == 1) o << v << '\\n'; std::cout << o.str(); }\n")
    exe = tmp_path / "fmt"
    subprocess.run(["g++", "-O0", "-o", str(exe), str(src)], check=True)
    rng = np.random.default_rng(3)
    vals = np.concatenate([rng.standard_normal(200) * 10.0 ** rng.integers(-300, 300, 200),
                           [0.0, -0.0, 1.0, 0.1, 1e-5, 123456789.0, 1e22, 5e-324, np.inf, -np.inf]])
    out = subprocess.run([str(exe)], input=vals.astype("<f8").tobytes(), capture_output=True, check=True).stdout
    assert out.decode().splitlines() == [io._g17(v) for v in vals]


def test_kernel_sweep_particle_sets():
    """tools/kernel_sweep.py (BASELINE config 5): 8 ppc in the ball, random F with singular
    values in [0.5, 2]."""
    import importlib.util
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "kernel_sweep.py")
    spec = importlib.util.spec_from_file_location("kernel_sweep", path)
    ks = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ks)
    p = ks.particles_for(16)
    n = p["x"].shape[0]
    assert n % 8 == 0 and n > 0
    assert np.all(np.linalg.norm(p["x"] - 0.5, axis=1) < 0.45 + 2.0 / 16)
    s = np.linalg.svd(p["F"], compute_uv=False)
    assert s.min() >= 0.5 - 1e-12 and s.max() <= 2.0 + 1e-12
    R = ks.rotations(np.random.default_rng(0), 50)
    assert np.allclose(np.einsum("nij,nkj->nik", R, R), np.eye(3)) and np.allclose(np.linalg.det(R), 1.0)


def test_bench_reference_arm_is_oracle_only_and_same_config():
    """bench.py --impl reference: the oracle on the full scene, sampled by the oracle itself; the
    product package is never imported; its config equals the GPU arm's (same workload dict)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    scene = os.path.join(root, "scenes", "cfg1_cube.json")
    code = f"""
import sys, json, types
sys.argv = ["bench.py", "--impl", "reference", "--scene", {scene!r}, "--steps", "1", "--warmup", "0"]
sys.path.insert(0, {root!r})
import bench
bench.main()
print(json.dumps({{"product_loaded": any(m.startswith("paper_1911_07913_b200") for m in sys.modules)}}))
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    ref, flag = lines[0], lines[1]
    assert flag["product_loaded"] is False
    assert ref["impl"] == "reference" and ref["steps"] == 1 and ref["cpu_baseline"]["kind"] == "port"
    from paper_1911_07913_b200 import load_scene_file, sample_scene_particles

    sys.path.insert(0, root)
    import bench

    sc = load_scene_file(scene)
    n = sample_scene_particles(sc)["x"].shape[0]
    assert ref["config"] == json.loads(json.dumps(bench.workload_config(sc.source, scene, n)))
