"""CPU-side checks of the product boundary: libhotb200.so loads and exports every symbol the
header declares; host-side sampling is byte-identical to the oracle (libstdc++ RNG stream,
simulation.hpp:94-254); the scene schema is as strict as scene.cpp; no device -> a clean
CUDA error, never a CPU fallback."""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_1911_07913_b200 import ParseError, capi, load_scene_file, parse_scene, sample_scene_particles

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "hot_c_api.h")).read()
    return sorted(set(re.findall(r"\b(hot_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = ctypes.CDLL(capi.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(capi.EXPORTS)
    assert capi.lib().hot_version() == 2


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {capi.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(ROOT, "scenes", "*.json"))))
def test_scene_sampling_matches_oracle_bitwise(path):
    sc = load_scene_file(path)
    p = sample_scene_particles(sc)  # every scene, the 4.0M-particle snow included
    o = O.Oracle(sc.dim)
    o.set_scene(sc.source)
    assert o.sample_scene() == p["x"].shape[0]
    q = o.get_particles()
    for k in ("x", "v", "mass", "volume", "F", "C", "material"):
        assert np.array_equal(p[k], q[k]), k


def test_sampling_2d_matches_oracle():
    sc = parse_scene("""{"dim": 2, "dx": 0.01, "seed": 13, "domain": {"min": [0, 0], "max": [0.64, 0.64]},
      "materials": [{"density": 2700.0, "youngs": 2.1e5, "poisson": 0.33}],
      "objects": [{"shape": {"kind": "sphere", "center": [0.32, 0.40], "radius": 0.09}, "material": 0,
                   "velocity": [0.0, -2.0], "initial_deformation": {"kind": "random_diagonal", "lo": 0.9, "hi": 1.1}}]}""")
    p = sample_scene_particles(sc)
    o = O.Oracle(2)
    o.set_scene(sc.source)
    o.sample_scene()
    q = o.get_particles()
    for k in ("x", "v", "F", "material"):
        assert np.array_equal(p[k], q[k]), k


def test_poisson_sampling_matches_oracle():
    sc = parse_scene("""{"dim": 3, "dx": 0.05, "seed": 3, "ppc": 2, "sampling": "poisson",
      "domain": {"min": [0, 0, 0], "max": [1, 1, 1]},
      "materials": [{"density": 1000.0, "youngs": 1e5, "poisson": 0.3}],
      "objects": [{"shape": {"kind": "sphere", "center": [0.5, 0.5, 0.5], "radius": 0.2}, "material": 0}]}""")
    p = sample_scene_particles(sc)
    o = O.Oracle(3)
    o.set_scene(sc.source)
    o.sample_scene()
    assert np.array_equal(p["x"], o.get_particles()["x"])


BASE = """{"dx": 0.01, "domain": {"min": [0, 0], "max": [1, 1]},
  "materials": [{"density": 1000.0, "youngs": 1e5, "poisson": 0.3}],
  "objects": [{"shape": {"kind": "box", "min": [0.1, 0.1], "max": [0.2, 0.2]}, "material": 0}] %s}"""


@pytest.mark.parametrize("extra,needle", [
    (', "bogus": 1', "unknown key 'bogus'"),
    (', "dim": 4', "scene.dim"),
    (', "levels": 0', "scene.levels"),
    (', "embedding": "cubic"', "scene.embedding"),
    (', "sampling": "grid"', "scene.sampling"),
    (', "colliders": [{"shape": {"kind": "half_space", "point": [0, 0]}}]', "missing required key 'normal'"),
])
def test_scene_schema_is_strict(extra, needle):  # scene.cpp:15-22, 190-294
    with pytest.raises(ParseError) as e:
        parse_scene(BASE % extra)
    assert needle in str(e.value)


def test_scene_objects_must_be_in_domain_and_reference_materials():
    with pytest.raises(ParseError):
        parse_scene(BASE.replace('"max": [0.2, 0.2]', '"max": [1.2, 0.2]') % "")
    with pytest.raises(ParseError):
        parse_scene(BASE.replace('"material": 0', '"material": 3') % "")
    with pytest.raises(ParseError):
        parse_scene(BASE.replace('"kind": "box", "min": [0.1, 0.1], "max": [0.2, 0.2]',
                                 '"kind": "half_space", "point": [0, 0], "normal": [0, 1]') % "")


def test_no_device_is_a_clean_error():
    if capi.lib().hot_device_count() > 0:
        pytest.skip("a GPU is present")
    from paper_1911_07913_b200 import CudaError, Simulation
    with pytest.raises(CudaError):
        Simulation(load_scene_file(os.path.join(ROOT, "scenes", "cfg1_cube.json")))
