"""B200-native HOT (Hierarchical Optimization Time Integration) implicit-MPM step.

The hot path (one implicit-Euler MPM step: binning + APIC P2G, the HOT solve = L-BFGS
initialised by a Galerkin-multigrid V-cycle, G2P + strain update + advection) runs as
hand-written sm_100a CUDA kernels in ``lib/libhotb200.so`` behind the C-ABI in
``include/hot_c_api.h``.  This package is the Python host surface mirroring the reference's
scene / simulation API (see ``sim.Simulation``).
"""
from .scene import ParseError, SceneConfig, load_scene_file, parse_scene  # noqa: F401
from .capi import (CudaError, DomainError, HotError, InvalidArgument, LogicError, SolverFailure,  # noqa: F401
                   Unsupported, sample_scene_particles)
from .sim import Simulation  # noqa: F401

__all__ = ["ParseError", "SceneConfig", "load_scene_file", "parse_scene", "Simulation", "sample_scene_particles",
           "SolverFailure", "InvalidArgument", "LogicError", "DomainError", "CudaError", "Unsupported", "HotError"]
