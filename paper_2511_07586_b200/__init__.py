"""B200-native Monte Carlo SBR radar-cross-section estimator (arXiv 2511.07586 hot path).

Drop-in for the reference CPU solver ``mcsbr::estimate``: host-side scene I/O
and solver types mirror the reference headers; all per-ray work runs in the
hand-written sm_100a CUDA kernels of ``libmcsbr_gpu.so`` (C ABI in
include/mcsbr_gpu.h).
"""
from .geometry import (SceneData, SceneError, Material, load_scene, load_scene_files, airframe,
                       builtin_scene, builtin_scene_names, make_builtin_scene, dihedral_grid,
                       coated_sphere, MeshBuilder)
from .solver import (Scene, Excitation, monostatic_excitation, bistatic_excitation, McConfig,
                     RouletteConfig, BranchStrategy, RngMode, Reduction, DetConfig, DetResult, solve, SweepResult, RunStats, McResult,
                     LaunchRect, StrataGrid, DomainError, estimate, estimate_batch, launch_plan,
                     launch_rect, rcs_m2, VV, HH, VH, HV, K_SPEED_OF_LIGHT)
from . import signal
from .signal import Window, RangeProfile, IsarImage, SignalError, range_profile, isar

__all__ = [
    "SceneData", "SceneError", "Material", "load_scene", "load_scene_files", "airframe", "builtin_scene",
    "builtin_scene_names", "make_builtin_scene", "dihedral_grid", "coated_sphere", "MeshBuilder",
    "Scene", "Excitation", "monostatic_excitation", "bistatic_excitation", "McConfig",
    "RouletteConfig", "BranchStrategy", "RngMode", "Reduction", "DetConfig", "DetResult", "solve", "SweepResult", "RunStats", "McResult",
    "LaunchRect", "StrataGrid", "DomainError", "estimate", "estimate_batch", "launch_plan",
    "launch_rect", "rcs_m2", "VV", "HH", "VH", "HV", "K_SPEED_OF_LIGHT",
    "signal", "Window", "RangeProfile", "IsarImage", "SignalError", "range_profile", "isar",
]
