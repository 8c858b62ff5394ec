"""ctypes mirror of include/mcsbr_gpu.h and the loader for the CUDA library.

The product library is ``paper_2511_07586_b200/libmcsbr_gpu.so`` (built in-tree
by ``__graft_entry__.build()`` / ``python -m paper_2511_07586_b200.build``).
There is no CPU fallback: if the library is missing the import of the
compute entry points raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCSBR_GPU_LIB") or os.path.join(_HERE, "libmcsbr_gpu.so")

MCSBR_OK = 0
MCSBR_EINVAL = -1
MCSBR_ENOMEM = -2
MCSBR_ECUDA = -3
MCSBR_ESCENE = -4
MCSBR_EDEVICE = -5

MCSBR_BRANCH_FIFTY_FIFTY = 0
MCSBR_BRANCH_FRESNEL = 1
MCSBR_RNG_REFERENCE = 0
MCSBR_RNG_PHILOX = 1
MCSBR_REDUCE_FAST = 0
MCSBR_REDUCE_EXACT = 1
MCSBR_EXACT_LIMBS = 4
MCSBR_MAX_BOUNCE_LIMIT = 64
MCSBR_COUNTER_WORDS = 256


class Triangle(C.Structure):
    _fields_ = [
        ("v0", C.c_uint32), ("v1", C.c_uint32), ("v2", C.c_uint32), ("_pad0", C.c_uint32),
        ("normal", C.c_double * 3),
        ("front_material", C.c_uint16), ("back_material", C.c_uint16),
        ("exterior_facing", C.c_uint8), ("_pad1", C.c_uint8 * 3),
    ]


TRIANGLE_DTYPE = np.dtype(
    {
        "names": ["v0", "v1", "v2", "_pad0", "normal", "front_material", "back_material",
                  "exterior_facing", "_pad1"],
        "formats": ["<u4", "<u4", "<u4", "<u4", ("<f8", 3), "<u2", "<u2", "u1", ("u1", 3)],
        "offsets": [0, 4, 8, 12, 16, 40, 42, 44, 45],
        "itemsize": 48,
    }
)


class Material(C.Structure):
    _fields_ = [("eps_r", C.c_double), ("mu_r", C.c_double), ("is_pec", C.c_uint8),
                ("_pad", C.c_uint8 * 7)]


MATERIAL_DTYPE = np.dtype(
    {"names": ["eps_r", "mu_r", "is_pec", "_pad"], "formats": ["<f8", "<f8", "u1", ("u1", 7)],
     "offsets": [0, 8, 16, 17], "itemsize": 24}
)


class Excitation(C.Structure):
    _fields_ = [
        ("k_inc", C.c_double * 3), ("pol_v", C.c_double * 3), ("pol_h", C.c_double * 3),
        ("k_scatter", C.c_double * 3), ("rx_v", C.c_double * 3), ("rx_h", C.c_double * 3),
        ("occlusion_enabled", C.c_uint8), ("_pad", C.c_uint8 * 7),
    ]


class Incidence(C.Structure):
    _fields_ = [("k_inc", C.c_double * 3), ("pol_v", C.c_double * 3), ("pol_h", C.c_double * 3),
                ("strata_per_wavelength", C.c_double)]


class Receiver(C.Structure):
    _fields_ = [("k_scatter", C.c_double * 3), ("rx_v", C.c_double * 3), ("rx_h", C.c_double * 3)]


class McConfigC(C.Structure):
    _fields_ = [
        ("strata_per_wavelength", C.c_double),
        ("samples_per_stratum", C.c_int32),
        ("branch_strategy", C.c_int32),
        ("roulette_enabled", C.c_int32),
        ("roulette_min_bounce", C.c_int32),
        ("roulette_q", C.c_double),
        ("max_bounce", C.c_int32),
        ("jitter", C.c_int32),
        ("seed", C.c_uint64),
        ("reference_wavelength", C.c_double),
        ("launch_padding", C.c_double),
        ("p_min", C.c_double),
        ("block_size", C.c_int32),
        ("rng_mode", C.c_int32),
        ("reduction", C.c_int32),
        ("parity_fp64_refine", C.c_int32),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("rays_launched", C.c_uint64), ("segments_traced", C.c_uint64),
        ("contributions", C.c_uint64), ("grazing_kills", C.c_uint64), ("cap_kills", C.c_uint64),
        ("occlusion_queries", C.c_uint64), ("peak_live_state_bytes", C.c_uint64),
        ("state_bytes_per_ray", C.c_uint64), ("block_size", C.c_uint64),
        ("n_rounds", C.c_uint32), ("_pad", C.c_uint32),
        ("rays_per_bounce", C.c_uint64 * MCSBR_MAX_BOUNCE_LIMIT),
        ("roulette_candidates", C.c_uint64 * MCSBR_MAX_BOUNCE_LIMIT),
        ("roulette_survivors", C.c_uint64 * MCSBR_MAX_BOUNCE_LIMIT),
        ("wall_ms", C.c_double), ("kernel_ms", C.c_double),
        ("forced_stack_bytes", C.c_uint64), ("device_stack_bytes", C.c_uint64),
        ("culled_launch_rays", C.c_uint64),
    ]


class DetConfigC(C.Structure):
    _fields_ = [
        ("rays_per_wavelength", C.c_double),
        ("max_bounce", C.c_int32),
        ("force_stack_accounting", C.c_int32),
        ("amplitude_cutoff", C.c_double),
        ("launch_padding", C.c_double),
        ("reference_wavelength", C.c_double),
        ("block_size", C.c_int32),
        ("_pad", C.c_int32),
    ]


CONTRIBUTION_DTYPE = np.dtype(
    {
        "names": ["a_j", "a_m", "phi_total", "exit_point", "bounce", "_pad", "order_key"],
        "formats": [("<f8", (2, 3, 2)), ("<f8", (2, 3, 2)), "<f8", ("<f8", 3), "<i4", "<i4", "<u8"],
        "offsets": [0, 96, 192, 200, 224, 228, 232],
        "itemsize": 240,
    }
)


class LaunchPlan(C.Structure):
    _fields_ = [
        ("center", C.c_double * 3), ("u_axis", C.c_double * 3), ("v_axis", C.c_double * 3),
        ("half_u", C.c_double), ("half_v", C.c_double), ("nu", C.c_int32), ("nv", C.c_int32),
        ("cell_area", C.c_double), ("entries", C.c_uint64),
    ]


assert C.sizeof(Triangle) == 48 and TRIANGLE_DTYPE.itemsize == 48
assert C.sizeof(Material) == 24
assert C.sizeof(Excitation) == 152
assert CONTRIBUTION_DTYPE.itemsize == 240


def ptr(a: np.ndarray | None, ctype=C.c_void_p):
    """Pointer to a C-contiguous numpy array (or NULL)."""
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(ctype)


_DP = C.POINTER(C.c_double)
_U32P = C.POINTER(C.c_uint32)
_U64P = C.POINTER(C.c_uint64)

# exported symbol -> (restype, argtypes); the CPU test suite checks that the
# built library exports exactly these (include/mcsbr_gpu.h).
SIGNATURES = {
    "mcsbr_gpu_last_error": (C.c_char_p, []),
    "mcsbr_gpu_abi_version": (C.c_int, []),
    "mcsbr_gpu_default_config": (None, [C.POINTER(McConfigC)]),
    "mcsbr_gpu_validate_config": (C.c_int, [C.POINTER(McConfigC)]),
    "mcsbr_gpu_scene_create": (
        C.c_int,
        [_DP, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, _DP, C.c_int,
         C.POINTER(C.c_void_p)],
    ),
    "mcsbr_gpu_scene_destroy": (None, [C.c_void_p]),
    "mcsbr_gpu_scene_create_multi": (
        C.c_int,
        [_DP, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, _DP, C.POINTER(C.c_int), C.c_int,
         C.POINTER(C.c_void_p)],
    ),
    "mcsbr_gpu_scene_devices": (C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    "mcsbr_gpu_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "mcsbr_gpu_scene_bounds": (C.c_int, [C.c_void_p, _DP, _DP, _DP]),
    "mcsbr_gpu_scene_bvh_info": (C.c_int, [C.c_void_p, _U32P, _U32P, _U32P, _DP]),
    "mcsbr_gpu_launch_plan": (
        C.c_int, [C.c_void_p, _DP, C.c_double, C.c_double, C.c_double, C.c_int32,
                  C.POINTER(LaunchPlan)],
    ),
    "mcsbr_gpu_intersect": (
        C.c_int, [C.c_void_p, _DP, _DP, _DP, C.c_uint32, C.c_int, _DP, _U32P],
    ),
    "mcsbr_gpu_intersect_device": (
        C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_int, C.c_void_p,
                  C.c_void_p, C.c_void_p],
    ),
    "mcsbr_gpu_estimate": (
        C.c_int,
        [C.c_void_p, C.POINTER(Excitation), _DP, C.c_uint32, C.POINTER(McConfigC), C.c_int, _DP,
         C.POINTER(Stats), C.c_void_p, C.c_uint64, _U64P],
    ),
    "mcsbr_gpu_default_det_config": (None, [C.POINTER(DetConfigC)]),
    "mcsbr_gpu_validate_det_config": (C.c_int, [C.POINTER(DetConfigC)]),
    "mcsbr_gpu_solve": (
        C.c_int,
        [C.c_void_p, C.POINTER(Excitation), _DP, C.c_uint32, C.POINTER(DetConfigC), C.c_int, _DP,
         C.POINTER(Stats), C.c_void_p, C.c_uint64, _U64P],
    ),
    "mcsbr_gpu_estimate_batch": (
        C.c_int,
        [C.c_void_p, C.POINTER(Incidence), C.c_uint32, C.POINTER(Receiver), C.c_uint32, C.c_int,
         _DP, C.c_uint32, C.POINTER(McConfigC), _DP, C.POINTER(Stats)],
    ),
    "mcsbr_gpu_trace_device": (
        C.c_int,
        [C.c_void_p, C.POINTER(Incidence), C.c_uint32, C.POINTER(Receiver), C.c_uint32, C.c_int,
         _DP, C.c_uint32, C.POINTER(McConfigC), C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
         C.c_void_p],
    ),
    "mcsbr_gpu_finalize": (C.c_int, [_DP, C.c_uint32, _DP, C.c_uint32, _DP]),
    "mcsbr_gpu_finalize_exact": (C.c_int, [C.POINTER(C.c_int64), C.c_uint32, _DP, C.c_uint32, _DP]),
    "mcsbr_gpu_decode_counters": (C.c_int, [_U64P, C.POINTER(Stats)]),
    "mcsbr_gpu_path_log": (
        C.c_int,
        [C.c_void_p, C.POINTER(Excitation), _DP, C.c_uint32, C.POINTER(McConfigC), C.c_uint64,
         C.c_uint32, _U32P, C.POINTER(C.c_uint8), _U64P],
    ),
    "mcsbr_gpu_range_profile": (
        C.c_int, [_DP, _DP, C.c_uint32, C.c_int, C.c_int, _DP, _DP, _DP],
    ),
    "mcsbr_gpu_isar": (
        C.c_int, [_DP, _DP, C.c_uint32, _DP, C.c_uint32, C.c_int, C.c_int, C.c_double, _DP, _DP, _DP,
                  _DP],
    ),
    "mcsbr_gpu_last_launch_count": (C.c_uint64, []),
    "mcsbr_gpu_kernel_timing": (None, [C.c_int]),
    "mcsbr_gpu_kernel_times": (C.c_int, [_DP, _U64P, _DP, _U64P]),
}

_lib = None


class McsbrError(RuntimeError):
    """Error raised from a non-zero status of the C ABI."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def lib() -> C.CDLL:
    """Load libmcsbr_gpu.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2511_07586_b200.build` "
                "(there is no CPU fallback)"
            )
        L = C.CDLL(LIB_PATH)
        lenient = os.environ.get("MCSBR_ABI_LENIENT") == "1"  # A/B tooling: older library builds
        for name, (res, args) in SIGNATURES.items():
            if lenient and not hasattr(L, name):
                continue
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(code: int) -> None:
    if code != 0:
        msg = lib().mcsbr_gpu_last_error()
        raise McsbrError(code, msg.decode() if msg else f"mcsbr error {code}")
