"""TEST INFRASTRUCTURE ONLY: ctypes access to the two CPU checkers.

* ``ref()``    -> oracle/_ref/libmcsbr_ref.so: the UNMODIFIED reference C++
  (proj/src) behind the extern "C" shim oracle/ref_shim.cpp.  Built here by
  ``make -C oracle ref`` (needs /root/reference); the built .so travels to the
  GPU box with the repo snapshot.
* ``port()``   -> oracle/libmcsbr_oracle.so: our C restatement
  (oracle/mcsbr_oracle.c), pinned bit-for-bit against ``ref()``.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product
(paper_2511_07586_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2511_07586_b200 import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmcsbr_ref.so")
# the reference with its solver TUs swapped for the product's drop-in
# (paper_2511_07586_b200/dropin/solver_b200.cpp): `make -C oracle dropin`
DROPIN_SO = os.path.join(HERE, "_ref", "libmcsbr_ref_b200.so")
PORT_SO = os.path.join(HERE, "libmcsbr_oracle.so")

_DP = C.POINTER(C.c_double)
_ref = None
_dropin = None
_port = None


def build(ref_too: bool = True) -> None:
    """Compile the C restatement and, when /root/reference exists, the reference
    and the drop-in integration library (needs the product library built first)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref_too and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref", "dropin"], check=True)


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
        _ref = _bind_shim(C.CDLL(REF_SO))
    return _ref


def have_dropin() -> bool:
    return os.path.exists(DROPIN_SO)


def dropin() -> C.CDLL:
    """The reference's own code with estimate()/solve() on the GPU (f3)."""
    global _dropin
    if _dropin is None:
        if not os.path.exists(DROPIN_SO):
            raise FileNotFoundError(f"{DROPIN_SO} not built (make -C oracle dropin)")
        _dropin = _bind_shim(C.CDLL(DROPIN_SO))
    return _dropin


def _bind_shim(L: C.CDLL) -> C.CDLL:
    L.ref_last_error.restype = C.c_char_p
    L.ref_counter_hash.restype = C.c_uint64
    L.ref_counter_hash.argtypes = [C.c_uint64] * 5
    L.ref_counter_uniform.restype = C.c_double
    L.ref_counter_uniform.argtypes = [C.c_uint64] * 5
    L.ref_fresnel.argtypes = [C.c_double, C.c_double, C.c_double, _DP]
    L.ref_sp_basis.argtypes = [_DP, _DP, C.c_double, C.c_double, _DP]
    L.ref_interface_transform.argtypes = [_DP, C.c_int, _DP, _DP, _DP]
    L.ref_branch_outcomes.argtypes = [_DP, _DP, _DP]
    L.ref_meca_currents.argtypes = [_DP, _DP, _DP, C.c_int, _DP]
    L.ref_meca_currents_hot.argtypes = [_DP, _DP, _DP, C.c_int, _DP, _DP, C.c_double, _DP]
    L.ref_evaluate_sweep.argtypes = [C.c_void_p, C.c_uint64, _DP, C.c_uint32, _DP, _DP, _DP, _DP]
    L.ref_monostatic_excitation.argtypes = [C.c_double, C.c_double, C.POINTER(A.Excitation)]
    L.ref_bistatic_excitation.argtypes = [C.c_double] * 4 + [C.POINTER(A.Excitation)]
    L.ref_scene_load.restype = C.c_void_p
    L.ref_scene_load.argtypes = [C.c_char_p, C.c_char_p]
    L.ref_scene_builtin.restype = C.c_void_p
    L.ref_scene_builtin.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), _DP, C.c_int]
    L.ref_builtin_text.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), _DP, C.c_int,
                                   C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64,
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    L.ref_scene_free.argtypes = [C.c_void_p]
    L.ref_scene_sizes.argtypes = [C.c_void_p] + [C.POINTER(C.c_uint32)] * 3
    L.ref_scene_export.argtypes = [C.c_void_p, _DP, C.c_void_p, C.c_void_p, _DP]
    L.ref_scene_from_arrays.restype = C.c_void_p
    L.ref_scene_from_arrays.argtypes = [_DP, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p,
                                        C.c_uint32]
    L.ref_intersect.argtypes = [C.c_void_p, _DP, _DP, _DP, C.c_uint64, C.c_int, _DP]
    L.ref_launch_rect.argtypes = [C.c_void_p, _DP, C.c_double, _DP]
    L.ref_build_strata.argtypes = [_DP, C.c_double, C.c_double, C.POINTER(C.c_int32), _DP]
    L.ref_sample_stratum.argtypes = [_DP, C.c_int32, C.c_int32, C.c_uint32, C.c_uint32,
                                     C.c_uint64, C.c_int, _DP]
    L.ref_estimate.argtypes = [C.c_void_p, C.POINTER(A.Excitation), _DP, C.c_uint32,
                               C.POINTER(A.McConfigC), C.c_int, _DP, C.POINTER(A.Stats),
                               C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
    L.ref_solve.argtypes = [C.c_void_p, C.POINTER(A.Excitation), _DP, C.c_uint32,
                            C.POINTER(A.DetConfigC), C.c_int, _DP, C.POINTER(A.Stats),
                            C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
    L.ref_sweep_csv.argtypes = [_DP, _DP, C.c_uint32, C.c_uint64, C.c_char_p, C.c_char_p,
                                C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64)]
    L.ref_stats_json.argtypes = [C.POINTER(A.Stats), C.c_char_p, C.c_char_p, C.c_uint64,
                                 C.POINTER(C.c_uint64)]
    L.ref_parse_config.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64)]
    L.ref_run_command.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.c_int,
                                  C.c_uint64]
    L.ref_slab_reflection.argtypes = [_DP, _DP, C.c_int, C.c_double, C.c_int, _DP]
    L.ref_range_profile.argtypes = [_DP, _DP, C.c_uint32, C.c_int, C.c_int, _DP, _DP, _DP]
    L.ref_isar.argtypes = [_DP, _DP, C.c_uint32, _DP, C.c_uint32, C.c_int, C.c_int, C.c_double,
                           _DP, _DP, _DP, _DP]
    L.ref_plate_rcs.restype = C.c_double
    L.ref_plate_rcs.argtypes = [C.c_double] * 3
    L.ref_sphere_go_rcs.restype = C.c_double
    L.ref_sphere_go_rcs.argtypes = [C.c_double]
    return L


def port() -> C.CDLL:
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build(ref_too=False)
        L = C.CDLL(PORT_SO)
        L.orc_last_error.restype = C.c_char_p
        L.orc_counter_hash.restype = C.c_uint64
        L.orc_counter_hash.argtypes = [C.c_uint64] * 5
        L.orc_counter_uniform.restype = C.c_double
        L.orc_counter_uniform.argtypes = [C.c_uint64] * 5
        L.orc_fresnel.argtypes = [C.c_double, C.c_double, C.c_double, _DP]
        L.orc_sp_basis.argtypes = [_DP, _DP, C.c_double, C.c_double, _DP]
        L.orc_interface_transform.argtypes = [_DP, C.c_int, _DP, _DP, _DP]
        L.orc_branch_outcomes.argtypes = [_DP, _DP, _DP]
        L.orc_meca_currents.argtypes = [_DP, _DP, _DP, C.c_int, _DP]
        L.orc_cdiv.argtypes = [_DP, _DP, _DP]
        L.orc_scene_create.restype = C.c_void_p
        L.orc_scene_create.argtypes = [_DP, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p,
                                       C.c_uint32]
        L.orc_scene_free.argtypes = [C.c_void_p]
        L.orc_scene_bounds.argtypes = [C.c_void_p, _DP]
        L.orc_intersect.argtypes = [C.c_void_p, _DP, _DP, _DP, C.c_uint64, C.c_int, _DP]
        L.orc_launch_rect.argtypes = [C.c_void_p, _DP, C.c_double, _DP]
        L.orc_estimate.argtypes = [C.c_void_p, C.POINTER(A.Excitation), _DP, C.c_uint32,
                                   C.POINTER(A.McConfigC), _DP, C.POINTER(A.Stats), C.c_void_p,
                                   C.c_uint64, C.POINTER(C.c_uint64)]
        L.orc_path_log.argtypes = [C.c_void_p, C.POINTER(A.Excitation), _DP, C.c_uint32,
                                   C.POINTER(A.McConfigC), C.c_uint64, C.c_uint64,
                                   C.POINTER(C.c_uint32), C.c_uint32, C.POINTER(C.c_uint8),
                                   C.POINTER(C.c_uint64)]
        L.orc_solve.argtypes = [C.c_void_p, C.POINTER(A.Excitation), _DP, C.c_uint32,
                                C.POINTER(A.DetConfigC), _DP, C.POINTER(A.Stats), C.c_void_p,
                                C.c_uint64, C.POINTER(C.c_uint64)]
        L.orc_estimate_range.argtypes = [C.c_void_p, C.POINTER(A.Excitation), _DP, C.c_uint32,
                                         C.POINTER(A.McConfigC), C.c_uint64, C.c_uint64, _DP,
                                         C.POINTER(A.Stats), C.POINTER(C.c_uint64)]
        _port = L
    return _port


def port_estimate_range(scene_h, exc, freqs, cfg, entry_begin, entry_end):
    """Raw [nf][4] complex sums over launch entries [entry_begin, entry_end)."""
    L = port()
    freqs = np.ascontiguousarray(freqs, dtype=np.float64)
    raw = np.zeros((len(freqs), 4, 2), dtype=np.float64)
    st = A.Stats()
    total = C.c_uint64(0)
    rc = L.orc_estimate_range(scene_h.h, C.byref(exc), dp(freqs), len(freqs), C.byref(cfg),
                              entry_begin, entry_end, dp(raw), C.byref(st), C.byref(total))
    if rc != 0:
        raise RuntimeError(L.orc_last_error().decode())
    return raw, st, total.value


def dp(a: np.ndarray):
    return a.ctypes.data_as(_DP)


# --------------------------------------------------------------------------
# scene handles over host SceneData (paper_2511_07586_b200.geometry.SceneData)

class _Handle:
    def __init__(self, lib, h, free):
        self.lib, self.h, self._free = lib, h, free

    def __del__(self):
        if self.h:
            self._free(self.h)
            self.h = None


def ref_scene(sd) -> _Handle:
    L = ref()
    h = L.ref_scene_from_arrays(dp(sd.vertices), len(sd.vertices), sd.triangles.ctypes.data,
                                len(sd.triangles), sd.materials.ctypes.data, len(sd.materials))
    if not h:
        raise RuntimeError(L.ref_last_error().decode())
    return _Handle(L, h, L.ref_scene_free)


def port_scene(sd) -> _Handle:
    L = port()
    h = L.orc_scene_create(dp(sd.vertices), len(sd.vertices), sd.triangles.ctypes.data,
                           len(sd.triangles), sd.materials.ctypes.data, len(sd.materials))
    if not h:
        raise RuntimeError(L.orc_last_error().decode())
    return _Handle(L, h, L.orc_scene_free)


def _estimate(fn, errfn, scene_h, exc, freqs, cfg, contributions, capacity, *pre):
    freqs = np.ascontiguousarray(freqs, dtype=np.float64)
    nf = len(freqs)
    values = np.zeros((4, max(nf, 1), 2), dtype=np.float64)
    st = A.Stats()
    contribs = None
    n_c = C.c_uint64(0)
    if contributions:
        contribs = np.zeros(capacity, dtype=A.CONTRIBUTION_DTYPE)
    rc = fn(scene_h, C.byref(exc), dp(freqs), nf, C.byref(cfg), *pre, dp(values), C.byref(st),
            contribs.ctypes.data if contribs is not None else None, capacity, C.byref(n_c))
    if rc != 0:
        raise RuntimeError(errfn().decode())
    out = {"values": values[..., 0] + 1j * values[..., 1], "stats": st}
    if contributions:
        out["contributions"] = contribs[: min(n_c.value, capacity)]
        out["n_contributions"] = n_c.value
    return out


def ref_estimate(scene_h, exc, freqs, cfg, workers=1, contributions=False, capacity=0):
    L = ref()
    return _estimate(L.ref_estimate, L.ref_last_error, scene_h.h, exc, freqs, cfg, contributions,
                     capacity, workers)


def port_estimate(scene_h, exc, freqs, cfg, contributions=False, capacity=0):
    L = port()
    return _estimate(L.orc_estimate, L.orc_last_error, scene_h.h, exc, freqs, cfg, contributions,
                     capacity)


def ref_solve(scene_h, exc, freqs, cfg, workers=1, contributions=False, capacity=0):
    L = ref()
    return _estimate(L.ref_solve, L.ref_last_error, scene_h.h, exc, freqs, cfg, contributions,
                     capacity, workers)


def port_solve(scene_h, exc, freqs, cfg, contributions=False, capacity=0):
    L = port()
    return _estimate(L.orc_solve, L.orc_last_error, scene_h.h, exc, freqs, cfg, contributions,
                     capacity)


def _text(fn, *args):
    n = C.c_uint64(0)
    rc = fn(*args, None, 0, C.byref(n))
    buf = C.create_string_buffer(n.value + 1)
    rc = fn(*args, buf, n.value + 1, C.byref(n))
    return rc, buf.value.decode()


def ref_sweep_csv(values, freqs, seed, solver, config_hash):
    """The reference's sweep_csv (runner.cpp:80-99) of a [4][nf] complex block."""
    v = np.ascontiguousarray(np.stack([np.real(values), np.imag(values)], axis=-1), dtype=np.float64)
    f = np.ascontiguousarray(freqs, dtype=np.float64)
    rc, t = _text(ref().ref_sweep_csv, dp(v), dp(f), len(f), seed, solver.encode(), config_hash.encode())
    if rc != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return t


def ref_stats_json(stats, solver):
    rc, t = _text(ref().ref_stats_json, C.byref(stats), solver.encode())
    if rc != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return t


def ref_parse_config(text):
    """(ok, config_hash or ConfigError message)."""
    rc, t = _text(ref().ref_parse_config, text.encode())
    if rc < 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return rc == 0, t


def ref_run_command(command, config_text, out_dir, workers=1, seed=None, lib=None):
    """run_command (runner.cpp:437-452) of the CPU reference, or of ``lib``
    (e.g. ``dropin()``: the same code with the solvers on the GPU)."""
    L = lib or ref()
    rc = L.ref_run_command(command.encode(), config_text.encode(), out_dir.encode(), workers,
                               0 if seed is None else 1, 0 if seed is None else seed)
    if rc < 0:
        raise RuntimeError(L.ref_last_error().decode())
    return rc


def port_path_log(scene_h, exc, freqs, cfg, first, n, stride):
    L = port()
    freqs = np.ascontiguousarray(freqs, dtype=np.float64)
    tri = np.zeros((n, stride), dtype=np.uint32)
    term = np.zeros(n, dtype=np.uint8)
    br = np.zeros(n, dtype=np.uint64)
    rc = L.orc_path_log(scene_h.h, C.byref(exc), dp(freqs), len(freqs), C.byref(cfg), first, n,
                        tri.ctypes.data_as(C.POINTER(C.c_uint32)), stride,
                        term.ctypes.data_as(C.POINTER(C.c_uint8)),
                        br.ctypes.data_as(C.POINTER(C.c_uint64)))
    if rc != 0:
        raise RuntimeError(L.orc_last_error().decode())
    return tri, term, br


def intersect(which: str, scene_h, o, d, t_min, mode):
    """mode 0 closest, 1 brute force, 2 occluded -> (n, 13) hit blocks."""
    L = ref() if which == "ref" else port()
    fn = L.ref_intersect if which == "ref" else L.orc_intersect
    o = np.ascontiguousarray(o, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    t_min = np.ascontiguousarray(t_min, dtype=np.float64)
    n = len(o)
    out = np.zeros((n, 13), dtype=np.float64)
    fn(scene_h.h, dp(o), dp(d), dp(t_min), n, mode, dp(out))
    return out
