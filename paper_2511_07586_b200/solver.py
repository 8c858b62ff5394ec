"""Host-side mirror of the reference solver interface, backed by the CUDA library.

Names, fields and error behaviour follow the reference's public headers so
code written against ``mcsbr::estimate`` reads the same here:

* ``Excitation``, ``monostatic_excitation``, ``bistatic_excitation``
  (proj/include/mcsbr/solver_common.hpp:16-30, proj/src/solver_common.cpp:15-49)
* ``McConfig`` / ``RouletteConfig`` / ``BranchStrategy`` (solver_mc.hpp:14-36)
* ``SweepResult`` / ``RunStats`` / ``McResult`` (farfield.hpp:73-80,
  solver_common.hpp:37-53, solver_mc.hpp:73-76)
* ``estimate(scene, excitation, frequencies, config, workers, contributions_out)``
  (solver_mc.hpp:81-83) -> ``mcsbr_gpu_estimate`` in libmcsbr_gpu.so.

Every call runs on the GPU through the C ABI (include/mcsbr_gpu.h); there is
no CPU fallback.  ``std::invalid_argument`` becomes ``ValueError`` with the
reference's message, ``SceneError`` stays ``SceneError``, in-kernel reference
throw sites (DomainError) become ``DomainError``.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi as A
from .geometry import SceneData, SceneError

K_SPEED_OF_LIGHT = 299792458.0
K_PI = 3.14159265358979323846

VV, HH, VH, HV = 0, 1, 2, 3  # PolChannel, farfield.hpp:61-63


class DomainError(RuntimeError):
    """mcsbr::DomainError (em_math.hpp:107-109), raised from device fault flags."""


def _raise(code: int) -> None:
    if code == 0:
        return
    msg = A.lib().mcsbr_gpu_last_error().decode()
    if code == A.MCSBR_EINVAL:
        raise ValueError(msg)
    if code == A.MCSBR_ESCENE:
        raise SceneError(msg)
    if code == A.MCSBR_EDEVICE:
        raise DomainError(msg)
    raise A.McsbrError(code, msg)


# ---------------------------------------------------------------------------
# excitation (solver_common.cpp:15-49)


@dataclass
class Excitation:
    k_inc: tuple = (0.0, 0.0, -1.0)
    pol_v: tuple = (1.0, 0.0, 0.0)
    pol_h: tuple = (0.0, 1.0, 0.0)
    k_scatter: tuple = (0.0, 0.0, 1.0)
    rx_v: tuple = (1.0, 0.0, 0.0)
    rx_h: tuple = (0.0, 1.0, 0.0)
    occlusion_enabled: bool = True

    def to_c(self) -> A.Excitation:
        e = A.Excitation()
        for name in ("k_inc", "pol_v", "pol_h", "k_scatter", "rx_v", "rx_h"):
            getattr(e, name)[:] = [float(x) for x in getattr(self, name)]
        e.occlusion_enabled = 1 if self.occlusion_enabled else 0
        return e

    def incidence(self, strata_per_wavelength: float = 0.0) -> A.Incidence:
        i = A.Incidence()
        i.k_inc[:] = list(map(float, self.k_inc))
        i.pol_v[:] = list(map(float, self.pol_v))
        i.pol_h[:] = list(map(float, self.pol_h))
        i.strata_per_wavelength = float(strata_per_wavelength)
        return i

    def receiver(self) -> A.Receiver:
        r = A.Receiver()
        r.k_scatter[:] = list(map(float, self.k_scatter))
        r.rx_v[:] = list(map(float, self.rx_v))
        r.rx_h[:] = list(map(float, self.rx_h))
        return r


def _spherical(theta_deg: float, phi_deg: float):
    th = theta_deg * K_PI / 180.0
    ph = phi_deg * K_PI / 180.0
    st, ct = math.sin(th), math.cos(th)
    sp, cp = math.sin(ph), math.cos(ph)
    return (st * cp, st * sp, ct), (ct * cp, ct * sp, -st), (-sp, cp, 0.0)


def monostatic_excitation(theta_deg: float, phi_deg: float) -> Excitation:
    r, t, p = _spherical(theta_deg, phi_deg)
    return Excitation(k_inc=(-r[0], -r[1], -r[2]), pol_v=t, pol_h=p, k_scatter=r, rx_v=t, rx_h=p)


def bistatic_excitation(theta_deg, phi_deg, rx_theta_deg, rx_phi_deg) -> Excitation:
    e = monostatic_excitation(theta_deg, phi_deg)
    r, t, p = _spherical(rx_theta_deg, rx_phi_deg)
    e.k_scatter, e.rx_v, e.rx_h = r, t, p
    return e


# ---------------------------------------------------------------------------
# config (solver_mc.hpp:14-36)


class BranchStrategy(enum.IntEnum):
    FIFTY_FIFTY = A.MCSBR_BRANCH_FIFTY_FIFTY
    FRESNEL = A.MCSBR_BRANCH_FRESNEL


class RngMode(enum.IntEnum):
    REFERENCE = A.MCSBR_RNG_REFERENCE  # parity: reproduces the reference's per-ray stream
    PHILOX = A.MCSBR_RNG_PHILOX        # statistical mode


class Reduction(enum.IntEnum):
    FAST = A.MCSBR_REDUCE_FAST    # fp64 atomics (summation order varies run to run)
    EXACT = A.MCSBR_REDUCE_EXACT  # 192-bit fixed-point integer sums: byte-reproducible


@dataclass
class RouletteConfig:
    enabled: bool = False
    q: float = 0.5
    min_bounce: int = 2


@dataclass
class McConfig:
    strata_per_wavelength: float = 10.0
    samples_per_stratum: int = 16
    branch_strategy: BranchStrategy = BranchStrategy.FRESNEL
    roulette: RouletteConfig = field(default_factory=RouletteConfig)
    max_bounce: int = 9
    seed: int = 1
    reference_wavelength: float = 0.0
    launch_padding: float = 0.0
    p_min: float = 0.05
    jitter: bool = True
    block_size: int = 8192
    rng_mode: RngMode = RngMode.REFERENCE
    reduction: Reduction = Reduction.FAST
    parity_fp64_refine: bool = True

    def to_c(self) -> A.McConfigC:
        c = A.McConfigC()
        c.strata_per_wavelength = float(self.strata_per_wavelength)
        c.samples_per_stratum = int(self.samples_per_stratum)
        c.branch_strategy = int(self.branch_strategy)
        c.roulette_enabled = 1 if self.roulette.enabled else 0
        c.roulette_min_bounce = int(self.roulette.min_bounce)
        c.roulette_q = float(self.roulette.q)
        c.max_bounce = int(self.max_bounce)
        c.jitter = 1 if self.jitter else 0
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        c.reference_wavelength = float(self.reference_wavelength)
        c.launch_padding = float(self.launch_padding)
        c.p_min = float(self.p_min)
        c.block_size = int(self.block_size)
        c.rng_mode = int(self.rng_mode)
        c.reduction = int(self.reduction)
        c.parity_fp64_refine = 1 if self.parity_fp64_refine else 0
        return c

    def validate(self) -> None:
        """McConfig::validate (solver_mc.cpp:10-17)."""
        _raise(A.lib().mcsbr_gpu_validate_config(C.byref(self.to_c())))


@dataclass
class DetConfig:
    """mcsbr::DetConfig (solver_det.hpp:12-22)."""
    rays_per_wavelength: float = 20.0
    max_bounce: int = 9
    amplitude_cutoff: float = 0.0
    force_stack_accounting: bool = False
    launch_padding: float = 0.0
    reference_wavelength: float = 0.0
    block_size: int = 8192

    def to_c(self) -> A.DetConfigC:
        c = A.DetConfigC()
        c.rays_per_wavelength = float(self.rays_per_wavelength)
        c.max_bounce = int(self.max_bounce)
        c.amplitude_cutoff = float(self.amplitude_cutoff)
        c.force_stack_accounting = 1 if self.force_stack_accounting else 0
        c.launch_padding = float(self.launch_padding)
        c.reference_wavelength = float(self.reference_wavelength)
        c.block_size = int(self.block_size)
        return c

    def validate(self) -> None:
        """DetConfig::validate (solver_det.cpp:11-17)."""
        _raise(A.lib().mcsbr_gpu_validate_det_config(C.byref(self.to_c())))


# ---------------------------------------------------------------------------
# results (farfield.hpp:73-80, solver_common.hpp:37-53)


@dataclass
class SweepResult:
    frequencies: np.ndarray
    values: np.ndarray  # complex [4][nf]: VV, HH, VH, HV
    solver: str = "mc"
    seed: int = 0
    rays_launched: int = 0
    contributions: int = 0


@dataclass
class RunStats:
    rays_per_bounce: list
    roulette_candidates: list
    roulette_survivors: list
    rays_launched: int = 0
    segments_traced: int = 0
    contributions: int = 0
    grazing_kills: int = 0
    cap_kills: int = 0
    occlusion_queries: int = 0
    peak_live_state_bytes: int = 0
    state_bytes_per_ray: int = 0
    block_size: int = 0
    wall_ms: float = 0.0
    kernel_ms: float = 0.0
    forced_stack_bytes: int = 0
    device_stack_bytes: int = 0
    culled_launch_rays: int = 0

    @staticmethod
    def from_c(st: A.Stats) -> "RunStats":
        n = st.n_rounds
        last_r = max([i + 1 for i in range(A.MCSBR_MAX_BOUNCE_LIMIT) if st.roulette_candidates[i]] or [0])
        return RunStats(
            rays_per_bounce=[int(x) for x in st.rays_per_bounce[:n]],
            roulette_candidates=[int(x) for x in st.roulette_candidates[:last_r]],
            roulette_survivors=[int(x) for x in st.roulette_survivors[:last_r]],
            rays_launched=st.rays_launched, segments_traced=st.segments_traced,
            contributions=st.contributions, grazing_kills=st.grazing_kills,
            cap_kills=st.cap_kills, occlusion_queries=st.occlusion_queries,
            peak_live_state_bytes=st.peak_live_state_bytes,
            state_bytes_per_ray=st.state_bytes_per_ray, block_size=st.block_size,
            wall_ms=st.wall_ms, kernel_ms=st.kernel_ms,
            forced_stack_bytes=st.forced_stack_bytes, device_stack_bytes=st.device_stack_bytes,
            culled_launch_rays=st.culled_launch_rays,
        )


@dataclass
class McResult:
    sweep: SweepResult
    stats: RunStats


@dataclass
class DetResult:
    sweep: SweepResult
    stats: RunStats


@dataclass
class LaunchRect:
    center: np.ndarray
    u_axis: np.ndarray
    v_axis: np.ndarray
    half_u: float
    half_v: float

    def area(self) -> float:
        return 4.0 * self.half_u * self.half_v


@dataclass
class StrataGrid:
    rect: LaunchRect
    nu: int
    nv: int
    cell_area: float

    @property
    def pdf_per_cell(self) -> float:
        return 1.0 / self.cell_area

    def cell_count(self) -> int:
        return self.nu * self.nv


# ---------------------------------------------------------------------------
# scene on the GPU


class Scene:
    """A finalized scene resident on one GPU (mcsbr::Scene, geometry.hpp:55-98).

    Wraps host ``SceneData`` (vertices / triangles / materials) and the device
    handle created by ``mcsbr_gpu_scene_create`` (upload + GPU BVH build).
    """

    def __init__(self, data: SceneData, device: int = 0, devices: list | None = None):
        """device: the GPU; devices: several GPUs (mcsbr_gpu_scene_create_multi:
        BVH built on devices[0], copied to the others; estimate / estimate_batch
        shard the launch entries over them)."""
        self.data = data
        self.devices = list(devices) if devices else [device]
        self.device = self.devices[0]
        self._h = C.c_void_p()
        L = A.lib()
        v = np.ascontiguousarray(data.vertices, dtype=np.float64)
        eps_i = data.eps_imag
        args = (v.ctypes.data_as(C.POINTER(C.c_double)), len(v), data.triangles.ctypes.data,
                len(data.triangles), data.materials.ctypes.data, len(data.materials),
                eps_i.ctypes.data_as(C.POINTER(C.c_double)) if eps_i is not None else None)
        if len(self.devices) == 1:
            _raise(L.mcsbr_gpu_scene_create(*args, self.device, C.byref(self._h)))
        else:
            dv = (C.c_int * len(self.devices))(*self.devices)
            _raise(L.mcsbr_gpu_scene_create_multi(*args, dv, len(self.devices), C.byref(self._h)))

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if self._h:
            A.lib().mcsbr_gpu_scene_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # Scene accessors (geometry.hpp:76-80)
    @property
    def vertices(self):
        return self.data.vertices

    @property
    def triangles(self):
        return self.data.triangles

    @property
    def materials(self):
        return self.data.materials

    def diameter(self) -> float:
        return self.data.diameter

    def self_intersection_epsilon(self) -> float:
        return 1e-6 * self.data.diameter

    def bounding_center(self) -> np.ndarray:
        return self.data.bounding_center

    def bounding_radius(self) -> float:
        return self.data.bounding_radius

    def ambient_index(self) -> float:
        return self.data.ambient_index()

    def bvh_info(self) -> dict:
        n, d, l, ms = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_double()
        _raise(A.lib().mcsbr_gpu_scene_bvh_info(self._h, C.byref(n), C.byref(d), C.byref(l),
                                                 C.byref(ms)))
        return {"nodes": n.value, "max_depth": d.value, "leaves": l.value, "build_ms": ms.value}

    def intersect_batch(self, origins, dirs, t_min, any_hit: bool = False):
        """Batched Scene::intersect (any_hit=False) or occlusion (True) on the GPU.
        Returns (t, triangle_id) with t = inf / id = 0xFFFFFFFF on a miss."""
        o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
        n = len(o)
        tm = np.ascontiguousarray(np.broadcast_to(np.asarray(t_min, dtype=np.float64), (n,)))
        t = np.empty(n, dtype=np.float64)
        ids = np.empty(n, dtype=np.uint32)
        DP = C.POINTER(C.c_double)
        _raise(A.lib().mcsbr_gpu_intersect(self._h, o.ctypes.data_as(DP), d.ctypes.data_as(DP),
                                           tm.ctypes.data_as(DP), n, 1 if any_hit else 0,
                                           t.ctypes.data_as(DP),
                                           ids.ctypes.data_as(C.POINTER(C.c_uint32))))
        return t, ids

    def intersect(self, origin, direction, t_min: float):
        t, ids = self.intersect_batch([origin], [direction], [t_min])
        if ids[0] == 0xFFFFFFFF:
            return None
        return float(t[0]), int(ids[0])

    def occluded(self, point, direction) -> bool:
        """Scene::occluded (geometry.cpp:242-244)."""
        t, ids = self.intersect_batch([point], [direction], [self.self_intersection_epsilon()],
                                      any_hit=True)
        return bool(ids[0] != 0xFFFFFFFF)


def launch_plan(scene: Scene, k_inc, padding: float, strata_per_wavelength: float,
                reference_wavelength: float, samples_per_stratum: int = 1):
    lp = A.LaunchPlan()
    k = (C.c_double * 3)(*map(float, k_inc))
    _raise(A.lib().mcsbr_gpu_launch_plan(scene.handle, k, float(padding),
                                         float(strata_per_wavelength),
                                         float(reference_wavelength), int(samples_per_stratum),
                                         C.byref(lp)))
    rect = LaunchRect(np.array(lp.center[:]), np.array(lp.u_axis[:]), np.array(lp.v_axis[:]),
                      lp.half_u, lp.half_v)
    return StrataGrid(rect, lp.nu, lp.nv, lp.cell_area), int(lp.entries)


def launch_rect(scene: Scene, k_inc, padding: float) -> LaunchRect:
    """launch_rect (geometry.cpp:246-275), computed by the library's host planner."""
    return launch_plan(scene, k_inc, padding, 1.0, 1.0, 1)[0].rect


# ---------------------------------------------------------------------------
# the estimator


def estimate(scene: Scene, excitation: Excitation, frequencies, config: McConfig,
             workers: int = 1, contributions_out: list | None = None,
             contributions_capacity: int = 1 << 22) -> McResult:
    """mcsbr::estimate (solver_mc.hpp:81-83) on the GPU.

    If ``contributions_out`` is a list, the emitted contributions are appended
    as a numpy structured array (CONTRIBUTION_DTYPE) sorted by order_key.
    """
    freqs = np.ascontiguousarray(np.asarray(frequencies, dtype=np.float64).reshape(-1))
    nf = len(freqs)
    values = np.zeros((4, max(nf, 1), 2), dtype=np.float64)
    st = A.Stats()
    cfg = config.to_c()
    exc = excitation.to_c()
    buf = None
    n_c = C.c_uint64(0)
    cap = 0
    if contributions_out is not None:
        cap = int(contributions_capacity)
        buf = np.zeros(cap, dtype=A.CONTRIBUTION_DTYPE)
    _raise(A.lib().mcsbr_gpu_estimate(
        scene.handle, C.byref(exc), freqs.ctypes.data_as(C.POINTER(C.c_double)), nf, C.byref(cfg),
        int(workers), values.ctypes.data_as(C.POINTER(C.c_double)), C.byref(st),
        buf.ctypes.data if buf is not None else None, cap, C.byref(n_c)))
    if contributions_out is not None:
        if n_c.value > cap:
            raise ValueError(f"contributions_out capacity {cap} < {n_c.value}")
        contributions_out.append(buf[: n_c.value].copy())
    stats = RunStats.from_c(st)
    sweep = SweepResult(frequencies=freqs, values=values[..., 0] + 1j * values[..., 1],
                        seed=config.seed, rays_launched=stats.rays_launched,
                        contributions=stats.contributions)
    return McResult(sweep=sweep, stats=stats)


def solve(scene: Scene, excitation: Excitation, frequencies, config: DetConfig,
          workers: int = 1, contributions_out: list | None = None,
          contributions_capacity: int = 1 << 22) -> DetResult:
    """mcsbr::solve (solver_det.hpp:29-31), the deterministic SBR baseline, on the GPU."""
    freqs = np.ascontiguousarray(np.asarray(frequencies, dtype=np.float64).reshape(-1))
    nf = len(freqs)
    values = np.zeros((4, max(nf, 1), 2), dtype=np.float64)
    st = A.Stats()
    cfg = config.to_c()
    exc = excitation.to_c()
    buf = None
    n_c = C.c_uint64(0)
    cap = 0
    if contributions_out is not None:
        cap = int(contributions_capacity)
        buf = np.zeros(cap, dtype=A.CONTRIBUTION_DTYPE)
    _raise(A.lib().mcsbr_gpu_solve(
        scene.handle, C.byref(exc), freqs.ctypes.data_as(C.POINTER(C.c_double)), nf, C.byref(cfg),
        int(workers), values.ctypes.data_as(C.POINTER(C.c_double)), C.byref(st),
        buf.ctypes.data if buf is not None else None, cap, C.byref(n_c)))
    if contributions_out is not None:
        if n_c.value > cap:
            raise ValueError(f"contributions_out capacity {cap} < {n_c.value}")
        contributions_out.append(buf[: n_c.value].copy())
    stats = RunStats.from_c(st)
    sweep = SweepResult(frequencies=freqs, values=values[..., 0] + 1j * values[..., 1],
                        solver="deterministic", seed=0, rays_launched=stats.rays_launched)
    return DetResult(sweep=sweep, stats=stats)


def path_log(scene: Scene, excitation: Excitation, frequencies, config: McConfig, n_paths: int,
             stride: int | None = None):
    """Per-path event log of the first n_paths launch entries (parity instrumentation):
    (tri_ids [n, stride] uint32, termination [n] uint8, branch bits [n] uint64)."""
    stride = int(stride or config.max_bounce)
    freqs = np.ascontiguousarray(np.asarray(frequencies, dtype=np.float64).reshape(-1))
    tri = np.zeros((n_paths, stride), dtype=np.uint32)
    term = np.zeros(n_paths, dtype=np.uint8)
    br = np.zeros(n_paths, dtype=np.uint64)
    cfg = config.to_c()
    _raise(A.lib().mcsbr_gpu_path_log(
        scene.handle, C.byref(excitation.to_c()), freqs.ctypes.data_as(C.POINTER(C.c_double)),
        len(freqs), C.byref(cfg), n_paths, stride, tri.ctypes.data_as(C.POINTER(C.c_uint32)),
        term.ctypes.data_as(C.POINTER(C.c_uint8)), br.ctypes.data_as(C.POINTER(C.c_uint64))))
    return tri, term, br


def estimate_batch(scene: Scene, incidences: list, receivers: list, frequencies,
                   config: McConfig, occlusion_enabled: bool = True):
    """Many incidences (e.g. an azimuth sweep) in ONE device launch.

    ``incidences`` is a list of (Excitation, strata_per_wavelength or 0);
    ``receivers[i]`` is the list of receiver Excitations (k_scatter, rx_v, rx_h
    used) of incidence i, all the same length.  Returns (values, RunStats)
    with values complex [n_inc][n_rx][4][nf].
    """
    freqs = np.ascontiguousarray(np.asarray(frequencies, dtype=np.float64).reshape(-1))
    n_inc = len(incidences)
    n_rx = len(receivers[0]) if receivers else 0
    # the C structs are plain doubles: pack them with numpy (one array per
    # call instead of a ctypes object per incidence / receiver)
    inc_np = np.array([(*e.k_inc, *e.pol_v, *e.pol_h, spw) for e, spw in incidences],
                      dtype=np.float64).reshape(n_inc, 10)
    rx_np = np.array([(*r.k_scatter, *r.rx_v, *r.rx_h) for rl in receivers for r in rl],
                     dtype=np.float64).reshape(n_inc * n_rx, 9)
    inc_arr = (A.Incidence * n_inc).from_buffer(inc_np)
    rx_arr = (A.Receiver * (n_inc * n_rx)).from_buffer(rx_np)
    values = np.zeros((n_inc, n_rx, 4, len(freqs), 2), dtype=np.float64)
    st = A.Stats()
    cfg = config.to_c()
    _raise(A.lib().mcsbr_gpu_estimate_batch(
        scene.handle, inc_arr, n_inc, rx_arr, n_rx, 1 if occlusion_enabled else 0,
        freqs.ctypes.data_as(C.POINTER(C.c_double)), len(freqs), C.byref(cfg),
        values.ctypes.data_as(C.POINTER(C.c_double)), C.byref(st)))
    return values[..., 0] + 1j * values[..., 1], RunStats.from_c(st)


def rcs_m2(values: np.ndarray) -> np.ndarray:
    """sigma = |S|^2 (m^2) from complex sqrt-RCS values."""
    return np.abs(values) ** 2
