"""Radar products from sweeps, computed on the GPU.

Mirrors proj/include/mcsbr/signal_processing.hpp: ``Window``, ``RangeProfile``,
``range_profile(sweep, channel, window, zero_pad)``, ``IsarImage``,
``isar(sweeps, angles_deg, channel, window, zero_pad, dynamic_floor_db)``,
``SignalError``.  The transforms run in csrc/imaging.cu through the C ABI.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _abi as A


class SignalError(RuntimeError):
    """mcsbr::SignalError (signal_processing.hpp:17-19)."""


class Window(enum.IntEnum):
    NONE = 0
    HANN = 1


@dataclass
class RangeProfile:
    range_m: np.ndarray
    mag_db: np.ndarray
    window: Window = Window.HANN
    zero_pad: int = 4
    bin_spacing: float = 0.0


@dataclass
class IsarImage:
    down_range_m: np.ndarray
    cross_range_m: np.ndarray
    mag_db: np.ndarray  # (rows = down range, cols = cross range)
    dynamic_floor_db: float = -40.0
    peak_db: float = 0.0
    window: Window = Window.HANN
    zero_pad: int = 4

    def at(self, row: int, col: int) -> float:
        return float(self.mag_db[row, col])


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = A.lib().mcsbr_gpu_last_error().decode()
    if rc == A.MCSBR_EINVAL:
        raise SignalError(msg)
    raise A.McsbrError(rc, msg)


_DP = C.POINTER(C.c_double)


def range_profile(sweep, channel: int, window: Window = Window.HANN, zero_pad: int = 4) -> RangeProfile:
    """signal_processing.cpp:66-89.  `sweep` is a SweepResult (values [4][nf])."""
    freqs = np.ascontiguousarray(sweep.frequencies, dtype=np.float64)
    vals = np.ascontiguousarray(np.asarray(sweep.values)[channel], dtype=np.complex128)
    m = len(freqs) * max(int(zero_pad), 1)
    r = np.zeros(m)
    db = np.zeros(m)
    bin_ = C.c_double(0.0)
    _check(A.lib().mcsbr_gpu_range_profile(vals.view(np.float64).ctypes.data_as(_DP),
                                           freqs.ctypes.data_as(_DP), len(freqs), int(window),
                                           int(zero_pad), r.ctypes.data_as(_DP), db.ctypes.data_as(_DP),
                                           C.byref(bin_)))
    return RangeProfile(r, db, Window(window), int(zero_pad), bin_.value)


def isar(sweeps, angles_deg, channel: int, window: Window = Window.HANN, zero_pad: int = 4,
         dynamic_floor_db: float = -40.0, frequencies=None) -> IsarImage:
    """signal_processing.cpp:91-162.  `sweeps`: a list of SweepResult (one per
    angle), or an array of values [na][4][nf] with `frequencies` given."""
    if isinstance(sweeps, np.ndarray):
        vals = np.ascontiguousarray(sweeps[:, channel, :], dtype=np.complex128)
        freqs = np.ascontiguousarray(frequencies, dtype=np.float64)
    else:
        if len(sweeps) == 0:
            raise SignalError("isar: one sweep per angle required")
        freqs = np.ascontiguousarray(sweeps[0].frequencies, dtype=np.float64)
        for s in sweeps:
            if len(s.frequencies) != len(freqs) or abs(s.frequencies[0] - freqs[0]) > 1e-3:
                raise SignalError("isar: sweeps must share one frequency grid")
        vals = np.ascontiguousarray(np.stack([np.asarray(s.values)[channel] for s in sweeps]),
                                    dtype=np.complex128)
    ang = np.ascontiguousarray(angles_deg, dtype=np.float64)
    if len(ang) != len(vals):
        raise SignalError("isar: one sweep per angle required")
    zp = max(int(zero_pad), 1)
    mr, mc = len(freqs) * zp, len(ang) * zp
    down, cross, db = np.zeros(mr), np.zeros(mc), np.zeros((mr, mc))
    peak = C.c_double(0.0)
    _check(A.lib().mcsbr_gpu_isar(vals.view(np.float64).ctypes.data_as(_DP), freqs.ctypes.data_as(_DP),
                                  len(freqs), ang.ctypes.data_as(_DP), len(ang), int(window), int(zero_pad),
                                  float(dynamic_floor_db), down.ctypes.data_as(_DP),
                                  cross.ctypes.data_as(_DP), db.ctypes.data_as(_DP), C.byref(peak)))
    return IsarImage(down, cross, db, float(dynamic_floor_db), peak.value, Window(window), int(zero_pad))
