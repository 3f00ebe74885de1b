"""Seeded synthetic input generator (ctypes wrapper over libsynth.so).

This module holds NO Katsevich arithmetic.  It produces:
  * exact analytic helical curved-detector (or, flags & 4, flat-detector) sinograms of ellipsoid phantoms
    (closed-form ray/ellipsoid chords; scan model of
    PAPER.md l.87-94 Eq. 1 and the curved detector of l.117 / l.311-349),
  * ground-truth phantom densities,
  * seeded random arrays.
Both the oracle (tests) and the CUDA path (tests, bench) consume its output.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")


class SynthScan(ctypes.Structure):
    _fields_ = [
        ("R", ctypes.c_double), ("D", ctypes.c_double), ("P", ctypes.c_double),
        ("lambda0", ctypes.c_double), ("z0", ctypes.c_double),
        ("n_rows", ctypes.c_int32), ("d_w", ctypes.c_double),
        ("n_cols", ctypes.c_int32), ("d_alpha", ctypes.c_double), ("alpha_offset", ctypes.c_double),
        ("views_per_turn", ctypes.c_int32), ("flat", ctypes.c_int32),
    ]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        l = ctypes.CDLL(_SO)
        dp = ctypes.POINTER(ctypes.c_double)
        l.synth_project.argtypes = [ctypes.POINTER(SynthScan), dp, ctypes.c_int32, ctypes.c_int64,
                                    ctypes.c_int32, ctypes.POINTER(ctypes.c_float)]
        l.synth_project.restype = None
        l.synth_ray_quadrature.argtypes = [ctypes.POINTER(SynthScan), dp, ctypes.c_int32,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_double]
        l.synth_ray_quadrature.restype = ctypes.c_double
        l.synth_phantom_eval.argtypes = [dp, ctypes.c_int32, dp, ctypes.c_int64, dp]
        l.synth_phantom_eval.restype = None
        _lib = l
    return _lib


def _scan(g: dict) -> SynthScan:
    return SynthScan(g["R"], g["D"], g["P"], g.get("lambda0", 0.0), g.get("z0", 0.0),
                     g["n_rows"], g["d_w"], g["n_cols"], g["d_alpha"], g.get("alpha_offset", 0.0),
                     g["views_per_turn"], 1 if g.get("flags", 0) & 4 else 0)


def _ell(ellipsoids) -> np.ndarray:
    e = np.ascontiguousarray(np.asarray(ellipsoids, dtype=np.float64).reshape(-1, 8))
    return e


def project(g: dict, ellipsoids, v0: int, n_views: int) -> np.ndarray:
    """Exact line integrals g[v][m][l] (float32) for views v0..v0+n_views-1."""
    e = _ell(ellipsoids)
    out = np.empty((n_views, g["n_rows"], g["n_cols"]), dtype=np.float32)
    s = _scan(g)
    lib().synth_project(ctypes.byref(s), e.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                        e.shape[0], v0, n_views, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
    return out


def ray_quadrature(g: dict, ellipsoids, lam: float, alpha: float, w: float,
                   t0: float, t1: float, h: float) -> float:
    e = _ell(ellipsoids)
    s = _scan(g)
    return lib().synth_ray_quadrature(ctypes.byref(s), e.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                      e.shape[0], lam, alpha, w, t0, t1, h)


def phantom_eval(ellipsoids, pts) -> np.ndarray:
    e = _ell(ellipsoids)
    p = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).reshape(-1, 3))
    out = np.empty(p.shape[0], dtype=np.float64)
    lib().synth_phantom_eval(e.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), e.shape[0],
                             p.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), p.shape[0],
                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


def volume_truth(cfg: dict, ellipsoids, pitch: int) -> np.ndarray:
    """f_true on the voxel grid of pitch `pitch`: [nz][ny][nx] (float64).
    Grid: x_i = (i - nx/2) dx, z_j = j P / nz + pitch P."""
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    x = (np.arange(nx) - nx / 2) * cfg["dx"]
    y = (np.arange(ny) - ny / 2) * cfg["dy"]
    z = np.arange(nz) * cfg["P"] / nz + pitch * cfg["P"]
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    pts = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    return phantom_eval(ellipsoids, pts).reshape(nz, ny, nx)


def random_array(shape, seed: int, scale: float = 1.0) -> np.ndarray:
    """Seeded float32 standard-normal array (for linearity / random-input tests)."""
    return (np.random.default_rng(seed).standard_normal(shape) * scale).astype(np.float32)
