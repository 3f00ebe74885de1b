"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over oracle/liboracle.so, the plain
double-precision CPU Katsevich reconstruction written from arXiv 2201.02309 §II
(see oracle.cpp for the per-function citations).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs may import this module.  It shares no code with paper_2201_02309_b200/.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")


class OraGeom(ctypes.Structure):
    _fields_ = [
        ("R", ctypes.c_double), ("D", ctypes.c_double), ("P", ctypes.c_double),
        ("lambda0", ctypes.c_double), ("z0", ctypes.c_double), ("r_fov", ctypes.c_double),
        ("n_rows", ctypes.c_int32), ("d_w", ctypes.c_double),
        ("n_cols", ctypes.c_int32), ("d_alpha", ctypes.c_double), ("alpha_offset", ctypes.c_double),
        ("views_per_turn", ctypes.c_int32),
        ("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("dx", ctypes.c_double), ("dy", ctypes.c_double),
        ("nz", ctypes.c_int32), ("n_psi", ctypes.c_int32), ("apod", ctypes.c_int32), ("flat", ctypes.c_int32),
    ]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared",
                               "-o", _SO, src])
    return _SO


_lib = None
_D = ctypes.POINTER(ctypes.c_double)
_F = ctypes.POINTER(ctypes.c_float)
_I32 = ctypes.POINTER(ctypes.c_int32)
_I64 = ctypes.POINTER(ctypes.c_int64)
_G = ctypes.POINTER(OraGeom)


def lib():
    global _lib
    if _lib is None:
        build()
        l = ctypes.CDLL(_SO)
        sig = {
            "ora_derived": (None, [_G, _D]),
            "ora_pi_line": (None, [_G, ctypes.c_double, ctypes.c_double, ctypes.c_double, _D, _D]),
            "ora_pi_lines": (None, [_G, _D, ctypes.c_int64, _D, _D]),
            "ora_w_kappa": (ctypes.c_double, [_G, ctypes.c_double, ctypes.c_double]),
            "ora_psi_hat": (ctypes.c_int, [_G, ctypes.c_double, ctypes.c_double, _D]),
            "ora_hilbert_kernel": (None, [_G, _D]),
            "ora_rebin_tables": (None, [_G, _I32, _D, _I32, _D]),
            "ora_bp_weights": (None, [_G, ctypes.c_int32, _I64, _I64, _D, _D]),
            "ora_pitch_slab": (None, [_G, ctypes.c_int32, _I64, _I64]),
            "ora_bp_weights_voxels": (None, [_G, ctypes.c_int32, _I32, ctypes.c_int64, _I64, _I64, _D, _D]),
            "ora_filter": (ctypes.c_int, [_G, _F, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, _D, _D, _D, _D]),
            "ora_backproject": (ctypes.c_int, [_G, ctypes.c_int32, _D, ctypes.c_int64, ctypes.c_int64, _D]),
            "ora_backproject_voxels": (ctypes.c_int, [_G, ctypes.c_int32, _D, ctypes.c_int64, ctypes.c_int64,
                                                      _I32, ctypes.c_int64, _D]),
            "ora_reconstruct": (ctypes.c_int, [_G, _F, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                               ctypes.c_int32, _D]),
            "ora_backproject_T": (None, [_G, ctypes.c_int32, _D, ctypes.c_int64, ctypes.c_int64, _D]),
            "ora_filter_T": (ctypes.c_int, [_G, _D, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int64, _D]),
            "ora_adjoint": (ctypes.c_int, [_G, _D, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                           ctypes.c_int64, _D]),
            "ora_project_ellipsoids": (None, [_G, _D, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, _D]),
            "ora_project_volume": (None, [_G, _F, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_int64, ctypes.c_int32, _D, _I64]),
            "ora_resample_alpha": (None, [_G, _D, ctypes.c_int64, ctypes.c_int32, _D]),
            "ora_add_noise": (ctypes.c_int, [_G, _D, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_uint64, ctypes.c_int, _D, _I64, _D]),
            "ora_filter_prepare": (ctypes.c_void_p, [_G]),
            "ora_filter_free": (None, [ctypes.c_void_p]),
            "ora_filter_run": (ctypes.c_int, [ctypes.c_void_p, _F, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_int64, _D, _D, _D, _D]),
            "ora_set_threads": (None, [ctypes.c_int]),
            "ora_deriv_half": (ctypes.c_int, [_G, _F, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_int64, _D]),
            "ora_filter_g1": (None, [_G, _D, ctypes.c_int64, _D, _D, _D, _D]),
            "ora_get_threads": (ctypes.c_int, []),
            "ora_philox": (None, [ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
                                  ctypes.POINTER(ctypes.c_uint32)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def geom(cfg: dict) -> OraGeom:
    return OraGeom(cfg["R"], cfg["D"], cfg["P"], cfg.get("lambda0", 0.0), cfg.get("z0", 0.0),
                   cfg.get("r_fov", 0.0), cfg["n_rows"], cfg["d_w"], cfg["n_cols"], cfg["d_alpha"],
                   cfg.get("alpha_offset", 0.0), cfg["views_per_turn"], cfg["nx"], cfg["ny"],
                   cfg["dx"], cfg.get("dy", cfg["dx"]), cfg["nz"], cfg.get("n_psi", 0),
                   1 if cfg.get("flags", 0) & 2 else 0,          # NEXT-4: Hann-apodised Hilbert (A26)
                   1 if cfg.get("flags", 0) & 4 else 0)          # NEXT-4: flat detector (A27)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def derived(cfg):
    out = np.zeros(8)
    g = geom(cfg)
    lib().ora_derived(ctypes.byref(g), _p(out, _D))
    keys = ["dlam", "h", "r_fov", "alpha_m", "psi_max", "dpsi", "kappa_scale", "n_psi"]
    d = dict(zip(keys, out.tolist()))
    d["n_psi"] = int(d["n_psi"])
    return d


def pi_line(cfg, x, y, z):
    g = geom(cfg)
    li, lo = ctypes.c_double(), ctypes.c_double()
    lib().ora_pi_line(ctypes.byref(g), x, y, z, ctypes.byref(li), ctypes.byref(lo))
    return li.value, lo.value


def pi_lines(cfg, pts):
    g = geom(cfg)
    p = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).reshape(-1, 3))
    li = np.empty(p.shape[0]); lo = np.empty(p.shape[0])
    lib().ora_pi_lines(ctypes.byref(g), _p(p, _D), p.shape[0], _p(li, _D), _p(lo, _D))
    return li, lo


def w_kappa(cfg, alpha, psi):
    g = geom(cfg)
    return lib().ora_w_kappa(ctypes.byref(g), alpha, psi)


def psi_hat(cfg, alpha, w):
    g = geom(cfg)
    out = ctypes.c_double()
    ok = lib().ora_psi_hat(ctypes.byref(g), alpha, w, ctypes.byref(out))
    return out.value if ok else None


def hilbert_kernel(cfg):
    g = geom(cfg)
    K = np.empty(2 * cfg["n_cols"] - 1)
    lib().ora_hilbert_kernel(ctypes.byref(g), _p(K, _D))
    return K


def rebin_tables(cfg):
    d = derived(cfg)
    npsi, nr, nc = d["n_psi"], cfg["n_rows"], cfg["n_cols"]
    fi = np.empty((npsi, nc), np.int32); ff = np.empty((npsi, nc))
    bi = np.empty((nr, nc), np.int32); bf = np.empty((nr, nc))
    g = geom(cfg)
    lib().ora_rebin_tables(ctypes.byref(g), _p(fi, _I32), _p(ff, _D), _p(bi, _I32), _p(bf, _D))
    return fi, ff, bi, bf


def bp_weights(cfg, pitch):
    shape = (cfg["nz"], cfg["ny"], cfg["nx"])
    kf = np.empty(shape, np.int64); kl = np.empty(shape, np.int64)
    wf = np.empty(shape); wl = np.empty(shape)
    g = geom(cfg)
    lib().ora_bp_weights(ctypes.byref(g), pitch, _p(kf, _I64), _p(kl, _I64), _p(wf, _D), _p(wl, _D))
    return kf, kl, wf, wl


def bp_weights_voxels(cfg, pitch, idx):
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int32).reshape(-1, 3))
    n = idx.shape[0]
    kf = np.empty(n, np.int64); kl = np.empty(n, np.int64); wf = np.empty(n); wl = np.empty(n)
    g = geom(cfg)
    lib().ora_bp_weights_voxels(ctypes.byref(g), pitch, _p(idx, _I32), n, _p(kf, _I64), _p(kl, _I64),
                                _p(wf, _D), _p(wl, _D))
    return kf, kl, wf, wl


def pitch_slab(cfg, pitch):
    g = geom(cfg)
    fv, nv = ctypes.c_int64(), ctypes.c_int64()
    lib().ora_pitch_slab(ctypes.byref(g), pitch, ctypes.byref(fv), ctypes.byref(nv))
    return fv.value, nv.value


def filter_views(cfg, sino, s0, v_first, n_out, stages=("gF",)):
    """Filter views [v_first, v_first+n_out).  Returns dict of requested stages
    among g2, g3, g4, gF (float64)."""
    d = derived(cfg)
    nr, nc, npsi = cfg["n_rows"], cfg["n_cols"], d["n_psi"]
    sino = np.ascontiguousarray(sino, dtype=np.float32)
    out = {}
    shapes = {"g2": (n_out, nr, nc), "g3": (n_out, npsi, nc), "g4": (n_out, npsi, nc), "gF": (n_out, nr, nc)}
    for s in stages:
        out[s] = np.empty(shapes[s])
    g = geom(cfg)
    rc = lib().ora_filter(ctypes.byref(g), _p(sino, _F), s0, sino.shape[0], v_first, n_out,
                          _p(out.get("g2"), _D), _p(out.get("g3"), _D), _p(out.get("g4"), _D),
                          _p(out.get("gF"), _D))
    if rc != 0:
        raise ValueError("oracle filter: sinogram does not cover the requested views")
    return out


class PreparedFilter:
    """Steps 1-6 with the per-geometry set-up (Hilbert kernel, rebin maps) built once, so that
    bench.py can time the filter alone; the same arithmetic as filter_views."""

    def __init__(self, cfg):
        self.cfg = cfg
        self._g = geom(cfg)
        self._ctx = lib().ora_filter_prepare(ctypes.byref(self._g))

    def gF(self, sino, s0, v_first, n_out):
        nr, nc = self.cfg["n_rows"], self.cfg["n_cols"]
        sino = np.ascontiguousarray(sino, dtype=np.float32)
        out = np.empty((n_out, nr, nc))
        rc = lib().ora_filter_run(self._ctx, _p(sino, _F), s0, sino.shape[0], v_first, n_out,
                                  None, None, None, _p(out, _D))
        if rc != 0:
            raise ValueError("oracle filter: sinogram does not cover the requested views")
        return out

    def __del__(self):
        if getattr(self, "_ctx", None):
            lib().ora_filter_free(self._ctx)
            self._ctx = None


def set_threads(n: int) -> None:
    """OpenMP threads of the following oracle calls (0: all processors)."""
    lib().ora_set_threads(int(n))


def get_threads() -> int:
    return int(lib().ora_get_threads())


def backproject(cfg, pitch, gF, gF0):
    gF = np.ascontiguousarray(gF, dtype=np.float64)
    vol = np.empty((cfg["nz"], cfg["ny"], cfg["nx"]))
    g = geom(cfg)
    rc = lib().ora_backproject(ctypes.byref(g), pitch, _p(gF, _D), gF0, gF.shape[0], _p(vol, _D))
    if rc:
        raise ValueError("oracle backproject: filtered views do not cover a PI-window")
    return vol


def backproject_voxels(cfg, pitch, gF, gF0, idx):
    gF = np.ascontiguousarray(gF, dtype=np.float64)
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int32).reshape(-1, 3))
    out = np.empty(idx.shape[0])
    g = geom(cfg)
    rc = lib().ora_backproject_voxels(ctypes.byref(g), pitch, _p(gF, _D), gF0, gF.shape[0],
                                      _p(idx, _I32), idx.shape[0], _p(out, _D))
    if rc:
        raise ValueError("oracle backproject: filtered views do not cover a PI-window")
    return out


def reconstruct(cfg, sino, s0, k0, n_pitches):
    sino = np.ascontiguousarray(sino, dtype=np.float32)
    vol = np.empty((n_pitches * cfg["nz"], cfg["ny"], cfg["nx"]))
    g = geom(cfg)
    rc = lib().ora_reconstruct(ctypes.byref(g), _p(sino, _F), s0, sino.shape[0], k0, n_pitches, _p(vol, _D))
    if rc:
        raise ValueError("oracle reconstruct: sinogram does not cover a requested pitch slab")
    return vol


# ---- NEXT-4: Noo's half-sample derivative (reading A25) ----

def half_sample_cfg(cfg):
    """Geometry of the half-shifted grid the half-sample derivative produces (reading A25): samples
    (λ_{k+½}, α_{l+½}, w_{m+½}) are those of a detector with one row and one column fewer (same
    spacings, offsets: α_{l+½} = (l - (n_c - 2)/2 + offset) Δα, w_{m+½} = (m - (n_r - 2)/2) Δw) on the
    same helix parametrised from λ0 + Δλ/2 and z0 + P Δλ / (4π) (Eq. 1: a(λ_{k+½}) = a'(λ_k)).  The
    voxel grid, FOV and pitch are unchanged; the κ-line count defaults to 2 (n_r - 1) + 1."""
    import math
    dlam = 2 * math.pi / cfg["views_per_turn"]
    return dict(cfg, n_rows=cfg["n_rows"] - 1, n_cols=cfg["n_cols"] - 1,
                lambda0=cfg.get("lambda0", 0.0) + 0.5 * dlam,
                z0=cfg.get("z0", 0.0) + cfg["P"] * dlam / (4 * math.pi))


def deriv_half(cfg, sino, s0, v_first, n_out):
    """g1 [n_out][rows-1][cols-1] on the half-shifted grid for half-views v_first+½ .. (raw views
    v_first .. v_first + n_out of a sinogram whose first view is s0)."""
    sino = np.ascontiguousarray(sino, dtype=np.float32)
    out = np.empty((n_out, cfg["n_rows"] - 1, cfg["n_cols"] - 1))
    g = geom(cfg)
    if lib().ora_deriv_half(ctypes.byref(g), _p(sino, _F), s0, sino.shape[0], v_first, n_out, _p(out, _D)):
        raise ValueError("oracle deriv_half: sinogram does not cover the requested views")
    return out


def filter_g1(cfg, g1, stages=("gF",)):
    """Steps 2-6 from step-1 output g1 [n][rows][cols] in geometry cfg."""
    d = derived(cfg)
    nr, nc, npsi = cfg["n_rows"], cfg["n_cols"], d["n_psi"]
    g1 = np.ascontiguousarray(g1, dtype=np.float64)
    n = g1.shape[0]
    shapes = {"g2": (n, nr, nc), "g3": (n, npsi, nc), "g4": (n, npsi, nc), "gF": (n, nr, nc)}
    out = {s: np.empty(shapes[s]) for s in stages}
    g = geom(cfg)
    lib().ora_filter_g1(ctypes.byref(g), _p(g1, _D), n, _p(out.get("g2"), _D), _p(out.get("g3"), _D),
                        _p(out.get("g4"), _D), _p(out.get("gF"), _D))
    return out


def reconstruct_half(cfg, sino, s0, k0, n_pitches):
    """reconstruct() with Noo's half-sample derivative (reading A25): per pitch, the half-shifted
    grid's slab [K_lo, K_hi] (its PI windows on the views λ_{k+½}), step 1 by the 2x2x2 cube from raw
    views K_lo .. K_hi + 1, steps 2-7 on the half-shifted grid."""
    vc = half_sample_cfg(cfg)
    vol = np.empty((n_pitches * cfg["nz"], cfg["ny"], cfg["nx"]))
    for i, k in enumerate(range(k0, k0 + n_pitches)):
        fv, nv = pitch_slab(vc, k)
        klo, n = fv + 1, nv - 2
        g1 = deriv_half(cfg, sino, s0, klo, n)
        gF = filter_g1(vc, g1)["gF"]
        vol[i * cfg["nz"]:(i + 1) * cfg["nz"]] = backproject(vc, k, gF, klo)
    return vol


# ---- adjoint (NEXT-1): transposes of the maps above, pinned by dot-product tests ----

def backproject_T(cfg, pitch, vol, gF0, gFn):
    """BP^T: volume of pitch `pitch` -> filtered-view adjoint [gFn][rows][cols] for views gF0.. ."""
    vol = np.ascontiguousarray(vol, dtype=np.float64)
    out = np.zeros((gFn, cfg["n_rows"], cfg["n_cols"]))
    g = geom(cfg)
    lib().ora_backproject_T(ctypes.byref(g), pitch, _p(vol, _D), gF0, gFn, _p(out, _D))
    return out


def filter_T(cfg, gFT, v_first, s0, sn):
    """F^T: filtered-view adjoint for views v_first.. -> raw-view adjoint for views s0..s0+sn-1."""
    gFT = np.ascontiguousarray(gFT, dtype=np.float64)
    out = np.zeros((sn, cfg["n_rows"], cfg["n_cols"]))
    g = geom(cfg)
    rc = lib().ora_filter_T(ctypes.byref(g), _p(gFT, _D), v_first, gFT.shape[0], s0, sn, _p(out, _D))
    if rc:
        raise ValueError("oracle filter_T: output views do not hold the +-1 halo")
    return out


def adjoint(cfg, vol, k0, n_pitches, s0, sn):
    """A^T of reconstruct(): volume [n_pitches*nz][ny][nx] -> sinogram adjoint [sn][rows][cols]."""
    vol = np.ascontiguousarray(vol, dtype=np.float64)
    out = np.empty((sn, cfg["n_rows"], cfg["n_cols"]))
    g = geom(cfg)
    rc = lib().ora_adjoint(ctypes.byref(g), _p(vol, _D), k0, n_pitches, s0, sn, _p(out, _D))
    if rc:
        raise ValueError("oracle adjoint: sinogram does not cover a requested pitch slab")
    return out


# ---- NEXT-3: data generation (P:l.353-404) ----

def project_ellipsoids(cfg, ellipsoids, v0, n_views):
    """Exact line integrals [n_views][rows][cols] (float64) of an ellipsoid phantom."""
    e = np.ascontiguousarray(np.asarray(ellipsoids, dtype=np.float64).reshape(-1, 8))
    out = np.empty((n_views, cfg["n_rows"], cfg["n_cols"]))
    g = geom(cfg)
    lib().ora_project_ellipsoids(ctypes.byref(g), _p(e, _D), e.shape[0], v0, n_views, _p(out, _D))
    return out


def project_volume(cfg, vol, zv0, dzv, v0, n_views):
    """Trilinear ray-marched line integrals of vol [nzv][ny][nx] (slices at zv0 + j dzv).
    Returns (sino float64, number of rays truncated by the volume's z extent)."""
    vol = np.ascontiguousarray(vol, dtype=np.float32)
    out = np.empty((n_views, cfg["n_rows"], cfg["n_cols"]))
    nt = ctypes.c_int64()
    g = geom(cfg)
    lib().ora_project_volume(ctypes.byref(g), _p(vol, _F), vol.shape[0], zv0, dzv, v0, n_views, _p(out, _D),
                             ctypes.byref(nt))
    return out, nt.value


def resample_alpha(cfg, sino, stride):
    """alpha_sp = alpha[0:stride:end], then linear interpolation back (edge hold)."""
    sino = np.ascontiguousarray(sino, dtype=np.float64)
    out = np.empty_like(sino)
    g = geom(cfg)
    lib().ora_resample_alpha(ctypes.byref(g), _p(sino, _D), sino.shape[0], stride, _p(out, _D))
    return out


def add_noise(cfg, sino, v_first, I0=1e5, var=0.5, seed=0, mode=0):
    """'Gaussian+Poisson' noise; returns (noisy float64, Poisson counts int64, M)."""
    sino = np.ascontiguousarray(sino, dtype=np.float64)
    out = np.empty_like(sino)
    counts = np.zeros(sino.shape, dtype=np.int64)
    M = ctypes.c_double()
    g = geom(cfg)
    rc = lib().ora_add_noise(ctypes.byref(g), _p(sino, _D), v_first, sino.shape[0], I0, var, seed, mode,
                             _p(out, _D), _p(counts, _I64), ctypes.byref(M))
    if rc:
        raise ValueError("oracle add_noise: max of the sinogram must be > 0")
    return out, counts, M.value


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().ora_philox(c, k, o)
    return list(o)
