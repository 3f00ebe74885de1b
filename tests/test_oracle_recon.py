"""Oracle pins — end-to-end reconstruction (step 7 and the whole pipeline):
zero / linearity, the uniform-ball density (pins the overall sign, reading A3),
the z-invariant elliptic-cylinder special case, and z-periodicity."""
import math

import numpy as np

from oracle import oracle
from synth import configs, synth


def test_zero_in_zero_out_and_linearity():
    cfg = configs.get("T1")
    v0, nv = cfg["scan_v0"], cfg["scan_nv"]
    shape = (nv, cfg["n_rows"], cfg["n_cols"])
    z = oracle.reconstruct(cfg, np.zeros(shape, np.float32), v0, 0, 1)
    assert np.abs(z).max() == 0.0
    rng = np.random.default_rng(7)
    # integer-valued inputs: 3g - 2h is exact in fp32, so linearity is exact up to fp64 rounding
    g = rng.integers(-50, 50, shape).astype(np.float32)
    h = rng.integers(-50, 50, shape).astype(np.float32)
    fg = oracle.reconstruct(cfg, g, v0, 0, 1)
    fh = oracle.reconstruct(cfg, h, v0, 0, 1)
    fgh = oracle.reconstruct(cfg, 3 * g - 2 * h, v0, 0, 1)
    assert np.abs(fgh - (3 * fg - 2 * fh)).max() < 1e-10 * np.abs(fgh).max()


def test_uniform_ball_density_and_sign():
    """Exact analytic projections of a uniform ball (ρ = 1, r = 120 mm) inside U and
    inside the pitch (C1 geometry): interior mean = +ρ within 0.5 %, flat within 0.5 %."""
    cfg = configs.get("C1")
    ball = configs.ball_phantom(0.5 * cfg["P"], inner=False)
    sino = synth.project(cfg, ball, cfg["scan_v0"], cfg["scan_nv"])
    vol = oracle.reconstruct(cfg, sino, cfg["scan_v0"], 0, 1)
    nx = cfg["nx"]
    x = (np.arange(nx) - nx / 2) * cfg["dx"]
    z = np.arange(cfg["nz"]) * cfg["P"] / cfg["nz"]
    Z, Y, X = np.meshgrid(z, x, x, indexing="ij")
    r = np.sqrt(X ** 2 + Y ** 2 + (Z - 0.5 * cfg["P"]) ** 2)
    inner = vol[r < 90.0]
    outer = vol[(r > 140.0) & (np.hypot(X, Y) < 200)]
    assert abs(inner.mean() - 1.0) < 5e-3
    assert inner.std() < 5e-3
    assert np.abs(outer).mean() < 0.03          # coarse 16 x 36.5 mm rows: streaks, no bias


def test_elliptic_cylinder_is_z_invariant():
    """Infinite elliptic cylinder along z: exact data is p2D(λ,α)·sqrt(D²+w²)/D, step 2
    makes it w-independent, so every slice reconstructs the same 2-D object (≈ ρ inside)."""
    R, D = 595.0, 1085.6
    cfg = dict(name="cyl", R=R, D=D, P=40.0, lambda0=0.4, z0=0.0, r_fov=0.0, n_rows=24, d_w=12.0, n_cols=121,
               d_alpha=7.5e-3, alpha_offset=0.25, views_per_turn=240, nx=40, ny=40, dx=6.0, dy=6.0, nz=6,
               n_psi=0)
    ph = np.array([[10.0, -5.0, 0.0, 80.0, 60.0, 0.0, 0.4, 1.0]])       # c <= 0: infinite cylinder
    v0, nv = -120, 560
    sino = synth.project(cfg, ph, v0, nv)
    vol = oracle.reconstruct(cfg, sino, v0, 0, 1)
    truth = synth.volume_truth(cfg, ph, 0)
    # slices agree up to discretisation (each slice uses a different set of views)
    spread = np.abs(vol - vol.mean(axis=0, keepdims=True))
    assert spread.mean() < 0.01
    x = (np.arange(40) - 20) * 6.0
    Y, X = np.meshgrid(x, x, indexing="ij")
    u = ((X - 10) * math.cos(0.4) + (Y + 5) * math.sin(0.4)) / 80
    v = (-(X - 10) * math.sin(0.4) + (Y + 5) * math.cos(0.4)) / 60
    deep = (u ** 2 + v ** 2) < 0.5
    assert spread[:, deep].max() < 0.02
    assert abs(vol[:, deep].mean() - 1.0) < 0.01
    assert np.abs(vol - truth)[:, deep].max() < 0.05


def test_z_periodic_phantom_gives_identical_pitches():
    """A phantom periodic in z with period P: pitch k and pitch k+1 agree to
    1e-5 max|f| (SPEC l.305/criterion 6) — the oracle recomputes every PI-window
    at absolute coordinates, so this checks its periodicity end to end."""
    cfg = configs.get("T2")
    P = cfg["P"]
    rows = [[0.0, 0.0, 0.0, 150.0, 120.0, 0.0, 0.2, 0.5]]                 # infinite cylinder
    for k in range(-4, 8):
        rows.append([40.0, -30.0, k * P + 0.37 * P, 60.0, 45.0, 7.0, 0.3, 0.4])
        rows.append([-70.0, 50.0, k * P + 0.8 * P, 30.0, 35.0, 4.0, -0.6, -0.2])
    ph = np.array(rows)
    vt = cfg["views_per_turn"]
    v0, nv = -vt, 5 * vt
    sino = synth.project(cfg, ph, v0, nv)
    vol = oracle.reconstruct(cfg, sino, v0, 1, 2)
    a, b = vol[: cfg["nz"]], vol[cfg["nz"]:]
    assert np.abs(a - b).max() < 1e-5 * np.abs(a).max()


def test_outside_fov_is_zero_and_slab_matches_survey_c1():
    cfg = configs.get("C1")
    assert oracle.pitch_slab(cfg, 0) == (-47, 222)          # C1 slab 222 = [-47, 174]
    assert oracle.pitch_slab(cfg, 3) == (-47 + 3 * 128, 222)
    d = oracle.derived(cfg)
    kf, kl, _, _ = oracle.bp_weights(cfg, 0)
    nx = cfg["nx"]
    x = (np.arange(nx) - nx / 2) * cfg["dx"]
    Y, X = np.meshgrid(x, x, indexing="ij")
    outside = X ** 2 + Y ** 2 >= d["r_fov"] ** 2
    assert (kl[:, outside] < kf[:, outside]).all()
