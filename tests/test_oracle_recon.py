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


def _registration_case():
    # 2 mm voxels, ~1 detector column and row per voxel at the isocentre, λ0 ≠ 0, z0 ≠ 0
    R, D, dx = 595.0, 1085.6, 2.0
    cfg = dict(name="reg", R=R, D=D, P=32.0, lambda0=0.7, z0=3.1, r_fov=0.0, n_rows=16, d_w=dx * D / R,
               n_cols=80, d_alpha=dx / R, alpha_offset=0.25, views_per_turn=360, nx=40, ny=40, dx=dx, dy=dx,
               nz=16, n_psi=0)
    c = (17.3, -9.1, 15.3)                    # off-centre, off-grid (voxel 28.65, 15.45, slice 7.65)
    # six nested balls (r = 1.5 .. 9 mm, ρ = 1/6 each): a radially symmetric object ~3 voxels in radius
    ph = np.array([[c[0], c[1], c[2], r, r, r, 0.0, 1.0 / 6] for r in (1.5, 3.0, 4.5, 6.0, 7.5, 9.0)])
    vt = cfg["views_per_turn"]
    v0, nv = -vt, 3 * vt
    return cfg, c, synth.project(cfg, ph, v0, nv), v0


def _centroid_error(vol, cfg, c):
    """Density-weighted centroid of the reconstruction over a 16^3-voxel box around the true
    centre, minus the true centre, in voxels (slice, y, x)."""
    nx, dz = cfg["nx"], cfg["P"] / cfg["nz"]
    ci = np.array([c[2] / dz, c[1] / cfg["dx"] + nx / 2, c[0] / cfg["dx"] + nx / 2])   # x_i = (i - nx/2) dx
    lo = np.floor(ci - 7).astype(int)
    hi = lo + 16
    b = vol[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]]
    T, Y, X = np.meshgrid(*[np.arange(a, e) for a, e in zip(lo, hi)], indexing="ij")
    w = b.sum()
    return np.array([(b * T).sum() / w, (b * Y).sum() / w, (b * X).sum() / w]) - ci


def test_registration_off_centre_small_ball():
    """Sub-voxel registration of the oracle: a radially symmetric ~3-voxel
    ball at an asymmetric, off-grid (x, y, z) under a helix with λ0 ≠ 0 and z0 ≠ 0 (Eq. 1,
    PAPER.md l.88; step 7 geometry l.155-171; grids x_i = (i - n/2)dx, α quarter offset l.328)
    reconstructs with its density centroid within 0.05 voxel of the true centre in x, y and z.
    The same check fails for each plausible registration slip — the quarter offset with the
    wrong sign, λ0 off by half a view, z0 off by half a slice — so it pins them."""
    import math
    cfg, c, sino, v0 = _registration_case()
    vol = oracle.reconstruct(cfg, sino, v0, 0, 1)
    err = _centroid_error(vol, cfg, c)
    assert np.abs(err).max() < 0.05, err
    vt = cfg["views_per_turn"]
    for key, val in [("alpha_offset", -0.25), ("lambda0", 0.7 + math.pi / vt), ("z0", 3.1 + 1.0)]:
        bad = oracle.reconstruct(dict(cfg, **{key: val}), sino, v0, 0, 1)
        assert np.abs(_centroid_error(bad, cfg, c)).max() > 0.06, key
