"""Oracle pins — NEXT-4 flat-detector variant (reading A27).  PAPER.md states the method for
the curved detector only (l.117, l.311-349) and implements it after [Noo2003a] (l.115), which also
gives the flat-detector form; the oracle's flat steps are pinned here by what does not depend on
reading that reference right:
  * the same object scanned by a curved and by a flat detector reconstructs to the same volume
    (the two are different discretisations of one inversion formula);
  * a uniform ball reconstructs to +ρ (sign and scale), an infinite cylinder is z-invariant;
  * sub-voxel registration of an off-centre small ball (u-offset and z registration of the plane);
  * κ-lines: the flat w_κ is the curved one divided by cos α at u = D tan α (the same κ-plane);
  * the adjoint's dot-product identity (stage by stage and for the layer).
Each fails for a plausible slip in the flat steps: a dropped (u²+D²)/D or uw/D derivative factor, the
curved length weight, a post-cosine left in, the curved Hilbert kernel, the curved u*/w*."""
import math

import numpy as np
import pytest

from oracle import oracle
from synth import configs, synth

FLAT = configs.FLAT


def test_flat_and_curved_reconstruct_the_same_object():
    """T3's scan of a Shepp-Logan phantom with its curved detector, and with a flat one (TF1: same
    helix, volume and rows; columns on the plane): the two reconstructions agree to 1 % of the
    contrast (RMSE; both are ~11 % from the voxelised phantom at these coarse grids), so every flat
    step matches its curved counterpart up to discretisation."""
    f = configs.get("TF1")
    c = configs.get("T3")
    sf = synth.project(f, f["phantom"], f["scan_v0"], f["scan_nv"])
    sc = synth.project(c, c["phantom"], c["scan_v0"], c["scan_nv"])
    vf = oracle.reconstruct(f, sf, f["scan_v0"], 0, 3)
    vc = oracle.reconstruct(c, sc, c["scan_v0"], 0, 3)
    assert np.sqrt(((vf - vc) ** 2).mean()) < 0.01
    assert np.abs(vf - vc).max() < 0.1
    truth = np.concatenate([synth.volume_truth(f, f["phantom"], k) for k in range(3)])
    ef, ec = np.sqrt(((vf - truth) ** 2).mean()), np.sqrt(((vc - truth) ** 2).mean())
    assert ef < 1.05 * ec
    # the flag matters: the flat data read with the curved steps is far off
    bad = oracle.reconstruct(dict(f, flags=0), sf, f["scan_v0"], 0, 3)
    assert np.sqrt(((bad - vc) ** 2).mean()) > 10 * np.sqrt(((vf - vc) ** 2).mean())


def _flat_c1():
    """C1's helix, ball and volume with a flat 16 x 96 detector (12 mm columns: u* up to 446 mm)."""
    return dict(configs.get("C1"), d_alpha=12.0, flags=FLAT, name="C1F")


def test_flat_uniform_ball_density_and_sign():
    cfg = _flat_c1()
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
    assert np.abs(outer).mean() < 0.03


def test_flat_elliptic_cylinder_is_z_invariant():
    R, D = 595.0, 1085.6
    cfg = dict(name="cylF", R=R, D=D, P=40.0, lambda0=0.4, z0=0.0, r_fov=0.0, n_rows=24, d_w=12.0, n_cols=121,
               d_alpha=8.2, alpha_offset=0.25, views_per_turn=240, nx=40, ny=40, dx=6.0, dy=6.0, nz=6,
               n_psi=0, flags=FLAT)
    ph = np.array([[10.0, -5.0, 0.0, 80.0, 60.0, 0.0, 0.4, 1.0]])
    v0, nv = -120, 560
    sino = synth.project(cfg, ph, v0, nv)
    vol = oracle.reconstruct(cfg, sino, v0, 0, 1)
    truth = synth.volume_truth(cfg, ph, 0)
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


def test_flat_registration_off_centre_small_ball():
    """As test_oracle_recon's registration pin, on a flat detector (1 column and row per voxel at the
    isocentre): the centroid lies within 0.05 voxel of the true centre; a quarter-offset sign slip or a
    z0 slip moves it past 0.06 voxel."""
    from tests.test_oracle_recon import _centroid_error
    R, D, dx = 595.0, 1085.6, 2.0
    cfg = dict(name="regF", R=R, D=D, P=32.0, lambda0=0.7, z0=3.1, r_fov=0.0, n_rows=16, d_w=dx * D / R,
               n_cols=80, d_alpha=dx * D / R, alpha_offset=0.25, views_per_turn=360, nx=40, ny=40, dx=dx,
               dy=dx, nz=16, n_psi=0, flags=FLAT)
    c = (17.3, -9.1, 15.3)
    ph = np.array([[c[0], c[1], c[2], r, r, r, 0.0, 1.0 / 6] for r in (1.5, 3.0, 4.5, 6.0, 7.5, 9.0)])
    vt = cfg["views_per_turn"]
    v0, nv = -vt, 3 * vt
    sino = synth.project(cfg, ph, v0, nv)
    vol = oracle.reconstruct(cfg, sino, v0, 0, 1)
    assert np.abs(_centroid_error(vol, cfg, c)).max() < 0.05
    for key, val in [("alpha_offset", -0.25), ("z0", 3.1 + 1.0)]:
        bad = oracle.reconstruct(dict(cfg, **{key: val}), sino, v0, 0, 1)
        assert np.abs(_centroid_error(bad, cfg, c)).max() > 0.06, key


def test_flat_kappa_lines_are_curved_ones_over_cos():
    """One κ-plane meets the cylinder at w_κ(α, ψ) (Eq. 11) and the plane at distance D at
    w_κ(α, ψ)/cos α, u = D tan α (the ray through a detector point keeps its direction)."""
    c = configs.get("T3")
    f = dict(c, flags=FLAT)
    for a in (-0.4, -0.1, 0.0, 0.23, 0.41):
        for psi in (-1.7, -0.8, -1e-9, 0.3, 1.2, 1.8):
            wc = oracle.w_kappa(c, a, psi)
            wf = oracle.w_kappa(f, c["D"] * math.tan(a), psi)
            assert abs(wf - wc / math.cos(a)) < 1e-12 * max(1.0, abs(wf))


def _rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


def test_flat_adjoint_dot_products():
    cfg = configs.get("TF1")
    rng = np.random.default_rng(4)
    fv, nv = oracle.pitch_slab(cfg, 0)
    gF = rng.standard_normal((nv - 2, cfg["n_rows"], cfg["n_cols"]))
    y = rng.standard_normal((cfg["nz"], cfg["ny"], cfg["nx"]))
    lhs = float(np.vdot(oracle.backproject(cfg, 0, gF, fv + 1), y))
    rhs = float(np.vdot(gF, oracle.backproject_T(cfg, 0, y, fv + 1, nv - 2)))
    assert _rel(lhs, rhs) < 1e-10
    n_out, s0 = 7, 50
    x = rng.standard_normal((n_out + 2, cfg["n_rows"], cfg["n_cols"])).astype(np.float32)
    g = oracle.filter_views(cfg, x, s0, s0 + 1, n_out)["gF"]
    yy = rng.standard_normal(g.shape)
    assert _rel(float(np.vdot(g, yy)), float(np.vdot(x.astype(np.float64), oracle.filter_T(cfg, yy, s0 + 1, s0, n_out + 2)))) < 1e-10
