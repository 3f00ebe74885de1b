"""Oracle pins — NEXT-4, Noo's half-sample derivative (reading A25; [Noo2003a] as cited
at PAPER.md l.115 for implementing Eq. (8)).  The 2x2x2-cube derivative is exact on affine data,
lands on the half-shifted samples (λ_{k+½}, α_{l+½}, w_{m+½}) to second order (and not on the
integer grid), the half-shifted grid's geometry reproduces the scan's rays there (independent
analytic projector), and the whole reconstruction keeps the ball density, the sign and the
registration pins of the centred scheme."""
import math

import numpy as np

from oracle import oracle
from synth import configs, synth


def _cfg(**kw):
    base = dict(R=595.0, D=1085.6, P=38.4, lambda0=0.3, z0=1.7, n_rows=12, d_w=2.0, n_cols=40,
                d_alpha=6e-3, alpha_offset=0.25, views_per_turn=360, nx=16, ny=16, dx=10.0, dy=10.0, nz=4)
    base.update(kw)
    return base


def _grids(cfg, nv, v0=0):
    lam = (np.arange(nv) + v0) * 2 * math.pi / cfg["views_per_turn"]
    al = (np.arange(cfg["n_cols"]) - (cfg["n_cols"] - 1) / 2 + cfg["alpha_offset"]) * cfg["d_alpha"]
    w = (np.arange(cfg["n_rows"]) - (cfg["n_rows"] - 1) / 2) * cfg["d_w"]
    return lam, al, w


def test_half_sample_derivative_exact_on_affine_data():
    """g = a λ + b α + c w + d: every 2x2 difference is exact, so g1 = a + b on every half sample."""
    cfg = _cfg()
    lam, al, w = _grids(cfg, 6)
    g = (3.0 * lam[:, None, None] - 2.0 * al[None, None, :] + 0.7 * w[None, :, None] + 5.0).astype(np.float32)
    g1 = oracle.deriv_half(cfg, g, 0, 0, 5)
    assert g1.shape == (5, cfg["n_rows"] - 1, cfg["n_cols"] - 1)
    assert np.abs(g1 - 1.0).max() < 2e-3          # fp32 rounding of the inputs (|g| ~ 10, Δα ~ 6e-3)


def test_half_sample_derivative_sits_on_the_half_shifted_grid():
    """Smooth g = sin(λ + 2α) + cos(w/7): g1 = 3 cos(λ + 2α) at (λ_{k+½}, α_{l+½}) to O(Δ²) (the
    w-average of the cos(w/7) term cancels in the differences); the same values compared with the
    integer grid (λ_k, α_l) are off by O(Δ) — a half-sample slip in either variable fails."""
    cfg = _cfg(views_per_turn=120, d_alpha=2e-2, n_cols=24)
    lam, al, w = _grids(cfg, 4)
    g = (np.sin(lam[:, None, None] + 2 * al[None, None, :]) + np.cos(w[None, :, None] / 7)).astype(np.float64)
    g1 = oracle.deriv_half(cfg, g.astype(np.float32), 0, 0, 3)
    lh, ah = 0.5 * (lam[:-1] + lam[1:]), 0.5 * (al[:-1] + al[1:])
    exact_half = 3 * np.cos(lh[:3, None, None] + 2 * ah[None, None, :])
    exact_int = 3 * np.cos(lam[:3, None, None] + 2 * al[None, None, :-1])
    e_half = np.abs(g1 - exact_half).max()
    e_int = np.abs(g1 - exact_int).max()
    assert e_half < 2e-3, e_half
    assert e_int > 20 * e_half, (e_int, e_half)


def test_half_sample_grid_geometry_matches_the_scan_rays():
    """half_sample_cfg's sample (k, m, l) is the scan's ray at (λ_{k+½}, α_{l+½}, w_{m+½}): exact
    line integrals of an ellipsoid phantom on the shifted grid (independent projector, synth/)
    equal the bilinear-free mid-point integrals obtained by projecting with the physical geometry
    evaluated at those parameters (one-sample detectors placed there)."""
    cfg = _cfg(n_rows=6, n_cols=8, d_alpha=2e-2, d_w=8.0)
    vc = oracle.half_sample_cfg(cfg)
    ph = np.array([[20.0, -15.0, 5.0, 60.0, 45.0, 50.0, 0.4, 1.0], [-30.0, 10.0, -4.0, 25.0, 30.0, 20.0, -0.2, 0.5]])
    shifted = synth.project(vc, ph, 3, 2)                      # views 3, 4 of the shifted grid
    dlam = 2 * math.pi / cfg["views_per_turn"]
    h = cfg["P"] / (2 * math.pi)
    lam, al, w = _grids(cfg, 1)
    for kk in range(2):
        lk = (3 + kk + 0.5) * dlam                             # λ_{k+½}
        for m in range(cfg["n_rows"] - 1):
            wm = 0.5 * (w[m] + w[m + 1])
            for l in range(cfg["n_cols"] - 1):
                al_ = 0.5 * (al[l] + al[l + 1])
                # a one-ray detector at (α, w) = (al_, wm) on the physical helix at λ = lk: view 0 of a
                # helix started at λ0 + lk, z0 + h lk; two rows ±wm (row 1 at +wm), one column at al_
                rows = dict(n_rows=1, d_w=1.0) if wm == 0 else dict(n_rows=2, d_w=2 * abs(wm))   # a row at wm
                pt = dict(cfg, lambda0=cfg["lambda0"] + lk, z0=cfg["z0"] + h * lk, n_cols=1, d_alpha=1.0,
                          alpha_offset=al_, **rows)
                v = synth.project(pt, ph, 0, 1)[0, 0 if wm <= 0 else 1, 0]
                assert abs(v - shifted[kk, m, l]) < 1e-4 * max(1.0, abs(v)), (kk, m, l)


def test_half_sample_uniform_ball_density_and_sign():
    """The C1 uniform ball (ρ = 1) reconstructed with the half-sample derivative: interior
    mean = +ρ within 0.5 % (as the centred scheme, tests/test_oracle_recon.py), flat within 1 % (one
    detector row fewer on C1's coarse 16-row detector: std 0.53 % vs 0.4 %)."""
    cfg = configs.get("C1")
    ball = configs.ball_phantom(0.5 * cfg["P"], inner=False)
    sino = synth.project(cfg, ball, cfg["scan_v0"], cfg["scan_nv"])
    vol = oracle.reconstruct_half(cfg, sino, cfg["scan_v0"], 0, 1)
    nx = cfg["nx"]
    x = (np.arange(nx) - nx / 2) * cfg["dx"]
    z = np.arange(cfg["nz"]) * cfg["P"] / cfg["nz"]
    Z, Y, X = np.meshgrid(z, x, x, indexing="ij")
    r = np.sqrt(X ** 2 + Y ** 2 + (Z - 0.5 * cfg["P"]) ** 2)
    inner = vol[r < 90.0]
    assert abs(inner.mean() - 1.0) < 5e-3
    assert inner.std() < 1e-2


def test_half_sample_registration():
    """The off-centre small-ball registration pin with the half-sample derivative: centroid within
    0.05 voxel of the truth (a half-view slip of the shifted helix start fails it)."""
    from tests.test_oracle_recon import _centroid_error, _registration_case
    cfg, c, sino, v0 = _registration_case()
    vol = oracle.reconstruct_half(cfg, sino, v0, 0, 1)
    assert np.abs(_centroid_error(vol, cfg, c)).max() < 0.05
