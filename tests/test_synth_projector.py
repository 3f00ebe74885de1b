"""Pins of the input generator (closed-form ray/ellipsoid chords)."""
import math

import numpy as np

from synth import configs, synth

SCAN = dict(R=595.0, D=1085.6, P=38.4, lambda0=0.3, z0=2.0, n_rows=5, d_w=2.0, n_cols=7, d_alpha=0.01,
            alpha_offset=0.0, views_per_turn=360)


def test_central_ray_through_sphere_is_diameter():
    # the central ray (α = 0, w = 0) of view 0 passes through the axis at height z0
    a, rho = 50.0, 0.7
    ph = np.array([[0.0, 0.0, SCAN["z0"], a, a, a, 0.0, rho]])
    g = synth.project(SCAN, ph, 0, 1)
    assert abs(g[0, 2, 3] - 2 * a * rho) < 1e-4


def test_ray_missing_everything_is_zero():
    ph = np.array([[0.0, 0.0, 500.0, 10.0, 10.0, 10.0, 0.0, 1.0]])
    assert np.abs(synth.project(SCAN, ph, 0, 3)).max() == 0.0


def _chord_by_bisection(ph, o, d, tmax=2000.0, h=0.05):
    """Line integral by locating every boundary crossing of the point-in-ellipsoid
    indicator (dense scan + bisection) — independent of the closed-form quadratic."""
    total = 0.0
    for cx, cy, cz, a, b, c, phi, rho in ph:
        def inside(t):
            p = o[None, :] + np.atleast_1d(t)[:, None] * d[None, :] - np.array([cx, cy, cz])
            u = (math.cos(phi) * p[:, 0] + math.sin(phi) * p[:, 1]) / a
            v = (-math.sin(phi) * p[:, 0] + math.cos(phi) * p[:, 1]) / b
            return u * u + v * v + (p[:, 2] / c) ** 2 <= 1.0
        t = np.arange(0.0, tmax, h)
        f = inside(t)
        edges = np.nonzero(f[1:] != f[:-1])[0]
        pts = []
        for e in edges:
            lo, hi = t[e], t[e + 1]
            flo = f[e]
            for _ in range(60):
                mid = 0.5 * (lo + hi)
                if inside(mid)[0] == flo:
                    lo = mid
                else:
                    hi = mid
            pts.append(0.5 * (lo + hi))
        assert len(pts) % 2 == 0
        total += rho * sum(pts[i + 1] - pts[i] for i in range(0, len(pts), 2))
    return total


def test_rotated_ellipsoid_matches_boundary_bisection():
    ph = np.array([[20.0, -15.0, 5.0, 60.0, 35.0, 25.0, 0.7, 1.3],
                   [-10.0, 30.0, -4.0, 40.0, 50.0, 30.0, -1.1, -0.4]])
    sc = dict(SCAN, n_rows=7, n_cols=9, d_w=6.0, d_alpha=0.02, alpha_offset=0.25)
    g = synth.project(sc, ph, 11, 2).astype(np.float64)
    checked = 0
    for iv in range(2):
        lam = (11 + iv) * 2 * math.pi / sc["views_per_turn"]
        c, s_ = math.cos(lam + sc["lambda0"]), math.sin(lam + sc["lambda0"])
        o = np.array([sc["R"] * c, sc["R"] * s_, sc["z0"] + sc["P"] * lam / (2 * math.pi)])
        for m in range(sc["n_rows"]):
            for l in range(sc["n_cols"]):
                al = (l - (sc["n_cols"] - 1) / 2 + sc["alpha_offset"]) * sc["d_alpha"]
                w = (m - (sc["n_rows"] - 1) / 2) * sc["d_w"]
                d = np.array([sc["D"] * (-math.sin(al) * s_ - math.cos(al) * c),
                              sc["D"] * (math.sin(al) * c - math.cos(al) * s_), w])
                d /= np.linalg.norm(d)
                ref = _chord_by_bisection(ph, o, d)
                assert abs(g[iv, m, l] - ref) <= 1e-6 * max(1.0, abs(ref))
                checked += ref != 0.0
    assert checked > 50


def test_infinite_cylinder_chord_independent_of_w():
    ph = np.array([[5.0, 0.0, 0.0, 70.0, 50.0, 0.0, 0.2, 1.0]])
    g = synth.project(SCAN, ph, 3, 2).astype(np.float64)
    D = SCAN["D"]
    w = (np.arange(5) - 2) * SCAN["d_w"]
    # chord along a tilted ray scales with sqrt(D² + w²)/D (the cylinder is z-invariant)
    ratio = g / g[:, 2:3, :]
    assert np.allclose(ratio, (np.sqrt(D ** 2 + w ** 2) / D)[None, :, None], rtol=1e-6)


def test_phantom_truth_and_configs():
    cfg = configs.get("C1")
    t = synth.volume_truth(cfg, cfg["phantom"], 0)
    assert t.max() == 1.5 and t.min() == 0.0
    assert configs.get("C5")["n_cols"] // 4 + 1 == 157          # α downsampling 627 -> 157 (P:l.394)
