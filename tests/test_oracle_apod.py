"""Oracle pins — NEXT-4, the Hann-apodised Hilbert filter (KATS_FLAG_HANN = 2, DESIGN.md reading
A26): step 4's kernel response -i sgn(σ) multiplied by the Hann window cos²(πσΔα) (1 at DC, 0 at
the Nyquist frequency), i.e. the band-limited kernel of reading A10 applied to the κ-line smoothed
by [1/4, 1/2, 1/4] along α.  Pinned by the delta response (closed form), the frequency response of
a sinusoid (the window, exactly, away from the detector edges), the ball density, and the adjoint's
dot-product identity."""
import math

import numpy as np

from oracle import oracle
from synth import configs, synth
from tests.test_oracle_filter import _cfg, _grid, _view_trick_sino


def _g4(cfg, H):
    """g4 of one view whose κ-lines all carry H (view trick: every κ-line sample on the rows)."""
    al, w = _grid(cfg)
    cw = np.sqrt(cfg["D"] ** 2 + w ** 2) / cfg["D"]
    g = _view_trick_sino(cfg, cw, H).astype(np.float32)
    return oracle.filter_views(cfg, g, -1, 0, 1, stages=("g3", "g4"))


def test_apodised_delta_response_closed_form():
    """A delta at column l0: g4[l] = ½K[l-l0] + ¼K[l-l0+1] + ¼K[l-l0-1] (K: reading A10's closed
    form), against the un-apodised kernel's own delta response K[l-l0]."""
    cfg = _cfg(n_rows=64, d_w=40.0, n_cols=41, flags=2)
    l0 = 20
    H = np.zeros(cfg["n_cols"]); H[l0] = 1.0
    out = _g4(cfg, H)
    g3, g4 = out["g3"][0], out["g4"][0]
    assert np.abs(g3 - g3[0][None, :]).max() < 1e-6 and abs(g3[0, l0] - 1.0) < 1e-6   # κ-lines unsmoothed
    da, nc = cfg["d_alpha"], cfg["n_cols"]
    K = lambda d: (2 * da / (math.pi * math.sin(d * da))) if d % 2 else 0.0
    want = np.array([0.5 * K(l - l0) + 0.25 * K(l - l0 + 1) + 0.25 * K(l - l0 - 1) for l in range(nc)])
    assert np.abs(g4[0] - want).max() < 1e-6 * np.abs(want).max()
    plain = _g4(dict(cfg, flags=0), H)["g4"][0, 0]
    assert np.abs(plain - np.array([K(l - l0) for l in range(nc)])).max() < 1e-6


def test_apodised_frequency_response_is_hann():
    """A sinusoid of f cycles per column on a long κ-line: away from the edges the apodised output
    is the plain output times cos²(πf) (the Hann window at that frequency), for several f."""
    cfg = _cfg(n_rows=64, d_w=40.0, n_cols=401, d_alpha=1e-3, flags=2)
    l = np.arange(cfg["n_cols"])
    mid = slice(150, 251)
    for f in (0.05, 0.15, 0.3, 0.45):
        H = np.cos(2 * math.pi * f * l)
        a = _g4(cfg, H)["g4"][0, 0]
        b = _g4(dict(cfg, flags=0), H)["g4"][0, 0]
        # interior: the smoothing of a pure cosine is exact except next to the edges (zeros beyond)
        ratio = np.dot(a[mid], b[mid]) / np.dot(b[mid], b[mid])
        assert abs(ratio - math.cos(math.pi * f) ** 2) < 2e-3, (f, ratio)


def test_apodised_uniform_ball_density():
    """The C1 uniform ball with the apodised filter: interior mean = +ρ within 0.5 % (the window is
    1 at DC), flat within 1 %."""
    cfg = dict(configs.get("C1"), flags=2)
    ball = configs.ball_phantom(0.5 * cfg["P"], inner=False)
    sino = synth.project(cfg, ball, cfg["scan_v0"], cfg["scan_nv"])
    vol = oracle.reconstruct(cfg, sino, cfg["scan_v0"], 0, 1)
    nx = cfg["nx"]
    x = (np.arange(nx) - nx / 2) * cfg["dx"]
    z = np.arange(cfg["nz"]) * cfg["P"] / cfg["nz"]
    Z, Y, X = np.meshgrid(z, x, x, indexing="ij")
    r = np.sqrt(X ** 2 + Y ** 2 + (Z - 0.5 * cfg["P"]) ** 2)
    inner = vol[r < 90.0]
    assert abs(inner.mean() - 1.0) < 5e-3
    assert inner.std() < 1e-2


def test_apodised_adjoint_dot_product():
    """<A x, y> = <x, A^T y> with the apodised forward and adjoint (T1, one pitch)."""
    cfg = dict(configs.get("T1"), flags=2)
    s0, sn = cfg["scan_v0"], cfg["scan_nv"]
    rng = np.random.default_rng(3)
    x = rng.standard_normal((sn, cfg["n_rows"], cfg["n_cols"])).astype(np.float32)
    y = rng.standard_normal((cfg["nz"], cfg["ny"], cfg["nx"]))
    ax = oracle.reconstruct(cfg, x, s0, 0, 1)
    aty = oracle.adjoint(cfg, y, 0, 1, s0, sn)
    lhs, rhs = float((ax * y).sum()), float((x.astype(np.float64) * aty).sum())
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), 1e-30) + 1e-12 * np.linalg.norm(ax) * np.linalg.norm(y)
