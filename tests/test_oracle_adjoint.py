"""Oracle adjoint (NEXT-1) pinned against the already-pinned
forward oracle by the dot-product identity <A x, y> = <x, A^T y>, which any
dropped term, wrong index, sign or transposed operand in A^T breaks.  Checked
per stage (backprojection, filter) and for the whole layer on several
configurations, with random x, y (fp64 arithmetic: the identity holds to
~1e-12 relative)."""
import numpy as np
import pytest

from oracle import oracle
from synth import configs

TOL = 1e-10


def _rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


@pytest.mark.parametrize("name", ["T1", "T2"])
def test_backprojection_adjoint_dot_product(name):
    cfg = configs.get(name)
    fv, nv = oracle.pitch_slab(cfg, 0)
    rng = np.random.default_rng(1)
    gF = rng.standard_normal((nv - 2, cfg["n_rows"], cfg["n_cols"]))
    y = rng.standard_normal((cfg["nz"], cfg["ny"], cfg["nx"]))
    lhs = float(np.vdot(oracle.backproject(cfg, 0, gF, fv + 1), y))
    rhs = float(np.vdot(gF, oracle.backproject_T(cfg, 0, y, fv + 1, nv - 2)))
    assert _rel(lhs, rhs) < TOL, (lhs, rhs)


@pytest.mark.parametrize("name", ["T1", "T3"])
def test_filter_adjoint_dot_product(name):
    cfg = configs.get(name)
    rng = np.random.default_rng(2)
    n_out, s0 = 9, 100
    sn = n_out + 2
    x = rng.standard_normal((sn, cfg["n_rows"], cfg["n_cols"])).astype(np.float32)
    gF = oracle.filter_views(cfg, x, s0, s0 + 1, n_out)["gF"]
    y = rng.standard_normal(gF.shape)
    lhs = float(np.vdot(gF, y))
    rhs = float(np.vdot(x.astype(np.float64), oracle.filter_T(cfg, y, s0 + 1, s0, sn)))
    assert _rel(lhs, rhs) < TOL, (lhs, rhs)


@pytest.mark.parametrize("name,pitches", [("T1", 1), ("T2", 2)])
def test_layer_adjoint_dot_product(name, pitches):
    cfg = configs.get(name)
    rng = np.random.default_rng(3)
    s0, sn = cfg["scan_v0"], cfg["scan_nv"]
    x = rng.standard_normal((sn, cfg["n_rows"], cfg["n_cols"])).astype(np.float32)
    y = rng.standard_normal((pitches * cfg["nz"], cfg["ny"], cfg["nx"]))
    lhs = float(np.vdot(oracle.reconstruct(cfg, x, s0, 0, pitches), y))
    aty = oracle.adjoint(cfg, y, 0, pitches, s0, sn)
    rhs = float(np.vdot(x.astype(np.float64), aty))
    assert _rel(lhs, rhs) < TOL, (lhs, rhs)
    # views outside every slab receive nothing
    fv, nv = oracle.pitch_slab(cfg, 0)
    assert np.all(aty[: fv - s0] == 0.0)


def test_adjoint_is_linear_and_zero_preserving():
    cfg = configs.get("T1")
    s0, sn = cfg["scan_v0"], cfg["scan_nv"]
    shape = (cfg["nz"], cfg["ny"], cfg["nx"])
    rng = np.random.default_rng(4)
    a, b = rng.standard_normal(shape), rng.standard_normal(shape)
    assert np.all(oracle.adjoint(cfg, np.zeros(shape), 0, 1, s0, sn) == 0.0)
    lhs = oracle.adjoint(cfg, 2.0 * a - 3.0 * b, 0, 1, s0, sn)
    rhs = 2.0 * oracle.adjoint(cfg, a, 0, 1, s0, sn) - 3.0 * oracle.adjoint(cfg, b, 0, 1, s0, sn)
    assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()
