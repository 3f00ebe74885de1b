"""GPU data generation (NEXT-3) through the C ABI against the oracle: analytic
and ray-marched projectors (fp32 output vs fp64 oracle), the α resampling, and
the noise model (Poisson draws bit-exact: both sides run the same Philox4x32-10
stream and the same fp64 PTRS decisions; outputs to fp32 rounding)."""
import numpy as np
import pytest

from tests.conftest import cuda_ok

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not cuda_ok():
        pytest.skip("no CUDA device")


def _plan(cfg):
    import paper_2201_02309_b200 as k
    p = k.Plan(cfg, device=0)
    p.precompute()
    return p


@pytest.mark.parametrize("name", ["T2", "T3", "C1"])
def test_project_ellipsoids_matches_oracle(name):
    from oracle import oracle
    from synth import configs
    cfg = configs.get(name)
    p = _plan(cfg)
    v0, nv = cfg["scan_v0"], min(cfg["scan_nv"], 40)
    got = p.project_ellipsoids(cfg["phantom"], v0, nv).cpu().numpy().astype(np.float64)
    ref = oracle.project_ellipsoids(cfg, cfg["phantom"], v0, nv)
    assert np.abs(got - ref).max() <= 1e-6 * max(1.0, np.abs(ref).max())


def test_project_volume_matches_oracle():
    import torch
    from oracle import oracle
    from synth import configs
    cfg = dict(configs.get("T2"), nx=64, ny=64, dx=4.0, dy=4.0, r_fov=0.0)
    import paper_2201_02309_b200 as k
    p = k.Plan(cfg, device=0)                                 # projection needs the geometry only
    rng = np.random.default_rng(5)
    nzv, zv0, dzv = 24, -40.0, 3.5
    vol = rng.uniform(0.0, 1.0, (nzv, cfg["ny"], cfg["nx"])).astype(np.float32)
    got, nt = p.project_volume(torch.from_numpy(vol).cuda(), zv0, dzv, -3, 6)
    ref, nt_ref = oracle.project_volume(cfg, vol, zv0, dzv, -3, 6)
    got = got.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-5
    assert np.abs(got - ref).max() <= 1e-4 * np.abs(ref).max()
    assert abs(nt - nt_ref) <= max(2, 0.01 * nt_ref)


@pytest.mark.parametrize("name", ["T1", "T3"])
def test_degrade_matches_oracle(name):
    import torch
    from oracle import oracle
    from synth import configs
    cfg = configs.get(name)
    p = _plan(cfg)
    v0, nv = 17, 30
    rng = np.random.default_rng(6)
    g = rng.uniform(0.0, 400.0, (nv, cfg["n_rows"], cfg["n_cols"])).astype(np.float32)
    out, counts, M = p.degrade(torch.from_numpy(g).cuda(), v0, alpha_stride=4, seed=11, return_counts=True)
    up = oracle.resample_alpha(cfg, g.astype(np.float64), 4)
    # the noise step on the same (fp32-rounded) upsampled values the GPU used
    up32 = up.astype(np.float32).astype(np.float64)
    ref, cref, Mref = oracle.add_noise(cfg, up32, v0, I0=1e5, var=0.5, seed=11)
    assert float(M.item()) == np.float32(Mref)
    c = counts.cpu().numpy()
    assert (c == cref).mean() >= 1 - 1e-5                     # Poisson draws: integer decisions in fp64 on both sides
    o = out.cpu().numpy().astype(np.float64)
    same = c == cref
    assert np.abs(o[same] - ref[same]).max() <= 1e-5 * Mref
    # noiseless mode returns the upsampled data
    z = p.degrade(torch.from_numpy(g).cuda(), v0, mode=1).cpu().numpy().astype(np.float64)
    assert np.abs(z - up32).max() <= 1e-5 * Mref
