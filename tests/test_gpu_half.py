"""GPU parity of NEXT-4, Noo's half-sample derivative (KATS_FLAG_HALF_SAMPLE; DESIGN.md reading
A25): the CUDA path through the C ABI against the oracle's half-sample reconstruction
(oracle.reconstruct_half, pinned in tests/test_oracle_half.py) on the same seeded sinograms,
the filtered views per stage, the batch entry point, the host-buffer entry point, and the
adjoint by the dot-product identity with the GPU forward.  Bars as tests/test_gpu_parity.py."""
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
    p = k.Plan(dict(cfg, flags=1), device=0)
    p.precompute()
    return p


def _case(name):
    from synth import configs, synth
    cfg = configs.get(name)
    sino = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    truth = np.concatenate([synth.volume_truth(cfg, cfg["phantom"], k) for k in range(cfg["n_pitches"])])
    return cfg, sino, float(truth.max() - truth.min())


@pytest.mark.parametrize("name", ["T1", "T2", "T3", "C1"])
def test_half_sample_reconstruct_matches_oracle(name):
    import torch
    from oracle import oracle
    cfg, sino, contrast = _case(name)
    ref = oracle.reconstruct_half(cfg, sino, cfg["scan_v0"], 0, cfg["n_pitches"])
    p = _plan(cfg)
    got = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"]).cpu().numpy()
    got = got.astype(np.float64)
    e = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert e <= 1e-4, f"rel L2 {e:.3e}"
    assert np.abs(got - ref).max() <= 1e-3 * contrast


@pytest.mark.parametrize("name", ["T1", "C1"])
def test_half_sample_filter_stages_match_oracle(name):
    """g3 and gF on the half-shifted grid (steps 1-6) within 1e-5 of the oracle."""
    import torch
    from oracle import oracle
    cfg, sino, _ = _case(name)
    vc = oracle.half_sample_cfg(cfg)
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)                        # raw views [K_lo, K_hi + 1]
    n = nv - 1
    out = p.filter(torch.from_numpy(sino).cuda(), cfg["scan_v0"], v0, n, stages=("g3", "gF"))
    torch.cuda.synchronize()
    g1 = oracle.deriv_half(cfg, sino, cfg["scan_v0"], v0, n)
    ref = oracle.filter_g1(vc, g1, stages=("g3", "gF"))
    for s in ("g3", "gF"):
        got = out[s].cpu().numpy().astype(np.float64)
        e = np.linalg.norm(got - ref[s]) / np.linalg.norm(ref[s])
        assert e <= 1e-5, f"{s}: rel L2 {e:.3e}"


def test_half_sample_batch_and_host_entry_points():
    """reconstruct_batch (3 one-pitch slabs of T2, each with its raw views K_lo .. K_hi + 1) against
    the oracle per slab; reconstruct_host equals the device path to fp32 rounding."""
    import torch
    from oracle import oracle
    from synth import configs, synth
    cfg = configs.get("T2")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    phs = [configs.shepp_logan(300.0 - 30 * b, 300.0, 0.5 * cfg["P"]) for b in range(3)]
    slabs = np.stack([synth.project(cfg, ph, v0, nv) for ph in phs])
    vols = p.reconstruct_batch(torch.from_numpy(slabs).cuda()).cpu().numpy()
    for b in range(3):
        ref = oracle.reconstruct_half(cfg, slabs[b], v0, 0, 1)
        assert np.linalg.norm(vols[b] - ref) / np.linalg.norm(ref) <= 1e-4
    sino = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    dev = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, 2).cpu().numpy()
    host = p.reconstruct_host(sino, cfg["scan_v0"], 0, 2).numpy()
    assert np.linalg.norm(host - dev) / np.linalg.norm(dev) <= 1e-6


@pytest.mark.parametrize("name", ["T3", "C1"])
def test_half_sample_adjoint_dot_product(name):
    """<A x, y> = <x, A^T y> with the half-sample forward and adjoint (K1^T of the 2x2x2 stencil)."""
    import torch
    from synth import configs
    cfg = configs.get(name)
    p = _plan(cfg)
    npit = cfg["n_pitches"]
    s0, sn = p.scan_views(0, npit)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((sn, cfg["n_rows"], cfg["n_cols"]), device="cuda", generator=g)
    y = torch.randn((npit * cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda", generator=g)
    ax = p.reconstruct(x, s0, 0, npit)
    aty = p.adjoint(y, s0, sn, 0, npit)
    torch.cuda.synchronize()
    lhs = float((ax.double() * y.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    scale = float(ax.double().norm() * y.double().norm())
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)


def test_half_sample_adjoint_batch_dot_product():
    import torch
    from synth import configs
    cfg = configs.get("T2")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    g = torch.Generator(device="cuda").manual_seed(6)
    x = torch.randn((3, nv, cfg["n_rows"], cfg["n_cols"]), device="cuda", generator=g)
    y = torch.randn((3, cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda", generator=g)
    ax = p.reconstruct_batch(x)
    aty = p.adjoint_batch(y)
    torch.cuda.synchronize()
    lhs = float((ax.double() * y.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    scale = float(ax.double().norm() * y.double().norm())
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)
