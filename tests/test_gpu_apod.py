"""GPU parity of NEXT-4's Hann-apodised Hilbert filter (KATS_FLAG_HANN; reading A26)
through the C ABI against the oracle (pinned in tests/test_oracle_apod.py): the volume, the filter
stages for each K3 kernel, the combination with the half-sample derivative, the host and batch
entry points, and the adjoint's dot-product identity.  Bars as tests/test_gpu_parity.py."""
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


def _case(name, flags):
    from synth import configs, synth
    cfg = dict(configs.get(name), flags=flags)
    sino = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    truth = np.concatenate([synth.volume_truth(cfg, cfg["phantom"], k) for k in range(cfg["n_pitches"])])
    return cfg, sino, float(truth.max() - truth.min())


@pytest.mark.parametrize("name,flags", [("T1", 2), ("T3", 2), ("C1", 2), ("T2", 3), ("C1", 3)])
def test_apodised_reconstruct_matches_oracle(name, flags):
    """flags 2: Hann-apodised Hilbert; 3: with the half-sample derivative as well."""
    import torch
    from oracle import oracle
    cfg, sino, contrast = _case(name, flags)
    rec = oracle.reconstruct_half if flags & 1 else oracle.reconstruct
    ref = rec(cfg, sino, cfg["scan_v0"], 0, cfg["n_pitches"])
    got = _plan(cfg).reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"])
    got = got.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-4
    assert np.abs(got - ref).max() <= 1e-3 * contrast


@pytest.mark.parametrize("hilbert", ["default", "ws", "tc", "fp32"])
def test_apodised_filter_stages_match_oracle(hilbert, monkeypatch):
    import torch
    from oracle import oracle
    if hilbert == "default":
        monkeypatch.delenv("KATS_HILBERT", raising=False)
    else:
        monkeypatch.setenv("KATS_HILBERT", hilbert)
    cfg, sino, _ = _case("C1", 2)
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    out = p.filter(torch.from_numpy(sino).cuda(), cfg["scan_v0"], v0 + 1, nv - 2, stages=("g3", "g4", "gF"))
    torch.cuda.synchronize()
    ref = oracle.filter_views(cfg, sino, cfg["scan_v0"], v0 + 1, nv - 2, stages=("g3", "g4", "gF"))
    for s in ("g3", "g4", "gF"):
        got = out[s].cpu().numpy().astype(np.float64)
        e = np.linalg.norm(got - ref[s]) / np.linalg.norm(ref[s])
        assert e <= 1e-5, f"{s}: rel L2 {e:.3e}"


@pytest.mark.parametrize("name", ["T3", "C1"])
def test_apodised_adjoint_dot_product(name):
    import torch
    from synth import configs
    cfg = dict(configs.get(name), flags=2)
    p = _plan(cfg)
    npit = cfg["n_pitches"]
    s0, sn = p.scan_views(0, npit)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn((sn, cfg["n_rows"], cfg["n_cols"]), device="cuda", generator=g)
    y = torch.randn((npit * cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda", generator=g)
    ax = p.reconstruct(x, s0, 0, npit)
    aty = p.adjoint(y, s0, sn, 0, npit)
    torch.cuda.synchronize()
    lhs = float((ax.double() * y.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    assert abs(lhs - rhs) <= 1e-5 * float(ax.double().norm() * y.double().norm())


def test_apodised_batch_and_host_entry_points():
    import torch
    from oracle import oracle
    from synth import configs, synth
    cfg = dict(configs.get("T2"), flags=2)
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    slabs = np.stack([synth.project(cfg, configs.random_ellipsoids(40 + b, 6, 180.0, -5.0, cfg["P"] + 5.0), v0, nv)
                      for b in range(4)])
    vols = p.reconstruct_batch(torch.from_numpy(slabs).cuda()).cpu().numpy()
    for b in (0, 3):
        ref = oracle.reconstruct(cfg, slabs[b], v0, 0, 1)
        assert np.linalg.norm(vols[b] - ref) / np.linalg.norm(ref) <= 1e-4
    sino = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    dev = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, 2).cpu().numpy()
    host = p.reconstruct_host(sino, cfg["scan_v0"], 0, 2).numpy()
    assert np.linalg.norm(host - dev) / np.linalg.norm(dev) <= 1e-6
