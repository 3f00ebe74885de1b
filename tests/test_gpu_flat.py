"""GPU parity of NEXT-4's flat-detector variant (KATS_FLAG_FLAT; reading A27): the CUDA path
through the C ABI against the oracle's flat reconstruction (pinned in tests/test_oracle_flat.py) on the
same seeded flat-detector sinograms — every step-7 kernel, the filtered views per stage, the batch and
host-buffer entry points, a full-size configuration on sampled voxels, the adjoint (dot-product identity
with the GPU forward, and against the oracle's adjoint) and the GPU projector.  Bars as
tests/test_gpu_parity.py."""
import numpy as np
import pytest

from tests.conftest import cuda_ok

pytestmark = pytest.mark.gpu

REL_L2, MAX_ABS_FRAC, STAGE_REL = 1e-4, 1e-3, 1e-5


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not cuda_ok():
        pytest.skip("no CUDA device")


def _plan(cfg):
    import paper_2201_02309_b200 as k
    p = k.Plan(cfg, device=0)
    p.precompute()
    return p


def _case(name):
    from synth import configs, synth
    cfg = configs.get(name)
    sino = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    truth = np.concatenate([synth.volume_truth(cfg, cfg["phantom"], k) for k in range(cfg["n_pitches"])])
    return cfg, sino, float(truth.max() - truth.min())


def _check(got, ref, contrast):
    got = np.asarray(got, dtype=np.float64)
    e = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert e <= REL_L2, f"rel L2 {e:.3e}"
    assert np.abs(got - ref).max() <= MAX_ABS_FRAC * contrast


@pytest.mark.parametrize("kernel", [None, "window", "tmem", "l1"])
def test_flat_reconstruct_matches_oracle(kernel, monkeypatch):
    """TF1 (3 pitches, ragged grid) with the default step-7 kernel (the small-grid L1 kernel) and each
    staged kernel forced: their flat column (u*/Δu = (D/Δu) u/v*) and row (D (z - z_src)/v*) maps."""
    import torch
    from oracle import oracle
    if kernel is None:
        monkeypatch.delenv("KATS_BP_KERNEL", raising=False)
    else:
        monkeypatch.setenv("KATS_BP_KERNEL", kernel)
    cfg, sino, contrast = _case("TF1")
    ref = oracle.reconstruct(cfg, sino, cfg["scan_v0"], 0, cfg["n_pitches"])
    p = _plan(cfg)
    got = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"]).cpu().numpy()
    if kernel in ("window", "tmem"):
        assert p.bp_kernel() == "k_bp_" + kernel
    _check(got, ref, contrast)


def test_flat_filter_stages_match_oracle():
    """g3 (steps 1-3: flat derivative, 2-D length weight, flat κ-lines), g4 (step 4: 1/(π(u-u')) on the
    tensor cores) and gF (steps 5-6, no post-cosine) within 1e-5 of the oracle."""
    import torch
    from oracle import oracle
    cfg, sino, _ = _case("TF1")
    p = _plan(cfg)
    v0, n = cfg["scan_v0"] + 3, 40
    out = p.filter(torch.from_numpy(sino).cuda(), cfg["scan_v0"], v0, n, stages=("g3", "g4", "gF"))
    torch.cuda.synchronize()
    ref = oracle.filter_views(cfg, sino, cfg["scan_v0"], v0, n, stages=("g3", "g4", "gF"))
    for s in ("g3", "g4", "gF"):
        got = out[s].cpu().numpy().astype(np.float64)
        e = np.linalg.norm(got - ref[s]) / np.linalg.norm(ref[s])
        assert e <= STAGE_REL, f"{s}: rel L2 {e:.3e}"


def test_flat_batch_and_host_entry_points():
    import torch
    from oracle import oracle
    from synth import configs, synth
    cfg = configs.get("TF1")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    phs = [configs.shepp_logan(110.0 - 15 * b, 80.0, 0.5 * cfg["P"]) for b in range(3)]
    slabs = np.stack([synth.project(cfg, ph, v0, nv) for ph in phs])
    vols = p.reconstruct_batch(torch.from_numpy(slabs).cuda()).cpu().numpy()
    for b in range(3):
        ref = oracle.reconstruct(cfg, slabs[b], v0, 0, 1)
        assert np.linalg.norm(vols[b] - ref) / np.linalg.norm(ref) <= REL_L2
    sino = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    dev = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, 3).cpu().numpy()
    host = p.reconstruct_host(sino, cfg["scan_v0"], 0, 3).numpy()
    assert np.linalg.norm(host - dev) / np.linalg.norm(dev) <= 1e-6


def test_flat_full_size_c2f_sampled():
    """C2F (C2's 256^2 x 64 volume, flat 36 x 368 detector, 2 pitches in one call, the window kernel)
    against the oracle on sampled voxels of both pitches (random, FOV rim, first/last slices)."""
    import torch
    from tests.test_gpu_fullsize import _samples, _oracle_voxels
    from synth import configs, synth
    cfg = configs.get("C2F")
    sino = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    p = _plan(cfg)
    vol = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, 2).cpu().numpy()
    assert p.bp_kernel() in ("k_bp_window", "k_bp_tmem")
    nz = cfg["nz"]
    for pitch in (0, 1):
        idx = _samples(cfg, 300, 10 + pitch)
        ref = _oracle_voxels(cfg, sino, cfg["scan_v0"], pitch, idx)
        got = vol[pitch * nz + idx[:, 2], idx[:, 1], idx[:, 0]].astype(np.float64)
        e = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert e <= REL_L2, f"pitch {pitch}: rel L2 {e:.3e}"
        assert np.abs(got - ref).max() <= MAX_ABS_FRAC


def test_flat_adjoint_dot_product_and_oracle():
    """<A x, y> = <x, A^T y> with the flat forward and adjoint (K1^T with the u and w stencils, K2^T with
    the 2-D length weight), and A^T y against the oracle's flat adjoint."""
    import torch
    from oracle import oracle
    from synth import configs
    cfg = configs.get("TF1")
    p = _plan(cfg)
    s0, sn = p.scan_views(0, 1)
    g = torch.Generator(device="cuda").manual_seed(8)
    x = torch.randn((sn, cfg["n_rows"], cfg["n_cols"]), device="cuda", generator=g)
    y = torch.randn((cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda", generator=g)
    ax = p.reconstruct(x, s0, 0, 1)
    aty = p.adjoint(y, s0, sn, 0, 1)
    torch.cuda.synchronize()
    lhs = float((ax.double() * y.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    scale = float(ax.double().norm() * y.double().norm())
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)
    ref = oracle.adjoint(cfg, y.cpu().numpy().astype(np.float64), 0, 1, s0, sn)
    got = aty.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-4


def test_flat_gpu_projector_matches_synth():
    """katsevich_project_ellipsoids on a flat-detector plan: exact chords along the flat rays."""
    import torch
    from synth import configs, synth
    cfg = configs.get("TF1")
    p = _plan(cfg)
    v0, nv = cfg["scan_v0"], 60
    got = p.project_ellipsoids(cfg["phantom"], v0, nv).cpu().numpy().astype(np.float64)
    ref = synth.project(cfg, cfg["phantom"], v0, nv).astype(np.float64)
    assert np.abs(got - ref).max() <= 1e-4 * np.abs(ref).max()


@pytest.mark.parametrize("n_slabs", [4, 2])
def test_flat_batch_window_kernel_matches_oracle(n_slabs, monkeypatch):
    """C5-shaped flat slabs (TF2: 10 slices, 18 rows) through the window kernel forced past the small-grid
    rule: four slabs per CTA on the byte ring of row-cropped boxes (4 slabs), two per CTA (2 slabs)."""
    import torch
    from oracle import oracle
    from synth import configs, synth
    monkeypatch.setenv("KATS_BP_KERNEL", "window")
    monkeypatch.delenv("KATS_BP_WINV", raising=False)
    cfg = configs.get("TF2")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    slabs, refs = [], []
    for b in range(n_slabs):
        ph = configs.random_ellipsoids(200 + b, 6, 180.0, -5.0, cfg["P"] + 5.0)
        slabs.append(synth.project(cfg, ph, v0, nv))
        refs.append(oracle.reconstruct(cfg, slabs[-1], v0, 0, 1))
    got = p.reconstruct_batch(torch.from_numpy(np.stack(slabs)).cuda()).cpu().numpy()
    assert p.bp_kernel() == "k_bp_window"
    for b in range(n_slabs):
        e = np.linalg.norm(got[b] - refs[b]) / np.linalg.norm(refs[b])
        assert e <= REL_L2, f"slab {b}: rel L2 {e:.3e}"


def test_flat_with_hann_filter_matches_oracle():
    """KATS_FLAG_FLAT | KATS_FLAG_HANN: the apodised kernel on the flat κ-lines."""
    import torch
    from oracle import oracle
    cfg, sino, contrast = _case("TF1")
    cfg = dict(cfg, flags=cfg["flags"] | 2)
    ref = oracle.reconstruct(cfg, sino, cfg["scan_v0"], 0, cfg["n_pitches"])
    p = _plan(cfg)
    got = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"]).cpu().numpy()
    _check(got, ref, contrast)


def test_flat_adjoint_batch_dot_product():
    """katsevich_adjoint_batch on flat slabs (TF2): <A x, y> = <x, A^T y> with the batch forward."""
    import torch
    from synth import configs
    cfg = configs.get("TF2")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn((2, nv, cfg["n_rows"], cfg["n_cols"]), device="cuda", generator=g)
    y = torch.randn((2, cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda", generator=g)
    ax = p.reconstruct_batch(x)
    aty = p.adjoint_batch(y)
    torch.cuda.synchronize()
    lhs = float((ax.double() * y.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    scale = float(ax.double().norm() * y.double().norm())
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)
