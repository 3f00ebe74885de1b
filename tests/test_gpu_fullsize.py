"""Full-size parity: the BASELINE configurations in the launch configuration
bench.py times (C4: all 8 pitches in one katsevich_reconstruct call; C5: the
16-slab batch through katsevich_reconstruct_batch; C2, C3), compared with the
CPU oracle on sampled voxels the oracle computes one by one (random voxels plus
the FOV rim, the first/last slices and the last pitch).  Bar: rel L2 over the
sample <= 1e-4, max abs <= 1e-3 x phantom contrast."""
import numpy as np
import pytest

from tests.conftest import cuda_ok

pytestmark = pytest.mark.gpu

REL_L2, MAX_ABS_FRAC = 1e-4, 1e-3


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not cuda_ok():
        pytest.skip("no CUDA device")


def _samples(cfg, n, seed, slices=None):
    rng = np.random.default_rng(seed)
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    js = rng.integers(0, nz, n) if slices is None else rng.choice(slices, n)
    idx = [np.stack([rng.integers(0, nx, n), rng.integers(0, ny, n), js], 1)]
    # FOV rim and corners, first and last slice
    t = np.linspace(0, 2 * np.pi, 48, endpoint=False)
    r = 0.5 * min(nx, ny) - 1
    rim = np.stack([(nx / 2 + r * np.cos(t)).astype(int), (ny / 2 + r * np.sin(t)).astype(int)], 1)
    zs = [0, nz - 1] if slices is None else list(slices)
    for z in zs:
        idx.append(np.concatenate([rim, np.full((len(rim), 1), z)], 1))
        idx.append(np.array([[0, 0, z], [nx - 1, 0, z], [0, ny - 1, z], [nx - 1, ny - 1, z]]))
    return np.clip(np.concatenate(idx), 0, [nx - 1, ny - 1, nz - 1]).astype(np.int32)


def _oracle_voxels(cfg, sino, s0, pitch, idx):
    from oracle import oracle
    kf, kl, _, _ = oracle.bp_weights_voxels(cfg, pitch, idx)
    m = kl >= kf
    lo, hi = int(kf[m].min()), int(kl[m].max())
    gF = oracle.filter_views(cfg, sino, s0, lo, hi - lo + 1)["gF"]
    return oracle.backproject_voxels(cfg, pitch, gF, lo, idx)


def _check(got, ref, contrast):
    e = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    mx = np.abs(got - ref).max()
    assert e <= REL_L2, f"rel L2 {e:.3e}"
    assert mx <= MAX_ABS_FRAC * contrast, f"max abs {mx:.3e} vs contrast {contrast}"


def _truth_contrast(cfg, ph, pitches):
    from synth import synth
    t = np.concatenate([synth.volume_truth(dict(cfg, nx=min(cfg["nx"], 128), ny=min(cfg["ny"], 128),
                                                dx=cfg["dx"] * cfg["nx"] / min(cfg["nx"], 128),
                                                dy=cfg["dx"] * cfg["ny"] / min(cfg["ny"], 128)), ph, k)
                        for k in pitches])
    return float(t.max() - t.min())


def test_c4_all_pitches_sampled():
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs, synth
    cfg = configs.get("C4")
    p = k.Plan(cfg, device=0)
    p.precompute()
    v0, nv = p.scan_views(0, cfg["n_pitches"])
    sino = synth.project(cfg, cfg["phantom"], v0, nv)
    vol = p.reconstruct(torch.from_numpy(sino).cuda(), v0, 0, cfg["n_pitches"])
    torch.cuda.synchronize()
    contrast = _truth_contrast(cfg, cfg["phantom"], [0])
    for pitch in range(cfg["n_pitches"]):                    # every pitch of the 512^3 volume
        idx = _samples(cfg, 600 if pitch in (0, 3, 7) else 250, 1 + pitch)
        ref = _oracle_voxels(cfg, sino, v0, pitch, idx)
        g = vol[pitch * cfg["nz"]:(pitch + 1) * cfg["nz"]].cpu().numpy()
        got = g[idx[:, 2], idx[:, 1], idx[:, 0]].astype(np.float64)
        _check(got, ref, contrast)


def test_c5_batch_sampled():
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs, synth
    cfg = configs.get("C5")
    p = k.Plan(cfg, device=0)
    p.precompute()
    v0, nv = p.pitch_views(0)
    phs = configs.c5_phantoms(16)
    slabs = np.stack([synth.project(cfg, ph, v0, nv) for ph in phs])
    vols = p.reconstruct_batch(torch.from_numpy(slabs).cuda())
    torch.cuda.synchronize()
    for b in range(16):                                        # every slab of the batch
        idx = _samples(cfg, 400 if b in (0, 9, 15) else 150, 10 + b)
        ref = _oracle_voxels(cfg, slabs[b], v0, 0, idx)
        g = vols[b].cpu().numpy()
        got = g[idx[:, 2], idx[:, 1], idx[:, 0]].astype(np.float64)
        _check(got, ref, _truth_contrast(cfg, phs[b], [0]))


def test_c2_sampled():
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs, synth
    cfg = configs.get("C2")
    p = k.Plan(cfg, device=0)
    p.precompute()
    sino = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    vol = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, 2)
    torch.cuda.synchronize()
    contrast = _truth_contrast(cfg, cfg["phantom"], [0, 1])
    for pitch in (0, 1):
        idx = _samples(cfg, 500, 20 + pitch)
        ref = _oracle_voxels(cfg, sino, cfg["scan_v0"], pitch, idx)
        g = vol[pitch * cfg["nz"]:(pitch + 1) * cfg["nz"]].cpu().numpy()
        _check(g[idx[:, 2], idx[:, 1], idx[:, 0]].astype(np.float64), ref, contrast)


def test_c3_edge_and_mid_slices_sampled():
    """C3 (one pitch, the one-view TMEM kernel with end views written ahead): the first two and
    last two slices — where the fractional end weights and the window flush edges live — and a
    mid slice, each with random voxels plus the FOV rim and the grid corners."""
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs, synth
    cfg = configs.get("C3")
    p = k.Plan(cfg, device=0)
    p.precompute()
    v0, nv = p.pitch_views(0)
    sino = synth.project(cfg, cfg["phantom"], v0, nv)
    vol = p.reconstruct(torch.from_numpy(sino).cuda(), v0, 0, 1)
    torch.cuda.synchronize()
    # the oracle filters the union of the sampled voxels' PI windows (~the whole slab)
    idx = _samples(cfg, 500, 30, slices=[0, 1, 31, 62, 63])
    ref = _oracle_voxels(cfg, sino, v0, 0, idx)
    g = vol.cpu().numpy()
    _check(g[idx[:, 2], idx[:, 1], idx[:, 0]].astype(np.float64), ref, _truth_contrast(cfg, cfg["phantom"], [0]))


def _dot_check(ax, y, x, aty):
    lhs = float((ax.double() * y.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    # Cauchy-Schwarz scale: |<Ax,y>| <= |Ax||y|, the scale of the rounding of either side
    scale = max(float(ax.double().norm() * y.double().norm()), float(x.double().norm() * aty.double().norm()))
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_dot_product(name):
    """<A x, y> = <x, A^T y> at the full BASELINE size, forward and adjoint in the launch
    configuration bench.py times (C4: all 8 pitches in one call; C3: the paper's 64 x 736 detector)."""
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs
    cfg = configs.get(name)
    npit = cfg["n_pitches"]
    p = k.Plan(cfg, device=0)
    p.precompute()
    s0, sn = p.scan_views(0, npit)
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn((sn, cfg["n_rows"], cfg["n_cols"]), device="cuda", generator=g)
    y = torch.randn((npit * cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda", generator=g)
    ax = p.reconstruct(x, s0, 0, npit)
    aty = p.adjoint(y, s0, sn, 0, npit)
    torch.cuda.synchronize()
    _dot_check(ax, y, x, aty)


def test_full_size_batch_dot_product():
    """The same identity for the C5 16-slab batch (reconstruct_batch / adjoint_batch)."""
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs
    cfg = configs.get("C5")
    p = k.Plan(cfg, device=0)
    p.precompute()
    v0, nv = p.pitch_views(0)
    B = cfg["batch"]
    g = torch.Generator(device="cuda").manual_seed(12)
    x = torch.randn((B, nv, cfg["n_rows"], cfg["n_cols"]), device="cuda", generator=g)
    y = torch.randn((B, cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda", generator=g)
    ax = p.reconstruct_batch(x)
    aty = p.adjoint_batch(y)
    torch.cuda.synchronize()
    _dot_check(ax, y, x, aty)
