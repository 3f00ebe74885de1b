"""GPU adjoint (NEXT-1) through the C ABI: katsevich_adjoint against the oracle's
adjoint (pinned by dot-product tests), the dot-product identity on the GPU
itself, and autograd through the layer.  Bar: rel L2 <= 1e-4 of the fp64
oracle, max abs <= 1e-3 x max|oracle| (fp32 with atomic summation)."""
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


@pytest.mark.parametrize("name,kernel", [("T1", None), ("T2", None), ("T3", None), ("C1", None),
                                         ("T2", "l1"), ("C1", "l1"), ("T3", "k4t1"), ("T3", "k4t2")])
def test_adjoint_matches_oracle(name, kernel, monkeypatch):
    """kernel None: the shared-memory box kernel (footprints on the detector);
    'l1': the checked, direct-scatter kernel (as for plans whose footprints may
    leave the detector); 'k4t1' / 'k4t2': K4^T over one / two views per thread."""
    import torch
    from oracle import oracle
    from synth import configs
    if kernel in ("k4t1", "k4t2"):
        monkeypatch.setenv("KATS_K4T_VPB", kernel[-1])
        monkeypatch.delenv("KATS_BP_KERNEL", raising=False)
    elif kernel:
        monkeypatch.setenv("KATS_BP_KERNEL", kernel)
    else:
        monkeypatch.delenv("KATS_BP_KERNEL", raising=False)
    cfg = configs.get(name)
    npit = cfg["n_pitches"]
    s0, sn = cfg["scan_v0"], cfg["scan_nv"]
    rng = np.random.default_rng(7)
    y = rng.standard_normal((npit * cfg["nz"], cfg["ny"], cfg["nx"])).astype(np.float32)
    ref = oracle.adjoint(cfg, y.astype(np.float64), 0, npit, s0, sn)
    p = _plan(cfg)
    got = p.adjoint(torch.from_numpy(y).cuda(), s0, sn, 0, npit).cpu().numpy().astype(np.float64)
    e = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    m = np.abs(got - ref).max() / np.abs(ref).max()
    assert e <= 1e-4, f"rel L2 {e:.3e}"
    assert m <= 1e-3, f"max abs / max {m:.3e}"


@pytest.mark.parametrize("name", ["T2", "C1"])
def test_gpu_dot_product(name):
    """<A x, y> = <x, A^T y> with the GPU forward and the GPU adjoint."""
    import torch
    from synth import configs
    cfg = configs.get(name)
    npit = cfg["n_pitches"]
    s0, sn = cfg["scan_v0"], cfg["scan_nv"]
    rng = np.random.default_rng(8)
    x = torch.from_numpy(rng.standard_normal((sn, cfg["n_rows"], cfg["n_cols"])).astype(np.float32)).cuda()
    y = torch.from_numpy(rng.standard_normal((npit * cfg["nz"], cfg["ny"], cfg["nx"])).astype(np.float32)).cuda()
    p = _plan(cfg)
    ax = p.reconstruct(x, s0, 0, npit)
    aty = p.adjoint(y, s0, sn, 0, npit)
    lhs = float((ax.double() * y.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    # Cauchy-Schwarz scale: |<Ax,y>| <= |Ax||y|, the scale of the rounding of either side
    scale = max(float(ax.double().norm() * y.double().norm()), float(x.double().norm() * aty.double().norm()))
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)


def test_autograd_gradient_is_the_adjoint():
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs
    cfg = configs.get("T2")
    npit = cfg["n_pitches"]
    s0, sn = cfg["scan_v0"], cfg["scan_nv"]
    p = _plan(cfg)
    rng = np.random.default_rng(9)
    x = torch.from_numpy(rng.standard_normal((sn, cfg["n_rows"], cfg["n_cols"])).astype(np.float32)).cuda()
    w = torch.from_numpy(rng.standard_normal((npit * cfg["nz"], cfg["ny"], cfg["nx"])).astype(np.float32)).cuda()
    x.requires_grad_(True)
    vol = k.autograd.reconstruct(p, x, s0, 0, npit)
    loss = (vol * w).sum()
    loss.backward()
    ref = p.adjoint(w, s0, sn, 0, npit)
    assert torch.allclose(x.grad, ref, rtol=0, atol=1e-6 * float(ref.abs().max()))
    # and the forward value is the plain reconstruction
    assert torch.equal(vol.detach(), p.reconstruct(x.detach(), s0, 0, npit))


def test_adjoint_batch_matches_oracle_and_autograd():
    """katsevich_adjoint_batch (training-shaped batches of one-pitch slabs) against the
    oracle adjoint of each slab, the batch dot-product identity, and autograd."""
    import torch
    import paper_2201_02309_b200 as k
    from oracle import oracle
    from synth import configs
    cfg = configs.get("T2")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    B = 3
    rng = np.random.default_rng(21)
    y = rng.standard_normal((B, cfg["nz"], cfg["ny"], cfg["nx"])).astype(np.float32)
    got = p.adjoint_batch(torch.from_numpy(y).cuda()).cpu().numpy().astype(np.float64)
    for b in range(B):
        ref = oracle.adjoint(cfg, y[b].astype(np.float64), 0, 1, v0, nv)
        e = np.linalg.norm(got[b] - ref) / np.linalg.norm(ref)
        assert e <= 1e-4, f"slab {b}: rel L2 {e:.3e}"
    x = torch.from_numpy(rng.standard_normal((B, nv, cfg["n_rows"], cfg["n_cols"])).astype(np.float32)).cuda()
    yy = torch.from_numpy(y).cuda()
    ax = p.reconstruct_batch(x)
    aty = p.adjoint_batch(yy)
    lhs = float((ax.double() * yy.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    scale = float(ax.double().norm() * yy.double().norm())
    assert abs(lhs - rhs) <= 1e-5 * scale
    x.requires_grad_(True)
    loss = (k.autograd.reconstruct_batch(p, x) * yy).sum()
    loss.backward()
    assert torch.allclose(x.grad, aty, rtol=0, atol=1e-6 * float(aty.abs().max()))


@pytest.mark.parametrize("name", ["C1", "T3"])
def test_adjoint_high_dynamic_range_constant_sign(name):
    """K5^T accumulates int32 fixed-point sums scaled per CTA by its largest contribution
    (backproject.cu k_bp_adjoint): with constant-sign y spanning six decades inside a tile the
    result must still match the oracle adjoint (rel L2 1e-4) — small contributions are rounded
    to 2^-22 of the tile's largest, and same-sign sums must not overflow."""
    import torch
    from oracle import oracle
    from synth import configs
    cfg = configs.get(name)
    npit = cfg["n_pitches"]
    s0, sn = cfg["scan_v0"], cfg["scan_nv"]
    rng = np.random.default_rng(9)
    y = np.exp(rng.uniform(-7.0, 7.0, (npit * cfg["nz"], cfg["ny"], cfg["nx"]))).astype(np.float32)
    ref = oracle.adjoint(cfg, y.astype(np.float64), 0, npit, s0, sn)
    got = _plan(cfg).adjoint(torch.from_numpy(y).cuda(), s0, sn, 0, npit).cpu().numpy().astype(np.float64)
    e = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert e <= 1e-4, f"rel L2 {e:.3e}"


def test_adjoint_batch_beyond_grid_z_limit():
    """A C5-geometry batch of 120 slabs: the per-slab stencil transposes and the end-view kernels
    exceed the 65535 limit of a single launch's grid.z and must be split; checked by
    the batch dot-product identity against the forward at the same size."""
    import torch
    from synth import configs
    cfg = configs.get("C5")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    B = 120
    g = torch.Generator(device="cuda").manual_seed(21)
    x = torch.randn((B, nv, cfg["n_rows"], cfg["n_cols"]), device="cuda", generator=g)
    y = torch.randn((B, cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda", generator=g)
    ax = p.reconstruct_batch(x)
    aty = p.adjoint_batch(y)
    torch.cuda.synchronize()
    lhs = float((ax.double() * y.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    scale = float(ax.double().norm() * y.double().norm())
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)
