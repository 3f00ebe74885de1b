"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded synthetic inputs.  Bar (BASELINE.json north_star): integer tables
bit-exact; fp32 volume rel L2 <= 1e-4 and max-abs <= 1e-3 x phantom contrast.
Per-stage intermediates: rel L2 <= 1e-5 (fp32 arithmetic vs fp64)."""
import functools

import numpy as np
import pytest

from tests.conftest import cuda_ok

pytestmark = pytest.mark.gpu

REL_L2 = 1e-4
MAX_ABS_FRAC = 1e-3
STAGE_REL = 1e-5


@functools.lru_cache(maxsize=None)
def _case(name):
    from oracle import oracle
    from synth import configs, synth
    cfg = configs.get(name)
    sino = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    ref = oracle.reconstruct(cfg, sino, cfg["scan_v0"], 0, cfg["n_pitches"])
    truth = np.concatenate([synth.volume_truth(cfg, cfg["phantom"], k) for k in range(cfg["n_pitches"])])
    return cfg, sino, ref, float(truth.max() - truth.min())


def _plan(cfg):
    import paper_2201_02309_b200 as k
    p = k.Plan(cfg, device=0)
    p.precompute()
    return p


def _check(got, ref, contrast, rel=REL_L2, frac=MAX_ABS_FRAC):
    got = np.asarray(got, dtype=np.float64)
    e = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)
    m = np.abs(got - ref).max()
    assert e <= rel, f"rel L2 {e:.3e} > {rel}"
    assert m <= frac * contrast, f"max abs {m:.3e} > {frac} x contrast {contrast:.3g}"
    return e, m


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not cuda_ok():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", ["T1", "T2", "T3", "C1"])
def test_reconstruct_matches_oracle(name):
    import torch
    cfg, sino, ref, contrast = _case(name)
    p = _plan(cfg)
    vol = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"])
    torch.cuda.synchronize()
    _check(vol.cpu().numpy(), ref, contrast)


@pytest.mark.parametrize("hilbert", ["default", "tc", "hk", "hk1", "ws", "fp32"])
@pytest.mark.parametrize("name", ["T1", "T3", "C1"])
def test_filter_stages_match_oracle(name, hilbert, monkeypatch):
    """Steps 1-6 per stage (g3, g4, gF) against the oracle; K3 on the tensor cores
    (3xTF32 GEMM: default choice, tap-streaming kernels, Hankel-core kernel) and as
    the fp32 direct convolution."""
    import torch
    from oracle import oracle
    if hilbert == "default":
        monkeypatch.delenv("KATS_HILBERT", raising=False)
    else:
        monkeypatch.setenv("KATS_HILBERT", hilbert)
    cfg, sino, _, _ = _case(name)
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    out = p.filter(torch.from_numpy(sino).cuda(), cfg["scan_v0"], v0 + 1, nv - 2, stages=("g3", "g4", "gF"))
    torch.cuda.synchronize()
    ref = oracle.filter_views(cfg, sino, cfg["scan_v0"], v0 + 1, nv - 2, stages=("g3", "g4", "gF"))
    for s in ("g3", "g4", "gF"):
        got = out[s].cpu().numpy().astype(np.float64)
        e = np.linalg.norm(got - ref[s]) / np.linalg.norm(ref[s])
        assert e <= STAGE_REL, f"{s}: rel L2 {e:.3e}"


@pytest.mark.parametrize("name", ["T1", "T2", "C1"])
def test_backproject_only_matches_oracle(name):
    """K5 alone, fed with the oracle's filtered views (rounded to fp32)."""
    import torch
    from oracle import oracle
    cfg, sino, _, contrast = _case(name)
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    gF = oracle.filter_views(cfg, sino, cfg["scan_v0"], v0 + 1, nv - 2)["gF"]
    gF32 = gF.astype(np.float32)
    ref = oracle.backproject(cfg, 0, gF32.astype(np.float64), v0 + 1)
    got = p.backproject(torch.from_numpy(gF32).cuda(), v0 + 1, 0)
    torch.cuda.synchronize()
    _check(got.cpu().numpy(), ref, contrast)


@pytest.mark.parametrize("n_slabs,winv,k12", [(3, None, None), (4, None, None), (4, "0", None), (3, None, "colv4")])
def test_batch_matches_oracle(n_slabs, winv, k12, monkeypatch):
    """Independent one-pitch slabs (C5-shaped, small): reconstruct_batch, odd and
    even batches (even batches may pair items per CTA in the window kernel), and
    the plain window kernel forced (KATS_BP_WINV=0), and K12 over 4 views per thread across
    slab ends (KATS_K12=colv4)."""
    import torch
    if k12 is None:
        monkeypatch.delenv("KATS_K12", raising=False)
    else:
        monkeypatch.setenv("KATS_K12", k12)
    from oracle import oracle
    from synth import configs, synth
    if winv is None:
        monkeypatch.delenv("KATS_BP_WINV", raising=False)
    else:
        monkeypatch.setenv("KATS_BP_WINV", winv)
    cfg = configs.get("T2")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    slabs, refs, contrasts = [], [], []
    for s in range(n_slabs):
        ph = configs.random_ellipsoids(s, 6, 180.0, -5.0, cfg["P"] + 5.0)
        sino = synth.project(cfg, ph, v0, nv)
        slabs.append(sino)
        refs.append(oracle.reconstruct(cfg, sino, v0, 0, 1))
        t = synth.volume_truth(cfg, ph, 0)
        contrasts.append(t.max() - t.min())
    got = p.reconstruct_batch(torch.from_numpy(np.stack(slabs)).cuda())
    torch.cuda.synchronize()
    for b in range(n_slabs):
        _check(got[b].cpu().numpy(), refs[b], contrasts[b])


@pytest.mark.parametrize("n_slabs,winv,crop", [(4, None, None), (8, None, None), (2, None, None), (4, "2", None),
                                              (4, "3", "0"), (4, "1", "1"), (3, "0", "1")])
def test_batch_window_kernel_matches_oracle(n_slabs, winv, crop, monkeypatch):
    """The window kernel on C5-shaped slabs (T2), forced past the small-grid rule: four slabs per
    CTA on the byte ring of row-cropped boxes (the default for batches of 4k slabs: C5), two slabs
    per CTA (ring), one slab, and the fixed-slot full-column boxes (KATS_BP_CROP=0)."""
    import torch
    from oracle import oracle
    from synth import configs, synth
    monkeypatch.setenv("KATS_BP_KERNEL", "window")
    for var, val in (("KATS_BP_WINV", winv), ("KATS_BP_CROP", crop)):
        if val is None:
            monkeypatch.delenv(var, raising=False)
        else:
            monkeypatch.setenv(var, val)
    cfg = configs.get("T2")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    slabs, refs, contrasts = [], [], []
    for s in range(n_slabs):
        ph = configs.random_ellipsoids(100 + s, 6, 180.0, -5.0, cfg["P"] + 5.0)
        sino = synth.project(cfg, ph, v0, nv)
        slabs.append(sino)
        refs.append(oracle.reconstruct(cfg, sino, v0, 0, 1))
        t = synth.volume_truth(cfg, ph, 0)
        contrasts.append(t.max() - t.min())
    got = p.reconstruct_batch(torch.from_numpy(np.stack(slabs)).cuda())
    torch.cuda.synchronize()
    assert p.bp_kernel() == "k_bp_window"
    for b in range(n_slabs):
        _check(got[b].cpu().numpy(), refs[b], contrasts[b])


def test_host_entry_point_matches_device():
    """The host entry point (copies overlapped; its K3 runs beside the backprojection as the
    fp32 direct convolution) agrees with the device path to fp32 rounding, and with the oracle."""
    import torch
    cfg, sino, ref, contrast = _case("T3")
    p = _plan(cfg)
    h = p.reconstruct_host(sino, cfg["scan_v0"], 0, cfg["n_pitches"])
    d = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"])
    torch.cuda.synchronize()
    hh, dd = h.numpy().astype(np.float64), d.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(hh - dd) <= 1e-6 * np.linalg.norm(dd)
    _check(h.numpy(), ref, contrast)


def test_deterministic_and_pitch_periodic():
    """Bitwise determinism; identical slabs at different pitches give bitwise
    identical volumes (same periodic tables, pitch-relative arithmetic)."""
    import torch
    cfg, sino, _, _ = _case("T2")
    p = _plan(cfg)
    vt = cfg["views_per_turn"]
    v0, nv = p.pitch_views(0)
    slab = sino[v0 - cfg["scan_v0"]: v0 - cfg["scan_v0"] + nv]
    a = p.reconstruct(torch.from_numpy(np.ascontiguousarray(slab)).cuda(), v0, 0, 1)
    b = p.reconstruct(torch.from_numpy(np.ascontiguousarray(slab)).cuda(), v0 + 5 * vt, 5, 1)
    c = p.reconstruct(torch.from_numpy(np.ascontiguousarray(slab)).cuda(), v0, 0, 1)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(a, c)


def test_coverage_error_names_pitches():
    import torch
    import paper_2201_02309_b200 as k
    cfg, sino, _, _ = _case("T1")
    p = _plan(cfg)
    with pytest.raises(k.KatsevichError) as ei:
        p.reconstruct(torch.from_numpy(sino[:40]).cuda(), cfg["scan_v0"], 0, 1)
    assert ei.value.code == -4 and "reconstructible" in str(ei.value)


@pytest.mark.parametrize("n_slabs,var,val", [(4, "KATS_BATCH_GROUPS", "2"), (8, "KATS_BATCH_GROUPS", "4"),
                                              (6, "KATS_BATCH_GROUPS", "3"), (7, "KATS_BATCH_SPLIT", "3,4"),
                                              (5, "KATS_BATCH_SPLIT", "1,2,2")])
def test_batch_groups_match_oracle(n_slabs, var, val, monkeypatch):
    """reconstruct_batch in slab groups (KATS_BATCH_GROUPS: group g+1 filtered while group g
    backprojects; KATS_BATCH_SPLIT: uneven groups) against the oracle per slab."""
    import torch
    from oracle import oracle
    from synth import configs, synth
    monkeypatch.delenv("KATS_BATCH_GROUPS", raising=False)
    monkeypatch.delenv("KATS_BATCH_SPLIT", raising=False)
    monkeypatch.setenv(var, val)
    cfg = configs.get("T2")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    slabs, refs = [], []
    for s in range(n_slabs):
        ph = configs.random_ellipsoids(30 + s, 6, 180.0, -5.0, cfg["P"] + 5.0)
        sino = synth.project(cfg, ph, v0, nv)
        slabs.append(sino)
        refs.append(oracle.reconstruct(cfg, sino, v0, 0, 1))
    got = p.reconstruct_batch(torch.from_numpy(np.stack(slabs)).cuda())
    torch.cuda.synchronize()
    for b in range(n_slabs):
        _check(got[b].cpu().numpy(), refs[b], 1.0)


@pytest.mark.parametrize("n_slabs,ni", [(4, "4"), (6, "2"), (3, "3")])
def test_batch_items_kernel_matches_oracle(n_slabs, ni, monkeypatch):
    """The items kernel (batches whose windows hold <= 8 slices, the default for C5-shaped batches:
    the slabs of a CTA share each view's geometry, per-lane window-relative TMEM accumulators)
    forced on T2 with 4, 2 and 3 slabs per CTA, against the oracle per slab."""
    import torch
    from oracle import oracle
    from synth import configs, synth
    monkeypatch.setenv("KATS_BP_ITEMS", ni)
    cfg = configs.get("T2")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    slabs, refs, contrasts = [], [], []
    for s in range(n_slabs):
        ph = configs.random_ellipsoids(10 + s, 6, 180.0, -5.0, cfg["P"] + 5.0)
        sino = synth.project(cfg, ph, v0, nv)
        slabs.append(sino)
        refs.append(oracle.reconstruct(cfg, sino, v0, 0, 1))
        t = synth.volume_truth(cfg, ph, 0)
        contrasts.append(t.max() - t.min())
    got = p.reconstruct_batch(torch.from_numpy(np.stack(slabs)).cuda())
    torch.cuda.synchronize()
    assert p.bp_kernel() == "k_bp_items"
    for b in range(n_slabs):
        _check(got[b].cpu().numpy(), refs[b], contrasts[b])


@pytest.mark.parametrize("vp", ["1", "2"])
def test_tmem_pitch_pairs_match_oracle(vp, monkeypatch):
    """The TMEM kernel with two pitches per CTA (KATS_BP_PP=2: shared windows and geometry, raw sums
    finished by k_bp_ends_add_t) on T2's two pitches, one and two views per pass."""
    import torch
    for env, val in (("KATS_BP_KERNEL", "tmem"), ("KATS_BP_PP", "2"), ("KATS_BP_VP", vp)):
        monkeypatch.setenv(env, val)
    cfg, sino, ref, contrast = _case("T2")
    p = _plan(cfg)
    vol = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"])
    torch.cuda.synchronize()
    assert p.bp_kernel() == "k_bp_tmem"
    _check(vol.cpu().numpy(), ref, contrast)


@pytest.mark.parametrize("variant,vp,kernel", [(None, None, "k_backproject"), ("tmem", None, "k_bp_tmem"),
                                               ("tmem", "1", "k_bp_tmem"), ("tmem", "2", "k_bp_tmem"),
                                               ("window", None, "k_bp_window"), ("window", "winv1", "k_bp_window"),
                                               ("l1", None, "k_backproject")])
def test_every_bp_kernel_variant_matches_oracle(variant, vp, kernel, monkeypatch):
    """Each step-7 kernel on C1 against the oracle: the default (C1's 16 column tiles are under
    one CTA per SM, so the z-chunked L1 kernel), the TMEM window (forced; one or two views per
    pass), the register window and the L1 path; the plan reports that the
    expected variant is the one that ran (katsevich_bp_kernel)."""
    import torch
    winv = "1" if vp == "winv1" else None
    vp = None if vp == "winv1" else vp
    for env, val in (("KATS_BP_KERNEL", variant), ("KATS_BP_VP", vp), ("KATS_BP_WINV", winv)):
        if val is None:
            monkeypatch.delenv(env, raising=False)
        else:
            monkeypatch.setenv(env, val)
    cfg, sino, ref, contrast = _case("C1")
    p = _plan(cfg)
    vol = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"])
    torch.cuda.synchronize()
    assert p.bp_kernel() == kernel
    _check(vol.cpu().numpy(), ref, contrast)


@pytest.mark.parametrize("name,mode", [("T2", "1"), ("T3", "1"), ("T2", "2"), ("T3", "2")])
def test_pipelined_reconstruct_matches_oracle(name, mode, monkeypatch):
    """KATS_PIPELINE=1 (per pitch) / 2 (pitch pairs, the odd last pitch alone): backprojections on
    two streams behind a high-priority filter stream (forked from and joined to the caller's
    stream) give the oracle's volume too."""
    import torch
    monkeypatch.setenv("KATS_PIPELINE", mode)
    cfg, sino, ref, contrast = _case(name)
    p = _plan(cfg)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        vol = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"], stream=s)
        host = vol.cpu()          # ordered after the join on the caller's stream
    _check(host.numpy(), ref, contrast)


@pytest.mark.parametrize("kernel,ends", [("tmem", "pre"), ("tmem", "inline"), ("window", None)])
def test_bp_end_views_ahead_or_inline(kernel, ends, monkeypatch):
    """The staged step-7 kernels finish a slice with its two fractional end views either
    written ahead by k_bp_ends (window kernel always; TMEM kernel with KATS_BP_ENDS=pre) or
    sampled in the flush (TMEM kernel, inline): against the oracle on C1."""
    import torch
    if ends is None:
        monkeypatch.delenv("KATS_BP_ENDS", raising=False)
    else:
        monkeypatch.setenv("KATS_BP_ENDS", ends)
    if kernel is None:
        monkeypatch.delenv("KATS_BP_KERNEL", raising=False)
    else:
        monkeypatch.setenv("KATS_BP_KERNEL", kernel)
    cfg, sino, ref, contrast = _case("C1")
    p = _plan(cfg)
    vol = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"])
    torch.cuda.synchronize()
    _check(vol.cpu().numpy(), ref, contrast)


@pytest.mark.parametrize("k12", ["wv", "rows", "sample", "col3", "col8", "tile", "colv2", "colv4"])
@pytest.mark.parametrize("name", ["T1", "C1"])
def test_k12_variants_match_oracle(name, k12, monkeypatch):
    """Steps 1-3 (g3) by the K12 kernels: the row form (default), one thread per sample, the column walk
    with a ragged κ-line segment (3 lines per thread; the default walks 8), the shared-memory
    tile, and the column walk over 2 / 4 views per thread (ragged view tails)."""
    import torch
    from oracle import oracle
    monkeypatch.setenv("KATS_K12", k12)
    monkeypatch.delenv("KATS_HILBERT", raising=False)
    cfg, sino, _, _ = _case(name)
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    out = p.filter(torch.from_numpy(sino).cuda(), cfg["scan_v0"], v0 + 1, nv - 2, stages=("g3", "gF"))
    torch.cuda.synchronize()
    ref = oracle.filter_views(cfg, sino, cfg["scan_v0"], v0 + 1, nv - 2, stages=("g3", "gF"))
    for s in ("g3", "gF"):
        got = out[s].cpu().numpy().astype(np.float64)
        e = np.linalg.norm(got - ref[s]) / np.linalg.norm(ref[s])
        assert e <= STAGE_REL, f"{s}: rel L2 {e:.3e}"


@pytest.mark.parametrize("name,n_psi", [("T1", 2), ("T1", 14), ("T3", 22), ("T3", 87), ("C1", 65)])
def test_reconstruct_n_psi_matches_oracle(name, n_psi):
    """Non-default κ-line counts (P:l.132 leaves n_ψ free; DESIGN A6 default 2 n_w + 1):
    the degenerate two-line case, n_w + 1 and ~4 n_w + 1 (more lines than a K3 tile holds).
    Same seeded sinogram, oracle and GPU built with the same n_ψ."""
    import torch
    from oracle import oracle
    cfg, sino, _, contrast = _case(name)
    cfg = dict(cfg, n_psi=n_psi)
    ref = oracle.reconstruct(cfg, sino, cfg["scan_v0"], 0, cfg["n_pitches"])
    p = _plan(cfg)
    assert p.table_info()["n_psi"] == n_psi
    vol = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"])
    torch.cuda.synchronize()
    _check(vol.cpu().numpy(), ref, contrast)


@pytest.mark.parametrize("k4", ["rows", "tile"])
@pytest.mark.parametrize("vpb", ["1", "2", "4"])
@pytest.mark.parametrize("name", ["T1", "T3"])
def test_k4_views_per_cta_match_oracle(name, vpb, k4, monkeypatch):
    """K4 (row form, default, and the round-1 tile kernel) with 1, 2 or 4 views per CTA
    (KATS_K4_VPB; ragged view tails): gF per stage and the reconstructed volume against the oracle."""
    import torch
    from oracle import oracle
    monkeypatch.setenv("KATS_K4_VPB", vpb)
    monkeypatch.setenv("KATS_K4", k4)
    cfg, sino, ref, contrast = _case(name)
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    out = p.filter(torch.from_numpy(sino).cuda(), cfg["scan_v0"], v0 + 1, nv - 3, stages=("gF",))
    vol = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"])
    torch.cuda.synchronize()
    gref = oracle.filter_views(cfg, sino, cfg["scan_v0"], v0 + 1, nv - 3, stages=("gF",))["gF"]
    got = out["gF"].cpu().numpy().astype(np.float64)
    assert np.linalg.norm(got - gref) / np.linalg.norm(gref) <= STAGE_REL
    _check(vol.cpu().numpy(), ref, contrast)


def test_registration_case_matches_oracle():
    """The oracle's registration pin (tests/test_oracle_recon.py: off-centre ~3-voxel ball,
    λ0, z0 ≠ 0, centroid within 0.05 voxel) on the GPU: whole volume within the parity bar, and
    the GPU reconstruction's own centroid within 0.05 voxel of the true centre."""
    import torch
    from oracle import oracle
    from tests.test_oracle_recon import _centroid_error, _registration_case
    cfg, c, sino, v0 = _registration_case()
    ref = oracle.reconstruct(cfg, sino, v0, 0, 1)
    p = _plan(cfg)
    vol = p.reconstruct(torch.from_numpy(sino).cuda(), v0, 0, 1).cpu().numpy().astype(np.float64)
    _check(vol, ref, 1.0)
    assert np.abs(_centroid_error(vol, cfg, c)).max() < 0.05


@pytest.mark.parametrize("n_slabs", [4, 6, 3])
def test_batch_host_entry_point_equals_device(n_slabs):
    """katsevich_reconstruct_batch_host (host slabs in, host volumes out, groups of slabs with the
    copies overlapped) gives the device batch path's volumes; checked on T2 with 4, 6 and 3 slabs
    (groups of 4, 2 and 1)."""
    import torch
    from synth import configs, synth
    cfg = configs.get("T2")
    p = _plan(cfg)
    v0, nv = p.pitch_views(0)
    slabs = np.stack([synth.project(cfg, configs.random_ellipsoids(20 + s, 6, 180.0, -5.0, cfg["P"] + 5.0), v0, nv)
                      for s in range(n_slabs)])
    dev = p.reconstruct_batch(torch.from_numpy(slabs).cuda()).cpu().numpy()
    host = p.reconstruct_batch_host(torch.from_numpy(slabs).pin_memory()).numpy()
    assert np.linalg.norm(host - dev) / np.linalg.norm(dev) <= 1e-6
