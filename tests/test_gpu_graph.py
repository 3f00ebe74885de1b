"""CUDA graphs: the device entry points are capturable (no host synchronisation or allocation inside
the call) — a captured reconstruction and batch reconstruction replay to results bitwise equal to the
eager calls, the adjoint to fp32 rounding (its atomics sum in a run-dependent order)."""
import pytest

from tests.conftest import cuda_ok

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not cuda_ok():
        pytest.skip("no CUDA device")


def _capture(fn, s):
    import gc
    import torch
    fn()                                   # warm: workspace, kernel attributes, tensor maps
    torch.cuda.synchronize()
    # plans freed by the garbage collector release device memory (cudaFree), which a stream capture
    # does not allow: collect them before capturing (katsevich_destroy is not capture-safe)
    gc.collect()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    return g


@pytest.mark.parametrize("name", ["C1", "T3"])
def test_graph_replay_reconstruct_and_adjoint(name):
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs, synth
    cfg = configs.get(name)
    p = k.Plan(cfg, device=0)
    p.precompute()
    npit = cfg["n_pitches"]
    v0, nv = p.scan_views(0, npit)
    x = torch.from_numpy(synth.project(cfg, cfg["phantom"], v0, nv)).cuda()
    ref = p.reconstruct(x, v0, 0, npit).clone()
    s = torch.cuda.Stream()
    out = torch.empty_like(ref)
    g = _capture(lambda: p.reconstruct(x, v0, 0, npit, out=out, stream=s), s)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    y = torch.randn(ref.shape, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
    aref = p.adjoint(y, v0, nv, 0, npit).clone()
    aout = torch.empty_like(aref)
    ga = _capture(lambda: p.adjoint(y, v0, nv, 0, npit, out=aout, stream=s), s)
    aout.zero_()
    ga.replay()
    torch.cuda.synchronize()
    # (K5^T reduces CTA boxes into the sinogram adjoint with float atomics: the summation order, hence
    # the last bits, varies from run to run, eager or replayed)
    assert float((aout - aref).double().norm()) <= 1e-5 * float(aref.double().norm())


@pytest.mark.parametrize("n_slabs", [4, 16])
def test_graph_replay_batch(n_slabs):
    """4 slabs: one filter pass and one step-7 launch; 16: the two slab groups (filter of group 2
    beside the backprojection of group 1 on forked streams, joined by events) captured as graph edges."""
    import numpy as np
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs, synth
    cfg = configs.get("T2")
    p = k.Plan(cfg, device=0)
    p.precompute()
    v0, nv = p.pitch_views(0)
    slabs = np.stack([synth.project(cfg, configs.random_ellipsoids(b, 5, 180.0, 0.0, cfg["P"]), v0, nv)
                      for b in range(n_slabs)])
    x = torch.from_numpy(slabs).cuda()
    ref = p.reconstruct_batch(x).clone()
    s = torch.cuda.Stream()
    out = torch.empty_like(ref)
    g = _capture(lambda: p.reconstruct_batch(x, out=out, stream=s), s)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_workspace_shared_across_streams():
    """The plan's cached workspace used back to back from the default stream and a side stream with
    no synchronisation in between (the binding orders the calls): every result equals the
    synchronised one, forward bitwise, adjoint to rounding."""
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs
    cfg = configs.get("C1")
    p = k.Plan(cfg, device=0)
    p.precompute()
    v0, nv = p.scan_views(0, 1)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((nv, cfg["n_rows"], cfg["n_cols"]), device="cuda", generator=g)
    y = torch.randn((cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda", generator=g)
    rref = p.reconstruct(x, v0, 0, 1).clone()
    aref = p.adjoint(y, v0, nv, 0, 1).clone()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    outs = []
    for i in range(6):
        st = s if i % 2 else None
        r = p.reconstruct(x, v0, 0, 1, stream=st)
        a = p.adjoint(y, v0, nv, 0, 1, stream=st)
        if st is not None:
            r.record_stream(s)
            a.record_stream(s)
            torch.cuda.current_stream().wait_stream(s)
        outs.append((r.clone(), a.clone()))
    torch.cuda.synchronize()
    for r, a in outs:
        assert torch.equal(r, rref)
        assert float((a - aref).double().norm()) <= 1e-5 * float(aref.double().norm())


def test_no_uninitialised_reads():
    """Every entry point's result is independent of what the reused device memory held: the caching
    allocator's free blocks filled with NaN before a fresh plan's calls change nothing."""
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs
    for name in ("C1", "T3"):
        cfg = configs.get(name)
        p = k.Plan(cfg, device=0)
        p.precompute()
        npit = min(cfg["n_pitches"], 2)
        v0, nv = p.scan_views(0, npit)
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.randn((nv, cfg["n_rows"], cfg["n_cols"]), device="cuda", generator=g)
        y = torch.randn((npit * cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda", generator=g)
        r0 = p.reconstruct(x, v0, 0, npit).clone()
        a0 = p.adjoint(y, v0, nv, 0, npit).clone()
        torch.cuda.synchronize()
        q = k.Plan(cfg, device=0)
        q.precompute()
        junk = torch.full((1 << 28,), float("nan"), device="cuda")
        torch.cuda.synchronize()
        del junk
        r1 = q.reconstruct(x, v0, 0, npit)
        a1 = q.adjoint(y, v0, nv, 0, npit)
        torch.cuda.synchronize()
        assert torch.equal(r1, r0), name
        assert bool(torch.isfinite(a1).all()), name
        assert float((a1 - a0).double().norm()) <= 1e-5 * float(a0.double().norm()), name


def test_graph_replay_adjoint_batch():
    """katsevich_adjoint_batch captured and replayed: equal to the eager call to fp32 rounding."""
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs
    cfg = configs.get("T2")
    p = k.Plan(cfg, device=0)
    p.precompute()
    g = torch.Generator(device="cuda").manual_seed(11)
    y = torch.randn((4, cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda", generator=g)
    aref = p.adjoint_batch(y).clone()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    out = torch.empty_like(aref)
    ga = _capture(lambda: p.adjoint_batch(y, out=out, stream=s), s)
    out.zero_()
    with torch.cuda.stream(s):
        ga.replay()
    torch.cuda.synchronize()
    assert float((out - aref).double().norm()) <= 1e-5 * float(aref.double().norm())
