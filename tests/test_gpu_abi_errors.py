"""The C ABI's documented error codes on a device plan (include/katsevich.h): NULL pointers,
counts out of range, a workspace smaller than katsevich_workspace_bytes, a sinogram that does not
cover the requested pitches, calls before katsevich_precompute — each returns its code, launches
nothing and leaves the output untouched; a valid call right after succeeds (the plan is reusable)."""
import ctypes

import pytest

from tests.conftest import cuda_ok

pytestmark = pytest.mark.gpu

OK, NULL, NOT_PRE, COVER, WS, ARG = 0, -1, -3, -4, -6, -9


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not cuda_ok():
        pytest.skip("no CUDA device")


def _v(t):
    return ctypes.c_void_p(t.data_ptr())


def test_entry_point_error_codes():
    import torch
    import paper_2201_02309_b200 as k
    from paper_2201_02309_b200._lib import lib
    from synth import configs
    cfg = configs.get("T1")
    L = lib()
    p = k.Plan(cfg, device=0)
    h = p._h
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    v0, nv = 0, 10
    sino = torch.zeros((nv, cfg["n_rows"], cfg["n_cols"]), device="cuda")
    vol = torch.full((cfg["nz"], cfg["ny"], cfg["nx"]), 7.0, device="cuda")
    ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    # before precompute
    assert L.katsevich_reconstruct(h, _v(sino), v0, nv, 0, 1, _v(vol), _v(ws), ws.numel(), s) == NOT_PRE
    p.precompute()
    f0, n0 = p.scan_views(0, 1)
    sino = torch.zeros((n0, cfg["n_rows"], cfg["n_cols"]), device="cuda")
    need = p.workspace_bytes(1)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    rec = L.katsevich_reconstruct
    assert rec(h, None, f0, n0, 0, 1, _v(vol), _v(ws), need, s) == NULL
    assert rec(h, _v(sino), f0, n0, 0, 1, None, _v(ws), need, s) == NULL
    assert rec(h, _v(sino), f0, n0, 0, 0, _v(vol), _v(ws), need, s) == ARG
    assert rec(h, _v(sino), f0, n0, 0, 1, _v(vol), _v(ws), need - 1, s) == WS
    assert rec(h, _v(sino), f0 + 1, n0 - 1, 0, 1, _v(vol), _v(ws), need, s) == COVER
    assert rec(h, _v(sino), f0, n0, 1, 1, _v(vol), _v(ws), need, s) == COVER
    torch.cuda.synchronize()
    assert bool((vol == 7.0).all())                      # nothing ran
    # batch and adjoint entry points
    fv, nvs = p.pitch_views(0)
    slabs = torch.zeros((2, nvs, cfg["n_rows"], cfg["n_cols"]), device="cuda")
    vols = torch.full((2, cfg["nz"], cfg["ny"], cfg["nx"]), 7.0, device="cuda")
    nb = p.workspace_bytes(2)
    wsb = torch.empty(nb, dtype=torch.uint8, device="cuda")
    assert L.katsevich_reconstruct_batch(h, _v(slabs), 0, _v(vols), _v(wsb), nb, s) == ARG
    assert L.katsevich_reconstruct_batch(h, _v(slabs), 2, _v(vols), _v(wsb), nb - 1, s) == WS
    na = p.adjoint_workspace_bytes(1)
    wsa = torch.empty(na, dtype=torch.uint8, device="cuda")
    out = torch.full_like(sino, 7.0)
    adj = L.katsevich_adjoint
    assert adj(h, _v(vol), 0, 1, _v(out), f0, 2, _v(wsa), na, s) == ARG
    assert adj(h, _v(vol), 0, 1, _v(out), f0 + 1, n0 - 1, _v(wsa), na, s) == COVER
    assert adj(h, _v(vol), 0, 1, _v(out), f0, n0, _v(wsa), na - 1, s) == WS
    torch.cuda.synchronize()
    assert bool((vols == 7.0).all()) and bool((out == 7.0).all())
    # the plan still works
    assert rec(h, _v(sino), f0, n0, 0, 1, _v(vol), _v(ws), need, s) == OK
    assert adj(h, _v(vol), 0, 1, _v(out), f0, n0, _v(wsa), na, s) == OK
    torch.cuda.synchronize()
    assert bool((vol == 0).all()) and bool((out == 0).all())      # zero sinogram -> zero volume; zero volume
