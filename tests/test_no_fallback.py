"""The product path has no CPU fallback: without the CUDA library the binding refuses to load, and a
host-only plan (cuda_device < 0: tables only) answers every compute entry point with
KATS_ERR_NO_DEVICE instead of computing anything (CPU-side checks; no GPU needed)."""
import ctypes

import pytest


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2201_02309_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "libkatsevich.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.lib()


def test_host_only_plan_refuses_compute():
    import paper_2201_02309_b200 as k
    from paper_2201_02309_b200._lib import lib
    from synth import configs
    p = k.Plan(configs.get("T1"), device=-1)
    p.precompute()
    L, h, z = lib(), p._h, ctypes.c_void_p(1)
    NO_DEVICE = -8
    assert L.katsevich_reconstruct(h, z, 0, 100, 0, 1, z, z, 1 << 30, None) == NO_DEVICE
    assert L.katsevich_reconstruct_batch(h, z, 1, z, z, 1 << 30, None) == NO_DEVICE
    assert L.katsevich_adjoint(h, z, 0, 1, z, 0, 100, z, 1 << 30, None) == NO_DEVICE
    assert L.katsevich_adjoint_batch(h, z, 1, z, z, 1 << 30, None) == NO_DEVICE
