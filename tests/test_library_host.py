"""CPU-side checks of the product library: the C ABI loads and exports every
symbol include/katsevich.h declares; host precompute (independent solvers)
reproduces the oracle's integer tables bit for bit and its fractions to 1e-9;
argument validation and error codes.  No compute kernel runs here."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2201_02309_b200 as k
from paper_2201_02309_b200 import _lib
from synth import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "katsevich.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(katsevich_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = _declared_symbols()
    assert len(names) >= 18
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), "binding must cover exactly the header"


def test_library_is_sm100a_code():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", ["T1", "T2", "T3", "C1", "C5", "TF1", "TF2", "C2F"])
def test_host_tables_bit_exact_vs_oracle(name):
    from oracle import oracle
    cfg = configs.get(name)
    if name == "C5":
        cfg = dict(cfg, nx=64, ny=64, dx=8.0, dy=8.0)       # same FOV, fewer voxels
    p = k.Plan(cfg, device=-1)
    p.precompute()
    t = p.export_tables()
    fi, ff, bi, bf = oracle.rebin_tables(cfg)
    assert np.array_equal(fi, t["fr_idx"]) and np.array_equal(bi, t["br_idx"])
    assert np.abs(ff - t["fr_frac"]).max() < 1e-9 and np.abs(bf - t["br_frac"]).max() < 1e-9
    kf, kl, wf, wl = oracle.bp_weights(cfg, 0)
    m = kl >= kf
    assert np.array_equal(np.where(m, kf, 0), t["pi_first"])
    assert np.array_equal(np.where(m, kl, -1), t["pi_last"])
    assert np.abs(wf - t["w_first"]).max() < 1e-9 and np.abs(wl - t["w_last"]).max() < 1e-9
    # periodic reuse: the oracle's pitch-k recomputation = pitch-0 table + k turns
    vt = cfg["views_per_turn"]
    kf3, kl3, wf3, _ = oracle.bp_weights(cfg, 3)
    assert np.array_equal(np.where(m, kf3 - 3 * vt, 0), t["pi_first"])
    assert np.abs(wf3 - t["w_first"]).max() < 1e-9
    fv, nv = p.pitch_views(0)
    assert (fv, nv) == oracle.pitch_slab(cfg, 0)
    assert p.pitch_views(5) == (fv + 5 * vt, nv)


@pytest.mark.slow
@pytest.mark.parametrize("name,pitch", [("C2", 1), ("C3", 0), ("C4", 7), ("C5", 0)])
def test_host_tables_bit_exact_full_configs(name, pitch):
    """North-star acceptance criterion 1 at the bench sizes (SURVEY §8(c) acceptance; PAPER.md
    l.191-231 precompute steps 1-3): the product's PI-limits (T_pi k_first/k_last), forward and
    backward rebin indices (T_fr, T_br) are bit-exact against the oracle's independent solvers on
    the FULL C2, C3, C4 grids and the real C5 256x256x10 grid; end weights and fractions to 1e-9.
    The oracle recomputes pitch `pitch` at absolute coordinates (no periodic reuse: C4 pitch 7 is
    the last pitch the bench reconstructs, C2 pitch 1 its second), so this also checks the
    periodic table against per-pitch recomputation at full size."""
    from oracle import oracle
    cfg = configs.get(name)
    p = k.Plan(cfg, device=-1)
    p.precompute()
    t = p.export_tables()
    fi, ff, bi, bf = oracle.rebin_tables(cfg)
    assert np.array_equal(fi, t["fr_idx"]) and np.array_equal(bi, t["br_idx"])
    assert np.abs(ff - t["fr_frac"]).max() < 1e-9 and np.abs(bf - t["br_frac"]).max() < 1e-9
    del fi, ff, bi, bf
    kf, kl, wf, wl = oracle.bp_weights(cfg, pitch)
    shift = pitch * cfg["views_per_turn"]
    m = kl >= kf
    assert m.sum() > 0.7 * m.size                              # the FOV covers most of the grid
    assert np.array_equal(np.where(m, kf - shift, 0), t["pi_first"])
    assert np.array_equal(np.where(m, kl - shift, -1), t["pi_last"])
    assert np.abs(np.where(m, wf, 0.0) - np.where(m, t["w_first"], 0.0)).max() < 1e-9
    assert np.abs(np.where(m, wl, 0.0) - np.where(m, t["w_last"], 0.0)).max() < 1e-9


def test_paper_layout_slab_and_td_coverage():
    """C5 (the paper's layout, zero-margin detector): no TD warning; slab [-125, 454]
    (SURVEY: BP views [-124, 453] + derivative halo)."""
    cfg = dict(configs.get("C5"), nx=128, ny=128, dx=4.0, dy=4.0)
    p = k.Plan(cfg, device=-1)
    assert p.precompute() == 0
    assert p.pitch_views(0) == (-125, 580)


def test_td_warning_when_rows_too_short():
    cfg = dict(configs.get("T1"), d_w=10.0)
    p = k.Plan(cfg, device=-1)
    with pytest.warns(UserWarning):
        rc = p.precompute()
    assert rc == _lib.KATS_WARN_TD_NOT_COVERED


@pytest.mark.parametrize("field,value", [("R", -1.0), ("D", 0.0), ("pitch", 0.0), ("views_per_turn", 2),
                                         ("n_cols", 1), ("n_rows", 1), ("d_w", 0.0), ("r_fov", 600.0),
                                         ("flags", 8), ("flags", 5), ("n_psi", 1), ("d_alpha", 0.5)])
def test_invalid_geometry_rejected(field, value):
    g = k.geometry_from_config(configs.get("T1"))
    setattr(g, field, value)
    h = ctypes.c_void_p()
    rc = _lib.lib().katsevich_plan_create(ctypes.byref(g), -1, ctypes.byref(h))
    assert rc == _lib.KATS_ERR_INVALID_GEOMETRY and not h.value


def test_null_and_state_errors():
    L = _lib.lib()
    assert L.katsevich_plan_create(None, -1, None) == _lib.KATS_ERR_NULL
    g = k.geometry_from_config(configs.get("T1"))
    h = ctypes.c_void_p()
    assert L.katsevich_plan_create(ctypes.byref(g), -1, ctypes.byref(h)) == 0
    fv, nv = ctypes.c_int64(), ctypes.c_int32()
    assert L.katsevich_pitch_views(h, 0, ctypes.byref(fv), ctypes.byref(nv)) == _lib.KATS_ERR_NOT_PRECOMPUTED
    assert L.katsevich_precompute(h, None) == 0
    # device entry points on a host-only plan
    assert L.katsevich_reconstruct(h, ctypes.c_void_p(1), 0, 10, 0, 1, ctypes.c_void_p(1), ctypes.c_void_p(1), 1 << 30,
                                   None) == _lib.KATS_ERR_NO_DEVICE
    assert L.katsevich_profile_enable(h, 1) == _lib.KATS_ERR_NO_DEVICE
    assert b"host-only" in L.katsevich_last_error_detail(h)
    assert L.katsevich_error_string(-4).startswith(b"sinogram")
    L.katsevich_destroy(h)
    L.katsevich_destroy(None)


def test_workspace_and_scan_views():
    cfg = configs.get("T3")
    p = k.Plan(cfg, device=-1)
    p.precompute()
    fv, nv = p.scan_views(1, 2)
    f1, n1 = p.pitch_views(1)
    f2, n2 = p.pitch_views(2)
    assert fv == f1 and fv + nv == f2 + n2
    b1, b3 = p.workspace_bytes(1), p.workspace_bytes(3)
    assert 0 < b1 < b3
    assert p.workspace_bytes(3, host=True) > b3


@pytest.mark.parametrize("nc", [96, 184, 368, 627, 736])
def test_hilbert_hankel_core_table(nc):
    """The tensor-core Hilbert's B operand (Hankel tap cores), read the way the
    UMMA descriptor walks it (core s = 2 (n >> 3) + (k' >> 2), row n & 7, column k' & 3), is the
    per-parity Toeplitz tap matrix K[2 (n - k) + 2 p - 1] (Eq. 12 split by output parity) with the
    K index reversed (k = NH - 1 - k'), split exactly into a TF32 hi part and an fp32 remainder."""
    rng = np.random.default_rng(nc)
    taps = rng.standard_normal(2 * nc - 1).astype(np.float32)
    NH = 32 * math.ceil(math.ceil(nc / 2) / 32)
    NS = NH // 2
    out = np.full(64 * NH, np.nan, np.float32)
    assert _lib.lib().katsevich_hilbert_hk_table(nc, taps.ctypes.data, out.ctypes.data, out.size - 1) != 0
    assert _lib.lib().katsevich_hilbert_hk_table(nc, taps.ctypes.data, out.ctypes.data, out.size) == 0
    t = out.reshape(2, 2, NS, 8, 4)
    n = np.arange(NH)[:, None]
    kp = np.arange(NH)[None, :]
    s = 2 * (n >> 3) + (kp >> 2)
    k = NH - 1 - kp
    for par in (0, 1):
        hi = t[par, 0][s, n & 7, kp & 3]
        lo = t[par, 1][s, n & 7, kp & 3]
        d = 2 * (n - k) + 2 * par - 1
        ref = np.where(np.abs(d) <= nc - 1, taps[np.clip(d + nc - 1, 0, 2 * nc - 2)], np.float32(0))
        assert np.array_equal(hi + lo, ref)
        assert not np.any(hi.view(np.uint32) & 0x1FFF)          # exactly representable in TF32


@pytest.mark.parametrize("name", ["T1", "T3", "C1"])
def test_half_sample_plan_tables_and_views(name):
    """KATS_FLAG_HALF_SAMPLE (NEXT-4, reading A25): the plan's tables are those of the half-shifted
    grid — bit-exact against the oracle's independent tables of oracle.half_sample_cfg — and a
    pitch's raw views are the shifted grid's slab [K_lo, K_hi] plus the one raw view above it."""
    from oracle import oracle
    cfg = dict(configs.get(name), flags=1)
    vc = oracle.half_sample_cfg(configs.get(name))
    p = k.Plan(cfg, device=-1)
    p.precompute()
    assert p.filtered_grid() == (cfg["n_rows"] - 1, cfg["n_cols"] - 1)
    t = p.export_tables()
    fi, ff, bi, bf = oracle.rebin_tables(vc)
    assert np.array_equal(fi, t["fr_idx"]) and np.array_equal(bi, t["br_idx"])
    assert np.abs(ff - t["fr_frac"]).max() < 1e-9 and np.abs(bf - t["br_frac"]).max() < 1e-9
    kf, kl, wf, wl = oracle.bp_weights(vc, 0)
    m = kl >= kf
    assert np.array_equal(np.where(m, kf, 0), t["pi_first"])
    assert np.array_equal(np.where(m, kl, -1), t["pi_last"])
    assert np.abs(wf - t["w_first"]).max() < 1e-9 and np.abs(wl - t["w_last"]).max() < 1e-9
    fv, nv = oracle.pitch_slab(vc, 2)                 # [K_lo - 1, K_hi + 1] of the shifted grid
    assert p.pitch_views(2) == (fv + 1, nv - 1)


def test_flat_flag_validation():
    """KATS_FLAG_FLAT (4) is accepted alone and with the Hann filter; with the half-sample derivative
    the plan is rejected (not supported)."""
    cfg = configs.get("TF1")
    for flags, ok in ((4, True), (4 | 2, True), (4 | 1, False)):
        if ok:
            k.Plan(dict(cfg, flags=flags), device=-1).precompute()
        else:
            with pytest.raises(k.KatsevichError):
                k.Plan(dict(cfg, flags=flags), device=-1)
