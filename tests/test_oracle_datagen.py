"""Oracle of the data-generation path (NEXT-3)
pinned against things other than itself: Philox4x32-10 known-answer vectors
(Random123), Poisson/normal moments, the noiseless identity and the delta-method
variance of the noise model, exactness properties of the α resampling, chord
closed forms, the independent input-generator projector (synth/) and dense
quadrature, and an analytic ball for the voxel projector."""
import numpy as np
import pytest

from oracle import oracle
from synth import configs, synth


def test_philox_known_answers():
    # Random123 kat_vectors, philox4x32 R=10
    assert oracle.philox([0, 0, 0, 0], [0, 0]) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert oracle.philox([0xffffffff] * 4, [0xffffffff] * 2) == [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert oracle.philox([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0]) == \
        [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


def _flat_cfg(n_views=1):
    cfg = dict(configs.get("T1"))
    return cfg


def test_noise_noiseless_mode_is_identity():
    cfg = configs.get("T1")
    rng = np.random.default_rng(0)
    g = rng.uniform(0.0, 300.0, (3, cfg["n_rows"], cfg["n_cols"]))
    out, _, M = oracle.add_noise(cfg, g, 5, mode=1)
    assert M == g.max()
    assert np.abs(out - g).max() <= 1e-9 * M


def test_noise_statistics_match_the_delta_method():
    """Poisson draws have mean = variance = t; the noisy-minus-clean spread matches
    M^2 (t + var) / t^2 to first order (SPEC add_noise)."""
    cfg = configs.get("T1")
    nv = 700                                                   # 700 x 13 x 45 = 409,500 samples
    g = np.full((nv, cfg["n_rows"], cfg["n_cols"]), 50.0)
    g[0, 0, 0] = 100.0                                         # M = 100 -> t = I0 e^-0.5
    out, counts, M = oracle.add_noise(cfg, g, 0, I0=1e5, var=0.5, seed=7)
    t = 1e5 * np.exp(-0.5)
    c = counts.ravel()[1:].astype(np.float64)
    assert abs(c.mean() - t) < 4 * np.sqrt(t / c.size)
    assert abs(c.var() / t - 1.0) < 0.02
    d = (out - g).ravel()[1:]
    pred = M * M * (t + 0.5) / (t * t)
    assert abs(d.var() / pred - 1.0) < 0.1
    # different seeds differ, the same seed reproduces bit for bit
    out2, counts2, _ = oracle.add_noise(cfg, g, 0, I0=1e5, var=0.5, seed=7)
    assert np.array_equal(counts, counts2) and np.array_equal(out, out2)
    _, counts3, _ = oracle.add_noise(cfg, g, 0, I0=1e5, var=0.5, seed=8)
    assert not np.array_equal(counts, counts3)


def test_noise_stream_is_independent_of_chunking():
    cfg = configs.get("T1")
    rng = np.random.default_rng(1)
    g = rng.uniform(10.0, 200.0, (6, cfg["n_rows"], cfg["n_cols"]))
    g[0, 0, 0] = g[3, 0, 0] = 250.0                           # same M for both halves
    _, c_all, _ = oracle.add_noise(cfg, g, 40, seed=3)
    _, c_a, _ = oracle.add_noise(cfg, g[:3], 40, seed=3)
    _, c_b, _ = oracle.add_noise(cfg, g[3:], 43, seed=3)
    assert np.array_equal(c_all, np.concatenate([c_a, c_b]))


def test_resample_alpha_properties():
    cfg = configs.get("T3")                                    # 131 columns
    nc = cfg["n_cols"]
    rng = np.random.default_rng(2)
    g = rng.standard_normal((2, cfg["n_rows"], nc))
    assert np.array_equal(oracle.resample_alpha(cfg, g, 1), g)
    up = oracle.resample_alpha(cfg, g, 4)
    assert np.array_equal(up[..., ::4], g[..., ::4])          # kept columns bit for bit
    assert np.allclose(oracle.resample_alpha(cfg, up, 4), up, rtol=0, atol=1e-12)   # idempotent
    # alpha-affine data is reproduced exactly up to the last kept column; held beyond it
    l = np.arange(nc, dtype=np.float64)
    aff = np.broadcast_to(3.0 - 0.25 * l, g.shape).copy()
    r = oracle.resample_alpha(cfg, aff, 4)
    last = 4 * ((nc - 1) // 4)
    assert np.allclose(r[..., :last + 1], aff[..., :last + 1], rtol=0, atol=1e-12)
    assert np.all(r[..., last:] == aff[..., last:last + 1])
    # paper: 627 channels, stride 4 -> 157 kept
    assert len(range(0, 627, 4)) == 157


def test_projector_central_sphere_chord():
    cfg = configs.get("T1")
    R = cfg["R"]
    # a sphere centred on the central ray of view 0 (alpha = 0, w = 0): chord = diameter
    nc, nr = cfg["n_cols"], cfg["n_rows"]
    # central ray exists only for odd counts with alpha_offset 0: use a custom detector
    c = dict(cfg, n_cols=1, n_rows=1, alpha_offset=0.0, lambda0=0.0, z0=0.0)
    a, rho = 37.5, 0.8
    out = oracle.project_ellipsoids(c, [[0.0, 0.0, 0.0, a, a, a, 0.3, rho]], 0, 1)
    assert abs(out[0, 0, 0] - 2 * a * rho) < 1e-9 * a


@pytest.mark.parametrize("name", ["T2", "T3"])
def test_projector_matches_input_generator_and_quadrature(name):
    cfg = configs.get(name)
    ph = cfg["phantom"]
    v0 = cfg["scan_v0"] + 3
    ref = synth.project(cfg, ph, v0, 2).astype(np.float64)
    got = oracle.project_ellipsoids(cfg, ph, v0, 2)
    assert np.abs(got - ref).max() <= 2e-6 * max(1.0, np.abs(ref).max())       # synth stores float32
    # one ray against dense quadrature of the phantom density along it
    lam = v0 * 2 * np.pi / cfg["views_per_turn"]
    l, m = cfg["n_cols"] // 3, cfg["n_rows"] // 2
    alpha = (l - 0.5 * (cfg["n_cols"] - 1) + cfg["alpha_offset"]) * cfg["d_alpha"]
    w = (m - 0.5 * (cfg["n_rows"] - 1)) * cfg["d_w"]
    q = synth.ray_quadrature(cfg, ph, lam, alpha, w, 0.0, 2.5 * cfg["R"], 0.01)
    assert abs(got[0, m, l] - q) < 1e-3 * max(1.0, abs(q))


def test_volume_projector_ball_against_analytic():
    """A voxelised ball (4^3 supersampled occupancy, 2 mm voxels) projected by ray
    marching vs the exact chords: relative RMSE < 0.5 % (SPEC project_numeric)."""
    cfg = dict(configs.get("T2"), nx=128, ny=128, dx=2.0, dy=2.0)
    nx, dx = cfg["nx"], cfg["dx"]
    zv0, dzv, nzv = -80.0, 2.0, 81
    rb = 60.0
    ball = [0.0, 0.0, 0.0, rb, rb, rb, 0.0, 1.0]
    ss = (np.arange(4) + 0.5) / 4 - 0.5
    xs = (np.arange(nx) - nx / 2) * dx
    zs = zv0 + np.arange(nzv) * dzv
    X, Y, Z = np.meshgrid(xs, xs, zs, indexing="ij")
    occ = np.zeros_like(X)
    for a in ss:
        for b in ss:
            for c in ss:
                occ += ((X + a * dx) ** 2 + (Y + b * dx) ** 2 + (Z + c * dzv) ** 2 <= rb * rb)
    vol = np.ascontiguousarray((occ / 64.0).transpose(2, 1, 0)).astype(np.float32)   # [z][y][x]
    # z0 = 0: the source is at z = 0 at view 0, so views near 0 cross the ball's centre plane
    got, ntr = oracle.project_volume(cfg, vol, zv0, dzv, -2, 4)
    ref = oracle.project_ellipsoids(cfg, [ball], -2, 4)
    mask = ref > 0.05 * ref.max()
    assert mask.sum() > 100
    rmse = np.sqrt(np.mean((got[mask] - ref[mask]) ** 2)) / np.sqrt(np.mean(ref[mask] ** 2))
    assert rmse < 5e-3, rmse
    # linearity and zero
    got2, _ = oracle.project_volume(cfg, 2 * vol, zv0, dzv, -2, 1)
    assert np.allclose(got2, 2 * got[:1], rtol=1e-12, atol=0)
    z, _ = oracle.project_volume(cfg, np.zeros_like(vol), zv0, dzv, 0, 1)
    assert np.all(z == 0.0)
