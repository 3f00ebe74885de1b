"""Workload configurations C1..C5 (BASELINE.json `configs`, SURVEY.md §8 concrete
configs table) plus small ragged test configurations.

Pure data: geometry numbers, grids, phantoms and generous scan view ranges.  No
Katsevich arithmetic lives here (the reconstructible slab of a pitch is computed
independently by the oracle and by the product).

Geometry conventions (§II / §III-C2, SURVEY.md §8(c) "Grids"):
  R helix radius, D source-to-detector distance, P table feed per turn [mm],
  "normalised pitch" = P / (n_rows d_w R / D)  (collimation at isocentre),
  α_l = (l-(n_cols-1)/2+alpha_offset) d_alpha, w_m = (m-(n_rows-1)/2) d_w,
  x_i = (i - nx/2) dx, z_j = j P / nz (+ k P for pitch k), view v <-> λ = 2π v / views_per_turn.
"""
from __future__ import annotations

import math

import numpy as np

# --- AAPM / Siemens-like physical scanner (K1) ---------
R_AAPM, D_AAPM = 595.0, 1085.6
DW_AAPM = 1.0947            # mm at the detector (0.6 mm at isocentre)
DALPHA_736 = 1.1844e-3      # rad, 736 columns -> half fan 24.97 deg


def _pitch_mm(norm_pitch, n_rows, d_w, R, D):
    return norm_pitch * n_rows * d_w * R / D


# --- phantoms (rows: cx, cy, cz, a, b, c, phi, rho) --------------------------
# 3-D Shepp-Logan, Kak & Slaney geometry with Toft's modified densities
# (unit-cube coordinates; scaled per config).
_SL3D = [
    # x0     y0      z0     a       b      c     phi(deg) rho
    (0.0,   0.0,    0.0,   0.69,   0.92,  0.90,    0.0,  1.0),
    (0.0,   0.0,    0.0,   0.6624, 0.874, 0.88,    0.0, -0.8),
    (-0.22, 0.0,   -0.25,  0.41,   0.16,  0.21,  108.0, -0.2),
    (0.22,  0.0,   -0.25,  0.31,   0.11,  0.22,   72.0, -0.2),
    (0.0,   0.35,  -0.25,  0.21,   0.25,  0.50,    0.0,  0.1),
    (0.0,   0.1,   -0.25,  0.046,  0.046, 0.046,   0.0,  0.1),
    (-0.08, -0.65, -0.25,  0.046,  0.023, 0.02,    0.0,  0.1),
    (0.06,  -0.65, -0.25,  0.046,  0.023, 0.02,   90.0,  0.1),
    (0.06,  -0.105, 0.625, 0.056,  0.04,  0.10,   90.0,  0.1),
    (0.0,   0.1,    0.625, 0.056,  0.056, 0.10,    0.0,  0.1),
]


def shepp_logan(scale_xy: float, scale_z: float, zc: float) -> np.ndarray:
    rows = []
    for x0, y0, z0, a, b, c, phi, rho in _SL3D:
        rows.append((x0 * scale_xy, y0 * scale_xy, zc + z0 * scale_z,
                     a * scale_xy, b * scale_xy, c * scale_z, math.radians(phi), rho))
    return np.array(rows, dtype=np.float64)


def ball_phantom(zc: float, inner: bool = True) -> np.ndarray:
    rows = [(0.0, 0.0, zc, 120.0, 120.0, 120.0, 0.0, 1.0)]
    if inner:
        rows += [(-40.0, 20.0, zc - 10.0, 30.0, 20.0, 40.0, 0.3, 0.5),
                 (45.0, -10.0, zc + 20.0, 25.0, 35.0, 30.0, -0.5, -0.3),
                 (0.0, -60.0, zc - 40.0, 15.0, 15.0, 50.0, 0.0, 0.2)]
    return np.array(rows, dtype=np.float64)


def random_ellipsoids(seed: int, n: int, r_max: float, z_lo: float, z_hi: float) -> np.ndarray:
    """Seeded random-ellipsoid phantom (C5): centres within r <= r_max."""
    rng = np.random.default_rng(seed)
    rows = [(0.0, 0.0, 0.5 * (z_lo + z_hi), r_max * 1.05, r_max * 0.9, 400.0, 0.0, 0.2)]  # body
    for _ in range(n - 1):
        r = r_max * math.sqrt(rng.uniform(0.0, 1.0)) * 0.85
        t = rng.uniform(0.0, 2 * math.pi)
        rows.append((r * math.cos(t), r * math.sin(t), rng.uniform(z_lo, z_hi),
                     rng.uniform(8.0, 50.0), rng.uniform(8.0, 50.0), rng.uniform(5.0, 30.0),
                     rng.uniform(0.0, math.pi), rng.uniform(-0.3, 0.8)))
    return np.array(rows, dtype=np.float64)


def _scan_range(views_per_turn: int, n_pitches: int, z0_turns: float = 0.0, first_pitch: int = 0):
    # generous: PI-windows of z in [kP,(k+1)P) stay within [-0.4, n+0.4] turns
    # of the helix parameter (shifted by -z0/P turns: λ = 2π(z - z0)/P on the axis)
    lo = int(math.floor((first_pitch - z0_turns - 0.4) * views_per_turn))
    hi = int(math.ceil((first_pitch + n_pitches - z0_turns + 0.4) * views_per_turn))
    return lo, hi - lo + 1


def _mk(name, *, R, D, P, n_rows, d_w, n_cols, d_alpha, views_per_turn, nx, ny, dx, nz,
        n_pitches, phantom, alpha_offset=0.25, lambda0=0.0, z0=0.0, n_psi=0, r_fov=0.0,
        batch=0, desc="", flags=0):
    v0, nv = _scan_range(views_per_turn, n_pitches, z0 / P)
    d = dict(name=name, desc=desc, R=R, D=D, P=P, lambda0=lambda0, z0=z0, r_fov=r_fov,
             n_rows=n_rows, d_w=d_w, n_cols=n_cols, d_alpha=d_alpha, alpha_offset=alpha_offset,
             views_per_turn=views_per_turn, nx=nx, ny=ny, dx=dx, dy=dx, nz=nz, n_psi=n_psi,
             n_pitches=n_pitches, phantom=phantom, scan_v0=v0, scan_nv=nv, batch=batch)
    if flags:
        d["flags"] = flags
    return d


FLAT = 4        # KATS_FLAG_FLAT: flat detector, d_alpha = column pitch [mm] on the plane at distance D


def get(name: str) -> dict:
    n = name.upper()
    if n == "C1":
        # 64^3 ball + ellipsoids, 16 x 96 curved detector, 128 views/turn, 2 turns, pitch 1.0
        P = _pitch_mm(1.0, 16, 36.491, R_AAPM, D_AAPM)           # 320.0 mm
        return _mk("C1", R=R_AAPM, D=D_AAPM, P=P, n_rows=16, d_w=36.491, n_cols=96,
                   d_alpha=9.0805e-3, views_per_turn=128, nx=64, ny=64, dx=5.0, nz=64,
                   n_pitches=1, phantom=ball_phantom(0.5 * P),
                   desc="64^3 ball+ellipsoids, 16x96, 128 v/turn, pitch 1.0")
    if n == "C2":
        P = _pitch_mm(1.5, 32, DW_AAPM, R_AAPM, D_AAPM)          # 28.8 mm
        return _mk("C2", R=R_AAPM, D=D_AAPM, P=P, n_rows=32, d_w=DW_AAPM, n_cols=368,
                   d_alpha=2 * DALPHA_736, views_per_turn=576, nx=256, ny=256, dx=1.0, nz=32,
                   n_pitches=2, phantom=shepp_logan(120.0, 120.0, P),
                   desc="256x256x64 Shepp-Logan, 32x368 (sparse 2x), 576 v/turn, pitch 1.5")
    if n == "C3":
        P = _pitch_mm(1.0, 64, DW_AAPM, R_AAPM, D_AAPM)          # 38.4 mm
        return _mk("C3", R=R_AAPM, D=D_AAPM, P=P, n_rows=64, d_w=DW_AAPM, n_cols=736,
                   d_alpha=DALPHA_736, views_per_turn=1152, nx=512, ny=512, dx=0.68, nz=64,
                   n_pitches=1, phantom=shepp_logan(180.0, 180.0, 0.5 * P),
                   desc="512x512 x one pitch, 64x736, 1152 v/turn, pitch 1.0")
    if n == "C4":
        P = _pitch_mm(1.5, 64, DW_AAPM, R_AAPM, D_AAPM)          # 57.6 mm
        return _mk("C4", R=R_AAPM, D=D_AAPM, P=P, n_rows=64, d_w=DW_AAPM, n_cols=184,
                   d_alpha=4 * DALPHA_736, views_per_turn=1152, nx=512, ny=512, dx=0.5, nz=64,
                   n_pitches=8, phantom=shepp_logan(120.0, 230.0, 230.0),
                   desc="512^3 long scan (8 pitches x 64), 64x184 (sparse 4x), 1152 v/turn, pitch 1.5")
    if n == "C5":
        # the paper's own layout (Table I) read with R=1085.6, D=595
        P = 7.0 * math.pi
        return _mk("C5", R=1085.6, D=595.0, P=P, n_rows=16, d_w=0.5176, n_cols=627,
                   d_alpha=math.pi / 2880.0, views_per_turn=360, nx=256, ny=256, dx=2.0, nz=10,
                   n_pitches=1, phantom=None, batch=16,
                   desc="batch of 16 one-pitch 256^2 x 10 slabs, 16x627, 360 v/turn, p=7pi")
    # ---- small ragged test configurations (not bench lines) ----
    if n == "T1":
        # tiny, ragged: 37x29 grid (not tile multiples), 7 slices, 13 x 45 detector
        R, D = R_AAPM, D_AAPM
        P = _pitch_mm(1.0, 13, 40.0, R, D)
        return _mk("T1", R=R, D=D, P=P, n_rows=13, d_w=40.0, n_cols=45, d_alpha=0.021,
                   views_per_turn=60, nx=37, ny=29, dx=9.0, nz=7, n_pitches=1,
                   phantom=ball_phantom(0.5 * P), lambda0=0.7, z0=3.1,
                   desc="tiny ragged test")
    if n == "T2":
        # small paper-layout-like (R, D swapped as the paper's numbers need), 2 pitches
        P = 7.0 * math.pi
        return _mk("T2", R=1085.6, D=595.0, P=P, n_rows=16, d_w=0.5176, n_cols=157,
                   d_alpha=4 * math.pi / 2880.0, views_per_turn=90, nx=48, ny=40, dx=10.0, nz=10,
                   n_pitches=2, phantom=shepp_logan(300.0, 300.0, P),
                   desc="paper-like geometry, sparse 4x columns, small grid, 2 pitches")
    if n == "T3":
        # wide-fan ragged config with odd numbers everywhere (stress edges)
        R, D = R_AAPM, D_AAPM
        P = _pitch_mm(1.2, 21, 3.3, R, D)
        return _mk("T3", R=R, D=D, P=P, n_rows=21, d_w=3.3, n_cols=131, d_alpha=6.6e-3,
                   views_per_turn=200, nx=61, ny=53, dx=4.1, nz=19, n_pitches=3,
                   phantom=shepp_logan(110.0, 80.0, 1.5 * P), lambda0=-1.3, z0=-7.0,
                   desc="ragged odd-sized config, 3 pitches")
    # ---- flat-detector variant (NEXT-4, reading A27): columns u_l = (l - (n-1)/2 + off) d_u ----
    if n == "TF1":
        # T3's scan and volume with a flat detector (131 x 7.2 mm columns cover u* = D tan α_m = 316 mm)
        R, D = R_AAPM, D_AAPM
        P = _pitch_mm(1.2, 21, 3.3, R, D)
        return _mk("TF1", R=R, D=D, P=P, n_rows=21, d_w=3.3, n_cols=131, d_alpha=7.2,
                   views_per_turn=200, nx=61, ny=53, dx=4.1, nz=19, n_pitches=3,
                   phantom=shepp_logan(110.0, 80.0, 1.5 * P), lambda0=-1.3, z0=-7.0, flags=FLAT,
                   desc="flat-detector ragged config, 3 pitches")
    if n == "TF2":
        # T2's paper-like helix and slab with a flat detector: 157 x 2.6 mm columns (u* up to 178 mm) and 18
        # rows (the flat Tam-Danielsson window is ~9 % taller at the edge columns than the curved one)
        P = 7.0 * math.pi
        return _mk("TF2", R=1085.6, D=595.0, P=P, n_rows=18, d_w=0.5176, n_cols=157,
                   d_alpha=2.6, views_per_turn=90, nx=48, ny=40, dx=10.0, nz=10,
                   n_pitches=2, phantom=shepp_logan(300.0, 300.0, P), flags=FLAT,
                   desc="paper-like geometry, flat detector, small grid, 2 pitches")
    if n == "C2F":
        # C2's volume and scan with a flat 36 x 368 detector (2 mm columns: u* up to 346 mm; 36 rows for
        # the flat Tam-Danielsson window, which widens by 1 + u^2/D^2 towards the edges)
        P = _pitch_mm(1.5, 32, DW_AAPM, R_AAPM, D_AAPM)          # 28.8 mm, as C2
        return _mk("C2F", R=R_AAPM, D=D_AAPM, P=P, n_rows=36, d_w=DW_AAPM, n_cols=368,
                   d_alpha=2.0, views_per_turn=576, nx=256, ny=256, dx=1.0, nz=32,
                   n_pitches=2, phantom=shepp_logan(120.0, 120.0, P), flags=FLAT,
                   desc="C2 volume, flat 36x368 detector (2 mm columns), 576 v/turn")
    raise KeyError(name)


BENCH_CONFIGS = ("C1", "C2", "C3", "C4", "C5")
TEST_CONFIGS = ("T1", "T2", "T3")


def c5_phantoms(batch: int = 16):
    cfg = get("C5")
    return [random_ellipsoids(s, 10, 200.0, -10.0, cfg["P"] + 10.0) for s in range(batch)]
