"""NEXT-4: the Hann-apodised Hilbert filter (KATS_FLAG_HANN, reading A26) against the
plain band-limited kernel (reading A10), on noiseless data and on data degraded by the paper's
'Gaussian+Poisson' model (P:l.396-404: I0 = 1e5, Gaussian variance 0.5; optionally also the
α-downsampling by --stride): error against the phantom's own voxel values in the smooth interior
(RMSE), over all voxels (rel L2), the noise standard deviation (noisy minus noiseless
reconstruction) in the smooth interior, and the resolution cost as the RMSE within two voxels of a
density jump on noiseless data.  Every step runs on the GPU (projector, degradation, reconstruction).

    python scripts/apod_study.py --config C2 [--stride 1] [--seed 0]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_02309_b200 as k  # noqa: E402
from synth import configs, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--stride", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    base = configs.get(a.config)
    truth = np.concatenate([synth.volume_truth(base, base["phantom"], j) for j in range(base["n_pitches"])])
    contrast = float(truth.max() - truth.min())
    ny, nx = truth.shape[1:]
    yy, xx = np.mgrid[0:ny, 0:nx]
    disc = np.hypot((xx - 0.5 * (nx - 1)) * base["dx"], (yy - 0.5 * (ny - 1)) * base["dx"]) < 0.9 * 0.5 * nx * base["dx"]
    from scipy import ndimage
    jump = np.zeros_like(truth, dtype=bool)
    for ax in (1, 2):
        jump |= np.abs(np.diff(truth, axis=ax, prepend=np.take(truth, [0], axis=ax))) > 0
    near = ndimage.binary_dilation(jump, iterations=2)
    smooth = ~near & disc[None]
    edges = near & disc[None]
    v0, nv = base["scan_v0"], base["scan_nv"]
    rows = {}
    for flags, name in ((0, "plain"), (2, "hann")):
        cfg = dict(base, flags=flags)
        p = k.Plan(cfg, device=0)
        p.precompute()
        clean = p.project_ellipsoids(base["phantom"], v0, nv)
        noisy = p.degrade(clean, v0, alpha_stride=a.stride, I0=1e5, gauss_var=0.5, seed=a.seed)
        if a.stride > 1:                      # the sparse-view clean reference: same resampling, no noise
            clean = p.degrade(clean, v0, alpha_stride=a.stride, I0=1e5, gauss_var=0.0, seed=a.seed, mode=1)
        rc = p.reconstruct(clean, v0, 0, base["n_pitches"]).cpu().numpy().astype(np.float64)
        rn = p.reconstruct(noisy, v0, 0, base["n_pitches"]).cpu().numpy().astype(np.float64)
        rows[name] = dict(
            rmse_smooth_noiseless=float(np.sqrt(np.mean((rc - truth)[smooth] ** 2)) / contrast),
            rmse_edges_noiseless=float(np.sqrt(np.mean((rc - truth)[edges] ** 2)) / contrast),
            rmse_smooth_noisy=float(np.sqrt(np.mean((rn - truth)[smooth] ** 2)) / contrast),
            noise_std_smooth=float(np.std((rn - rc)[smooth]) / contrast),
            rel_l2_all_noiseless=float(np.linalg.norm(rc - truth) / np.linalg.norm(truth)),
            rel_l2_all_noisy=float(np.linalg.norm(rn - truth) / np.linalg.norm(truth)))
        del p
    out = dict(config=a.config, stride=a.stride, seed=a.seed, I0=1e5, gauss_var=0.5,
               smooth_voxels=int(smooth.sum()), edge_voxels=int(edges.sum()), **rows)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
