"""NEXT-4: accuracy / cost of the κ-line count n_ψ (P:l.132 leaves it free; DESIGN A6 takes
2 n_w + 1).  GPU reconstruction of a seeded analytic phantom for several n_ψ; error against
the phantom's own voxel values inside the reconstructible region, and device time per step.

    python scripts/npsi_study.py --config C2 [--reps 5]
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
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    base = configs.get(a.config)
    nw = base["n_rows"]
    sino = torch.from_numpy(synth.project(base, base["phantom"], base["scan_v0"], base["scan_nv"])).cuda()
    truth = np.concatenate([synth.volume_truth(base, base["phantom"], j) for j in range(base["n_pitches"])])
    contrast = float(truth.max() - truth.min())
    # in-plane disc inside r_fov, axially all slices; edges of the phantom (within 1.5 voxels of a
    # density jump) are excluded so the number measures the filter, not the voxel-sampling of a step
    ny, nx = truth.shape[1:]
    yy, xx = np.mgrid[0:ny, 0:nx]
    rx = (xx - 0.5 * (nx - 1)) * base["dx"]
    ry = (yy - 0.5 * (ny - 1)) * base["dx"]
    disc = np.hypot(rx, ry) < 0.9 * 0.5 * nx * base["dx"]
    from scipy import ndimage
    jump = np.zeros_like(truth, dtype=bool)
    for ax in (1, 2):
        jump |= np.abs(np.diff(truth, axis=ax, prepend=np.take(truth, [0], axis=ax))) > 0
    smooth = ~ndimage.binary_dilation(jump, iterations=2) & disc[None]
    rows = []
    for n_psi in (nw // 2 + 1, nw + 1, 2 * nw + 1, 4 * nw + 1, 8 * nw + 1):
        cfg = dict(base, n_psi=n_psi)
        p = k.Plan(cfg, device=0)
        p.precompute()
        vol = p.reconstruct(sino, cfg["scan_v0"], 0, cfg["n_pitches"])
        for _ in range(2):
            p.reconstruct(sino, cfg["scan_v0"], 0, cfg["n_pitches"], out=vol)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            p.reconstruct(sino, cfg["scan_v0"], 0, cfg["n_pitches"], out=vol)
        e1.record()
        torch.cuda.synchronize()
        v = vol.cpu().numpy().astype(np.float64)
        d = (v - truth)[smooth]
        rows.append(dict(n_psi=n_psi, ms=e0.elapsed_time(e1) / a.reps,
                         rmse_smooth_over_contrast=float(np.sqrt(np.mean(d ** 2)) / contrast),
                         max_abs_smooth_over_contrast=float(np.abs(d).max() / contrast),
                         rel_l2_all=float(np.linalg.norm(v - truth) / np.linalg.norm(truth)),
                         smooth_voxels=int(smooth.sum())))
        print(json.dumps(dict(config=a.config, **rows[-1])), flush=True)
        del p


if __name__ == "__main__":
    main()
