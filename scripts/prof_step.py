"""Small driver for ncu captures: one reconstruction of `--pitches` pitches of a
config with seeded random data (kernel control flow does not depend on values)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2201_02309_b200 as k
from synth import configs, synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--pitches", type=int, default=1)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg = configs.get(a.config)
p = k.Plan(cfg, device=0)
p.precompute()
if cfg.get("batch"):
    v0, nv = p.pitch_views(0)
    x = torch.from_numpy(synth.random_array((cfg["batch"], nv, cfg["n_rows"], cfg["n_cols"]), 1)).cuda()
    for _ in range(a.reps):
        p.reconstruct_batch(x)
else:
    v0, nv = p.scan_views(0, a.pitches)
    x = torch.from_numpy(synth.random_array((nv, cfg["n_rows"], cfg["n_cols"]), 1)).cuda()
    for _ in range(a.reps):
        p.reconstruct(x, v0, 0, a.pitches)
torch.cuda.synchronize()
print("ok", p.profile_read()["total_launches"])
