"""Small reconstructions for compute-sanitizer runs (T2 batch + T3 multi-pitch + C1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_02309_b200 as k
from synth import configs, synth
for name in ("T3", "C1"):
    cfg = configs.get(name)
    p = k.Plan(cfg, device=0); p.precompute()
    sino = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    v = p.reconstruct(torch.from_numpy(sino).cuda(), cfg["scan_v0"], 0, cfg["n_pitches"])
cfg = configs.get("T2"); p = k.Plan(cfg, device=0); p.precompute()
v0, nv = p.pitch_views(0)
slabs = np.stack([synth.project(cfg, configs.random_ellipsoids(s, 6, 180.0, -5.0, cfg["P"] + 5.0), v0, nv) for s in range(3)])
p.reconstruct_batch(torch.from_numpy(slabs).cuda())
torch.cuda.synchronize(); print("ok")
