"""Per-stage kernel times of one reconstruction (single-launch form, KATS_PIPELINE=0) for a config."""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("KATS_PIPELINE", "0")
import torch
import paper_2201_02309_b200 as k
from synth import configs, synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--pitches", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = configs.get(a.config)
p = k.Plan(cfg, device=0)
p.precompute()
npit = a.pitches or cfg.get("n_pitches", 1)
if cfg.get("batch"):
    v0, nv = p.pitch_views(0)
    x = torch.from_numpy(synth.random_array((cfg["batch"], nv, cfg["n_rows"], cfg["n_cols"]), 1)).cuda()
    run = lambda: p.reconstruct_batch(x)
else:
    v0, nv = p.scan_views(0, npit)
    x = torch.from_numpy(synth.random_array((nv, cfg["n_rows"], cfg["n_cols"]), 1)).cuda()
    run = lambda: p.reconstruct(x, v0, 0, npit)
run(); torch.cuda.synchronize()
p.profile_read(reset=True); p.profile_enable(True)
for _ in range(a.reps):
    run()
torch.cuda.synchronize()
st = p.profile_read(reset=True)
out = {s: {"ms_per_rep": st["ms"][s] / a.reps, "launches_per_rep": st["launches"][s] // a.reps} for s in st["ms"] if st["launches"][s]}
print(json.dumps({"config": a.config, "pitches": npit, "bp_kernel": p.bp_kernel(), "stages": out}))
