"""Timeline of one C4 host-buffer reconstruction (katsevich_reconstruct_host): per-launch stage
intervals from the library's in-run CUDA events (KATS_PROFILE_DUMP=1 prints them), wall time around
the call.  Usage: KATS_PROFILE_DUMP=1 python scripts/host_timeline.py [C4]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2201_02309_b200 as k
from synth import configs, synth
cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "C4")
p = k.Plan(cfg, device=0); p.precompute()
npit = cfg["n_pitches"]
v0, nv = p.scan_views(0, npit)
x = torch.from_numpy(synth.random_array((nv, cfg["n_rows"], cfg["n_cols"]), 1)).pin_memory()
out = torch.empty((npit * cfg["nz"], cfg["ny"], cfg["nx"]), dtype=torch.float32).pin_memory()
for _ in range(3):
    p.reconstruct_host(x, v0, 0, npit, out_host=out)
torch.cuda.synchronize()
p.profile_read(reset=True); p.profile_enable(True)
t0 = time.perf_counter()
p.reconstruct_host(x, v0, 0, npit, out_host=out)
t1 = time.perf_counter()
st = p.profile_read(reset=True)
print("wall ms", (t1 - t0) * 1e3, "busy", st["busy_ms"], file=sys.stderr)
