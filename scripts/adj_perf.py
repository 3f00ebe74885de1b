"""Adjoint step timing and per-stage split at a config (profiling events)."""
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
import paper_2201_02309_b200 as k
from synth import configs
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = configs.get(name); npit = cfg["n_pitches"]
p = k.Plan(cfg, device=0); p.precompute()
s0, sn = p.scan_views(0, npit)
y = torch.randn((npit * cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda")
out = torch.empty((sn, cfg["n_rows"], cfg["n_cols"]), device="cuda")
for _ in range(2): p.adjoint(y, s0, sn, 0, npit, out=out)
torch.cuda.synchronize()
p.profile_read(reset=True); p.profile_enable(True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
n = 3
for _ in range(n): p.adjoint(y, s0, sn, 0, npit, out=out)
b.record(); torch.cuda.synchronize()
st = p.profile_read(reset=True)
print(json.dumps({"config": name, "ms_per_step": a.elapsed_time(b) / n,
                  "stages_ms": {s: v / n for s, v in st["ms"].items() if v}}))
