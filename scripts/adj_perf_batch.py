"""Batch adjoint step timing at a batch config (C5)."""
import sys, json, torch
sys.path.insert(0, ".")
import paper_2201_02309_b200 as k
from synth import configs
cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "C5")
p = k.Plan(cfg, device=0); p.precompute()
B = cfg["batch"]
y = torch.randn((B, cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda")
for _ in range(2): p.adjoint_batch(y)
torch.cuda.synchronize()
p.profile_read(reset=True); p.profile_enable(True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); n = 5
for _ in range(n): p.adjoint_batch(y)
b.record(); torch.cuda.synchronize()
st = p.profile_read(reset=True)
print(json.dumps({"config": cfg["name"], "ms_per_batch": a.elapsed_time(b) / n,
                  "stages_ms": {s: v / n for s, v in st["ms"].items() if v}}))
