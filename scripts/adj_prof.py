import sys, torch
sys.path.insert(0, ".")
import paper_2201_02309_b200 as k
from synth import configs
cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "C4")
p = k.Plan(cfg, device=0); p.precompute()
s0, sn = p.scan_views(0, 1)
y = torch.randn((cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda")
for _ in range(2): p.adjoint(y, s0, sn, 0, 1)
torch.cuda.synchronize(); print("ok")
