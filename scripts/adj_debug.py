import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2201_02309_b200 as k
from synth import configs
name = sys.argv[1] if len(sys.argv) > 1 else "T2"
order = sys.argv[2] if len(sys.argv) > 2 else "fa"
cfg = configs.get(name); npit = cfg["n_pitches"]; s0, sn = cfg["scan_v0"], cfg["scan_nv"]
p = k.Plan(cfg, device=0); p.precompute()
print("fwd ws", p.workspace_bytes(npit), "adj ws", p.adjoint_workspace_bytes(npit), flush=True)
rng = np.random.default_rng(8)
x = torch.from_numpy(rng.standard_normal((sn, cfg["n_rows"], cfg["n_cols"])).astype(np.float32)).cuda()
y = torch.from_numpy(rng.standard_normal((npit * cfg["nz"], cfg["ny"], cfg["nx"])).astype(np.float32)).cuda()
for op in order:
    if op == "f":
        ax = p.reconstruct(x, s0, 0, npit); torch.cuda.synchronize(); print("forward ok", p.bp_kernel(), flush=True)
    else:
        aty = p.adjoint(y, s0, sn, 0, npit); torch.cuda.synchronize(); print("adjoint ok", flush=True)
