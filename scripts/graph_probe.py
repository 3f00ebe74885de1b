import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_2201_02309_b200 as k
from synth import configs, synth
for name in ["C1", "T3"]:
    cfg = configs.get(name)
    p = k.Plan(cfg, device=0); p.precompute()
    npit = cfg["n_pitches"]
    v0, nv = p.scan_views(0, npit)
    x = torch.from_numpy(synth.project(cfg, cfg["phantom"], v0, nv)).cuda()
    out = torch.empty((npit * cfg["nz"], cfg["ny"], cfg["nx"]), device="cuda")
    ref = p.reconstruct(x, v0, 0, npit).clone()
    s = torch.cuda.Stream()
    ws_bytes = p.workspace_bytes(npit)
    with torch.cuda.stream(s):
        for _ in range(3): p.reconstruct(x, v0, 0, npit, out=out, stream=s)   # warm (workspace, attributes)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            p.reconstruct(x, v0, 0, npit, out=out, stream=s)
    except Exception as e:
        print(name, "capture failed:", repr(e)[:300]); continue
    out.zero_(); g.replay(); torch.cuda.synchronize()
    print(name, "graph == eager:", torch.equal(out, ref))
    for mode in ("eager", "graph"):
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(200):
            if mode == "graph": g.replay()
            else: p.reconstruct(x, v0, 0, npit, out=out, stream=torch.cuda.current_stream())
        torch.cuda.synchronize(); print(name, mode, "ms/step", (time.perf_counter() - t) / 200 * 1e3)
