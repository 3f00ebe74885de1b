"""Round-2 repro: an eager adjoint on the default stream followed at once by one on a side stream
(no synchronisation) raced on the plan's cached workspace before the binding ordered them
(Plan._ws_use); now every line prints ~1e-7."""
import sys, gc, torch, numpy as np
sys.path.insert(0, '.')
import paper_2201_02309_b200 as k
from synth import configs, synth
rel = lambda a, b: float((a - b).double().norm() / b.double().norm())

def seq(name, check_oracle=False):
    cfg = configs.get(name)
    p = k.Plan(cfg, device=0); p.precompute()
    npit = cfg["n_pitches"]
    v0, nv = p.scan_views(0, npit)
    x = torch.from_numpy(synth.project(cfg, cfg["phantom"], v0, nv)).cuda()
    ref = p.reconstruct(x, v0, 0, npit).clone()
    s = torch.cuda.Stream()
    out = torch.empty_like(ref)
    fn = lambda: p.reconstruct(x, v0, 0, npit, out=out, stream=s)
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    out.zero_(); g.replay(); torch.cuda.synchronize()
    print(name, "fwd graph", rel(out, ref))
    y = torch.randn(ref.shape, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
    aref = p.adjoint(y, v0, nv, 0, npit).clone()
    a2 = p.adjoint(y, v0, nv, 0, npit).clone()
    if check_oracle:
        from oracle import oracle
        oref = oracle.adjoint(cfg, y.cpu().numpy().astype(np.float64), 0, npit, v0, nv)
        print(name, "eager vs oracle", float(np.linalg.norm(aref.cpu().numpy() - oref) / np.linalg.norm(oref)))
    aout = torch.empty_like(aref)
    fa = lambda: p.adjoint(y, v0, nv, 0, npit, out=aout, stream=s)
    fa(); torch.cuda.synchronize()
    print(name, "eager-eager", rel(a2, aref), "warm on s", rel(aout, aref))
    ga = torch.cuda.CUDAGraph()
    with torch.cuda.graph(ga, stream=s):
        fa()
    aout.zero_(); ga.replay(); torch.cuda.synchronize()
    print(name, "adj graph", rel(aout, aref))
    return p, g, ga

keep = seq("C1")
if len(sys.argv) > 1 and sys.argv[1] == "drop":
    del keep; gc.collect(); torch.cuda.synchronize()
keep2 = seq("T3", check_oracle=True)
