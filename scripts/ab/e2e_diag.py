"""Diagnose the host entry point: copy bandwidths, device-only step, host-path step."""
import time, torch, numpy as np, sys
sys.path.insert(0, ".")
import paper_2201_02309_b200 as k
from synth import configs

cfg = configs.get("C4")
p = k.Plan(cfg, device=0); p.precompute()
v0, nv = p.scan_views(0, cfg["n_pitches"])
rng = np.random.default_rng(0)
host = torch.from_numpy(rng.standard_normal((nv, cfg["n_rows"], cfg["n_cols"]), dtype=np.float32)).pin_memory()
dev = host.cuda()
out = torch.empty((cfg["n_pitches"] * cfg["nz"], cfg["ny"], cfg["nx"]), dtype=torch.float32).pin_memory()
dvol = torch.empty(out.shape, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()

def t_events(fn, n=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(n): fn()
    b.record(s); torch.cuda.synchronize()
    return a.elapsed_time(b) / n

with torch.cuda.stream(s):
    h2d = t_events(lambda: dev.copy_(host, non_blocking=True))
    d2h = t_events(lambda: out.copy_(dvol, non_blocking=True))
print(f"H2D {host.numel()*4/1e6:.0f} MB {h2d:.2f} ms = {host.numel()*4/h2d/1e6:.1f} GB/s")
print(f"D2H {out.numel()*4/1e6:.0f} MB {d2h:.2f} ms = {out.numel()*4/d2h/1e6:.1f} GB/s")
ws = p._workspace(p.workspace_bytes(cfg["n_pitches"]))
def dev_step():
    p.reconstruct(dev, v0, 0, cfg["n_pitches"], out=dvol, stream=s)
print(f"device step {t_events(dev_step):.2f} ms")
for _ in range(2): p.reconstruct_host(host, v0, 0, cfg["n_pitches"], out_host=out, stream=s)
torch.cuda.synchronize()
for rep in range(3):
    t = time.perf_counter(); n = 5
    for _ in range(n): p.reconstruct_host(host, v0, 0, cfg["n_pitches"], out_host=out, stream=s)
    torch.cuda.synchronize()
    print(f"host step {(time.perf_counter()-t)*1e3/n:.2f} ms")
# CPU-side enqueue cost of one host call (GPU work included, synchronous)
t = time.perf_counter(); p.reconstruct_host(host, v0, 0, cfg["n_pitches"], out_host=out, stream=s); print(f"single call {(time.perf_counter()-t)*1e3:.2f} ms")
p.profile_enable(True)
p.reconstruct_host(host, v0, 0, cfg["n_pitches"], out_host=out, stream=s)
st = p.profile_read()
print("profiled stages in host call:", {kk: round(v, 2) for kk, v in st["ms"].items()})
