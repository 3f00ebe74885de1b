"""Whole-workload CPU oracle runs (SURVEY §8(d) "Oracle timing"): every config C1-C5 reconstructed
completely by the fp64 oracle on all host cores — filter (steps 1-6) and backprojection (step 7)
timed separately, the oracle's precompute (rebin maps + PI windows of one pitch) separately — plus
C1 single-thread.  Seeded synthetic inputs (the configs' analytic phantoms; C5: 16 seeded slabs).
Writes one JSON object (stdout).  Test infrastructure: runs the oracle only."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
from synth import configs, synth  # noqa: E402


def run(name, threads=0):
    oracle.set_threads(threads)
    cfg = configs.get(name)
    t0 = time.perf_counter()
    oracle.rebin_tables(cfg)
    kf, kl, _, _ = oracle.bp_weights(cfg, 0)
    t_pre = time.perf_counter() - t0
    U_pitch = int(np.where(kl >= kf, kl - kf + 1, 0).sum())
    filt = oracle.PreparedFilter(cfg)
    items = [(k, None) for k in range(cfg["n_pitches"])] if not cfg.get("batch") else \
        [(0, ph) for ph in configs.c5_phantoms(cfg["batch"])]
    t_f = t_b = 0.0
    n_views = 0
    for k, ph in items:
        fv, nv = oracle.pitch_slab(cfg, k)
        sino = synth.project(cfg, cfg["phantom"] if ph is None else ph, fv, nv)
        t0 = time.perf_counter()
        gF = filt.gF(sino, fv, fv + 1, nv - 2)
        t_f += time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.backproject(cfg, k, gF, fv + 1)
        t_b += time.perf_counter() - t0
        n_views += nv - 2
    U = U_pitch * len(items)
    return {"config": name, "threads": oracle.get_threads(), "items": len(items), "updates": U,
            "filtered_views": n_views, "seconds_filter": t_f, "seconds_backprojection": t_b,
            "seconds_total": t_f + t_b, "updates_per_s": U / (t_f + t_b),
            "seconds_precompute_one_pitch": t_pre}


if __name__ == "__main__":
    out = {"host_cores": len(os.sched_getaffinity(0)), "runs": []}
    out["runs"].append(run("C1", threads=1))
    for name in ("C1", "C2", "C3", "C5", "C4"):
        out["runs"].append(run(name))
        print(json.dumps(out["runs"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out))
