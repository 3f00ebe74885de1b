"""bench.py — device-timed Katsevich reconstruction throughput (BASELINE.json metric:
voxel-view updates/s and volumes/s).

Workload (N=1): C4 — 512^3 long helical scan (8 pitches x 64 slices), 64 x 184
curved detector (sparse 4x), 1152 views/turn, normalised pitch 1.5
(BASELINE.json configs[3]; the config the metric's 1/2/4/8-GPU numbers are
quoted on).  One step = one full reconstruction of the rank's pitches
(filter steps 1-6 on every needed view + PI-limited backprojection of every
pitch), inputs already resident in HBM.

Multi-GPU (torchrun): the C4 scan's 8 pitches split across the
N ranks (strong scaling): rank r reconstructs pitches [8r/N, 8(r+1)/N) from
the views they need (its pitches plus the PI-window overlap) and NCCL gathers
the volume slabs to rank 0 INSIDE the timed region, point to point, per pitch
group: the send of group i overlaps the backprojection of group i+1
(katsevich_reconstruct_grouped marks each group with a CUDA event).  The
compute-only time (no gather) is reported beside it.  `--scaling weak`: every
rank reconstructs its own 8 pitches of an 8N-pitch scan, no collective.

`--impl reference`: the CPU oracle (oracle/) timed on the host cores, each step
one whole slice of the workload (every voxel of the slice and the filtering of
every view its PI windows need), measured, not extrapolated.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# --- clocks sampling during the timed region (nvidia-smi) ------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0])); mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --- workload ----------------------------------------------------------------
def workload(name: str):
    from synth import configs
    cfg = configs.get(name)
    return cfg


def rank_phantom(cfg, first_pitch):
    """The config phantom, shifted so each rank's pitch block sees the same object."""
    ph = np.array(cfg["phantom"], dtype=np.float64).copy()
    ph[:, 2] += first_pitch * cfg["P"]
    return ph


def count_updates(plan) -> int:
    """U = Σ_voxels #{k : ω_k > 0} for one pitch (identical for every pitch)."""
    t = plan.export_tables()
    m = t["pi_last"] >= t["pi_first"]
    n = (t["pi_last"] - t["pi_first"] + 1)[m].astype(np.int64)
    # views with zero end weight never occur under reading A12 (no zero-weight ends)
    return int(n.sum())


def bp_flops_per_update():
    # algorithmic FP32 work of one voxel-view update:
    # w* position FFMA (2) + 2 column lerps (2 x (FADD+FFMA) = 6) + row lerp (3)
    # + weighted accumulate FFMA with 1/v* (2)  = 13 flops
    return 13.0


def bp_smem_bytes_per_update():
    # algorithmic on-chip gather of one update: the bilinear sample of gF at (α*, w*) reads
    # 4 fp32 neighbours = 16 B (held as one (s', s', d, d) quad)
    return 16.0


def smem_peak_gbs(sm_mhz):
    """K5's roofline denominator: the MEASURED LDS.128 throughput of this GPU model
    (scripts/micro/smem_peak.cu, profiles/smem_peak.json) when present, else the derived
    148 SMs x 128 B/clk (one LSU wavefront per clock) at sm_mhz.  Returns (GB/s, source)."""
    try:
        with open(os.path.join(ROOT, "profiles", "smem_peak.json")) as f:
            d = json.load(f)
        return float(d["smem_lds128_gbs"]), ("measured LDS.128 throughput (scripts/micro/smem_peak.cu, "
                                              f"profiles/smem_peak.json: {d['bytes_per_clk_per_sm_at_max']:.1f} "
                                              "B/clk/SM at the max clock)")
    except Exception:
        return 148 * 128 * sm_mhz * 1e6 / 1e9, f"derived: 148 SMs x 128 B/clk x {sm_mhz} MHz"


PAPER_CONTEXT = {
    "reported": "no reconstruction time or throughput for the Katsevich layer (BASELINE.md section 1)",
    "closest": "full network training step (sinogram CNN + Katsevich layer + image CNN, fwd+bwd) about 5-6 s, "
               "batch 1, one 581-view x 16 x 627 slab -> 512x512x10, NVIDIA RTX A6000, TensorFlow 2.5 (P:l.302-304)",
    "derived_bound": ">= ~9e7 voxel-view updates/s on the A6000 if the whole step were the layer (BASELINE.md)",
}


def n_filtered_views(plan, cfg, n_items, batch):
    ti = plan.table_info()
    per_slab = ti["bp_hi"] - ti["bp_lo"] + 1
    if batch:
        return per_slab * batch
    return (n_items - 1) * cfg["views_per_turn"] + per_slab          # filter-once over the union


def filter_stage_rooflines(plan, cfg, stats, steps, nu, hbm_peak):
    """Achieved GB/s of each filter stage's ALGORITHMIC HBM bytes as SURVEY §8(d) counts them (each
    input read once, each output written once, 4 B per fp32 element: K12 reads the raw views and
    writes g3, K3 reads g3 and writes g4, K4 reads g4 and writes gF) against the HBM peak.  K4 in
    fact writes gF as 2x2 tap quads (16 B per (row + 2, column)): those bytes are
    reported beside, not counted."""
    npsi = plan.table_info()["n_psi"]
    nr, nc = cfg["n_rows"], cfg["n_cols"]
    by = {"K12_deriv_fwd_rebin": 4.0 * (nu + 2) * nr * nc + 4.0 * nu * npsi * nc,
          "K3_hilbert": 8.0 * nu * npsi * nc,
          "K4_bwd_rebin_cos": 4.0 * nu * npsi * nc + 4.0 * nu * nr * nc}
    out = {}
    for k, b in by.items():
        ms = stats["busy_ms"].get(k, 0.0) / steps
        if ms > 0:
            gbs = b / (ms * 1e-3) / 1e9
            out[k] = {"ms_per_step": ms, "algorithmic_bytes": b, "achieved_gbs": gbs, "hbm_peak_gbs": hbm_peak,
                      "frac": gbs / hbm_peak}
    if "K4_bwd_rebin_cos" in out:
        out["K4_bwd_rebin_cos"]["quad_bytes_written"] = 16.0 * nu * nc * (nr + 2)
    return out


def ncu_traffic(config_name):
    """dram bytes per K5 launch from the committed ncu --set full summary, if present."""
    path = os.path.join(ROOT, "profiles", "ncu_k5_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        if d.get("config") == config_name:                     # (single-config form)
            return d.get("dram_bytes_per_launch")
        if isinstance(d.get(config_name), dict):               # keyed by config
            return d[config_name].get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2201_02309_b200 as k
    from synth import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    cfg = workload(args.config)
    pitches = cfg["n_pitches"]
    batch = cfg.get("batch", 0)
    plan = k.Plan(cfg, device=local)
    t0 = time.perf_counter()
    plan.precompute()
    t_pre = time.perf_counter() - t0
    vt = cfg["views_per_turn"]

    # ---- inputs (seeded, synthetic; generated on the host, moved to HBM before timing) ----
    from paper_2201_02309_b200 import dist as kd
    gather = False
    if batch:
        from synth import configs
        v0, nv = plan.pitch_views(0)
        phs = configs.c5_phantoms(batch)
        host_in = np.stack([synth.project(cfg, phs[b], v0, nv) for b in range(batch)])
        first_pitch, n_items = 0, batch
    else:
        if args.scaling == "weak":
            shards = [kd.weak_shard(pitches, r) for r in range(world)]
        else:  # strong (default): the config's pitches split [P r / N, P (r+1) / N)
            shards = kd.pitch_shards(cfg["n_pitches"], world)
        me = shards[rank]
        first_pitch, pitches = me.first_pitch, me.n_pitches
        if pitches < 1:
            raise SystemExit(f"rank {rank}: no pitch to reconstruct ({cfg['n_pitches']} pitches over {world} ranks)")
        v0, nv = plan.scan_views(first_pitch, pitches)
        host_in = synth.project(cfg, rank_phantom(cfg, first_pitch - (first_pitch % cfg["n_pitches"])), v0, nv)
        n_items = pitches
        gather = world > 1 and args.scaling == "strong" and not args.no_gather
    dev_in = torch.from_numpy(host_in).to(dev)
    vol_shape = (n_items * cfg["nz"], cfg["ny"], cfg["nx"]) if not batch else (batch, cfg["nz"], cfg["ny"], cfg["nx"])
    stream = torch.cuda.current_stream(dev)
    groups, gobj, full, evs, side = 1, None, None, None, None
    if gather:
        # rank 0 owns the whole volume and reconstructs its own pitches straight into its slice;
        # the others send each pitch group as soon as its backprojection is done
        groups = max(1, min(args.gather_groups, pitches))
        gobj = kd.SlabGather(shards, cfg["nz"], parts=groups)
        if rank == 0:
            full = torch.empty((cfg["n_pitches"] * cfg["nz"], cfg["ny"], cfg["nx"]), dtype=torch.float32, device=dev)
            out = full[gobj.rows(me)]
        else:
            out = torch.empty(vol_shape, dtype=torch.float32, device=dev)
        evs = [torch.cuda.Event() for _ in range(groups)]
        for e in evs:
            e.record(stream)                  # creates the events (handles for the C ABI)
        side = torch.cuda.Stream(dev)
    else:
        out = torch.empty(vol_shape, dtype=torch.float32, device=dev)

    def step(with_gather=True):
        if batch:
            plan.reconstruct_batch(dev_in, out=out, stream=stream)
            return
        if not (gather and with_gather):
            plan.reconstruct(dev_in, v0, first_pitch, pitches, out=out, stream=stream)
            return
        works = gobj.post_recvs(full) if rank == 0 else []
        plan.reconstruct_grouped(dev_in, v0, first_pitch, pitches, groups, group_events=evs, out=out, stream=stream)
        if rank != 0:
            for i in range(groups):
                with torch.cuda.stream(side):          # the send of group i waits for group i only
                    side.wait_event(evs[i])
                    works.append(gobj.send(rank, i, out[gobj.local_rows(rank, i)]))
        for w in works:
            w.wait()                                   # the caller's stream waits for the transfers

    def timed_loop(n, with_gather=True):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            step(with_gather)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([t], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)     # max over ranks
            t = float(tt.item())
        return t

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    compute_only_ms = None
    if gather:
        for _ in range(max(1, args.warmup // 2)):
            step(False)
        compute_only_ms = timed_loop(args.steps, False) / args.steps
    plan.profile_read(reset=True)
    plan.profile_enable(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ms = timed_loop(args.steps)
    clk = clocks.stop()
    stats = plan.profile_read(reset=True)
    plan.profile_enable(False)
    ms_step = ms / args.steps
    step_bp_kernel = plan.bp_kernel()          # the timed step's step-7 kernel (before the e2e / adjoint runs)

    # ---- the same step replayed from a captured CUDA graph (every device entry point is capturable:
    # no host synchronisation or allocation inside); single process only ----
    graph = None
    if world == 1 and not args.no_graph:
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(stream)

        def gstep():
            if batch:
                plan.reconstruct_batch(dev_in, out=out, stream=gs)
            else:
                plan.reconstruct(dev_in, v0, first_pitch, pitches, out=out, stream=gs)
        gstep()                                              # warm on the capture stream
        torch.cuda.synchronize()
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg, stream=gs):
            gstep()
        with torch.cuda.stream(gs):                          # replays go to the current stream
            for _ in range(args.warmup):
                cg.replay()
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(gs)
            for _ in range(args.steps):
                cg.replay()
            g1.record(gs)
        torch.cuda.synchronize()
        graph = {"ms_per_step": g0.elapsed_time(g1) / args.steps,
                 "what": "the timed step captured once into a CUDA graph (torch.cuda.graph) and replayed"}
        del cg

    # ---- K5 in isolation: the same step with one backprojection launch over all of the rank's
    # pitches after all filtering (KATS_PIPELINE=0, the default), so no other kernel shares the GPU
    # with it (differs from the timed region only when KATS_PIPELINE=1 is set) ----
    iso = None
    st_iso = None
    saved = {e: os.environ.get(e) for e in ("KATS_PIPELINE", "KATS_FILTER_STREAMS", "KATS_BATCH_GROUPS")}
    os.environ["KATS_PIPELINE"] = "0"
    os.environ["KATS_FILTER_STREAMS"] = "1"       # one filter stream: every kernel runs alone
    os.environ["KATS_BATCH_GROUPS"] = "1"         # batches: one step-7 launch after all filtering
    step()
    torch.cuda.synchronize()
    plan.profile_read(reset=True)
    plan.profile_enable(True)
    n_iso = 3
    for _ in range(n_iso):
        step()
    torch.cuda.synchronize()
    st_iso = plan.profile_read(reset=True)
    plan.profile_enable(False)
    for e, v in saved.items():
        if v is None:
            os.environ.pop(e, None)
        else:
            os.environ[e] = v
    k = "K5_backproject"
    iso = {"k5_ms_per_launch": st_iso["ms"][k] / max(1, st_iso["launches"][k]),
           "launches": st_iso["launches"][k] // n_iso}
    st_iso = {"busy_ms": dict(st_iso["ms"]), "n": n_iso}

    # ---- e2e: host (pinned) in -> host out through katsevich_reconstruct_host ----
    e2e = None
    if True:
        pin_in = torch.from_numpy(host_in).pin_memory()
        pin_out = torch.empty(vol_shape, dtype=torch.float32).pin_memory()
        if batch:       # the training batch from host memory: katsevich_reconstruct_batch_host
            run_host = lambda: plan.reconstruct_batch_host(pin_in, out_host=pin_out, stream=stream)
        else:
            run_host = lambda: plan.reconstruct_host(pin_in, v0, first_pitch, pitches, out_host=pin_out, stream=stream)
        for _ in range(2):
            run_host()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t1 = time.perf_counter()
        ne = max(3, min(args.steps, 10))
        for _ in range(ne):
            run_host()
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t1) * 1e3 / ne
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"ms_per_step": e2e_ms, "h2d": pin_in.numel() * 4, "d2h": pin_out.numel() * 4}

    # ---- adjoint (NEXT-1): the transpose of the same step, volume -> sinogram, device-resident ----
    adj = None
    if not args.no_adjoint:
        vol_y = torch.randn(out.shape, device=dev, generator=torch.Generator(device=dev).manual_seed(11))
        sino_t = torch.empty(tuple(host_in.shape), dtype=torch.float32, device=dev)
        if batch:      # training-shaped batches: katsevich_adjoint_batch
            run_adj = lambda: plan.adjoint_batch(vol_y, out=sino_t, stream=stream)
        else:
            run_adj = lambda: plan.adjoint(vol_y, v0, sino_t.shape[0], first_pitch, pitches, out=sino_t,
                                           stream=stream)
        for _ in range(args.warmup):
            run_adj()
        torch.cuda.synchronize()
        plan.profile_read(reset=True)
        plan.profile_enable(True)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(args.steps):
            run_adj()
        a1.record(stream)
        torch.cuda.synchronize()
        st_adj = plan.profile_read(reset=True)
        plan.profile_enable(False)
        adj_ms = a0.elapsed_time(a1) / args.steps
        if world > 1:
            t = torch.tensor([adj_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            adj_ms = float(t.item())
        adj = {"ms_per_step": adj_ms, "k5T_ms_per_step": st_adj["ms"]["K5_backproject"] / args.steps}
        del vol_y, sino_t

    # ---- data generation (NEXT-3): projection of the workload's phantom over the rank's scan,
    # ray marching through the reconstructed volume (a view subset), sparse-view + noise degradation ----
    dg = None
    if not batch and not args.no_datagen:
        nvs = host_in.shape[0]
        sino_g = torch.empty(tuple(host_in.shape), dtype=torch.float32, device=dev)
        nvv = min(64, nvs)
        sino_v = torch.empty((nvv,) + tuple(host_in.shape[1:]), dtype=torch.float32, device=dev)
        zf, dzv = float(first_pitch * cfg["P"]), cfg["P"] / cfg["nz"]

        def timed(fn, reps):
            for _ in range(max(1, args.warmup)):
                fn()
            torch.cuda.synchronize()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            for _ in range(reps):
                fn()
            b1.record(stream)
            torch.cuda.synchronize()
            return b0.elapsed_time(b1) / reps

        ph = cfg["phantom"]
        ms_pe = timed(lambda: plan.project_ellipsoids(ph, v0, nvs, out=sino_g, stream=stream), args.steps)
        ms_pv = timed(lambda: plan.project_volume(out, zf, dzv, v0 + nvs // 2, nvv, out=sino_v, stream=stream), 3)
        ms_dg = timed(lambda: plan.degrade(sino_g, v0, 4, 1e5, 0.5, 1234, stream=stream), args.steps)
        rays = nvs * cfg["n_rows"] * cfg["n_cols"]
        dg = {"project_ellipsoids": {"value": rays / (ms_pe * 1e-3), "unit": "rays/s", "ms": ms_pe, "rays": rays,
                                     "ellipsoids": len(ph), "precision": "f64"},
              "project_volume": {"value": nvv * cfg["n_rows"] * cfg["n_cols"] / (ms_pv * 1e-3), "unit": "rays/s",
                                 "ms": ms_pv, "views": nvv,
                                 "volume_xyz": [cfg["nx"], cfg["ny"], int(out.shape[0])], "precision": "f32"},
              "degrade": {"value": rays / (ms_dg * 1e-3), "unit": "samples/s", "ms": ms_dg,
                          "what": "alpha stride 4 + 'Gaussian+Poisson' (I0 1e5, var 0.5), Philox4x32-10"}}
        del sino_g, sino_v

    # ---- method variants (NEXT-4): the same step with Noo's half-sample derivative and with the
    # Hann-apodised filter at this config, and the flat-detector counterpart config where one exists
    # (C2 -> C2F); device-resident, CUDA events, one process (rank 0 of a single-rank run) ----
    var = None
    if world == 1 and not args.no_variants:
        from synth import configs as _cf

        import paper_2201_02309_b200 as _kpkg

        def vstep(vcfg, reuse_input):
            vp = _kpkg.Plan(vcfg, device=local)
            vp.precompute()
            if batch:
                a0_, n_ = vp.pitch_views(0)
                x = dev_in if reuse_input else torch.from_numpy(
                    np.stack([synth.project(vcfg, phs[b], a0_, n_) for b in range(batch)])).to(dev)
                o = torch.empty(vol_shape, dtype=torch.float32, device=dev)
                fn = lambda: vp.reconstruct_batch(x, out=o, stream=stream)
            else:
                a0_, n_ = vp.scan_views(first_pitch, pitches)
                x = dev_in if reuse_input else torch.from_numpy(
                    synth.project(vcfg, rank_phantom(vcfg, first_pitch - (first_pitch % vcfg["n_pitches"])), a0_, n_)).to(dev)
                o = torch.empty((pitches * vcfg["nz"], vcfg["ny"], vcfg["nx"]), dtype=torch.float32, device=dev)
                fn = lambda: vp.reconstruct(x, a0_, first_pitch, pitches, out=o, stream=stream)
            for _ in range(args.warmup):
                fn()
            torch.cuda.synchronize()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            for _ in range(args.steps):
                fn()
            b1.record(stream)
            torch.cuda.synchronize()
            ms = b0.elapsed_time(b1) / args.steps
            u = count_updates(vp) * n_items
            del x, o
            return {"ms_per_step": ms, "value": u / (ms * 1e-3), "unit": "updates/s", "bp_kernel": vp.bp_kernel()}

        var = {"half_sample": dict(vstep(dict(cfg, flags=1), False), flags=1,
                                   what="Noo's 2x2x2 half-sample derivative (reading A25), same scan"),
               "hann": dict(vstep(dict(cfg, flags=2), True), flags=2,
                            what="Hann-apodised Hilbert filter (reading A26), same input")}
        try:
            fcfg = _cf.get(cfg["name"] + "F")
        except KeyError:
            fcfg = None
        if fcfg is not None and not batch:
            var["flat"] = dict(vstep(fcfg, False), config=fcfg["name"],
                               what="flat-detector counterpart (reading A27): " + fcfg["desc"])
        torch.cuda.synchronize()

    items_all, launches_all = n_items, stats["total_launches"]
    if world > 1:
        tt = torch.tensor([n_items, launches_all], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        items_all, launches_all = int(tt[0].item()), int(tt[1].item())
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    U_pitch = count_updates(plan)
    U_rank = U_pitch * n_items
    U_all = U_pitch * items_all                    # units every rank processed
    vols_all = items_all / (cfg["n_pitches"] if not batch else batch)
    value = U_all / (ms_step * 1e-3)
    # roofline of the dominant kernel (K5 backprojection), CUDA events recorded by the library on
    # the launching streams. Per-pitch K5 launches run on two alternating streams and overlap, so
    # the K5 time is its busy time (union of its launch intervals) per step, not a sum of durations.
    k5 = "K5_backproject"
    k5_launches_per_step = max(1, stats["launches"][k5] // args.steps)
    k5_ms_launch = stats["ms"][k5] / max(1, stats["launches"][k5])
    k5_busy = stats["busy_ms"][k5] / args.steps
    achieved_tflops = U_rank * bp_flops_per_update() / (k5_busy * 1e-3) / 1e12
    peaks, src = _peaks()
    fp32_peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    smem_peak, smem_src = smem_peak_gbs(peaks.get("sm_max_mhz", 1965.0))
    achieved_smem = U_rank * bp_smem_bytes_per_update() / (k5_busy * 1e-3) / 1e9
    bp_kernel = step_bp_kernel
    share = {s: stats["busy_ms"][s] / args.steps / ms_step for s in stats["busy_ms"] if stats["busy_ms"][s] > 0}
    line = {
        "metric": "voxel-view updates/s",
        "value": value,
        "unit": "updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak" if (args.scaling == "weak" or batch) else "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded analytic Shepp-Logan helical projections, synth/)",
        "config": {"workload": f"{cfg['name']}: {cfg['desc']}", "volume_xyz": [cfg["nx"], cfg["ny"], cfg["nz"] * cfg["n_pitches"]],
                   "detector": [cfg["n_rows"], cfg["n_cols"]], "views_per_turn": vt,
                   "scan_views_per_rank": int(host_in.shape[0]) if not batch else int(host_in.shape[1]),
                   "pitches_per_rank": n_items,
                   "parallelism": (f"pitch-sharded x{world}" + (f", NCCL point-to-point gather of the volume slabs to "
                                   f"rank 0 inside the timed region ({groups} overlapped pitch groups per rank)"
                                   if gather else "")) if not batch else f"batch replicas x{world}",
                   "l2": "inputs larger than L2 (scan %.0f MB, filtered views %.0f MB > 126 MB L2)" % (
                       host_in.nbytes / 1e6,
                       16.0 * n_filtered_views(plan, cfg, n_items, batch) * cfg["n_cols"] * (cfg["n_rows"] + 2) / 1e6)},
        "volumes_per_s": vols_all / (ms_step * 1e-3),
        "updates_per_step": U_all,
        "compute_only": None if compute_only_ms is None else {
            "ms_per_step": compute_only_ms, "value": U_all / (compute_only_ms * 1e-3), "unit": "updates/s",
            "note": "the same step without the gather (max over ranks)"},
        "gpu_launches": launches_all,
        "stage_busy_share_of_step": share,
        "filter_stages": filter_stage_rooflines(plan, cfg, stats, args.steps, n_filtered_views(plan, cfg, n_items, batch),
                                                peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])),
        "filter_stages_isolated": filter_stage_rooflines(plan, cfg, st_iso, st_iso["n"],
                                                         n_filtered_views(plan, cfg, n_items, batch),
                                                         peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])),
        "paper_context": PAPER_CONTEXT,
        "precompute_s": t_pre,
        "roofline": {"bound": "smem", "kernel": bp_kernel, "achieved": achieved_smem, "peak": smem_peak,
                     "unit": "GB/s", "frac": achieved_smem / smem_peak,
                     "traffic": ncu_traffic(cfg["name"]),
                     "bytes_per_update": bp_smem_bytes_per_update(),
                     "k5_busy_ms_per_step": k5_busy, "k5_launches_per_step": k5_launches_per_step,
                     "k5_ms_per_launch": k5_ms_launch, "k5_updates_per_s": U_rank / (k5_busy * 1e-3),
                     "peak_source": smem_src + "; DESIGN.md §5",
                     "secondary_hbm": None if not ncu_traffic(cfg["name"]) else {
                         "achieved": ncu_traffic(cfg["name"]) / (k5_ms_launch * 1e-3) / 1e9,
                         "peak": peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]), "unit": "GB/s",
                         "note": "ncu DRAM bytes of one K5 launch (profiles/ncu_k5_traffic.json) / the timed "
                                 "region's average K5 launch time: far from bound"},
                     "secondary_alu": {"achieved": achieved_tflops, "peak": fp32_peak, "unit": "TFLOP/s",
                                       "frac": achieved_tflops / fp32_peak,
                                       "flops_per_update": bp_flops_per_update()},
                     "note": "achieved = 16 B x updates per step / K5 busy time per step in the timed "
                             "region (per-pitch K5 launches overlap each other and the filter there, so "
                             "this is a lower bound); isolated = one K5 launch for all pitches, alone",
                     "isolated": None if iso is None else {
                         "k5_ms_per_launch": iso["k5_ms_per_launch"], "k5_launches_per_step": iso["launches"],
                         "achieved": U_rank * bp_smem_bytes_per_update()
                         / (iso["k5_ms_per_launch"] * max(1, iso["launches"]) * 1e-3) / 1e9,
                         "frac": U_rank * bp_smem_bytes_per_update()
                         / (iso["k5_ms_per_launch"] * max(1, iso["launches"]) * 1e-3) / 1e9 / smem_peak}},
        "clocks": clk,
    }
    if dg:
        line["datagen"] = dg
    if var:
        line["variants"] = var
    if graph:
        graph["value"] = U_all / (graph["ms_per_step"] * 1e-3)
        graph["unit"] = "updates/s"
        line["cuda_graph"] = graph
    if adj:
        line["adjoint"] = {"metric": "voxel-view updates/s (transpose: volume -> sinogram)",
                           "value": U_all / (adj["ms_per_step"] * 1e-3), "unit": "updates/s",
                           "ms_per_step": adj["ms_per_step"], "k5T_ms_per_step": adj["k5T_ms_per_step"],
                           "note": ("katsevich_adjoint_batch over the same slabs" if batch else
                                    "katsevich_adjoint over the same pitches") + ", inputs resident, CUDA events"}
    if e2e:
        line["e2e"] = {"value": U_all / (e2e["ms_per_step"] * 1e-3), "unit": "updates/s",
                       "ms_per_step": e2e["ms_per_step"],
                       "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"]}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# --- CPU oracle timing (measured on bounded samples, no extrapolation) -------
def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


class OracleSlice:
    """One whole slice of the workload as the oracle's unit of timed work: every voxel of slice j
    of pitch 0 (step 7 over each voxel's PI window) and steps 1-6 on every view those windows
    need, from seeded random data of the workload's shape.  The oracle's per-geometry filter set-up
    (Hilbert kernel, rebin maps) is built once outside the timed calls (oracle.PreparedFilter)."""

    def __init__(self, cfg):
        from oracle import oracle
        self.cfg = cfg
        t0 = time.perf_counter()
        self.filt = oracle.PreparedFilter(cfg)
        self.t_filter_setup = time.perf_counter() - t0

    def run(self, j, seed=0):
        from oracle import oracle
        from synth import synth
        cfg = self.cfg
        nx, ny = cfg["nx"], cfg["ny"]
        iy, ix = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        idx = np.stack([ix.ravel(), iy.ravel(), np.full(nx * ny, j)], 1).astype(np.int32)
        kf, kl, _, _ = oracle.bp_weights_voxels(cfg, 0, idx)      # tables: not timed (precompute)
        m = kl >= kf
        lo, hi = int(kf[m].min()), int(kl[m].max())
        n = hi - lo + 1
        raw = synth.random_array((n + 2, cfg["n_rows"], cfg["n_cols"]), seed)
        t0 = time.perf_counter()
        gF = self.filt.gF(raw, lo - 1, lo, n)
        t_f = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.backproject_voxels(cfg, 0, gF, lo, idx)
        t_b = time.perf_counter() - t0
        return dict(updates=int(np.where(m, kl - kf + 1, 0).sum()), views=n, voxels=nx * ny, t_filter=t_f,
                    t_bp=t_b, slice=j)


def cpu_baseline(cfg):
    """The oracle (fp64, OpenMP) on this host, measured: (1) one whole slice of the workload —
    every voxel and the filtering of every view it needs — the rate of the metric; (2) the
    oracle's own precompute for one pitch (rebin maps + PI windows of every voxel, P:l.265
    "implemented by the CPU"); (3) the whole C1 reconstruction (BASELINE configs[0], "CPU oracle
    in seconds") single-thread and all-core."""
    from oracle import oracle
    from synth import configs, synth
    oracle.set_threads(0)
    threads = oracle.get_threads()
    t0 = time.perf_counter()
    oracle.rebin_tables(cfg)
    oracle.bp_weights(cfg, 0)
    t_pre = time.perf_counter() - t0
    sl = OracleSlice(cfg)
    r = sl.run(cfg["nz"] // 2)
    t = r["t_filter"] + r["t_bp"]
    c1 = configs.get("C1")
    sino1 = synth.project(c1, c1["phantom"], c1["scan_v0"], c1["scan_nv"])
    kf1, kl1, _, _ = oracle.bp_weights(c1, 0)
    u1 = int(np.where(kl1 >= kf1, kl1 - kf1 + 1, 0).sum())
    c1t = {}
    for nt in (1, threads):
        oracle.set_threads(nt)
        t0 = time.perf_counter()
        oracle.reconstruct(c1, sino1, c1["scan_v0"], 0, 1)
        c1t[nt] = time.perf_counter() - t0
    oracle.set_threads(0)
    return {"value": r["updates"] / t, "unit": "updates/s", "cores": threads, "kind": "oracle",
            "sample": (f"{cfg['name']} slice {r['slice']} of pitch 0, measured whole: all {r['voxels']} voxels "
                       f"({r['updates']} voxel-view updates) + steps 1-6 on the {r['views']} views their PI "
                       f"windows need; seeded random data, fp64, {threads} OpenMP threads"),
            "seconds": t, "seconds_filter": r["t_filter"], "seconds_backprojection": r["t_bp"],
            "seconds_per_view_filter": r["t_filter"] / r["views"], "seconds_per_update": r["t_bp"] / r["updates"],
            "precompute_seconds": {"tables_one_pitch": t_pre, "filter_setup": sl.t_filter_setup,
                                   "what": "oracle rebin maps + PI windows of every voxel of one pitch (bisection)"},
            "c1_full_reconstruction_seconds": {"threads_1": c1t[1], f"threads_{threads}": c1t[threads],
                                               "updates": u1,
                                               "what": "whole C1 pitch (64^3, filter + backprojection) incl. the "
                                                       "oracle's per-call rebin maps and PI windows"}}


def run_reference(args):
    """The base contract's reference arm for this tier: the CPU oracle, unmodified, timed on the
    host cores.  Each step is one whole slice of the workload (OracleSlice, the slices taken in
    turn), so a step is a bounded, fully measured piece of the same work; value = updates of the
    K timed steps / their time."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle
    cfg = workload(args.config)
    oracle.set_threads(0)
    threads = oracle.get_threads()
    sl = OracleSlice(cfg)
    nz = cfg["nz"]
    for i in range(args.warmup):
        sl.run((nz // 2 + i) % nz, seed=i)
    runs = [sl.run((nz // 2 + args.warmup + i) % nz, seed=args.warmup + i) for i in range(args.steps)]
    t = sum(r["t_filter"] + r["t_bp"] for r in runs)
    upd = sum(r["updates"] for r in runs)
    value = upd / t
    line = {"impl": "reference", "metric": "voxel-view updates/s", "value": value, "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3 / args.steps,
            "higher_is_better": True, "vs_baseline": None, "dtype": "f64",
            # (our arm's rule for the same config: batches and --scaling weak are weak, else strong)
            "scaling": "weak" if (args.scaling == "weak" or cfg.get("batch")) else "strong",
            "data": "synthetic (seeded random arrays of the workload's shapes)",
            "config": {"workload": f"{cfg['name']}: {cfg['desc']}",
                       "step": "one whole slice of pitch 0 (all its voxels + the filtering of the views they need)"},
            "cpu_baseline": {"value": value, "unit": "updates/s", "cores": threads, "kind": "oracle",
                             "sample": f"per step one whole {cfg['name']} slice ({runs[0]['voxels']} voxels, "
                                       f"~{upd // args.steps} updates, ~{runs[0]['views']} filtered views), measured"},
            "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): the config's pitches split over the ranks + NCCL gather to rank 0; "
                         "weak: 8 pitches per rank of a longer scan, no collective")
    ap.add_argument("--no-gather", action="store_true", help="strong scaling without the volume gather")
    ap.add_argument("--gather-groups", type=int, default=2,
                    help="pitch groups per rank whose sends overlap the next group's backprojection")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-adjoint", action="store_true", help="skip the adjoint (NEXT-1) measurement")
    ap.add_argument("--no-datagen", action="store_true", help="skip the data-generation (NEXT-3) measurement")
    ap.add_argument("--no-variants", action="store_true", help="skip the method-variant (NEXT-4) measurements")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
