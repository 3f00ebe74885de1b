"""bench.py — device-timed Katsevich reconstruction throughput (BASELINE.json metric:
voxel-view updates/s and volumes/s).

Workload (N=1): C4 — 512^3 long helical scan (8 pitches x 64 slices), 64 x 184
curved detector (sparse 4x), 1152 views/turn, normalised pitch 1.5
(BASELINE.json configs[3]; the config the metric's 1/2/4/8-GPU numbers are
quoted on).  One step = one full reconstruction of the rank's pitches
(filter steps 1-6 on every needed view + PI-limited backprojection of every
pitch), inputs already resident in HBM.

Multi-GPU (torchrun): pitch sharding, weak scaling — rank r reconstructs its
own 8 pitches [8r, 8r+8) of an (8N)-pitch scan from its own view range; no
collective on the data path.  `--gather` adds the NCCL
gather of the volume slabs to rank 0 inside the timed region.

`--impl reference`: the CPU oracle (oracle/) timed on the host cores on a
bounded sample of the same workload, extrapolated to the same metric.
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
    # shared-memory data pipe: 128 B/clk per SM (1 LSU wavefront/clk), 148 SMs
    return 148 * 128 * sm_mhz * 1e6 / 1e9


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
    """Achieved GB/s of each filter stage's ALGORITHMIC HBM bytes (each input read once, each output
    written once; g3/g4 of a 256-view chunk may in fact stay in L2) against the HBM peak."""
    npsi = plan.table_info()["n_psi"]
    nr, nc = cfg["n_rows"], cfg["n_cols"]
    by = {"K12_deriv_fwd_rebin": 4.0 * (nu + 2) * nr * nc + 4.0 * nu * npsi * nc,
          "K3_hilbert": 8.0 * nu * npsi * nc,
          "K4_bwd_rebin_cos": 4.0 * nu * npsi * nc + 16.0 * nu * nc * (nr + 2)}
    out = {}
    for k, b in by.items():
        ms = stats["busy_ms"].get(k, 0.0) / steps
        if ms > 0:
            gbs = b / (ms * 1e-3) / 1e9
            out[k] = {"ms_per_step": ms, "algorithmic_bytes": b, "achieved_gbs": gbs, "hbm_peak_gbs": hbm_peak,
                      "frac": gbs / hbm_peak}
    return out


def ncu_traffic(config_name):
    """dram bytes per K5 launch from the committed ncu --set full summary, if present."""
    path = os.path.join(ROOT, "profiles", "ncu_k5_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        if d.get("config") == config_name:
            return d.get("dram_bytes_per_launch")
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
    if batch:
        from synth import configs
        v0, nv = plan.pitch_views(0)
        phs = configs.c5_phantoms(batch)
        host_in = np.stack([synth.project(cfg, phs[b], v0, nv) for b in range(batch)])
        first_pitch, n_items = 0, batch
    else:
        if args.scaling == "weak":
            first_pitch = rank * pitches
        else:  # strong: the config's pitches split across ranks
            per = math.ceil(pitches / world)
            first_pitch = rank * per
            pitches = max(0, min(per, cfg["n_pitches"] - first_pitch))
        v0, nv = plan.scan_views(first_pitch, pitches)
        host_in = synth.project(cfg, rank_phantom(cfg, first_pitch - (first_pitch % cfg["n_pitches"])), v0, nv)
        n_items = pitches
    dev_in = torch.from_numpy(host_in).to(dev)
    vol_shape = (n_items * cfg["nz"], cfg["ny"], cfg["nx"]) if not batch else (batch, cfg["nz"], cfg["ny"], cfg["nx"])
    out = torch.empty(vol_shape, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        if batch:
            plan.reconstruct_batch(dev_in, out=out, stream=stream)
        else:
            plan.reconstruct(dev_in, v0, first_pitch, pitches, out=out, stream=stream)

    gather_buf = None
    if args.gather and world > 1:
        gather_buf = [torch.empty_like(out) for _ in range(world)] if rank == 0 else None

    def maybe_gather():
        if args.gather and world > 1:
            dist.gather(out, gather_buf, dst=0)

    for _ in range(args.warmup):
        step(); maybe_gather()
    torch.cuda.synchronize()
    plan.profile_read(reset=True)
    plan.profile_enable(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(); maybe_gather()
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    stats = plan.profile_read(reset=True)
    plan.profile_enable(False)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        if world > 1:
            dist.barrier()
    ms_step = ms / args.steps

    # ---- K5 in isolation: the same step with one backprojection launch over all of the rank's
    # pitches after all filtering (KATS_PIPELINE=0, the default), so no other kernel shares the GPU
    # with it (differs from the timed region only when KATS_PIPELINE=1 is set) ----
    iso = None
    if not batch:
        old_env = os.environ.get("KATS_PIPELINE")
        os.environ["KATS_PIPELINE"] = "0"
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
        if old_env is None:
            del os.environ["KATS_PIPELINE"]
        else:
            os.environ["KATS_PIPELINE"] = old_env
        k = "K5_backproject"
        iso = {"k5_ms_per_launch": st_iso["ms"][k] / max(1, st_iso["launches"][k]),
               "launches": st_iso["launches"][k] // n_iso}

    # ---- e2e: host (pinned) in -> host out through katsevich_reconstruct_host ----
    e2e = None
    if not batch:
        pin_in = torch.from_numpy(host_in).pin_memory()
        pin_out = torch.empty(vol_shape, dtype=torch.float32).pin_memory()
        for _ in range(2):
            plan.reconstruct_host(pin_in, v0, first_pitch, pitches, out_host=pin_out, stream=stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t1 = time.perf_counter()
        ne = max(3, min(args.steps, 10))
        for _ in range(ne):
            plan.reconstruct_host(pin_in, v0, first_pitch, pitches, out_host=pin_out, stream=stream)
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

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    U_pitch = count_updates(plan)
    U_rank = U_pitch * n_items
    U_all = U_rank * world
    vols_all = (n_items * world) / (cfg["n_pitches"] if not batch else batch)
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
    smem_peak = smem_peak_gbs(peaks.get("sm_max_mhz", 1965.0))
    achieved_smem = U_rank * bp_smem_bytes_per_update() / (k5_busy * 1e-3) / 1e9
    bp_kernel = plan.bp_kernel()
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
                   "pitches_per_rank": n_items, "parallelism": f"pitch-sharded x{world}",
                   "l2": "inputs larger than L2 (scan %.0f MB, filtered views %.0f MB > 126 MB L2)" % (
                       host_in.nbytes / 1e6, host_in.nbytes / 1e6)},
        "volumes_per_s": vols_all / (ms_step * 1e-3),
        "updates_per_step": U_all,
        "gpu_launches": stats["total_launches"],
        "stage_busy_share_of_step": share,
        "filter_stages": filter_stage_rooflines(plan, cfg, stats, args.steps, n_filtered_views(plan, cfg, n_items, batch),
                                                peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])),
        "paper_context": PAPER_CONTEXT,
        "precompute_s": t_pre,
        "roofline": {"bound": "smem", "kernel": bp_kernel, "achieved": achieved_smem, "peak": smem_peak,
                     "unit": "GB/s", "frac": achieved_smem / smem_peak,
                     "traffic": ncu_traffic(cfg["name"]),
                     "bytes_per_update": bp_smem_bytes_per_update(),
                     "k5_busy_ms_per_step": k5_busy, "k5_launches_per_step": k5_launches_per_step,
                     "k5_ms_per_launch": k5_ms_launch, "k5_updates_per_s": U_rank / (k5_busy * 1e-3),
                     "peak_source": f"148 SMs x 128 B/clk shared-memory pipe x {peaks.get('sm_max_mhz', 1965.0)} MHz "
                                    f"({src} sm_max); DESIGN.md §5",
                     "secondary_hbm": None if not ncu_traffic(cfg["name"]) else {
                         "achieved": ncu_traffic(cfg["name"]) / (iso["k5_ms_per_launch"] * 1e-3) / 1e9
                         if iso else None,
                         "peak": peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]), "unit": "GB/s",
                         "note": "ncu DRAM bytes of one 8-pitch K5 launch / its isolated time: far from bound"},
                     "secondary_alu": {"achieved": achieved_tflops, "peak": fp32_peak, "unit": "TFLOP/s",
                                       "frac": achieved_tflops / fp32_peak,
                                       "flops_per_update": bp_flops_per_update()},
                     "note": "achieved = 16 B x updates per step / K5 busy time per step in the timed "
                             "region (per-pitch K5 launches overlap each other and the filter there, so "
                             "this is a lower bound); isolated = one K5 launch for all pitches, alone",
                     "isolated": None if iso is None else {
                         "k5_ms_per_launch": iso["k5_ms_per_launch"],
                         "achieved": U_rank * bp_smem_bytes_per_update() / (iso["k5_ms_per_launch"] * 1e-3) / 1e9,
                         "frac": U_rank * bp_smem_bytes_per_update() / (iso["k5_ms_per_launch"] * 1e-3) / 1e9 / smem_peak}},
        "clocks": clk,
    }
    if dg:
        line["datagen"] = dg
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


# --- CPU oracle timing (bounded sample, extrapolated) -----------------------
def _oracle_sample(cfg, seed=0, n_b=32768):
    """Time the oracle on a bounded sample of one pitch of `cfg`:
    (a) steps 1-6 on 132 views minus the separately timed rebin-map setup
    the oracle runs in each call, (b) step 7 on n_b
    uniformly sampled voxels of the pitch (random filtered data).  The pitch's
    update count and slab length are estimated from the same sample."""
    from oracle import oracle
    from synth import synth
    rng = np.random.default_rng(seed)
    t0 = time.perf_counter()
    oracle.rebin_tables(cfg)                      # the oracle's per-call setup inside filter_views
    t_setup = time.perf_counter() - t0
    n_f = 132
    raw = synth.random_array((n_f + 2, cfg["n_rows"], cfg["n_cols"]), seed)
    t0 = time.perf_counter()
    oracle.filter_views(cfg, raw, 0, 1, n_f)
    t_f = max(1e-12, (time.perf_counter() - t0 - t_setup) / n_f)
    idx = np.stack([rng.integers(0, cfg["nx"], n_b), rng.integers(0, cfg["ny"], n_b),
                    rng.integers(0, cfg["nz"], n_b)], 1)
    kf, kl, _, _ = oracle.bp_weights_voxels(cfg, 0, idx)
    m = kl >= kf
    k_lo, k_hi = int(kf[m].min()), int(kl[m].max())
    u = np.where(m, kl - kf + 1, 0)
    gF = rng.standard_normal((k_hi - k_lo + 1, cfg["n_rows"], cfg["n_cols"]))
    t0 = time.perf_counter()
    oracle.backproject_voxels(cfg, 0, gF, k_lo, idx)
    t_b = time.perf_counter() - t0
    u_s = int(u.sum())
    t_u = t_b / max(1, u_s)
    n_vox = cfg["nx"] * cfg["ny"] * cfg["nz"]
    return dict(t_f=t_f, t_setup=t_setup, t_u=t_u, U_pitch=int(u.mean() * n_vox), nbp=k_hi - k_lo + 1,
                sample=f"steps 1-6 on {n_f} views and step 7 on {n_b} uniformly sampled voxels ({u_s} updates) of pitch 0")


def _extrapolate(cfg, s):
    n_p = cfg["n_pitches"] if not cfg.get("batch") else cfg["batch"]
    # the oracle filters each pitch's slab (no filter-once) and backprojects every voxel
    t_total = s["t_setup"] + n_p * (s["nbp"] * s["t_f"] + s["U_pitch"] * s["t_u"])
    return n_p * s["U_pitch"] / t_total, t_total, n_p


def cpu_baseline(cfg):
    s = _oracle_sample(cfg)
    value, t_total, n_p = _extrapolate(cfg, s)
    return {"value": value, "unit": "updates/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": s["sample"] + f"; extrapolated to {n_p} pitches x ({s['nbp']} views + {s['U_pitch']:.4g} updates)",
            "seconds_per_view_filter": s["t_f"], "seconds_per_update": s["t_u"],
            "extrapolated_seconds": t_total}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = workload(args.config)
    samples = []
    for i in range(args.warmup + args.steps):
        s = _oracle_sample(cfg, seed=i, n_b=8192)
        if i >= args.warmup:
            samples.append(s)
    s = dict(samples[0])
    for key in ("t_f", "t_setup", "t_u"):
        s[key] = float(np.median([x[key] for x in samples]))
    value, t_total, n_p = _extrapolate(cfg, s)
    line = {"impl": "reference", "metric": "voxel-view updates/s", "value": value, "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_total * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded random arrays of the workload's shapes)",
            "config": {"workload": f"{cfg['name']}: {cfg['desc']}"},
            "cpu_baseline": {"value": value, "unit": "updates/s", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": "per step: " + s["sample"] + "; median over steps, extrapolated"},
            "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--gather", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-adjoint", action="store_true", help="skip the adjoint (NEXT-1) measurement")
    ap.add_argument("--no-datagen", action="store_true", help="skip the data-generation (NEXT-3) measurement")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
