"""Pitch-sharded multi-process reconstruction through libkatsevich: two
processes on cuda:0 each reconstruct their block of C4's 8 pitches through the C ABI, in
bench.py's sub-blocks, and send each finished sub-block to rank 0 (gloo moves CPU copies:
one GPU here, and kernels of different ranks never wait on one another).  The gathered
volume must equal the single-process 8-pitch reconstruction bit for bit (each filtered view
depends only on raw views v-1..v+1 and every pitch shares the same periodic tables)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests.conftest import cuda_ok

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ret):
    import torch
    import torch.distributed as dist

    import paper_2201_02309_b200 as k
    from paper_2201_02309_b200 import dist as kd
    from synth import configs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = configs.get("C4")
    nz, npit = cfg["nz"], cfg["n_pitches"]
    plan = k.Plan(cfg, device=0)
    plan.precompute()
    shards = kd.pitch_shards(npit, world)
    me = shards[rank]
    g = kd.SlabGather(shards, nz, parts=2)
    v0, nv = plan.scan_views(me.first_pitch, me.n_pitches)
    sino = plan.project_ellipsoids(cfg["phantom"], v0, nv)       # GPU projector: identical per ray
    shape = (npit * nz, cfg["ny"], cfg["nx"])
    full = torch.full(shape, float("nan")) if rank == 0 else None
    local = torch.empty((me.n_pitches * nz, cfg["ny"], cfg["nx"]))
    works = g.post_recvs(full) if rank == 0 else []
    for i, b in enumerate(g.blocks[rank]):
        vol = plan.reconstruct(sino, v0, b.first_pitch, b.n_pitches).cpu()
        if rank == 0:
            full[g.rows(b)] = vol
        else:
            local[g.local_rows(rank, i)] = vol
            works.append(g.send(rank, i, local[g.local_rows(rank, i)]))
    for w in works:
        w.wait()
    if rank == 0:
        s0, sn = plan.scan_views(0, npit)
        ref = plan.reconstruct(plan.project_ellipsoids(cfg["phantom"], s0, sn), s0, 0, npit).cpu()
        ret["equal"] = bool(torch.equal(full, ref))
        ret["nonzero"] = float(ref.abs().max())
    dist.destroy_process_group()


def test_two_process_pitch_sharded_c4_equals_single_process():
    if not cuda_ok():
        pytest.skip("no CUDA device")
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.start_processes(_worker, args=(2, _free_port(), ret), nprocs=2, start_method="spawn")
    assert ret["nonzero"] > 0.5
    assert ret["equal"], "gathered sharded C4 volume differs from the single-process volume"


def test_reconstruct_grouped_equals_reconstruct_and_marks_groups():
    """katsevich_reconstruct_grouped (bench.py's overlapped gather): the same volume bit for bit
    as katsevich_reconstruct, and every group's event completes."""
    if not cuda_ok():
        pytest.skip("no CUDA device")
    import torch
    import paper_2201_02309_b200 as k
    from synth import configs
    cfg = configs.get("T3")
    p = k.Plan(cfg, device=0)
    p.precompute()
    s0, sn = p.scan_views(0, 3)
    sino = p.project_ellipsoids(cfg["phantom"], s0, sn)
    ref = p.reconstruct(sino, s0, 0, 3)
    evs = [torch.cuda.Event() for _ in range(3)]
    for e in evs:
        e.record()
    got = p.reconstruct_grouped(sino, s0, 0, 3, 3, group_events=evs)
    torch.cuda.synchronize()
    assert all(e.query() for e in evs)
    assert torch.equal(got, ref)
    got2 = p.reconstruct_grouped(sino, s0, 0, 3, 2)
    assert torch.equal(got2, ref)
    with pytest.raises(Exception):
        p.reconstruct_grouped(sino, s0, 0, 3, 4)
