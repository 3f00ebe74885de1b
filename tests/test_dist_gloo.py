"""Multi-process pitch sharding on CPU (gloo, world size 2).

Each rank takes its pitch block and the scan views that block needs, reconstructs
them (the CPU oracle stands in for the GPU here — only the host-side sharding,
view slicing and gather are under test), and rank 0 checks that the gathered
volume equals the single-process reconstruction bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2201_02309_b200 import dist as kd


def test_pitch_shards_balanced_and_contiguous():
    s = kd.pitch_shards(8, 3)
    assert [x.n_pitches for x in s] == [3, 3, 2]
    assert [x.first_pitch for x in s] == [0, 3, 6]
    s = kd.pitch_shards(2, 4, first_pitch=5)
    assert [(x.first_pitch, x.n_pitches) for x in s] == [(5, 1), (6, 1), (7, 0), (7, 0)]
    w = kd.weak_shard(8, 3)
    assert (w.first_pitch, w.n_pitches) == (24, 8)


def test_shard_views_union():
    pv = lambda k: (k * 100 - 13, 150)                 # slab of pitch k
    assert kd.shard_views(pv, kd.Shard(0, 2, 3)) == (187, 350)
    assert kd.shard_views(pv, kd.Shard(0, 2, 0)) == (0, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_name, ret):
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from synth import configs, synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = configs.get(cfg_name)
    scan = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    shards = kd.pitch_shards(cfg["n_pitches"], world)
    me = shards[rank]
    pv = lambda k: oracle.pitch_slab(cfg, k)
    v0, nv = kd.shard_views(pv, me)
    local_scan = kd.slice_scan(scan, cfg["scan_v0"], v0, nv)
    vol = oracle.reconstruct(cfg, local_scan, v0, me.first_pitch, me.n_pitches) if me.n_pitches else \
        np.zeros((0, cfg["ny"], cfg["nx"]))
    full = kd.gather_volumes(torch.from_numpy(vol), shards, cfg["nz"])
    if rank == 0:
        ref = oracle.reconstruct(cfg, scan, cfg["scan_v0"], 0, cfg["n_pitches"])
        ret["equal"] = bool(np.array_equal(full.numpy(), ref))
        ret["shape"] = tuple(full.shape)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_reconstruction_equals_single_process(world):
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), "T3", ret), nprocs=world, start_method="spawn")
    assert ret["equal"], "gathered sharded volume differs from the single-process volume"
    assert ret["shape"][0] == 3 * 19
