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


def _adj_worker(rank, world, port, cfg_name, ret):
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from synth import configs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = configs.get(cfg_name)
    s0, sn = cfg["scan_v0"], cfg["scan_nv"]
    rng = np.random.default_rng(12)
    y = rng.standard_normal((cfg["n_pitches"] * cfg["nz"], cfg["ny"], cfg["nx"]))   # d loss / d volume
    shards = kd.pitch_shards(cfg["n_pitches"], world)
    pv = lambda k: oracle.pitch_slab(cfg, k)
    ranges = [kd.shard_views(pv, s) for s in shards]
    me = shards[rank]
    v0, nv = ranges[rank]
    ylocal = y[me.first_pitch * cfg["nz"]:(me.first_pitch + me.n_pitches) * cfg["nz"]]
    # this rank's part of the layer's adjoint over its own views (the GPU would run katsevich_adjoint)
    g = torch.from_numpy(oracle.adjoint(cfg, ylocal, me.first_pitch, me.n_pitches, v0, nv))
    kd.reduce_view_halos(g, ranges)
    ref = oracle.adjoint(cfg, y, 0, cfg["n_pitches"], s0, sn)[v0 - s0:v0 - s0 + nv]
    ret[rank] = float(np.abs(g.numpy() - ref).max() / np.abs(ref).max())
    dist.destroy_process_group()


def test_sharded_adjoint_with_halo_reduction_equals_single_process():
    """Training a pitch-sharded layer: the per-rank adjoints summed over the
    overlapping view halos equal the single-process adjoint on every rank's range."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_adj_worker, args=(world, port, "T2", ret), nprocs=world, join=True)
    assert set(ret.keys()) == {0, 1}
    for r in range(world):
        assert ret[r] <= 1e-12, ret[r]


def test_view_range_precondition():
    kd.check_view_ranges([(0, 10), (6, 10), (14, 10)])            # neighbours overlap: fine
    with pytest.raises(ValueError):
        kd.check_view_ranges([(0, 10), (5, 10), (8, 10)])          # ranks 0 and 2 overlap
    with pytest.raises(ValueError):
        kd.check_view_ranges([(10, 5), (0, 5)])                     # not increasing
