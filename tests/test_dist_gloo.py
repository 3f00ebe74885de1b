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


def _slab_gather_worker(rank, world, port, cfg_name, parts, ret):
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from synth import configs, synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = configs.get(cfg_name)
    nz = cfg["nz"]
    scan = synth.project(cfg, cfg["phantom"], cfg["scan_v0"], cfg["scan_nv"])
    shards = kd.pitch_shards(cfg["n_pitches"], world)
    me = shards[rank]
    g = kd.SlabGather(shards, nz, parts=parts)
    shape = (cfg["n_pitches"] * nz, cfg["ny"], cfg["nx"])
    full = torch.full(shape, float("nan"), dtype=torch.float64) if rank == 0 else None
    local = None if rank == 0 else torch.empty((me.n_pitches * nz, cfg["ny"], cfg["nx"]), dtype=torch.float64)
    works = g.post_recvs(full) if rank == 0 else []
    pv = lambda k: oracle.pitch_slab(cfg, k)
    for i, b in enumerate(g.blocks[rank]):            # bench.py's step: sub-block by sub-block
        v0, nv = kd.shard_views(pv, b)
        vol = torch.from_numpy(oracle.reconstruct(cfg, kd.slice_scan(scan, cfg["scan_v0"], v0, nv), v0,
                                                  b.first_pitch, b.n_pitches))
        if rank == 0:
            full[g.rows(b)] = vol
        else:
            local[g.local_rows(rank, i)] = vol
            works.append(g.send(rank, i, local[g.local_rows(rank, i)]))
    for w in works:
        w.wait()
    if rank == 0:
        ref = oracle.reconstruct(cfg, scan, cfg["scan_v0"], 0, cfg["n_pitches"])
        ret["equal"] = bool(np.array_equal(full.numpy(), ref))
        ret["blocks"] = [[(b.first_pitch, b.n_pitches) for b in bl] for bl in g.blocks]
    dist.destroy_process_group()


def test_slab_gather_overlapped_sub_blocks_equal_single_process():
    """bench.py's multi-GPU step on CPU: rank r of 2 reconstructs its pitch block of T3 in
    sub-blocks, each sent to rank 0 (isend/irecv into its slice of the full volume) as soon as
    it is done; the gathered volume equals the single-process reconstruction bit for bit."""
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.start_processes(_slab_gather_worker, args=(2, _free_port(), "T3", 2, ret), nprocs=2, start_method="spawn")
    assert ret["blocks"] == [[(0, 1), (1, 1)], [(2, 1)]]
    assert ret["equal"], "gathered volume differs from the single-process volume"


def test_sub_blocks_and_rows():
    s = kd.pitch_shards(8, 2)
    g = kd.SlabGather(s, nz=64, parts=2)
    assert [[(b.first_pitch, b.n_pitches) for b in bl] for bl in g.blocks] == [[(0, 2), (2, 2)], [(4, 2), (6, 2)]]
    assert g.rows(g.blocks[1][1]) == slice(6 * 64, 8 * 64)
    assert g.local_rows(1, 1) == slice(2 * 64, 4 * 64)
    assert [len(b) for b in kd.SlabGather(kd.pitch_shards(8, 8), 64, parts=2).blocks] == [1] * 8
