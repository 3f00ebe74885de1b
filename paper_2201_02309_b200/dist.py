"""Multi-GPU pitch sharding (host logic; one process per GPU, torch.distributed).

Pitches are independent given their slab and share every periodic table
(PAPER.md l.174-185, l.246, l.265), so a long scan shards by pitch (z-slab):
rank r reconstructs a contiguous block of pitches from the views that block
needs (its pitches plus the PI-window overlap).  The only collective is the
optional gather of the volume slabs (NCCL over NVLink on B200; gloo in the
CPU tests).  Training through the layer (the adjoint, NEXT-1) has one real
exchange: neighbouring ranks' view ranges overlap by the PI-window halo, so
their sinogram adjoints must be summed there (reduce_view_halos).  Nothing
here computes the method: reconstruction and adjoint run in libkatsevich.so.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    first_pitch: int
    n_pitches: int


def pitch_shards(total_pitches: int, world: int, first_pitch: int = 0):
    """Contiguous, balanced split of pitches [first_pitch, first_pitch + total) over
    `world` ranks (the first total % world ranks get one extra pitch)."""
    if world < 1 or total_pitches < 0:
        raise ValueError("world >= 1 and total_pitches >= 0 required")
    base, extra = divmod(total_pitches, world)
    out, p = [], first_pitch
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append(Shard(r, p, n))
        p += n
    return out


def weak_shard(pitches_per_rank: int, rank: int) -> Shard:
    """Weak scaling: every rank owns the same number of pitches of a longer scan."""
    return Shard(rank, rank * pitches_per_rank, pitches_per_rank)


def shard_views(pitch_views, shard: Shard):
    """Views [v0, v0 + nv) shard needs, from `pitch_views(k) -> (first_view, n_views)`
    (e.g. Plan.pitch_views): union of its pitches' slabs (halo included)."""
    if shard.n_pitches == 0:
        return 0, 0
    f0, n0 = pitch_views(shard.first_pitch)
    f1, n1 = pitch_views(shard.first_pitch + shard.n_pitches - 1)
    return f0, f1 + n1 - f0


def slice_scan(scan, scan_first_view: int, v0: int, nv: int):
    """The rank's sub-range of a full scan array [views][rows][cols]."""
    a = v0 - scan_first_view
    if a < 0 or a + nv > scan.shape[0]:
        raise ValueError(f"scan views [{scan_first_view}, {scan_first_view + scan.shape[0]}) "
                         f"do not cover [{v0}, {v0 + nv})")
    return scan[a:a + nv]


def gather_volumes(local, shards, nz: int, dst: int = 0, group=None):
    """Gather per-rank volume slabs [n_pitches*nz][ny][nx] to rank `dst`.
    Unequal shards are padded to the largest for the collective and trimmed.
    Returns the stacked volume on `dst`, None elsewhere."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    assert len(shards) == world
    max_p = max(s.n_pitches for s in shards)
    ny, nx = local.shape[-2], local.shape[-1]
    buf = torch.zeros((max_p * nz, ny, nx), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    if rank == dst:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, parts, dst=dst, group=group)
        return torch.cat([parts[s.rank][: s.n_pitches * nz] for s in shards], dim=0)
    dist.gather(buf, None, dst=dst, group=group)
    return None


def sub_blocks(shard: Shard, parts: int):
    """Split a rank's pitch block into min(parts, n_pitches) contiguous sub-blocks, sub-block i =
    pitches [n i / parts, n (i + 1) / parts) of the block — the pitch groups of
    katsevich_reconstruct_grouped, and the unit of the overlapped gather (sub-block i travels while
    sub-block i+1 is backprojected)."""
    n = shard.n_pitches
    g = max(1, min(parts, n))
    return [Shard(shard.rank, shard.first_pitch + n * i // g, n * (i + 1) // g - n * i // g)
            for i in range(g)] if n else []


class SlabGather:
    """Point-to-point gather of every rank's volume slabs into rank `dst`'s full volume
    (NCCL carries only the gather of the pitch slabs), per sub-block so that
    the transfer of a finished sub-block overlaps the reconstruction of the next one.

    Every transfer is one isend/irecv pair between the owner and `dst` (the same pattern on both
    sides, so NCCL uses the same two-rank communicator for the pair); `dst` writes its own
    sub-blocks directly into its slice of `full` and receives the others there (no staging copy).
    Usage per step:  works = g.post_recvs(full) on dst (its own sub-block i goes straight into
    full[g.rows(g.blocks[dst][i])]); on the others, after sub-block i is reconstructed into
    local[g.local_rows(rank, i)]:  works.append(g.send(rank, i, that slice)); finally
    for w in works: w.wait()."""

    def __init__(self, shards, nz: int, parts: int = 2, dst: int = 0, group=None):
        self.shards = list(shards)
        self.nz = nz
        self.dst = dst
        self.group = group
        self.base = self.shards[0].first_pitch
        self.blocks = [sub_blocks(s, parts) for s in self.shards]

    def rows(self, block: Shard):
        """Slice of the full (gathered) volume's slices holding `block`."""
        a = (block.first_pitch - self.base) * self.nz
        return slice(a, a + block.n_pitches * self.nz)

    def local_rows(self, rank: int, i: int):
        """Slice of rank `rank`'s own volume [n_pitches*nz] holding its sub-block i."""
        b = self.blocks[rank][i]
        a = (b.first_pitch - self.shards[rank].first_pitch) * self.nz
        return slice(a, a + b.n_pitches * self.nz)

    def post_recvs(self, full):
        import torch.distributed as dist
        works = []
        for r, blocks in enumerate(self.blocks):
            if r == self.dst:
                continue
            for b in blocks:
                works.append(dist.irecv(full[self.rows(b)], src=r, group=self.group))
        return works

    def send(self, rank: int, i: int, tensor):
        import torch.distributed as dist
        assert rank != self.dst
        return dist.isend(tensor, dst=self.dst, group=self.group)


def check_view_ranges(view_ranges):
    """reduce_view_halos' precondition: increasing starts, overlaps only between neighbours."""
    starts = [v for v, n in view_ranges if n]
    if starts != sorted(starts):
        raise ValueError("view ranges must be in increasing order of their first view")
    for a in range(len(view_ranges)):
        for b in range(a + 2, len(view_ranges)):
            va, na = view_ranges[a]
            vb, nb = view_ranges[b]
            if na and nb and vb < va + na:
                raise ValueError(f"ranks {a} and {b} are not neighbours but their view ranges overlap")


def reduce_view_halos(local, view_ranges, group=None):
    """Sum the overlapping parts of per-rank view arrays in place (owner computes).

    local        this rank's array [nv_r][rows][cols] for views [v0_r, v0_r + nv_r)
    view_ranges  [(v0_r, nv_r)] for every rank, increasing v0_r; only neighbouring
                 ranges may overlap (the PI-window halo of a pitch block).
    After the call every rank holds, over its whole range, the sum of all ranks'
    contributions — e.g. the sinogram gradient of a pitch-sharded reconstruction,
    whose per-rank adjoints overlap where the slabs do.  One batched point-to-point
    exchange with each neighbour (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    assert len(view_ranges) == world
    check_view_ranges(view_ranges)
    v0, nv = view_ranges[rank]

    def overlap(r):
        va, na = view_ranges[r]
        lo, hi = max(v0, va), min(v0 + nv, va + na)
        return (lo, hi) if na and nv and lo < hi else None

    ops, recv = [], []
    for nb in (rank - 1, rank + 1):
        if 0 <= nb < world:
            o = overlap(nb)
            if o is None:
                continue
            lo, hi = o
            send = local[lo - v0:hi - v0].contiguous()
            buf = torch.empty_like(send)
            ops.append(dist.P2POp(dist.isend, send, nb, group))
            ops.append(dist.P2POp(dist.irecv, buf, nb, group))
            recv.append((lo, hi, buf))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for lo, hi, buf in recv:
        local[lo - v0:hi - v0] += buf
    return local
