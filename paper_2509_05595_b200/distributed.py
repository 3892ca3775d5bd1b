"""Multi-GPU partitioning of the remesh path: one process per GPU.

* Batch (C5): independent meshes, LPT-assigned to ranks by face count; no collective on the
  data path (only the final stats gather).
* Large grid (C4): the SDF lattice split into z-slabs of lattice planes; every rank computes
  its slab on its GPU, then one halo plane is exchanged with each neighbour (NCCL send/recv
  over NVLink) and the slabs are gathered on rank 0, which runs DMC (and QEM) — simplification
  stays single-GPU per mesh.

The exchange helpers take a torch.distributed process group, so the same code runs on NCCL
(GPU tensors) and on gloo (CPU tensors, tests/test_distributed.py).
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np


def slab_ranges(R: int, world: int):
    """Balanced split of the R+1 lattice planes: [(z0, z1)) per rank, contiguous, ordered."""
    n = R + 1
    base, extra = divmod(n, world)
    out, z = [], 0
    for r in range(world):
        c = base + (1 if r < extra else 0)
        out.append((z, z + c))
        z += c
    return out


def exchange_halo_and_gather(slab, R: int, rank: int, world: int, dist, group=None):
    """slab: tensor [planes, R+1, R+1] of this rank's planes.  Returns (halo, full):
    halo = the first plane of rank+1 (the top cell layer's missing corners; None on the last
    rank); full = the concatenated lattice on rank 0 (None elsewhere)."""
    import torch

    n1 = R + 1
    ranges = slab_ranges(R, world)
    halo = None
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, slab[0].contiguous(), rank - 1, group))
    if rank < world - 1:
        halo = torch.empty((n1, n1), dtype=slab.dtype, device=slab.device)
        ops.append(dist.P2POp(dist.irecv, halo, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    full = None
    if rank == 0:
        full = torch.empty((n1, n1, n1), dtype=slab.dtype, device=slab.device)
        z0, z1 = ranges[0]
        full[z0:z1] = slab
        ops = [dist.P2POp(dist.irecv, full[ranges[r][0]:ranges[r][1]], r, group) for r in range(1, world)]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
    else:
        for req in dist.batch_isend_irecv([dist.P2POp(dist.isend, slab.contiguous(), 0, group)]):
            req.wait()
    return halo, full


def distributed_sdf(compute_slab: Callable[[int, int], object], R: int, rank: int, world: int, dist, group=None):
    """compute_slab(z0, z1) -> tensor [z1-z0, R+1, R+1] on this rank's device.  Returns
    (halo, full) as exchange_halo_and_gather."""
    z0, z1 = slab_ranges(R, world)[rank]
    slab = compute_slab(z0, z1)
    return exchange_halo_and_gather(slab, R, rank, world, dist, group)


def gpu_slab_fn(mesh, R: int, eps: float | None = None):
    """compute_slab for the CUDA path: pamopt_cu_compute_sdf_slab into a torch CUDA tensor."""
    import torch

    from . import api

    def fn(z0: int, z1: int):
        g = api.compute_sdf_slab(mesh, R, z0, z1, eps)
        t = torch.empty((z1 - z0, R + 1, R + 1), dtype=torch.float32, device="cuda")
        g.copy_to_device(t.data_ptr())
        g.free()
        return t

    return fn


# ------------------------------------------------------------------------------ batch
def lpt_assign(sizes: Sequence[int], world: int):
    """Longest-processing-time-first: meshes sorted by size (desc, index tie-break) go to the
    currently least-loaded rank (lowest rank on ties).  Deterministic."""
    order = sorted(range(len(sizes)), key=lambda i: (-int(sizes[i]), i))
    load = [0] * world
    out = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += int(sizes[i])
    return out


def run_batch(meshes, rank: int, world: int, work: Callable, dist=None, group=None):
    """Runs work(i, mesh) for this rank's LPT share; gathers [(index, result)] on every rank
    (object all_gather: control metadata only, never mesh data)."""
    sizes = [len(m[1]) for m in meshes]
    mine = lpt_assign(sizes, world)[rank]
    local = [(i, work(i, meshes[i])) for i in mine]
    if dist is None or world == 1:
        return sorted(local)
    gathered = [None] * world
    dist.all_gather_object(gathered, local, group=group)
    return sorted(x for part in gathered for x in part)


def makespan(sizes: Sequence[int], world: int) -> float:
    """Load of the most loaded rank under lpt_assign, relative to a perfect split."""
    a = lpt_assign(sizes, world)
    loads = [sum(int(sizes[i]) for i in part) for part in a]
    return max(loads) / (sum(int(s) for s in sizes) / world)


__all__ = ["slab_ranges", "exchange_halo_and_gather", "distributed_sdf", "gpu_slab_fn", "lpt_assign",
           "run_batch", "makespan"]
_ = np
