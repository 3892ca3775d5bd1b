"""Multi-GPU partitioning of the remesh path: one process per GPU.

* Batch (C5): independent meshes, LPT-assigned to ranks by face count; no collective on the
  data path (only the final stats gather).
* Large grid (C4): the SDF lattice split into z-slabs of lattice planes; every rank computes
  its slab on its GPU, exchanges HALO=2 planes with each neighbour (NCCL send/recv over
  NVLink), runs DMC on its own cell layers (slab-local, pamopt_cu_dmc_extract_slab), and the
  slab meshes are gathered on rank 0 after an all-gather of their counts; the concatenation is
  bit-identical to the whole-grid extract.  Simplification stays single-GPU per mesh.
  (exchange_halo_and_gather keeps the older whole-lattice gather for tests/diagnostics.)

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


# ------------------------------------------------------------------- slab-local DMC (C4)
HALO = 2  # planes per side: a cell needs its top plane, the lending layer below, and the C16/C19
#           neighbour-case probe one layer further (dual_mc.cu k_patch_count)


def own_cell_layers(R: int, world: int, rank: int):
    """Cell layers [z0, z1) whose corner-0 quads this rank emits (its plane range, minus plane R)."""
    z0, z1 = slab_ranges(R, world)[rank]
    return z0, min(z1, R)


def resident_planes(R: int, world: int, rank: int):
    """Lattice planes a rank must hold for slab-local DMC: [z0 - HALO, z1 + HALO) clipped."""
    z0, z1 = slab_ranges(R, world)[rank]
    return max(z0 - HALO, 0), min(z1 + HALO, R + 1)


def exchange_halo2(slab, R: int, rank: int, world: int, dist, group=None):
    """slab: [z1-z0, R+1, R+1] (this rank's planes).  Returns the resident planes
    (resident_planes(R, world, rank)): HALO planes from each neighbour over P2P send/recv."""
    import torch

    assert slab.shape[0] >= HALO or world == 1, "each rank needs at least HALO planes"
    ops, lo, hi = [], None, None
    if rank > 0:
        lo = torch.empty((HALO,) + tuple(slab.shape[1:]), dtype=slab.dtype, device=slab.device)
        ops.append(dist.P2POp(dist.isend, slab[:HALO].contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, lo, rank - 1, group))
    if rank < world - 1:
        hi = torch.empty((HALO,) + tuple(slab.shape[1:]), dtype=slab.dtype, device=slab.device)
        ops.append(dist.P2POp(dist.isend, slab[-HALO:].contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, hi, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    parts = [x for x in (lo, slab, hi) if x is not None]
    return parts[0] if len(parts) == 1 else torch.cat(parts, 0)


def slab_offsets(counts):
    """counts[r] = (nvp_own, n_extra, nf) per rank ->
    per-rank (patch_base, extra_base, face_base) and totals (NVP, NEX, NF).  The assembled mesh is
    [every slab's patch vertices (z order), every slab's 4-split vertices], faces in z order —
    the whole-grid extract's P11 order."""
    counts = [tuple(int(x) for x in c) for c in counts]
    nvp = sum(c[0] for c in counts)
    out, p, e, fo = [], 0, 0, 0
    for c in counts:
        out.append((p, nvp + e, fo))
        p += c[0]
        e += c[1]
        fo += c[2]
    return out, (nvp, e, fo)


def distributed_dmc(piece, R: int, rank: int, world: int, dist, group=None, device=None):
    """Assembles slab-local extracts on rank 0.  piece: this rank's extract, with attributes
    nvp_own, n_extra, nf, rebase(patch_base, nvp_own, extra_base) and tensors() -> (V [nv,3] f64,
    F [nf,3] i32) after rebase.  Counts are all-gathered; then rank 0 receives every slab's
    patch vertices, split vertices and faces straight into place.  Returns (V, F) on rank 0,
    None elsewhere."""
    import torch

    mine = torch.tensor([piece.nvp_own, piece.n_extra, piece.nf], dtype=torch.int64, device=device)
    if world > 1:
        allc = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allc, mine, group=group)
        counts = [c.tolist() for c in allc]
    else:
        counts = [mine.tolist()]
    offs, (nvp, nex, nf) = slab_offsets(counts)
    pb, eb, fb = offs[rank]
    piece.rebase(pb, piece.nvp_own, eb)
    V, F = piece.tensors()
    if rank != 0:
        ops = []
        if piece.nvp_own:
            ops.append(dist.P2POp(dist.isend, V[:piece.nvp_own].contiguous(), 0, group))
        if piece.n_extra:
            ops.append(dist.P2POp(dist.isend, V[piece.nvp_own:].contiguous(), 0, group))
        if piece.nf:
            ops.append(dist.P2POp(dist.isend, F.contiguous(), 0, group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return None
    Vt = torch.empty((nvp + nex, 3), dtype=V.dtype, device=V.device)
    Ft = torch.empty((nf, 3), dtype=F.dtype, device=F.device)
    Vt[pb:pb + piece.nvp_own] = V[:piece.nvp_own]
    Vt[eb:eb + piece.n_extra] = V[piece.nvp_own:]
    Ft[fb:fb + piece.nf] = F
    ops = []
    for r in range(1, world):
        c = counts[r]
        p, e, f0 = offs[r]
        if c[0]:
            ops.append(dist.P2POp(dist.irecv, Vt[p:p + c[0]], r, group))
        if c[1]:
            ops.append(dist.P2POp(dist.irecv, Vt[e:e + c[1]], r, group))
        if c[2]:
            ops.append(dist.P2POp(dist.irecv, Ft[f0:f0 + c[2]], r, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return Vt, Ft


class GpuSlabPiece:
    """distributed_dmc piece backed by the CUDA slab extract (pamopt_cu_dmc_extract_slab)."""

    def __init__(self, resident, R: int, pz0: int, own_z0: int, own_z1: int, ctx, beta: float | None = None):
        import torch

        from . import api

        torch.cuda.current_stream().synchronize()  # resident planes were written on torch's stream
        g = api.DeviceGrid.slab_from_device(resident.data_ptr(), R, pz0, pz0 + resident.shape[0], ctx)
        try:
            self.mesh, self.nvp_own, self.n_extra = api.extract_slab(
                g, own_z0, own_z1, api.DEFAULT_BETA if beta is None else beta)
        finally:
            g.free()
        self.nf = self.mesh.size()[1]
        self.device = resident.device

    def rebase(self, patch_base, nvp_own, extra_base):
        self.mesh.rebase(patch_base, nvp_own, extra_base)

    def tensors(self):
        import torch

        nv, nf = self.mesh.size()
        V = torch.empty((nv, 3), dtype=torch.float64, device=self.device)
        F = torch.empty((nf, 3), dtype=torch.int32, device=self.device)
        self.mesh.copy_to_device(V.data_ptr() if nv else None, F.data_ptr() if nf else None)
        return V, F

    def free(self):
        self.mesh.free()


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


__all__ = ["slab_ranges", "exchange_halo_and_gather", "distributed_sdf", "gpu_slab_fn", "own_cell_layers",
           "resident_planes", "exchange_halo2", "slab_offsets", "distributed_dmc", "GpuSlabPiece", "lpt_assign",
           "run_batch", "makespan"]
_ = np
