"""Multi-process (gloo, world_size 2 and 3) tests of the host-side partitioning: z-slab halo
exchange + gather (the C4 path) and the LPT batch distribution (the C5 path).  The slab
contents come from the oracle so the assembled lattice can be compared bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_05595_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, R, full, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.from_numpy(full.reshape(R + 1, R + 1, R + 1))
        halo, got = D.distributed_sdf(lambda z0, z1: g[z0:z1].clone(), R, rank, world, dist)
        z0, z1 = D.slab_ranges(R, world)[rank]
        ok_halo = halo is None if rank == world - 1 else torch.equal(halo, g[z1])
        ok_full = True if rank != 0 else torch.equal(got, g)
        res = D.run_batch([(None, np.zeros((n, 3))) for n in (50, 10, 40, 20, 30)], rank, world,
                          lambda i, m: len(m[1]) * 2, dist)
        q.put((rank, ok_halo, ok_full, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_halo_gather_and_batch(oracle, world):
    from paper_2509_05595_b200 import fixtures as FX
    v, f = FX.icosphere(2)
    R = 16
    v, _ = FX.normalize_unit_cube(v, 6.0 / R)
    _, sdf = oracle.compute_udf_sdf(v, f, R)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, R, sdf, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_halo, ok_full, res in out:
        assert ok_halo and ok_full, rank
        assert res == [(0, 100), (1, 20), (2, 80), (3, 40), (4, 60)]


def test_slab_ranges_cover_lattice():
    for R in (8, 64, 1024):
        for w in (1, 2, 3, 4, 8):
            r = D.slab_ranges(R, w)
            assert r[0][0] == 0 and r[-1][1] == R + 1
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1


def test_lpt_assign_deterministic_and_balanced():
    from paper_2509_05595_b200 import fixtures as FX
    sizes = (np.exp(np.log(5e4) + (np.log(2e6) - np.log(5e4)) * FX.Rng(5).uniform(64))).astype(int)
    for w in (1, 2, 4, 8):
        a = D.lpt_assign(sizes, w)
        assert sorted(i for part in a for i in part) == list(range(64))
        assert a == D.lpt_assign(sizes, w)
        assert D.makespan(sizes, w) < 1.25


class _OraclePiece:
    """distributed_dmc piece backed by the oracle's slab restatement (CPU tensors, gloo)."""

    def __init__(self, oracle, resident, R, pz0, oz0, oz1):
        d = oracle.dmc_extract_slab(resident.numpy(), R, pz0, oz0, oz1)
        self.V, self.F = d["vertices"], d["faces"]
        self.nvp_own, self.n_extra, self.nf = d["nvp_own"], d["n_extra"], len(d["faces"])

    def rebase(self, pb, nvp, eb):
        F = self.F.astype(np.int64)
        self.F = np.where(F < nvp, pb + F, eb + (F - nvp)).astype(np.int32)

    def tensors(self):
        return torch.from_numpy(self.V), torch.from_numpy(self.F)


def _dmc_worker(rank, world, port, R, full, q):
    import sys
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import pyoracle as oracle
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.from_numpy(full.reshape(R + 1, R + 1, R + 1))
        z0, z1 = D.slab_ranges(R, world)[rank]
        res = D.exchange_halo2(g[z0:z1].clone(), R, rank, world, dist)
        pz0, pz1 = D.resident_planes(R, world, rank)
        ok_res = torch.equal(res, g[pz0:pz1])
        oz0, oz1 = D.own_cell_layers(R, world, rank)
        out = D.distributed_dmc(_OraclePiece(oracle, res, R, pz0, oz0, oz1), R, rank, world, dist)
        got = None if out is None else (out[0].numpy().copy(), out[1].numpy().copy())
        q.put((rank, ok_res, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_local_dmc_gather(oracle, world):
    """C4 data path on gloo: HALO=2 plane exchange, slab-local DMC (oracle), count all-gather,
    rebase, P2P gather on rank 0 -> bit-identical to the whole-grid extract."""
    from paper_2509_05595_b200 import fixtures as FX
    v, f = FX.icosphere(3)
    R = 24
    v, _ = FX.normalize_unit_cube(v, 6.0 / R)
    _, sdf = oracle.compute_udf_sdf(v, f, R)
    full = oracle.dmc_extract(sdf, R)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dmc_worker, args=(r, world, port, R, sdf, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_res, got in out:
        assert ok_res, rank
        if rank == 0:
            V, F = got
            assert np.array_equal(F, full["faces"])
            assert np.array_equal(V.view(np.uint64), full["vertices"].view(np.uint64))
        else:
            assert got is None
