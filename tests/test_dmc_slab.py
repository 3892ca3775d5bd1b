"""Slab-local DMC: every rank extracts its own cell layers from its resident
planes (own slab + HALO planes per side); rebasing the face indices and concatenating [patch
vertices of every slab, 4-split vertices of every slab, faces of every slab] must reproduce the
whole-grid extract bit for bit.  CPU side: the oracle's slab restatement, assembled with the same
host code the multi-GPU path uses (paper_2509_05595_b200.distributed)."""
import numpy as np
import pytest

from paper_2509_05595_b200 import distributed as D
from paper_2509_05595_b200 import fixtures as FX


def rebase_np(F, pb, nvp, eb):
    F = F.astype(np.int64)
    return np.where(F < nvp, pb + F, eb + (F - nvp)).astype(np.int32)


def assemble(pieces):
    """pieces: [(V, F, nvp_own, n_extra)] in rank order -> (V, F) of the whole mesh."""
    offs, (nvp, nex, nf) = D.slab_offsets([(p[2], p[3], len(p[1])) for p in pieces])
    V = np.empty((nvp + nex, 3))
    F = np.empty((nf, 3), np.int32)
    for (v, f, n, e), (pb, eb, fb) in zip(pieces, offs):
        V[pb:pb + n] = v[:n]
        V[eb:eb + e] = v[n:]
        F[fb:fb + len(f)] = rebase_np(f, pb, n, eb)
    return V, F


def random_sdf(R, seed):
    """Random signs everywhere: dense ambiguous faces and C16/C19 doubly-covered pairs."""
    rng = FX.Rng(seed)
    return (rng.uniform((R + 1) ** 3) * 2.0 - 1.0).astype(np.float32)


def slab_pieces(oracle, sdf, R, world):
    g = sdf.reshape(R + 1, R + 1, R + 1)
    out = []
    for r in range(world):
        pz0, pz1 = D.resident_planes(R, world, r)
        oz0, oz1 = D.own_cell_layers(R, world, r)
        d = oracle.dmc_extract_slab(g[pz0:pz1], R, pz0, oz0, oz1)
        out.append((d["vertices"], d["faces"], d["nvp_own"], d["n_extra"]))
    return out


def grids(oracle):
    v, f = FX.icosphere(3)
    R = 32
    v, _ = FX.normalize_unit_cube(v, 6.0 / R)
    _, sdf = oracle.compute_udf_sdf(v, f, R)
    yield "icosphere", sdf, R
    yield "random16", random_sdf(16, 7), 16
    yield "random32", random_sdf(32, 8), 32


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_oracle_slab_assembly_equals_whole_grid(oracle, world):
    for name, sdf, R in grids(oracle):
        full = oracle.dmc_extract(sdf, R)
        V, F = assemble(slab_pieces(oracle, sdf, R, world))
        assert np.array_equal(F, full["faces"]), name
        assert np.array_equal(V.view(np.uint64), full["vertices"].view(np.uint64)), name


def test_slab_layers_and_residency():
    for R in (16, 64, 1024):
        for w in (1, 2, 3, 8):
            own = [D.own_cell_layers(R, w, r) for r in range(w)]
            assert own[0][0] == 0 and own[-1][1] == R
            assert all(a[1] == b[0] for a, b in zip(own, own[1:]))
            for r in range(w):
                pz0, pz1 = D.resident_planes(R, w, r)
                assert pz0 == max(own[r][0] - D.HALO, 0) and pz1 >= min(own[r][1] + D.HALO, R + 1)
