"""GPU slab-local DMC (pamopt_cu_dmc_extract_slab): every slab piece equals the
oracle's slab restatement bit for bit, and the assembled pieces equal the whole-grid GPU extract."""
import numpy as np
import pytest

from paper_2509_05595_b200 import distributed as D
from paper_2509_05595_b200 import fixtures as FX

from tests.test_dmc_slab import assemble, grids, random_sdf

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("world", [2, 3, 5])
def test_gpu_slab_pieces_match_oracle_and_assemble(api, oracle, world):
    cases = list(grids(oracle))
    v, f, R, _ = FX.make_config("c1")
    _, sdf = oracle.compute_udf_sdf(v, f, R)
    cases.append(("c1", sdf, R))
    cases.append(("random64", random_sdf(64, 9), 64))
    for name, sdf, R in cases:
        g = sdf.reshape(R + 1, R + 1, R + 1)
        pieces = []
        for r in range(world):
            pz0, pz1 = D.resident_planes(R, world, r)
            oz0, oz1 = D.own_cell_layers(R, world, r)
            grid = api.DeviceGrid.slab_upload(g[pz0:pz1], R, pz0)
            m, nvp, nex = api.extract_slab(grid, oz0, oz1)
            gv, gf = m.download()
            m.free()
            grid.free()
            ref = oracle.dmc_extract_slab(g[pz0:pz1], R, pz0, oz0, oz1)
            assert (nvp, nex) == (ref["nvp_own"], ref["n_extra"]), (name, r)
            assert np.array_equal(gf, ref["faces"]), (name, r)
            assert np.array_equal(_bits(gv), _bits(ref["vertices"])), (name, r)
            pieces.append((gv, gf, nvp, nex))
        V, F = assemble(pieces)
        whole = api.extract(api.DeviceGrid.upload(sdf, R))
        wv, wf = whole.download()
        assert np.array_equal(F, wf) and np.array_equal(_bits(V), _bits(wv)), name


def test_gpu_distributed_dmc_single_rank(api, oracle):
    """The multi-GPU assembly code path (GpuSlabPiece + distributed_dmc) at world size 1."""
    import torch
    v, f, R, _ = FX.make_config("c1")
    _, sdf = oracle.compute_udf_sdf(v, f, R)
    ctx = api.default_context()
    t = torch.from_numpy(sdf.reshape(R + 1, R + 1, R + 1)).cuda()
    piece = D.GpuSlabPiece(t, R, 0, 0, R, ctx)
    V, F = D.distributed_dmc(piece, R, 0, 1, None, device=t.device)
    piece.free()
    full = oracle.dmc_extract(sdf, R)
    assert np.array_equal(F.cpu().numpy(), full["faces"])
    assert np.array_equal(_bits(V.cpu().numpy()), _bits(full["vertices"]))


def test_gpu_slab_errors(api):
    from paper_2509_05595_b200._lib import PamoptInvalidArgument
    R = 16
    s = random_sdf(R, 3).reshape(R + 1, R + 1, R + 1)
    grid = api.DeviceGrid.slab_upload(s[4:10], R, 4)
    with pytest.raises(PamoptInvalidArgument):
        api.extract_slab(grid, 5, 9)   # needs planes [3, 11)
    with pytest.raises(PamoptInvalidArgument):
        api.extract_slab(grid, 7, 6)   # empty own range
    m, _, _ = api.extract_slab(grid, 6, 8)
    m.free()


def test_extract_slab_nccl_world1_equals_whole_grid(api):
    """The C-ABI slab path over a real NCCL communicator (ncclCommInitAll on this one GPU): at
    world = 1 it must reproduce the whole-grid extract exactly (multi-rank exchange logic is the
    same code with neighbours; the Python twin is covered at world 2/3 with gloo)."""
    from paper_2509_05595_b200 import fixtures as FX
    v, f = FX.icosphere(4)
    R = 64
    v, _ = FX.normalize_unit_cube(v * (1.0 + 0.01 * FX.Rng(2).normal(len(v)))[:, None], 6.0 / R)
    whole_v, whole_f = api.extract(api.compute_sdf((v, f), R)).download()
    comms = api.nccl_comm_init_all([0])
    try:
        out, counts = api.extract_slab_nccl((v, f), R, 0, 1, comms[0])
        gv, gf = out.download()
    finally:
        api.nccl_comm_destroy(comms[0])
    assert np.array_equal(gf, whole_f) and np.array_equal(gv.view(np.uint64), whole_v.view(np.uint64))
    assert counts[2] == len(whole_f)
    out2, _ = api.extract_slab_nccl((v, f), R, 0, 1, None)  # world 1 needs no communicator
    assert np.array_equal(out2.download()[1], whole_f)
