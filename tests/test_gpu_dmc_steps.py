"""SPEC-granular dual_mc operations through the C-ABI, each against the oracle:
interpolate_patch_vertex, classify_voxels / build_patches / build_quads views, and
triangulate_quads on explicit quads (which recomposes extract exactly).  Plus SPEC acceptance
criterion #2 at its stated size: 100 random 32^3 grids -> manifold, intersection-free meshes
(SPEC.md:808), each bit-identical to the oracle's extraction."""
import numpy as np
import pytest

from paper_2509_05595_b200 import fixtures as FX

pytestmark = pytest.mark.gpu


def u64(a):
    return np.ascontiguousarray(a).view(np.uint64)


def test_interpolate_patch_vertex_spec_examples(api, oracle):
    p0 = np.array([[0.0, 0.0, 0.0]] * 3)
    p1 = np.array([[1.0, 0.0, 0.0]] * 3)
    out = api.interpolate_patch_vertex(p0, p1, [-0.5, 0.0, -0.4], [0.5, -1.0, 0.6], beta=5.0)
    assert out[0, 0] == 0.5  # f0 = -f1 -> midpoint
    assert abs(out[1, 0] - 1.0 / (1.0 + np.exp(2.5))) < 1e-15  # t = 0 -> 0.07586
    sharp = api.interpolate_patch_vertex(p0[:1], p1[:1], [-0.4], [0.6], beta=500.0)
    assert sharp[0, 0] < 1e-20  # beta -> inf: step at 1/2
    with pytest.raises(api._lib.PamoptInvalidArgument):
        api.interpolate_patch_vertex(p0[:1], p1[:1], [0.2], [0.5])


def test_interpolate_patch_vertex_matches_oracle(api, oracle):
    rng = np.random.default_rng(3)
    n = 4096
    p0 = rng.uniform(-1, 1, (n, 3))
    p1 = p0 + rng.uniform(-0.01, 0.01, (n, 3))
    f0 = rng.uniform(-1, 1, n).astype(np.float32)
    f1 = (-np.sign(f0) * rng.uniform(1e-6, 1, n)).astype(np.float32)
    f1[f0 < 0] = np.abs(f1[f0 < 0])
    got = api.interpolate_patch_vertex(p0, p1, f0, f1)
    t = -f0.astype(np.float64) / (f1.astype(np.float64) - f0.astype(np.float64))
    ts = np.array([oracle.sigmoid(x, 5.0) for x in t])
    ref = p0 + ts[:, None] * (p1 - p0)
    assert np.array_equal(u64(got), u64(ref))


@pytest.fixture(scope="module")
def sdf32(oracle):
    v, f, _, _ = FX.make_config("c1")
    v, _ = FX.normalize_unit_cube(v, 6.0 / 32)
    _, sdf = oracle.compute_udf_sdf(v, f, 32)
    return sdf


def test_dmc_stage_views_match_oracle(api, oracle, sdf32):
    R = 32
    d = oracle.dmc_extract(sdf32, R)
    g = api.DeviceGrid.upload(sdf32, R)
    s = api.dmc_stages(g)
    assert np.array_equal(s["cells"], d["cells"]) and np.array_equal(s["cases"], d["cases"])
    assert np.array_equal(s["flips"], d["flips"])
    assert np.array_equal(s["patch_first"], d["patch_first"])
    assert np.array_equal(u64(s["patch_vertices"]), u64(d["vertices"][: d["n_patch_vertices"]]))
    assert np.array_equal(s["quads"], d["quads"]) and np.array_equal(s["quad_edges"], d["quad_edges"])
    assert np.array_equal(s["quad_samples"].view(np.uint32), d["quad_samples"].view(np.uint32))
    assert np.array_equal(s["quad_split"], d["quad_split"])


def test_triangulate_quads_recomposes_extract(api, oracle, sdf32):
    R = 32
    g = api.DeviceGrid.upload(sdf32, R)
    s = api.dmc_stages(g)
    m = api.triangulate_quads(R, s["patch_vertices"], s["quads"], s["quad_edges"], s["quad_samples"])
    tv, tf = m.download()
    ev, ef = api.extract(g).download()
    assert np.array_equal(tf, ef) and np.array_equal(u64(tv), u64(ev))
    # per-quad triangle counts follow the split decision
    assert len(tf) == 2 * len(s["quads"]) + 2 * int((s["quad_split"] == 3).sum())


def test_classify_voxels_spec_examples(api):
    R = 8
    g = np.ones((R + 1) ** 3, np.float32)
    s = api.dmc_stages(api.DeviceGrid.upload(g, R))
    assert len(s["cells"]) == 0 and len(s["quads"]) == 0  # all-positive grid
    g = g.reshape(R + 1, R + 1, R + 1)
    g[4, 4, 4] = -1.0  # one negative sample: its 8 cells are active, one patch of 3 edges each
    s = api.dmc_stages(api.DeviceGrid.upload(g.ravel(), R))
    assert len(s["cells"]) == 8 and len(s["patch_vertices"]) == 8
    assert len(s["quads"]) == 6  # a closed quad polyhedron around the sample (V - E + F = 2)
    m = api.extract(api.DeviceGrid.upload(g.ravel(), R))
    t = api.analyze_topology(m)
    assert t["manifold"] and t["watertight"] and t["euler"] == 2


def test_random_grids_acceptance_100x32(api, oracle):
    """SPEC.md:808 acceptance #2: 100 random 32^3 grids (uniform in [-1, 1], boundary samples
    positive so the negative region is strictly interior) -> 0 self-intersecting
    outputs, 100% manifold and watertight; each GPU extraction equals the oracle's bit for bit."""
    R = 32
    for seed in range(100):
        g = np.random.default_rng(1000 + seed).uniform(-1, 1, (R + 1) ** 3).astype(np.float32)
        g3 = g.reshape(R + 1, R + 1, R + 1)
        for sl in (0, -1):
            g3[sl, :, :] = 1
            g3[:, sl, :] = 1
            g3[:, :, sl] = 1
        gv, gf = api.extract(api.DeviceGrid.upload(g, R)).download()
        d = oracle.dmc_extract(g, R)
        assert np.array_equal(gf, d["faces"]) and np.array_equal(u64(gv), u64(d["vertices"])), seed
        t = api.analyze_topology((gv, gf))
        assert t["manifold"] and t["watertight"], seed
        assert len(api.detect_self_intersections((gv, gf))) == 0, seed
