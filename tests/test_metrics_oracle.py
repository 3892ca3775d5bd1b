"""Oracle restatement of the certification / metrics operations pinned
against the reference itself: golden vectors from oracle/_ref (tests/golden/ref_metrics.npz,
made by tests/golden/make_golden_metrics.py) and, when /root/reference is present, live calls.
Plus the SPEC quality_metrics known answers."""
import numpy as np
import pytest

from tests.metrics_corpus import nearest_cases, topology_corpus

GOLD = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "ref_metrics.npz"))


def test_topology_matches_reference_golden(oracle):
    for name, (v, f) in topology_corpus().items():
        t = oracle.topology(f, len(v))
        s = GOLD[f"topo_{name}_summary"]
        assert [t["manifold"], t["watertight"], t["euler"], t["boundary_edges"]] == list(s), name
        assert np.array_equal(t["nonmanifold_edges"], GOLD[f"topo_{name}_edges"]), name
        assert np.array_equal(t["nonmanifold_vertices"], GOLD[f"topo_{name}_verts"]), name


def test_nearest_matches_reference_golden(oracle):
    for name, v, f, p in nearest_cases():
        face, dist, clo = oracle.nearest(v, f, p)
        assert np.array_equal(face, GOLD[f"near_{name}_face"]), name
        assert np.array_equal(dist.view(np.uint64), GOLD[f"near_{name}_dist_bits"]), name
        assert np.array_equal(clo.view(np.uint64), GOLD[f"near_{name}_closest_bits"]), name


def test_live_reference_topology_on_dmc_mesh(oracle):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (no /root/reference)")
    from paper_2509_05595_b200 import fixtures as FX
    v, f = FX.icosphere(3)
    R = 32
    v, _ = FX.normalize_unit_cube(v, 6.0 / R)
    _, sdf = oracle.compute_udf_sdf(v, f, R)
    d = oracle.dmc_extract(sdf, R)
    a = oracle.topology(d["faces"], len(d["vertices"]))
    b = oracle.ref_topology_full(d["vertices"], d["faces"])
    assert a["watertight"] and a["manifold"]
    for k in a:
        assert np.array_equal(a[k], b[k]) if isinstance(a[k], np.ndarray) else a[k] == b[k], k


def _squares(h):
    v = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], float)
    f = np.array([[0, 1, 2], [0, 2, 3]], np.int32)
    return v, f, v + np.array([0, 0, h]), f


def test_metrics_known_answers(oracle):
    """SPEC quality_metrics examples: parallel unit squares at gap h -> CD = 2h^2, HD = h;
    identical meshes -> 0; equilateral -> 60 deg, right isosceles -> 45 deg."""
    h = 0.125
    va, fa, vb, fb = _squares(h)
    assert abs(oracle.chamfer(va, fa, vb, fb, 2048) - 2 * h * h) < 1e-12
    assert abs(oracle.hausdorff(va, fa, vb, fb, 2048) - h) < 1e-12
    assert oracle.chamfer(va, fa, va, fa, 2048) < 1e-12
    assert abs(oracle.min_internal_angle(np.array([[0, 0, 0], [1, 0, 0], [0.5, np.sqrt(3) / 2, 0]]),
                                         np.array([[0, 1, 2]], np.int32)) - 60.0) < 1e-9
    assert abs(oracle.min_internal_angle(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]]),
                                         np.array([[0, 1, 2]], np.int32)) - 45.0) < 1e-9
    with pytest.raises(ValueError):
        oracle.chamfer(va, np.array([[0, 0, 1]], np.int32), vb, fb, 16)


def test_sampler_is_area_weighted_and_on_surface(oracle):
    from paper_2509_05595_b200 import fixtures as FX
    v, f = FX.uv_sphere(20, 20)  # face areas vary with latitude
    pts, fid, area = oracle.sample(v, f, 200000, 5)
    a, b, c = v[f[fid, 0]], v[f[fid, 1]], v[f[fid, 2]]
    n = np.cross(b - a, c - a)
    assert np.abs(np.einsum("ij,ij->i", pts - a, n)).max() < 1e-12 * max(1.0, np.abs(n).max())
    # area weighting: sample counts per face track the areas
    A = 0.5 * np.linalg.norm(np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]]), axis=1)
    assert abs(A.sum() - area) < 1e-12 * A.sum()
    cnt = np.bincount(fid, minlength=len(f))
    assert np.corrcoef(cnt, A)[0, 1] > 0.97
    assert np.array_equal(oracle.sample(v, f, 100, 5)[0], pts[:100])  # counter-based: prefix-stable
