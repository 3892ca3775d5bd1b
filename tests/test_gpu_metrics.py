"""GPU certification / quality metrics against the reference's own
analyze_topology / nearest_primitive (golden vectors from oracle/_ref) and the oracle restatement."""
import numpy as np
import pytest

from paper_2509_05595_b200 import fixtures as FX
from tests.metrics_corpus import nearest_cases, topology_corpus
from tests.test_metrics_oracle import GOLD, _squares

pytestmark = pytest.mark.gpu


def _u64(a):
    return np.ascontiguousarray(a).view(np.uint64)


def test_topology_matches_reference(api, oracle):
    for name, (v, f) in topology_corpus().items():
        t = api.analyze_topology((v, f))
        s = GOLD[f"topo_{name}_summary"]
        assert [t["manifold"], t["watertight"], t["euler"], t["boundary_edges"]] == list(s), name
        assert np.array_equal(t["nonmanifold_edges"], GOLD[f"topo_{name}_edges"]), name
        assert np.array_equal(t["nonmanifold_vertices"], GOLD[f"topo_{name}_verts"]), name


def test_topology_on_pipeline_meshes(api, oracle, c1):
    g = api.compute_sdf((c1["v"], c1["f"]), c1["R"])
    d = api.extract(g)
    dv, df = d.download()
    for v, f in ((dv, df), (c1["v"], c1["f"])):
        t = api.analyze_topology((v, f))
        o = oracle.topology(f, len(v))
        for k in t:
            assert np.array_equal(t[k], o[k]) if isinstance(t[k], np.ndarray) else t[k] == o[k], k
    assert api.analyze_topology(d)["watertight"]


def test_nearest_matches_reference(api):
    for name, v, f, p in nearest_cases():
        face, dist, clo = api.nearest_primitive((v, f), p)
        assert np.array_equal(face, GOLD[f"near_{name}_face"]), name
        assert np.array_equal(_u64(dist), GOLD[f"near_{name}_dist_bits"]), name
        assert np.array_equal(_u64(clo), GOLD[f"near_{name}_closest_bits"]), name


def test_nearest_large_vs_oracle(api, oracle):
    v, f, _, _ = FX.make_config("c2")
    rng = FX.Rng(11)
    p = rng.uniform(3 * 1500).reshape(-1, 3) * 1.2 - 0.1
    p[:500] = v[f[:500, 0]] * 0.5 + v[f[:500, 1]] * 0.5  # on edges: many near-ties
    got = api.nearest_primitive((v, f), p)
    ref = oracle.nearest(v, f, p)
    for a, b in zip(got, ref):
        assert np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))


def test_sampler_bit_exact(api, oracle, c1):
    for n, seed in ((1000, 1), (50000, 42)):
        gp, gf, ga = api.sample_points((c1["v"], c1["f"]), n, seed)
        op, of, oa = oracle.sample(c1["v"], c1["f"], n, seed)
        assert np.array_equal(gf, of) and np.array_equal(_u64(gp), _u64(op))
        assert abs(ga - oa) <= 1e-12 * oa


def test_chamfer_hausdorff_angle_vs_oracle(api, oracle, c1):
    v, f = c1["v"], c1["f"]
    out = api.run_pipeline(v, f, c1["R"], c1["target"])
    a, b = (v, f), (out.vertices, out.faces)
    for n in (1024, 8192):
        cd = api.chamfer(a, b, n, 7)
        hd = api.hausdorff(a, b, n, 7)
        ocd = oracle.chamfer(v, f, out.vertices, out.faces, n, 7)
        ohd = oracle.hausdorff(v, f, out.vertices, out.faces, n, 7)
        assert abs(cd - ocd) <= 1e-12 * ocd and hd == ohd
    assert abs(api.min_internal_angle(b) - oracle.min_internal_angle(*b)) < 1e-12
    h = 0.125
    va, fa, vb, fb = _squares(h)
    assert abs(api.chamfer((va, fa), (vb, fb), 2048) - 2 * h * h) < 1e-12
    assert abs(api.hausdorff((va, fa), (vb, fb), 2048) - h) < 1e-12


def test_report_and_errors(api, c1):
    from paper_2509_05595_b200._lib import PamoptInvalidArgument
    out = api.run_pipeline(c1["v"], c1["f"], c1["R"], c1["target"])
    r = api.mesh_report((out.vertices, out.faces), (c1["v"], c1["f"]), 4096)
    assert r["manifold"] and r["watertight"] and r["intersection_free"]
    assert r["n_faces"] == len(out.faces) and 0 < r["min_angle_deg"] <= 60.0 and 0 <= r["cd"] < 1e-3
    r0 = api.mesh_report((out.vertices, out.faces))
    assert np.isnan(r0["cd"]) and r0["watertight"]
    flat = (np.zeros((3, 3)), np.array([[0, 1, 2]], np.int32))
    with pytest.raises(PamoptInvalidArgument):
        api.chamfer(flat, (out.vertices, out.faces), 64)
    with pytest.raises(PamoptInvalidArgument):
        api.analyze_topology((np.zeros((3, 3)), np.array([[0, 1, 5]], np.int32)))
    face, dist, _ = api.nearest_primitive((np.zeros((0, 3)), np.zeros((0, 3), np.int32)), np.zeros((2, 3)))
    assert (face == -1).all() and np.isinf(dist).all()
