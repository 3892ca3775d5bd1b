"""GPU edge cases and error behaviour (SPEC.md error clauses; reference exception mapping),
plus larger-input parity (C2 scale) and determinism."""
import numpy as np
import pytest

from paper_2509_05595_b200 import fixtures as FX

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def test_empty_inputs(api):
    v = np.zeros((0, 3))
    f = np.zeros((0, 3), np.int32)
    g = api.compute_udf((v, f), 16)
    assert np.isinf(g.download()).all()                       # SPEC.md:201 empty -> +INF
    s = api.compute_sdf((v, f), 16).download()
    assert (s == 1.0).all()                                   # sentinel -> +1.0
    m = api.extract(api.DeviceGrid.upload(s, 16))             # all positive -> empty mesh
    assert m.size() == (0, 0)
    assert len(api.detect_self_intersections((v, f))) == 0


def test_invalid_arguments_raise(api, c1):
    from paper_2509_05595_b200._lib import PamoptInvalidArgument
    with pytest.raises(PamoptInvalidArgument):
        api.compute_udf((c1["v"], c1["f"]), 100)              # R not a power of two
    for R in (2048, 4096):  # 32-bit cell ids: R is capped at 1024 before anything is allocated
        with pytest.raises(PamoptInvalidArgument):
            api.compute_sdf((c1["v"], c1["f"]), R)
        with pytest.raises(PamoptInvalidArgument):
            api.remesh_device(api.DeviceMesh.upload(c1["v"], c1["f"]), R, 100)
    g = api.compute_udf((c1["v"], c1["f"]), 32)
    with pytest.raises(PamoptInvalidArgument):
        api.udf_to_sdf(g, 0.5)                                # eps out of range
    # non-manifold input to simplify: three faces on one edge
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1]], float)
    f = np.array([[0, 1, 2], [1, 0, 3], [0, 1, 4]], np.int32)
    with pytest.raises(PamoptInvalidArgument):
        api.simplify_to((v, f), 1)


def test_simplify_target_not_below_faces_is_identity(api):
    v, f = FX.icosphere(2)
    m, st = api.simplify_to((v, f), 10_000)
    vo, fo = m.download()
    assert np.array_equal(fo, f) and np.array_equal(bits(vo), bits(v))
    assert st["iterations"] == 0


def test_tetrahedron_cannot_simplify(api, oracle):
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    f = np.array([[0, 2, 1], [0, 1, 3], [1, 2, 3], [0, 3, 2]], np.int32)
    m, st = api.simplify_to((v, f), 1)                        # every edge fails the link condition
    vo, fo = m.download()
    assert len(fo) == 4
    ro = oracle.simplify(v, f, 1)
    assert np.array_equal(fo, ro[1]) and st["iterations"] == ro[2]["iterations"]


def test_open_mesh_simplify_parity(api, oracle):
    """Boundary edges / virtual boundary vertex of the link condition (mesh.cpp:298-356)."""
    n = 40
    xs = np.linspace(0, 1, n)
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    rng = FX.Rng(21)
    Z = 0.05 * np.sin(6 * X) * np.cos(5 * Y) + 0.002 * rng.uniform(n * n).reshape(n, n)
    v = np.stack([X, Y, Z], -1).reshape(-1, 3)
    f = []
    for i in range(n - 1):
        for j in range(n - 1):
            a, b, c, d = i * n + j, (i + 1) * n + j, (i + 1) * n + j + 1, i * n + j + 1
            f += [[a, b, c], [a, c, d]]
    f = np.array(f, np.int32)
    vo, fo, st = oracle.simplify(v, f, 300)
    m, gst = api.simplify_to((v, f), 300)
    gv, gf = m.download()
    assert np.array_equal(gf, fo) and np.array_equal(bits(gv), bits(vo))
    assert gst["iterations"] == st["iterations"]


def test_pipeline_deterministic(api, c1):
    a = api.run_pipeline(c1["v"], c1["f"], c1["R"], c1["target"])
    b = api.run_pipeline(c1["v"], c1["f"], c1["R"], c1["target"])
    assert np.array_equal(a.faces, b.faces) and np.array_equal(bits(a.vertices), bits(b.vertices))


def test_c2_udf_dmc_and_soup_intersections_parity(api, oracle):
    """C2 scale: 200k-triangle interpenetrating soup at R=256 — UDF/SDF grid, DMC mesh and the
    self-intersection pairs of the raw soup, all bit-exact against the oracle."""
    v, f, R, _ = FX.make_config("c2")
    udf, sdf = oracle.compute_udf_sdf(v, f, R)
    g = api.compute_sdf((v, f), R)
    assert np.array_equal(bits(g.download()), bits(sdf))
    d = oracle.dmc_extract(sdf, R)
    mv, mf = api.extract(g).download()
    assert np.array_equal(mf, d["faces"]) and np.array_equal(bits(mv), bits(d["vertices"]))
    # raw soup: interpenetrating primitives -> many true intersections
    sub = f[:40000]
    got = api.detect_self_intersections((v, sub))
    ref = oracle.self_intersections(v, sub)
    assert len(ref) > 100 and np.array_equal(got, ref)


def test_hierarchy_levels_c1_scale(api, oracle, c1):
    for r in (8, 32, 128):
        got = api.build_hierarchy_pairs((c1["v"], c1["f"]), c1["R"], r)
        ref = oracle.hierarchy_pairs(c1["v"], c1["f"], c1["R"], r)
        assert np.array_equal(got, ref), r


def test_concurrent_contexts_match_sequential(api):
    """Distinct contexts on distinct host threads (the C5 batch path) give the same outputs as
    sequential runs: contexts share nothing but the device."""
    import threading
    cases = [FX.make_config("c1")[:2] + (128, 3000), (FX.soup(6, 5000, seed=11)) + (128, 4000)]
    cases = [(FX.normalize_unit_cube(v, 6.0 / R)[0], f, R, t) for v, f, R, t in cases]
    seq = [api.run_pipeline(v, f, R, t) for v, f, R, t in cases]
    out = [None] * len(cases)

    def work(k):
        ctx = api.Context(0)
        v, f, R, t = cases[k]
        m = api.DeviceMesh.upload(v, f, ctx)
        o, st, tm = api.remesh_device(m, R, t)
        out[k] = o.download()
        o.free()
        m.free()
        ctx.close()

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(cases))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for s, (ov, of) in zip(seq, out):
        assert np.array_equal(of, s.faces) and np.array_equal(bits(ov), bits(s.vertices))
