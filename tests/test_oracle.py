"""CPU tests of the oracle (the checker): pinned against the reference's own code through the
committed golden fixtures (tests/golden, made by tests/golden/make_golden.py from the reference
translation units), against the live compiled reference when oracle/_ref is present, and against
the SPEC known answers."""
import json
import os

import numpy as np
import pytest

from paper_2509_05595_b200 import fixtures as FX

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


# ---------------------------------------------------------------- golden (reference-made)
def test_distance_matches_reference_golden(oracle):
    g = np.load(os.path.join(GOLD, "ref_distance.npz"))
    d = oracle.point_triangle_sq(g["p"], g["a"], g["b"], g["c"])
    assert np.array_equal(bits(d), g["d2_bits"])


def test_link_condition_matches_reference_golden(oracle):
    g = np.load(os.path.join(GOLD, "ref_link.npz"))
    names = sorted({k.rsplit("_", 1)[0] for k in g.files})
    for n in names:
        got = oracle.link_condition(g[n + "_v"], g[n + "_f"], g[n + "_e"])
        assert np.array_equal(got, g[n + "_r"]), n
    # tetrahedron edges fail, icosphere interior edges pass
    assert not g["tetra_r"].any()
    assert g["icosphere2_r"].all()


def test_collapse_undo_matches_reference_golden(oracle):
    """The oracle's collapse semantics (used inside simplify) reproduce mesh.cpp:363-416."""
    g = np.load(os.path.join(GOLD, "ref_collapse.npz"))
    # undo restores bit-exactly
    assert np.array_equal(bits(g["undo_v"]), bits(g["v"]))
    assert np.array_equal(g["undo_f"], g["f"])
    top = json.load(open(os.path.join(GOLD, "ref_topology.json")))
    assert top["icosphere2_collapsed"]["manifold"] and top["icosphere2_collapsed"]["euler"] == 2


def test_overlap_pairs_match_reference_lbvh_golden(oracle):
    g = np.load(os.path.join(GOLD, "ref_bvh_pairs.npz"))
    got = oracle.overlap_pairs(g["v"], g["f"])
    ref = g["pairs"]
    key = lambda p: set(map(tuple, p.tolist()))
    assert key(got) == key(ref)


def test_normalize_matches_reference_golden():
    g = np.load(os.path.join(GOLD, "ref_normalize.npz"))
    out, (scale, tr) = FX.normalize_unit_cube(g["v_in"], 6.0 / 128)
    assert np.array_equal(bits(out), bits(g["v_out"]))
    assert scale == g["st"][0] and np.array_equal(tr, g["st"][1:])


def test_dmc_table_snapshot(oracle):
    snap = np.array(json.load(open(os.path.join(GOLD, "dmc_table.json")))["table"], np.int32)
    assert np.array_equal(oracle.dmc_table(), snap)


# ---------------------------------------------------------------- live reference (if built)
ref_only = pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(GOLD), "..", "oracle", "_ref",
                                                             "libpamopt_ref.so")), reason="oracle/_ref not built")


@ref_only
def test_link_condition_live_reference_random_meshes(oracle):
    v, f = FX.icosphere(3)
    rng = np.random.default_rng(1)
    # random collapses create low-valence / pinched neighbourhoods
    e = np.unique(np.sort(np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]]), 1), axis=0)
    pick = e[rng.choice(len(e), 300, replace=False)]
    ok, cv, cf = oracle.ref_collapse_sequence(v, f, pick, v[pick[:, 0]])
    e2 = np.unique(np.sort(np.concatenate([cf[:, [0, 1]], cf[:, [1, 2]], cf[:, [2, 0]]]), 1), axis=0).astype(np.int32)
    assert np.array_equal(oracle.link_condition(cv, cf, e2), oracle.ref_link_condition(cv, cf, e2))


@ref_only
def test_topology_of_dmc_output_live_reference(oracle):
    R = 32
    for seed in range(3):
        g = np.random.default_rng(seed).uniform(-1, 1, (R + 1) ** 3).astype(np.float32)
        g3 = g.reshape(R + 1, R + 1, R + 1)
        for sl in (0, -1):
            g3[sl, :, :] = 1
            g3[:, sl, :] = 1
            g3[:, :, sl] = 1
        d = oracle.dmc_extract(g, R)
        t = oracle.ref_topology(d["vertices"], d["faces"])
        assert t["manifold"] and t["watertight"], t


# ---------------------------------------------------------------- SPEC known answers
def test_spec_distance_examples(oracle):
    # unit square at z=0.5, R=16 -> 0 and 1/16
    sq = np.array([[0.25, 0.25, 0.5], [0.75, 0.25, 0.5], [0.75, 0.75, 0.5], [0.25, 0.75, 0.5]])
    f = np.array([[0, 1, 2], [0, 2, 3]], np.int32)
    R = 16
    udf, sdf = oracle.compute_udf_sdf(sq, f, R)
    g = udf.reshape(R + 1, R + 1, R + 1)
    assert g[8, 8, 8] == 0.0
    assert g[9, 8, 8] == np.float32(1 / 16)
    assert np.isinf(g[0, 0, 0])
    s = sdf.reshape(R + 1, R + 1, R + 1)
    assert s[0, 0, 0] == 1.0                       # sentinel -> +1.0
    assert s[8, 8, 8] == np.float32(-0.9 / R)      # u = 0 -> -eps


def test_spec_sigmoid_examples(oracle):
    assert abs(oracle.sigmoid(0.0, 5.0) - 0.07585818002124355) < 1e-15
    assert oracle.sigmoid(0.5, 5.0) == 0.5
    assert oracle.sigmoid(0.4, 500.0) < 1e-20
    for x in np.linspace(-700, 700, 1401):
        assert abs(oracle.det_exp(x) - np.exp(x)) <= 4e-16 * np.exp(x)


def test_dmc_table_invariants(oracle):
    t = oracle.dmc_table()
    assert t[0, 0] == 0 and t[255, 0] == 0
    for c in range(256):
        union = int(np.bitwise_or.reduce(t[c, 1:5]))
        comp = int(np.bitwise_or.reduce(t[255 - c, 1:5]))
        assert union == comp                                               # SPEC.md:247,313 (P12)
        assert bin(t[c, 5]).count("1") <= 1


def test_dmc_single_negative_corner(oracle):
    # one negative corner -> one patch of 3 edges
    t = oracle.dmc_table()
    for c in range(8):
        assert t[1 << c, 0] == 1 and bin(t[1 << c, 1]).count("1") == 3


def test_dmc_sphere_and_torus_euler(oracle):
    R = 32
    x = np.arange(R + 1) / R
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    sph = (np.sqrt((X - .5) ** 2 + (Y - .5) ** 2 + (Z - .5) ** 2) - 0.3).astype(np.float32)
    d = oracle.dmc_extract(sph.transpose(2, 1, 0).ravel(), R)
    V, F = len(d["vertices"]), len(d["faces"])
    assert V - F * 3 // 2 + F == 2
    q = np.sqrt((X - .5) ** 2 + (Y - .5) ** 2)
    tor = (np.sqrt((q - 0.3) ** 2 + (Z - .5) ** 2) - 0.1).astype(np.float32)
    d = oracle.dmc_extract(tor.transpose(2, 1, 0).ravel(), R)
    V, F = len(d["vertices"]), len(d["faces"])
    assert V - F * 3 // 2 + F == 0
    assert len(oracle.self_intersections(d["vertices"], d["faces"])) == 0


@pytest.mark.parametrize("seed", range(6))
def test_dmc_random_grids_manifold_intersection_free(oracle, seed):
    """SPEC.md:310,808 (scaled): random 32^3 grids -> manifold, watertight, 0 intersections."""
    R = 32
    g = np.random.default_rng(100 + seed).uniform(-1, 1, (R + 1) ** 3).astype(np.float32)
    g3 = g.reshape(R + 1, R + 1, R + 1)
    for sl in (0, -1):
        g3[sl, :, :] = 1
        g3[:, sl, :] = 1
        g3[:, :, sl] = 1
    d = oracle.dmc_extract(g, R)
    assert len(oracle.self_intersections(d["vertices"], d["faces"])) == 0
    # every edge shared by exactly two faces
    f = d["faces"]
    e = np.sort(np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]]), 1)
    _, cnt = np.unique(e, axis=0, return_counts=True)
    assert (cnt == 2).all()


def test_udf_filter_soundness_vs_brute_force(oracle):
    """in-band UDF == brute-force all-triangle minima (soup <= 1k, R <= 32)."""
    rng = FX.Rng(9)
    n = 300
    a = 0.15 + 0.7 * rng.uniform(3 * n).reshape(n, 3)
    v = (a[:, None, :] + 0.12 * (rng.uniform(9 * n).reshape(n, 3, 3) - 0.5)).reshape(-1, 3)
    f = np.arange(3 * n, dtype=np.int32).reshape(n, 3)
    R = 32
    u, _ = oracle.compute_udf_sdf(v, f, R)
    b = oracle.brute_udf(v, f, R)
    band = b <= 3.0 / R
    assert np.array_equal(bits(u[band].astype(np.float64)), bits(b[band].astype(np.float64)))
    # monotone hierarchy: level pairs are subsets of parent pairs
    prev = None
    r = 8
    while r <= R:
        cur = oracle.hierarchy_pairs(v, f, R, r)
        if prev is not None:
            rp = r // 2
            cx, cy, cz = cur[:, 0] % r, (cur[:, 0] // r) % r, cur[:, 0] // (r * r)
            parent = (cx // 2) + rp * ((cy // 2) + rp * (cz // 2))
            pp = set(zip(prev[:, 0].tolist(), prev[:, 1].tolist()))
            assert all((int(p), int(t)) in pp for p, t in zip(parent, cur[:, 1]))
        prev = cur
        r *= 2


def test_self_intersection_duplicate_face(oracle):
    """icosphere + one duplicated face -> exactly the duplicate pair(s)."""
    v, f = FX.icosphere(2)
    assert len(oracle.self_intersections(v, f)) == 0
    f2 = np.concatenate([f, f[7:8]])
    pr = oracle.self_intersections(v, f2)
    assert pr.tolist() == [[7, len(f)]]


def test_simplify_icosphere_properties(oracle):
    """icosphere 1280 -> 80 faces, manifold, chi=2, zero intersections."""
    v, f = FX.icosphere(3)
    vo, fo, st = oracle.simplify(v, f, 80)
    assert len(fo) <= 80
    e = np.sort(np.concatenate([fo[:, [0, 1]], fo[:, [1, 2]], fo[:, [2, 0]]]), 1)
    ue, cnt = np.unique(e, axis=0, return_counts=True)
    assert (cnt == 2).all()
    assert len(vo) - len(ue) + len(fo) == 2
    assert len(oracle.self_intersections(vo, fo)) == 0
    # target >= faces -> unchanged
    vo2, fo2, _ = oracle.simplify(v, f, 5000)
    assert np.array_equal(fo2, f) and np.array_equal(bits(vo2), bits(v))


def test_simplify_deterministic_across_workers(oracle):
    """identical output for any worker count."""
    v, f = FX.icosphere(3)
    v = v * (1 + 0.05 * FX.Rng(4).normal(len(v)))[:, None]
    oracle.set_workers(1)
    a = oracle.simplify(v, f, 200)
    oracle.set_workers(os.cpu_count() or 4)
    b = oracle.simplify(v, f, 200)
    assert np.array_equal(a[1], b[1]) and np.array_equal(bits(a[0]), bits(b[0]))


def test_oracle_link_condition_high_valence_matches_reference(oracle):
    """Valence 600-1000 (tests/golden/make_golden_valence.py, the reference's own
    link_condition_holds): the oracle restatement has no capacity limit either."""
    g = np.load(os.path.join(GOLD, "ref_link_valence.npz"))
    for n in sorted({k.rsplit("_", 1)[0] for k in g.files}):
        got = oracle.link_condition(g[f"{n}_v"], g[f"{n}_f"], g[f"{n}_e"])
        assert np.array_equal(got.astype(np.int8), g[f"{n}_r"]), n
