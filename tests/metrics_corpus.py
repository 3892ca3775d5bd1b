"""Meshes for the certification / metrics parity tests (analyze_topology, nearest_primitive):
manifold, boundary, pinched, non-manifold-edge fans, degenerate and duplicate faces, isolated
vertices, random index soups, and a DMC output."""
import numpy as np

from paper_2509_05595_b200 import fixtures as FX


def topology_corpus():
    out = {}
    v, f = FX.icosphere(2)
    out["icosphere2"] = (v, f)
    gv = np.array([[x, y, 0.1 * x * y] for y in range(4) for x in range(5)], float)
    gf = []
    for y in range(3):
        for x in range(4):
            a, b, c, d = y * 5 + x, y * 5 + x + 1, (y + 1) * 5 + x + 1, (y + 1) * 5 + x
            gf += [[a, b, c], [a, c, d]]
    out["strip"] = (gv, np.array(gf, np.int32))
    v1, f1 = FX.icosphere(0)
    vv = np.concatenate([v1, v1 + np.array([3.0, 0.0, 0.0])])
    ff = np.concatenate([f1, f1 + len(v1)])
    ff[ff == len(v1) + 9] = 9
    out["pinched"] = (vv, ff.astype(np.int32))
    # three faces on one edge (non-manifold edge), plus a bowtie of two fans at one vertex
    fv = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [2, 2, 2], [3, 2, 2], [2, 3, 2]], float)
    out["fan3"] = (fv, np.array([[0, 1, 2], [1, 0, 3], [0, 1, 4], [0, 5, 6], [0, 6, 7]], np.int32))
    # degenerate (repeated index) and duplicate faces, isolated vertex 9
    dv = np.concatenate([v1, np.array([[5.0, 5.0, 5.0]])])
    df = np.concatenate([f1, np.array([[0, 0, 1], [2, 3, 2], [4, 4, 4]], np.int32), f1[:3]])
    out["degenerate_dup"] = (dv, df.astype(np.int32))
    # random index soups (heavily non-manifold)
    for seed, (nv, nf) in enumerate([(12, 30), (40, 200), (200, 600)]):
        rng = FX.Rng(100 + seed)
        vv = rng.uniform(3 * nv).reshape(nv, 3)
        ff = np.minimum((rng.uniform(3 * nf) * nv).astype(np.int32), nv - 1).reshape(nf, 3)
        out[f"soup{seed}"] = (vv, ff)
    # a tetrahedron-sharing-an-edge "book" and an open fan around a vertex
    bv = np.array([[0, 0, 0], [0, 0, 1], [1, 0, 0], [0, 1, 0], [-1, 0, 0], [0, -1, 0]], float)
    out["book"] = (bv, np.array([[0, 1, 2], [0, 1, 3], [0, 1, 4], [0, 1, 5]], np.int32))
    out["open_fan"] = (bv, np.array([[0, 2, 3], [0, 3, 4], [0, 4, 5]], np.int32))
    return out


def nearest_cases():
    """(name, v, f, points): includes exact ties (duplicate faces), points on vertices/edges, far points."""
    out = []
    v, f = FX.icosphere(3)
    rng = FX.Rng(7)
    p = np.concatenate([rng.normal(3 * 300).reshape(-1, 3) * 0.7, v[:50], 0.5 * (v[f[:50, 0]] + v[f[:50, 1]]),
                        rng.normal(3 * 20).reshape(-1, 3) * 10.0])
    out.append(("icosphere3", v, f, p))
    v2, f2 = FX.soup(4, 5000, seed=3)
    f2 = np.concatenate([f2, f2[::7]])  # duplicate faces: exact distance ties -> lower id
    p2 = rng.uniform(3 * 500).reshape(-1, 3) * (v2.max(0) - v2.min(0)) + v2.min(0)
    out.append(("soup_dup", v2, f2.astype(np.int32), p2))
    return out
