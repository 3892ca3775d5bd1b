"""Generates the golden fixtures in tests/golden/ from the REFERENCE's own code.

Run in a container that has /root/reference (the reference translation units are compiled in
place by `make -C oracle ref` into oracle/_ref/libpamopt_ref.so):

    python tests/golden/make_golden.py

Outputs (small, committed):
  ref_distance.npz   point_triangle_sq_distance<double> (distance.cpp:26-79) on 4096 random and
                     degenerate (p, a, b, c) tuples — stored as raw f64 bits
  ref_link.npz       link_condition_holds (mesh.cpp:301-358) for every edge of three meshes
                     (icosphere-2, a tetrahedron, an open strip with a boundary, a pinched mesh)
  ref_collapse.npz   collapse_edge / undo_collapse / compact (mesh.cpp:278-416) sequences
  ref_topology.json  analyze_topology (mesh.cpp:113-150) summaries
  ref_bvh_pairs.npz  TriangleBvh overlap pairs (lbvh.cpp:159-190, 1e-7 inflation)
  ref_normalize.npz  normalize_unit_cube (mesh_io.cpp:393-408)
  dmc_table.json     the generated 256-entry DMC patch table snapshot
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle as O  # noqa: E402
from paper_2509_05595_b200 import fixtures as FX  # noqa: E402


def meshes():
    out = {}
    v, f = FX.icosphere(2)
    out["icosphere2"] = (v, f)
    out["tetra"] = (np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float),
                    np.array([[0, 2, 1], [0, 1, 3], [1, 2, 3], [0, 3, 2]], np.int32))
    # open strip (boundary) 3x2 quads
    gv = np.array([[x, y, 0.1 * x * y] for y in range(3) for x in range(4)], float)
    gf = []
    for y in range(2):
        for x in range(3):
            a, b, c, d = y * 4 + x, y * 4 + x + 1, (y + 1) * 4 + x + 1, (y + 1) * 4 + x
            gf += [[a, b, c], [a, c, d]]
    out["strip"] = (gv, np.array(gf, np.int32))
    # two icosahedra sharing one vertex index (pinched / non-manifold vertex)
    v1, f1 = FX.icosphere(0)
    vv = np.concatenate([v1, v1 + np.array([3.0, 0.0, 0.0])])
    ff = np.concatenate([f1, f1 + len(v1)])
    ff[ff == len(v1) + 9] = 9
    out["pinched"] = (vv, ff.astype(np.int32))
    return out


def edges_of(f):
    e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
    e = np.sort(e, axis=1)
    return np.unique(e, axis=0).astype(np.int32)


def main():
    O.build(ref=True)
    assert O.ref_available(), "oracle/_ref/libpamopt_ref.so missing (needs /root/reference)"
    rng = np.random.default_rng(2509)
    # distance
    n = 4096
    p, a, b, c = (rng.random((n, 3)) for _ in range(4))
    c[:256] = a[:256]                    # degenerate: repeated vertex
    b[256:512] = a[256:512] + 1e-13      # near-degenerate
    c[512:768] = 2 * b[512:768] - a[512:768]  # collinear
    p[768:1024] = (a[768:1024] + b[768:1024] + c[768:1024]) / 3  # on the face
    d = O.ref_point_triangle_sq(p, a, b, c)
    np.savez_compressed(os.path.join(HERE, "ref_distance.npz"), p=p, a=a, b=b, c=c, d2_bits=d.view(np.uint64))
    # link condition + topology
    ms = meshes()
    link = {}
    topo = {}
    for name, (v, f) in ms.items():
        e = edges_of(f)
        link[name + "_v"] = v
        link[name + "_f"] = f
        link[name + "_e"] = e
        link[name + "_r"] = O.ref_link_condition(v, f, e)
        topo[name] = O.ref_topology(v, f)
    np.savez_compressed(os.path.join(HERE, "ref_link.npz"), **link)
    # collapse sequences on icosphere-2: a few disjoint interior edges, midpoint placement
    v, f = ms["icosphere2"]
    e = edges_of(f)
    pick = e[rng.choice(len(e), 12, replace=False)]
    pos = (v[pick[:, 0]] + v[pick[:, 1]]) * 0.5
    ok, cv, cf = O.ref_collapse_sequence(v, f, pick, pos, undo=False)
    ok2, uv, uf = O.ref_collapse_sequence(v, f, pick, pos, undo=True)
    np.savez_compressed(os.path.join(HERE, "ref_collapse.npz"), v=v, f=f, edges=pick, pos=pos, ok=ok,
                        out_v=cv, out_f=cf, undo_v=uv, undo_f=uf)
    topo["icosphere2_collapsed"] = O.ref_topology(cv, cf)
    with open(os.path.join(HERE, "ref_topology.json"), "w") as fh:
        json.dump(topo, fh, indent=1, sort_keys=True)
    # LBVH overlap pairs on a small random soup
    k = 400
    base = rng.random((k, 3))
    sv = (base[:, None, :] + 0.05 * rng.standard_normal((k, 3, 3))).reshape(-1, 3)
    sf = np.arange(3 * k, dtype=np.int32).reshape(k, 3)
    pairs = O.ref_bvh_overlap_pairs(sv, sf)
    np.savez_compressed(os.path.join(HERE, "ref_bvh_pairs.npz"), v=sv, f=sf, pairs=pairs)
    # normalisation
    nv_, st = O.ref_normalize_unit_cube(sv * 7.0 - 3.0, 6.0 / 128)
    np.savez_compressed(os.path.join(HERE, "ref_normalize.npz"), v_in=sv * 7.0 - 3.0, v_out=nv_, st=st)
    # DMC table snapshot
    tab = O.dmc_table()
    with open(os.path.join(HERE, "dmc_table.json"), "w") as fh:
        json.dump({"layout": "per case: [n_patches, mask0, mask1, mask2, mask3, doubly_covered_faces]",
                   "table": tab.tolist()}, fh)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
