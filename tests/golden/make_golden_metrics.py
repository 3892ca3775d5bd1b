"""Generates tests/golden/ref_metrics.npz from the reference itself (oracle/_ref, compiled from
/root/reference/proj/src by oracle/Makefile): analyze_topology summaries + non-manifold lists
(mesh.cpp:113-150) over tests/metrics_corpus.topology_corpus(), and
TriangleBvh::nearest_primitive (lbvh.cpp:192-237) over tests/metrics_corpus.nearest_cases().
Run here (needs /root/reference): python tests/golden/make_golden_metrics.py"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import pyoracle as O  # noqa: E402
from metrics_corpus import nearest_cases, topology_corpus  # noqa: E402


def main():
    O.build(ref=True)
    assert O.ref_available(), "oracle/_ref/libpamopt_ref.so missing (needs /root/reference)"
    out = {}
    for name, (v, f) in topology_corpus().items():
        t = O.ref_topology_full(v, f)
        out[f"topo_{name}_summary"] = np.array([t["manifold"], t["watertight"], t["euler"], t["boundary_edges"]],
                                               np.int64)
        out[f"topo_{name}_edges"] = t["nonmanifold_edges"]
        out[f"topo_{name}_verts"] = t["nonmanifold_vertices"]
    for name, v, f, p in nearest_cases():
        face, dist, clo = O.ref_nearest(v, f, p)
        out[f"near_{name}_face"] = face
        out[f"near_{name}_dist_bits"] = dist.view(np.uint64)
        out[f"near_{name}_closest_bits"] = clo.view(np.uint64)
    np.savez_compressed(os.path.join(HERE, "ref_metrics.npz"), **out)


if __name__ == "__main__":
    main()
