"""Generates tests/golden/ref_ingest.npz: the reference's own load_mesh (mesh_io.cpp:372-385,
compiled from /root/reference/proj/src into oracle/_ref) on every file of
tests/ingest_corpus.corpus().  Run here (needs /root/reference):
python tests/golden/make_golden_ingest.py"""
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import pyoracle as O  # noqa: E402
from ingest_corpus import corpus  # noqa: E402


def main():
    O.build(ref=True)
    out = {}
    for name, (ext, data) in corpus().items():
        with tempfile.NamedTemporaryFile(suffix="." + ext, delete=False) as fh:
            fh.write(data)
            path = fh.name
        try:
            v, f, st = O.ref_load_mesh(path)
        finally:
            os.unlink(path)
        out[f"{name}_v_bits"] = v.view(np.uint64)
        out[f"{name}_f"] = f
        out[f"{name}_stats"] = np.array([st["degenerate_faces_dropped"], st["polygons_triangulated"],
                                         st["vertices_welded"]], np.int64)
    np.savez_compressed(os.path.join(HERE, "ref_ingest.npz"), **out)


if __name__ == "__main__":
    main()
