"""Generates tests/golden/tri_corpus_10100.npz: SPEC acceptance criterion #3's corpus size
(SPEC.md:809, 10,100 generated pairs covering coplanar, sharp, vertex-sharing and edge-sharing
cases; tests/tri_corpus.py, seed 11) with the verdicts and pair classes of the independent
exact rational-arithmetic oracle (tests/exact_tri.py).

    python tests/golden/make_golden_tri.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from tests.exact_tri import classify_pairs, verdict_pairs  # noqa: E402
from tests.tri_corpus import corpus  # noqa: E402

if __name__ == "__main__":
    v, f, p = corpus(10100, seed=11)
    r = np.array(verdict_pairs(v.tolist(), f.tolist(), p.tolist()), np.int8)
    sh, cp = classify_pairs(v.tolist(), f.tolist(), p.tolist())
    np.savez_compressed(os.path.join(HERE, "tri_corpus_10100.npz"), verdict=r, shared=np.array(sh, np.int8),
                        coplanar=np.array(cp, np.int8))
    print(len(r), "pairs,", int(r.sum()), "intersecting,", int(np.sum(cp)), "coplanar")
