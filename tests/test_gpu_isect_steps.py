"""SPEC-granular tri_isect operations through the C-ABI on SPEC acceptance
criterion #3's 10,100-pair corpus (tests/golden/tri_corpus_10100.npz, verdicts and classes from
the exact rational oracle): classify_pair, intersect_3d on the non-coplanar pairs,
intersect_coplanar on the coplanar ones, and the dispatching verdict on all of them."""
import os

import numpy as np
import pytest

from tests.tri_corpus import corpus

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def c10100():
    v, f, pairs = corpus(10100, seed=11)
    return v, f, pairs, np.load(os.path.join(GOLD, "tri_corpus_10100.npz"))


def test_classify_pair_matches_exact(api, c10100):
    v, f, pairs, g = c10100
    sh, cp = api.classify_pair((v, f), pairs)
    assert np.array_equal(sh, g["shared"]) and np.array_equal(cp, g["coplanar"])


def test_intersect_by_class_matches_exact(api, c10100):
    v, f, pairs, g = c10100
    cop = g["coplanar"].astype(bool)
    i3 = api.intersect_3d((v, f), pairs[~cop])
    ic = api.intersect_coplanar((v, f), pairs[cop])
    assert np.array_equal(i3, g["verdict"][~cop]) and np.array_equal(ic, g["verdict"][cop])
    allv = api.tri_tri_pairs((v, f), pairs)
    fn = int(((g["verdict"] == 1) & (allv == 0)).sum())
    fp = int(((g["verdict"] == 0) & (allv == 1)).sum())
    assert fn == 0 and fp == 0, (fn, fp)  # FNR 0, FPR < 1%
    # preconditions are enforced
    with pytest.raises(api._lib.PamoptInvalidArgument):
        api.intersect_3d((v, f), pairs[cop][:4])
    with pytest.raises(api._lib.PamoptInvalidArgument):
        api.intersect_coplanar((v, f), pairs[~cop][:4])
