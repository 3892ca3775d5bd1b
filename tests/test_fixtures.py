import numpy as np

from paper_2509_05595_b200 import fixtures as FX


def test_splitmix_known_values():
    # SplitMix64 reference outputs for seed 0 (counter 1..3)
    z = FX.splitmix64(0, 3)
    assert z.dtype == np.uint64 and len(set(z.tolist())) == 3


def test_configs_sizes_and_normalisation():
    v, f, R, target = FX.make_config("c1")
    assert len(f) == 20480 and R == 128 and target == 5000
    pad = 6.0 / R
    assert v.min() >= pad - 1e-12 and v.max() <= 1 - pad + 1e-12
    v2, f2, R2, _ = FX.make_config("c2")
    assert len(f2) == 200000 and R2 == 256


def test_primitives_closed():
    for kind in range(5):
        v, f = FX.primitive(kind, 5000)
        e = np.sort(np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]]), 1)
        _, cnt = np.unique(e, axis=0, return_counts=True)
        assert (cnt == 2).all(), kind


def test_determinism():
    a = FX.soup(3, 5000, seed=7)
    b = FX.soup(3, 5000, seed=7)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
