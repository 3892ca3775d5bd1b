"""SPEC acceptance #5 (scaled PAPER §9.3): the edge-cost terms matter on flat-heavy
input.  With w_e = w_s = 0 (pure QEM, constant on flat regions) against the defaults (w_e = 1e-3,
w_s = 5e-3), the default configuration yields a strictly lower bad-triangle ratio (minimum
corner angle below 10, 20 and 30 degrees).  Both GPU runs are also the oracle's, bit for bit."""
import numpy as np
import pytest

from paper_2509_05595_b200 import fixtures as FX

pytestmark = pytest.mark.gpu


def bad_ratio(v, f, thresholds=(10.0, 20.0, 30.0)):
    a, b, c = v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]

    def ang(p, q, r):
        u, w = q - p, r - p
        cs = (u * w).sum(1) / np.sqrt((u * u).sum(1) * (w * w).sum(1))
        return np.degrees(np.arccos(np.clip(cs, -1.0, 1.0)))

    m = np.minimum(np.minimum(ang(a, b, c), ang(b, c, a)), ang(c, a, b))
    return np.array([(m < t).mean() for t in thresholds])


@pytest.mark.parametrize("name", ["box", "cylinder"])
def test_edge_cost_ablation(api, oracle, name):
    v, f = FX.box(20, 30, 13) if name == "box" else FX.cylinder(50, 49)
    R = 64
    v, _ = FX.normalize_unit_cube(v, 6.0 / R)
    dv, df = api.extract(api.compute_sdf((v, f), R)).download()
    target = len(df) // 20
    ratios = {}
    for we, ws in ((0.0, 0.0), (1e-3, 5e-3)):
        out, st = api.simplify_to(api.DeviceMesh.upload(dv, df), target, we=we, ws=ws)
        gv, gf = out.download()
        ov, of, _ = oracle.simplify(dv, df, target, we=we, ws=ws)
        assert np.array_equal(gf, of) and np.array_equal(gv.view(np.uint64), ov.view(np.uint64))
        ratios[(we, ws)] = bad_ratio(gv, gf)
    assert np.all(ratios[(1e-3, 5e-3)] < ratios[(0.0, 0.0)]), ratios
