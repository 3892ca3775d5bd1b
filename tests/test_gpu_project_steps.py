"""Stage 3 step oracle: every recorded Newton iteration of the GPU safe_project is replayed on the
CPU (oracle/project_ref.py) and each piece of the step is checked on its own:

  refresh     S2M targets = nearest points of M_in (every `refresh` iterations, frozen between),
              M2S stencils = nearest face of S per sample with its class (frozen between),
              samples = the pinned sampler's
  contacts    the GPU's contact set = the brute-force set of point-triangle / edge-edge pairs
              sharing no vertex with d < d̂, with the same classes
  energy      B(X) and its gradient from the CPU restatement (autograd), rel 1e-10
  direction   the GPU's PCG solution meets the CG contract under the CPU's SPD-projected Hessian:
              |H p + g| <= cg_tol |g| (when CG stopped before its cap) and g.p < 0
  ACCD        t_max = the CPU's conservative advancement over the swept primitive pairs
  line search alpha = min(1, 0.9 t_max) / 2^(tries-1); X' = X + alpha p bit for bit;
              B(X') recomputed with the contacts at X' < B(X); X' intersection-free (exact)

Fixtures: "pull", two concentric icospheres 8e-4 apart (inside the barrier distance d̂ = 1e-3,
so the point-triangle and edge-edge barrier terms are active from the first iteration) projected
onto a wavy pair of shells that pulls the walls together; "collide", two spheres 5e-4 apart
projected onto an overlapping pair, so ACCD bounds the steps."""
import numpy as np
import pytest

from paper_2509_05595_b200 import fixtures as FX

pytestmark = pytest.mark.gpu

ITERS = 11  # iterations 0..10: two refreshes (0 and 10) with the default period


def _shells(gap=8e-4, wave=0.01):
    """"pull": inner shell r = 1, outer r = 1 + gap (inside d̂ everywhere); M_in = the pair at
    radii (1, 1 + gap / 2) times a smooth wave, so the distance terms pull the walls together."""
    v, f = FX.icosphere(3)
    n = len(v)
    r_out = 1.0 + gap
    vs = np.concatenate([v, v * r_out])
    fs = np.concatenate([f[:, ::-1], f + n]).astype(np.int32)
    s = 1.0 + wave * np.sin(3 * v[:, :1]) * np.cos(2 * v[:, 1:2])
    vin = np.concatenate([v * s, v * (r_out - 0.5 * gap) * s])
    return vs, fs, vin, fs.copy()


def _collide(gap=5e-4, shift=0.05):
    """"collide": two unit spheres side by side, their facing extreme vertices gap apart; M_in =
    the same spheres moved `shift` toward each other (overlapping), so the Newton direction drives
    the walls through each other and ACCD bounds the step."""
    v, f = FX.icosphere(3)
    n = len(v)
    a = v + [-1.0 - gap / 2, 0, 0]
    b = v + [1.0 + gap / 2, 0, 0]
    vs = np.concatenate([a, b])
    fs = np.concatenate([f, f + n]).astype(np.int32)
    vin = np.concatenate([a + [shift, 0, 0], b - [shift, 0, 0]])
    return vs, fs, vin, fs.copy()


CASES = {"pull": _shells, "collide": _collide}


@pytest.fixture(scope="module", params=sorted(CASES))
def run(api, request):
    vs, fs, vin, fin = CASES[request.param]()
    m = api.DeviceMesh.upload(vs, fs)
    st, tr = api.safe_project_traced(m, (vin, fin), ITERS, iterations=ITERS)
    return vs, fs, vin, fin, st, tr


def _rows(a):
    a = np.asarray(a, np.int64).reshape(-1, 6)
    return a[np.lexsort(a.T[::-1])]


def test_trace_is_complete(run):
    vs, fs, vin, fin, st, tr = run
    assert st["iterations"] == ITERS and len(tr["X"]) == ITERS
    assert np.array_equal(tr["X"][0], vs)
    assert len(tr["contacts"][0]) > 0  # the barrier is active from the first iteration
    kinds = set(np.concatenate([c[:, 0] for c in tr["contacts"]]).tolist())
    assert kinds == {4, 5}
    sc = tr["scalars"]
    assert (sc[:, 6] == 1).all() and (sc[:, 5] < sc[:, 0]).all()
    assert (sc[:, 2] < tr["params"]["cg_max"]).any()  # the CG residual check is exercised
    if np.abs(vs[:, 0]).max() > 1.5:  # "collide": ACCD bounds the steps
        assert (sc[:, 3] < 1.0).any()


def test_refresh_targets_and_samples(run, oracle):
    from oracle import project_ref as PR
    vs, fs, vin, fin, st, tr = run
    P = tr["params"]
    ys, _, _ = oracle.sample(vin, fin, int(P["samples"]), int(P["seed"]))
    assert np.array_equal(ys.view(np.uint64), tr["samples"].view(np.uint64))
    for it in range(len(tr["X"])):
        X = tr["X"][it]
        if it % int(P["refresh"]) == 0:
            _, _, clo = oracle.nearest(vin, fin, X)
            assert np.abs(clo - tr["targets"][it]).max() <= 1e-14, it
            face, d, _ = oracle.nearest(X, fs, ys)
            got = tr["m2s"][it]
            same = (np.sort(fs[face], 1) == np.sort(got[:, :3], 1)).all(1)
            if not same.all():  # ties only: the GPU's face is as near as the oracle's
                _, dg = PR.pt_distance2(np.concatenate([X, ys]), len(X) + np.nonzero(~same)[0],
                                        got[~same, :3].astype(np.int64))
                assert np.allclose(np.sqrt(dg), d[~same], rtol=0, atol=1e-15), it
            cls = PR.pt_class(ys, X[got[:, 0]], X[got[:, 1]], X[got[:, 2]])
            assert np.array_equal(cls, got[:, 3]), it
        else:  # frozen between refreshes
            assert np.array_equal(tr["targets"][it], tr["targets"][it - 1])
            assert np.array_equal(tr["m2s"][it], tr["m2s"][it - 1])


def test_contact_sets(run):
    from oracle import project_ref as PR
    vs, fs, vin, fin, st, tr = run
    dhat = tr["params"]["dhat"]
    for it in range(len(tr["X"])):
        ref = PR.contacts(tr["X"][it], fs, dhat)
        assert np.array_equal(_rows(ref), _rows(tr["contacts"][it])), it


@pytest.fixture(scope="module")
def replay(run):
    """Per iteration: (oracle B, oracle g, GPU scalars) and the CPU Hessian."""
    from oracle import project_ref as PR
    vs, fs, vin, fin, st, tr = run
    O = PR.StepOracle(vs, fs, vin, fin, tr["params"])
    out = []
    for it in range(len(tr["X"])):
        args = (tr["X"][it], tr["targets"][it], tr["m2s"][it], tr["samples"], tr["contacts"][it])
        B, g, parts = O.energy_grad(*args)
        out.append((B, g, parts, O.hessian_spd(*args), args))
    return O, out


def test_energy_and_gradient(run, replay):
    vs, fs, vin, fin, st, tr = run
    O, out = replay
    for it, (B, g, parts, _, _) in enumerate(out):
        sc = tr["scalars"][it]
        assert abs(B - sc[0]) <= 1e-10 * abs(B), (it, B, sc[0], parts)
        gg = tr["grad"][it].ravel()
        assert np.abs(gg - g.ravel()).max() <= 1e-9 * np.abs(g).max(), it
        assert abs(np.linalg.norm(gg) - sc[1]) <= 1e-12 * sc[1]
        kinds = set(tr["contacts"][it][:, 0].tolist())
        assert (parts.get("pt", 0.0) > 0.0) == (4 in kinds) and (parts.get("ee", 0.0) > 0.0) == (5 in kinds)
        if it > 0:
            assert parts["elastic"] > 0.0 and parts["bend"] > 0.0
    assert abs(out[0][0] - st["energy0"]) <= 1e-10 * out[0][0]


def test_newton_direction_meets_cg_contract(run, replay):
    vs, fs, vin, fin, st, tr = run
    O, out = replay
    P = tr["params"]
    for it, (B, g, _, H, _) in enumerate(out):
        p = tr["dir"][it].ravel()
        gg = g.ravel()
        assert gg @ p < 0, it
        res = np.linalg.norm(H @ p + gg) / np.linalg.norm(gg)
        if tr["scalars"][it][2] < P["cg_max"]:
            assert res <= 1.05 * P["cg_tol"], (it, res)


def test_accd_bound_and_line_search(run, replay, oracle):
    from oracle import project_ref as PR
    vs, fs, vin, fin, st, tr = run
    O, out = replay
    P = tr["params"]
    dhat = P["dhat"]
    n = len(tr["X"])
    for it in range(n):
        X, p = tr["X"][it], tr["dir"][it]
        B0, tmax, alpha, B1, acc, tries = tr["scalars"][it][[0, 3, 4, 5, 6, 7]]
        ptq, eeq = PR.swept_pairs(X, p, fs, dhat)
        t_ref = min(PR.accd(X, p, ptq, False, 0.1 * dhat).min(initial=1.0),
                    PR.accd(X, p, eeq, True, 0.1 * dhat).min(initial=1.0))
        assert abs(t_ref - tmax) <= 1e-9 * max(t_ref, 1e-300), (it, t_ref, tmax)
        a = min(1.0, 0.9 * tmax)
        for _ in range(int(tries) - 1):
            a *= 0.5
        assert a == alpha, it
        assert acc == 1.0, it
        Xn = X + alpha * p
        if it + 1 < n:
            assert np.array_equal(Xn.view(np.uint64), tr["X"][it + 1].view(np.uint64)), it
        cont = PR.contacts(Xn, fs, dhat)
        b1 = O.energy(Xn, tr["targets"][it], tr["m2s"][it], tr["samples"], cont)
        assert abs(b1 - B1) <= 1e-10 * abs(b1), (it, b1, B1)
        assert B1 < B0, it
        assert len(oracle.self_intersections(Xn, fs)) == 0, it
