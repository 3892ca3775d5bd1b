"""The stage-3 step oracle (oracle/project_ref.py) against SPEC.md's own examples for the energy
terms, the barrier, the contact rule and ACCD, before it is trusted as the
checker of the GPU trace (tests/test_gpu_project_steps.py).  CPU only."""
import numpy as np
import pytest

from oracle import project_ref as PR

PARAMS = dict(samples=4, seed=1, kdis=1e3, kelas=0.1, kbend=0.01, kbar=1e2, dhat=1e-3, elas_tau=1e-12,
              elas_power=1, refresh=10, cg_tol=1e-3, cg_max=1000)


def _oracle(X0, F):
    return PR.StepOracle(X0, F, X0, F, PARAMS)


def _parts(O, X):
    m2s = np.zeros((0, 4), np.int32)
    return O.energy_grad(X, X, m2s, np.zeros((0, 3)), np.zeros((0, 6), np.int64))[2]


def test_elastic_stretch_and_rigid_invariance():
    X0 = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    F = np.array([[0, 1, 2]])
    O = _oracle(X0, F)
    lam = 1.3
    p = _parts(O, X0 * lam)
    # F^T F = lam^2 I -> |F^T F - I|_F = sqrt(2) (lam^2 - 1); E = 1/4 A0 k_elas |.|
    assert p["elastic"] == pytest.approx(0.25 * 0.5 * 0.1 * np.sqrt(2) * (lam * lam - 1), rel=1e-12)
    c, s = np.cos(0.7), np.sin(0.7)
    Rm = np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])
    assert _parts(O, X0 @ Rm.T + [3, -2, 1])["elastic"] <= 1e-10


def test_bending_hinge_known_answer():
    # two unit right triangles sharing the edge (0, 1), flat at rest
    X0 = np.array([[0, 0, 0], [1, 0, 0], [0.5, 1, 0], [0.5, -1, 0]], float)
    F = np.array([[0, 1, 2], [1, 0, 3]])
    O = _oracle(X0, F)
    assert len(O.rest["hinges"]) == 1 and abs(O.rest["theta0"][0]) < 1e-15
    th = 0.3
    X = X0.copy()
    X[3] = [0.5, -np.cos(th), np.sin(th)]  # rotate the second wing about the hinge by th
    got = _parts(O, X)["bend"]
    assert got == pytest.approx(0.5 * 0.01 * 1.0 * th * th, rel=1e-12)


def test_barrier_half_dhat():
    dhat = PARAMS["dhat"]
    X0 = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.2, 0.2, 0.5 * dhat]], float)
    F = np.array([[0, 1, 2]])
    O = PR.StepOracle(X0[:3], F, X0[:3], F, PARAMS)
    O.nv = 4
    O.t["s0"] = PR.torch.zeros(4, dtype=PR.torch.float64)
    cont = PR.contacts(X0, F, dhat)
    assert cont.tolist() == [[PR.PT, 6, 3, 0, 1, 2]]
    B, _, parts = O.energy_grad(X0, X0, np.zeros((0, 4), np.int32), np.zeros((0, 3)), cont)
    # b(d̂/2) = (d̂^2 / 4) ln 2
    assert parts["pt"] == pytest.approx(PARAMS["kbar"] * dhat * dhat / 4 * np.log(2), rel=1e-12)


def test_contacts_exclude_shared_vertices_and_far_pairs():
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    F = np.array([[0, 1, 2], [0, 1, 3]])  # two faces sharing an edge: no contact pairs
    assert len(PR.contacts(X, F, 1e-3)) == 0
    X2 = np.concatenate([X[:3], X[:3] + [0, 0, 5e-4]])
    F2 = np.array([[0, 1, 2], [3, 5, 4]])  # parallel plates 5e-4 apart
    c = PR.contacts(X2, F2, 1e-3)
    assert set(c[:, 0].tolist()) == {PR.PT, PR.EE}
    assert len(PR.contacts(X2 * [1, 1, 4], F2, 1e-3)) == 0  # 2e-3 apart


def test_accd_parallel_plates():
    g = 5e-4
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, g], [1, 0, g], [0, 1, g]], float)
    F = np.array([[0, 1, 2], [3, 5, 4]])
    p = np.zeros_like(X)
    p[3:, 2] = -2 * g  # the top plate would pass through the bottom one at t = 1/2
    ptq, eeq = PR.swept_pairs(X, p, F, 1e-3)
    t = min(PR.accd(X, p, ptq, False, 1e-4).min(), PR.accd(X, p, eeq, True, 1e-4).min(initial=1.0))
    assert 0 < t < 0.5
    # the gap after the bounded step stays positive
    assert g - 2 * g * t > 0


def test_gradient_matches_finite_differences():
    from paper_2509_05595_b200 import fixtures as FX
    v, f = FX.icosphere(1)
    rng = np.random.default_rng(0)
    X = v + 0.01 * rng.normal(size=v.shape)
    O = PR.StepOracle(v, f.astype(np.int64), v, f.astype(np.int64), PARAMS)
    tg = v * 1.01
    m2s = np.zeros((0, 4), np.int32)
    B, g, _ = O.energy_grad(X, tg, m2s, np.zeros((0, 3)), np.zeros((0, 6), np.int64))
    h = 1e-6
    for i, k in [(0, 0), (5, 1), (11, 2)]:
        Xp, Xm = X.copy(), X.copy()
        Xp[i, k] += h
        Xm[i, k] -= h
        fd = (O.energy(Xp, tg, m2s, np.zeros((0, 3)), np.zeros((0, 6))) -
              O.energy(Xm, tg, m2s, np.zeros((0, 3)), np.zeros((0, 6)))) / (2 * h)
        assert g[i, k] == pytest.approx(fd, rel=1e-5, abs=1e-8)
    H = O.hessian_spd(X, tg, m2s, np.zeros((0, 3)), np.zeros((0, 6), np.int64))
    assert abs(H - H.T).max() <= 1e-12 * abs(H).max()
    assert np.linalg.eigvalsh(H.toarray()).min() > 0
