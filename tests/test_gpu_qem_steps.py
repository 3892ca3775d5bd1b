"""SPEC-granular stage-2 operations through the C-ABI, each against the
oracle (and the reference's own link condition, tests/golden/ref_link*.npz):

  quadrics, edge_cost, pack_cost, link_condition_holds (unbounded valence),
  and Algorithm 1 one step at a time (pamopt_cu_qem_*: prepare -> propagate_and_mark ->
  collapse_batch -> undo_loop -> end_iteration), compared array for array with the oracle's
  record of the same iteration (oracle.simplify_trace)."""
import os

import numpy as np
import pytest

from paper_2509_05595_b200 import fixtures as FX

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def noisy_sphere(sub=3, seed=1):
    v, f = FX.icosphere(sub)
    return v * (1.0 + 0.01 * FX.Rng(seed).normal(len(v)))[:, None], f


def edges_of(f):
    e = np.sort(np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]]), axis=1)
    return np.unique(e, axis=0).astype(np.int32)


def u64(a):
    return np.ascontiguousarray(a).view(np.uint64)


def test_quadrics_and_edge_cost_match_oracle(api, oracle):
    v, f = noisy_sphere(3)
    assert np.array_equal(u64(api.quadrics((v, f))), u64(oracle.quadrics(v, f)))
    e = edges_of(f)
    gc, gp = api.edge_cost((v, f), e)
    oc, op = oracle.edge_cost(v, f, e)
    assert np.array_equal(u64(gc), u64(oc)) and np.array_equal(u64(gp), u64(op))


def test_pack_cost_spec_examples(api):
    # pack(0, 0) = 0; cost ties broken by the id; monotone in the cost
    assert api.pack_cost([0.0], [0])[0] == 0
    k = api.pack_cost([1.5, 1.5], [3, 7])
    assert k[0] < k[1]
    assert api.pack_cost([-2.0], [5])[0] == 5  # negative clamps to 0
    rng = np.random.default_rng(7)
    c = np.concatenate([rng.exponential(1.0, 500_000), rng.uniform(0, 1e-30, 250_000), rng.uniform(0, 1e30, 250_000)])
    ids = rng.integers(0, 2**32, len(c), dtype=np.uint64).astype(np.uint32)
    keys = api.pack_cost(c, ids)
    ref = (np.float32(c).view(np.uint32).astype(np.uint64) << np.uint64(32)) | ids.astype(np.uint64)
    assert np.array_equal(keys, ref)
    a, b = c[0::2], c[1::2]  # 10^6 random values -> 5e5 pairs: float order <=> key order
    ka, kb = keys[0::2] >> np.uint64(32), keys[1::2] >> np.uint64(32)
    fa, fb = np.float32(a), np.float32(b)
    assert np.all((fa < fb) == (ka < kb)) and np.all((fa == fb) == (ka == kb))
    with pytest.raises(api._lib.PamoptError):
        api.pack_cost([1.0, float("nan")], [0, 1])


@pytest.mark.parametrize("golden", ["ref_link.npz", "ref_link_valence.npz"])
def test_link_condition_matches_reference(api, golden):
    g = np.load(os.path.join(GOLD, golden))
    names = sorted({k.rsplit("_", 1)[0] for k in g.files})
    for n in names:
        got = api.link_condition((g[f"{n}_v"], g[f"{n}_f"]), g[f"{n}_e"])
        assert np.array_equal(got, g[f"{n}_r"].astype(bool)), n


def test_link_condition_unknown_edge_raises(api):
    v, f = noisy_sphere(1)
    known = {tuple(e) for e in edges_of(f).tolist()}
    b = next(j for j in range(1, len(v)) if (0, j) not in known)
    with pytest.raises(api._lib.PamoptInvalidArgument):
        api.link_condition((v, f), [[0, b]])


def test_high_valence_simplify_matches_oracle(api, oracle):
    """A 1000-valent apex pair (no fixed per-thread capacity remains)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("mgv", os.path.join(GOLD, "make_golden_valence.py"))
    mgv = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mgv)
    v, f = mgv.bipyramid(1000)
    vo, fo, st = oracle.simplify(v, f, 200)
    out, gs = api.simplify_to(api.DeviceMesh.upload(v, f), 200)
    gv, gf = out.download()
    assert np.array_equal(gs["per_iter_collapses"], st["per_iter_collapses"])
    assert np.array_equal(gf, fo) and np.array_equal(u64(gv), u64(vo))


def step_compare(api, oracle, v, f, target, iters):
    """Runs the GPU step API for max(iters) iterations and compares each listed iteration with the
    oracle's record of it."""
    m = api.DeviceMesh.upload(v, f)
    q = api.QemRun(m, target)
    seen = 0
    for it in range(1, max(iters) + 1):
        assert not q.done()
        ne = q.prepare()
        e = q.edges()
        nm = q.propagate_and_mark()
        ids, fkeys = q.marked()
        ok = q.collapse_batch()
        rounds, napplied, applied = q.undo_loop()
        X, F, falive = q.state_mesh()
        q.end_iteration()
        if it not in iters:
            continue
        t = oracle.simplify_trace(v, f, target, it)
        assert ne == len(t["edges"]) and np.array_equal(e["edges"], t["edges"]), it
        assert np.array_equal(e["keys"], t["keys"]), it
        valid = t["keys"] != np.uint64(2**64 - 1)
        assert np.array_equal(u64(e["place"][valid]), u64(t["place"][valid])), it
        assert np.array_equal(fkeys, t["face_keys"]), it
        order = np.argsort(ids)  # GPU lists marked edges in key order, the oracle in id order
        assert nm == len(t["marked"]) and np.array_equal(ids[order].astype(np.int64), t["marked"]), it
        assert np.array_equal(ok[order], t["link_ok"]), it
        assert np.array_equal(np.sort(ids[applied.astype(bool)]).astype(np.int64), t["applied"]), it
        assert rounds == t["rounds"], it
        assert np.array_equal(falive, t["falive"]) and np.array_equal(F, t["F"]) and np.array_equal(u64(X), u64(t["X"]))
        seen += 1
    assert seen == len(iters)
    q.close()


def test_qem_steps_match_oracle_trace(api, oracle):
    v, f = noisy_sphere(4)
    step_compare(api, oracle, v, f, 300, [1, 2, 4])


def test_qem_steps_with_undo_rounds_match_oracle_trace(api, oracle):
    v, f = FX.nested_shells(3, 0.01, 3, 7)
    t = [oracle.simplify_trace(v, f, 150, it)["rounds"] for it in (4, 11, 28)]
    assert t == [1, 2, 3]  # one, two and three undo rounds
    step_compare(api, oracle, v, f, 150, [4, 11, 28])


def test_qem_step_loop_equals_simplify_to(api):
    v, f = noisy_sphere(4)
    m = api.DeviceMesh.upload(v, f)
    q = api.QemRun(m, 500)
    while not q.done():
        q.prepare()
        q.propagate_and_mark()
        q.collapse_batch()
        q.undo_loop()
        q.end_iteration()
    st = q.finish()
    q.close()
    sv, sf = m.download()
    out, gs = api.simplify_to(api.DeviceMesh.upload(v, f), 500)
    gv, gf = out.download()
    assert np.array_equal(sf, gf) and np.array_equal(u64(sv), u64(gv))
    assert st["undo_hist"] == gs["undo_hist"] and st["iterations"] == gs["iterations"]
