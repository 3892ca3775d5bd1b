"""run_pipeline through the C-ABI: normalise -> stage 1 -> certify -> stage 2 ->
certify -> [stage 3 -> certify] -> denormalise, plus SPEC acceptance criteria #1 and #4 on the
generated 20-fixture defect corpus: 100% manifold, watertight and exact-check
intersection-free outputs at R in {64, 128} with a 1% face target, and the undo-round statistics
of every simplification batch."""
import numpy as np
import pytest

from paper_2509_05595_b200 import fixtures as FX

pytestmark = pytest.mark.gpu


def u64(a):
    return np.ascontiguousarray(a).view(np.uint64)


def test_run_pipeline_equals_stagewise(api):
    v, f = FX.icosphere(5)
    v = v * (1.0 + 0.01 * FX.Rng(1).normal(len(v)))[:, None] * 3.0 + np.array([1.0, -2.0, 0.5])
    R, target = 128, 5000
    out, rep = api.run_certified_pipeline((v, f), target_faces=target, resolution=R)
    assert rep["failed_stage"] == 0 and rep["resolution"] == R and rep["target_faces"] == target
    for s in rep["stages"]:
        assert s["manifold"] and s["watertight"] and s["intersection_free"]
    assert rep["stages"][1]["n_faces"] <= target
    # the same computation stage by stage through the public API
    m = api.DeviceMesh.upload(v, f)
    scale, t = api.normalize_unit_cube(m, 6.0 / R)
    o2, _, _ = api.remesh_device(m, R, target)
    api.denormalize(o2, scale, t)
    a_v, a_f = out.download()
    b_v, b_f = o2.download()
    assert np.array_equal(a_f, b_f) and np.array_equal(u64(a_v), u64(b_v))
    assert rep["scale_translation"] == [scale, *t]


def test_run_pipeline_auto_resolution_and_ratio(api):
    v, f = FX.icosphere(4)
    out, rep = api.run_certified_pipeline((v, f), target_ratio=0.05)  # 5120 faces -> target 256
    assert rep["target_faces"] == 256 and rep["resolution"] == 128  # target < 1000
    # two offset shells 1.8 voxels apart: the undo loop can stall above the target
    assert rep["stages"][1]["n_faces"] <= 256 or rep["stalled"]


def test_run_pipeline_with_projection(api):
    v, f = FX.icosphere(4)
    v = v * (1.0 + 0.02 * FX.Rng(3).normal(len(v)))[:, None]
    out, rep = api.run_certified_pipeline((v, f), target_faces=600, resolution=64, run_projection=True)
    assert len(rep["stages"]) == 3 and rep["stages"][2]["intersection_free"]
    assert rep["stages"][2]["n_faces"] == rep["stages"][1]["n_faces"]  # connectivity unchanged
    assert rep["stages"][2]["cd"] <= rep["stages"][1]["cd"]


def test_defect_corpus_acceptance(api):
    """SPEC.md:805 #1 (guarantees) and #4 (undo statistics) on 20 defect fixtures, 5k-300k faces."""
    hist = np.zeros(8, np.int64)
    for i, (v, f, R, target) in enumerate(FX.defect_corpus(20)):
        out, rep = api.run_certified_pipeline((v, f), target_faces=target, resolution=R, report_samples=4096)
        assert rep["failed_stage"] == 0, i
        for s in rep["stages"]:
            assert s["manifold"] and s["watertight"] and s["intersection_free"], (i, s)
        assert rep["stages"][1]["n_faces"] <= target or rep["stalled"], i
        hist += np.array(rep["simplify"]["undo_hist"])
    batches = hist.sum()
    assert hist[4:].sum() == 0  # 100% of batches within 3 undo rounds
    frac1 = hist[:2].sum() / batches
    print(f"undo rounds histogram over {batches} batches: {hist[:4].tolist()}, <=1 round: {frac1:.4f}")
