"""compute-sanitizer target: one small UDF -> DMC -> QEM pass (noisy icosphere-4, R=64, 600 faces)
plus a self-intersection detection and the stepwise QEM API, exercising every hot-path kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05595_b200 import api, fixtures as FX  # noqa: E402

v, f = FX.icosphere(4)
R = 64
v, _ = FX.normalize_unit_cube(v * (1.0 + 0.01 * FX.Rng(1).normal(len(v)))[:, None], 6.0 / R)
m = api.DeviceMesh.upload(v, f)
out, st, tm = api.remesh_device(m, R, 600)
print("remesh", out.size(), st["iterations"], st["undo_hist"][:3])
print("pairs", len(api.detect_self_intersections(out)))
sv, sf = FX.nested_shells(2, 0.01, 3, 7)
o2, s2 = api.simplify_to(api.DeviceMesh.upload(sv, sf), 200)
print("shells", o2.size(), s2["max_undo_rounds"])
