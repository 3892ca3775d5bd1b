"""Stage-3 diagnostics: SPEC example (decimated icosphere projected onto the dense one)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2509_05595_b200 import api, fixtures as FX
for bump in (0.0, 0.05):
    v, f = FX.icosphere(4)
    v = v * (1.0 + bump * np.sin(5 * v[:, :1]) * np.cos(4 * v[:, 1:2]))
    dense = (v, f)
    for target in (600, 2000):
        low, st = api.simplify_to(dense, target)
        lv, lf = low.download()
        m = api.DeviceMesh.upload(lv, lf)
        t = time.time()
        s = api.safe_project(m, dense)
        dt = time.time() - t
        pv, _ = m.download()
        c0, c1 = api.chamfer((lv, lf), dense, 16384, 3), api.chamfer((pv, lf), dense, 16384, 3)
        h0, h1 = api.hausdorff((lv, lf), dense, 16384, 3), api.hausdorff((pv, lf), dense, 16384, 3)
        print("bump", bump, "faces", len(lf), "it", s["iterations"], "cg", s["cg_iterations"], "E %.4g -> %.4g" % (s["energy0"], s["energy"]),
              "CD %.3e -> %.3e HD %.3e -> %.3e" % (c0, c1, h0, h1), "isect", len(api.detect_self_intersections((pv, lf))),
              "%.2fs" % dt, flush=True)

# pipeline case: the stage-2 output sits on the eps-offset surface; stage 3 pulls it back
v, f, R, target = FX.make_config("c1")
out = api.run_pipeline(v, f, R, target)
m = api.DeviceMesh.upload(out.vertices, out.faces)
t = time.time()
s = api.safe_project(m, (v, f))
dt = time.time() - t
pv, _ = m.download()
c0, c1 = api.chamfer((out.vertices, out.faces), (v, f), 16384, 3), api.chamfer((pv, out.faces), (v, f), 16384, 3)
h0, h1 = api.hausdorff((out.vertices, out.faces), (v, f), 16384, 3), api.hausdorff((pv, out.faces), (v, f), 16384, 3)
print("C1 pipeline", len(out.faces), s, "CD %.3e -> %.3e HD %.3e -> %.3e" % (c0, c1, h0, h1),
      "isect", len(api.detect_self_intersections((pv, out.faces))), "%.2fs" % dt, flush=True)
