"""Stage-3 smoke: decimated icosphere projected onto the dense one (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2509_05595_b200 import api, fixtures as FX
v, f = FX.icosphere(4)
v = v * (1.0 + 0.05 * np.sin(5 * v[:, :1]) * np.cos(4 * v[:, 1:2]))   # bumpy target
dense = (v, f)
low, st = api.simplify_to(dense, 600)
lv, lf = low.download()
print("low", lv.shape, lf.shape, flush=True)
cd0 = api.chamfer((lv, lf), dense, 8192, 3)
hd0 = api.hausdorff((lv, lf), dense, 8192, 3)
m = api.DeviceMesh.upload(lv, lf)
t = time.time()
stats = api.safe_project(m, dense, iterations=int(sys.argv[1]) if len(sys.argv) > 1 else 10)
dt = time.time() - t
pv, pf = m.download()
cd1 = api.chamfer((pv, pf), dense, 8192, 3)
hd1 = api.hausdorff((pv, pf), dense, 8192, 3)
print(stats, "time %.2fs" % dt, flush=True)
print("CD %.3e -> %.3e  HD %.3e -> %.3e" % (cd0, cd1, hd0, hd1), "isect", len(api.detect_self_intersections((pv, pf))),
      "moved", float(np.abs(pv - lv).max()), flush=True)
