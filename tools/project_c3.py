"""Stage-3 timing on a config's pipeline output (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05595_b200 import api, fixtures as FX
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
v, f, R, target = FX.make_config(name)
out = api.run_pipeline(v, f, R, target)
m = api.DeviceMesh.upload(out.vertices, out.faces)
inp = api.DeviceMesh.upload(v, f)
t = time.time()
s = api.safe_project(m, inp)
dt = time.time() - t
pv, pf = m.download()
c0, c1 = api.chamfer((out.vertices, out.faces), inp, 16384, 3), api.chamfer((pv, pf), inp, 16384, 3)
print(name, len(out.faces), s, "CD %.3e -> %.3e" % (c0, c1), "isect", len(api.detect_self_intersections((pv, pf))),
      "%.2fs" % dt, flush=True)
