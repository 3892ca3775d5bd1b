import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2509_05595_b200 import api, fixtures as FX
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
v, f, R, target = FX.make_config(name)
g = api.compute_sdf((v, f), R)
m = api.extract(g)
dv, df = m.download()
print("dmc", dv.shape, df.shape, flush=True)
t0 = time.time(); pr = api.detect_self_intersections((dv, df)); print("dmc isect", len(pr), time.time() - t0, pr[:10], flush=True)
if len(pr):
    for a, b in pr[:5]:
        print(a, b, df[a], df[b], dv[df[a]].tolist(), dv[df[b]].tolist())
np.savez_compressed("gpurun_out/dmc_%s_pairs.npz" % name, pairs=pr)
m2, st = api.simplify_to((dv, df), target)
print({k: v for k, v in st.items() if k != "per_iter_collapses"})
pc = st["per_iter_collapses"]
print("per-iter", pc[:30].tolist(), pc[-30:].tolist())
