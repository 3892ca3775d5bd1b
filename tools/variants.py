import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2509_05595_b200 import api, fixtures as FX
R = 512
for scale, spread in [((0.06, 0.2), (0.2, 0.8)), ((0.04, 0.12), (0.08, 0.92)), ((0.05, 0.15), (0.1, 0.9)), ((0.03, 0.09), (0.06, 0.94))]:
    v, f = FX.soup(100, 10000, seed=3, scale=scale, spread=spread)
    v, f = FX.inject_defects(v, f, seed=3)
    f = f[:1_000_000]
    v, _ = FX.normalize_unit_cube(v, 6.0 / R)
    g = api.compute_sdf((v, f), R)
    m = api.extract(g)
    nv, nf = m.size()
    chi = nv - nf * 3 // 2 + nf
    t0 = time.time()
    m2, st = api.simplify_to(m, 50000)
    print(scale, spread, "dmc", nv, nf, "chi", chi, "-> faces", m2.size()[1], "iters", st["iterations"], "t", round(time.time() - t0, 2), flush=True)
