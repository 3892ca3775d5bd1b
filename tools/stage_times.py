"""Per-stage GPU timings of the pipeline on the BASELINE configs (diagnostic)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2509_05595_b200 import api, fixtures as FX

for name in sys.argv[1:] or ["c1", "c2", "c3"]:
    t0 = time.time()
    v, f, R, target = FX.make_config(name)
    tg = time.time() - t0
    m = api.DeviceMesh.upload(v, f)
    for rep in range(3):
        out, st, tm = api.remesh_device(m, R, target)
        nv, nf = out.size()
        print(name, f"gen {tg:.1f}s F={len(f)} R={R}", {k: round(x, 3) if isinstance(x, float) else x for k, x in tm.items()},
              "out", nf, "iters", st["iterations"], "undo", st["undo_hist"][:4], "maxround", st["max_undo_rounds"], flush=True)
