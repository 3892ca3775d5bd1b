import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2509_05595_b200 import api, fixtures as FX
ms = FX.c5_batch(14)
for i in (4, 13):
    v, f, R, t = ms[i]
    ctx = api.Context(0)
    d = api.DeviceMesh.upload(v, f, ctx)
    out, st, tm = api.remesh_device(d, R, t)
    vo, fo = out.download()
    deg = np.bincount(fo.ravel(), minlength=len(vo))
    print(i, "faces", len(fo), "max deg", deg.max(), "p99", np.percentile(deg, 99), "mean", deg.mean(), "n>32", (deg > 32).sum(), "n>64", (deg>64).sum(), flush=True)
