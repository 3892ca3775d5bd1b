"""Per-mesh timing/stats of the C5 batch (diagnostic)."""
import sys, time, json
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_05595_b200 import api, fixtures as FX

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
meshes = FX.c5_batch(n)
ctx = api.Context(0)
tot = 0
for i, (v, f, R, target) in enumerate(meshes):
    d = api.DeviceMesh.upload(v, f, ctx)
    out, st, tm = api.remesh_device(d, R, target); out.free()
    torch.cuda.synchronize()
    t = time.perf_counter()
    out, st, tm = api.remesh_device(d, R, target)
    ctx.synchronize()
    dt = (time.perf_counter() - t) * 1e3
    tot += dt
    print(i, i % 3, "F", len(f), "R", R, "target", target, "dmcF", tm["dmc_faces"], "out", out.size()[1],
          "iters", st["iterations"], "undo", st.get("undo_hist"), "ms %.1f" % dt, {k: round(tm[k], 1) for k in ("udf_ms", "dmc_ms", "simplify_ms")}, flush=True)
    out.free(); d.free()
print("total ms", tot)
