"""Stage-3 kernel-time breakdown on a config's pipeline output (PAMOPT_PROFILE=2 style, via the ctx API)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05595_b200 import api, fixtures as FX
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
v, f, R, target = FX.make_config(name)
out = api.run_pipeline(v, f, R, target)
ctx = api.default_context()
m = api.DeviceMesh.upload(out.vertices, out.faces, ctx)
inp = api.DeviceMesh.upload(v, f, ctx)
ctx.profile(True)
t = time.time()
s = api.safe_project(m, inp, iterations=10)
dt = time.time() - t
kt = ctx.kernel_times()
ctx.profile(False)
tot = sum(ms for ms, _ in kt.values())
print(name, "wall %.2fs kernels %.2fs" % (dt, tot / 1e3), s)
for k, (ms, n) in sorted(kt.items(), key=lambda kv: -kv[1][0])[:15]:
    print("  %-28s %9.1f ms %7d" % (k, ms, n))
