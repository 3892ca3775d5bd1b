import faulthandler, sys, time, os
faulthandler.dump_traceback_later(45, repeat=True)
sys.path.insert(0, os.getcwd())
t0 = time.time()
def log(*a):
    print(f"[{time.time()-t0:7.2f}]", *a, flush=True)
from paper_2509_05595_b200 import api, fixtures as FX
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
v, f, R, target = FX.make_config(name)
log("fixture", len(f))
m = api.DeviceMesh.upload(v, f); log("upload")
g = api.compute_sdf(m, R); api.default_context().synchronize(); log("sdf")
d = api.extract(g); log("extract", d.size())
dv, df = d.download(); log("download")
out, st = api.simplify_to(d, target); log("simplify", st["iterations"], out.size())
