"""PAMOPT_PROFILE phase / per-kernel breakdown for one C5 mesh (index) or a config (c1..c3); two\npasses, the second one warm."""
import os, sys
os.environ["PAMOPT_PROFILE"] = os.environ.get("PAMOPT_PROFILE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05595_b200 import api, fixtures as FX
arg = sys.argv[1] if len(sys.argv) > 1 else "13"
if arg.startswith("c"):
    i = arg
    v, f, R, target = FX.make_config(arg)
else:
    i = int(arg)
    v, f, R, target = FX.c5_batch(i + 1)[i]
ctx = api.Context(0)
for rep in range(2):  # the first pass pays the lazy module loads; read the second report
    d = api.DeviceMesh.upload(v, f, ctx)
    out, st, tm = api.remesh_device(d, R, target)
    print(i, rep, st["iterations"], tm, flush=True)
