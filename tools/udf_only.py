"""Driver for UDF-stage ncu captures: one compute_sdf pass of a config (default c3)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05595_b200 import api, fixtures as FX
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
v, f, R, target = FX.make_config(name)
m = api.DeviceMesh.upload(v, f)
g = api.compute_sdf(m, R)
g.download()
print("ok")
