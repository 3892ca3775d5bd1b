"""Driver for ncu captures: one device-resident pipeline pass of a config (default c2)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05595_b200 import api, fixtures as FX
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
v, f, R, target = FX.make_config(name)
m = api.DeviceMesh.upload(v, f)
out, st, tm = api.remesh_device(m, R, target)
print(name, tm, st["iterations"])
