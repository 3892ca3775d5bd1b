import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2509_05595_b200 import api, fixtures as FX
R = 16
rng = FX.Rng(7)
s = (rng.uniform((R + 1) ** 3) * 2 - 1).astype(np.float32).reshape(R + 1, R + 1, R + 1)
g = api.DeviceGrid.upload(s, R)
m = api.extract(g)
print("full", m.size(), flush=True)
gs = api.DeviceGrid.slab_upload(s[0:11], R, 0)
m2, a, b = api.extract_slab(gs, 0, 9)
print("slab", m2.size(), a, b, flush=True)
