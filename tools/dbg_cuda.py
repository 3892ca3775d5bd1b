"""Minimal CUDA liveness probe: torch H2D copy, then the library's context + mesh upload."""
import faulthandler, os, sys, time
faulthandler.dump_traceback_later(30, repeat=True)
sys.path.insert(0, os.getcwd())
t0 = time.time()
def log(*a):
    print(f"[{time.time()-t0:7.2f}]", *a, flush=True)
if "torch" in sys.argv:
    import torch
    x = torch.arange(10, device="cuda"); torch.cuda.synchronize(); log("torch ok", int(x.sum()))
import numpy as np
from paper_2509_05595_b200 import api, _lib
log("lib", _lib.LIB_PATH)
c = api.Context(0); log("ctx")
m = api.DeviceMesh.upload(np.zeros((3, 3)), np.array([[0, 1, 2]], np.int32), c); log("upload")
c.synchronize(); log("sync")
