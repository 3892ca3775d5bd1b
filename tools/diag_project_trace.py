"""Print the per-iteration scalars of the stage-3 step-oracle fixtures (tests/test_gpu_project_steps.py):
B0, |g|, CG iterations, ACCD t_max, alpha, B1, accepted, line-search tries."""
import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_2509_05595_b200 import api
from test_gpu_project_steps import ITERS, CASES
np.set_printoptions(linewidth=200, precision=6)
for name, make in sorted(CASES.items()):
    vs, fs, vin, fin = make()
    m = api.DeviceMesh.upload(vs, fs)
    st, tr = api.safe_project_traced(m, (vin, fin), ITERS, iterations=ITERS)
    print(name, st)
    print(tr["scalars"])
    print([len(c) for c in tr["contacts"]])
