import sys, os, time
os.environ["PAMOPT_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_05595_b200 import api, fixtures as FX
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
v, f, R, target = FX.make_config(name)
g = api.compute_sdf((v, f), R)
m = api.extract(g)
dv, df = m.download()
t0 = time.time()
m2, st = api.simplify_to((dv, df), target)
print(name, "wall", time.time() - t0, {k: v for k, v in st.items() if k != "per_iter_collapses"}, flush=True)
