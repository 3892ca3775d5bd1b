"""ncu CSV (gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum of one UDF pass,
tools/udf_only.py) -> profiles/<round>_udf_traffic_<cfg>.json, read by bench.py as roofline.traffic.
usage: udf_traffic.py <ncu.csv> <cfg> <out.json>"""
import collections
import csv
import json
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2509_05595_b200 import fixtures as FX  # noqa: E402

src, cfg, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = collections.defaultdict(lambda: collections.defaultdict(float))
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    try:
        val = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    name = r[ki].split("(")[0].split("::")[-1]
    per[name][r[mi]] += val
v, f, R, _ = FX.make_config(cfg)
rd = sum(m["dram__bytes_read.sum"] for m in per.values())
wr = sum(m["dram__bytes_write.sum"] for m in per.values())
res = {"source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, "
                 f"python tools/udf_only.py {cfg} (one {cfg.upper()} UDF pass)",
       "stage": "udf", "config": cfg.upper(), "dram_bytes": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
       "kernel_ns_sum": int(sum(m["gpu__time_duration.sum"] for m in per.values())),
       "algorithmic_bytes": int(4 * (R + 1) ** 3 + 36 * len(f)),
       "per_kernel": {k: {mk: int(mv) for mk, mv in m.items()} for k, m in per.items()}}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: res[k] for k in ("dram_bytes", "kernel_ns_sum", "algorithmic_bytes")}))
