"""Aggregate an ncu --csv launch list by kernel (gpu__time_duration.sum, and the DRAM bytes when
the capture has dram__bytes_{read,write}.sum):

    python tools/agg_launches.py <csv or csv.gz> [top] [--json out.json]

The JSON form (per kernel: ms, launches, dram bytes; per stage totals) is what bench.py reads as
the ncu traffic of each stage (profiles/r02_stage_traffic_c3.json)."""
import collections
import csv
import gzip
import json
import sys

# kernel -> pipeline stage (the stage that launches it in remesh_device)
UDF = {"k_prep", "k_level0", "k_refine", "k_brick_count", "k_brick_scatter", "k_brick_items", "k_make_items",
       "k_brick", "k_finalize", "k_validate"}
DMC = {"k_classify_count", "k_classify_write", "k_patch_count", "k_patch_vertices", "k_quad_count", "k_quad_write",
       "k_own_split", "k_pack_signs"}


def stage_of(name: str, seen_qem: bool) -> str:
    if name in UDF:
        return "udf"
    if name in DMC:
        return "dmc"
    if not seen_qem and ("scan" in name or "Scan" in name):
        return "udf_dmc_scan"
    return "qem"


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as fh:
        rows = list(csv.reader(fh))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            val = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].replace("<unnamed>", "anon").replace("(anonymous namespace)", "anon")
        name = name.split("(")[0].split("::")[-1].strip()
        rec = launches.setdefault(r[ii], {"kernel": name})
        rec[r[mi]] = val
    return list(launches.values())


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 25
    L = load(path)
    agg = collections.defaultdict(lambda: {"ns": 0.0, "launches": 0, "dram": 0.0})
    stages = collections.defaultdict(lambda: {"ns": 0.0, "dram": 0.0, "launches": 0})
    seen_qem = False
    for r in L:
        k = r["kernel"]
        a = agg[k]
        ns = r.get("gpu__time_duration.sum", 0.0)
        dram = r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
        a["ns"] += ns
        a["launches"] += 1
        a["dram"] += dram
        st = stage_of(k, seen_qem)
        if k in ("k_deg", "k_quadrics"):
            seen_qem = True
            st = "qem"
        s = stages[st]
        s["ns"] += ns
        s["dram"] += dram
        s["launches"] += 1
    tot = sum(a["ns"] for a in agg.values())
    print(f"total {tot / 1e6:.2f} ms, {len(L)} launches")
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["ns"])[:top]:
        print(f"{a['ns'] / 1e6:9.3f} ms {a['launches']:6d}  {a['dram'] / 1e6:10.1f} MB  {k}")
    for s, v in stages.items():
        print(f"stage {s}: {v['ns'] / 1e6:.2f} ms, {v['dram'] / 1e6:.1f} MB DRAM, {v['launches']} launches")
    if "--json" in sys.argv:
        out = sys.argv[sys.argv.index("--json") + 1]
        with open(out, "w") as fh:
            json.dump({"source": path, "note": "ncu --clock-control none, serialised cold-cache launches",
                       "stages": {s: {"ms": round(v["ns"] / 1e6, 3), "dram_bytes": int(v["dram"]),
                                      "launches": v["launches"]} for s, v in stages.items()},
                       "kernels": {k: {"ms": round(a["ns"] / 1e6, 3), "launches": a["launches"],
                                       "dram_bytes": int(a["dram"])} for k, a in agg.items()}}, fh, indent=1)


if __name__ == "__main__":
    main()
