"""Builds the sm_100a shared library `libpamopt_cu.so` in-tree with nvcc.

Every translation unit is compiled with `--fmad=false` (no FMA contraction: the FP64
decision arithmetic must round exactly like the pinned scalar formulas),
`-lineinfo` (ncu source attribution) and `-gencode arch=compute_100a,code=sm_100a`.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpamopt_cu.so")
OBJ = os.path.join(HERE, "build_obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
SOURCES = ["capi.cu", "udf.cu", "dmc.cu", "isect.cu", "simplify.cu", "metrics.cu", "ingest.cu", "project.cu",
           "slab_nccl.cu", "ingest_text.cu"]


def _stale(src_files, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_files)


def build(verbose: bool = False, force: bool = False, defines=(), tag: str = "") -> str:
    """defines/tag: an A/B variant (-D flags) built into build_obj/<tag>/ and libpamopt_cu_<tag>.so;
    select it at run time with PAMOPT_LIB=<path> (experiments only)."""
    out = OUT if not tag else OUT.replace(".so", f"_{tag}.so")
    obj_dir = OBJ if not tag else os.path.join(OBJ, tag)
    os.makedirs(obj_dir, exist_ok=True)
    extra = [f"-D{d}" for d in defines]
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    headers.append(os.path.join(HERE, "..", "include", "pamopt_cu.h"))
    objs = []
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(obj_dir, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale([src] + headers, obj):
            jobs.append([NVCC, *FLAGS, *extra, "-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr, file=sys.stderr)

    with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs) or 1)) as ex:
        list(ex.map(run, jobs))
    if jobs or _stale(objs, out):
        run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs, "-lcudart", "-ldl"])
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    tags = [a[6:] for a in sys.argv[1:] if a.startswith("--tag=")]
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, defines=defs, tag=tags[0] if tags else ""))
