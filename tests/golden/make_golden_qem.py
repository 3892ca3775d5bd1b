"""Generates tests/golden/ref_qem_{c2,c3}.json: the ORACLE's full stage-2 run (simplify_to,
SPEC.md:539-547, with the undo loop of SPEC.md:530-538) on the oracle's own stage-1 output for the
BASELINE configs C2 (200k-tri soup, R=256, target 20k) and C3 (1M-tri soup, R=512, target 50k).

The oracle (oracle/src, test infrastructure) is the CPU restatement of the reference algorithm;
its UDF/DMC are bit-identical to the CUDA path (tests/test_gpu_full_size.py), so the QEM input
is identical on both sides.  These runs take minutes of host CPU (C3: ~10 min on 8 cores), too
long for every GPU test session, so the GPU tests compare against this committed record:

    per_iter_collapses   successful collapses per iteration (the collapse-set sequence)
    undo_hist            batches needing k undo rounds
    iterations, nf_out, nv_out, face_iterations, collapses, undone, link_failures
    faces_sha256 / vertices_sha256   output IndexedMesh bytes (i32 faces, f64 vertex bits)
    stage_seconds        measured wall time of each oracle stage here, with the core count

    python tests/golden/make_golden_qem.py [c2] [c3]
"""
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle as O  # noqa: E402
from paper_2509_05595_b200 import fixtures as FX  # noqa: E402


def sha(a) -> str:
    import numpy as np
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(name: str) -> dict:
    v, f, R, target = FX.make_config(name)
    t0 = time.time()
    _, sdf = O.compute_udf_sdf(v, f, R)
    t1 = time.time()
    d = O.dmc_extract(sdf, R)
    t2 = time.time()
    vo, fo, st = O.simplify(d["vertices"], d["faces"], target)
    t3 = time.time()
    per = [int(x) for x in st.pop("per_iter_collapses")]
    out = dict(config=name, R=R, target=target, faces_in=int(len(f)), dmc_faces=int(len(d["faces"])),
               dmc_vertices=int(len(d["vertices"])), dmc_faces_sha256=sha(d["faces"]),
               dmc_vertices_sha256=sha(d["vertices"]), **st, per_iter_collapses=per,
               faces_sha256=sha(fo), vertices_sha256=sha(vo),
               stage_seconds=dict(udf=t1 - t0, dmc=t2 - t1, qem=t3 - t2), cores=os.cpu_count())
    return out


if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if a in ("c2", "c3")] or ["c2", "c3"]
    for n in names:
        r = run(n)
        with open(os.path.join(HERE, f"ref_qem_{n}.json"), "w") as fh:
            json.dump(r, fh, indent=1)
        print(n, r["nf_out"], r["iterations"], r["undo_hist"], r["stage_seconds"], flush=True)
