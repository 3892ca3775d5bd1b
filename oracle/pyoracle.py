"""ctypes bindings of the ORACLE — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may
import this module, and only as the checker.  The product package
(paper_2509_05595_b200/) never imports it.

Two shared libraries:
  oracle/liboracle.so          CPU restatement of the hot path (oracle/src, this repo)
  oracle/_ref/libpamopt_ref.so the reference's own translation units compiled in place
                               (oracle/Makefile `ref`); absent on machines without it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        L.orc_set_workers.argtypes = [C.c_int]
        L.orc_hierarchy_pairs.restype = C.c_int64
        L.orc_hierarchy_pairs.argtypes = [f64p, i32p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_int64]
        L.orc_compute_udf_sdf.restype = C.c_int64
        L.orc_compute_udf_sdf.argtypes = [f64p, i32p, C.c_int64, C.c_int, C.c_double, C.c_void_p, C.c_void_p]
        L.orc_brute_udf.argtypes = [f64p, i32p, C.c_int64, C.c_int, f32p]
        L.orc_point_triangle_sq_batch.argtypes = [f64p, f64p, f64p, f64p, C.c_int64, f64p]
        L.orc_det_exp.restype = C.c_double
        L.orc_det_exp.argtypes = [C.c_double]
        L.orc_sigmoid.restype = C.c_double
        L.orc_sigmoid.argtypes = [C.c_double, C.c_double]
        L.orc_dmc_table.argtypes = [i32p]
        L.orc_dmc_patches.argtypes = [C.c_int, C.c_int, i32p]
        L.orc_dmc_extract.argtypes = [f32p, C.c_int, C.c_double, i64p]
        L.orc_dmc_fetch.argtypes = [C.c_void_p] * 5
        L.orc_dmc_stages.argtypes = [C.c_void_p] * 6
        L.orc_dmc_extract_slab.argtypes = [f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, i64p]
        L.orc_tri_tri_pairs.argtypes = [f64p, i32p, i32p, C.c_int64, i32p]
        L.orc_orient3d.restype = C.c_int
        L.orc_orient3d.argtypes = [f64p, f64p, f64p, f64p]
        L.orc_self_intersections.restype = C.c_int64
        L.orc_self_intersections.argtypes = [f64p, C.c_int64, i32p, C.c_int64, C.c_void_p, C.c_int64]
        L.orc_overlap_pairs.restype = C.c_int64
        L.orc_overlap_pairs.argtypes = [f64p, i32p, C.c_int64, C.c_void_p, C.c_int64]
        L.orc_simplify.restype = C.c_int
        L.orc_simplify.argtypes = [f64p, C.c_int64, i32p, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int, i64p]
        L.orc_simplify_fetch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_link_condition.argtypes = [f64p, C.c_int64, i32p, C.c_int64, i32p, C.c_int64, i32p]
        L.orc_simplify_trace.restype = C.c_int
        L.orc_simplify_trace.argtypes = [f64p, C.c_int64, i32p, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int,
                                         C.c_int64, i64p]
        L.orc_trace_fetch.argtypes = [C.c_void_p] * 10
        L.orc_quadrics.argtypes = [f64p, C.c_int64, i32p, C.c_int64, f64p]
        L.orc_edge_cost.argtypes = [f64p, C.c_int64, i32p, C.c_int64, i32p, C.c_int64, C.c_double, C.c_double, f64p, f64p]
        L.orc_topology.argtypes = [i32p, C.c_int64, C.c_int64, i64p]
        L.orc_topology_lists.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_nearest.argtypes = [f64p, i32p, C.c_int64, f64p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_sample.restype = C.c_int
        L.orc_sample.argtypes = [f64p, i32p, C.c_int64, C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_max_corner_cos.restype = C.c_double
        L.orc_max_corner_cos.argtypes = [f64p, i32p, C.c_int64]
        _LIB = L
    return _LIB


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libpamopt_ref.so"))


def ref():
    global _REF
    if _REF is None:
        L = C.CDLL(os.path.join(HERE, "_ref", "libpamopt_ref.so"))
        L.ref_set_workers.argtypes = [C.c_int]
        L.ref_point_triangle_sq_distance.argtypes = [f64p, f64p, f64p, f64p, C.c_int64, f64p, C.c_void_p]
        L.ref_analyze_topology.restype = C.c_int
        L.ref_analyze_topology.argtypes = [f64p, C.c_int64, i32p, C.c_int64, i64p]
        L.ref_link_condition.restype = C.c_int
        L.ref_link_condition.argtypes = [f64p, C.c_int64, i32p, C.c_int64, i32p, C.c_int64, i32p]
        L.ref_collapse_sequence.restype = C.c_int
        L.ref_collapse_sequence.argtypes = [f64p, C.c_int64, i32p, C.c_int64, i32p, f64p, C.c_int64, C.c_int,
                                            i32p, f64p, i32p, i64p, i64p]
        L.ref_bvh_overlap_pairs.restype = C.c_int64
        L.ref_bvh_overlap_pairs.argtypes = [f64p, C.c_int64, i32p, C.c_int64, C.c_void_p, C.c_int64]
        L.ref_normalize_unit_cube.restype = C.c_int
        L.ref_normalize_unit_cube.argtypes = [f64p, C.c_int64, C.c_double, f64p]
        L.ref_analyze_topology_lists.restype = C.c_int
        L.ref_analyze_topology_lists.argtypes = [f64p, C.c_int64, i32p, C.c_int64, C.c_void_p, C.c_void_p]
        L.ref_load_mesh.restype = C.c_int
        L.ref_load_mesh.argtypes = [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), i64p]
        L.ref_load_fetch.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_nearest_primitive.restype = C.c_int
        L.ref_nearest_primitive.argtypes = [f64p, C.c_int64, i32p, C.c_int64, f64p, C.c_int64, C.c_void_p,
                                            C.c_void_p, C.c_void_p]
        _REF = L
    return _REF


def _vf(v, f):
    return np.ascontiguousarray(v, np.float64).reshape(-1, 3), np.ascontiguousarray(f, np.int32).reshape(-1, 3)


def set_workers(n: int) -> None:
    lib().orc_set_workers(int(n))


# ---------------------------------------------------------------- stage 1a
def hierarchy_pairs(v, f, R: int, r: int) -> np.ndarray:
    v, f = _vf(v, f)
    n = lib().orc_hierarchy_pairs(v.ravel(), f.ravel(), len(f), R, r, None, 0)
    out = np.empty((n, 2), np.int64)
    lib().orc_hierarchy_pairs(v.ravel(), f.ravel(), len(f), R, r, out.ctypes.data, n)
    return out


def compute_udf_sdf(v, f, R: int, eps: float | None = None):
    v, f = _vf(v, f)
    eps = 0.9 / R if eps is None else eps
    n = (R + 1) ** 3
    udf = np.empty(n, np.float32)
    sdf = np.empty(n, np.float32)
    lib().orc_compute_udf_sdf(v.ravel(), f.ravel(), len(f), R, eps, udf.ctypes.data, sdf.ctypes.data)
    return udf, sdf


def brute_udf(v, f, R: int) -> np.ndarray:
    v, f = _vf(v, f)
    out = np.empty((R + 1) ** 3, np.float32)
    lib().orc_brute_udf(v.ravel(), f.ravel(), len(f), R, out)
    return out


def point_triangle_sq(p, a, b, c) -> np.ndarray:
    p, a, b, c = (np.ascontiguousarray(x, np.float64).reshape(-1, 3) for x in (p, a, b, c))
    out = np.empty(len(p), np.float64)
    lib().orc_point_triangle_sq_batch(p.ravel(), a.ravel(), b.ravel(), c.ravel(), len(p), out)
    return out


def det_exp(x: float) -> float:
    return lib().orc_det_exp(float(x))


def sigmoid(t: float, beta: float) -> float:
    return lib().orc_sigmoid(float(t), float(beta))


# ---------------------------------------------------------------- stage 1b
def dmc_table() -> np.ndarray:
    out = np.empty(256 * 6, np.int32)
    lib().orc_dmc_table(out)
    return out.reshape(256, 6)


def dmc_patches(case: int, flip: int):
    out = np.empty(5, np.int32)
    lib().orc_dmc_patches(case, flip, out)
    return out


def dmc_extract(sdf, R: int, beta: float = 5.0) -> dict:
    sdf = np.ascontiguousarray(sdf, np.float32).ravel()
    sizes = np.zeros(5, np.int64)
    lib().orc_dmc_extract(sdf, R, beta, sizes)
    na, nv, nf = int(sizes[0]), int(sizes[1]), int(sizes[2])
    cells = np.empty(na, np.int64)
    cases = np.empty(na, np.uint8)
    flips = np.empty(na, np.uint8)
    verts = np.empty((nv, 3), np.float64)
    faces = np.empty((nf, 3), np.int32)
    lib().orc_dmc_fetch(cells.ctypes.data, cases.ctypes.data, flips.ctypes.data, verts.ctypes.data,
                        faces.ctypes.data)
    out = dict(cells=cells, cases=cases, flips=flips, vertices=verts, faces=faces,
               n_quads=int(sizes[3]), n_split4=int(sizes[4]))
    # build_patches / build_quads views of the same run
    st = np.zeros(2, np.int64)
    lib().orc_dmc_stages(st.ctypes.data, None, None, None, None, None)
    nq = int(st[1])
    vbase = np.empty(na, np.int64)
    quads = np.empty((nq, 4), np.int32)
    qedge = np.empty(nq, np.int64)
    qf = np.empty((nq, 2), np.float32)
    qsplit = np.empty(nq, np.uint8)
    lib().orc_dmc_stages(st.ctypes.data, vbase.ctypes.data, quads.ctypes.data, qedge.ctypes.data, qf.ctypes.data,
                         qsplit.ctypes.data)
    out.update(patch_first=vbase, n_patch_vertices=int(st[0]), quads=quads, quad_edges=qedge, quad_samples=qf,
               quad_split=qsplit)
    return out


def dmc_extract_slab(planes, R: int, pz0: int, own_z0: int, own_z1: int, beta: float = 5.0) -> dict:
    """Slab-local DMC over resident planes [pz0, pz0 + len(planes)): vertices =
    [own patch vertices, 4-split vertices]; face indices relative to the first own patch vertex."""
    planes = np.ascontiguousarray(planes, np.float32)
    pz1 = pz0 + planes.size // ((R + 1) * (R + 1))
    sizes = np.zeros(7, np.int64)
    lib().orc_dmc_extract_slab(planes.ravel(), R, pz0, pz1, own_z0, own_z1, beta, sizes)
    na, nv, nf = int(sizes[0]), int(sizes[1]), int(sizes[2])
    verts = np.empty((nv, 3), np.float64)
    faces = np.empty((nf, 3), np.int32)
    lib().orc_dmc_fetch(None, None, None, verts.ctypes.data, faces.ctypes.data)
    return dict(vertices=verts, faces=faces, nvp_own=int(sizes[5]), n_extra=int(sizes[6]))


# ---------------------------------------------------------------- tri_isect
def tri_tri_pairs(v, f, pairs) -> np.ndarray:
    v, f = _vf(v, f)
    pairs = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
    out = np.empty(len(pairs), np.int32)
    lib().orc_tri_tri_pairs(v.ravel(), f.ravel(), pairs.ravel(), len(pairs), out)
    return out


def orient3d(a, b, c, d) -> int:
    return lib().orc_orient3d(*(np.ascontiguousarray(x, np.float64) for x in (a, b, c, d)))


def self_intersections(v, f) -> np.ndarray:
    v, f = _vf(v, f)
    n = lib().orc_self_intersections(v.ravel(), len(v), f.ravel(), len(f), None, 0)
    out = np.empty((n, 2), np.int32)
    lib().orc_self_intersections(v.ravel(), len(v), f.ravel(), len(f), out.ctypes.data, n)
    return out


def overlap_pairs(v, f) -> np.ndarray:
    v, f = _vf(v, f)
    n = lib().orc_overlap_pairs(v.ravel(), f.ravel(), len(f), None, 0)
    out = np.empty((n, 2), np.int32)
    lib().orc_overlap_pairs(v.ravel(), f.ravel(), len(f), out.ctypes.data, n)
    return out


# ---------------------------------------------------------------- stage 2
STAT_KEYS = ["iterations", "collapses", "undone", "link_failures", "max_undo_rounds", "error",
             "nv_out", "nf_out"]


def simplify(v, f, target: int, we: float = 1e-3, ws: float = 5e-3, tolerance: int = 4):
    v, f = _vf(v, f)
    st = np.zeros(17, np.int64)
    rc = lib().orc_simplify(v.ravel(), len(v), f.ravel(), len(f), int(target), we, ws, tolerance, st)
    if rc != 0:
        raise ValueError("oracle simplify: NaN edge cost")
    stats = {k: int(st[i]) for i, k in enumerate(STAT_KEYS)}
    stats["undo_hist"] = [int(x) for x in st[8:16]]
    stats["face_iterations"] = int(st[16])
    nv, nf = stats["nv_out"], stats["nf_out"]
    vo = np.empty((nv, 3), np.float64)
    fo = np.empty((nf, 3), np.int32)
    per_iter = np.empty(stats["iterations"], np.int64)
    lib().orc_simplify_fetch(vo.ctypes.data, fo.ctypes.data, per_iter.ctypes.data)
    stats["per_iter_collapses"] = per_iter
    return vo, fo, stats


def simplify_trace(v, f, target: int, iteration: int, we: float = 1e-3, ws: float = 5e-3, tolerance: int = 4):
    """Step-level record of one simplify_to iteration (1-based): edges, keys, placements, face
    keys, marked edge ids, link results, applied edge ids, undo rounds and the mesh after it."""
    v, f = _vf(v, f)
    sz = np.zeros(6, np.int64)
    rc = lib().orc_simplify_trace(v.ravel(), len(v), f.ravel(), len(f), int(target), we, ws, tolerance,
                                  int(iteration), sz)
    if rc < 0:
        raise ValueError("oracle simplify: NaN edge cost")
    if rc > 0:
        raise ValueError("oracle simplify: the run ended before that iteration")
    ne, nf, nm, na, rounds, nv = (int(x) for x in sz)
    t = dict(edges=np.empty((ne, 2), np.int32), keys=np.empty(ne, np.uint64), place=np.empty((ne, 3)),
             face_keys=np.empty(nf, np.uint64), marked=np.empty(nm, np.int64), link_ok=np.empty(nm, np.uint8),
             applied=np.empty(na, np.int64), X=np.empty((nv, 3)), F=np.empty((nf, 3), np.int32),
             falive=np.empty(nf, np.uint8))
    order = ["edges", "keys", "place", "face_keys", "marked", "link_ok", "applied", "X", "F", "falive"]
    lib().orc_trace_fetch(*[t[k].ctypes.data for k in order])
    t["rounds"] = rounds
    return t


def quadrics(v, f) -> np.ndarray:
    v, f = _vf(v, f)
    out = np.empty((len(v), 10))
    lib().orc_quadrics(v.ravel(), len(v), f.ravel(), len(f), out.ravel())
    return out


def edge_cost(v, f, edges, we: float = 1e-3, ws: float = 5e-3):
    v, f = _vf(v, f)
    e = np.ascontiguousarray(edges, np.int32).reshape(-1, 2)
    cost = np.empty(len(e))
    place = np.empty((len(e), 3))
    lib().orc_edge_cost(v.ravel(), len(v), f.ravel(), len(f), e.ravel(), len(e), we, ws, cost, place.ravel())
    return cost, place


def link_condition(v, f, edges) -> np.ndarray:
    v, f = _vf(v, f)
    edges = np.ascontiguousarray(edges, np.int32).reshape(-1, 2)
    out = np.empty(len(edges), np.int32)
    lib().orc_link_condition(v.ravel(), len(v), f.ravel(), len(f), edges.ravel(), len(edges), out)
    return out


# ---------------------------------------------------------------- reference primitives
def ref_point_triangle_sq(p, a, b, c) -> np.ndarray:
    p, a, b, c = (np.ascontiguousarray(x, np.float64).reshape(-1, 3) for x in (p, a, b, c))
    out = np.empty(len(p), np.float64)
    ref().ref_point_triangle_sq_distance(p.ravel(), a.ravel(), b.ravel(), c.ravel(), len(p), out, None)
    return out


def ref_topology(v, f) -> dict:
    v, f = _vf(v, f)
    out = np.zeros(6, np.int64)
    rc = ref().ref_analyze_topology(v.ravel(), len(v), f.ravel(), len(f), out)
    assert rc == 0
    return dict(manifold=bool(out[0]), watertight=bool(out[1]), euler=int(out[2]),
                boundary_edges=int(out[3]), nonmanifold_edges=int(out[4]), nonmanifold_vertices=int(out[5]))


def ref_link_condition(v, f, edges) -> np.ndarray:
    v, f = _vf(v, f)
    edges = np.ascontiguousarray(edges, np.int32).reshape(-1, 2)
    out = np.empty(len(edges), np.int32)
    assert ref().ref_link_condition(v.ravel(), len(v), f.ravel(), len(f), edges.ravel(), len(edges), out) == 0
    return out


def ref_collapse_sequence(v, f, edges, pos, undo=False):
    v, f = _vf(v, f)
    edges = np.ascontiguousarray(edges, np.int32).reshape(-1, 2)
    pos = np.ascontiguousarray(pos, np.float64).reshape(-1, 3)
    ok = np.empty(len(edges), np.int32)
    ov = np.empty_like(v)
    of = np.empty_like(f)
    nv = np.zeros(1, np.int64)
    nf = np.zeros(1, np.int64)
    assert ref().ref_collapse_sequence(v.ravel(), len(v), f.ravel(), len(f), edges.ravel(), pos.ravel(),
                                       len(edges), int(undo), ok, ov.ravel(), of.ravel(), nv, nf) == 0
    return ok, ov[: nv[0]], of[: nf[0]]


def ref_bvh_overlap_pairs(v, f) -> np.ndarray:
    v, f = _vf(v, f)
    n = ref().ref_bvh_overlap_pairs(v.ravel(), len(v), f.ravel(), len(f), None, 0)
    out = np.empty((n, 2), np.int32)
    ref().ref_bvh_overlap_pairs(v.ravel(), len(v), f.ravel(), len(f), out.ctypes.data, n)
    return out


def ref_normalize_unit_cube(v, padding: float):
    v = np.ascontiguousarray(v, np.float64).reshape(-1, 3).copy()
    st = np.zeros(4, np.float64)
    assert ref().ref_normalize_unit_cube(v.ravel(), len(v), padding, st) == 0
    return v, st


# ---------------------------------------------------------------- certification / metrics
SAMPLE_SEED_B = 0x632BE59BD9B4E019  # seed offset of the second mesh's samples (chamfer/hausdorff)


def topology(f, nv: int) -> dict:
    """analyze_topology restatement (mesh.cpp:113-150) with the non-manifold lists."""
    f = np.ascontiguousarray(f, np.int32).reshape(-1, 3)
    out = np.zeros(6, np.int64)
    lib().orc_topology(f, len(f), int(nv), out)
    edges = np.empty(int(out[4]), np.int64)
    verts = np.empty(int(out[5]), np.int32)
    lib().orc_topology_lists(edges.ctypes.data, verts.ctypes.data)
    return dict(manifold=bool(out[0]), watertight=bool(out[1]), euler=int(out[2]), boundary_edges=int(out[3]),
                nonmanifold_edges=np.stack([edges >> 32, edges & 0xffffffff], 1).astype(np.int32),
                nonmanifold_vertices=verts)


def nearest(v, f, pts):
    """Brute-force nearest face per point (lbvh.cpp:192-237 semantics): (face, dist, closest)."""
    v, f = _vf(v, f)
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    face = np.empty(len(pts), np.int32)
    dist = np.empty(len(pts))
    clo = np.empty((len(pts), 3))
    lib().orc_nearest(v, f, len(f), pts.ravel(), len(pts), face.ctypes.data, dist.ctypes.data, clo.ctypes.data)
    return face, dist, clo


def sample(v, f, n: int, seed: int):
    """Pinned area-weighted sampler -> (points [n,3], face ids, total area); None for zero area."""
    v, f = _vf(v, f)
    pts = np.empty((n, 3))
    fid = np.empty(n, np.int32)
    area = C.c_double()
    rc = lib().orc_sample(v, f, len(f), int(n), int(seed) & (2**64 - 1), pts.ctypes.data, fid.ctypes.data,
                          C.byref(area))
    if rc != 0:
        return None
    return pts, fid, area.value


def _directed(va, fa, vb, fb, n, seed):
    s = sample(va, fa, n, seed)
    if s is None:
        raise ValueError("zero-area mesh")
    _, d, _ = nearest(vb, fb, s[0])
    return d, s[2]


def chamfer(va, fa, vb, fb, n: int = 16384, seed: int = 42) -> float:
    """(A(a)/n) sum d^2(s_i(a), b) + (A(b)/n) sum d^2(t_j(b), a) (SPEC quality_metrics)."""
    da, aa = _directed(va, fa, vb, fb, n, seed)
    db, ab = _directed(vb, fb, va, fa, n, seed + SAMPLE_SEED_B)
    return aa / n * float(np.sum(da * da)) + ab / n * float(np.sum(db * db))


def hausdorff(va, fa, vb, fb, n: int = 16384, seed: int = 42) -> float:
    da, _ = _directed(va, fa, vb, fb, n, seed)
    db, _ = _directed(vb, fb, va, fa, n, seed + SAMPLE_SEED_B)
    return float(max(da.max(), db.max()))


def min_internal_angle(v, f) -> float:
    v, f = _vf(v, f)
    c = lib().orc_max_corner_cos(v, f, len(f))
    return float(np.degrees(np.arccos(c)))


def ref_topology_full(v, f) -> dict:
    v, f = _vf(v, f)
    out = np.zeros(6, np.int64)
    rc = ref().ref_analyze_topology(v, len(v), f, len(f), out)
    assert rc == 0
    edges = np.empty(int(out[4]), np.int64)
    verts = np.empty(int(out[5]), np.int32)
    rc = ref().ref_analyze_topology_lists(v, len(v), f, len(f), edges.ctypes.data, verts.ctypes.data)
    assert rc == 0
    return dict(manifold=bool(out[0]), watertight=bool(out[1]), euler=int(out[2]), boundary_edges=int(out[3]),
                nonmanifold_edges=np.stack([edges >> 32, edges & 0xffffffff], 1).astype(np.int32),
                nonmanifold_vertices=verts)


def ref_nearest(v, f, pts):
    v, f = _vf(v, f)
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    face = np.empty(len(pts), np.int32)
    dist = np.empty(len(pts))
    clo = np.empty((len(pts), 3))
    rc = ref().ref_nearest_primitive(v, len(v), f, len(f), pts.ravel(), len(pts), face.ctypes.data,
                                     dist.ctypes.data, clo.ctypes.data)
    assert rc == 0
    return face, dist, clo


# ---------------------------------------------------------------- ingest (mesh_io.cpp)
def ref_load_mesh(path: str):
    """The reference's own load_mesh: (vertices, faces, stats dict) or None on a load error."""
    nv, nf = C.c_int64(), C.c_int64()
    st = np.zeros(3, np.int64)
    if ref().ref_load_mesh(path.encode(), C.byref(nv), C.byref(nf), st) != 0:
        return None
    v = np.empty((nv.value, 3))
    f = np.empty((nf.value, 3), np.int32)
    ref().ref_load_fetch(v.ctypes.data, f.ctypes.data)
    return v, f, dict(degenerate_faces_dropped=int(st[0]), polygons_triangulated=int(st[1]),
                      vertices_welded=int(st[2]))


def load_stl_binary(data: bytes):
    """Restatement of load_stl's binary branch + StlWelder (mesh_io.cpp:291-366): corners welded
    by exact equality (bit patterns; a NaN corner is never equal), first-occurrence numbering,
    faces with repeated indices dropped (add_polygon, mesh_io.cpp:32-42)."""
    count = int(np.frombuffer(data[80:84], np.uint32)[0])
    rec = np.frombuffer(data[84:84 + 50 * count], np.uint8).reshape(count, 50)
    pts = rec[:, 12:48].copy().view(np.float32).reshape(count * 3, 3)
    ids, verts, welded = {}, [], 0
    vid = np.empty(count * 3, np.int64)
    for c, p in enumerate(pts):
        if np.isnan(p).any():
            vid[c] = len(verts)
            verts.append(p.astype(np.float64))
            continue
        key = p.tobytes()
        if key in ids:
            vid[c] = ids[key]
            welded += 1
        else:
            ids[key] = vid[c] = len(verts)
            verts.append(p.astype(np.float64))
    tri = vid.reshape(count, 3)
    keep = (tri[:, 0] != tri[:, 1]) & (tri[:, 1] != tri[:, 2]) & (tri[:, 0] != tri[:, 2])
    v = np.array(verts, np.float64).reshape(-1, 3)
    return v, tri[keep].astype(np.int32), dict(degenerate_faces_dropped=int((~keep).sum()), polygons_triangulated=0,
                                               vertices_welded=welded)
