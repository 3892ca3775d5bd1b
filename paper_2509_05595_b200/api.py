"""Python host mirror of the reference's SPEC operations over the C-ABI (libpamopt_cu.so).

Names follow the reference (SPEC.md `[OP]`s / proj/include/pamopt): `compute_udf`,
`udf_to_sdf`, `build_hierarchy` (debug view), `extract`, `detect_self_intersections`,
`simplify_to`, `run_pipeline`.  Everything runs on the GPU; errors surface as
`PamoptInvalidArgument` (std::invalid_argument in the reference) or `PamoptError`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib, ptr

DEFAULT_BETA = 5.0
DEFAULT_WE = 1e-3
DEFAULT_WS = 5e-3
DEFAULT_TOL = 4


def default_eps(R: int) -> float:
    return 0.9 / R


class Context:
    """One device + one CUDA stream (pamopt_cu_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().pamopt_cu_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device

    @property
    def stream(self) -> int:
        return int(lib().pamopt_cu_ctx_stream(self.h) or 0)

    def synchronize(self) -> None:
        check(lib().pamopt_cu_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        return int(lib().pamopt_cu_ctx_launches(self.h))

    def profile(self, on: bool = True) -> None:
        """Per-kernel device-time accounting (events around every launch; perturbs timing)."""
        check(lib().pamopt_cu_ctx_profile(self.h, 1 if on else 0))

    def kernel_times(self) -> dict:
        """{kernel: (ms, launches)} accumulated since profile(True)."""
        n = lib().pamopt_cu_ctx_kernel_times(self.h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        lib().pamopt_cu_ctx_kernel_times(self.h, buf, len(buf))
        out = {}
        for line in buf.value.decode().splitlines():
            name, ms, cnt = line.split("\t")
            out[name] = (float(ms), int(cnt))
        return out

    def close(self) -> None:
        if self.h:
            lib().pamopt_cu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class DeviceMesh:
    """Device-resident IndexedMesh (mesh.hpp:18-33)."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    @classmethod
    def upload(cls, vertices, faces, ctx: Context | None = None) -> "DeviceMesh":
        ctx = ctx or default_context()
        v = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
        f = np.ascontiguousarray(faces, np.int32).reshape(-1, 3)
        h = C.c_void_p()
        check(lib().pamopt_cu_mesh_upload(ctx.h, ptr(v), len(v), ptr(f), len(f), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_device(cls, vptr: int, nv: int, fptr: int, nf: int, ctx: Context | None = None) -> "DeviceMesh":
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib().pamopt_cu_mesh_from_device(ctx.h, C.c_void_p(vptr), nv, C.c_void_p(fptr), nf, C.byref(h)))
        return cls(h, ctx)

    def size(self):
        nv, nf = C.c_int64(), C.c_int64()
        check(lib().pamopt_cu_mesh_size(self.h, C.byref(nv), C.byref(nf)))
        return nv.value, nf.value

    def download(self):
        nv, nf = self.size()
        v = np.empty((nv, 3), np.float64)
        f = np.empty((nf, 3), np.int32)
        check(lib().pamopt_cu_mesh_download(self.h, ptr(v), ptr(f)))
        return v, f

    def rebase(self, patch_base: int, nvp_own: int, extra_base: int) -> None:
        """Face indices -> global ids of the assembled slab mesh (pamopt_cu_mesh_rebase)."""
        check(lib().pamopt_cu_mesh_rebase(self.h, int(patch_base), int(nvp_own), int(extra_base)))

    def copy_to_device(self, vptr: int | None, fptr: int | None) -> None:
        check(lib().pamopt_cu_mesh_copy_to_device(self.h, C.c_void_p(vptr) if vptr else None,
                                                   C.c_void_p(fptr) if fptr else None))

    def free(self):
        if self.h:
            lib().pamopt_cu_mesh_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class DeviceGrid:
    """Device-resident ScalarGrid ((R+1)^3 f32, x-fastest), or a z-slab of it
    (lattice planes [z0, z1))."""

    def __init__(self, handle, ctx: Context, R: int):
        self.h = handle
        self.ctx = ctx
        self.R = R
        z0, z1 = C.c_int32(), C.c_int32()
        check(lib().pamopt_cu_grid_slab(handle, C.byref(z0), C.byref(z1)))
        self.z0, self.z1 = z0.value, z1.value

    @property
    def planes(self) -> int:
        return self.z1 - self.z0

    @classmethod
    def from_device(cls, ptr: int, R: int, ctx: Context | None = None) -> "DeviceGrid":
        """Full (R+1)^3 grid copied from a device buffer (e.g. a torch tensor's data_ptr)."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib().pamopt_cu_grid_from_device(ctx.h, int(R), C.c_void_p(ptr), C.byref(h)))
        return cls(h, ctx, R)

    def copy_to_device(self, ptr: int) -> None:
        check(lib().pamopt_cu_grid_copy_to_device(self.h, C.c_void_p(ptr)))

    @classmethod
    def slab_from_device(cls, ptr: int, R: int, z0: int, z1: int, ctx: Context | None = None) -> "DeviceGrid":
        """z-slab (lattice planes [z0, z1)) copied from a device buffer."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib().pamopt_cu_grid_slab_from_device(ctx.h, int(R), int(z0), int(z1), C.c_void_p(ptr), C.byref(h)))
        return cls(h, ctx, R)

    @classmethod
    def slab_upload(cls, planes, R: int, z0: int, ctx: Context | None = None) -> "DeviceGrid":
        """z-slab from host samples: planes [z0, z0 + len) of the (R+1)^3 lattice."""
        ctx = ctx or default_context()
        s = np.ascontiguousarray(planes, np.float32).ravel()
        n = s.size // ((R + 1) * (R + 1))
        assert s.size == n * (R + 1) * (R + 1)
        h = C.c_void_p()
        check(lib().pamopt_cu_grid_slab_upload(ctx.h, int(R), int(z0), int(z0 + n), ptr(s), C.byref(h)))
        return cls(h, ctx, R)

    @classmethod
    def upload(cls, samples, R: int, ctx: Context | None = None) -> "DeviceGrid":
        ctx = ctx or default_context()
        s = np.ascontiguousarray(samples, np.float32).ravel()
        assert s.size == (R + 1) ** 3
        h = C.c_void_p()
        check(lib().pamopt_cu_grid_upload(ctx.h, R, ptr(s), C.byref(h)))
        return cls(h, ctx, R)

    def download(self) -> np.ndarray:
        out = np.empty((self.R + 1) ** 2 * self.planes, np.float32)
        check(lib().pamopt_cu_grid_download(self.h, ptr(out)))
        return out

    def free(self):
        if self.h:
            lib().pamopt_cu_grid_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _mesh(m, ctx=None) -> DeviceMesh:
    if isinstance(m, DeviceMesh):
        return m
    v, f = m
    return DeviceMesh.upload(v, f, ctx)


# ------------------------------------------------------------------ voxel_field (stage 1a)
def compute_udf(mesh, R: int, ctx: Context | None = None) -> DeviceGrid:
    """build_hierarchy + compute_udf."""
    m = _mesh(mesh, ctx)
    h = C.c_void_p()
    check(lib().pamopt_cu_compute_udf(m.ctx.h, m.h, int(R), C.byref(h)))
    return DeviceGrid(h, m.ctx, R)


def udf_to_sdf(grid: DeviceGrid, eps: float | None = None) -> DeviceGrid:
    """In place."""
    check(lib().pamopt_cu_udf_to_sdf(grid.h, default_eps(grid.R) if eps is None else float(eps)))
    return grid


def compute_sdf(mesh, R: int, eps: float | None = None, ctx: Context | None = None) -> DeviceGrid:
    m = _mesh(mesh, ctx)
    h = C.c_void_p()
    check(lib().pamopt_cu_compute_sdf(m.ctx.h, m.h, int(R), default_eps(R) if eps is None else float(eps),
                                      C.byref(h)))
    return DeviceGrid(h, m.ctx, R)


def compute_sdf_slab(mesh, R: int, z0: int, z1: int, eps: float | None = None,
                     ctx: Context | None = None) -> DeviceGrid:
    """SDF lattice planes [z0, z1) only — one rank's share of the z-slab decomposition."""
    m = _mesh(mesh, ctx)
    h = C.c_void_p()
    check(lib().pamopt_cu_compute_sdf_slab(m.ctx.h, m.h, int(R), default_eps(R) if eps is None else float(eps),
                                           int(z0), int(z1), C.byref(h)))
    return DeviceGrid(h, m.ctx, R)


def build_hierarchy_pairs(mesh, R: int, r: int, ctx: Context | None = None) -> np.ndarray:
    """Surviving (cell, tri) pairs of level r, sorted (VoxelHierarchy view)."""
    m = _mesh(mesh, ctx)
    n = C.c_int64()
    check(lib().pamopt_cu_hierarchy_pairs(m.ctx.h, m.h, int(R), int(r), None, 0, C.byref(n)))
    out = np.empty((n.value, 2), np.int64)
    check(lib().pamopt_cu_hierarchy_pairs(m.ctx.h, m.h, int(R), int(r), ptr(out), n.value, C.byref(n)))
    return out


# ------------------------------------------------------------------ dual_mc (stage 1b)
def extract(grid: DeviceGrid, beta: float = DEFAULT_BETA) -> DeviceMesh:
    """dual_mc::extract."""
    h = C.c_void_p()
    check(lib().pamopt_cu_dmc_extract(grid.h, float(beta), C.byref(h)))
    return DeviceMesh(h, grid.ctx)


def extract_slab(grid: DeviceGrid, own_z0: int, own_z1: int, beta: float = DEFAULT_BETA):
    """Slab-local extract.  Returns (DeviceMesh, nvp_own, n_extra); the mesh's
    vertices are [own patch vertices, 4-split vertices] and its face indices are relative to the
    first own patch vertex until DeviceMesh.rebase."""
    h = C.c_void_p()
    counts = (C.c_int64 * 2)()
    check(lib().pamopt_cu_dmc_extract_slab(grid.h, int(own_z0), int(own_z1), float(beta), C.byref(h), counts))
    return DeviceMesh(h, grid.ctx), int(counts[0]), int(counts[1])


def nccl_comm_init_all(devices) -> list:
    """ncclCommInitAll for one host process driving several GPUs (returns the ncclComm_t handles)."""
    d = np.ascontiguousarray(devices, np.int32)
    comms = (C.c_void_p * len(d))()
    check(lib().pamopt_cu_nccl_comm_init_all(len(d), ptr(d), comms))
    return list(comms)


def nccl_comm_destroy(comm) -> None:
    check(lib().pamopt_cu_nccl_comm_destroy(C.c_void_p(comm)))


def extract_slab_nccl(mesh, R: int, rank: int, world: int, comm=None, eps: float | None = None,
                      beta: float = DEFAULT_BETA, ctx: Context | None = None):
    """The C4 slab path of one rank over NCCL (pamopt_cu_extract_slab_nccl): returns (DeviceMesh on
    rank 0 / None elsewhere, this slab's (patch vertices, split vertices, faces) counts)."""
    m = _mesh(mesh, ctx)
    h = C.c_void_p()
    counts = np.zeros(3, np.int64)
    check(lib().pamopt_cu_extract_slab_nccl(m.ctx.h, m.h, int(R), default_eps(R) if eps is None else float(eps),
                                            float(beta), int(rank), int(world), C.c_void_p(comm), C.byref(h),
                                            ptr(counts)))
    return (DeviceMesh(h, m.ctx) if h.value else None), counts


def dmc_active_cells(grid: DeviceGrid):
    n = C.c_int64()
    check(lib().pamopt_cu_dmc_active_cells(grid.h, None, None, None, 0, C.byref(n)))
    cells = np.empty(n.value, np.int64)
    cases = np.empty(n.value, np.uint8)
    flips = np.empty(n.value, np.uint8)
    check(lib().pamopt_cu_dmc_active_cells(grid.h, ptr(cells), ptr(cases), ptr(flips), n.value, C.byref(n)))
    return cells, cases, flips


def dmc_stages(grid: DeviceGrid, beta: float = DEFAULT_BETA) -> dict:
    """classify_voxels + build_patches + build_quads as separate views: active
    cells, patch vertices with each active cell's first patch vertex, and the quads (patch-vertex
    ids, valid edge = lower lattice vertex * 3 + axis, its two samples, triangulate_quads' split)."""
    counts = np.zeros(3, np.int64)
    check(lib().pamopt_cu_dmc_stages(grid.h, float(beta), ptr(counts)))
    na, nv, nq = (int(x) for x in counts)
    pv = np.empty((nv, 3))
    first = np.empty(na, np.int64)
    check(lib().pamopt_cu_dmc_build_patches(grid.h, ptr(pv), ptr(first)))
    quads = np.empty((nq, 4), np.int32)
    edges = np.empty(nq, np.int64)
    samples = np.empty((nq, 2), np.float32)
    split = np.empty(nq, np.uint8)
    check(lib().pamopt_cu_dmc_build_quads(grid.h, ptr(quads), ptr(edges), ptr(samples), ptr(split)))
    cells, cases, flips = dmc_active_cells(grid)
    return dict(cells=cells, cases=cases, flips=flips, patch_vertices=pv, patch_first=first, quads=quads,
                quad_edges=edges, quad_samples=samples, quad_split=split)


def triangulate_quads(R: int, patch_vertices, quads, quad_edges, quad_samples, beta: float = DEFAULT_BETA,
                      ctx: Context | None = None) -> DeviceMesh:
    """triangulate_quads on explicit quads -> DeviceMesh."""
    ctx = ctx or default_context()
    pv = np.ascontiguousarray(patch_vertices, np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(quads, np.int32).reshape(-1, 4)
    e = np.ascontiguousarray(quad_edges, np.int64).ravel()
    s_ = np.ascontiguousarray(quad_samples, np.float32).reshape(-1, 2)
    h = C.c_void_p()
    check(lib().pamopt_cu_triangulate_quads(ctx.h, int(R), ptr(pv), len(pv), ptr(q), ptr(e), ptr(s_), len(q),
                                            float(beta), C.byref(h)))
    return DeviceMesh(h, ctx)


def interpolate_patch_vertex(p0, p1, f0, f1, beta: float = DEFAULT_BETA, ctx: Context | None = None) -> np.ndarray:
    """interpolate_patch_vertex for arrays of edges; raises for equal signs."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(p0, np.float64).reshape(-1, 3)
    b = np.ascontiguousarray(p1, np.float64).reshape(-1, 3)
    x = np.ascontiguousarray(f0, np.float32).ravel()
    y = np.ascontiguousarray(f1, np.float32).ravel()
    out = np.empty((len(a), 3))
    check(lib().pamopt_cu_interpolate_patch_vertex(ctx.h, ptr(a), ptr(b), ptr(x), ptr(y), len(a), float(beta),
                                                   ptr(out)))
    return out


def dmc_table() -> np.ndarray:
    out = np.empty(256 * 6, np.int32)
    check(lib().pamopt_cu_dmc_table(ptr(out)))
    return out.reshape(256, 6)


# ------------------------------------------------------------------ tri_isect
def detect_self_intersections(mesh, ctx: Context | None = None) -> np.ndarray:
    """Sorted (f1<f2) intersecting face pairs."""
    m = _mesh(mesh, ctx)
    n = C.c_int64()
    check(lib().pamopt_cu_self_intersections(m.h, None, 0, C.byref(n)))
    out = np.empty((n.value, 2), np.int32)
    check(lib().pamopt_cu_self_intersections(m.h, ptr(out), n.value, C.byref(n)))
    return out


def tri_tri_pairs(mesh, pairs, ctx: Context | None = None) -> np.ndarray:
    m = _mesh(mesh, ctx)
    p = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
    out = np.empty(len(p), np.int32)
    check(lib().pamopt_cu_tri_tri_pairs(m.h, ptr(p), len(p), ptr(out)))
    return out


def classify_pair(mesh, pairs, ctx: Context | None = None):
    """classify_pair: (shared-vertex count, coplanar flag) per pair."""
    m = _mesh(mesh, ctx)
    p = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
    sh = np.empty(len(p), np.int32)
    cp = np.empty(len(p), np.int32)
    check(lib().pamopt_cu_classify_pair(m.h, ptr(p), len(p), ptr(sh), ptr(cp)))
    return sh, cp


def intersect_3d(mesh, pairs, ctx: Context | None = None) -> np.ndarray:
    """intersect_3d for non-coplanar pairs; raises for a coplanar pair."""
    m = _mesh(mesh, ctx)
    p = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
    out = np.empty(len(p), np.int32)
    check(lib().pamopt_cu_intersect_3d(m.h, ptr(p), len(p), ptr(out)))
    return out


def intersect_coplanar(mesh, pairs, ctx: Context | None = None) -> np.ndarray:
    """intersect_coplanar for coplanar pairs; raises for a non-coplanar pair."""
    m = _mesh(mesh, ctx)
    p = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
    out = np.empty(len(p), np.int32)
    check(lib().pamopt_cu_intersect_coplanar(m.h, ptr(p), len(p), ptr(out)))
    return out


# ------------------------------------------------------------------ simplify (stage 2)
def _params(we, ws, tolerance, stall=10) -> _lib.SimplifyParams:
    return _lib.SimplifyParams(float(we), float(ws), int(tolerance), int(stall))


def simplify_to(mesh, target_faces: int, we: float = DEFAULT_WE, ws: float = DEFAULT_WS,
                tolerance: int = DEFAULT_TOL, ctx: Context | None = None, per_iter_cap: int = 100000):
    """simplify_to.  Simplifies a DeviceMesh in place; returns (mesh, stats)."""
    m = _mesh(mesh, ctx)
    st = _lib.SimplifyStats()
    per = np.zeros(per_iter_cap, np.int64)
    p = _params(we, ws, tolerance)
    check(lib().pamopt_cu_simplify(m.h, int(target_faces), C.byref(p), C.byref(st), ptr(per), per_iter_cap))
    stats = st.as_dict()
    stats["per_iter_collapses"] = per[: stats["iterations"]].copy()
    return m, stats


# ------------------------------------------------- stage 2, SPEC-granular operations
def _edges_arr(edges) -> np.ndarray:
    return np.ascontiguousarray(edges, np.int32).reshape(-1, 2)


def quadrics(mesh, ctx: Context | None = None) -> np.ndarray:
    """Quadric per vertex: (nv, 10) = xx xy xz xw yy yz yw zz zw ww."""
    m = _mesh(mesh, ctx)
    nv, _ = m.size()
    out = np.empty((nv, 10))
    check(lib().pamopt_cu_quadrics(m.h, ptr(out)))
    return out


def edge_cost(mesh, edges, we: float = DEFAULT_WE, ws: float = DEFAULT_WS, ctx: Context | None = None):
    """edge_cost of explicit edges: (cost[n], placement[n, 3])."""
    m = _mesh(mesh, ctx)
    e = _edges_arr(edges)
    cost = np.empty(len(e))
    place = np.empty((len(e), 3))
    check(lib().pamopt_cu_edge_cost(m.h, ptr(e), len(e), float(we), float(ws), ptr(cost), ptr(place)))
    return cost, place


def pack_cost(cost, edge_ids, ctx: Context | None = None) -> np.ndarray:
    """pack_cost on the GPU; PamoptError (ENUMERIC) for a NaN cost."""
    ctx = ctx or default_context()
    c = np.ascontiguousarray(cost, np.float64).ravel()
    ids = np.ascontiguousarray(edge_ids, np.uint32).ravel()
    keys = np.empty(len(c), np.uint64)
    check(lib().pamopt_cu_pack_cost(ctx.h, ptr(c), ptr(ids), len(c), ptr(keys)))
    return keys


def link_condition(mesh, edges, ctx: Context | None = None) -> np.ndarray:
    """HalfEdgeAdjacency::link_condition_holds (mesh.cpp:301-358) per edge (bool); raises
    PamoptInvalidArgument for a pair that is not an edge (mesh.cpp:302)."""
    m = _mesh(mesh, ctx)
    e = _edges_arr(edges)
    out = np.empty(len(e), np.int32)
    check(lib().pamopt_cu_link_condition(m.h, ptr(e), len(e), ptr(out)))
    return out.astype(bool)


class QemRun:
    """Algorithm 1 one SPEC operation at a time (pamopt_cu_qem_*): the same code simplify_to
    runs.  Per iteration: prepare(), propagate_and_mark(), collapse_batch(), undo_loop(),
    end_iteration(); finish() compacts the mesh."""

    def __init__(self, mesh: DeviceMesh, target_faces: int, we: float = DEFAULT_WE, ws: float = DEFAULT_WS,
                 tolerance: int = DEFAULT_TOL):
        self.mesh = mesh
        self.h = C.c_void_p()
        p = _params(we, ws, tolerance)
        check(lib().pamopt_cu_qem_create(mesh.h, int(target_faces), C.byref(p), C.byref(self.h)))
        self.ne = self.nm = 0

    def done(self) -> bool:
        d = C.c_int32()
        check(lib().pamopt_cu_qem_done(self.h, C.byref(d)))
        return bool(d.value)

    def prepare(self) -> int:
        n = C.c_int64()
        check(lib().pamopt_cu_qem_prepare(self.h, C.byref(n)))
        self.ne = n.value
        return self.ne

    def edges(self) -> dict:
        n = self.ne
        e = np.empty((n, 2), np.int32)
        k = np.empty(n, np.uint64)
        p = np.empty((n, 3))
        v = np.empty(n, np.uint8)
        check(lib().pamopt_cu_qem_edges(self.h, ptr(e), ptr(k), ptr(p), ptr(v), n))
        return dict(edges=e, keys=k, place=p, valid=v)

    def propagate_and_mark(self) -> int:
        n = C.c_int64()
        check(lib().pamopt_cu_qem_propagate_and_mark(self.h, C.byref(n)))
        self.nm = n.value
        return self.nm

    def marked(self):
        ids = np.empty(self.nm, np.uint32)
        _, nf = self.state_sizes()
        fk = np.empty(nf, np.uint64)
        check(lib().pamopt_cu_qem_marked(self.h, ptr(ids), self.nm, ptr(fk), nf))
        return ids, fk

    def collapse_batch(self) -> np.ndarray:
        ok = np.empty(self.nm, np.uint8)
        check(lib().pamopt_cu_qem_collapse_batch(self.h, ptr(ok), self.nm))
        return ok

    def undo_loop(self):
        r, n = C.c_int32(), C.c_int64()
        applied = np.empty(self.nm, np.uint8)
        check(lib().pamopt_cu_qem_undo_loop(self.h, C.byref(r), C.byref(n), ptr(applied), self.nm))
        return r.value, n.value, applied

    def end_iteration(self) -> int:
        a = C.c_int64()
        check(lib().pamopt_cu_qem_end_iteration(self.h, C.byref(a)))
        return a.value

    def state_sizes(self):
        nv, nf = C.c_int64(), C.c_int64()
        check(lib().pamopt_cu_qem_mesh(self.h, None, None, None, C.byref(nv), C.byref(nf)))
        return nv.value, nf.value

    def state_mesh(self):
        nv, nf = self.state_sizes()
        v = np.empty((nv, 3))
        f = np.empty((nf, 3), np.int32)
        a = np.empty(nf, np.uint8)
        n1, n2 = C.c_int64(), C.c_int64()
        check(lib().pamopt_cu_qem_mesh(self.h, ptr(v), ptr(f), ptr(a), C.byref(n1), C.byref(n2)))
        return v, f, a

    def finish(self) -> dict:
        st = _lib.SimplifyStats()
        check(lib().pamopt_cu_qem_finish(self.h, C.byref(st)))
        return st.as_dict()

    def close(self):
        if self.h:
            lib().pamopt_cu_qem_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ pipeline (stages 1-2)
@dataclass
class RemeshResult:
    vertices: np.ndarray
    faces: np.ndarray
    stats: dict = field(default_factory=dict)
    times: dict = field(default_factory=dict)


def run_pipeline(vertices, faces, R: int, target_faces: int, eps: float | None = None,
                 beta: float = DEFAULT_BETA, we: float = DEFAULT_WE, ws: float = DEFAULT_WS,
                 tolerance: int = DEFAULT_TOL, ctx: Context | None = None) -> RemeshResult:
    """UDF -> SDF -> DMC -> QEM (run_pipeline stages 1-2) through the host
    C-ABI entry (pamopt_cu_remesh_host): host arrays in, host arrays out."""
    ctx = ctx or default_context()
    v = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
    f = np.ascontiguousarray(faces, np.int32).reshape(-1, 3)
    nv, nf = C.c_int64(), C.c_int64()
    st = _lib.SimplifyStats()
    tm = _lib.StageTimes()
    p = _params(we, ws, tolerance)
    check(lib().pamopt_cu_remesh_host(ctx.h, ptr(v), len(v), ptr(f), len(f), int(R),
                                      default_eps(R) if eps is None else float(eps), float(beta), int(target_faces),
                                      C.byref(p), C.byref(nv), C.byref(nf), C.byref(st), C.byref(tm)))
    vo = np.empty((nv.value, 3), np.float64)
    fo = np.empty((nf.value, 3), np.int32)
    check(lib().pamopt_cu_remesh_fetch(ctx.h, ptr(vo), ptr(fo)))
    return RemeshResult(vo, fo, st.as_dict(), tm.as_dict())


class CertificationError(_lib.PamoptError):
    """A run_pipeline stage failed its certification; .mesh is that stage's output."""

    def __init__(self, code, msg, mesh, report):
        super().__init__(code, msg)
        self.mesh = mesh
        self.report = report


def run_certified_pipeline(mesh, target_faces: int = 0, target_ratio: float = 0.01, resolution: int = 0,
                           run_projection: bool = False, eps: float = 0.0, beta: float = DEFAULT_BETA,
                           we: float = DEFAULT_WE, ws: float = DEFAULT_WS, tolerance: int = DEFAULT_TOL,
                           report_samples: int = 16384, seed: int = 42, ctx: Context | None = None):
    """run_pipeline: normalise a copy of the raw input, stage 1 (UDF -> DMC),
    certify (manifold, watertight, exact intersection check), stage 2 (QEM), certify (+ face
    target or the stall rule), optional stage 3 (safe projection), certify, denormalise.
    Returns (DeviceMesh, report dict); raises CertificationError if a stage fails."""
    m = _mesh(mesh, ctx)
    cfg = _lib.PipelineConfig()
    check(lib().pamopt_cu_pipeline_defaults(C.byref(cfg)))
    cfg.resolution = int(resolution)
    cfg.run_projection = 1 if run_projection else 0
    cfg.target_faces = int(target_faces)
    cfg.target_ratio = float(target_ratio)
    cfg.beta = float(beta)
    cfg.eps = float(eps)
    cfg.simplify = _params(we, ws, tolerance)
    cfg.report_samples = int(report_samples)
    cfg.seed = int(seed)
    h = C.c_void_p()
    rep = _lib.PipelineReport()
    rc = lib().pamopt_cu_run_pipeline(m.ctx.h, m.h, C.byref(cfg), C.byref(h), C.byref(rep))
    if rc == _lib.ECERT:
        raise CertificationError(rc, lib().pamopt_cu_last_error().decode(), DeviceMesh(h, m.ctx), rep.as_dict())
    check(rc)
    return DeviceMesh(h, m.ctx), rep.as_dict()


def remesh_device(mesh: DeviceMesh, R: int, target_faces: int, eps: float | None = None, beta: float = DEFAULT_BETA,
                  we: float = DEFAULT_WE, ws: float = DEFAULT_WS, tolerance: int = DEFAULT_TOL):
    """Device-resident pipeline (pamopt_cu_remesh): returns (DeviceMesh, stats, times)."""
    h = C.c_void_p()
    st = _lib.SimplifyStats()
    tm = _lib.StageTimes()
    p = _params(we, ws, tolerance)
    check(lib().pamopt_cu_remesh(mesh.ctx.h, mesh.h, int(R), default_eps(R) if eps is None else float(eps),
                                 float(beta), int(target_faces), C.byref(p), C.byref(h), C.byref(st), C.byref(tm)))
    return DeviceMesh(h, mesh.ctx), st.as_dict(), tm.as_dict()


# ------------------------------------------------------- certification / quality metrics
SAMPLE_SEED_B = 0x632BE59BD9B4E019


def analyze_topology(mesh, ctx: Context | None = None) -> dict:
    """analyze_topology (mesh.cpp:113-150) on the GPU: TopologySummary with the lists."""
    m = _mesh(mesh, ctx)
    t = _lib.Topology()
    check(lib().pamopt_cu_analyze_topology(m.h, C.byref(t), None, 0, None, 0))
    e = np.empty((t.n_nonmanifold_edges, 2), np.int32)
    v = np.empty(t.n_nonmanifold_vertices, np.int32)
    check(lib().pamopt_cu_analyze_topology(m.h, C.byref(t), ptr(e), len(e), ptr(v), len(v)))
    return dict(manifold=bool(t.manifold), watertight=bool(t.watertight), euler=int(t.euler_characteristic),
                boundary_edges=int(t.boundary_edge_count), nonmanifold_edges=e, nonmanifold_vertices=v)


def nearest_primitive(mesh, points, ctx: Context | None = None):
    """TriangleBvh::nearest_primitive (lbvh.cpp:192-237) per point: (face, distance, closest)."""
    m = _mesh(mesh, ctx)
    p = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    face = np.empty(len(p), np.int32)
    dist = np.empty(len(p))
    clo = np.empty((len(p), 3))
    check(lib().pamopt_cu_nearest_primitive(m.h, ptr(p), len(p), ptr(face), ptr(dist), ptr(clo)))
    return face, dist, clo


def sample_points(mesh, n: int, seed: int, ctx: Context | None = None):
    """The pinned area-weighted sampler: (points [n,3], face ids, total area)."""
    m = _mesh(mesh, ctx)
    pts = np.empty((n, 3))
    fid = np.empty(n, np.int32)
    area = C.c_double()
    check(lib().pamopt_cu_sample_points(m.h, int(n), int(seed) & (2**64 - 1), ptr(pts), ptr(fid), C.byref(area)))
    return pts, fid, area.value


def chamfer(a, b, n_samples: int = 16384, seed: int = 42, ctx: Context | None = None) -> float:
    ma, mb = _mesh(a, ctx), _mesh(b, ctx)
    out = C.c_double()
    check(lib().pamopt_cu_chamfer(ma.h, mb.h, int(n_samples), int(seed) & (2**64 - 1), C.byref(out)))
    return out.value


def hausdorff(a, b, n_samples: int = 16384, seed: int = 42, ctx: Context | None = None) -> float:
    ma, mb = _mesh(a, ctx), _mesh(b, ctx)
    out = C.c_double()
    check(lib().pamopt_cu_hausdorff(ma.h, mb.h, int(n_samples), int(seed) & (2**64 - 1), C.byref(out)))
    return out.value


def min_internal_angle(mesh, ctx: Context | None = None) -> float:
    m = _mesh(mesh, ctx)
    out = C.c_double()
    check(lib().pamopt_cu_min_internal_angle(m.h, C.byref(out)))
    return out.value


def mesh_report(mesh, reference=None, n_samples: int = 16384, seed: int = 42, ctx: Context | None = None) -> dict:
    """MeshReport (SPEC quality_metrics): cd/hd vs reference (NaN without one), min angle,
    manifold, watertight, intersection_free, counts."""
    m = _mesh(mesh, ctx)
    r = _mesh(reference, m.ctx) if reference is not None else None  # keep alive across the call
    out = _lib.MeshReport()
    check(lib().pamopt_cu_report(r.h if r is not None else None, m.h, int(n_samples), int(seed) & (2**64 - 1),
                                 C.byref(out)))
    d = out.as_dict()
    for k in ("manifold", "watertight", "intersection_free"):
        d[k] = bool(d[k])
    return d


# ------------------------------------------------------------------ ingest
def load_mesh_bytes(data: bytes, fmt: str, ctx: Context | None = None):
    """OBJ / PLY / STL bytes -> (DeviceMesh, LoadStats dict) with the reference's load_mesh
    semantics (mesh_io.cpp:46-384): binary bodies decoded and STL corners welded on the GPU."""
    ctx = ctx or default_context()
    buf = np.frombuffer(data, dtype=np.uint8)
    h = C.c_void_p()
    st = _lib.LoadStats()
    fn = {"stl": lib().pamopt_cu_load_stl, "ply": lib().pamopt_cu_load_ply, "obj": lib().pamopt_cu_load_obj}[fmt.lower()]
    check(fn(ctx.h, buf.ctypes.data, len(buf), C.byref(h), C.byref(st)))
    return DeviceMesh(h, ctx), st.as_dict()


def load_mesh(path: str, ctx: Context | None = None):
    """load_mesh (mesh_io.cpp:372-385) for .obj / .ply / .stl files."""
    ext = path.rsplit(".", 1)[-1].lower()
    with open(path, "rb") as fh:
        return load_mesh_bytes(fh.read(), ext, ctx)


def normalize_unit_cube(mesh: DeviceMesh, padding: float):
    """In place (mesh_io.cpp:393-408); returns (scale, translation)."""
    out = (C.c_double * 4)()
    check(lib().pamopt_cu_normalize_unit_cube(mesh.h, float(padding), out))
    return out[0], (out[1], out[2], out[3])


def denormalize(mesh: DeviceMesh, scale: float, translation) -> None:
    """In place (mesh_io.cpp:410-412): v = (v - translation) / scale."""
    st = (C.c_double * 4)(float(scale), *(float(t) for t in translation))
    check(lib().pamopt_cu_denormalize(mesh.h, st))


# ------------------------------------------------------------------ stage 3 (SPEC.md safe_project)
def project_defaults() -> dict:
    p = _lib.ProjectParams()
    check(lib().pamopt_cu_project_defaults(C.byref(p)))
    return {k: getattr(p, k) for k, _ in p._fields_}


def safe_project(mesh_s: DeviceMesh, mesh_in, **overrides):
    """project(mesh_s, mesh_in, params): deforms mesh_s in place (intersection-free trajectory);
    returns the stats dict.  Keyword overrides: iterations, refresh, samples, kdis, ..."""
    p = _lib.ProjectParams()
    check(lib().pamopt_cu_project_defaults(C.byref(p)))
    for k, v in overrides.items():
        setattr(p, k, v)
    mi = _mesh(mesh_in, mesh_s.ctx)
    st = _lib.ProjectStats()
    check(lib().pamopt_cu_safe_project(mesh_s.h, mi.h, C.byref(p), C.byref(st)))
    return st.as_dict()


def safe_project_traced(mesh_s: DeviceMesh, mesh_in, record: int, contact_cap: int = 1 << 16, **overrides):
    """safe_project with a per-iteration record of the first `record` Newton iterations (the
    step oracle's input): X, grad, dir, targets (record x nv x 3), m2s (record x m x 4),
    contacts (list of (n, 6) arrays), scalars (record x 8: B0, |g|, CG its, t_max, alpha, B1,
    accepted, tries), samples (m x 3).  Returns (stats, trace dict)."""
    p = _lib.ProjectParams()
    check(lib().pamopt_cu_project_defaults(C.byref(p)))
    for k, v in overrides.items():
        setattr(p, k, v)
    mi = _mesh(mesh_in, mesh_s.ctx)
    nv, m, K = mesh_s.size()[0], int(p.samples), int(record)
    buf = {"X": np.zeros((K, nv, 3)), "grad": np.zeros((K, nv, 3)), "dir": np.zeros((K, nv, 3)),
           "targets": np.zeros((K, nv, 3)), "m2s": np.zeros((K, m, 4), np.int32),
           "contacts": np.zeros((K, contact_cap, 6), np.int32), "n_contacts": np.zeros(K, np.int64),
           "scalars": np.full((K, 8), np.nan), "samples": np.zeros((m, 3))}
    tr = _lib.ProjectTrace(K, contact_cap, *(buf[k].ctypes.data for k in
                                             ("X", "grad", "dir", "targets", "m2s", "contacts", "n_contacts",
                                              "scalars", "samples")))
    st = _lib.ProjectStats()
    check(lib().pamopt_cu_safe_project_traced(mesh_s.h, mi.h, C.byref(p), C.byref(st), C.byref(tr)))
    n_it = min(K, int(st.iterations))
    buf["contacts"] = [buf["contacts"][i, :min(int(buf["n_contacts"][i]), contact_cap)].copy() for i in range(n_it)]
    for k in ("X", "grad", "dir", "targets", "m2s", "scalars", "n_contacts"):
        buf[k] = buf[k][:n_it]
    buf["params"] = {k: getattr(p, k) for k, _ in p._fields_}
    return st.as_dict(), buf


TERMS = {"s2m": 0, "m2s": 1, "elastic": 2, "bending": 3, "pt": 4, "ee": 5}


def project_term(term: str, coords, rest=None, cls: int = 0, ctx: Context | None = None, **overrides):
    """One stage-3 energy stencil on the GPU: (value, gradient, SPD-projected Hessian)."""
    ctx = ctx or default_context()
    x = np.ascontiguousarray(coords, np.float64).reshape(-1, 3)
    r = np.zeros(16)
    if rest is not None:
        r[:len(rest)] = rest
    p = _lib.ProjectParams()
    check(lib().pamopt_cu_project_defaults(C.byref(p)))
    for k, v in overrides.items():
        setattr(p, k, v)
    out = np.zeros(1 + 12 + 144)
    check(lib().pamopt_cu_project_term(ctx.h, TERMS[term], int(cls), ptr(x), len(x), ptr(r), C.byref(p), ptr(out)))
    n = 3 * len(x)
    return out[0], out[1:1 + n].copy(), out[13:13 + n * n].reshape(n, n).copy()
