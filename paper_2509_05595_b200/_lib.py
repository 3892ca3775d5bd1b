"""ctypes binding of libpamopt_cu.so (the C-ABI in include/pamopt_cu.h).

There is no fallback: if the shared library is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PAMOPT_LIB") or os.path.join(HERE, "libpamopt_cu.so")  # PAMOPT_LIB: A/B variants only

OK, EINVAL, ECUDA, ENOMEM, ENUMERIC, ECAP, ECERT, EIO = 0, -1, -2, -3, -4, -5, -6, -7


class SimplifyParams(C.Structure):
    _fields_ = [("w_e", C.c_double), ("w_s", C.c_double), ("tolerance", C.c_int32),
                ("stall_iterations", C.c_int32)]


class SimplifyStats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("collapses", C.c_int64), ("undone", C.c_int64),
                ("link_failures", C.c_int64), ("max_undo_rounds", C.c_int64), ("undo_hist", C.c_int64 * 8),
                ("face_iterations", C.c_int64), ("alg_bytes", C.c_int64)]

    def as_dict(self) -> dict:
        return {"iterations": self.iterations, "collapses": self.collapses, "undone": self.undone,
                "link_failures": self.link_failures, "max_undo_rounds": self.max_undo_rounds,
                "undo_hist": list(self.undo_hist), "face_iterations": self.face_iterations,
                "alg_bytes": self.alg_bytes}


class StageTimes(C.Structure):
    _fields_ = [("udf_ms", C.c_float), ("dmc_ms", C.c_float), ("simplify_ms", C.c_float), ("total_ms", C.c_float),
                ("dmc_faces", C.c_int64), ("dmc_vertices", C.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class LoadStats(C.Structure):
    _fields_ = [("degenerate_faces_dropped", C.c_int64), ("polygons_triangulated", C.c_int64),
                ("vertices_welded", C.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class ProjectParams(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("refresh", C.c_int32), ("cg_max", C.c_int32), ("elas_power", C.c_int32),
                ("samples", C.c_int64), ("seed", C.c_uint64), ("kdis", C.c_double), ("kelas", C.c_double),
                ("kbend", C.c_double), ("kbar", C.c_double), ("dhat", C.c_double), ("cg_tol", C.c_double),
                ("elas_tau", C.c_double)]


class ProjectStats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("cg_iterations", C.c_int64), ("refreshes", C.c_int64),
                ("converged", C.c_int64), ("energy0", C.c_double), ("energy", C.c_double),
                ("grad_norm", C.c_double), ("last_alpha", C.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class ProjectTrace(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("contact_cap", C.c_int64), ("X", C.c_void_p), ("grad", C.c_void_p),
                ("dir", C.c_void_p), ("targets", C.c_void_p), ("m2s", C.c_void_p), ("contacts", C.c_void_p),
                ("n_contacts", C.c_void_p), ("scalars", C.c_void_p), ("samples", C.c_void_p)]


class Topology(C.Structure):
    _fields_ = [("manifold", C.c_int32), ("watertight", C.c_int32), ("euler_characteristic", C.c_int64),
                ("boundary_edge_count", C.c_int64), ("n_nonmanifold_edges", C.c_int64),
                ("n_nonmanifold_vertices", C.c_int64)]


class MeshReport(C.Structure):
    _fields_ = [("cd", C.c_double), ("hd", C.c_double), ("min_angle_deg", C.c_double), ("manifold", C.c_int32),
                ("watertight", C.c_int32), ("intersection_free", C.c_int32), ("pad_", C.c_int32),
                ("n_faces", C.c_int64), ("n_vertices", C.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad_"}


class PipelineConfig(C.Structure):
    _fields_ = [("resolution", C.c_int32), ("run_projection", C.c_int32), ("target_faces", C.c_int64),
                ("target_ratio", C.c_double), ("beta", C.c_double), ("eps", C.c_double),
                ("simplify", SimplifyParams), ("report_samples", C.c_int64), ("seed", C.c_uint64)]


class PipelineReport(C.Structure):
    _fields_ = [("stage", MeshReport * 3), ("failed_stage", C.c_int32), ("stalled", C.c_int32),
                ("resolution", C.c_int32), ("projected", C.c_int32), ("faces_in", C.c_int64),
                ("target_faces", C.c_int64), ("simplify", SimplifyStats), ("stage_ms", C.c_float * 4),
                ("total_ms", C.c_float), ("pad_", C.c_float), ("scale_translation", C.c_double * 4)]

    def as_dict(self) -> dict:
        n = 3 if self.projected else 2
        return {"stages": [self.stage[i].as_dict() for i in range(n)], "failed_stage": self.failed_stage,
                "stalled": bool(self.stalled), "resolution": self.resolution, "faces_in": self.faces_in,
                "target_faces": self.target_faces, "simplify": self.simplify.as_dict(),
                "stage_ms": {"stage1": self.stage_ms[0], "stage2": self.stage_ms[1], "stage3": self.stage_ms[2],
                             "certification": self.stage_ms[3]},
                "total_ms": self.total_ms, "scale_translation": list(self.scale_translation)}


class PamoptError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class PamoptInvalidArgument(PamoptError, ValueError):
    """Maps PAMOPT_CU_EINVAL (the reference's std::invalid_argument, mesh.cpp:186-187,302)."""


_L = None

vp = C.c_void_p
i64 = C.c_int64
i32 = C.c_int32
dbl = C.c_double
P = C.POINTER

_SIGS = {
    "pamopt_cu_last_error": (C.c_char_p, []),
    "pamopt_cu_version": (C.c_char_p, []),
    "pamopt_cu_ctx_create": (C.c_int, [i32, P(vp)]),
    "pamopt_cu_ctx_destroy": (C.c_int, [vp]),
    "pamopt_cu_ctx_stream": (vp, [vp]),
    "pamopt_cu_ctx_synchronize": (C.c_int, [vp]),
    "pamopt_cu_ctx_launches": (i64, [vp]),
    "pamopt_cu_ctx_profile": (C.c_int, [vp, i32]),
    "pamopt_cu_ctx_kernel_times": (i64, [vp, vp, i64]),
    "pamopt_cu_mesh_upload": (C.c_int, [vp, vp, i64, vp, i64, P(vp)]),
    "pamopt_cu_mesh_from_device": (C.c_int, [vp, vp, i64, vp, i64, P(vp)]),
    "pamopt_cu_mesh_size": (C.c_int, [vp, P(i64), P(i64)]),
    "pamopt_cu_mesh_download": (C.c_int, [vp, vp, vp]),
    "pamopt_cu_mesh_copy_to_device": (C.c_int, [vp, vp, vp]),
    "pamopt_cu_mesh_free": (C.c_int, [vp]),
    "pamopt_cu_load_stl": (C.c_int, [vp, vp, i64, P(vp), P(LoadStats)]),
    "pamopt_cu_load_ply": (C.c_int, [vp, vp, i64, P(vp), P(LoadStats)]),
    "pamopt_cu_load_obj": (C.c_int, [vp, vp, i64, P(vp), P(LoadStats)]),
    "pamopt_cu_normalize_unit_cube": (C.c_int, [vp, dbl, vp]),
    "pamopt_cu_denormalize": (C.c_int, [vp, vp]),
    "pamopt_cu_pipeline_defaults": (C.c_int, [P(PipelineConfig)]),
    "pamopt_cu_run_pipeline": (C.c_int, [vp, vp, P(PipelineConfig), P(vp), P(PipelineReport)]),
    "pamopt_cu_compute_udf": (C.c_int, [vp, vp, i32, P(vp)]),
    "pamopt_cu_udf_to_sdf": (C.c_int, [vp, dbl]),
    "pamopt_cu_compute_sdf": (C.c_int, [vp, vp, i32, dbl, P(vp)]),
    "pamopt_cu_compute_sdf_slab": (C.c_int, [vp, vp, i32, dbl, i32, i32, P(vp)]),
    "pamopt_cu_grid_slab": (C.c_int, [vp, P(i32), P(i32)]),
    "pamopt_cu_grid_copy_to_device": (C.c_int, [vp, vp]),
    "pamopt_cu_grid_from_device": (C.c_int, [vp, i32, vp, P(vp)]),
    "pamopt_cu_grid_upload": (C.c_int, [vp, i32, vp, P(vp)]),
    "pamopt_cu_grid_slab_from_device": (C.c_int, [vp, i32, i32, i32, vp, P(vp)]),
    "pamopt_cu_grid_slab_upload": (C.c_int, [vp, i32, i32, i32, vp, P(vp)]),
    "pamopt_cu_grid_resolution": (C.c_int, [vp, P(i32)]),
    "pamopt_cu_grid_download": (C.c_int, [vp, vp]),
    "pamopt_cu_grid_free": (C.c_int, [vp]),
    "pamopt_cu_hierarchy_pairs": (C.c_int, [vp, vp, i32, i32, vp, i64, P(i64)]),
    "pamopt_cu_dmc_extract": (C.c_int, [vp, dbl, P(vp)]),
    "pamopt_cu_dmc_extract_slab": (C.c_int, [vp, i32, i32, dbl, P(vp), P(i64)]),
    "pamopt_cu_mesh_rebase": (C.c_int, [vp, i64, i64, i64]),
    "pamopt_cu_extract_slab_nccl": (C.c_int, [vp, vp, i32, dbl, dbl, i32, i32, vp, P(vp), vp]),
    "pamopt_cu_nccl_comm_init_all": (C.c_int, [i32, vp, vp]),
    "pamopt_cu_nccl_comm_destroy": (C.c_int, [vp]),
    "pamopt_cu_dmc_active_cells": (C.c_int, [vp, vp, vp, vp, i64, P(i64)]),
    "pamopt_cu_dmc_table": (C.c_int, [vp]),
    "pamopt_cu_dmc_stages": (C.c_int, [vp, dbl, vp]),
    "pamopt_cu_dmc_build_patches": (C.c_int, [vp, vp, vp]),
    "pamopt_cu_dmc_build_quads": (C.c_int, [vp, vp, vp, vp, vp]),
    "pamopt_cu_triangulate_quads": (C.c_int, [vp, i32, vp, i64, vp, vp, vp, i64, dbl, P(vp)]),
    "pamopt_cu_interpolate_patch_vertex": (C.c_int, [vp, vp, vp, vp, vp, i64, dbl, vp]),
    "pamopt_cu_self_intersections": (C.c_int, [vp, vp, i64, P(i64)]),
    "pamopt_cu_tri_tri_pairs": (C.c_int, [vp, vp, i64, vp]),
    "pamopt_cu_classify_pair": (C.c_int, [vp, vp, i64, vp, vp]),
    "pamopt_cu_intersect_3d": (C.c_int, [vp, vp, i64, vp]),
    "pamopt_cu_intersect_coplanar": (C.c_int, [vp, vp, i64, vp]),
    "pamopt_cu_simplify": (C.c_int, [vp, i64, P(SimplifyParams), P(SimplifyStats), vp, i64]),
    "pamopt_cu_quadrics": (C.c_int, [vp, vp]),
    "pamopt_cu_edge_cost": (C.c_int, [vp, vp, i64, dbl, dbl, vp, vp]),
    "pamopt_cu_pack_cost": (C.c_int, [vp, vp, vp, i64, vp]),
    "pamopt_cu_link_condition": (C.c_int, [vp, vp, i64, vp]),
    "pamopt_cu_qem_create": (C.c_int, [vp, i64, P(SimplifyParams), P(vp)]),
    "pamopt_cu_qem_done": (C.c_int, [vp, P(i32)]),
    "pamopt_cu_qem_prepare": (C.c_int, [vp, P(i64)]),
    "pamopt_cu_qem_edges": (C.c_int, [vp, vp, vp, vp, vp, i64]),
    "pamopt_cu_qem_propagate_and_mark": (C.c_int, [vp, P(i64)]),
    "pamopt_cu_qem_marked": (C.c_int, [vp, vp, i64, vp, i64]),
    "pamopt_cu_qem_collapse_batch": (C.c_int, [vp, vp, i64]),
    "pamopt_cu_qem_undo_loop": (C.c_int, [vp, P(i32), P(i64), vp, i64]),
    "pamopt_cu_qem_end_iteration": (C.c_int, [vp, P(i64)]),
    "pamopt_cu_qem_mesh": (C.c_int, [vp, vp, vp, vp, P(i64), P(i64)]),
    "pamopt_cu_qem_finish": (C.c_int, [vp, P(SimplifyStats)]),
    "pamopt_cu_qem_destroy": (C.c_int, [vp]),
    "pamopt_cu_analyze_topology": (C.c_int, [vp, P(Topology), vp, i64, vp, i64]),
    "pamopt_cu_nearest_primitive": (C.c_int, [vp, vp, i64, vp, vp, vp]),
    "pamopt_cu_sample_points": (C.c_int, [vp, i64, C.c_uint64, vp, vp, P(dbl)]),
    "pamopt_cu_chamfer": (C.c_int, [vp, vp, i64, C.c_uint64, P(dbl)]),
    "pamopt_cu_hausdorff": (C.c_int, [vp, vp, i64, C.c_uint64, P(dbl)]),
    "pamopt_cu_min_internal_angle": (C.c_int, [vp, P(dbl)]),
    "pamopt_cu_report": (C.c_int, [vp, vp, i64, C.c_uint64, P(MeshReport)]),
    "pamopt_cu_project_defaults": (C.c_int, [P(ProjectParams)]),
    "pamopt_cu_safe_project": (C.c_int, [vp, vp, P(ProjectParams), P(ProjectStats)]),
    "pamopt_cu_safe_project_traced": (C.c_int, [vp, vp, P(ProjectParams), P(ProjectStats), P(ProjectTrace)]),
    "pamopt_cu_project_term": (C.c_int, [vp, i32, i32, vp, i32, vp, P(ProjectParams), vp]),
    "pamopt_cu_remesh": (C.c_int, [vp, vp, i32, dbl, dbl, i64, P(SimplifyParams), P(vp), P(SimplifyStats),
                                   P(StageTimes)]),
    "pamopt_cu_remesh_host": (C.c_int, [vp, vp, i64, vp, i64, i32, dbl, dbl, i64, P(SimplifyParams), P(i64),
                                        P(i64), P(SimplifyStats), P(StageTimes)]),
    "pamopt_cu_remesh_fetch": (C.c_int, [vp, vp, vp]),
}

EXPORTS = tuple(_SIGS)


def lib():
    global _L
    if _L is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("PAMOPT_LIB") and not hasattr(L, name):
                continue  # A/B variant library built from another revision
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _L = L
    return _L


def check(rc: int) -> None:
    if rc != OK:
        msg = lib().pamopt_cu_last_error().decode()
        if rc == EINVAL:
            raise PamoptInvalidArgument(rc, msg)
        raise PamoptError(rc, msg)


def ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)
