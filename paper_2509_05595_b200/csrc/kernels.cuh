// kernels.cuh — host-side entry points of the device modules (udf.cu, dmc.cu, isect.cu,
// simplify.cu), called by the C-ABI layer in capi.cu.
#pragma once

#include <vector>

#include "common.cuh"

namespace pcu {

// ---- stage 1a (udf.cu)
// mode 0: UDF (+INF sentinel); mode 1: fused SDF (u - eps, sentinel +1.0)
// z-slab: only lattice planes [z0, z1) are computed and written (z1 < 0: the whole grid)
void udf_run(Ctx& ctx, const double* dV, int64_t nv, const int32_t* dF, int64_t nf, int R, int mode, double eps,
             float* d_out, int z0 = 0, int z1 = -1);
void udf_to_sdf_inplace(Ctx& ctx, float* g, int64_t n, double eps);
std::vector<int64_t> hierarchy_pairs(Ctx& ctx, const double* dV, const int32_t* dF, int64_t nf, int R, int r);

// ---- stage 1b (dmc.cu)
struct DmcResult {
  DevBuf<uint32_t> cells;
  DevBuf<uint8_t> cases, flips;
  uint32_t n_active = 0;
  DevBuf<double> V;
  DevBuf<int32_t> F;
  uint64_t nv = 0, nf = 0, n_quads = 0;
  uint64_t nvp_own = 0, n_extra = 0;  // V = [own patch vertices, extra (4-split) vertices]
};
void dmc_extract(Ctx& ctx, const float* d_sdf, int R, double beta, DmcResult& res);
// z-slab extraction: d_planes holds lattice planes [pz0, pz1); cells of layers
// [own_z0, own_z1) emit faces; the layer below only lends vertex ids.  Face indices are relative
// to the first own patch vertex (negative = the previous slab's top layer); see mesh_rebase.
void dmc_extract_slab(Ctx& ctx, const float* d_planes, int R, int pz0, int pz1, int own_z0, int own_z1, double beta,
                      DmcResult& res);
// F[i] -> patch_base + F[i] if F[i] < nvp_own, else extra_base + (F[i] - nvp_own)
void mesh_rebase(Ctx& ctx, int32_t* dF, int64_t nidx, int64_t patch_base, int64_t nvp_own, int64_t extra_base);
void dmc_table_host(int32_t* out);

// ---- certification / quality metrics (metrics.cu)
struct TopologyResult {
  int32_t manifold = 0, watertight = 0;
  int64_t euler = 0, boundary = 0;
  std::vector<uint64_t> nm_edges;  // (a<<32|b), ascending
  std::vector<int32_t> nm_verts;   // ascending
};
void analyze_topology(Ctx& ctx, const int32_t* dF, int64_t nf, int64_t nv, TopologyResult& out);
// nearest face per point (lbvh.cpp:192-237 semantics): squared distance, face (-1: none), closest
void nearest_primitive(Ctx& ctx, const double* dV, const int32_t* dF, int64_t nf, const double* d_pts, int64_t n,
                       int32_t* d_face, double* d_d2, double* d_closest);
// pinned area-weighted sampler; false for a zero-area (or empty) mesh
bool sample_points(Ctx& ctx, const double* dV, const int32_t* dF, int64_t nf, int64_t n, uint64_t seed,
                   double* d_pts, int32_t* d_fid, double* total_area);
void directed_d2(Ctx& ctx, const double* Va, const int32_t* Fa, int64_t nfa, const double* Vb, const int32_t* Fb,
                 int64_t nfb, int64_t n, uint64_t seed, double& sum_d2, double& max_d2, double& area_a);
double max_corner_cos(Ctx& ctx, const double* dV, const int32_t* dF, int64_t nf);
std::vector<int32_t> index_range(Ctx& ctx, const int32_t* d, int64_t n);  // {min, max}
// IndexedMesh::validate (mesh.cpp:31-43): throws EINVAL naming the first invalid face
void validate_mesh(Ctx& ctx, const int32_t* dF, int64_t nf, int64_t nv);

// ---- stage 3: safe projection (project.cu, SPEC.md safe_project)
struct ProjectParams {
  int iterations = 50, refresh = 10, cg_max = 1000, elas_power = 1;
  int64_t samples = 16384;
  uint64_t seed = 42;
  double kdis = 1e3, kelas = 1e-1, kbend = 1e-2, kbar = 1e2, dhat = 1e-3, cg_tol = 1e-3, elas_tau = 1e-12;
};
struct ProjectStats {
  int64_t iterations = 0, cg_iterations = 0, refreshes = 0, converged = 0;
  double energy0 = 0, energy = 0, grad_norm = 0, last_alpha = 0;
};
// deforms dV (mesh_s vertices) in place; connectivity unchanged
void safe_project(Ctx& ctx, double* dV, int64_t nv, const int32_t* dF, int64_t nf, const double* dVin,
                  const int32_t* dFin, int64_t nfin, const ProjectParams& params, ProjectStats& stats);

// one term stencil evaluated on the GPU (unit checks): out = {value, grad[12], projected H[144]}
void project_term_probe(Ctx& ctx, int term, int cls, const double* coords, int nv, const double* rest,
                        const ProjectParams& params, double* out);

// ---- ingest (ingest.cu)
struct IngestResult {
  DevBuf<double> V;
  DevBuf<int32_t> F;
  int64_t nv = 0, nf = 0, welded = 0, degenerate_dropped = 0;
};
// body offsets/types of a binary little-endian PLY (header parsed on the host); types: 0 float,
// 1 double, 2 int32, 3 uint32, 4 int8, 5 uint8, 6 int16, 7 uint16
struct PlyBinaryLayout {
  int64_t vbase = 0, vstride = 0, nvert = 0;
  int off[3] = {0, 0, 0}, type[3] = {0, 0, 0};
  int64_t fbase = 0, fstride = 0, nface = 0;
  int count_off = 0, count_type = 5, index_off = 1, index_type = 2;
};
void load_stl_binary(Ctx& ctx, const uint8_t* d_bytes, int64_t nbytes, uint32_t count, IngestResult& out);
void load_ply_binary(Ctx& ctx, const uint8_t* d_bytes, const PlyBinaryLayout& layout, IngestResult& out);
void normalize_unit_cube(Ctx& ctx, double* dV, int64_t nv, double padding, double* scale_translation);

// ---- tri_isect (isect.cu)
// all intersecting pairs (i<j) among faces with alive[i] (alive may be null); if `query` is
// non-null only pairs with at least one query face are reported.  Result sorted (host).
std::vector<int32_t> self_intersections(Ctx& ctx, const double* dV, int64_t nv, const int32_t* dF, int64_t nf,
                                        const uint8_t* d_alive, const uint8_t* d_query);
void tri_tri_pairs(Ctx& ctx, const double* dV, const int32_t* dF, const int32_t* d_pairs, int64_t n, int32_t* d_out);

// Broad phase + narrow phase of the QEM undo loop, asynchronous: results (found pairs, buffer
// overflow) are left in device scalars; detect_scalars_ptr/size let the caller fetch them in
// the same host synchronisation as its own counters.  d_owner[f] >= 0 names the applied collapse
// that modified face f (owner is set only for applied collapses and cleared on revert).
struct IsectScratch;
void undo_detect_async(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf,
                       const uint8_t* d_falive, const int32_t* d_query_faces, int64_t n_query, const int32_t* d_owner,
                       uint8_t* d_revert);
void undo_detect_restored_async(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf,
                                const uint8_t* d_falive, const int32_t* d_restored, int64_t n_restored,
                                const int32_t* d_owned, int64_t n_owned, const int32_t* d_owner,
                                uint8_t* d_revert);
void boxes_init(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf, const uint8_t* d_alive);
void boxes_update(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, const int32_t* ids, int64_t n,
                  const uint8_t* d_alive);
const void* detect_scalars_ptr(IsectScratch& S);
size_t detect_scalars_size();
void detect_grow(IsectScratch& S, unsigned long long ncand);
void detect_read(const void* host_copy, unsigned long long* found, int* redo, unsigned long long* ncand);
IsectScratch* isect_scratch_create();
void isect_scratch_destroy(IsectScratch* s);

// ---- stage 2 (simplify.cu)
struct SimplifyParams {
  double we = 1e-3, ws = 5e-3;
  int tolerance = 4, stall = 10;
};
struct SimplifyStats {
  int64_t iterations = 0, collapses = 0, undone = 0, link_failures = 0, max_undo_rounds = 0;
  int64_t undo_hist[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t face_iterations = 0, alg_bytes = 0;
  std::vector<int64_t> per_iter;
};
// Simplifies in place.  On return dV/dF hold the compacted mesh (sizes updated).
void simplify_run(Ctx& ctx, DevBuf<double>& V, DevBuf<int32_t>& F, int64_t& nv, int64_t& nf, int64_t target,
                  const SimplifyParams& P, SimplifyStats& S);

}  // namespace pcu
