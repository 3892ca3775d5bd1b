// kernels.cuh — host-side entry points of the device modules (udf.cu, dmc.cu, isect.cu,
// simplify.cu), called by the C-ABI layer in capi.cu.
#pragma once

#include <vector>

#include "common.cuh"

namespace pcu {

// ---- stage 1a (udf.cu)
// mode 0: UDF (+INF sentinel); mode 1: fused SDF (u - eps, sentinel +1.0)
// z-slab: only lattice planes [z0, z1) are computed and written (z1 < 0: the whole grid)
// d_signs (optional): the DMC sign mask of the written planes, (z1-z0)*(R+1) rows of
// ceil((R+1)/32) words; bit x&31 of word x>>5 = (sample < 0)
void udf_run(Ctx& ctx, const double* dV, int64_t nv, const int32_t* dF, int64_t nf, int R, int mode, double eps,
             float* d_out, int z0 = 0, int z1 = -1, uint32_t* d_signs = nullptr);
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
  // stage views (whole-grid extract with want_stages): build_patches / build_quads
  bool want_stages = false;
  DevBuf<uint32_t> vbase;  // first patch vertex per active cell
  uint64_t nv_patch = 0;
  DevBuf<int32_t> quads;   // 4 patch-vertex ids per quad (oriented - -> +)
  DevBuf<int64_t> qedge;   // lower lattice vertex * 3 + axis
  DevBuf<float> qf;        // samples at the edge's lower / upper vertex
  DevBuf<uint8_t> qsplit;  // 1: diagonal 0-2, 2: diagonal 1-3, 3: four triangles
};
// d_signs: the sign mask udf_run can emit for the same planes (NULL: packed here, one read)
void dmc_extract(Ctx& ctx, const float* d_sdf, int R, double beta, DmcResult& res, const uint32_t* d_signs = nullptr);
// z-slab extraction: d_planes holds lattice planes [pz0, pz1); cells of layers
// [own_z0, own_z1) emit faces; the layer below only lends vertex ids.  Face indices are relative
// to the first own patch vertex (negative = the previous slab's top layer); see mesh_rebase.
void dmc_extract_slab(Ctx& ctx, const float* d_planes, int R, int pz0, int pz1, int own_z0, int own_z1, double beta,
                      DmcResult& res, const uint32_t* d_signs = nullptr);
// F[i] -> patch_base + F[i] if F[i] < nvp_own, else extra_base + (F[i] - nvp_own)
void mesh_rebase(Ctx& ctx, int32_t* dF, int64_t nidx, int64_t patch_base, int64_t nvp_own, int64_t extra_base);
void dmc_table_host(int32_t* out);
// triangulate_quads on explicit quads (patch vertices + quads + valid-edge data): V = [patch
// vertices, extra vertices in quad order], faces in quad order
void triangulate_quads(Ctx& ctx, const double* d_patch_v, int64_t nv_patch, const int32_t* d_quads,
                       const int64_t* d_qedge, const float* d_qf, int64_t nq, int R, double beta, DevBuf<double>& V,
                       DevBuf<int32_t>& F, int64_t& nv, int64_t& nf);
// returns the number of entries whose samples do not change sign (SPEC.md:270 error)
int64_t interpolate_patch_vertex(Ctx& ctx, const double* d_p0, const double* d_p1, const float* d_f0, const float* d_f1,
                                 int64_t n, double beta, double* d_out);

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
// per-iteration record of the solve (host buffers, any may be null) for the step oracle in
// tests/test_gpu_project_steps.py: iterations [0, max_iters) are recorded
struct ProjectTrace {
  int max_iters = 0;
  int64_t contact_cap = 0;
  double* X = nullptr;          // max_iters x 3nv: positions at the start of the iteration
  double* grad = nullptr;       // max_iters x 3nv: assembled gradient
  double* dir = nullptr;        // max_iters x 3nv: PCG solution p of H p = -g
  double* targets = nullptr;    // max_iters x 3nv: S2M targets in use
  int32_t* m2s = nullptr;       // max_iters x m x 4: M2S stencil (3 vertices, frozen class)
  int32_t* contacts = nullptr;  // max_iters x contact_cap x 6: term, class, 4 vertices
  int64_t* n_contacts = nullptr;
  double* scalars = nullptr;    // max_iters x 8: B0, |g|, CG iterations, t_max, alpha, B1, accepted, tries
  double* samples = nullptr;    // 3m: the M2S samples on M_in
};
// deforms dV (mesh_s vertices) in place; connectivity unchanged
void safe_project(Ctx& ctx, double* dV, int64_t nv, const int32_t* dF, int64_t nf, const double* dVin,
                  const int32_t* dFin, int64_t nfin, const ProjectParams& params, ProjectStats& stats,
                  ProjectTrace* trace = nullptr);

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
// false (nothing decoded) when a face list is not a triangle: the layout is not fixed-size
bool load_ply_binary(Ctx& ctx, const uint8_t* d_bytes, const PlyBinaryLayout& layout, IngestResult& out);
// text formats (ingest_text.cu): OBJ, ASCII STL (GPU weld), PLY record by record
void load_obj_text(Ctx& ctx, const char* b, int64_t n, IngestResult& out, int64_t* triangulated);
void load_stl_ascii(Ctx& ctx, const char* b, int64_t n, IngestResult& out);
void load_ply_host(Ctx& ctx, const char* b, int64_t n, IngestResult& out, int64_t* triangulated);
// denormalize (mesh_io.cpp:410-412) with {scale, tx, ty, tz} from normalize_unit_cube
void denormalize(Ctx& ctx, double* dV, int64_t nv, const double* scale_translation);
void normalize_unit_cube(Ctx& ctx, double* dV, int64_t nv, double padding, double* scale_translation);

// ---- tri_isect (isect.cu)
// all intersecting pairs (i<j) among faces with alive[i] (alive may be null); if `query` is
// non-null only pairs with at least one query face are reported.  Result sorted (host).
std::vector<int32_t> self_intersections(Ctx& ctx, const double* dV, int64_t nv, const int32_t* dF, int64_t nf,
                                        const uint8_t* d_alive, const uint8_t* d_query);
void tri_tri_pairs(Ctx& ctx, const double* dV, const int32_t* dF, const int32_t* d_pairs, int64_t n, int32_t* d_out);
// classify_pair (shared count, coplanar flag) and the class-restricted verdicts (mode 1:
// intersect_3d, mode 2: intersect_coplanar; -1 = precondition violated)
void classify_pairs(Ctx& ctx, const double* dV, const int32_t* dF, const int32_t* d_pairs, int64_t n, int32_t* d_shared,
                    int32_t* d_coplanar);
void verdict_by_class(Ctx& ctx, const double* dV, const int32_t* dF, const int32_t* d_pairs, int64_t n, int mode,
                      int32_t* d_out);

// Broad phase + narrow phase of the QEM undo loop, asynchronous: results (found pairs, buffer
// overflow) are left in device scalars; detect_scalars_ptr/size let the caller fetch them in
// the same host synchronisation as its own counters.  d_owner[f] >= 0 names the applied collapse
// that modified face f (owner is set only for applied collapses and cleared on revert).
struct IsectScratch;
void undo_detect_async(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf,
                       const uint8_t* d_falive, const int32_t* d_query_faces, int64_t n_query, const int32_t* d_owner,
                       uint8_t* d_revert, std::initializer_list<FillRange> resets = {});
void undo_detect_restored_async(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf,
                                const uint8_t* d_falive, const int32_t* d_restored, int64_t n_restored,
                                const int32_t* d_owned, int64_t n_owned, const int32_t* d_owner,
                                uint8_t* d_revert, std::initializer_list<FillRange> resets = {});
void boxes_init(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf, const uint8_t* d_alive);
void boxes_update(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, const int32_t* ids, int64_t n,
                  const uint8_t* d_alive);
const void* detect_scalars_ptr(IsectScratch& S);
size_t detect_scalars_size();
void detect_grow(IsectScratch& S, unsigned long long ncand);
void detect_read(const void* host_copy, unsigned long long* found, int* redo, unsigned long long* ncand,
                 unsigned long long* ncls = nullptr);
IsectScratch* isect_scratch_create();
void isect_scratch_destroy(IsectScratch* s);

// ---- C4 slab path over NCCL (slab_nccl.cu): NCCL resolved at run time from the process
void* nccl_comm_init_all(int ndev, const int* devs, void** comms);
void nccl_comm_destroy(void* comm);
// rank 0 gets the assembled mesh in Vout/Fout (nv_out/nf_out); others get nv_out = nf_out = 0
void slab_extract_nccl(Ctx& ctx, const double* dV, int64_t nv, const int32_t* dF, int64_t nf, int R, double eps,
                       double beta, int rank, int world, void* comm, DevBuf<double>& Vout, DevBuf<int32_t>& Fout,
                       int64_t& nv_out, int64_t& nf_out, int64_t counts[3]);

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
// Stepwise QEM run (one object per simplify_to).  The mesh buffers are
// simplified in place; qem_finish compacts them.  Steps must be called in order per iteration.
struct QemState;
QemState* qem_create(Ctx& ctx, DevBuf<double>& V, DevBuf<int32_t>& F, int64_t& nv, int64_t& nf, int64_t target,
                     const SimplifyParams& P, SimplifyStats& S);
void qem_destroy(QemState* q);
bool qem_done(const QemState* q);
void qem_prepare(QemState* q);
void qem_propagate_and_mark(QemState* q);
void qem_collapse_batch(QemState* q);
void qem_undo_loop(QemState* q);
void qem_end_iteration(QemState* q);
void qem_finish(QemState* q);
int qem_phase(const QemState* q);
// device views of the current iteration (valid until the next step)
struct QemView {
  int64_t nv = 0, nf = 0, ne = 0, nm = 0, alive_faces = 0, succ = 0;
  int rounds = 0;
  const double* X = nullptr;
  const int32_t* F = nullptr;
  const uint8_t *falive = nullptr, *valive = nullptr;
  const double* Q = nullptr;
  const int32_t *ea = nullptr, *eb = nullptr;
  const uint64_t* key = nullptr;
  const double* place = nullptr;
  const uint8_t* valid = nullptr;
  const uint64_t* marked_sorted = nullptr;
  const uint32_t* rem = nullptr;
  const uint8_t* applied = nullptr;
};
QemView qem_view(QemState* q);
void qem_face_keys(QemState* q, uint64_t* d_out);  // per face: min key of its vertices' valid edges
// standalone SPEC operations on a whole mesh (every face alive); device arrays
void quadrics_of(Ctx& ctx, const double* X, const int32_t* F, int64_t nv, int64_t nf, double* dQ);
void edge_cost_of(Ctx& ctx, const double* X, const int32_t* F, int64_t nv, int64_t nf, const int32_t* d_edges,
                  int64_t n, double we, double ws, double* d_cost, double* d_place);
int64_t pack_cost_of(Ctx& ctx, const double* d_cost, const uint32_t* d_ids, int64_t n, uint64_t* d_keys);  // #NaN
void link_condition_of(Ctx& ctx, const int32_t* F, int64_t nv, int64_t nf, const int32_t* d_edges, int64_t n,
                       int32_t* d_out);  // 1 / 0, -1 = not an edge
// Simplifies in place.  On return dV/dF hold the compacted mesh (sizes updated).
void simplify_run(Ctx& ctx, DevBuf<double>& V, DevBuf<int32_t>& F, int64_t& nv, int64_t& nf, int64_t target,
                  const SimplifyParams& P, SimplifyStats& S);

}  // namespace pcu
