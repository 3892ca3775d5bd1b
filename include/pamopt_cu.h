/* pamopt_cu.h — C-ABI of the B200-native remesh hot path (UDF -> DMC -> QEM with
 * self-intersection undo).  Plain pointers and sizes only; no torch or C++ types.
 *
 * The reference (`/root/reference/proj`, namespace pamopt) is an in-process C++ library with
 * no FFI; its hot-path modules exist only as SPEC operations (the .cpp files
 * are listed at proj/CMakeLists.txt:19-23,26 but absent).  Each entry below replaces one
 * reference operation; the C++ drop-in headers in include/pamopt/ wrap them under the
 * reference names:
 *
 *   pamopt_cu_mesh_*            IndexedMesh (mesh.hpp:18-33): f64 AoS vertices, i32 faces
 *   pamopt_cu_compute_udf       build_hierarchy + compute_udf
 *   pamopt_cu_udf_to_sdf        udf_to_sdf
 *   pamopt_cu_hierarchy_pairs   VoxelHierarchy level view, debug/parity
 *   pamopt_cu_dmc_extract       dual_mc::extract
 *   pamopt_cu_self_intersections  detect_self_intersections
 *   pamopt_cu_tri_tri_pairs     classify_pair + intersect_3d/intersect_coplanar
 *   pamopt_cu_simplify          simplify_to
 *   pamopt_cu_remesh            run_pipeline stages 1-2 (stage 3 excluded)
 *
 * Conventions.  Every function returns PAMOPT_CU_OK (0) or a negative status; the message
 * of the last failure on the calling thread is pamopt_cu_last_error().  The C++ wrappers map
 * PAMOPT_CU_EINVAL to std::invalid_argument (mesh.cpp:186-187,302) and the others to
 * std::runtime_error.  A context binds one device and one CUDA stream; handles created from a
 * context run on its stream.  Calls on distinct contexts are thread-safe.  Variable-size
 * results are count-then-fill (pass NULL to get the count), mirroring the 2-kernel gather.
 */
#ifndef PAMOPT_CU_H_
#define PAMOPT_CU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PAMOPT_CU_OK 0
#define PAMOPT_CU_EINVAL -1   /* invalid argument / invalid mesh / out-of-range parameter */
#define PAMOPT_CU_ECUDA -2    /* CUDA runtime failure */
#define PAMOPT_CU_ENOMEM -3   /* device allocation failure */
#define PAMOPT_CU_ENUMERIC -4 /* NaN edge cost */
#define PAMOPT_CU_ECAP -5     /* reserved (no fixed per-element capacity remains) */
#define PAMOPT_CU_EIO -7      /* malformed / truncated / empty mesh file (std::runtime_error, mesh_io.cpp:17-21) */

typedef struct pamopt_cu_ctx_s* pamopt_cu_ctx;
typedef struct pamopt_cu_mesh_s* pamopt_cu_mesh;
typedef struct pamopt_cu_grid_s* pamopt_cu_grid;

/* simplify parameters */
typedef struct {
  double w_e;             /* edge-length weight, default 1e-3 */
  double w_s;             /* skinny-triangle weight, default 5e-3 */
  int32_t tolerance;      /* invalid-flag retention, default 4 */
  int32_t stall_iterations; /* stall rule, default 10 */
} pamopt_cu_simplify_params;

typedef struct {
  int64_t iterations;
  int64_t collapses;
  int64_t undone;
  int64_t link_failures;
  int64_t max_undo_rounds;
  int64_t undo_hist[8]; /* batches needing k undo rounds (index 7 = 7 or more) */
  int64_t face_iterations; /* sum over iterations of the alive face count (work units) */
  int64_t alg_bytes;       /* SURVEY §8(d) QEM algorithmic bytes: sum 28 F_i + 92 V_i + 8 E_i */
} pamopt_cu_simplify_stats;

typedef struct {
  float udf_ms;      /* build_hierarchy + compute_udf + udf_to_sdf */
  float dmc_ms;      /* extract */
  float simplify_ms; /* simplify_to incl. undo loops */
  float total_ms;
  int64_t dmc_faces;
  int64_t dmc_vertices;
} pamopt_cu_stage_times;

const char* pamopt_cu_last_error(void);
const char* pamopt_cu_version(void);

/* ---- context ---------------------------------------------------------------------- */
int pamopt_cu_ctx_create(int32_t device, pamopt_cu_ctx* out);
int pamopt_cu_ctx_destroy(pamopt_cu_ctx ctx);
/* the cudaStream_t the context launches on (for event timing by the caller) */
void* pamopt_cu_ctx_stream(pamopt_cu_ctx ctx);
int pamopt_cu_ctx_synchronize(pamopt_cu_ctx ctx);
/* number of kernels this context launched since creation (telemetry) */
int64_t pamopt_cu_ctx_launches(pamopt_cu_ctx ctx);
/* per-kernel device-time accounting (CUDA events around every launch; diagnostics only, it
 * perturbs timing): on != 0 starts a fresh tally.  kernel_times writes
 * "name\tms\tlaunches\n" lines (NUL-terminated, truncated to cap) and returns the full length. */
int pamopt_cu_ctx_profile(pamopt_cu_ctx ctx, int on);
int64_t pamopt_cu_ctx_kernel_times(pamopt_cu_ctx ctx, char* buf, int64_t cap);

/* ---- meshes (IndexedMesh) ------------------------------------------------------------ */
int pamopt_cu_mesh_upload(pamopt_cu_ctx ctx, const double* vertices, int64_t nv,
                          const int32_t* faces, int64_t nf, pamopt_cu_mesh* out);
/* same, from device pointers (copied device-to-device) */
int pamopt_cu_mesh_from_device(pamopt_cu_ctx ctx, const double* d_vertices, int64_t nv,
                               const int32_t* d_faces, int64_t nf, pamopt_cu_mesh* out);
int pamopt_cu_mesh_size(pamopt_cu_mesh mesh, int64_t* nv, int64_t* nf);
int pamopt_cu_mesh_download(pamopt_cu_mesh mesh, double* vertices, int32_t* faces);
/* device-to-device copy into caller buffers (NCCL gather of slab meshes); either may be NULL */
int pamopt_cu_mesh_copy_to_device(pamopt_cu_mesh mesh, double* d_vertices, int32_t* d_faces);
int pamopt_cu_mesh_free(pamopt_cu_mesh mesh);

/* ---- ingest: file bytes in host memory -> device mesh --------------- */
/* LoadStats (mesh_io.hpp:11-15) */
typedef struct {
  int64_t degenerate_faces_dropped;
  int64_t polygons_triangulated;
  int64_t vertices_welded;
} pamopt_cu_load_stats;
/* load_stl (mesh_io.cpp:309-366), binary or ASCII: corners welded by exact equality on the GPU,
 * vertices in first-occurrence order, repeated-index faces dropped.  Errors -> PAMOPT_CU_EIO. */
int pamopt_cu_load_stl(pamopt_cu_ctx ctx, const void* bytes, int64_t nbytes, pamopt_cu_mesh* out,
                       pamopt_cu_load_stats* stats);
/* load_ply (mesh_io.cpp:135-255): binary_little_endian bodies with 3-index face lists (the
 * reference writer's layout) are decoded on the GPU; ASCII bodies and variable-length face lists
 * are decoded record by record (polygons fanned, mesh_io.cpp:32-42).  Errors -> PAMOPT_CU_EIO. */
int pamopt_cu_load_ply(pamopt_cu_ctx ctx, const void* bytes, int64_t nbytes, pamopt_cu_mesh* out,
                       pamopt_cu_load_stats* stats);
/* load_obj (mesh_io.cpp:46-82): v / f lines, 1-based and negative (relative) indices, /vt/vn
 * suffixes ignored, polygons fanned (mesh_io.cpp:32-42).  Errors -> PAMOPT_CU_EIO. */
int pamopt_cu_load_obj(pamopt_cu_ctx ctx, const void* bytes, int64_t nbytes, pamopt_cu_mesh* out,
                       pamopt_cu_load_stats* stats);
/* normalize_unit_cube (mesh_io.cpp:393-408), in place; scale_translation = {scale, tx, ty, tz} or NULL */
int pamopt_cu_normalize_unit_cube(pamopt_cu_mesh mesh, double padding, double* scale_translation);
/* denormalize (mesh_io.cpp:410-412), in place: v = (v - t) / scale */
int pamopt_cu_denormalize(pamopt_cu_mesh mesh, const double* scale_translation);

/* ---- stage 1a: voxel_field --------------------------------------------------------- */
/* R: power of two >= 8.  Returns the UDF lattice ((R+1)^3 f32, x-fastest, +INF sentinel). */
int pamopt_cu_compute_udf(pamopt_cu_ctx ctx, pamopt_cu_mesh mesh, int32_t R, pamopt_cu_grid* out);
/* in place; PAMOPT_CU_EINVAL unless sqrt(3)/(2R) <= eps <= 3/R - sqrt(3)/(2R) */
int pamopt_cu_udf_to_sdf(pamopt_cu_grid grid, double eps);
/* fused compute_udf + udf_to_sdf (the pipeline path) */
int pamopt_cu_compute_sdf(pamopt_cu_ctx ctx, pamopt_cu_mesh mesh, int32_t R, double eps,
                          pamopt_cu_grid* out);
/* z-slab of the SDF lattice: planes [z0, z1) only (multi-GPU slab decomposition) */
int pamopt_cu_compute_sdf_slab(pamopt_cu_ctx ctx, pamopt_cu_mesh mesh, int32_t R, double eps, int32_t z0,
                               int32_t z1, pamopt_cu_grid* out);
int pamopt_cu_grid_slab(pamopt_cu_grid grid, int32_t* z0, int32_t* z1);
/* device-to-device exchange with caller buffers (NCCL halo exchange / gather) */
int pamopt_cu_grid_copy_to_device(pamopt_cu_grid grid, void* dst);
int pamopt_cu_grid_from_device(pamopt_cu_ctx ctx, int32_t R, const float* src, pamopt_cu_grid* out);
/* a z-slab grid holding lattice planes [z0, z1) from device (src) or host (samples) memory */
int pamopt_cu_grid_slab_from_device(pamopt_cu_ctx ctx, int32_t R, int32_t z0, int32_t z1, const float* src,
                                    pamopt_cu_grid* out);
int pamopt_cu_grid_slab_upload(pamopt_cu_ctx ctx, int32_t R, int32_t z0, int32_t z1, const float* samples,
                               pamopt_cu_grid* out);
int pamopt_cu_grid_upload(pamopt_cu_ctx ctx, int32_t R, const float* samples, pamopt_cu_grid* out);
int pamopt_cu_grid_resolution(pamopt_cu_grid grid, int32_t* R);
int pamopt_cu_grid_download(pamopt_cu_grid grid, float* samples);
int pamopt_cu_grid_free(pamopt_cu_grid grid);
/* surviving (cell, triangle) pairs of hierarchy level r (8 <= r <= R), sorted by (cell, tri);
 * pairs = int64[2*n] or NULL (count only).  Debug/parity view of build_hierarchy. */
int pamopt_cu_hierarchy_pairs(pamopt_cu_ctx ctx, pamopt_cu_mesh mesh, int32_t R, int32_t r,
                              int64_t* pairs, int64_t cap, int64_t* n);

/* ---- stage 1b: dual_mc -------------------------------------------------------------- */
int pamopt_cu_dmc_extract(pamopt_cu_grid sdf, double beta, pamopt_cu_mesh* out);
/* slab-local extract: the grid holds planes [z0, z1) covering [own_z0-2,
 * own_z1+2) clipped to the lattice; cells of layers [own_z0, own_z1) emit the faces of their
 * corner-0 edges, in the same order as the whole-grid extract.  out mesh V = [own patch
 * vertices (counts[0]), 4-split vertices (counts[1])]; face indices are relative to the first own
 * patch vertex, negative ones naming the previous slab's top layer.  Assemble with
 * pamopt_cu_mesh_rebase: concatenating every slab's patch vertices, then every slab's split
 * vertices, reproduces the whole-grid mesh bit for bit. */
int pamopt_cu_dmc_extract_slab(pamopt_cu_grid sdf, int32_t own_z0, int32_t own_z1, double beta,
                               pamopt_cu_mesh* out, int64_t counts[2]);
/* The whole C4 slab path for a C++ host, one rank (process or thread) per GPU over an NCCL
 * communicator (ncclComm_t passed as void*; world == 1 may pass NULL): the SDF of this rank's
 * lattice planes, a HALO=2-plane ncclSend/ncclRecv exchange with the z-neighbours, slab-local
 * DMC, an ncclAllGather of the counts and a grouped send of every slab mesh into place on rank
 * 0.  Rank 0's out is the assembled mesh, bit-identical to pamopt_cu_dmc_extract of the whole
 * grid; other ranks get out = NULL.  counts = this slab's {patch vertices, split vertices,
 * faces}.  NCCL is resolved at run time from the process (libnccl.so.2); none -> ECUDA. */
int pamopt_cu_extract_slab_nccl(pamopt_cu_ctx ctx, pamopt_cu_mesh mesh, int32_t R, double eps, double beta,
                                int32_t rank, int32_t world, void* nccl_comm, pamopt_cu_mesh* out, int64_t counts[3]);
/* ncclCommInitAll for a single host process driving ndev GPUs: comms[ndev] */
int pamopt_cu_nccl_comm_init_all(int32_t ndev, const int32_t* devices, void** comms);
int pamopt_cu_nccl_comm_destroy(void* comm);
/* in place: F -> patch_base + F if F < nvp_own, else extra_base + (F - nvp_own) */
int pamopt_cu_mesh_rebase(pamopt_cu_mesh mesh, int64_t patch_base, int64_t nvp_own, int64_t extra_base);
/* active cells of the last extract on this grid: linear cell index, case, flip mask */
int pamopt_cu_dmc_active_cells(pamopt_cu_grid sdf, int64_t* cells, uint8_t* cases,
                               uint8_t* flips, int64_t cap, int64_t* n);
/* the 256-entry patch table: per case {n, mask0..3, doubly-covered faces} (int32[256*6]) */
int pamopt_cu_dmc_table(int32_t* out);

/* SPEC-granular dual_mc operations.  pamopt_cu_dmc_stages runs classify_voxels
 * + build_patches + build_quads on a whole grid and keeps the views on the grid handle:
 * counts = {n_active, n_patch_vertices, n_quads}. */
int pamopt_cu_dmc_stages(pamopt_cu_grid sdf, double beta, int64_t counts[3]);
/* build_patches view: patch vertices double[3 n_patch_vertices] in (active cell, patch) order and
 * the first patch vertex of every active cell, int64[n_active]; either may be NULL */
int pamopt_cu_dmc_build_patches(pamopt_cu_grid sdf, double* vertices, int64_t* patch_first);
/* build_quads view, one quad per valid interior grid edge in output order: quads int32[4 n]
 * (patch-vertex ids, oriented negative -> positive), edges int64[n] = lower lattice vertex
 * linear index * 3 + axis, samples float[2 n] at the edge's lower / upper vertex, split uint8[n]
 * = triangulate_quads' decision (1 diagonal 0-2, 2 diagonal 1-3, 3 four triangles) */
int pamopt_cu_dmc_build_quads(pamopt_cu_grid sdf, int32_t* quads, int64_t* edges, float* samples, uint8_t* split);
/* triangulate_quads on explicit quads: out mesh V = [patch vertices, the
 * extra 4-split vertices in quad order], faces in quad order (== extract for build_quads' output) */
int pamopt_cu_triangulate_quads(pamopt_cu_ctx ctx, int32_t R, const double* patch_vertices, int64_t n_vertices,
                                const int32_t* quads, const int64_t* edges, const float* samples, int64_t n_quads,
                                double beta, pamopt_cu_mesh* out);
/* interpolate_patch_vertex for n edges: p0, p1 double[3n], f0, f1 float[n] ->
 * out double[3n]; PAMOPT_CU_EINVAL if some f0, f1 do not change sign (those outputs are 0) */
int pamopt_cu_interpolate_patch_vertex(pamopt_cu_ctx ctx, const double* p0, const double* p1, const float* f0,
                                       const float* f1, int64_t n, double beta, double* out);

/* ---- tri_isect ------------------------------------------------------------------------ */
/* all intersecting face pairs (f1<f2), sorted; pairs = int32[2*n] or NULL */
int pamopt_cu_self_intersections(pamopt_cu_mesh mesh, int32_t* pairs, int64_t cap, int64_t* n);
/* narrow-phase verdict for explicit face pairs (host arrays) */
int pamopt_cu_tri_tri_pairs(pamopt_cu_mesh mesh, const int32_t* pairs, int64_t n, int32_t* out);
/* classify_pair: shared-vertex count by index (3 = duplicate face) and the
 * exact coplanarity flag (a degenerate face counts as coplanar); either output may be NULL */
int pamopt_cu_classify_pair(pamopt_cu_mesh mesh, const int32_t* pairs, int64_t n, int32_t* shared, int32_t* coplanar);
/* intersect_3d / intersect_coplanar for pairs of that class:
 * out int32[n] = 1/0; PAMOPT_CU_EINVAL if some pair violates the class precondition (out -1) */
int pamopt_cu_intersect_3d(pamopt_cu_mesh mesh, const int32_t* pairs, int64_t n, int32_t* out);
int pamopt_cu_intersect_coplanar(pamopt_cu_mesh mesh, const int32_t* pairs, int64_t n, int32_t* out);

/* ---- stage 2: simplify ---------------------------------------------------------------- */
/* in place; on success the mesh is compacted (mesh.cpp:278-292).  PAMOPT_CU_EINVAL for a
 * non-manifold input.  per_iter_collapses may be NULL. */
int pamopt_cu_simplify(pamopt_cu_mesh mesh, int64_t target_faces,
                       const pamopt_cu_simplify_params* params, pamopt_cu_simplify_stats* stats,
                       int64_t* per_iter_collapses, int64_t per_iter_cap);

/* ---- stage 2, SPEC-granular operations ------------------------------ */
/* Quadric per vertex, area-weighted unit-plane quadrics gathered in ascending
 * face id: out double[10 nv] = {xx, xy, xz, xw, yy, yz, yw, zz, zw, ww} */
int pamopt_cu_quadrics(pamopt_cu_mesh mesh, double* out);
/* edge_cost of n explicit edges (int32[2n]) under the mesh's quadrics:
 * cost double[n], placement double[3n] (adjugate solve or the {mid, a, b} fallback, P8) */
int pamopt_cu_edge_cost(pamopt_cu_mesh mesh, const int32_t* edges, int64_t n, double w_e, double w_s, double* cost,
                        double* placement);
/* pack_cost: key = f32 bits(max(cost, 0)) << 32 | id; PAMOPT_CU_ENUMERIC if any
 * cost is NaN (the keys of the other entries are still written) */
int pamopt_cu_pack_cost(pamopt_cu_ctx ctx, const double* cost, const uint32_t* edge_ids, int64_t n, uint64_t* keys);
/* HalfEdgeAdjacency::link_condition_holds (mesh.cpp:301-358) for n edges: out int32[n] = 1/0;
 * PAMOPT_CU_EINVAL (std::invalid_argument, mesh.cpp:302) if a pair is not an edge of the mesh,
 * out[i] = -1 for it.  Unbounded valence. */
int pamopt_cu_link_condition(pamopt_cu_mesh mesh, const int32_t* edges, int64_t n, int32_t* out);

/* Algorithm 1 one step at a time on a device mesh (simplified in place; the mesh handle must
 * outlive the state).  Per iteration, in order: prepare (edges + edge_cost + pack_cost),
 * propagate_and_mark, collapse_batch, undo_loop, end_iteration; qem_finish compacts the mesh.
 * pamopt_cu_simplify is exactly this loop.  Calls out of order -> PAMOPT_CU_EINVAL. */
typedef struct pamopt_cu_qem_s* pamopt_cu_qem;
int pamopt_cu_qem_create(pamopt_cu_mesh mesh, int64_t target_faces, const pamopt_cu_simplify_params* params,
                         pamopt_cu_qem* out);
/* 1 when simplify_to's loop would stop: alive faces <= target, or the stall rule */
int pamopt_cu_qem_done(pamopt_cu_qem q, int32_t* done);
int pamopt_cu_qem_prepare(pamopt_cu_qem q, int64_t* n_edges);
/* this iteration's edges (lexicographic ids, P5): int32[2 ne]; keys uint64[ne] (~0 = invalid
 * edge); placements double[3 ne]; valid uint8[ne]; any output may be NULL */
int pamopt_cu_qem_edges(pamopt_cu_qem q, int32_t* edges, uint64_t* keys, double* placements, uint8_t* valid,
                        int64_t cap);
int pamopt_cu_qem_propagate_and_mark(pamopt_cu_qem q, int64_t* n_marked);
/* marked (independent) edges in ascending key order; face_keys = per face slot min key (~0 for
 * a dead face), uint64[nf] with nf from pamopt_cu_qem_mesh; either may be NULL */
int pamopt_cu_qem_marked(pamopt_cu_qem q, uint32_t* edge_ids, int64_t cap, uint64_t* face_keys, int64_t cap_faces);
/* link condition + overshoot trim + parallel collapse; link_ok uint8[n_marked] (key order) */
int pamopt_cu_qem_collapse_batch(pamopt_cu_qem q, uint8_t* link_ok, int64_t cap);
/* detect -> revert -> repeat; applied uint8[n_marked] = collapse still applied (key order) */
int pamopt_cu_qem_undo_loop(pamopt_cu_qem q, int32_t* rounds, int64_t* n_applied, uint8_t* applied, int64_t cap);
int pamopt_cu_qem_end_iteration(pamopt_cu_qem q, int64_t* alive_faces);
/* the working mesh with tombstones (ids stable until compaction): vertices double[3 nv],
 * faces int32[3 nf], face_alive uint8[nf]; NULL outputs = sizes only */
int pamopt_cu_qem_mesh(pamopt_cu_qem q, double* vertices, int32_t* faces, uint8_t* face_alive, int64_t* nv,
                       int64_t* nf);
int pamopt_cu_qem_finish(pamopt_cu_qem q, pamopt_cu_simplify_stats* stats);
int pamopt_cu_qem_destroy(pamopt_cu_qem q);

/* ---- certification and quality metrics ---------------------------- */
/* analyze_topology (mesh.cpp:113-150; TopologySummary mesh.hpp:44-51) */
typedef struct {
  int32_t manifold;
  int32_t watertight;
  int64_t euler_characteristic;
  int64_t boundary_edge_count;
  int64_t n_nonmanifold_edges;
  int64_t n_nonmanifold_vertices;
} pamopt_cu_topology;
/* lists (count-then-fill): nonmanifold_edges = int32[2*cap_edges] (a<b, ascending),
 * nonmanifold_vertices = int32[cap_vertices] (ascending); either may be NULL */
int pamopt_cu_analyze_topology(pamopt_cu_mesh mesh, pamopt_cu_topology* out, int32_t* nonmanifold_edges,
                               int64_t cap_edges, int32_t* nonmanifold_vertices, int64_t cap_vertices);
/* TriangleBvh::nearest_primitive (lbvh.cpp:192-237) for n host points: face (-1 for an empty
 * mesh), distance, closest point (double[3n]); ties go to the lower face id.  Any output may be NULL. */
int pamopt_cu_nearest_primitive(pamopt_cu_mesh mesh, const double* points, int64_t n, int32_t* face,
                                double* distance, double* closest);
/* the pinned area-weighted sampler: points double[3n], faces int32[n] (may be NULL) */
int pamopt_cu_sample_points(pamopt_cu_mesh mesh, int64_t n, uint64_t seed, double* points, int32_t* faces,
                            double* total_area);
/* quality_metrics: squared-distance Chamfer and sampled symmetric Hausdorff with n
 * samples per direction (mesh a uses seed, mesh b seed + 0x632BE59BD9B4E019); EINVAL for a
 * zero-area mesh */
int pamopt_cu_chamfer(pamopt_cu_mesh a, pamopt_cu_mesh b, int64_t n_samples, uint64_t seed, double* out);
int pamopt_cu_hausdorff(pamopt_cu_mesh a, pamopt_cu_mesh b, int64_t n_samples, uint64_t seed, double* out);
/* minimum corner angle in degrees; a zero-area face counts as 0 */
int pamopt_cu_min_internal_angle(pamopt_cu_mesh mesh, double* degrees);
/* MeshReport (SPEC.md quality_metrics): every field in one call; reference may be NULL (cd/hd = NaN) */
typedef struct {
  double cd;
  double hd;
  double min_angle_deg;
  int32_t manifold;
  int32_t watertight;
  int32_t intersection_free;
  int32_t pad_;
  int64_t n_faces;
  int64_t n_vertices;
} pamopt_cu_mesh_report;
int pamopt_cu_report(pamopt_cu_mesh reference, pamopt_cu_mesh mesh, int64_t n_samples, uint64_t seed,
                     pamopt_cu_mesh_report* out);

/* ---- stage 3: safe projection (SPEC.md safe_project; Algorithm 2) --------------- */
typedef struct {
  int32_t iterations;  /* T = 50 */
  int32_t refresh;     /* nearest-target refresh period, 10 */
  int32_t cg_max;      /* 1000 */
  int32_t elas_power;  /* 1 = |F^T F - I|_F as printed (C1-smoothed below elas_tau); 2 = squared */
  int64_t samples;     /* m = 16384 surface samples of the input mesh */
  uint64_t seed;
  double kdis, kelas, kbend, kbar, dhat, cg_tol, elas_tau;
} pamopt_cu_project_params;
typedef struct {
  int64_t iterations, cg_iterations, refreshes, converged;
  double energy0, energy, grad_norm, last_alpha;
} pamopt_cu_project_stats;
int pamopt_cu_project_defaults(pamopt_cu_project_params* out);
/* project(mesh_s, mesh_in): deforms mesh_s's vertices in place toward mesh_in along an
 * intersection-free piecewise-linear trajectory; connectivity unchanged.  EINVAL if mesh_s
 * self-intersects or has a degenerate face. */
int pamopt_cu_safe_project(pamopt_cu_mesh mesh_s, pamopt_cu_mesh mesh_in, const pamopt_cu_project_params* params,
                           pamopt_cu_project_stats* stats);

/* the same solve with a per-iteration record (host buffers; any pointer may be null) so a CPU
 * restatement can replay each Newton step: iterations [0, max_iters) are recorded.  m = samples.
 * X/grad/dir/targets: max_iters x 3nv; m2s: max_iters x m x 4 (face vertices, frozen class);
 * contacts: max_iters x contact_cap x 6 (term 4 PT / 5 EE, class, 4 vertices), n_contacts:
 * max_iters; scalars: max_iters x 8 = {B0, |g|, CG iterations, ACCD t_max, alpha, B(x + alpha p),
 * accepted, line-search tries}; samples: 3m */
typedef struct {
  int32_t max_iters;
  int64_t contact_cap;
  double *X, *grad, *dir, *targets;
  int32_t *m2s, *contacts;
  int64_t* n_contacts;
  double *scalars, *samples;
} pamopt_cu_project_trace;
int pamopt_cu_safe_project_traced(pamopt_cu_mesh mesh_s, pamopt_cu_mesh mesh_in, const pamopt_cu_project_params* params,
                                  pamopt_cu_project_stats* stats, const pamopt_cu_project_trace* trace);

/* one stage-3 energy stencil on the GPU (unit checks of the terms).  term: 0 S2M, 1 M2S,
 * 2 elastic, 3 bending, 4 point-triangle barrier, 5 edge-edge barrier; cls: the frozen distance
 * class (M2S / barrier); coords: nv (1, 3 or 4) vertices; rest[16] = {s0, ytgt[3], ys[3], m2s_w,
 * dminv[4], a0, theta0, l0, -}; out = {value, gradient[12], SPD-projected Hessian[144]} */
int pamopt_cu_project_term(pamopt_cu_ctx ctx, int32_t term, int32_t cls, const double* coords, int32_t nv,
                           const double* rest, const pamopt_cu_project_params* params, double* out);

/* ---- run_pipeline: normalise -> stage 1 -> certify -> stage 2 -> certify ->
 * [stage 3 -> certify] -> denormalise, with a MeshReport per stage ------------------------- */
#define PAMOPT_CU_ECERT -6 /* a stage certification failed (nonzero exit) */
typedef struct {
  int32_t resolution;      /* R; 0 = the SPEC auto rule (256; 128 if target < 1000; 64 if < 50) */
  int32_t run_projection;  /* stage 3 (safe projection) after stage 2 */
  int64_t target_faces;    /* > 0, or 0 to use target_ratio */
  double target_ratio;     /* target = max(4, ratio * input faces) when target_faces == 0 */
  double beta;             /* DMC sigmoid sharpness, 5 */
  double eps;              /* band offset; 0 = 0.9 / R */
  pamopt_cu_simplify_params simplify;
  int64_t report_samples;  /* Chamfer / Hausdorff samples per side, 16384 */
  uint64_t seed;           /* 42 */
} pamopt_cu_pipeline_config;
typedef struct {
  /* per stage, against the (normalised) input: stage[0] DMC, stage[1] QEM, stage[2] projection */
  pamopt_cu_mesh_report stage[3];
  int32_t failed_stage;    /* 0 = every certification passed, else the failing stage (1..3) */
  int32_t stalled;         /* stage 2 stopped by the stall rule above the target */
  int32_t resolution;
  int32_t projected;
  int64_t faces_in, target_faces;
  pamopt_cu_simplify_stats simplify;
  float stage_ms[4];       /* stage 1 (UDF+DMC), stage 2 (QEM), stage 3, certification + reports */
  float total_ms;
  float pad_;
  double scale_translation[4];
} pamopt_cu_pipeline_report;
int pamopt_cu_pipeline_defaults(pamopt_cu_pipeline_config* out);
/* input: the raw mesh (any coordinates; it is copied, not modified).  out: the denormalised
 * output; on a certification failure returns PAMOPT_CU_ECERT with out = the failing stage's
 * mesh (normalised coordinates, the diagnostic dump) and report->failed_stage set. */
int pamopt_cu_run_pipeline(pamopt_cu_ctx ctx, pamopt_cu_mesh input, const pamopt_cu_pipeline_config* config,
                           pamopt_cu_mesh* out, pamopt_cu_pipeline_report* report);

/* ---- pipeline: UDF -> SDF -> DMC -> QEM ------------------------------------------------ */
int pamopt_cu_remesh(pamopt_cu_ctx ctx, pamopt_cu_mesh input, int32_t R, double eps, double beta,
                     int64_t target_faces, const pamopt_cu_simplify_params* params,
                     pamopt_cu_mesh* out, pamopt_cu_simplify_stats* stats,
                     pamopt_cu_stage_times* times);
/* same, host buffers in and out (the end-to-end entry the reference's caller would bind);
 * out_vertices/out_faces must hold the returned sizes: call with NULL outputs first is NOT
 * supported — the result is retained in the context until the next call and fetched with
 * pamopt_cu_remesh_fetch. */
int pamopt_cu_remesh_host(pamopt_cu_ctx ctx, const double* vertices, int64_t nv,
                          const int32_t* faces, int64_t nf, int32_t R, double eps, double beta,
                          int64_t target_faces, const pamopt_cu_simplify_params* params,
                          int64_t* out_nv, int64_t* out_nf, pamopt_cu_simplify_stats* stats,
                          pamopt_cu_stage_times* times);
int pamopt_cu_remesh_fetch(pamopt_cu_ctx ctx, double* vertices, int32_t* faces);

#ifdef __cplusplus
}
#endif

#endif /* PAMOPT_CU_H_ */
