// pamopt/pipeline.hpp — the reference's missing run_pipeline (proj/CMakeLists.txt:28
// `src/pipeline.cpp`) on the GPU, device resident between stages:
//   remesh()        stages 1-2 (UDF -> SDF -> DMC -> QEM) of a normalised mesh, the hot path;
//   run_pipeline()  normalise -> stage 1 -> certify -> stage 2 -> certify -> [stage 3 (safe
//                   projection) -> certify] -> denormalise, with a MeshReport per stage.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "pamopt/cuda_detail.hpp"
#include "pamopt/simplify.hpp"

namespace pamopt {

struct StageTimings {
  float udf_ms = 0, dmc_ms = 0, simplify_ms = 0, total_ms = 0;
  int64_t dmc_faces = 0, dmc_vertices = 0;
};

/// The mesh must already be normalised with normalize_unit_cube(mesh, 6.0 / R)
/// (mesh_io.hpp:42, padding rule SPEC.md:141).  eps <= 0 selects the default 0.9 / R.
inline IndexedMesh remesh(const IndexedMesh& normalized, int R, int64_t target_faces, const SimplifyParams& p = {},
                          double eps = 0.0, double beta = 5.0, SimplifyStats* stats = nullptr,
                          StageTimings* timings = nullptr) {
  cuda::Context& ctx = cuda::Context::thread_default();
  std::vector<double> v(3 * normalized.vertices.size());
  std::vector<int32_t> f(3 * normalized.faces.size());
  for (size_t i = 0; i < normalized.vertices.size(); ++i)
    for (int k = 0; k < 3; ++k) v[3 * i + k] = normalized.vertices[i][k];
  for (size_t i = 0; i < normalized.faces.size(); ++i)
    for (int k = 0; k < 3; ++k) f[3 * i + k] = normalized.faces[i][k];
  const pamopt_cu_simplify_params cp{p.w_e, p.w_s, p.tolerance, p.stall_iterations};
  pamopt_cu_simplify_stats st{};
  pamopt_cu_stage_times tm{};
  int64_t nv = 0, nf = 0;
  cuda::check(pamopt_cu_remesh_host(ctx.get(), v.data(), static_cast<int64_t>(normalized.vertices.size()), f.data(),
                                    static_cast<int64_t>(normalized.faces.size()), R, eps > 0 ? eps : 0.9 / R, beta,
                                    target_faces, &cp, &nv, &nf, &st, &tm));
  std::vector<double> ov(3 * nv);
  std::vector<int32_t> of(3 * nf);
  cuda::check(pamopt_cu_remesh_fetch(ctx.get(), ov.data(), of.data()));
  IndexedMesh out;
  out.vertices.resize(nv);
  out.faces.resize(nf);
  for (int64_t i = 0; i < nv; ++i) out.vertices[i] = Vec3d(ov[3 * i], ov[3 * i + 1], ov[3 * i + 2]);
  for (int64_t i = 0; i < nf; ++i) out.faces[i] = Vec3i(of[3 * i], of[3 * i + 1], of[3 * i + 2]);
  if (stats) {
    stats->iterations = st.iterations;
    stats->collapses = st.collapses;
    stats->undone = st.undone;
    stats->link_failures = st.link_failures;
    stats->max_undo_rounds = st.max_undo_rounds;
    for (int k = 0; k < 8; ++k) stats->undo_hist[k] = st.undo_hist[k];
  }
  if (timings) *timings = StageTimings{tm.udf_ms, tm.dmc_ms, tm.simplify_ms, tm.total_ms, tm.dmc_faces, tm.dmc_vertices};
  return out;
}

/// PipelineConfig.  resolution 0 = the SPEC auto rule.
struct PipelineConfig {
  int resolution = 0;
  int64_t target_faces = 0;   // 0: use target_ratio
  double target_ratio = 0.01;
  bool run_projection = false;
  double beta = 5.0, eps = 0.0;
  SimplifyParams simplify{};
  int64_t report_samples = 16384;
  uint64_t seed = 42;
};

/// MeshReport per stage (SPEC.md quality_metrics; CD/HD against the normalised input).
struct StageReport {
  double cd = 0, hd = 0, min_angle_deg = 0;
  bool manifold = false, watertight = false, intersection_free = false;
  int64_t faces = 0, vertices = 0;
};

struct PipelineResult {
  IndexedMesh mesh;                 // denormalised to the input's coordinates
  std::vector<StageReport> stages;  // stage 1, 2 (and 3 with projection)
  bool stalled = false;
  int resolution = 0;
  int64_t target_faces = 0;
  SimplifyStats simplify;
  float stage_ms[4] = {0, 0, 0, 0};  // stage 1, 2, 3, certification
  float total_ms = 0;
};

/// Thrown when a stage certification fails ("nonzero exit with stage name and
/// diagnostic dump"); dump() is that stage's mesh in normalised coordinates.
class CertificationError : public std::runtime_error {
 public:
  CertificationError(const std::string& m, int stage, IndexedMesh dump)
      : std::runtime_error(m), stage_(stage), dump_(std::move(dump)) {}
  int stage() const { return stage_; }
  const IndexedMesh& dump() const { return dump_; }

 private:
  int stage_;
  IndexedMesh dump_;
};

/// run_pipeline on an in-memory raw mesh (load_mesh, mesh_io.hpp:23, is the
/// caller's): normalise, stage 1, certify, stage 2, certify, [stage 3, certify], denormalise.
inline PipelineResult run_pipeline(const IndexedMesh& input, const PipelineConfig& c = {}) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, input);
  pamopt_cu_pipeline_config cfg{};
  cuda::check(pamopt_cu_pipeline_defaults(&cfg));
  cfg.resolution = c.resolution;
  cfg.run_projection = c.run_projection ? 1 : 0;
  cfg.target_faces = c.target_faces;
  cfg.target_ratio = c.target_ratio;
  cfg.beta = c.beta;
  cfg.eps = c.eps;
  cfg.simplify = pamopt_cu_simplify_params{c.simplify.w_e, c.simplify.w_s, c.simplify.tolerance,
                                           c.simplify.stall_iterations};
  cfg.report_samples = c.report_samples;
  cfg.seed = c.seed;
  pamopt_cu_mesh out = nullptr;
  pamopt_cu_pipeline_report rep{};
  const int rc = pamopt_cu_run_pipeline(ctx.get(), dm.get(), &cfg, &out, &rep);
  if (rc == PAMOPT_CU_ECERT) {
    const std::string msg = pamopt_cu_last_error();
    throw CertificationError(msg, rep.failed_stage, cuda::DeviceMesh(out).download());
  }
  cuda::check(rc);
  PipelineResult r;
  r.mesh = cuda::DeviceMesh(out).download();
  for (int s = 0; s < (rep.projected ? 3 : 2); ++s) {
    const pamopt_cu_mesh_report& m = rep.stage[s];
    r.stages.push_back(StageReport{m.cd, m.hd, m.min_angle_deg, m.manifold != 0, m.watertight != 0,
                                   m.intersection_free != 0, m.n_faces, m.n_vertices});
  }
  r.stalled = rep.stalled != 0;
  r.resolution = rep.resolution;
  r.target_faces = rep.target_faces;
  r.simplify.iterations = rep.simplify.iterations;
  r.simplify.collapses = rep.simplify.collapses;
  r.simplify.undone = rep.simplify.undone;
  r.simplify.link_failures = rep.simplify.link_failures;
  r.simplify.max_undo_rounds = rep.simplify.max_undo_rounds;
  for (int k = 0; k < 8; ++k) r.simplify.undo_hist[k] = rep.simplify.undo_hist[k];
  for (int k = 0; k < 4; ++k) r.stage_ms[k] = rep.stage_ms[k];
  r.total_ms = rep.total_ms;
  return r;
}

}  // namespace pamopt
