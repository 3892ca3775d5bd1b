// pamopt/pipeline.hpp — stages 1-2 of the reference's missing run_pipeline
// (proj/CMakeLists.txt:28 `src/pipeline.cpp`): UDF -> SDF -> DMC -> QEM on the
// GPU in one call, device resident between stages.  Stage 3 (safe projection) is out of scope.
#pragma once

#include <cstdint>
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

}  // namespace pamopt
