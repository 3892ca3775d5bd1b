// pamopt/safe_project.hpp — drop-in for the reference's missing stage-3 module (SPEC.md
// safe_project; Algorithm 2): project(mesh_s, mesh_in, params) deforms mesh_s toward
// mesh_in along an intersection-free piecewise-linear trajectory, on the GPU.
#pragma once

#include "pamopt/cuda_detail.hpp"

namespace pamopt {

/// SPEC ProjectionState weights and iteration controls (defaults: T=50, refresh 10, m=16384,
/// k_dis=1e3, k_elas=1e-1, k_bend=1e-2, k_bar=1e2, d̂=1e-3).
inline pamopt_cu_project_params default_projection_params() {
  pamopt_cu_project_params p{};
  cuda::check(pamopt_cu_project_defaults(&p));
  return p;
}

/// SPEC [OP] project: returns the deformed mesh (same connectivity as mesh_s).
inline IndexedMesh project(const IndexedMesh& mesh_s, const IndexedMesh& mesh_in,
                           const pamopt_cu_project_params& params = default_projection_params(),
                           pamopt_cu_project_stats* stats = nullptr) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh s(ctx, mesh_s), in(ctx, mesh_in);
  pamopt_cu_project_stats st{};
  cuda::check(pamopt_cu_safe_project(s.get(), in.get(), &params, &st));
  if (stats) *stats = st;
  return s.download();
}

}  // namespace pamopt
