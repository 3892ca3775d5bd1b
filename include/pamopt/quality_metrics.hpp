// pamopt/quality_metrics.hpp — drop-in for the reference's missing quality_metrics module
// (SPEC.md quality_metrics: chamfer, hausdorff, min_internal_angle, MeshReport) and GPU
// twins of the certification calls the reference runs on the CPU:
//   pamopt::cuda::analyze_topology   == pamopt::analyze_topology        (mesh.cpp:113-150)
//   pamopt::cuda::nearest_primitives == TriangleBvh::nearest_primitive  (lbvh.cpp:192-237), batched
// Both return the reference's own types and equal its results bit for bit
// (tests/test_gpu_metrics.py against golden vectors from the reference).
#pragma once

#include <cstdint>
#include <vector>

#include "pamopt/cuda_detail.hpp"
#include "pamopt/lbvh.hpp"

namespace pamopt {

/// SPEC quality_metrics MeshReport.
struct MeshReport {
  double cd = 0, hd = 0, min_angle_deg = 0;
  bool manifold = false, watertight = false, intersection_free = false;
  int64_t face_count = 0, vertex_count = 0;
};

namespace cuda {

inline TopologySummary analyze_topology(const IndexedMesh& mesh) {
  Context& ctx = Context::thread_default();
  DeviceMesh dm(ctx, mesh);
  pamopt_cu_topology t{};
  check(pamopt_cu_analyze_topology(dm.get(), &t, nullptr, 0, nullptr, 0));
  std::vector<int32_t> e(2 * t.n_nonmanifold_edges), v(t.n_nonmanifold_vertices);
  check(pamopt_cu_analyze_topology(dm.get(), &t, e.data(), t.n_nonmanifold_edges, v.data(),
                                   t.n_nonmanifold_vertices));
  TopologySummary s;
  s.manifold = t.manifold != 0;
  s.watertight = t.watertight != 0;
  s.euler_characteristic = static_cast<int>(t.euler_characteristic);
  s.boundary_edge_count = static_cast<int>(t.boundary_edge_count);
  for (int64_t i = 0; i < t.n_nonmanifold_edges; ++i) s.nonmanifold_edges.emplace_back(e[2 * i], e[2 * i + 1]);
  s.nonmanifold_vertices.assign(v.begin(), v.end());
  return s;
}

inline std::vector<NearestHit> nearest_primitives(const IndexedMesh& mesh, const std::vector<Vec3d>& points) {
  Context& ctx = Context::thread_default();
  DeviceMesh dm(ctx, mesh);
  const int64_t n = static_cast<int64_t>(points.size());
  std::vector<double> p(3 * n), dist(n), clo(3 * n);
  std::vector<int32_t> face(n);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) p[3 * i + k] = points[i][k];
  check(pamopt_cu_nearest_primitive(dm.get(), p.data(), n, face.data(), dist.data(), clo.data()));
  std::vector<NearestHit> out(n);
  for (int64_t i = 0; i < n; ++i) {
    out[i].primitive = face[i];
    out[i].distance = dist[i];
    out[i].point = Vec3d(clo[3 * i], clo[3 * i + 1], clo[3 * i + 2]);
  }
  return out;
}

}  // namespace cuda

inline double chamfer(const IndexedMesh& a, const IndexedMesh& b, int64_t n_samples = 16384, uint64_t seed = 42) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh da(ctx, a), db(ctx, b);
  double out = 0;
  cuda::check(pamopt_cu_chamfer(da.get(), db.get(), n_samples, seed, &out));
  return out;
}

inline double hausdorff(const IndexedMesh& a, const IndexedMesh& b, int64_t n_samples = 16384, uint64_t seed = 42) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh da(ctx, a), db(ctx, b);
  double out = 0;
  cuda::check(pamopt_cu_hausdorff(da.get(), db.get(), n_samples, seed, &out));
  return out;
}

inline double min_internal_angle(const IndexedMesh& mesh) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  double out = 0;
  cuda::check(pamopt_cu_min_internal_angle(dm.get(), &out));
  return out;
}

/// cd/hd against `reference` (pass nullptr to skip them: NaN), plus the certification flags.
inline MeshReport mesh_report(const IndexedMesh& mesh, const IndexedMesh* reference = nullptr,
                              int64_t n_samples = 16384, uint64_t seed = 42) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  cuda::DeviceMesh dr;
  if (reference) dr = cuda::DeviceMesh(ctx, *reference);
  pamopt_cu_mesh_report r{};
  cuda::check(pamopt_cu_report(reference ? dr.get() : nullptr, dm.get(), n_samples, seed, &r));
  MeshReport o;
  o.cd = r.cd;
  o.hd = r.hd;
  o.min_angle_deg = r.min_angle_deg;
  o.manifold = r.manifold != 0;
  o.watertight = r.watertight != 0;
  o.intersection_free = r.intersection_free != 0;
  o.face_count = r.n_faces;
  o.vertex_count = r.n_vertices;
  return o;
}

}  // namespace pamopt
