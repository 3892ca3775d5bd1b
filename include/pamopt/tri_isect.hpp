// pamopt/tri_isect.hpp — drop-in for the reference's missing tri_isect module
// (proj/CMakeLists.txt:23).  Detection = grid broad phase (superset of the
// reference LBVH's inflated-AABB pairs, lbvh.cpp:182-190) + exact narrow phase, on the GPU.
#pragma once

#include <utility>
#include <vector>

#include "pamopt/cuda_detail.hpp"

namespace pamopt {

/// all unordered intersecting face pairs (f1 < f2), sorted.
inline std::vector<std::pair<int, int>> detect_self_intersections(const IndexedMesh& mesh) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  int64_t n = 0;
  cuda::check(pamopt_cu_self_intersections(dm.get(), nullptr, 0, &n));
  std::vector<int32_t> buf(2 * n);
  cuda::check(pamopt_cu_self_intersections(dm.get(), buf.data(), n, &n));
  std::vector<std::pair<int, int>> out(n);
  for (int64_t i = 0; i < n; ++i) out[i] = {buf[2 * i], buf[2 * i + 1]};
  return out;
}

/// classify_pair + intersect_3d / intersect_coplanar for explicit pairs.
inline std::vector<bool> faces_intersect(const IndexedMesh& mesh, const std::vector<std::pair<int, int>>& pairs) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  std::vector<int32_t> p(2 * pairs.size());
  for (size_t i = 0; i < pairs.size(); ++i) {
    p[2 * i] = pairs[i].first;
    p[2 * i + 1] = pairs[i].second;
  }
  std::vector<int32_t> r(pairs.size());
  cuda::check(pamopt_cu_tri_tri_pairs(dm.get(), p.data(), static_cast<int64_t>(pairs.size()), r.data()));
  return std::vector<bool>(r.begin(), r.end());
}

/// SPEC.md:404-418 PairClass.
struct PairClass {
  int shared_vertex_count = 0;
  bool coplanar = false;
};

namespace detail {
inline std::vector<int32_t> flat_pairs(const std::vector<std::pair<int, int>>& pairs) {
  std::vector<int32_t> p(2 * pairs.size());
  for (size_t i = 0; i < pairs.size(); ++i) {
    p[2 * i] = pairs[i].first;
    p[2 * i + 1] = pairs[i].second;
  }
  return p;
}
}  // namespace detail

/// classify_pair for face pairs of a mesh.
inline std::vector<PairClass> classify_pair(const IndexedMesh& mesh, const std::vector<std::pair<int, int>>& pairs) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  const std::vector<int32_t> p = detail::flat_pairs(pairs);
  std::vector<int32_t> s(pairs.size()), c(pairs.size());
  cuda::check(pamopt_cu_classify_pair(dm.get(), p.data(), static_cast<int64_t>(pairs.size()), s.data(), c.data()));
  std::vector<PairClass> out(pairs.size());
  for (size_t i = 0; i < pairs.size(); ++i) out[i] = PairClass{s[i], c[i] != 0};
  return out;
}

/// intersect_3d / intersect_coplanar; std::invalid_argument
/// when a pair does not satisfy the class precondition.
inline std::vector<bool> intersect_3d(const IndexedMesh& mesh, const std::vector<std::pair<int, int>>& pairs) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  const std::vector<int32_t> p = detail::flat_pairs(pairs);
  std::vector<int32_t> r(pairs.size());
  cuda::check(pamopt_cu_intersect_3d(dm.get(), p.data(), static_cast<int64_t>(pairs.size()), r.data()));
  return std::vector<bool>(r.begin(), r.end());
}
inline std::vector<bool> intersect_coplanar(const IndexedMesh& mesh, const std::vector<std::pair<int, int>>& pairs) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  const std::vector<int32_t> p = detail::flat_pairs(pairs);
  std::vector<int32_t> r(pairs.size());
  cuda::check(pamopt_cu_intersect_coplanar(dm.get(), p.data(), static_cast<int64_t>(pairs.size()), r.data()));
  return std::vector<bool>(r.begin(), r.end());
}

}  // namespace pamopt
