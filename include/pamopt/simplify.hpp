// pamopt/simplify.hpp — drop-in for the reference's missing simplify module
// (proj/CMakeLists.txt:24): parallel QEM with cost propagation, link
// condition (mesh.cpp:301-358 semantics), collapse/undo and the self-intersection undo loop.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <vector>

#include "pamopt/cuda_detail.hpp"

namespace pamopt {

/// SPEC.md:566 parameters (PAPER.md:145,238 defaults).
struct SimplifyParams {
  double w_e = 1e-3;
  double w_s = 5e-3;
  int tolerance = 4;
  int stall_iterations = 10;
};

struct SimplifyStats {
  int64_t iterations = 0, collapses = 0, undone = 0, link_failures = 0, max_undo_rounds = 0;
  int64_t undo_hist[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

/// (f32 bits of max(cost,0)) << 32 | edge id; NaN -> std::domain_error.
inline uint64_t pack_cost(double cost, uint32_t edge_id) {
  if (cost != cost) throw std::domain_error("pack_cost: NaN cost");
  const float f = static_cast<float>(cost < 0.0 ? 0.0 : cost);
  uint32_t bits;
  std::memcpy(&bits, &f, 4);
  return (static_cast<uint64_t>(bits) << 32) | edge_id;
}

/// Quadric per vertex: {xx, xy, xz, xw, yy, yz, yw, zz, zw, ww}.
inline std::vector<std::array<double, 10>> compute_quadrics(const IndexedMesh& mesh) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  std::vector<std::array<double, 10>> q(mesh.vertices.size());
  cuda::check(pamopt_cu_quadrics(dm.get(), q.empty() ? nullptr : q[0].data()));
  return q;
}

struct EdgeCost {
  double cost = 0.0;
  Vec3d placement = Vec3d::Zero();
};

/// edge_cost of explicit edges under the mesh's quadrics (Eq. 1).
inline std::vector<EdgeCost> edge_cost(const IndexedMesh& mesh, const std::vector<EdgeKey>& edges,
                                       const SimplifyParams& p = {}) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  std::vector<int32_t> e(2 * edges.size());
  for (size_t i = 0; i < edges.size(); ++i) {
    e[2 * i] = edges[i].a;
    e[2 * i + 1] = edges[i].b;
  }
  std::vector<double> c(edges.size()), x(3 * edges.size());
  cuda::check(pamopt_cu_edge_cost(dm.get(), e.data(), static_cast<int64_t>(edges.size()), p.w_e, p.w_s, c.data(),
                                  x.data()));
  std::vector<EdgeCost> out(edges.size());
  for (size_t i = 0; i < edges.size(); ++i) out[i] = EdgeCost{c[i], Vec3d(x[3 * i], x[3 * i + 1], x[3 * i + 2])};
  return out;
}

/// HalfEdgeAdjacency::link_condition_holds (mesh.cpp:301-358) for many edges at once;
/// std::invalid_argument for a pair that is not an edge (mesh.cpp:302).
inline std::vector<bool> link_condition_holds(const IndexedMesh& mesh, const std::vector<EdgeKey>& edges) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  std::vector<int32_t> e(2 * edges.size()), r(edges.size());
  for (size_t i = 0; i < edges.size(); ++i) {
    e[2 * i] = edges[i].a;
    e[2 * i + 1] = edges[i].b;
  }
  cuda::check(pamopt_cu_link_condition(dm.get(), e.data(), static_cast<int64_t>(edges.size()), r.data()));
  return std::vector<bool>(r.begin(), r.end());
}

/// Algorithm 1 one SPEC operation at a time (the code simplify_to runs): per iteration
/// prepare() (edges + edge_cost + pack_cost), propagate_and_mark(), collapse_batch(),
/// undo_loop(), end_iteration(); finish() compacts and returns the mesh.
class SimplifySession {
 public:
  SimplifySession(const IndexedMesh& mesh, int64_t target_faces, const SimplifyParams& p = {})
      : dm_(cuda::Context::thread_default(), mesh) {
    const pamopt_cu_simplify_params cp{p.w_e, p.w_s, p.tolerance, p.stall_iterations};
    cuda::check(pamopt_cu_qem_create(dm_.get(), target_faces, &cp, &q_));
  }
  ~SimplifySession() { pamopt_cu_qem_destroy(q_); }
  SimplifySession(const SimplifySession&) = delete;
  SimplifySession& operator=(const SimplifySession&) = delete;
  bool done() const {
    int32_t d = 0;
    cuda::check(pamopt_cu_qem_done(q_, &d));
    return d != 0;
  }
  /// edge ids = lexicographic ranks (P5); keys[i] = pack_cost(cost, i) or ~0 for an invalid edge
  std::vector<uint64_t> prepare(std::vector<EdgeKey>* edges = nullptr) {
    int64_t ne = 0;
    cuda::check(pamopt_cu_qem_prepare(q_, &ne));
    std::vector<int32_t> e(2 * ne);
    std::vector<uint64_t> keys(ne);
    cuda::check(pamopt_cu_qem_edges(q_, e.data(), keys.data(), nullptr, nullptr, ne));
    if (edges) {
      edges->clear();
      for (int64_t i = 0; i < ne; ++i) edges->push_back(EdgeKey(e[2 * i], e[2 * i + 1]));
    }
    return keys;
  }
  /// independent edge ids in ascending key order
  std::vector<uint32_t> propagate_and_mark() {
    int64_t nm = 0;
    cuda::check(pamopt_cu_qem_propagate_and_mark(q_, &nm));
    marked_.resize(nm);
    cuda::check(pamopt_cu_qem_marked(q_, marked_.data(), nm, nullptr, 0));
    return marked_;
  }
  /// per marked edge: link condition held
  std::vector<bool> collapse_batch() {
    std::vector<uint8_t> ok(marked_.size());
    cuda::check(pamopt_cu_qem_collapse_batch(q_, ok.data(), static_cast<int64_t>(ok.size())));
    return std::vector<bool>(ok.begin(), ok.end());
  }
  /// undo rounds of this batch; applied[i] = marked edge i is still collapsed
  int undo_loop(std::vector<bool>* applied = nullptr) {
    int32_t rounds = 0;
    int64_t n = 0;
    std::vector<uint8_t> a(marked_.size());
    cuda::check(pamopt_cu_qem_undo_loop(q_, &rounds, &n, a.data(), static_cast<int64_t>(a.size())));
    if (applied) *applied = std::vector<bool>(a.begin(), a.end());
    return rounds;
  }
  int64_t end_iteration() {
    int64_t alive = 0;
    cuda::check(pamopt_cu_qem_end_iteration(q_, &alive));
    return alive;
  }
  IndexedMesh finish(SimplifyStats* stats = nullptr) {
    pamopt_cu_simplify_stats st{};
    cuda::check(pamopt_cu_qem_finish(q_, &st));
    if (stats) {
      stats->iterations = st.iterations;
      stats->collapses = st.collapses;
      stats->undone = st.undone;
      stats->link_failures = st.link_failures;
      stats->max_undo_rounds = st.max_undo_rounds;
      for (int k = 0; k < 8; ++k) stats->undo_hist[k] = st.undo_hist[k];
    }
    return dm_.download();
  }

 private:
  cuda::DeviceMesh dm_;
  pamopt_cu_qem q_ = nullptr;
  std::vector<uint32_t> marked_;
};

/// SPEC.md:539-547.  Returns the compacted simplified mesh; std::invalid_argument for a
/// non-manifold input.
inline IndexedMesh simplify_to(const IndexedMesh& mesh, int64_t target_faces, const SimplifyParams& p = {},
                               SimplifyStats* stats = nullptr) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  const pamopt_cu_simplify_params cp{p.w_e, p.w_s, p.tolerance, p.stall_iterations};
  pamopt_cu_simplify_stats st{};
  cuda::check(pamopt_cu_simplify(dm.get(), target_faces, &cp, &st, nullptr, 0));
  if (stats) {
    stats->iterations = st.iterations;
    stats->collapses = st.collapses;
    stats->undone = st.undone;
    stats->link_failures = st.link_failures;
    stats->max_undo_rounds = st.max_undo_rounds;
    for (int k = 0; k < 8; ++k) stats->undo_hist[k] = st.undo_hist[k];
  }
  return dm.download();
}

}  // namespace pamopt
