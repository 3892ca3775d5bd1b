// pamopt/simplify.hpp — drop-in for the reference's missing simplify module
// (proj/CMakeLists.txt:24): parallel QEM with cost propagation, link
// condition (mesh.cpp:301-358 semantics), collapse/undo and the self-intersection undo loop.
#pragma once

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
