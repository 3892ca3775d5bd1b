// pamopt/dual_mc.hpp — drop-in for the reference's missing dual_mc / dual_mc_table modules
// (proj/CMakeLists.txt:20-21).  The patch table, active-cell classification,
// patches, quads and the envelope quad division run on the GPU (include/pamopt_cu.h).
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "pamopt/cuda_detail.hpp"
#include "pamopt/voxel_field.hpp"

namespace pamopt {

/// per case, the patches as 12-bit edge masks; doubly-covered faces
/// (the ambiguous faces the C16/C19 rule may flip).
struct DmcTable {
  struct Entry {
    int patches = 0;
    std::array<uint16_t, 4> mask{};
    uint8_t doubly_covered = 0;
  };
  std::array<Entry, 256> entries;
  static DmcTable generate() {
    std::vector<int32_t> t(256 * 6);
    cuda::check(pamopt_cu_dmc_table(t.data()));
    DmcTable d;
    for (int c = 0; c < 256; ++c) {
      d.entries[c].patches = t[6 * c];
      for (int k = 0; k < 4; ++k) d.entries[c].mask[k] = static_cast<uint16_t>(t[6 * c + 1 + k]);
      d.entries[c].doubly_covered = static_cast<uint8_t>(t[6 * c + 5]);
    }
    return d;
  }
};

/// watertight, manifold, self-intersection-free triangle mesh of an SDF grid.
inline IndexedMesh extract(const ScalarGrid& grid, double beta = 5.0) {
  cuda::Context& ctx = cuda::Context::thread_default();
  pamopt_cu_grid g = nullptr;
  cuda::check(pamopt_cu_grid_upload(ctx.get(), grid.resolution, grid.samples.data(), &g));
  pamopt_cu_mesh m = nullptr;
  const int rc = pamopt_cu_dmc_extract(g, beta, &m);
  pamopt_cu_grid_free(g);
  cuda::check(rc);
  return cuda::DeviceMesh(m).download();
}

/// active cells (linear index, 8-bit case) in x-fastest order.
inline std::vector<std::pair<int64_t, uint8_t>> classify_voxels(const ScalarGrid& grid) {
  cuda::Context& ctx = cuda::Context::thread_default();
  pamopt_cu_grid g = nullptr;
  cuda::check(pamopt_cu_grid_upload(ctx.get(), grid.resolution, grid.samples.data(), &g));
  pamopt_cu_mesh m = nullptr;
  int rc = pamopt_cu_dmc_extract(g, 5.0, &m);
  pamopt_cu_mesh_free(m);
  std::vector<std::pair<int64_t, uint8_t>> out;
  if (rc == PAMOPT_CU_OK) {
    int64_t n = 0;
    rc = pamopt_cu_dmc_active_cells(g, nullptr, nullptr, nullptr, 0, &n);
    std::vector<int64_t> cells(n);
    std::vector<uint8_t> cases(n);
    if (rc == PAMOPT_CU_OK) rc = pamopt_cu_dmc_active_cells(g, cells.data(), cases.data(), nullptr, n, &n);
    for (int64_t i = 0; i < n; ++i) out.emplace_back(cells[i], cases[i]);
  }
  pamopt_cu_grid_free(g);
  cuda::check(rc);
  return out;
}

}  // namespace pamopt
