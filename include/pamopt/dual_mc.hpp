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

/// interpolate_patch_vertex: v0 + t'(v1 - v0), t = -f0/(f1 - f0),
/// t' = 1/(1 + exp(-beta (t - 1/2))); std::invalid_argument when f0, f1 share a sign.
inline Vec3d interpolate_patch_vertex(const Vec3d& v0, const Vec3d& v1, float f0, float f1, double beta = 5.0) {
  cuda::Context& ctx = cuda::Context::thread_default();
  const double p0[3] = {v0[0], v0[1], v0[2]}, p1[3] = {v1[0], v1[1], v1[2]};
  double o[3];
  cuda::check(pamopt_cu_interpolate_patch_vertex(ctx.get(), p0, p1, &f0, &f1, 1, beta, o));
  return Vec3d(o[0], o[1], o[2]);
}

/// build_patches + build_quads views and triangulate_quads.
struct PatchSoup {
  std::vector<Vec3d> vertices;       // (active cell, patch) order
  std::vector<int64_t> patch_first;  // first patch vertex of each active cell
};
struct QuadMesh {
  std::vector<std::array<int32_t, 4>> quads;  // patch-vertex ids, oriented negative -> positive
  std::vector<int64_t> edges;                 // valid grid edge: lower lattice vertex * 3 + axis
  std::vector<std::array<float, 2>> samples;  // SDF at the edge's lower / upper vertex
  std::vector<uint8_t> split;                 // 1: diagonal 0-2, 2: diagonal 1-3, 3: four triangles
};

inline void dmc_stages(const ScalarGrid& grid, PatchSoup& patches, QuadMesh& quads, double beta = 5.0) {
  cuda::Context& ctx = cuda::Context::thread_default();
  pamopt_cu_grid g = nullptr;
  cuda::check(pamopt_cu_grid_upload(ctx.get(), grid.resolution, grid.samples.data(), &g));
  int64_t c[3] = {0, 0, 0};
  int rc = pamopt_cu_dmc_stages(g, beta, c);
  if (rc == PAMOPT_CU_OK) {
    std::vector<double> v(3 * c[1]);
    patches.patch_first.resize(c[0]);
    rc = pamopt_cu_dmc_build_patches(g, v.data(), patches.patch_first.data());
    patches.vertices.resize(c[1]);
    for (int64_t i = 0; i < c[1]; ++i) patches.vertices[i] = Vec3d(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  }
  if (rc == PAMOPT_CU_OK) {
    quads.quads.resize(c[2]);
    quads.edges.resize(c[2]);
    quads.samples.resize(c[2]);
    quads.split.resize(c[2]);
    rc = pamopt_cu_dmc_build_quads(g, c[2] ? quads.quads[0].data() : nullptr, quads.edges.data(),
                                   c[2] ? quads.samples[0].data() : nullptr, quads.split.data());
  }
  pamopt_cu_grid_free(g);
  cuda::check(rc);
}

inline IndexedMesh triangulate_quads(int R, const PatchSoup& patches, const QuadMesh& q, double beta = 5.0) {
  cuda::Context& ctx = cuda::Context::thread_default();
  std::vector<double> v(3 * patches.vertices.size());
  for (size_t i = 0; i < patches.vertices.size(); ++i)
    for (int k = 0; k < 3; ++k) v[3 * i + k] = patches.vertices[i][k];
  pamopt_cu_mesh m = nullptr;
  cuda::check(pamopt_cu_triangulate_quads(ctx.get(), R, v.data(), static_cast<int64_t>(patches.vertices.size()),
                                          q.quads.empty() ? nullptr : q.quads[0].data(), q.edges.data(),
                                          q.samples.empty() ? nullptr : q.samples[0].data(),
                                          static_cast<int64_t>(q.quads.size()), beta, &m));
  return cuda::DeviceMesh(m).download();
}

}  // namespace pamopt
