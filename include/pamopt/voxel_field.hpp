// pamopt/voxel_field.hpp — drop-in for the reference's missing voxel_field module
// (proj/CMakeLists.txt:19 `src/voxel_field.cpp`).  Same OP names and meaning;
// the computation runs on the GPU through the C-ABI (include/pamopt_cu.h).
#pragma once

#include <cmath>
#include <cstdint>
#include <utility>
#include <vector>

#include "pamopt/cuda_detail.hpp"

namespace pamopt {

/// (R+1)^3 lattice samples, x-fastest, +INF sentinel (UDF) / +1.0 (SDF).
struct ScalarGrid {
  int resolution = 0;           // R_DMC (cells per axis)
  float band = 0.f;             // 3 / R
  float epsilon = NAN;          // set by udf_to_sdf
  std::vector<float> samples;   // (R+1)^3
  float at(int x, int y, int z) const {
    const int64_t n = resolution + 1;
    return samples[x + n * (y + n * static_cast<int64_t>(z))];
  }
};

/// per level (resolution, surviving (cell, triangle) pairs sorted).
struct VoxelHierarchy {
  struct Level {
    int resolution = 0;
    std::vector<std::pair<int64_t, int>> pairs;  // (linear cell index at this level, triangle id)
  };
  int resolution = 0;
  std::vector<Level> levels;  // coarsest (8) -> finest (R)
};

/// SPEC.md:176-184.  batch_size is accepted for interface parity: the device path streams all
/// triangles at once (the result is batch-invariant by definition).
inline VoxelHierarchy build_hierarchy(const IndexedMesh& mesh, int R, int batch_size = 1 << 20) {
  (void)batch_size;
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  VoxelHierarchy h;
  h.resolution = R;
  for (int r = 8; r <= R; r *= 2) {
    int64_t n = 0;
    cuda::check(pamopt_cu_hierarchy_pairs(ctx.get(), dm.get(), R, r, nullptr, 0, &n));
    std::vector<int64_t> buf(2 * n);
    cuda::check(pamopt_cu_hierarchy_pairs(ctx.get(), dm.get(), R, r, buf.data(), n, &n));
    VoxelHierarchy::Level L;
    L.resolution = r;
    L.pairs.resize(n);
    for (int64_t i = 0; i < n; ++i) L.pairs[i] = {buf[2 * i], static_cast<int>(buf[2 * i + 1])};
    h.levels.push_back(std::move(L));
  }
  return h;
}

/// SPEC.md:194-202 (fused with build_hierarchy on the device).
inline ScalarGrid compute_udf(const IndexedMesh& mesh, int R) {
  cuda::Context& ctx = cuda::Context::thread_default();
  cuda::DeviceMesh dm(ctx, mesh);
  pamopt_cu_grid g = nullptr;
  cuda::check(pamopt_cu_compute_udf(ctx.get(), dm.get(), R, &g));
  ScalarGrid out;
  out.resolution = R;
  out.band = static_cast<float>(3.0 / R);
  const int64_t n = R + 1;
  out.samples.resize(n * n * n);
  const int rc = pamopt_cu_grid_download(g, out.samples.data());
  pamopt_cu_grid_free(g);
  cuda::check(rc);
  return out;
}

/// SPEC.md:203-211.  Throws std::invalid_argument when eps is outside
/// [sqrt(3)/(2R), 3/R - sqrt(3)/(2R)].
inline void udf_to_sdf(ScalarGrid& grid, double epsilon) {
  cuda::Context& ctx = cuda::Context::thread_default();
  pamopt_cu_grid g = nullptr;
  cuda::check(pamopt_cu_grid_upload(ctx.get(), grid.resolution, grid.samples.data(), &g));
  int rc = pamopt_cu_udf_to_sdf(g, epsilon);
  if (rc == PAMOPT_CU_OK) rc = pamopt_cu_grid_download(g, grid.samples.data());
  pamopt_cu_grid_free(g);
  cuda::check(rc);
  grid.epsilon = static_cast<float>(epsilon);
}

}  // namespace pamopt
