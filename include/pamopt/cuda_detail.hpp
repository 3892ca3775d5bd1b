// pamopt/cuda_detail.hpp — shared plumbing of the drop-in headers (voxel_field.hpp,
// dual_mc.hpp, tri_isect.hpp, simplify.hpp, pipeline.hpp): status -> exception mapping,
// RAII handles and a per-thread device context.  Header-only; links against libpamopt_cu.so.
//
// Error mapping (the reference's conventions):
//   PAMOPT_CU_EINVAL            -> std::invalid_argument  (mesh.cpp:186-187,302)
//   PAMOPT_CU_ENUMERIC          -> std::domain_error      (NaN cost)
//   everything else             -> std::runtime_error
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "pamopt/mesh.hpp"
#include "pamopt_cu.h"

namespace pamopt {
namespace cuda {

inline void check(int rc) {
  if (rc == PAMOPT_CU_OK) return;
  const std::string msg = std::string("pamopt_cu: ") + pamopt_cu_last_error();
  if (rc == PAMOPT_CU_EINVAL) throw std::invalid_argument(msg);
  if (rc == PAMOPT_CU_ENUMERIC) throw std::domain_error(msg);
  throw std::runtime_error(msg);
}

/// Device + stream binding.  One per host thread by default (calls on distinct contexts are
/// thread-safe; the reference's worker-count global has no GPU analogue).
class Context {
 public:
  explicit Context(int device = 0) { check(pamopt_cu_ctx_create(device, &h_)); }
  ~Context() { pamopt_cu_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  pamopt_cu_ctx get() const { return h_; }
  static Context& thread_default() {
    thread_local Context ctx(0);
    return ctx;
  }

 private:
  pamopt_cu_ctx h_ = nullptr;
};

/// Device-resident IndexedMesh.
class DeviceMesh {
 public:
  DeviceMesh() = default;
  DeviceMesh(Context& ctx, const IndexedMesh& m) {
    std::vector<double> v(3 * m.vertices.size());
    std::vector<int32_t> f(3 * m.faces.size());
    for (size_t i = 0; i < m.vertices.size(); ++i)
      for (int k = 0; k < 3; ++k) v[3 * i + k] = m.vertices[i][k];
    for (size_t i = 0; i < m.faces.size(); ++i)
      for (int k = 0; k < 3; ++k) f[3 * i + k] = m.faces[i][k];
    check(pamopt_cu_mesh_upload(ctx.get(), v.data(), static_cast<int64_t>(m.vertices.size()), f.data(),
                                static_cast<int64_t>(m.faces.size()), &h_));
  }
  explicit DeviceMesh(pamopt_cu_mesh h) : h_(h) {}
  ~DeviceMesh() { pamopt_cu_mesh_free(h_); }
  DeviceMesh(DeviceMesh&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  DeviceMesh& operator=(DeviceMesh&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  pamopt_cu_mesh get() const { return h_; }
  IndexedMesh download() const {
    int64_t nv = 0, nf = 0;
    check(pamopt_cu_mesh_size(h_, &nv, &nf));
    std::vector<double> v(3 * nv);
    std::vector<int32_t> f(3 * nf);
    check(pamopt_cu_mesh_download(h_, v.data(), f.data()));
    IndexedMesh m;
    m.vertices.resize(nv);
    m.faces.resize(nf);
    for (int64_t i = 0; i < nv; ++i) m.vertices[i] = Vec3d(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    for (int64_t i = 0; i < nf; ++i) m.faces[i] = Vec3i(f[3 * i], f[3 * i + 1], f[3 * i + 2]);
    return m;
  }

 private:
  pamopt_cu_mesh h_ = nullptr;
};

}  // namespace cuda
}  // namespace pamopt
