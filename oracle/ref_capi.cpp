// C wrapper over the REFERENCE's own translation units — TEST INFRASTRUCTURE ONLY.
//
// Built by oracle/Makefile (target `ref`) together with
//   /root/reference/proj/src/{distance,mesh,lbvh,parallel,mesh_io}.cpp
// into oracle/_ref/libpamopt_ref.so.  Only tests/ and bench.py's reference arm
// load it, to pin the oracle restatement (oracle/src) against the reference's
// actual code: point_triangle_sq_distance (distance.cpp:26-79),
// HalfEdgeAdjacency::link_condition_holds / collapse_edge / undo_collapse
// (mesh.cpp:301-416), analyze_topology (mesh.cpp:113-150) and the LBVH overlap
// semantics (lbvh.cpp:159-190, inflation lbvh.hpp:72).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "pamopt/distance.hpp"
#include "pamopt/lbvh.hpp"
#include "pamopt/mesh.hpp"
#include "pamopt/mesh_io.hpp"
#include "pamopt/parallel.hpp"

using namespace pamopt;

namespace {
IndexedMesh make_mesh(const double* v, int64_t nv, const int32_t* f, int64_t nf) {
  IndexedMesh m;
  m.vertices.resize(nv);
  for (int64_t i = 0; i < nv; ++i) m.vertices[i] = Vec3d(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  m.faces.resize(nf);
  for (int64_t i = 0; i < nf; ++i) m.faces[i] = Vec3i(f[3 * i], f[3 * i + 1], f[3 * i + 2]);
  return m;
}
// The reference pool aborts at process exit once its threads exist (parallel.cpp:24-92,
// SURVEY §0.6); a single worker keeps every loop serial so no thread is ever created.
[[maybe_unused]] const int kSerial = (set_worker_count(1), 0);
}  // namespace

extern "C" {

void ref_set_workers(int n) { set_worker_count(n); }

// distance.cpp:26-79 (double instantiation), batched.
void ref_point_triangle_sq_distance(const double* p, const double* a, const double* b,
                                    const double* c, int64_t n, double* out, int32_t* region) {
  for (int64_t i = 0; i < n; ++i) {
    TriRegion r;
    out[i] = point_triangle_sq_distance<double>(
        Vec3d(p[3 * i], p[3 * i + 1], p[3 * i + 2]), Vec3d(a[3 * i], a[3 * i + 1], a[3 * i + 2]),
        Vec3d(b[3 * i], b[3 * i + 1], b[3 * i + 2]), Vec3d(c[3 * i], c[3 * i + 1], c[3 * i + 2]),
        nullptr, &r);
    if (region) region[i] = static_cast<int32_t>(r);
  }
}

// mesh.cpp:113-150.  out = {manifold, watertight, euler, boundary_edges, n_nonmanifold_edges, n_nonmanifold_vertices}
int ref_analyze_topology(const double* v, int64_t nv, const int32_t* f, int64_t nf, int64_t* out) {
  try {
    IndexedMesh m = make_mesh(v, nv, f, nf);
    TopologySummary s = analyze_topology(m);
    out[0] = s.manifold;
    out[1] = s.watertight;
    out[2] = s.euler_characteristic;
    out[3] = s.boundary_edge_count;
    out[4] = static_cast<int64_t>(s.nonmanifold_edges.size());
    out[5] = static_cast<int64_t>(s.nonmanifold_vertices.size());
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// mesh.cpp:113-150, the lists: nonmanifold edges as (a<<32|b) in std::map order, vertices ascending
int ref_analyze_topology_lists(const double* v, int64_t nv, const int32_t* f, int64_t nf, int64_t* edges,
                               int32_t* verts) {
  try {
    IndexedMesh m = make_mesh(v, nv, f, nf);
    TopologySummary s = analyze_topology(m);
    for (size_t i = 0; i < s.nonmanifold_edges.size(); ++i)
      edges[i] = (static_cast<int64_t>(s.nonmanifold_edges[i].a) << 32) | static_cast<uint32_t>(s.nonmanifold_edges[i].b);
    for (size_t i = 0; i < s.nonmanifold_vertices.size(); ++i) verts[i] = s.nonmanifold_vertices[i];
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// mesh_io.cpp:372-385: load_mesh; the result is kept for ref_load_fetch.  stats = {degenerate
// faces dropped, polygons triangulated, vertices welded}; returns 0, or -1 on a load error
static IndexedMesh g_loaded;
int ref_load_mesh(const char* path, int64_t* nv, int64_t* nf, int64_t* stats) {
  try {
    LoadStats st;
    g_loaded = load_mesh(path, &st);
    *nv = g_loaded.vertex_count();
    *nf = g_loaded.face_count();
    stats[0] = st.degenerate_faces_dropped;
    stats[1] = st.polygons_triangulated;
    stats[2] = st.vertices_welded;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}
void ref_load_fetch(double* v, int32_t* f) {
  for (int i = 0; i < g_loaded.vertex_count(); ++i)
    for (int k = 0; k < 3; ++k) v[3 * i + k] = g_loaded.vertices[i][k];
  for (int i = 0; i < g_loaded.face_count(); ++i)
    for (int k = 0; k < 3; ++k) f[3 * i + k] = g_loaded.faces[i][k];
}

// lbvh.cpp:192-237: TriangleBvh::nearest_primitive for a batch of points
int ref_nearest_primitive(const double* v, int64_t nv, const int32_t* f, int64_t nf, const double* pts, int64_t n,
                          int32_t* face, double* dist, double* closest) {
  try {
    IndexedMesh m = make_mesh(v, nv, f, nf);
    const TriangleBvh bvh = TriangleBvh::build(m);
    for (int64_t i = 0; i < n; ++i) {
      const NearestHit h = bvh.nearest_primitive(m, Vec3d(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
      face[i] = h.primitive;
      dist[i] = h.distance;
      for (int k = 0; k < 3; ++k) closest[3 * i + k] = h.point[k];
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// mesh.cpp:301-358 for a list of edges (a,b); result 1/0, -1 = unknown edge (invalid_argument).
int ref_link_condition(const double* v, int64_t nv, const int32_t* f, int64_t nf,
                       const int32_t* edges, int64_t ne, int32_t* out) {
  try {
    IndexedMesh m = make_mesh(v, nv, f, nf);
    HalfEdgeAdjacency adj(m);
    for (int64_t i = 0; i < ne; ++i) {
      try {
        out[i] = adj.link_condition_holds(edges[2 * i], edges[2 * i + 1]) ? 1 : 0;
      } catch (const std::invalid_argument&) {
        out[i] = -1;
      }
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// Sequential collapse_edge (mesh.cpp:363-395) of (a_i,b_i) to pos_i, then compact()
// (mesh.cpp:278-292).  ok[i] = 1 if applied.  Output mesh sizes returned via out_nv/out_nf;
// out_v/out_f must hold nv / nf entries.  If undo != 0 every applied collapse is undone in
// reverse order (mesh.cpp:397-416) before compaction.
int ref_collapse_sequence(const double* v, int64_t nv, const int32_t* f, int64_t nf,
                          const int32_t* edges, const double* pos, int64_t ne, int undo,
                          int32_t* ok, double* out_v, int32_t* out_f, int64_t* out_nv,
                          int64_t* out_nf) {
  try {
    IndexedMesh m = make_mesh(v, nv, f, nf);
    HalfEdgeAdjacency adj(m);
    std::vector<CollapseRecord> recs;
    for (int64_t i = 0; i < ne; ++i) {
      try {
        auto r = adj.collapse_edge(edges[2 * i], edges[2 * i + 1],
                                   Vec3d(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]));
        ok[i] = r.has_value() ? 1 : 0;
        if (r) recs.push_back(std::move(*r));
      } catch (const std::invalid_argument&) {
        ok[i] = -1;  // the edge no longer exists (mesh.cpp:302)
      }
    }
    if (undo)
      for (auto it = recs.rbegin(); it != recs.rend(); ++it) adj.undo_collapse(*it);
    IndexedMesh c = adj.compact();
    *out_nv = c.vertex_count();
    *out_nf = c.face_count();
    for (int i = 0; i < c.vertex_count(); ++i)
      for (int k = 0; k < 3; ++k) out_v[3 * i + k] = c.vertices[i][k];
    for (int i = 0; i < c.face_count(); ++i)
      for (int k = 0; k < 3; ++k) out_f[3 * i + k] = c.faces[i][k];
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// All unordered face pairs (i<j) whose inflated boxes overlap: TriangleBvh::build +
// query_overlaps per face (lbvh.cpp:159-190).  Count-then-fill: call with pairs=nullptr
// to get the count.
int64_t ref_bvh_overlap_pairs(const double* v, int64_t nv, const int32_t* f, int64_t nf,
                              int32_t* pairs, int64_t cap) {
  IndexedMesh m = make_mesh(v, nv, f, nf);
  TriangleBvh bvh = TriangleBvh::build(m);
  int64_t n = 0;
  for (int i = 0; i < m.face_count(); ++i) {
    const Vec3i& t = m.faces[i];
    Aabb box = triangle_aabb(m.vertices[t[0]], m.vertices[t[1]], m.vertices[t[2]]);
    box.inflate(TriangleBvh::kInflation);
    for (int j : bvh.query_overlaps(box, i)) {
      if (j <= i) continue;
      if (pairs && n < cap) {
        pairs[2 * n] = i;
        pairs[2 * n + 1] = j;
      }
      ++n;
    }
  }
  return n;
}

// mesh_io.cpp:393-408
int ref_normalize_unit_cube(double* v, int64_t nv, double padding, double* scale_translation) {
  try {
    IndexedMesh m;
    m.vertices.resize(nv);
    for (int64_t i = 0; i < nv; ++i) m.vertices[i] = Vec3d(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    NormalizationTransform t = normalize_unit_cube(m, padding);
    for (int64_t i = 0; i < nv; ++i)
      for (int k = 0; k < 3; ++k) v[3 * i + k] = m.vertices[i][k];
    scale_translation[0] = t.scale;
    for (int k = 0; k < 3; ++k) scale_translation[1 + k] = t.translation[k];
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
