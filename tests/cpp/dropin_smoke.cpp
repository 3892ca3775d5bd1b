// Drop-in smoke test: the reference's own C++ types and algorithms (IndexedMesh,
// normalize_unit_cube, analyze_topology — compiled from /root/reference/proj/src) driving the
// GPU path through include/pamopt/*.hpp, exactly as a reference caller would.
// Built by tests/cpp/Makefile into tests/cpp/_bin/ (git-ignored, travels to the GPU box).
#include <cmath>
#include <cstdio>
#include <map>

#include "pamopt/dual_mc.hpp"
#include "pamopt/lbvh.hpp"
#include "pamopt/mesh.hpp"
#include "pamopt/mesh_io.hpp"
#include "pamopt/pipeline.hpp"
#include "pamopt/quality_metrics.hpp"
#include "pamopt/safe_project.hpp"
#include "pamopt/simplify.hpp"
#include "pamopt/tri_isect.hpp"
#include "pamopt/voxel_field.hpp"

using namespace pamopt;

static IndexedMesh icosphere(int sub) {
  const double t = (1.0 + std::sqrt(5.0)) / 2.0;
  IndexedMesh m;
  const double v[12][3] = {{-1, t, 0}, {1, t, 0}, {-1, -t, 0}, {1, -t, 0}, {0, -1, t}, {0, 1, t},
                           {0, -1, -t}, {0, 1, -t}, {t, 0, -1}, {t, 0, 1}, {-t, 0, -1}, {-t, 0, 1}};
  for (auto& p : v) {
    Vec3d q(p[0], p[1], p[2]);
    m.vertices.push_back(q / q.norm());
  }
  const int f[20][3] = {{0, 11, 5}, {0, 5, 1}, {0, 1, 7}, {0, 7, 10}, {0, 10, 11}, {1, 5, 9}, {5, 11, 4},
                        {11, 10, 2}, {10, 7, 6}, {7, 1, 8}, {3, 9, 4}, {3, 4, 2}, {3, 2, 6}, {3, 6, 8},
                        {3, 8, 9}, {4, 9, 5}, {2, 4, 11}, {6, 2, 10}, {8, 6, 7}, {9, 8, 1}};
  for (auto& q : f) m.faces.push_back(Vec3i(q[0], q[1], q[2]));
  for (int s = 0; s < sub; ++s) {
    std::map<std::pair<int, int>, int> mid;
    auto midpoint = [&](int a, int b) {
      auto key = std::make_pair(std::min(a, b), std::max(a, b));
      auto it = mid.find(key);
      if (it != mid.end()) return it->second;
      Vec3d p = m.vertices[a] + m.vertices[b];
      m.vertices.push_back(p / p.norm());
      return mid[key] = m.vertex_count() - 1;
    };
    std::vector<Vec3i> nf;
    for (const Vec3i& t3 : m.faces) {
      const int a = midpoint(t3[0], t3[1]), b = midpoint(t3[1], t3[2]), c = midpoint(t3[2], t3[0]);
      nf.push_back(Vec3i(t3[0], a, c));
      nf.push_back(Vec3i(t3[1], b, a));
      nf.push_back(Vec3i(t3[2], c, b));
      nf.push_back(Vec3i(a, b, c));
    }
    m.faces = nf;
  }
  return m;
}

int main() {
  const int R = 64;
  IndexedMesh in = icosphere(4);
  normalize_unit_cube(in, 6.0 / R);                  // reference mesh_io.cpp:393-408
  ScalarGrid g = compute_udf(in, R);                 // GPU
  udf_to_sdf(g, 0.9 / R);                            // GPU
  IndexedMesh d = extract(g);                        // GPU
  const TopologySummary td = analyze_topology(d);    // reference mesh.cpp:113-150
  const auto pd = detect_self_intersections(d);      // GPU
  SimplifyStats st;
  IndexedMesh s = simplify_to(d, 1000, SimplifyParams{}, &st);  // GPU
  const TopologySummary ts = analyze_topology(s);
  const auto ps = detect_self_intersections(s);
  StageTimings tm;
  IndexedMesh e = remesh(in, R, 1000, SimplifyParams{}, 0.0, 5.0, nullptr, &tm);
  const bool same = e.faces == s.faces && e.vertices == s.vertices;
  // GPU certification twins vs the reference's own CPU implementations
  const TopologySummary tg = cuda::analyze_topology(d);
  const bool topo_same = tg.manifold == td.manifold && tg.watertight == td.watertight &&
                         tg.euler_characteristic == td.euler_characteristic &&
                         tg.boundary_edge_count == td.boundary_edge_count &&
                         tg.nonmanifold_edges == td.nonmanifold_edges &&
                         tg.nonmanifold_vertices == td.nonmanifold_vertices;
  const TriangleBvh bvh = TriangleBvh::build(s);
  std::vector<Vec3d> q;
  for (int i = 0; i < 512; ++i) q.push_back(d.vertices[(i * 7919) % d.vertex_count()] * 1.01);
  const std::vector<NearestHit> hg = cuda::nearest_primitives(s, q);
  bool near_same = true;
  for (size_t i = 0; i < q.size(); ++i) {
    const NearestHit h = bvh.nearest_primitive(s, q[i]);  // reference lbvh.cpp:192-237
    near_same = near_same && h.primitive == hg[i].primitive && h.distance == hg[i].distance && h.point == hg[i].point;
  }
  const MeshReport rep = mesh_report(s, &in, 4096);
  pamopt_cu_project_params pp = default_projection_params();
  pp.iterations = 10;
  const IndexedMesh pj = project(s, in, pp);  // stage 3 (SPEC safe_project)
  const MeshReport rep3 = mesh_report(pj, &in, 4096);
  const bool proj_ok = pj.faces == s.faces && rep3.intersection_free && rep3.cd < rep.cd;
  // SPEC-granular operations against the reference's own code
  IndexedMesh dcopy = d;
  HalfEdgeAdjacency adj(dcopy);  // reference mesh.cpp:185-197
  std::vector<EdgeKey> ek;
  for (int f = 0; f < d.face_count() && ek.size() < 3000; f += 3) ek.push_back(EdgeKey(d.faces[f][0], d.faces[f][1]));
  const std::vector<bool> lk = link_condition_holds(d, ek);
  bool link_same = true;
  for (size_t i = 0; i < ek.size(); ++i) link_same = link_same && lk[i] == adj.link_condition_holds(ek[i].a, ek[i].b);
  SimplifySession sess(d, 1000);
  while (!sess.done()) {
    sess.prepare();
    sess.propagate_and_mark();
    sess.collapse_batch();
    sess.undo_loop();
    sess.end_iteration();
  }
  const IndexedMesh ss = sess.finish();
  const bool steps_same = ss.faces == s.faces && ss.vertices == s.vertices;
  PatchSoup soup;
  QuadMesh qm;
  dmc_stages(g, soup, qm);
  const IndexedMesh tq = triangulate_quads(R, soup, qm);
  const bool dmc_steps_same = tq.faces == d.faces && tq.vertices == d.vertices;
  // run_pipeline on the raw (un-normalised) input: certified, and equal to the reference's own
  // normalise -> remesh -> denormalise (mesh_io.cpp:393-412)
  IndexedMesh raw = icosphere(4);
  for (Vec3d& v : raw.vertices) v = v * 3.0 + Vec3d(1.0, -2.0, 0.5);
  PipelineConfig pc;
  pc.resolution = R;
  pc.target_faces = 1000;
  const PipelineResult pr = run_pipeline(raw, pc);
  IndexedMesh nr = raw;
  const NormalizationTransform nt = normalize_unit_cube(nr, 6.0 / R);
  IndexedMesh er = remesh(nr, R, 1000);
  denormalize(er, nt);
  const bool pipe_ok = pr.mesh.faces == er.faces && pr.mesh.vertices == er.vertices && pr.stages.size() == 2 &&
                       pr.stages[0].manifold && pr.stages[0].watertight && pr.stages[0].intersection_free &&
                       pr.stages[1].intersection_free && pr.mesh.face_count() <= 1000;
  std::printf("{\"dmc_faces\": %d, \"dmc_manifold\": %d, \"dmc_watertight\": %d, \"dmc_euler\": %d, "
              "\"dmc_isect\": %zu, \"out_faces\": %d, \"out_manifold\": %d, \"out_euler\": %d, \"out_isect\": %zu, "
              "\"iterations\": %lld, \"pipeline_equal\": %d, \"total_ms\": %.3f, \"topology_equal\": %d, "
              "\"nearest_equal\": %d, \"cd\": %.3e, \"hd\": %.3e, \"min_angle\": %.2f, \"projected_cd\": %.3e, "
              "\"projection_ok\": %d, \"link_equal\": %d, \"qem_steps_equal\": %d, \"dmc_steps_equal\": %d, "
              "\"run_pipeline_ok\": %d}\n",
              d.face_count(), td.manifold, td.watertight, td.euler_characteristic, pd.size(), s.face_count(),
              ts.manifold, ts.euler_characteristic, ps.size(), static_cast<long long>(st.iterations), same,
              tm.total_ms, topo_same, near_same, rep.cd, rep.hd, rep.min_angle_deg, rep3.cd, proj_ok, link_same,
              steps_same, dmc_steps_same, pipe_ok);
  const bool ok = td.manifold && td.watertight && pd.empty() && ts.manifold && ps.empty() && s.face_count() <= 1000 &&
                  same && topo_same && near_same && rep.watertight && rep.intersection_free && proj_ok && link_same &&
                  steps_same && dmc_steps_same && pipe_ok;
  std::fflush(stdout);
  std::_Exit(ok ? 0 : 1);  // parallel.cpp pool: never run static destructors
}
