// ORACLE (test infrastructure only) — stage 2: parallel intersection-free QEM
// simplification (Algorithm 1), restated from SPEC.md:473-574 and PAPER.md:117-165,229-238,
// on top of the reference's link condition / collapse / undo semantics (mesh.cpp:301-416).
//
// Pinned semantics (SURVEY pins P5-P10):
//   quadrics  K_v = sum over incident faces in ascending face id of A_f * p p^T (unit plane p,
//             area A_f); merged K_a + K_b on collapse, restored on undo
//   edges     ids = lexicographic rank of (a<b) over the edges of alive faces at iteration start
//   cost      Eq. 1: Q(x) + w_e*|ab| + w_s * sum over post-collapse ring faces (ascending id)
//             of (1 - 4*sqrt(3)*A/(l01+l12+l20)); placement = argmin of the merged quadric
//             (adjugate inverse), falling back to the cheapest of {mid, a, b} when
//             det == 0 or ||A||_1 * ||A^-1||_1 > 1e8
//   key       (f32 bits of max(cost,0)) << 32 | edge id; NaN -> error
//   marking   face key = min over edges whose ring holds it = min of its vertices' incident
//             edge keys; an edge is marked iff every face of ring(a) ∪ ring(b) holds its key
//             (invalid edges take no part, P7)
//   collapse  link condition (mesh.cpp:301-358) on the pre-batch mesh for every marked edge;
//             failures flagged invalid; if the batch would undershoot the target only the
//             smallest keys are kept (P9); b merges into a (mesh.cpp:363-395, P6)
//   undo      repeat: intersecting pairs (exact verdict, isect.cpp) among alive faces that
//             touch a face owned by an applied collapse of this batch -> revert every applied
//             collapse owning either face and flag it invalid (P10); until clean
//   flags     invalid flags live one iteration; an iteration with zero successful collapses
//             keeps (accumulates) them, for at most `tolerance` such iterations
//   stop      alive faces <= target, or 10 consecutive iterations without a collapse
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <set>
#include <vector>

#include "geom.hpp"
#include "par.hpp"

namespace orc {

bool tri_tri_verdict(const int32_t* t1, const int32_t* t2, const double* v);
std::vector<std::pair<int32_t, int32_t>> detect_pairs(const double* v, const int32_t* f, int64_t nf,
                                                      const uint8_t* alive, const uint8_t* query);

namespace simp {

constexpr double k4Sqrt3 = 6.928203230275509;

struct Quadric {
  double q[10];
};

struct Params {
  double we, ws;
  int tolerance;
  int stall;
};

struct Mesh {
  std::vector<double> X;  // 3V
  std::vector<int32_t> F; // 3F
  std::vector<uint8_t> valive, falive;
  std::vector<Quadric> Q;
  int64_t nv = 0, nf = 0, alive_faces = 0;
  V3 pos(int v) const { return v3(X[3 * v], X[3 * v + 1], X[3 * v + 2]); }
  const int32_t* face(int f) const { return &F[3 * f]; }
};

static void face_quadric(const Mesh& m, int f, double* out) {
  const int32_t* t = m.face(f);
  const V3 p0 = m.pos(t[0]), p1 = m.pos(t[1]), p2 = m.pos(t[2]);
  const V3 n = cross(p1 - p0, p2 - p0);
  const double len = std::sqrt(sqnorm(n));
  if (!(len > 0.0)) {
    for (int k = 0; k < 10; ++k) out[k] = 0.0;
    return;
  }
  const double a = n.x / len, b = n.y / len, c = n.z / len;
  const double d = -((a * p0.x + b * p0.y) + c * p0.z);
  const double w = 0.5 * len;
  out[0] = w * (a * a); out[1] = w * (a * b); out[2] = w * (a * c); out[3] = w * (a * d);
  out[4] = w * (b * b); out[5] = w * (b * c); out[6] = w * (b * d);
  out[7] = w * (c * c); out[8] = w * (c * d);
  out[9] = w * (d * d);
}

static double qeval(const double* q, V3 p) {
  const double x = p.x, y = p.y, z = p.z;
  double r = q[0] * x * x;
  r = r + 2.0 * q[1] * x * y;
  r = r + 2.0 * q[2] * x * z;
  r = r + 2.0 * q[3] * x;
  r = r + q[4] * y * y;
  r = r + 2.0 * q[5] * y * z;
  r = r + 2.0 * q[6] * y;
  r = r + q[7] * z * z;
  r = r + 2.0 * q[8] * z;
  r = r + q[9];
  return r < 0.0 ? 0.0 : r;
}

// CSR vertex -> alive faces (ascending face id)
struct Incidence {
  std::vector<int64_t> off;
  std::vector<int32_t> idx;
  const int32_t* begin(int v) const { return idx.data() + off[v]; }
  const int32_t* end(int v) const { return idx.data() + off[v + 1]; }
  int64_t size(int v) const { return off[v + 1] - off[v]; }
};

static Incidence build_incidence(const Mesh& m) {
  Incidence I;
  I.off.assign(m.nv + 1, 0);
  for (int64_t f = 0; f < m.nf; ++f)
    if (m.falive[f])
      for (int k = 0; k < 3; ++k) I.off[m.F[3 * f + k] + 1]++;
  for (int64_t v = 0; v < m.nv; ++v) I.off[v + 1] += I.off[v];
  I.idx.resize(I.off[m.nv]);
  std::vector<int64_t> cur(I.off.begin(), I.off.end() - 1);
  for (int64_t f = 0; f < m.nf; ++f)
    if (m.falive[f])
      for (int k = 0; k < 3; ++k) I.idx[cur[m.F[3 * f + k]]++] = static_cast<int32_t>(f);
  return I;
}

static bool has(const int32_t* t, int v) { return t[0] == v || t[1] == v || t[2] == v; }

static double ring_skinny(const Mesh& m, const Incidence& I, int a, int b, V3 x) {
  // union of faces(a), faces(b) in ascending id, skipping faces holding both
  const int32_t *ia = I.begin(a), *ea = I.end(a), *ib = I.begin(b), *eb = I.end(b);
  double cs = 0.0;
  while (ia != ea || ib != eb) {
    int f;
    if (ib == eb || (ia != ea && *ia < *ib)) f = *ia++;
    else if (ia == ea || *ib < *ia) f = *ib++;
    else { f = *ia++; ++ib; }
    const int32_t* t = m.face(f);
    if (has(t, a) && has(t, b)) continue;
    V3 P[3];
    for (int k = 0; k < 3; ++k) P[k] = (t[k] == a || t[k] == b) ? x : m.pos(t[k]);
    const V3 n = cross(P[1] - P[0], P[2] - P[0]);
    const double area = 0.5 * std::sqrt(sqnorm(n));
    const double l01 = sqnorm(P[1] - P[0]), l12 = sqnorm(P[2] - P[1]), l20 = sqnorm(P[0] - P[2]);
    const double den = (l01 + l12) + l20;
    const double c = den > 0.0 ? (k4Sqrt3 * area) / den : 0.0;
    cs = cs + (1.0 - c);
  }
  return cs;
}

struct CostOut {
  double cost;
  V3 x;
};

static CostOut edge_cost(const Mesh& m, const Incidence& I, int a, int b, const Params& P) {
  double q[10];
  for (int k = 0; k < 10; ++k) q[k] = m.Q[a].q[k] + m.Q[b].q[k];
  const V3 pa = m.pos(a), pb = m.pos(b);
  const double l = std::sqrt(sqnorm(pa - pb));
  const double m00 = q[0], m01 = q[1], m02 = q[2], m10 = q[1], m11 = q[4], m12 = q[5], m20 = q[2],
               m21 = q[5], m22 = q[7];
  const double det = m00 * (m11 * m22 - m12 * m21) - m01 * (m10 * m22 - m12 * m20) +
                     m02 * (m10 * m21 - m11 * m20);
  bool ok = det != 0.0;
  V3 x{0, 0, 0};
  if (ok) {
    const double rdet = 1.0 / det;  // adjugate * (1/det)
    const double i00 = (m11 * m22 - m12 * m21) * rdet, i01 = (m02 * m21 - m01 * m22) * rdet,
                 i02 = (m01 * m12 - m02 * m11) * rdet, i10 = (m12 * m20 - m10 * m22) * rdet,
                 i11 = (m00 * m22 - m02 * m20) * rdet, i12 = (m02 * m10 - m00 * m12) * rdet,
                 i20 = (m10 * m21 - m11 * m20) * rdet, i21 = (m01 * m20 - m00 * m21) * rdet,
                 i22 = (m00 * m11 - m01 * m10) * rdet;
    auto colmax = [](double c0, double c1, double c2) {
      return std::max(std::max(c0, c1), c2);
    };
    const double nA = colmax((std::fabs(m00) + std::fabs(m10)) + std::fabs(m20),
                             (std::fabs(m01) + std::fabs(m11)) + std::fabs(m21),
                             (std::fabs(m02) + std::fabs(m12)) + std::fabs(m22));
    const double nI = colmax((std::fabs(i00) + std::fabs(i10)) + std::fabs(i20),
                             (std::fabs(i01) + std::fabs(i11)) + std::fabs(i21),
                             (std::fabs(i02) + std::fabs(i12)) + std::fabs(i22));
    const double cond = nA * nI;
    if (!(cond <= 1e8)) ok = false;
    else {
      const double b0 = q[3], b1 = q[6], b2 = q[8];
      x = v3(-((i00 * b0 + i01 * b1) + i02 * b2), -((i10 * b0 + i11 * b1) + i12 * b2),
             -((i20 * b0 + i21 * b1) + i22 * b2));
    }
  }
  auto full = [&](V3 p) {
    return (qeval(q, p) + P.we * l) + P.ws * ring_skinny(m, I, a, b, p);
  };
  if (ok) return CostOut{full(x), x};
  const V3 cand[3] = {v3((pa.x + pb.x) * 0.5, (pa.y + pb.y) * 0.5, (pa.z + pb.z) * 0.5), pa, pb};
  CostOut best{full(cand[0]), cand[0]};
  for (int k = 1; k < 3; ++k) {
    const double c = full(cand[k]);
    if (c < best.cost) best = CostOut{c, cand[k]};
  }
  return best;
}

// ---- link condition: restatement of mesh.cpp:301-358 over the incidence lists -----------
static bool is_boundary_vertex(const Mesh& m, const Incidence& I, int v) {
  std::vector<int> ring;
  for (const int32_t* p = I.begin(v); p != I.end(v); ++p) {
    const int32_t* t = m.face(*p);
    for (int k = 0; k < 3; ++k)
      if (t[k] != v) ring.push_back(t[k]);
  }
  std::sort(ring.begin(), ring.end());
  for (size_t i = 0; i < ring.size();) {
    size_t j = i;
    while (j < ring.size() && ring[j] == ring[i]) ++j;
    if (j - i == 1) return true;
    i = j;
  }
  return false;
}
static int faces_of_edge_count(const Mesh& m, const Incidence& I, int a, int b, int32_t* out = nullptr) {
  int n = 0;
  for (const int32_t* p = I.begin(a); p != I.end(a); ++p)
    if (has(m.face(*p), b)) {
      if (out) out[n] = *p;
      ++n;
    }
  return n;
}

static bool link_condition(const Mesh& m, const Incidence& I, int a, int b) {
  constexpr int VB = -2;
  auto link_vertices = [&](int v) {
    std::set<int> out;
    for (const int32_t* p = I.begin(v); p != I.end(v); ++p) {
      const int32_t* t = m.face(*p);
      for (int k = 0; k < 3; ++k)
        if (t[k] != v) out.insert(t[k]);
    }
    if (is_boundary_vertex(m, I, v)) out.insert(VB);
    return out;
  };
  const std::set<int> la = link_vertices(a), lb = link_vertices(b);
  std::set<int> common;
  std::set_intersection(la.begin(), la.end(), lb.begin(), lb.end(), std::inserter(common, common.begin()));
  std::set<int> link_ab;
  const int nfe = faces_of_edge_count(m, I, a, b, nullptr);
  std::vector<int32_t> fev(nfe);
  faces_of_edge_count(m, I, a, b, fev.data());
  for (int32_t f : fev) {
    const int32_t* t = m.face(f);
    for (int k = 0; k < 3; ++k)
      if (t[k] != a && t[k] != b) link_ab.insert(t[k]);
  }
  if (nfe == 1) link_ab.insert(VB);
  if (common != link_ab) return false;
  for (int x : common) {
    if (x == VB) continue;
    for (int y : common) {
      if (y == VB || y <= x) continue;
      bool in_la = false, in_lb = false;
      for (const int32_t* p = I.begin(x); p != I.end(x); ++p) {
        const int32_t* t = m.face(*p);
        if (!has(t, y)) continue;
        if (has(t, a)) in_la = true;
        if (has(t, b)) in_lb = true;
      }
      if (in_la && in_lb) return false;
    }
    if (common.count(VB)) {
      if (faces_of_edge_count(m, I, a, x) == 1 && faces_of_edge_count(m, I, b, x) == 1) return false;
    }
  }
  return true;
}

struct Collapse {
  int a, b;
  V3 x;
  uint64_t key;
  V3 old_x;
  Quadric old_q;
  std::vector<std::pair<int, std::array<int32_t, 3>>> bfaces;  // pre-collapse faces of b
  std::vector<int> owned;                                      // faces holding a afterwards
  bool applied = false;
};

struct Stats {
  int64_t iterations = 0;
  int64_t collapses = 0;
  int64_t undone = 0;
  int64_t link_failures = 0;
  int64_t undo_hist[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // batches needing k undo rounds (7 = >=7)
  int64_t max_undo_rounds = 0;
  int64_t face_iterations = 0;
  int error = 0;
};

// Step-level record of one iteration (granular parity tests of the SPEC operations)
struct Trace {
  int64_t iter = 0;  // 1-based iteration to record; the run stops after it
  std::vector<std::pair<int32_t, int32_t>> edges;
  std::vector<uint64_t> keys;       // ~0 for an invalid edge
  std::vector<double> place;        // 3 per edge
  std::vector<uint64_t> face_keys;  // per face slot, ~0 for a dead face
  std::vector<int64_t> marked;      // edge ids, ascending
  std::vector<uint8_t> link_ok;     // per marked edge
  std::vector<int64_t> applied;     // edge ids of the collapses that survived the undo loop
  int64_t rounds = 0;
  std::vector<double> X;
  std::vector<int32_t> F;
  std::vector<uint8_t> falive;
};

// ORC_PROFILE=1: per-phase wall seconds on stderr (diagnostics of the CPU baseline only)
struct PhaseTimer {
  bool on = std::getenv("ORC_PROFILE") != nullptr;
  double t[10] = {0};
  std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
  void mark(int i) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    t[i] += std::chrono::duration<double>(now - last).count();
    last = now;
  }
  ~PhaseTimer() {
    if (on)
      std::fprintf(stderr, "orc simplify s: incidence %.2f edges %.2f cost %.2f mark %.2f link %.2f collapse %.2f "
                   "detect %.2f revert %.2f flags %.2f\n", t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8]);
  }
};

static void run(Mesh& m, int64_t target, const Params& P, Stats& S,
                std::vector<int64_t>* per_iter_collapses, Trace* tr = nullptr) {
  PhaseTimer T;
  // initial quadrics, gathered in ascending face id
  m.Q.assign(m.nv, Quadric{});
  for (auto& q : m.Q) std::fill(q.q, q.q + 10, 0.0);
  for (int64_t f = 0; f < m.nf; ++f) {
    if (!m.falive[f]) continue;
    double fq[10];
    face_quadric(m, static_cast<int>(f), fq);
    for (int k = 0; k < 3; ++k) {
      Quadric& Q = m.Q[m.F[3 * f + k]];
      for (int i = 0; i < 10; ++i) Q.q[i] = Q.q[i] + fq[i];
    }
  }
  std::set<std::pair<int, int>> invalid;
  int retain = 0, zero_run = 0;
  while (m.alive_faces > target && zero_run < P.stall) {
    S.iterations++;
    S.face_iterations += m.alive_faces;
    T.mark(8);
    const Incidence I = build_incidence(m);
    T.mark(0);
    // edges in lexicographic order
    // (per vertex: sorted unique upper neighbours, counted then written at scanned offsets)
    auto upper = [&](int64_t v, std::vector<int32_t>& nb) {
      nb.clear();
      for (const int32_t* p = I.begin(static_cast<int>(v)); p != I.end(static_cast<int>(v)); ++p) {
        const int32_t* t = m.face(*p);
        for (int k = 0; k < 3; ++k)
          if (t[k] > v) nb.push_back(t[k]);
      }
      std::sort(nb.begin(), nb.end());
      nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
    };
    std::vector<int64_t> eoff(m.nv + 1, 0);
    constexpr int64_t kVChunk = 4096;
    const int64_t nvc = (m.nv + kVChunk - 1) / kVChunk;
    parallel_for(nvc, [&](int64_t c) {
      std::vector<int32_t> nb;
      for (int64_t v = c * kVChunk; v < std::min<int64_t>(m.nv, (c + 1) * kVChunk); ++v) {
        upper(v, nb);
        eoff[v + 1] = static_cast<int64_t>(nb.size());
      }
    }, 1);
    for (int64_t v = 0; v < m.nv; ++v) eoff[v + 1] += eoff[v];
    std::vector<std::pair<int32_t, int32_t>> edges(eoff[m.nv]);
    parallel_for(nvc, [&](int64_t c) {
      std::vector<int32_t> nb;
      for (int64_t v = c * kVChunk; v < std::min<int64_t>(m.nv, (c + 1) * kVChunk); ++v) {
        upper(v, nb);
        for (size_t i = 0; i < nb.size(); ++i) edges[eoff[v] + i] = {static_cast<int32_t>(v), nb[i]};
      }
    }, 1);
    T.mark(1);
    const int64_t ne = static_cast<int64_t>(edges.size());
    std::vector<uint64_t> key(ne, ~0ull);
    std::vector<V3> place(ne);
    std::vector<uint8_t> valid(ne, 1);
    int err = 0;
    if (!invalid.empty())
      parallel_for(ne, [&](int64_t e) {
        if (invalid.count(edges[e])) valid[e] = 0;
      }, 4096);
    parallel_for(ne, [&](int64_t e) {
      if (!valid[e]) return;
      const CostOut c = edge_cost(m, I, edges[e].first, edges[e].second, P);
      if (c.cost != c.cost) {
        err = 1;
        return;
      }
      const float cf = static_cast<float>(c.cost < 0.0 ? 0.0 : c.cost);
      uint32_t bits;
      std::memcpy(&bits, &cf, 4);
      key[e] = (static_cast<uint64_t>(bits) << 32) | static_cast<uint64_t>(e);
      place[e] = c.x;
    }, 512);
    if (err) {
      S.error = 1;
      return;
    }
    T.mark(2);
    std::vector<uint64_t> vmin(m.nv, ~0ull), vfmin(m.nv, ~0ull);
    for (int64_t e = 0; e < ne; ++e) {
      if (!valid[e]) continue;
      vmin[edges[e].first] = std::min(vmin[edges[e].first], key[e]);
      vmin[edges[e].second] = std::min(vmin[edges[e].second], key[e]);
    }
    for (int64_t f = 0; f < m.nf; ++f) {
      if (!m.falive[f]) continue;
      const int32_t* t = m.face(static_cast<int>(f));
      const uint64_t fk = std::min(std::min(vmin[t[0]], vmin[t[1]]), vmin[t[2]]);
      for (int k = 0; k < 3; ++k) vfmin[t[k]] = std::min(vfmin[t[k]], fk);
    }
    std::vector<int64_t> marked;
    for (int64_t e = 0; e < ne; ++e)
      if (valid[e] && key[e] == vfmin[edges[e].first] && key[e] == vfmin[edges[e].second])
        marked.push_back(e);
    const bool rec = tr && S.iterations == tr->iter;
    if (rec) {
      tr->edges = edges;
      tr->keys = key;
      tr->place.resize(3 * ne);
      for (int64_t e = 0; e < ne; ++e) {
        tr->place[3 * e] = place[e].x;
        tr->place[3 * e + 1] = place[e].y;
        tr->place[3 * e + 2] = place[e].z;
      }
      tr->face_keys.assign(m.nf, ~0ull);
      for (int64_t f = 0; f < m.nf; ++f)
        if (m.falive[f]) {
          const int32_t* t = m.face(static_cast<int>(f));
          tr->face_keys[f] = std::min(std::min(vmin[t[0]], vmin[t[1]]), vmin[t[2]]);
        }
      tr->marked = marked;
    }
    T.mark(3);
    // link condition on the pre-batch mesh
    std::vector<uint8_t> pass(marked.size());
    parallel_for(static_cast<int64_t>(marked.size()), [&](int64_t i) {
      pass[i] = link_condition(m, I, edges[marked[i]].first, edges[marked[i]].second) ? 1 : 0;
    }, 64);
    T.mark(4);
    if (rec) tr->link_ok = pass;
    std::set<std::pair<int, int>> new_invalid;
    std::vector<int64_t> sel;
    for (size_t i = 0; i < marked.size(); ++i) {
      if (pass[i]) sel.push_back(marked[i]);
      else {
        new_invalid.insert(edges[marked[i]]);
        S.link_failures++;
      }
    }
    // overshoot trim (P9)
    {
      int64_t removed = 0;
      for (int64_t e : sel) removed += faces_of_edge_count(m, I, edges[e].first, edges[e].second);
      if (m.alive_faces - removed < target) {
        std::vector<int64_t> byk = sel;
        std::sort(byk.begin(), byk.end(), [&](int64_t x, int64_t y) { return key[x] < key[y]; });
        std::vector<int64_t> keep;
        int64_t rem = 0;
        for (int64_t e : byk) {
          if (m.alive_faces - rem <= target) break;
          keep.push_back(e);
          rem += faces_of_edge_count(m, I, edges[e].first, edges[e].second);
        }
        std::sort(keep.begin(), keep.end());
        sel = keep;
      }
    }
    // collapse (regions are disjoint: order irrelevant; ascending edge id)
    std::vector<Collapse> cols(sel.size());
    std::vector<int32_t> owner(m.nf, -1);
    for (size_t ci = 0; ci < sel.size(); ++ci) {
      Collapse& C = cols[ci];
      const int a = edges[sel[ci]].first, b = edges[sel[ci]].second;
      C.a = a;
      C.b = b;
      C.x = place[sel[ci]];
      C.key = key[sel[ci]];
      C.old_x = m.pos(a);
      C.old_q = m.Q[a];
      for (const int32_t* p = I.begin(b); p != I.end(b); ++p) {
        const int32_t* t = m.face(*p);
        C.bfaces.push_back({*p, {t[0], t[1], t[2]}});
      }
      for (auto& bf : C.bfaces) {
        int32_t* t = &m.F[3 * bf.first];
        if (has(t, a)) {
          m.falive[bf.first] = 0;
          m.alive_faces--;
        } else {
          for (int k = 0; k < 3; ++k)
            if (t[k] == b) t[k] = a;
        }
      }
      m.X[3 * a] = C.x.x;
      m.X[3 * a + 1] = C.x.y;
      m.X[3 * a + 2] = C.x.z;
      for (int i = 0; i < 10; ++i) m.Q[a].q[i] = m.Q[a].q[i] + m.Q[b].q[i];
      m.valive[b] = 0;
      C.applied = true;
      for (const int32_t* p = I.begin(a); p != I.end(a); ++p)
        if (m.falive[*p]) C.owned.push_back(*p);
      for (auto& bf : C.bfaces)
        if (m.falive[bf.first]) C.owned.push_back(bf.first);
      std::sort(C.owned.begin(), C.owned.end());
      for (int f : C.owned) owner[f] = static_cast<int32_t>(ci);
    }
    T.mark(5);
    // undo loop
    int rounds = 0;
    while (true) {
      std::vector<uint8_t> query(m.nf, 0);
      bool any = false;
      for (auto& C : cols)
        if (C.applied)
          for (int f : C.owned) {
            query[f] = 1;
            any = true;
          }
      if (!any) break;
      const auto pairs = detect_pairs(m.X.data(), m.F.data(), m.nf, m.falive.data(), query.data());
      T.mark(6);
      if (pairs.empty()) break;
      ++rounds;
      std::vector<uint8_t> revert(cols.size(), 0);
      for (auto& pr : pairs) {
        for (int f : {pr.first, pr.second}) {
          const int o = owner[f];
          if (o >= 0 && cols[o].applied) revert[o] = 1;
        }
      }
      for (size_t ci = 0; ci < cols.size(); ++ci) {
        if (!revert[ci]) continue;
        Collapse& C = cols[ci];
        for (auto& bf : C.bfaces) {
          if (!m.falive[bf.first]) m.alive_faces++;
          m.falive[bf.first] = 1;
          for (int k = 0; k < 3; ++k) m.F[3 * bf.first + k] = bf.second[k];
        }
        m.X[3 * C.a] = C.old_x.x;
        m.X[3 * C.a + 1] = C.old_x.y;
        m.X[3 * C.a + 2] = C.old_x.z;
        m.Q[C.a] = C.old_q;
        m.valive[C.b] = 1;
        C.applied = false;
        for (int f : C.owned) owner[f] = -1;
        new_invalid.insert({C.a, C.b});
        S.undone++;
      }
    }
    T.mark(7);
    S.undo_hist[std::min(rounds, 7)]++;
    S.max_undo_rounds = std::max<int64_t>(S.max_undo_rounds, rounds);
    int64_t succ = 0;
    for (auto& C : cols) succ += C.applied;
    S.collapses += succ;
    if (per_iter_collapses) per_iter_collapses->push_back(succ);
    if (rec) {
      for (size_t ci = 0; ci < cols.size(); ++ci)
        if (cols[ci].applied) tr->applied.push_back(sel[ci]);
      tr->rounds = rounds;
      tr->X = m.X;
      tr->F = m.F;
      tr->falive = m.falive;
    }
    if (succ > 0) {
      invalid = new_invalid;
      retain = 0;
      zero_run = 0;
    } else {
      ++zero_run;
      ++retain;
      if (retain >= P.tolerance) {
        invalid = new_invalid;
        retain = 0;
      } else {
        invalid.insert(new_invalid.begin(), new_invalid.end());
      }
    }
    if (rec) return;
  }
}

}  // namespace simp
}  // namespace orc

using namespace orc;
using namespace orc::simp;

namespace {
std::vector<double> g_v;
std::vector<int32_t> g_f;
std::vector<int64_t> g_iters;
}  // namespace

extern "C" {

// simplify_to.  stats_out (int64[17]):
//  [iterations, collapses, undone, link_failures, max_undo_rounds, error, nv_out, nf_out,
//   undo_hist[0..7], face_iterations]
int orc_simplify(const double* v, int64_t nv, const int32_t* f, int64_t nf, int64_t target,
                 double we, double ws, int tolerance, int64_t* stats_out) {
  Mesh m;
  m.nv = nv;
  m.nf = nf;
  m.X.assign(v, v + 3 * nv);
  m.F.assign(f, f + 3 * nf);
  m.valive.assign(nv, 1);
  m.falive.assign(nf, 1);
  m.alive_faces = nf;
  Params P{we, ws, tolerance, 10};
  Stats S;
  g_iters.clear();
  run(m, target, P, S, &g_iters);
  // compact (mesh.cpp:278-292): alive vertices with >=1 alive face, order preserving
  std::vector<int64_t> used(nv, 0);
  for (int64_t i = 0; i < nf; ++i)
    if (m.falive[i])
      for (int k = 0; k < 3; ++k) used[m.F[3 * i + k]] = 1;
  std::vector<int32_t> remap(nv, -1);
  g_v.clear();
  g_f.clear();
  for (int64_t i = 0; i < nv; ++i)
    if (m.valive[i] && used[i]) {
      remap[i] = static_cast<int32_t>(g_v.size() / 3);
      for (int k = 0; k < 3; ++k) g_v.push_back(m.X[3 * i + k]);
    }
  for (int64_t i = 0; i < nf; ++i)
    if (m.falive[i])
      for (int k = 0; k < 3; ++k) g_f.push_back(remap[m.F[3 * i + k]]);
  stats_out[0] = S.iterations;
  stats_out[1] = S.collapses;
  stats_out[2] = S.undone;
  stats_out[3] = S.link_failures;
  stats_out[4] = S.max_undo_rounds;
  stats_out[5] = S.error;
  stats_out[6] = static_cast<int64_t>(g_v.size() / 3);
  stats_out[7] = static_cast<int64_t>(g_f.size() / 3);
  for (int k = 0; k < 8; ++k) stats_out[8 + k] = S.undo_hist[k];
  stats_out[16] = S.face_iterations;
  return S.error ? -1 : 0;
}

void orc_simplify_fetch(double* v, int32_t* f, int64_t* per_iter) {
  if (v) std::memcpy(v, g_v.data(), g_v.size() * 8);
  if (f) std::memcpy(f, g_f.data(), g_f.size() * 4);
  if (per_iter) std::memcpy(per_iter, g_iters.data(), g_iters.size() * 8);
}

// Step-level record of iteration `iter` of simplify_to (granular parity of edge_cost, pack_cost,
// propagate_and_mark, collapse_batch, undo_loop).  sizes_out (int64[6]): ne, nf, nmarked,
// napplied, rounds, nv.  Fetch with orc_trace_fetch.
namespace {
Trace g_trace;
}
int orc_simplify_trace(const double* v, int64_t nv, const int32_t* f, int64_t nf, int64_t target, double we,
                       double ws, int tolerance, int64_t iter, int64_t* sizes_out) {
  Mesh m;
  m.nv = nv;
  m.nf = nf;
  m.X.assign(v, v + 3 * nv);
  m.F.assign(f, f + 3 * nf);
  m.valive.assign(nv, 1);
  m.falive.assign(nf, 1);
  m.alive_faces = nf;
  Params P{we, ws, tolerance, 10};
  Stats S;
  g_trace = Trace();
  g_trace.iter = iter;
  run(m, target, P, S, nullptr, &g_trace);
  sizes_out[0] = static_cast<int64_t>(g_trace.edges.size());
  sizes_out[1] = nf;
  sizes_out[2] = static_cast<int64_t>(g_trace.marked.size());
  sizes_out[3] = static_cast<int64_t>(g_trace.applied.size());
  sizes_out[4] = g_trace.rounds;
  sizes_out[5] = nv;
  return S.error ? -1 : (g_trace.X.empty() ? 1 : 0);
}

void orc_trace_fetch(int32_t* edges, uint64_t* keys, double* place, uint64_t* face_keys, int64_t* marked,
                     uint8_t* link_ok, int64_t* applied, double* X, int32_t* F, uint8_t* falive) {
  const Trace& t = g_trace;
  for (size_t e = 0; e < t.edges.size(); ++e) {
    edges[2 * e] = t.edges[e].first;
    edges[2 * e + 1] = t.edges[e].second;
  }
  std::memcpy(keys, t.keys.data(), t.keys.size() * 8);
  std::memcpy(place, t.place.data(), t.place.size() * 8);
  std::memcpy(face_keys, t.face_keys.data(), t.face_keys.size() * 8);
  std::memcpy(marked, t.marked.data(), t.marked.size() * 8);
  std::memcpy(link_ok, t.link_ok.data(), t.link_ok.size());
  std::memcpy(applied, t.applied.data(), t.applied.size() * 8);
  std::memcpy(X, t.X.data(), t.X.size() * 8);
  std::memcpy(F, t.F.data(), t.F.size() * 4);
  std::memcpy(falive, t.falive.data(), t.falive.size());
}

// Quadric per vertex, gathered in ascending face id: double[10 nv]
void orc_quadrics(const double* v, int64_t nv, const int32_t* f, int64_t nf, double* out) {
  Mesh m;
  m.nv = nv;
  m.nf = nf;
  m.X.assign(v, v + 3 * nv);
  m.F.assign(f, f + 3 * nf);
  std::fill(out, out + 10 * nv, 0.0);
  for (int64_t i = 0; i < nf; ++i) {
    double fq[10];
    face_quadric(m, static_cast<int>(i), fq);
    for (int k = 0; k < 3; ++k) {
      double* q = out + 10 * m.F[3 * i + k];
      for (int j = 0; j < 10; ++j) q[j] = q[j] + fq[j];
    }
  }
}

// edge_cost of explicit edges under the mesh's initial quadrics
void orc_edge_cost(const double* v, int64_t nv, const int32_t* f, int64_t nf, const int32_t* edges, int64_t ne,
                   double we, double ws, double* cost, double* place) {
  Mesh m;
  m.nv = nv;
  m.nf = nf;
  m.X.assign(v, v + 3 * nv);
  m.F.assign(f, f + 3 * nf);
  m.falive.assign(nf, 1);
  m.Q.assign(nv, Quadric{});
  orc_quadrics(v, nv, f, nf, reinterpret_cast<double*>(m.Q.data()));
  const Incidence I = build_incidence(m);
  const Params P{we, ws, 4, 10};
  for (int64_t i = 0; i < ne; ++i) {
    const CostOut c = edge_cost(m, I, edges[2 * i], edges[2 * i + 1], P);
    cost[i] = c.cost;
    place[3 * i] = c.x.x;
    place[3 * i + 1] = c.x.y;
    place[3 * i + 2] = c.x.z;
  }
}

// Link condition restatement over an arbitrary mesh (checked against the reference).
void orc_link_condition(const double* v, int64_t nv, const int32_t* f, int64_t nf,
                        const int32_t* edges, int64_t ne, int32_t* out) {
  Mesh m;
  m.nv = nv;
  m.nf = nf;
  m.X.assign(v, v + 3 * nv);
  m.F.assign(f, f + 3 * nf);
  m.falive.assign(nf, 1);
  const Incidence I = build_incidence(m);
  for (int64_t i = 0; i < ne; ++i) {
    const int a = edges[2 * i], b = edges[2 * i + 1];
    if (faces_of_edge_count(m, I, a, b) == 0) {
      out[i] = -1;
      continue;
    }
    out[i] = link_condition(m, I, a, b) ? 1 : 0;
  }
}

}  // extern "C"
