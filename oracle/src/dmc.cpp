// ORACLE (test infrastructure only) — stage 1b: Dual Marching Cubes with the paper's
// intersection corrections, restated from SPEC.md:238-334 and PAPER.md:85-114,716-772.
//
// Pinned semantics:
//   corners  c = x | y<<1 | z<<2;  case = OR over corners of (s_c < 0) << c  (sign(0)=+)
//   edges    e = 4*axis + sub; x-edges sub = y+2z, y-edges sub = x+2z, z-edges sub = x+2y
//   faces    f = 2*axis + side
//   patches  = cycles of the face pairing graph: on every face the sign-change edges are paired;
//              an ambiguous face (alternating corner signs) pairs the two edges around each
//              POSITIVE corner (negative corners connected) — resolution S; the flipped
//              resolution T pairs the edges around each NEGATIVE corner.
//   C16/C19 (Wenger) fix: a face f of a cell is "doubly covered" when both S-segments on f
//              belong to one patch.  If the two cells sharing an ambiguous face are BOTH doubly
//              covered on it, that face uses resolution T in both cells (otherwise four quads
//              would share one dual edge).
//   vertex   patch vertex = centroid (sum in ascending edge id, then /n) of the sigmoid-
//              smoothed crossings p0 + t'(p1-p0), t = -f0/(f1-f0), t' = 1/(1+exp(-beta(t-1/2)))
//   order    vertices: (active cell linear index, patch index by lowest edge id), then the extra
//              4-split vertices in quad order; quads: (lower grid-vertex linear index, axis)
//   quad     cells around an axis-a edge at offsets (b,c) = (-1,-1),(0,-1),(0,0),(-1,0),
//              b=(a+1)%3, c=(a+2)%3; reversed when the lower endpoint is the positive one so
//              the normal points from the negative toward the positive endpoint
//   split    concavity with l = previous, r = next quad vertex; one
//              concave diagonal -> split along it; both -> 4 triangles around the smoothed
//              crossing of the valid edge; none -> diagonal maximising the minimum angle
//              (compare the largest corner cosine; tie -> diagonal 0-2).
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "geom.hpp"
#include "par.hpp"

namespace orc {
namespace dmc {

struct Edge {
  int c0, c1, axis;
};

static Edge edge_of(int e) {
  const int axis = e / 4, sub = e % 4, u = sub & 1, w = sub >> 1;
  int c0;
  if (axis == 0) c0 = (u << 1) | (w << 2);
  else if (axis == 1) c0 = u | (w << 2);
  else c0 = u | (w << 1);
  return Edge{c0, c0 | (1 << axis), axis};
}

static int edge_index(int axis, int c0) {  // edge along `axis` whose lower corner is c0
  const int x = c0 & 1, y = (c0 >> 1) & 1, z = (c0 >> 2) & 1;
  if (axis == 0) return 0 + y + 2 * z;
  if (axis == 1) return 4 + x + 2 * z;
  return 8 + x + 2 * y;
}

// Face f = 2*axis+side: its 4 corners in cyclic order and the edge between consecutive ones.
struct Face {
  int corner[4];
  int edge[4];  // edge[i] joins corner[i] and corner[(i+1)%4]
};

static Face face_of(int f) {
  const int axis = f / 2, side = f % 2;
  const int b = (axis + 1) % 3, c = (axis + 2) % 3;
  Face F;
  const int cyc[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
  for (int i = 0; i < 4; ++i)
    F.corner[i] = (side << axis) | (cyc[i][0] << b) | (cyc[i][1] << c);
  for (int i = 0; i < 4; ++i) {
    const int p = F.corner[i], q = F.corner[(i + 1) % 4];
    const int diff = p ^ q;
    const int ax = diff == 1 ? 0 : (diff == 2 ? 1 : 2);
    F.edge[i] = edge_index(ax, p & q);
  }
  return F;
}

struct Patches {
  int n = 0;
  uint16_t mask[4] = {0, 0, 0, 0};
  int8_t edge_patch[12];
};

static bool ambiguous(int cs, const Face& F) {
  const int s0 = (cs >> F.corner[0]) & 1, s1 = (cs >> F.corner[1]) & 1, s2 = (cs >> F.corner[2]) & 1,
            s3 = (cs >> F.corner[3]) & 1;
  return s0 == s2 && s1 == s3 && s0 != s1;
}

// Patches of case `cs` with resolution T on the faces of `flip`.
static Patches make_patches(int cs, int flip) {
  int partner[12][2];
  int deg[12] = {0};
  for (int f = 0; f < 6; ++f) {
    const Face F = face_of(f);
    bool cross[4];
    int ncross = 0;
    for (int i = 0; i < 4; ++i) {
      cross[i] = ((cs >> F.corner[i]) & 1) != ((cs >> F.corner[(i + 1) % 4]) & 1);
      ncross += cross[i];
    }
    auto link = [&](int e1, int e2) {
      partner[e1][deg[e1]++] = e2;
      partner[e2][deg[e2]++] = e1;
    };
    if (ncross == 2) {
      int a = -1, b = -1;
      for (int i = 0; i < 4; ++i)
        if (cross[i]) (a < 0 ? a : b) = F.edge[i];
      link(a, b);
    } else if (ncross == 4) {
      // corner i is between edge[i-1] and edge[i]
      const bool use_t = (flip >> f) & 1;
      for (int i = 0; i < 4; ++i) {
        const bool neg = (cs >> F.corner[i]) & 1;
        if (neg == use_t) link(F.edge[(i + 3) % 4], F.edge[i]);
      }
    }
  }
  Patches P;
  for (int e = 0; e < 12; ++e) P.edge_patch[e] = -1;
  for (int e = 0; e < 12; ++e) {
    if (deg[e] == 0 || P.edge_patch[e] >= 0) continue;
    // walk the cycle starting at e (lowest unassigned edge => patches ordered by lowest edge)
    uint16_t m = 0;
    int prev = -1, cur = e;
    while (true) {
      m |= static_cast<uint16_t>(1u << cur);
      P.edge_patch[cur] = static_cast<int8_t>(P.n);
      const int nxt = partner[cur][0] != prev ? partner[cur][0] : partner[cur][1];
      prev = cur;
      cur = nxt;
      if (cur == e) break;
    }
    P.mask[P.n++] = m;
  }
  return P;
}

// Faces on which both S-segments of an ambiguous face lie in one patch.
static int doubly_covered(int cs) {
  const Patches P = make_patches(cs, 0);
  int m = 0;
  for (int f = 0; f < 6; ++f) {
    const Face F = face_of(f);
    if (!ambiguous(cs, F)) continue;
    if (P.edge_patch[F.edge[0]] == P.edge_patch[F.edge[1]] &&
        P.edge_patch[F.edge[1]] == P.edge_patch[F.edge[2]] &&
        P.edge_patch[F.edge[2]] == P.edge_patch[F.edge[3]])
      m |= 1 << f;
  }
  return m;
}

struct Table {
  Patches base[256];
  int dc[256];
  Table() {
    for (int cs = 0; cs < 256; ++cs) {
      base[cs] = make_patches(cs, 0);
      dc[cs] = doubly_covered(cs);
    }
  }
};

static const Table& table() {
  static Table t;
  return t;
}

}  // namespace dmc
}  // namespace orc

using namespace orc;
using namespace orc::dmc;

namespace {

struct Grid {
  const float* s;
  int R;
  int64_t n1;
  int64_t zb;  // global z of the first resident plane (z-slab restatement)
  float at(int64_t x, int64_t y, int64_t z) const { return s[x + n1 * (y + n1 * (z - zb))]; }
  int case_of(int64_t x, int64_t y, int64_t z) const {
    int cs = 0;
    for (int c = 0; c < 8; ++c)
      if (at(x + (c & 1), y + ((c >> 1) & 1), z + ((c >> 2) & 1)) < 0.0f) cs |= 1 << c;
    return cs;
  }
};

// the effective flip mask of a cell (C16/C19 neighbour rule)
int flip_mask(const Grid& g, int64_t x, int64_t y, int64_t z, int cs) {
  const int dc = table().dc[cs];
  if (!dc) return 0;
  int flip = 0;
  for (int f = 0; f < 6; ++f) {
    if (!((dc >> f) & 1)) continue;
    const int axis = f / 2, side = f % 2;
    int64_t n[3] = {x, y, z};
    n[axis] += side ? 1 : -1;
    if (n[axis] < 0 || n[axis] >= g.R) continue;
    const int ncs = g.case_of(n[0], n[1], n[2]);
    const int nf = 2 * axis + (1 - side);
    if ((table().dc[ncs] >> nf) & 1) flip |= 1 << f;
  }
  return flip;
}

V3 grid_point(int64_t x, int64_t y, int64_t z, int R) {
  return v3(static_cast<double>(x) / R, static_cast<double>(y) / R, static_cast<double>(z) / R);
}

V3 crossing(V3 p0, V3 p1, float f0, float f1, double beta) {
  const double t = -static_cast<double>(f0) / (static_cast<double>(f1) - static_cast<double>(f0));
  const double ts = sigmoid_t(t, beta);
  return v3(p0.x + ts * (p1.x - p0.x), p0.y + ts * (p1.y - p0.y), p0.z + ts * (p1.z - p0.z));
}

struct DmcOut {
  std::vector<int64_t> cells;
  std::vector<uint8_t> cases;
  std::vector<uint8_t> flips;
  std::vector<int64_t> vbase;
  std::vector<double> verts;
  std::vector<int32_t> faces;
  int64_t nquads = 0;
  int64_t nsplit4 = 0;
  // build_quads view: patch-vertex ids (4 per quad), lower vertex * 3 + axis, samples, split
  std::vector<int32_t> quads;
  std::vector<int64_t> qedge;
  std::vector<float> qf;
  std::vector<uint8_t> qsplit;
  int64_t nvp_own = 0;  // patch vertices of the own layers (slab mode)
  int64_t n_extra = 0;
};

// Whole grid: pz0 = 0, own layers [0, R).  Slab: the resident planes start at pz0; cells of layers
// [own_z0, own_z1) emit quads, the layer below only provides vertex ids; the output drops the
// vertices below the own layers and shifts every face index by their count.
void run_dmc(const float* sdf, int R, double beta, DmcOut& out, int64_t pz0 = 0, int64_t own_z0 = 0,
             int64_t own_z1 = -1) {
  if (own_z1 < 0) own_z1 = R;
  Grid g{sdf, R, static_cast<int64_t>(R) + 1, pz0};
  const int64_t cz0 = own_z0 > 0 ? own_z0 - 1 : 0;
  const int64_t cbeg = static_cast<int64_t>(R) * R * cz0;
  const int64_t ncell = static_cast<int64_t>(R) * R * own_z1;
  // classify (dense scan, per-thread chunks then ordered concatenation)
  const int64_t chunk = 1 << 16;
  const int64_t nchunks = (ncell - cbeg + chunk - 1) / chunk;
  std::vector<std::vector<int64_t>> part(nchunks);
  parallel_for(nchunks, [&](int64_t ci) {
    for (int64_t c = cbeg + ci * chunk; c < std::min(ncell, cbeg + (ci + 1) * chunk); ++c) {
      const int64_t x = c % R, y = (c / R) % R, z = c / (static_cast<int64_t>(R) * R);
      const int cs = g.case_of(x, y, z);
      if (cs != 0 && cs != 255) part[ci].push_back(c);
    }
  }, 1);
  for (auto& p : part) out.cells.insert(out.cells.end(), p.begin(), p.end());
  const int64_t na = static_cast<int64_t>(out.cells.size());
  out.cases.resize(na);
  out.flips.resize(na);
  out.vbase.resize(na + 1);
  std::vector<Patches> patches(na);
  parallel_for(na, [&](int64_t i) {
    const int64_t c = out.cells[i];
    const int64_t x = c % R, y = (c / R) % R, z = c / (static_cast<int64_t>(R) * R);
    const int cs = g.case_of(x, y, z);
    const int fl = flip_mask(g, x, y, z, cs);
    out.cases[i] = static_cast<uint8_t>(cs);
    out.flips[i] = static_cast<uint8_t>(fl);
    patches[i] = fl ? make_patches(cs, fl) : table().base[cs];
  });
  out.vbase[0] = 0;
  for (int64_t i = 0; i < na; ++i) out.vbase[i + 1] = out.vbase[i] + patches[i].n;
  const int64_t nv_patch = out.vbase[na];
  out.verts.resize(3 * nv_patch);
  parallel_for(na, [&](int64_t i) {
    const int64_t c = out.cells[i];
    const int64_t x = c % R, y = (c / R) % R, z = c / (static_cast<int64_t>(R) * R);
    const Patches& P = patches[i];
    for (int p = 0; p < P.n; ++p) {
      V3 sum = v3(0, 0, 0);
      int cnt = 0;
      for (int e = 0; e < 12; ++e) {
        if (!((P.mask[p] >> e) & 1)) continue;
        const Edge E = edge_of(e);
        const int64_t x0 = x + (E.c0 & 1), y0 = y + ((E.c0 >> 1) & 1), z0 = z + ((E.c0 >> 2) & 1);
        const int64_t x1 = x + (E.c1 & 1), y1 = y + ((E.c1 >> 1) & 1), z1 = z + ((E.c1 >> 2) & 1);
        const V3 q = crossing(grid_point(x0, y0, z0, R), grid_point(x1, y1, z1, R), g.at(x0, y0, z0),
                              g.at(x1, y1, z1), beta);
        sum = v3(sum.x + q.x, sum.y + q.y, sum.z + q.z);
        ++cnt;
      }
      const int64_t vi = out.vbase[i] + p;
      out.verts[3 * vi] = sum.x / cnt;
      out.verts[3 * vi + 1] = sum.y / cnt;
      out.verts[3 * vi + 2] = sum.z / cnt;
    }
  });
  // vertex id of (cell, local edge)
  auto vid = [&](int64_t x, int64_t y, int64_t z, int e) -> int64_t {
    const int64_t c = x + static_cast<int64_t>(R) * (y + static_cast<int64_t>(R) * z);
    const auto it = std::lower_bound(out.cells.begin(), out.cells.end(), c);
    const int64_t i = it - out.cells.begin();
    return out.vbase[i] + patches[i].edge_patch[e];
  };
  // quads + triangulation, ordered by (cell, axis)
  struct QuadOut {
    int64_t q[4];
    int64_t edge;
    float f0, f1;
    int code;  // 1: diagonal 0-2, 2: diagonal 1-3, 3: four triangles
    int ntri;  // 2 or 4
    V3 extra;
    int32_t tri[4][3];  // local: 0..3 quad corners, 4 = extra vertex
  };
  std::vector<std::array<QuadOut, 3>> qo(na);
  std::vector<uint8_t> qmask(na, 0);
  parallel_for(na, [&](int64_t i) {
    const int64_t c = out.cells[i];
    const int64_t xyz[3] = {c % R, (c / R) % R, c / (static_cast<int64_t>(R) * R)};
    for (int a = 0; a < 3 && xyz[2] >= own_z0; ++a) {
      const int b = (a + 1) % 3, cc = (a + 2) % 3;
      if (xyz[b] < 1 || xyz[cc] < 1) continue;  // lower vertex coordinate must be in [1, R-1]
      int64_t up[3] = {xyz[0], xyz[1], xyz[2]};
      up[a] += 1;
      const float f0 = g.at(xyz[0], xyz[1], xyz[2]);
      const float f1 = g.at(up[0], up[1], up[2]);
      if ((f0 < 0.0f) == (f1 < 0.0f)) continue;
      const int offs[4][2] = {{-1, -1}, {0, -1}, {0, 0}, {-1, 0}};
      int64_t q[4];
      for (int k = 0; k < 4; ++k) {
        int64_t cl[3] = {xyz[0], xyz[1], xyz[2]};
        cl[b] += offs[k][0];
        cl[cc] += offs[k][1];
        // local corner of the edge's lower end inside that cell
        int c0 = 0;
        if (offs[k][0] == -1) c0 |= 1 << b;
        if (offs[k][1] == -1) c0 |= 1 << cc;
        q[k] = vid(cl[0], cl[1], cl[2], edge_index(a, c0));
      }
      const bool lower_neg = f0 < 0.0f;
      if (!lower_neg) std::swap(q[1], q[3]);
      const V3 plo = grid_point(xyz[0], xyz[1], xyz[2], R), phi = grid_point(up[0], up[1], up[2], R);
      const V3 vp = lower_neg ? phi : plo, vn = lower_neg ? plo : phi;
      V3 P[4];
      for (int k = 0; k < 4; ++k) P[k] = v3(out.verts[3 * q[k]], out.verts[3 * q[k] + 1], out.verts[3 * q[k] + 2]);
      bool conc[4];
      for (int k = 0; k < 4; ++k) {
        const V3 L = P[(k + 3) % 4], Rr = P[(k + 1) % 4];
        const double t1 = dot(P[k] - vp, cross(L - vp, Rr - vp));
        const double t2 = dot(P[k] - vn, cross(L - vn, Rr - vn));
        conc[k] = t1 < 0.0 || t2 > 0.0;
      }
      const bool d02 = conc[0] || conc[2], d13 = conc[1] || conc[3];
      QuadOut Q;
      for (int k = 0; k < 4; ++k) Q.q[k] = q[k];
      Q.edge = (xyz[0] + (R + 1) * (xyz[1] + static_cast<int64_t>(R + 1) * xyz[2])) * 3 + a;
      Q.f0 = f0;
      Q.f1 = f1;
      auto set2 = [&](bool diag02) {
        Q.ntri = 2;
        Q.code = diag02 ? 1 : 2;
        if (diag02) {
          const int32_t t[2][3] = {{0, 1, 2}, {0, 2, 3}};
          std::memcpy(Q.tri, t, sizeof(t));
        } else {
          const int32_t t[2][3] = {{0, 1, 3}, {1, 2, 3}};
          std::memcpy(Q.tri, t, sizeof(t));
        }
      };
      if (d02 && !d13) set2(true);
      else if (d13 && !d02) set2(false);
      else if (d02 && d13) {
        Q.ntri = 4;
        Q.code = 3;
        Q.extra = crossing(plo, phi, f0, f1, beta);
        const int32_t t[4][3] = {{0, 1, 4}, {1, 2, 4}, {2, 3, 4}, {3, 0, 4}};
        std::memcpy(Q.tri, t, sizeof(t));
      } else {
        auto maxcos = [&](int i0, int i1, int i2) {
          const V3 T[3] = {P[i0], P[i1], P[i2]};
          double m = -2.0;
          for (int k = 0; k < 3; ++k) {
            const V3 u = T[(k + 1) % 3] - T[k], w = T[(k + 2) % 3] - T[k];
            const double cs = dot(u, w) / std::sqrt(sqnorm(u) * sqnorm(w));
            if (cs > m) m = cs;
          }
          return m;
        };
        const double m02 = std::max(maxcos(0, 1, 2), maxcos(0, 2, 3));
        const double m13 = std::max(maxcos(0, 1, 3), maxcos(1, 2, 3));
        set2(m02 <= m13);
      }
      qo[i][a] = Q;
      qmask[i] |= static_cast<uint8_t>(1 << a);
    }
  });
  int64_t extra = 0;
  for (int64_t i = 0; i < na; ++i)
    for (int a = 0; a < 3; ++a)
      if ((qmask[i] >> a) & 1) {
        const QuadOut& Q = qo[i][a];
        ++out.nquads;
        for (int k = 0; k < 4; ++k) out.quads.push_back(static_cast<int32_t>(Q.q[k]));
        out.qedge.push_back(Q.edge);
        out.qf.push_back(Q.f0);
        out.qf.push_back(Q.f1);
        out.qsplit.push_back(static_cast<uint8_t>(Q.code));
        int64_t ids[5] = {Q.q[0], Q.q[1], Q.q[2], Q.q[3], -1};
        if (Q.ntri == 4) {
          ids[4] = nv_patch + extra++;
          out.verts.push_back(Q.extra.x);
          out.verts.push_back(Q.extra.y);
          out.verts.push_back(Q.extra.z);
          ++out.nsplit4;
        }
        for (int t = 0; t < Q.ntri; ++t)
          for (int k = 0; k < 3; ++k) out.faces.push_back(static_cast<int32_t>(ids[Q.tri[t][k]]));
      }
  // drop the lending layer's vertices (slab mode); whole grid: shift = 0
  const int64_t cown = static_cast<int64_t>(R) * R * own_z0;
  const int64_t i0 = std::lower_bound(out.cells.begin(), out.cells.end(), cown) - out.cells.begin();
  const int64_t shift = out.vbase[i0];
  out.verts.erase(out.verts.begin(), out.verts.begin() + 3 * shift);
  for (auto& x : out.faces) x = static_cast<int32_t>(x - shift);
  out.nvp_own = nv_patch - shift;
  out.n_extra = extra;
}

}  // namespace

extern "C" {

// Table views for the golden snapshot / invariants.
// out: per case  [n, mask0..mask3, dc]  (6 ints)
void orc_dmc_table(int32_t* out) {
  for (int cs = 0; cs < 256; ++cs) {
    const Patches& P = table().base[cs];
    out[6 * cs] = P.n;
    for (int k = 0; k < 4; ++k) out[6 * cs + 1 + k] = P.mask[k];
    out[6 * cs + 5] = table().dc[cs];
  }
}

// patches for (case, flip mask): out = [n, mask0..mask3]
void orc_dmc_patches(int cs, int flip, int32_t* out) {
  const Patches P = make_patches(cs, flip);
  out[0] = P.n;
  for (int k = 0; k < 4; ++k) out[1 + k] = P.mask[k];
}

static DmcOut g_last;

// extract(grid, beta).  Result kept in a static; fetch with orc_dmc_fetch.
// sizes = {n_active, n_verts, n_faces, n_quads, n_split4}
void orc_dmc_extract(const float* sdf, int R, double beta, int64_t* sizes) {
  g_last = DmcOut();
  run_dmc(sdf, R, beta, g_last);
  sizes[0] = static_cast<int64_t>(g_last.cells.size());
  sizes[1] = static_cast<int64_t>(g_last.verts.size() / 3);
  sizes[2] = static_cast<int64_t>(g_last.faces.size() / 3);
  sizes[3] = g_last.nquads;
  sizes[4] = g_last.nsplit4;
}

// slab-local extract: planes [pz0, pz1) resident; sizes as orc_dmc_extract plus
// {nvp_own, n_extra}
void orc_dmc_extract_slab(const float* planes, int R, int pz0, int pz1, int own_z0, int own_z1, double beta,
                          int64_t* sizes) {
  (void)pz1;
  g_last = DmcOut();
  run_dmc(planes, R, beta, g_last, pz0, own_z0, own_z1);
  sizes[0] = static_cast<int64_t>(g_last.cells.size());
  sizes[1] = static_cast<int64_t>(g_last.verts.size() / 3);
  sizes[2] = static_cast<int64_t>(g_last.faces.size() / 3);
  sizes[3] = g_last.nquads;
  sizes[4] = g_last.nsplit4;
  sizes[5] = g_last.nvp_own;
  sizes[6] = g_last.n_extra;
}

// build_patches / build_quads views of the last whole-grid extract: sizes {n_patch_vertices,
// n_quads}; vbase int64[n_active], quads int32[4n], qedge int64[n], qf float[2n], qsplit uint8[n]
void orc_dmc_stages(int64_t* sizes, int64_t* vbase, int32_t* quads, int64_t* qedge, float* qf, uint8_t* qsplit) {
  sizes[0] = g_last.nvp_own;
  sizes[1] = g_last.nquads;
  if (vbase) std::memcpy(vbase, g_last.vbase.data(), (g_last.vbase.size() - 1) * 8);
  if (quads) std::memcpy(quads, g_last.quads.data(), g_last.quads.size() * 4);
  if (qedge) std::memcpy(qedge, g_last.qedge.data(), g_last.qedge.size() * 8);
  if (qf) std::memcpy(qf, g_last.qf.data(), g_last.qf.size() * 4);
  if (qsplit) std::memcpy(qsplit, g_last.qsplit.data(), g_last.qsplit.size());
}

void orc_dmc_fetch(int64_t* cells, uint8_t* cases, uint8_t* flips, double* verts, int32_t* faces) {
  if (cells) std::memcpy(cells, g_last.cells.data(), g_last.cells.size() * 8);
  if (cases) std::memcpy(cases, g_last.cases.data(), g_last.cases.size());
  if (flips) std::memcpy(flips, g_last.flips.data(), g_last.flips.size());
  if (verts) std::memcpy(verts, g_last.verts.data(), g_last.verts.size() * 8);
  if (faces) std::memcpy(faces, g_last.faces.data(), g_last.faces.size() * 4);
}

}  // extern "C"
