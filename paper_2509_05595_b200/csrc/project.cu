// project.cu — stage 3, safe projection (SPEC.md safe_project; §6, Algorithm 2,
// Appendix 2.2), on the GPU.
//
// B(X) = k_dis (E_S2M + E_M2S) + k_elas E_elas + k_bend E_bend + k_bar Σ_c b(d_c), minimised by
// projected Newton:
//   * every term is a stencil (S2M: 1 vertex, M2S/elastic: a triangle, bending: a hinge, barrier:
//     a point-triangle or edge-edge contact); one thread per stencil evaluates the closed form on
//     second-order forward-mode jets (ad.cuh), so gradients and Hessian blocks are exact, and
//     projects its block to SPD by a Jacobi eigen-clamp (eigenvalues < 1e-10 -> 1e-10);
//   * accumulation is deterministic: stencils write per-slot contributions, and a per-vertex CSR
//     of slots (sorted once per assembly) sums them in a fixed order — gradient, diagonal and
//     every CG product;
//   * the Newton direction solves H p = -g by Jacobi-preconditioned CG (|r| <= 1e-3 |g|, <= 1000
//     iterations);
//   * the step is bounded by additive CCD over point-triangle / edge-edge pairs from a sweep of
//     the d̂-inflated swept boxes (conservative advancement: the pair's distance can shrink at
//     most by l_p per unit step, l_p from the centred displacements), times 0.9; a backtracking
//     line search then halves it until B decreases and the exact self-intersection check of
//     the new mesh is empty (<= 64 halvings);
//   * nearest targets (S2M: LBVH nearest point on M_in per vertex; M2S: nearest face of S per
//     sample, with its distance class frozen) refresh every `refresh` iterations.
// Contacts sharing a vertex are excluded from the barrier (SPEC DESIGN DECISIONS); adjacent
// safety is carried by the exact post-check.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "ad.cuh"
#include "common.cuh"
#include "kernels.cuh"

namespace pcu {
namespace {

using ad::J2;
using ad::V;

constexpr int kMaxN = 12;     // stencil coordinates (4 vertices)
constexpr int kBlk = 144;     // block stride (12 x 12)
enum Term : int { kS2M = 0, kM2S = 1, kElas = 2, kBend = 3, kPT = 4, kEE = 5 };

struct Stencil {
  int term;
  int nv;       // vertices (1, 3 or 4)
  int v[4];     // vertex ids
  int param;    // index into the term's parameter arrays
  int cls;      // distance class (M2S, contacts)
};

struct Params {
  double kdis, kelas, kbend, kbar, dhat, elas_tau;
  int elas_power;
};

struct TermData {
  const double* X0;
  const double* s0;       // per-vertex rest area (S2M weight)
  const double* ytgt;     // S2M targets (3n)
  const double* ys;       // M2S samples (3m)
  double m2s_w;           // A(M_in) / m
  const double* dminv;    // elastic: rest Dm^-1 (4 per face)
  const double* a0;       // elastic: rest area per face
  const double* theta0;   // bending: rest dihedral per hinge
  const double* l0;       // bending: rest edge length per hinge
};

// ---------------------------------------------------------------- distance classes
// point-triangle: 0..2 point-vertex t_k, 3..5 point-edge (t0t1, t1t2, t2t0), 6 point-plane
__device__ int pt_class(const double* p, const double* t0, const double* t1, const double* t2) {
  double e0[3], e1[3], w[3], n[3];
  for (int k = 0; k < 3; ++k) {
    e0[k] = t1[k] - t0[k];
    e1[k] = t2[k] - t0[k];
    w[k] = p[k] - t0[k];
  }
  n[0] = e0[1] * e1[2] - e0[2] * e1[1];
  n[1] = e0[2] * e1[0] - e0[0] * e1[2];
  n[2] = e0[0] * e1[1] - e0[1] * e1[0];
  const double nn = n[0] * n[0] + n[1] * n[1] + n[2] * n[2];
  if (nn > 0.0) {
    const double d00 = e0[0] * e0[0] + e0[1] * e0[1] + e0[2] * e0[2];
    const double d01 = e0[0] * e1[0] + e0[1] * e1[1] + e0[2] * e1[2];
    const double d11 = e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2];
    const double d20 = w[0] * e0[0] + w[1] * e0[1] + w[2] * e0[2];
    const double d21 = w[0] * e1[0] + w[1] * e1[1] + w[2] * e1[2];
    const double den = d00 * d11 - d01 * d01;
    const double bv = (d11 * d20 - d01 * d21) / den, bw = (d00 * d21 - d01 * d20) / den;
    if (bv > 0.0 && bw > 0.0 && bv + bw < 1.0) return 6;
  }
  const double* T[3] = {t0, t1, t2};
  double best = 1e300;
  int cls = 0;
  for (int e = 0; e < 3; ++e) {
    const double* a = T[e];
    const double* b = T[(e + 1) % 3];
    double ab[3], ap[3];
    for (int k = 0; k < 3; ++k) {
      ab[k] = b[k] - a[k];
      ap[k] = p[k] - a[k];
    }
    const double den = ab[0] * ab[0] + ab[1] * ab[1] + ab[2] * ab[2];
    double t = den > 0.0 ? (ap[0] * ab[0] + ap[1] * ab[1] + ap[2] * ab[2]) / den : 0.0;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    double d2 = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double q = ap[k] - t * ab[k];
      d2 += q * q;
    }
    if (d2 < best) {
      best = d2;
      cls = t <= 0.0 ? e : (t >= 1.0 ? (e + 1) % 3 : 3 + e);
    }
  }
  return cls;
}

// edge-edge: 0..3 point-point (a0b0, a0b1, a1b0, a1b1), 4..7 point-edge (a0-b, a1-b, b0-a,
// b1-a), 8 line-line
__device__ int ee_class(const double* a0, const double* a1, const double* b0, const double* b1) {
  double u[3], v[3], w[3];
  for (int k = 0; k < 3; ++k) {
    u[k] = a1[k] - a0[k];
    v[k] = b1[k] - b0[k];
    w[k] = a0[k] - b0[k];
  }
  const double a = u[0] * u[0] + u[1] * u[1] + u[2] * u[2], b = u[0] * v[0] + u[1] * v[1] + u[2] * v[2];
  const double c = v[0] * v[0] + v[1] * v[1] + v[2] * v[2], d = u[0] * w[0] + u[1] * w[1] + u[2] * w[2];
  const double e = v[0] * w[0] + v[1] * w[1] + v[2] * w[2];
  const double D = a * c - b * b;
  // candidates: interior-interior when not (near) parallel, else the point-edge / point-point
  if (D > 1e-12 * a * c) {
    const double s = (b * e - c * d) / D, t = (a * e - b * d) / D;
    if (s > 0.0 && s < 1.0 && t > 0.0 && t < 1.0) return 8;
  }
  // best of the four endpoint-to-segment distances
  const double* P[4] = {a0, a1, b0, b1};
  const double* S0[4] = {b0, b0, a0, a0};
  const double* S1[4] = {b1, b1, a1, a1};
  double best = 1e300;
  int cls = 0;
  for (int q = 0; q < 4; ++q) {
    double sv[3], sp[3];
    for (int k = 0; k < 3; ++k) {
      sv[k] = S1[q][k] - S0[q][k];
      sp[k] = P[q][k] - S0[q][k];
    }
    const double den = sv[0] * sv[0] + sv[1] * sv[1] + sv[2] * sv[2];
    double t = den > 0.0 ? (sp[0] * sv[0] + sp[1] * sv[1] + sp[2] * sv[2]) / den : 0.0;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    double d2 = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double r = sp[k] - t * sv[k];
      d2 += r * r;
    }
    if (d2 < best) {
      best = d2;
      if (t > 0.0 && t < 1.0) cls = 4 + q;
      else if (q < 2) cls = (q == 0 ? 0 : 2) + (t >= 1.0 ? 1 : 0);   // a_q with b0/b1
      else cls = (t >= 1.0 ? 2 : 0) + (q == 2 ? 0 : 1);              // a0/a1 with b_q
    }
  }
  return cls;
}

template <class T>
__device__ T d2_pp(const V<T>& a, const V<T>& b) {
  const V<T> d = a - b;
  return ad::dot(d, d);
}
template <class T>
__device__ T d2_pe(const V<T>& p, const V<T>& a, const V<T>& b) {
  const V<T> c = ad::cross(a - p, b - p), e = b - a;
  return ad::dot(c, c) / ad::dot(e, e);
}
template <class T>
__device__ T d2_plane(const V<T>& p, const V<T>& t0, const V<T>& t1, const V<T>& t2) {
  const V<T> n = ad::cross(t1 - t0, t2 - t0);
  const T s = ad::dot(p - t0, n);
  return s * s / ad::dot(n, n);
}
template <class T>
__device__ T d2_pt_class(const V<T>& p, const V<T>* t, int cls) {
  if (cls < 3) return d2_pp(p, t[cls]);
  if (cls < 6) return d2_pe(p, t[cls - 3], t[(cls - 2) % 3]);
  return d2_plane(p, t[0], t[1], t[2]);
}
template <class T>
__device__ T d2_ee_class(const V<T>& a0, const V<T>& a1, const V<T>& b0, const V<T>& b1, int cls) {
  switch (cls) {
    case 0: return d2_pp(a0, b0);
    case 1: return d2_pp(a0, b1);
    case 2: return d2_pp(a1, b0);
    case 3: return d2_pp(a1, b1);
    case 4: return d2_pe(a0, b0, b1);
    case 5: return d2_pe(a1, b0, b1);
    case 6: return d2_pe(b0, a0, a1);
    case 7: return d2_pe(b1, a0, a1);
    default: {
      const V<T> n = ad::cross(a1 - a0, b1 - b0);
      const T s = ad::dot(b0 - a0, n);
      return s * s / ad::dot(n, n);
    }
  }
}

// barrier b(d) = -(d - d̂)^2 ln(d / d̂) for 0 < d < d̂ (PAPER.md Eq. barrier)
template <class T>
__device__ T barrier_of_d2(const T& d2, double dhat) {
  const T d = ad::sqrt(d2);
  const T u = d - dhat;
  return -1.0 * (u * u) * ad::log(d / dhat);
}

// ------------------------------------------------------------------------- the terms
// G selects the terms compiled into an instantiation (0: all, for values; 1: the 1-vertex term;
// 3: the triangle terms; 4: the 4-vertex terms) so each jet size only carries its own stencils
template <class T, int G>
__device__ T term_value(const Stencil& S, const V<T>* x, const TermData& D, const Params& P) {
  if constexpr (G == 0 || G == 1) {
    if (S.term == kS2M) {
      const V<T> y{T(D.ytgt[3 * S.v[0]]), T(D.ytgt[3 * S.v[0] + 1]), T(D.ytgt[3 * S.v[0] + 2])};
      return (P.kdis * D.s0[S.v[0]]) * d2_pp(x[0], y);
    }
  }
  if constexpr (G == 0 || G == 3) {
    if (S.term == kM2S) {
      const V<T> y{T(D.ys[3 * S.param]), T(D.ys[3 * S.param + 1]), T(D.ys[3 * S.param + 2])};
      return (P.kdis * D.m2s_w) * d2_pt_class(y, x, S.cls);
    }
    if (S.term == kElas) {
      // F = Ds Dm^-1 (3x2); C = F^T F; E = 1/4 A0 |C - I|_F^p
      const double* mi = D.dminv + 4 * S.param;
      const V<T> e1 = x[1] - x[0], e2 = x[2] - x[0];
      const V<T> f1 = ad::scale(T(mi[0]), e1) + ad::scale(T(mi[2]), e2);  // column 1 of F
      const V<T> f2 = ad::scale(T(mi[1]), e1) + ad::scale(T(mi[3]), e2);  // column 2
      const T c11 = ad::dot(f1, f1) - 1.0, c22 = ad::dot(f2, f2) - 1.0, c12 = ad::dot(f1, f2);
      const T s = c11 * c11 + c22 * c22 + 2.0 * (c12 * c12);
      const double w = 0.25 * D.a0[S.param] * P.kelas;
      if (P.elas_power == 2) return w * s;
      // |.|_F (power 1, as printed): below tau, sqrt(s) is replaced by the C1 blend
      // s (3 tau - s) / (2 tau^1.5) (value and slope match at tau, value 0 at the rest state)
      const double tau = P.elas_tau;
      if (ad::value(s) < tau) return w * (s * (3.0 * tau - s)) * (0.5 / (tau * ::sqrt(tau)));
      return w * ad::sqrt(s);
    }
  }
  if constexpr (G == 0 || G == 4) {
    if (S.term == kBend) {
      // hinge (i, j | k, l): faces (i, j, k) and (j, i, l); signed dihedral, flat = 0
      const V<T> e = x[1] - x[0];
      const V<T> n0 = ad::cross(e, x[2] - x[0]), n1 = ad::cross(x[3] - x[0], e);
      const T el = ad::sqrt(ad::dot(e, e));
      const T sn = ad::dot(ad::cross(n0, n1), e) / el, cs = ad::dot(n0, n1);
      const T th = ad::atan2(sn, cs);
      const T dth = th - D.theta0[S.param];
      return (0.5 * P.kbend * D.l0[S.param]) * (dth * dth);
    }
    if (S.term == kPT) return P.kbar * barrier_of_d2(d2_pt_class(x[0], x + 1, S.cls), P.dhat);
    if (S.term == kEE) return P.kbar * barrier_of_d2(d2_ee_class(x[0], x[1], x[2], x[3], S.cls), P.dhat);
  }
  return T(0.0);
}

// Jacobi eigen-decomposition of a symmetric n x n block (in place) and the SPD clamp
__device__ void spd_project(double* H, int n) {
  double A[kMaxN][kMaxN], Vv[kMaxN][kMaxN];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      A[i][j] = 0.5 * (H[i * n + j] + H[j * n + i]);
      Vv[i][j] = i == j ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += A[i][j] * A[i][j];
        if (i != j) off += A[i][j] * A[i][j];
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (A[p][q] == 0.0) continue;
        const double th = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + ::sqrt(th * th + 1.0));
        const double c = 1.0 / ::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = Vv[k][p], vkq = Vv[k][q];
          Vv[k][p] = c * vkp - s * vkq;
          Vv[k][q] = s * vkp + c * vkq;
        }
      }
  }
  double lam[kMaxN];
  for (int i = 0; i < n; ++i) lam[i] = A[i][i] < 1e-10 ? 1e-10 : A[i][i];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double sum = 0.0;
      for (int k = 0; k < n; ++k) sum += Vv[i][k] * lam[k] * Vv[j][k];
      H[i * n + j] = sum;
    }
}

// ----------------------------------------------------------------------- assembly
// value per stencil; with `deriv`, also the gradient into slots (3 per stencil vertex) and the
// projected Hessian block
template <int N>
__device__ void eval_stencil(const Stencil& S, const double* X, const TermData& D, const Params& P, double* val,
                             double* gslot, double* blk) {
  V<J2<N>> x[4];
  for (int a = 0; a < S.nv; ++a)
    x[a] = V<J2<N>>{J2<N>::var(3 * a, X[3 * S.v[a]]), J2<N>::var(3 * a + 1, X[3 * S.v[a] + 1]),
                    J2<N>::var(3 * a + 2, X[3 * S.v[a] + 2])};
  const J2<N> e = term_value<J2<N>, (N == 3 ? 1 : (N == 9 ? 3 : 4))>(S, x, D, P);
  *val = e.v;
  for (int i = 0; i < N; ++i) gslot[i] = e.g[i];
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) blk[i * N + j] = ad::hess(e, i, j);
  spd_project(blk, N);
}

__global__ void k_assemble(const Stencil* __restrict__ st, int64_t ns, const double* __restrict__ X, TermData D,
                           Params P, double* __restrict__ val, double* __restrict__ gslot, double* __restrict__ blk) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= ns) return;
  const Stencil S = st[s];
  double* g = gslot + kMaxN * s;
  double* b = blk + kBlk * s;
  if (S.nv == 1) eval_stencil<3>(S, X, D, P, val + s, g, b);
  else if (S.nv == 3) eval_stencil<9>(S, X, D, P, val + s, g, b);
  else eval_stencil<12>(S, X, D, P, val + s, g, b);
}

__global__ void k_values(const Stencil* __restrict__ st, int64_t ns, const double* __restrict__ X, TermData D,
                         Params P, double* __restrict__ val, unsigned long long* __restrict__ bad) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= ns) return;
  const Stencil S = st[s];
  V<double> x[4];
  for (int a = 0; a < S.nv; ++a) x[a] = V<double>{X[3 * S.v[a]], X[3 * S.v[a] + 1], X[3 * S.v[a] + 2]};
  const double e = term_value<double, 0>(S, x, D, P);
  val[s] = e;
  if (!(e == e) || isinf(e)) atomicOr(bad, 1ull);
}


// slot keys (vertex << 32 | stencil * 4 + local) for the deterministic per-vertex gather
__global__ void k_slot_keys(const Stencil* __restrict__ st, int64_t ns, uint64_t* __restrict__ keys) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= ns) return;
  const Stencil S = st[s];
  for (int a = 0; a < 4; ++a)
    keys[4 * s + a] = a < S.nv ? (static_cast<uint64_t>(S.v[a]) << 32) | static_cast<uint64_t>(4 * s + a) : ~0ull;
}
__global__ void k_slot_csr(const uint64_t* __restrict__ keys, int64_t n, int64_t nv, uint32_t* __restrict__ vstart) {
  // vstart[v] = first sorted position with vertex >= v (n for the tail); keys are sorted
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i > n) return;
  const int64_t vi = i < n && keys[i] != ~0ull ? static_cast<int64_t>(keys[i] >> 32) : nv;
  const int64_t vp = i == 0 ? -1 : (keys[i - 1] != ~0ull ? static_cast<int64_t>(keys[i - 1] >> 32) : nv);
  for (int64_t v = vp + 1; v <= vi && v <= nv; ++v) vstart[v] = static_cast<uint32_t>(i);
}
// out[v][k] = sum over the vertex's slots (ascending stencil order) of slot[.][k]
__global__ void k_gather(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vstart, int64_t nv,
                         const double* __restrict__ slot, double* __restrict__ out) {
  const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (v >= nv) return;
  double a = 0.0, b = 0.0, c = 0.0;
  for (uint32_t i = vstart[v]; i < vstart[v + 1]; ++i) {
    const uint64_t key = keys[i] & 0xffffffffu;  // 4 * stencil + local
    const double* g = slot + kMaxN * (key >> 2) + 3 * (key & 3);
    a += g[0];
    b += g[1];
    c += g[2];
  }
  out[3 * v] = a;
  out[3 * v + 1] = b;
  out[3 * v + 2] = c;
}

// ------------------------------------------------------------------------ vector ops
__global__ void k_xpay(int64_t n, const double* __restrict__ x, double a, double* __restrict__ y) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = x[i] + a * y[i];
}
__global__ void k_mul(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ o) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) o[i] = a[i] * b[i];
}
__global__ void k_step(int64_t n, const double* __restrict__ x, double a, const double* __restrict__ p,
                       double* __restrict__ o) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) o[i] = x[i] + a * p[i];
}

// ---- global block-sparse (BSR, 3x3 blocks) matrix from the projected stencil blocks: the
// sparsity is every (vertex, vertex) pair of every stencil; contributions to a block are summed
// in stencil order (a stable key sort), so the matrix is deterministic.
__global__ void k_pair_keys(const Stencil* __restrict__ st, int64_t ns, uint64_t* __restrict__ keys,
                            uint32_t* __restrict__ vals) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= ns) return;
  const Stencil S = st[s];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      const int64_t k = 16 * s + 4 * a + b;
      const bool on = a < S.nv && b < S.nv;
      keys[k] = on ? (static_cast<uint64_t>(S.v[a]) << 32) | static_cast<uint32_t>(S.v[b]) : ~0ull;
      vals[k] = static_cast<uint32_t>(k);
    }
}
__global__ void k_key_heads(const uint64_t* __restrict__ keys, int64_t n, uint32_t* __restrict__ head) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) head[i] = (keys[i] != ~0ull && (i == 0 || keys[i] != keys[i - 1])) ? 1u : 0u;
}
__global__ void k_bsr_fill(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                           const uint32_t* __restrict__ head, const uint32_t* __restrict__ hpos, int64_t n,
                           const Stencil* __restrict__ st, const double* __restrict__ blk, int32_t* __restrict__ bcol,
                           int32_t* __restrict__ brow, double* __restrict__ bval) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n || !head[i]) return;
  const uint32_t b = hpos[i];
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t j = i; j < n && keys[j] == keys[i]; ++j) {
    const uint32_t v = vals[j];
    const int64_t s = v >> 4;
    const int a = (v >> 2) & 3, c = v & 3;
    const int m = 3 * st[s].nv;
    const double* B = blk + kBlk * s;
    for (int r = 0; r < 3; ++r)
      for (int q = 0; q < 3; ++q) acc[3 * r + q] += B[(3 * a + r) * m + 3 * c + q];
  }
  brow[b] = static_cast<int32_t>(keys[i] >> 32);
  bcol[b] = static_cast<int32_t>(keys[i] & 0xffffffffu);
  for (int k = 0; k < 9; ++k) bval[9 * static_cast<int64_t>(b) + k] = acc[k];
}
__global__ void k_compact_u64(const uint64_t* __restrict__ in, const uint32_t* __restrict__ keep,
                              const uint32_t* __restrict__ pos, int64_t n, uint64_t* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n && keep[i]) out[pos[i]] = in[i];
}
__global__ void k_row_start(const int32_t* __restrict__ brow, int64_t nb, int64_t nv, uint32_t* __restrict__ rs) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i > nb) return;
  const int64_t vi = i < nb ? brow[i] : nv;
  const int64_t vp = i == 0 ? -1 : brow[i - 1];
  for (int64_t v = vp + 1; v <= vi && v <= nv; ++v) rs[v] = static_cast<uint32_t>(i);
}
__global__ void k_bsr_mv(const uint32_t* __restrict__ rs, const int32_t* __restrict__ bcol,
                         const double* __restrict__ bval, int64_t nv, const double* __restrict__ x,
                         double* __restrict__ y) {
  const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (v >= nv) return;
  double a = 0.0, b = 0.0, c = 0.0;
  for (uint32_t k = rs[v]; k < rs[v + 1]; ++k) {
    const double* B = bval + 9 * static_cast<int64_t>(k);
    const int j = bcol[k];
    const double x0 = x[3 * j], x1 = x[3 * j + 1], x2 = x[3 * j + 2];
    a += (B[0] * x0 + B[1] * x1) + B[2] * x2;
    b += (B[3] * x0 + B[4] * x1) + B[5] * x2;
    c += (B[6] * x0 + B[7] * x1) + B[8] * x2;
  }
  y[3 * v] = a;
  y[3 * v + 1] = b;
  y[3 * v + 2] = c;
}
// block-Jacobi preconditioner: the inverse of every vertex's 3x3 diagonal block (SPD)
__global__ void k_bsr_dinv(const uint32_t* __restrict__ rs, const int32_t* __restrict__ bcol,
                           const double* __restrict__ bval, int64_t nv, double* __restrict__ dinv) {
  const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (v >= nv) return;
  double a[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (uint32_t k = rs[v]; k < rs[v + 1]; ++k)
    if (bcol[k] == v)
      for (int q = 0; q < 9; ++q) a[q] += bval[9 * static_cast<int64_t>(k) + q];
  const double c00 = a[4] * a[8] - a[5] * a[7], c01 = a[5] * a[6] - a[3] * a[8], c02 = a[3] * a[7] - a[4] * a[6];
  const double det = a[0] * c00 + a[1] * c01 + a[2] * c02;
  double* o = dinv + 9 * v;
  if (!(det > 0.0)) {  // isolated vertex: identity
    for (int q = 0; q < 9; ++q) o[q] = (q % 4 == 0) ? 1.0 : 0.0;
    return;
  }
  const double id = 1.0 / det;
  o[0] = c00 * id;
  o[1] = (a[2] * a[7] - a[1] * a[8]) * id;
  o[2] = (a[1] * a[5] - a[2] * a[4]) * id;
  o[3] = c01 * id;
  o[4] = (a[0] * a[8] - a[2] * a[6]) * id;
  o[5] = (a[2] * a[3] - a[0] * a[5]) * id;
  o[6] = c02 * id;
  o[7] = (a[1] * a[6] - a[0] * a[7]) * id;
  o[8] = (a[0] * a[4] - a[1] * a[3]) * id;
}
__global__ void k_bprecond(int64_t nv, const double* __restrict__ dinv, const double* __restrict__ r,
                           double* __restrict__ z) {
  const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (v >= nv) return;
  const double* M = dinv + 9 * v;
  const double r0 = r[3 * v], r1 = r[3 * v + 1], r2 = r[3 * v + 2];
  z[3 * v] = (M[0] * r0 + M[1] * r1) + M[2] * r2;
  z[3 * v + 1] = (M[3] * r0 + M[4] * r1) + M[5] * r2;
  z[3 * v + 2] = (M[6] * r0 + M[7] * r1) + M[8] * r2;
}

// CG with device-resident scalars (no host round trip per iteration).  sc[0] = rz, sc[1] = qAq,
// sc[2] = rz_new, sc[3] = rr; every scalar comes from a CUB reduction of elementwise products.
__global__ void k_cg_step(int64_t n, const double* __restrict__ sc, const double* __restrict__ q,
                          const double* __restrict__ Ap, double* __restrict__ x, double* __restrict__ r,
                          double* __restrict__ prr) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double qaq = sc[1];
  const double alpha = qaq > 0.0 ? sc[0] / qaq : 0.0;
  x[i] += alpha * q[i];
  const double ri = r[i] - alpha * Ap[i];
  r[i] = ri;
  prr[i] = ri * ri;
}
__global__ void k_cg_dir(int64_t n, const double* __restrict__ sc, const double* __restrict__ z, double* __restrict__ q) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double beta = sc[0] != 0.0 ? sc[2] / sc[0] : 0.0;
  q[i] = z[i] + beta * q[i];
}
__global__ void k_cg_shift(double* __restrict__ sc) { sc[0] = sc[2]; }

// --------------------------------------------------------------------- broad phase
// face boxes over [X, X + p] inflated by `pad` (p may be null)
__global__ void k_swept_boxes(const double* __restrict__ X, const double* __restrict__ p, const int32_t* __restrict__ F,
                              int64_t nf, double pad, double* __restrict__ box, uint64_t* __restrict__ key) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int c = 0; c < 3; ++c) {
    const int v = F[3 * f + c];
    for (int k = 0; k < 3; ++k) {
      const double a = X[3 * v + k], b = p ? a + p[3 * v + k] : a;
      lo[k] = fmin(lo[k], fmin(a, b));
      hi[k] = fmax(hi[k], fmax(a, b));
    }
  }
  for (int k = 0; k < 3; ++k) {
    box[6 * f + k] = lo[k] - pad;
    box[6 * f + 3 + k] = hi[k] + pad;
  }
  // sort key: lo.x as an order-preserving integer, face id in the low bits
  const float fx = static_cast<float>(lo[0] - pad);
  const unsigned u = __float_as_uint(fx);
  const unsigned kx = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  key[f] = (static_cast<uint64_t>(kx) << 32) | static_cast<uint32_t>(f);
}

__device__ inline bool shares(const int32_t* a, const int32_t* b) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (a[i] == b[j]) return true;
  return false;
}

// sweep over faces sorted by lo.x: candidate face pairs with overlapping boxes (either order
// emitted once, i < j in sorted order).  Vertex-sharing pairs are kept: the caller splits them
// into point-triangle / edge-edge stencils and drops only the vertex-sharing primitives.
__global__ void k_sweep(const uint64_t* __restrict__ sorted, int64_t nf, const double* __restrict__ box,
                        uint64_t* __restrict__ pairs, uint64_t cap, unsigned long long* __restrict__ np) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nf) return;
  const int32_t a = static_cast<int32_t>(sorted[i] & 0xffffffffu);
  const double* A = box + 6 * a;
  for (int64_t j = i + 1; j < nf; ++j) {
    const int32_t b = static_cast<int32_t>(sorted[j] & 0xffffffffu);
    const double* Bx = box + 6 * b;
    // the sort key is lo.x rounded to f32: faces with equal keys may be out of order in double,
    // so stop only once lo.x is past A's hi.x by more than that rounding, and test x exactly
    if (Bx[0] - 1e-6 * fabs(Bx[0]) > A[3]) break;
    if (Bx[0] > A[3] || Bx[3] < A[0]) continue;
    if (Bx[1] > A[4] || Bx[4] < A[1] || Bx[2] > A[5] || Bx[5] < A[2]) continue;
    const unsigned long long k = atomicAdd(np, 1ull);
    if (k < cap) pairs[k] = (static_cast<uint64_t>(min(a, b)) << 32) | static_cast<uint32_t>(max(a, b));
  }
}

// face pairs -> primitive keys: PT (vertex, face) and EE (edge id pair), vertex-sharing dropped
__global__ void k_primitives(const uint64_t* __restrict__ pairs, int64_t n, const int32_t* __restrict__ F,
                             const int32_t* __restrict__ fedge, const int32_t* __restrict__ edges,
                             uint64_t* __restrict__ pt, unsigned long long* __restrict__ npt, uint64_t* __restrict__ ee,
                             unsigned long long* __restrict__ nee) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int32_t fa = static_cast<int32_t>(pairs[i] >> 32), fb = static_cast<int32_t>(pairs[i] & 0xffffffffu);
  const int32_t* A = F + 3 * fa;
  const int32_t* B = F + 3 * fb;
  for (int s = 0; s < 2; ++s) {
    const int32_t* P = s ? B : A;
    const int32_t* T = s ? A : B;
    const int32_t tf = s ? fa : fb;
    for (int k = 0; k < 3; ++k) {
      const int32_t v = P[k];
      if (v == T[0] || v == T[1] || v == T[2]) continue;
      pt[atomicAdd(npt, 1ull)] = (static_cast<uint64_t>(v) << 32) | static_cast<uint32_t>(tf);
    }
  }
  for (int x = 0; x < 3; ++x)
    for (int y = 0; y < 3; ++y) {
      const int32_t e1 = fedge[3 * fa + x], e2 = fedge[3 * fb + y];
      if (e1 == e2) continue;
      const int32_t a0 = edges[2 * e1], a1 = edges[2 * e1 + 1], b0 = edges[2 * e2], b1 = edges[2 * e2 + 1];
      if (a0 == b0 || a0 == b1 || a1 == b0 || a1 == b1) continue;
      ee[atomicAdd(nee, 1ull)] = (static_cast<uint64_t>(min(e1, e2)) << 32) | static_cast<uint32_t>(max(e1, e2));
    }
}

// ACCD (additive CCD as conservative advancement) for one primitive pair; returns the safe
// fraction of the step in (0, 1]
template <bool EE>
__device__ double accd_pair(const double* X, const double* p, const int* v, double margin) {
  double x[4][3], d[4][3], mean[3] = {0, 0, 0};
  for (int a = 0; a < 4; ++a)
    for (int k = 0; k < 3; ++k) {
      x[a][k] = X[3 * v[a] + k];
      d[a][k] = p[3 * v[a] + k];
      mean[k] += 0.25 * d[a][k];
    }
  double m0 = 0.0, m1 = 0.0;  // max centred displacement of the two primitives
  for (int a = 0; a < 4; ++a) {
    double s = 0.0;
    for (int k = 0; k < 3; ++k) s += (d[a][k] - mean[k]) * (d[a][k] - mean[k]);
    const double l = ::sqrt(s);
    if (EE ? a < 2 : a == 0) m0 = fmax(m0, l);
    else m1 = fmax(m1, l);
  }
  const double lp = m0 + m1;
  if (!(lp > 0.0)) return 1.0;
  // margin: the SPEC's 0.1 d̂, or 10% of the current gap when the pair is already closer than that
  // (the standard ACCD slack), so a close pair still lets the step advance
  {
    V<double> q[4];
    for (int a = 0; a < 4; ++a) q[a] = V<double>{x[a][0], x[a][1], x[a][2]};
    const double d0 = ::sqrt(fmax(EE ? d2_ee_class(q[0], q[1], q[2], q[3], ee_class(x[0], x[1], x[2], x[3]))
                                     : d2_pt_class(q[0], q + 1, pt_class(x[0], x[1], x[2], x[3])),
                                  0.0));
    margin = fmin(margin, 0.1 * d0);
  }
  double t = 0.0;
  for (int it = 0; it < 64; ++it) {
    double y[4][3];
    for (int a = 0; a < 4; ++a)
      for (int k = 0; k < 3; ++k) y[a][k] = x[a][k] + t * d[a][k];
    int cls;
    double dist2;
    V<double> q[4];
    for (int a = 0; a < 4; ++a) q[a] = V<double>{y[a][0], y[a][1], y[a][2]};
    if (EE) {
      cls = ee_class(y[0], y[1], y[2], y[3]);
      dist2 = d2_ee_class(q[0], q[1], q[2], q[3], cls);
    } else {
      cls = pt_class(y[0], y[1], y[2], y[3]);
      dist2 = d2_pt_class(q[0], q + 1, cls);
    }
    const double dist = ::sqrt(fmax(dist2, 0.0));
    if (dist <= margin) return t;
    t += 0.9 * (dist - margin) / lp;
    if (t >= 1.0) return 1.0;
  }
  return t;
}

__global__ void k_accd(const uint64_t* __restrict__ pt, int64_t npt, const uint64_t* __restrict__ ee, int64_t nee,
                       const int32_t* __restrict__ F, const int32_t* __restrict__ edges, const double* __restrict__ X,
                       const double* __restrict__ p, double margin, unsigned long long* __restrict__ tmin_bits) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= npt + nee) return;
  int v[4];
  double t;
  if (i < npt) {
    const int32_t pv = static_cast<int32_t>(pt[i] >> 32), f = static_cast<int32_t>(pt[i] & 0xffffffffu);
    v[0] = pv;
    v[1] = F[3 * f];
    v[2] = F[3 * f + 1];
    v[3] = F[3 * f + 2];
    t = accd_pair<false>(X, p, v, margin);
  } else {
    const int64_t j = i - npt;
    const int32_t e1 = static_cast<int32_t>(ee[j] >> 32), e2 = static_cast<int32_t>(ee[j] & 0xffffffffu);
    v[0] = edges[2 * e1];
    v[1] = edges[2 * e1 + 1];
    v[2] = edges[2 * e2];
    v[3] = edges[2 * e2 + 1];
    t = accd_pair<true>(X, p, v, margin);
  }
  atomicMin(tmin_bits, static_cast<unsigned long long>(__double_as_longlong(t)));  // t >= 0: bit order
}

// active contacts (d < d̂) -> barrier stencils (classes frozen at X)
__global__ void k_contacts(const uint64_t* __restrict__ pt, int64_t npt, const uint64_t* __restrict__ ee, int64_t nee,
                           const int32_t* __restrict__ F, const int32_t* __restrict__ edges, const double* __restrict__ X,
                           double dhat, Stencil* __restrict__ out, uint32_t* __restrict__ flag,
                           unsigned long long* __restrict__ touching) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= npt + nee) return;
  Stencil S;
  S.nv = 4;
  S.param = 0;
  double y[4][3];
  double d2;
  if (i < npt) {
    const int32_t pv = static_cast<int32_t>(pt[i] >> 32), f = static_cast<int32_t>(pt[i] & 0xffffffffu);
    S.term = kPT;
    S.v[0] = pv;
    S.v[1] = F[3 * f];
    S.v[2] = F[3 * f + 1];
    S.v[3] = F[3 * f + 2];
  } else {
    const int64_t j = i - npt;
    const int32_t e1 = static_cast<int32_t>(ee[j] >> 32), e2 = static_cast<int32_t>(ee[j] & 0xffffffffu);
    S.term = kEE;
    S.v[0] = edges[2 * e1];
    S.v[1] = edges[2 * e1 + 1];
    S.v[2] = edges[2 * e2];
    S.v[3] = edges[2 * e2 + 1];
  }
  for (int a = 0; a < 4; ++a)
    for (int k = 0; k < 3; ++k) y[a][k] = X[3 * S.v[a] + k];
  V<double> q[4];
  for (int a = 0; a < 4; ++a) q[a] = V<double>{y[a][0], y[a][1], y[a][2]};
  if (S.term == kPT) {
    S.cls = pt_class(y[0], y[1], y[2], y[3]);
    d2 = d2_pt_class(q[0], q + 1, S.cls);
  } else {
    S.cls = ee_class(y[0], y[1], y[2], y[3]);
    d2 = d2_ee_class(q[0], q[1], q[2], q[3], S.cls);
  }
  if (!(d2 > 0.0)) atomicAdd(touching, 1ull);
  // every candidate writes its stencil and an "active" flag at its own position; the caller
  // compacts them in candidate order (a scan), so the stencil order is deterministic
  out[i] = S;
  flag[i] = (d2 < dhat * dhat && d2 > 0.0) ? 1u : 0u;
}

__global__ void k_compact_contacts(const Stencil* __restrict__ in, const uint32_t* __restrict__ flag,
                                   const uint32_t* __restrict__ pos, int64_t n, Stencil* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n && flag[i]) out[pos[i]] = in[i];
}

// M2S stencils: nearest face of S per sample (from the LBVH query) with its class frozen
__global__ void k_m2s_stencils(const int32_t* __restrict__ face, int64_t m, const int32_t* __restrict__ F,
                               const double* __restrict__ X, const double* __restrict__ ys, Stencil* __restrict__ out) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= m) return;
  const int f = face[s];
  Stencil S;
  S.term = kM2S;
  S.nv = 3;
  S.param = static_cast<int>(s);
  for (int k = 0; k < 3; ++k) S.v[k] = F[3 * f + k];
  S.v[3] = -1;
  S.cls = pt_class(ys + 3 * s, X + 3 * S.v[0], X + 3 * S.v[1], X + 3 * S.v[2]);
  out[s] = S;
}

// ------------------------------------------------------------------------ rest state
__global__ void k_rest_faces(const double* __restrict__ X, const int32_t* __restrict__ F, int64_t nf,
                             double* __restrict__ dminv, double* __restrict__ a0, unsigned long long* __restrict__ bad) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  const double* x0 = X + 3 * F[3 * f];
  const double* x1 = X + 3 * F[3 * f + 1];
  const double* x2 = X + 3 * F[3 * f + 2];
  double e1[3], e2[3];
  for (int k = 0; k < 3; ++k) {
    e1[k] = x1[k] - x0[k];
    e2[k] = x2[k] - x0[k];
  }
  // 2D frame: u = e1/|e1|, w = n x u
  const double l1 = ::sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
  const double n[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
  const double nl = ::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
  if (!(l1 > 0.0) || !(nl > 0.0)) {
    atomicAdd(bad, 1ull);
    return;
  }
  const double u[3] = {e1[0] / l1, e1[1] / l1, e1[2] / l1};
  const double w[3] = {(n[1] * u[2] - n[2] * u[1]) / nl, (n[2] * u[0] - n[0] * u[2]) / nl,
                       (n[0] * u[1] - n[1] * u[0]) / nl};
  // Dm = [[e1.u, e2.u], [e1.w, e2.w]]
  const double m00 = l1, m01 = e2[0] * u[0] + e2[1] * u[1] + e2[2] * u[2];
  const double m10 = 0.0, m11 = e2[0] * w[0] + e2[1] * w[1] + e2[2] * w[2];
  const double det = m00 * m11 - m01 * m10;
  dminv[4 * f] = m11 / det;
  dminv[4 * f + 1] = -m01 / det;
  dminv[4 * f + 2] = -m10 / det;
  dminv[4 * f + 3] = m00 / det;
  a0[f] = 0.5 * nl;
}

// one stencil on one thread (unit checks of the terms, tests/test_gpu_project.py): the rest
// data arrive in small device arrays laid out like the solver's (X holds the stencil vertices
// 0..nv-1, X0 their rest positions)
__global__ void k_term_probe(Stencil S, const double* __restrict__ X, TermData D, Params P, double* __restrict__ out) {
  double val = 0.0, g[kMaxN], H[kBlk];
  if (S.nv == 1) eval_stencil<3>(S, X, D, P, &val, g, H);
  else if (S.nv == 3) eval_stencil<9>(S, X, D, P, &val, g, H);
  else eval_stencil<12>(S, X, D, P, &val, g, H);
  out[0] = val;
  const int n = 3 * S.nv;
  for (int i = 0; i < n; ++i) out[1 + i] = g[i];
  for (int i = 0; i < n * n; ++i) out[1 + kMaxN + i] = H[i];
}

// hinge rest state: theta0 (same signed dihedral as the bending term) and |x_i - x_j|
__global__ void k_hinge_rest(const double* __restrict__ X, const int32_t* __restrict__ hinge, int64_t nh,
                             double* __restrict__ theta0, double* __restrict__ l0) {
  const int64_t h = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (h >= nh) return;
  V<double> x[4];
  for (int a = 0; a < 4; ++a) {
    const int v = hinge[4 * h + a];
    x[a] = V<double>{X[3 * v], X[3 * v + 1], X[3 * v + 2]};
  }
  const V<double> e = x[1] - x[0];
  const V<double> n0 = ad::cross(e, x[2] - x[0]), n1 = ad::cross(x[3] - x[0], e);
  const double el = ::sqrt(ad::dot(e, e));
  theta0[h] = ::atan2(ad::dot(ad::cross(n0, n1), e) / el, ad::dot(n0, n1));
  l0[h] = el;
}

// ============================================================================ host
double dev_sum(Ctx& ctx, const double* d, int64_t n) {
  if (n <= 0) return 0.0;
  DevBuf<double> out(1, ctx.stream);
  size_t need = 0;
  cub::DeviceReduce::Sum(nullptr, need, d, out.get(), n, ctx.stream);
  DevBuf<uint8_t> tmp(need ? need : 1, ctx.stream);
  PCU_CUDA(cub::DeviceReduce::Sum(tmp.get(), need, d, out.get(), n, ctx.stream));
  ++ctx.launches;
  return read_scalar(ctx, out.get());
}

struct Assembly {
  DevBuf<Stencil> st;
  int64_t ns = 0;
  DevBuf<double> val, gslot, blk;
  DevBuf<uint64_t> keys, keys2;
  DevBuf<uint32_t> vstart;
};

}  // namespace

void safe_project(Ctx& ctx, double* dV, int64_t nv, const int32_t* dF, int64_t nf, const double* dVin,
                  const int32_t* dFin, int64_t nfin, const ProjectParams& PP, ProjectStats& stats,
                  ProjectTrace* tr) {
  cudaStream_t st = ctx.stream;
  PCU_REQUIRE(nv > 0 && nf > 0 && nfin > 0, PAMOPT_CU_EINVAL, "safe_project: empty mesh");
  const std::vector<int32_t> sip = self_intersections(ctx, dV, nv, dF, nf, nullptr, nullptr);
  PCU_REQUIRE(sip.empty(), PAMOPT_CU_EINVAL, "safe_project: the input mesh self-intersects (infeasible)");
  Params P{PP.kdis, PP.kelas, PP.kbend, PP.kbar, PP.dhat, PP.elas_tau, PP.elas_power};
  // ---- topology (host; setup only): unique edges, per-face edge ids, interior hinges
  std::vector<int32_t> hF(3 * nf);
  PCU_CUDA(cudaMemcpyAsync(hF.data(), dF, 3 * nf * 4, cudaMemcpyDeviceToHost, st));
  PCU_CUDA(cudaStreamSynchronize(st));
  std::vector<std::pair<uint64_t, int32_t>> he(3 * nf);  // (edge key, face * 3 + k)
  for (int64_t f = 0; f < nf; ++f)
    for (int k = 0; k < 3; ++k) {
      const uint32_t a = hF[3 * f + k], b = hF[3 * f + (k + 1) % 3];
      he[3 * f + k] = {(static_cast<uint64_t>(std::min(a, b)) << 32) | std::max(a, b), static_cast<int32_t>(3 * f + k)};
    }
  std::sort(he.begin(), he.end());
  std::vector<int32_t> edges, fedge(3 * nf), hinge;
  for (size_t i = 0; i < he.size();) {
    size_t j = i;
    while (j < he.size() && he[j].first == he[i].first) ++j;
    const int32_t eid = static_cast<int32_t>(edges.size() / 2);
    edges.push_back(static_cast<int32_t>(he[i].first >> 32));
    edges.push_back(static_cast<int32_t>(he[i].first & 0xffffffffu));
    for (size_t q = i; q < j; ++q) fedge[he[q].second] = eid;
    if (j - i == 2) {  // interior edge: (i, j) as in the first face, k/l the opposite corners
      const int32_t c0 = he[i].second, c1 = he[i + 1].second;
      const int32_t f0 = c0 / 3, k0 = c0 % 3, f1 = c1 / 3, k1 = c1 % 3;
      const int32_t vi = hF[3 * f0 + k0], vj = hF[3 * f0 + (k0 + 1) % 3];
      hinge.insert(hinge.end(), {vi, vj, hF[3 * f0 + (k0 + 2) % 3], hF[3 * f1 + (k1 + 2) % 3]});
    }
    i = j;
  }
  const int64_t ne = static_cast<int64_t>(edges.size() / 2), nh = static_cast<int64_t>(hinge.size() / 4);
  DevBuf<int32_t> dEdges(2 * ne, st), dFedge(3 * nf, st), dHinge(4 * (nh ? nh : 1), st);
  PCU_CUDA(cudaMemcpyAsync(dEdges.get(), edges.data(), 2 * ne * 4, cudaMemcpyHostToDevice, st));
  PCU_CUDA(cudaMemcpyAsync(dFedge.get(), fedge.data(), 3 * nf * 4, cudaMemcpyHostToDevice, st));
  if (nh) PCU_CUDA(cudaMemcpyAsync(dHinge.get(), hinge.data(), 4 * nh * 4, cudaMemcpyHostToDevice, st));
  // ---- rest state
  DevBuf<double> X0(3 * nv, st), dminv(4 * nf, st), a0(nf, st), theta0(nh ? nh : 1, st), l0(nh ? nh : 1, st);
  PCU_CUDA(cudaMemcpyAsync(X0.get(), dV, 3 * nv * 8, cudaMemcpyDeviceToDevice, st));
  DevBuf<unsigned long long> flag(2, st);
  PCU_CUDA(cudaMemsetAsync(flag.get(), 0, 16, st));
  PCU_LAUNCH(ctx, k_rest_faces, grid_for(nf, 128), 128, 0, dV, dF, nf, dminv.get(), a0.get(), flag.get());
  PCU_REQUIRE(read_scalar(ctx, flag.get()) == 0, PAMOPT_CU_EINVAL, "safe_project: degenerate rest face");
  if (nh) PCU_LAUNCH(ctx, k_hinge_rest, grid_for(nh, 128), 128, 0, dV, dHinge.get(), nh, theta0.get(), l0.get());
  std::vector<double> ha0(nf), hs0(nv, 0.0);
  PCU_CUDA(cudaMemcpyAsync(ha0.data(), a0.get(), nf * 8, cudaMemcpyDeviceToHost, st));
  PCU_CUDA(cudaStreamSynchronize(st));
  for (int64_t f = 0; f < nf; ++f)
    for (int k = 0; k < 3; ++k) hs0[hF[3 * f + k]] += ha0[f] / 3.0;  // barycentric "Voronoi" areas
  DevBuf<double> s0(nv, st);
  PCU_CUDA(cudaMemcpyAsync(s0.get(), hs0.data(), nv * 8, cudaMemcpyHostToDevice, st));
  // ---- samples on M_in
  const int64_t m = PP.samples;
  DevBuf<double> ys(3 * m, st), ytgt(3 * nv, st), scratch_d2(std::max(nv, m), st);
  DevBuf<int32_t> sface(std::max(nv, m), st);
  double ain = 0.0;
  PCU_REQUIRE(sample_points(ctx, dVin, dFin, nfin, m, PP.seed, ys.get(), nullptr, &ain), PAMOPT_CU_EINVAL,
              "safe_project: zero-area input mesh");
  if (tr && tr->samples) PCU_CUDA(cudaMemcpyAsync(tr->samples, ys.get(), 3 * m * 8, cudaMemcpyDeviceToHost, st));
  TermData D{X0.get(), s0.get(), ytgt.get(), ys.get(), ain / static_cast<double>(m), dminv.get(), a0.get(),
             theta0.get(), l0.get()};
  // ---- static stencils: S2M, elastic, bending
  std::vector<Stencil> hst;
  hst.reserve(nv + nf + nh);
  for (int64_t v = 0; v < nv; ++v) hst.push_back(Stencil{kS2M, 1, {static_cast<int>(v), -1, -1, -1}, 0, 0});
  for (int64_t f = 0; f < nf; ++f)
    hst.push_back(Stencil{kElas, 3, {hF[3 * f], hF[3 * f + 1], hF[3 * f + 2], -1}, static_cast<int>(f), 0});
  for (int64_t h = 0; h < nh; ++h)
    hst.push_back(Stencil{kBend, 4, {hinge[4 * h], hinge[4 * h + 1], hinge[4 * h + 2], hinge[4 * h + 3]},
                          static_cast<int>(h), 0});
  const int64_t nstatic = static_cast<int64_t>(hst.size());
  // stencil layout: [static | M2S (m) | contacts]
  int64_t ccap = 4096;
  DevBuf<Stencil> stc;
  auto ensure_st = [&](int64_t ncont) {
    const int64_t need = nstatic + m + ncont;
    if (static_cast<int64_t>(stc.n) < need) {
      DevBuf<Stencil> n2(need + 4096, st);
      if (stc.n) PCU_CUDA(cudaMemcpyAsync(n2.get(), stc.get(), (nstatic + m) * sizeof(Stencil), cudaMemcpyDeviceToDevice, st));
      else PCU_CUDA(cudaMemcpyAsync(n2.get(), hst.data(), nstatic * sizeof(Stencil), cudaMemcpyHostToDevice, st));
      stc = std::move(n2);
    }
  };
  ensure_st(ccap);

  // ---- broad phase -> contact primitives (deduplicated) for positions X (+ p when sweeping)
  DevBuf<double> box(6 * nf, st);
  DevBuf<uint64_t> bkey(nf, st), bkey2(nf, st);
  DevBuf<uint64_t> fpairs, pt, ee, ubuf;
  DevBuf<uint32_t> uhead, upos;
  int64_t npt = 0, nee = 0;
  auto primitives = [&](const double* X, const double* p, double pad) {
    PCU_LAUNCH(ctx, k_swept_boxes, grid_for(nf, 256), 256, 0, X, p, dF, nf, pad, box.get(), bkey.get());
    sort_pairs_u64(ctx, bkey.get(), nf);
    uint64_t cap = std::max<uint64_t>(fpairs.n, 16 * static_cast<uint64_t>(nf) + 1024);
    for (;;) {
      fpairs.ensure(cap, st);
      PCU_CUDA(cudaMemsetAsync(flag.get(), 0, 8, st));
      PCU_LAUNCH(ctx, k_sweep, grid_for(nf, 128), 128, 0, bkey.get(), nf, box.get(), fpairs.get(), cap, flag.get());
      const unsigned long long np = read_scalar(ctx, flag.get());
      if (np <= cap) {
        pt.ensure(6 * np + 16, st);
        ee.ensure(9 * np + 16, st);
        DevBuf<unsigned long long> c2(2, st);
        PCU_CUDA(cudaMemsetAsync(c2.get(), 0, 16, st));
        if (np) PCU_LAUNCH(ctx, k_primitives, grid_for(np, 128), 128, 0, fpairs.get(), static_cast<int64_t>(np), dF,
                           dFedge.get(), dEdges.get(), pt.get(), c2.get(), ee.get(), c2.get() + 1);
        unsigned long long h2[2];
        PCU_CUDA(cudaMemcpyAsync(h2, c2.get(), 16, cudaMemcpyDeviceToHost, st));
        PCU_CUDA(cudaStreamSynchronize(st));
        // dedup on the device (sort, head flags, scan, compact) — a primitive pair can come from
        // several face pairs
        auto uniq = [&](DevBuf<uint64_t>& a, int64_t n) -> int64_t {
          if (n <= 1) return n;
          sort_pairs_u64(ctx, a.get(), n);
          uhead.ensure(n, st);
          upos.ensure(n, st);
          ubuf.ensure(n, st);
          PCU_LAUNCH(ctx, k_key_heads, grid_for(n, 256), 256, 0, a.get(), n, uhead.get());
          exclusive_scan_u32(ctx, uhead.get(), upos.get(), n);
          const int64_t u = static_cast<int64_t>(read_scalar(ctx, upos.get() + n - 1)) + read_scalar(ctx, uhead.get() + n - 1);
          PCU_LAUNCH(ctx, k_compact_u64, grid_for(n, 256), 256, 0, a.get(), uhead.get(), upos.get(), n, ubuf.get());
          PCU_CUDA(cudaMemcpyAsync(a.get(), ubuf.get(), u * 8, cudaMemcpyDeviceToDevice, st));
          return u;
        };
        npt = uniq(pt, static_cast<int64_t>(h2[0]));
        nee = uniq(ee, static_cast<int64_t>(h2[1]));
        return;
      }
      cap = np + np / 4 + 1024;
    }
  };

  Assembly A;
  DevBuf<Stencil> cand;
  DevBuf<uint32_t> cflag, cpos;
  auto build_contacts = [&](const double* X, int64_t& ncont, bool& touching) {
    primitives(X, nullptr, P.dhat);
    const int64_t nc = npt + nee;
    ncont = 0;
    touching = false;
    if (nc == 0) return;
    cand.ensure(nc, st);
    cflag.ensure(nc, st);
    cpos.ensure(nc, st);
    PCU_CUDA(cudaMemsetAsync(flag.get(), 0, 8, st));
    PCU_LAUNCH(ctx, k_contacts, grid_for(nc, 128), 128, 0, pt.get(), npt, ee.get(), nee, dF, dEdges.get(), X, P.dhat,
               cand.get(), cflag.get(), flag.get());
    exclusive_scan_u32(ctx, cflag.get(), cpos.get(), nc);
    ncont = static_cast<int64_t>(read_scalar(ctx, cpos.get() + nc - 1)) + read_scalar(ctx, cflag.get() + nc - 1);
    touching = read_scalar(ctx, flag.get()) != 0;
    if (ncont > ccap) ccap = ncont + 1024;
    ensure_st(ccap);
    PCU_LAUNCH(ctx, k_compact_contacts, grid_for(nc, 128), 128, 0, cand.get(), cflag.get(), cpos.get(), nc,
               stc.get() + nstatic + m);
  };
  auto energy = [&](const double* X, int64_t ns, bool& bad) {
    A.val.ensure(ns, st);
    PCU_CUDA(cudaMemsetAsync(flag.get(), 0, 8, st));
    PCU_LAUNCH(ctx, k_values, grid_for(ns, 128), 128, 0, stc.get(), ns, X, D, P, A.val.get(), flag.get());
    bad = read_scalar(ctx, flag.get()) != 0;
    return dev_sum(ctx, A.val.get(), ns);
  };
  const int64_t n3 = 3 * nv;
  DevBuf<double> g(n3, st), pdir(n3, st), r(n3, st), z(n3, st), q(n3, st), Ap(n3, st), tmpv(n3, st),
      Xn(n3, st);
  auto gather = [&](const double* slots, double* out) {
    PCU_LAUNCH(ctx, k_gather, grid_for(nv, 256), 256, 0, A.keys2.get(), A.vstart.get(), nv, slots, out);
  };
  DevBuf<double> sc(4, st), tmp2(n3, st), bval, dinv;
  DevBuf<uint64_t> bk, bk2;
  DevBuf<uint32_t> bvl, bvl2, bhead, bhpos, rstart;
  DevBuf<int32_t> bcol, brow;
  int64_t nblk = 0;
  DevBuf<uint8_t> red_tmp;
  size_t red_bytes = 0;
  auto dev_sum_to = [&](const double* d, int64_t n, double* out) {  // deterministic CUB sum into device memory
    size_t need = 0;
    cub::DeviceReduce::Sum(nullptr, need, d, out, n, st);
    if (need > red_bytes) {
      red_tmp.alloc(need, st);
      red_bytes = need;
    }
    PCU_CUDA(cub::DeviceReduce::Sum(red_tmp.get(), need, d, out, n, st));
    ++ctx.launches;
  };
  auto dot = [&](const double* a, const double* b) {
    PCU_LAUNCH(ctx, k_mul, grid_for(n3, 256), 256, 0, n3, a, b, tmpv.get());
    return dev_sum(ctx, tmpv.get(), n3);
  };

  stats = ProjectStats();
  std::vector<Stencil> hrec;
  auto rec_vec = [&](double* base, int it, const double* dsrc) {  // one 3nv record
    if (base) PCU_CUDA(cudaMemcpyAsync(base + static_cast<size_t>(it) * n3, dsrc, n3 * 8, cudaMemcpyDeviceToHost, st));
  };
  auto rec_stencils = [&](int32_t* base, int64_t stride, int width, const Stencil* dsrc, int64_t n) {
    hrec.resize(n);
    if (n) PCU_CUDA(cudaMemcpyAsync(hrec.data(), dsrc, n * sizeof(Stencil), cudaMemcpyDeviceToHost, st));
    PCU_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < n && i < stride; ++i) {
      int32_t* o = base + width * i;
      if (width == 6) {
        o[0] = hrec[i].term;
        o[1] = hrec[i].cls;
        for (int k = 0; k < 4; ++k) o[2 + k] = hrec[i].v[k];
      } else {
        for (int k = 0; k < 3; ++k) o[k] = hrec[i].v[k];
        o[3] = hrec[i].cls;
      }
    }
  };
  for (int it = 0; it < PP.iterations; ++it) {
    const bool rec = tr && it < tr->max_iters;
    double* rs = rec && tr->scalars ? tr->scalars + 8 * static_cast<size_t>(it) : nullptr;
    if (rec) rec_vec(tr->X, it, dV);
    if (it % PP.refresh == 0) {
      // S2M targets: nearest points of M_in; M2S: nearest faces of S(X) with frozen classes
      nearest_primitive(ctx, dVin, dFin, nfin, dV, nv, sface.get(), scratch_d2.get(), ytgt.get());
      nearest_primitive(ctx, dV, dF, nf, ys.get(), m, sface.get(), scratch_d2.get(), nullptr);
      PCU_LAUNCH(ctx, k_m2s_stencils, grid_for(m, 128), 128, 0, sface.get(), m, dF, dV, ys.get(), stc.get() + nstatic);
      ++stats.refreshes;
    }
    int64_t ncont = 0;
    bool touching = false;
    build_contacts(dV, ncont, touching);
    PCU_REQUIRE(!touching, PAMOPT_CU_ENUMERIC, "safe_project: a contact pair reached distance 0 (infeasible)");
    const int64_t ns = nstatic + m + ncont;
    if (rec) {
      rec_vec(tr->targets, it, ytgt.get());
      if (tr->m2s) rec_stencils(tr->m2s + static_cast<size_t>(it) * 4 * m, m, 4, stc.get() + nstatic, m);
      if (tr->contacts)
        rec_stencils(tr->contacts + static_cast<size_t>(it) * 6 * tr->contact_cap, tr->contact_cap, 6,
                     stc.get() + nstatic + m, ncont);
      if (tr->n_contacts) tr->n_contacts[it] = ncont;
    }
    // ---- assemble gradient + projected Hessian blocks
    A.val.ensure(ns, st);
    A.gslot.ensure(kMaxN * ns, st);
    A.blk.ensure(kBlk * ns, st);
    A.keys.ensure(4 * ns, st);
    A.keys2.ensure(4 * ns, st);
    A.vstart.ensure(nv + 1, st);
    PCU_LAUNCH(ctx, k_assemble, grid_for(ns, 64), 64, 0, stc.get(), ns, dV, D, P, A.val.get(), A.gslot.get(),
               A.blk.get());
    const double B0 = dev_sum(ctx, A.val.get(), ns);
    PCU_LAUNCH(ctx, k_slot_keys, grid_for(ns, 256), 256, 0, stc.get(), ns, A.keys.get());
    PCU_CUDA(cudaMemcpyAsync(A.keys2.get(), A.keys.get(), 4 * ns * 8, cudaMemcpyDeviceToDevice, st));
    sort_pairs_u64(ctx, A.keys2.get(), 4 * ns);
    PCU_LAUNCH(ctx, k_slot_csr, grid_for(4 * ns + 1, 256), 256, 0, A.keys2.get(), 4 * ns, nv, A.vstart.get());
    gather(A.gslot.get(), g.get());
    if (rec) rec_vec(tr->grad, it, g.get());
    {  // global BSR matrix (3x3 blocks), deterministic summation in stencil order
      const int64_t np = 16 * ns;
      bk.ensure(np, st);
      bk2.ensure(np, st);
      bvl.ensure(np, st);
      bvl2.ensure(np, st);
      bhead.ensure(np, st);
      bhpos.ensure(np, st);
      PCU_LAUNCH(ctx, k_pair_keys, grid_for(ns, 128), 128, 0, stc.get(), ns, bk.get(), bvl.get());
      size_t need = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, need, bk.get(), bk2.get(), bvl.get(), bvl2.get(), static_cast<int>(np), 0,
                                      64, st);
      if (need > red_bytes) {
        red_tmp.alloc(need, st);
        red_bytes = need;
      }
      PCU_CUDA(cub::DeviceRadixSort::SortPairs(red_tmp.get(), need, bk.get(), bk2.get(), bvl.get(), bvl2.get(),
                                               static_cast<int>(np), 0, 64, st));
      ++ctx.launches;
      PCU_LAUNCH(ctx, k_key_heads, grid_for(np, 256), 256, 0, bk2.get(), np, bhead.get());
      exclusive_scan_u32(ctx, bhead.get(), bhpos.get(), np);
      nblk = static_cast<int64_t>(read_scalar(ctx, bhpos.get() + np - 1)) + read_scalar(ctx, bhead.get() + np - 1);
      bcol.ensure(nblk, st);
      brow.ensure(nblk, st);
      bval.ensure(9 * nblk, st);
      rstart.ensure(nv + 1, st);
      PCU_LAUNCH(ctx, k_bsr_fill, grid_for(np, 128), 128, 0, bk2.get(), bvl2.get(), bhead.get(), bhpos.get(), np,
                 stc.get(), A.blk.get(), bcol.get(), brow.get(), bval.get());
      PCU_LAUNCH(ctx, k_row_start, grid_for(nblk + 1, 256), 256, 0, brow.get(), nblk, nv, rstart.get());
      dinv.ensure(9 * nv, st);
      PCU_LAUNCH(ctx, k_bsr_dinv, grid_for(nv, 256), 256, 0, rstart.get(), bcol.get(), bval.get(), nv, dinv.get());
    }
    // ---- PCG: H p = -g
    const double gnorm = ::sqrt(dot(g.get(), g.get()));
    stats.grad_norm = gnorm;
    if (!(gnorm > 0.0)) break;
    PCU_CUDA(cudaMemsetAsync(pdir.get(), 0, n3 * 8, st));
    PCU_CUDA(cudaMemcpyAsync(r.get(), g.get(), n3 * 8, cudaMemcpyDeviceToDevice, st));
    PCU_LAUNCH(ctx, k_xpay, grid_for(n3, 256), 256, 0, n3, pdir.get(), -1.0, r.get());  // r = -g
    PCU_LAUNCH(ctx, k_bprecond, grid_for(nv, 256), 256, 0, nv, dinv.get(), r.get(), z.get());
    PCU_CUDA(cudaMemcpyAsync(q.get(), z.get(), n3 * 8, cudaMemcpyDeviceToDevice, st));
    PCU_LAUNCH(ctx, k_mul, grid_for(n3, 256), 256, 0, n3, r.get(), z.get(), tmpv.get());
    dev_sum_to(tmpv.get(), n3, sc.get());
    const double tol2 = PP.cg_tol * PP.cg_tol * gnorm * gnorm;
    int cg = 0;
    auto cg_iter = [&]() {
      PCU_LAUNCH(ctx, k_bsr_mv, grid_for(nv, 128), 128, 0, rstart.get(), bcol.get(), bval.get(), nv, q.get(), Ap.get());
      PCU_LAUNCH(ctx, k_mul, grid_for(n3, 256), 256, 0, n3, q.get(), Ap.get(), tmpv.get());
      dev_sum_to(tmpv.get(), n3, sc.get() + 1);
      PCU_LAUNCH(ctx, k_cg_step, grid_for(n3, 256), 256, 0, n3, sc.get(), q.get(), Ap.get(), pdir.get(), r.get(),
                 tmp2.get());
      PCU_LAUNCH(ctx, k_bprecond, grid_for(nv, 256), 256, 0, nv, dinv.get(), r.get(), z.get());
      PCU_LAUNCH(ctx, k_mul, grid_for(n3, 256), 256, 0, n3, r.get(), z.get(), tmpv.get());
      dev_sum_to(tmpv.get(), n3, sc.get() + 2);
      dev_sum_to(tmp2.get(), n3, sc.get() + 3);
      PCU_LAUNCH(ctx, k_cg_dir, grid_for(n3, 256), 256, 0, n3, sc.get(), z.get(), q.get());
      PCU_LAUNCH(ctx, k_cg_shift, 1, 1, 0, sc.get());
    };
    auto converged = [&]() {
      double h[4];
      PCU_CUDA(cudaMemcpyAsync(h, sc.get(), 32, cudaMemcpyDeviceToHost, st));
      PCU_CUDA(cudaStreamSynchronize(st));
      return h[3] <= tol2 || !(h[1] > 0.0);
    };
    constexpr int kChunk = 16;  // CG iterations per convergence check
    if (!ctx.prof.kt) {
      // the 16-iteration chunk is captured once per Newton step into a CUDA graph and replayed:
      // the CG kernels are tiny, so launch latency, not work, bounds them
      cudaGraph_t graph = nullptr;
      cudaGraphExec_t exec = nullptr;
      PCU_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      for (int k = 0; k < kChunk; ++k) cg_iter();
      PCU_CUDA(cudaStreamEndCapture(st, &graph));
      PCU_CUDA(cudaGraphInstantiate(&exec, graph, 0));
      for (; cg < PP.cg_max;) {
        PCU_CUDA(cudaGraphLaunch(exec, st));
        cg += kChunk;
        if (converged()) break;
      }
      cudaGraphExecDestroy(exec);
      cudaGraphDestroy(graph);
    } else {
      for (; cg < PP.cg_max;) {
        for (int k = 0; k < kChunk; ++k) cg_iter();
        cg += kChunk;
        if (converged()) break;
      }
    }
    stats.cg_iterations += cg;
    if (rec) rec_vec(tr->dir, it, pdir.get());
    // ---- ACCD step bound over the swept primitives
    primitives(dV, pdir.get(), P.dhat);
    DevBuf<unsigned long long> tb(1, st);
    const double one = 1.0;
    unsigned long long onebits;
    std::memcpy(&onebits, &one, 8);
    PCU_CUDA(cudaMemcpyAsync(tb.get(), &onebits, 8, cudaMemcpyHostToDevice, st));
    if (npt + nee)
      PCU_LAUNCH(ctx, k_accd, grid_for(npt + nee, 128), 128, 0, pt.get(), npt, ee.get(), nee, dF, dEdges.get(), dV,
                 pdir.get(), 0.1 * P.dhat, tb.get());
    const unsigned long long tbits = read_scalar(ctx, tb.get());
    double tmax;
    std::memcpy(&tmax, &tbits, 8);
    double alpha = std::min(1.0, 0.9 * tmax);
    // ---- backtracking line search: B decreases and the exact check finds no intersection
    bool accepted = false;
    int tries = 0;
    for (int ls = 0; ls < 64 && alpha > 0.0; ++ls, alpha *= 0.5) {
      ++tries;
      PCU_LAUNCH(ctx, k_step, grid_for(n3, 256), 256, 0, n3, dV, alpha, pdir.get(), Xn.get());
      int64_t nc2 = 0;
      bool touch2 = false;
      build_contacts(Xn.get(), nc2, touch2);
      if (touch2) continue;
      bool bad = false;
      const double B1 = energy(Xn.get(), nstatic + m + nc2, bad);
      if (bad || !(B1 < B0)) continue;
      if (!self_intersections(ctx, Xn.get(), nv, dF, nf, nullptr, nullptr).empty()) continue;
      accepted = true;
      stats.energy = B1;
      break;
    }
    if (it == 0) stats.energy0 = B0;
    stats.iterations = it + 1;
    if (rs) {
      const double r8[8] = {B0, gnorm, static_cast<double>(cg), tmax, alpha, accepted ? stats.energy : B0,
                            accepted ? 1.0 : 0.0, static_cast<double>(tries)};
      std::memcpy(rs, r8, sizeof(r8));
    }
    if (!accepted) {  // no decrease along a feasible step: converged
      stats.energy = B0;
      stats.converged = 1;
      break;
    }
    PCU_CUDA(cudaMemcpyAsync(dV, Xn.get(), n3 * 8, cudaMemcpyDeviceToDevice, st));
    stats.last_alpha = alpha;
  }
  PCU_CUDA(cudaStreamSynchronize(st));
}

void project_term_probe(Ctx& ctx, int term, int cls, const double* coords, int nv, const double* rest,
                        const ProjectParams& PP, double* out) {
  // rest: {s0, ytgt[3], ys[3], m2s_w}  (S2M / M2S), {dminv[4], a0} (elastic), {theta0, l0} (bending)
  cudaStream_t st = ctx.stream;
  PCU_REQUIRE(nv == 1 || nv == 3 || nv == 4, PAMOPT_CU_EINVAL, "term probe: 1, 3 or 4 vertices");
  DevBuf<double> X(3 * nv, st), R(16, st), o(1 + kMaxN + kBlk, st);
  PCU_CUDA(cudaMemcpyAsync(X.get(), coords, 3 * nv * 8, cudaMemcpyHostToDevice, st));
  PCU_CUDA(cudaMemcpyAsync(R.get(), rest, 16 * 8, cudaMemcpyHostToDevice, st));
  const double* r = R.get();
  TermData D{X.get(), r + 0, r + 1, r + 4, rest[7], r + 8, r + 12, r + 13, r + 14};
  Params P{PP.kdis, PP.kelas, PP.kbend, PP.kbar, PP.dhat, PP.elas_tau, PP.elas_power};
  Stencil S{term, nv, {0, nv > 1 ? 1 : -1, nv > 2 ? 2 : -1, nv > 3 ? 3 : -1}, 0, cls};
  PCU_LAUNCH(ctx, k_term_probe, 1, 1, 0, S, X.get(), D, P, o.get());
  PCU_CUDA(cudaMemcpyAsync(out, o.get(), (1 + kMaxN + kBlk) * 8, cudaMemcpyDeviceToHost, st));
  PCU_CUDA(cudaStreamSynchronize(st));
}

}  // namespace pcu
