// ORACLE — CPU restatement of the remesh hot path.  TEST INFRASTRUCTURE ONLY:
// loaded by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm as the checker.  Never linked into the product (paper_2509_05595_b200/).
//
// geom.hpp: pinned geometric arithmetic shared by the oracle modules.
//   * vector ops follow the Eigen fixed-size-3 order pinned in oracle/eigen_shim
//     (dot = (x0y0 + x1y1) + x2y2; Eigen cross formula);
//   * point_segment / point_triangle squared distance restate
//     /root/reference/proj/src/distance.cpp:10-79 operation for operation
//     (checked bit-exactly against the compiled reference in tests/test_oracle_ref.py);
//   * exact orientation predicates (Shewchuk-style static filter + exact expansion
//     arithmetic) used by tri_isect — exact verdicts by construction;
//   * det_exp: the pinned exponential used by the DMC sigmoid.
// Built with -ffp-contract=off: no FMA contraction anywhere.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>

namespace orc {

struct V3 {
  double x, y, z;
};

inline V3 v3(double x, double y, double z) { return V3{x, y, z}; }
inline V3 operator+(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(double s, V3 a) { return V3{a.x * s, a.y * s, a.z * s}; }
inline double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline double sqnorm(V3 a) { return dot(a, a); }
inline V3 cross(V3 a, V3 b) {
  return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double get(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

// distance.cpp:10-21
inline double point_segment_sq(V3 p, V3 a, V3 b, double* t_out = nullptr) {
  const V3 ab = b - a;
  const double denom = sqnorm(ab);
  double t = denom > 0.0 ? dot(p - a, ab) / denom : 0.0;
  t = t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t);  // std::clamp
  const V3 q = a + t * ab;
  if (t_out) *t_out = t;
  return sqnorm(p - q);
}

// distance.cpp:26-79: face-projection candidate, then the three edges with strict '<'.
inline double point_triangle_sq(V3 p, V3 a, V3 b, V3 c) {
  const V3 n = cross(b - a, c - a);
  const double nn = sqnorm(n);
  double best = std::numeric_limits<double>::infinity();
  if (nn > 0.0) {
    const V3 ap = p - a;
    const double dist_n = dot(ap, n);
    const V3 proj = p - (dist_n / nn) * n;
    const V3 v0 = b - a, v1 = c - a, v2 = proj - a;
    const double d00 = sqnorm(v0), d01 = dot(v0, v1), d11 = sqnorm(v1);
    const double d20 = dot(v2, v0), d21 = dot(v2, v1);
    const double denom = d00 * d11 - d01 * d01;
    if (denom > 0.0) {
      const double v = (d11 * d20 - d01 * d21) / denom;
      const double w = (d00 * d21 - d01 * d20) / denom;
      if (v >= 0.0 && w >= 0.0 && v + w <= 1.0) best = dist_n * dist_n / nn;
    }
  }
  const double e0 = point_segment_sq(p, a, b);
  if (e0 < best) best = e0;
  const double e1 = point_segment_sq(p, b, c);
  if (e1 < best) best = e1;
  const double e2 = point_segment_sq(p, c, a);
  if (e2 < best) best = e2;
  return best;
}

// ---------------------------------------------------------------------------
// Exact arithmetic (expansions).  Dekker split / two-product: exact without FMA.

namespace exact {

constexpr double kSplitter = 134217729.0;  // 2^27 + 1

inline void two_sum(double a, double b, double& x, double& y) {
  x = a + b;
  const double bv = x - a;
  const double av = x - bv;
  y = (a - av) + (b - bv);
}
inline void two_diff(double a, double b, double& x, double& y) {
  x = a - b;
  const double bv = a - x;
  const double av = x + bv;
  y = (a - av) + (bv - b);
}
inline void split(double a, double& hi, double& lo) {
  const double c = kSplitter * a;
  const double abig = c - a;
  hi = c - abig;
  lo = a - hi;
}
inline void two_product(double a, double b, double& x, double& y) {
  x = a * b;
  double ahi, alo, bhi, blo;
  split(a, ahi, alo);
  split(b, bhi, blo);
  const double err1 = x - (ahi * bhi);
  const double err2 = err1 - (alo * bhi);
  const double err3 = err2 - (ahi * blo);
  y = (alo * blo) - err3;
}

// h = e + b (grow_expansion_zeroelim); e nonoverlapping, increasing magnitude.
inline int grow(int elen, const double* e, double b, double* h) {
  double q = b, hh;
  int hi = 0;
  for (int i = 0; i < elen; ++i) {
    double qn;
    two_sum(q, e[i], qn, hh);
    q = qn;
    if (hh != 0.0) h[hi++] = hh;
  }
  if (q != 0.0 || hi == 0) h[hi++] = q;
  return hi;
}

// h = e + f  (repeated grow; O(elen*flen) but robust for the small sizes used here)
inline int sum(int elen, const double* e, int flen, const double* f, double* h, double* tmp) {
  int n = elen;
  for (int i = 0; i < elen; ++i) h[i] = e[i];
  for (int j = 0; j < flen; ++j) {
    n = grow(n, h, f[j], tmp);
    for (int i = 0; i < n; ++i) h[i] = tmp[i];
  }
  return n;
}

// h = e * b (scale_expansion_zeroelim)
inline int scale(int elen, const double* e, double b, double* h) {
  double q, hh, product1, product0, sum_;
  int hi = 0;
  two_product(e[0], b, q, hh);
  if (hh != 0.0) h[hi++] = hh;
  for (int i = 1; i < elen; ++i) {
    two_product(e[i], b, product1, product0);
    two_sum(q, product0, sum_, hh);
    if (hh != 0.0) h[hi++] = hh;
    double qn;
    two_sum(product1, sum_, qn, hh);
    q = qn;
    if (hh != 0.0) h[hi++] = hh;
  }
  if (q != 0.0 || hi == 0) h[hi++] = q;
  return hi;
}

// h = e * f
inline int mul(int elen, const double* e, int flen, const double* f, double* h) {
  double part[64], acc[256], tmp[256];
  int alen = 1;
  acc[0] = 0.0;
  for (int j = 0; j < flen; ++j) {
    const int plen = scale(elen, e, f[j], part);
    double out[256];
    alen = sum(alen, acc, plen, part, out, tmp);
    for (int i = 0; i < alen; ++i) acc[i] = out[i];
  }
  for (int i = 0; i < alen; ++i) h[i] = acc[i];
  return alen;
}

inline int sign_of(int n, const double* e) {
  for (int i = n - 1; i >= 0; --i) {
    if (e[i] > 0.0) return 1;
    if (e[i] < 0.0) return -1;
  }
  return 0;
}

inline int neg(int n, const double* e, double* h) {
  for (int i = 0; i < n; ++i) h[i] = -e[i];
  return n;
}

}  // namespace exact

// orient2d(a,b,c) = det[[ax-cx, ay-cy],[bx-cx, by-cy]]; exact sign.
inline int orient2d(double ax, double ay, double bx, double by, double cx, double cy) {
  const double detleft = (ax - cx) * (by - cy);
  const double detright = (ay - cy) * (bx - cx);
  const double det = detleft - detright;
  const double detsum = std::fabs(detleft) + std::fabs(detright);
  const double eps = 1.1102230246251565e-16;  // 2^-53
  const double bound = (3.0 + 16.0 * eps) * eps * detsum;
  if (det > bound) return 1;
  if (-det > bound) return -1;
  using namespace exact;
  double acx[2], acy[2], bcx[2], bcy[2];
  two_diff(ax, cx, acx[1], acx[0]);
  two_diff(ay, cy, acy[1], acy[0]);
  two_diff(bx, cx, bcx[1], bcx[0]);
  two_diff(by, cy, bcy[1], bcy[0]);
  double l[16], r[16], nr[16], s[32], tmp[32];
  const int ll = mul(2, acx, 2, bcy, l);
  const int rl = mul(2, acy, 2, bcx, r);
  neg(rl, r, nr);
  const int sl = sum(ll, l, rl, nr, s, tmp);
  return sign_of(sl, s);
}

// orient3d(a,b,c,d) = det[a-d, b-d, c-d] (Shewchuk's convention); exact sign.
inline int orient3d(V3 a, V3 b, V3 c, V3 d) {
  const double adx = a.x - d.x, bdx = b.x - d.x, cdx = c.x - d.x;
  const double ady = a.y - d.y, bdy = b.y - d.y, cdy = c.y - d.y;
  const double adz = a.z - d.z, bdz = b.z - d.z, cdz = c.z - d.z;
  const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
  const double cdxady = cdx * ady, adxcdy = adx * cdy;
  const double adxbdy = adx * bdy, bdxady = bdx * ady;
  const double det =
      adz * (bdxcdy - cdxbdy) + bdz * (cdxady - adxcdy) + cdz * (adxbdy - bdxady);
  const double perm = (std::fabs(bdxcdy) + std::fabs(cdxbdy)) * std::fabs(adz) +
                      (std::fabs(cdxady) + std::fabs(adxcdy)) * std::fabs(bdz) +
                      (std::fabs(adxbdy) + std::fabs(bdxady)) * std::fabs(cdz);
  const double eps = 1.1102230246251565e-16;
  const double bound = (7.0 + 56.0 * eps) * eps * perm;
  if (det > bound) return 1;
  if (-det > bound) return -1;
  using namespace exact;
  double ax_[2], ay_[2], az_[2], bx_[2], by_[2], bz_[2], cx_[2], cy_[2], cz_[2];
  two_diff(a.x, d.x, ax_[1], ax_[0]);
  two_diff(a.y, d.y, ay_[1], ay_[0]);
  two_diff(a.z, d.z, az_[1], az_[0]);
  two_diff(b.x, d.x, bx_[1], bx_[0]);
  two_diff(b.y, d.y, by_[1], by_[0]);
  two_diff(b.z, d.z, bz_[1], bz_[0]);
  two_diff(c.x, d.x, cx_[1], cx_[0]);
  two_diff(c.y, d.y, cy_[1], cy_[0]);
  two_diff(c.z, d.z, cz_[1], cz_[0]);
  // minor(u,v) = u1*v2 - u2*v1 pieces
  auto minor2 = [](const double* p, const double* q, const double* r, const double* s,
                   double* out) {  // p*q - r*s
    double m1[16], m2[16], nm2[16], tmp[32];
    const int l1 = exact::mul(2, p, 2, q, m1);
    const int l2 = exact::mul(2, r, 2, s, m2);
    exact::neg(l2, m2, nm2);
    return exact::sum(l1, m1, l2, nm2, out, tmp);
  };
  double mA[32], mB[32], mC[32];
  const int la = minor2(bx_, cy_, cx_, by_, mA);  // bdx*cdy - cdx*bdy
  const int lb = minor2(cx_, ay_, ax_, cy_, mB);  // cdx*ady - adx*cdy
  const int lc = minor2(ax_, by_, bx_, ay_, mC);  // adx*bdy - bdx*ady
  double t1[128], t2[128], t3[128], s12[256], s123[256], tmp[256];
  const int l1 = mul(la, mA, 2, az_, t1);
  const int l2 = mul(lb, mB, 2, bz_, t2);
  const int l3 = mul(lc, mC, 2, cz_, t3);
  const int n12 = sum(l1, t1, l2, t2, s12, tmp);
  const int n123 = sum(n12, s12, l3, t3, s123, tmp);
  return sign_of(n123, s123);
}

// ---------------------------------------------------------------------------
// Pinned exponential (SPEC.md:269 t' = 1/(1+exp(-beta(t-1/2)))).  Both sides of the
// parity contract evaluate exp with this exact op sequence so the sigmoid — and
// therefore every DMC vertex and every decision taken on it — is bit-identical:
//   k = floor(x*log2(e) + 1/2);  r = (x - k*LN2_HI) - k*LN2_LO;
//   p = 1 + r + r^2/2! + ... + r^13/13!   (Horner, reciprocal-factorial constants)
//   exp(x) = p * 2^k   (2^k assembled from bits; two steps when k < -1022)
inline double pow2i(int k) {
  // k in [-1022, 1023]
  const uint64_t bits = static_cast<uint64_t>(k + 1023) << 52;
  double r;
  std::memcpy(&r, &bits, 8);
  return r;
}

inline double det_exp(double x) {
  if (x != x) return x;
  if (x > 709.0) return std::numeric_limits<double>::infinity();
  if (x < -745.0) return 0.0;
  const double kLog2e = 1.4426950408889634;
  const double kLn2Hi = 6.93147180369123816490e-01;
  const double kLn2Lo = 1.90821492927058770002e-10;
  const double kd = std::floor(x * kLog2e + 0.5);
  const int k = static_cast<int>(kd);
  const double r = (x - kd * kLn2Hi) - kd * kLn2Lo;
  static const double c[14] = {1.0,
                               1.0,
                               0.5,
                               1.6666666666666666e-01,
                               4.1666666666666664e-02,
                               8.3333333333333332e-03,
                               1.3888888888888889e-03,
                               1.9841269841269841e-04,
                               2.4801587301587302e-05,
                               2.7557319223985893e-06,
                               2.7557319223985888e-07,
                               2.5052108385441720e-08,
                               2.0876756987868100e-09,
                               1.6059043836821613e-10};
  double p = c[13];
  for (int i = 12; i >= 0; --i) p = p * r + c[i];
  if (k >= -1022) return p * pow2i(k);
  return (p * pow2i(k + 600)) * pow2i(-600);
}

inline double sigmoid_t(double t, double beta) {
  return 1.0 / (1.0 + det_exp(-beta * (t - 0.5)));
}

}  // namespace orc
