// exact.cuh — exact orientation predicates for the self-intersection narrow phase.
//
// Fast path: the double-precision determinant with Shewchuk's static error bound (certifies the
// sign for all but near-degenerate inputs).  Slow path (rare): exact evaluation with
// floating-point expansions (Dekker two-product, no FMA needed) so every verdict of the
// narrow phase is exact and therefore identical on every device (0% FNR).
#pragma once

#include "common.cuh"

namespace pcu {
namespace xp {

__device__ __forceinline__ void two_sum(double a, double b, double& x, double& y) {
  x = a + b;
  const double bv = x - a;
  const double av = x - bv;
  y = (a - av) + (b - bv);
}
__device__ __forceinline__ void two_diff(double a, double b, double& x, double& y) {
  x = a - b;
  const double bv = a - x;
  const double av = x + bv;
  y = (a - av) + (bv - b);
}
__device__ __forceinline__ void two_prod(double a, double b, double& x, double& y) {
  x = a * b;
  const double ca = 134217729.0 * a, cb = 134217729.0 * b;
  const double ahi = ca - (ca - a), alo = a - ahi;
  const double bhi = cb - (cb - b), blo = b - bhi;
  const double e1 = x - (ahi * bhi);
  const double e2 = e1 - (alo * bhi);
  const double e3 = e2 - (ahi * blo);
  y = (alo * blo) - e3;
}

// h <- e + b  (zero-eliminating grow); returns new length.  h may alias e.
__device__ inline int grow(int elen, double* e, double b) {
  double q = b;
  int hi = 0;
  for (int i = 0; i < elen; ++i) {
    double s, err;
    two_sum(q, e[i], s, err);
    q = s;
    if (err != 0.0) e[hi++] = err;
  }
  if (q != 0.0 || hi == 0) e[hi++] = q;
  return hi;
}

// acc += e * b
__device__ inline int acc_scale(int alen, double* acc, int elen, const double* e, double b) {
  for (int i = 0; i < elen; ++i) {
    double p1, p0;
    two_prod(e[i], b, p1, p0);
    alen = grow(alen, acc, p0);
    alen = grow(alen, acc, p1);
  }
  return alen;
}

__device__ inline int sign_of(int n, const double* e) {
  for (int i = n - 1; i >= 0; --i) {
    if (e[i] > 0.0) return 1;
    if (e[i] < 0.0) return -1;
  }
  return 0;
}

// out = p*q - r*s for 2-term expansions (length <= 16)
__device__ inline int minor2(const double* p, const double* q, const double* r, const double* s, double* out) {
  int n = 1;
  out[0] = 0.0;
  for (int j = 0; j < 2; ++j) n = acc_scale(n, out, 2, p, q[j]);
  double nr[2] = {-r[0], -r[1]};
  for (int j = 0; j < 2; ++j) n = acc_scale(n, out, 2, nr, s[j]);
  return n;
}

}  // namespace xp

__device__ inline int orient2d_exact(double ax, double ay, double bx, double by, double cx, double cy) {
  double acx[2], acy[2], bcx[2], bcy[2];
  xp::two_diff(ax, cx, acx[1], acx[0]);
  xp::two_diff(ay, cy, acy[1], acy[0]);
  xp::two_diff(bx, cx, bcx[1], bcx[0]);
  xp::two_diff(by, cy, bcy[1], bcy[0]);
  double m[40];
  const int n = xp::minor2(acx, bcy, acy, bcx, m);
  return xp::sign_of(n, m);
}

// orient2d(a,b,c) = sign det[[ax-cx, ay-cy],[bx-cx, by-cy]]
__device__ __forceinline__ int orient2d(double ax, double ay, double bx, double by, double cx, double cy) {
  const double detleft = (ax - cx) * (by - cy);
  const double detright = (ay - cy) * (bx - cx);
  const double det = detleft - detright;
  const double detsum = fabs(detleft) + fabs(detright);
  const double bound = (3.0 + 16.0 * 1.1102230246251565e-16) * 1.1102230246251565e-16 * detsum;
  if (det > bound) return 1;
  if (-det > bound) return -1;
  return orient2d_exact(ax, ay, bx, by, cx, cy);
}

__device__ __noinline__ int orient3d_exact(D3 a, D3 b, D3 c, D3 d) {
  double ax[2], ay[2], az[2], bx[2], by[2], bz[2], cx[2], cy[2], cz[2];
  xp::two_diff(a.x, d.x, ax[1], ax[0]);
  xp::two_diff(a.y, d.y, ay[1], ay[0]);
  xp::two_diff(a.z, d.z, az[1], az[0]);
  xp::two_diff(b.x, d.x, bx[1], bx[0]);
  xp::two_diff(b.y, d.y, by[1], by[0]);
  xp::two_diff(b.z, d.z, bz[1], bz[0]);
  xp::two_diff(c.x, d.x, cx[1], cx[0]);
  xp::two_diff(c.y, d.y, cy[1], cy[0]);
  xp::two_diff(c.z, d.z, cz[1], cz[0]);
  double m[40];
  double acc[400];
  int an = 1;
  acc[0] = 0.0;
  int mn = xp::minor2(bx, cy, cx, by, m);  // bdx*cdy - cdx*bdy, times adz
  for (int j = 0; j < 2; ++j) an = xp::acc_scale(an, acc, mn, m, az[j]);
  mn = xp::minor2(cx, ay, ax, cy, m);      // cdx*ady - adx*cdy, times bdz
  for (int j = 0; j < 2; ++j) an = xp::acc_scale(an, acc, mn, m, bz[j]);
  mn = xp::minor2(ax, by, bx, ay, m);      // adx*bdy - bdx*ady, times cdz
  for (int j = 0; j < 2; ++j) an = xp::acc_scale(an, acc, mn, m, cz[j]);
  return xp::sign_of(an, acc);
}

// The certified part of orient3d: the sign where the floating-point filter (or coincident
// points) decides it, else 2.  Kernels that call only this carry none of the expansion
// arithmetic's registers.
__device__ __forceinline__ int orient3d_filtered(D3 a, D3 b, D3 c, D3 d) {
  const double adx = a.x - d.x, bdx = b.x - d.x, cdx = c.x - d.x;
  const double ady = a.y - d.y, bdy = b.y - d.y, cdy = c.y - d.y;
  const double adz = a.z - d.z, bdz = b.z - d.z, cdz = c.z - d.z;
  const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
  const double cdxady = cdx * ady, adxcdy = adx * cdy;
  const double adxbdy = adx * bdy, bdxady = bdx * ady;
  const double det = adz * (bdxcdy - cdxbdy) + bdz * (cdxady - adxcdy) + cdz * (adxbdy - bdxady);
  const double perm = (fabs(bdxcdy) + fabs(cdxbdy)) * fabs(adz) + (fabs(cdxady) + fabs(adxcdy)) * fabs(bdz) +
                      (fabs(adxbdy) + fabs(bdxady)) * fabs(cdz);
  const double bound = (7.0 + 56.0 * 1.1102230246251565e-16) * 1.1102230246251565e-16 * perm;
  if (det > bound) return 1;
  if (-det > bound) return -1;
  auto same = [](D3 p, D3 q) { return p.x == q.x && p.y == q.y && p.z == q.z; };
  if (same(a, b) || same(a, c) || same(a, d) || same(b, c) || same(b, d) || same(c, d)) return 0;
  return 2;
}

// orient3d(a,b,c,d) = sign det[a-d, b-d, c-d]
__device__ __forceinline__ int orient3d(D3 a, D3 b, D3 c, D3 d) {
  const double adx = a.x - d.x, bdx = b.x - d.x, cdx = c.x - d.x;
  const double ady = a.y - d.y, bdy = b.y - d.y, cdy = c.y - d.y;
  const double adz = a.z - d.z, bdz = b.z - d.z, cdz = c.z - d.z;
  const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
  const double cdxady = cdx * ady, adxcdy = adx * cdy;
  const double adxbdy = adx * bdy, bdxady = bdx * ady;
  const double det = adz * (bdxcdy - cdxbdy) + bdz * (cdxady - adxcdy) + cdz * (adxbdy - bdxady);
  const double perm = (fabs(bdxcdy) + fabs(cdxbdy)) * fabs(adz) + (fabs(cdxady) + fabs(adxcdy)) * fabs(bdz) +
                      (fabs(adxbdy) + fabs(bdxady)) * fabs(cdz);
  const double bound = (7.0 + 56.0 * 1.1102230246251565e-16) * 1.1102230246251565e-16 * perm;
  if (det > bound) return 1;
  if (-det > bound) return -1;
  // coincident points give an exact zero without the expansion arithmetic
  auto same = [](D3 p, D3 q) { return p.x == q.x && p.y == q.y && p.z == q.z; };
  if (same(a, b) || same(a, c) || same(a, d) || same(b, c) || same(b, d) || same(c, d)) return 0;
  return orient3d_exact(a, b, c, d);
}

}  // namespace pcu
