// ad.cuh — forward-mode second-order automatic differentiation for the stage-3 energy stencils
// (SPEC.md safe_project; Appendix 2.2).  J2<N> carries a value, its gradient and its
// symmetric Hessian with respect to N stencil coordinates (only the upper triangle h[i][j],
// j >= i, is propagated; read it through hess()), so every term's gradient and Hessian block
// are exact derivatives of one closed-form expression.  The same templates
// instantiated on `double` give value-only evaluations (line search).
#pragma once

#include <cmath>

namespace pcu {
namespace ad {

template <int N>
struct J2 {
  double v;
  double g[N];
  double h[N][N];
  __host__ __device__ J2() : v(0.0) {
    #pragma unroll 1
  for (int i = 0; i < N; ++i) {
      g[i] = 0.0;
      for (int j = i; j < N; ++j) h[i][j] = 0.0;
    }
  }
  __host__ __device__ J2(double c) : v(c) {  // NOLINT: constants promote implicitly
    #pragma unroll 1
  for (int i = 0; i < N; ++i) {
      g[i] = 0.0;
      for (int j = i; j < N; ++j) h[i][j] = 0.0;
    }
  }
  __host__ __device__ static J2 var(int i, double x) {
    J2 r(x);
    r.g[i] = 1.0;
    return r;
  }
};

template <int N>
__host__ __device__ inline J2<N> operator+(const J2<N>& a, const J2<N>& b) {
  J2<N> r;
  r.v = a.v + b.v;
  #pragma unroll 1
  for (int i = 0; i < N; ++i) {
    r.g[i] = a.g[i] + b.g[i];
    for (int j = i; j < N; ++j) r.h[i][j] = a.h[i][j] + b.h[i][j];
  }
  return r;
}
template <int N>
__host__ __device__ inline J2<N> operator-(const J2<N>& a, const J2<N>& b) {
  J2<N> r;
  r.v = a.v - b.v;
  #pragma unroll 1
  for (int i = 0; i < N; ++i) {
    r.g[i] = a.g[i] - b.g[i];
    for (int j = i; j < N; ++j) r.h[i][j] = a.h[i][j] - b.h[i][j];
  }
  return r;
}
template <int N>
__host__ __device__ inline J2<N> operator-(const J2<N>& a) {
  J2<N> r;
  r.v = -a.v;
  #pragma unroll 1
  for (int i = 0; i < N; ++i) {
    r.g[i] = -a.g[i];
    for (int j = i; j < N; ++j) r.h[i][j] = -a.h[i][j];
  }
  return r;
}
template <int N>
__host__ __device__ inline J2<N> operator*(const J2<N>& a, const J2<N>& b) {
  J2<N> r;
  r.v = a.v * b.v;
  #pragma unroll 1
  for (int i = 0; i < N; ++i) {
    r.g[i] = a.v * b.g[i] + b.v * a.g[i];
    for (int j = i; j < N; ++j)
      r.h[i][j] = a.v * b.h[i][j] + b.v * a.h[i][j] + a.g[i] * b.g[j] + b.g[i] * a.g[j];
  }
  return r;
}
template <int N>
__host__ __device__ inline J2<N> operator*(double c, const J2<N>& a) {
  J2<N> r;
  r.v = c * a.v;
  #pragma unroll 1
  for (int i = 0; i < N; ++i) {
    r.g[i] = c * a.g[i];
    for (int j = i; j < N; ++j) r.h[i][j] = c * a.h[i][j];
  }
  return r;
}
template <int N>
__host__ __device__ inline J2<N> operator*(const J2<N>& a, double c) {
  return c * a;
}
template <int N>
__host__ __device__ inline J2<N> operator+(const J2<N>& a, double c) {
  J2<N> r = a;
  r.v += c;
  return r;
}
template <int N>
__host__ __device__ inline J2<N> operator-(const J2<N>& a, double c) {
  J2<N> r = a;
  r.v -= c;
  return r;
}
template <int N>
__host__ __device__ inline J2<N> operator-(double c, const J2<N>& a) {
  return (-a) + c;
}

// f(a) with f' = d1, f'' = d2 at a.v
template <int N>
__host__ __device__ inline J2<N> chain(const J2<N>& a, double f, double d1, double d2) {
  J2<N> r;
  r.v = f;
  #pragma unroll 1
  for (int i = 0; i < N; ++i) {
    r.g[i] = d1 * a.g[i];
    for (int j = i; j < N; ++j) r.h[i][j] = d1 * a.h[i][j] + d2 * a.g[i] * a.g[j];
  }
  return r;
}
template <int N>
__host__ __device__ inline J2<N> recip(const J2<N>& a) {
  const double inv = 1.0 / a.v;
  return chain(a, inv, -inv * inv, 2.0 * inv * inv * inv);
}
template <int N>
__host__ __device__ inline J2<N> operator/(const J2<N>& a, const J2<N>& b) {
  return a * recip(b);
}
template <int N>
__host__ __device__ inline J2<N> operator/(const J2<N>& a, double c) {
  return (1.0 / c) * a;
}
template <int N>
__host__ __device__ inline J2<N> sqrt(const J2<N>& a) {
  const double s = ::sqrt(a.v);
  return chain(a, s, 0.5 / s, -0.25 / (s * a.v));
}
template <int N>
__host__ __device__ inline J2<N> log(const J2<N>& a) {
  return chain(a, ::log(a.v), 1.0 / a.v, -1.0 / (a.v * a.v));
}
// atan2(y, x) as a function of two jets
template <int N>
__host__ __device__ inline J2<N> atan2(const J2<N>& y, const J2<N>& x) {
  const double r2 = x.v * x.v + y.v * y.v, r4 = r2 * r2;
  const double fy = x.v / r2, fx = -y.v / r2;
  const double fyy = -2.0 * x.v * y.v / r4, fxx = 2.0 * x.v * y.v / r4, fxy = (y.v * y.v - x.v * x.v) / r4;
  J2<N> r;
  r.v = ::atan2(y.v, x.v);
  #pragma unroll 1
  for (int i = 0; i < N; ++i) {
    r.g[i] = fy * y.g[i] + fx * x.g[i];
    for (int j = i; j < N; ++j)
      r.h[i][j] = fy * y.h[i][j] + fx * x.h[i][j] + fyy * y.g[i] * y.g[j] + fxx * x.g[i] * x.g[j] +
                  fxy * (y.g[i] * x.g[j] + x.g[i] * y.g[j]);
  }
  return r;
}

// double overloads: the same templates evaluate values only
__host__ __device__ inline double sqrt(double a) { return ::sqrt(a); }
__host__ __device__ inline double log(double a) { return ::log(a); }
__host__ __device__ inline double atan2(double y, double x) { return ::atan2(y, x); }

template <int N>
__host__ __device__ inline double hess(const J2<N>& a, int i, int j) {
  return i <= j ? a.h[i][j] : a.h[j][i];
}

__host__ __device__ inline double value(double a) { return a; }
template <int N>
__host__ __device__ inline double value(const J2<N>& a) {
  return a.v;
}

// 3-vectors of a scalar type
template <class T>
struct V {
  T x, y, z;
};
template <class T>
__host__ __device__ inline V<T> operator-(const V<T>& a, const V<T>& b) {
  return V<T>{a.x - b.x, a.y - b.y, a.z - b.z};
}
template <class T>
__host__ __device__ inline V<T> operator+(const V<T>& a, const V<T>& b) {
  return V<T>{a.x + b.x, a.y + b.y, a.z + b.z};
}
template <class T>
__host__ __device__ inline T dot(const V<T>& a, const V<T>& b) {
  return (a.x * b.x + a.y * b.y) + a.z * b.z;
}
template <class T>
__host__ __device__ inline V<T> cross(const V<T>& a, const V<T>& b) {
  return V<T>{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class T>
__host__ __device__ inline V<T> scale(const T& s, const V<T>& a) {
  return V<T>{s * a.x, s * a.y, s * a.z};
}

}  // namespace ad
}  // namespace pcu
