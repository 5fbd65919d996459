// Small host geometry / quadrature / polynomial toolkit for the setup code.
// Operation order follows the reference primitives so derived operator data
// is bitwise comparable: Vec2 and polygon formulas (include/ucfv/geometry.hpp),
// Gauss-Legendre by Newton on P_n (src/quadrature.cpp:9-39), Duffy-collapsed
// triangle rules (quadrature.cpp:45-64) and polygon splitting (:68-91).
#pragma once

#include <cmath>
#include <vector>

namespace ucfvb {

struct Vec2 {
  double x = 0.0, y = 0.0;
  Vec2() = default;
  Vec2(double a, double b) : x(a), y(b) {}
  Vec2 operator+(const Vec2& o) const { return {x + o.x, y + o.y}; }
  Vec2 operator-(const Vec2& o) const { return {x - o.x, y - o.y}; }
  Vec2 operator*(double s) const { return {x * s, y * s}; }
  Vec2 operator/(double s) const { return {x / s, y / s}; }
};
inline Vec2 operator*(double s, const Vec2& v) { return v * s; }
inline double cross(const Vec2& a, const Vec2& b) { return a.x * b.y - a.y * b.x; }
inline double norm(const Vec2& v) { return std::sqrt(v.x * v.x + v.y * v.y); }

inline double polygon_signed_area(const std::vector<Vec2>& p) {
  double a = 0.0;
  const size_t n = p.size();
  for (size_t i = 0; i < n; ++i) a += cross(p[i], p[(i + 1) % n]);
  return 0.5 * a;
}

inline Vec2 polygon_centroid(const std::vector<Vec2>& p) {
  double a = 0.0;
  Vec2 c;
  const size_t n = p.size();
  for (size_t i = 0; i < n; ++i) {
    const Vec2& u = p[i];
    const Vec2& v = p[(i + 1) % n];
    const double w = cross(u, v);
    a += w;
    c = c + (u + v) * w;
  }
  return c / (3.0 * a);
}

struct GaussRule {
  std::vector<double> nodes, weights;
};

// n-point Gauss-Legendre rule on [-1, 1]
inline GaussRule gauss_legendre(int n) {
  GaussRule r;
  r.nodes.assign(n, 0.0);
  r.weights.assign(n, 0.0);
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dpn = 0.0;
    for (int it = 0; it < 100; ++it) {
      double pn = 1.0, pm = 0.0;
      for (int j = 0; j < n; ++j) {
        const double pmm = pm;
        pm = pn;
        pn = ((2.0 * j + 1.0) * x * pm - j * pmm) / (j + 1.0);
      }
      dpn = n * (x * pn - pm) / (x * x - 1.0);
      const double step = pn / dpn;
      x -= step;
      if (std::abs(step) < 1e-15) break;
    }
    r.nodes[i] = -x;
    r.nodes[n - 1 - i] = x;
    const double w = 2.0 / ((1.0 - x * x) * dpn * dpn);
    r.weights[i] = w;
    r.weights[n - 1 - i] = w;
  }
  return r;
}

struct QPoint {
  Vec2 p;
  double w;
};

// collapsed (Duffy) tensor rule on triangle (a, b, c), exact to total degree `degree`
inline void triangle_rule(const Vec2& a, const Vec2& b, const Vec2& c, int degree, std::vector<QPoint>& out) {
  const int n = (degree + 3) / 2;
  static thread_local int cached_n = -1;
  static thread_local GaussRule g;
  if (cached_n != n) {
    g = gauss_legendre(n);
    cached_n = n;
  }
  const double area2 = cross(b - a, c - a);
  for (int i = 0; i < n; ++i) {
    const double u = 0.5 * (g.nodes[i] + 1.0);
    for (int j = 0; j < n; ++j) {
      const double v = 0.5 * (g.nodes[j] + 1.0);
      const double t = v * (1.0 - u);
      const Vec2 p = a + u * (b - a) + t * (c - a);
      const double jac = 0.25 * (1.0 - u);
      out.push_back({p, g.weights[i] * g.weights[j] * jac * area2});
    }
  }
}

inline void polygon_rule(const std::vector<Vec2>& poly, int degree, std::vector<QPoint>& out) {
  out.clear();
  if (degree < 0) degree = 0;
  if (poly.size() == 3) {
    triangle_rule(poly[0], poly[1], poly[2], degree, out);
  } else if (poly.size() == 4) {
    const double a0 = cross(poly[1] - poly[0], poly[2] - poly[0]);
    const double a1 = cross(poly[2] - poly[0], poly[3] - poly[0]);
    if (a0 > 0.0 && a1 > 0.0) {
      triangle_rule(poly[0], poly[1], poly[2], degree, out);
      triangle_rule(poly[0], poly[2], poly[3], degree, out);
    } else {
      triangle_rule(poly[1], poly[2], poly[3], degree, out);
      triangle_rule(poly[1], poly[3], poly[0], degree, out);
    }
  } else {
    const Vec2 c = polygon_centroid(poly);
    for (size_t i = 0; i < poly.size(); ++i) triangle_rule(c, poly[i], poly[(i + 1) % poly.size()], degree, out);
  }
}

}  // namespace ucfvb
