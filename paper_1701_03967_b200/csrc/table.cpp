// Host spectral-table builder.  See table.hpp for the reference citations.
// All routines are written for double only (the runtime precision of the
// reference, types.hpp:20-23); loop orders follow the reference's small dense
// kit so the resulting tables agree with it to the last bit in practice
// (checked by tests/test_gpu_parity.py::test_table_matches_reference).
#include "table.hpp"

#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <atomic>

#include <unistd.h>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <utility>

namespace sfem_b200 {
namespace {

[[noreturn]] void fail(const std::string& msg) { throw std::runtime_error(msg); }

struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rr, int cc) : r(rr), c(cc), a(static_cast<size_t>(rr) * cc, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) * c + j]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) * c + j]; }
};

Mat matmul(const Mat& x, const Mat& y) {
  Mat z(x.r, y.c);
  for (int i = 0; i < x.r; ++i)
    for (int k = 0; k < x.c; ++k) {
      const double xik = x(i, k);
      for (int j = 0; j < y.c; ++j) z(i, j) += xik * y(k, j);
    }
  return z;
}

Mat transpose(const Mat& x) {
  Mat z(x.c, x.r);
  for (int i = 0; i < x.r; ++i)
    for (int j = 0; j < x.c; ++j) z(j, i) = x(i, j);
  return z;
}

double dot(const std::vector<double>& x, const std::vector<double>& y) {
  double s = 0;
  for (size_t i = 0; i < x.size(); ++i) s += x[i] * y[i];
  return s;
}

// ---- quadrature / Lagrange (quadrature.hpp:18-74, lagrange.hpp:11-47) ----
void legendre_eval(int m, double x, double& p, double& dp) {
  double p0 = 1, p1 = x;
  if (m == 0) {
    p = p0;
    dp = 0;
    return;
  }
  for (int k = 2; k <= m; ++k) {
    const double pk = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    p0 = p1;
    p1 = pk;
  }
  p = p1;
  dp = m * (x * p1 - p0) / (x * x - 1.0);
}

void gauss_legendre(int m, std::vector<double>& nodes, std::vector<double>& weights) {
  nodes.assign(m, 0.0);
  weights.assign(m, 0.0);
  const double eps = std::numeric_limits<double>::epsilon();
  const int half = m / 2;
  for (int i = 0; i < half; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (m + 0.5));
    double p, dp;
    for (int it = 0; it < 200; ++it) {
      legendre_eval(m, x, p, dp);
      const double dx = p / dp;
      x -= dx;
      if (std::abs(dx) <= 2 * eps * (1 + std::abs(x))) break;
    }
    legendre_eval(m, x, p, dp);
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    nodes[m - 1 - i] = x;
    nodes[i] = -x;
    weights[i] = w;
    weights[m - 1 - i] = w;
  }
  if (m % 2 == 1) {
    double p, dp;
    legendre_eval(m, 0.0, p, dp);
    nodes[half] = 0.0;
    weights[half] = 2.0 / (dp * dp);
  }
}

double lagrange_value(const std::vector<double>& nodes, int l, double x) {
  double v = 1;
  for (size_t m = 0; m < nodes.size(); ++m) {
    if (static_cast<int>(m) == l) continue;
    v *= (x - nodes[m]) / (nodes[l] - nodes[m]);
  }
  return v;
}

double lagrange_derivative(const std::vector<double>& nodes, int l, double x) {
  double sum = 0, denom = 1;
  for (size_t m = 0; m < nodes.size(); ++m) {
    if (static_cast<int>(m) == l) continue;
    denom *= nodes[l] - nodes[m];
    double term = 1;
    for (size_t r = 0; r < nodes.size(); ++r) {
      if (static_cast<int>(r) == l || r == m) continue;
      term *= x - nodes[r];
    }
    sum += term;
  }
  return sum / denom;
}

// ---- dense eigen kit (smallmat.hpp:72-214) ----
Mat cholesky_lower(const Mat& m) {
  const int n = m.r;
  Mat l(n, n);
  for (int j = 0; j < n; ++j) {
    double d = m(j, j);
    for (int k = 0; k < j; ++k) d -= l(j, k) * l(j, k);
    if (!(d > 0)) fail("cholesky: matrix not positive definite");
    l(j, j) = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double s = m(i, j);
      for (int k = 0; k < j; ++k) s -= l(i, k) * l(j, k);
      l(i, j) = s / l(j, j);
    }
  }
  return l;
}

std::vector<double> solve_lower(const Mat& l, std::vector<double> b) {
  for (int i = 0; i < l.r; ++i) {
    for (int k = 0; k < i; ++k) b[i] -= l(i, k) * b[k];
    b[i] /= l(i, i);
  }
  return b;
}

std::vector<double> solve_lower_transposed(const Mat& l, std::vector<double> b) {
  for (int i = l.r - 1; i >= 0; --i) {
    for (int k = i + 1; k < l.r; ++k) b[i] -= l(k, i) * b[k];
    b[i] /= l(i, i);
  }
  return b;
}

void jacobi_eigensymm(Mat m, std::vector<double>& values, Mat& vecs) {
  const int n = m.r;
  vecs = Mat(n, n);
  for (int i = 0; i < n; ++i) vecs(i, i) = 1;
  values.assign(n, 0.0);
  if (n == 0) return;
  const double eps = std::numeric_limits<double>::epsilon();
  for (int sweep = 0; sweep < 128; ++sweep) {
    double off = 0, diag = 0;
    for (int i = 0; i < n; ++i) {
      diag += std::abs(m(i, i));
      for (int j = i + 1; j < n; ++j) off += std::abs(m(i, j));
    }
    if (!(off > eps * (diag + off))) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = m(p, q);
        if (std::abs(apq) <= eps * eps * (std::abs(m(p, p)) + std::abs(m(q, q)))) continue;
        const double tau = (m(q, q) - m(p, p)) / (2 * apq);
        const double t = tau >= 0 ? 1.0 / (tau + std::sqrt(1.0 + tau * tau))
                                  : -1.0 / (-tau + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double mkp = m(k, p), mkq = m(k, q);
          m(k, p) = c * mkp - s * mkq;
          m(k, q) = s * mkp + c * mkq;
        }
        for (int k = 0; k < n; ++k) {
          const double mpk = m(p, k), mqk = m(q, k);
          m(p, k) = c * mpk - s * mqk;
          m(q, k) = s * mpk + c * mqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = vecs(k, p), vkq = vecs(k, q);
          vecs(k, p) = c * vkp - s * vkq;
          vecs(k, q) = s * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < n; ++i) values[i] = m(i, i);
}

void pencil_eigensymm(const Mat& a, const Mat& b, std::vector<double>& values, Mat& vecs) {
  const int n = a.r;
  values.assign(n, 0.0);
  vecs = Mat(n, n);
  if (n == 0) return;
  const Mat l = cholesky_lower(b);
  Mat m(n, n);
  for (int j = 0; j < n; ++j) {
    std::vector<double> col(n);
    for (int i = 0; i < n; ++i) col[i] = a(i, j);
    col = solve_lower(l, std::move(col));
    for (int i = 0; i < n; ++i) m(i, j) = col[i];
  }
  for (int i = 0; i < n; ++i) {
    std::vector<double> row(n);
    for (int j = 0; j < n; ++j) row[j] = m(i, j);
    row = solve_lower(l, std::move(row));
    for (int j = 0; j < n; ++j) m(i, j) = row[j];
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const double v = (m(i, j) + m(j, i)) / 2;
      m(i, j) = v;
      m(j, i) = v;
    }
  std::vector<double> w;
  Mat y;
  jacobi_eigensymm(std::move(m), w, y);
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int x, int z) { return w[x] < w[z]; });
  for (int j = 0; j < n; ++j) {
    std::vector<double> col(n);
    for (int i = 0; i < n; ++i) col[i] = y(i, order[j]);
    col = solve_lower_transposed(l, std::move(col));
    for (int i = 0; i < n; ++i) vecs(i, j) = col[i];
    values[j] = w[order[j]];
  }
}

// ---- element (element.hpp:85-347) ----
void symmetrize_bisymmetric(Mat& m) {
  const int n = m.r - 1;
  for (int i = 0; i <= n; ++i)
    for (int j = i; j <= n; ++j) {
      const double v = (m(i, j) + m(j, i)) / 2;
      m(i, j) = v;
      m(j, i) = v;
    }
  for (int i = 0; i <= n; ++i)
    for (int j = 0; j <= n; ++j) {
      const int fi = n - i, fj = n - j;
      if (std::make_pair(fi, fj) > std::make_pair(i, j)) m(fi, fj) = m(i, j);
    }
}

struct Blocks {
  double corner = 0, cross = 0;
  std::vector<double> edge, edge_rev;
  Mat interior;
};

Blocks carve(const Mat& m) {
  const int n = m.r - 1;
  Blocks b;
  b.corner = m(0, 0);
  b.cross = m(0, n);
  const int mm = n - 1 > 0 ? n - 1 : 0;
  b.edge.resize(mm);
  b.edge_rev.resize(mm);
  b.interior = Mat(mm, mm);
  for (int i = 1; i < n; ++i) {
    b.edge[i - 1] = m(i, 0);
    b.edge_rev[i - 1] = m(i, n);
    for (int j = 1; j < n; ++j) b.interior(i - 1, j - 1) = m(i, j);
  }
  return b;
}

Mat parity_basis(int m, int sign) {
  const int half = m / 2;
  const int dim = sign > 0 ? (m + 1) / 2 : m / 2;
  Mat u(m, dim);
  const double r = 1.0 / std::sqrt(2.0);
  for (int i = 0; i < half; ++i) {
    u(i, i) = r;
    u(m - 1 - i, i) = sign > 0 ? r : -r;
  }
  if (sign > 0 && m % 2 == 1) u(half, dim - 1) = 1;
  return u;
}

void parity_pencil_eig(const Mat& a, const Mat& b, std::vector<double>& values, Mat& vecs,
                       std::vector<int>& parity) {
  const int m = a.r;
  values.assign(m, 0.0);
  vecs = Mat(m, m);
  parity.assign(m, 0);
  if (m == 0) return;
  struct Pair {
    double value;
    std::vector<double> vec;
    int parity;
  };
  std::vector<Pair> pairs;
  for (int sign : {+1, -1}) {
    const Mat u = parity_basis(m, sign);
    if (u.c == 0) continue;
    const Mat ut = transpose(u);
    const Mat ar = matmul(ut, matmul(a, u));
    const Mat br = matmul(ut, matmul(b, u));
    std::vector<double> w;
    Mat y;
    pencil_eigensymm(ar, br, w, y);
    for (int j = 0; j < u.c; ++j) {
      Pair p;
      p.value = w[j];
      p.parity = sign;
      p.vec.assign(m, 0.0);
      for (int i = 0; i < m; ++i) {
        double s = 0;
        for (int k = 0; k < u.c; ++k) s += u(i, k) * y(k, j);
        p.vec[i] = s;
      }
      pairs.push_back(std::move(p));
    }
  }
  std::sort(pairs.begin(), pairs.end(), [](const Pair& x, const Pair& y) { return x.value < y.value; });
  for (int j = 0; j < m; ++j) {
    double peak = 0;
    for (double v : pairs[j].vec) peak = std::max(peak, std::abs(v));
    for (int i = 0; i < m; ++i)
      if (std::abs(pairs[j].vec[i]) > peak / 1048576.0) {
        if (pairs[j].vec[i] < 0)
          for (double& v : pairs[j].vec) v = -v;
        break;
      }
    values[j] = pairs[j].value;
    parity[j] = pairs[j].parity;
    for (int i = 0; i < m; ++i) vecs(i, j) = pairs[j].vec[i];
  }
}

struct Element {
  int n = 0;
  Mat stiffness, mass;
  Blocks sb, mb;
};

Element build_element(int n) {
  if (n < 1 || n > 9)
    fail("build_element_matrices: order " + std::to_string(n) + " outside [1, 9]");
  std::vector<double> nodes(n + 1);
  for (int k = 0; k <= n; ++k) nodes[k] = static_cast<double>(2 * k - n) / static_cast<double>(n);
  std::vector<double> gn, gw;
  gauss_legendre(n + 1, gn, gw);
  Mat vals(n + 1, n + 1), ders(n + 1, n + 1);
  for (int l = 0; l <= n; ++l)
    for (int g = 0; g <= n; ++g) {
      vals(l, g) = lagrange_value(nodes, l, gn[g]);
      ders(l, g) = lagrange_derivative(nodes, l, gn[g]);
    }
  Element em;
  em.n = n;
  em.stiffness = Mat(n + 1, n + 1);
  em.mass = Mat(n + 1, n + 1);
  for (int k = 0; k <= n; ++k)
    for (int l = 0; l <= n; ++l) {
      double sa = 0, sc = 0;
      for (int g = 0; g <= n; ++g) {
        sa += gw[g] * ders(k, g) * ders(l, g);
        sc += gw[g] * vals(k, g) * vals(l, g);
      }
      em.stiffness(k, l) = sa;
      em.mass(k, l) = sc;
    }
  symmetrize_bisymmetric(em.stiffness);
  symmetrize_bisymmetric(em.mass);
  em.sb = carve(em.stiffness);
  em.mb = carve(em.mass);
  return em;
}

struct Interior {
  std::vector<double> values;
  Mat vectors;
  std::vector<int> parity;
  std::vector<double> edge_stiff, edge_mass;
};

Interior interior_eigensystem(const Element& em) {
  const int m = em.n - 1;
  Interior es;
  parity_pencil_eig(em.sb.interior, em.mb.interior, es.values, es.vectors, es.parity);
  for (int j = 0; j + 1 < m; ++j) {
    const double gap = es.values[j + 1] - es.values[j];
    if (!(gap > 1e-12 * (1 + std::abs(es.values[j + 1]))))
      fail("interior_eigensystem: eigenvalue multiplicity between l=" + std::to_string(j + 1) +
           " and l=" + std::to_string(j + 2) + " at order " + std::to_string(em.n));
  }
  es.edge_stiff.resize(m);
  es.edge_mass.resize(m);
  for (int l = 0; l < m; ++l) {
    std::vector<double> e(m);
    for (int i = 0; i < m; ++i) e[i] = es.vectors(i, l);
    es.edge_stiff[l] = dot(em.sb.edge, e);
    es.edge_mass[l] = dot(em.mb.edge, e);
  }
  return es;
}

// ---- theta equation (spectral.hpp:26-193) ----
struct ThetaEq {
  double affine_a, affine_b;
  std::vector<double> pole, coef, num_a, num_c;
  ThetaEq(const Interior& es, const Element& em, double theta) {
    affine_a = em.sb.corner + theta * em.sb.cross;
    affine_b = em.mb.corner + theta * em.mb.cross;
    const int m = em.n - 1;
    for (int l = 0; l < m; ++l) {
      pole.push_back(es.values[l]);
      coef.push_back(1.0 + theta * static_cast<double>(es.parity[l]));
      num_a.push_back(es.edge_stiff[l]);
      num_c.push_back(es.edge_mass[l]);
    }
  }
  double value(double x) const {
    double s = affine_a - x * affine_b;
    for (size_t l = 0; l < pole.size(); ++l) {
      const double d = num_a[l] - x * num_c[l];
      s += coef[l] * d * d / (x - pole[l]);
    }
    return s;
  }
  double derivative(double x) const {
    double s = -affine_b;
    for (size_t l = 0; l < pole.size(); ++l) {
      const double d = num_a[l] - x * num_c[l];
      const double u = x - pole[l];
      s += coef[l] * (-2.0 * num_c[l] * d * u - d * d) / (u * u);
    }
    return s;
  }
};

double refine_root(const ThetaEq& eq, double lo, double hi) {
  const double eps = std::numeric_limits<double>::epsilon();
  double x = (lo + hi) / 2;
  for (int it = 0; it < 500; ++it) {
    const double g = eq.value(x);
    if (g > 0)
      lo = x;
    else if (g < 0)
      hi = x;
    else
      return x;
    const double width = hi - lo;
    if (!(width > 4 * eps * (std::abs(lo) + std::abs(hi)))) break;
    const double dg = eq.derivative(x);
    double next = x - g / dg;
    if (!(next > lo) || !(next < hi)) next = (lo + hi) / 2;
    x = next;
  }
  return (lo + hi) / 2;
}

std::vector<double> solve_theta(const Interior& es, const Element& em, double theta) {
  const int n = em.n;
  if (n == 1)
    return {(em.sb.corner + theta * em.sb.cross) / (em.mb.corner + theta * em.mb.cross)};
  const ThetaEq eq(es, em, theta);
  const int m = n - 1;
  const auto bracket_fail = [&](const std::string& what) {
    fail("solve_theta_equation: " + what + " (order " + std::to_string(n) + ", theta " +
         std::to_string(theta) + ")");
  };
  const auto right_of_pole = [&](int l) {
    const double p = eq.pole[l];
    const double gap = (l + 1 < m ? eq.pole[l + 1] : 2 * p + 1) - p;
    double d = gap / 8;
    for (int it = 0; it < 2000; ++it) {
      if (eq.value(p + d) > 0) return p + d;
      d /= 2;
      if (!(p + d > p)) break;
    }
    bracket_fail("no positive bracket right of pole " + std::to_string(l + 1));
    return p;
  };
  const auto left_of_pole = [&](int l) {
    const double p = eq.pole[l];
    const double gap = p - (l > 0 ? eq.pole[l - 1] : 0.0);
    double d = gap / 8;
    for (int it = 0; it < 2000; ++it) {
      if (eq.value(p - d) < 0) return p - d;
      d /= 2;
      if (!(p - d < p)) break;
    }
    bracket_fail("no negative bracket left of pole " + std::to_string(l + 1));
    return p;
  };
  std::vector<double> roots;
  {
    double lo = 0;
    if (!(eq.value(lo) > 0)) {
      double step = eq.pole[0] / 4;
      bool found = false;
      for (int it = 0; it < 64 && !found; ++it, step *= 2) {
        lo = -step;
        found = eq.value(lo) > 0;
      }
      if (!found) bracket_fail("no positive bracket below the first pole");
    }
    roots.push_back(refine_root(eq, lo, left_of_pole(0)));
  }
  for (int l = 0; l + 1 < m; ++l) roots.push_back(refine_root(eq, right_of_pole(l), left_of_pole(l + 1)));
  {
    double hi = 4 * eq.pole[m - 1] + 4 * std::abs(eq.affine_a) + 4;
    const double cap = 64 * hi;
    while (!(eq.value(hi) < 0)) {
      hi *= 2;
      if (hi > cap) bracket_fail("outer bracket cap reached");
    }
    roots.push_back(refine_root(eq, right_of_pole(m - 1), hi));
  }
  for (int i = 0; i + 1 < n; ++i)
    if (!(roots[i] < roots[i + 1])) bracket_fail("roots not strictly increasing");
  return roots;
}

std::vector<double> interior_solution(const Interior& es, int order, double lambda) {
  const int m = order - 1;
  std::vector<double> p(m, 0.0);
  for (int l = 0; l < m; ++l) {
    const double d = lambda - es.values[l];
    if (!(std::abs(d) > 1e-8 * (1 + std::abs(es.values[l]))))
      fail("interior_solution: lambda within pole tolerance of interior eigenvalue l=" + std::to_string(l + 1));
    const double w = (es.edge_stiff[l] - lambda * es.edge_mass[l]) / d;
    for (int i = 0; i < m; ++i) p[i] += w * es.vectors(i, l);
  }
  return p;
}

}  // namespace

void load_quadrature(int n, std::vector<double>& nodes, std::vector<double>& weighted) {
  // axis_quad (reference poisson.cpp:481-495): (n+1)-point Gauss rule and
  // weighted[loc * (n+1) + g] = w_g * phi_loc(xi_g) on the equispaced nodes
  if (n < 1 || n > 9) fail("fem_load: order " + std::to_string(n) + " outside [1, 9]");
  std::vector<double> w;
  gauss_legendre(n + 1, nodes, w);
  std::vector<double> eq(n + 1);
  for (int k = 0; k <= n; ++k) eq[k] = static_cast<double>(2 * k - n) / static_cast<double>(n);
  weighted.assign(static_cast<size_t>(n + 1) * (n + 1), 0.0);
  for (int loc = 0; loc <= n; ++loc)
    for (int g = 0; g <= n; ++g) weighted[static_cast<size_t>(loc) * (n + 1) + g] = w[g] * lagrange_value(eq, loc, nodes[g]);
}

namespace {

// finalize_table (spectral.cpp:21-79): the per-frequency data derived from the
// primaries (theta, values, p, norm_sq).  Shared by the builder and the file
// loaders, as in the reference (spectral.cpp:112, 235).
void finalize_host_table(HostTable& t, const Blocks& mb) {
  const int n = t.order, K = t.elements, m = n - 1;
  t.half_cos.resize(K - 1);
  t.half_sin.resize(K - 1);
  for (int k = 1; k < K; ++k) {
    t.half_cos[k - 1] = std::cos(M_PI * k / (2.0 * K));
    t.half_sin[k - 1] = std::sin(M_PI * k / (2.0 * K));
  }
  const size_t pairs = static_cast<size_t>(K - 1) * n;
  t.q.resize(pairs * m);
  t.nodal_weight.resize(pairs);
  for (size_t idx = 0; idx < pairs; ++idx) {
    const double theta = t.theta[idx / n];
    const double* p = t.p.data() + idx * m;
    double* q = t.q.data() + idx * m;
    double edge_dot = 0, edge_dot_rev = 0;
    for (int i = 0; i < m; ++i) {
      double s = mb.edge[i];
      for (int j = 0; j < m; ++j) s += mb.interior(i, j) * p[j];
      q[i] = s;
      edge_dot += mb.edge[i] * p[i];
      edge_dot_rev += mb.edge[i] * p[m - 1 - i];
    }
    t.nodal_weight[idx] = 2.0 * (mb.corner + edge_dot + theta * (mb.cross + edge_dot_rev));
  }
  t.eig_coeff.clear();
  t.eig_coeff.reserve(static_cast<size_t>(n) * K - 1);
  for (int l = 0; l < m; ++l) t.eig_coeff.push_back(t.interior_values[l]);
  for (size_t idx = 0; idx < pairs; ++idx) t.eig_coeff.push_back(t.values[idx]);
}

// Element data and the sized per-k arrays shared by the builder and the loaders.
HostTable table_skeleton(const Element& em, int K) {
  const int n = em.n, m = n - 1;
  HostTable t;
  t.order = n;
  t.elements = K;
  t.stiffness = em.stiffness.a;
  t.mass = em.mass.a;
  t.mass_interior = em.mb.interior.a;
  t.interior_values.assign(m, 0.0);
  t.interior_vectors.assign(static_cast<size_t>(m) * m, 0.0);
  t.theta.resize(K - 1);
  const double pi = std::acos(-1.0);
  for (int k = 1; k < K; ++k) t.theta[k - 1] = std::cos(pi * static_cast<double>(k) / static_cast<double>(K));
  t.values.resize(static_cast<size_t>(K - 1) * n);
  t.norm_sq.resize(t.values.size());
  t.p.resize(t.values.size() * m);
  return t;
}

}  // namespace

HostTable build_host_table(int n, int K) {
  if (K < 2) fail("spectral table: need at least two elements");
  const Element em = build_element(n);
  Interior es;
  if (n >= 2) es = interior_eigensystem(em);
  const int m = n - 1;
  HostTable t = table_skeleton(em, K);
  t.interior_values = es.values;
  t.interior_vectors = es.vectors.a;
  const Blocks& mb = em.mb;
  // The reference builds frequency by frequency on one thread
  // (spectral.hpp:228-277); every k is independent (one theta-equation root
  // solve and n interior solutions), so the cold build runs them in parallel.
  // A failure reports the lowest failing k, as the serial loop would.
  int bad_k = K;
  std::string bad_msg;
#pragma omp parallel for schedule(dynamic, 4) if (K > 64)
  for (int k = 1; k < K; ++k) {
    try {
      const double theta = t.theta[k - 1];
      const std::vector<double> roots = solve_theta(es, em, theta);
      for (int l = 1; l <= n; ++l) {
        const double lambda = roots[l - 1];
        const size_t idx = static_cast<size_t>(k - 1) * n + (l - 1);
        t.values[idx] = lambda;
        std::vector<double> p(m);
        if (m > 0) p = interior_solution(es, n, lambda);
        for (int i = 0; i < m; ++i) t.p[idx * m + i] = p[i];
        std::vector<double> cp(m, 0.0);
        for (int i = 0; i < m; ++i) {
          double s = 0;
          for (int j = 0; j < m; ++j) s += mb.interior(i, j) * p[j];
          cp[i] = s;
        }
        double term_direct = mb.corner, term_rev = mb.cross;
        for (int i = 0; i < m; ++i) {
          const double w = cp[i] + 2 * mb.edge[i];
          term_direct += w * p[i];
          term_rev += w * p[m - 1 - i];
        }
        const double norm_sq = static_cast<double>(K) * (term_direct + theta * term_rev);
        if (!(norm_sq > 0))
          fail("spectral table: nonpositive squared norm at k=" + std::to_string(k) + " l=" + std::to_string(l));
        t.norm_sq[idx] = norm_sq;
      }
    } catch (const std::exception& e) {
#pragma omp critical(sfem_table_build_fail)
      if (k < bad_k) {
        bad_k = k;
        bad_msg = e.what();
      }
    }
  }
  if (bad_k < K) fail(bad_msg);
  finalize_host_table(t, mb);
  return t;
}

// ---------------------------------------------------------------------------
// Table files (reference save_table / load_table / build_and_save_table,
// spectral.cpp:81-236) and the cache directory of TableSet (poisson.cpp:49-73).
// ---------------------------------------------------------------------------
namespace {

constexpr char kBinaryMagic[8] = {'S', 'F', 'E', 'M', 'B', '1', '\0', '\0'};

// format_records (spectral.cpp:81-105) at 17 significant digits: the k = 0
// records carry (lambda0_l, e^(l), K), the others (lambda_kl, p_kl, ||s_kl||^2).
std::string format_text(const HostTable& t) {
  const int n = t.order, K = t.elements, m = n - 1;
  std::string out = "SFEM1 " + std::to_string(n) + " " + std::to_string(K) + " 17\n";
  out.reserve(out.size() + static_cast<size_t>(n) * K * (n + 4) * 25);
  char buf[64];
  auto num = [&](double v) {
    std::snprintf(buf, sizeof buf, " %.*g", 17, v);
    out += buf;
  };
  for (int l = 1; l <= m; ++l) {
    out += "0 " + std::to_string(l);
    num(t.interior_values[l - 1]);
    for (int i = 0; i < m; ++i) num(t.interior_vectors[static_cast<size_t>(i) * m + (l - 1)]);
    num(static_cast<double>(K));
    out += '\n';
  }
  for (int k = 1; k < K; ++k)
    for (int l = 1; l <= n; ++l) {
      const size_t idx = static_cast<size_t>(k - 1) * n + (l - 1);
      out += std::to_string(k) + " " + std::to_string(l);
      num(t.values[idx]);
      for (int i = 0; i < m; ++i) num(t.p[idx * m + i]);
      num(t.norm_sq[idx]);
      out += '\n';
    }
  return out;
}

uint64_t fnv1a(const void* data, size_t bytes, uint64_t h = 1469598103934665603ull) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < bytes; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

// The primaries in file order: interior values, interior vectors (row-major
// [i][l-1]), then per (k, l) values, norm_sq, p.
std::vector<std::vector<double>*> binary_parts(HostTable& t) {
  return {&t.interior_values, &t.interior_vectors, &t.values, &t.norm_sq, &t.p};
}

std::string read_file(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) fail("load_table: cannot open '" + path + "'");
  std::string s;
  char buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, got);
  std::fclose(f);
  return s;
}

void write_file(const std::string& path, const std::string& data) {
  // Write to a temporary name and rename, so a concurrent reader of the cache
  // never sees a partial file (the reference writes in place, spectral.cpp:117-124).
  static std::atomic<int> serial{0};
  const std::string tmp = path + ".tmp" + std::to_string(static_cast<long long>(getpid())) + "_" +
                          std::to_string(serial.fetch_add(1));
  std::FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) fail("save_table: cannot open '" + path + "' for writing");
  const bool ok = std::fwrite(data.data(), 1, data.size(), f) == data.size();
  if (std::fclose(f) != 0 || !ok || std::rename(tmp.c_str(), path.c_str()) != 0) {
    std::remove(tmp.c_str());
    fail("save_table: write failed for '" + path + "'");
  }
}

struct Tokens {
  const char* p;
  const char* end;
  void skip() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r')) ++p;
  }
  bool word(std::string& w) {
    skip();
    const char* s = p;
    while (p < end && !(*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r')) ++p;
    w.assign(s, p);
    return p > s;
  }
  bool integer(int& v) {
    skip();
    auto r = std::from_chars(p, end, v);
    if (r.ec != std::errc()) return false;
    p = r.ptr;
    return true;
  }
  bool real(double& v) {
    skip();
    auto r = std::from_chars(p, end, v);
    if (r.ec != std::errc()) return false;
    p = r.ptr;
    return true;
  }
};

void check_header(int fn, int fk, int n, int K) {
  if (fn != n || fk != K)
    fail("load_table: file holds order " + std::to_string(fn) + ", elements " + std::to_string(fk) +
         " but order " + std::to_string(n) + ", elements " + std::to_string(K) + " were requested");
  if (!(n >= 1 && K >= 2 && n <= 9)) fail("load_table: header values out of range");
}

HostTable parse_text(const std::string& s, const std::string& path, int n, int K) {
  Tokens in{s.data(), s.data() + s.size()};
  std::string magic;
  int fn = 0, fk = 0, digits = 0;
  if (!(in.word(magic) && in.integer(fn) && in.integer(fk) && in.integer(digits)))
    fail("load_table: malformed header in '" + path + "'");
  if (magic != "SFEM1") fail("load_table: unsupported format '" + magic + "' in '" + path + "'");
  check_header(fn, fk, n, K);
  const int m = n - 1;
  HostTable t = table_skeleton(build_element(n), K);
  const size_t expected = static_cast<size_t>(n) * K - 1;
  std::vector<double> vec(m);
  for (size_t rec = 0; rec < expected; ++rec) {
    int k = 0, l = 0;
    double lambda = 0, norm = 0;
    if (!(in.integer(k) && in.integer(l) && in.real(lambda)))
      fail("load_table: truncated or corrupt record " + std::to_string(rec + 1) + " in '" + path + "'");
    for (int i = 0; i < m; ++i)
      if (!in.real(vec[i])) fail("load_table: truncated interior vector in record " + std::to_string(rec + 1));
    if (!in.real(norm)) fail("load_table: truncated record " + std::to_string(rec + 1));
    if (k == 0) {
      if (l < 1 || l > m) fail("load_table: zero-frequency record with bad index");
      t.interior_values[l - 1] = lambda;
      for (int i = 0; i < m; ++i) t.interior_vectors[static_cast<size_t>(i) * m + (l - 1)] = vec[i];
    } else {
      if (k < 1 || k >= K || l < 1 || l > n) fail("load_table: record index out of range");
      const size_t idx = static_cast<size_t>(k - 1) * n + (l - 1);
      t.values[idx] = lambda;
      for (int i = 0; i < m; ++i) t.p[idx * m + i] = vec[i];
      t.norm_sq[idx] = norm;
    }
  }
  std::string trailing;
  if (in.word(trailing)) fail("load_table: unexpected trailing data in '" + path + "'");
  return t;
}

HostTable parse_binary(const std::string& s, const std::string& path, int n, int K) {
  struct Header {
    char magic[8];
    int32_t order, elements, digits, reserved;
    uint64_t count;
  } h;
  if (s.size() < sizeof h) fail("load_table: malformed header in '" + path + "'");
  std::memcpy(&h, s.data(), sizeof h);
  check_header(h.order, h.elements, n, K);
  HostTable t = table_skeleton(build_element(n), K);
  size_t count = 0;
  for (auto* v : binary_parts(t)) count += v->size();
  if (h.count != count || s.size() != sizeof h + count * sizeof(double) + sizeof(uint64_t))
    fail("load_table: truncated or corrupt payload in '" + path + "'");
  const char* p = s.data() + sizeof h;
  uint64_t sum;
  std::memcpy(&sum, p + count * sizeof(double), sizeof sum);
  if (sum != fnv1a(p, count * sizeof(double))) fail("load_table: checksum mismatch in '" + path + "'");
  for (auto* v : binary_parts(t)) {
    std::memcpy(v->data(), p, v->size() * sizeof(double));
    p += v->size() * sizeof(double);
  }
  return t;
}

}  // namespace

void save_host_table(const HostTable& t, const std::string& path, int format) {
  if (format == kTableText) {
    write_file(path, format_text(t));
    return;
  }
  if (format != kTableBinary) fail("save_table: unknown format " + std::to_string(format));
  HostTable c = t;  // binary_parts wants mutable vectors
  size_t count = 0;
  for (auto* v : binary_parts(c)) count += v->size();
  std::string out(sizeof(kBinaryMagic) + 4 * sizeof(int32_t) + sizeof(uint64_t), '\0');
  char* w = out.data();
  std::memcpy(w, kBinaryMagic, sizeof kBinaryMagic);
  const int32_t hdr[4] = {t.order, t.elements, 17, 0};
  std::memcpy(w + 8, hdr, sizeof hdr);
  const uint64_t cnt = count;
  std::memcpy(w + 24, &cnt, sizeof cnt);
  const size_t payload_at = out.size();
  for (auto* v : binary_parts(c)) out.append(reinterpret_cast<const char*>(v->data()), v->size() * sizeof(double));
  const uint64_t sum = fnv1a(out.data() + payload_at, count * sizeof(double));
  out.append(reinterpret_cast<const char*>(&sum), sizeof sum);
  write_file(path, out);
}

HostTable load_host_table(const std::string& path, int n, int K) {
  const std::string s = read_file(path);
  HostTable t = (s.size() >= 8 && std::memcmp(s.data(), kBinaryMagic, 8) == 0) ? parse_binary(s, path, n, K)
                                                                                  : parse_text(s, path, n, K);
  // the reference rebuilds the derived data after a load (spectral.cpp:209-235)
  finalize_host_table(t, build_element(n).mb);
  return t;
}

std::string table_cache_path(const std::string& dir, int n, int K, int format) {
  return dir + "/sfem_table_n" + std::to_string(n) + "_K" + std::to_string(K) +
         (format == kTableBinary ? ".bin" : ".txt");
}

HostTable cached_host_table(const TableCache& cache, int n, int K, int* source) {
  if (source) *source = 0;
  if (cache.dir.empty()) return build_host_table(n, K);
  // TableSet::get (poisson.cpp:49-73): a stale or unreadable entry is rebuilt.
  // The binary entry is tried first, then the reference's text entry, so a
  // cache directory the reference filled is used as is.
  for (int format : {kTableBinary, kTableText}) {
    try {
      HostTable t = load_host_table(table_cache_path(cache.dir, n, K, format), n, K);
      if (source) *source = 1 + format;
      return t;
    } catch (const std::exception&) {
    }
  }
  HostTable t = build_host_table(n, K);
  if (cache.write) save_host_table(t, table_cache_path(cache.dir, n, K, cache.format), cache.format);
  return t;
}

DeviceTableData derive_device_data(const HostTable& t) {
  const int n = t.order, K = t.elements, m = n - 1, N = K;
  const int half = m / 2, ne = n / 2;
  DeviceTableData d;
  d.n = n;
  d.K = K;
  const size_t nn = static_cast<size_t>(n) * n;
  d.mix_fwd_w.assign((K - 1) * nn, 0.0);
  d.mix_fwd_d.assign((K - 1) * nn, 0.0);
  d.mix_inv.assign((K - 1) * nn, 0.0);
  // Slot order s: 0 = nodal DST-I, 1+i (i < ne) = even part via DST-II,
  // 1+ne+i (i < no) = odd part via DCT-II.  The reference folds neighbouring
  // elements before a DST-I (eigenbasis.cpp:46-59, 87-100); by
  //   DST-I(fold_e)_k = 2 cos(pi k/2K) DST-II(g)_k,
  //   DST-I(fold_o)_k = -2 sin(pi k/2K) DCT-II(h)_k
  // the same numbers come from half-sample transforms of the unfolded rows,
  // which pair two per complex FFT.  Those factors and 1/||s||^2 are folded
  // into the per-frequency mixes here.
  for (int k = 1; k < K; ++k) {
    const double c2 = 2.0 * t.half_cos[k - 1], s2 = -2.0 * t.half_sin[k - 1];
    for (int l = 0; l < n; ++l) {
      const size_t idx = static_cast<size_t>(k - 1) * n + l;
      const double inv = 1.0 / t.norm_sq[idx];
      const double* p = t.p.data() + idx * m;
      const double* q = t.q.data() + idx * m;
      double* fw = d.mix_fwd_w.data() + (k - 1) * nn + static_cast<size_t>(l) * n;
      double* fd = d.mix_fwd_d.data() + (k - 1) * nn + static_cast<size_t>(l) * n;
      fw[0] = inv;
      fd[0] = t.nodal_weight[idx] * inv;
      d.mix_inv[(k - 1) * nn + 0 * n + l] = 1.0;
      for (int i = 0; i < ne; ++i) {
        const double pe = i < half ? 0.5 * (p[i] + p[m - 1 - i]) : p[half];
        const double qe = i < half ? 0.5 * (q[i] + q[m - 1 - i]) : q[half];
        fw[1 + i] = c2 * pe * inv;
        fd[1 + i] = c2 * qe * inv;
        d.mix_inv[(k - 1) * nn + static_cast<size_t>(1 + i) * n + l] = c2 * pe;
      }
      for (int i = 0; i < half; ++i) {
        const double po = 0.5 * (p[i] - p[m - 1 - i]);
        const double qo = 0.5 * (q[i] - q[m - 1 - i]);
        fw[1 + ne + i] = s2 * po * inv;
        fd[1 + ne + i] = s2 * qo * inv;
        d.mix_inv[(k - 1) * nn + static_cast<size_t>(1 + ne + i) * n + l] = s2 * po;
      }
    }
  }
  d.e0_fwd_w.assign(static_cast<size_t>(m) * m, 0.0);
  d.e0_fwd_d.assign(static_cast<size_t>(m) * m, 0.0);
  d.e0_inv.assign(static_cast<size_t>(m) * m, 0.0);
  for (int i = 0; i < m; ++i)
    for (int l = 0; l < m; ++l) {
      const double e = t.interior_vectors[static_cast<size_t>(i) * m + l];
      d.e0_inv[static_cast<size_t>(i) * m + l] = e;
      d.e0_fwd_w[static_cast<size_t>(i) * m + l] = e / K;
      double ce = 0;  // (C~ e^(l))_i
      for (int j = 0; j < m; ++j)
        ce += t.mass_interior[static_cast<size_t>(i) * m + j] * t.interior_vectors[static_cast<size_t>(j) * m + l];
      d.e0_fwd_d[static_cast<size_t>(i) * m + l] = ce / K;
    }
  d.eig = t.eig_coeff;
  // norm_sq in coefficient order: the fused last-axis sweep runs the forward
  // mix with the synthesis matrix (mix_fwd_w[k][l][s] = mix_inv[k][s][l] /
  // norm_sq[k][l], exactly as formed above) and folds 1/norm_sq into the
  // symbol divide, so one matrix per frequency serves both mixes.
  d.nsq.assign(static_cast<size_t>(n) * K - 1, 1.0);
  for (int k = 1; k < K; ++k)
    for (int l = 0; l < n; ++l) d.nsq[m + static_cast<size_t>(k - 1) * n + l] = t.norm_sq[static_cast<size_t>(k - 1) * n + l];
  d.mixT_w.assign(nn * K, 0.0);
  d.mixT_d.assign(nn * K, 0.0);
  d.mixT_i.assign(nn * K, 0.0);
  for (int k = 1; k < K; ++k)
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) {
        const size_t src = (k - 1) * nn + static_cast<size_t>(a) * n + b;
        const size_t dst = (static_cast<size_t>(a) * n + b) * K + k;
        // fast kernels: the 1/2 of the nodal DST-I post-processing lives in the
        // nodal column (forward, s = 0) / nodal row (inverse, s = 0) of the mix
        d.mixT_w[dst] = d.mix_fwd_w[src] * (b == 0 ? 0.5 : 1.0);
        d.mixT_d[dst] = d.mix_fwd_d[src] * (b == 0 ? 0.5 : 1.0);
        d.mixT_i[dst] = d.mix_inv[src] * (a == 0 ? 0.5 : 1.0);
      }
  d.tw.resize(2 * N);
  d.mk.resize(2 * N);
  d.mkh.resize(2 * N);
  d.om.resize(2 * N);
  const long double PI = 3.14159265358979323846264338327950288L;
  for (int j = 0; j < N; ++j) {
    const long double a = -2.0L * PI * j / N;
    d.tw[2 * j] = static_cast<double>(cosl(a));
    d.tw[2 * j + 1] = static_cast<double>(sinl(a));
    const long double b = PI * j / (2.0L * N);
    d.mk[2 * j] = static_cast<double>(cosl(b));
    d.mk[2 * j + 1] = static_cast<double>(-sinl(b));
    d.mkh[2 * j] = static_cast<double>(0.5L * cosl(b));
    d.mkh[2 * j + 1] = static_cast<double>(0.5L * sinl(b));
    const long double c = PI * j / N;
    d.om[2 * j] = static_cast<double>(cosl(c));
    d.om[2 * j + 1] = static_cast<double>(-sinl(c));
  }
  return d;
}

}  // namespace sfem_b200
