// C++ parity tests through include/sfem_b200.hpp (the reference-shaped API),
// restating the reference's own test cases (proj/tests/test_eigenbasis.cpp,
// test_poisson.cpp).  Built and run by tests/test_cpp_api.py (GPU).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <random>
#include <vector>

#include "sfem_b200.hpp"

using namespace sfem_b200;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                            \
  do {                                                                         \
    if (cond) {                                                                \
      ++g_pass;                                                                \
    } else {                                                                   \
      ++g_fail;                                                                \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);              \
    }                                                                          \
  } while (0)
#define CHECK_THROWS(expr)                                                     \
  do {                                                                         \
    bool thrown = false;                                                       \
    try {                                                                      \
      expr;                                                                    \
    } catch (const Error&) {                                                   \
      thrown = true;                                                           \
    }                                                                          \
    CHECK(thrown);                                                             \
  } while (0)

static GridFunction1D random_grid(int n, int K, unsigned seed) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  GridFunction1D g = GridFunction1D::zeros(n, K);
  for (int j = 1; j < K; ++j) g.nodal[j] = u(rng);
  for (auto& v : g.interior) v = u(rng);
  return g;
}

static CoefficientArray1D random_coeffs(int n, int K, unsigned seed) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  CoefficientArray1D c = CoefficientArray1D::zeros(n, K);
  for (auto& v : c.data) v = u(rng);
  return c;
}

static double max_diff(const std::vector<double>& a, const std::vector<double>& b) {
  double w = 0;
  for (size_t i = 0; i < a.size(); ++i) w = std::max(w, std::abs(a[i] - b[i]));
  return w;
}

// test_eigenbasis.cpp:106-123
static void roundtrip_identities(TableSet& tables) {
  for (int n : {1, 2, 3, 5, 9})
    for (int K : {2, 3, 4, 8, 31, 64}) {
      const auto& t = tables.get(n, K);
      const auto c = random_coeffs(n, K, 1000u + n * 64 + K);
      const auto back = decompose(synthesize(c, t), t);
      CHECK(max_diff(c.data, back.data) <= 1e-11);
      const auto g = random_grid(n, K, 2000u + n * 64 + K);
      const auto gb = synthesize(decompose(g, t), t);
      CHECK(max_diff(g.nodal, gb.nodal) <= 1e-11);
      CHECK(max_diff(g.interior, gb.interior) <= 1e-11);
    }
}

// test_eigenbasis.cpp:198-205
static void dimension_mismatches(TableSet& tables) {
  const auto& t = tables.get(2, 4);
  const auto g = random_grid(2, 5, 1);
  CHECK_THROWS(decompose(g, t));
  CHECK_THROWS(decompose_weighted(g, t));
  const auto c = random_coeffs(3, 4, 1);
  CHECK_THROWS(synthesize(c, t));
}

// Dense Kronecker reference (oracle.cpp:146-184) on the interleaved dof order.
static std::vector<double> dense_solve_2d(int n, int K, double shift, const std::vector<double>& rhs) {
  // element matrices for n = 2 on [-1,1] (exact): stiffness / mass
  const double A[3][3] = {{7.0 / 6, -4.0 / 3, 1.0 / 6}, {-4.0 / 3, 8.0 / 3, -4.0 / 3}, {1.0 / 6, -4.0 / 3, 7.0 / 6}};
  const double M[3][3] = {{4.0 / 15, 2.0 / 15, -1.0 / 15}, {2.0 / 15, 16.0 / 15, 2.0 / 15}, {-1.0 / 15, 2.0 / 15, 4.0 / 15}};
  const int L = n * K - 1;
  auto dof = [&](int e, int loc) {
    if (loc == 0) return e == 0 ? -1 : e * n - 1;
    if (loc == n) return e == K - 1 ? -1 : (e + 1) * n - 1;
    return e * n + loc - 1;
  };
  std::vector<double> a1(L * L, 0.0), c1(L * L, 0.0);
  for (int e = 0; e < K; ++e)
    for (int i = 0; i <= n; ++i)
      for (int j = 0; j <= n; ++j) {
        const int gi = dof(e, i), gj = dof(e, j);
        if (gi < 0 || gj < 0) continue;
        a1[gi * L + gj] += A[i][j];
        c1[gi * L + gj] += M[i][j];
      }
  const double f = 4.0 * K * K;  // 4/h^2 on the unit square
  const int U = L * L;
  std::vector<double> S(static_cast<size_t>(U) * U, 0.0), x = rhs;
  for (int i0 = 0; i0 < L; ++i0)
    for (int i1 = 0; i1 < L; ++i1)
      for (int j0 = 0; j0 < L; ++j0)
        for (int j1 = 0; j1 < L; ++j1)
          S[static_cast<size_t>(i0 * L + i1) * U + (j0 * L + j1)] =
              f * (a1[i0 * L + j0] * c1[i1 * L + j1] + c1[i0 * L + j0] * a1[i1 * L + j1]) +
              shift * c1[i0 * L + j0] * c1[i1 * L + j1];
  // Gaussian elimination (SPD, no pivoting needed)
  for (int k = 0; k < U; ++k)
    for (int i = k + 1; i < U; ++i) {
      const double r = S[static_cast<size_t>(i) * U + k] / S[static_cast<size_t>(k) * U + k];
      if (r == 0) continue;
      for (int j = k; j < U; ++j) S[static_cast<size_t>(i) * U + j] -= r * S[static_cast<size_t>(k) * U + j];
      x[i] -= r * x[k];
    }
  for (int i = U - 1; i >= 0; --i) {
    double s = x[i];
    for (int j = i + 1; j < U; ++j) s -= S[static_cast<size_t>(i) * U + j] * x[j];
    x[i] = s / S[static_cast<size_t>(i) * U + i];
  }
  return x;
}

// test_poisson.cpp:151-160 (2D solve vs the dense Kronecker system), through
// solve_with_load on the reference's GridFunctionND layout.
static void solve_vs_dense(TableSet& tables) {
  const int n = 2, K = 4, L = n * K - 1;
  ProblemSpec spec;
  spec.dimension = 2;
  spec.lengths = {1.0, 1.0};
  spec.elements = {K, K};
  spec.orders = {n, n};
  spec.shift = 1.0;
  std::mt19937 rng(7);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::vector<double> rhs(L * L);
  for (auto& v : rhs) v = u(rng);
  // dof -> class arrays
  GridFunctionND load = GridFunctionND::zeros(spec.axis_specs());
  auto cls = [&](int t, int& interior, int& idx) {
    const int r = t % n;
    interior = r != n - 1;
    idx = interior ? (t / n) * (n - 1) + r : t / n + 1;
  };
  for (int t0 = 0; t0 < L; ++t0)
    for (int t1 = 0; t1 < L; ++t1) {
      int m0, i0, m1, i1;
      cls(t0, m0, i0);
      cls(t1, m1, i1);
      const unsigned mask = m0 | (m1 << 1);
      const int e1 = load.class_extents(mask)[1];
      load.classes[mask][static_cast<size_t>(i0) * e1 + i1] = rhs[t0 * L + t1];
    }
  const SolveReport rep = solve_with_load(spec, load, tables);
  const std::vector<double> want = dense_solve_2d(n, K, spec.shift, rhs);
  double worst = 0, scale = 0;
  for (int t0 = 0; t0 < L; ++t0)
    for (int t1 = 0; t1 < L; ++t1) {
      int m0, i0, m1, i1;
      cls(t0, m0, i0);
      cls(t1, m1, i1);
      const unsigned mask = m0 | (m1 << 1);
      const int e1 = rep.solution.class_extents(mask)[1];
      worst = std::max(worst, std::abs(rep.solution.classes[mask][static_cast<size_t>(i0) * e1 + i1] - want[t0 * L + t1]));
      scale = std::max(scale, std::abs(want[t0 * L + t1]));
    }
  CHECK(worst <= 1e-10 * std::max(1.0, scale));
  // boundary slots are zero (enforce_boundary)
  CHECK(rep.solution.classes[0][0] == 0.0);
  CHECK(rep.seconds_solve >= 0.0);
}

// test_poisson.cpp:276-291
static void rejects_invalid(TableSet& tables) {
  ProblemSpec spec;
  spec.dimension = 2;
  spec.lengths = {1.0, 1.0};
  spec.elements = {4, 4};
  spec.orders = {2, 2};
  spec.shift = -2 * M_PI * M_PI - 1;
  GridFunctionND load = GridFunctionND::zeros(spec.axis_specs());
  CHECK_THROWS(solve_with_load(spec, load, tables));
  ProblemSpec bad = spec;
  bad.shift = 1.0;
  bad.elements = {4};
  CHECK_THROWS(bad.validate());
  // algorithm (b) needs dimension >= 2 (poisson.cpp:674)
  ProblemSpec one;
  one.dimension = 1;
  one.lengths = {1.0};
  one.elements = {4};
  one.orders = {2};
  one.shift = 1.0;
  GridFunctionND load1 = GridFunctionND::zeros(one.axis_specs());
  SolveOptions opt;
  opt.algorithm = Algorithm::PartialDiagonalization;
  CHECK_THROWS(solve_with_load(one, load1, tables, opt));
}

// test_poisson.cpp:355-362 (bitwise reproducibility)
static void deterministic(TableSet& tables) {
  ProblemSpec spec;
  spec.dimension = 3;
  spec.lengths = {1.0, 1.0, 1.0};
  spec.elements = {8, 8, 8};
  spec.orders = {9, 9, 9};
  spec.shift = 0.0;
  Plan plan(tables.context(), spec);
  const int L = 9 * 8 - 1;
  std::vector<double> f(static_cast<size_t>(L) * L * L), u1(f.size()), u2(f.size());
  std::mt19937 rng(3);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (auto& v : f) v = u(rng);
  plan.solve_dof(f.data(), u1.data());
  plan.solve_dof(f.data(), u2.data());
  CHECK(max_diff(u1, u2) == 0.0);
}

// solve(spec, options) of the reference's manufactured cases, every step on
// the device: the residual check (poisson.cpp:785-789) and the discretisation
// error (test_poisson.cpp convergence tests: high order, error shrinks with K)
static void manufactured_solve() {
  for (int K : {4, 8}) {
    ProblemSpec spec;
    spec.dimension = 2;
    spec.lengths = {1.0, 1.0};
    spec.elements = {K, K};
    spec.orders = {4, 4};
    spec.shift = 1.0;
    SolveOptions opt;
    opt.compute_residual = true;
    const SolveReport r = solve(spec, Field::manufactured("poisson2d"), opt);
    CHECK(r.residual_rel.has_value() && *r.residual_rel < 1e-11);
    CHECK(r.error_uniform.has_value() && *r.error_uniform < (K == 4 ? 5e-2 : 5e-3));
    CHECK(r.seconds_solve > 0 && r.seconds_load > 0);
    CHECK(r.solution.classes.size() == 4);
  }
  CHECK_THROWS(Field::manufactured("nope"));
}

// A (A^-1 f) == f through the dense-dof operator
static void operator_inverts_solve(TableSet& tables) {
  ProblemSpec spec;
  spec.dimension = 3;
  spec.lengths = {1.0, 2.0, 1.0};
  spec.elements = {5, 4, 6};
  spec.orders = {3, 2, 4};
  spec.shift = 0.5;
  Plan plan(tables.context(), spec);
  std::vector<double> f(static_cast<size_t>(plan.unknowns())), u(f.size()), y(f.size());
  std::mt19937 rng(9);
  std::uniform_real_distribution<double> d(-1.0, 1.0);
  for (auto& v : f) v = d(rng);
  plan.solve_dof(f.data(), u.data());
  plan.apply_operator_dof(u.data(), y.data());
  CHECK(max_diff(y, f) < 1e-11);
}

// algorithm (b) agrees with algorithm (a) (both solve the same system)
static void partial_matches_full(TableSet& tables) {
  ProblemSpec spec;
  spec.dimension = 3;
  spec.lengths = {1.0, 1.0, 1.0};
  spec.elements = {6, 5, 4};
  spec.orders = {9, 3, 2};
  spec.shift = 0.0;
  GridFunctionND load = GridFunctionND::zeros(spec.axis_specs());
  std::mt19937 rng(11);
  std::uniform_real_distribution<double> d(-1.0, 1.0);
  for (auto& c : load.classes)
    for (auto& v : c) v = d(rng);
  load = classes_from_dof(spec.axis_specs(), [&] {
    // round trip through the dof layout zeroes the boundary slots
    std::vector<double> dof(static_cast<size_t>(53 * 14 * 7));
    for (auto& v : dof) v = d(rng);
    return dof;
  }());
  SolveOptions a, b;
  b.algorithm = Algorithm::PartialDiagonalization;
  const SolveReport ra = solve_with_load(spec, load, tables, a);
  const SolveReport rb = solve_with_load(spec, load, tables, b);
  double w = 0, nrm = 0;
  for (size_t c = 0; c < ra.solution.classes.size(); ++c)
    for (size_t i = 0; i < ra.solution.classes[c].size(); ++i) {
      w = std::max(w, std::abs(ra.solution.classes[c][i] - rb.solution.classes[c][i]));
      nrm = std::max(nrm, std::abs(ra.solution.classes[c][i]));
    }
  CHECK(w <= 1e-12 * nrm);
}

// Table files and the cache directory (spectral.cpp:81-236, poisson.cpp:49-73):
// a table saved and loaded back in either format transforms bit for bit like
// the built one; a second TableSet over the same directory loads the entry;
// a file for another (n, K) is refused with load_table's message.
static void table_files() {
  Context& ctx = default_context();
  const std::string dir = std::string(std::getenv("TMPDIR") ? std::getenv("TMPDIR") : "/tmp") + "/sfem_cpp_tables_" +
                          std::to_string(static_cast<long long>(std::random_device{}()));
  std::system(("mkdir -p " + dir).c_str());
  SpectralTable built(ctx, 4, 24);
  const GridFunction1D g = random_grid(4, 24, 11);
  const std::vector<double> want = decompose_weighted(g, built).data;
  for (TableFormat f : {TableFormat::Text, TableFormat::Binary}) {
    const std::string path = dir + (f == TableFormat::Text ? "/t.txt" : "/t.bin");
    built.save(path, f);
    auto loaded = SpectralTable::load(ctx, path, 4, 24);
    CHECK(max_diff(decompose_weighted(g, *loaded).data, want) == 0.0);
    CHECK(loaded->eigenvalues_coeff_order() == built.eigenvalues_coeff_order());
    CHECK_THROWS(SpectralTable::load(ctx, path, 4, 25));
  }
  build_and_save_table(3, 10, dir + "/sfem_table_n3_K10.txt");
  {
    Context c2(0);
    TableSet cached(c2, dir, true, TableFormat::Binary);
    const auto& t = cached.get(3, 10);  // loads the text entry
    SpectralTable fresh(ctx, 3, 10);
    CHECK(t.eigenvalues_coeff_order() == fresh.eigenvalues_coeff_order());
    cached.get(5, 12);  // built, then written as .bin
  }
  std::FILE* f = std::fopen((dir + "/sfem_table_n5_K12.bin").c_str(), "rb");
  CHECK(f != nullptr);
  if (f) std::fclose(f);
  std::system(("rm -rf " + dir).c_str());
}

// test_eigenbasis.cpp:40-50, 125-135: synthesize(indicator (k, l)) is the
// materialised eigenvector; both DirectRoutes give the same coefficients.
static void eigenvectors_and_routes(TableSet& tables) {
  for (int n : {1, 3, 9})
    for (int K : {4, 11}) {
      const auto& t = tables.get(n, K);
      for (int k = 0; k < K; ++k)
        for (int l = 1; l <= (k == 0 ? n - 1 : n); ++l) {
          CoefficientArray1D c = CoefficientArray1D::zeros(n, K);
          c.at(k, l) = 1.0;
          const GridFunction1D s = synthesize(c, t), want = materialize_eigenvector(t, k, l);
          CHECK(max_diff(s.to_dof(), want.to_dof()) <= 1e-12);
        }
      const GridFunction1D g = random_grid(n, K, 5);
      const auto a = decompose(g, t, DirectRoute::Spectral), b = decompose(g, t, DirectRoute::MassApply);
      CHECK(max_diff(a.data, b.data) <= 1e-12);
    }
  CHECK_THROWS(materialize_eigenvector(tables.get(3, 4), 4, 1));
  CHECK_THROWS(materialize_eigenvector(tables.get(3, 4), 0, 3));
}

int main() {
  TableSet tables;
  table_files();
  eigenvectors_and_routes(tables);
  roundtrip_identities(tables);
  dimension_mismatches(tables);
  solve_vs_dense(tables);
  rejects_invalid(tables);
  deterministic(tables);
  manufactured_solve();
  operator_inverts_solve(tables);
  partial_matches_full(tables);
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
