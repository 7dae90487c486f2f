// sfem_b200.hpp -- header-only C++ mirror of the reference solver API over the
// C-ABI in sfem_cuda.h.  A user of the reference (namespace sfem, proj/include/
// sfem/*.hpp) switches by including this header and using namespace
// sfem_b200: the names, argument meaning and error behaviour of the hot-path
// entry points are the reference's:
//
//   reference (file:line)                      here
//   sfem::Error (types.hpp:9-18)               sfem_b200::Error
//   ProblemSpec (poisson.hpp:29-41)            ProblemSpec (+ optional per-axis coefficients)
//   SolveOptions / SolveReport (64-78)         SolveOptions / SolveReport
//   TableSet::get (poisson.hpp:54)             TableSet::get -> const SpectralTable&
//   solve_with_load (poisson.hpp:90-91)        solve_with_load (GridFunctionND in/out)
//   GridFunctionND (ndgrid.hpp:43-57)          GridFunctionND (2^N parity-class arrays)
//   GridFunction1D / CoefficientArray1D        GridFunction1D / CoefficientArray1D
//     (grid1d.hpp:13-61)
//   synthesize / decompose / decompose_weighted  same (eigenbasis.hpp:76-79)
//   lines::* raw forms (eigenbasis.hpp:50-55)  lines::* on dof-layout batches
//
// The right-hand-side closure / fem_load_average of the reference are outside
// the accelerated path; loads are passed in, as solve_with_load does.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sfem_cuda.h"

namespace sfem_b200 {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

[[noreturn]] inline void fail(const std::string& msg) { throw Error(msg); }
inline void require(bool cond, const std::string& msg) {
  if (!cond) fail(msg);
}
inline void check(int status) {
  if (status != 0) throw Error(sfem_cuda_last_error());
}

// ---------------------------------------------------------------------------
// Device context (one per GPU; owns the stream)
// ---------------------------------------------------------------------------
class Context {
 public:
  explicit Context(int device = 0) { check(sfem_cuda_ctx_create(device, &h_)); }
  ~Context() { sfem_cuda_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  sfem_ctx handle() const { return h_; }

 private:
  sfem_ctx h_ = nullptr;
};

inline Context& default_context() {
  static Context ctx(0);
  return ctx;
}

// ---------------------------------------------------------------------------
// 1D types (grid1d.hpp:13-61)
// ---------------------------------------------------------------------------
struct GridFunction1D {
  int order = 0, elements = 0;
  std::vector<double> nodal;     // K+1, boundary entries zero
  std::vector<double> interior;  // K*(n-1), element-major

  static GridFunction1D zeros(int n, int K) {
    GridFunction1D g;
    g.order = n;
    g.elements = K;
    g.nodal.assign(K + 1, 0.0);
    g.interior.assign(static_cast<size_t>(K) * (n - 1), 0.0);
    return g;
  }
  int dof_count() const { return order * elements - 1; }
  // interleaved dof vector (banded.cpp:87-96 ordering)
  std::vector<double> to_dof() const {
    const int n = order, K = elements, m = n - 1;
    std::vector<double> v(static_cast<size_t>(n) * K - 1);
    for (int e = 0; e < K; ++e) {
      for (int c = 0; c < m; ++c) v[static_cast<size_t>(e) * n + c] = interior[static_cast<size_t>(e) * m + c];
      if (e + 1 < K) v[static_cast<size_t>(e + 1) * n - 1] = nodal[e + 1];
    }
    return v;
  }
  static GridFunction1D from_dof(const double* v, int n, int K) {
    GridFunction1D g = zeros(n, K);
    const int m = n - 1;
    for (int e = 0; e < K; ++e) {
      for (int c = 0; c < m; ++c) g.interior[static_cast<size_t>(e) * m + c] = v[static_cast<size_t>(e) * n + c];
      if (e + 1 < K) g.nodal[e + 1] = v[static_cast<size_t>(e + 1) * n - 1];
    }
    return g;
  }
};

struct CoefficientArray1D {
  int order = 0, elements = 0;
  std::vector<double> data;  // n*K-1, frequency-major
  static CoefficientArray1D zeros(int n, int K) {
    CoefficientArray1D c;
    c.order = n;
    c.elements = K;
    c.data.assign(static_cast<size_t>(n) * K - 1, 0.0);
    return c;
  }
  int index(int k, int l) const { return k == 0 ? l - 1 : (order - 1) + (k - 1) * order + (l - 1); }
  double& at(int k, int l) { return data[index(k, l)]; }
  double at(int k, int l) const { return data[index(k, l)]; }
};

// ---------------------------------------------------------------------------
// Spectral table (device) and TableSet (poisson.hpp:48-62)
// ---------------------------------------------------------------------------
enum class TableFormat { Text = SFEM_TABLE_TEXT, Binary = SFEM_TABLE_BINARY };

class SpectralTable {
 public:
  SpectralTable(Context& ctx, int order, int elements) : order(order), elements(elements) {
    check(sfem_cuda_table_create(ctx.handle(), order, elements, &h_));
  }
  // load_table (spectral.hpp:326): the reference's SFEM1 text files or our SFEMB1 binary ones.
  static std::unique_ptr<SpectralTable> load(Context& ctx, const std::string& path, int order, int elements) {
    sfem_table h = nullptr;
    check(sfem_cuda_table_load(ctx.handle(), path.c_str(), order, elements, &h));
    return std::unique_ptr<SpectralTable>(new SpectralTable(h, order, elements));
  }
  ~SpectralTable() { sfem_cuda_table_destroy(h_); }
  SpectralTable(const SpectralTable&) = delete;
  SpectralTable& operator=(const SpectralTable&) = delete;
  sfem_table handle() const { return h_; }
  int coeff_count() const { return order * elements - 1; }
  std::vector<double> eigenvalues_coeff_order() const {
    std::vector<double> e(coeff_count());
    check(sfem_cuda_table_export(h_, nullptr, nullptr, nullptr, nullptr, nullptr, e.data()));
    return e;
  }
  // save_table (spectral.hpp:325); Text writes the reference's file byte for byte.
  void save(const std::string& path, TableFormat format = TableFormat::Text) const {
    check(sfem_cuda_table_save(h_, path.c_str(), static_cast<int>(format)));
  }
  const int order, elements;

 private:
  SpectralTable(sfem_table h, int order, int elements) : order(order), elements(elements), h_(h) {}
  sfem_table h_ = nullptr;
};

// build_and_save_table (spectral.hpp:320-321), host only.
inline void build_and_save_table(int order, int elements, const std::string& path,
                                 TableFormat format = TableFormat::Text) {
  check(sfem_cuda_table_file_build(order, elements, path.c_str(), static_cast<int>(format)));
}

// TableSet(cache_dir, write_cache) as the reference's constructor (poisson.hpp:50-52): the
// cache directory is set on the context, so the plans built on it use it too.
class TableSet {
 public:
  explicit TableSet(Context& ctx = default_context(), const std::string& cache_dir = {}, bool write_cache = false,
                    TableFormat format = TableFormat::Binary)
      : ctx_(ctx) {
    if (!cache_dir.empty())
      check(sfem_cuda_ctx_set_table_cache(ctx.handle(), cache_dir.c_str(),
                                          (write_cache ? SFEM_TABLE_CACHE_WRITE : 0) |
                                              (format == TableFormat::Binary ? SFEM_TABLE_CACHE_BINARY : 0)));
  }
  const SpectralTable& get(int order, int elements) {
    auto key = std::make_pair(order, elements);
    auto it = tables_.find(key);
    if (it == tables_.end()) it = tables_.emplace(key, std::make_unique<SpectralTable>(ctx_, order, elements)).first;
    return *it->second;
  }
  Context& context() { return ctx_; }

 private:
  Context& ctx_;
  std::map<std::pair<int, int>, std::unique_ptr<SpectralTable>> tables_;
};

// ---------------------------------------------------------------------------
// 1D API (eigenbasis.hpp:50-79)
// ---------------------------------------------------------------------------
namespace lines {
// `count` dof-layout lines of length n*K-1 (line-major) -> coefficients, etc.
inline void decompose_weighted(const SpectralTable& t, const double* in, double* out, long long count = 1) {
  check(sfem_cuda_lines_host(t.handle(), SFEM_OP_DECOMPOSE_WEIGHTED, count, in, out));
}
inline void decompose(const SpectralTable& t, const double* in, double* out, long long count = 1) {
  check(sfem_cuda_lines_host(t.handle(), SFEM_OP_DECOMPOSE, count, in, out));
}
inline void synthesize(const SpectralTable& t, const double* in, double* out, long long count = 1) {
  check(sfem_cuda_lines_host(t.handle(), SFEM_OP_SYNTHESIZE, count, in, out));
}
}  // namespace lines

inline GridFunction1D synthesize(const CoefficientArray1D& coeffs, const SpectralTable& table) {
  require(coeffs.order == table.order && coeffs.elements == table.elements,
          "synthesize: coefficient array does not match the table");
  std::vector<double> v(coeffs.data.size());
  lines::synthesize(table, coeffs.data.data(), v.data());
  return GridFunction1D::from_dof(v.data(), table.order, table.elements);
}

inline CoefficientArray1D decompose_weighted(const GridFunction1D& y, const SpectralTable& table) {
  require(y.order == table.order && y.elements == table.elements,
          "decompose_weighted: grid function does not match the table");
  CoefficientArray1D c = CoefficientArray1D::zeros(table.order, table.elements);
  const std::vector<double> v = y.to_dof();
  lines::decompose_weighted(table, v.data(), c.data.data());
  return c;
}

// apply_mass_1d / apply_stiffness_1d (grid1d.hpp:66-69), on the device; the
// element matrices are those of the table's order.
inline GridFunction1D apply_mass_1d(const GridFunction1D& v, const SpectralTable& table) {
  require(v.order == table.order, "apply_mass_1d: order mismatch");
  std::vector<double> x = v.to_dof(), y(x.size());
  check(sfem_cuda_lines_host(table.handle(), SFEM_OP_APPLY_MASS, 1, x.data(), y.data()));
  return GridFunction1D::from_dof(y.data(), v.order, v.elements);
}
inline GridFunction1D apply_stiffness_1d(const GridFunction1D& v, const SpectralTable& table) {
  require(v.order == table.order, "apply_stiffness_1d: order mismatch");
  std::vector<double> x = v.to_dof(), y(x.size());
  check(sfem_cuda_lines_host(table.handle(), SFEM_OP_APPLY_STIFFNESS, 1, x.data(), y.data()));
  return GridFunction1D::from_dof(y.data(), v.order, v.elements);
}

// materialize_eigenvector (spectral.hpp:330)
inline GridFunction1D materialize_eigenvector(const SpectralTable& table, int k, int l) {
  std::vector<double> y(table.coeff_count());
  check(sfem_cuda_table_eigenvector(table.handle(), k, l, y.data()));
  return GridFunction1D::from_dof(y.data(), table.order, table.elements);
}

// DirectRoute (eigenbasis.hpp:28): Spectral runs F_n, MassApply the mass
// operator followed by FC_n (the reference's cross-check route).
enum class DirectRoute { Spectral, MassApply };

inline CoefficientArray1D decompose(const GridFunction1D& w, const SpectralTable& table,
                                    DirectRoute route = DirectRoute::Spectral) {
  require(w.order == table.order && w.elements == table.elements,
          "decompose: grid function does not match the table");
  if (route == DirectRoute::MassApply) return decompose_weighted(apply_mass_1d(w, table), table);
  CoefficientArray1D c = CoefficientArray1D::zeros(table.order, table.elements);
  const std::vector<double> v = w.to_dof();
  lines::decompose(table, v.data(), c.data.data());
  return c;
}

// ---------------------------------------------------------------------------
// N-D problem (poisson.hpp:29-91, ndgrid.hpp:18-57)
// ---------------------------------------------------------------------------
struct AxisSpec {
  int elements = 0, order = 0;
  int nodal_extent() const { return elements + 1; }
  int interior_extent() const { return elements * (order - 1); }
  int dof_extent() const { return elements * order - 1; }
};

struct GridFunctionND {
  std::vector<AxisSpec> axes;
  std::vector<std::vector<double>> classes;  // 2^N; mask bit i = interior on axis i
  int dim() const { return static_cast<int>(axes.size()); }
  std::vector<int> class_extents(unsigned mask) const {
    std::vector<int> e(axes.size());
    for (size_t i = 0; i < axes.size(); ++i)
      e[i] = (mask >> i & 1u) ? axes[i].interior_extent() : axes[i].nodal_extent();
    return e;
  }
  static GridFunctionND zeros(std::vector<AxisSpec> axes) {
    GridFunctionND g;
    g.axes = std::move(axes);
    g.classes.resize(size_t{1} << g.axes.size());
    for (unsigned mask = 0; mask < g.classes.size(); ++mask) {
      size_t total = 1;
      for (int e : g.class_extents(mask)) total *= static_cast<size_t>(e);
      g.classes[mask].assign(total, 0.0);
    }
    return g;
  }
};

enum class Algorithm { FullDiagonalization, PartialDiagonalization };

struct ProblemSpec {
  int dimension = 0;
  std::vector<double> lengths;       // X_i > 0
  std::vector<int> elements;         // K_i >= 2
  std::vector<int> orders;           // n_i in 1..9
  double shift = 0;                  // alpha
  std::vector<double> coefficients;  // a_i (empty = all ones; the reference's case)

  std::vector<AxisSpec> axis_specs() const {
    std::vector<AxisSpec> a(dimension);
    for (int i = 0; i < dimension; ++i) a[i] = AxisSpec{elements[i], orders[i]};
    return a;
  }
  double shift_lower_bound() const {
    double s = 0;
    for (int i = 0; i < dimension; ++i)
      s += (coefficients.empty() ? 1.0 : coefficients[i]) / (lengths[i] * lengths[i]);
    return -M_PI * M_PI * s;
  }
  void validate() const {  // poisson.cpp:32-47
    require(dimension >= 1, "problem: dimension must be at least 1");
    require(static_cast<int>(lengths.size()) == dimension && static_cast<int>(elements.size()) == dimension &&
                static_cast<int>(orders.size()) == dimension,
            "problem: lengths/elements/orders must all have `dimension` entries");
    for (int i = 0; i < dimension; ++i) {
      require(lengths[i] > 0, "problem: box length must be positive (axis " + std::to_string(i + 1) + ")");
      require(elements[i] >= 2, "problem: need at least 2 elements (axis " + std::to_string(i + 1) + ")");
      require(orders[i] >= 1 && orders[i] <= 9, "problem: order out of range (axis " + std::to_string(i + 1) + ")");
    }
    if (!(shift > shift_lower_bound()))
      fail("problem: shift " + std::to_string(shift) + " must exceed " + std::to_string(shift_lower_bound()) +
           " for a positive definite operator");
  }
};

struct SolveOptions {
  Algorithm algorithm = Algorithm::FullDiagonalization;
  int threads = 0;  // accepted for interface parity (device parallelism is fixed)
  bool compute_residual = false;
  TableSet* tables = nullptr;
};

struct SolveReport {
  GridFunctionND solution;
  double seconds_solve = 0;
  double seconds_load = 0;
  std::optional<double> residual_rel;
  std::optional<double> error_uniform;
};

// A built-in right-hand side: the device stand-in for ProblemSpec::rhs /
// exact (poisson.hpp:39-40), see sfem_cuda_fem_load.
struct Field {
  int kind = SFEM_FIELD_CONSTANT;
  std::vector<double> params{1.0};
  static Field constant(double v) { return Field{SFEM_FIELD_CONSTANT, {v}}; }
  static Field sines(double amp, const std::vector<double>& k) {
    Field f{SFEM_FIELD_SINES, {amp}};
    f.params.insert(f.params.end(), k.begin(), k.end());
    return f;
  }
  // the reference's manufactured cases by name (cases.cpp:61-78)
  static Field manufactured(const std::string& name) {
    if (name == "sin1d") return Field{SFEM_FIELD_SIN1D, {}};
    if (name == "poisson2d") return Field{SFEM_FIELD_POISSON2D, {}};
    if (name == "poisson3d") return Field{SFEM_FIELD_POISSON3D, {}};
    if (name == "constant1d" || name == "constant2d" || name == "constant3d") return constant(1.0);
    fail("unknown case '" + name + "' (known: sin1d, poisson2d, poisson3d, constant1d, constant2d, constant3d)");
  }
};

// dense dof tensor <-> 2^N class arrays (per axis: dof t with t % n == n-1 is
// node (t+1)/n, else interior index (t/n)*(n-1) + t%n; ndgrid.hpp:43-57)
inline GridFunctionND classes_from_dof(const std::vector<AxisSpec>& axes, const std::vector<double>& dof) {
  GridFunctionND g = GridFunctionND::zeros(axes);
  const int N = static_cast<int>(axes.size());
  std::vector<long long> ext(N);
  for (int i = 0; i < N; ++i) ext[i] = static_cast<long long>(axes[i].order) * axes[i].elements - 1;
  std::vector<long long> t(N, 0);
  for (size_t flat = 0; flat < dof.size(); ++flat) {
    unsigned mask = 0;
    long long off = 0;
    for (int i = 0; i < N; ++i) {
      const int n = axes[i].order;
      const bool node = t[i] % n == n - 1;
      if (!node) mask |= 1u << i;
    }
    const std::vector<int> cext = g.class_extents(mask);
    for (int i = 0; i < N; ++i) {
      const int n = axes[i].order;
      const long long idx = (t[i] % n == n - 1) ? (t[i] + 1) / n : (t[i] / n) * (n - 1) + t[i] % n;
      off = off * cext[i] + idx;
    }
    g.classes[mask][static_cast<size_t>(off)] = dof[flat];
    for (int i = N - 1; i >= 0; --i) {
      if (++t[i] < ext[i]) break;
      t[i] = 0;
    }
  }
  return g;
}

// A device plan for one ProblemSpec (sfem_cuda_plan_create).
class Plan {
 public:
  Plan(Context& ctx, const ProblemSpec& spec) : spec_(spec) {
    spec.validate();
    check(sfem_cuda_plan_create(ctx.handle(), spec.dimension, spec.orders.data(), spec.elements.data(),
                                spec.lengths.data(), spec.coefficients.empty() ? nullptr : spec.coefficients.data(),
                                spec.shift, &h_));
  }
  ~Plan() { sfem_cuda_plan_destroy(h_); }
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;
  sfem_plan handle() const { return h_; }
  // SolveOptions::algorithm (poisson.hpp:64-70): FullDiagonalization (a) or
  // PartialDiagonalization (b, poisson.cpp:671-745; dimension >= 2)
  void set_algorithm(Algorithm a) {
    check(sfem_cuda_plan_set_algorithm(h_, a == Algorithm::FullDiagonalization ? 0 : 1));
  }
  // dense dof-layout load -> u (host buffers); returns device-timed seconds
  double solve_dof(const double* load, double* u) {
    double sec = 0;
    check(sfem_cuda_solve_host(h_, load, u, &sec));
    return sec;
  }
  long long unknowns() const {
    long long u = 0;
    check(sfem_cuda_plan_shape(h_, nullptr, nullptr, &u));
    return u;
  }
  // y = A v on dense dof tensors (apply_operator, poisson.cpp:749-769)
  void apply_operator_dof(const double* v, double* y) { check(sfem_cuda_apply_operator_host(h_, v, y)); }
  // the reference's solve(spec, options) of a field, every step on the device
  SolveReport solve_field(const Field& f, bool compute_residual) {
    std::vector<double> u(static_cast<size_t>(unknowns()));
    double rep[4];
    check(sfem_cuda_solve_field(h_, f.kind, f.params.empty() ? nullptr : f.params.data(),
                                static_cast<int>(f.params.size()), compute_residual ? 1 : 0, u.data(), rep));
    SolveReport r;
    r.solution = classes_from_dof(spec_.axis_specs(), u);
    r.seconds_load = rep[0];
    r.seconds_solve = rep[1];
    if (!std::isnan(rep[2])) r.residual_rel = rep[2];
    if (!std::isnan(rep[3])) r.error_uniform = rep[3];
    return r;
  }
  GridFunctionND solve_classes(const GridFunctionND& load, double* seconds) {
    GridFunctionND out = GridFunctionND::zeros(spec_.axis_specs());
    std::vector<const double*> in(load.classes.size());
    std::vector<double*> o(out.classes.size());
    for (size_t i = 0; i < in.size(); ++i) {
      in[i] = load.classes[i].data();
      o[i] = out.classes[i].data();
    }
    check(sfem_cuda_solve_classes(h_, in.data(), o.data(), seconds));
    return out;
  }

 private:
  ProblemSpec spec_;
  sfem_plan h_ = nullptr;
};

// solve_with_load (poisson.hpp:90-91), algorithm (a) on the GPU.
inline SolveReport solve_with_load(const ProblemSpec& spec, const GridFunctionND& load, TableSet& tables,
                                   const SolveOptions& options = {}) {
  spec.validate();
  require(load.dim() == spec.dimension, "solve: load dimension does not match the problem");
  Plan plan(tables.context(), spec);
  plan.set_algorithm(options.algorithm);
  SolveReport r;
  r.solution = plan.solve_classes(load, &r.seconds_solve);
  return r;
}

// solve (poisson.hpp:86; poisson.cpp:796-808): FEM load of `rhs`, the solve,
// and on request the residual check / uniform error, all on the GPU.
inline SolveReport solve(const ProblemSpec& spec, const Field& rhs, const SolveOptions& options = {}) {
  spec.validate();
  static TableSet local;
  TableSet& tables = options.tables ? *options.tables : local;
  Plan plan(tables.context(), spec);
  plan.set_algorithm(options.algorithm);
  return plan.solve_field(rhs, options.compute_residual);
}

}  // namespace sfem_b200
