// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE, not product code.
//
// A thin C-ABI over the reference's own library, compiled from the reference
// sources where they lie (/root/reference/proj/src, see oracle/Makefile) into
// oracle/_ref/libsfem_ref.so.  Only tests/, __graft_entry__.smoke() and the
// CPU legs of bench.py load it, and only as the checker / CPU baseline.
//
// Data crosses this boundary in the interleaved dof layout (per axis, dof
// t = e*n + c is interior component c of element e, t = j*n - 1 is node j;
// extent n*K-1, last axis fastest) -- the same layout the product uses.  The
// class-array <-> dof mapping restates oracle::pack_nd / unpack_nd
// (reference proj/src/oracle.cpp:86-144) and gather/scatter_dof_line
// (proj/src/banded.cpp:87-107, called directly).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "sfem/banded.hpp"
#include "sfem/cases.hpp"
#include "sfem/eigenbasis.hpp"
#include "sfem/grid1d.hpp"
#include "sfem/poisson.hpp"
#include "sfem/spectral.hpp"
#include "sfem/trig.hpp"

using namespace sfem;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Per-axis map dof index -> (interior flag, class index); proj/src/oracle.cpp:89-107.
struct AxisMap {
  std::vector<std::int64_t> cls;
  std::vector<unsigned char> interior;
  AxisMap(int n, int K) {
    const int L = n * K - 1;
    cls.resize(L);
    interior.resize(L);
    for (int t = 0; t < L; ++t) {
      const int r = t % n;
      if (r == n - 1) {
        interior[t] = 0;
        cls[t] = t / n + 1;
      } else {
        interior[t] = 1;
        cls[t] = static_cast<std::int64_t>(t / n) * (n - 1) + r;
      }
    }
  }
};

// Walk every dof of the tensor and hand (flat dof index, class mask, class offset) to f.
template <class F>
void for_each_dof(const std::vector<AxisSpec>& axes, F&& f) {
  const int N = static_cast<int>(axes.size());
  std::vector<AxisMap> maps;
  std::vector<int> ext(N);
  for (int i = 0; i < N; ++i) {
    maps.emplace_back(axes[i].order, axes[i].elements);
    ext[i] = axes[i].dof_extent();
  }
  const unsigned nclass = 1u << N;
  std::vector<TensorShape> shapes;
  for (unsigned mask = 0; mask < nclass; ++mask) {
    std::vector<int> ce(N);
    for (int i = 0; i < N; ++i)
      ce[i] = (mask >> i & 1u) ? axes[i].interior_extent() : axes[i].nodal_extent();
    shapes.emplace_back(ce);
  }
  const TensorShape shape(ext);
  // Parallel over the slowest axis.
#pragma omp parallel for schedule(static)
  for (int i0 = 0; i0 < ext[0]; ++i0) {
    std::vector<int> idx(N, 0);
    idx[0] = i0;
    const std::int64_t inner = shape.total / ext[0];
    for (std::int64_t r = 0; r < inner; ++r) {
      unsigned mask = 0;
      for (int i = 0; i < N; ++i)
        if (maps[i].interior[idx[i]]) mask |= 1u << i;
      std::int64_t off = 0;
      for (int i = 0; i < N; ++i) off += maps[i].cls[idx[i]] * shapes[mask].stride[i];
      f(static_cast<std::int64_t>(i0) * inner + r, mask, off);
      for (int i = N - 1; i >= 1; --i) {
        if (++idx[i] < ext[i]) break;
        idx[i] = 0;
      }
    }
  }
}

GridFunctionND grid_from_dof(const std::vector<AxisSpec>& axes, const double* dof) {
  GridFunctionND g = GridFunctionND::zeros(axes);
  for_each_dof(axes, [&](std::int64_t flat, unsigned mask, std::int64_t off) {
    g.classes[mask][off] = dof[flat];
  });
  return g;
}

void grid_to_dof(const GridFunctionND& g, double* dof) {
  for_each_dof(g.axes, [&](std::int64_t flat, unsigned mask, std::int64_t off) {
    dof[flat] = g.classes[mask][off];
  });
}

ProblemSpec make_spec(int dim, const int* orders, const int* elements, const double* lengths, double shift) {
  ProblemSpec spec;
  spec.dimension = dim;
  spec.orders.assign(orders, orders + dim);
  spec.elements.assign(elements, elements + dim);
  spec.lengths.assign(lengths, lengths + dim);
  spec.shift = shift;
  return spec;
}

void export_table(const SpectralTable1D& t, double* theta, double* half_cos, double* half_sin, double* values,
                  double* norm_sq, double* nodal_weight, double* p, double* q, double* interior_values,
                  double* interior_vectors, double* eig_coeff) {
  const int m = t.order - 1;
  auto cp = [](const std::vector<double>& v, double* dst) {
    if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(double));
  };
  cp(t.theta, theta);
  cp(t.half_cos, half_cos);
  cp(t.half_sin, half_sin);
  cp(t.values, values);
  cp(t.norm_sq, norm_sq);
  cp(t.nodal_weight, nodal_weight);
  cp(t.p, p);
  cp(t.q, q);
  if (m > 0) {
    cp(t.interior.values, interior_values);
    cp(t.interior.vectors.a, interior_vectors);
  }
  cp(t.eigenvalues_coeff_order(), eig_coeff);
}

TableSet& tables() {
  static TableSet t;
  return t;
}

}  // namespace

extern "C" {

const char* sfemref_last_error() { return g_err.c_str(); }

int sfemref_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

unsigned long long sfemref_trig_invocations() { return trig::invocation_count(); }

// kind 0: dst1 (len = K-1), 1: dst3_synthesis (len = K), 2: dct3_synthesis (len = K).
int sfemref_trig(int kind, int len, const double* in, double* out) {
  return guarded([&] {
    std::vector<double> r;
    std::span<const double> x(in, static_cast<size_t>(len));
    if (kind == 0) r = trig::dst1(x);
    else if (kind == 1) r = trig::dst3_synthesis(x);
    else r = trig::dct3_synthesis(x);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

// Table export (spectral.hpp:281-312).  Arrays sized by the caller:
// theta/half_cos/half_sin K-1; values/norm_sq/nodal_weight (K-1)n;
// p/q (K-1)n(n-1); interior_values n-1; interior_vectors (n-1)^2 row-major
// (row i, column l-1 = e^(l)); eig_coeff nK-1.
int sfemref_table(int n, int K, double* theta, double* half_cos, double* half_sin, double* values,
                  double* norm_sq, double* nodal_weight, double* p, double* q, double* interior_values,
                  double* interior_vectors, double* eig_coeff) {
  return guarded([&] {
    export_table(tables().get(n, K), theta, half_cos, half_sin, values, norm_sq, nodal_weight, p, q,
                 interior_values, interior_vectors, eig_coeff);
  });
}

// Table files (spectral.cpp:81-236): save_table of the (memoised) table.
int sfemref_save_table(int n, int K, const char* path) {
  return guarded([&] { save_table(tables().get(n, K), path); });
}

// load_table, then the export of sfemref_table.
int sfemref_load_table(const char* path, int n, int K, double* theta, double* half_cos, double* half_sin,
                       double* values, double* norm_sq, double* nodal_weight, double* p, double* q,
                       double* interior_values, double* interior_vectors, double* eig_coeff) {
  return guarded([&] {
    const SpectralTable1D t = load_table(path, n, K);
    export_table(t, theta, half_cos, half_sin, values, norm_sq, nodal_weight, p, q, interior_values,
                 interior_vectors, eig_coeff);
  });
}

// A fresh TableSet over a cache directory (poisson.cpp:49-73), then the export.
int sfemref_tableset_get(const char* dir, int write_cache, int n, int K, double* theta, double* half_cos,
                         double* half_sin, double* values, double* norm_sq, double* nodal_weight, double* p,
                         double* q, double* interior_values, double* interior_vectors, double* eig_coeff) {
  return guarded([&] {
    TableSet ts(Precision::Double, dir, write_cache != 0);
    export_table(ts.get(n, K), theta, half_cos, half_sin, values, norm_sq, nodal_weight, p, q, interior_values,
                 interior_vectors, eig_coeff);
  });
}

// apply_mass_1d (kind 0) / apply_stiffness_1d (kind 1) (grid1d.cpp:33-47) on
// `count` dof-layout lines.
int sfemref_apply_1d(int kind, int n, int K, long long count, const double* in, double* out) {
  return guarded([&] {
    const SpectralTable1D& t = tables().get(n, K);
    const int L = n * K - 1;
    for (long long b = 0; b < count; ++b) {
      GridFunction1D g = GridFunction1D::zeros(n, K);
      scatter_dof_line(n, K, in + b * L, g.nodal.data(), 1, g.interior.data(), 1);
      const GridFunction1D y = kind == 0 ? apply_mass_1d(g, t.element) : apply_stiffness_1d(g, t.element);
      gather_dof_line(n, K, y.nodal.data(), 1, y.interior.data(), 1, out + b * L);
    }
  });
}

// materialize_eigenvector (spectral.cpp:238-265), dof layout.
int sfemref_eigenvector(int n, int K, int k, int l, double* out) {
  return guarded([&] {
    const GridFunction1D g = materialize_eigenvector(tables().get(n, K), k, l);
    gather_dof_line(n, K, g.nodal.data(), 1, g.interior.data(), 1, out);
  });
}

// Element matrices (element.hpp:258-295), (n+1)^2 row-major each.
int sfemref_element(int n, double* stiffness, double* mass) {
  return guarded([&] {
    const ElementMatrices em = build_element_matrices<double>(n);
    std::memcpy(stiffness, em.stiffness.a.data(), em.stiffness.a.size() * sizeof(double));
    std::memcpy(mass, em.mass.a.data(), em.mass.a.size() * sizeof(double));
  });
}

// 1D line transforms on a line-major batch in dof layout (length nK-1 each).
// op 0: lines::decompose_weighted (eigenbasis.cpp:63-101)
// op 1: lines::decompose          (eigenbasis.cpp:103-142)
// op 2: lines::synthesize         (eigenbasis.cpp:144-225)
// op 3: lines::decompose_weighted_block (248-331), 32-line slot-major tiles
// op 4: lines::synthesize_block (333-444), 32-line tiles
int sfemref_lines(int op, int n, int K, long long count, const double* in, double* out) {
  return guarded([&] {
    const SpectralTable1D& t = tables().get(n, K);
    const int L = n * K - 1, m = n - 1;
    if (op <= 2) {
#pragma omp parallel
      {
        LineWork w;
        std::vector<double> nodal(K + 1), inter(static_cast<size_t>(K) * m), coef(L);
#pragma omp for schedule(static)
        for (long long b = 0; b < count; ++b) {
          const double* src = in + b * L;
          double* dst = out + b * L;
          if (op == 2) {
            lines::synthesize(t, src, nodal.data(), inter.data(), w);
            gather_dof_line(n, K, nodal.data(), 1, inter.data(), 1, dst);
          } else {
            scatter_dof_line(n, K, src, nodal.data(), 1, inter.data(), 1);
            if (op == 0) lines::decompose_weighted(t, nodal.data(), inter.data(), dst, w);
            else lines::decompose(t, nodal.data(), inter.data(), dst, w);
          }
        }
      }
    } else {
      const int B = 32;
#pragma omp parallel
      {
        lines::BlockWork w;
        std::vector<double> nodal(static_cast<size_t>(K + 1) * B), inter(static_cast<size_t>(K) * m * B),
            coef(static_cast<size_t>(L) * B), tmp(L);
#pragma omp for schedule(static)
        for (long long b0 = 0; b0 < count; b0 += B) {
          const int c = static_cast<int>(std::min<long long>(B, count - b0));
          if (op == 3) {
            for (int b = 0; b < c; ++b) {
              std::vector<double> nd(K + 1), it(static_cast<size_t>(K) * m);
              scatter_dof_line(n, K, in + (b0 + b) * L, nd.data(), 1, it.data(), 1);
              for (int j = 0; j <= K; ++j) nodal[static_cast<size_t>(j) * c + b] = nd[j];
              for (size_t j = 0; j < it.size(); ++j) inter[j * c + b] = it[j];
            }
            lines::decompose_weighted_block(t, nodal.data(), inter.data(), coef.data(), c, w);
            for (int b = 0; b < c; ++b)
              for (int j = 0; j < L; ++j) out[(b0 + b) * L + j] = coef[static_cast<size_t>(j) * c + b];
          } else {
            for (int b = 0; b < c; ++b)
              for (int j = 0; j < L; ++j) coef[static_cast<size_t>(j) * c + b] = in[(b0 + b) * L + j];
            lines::synthesize_block(t, coef.data(), nodal.data(), inter.data(), c, w);
            for (int b = 0; b < c; ++b) {
              std::vector<double> nd(K + 1), it(static_cast<size_t>(K) * m);
              for (int j = 0; j <= K; ++j) nd[j] = nodal[static_cast<size_t>(j) * c + b];
              for (size_t j = 0; j < it.size(); ++j) it[j] = inter[j * c + b];
              gather_dof_line(n, K, nd.data(), 1, it.data(), 1, out + (b0 + b) * L);
            }
          }
        }
      }
    }
  });
}

// Full solve, algorithm (a) (poisson.cpp:771-794 -> 637-669) on a dof-layout
// load; u in dof layout.  seconds = SolveReport::seconds_solve.
int sfemref_solve(int dim, const int* orders, const int* elements, const double* lengths, double shift,
                  int algorithm, int threads, const double* load_dof, double* u_dof, double* seconds) {
  return guarded([&] {
    const ProblemSpec spec = make_spec(dim, orders, elements, lengths, shift);
    spec.validate();
    const GridFunctionND load = grid_from_dof(spec.axis_specs(), load_dof);
    SolveOptions opt;
    opt.algorithm = algorithm == 1 ? Algorithm::PartialDiagonalization : Algorithm::FullDiagonalization;
    opt.threads = threads;
    const SolveReport rep = solve_with_load(spec, load, tables(), opt);
    if (seconds) *seconds = rep.seconds_solve;
    grid_to_dof(rep.solution, u_dof);
  });
}

// `reps` timed solve_with_load calls of one load (the bench's CPU legs): the
// dof -> class conversion is done once, each call's own seconds_solve
// (poisson.cpp:781-785) lands in seconds[i]; the tables are built untimed by
// the first call (poisson.cpp:776-779), as in every reference solve.
int sfemref_solve_repeat(int dim, const int* orders, const int* elements, const double* lengths, double shift,
                         int threads, int reps, const double* load_dof, double* seconds) {
  return guarded([&] {
    const ProblemSpec spec = make_spec(dim, orders, elements, lengths, shift);
    spec.validate();
    const GridFunctionND load = grid_from_dof(spec.axis_specs(), load_dof);
    SolveOptions opt;
    opt.algorithm = Algorithm::FullDiagonalization;
    opt.threads = threads;
    for (int r = 0; r < reps; ++r) seconds[r] = solve_with_load(spec, load, tables(), opt).seconds_solve;
  });
}

// Operator apply (poisson.cpp:749-769) on dof-layout data (verification only).
int sfemref_apply_operator(int dim, const int* orders, const int* elements, const double* lengths,
                           double shift, const double* v_dof, double* out_dof) {
  return guarded([&] {
    const ProblemSpec spec = make_spec(dim, orders, elements, lengths, shift);
    const GridFunctionND v = grid_from_dof(spec.axis_specs(), v_dof);
    grid_to_dof(apply_operator(spec, v), out_dof);
  });
}

// FEM load average (poisson.cpp:471-569) of f = amp * prod_i sin(freq_i * pi * x_i)
// on the box `lengths` (config 3: amp = 9 pi^2 + 1, freq = (1, 2), unit square).
int sfemref_fem_load_sines(int dim, const int* orders, const int* elements, const double* lengths,
                           double amp, const double* freq, double* load_dof) {
  return guarded([&] {
    ProblemSpec spec = make_spec(dim, orders, elements, lengths, 0.0);
    std::vector<double> fr(freq, freq + dim);
    spec.rhs = [amp, fr](std::span<const double> x) {
      double v = amp;
      for (size_t i = 0; i < x.size(); ++i) v *= std::sin(fr[i] * M_PI * x[i]);
      return v;
    };
    grid_to_dof(fem_load_average(spec), load_dof);
  });
}

// FEM load average (poisson.cpp:471-569) of a manufactured case's right-hand
// side (make_problem, cases.cpp:81-95: -Lap u + shift u, or 1 for constantNd).
int sfemref_fem_load_case(const char* name, int dim, const int* orders, const int* elements, const double* lengths,
                          double shift, double* load_dof) {
  return guarded([&] {
    const ManufacturedCase& c = manufactured_case(name);
    require(c.dimension == dim, "fem_load_case: dimension mismatch");
    ProblemSpec spec = make_problem(c, shift, std::vector<int>(elements, elements + dim),
                                    std::vector<int>(orders, orders + dim), std::vector<double>(lengths, lengths + dim));
    grid_to_dof(fem_load_average(spec), load_dof);
  });
}

// The reference's end-to-end solve(spec, options) (poisson.cpp:796-808) of a
// manufactured case with compute_residual: solution (dof layout),
// residual_rel and error_uniform (NaN when the case has no exact solution).
int sfemref_solve_case(const char* name, int dim, const int* orders, const int* elements, const double* lengths,
                       double shift, double* u_dof, double* residual_rel, double* error_uniform) {
  return guarded([&] {
    const ManufacturedCase& c = manufactured_case(name);
    require(c.dimension == dim, "solve_case: dimension mismatch");
    ProblemSpec spec = make_problem(c, shift, std::vector<int>(elements, elements + dim),
                                    std::vector<int>(orders, orders + dim), std::vector<double>(lengths, lengths + dim));
    SolveOptions opt;
    opt.compute_residual = true;
    const SolveReport rep = solve(spec, opt);
    grid_to_dof(rep.solution, u_dof);
    *residual_rel = rep.residual_rel.value_or(std::nan(""));
    *error_uniform = rep.error_uniform.value_or(std::nan(""));
  });
}

// The reference's fixture generator: std::mt19937(seed) +
// uniform_real_distribution(lo, hi) (test_trig.cpp:14-20, verify.cpp:43-49).
void sfemref_uniform(unsigned seed, long long count, double lo, double hi, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(lo, hi);
  for (long long i = 0; i < count; ++i) out[i] = u(rng);
}

}  // extern "C"
