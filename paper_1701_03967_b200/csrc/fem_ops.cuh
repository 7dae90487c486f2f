// Device FEM load averaging, operator application and residual / error
// reductions (fem_ops.cu).
#pragma once

#include <cuda_runtime.h>

#include "sweep.cuh"

namespace sfem_b200 {

constexpr int kMaxNP = 10;  // n + 1 for n <= 9

enum FieldKind { kFieldConstant = 0, kFieldSines = 1, kFieldSin1d = 2, kFieldPoisson2d = 3, kFieldPoisson3d = 4 };

// A right-hand side / manufactured solution.  kFieldConstant: p[0].
// kFieldSines: p[0] amp, p[1..dim] wave numbers k_i (f = amp prod sin(k_i pi x_i)),
// p[1 + kMaxDim] the exact solution's amplitude.  Cases: shift (the plan's).
struct FieldArgs {
  int kind, dim;
  double shift;
  double p[2 + kMaxDim];
};

// Load averaging geometry: per axis order n, np = n + 1 Gauss points, K,
// h, dof extent / stride of the output tensor, Gauss nodes and the weighted
// basis wq[loc * np + g] = w_g phi_loc(xi_g) (poisson.cpp:481-495).
struct LoadArgs {
  int dim;
  int n[kMaxDim], np[kMaxDim], K[kMaxDim];
  double h[kMaxDim];
  long long ext[kMaxDim], st[kMaxDim];
  double gnode[kMaxDim][kMaxNP];
  double wq[kMaxDim][kMaxNP * kMaxNP];
};

// One operator sweep along an axis of a dof tensor: lines = outer x inner
// (strided: line start o*L*inner + i, position stride inner; rows: outer rows
// at o*pitch), element matrices M (mass) and S (stiffness) of order n, fac =
// f_axis, shift (first sweep only).  Padding columns (i % pitch >= last) are
// skipped.
struct OpAxisArgs {
  int n, K;
  long long L, outer, inner, pitch, last;
  double fac, shift;
  double M[kMaxNP][kMaxNP], S[kMaxNP][kMaxNP];
};

// Separable load: out[t] = amp * prod_i B_i[t_i] over the padded tensor
// (total = rows * pitch elements; padding written as zero).
struct SepArgs {
  int dim;
  long long total;
  double amp;
  long long ext[kMaxDim], st[kMaxDim], boff[kMaxDim];
  long long pitch;
};

struct ErrArgs {
  int dim;
  long long total;
  int n[kMaxDim];
  long long ext[kMaxDim], st[kMaxDim];
  double h[kMaxDim];
};

cudaError_t launch_op_axis(const double* pin, double* pout, double* q, const double* f, const OpAxisArgs& a,
                           bool rows, bool first, bool last, bool resid, unsigned long long* red, cudaStream_t s);
cudaError_t launch_fem_load(double* out, const LoadArgs& a, const FieldArgs& fa, int num_sms, cudaStream_t s);
cudaError_t launch_fem_load_separable(double* out, const double* Bv, const SepArgs& a, int num_sms, cudaStream_t s);
cudaError_t launch_max_error(const double* u, const ErrArgs& a, const FieldArgs& fa, unsigned long long* red,
                             int num_sms, cudaStream_t s);

}  // namespace sfem_b200
