// Algorithm (b)'s line solves along axis 0 (banded.cu).
#pragma once

#include <cuda_runtime.h>

#include "sweep.cuh"

namespace sfem_b200 {

constexpr int kMaxM = 8;  // n - 1 for n <= 9

// One axis-0 solve over a dof tensor: lines o * L * inner + i (i < inner,
// padding columns i % pitch >= last skipped), position stride inner.  The
// axis-0 element data: order n, K elements, f0 = a0 * 4 / h0^2, corner /
// cross entries of the element stiffness (A) and mass (C), the interior
// eigenbasis V[c][l] (C-orthonormal), its eigenvalues lam, and the projected
// edge columns P*0[l] = sum_c V[c][l] *[1 + c][0], P*n[l] = ... [1 + c][n].
// sigma of a line = shift + sum_{ax = nfreq-1 .. 0} f[ax] eig[ax][t_ax], t
// decoded from i row-major over fext (the last with extent pitch).
struct BandArgs {
  int n, K;
  long long L, inner, outer, pitch, last;
  double f0, shift;
  int nfreq;
  long long fext[kMaxDim];
  const double* eig[kMaxDim];
  double f[kMaxDim];
  double A00, A0n, C00, C0n;
  double lam[kMaxM], PA0[kMaxM], PAn[kMaxM], PC0[kMaxM], PCn[kMaxM];
  double V[kMaxM][kMaxM];
};

// cbuf: K * inner * outer doubles of Thomas coefficients.  *fail receives
// the smallest failing line index (atomicMin) when a pivot is not positive.
cudaError_t launch_band_lines(double* data, double* cbuf, const BandArgs& a, unsigned long long* fail,
                              cudaStream_t s);

}  // namespace sfem_b200
