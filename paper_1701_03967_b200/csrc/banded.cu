// Algorithm (b), partial diagonalisation (reference run_partial_diagonalization,
// poisson.cpp:671-745): after the forward expansions along axes 1..N-1, every
// line along axis 0 solves (f0 A + sigma C) u = rhs with sigma = shift +
// sum_{i>=1} f_i lambda_i[t_i] (summed i = N-1 .. 1, poisson.cpp:703-710).
// The reference factors the assembled band matrix per line (band_cholesky /
// band_solve, banded.cpp:48-85).  Here the element structure is used instead:
//
//   * the interior block K_ii = f0 A_ii + sigma C_ii of every element is
//     diagonal in the interior eigenbasis V (A_ii V = C_ii V Lambda,
//     V^T C_ii V = I; the table's interior eigensystem), so
//     K_ii^-1 = V diag(1 / (f0 lambda_l + sigma)) V^T -- no per-line
//     factorisation, V is line-independent (kernel parameter, broadcast);
//   * eliminating the interiors (static condensation) leaves a symmetric
//     tridiagonal system on the nodes with constant coefficients
//     D = S00 + S11, E = S01 (S the element Schur complement), solved by the
//     Thomas recurrence;
//   * one thread per line, lanes over the contiguous last-axis index
//     (coalesced), two passes along the line: forward (r = V^T f_int stored
//     in place of f_int, condensed rhs, Thomas forward: d' in place of the
//     nodal rhs, c' to a scratch column), backward (nodal u, then
//     u_int = V (diag(D) (r - u_l q0 - u_r qn))).
//
// Same solution as the band Cholesky up to rounding (both are backward
// stable eliminations of an SPD system); tests compare with the reference's
// algorithm (b) and with algorithm (a).
#include <cuda_runtime.h>

#include "banded.cuh"

namespace sfem_b200 {
namespace band {

template <int NP>
__global__ void __launch_bounds__(128) band_lines(double* data, double* cbuf, const __grid_constant__ BandArgs a,
                                                  unsigned long long* fail) {
  constexpr int n = NP - 1, m = NP - 2 > 0 ? NP - 2 : 0, MM = m > 0 ? m : 1;
  const long long nl = a.inner * a.outer;
  const long long line = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (line >= nl) return;
  const long long o = line / a.inner, i = line - o * a.inner;
  if (i % a.pitch >= a.last) return;  // padding column of the last axis
  // sigma = shift + sum_{i = N-1 .. 1} f_i lambda_i[t_i] (reference order)
  double sigma = a.shift;
  {
    long long rem = i;
    for (int ax = a.nfreq - 1; ax >= 0; --ax) {
      const long long ext = ax == a.nfreq - 1 ? a.pitch : a.fext[ax];
      const long long t = rem % ext;
      rem /= ext;
      sigma += a.f[ax] * a.eig[ax][t];
    }
  }
  const double f0 = a.f0;
  double Dl[MM], q0[MM], qn[MM];
  double S00 = f0 * a.A00 + sigma * a.C00, S01 = f0 * a.A0n + sigma * a.C0n, S11 = S00;
#pragma unroll
  for (int l = 0; l < m; ++l) {
    const double den = fma(f0, a.lam[l], sigma);
    if (!(den > 0)) atomicMin(fail, static_cast<unsigned long long>(line));
    Dl[l] = 1.0 / den;
    q0[l] = fma(f0, a.PA0[l], sigma * a.PC0[l]);
    qn[l] = fma(f0, a.PAn[l], sigma * a.PCn[l]);
    S00 -= q0[l] * q0[l] * Dl[l];
    S01 -= q0[l] * qn[l] * Dl[l];
    S11 -= qn[l] * qn[l] * Dl[l];
  }
  const double D = S00 + S11, E = S01;
  const long long st = a.inner;
  double* base = data + o * a.L * a.inner + i;
  double* cb = cbuf + line;
  const long long cst = nl;
  // forward: r_e = V^T f_int(e) in place; g_j = f_j - w_{e-1}[n-side] - w_e[0-side]
  double wprev = 0.0, cprev = 0.0, dprev = 0.0;
  for (int e = 0; e < a.K; ++e) {
    double r[MM];
    double w0 = 0.0, wn = 0.0;
    if (m > 0) {
      double fi[MM];
#pragma unroll
      for (int c = 0; c < m; ++c) fi[c] = base[(static_cast<long long>(e) * n + c) * st];
#pragma unroll
      for (int l = 0; l < m; ++l) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < m; ++c) s = fma(a.V[c][l], fi[c], s);
        r[l] = s;
        w0 = fma(q0[l] * Dl[l], s, w0);
        wn = fma(qn[l] * Dl[l], s, wn);
      }
#pragma unroll
      for (int l = 0; l < m; ++l) base[(static_cast<long long>(e) * n + l) * st] = r[l];
    }
    if (e > 0) {  // node j = e (position e*n - 1): Thomas forward
      const long long pj = (static_cast<long long>(e) * n - 1) * st;
      const double g = base[pj] - wprev - w0;
      const double den = e == 1 ? D : fma(-E, cprev, D);
      if (!(den > 0)) atomicMin(fail, static_cast<unsigned long long>(line));
      const double inv = 1.0 / den;
      const double c = E * inv;
      const double d = (e == 1 ? g : fma(-E, dprev, g)) * inv;
      base[pj] = d;
      cb[static_cast<long long>(e) * cst] = c;
      cprev = c;
      dprev = d;
    }
    wprev = wn;
  }
  // backward: nodes K-1 .. 1, interiors K-1 .. 0
  double uright = 0.0;  // node K (boundary)
  for (int e = a.K - 1; e >= 0; --e) {
    double uleft = 0.0;
    if (e > 0) {
      const long long pj = (static_cast<long long>(e) * n - 1) * st;
      const double d = base[pj];
      uleft = e == a.K - 1 ? d : fma(-cb[static_cast<long long>(e) * cst], uright, d);
      base[pj] = uleft;
    }
    if (m > 0) {
      double t[MM];
#pragma unroll
      for (int l = 0; l < m; ++l) {
        const double rl = base[(static_cast<long long>(e) * n + l) * st];
        t[l] = Dl[l] * fma(-uleft, q0[l], fma(-uright, qn[l], rl));
      }
#pragma unroll
      for (int c = 0; c < m; ++c) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < m; ++l) s = fma(a.V[c][l], t[l], s);
        base[(static_cast<long long>(e) * n + c) * st] = s;
      }
    }
    uright = uleft;
  }
}

}  // namespace band

cudaError_t launch_band_lines(double* data, double* cbuf, const BandArgs& a, unsigned long long* fail,
                              cudaStream_t s) {
  const long long nl = a.inner * a.outer;
  const unsigned grid = static_cast<unsigned>((nl + 127) / 128);
  if (grid == 0) return cudaSuccess;
  switch (a.n + 1) {
#define SFEM_BAND_CASE(NP) \
  case NP:                 \
    band::band_lines<NP><<<grid, 128, 0, s>>>(data, cbuf, a, fail); \
    break;
    SFEM_BAND_CASE(2)
    SFEM_BAND_CASE(3)
    SFEM_BAND_CASE(4)
    SFEM_BAND_CASE(5)
    SFEM_BAND_CASE(6)
    SFEM_BAND_CASE(7)
    SFEM_BAND_CASE(8)
    SFEM_BAND_CASE(9)
    SFEM_BAND_CASE(10)
#undef SFEM_BAND_CASE
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace sfem_b200
