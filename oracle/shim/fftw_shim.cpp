// oracle/shim/fftw_shim.cpp -- TEST INFRASTRUCTURE, not product code.
//
// A from-scratch implementation of the FFTW3 r2r entry points the reference's
// trig module binds (reference proj/src/trig.cpp:20-21, 43, 47-48, 56, 76, 91),
// so that the reference's own hot-path translation units can be compiled
// unchanged into oracle/_ref (see oracle/Makefile).  FFTW itself (an unpinned
// dependency, proj/CMakeLists.txt:15-16) is not in this image.
//
// Definitions restated from FFTW's published manual (section "1d Real-odd
// DFTs (DSTs)" / "1d Real-even DFTs (DCTs)"), n = logical length:
//   RODFT00: Y_k = 2 sum_{j=0}^{n-1} X_j sin(pi (j+1)(k+1)/(n+1))
//   RODFT01: Y_k = (-1)^k X_{n-1} + 2 sum_{j=0}^{n-2} X_j sin(pi (j+1)(2k+1)/(2n))
//   REDFT01: Y_k = X_0 + 2 sum_{j=1}^{n-1} X_j cos(pi j (2k+1)/(2n))
// The reference rescales these into the plain sums of trig.hpp:3-7; its own
// tests pin the result (test_trig.cpp:30-102), and tests/test_oracle.py
// re-runs those cases against this shim.
//
// Algorithms: O(n log n) through a mixed-radix complex FFT (radix 4/2/3/5 and
// a generic small-prime DFT).  DST-I uses the real-data recurrence form for
// even n+1 and an odd-extension complex FFT otherwise; DCT-III uses Makhoul's
// n-point reordering; DST-III maps to DCT-III by index reversal.  Execution is
// re-entrant (plans are read-only, scratch is thread_local), as the reference
// requires for its OpenMP sweeps (trig.cpp:22-24).

#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {

using cd = std::complex<double>;

// ---------------------------------------------------------------- complex FFT
struct CFFT {
  int n = 0;
  std::vector<int> fac;
  std::vector<cd> tw;  // exp(-2 pi i t / n), t = 0..n-1

  explicit CFFT(int len) : n(len) {
    int m = len;
    while (m % 4 == 0) { fac.push_back(4); m /= 4; }
    while (m % 2 == 0) { fac.push_back(2); m /= 2; }
    for (int p = 3; m > 1; p += 2)
      while (m % p == 0) { fac.push_back(p); m /= p; }
    tw.resize(n);
    for (int t = 0; t < n; ++t) {
      const long double a = -2.0L * 3.14159265358979323846264338327950288L * t / n;
      tw[t] = cd(static_cast<double>(cosl(a)), static_cast<double>(sinl(a)));
    }
  }

  // out (contiguous, length len) = DFT of in[0], in[is], ..., forward sign.
  void rec(const cd* in, long is, cd* out, int len, int fi, std::vector<cd>& tmp) const {
    if (len == 1) { out[0] = in[0]; return; }
    const int r = fac[fi], m = len / r;
    for (int q = 0; q < r; ++q) rec(in + q * is, is * r, out + q * m, m, fi + 1, tmp);
    const int step = n / len;  // W_len^e = tw[e*step]
    if (r == 2) {
      for (int k = 0; k < m; ++k) {
        const cd a = out[k], b = out[m + k] * tw[k * step];
        out[k] = a + b;
        out[m + k] = a - b;
      }
    } else if (r == 4) {
      for (int k = 0; k < m; ++k) {
        const cd a0 = out[k];
        const cd a1 = out[m + k] * tw[k * step];
        const cd a2 = out[2 * m + k] * tw[2 * k * step];
        const cd a3 = out[3 * m + k] * tw[3 * k * step];
        const cd s02 = a0 + a2, d02 = a0 - a2, s13 = a1 + a3, d13 = a1 - a3;
        const cd jd13(d13.imag(), -d13.real());  // -i * d13
        out[k] = s02 + s13;
        out[m + k] = d02 + jd13;
        out[2 * m + k] = s02 - s13;
        out[3 * m + k] = d02 - jd13;
      }
    } else {
      if (static_cast<int>(tmp.size()) < 2 * r) tmp.resize(2 * r);
      cd* t = tmp.data();
      cd* o = t + r;
      const int rstep = n / r;
      for (int k = 0; k < m; ++k) {
        for (int q = 0; q < r; ++q) t[q] = out[q * m + k] * tw[static_cast<long>(q) * k * step % n];
        for (int p = 0; p < r; ++p) {
          cd s = 0;
          for (int q = 0; q < r; ++q) s += t[q] * tw[static_cast<long>(q * p % r) * rstep];
          o[p] = s;
        }
        for (int p = 0; p < r; ++p) out[p * m + k] = o[p];
      }
    }
  }

  void forward(const cd* in, cd* out, std::vector<cd>& tmp) const { rec(in, 1, out, n, 0, tmp); }
};

struct Scratch {
  std::vector<cd> a, b, t;
  std::vector<double> x, y;
};
Scratch& scratch() {
  thread_local Scratch s;
  return s;
}

// ------------------------------------------------------------- real kernels
// DST-I of x[0..n-1] (logical x_1..x_{N-1}, N = n+1): S_k = sum x_j sin(pi j k / N).
struct DST1 {
  int n, N;
  bool even;
  CFFT fft;
  std::vector<double> s;     // sin(pi j / N)
  std::vector<cd> unpack;    // exp(-2 pi i k / N), k < N/2
  explicit DST1(int len) : n(len), N(len + 1), even((len + 1) % 2 == 0), fft(even ? (len + 1) / 2 : 2 * (len + 1)) {
    s.resize(N);
    for (int j = 0; j < N; ++j) s[j] = static_cast<double>(sinl(3.14159265358979323846264338327950288L * j / N));
    if (even) {
      unpack.resize(N / 2 + 1);
      for (int k = 0; k <= N / 2; ++k) {
        const long double a = -2.0L * 3.14159265358979323846264338327950288L * k / N;
        unpack[k] = cd(static_cast<double>(cosl(a)), static_cast<double>(sinl(a)));
      }
    }
  }
  // S[k-1] for k = 1..n
  void run(const double* x, double* S) const {
    Scratch& sc = scratch();
    if (!even) {
      const int L = 2 * N;
      sc.a.assign(L, cd(0));
      sc.b.resize(L);
      for (int j = 1; j < N; ++j) {
        sc.a[j] = x[j - 1];
        sc.a[L - j] = -x[j - 1];
      }
      fft.forward(sc.a.data(), sc.b.data(), sc.t);
      for (int k = 1; k < N; ++k) S[k - 1] = -0.5 * sc.b[k].imag();
      return;
    }
    // w_j = sin(pi j/N)(x_j + x_{N-j}) + (x_j - x_{N-j})/2, w_0 = 0; real DFT.
    const int h = N / 2;
    sc.x.resize(N);
    sc.x[0] = 0.0;
    for (int j = 1; j < N; ++j) {
      const double xj = x[j - 1], xr = x[N - j - 1];
      sc.x[j] = s[j] * (xj + xr) + 0.5 * (xj - xr);
    }
    sc.a.resize(h);
    sc.b.resize(h);
    for (int t = 0; t < h; ++t) sc.a[t] = cd(sc.x[2 * t], sc.x[2 * t + 1]);
    fft.forward(sc.a.data(), sc.b.data(), sc.t);
    // W_k for k = 0..h-1 (W real DFT of w)
    double odd = 0.0;
    for (int k = 0; k < h; ++k) {
      const cd zk = sc.b[k], zc = std::conj(sc.b[(h - k) % h]);
      const cd W = 0.5 * (zk + zc) + cd(0, -0.5) * unpack[k] * (zk - zc);
      if (k == 0) {
        odd = 0.5 * W.real();
      } else {
        S[2 * k - 1] = -W.imag();  // S_{2k}
        odd += W.real();
      }
      S[2 * k] = odd;  // S_{2k+1}
    }
  }
};

// DCT-III of a[0..n-1]: y_j = sum_k a_k cos(pi k (2j+1)/(2n)), via Makhoul.
struct DCT3 {
  int n;
  CFFT fft;
  std::vector<cd> tw;  // 0.5 * exp(+i pi k/(2n))
  explicit DCT3(int len) : n(len), fft(len) {
    tw.resize(n);
    for (int k = 0; k < n; ++k) {
      const long double a = 3.14159265358979323846264338327950288L * k / (2.0L * n);
      tw[k] = 0.5 * cd(static_cast<double>(cosl(a)), static_cast<double>(sinl(a)));
    }
  }
  void run(const double* a, double* y) const {
    Scratch& sc = scratch();
    sc.a.resize(n);
    sc.b.resize(n);
    // u_t = sum_k V_k e^{+2 pi i k t/n} = conj(FFT(conj V))_t
    sc.a[0] = cd(a[0], 0.0);
    for (int k = 1; k < n; ++k) sc.a[k] = std::conj(tw[k] * cd(a[k], -a[n - k]));
    fft.forward(sc.a.data(), sc.b.data(), sc.t);
    for (int t = 0; 2 * t < n; ++t) y[2 * t] = sc.b[t].real();
    for (int t = 0; 2 * t + 1 < n; ++t) y[2 * t + 1] = sc.b[n - 1 - t].real();
  }
};

}  // namespace

struct fftw_plan_s {
  int kind, n, howmany, istride, idist, ostride, odist;
  DST1* dst1 = nullptr;
  DCT3* dct3 = nullptr;
};

extern "C" {

fftw_plan fftw_plan_many_r2r(int rank, const int* n, int howmany, double*, const int* inembed,
                             int istride, int idist, double*, const int* onembed, int ostride,
                             int odist, const fftw_r2r_kind* kind, unsigned) {
  if (rank != 1 || n == nullptr || n[0] < 1 || howmany < 1 || inembed || onembed) return nullptr;
  const int k = kind[0];
  if (k != FFTW_RODFT00 && k != FFTW_RODFT01 && k != FFTW_REDFT01) return nullptr;
  auto* p = new fftw_plan_s{k, n[0], howmany, istride, idist, ostride, odist};
  if (k == FFTW_RODFT00)
    p->dst1 = new DST1(n[0]);
  else
    p->dct3 = new DCT3(n[0]);
  return p;
}

fftw_plan fftw_plan_r2r_1d(int n, double* in, double* out, fftw_r2r_kind kind, unsigned flags) {
  return fftw_plan_many_r2r(1, &n, 1, in, nullptr, 1, 1, out, nullptr, 1, 1, &kind, flags);
}

void fftw_execute_r2r(const fftw_plan p, double* in, double* out) {
  const int n = p->n;
  Scratch& sc = scratch();
  thread_local std::vector<double> xin, yout;
  xin.resize(n);
  yout.resize(n);
  for (int b = 0; b < p->howmany; ++b) {
    const double* src = in + static_cast<long>(b) * p->idist;
    double* dst = out + static_cast<long>(b) * p->odist;
    for (int j = 0; j < n; ++j) xin[j] = src[static_cast<long>(j) * p->istride];
    if (p->kind == FFTW_RODFT00) {
      p->dst1->run(xin.data(), yout.data());
      for (int j = 0; j < n; ++j) yout[j] *= 2.0;
    } else if (p->kind == FFTW_REDFT01) {
      // Y = 2 * DCT3(a) with a_0 = X_0 / 2.
      xin[0] *= 0.5;
      p->dct3->run(xin.data(), yout.data());
      for (int j = 0; j < n; ++j) yout[j] *= 2.0;
    } else {
      // RODFT01: Y = 2 * DST3(b), b_{j+1} = X_j, b_n = X_{n-1}/2;
      // DST3(b)_j = (-1)^(j-1) DCT3(bt)_j with bt_k = b_{n-k}.
      sc.y.resize(n);
      sc.y[0] = 0.5 * xin[n - 1];
      for (int k = 1; k < n; ++k) sc.y[k] = xin[n - 1 - k];
      p->dct3->run(sc.y.data(), yout.data());
      for (int j = 0; j < n; ++j) yout[j] *= (j % 2 == 0) ? 2.0 : -2.0;
    }
    for (int j = 0; j < n; ++j) dst[static_cast<long>(j) * p->ostride] = yout[j];
  }
}

void fftw_destroy_plan(fftw_plan p) {
  if (!p) return;
  delete p->dst1;
  delete p->dct3;
  delete p;
}

}  // extern "C"
