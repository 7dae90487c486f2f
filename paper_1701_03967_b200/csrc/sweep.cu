// Generic sweep kernels: the eigen-expansion of the 1D high-order FEM operator
// applied along one axis of a dof tensor, for any (n, K).
//
// One CTA owns a tile of B lines.  The tile is staged in shared memory in
// position-major layout T[pos][b]; the n length-(K-1) sine transforms of every
// line are recast as n/2 complex K-point FFTs:
//   * interior pair i (components i and m-1-i): DCT-II of h = r_i - r_{m-1-i}
//     and DST-II of g = r_i + r_{m-1-i} share one FFT (Makhoul reordering);
//     this equals the reference's fold + DST-I (eigenbasis.cpp:46-59, 87-100);
//   * the middle component (m odd) pairs with the same component of line b+B/2;
//   * the nodal DST-I (trig.cpp:71-79) of lines b and b+B/2 share two FFTs.
// The inverse runs the transposed pipeline: per-frequency mixes, then paired
// DCT-III transforms (DST-III by index reversal), as eigenbasis.cpp:144-225.
// FFTs are shared-memory Stockham passes over all jobs of the tile.
#include <cstdio>

#include "sweep.cuh"

namespace sfem_b200 {
namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// -i * a
__device__ __forceinline__ double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }

struct Geometry {
  int B, Bh, Bm, J;
  int n, m, half, ne, N, L;
};

__device__ __forceinline__ Geometry geometry(const DevTable& t, int B) {
  Geometry g;
  g.B = B;
  g.Bh = (B + 1) / 2;
  g.n = t.n;
  g.m = t.m;
  g.half = t.half;
  g.ne = t.ne;
  g.N = t.K;
  g.L = t.L;
  g.Bm = (t.m & 1) ? g.Bh : 0;
  g.J = B * t.half + g.Bm + 2 * g.Bh;
  return g;
}

// Makhoul reorder: FFT input slot t holds element 2t (first half) or 2N-1-2t.
__device__ __forceinline__ int makhoul_src(int t, int N) { return (2 * t < N) ? 2 * t : 2 * N - 1 - 2 * t; }

// Stockham autosort FFT (forward sign) over J interleaved jobs, X[t*J + job].
// Returns the buffer holding the result.
__device__ double2* fft_passes(double2* X, double2* Y, const DevTable& t, int J) {
  const int N = t.K;
  int Ns = 1;
  for (int p = 0; p < t.npass; ++p) {
    const int r = t.radix[p];
    const int Nr = N / r;
    const int tstep = N / (Ns * r);
    const int items = Nr * J;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int job = it % J;
      const int j = it / J;
      const int k = j % Ns;
      const int outb = (j / Ns) * Ns * r + k;
      if (r == 2) {
        double2 a0 = X[j * J + job];
        double2 a1 = cmul(X[(j + Nr) * J + job], t.tw[(k * tstep) % N]);
        Y[outb * J + job] = cadd(a0, a1);
        Y[(outb + Ns) * J + job] = csub(a0, a1);
      } else if (r == 4) {
        double2 a0 = X[j * J + job];
        double2 a1 = cmul(X[(j + Nr) * J + job], t.tw[(k * tstep) % N]);
        double2 a2 = cmul(X[(j + 2 * Nr) * J + job], t.tw[(2 * k * tstep) % N]);
        double2 a3 = cmul(X[(j + 3 * Nr) * J + job], t.tw[(3 * k * tstep) % N]);
        const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2), s13 = cadd(a1, a3), d13 = csub(a1, a3);
        const double2 jd = cmul_mi(d13);
        Y[outb * J + job] = cadd(s02, s13);
        Y[(outb + Ns) * J + job] = cadd(d02, jd);
        Y[(outb + 2 * Ns) * J + job] = csub(s02, s13);
        Y[(outb + 3 * Ns) * J + job] = csub(d02, jd);
      } else {
        // generic radix: each output gathers all r twiddled inputs
        const int rstep = N / r;
        for (int pp = 0; pp < r; ++pp) {
          double2 s = make_double2(0.0, 0.0);
          for (int q = 0; q < r; ++q) {
            double2 a = X[(j + q * Nr) * J + job];
            const long long e1 = (static_cast<long long>(q) * k * tstep) % N;
            a = cmul(a, t.tw[e1]);
            s = cadd(s, cmul(a, t.tw[((q * pp) % r) * rstep]));
          }
          Y[(outb + pp * Ns) * J + job] = s;
        }
      }
    }
    __syncthreads();
    double2* tmp = X;
    X = Y;
    Y = tmp;
    Ns *= r;
  }
  return X;
}

// --------------------------------------------------------------- forward
__device__ void forward_fill(const Geometry& g, const DevTable& t, const double* T, double* C0, double2* W) {
  const int B = g.B, N = g.N, n = g.n, m = g.m, J = g.J;
  const int npair = B * g.half;
  for (int it = threadIdx.x; it < N * J; it += blockDim.x) {
    const int job = it % J;
    const int tt = it / J;
    double2 z;
    if (job < npair) {
      const int i = job / B, b = job % B;
      const int e = makhoul_src(tt, N);
      const double ri = T[(e * n + i) * B + b], rr = T[(e * n + m - 1 - i) * B + b];
      const double h = ri - rr;
      double gg = ri + rr;
      if (e & 1) gg = -gg;
      z = make_double2(h, gg);
    } else if (job < npair + g.Bm) {
      const int b = job - npair, b2 = b + g.Bh;
      const int e = makhoul_src(tt, N);
      double g1 = T[(e * n + g.half) * B + b];
      double g2 = b2 < B ? T[(e * n + g.half) * B + b2] : 0.0;
      if (e & 1) {
        g1 = -g1;
        g2 = -g2;
      }
      z = make_double2(g1, g2);
    } else {
      const int jb = job - npair - g.Bm;
      const int b = jb % g.Bh, which = jb / g.Bh, b2 = b + g.Bh;
      double x1 = 0.0, x2 = 0.0;
      if (tt > 0) {
        x1 = T[(tt * n - 1) * B + b];
        x2 = b2 < B ? T[(tt * n - 1) * B + b2] : 0.0;
      }
      z = make_double2(x1, x2);
      if (which) z = cmul(z, t.om[tt]);
    }
    W[tt * J + job] = z;
  }
  // zero-frequency centre (eigenbasis.cpp:31-40)
  for (int it = threadIdx.x; it < m * B; it += blockDim.x) {
    const int i = it / B, b = it % B;
    double s = 0.0;
    for (int e = 0; e < N; ++e) s += (e & 1) ? -T[(e * n + m - 1 - i) * B + b] : T[(e * n + i) * B + b];
    C0[i * B + b] = s;
  }
}

// FFT results -> per-(k, slot, line) real values S[((k-1) n + s) B + b].
__device__ void forward_post(const Geometry& g, const DevTable& t, const double2* R, double* S) {
  const int B = g.B, N = g.N, n = g.n, J = g.J;
  const int npair = B * g.half;
  for (int it = threadIdx.x; it < (N - 1) * J; it += blockDim.x) {
    const int job = it % J;
    const int k = 1 + it / J;
    if (job < npair + g.Bm) {
      const double2 zk = R[k * J + job], zc = R[(N - k) * J + job];
      // V1 = (Z_k + conj Z_{N-k})/2, V2 = (Z_k - conj Z_{N-k})/(2i)
      const double2 v1 = make_double2(0.5 * (zk.x + zc.x), 0.5 * (zk.y - zc.y));
      const double2 v2 = make_double2(0.5 * (zk.y + zc.y), -0.5 * (zk.x - zc.x));
      const double2 w = t.mk[k];
      const double r1 = w.x * v1.x - w.y * v1.y;  // DCT-II of the real part
      const double r2 = w.x * v2.x - w.y * v2.y;  // DCT-II of the imaginary part
      if (job < npair) {
        const int i = job / B, b = job % B;
        S[((k - 1) * n + 1 + g.ne + i) * B + b] = r1;       // H_k
        S[((N - k - 1) * n + 1 + i) * B + b] = r2;          // G_{N-k} = DCT2(g~)_k
      } else {
        const int b = job - npair, b2 = b + g.Bh;
        S[((N - k - 1) * n + 1 + g.half) * B + b] = r1;
        if (b2 < B) S[((N - k - 1) * n + 1 + g.half) * B + b2] = r2;
      }
    } else {
      const int jb = job - npair - g.Bm;
      const int b = jb % g.Bh, which = jb / g.Bh, b2 = b + g.Bh;
      if ((k & 1) != which) continue;  // A-job gives even k, B-job odd k
      double2 d;
      if (!which) {
        const int kp = k / 2;
        d = csub(R[(N - kp) * J + job], R[kp * J + job]);
      } else {
        const int kp = (k - 1) / 2;
        d = csub(R[(N - 1 - kp) * J + job], R[kp * J + job]);
      }
      // X = d / (2i)
      S[((k - 1) * n + 0) * B + b] = 0.5 * d.y;
      if (b2 < B) S[((k - 1) * n + 0) * B + b2] = -0.5 * d.x;
    }
  }
}

// --------------------------------------------------------------- inverse
__device__ void inverse_fill(const Geometry& g, const DevTable& t, const double* S, double2* W) {
  const int B = g.B, N = g.N, n = g.n, J = g.J;
  const int npair = B * g.half;
  for (int it = threadIdx.x; it < N * J; it += blockDim.x) {
    const int job = it % J;
    const int tt = it / J;
    double2 z = make_double2(0.0, 0.0);
    if (job < npair + g.Bm) {
      if (tt > 0) {
        const double2 w = t.mkh[tt];
        double ax, ar, bx, br;  // V1 = w (ax - i ar), V2 = w (bx - i br)
        if (job < npair) {
          const int i = job / B, b = job % B;
          ax = S[((tt - 1) * n + 1 + g.ne + i) * B + b];
          ar = S[((N - tt - 1) * n + 1 + g.ne + i) * B + b];
          bx = S[((N - tt - 1) * n + 1 + i) * B + b];   // b~_t = b_{N-t}
          br = S[((tt - 1) * n + 1 + i) * B + b];       // b~_{N-t} = b_t
        } else {
          const int b = job - npair, b2 = b + g.Bh;
          ax = S[((N - tt - 1) * n + 1 + g.half) * B + b];
          ar = S[((tt - 1) * n + 1 + g.half) * B + b];
          bx = b2 < B ? S[((N - tt - 1) * n + 1 + g.half) * B + b2] : 0.0;
          br = b2 < B ? S[((tt - 1) * n + 1 + g.half) * B + b2] : 0.0;
        }
        const double2 v1 = cmul(w, make_double2(ax, -ar));
        const double2 v2 = cmul(w, make_double2(bx, -br));
        // conj(V1 + i V2): the inverse DFT runs as a forward FFT of the conjugate
        z = make_double2(v1.x - v2.y, -(v1.y + v2.x));
      }
    } else {
      const int jb = job - npair - g.Bm;
      const int b = jb % g.Bh, which = jb / g.Bh, b2 = b + g.Bh;
      if (tt > 0) {
        z = make_double2(S[((tt - 1) * n) * B + b], b2 < B ? S[((tt - 1) * n) * B + b2] : 0.0);
        if (which) z = cmul(z, t.om[tt]);
      }
    }
    W[tt * J + job] = z;
  }
}

__device__ void inverse_post(const Geometry& g, const double2* R, const double* C0, double* T) {
  const int B = g.B, N = g.N, n = g.n, m = g.m, J = g.J;
  const int npair = B * g.half;
  for (int it = threadIdx.x; it < N * J; it += blockDim.x) {
    const int job = it % J;
    const int tt = it / J;
    if (job < npair + g.Bm) {
      const double2 u = R[tt * J + job];  // conj taken below
      const double ure = u.x, uim = -u.y;
      const int e = makhoul_src(tt, N);
      const bool odd = e & 1;
      if (job < npair) {
        const int i = job / B, b = job % B;
        const double o = ure;
        const double ev = odd ? -uim : uim;
        const double ci = odd ? -C0[(m - 1 - i) * B + b] : C0[i * B + b];
        const double cr = odd ? -C0[i * B + b] : C0[(m - 1 - i) * B + b];
        T[(e * n + i) * B + b] = ci + ev + o;
        T[(e * n + m - 1 - i) * B + b] = cr + ev - o;
      } else {
        const int b = job - npair, b2 = b + g.Bh;
        const int hc = g.half;
        const double c1 = odd ? -C0[hc * B + b] : C0[hc * B + b];
        T[(e * n + hc) * B + b] = c1 + (odd ? -ure : ure);
        if (b2 < B) {
          const double c2 = odd ? -C0[hc * B + b2] : C0[hc * B + b2];
          T[(e * n + hc) * B + b2] = c2 + (odd ? -uim : uim);
        }
      }
    } else {
      const int jb = job - npair - g.Bm;
      const int b = jb % g.Bh, which = jb / g.Bh, b2 = b + g.Bh;
      const int j = tt;  // nodal index handled by this item
      if (j < 1 || j > N - 1 || (j & 1) != which) continue;
      double2 d;
      if (!which) {
        const int kp = j / 2;
        d = csub(R[(N - kp) * J + job], R[kp * J + job]);
      } else {
        const int kp = (j - 1) / 2;
        d = csub(R[(N - 1 - kp) * J + job], R[kp * J + job]);
      }
      T[(j * n - 1) * B + b] = 0.5 * d.y;
      if (b2 < B) T[(j * n - 1) * B + b2] = -0.5 * d.x;
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) sweep_kernel(DevTable t, LineSet ls, int analysis, SymbolInfo sym, int B,
                                                    double* gwork) {
  extern __shared__ double smem[];
  const Geometry g = geometry(t, B);
  const int L = g.L, N = g.N, n = g.n, m = g.m;
  double* T = smem;
  double* C0 = T + static_cast<size_t>(L) * B;
  double* base = C0 + static_cast<size_t>(m) * B;  // B doubles: symbol base per line
  long long* off = reinterpret_cast<long long*>(base + B);
  const size_t head = static_cast<size_t>(L) * B + static_cast<size_t>(m) * B + 2 * static_cast<size_t>(B);
  // FFT work buffers: shared memory, or (long lines) a per-CTA slice of a
  // global scratch array that stays L2-resident
  double2* W0 = gwork ? reinterpret_cast<double2*>(gwork + static_cast<size_t>(blockIdx.x) * 4 * g.J * N)
                      : reinterpret_cast<double2*>(smem + head + (head & 1));
  double2* W1 = W0 + static_cast<size_t>(g.J) * N;

  const long long l0 = static_cast<long long>(blockIdx.x) * B;
  const int Bv = static_cast<int>(min(static_cast<long long>(B), ls.nlines - l0));

  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const long long l = l0 + b;
    const long long r = l / ls.ninner;
    off[b] = (r / ls.n1) * ls.os2 + (r % ls.n1) * ls.os1 + (l % ls.ninner) * ls.is;
    if (MODE == kForwardDivideInverse) {
      double s = sym.shift;
      long long rem = l;
      double terms[kMaxDim];
      for (int i = sym.nlead - 1; i >= 0; --i) {
        const long long a = rem % sym.lead_ext[i];
        rem /= sym.lead_ext[i];
        terms[i] = (l < ls.nlines) ? sym.lead_f[i] * sym.lead_eig[i][a] : 0.0;
      }
      for (int i = 0; i < sym.nlead; ++i) s += terms[i];
      base[b] = s;
    }
  }
  __syncthreads();

  // load tile
  const long long ps = ls.ps;
  for (int it = threadIdx.x; it < L * B; it += blockDim.x) {
    int b, pos;
    if (ls.contiguous) {
      b = it / L;
      pos = it % L;
    } else {
      pos = it / B;
      b = it % B;
    }
    T[pos * B + b] = (b < Bv) ? ls.src[off[b] + pos * ps] : 0.0;
  }
  __syncthreads();

  if (MODE != kInverse) {
    forward_fill(g, t, T, C0, W0);
    __syncthreads();
    double2* R = fft_passes(W0, W1, t, g.J);
    double* S = reinterpret_cast<double*>(R == W0 ? W1 : W0);
    forward_post(g, t, R, S);
    __syncthreads();
    const double* mix = analysis == kDirect ? t.mix_fwd_d : t.mix_fwd_w;
    const double* e0 = analysis == kDirect ? t.e0_fwd_d : t.e0_fwd_w;
    for (int it = threadIdx.x; it < (N - 1) * B; it += blockDim.x) {
      const int k = 1 + it / B, b = it % B;
      const double* M = mix + static_cast<size_t>(k - 1) * n * n;
      const double* v = S + static_cast<size_t>((k - 1) * n) * B + b;
      for (int l = 0; l < n; ++l) {
        double c = 0.0;
        for (int s = 0; s < n; ++s) c += M[l * n + s] * v[s * B];
        const int pos = m + (k - 1) * n + l;
        if (MODE == kForwardDivideInverse) c /= (base[b] + sym.f_last * t.eig[pos]);
        T[pos * B + b] = c;
      }
    }
    for (int it = threadIdx.x; it < m * B; it += blockDim.x) {
      const int l = it / B, b = it % B;
      double c = 0.0;
      for (int i = 0; i < m; ++i) c += C0[i * B + b] * e0[i * m + l];
      if (MODE == kForwardDivideInverse) c /= (base[b] + sym.f_last * t.eig[l]);
      T[l * B + b] = c;
    }
    __syncthreads();
  }

  if (MODE != kForward) {
    double* S = reinterpret_cast<double*>(W1);
    for (int it = threadIdx.x; it < (N - 1) * B; it += blockDim.x) {
      const int k = 1 + it / B, b = it % B;
      const double* M = t.mix_inv + static_cast<size_t>(k - 1) * n * n;
      double c[16];
      for (int l = 0; l < n; ++l) c[l] = T[(m + (k - 1) * n + l) * B + b];
      for (int s = 0; s < n; ++s) {
        double u = 0.0;
        for (int l = 0; l < n; ++l) u += M[s * n + l] * c[l];
        S[((k - 1) * n + s) * B + b] = u;
      }
    }
    for (int it = threadIdx.x; it < m * B; it += blockDim.x) {
      const int i = it / B, b = it % B;
      double c = 0.0;
      for (int l = 0; l < m; ++l) c += t.e0_inv[i * m + l] * T[l * B + b];
      C0[i * B + b] = c;
    }
    __syncthreads();
    inverse_fill(g, t, S, W0);
    __syncthreads();
    double2* R = fft_passes(W0, W1, t, g.J);
    inverse_post(g, R, C0, T);
    __syncthreads();
  }

  for (int it = threadIdx.x; it < L * B; it += blockDim.x) {
    int b, pos;
    if (ls.contiguous) {
      b = it / L;
      pos = it % L;
    } else {
      pos = it / B;
      b = it % B;
    }
    if (b < Bv) ls.dst[off[b] + pos * ps] = T[pos * B + b];
  }
}

}  // namespace

size_t sweep_work_doubles(const DevTable& t, int B) {
  const int Bh = (B + 1) / 2;
  const int J = B * t.half + ((t.m & 1) ? Bh : 0) + 2 * Bh;
  return 4 * static_cast<size_t>(J) * t.K;
}

size_t sweep_smem_bytes(const DevTable& t, int B, bool global_work) {
  size_t doubles = static_cast<size_t>(t.L) * B + static_cast<size_t>(t.m) * B + 2 * static_cast<size_t>(B);
  doubles += (doubles & 1);
  if (!global_work) doubles += sweep_work_doubles(t, B);
  return doubles * sizeof(double);
}

cudaError_t launch_sweep(const DevTable& t, const LineSet& lines, int mode, int analysis,
                         const SymbolInfo* sym, int B, cudaStream_t stream, double* gwork) {
  if (lines.nlines <= 0) return cudaSuccess;
  const size_t smem = sweep_smem_bytes(t, B, gwork != nullptr);
  const long long tiles = (lines.nlines + B - 1) / B;
  SymbolInfo s{};
  if (sym) s = *sym;
  const dim3 grid(static_cast<unsigned>(tiles));
  cudaError_t err = cudaSuccess;
  switch (mode) {
    case kForward:
      err = cudaFuncSetAttribute(sweep_kernel<kForward>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (err == cudaSuccess) sweep_kernel<kForward><<<grid, 256, smem, stream>>>(t, lines, analysis, s, B, gwork);
      break;
    case kInverse:
      err = cudaFuncSetAttribute(sweep_kernel<kInverse>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (err == cudaSuccess) sweep_kernel<kInverse><<<grid, 256, smem, stream>>>(t, lines, analysis, s, B, gwork);
      break;
    default:
      err = cudaFuncSetAttribute(sweep_kernel<kForwardDivideInverse>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
      if (err == cudaSuccess)
        sweep_kernel<kForwardDivideInverse><<<grid, 256, smem, stream>>>(t, lines, analysis, s, B, gwork);
      break;
  }
  if (err != cudaSuccess) return err;
  return cudaGetLastError();
}

}  // namespace sfem_b200
