// The steps either side of the solve, on the device (SURVEY.md 8(f) ranks 1
// and 3):
//
//   * FEM load averaging (reference fem_load_average, poisson.cpp:471-569):
//     per element, f on the tensor Gauss grid (n_i + 1 points per axis), one
//     contraction per axis with w_g * phi_loc(xi_g) (axis_quad,
//     poisson.cpp:481-495), then the local load is added into the dof tensor
//     with the boundary contributions dropped.  One warp per element; the
//     elements are swept in 2^N parity colours (elements of one colour share
//     no dof), so the adds need no atomics and every dof sums its element
//     contributions in a fixed order: deterministic run to run.
//   * Operator application A v (apply_operator, poisson.cpp:749-769) with
//     A = sum_i f_i (x)_{j != i} M_j (x) S_i + shift (x)_j M_j, as one sweep
//     per axis carrying two tensors:  P <- M P,  Q <- M Q + f S P  (Q starts
//     as shift * v), so N sweeps instead of the reference's (N + 1) N stencil
//     passes.  Each sweep walks the elements of a line once (the 1-D operator
//     is element-local, apply_element_stencil grid1d.cpp:7-29), in place.
//     Strided axes: one thread per line (lanes over the contiguous index:
//     coalesced).  Last axis: one warp per row, lanes over elements, node
//     sums through a shuffle.
//   * The residual check of solve_with_load (poisson.cpp:785-789,
//     max|A u - f| / max|f|) fused into the last operator sweep, and the
//     uniform error against a manufactured solution (max_error_vs,
//     ndgrid.cpp:80-101, at the dof coordinates of axis_coordinate,
//     ndgrid.cpp:71-78), both as deterministic max-reductions.
#include <cuda_runtime.h>

#include <algorithm>

#include "fem_ops.cuh"

namespace sfem_b200 {
namespace femops {

constexpr double kPi = 3.14159265358979323846;

// ---------------------------------------------------------------------------
// Right-hand sides / exact solutions (reference cases.cpp:11-55 and the
// product-of-sines load of BASELINE config 3).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double field_value(const FieldArgs& fa, const double* x, bool exact) {
  switch (fa.kind) {
    case kFieldConstant:
      return exact ? 0.0 : fa.p[0];
    case kFieldSines: {  // amp * prod sin(k_i pi x_i); exact: / (sum a_i (k_i pi)^2 + shift)
      double v = exact ? fa.p[1 + kMaxDim] : fa.p[0];
      for (int i = 0; i < fa.dim; ++i) v *= sin(fa.p[1 + i] * kPi * x[i]);
      return v;
    }
    case kFieldSin1d: {  // u = sin(pi x) e^x
      const double s = sin(kPi * x[0]), c = cos(kPi * x[0]), ex = exp(x[0]);
      const double u = s * ex;
      if (exact) return u;
      const double lap = ((1.0 - kPi * kPi) * s + 2.0 * kPi * c) * ex;
      return -lap + fa.shift * u;
    }
    case kFieldPoisson2d: {  // u = sin(2 pi x1) sin(3 pi x2) cosh(sqrt2 x1 - x2)
      const double s1 = sin(2 * kPi * x[0]), c1 = cos(2 * kPi * x[0]);
      const double s2 = sin(3 * kPi * x[1]), c2 = cos(3 * kPi * x[1]);
      const double w = sqrt(2.0) * x[0] - x[1];
      const double ch = cosh(w), sh = sinh(w);
      const double u = s1 * s2 * ch;
      if (exact) return u;
      const double lap = (-13.0 * kPi * kPi + 3.0) * s1 * s2 * ch +
                         2.0 * sh * (2.0 * sqrt(2.0) * kPi * c1 * s2 - 3.0 * kPi * s1 * c2);
      return -lap + fa.shift * u;
    }
    case kFieldPoisson3d: {  // u = s1 s2 s3 cosh(sqrt2 x1 - x2 + x3/sqrt3)
      const double s1 = sin(2 * kPi * x[0]), c1 = cos(2 * kPi * x[0]);
      const double s2 = sin(3 * kPi * x[1]), c2 = cos(3 * kPi * x[1]);
      const double s3 = sin(4 * kPi * x[2]), c3 = cos(4 * kPi * x[2]);
      const double w = sqrt(2.0) * x[0] - x[1] + x[2] / sqrt(3.0);
      const double ch = cosh(w), sh = sinh(w);
      const double u = s1 * s2 * s3 * ch;
      if (exact) return u;
      const double lap = (-29.0 * kPi * kPi + 10.0 / 3.0) * s1 * s2 * s3 * ch +
                         2.0 * sh *
                             (2.0 * sqrt(2.0) * kPi * c1 * s2 * s3 - 3.0 * kPi * s1 * c2 * s3 +
                              4.0 * kPi / sqrt(3.0) * s1 * s2 * c3);
      return -lap + fa.shift * u;
    }
  }
  return 0.0;
}

// ---------------------------------------------------------------------------
// FEM load: one warp per element of parity colour `color`.
// ---------------------------------------------------------------------------
__global__ void fem_load_color(double* __restrict__ out, const __grid_constant__ LoadArgs a, FieldArgs fa,
                               unsigned color) {
  extern __shared__ double lsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  int tens = 1;
  for (int i = 0; i < a.dim; ++i) tens *= a.np[i];
  double* vals = lsm + static_cast<size_t>(warp) * 2 * tens;
  double* scr = vals + tens;
  // elements of this colour: e_i = 2 c_i + bit_i(color), c_i < cnt_i
  long long cnt[kMaxDim];
  long long total = 1;
  for (int i = 0; i < a.dim; ++i) {
    const int par = (color >> i) & 1u;
    cnt[i] = (a.K[i] - par + 1) / 2;
    total *= cnt[i];
  }
  for (long long w = static_cast<long long>(blockIdx.x) * nwarps + warp; w < total;
       w += static_cast<long long>(gridDim.x) * nwarps) {
    int e[kMaxDim];
    long long r = w;
    for (int i = a.dim - 1; i >= 0; --i) {
      e[i] = static_cast<int>(2 * (r % cnt[i]) + ((color >> i) & 1u));
      r /= cnt[i];
    }
    // f on the tensor Gauss grid (g flat, last axis fastest)
    for (int g = lane; g < tens; g += 32) {
      double x[kMaxDim];
      int rem = g;
      for (int i = a.dim - 1; i >= 0; --i) {
        const int gi = rem % a.np[i];
        rem /= a.np[i];
        x[i] = (e[i] + 0.5 * (a.gnode[i][gi] + 1.0)) * a.h[i];
      }
      vals[g] = field_value(fa, x, false);
    }
    __syncwarp();
    // contract axes N-1 .. 0 (poisson.cpp:527-540 order)
    for (int ax = a.dim - 1; ax >= 0; --ax) {
      int inner = 1;
      for (int i = ax + 1; i < a.dim; ++i) inner *= a.np[i];
      const int s = a.np[ax];
      for (int idx = lane; idx < tens; idx += 32) {
        const int in = idx % inner, os = idx / inner, loc = os % s, o = os / s;
        const double* wv = a.wq[ax] + loc * s;
        const double* src = vals + static_cast<size_t>(o) * s * inner + in;
        double acc = 0.0;
        for (int g = 0; g < s; ++g) acc = fma(wv[g], src[g * inner], acc);
        scr[idx] = acc;
      }
      __syncwarp();
      double* t = vals;
      vals = scr;
      scr = t;
    }
    // add into the dof tensor; boundary contributions dropped
    for (int l = lane; l < tens; l += 32) {
      int rem = l;
      long long off = 0;
      bool keep = true;
      for (int i = a.dim - 1; i >= 0; --i) {
        const int loc = rem % a.np[i];
        rem /= a.np[i];
        const long long t = static_cast<long long>(e[i]) * a.n[i] - 1 + loc;  // dof coordinate
        if (t < 0 || t >= a.ext[i]) keep = false;
        off += t * a.st[i];
      }
      if (keep) out[off] += vals[l];
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Separable fields (constant, product of sines): the element loads are rank
// one, so the assembled load is amp * outer product of the assembled 1-D
// loads B_i (sum over the elements containing dof t_i of b_i[e][loc]); one
// write per dof.  B = concatenated per-axis vectors, boff[i] their offsets.
// ---------------------------------------------------------------------------
__global__ void fem_load_separable(double* __restrict__ out, const double* __restrict__ Bv, SepArgs a) {
  for (long long l = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; l < a.total;
       l += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long rem = l, off = 0;
    double v = a.amp;
    bool pad = false;
    for (int i = a.dim - 1; i >= 0; --i) {
      const long long ext = i == a.dim - 1 ? a.pitch : a.ext[i];
      const long long t = rem % ext;
      rem /= ext;
      off += t * a.st[i];
      if (t >= a.ext[i]) pad = true;
      else v *= __ldg(Bv + a.boff[i] + t);
    }
    out[off] = pad ? 0.0 : v;
  }
}

// ---------------------------------------------------------------------------
// Operator sweeps.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void atomic_max_pos(unsigned long long* p, double v) {
  atomicMax(p, static_cast<unsigned long long>(__double_as_longlong(v)));  // v >= 0: bit order = value order
}

// block max of (a, b) into red[0], red[1]
__device__ __forceinline__ void block_max2(double a, double b, unsigned long long* red) {
  __shared__ double sa[32], sb[32];
  for (int o = 16; o > 0; o >>= 1) {
    a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) {
    sa[warp] = a;
    sb[warp] = b;
  }
  __syncthreads();
  if (warp == 0) {
    a = lane < nw ? sa[lane] : 0.0;
    b = lane < nw ? sb[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0) {
      atomic_max_pos(&red[0], a);
      atomic_max_pos(&red[1], b);
    }
  }
}

// Element contributions of one element: zm = M x_P, zs = S x_P, zq = M x_Q.
template <int NP, bool FIRST>
__device__ __forceinline__ void element_apply(const OpAxisArgs& a, const double (&xp)[NP], const double (&xq)[NP],
                                              double (&zp)[NP], double (&zq)[NP]) {
#pragma unroll
  for (int r = 0; r < NP; ++r) {
    double m = 0.0, s = 0.0, q = 0.0;
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      m = fma(a.M[r][c], xp[c], m);
      s = fma(a.S[r][c], xp[c], s);
      if (!FIRST) q = fma(a.M[r][c], xq[c], q);
    }
    zp[r] = m;
    zq[r] = fma(a.fac, s, FIRST ? a.shift * m : q);
  }
}

// Strided axis: thread per line.  FIRST: P_in = v (read only), Q_in = shift*v.
// LAST: no P output; Q to qout, or (RESID) max|Q - f| and max|f| into red.
template <int NP, bool FIRST, bool LAST, bool RESID>
__global__ void __launch_bounds__(256) op_strided(const double* pin, double* pout, double* qio, const double* f,
                                                  OpAxisArgs a, unsigned long long* red) {
  constexpr int n = NP - 1;
  const long long nl = a.outer * a.inner;
  long long l = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  double rmax = 0.0, fmaxv = 0.0;
  if (l < nl && (l % a.inner) % a.pitch < a.last) {
    const long long o = l / a.inner, i = l - o * a.inner;
    const long long base = o * a.L * a.inner + i;
    const long long st = a.inner;
    double xp[NP], xq[NP], zp[NP], zq[NP];
    double lp = 0.0, lq = 0.0, cp = 0.0, cq = 0.0;  // raw left node, carried right-node sums
    for (int e = 0; e < a.K; ++e) {
      const long long t0 = static_cast<long long>(e) * n - 1;  // left node position
      xp[0] = lp;
      xq[0] = lq;
#pragma unroll
      for (int c = 1; c < NP; ++c) {
        const long long t = t0 + c;
        const bool in = t < a.L;
        xp[c] = in ? pin[base + t * st] : 0.0;
        if (!FIRST) xq[c] = in ? qio[base + t * st] : 0.0;
      }
      element_apply<NP, FIRST>(a, xp, xq, zp, zq);
#pragma unroll
      for (int c = 0; c < n; ++c) {
        const long long t = t0 + c;
        if (t < 0) continue;
        const double vp = c == 0 ? cp + zp[0] : zp[c];
        const double vq = c == 0 ? cq + zq[0] : zq[c];
        if (!LAST) pout[base + t * st] = vp;
        if (RESID) {
          const double fv = f[base + t * st];
          rmax = fmax(rmax, fabs(vq - fv));
          fmaxv = fmax(fmaxv, fabs(fv));
        } else {
          qio[base + t * st] = vq;
        }
      }
      cp = zp[n];
      cq = zq[n];
      lp = xp[n];
      lq = FIRST ? 0.0 : xq[n];
    }
  }
  if (RESID) block_max2(rmax, fmaxv, red);
}

// Last axis: one warp per row, lanes over elements (chunks of 32).
template <int NP, bool FIRST, bool LAST, bool RESID>
__global__ void __launch_bounds__(256) op_rows(const double* pin, double* pout, double* qio, const double* f,
                                               OpAxisArgs a, unsigned long long* red) {
  constexpr int n = NP - 1;
  const int lane = threadIdx.x & 31;
  const long long row = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  double rmax = 0.0, fmaxv = 0.0;
  if (row < a.outer) {
    const long long base = row * a.pitch;
    double cp = 0.0, cq = 0.0;  // right-node sums of the previous chunk's last element
    for (int e0 = 0; e0 < a.K; e0 += 32) {
      const int e = e0 + lane;
      const bool ok = e < a.K;
      const long long t0 = static_cast<long long>(e) * n - 1;
      double xp[NP], xq[NP], zp[NP], zq[NP];
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const long long t = t0 + c;
        const bool in = ok && t >= 0 && t < a.L;
        xp[c] = in ? pin[base + t] : 0.0;
        if (!FIRST) xq[c] = in ? qio[base + t] : 0.0;
      }
      element_apply<NP, FIRST>(a, xp, xq, zp, zq);
      // right-node sums of the left neighbour (all loads of the chunk are done
      // once the shuffle returns: in-place stores below are safe)
      double np_ = __shfl_up_sync(0xffffffffu, zp[n], 1);
      double nq_ = __shfl_up_sync(0xffffffffu, zq[n], 1);
      if (lane == 0) {
        np_ = cp;
        nq_ = cq;
      }
      cp = __shfl_sync(0xffffffffu, zp[n], 31);
      cq = __shfl_sync(0xffffffffu, zq[n], 31);
      if (ok) {
#pragma unroll
        for (int c = 0; c < n; ++c) {
          const long long t = t0 + c;
          if (t < 0) continue;
          const double vp = c == 0 ? np_ + zp[0] : zp[c];
          const double vq = c == 0 ? nq_ + zq[0] : zq[c];
          if (!LAST) pout[base + t] = vp;
          if (RESID) {
            const double fv = f[base + t];
            rmax = fmax(rmax, fabs(vq - fv));
            fmaxv = fmax(fmaxv, fabs(fv));
          } else {
            qio[base + t] = vq;
          }
        }
      }
    }
  }
  if (RESID) block_max2(rmax, fmaxv, red);
}

// max |u - exact(x)| over the dofs (and max |u| for scale).
__global__ void max_error_kernel(const double* __restrict__ u, ErrArgs a, FieldArgs fa, unsigned long long* red) {
  const long long nl = a.total;
  double worst = 0.0, umax = 0.0;
  for (long long l = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; l < nl;
       l += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long rem = l, off = 0;
    double x[kMaxDim];
    for (int i = a.dim - 1; i >= 0; --i) {
      const long long t = rem % a.ext[i];
      rem /= a.ext[i];
      off += t * a.st[i];
      // dof t: node j = (t+1)/n when (t+1) % n == 0, else interior of element t/n
      const long long j1 = t + 1;
      const long long e = j1 / a.n[i], c = j1 % a.n[i];
      x[i] = c == 0 ? a.h[i] * static_cast<double>(e)
                    : a.h[i] * (static_cast<double>(t / a.n[i]) + static_cast<double>(t % a.n[i] + 1) / a.n[i]);
    }
    const double v = u[off];
    worst = fmax(worst, fabs(v - field_value(fa, x, true)));
    umax = fmax(umax, fabs(v));
  }
  block_max2(worst, umax, red);
}

template <int NP>
cudaError_t launch_op_np(const double* pin, double* pout, double* q, const double* f, const OpAxisArgs& a, bool rows,
                         bool first, bool last, bool resid, unsigned long long* red, cudaStream_t s) {
  const long long threads = rows ? a.outer * 32 : a.outer * a.inner;
  const unsigned grid = static_cast<unsigned>((threads + 255) / 256);
  if (grid == 0) return cudaSuccess;
#define SFEM_OP_GO(KERN, F, L, R) KERN<NP, F, L, R><<<grid, 256, 0, s>>>(pin, pout, q, f, a, red)
#define SFEM_OP_SEL(KERN)                        \
  if (first && last && resid)                    \
    SFEM_OP_GO(KERN, true, true, true);          \
  else if (first && last)                        \
    SFEM_OP_GO(KERN, true, true, false);         \
  else if (first)                                \
    SFEM_OP_GO(KERN, true, false, false);        \
  else if (last && resid)                        \
    SFEM_OP_GO(KERN, false, true, true);         \
  else if (last)                                 \
    SFEM_OP_GO(KERN, false, true, false);        \
  else                                           \
    SFEM_OP_GO(KERN, false, false, false);
  if (rows) {
    SFEM_OP_SEL(op_rows)
  } else {
    SFEM_OP_SEL(op_strided)
  }
#undef SFEM_OP_SEL
#undef SFEM_OP_GO
  return cudaGetLastError();
}

}  // namespace femops

cudaError_t launch_op_axis(const double* pin, double* pout, double* q, const double* f, const OpAxisArgs& a,
                           bool rows, bool first, bool last, bool resid, unsigned long long* red, cudaStream_t s) {
  using namespace femops;
  switch (a.n + 1) {
    case 2: return launch_op_np<2>(pin, pout, q, f, a, rows, first, last, resid, red, s);
    case 3: return launch_op_np<3>(pin, pout, q, f, a, rows, first, last, resid, red, s);
    case 4: return launch_op_np<4>(pin, pout, q, f, a, rows, first, last, resid, red, s);
    case 5: return launch_op_np<5>(pin, pout, q, f, a, rows, first, last, resid, red, s);
    case 6: return launch_op_np<6>(pin, pout, q, f, a, rows, first, last, resid, red, s);
    case 7: return launch_op_np<7>(pin, pout, q, f, a, rows, first, last, resid, red, s);
    case 8: return launch_op_np<8>(pin, pout, q, f, a, rows, first, last, resid, red, s);
    case 9: return launch_op_np<9>(pin, pout, q, f, a, rows, first, last, resid, red, s);
    case 10: return launch_op_np<10>(pin, pout, q, f, a, rows, first, last, resid, red, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_fem_load(double* out, const LoadArgs& a, const FieldArgs& fa, int num_sms, cudaStream_t s) {
  int tens = 1;
  for (int i = 0; i < a.dim; ++i) tens *= a.np[i];
  const size_t per_warp = 2 * static_cast<size_t>(tens) * sizeof(double);
  int warps = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, (48 * 1024) / per_warp)));
  const size_t smem = per_warp * warps;
  if (smem > 48 * 1024) {
    const cudaError_t e =
        cudaFuncSetAttribute(femops::fem_load_color, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  long long elems = 1;
  for (int i = 0; i < a.dim; ++i) elems *= a.K[i];
  const long long per_color = (elems >> a.dim) + 1;
  const long long want = (per_color + warps - 1) / warps;
  const unsigned grid = static_cast<unsigned>(std::max<long long>(1, std::min<long long>(want, 64LL * num_sms)));
  for (unsigned color = 0; color < (1u << a.dim); ++color) {
    femops::fem_load_color<<<grid, 32 * warps, smem, s>>>(out, a, fa, color);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_fem_load_separable(double* out, const double* Bv, const SepArgs& a, int num_sms, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(
      std::max<long long>(1, std::min<long long>((a.total + 255) / 256, 32LL * num_sms)));
  femops::fem_load_separable<<<grid, 256, 0, s>>>(out, Bv, a);
  return cudaGetLastError();
}

cudaError_t launch_max_error(const double* u, const ErrArgs& a, const FieldArgs& fa, unsigned long long* red,
                             int num_sms, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(
      std::max<long long>(1, std::min<long long>((a.total + 255) / 256, 16LL * num_sms)));
  femops::max_error_kernel<<<grid, 256, 0, s>>>(u, a, fa, red);
  return cudaGetLastError();
}

}  // namespace sfem_b200
