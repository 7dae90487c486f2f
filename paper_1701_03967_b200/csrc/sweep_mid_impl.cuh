// Sweep kernels for mid-length lines (templates; instantiated by sweep_mid.cu
// for the tuned shapes and by sweep_mid_k*.cu for the general ones) (n*K ~ 1000-10000): C5's (n, K) in
// {(1,1024), (2,512), (4,256), (9,114)} and C3's (9,1024).
//
// Same mathematics as sweep.cu (reference eigenbasis.cpp:63-225),
// specialised at compile time on (n, K, lines per tile B, threads) and laid
// out for one large tile per CTA:
//   * one shared-memory region is reused in place for every stage: the tile
//     T[pos][b], the FFT buffer W[t][job] (complex) and the per-frequency slots
//     S, which are stored at the tile positions of the coefficients they
//     become (S row r <-> tile position m + r).  Stages that permute data move
//     it through registers ("bridges": every thread loads its items, barrier,
//     every thread stores);
//   * FFTs are in-place Stockham passes with compile-time radices (16/8/4/2
//     register butterflies, odd radices 3 and 19 as direct DFTs);
//   * the n x n mix of a frequency touches only that frequency's n slots of a
//     line, so it runs in place per (k, line) item; the last-axis kernel does
//     forward mix, symbol divide and inverse mix of an item in registers;
//   * the zero-frequency centre sums (eigenbasis.cpp:31-40) are chunked over
//     all threads and reduced in a fixed order (deterministic).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "fft_reg.cuh"
#include "sweep.cuh"

#ifndef SFEM_MID_R16
#define SFEM_MID_R16 1
#endif
// CTAs of at least this many threads hold one radix-16 item per thread, so
// they take the short radix plans regardless of the job count.
#ifndef SFEM_MID_FEW_TH
#define SFEM_MID_FEW_TH 512
#endif
#ifndef SFEM_MID_C2_TH
#define SFEM_MID_C2_TH 512
#endif
// C3 (n = 9, K = 1024, two lines: J = 10 jobs): 10 x 1024 / 16 = 640 radix-16 items
#ifndef SFEM_MID_C3_TH
#define SFEM_MID_C3_TH 640
#endif
#ifndef SFEM_MID_KMIX
#define SFEM_MID_KMIX 1
#endif
// Lines per (k >= 1) mix item, at most SFEM_MID_MIXG (1, 2 or 4; G lines need
// B % G == 0; 4 only in the fused kernel and for n <= 5, to stay in
// registers).  G lines per item divide the matrix loads per FMA by G.
// Measured (profiles/r1m_mid_mixg*): G = 2 vs 1: C3 -9 %, C5 -4.5..-8 %;
// G = 4 vs 2: fused C5 sweeps -1.4..-2.7 %, strided ones +1..+7 % (kept
// at 2 there).
#ifndef SFEM_MID_MIXG
#define SFEM_MID_MIXG 4
#endif
#ifndef SFEM_MID_ROWS_BULK
#define SFEM_MID_ROWS_BULK 1
#endif

namespace sfem_b200 {
namespace mid {

using namespace reg;

#include "phase_timing.cuh"

// ROWS: tile stored line-major T[b][pos] (line pitch LP, odd: conflict-free
// for lanes over lines), used when lines are rows of the tensor; otherwise
// position-major T[pos][b] (strided axes, lanes over the 8 adjacent lines).
//
// CM (strided TMA tiles of 8 lines, n a power of two): component-major tile
// T[s][e & 1][e >> 1][b] for position e * n + s.  In the dense T[pos][b]
// layout a tile row is 64 bytes, and both access families of the stages --
// a warp's items at consecutive frequencies / elements (rows n apart) and at
// consecutive Makhoul indices (elements 2 apart) -- keep to one half of the
// 128-byte bank line for even n (C5 n=4: 432M of 1,161M shared wavefronts
// excess, profiles/r4d_ncu_full_c5n4.json).  Here consecutive elements of one
// component alternate between two planes and consecutive even (odd) elements
// are adjacent 64-byte rows, so either family covers whole bank lines.  The
// TMA unit writes this layout itself (5-D boxes, sweep_mid_tma_cm).
template <int NN, int K, int BB, int TH, bool ROWS_, bool GW = false, bool CM_ = false>
struct Cfg {
  static constexpr int n = NN, m = NN - 1, half = m / 2, ne = NN / 2, N = K, L = NN * K - 1;
  static constexpr bool ROWS = ROWS_;
  static constexpr bool CM = CM_;
  static_assert(!CM_ || (!ROWS_ && !GW && BB == 8 && (NN & (NN - 1)) == 0 && NN >= 2 && K % 2 == 0),
                "component-major tiles: strided, 8 lines, n a power of two, even K");
  // PAD (one-line tiles): lanes run ALONG the line, at strides of n or 2n
  // doubles (fills, posts, mixes), i.e. onto 2-4 bank pairs; one pad double
  // per 16 positions spreads 16 consecutive elements / frequencies over all
  // 16 bank pairs (C2: shared wavefronts 52M -> ideal 8M in the forward fill).
  static constexpr bool PAD = BB == 1 && !GW;
  // Row tiles of B > 1 lines: rows move as one bulk copy each (cp.async.bulk,
  // 16-byte aligned, L rounded up to even doubles), so the row pitch is even:
  // 2 mod 16 doubles keeps the 8 lines of a tile on 8 different bank pairs.
  // (SFEM_MID_ROWS_BULK=0: odd pitch and 8-byte cp.async copies.)
  static constexpr bool BULK = SFEM_MID_ROWS_BULK && ROWS_ && BB > 1 && !GW;
  static constexpr int LB = (L + 1) & ~1;  // doubles per bulk row copy
  static constexpr int LP = PAD ? ((L + (L >> 4) + 1) | 1) : (BULK ? ((LB + 15) / 16 * 16 + 2) : (L | 1));
  static constexpr int PSTR = ROWS ? 1 : BB;  // position stride in the tile (not with PAD: use ix)
  __device__ __forceinline__ static constexpr int ix(int pos, int b) {
    if (CM) {
      const int e = pos / NN, s = pos - e * NN;
      return ((s * 2 + (e & 1)) * (K / 2) + (e >> 1)) * BB + b;
    }
    return PAD ? pos + (pos >> 4) : (ROWS ? b * LP + pos : pos * BB + b);
  }
  // CM: index of component s of element e
  __device__ __forceinline__ static constexpr int ixe(int e, int s, int b) {
    return ((s * 2 + (e & 1)) * (K / 2) + (e >> 1)) * BB + b;
  }
  // position e * n + c (0 <= c < n) given as element and component
  __device__ __forceinline__ static constexpr int ixp(int e, int c, int b) {
    return CM ? ixe(e, c, b) : ix(e * NN + c, b);
  }
  static constexpr int B = BB, Bh = (BB + 1) / 2, Bm = (m & 1) ? Bh : 0;
  static constexpr int NPAIR = B * half;
  // PK (one-line tiles, m odd; C2's n = 4, K = 4096): the middle job's second
  // line is a phantom, so its imaginary part carries the line's nodal values
  // instead and yields the even-index half of the nodal DST-I (forward: X_2k'
  // = (Re Z_k' - Re Z_{N-k'}) / 2; inverse: the antisymmetrised slots
  // (s_t - s_{N-t}) / 2 ride in the real part and come back as Im u_k').  Only
  // the odd-index nodal job remains: J = half + 2 jobs instead of half + 3, which
  // is what lets a K = 4096 line's FFT work fit in shared memory (192 KB).
  static constexpr bool PK = !GW && BB == 1 && (m & 1) != 0;
  static constexpr int ND = PK ? 1 : 2 * Bh;  // nodal jobs
  static constexpr int J = NPAIR + Bm + ND;
  static constexpr int THREADS = TH;
  static constexpr int WD = 2 * J * K;  // FFT buffer (doubles)
  static constexpr int TD = CM ? NN * K * B : ((ROWS || PAD) ? LP : L) * B;  // tile (doubles)
  static constexpr int REGION = (GW || TD > WD) ? TD : WD;  // GW: FFT work in global scratch
  static constexpr int NCEN = m * B;  // centre sums
  static constexpr int CHUNKS = NCEN > 0 ? (TH / NCEN > 0 ? TH / NCEN : 1) : 1;
  // elements per chunk; CM: twice an odd count, so the chunks of the lanes of a warp start in alternate bank halves
  static constexpr int ECH0 = (K + CHUNKS - 1) / CHUNKS;
  static constexpr int ECH = CM ? (((ECH0 + 1) / 2) | 1) * 2 : ECH0;
  static constexpr int C0_OFF = REGION;
  static constexpr int PS_OFF = C0_OFF + (NCEN > 0 ? NCEN : 1);
  static constexpr int BASE_OFF = PS_OFF + (NCEN > 0 ? CHUNKS * NCEN : 1);
  static constexpr int TOTAL = BASE_OFF + B;
  static constexpr size_t SMEM = static_cast<size_t>(TOTAL) * sizeof(double);
};

// Radix plans (product = K), chosen so that one pass keeps at most ~24
// complex values per thread in flight (FEW: at most 8 jobs per tile, where
// a radix-16 pass still fits).
template <int K, bool FEW>
struct Plan;
template <bool FEW>
struct Plan<1024, FEW> {
#if SFEM_MID_R16
  static constexpr int NP = FEW ? 3 : 4;
  static constexpr int R[4] = {FEW ? 16 : 8, 8, FEW ? 8 : 4, 4};
#else
  static constexpr int NP = 4;
  static constexpr int R[4] = {8, 8, 4, 4};
#endif
};
template <bool FEW>
struct Plan<2048, FEW> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {16, 16, 8};
};
template <bool FEW>
struct Plan<512, FEW> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {8, 8, 8};
};
template <bool FEW>
struct Plan<256, FEW> {
  static constexpr int NP = 2;
  static constexpr int R[2] = {16, 16};
};
template <bool FEW>
struct Plan<128, FEW> {
  static constexpr int NP = FEW ? 2 : 3;
  static constexpr int R[3] = {FEW ? 16 : 8, FEW ? 8 : 4, 4};
};
template <bool FEW>
struct Plan<64, FEW> {
  static constexpr int NP = 2;
  static constexpr int R[2] = {8, 8};
};
template <bool FEW>
struct Plan<32, FEW> {
  static constexpr int NP = 2;
  static constexpr int R[2] = {8, 4};
};
template <bool FEW>
struct Plan<16, FEW> {
  static constexpr int NP = 1;
  static constexpr int R[1] = {16};
};
template <bool FEW>
struct Plan<4096, FEW> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {16, 16, 16};
};
template <bool FEW>
struct Plan<114, FEW> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {2, 3, 19};
};

// Non-power-of-two K (3 * 2^j, 5 * 2^j, 2^i * 5^j): odd radices run as
// direct DFTs by conjugate pairs (dft_direct).  FEW: radix 16 where it fits.
template <bool FEW>
struct Plan<24, FEW> {
  static constexpr int NP = 2;
  static constexpr int R[2] = {8, 3};
};
template <>
struct Plan<48, true> {
  static constexpr int NP = 2;
  static constexpr int R[2] = {16, 3};
};
template <>
struct Plan<48, false> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {8, 2, 3};
};
template <bool FEW>
struct Plan<96, FEW> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {8, 4, 3};
};
template <>
struct Plan<192, true> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {16, 4, 3};
};
template <>
struct Plan<192, false> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {8, 8, 3};
};
template <>
struct Plan<384, true> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {16, 8, 3};
};
template <>
struct Plan<384, false> {
  static constexpr int NP = 4;
  static constexpr int R[4] = {8, 8, 2, 3};
};
template <>
struct Plan<768, true> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {16, 16, 3};
};
template <>
struct Plan<768, false> {
  static constexpr int NP = 4;
  static constexpr int R[4] = {8, 8, 4, 3};
};
template <bool FEW>
struct Plan<40, FEW> {
  static constexpr int NP = 2;
  static constexpr int R[2] = {8, 5};
};
template <>
struct Plan<80, true> {
  static constexpr int NP = 2;
  static constexpr int R[2] = {16, 5};
};
template <>
struct Plan<80, false> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {8, 2, 5};
};
template <bool FEW>
struct Plan<160, FEW> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {8, 4, 5};
};
template <>
struct Plan<320, true> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {16, 4, 5};
};
template <>
struct Plan<320, false> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {8, 8, 5};
};
template <bool FEW>
struct Plan<100, FEW> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {4, 5, 5};
};
template <bool FEW>
struct Plan<200, FEW> {
  static constexpr int NP = 3;
  static constexpr int R[3] = {8, 5, 5};
};
template <bool FEW>
struct Plan<1000, FEW> {
  static constexpr int NP = 4;
  static constexpr int R[4] = {8, 5, 5, 5};
};

__device__ __forceinline__ int makhoul_src(int t, int N) { return (2 * t < N) ? 2 * t : 2 * N - 1 - 2 * t; }

// Direct DFT of odd length R (K = 114: R = 19) with roots from the K-point
// twiddle table, by conjugate pairs: with s_q = x_q + x_{R-q}, d_q = x_q -
// x_{R-q} and theta = 2 pi q p / R,
//   y_p     = x_0 + sum_q s_q cos(theta) - i sum_q d_q sin(theta)
//   y_{R-p} = x_0 + sum_q s_q cos(theta) + i sum_q d_q sin(theta),
// so an output pair costs 4 (R-1)/2 real FMAs and the (R-1)/2 roots are
// loaded once per butterfly (was R-1 complex products and loads per output).
template <int R, int K>
__device__ __forceinline__ void dft_direct(double2 (&x)[R], const double2* __restrict__ tw) {
  constexpr int H = (R - 1) / 2;
  double cs[H + 1], sn[H + 1];  // cos / sin (2 pi j / R), j = 1..H
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    const double2 w = __ldg(tw + j * (K / R));  // exp(-2 pi i j / R)
    cs[j] = w.x;
    sn[j] = -w.y;
  }
  double2 sq[H + 1], dq[H + 1];
  double2 y0 = x[0];
#pragma unroll
  for (int q = 1; q <= H; ++q) {
    sq[q] = c_add(x[q], x[R - q]);
    dq[q] = c_sub(x[q], x[R - q]);
    y0 = c_add(y0, sq[q]);
  }
#pragma unroll
  for (int p = 1; p <= H; ++p) {
    double2 a = x[0], b = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 1; q <= H; ++q) {
      const int j = (q * p) % R;
      const double c = j <= H ? cs[j] : cs[R - j];
      const double sv = j <= H ? sn[j] : -sn[R - j];
      a.x = fma(sq[q].x, c, a.x);
      a.y = fma(sq[q].y, c, a.y);
      b.x = fma(dq[q].x, sv, b.x);
      b.y = fma(dq[q].y, sv, b.y);
    }
    x[p] = make_double2(a.x + b.y, a.y - b.x);
    x[R - p] = make_double2(a.x - b.y, a.y + b.x);
  }
  x[0] = y0;
}

template <int R, int K>
__device__ __forceinline__ void dft(double2 (&x)[R], const double2* __restrict__ tw) {
  if constexpr (R == 2 || R == 4 || R == 8 || R == 16)
    Dft<R>::run(x);
  else if constexpr (R == 3) {
    // exp(-2 pi i/3) = -1/2 - i sqrt(3)/2
    constexpr double s3 = 0.86602540378443864676;
    const double2 a = x[0], b = x[1], c = x[2];
    const double2 t = c_add(b, c), d = c_sub(b, c);
    x[0] = c_add(a, t);
    const double2 u = make_double2(fma(-0.5, t.x, a.x), fma(-0.5, t.y, a.y));
    // -i sqrt3/2 d
    const double2 v = make_double2(s3 * d.y, -s3 * d.x);
    x[1] = c_add(u, v);
    x[2] = c_sub(u, v);
  } else {
    dft_direct<R, K>(x, tw);
  }
}

// One in-place Stockham pass of radix R after NS points are done, over all J
// interleaved jobs of W[t * J + job].
template <class C, int R, int NS>
__device__ __forceinline__ void fft_pass(double2* W, const double2* __restrict__ tw) {
  constexpr int N = C::N, J = C::J, NR = N / R, ITEMS = NR * J;
  constexpr int IPT = (ITEMS + C::THREADS - 1) / C::THREADS;
  constexpr int TSTEP = N / (NS * R);
  double2 v[IPT][R];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int it = threadIdx.x + i * C::THREADS;
    if (it < ITEMS) {
      const int job = it % J, j = it / J, k = j % NS;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        double2 a = W[(j + q * NR) * J + job];
        if (NS > 1 && q > 0) a = c_mul(a, __ldg(tw + (q * k * TSTEP) % N));
        v[i][q] = a;
      }
      dft<R, N>(v[i], tw);
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int it = threadIdx.x + i * C::THREADS;
    if (it < ITEMS) {
      const int job = it % J, j = it / J, k = j % NS;
      const int outb = (j / NS) * NS * R + k;
#pragma unroll
      for (int pp = 0; pp < R; ++pp) W[(outb + pp * NS) * J + job] = v[i][pp];
    }
  }
  __syncthreads();
}

#ifndef SFEM_MID_DIAG_SKIP
#define SFEM_MID_DIAG_SKIP 0  // diagnostics builds only: 1 skips the FFT passes, 2 the mixes, 3 the fills
#endif
// Radix-16 plans where a radix-16 pass keeps one butterfly per thread
// (SFEM_MID_FEW_RULE = 1: J * N / 16 <= threads, else spills), or with at
// most 8 jobs per tile (rule 0, the original).
#ifndef SFEM_MID_FEW_RULE
#define SFEM_MID_FEW_RULE 0
#endif
template <class C>
__host__ __device__ constexpr bool few_plan() {
  return SFEM_MID_FEW_RULE ? (C::J * (C::N / 16) <= C::THREADS || C::THREADS >= SFEM_MID_FEW_TH)
                           : (C::J <= 8 || C::THREADS >= SFEM_MID_FEW_TH);
}

// One thread group per job (C2's packed one-line tiles: J = 3 jobs x 256
// radix-16 butterflies = 768 threads): the passes of a job only depend on that
// job's data, so each group of N/R threads runs its job's passes behind its
// own named barrier and the three groups drift apart -- one group's
// shared-memory phase overlaps another's butterflies (with block barriers all
// 24 warps sat in the same phase of every pass).
#ifndef SFEM_MID_GROUPED_FFT
#define SFEM_MID_GROUPED_FFT 0  // measured slower on C2 (1.01 -> 1.28 ms: the job-major thread map makes the first pass's stores 8-way conflicted)
#endif
template <class C, int R>
__host__ __device__ constexpr bool grouped_fft() {
  return SFEM_MID_GROUPED_FFT && C::PK && C::THREADS == C::J * (C::N / R) && (C::N / R) % 32 == 0 && C::J <= 15;
}

template <class C, int R, int NS>
__device__ __forceinline__ void fft_pass_grouped(double2* W, const double2* __restrict__ tw) {
  constexpr int N = C::N, J = C::J, NR = N / R;
  constexpr int TSTEP = N / (NS * R);
  const int job = threadIdx.x / NR, j = threadIdx.x - job * NR, k = j % NS;
  double2 v[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    double2 a = W[(j + q * NR) * J + job];
    if (NS > 1 && q > 0) a = c_mul(a, __ldg(tw + (q * k * TSTEP) % N));
    v[q] = a;
  }
  dft<R, N>(v, tw);
  asm volatile("bar.sync %0, %1;" ::"r"(1 + job), "r"(NR) : "memory");
  const int outb = (j / NS) * NS * R + k;
#pragma unroll
  for (int pp = 0; pp < R; ++pp) W[(outb + pp * NS) * J + job] = v[pp];
  asm volatile("bar.sync %0, %1;" ::"r"(1 + job), "r"(NR) : "memory");
}

template <class C, int P = 0, int NS = 1>
__device__ __forceinline__ void fft(double2* W, const double2* __restrict__ tw) {
  using PL = Plan<C::N, few_plan<C>()>;
  if constexpr (P < PL::NP && SFEM_MID_DIAG_SKIP != 1) {
    constexpr int R = PL::R[P];
    if constexpr (grouped_fft<C, R>()) {
      fft_pass_grouped<C, R, NS>(W, tw);
      if constexpr (P + 1 == PL::NP) __syncthreads();  // the post stage reads every job
    } else {
      fft_pass<C, R, NS>(W, tw);
    }
    fft<C, P + 1, NS * R>(W, tw);
  }
}

// Item -> (job, index) for the fill / post stages with warps uniform in the
// job kind: items are grouped pair jobs | middle jobs | nodal jobs, each
// group index-major with its jobs fastest (consecutive lanes write
// consecutive W entries of one index: conflict-free).
template <class C, int NT>
__device__ __forceinline__ void item_job(int it, int& job, int& t) {
  constexpr int NP = C::NPAIR, NM = C::Bm, ND = C::ND;
  constexpr int P = NP * NT, PM = (NP + NM) * NT;
  if (NP > 0 && it < P) {
    job = it % (NP > 0 ? NP : 1);
    t = it / (NP > 0 ? NP : 1);
  } else if (NM > 0 && it < PM) {
    const int r = it - P;
    job = NP + r % (NM > 0 ? NM : 1);
    t = r / (NM > 0 ? NM : 1);
  } else {
    const int r = it - PM;
    job = NP + NM + r % ND;
    t = r / ND;
  }
}

// Out-of-place Stockham passes X -> Y (global-memory work buffers for lines
// too long for shared memory): one item at a time per thread, no bridge.
template <class C, int R, int NS>
__device__ __forceinline__ void fft_pass_oop(const double2* X, double2* Y, const double2* __restrict__ tw) {
  constexpr int N = C::N, J = C::J, NR = N / R, ITEMS = NR * J;
  constexpr int TSTEP = N / (NS * R);
  for (int it = threadIdx.x; it < ITEMS; it += C::THREADS) {
    const int job = it % J, j = it / J, k = j % NS;
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      double2 a = X[(j + q * NR) * J + job];
      if (NS > 1 && q > 0) a = c_mul(a, __ldg(tw + (q * k * TSTEP) % N));
      v[q] = a;
    }
    dft<R, N>(v, tw);
    const int outb = (j / NS) * NS * R + k;
#pragma unroll
    for (int pp = 0; pp < R; ++pp) Y[(outb + pp * NS) * J + job] = v[pp];
  }
  __syncthreads();
}

// Global FFT work slices (sweep_mid_gw): every dead slice is dropped from L2
// without write-back as soon as a pass has consumed it, so at most one dirty
// slice per CTA competes for L2.  With both slices only discarded at exit,
// C2 wrote 3.61 GB to DRAM per launch against 0.54 GB of results
// (profiles/r1n_ncu_full_c2.json): the 148 x 0.52 MB of work slices were
// being evicted dirty.
#ifndef SFEM_MID_GW_DISCARD
#define SFEM_MID_GW_DISCARD 1
#endif
template <class C>
__device__ __forceinline__ void discard_l2(const double2* W) {
  constexpr int LINES = (C::J * C::N * 16) / 128;
  const char* wb = reinterpret_cast<const char*>(W);
  for (int i = threadIdx.x; i < LINES; i += C::THREADS)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(wb + static_cast<size_t>(i) * 128) : "memory");
}

// Returns the buffer holding the result.
template <class C, int P = 0, int NS = 1>
__device__ __forceinline__ double2* fft_oop(double2* X, double2* Y, const double2* __restrict__ tw) {
  using PL = Plan<C::N, few_plan<C>()>;
  if constexpr (P < PL::NP) {
    constexpr int R = PL::R[P];
    fft_pass_oop<C, R, NS>(X, Y, tw);  // ends with a barrier: X is dead
#if SFEM_MID_GW_DISCARD
    discard_l2<C>(X);
    __syncthreads();  // the discards land before the next pass writes X
#endif
    return fft_oop<C, P + 1, NS * R>(Y, X, tw);
  } else {
    return X;
  }
}

// ------------------------------------------------------------ forward fill
// W[t][job] from the tile (bridge), plus the chunked centre partial sums.
// SEP: the tile T is a separate staging buffer, so W is written directly
// (no bridge); otherwise T aliases the region R.
template <class C, bool SEP = false>
__device__ __forceinline__ void forward_fill(const double* T, double* R, double* PS, const double2* __restrict__ om) {
  constexpr int N = C::N, n = C::n, m = C::m, B = C::B, Bh = C::Bh, J = C::J, NPAIR = C::NPAIR;
  constexpr int ITEMS = SFEM_MID_DIAG_SKIP == 3 ? 0 : N * J, IPT = (N * J + C::THREADS - 1) / C::THREADS;
  double2* W = reinterpret_cast<double2*>(R);
  double2 z[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int it = threadIdx.x + i * C::THREADS;
    z[i] = make_double2(0.0, 0.0);
    if (it < ITEMS) {
      int job, tt;
      item_job<C, N>(it, job, tt);
      if (job < NPAIR) {
        const int ii = job / B, b = job % B;
        const int e = makhoul_src(tt, N);
        const double ri = T[C::ixp(e, ii, b)], rr = T[C::ixp(e, m - 1 - ii, b)];
        double gg = ri + rr;
        if (e & 1) gg = -gg;
        z[i] = make_double2(ri - rr, gg);
      } else if (job < NPAIR + C::Bm) {
        const int b = job - NPAIR, b2 = b + Bh;
        const int e = makhoul_src(tt, N);
        double g1 = T[C::ixp(e, C::half, b)];
        double g2 = b2 < B ? T[C::ixp(e, C::half, b2)] : 0.0;
        if (e & 1) {
          g1 = -g1;
          g2 = -g2;
        }
        if (C::PK) g2 = tt > 0 ? T[C::ixp(tt - 1, n - 1, b)] : 0.0;  // nodal values (even-index DST-I half)
        z[i] = make_double2(g1, g2);
      } else {
        const int jb = job - NPAIR - C::Bm;
        const int b = jb % Bh, which = C::PK ? 1 : jb / Bh, b2 = b + Bh;
        if (tt > 0) {
          z[i] = make_double2(T[C::ixp(tt - 1, n - 1, b)], b2 < B ? T[C::ixp(tt - 1, n - 1, b2)] : 0.0);
          if (which) z[i] = c_mul(z[i], __ldg(om + tt));
        }
      }
      if (SEP) W[tt * J + job] = z[i];
    }
  }
  // centre partials: sum (i, b) over elements [c * ECH, (c+1) * ECH)
  double part = 0.0;
  const int cit = threadIdx.x;
  if constexpr (C::NCEN > 0) {
    if (cit < C::CHUNKS * C::NCEN) {
      const int s = cit % C::NCEN, c = cit / C::NCEN;
      const int ii = s / B, b = s % B;
      const int e0 = c * C::ECH, e1 = min(N, e0 + C::ECH);
      for (int e = e0; e < e1; ++e) part += (e & 1) ? -T[C::ixp(e, m - 1 - ii, b)] : T[C::ixp(e, ii, b)];
    }
  }
  if (!SEP) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int it = threadIdx.x + i * C::THREADS;
      if (it < ITEMS) {
        int job, tt;
        item_job<C, N>(it, job, tt);
        W[tt * J + job] = z[i];
      }
    }
  }
  if (C::NCEN > 0 && cit < C::CHUNKS * C::NCEN) PS[cit] = part;  // NCEN = 0: no centre (n = 1)
  __syncthreads();
}

// ---- fill fused into the first pass (in-place kernels) ----------------------
// The first Stockham pass (NS = 1, no twiddles) reads its butterfly inputs
// straight from the tile (forward) or the slots (inverse) instead of from a
// W buffer a separate fill stage wrote: one write and one read of the whole
// FFT buffer and two block barriers fewer per transform.  Items are grouped by
// job kind (item_job) so a warp's element code is uniform.
template <class C>
__device__ __forceinline__ double2 forward_elem(const double* T, int job, int tt, const double2* __restrict__ om) {
  constexpr int N = C::N, n = C::n, m = C::m, B = C::B, Bh = C::Bh, NPAIR = C::NPAIR;
  double2 z = make_double2(0.0, 0.0);
  if (job < NPAIR) {
    const int ii = job / B, b = job % B;
    const int e = makhoul_src(tt, N);
    const double ri = T[C::ixp(e, ii, b)], rr = T[C::ixp(e, m - 1 - ii, b)];
    double gg = ri + rr;
    if (e & 1) gg = -gg;
    z = make_double2(ri - rr, gg);
  } else if (job < NPAIR + C::Bm) {
    const int b = job - NPAIR, b2 = b + Bh;
    const int e = makhoul_src(tt, N);
    double g1 = T[C::ixp(e, C::half, b)];
    double g2 = b2 < B ? T[C::ixp(e, C::half, b2)] : 0.0;
    if (e & 1) {
      g1 = -g1;
      g2 = -g2;
    }
    if (C::PK) g2 = tt > 0 ? T[C::ixp(tt - 1, n - 1, b)] : 0.0;
    z = make_double2(g1, g2);
  } else {
    const int jb = job - NPAIR - C::Bm;
    const int b = jb % Bh, which = C::PK ? 1 : jb / Bh, b2 = b + Bh;
    if (tt > 0) {
      z = make_double2(T[C::ixp(tt - 1, n - 1, b)], b2 < B ? T[C::ixp(tt - 1, n - 1, b2)] : 0.0);
      if (which) z = c_mul(z, __ldg(om + tt));
    }
  }
  return z;
}

template <class C>
__device__ __forceinline__ void centre_partials(const double* T, double* PS) {
  constexpr int N = C::N, n = C::n, m = C::m, B = C::B;
  if constexpr (C::NCEN > 0) {
    const int cit = threadIdx.x;
    if (cit < C::CHUNKS * C::NCEN) {
      // CM: a warp covers four consecutive chunks of one component (rows of one plane pair)
      const int s = C::CM ? (cit / (B * C::CHUNKS)) * B + cit % B : cit % C::NCEN;
      const int c = C::CM ? (cit / B) % C::CHUNKS : cit / C::NCEN;
      const int ii = s / B, b = s % B;
      const int e0 = c * C::ECH, e1 = min(N, e0 + C::ECH);
      double part = 0.0;
      for (int e = e0; e < e1; ++e) part += (e & 1) ? -T[C::ixp(e, m - 1 - ii, b)] : T[C::ixp(e, ii, b)];
      PS[c * C::NCEN + s] = part;
    }
  }
}

// First pass of radix R with element source `elem(job, t)`; W aliases the
// source, so every thread loads all its inputs before the barrier.
template <class C, int R, class F>
__device__ __forceinline__ void fft_pass_first(double2* W, const double2* __restrict__ tw, F elem) {
  constexpr int N = C::N, J = C::J, NR = N / R, ITEMS = NR * J;
  constexpr int IPT = (ITEMS + C::THREADS - 1) / C::THREADS;
  double2 v[IPT][R];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int it = threadIdx.x + i * C::THREADS;
    if (it < ITEMS) {
      int job, j;
      item_job<C, NR>(it, job, j);
#pragma unroll
      for (int q = 0; q < R; ++q) v[i][q] = elem(job, j + q * NR);
      dft<R, N>(v[i], tw);
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int it = threadIdx.x + i * C::THREADS;
    if (it < ITEMS) {
      int job, j;
      item_job<C, NR>(it, job, j);
#pragma unroll
      for (int pp = 0; pp < R; ++pp) W[(j * R + pp) * J + job] = v[i][pp];
    }
  }
  __syncthreads();
}

#ifndef SFEM_MID_FUSED_FILL
#define SFEM_MID_FUSED_FILL 1
#endif

// Forward transform of the tile in R (in place): fill + FFT, W = R.
template <class C>
__device__ __forceinline__ void forward_fft_inplace(double* R, double* PS, const double2* __restrict__ tw,
                                                    const double2* __restrict__ om) {
  using PL = Plan<C::N, few_plan<C>()>;
  double2* W = reinterpret_cast<double2*>(R);
  // (not for the one-line tiles of C2: 1.01 -> 1.11 ms there)
  if constexpr (SFEM_MID_FUSED_FILL && !C::PAD) {
    centre_partials<C>(R, PS);
    fft_pass_first<C, PL::R[0]>(W, tw, [&](int job, int t) { return forward_elem<C>(R, job, t, om); });
    fft<C, 1, PL::R[0]>(W, tw);
  } else {
    forward_fill<C>(R, R, PS, om);
    fft<C>(W, tw);
  }
}

// C0[s] = sum over chunks in order.
template <class C>
__device__ __forceinline__ void centre_reduce(const double* PS, double* C0) {
  for (int s = threadIdx.x; s < C::NCEN; s += C::THREADS) {
    double acc = 0.0;
#pragma unroll 4
    for (int c = 0; c < C::CHUNKS; ++c) acc += PS[c * C::NCEN + s];
    C0[s] = acc;
  }
}

// ------------------------------------------------------------ forward post
// FFT results -> slots S (at tile positions m + (k-1) n + s), bridge.
// One post item: up to two slot values and their tile indices (-1: none).
struct Out2 {
  double v1, v2;
  int i1, i2;
};

template <class C>
__device__ __forceinline__ Out2 forward_post_item(const double2* Z, int it, const double2* __restrict__ mk) {
  constexpr int N = C::N, n = C::n, m = C::m, B = C::B, Bh = C::Bh, J = C::J, NPAIR = C::NPAIR;
  Out2 o{0.0, 0.0, -1, -1};
  int job, k;
  item_job<C, N - 1>(it, job, k);
  k += 1;
  if (job < NPAIR + C::Bm) {
    const double2 zk = Z[k * J + job], zc = Z[(N - k) * J + job];
    const double2 w = __ldg(mk + k);
    // r1 = Re(mk_k V1), r2 = Re(mk_k V2), V1 = (Z_k + conj Z_{N-k})/2, V2 = (Z_k - conj Z_{N-k})/(2i)
    const double a1 = 0.5 * (zk.x + zc.x), b1 = 0.5 * (zk.y - zc.y);
    const double a2 = 0.5 * (zk.y + zc.y), b2 = -0.5 * (zk.x - zc.x);
    o.v1 = w.x * a1 - w.y * b1;
    o.v2 = w.x * a2 - w.y * b2;
    if (job < NPAIR) {
      const int ii = job / B, b = job % B;
      o.i1 = C::ixp(k, C::ne + ii, b);  // H_k
      o.i2 = C::ixp(N - k, ii, b);      // G_{N-k}
    } else {
      const int b = job - NPAIR, bb = b + Bh;
      o.i1 = C::ixp(N - k, C::half, b);
      if (bb < B) o.i2 = C::ixp(N - k, C::half, bb);
      if (C::PK && (k & 1) == 0) {
        // even nodal frequency k = 2 kp from the imaginary payload
        const int kp = k / 2;
        o.v2 = 0.5 * (Z[kp * J + job].x - Z[(N - kp) * J + job].x);
        o.i2 = C::ixp(k - 1, n - 1, b);
      }
    }
  } else {
    const int jb = job - NPAIR - C::Bm;
    const int b = jb % Bh, which = C::PK ? 1 : jb / Bh, bb = b + Bh;
    if ((k & 1) == which) {
      double2 d;
      if (!which) {
        const int kp = k / 2;
        d = c_sub(Z[(N - kp) * J + job], Z[kp * J + job]);
      } else {
        const int kp = (k - 1) / 2;
        d = c_sub(Z[(N - 1 - kp) * J + job], Z[kp * J + job]);
      }
      // X = d / (2i)
      o.v1 = 0.5 * d.y;
      o.v2 = -0.5 * d.x;
      o.i1 = C::ixp(k - 1, n - 1, b);
      if (bb < B) o.i2 = C::ixp(k - 1, n - 1, bb);
    }
  }
  return o;
}

// Runs ITEMS items of f into the tile R: bridged (all items loaded, barrier,
// all stored) when the source aliases R, direct otherwise.
template <class C, bool SEP, int ITEMS, class F>
__device__ __forceinline__ void run_out2(double* R, F f) {
  if constexpr (SEP) {
    for (int it = threadIdx.x; it < ITEMS; it += C::THREADS) {
      const Out2 o = f(it);
      if (o.i1 >= 0) R[o.i1] = o.v1;
      if (o.i2 >= 0) R[o.i2] = o.v2;
    }
  } else {
    // Only the values cross the barrier in registers; the target indices are
    // recomputed afterwards (f is called again and only its index part is
    // used, so its loads are dead): 4 registers per item instead of 6, which
    // is what spilled in the 20-items-per-thread tiles.
    constexpr int IPT = (ITEMS + C::THREADS - 1) / C::THREADS;
    double v1[IPT], v2[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int it = threadIdx.x + i * C::THREADS;
      v1[i] = v2[i] = 0.0;
      if (it < ITEMS) {
        const Out2 o = f(it);
        v1[i] = o.v1;
        v2[i] = o.v2;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int it = threadIdx.x + i * C::THREADS;
      if (it < ITEMS) {
        const Out2 o = f(it);
        if (o.i1 >= 0) R[o.i1] = v1[i];
        if (o.i2 >= 0) R[o.i2] = v2[i];
      }
    }
  }
  __syncthreads();
}

// FFT results -> slots S (at tile positions m + (k-1) n + s).
template <class C, bool SEP = false>
__device__ __forceinline__ void forward_post(const double2* Z, double* R, const double2* __restrict__ mk) {
  run_out2<C, SEP, (C::N - 1) * C::J>(R, [&](int it) { return forward_post_item<C>(Z, it, mk); });
}

// ------------------------------------------------------------ mixes
// Symbol divide c / d (d > 0): MUFU reciprocal seed, one Newton step, one
// residual correction of the quotient -- within 1 ulp of IEEE division (the
// fast kernels' sym_div, measured over 2^30 quotients by tools/div_ulp.cu)
// at a third of the instructions of the IEEE division sequence.
#ifndef SFEM_MID_FAST_DIV
#define SFEM_MID_FAST_DIV 1
#endif
__device__ __forceinline__ double mid_div(double c, double d) {
#if SFEM_MID_FAST_DIV
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = fma(r, fma(-d, r, 1.0), r);
  const double q = c * r;
  return fma(fma(-d, q, c), r, q);
#else
  return c / d;
#endif
}

// Per (k >= 1, line) item, in place at tile positions m + (k-1) n + [0, n):
//   MODE kForward:             c = Mf v
//   MODE kInverse:             u = Mi c
//   MODE kForwardDivideInverse u = Mi (Mf v / denom)
// Items (K-1)*B .. (K-1)*B + B - 1 are the centre blocks of the lines.
//
// SFEM_MID_KMIX (default): the matrices are the k-contiguous copies mixT_w/d
// ([l][s][k]) and mixT_i ([s][l][k]).  Items run b-fastest, so a warp covers
// 32/B consecutive frequencies and one matrix load is one or a few 32-byte
// sectors instead of 32/B of them (the per-frequency [k][l][s] layout).
// C3 (n=9, K=1024: 0.66 MB per matrix set, not L1-resident): solve 8.30 ->
// 4.92 ms; C5 n=4 / n=9: -6 % / -5 % (bitwise-identical results).
template <class C, int MODE>
__device__ __forceinline__ void mix(const double* Tin, double* T, double* C0, const double* __restrict__ mixF,
                                    const double* __restrict__ e0F, const double* __restrict__ mixI,
                                    const double* __restrict__ e0I, const double* base,
                                    const double* __restrict__ eig, double f_last,
                                    const double* __restrict__ eigT = nullptr) {
  constexpr int N = C::N, n = C::n, m = C::m, B = C::B;
#if SFEM_MID_KMIX
#define MIDX(a, b) (((a) * n + (b)) * N)
#else
#define MIDX(a, b) ((a) * n + (b))
#endif
  // G lines per (k >= 1) item: one matrix load feeds G FMAs (SFEM_MID_MIXG).
  constexpr int G = (SFEM_MID_MIXG >= 4 && MODE == kForwardDivideInverse && B % 4 == 0 && 4 * n <= 20) ? 4
                    : (SFEM_MID_MIXG >= 2 && B % 2 == 0)              ? 2
                                                                       : 1;
  constexpr int BG = B / G;
  constexpr int KITEMS = (N - 1) * BG;
  constexpr int ITEMS = (SFEM_MID_DIAG_SKIP == 2) ? 0 : KITEMS + B;
  for (int it = threadIdx.x; it < ITEMS; it += C::THREADS) {
    if (it < KITEMS) {
      const int k = 1 + it / BG, b0 = (it % BG) * G;
      double v[G][n], c[G][n];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double* pin = Tin + C::ix(m + (k - 1) * n, b0 + g);
#pragma unroll
        for (int s = 0; s < n; ++s)
          v[g][s] = C::CM ? Tin[C::ixe(k - 1 + (s > 0), s > 0 ? s - 1 : n - 1, b0 + g)]
                          : (C::PAD ? Tin[C::ix(m + (k - 1) * n + s, b0 + g)] : pin[s * C::PSTR]);
      }
      if (MODE != kInverse) {
#if SFEM_MID_KMIX
        const double* M = mixF + k;
#pragma unroll
        for (int g = 0; g < G; ++g) v[g][0] *= 2.0;  // the nodal column of mixT_* carries a factor 1/2 (exact)
#else
        const double* M = mixF + static_cast<size_t>(k - 1) * n * n;
#endif
#pragma unroll
        for (int l = 0; l < n; ++l) {
          double acc[G];
#pragma unroll
          for (int g = 0; g < G; ++g) acc[g] = 0.0;
#pragma unroll
          for (int s = 0; s < n; ++s) {
            const double mv = __ldg(M + MIDX(l, s));
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = fma(mv, v[g][s], acc[g]);
          }
          if (MODE == kForwardDivideInverse) {
            const double ev = __ldg(eigT + l * N + k);  // k-contiguous copy: lanes over k read one line
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = mid_div(acc[g], base[b0 + g] + f_last * ev);
          }
#pragma unroll
          for (int g = 0; g < G; ++g) c[g][l] = acc[g];
        }
      } else {
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int l = 0; l < n; ++l) c[g][l] = v[g][l];
      }
      if (MODE != kForward) {
#if SFEM_MID_KMIX
        const double* M = mixI + k;
#else
        const double* M = mixI + static_cast<size_t>(k - 1) * n * n;
#endif
#pragma unroll
        for (int s = 0; s < n; ++s) {
          double acc[G];
#pragma unroll
          for (int g = 0; g < G; ++g) acc[g] = 0.0;
#pragma unroll
          for (int l = 0; l < n; ++l) {
            const double mv = __ldg(M + MIDX(s, l));
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = fma(mv, c[g][l], acc[g]);
          }
#pragma unroll
          for (int g = 0; g < G; ++g) v[g][s] = acc[g];
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
#if SFEM_MID_KMIX
          v[g][0] *= 2.0;  // nodal row of mixT_i carries 1/2 (exact)
#endif
          double* p = T + C::ix(m + (k - 1) * n, b0 + g);
#pragma unroll
          for (int s = 0; s < n; ++s)
            (C::CM ? T[C::ixe(k - 1 + (s > 0), s > 0 ? s - 1 : n - 1, b0 + g)]
                   : (C::PAD ? T[C::ix(m + (k - 1) * n + s, b0 + g)] : p[s * C::PSTR])) = v[g][s];
        }
      } else {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          double* p = T + C::ix(m + (k - 1) * n, b0 + g);
#pragma unroll
          for (int l = 0; l < n; ++l)
            (C::CM ? T[C::ixe(k - 1 + (l > 0), l > 0 ? l - 1 : n - 1, b0 + g)]
                   : (C::PAD ? T[C::ix(m + (k - 1) * n + l, b0 + g)] : p[l * C::PSTR])) = c[g][l];
        }
      }
    } else if (m > 0) {
      // centre block of line b: coefficients l < m (k = 0)
      const int b = it - KITEMS;
      double c[m > 0 ? m : 1];
      if (MODE != kInverse) {
#pragma unroll
        for (int l = 0; l < m; ++l) {
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < m; ++i) acc = fma(C0[i * B + b], __ldg(e0F + i * m + l), acc);
          if (MODE == kForwardDivideInverse) acc = mid_div(acc, base[b] + f_last * __ldg(eig + l));
          c[l] = acc;
        }
      } else {
#pragma unroll
        for (int l = 0; l < m; ++l) c[l] = Tin[C::ixp(0, l, b)];
      }
      if (MODE == kForward) {
#pragma unroll
        for (int l = 0; l < m; ++l) T[C::ixp(0, l, b)] = c[l];
      } else {
        // centre of the synthesis: C0[i] = sum_l e0_inv[i][l] c[l]
#pragma unroll
        for (int i = 0; i < m; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < m; ++l) acc = fma(__ldg(e0I + i * m + l), c[l], acc);
          C0[i * B + b] = acc;
        }
      }
    }
  }
  __syncthreads();
}

#undef MIDX

// ------------------------------------------------------------ inverse fill
template <class C>
__device__ __forceinline__ double2 inverse_elem(const double* T, int job, int tt, const double2* __restrict__ mkh,
                                                const double2* __restrict__ om);

template <class C>
__device__ __forceinline__ double2 inverse_fill_item(const double* T, int it, int& widx,
                                                     const double2* __restrict__ mkh, const double2* __restrict__ om) {
  int job, tt;
  item_job<C, C::N>(it, job, tt);
  widx = tt * C::J + job;
  return inverse_elem<C>(T, job, tt, mkh, om);
}

template <class C>
__device__ __forceinline__ double2 inverse_elem(const double* T, int job, int tt, const double2* __restrict__ mkh,
                                                const double2* __restrict__ om) {
  constexpr int N = C::N, n = C::n, m = C::m, B = C::B, Bh = C::Bh, NPAIR = C::NPAIR;
  double2 z = make_double2(0.0, 0.0);
  if (tt > 0) {
    if (job < NPAIR + C::Bm) {
      const double2 w = __ldg(mkh + tt);
      double ax, ar, bx, br;  // V1 = w (ax - i ar), V2 = w (bx - i br)
      if (job < NPAIR) {
        const int ii = job / B, b = job % B;
        ax = T[C::ixp(tt, C::ne + ii, b)];
        ar = T[C::ixp(N - tt, C::ne + ii, b)];
        bx = T[C::ixp(N - tt, ii, b)];
        br = T[C::ixp(tt, ii, b)];
      } else {
        const int b = job - NPAIR, b2 = b + Bh;
        ax = T[C::ixp(N - tt, C::half, b)];
        ar = T[C::ixp(tt, C::half, b)];
        bx = b2 < B ? T[C::ixp(N - tt, C::half, b2)] : 0.0;
        br = b2 < B ? T[C::ixp(tt, C::half, b2)] : 0.0;
      }
      const double2 v1 = c_mul(w, make_double2(ax, -ar));
      const double2 v2 = c_mul(w, make_double2(bx, -br));
      // conj(V1 + i V2): the inverse DFT runs as a forward FFT of the conjugate
      z = make_double2(v1.x - v2.y, -(v1.y + v2.x));
      if (C::PK && job >= NPAIR) {
        // + (s_t - s_{N-t}) / 2 (antisymmetric, real): its inverse DFT is i * sum_t s_t sin(2 pi t j / N)
        const int b = job - NPAIR;
        z.x += 0.5 * (T[C::ixp(tt - 1, n - 1, b)] - T[C::ixp(N - tt - 1, n - 1, b)]);
      }
    } else {
      const int jb = job - NPAIR - C::Bm;
      const int b = jb % Bh, which = C::PK ? 1 : jb / Bh, b2 = b + Bh;
      z = make_double2(T[C::ixp(tt - 1, n - 1, b)], b2 < B ? T[C::ixp(tt - 1, n - 1, b2)] : 0.0);
      if (which) z = c_mul(z, __ldg(om + tt));
    }
  }
  return z;
}

// Slots (tile) -> W; bridged when W aliases the tile.
template <class C, bool SEP = false>
__device__ __forceinline__ void inverse_fill(const double* T, double2* W, const double2* __restrict__ mkh,
                                             const double2* __restrict__ om) {
  constexpr int ITEMS = SFEM_MID_DIAG_SKIP == 3 ? 0 : C::N * C::J;
  if constexpr (SEP) {
    for (int it = threadIdx.x; it < ITEMS; it += C::THREADS) {
      int widx;
      const double2 z = inverse_fill_item<C>(T, it, widx, mkh, om);
      W[widx] = z;
    }
  } else {
    constexpr int IPT = (C::N * C::J + C::THREADS - 1) / C::THREADS;
    double2 z[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int it = threadIdx.x + i * C::THREADS;
      int widx;
      if (it < ITEMS) z[i] = inverse_fill_item<C>(T, it, widx, mkh, om);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int it = threadIdx.x + i * C::THREADS;
      if (it < ITEMS) {
        int job, tt;
        item_job<C, C::N>(it, job, tt);
        W[tt * C::J + job] = z[i];
      }
    }
  }
  __syncthreads();
}

// Inverse transform of the slots in R (in place): fill + FFT, W = R.
template <class C>
__device__ __forceinline__ void inverse_fft_inplace(double* R, const double2* __restrict__ tw,
                                                    const double2* __restrict__ mkh, const double2* __restrict__ om) {
  using PL = Plan<C::N, few_plan<C>()>;
  double2* W = reinterpret_cast<double2*>(R);
  if constexpr (SFEM_MID_FUSED_FILL && !C::PAD) {
    fft_pass_first<C, PL::R[0]>(W, tw, [&](int job, int t) { return inverse_elem<C>(R, job, t, mkh, om); });
    fft<C, 1, PL::R[0]>(W, tw);
  } else {
    inverse_fill<C>(R, W, mkh, om);
    fft<C>(W, tw);
  }
}

// ------------------------------------------------------------ inverse post
template <class C>
__device__ __forceinline__ Out2 inverse_post_item(const double2* Z, int it, const double* C0) {
  constexpr int N = C::N, n = C::n, m = C::m, B = C::B, Bh = C::Bh, J = C::J, NPAIR = C::NPAIR;
  Out2 o{0.0, 0.0, -1, -1};
  int job, tt;
  item_job<C, N>(it, job, tt);
  if (job < NPAIR + C::Bm) {
    const double2 u = Z[tt * J + job];
    const double ure = u.x, uim = -u.y;
    const int e = makhoul_src(tt, N);
    const bool odd = e & 1;
    if (job < NPAIR) {
      const int ii = job / B, b = job % B;
      const double ev = odd ? -uim : uim;
      const double ci = odd ? -C0[(m - 1 - ii) * B + b] : C0[ii * B + b];
      const double cr = odd ? -C0[ii * B + b] : C0[(m - 1 - ii) * B + b];
      o.v1 = ci + ev + ure;
      o.v2 = cr + ev - ure;
      o.i1 = C::ixp(e, ii, b);
      o.i2 = C::ixp(e, m - 1 - ii, b);
    } else {
      const int b = job - NPAIR, b2 = b + Bh;
      constexpr int hc = C::half;
      const double c1 = odd ? -C0[hc * B + b] : C0[hc * B + b];
      o.v1 = c1 + (odd ? -ure : ure);
      o.i1 = C::ixp(e, hc, b);
      if (b2 < B) {
        const double c2 = odd ? -C0[hc * B + b2] : C0[hc * B + b2];
        o.v2 = c2 + (odd ? -uim : uim);
        o.i2 = C::ixp(e, hc, b2);
      }
      if (C::PK && tt >= 1 && 2 * tt <= N - 1) {
        o.v2 = uim;  // node 2 tt
        o.i2 = C::ix(2 * tt * n - 1, b);
      }
    }
  } else {
    const int jb = job - NPAIR - C::Bm;
    const int b = jb % Bh, which = C::PK ? 1 : jb / Bh, b2 = b + Bh;
    const int j = tt;
    if (j >= 1 && j <= N - 1 && (j & 1) == which) {
      double2 d;
      if (!which) {
        const int kp = j / 2;
        d = c_sub(Z[(N - kp) * J + job], Z[kp * J + job]);
      } else {
        const int kp = (j - 1) / 2;
        d = c_sub(Z[(N - 1 - kp) * J + job], Z[kp * J + job]);
      }
      o.v1 = 0.5 * d.y;
      o.i1 = C::ixp(j - 1, n - 1, b);
      if (b2 < B) {
        o.v2 = -0.5 * d.x;
        o.i2 = C::ixp(j - 1, n - 1, b2);
      }
    }
  }
  return o;
}

// FFT results + centre -> the line tile R.
template <class C, bool SEP = false>
__device__ __forceinline__ void inverse_post(const double2* Z, double* R, const double* C0) {
  run_out2<C, SEP, C::N * C::J>(R, [&](int it) { return inverse_post_item<C>(Z, it, C0); });
}

// ------------------------------------------------------------ kernel
// Resident CTAs per SM asked of ptxas: two for CTAs of up to 384 threads
// (four / two for 128 / 256), one above.
__host__ __device__ constexpr int mid_min_blocks(int th) { return th <= 256 ? 512 / th : (th <= 384 ? 2 : 1); }
// n = 1 tiles (no mixes, 65 KB of shared memory): three CTAs per SM (85 registers), C5 n=1 60.5 -> 56.1 ms
#ifndef SFEM_MID_MINB_N1
#define SFEM_MID_MINB_N1 3
#endif
__host__ __device__ constexpr int mid_min_blocks_n(int nn, int th) {
  return (nn == 1 && th == 256) ? SFEM_MID_MINB_N1 : mid_min_blocks(th);
}

__device__ __forceinline__ unsigned mid_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}

__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}

// Strided tiles whose B lines are adjacent, 16-byte aligned and all present:
// each position row (B doubles, contiguous in both places) moves as B/2
// 16-byte copies / stores instead of B 8-byte ones.
template <class C>
__device__ __forceinline__ bool vec_tile(const long long* off, int Bv, long long ps, const double* src,
                                         const double* dst) {
  if constexpr (C::ROWS || (C::B & 1)) return false;
  bool ok = Bv == C::B && (off[0] & 1) == 0 && (ps & 1) == 0 &&
            ((reinterpret_cast<unsigned long long>(src) | reinterpret_cast<unsigned long long>(dst)) & 15) == 0;
#pragma unroll
  for (int b = 1; b < C::B; ++b) ok = ok && off[b] == off[0] + b;
  return ok;
}

template <int NN, int K, int BB, int TH, int MODE, bool ROWS>
__global__ void __launch_bounds__(TH, mid_min_blocks_n(NN, TH))  // <= 128 registers
    sweep_mid(DevTable t, LineSet ls, SymbolInfo sym, const double* __restrict__ mixF,
              const double* __restrict__ e0F) {
  using C = Cfg<NN, K, BB, TH, ROWS>;
  constexpr int B = C::B, L = C::L;
  extern __shared__ __align__(128) double smem[];
  double* R = smem;
  double* C0 = smem + C::C0_OFF;
  double* PS = smem + C::PS_OFF;
  double* base = smem + C::BASE_OFF;
  __shared__ long long off[B];
  SFEM_PT_DECL;
  SFEM_PT(0);

  const long long l0 = static_cast<long long>(blockIdx.x) * B;
  const int Bv = static_cast<int>(min(static_cast<long long>(B), ls.nlines - l0));
  if (threadIdx.x < B) {
    const int b = threadIdx.x;
    const long long l = l0 + b;
    const long long r = l / ls.ninner;
    off[b] = l < ls.nlines ? (r / ls.n1) * ls.os2 + (r % ls.n1) * ls.os1 + (l % ls.ninner) * ls.is : 0;
    if (MODE == kForwardDivideInverse && sym.xblk > 0) {
      // blocked 3-D layout (capi.cu build_blocked_steps): row (x_hi, y, x_lo), x = x_hi*xblk + x_lo
      const long long lb = l < ls.nlines ? l : 0;
      const long long xlo = lb % sym.xblk, r1 = lb / sym.xblk;
      const long long y = r1 % sym.lead_ext[1], xhi = r1 / sym.lead_ext[1];
      const long long x = min(xhi * sym.xblk + xlo, sym.x_ext - 1);  // padding rows: any finite base
      const double t0 = sym.lead_f[0] * sym.lead_eig[0][x], t1 = sym.lead_f[1] * sym.lead_eig[1][y];
      base[b] = (sym.shift + t0) + t1;
    } else if (MODE == kForwardDivideInverse) {
      // base = shift + sum_{i<N-1} f_i lambda_i (poisson.cpp:586-590 order)
      long long rem = l < ls.nlines ? l : 0;
      double terms[kMaxDim];
#pragma unroll
      for (int i = kMaxDim - 1; i >= 0; --i) {
        terms[i] = 0.0;
        if (i < sym.nlead) {
          const long long a = rem % sym.lead_ext[i];
          rem /= sym.lead_ext[i];
          terms[i] = sym.lead_f[i] * sym.lead_eig[i][a];
        }
      }
      double s = sym.shift;
#pragma unroll
      for (int i = 0; i < kMaxDim; ++i)
        if (i < sym.nlead) s += terms[i];
      base[b] = s;
    }
  }
  __syncthreads();

  // tile load, all copies in flight at once (phantom lines zero-filled)
  const long long ps = ls.ps;
  const bool vec = vec_tile<C>(off, Bv, ps, ls.src, ls.dst);
  // rows as bulk copies: 16-byte aligned rows with room for the even length
  __shared__ unsigned long long rowbar;
  bool bulk = false;
  if constexpr (C::BULK) {
    bulk = ((reinterpret_cast<unsigned long long>(ls.src) | reinterpret_cast<unsigned long long>(ls.dst)) & 15) == 0 &&
           ((ls.os1 | ls.os2 | ls.is) & 1) == 0 && (ls.nlines == 1 || C::LB <= (ls.ninner > 1 ? ls.is : ls.os1));
  }
  if (bulk) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mid_smem_u32(&rowbar)), "r"(1) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mid_smem_u32(&rowbar)),
                   "r"(static_cast<unsigned>(Bv * C::LB * sizeof(double)))
                   : "memory");
    }
    __syncthreads();
    if (threadIdx.x < Bv)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       mid_smem_u32(R + C::ix(0, threadIdx.x))),
                   "l"(ls.src + off[threadIdx.x]), "r"(static_cast<unsigned>(C::LB * sizeof(double))),
                   "r"(mid_smem_u32(&rowbar))
                   : "memory");
    for (int it = threadIdx.x; it < (B - Bv) * C::LP; it += TH) R[Bv * C::LP + it] = 0.0;  // phantom rows
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(mid_smem_u32(&rowbar)),
        "r"(0)
        : "memory");
  } else if (ROWS) {
    // row by row: the inner loop is one add per element (a flat index costs a
    // division and an offset lookup per 8-byte copy)
#pragma unroll 1
    for (int b = 0; b < B; ++b) {
      const double* src = ls.src + off[b];
      double* dstrow = R + C::ix(0, b);
      const bool ok = b < Bv;
      if (C::PAD) {
        for (int pos = threadIdx.x; pos < L; pos += TH) cp_async8(R + C::ix(pos, b), src + pos, ok);
      } else {
#pragma unroll 4
        for (int pos = threadIdx.x; pos < L; pos += TH) cp_async8(dstrow + pos, src + pos, ok);
      }
    }
  } else if (vec) {
    constexpr int B2 = B / 2;
    const double* src = ls.src + off[0];
    for (int it = threadIdx.x; it < L * B2; it += TH) {
      const int pos = it / B2, b2 = it - pos * B2;
      cp_async16(R + 2 * it, src + pos * ps + 2 * b2);
    }
  } else {
    for (int it = threadIdx.x; it < L * B; it += TH) {
      const int pos = it / B, b = it % B;
      cp_async8(R + C::ix(pos, b), ls.src + off[b] + pos * ps, b < Bv);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  SFEM_PT(1);

  if (MODE != kInverse) {
    forward_fft_inplace<C>(R, PS, t.tw, t.om);
    centre_reduce<C>(PS, C0);  // PS / C0 are outside the region
    forward_post<C>(reinterpret_cast<const double2*>(R), R, t.mk);
  }
  SFEM_PT(2);
  mix<C, MODE>(R, R, C0, mixF, e0F, SFEM_MID_KMIX ? t.mixT_i : t.mix_inv, t.e0_inv, base, t.eig, sym.f_last, t.eigT);
  SFEM_PT(3);
  if (MODE != kForward) {
    inverse_fft_inplace<C>(R, t.tw, t.mkh, t.om);
    inverse_post<C>(reinterpret_cast<const double2*>(R), R, C0);
  }
  SFEM_PT(4);

  if (bulk) {
    if (C::LB > L && threadIdx.x < B) R[C::ix(L, threadIdx.x)] = 0.0;  // the row's pad element
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x < Bv) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(ls.dst + off[threadIdx.x]),
                   "r"(mid_smem_u32(R + C::ix(0, threadIdx.x))), "r"(static_cast<unsigned>(C::LB * sizeof(double)))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
  } else if (ROWS) {
#pragma unroll 1
    for (int b = 0; b < Bv; ++b) {
      double* dst = ls.dst + off[b];
      const double* srow = R + C::ix(0, b);
      if (C::PAD) {
        for (int pos = threadIdx.x; pos < L; pos += TH) dst[pos] = R[C::ix(pos, b)];
      } else {
#pragma unroll 4
        for (int pos = threadIdx.x; pos < L; pos += TH) dst[pos] = srow[pos];
      }
    }
  } else if (vec) {
    constexpr int B2 = B / 2;
    double* dst = ls.dst + off[0];
    for (int it = threadIdx.x; it < L * B2; it += TH) {
      const int pos = it / B2, b2 = it - pos * B2;
      *reinterpret_cast<double2*>(dst + pos * ps + 2 * b2) = *reinterpret_cast<const double2*>(R + 2 * it);
    }
  } else {
    for (int it = threadIdx.x; it < L * B; it += TH) {
      const int pos = it / B, b = it % B;
      if (b < Bv) ls.dst[off[b] + pos * ps] = R[C::ix(pos, b)];
    }
  }
  SFEM_PT(5);
  SFEM_PT_FLUSH(20 + MODE);
}


// ---------------------------------------------------------------------------
// Strided sweeps with the tile moved by TMA (same stages as sweep_mid, same
// dense tile layout T[pos][b]): the tensor is viewed as 4-D {last axis, swept
// axis, outer axes} (TmaGeom, sweep.cuh); a tile is BB consecutive last-axis
// indices x all positions at one (c2, c3), brought in by nbox box copies
// {BB, boxp} issued by one thread and signalled on an mbarrier, and written
// back by nbox tensor stores.  Lines / positions outside the tensor are
// zero-filled on load and clipped on store by the TMA unit, so partial tiles
// need no per-line bookkeeping.  Replaces 2 x L*BB/2 16-byte cp.async / store
// instructions per tile (a quarter of the kernel's instructions at C5 n = 4).
// ---------------------------------------------------------------------------
template <int NN, int K, int BB, int TH>
struct TmaShape {
  using C = Cfg<NN, K, BB, TH, false>;
  static constexpr int NBOX = (C::L + 255) / 256;
  // every box starts 128-byte aligned in shared memory: BOXP * BB a multiple of 16 doubles
  static constexpr int BALIGN = BB % 16 == 0 ? 1 : (BB % 8 == 0 ? 2 : (BB % 4 == 0 ? 4 : (BB % 2 == 0 ? 8 : 16)));
  static constexpr int BOXP = ((C::L + NBOX - 1) / NBOX + BALIGN - 1) / BALIGN * BALIGN;
  // the boxes' zero-filled tail rows must fit the region; 16-byte box rows at least
  static constexpr bool OK = NBOX * BOXP * BB <= C::REGION && (BB * 8) % 16 == 0;
  // the mbarrier lives behind the regular layout
  static constexpr int BAR_OFF = (C::TOTAL + 1) & ~1;
  static constexpr size_t SMEM = static_cast<size_t>(BAR_OFF + 2) * sizeof(double);
};

template <int NN, int K, int BB, int TH, int MODE>
__global__ void __launch_bounds__(TH, mid_min_blocks_n(NN, TH))
    sweep_mid_tma(DevTable t, const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap smap,
                  TmaGeom geo, const double* __restrict__ mixF, const double* __restrict__ e0F) {
  using C = Cfg<NN, K, BB, TH, false>;
  using TS = TmaShape<NN, K, BB, TH>;
  extern __shared__ __align__(128) double smem[];  // no static shared memory: the tile starts 128-byte aligned
  double* R = smem;
  double* C0 = smem + C::C0_OFF;
  double* PS = smem + C::PS_OFF;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + TS::BAR_OFF);
  SFEM_PT_DECL;
  SFEM_PT(0);
  int c0, c2, c3;
  if (gridDim.y > 1 || gridDim.z > 1 || geo.ntiles == geo.nblk0) {
    c0 = static_cast<int>(blockIdx.x) * BB;
    c2 = static_cast<int>(blockIdx.y);
    c3 = static_cast<int>(blockIdx.z);
  } else {
    const long long tile = blockIdx.x;
    c0 = static_cast<int>(tile % geo.nblk0) * BB;
    const long long rest = tile / geo.nblk0;
    c2 = static_cast<int>(rest % geo.ext2);
    c3 = static_cast<int>(rest / geo.ext2);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mid_smem_u32(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    // bytes of the tile's boxes; the one box of a blocked swept axis brings xblk * ceil(L / xblk) rows
    const unsigned tile_bytes =
        geo.ld_mode == kBoxSwept
            ? static_cast<unsigned>((C::L + geo.xblk - 1) / geo.xblk * geo.xblk * BB * sizeof(double))
            : static_cast<unsigned>(TS::NBOX * TS::BOXP * BB * sizeof(double));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mid_smem_u32(bar)), "r"(tile_bytes)
                 : "memory");
    // box coordinates (sweep.cuh BoxMode): plain {c0, j*boxp, c2, c3}; swept axis stored blocked: one box
    // {BB, xblk, nhi, 1} at {c0, 0, 0, c2}; the tile's fixed coordinate blocked: {c0, j*boxp, c2 % xblk, c2 / xblk}
    if (geo.ld_mode == kBoxSwept) {
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
          "[%6];\n" ::"r"(mid_smem_u32(R)),
          "l"(&tmap), "r"(c0), "r"(0), "r"(0), "r"(c2), "r"(mid_smem_u32(bar))
          : "memory");
    } else {
      const int k2 = geo.ld_mode == kBoxSplit ? c2 % geo.xblk : c2, k3 = geo.ld_mode == kBoxSplit ? c2 / geo.xblk : c3;
#pragma unroll 1
      for (int j = 0; j < TS::NBOX; ++j)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
            "[%6];\n" ::"r"(mid_smem_u32(R + j * TS::BOXP * BB)),
            "l"(&tmap), "r"(c0), "r"(j * TS::BOXP), "r"(k2), "r"(k3), "r"(mid_smem_u32(bar))
            : "memory");
    }
    if (geo.prefetch > 0 && geo.ld_mode == kBoxPlain) {
      // L2 prefetch of the tile the next CTA on this SM will load (one resident
      // wave ahead).  Only for sweeps whose positions are a few KB apart: C5
      // n=4 axis-1 sweeps -6 %, but +22 % along axis 0, whose rows are planes
      // apart (profiles/r3z4_mid_tma_prefetch.txt), so the host turns it on per sweep.
      const long long lin = (static_cast<long long>(c3) * geo.ext2 + c2) * geo.nblk0 + c0 / BB;
      const long long nxt = lin + geo.prefetch;
      if (nxt < geo.ntiles) {
        const int p0 = static_cast<int>(nxt % geo.nblk0) * BB;
        const long long rest = nxt / geo.nblk0;
        const int p2 = static_cast<int>(rest % geo.ext2), p3 = static_cast<int>(rest / geo.ext2);
#pragma unroll 1
        for (int j = 0; j < TS::NBOX; ++j)
          asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];\n" ::"l"(&tmap), "r"(p0),
                       "r"(j * TS::BOXP), "r"(p2), "r"(p3)
                       : "memory");
      }
    }
  }
  __syncthreads();  // the barrier is initialised before anyone polls it
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(mid_smem_u32(bar)),
      "r"(0)
      : "memory");
  SFEM_PT(1);
  SymbolInfo nosym{};
  if (MODE != kInverse) {
    forward_fft_inplace<C>(R, PS, t.tw, t.om);
    centre_reduce<C>(PS, C0);
    forward_post<C>(reinterpret_cast<const double2*>(R), R, t.mk);
  }
  SFEM_PT(2);
  mix<C, MODE>(R, R, C0, mixF, e0F, SFEM_MID_KMIX ? t.mixT_i : t.mix_inv, t.e0_inv, nullptr, t.eig, nosym.f_last);
  SFEM_PT(3);
  if (MODE != kForward) {
    inverse_fft_inplace<C>(R, t.tw, t.mkh, t.om);
    inverse_post<C>(reinterpret_cast<const double2*>(R), R, C0);
  }
  SFEM_PT(4);
  // every stage above ends with a block barrier; make the generic-proxy
  // writes of the tile visible to the async proxy before the tensor stores
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    if (geo.st_mode == kBoxSwept) {
      asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n" ::"l"(&smap),
                   "r"(c0), "r"(0), "r"(0), "r"(c2), "r"(mid_smem_u32(R))
                   : "memory");
    } else {
      const int k2 = geo.st_mode == kBoxSplit ? c2 % geo.xblk : c2, k3 = geo.st_mode == kBoxSplit ? c2 / geo.xblk : c3;
#pragma unroll 1
      for (int j = 0; j < TS::NBOX; ++j)
        asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n" ::"l"(&smap),
                     "r"(c0), "r"(j * TS::BOXP), "r"(k2), "r"(k3), "r"(mid_smem_u32(R + j * TS::BOXP * BB))
                     : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
  }
  SFEM_PT(5);
  SFEM_PT_FLUSH(30 + MODE);
}

template <int NN, int K, int BB, int TH>
cudaError_t launch_tma(const DevTable& t, const void* tmap, const TmaGeom& geo, int mode, int analysis,
                       cudaStream_t stream, const void* smap_in = nullptr) {
  using TS = TmaShape<NN, K, BB, TH>;
  if constexpr (!TS::OK) {
    return cudaErrorNotSupported;
  } else {
    if (mode == kForwardDivideInverse || geo.nbox != TS::NBOX || geo.boxp != TS::BOXP) return cudaErrorInvalidValue;
    using C = Cfg<NN, K, BB, TH, false>;
    if ((geo.ld_mode == kBoxSwept || geo.st_mode == kBoxSwept) &&
        (geo.xblk <= 0 || (C::L + geo.xblk - 1) / geo.xblk * geo.xblk * BB > C::REGION))
      return cudaErrorInvalidValue;
    const double* mixF = SFEM_MID_KMIX ? (analysis == kDirect ? t.mixT_d : t.mixT_w)
                                       : (analysis == kDirect ? t.mix_fwd_d : t.mix_fwd_w);
    const double* e0F = analysis == kDirect ? t.e0_fwd_d : t.e0_fwd_w;
    const CUtensorMap* map = static_cast<const CUtensorMap*>(tmap);
    const CUtensorMap* smap = smap_in ? static_cast<const CUtensorMap*>(smap_in) : map;  // in place: one map
    const long long ext3 = geo.ntiles / (geo.nblk0 * geo.ext2);
    const bool grid3 = geo.nblk0 < (1LL << 31) && geo.ext2 <= 65535 && ext3 <= 65535;
    const dim3 grid = grid3 ? dim3(static_cast<unsigned>(geo.nblk0), static_cast<unsigned>(geo.ext2),
                                   static_cast<unsigned>(ext3))
                            : dim3(static_cast<unsigned>(geo.ntiles));
    cudaError_t err;
    if (mode == kForward) {
      auto kern = sweep_mid_tma<NN, K, BB, TH, kForward>;
      err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(TS::SMEM));
      if (err != cudaSuccess) return err;
      kern<<<grid, TH, TS::SMEM, stream>>>(t, *map, *smap, geo, mixF, e0F);
    } else {
      auto kern = sweep_mid_tma<NN, K, BB, TH, kInverse>;
      err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(TS::SMEM));
      if (err != cudaSuccess) return err;
      kern<<<grid, TH, TS::SMEM, stream>>>(t, *map, *smap, geo, mixF, e0F);
    }
    return cudaGetLastError();
  }
}

// Component-major tiles (Cfg::CM) by 5-D tensor copies.  The tensor is viewed
// as {last axis, e >> 1, e & 1, s, outer axis} for position e * n + s of the
// swept axis, so one box {8, K/2, 2, n-1, 1} lands as the planes [s][e & 1] of
// components s < n-1; the last component's planes (the line has no position
// n K - 1) come by two boxes {8, K/2, 1, 1, 1}: even elements through mapB,
// odd ones through mapC, whose tensor ends one element early so the TMA unit
// clips the missing position (zero-filled on load, skipped on store).
template <int NN, int K, int BB, int TH>
struct TmaShapeCM {
  using C = Cfg<NN, K, BB, TH, false, false, true>;
  static constexpr bool OK = BB == 8 && NN >= 2 && K / 2 <= 256 && NN * K * BB <= C::REGION;
  static constexpr int PLANE = (K / 2) * BB;  // doubles per [s][e & 1] plane
  static constexpr int BAR_OFF = (C::TOTAL + 1) & ~1;
  static constexpr size_t SMEM = static_cast<size_t>(BAR_OFF + 2) * sizeof(double);
};

template <int NN, int K, int BB, int TH, int MODE>
__global__ void __launch_bounds__(TH, mid_min_blocks_n(NN, TH))
    sweep_mid_tma_cm(DevTable t, const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     const __grid_constant__ CUtensorMap mapC, TmaGeom geo, const double* __restrict__ mixF,
                     const double* __restrict__ e0F) {
  using C = Cfg<NN, K, BB, TH, false, false, true>;
  using TS = TmaShapeCM<NN, K, BB, TH>;
  extern __shared__ __align__(128) double smem[];
  double* R = smem;
  double* C0 = smem + C::C0_OFF;
  double* PS = smem + C::PS_OFF;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + TS::BAR_OFF);
  SFEM_PT_DECL;
  SFEM_PT(0);
  int c0, c2;
  if (gridDim.y > 1 || geo.ntiles == geo.nblk0) {
    c0 = static_cast<int>(blockIdx.x) * BB;
    c2 = static_cast<int>(blockIdx.y);
  } else {
    const long long tile = blockIdx.x;
    c0 = static_cast<int>(tile % geo.nblk0) * BB;
    c2 = static_cast<int>(tile / geo.nblk0);
  }
  double* RB = R + (NN - 1) * 2 * TS::PLANE;  // planes of the last component
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mid_smem_u32(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mid_smem_u32(bar)),
                 "r"(static_cast<unsigned>(NN * 2 * TS::PLANE * sizeof(double)))
                 : "memory");
    if (NN > 1)
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
          "%6}], [%7];\n" ::"r"(mid_smem_u32(R)),
          "l"(&mapA), "r"(c0), "r"(0), "r"(0), "r"(0), "r"(c2), "r"(mid_smem_u32(bar))
          : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];\n" ::"r"(mid_smem_u32(RB)),
        "l"(&mapB), "r"(c0), "r"(0), "r"(0), "r"(NN - 1), "r"(c2), "r"(mid_smem_u32(bar))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];\n" ::"r"(mid_smem_u32(RB + TS::PLANE)),
        "l"(&mapC), "r"(c0), "r"(0), "r"(0), "r"(0), "r"(c2), "r"(mid_smem_u32(bar))
        : "memory");
    if (geo.prefetch > 0) {
      const long long lin = static_cast<long long>(c2) * geo.nblk0 + c0 / BB;
      const long long nxt = lin + geo.prefetch;
      if (nxt < geo.ntiles) {
        const int p0 = static_cast<int>(nxt % geo.nblk0) * BB, p2 = static_cast<int>(nxt / geo.nblk0);
        if (NN > 1)
          asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global [%0, {%1, %2, %3, %4, %5}];\n" ::"l"(&mapA), "r"(p0),
                       "r"(0), "r"(0), "r"(0), "r"(p2)
                       : "memory");
        asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global [%0, {%1, %2, %3, %4, %5}];\n" ::"l"(&mapB), "r"(p0),
                     "r"(0), "r"(0), "r"(NN - 1), "r"(p2)
                     : "memory");
        asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global [%0, {%1, %2, %3, %4, %5}];\n" ::"l"(&mapC), "r"(p0),
                     "r"(0), "r"(0), "r"(0), "r"(p2)
                     : "memory");
      }
    }
  }
  __syncthreads();  // the barrier is initialised before anyone polls it
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(mid_smem_u32(bar)),
      "r"(0)
      : "memory");
  SFEM_PT(1);
  SymbolInfo nosym{};
  if (MODE != kInverse) {
    forward_fft_inplace<C>(R, PS, t.tw, t.om);
    centre_reduce<C>(PS, C0);
    forward_post<C>(reinterpret_cast<const double2*>(R), R, t.mk);
  }
  SFEM_PT(2);
  mix<C, MODE>(R, R, C0, mixF, e0F, SFEM_MID_KMIX ? t.mixT_i : t.mix_inv, t.e0_inv, nullptr, t.eig, nosym.f_last);
  SFEM_PT(3);
  if (MODE != kForward) {
    inverse_fft_inplace<C>(R, t.tw, t.mkh, t.om);
    inverse_post<C>(reinterpret_cast<const double2*>(R), R, C0);
  }
  SFEM_PT(4);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    if (NN > 1)
      asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n" ::"l"(&mapA),
                   "r"(c0), "r"(0), "r"(0), "r"(0), "r"(c2), "r"(mid_smem_u32(R))
                   : "memory");
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n" ::"l"(&mapB),
                 "r"(c0), "r"(0), "r"(0), "r"(NN - 1), "r"(c2), "r"(mid_smem_u32(RB))
                 : "memory");
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n" ::"l"(&mapC),
                 "r"(c0), "r"(0), "r"(0), "r"(0), "r"(c2), "r"(mid_smem_u32(RB + TS::PLANE))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
  }
  SFEM_PT(5);
  SFEM_PT_FLUSH(30 + MODE);
}

// maps[0..2] = mapA, mapB, mapC (64-byte aligned CUtensorMaps)
template <int NN, int K, int BB, int TH>
cudaError_t launch_tma_cm(const DevTable& t, const void* maps, const TmaGeom& geo, int mode, int analysis,
                          cudaStream_t stream) {
  using TS = TmaShapeCM<NN, K, BB, TH>;
  if constexpr (!TS::OK) {
    return cudaErrorNotSupported;
  } else {
    if (mode == kForwardDivideInverse) return cudaErrorInvalidValue;
    const double* mixF = SFEM_MID_KMIX ? (analysis == kDirect ? t.mixT_d : t.mixT_w)
                                       : (analysis == kDirect ? t.mix_fwd_d : t.mix_fwd_w);
    const double* e0F = analysis == kDirect ? t.e0_fwd_d : t.e0_fwd_w;
    const CUtensorMap* map = static_cast<const CUtensorMap*>(maps);
    const long long rest = geo.ntiles / geo.nblk0;
    const bool grid2 = geo.nblk0 < (1LL << 31) && rest <= 65535;
    const dim3 grid = grid2 ? dim3(static_cast<unsigned>(geo.nblk0), static_cast<unsigned>(rest))
                            : dim3(static_cast<unsigned>(geo.ntiles));
    cudaError_t err;
    if (mode == kForward) {
      auto kern = sweep_mid_tma_cm<NN, K, BB, TH, kForward>;
      err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(TS::SMEM));
      if (err != cudaSuccess) return err;
      kern<<<grid, TH, TS::SMEM, stream>>>(t, map[0], map[1], map[2], geo, mixF, e0F);
    } else {
      auto kern = sweep_mid_tma_cm<NN, K, BB, TH, kInverse>;
      err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(TS::SMEM));
      if (err != cudaSuccess) return err;
      kern<<<grid, TH, TS::SMEM, stream>>>(t, map[0], map[1], map[2], geo, mixF, e0F);
    }
    return cudaGetLastError();
  }
}

// Lines too long for an FFT buffer in shared memory (C2: n=4, K=4096): the
// tile stays in shared memory, the J*K complex FFT work of the CTA lives in
// two slices of a global scratch array (L2-resident while the CTA runs; the
// slices are discarded from L2 at exit, so they never reach HBM).
template <int NN, int K, int BB, int TH, int MODE, bool ROWS>
__global__ void __launch_bounds__(TH, 1)
    sweep_mid_gw(DevTable t, LineSet ls, SymbolInfo sym, const double* __restrict__ mixF,
                 const double* __restrict__ e0F, double* gwork) {
  using C = Cfg<NN, K, BB, TH, ROWS, true>;
  constexpr int B = C::B, L = C::L, JK = C::J * C::N;
  extern __shared__ __align__(16) double smem[];
  double* R = smem;  // tile and slots (REGION >= TD)
  double* C0 = smem + C::C0_OFF;
  double* PS = smem + C::PS_OFF;
  double* base = smem + C::BASE_OFF;
  __shared__ long long off[B];
  double2* W0 = reinterpret_cast<double2*>(gwork) + static_cast<size_t>(blockIdx.x) * 2 * JK;
  double2* W1 = W0 + JK;

  const long long l0 = static_cast<long long>(blockIdx.x) * B;
  const int Bv = static_cast<int>(min(static_cast<long long>(B), ls.nlines - l0));
  if (threadIdx.x < B) {
    const int b = threadIdx.x;
    const long long l = l0 + b;
    const long long r = l / ls.ninner;
    off[b] = l < ls.nlines ? (r / ls.n1) * ls.os2 + (r % ls.n1) * ls.os1 + (l % ls.ninner) * ls.is : 0;
    if (MODE == kForwardDivideInverse) {
      long long rem = l < ls.nlines ? l : 0;
      double terms[kMaxDim];
#pragma unroll
      for (int i = kMaxDim - 1; i >= 0; --i) {
        terms[i] = 0.0;
        if (i < sym.nlead) {
          const long long a = rem % sym.lead_ext[i];
          rem /= sym.lead_ext[i];
          terms[i] = sym.lead_f[i] * sym.lead_eig[i][a];
        }
      }
      double sb = sym.shift;
#pragma unroll
      for (int i = 0; i < kMaxDim; ++i)
        if (i < sym.nlead) sb += terms[i];
      base[b] = sb;
    }
  }
  __syncthreads();
  const long long ps = ls.ps;
  if (ROWS) {
    for (int it = threadIdx.x; it < L * B; it += TH) {
      const int b = it / L, pos = it - b * L;
      cp_async8(R + C::ix(pos, b), ls.src + off[b] + pos, b < Bv);
    }
  } else {
    for (int it = threadIdx.x; it < L * B; it += TH) {
      const int pos = it / B, b = it % B;
      cp_async8(R + it, ls.src + off[b] + pos * ps, b < Bv);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  const double2* Zf = W0;
  if (MODE != kInverse) {
    forward_fill<C, true>(R, reinterpret_cast<double*>(W0), PS, t.om);
    Zf = fft_oop<C>(W0, W1, t.tw);
    centre_reduce<C>(PS, C0);
    forward_post<C, true>(Zf, R, t.mk);
  }
  mix<C, MODE>(R, R, C0, mixF, e0F, SFEM_MID_KMIX ? t.mixT_i : t.mix_inv, t.e0_inv, base, t.eig, sym.f_last, t.eigT);
  if (MODE != kForward) {
#if SFEM_MID_GW_DISCARD
    if (MODE == kForwardDivideInverse) {  // the forward result is dead (mix ended with a barrier)
      discard_l2<C>(Zf);
      __syncthreads();
    }
#endif
    inverse_fill<C, true>(R, W0, t.mkh, t.om);
    const double2* Z = fft_oop<C>(W0, W1, t.tw);
    inverse_post<C, true>(Z, R, C0);
  }
  if (ROWS) {
    for (int it = threadIdx.x; it < L * B; it += TH) {
      const int b = it / L, pos = it - b * L;
      if (b < Bv) ls.dst[off[b] + pos] = R[C::ix(pos, b)];
    }
  } else {
    for (int it = threadIdx.x; it < L * B; it += TH) {
      const int pos = it / B, b = it % B;
      if (b < Bv) ls.dst[off[b] + pos * ps] = R[it];
    }
  }
  // the work slices are dead: drop them from L2 without write-back
  char* wb = reinterpret_cast<char*>(W0);
  for (int i = threadIdx.x; i < (2 * JK * 16) / 128; i += TH)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(wb + static_cast<size_t>(i) * 128) : "memory");
}

template <int NN, int K, int BB, int TH>
cudaError_t launch_gw(const DevTable& t, const LineSet& ls, int mode, int analysis, const SymbolInfo* sym,
                      double* gwork, cudaStream_t stream) {
  const double* mixF = SFEM_MID_KMIX ? (analysis == kDirect ? t.mixT_d : t.mixT_w)
                                     : (analysis == kDirect ? t.mix_fwd_d : t.mix_fwd_w);
  const double* e0F = analysis == kDirect ? t.e0_fwd_d : t.e0_fwd_w;
  SymbolInfo s{};
  if (sym) s = *sym;
  const dim3 grid(static_cast<unsigned>((ls.nlines + BB - 1) / BB));
  cudaError_t err = cudaSuccess;
  auto go = [&](auto kern, size_t smem) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (err != cudaSuccess) return;
    kern<<<grid, TH, smem, stream>>>(t, ls, s, mixF, e0F, gwork);
    err = cudaGetLastError();
  };
  // shared memory: the tile only (the FFT buffers are global)
  constexpr size_t SR = Cfg<NN, K, BB, TH, true, true>::SMEM, SS = Cfg<NN, K, BB, TH, false, true>::SMEM;
  if (mode == kForwardDivideInverse) {
    if (!ls.contiguous) return cudaErrorNotSupported;
    go(sweep_mid_gw<NN, K, BB, TH, kForwardDivideInverse, true>, SR);
  } else if (mode == kForward) {
    ls.contiguous ? go(sweep_mid_gw<NN, K, BB, TH, kForward, true>, SR)
                  : go(sweep_mid_gw<NN, K, BB, TH, kForward, false>, SS);
  } else {
    ls.contiguous ? go(sweep_mid_gw<NN, K, BB, TH, kInverse, true>, SR)
                  : go(sweep_mid_gw<NN, K, BB, TH, kInverse, false>, SS);
  }
  return err;
}

template <int NN, int K, int BB, int TH>
cudaError_t launch(const DevTable& t, const LineSet& ls, int mode, int analysis, const SymbolInfo* sym,
                   cudaStream_t stream) {
  const double* mixF = SFEM_MID_KMIX ? (analysis == kDirect ? t.mixT_d : t.mixT_w)
                                     : (analysis == kDirect ? t.mix_fwd_d : t.mix_fwd_w);
  const double* e0F = analysis == kDirect ? t.e0_fwd_d : t.e0_fwd_w;
  SymbolInfo s{};
  if (sym) s = *sym;
  const dim3 grid(static_cast<unsigned>((ls.nlines + BB - 1) / BB));
  cudaError_t err = cudaSuccess;
  auto go = [&](auto kern, size_t smem) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (err != cudaSuccess) return;
    kern<<<grid, TH, smem, stream>>>(t, ls, s, mixF, e0F);
    err = cudaGetLastError();
  };
  using CR = Cfg<NN, K, BB, TH, true>;
  using CS = Cfg<NN, K, BB, TH, false>;
  if (mode == kForwardDivideInverse) {
    if (!ls.contiguous) return cudaErrorNotSupported;
    go(sweep_mid<NN, K, BB, TH, kForwardDivideInverse, true>, CR::SMEM);
  } else if (mode == kForward) {
    ls.contiguous ? go(sweep_mid<NN, K, BB, TH, kForward, true>, CR::SMEM)
                  : go(sweep_mid<NN, K, BB, TH, kForward, false>, CS::SMEM);
  } else {
    ls.contiguous ? go(sweep_mid<NN, K, BB, TH, kInverse, true>, CR::SMEM)
                  : go(sweep_mid<NN, K, BB, TH, kInverse, false>, CS::SMEM);
  }
  return err;
}

// Tile shape for the general (n, K) instantiations: the most lines per tile
// (8, 4, 2) whose shared region fits two 256-thread CTAs per SM, else two
// lines with one 512-thread CTA per SM, else none (generic kernels).
template <int NN, int K>
struct AutoShape {
  template <int BB, int TH>
  static constexpr bool fits(size_t budget) {
    return Cfg<NN, K, BB, TH, true>::SMEM <= budget && Cfg<NN, K, BB, TH, false>::SMEM <= budget;
  }
  static constexpr int B = fits<8, 256>(110 * 1024) ? 8 : fits<4, 256>(110 * 1024) ? 4
                           : fits<2, 256>(110 * 1024) ? 2 : fits<2, 512>(220 * 1024) ? 2 : 0;
  static constexpr int TH = (B == 2 && !fits<2, 256>(110 * 1024)) ? 512 : 256;
};

// (n, K) served elsewhere: the K = 64 register-FFT kernels (sweep_fast.cu)
// and the tuned shapes of launch_sweep_mid below.
template <int NN, int K>
constexpr bool served_elsewhere() {
  return (K == 64 && NN >= 2) || (NN == 2 && K == 512) || (K == 1024 && (NN == 1 || NN == 9)) ||
         (NN == 4 && K == 256);
}

template <int NN, int K>
cudaError_t launch_auto(const DevTable& t, const LineSet& ls, int mode, int analysis, const SymbolInfo* sym,
                        cudaStream_t stream) {
  using S = AutoShape<NN, K>;
  if constexpr (S::B == 0 || served_elsewhere<NN, K>()) {
    return cudaErrorNotSupported;
  } else {
    return launch<NN, K, S::B, S::TH>(t, ls, mode, analysis, sym, stream);
  }
}

template <int K>
cudaError_t launch_auto_n(const DevTable& t, const LineSet& ls, int mode, int analysis, const SymbolInfo* sym,
                          cudaStream_t stream) {
  switch (t.n) {
    case 1: return launch_auto<1, K>(t, ls, mode, analysis, sym, stream);
    case 2: return launch_auto<2, K>(t, ls, mode, analysis, sym, stream);
    case 3: return launch_auto<3, K>(t, ls, mode, analysis, sym, stream);
    case 4: return launch_auto<4, K>(t, ls, mode, analysis, sym, stream);
    case 5: return launch_auto<5, K>(t, ls, mode, analysis, sym, stream);
    case 6: return launch_auto<6, K>(t, ls, mode, analysis, sym, stream);
    case 7: return launch_auto<7, K>(t, ls, mode, analysis, sym, stream);
    case 8: return launch_auto<8, K>(t, ls, mode, analysis, sym, stream);
    case 9: return launch_auto<9, K>(t, ls, mode, analysis, sym, stream);
    default: return cudaErrorNotSupported;
  }
}

// General shapes, strided sweeps with TMA tiles (sweep_mid_tma): the same
// tile shape as launch_auto; lines per tile 0 when the shape has no TMA kernel.
template <int NN, int K>
constexpr int auto_tma_lines() {
  using S = AutoShape<NN, K>;
  if constexpr (S::B < 2 || served_elsewhere<NN, K>()) {
    return 0;
  } else {
    return TmaShape<NN, K, S::B, S::TH>::OK ? S::B : 0;
  }
}

template <int NN, int K>
cudaError_t launch_auto_tma(const DevTable& t, const void* tmap, const TmaGeom& geo, int mode, int analysis,
                            cudaStream_t stream) {
  if constexpr (auto_tma_lines<NN, K>() == 0) {
    return cudaErrorNotSupported;
  } else {
    using S = AutoShape<NN, K>;
    return launch_tma<NN, K, S::B, S::TH>(t, tmap, geo, mode, analysis, stream);
  }
}

template <int K>
cudaError_t launch_auto_tma_n(const DevTable& t, const void* tmap, const TmaGeom& geo, int mode, int analysis,
                              cudaStream_t stream) {
  switch (t.n) {
    case 1: return launch_auto_tma<1, K>(t, tmap, geo, mode, analysis, stream);
    case 2: return launch_auto_tma<2, K>(t, tmap, geo, mode, analysis, stream);
    case 3: return launch_auto_tma<3, K>(t, tmap, geo, mode, analysis, stream);
    case 4: return launch_auto_tma<4, K>(t, tmap, geo, mode, analysis, stream);
    case 5: return launch_auto_tma<5, K>(t, tmap, geo, mode, analysis, stream);
    case 6: return launch_auto_tma<6, K>(t, tmap, geo, mode, analysis, stream);
    case 7: return launch_auto_tma<7, K>(t, tmap, geo, mode, analysis, stream);
    case 8: return launch_auto_tma<8, K>(t, tmap, geo, mode, analysis, stream);
    case 9: return launch_auto_tma<9, K>(t, tmap, geo, mode, analysis, stream);
    default: return cudaErrorNotSupported;
  }
}

template <int K>
int auto_tma_lines_n(int n) {
  switch (n) {
    case 1: return auto_tma_lines<1, K>();
    case 2: return auto_tma_lines<2, K>();
    case 3: return auto_tma_lines<3, K>();
    case 4: return auto_tma_lines<4, K>();
    case 5: return auto_tma_lines<5, K>();
    case 6: return auto_tma_lines<6, K>();
    case 7: return auto_tma_lines<7, K>();
    case 8: return auto_tma_lines<8, K>();
    case 9: return auto_tma_lines<9, K>();
    default: return 0;
  }
}

// General shapes with component-major strided tiles (Cfg::CM): eight-line tiles of the orders 2 and 4 whose
// planes fit the TMA box (K / 2 <= 256): 3-D n=2 K=128 / 256 -6.6 / -5.2 %, n=4 K=128 / 100 -3.8 / -3.6 %, bitwise
// identical; n = 8 measured neutral to +1.8 % and left on the dense tiles (profiles/r5d_mid_cm_general_shapes.txt).
template <int NN, int K>
constexpr bool auto_tma_cm() {
  if constexpr (auto_tma_lines<NN, K>() != 8 || (NN != 2 && NN != 4) || K % 2 != 0) {
    return false;
  } else {
    return TmaShapeCM<NN, K, 8, AutoShape<NN, K>::TH>::OK;
  }
}

template <int NN, int K>
cudaError_t launch_auto_tma_cm(const DevTable& t, const void* maps, const TmaGeom& geo, int mode, int analysis,
                               cudaStream_t stream) {
  if constexpr (!auto_tma_cm<NN, K>()) {
    return cudaErrorNotSupported;
  } else {
    return launch_tma_cm<NN, K, 8, AutoShape<NN, K>::TH>(t, maps, geo, mode, analysis, stream);
  }
}

template <int K>
cudaError_t launch_auto_tma_cm_n(const DevTable& t, const void* maps, const TmaGeom& geo, int mode, int analysis,
                                 cudaStream_t stream) {
  switch (t.n) {
    case 2: return launch_auto_tma_cm<2, K>(t, maps, geo, mode, analysis, stream);
    case 4: return launch_auto_tma_cm<4, K>(t, maps, geo, mode, analysis, stream);
    case 8: return launch_auto_tma_cm<8, K>(t, maps, geo, mode, analysis, stream);
    default: return cudaErrorNotSupported;
  }
}

template <int K>
bool auto_tma_cm_n(int n) {
  switch (n) {
    case 2: return auto_tma_cm<2, K>();
    case 4: return auto_tma_cm<4, K>();
    case 8: return auto_tma_cm<8, K>();
    default: return false;
  }
}

template <int K>
bool auto_ok_n(int n) {
  switch (n) {
    case 1: return AutoShape<1, K>::B > 0;
    case 2: return AutoShape<2, K>::B > 0;
    case 3: return AutoShape<3, K>::B > 0;
    case 4: return AutoShape<4, K>::B > 0;
    case 5: return AutoShape<5, K>::B > 0;
    case 6: return AutoShape<6, K>::B > 0;
    case 7: return AutoShape<7, K>::B > 0;
    case 8: return AutoShape<8, K>::B > 0;
    case 9: return AutoShape<9, K>::B > 0;
    default: return false;
  }
}

}  // namespace mid
}  // namespace sfem_b200
