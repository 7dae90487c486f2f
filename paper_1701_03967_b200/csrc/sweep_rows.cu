// Fused last-axis sweep, K = 64: forward FC_n + symbol divide + inverse F_n
// of 8 rows per CTA (reference forward_axis / scale_by_symbol / inverse_axis
// on the contiguous axis, poisson.cpp:283-291, 573-631, 360-368, with
// lines::decompose_weighted / synthesize, eigenbasis.cpp:63-101, 144-225).
//
// Same arithmetic as sweep_bulk_rows (sweep_fast.cu), laid out
// so that every FFT exchange stays inside one warp:
//   * a job (one complex 64-point FFT: an interior pair (i, m-1-i) of a line,
//     a nodal half of a line pair, or a middle component of a line pair) is
//     four lanes of ONE warp (lane = 4 * slot + tau), eight jobs per warp;
//     lane tau holds residue classes (c, 8-c) in pass 1 and output classes
//     (q, 8-q) in pass 2, so the Makhoul / DST-I pre- and post-processing are
//     lane-local and the pass-1 -> pass-2 transpose is a warp-private
//     shared-memory exchange ordered by __syncwarp, not __syncthreads;
//   * the job's exchange slot (65 complex) also holds the two coefficient-side
//     rows it produces (S rows, 65 doubles each), so the forward
//     post-processing and the inverse pre-processing touch only their own warp's
//     slots;
//   * the per-frequency mixes run per (k, 4-line group) item with the two
//     groups of one k in adjacent lanes (one matrix load serves both), and the
//     forward mix, divide and inverse mix of an item run back to back (the
//     coefficients go through a thread-private scratch row, no barrier);
//   * pair jobs of one warp cover two components (i, i+1) x four lines and the
//     row tile has a pitch of 8 mod 16 doubles: a warp's tile loads and stores
//     hit all 16 bank pairs twice (conflict-free).
// Five block barriers per tile (tile in -> exchange slots, forward S complete,
// mixed S complete, exchange reads done -> output tile, output tile complete),
// against twelve in sweep_bulk_rows.
#include <cuda.h>

#include <type_traits>

#include "fft_reg.cuh"
#include "sweep.cuh"

// Resident CTAs per SM asked of ptxas: 3 (128 registers) for n >= 6; 4 (96
// registers) for n <= 5, whose mix items hold fewer values (measured
// profiles/r2l_rows_ab.txt: n = 2 / 4 / 5 fused sweeps -12 / -6 / -7 %, n = 9
// +75 % from spills).
#ifndef SFEM_ROWS_MINB
#define SFEM_ROWS_MINB(NN) ((NN) <= 5 ? 4 : 3)
#endif

namespace sfem_b200 {
namespace rows {

using namespace reg;

constexpr int N = 64, R = 8, G = 8, B = 8;
// Job slot: 68 complex.  The exchange X[q][c] (8 x 8 complex) is stored at
// q*8 + (c ^ q), and consecutive jobs start 4 bank quads apart (68 = 4 mod 8):
// the eight lanes of a 128-bit access phase (two jobs x four taus) then hit
// eight distinct quads in both the pass-1 stores and the pass-2 loads.  The
// job's two S rows (65 doubles each) start at +0 or +4 doubles (bit 1 of the
// job index), so the 16 lanes of a 64-bit phase (four jobs x four taus) hit 16
// distinct bank pairs in the S-row accesses.
constexpr int XJOB = 136;  // doubles per job slot
constexpr int SR = 65;     // doubles per S row (index k = 1..63 used)
__host__ __device__ constexpr int sbase(int j) { return j * XJOB + 4 * ((j >> 1) & 1); }

template <int V, int A>
constexpr int round_up(int v = V) {
  return (v + A - 1) / A * A;
}

template <int NN>
struct Cfg {
  static constexpr int M = NN - 1, HALF = M / 2, NE = NN / 2, MODD = M & 1;
  static constexpr int L = NN * N - 1;
  static constexpr int NPAIR = B * HALF, NNOD = B, NMID = MODD ? B / 2 : 0;
  static constexpr int NJOB = NPAIR + NNOD + NMID;
  static constexpr int PAIR_WARPS = NPAIR / 8;
  static constexpr int FFT_WARPS = (NJOB + 7) / 8;
  static constexpr int ITEMS = N * 2;  // mix item slots (k = 1..64, 4-line group); k = 64 is idle
  static constexpr int THREADS = (32 * FFT_WARPS > round_up<ITEMS + B, 32>()) ? 32 * FFT_WARPS
                                                                            : round_up<ITEMS + B, 32>();
  static constexpr int P = (L + 1) & ~1;                   // doubles per row copy (16-byte multiple)
  static constexpr int RP = P + ((8 - P) % 16 + 16) % 16;  // row pitch, 8 mod 16 doubles
  static constexpr int TILE_D = B * RP;
  static constexpr int X_D = NJOB * XJOB;
  static constexpr int REGION = round_up<(TILE_D > X_D ? TILE_D : X_D), 16>();
  static constexpr int MB = (M > 0 ? M : 1) * B;
  static constexpr int C0_OFF = REGION;          // 4 per-tau centre partial blocks [tau][i][b]
  static constexpr int CI_OFF = C0_OFF + 4 * MB;  // inverse centre terms [i][b]
  static constexpr int BASE_OFF = CI_OFF + MB;
  static constexpr int BAR_OFF = round_up<BASE_OFF + B, 2>();
  static constexpr int TAB_OFF = BAR_OFF + 2;     // tw | mkh | om, N complex each
  static constexpr int SOFF_OFF = TAB_OFF + 6 * N;  // S-row offsets [g][slot][4 lines] (ints; rolled mixes)
  static constexpr int TOTAL_D = SOFF_OFF + (2 * NN * 4 + 1) / 2 + 2;
  static constexpr size_t SMEM = static_cast<size_t>(TOTAL_D) * sizeof(double);
};

// ---------------------------------------------------------------------------
// Job roles and the S-row placement.
// ---------------------------------------------------------------------------
struct Job {
  int kind;  // 0 pair, 1 nodal, 2 middle, 3 none
  int j;     // job index (slot)
  int i;     // pair: component; middle: HALF
  int b;     // pair: line; nodal / middle: first line of the pair (second = b + 4)
  int which; // nodal: 0 even outputs, 1 odd outputs
  int tau, c1, c2, q1, q2;
};

template <int NN>
__device__ __forceinline__ Job job_of(int tid) {
  using C = Cfg<NN>;
  const int warp = tid >> 5, lane = tid & 31, js = lane >> 2;
  Job o{3, -1, 0, 0, 0, lane & 3, 0, 0, 0, 0};
  const int j = warp * 8 + js;
  if (j < C::NPAIR) {
    o.kind = 0;
    o.j = j;
    if constexpr (C::HALF % 2 == 0) {
      // warp: components (i0, i0 + 1) x four lines (conflict-free tile access)
      constexpr int HP = C::HALF / 2 > 0 ? C::HALF / 2 : 1;
      o.i = 2 * (warp % HP) + (js & 1);
      o.b = 4 * (warp / HP) + (js >> 1);
    } else {
      o.i = j / B;
      o.b = j % B;
    }
  } else if (j < C::NPAIR + C::NNOD) {
    o.kind = 1;
    o.j = j;
    o.which = (j - C::NPAIR) >> 2;
    o.b = (j - C::NPAIR) & 3;
  } else if (j < C::NJOB) {
    o.kind = 2;
    o.j = j;
    o.i = C::HALF;
    o.b = j - C::NPAIR - C::NNOD;
  }
  o.c1 = o.tau;
  o.c2 = o.tau == 0 ? G / 2 : G - o.tau;
  o.q1 = o.tau;
  o.q2 = (o.kind == 1 && o.which == 1) ? R - 1 - o.tau : (o.tau == 0 ? R / 2 : R - o.tau);
  return o;
}

// Job index of pair (i, b) (inverse of job_of for pair jobs).
template <int NN>
__device__ __forceinline__ int pair_job(int i, int b) {
  using C = Cfg<NN>;
  if constexpr (C::HALF % 2 == 0) {
    constexpr int HP = C::HALF / 2 > 0 ? C::HALF / 2 : 1;
    const int warp = (b >> 2) * HP + (i >> 1);
    return warp * 8 + ((b & 3) << 1) + (i & 1);
  } else {
    return i * B + b;
  }
}

// Offset (doubles, from the region start) of S row (slot s, line b).
// Slots: 0 nodal, 1..HALF even parts of pairs, 1+HALF middle (m odd),
// 1+NE.. odd parts of pairs (the reference's fold order, eigenbasis.cpp:46-59).
template <int NN>
__device__ __forceinline__ int srow(int s, int b) {
  using C = Cfg<NN>;
  if (s == 0) return sbase(C::NPAIR + b);  // nodal job (which = b >> 2, line pair b & 3)
  if (C::MODD && s == 1 + C::HALF) return sbase(C::NPAIR + C::NNOD + (b & 3)) + (b >> 2) * SR;
  if (s <= C::HALF) return sbase(pair_job<NN>(s - 1, b));
  return sbase(pair_job<NN>(s - 1 - C::NE, b)) + SR;
}

// Partner value of output class member (h, P): pairing (q, R-q) with tau = 0
// -> (0, R/2): partner of k is N-k; pairing (q, R-1-q) (odd-frequency DST-I
// half): partner of k' is N-1-k'.
template <int P>
__device__ __forceinline__ double2 partner(const double2 (&w1)[G], const double2 (&w2)[G], int tau, int h,
                                           bool shifted) {
  if (shifted || tau != 0) return h == 0 ? w2[G - 1 - P] : w1[G - 1 - P];
  return h == 0 ? w1[(G - P) % G] : w2[G - 1 - P];
}

template <int NN_, int I = 0>
struct Unroll {
  template <class F>
  __device__ __forceinline__ static void run(F&& f) {
    if constexpr (I < NN_) {
      f(std::integral_constant<int, I>{});
      Unroll<NN_, I + 1>::run(f);
    }
  }
};

// Read-only load that the compiler may neither merge with an identical
// earlier load nor hoist: the forward and inverse mixes read the same matrix
// entries, and keeping the forward loads live for the inverse costs 2 x n^2
// registers.
__device__ __forceinline__ double ldg_once(const double* p) {
#ifdef SFEM_ROWS_LDG_PLAIN
  return __ldg(p);
#else
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#endif
}
#ifdef SFEM_ROWS_NOFENCE
#define SFEM_ROWS_FENCE()
#else
#define SFEM_ROWS_FENCE() asm volatile("" ::: "memory")
#endif

// Shared-memory load the compiler may not replace by the value it just
// stored there (the mix parks its coefficients in smem to free registers).
__device__ __forceinline__ double lds_once(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return v;
}

__device__ __forceinline__ int opaque_tid() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}

// c / d (the symbol divide): MUFU reciprocal seed, one Newton step and one
// residual correction of the quotient (sweep_fast.cu sym_div; within 1 ulp of
// the IEEE quotient, tools/div_ulp.cu).
__device__ __forceinline__ double sym_div(double c, double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = fma(r, fma(-d, r, 1.0), r);
  const double q = c * r;
  return fma(fma(-d, q, c), r, q);
}

// ---------------------------------------------------------------------------
// Forward: tile rows -> pass 1 -> warp exchange -> pass 2 -> S rows (+ centre
// partial sums).  T: row tile (row b at T + b*RP); X: region (job slots).
// ---------------------------------------------------------------------------
template <int NN>
__device__ __forceinline__ void forward_job(const Job& jb, const double* T, double* X, double* C0,
                                            const double2* tw, const double2* mkh, const double2* om) {
  using C = Cfg<NN>;
  constexpr int M = C::M, HALF = C::HALF;
  double2* Xj = reinterpret_cast<double2*>(X + (jb.kind < 3 ? jb.j : 0) * XJOB);
  double2 v[2][R];
  double cen_a = 0.0, cen_b = 0.0;
  if (jb.kind == 0 || jb.kind == 2) {
    const double* ra = T + jb.b * C::RP;
    const double* pa = ra + jb.i;
    const double* pb = jb.kind == 0 ? ra + (M - 1 - jb.i) : T + (jb.b + 4) * C::RP + HALF;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = h == 0 ? jb.c1 : jb.c2;
      const double* fa = pa + (2 * c) * NN;
      const double* fb = pb + (2 * c) * NN;
      const double* sa = pa + (N - 1 - 2 * c) * NN;
      const double* sb = pb + (N - 1 - 2 * c) * NN;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool first = r < R / 2;
        const int off = first ? r * (2 * G) * NN : -(r - R / 2) * (2 * G) * NN;
        const double x = (first ? fa : sa)[off];
        const double y = (first ? fb : sb)[off];
        double2 z;
        if (jb.kind == 0) {
          if (first) {
            cen_a += x;
            cen_b += y;
          } else {
            cen_a -= y;
            cen_b -= x;
          }
          const double g = x + y;
          z = make_double2(x - y, first ? g : -g);
        } else {
          z = first ? make_double2(x, y) : make_double2(-x, -y);
          cen_a += z.x;
          cen_b += z.y;
        }
        v[h][r] = z;
      }
    }
  } else if (jb.kind == 1) {
    const double* pa = T + jb.b * C::RP - 1;
    const double* pb = T + (jb.b + 4) * C::RP - 1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = h == 0 ? jb.c1 : jb.c2;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = c + G * r;
        double2 z = make_double2(0.0, 0.0);
        if (t > 0) z = make_double2(pa[t * NN], pb[t * NN]);
        if (jb.which) z = c_mul(z, om[t]);
        v[h][r] = z;
      }
    }
  }
  if (jb.kind == 0) {
    C0[jb.tau * C::MB + jb.i * B + jb.b] = cen_a;
    C0[jb.tau * C::MB + (M - 1 - jb.i) * B + jb.b] = cen_b;
  } else if (jb.kind == 2) {
    C0[jb.tau * C::MB + HALF * B + jb.b] = cen_a;
    C0[jb.tau * C::MB + HALF * B + jb.b + 4] = cen_b;
  }
  __syncthreads();  // (B1) every job's tile reads are done: the slots alias the tile
  if (jb.kind < 3) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = h == 0 ? jb.c1 : jb.c2;
      Dft<R>::run(v[h]);
#pragma unroll
      for (int q = 0; q < R; ++q) Xj[q * G + (c ^ q)] = q == 0 ? v[h][q] : c_mul(v[h][q], tw[(c * q) % N]);
    }
  }
  __syncwarp();
  double2 w1[G], w2[G];
  if (jb.kind < 3) {
#pragma unroll
    for (int c = 0; c < G; ++c) {
      w1[c] = Xj[jb.q1 * G + (c ^ jb.q1)];
      w2[c] = Xj[jb.q2 * G + (c ^ jb.q2)];
    }
  }
  __syncwarp();  // the warp's slots are read: S rows overwrite them
  if (jb.kind == 3) return;
  Dft<G>::run(w1);
  Dft<G>::run(w2);
  if (jb.kind != 1) {
    double* sA = X + sbase(jb.j) + SR;  // pair: H_k row (odd part); middle: line b + 4's row
    double* sB = X + sbase(jb.j);       // pair: G_{N-k} row (even part); middle: line b's row
    if (jb.kind == 2) {
      double* t_ = sA;
      sA = sB;
      sB = t_;
    }
    // r1 = Re(mk_k V1), r2 = Re(mk_k V2), V1 = (Z_k + conj Z_{N-k})/2,
    // V2 = (Z_k - conj Z_{N-k})/(2i); the 1/2 is folded into mkh.  One pass over
    // the (k, N-k) pairs: both outputs share the four sums / differences and a
    // pair's values are dead once emitted (sweep_fast.cu forward_post):
    //   tau != 0: (w1[p], w2[7-p]); tau == 0: class 0 pairs with itself
    //   (w1[p], w1[8-p]) p = 1..3, k = 32 alone; class 4 (w2[p], w2[7-p]) p = 0..3
    auto emit_pair = [&](int k, const double2 zk, const double2 zc, bool both) {
      const double sx = zk.x + zc.x, dy = zk.y - zc.y, sy = zk.y + zc.y, dx = zk.x - zc.x;
      const double2 w = mkh[k];
      const double r1 = fma(w.x, sx, w.y * dy), r2 = fma(w.x, sy, -w.y * dx);
      if (jb.kind == 0) {
        sA[k] = r1;
        sB[N - k] = r2;
      } else {
        sA[N - k] = r1;
        sB[N - k] = r2;
      }
      if (both) {
        // mkh[N-k] = 0.5 exp(i pi/2 - i pi k/2N) = (w.y, w.x): no second table load
        const double2 u = make_double2(w.y, w.x);
        const double t1 = fma(u.x, sx, -u.y * dy), t2 = fma(u.x, sy, u.y * dx);
        if (jb.kind == 0) {
          sA[N - k] = t1;
          sB[k] = t2;
        } else {
          sA[k] = t1;
          sB[k] = t2;
        }
      }
    };
    const bool t0 = jb.tau == 0;
    Unroll<G>::run([&](auto PP) {
      constexpr int p = decltype(PP)::value;
      const double2 y = t0 ? w1[(G - p) % G] : w2[G - 1 - p];
      const bool active = !t0 || (p >= 1 && p <= G / 2);
      if (active) emit_pair(jb.q1 + R * p, w1[p], y, !t0 || p < G / 2);
    });
    if (t0) {
      Unroll<G / 2>::run([&](auto PP) {
        constexpr int p = decltype(PP)::value;
        emit_pair(jb.q2 + R * p, w2[p], w2[G - 1 - p], true);
      });
    }
  } else {
    double* s0a = X + srow<NN>(0, jb.b);
    double* s0b = X + srow<NN>(0, jb.b + 4);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = h == 0 ? jb.q1 : jb.q2;
      Unroll<G>::run([&](auto PP) {
        constexpr int p = decltype(PP)::value;
        const int kp = q + R * p;
        if (jb.which == 0 ? (kp < 1 || kp >= N / 2) : (kp >= N / 2)) return;
        const int kout = 2 * kp + jb.which;
        const double2 zk = h == 0 ? w1[p] : w2[p];
        const double2 zc = partner<p>(w1, w2, jb.tau, h, jb.which == 1);
        // X = (Z_partner - Z_k) / (2i); the 1/2 is folded into the nodal mix column
        s0a[kout] = zc.y - zk.y;
        s0b[kout] = zk.x - zc.x;
      });
    }
  }
}

// ---------------------------------------------------------------------------
// Inverse: S rows (+ centre terms) -> pass 1 -> warp exchange -> pass 2 ->
// row tile.
// ---------------------------------------------------------------------------
template <int NN>
__device__ __forceinline__ void inverse_job(const Job& jb, double* T, double* X, const double* CI,
                                            const double2* tw, const double2* mkh, const double2* om) {
  using C = Cfg<NN>;
  constexpr int M = C::M, HALF = C::HALF;
  double2* Xj = reinterpret_cast<double2*>(X + (jb.kind < 3 ? jb.j : 0) * XJOB);
  double2 v[2][R];
  if (jb.kind == 1) {
    const double* s0a = X + srow<NN>(0, jb.b);
    const double* s0b = X + srow<NN>(0, jb.b + 4);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = h == 0 ? jb.c1 : jb.c2;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = c + G * r;
        double2 z = make_double2(0.0, 0.0);
        if (t > 0) z = make_double2(s0a[t], s0b[t]);
        if (jb.which) z = c_mul(z, om[t]);
        v[h][r] = z;
      }
    }
  } else if (jb.kind == 0 || jb.kind == 2) {
    // real part: DCT-III of a (pair: odd part of line b; middle: reversed even
    // slot of line b); imaginary part: DCT-III of b~ (reversed even slot)
    const double* A = X + sbase(jb.j) + (jb.kind == 0 ? SR : 0);
    const double* Bs = X + sbase(jb.j) + (jb.kind == 0 ? 0 : SR);
#if SFEM_ROWS_INV_PAIRS
    // One evaluation per (t, N-t) pair: the pair shares its four slot values,
    // the table entry (mkh[N-t] is mkh[t] with its components swapped) and
    // the two products -- V1' = conj(V1), V2' = conj(V2), so z_t = conj(V1 + i V2)
    // and z_{N-t} = V1 - i V2.  Half the slot and table loads and half the
    // products of the per-element form.  tau != 0: t = c1 + 8p pairs with class
    // c2 at index 7-p; tau == 0: class 0 pairs with itself (t = 8p, p = 1..3;
    // t = 32 alone; t = 0 unused) and so does class 4 (t = 4 + 8r, r = 0..3).
    const bool t0 = jb.tau == 0;
    double2 za[R], zb[R];
    Unroll<R>::run([&](auto P_) {
      constexpr int p = decltype(P_)::value;
      constexpr int T0[8] = {4, 8, 16, 24, 32, 12, 20, 28};
      const int t = t0 ? T0[p] : jb.tau + G * p;
      const double2 w = mkh[t];
      double ax, ar;
      if (jb.kind == 0) {
        ax = A[t];
        ar = A[N - t];
      } else {
        ax = A[N - t];
        ar = A[t];
      }
      const double bx = Bs[N - t], br = Bs[t];
      // V1 = w (ax - i ar), V2 = w (bx - i br)
      const double v1x = fma(w.x, ax, w.y * ar), v1y = fma(w.y, ax, -w.x * ar);
      const double v2x = fma(w.x, bx, w.y * br), v2y = fma(w.y, bx, -w.x * br);
      za[p] = make_double2(v1x - v2y, -(v1y + v2x));
      zb[p] = make_double2(v1x + v2y, v1y - v2x);
    });
    const double2 zero = make_double2(0.0, 0.0);
    v[0][0] = t0 ? zero : za[0];
    v[0][1] = za[1];
    v[0][2] = za[2];
    v[0][3] = za[3];
    v[0][4] = za[4];
    v[0][5] = t0 ? zb[3] : za[5];
    v[0][6] = t0 ? zb[2] : za[6];
    v[0][7] = t0 ? zb[1] : za[7];
    v[1][0] = t0 ? za[0] : zb[7];
    v[1][1] = t0 ? za[5] : zb[6];
    v[1][2] = t0 ? za[6] : zb[5];
    v[1][3] = t0 ? za[7] : zb[4];
    v[1][4] = t0 ? zb[7] : zb[3];
    v[1][5] = t0 ? zb[6] : zb[2];
    v[1][6] = t0 ? zb[5] : zb[1];
    v[1][7] = zb[0];
#else
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = h == 0 ? jb.c1 : jb.c2;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = c + G * r;
        double2 z = make_double2(0.0, 0.0);
        if (t > 0) {
          const double2 w = mkh[t];
          double ax, ar;
          if (jb.kind == 0) {
            ax = A[t];
            ar = A[N - t];
          } else {
            ax = A[N - t];
            ar = A[t];
          }
          const double bx = Bs[N - t], br = Bs[t];
          // V1 = w (ax - i ar), V2 = w (bx - i br); z = conj(V1 + i V2)
          const double v1x = fma(w.x, ax, w.y * ar), v1y = fma(w.y, ax, -w.x * ar);
          const double v2x = fma(w.x, bx, w.y * br), v2y = fma(w.y, bx, -w.x * br);
          z = make_double2(v1x - v2y, -(v1y + v2x));
        }
        v[h][r] = z;
      }
    }
#endif
  }
  __syncwarp();  // the warp's S rows are read: exchange data overwrites them
  if (jb.kind < 3) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = h == 0 ? jb.c1 : jb.c2;
      Dft<R>::run(v[h]);
#pragma unroll
      for (int q = 0; q < R; ++q) Xj[q * G + (c ^ q)] = q == 0 ? v[h][q] : c_mul(v[h][q], tw[(c * q) % N]);
    }
  }
  __syncwarp();
  double2 w[2][G];
  if (jb.kind < 3) {
#pragma unroll
    for (int c = 0; c < G; ++c) {
      w[0][c] = Xj[jb.q1 * G + (c ^ jb.q1)];
      w[1][c] = Xj[jb.q2 * G + (c ^ jb.q2)];
    }
  }
  __syncthreads();  // (B4) every slot is read: the output tile overwrites them
  if (jb.kind == 3) return;
  Dft<G>::run(w[0]);
  Dft<G>::run(w[1]);
  if (jb.kind == 1) {
    double* oa = T + jb.b * C::RP - 1;
    double* ob = T + (jb.b + 4) * C::RP - 1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = h == 0 ? jb.q1 : jb.q2;
      Unroll<G>::run([&](auto PP) {
        constexpr int p = decltype(PP)::value;
        const int kp = q + R * p;
        if (jb.which == 0 ? (kp < 1 || kp >= N / 2) : (kp >= N / 2)) return;
        const double2 zk = w[h][p];
        const double2 zc = partner<p>(w[0], w[1], jb.tau, h, jb.which == 1);
        // nodal j = 2 kp + which at position j*NN - 1 (the 1/2 of
        // X = (Z_partner - Z_k)/(2i) is folded into the inverse mix row s = 0)
        const int pos = (2 * kp + jb.which) * NN;
        oa[pos] = zc.y - zk.y;
        ob[pos] = zk.x - zc.x;
      });
    }
    return;
  }
  // u_t = conj(result_t): o = Re u, e~ = Im u at element e = makhoul_src(t)
  double* oi = T + jb.b * C::RP + (jb.kind == 0 ? jb.i : HALF);
  double* orr = jb.kind == 0 ? T + jb.b * C::RP + (M - 1 - jb.i) : T + (jb.b + 4) * C::RP + HALF;
  double ci_e, cr_e;  // centre terms for even elements (odd elements: -cr_e / -ci_e)
  if (jb.kind == 0) {
    ci_e = CI[jb.i * B + jb.b];
    cr_e = CI[(M - 1 - jb.i) * B + jb.b];
  } else {
    ci_e = CI[HALF * B + jb.b];
    cr_e = CI[HALF * B + jb.b + 4];
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = h == 0 ? jb.q1 : jb.q2;
    double* fi = oi + (2 * q) * NN;
    double* fr = orr + (2 * q) * NN;
    double* si = oi + (N - 1 - 2 * q) * NN;
    double* sr = orr + (N - 1 - 2 * q) * NN;
#pragma unroll
    for (int p = 0; p < G; ++p) {
      const double2 res = w[h][p];
      const double ure = res.x, uim = -res.y;
      const bool first = p < G / 2;  // element e even (first half) / odd
      const int off = first ? p * (2 * R) * NN : -(p - G / 2) * (2 * R) * NN;
      double vi, vr;
      if (jb.kind == 0) {
        if (first) {
          vi = ci_e + uim + ure;
          vr = cr_e + uim - ure;
        } else {
          vi = -cr_e - uim + ure;
          vr = -ci_e - uim - ure;
        }
      } else {
        vi = first ? ci_e + ure : -ci_e - ure;
        vr = first ? cr_e + uim : -cr_e - uim;
      }
      (first ? fi : si)[off] = vi;
      (first ? fr : sr)[off] = vr;
    }
  }
}

// ---------------------------------------------------------------------------
// Mixes.  Item (k, g): frequency k = 1..N-1, lines 4g..4g+3; the two items of
// one k are adjacent lanes (one matrix load serves both).  Forward mix (the
// synthesis matrix read transposed, 1/norm_sq in the denominator; table.cpp
// derive_device_data), divide, inverse mix.  The item's S entries are loaded
// once, its coefficients are parked in those same entries (slot l <- c_l) and
// reloaded for the inverse mix, whose results overwrite them: every access is
// the item's own, so no barrier separates the three steps.
// ---------------------------------------------------------------------------
template <int NN>
__host__ __device__ constexpr int srow_c(int s, int b) {
  // constexpr twin of srow (same placement)
  using C = Cfg<NN>;
  if (s == 0) return sbase(C::NPAIR + b);
  if (C::MODD && s == 1 + C::HALF) return sbase(C::NPAIR + C::NNOD + (b & 3)) + (b >> 2) * SR;
  const bool odd = s > C::HALF + C::MODD;
  const int i = odd ? s - 1 - C::NE : s - 1;
  int j = 0;
  if (C::HALF % 2 == 0) {
    const int HP = C::HALF / 2 > 0 ? C::HALF / 2 : 1;
    j = ((b >> 2) * HP + (i >> 1)) * 8 + ((b & 3) << 1) + (i & 1);
  } else {
    j = i * B + b;
  }
  return sbase(j) + (odd ? SR : 0);
}

// Rolled mixes (SFEM_ROWS_ROLLED_MIX, default): the column loops of the two
// mixes are real loops (the 9 x 4 FMAs of a column stay unrolled), with the
// slot offsets of a column's four results read from a small shared table.
// The unrolled form is ~1800 straight-line instructions executed once per
// tile and warp; with three CTAs in different phases the fused kernel's 93 KB
// of code did not stay in the instruction caches (ncu: no_instruction was the
// top stall reason, 1.2-2.7 per issue).
#ifndef SFEM_ROWS_MIX_PREFETCH
#define SFEM_ROWS_MIX_PREFETCH 0
#endif
#ifndef SFEM_ROWS_INV_PAIRS
#define SFEM_ROWS_INV_PAIRS 1
#endif
#ifndef SFEM_ROWS_ROLLED_MIX
#define SFEM_ROWS_ROLLED_MIX 1
#endif

template <int NN>
__device__ __forceinline__ void mix_item_rolled(int item, double* X, const double* __restrict__ mixT,
                                                const double* __restrict__ eig, const double* __restrict__ nsq,
                                                const double* base, double f_last, const int* soff) {
  using C = Cfg<NN>;
  const int k = 1 + (item & 15) + 16 * (item >> 5), g = (item >> 4) & 1;
  constexpr int S_PAIR = C::HALF > 0 ? 1 : (C::MODD ? 1 + C::HALF : 0);
  constexpr int OG_NOD = srow_c<NN>(0, 4) - srow_c<NN>(0, 0);
  constexpr int OG_PAIR = srow_c<NN>(S_PAIR, 4) - srow_c<NN>(S_PAIR, 0);
  constexpr int OG_MID = C::MODD ? srow_c<NN>(1 + C::HALF, 4) - srow_c<NN>(1 + C::HALF, 0) : 0;
  double* const xn = X + k + g * OG_NOD;
  double* const xp = X + k + g * OG_PAIR;
  double* const xm = X + k + g * OG_MID;
  auto at = [&](auto S_, int bb) -> double& {
    constexpr int s = decltype(S_)::value;
    double* const base_ = s == 0 ? xn : ((C::MODD && s == 1 + C::HALF) ? xm : xp);
    return base_[srow_c<NN>(s, bb)];
  };
  double* const Xk = X + k;
  const int4* so = reinterpret_cast<const int4*>(soff) + g * NN;  // [slot] -> offsets of lines 4g .. 4g+3
  double vv[NN][4];
  Unroll<NN>::run([&](auto S_) {
    constexpr int s = decltype(S_)::value;
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) vv[s][bb] = at(S_, bb);
  });
  double bs[4];
#pragma unroll
  for (int bb = 0; bb < 4; ++bb) bs[bb] = base[4 * g + bb];
  const double* mk = mixT + k;
#if SFEM_ROWS_MIX_PREFETCH
  // software pipeline: column l+1's matrix entries are loaded before column
  // l's divides (their dependent chains then hide the L1 latency)
  double mvn[NN];
#pragma unroll
  for (int s = 0; s < NN; ++s) mvn[s] = __ldg(mk + s * NN * N);
#endif
#pragma unroll 1
  for (int l = 0; l < NN; ++l) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const double* ml = mk + l * N;
#if SFEM_ROWS_MIX_PREFETCH
#pragma unroll
    for (int s = 0; s < NN; ++s) {
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) acc[bb] = fma(mvn[s], vv[s][bb], acc[bb]);
    }
    if (l + 1 < NN) {
#pragma unroll
      for (int s = 0; s < NN; ++s) mvn[s] = __ldg(ml + N + s * NN * N);
    }
#else
#pragma unroll
    for (int s = 0; s < NN; ++s) {
      const double mv = __ldg(ml + s * NN * N);
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) acc[bb] = fma(mv, vv[s][bb], acc[bb]);
    }
#endif
    const double lam = f_last * __ldg(eig + l * N + k), ns = __ldg(nsq + l * N + k);
    const int4 o = so[l];
    Xk[o.x] = sym_div(acc[0], (bs[0] + lam) * ns);
    Xk[o.y] = sym_div(acc[1], (bs[1] + lam) * ns);
    Xk[o.z] = sym_div(acc[2], (bs[2] + lam) * ns);
    Xk[o.w] = sym_div(acc[3], (bs[3] + lam) * ns);
  }
  __threadfence_block();
  double cv[NN][4];
  Unroll<NN>::run([&](auto L_) {
    constexpr int l = decltype(L_)::value;
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) cv[l][bb] = lds_once(&at(L_, bb));
  });
#pragma unroll 1
  for (int sI = 0; sI < NN; ++sI) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const double* ms = mk + sI * NN * N;
#pragma unroll
    for (int l = 0; l < NN; ++l) {
      const double mv = __ldg(ms + l * N);
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) acc[bb] = fma(mv, cv[l][bb], acc[bb]);
    }
    const int4 o = so[sI];
    Xk[o.x] = acc[0];
    Xk[o.y] = acc[1];
    Xk[o.z] = acc[2];
    Xk[o.w] = acc[3];
  }
}

template <int NN>
__device__ __forceinline__ void mix_item(int item, double* X, const double* __restrict__ mixT,
                                         const double* __restrict__ eig, const double* __restrict__ nsq,
                                         const double* base, double f_last) {
  using C = Cfg<NN>;
  constexpr int M = C::M;
  // lanes 0-15 / 16-31 of a warp: the same 16 frequencies, line groups 0 / 1
  // (one matrix load serves both halves; a 64-bit phase sees 16 distinct k)
  const int k = 1 + (item & 15) + 16 * (item >> 5), g = (item >> 4) & 1;
  // S entry (s, line 4g + bb) of this k: one base pointer per slot class
  // (the line-group step is the same for all slots of a class), the rest
  // compile-time offsets
  constexpr int S_PAIR = C::HALF > 0 ? 1 : (C::MODD ? 1 + C::HALF : 0);
  constexpr int OG_NOD = srow_c<NN>(0, 4) - srow_c<NN>(0, 0);
  constexpr int OG_PAIR = srow_c<NN>(S_PAIR, 4) - srow_c<NN>(S_PAIR, 0);
  constexpr int OG_MID = C::MODD ? srow_c<NN>(1 + C::HALF, 4) - srow_c<NN>(1 + C::HALF, 0) : 0;
  double* const xn = X + k + g * OG_NOD;
  double* const xp = X + k + g * OG_PAIR;
  double* const xm = X + k + g * OG_MID;
  auto at = [&](auto S_, int bb) -> double& {
    constexpr int s = decltype(S_)::value;
    double* const base_ = s == 0 ? xn : ((C::MODD && s == 1 + C::HALF) ? xm : xp);
    return base_[srow_c<NN>(s, bb)];
  };
  double vv[NN][4];
  Unroll<NN>::run([&](auto S_) {
    constexpr int s = decltype(S_)::value;
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) vv[s][bb] = at(S_, bb);
  });
  double bs[4];
#pragma unroll
  for (int bb = 0; bb < 4; ++bb) bs[bb] = base[4 * g + bb];
  const double* mk = mixT + k;
  Unroll<NN>::run([&](auto L_) {
    constexpr int l = decltype(L_)::value;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int s = 0; s < NN; ++s) {
      const double mv = ldg_once(mk + (s * NN + l) * N);
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) acc[bb] = fma(mv, vv[s][bb], acc[bb]);
    }
    const double lam = f_last * __ldg(eig + l * N + k), ns = __ldg(nsq + l * N + k);  // eigT / nsqT ([l][k])
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) at(L_, bb) = sym_div(acc[bb], (bs[bb] + lam) * ns);
    SFEM_ROWS_FENCE();  // one column of matrix loads in flight at a time (register budget)
  });
#ifdef SFEM_ROWS_DIAG_FWDONLY
  return;
#endif
  __threadfence_block();  // keep the coefficient reloads after the forward mix (register budget)
  double cv[NN][4];
  Unroll<NN>::run([&](auto L_) {
    constexpr int l = decltype(L_)::value;
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) cv[l][bb] = lds_once(&at(L_, bb));
  });
  Unroll<NN>::run([&](auto S_) {
    constexpr int s = decltype(S_)::value;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int l = 0; l < NN; ++l) {
      const double mv = ldg_once(mk + (s * NN + l) * N);
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) acc[bb] = fma(mv, cv[l][bb], acc[bb]);
    }
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) at(S_, bb) = acc[bb];
    SFEM_ROWS_FENCE();
  });
}

// k = 0 block of line b: centre sums -> m x m forward -> divide -> m x m
// inverse -> inverse centre terms CI[.][b].
template <int NN>
__device__ __forceinline__ void mix_zero(int b, const double* C0, double* CI, const double* __restrict__ e0f,
                                         const double* __restrict__ e0i, const double* __restrict__ eig,
                                         const double* base, double f_last) {
  using C = Cfg<NN>;
  constexpr int M = C::M;
  if constexpr (M > 0) {
    double cs[M], c0[M];
#pragma unroll
    for (int ii = 0; ii < M; ++ii) {
      const int o = ii * B + b;
      cs[ii] = ((C0[o] + C0[C::MB + o]) + C0[2 * C::MB + o]) + C0[3 * C::MB + o];
    }
#pragma unroll
    for (int l = 0; l < M; ++l) {
      double acc = 0.0;
#pragma unroll
      for (int ii = 0; ii < M; ++ii) acc = fma(cs[ii], __ldg(e0f + ii * M + l), acc);
      c0[l] = sym_div(acc, base[b] + f_last * __ldg(eig + l));
    }
#pragma unroll
    for (int ii = 0; ii < M; ++ii) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < M; ++l) acc = fma(__ldg(e0i + ii * M + l), c0[l], acc);
      CI[ii * B + b] = acc;
    }
  }
}

// FFT tables (tw | mkh | om, N complex each) in constant memory
// (SFEM_ROWS_CONST_TAB): the lookups leave the L1 / shared data pipe, which is
// what bounds this kernel, for the constant cache.  They depend on N = 64 only.
#ifndef SFEM_ROWS_CONST_TAB
#define SFEM_ROWS_CONST_TAB 0
#endif
__constant__ double2 c_tab64[3 * N];

template <int NN>
__global__ void __launch_bounds__(Cfg<NN>::THREADS, SFEM_ROWS_MINB(NN))
    sweep_rows_fused(DevTable t, double* data, RowSegs segs, long long nrows, SymbolInfo sym,
                     const double* __restrict__ e0F) {
  using C = Cfg<NN>;
  extern __shared__ __align__(128) double smem[];
  double* T = smem;  // row tile / job slots / mix scratch (aliased, phases separated by barriers)
  double* C0 = smem + C::C0_OFF;
  double* CI = smem + C::CI_OFF;
  double* base = smem + C::BASE_OFF;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + C::BAR_OFF);
#if SFEM_ROWS_CONST_TAB
  const double2* tw = c_tab64;
  const double2* mkh = c_tab64 + N;
  const double2* om = c_tab64 + 2 * N;
#else
  double2* tw = reinterpret_cast<double2*>(smem + C::TAB_OFF);
  double2* mkh = tw + N;
  double2* om = mkh + N;
#endif
  int* soff = reinterpret_cast<int*>(smem + C::SOFF_OFF);
  const int tid = threadIdx.x;
  const long long l0 = static_cast<long long>(blockIdx.x) * B;
  const int Bv = static_cast<int>(min(static_cast<long long>(B), nrows - l0));
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    mbar_expect_tx(bar, static_cast<unsigned>(Bv * C::P * sizeof(double)));
  }
  __syncthreads();  // barrier initialised and armed before any copy completes
  for (int i = tid; i < Bv * segs.n; i += C::THREADS) {
    const int b = i / segs.n, sg = i - b * segs.n;
    bulk_load(T + b * C::RP + segs.pos0[sg], data + segs.off[sg] + (l0 + b) * segs.stride[sg],
              segs.len[sg] * sizeof(double), bar);
  }
  for (int i = tid; i < (B - Bv) * C::RP; i += C::THREADS) T[Bv * C::RP + i] = 0.0;  // phantom rows
  if (tid < B && sym.xblk > 0) {
    // blocked 3-D layout: row (x_hi, y, x_lo), x = x_hi*xblk + x_lo
    const long long l = l0 + tid < nrows ? l0 + tid : 0;
    const long long xlo = l % sym.xblk, r1 = l / sym.xblk;
    const long long y = r1 % sym.lead_ext[1], xhi = r1 / sym.lead_ext[1];
    const long long x = min(xhi * sym.xblk + xlo, sym.x_ext - 1);  // padding rows: any finite base
    const double t0 = sym.lead_f[0] * sym.lead_eig[0][x], t1 = sym.lead_f[1] * sym.lead_eig[1][y];
    base[tid] = (sym.shift + t0) + t1;
  } else if (tid < B) {
    // base = shift + sum_{i<N-1} f_i lambda_i (poisson.cpp:586-590 order)
    const long long l = l0 + tid;
    long long rem = l < nrows ? l : 0;
    double terms[kMaxDim];
#pragma unroll
    for (int ii = kMaxDim - 1; ii >= 0; --ii) {
      terms[ii] = 0.0;
      if (ii < sym.nlead) {
        const long long a = rem % sym.lead_ext[ii];
        rem /= sym.lead_ext[ii];
        terms[ii] = sym.lead_f[ii] * sym.lead_eig[ii][a];
      }
    }
    double sacc = sym.shift;
#pragma unroll
    for (int ii = 0; ii < kMaxDim; ++ii)
      if (ii < sym.nlead) sacc += terms[ii];
    base[tid] = sacc;
  }
#if !SFEM_ROWS_CONST_TAB
  for (int i = tid; i < N; i += C::THREADS) {
    tw[i] = t.tw[i];
    mkh[i] = t.mkh[i];
    om[i] = t.om[i];
  }
#endif
#if SFEM_ROWS_ROLLED_MIX
  if (tid < 2 * NN * 4) soff[tid] = srow<NN>((tid >> 2) % NN, 4 * (tid / (4 * NN)) + (tid & 3));
#endif
  __syncthreads();  // tables, bases, phantom rows
  mbar_wait(bar, 0);
  const Job jb = job_of<NN>(tid);
  forward_job<NN>(jb, T, T, C0, tw, mkh, om);  // contains B1
  __syncthreads();                              // (B2) S rows and centre partials complete
#ifndef SFEM_ROWS_DIAG_NOMIX
  if (tid < C::ITEMS) {
    // rolled for the large orders only (n = 9: 1.50 -> 1.33 ms; n <= 7: +-2 %, their code is smaller)
    if ((tid & 15) + 16 * (tid >> 5) < N - 1) {
      if constexpr (SFEM_ROWS_ROLLED_MIX && NN >= 8)
        mix_item_rolled<NN>(tid, T, t.mixT_i, t.eigT, t.nsqT, base, sym.f_last, soff);
      else
        mix_item<NN>(tid, T, t.mixT_i, t.eigT, t.nsqT, base, sym.f_last);
    }
  }
#else
  if (false) {
  }
#endif
  else if (tid - C::ITEMS < B)
    mix_zero<NN>(tid - C::ITEMS, C0, CI, e0F, t.e0_inv, t.eig, base, sym.f_last);
  __syncthreads();  // (B3) mixed S rows and inverse centre terms complete
  inverse_job<NN>(jb, T, T, CI, tw, mkh, om);  // contains B4
  if (C::P > C::L) {
    if (tid < B) T[tid * C::RP + C::L] = 0.0;  // row padding element (written by no job)
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();  // (B5) output tile complete
  for (int i = tid; i < Bv * segs.n; i += C::THREADS) {
    const int b = i / segs.n, sg = i - b * segs.n;
    bulk_store(data + segs.off[sg] + (l0 + b) * segs.stride[sg], T + b * C::RP + segs.pos0[sg],
               segs.len[sg] * sizeof(double));
  }
  if (tid < Bv * segs.n) {
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
  }
}

template <int NN>
cudaError_t launch_nn(const DevTable& t, double* data, const RowSegs& segs, long long nrows, const SymbolInfo& sym,
                      cudaStream_t stream) {
  using C = Cfg<NN>;
  int row_len = 0;
  for (int sg = 0; sg < segs.n; ++sg) row_len += segs.len[sg];
  if (segs.n < 1 || segs.n > kMaxSeg || row_len != C::P) return cudaErrorInvalidValue;
  auto kern = sweep_rows_fused<NN>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (err != cudaSuccess) return err;
#if SFEM_ROWS_CONST_TAB
  {
    static bool done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !done[dev]) {
      err = cudaMemcpyToSymbolAsync(c_tab64, t.tw, N * sizeof(double2), 0, cudaMemcpyDeviceToDevice, stream);
      if (err == cudaSuccess)
        err = cudaMemcpyToSymbolAsync(c_tab64, t.mkh, N * sizeof(double2), N * sizeof(double2),
                                      cudaMemcpyDeviceToDevice, stream);
      if (err == cudaSuccess)
        err = cudaMemcpyToSymbolAsync(c_tab64, t.om, N * sizeof(double2), 2 * N * sizeof(double2),
                                      cudaMemcpyDeviceToDevice, stream);
      if (err != cudaSuccess) return err;
      done[dev] = true;
    }
  }
#endif
  const dim3 grid(static_cast<unsigned>((nrows + B - 1) / B));
  kern<<<grid, C::THREADS, C::SMEM, stream>>>(t, data, segs, nrows, sym, t.e0_fwd_w);
  return cudaGetLastError();
}

}  // namespace rows

bool has_rows_fused(int n, int K) { return K == 64 && n >= 2 && n <= 9; }

cudaError_t launch_sweep_rows_fused(const DevTable& t, double* data, const RowSegs& segs, long long nrows,
                                    const SymbolInfo& sym, cudaStream_t stream) {
  if (!has_rows_fused(t.n, t.K)) return cudaErrorNotSupported;
  if (nrows <= 0) return cudaSuccess;
  switch (t.n) {
    case 2: return rows::launch_nn<2>(t, data, segs, nrows, sym, stream);
    case 3: return rows::launch_nn<3>(t, data, segs, nrows, sym, stream);
    case 4: return rows::launch_nn<4>(t, data, segs, nrows, sym, stream);
    case 5: return rows::launch_nn<5>(t, data, segs, nrows, sym, stream);
    case 6: return rows::launch_nn<6>(t, data, segs, nrows, sym, stream);
    case 7: return rows::launch_nn<7>(t, data, segs, nrows, sym, stream);
    case 8: return rows::launch_nn<8>(t, data, segs, nrows, sym, stream);
    case 9: return rows::launch_nn<9>(t, data, segs, nrows, sym, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace sfem_b200
