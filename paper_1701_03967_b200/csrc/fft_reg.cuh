// Register-resident small DFTs (compile-time size), forward sign exp(-2 pi i/R).
#pragma once

#include <cuda_runtime.h>

namespace sfem_b200 {
namespace reg {

__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 c_mulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}

// cos(2 pi j / 16), j = 0..16
__device__ __forceinline__ constexpr double cos16(int j) {
  constexpr double c[17] = {1.0,
                            0.92387953251128675613,
                            0.70710678118654752440,
                            0.38268343236508977173,
                            0.0,
                            -0.38268343236508977173,
                            -0.70710678118654752440,
                            -0.92387953251128675613,
                            -1.0,
                            -0.92387953251128675613,
                            -0.70710678118654752440,
                            -0.38268343236508977173,
                            0.0,
                            0.38268343236508977173,
                            0.70710678118654752440,
                            0.92387953251128675613,
                            1.0};
  return c[j];
}

// x * exp(-2 pi i J / R) for compile-time J, R (R | 16)
template <int R, int J>
__device__ __forceinline__ double2 twiddle(double2 x) {
  constexpr int j16 = (J * (16 / R)) % 16;
  if constexpr (j16 == 0) {
    return x;
  } else if constexpr (j16 == 4) {  // -i
    return make_double2(x.y, -x.x);
  } else if constexpr (j16 == 8) {
    return make_double2(-x.x, -x.y);
  } else if constexpr (j16 == 12) {  // +i
    return make_double2(-x.y, x.x);
  } else if constexpr (j16 == 2) {  // (1 - i)/sqrt2
    constexpr double s = 0.70710678118654752440;
    return make_double2(s * (x.x + x.y), s * (x.y - x.x));
  } else if constexpr (j16 == 6) {  // (-1 - i)/sqrt2
    constexpr double s = 0.70710678118654752440;
    return make_double2(s * (x.y - x.x), -s * (x.x + x.y));
  } else if constexpr (j16 == 10) {  // (-1 + i)/sqrt2
    constexpr double s = 0.70710678118654752440;
    return make_double2(-s * (x.x + x.y), s * (x.x - x.y));
  } else if constexpr (j16 == 14) {  // (1 + i)/sqrt2
    constexpr double s = 0.70710678118654752440;
    return make_double2(s * (x.x - x.y), s * (x.x + x.y));
  } else {
    constexpr double c = cos16(j16);
    constexpr double sn = cos16((j16 + 12) % 16);  // sin(2 pi j/16) = cos(2 pi (j-4)/16)
    // multiply by (c - i sn)
    return make_double2(fma(x.x, c, x.y * sn), fma(x.y, c, -x.x * sn));
  }
}

// In-place DFT of length R (1, 2, 4, 8, 16), natural order in and out.
template <int R>
struct Dft {
  template <int J>
  __device__ __forceinline__ static void split(double2 (&x)[R], double2 (&a)[R / 2], double2 (&b)[R / 2]) {
    if constexpr (J < R / 2) {
      a[J] = c_add(x[J], x[J + R / 2]);
      b[J] = twiddle<R, J>(c_sub(x[J], x[J + R / 2]));
      split<J + 1>(x, a, b);
    }
  }
  __device__ __forceinline__ static void run(double2 (&x)[R]) {
    double2 a[R / 2], b[R / 2];
    split<0>(x, a, b);
    Dft<R / 2>::run(a);
    Dft<R / 2>::run(b);
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      x[2 * k] = a[k];
      x[2 * k + 1] = b[k];
    }
  }
};
template <>
struct Dft<1> {
  __device__ __forceinline__ static void run(double2 (&)[1]) {}
};
template <>
struct Dft<2> {
  __device__ __forceinline__ static void run(double2 (&x)[2]) {
    const double2 a = x[0], b = x[1];
    x[0] = c_add(a, b);
    x[1] = c_sub(a, b);
  }
};

}  // namespace reg
}  // namespace sfem_b200
