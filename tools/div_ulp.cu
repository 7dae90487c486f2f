// Max ulp distance of the sweep kernels' branch-free divide (1 or 2 Newton
// steps on the MUFU reciprocal seed) from the IEEE quotient, over random
// positive denominators spanning 1e-3 .. 1e9 (GPU box:  nvcc -arch=sm_100a
// tools/div_ulp.cu -o /tmp/div_ulp && /tmp/div_ulp).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>

template <int NEWTON>
__device__ double sym_div(double c, double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = fma(r, fma(-d, r, 1.0), r);
  if (NEWTON > 1) r = fma(r, fma(-d, r, 1.0), r);
  const double q = c * r;
  return fma(fma(-d, q, c), r, q);
}

__device__ unsigned long long hash(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}
__device__ double u01(unsigned long long h) { return (h >> 11) * (1.0 / 9007199254740992.0); }

template <int NEWTON>
__global__ void kern(long long n, unsigned long long* maxulp, unsigned long long* nexact) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned long long mu = 0, ex = 0;
  for (; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double c = 2.0 * u01(hash(2 * i)) - 1.0;
    const double d = exp(log(1e-3) + u01(hash(2 * i + 1)) * (log(1e9) - log(1e-3)));
    const double a = sym_div<NEWTON>(c, d), b = c / d;
    long long ia = __double_as_longlong(a), ib = __double_as_longlong(b);
    unsigned long long diff = (unsigned long long)(ia > ib ? ia - ib : ib - ia);
    if (diff > mu) mu = diff;
    ex += diff == 0;
  }
  atomicMax(maxulp, mu);
  atomicAdd(nexact, ex);
}

int main() {
  unsigned long long *m, *e;
  cudaMallocManaged(&m, 8);
  cudaMallocManaged(&e, 8);
  const long long n = 1LL << 30;
  for (int nw = 1; nw <= 2; ++nw) {
    *m = 0; *e = 0;
    if (nw == 1) kern<1><<<1184, 256>>>(n, m, e); else kern<2><<<1184, 256>>>(n, m, e);
    cudaDeviceSynchronize();
    printf("newton=%d: max ulp %llu, exact %.6f of %lld\n", nw, *m, (double)*e / n, n);
  }
  return 0;
}
