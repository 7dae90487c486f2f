// Slot-major class tiles <-> slot-major dof tiles for the batched line API
// (reference lines::decompose_weighted_block / synthesize_block,
// eigenbasis.hpp:66-73: the value at position j of line b sits at
// [j*count + b]; nodal tile (K+1) x count with the boundary slots, interior
// tile K*(n-1) x count element-major).  The dof tile has one row per dof
// t = e*n + c (interior component c of element e) or t = j*n - 1 (node j),
// n*K - 1 rows of `count` entries, which is what the strided sweeps run on.
#include <cuda_runtime.h>

#include "sweep.cuh"

namespace sfem_b200 {
namespace {

template <bool TO_DOF>
__global__ void __launch_bounds__(256) class_tiles(int n, int K, long long count, double* nodal, double* interior,
                                                   double* dof) {
  const long long L = static_cast<long long>(n) * K - 1;
  const long long total = L * count;
  const int m = n - 1;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total; i += 256LL * gridDim.x) {
    const long long t = i / count, b = i - t * count;
    const long long e = t / n;
    const int c = static_cast<int>(t - e * n);
    double* cls = c == m ? nodal + (e + 1) * count + b : interior + (e * m + c) * count + b;
    if (TO_DOF)
      dof[i] = *cls;
    else
      *cls = dof[i];
  }
  if (!TO_DOF) {
    // boundary slots of the nodal tile are written as zero (eigenbasis.cpp:353-356)
    for (long long b = blockIdx.x * 256LL + threadIdx.x; b < count; b += 256LL * gridDim.x) {
      nodal[b] = 0.0;
      nodal[static_cast<long long>(K) * count + b] = 0.0;
    }
  }
}

}  // namespace

cudaError_t launch_class_tiles(int n, int K, long long count, double* nodal, double* interior, double* dof,
                               bool to_dof, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const long long total = (static_cast<long long>(n) * K - 1) * count;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  if (to_dof)
    class_tiles<true><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(n, K, count, nodal, interior, dof);
  else
    class_tiles<false><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(n, K, count, nodal, interior, dof);
  return cudaGetLastError();
}

}  // namespace sfem_b200
