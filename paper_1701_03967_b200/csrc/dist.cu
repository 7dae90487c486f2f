// Slab transposes for the multi-GPU solve.
//
// The x-slab of a rank is a local dof tensor [lx][L1][rest...] (last axis
// padded); the exchange buffer is the same data transposed to [L1*R][bpitch]
// (bpitch = lx rounded up to even, the pad column zero),
// R = prod(L2..L_{N-1}), i.e. destination-major blocks [ly_s][R][lx] in rank
// order (the a1 slabs of the destinations are contiguous and ordered), ready
// for an all-to-all with split sizes lx*ly_s*R.
#include <cuda_runtime.h>

#include "dist.cuh"

namespace sfem_b200 {
namespace {

constexpr int TT = 32;  // transpose tile

// The x-slab is walked as (a0l, z, i): i = the contiguous last axis (extent
// EI = L_{N-1}; for N = 2 it is axis 1 itself), z = the remaining middle
// coordinates (a1 [, a2]), so q = z * EI + i and the x offset is
// a0l * st0 + zoff(z) + i: no per-element division.  One CTA moves a 32 x 32
// (i, a0l) tile at one z through padded shared memory (both global sides
// coalesced).
template <bool TO_BUF>
__global__ void __launch_bounds__(TT * 8) slab_transpose(SlabView v, double* x, double* buf) {
  __shared__ double tile[TT][TT + 1];
  const int tx = threadIdx.x & (TT - 1), ty = threadIdx.x / TT;  // 32 x 8 threads
  const long long EI = v.nrest == 0 ? v.Q : (v.nrest == 1 ? v.R : v.e3);
  const long long Z = v.Q / EI;
  const long long i0 = static_cast<long long>(blockIdx.x) * TT;
  const long long a00 = static_cast<long long>(blockIdx.y) * TT;
  for (long long z = blockIdx.z; z < Z; z += gridDim.z) {
    long long zoff;
    if (v.nrest == 0) {
      zoff = 0;
    } else if (v.nrest == 1) {
      zoff = z * v.st1;
    } else {
      const long long R2 = v.R / v.e3;  // extent of axis 2
      const long long a1 = z / R2, a2 = z - a1 * R2;
      zoff = a1 * v.st1 + a2 * v.st2;
    }
    const long long q0 = z * EI + i0;
    if (TO_BUF) {
      // read x with lanes over i (contiguous), write buf with lanes over a0
#pragma unroll
      for (int j = ty; j < TT; j += 8) {
        const long long a0 = a00 + j, i = i0 + tx;
        if (a0 < v.lx && i < EI) tile[j][tx] = x[a0 * v.st0 + zoff + i];
      }
      __syncthreads();
#pragma unroll
      for (int j = ty; j < TT; j += 8) {
        const long long i = i0 + j, a0 = a00 + tx;
        if (i < EI) {
          if (a0 < v.lx) buf[(q0 + j) * v.bpitch + a0] = tile[tx][j];
          if (a0 == v.lx && a0 < v.bpitch) buf[(q0 + j) * v.bpitch + a0] = 0.0;  // pad column
        }
      }
    } else {
#pragma unroll
      for (int j = ty; j < TT; j += 8) {
        const long long i = i0 + j, a0 = a00 + tx;
        if (a0 < v.lx && i < EI) tile[tx][j] = buf[(q0 + j) * v.bpitch + a0];
      }
      __syncthreads();
#pragma unroll
      for (int j = ty; j < TT; j += 8) {
        const long long a0 = a00 + j, i = i0 + tx;
        if (a0 < v.lx && i < EI) x[a0 * v.st0 + zoff + i] = tile[j][tx];
      }
    }
    __syncthreads();  // tile reused for the next z
  }
}

}  // namespace

cudaError_t launch_slab_transpose(const SlabView& v, double* x, double* buf, bool to_buf, cudaStream_t stream) {
  if (v.lx <= 0 || v.Q <= 0) return cudaSuccess;
  const long long EI = v.nrest == 0 ? v.Q : (v.nrest == 1 ? v.R : v.e3);
  const long long Z = v.Q / EI;
  const dim3 grid(static_cast<unsigned>((EI + TT - 1) / TT), static_cast<unsigned>((v.lx + TT - 1) / TT),
                  static_cast<unsigned>(Z < 65535 ? Z : 65535));
  if (to_buf)
    slab_transpose<true><<<grid, TT * 8, 0, stream>>>(v, x, buf);
  else
    slab_transpose<false><<<grid, TT * 8, 0, stream>>>(v, x, buf);
  return cudaGetLastError();
}

}  // namespace sfem_b200
