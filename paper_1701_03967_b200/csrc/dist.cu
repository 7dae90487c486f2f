// Slab transposes for the multi-GPU solve.
//
// The x-slab of a rank is a local dof tensor [lx][L1][rest...] (last axis
// padded); the exchange buffer is the same data transposed to [L1*R][lx],
// R = prod(L2..L_{N-1}), i.e. destination-major blocks [ly_s][R][lx] in rank
// order (the a1 slabs of the destinations are contiguous and ordered), ready
// for an all-to-all with split sizes lx*ly_s*R.
#include <cuda_runtime.h>

#include "dist.cuh"

namespace sfem_b200 {
namespace {

constexpr int TT = 32;  // transpose tile

// x offset of (a0l, q) with q = a1 * R + r, r decoded over the rest axes.
__device__ __forceinline__ long long x_offset(const SlabView& v, long long a0l, long long q) {
  const long long a1 = q / v.R, r = q - a1 * v.R;
  long long off = a0l * v.st0 + a1 * v.st1;
  // rest axes 2..N-1 (at most two): r = r2 * e3 + r3
  if (v.nrest == 1) {
    off += r;  // last axis, unit stride
  } else if (v.nrest == 2) {
    const long long r2 = r / v.e3, r3 = r - r2 * v.e3;
    off += r2 * v.st2 + r3;
  }
  return off;
}

template <bool TO_BUF>
__global__ void __launch_bounds__(TT * 8) slab_transpose(SlabView v, double* x, double* buf) {
  __shared__ double tile[TT][TT + 1];
  const long long q0 = static_cast<long long>(blockIdx.x) * TT;
  const long long a00 = static_cast<long long>(blockIdx.y) * TT;
  const int tx = threadIdx.x & (TT - 1), ty = threadIdx.x / TT;  // 32 x 8 threads
  if (TO_BUF) {
    // read x with lanes over q (contiguous along the last axis), write buf with lanes over a0
    for (int j = ty; j < TT; j += 8) {
      const long long a0 = a00 + j, q = q0 + tx;
      if (a0 < v.lx && q < v.Q) tile[j][tx] = x[x_offset(v, a0, q)];
    }
    __syncthreads();
    for (int j = ty; j < TT; j += 8) {
      const long long q = q0 + j, a0 = a00 + tx;
      if (a0 < v.lx && q < v.Q) buf[q * v.lx + a0] = tile[tx][j];
    }
  } else {
    for (int j = ty; j < TT; j += 8) {
      const long long q = q0 + j, a0 = a00 + tx;
      if (a0 < v.lx && q < v.Q) tile[tx][j] = buf[q * v.lx + a0];
    }
    __syncthreads();
    for (int j = ty; j < TT; j += 8) {
      const long long a0 = a00 + j, q = q0 + tx;
      if (a0 < v.lx && q < v.Q) x[x_offset(v, a0, q)] = tile[j][tx];
    }
  }
}

}  // namespace

cudaError_t launch_slab_transpose(const SlabView& v, double* x, double* buf, bool to_buf, cudaStream_t stream) {
  if (v.lx <= 0 || v.Q <= 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((v.Q + TT - 1) / TT), static_cast<unsigned>((v.lx + TT - 1) / TT));
  if (to_buf)
    slab_transpose<true><<<grid, TT * 8, 0, stream>>>(v, x, buf);
  else
    slab_transpose<false><<<grid, TT * 8, 0, stream>>>(v, x, buf);
  return cudaGetLastError();
}

}  // namespace sfem_b200
