// Probe: 2-D TMA row boxes with element-granular (negative) start coordinates.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap map, double* out, int nbr, int B) {
  extern __shared__ __align__(128) double smem[];
  __shared__ unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(B * nbr * 2048) : "memory");
  }
  __syncthreads();
  for (int it = threadIdx.x; it < B * nbr; it += blockDim.x) {
    const int b = it / nbr, j = it - b * nbr;
    const int c0 = MODE == 0 ? j * 256 : j * 256 - b;
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
                 "r"(su32(smem + (b * nbr + j) * 256)), "l"(&map), "r"(c0), "r"(b), "r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < B * nbr * 256; i += blockDim.x) out[i] = smem[i];
}
int main() {
  const int L = 1023, rows = 9, pitch = 1024, B = 8, nbr = 5;
  std::vector<double> h(rows * pitch);
  for (int r = 0; r < rows; ++r) for (int p = 0; p < pitch; ++p) h[r * pitch + p] = r * 10000 + p;
  double *d, *o; cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, B * nbr * 256 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  alignas(64) CUtensorMap map;
  cuuint64_t dims[2] = {L, rows}; cuuint64_t strides[1] = {pitch * 8}; cuuint32_t box[2] = {256, 1}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int mode = 0; mode < 2; ++mode) {
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, B * nbr * 2048);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, B * nbr * 2048);
    if (mode == 0) k<0><<<1, 128, B * nbr * 2048>>>(map, o, nbr, B); else k<1><<<1, 128, B * nbr * 2048>>>(map, o, nbr, B);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<double> g(B * nbr * 256);
    cudaMemcpy(g.data(), o, g.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int b = 0; b < B; ++b) for (int i = 0; i < nbr * 256; ++i) {
      const int pos = mode == 0 ? i : i - b;
      const double want = (pos >= 0 && pos < L) ? b * 10000 + pos : 0.0;
      if (g[b * nbr * 256 + i] != want) { if (bad < 5) printf("  b %d i %d got %g want %g\n", b, i, g[b * nbr * 256 + i], want); ++bad; }
    }
    printf("mode %d mismatches %d\n", mode, bad);
  }
  return 0;
}
