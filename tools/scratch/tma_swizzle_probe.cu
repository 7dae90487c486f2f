// Probe: where a 2-D TMA box of 64-byte rows (8 doubles) lands in shared
// memory under CU_TENSOR_MAP_SWIZZLE_128B, against the index formula the mid
// kernels use: idx = pos * 8 + b; idx ^ (((idx >> 4) & 7) << 1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/swz tools/scratch/tma_swizzle_probe.cu && /tmp/swz
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
constexpr int ROWS = 256, NBOX = 2;
__global__ void k(const __grid_constant__ CUtensorMap map, double* out, unsigned* base, int do_store, int padd) {
  extern __shared__ __align__(1024) double smem[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + NBOX * (ROWS * 8 + 16));
  if (threadIdx.x == 0) {
    *base = su32(smem);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(NBOX * ROWS * 64) : "memory");
    for (int j = 0; j < NBOX; ++j)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
                   "r"(su32(smem + j * (ROWS * 8 + padd))), "l"(&map), "r"(8), "r"(j * ROWS), "r"(su32(bar)) : "memory");
  }
  __syncthreads();
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < NBOX * ROWS * 8; i += blockDim.x) out[i] = smem[i + (i / (ROWS * 8)) * padd];
  // store back through the same map (shifted by 16 columns) to check the store side un-swizzles
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0 && do_store) {
    for (int j = 0; j < NBOX; ++j)
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(&map), "r"(24),
                   "r"(j * ROWS), "r"(su32(smem + j * (ROWS * 8 + padd))) : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}
int main(int argc, char** argv) {
  const int swz = argc > 1 ? atoi(argv[1]) : 3, do_store = argc > 2 ? atoi(argv[2]) : 1, padd = argc > 3 ? atoi(argv[3]) : 0;
  const int rows = 600, pitch = 64;
  std::vector<double> h(rows * pitch);
  for (int r = 0; r < rows; ++r) for (int p = 0; p < pitch; ++p) h[r * pitch + p] = r * 100 + p;
  double *d, *o; unsigned* bp;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, NBOX * ROWS * 64); cudaMalloc(&bp, 4);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  alignas(64) CUtensorMap map;
  cuuint64_t dims[2] = {pitch, rows}; cuuint64_t strides[1] = {pitch * 8}; cuuint32_t box[2] = {8, ROWS}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   static_cast<CUtensorMapSwizzle>(swz), CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("pad doubles %d: ", padd); printf("swizzle mode %d store %d encode %d\n", swz, do_store, (int)r);
  const int sm = NBOX * (ROWS * 64 + 128) + 16;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k<<<1, 128, sm>>>(map, o, bp, do_store, padd);
  cudaError_t e = cudaDeviceSynchronize();
  printf("run: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  unsigned base; cudaMemcpy(&base, bp, 4, cudaMemcpyDeviceToHost);
  printf("dynamic shared base 0x%x (mod 1024 = %u)\n", base, base % 1024);
  std::vector<double> g(NBOX * ROWS * 8);
  cudaMemcpy(g.data(), o, g.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int pos = 0; pos < NBOX * ROWS; ++pos) for (int b = 0; b < 8; ++b) {
    const int idx = pos * 8 + b, sw = swz == 3 ? idx ^ (((idx >> 4) & 7) << 1) : (swz == 2 ? idx ^ (((idx >> 4) & 3) << 1) : idx);
    const double want = pos * 100 + 8 + b;
    if (g[sw] != want) { if (bad < 8) printf("  pos %d b %d: smem[%d] = %g want %g\n", pos, b, sw, g[sw], want); ++bad; }
  }
  printf("swizzle formula mismatches %d of %d\n", bad, NBOX * ROWS * 8);
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  int sbad = 0;
  for (int r2 = 0; r2 < NBOX * ROWS; ++r2) for (int b = 0; b < 8; ++b)
    if (h[r2 * pitch + 24 + b] != r2 * 100 + 8 + b) ++sbad;
  printf("store-side mismatches %d\n", sbad);
  return bad || sbad;
}
