// tools/fp64_probe.cu -- FP64 pipe microbenchmark on the B200 (SURVEY.md 7.4
// item 1 asked for it): DFMA throughput, DMMA (mma.sync f64) throughput, and
// both at once (separate pipes or one?), plus 64-bit shuffle throughput.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b, int mode) {
  // mode 0: all warps DFMA; mode 1: even warps DFMA, odd warps DMMA; mode 2: all DMMA
  const int warp = threadIdx.x >> 5;
  const bool do_mma = mode == 2 || (mode == 1 && (warp & 1));
  if (!do_mma) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = a * (threadIdx.x + i);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345) out[threadIdx.x] = s;
  } else {
    double acc[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
    double fa = a * threadIdx.x, fb = b;
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[i][0]), "+d"(acc[i][1])
                     : "d"(fa), "d"(fb));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
    if (s == 1.2345) out[threadIdx.x] = s;
  }
}

__global__ void shfl_kernel(double* out, double a) {
  double x = a * threadIdx.x, y = a + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
    x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
    y = __shfl_xor_sync(0xffffffffu, y, 2) + 1.0;
  }
  if (x + y == 1.2345) out[threadIdx.x] = x;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s, %d SMs, clock %d MHz\n", prop.name, prop.multiProcessorCount, clk / 1000);
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms = prop.multiProcessorCount;
  for (int warps : {8, 16, 32}) {
    for (int mode = 0; mode < 3; ++mode) {
      const int blocks = sms * 2;
      dfma_kernel<<<blocks, 32 * warps>>>(out, 1.0000001, 1e-9, mode);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) dfma_kernel<<<blocks, 32 * warps>>>(out, 1.0000001, 1e-9, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      const double nthreads = static_cast<double>(blocks) * 32 * warps;
      double fma_warps = 0, mma_warps = 0;
      const double total_warps = nthreads / 32;
      if (mode == 0) fma_warps = total_warps;
      if (mode == 1) fma_warps = mma_warps = total_warps / 2;
      if (mode == 2) mma_warps = total_warps;
      // DFMA: 2 flop per lane per fma; DMMA m8n8k4: 2*8*8*4 = 512 flop per warp instruction
      const double fma_flop = fma_warps * 32 * 8.0 * ITERS * 2;
      const double mma_flop = mma_warps * 4.0 * (ITERS / 4) * 512;
      printf("warps/CTA %2d mode %d (%s): %.3f ms  DFMA %.2f TF/s  DMMA %.2f TF/s  total %.2f TF/s\n", warps, mode,
             mode == 0 ? "dfma" : mode == 1 ? "half/half" : "dmma", ms, fma_flop / ms / 1e9, mma_flop / ms / 1e9,
             (fma_flop + mma_flop) / ms / 1e9);
    }
  }
  {
    const int blocks = sms * 2, th = 1024;
    shfl_kernel<<<blocks, th>>>(out, 1.0);
    cudaEventRecord(e0);
    shfl_kernel<<<blocks, th>>>(out, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double shfl = 2.0 * 2 * ITERS * (blocks * th / 32.0);  // warp SHFL.32 instructions (2 per double)
    printf("shfl: %.3f ms, %.2f warp-SHFL/clk/SM (at %d MHz)\n", ms, shfl / (ms * 1e-3) / sms / (clk * 1e3),
           clk / 1000);
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
