// DFMA dependent-issue latency and single-warp throughput vs ILP on sm_100a
// (how many independent FP64 chains a warp needs to keep its SMSP's FP64
// pipe busy).  nvcc -arch=sm_100a -O3 -o /tmp/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chain(double* out, long long* cycles, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = a * (threadIdx.x + i + 1);
  constexpr int ITERS = 4096;
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; it += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = (t1 - t0);
}

template <int ILP>
void run(int warps, double* out, long long* cyc) {
  chain<ILP><<<148, 32 * warps>>>(out, cyc, 1.0000001, 1e-9);
  cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  printf("warps/SM %2d ILP %2d: %.2f cycles per dependent DFMA step, %.3f DFMA warp-instr/clk/SM\n", warps, ILP,
         c / 4096.0, warps * ILP * 4096.0 / c);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  for (int warps : {1, 4, 8, 16}) {
    run<1>(warps, out, cyc);
    run<2>(warps, out, cyc);
    run<4>(warps, out, cyc);
    run<8>(warps, out, cyc);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
