// A C++ host on the bare C-ABI (include/sfem_cuda.h + the CUDA runtime, no
// torch, no Python): (1) the slot-major batched line API with the reference's
// own arguments (lines::decompose_weighted_block / synthesize_block,
// eigenbasis.hpp:66-73) against the per-line entry, and (2) a slab solve whose
// exchange the library owns (NCCL communicator from a unique id, grouped
// ncclSend / ncclRecv inside sfem_cuda_dist_solve), one rank, against the
// single-GPU plan.  Built and run by tests/test_cpp_api.py (GPU).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "sfem_cuda.h"

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    if (cond) {                                                   \
      ++g_pass;                                                   \
    } else {                                                      \
      ++g_fail;                                                   \
      std::printf("FAIL %s:%d: %s (%s)\n", __FILE__, __LINE__, #cond, sfem_cuda_last_error()); \
    }                                                             \
  } while (0)
#define OK(call) CHECK((call) == 0)

static double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1));
}

template <class T>
static T* to_device(const std::vector<T>& v) {
  T* d = nullptr;
  cudaMalloc(&d, std::max<size_t>(v.size(), 1) * sizeof(T));
  cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return d;
}

static void block_api(sfem_ctx ctx, int n, int K, int count) {
  sfem_table t = nullptr;
  OK(sfem_cuda_table_create(ctx, n, K, &t));
  const int L = n * K - 1, m = n - 1;
  std::mt19937 rng(7u + n * 100 + K);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  // dof-layout lines and the same data as slot-major class tiles
  std::vector<double> lines(static_cast<size_t>(count) * L);
  for (auto& v : lines) v = u(rng);
  std::vector<double> nodal(static_cast<size_t>(K + 1) * count, 0.0), inter(static_cast<size_t>(K) * m * count, 0.0);
  for (int b = 0; b < count; ++b)
    for (int tt = 0; tt < L; ++tt) {
      const int e = tt / n, c = tt % n;
      const double v = lines[static_cast<size_t>(b) * L + tt];
      if (c == m) nodal[static_cast<size_t>(e + 1) * count + b] = v;
      else inter[static_cast<size_t>(e * m + c) * count + b] = v;
    }
  for (int b = 0; b < count; ++b) {  // boundary slots: ignored by the analyses
    nodal[b] = 3.0;
    nodal[static_cast<size_t>(K) * count + b] = -2.0;
  }
  std::vector<double> want(lines.size());
  OK(sfem_cuda_lines_host(t, SFEM_OP_DECOMPOSE_WEIGHTED, count, lines.data(), want.data()));
  double* dn = to_device(nodal);
  double* di = to_device(inter);
  double* dc = nullptr;
  cudaMalloc(&dc, lines.size() * sizeof(double));
  OK(sfem_cuda_lines_block_device(t, SFEM_OP_DECOMPOSE_WEIGHTED, count, dn, m ? di : nullptr, dc, nullptr));
  cudaDeviceSynchronize();
  std::vector<double> coef(lines.size()), got(lines.size());
  cudaMemcpy(coef.data(), dc, coef.size() * sizeof(double), cudaMemcpyDeviceToHost);
  for (int b = 0; b < count; ++b)
    for (int j = 0; j < L; ++j) got[static_cast<size_t>(b) * L + j] = coef[static_cast<size_t>(j) * count + b];
  CHECK(rel_l2(got, want) <= 1e-12);
  // synthesis of those coefficients back into class tiles = the input (F_n^-1 FC_n is not the
  // identity; compare with the per-line synthesis instead)
  std::vector<double> wsyn(lines.size());
  OK(sfem_cuda_lines_host(t, SFEM_OP_SYNTHESIZE, count, want.data(), wsyn.data()));
  cudaMemset(dn, 0xff, nodal.size() * sizeof(double));
  OK(sfem_cuda_lines_block_device(t, SFEM_OP_SYNTHESIZE, count, dn, m ? di : nullptr, dc, nullptr));
  cudaDeviceSynchronize();
  cudaMemcpy(nodal.data(), dn, nodal.size() * sizeof(double), cudaMemcpyDeviceToHost);
  cudaMemcpy(inter.data(), di, inter.size() * sizeof(double), cudaMemcpyDeviceToHost);
  std::vector<double> gsyn(lines.size());
  bool zero_bc = true;
  for (int b = 0; b < count; ++b) {
    zero_bc = zero_bc && nodal[b] == 0.0 && nodal[static_cast<size_t>(K) * count + b] == 0.0;
    for (int tt = 0; tt < L; ++tt) {
      const int e = tt / n, c = tt % n;
      gsyn[static_cast<size_t>(b) * L + tt] = c == m ? nodal[static_cast<size_t>(e + 1) * count + b]
                                                     : inter[static_cast<size_t>(e * m + c) * count + b];
    }
  }
  CHECK(zero_bc);
  CHECK(rel_l2(gsyn, wsyn) <= 1e-12);
  // element-stride entry on the slot-major dof tile, in place
  std::vector<double> tile(lines.size());
  for (int b = 0; b < count; ++b)
    for (int j = 0; j < L; ++j) tile[static_cast<size_t>(j) * count + b] = lines[static_cast<size_t>(b) * L + j];
  double* dt = to_device(tile);
  OK(sfem_cuda_lines_strided_device(t, SFEM_OP_DECOMPOSE_WEIGHTED, count, dt, dt, count, 1, nullptr));
  cudaDeviceSynchronize();
  cudaMemcpy(tile.data(), dt, tile.size() * sizeof(double), cudaMemcpyDeviceToHost);
  for (int b = 0; b < count; ++b)
    for (int j = 0; j < L; ++j) got[static_cast<size_t>(b) * L + j] = tile[static_cast<size_t>(j) * count + b];
  CHECK(rel_l2(got, want) <= 1e-12);
  CHECK(sfem_cuda_lines_strided_device(t, SFEM_OP_DECOMPOSE_WEIGHTED, count, dt, dt, count > 1 ? count - 1 : 0, 1,
                                       nullptr) != 0);
  cudaFree(dn);
  cudaFree(di);
  cudaFree(dc);
  cudaFree(dt);
  OK(sfem_cuda_table_destroy(t));
}

static void nccl_one_rank(sfem_ctx ctx, int dim, const int* orders, const int* elements, int chunks) {
  std::vector<double> lengths(dim, 1.0);
  const double shift = 0.5;
  sfem_plan plan = nullptr;
  OK(sfem_cuda_plan_create(ctx, dim, orders, elements, lengths.data(), nullptr, shift, &plan));
  long long ext[4], pitch = 0, unknowns = 0;
  OK(sfem_cuda_plan_shape(plan, ext, &pitch, &unknowns));
  std::mt19937 rng(11);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::vector<double> f(unknowns), want(unknowns);
  for (auto& v : f) v = u(rng);
  OK(sfem_cuda_solve_host(plan, f.data(), want.data(), nullptr));

  sfem_dist dist = nullptr;
  OK(sfem_cuda_dist_create(ctx, dim, orders, elements, lengths.data(), nullptr, shift, 1, 0, &dist));
  long long info[10], sc[1], rc[1];
  OK(sfem_cuda_dist_shape(dist, info, sc, rc));
  unsigned char id[SFEM_NCCL_UNIQUE_ID_BYTES];
  OK(sfem_cuda_nccl_unique_id(id));
  OK(sfem_cuda_dist_comm_init(dist, id, chunks));
  const long long xpitch = info[7], rows = unknowns / ext[dim - 1];
  double* dx = nullptr;
  cudaMalloc(&dx, info[4] * sizeof(double));
  cudaMemset(dx, 0, info[4] * sizeof(double));
  cudaMemcpy2D(dx, xpitch * sizeof(double), f.data(), ext[dim - 1] * sizeof(double), ext[dim - 1] * sizeof(double),
               rows, cudaMemcpyHostToDevice);
  OK(sfem_cuda_dist_solve(dist, dx, nullptr));
  double ms[6];
  long long sent = -1;
  OK(sfem_cuda_dist_solve_stats(dist, ms, &sent));
  std::vector<double> got(unknowns);
  cudaMemcpy2D(got.data(), ext[dim - 1] * sizeof(double), dx, xpitch * sizeof(double), ext[dim - 1] * sizeof(double),
               rows, cudaMemcpyDeviceToHost);
  CHECK(rel_l2(got, want) <= 1e-13);
  CHECK(sent == 0 && ms[5] > 0);
  std::printf("nccl one-rank solve dim %d: rel-L2 %.2e, %.3f ms (fwd %.3f, x1 %.3f, axis0 %.3f, x2 %.3f, inv %.3f)\n",
              dim, rel_l2(got, want), ms[5], ms[0], ms[1], ms[2], ms[3], ms[4]);
  cudaFree(dx);
  OK(sfem_cuda_dist_destroy(dist));
  OK(sfem_cuda_plan_destroy(plan));
}

int main() {
  sfem_ctx ctx = nullptr;
  if (sfem_cuda_ctx_create(0, &ctx) != 0) {
    std::printf("no context: %s\n", sfem_cuda_last_error());
    return 2;
  }
  block_api(ctx, 3, 8, 5);
  block_api(ctx, 9, 64, 32);
  block_api(ctx, 1, 16, 7);
  block_api(ctx, 4, 256, 9);
  {
    const int o[3] = {2, 3, 2}, e[3] = {16, 9, 5};
    nccl_one_rank(ctx, 3, o, e, 3);
  }
  {
    const int o[2] = {9, 9}, e[2] = {64, 64};
    nccl_one_rank(ctx, 2, o, e, 2);
  }
  OK(sfem_cuda_ctx_destroy(ctx));
  std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
