// C-ABI implementation (include/sfem_cuda.h): contexts, device tables, solve
// plans and the sweep schedule of algorithm (a).
//
// Schedule for an N-D solve on a dof tensor (reference run_full_diagonalization,
// poisson.cpp:637-669, which sweeps forward 0..N-1, divides, then inverts
// N-1..0):
//   forward sweeps along axes 0..N-2            (strided lines, tiles of B
//                                                 adjacent lines)
//   one fused sweep along the last axis:        forward + symbol divide +
//                                                 inverse, data never leaves
//                                                 shared memory in between
//   inverse sweeps along axes N-2..0
// = 2N-1 launches and 2N-1 passes over HBM instead of 2N.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only: the library is dlopen-ed (libnccl.so.2), never linked

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sfem_cuda.h"
#include "dist.cuh"
#include "banded.cuh"
#include "fem_ops.cuh"
#include "sweep.cuh"
#include "table.hpp"

using namespace sfem_b200;

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  } catch (...) {
    g_err = "unknown error";
    return 1;
  }
}

[[noreturn]] void fail(const std::string& msg) { throw std::runtime_error(msg); }
void require(bool c, const std::string& msg) {
  if (!c) fail(msg);
}

std::vector<int> factor_radices(int N) {
  std::vector<int> r;
  int m = N;
  while (m % 4 == 0) {
    r.push_back(4);
    m /= 4;
  }
  while (m % 2 == 0) {
    r.push_back(2);
    m /= 2;
  }
  for (int p = 3; m > 1; p += 2)
    while (m % p == 0) {
      r.push_back(p);
      m /= p;
    }
  return r;
}

constexpr size_t kSmemMax = 227 * 1024;

// SFEM_GENERIC=1 forces the generic shared-memory kernels (tests compare both).
bool fast_enabled() {
  const char* e = std::getenv("SFEM_GENERIC");
  return !(e && e[0] == '1');
}

}  // namespace

struct sfem_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  double* scratch = nullptr;
  size_t scratch_doubles = 0;
  // The scratch is shared by every plan and lines call of the context, each
  // on the caller's stream: the last user's stream and an event after its
  // launch order a user on another stream behind it (scratch_for/scratch_done).
  cudaEvent_t scratch_ev = nullptr;
  cudaStream_t scratch_stream = nullptr;
  bool scratch_pending = false;
  TableCache table_cache;  // TableSet's cache directory (poisson.cpp:49-73); empty = none
};

struct sfem_table_s {
  sfem_ctx ctx = nullptr;
  HostTable host;
  double* dbuf = nullptr;
  DevTable dev{};
};

namespace {

void upload_table(sfem_table_s* t) {
  const DeviceTableData d = derive_device_data(t->host);
  std::vector<const std::vector<double>*> parts = {&d.mix_fwd_w, &d.mix_fwd_d, &d.mix_inv, &d.e0_fwd_w,
                                                   &d.e0_fwd_d,  &d.e0_inv,    &d.eig,     &d.tw,
                                                   &d.mk,        &d.mkh,       &d.om,
                                                   &d.mixT_w,    &d.mixT_d,    &d.mixT_i,    &d.nsq};
  // k-contiguous per-(l, k) copies of the eigenvalues and norms (coefficient
  // order m + (k-1) n + l -> [l][k]): lanes over consecutive k read one line
  std::vector<double> eigT(static_cast<size_t>(d.n) * d.K, 0.0), nsqT(static_cast<size_t>(d.n) * d.K, 1.0);
  for (int k = 1; k < d.K; ++k)
    for (int l = 0; l < d.n; ++l) {
      eigT[static_cast<size_t>(l) * d.K + k] = d.eig[(d.n - 1) + static_cast<size_t>(k - 1) * d.n + l];
      nsqT[static_cast<size_t>(l) * d.K + k] = d.nsq[(d.n - 1) + static_cast<size_t>(k - 1) * d.n + l];
    }
  parts.push_back(&eigT);
  parts.push_back(&nsqT);
  std::vector<size_t> offs;
  size_t total = 0;
  for (size_t i = 0; i < parts.size(); ++i) {
    // the k-contiguous arrays (index k >= 1 used) start one double before a
    // 128-byte boundary: a warp's 16 consecutive frequencies k = 1 + 16 j ..
    // are one aligned line (two L1 tag requests per load otherwise)
    const bool kcont = i >= 11 && i != 14;
    if (kcont) total = ((total + 1 + 15) & ~static_cast<size_t>(15)) - 1;
    offs.push_back(total);
    total += (parts[i]->size() + 1) & ~static_cast<size_t>(1);  // keep 16-byte alignment
    if (kcont) total = (total + 1) & ~static_cast<size_t>(1);
  }
  std::vector<double> packed(total, 0.0);
  for (size_t i = 0; i < parts.size(); ++i)
    std::copy(parts[i]->begin(), parts[i]->end(), packed.begin() + offs[i]);
  ck(cudaSetDevice(t->ctx->device), "cudaSetDevice");
  ck(cudaMalloc(&t->dbuf, std::max<size_t>(total, 2) * sizeof(double)), "cudaMalloc(table)");
  ck(cudaMemcpy(t->dbuf, packed.data(), total * sizeof(double), cudaMemcpyHostToDevice), "upload table");
  DevTable& v = t->dev;
  v.n = d.n;
  v.K = d.K;
  v.m = d.n - 1;
  v.half = v.m / 2;
  v.ne = d.n / 2;
  v.L = d.n * d.K - 1;
  v.mix_fwd_w = t->dbuf + offs[0];
  v.mix_fwd_d = t->dbuf + offs[1];
  v.mix_inv = t->dbuf + offs[2];
  v.e0_fwd_w = t->dbuf + offs[3];
  v.e0_fwd_d = t->dbuf + offs[4];
  v.e0_inv = t->dbuf + offs[5];
  v.eig = t->dbuf + offs[6];
  v.tw = reinterpret_cast<const double2*>(t->dbuf + offs[7]);
  v.mk = reinterpret_cast<const double2*>(t->dbuf + offs[8]);
  v.mkh = reinterpret_cast<const double2*>(t->dbuf + offs[9]);
  v.om = reinterpret_cast<const double2*>(t->dbuf + offs[10]);
  v.mixT_w = t->dbuf + offs[11];
  v.mixT_d = t->dbuf + offs[12];
  v.mixT_i = t->dbuf + offs[13];
  v.nsq = t->dbuf + offs[14];
  v.eigT = t->dbuf + offs[15];
  v.nsqT = t->dbuf + offs[16];
  const std::vector<int> r = factor_radices(d.K);
  require(static_cast<int>(r.size()) <= kMaxPasses, "table: too many FFT passes");
  v.npass = static_cast<int>(r.size());
  for (size_t i = 0; i < r.size(); ++i) v.radix[i] = r[i];
}

// Largest tile (lines per CTA) that fits shared memory; prefer two CTAs/SM.
// Lines too long for any shared-memory tile keep one line per CTA in shared
// memory and move the FFT work buffers to global scratch (*gwork = true).
int choose_tile(const DevTable& t, long long nlines, bool* gwork = nullptr) {
  const int cands[] = {16, 8, 4, 2, 1};
  if (gwork) *gwork = false;
  for (int B : cands) {
    if (B > 1 && B > nlines) continue;
    if (sweep_smem_bytes(t, B) <= kSmemMax / 2) return B;
  }
  for (int B : cands) {
    if (B > 1 && B > nlines) continue;
    if (sweep_smem_bytes(t, B) <= kSmemMax) return B;
  }
  if (gwork && sweep_smem_bytes(t, 1, true) <= kSmemMax) {
    *gwork = true;
    return 1;
  }
  fail("sfem_cuda: line length " + std::to_string(t.L) + " (n=" + std::to_string(t.n) + ", K=" +
       std::to_string(t.K) + ") exceeds the shared-memory tile of this build");
}

struct Step {
  int axis;
  int mode;
  sfem_table_s* table = nullptr;  // table of the swept axis
  bool use_fast = true;
  LineSet ls;  // src/dst filled at launch
  int B;
  bool gwork = false;  // FFT work buffers in global scratch (long lines)
  SymbolInfo sym;
  // TMA description (strided steps): tensor map for the data pointer it was
  // encoded for, re-encoded when the pointer changes.
  bool tma = false;
  bool mid_tma = false;    // sweep_mid_tma (tile of box[0] lines)
  bool bulk_rows = false;  // fused last-axis sweep with per-row bulk copies
  TmaGeom geo{};
  cuuint64_t dims[4] = {1, 1, 1, 1}, strides[3] = {0, 0, 0};
  cuuint32_t box[4] = {0, 0, 0, 0};  // {0,..}: the plain box {8, boxp, 1, 1}
  const double* map_ptr = nullptr;
  alignas(64) CUtensorMap map;
  // out of place (blocked schedule): load from buffer src_buf, store through
  // smap into dst_buf (0 = the caller's tensor, 1 = the plan's blocked scratch)
  int src_buf = 0, dst_buf = 0;
  cuuint64_t sdims[4] = {1, 1, 1, 1}, sstrides[3] = {0, 0, 0};
  cuuint32_t sbox[4] = {0, 0, 0, 0};
  const double* smap_ptr = nullptr;
  alignas(64) CUtensorMap smap;
  // component-major mid tiles (mid_tma_cm): three 5-D maps (sweep.cuh)
  bool mid_cm = false;
  long long cm_st_pos = 0, cm_st_outer = 0, cm_ext_outer = 1;  // strides (elements) / extent of the 5-D view
  const double* cm_ptr = nullptr;
  alignas(64) CUtensorMap cm_maps[3];
};

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q), "cudaGetDriverEntryPoint");
    require(q == cudaDriverEntryPointSuccess && p != nullptr, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

void encode4(CUtensorMap* m, const double* data, const cuuint64_t* dims, const cuuint64_t* strides,
             const cuuint32_t* box_in, int boxp) {
  const cuuint32_t plain[4] = {8u, static_cast<cuuint32_t>(boxp), 1u, 1u};
  const cuuint32_t* box = box_in[0] ? box_in : plain;
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(data), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
}

// 5-D view {last axis, e >> 1, e & 1, s, outer} of position e * n + s of the swept axis
void encode5(CUtensorMap* m, const double* data, long long ext0, long long ext1, long long ext2, long long ext3,
             long long ext4, long long st_pos, long long st_outer, int n, const cuuint32_t* box) {
  const cuuint64_t dims[5] = {static_cast<cuuint64_t>(ext0), static_cast<cuuint64_t>(ext1), static_cast<cuuint64_t>(ext2),
                              static_cast<cuuint64_t>(ext3), static_cast<cuuint64_t>(ext4)};
  const cuuint64_t strides[4] = {static_cast<cuuint64_t>(2 * n * st_pos * 8), static_cast<cuuint64_t>(n * st_pos * 8),
                                 static_cast<cuuint64_t>(st_pos * 8), static_cast<cuuint64_t>(st_outer * 8)};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(data), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail("cuTensorMapEncodeTiled (5-D) failed (" + std::to_string(static_cast<int>(r)) + ")");
}

void encode_cm_maps(Step& s, const double* data) {
  if (s.cm_ptr == data) return;
  const int n = s.table->dev.n, K = s.table->dev.K;
  const long long e0 = static_cast<long long>(s.geo.ext0), eo = s.cm_ext_outer;
  const cuuint32_t boxA[5] = {8u, static_cast<cuuint32_t>(K / 2), 2u, static_cast<cuuint32_t>(n - 1), 1u};
  const cuuint32_t boxB[5] = {8u, static_cast<cuuint32_t>(K / 2), 1u, 1u, 1u};
  encode5(&s.cm_maps[0], data, e0, K / 2, 2, n, eo, s.cm_st_pos, s.cm_st_outer, n, boxA);
  encode5(&s.cm_maps[1], data, e0, K / 2, 2, n, eo, s.cm_st_pos, s.cm_st_outer, n, boxB);
  // odd elements of the last component: positions (2 e' + 1) n + n - 1, e' < K/2 - 1
  encode5(&s.cm_maps[2], data + (2 * n - 1) * s.cm_st_pos, e0, K / 2 - 1, 1, 1, eo, s.cm_st_pos, s.cm_st_outer, n, boxB);
  s.cm_ptr = data;
}

void encode_map(Step& s, const double* data) {
  if (s.map_ptr == data) return;
  encode4(&s.map, data, s.dims, s.strides, s.box, s.geo.boxp);
  s.map_ptr = data;
}

void encode_smap(Step& s, const double* data) {
  if (s.smap_ptr == data) return;
  encode4(&s.smap, data, s.sdims, s.sstrides, s.sbox, s.geo.boxp);
  s.smap_ptr = data;
}

}  // namespace

// Per-context scratch for global-work sweeps (grown on demand).  A caller on
// `stream` waits for the previous user's launch if that ran on another stream;
// growing it synchronises the device (the old buffer may be in use anywhere).
static double* scratch_for(sfem_ctx ctx, size_t doubles, cudaStream_t stream) {
  if (doubles > ctx->scratch_doubles) {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (ctx->scratch) {
      ck(cudaDeviceSynchronize(), "sync");
      ck(cudaFree(ctx->scratch), "cudaFree(scratch)");
    }
    ctx->scratch = nullptr;
    ctx->scratch_pending = false;
    ck(cudaMalloc(&ctx->scratch, doubles * sizeof(double)), "cudaMalloc(scratch)");
    ctx->scratch_doubles = doubles;
  }
  if (!ctx->scratch_ev) ck(cudaEventCreateWithFlags(&ctx->scratch_ev, cudaEventDisableTiming), "event");
  if (ctx->scratch_pending && ctx->scratch_stream != stream)
    ck(cudaStreamWaitEvent(stream, ctx->scratch_ev, 0), "scratch: wait for the previous user");
  return ctx->scratch;
}

// After a launch that used the scratch on `stream`.
static void scratch_done(sfem_ctx ctx, cudaStream_t stream) {
  ck(cudaEventRecord(ctx->scratch_ev, stream), "event");
  ctx->scratch_stream = stream;
  ctx->scratch_pending = true;
}

namespace {

// A local dof tensor the steps run on: extents (last axis padded to pitch),
// the table / symbol factor of each of its axes (eig_off shifts an axis's
// eigenvalue array for slabs that start at a global offset).
struct View {
  int N = 0;
  std::vector<long long> ext;
  long long pitch = 0;
  std::vector<sfem_table_s*> tables;
  std::vector<double> factors;
  std::vector<long long> eig_off;
  double shift = 0;
  bool use_fast = true;
  long long rows() const {
    long long r = 1;
    for (int i = 0; i < N - 1; ++i) r *= ext[i];
    return r;
  }
  std::vector<long long> strides() const {
    std::vector<long long> st(N);
    st[N - 1] = 1;
    if (N >= 2) st[N - 2] = pitch;
    for (int i = N - 3; i >= 0; --i) st[i] = st[i + 1] * ext[i + 1];
    return st;
  }
};

bool mid_tma_prefetch() {
  static const bool v = [] {
    const char* e = std::getenv("SFEM_MID_PREFETCH");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Sweep along strided axis a (a < N-1) of view v.
Step strided_step(const View& v, int a, int mode) {
  const int N = v.N;
  const std::vector<long long> st = v.strides();
  Step s{};
  s.axis = a;
  s.mode = mode;
  s.table = v.tables[a];
  s.use_fast = v.use_fast;
  LineSet& ls = s.ls;
  ls.ninner = v.ext[N - 1];
  ls.is = 1;
  std::vector<int> outer;
  for (int i = 0; i < N - 1; ++i)
    if (i != a) outer.push_back(i);
  ls.n1 = 1;
  ls.os1 = 0;
  ls.os2 = 0;
  if (outer.size() >= 1) {
    ls.n1 = v.ext[outer.back()];
    ls.os1 = st[outer.back()];
  }
  if (outer.size() == 2) ls.os2 = st[outer[0]];
  long long nl = ls.ninner;
  for (int i : outer) nl *= v.ext[i];
  ls.nlines = nl;
  ls.ps = st[a];
  ls.contiguous = 0;
  s.B = choose_tile(v.tables[a]->dev, nl, &s.gwork);
  const DevTable& dt = v.tables[a]->dev;
  if (v.use_fast && has_tma_sweep(dt.n, dt.K) && (v.pitch * 8) % 16 == 0) {
    s.tma = true;
    long long total_bytes = 8 * v.rows() * v.pitch;
    total_bytes = (total_bytes + 15) & ~15LL;
    s.dims[0] = v.ext[N - 1];
    s.dims[1] = v.ext[a];
    s.strides[0] = st[a] * 8;
    s.strides[1] = s.strides[2] = total_bytes;
    if (outer.size() >= 1) {
      s.dims[2] = v.ext[outer.back()];
      s.strides[1] = st[outer.back()] * 8;
    }
    if (outer.size() == 2) {
      s.dims[3] = v.ext[outer[0]];
      s.strides[2] = st[outer[0]] * 8;
    }
    s.geo.nbox = static_cast<int>((v.ext[a] + 255) / 256);
    s.geo.boxp = static_cast<int>((v.ext[a] + s.geo.nbox - 1) / s.geo.nbox);
    s.geo.nblk0 = (v.ext[N - 1] + 7) / 8;
    s.geo.ext0 = v.ext[N - 1];
    s.geo.ext2 = static_cast<long long>(s.dims[2]);
    s.geo.ntiles = s.geo.nblk0 * static_cast<long long>(s.dims[2]) * static_cast<long long>(s.dims[3]);
  } else if (v.use_fast && mid_tma_lines(dt.n, dt.K) > 0 && (v.pitch * 8) % 16 == 0 && v.ext[N - 1] >= 2) {
    // mid kernels: the same 4-D view, tiles of `tb` last-axis indices
    const int tb = mid_tma_lines(dt.n, dt.K);
    s.mid_tma = true;
    long long total_bytes = 8 * v.rows() * v.pitch;
    total_bytes = (total_bytes + 15) & ~15LL;
    s.dims[0] = v.ext[N - 1];
    s.dims[1] = v.ext[a];
    s.strides[0] = st[a] * 8;
    s.strides[1] = s.strides[2] = total_bytes;
    if (outer.size() >= 1) {
      s.dims[2] = v.ext[outer.back()];
      s.strides[1] = st[outer.back()] * 8;
    }
    if (outer.size() == 2) {
      s.dims[3] = v.ext[outer[0]];
      s.strides[2] = st[outer[0]] * 8;
    }
    s.geo.nbox = static_cast<int>((v.ext[a] + 255) / 256);
    s.geo.boxp = static_cast<int>((v.ext[a] + s.geo.nbox - 1) / s.geo.nbox);
    // boxes start 128-byte aligned in shared memory: boxp * tb a multiple of 16 doubles
    const int balign = tb % 16 == 0 ? 1 : (tb % 8 == 0 ? 2 : (tb % 4 == 0 ? 4 : (tb % 2 == 0 ? 8 : 16)));
    s.geo.boxp = (s.geo.boxp + balign - 1) / balign * balign;
    s.geo.nblk0 = (v.ext[N - 1] + tb - 1) / tb;
    s.geo.ext0 = v.ext[N - 1];
    s.geo.ext2 = static_cast<long long>(s.dims[2]);
    s.geo.ntiles = s.geo.nblk0 * static_cast<long long>(s.dims[2]) * static_cast<long long>(s.dims[3]);
    s.box[0] = static_cast<cuuint32_t>(tb);
    s.box[1] = static_cast<cuuint32_t>(s.geo.boxp);
    s.box[2] = s.box[3] = 1;
    // L2 prefetch one resident wave ahead where the tile's rows are close (<= 16 KB apart)
    s.geo.prefetch = (st[a] * 8 <= 16384 && mid_tma_prefetch()) ? 2 * 148 : 0;
    // component-major tiles: one outer axis at most (the 5-D view has no room for two)
    if (tb == 8 && outer.size() <= 1 && mid_tma_cm(dt.n, dt.K)) {
      s.mid_cm = true;
      s.cm_st_pos = st[a];
      s.cm_st_outer = outer.empty() ? static_cast<long long>(total_bytes / 8) : st[outer.back()];
      s.cm_ext_outer = outer.empty() ? 1 : v.ext[outer.back()];
    }
  }
  return s;
}

// Sweep along the last (contiguous) axis; mode kForwardDivideInverse fuses the
// symbol divide with the view's leading axes as the symbol's leading terms.
Step rows_step(const View& v, int mode) {
  const int N = v.N;
  Step s{};
  s.axis = N - 1;
  s.mode = mode;
  s.table = v.tables[N - 1];
  s.use_fast = v.use_fast;
  LineSet& ls = s.ls;
  ls.nlines = v.rows();
  ls.ninner = 1;
  ls.n1 = ls.nlines;
  ls.is = 0;
  ls.os1 = v.pitch;
  ls.os2 = 0;
  ls.ps = 1;
  ls.contiguous = 1;
  SymbolInfo& sy = s.sym;
  sy.nlead = N - 1;
  for (int i = 0; i < N - 1; ++i) {
    sy.lead_ext[i] = v.ext[i];
    sy.lead_eig[i] = v.tables[i]->dev.eig + v.eig_off[i];
    sy.lead_f[i] = v.factors[i];
  }
  sy.shift = v.shift;
  sy.f_last = v.factors[N - 1];
  s.B = choose_tile(v.tables[N - 1]->dev, ls.nlines, &s.gwork);
  const DevTable& dt = v.tables[N - 1]->dev;
  // bulk row copies move L rounded up to even doubles per row
  s.bulk_rows = v.use_fast && has_bulk_rows(dt.n, dt.K) && (v.pitch * 8) % 16 == 0 && ((dt.L + 1) & ~1) <= v.pitch;
  return s;
}

// Row sweeps with per-row bulk copies: the fused forward + divide + inverse
// runs the warp-local-job kernel (sweep_rows.cu) unless SFEM_ROWS_V1=1 selects
// the block-synchronous one (sweep_fast.cu sweep_bulk_rows, kept for A/B).
bool rows_v1() {
  const char* e = std::getenv("SFEM_ROWS_V1");
  return e && e[0] == '1';
}

cudaError_t launch_rows(const DevTable& dt, double* data, const RowSegs& rs, long long nrows, int mode,
                        const SymbolInfo& sym, cudaStream_t stream) {
  if (mode == kForwardDivideInverse && !rows_v1() && has_rows_fused(dt.n, dt.K))
    return launch_sweep_rows_fused(dt, data, rs, nrows, sym, stream);
  return launch_sweep_bulk_rows(dt, data, rs, nrows, mode, kWeighted, sym, stream);
}

// Launch a list of steps on `data` (in place).
void launch_steps(std::vector<Step>& steps, double* user, sfem_ctx ctx, cudaStream_t stream,
                  std::vector<cudaEvent_t>* kev, double* scratch = nullptr) {
  for (size_t i = 0; i < steps.size(); ++i) {
    Step& s = steps[i];
    double* data = s.src_buf ? scratch : user;
    double* dst = s.dst_buf ? scratch : user;
    s.ls.src = data;
    s.ls.dst = data;
    if (kev) ck(cudaEventRecord((*kev)[i], stream), "event");
    const DevTable& dt = s.table->dev;
    const SymbolInfo* sym = s.mode == kForwardDivideInverse ? &s.sym : nullptr;
    const bool aligned = (reinterpret_cast<unsigned long long>(data) % 16) == 0;
    if (s.tma && data != dst) {  // blocked schedule: out-of-place TMA sweep
      require(aligned && reinterpret_cast<unsigned long long>(dst) % 16 == 0, "blocked sweep: unaligned tensor");
      encode_map(s, data);
      encode_smap(s, dst);
      ck(launch_sweep_tma(dt, &s.map, &s.smap, s.geo, s.mode, kWeighted, stream), "tma sweep launch");
    } else if (s.tma && aligned) {
      encode_map(s, data);
      ck(launch_sweep_tma(dt, &s.map, nullptr, s.geo, s.mode, kWeighted, stream), "tma sweep launch");
    } else if (s.mid_tma && s.mid_cm && aligned) {
      encode_cm_maps(s, data);
      ck(launch_sweep_mid_tma_cm(dt, s.cm_maps, s.geo, s.mode, kWeighted, stream), "mid tma (component-major) sweep launch");
    } else if (s.mid_tma && aligned && (data != dst || s.geo.ld_mode != kBoxPlain)) {  // blocked schedule (mid)
      require(reinterpret_cast<unsigned long long>(dst) % 16 == 0, "blocked sweep: unaligned tensor");
      encode_map(s, data);
      if (data != dst) encode_smap(s, dst);
      ck(launch_sweep_mid_tma(dt, &s.map, s.geo, s.mode, kWeighted, stream, data != dst ? &s.smap : nullptr),
         "mid tma sweep launch (blocked)");
    } else if (s.mid_tma && aligned) {
      encode_map(s, data);
      ck(launch_sweep_mid_tma(dt, &s.map, s.geo, s.mode, kWeighted, stream), "mid tma sweep launch");
    } else if (s.bulk_rows && aligned) {
      RowSegs rs{};
      rs.n = 1;
      rs.pos0[0] = 0;
      rs.len[0] = static_cast<int>((dt.L + 1) & ~1);
      rs.off[0] = 0;
      rs.stride[0] = s.ls.os1;
      ck(launch_rows(dt, data, rs, s.ls.nlines, s.mode, s.sym, stream), "bulk rows sweep launch");
    } else if (s.use_fast && has_fast_sweep(dt.n, dt.K, s.mode, s.ls.contiguous)) {
      ck(launch_sweep_fast(dt, s.ls, s.mode, kWeighted, sym, stream), "fast sweep launch");
    } else if (s.use_fast && has_mid_sweep(dt.n, dt.K)) {
      const size_t wd = mid_work_doubles(dt.n, dt.K, s.ls.nlines);
      double* gw = wd ? scratch_for(ctx, wd, stream) : nullptr;
      ck(launch_sweep_mid(dt, s.ls, s.mode, kWeighted, sym, stream, gw), "mid sweep launch");
      if (gw) scratch_done(ctx, stream);
    } else {
      double* gw = nullptr;
      if (s.gwork) gw = scratch_for(ctx, sweep_work_doubles(dt, s.B) * ((s.ls.nlines + s.B - 1) / s.B), stream);
      ck(launch_sweep(dt, s.ls, s.mode, kWeighted, sym, s.B, stream, gw), "sweep launch");
      if (gw) scratch_done(ctx, stream);
    }
  }
  if (kev) ck(cudaEventRecord((*kev)[steps.size()], stream), "event");
}

}  // namespace

struct sfem_plan_s {
  sfem_ctx ctx = nullptr;
  int dim = 0;
  std::vector<int> orders, elements;
  std::vector<double> lengths, coeffs, factors;
  double shift = 0;
  std::vector<std::unique_ptr<sfem_table_s>> owned;
  std::vector<sfem_table_s*> tables;  // per axis
  std::vector<long long> ext;
  long long pitch = 0;        // the plan's own padded pitch (fixed at creation; sizes dwork / fbuf / dstage)
  long long steps_pitch = 0;  // the caller pitch `steps` were last built for
  long long rows = 0;  // product of leading extents
  std::vector<Step> steps;
  int algorithm = 0;            // 0: full diagonalisation (a), 1: partial (b)
  std::vector<Step> pfwd, pinv; // algorithm (b): forward / inverse sweeps of axes N-1 .. 1
  BandArgs band{};              // algorithm (b): the axis-0 line solves
  double* cbuf = nullptr;       // their Thomas coefficients
  size_t cbuf_cap = 0;          // doubles allocated in cbuf
  unsigned long long* dfail = nullptr;
  unsigned long long* hfail = nullptr;  // pinned copy of the failure flag
  bool blocked = false;         // 3-D blocked schedule (build_blocked_steps)
  double* bwork = nullptr;      // its scratch tensor [x_hi][L1][x_lo][bpitch]
  size_t belems = 0;
  size_t bwork_cap = 0;         // doubles allocated in bwork
  // plan-owned scratch (bwork, cbuf) is shared by solves on any stream: a
  // solve on another stream than the previous one waits for it
  cudaEvent_t busy_ev = nullptr;
  cudaStream_t busy_stream = nullptr;
  long long bpitch = 0;
  double* dwork = nullptr;
  double* dstage = nullptr;  // dense host-transfer staging
  // pipelined host solves (sfem_cuda_solve_host_batch): kSlots in-flight
  // problems, so the H2D of i+1 and the D2H of i-1 run during the solve of i
  static constexpr int kSlots = 3;
  double* pwork[kSlots] = {};
  double* pstage[kSlots] = {};
  cudaStream_t pin = nullptr, pout = nullptr;
  cudaEvent_t e_in[kSlots] = {}, e_comp[kSlots] = {}, e_out[kSlots] = {};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> kev;
  bool use_fast = true;
  // operator / residual scratch (P and Q tensors, padded) and reduction slots
  double* opwork[2] = {nullptr, nullptr};
  size_t opwork_cap[2] = {0, 0};  // doubles allocated per operator scratch tensor
  unsigned long long* dred = nullptr;
  double* fbuf = nullptr;      // device load of sfem_cuda_solve_field / operator output
  double* load_vec = nullptr;  // per-axis 1-D loads of separable fields
  size_t load_vec_cap = 0;
};

namespace {

View plan_view(const sfem_plan_s* p, long long pitch) {
  View v;
  v.N = p->dim;
  v.ext = p->ext;
  v.pitch = pitch;
  v.tables = p->tables;
  v.factors = p->factors;
  v.eig_off.assign(p->dim, 0);
  v.shift = p->shift;
  v.use_fast = p->use_fast;
  return v;
}

// Blocked schedule (3-D, TMA kernels on axes 0 and 1, bulk rows on axis 2):
// axis 0 is split x = x_hi*xblk + x_lo and stored in the plan's scratch as
// [x_hi][L1][x_lo][bpitch] (x_lo between y and z), so the axis-0 sweep reads
// groups of xblk 64-byte rows 8*bpitch bytes apart instead of 575 rows
// 2.65 MB apart (one DRAM page / TLB reach each; copy-only TMA time 0.98 ms
// vs 0.47 ms for axis 1, profiles/r1g_*).  Order: axis 1 forward
// (caller's tensor -> scratch), axis 0 forward (scratch, in place), fused
// axis 2 (scratch), axis 0 inverse, axis 1 inverse (scratch -> caller's).
constexpr int kXBlk = 8;

bool blocked_ok(const sfem_plan_s* p, long long pitch) {
  if (p->dim != 3 || !p->use_fast || std::getenv("SFEM_PLAIN")) return false;
  const DevTable& t0 = p->tables[0]->dev;
  const DevTable& t1 = p->tables[1]->dev;
  const DevTable& t2 = p->tables[2]->dev;
  const long long nhi = (p->ext[0] + kXBlk - 1) / kXBlk;
  return has_tma_sweep(t0.n, t0.K) && has_tma_sweep(t1.n, t1.K) && has_bulk_rows(t2.n, t2.K) &&
         kXBlk * nhi <= 576 && nhi <= 256 && (pitch * 8) % 16 == 0 && ((t2.L + 1) & ~1) <= pitch;
}

void build_blocked_steps(sfem_plan_s* p, long long pitch) {
  const long long L0 = p->ext[0], L1 = p->ext[1], L2 = p->ext[2];
  const long long bp = (L2 + 3) & ~3LL, X = kXBlk, nhi = (L0 + X - 1) / X;
  p->bpitch = bp;
  p->belems = static_cast<size_t>(nhi) * X * L1 * bp;
  const View v = plan_view(p, pitch);
  // blocked tensor strides (bytes): z 8, x_lo bp*8, y X*bp*8, x_hi L1*X*bp*8
  const cuuint64_t sxlo = bp * 8, sy = X * bp * 8, sxhi = L1 * X * bp * 8;
  auto axis1 = [&](int mode) {
    Step s = strided_step(v, 1, mode);  // plain geometry: d0 z, d1 y (swept), d2 x
    require(s.tma, "blocked schedule: axis-1 TMA step");
    // the blocked side: {z, y, x_lo, x_hi}, the tile's x split
    cuuint64_t* bd = mode == kForward ? s.sdims : s.dims;
    cuuint64_t* bs = mode == kForward ? s.sstrides : s.strides;
    const cuuint64_t pd[4] = {s.dims[0], s.dims[1], s.dims[2], s.dims[3]};
    const cuuint64_t ps[3] = {s.strides[0], s.strides[1], s.strides[2]};
    if (mode == kForward) {
      for (int i = 0; i < 4; ++i) s.dims[i] = pd[i];
      for (int i = 0; i < 3; ++i) s.strides[i] = ps[i];
    } else {
      for (int i = 0; i < 4; ++i) s.sdims[i] = pd[i];
      for (int i = 0; i < 3; ++i) s.sstrides[i] = ps[i];
    }
    bd[0] = L2;
    bd[1] = L1;
    bd[2] = X;
    bd[3] = nhi;
    bs[0] = sy;
    bs[1] = sxlo;
    bs[2] = sxhi;
    s.geo.xblk = X;
    s.geo.ld_mode = mode == kForward ? kBoxPlain : kBoxSplit;
    s.geo.st_mode = mode == kForward ? kBoxSplit : kBoxPlain;
    s.src_buf = mode == kForward ? 0 : 1;
    s.dst_buf = mode == kForward ? 1 : 0;
    return s;
  };
  auto axis0 = [&](int mode) {
    Step s = strided_step(v, 0, mode);  // table / line set of axis 0; geometry replaced
    require(s.tma, "blocked schedule: axis-0 TMA step");
    s.dims[0] = L2;
    s.dims[1] = X;
    s.dims[2] = nhi;
    s.dims[3] = L1;
    s.strides[0] = sxlo;
    s.strides[1] = sxhi;
    s.strides[2] = sy;
    s.box[0] = 8;
    s.box[1] = static_cast<cuuint32_t>(X);
    s.box[2] = static_cast<cuuint32_t>(nhi);
    s.box[3] = 1;
    s.geo.nbox = 1;
    s.geo.boxp = static_cast<int>(X * nhi);
    s.geo.nblk0 = (L2 + 7) / 8;
    s.geo.ext0 = L2;
    s.geo.ext2 = L1;
    s.geo.ntiles = s.geo.nblk0 * L1;
    s.geo.xblk = X;
    s.geo.ld_mode = s.geo.st_mode = kBoxSwept;
    s.src_buf = s.dst_buf = 1;
    return s;
  };
  Step rows = rows_step(v, kForwardDivideInverse);
  require(rows.bulk_rows, "blocked schedule: bulk-row step");
  rows.ls.nlines = nhi * L1 * X;
  rows.ls.n1 = rows.ls.nlines;
  rows.ls.os1 = bp;
  SymbolInfo& sy_ = rows.sym;
  sy_.nlead = 3;
  sy_.lead_ext[0] = nhi;
  sy_.lead_ext[1] = L1;
  sy_.lead_ext[2] = X;
  sy_.xblk = static_cast<int>(X);
  sy_.x_ext = L0;
  rows.src_buf = rows.dst_buf = 1;
  p->steps.clear();
  p->steps.push_back(axis1(kForward));
  p->steps.push_back(axis0(kForward));
  p->steps.push_back(rows);
  p->steps.push_back(axis0(kInverse));
  p->steps.push_back(axis1(kInverse));
  p->blocked = true;
}

// The same schedule for the mid kernels (sweep_mid_tma with box modes, sweep_mid rows with the blocked row
// order in the symbol): shapes mid_tma_blocked() names, all three axes on one table.
// rows per group of the blocked axis in the mid schedule (SFEM_MID_XBLK: A/B)
long long mid_xblk() {
  static const long long v = [] {
    const char* e = std::getenv("SFEM_MID_XBLK");
    const long long x = e ? std::atoll(e) : 0;
    return (x >= 2 && x <= 256) ? x : static_cast<long long>(kXBlk);
  }();
  return v;
}

bool blocked_mid_ok(const sfem_plan_s* p, long long pitch) {
  if (p->dim != 3 || !p->use_fast || std::getenv("SFEM_PLAIN")) return false;
  const DevTable& t0 = p->tables[0]->dev;
  if (p->tables[1] != p->tables[0] || p->tables[2] != p->tables[0]) return false;
  if (!mid_tma_blocked(t0.n, t0.K) || mid_tma_lines(t0.n, t0.K) <= 0 || mid_tma_cm(t0.n, t0.K)) return false;
  const long long nhi = (p->ext[0] + mid_xblk() - 1) / mid_xblk();
  const long long tb = mid_tma_lines(t0.n, t0.K), nbox = (p->ext[0] + 255) / 256;
  const long long balign = tb % 16 == 0 ? 1 : (tb % 8 == 0 ? 2 : (tb % 4 == 0 ? 4 : (tb % 2 == 0 ? 8 : 16)));
  const long long boxp = ((p->ext[0] + nbox - 1) / nbox + balign - 1) / balign * balign;  // as strided_step
  (void)nbox;
  (void)boxp;
  // one box {lines, xblk, nhi, 1} brings the swept axis (the launch checks that it fits the shared region)
  return nhi <= 256 && (pitch * 8) % 16 == 0 && p->ext[2] >= 2;
}

void build_blocked_mid_steps(sfem_plan_s* p, long long pitch) {
  const long long L0 = p->ext[0], L1 = p->ext[1], L2 = p->ext[2];
  const long long bp = (L2 + 3) & ~3LL, X = mid_xblk(), nhi = (L0 + X - 1) / X;
  p->bpitch = bp;
  p->belems = static_cast<size_t>(nhi) * X * L1 * bp;
  const View v = plan_view(p, pitch);
  const cuuint64_t sxlo = bp * 8, sy = X * bp * 8, sxhi = L1 * X * bp * 8;
  auto axis1 = [&](int mode) {
    Step s = strided_step(v, 1, mode);  // plain geometry: d0 z, d1 y (swept), d2 x
    require(s.mid_tma && !s.mid_cm, "blocked schedule (mid): axis-1 TMA step");
    for (int i = 0; i < 4; ++i) s.sdims[i] = s.dims[i], s.sbox[i] = s.box[i];
    for (int i = 0; i < 3; ++i) s.sstrides[i] = s.strides[i];
    // the blocked side: {z, y, x_lo, x_hi}, the tile's x split
    cuuint64_t* bd = mode == kForward ? s.sdims : s.dims;
    cuuint64_t* bs = mode == kForward ? s.sstrides : s.strides;
    bd[0] = L2;
    bd[1] = L1;
    bd[2] = X;
    bd[3] = nhi;
    bs[0] = sy;
    bs[1] = sxlo;
    bs[2] = sxhi;
    s.geo.xblk = X;
    s.geo.ld_mode = mode == kForward ? kBoxPlain : kBoxSplit;
    s.geo.st_mode = mode == kForward ? kBoxSplit : kBoxPlain;
    s.src_buf = mode == kForward ? 0 : 1;
    s.dst_buf = mode == kForward ? 1 : 0;
    return s;
  };
  auto axis0 = [&](int mode) {
    Step s = strided_step(v, 0, mode);  // table / line set of axis 0; geometry replaced
    require(s.mid_tma && !s.mid_cm, "blocked schedule (mid): axis-0 TMA step");
    const long long tb = s.box[0];
    s.dims[0] = L2;
    s.dims[1] = X;
    s.dims[2] = nhi;
    s.dims[3] = L1;
    s.strides[0] = sxlo;
    s.strides[1] = sxhi;
    s.strides[2] = sy;
    s.box[1] = static_cast<cuuint32_t>(X);
    s.box[2] = static_cast<cuuint32_t>(nhi);
    s.box[3] = 1;
    s.geo.nblk0 = (L2 + tb - 1) / tb;
    s.geo.ext0 = L2;
    s.geo.ext2 = L1;
    s.geo.ntiles = s.geo.nblk0 * L1;
    s.geo.xblk = X;
    s.geo.ld_mode = s.geo.st_mode = kBoxSwept;
    s.geo.prefetch = 0;
    s.src_buf = s.dst_buf = 1;
    return s;
  };
  Step rows = rows_step(v, kForwardDivideInverse);
  rows.ls.nlines = nhi * L1 * X;
  rows.ls.n1 = rows.ls.nlines;
  rows.ls.os1 = bp;
  rows.bulk_rows = false;
  SymbolInfo& sy_ = rows.sym;
  sy_.nlead = 3;
  sy_.lead_ext[0] = nhi;
  sy_.lead_ext[1] = L1;
  sy_.lead_ext[2] = X;
  sy_.xblk = static_cast<int>(X);
  sy_.x_ext = L0;
  rows.src_buf = rows.dst_buf = 1;
  p->steps.clear();
  p->steps.push_back(axis1(kForward));
  p->steps.push_back(axis0(kForward));
  p->steps.push_back(rows);
  p->steps.push_back(axis0(kInverse));
  p->steps.push_back(axis1(kInverse));
  p->blocked = true;
}

void build_steps(sfem_plan_s* p, long long pitch) {
  const int N = p->dim;
  p->blocked = false;
  if (blocked_ok(p, pitch)) {
    build_blocked_steps(p, pitch);
    return;
  }
  if (blocked_mid_ok(p, pitch)) {
    build_blocked_mid_steps(p, pitch);
    return;
  }
  const View v = plan_view(p, pitch);
  p->steps.clear();
  for (int a = 0; a < N - 1; ++a) p->steps.push_back(strided_step(v, a, kForward));
  p->steps.push_back(rows_step(v, kForwardDivideInverse));
  for (int a = N - 2; a >= 0; --a) p->steps.push_back(strided_step(v, a, kInverse));
}

// Algorithm (b) (poisson.cpp:671-745): forward expansions along axes N-1..1
// (the last axis as rows), the axis-0 line solves (banded.cu), inverse
// expansions along axes 1..N-1.
void build_partial_steps(sfem_plan_s* p, long long pitch) {
  const int N = p->dim;
  const View v = plan_view(p, pitch);
  p->pfwd.clear();
  p->pinv.clear();
  p->pfwd.push_back(rows_step(v, kForward));
  for (int a = N - 2; a >= 1; --a) p->pfwd.push_back(strided_step(v, a, kForward));
  for (int a = 1; a <= N - 2; ++a) p->pinv.push_back(strided_step(v, a, kInverse));
  p->pinv.push_back(rows_step(v, kInverse));
  BandArgs& b = p->band;
  b = BandArgs{};
  const HostTable& h = p->tables[0]->host;
  const int n = p->orders[0], np = n + 1, m = n - 1;
  b.n = n;
  b.K = p->elements[0];
  b.L = p->ext[0];
  std::vector<long long> st(N);
  st[N - 1] = 1;
  if (N >= 2) st[N - 2] = pitch;
  for (int i = N - 3; i >= 0; --i) st[i] = st[i + 1] * p->ext[i + 1];
  b.inner = st[0];
  b.outer = 1;
  b.pitch = pitch;
  b.last = p->ext[N - 1];
  b.f0 = p->factors[0];
  b.shift = p->shift;
  b.nfreq = N - 1;
  for (int i = 1; i < N; ++i) {
    b.fext[i - 1] = p->ext[i];
    b.eig[i - 1] = p->tables[i]->dev.eig;
    b.f[i - 1] = p->factors[i];
  }
  auto A = [&](int r, int c) { return h.stiffness[static_cast<size_t>(r) * np + c]; };
  auto C = [&](int r, int c) { return h.mass[static_cast<size_t>(r) * np + c]; };
  b.A00 = A(0, 0);
  b.A0n = A(0, n);
  b.C00 = C(0, 0);
  b.C0n = C(0, n);
  for (int l = 0; l < m; ++l) {
    b.lam[l] = h.interior_values[l];
    double pa0 = 0, pan = 0, pc0 = 0, pcn = 0;
    for (int c = 0; c < m; ++c) {
      const double vcl = h.interior_vectors[static_cast<size_t>(c) * m + l];
      b.V[c][l] = vcl;
      pa0 += vcl * A(1 + c, 0);
      pan += vcl * A(1 + c, n);
      pc0 += vcl * C(1 + c, 0);
      pcn += vcl * C(1 + c, n);
    }
    b.PA0[l] = pa0;
    b.PAn[l] = pan;
    b.PC0[l] = pc0;
    b.PCn[l] = pcn;
  }
}

// Grow a device buffer to at least `need` doubles (contents not kept).  The
// old buffer may still be read by work queued on `stream` or another stream,
// so the device is synchronised before it is freed (cold path: first use or a
// larger caller pitch).
void ensure_capacity(double*& buf, size_t& cap, size_t need, const char* what) {
  if (buf && cap >= need) return;
  if (buf) {
    ck(cudaDeviceSynchronize(), "sync before realloc");
    ck(cudaFree(buf), "cudaFree");
    buf = nullptr;
    cap = 0;
  }
  ck(cudaMalloc(&buf, std::max<size_t>(need, 1) * sizeof(double)), what);
  cap = need;
}

void run_partial(sfem_plan_s* p, double* data, long long pitch, cudaStream_t stream) {
  if (pitch != p->band.pitch || p->pfwd.empty()) build_partial_steps(p, pitch);
  const size_t lines = static_cast<size_t>(p->band.inner * p->band.outer);
  // the line count includes the caller's pitch: grow the coefficient scratch with it
  ensure_capacity(p->cbuf, p->cbuf_cap, static_cast<size_t>(p->band.K) * lines, "cudaMalloc(band scratch)");
  if (!p->dfail) {
    ck(cudaMalloc(&p->dfail, sizeof(unsigned long long)), "cudaMalloc(flag)");
    ck(cudaMallocHost(&p->hfail, sizeof(unsigned long long)), "cudaMallocHost(flag)");
  }
  ck(cudaMemsetAsync(p->dfail, 0xff, sizeof(unsigned long long), stream), "memset(flag)");
  launch_steps(p->pfwd, data, p->ctx, stream, nullptr);
  ck(launch_band_lines(data, p->cbuf, p->band, p->dfail, stream), "band line solves");
  ck(cudaMemcpyAsync(p->hfail, p->dfail, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream), "flag");
  launch_steps(p->pinv, data, p->ctx, stream, nullptr);
}

// After a synchronised algorithm-(b) solve: the reference's error for an
// indefinite line (poisson.cpp:720-725), with its line index r (row-major
// over the frequency extents of axes 1..N-1).
void check_partial(const sfem_plan_s* p) {
  if (p->algorithm != 1 || !p->hfail || *p->hfail == ~0ULL) return;
  long long rem = static_cast<long long>(*p->hfail), r = 0, mul = 1;
  double sigma = p->shift;
  const int N = p->dim;
  std::vector<long long> t(N, 0);
  for (int ax = N - 1; ax >= 1; --ax) {
    const long long ext = ax == N - 1 ? p->band.pitch : p->ext[ax];
    t[ax] = rem % ext;
    rem /= ext;
  }
  for (int ax = N - 1; ax >= 1; --ax) {
    r += t[ax] * mul;
    mul *= p->ext[ax];
    sigma += p->factors[ax] * p->tables[ax]->host.eig_coeff[t[ax]];
  }
  fail("solve: indefinite 1D system at transformed frequency " + std::to_string(r) + " (sigma " +
       std::to_string(sigma) + "); shift too negative");
}

void run_steps_impl(sfem_plan_s* p, double* data, long long pitch, cudaStream_t stream, bool events) {
  if (p->algorithm == 1) {
    run_partial(p, data, pitch, stream);
    return;
  }
  // Steps are rebuilt for a new caller pitch; p->pitch (the plan's own
  // padded pitch, which sizes dwork / fbuf / dstage) never changes.
  if (pitch != p->steps_pitch) build_steps(p, pitch), p->steps_pitch = pitch;
  if (p->blocked && p->bwork_cap < p->belems) {
    ensure_capacity(p->bwork, p->bwork_cap, p->belems, "cudaMalloc(blocked scratch)");
    ck(cudaMemsetAsync(p->bwork, 0, p->belems * sizeof(double), stream), "memset(blocked scratch)");
  }
  launch_steps(p->steps, data, p->ctx, stream, events ? &p->kev : nullptr, p->bwork);
}

void run_steps(sfem_plan_s* p, double* data, long long pitch, cudaStream_t stream, bool events) {
  if (!p->busy_ev) ck(cudaEventCreateWithFlags(&p->busy_ev, cudaEventDisableTiming), "event");
  if (p->busy_stream && p->busy_stream != stream)
    ck(cudaStreamWaitEvent(stream, p->busy_ev, 0), "plan: wait for the previous solve");
  run_steps_impl(p, data, pitch, stream, events);
  ck(cudaEventRecord(p->busy_ev, stream), "event");
  p->busy_stream = stream;
}

// Reference ProblemSpec::validate (poisson.cpp:32-47), with per-axis coefficients.
void validate(int dim, const int* orders, const int* elements, const double* lengths, const double* coeffs,
              double shift) {
  require(dim >= 1, "problem: dimension must be at least 1");
  require(dim <= kMaxDim, "problem: dimension above " + std::to_string(kMaxDim) + " is not supported by this build");
  double bound = 0;
  for (int i = 0; i < dim; ++i) {
    require(lengths[i] > 0, "problem: box length must be positive (axis " + std::to_string(i + 1) + ")");
    require(elements[i] >= 2, "problem: need at least 2 elements (axis " + std::to_string(i + 1) + ")");
    require(orders[i] >= 1 && orders[i] <= 9, "problem: order out of range (axis " + std::to_string(i + 1) + ")");
    const double a = coeffs ? coeffs[i] : 1.0;
    require(a > 0, "problem: diffusion coefficient must be positive (axis " + std::to_string(i + 1) + ")");
    bound += a / (lengths[i] * lengths[i]);
  }
  const double lower = -M_PI * M_PI * bound;
  if (!(shift > lower))
    fail("problem: shift " + std::to_string(shift) + " must exceed " + std::to_string(lower) +
         " for a positive definite operator");
}

// detail::scale_by_symbol's failure path (poisson.cpp:602-630): the first
// index in row-major order whose denominator is <= 0, decoded to (k, l).
void check_symbol(const sfem_plan_s* p) {
  const int N = p->dim;
  std::vector<double> mins(N);
  for (int i = 0; i < N; ++i) {
    const auto& e = p->tables[i]->host.eig_coeff;
    mins[i] = p->factors[i] * *std::min_element(e.begin(), e.end());
  }
  double total = p->shift;
  for (int i = 0; i < N; ++i) total += mins[i];
  if (total > 0) return;
  std::vector<int> idx(N, 0);
  double prefix = p->shift;
  for (int i = 0; i < N; ++i) {
    double tail = 0;
    for (int j = i + 1; j < N; ++j) tail += mins[j];
    const auto& e = p->tables[i]->host.eig_coeff;
    for (size_t t = 0; t < e.size(); ++t)
      if (prefix + p->factors[i] * e[t] + tail <= 0 || t + 1 == e.size()) {
        idx[i] = static_cast<int>(t);
        prefix += p->factors[i] * e[t];
        break;
      }
  }
  double denom = p->shift;
  std::string where;
  for (int i = 0; i < N; ++i) {
    denom += p->factors[i] * p->tables[i]->host.eig_coeff[idx[i]];
    const int n = p->orders[i];
    int k, l;
    if (idx[i] < n - 1) {
      k = 0;
      l = idx[i] + 1;
    } else {
      k = (idx[i] - (n - 1)) / n + 1;
      l = (idx[i] - (n - 1)) % n + 1;
    }
    where += (i ? ", " : "") + std::string("k") + std::to_string(i + 1) + "=" + std::to_string(k) + " l" +
             std::to_string(i + 1) + "=" + std::to_string(l);
  }
  fail("solve: nonpositive denominator " + std::to_string(denom) + " at (" + where + "); shift too negative");
}

void ensure_work(sfem_plan_s* p) {
  if (p->dwork) return;
  ck(cudaSetDevice(p->ctx->device), "cudaSetDevice");
  ck(cudaMalloc(&p->dwork, static_cast<size_t>(p->rows) * p->pitch * sizeof(double)), "cudaMalloc(work)");
}

double event_seconds(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  ck(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
  return ms * 1e-3;
}

// ---- class-array (GridFunctionND) <-> dof tensor on the host ----
// Mapping restated from the reference's oracle::pack_nd / unpack_nd
// (oracle.cpp:86-144).
template <bool TO_DOF>
void classes_dof(const sfem_plan_s* p, const double* const* cls_in, double* const* cls_out, const double* dof_in,
                 double* dof_out) {
  const int N = p->dim;
  std::vector<std::vector<long long>> cidx(N);
  std::vector<std::vector<unsigned char>> inter(N);
  for (int i = 0; i < N; ++i) {
    const int n = p->orders[i];
    cidx[i].resize(p->ext[i]);
    inter[i].resize(p->ext[i]);
    for (long long t = 0; t < p->ext[i]; ++t) {
      const long long r = t % n;
      if (r == n - 1) {
        inter[i][t] = 0;
        cidx[i][t] = t / n + 1;
      } else {
        inter[i][t] = 1;
        cidx[i][t] = (t / n) * (n - 1) + r;
      }
    }
  }
  const unsigned ncls = 1u << N;
  std::vector<std::vector<long long>> cstride(ncls, std::vector<long long>(N));
  for (unsigned mask = 0; mask < ncls; ++mask) {
    long long s = 1;
    for (int i = N - 1; i >= 0; --i) {
      cstride[mask][i] = s;
      const long long e = (mask >> i & 1u) ? static_cast<long long>(p->elements[i]) * (p->orders[i] - 1)
                                           : p->elements[i] + 1;
      s *= e;
    }
  }
  long long total = 1;
  for (int i = 0; i < N; ++i) total *= p->ext[i];
  const long long last = p->ext[N - 1];
#pragma omp parallel for schedule(static)
  for (long long row = 0; row < total / last; ++row) {
    std::vector<long long> idx(N, 0);
    long long rem = row;
    for (int i = N - 2; i >= 0; --i) {
      idx[i] = rem % p->ext[i];
      rem /= p->ext[i];
    }
    for (long long t = 0; t < last; ++t) {
      idx[N - 1] = t;
      unsigned mask = 0;
      for (int i = 0; i < N; ++i)
        if (inter[i][idx[i]]) mask |= 1u << i;
      long long off = 0;
      for (int i = 0; i < N; ++i) off += cidx[i][idx[i]] * cstride[mask][i];
      if (TO_DOF)
        dof_out[row * last + t] = cls_in[mask][off];
      else
        cls_out[mask][off] = dof_in[row * last + t];
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// Multi-GPU slab plan.  Rank r holds the x-slab of axis-0 rows
// [x0_r, x0_r + lx_r) (all other axes; last axis padded) and, between the two
// exchanges, the y-slab of axis-1 rows [y0_r, y0_r + ly_r) stored as
// [ly][R][P0] with axis 0 contiguous (R = prod of the extents of axes 2..N-1).
// ---------------------------------------------------------------------------
struct sfem_dist_s {
  sfem_ctx ctx = nullptr;
  int dim = 0, nranks = 1, rank = 0;
  std::vector<std::unique_ptr<sfem_table_s>> owned;
  std::vector<sfem_table_s*> tables;
  std::vector<long long> ext;
  std::vector<double> factors;
  double shift = 0;
  std::vector<long long> x0, lx, lxp, y0, ly;  // lxp: lx rounded up to even (exchange block pitch)
  long long R = 1, xpitch = 0, ypitch = 0;
  bool fused_y = false;  // AXIS0 runs on the exchange buffer in place (no UNPACK1 / PACK2)
  RowSegs ysegs{};
  View xv, yv;
  std::vector<Step> phaseA, phaseB, phaseC;
  SlabView sv{};
  // ---- library-owned solve (sfem_cuda_dist_solve): buffers, chunk schedule, communicator ----
  int C = 0;                                  // chunks per exchange (0 = not set up)
  std::vector<std::vector<long long>> xc0, xw;  // [rank][chunk]: chunk rows of that rank's x-slab (even starts)
  std::vector<std::vector<long long>> yc0, yw;  // [rank][chunk]: chunk rows of that rank's y range
  std::vector<std::vector<Step>> stepsA;      // forward local, per x-chunk
  std::vector<SlabView> svc;                  // slab transposes, per x-chunk
  std::vector<std::vector<Step>> stepsB;      // axis 0, per y-chunk (y-slab path)
  std::vector<RowSegs> segsB;                 // axis 0 in place on the exchange buffer, per y-chunk (K = 64 path)
  double *bufA = nullptr, *bufB = nullptr, *ybuf = nullptr;
  ncclComm_t comm = nullptr;
  cudaStream_t cs = nullptr;                  // exchange stream
  std::vector<cudaEvent_t> ev;                // 2C + 2 events
  double phase_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long bytes_sent = 0;                   // per solve, to other ranks (NVLink)
};

namespace {

// Axis-0 slabs: even sizes (pairs of rows split as evenly as possible), the
// odd remainder taken off the last non-empty slab, so every slab starts at an
// even row and every exchange block row (padded to lxp = lx rounded up to
// even) is a 16-byte multiple at a 16-byte offset.
std::vector<long long> balanced_even(long long n, int parts, std::vector<long long>& off) {
  const long long pairs = (n + 1) / 2;
  std::vector<long long> len(parts);
  off.assign(parts, 0);
  long long acc = 0;
  for (int r = 0; r < parts; ++r) {
    len[r] = 2 * (pairs / parts + (r < pairs % parts ? 1 : 0));
    off[r] = acc;
    acc += len[r];
  }
  if (acc > n)
    for (int r = parts - 1; r >= 0; --r)
      if (len[r] > 0) {
        len[r] -= acc - n;
        break;
      }
  return len;
}

std::vector<long long> balanced(long long n, int parts, std::vector<long long>& off) {
  std::vector<long long> len(parts);
  off.assign(parts, 0);
  long long acc = 0;
  for (int r = 0; r < parts; ++r) {
    len[r] = n / parts + (r < n % parts ? 1 : 0);
    off[r] = acc;
    acc += len[r];
  }
  return len;
}

}  // namespace

namespace {

int device_sms(int device) {
  int n = 0;
  ck(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device), "cudaDeviceGetAttribute");
  return n;
}

// Field description for the load / error kernels, validated against the plan.
FieldArgs make_field(const sfem_plan_s* p, int field, const double* params, int nparams) {
  FieldArgs fa{};
  fa.kind = field;
  fa.dim = p->dim;
  fa.shift = p->shift;
  auto unit_coeffs = [&] {
    for (double c : p->coeffs)
      require(c == 1.0, "fem_load: the manufactured cases are defined for unit coefficients (cases.cpp:81-95)");
  };
  switch (field) {
    case SFEM_FIELD_CONSTANT:
      require(params && nparams >= 1, "fem_load: CONSTANT needs params[0]");
      fa.p[0] = params[0];
      break;
    case SFEM_FIELD_SINES: {
      require(params && nparams >= 1 + p->dim, "fem_load: SINES needs amp and one wave number per axis");
      fa.p[0] = params[0];
      double denom = p->shift;
      for (int i = 0; i < p->dim; ++i) {
        fa.p[1 + i] = params[1 + i];
        const double k = params[1 + i] * M_PI;
        denom += p->coeffs[i] * k * k;
      }
      fa.p[1 + kMaxDim] = denom != 0.0 ? params[0] / denom : 0.0;
      break;
    }
    case SFEM_FIELD_SIN1D:
      require(p->dim == 1, "fem_load: case sin1d is 1-D");
      unit_coeffs();
      break;
    case SFEM_FIELD_POISSON2D:
      require(p->dim == 2, "fem_load: case poisson2d is 2-D");
      unit_coeffs();
      break;
    case SFEM_FIELD_POISSON3D:
      require(p->dim == 3, "fem_load: case poisson3d is 3-D");
      unit_coeffs();
      break;
    default:
      fail("fem_load: unknown field " + std::to_string(field));
  }
  return fa;
}

// dof-tensor strides (last axis padded to pitch)
std::vector<long long> dof_strides(const sfem_plan_s* p, long long pitch) {
  std::vector<long long> st(p->dim);
  st[p->dim - 1] = 1;
  if (p->dim >= 2) st[p->dim - 2] = pitch;
  for (int i = p->dim - 3; i >= 0; --i) st[i] = st[i + 1] * p->ext[i + 1];
  return st;
}

size_t padded_elems(const sfem_plan_s* p, long long pitch) { return static_cast<size_t>(p->rows) * pitch; }

// A v into q_out (or, with f, max|A v - f| and max|f| into p->dred): one sweep
// per axis 0..N-1 carrying P (scratch) and Q (q_out or scratch), fem_ops.cu.
void apply_sweeps(sfem_plan_s* p, const double* v, double* q_out, const double* f, long long pitch,
                  cudaStream_t s) {
  const size_t elems = padded_elems(p, pitch);
  const int nbuf = f ? 2 : 1;
  for (int b = 0; b < nbuf; ++b) ensure_capacity(p->opwork[b], p->opwork_cap[b], elems, "cudaMalloc(operator scratch)");
  double* P = p->opwork[0];
  double* Q = f ? p->opwork[1] : q_out;
  const std::vector<long long> st = dof_strides(p, pitch);
  const int N = p->dim;
  for (int a = 0; a < N; ++a) {
    OpAxisArgs A{};
    const HostTable& h = p->tables[a]->host;
    A.n = p->orders[a];
    A.K = p->elements[a];
    A.L = p->ext[a];
    A.pitch = pitch;
    A.last = p->ext[N - 1];
    A.fac = p->factors[a];
    A.shift = p->shift;
    const int np = A.n + 1;
    for (int r = 0; r < np; ++r)
      for (int c = 0; c < np; ++c) {
        A.M[r][c] = h.mass[static_cast<size_t>(r) * np + c];
        A.S[r][c] = h.stiffness[static_cast<size_t>(r) * np + c];
      }
    const bool rows = a == N - 1;
    A.outer = 1;
    for (int i = 0; i < (rows ? N - 1 : a); ++i) A.outer *= p->ext[i];
    A.inner = rows ? 1 : st[a];
    const bool first = a == 0, last = a == N - 1;
    ck(launch_op_axis(first ? v : P, P, Q, f, A, rows, first, last, f != nullptr && last, p->dred, s),
       "operator sweep");
  }
}

// 3-D tensor map {d0 = last axis (box 8), d1 (box b), d2 (box 1)} over `base`.
void encode_map3(CUtensorMap* m, void* base, long long e0, long long e1, long long e2, long long s1_bytes,
                 long long s2_bytes, int box1) {
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(e0), static_cast<cuuint64_t>(e1), static_cast<cuuint64_t>(e2)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(s1_bytes), static_cast<cuuint64_t>(s2_bytes)};
  const cuuint32_t box[3] = {8u, static_cast<cuuint32_t>(box1), 1u};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail("cuTensorMapEncodeTiled (peer map) failed (" + std::to_string(static_cast<int>(r)) + ")");
}

// boxes of at most 256 rows, even (128-byte aligned shared-memory starts)
void box_split(long long n, int& nbox, int& b) {
  nbox = static_cast<int>(std::max<long long>(1, (n + 255) / 256));
  b = static_cast<int>((n + nbox - 1) / nbox);
  b += b & 1;
  if (b > 256) {
    ++nbox;
    b = static_cast<int>((n + nbox - 1) / nbox);
    b += b & 1;
  }
}

double red_to_double(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
}

}  // namespace

// NVLink slab decomposition with the exchanges fused into the sweeps (3-D,
// K = 64 tables on axes 0 and 1).  Rank r owns the x-slab [L1][lx_r][pitch]
// (axis-0 rows x0_r.., laid out x, y, z) and the y-slab [ly_r][L0][pitch]
// (axis-1 rows y0_r.., laid out y, x, z).
struct sfem_peer_s {
  sfem_ctx ctx = nullptr;
  int dim = 0, nranks = 1, rank = 0;
  std::vector<std::unique_ptr<sfem_table_s>> owned;
  std::vector<sfem_table_s*> tables;
  std::vector<long long> ext;
  std::vector<double> factors;
  double shift = 0;
  std::vector<long long> x0, lx, y0, ly;
  long long pitch = 0, x_elems = 0, y_elems = 0;
  View xv, yv;
  std::vector<Step> fwd_rows, inv_local;
  Step fwd_y, axis0;
  double* xbuf = nullptr;
  double* ybuf = nullptr;
  unsigned long long* flags = nullptr;
  bool bound = false, device_barrier = false;
  ScatterMaps fwd_sc{}, ax_sc{};
  PeerFlags pf{};
  unsigned long long epoch = 0;
};

extern "C" {

int sfem_cuda_version(void) { return 100; }

const char* sfem_cuda_last_error(void) { return g_err.c_str(); }

int sfem_cuda_ctx_create(int device, sfem_ctx* out) {
  return guarded([&] {
    require(out != nullptr, "ctx_create: null output");
    int count = 0;
    ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    require(device >= 0 && device < count, "ctx_create: no CUDA device " + std::to_string(device));
    ck(cudaSetDevice(device), "cudaSetDevice");
    auto* c = new sfem_ctx_s;
    c->device = device;
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    *out = c;
  });
}

int sfem_cuda_ctx_destroy(sfem_ctx ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->scratch) cudaFree(ctx->scratch);
    if (ctx->scratch_ev) cudaEventDestroy(ctx->scratch_ev);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int sfem_cuda_ctx_stream(sfem_ctx ctx, void** stream) {
  return guarded([&] {
    require(ctx && stream, "ctx_stream: null argument");
    *stream = ctx->stream;
  });
}

int sfem_cuda_table_create(sfem_ctx ctx, int order, int elements, sfem_table* out) {
  return guarded([&] {
    require(ctx && out, "table_create: null argument");
    auto t = std::make_unique<sfem_table_s>();
    t->ctx = ctx;
    t->host = cached_host_table(ctx->table_cache, order, elements);
    upload_table(t.get());
    *out = t.release();
  });
}

int sfem_cuda_ctx_set_table_cache(sfem_ctx ctx, const char* dir, int flags) {
  return guarded([&] {
    require(ctx != nullptr, "set_table_cache: null context");
    require((flags & ~3) == 0, "set_table_cache: unknown flags");
    ctx->table_cache.dir = dir ? dir : "";
    ctx->table_cache.write = (flags & SFEM_TABLE_CACHE_WRITE) != 0;
    ctx->table_cache.format = (flags & SFEM_TABLE_CACHE_BINARY) ? kTableBinary : kTableText;
  });
}

int sfem_cuda_table_load(sfem_ctx ctx, const char* path, int order, int elements, sfem_table* out) {
  return guarded([&] {
    require(ctx && path && out, "table_load: null argument");
    auto t = std::make_unique<sfem_table_s>();
    t->ctx = ctx;
    t->host = load_host_table(path, order, elements);
    upload_table(t.get());
    *out = t.release();
  });
}

int sfem_cuda_table_save(sfem_table t, const char* path, int format) {
  return guarded([&] {
    require(t && path, "table_save: null argument");
    save_host_table(t->host, path, format);
  });
}

int sfem_cuda_table_file_build(int order, int elements, const char* path, int format) {
  return guarded([&] {
    require(path != nullptr, "build_and_save_table: null path");
    save_host_table(build_host_table(order, elements), path, format);
  });
}

int sfem_cuda_table_file_read(const char* path, int order, int elements, double* values, double* norm_sq,
                              double* p, double* interior_values, double* interior_vectors, double* eig_coeff) {
  return guarded([&] {
    require(path != nullptr, "load_table: null path");
    const HostTable h = load_host_table(path, order, elements);
    auto cp = [](const std::vector<double>& v, double* dst) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    cp(h.values, values);
    cp(h.norm_sq, norm_sq);
    cp(h.p, p);
    cp(h.interior_values, interior_values);
    cp(h.interior_vectors, interior_vectors);
    cp(h.eig_coeff, eig_coeff);
  });
}

int sfem_cuda_table_eigenvector(sfem_table t, int k, int l, double* out) {
  return guarded([&] {
    require(t && out, "materialize_eigenvector: null argument");
    const HostTable& h = t->host;
    const int n = h.order, K = h.elements, m = n - 1;
    require(k >= 0 && k < K, "materialize_eigenvector: frequency out of range");
    require(l >= 1 && l <= (k == 0 ? m : n), "materialize_eigenvector: branch out of range");
    // spectral.cpp:238-265, written in the dof layout (node j at j*n - 1,
    // interior i of element j-1 at (j-1)*n + i)
    const double pi = M_PI;
    std::fill(out, out + (static_cast<size_t>(n) * K - 1), 0.0);
    if (k == 0) {
      for (int j = 1; j <= K; ++j)
        for (int i = 0; i < m; ++i)
          out[static_cast<size_t>(j - 1) * n + i] =
              (j % 2 == 1) ? h.interior_vectors[static_cast<size_t>(i) * m + (l - 1)]
                           : -h.interior_vectors[static_cast<size_t>(m - 1 - i) * m + (l - 1)];
      return;
    }
    for (int j = 1; j < K; ++j) out[static_cast<size_t>(j) * n - 1] = std::sin(pi * k * j / static_cast<double>(K));
    const double* p = h.p.data() + (static_cast<size_t>(k - 1) * n + (l - 1)) * m;
    for (int j = 1; j <= K; ++j) {
      const double s_left = std::sin(pi * k * (j - 1) / static_cast<double>(K));
      const double s_right = std::sin(pi * k * j / static_cast<double>(K));
      for (int i = 0; i < m; ++i) out[static_cast<size_t>(j - 1) * n + i] = p[i] * s_left + p[m - 1 - i] * s_right;
    }
  });
}

int sfem_cuda_table_destroy(sfem_table t) {
  return guarded([&] {
    if (!t) return;
    if (t->dbuf) cudaFree(t->dbuf);
    delete t;
  });
}

int sfem_cuda_table_export(sfem_table t, double* values, double* norm_sq, double* p, double* interior_values,
                           double* interior_vectors, double* eig_coeff) {
  return guarded([&] {
    require(t != nullptr, "table_export: null table");
    auto cp = [](const std::vector<double>& v, double* dst) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    cp(t->host.values, values);
    cp(t->host.norm_sq, norm_sq);
    cp(t->host.p, p);
    cp(t->host.interior_values, interior_values);
    cp(t->host.interior_vectors, interior_vectors);
    cp(t->host.eig_coeff, eig_coeff);
  });
}

namespace {
// One line transform (op = SFEM_OP_DECOMPOSE_WEIGHTED / DECOMPOSE / SYNTHESIZE)
// over a LineSet with the fastest kernel compiled for the table.
void launch_lines(sfem_table t, const LineSet& ls, int op, cudaStream_t s) {
  const int mode = op == SFEM_OP_SYNTHESIZE ? kInverse : kForward;
  const int analysis = op == SFEM_OP_DECOMPOSE ? kDirect : kWeighted;
  const long long count = ls.nlines;
  if (fast_enabled() && has_fast_sweep(t->dev.n, t->dev.K, mode, ls.contiguous)) {
    ck(launch_sweep_fast(t->dev, ls, mode, analysis, nullptr, s), "lines launch (fast)");
  } else if (fast_enabled() && has_mid_sweep(t->dev.n, t->dev.K)) {
    const size_t wd = mid_work_doubles(t->dev.n, t->dev.K, count);
    double* gw = wd ? scratch_for(t->ctx, wd, s) : nullptr;
    ck(launch_sweep_mid(t->dev, ls, mode, analysis, nullptr, s, gw), "lines launch (mid)");
    if (gw) scratch_done(t->ctx, s);
  } else {
    bool gwork = false;
    const int B = choose_tile(t->dev, count, &gwork);
    double* gw = gwork ? scratch_for(t->ctx, sweep_work_doubles(t->dev, B) * ((count + B - 1) / B), s) : nullptr;
    ck(launch_sweep(t->dev, ls, mode, analysis, nullptr, B, s, gw), "lines launch");
    if (gw) scratch_done(t->ctx, s);
  }
}
}  // namespace

int sfem_cuda_lines_device(sfem_table t, int op, long long count, const double* d_in, long long in_pitch,
                           double* d_out, long long out_pitch, void* stream) {
  return guarded([&] {
    require(t != nullptr, "lines: null table");
    require(op >= 0 && op <= SFEM_OP_APPLY_STIFFNESS, "lines: unknown op");
    require(count >= 0, "lines: negative count");
    const long long L = t->dev.L;
    require(in_pitch >= L && out_pitch >= L, "lines: pitch smaller than the line length");
    if (count == 0) return;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->ctx->stream;
    ck(cudaSetDevice(t->ctx->device), "cudaSetDevice");
    const double* src = d_in;
    if (in_pitch != out_pitch) {
      ck(cudaMemcpy2DAsync(d_out, out_pitch * sizeof(double), d_in, in_pitch * sizeof(double), L * sizeof(double),
                           count, cudaMemcpyDeviceToDevice, s),
         "lines: repitch");
      src = d_out;
    }
    if (op == SFEM_OP_APPLY_MASS || op == SFEM_OP_APPLY_STIFFNESS) {
      // apply_mass_1d / apply_stiffness_1d (grid1d.cpp:33-47): the element
      // stencil as one operator sweep along the rows, y = shift M v + fac S v
      // with (shift, fac) = (1, 0) or (0, 1) (fem_ops.cu op_rows; in place).
      OpAxisArgs a{};
      const int np = t->dev.n + 1;
      a.n = t->dev.n;
      a.K = t->dev.K;
      a.L = L;
      a.outer = count;
      a.inner = 1;
      a.pitch = out_pitch;
      a.last = L;
      a.shift = op == SFEM_OP_APPLY_MASS ? 1.0 : 0.0;
      a.fac = op == SFEM_OP_APPLY_MASS ? 0.0 : 1.0;
      for (int r = 0; r < np; ++r)
        for (int c = 0; c < np; ++c) {
          a.M[r][c] = t->host.mass[static_cast<size_t>(r) * np + c];
          a.S[r][c] = t->host.stiffness[static_cast<size_t>(r) * np + c];
        }
      ck(launch_op_axis(src, nullptr, d_out, nullptr, a, true, true, true, false, nullptr, s), "lines: element stencil");
      return;
    }
    LineSet ls{};
    ls.src = src;
    ls.dst = d_out;
    ls.nlines = count;
    ls.ninner = 1;
    ls.n1 = count;
    ls.is = 0;
    ls.os1 = out_pitch;
    ls.os2 = 0;
    ls.ps = 1;
    ls.contiguous = 1;
    launch_lines(t, ls, op, s);
  });
}

int sfem_cuda_lines_strided_device(sfem_table t, int op, long long count, const double* d_in, double* d_out,
                                   long long pos_stride, long long line_stride, void* stream) {
  return guarded([&] {
    require(t != nullptr, "lines: null table");
    require(op >= SFEM_OP_DECOMPOSE_WEIGHTED && op <= SFEM_OP_SYNTHESIZE, "lines_strided: unknown op");
    require(count >= 0, "lines: negative count");
    require(d_in && d_out, "lines_strided: null buffer");
    require(pos_stride >= 1 && line_stride >= 1, "lines_strided: strides must be positive");
    const long long L = t->dev.L;
    // the (position, line) index map must be one-to-one
    require((pos_stride >= count * line_stride) || (line_stride >= L * pos_stride),
            "lines_strided: lines overlap (need pos_stride >= count*line_stride or line_stride >= L*pos_stride)");
    if (count == 0) return;
    if (pos_stride == 1) {  // rows: the line-major entry
      if (sfem_cuda_lines_device(t, op, count, d_in, line_stride, d_out, line_stride, stream) != 0)
        throw std::runtime_error(g_err);
      return;
    }
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->ctx->stream;
    ck(cudaSetDevice(t->ctx->device), "cudaSetDevice");
    LineSet ls{};
    ls.src = d_in;
    ls.dst = d_out;
    ls.nlines = count;
    ls.ninner = count;
    ls.n1 = 1;
    ls.is = line_stride;
    ls.os1 = 0;
    ls.os2 = 0;
    ls.ps = pos_stride;
    ls.contiguous = 0;
    launch_lines(t, ls, op, s);
  });
}

int sfem_cuda_lines_block_device(sfem_table t, int op, long long count, double* d_nodal, double* d_interior,
                                 double* d_coeffs, void* stream) {
  return guarded([&] {
    require(t != nullptr, "lines: null table");
    require(op >= SFEM_OP_DECOMPOSE_WEIGHTED && op <= SFEM_OP_SYNTHESIZE, "lines_block: unknown op");
    require(count >= 0, "lines: negative count");
    const int n = t->dev.n, K = t->dev.K;
    require(d_nodal && d_coeffs && (d_interior || n == 1), "lines_block: null tile");
    if (count == 0) return;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->ctx->stream;
    ck(cudaSetDevice(t->ctx->device), "cudaSetDevice");
    const long long L = t->dev.L;
    LineSet ls{};
    ls.nlines = count;
    ls.ninner = count;
    ls.n1 = 1;
    ls.is = 1;
    ls.os1 = 0;
    ls.os2 = 0;
    ls.ps = count;
    ls.contiguous = 0;
    if (op != SFEM_OP_SYNTHESIZE) {
      // class tiles -> dof tile (in the coefficient tile's storage: same shape), transformed in place
      ck(launch_class_tiles(n, K, count, d_nodal, d_interior, d_coeffs, true, s), "lines_block: gather");
      ls.src = d_coeffs;
      ls.dst = d_coeffs;
      launch_lines(t, ls, op, s);
    } else {
      // coefficients stay untouched: the sweep writes a temporary dof tile
      double* tmp = nullptr;
      ck(cudaMallocAsync(&tmp, static_cast<size_t>(L) * count * sizeof(double), s), "lines_block: cudaMallocAsync");
      ls.src = d_coeffs;
      ls.dst = tmp;
      try {
        launch_lines(t, ls, op, s);
        ck(launch_class_tiles(n, K, count, d_nodal, d_interior, tmp, false, s), "lines_block: scatter");
      } catch (...) {
        cudaFreeAsync(tmp, s);
        throw;
      }
      ck(cudaFreeAsync(tmp, s), "lines_block: cudaFreeAsync");
    }
  });
}

int sfem_cuda_lines_host(sfem_table t, int op, long long count, const double* h_in, double* h_out) {
  return guarded([&] {
    require(t != nullptr, "lines: null table");
    const long long L = t->dev.L;
    if (count == 0) return;
    ck(cudaSetDevice(t->ctx->device), "cudaSetDevice");
    cudaStream_t s = t->ctx->stream;
    double* d = nullptr;
    const size_t bytes = static_cast<size_t>(count) * L * sizeof(double);
    ck(cudaMallocAsync(&d, bytes, s), "cudaMallocAsync");
    ck(cudaMemcpyAsync(d, h_in, bytes, cudaMemcpyHostToDevice, s), "H2D");
    if (sfem_cuda_lines_device(t, op, count, d, L, d, L, s) != 0) {
      cudaFreeAsync(d, s);
      throw std::runtime_error(g_err);
    }
    ck(cudaMemcpyAsync(h_out, d, bytes, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaFreeAsync(d, s), "cudaFreeAsync");
    ck(cudaStreamSynchronize(s), "sync");
  });
}

int sfem_cuda_plan_create(sfem_ctx ctx, int dim, const int* orders, const int* elements, const double* lengths,
                          const double* coefficients, double shift, sfem_plan* out) {
  return guarded([&] {
    require(ctx && orders && elements && lengths && out, "plan_create: null argument");
    validate(dim, orders, elements, lengths, coefficients, shift);
    auto p = std::make_unique<sfem_plan_s>();
    p->ctx = ctx;
    p->dim = dim;
    p->orders.assign(orders, orders + dim);
    p->elements.assign(elements, elements + dim);
    p->lengths.assign(lengths, lengths + dim);
    p->coeffs.assign(dim, 1.0);
    if (coefficients) p->coeffs.assign(coefficients, coefficients + dim);
    p->shift = shift;
    p->use_fast = fast_enabled();
    std::map<std::pair<int, int>, sfem_table_s*> cache;
    for (int i = 0; i < dim; ++i) {
      const auto key = std::make_pair(orders[i], elements[i]);
      auto it = cache.find(key);
      if (it == cache.end()) {
        auto t = std::make_unique<sfem_table_s>();
        t->ctx = ctx;
        t->host = cached_host_table(ctx->table_cache, orders[i], elements[i]);
        upload_table(t.get());
        it = cache.emplace(key, t.get()).first;
        p->owned.push_back(std::move(t));
      }
      p->tables.push_back(it->second);
      // f_i = a_i * 4 / h_i^2 (axis_scale_factors, poisson.cpp:398-405)
      const double h = lengths[i] / elements[i];
      p->factors.push_back(p->coeffs[i] * (4.0 / (h * h)));
      p->ext.push_back(static_cast<long long>(orders[i]) * elements[i] - 1);
    }
    check_symbol(p.get());
    p->rows = 1;
    for (int i = 0; i < dim - 1; ++i) p->rows *= p->ext[i];
    const long long last = p->ext[dim - 1];
    p->pitch = (last + 3) & ~3LL;  // 32-byte rows
    build_steps(p.get(), p->pitch);
    p->steps_pitch = p->pitch;
    ck(cudaEventCreate(&p->ev[0]), "event");
    ck(cudaEventCreate(&p->ev[1]), "event");
    p->kev.resize(p->steps.size() + 1);
    for (auto& e : p->kev) ck(cudaEventCreate(&e), "event");
    *out = p.release();
  });
}

int sfem_cuda_plan_destroy(sfem_plan p) {
  return guarded([&] {
    if (!p) return;
    cudaSetDevice(p->ctx->device);
    if (p->dwork) cudaFree(p->dwork);
    if (p->bwork) cudaFree(p->bwork);
    if (p->busy_ev) cudaEventDestroy(p->busy_ev);
    if (p->cbuf) cudaFree(p->cbuf);
    if (p->dfail) cudaFree(p->dfail);
    if (p->hfail) cudaFreeHost(p->hfail);
    if (p->dstage) cudaFree(p->dstage);
    for (int b = 0; b < sfem_plan_s::kSlots; ++b) {
      if (p->pwork[b]) cudaFree(p->pwork[b]);
      if (p->pstage[b]) cudaFree(p->pstage[b]);
      if (p->e_in[b]) cudaEventDestroy(p->e_in[b]);
      if (p->e_comp[b]) cudaEventDestroy(p->e_comp[b]);
      if (p->e_out[b]) cudaEventDestroy(p->e_out[b]);
    }
    for (auto* w : p->opwork)
      if (w) cudaFree(w);
    if (p->dred) cudaFree(p->dred);
    if (p->load_vec) cudaFree(p->load_vec);
    if (p->fbuf) cudaFree(p->fbuf);
    if (p->pin) cudaStreamDestroy(p->pin);
    if (p->pout) cudaStreamDestroy(p->pout);
    for (auto& t : p->owned)
      if (t->dbuf) cudaFree(t->dbuf);
    for (auto e : p->ev)
      if (e) cudaEventDestroy(e);
    for (auto e : p->kev)
      if (e) cudaEventDestroy(e);
    delete p;
  });
}

int sfem_cuda_plan_shape(sfem_plan p, long long* extents, long long* pitch, long long* unknowns) {
  return guarded([&] {
    require(p != nullptr, "plan_shape: null plan");
    long long u = 1;
    for (int i = 0; i < p->dim; ++i) {
      if (extents) extents[i] = p->ext[i];
      u *= p->ext[i];
    }
    const long long last = p->ext[p->dim - 1];
    if (pitch) *pitch = (last + 3) & ~3LL;
    if (unknowns) *unknowns = u;
  });
}

int sfem_cuda_plan_launches(sfem_plan p, int* launches) {
  return guarded([&] {
    require(p && launches, "plan_launches: null argument");
    *launches = static_cast<int>(p->steps.size());
  });
}

int sfem_cuda_solve_device(sfem_plan p, double* d_data, long long pitch, void* stream) {
  return guarded([&] {
    require(p && d_data, "solve_device: null argument");
    require(pitch >= p->ext[p->dim - 1], "solve_device: pitch smaller than the last extent");
    ck(cudaSetDevice(p->ctx->device), "cudaSetDevice");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : p->ctx->stream;
    run_steps(p, d_data, pitch, s, false);
  });
}

int sfem_cuda_solve_host(sfem_plan p, const double* h_load, double* h_u, double* seconds) {
  return guarded([&] {
    require(p && h_load && h_u, "solve_host: null argument");
    ck(cudaSetDevice(p->ctx->device), "cudaSetDevice");
    // Host <-> device as dense 1-D copies (full PCIe rate), re-pitched on the
    // device into the padded (TMA-compatible) work tensor.
    const long long last = p->ext[p->dim - 1];
    const long long pitch = (last + 3) & ~3LL;
    ensure_work(p);
    cudaStream_t s = p->ctx->stream;
    const size_t dense = static_cast<size_t>(p->rows) * last;
    if (!p->dstage) ck(cudaMalloc(&p->dstage, dense * sizeof(double)), "cudaMalloc(stage)");
    double* stage = p->dstage;
    ck(cudaMemcpyAsync(stage, h_load, dense * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    ck(cudaMemcpy2DAsync(p->dwork, pitch * sizeof(double), stage, last * sizeof(double), last * sizeof(double),
                         p->rows, cudaMemcpyDeviceToDevice, s),
       "repitch");
    ck(cudaEventRecord(p->ev[0], s), "event");
    run_steps(p, p->dwork, pitch, s, false);
    ck(cudaEventRecord(p->ev[1], s), "event");
    ck(cudaMemcpy2DAsync(stage, last * sizeof(double), p->dwork, pitch * sizeof(double), last * sizeof(double),
                         p->rows, cudaMemcpyDeviceToDevice, s),
       "repitch");
    ck(cudaMemcpyAsync(h_u, stage, dense * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    check_partial(p);
    if (seconds) *seconds = event_seconds(p->ev[0], p->ev[1]);
  });
}

int sfem_cuda_solve_host_batch(sfem_plan p, long long count, const double* const* h_loads, double* const* h_us) {
  return guarded([&] {
    require(p && h_loads && h_us && count >= 0, "solve_host_batch: bad argument");
    ck(cudaSetDevice(p->ctx->device), "cudaSetDevice");
    const long long last = p->ext[p->dim - 1];
    const long long pitch = (last + 3) & ~3LL;
    const size_t dense = static_cast<size_t>(p->rows) * last;
    const size_t padded = static_cast<size_t>(p->rows) * pitch;
    if (!p->pin) {
      ck(cudaStreamCreateWithFlags(&p->pin, cudaStreamNonBlocking), "stream");
      ck(cudaStreamCreateWithFlags(&p->pout, cudaStreamNonBlocking), "stream");
      for (int b = 0; b < sfem_plan_s::kSlots; ++b) {
        ck(cudaMalloc(&p->pwork[b], padded * sizeof(double)), "cudaMalloc(work)");
        ck(cudaMalloc(&p->pstage[b], dense * sizeof(double)), "cudaMalloc(stage)");
        ck(cudaEventCreateWithFlags(&p->e_in[b], cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&p->e_comp[b], cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&p->e_out[b], cudaEventDisableTiming), "event");
        ck(cudaEventRecord(p->e_out[b], p->pout), "event");
      }
    }
    cudaStream_t sc = p->ctx->stream;
    // problem i uses slot b = i % kSlots: H2D of i+1 and D2H of i-1 overlap the
    // solve of i (three streams; PCIe moves both directions at once)
    for (long long i = 0; i < count; ++i) {
      const int b = static_cast<int>(i % sfem_plan_s::kSlots);
      ck(cudaStreamWaitEvent(p->pin, p->e_out[b], 0), "wait");
      ck(cudaMemcpyAsync(p->pstage[b], h_loads[i], dense * sizeof(double), cudaMemcpyHostToDevice, p->pin), "H2D");
      ck(cudaEventRecord(p->e_in[b], p->pin), "event");
      ck(cudaStreamWaitEvent(sc, p->e_in[b], 0), "wait");
      ck(cudaMemcpy2DAsync(p->pwork[b], pitch * sizeof(double), p->pstage[b], last * sizeof(double),
                           last * sizeof(double), p->rows, cudaMemcpyDeviceToDevice, sc),
         "repitch");
      run_steps(p, p->pwork[b], pitch, sc, false);
      ck(cudaMemcpy2DAsync(p->pstage[b], last * sizeof(double), p->pwork[b], pitch * sizeof(double),
                           last * sizeof(double), p->rows, cudaMemcpyDeviceToDevice, sc),
         "repitch");
      ck(cudaEventRecord(p->e_comp[b], sc), "event");
      ck(cudaStreamWaitEvent(p->pout, p->e_comp[b], 0), "wait");
      ck(cudaMemcpyAsync(h_us[i], p->pstage[b], dense * sizeof(double), cudaMemcpyDeviceToHost, p->pout), "D2H");
      ck(cudaEventRecord(p->e_out[b], p->pout), "event");
    }
    ck(cudaStreamSynchronize(p->pout), "sync");
    ck(cudaStreamSynchronize(sc), "sync");
  });
}

int sfem_cuda_solve_classes(sfem_plan p, const double* const* h_load_classes, double* const* h_u_classes,
                            double* seconds) {
  return guarded([&] {
    require(p && h_load_classes && h_u_classes, "solve_classes: null argument");
    long long total = 1;
    for (int i = 0; i < p->dim; ++i) total *= p->ext[i];
    std::vector<double> dof(static_cast<size_t>(total));
    classes_dof<true>(p, h_load_classes, nullptr, nullptr, dof.data());
    if (sfem_cuda_solve_host(p, dof.data(), dof.data(), seconds) != 0) throw std::runtime_error(g_err);
    // boundary slots (and anything not covered by a dof) are zero
    const unsigned ncls = 1u << p->dim;
    for (unsigned mask = 0; mask < ncls; ++mask) {
      long long sz = 1;
      for (int i = 0; i < p->dim; ++i)
        sz *= (mask >> i & 1u) ? static_cast<long long>(p->elements[i]) * (p->orders[i] - 1) : p->elements[i] + 1;
      std::fill(h_u_classes[mask], h_u_classes[mask] + sz, 0.0);
    }
    classes_dof<false>(p, nullptr, h_u_classes, dof.data(), nullptr);
  });
}

int sfem_cuda_solve_device_timed(sfem_plan p, double* d_data, long long pitch, int reps, double* total_ms,
                                 double* kernel_ms) {
  return guarded([&] {
    require(p && d_data && reps >= 1, "solve_device_timed: bad argument");
    ck(cudaSetDevice(p->ctx->device), "cudaSetDevice");
    cudaStream_t s = p->ctx->stream;
    if (p->algorithm == 1) {  // algorithm (b): whole-solve time only
      ck(cudaEventRecord(p->ev[0], s), "event");
      for (int r = 0; r < reps; ++r) run_steps(p, d_data, pitch, s, false);
      ck(cudaEventRecord(p->ev[1], s), "event");
      ck(cudaStreamSynchronize(s), "sync");
      if (total_ms) *total_ms = event_seconds(p->ev[0], p->ev[1]) * 1e3 / reps;
      if (kernel_ms)
        for (size_t i = 0; i < p->steps.size(); ++i) kernel_ms[i] = 0.0;
      return;
    }
    std::vector<double> acc(p->steps.size(), 0.0);
    double total = 0;
    for (int r = 0; r < reps; ++r) {
      run_steps(p, d_data, pitch, s, true);
      ck(cudaStreamSynchronize(s), "sync");
      for (size_t i = 0; i < p->steps.size(); ++i) acc[i] += event_seconds(p->kev[i], p->kev[i + 1]) * 1e3;
      total += event_seconds(p->kev[0], p->kev[p->steps.size()]) * 1e3;
    }
    if (total_ms) *total_ms = total / reps;
    if (kernel_ms)
      for (size_t i = 0; i < acc.size(); ++i) kernel_ms[i] = acc[i] / reps;
  });
}


int sfem_cuda_dist_create(sfem_ctx ctx, int dim, const int* orders, const int* elements, const double* lengths,
                          const double* coefficients, double shift, int nranks, int rank, sfem_dist* out) {
  return guarded([&] {
    require(ctx && orders && elements && lengths && out, "dist_create: null argument");
    require(dim >= 2, "dist_create: the slab decomposition needs dimension >= 2");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "dist_create: bad rank / nranks");
    validate(dim, orders, elements, lengths, coefficients, shift);
    auto d = std::make_unique<sfem_dist_s>();
    d->ctx = ctx;
    d->dim = dim;
    d->nranks = nranks;
    d->rank = rank;
    d->shift = shift;
    std::map<std::pair<int, int>, sfem_table_s*> cache;
    for (int i = 0; i < dim; ++i) {
      const auto key = std::make_pair(orders[i], elements[i]);
      auto it = cache.find(key);
      if (it == cache.end()) {
        auto t = std::make_unique<sfem_table_s>();
        t->ctx = ctx;
        t->host = cached_host_table(ctx->table_cache, orders[i], elements[i]);
        upload_table(t.get());
        it = cache.emplace(key, t.get()).first;
        d->owned.push_back(std::move(t));
      }
      d->tables.push_back(it->second);
      const double h = lengths[i] / elements[i];
      d->factors.push_back((coefficients ? coefficients[i] : 1.0) * (4.0 / (h * h)));
      d->ext.push_back(static_cast<long long>(orders[i]) * elements[i] - 1);
    }
    require(d->ext[0] >= nranks && d->ext[1] >= nranks, "dist_create: fewer slab rows than ranks");
    d->lx = balanced_even(d->ext[0], nranks, d->x0);
    d->ly = balanced(d->ext[1], nranks, d->y0);
    d->lxp.resize(nranks);
    for (int p = 0; p < nranks; ++p) d->lxp[p] = d->lx[p] + (d->lx[p] & 1);
    for (int i = 2; i < dim; ++i) d->R *= d->ext[i];
    d->xpitch = (d->ext[dim - 1] + 3) & ~3LL;
    d->ypitch = (d->ext[0] + 3) & ~3LL;
    const bool fast = fast_enabled();
    // x view: [lx][L1]..[L_{N-1}]
    View& xv = d->xv;
    xv.N = dim;
    xv.ext = d->ext;
    xv.ext[0] = d->lx[rank];
    xv.pitch = d->xpitch;
    xv.tables = d->tables;
    xv.factors = d->factors;
    xv.eig_off.assign(dim, 0);
    xv.shift = shift;
    xv.use_fast = fast;
    // y view: [ly][L2]..[L_{N-1}][L0] (axis 0 last, contiguous)
    View& yv = d->yv;
    yv.N = dim;
    yv.ext.clear();
    yv.tables.clear();
    yv.factors.clear();
    yv.eig_off.clear();
    for (int i = 1; i < dim; ++i) {
      yv.ext.push_back(i == 1 ? d->ly[rank] : d->ext[i]);
      yv.tables.push_back(d->tables[i]);
      yv.factors.push_back(d->factors[i]);
      yv.eig_off.push_back(i == 1 ? d->y0[rank] : 0);
    }
    yv.ext.push_back(d->ext[0]);
    yv.tables.push_back(d->tables[0]);
    yv.factors.push_back(d->factors[0]);
    yv.eig_off.push_back(0);
    yv.pitch = d->ypitch;
    yv.shift = shift;
    yv.use_fast = fast;
    // phase A: forward along axes N-1 (rows) and N-2..1 (strided) on the x-slab
    if (xv.ext[0] > 0) {
      d->phaseA.push_back(rows_step(xv, kForward));
      for (int a = dim - 2; a >= 1; --a) d->phaseA.push_back(strided_step(xv, a, kForward));
      for (int a = 1; a <= dim - 2; ++a) d->phaseC.push_back(strided_step(xv, a, kInverse));
      d->phaseC.push_back(rows_step(xv, kInverse));
    }
    // phase B: fused forward + divide + inverse along axis 0 on the y-slab, or
    // (K = 64 tables) straight on the source-major blocks of the exchange
    // buffer: row q of the y-slab is the concatenation over sources p of
    // buf[lyR * x0_p + q * lxp_p + (0 .. lxp_p)]
    if (yv.ext[0] > 0) d->phaseB.push_back(rows_step(yv, kForwardDivideInverse));
    {
      const long long lyR = d->ly[rank] * d->R;
      const DevTable& t0 = d->tables[0]->dev;
      d->fused_y = fast && nranks <= kMaxSeg && has_bulk_rows(t0.n, t0.K) && lyR > 0 && !d->phaseB.empty() &&
                   d->phaseB[0].bulk_rows;
      if (d->fused_y) {
        RowSegs& rs = d->ysegs;
        rs.n = 0;
        for (int p = 0; p < nranks; ++p) {
          if (d->lx[p] == 0) continue;
          rs.pos0[rs.n] = static_cast<int>(d->x0[p]);
          rs.len[rs.n] = static_cast<int>(d->lxp[p]);
          rs.off[rs.n] = lyR * d->x0[p];
          rs.stride[rs.n] = d->lxp[p];
          ++rs.n;
        }
      }
    }
    // transpose view of the x-slab
    const std::vector<long long> st = xv.strides();
    SlabView& sv = d->sv;
    sv.lx = d->lx[rank];
    sv.bpitch = d->lxp[rank];
    sv.R = d->R;
    sv.Q = d->ext[1] * d->R;
    sv.st0 = st[0];
    sv.st1 = st[1];
    sv.nrest = dim - 2;
    sv.st2 = dim >= 4 ? st[2] : 0;
    sv.e3 = dim >= 4 ? d->ext[3] : 1;
    require(dim <= 4, "dist_create: dimension above 4 is not supported by this build");
    *out = d.release();
  });
}

namespace {
void dist_teardown(sfem_dist_s* d);
}

int sfem_cuda_dist_destroy(sfem_dist d) {
  return guarded([&] {
    if (!d) return;
    cudaSetDevice(d->ctx->device);
    dist_teardown(d);
    for (auto& t : d->owned)
      if (t->dbuf) cudaFree(t->dbuf);
    delete d;
  });
}

int sfem_cuda_dist_shape(sfem_dist d, long long* info, long long* send_counts, long long* recv_counts) {
  return guarded([&] {
    require(d && info, "dist_shape: null argument");
    const int r = d->rank;
    info[0] = d->x0[r];
    info[1] = d->lx[r];
    info[2] = d->y0[r];
    info[3] = d->ly[r];
    info[4] = d->xv.rows() * d->xpitch;  // x-slab elements (padded)
    info[5] = d->fused_y ? 0 : d->ly[r] * d->R * d->ypitch;  // y-slab elements (unused when fused)
    long long sx = 0, rx = 0;
    for (int p = 0; p < d->nranks; ++p) {
      const long long sc = d->lxp[r] * d->ly[p] * d->R;  // exchange 1: to p (blocks [ly_p R][lxp_r])
      const long long rc = d->lxp[p] * d->ly[r] * d->R;  // exchange 1: from p
      if (send_counts) send_counts[p] = sc;
      if (recv_counts) recv_counts[p] = rc;
      sx += sc;
      rx += rc;
    }
    info[6] = std::max(sx, rx);  // exchange buffer elements (each direction)
    info[7] = d->xpitch;
    info[8] = d->ypitch;
    info[9] = d->R;
  });
}

int sfem_cuda_dist_phase(sfem_dist d, int phase, double* x, double* y, double* buf, void* stream) {
  return guarded([&] {
    require(d != nullptr, "dist_phase: null plan");
    ck(cudaSetDevice(d->ctx->device), "cudaSetDevice");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
    const int r = d->rank;
    const long long lyR = d->ly[r] * d->R;
    switch (phase) {
      case SFEM_DIST_FORWARD_LOCAL:
        launch_steps(d->phaseA, x, d->ctx, s, nullptr);
        break;
      case SFEM_DIST_PACK1:  // x-slab -> [L1*R][lx] (destination-major blocks)
        ck(launch_slab_transpose(d->sv, x, buf, true, s), "slab transpose");
        break;
      case SFEM_DIST_UNPACK1:  // blocks [ly*R][lxp_p] from each source p -> y rows, columns x0_p..
        if (d->fused_y) break;
        for (int p = 0; p < d->nranks; ++p) {
          if (d->lx[p] == 0 || lyR == 0) continue;
          ck(cudaMemcpy2DAsync(y + d->x0[p], d->ypitch * sizeof(double), buf + lyR * d->x0[p],
                               d->lxp[p] * sizeof(double), d->lx[p] * sizeof(double), lyR,
                               cudaMemcpyDeviceToDevice, s),
             "unpack1");
        }
        break;
      case SFEM_DIST_AXIS0:
        if (d->fused_y) {
          const Step& st = d->phaseB[0];
          ck(launch_rows(st.table->dev, buf, d->ysegs, lyR, kForwardDivideInverse, st.sym, s),
             "axis0 (exchange buffer)");
        } else {
          launch_steps(d->phaseB, y, d->ctx, s, nullptr);
        }
        break;
      case SFEM_DIST_PACK2:  // y rows, columns x0_p.. -> blocks [ly*R][lxp_p] for each destination p
        if (d->fused_y) break;
        for (int p = 0; p < d->nranks; ++p) {
          if (d->lx[p] == 0 || lyR == 0) continue;
          ck(cudaMemcpy2DAsync(buf + lyR * d->x0[p], d->lxp[p] * sizeof(double), y + d->x0[p],
                               d->ypitch * sizeof(double), d->lx[p] * sizeof(double), lyR,
                               cudaMemcpyDeviceToDevice, s),
             "pack2");
        }
        break;
      case SFEM_DIST_UNPACK2:  // [L1*R][lx] (source-major blocks) -> x-slab
        ck(launch_slab_transpose(d->sv, x, buf, false, s), "slab transpose");
        break;
      case SFEM_DIST_INVERSE_LOCAL:
        launch_steps(d->phaseC, x, d->ctx, s, nullptr);
        break;
      default:
        fail("dist_phase: unknown phase");
    }
  });
}


// ---------------------------------------------------------------------------
// Library-owned distributed solve: NCCL communicator, buffers and the chunked
// exchange schedule behind one call (sfem_cuda_dist_solve).
//
// Both exchanges are split into C chunks so that NVLink traffic overlaps the
// sweeps that produce it:
//   exchange 1: the x-slab is cut into C row chunks (even starts).  Chunk c is
//     swept forward (rows + strided axes 1..N-2), transposed into its part of
//     buffer A ([Q][wp_c] at A + Q*xc0_c, destination-major blocks) and handed
//     to the exchange stream, which sends it while chunk c+1 is swept.  The
//     receiver stores the block of (source s, chunk c) at
//     B + lyR*(x0_s + xc0_{s,c}): the y-slab row q is then the concatenation
//     of one segment per (source, chunk), which is what the axis-0 sweep reads
//     (RowSegs, K = 64 tables) or UNPACK1 copies into the y-slab.
//   exchange 2: the rank's y range is cut into C chunks; after the fused
//     axis-0 sweep of chunk c, its rows of every (destination, x-chunk) block
//     go back while chunk c+1 is swept.  They land in A where PACK1 read them.
// Messages between a pair of ranks are issued in the same order on both sides
// (x-chunk ascending), inside one ncclGroup per chunk.
// ---------------------------------------------------------------------------
namespace {

struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclGetVersion) GetVersion = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // a process that already loaded NCCL (torch) keeps its copy: same soname
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return a;
    auto sym = [&](const char* n) { return dlsym(a.h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.GetVersion = reinterpret_cast<decltype(a.GetVersion)>(sym("ncclGetVersion"));
    return a;
  }();
  require(api.h && api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
              api.GroupEnd,
          "NCCL: libnccl.so.2 could not be loaded (it is opened at run time; put it on the library path)");
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "error";
    fail(std::string("NCCL: ") + what + ": " + msg);
  }
}

long long even_up(long long v) { return v + (v & 1); }

// One message of an exchange chunk: `count` doubles at `off` of the local
// send (or receive) buffer, to (from) rank `peer`.
struct Msg {
  int peer;
  long long off, count;
};

// Exchange 1, x-chunk c: what rank r sends / receives.
void msgs1(const sfem_dist_s* d, int r, int c, std::vector<Msg>& sends, std::vector<Msg>& recvs) {
  const long long Q = d->ext[1] * d->R;
  sends.clear();
  recvs.clear();
  const long long w = d->xw[r][c], wp = even_up(w);
  for (int p = 0; p < d->nranks; ++p) {
    if (w > 0 && d->ly[p] > 0)
      sends.push_back({p, Q * d->xc0[r][c] + d->y0[p] * d->R * wp, d->ly[p] * d->R * wp});
    const long long ws = d->xw[p][c];
    if (ws > 0 && d->ly[r] > 0)
      recvs.push_back({p, d->ly[r] * d->R * (d->x0[p] + d->xc0[p][c]), d->ly[r] * d->R * even_up(ws)});
  }
}

// Exchange 2, y-chunk c of the sender: rank r's sends (from B, as the y-side
// rank) and receives (into A, as the x-side rank), x-chunk ascending per peer.
void msgs2(const sfem_dist_s* d, int r, int c, std::vector<Msg>& sends, std::vector<Msg>& recvs) {
  const long long Q = d->ext[1] * d->R;
  sends.clear();
  recvs.clear();
  const long long lyR = d->ly[r] * d->R;
  for (int p = 0; p < d->nranks; ++p)
    for (int cx = 0; cx < d->C; ++cx) {
      const long long wpp = even_up(d->xw[p][cx]);
      if (d->xw[p][cx] > 0 && d->yw[r][c] > 0)
        sends.push_back({p, lyR * (d->x0[p] + d->xc0[p][cx]) + d->yc0[r][c] * d->R * wpp, d->yw[r][c] * d->R * wpp});
      const long long wpr = even_up(d->xw[r][cx]);
      if (d->xw[r][cx] > 0 && d->yw[p][c] > 0)
        recvs.push_back({p, Q * d->xc0[r][cx] + (d->y0[p] + d->yc0[p][c]) * d->R * wpr, d->yw[p][c] * d->R * wpr});
    }
}

long long dist_buf_elems(const sfem_dist_s* d) {
  long long sx = 0, rx = 0;
  const int r = d->rank;
  for (int p = 0; p < d->nranks; ++p) {
    sx += d->lxp[r] * d->ly[p] * d->R;
    rx += d->lxp[p] * d->ly[r] * d->R;
  }
  return std::max<long long>(std::max(sx, rx), 2);
}

// Chunk schedule and plan-owned buffers (idempotent for the same C).
void dist_setup(sfem_dist_s* d, int chunks) {
  require(chunks >= 1 && chunks <= 16, "dist: chunks must be in 1..16");
  if (d->C == chunks) return;
  require(d->C == 0, "dist: the chunk count of a set-up plan cannot change");
  ck(cudaSetDevice(d->ctx->device), "cudaSetDevice");
  const int P = d->nranks, r = d->rank, dim = d->dim;
  int C = chunks;
  if (d->fused_y) {
    int nonempty = 0;
    for (int p = 0; p < P; ++p) nonempty += d->lx[p] > 0;
    while (C > 1 && nonempty * C > kMaxSeg) --C;
  }
  d->xc0.assign(P, {});
  d->xw.assign(P, {});
  d->yc0.assign(P, {});
  d->yw.assign(P, {});
  for (int p = 0; p < P; ++p) {
    d->xw[p] = balanced_even(d->lx[p], C, d->xc0[p]);
    d->yw[p] = balanced(d->ly[p], C, d->yc0[p]);
  }
  d->C = C;
  const std::vector<long long> st = d->xv.strides();
  d->stepsA.assign(C, {});
  d->svc.assign(C, SlabView{});
  for (int c = 0; c < C; ++c) {
    View v = d->xv;
    v.ext[0] = d->xw[r][c];
    if (v.ext[0] > 0) {
      d->stepsA[c].push_back(rows_step(v, kForward));
      for (int a = dim - 2; a >= 1; --a) d->stepsA[c].push_back(strided_step(v, a, kForward));
    }
    SlabView sv = d->sv;
    sv.lx = d->xw[r][c];
    sv.bpitch = even_up(sv.lx);
    d->svc[c] = sv;
  }
  d->stepsB.assign(C, {});
  d->segsB.assign(C, RowSegs{});
  const long long lyR = d->ly[r] * d->R;
  for (int c = 0; c < C; ++c) {
    if (d->yw[r][c] == 0) continue;
    if (d->fused_y) {
      RowSegs& rs = d->segsB[c];
      rs.n = 0;
      for (int p = 0; p < P; ++p)
        for (int cx = 0; cx < C; ++cx) {
          if (d->xw[p][cx] == 0) continue;
          const long long wp = even_up(d->xw[p][cx]);
          rs.pos0[rs.n] = static_cast<int>(d->x0[p] + d->xc0[p][cx]);
          rs.len[rs.n] = static_cast<int>(wp);
          rs.off[rs.n] = lyR * (d->x0[p] + d->xc0[p][cx]) + d->yc0[r][c] * d->R * wp;
          rs.stride[rs.n] = wp;
          ++rs.n;
        }
    }
    View v = d->yv;
    v.ext[0] = d->yw[r][c];
    v.eig_off[0] = d->y0[r] + d->yc0[r][c];
    d->stepsB[c].push_back(rows_step(v, kForwardDivideInverse));
  }
  const size_t nb = static_cast<size_t>(dist_buf_elems(d)) * sizeof(double);
  ck(cudaMalloc(&d->bufA, nb), "dist: cudaMalloc (exchange buffer A)");
  ck(cudaMalloc(&d->bufB, nb), "dist: cudaMalloc (exchange buffer B)");
  ck(cudaMemset(d->bufA, 0, nb), "dist: memset");
  ck(cudaMemset(d->bufB, 0, nb), "dist: memset");
  if (!d->fused_y && lyR > 0) {
    const size_t ny = static_cast<size_t>(lyR) * d->ypitch * sizeof(double);
    ck(cudaMalloc(&d->ybuf, ny), "dist: cudaMalloc (y-slab)");
    ck(cudaMemset(d->ybuf, 0, ny), "dist: memset");
  }
  ck(cudaStreamCreateWithFlags(&d->cs, cudaStreamNonBlocking), "dist: stream");
  d->ev.resize(2 * C + 8);
  for (auto& e : d->ev) ck(cudaEventCreate(&e), "dist: event");
  (void)st;
}

void dist_teardown(sfem_dist_s* d) {
  if (d->comm) {
    nccl().CommDestroy(d->comm);
    d->comm = nullptr;
  }
  for (auto& e : d->ev) cudaEventDestroy(e);
  d->ev.clear();
  if (d->cs) cudaStreamDestroy(d->cs);
  d->cs = nullptr;
  for (double** b : {&d->bufA, &d->bufB, &d->ybuf}) {
    if (*b) cudaFree(*b);
    *b = nullptr;
  }
}

// The compute of one rank between the exchanges, chunk by chunk (stream s).
void dist_forward_chunk(sfem_dist_s* d, double* x, int c, cudaStream_t s) {
  const int r = d->rank;
  if (d->xw[r][c] == 0) return;
  const long long st0 = d->xv.strides()[0];
  const long long Q = d->ext[1] * d->R;
  double* xc = x + d->xc0[r][c] * st0;
  launch_steps(d->stepsA[c], xc, d->ctx, s, nullptr);
  ck(launch_slab_transpose(d->svc[c], xc, d->bufA + Q * d->xc0[r][c], true, s), "slab transpose");
}

void dist_unpack1(sfem_dist_s* d, cudaStream_t s) {
  if (d->fused_y) return;
  const int r = d->rank;
  const long long lyR = d->ly[r] * d->R;
  if (lyR == 0) return;
  for (int p = 0; p < d->nranks; ++p)
    for (int cx = 0; cx < d->C; ++cx) {
      const long long w = d->xw[p][cx];
      if (w == 0) continue;
      const long long pos = d->x0[p] + d->xc0[p][cx];
      ck(cudaMemcpy2DAsync(d->ybuf + pos, d->ypitch * sizeof(double), d->bufB + lyR * pos,
                           even_up(w) * sizeof(double), w * sizeof(double), lyR, cudaMemcpyDeviceToDevice, s),
         "unpack1");
    }
}

void dist_axis0_chunk(sfem_dist_s* d, int c, cudaStream_t s) {
  const int r = d->rank;
  const long long nq = d->yw[r][c] * d->R;
  if (nq == 0) return;
  if (d->fused_y) {
    const Step& st = d->stepsB[c][0];
    ck(launch_rows(st.table->dev, d->bufB, d->segsB[c], nq, kForwardDivideInverse, st.sym, s),
       "axis0 (exchange buffer)");
    return;
  }
  const long long lyR = d->ly[r] * d->R;
  const long long q0 = d->yc0[r][c] * d->R;
  launch_steps(d->stepsB[c], d->ybuf + q0 * d->ypitch, d->ctx, s, nullptr);
  for (int p = 0; p < d->nranks; ++p)  // PACK2 of the chunk's rows
    for (int cx = 0; cx < d->C; ++cx) {
      const long long w = d->xw[p][cx];
      if (w == 0) continue;
      const long long pos = d->x0[p] + d->xc0[p][cx], wp = even_up(w);
      ck(cudaMemcpy2DAsync(d->bufB + lyR * pos + q0 * wp, wp * sizeof(double), d->ybuf + q0 * d->ypitch + pos,
                           d->ypitch * sizeof(double), w * sizeof(double), nq, cudaMemcpyDeviceToDevice, s),
         "pack2");
    }
}

void dist_inverse(sfem_dist_s* d, double* x, cudaStream_t s) {
  const int r = d->rank;
  const long long st0 = d->xv.strides()[0];
  const long long Q = d->ext[1] * d->R;
  for (int c = 0; c < d->C; ++c) {
    if (d->xw[r][c] == 0) continue;
    ck(launch_slab_transpose(d->svc[c], x + d->xc0[r][c] * st0, d->bufA + Q * d->xc0[r][c], false, s),
       "slab transpose");
  }
  launch_steps(d->phaseC, x, d->ctx, s, nullptr);
}

void nccl_exchange(sfem_dist_s* d, const std::vector<Msg>& sends, const double* sbuf, const std::vector<Msg>& recvs,
                   double* rbuf) {
  NcclApi& n = nccl();
  nck(n.GroupStart(), "ncclGroupStart");
  for (const Msg& m : sends)
    nck(n.Send(sbuf + m.off, static_cast<size_t>(m.count), ncclDouble, m.peer, d->comm, d->cs), "ncclSend");
  for (const Msg& m : recvs)
    nck(n.Recv(rbuf + m.off, static_cast<size_t>(m.count), ncclDouble, m.peer, d->comm, d->cs), "ncclRecv");
  nck(n.GroupEnd(), "ncclGroupEnd");
}

}  // namespace

int sfem_cuda_nccl_unique_id(void* id) {
  return guarded([&] {
    require(id != nullptr, "nccl_unique_id: null argument");
    static_assert(sizeof(ncclUniqueId) == SFEM_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    nck(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof u);
  });
}

int sfem_cuda_dist_setup(sfem_dist d, int chunks) {
  return guarded([&] {
    require(d != nullptr, "dist_setup: null plan");
    dist_setup(d, chunks > 0 ? chunks : 4);
  });
}

int sfem_cuda_dist_messages(sfem_dist d, int step, int chunk, int capacity, int* n_send, int* n_recv, int* peers,
                            long long* offsets, long long* counts) {
  return guarded([&] {
    require(d && n_send && n_recv, "dist_messages: null argument");
    require(d->C > 0, "dist_messages: plan not set up (sfem_cuda_dist_setup / dist_comm_init)");
    require((step == 1 || step == 2) && chunk >= 0 && chunk < d->C, "dist_messages: bad step / chunk");
    std::vector<Msg> sends, recvs;
    if (step == 1)
      msgs1(d, d->rank, chunk, sends, recvs);
    else
      msgs2(d, d->rank, chunk, sends, recvs);
    *n_send = static_cast<int>(sends.size());
    *n_recv = static_cast<int>(recvs.size());
    require(static_cast<int>(sends.size() + recvs.size()) <= capacity || !peers,
            "dist_messages: capacity too small");
    if (!peers || !offsets || !counts) return;
    int i = 0;
    for (const auto* list : {&sends, &recvs})
      for (const Msg& m : *list) {
        peers[i] = m.peer;
        offsets[i] = m.off;
        counts[i] = m.count;
        ++i;
      }
  });
}

int sfem_cuda_dist_comm_init(sfem_dist d, const void* id, int chunks) {
  return guarded([&] {
    require(d && id, "dist_comm_init: null argument");
    require(d->comm == nullptr, "dist_comm_init: the plan already has a communicator");
    dist_setup(d, chunks > 0 ? chunks : (d->C > 0 ? d->C : 4));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    nck(nccl().CommInitRank(&d->comm, d->nranks, u, d->rank), "ncclCommInitRank");
  });
}

int sfem_cuda_dist_solve(sfem_dist d, double* d_x, void* stream) {
  return guarded([&] {
    require(d && d->comm, "dist_solve: no communicator (call sfem_cuda_dist_comm_init first)");
    require(d_x != nullptr || d->lx[d->rank] == 0, "dist_solve: null x-slab");
    ck(cudaSetDevice(d->ctx->device), "cudaSetDevice");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
    const int C = d->C, r = d->rank;
    std::vector<Msg> sends, recvs;
    cudaEvent_t* ev = d->ev.data();
    cudaEvent_t *t0 = ev + 2 * C, *t1 = t0 + 1, *t2 = t0 + 2, *t3 = t0 + 3, *t4 = t0 + 4, *t5 = t0 + 5;
    long long sent = 0;
    ck(cudaEventRecord(*t0, s), "event");
    ck(cudaStreamWaitEvent(d->cs, *t0, 0), "wait");  // the exchange stream starts behind earlier work on s
    for (int c = 0; c < C; ++c) {
      dist_forward_chunk(d, d_x, c, s);
      ck(cudaEventRecord(ev[c], s), "event");
      ck(cudaStreamWaitEvent(d->cs, ev[c], 0), "wait");
      msgs1(d, r, c, sends, recvs);
      for (const Msg& m : sends) sent += m.peer != r ? m.count : 0;
      nccl_exchange(d, sends, d->bufA, recvs, d->bufB);
    }
    ck(cudaEventRecord(*t1, s), "event");  // forward compute done
    ck(cudaEventRecord(*t2, d->cs), "event");
    ck(cudaStreamWaitEvent(s, *t2, 0), "wait");  // exchange 1 complete
    dist_unpack1(d, s);
    for (int c = 0; c < C; ++c) {
      dist_axis0_chunk(d, c, s);
      ck(cudaEventRecord(ev[C + c], s), "event");
      ck(cudaStreamWaitEvent(d->cs, ev[C + c], 0), "wait");
      msgs2(d, r, c, sends, recvs);
      for (const Msg& m : sends) sent += m.peer != r ? m.count : 0;
      nccl_exchange(d, sends, d->bufB, recvs, d->bufA);
    }
    ck(cudaEventRecord(*t3, s), "event");  // axis-0 compute done
    ck(cudaEventRecord(*t4, d->cs), "event");
    ck(cudaStreamWaitEvent(s, *t4, 0), "wait");  // exchange 2 complete
    dist_inverse(d, d_x, s);
    ck(cudaEventRecord(*t5, s), "event");
    d->bytes_sent = sent * static_cast<long long>(sizeof(double));
  });
}

int sfem_cuda_dist_solve_stats(sfem_dist d, double* phase_ms, long long* bytes_sent) {
  return guarded([&] {
    require(d && d->C > 0 && d->ev.size() >= static_cast<size_t>(2 * d->C + 6), "dist_solve_stats: plan not set up");
    ck(cudaSetDevice(d->ctx->device), "cudaSetDevice");
    cudaEvent_t* t = d->ev.data() + 2 * d->C;
    ck(cudaEventSynchronize(t[5]), "event sync");
    auto ms = [&](int a, int b) {
      float v = 0;
      ck(cudaEventElapsedTime(&v, t[a], t[b]), "elapsed");
      return static_cast<double>(v);
    };
    if (phase_ms) {
      phase_ms[0] = ms(0, 1);  // forward local + pack (all chunks)
      phase_ms[1] = ms(1, 2);  // exchange 1 not hidden behind the forward sweeps
      phase_ms[2] = ms(2, 3);  // (unpack +) axis 0 (+ pack), all chunks
      phase_ms[3] = ms(3, 4);  // exchange 2 not hidden behind the axis-0 sweeps
      phase_ms[4] = ms(4, 5);  // unpack + inverse local
      phase_ms[5] = ms(0, 5);  // whole solve
    }
    if (bytes_sent) *bytes_sent = d->bytes_sent;
  });
}

// All ranks of a solve in one process on one device (the single-GPU check of
// the chunk schedule): same phases, chunks and message lists as
// sfem_cuda_dist_solve, the messages moved by device copies.  Messages of a
// pair are matched in issue order, as NCCL matches them.
int sfem_cuda_dist_solve_group(sfem_dist* ds, int n, double* const* d_xs, void* stream) {
  return guarded([&] {
    require(ds && d_xs && n >= 1, "dist_solve_group: null argument");
    for (int r = 0; r < n; ++r) {
      require(ds[r] && ds[r]->nranks == n && ds[r]->rank == r, "dist_solve_group: plans must be ranks 0..n-1 of n");
      require(ds[r]->C > 0 && ds[r]->C == ds[0]->C, "dist_solve_group: set the plans up with one chunk count");
      require(ds[r]->ctx->device == ds[0]->ctx->device, "dist_solve_group: one device");
    }
    ck(cudaSetDevice(ds[0]->ctx->device), "cudaSetDevice");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ds[0]->ctx->stream;
    const int C = ds[0]->C;
    std::vector<std::vector<Msg>> sends(n), recvs(n);
    auto exchange = [&](int step) {
      for (int dst = 0; dst < n; ++dst)
        for (int src = 0; src < n; ++src) {
          std::vector<const Msg*> out, in;
          for (const Msg& m : sends[src])
            if (m.peer == dst) out.push_back(&m);
          for (const Msg& m : recvs[dst])
            if (m.peer == src) in.push_back(&m);
          require(out.size() == in.size(), "dist_solve_group: send / receive lists disagree");
          for (size_t i = 0; i < out.size(); ++i) {
            require(out[i]->count == in[i]->count, "dist_solve_group: message sizes disagree");
            const double* sb = step == 1 ? ds[src]->bufA : ds[src]->bufB;
            double* rb = step == 1 ? ds[dst]->bufB : ds[dst]->bufA;
            ck(cudaMemcpyAsync(rb + in[i]->off, sb + out[i]->off, out[i]->count * sizeof(double),
                               cudaMemcpyDeviceToDevice, s),
               "dist_solve_group: copy");
          }
        }
    };
    for (int c = 0; c < C; ++c) {
      for (int r = 0; r < n; ++r) {
        dist_forward_chunk(ds[r], d_xs[r], c, s);
        msgs1(ds[r], r, c, sends[r], recvs[r]);
      }
      exchange(1);
    }
    for (int r = 0; r < n; ++r) dist_unpack1(ds[r], s);
    for (int c = 0; c < C; ++c) {
      for (int r = 0; r < n; ++r) {
        dist_axis0_chunk(ds[r], c, s);
        msgs2(ds[r], r, c, sends[r], recvs[r]);
      }
      exchange(2);
    }
    for (int r = 0; r < n; ++r) dist_inverse(ds[r], d_xs[r], s);
  });
}

int sfem_cuda_fem_load(sfem_plan p, int field, const double* params, int nparams, double* d_load, long long pitch,
                       void* stream) {
  return guarded([&] {
    require(p && d_load, "fem_load: null argument");
    require(pitch >= p->ext[p->dim - 1], "fem_load: pitch smaller than the last extent");
    ck(cudaSetDevice(p->ctx->device), "cudaSetDevice");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : p->ctx->stream;
    const FieldArgs fa = make_field(p, field, params, nparams);
    LoadArgs a{};
    a.dim = p->dim;
    const std::vector<long long> st = dof_strides(p, pitch);
    for (int i = 0; i < p->dim; ++i) {
      a.n[i] = p->orders[i];
      a.np[i] = p->orders[i] + 1;
      a.K[i] = p->elements[i];
      a.h[i] = p->lengths[i] / p->elements[i];
      a.ext[i] = p->ext[i];
      a.st[i] = st[i];
      std::vector<double> nodes, wq;
      load_quadrature(p->orders[i], nodes, wq);
      for (int g = 0; g <= p->orders[i]; ++g) a.gnode[i][g] = nodes[g];
      std::copy(wq.begin(), wq.end(), a.wq[i]);
    }
    if (field == SFEM_FIELD_CONSTANT || field == SFEM_FIELD_SINES) {
      // separable: per-axis assembled 1-D loads of g_i (1, or sin(k_i pi x)),
      // following the element loop of poisson.cpp:499-569 per axis
      SepArgs sa{};
      sa.dim = p->dim;
      sa.total = static_cast<long long>(padded_elems(p, pitch));
      sa.amp = fa.p[0];
      sa.pitch = pitch;
      std::vector<double> B;
      for (int i = 0; i < p->dim; ++i) {
        const int n = a.n[i], np = n + 1, K = a.K[i];
        sa.ext[i] = a.ext[i];
        sa.st[i] = a.st[i];
        sa.boff[i] = static_cast<long long>(B.size());
        B.resize(B.size() + a.ext[i], 0.0);
        double* Bi = B.data() + sa.boff[i];
        for (int e = 0; e < K; ++e)
          for (int loc = 0; loc <= n; ++loc) {
            const long long t = static_cast<long long>(e) * n - 1 + loc;
            if (t < 0 || t >= a.ext[i]) continue;
            double acc = 0;
            for (int g = 0; g < np; ++g) {
              const double x = (e + 0.5 * (a.gnode[i][g] + 1.0)) * a.h[i];
              const double gv = field == SFEM_FIELD_SINES ? std::sin(fa.p[1 + i] * M_PI * x) : 1.0;
              acc += a.wq[i][loc * np + g] * gv;
            }
            Bi[t] += acc;
          }
      }
      if (B.size() > p->load_vec_cap) {
        if (p->load_vec) ck(cudaFree(p->load_vec), "cudaFree");
        p->load_vec = nullptr;
        ck(cudaMalloc(&p->load_vec, B.size() * sizeof(double)), "cudaMalloc(load vectors)");
        p->load_vec_cap = B.size();
      }
      ck(cudaMemcpyAsync(p->load_vec, B.data(), B.size() * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
      ck(launch_fem_load_separable(d_load, p->load_vec, sa, device_sms(p->ctx->device), s), "fem_load kernel");
      ck(cudaStreamSynchronize(s), "sync");  // B (host) is released on return
      return;
    }
    ck(cudaMemsetAsync(d_load, 0, padded_elems(p, pitch) * sizeof(double), s), "memset(load)");
    ck(launch_fem_load(d_load, a, fa, device_sms(p->ctx->device), s), "fem_load kernel");
  });
}

int sfem_cuda_apply_operator(sfem_plan p, const double* d_v, double* d_y, long long pitch, void* stream) {
  return guarded([&] {
    require(p && d_v && d_y, "apply_operator: null argument");
    require(d_v != d_y, "apply_operator: v and y must be distinct");
    require(pitch >= p->ext[p->dim - 1], "apply_operator: pitch smaller than the last extent");
    ck(cudaSetDevice(p->ctx->device), "cudaSetDevice");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : p->ctx->stream;
    apply_sweeps(p, d_v, d_y, nullptr, pitch, s);
  });
}

int sfem_cuda_residual(sfem_plan p, const double* d_u, const double* d_f, long long pitch, double* residual_rel) {
  return guarded([&] {
    require(p && d_u && d_f && residual_rel, "residual: null argument");
    require(pitch >= p->ext[p->dim - 1], "residual: pitch smaller than the last extent");
    ck(cudaSetDevice(p->ctx->device), "cudaSetDevice");
    cudaStream_t s = p->ctx->stream;
    if (!p->dred) ck(cudaMalloc(&p->dred, 2 * sizeof(unsigned long long)), "cudaMalloc(reduction)");
    ck(cudaMemsetAsync(p->dred, 0, 2 * sizeof(unsigned long long), s), "memset");
    apply_sweeps(p, d_u, nullptr, d_f, pitch, s);
    unsigned long long h[2];
    ck(cudaMemcpyAsync(h, p->dred, sizeof h, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    const double num = red_to_double(h[0]), den = red_to_double(h[1]);
    *residual_rel = num / (den > 0 ? den : 1.0);  // poisson.cpp:786-788
  });
}

int sfem_cuda_max_error(sfem_plan p, int field, const double* params, int nparams, const double* d_u, long long pitch,
                        double* error) {
  return guarded([&] {
    require(p && d_u && error, "max_error: null argument");
    require(field != SFEM_FIELD_CONSTANT, "max_error: the CONSTANT field has no closed-form solution");
    ck(cudaSetDevice(p->ctx->device), "cudaSetDevice");
    cudaStream_t s = p->ctx->stream;
    const FieldArgs fa = make_field(p, field, params, nparams);
    ErrArgs a{};
    a.dim = p->dim;
    a.total = 1;
    const std::vector<long long> st = dof_strides(p, pitch);
    for (int i = 0; i < p->dim; ++i) {
      a.n[i] = p->orders[i];
      a.ext[i] = p->ext[i];
      a.st[i] = st[i];
      a.h[i] = p->lengths[i] / p->elements[i];
      a.total *= p->ext[i];
    }
    if (!p->dred) ck(cudaMalloc(&p->dred, 2 * sizeof(unsigned long long)), "cudaMalloc(reduction)");
    ck(cudaMemsetAsync(p->dred, 0, 2 * sizeof(unsigned long long), s), "memset");
    ck(launch_max_error(d_u, a, fa, p->dred, device_sms(p->ctx->device), s), "max_error kernel");
    unsigned long long h[2];
    ck(cudaMemcpyAsync(h, p->dred, sizeof h, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    *error = red_to_double(h[0]);
  });
}


int sfem_cuda_peer_create(sfem_ctx ctx, int dim, const int* orders, const int* elements, const double* lengths,
                          const double* coefficients, double shift, int nranks, int rank, sfem_peer* out) {
  return guarded([&] {
    require(ctx && orders && elements && lengths && out, "peer_create: null argument");
    require(dim == 3, "peer_create: the fused NVLink decomposition is 3-D");
    require(nranks >= 1 && nranks <= kMaxPeer && rank >= 0 && rank < nranks, "peer_create: bad rank / nranks");
    validate(dim, orders, elements, lengths, coefficients, shift);
    auto d = std::make_unique<sfem_peer_s>();
    d->ctx = ctx;
    d->dim = dim;
    d->nranks = nranks;
    d->rank = rank;
    d->shift = shift;
    std::map<std::pair<int, int>, sfem_table_s*> cache;
    for (int i = 0; i < dim; ++i) {
      const auto key = std::make_pair(orders[i], elements[i]);
      auto it = cache.find(key);
      if (it == cache.end()) {
        auto t = std::make_unique<sfem_table_s>();
        t->ctx = ctx;
        t->host = cached_host_table(ctx->table_cache, orders[i], elements[i]);
        upload_table(t.get());
        it = cache.emplace(key, t.get()).first;
        d->owned.push_back(std::move(t));
      }
      d->tables.push_back(it->second);
      const double h = lengths[i] / elements[i];
      d->factors.push_back((coefficients ? coefficients[i] : 1.0) * (4.0 / (h * h)));
      d->ext.push_back(static_cast<long long>(orders[i]) * elements[i] - 1);
    }
    for (int i = 0; i < 2; ++i)
      require(has_tma_sweep(d->tables[i]->dev.n, d->tables[i]->dev.K) && fast_enabled(),
              "peer_create: axes 0 and 1 need the K = 64 TMA kernels");
    require(d->ext[0] >= 2 * nranks && d->ext[1] >= 2 * nranks, "peer_create: fewer slab rows than ranks");
    d->lx = balanced_even(d->ext[0], nranks, d->x0);
    d->ly = balanced_even(d->ext[1], nranks, d->y0);
    for (int p = 0; p < nranks; ++p) require(d->lx[p] > 0 && d->ly[p] > 0, "peer_create: empty slab");
    d->pitch = (d->ext[2] + 3) & ~3LL;
    const long long L0 = d->ext[0], L1 = d->ext[1], L2 = d->ext[2];
    d->x_elems = L1 * d->lx[rank] * d->pitch;
    d->y_elems = d->ly[rank] * L0 * d->pitch;
    auto view = [&](long long e0, long long e1, int t0, int t1) {
      View v;
      v.N = 3;
      v.ext = {e0, e1, L2};
      v.pitch = d->pitch;
      v.tables = {d->tables[t0], d->tables[t1], d->tables[2]};
      v.factors = {d->factors[t0], d->factors[t1], d->factors[2]};
      v.eig_off.assign(3, 0);
      v.shift = shift;
      v.use_fast = true;
      return v;
    };
    d->xv = view(d->lx[rank], L1, 0, 1);  // [x][y][z]
    d->yv = view(d->ly[rank], L0, 1, 0);  // [y][x][z]
    d->fwd_rows.push_back(rows_step(d->xv, kForward));
    d->fwd_y = strided_step(d->xv, 1, kForward);
    d->axis0 = strided_step(d->yv, 1, kForward);
    d->inv_local.push_back(strided_step(d->xv, 1, kInverse));
    d->inv_local.push_back(rows_step(d->xv, kInverse));
    require(d->fwd_y.tma && d->axis0.tma, "peer_create: TMA kernels unavailable");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    ck(cudaMalloc(&d->xbuf, d->x_elems * sizeof(double)), "cudaMalloc(x-slab)");
    ck(cudaMalloc(&d->ybuf, d->y_elems * sizeof(double)), "cudaMalloc(y-slab)");
    // kMaxPeer arrival words (written by the peers) + this rank's timeout word
    ck(cudaMalloc(&d->flags, (kMaxPeer + 1) * sizeof(unsigned long long)), "cudaMalloc(flags)");
    ck(cudaMemset(d->xbuf, 0, d->x_elems * sizeof(double)), "memset");
    ck(cudaMemset(d->ybuf, 0, d->y_elems * sizeof(double)), "memset");
    ck(cudaMemset(d->flags, 0, (kMaxPeer + 1) * sizeof(unsigned long long)), "memset");
    d->pf.timeout = d->flags + kMaxPeer;
    *out = d.release();
  });
}

int sfem_cuda_peer_destroy(sfem_peer d) {
  return guarded([&] {
    if (!d) return;
    cudaSetDevice(d->ctx->device);
    if (d->xbuf) cudaFree(d->xbuf);
    if (d->ybuf) cudaFree(d->ybuf);
    if (d->flags) cudaFree(d->flags);
    for (auto& t : d->owned)
      if (t->dbuf) cudaFree(t->dbuf);
    delete d;
  });
}

int sfem_cuda_peer_shape(sfem_peer d, long long* info) {
  return guarded([&] {
    require(d && info, "peer_shape: null argument");
    const int r = d->rank;
    const long long v[8] = {d->x0[r], d->lx[r], d->y0[r], d->ly[r], d->x_elems, d->y_elems, d->pitch, d->nranks};
    std::copy(v, v + 8, info);
  });
}

int sfem_cuda_peer_buffers(sfem_peer d, void** x_slab, void** y_slab, void** flags) {
  return guarded([&] {
    require(d != nullptr, "peer_buffers: null plan");
    if (x_slab) *x_slab = d->xbuf;
    if (y_slab) *y_slab = d->ybuf;
    if (flags) *flags = d->flags;
  });
}

int sfem_cuda_peer_bind(sfem_peer d, void* const* x_slabs, void* const* y_slabs, void* const* flags) {
  return guarded([&] {
    require(d && x_slabs && y_slabs, "peer_bind: null argument");
    const int P = d->nranks, r = d->rank;
    const long long L0 = d->ext[0], L1 = d->ext[1], L2 = d->ext[2], pitch = d->pitch;
    require(x_slabs[r] == d->xbuf && y_slabs[r] == d->ybuf, "peer_bind: own slot must hold this rank's slabs");
    // forward exchange: tile rows y0_q.. of the axis-1 sweep -> rank q's y-slab
    // viewed {z, y_local, x}: box {8, b, 1} at (c0, j b, x0_r + x_local)
    ScatterMaps& f = d->fwd_sc;
    f.npeer = P;
    f.fbase = d->x0[r];
    for (int q = 0; q < P; ++q) {
      f.r0[q] = static_cast<int>(d->y0[q]);
      f.n[q] = static_cast<int>(d->ly[q]);
      box_split(d->ly[q], f.nbox[q], f.b[q]);
      encode_map3(&f.map[q], y_slabs[q], L2, d->ly[q], L0, L0 * pitch * 8, pitch * 8, f.b[q]);
    }
    // return exchange: tile rows x0_p.. of the axis-0 sweep -> rank p's x-slab
    // viewed {z, x_local, y}: box {8, b, 1} at (c0, j b, y0_r + y_local)
    ScatterMaps& a = d->ax_sc;
    a.npeer = P;
    a.fbase = d->y0[r];
    for (int p = 0; p < P; ++p) {
      a.r0[p] = static_cast<int>(d->x0[p]);
      a.n[p] = static_cast<int>(d->lx[p]);
      box_split(d->lx[p], a.nbox[p], a.b[p]);
      encode_map3(&a.map[p], x_slabs[p], L2, d->lx[p], L1, L1 * pitch * 8, pitch * 8, a.b[p]);
    }
    d->device_barrier = flags != nullptr;
    if (flags)
      for (int q = 0; q < P; ++q) d->pf.f[q] = static_cast<unsigned long long*>(flags[q]);
    encode_map(d->fwd_y, d->xbuf);
    encode_map(d->axis0, d->ybuf);
    d->bound = true;
  });
}

int sfem_cuda_peer_phase(sfem_peer d, int phase, void* stream) {
  return guarded([&] {
    require(d != nullptr, "peer_phase: null plan");
    require(d->bound, "peer_phase: peers not bound (sfem_cuda_peer_bind)");
    ck(cudaSetDevice(d->ctx->device), "cudaSetDevice");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
    const PeerDivide none{};
    switch (phase) {
      case SFEM_PEER_FORWARD:
        launch_steps(d->fwd_rows, d->xbuf, d->ctx, s, nullptr);
        ck(launch_sweep_tma_scatter(d->tables[1]->dev, &d->fwd_y.map, d->fwd_y.geo, kForward, d->fwd_sc, none, s),
           "peer forward exchange sweep");
        break;
      case SFEM_PEER_AXIS0: {
        PeerDivide dv{};
        dv.shift = d->shift;
        dv.f1 = d->factors[1];
        dv.f2 = d->factors[2];
        dv.f_last = d->factors[0];
        dv.eig1 = d->tables[1]->dev.eig + d->y0[d->rank];
        dv.eig2 = d->tables[2]->dev.eig;
        ck(launch_sweep_tma_scatter(d->tables[0]->dev, &d->axis0.map, d->axis0.geo, kForwardDivideInverse, d->ax_sc,
                                    dv, s),
           "peer axis-0 exchange sweep");
        break;
      }
      case SFEM_PEER_INVERSE:
        launch_steps(d->inv_local, d->xbuf, d->ctx, s, nullptr);
        break;
      case SFEM_PEER_BARRIER:
        if (d->device_barrier) ck(launch_peer_barrier(d->pf, d->nranks, d->rank, ++d->epoch, s), "peer barrier");
        break;
      default:
        fail("peer_phase: unknown phase");
    }
  });
}

int sfem_cuda_peer_status(sfem_peer d, void* stream, long long* timed_out_epoch) {
  return guarded([&] {
    require(d && timed_out_epoch, "peer_status: null argument");
    ck(cudaSetDevice(d->ctx->device), "cudaSetDevice");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
    ck(cudaStreamSynchronize(s), "peer_status: sync");
    unsigned long long v = 0;
    ck(cudaMemcpy(&v, d->pf.timeout, sizeof v, cudaMemcpyDeviceToHost), "peer_status: read");
    *timed_out_epoch = static_cast<long long>(v);
  });
}

int sfem_cuda_ipc_get_handle(void* d_ptr, void* handle) {
  return guarded([&] {
    require(d_ptr && handle, "ipc_get_handle: null argument");
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, d_ptr), "cudaIpcGetMemHandle");
    std::memcpy(handle, &h, sizeof h);
  });
}

int sfem_cuda_ipc_open_handle(const void* handle, void** d_ptr) {
  return guarded([&] {
    require(d_ptr && handle, "ipc_open_handle: null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    ck(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  });
}

int sfem_cuda_ipc_close(void* d_ptr) {
  return guarded([&] { ck(cudaIpcCloseMemHandle(d_ptr), "cudaIpcCloseMemHandle"); });
}


int sfem_cuda_solve_field(sfem_plan p, int field, const double* params, int nparams, int compute_residual,
                          double* h_u, double* report) {
  return guarded([&] {
    require(p && report, "solve_field: null argument");
    ck(cudaSetDevice(p->ctx->device), "cudaSetDevice");
    cudaStream_t s = p->ctx->stream;
    const long long last = p->ext[p->dim - 1], pitch = p->pitch;
    ensure_work(p);
    const size_t elems = padded_elems(p, pitch);
    if (!p->fbuf) ck(cudaMalloc(&p->fbuf, elems * sizeof(double)), "cudaMalloc(load)");
    cudaEvent_t ev[3];
    for (auto& e : ev) ck(cudaEventCreate(&e), "event");
    struct Ev {
      cudaEvent_t* e;
      ~Ev() {
        for (int i = 0; i < 3; ++i) cudaEventDestroy(e[i]);
      }
    } guard{ev};
    ck(cudaEventRecord(ev[0], s), "event");
    if (sfem_cuda_fem_load(p, field, params, nparams, p->fbuf, pitch, s) != 0) throw std::runtime_error(g_err);
    ck(cudaEventRecord(ev[1], s), "event");
    ck(cudaMemcpyAsync(p->dwork, p->fbuf, elems * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
    ck(cudaEventRecord(ev[2], s), "event");
    run_steps(p, p->dwork, pitch, s, false);
    ck(cudaEventRecord(p->ev[1], s), "event");
    ck(cudaStreamSynchronize(s), "sync");
    report[0] = event_seconds(ev[0], ev[1]);  // seconds_load
    report[1] = event_seconds(ev[2], p->ev[1]);  // seconds_solve
    report[2] = std::nan("");
    report[3] = std::nan("");
    if (compute_residual && sfem_cuda_residual(p, p->dwork, p->fbuf, pitch, &report[2]) != 0)
      throw std::runtime_error(g_err);
    if (field != SFEM_FIELD_CONSTANT &&
        sfem_cuda_max_error(p, field, params, nparams, p->dwork, pitch, &report[3]) != 0)
      throw std::runtime_error(g_err);
    if (h_u) {
      const size_t dense = static_cast<size_t>(p->rows) * last;
      if (!p->dstage) ck(cudaMalloc(&p->dstage, dense * sizeof(double)), "cudaMalloc(stage)");
      ck(cudaMemcpy2DAsync(p->dstage, last * sizeof(double), p->dwork, pitch * sizeof(double), last * sizeof(double),
                           p->rows, cudaMemcpyDeviceToDevice, s),
         "repitch");
      ck(cudaMemcpyAsync(h_u, p->dstage, dense * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaStreamSynchronize(s), "sync");
    }
  });
}

int sfem_cuda_apply_operator_host(sfem_plan p, const double* h_v, double* h_y) {
  return guarded([&] {
    require(p && h_v && h_y, "apply_operator_host: null argument");
    ck(cudaSetDevice(p->ctx->device), "cudaSetDevice");
    cudaStream_t s = p->ctx->stream;
    const long long last = p->ext[p->dim - 1], pitch = p->pitch;
    ensure_work(p);
    const size_t elems = padded_elems(p, pitch), dense = static_cast<size_t>(p->rows) * last;
    if (!p->fbuf) ck(cudaMalloc(&p->fbuf, elems * sizeof(double)), "cudaMalloc(load)");
    if (!p->dstage) ck(cudaMalloc(&p->dstage, dense * sizeof(double)), "cudaMalloc(stage)");
    ck(cudaMemcpyAsync(p->dstage, h_v, dense * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    ck(cudaMemcpy2DAsync(p->dwork, pitch * sizeof(double), p->dstage, last * sizeof(double), last * sizeof(double),
                         p->rows, cudaMemcpyDeviceToDevice, s),
       "repitch");
    apply_sweeps(p, p->dwork, p->fbuf, nullptr, pitch, s);
    ck(cudaMemcpy2DAsync(p->dstage, last * sizeof(double), p->fbuf, pitch * sizeof(double), last * sizeof(double),
                         p->rows, cudaMemcpyDeviceToDevice, s),
       "repitch");
    ck(cudaMemcpyAsync(h_y, p->dstage, dense * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
  });
}


int sfem_cuda_plan_set_algorithm(sfem_plan p, int algorithm) {
  return guarded([&] {
    require(p != nullptr, "plan_set_algorithm: null plan");
    require(algorithm == 0 || algorithm == 1, "plan_set_algorithm: algorithm must be 0 (full) or 1 (partial)");
    if (algorithm == 1) require(p->dim >= 2, "solve: partial diagonalization needs dimension >= 2");
    p->algorithm = algorithm;
    p->pfwd.clear();
  });
}

}  // extern "C"
