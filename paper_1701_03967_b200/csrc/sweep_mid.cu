// Dispatch of the mid-length line kernels (templates in sweep_mid_impl.cuh):
// the tuned shapes are instantiated here, the general shapes in
// sweep_mid_k{16,...,2048}.cu (powers of two) and sweep_mid_k{24,...,1000}.cu
// (3 * 2^j, 5 * 2^j, 2^i * 5^j), one translation unit per K, built in parallel.
#include <cstdlib>

#include "sweep_mid_impl.cuh"

namespace sfem_b200 {
namespace mid {

SFEM_PHASE_EXPORT(sfem_debug_phase_records_mid)

extern template cudaError_t launch_auto_n<16>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                 cudaStream_t);
extern template cudaError_t launch_auto_n<32>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                 cudaStream_t);
extern template cudaError_t launch_auto_n<64>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                 cudaStream_t);
extern template cudaError_t launch_auto_n<128>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                 cudaStream_t);
extern template cudaError_t launch_auto_n<256>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                 cudaStream_t);
extern template cudaError_t launch_auto_n<512>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                 cudaStream_t);
extern template cudaError_t launch_auto_n<1024>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<2048>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);

extern template cudaError_t launch_auto_n<24>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<40>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<48>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<80>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<96>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<100>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<160>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<192>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<200>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<320>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<384>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<768>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_n<1000>(const DevTable&, const LineSet&, int, int, const SymbolInfo*,
                                                  cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<16>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<24>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<32>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<40>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<48>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<64>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<80>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<96>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<100>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<128>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<160>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<192>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<200>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<256>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<320>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<384>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_cm_n<512>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                        cudaStream_t);
extern template cudaError_t launch_auto_tma_n<16>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<24>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<32>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<40>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<48>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<64>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<80>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<96>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<100>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<128>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<160>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<192>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<200>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<256>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<320>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<384>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<512>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<768>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<1000>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<1024>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
extern template cudaError_t launch_auto_tma_n<2048>(const DevTable&, const void*, const TmaGeom&, int, int,
                                                     cudaStream_t);
}  // namespace mid

// Lines per tile and threads per CTA of the C5 shapes.
// n = 1 (K = 1024): four lines (J = 4 jobs, 65 KB) and 256 threads give two
// CTAs per SM instead of one 131 KB tile (C5 n=1 67.7 -> 64.3 ms)
#ifndef SFEM_MID_B_N1
#define SFEM_MID_B_N1 4
#endif
#ifndef SFEM_MID_TH_N1
#define SFEM_MID_TH_N1 256
#endif
#ifndef SFEM_MID_B_N2
#define SFEM_MID_B_N2 8
#endif
// Threads: one radix-16 / radix-8 butterfly per thread and pass (J * K / R
// items), so a pass keeps R complex values per thread, not 2R (spills):
// n = 2: J = 12 jobs x 512 / 8 = 768 items = 2 x 384; n = 4: 20 x 256 / 16 = 320.
#ifndef SFEM_MID_TH_N2
#define SFEM_MID_TH_N2 384
#endif
#ifndef SFEM_MID_B_N4
#define SFEM_MID_B_N4 8
#endif
#ifndef SFEM_MID_TH_N4
#define SFEM_MID_TH_N4 320
#endif
#ifndef SFEM_MID_B_N9
#define SFEM_MID_B_N9 8
#endif
#ifndef SFEM_MID_TH_N9
#define SFEM_MID_TH_N9 256
#endif

// General shapes: every order at the power-of-two K below (tile shape from
// mid::AutoShape).
#ifndef SFEM_MID_AUTO
#define SFEM_MID_AUTO 1
#endif
bool mid_auto(int n, int K) {
#if SFEM_MID_AUTO
  switch (K) {
    case 16: return mid::auto_ok_n<16>(n);
    case 32: return mid::auto_ok_n<32>(n);
    case 64: return mid::auto_ok_n<64>(n);
    case 128: return mid::auto_ok_n<128>(n);
    case 256: return mid::auto_ok_n<256>(n);
    case 512: return mid::auto_ok_n<512>(n);
    case 1024: return n != 1 && n != 9 && mid::auto_ok_n<1024>(n);
    case 2048: return mid::auto_ok_n<2048>(n);
    case 24: return mid::auto_ok_n<24>(n);
    case 40: return mid::auto_ok_n<40>(n);
    case 48: return mid::auto_ok_n<48>(n);
    case 80: return mid::auto_ok_n<80>(n);
    case 96: return mid::auto_ok_n<96>(n);
    case 100: return mid::auto_ok_n<100>(n);
    case 160: return mid::auto_ok_n<160>(n);
    case 192: return mid::auto_ok_n<192>(n);
    case 200: return mid::auto_ok_n<200>(n);
    case 320: return mid::auto_ok_n<320>(n);
    case 384: return mid::auto_ok_n<384>(n);
    case 768: return mid::auto_ok_n<768>(n);
    case 1000: return mid::auto_ok_n<1000>(n);
    default: return false;
  }
#else
  (void)n;
  (void)K;
  return false;
#endif
}

// Strided sweeps of the tuned shapes move their tiles by TMA (sweep_mid_tma);
// SFEM_MID_TMA=0 keeps the cp.async kernels (A/B).
static bool mid_tma_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("SFEM_MID_TMA");
    return !(e && e[0] == '0');
  }();
  return v;
}

bool mid_auto(int n, int K);

int mid_tma_lines(int n, int K) {
  if (!mid_tma_enabled()) return 0;
  if (n == 1 && K == 1024) return SFEM_MID_B_N1;
  if (n == 2 && K == 512) return SFEM_MID_B_N2;
  if (n == 4 && K == 256) return SFEM_MID_B_N4;
  if (n == 9 && K == 114) return SFEM_MID_B_N9;
  if (n == 9 && K == 1024) return 2;
#if SFEM_MID_AUTO
  if (!mid_auto(n, K)) return 0;
  switch (K) {
    case 16: return mid::auto_tma_lines_n<16>(n);
    case 24: return mid::auto_tma_lines_n<24>(n);
    case 32: return mid::auto_tma_lines_n<32>(n);
    case 40: return mid::auto_tma_lines_n<40>(n);
    case 48: return mid::auto_tma_lines_n<48>(n);
    case 64: return mid::auto_tma_lines_n<64>(n);
    case 80: return mid::auto_tma_lines_n<80>(n);
    case 96: return mid::auto_tma_lines_n<96>(n);
    case 100: return mid::auto_tma_lines_n<100>(n);
    case 128: return mid::auto_tma_lines_n<128>(n);
    case 160: return mid::auto_tma_lines_n<160>(n);
    case 192: return mid::auto_tma_lines_n<192>(n);
    case 200: return mid::auto_tma_lines_n<200>(n);
    case 256: return mid::auto_tma_lines_n<256>(n);
    case 320: return mid::auto_tma_lines_n<320>(n);
    case 384: return mid::auto_tma_lines_n<384>(n);
    case 512: return mid::auto_tma_lines_n<512>(n);
    case 768: return mid::auto_tma_lines_n<768>(n);
    case 1000: return mid::auto_tma_lines_n<1000>(n);
    case 1024: return mid::auto_tma_lines_n<1024>(n);
    case 2048: return mid::auto_tma_lines_n<2048>(n);
    default: return 0;
  }
#else
  return 0;
#endif
}

// Component-major strided tiles (Cfg::CM): the even orders of the tuned shapes,
// whose dense 64-byte tile rows keep a warp on one half of the bank line.
#ifndef SFEM_MID_CM
#define SFEM_MID_CM 1
#endif
bool mid_tma_cm(int n, int K) {
#if SFEM_MID_CM
  static const bool on = [] {
    const char* e = std::getenv("SFEM_MID_CM");
    return !(e && e[0] == '0');
  }();
  if (!on || !mid_tma_enabled()) return false;
  if ((n == 4 && K == 256 && SFEM_MID_B_N4 == 8) || (n == 2 && K == 512 && SFEM_MID_B_N2 == 8)) return true;
#if SFEM_MID_AUTO
  if (!mid_auto(n, K)) return false;
  switch (K) {
    case 16: return mid::auto_tma_cm_n<16>(n);
    case 24: return mid::auto_tma_cm_n<24>(n);
    case 32: return mid::auto_tma_cm_n<32>(n);
    case 40: return mid::auto_tma_cm_n<40>(n);
    case 48: return mid::auto_tma_cm_n<48>(n);
    case 64: return mid::auto_tma_cm_n<64>(n);
    case 80: return mid::auto_tma_cm_n<80>(n);
    case 96: return mid::auto_tma_cm_n<96>(n);
    case 100: return mid::auto_tma_cm_n<100>(n);
    case 128: return mid::auto_tma_cm_n<128>(n);
    case 160: return mid::auto_tma_cm_n<160>(n);
    case 192: return mid::auto_tma_cm_n<192>(n);
    case 200: return mid::auto_tma_cm_n<200>(n);
    case 256: return mid::auto_tma_cm_n<256>(n);
    case 320: return mid::auto_tma_cm_n<320>(n);
    case 384: return mid::auto_tma_cm_n<384>(n);
    case 512: return mid::auto_tma_cm_n<512>(n);
    default: return false;
  }
#else
  return false;
#endif
#else
  (void)n;
  (void)K;
  return false;
#endif
}

cudaError_t launch_sweep_mid_tma_cm(const DevTable& t, const void* maps, const TmaGeom& geo, int mode, int analysis,
                                    cudaStream_t stream) {
  if (geo.ntiles <= 0) return cudaSuccess;
#if SFEM_MID_CM
  if (t.n == 4 && t.K == 256) return mid::launch_tma_cm<4, 256, 8, SFEM_MID_TH_N4>(t, maps, geo, mode, analysis, stream);
  if (t.n == 2 && t.K == 512) return mid::launch_tma_cm<2, 512, 8, SFEM_MID_TH_N2>(t, maps, geo, mode, analysis, stream);
#if SFEM_MID_AUTO
  switch (t.K) {
    case 16: return mid::launch_auto_tma_cm_n<16>(t, maps, geo, mode, analysis, stream);
    case 24: return mid::launch_auto_tma_cm_n<24>(t, maps, geo, mode, analysis, stream);
    case 32: return mid::launch_auto_tma_cm_n<32>(t, maps, geo, mode, analysis, stream);
    case 40: return mid::launch_auto_tma_cm_n<40>(t, maps, geo, mode, analysis, stream);
    case 48: return mid::launch_auto_tma_cm_n<48>(t, maps, geo, mode, analysis, stream);
    case 64: return mid::launch_auto_tma_cm_n<64>(t, maps, geo, mode, analysis, stream);
    case 80: return mid::launch_auto_tma_cm_n<80>(t, maps, geo, mode, analysis, stream);
    case 96: return mid::launch_auto_tma_cm_n<96>(t, maps, geo, mode, analysis, stream);
    case 100: return mid::launch_auto_tma_cm_n<100>(t, maps, geo, mode, analysis, stream);
    case 128: return mid::launch_auto_tma_cm_n<128>(t, maps, geo, mode, analysis, stream);
    case 160: return mid::launch_auto_tma_cm_n<160>(t, maps, geo, mode, analysis, stream);
    case 192: return mid::launch_auto_tma_cm_n<192>(t, maps, geo, mode, analysis, stream);
    case 200: return mid::launch_auto_tma_cm_n<200>(t, maps, geo, mode, analysis, stream);
    case 256: return mid::launch_auto_tma_cm_n<256>(t, maps, geo, mode, analysis, stream);
    case 320: return mid::launch_auto_tma_cm_n<320>(t, maps, geo, mode, analysis, stream);
    case 384: return mid::launch_auto_tma_cm_n<384>(t, maps, geo, mode, analysis, stream);
    case 512: return mid::launch_auto_tma_cm_n<512>(t, maps, geo, mode, analysis, stream);
    default: break;
  }
#endif
#endif
  return cudaErrorNotSupported;
}

// Shapes whose 3-D solves run the blocked schedule (capi.cu build_blocked_mid_steps): axis 0 stored as
// (x_hi, y, x_lo, z) in a plan scratch, so an axis-0 tile's rows are 8-row groups instead of one row per plane.
// n = 1, K = 1024 (C5): 32-byte tile rows, 1,023 of them each in its own 2 MB page along axis 0.  Measured and left
// off for n = 9, K = 114 (64-byte rows: 46.2 -> 46.8 ms, profiles/r4s_mid_blocked_n9_rejected.txt).
// SFEM_MID_BLOCKED=0 turns it off (A/B).
bool mid_tma_blocked(int n, int K) {
  static const bool on = [] {
    const char* e = std::getenv("SFEM_MID_BLOCKED");
    return !(e && e[0] == '0');
  }();
  return on && mid_tma_enabled() && n == 1 && K == 1024;
}

cudaError_t launch_sweep_mid_tma(const DevTable& t, const void* tmap, const TmaGeom& geo, int mode, int analysis,
                                 cudaStream_t stream, const void* smap) {
  if (geo.ntiles <= 0) return cudaSuccess;
  if (t.n == 1 && t.K == 1024)
    return mid::launch_tma<1, 1024, SFEM_MID_B_N1, SFEM_MID_TH_N1>(t, tmap, geo, mode, analysis, stream, smap);
  if (t.n == 2 && t.K == 512)
    return mid::launch_tma<2, 512, SFEM_MID_B_N2, SFEM_MID_TH_N2>(t, tmap, geo, mode, analysis, stream);
  if (t.n == 4 && t.K == 256)
    return mid::launch_tma<4, 256, SFEM_MID_B_N4, SFEM_MID_TH_N4>(t, tmap, geo, mode, analysis, stream);
  if (t.n == 9 && t.K == 114)
    return mid::launch_tma<9, 114, SFEM_MID_B_N9, SFEM_MID_TH_N9>(t, tmap, geo, mode, analysis, stream, smap);
  if (smap != nullptr && smap != tmap) return cudaErrorNotSupported;
  if (t.n == 9 && t.K == 1024) return mid::launch_tma<9, 1024, 2, SFEM_MID_C3_TH>(t, tmap, geo, mode, analysis, stream);
#if SFEM_MID_AUTO
  switch (t.K) {
    case 16: return mid::launch_auto_tma_n<16>(t, tmap, geo, mode, analysis, stream);
    case 24: return mid::launch_auto_tma_n<24>(t, tmap, geo, mode, analysis, stream);
    case 32: return mid::launch_auto_tma_n<32>(t, tmap, geo, mode, analysis, stream);
    case 40: return mid::launch_auto_tma_n<40>(t, tmap, geo, mode, analysis, stream);
    case 48: return mid::launch_auto_tma_n<48>(t, tmap, geo, mode, analysis, stream);
    case 64: return mid::launch_auto_tma_n<64>(t, tmap, geo, mode, analysis, stream);
    case 80: return mid::launch_auto_tma_n<80>(t, tmap, geo, mode, analysis, stream);
    case 96: return mid::launch_auto_tma_n<96>(t, tmap, geo, mode, analysis, stream);
    case 100: return mid::launch_auto_tma_n<100>(t, tmap, geo, mode, analysis, stream);
    case 128: return mid::launch_auto_tma_n<128>(t, tmap, geo, mode, analysis, stream);
    case 160: return mid::launch_auto_tma_n<160>(t, tmap, geo, mode, analysis, stream);
    case 192: return mid::launch_auto_tma_n<192>(t, tmap, geo, mode, analysis, stream);
    case 200: return mid::launch_auto_tma_n<200>(t, tmap, geo, mode, analysis, stream);
    case 256: return mid::launch_auto_tma_n<256>(t, tmap, geo, mode, analysis, stream);
    case 320: return mid::launch_auto_tma_n<320>(t, tmap, geo, mode, analysis, stream);
    case 384: return mid::launch_auto_tma_n<384>(t, tmap, geo, mode, analysis, stream);
    case 512: return mid::launch_auto_tma_n<512>(t, tmap, geo, mode, analysis, stream);
    case 768: return mid::launch_auto_tma_n<768>(t, tmap, geo, mode, analysis, stream);
    case 1000: return mid::launch_auto_tma_n<1000>(t, tmap, geo, mode, analysis, stream);
    case 1024: return mid::launch_auto_tma_n<1024>(t, tmap, geo, mode, analysis, stream);
    case 2048: return mid::launch_auto_tma_n<2048>(t, tmap, geo, mode, analysis, stream);
    default: break;
  }
#endif
  return cudaErrorNotSupported;
}

bool has_mid_sweep(int n, int K) {
  return (n == 1 && K == 1024) || (n == 2 && K == 512) || (n == 4 && K == 256) || (n == 9 && K == 114) ||
         (n == 9 && K == 1024) || (n == 4 && K == 4096) || mid_auto(n, K);
}

// C2 (n = 4, K = 4096): one-line tiles with the packed middle / nodal job keep
// the FFT work in shared memory (mid::Cfg::PK); SFEM_C2_GW=1 selects the older
// kernel with the work in global scratch (kept for A/B).
#ifndef SFEM_MID_C2_PK_TH
#define SFEM_MID_C2_PK_TH 768
#endif
static bool c2_gw() {
  static const bool v = [] {
    const char* e = std::getenv("SFEM_C2_GW");
    return e && e[0] == '1';
  }();
  return v;
}

size_t mid_work_doubles(int n, int K, long long nlines) {
  if (n == 4 && K == 4096 && c2_gw()) {  // B = 1: jobs = 1 pair + 1 middle + 2 nodal
    return static_cast<size_t>(nlines) * 2 * 2 * 4 * 4096;
  }
  return 0;
}

cudaError_t launch_sweep_mid(const DevTable& t, const LineSet& ls, int mode, int analysis, const SymbolInfo* sym,
                             cudaStream_t stream, double* gwork) {
  if (ls.nlines <= 0) return cudaSuccess;
  if (t.n == 4 && t.K == 4096) {
    if (!c2_gw()) return mid::launch<4, 4096, 1, SFEM_MID_C2_PK_TH>(t, ls, mode, analysis, sym, stream);
    if (!gwork) return cudaErrorInvalidValue;
    return mid::launch_gw<4, 4096, 1, SFEM_MID_C2_TH>(t, ls, mode, analysis, sym, gwork, stream);
  }
  // (lines per tile, threads) per shape
  if (t.n == 1 && t.K == 1024)
    return mid::launch<1, 1024, SFEM_MID_B_N1, SFEM_MID_TH_N1>(t, ls, mode, analysis, sym, stream);
  if (t.n == 2 && t.K == 512)
    return mid::launch<2, 512, SFEM_MID_B_N2, SFEM_MID_TH_N2>(t, ls, mode, analysis, sym, stream);
  if (t.n == 4 && t.K == 256)
    return mid::launch<4, 256, SFEM_MID_B_N4, SFEM_MID_TH_N4>(t, ls, mode, analysis, sym, stream);
  if (t.n == 9 && t.K == 114)
    return mid::launch<9, 114, SFEM_MID_B_N9, SFEM_MID_TH_N9>(t, ls, mode, analysis, sym, stream);
  if (t.n == 9 && t.K == 1024) return mid::launch<9, 1024, 2, SFEM_MID_C3_TH>(t, ls, mode, analysis, sym, stream);
#if SFEM_MID_AUTO
  if (mid_auto(t.n, t.K)) {
    switch (t.K) {
      case 16: return mid::launch_auto_n<16>(t, ls, mode, analysis, sym, stream);
      case 32: return mid::launch_auto_n<32>(t, ls, mode, analysis, sym, stream);
      case 64: return mid::launch_auto_n<64>(t, ls, mode, analysis, sym, stream);
      case 128: return mid::launch_auto_n<128>(t, ls, mode, analysis, sym, stream);
      case 256: return mid::launch_auto_n<256>(t, ls, mode, analysis, sym, stream);
      case 512: return mid::launch_auto_n<512>(t, ls, mode, analysis, sym, stream);
      case 1024: return mid::launch_auto_n<1024>(t, ls, mode, analysis, sym, stream);
      case 2048: return mid::launch_auto_n<2048>(t, ls, mode, analysis, sym, stream);
      case 24: return mid::launch_auto_n<24>(t, ls, mode, analysis, sym, stream);
      case 40: return mid::launch_auto_n<40>(t, ls, mode, analysis, sym, stream);
      case 48: return mid::launch_auto_n<48>(t, ls, mode, analysis, sym, stream);
      case 80: return mid::launch_auto_n<80>(t, ls, mode, analysis, sym, stream);
      case 96: return mid::launch_auto_n<96>(t, ls, mode, analysis, sym, stream);
      case 100: return mid::launch_auto_n<100>(t, ls, mode, analysis, sym, stream);
      case 160: return mid::launch_auto_n<160>(t, ls, mode, analysis, sym, stream);
      case 192: return mid::launch_auto_n<192>(t, ls, mode, analysis, sym, stream);
      case 200: return mid::launch_auto_n<200>(t, ls, mode, analysis, sym, stream);
      case 320: return mid::launch_auto_n<320>(t, ls, mode, analysis, sym, stream);
      case 384: return mid::launch_auto_n<384>(t, ls, mode, analysis, sym, stream);
      case 768: return mid::launch_auto_n<768>(t, ls, mode, analysis, sym, stream);
      case 1000: return mid::launch_auto_n<1000>(t, ls, mode, analysis, sym, stream);
      default: break;
    }
  }
#endif
  return cudaErrorNotSupported;
}

}  // namespace sfem_b200
