// Per-CTA phase timestamps for diagnostic builds (-DSFEM_PHASE_TIMING=1).
// Included inside a kernel namespace; each translation unit gets its own
// record buffer and exports it with SFEM_PHASE_EXPORT(name) (not part of
// include/sfem_cuda.h): tools/phase_times.py reads the records back.
// Points: 0 start, 1 tile landed, 2..3 kernel-specific, 4 computed,
// 5 stored/drained.
#pragma once

#ifndef SFEM_PHASE_TIMING
#define SFEM_PHASE_TIMING 0
#endif

#if SFEM_PHASE_TIMING
struct PhaseRec {
  unsigned long long t[6];    // clock64 at the phase points
  unsigned long long g0, g5;  // globaltimer (ns) at start / end
  int tile, smid, kind, pad;
};
constexpr int kMaxPhaseRecs = 1 << 20;
static __device__ PhaseRec g_phase[kMaxPhaseRecs];
static __device__ unsigned int g_phase_n;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SFEM_PT(i)                \
  if (threadIdx.x == 0) {         \
    pt[i] = clock64();            \
    if (i == 0) pg0 = gtimer();   \
    if (i == 5) pg5 = gtimer();   \
  }
#define SFEM_PT_DECL unsigned long long pt[6] = {0, 0, 0, 0, 0, 0}, pg0 = 0, pg5 = 0
#define SFEM_PT_FLUSH(KIND)                                  \
  if (threadIdx.x == 0) {                                    \
    const unsigned idx_ = atomicAdd(&g_phase_n, 1u);         \
    if (idx_ < kMaxPhaseRecs) {                              \
      PhaseRec r_;                                           \
      for (int i_ = 0; i_ < 6; ++i_) r_.t[i_] = pt[i_];      \
      r_.g0 = pg0;                                           \
      r_.g5 = pg5;                                           \
      r_.tile = blockIdx.x;                                  \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(r_.smid));  \
      r_.kind = (KIND);                                      \
      r_.pad = 0;                                            \
      g_phase[idx_] = r_;                                    \
    }                                                        \
  }
// Copies up to `cap` records (12 x u64 each: clk0..clk5, gt0, gt5, tile,
// smid, kind, 0) to host, resets the counter; returns the count, -1 on error.
#define SFEM_PHASE_EXPORT(NAME)                                                             \
  extern "C" long long NAME(unsigned long long* host, long long cap) {                      \
    unsigned int n = 0;                                                                     \
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;                                  \
    if (cudaMemcpyFromSymbol(&n, g_phase_n, sizeof(n)) != cudaSuccess) return -1;           \
    long long m = n < static_cast<unsigned>(kMaxPhaseRecs) ? n : kMaxPhaseRecs;             \
    if (m > cap) m = cap;                                                                   \
    PhaseRec* tmp = new PhaseRec[m > 0 ? m : 1];                                            \
    if (m > 0 && cudaMemcpyFromSymbol(tmp, g_phase, m * sizeof(PhaseRec)) != cudaSuccess) { \
      delete[] tmp;                                                                         \
      return -1;                                                                            \
    }                                                                                       \
    for (long long i = 0; i < m; ++i) {                                                     \
      unsigned long long* h = host + 12 * i;                                                \
      for (int j = 0; j < 6; ++j) h[j] = tmp[i].t[j];                                       \
      h[6] = tmp[i].g0;                                                                     \
      h[7] = tmp[i].g5;                                                                     \
      h[8] = tmp[i].tile;                                                                   \
      h[9] = tmp[i].smid;                                                                   \
      h[10] = tmp[i].kind;                                                                  \
      h[11] = 0;                                                                            \
    }                                                                                       \
    delete[] tmp;                                                                           \
    const unsigned int zero = 0;                                                            \
    cudaMemcpyToSymbol(g_phase_n, &zero, sizeof(zero));                                     \
    return m;                                                                               \
  }
#else
#define SFEM_PT(i)
#define SFEM_PT_DECL
#define SFEM_PT_FLUSH(KIND)
#define SFEM_PHASE_EXPORT(NAME)
#endif
