// Device-side parameter blocks shared by the sweep kernels and the host
// orchestrator (capi.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

namespace sfem_b200 {

constexpr int kMaxDim = 4;
constexpr int kMaxPasses = 24;

// One (n, K) spectral table in device memory (see table.hpp / DESIGN.md 3).
struct DevTable {
  int n, K, m, half, ne, L;
  const double* mix_fwd_w;  // (K-1) x n x n, [k-1][l][s]
  const double* mix_fwd_d;
  const double* mix_inv;    // (K-1) x n x n, [k-1][s][l]
  const double* e0_fwd_w;   // m x m, [i][l]
  const double* e0_fwd_d;
  const double* e0_inv;
  const double* eig;        // L, coefficient order
  const double* nsq;        // L, norm_sq in coefficient order (1 for k = 0)
  const double* mixT_w;     // n x n x K, [l][s][k] (k-contiguous copies of mix_fwd_w; k = 0 unused)
  const double* mixT_d;     // same for mix_fwd_d
  const double* mixT_i;     // n x n x K, [s][l][k] copy of mix_inv
  const double* eigT;       // n x K, [l][k]: eig[m + (k-1) n + l] (k = 0 unused)
  const double* nsqT;       // n x K, [l][k]: nsq[m + (k-1) n + l]
  const double2* tw;        // N: exp(-2 pi i t/N)
  const double2* mk;        // N: exp(-i pi k/(2N))
  const double2* mkh;       // N: 0.5 exp(+i pi k/(2N))
  const double2* om;        // N: exp(-i pi j/N)
  int npass;
  int radix[kMaxPasses];    // Stockham pass radices, product = K
};

// A set of lines along one axis of a tensor.  Line l (0 <= l < nlines) is
// split as l = (o2 * n1 + o1) * ninner + i and starts at
// o2*os2 + o1*os1 + i*is; position p of the line is at start + p*ps.  Tiles
// are read from `src` and written to `dst` at the same offsets (in place when
// equal).
struct LineSet {
  const double* src;
  double* dst;
  long long nlines;
  long long ninner, n1;
  long long is, os1, os2, ps;
  int contiguous;  // ps == 1: lines are rows (tile loads run along the line)
};

// Symbol data for the fused last-axis kernel: a line's leading coordinates
// (row-major over the leading axes) give base = shift + sum_i f_i lambda_i[a_i]
// (poisson.cpp:586-590 order), then denom = base + f_last * lambda_last[p].
struct SymbolInfo {
  int nlead;
  long long lead_ext[kMaxDim];
  const double* lead_eig[kMaxDim];
  double lead_f[kMaxDim];
  double shift;
  double f_last;
  // xblk > 0 (3-D blocked layout): rows are ordered (x_hi, y, x_lo) with
  // lead_ext {nhi, L1, xblk}; x = x_hi*xblk + x_lo indexes lead_eig[0]
  // (x >= x_ext: a padding row), y lead_eig[1].
  int xblk;
  long long x_ext;
};

enum SweepMode { kForward = 0, kInverse = 1, kForwardDivideInverse = 2 };

// Tile decomposition for the TMA strided kernels: the tensor is viewed as 4-D
// (d0 = last axis, d1 = swept axis, d2/d3 = remaining axes, size 1 if absent);
// a tile is 8 consecutive d0 indices x all d1 positions at one (d2, d3).
//
// Box coordinates per tensor map (TmaGeom::ld_mode / st_mode), the tile being
// (c0 = first last-axis index, c2, c3) of the grid:
//   kBoxPlain    (c0, j*boxp, c2, c3)               box {8, boxp, 1, 1}
//   kBoxSwept    (c0, 0, 0, c2): the swept axis is stored blocked as
//                (x_hi, x_lo) with x = x_hi*xblk + x_lo; one box
//                {8, xblk, nhi, 1} brings all positions (nbox = 1)
//   kBoxSplit    (c0, j*boxp, c2 % xblk, c2 / xblk): the tile's fixed
//                coordinate c2 is blocked in this tensor
enum BoxMode { kBoxPlain = 0, kBoxSwept = 1, kBoxSplit = 2 };
struct TmaGeom {
  int nbox, boxp;      // boxes along d1 (boxp positions each, nbox*boxp >= L)
  long long nblk0;     // ceil(L_d0 / 8)
  long long ext0;      // L_d0 (extent of the last axis)
  long long ext2;      // extent of d2
  long long ntiles;    // nblk0 * ext2 * ext3
  int ld_mode, st_mode, xblk;
  int prefetch;        // mid kernels: L2-prefetch the tile this many tiles ahead (0 = off)
};

// Strided sweep through TMA (sweep_fast.cu).  `tmap` / `smap` are CUtensorMaps
// (64-byte aligned opaque blobs) of the tensor the tile is loaded from and
// stored to (the same map for an in-place sweep).
cudaError_t launch_sweep_tma(const DevTable& t, const void* tmap, const void* smap, const TmaGeom& geo, int mode,
                             int analysis, cudaStream_t stream);
bool has_tma_sweep(int n, int K);
// Fused last-axis sweep with per-row bulk copies (K = 64 specialisations).
// A row is the concatenation of `n` segments: segment s of row q holds
// positions [pos0[s], pos0[s] + len[s]) at base + off[s] + q * stride[s]
// (elements; every offset, stride and length even so the copies are 16-byte
// aligned).  One segment (off 0, stride = pitch, len = L rounded up to even)
// is a plain dof tensor; the multi-GPU axis-0 sweep reads and writes the
// source-major blocks of the exchange buffer directly.  In place.  `mode`:
// kForward / kInverse / kForwardDivideInverse (sym used by the latter only).
constexpr int kMaxSeg = 32;  // ranks x exchange chunks (multi-GPU axis-0 sweep)
struct RowSegs {
  int n;
  int pos0[kMaxSeg], len[kMaxSeg];
  long long off[kMaxSeg], stride[kMaxSeg];
};
bool has_bulk_rows(int n, int K);

// Strided TMA sweep whose tile stores go to other ranks' tensors (NVLink peer
// memory; local buffers in the single-device loopback): peer q receives tile
// rows [r0[q], r0[q] + n[q]) through map[q], a 3-D tensor map {last axis,
// target rows, fixed} with box {8, b[q], 1}, at coordinates
// (c0, j * b[q], fbase + c2) for boxes j < nbox[q] (c0: the tile's first
// last-axis index, c2: the tile's fixed coordinate of the load geometry).
// MODE kForward (axis-1 forward on the x-slab) or kForwardDivideInverse (the
// axis-0 sweep on the y-slab, divide base = (shift + f1 eig1[c2]) + f2 eig2[z],
// then + f_last eig[pos] of the swept table).
constexpr int kMaxPeer = 8;
struct alignas(64) ScatterMaps {
  CUtensorMap map[kMaxPeer];
  int npeer;
  long long fbase;
  int r0[kMaxPeer], n[kMaxPeer], b[kMaxPeer], nbox[kMaxPeer];
};
struct PeerDivide {
  double shift, f1, f2, f_last;
  const double* eig1;  // already offset to the rank's first row
  const double* eig2;
};
cudaError_t launch_sweep_tma_scatter(const DevTable& t, const void* tmap, const TmaGeom& geo, int mode,
                                     const ScatterMaps& sc, const PeerDivide& dv, cudaStream_t stream);
// Device barrier among ranks over peer-mapped flag words: rank `rank` writes
// `epoch` into flags[q][rank] of every q and waits until its own
// flags[rank][0..nranks) all reach `epoch` (system-scope release / acquire).
struct PeerFlags {
  unsigned long long* f[kMaxPeer];
  unsigned long long* timeout;  // this rank's word: epoch of a barrier that timed out (0 = none)
};
cudaError_t launch_peer_barrier(const PeerFlags& fl, int nranks, int rank, unsigned long long epoch,
                                cudaStream_t stream);
cudaError_t launch_sweep_bulk_rows(const DevTable& t, double* data, const RowSegs& segs, long long nrows, int mode,
                                   int analysis, const SymbolInfo& sym, cudaStream_t stream);
enum AnalysisKind { kWeighted = 0, kDirect = 1 };
// Fused last-axis sweep (forward + divide + inverse) with warp-local FFT jobs
// (sweep_rows.cu); same row segments as launch_sweep_bulk_rows.
bool has_rows_fused(int n, int K);
cudaError_t launch_sweep_rows_fused(const DevTable& t, double* data, const RowSegs& segs, long long nrows,
                                    const SymbolInfo& sym, cudaStream_t stream);

// Shared-memory bytes needed for a tile of B lines of table t (FFT work
// buffers excluded when they live in global scratch).
size_t sweep_smem_bytes(const DevTable& t, int B, bool global_work = false);
// Doubles of FFT work buffer per tile (global scratch mode: per CTA).
size_t sweep_work_doubles(const DevTable& t, int B);

// Fast path (sweep_fast.cu) for the (n, K) it was compiled for; returns
// cudaErrorNotSupported when no specialisation exists.
cudaError_t launch_sweep_fast(const DevTable& t, const LineSet& lines, int mode, int analysis,
                              const SymbolInfo* sym, cudaStream_t stream);
bool has_fast_sweep(int n, int K, int mode, int contiguous);

// Mid-length line kernels (sweep_mid.cu) for the (n, K) they were compiled for.
// Lines too long for shared-memory FFT buffers run them in global scratch:
// mid_work_doubles (0 when none is needed) sizes the `gwork` argument.
bool has_mid_sweep(int n, int K);
size_t mid_work_doubles(int n, int K, long long nlines);
cudaError_t launch_sweep_mid(const DevTable& t, const LineSet& lines, int mode, int analysis,
                             const SymbolInfo* sym, cudaStream_t stream, double* gwork = nullptr);
// Strided mid-kernel sweeps with TMA tiles (the tuned shapes): lines per tile
// (0: no TMA kernel for this table) and the launch.  `tmap`: 4-D tensor map
// {last axis, swept axis, outer, outer} with box {lines, geo.boxp, 1, 1};
// geo.nblk0 counts tiles of `lines` last-axis indices.  In place.
int mid_tma_lines(int n, int K);
// `smap` (blocked 3-D schedule of the shapes mid_tma_blocked() names): the map the tile is stored through when
// it differs from `tmap`; geo.ld_mode / st_mode / xblk give the box coordinates of either side (BoxMode).
cudaError_t launch_sweep_mid_tma(const DevTable& t, const void* tmap, const TmaGeom& geo, int mode, int analysis,
                                 cudaStream_t stream, const void* smap = nullptr);
bool mid_tma_blocked(int n, int K);
// Component-major tiles (sweep_mid_tma_cm, sweep_mid_impl.cuh) for tensors of
// at most three axes: `maps` are three consecutive CUtensorMaps over the 5-D
// view {last axis, e >> 1, e & 1, s, outer axis} of position e * n + s:
// box {8, K/2, 2, n-1, 1}; box {8, K/2, 1, 1, 1}; the same box over the tensor
// starting at position 2n - 1 with K/2 - 1 entries along the second axis.
// SFEM_MID_CM=0 turns the layout off (A/B).
bool mid_tma_cm(int n, int K);
cudaError_t launch_sweep_mid_tma_cm(const DevTable& t, const void* maps, const TmaGeom& geo, int mode, int analysis,
                                    cudaStream_t stream);

// Slot-major class tiles (nodal (K+1) x count, interior K*(n-1) x count,
// [j*count + b]) <-> the slot-major dof tile (n*K-1) x count (lines_block.cu).
cudaError_t launch_class_tiles(int n, int K, long long count, double* nodal, double* interior, double* dof,
                               bool to_dof, cudaStream_t stream);

// Launch one sweep over `lines` with tiles of B lines.
cudaError_t launch_sweep(const DevTable& t, const LineSet& lines, int mode, int analysis,
                         const SymbolInfo* sym, int B, cudaStream_t stream, double* gwork = nullptr);

}  // namespace sfem_b200
