// Host-side spectral table builder (cold path, runs once per (n, K) before any
// device work).  Re-implements, from the reference's published algorithm, the
// data the sweeps consume:
//   element matrices          reference include/sfem/element.hpp:258-295
//   interior pencil eigenpairs element.hpp:140-198, 313-347 (Cholesky+Jacobi,
//                              smallmat.hpp:72-214)
//   theta-equation roots      spectral.hpp:26-193
//   interior vectors / norms  spectral.hpp:198-277
//   finalised per-k data      spectral.cpp:21-79
// and then derives the device-side mix matrices that fold the half-angle
// twiddles and 1/||s||^2 into one n x n matrix per frequency.
#pragma once

#include <string>
#include <vector>

namespace sfem_b200 {

struct HostTable {
  int order = 0, elements = 0;  // n, K
  // element data
  std::vector<double> stiffness, mass;  // (n+1)^2 row-major
  std::vector<double> mass_interior;    // m x m
  // interior eigensystem (m = n-1)
  std::vector<double> interior_values;   // m
  std::vector<double> interior_vectors;  // m x m row-major, column l-1 = e^(l)
  // per frequency k = 1..K-1, l = 1..n, index (k-1)*n + (l-1)
  std::vector<double> theta, half_cos, half_sin;  // K-1
  std::vector<double> values, norm_sq, nodal_weight;
  std::vector<double> p, q;  // ((k-1)*n + l-1) * m + i
  std::vector<double> eig_coeff;  // n*K-1 eigenvalues in coefficient order

  int m() const { return order - 1; }
  int coeff_count() const { return order * elements - 1; }
};

// Builds the table; throws std::runtime_error with the reference's messages
// on failure (bracketing, nonpositive norms, order out of range).
HostTable build_host_table(int n, int K);

// Device-ready arrays for the sweep kernels (see sweep.cu for their use).
struct DeviceTableData {
  int n = 0, K = 0;
  std::vector<double> mix_fwd_w;   // (K-1) x n(l) x n(s): FC_n analysis
  std::vector<double> mix_fwd_d;   // (K-1) x n(l) x n(s): F_n analysis
  std::vector<double> mix_inv;     // (K-1) x n(s) x n(l): synthesis
  std::vector<double> e0_fwd_w;    // m x m [i][l] = e_i^(l) / K
  std::vector<double> e0_fwd_d;    // m x m [j][l] = (C~ e^(l))_j / K
  std::vector<double> e0_inv;      // m x m [i][l] = e_i^(l)
  std::vector<double> eig;         // n*K-1
  std::vector<double> nsq;         // n*K-1: ||s_k^(l)||^2 in coefficient order (1 in the k = 0 block)
  std::vector<double> mixT_w, mixT_d, mixT_i;  // n x n x K, k-contiguous (see sweep.cuh)
  std::vector<double> tw;          // 2N: exp(-2 pi i t/N)   (re, im interleaved)
  std::vector<double> mk;          // 2N: exp(-i pi k/(2N))
  std::vector<double> mkh;         // 2N: 0.5 exp(+i pi k/(2N))
  std::vector<double> om;          // 2N: exp(-i pi j/N)
};

DeviceTableData derive_device_data(const HostTable& t);

// Table files (reference save_table / load_table / build_and_save_table,
// spectral.hpp:316-330, spectral.cpp:81-236).  kTableText is the reference's
// SFEM1 text format, written byte for byte as the reference writes it (17
// significant digits) and read as the reference reads it; kTableBinary
// ("SFEMB1") carries the same primaries as raw doubles with an FNV-1a
// checksum (bit-exact, no text parse).  Loading sniffs the format and
// rebuilds the derived data (spectral.cpp:209-235).  Errors throw
// std::runtime_error with the reference's messages.
enum { kTableText = 0, kTableBinary = 1 };
void save_host_table(const HostTable& t, const std::string& path, int format);
HostTable load_host_table(const std::string& path, int n, int K);

// TableSet's on-disk cache (poisson.cpp:49-73): `dir` empty = no cache.
struct TableCache {
  std::string dir;
  bool write = true;
  int format = kTableBinary;
};
std::string table_cache_path(const std::string& dir, int n, int K, int format);
// source (optional): 0 built, 1 loaded from the text entry, 2 from the binary one.
HostTable cached_host_table(const TableCache& cache, int n, int K, int* source = nullptr);

// Gauss nodes (n+1 points) and weighted[loc*(n+1)+g] = w_g phi_loc(xi_g) of the
// load averaging (reference axis_quad, poisson.cpp:481-495).
void load_quadrature(int n, std::vector<double>& nodes, std::vector<double>& weighted);

}  // namespace sfem_b200
