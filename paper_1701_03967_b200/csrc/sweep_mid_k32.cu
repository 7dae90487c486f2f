// General-shape mid kernels for K = 32, every order (mid::AutoShape); see
// sweep_mid.cu.  One translation unit per K so the library builds in parallel.
#include "sweep_mid_impl.cuh"

namespace sfem_b200 {
namespace mid {
template cudaError_t launch_auto_n<32>(const DevTable&, const LineSet&, int, int, const SymbolInfo*, cudaStream_t);
template cudaError_t launch_auto_tma_n<32>(const DevTable&, const void*, const TmaGeom&, int, int, cudaStream_t);
template cudaError_t launch_auto_tma_cm_n<32>(const DevTable&, const void*, const TmaGeom&, int, int, cudaStream_t);
}  // namespace mid
}  // namespace sfem_b200
