// Multi-GPU slab transposes (dist.cu).
#pragma once

#include <cuda_runtime.h>

namespace sfem_b200 {

// x-slab [lx][L1][rest] viewed as (a0l, q) with q = a1 * R + r.
struct SlabView {
  long long lx;   // local rows of axis 0
  long long bpitch;  // exchange-buffer row pitch (lx rounded up to even; pad column written as 0)
  long long Q;    // L1 * R
  long long R;    // product of the rest extents (1 for N = 2)
  long long st0;  // x stride of axis 0 (elements)
  long long st1;  // x stride of axis 1
  long long st2;  // x stride of axis 2 (nrest == 2)
  long long e3;   // extent of axis 3 (nrest == 2)
  int nrest;      // number of axes after axis 1 (0, 1 or 2)
};

// to_buf: x-slab -> buf[q][a0l]; otherwise the inverse.
cudaError_t launch_slab_transpose(const SlabView& v, double* x, double* buf, bool to_buf, cudaStream_t stream);

}  // namespace sfem_b200
