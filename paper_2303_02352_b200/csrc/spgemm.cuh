// spgemm.cuh -- general C = A*B (host CSR in/out, device compute) in the
// reference's spgemm_local summation order (csr.cpp:206-272).
#pragma once

#include <cuda_runtime.h>

#include "mmio.cuh"

namespace pb {

// A: an x am (row_ptr, col, val), B: am x bm.  Columns need not be sorted;
// duplicates are summed like any other contribution.
HostCsr spgemm(int64_t an, int64_t am, const int64_t* a_rp, const int64_t* a_col, const double* a_val, int64_t bm,
               const int64_t* b_rp, const int64_t* b_col, const double* b_val, cudaStream_t s);

}  // namespace pb
