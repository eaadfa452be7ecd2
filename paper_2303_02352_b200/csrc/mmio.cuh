// mmio.cuh -- MatrixMarket ingest (mm_io.cpp) into a host CSR; row blocks of it
// are handed out as distribute_matrix does (dist.cpp:349-363).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace pb {

struct HostCsr {
    int64_t nrows = 0, ncols = 0;
    std::vector<int64_t> row_ptr;  // nrows+1
    std::vector<int64_t> col;      // global, strictly ascending per row
    std::vector<double> val;
};

HostCsr read_matrix_market(const std::string& path);
void write_matrix_market(const std::string& path, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                         const int64_t* col, const double* val);

}  // namespace pb
