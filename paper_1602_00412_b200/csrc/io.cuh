// io.cuh -- parallel ingestion of row-stream files (see io.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <string>

namespace sfdg {

// Reads a MatrixMarket coordinate file or a plain "col:value" file (plain_cols = column
// count; 0 = the file must be MatrixMarket), the reference's open_row_stream contract
// (core/src/io.cpp:170-189). Rows are delivered in file order as CSR batches (row_ptr
// relative, nrows + 1 entries) to `sink`; *d_out is set before the first batch. Errors
// throw invalid_argument with the reference's messages after the rows before the bad line
// were delivered.
void read_row_stream(const std::string& path, size_t plain_cols, size_t window_bytes, size_t* d_out,
                     const std::function<void(const int64_t*, const uint32_t*, const double*, size_t)>& sink);

}  // namespace sfdg
