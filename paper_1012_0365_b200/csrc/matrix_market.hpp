// Matrix Market I/O (core/matrix_market.hpp), host side.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace blws {

using Index = std::int64_t;

struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void mm_write_dense(const std::string& path, Index rows, Index cols, const double* a, Index lda);
void mm_write_sparse(const std::string& path, Index rows, Index cols, Index nnz, const std::int64_t* colptr,
                     const std::int32_t* rowidx, const double* values);
/// data == nullptr: size query only.
void mm_read_dense(const std::string& path, Index* rows, Index* cols, std::vector<double>* data);
/// CSC (rows ascending within each column, as Eigen's setFromTriplets + makeCompressed).
void mm_read_sparse(const std::string& path, Index* rows, Index* cols, std::vector<std::int64_t>* colptr,
                    std::vector<std::int32_t>* rowidx, std::vector<double>* values);

}  // namespace blws
