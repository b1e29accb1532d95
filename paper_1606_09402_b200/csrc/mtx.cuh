// Matrix Market read / write (host side, sparse_csr.cpp:42-64).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"

namespace qbgpu {

struct MtxInfo {
    bool coordinate;
    std::int64_t m, n, nnz;
};

MtxInfo mtx_info(const std::string& path);
void mtx_read_csr(const std::string& path, MtxInfo& info, std::vector<std::int64_t>& rp,
                  std::vector<std::int32_t>& ci, std::vector<double>& v);
void mtx_read_dense(const std::string& path, MtxInfo& info, std::vector<double>& a);
void mtx_write_csr(const std::string& path, std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                   const std::int32_t* ci, const double* v);
void mtx_write_dense(const std::string& path, std::int64_t m, std::int64_t n, const double* a, std::int64_t lda);

}  // namespace qbgpu
