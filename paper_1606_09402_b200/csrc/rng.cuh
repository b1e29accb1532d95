// Device Gaussian generator bit-compatible (integer stream) with the reference
// RngStream (/root/reference/proj/src/rng.cpp). See rng.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace qbgpu {

constexpr int kJumpLevels = 64;  // T^(2^k), k < 64

// Device copy of the xoshiro256 jump matrices (512 KB), uploaded once per context.
class RngTables {
public:
    RngTables() = default;
    RngTables(const RngTables&) = delete;
    RngTables& operator=(const RngTables&) = delete;
    ~RngTables();
    const std::uint64_t* device();

private:
    std::uint64_t* dev_ = nullptr;
};

// State of RngStream(seed, stream) before its first draw (rng.cpp:28-34).
void stream_origin(std::uint64_t seed, std::uint64_t stream, std::uint64_t (&s)[4]);
std::uint64_t host_next_u64(std::uint64_t (&s)[4]);

// Writes gaussians g0 .. g0 + rows*cols - 1 of stream (seed, stream) into `out`
// in column-major fill order (element e -> (e % rows, e / rows)), i.e. exactly what
// gaussian(rows, cols, rng) returns after g0 earlier next_gaussian() draws.
void gaussian_fill(cudaStream_t st, RngTables& tables, std::uint64_t seed, std::uint64_t stream,
                   std::uint64_t g0, const MatView& out);

}  // namespace qbgpu
