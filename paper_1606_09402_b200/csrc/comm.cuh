// NCCL plumbing for row-sharded A (one process per GPU). NCCL is loaded with
// dlopen only when world > 1, so a single-GPU run never touches it and the
// library does not pin a particular libnccl at link time (torch ships its own).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace qbgpu {

class Comm {
public:
    Comm(int rank, int world, const void* unique_id128);
    ~Comm();
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;

    int rank() const { return rank_; }
    int world() const { return world_; }
    // In-place sum over ranks on `st` (ncclAllReduce, ncclDouble, ncclSum).
    void allreduce_sum(double* p, std::size_t count, cudaStream_t st);

    static void unique_id(void* out128);

private:
    int rank_, world_;
    void* comm_ = nullptr;
};

}  // namespace qbgpu
