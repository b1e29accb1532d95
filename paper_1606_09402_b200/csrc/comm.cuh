// NCCL plumbing for row-sharded A (one process per GPU). NCCL is loaded with
// dlopen only when world > 1, so a single-GPU run never touches it and the
// library does not pin a particular libnccl at link time (torch ships its own).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

namespace qbgpu {

// In-process rank group on ONE device (test harness for the row-sharded engine): every rank is a
// Context driven by its own host thread; allreduce_sum synchronizes the rank's stream, meets the
// others at a host barrier, and rank 0 sums the buffers in rank order (deterministic, the same
// order NCCL's ring would not guarantee). Kernels never wait on each other — only host threads do.
struct LocalGroup {
    explicit LocalGroup(int w)
        : world(w), ptrs(static_cast<std::size_t>(w), nullptr), cptrs(static_cast<std::size_t>(w), nullptr) {}
    ~LocalGroup();
    void barrier();
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned gen = 0;
    std::vector<double*> ptrs;
    std::vector<const double*> cptrs;
    double* sum = nullptr;
    std::size_t cap = 0;
};

class Comm {
public:
    Comm(int rank, int world, const void* unique_id128);
    Comm(int rank, int world, std::shared_ptr<LocalGroup> group);  // in-process loopback (tests)
    ~Comm();
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;

    int rank() const { return rank_; }
    int world() const { return world_; }
    // In-place sum over ranks on `st` (ncclAllReduce, ncclDouble, ncclSum).
    void allreduce_sum(double* p, std::size_t count, cudaStream_t st);
    // recv (recvcount) = block `rank` of the sum over ranks of send (world * recvcount)
    // (ncclReduceScatter, ncclDouble, ncclSum).
    void reduce_scatter_sum(const double* send, double* recv, std::size_t recvcount, cudaStream_t st);
    // recv (world * sendcount) = the send blocks of all ranks in rank order (ncclAllGather).
    void all_gather(const double* send, double* recv, std::size_t sendcount, cudaStream_t st);

    static void unique_id(void* out128);

private:
    int rank_, world_;
    void* comm_ = nullptr;
    std::shared_ptr<LocalGroup> local_;
};

}  // namespace qbgpu
