// NCCL over NVLink/NVSwitch for the row-sharded path: the only
// collectives are the n x w allreduce after every A^T pass and the small Gram
// allreduces (k x b, b x b) plus one scalar for ||A||_F^2.

#include "comm.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

namespace qbgpu {

namespace {

struct NcclApi {
    void* handle = nullptr;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclReduceScatter) reduce_scatter = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            a.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (a.handle) break;
        }
        if (!a.handle) return;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.handle, "ncclGetUniqueId"));
        a.init_rank = reinterpret_cast<decltype(a.init_rank)>(dlsym(a.handle, "ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(a.handle, "ncclAllReduce"));
        a.reduce_scatter = reinterpret_cast<decltype(a.reduce_scatter)>(dlsym(a.handle, "ncclReduceScatter"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(a.handle, "ncclAllGather"));
        a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(a.handle, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.handle, "ncclGetErrorString"));
    });
    if (!a.handle || !a.get_unique_id || !a.init_rank || !a.all_reduce || !a.reduce_scatter || !a.all_gather ||
        !a.destroy)
        throw QbError(kError, "NCCL (libnccl.so.2) is not available");
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* msg = api().error_string ? api().error_string(r) : "nccl error";
        throw QbError(kError, std::string(what) + ": " + msg);
    }
}

}  // namespace

LocalGroup::~LocalGroup() {
    if (sum) cudaFree(sum);
}

void LocalGroup::barrier() {
    std::unique_lock<std::mutex> l(mu);
    const unsigned g = gen;
    if (++arrived == world) {
        arrived = 0;
        ++gen;
        cv.notify_all();
    } else {
        cv.wait(l, [&] { return gen != g; });
    }
}

namespace {
__global__ void local_add_kernel(double* __restrict__ d, const double* __restrict__ s, std::size_t n) {
    for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::size_t>(gridDim.x) * blockDim.x)
        d[i] += s[i];
}
}  // namespace

Comm::Comm(int rank, int world, std::shared_ptr<LocalGroup> group) : rank_(rank), world_(world), local_(std::move(group)) {
    if (!local_ || world != local_->world || rank < 0 || rank >= world) throw QbError(kDimensionError, "bad local group");
}

Comm::Comm(int rank, int world, const void* unique_id128) : rank_(rank), world_(world) {
    if (world < 1 || rank < 0 || rank >= world) throw QbError(kDimensionError, "bad rank/world");
    if (!unique_id128) throw QbError(kError, "NCCL communicator needs a unique id");
    ncclUniqueId id;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(&id, unique_id128, sizeof(id));
    ncclComm_t c = nullptr;
    check(api().init_rank(&c, world, id, rank), "ncclCommInitRank");
    comm_ = c;
}

Comm::~Comm() {
    if (comm_) api().destroy(static_cast<ncclComm_t>(comm_));
}

void Comm::allreduce_sum(double* p, std::size_t count, cudaStream_t st) {
    if (local_) {
        LocalGroup& g = *local_;
        QB_CUDA(cudaStreamSynchronize(st));
        g.ptrs[static_cast<std::size_t>(rank_)] = p;
        g.barrier();
        if (rank_ == 0 && count) {
            if (g.cap < count) {
                if (g.sum) QB_CUDA(cudaFree(g.sum));
                QB_CUDA(cudaMalloc(&g.sum, count * sizeof(double)));
                g.cap = count;
            }
            QB_CUDA(cudaMemcpyAsync(g.sum, g.ptrs[0], count * sizeof(double), cudaMemcpyDeviceToDevice, st));
            for (int r = 1; r < world_; ++r)
                local_add_kernel<<<static_cast<unsigned>(std::min<std::size_t>((count + 255) / 256, 1024)), 256, 0, st>>>(
                    g.sum, g.ptrs[static_cast<std::size_t>(r)], count);
            QB_CUDA(cudaStreamSynchronize(st));
        }
        g.barrier();
        if (count) QB_CUDA(cudaMemcpyAsync(p, g.sum, count * sizeof(double), cudaMemcpyDeviceToDevice, st));
        QB_CUDA(cudaStreamSynchronize(st));
        g.barrier();
        return;
    }
    if (!comm_ || count == 0) return;
    check(api().all_reduce(p, p, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm_), st),
          "ncclAllReduce");
}

void Comm::reduce_scatter_sum(const double* send, double* recv, std::size_t recvcount, cudaStream_t st) {
    if (local_) {
        // loopback: rank 0 sums the full send buffers in rank order, every rank copies its block
        LocalGroup& g = *local_;
        const std::size_t total = recvcount * static_cast<std::size_t>(world_);
        QB_CUDA(cudaStreamSynchronize(st));
        g.cptrs[static_cast<std::size_t>(rank_)] = send;
        g.barrier();
        if (rank_ == 0 && total) {
            if (g.cap < total) {
                if (g.sum) QB_CUDA(cudaFree(g.sum));
                QB_CUDA(cudaMalloc(&g.sum, total * sizeof(double)));
                g.cap = total;
            }
            QB_CUDA(cudaMemcpyAsync(g.sum, g.cptrs[0], total * sizeof(double), cudaMemcpyDeviceToDevice, st));
            for (int r = 1; r < world_; ++r)
                local_add_kernel<<<static_cast<unsigned>(std::min<std::size_t>((total + 255) / 256, 1024)), 256, 0, st>>>(
                    g.sum, g.cptrs[static_cast<std::size_t>(r)], total);
            QB_CUDA(cudaStreamSynchronize(st));
        }
        g.barrier();
        if (recvcount)
            QB_CUDA(cudaMemcpyAsync(recv, g.sum + static_cast<std::size_t>(rank_) * recvcount, recvcount * sizeof(double),
                                    cudaMemcpyDeviceToDevice, st));
        QB_CUDA(cudaStreamSynchronize(st));
        g.barrier();
        return;
    }
    if (!comm_) {
        if (recvcount && recv != send)
            QB_CUDA(cudaMemcpyAsync(recv, send, recvcount * sizeof(double), cudaMemcpyDeviceToDevice, st));
        return;
    }
    if (recvcount == 0) return;
    check(api().reduce_scatter(send, recv, recvcount, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm_), st),
          "ncclReduceScatter");
}

void Comm::all_gather(const double* send, double* recv, std::size_t sendcount, cudaStream_t st) {
    if (local_) {
        // loopback: every rank writes its block of a shared buffer, then copies the whole buffer
        LocalGroup& g = *local_;
        const std::size_t total = sendcount * static_cast<std::size_t>(world_);
        QB_CUDA(cudaStreamSynchronize(st));
        g.barrier();
        if (rank_ == 0 && g.cap < total) {
            if (g.sum) QB_CUDA(cudaFree(g.sum));
            QB_CUDA(cudaMalloc(&g.sum, total * sizeof(double)));
            g.cap = total;
        }
        g.barrier();
        if (sendcount)
            QB_CUDA(cudaMemcpyAsync(g.sum + static_cast<std::size_t>(rank_) * sendcount, send, sendcount * sizeof(double),
                                    cudaMemcpyDeviceToDevice, st));
        QB_CUDA(cudaStreamSynchronize(st));
        g.barrier();
        if (total) QB_CUDA(cudaMemcpyAsync(recv, g.sum, total * sizeof(double), cudaMemcpyDeviceToDevice, st));
        QB_CUDA(cudaStreamSynchronize(st));
        g.barrier();
        return;
    }
    if (!comm_) {
        if (sendcount && recv != send)
            QB_CUDA(cudaMemcpyAsync(recv, send, sendcount * sizeof(double), cudaMemcpyDeviceToDevice, st));
        return;
    }
    if (sendcount == 0) return;
    check(api().all_gather(send, recv, sendcount, ncclDouble, static_cast<ncclComm_t>(comm_), st), "ncclAllGather");
}

void Comm::unique_id(void* out128) {
    ncclUniqueId id;
    check(api().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
}

}  // namespace qbgpu
