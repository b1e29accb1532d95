// Shared device/host helpers for the qbfac B200 path (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace qbgpu {

// Status codes of the C-ABI (include/qbfac_gpu.h); they mirror the reference's
// exception hierarchy (/root/reference/proj/include/qbfac/types.hpp:16-66).
enum Status : int {
    kOk = 0,
    kDimensionError = 1,
    kSingularityError = 2,
    kToleranceFloorError = 3,
    kFormatError = 4,
    kResourceError = 5,
    kError = 6,
    kInternal = 7,
};

struct QbError : std::runtime_error {
    int status;
    std::int64_t diag_index = 0;
    double floor = 0.0;
    QbError(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    const int st = (e == cudaErrorMemoryAllocation) ? kResourceError : kError;
    throw QbError(st, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                          std::to_string(line) + ")");
}

#define QB_CUDA(call)                                                     \
    do {                                                                  \
        cudaError_t qb_e_ = (call);                                       \
        if (qb_e_ != cudaSuccess) ::qbgpu::throw_cuda(qb_e_, #call, __FILE__, __LINE__); \
    } while (0)

// Every kernel launch of the library is followed by QB_LAUNCH_CHECK(), which
// also counts it: process-wide, and for the context whose C-ABI call is running on this
// thread (qbfac_gpu_kernel_launches(ctx); the C-ABI guard installs t_launch_counter).
extern std::atomic<long long> g_kernel_launches;
extern thread_local long long* t_launch_counter;
#define QB_LAUNCH_CHECK()                                   \
    do {                                                    \
        ::qbgpu::g_kernel_launches.fetch_add(1, std::memory_order_relaxed); \
        if (::qbgpu::t_launch_counter) ++*::qbgpu::t_launch_counter; \
        QB_CUDA(cudaPeekAtLastError());                     \
    } while (0)

// One-time, per-DEVICE kernel setup (cudaFuncSetAttribute and occupancy queries are
// per-device state): `init` runs once for each device a process launches on, under
// std::call_once, and its value (e.g. resident CTAs per SM) is cached per device.
template <typename T>
class PerDevice {
public:
    template <typename F>
    T get(F&& init) {
        int dev = 0;
        QB_CUDA(cudaGetDevice(&dev));
        if (dev < 0 || dev >= kMax) throw QbError(kError, "device ordinal out of range");
        std::call_once(once_[dev], [&] { val_[dev] = init(); });
        return val_[dev];
    }

private:
    static constexpr int kMax = 64;
    std::once_flag once_[kMax];
    T val_[kMax] = {};
};

inline std::int64_t round_up(std::int64_t x, std::int64_t a) { return (x + a - 1) / a * a; }
inline std::int64_t ceil_div(std::int64_t x, std::int64_t a) { return (x + a - 1) / a; }

// A strided view of a logical rows x cols FP64 matrix in device memory.
// rowmajor == false: element (i, j) at p[i + j*ld]   (column-major, the reference's layout)
// rowmajor == true : element (i, j) at p[i*ld + j]
struct MatView {
    double* p = nullptr;
    std::int64_t rows = 0, cols = 0, ld = 0;
    bool rowmajor = false;

    __host__ __device__ double* at(std::int64_t i, std::int64_t j) const {
        return rowmajor ? p + i * ld + j : p + i + j * ld;
    }
    // Logical transpose (no data movement).
    MatView t() const { return MatView{p, cols, rows, ld, !rowmajor}; }
    // Sub-block [r0, r0+nr) x [c0, c0+nc).
    MatView block(std::int64_t r0, std::int64_t c0, std::int64_t nr, std::int64_t nc) const {
        return MatView{at(r0, c0), nr, nc, ld, rowmajor};
    }
    MatView cols_range(std::int64_t c0, std::int64_t nc) const { return block(0, c0, rows, nc); }
    MatView rows_range(std::int64_t r0, std::int64_t nr) const { return block(r0, 0, nr, cols); }
};

// Programmatic dependent launch (PDL): GEMM and split-K-reduce launches may start while the
// previous kernel on the stream drains; they execute griddepcontrol.wait before touching memory,
// and each GEMM CTA signals launch_dependents once its last work item is done.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("QBFAC_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    QB_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

}  // namespace qbgpu
