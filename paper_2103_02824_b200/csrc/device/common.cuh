// Shared device utilities: error checks, launch accounting, warp reductions.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../host/mesh.hpp"

namespace ksb {

#define KSB_CUDA_CHECK(expr)                                                                  \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            ::ksb::raise(KSB_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));       \
    } while (0)

constexpr int kSMs = 148;  // B200

/// Device context: one stream, launch counters, optional per-kernel event timing.
struct Ctx {
    int device = 0;
    int sm_count = kSMs;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;              // side stream for work independent of the critical path
    cudaEvent_t fork = nullptr, join = nullptr;
    bool profiling = false;
    int64_t launches = 0;
    struct Timer {
        double ms = 0;
        int64_t count = 0;
    };
    std::map<std::string, Timer> timers;
    std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> event_pool;

    cudaEvent_t take_event();
    void begin(const char* name, cudaEvent_t* e0);
    void end(const char* name, cudaEvent_t e0);
    void harvest();  // fold completed pending timings into timers (syncs the stream)
};

/// RAII-free launch helper: counts the launch and brackets it with events when profiling.
template <typename Kernel, typename... Args>
inline void launch(Ctx& c, const char* name, Kernel k, dim3 grid, dim3 block, size_t smem, Args... args) {
    cudaEvent_t e0 = nullptr;
    if (c.profiling) c.begin(name, &e0);
    k<<<grid, block, smem, c.stream>>>(args...);
    ++c.launches;
    KSB_CUDA_CHECK(cudaGetLastError());
    if (c.profiling) c.end(name, e0);
}

/// same as launch() on an explicit stream (the context's side stream)
template <typename Kernel, typename... Args>
inline void launch_on(Ctx& c, cudaStream_t st, const char* name, Kernel k, dim3 grid, dim3 block, size_t smem,
                      Args... args) {
    cudaStream_t keep = c.stream;
    c.stream = st;  // profiling events go to the launching stream
    cudaEvent_t e0 = nullptr;
    if (c.profiling) c.begin(name, &e0);
    k<<<grid, block, smem, st>>>(args...);
    ++c.launches;
    const cudaError_t err = cudaGetLastError();
    if (c.profiling) c.end(name, e0);
    c.stream = keep;
    if (err != cudaSuccess) ::ksb::raise(KSB_CUDA, std::string("launch: ") + cudaGetErrorString(err));
}

/// make `to` wait for everything issued so far on `from`
inline void stream_wait(Ctx& c, cudaStream_t from, cudaStream_t to, cudaEvent_t ev) {
    KSB_CUDA_CHECK(cudaEventRecord(ev, from));
    KSB_CUDA_CHECK(cudaStreamWaitEvent(to, ev, 0));
    (void)c;
}

inline int ceil_div(int64_t a, int64_t b) { return int((a + b - 1) / b); }

/// number of blocks of `kernel` that are co-resident on the whole GPU (one full wave).
/// Streaming kernels sized to one wave sweep the rows in lock-step, which keeps the
/// gathered neighbour rows of an SpMM inside L2 instead of re-fetching them per wave.
template <typename Kernel>
inline int resident_grid(const Ctx& c, Kernel k, int block, size_t smem) {
    static std::map<std::pair<const void*, size_t>, int> cache;
    const auto key = std::make_pair(reinterpret_cast<const void*>(k), smem * 4096 + size_t(block));
    auto it = cache.find(key);
    if (it != cache.end()) return it->second * c.sm_count;
    int n = 0;
    KSB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, block, smem));
    n = n > 0 ? n : 1;
    cache.emplace(key, n);
    return n * c.sm_count;
}

__device__ __forceinline__ double warp_sum(double v, unsigned mask = 0xffffffffu) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
    return v;
}

} // namespace ksb
