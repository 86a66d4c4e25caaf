// cc_internal.h -- host-side internals shared by the libcc.so translation units.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "../../include/cc.h"

namespace ccb {

// Thread-local detail string for cc_last_error().
void set_error(const std::string& msg);
cc_status cuda_fail(cudaError_t e, const char* where);

// Cumulative count of kernels this library launched (bench evidence).
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int num_sms();
// Blocks of a grid-strided kernel: num_sms() * per_sm, unless a test set an
// override (cc_bench_set_grid) -- such kernels are correct for any grid size.
unsigned grid_blocks(unsigned per_sm);
extern std::atomic<unsigned> g_grid_override;
// One wave of a grid-strided kernel: num_sms() x the blocks of `block` threads
// that fit on one SM (occupancy query, cached per kernel), so static grid-stride
// work splits never leave a partial second wave; the test override applies.
unsigned resident_blocks(const void* kernel, int block);
template <class K>
inline unsigned resident_grid(K* kernel, int block)
{
    return resident_blocks(reinterpret_cast<const void*>(kernel), block);
}
bool is_device_ptr(const void* p);

// Where an array argument lives: device memory, pinned host memory (device-
// accessible through UVA: used in place, zero-copy), or pageable host memory
// (staged through device scratch).
enum MemKind { MEM_DEVICE = 0, MEM_PINNED = 1, MEM_PAGEABLE = 2 };
MemKind mem_kind(const void* p, void** dev_alias);

// Stream-ordered scratch from the device's default memory pool (cached).
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s);
void scratch_free(void* p, cudaStream_t s);

constexpr int kBlock = 256;

#define CC_CUDA_TRY(expr)                                         \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return ::ccb::cuda_fail(_e, #expr); \
    } while (0)

// Launch-error check after a <<<>>> launch.
#define CC_LAUNCH_CHECK(name)                                     \
    do {                                                          \
        ::ccb::count_launch();                                    \
        cudaError_t _e = cudaGetLastError();                      \
        if (_e != cudaSuccess) return ::ccb::cuda_fail(_e, name); \
    } while (0)

// Launch with programmatic dependent launch (PDL) allowed: the kernel may be
// scheduled while the previous kernel of the stream still runs; it must execute
// pdl_wait() before touching memory the previous kernel writes.
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, Args... args);

// launch_pdl, or an ordinary launch (full dependency on the previous work of the
// stream, its writes visible from the kernel's first instruction) when !pdl
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl_if(bool pdl, void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t s,
                                 Args... args)
{
    if (pdl) return launch_pdl(kernel, grid, block, s, args...);
    kernel<<<grid, block, 0, s>>>(static_cast<KArgs>(args)...);
    return cudaGetLastError();
}

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Device pipeline entry points (device pointers only; validated args).
cc_status static_pipeline(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, uint32_t* P,
                          uint32_t* labels_out, uint32_t* edges, int64_t* num_edges, bool sf, const cc_opts& o,
                          cudaStream_t s);
cc_status amsf_pipeline(const int64_t* off, const uint32_t* adj, const float* w, uint32_t n, int64_t m, double eps,
                        uint32_t* edges, float* edge_w, int64_t* num_edges, double* total, const cc_opts& o,
                        cudaStream_t s);
cc_status validate_csr(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, cudaStream_t s);

}  // namespace ccb
