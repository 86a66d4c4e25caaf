// cc_bench.cu -- K10 measurement-floor kernels (include/cc_bench.h).
//
// MapEdges / GatherEdges (Table 8) on the device CSR, a uniform
// random 4-byte gather (the random-sector ceiling) and a streaming copy.
#include <cuda_runtime.h>

#include "../../include/cc_bench.h"
#include "cc_device.cuh"
#include "cc_internal.h"

namespace ccb {

// Edge-balanced sweep: warp c owns adjacency entries [c*kChunk, (c+1)*kChunk)
// whatever the degrees (hubs are split across warps), finds the owner of its
// first entry by a binary search of the offsets, then reads 4 entries per lane
// per iteration (coalesced, 4 loads in flight).  Each lane follows the owner of
// its next entry with a monotone pointer and adds its running sum into out[]
// with one atomic whenever the owner changes (out is zeroed first).
constexpr int64_t kChunk = 4096;

template <bool GATHER>
__global__ void __launch_bounds__(kBlock) k_edges(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                  uint32_t n, int64_t m, const uint32_t* __restrict__ x,
                                                  uint32_t* __restrict__ out)
{
    const unsigned lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c0 = warp * kChunk; c0 < m; c0 += nwarps * kChunk) {
        const int64_t c1 = min(c0 + kChunk, m);
        uint32_t lo = 0, hi = n;                           // largest v with off[v] <= c0
        if (lane == 0) {
            while (hi - lo > 1) {
                const uint32_t mid = lo + (hi - lo) / 2;
                if (off[mid] <= c0) lo = mid; else hi = mid;
            }
        }
        uint32_t own = __shfl_sync(0xffffffffu, lo, 0);
        int64_t own_end = off[own + 1];
        uint32_t run = 0;
        for (int64_t i0 = c0 + lane; i0 < c1; i0 += 128) {
            uint32_t val[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t i = i0 + 32 * j;
                uint32_t a = 0xFFFFFFFFu;
                if (i < c1) a = __ldcs(adj + i);
                val[j] = (i < c1) ? (GATHER ? x[a] : (a != 0xFFFFFFFFu ? 1u : 0u)) : 0u;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t i = i0 + 32 * j;
                if (i >= c1) break;
                if (i >= own_end) {                         // move to the owner of entry i
                    if (run) atomicAdd(out + own, run);
                    run = 0;
                    do {
                        ++own;
                        own_end = off[own + 1];
                    } while (own_end <= i);
                }
                run += val[j];
            }
        }
        if (run) atomicAdd(out + own, run);
    }
}

__global__ void __launch_bounds__(kBlock) k_random_gather(const uint32_t* __restrict__ x, uint64_t len,
                                                          uint64_t count, uint64_t seed, uint32_t* out)
{
    uint32_t acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // 16 independent loads in flight per thread: the probe (scripts/probe/randgather.cu)
    // found this, with a 32-blocks-per-SM grid, the fastest configuration on B200
    for (; i + 15 * stride < count; i += 16 * stride) {
        uint32_t t[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint64_t r = splitmix64(seed + i + j * stride);
            t[j] = __ldcg(x + (((r & 0xFFFFFFFFull) * len) >> 32));
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += t[j];
    }
    for (; i < count; i += stride) {
        const uint64_t r = splitmix64(seed + i);
        acc += __ldcg(x + (((r & 0xFFFFFFFFull) * len) >> 32));
    }
    acc = __reduce_add_sync(0xffffffffu, acc);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

__global__ void __launch_bounds__(kBlock) k_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t n4)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) dst[i] = src[i];
}

}  // namespace ccb

using namespace ccb;

extern "C" {

cc_status cc_bench_map_edges(const int64_t* offsets, const uint32_t* adj, uint32_t n, uint32_t* out, void* stream)
{
    if (n == 0) return CC_OK;
    if (!offsets || !adj || !out) return CC_EINVAL;
    int64_t m = 0;
    cudaStream_t s = (cudaStream_t)stream;
    CC_CUDA_TRY(cudaMemcpyAsync(&m, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CC_CUDA_TRY(cudaStreamSynchronize(s));
    CC_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(uint32_t) * n, s));
    k_edges<false><<<num_sms() * 16, kBlock, 0, s>>>(offsets, adj, n, m, nullptr, out);
    CC_LAUNCH_CHECK("k_edges<map>");
    return CC_OK;
}

cc_status cc_bench_gather_edges(const int64_t* offsets, const uint32_t* adj, uint32_t n, const uint32_t* x,
                                uint32_t* out, void* stream)
{
    if (n == 0) return CC_OK;
    if (!offsets || !adj || !out || !x) return CC_EINVAL;
    int64_t m = 0;
    cudaStream_t s = (cudaStream_t)stream;
    CC_CUDA_TRY(cudaMemcpyAsync(&m, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CC_CUDA_TRY(cudaStreamSynchronize(s));
    CC_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(uint32_t) * n, s));
    k_edges<true><<<num_sms() * 16, kBlock, 0, s>>>(offsets, adj, n, m, x, out);
    CC_LAUNCH_CHECK("k_edges<gather>");
    return CC_OK;
}

cc_status cc_bench_random_gather(const uint32_t* x, uint64_t len, uint64_t count, uint64_t seed, uint32_t* out,
                                 void* stream)
{
    if (!x || !out || len == 0) return CC_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    CC_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(uint32_t), s));
    k_random_gather<<<num_sms() * 32, kBlock, 0, s>>>(x, len, count, seed, out);
    CC_LAUNCH_CHECK("k_random_gather");
    return CC_OK;
}

cc_status cc_bench_copy(const uint32_t* src, uint32_t* dst, uint64_t words, void* stream)
{
    if (!src || !dst || (words & 3)) return CC_EINVAL;
    k_copy<<<num_sms() * 8, kBlock, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dst, words / 4);
    CC_LAUNCH_CHECK("k_copy");
    return CC_OK;
}

cc_status cc_bench_set_l2_fetch(int bytes, int* prev)
{
    size_t old = 0;
    CC_CUDA_TRY(cudaDeviceGetLimit(&old, cudaLimitMaxL2FetchGranularity));
    if (prev) *prev = (int)old;
    CC_CUDA_TRY(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes));
    return CC_OK;
}

uint64_t cc_bench_launch_count(void) { return g_launches.load(); }

unsigned cc_bench_set_grid(unsigned blocks) { return g_grid_override.exchange(blocks); }

}  // extern "C"
