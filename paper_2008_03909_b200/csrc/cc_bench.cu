// cc_bench.cu -- K10 measurement-floor kernels (include/cc_bench.h).
//
// MapEdges / GatherEdges (Table 8) on the device CSR, a uniform
// random 4-byte gather (the random-sector ceiling) and a streaming copy.
#include <cuda_runtime.h>

#include "../../include/cc_bench.h"
#include "cc_device.cuh"
#include "cc_internal.h"

namespace ccb {

// One warp per tile of 32 consecutive vertices: the warp sweeps the tile's
// concatenated lists with coalesced loads; each entry's owner lane is found by
// a binary search over the 33 tile offsets in shared memory and its value is
// accumulated with a shared-memory atomic (segmented reduction).
template <bool GATHER>
__global__ void __launch_bounds__(kBlock) k_edges(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                  uint32_t n, const uint32_t* __restrict__ x,
                                                  uint32_t* __restrict__ out)
{
    __shared__ int64_t s_off[kBlock / 32][33];
    __shared__ uint32_t s_acc[kBlock / 32][32];
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = warp * 32; t < n; t += nwarps * 32) {
        const uint64_t v = t + lane;
        const int64_t m_end = off[n];
        s_off[w][lane] = v < n ? off[v] : m_end;
        if (lane == 0) s_off[w][32] = (t + 32 < n) ? off[t + 32] : m_end;
        s_acc[w][lane] = 0;
        __syncwarp();
        const int64_t tb = s_off[w][0], te = s_off[w][32];
        for (int64_t i = tb + lane; i < te; i += 32) {
            const uint32_t a = ld_stream_u32(adj + i);
            const uint32_t val = GATHER ? x[a] : (a != 0xFFFFFFFFu ? 1u : 0u);
            int lo = 0, hi = 31;                     // owner: last lane with s_off <= i
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_off[w][mid] <= i) lo = mid; else hi = mid - 1;
            }
            atomicAdd(&s_acc[w][lo], val);
        }
        __syncwarp();
        if (v < n) out[v] = s_acc[w][lane];
        __syncwarp();
    }
}

__global__ void __launch_bounds__(kBlock) k_random_gather(const uint32_t* __restrict__ x, uint64_t len,
                                                          uint64_t count, uint64_t seed, uint32_t* out)
{
    uint32_t acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
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
    k_edges<false><<<num_sms() * 16, kBlock, 0, (cudaStream_t)stream>>>(offsets, adj, n, nullptr, out);
    CC_LAUNCH_CHECK("k_edges<map>");
    return CC_OK;
}

cc_status cc_bench_gather_edges(const int64_t* offsets, const uint32_t* adj, uint32_t n, const uint32_t* x,
                                uint32_t* out, void* stream)
{
    if (n == 0) return CC_OK;
    if (!offsets || !adj || !out || !x) return CC_EINVAL;
    k_edges<true><<<num_sms() * 16, kBlock, 0, (cudaStream_t)stream>>>(offsets, adj, n, x, out);
    CC_LAUNCH_CHECK("k_edges<gather>");
    return CC_OK;
}

cc_status cc_bench_random_gather(const uint32_t* x, uint64_t len, uint64_t count, uint64_t seed, uint32_t* out,
                                 void* stream)
{
    if (!x || !out || len == 0) return CC_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    CC_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(uint32_t), s));
    k_random_gather<<<num_sms() * 16, kBlock, 0, s>>>(x, len, count, seed, out);
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

}  // extern "C"
