// cc_common.cuh -- device helpers shared by the static (cc_static.cu) and AMSF
// (cc_amsf.cu) pipelines: warp/block scans, queue appends, and the Filter of
// Alg. 2 that compacts the forest slots (static kernels: one copy per
// translation unit).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "cc_internal.h"

namespace ccb {

constexpr uint32_t kSentinel = 0xFFFFFFFFu;
constexpr int kFItems = 16;                  // forest/SV scans: slots per thread
constexpr int kFTile = kBlock * kFItems;     // forest/SV scans: slots per block

// Exclusive warp prefix of c and one atomicAdd per warp; every lane must call.
static __device__ __forceinline__ unsigned long long warp_append(unsigned long long* counter, uint32_t c)
{
    const unsigned lane = threadIdx.x & 31;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += t;
    }
    uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(counter, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    return base + incl - c;
}

static __device__ __forceinline__ void warp_count(uint64_t* ctr, uint32_t c)
{
    if (!ctr) return;
    uint32_t s = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(reinterpret_cast<unsigned long long*>(ctr), (unsigned long long)s);
}

// Block-wide exclusive scan of one value per thread; *total = block sum.
static __device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* total)
{
    constexpr int NW = kBlock / 32;
    __shared__ uint32_t ws[NW];
    __shared__ uint32_t tot;
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += t;
    }
    if (lane == 31) ws[w] = incl;
    __syncthreads();
    if (w == 0) {
        const uint32_t sv = lane < (unsigned)NW ? ws[lane] : 0u;
        uint32_t si = sv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= (unsigned)o) si += t;
        }
        if (lane < (unsigned)NW) ws[lane] = si - sv;
        if (lane == (unsigned)NW - 1) tot = si;
    }
    __syncthreads();
    const uint32_t r = ws[w] + incl - x;
    *total = tot;
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// K7: Filter -- stable compaction of the non-sentinel forest slots.

static __global__ void __launch_bounds__(kBlock) k_forest_count(const uint2* F, uint32_t n, uint32_t* block_cnt)
{
    uint32_t tot;
    const uint64_t base = (uint64_t)blockIdx.x * kFTile + (uint64_t)threadIdx.x * kFItems;
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < kFItems; ++j)
        if (base + j < n && F[base + j].x != kSentinel) ++c;
    block_excl_scan(c, &tot);
    if (threadIdx.x == 0) block_cnt[blockIdx.x] = tot;
}

// single CTA: exclusive scan of the per-block counts (64-bit running total)
static __global__ void __launch_bounds__(kBlock) k_forest_scan(const uint32_t* block_cnt, uint32_t nb,
                                                        unsigned long long* block_off, int64_t* num_edges)
{
    uint32_t tot;
    unsigned long long carry = 0;
    for (uint32_t base = 0; base < nb; base += kBlock) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t x = i < nb ? block_cnt[i] : 0;
        const uint32_t ex = block_excl_scan(x, &tot);
        if (i < nb) block_off[i] = carry + ex;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *num_edges = (int64_t)carry;
}

// Fw / out_w (optional, AMSF): the weight stored with each slot, compacted alongside
static __global__ void __launch_bounds__(kBlock) k_forest_write(const uint2* F, uint32_t n,
                                                                const unsigned long long* block_off,
                                                                uint32_t* edges, const float* Fw = nullptr,
                                                                float* out_w = nullptr)
{
    uint32_t tot;
    const uint64_t base = (uint64_t)blockIdx.x * kFTile + (uint64_t)threadIdx.x * kFItems;
    uint2 f[kFItems];
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < kFItems; ++j) {
        f[j] = (base + j < n) ? F[base + j] : make_uint2(kSentinel, kSentinel);
        c += f[j].x != kSentinel;
    }
    uint32_t ex = block_excl_scan(c, &tot);
    unsigned long long o = block_off[blockIdx.x] + ex;
#pragma unroll
    for (int j = 0; j < kFItems; ++j)
        if (f[j].x != kSentinel) {
            reinterpret_cast<uint2*>(edges)[o] = f[j];
            if (out_w) out_w[o] = Fw[base + j];
            ++o;
        }
}

}  // namespace ccb
