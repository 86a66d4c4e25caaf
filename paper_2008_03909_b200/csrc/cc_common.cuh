// cc_common.cuh -- device helpers shared by the static (cc_static.cu) and AMSF
// (cc_amsf.cu) pipelines: warp/block scans, queue appends, and the Filter of
// Alg. 2 that compacts the forest slots (static kernels: one copy per
// translation unit).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "cc_device.cuh"
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

// Order-free append of a warp's kept items through a per-warp shared-memory
// buffer of CAP entries: one atomicAdd on the output counter per ~CAP items
// instead of one per 32 (a single counter takes its atomics one at a time at
// its L2 slice: ~1.3 ns each, 100 ms for the 79M appends of SV's edge copy at
// C4 k = 0), and the items leave in coalesced runs.  Every lane of the warp
// calls put() / flush() together.
template <class T, int CAP>
struct WarpBuf {
    T* buf;            // this warp's CAP shared-memory entries
    uint32_t fill;     // warp-uniform
    __device__ __forceinline__ void put(bool keep, const T& x, unsigned long long* counter, T* out)
    {
        const unsigned lane = threadIdx.x & 31;
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) buf[fill + __popc(m & ((1u << lane) - 1u))] = x;
        fill += __popc(m);
        if (fill > CAP - 32) flush(counter, out);
    }
    __device__ __forceinline__ void flush(unsigned long long* counter, T* out)
    {
        const unsigned lane = threadIdx.x & 31;
        __syncwarp();
        unsigned long long base = 0;
        if (lane == 0 && fill) base = atomicAdd(counter, (unsigned long long)fill);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (uint32_t j = lane; j < fill; j += 32) out[base + j] = buf[j];
        __syncwarp();
        fill = 0;
    }
};

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

// single CTA: exclusive scan of per-block counts (64-bit running total); used by
// the contracted link's rank scan
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


// ---------------------------------------------------------------------------
// K1': UF-Rem-CAS + SplitAtomicOne links with lane refill (the static k-out link
// and the incremental insert phase).
//
// The link kernel is latency-bound: every Rem-loop step is a dependent random
// load, and in k_link_pending a warp keeps stepping until its slowest lane's
// link is done, so on average half the lanes idle (ncu: 15 of 32 threads per
// instruction).  Here each warp streams its pending links through a 32-entry
// register buffer (one coalesced pend load + the P[u], P[v] gathers of all 32
// entries, issued one buffer ahead so they are in flight while the current one
// is consumed); a lane whose link finished takes the next buffered entry by a
// shuffle, and entries whose first parents are already equal retire without
// occupying a lane.  Every loop iteration then does one Rem step (one load, or
// a CAS) on every lane that holds a link.  The step is exactly link_rem_from's
// iteration (readings R1, R6), so the result is the same partition.
#ifndef CC_REFILL_MINB
#define CC_REFILL_MINB 6
#endif
// The link count is *count_dev when given (the static path: k_sample_init's
// append counter), else count_host (an incremental batch).
template <bool SF>
static __global__ void __launch_bounds__(kBlock, CC_REFILL_MINB) k_link_refill(
    uint32_t* P, const uint2* __restrict__ pend, const unsigned long long* count_dev, unsigned long long count_host,
    uint2* F, cc_counters* cnt, const unsigned int* skip_if)
{
    pdl_trigger();
    pdl_wait();
    if (skip_if && *skip_if) return;                 // the device-side kernel choice picked k_link_pending
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const unsigned long long total = count_dev ? *count_dev : count_host;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long chunk = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    // next buffer: entry chunk*32 + lane with its first two parent reads in flight
    uint2 nb = make_uint2(0u, 0u);
    uint32_t npu = 0, npv = 0, navail = 0;
    auto fetch = [&]() {
        const unsigned long long b0 = chunk * 32;
        navail = b0 < total ? (uint32_t)min(32ull, total - b0) : 0u;
        const bool ok = lane < navail;
        nb = ok ? pend[b0 + lane] : make_uint2(0u, 0u);
        npu = ok ? ld_link(P + nb.x) : 0u;
        npv = ok ? ld_link(P + nb.y) : 0u;
        chunk += nwarps;
    };
    fetch();
    uint2 cb = nb;
    uint32_t cpu = npu, cpv = npv, cavail = navail, cpos = 0;
    if (cavail) fetch();
    bool act = false;
    uint32_t u = 0, v = 0, ru = 0, rv = 0, pu = 0, pv = 0;
    uint32_t hooked = 0, steps = 0, fails = 0;
    while (true) {
        // refill idle lanes from the buffer (warp-uniform loop)
        unsigned need = __ballot_sync(0xffffffffu, !act);
        while (need && cavail) {
            const uint32_t src = cpos + __popc(need & lt_mask);
            const uint32_t sl = src & 31;
            const uint32_t xu = __shfl_sync(0xffffffffu, cb.x, sl), xv = __shfl_sync(0xffffffffu, cb.y, sl);
            const uint32_t xpu = __shfl_sync(0xffffffffu, cpu, sl), xpv = __shfl_sync(0xffffffffu, cpv, sl);
            if (!act && src < cavail && xpu != xpv) {        // equal first parents: already one set
                act = true;
                u = ru = xu;
                v = rv = xv;
                pu = xpu;
                pv = xpv;
            }
            cpos = min(cavail, cpos + (uint32_t)__popc(need));
            if (cpos == cavail) {                            // buffer used up: rotate in the prefetched one
                cb = nb;
                cpu = npu;
                cpv = npv;
                cavail = navail;
                cpos = 0;
                if (cavail) fetch();
            }
            need = __ballot_sync(0xffffffffu, !act);
        }
        if (!__any_sync(0xffffffffu, act)) break;           // buffer empty and every link done
        if (act) {                                           // one iteration of link_rem_from
            ++steps;
            if (pu < pv) {
                uint32_t t = ru; ru = rv; rv = t;
                t = pu; pu = pv; pv = t;
            }
            if (ru == pu) {                                  // ru is a root: hook it under pv
                const uint32_t old = cas(P + ru, ru, pv);
                if (old == ru) {
                    if (SF) F[ru] = make_uint2(u, v);
                    ++hooked;
                    act = false;
                } else {
                    ++fails;
                    pu = old;
                    pv = ld_link(P + rv);
                }
            } else {
                const uint32_t w = ld_link(P + pu);          // SplitAtomicOne on ru
                if (w != pu) cas(P + ru, pu, w);
                ru = pu;
                pu = w;
            }
            if (act && pu == pv) act = false;
        }
    }
    if (cnt) {
        warp_count(&cnt->sample_hooks, hooked);
        warp_count(&cnt->link_steps, steps);
        warp_count(&cnt->cas_failures, fails);
    }
}


// Filter in ONE pass (decoupled look-back): a block takes the next tile of kFTile
// slots by ticket; each warp owns kFTile/8 consecutive slots and counts them with
// ballots; the block publishes its count, adds up its predecessors' published
// counts / prefixes, publishes its inclusive prefix, and each warp writes its
// slots in order (re-reading them, still in L2) at ballot-ranked positions.  F is
// read from DRAM once, and a tile needs three block barriers, not one per slot
// round.  status[] (one word per tile) and *ticket start at zero; the last tile
// stores the total in *num_edges.
static __global__ void __launch_bounds__(kBlock) k_forest_filter(const uint2* F, uint32_t n, uint32_t ntiles,
                                                                 unsigned long long* status, unsigned int* ticket,
                                                                 uint32_t* edges, int64_t* num_edges,
                                                                 const float* Fw = nullptr, float* out_w = nullptr)
{
    pdl_trigger();
    pdl_wait();
    constexpr unsigned long long kAgg = 1ull << 62, kPre = 2ull << 62, kVal = (1ull << 62) - 1;
    constexpr int NW = kBlock / 32, SEG = kFTile / NW;      // slots per warp
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_wc[NW];
    __shared__ unsigned long long s_wo[NW];
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t seg = (uint64_t)tile * kFTile + (uint64_t)w * SEG;
    uint32_t c = 0;
#pragma unroll 4
    for (int r = 0; r < SEG / 32; ++r) {
        const uint64_t i = seg + (uint64_t)r * 32 + lane;
        c += __popc(__ballot_sync(0xffffffffu, i < n && F[i].x != kSentinel));
    }
    if (lane == 0) s_wc[w] = c;
    __syncthreads();
    if (w == 0) {                                            // warp 0: publish + look back 32 tiles at a time
        unsigned long long agg = 0;
        for (int k = 0; k < NW; ++k) agg += s_wc[k];
        if (lane == 0) atomicExch(status + tile, (tile == 0 ? kPre : kAgg) | agg);
        unsigned long long excl = 0;
        int64_t p = (int64_t)tile - 1;
        while (p >= 0) {
            const int64_t q = p - lane;
            unsigned long long st = q >= 0 ? atomicAdd(status + q, 0ull) : kPre;   // before tile 0: prefix 0
            const unsigned pre = __ballot_sync(0xffffffffu, (st & kPre) != 0);
            const unsigned none = __ballot_sync(0xffffffffu, (st & ~kVal) == 0);
            // lanes up to the first published prefix (lane order = descending tile)
            const int lim = pre ? __ffs(pre) - 1 : 31;
            const unsigned upto = lim == 31 ? 0xffffffffu : ((2u << lim) - 1u);
            if (none & upto) continue;                       // a tile in the window has not published: re-read
            unsigned long long v = (lane <= (unsigned)lim && q >= 0) ? (st & kVal) : 0ull;
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);   // 64-bit sum
            excl += v;
            if (pre) break;
            p -= 32;
        }
        if (lane == 0) {
            if (tile) atomicExch(status + tile, kPre | (excl + agg));
            unsigned long long acc = excl;
            for (int k = 0; k < NW; ++k) {
                s_wo[k] = acc;
                acc += s_wc[k];
            }
            if (tile == ntiles - 1) *num_edges = (int64_t)(excl + agg);
        }
    }
    __syncthreads();
    unsigned long long o = s_wo[w];
#pragma unroll 4
    for (int r = 0; r < SEG / 32; ++r) {
        const uint64_t i = seg + (uint64_t)r * 32 + lane;
        const uint2 f = i < n ? F[i] : make_uint2(kSentinel, kSentinel);
        const bool keep = f.x != kSentinel;
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const unsigned long long pos = o + __popc(mk & lt);
            reinterpret_cast<uint2*>(edges)[pos] = f;
            if (out_w) out_w[pos] = Fw[i];
        }
        o += __popc(mk);
    }
}

}  // namespace ccb
