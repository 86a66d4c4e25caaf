// cc_amsf.cu -- approximate minimum spanning forest, AMSF-NF-S (NEXT-4).
//
// Sec. 5.1 of the paper.  The folklore algorithm:
// bucket the edges by weight, [W_min (1+eps)^i, W_min (1+eps)^(i+1)), process
// the buckets from light to heavy, and in each one add to the forest the edges
// that join two different components of the labeling built so far.  NF
// (P:1819-1822): the CSR is never mutated, every round reads the lists again.
// S: each round finds the largest component L_max of the current
// labeling and skips its vertices -- an edge leaving it is seen from its other
// endpoint (the weights are symmetric, so both directions share a bucket).
// Every union is UF-Rem-CAS + SplitAtomicOne on ONE persistent
// parent array; the edge whose CAS hooks a root is recorded at that root (the
// rule of Alg. 2), so a root is recorded at most once over all
// rounds and the slots form the forest U F_i.
//
// B200 layout of a round (one persistent-grid kernel, no host round trip):
//   active list  -- the vertices that may still have work: those carried over
//                   from the previous round plus those whose lightest edge
//                   falls in this bucket (a counting sort by that bucket,
//                   computed once).  A vertex leaves the list for good when
//                   its heaviest edge is below the bucket, or when its root is
//                   the skipped component's (if a later round's L_max is a
//                   different component the list is rebuilt from scratch).
//   edge sweep   -- a warp takes up to 32 active vertices and sweeps their
//                   concatenated lists 32 entries at a time (prefix sums +
//                   shuffle search, as in the static finish): each lane reads
//                   one weight (coalesced) and only an in-bucket edge reads its
//                   endpoint and runs a link.
// CC_FLAG_AMSF_PLAIN drops the per-vertex [min, max] weight index: every
// non-skipped vertex is active and fully inspected in every round, as the
// paper states NF-S.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cc_common.cuh"
#include "cc_device.cuh"
#include "cc_internal.h"

namespace ccb {

namespace {

constexpr uint32_t kPosInfBits = 0x7F800000u;     // +inf as float bits
constexpr uint64_t AMSF_IDENT_STREAM = 19;        // per-round L_max samples: index = round * 2^20 + i

struct AmsfCtl {
    unsigned long long cnt[2];   // carry-list lengths (ping-pong)
    unsigned int wmin_bits;      // min / max weight (positive floats order like their bits)
    unsigned int wmax_bits;
    unsigned int bad;            // a weight <= 0 or not finite
    unsigned int anchor;         // a vertex of the component whose vertices are being dropped
    unsigned int skip_root;      // its root at the start of the current round
    unsigned int rebuild;        // this round's input is order[0 .. start[i+1])
    unsigned long long chunks;   // long-list pieces queued this round
};

constexpr int64_t kAmsfChunk = 2048;   // lists longer than this are split across warps
// cc_counters.amsf_links (in-bucket edges linked) is counted only in a diagnostics
// build (-DCC_AMSF_COUNT_LINKS): the counter costs the edge sweeps registers and
// occupancy (NF-S as stated: 98 -> 118 ms on C3)
#ifdef CC_AMSF_COUNT_LINKS
#define CC_AMSF_LINK_INC(x) (++(x))
#define CC_AMSF_LINK_FLUSH(cnt, x) warp_count(&(cnt)->amsf_links, (x))
#else
#define CC_AMSF_LINK_INC(x) ((void)0)
#define CC_AMSF_LINK_FLUSH(cnt, x) ((void)(x))
#endif
#ifndef CC_AMSF_IDX_MIN
#define CC_AMSF_IDX_MIN 256
#endif
constexpr int64_t kIdxMin = CC_AMSF_IDX_MIN;   // lists longer than this get the bucket index
constexpr int64_t kIdxWarpMax = 4096;  // ... built by one warp up to this length, else one CTA
constexpr uint32_t kIdxWarpBins = 512; // the warp build needs nb + 1 <= this

// Record for AMSF hooks: the edge and its weight at the hooked root.
struct ForestW {
    uint2* F;
    float* Fw;
    float w;
    __device__ __forceinline__ void record(uint32_t r, uint32_t u, uint32_t v) const
    {
        F[r] = make_uint2(u, v);
        Fw[r] = w;
    }
};

__device__ __forceinline__ bool good_weight(float x) { return x > 0.0f && x < __int_as_float((int)kPosInfBits); }

// Per-vertex lightest / heaviest edge weight and the global range, streamed in
// ENTRY tiles: block t reads the kWrTile weights [t*kWrTile, (t+1)*kWrTile)
// coalesced (16 per thread, float4 loads), whatever the list lengths.  tile_vs[t]
// (written by k_amsf_init) is the vertex owning the tile's first entry; a thread
// finds the owner of its first entry by a binary search of the offsets within the
// tile's vertex range (staged in shared memory), then walks the list boundaries
// forward.  Per
// vertex min / max are combined in shared memory; a vertex wholly inside the tile
// is stored plainly, one that straddles a tile boundary is combined by global
// atomics into vi[v].x / .y (initialised to +inf / 0 by k_amsf_init).  (The thread-
// per-vertex version walked each short list serially: 12.7 ms on C4, latency-bound.)
#ifndef CC_AMSF_WR_STAGE
#define CC_AMSF_WR_STAGE 0
#endif
#ifndef CC_AMSF_WR_ITEMS
#define CC_AMSF_WR_ITEMS 16
#endif
constexpr int kWrItems = CC_AMSF_WR_ITEMS;
constexpr int64_t kWrTile = (int64_t)kBlock * kWrItems;
constexpr uint32_t kWrCap = 2048;          // vertices per tile combined in shared memory
__global__ void __launch_bounds__(kBlock) k_amsf_wrange(const int64_t* __restrict__ off, const float* __restrict__ w,
                                                        uint32_t n, int64_t m, const uint32_t* __restrict__ tile_vs,
                                                        uint4* vi, AmsfCtl* ac)
{
    __shared__ uint32_t s_lo[kWrCap], s_hi[kWrCap];
#if CC_AMSF_WR_STAGE
    __shared__ int64_t s_off[kWrCap + 1];
#endif
    const unsigned lane = threadIdx.x & 31;
    const uint64_t ntiles = (uint64_t)((m + kWrTile - 1) / kWrTile);
    const bool vec = ((uintptr_t)w & 15u) == 0;
    uint32_t gmin = kPosInfBits, gmax = 0, bad = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t E0 = (int64_t)t * kWrTile, E1 = min(E0 + kWrTile, m);
        const uint32_t vs = tile_vs[t];
        const uint32_t ve = t + 1 < ntiles ? tile_vs[t + 1] : n - 1;     // owner of entry E1 (or the last)
        const uint32_t nv = min(ve - vs + 1, kWrCap);
        const uint32_t no = min(ve - vs + 2, kWrCap + 1);          // offsets staged: off[vs .. vs + no)
        for (uint32_t j = threadIdx.x; j < nv; j += blockDim.x) {
            s_lo[j] = kPosInfBits;
            s_hi[j] = 0;
        }
#if CC_AMSF_WR_STAGE
        for (uint32_t j = threadIdx.x; j < no; j += blockDim.x) s_off[j] = off[vs + j];
        __syncthreads();
        auto offat = [&](uint32_t v) -> int64_t { return v - vs < no ? s_off[v - vs] : off[v]; };
#else
        __syncthreads();
        auto offat = [&](uint32_t v) -> int64_t { return off[v]; };
        (void)no;
#endif
        const int64_t e0 = E0 + (int64_t)threadIdx.x * kWrItems;
        if (e0 < E1) {
            // owner of e0: the largest v in [vs, ve] with off[v] <= e0
            uint32_t lo = vs, hi = ve;
            while (lo < hi) {
                const uint32_t mid = lo + (hi - lo + 1) / 2;
                if (offat(mid) <= e0) lo = mid; else hi = mid - 1;
            }
            uint32_t owner = lo;
            int64_t nxt = offat(owner + 1);
            float x[kWrItems];
            if (vec && e0 + kWrItems <= E1) {
#pragma unroll
                for (int q = 0; q < kWrItems / 4; ++q) {
                    const float4 f = __ldg(reinterpret_cast<const float4*>(w + e0) + q);
                    x[4 * q] = f.x; x[4 * q + 1] = f.y; x[4 * q + 2] = f.z; x[4 * q + 3] = f.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < kWrItems; ++q) x[q] = e0 + q < E1 ? __ldg(w + e0 + q) : 1.0f;
            }
            uint32_t vlo = kPosInfBits, vhi = 0;
            bool any = false;
            auto flush = [&]() {
                if (!any) return;
                const uint32_t j = owner - vs;
                if (j < kWrCap) {
                    atomicMin(s_lo + j, vlo);
                    atomicMax(s_hi + j, vhi);
                } else {
                    atomicMin(reinterpret_cast<uint32_t*>(vi + owner), vlo);
                    atomicMax(reinterpret_cast<uint32_t*>(vi + owner) + 1, vhi);
                }
                gmin = min(gmin, vlo);
                gmax = max(gmax, vhi);
            };
            if (e0 + kWrItems <= E1 && nxt >= e0 + kWrItems) {
                // fast path (inside one list, the common case for the long lists that hold
                // most entries): no boundary tests; a weight is good iff 0 < bits < +inf bits
#pragma unroll
                for (int q = 0; q < kWrItems; ++q) {
                    const uint32_t bits = __float_as_uint(x[q]);
                    bad |= (bits - 1u) >= (kPosInfBits - 1u) ? 1u : 0u;
                    vlo = min(vlo, bits & 0x7FFFFFFFu);
                    vhi = max(vhi, bits & 0x7FFFFFFFu);
                }
                any = true;
            } else
#pragma unroll
            for (int q = 0; q < kWrItems; ++q) {
                const int64_t e = e0 + q;
                if (e < E1) {
                    while (e >= nxt) {                   // next list (zero-length lists skipped)
                        flush();
                        ++owner;
                        nxt = offat(owner + 1);
                        vlo = kPosInfBits;
                        vhi = 0;
                        any = false;
                    }
                    if (!good_weight(x[q])) bad = 1;
                    const uint32_t bits = __float_as_uint(x[q]) & 0x7FFFFFFFu;
                    vlo = min(vlo, bits);
                    vhi = max(vhi, bits);
                    any = true;
                }
            }
            // the last segment: inside a long list every lane of the warp has the same
            // owner -- reduce it in the warp first (one shared atomic, not 32)
            const unsigned am = __activemask();
            const uint32_t o0 = __shfl_sync(am, owner, __ffs(am) - 1);
            if (__all_sync(am, any && owner == o0)) {
                vlo = __reduce_min_sync(am, vlo);
                vhi = __reduce_max_sync(am, vhi);
                if (lane == (unsigned)(__ffs(am) - 1)) flush();
                gmin = min(gmin, vlo);
                gmax = max(gmax, vhi);
            } else {
                flush();
            }
        }
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < nv; j += blockDim.x) {
            if (s_lo[j] == kPosInfBits && s_hi[j] == 0) continue;          // no entry in this tile
            const uint32_t v = vs + j;
            if (offat(v) >= E0 && offat(v + 1) <= E1) {
                *reinterpret_cast<uint2*>(vi + v) = make_uint2(s_lo[j], s_hi[j]);
            } else {
                atomicMin(reinterpret_cast<uint32_t*>(vi + v), s_lo[j]);
                atomicMax(reinterpret_cast<uint32_t*>(vi + v) + 1, s_hi[j]);
            }
        }
        __syncthreads();
    }
    gmin = __reduce_min_sync(0xffffffffu, gmin);
    gmax = __reduce_max_sync(0xffffffffu, gmax);
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0) {
        if (gmin != kPosInfBits) atomicMin(&ac->wmin_bits, gmin);
        if (gmax) atomicMax(&ac->wmax_bits, gmax);
        if (bad) atomicOr(&ac->bad, 1u);
    }
}

// P, the weight ranges and the forest slots; and tile_vs[t] = the vertex whose list
// holds entry t * kWrTile (the first entry of wrange tile t).
__global__ void k_amsf_init(const int64_t* __restrict__ off, uint32_t* P, uint4* vi, uint2* F,
                            uint32_t n, uint32_t* tile_vs)
{
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        P[v] = (uint32_t)v;
        vi[v] = make_uint4(kPosInfBits, 0u, kSentinel, 0u);
        F[v] = make_uint2(kSentinel, kSentinel);
        if (tile_vs) {
            const int64_t b = off[v], e = off[v + 1];
            for (int64_t t = (b + kWrTile - 1) / kWrTile; t * kWrTile < e; ++t) tile_vs[t] = (uint32_t)v;
        }
    }
}

// bucket of a weight: the i with b[i] <= x < b[i+1] (b[0] = W_min <= x)
__device__ __forceinline__ uint32_t bucket_of(const double* b, uint32_t nb, float x)
{
    const double d = (double)x;
    uint32_t lo = 0, hi = nb;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (b[mid] <= d) lo = mid; else hi = mid;
    }
    return lo;
}

// activation bucket of every non-isolated vertex (its lightest edge's bucket;
// 0 in PLAIN mode) and the histogram of those buckets: per block a shared-
// memory histogram (when the buckets fit), one global atomic per non-empty bin
constexpr uint32_t kSmemBins = 4096;
constexpr uint32_t kIdxBins = 4000;      // the hub bucket index is built when nb <= this
__global__ void __launch_bounds__(kBlock) k_amsf_first(const uint4* vi, uint32_t n,
                                                       const double* b, uint32_t nb, bool plain, uint32_t* fb,
                                                       unsigned long long* hist)
{
    __shared__ uint32_t sh[kSmemBins];
    const bool local = nb <= kSmemBins;
    if (local)
        for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 r = *reinterpret_cast<const uint2*>(vi + v);
        if (!r.y) continue;                                   // isolated
        const uint32_t f = plain ? 0u : bucket_of(b, nb, __uint_as_float(r.x));
        fb[v] = f;
        if (local) atomicAdd(sh + f, 1u);
        else atomicAdd(hist + f, 1ull);
    }
    __syncthreads();
    if (local)
        for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
            if (sh[i]) atomicAdd(hist + i, (unsigned long long)sh[i]);
}

// exclusive scan of the histogram (nb + 1 entries, one block)
__global__ void __launch_bounds__(kBlock) k_amsf_scan(unsigned long long* hist, uint32_t nb)
{
    __shared__ unsigned long long carry;
    __shared__ unsigned long long ws[kBlock / 32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const unsigned lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    for (uint32_t base = 0; base <= nb; base += kBlock) {
        const uint32_t i = base + threadIdx.x;
        const unsigned long long x = i <= nb ? hist[i] : 0ull;
        unsigned long long incl = x;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (unsigned)o) incl += t;
        }
        if (lane == 31) ws[wi] = incl;
        __syncthreads();
        unsigned long long wb = 0;
        for (unsigned j = 0; j < wi; ++j) wb += ws[j];
        const unsigned long long c = carry;
        if (i <= nb) hist[i] = c + wb + incl - x;
        __syncthreads();
        if (threadIdx.x == kBlock - 1) carry = c + wb + incl;
        __syncthreads();
    }
}

// order[] by activation bucket: per block tile of 8 * kBlock vertices, ranks within
// the tile from shared atomics, one global range per non-empty bin and tile
__global__ void __launch_bounds__(kBlock) k_amsf_scatter(const uint4* vi, const uint32_t* fb, uint32_t n,
                                                         uint32_t nb, unsigned long long* cursor, uint32_t* order)
{
    constexpr int V = 8;
    __shared__ uint32_t sc[kSmemBins];
    __shared__ unsigned long long sb[kSmemBins];
    const bool local = nb <= kSmemBins;
    for (uint64_t t0 = (uint64_t)blockIdx.x * (kBlock * V); t0 < n; t0 += (uint64_t)gridDim.x * (kBlock * V)) {
        bool act[V];
        uint32_t f[V], rank[V];
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const uint64_t v = t0 + (uint64_t)k * kBlock + threadIdx.x;
            act[k] = v < n && reinterpret_cast<const uint2*>(vi + v)->y != 0;
            f[k] = act[k] ? fb[v] : 0u;
        }
        if (!local) {
#pragma unroll
            for (int k = 0; k < V; ++k)
                if (act[k]) order[atomicAdd(cursor + f[k], 1ull)] = (uint32_t)(t0 + (uint64_t)k * kBlock + threadIdx.x);
            continue;
        }
#pragma unroll
        for (int k = 0; k < V; ++k)
            if (act[k]) sc[f[k]] = 0;                        // clear only the bins this tile touches
        __syncthreads();
#pragma unroll
        for (int k = 0; k < V; ++k) rank[k] = act[k] ? atomicAdd(sc + f[k], 1u) : 0u;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < V; ++k)
            if (act[k] && rank[k] == 0) sb[f[k]] = atomicAdd(cursor + f[k], (unsigned long long)sc[f[k]]);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < V; ++k)
            if (act[k]) order[sb[f[k]] + rank[k]] = (uint32_t)(t0 + (uint64_t)k * kBlock + threadIdx.x);
        __syncthreads();
    }
}

// S: L_max of the current labeling (IdentifyFrequent: the mode of the
// roots of S seeded samples, ties to the smaller label), kept as the "anchor"
// of the skipped component.  The dropped vertices all lie in the anchor's
// component (components only merge, so it only grows); if L_max is now a
// different component -- seen by more samples than the anchor's -- the anchor
// moves there and this round rebuilds its input from every activated vertex.
constexpr int kIdTable = 4096;
#ifndef CC_AMSF_ANCHOR_DIV
#define CC_AMSF_ANCHOR_DIV 256
#endif
__global__ void __launch_bounds__(1024) k_amsf_lmax(uint32_t* P, uint32_t n, uint64_t seed, uint32_t round,
                                                    uint32_t samples, AmsfCtl* ac)
{
    pdl_trigger();
    pdl_wait();
    __shared__ uint32_t keys[kIdTable];
    __shared__ uint32_t cnts[kIdTable];
    __shared__ unsigned long long best[32];
    __shared__ uint32_t s_ra, s_cnt_ra;
    const int t = threadIdx.x;
    for (int i = t; i < kIdTable; i += blockDim.x) {
        keys[i] = kSentinel;
        cnts[i] = 0;
    }
    if (t == 0) {
        s_ra = ac->anchor == kSentinel ? kSentinel : find_halve_quiet(P, ac->anchor);   // no hook runs now
        s_cnt_ra = 0;
    }
    __syncthreads();
    for (int i = t; i < (int)samples; i += blockDim.x) {
        const uint32_t sv = uniform_below(mix(seed, AMSF_IDENT_STREAM, ((uint64_t)round << 20) + (uint64_t)i), n);
        const uint32_t lab = find_halve_quiet(P, sv);
        if (lab == s_ra) atomicAdd(&s_cnt_ra, 1u);
        uint32_t h = (lab * 0x9E3779B1u) >> 20;
        while (true) {
            const uint32_t old = atomicCAS(&keys[h], kSentinel, lab);
            if (old == kSentinel || old == lab) {
                atomicAdd(&cnts[h], 1u);
                break;
            }
            h = (h + 1) & (kIdTable - 1);
        }
    }
    __syncthreads();
    unsigned long long key = 0;
    for (int i = t; i < kIdTable; i += blockDim.x)
        if (cnts[i]) {
            const unsigned long long k2 = ((unsigned long long)cnts[i] << 32) | (unsigned long long)(kSentinel - keys[i]);
            key = key > k2 ? key : k2;
        }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
        key = key > y ? key : y;
    }
    if ((t & 31) == 0) best[t >> 5] = key;
    __syncthreads();
    if (t < 32) {
        key = t < (int)(blockDim.x >> 5) ? best[t] : 0;
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
            key = key > y ? key : y;
        }
        if (t == 0) {
            const uint32_t lm = kSentinel - (uint32_t)(key & 0xFFFFFFFFull);
            const uint32_t cnt_lm = (uint32_t)(key >> 32);
            // a component seen by under 1/256 of the samples (4 of 1024) is not worth skipping (while the
            // labeling is all singletons every sample is its own mode): start, or move, the
            // anchor only for a component at least that large
            const bool big = (uint64_t)cnt_lm * CC_AMSF_ANCHOR_DIV >= samples;
            ac->rebuild = 0;
            if (s_ra == kSentinel) {
                if (big) ac->anchor = lm;                 // nothing dropped yet: no rebuild needed
            } else if (big && lm != s_ra && cnt_lm > s_cnt_ra) {
                ac->anchor = lm;                          // a different, larger component
                ac->rebuild = 1;
            }
            ac->skip_root = ac->anchor == kSentinel ? kSentinel : (ac->anchor == lm ? lm : s_ra);
        }
    }
}

// One round (bucket i = [blo, bhi)): the active list is the carry list plus the
// vertices activated in this bucket (order[start[i] .. start[i+1])), or, after
// an anchor move, order[0 .. start[i+1]).  Survivors are appended to the next
// carry list.
#ifndef CC_AMSF_ROUND_MINB
#define CC_AMSF_ROUND_MINB 4
#endif
constexpr int kCarryBuf = 256;

template <int MODE>
__global__ void __launch_bounds__(kBlock, CC_AMSF_ROUND_MINB) k_amsf_round(
    const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, const float* __restrict__ w, uint32_t* P,
    const uint4* __restrict__ vi, const uint32_t* __restrict__ order,
    const unsigned long long* __restrict__ start, uint32_t round, double blo, double bhi,
    const uint32_t* __restrict__ carry_in, AmsfCtl* ac, int in_slot, uint32_t* carry_out, bool skip, bool plain,
    uint2* F, float* Fw, uint2* chq, const unsigned long long* __restrict__ hstart,
    const uint32_t* __restrict__ hidx, uint32_t nbk, cc_counters* cnt)
{
    pdl_trigger();
    pdl_wait();
    const unsigned lane = threadIdx.x & 31;
    const bool rebuild = ac->rebuild != 0;
    const unsigned long long s0 = rebuild ? 0ull : start[round], s1 = start[round + 1];
    const unsigned long long n1 = rebuild ? 0ull : ac->cnt[in_slot];
    const unsigned long long total = n1 + (s1 - s0);
    const uint32_t skip_root = skip ? ac->skip_root : kSentinel;
    unsigned long long* out_cnt = &ac->cnt[in_slot ^ 1];
    const unsigned long long warp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    const unsigned cpw = (unsigned)max(1ull, min(32ull, (total + nwarps - 1) / nwarps));
    __shared__ uint32_t s_carry[kBlock / 32][kCarryBuf];
    WarpBuf<uint32_t, kCarryBuf> carry{s_carry[threadIdx.x >> 5], 0u};   // survivors, one atomic per ~kCarryBuf
    uint32_t visits = 0, hooks = 0, links = 0;
    unsigned long long scanned = 0;
    for (unsigned long long base = warp * cpw; base < total; base += nwarps * cpw) {
        const unsigned long long i = base + lane;
        const bool cand = lane < cpw && i < total;
        const uint32_t u = cand ? (i < n1 ? carry_in[i] : order[s0 + (i - n1)]) : 0u;
        bool keep = false, work = false;
        uint32_t hub = kSentinel;
        if (cand) {
            ++visits;
            // [lightest, heaviest] weight bits, hub id (not needed as NF-S is stated: PLAIN)
            const uint4 vv = plain ? make_uint4(0u, 0u, kSentinel, 0u) : vi[u];
            hub = vv.z;
            const double hi_w = plain ? INFINITY : (double)__uint_as_float(vv.y);
            const double lo_w = plain ? 0.0 : (double)__uint_as_float(vv.x);
            // FindAtomicSplit (hooks run concurrently): walks stay short on chain-shaped inputs
            if (hi_w >= blo && !(skip_root != kSentinel && find_split(P, u) == skip_root)) {
                keep = hi_w >= bhi;                            // edges left for later buckets
                work = lo_w < bhi;                             // maybe an edge in this bucket
            }
        }
        carry.put(keep, u, out_cnt, carry_out);
        const int64_t b = work ? off[u] : 0;
        const int64_t dfull = work ? off[u + 1] - b : 0;
        // an indexed list (> kIdxMin entries, bucket index built) contributes only this
        // bucket's entries, read through hidx from `base`; a range (or, without the
        // index, a list) longer than kAmsfChunk is cut into pieces for any warp
        const bool indexed = hstart && dfull > kIdxMin;
        int64_t len = dfull, rbase = b;
        if (indexed) {
            const unsigned long long* hs = hstart + (uint64_t)hub * (nbk + 1);
            rbase = (int64_t)hs[round];
            len = (int64_t)hs[round + 1] - rbase;
        }
        const bool big = len > kAmsfChunk;
        if (big) {
            const uint32_t nch = (uint32_t)((len + kAmsfChunk - 1) / kAmsfChunk);
            const unsigned long long q = atomicAdd(&ac->chunks, (unsigned long long)nch);
            for (uint32_t c = 0; c < nch; ++c) chq[q + c] = make_uint2(u, c);
        }
        const uint32_t d = big ? 0u : (uint32_t)len;
        uint32_t incl = d;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (unsigned)o) incl += t;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - d;
        scanned += lane == 0 ? tot : 0u;
        // 4 entries per lane per sweep step: owners by shuffle search, then the 4 weight
        // loads in flight together
        for (uint32_t t0 = 0; t0 < tot; t0 += 128) {
            uint32_t ou[4];
            int64_t ex[4];
            float x[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t t = t0 + 32 * j + lane;
                int lo = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const uint32_t pe = __shfl_sync(0xffffffffu, excl, lo + step);
                    if (pe <= t) lo += step;
                }
                ou[j] = __shfl_sync(0xffffffffu, u, lo);
                const int64_t ob = __shfl_sync(0xffffffffu, rbase, lo);
                const bool oi = __shfl_sync(0xffffffffu, indexed, lo);
                const int64_t oo = __shfl_sync(0xffffffffu, b, lo);
                const uint32_t oex = __shfl_sync(0xffffffffu, excl, lo);
                ex[j] = t < tot ? (oi ? oo + (int64_t)hidx[ob + (t - oex)] : ob + (t - oex)) : -1;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = ex[j] >= 0 ? w[ex[j]] : 0.0f;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double xd = (double)x[j];
                if (ex[j] >= 0 && xd >= blo && xd < bhi) {
                    CC_AMSF_LINK_INC(links);
                    hooks += link<MODE>(P, ou[j], adj[ex[j]], ForestW{F, Fw, x[j]});
                }
            }
            __syncwarp();
        }
    }
    carry.flush(out_cnt, carry_out);
    if (cnt) {
        warp_count(&cnt->amsf_visits, visits);
        warp_count(&cnt->amsf_hooks, hooks);
        CC_AMSF_LINK_FLUSH(cnt, links);
        const unsigned long long sc = __reduce_add_sync(0xffffffffu, (uint32_t)min(scanned, 0xFFFFFFFFull));
        if (lane == 0 && sc) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt->amsf_edges), sc);
    }
}

// The long lists of this round, indexed (hub bucket index): a piece is up to
// kAmsfChunk of the hub's entries of THIS bucket, read through hidx -- every entry
// is in the bucket, so no weight test is needed and each hub edge is read in one
// round only.
template <int MODE>
__global__ void __launch_bounds__(kBlock) k_amsf_hub_pieces(const int64_t* __restrict__ off,
                                                            const uint32_t* __restrict__ adj,
                                                            const float* __restrict__ w, uint32_t* P, uint32_t round,
                                                            const uint2* __restrict__ chq, const AmsfCtl* ac,
                                                            const uint4* __restrict__ vi,
                                                            const unsigned long long* __restrict__ hstart,
                                                            const uint32_t* __restrict__ hidx, uint32_t nbk, uint2* F,
                                                            float* Fw, cc_counters* cnt)
{
    pdl_trigger();
    pdl_wait();
    const unsigned lane = threadIdx.x & 31;
    const unsigned long long total = ac->chunks;
    const unsigned long long warp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    uint32_t hooks = 0, links = 0;
    unsigned long long scanned = 0;
    for (unsigned long long q = warp; q < total; q += nwarps) {
        const uint2 item = chq[q];
        const unsigned long long* hs = hstart + (uint64_t)vi[item.x].z * (nbk + 1);
        const unsigned long long s0 = hs[round] + (unsigned long long)item.y * kAmsfChunk;
        const unsigned long long s1 = min(hs[round + 1], s0 + kAmsfChunk);
        const int64_t o = off[item.x];
        scanned += lane == 0 ? s1 - s0 : 0ull;
        for (unsigned long long x0 = s0 + lane; x0 < s1; x0 += 32 * 4) {
            int64_t e[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) e[j] = x0 + 32 * j < s1 ? o + hidx[x0 + 32 * j] : -1;
            float wx[4];
            uint32_t vx[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                wx[j] = e[j] >= 0 ? w[e[j]] : 0.0f;
                vx[j] = e[j] >= 0 ? adj[e[j]] : 0u;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (e[j] >= 0) {
                    CC_AMSF_LINK_INC(links);
                    hooks += link<MODE>(P, item.x, vx[j], ForestW{F, Fw, wx[j]});
                }
        }
    }
    if (cnt) {
        warp_count(&cnt->amsf_hooks, hooks);
        CC_AMSF_LINK_FLUSH(cnt, links);
        const unsigned long long sc = __reduce_add_sync(0xffffffffu, (uint32_t)min(scanned, 0xFFFFFFFFull));
        if (lane == 0 && sc) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt->amsf_edges), sc);
    }
}

// Bucket index (built once): the vertices with more than kIdxMin entries,
// vi[v].z = their index h, and per hub its entries (offsets relative to off[v])
// grouped by bucket: hidx[hstart[h][i] .. hstart[h][i+1]) are the bucket-i
// entries (absolute 64-bit starts, so a visit reads one line of hstart).  A
// visit of the round kernel reads its vertex's lightest / heaviest weight and
// hub id in ONE 16-byte vi load (three separate arrays made it three random
// sectors; the rounds are bound by these per-visit gathers).
// (Storing (neighbour, weight) pairs instead, so that a round reads its edges
// contiguously, was measured: the rounds stay bound by the links' P gathers
// (32.0 vs 29.9 ms on C4) and the build moves 8 B more per entry.)
// The lists to index: kIdxMin < d <= kIdxWarpMax go to queue 0 (one warp each),
// longer ones to queue 1 (one CTA each).  Each list's hidx region is claimed
// from a cursor (64-bit block prefix, one atomic per block): regions are
// disjoint, their order does not matter.
// Block-wide exclusive scan of three per-thread counts at once (two 32-bit queue
// counts, one 64-bit region size), with ONE global atomic per counter and block:
// per-warp atomics on three hot addresses made k_amsf_hubs atomic-bound (2.9 ms
// on C4 for a 1 GB offsets read).
struct Append3 {
    unsigned long long p0, p1, r;
};
__device__ __forceinline__ Append3 block_append3(uint32_t c0, uint32_t c1, unsigned long long r,
                                                 unsigned long long* hcount)
{
    constexpr int NW = kBlock / 32;
    __shared__ unsigned long long s_w[3][NW];
    __shared__ unsigned long long s_base[3];
    const unsigned lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    unsigned long long i0 = c0, i1 = c1, ir = r;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long a = __shfl_up_sync(0xffffffffu, i0, o);
        const unsigned long long b = __shfl_up_sync(0xffffffffu, i1, o);
        const unsigned long long c = __shfl_up_sync(0xffffffffu, ir, o);
        if (lane >= (unsigned)o) {
            i0 += a;
            i1 += b;
            ir += c;
        }
    }
    if (lane == 31) {
        s_w[0][wi] = i0;
        s_w[1][wi] = i1;
        s_w[2][wi] = ir;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned long long acc = 0;
        for (int k = 0; k < NW; ++k) {
            const unsigned long long x = s_w[threadIdx.x][k];
            s_w[threadIdx.x][k] = acc;
            acc += x;
        }
        s_base[threadIdx.x] = acc ? atomicAdd(hcount + threadIdx.x, acc) : 0ull;
    }
    __syncthreads();
    Append3 a;
    a.p0 = s_base[0] + s_w[0][wi] + i0 - c0;
    a.p1 = s_base[1] + s_w[1][wi] + i1 - c1;
    a.r = s_base[2] + s_w[2][wi] + ir - r;
    __syncthreads();
    return a;
}

constexpr int kHubV = 8;                  // vertices per thread in k_amsf_hubs
__global__ void __launch_bounds__(kBlock) k_amsf_hubs(const int64_t* __restrict__ off, uint32_t n, uint32_t* q0,
                                                      uint32_t* q1, unsigned long long* qb0, unsigned long long* qb1,
                                                      unsigned long long* hcount)
{
    constexpr uint64_t T = (uint64_t)kBlock * kHubV;
    for (uint64_t t0 = (uint64_t)blockIdx.x * T; t0 < n; t0 += (uint64_t)gridDim.x * T) {
        int64_t d[kHubV];
        uint32_t c0 = 0, c1 = 0;
        unsigned long long r = 0;
#pragma unroll
        for (int j = 0; j < kHubV; ++j) {
            const uint64_t v = t0 + (uint64_t)j * kBlock + threadIdx.x;
            d[j] = v < n ? off[v + 1] - off[v] : 0;
            c0 += d[j] > kIdxMin && d[j] <= kIdxWarpMax;
            c1 += d[j] > kIdxWarpMax;
            r += d[j] > kIdxMin ? (unsigned long long)d[j] : 0ull;
        }
        Append3 a = block_append3(c0, c1, r, hcount);
#pragma unroll
        for (int j = 0; j < kHubV; ++j) {
            const uint64_t v = t0 + (uint64_t)j * kBlock + threadIdx.x;
            if (d[j] <= kIdxMin) continue;
            if (d[j] <= kIdxWarpMax) {
                q0[a.p0] = (uint32_t)v;
                qb0[a.p0++] = a.r;
            } else {
                q1[a.p1] = (uint32_t)v;
                qb1[a.p1++] = a.r;
            }
            a.r += (unsigned long long)d[j];
        }
    }
}

// one block per hub: bucket histogram in shared memory, exclusive scan, then the
// entries placed by a shared cursor (order within a bucket is arbitrary).  The
// bucket of a weight is estimated from log2(x / W_min) / log2(1 + eps) and then
// settled by the exact fp64 comparisons b_i <= x < b_(i+1) (reading R25).
__device__ __forceinline__ uint32_t bucket_fast(const float* fb, uint32_t nb, float x, float wmin, float inv_l2g)
{
    // fb[i] = the smallest float >= b_i, so for a float weight x the exact rule
    // b_i <= (double)x (reading R25) is the float compare fb[i] <= x
    int i = (int)(__log2f(x / wmin) * inv_l2g);
    i = max(0, min((int)nb - 1, i));
    while (i + 1 < (int)nb && fb[i + 1] <= x) ++i;
    while (i > 0 && fb[i] > x) --i;
    return (uint32_t)i;
}

// Warp-aggregated shared-memory bin updates: lanes with the same bin (Exp(1)
// weights crowd a dozen buckets) are combined by __match_any_sync, so one lane
// per distinct bin issues the atomic.  key = kSentinel for an idle lane.
#ifndef CC_AMSF_AGG
#define CC_AMSF_AGG 0
#endif
__device__ __forceinline__ void agg_count(uint32_t* hist, uint32_t key)
{
    if (!CC_AMSF_AGG) {
        if (key != kSentinel) atomicAdd(hist + key, 1u);
        return;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (key != kSentinel && (threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(hist + key, __popc(peers));
}
// ... and the slot of this lane's entry: the leader reserves popc(peers) slots,
// each peer takes its rank among them.
__device__ __forceinline__ uint32_t agg_slot(uint32_t* hist, uint32_t key)
{
    if (!CC_AMSF_AGG) return key != kSentinel ? atomicAdd(hist + key, 1u) : 0u;
    const unsigned lane = threadIdx.x & 31;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (key != kSentinel && lane == (unsigned)leader) base = atomicAdd(hist + key, __popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + __popc(peers & ((1u << lane) - 1u));
}
#ifndef CC_AMSF_IDX_ILP
#define CC_AMSF_IDX_ILP 8
#endif
constexpr int kIdxILP = CC_AMSF_IDX_ILP;    // weights in flight per lane in the index builds

__global__ void __launch_bounds__(1024) k_amsf_hub_index(const int64_t* __restrict__ off,
                                                         const float* __restrict__ w, const uint32_t* q1,
                                                         const unsigned long long* qb1,
                                                         const unsigned long long* hcount, const float* bnd,
                                                         uint32_t nbk, float wmin, float inv_l2g, uint4* vi,
                                                         unsigned long long* hstart, uint32_t* hidx)
{
    __shared__ uint32_t sh[kIdxBins + 1];
    __shared__ float sb[kIdxBins + 1];
    for (uint32_t i = threadIdx.x; i <= nbk; i += blockDim.x) sb[i] = bnd[i];
    const unsigned long long H0 = hcount[0], H1 = hcount[1];
    for (unsigned long long p = blockIdx.x; p < H1; p += gridDim.x) {
        const uint32_t v = q1[p];
        const unsigned long long h = H0 + p;
        const int64_t b = off[v], d = off[v + 1] - b;
        if (threadIdx.x == 0) {
            reinterpret_cast<uint32_t*>(vi + v)[2] = (uint32_t)h;
        }
        for (uint32_t i = threadIdx.x; i <= nbk; i += blockDim.x) sh[i] = 0;
        __syncthreads();
        for (int64_t x0 = threadIdx.x; x0 - threadIdx.x < d; x0 += (int64_t)blockDim.x * kIdxILP) {
            float f[kIdxILP];
#pragma unroll
            for (int q = 0; q < kIdxILP; ++q) {
                const int64_t x = x0 + (int64_t)q * blockDim.x;
                f[q] = x < d ? __ldg(w + b + x) : 0.0f;
            }
#pragma unroll
            for (int q = 0; q < kIdxILP; ++q) {
                const int64_t x = x0 + (int64_t)q * blockDim.x;
                agg_count(sh, x < d ? bucket_fast(sb, nbk, f[q], wmin, inv_l2g) : kSentinel);
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {                               // exclusive scan (nbk <= kIdxBins), one warp
            uint32_t carry = 0;
            for (uint32_t base = 0; base <= nbk; base += 32) {
                const uint32_t i = base + threadIdx.x;
                const uint32_t c = i <= nbk ? sh[i] : 0u;
                uint32_t incl = c;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (threadIdx.x >= (unsigned)o) incl += t;
                }
                if (i <= nbk) sh[i] = carry + incl - c;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        __syncthreads();
        unsigned long long* hs = hstart + h * (nbk + 1);          // absolute bucket starts in hidx
        for (uint32_t i = threadIdx.x; i <= nbk; i += blockDim.x) hs[i] = qb1[p] + sh[i];
        __syncthreads();
        const unsigned long long hb = qb1[p];
        for (int64_t x0 = threadIdx.x; x0 - threadIdx.x < d; x0 += (int64_t)blockDim.x * kIdxILP) {
            float f[kIdxILP];
#pragma unroll
            for (int q = 0; q < kIdxILP; ++q) {
                const int64_t x = x0 + (int64_t)q * blockDim.x;
                f[q] = x < d ? __ldg(w + b + x) : 0.0f;
            }
#pragma unroll
            for (int q = 0; q < kIdxILP; ++q) {
                const int64_t x = x0 + (int64_t)q * blockDim.x;
                const uint32_t key = x < d ? bucket_fast(sb, nbk, f[q], wmin, inv_l2g) : kSentinel;
                const uint32_t slot = agg_slot(sh, key);
                if (x < d) hidx[hb + slot] = (uint32_t)x;
            }
        }
        __syncthreads();
    }
}

// The same index for lists of kIdxMin < d <= kIdxWarpMax entries, one warp per
// list (a per-warp shared histogram of nbk + 1 <= kIdxWarpBins bins).
constexpr int kIdxWBlock = 128;           // k_amsf_idx_warp block (4 warps: per-warp keys + bins in smem)
__global__ void __launch_bounds__(kIdxWBlock) k_amsf_idx_warp(const int64_t* __restrict__ off,
                                                          const float* __restrict__ w, const uint32_t* q0,
                                                          const unsigned long long* qb0,
                                                          const unsigned long long* hcount, const float* bnd,
                                                          uint32_t nbk, float wmin, float inv_l2g, uint4* vi,
                                                          unsigned long long* hstart, uint32_t* hidx)
{
    __shared__ uint32_t sh[kIdxWBlock / 32][kIdxWarpBins];
    __shared__ float sb[kIdxWarpBins];
    __shared__ uint8_t skey[kIdxWBlock / 32][kIdxWarpMax];     // pass-1 bucket keys (nbk < 256)
    const bool stage = nbk < 256;
    for (uint32_t i = threadIdx.x; i <= nbk; i += blockDim.x) sb[i] = bnd[i];
    __syncthreads();
    const unsigned lane = threadIdx.x & 31;
    uint32_t* hw = sh[threadIdx.x >> 5];
    const unsigned long long H0 = hcount[0];
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    for (unsigned long long h = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; h < H0; h += nwarps) {
        const uint32_t v = q0[h];
        const int64_t b = off[v], d = off[v + 1] - b;
        if (lane == 0) {
            reinterpret_cast<uint32_t*>(vi + v)[2] = (uint32_t)h;
        }
        for (uint32_t i = lane; i <= nbk; i += 32) hw[i] = 0;
        __syncwarp();
        uint8_t* kw = skey[threadIdx.x >> 5];
        for (int64_t x0 = lane; x0 - lane < d; x0 += 32 * kIdxILP) {
            float f[kIdxILP];
#pragma unroll
            for (int q = 0; q < kIdxILP; ++q) f[q] = x0 + 32 * q < d ? __ldg(w + b + x0 + 32 * q) : 0.0f;
#pragma unroll
            for (int q = 0; q < kIdxILP; ++q) {
                const int64_t x = x0 + 32 * q;
                const uint32_t key = x < d ? bucket_fast(sb, nbk, f[q], wmin, inv_l2g) : kSentinel;
                agg_count(hw, key);
                if (stage && x < d) kw[x] = (uint8_t)key;
            }
        }
        __syncwarp();
        uint32_t carry = 0;                                     // exclusive scan of the bins
        for (uint32_t b0 = 0; b0 <= nbk; b0 += 32) {
            const uint32_t i = b0 + lane;
            const uint32_t c = i <= nbk ? hw[i] : 0u;
            uint32_t incl = c;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (unsigned)o) incl += t;
            }
            if (i <= nbk) hw[i] = carry + incl - c;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        unsigned long long* hs = hstart + h * (nbk + 1);          // absolute bucket starts in hidx
        for (uint32_t i = lane; i <= nbk; i += 32) hs[i] = qb0[h] + hw[i];
        __syncwarp();
        const unsigned long long hb = qb0[h];
        if (stage) {                                            // keys from pass 1: no second weight read
            for (int64_t x = lane; x - lane < d; x += 32) {
                const uint32_t key = x < d ? (uint32_t)kw[x] : kSentinel;
                const uint32_t slot = agg_slot(hw, key);
                if (x < d) hidx[hb + slot] = (uint32_t)x;
            }
        } else {
            for (int64_t x0 = lane; x0 - lane < d; x0 += 32 * kIdxILP) {
                float f[kIdxILP];
#pragma unroll
                for (int q = 0; q < kIdxILP; ++q) f[q] = x0 + 32 * q < d ? __ldg(w + b + x0 + 32 * q) : 0.0f;
#pragma unroll
                for (int q = 0; q < kIdxILP; ++q) {
                    const int64_t x = x0 + 32 * q;
                    const uint32_t key = x < d ? bucket_fast(sb, nbk, f[q], wmin, inv_l2g) : kSentinel;
                    const uint32_t slot = agg_slot(hw, key);
                    if (x < d) hidx[hb + slot] = (uint32_t)x;
                }
            }
        }
        __syncwarp();
    }
}

// The long lists of this round: one warp per kAmsfChunk-entry piece.
template <int MODE, bool VEC>
__global__ void __launch_bounds__(kBlock) k_amsf_chunks(const int64_t* __restrict__ off,
                                                        const uint32_t* __restrict__ adj, const float* __restrict__ w,
                                                        uint32_t* P, double blo, double bhi,
                                                        const uint2* __restrict__ chq, const AmsfCtl* ac, uint2* F,
                                                        float* Fw, cc_counters* cnt)
{
    pdl_trigger();
    pdl_wait();
    const unsigned lane = threadIdx.x & 31;
    const unsigned long long total = ac->chunks;
    const unsigned long long warp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    uint32_t hooks = 0, links = 0;
    unsigned long long scanned = 0;
    for (unsigned long long q = warp; q < total; q += nwarps) {
        const uint2 item = chq[q];
        const int64_t b = off[item.x] + (int64_t)item.y * kAmsfChunk;
        const int64_t e = min(off[item.x + 1], b + kAmsfChunk);
        scanned += lane == 0 ? (unsigned long long)(e - b) : 0ull;
        if (VEC) {
            // 16-byte weight loads from the aligned quad containing b: 4 in flight per lane
            // (16 weights), entries outside [b, e) ignored
            const float4* w4 = reinterpret_cast<const float4*>(w);
            for (int64_t q0 = (b >> 2) + lane; q0 * 4 < e; q0 += 32 * 4) {
                float4 wq[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t x0 = (q0 + 32 * j) * 4;
                    // the whole quad only when it ends inside the piece (e <= m, so never past
                    // the end of w); a quad straddling e takes its entries below e one by one
                    if (x0 + 4 <= e) {
                        wq[j] = w4[q0 + 32 * j];
                    } else {
                        wq[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (x0 < e) wq[j].x = w[x0];
                        if (x0 + 1 < e) wq[j].y = w[x0 + 1];
                        if (x0 + 2 < e) wq[j].z = w[x0 + 2];
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float v4[4] = {wq[j].x, wq[j].y, wq[j].z, wq[j].w};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int64_t x = (q0 + 32 * j) * 4 + c;
                        const double xd = (double)v4[c];
                        if (x >= b && x < e && xd >= blo && xd < bhi) {
                            CC_AMSF_LINK_INC(links);
                            hooks += link<MODE>(P, item.x, adj[x], ForestW{F, Fw, v4[c]});
                        }
                    }
                }
            }
        } else {
            // 8 weight loads in flight per lane (the sweep is latency-bound otherwise)
            for (int64_t x0 = b + lane; x0 < e; x0 += 32 * 8) {
                float wx[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) wx[j] = x0 + 32 * j < e ? w[x0 + 32 * j] : 0.0f;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const double xd = (double)wx[j];
                    if (xd >= blo && xd < bhi) {
                        CC_AMSF_LINK_INC(links);
                        hooks += link<MODE>(P, item.x, adj[x0 + 32 * j], ForestW{F, Fw, wx[j]});
                    }
                }
            }
        }
    }
    if (cnt) {
        warp_count(&cnt->amsf_hooks, hooks);
        CC_AMSF_LINK_FLUSH(cnt, links);
        const unsigned long long sc = __reduce_add_sync(0xffffffffu, (uint32_t)min(scanned, 0xFFFFFFFFull));
        if (lane == 0 && sc) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt->amsf_edges), sc);
    }
}

__global__ void k_amsf_next(AmsfCtl* ac, int in_slot, cc_counters* cnt)
{
    pdl_trigger();
    pdl_wait();
    ac->chunks = 0;
    ac->cnt[in_slot] = 0;                                      // becomes the next round's output
    if (cnt) {
        cnt->amsf_rounds += 1;
        cnt->amsf_rebuilds += ac->rebuild;
    }
}

// sum of the forest weights (fp64)
__global__ void __launch_bounds__(kBlock) k_amsf_total(const float* ew, const int64_t* ne, double* total)
{
    const uint64_t k = (uint64_t)*ne;
    double s = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x)
        s += (double)ew[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(total, s);
}

template <int MODE>
cc_status amsf_run(const int64_t* off, const uint32_t* adj, const float* w, uint32_t n, int64_t m, double eps,
                   uint32_t* edges, float* edge_w, int64_t* num_edges, double* total, const cc_opts& o,
                   cudaStream_t s)
{
    const bool skip = !(o.flags & CC_FLAG_NO_SKIP);
    const bool plain = (o.flags & CC_FLAG_AMSF_PLAIN) != 0;
    bool index = false;                       // hub bucket index (set once nb is known)
    const char* tr = std::getenv("CC_AMSF_TRACE");
    const bool trace = tr && tr[0] == '1';
    AmsfCtl* ac = nullptr;
    uint32_t *P = nullptr, *fb = nullptr, *order = nullptr;
    uint4* vi = nullptr;                      // per vertex: lightest / heaviest weight bits, hub id
    uint32_t* carry[2] = {nullptr, nullptr};
    uint2* F = nullptr;
    uint2* chq = nullptr;
    uint32_t *hubs = nullptr, *hidx = nullptr;
    unsigned long long *hdeg = nullptr, *hstart = nullptr, *hcount = nullptr;
    float* Fw = nullptr;
    double* bd = nullptr;
    float* bfl = nullptr;
    std::vector<float> fbv;
    unsigned long long *start = nullptr, *cursor = nullptr;
    uint32_t* fcnt = nullptr;
    unsigned long long* foff = nullptr;
    uint32_t* tile_vs = nullptr;
    const uint32_t nfb = (uint32_t)(((uint64_t)n + kFTile - 1) / kFTile);
    auto body = [&]() -> cc_status {
        CC_CUDA_TRY(scratch_alloc((void**)&ac, sizeof(AmsfCtl), s));
        CC_CUDA_TRY(scratch_alloc((void**)&P, sizeof(uint32_t) * n, s));
        CC_CUDA_TRY(scratch_alloc((void**)&vi, sizeof(uint4) * n, s));
        CC_CUDA_TRY(scratch_alloc((void**)&F, sizeof(uint2) * n, s));
        CC_CUDA_TRY(scratch_alloc((void**)&Fw, sizeof(float) * n, s));
        AmsfCtl h0{};
        h0.wmin_bits = kPosInfBits;
        h0.anchor = kSentinel;
        h0.skip_root = kSentinel;
        CC_CUDA_TRY(cudaMemcpyAsync(ac, &h0, sizeof(h0), cudaMemcpyHostToDevice, s));
        const uint64_t ntiles = (uint64_t)((m + kWrTile - 1) / kWrTile);
        if (m > 0) CC_CUDA_TRY(scratch_alloc((void**)&tile_vs, sizeof(uint32_t) * ntiles, s));
        k_amsf_init<<<grid_blocks(8), kBlock, 0, s>>>(off, P, vi, F, n, m > 0 ? tile_vs : nullptr);
        CC_LAUNCH_CHECK("k_amsf_init");
        if (m > 0) {
            k_amsf_wrange<<<grid_blocks(16), kBlock, 0, s>>>(off, w, n, m, tile_vs, vi, ac);
            CC_LAUNCH_CHECK("k_amsf_wrange");
        }
        AmsfCtl h{};
        CC_CUDA_TRY(cudaMemcpyAsync(&h, ac, sizeof(h), cudaMemcpyDeviceToHost, s));
        CC_CUDA_TRY(cudaStreamSynchronize(s));
        if (h.bad) {
            set_error("cc_amsf: a weight is <= 0 or not finite");
            return CC_EINVAL;
        }
        uint32_t nb = 0;
        std::vector<double> b;
        if (m > 0) {
            // bucket boundaries (reading R25): b_0 = W_min, b_(i+1) = b_i * (1 + eps), up to
            // the first one above W_max -- the same fp64 product chain as the oracle
            float fmin, fmax;
            std::memcpy(&fmin, &h.wmin_bits, 4);
            std::memcpy(&fmax, &h.wmax_bits, 4);
            const double wmin = fmin, wmax = fmax;
            const double g = 1.0 + eps;
            b.push_back(wmin);
            while (b.back() * g <= wmax) {
                b.push_back(b.back() * g);
                if (b.size() > (1u << 24)) {
                    set_error("cc_amsf: more than 2^24 weight buckets (eps too small)");
                    return CC_ERANGE;
                }
            }
            b.push_back(b.back() * g);
            nb = (uint32_t)(b.size() - 1);
            index = !plain && nb <= kIdxBins && !(o.flags & CC_FLAG_AMSF_NO_INDEX);
            CC_CUDA_TRY(scratch_alloc((void**)&bd, sizeof(double) * b.size(), s));
            CC_CUDA_TRY(cudaMemcpyAsync(bd, b.data(), sizeof(double) * b.size(), cudaMemcpyHostToDevice, s));
            // the same boundaries as float thresholds: fb_i = the smallest float >= b_i, so that
            // b_i <= (double)x  <=>  fb_i <= x for every float weight x (exact, reading R25)
            fbv.resize(b.size());
            for (size_t k = 0; k < b.size(); ++k) {
                float f = (float)b[k];
                if ((double)f < b[k]) f = std::nextafter(f, INFINITY);
                fbv[k] = f;
            }
            CC_CUDA_TRY(scratch_alloc((void**)&bfl, sizeof(float) * fbv.size(), s));
            CC_CUDA_TRY(cudaMemcpyAsync(bfl, fbv.data(), sizeof(float) * fbv.size(), cudaMemcpyHostToDevice, s));
            CC_CUDA_TRY(scratch_alloc((void**)&fb, sizeof(uint32_t) * n, s));
            CC_CUDA_TRY(scratch_alloc((void**)&order, sizeof(uint32_t) * n, s));
            CC_CUDA_TRY(scratch_alloc((void**)&carry[0], sizeof(uint32_t) * n, s));
            CC_CUDA_TRY(scratch_alloc((void**)&carry[1], sizeof(uint32_t) * n, s));
            // long-list pieces of one round: at most one per kAmsfChunk adjacency entries (+1 per vertex)
            CC_CUDA_TRY(scratch_alloc((void**)&chq, sizeof(uint2) * (size_t)(m / kAmsfChunk + std::min<int64_t>(n, m / kAmsfChunk + 1) + 1), s));
            CC_CUDA_TRY(scratch_alloc((void**)&start, sizeof(unsigned long long) * (nb + 1), s));
            CC_CUDA_TRY(scratch_alloc((void**)&cursor, sizeof(unsigned long long) * (nb + 1), s));
            CC_CUDA_TRY(cudaMemsetAsync(start, 0, sizeof(unsigned long long) * (nb + 1), s));
            // activation order: non-isolated vertices by the bucket of their lightest edge
            k_amsf_first<<<grid_blocks(8), kBlock, 0, s>>>(vi, n, bd, nb, plain, fb, start);
            CC_LAUNCH_CHECK("k_amsf_first");
            k_amsf_scan<<<1, kBlock, 0, s>>>(start, nb);
            CC_LAUNCH_CHECK("k_amsf_scan");
            CC_CUDA_TRY(cudaMemcpyAsync(cursor, start, sizeof(unsigned long long) * (nb + 1), cudaMemcpyDeviceToDevice, s));
            k_amsf_scatter<<<grid_blocks(8), kBlock, 0, s>>>(vi, fb, n, nb, cursor, order);
            CC_LAUNCH_CHECK("k_amsf_scatter");
            if (index) {
                // bucket index: lists longer than kIdxMin grouped by bucket, once; the list
                // counts are read back (one more host sync) to size the per-list bucket starts
                const uint64_t qcap0 = std::max<uint64_t>(1, std::min<uint64_t>(n, (uint64_t)m / (kIdxMin + 1) + 1));
                const uint64_t qcap1 = std::max<uint64_t>(1, std::min<uint64_t>(n, (uint64_t)m / (kIdxWarpMax + 1) + 1));
                CC_CUDA_TRY(scratch_alloc((void**)&hubs, sizeof(uint32_t) * (qcap0 + qcap1), s));
                CC_CUDA_TRY(scratch_alloc((void**)&hdeg, sizeof(unsigned long long) * (qcap0 + qcap1), s));
                CC_CUDA_TRY(scratch_alloc((void**)&hcount, 3 * sizeof(unsigned long long), s));
                CC_CUDA_TRY(cudaMemsetAsync(hcount, 0, 3 * sizeof(unsigned long long), s));
                uint32_t *q0 = hubs, *q1 = hubs + qcap0;
                unsigned long long *qb0 = hdeg, *qb1 = hdeg + qcap0;
                k_amsf_hubs<<<grid_blocks(8), kBlock, 0, s>>>(off, n, q0, q1, qb0, qb1, hcount);
                CC_LAUNCH_CHECK("k_amsf_hubs");
                unsigned long long hc[3] = {0, 0, 0};
                CC_CUDA_TRY(cudaMemcpyAsync(hc, hcount, sizeof(hc), cudaMemcpyDeviceToHost, s));
                CC_CUDA_TRY(cudaStreamSynchronize(s));
                const uint64_t H = hc[0] + hc[1];
                CC_CUDA_TRY(scratch_alloc((void**)&hstart, sizeof(unsigned long long) * std::max<uint64_t>(H, 1) * (nb + 1), s));
                CC_CUDA_TRY(scratch_alloc((void**)&hidx, sizeof(uint32_t) * std::max<uint64_t>(hc[2], 1), s));
                const float wmin_f = (float)b[0], il2g = (float)(1.0 / std::log2(1.0 + eps));
                if (hc[0]) {
                    if (nb + 1 <= kIdxWarpBins) {
                        k_amsf_idx_warp<<<grid_blocks(16), kIdxWBlock, 0, s>>>(off, w, q0, qb0, hcount, bfl, nb, wmin_f, il2g, vi,
                                                                  hstart, hidx);
                        CC_LAUNCH_CHECK("k_amsf_idx_warp");
                    } else {
                        index = false;                      // too many buckets for the warp build: no index
                    }
                }
                if (index && hc[1]) {
                    k_amsf_hub_index<<<grid_blocks(2), 1024, 0, s>>>(off, w, q1, qb1, hcount, bfl, nb, wmin_f, il2g, vi, hstart,
                                                              hidx);
                    CC_LAUNCH_CHECK("k_amsf_hub_index");
                }
            }
        }
        // the rounds: bucket i = [b_i, b_(i+1)), lightest first
        for (uint32_t i = 0; i < nb; ++i) {
            const int in_slot = i & 1;
            if (skip) {
                CC_CUDA_TRY(launch_pdl(k_amsf_lmax, 1, 1024, s, P, n, o.seed, i, o.samples, ac));
                CC_LAUNCH_CHECK("k_amsf_lmax");
            }
            CC_CUDA_TRY(launch_pdl(k_amsf_round<MODE>, resident_grid(k_amsf_round<MODE>, kBlock), kBlock, s, off, adj, w, P, vi, order, start, i, b[i], b[i + 1],
                                                          carry[in_slot], ac, in_slot, carry[in_slot ^ 1],
                                                          skip, plain, F, Fw, chq, index ? hstart : nullptr,
                                                          hidx, nb, o.counters));
            CC_LAUNCH_CHECK("k_amsf_round");
            if (index)
                CC_CUDA_TRY(launch_pdl(k_amsf_hub_pieces<MODE>, resident_grid(k_amsf_hub_pieces<MODE>, kBlock), kBlock, s, off, adj, w, P, i, chq, ac, vi, hstart, hidx,
                                                                   nb, F, Fw, o.counters));
            else if (((uintptr_t)w & 15u) == 0)
                CC_CUDA_TRY(launch_pdl(k_amsf_chunks<MODE, true>, resident_grid(k_amsf_chunks<MODE, true>, kBlock), kBlock, s, off, adj, w, P, b[i], b[i + 1], chq, ac, F, Fw,
                                                                     o.counters));
            else
                CC_CUDA_TRY(launch_pdl(k_amsf_chunks<MODE, false>, resident_grid(k_amsf_chunks<MODE, false>, kBlock), kBlock, s, off, adj, w, P, b[i], b[i + 1], chq, ac, F,
                                                                      Fw, o.counters));
            CC_LAUNCH_CHECK("k_amsf_chunks");
            CC_CUDA_TRY(launch_pdl(k_amsf_next, 1, 1, s, ac, in_slot, o.counters));
            CC_LAUNCH_CHECK("k_amsf_next");
            if (trace && o.counters) {                       // diagnostics only (CC_AMSF_TRACE=1)
                cc_counters c{};
                AmsfCtl hc{};
                CC_CUDA_TRY(cudaMemcpyAsync(&c, o.counters, sizeof(c), cudaMemcpyDeviceToHost, s));
                CC_CUDA_TRY(cudaMemcpyAsync(&hc, ac, sizeof(hc), cudaMemcpyDeviceToHost, s));
                CC_CUDA_TRY(cudaStreamSynchronize(s));
                std::fprintf(stderr, "amsf round %u visits %llu edges %llu hooks %llu carry %llu anchor %u skip %u\n", i,
                             (unsigned long long)c.amsf_visits, (unsigned long long)c.amsf_edges,
                             (unsigned long long)c.amsf_hooks, hc.cnt[in_slot ^ 1], hc.anchor, hc.skip_root);
            }
        }
        // Filter: the non-empty slots, in slot order, with their weights
        CC_CUDA_TRY(scratch_alloc((void**)&fcnt, sizeof(uint32_t), s));
        CC_CUDA_TRY(scratch_alloc((void**)&foff, sizeof(unsigned long long) * nfb, s));
        CC_CUDA_TRY(cudaMemsetAsync(fcnt, 0, sizeof(uint32_t), s));
        CC_CUDA_TRY(cudaMemsetAsync(foff, 0, sizeof(unsigned long long) * nfb, s));
        float* ew = edge_w;
        if (!ew && total) {
            CC_CUDA_TRY(scratch_alloc((void**)&ew, sizeof(float) * n, s));
        }
        k_forest_filter<<<nfb, kBlock, 0, s>>>(F, n, nfb, foff, fcnt, edges, num_edges, Fw, ew);
        CC_LAUNCH_CHECK("k_forest_filter");
        if (total) {
            CC_CUDA_TRY(cudaMemsetAsync(total, 0, sizeof(double), s));
            k_amsf_total<<<grid_blocks(4), kBlock, 0, s>>>(ew, num_edges, total);
            CC_LAUNCH_CHECK("k_amsf_total");
        }
        if (ew != edge_w) scratch_free(ew, s);
        return CC_OK;
    };
    const cc_status rc = body();
    for (void* p : {(void*)ac, (void*)P, (void*)vi, (void*)fb, (void*)order, (void*)carry[0],
                    (void*)carry[1], (void*)F, (void*)Fw, (void*)chq, (void*)hubs, (void*)hstart,
                    (void*)hidx, (void*)hdeg, (void*)hcount, (void*)bd, (void*)bfl, (void*)start, (void*)cursor, (void*)fcnt,
                    (void*)foff, (void*)tile_vs})
        scratch_free(p, s);
    return rc;
}

}  // namespace

cc_status amsf_pipeline(const int64_t* off, const uint32_t* adj, const float* w, uint32_t n, int64_t m, double eps,
                        uint32_t* edges, float* edge_w, int64_t* num_edges, double* total, const cc_opts& o,
                        cudaStream_t s)
{
    if (o.flags & CC_FLAG_UF_ASYNC) return amsf_run<2>(off, adj, w, n, m, eps, edges, edge_w, num_edges, total, o, s);
    if (o.flags & CC_FLAG_HALVE) return amsf_run<1>(off, adj, w, n, m, eps, edges, edge_w, num_edges, total, o, s);
    return amsf_run<0>(off, adj, w, n, m, eps, edges, edge_w, num_edges, total, o, s);
}

}  // namespace ccb
