// cc_static.cu -- static connectivity / spanning forest pipeline (H1-H7).
//
// Alg. 1 / Alg. 2 on one B200, stream-ordered with
// no host synchronisation: L_max, every queue length and every kernel choice
// stay in device memory.  Every kernel is a programmatic dependent launch
// (launch_pdl; pdl_trigger + pdl_wait at its entry).
//
//   K0 k_sample_init  H1 P[v] = v fused with the first k-out round: each vertex
//                     u with first neighbour v0 < u sets P[u] = v0 by a plain
//                     store (u is still a singleton root and only u writes
//                     slot u in this kernel, so this IS Union(u, v0) of
//                     Alg. 4 P:3952 with the min orientation of R1).  All other
//                     sampled edges (v0 > u, j = 1..k-1) go to a pending list;
//                     a bitmap marks vertices whose list was not wholly sampled
//                     (degree skip).
//   Kp k_probe        round-0 chain depth from 1024 seeded walks: gates the mid
//                     compress and picks the link kernel (device-side flag)
//   Kc k_compress     pointer-jumping compress ("fully compress"),
//                     root walks halving deep chains (root_halve)
//   K1 k_link_pending UF-Rem-CAS + SplitAtomicOne links of the pending sampled
//                     edges, one per thread (short chains: the default on RMAT/ER),
//      k_link_refill  or with lane refill (long chains: grid-like ids; cc_common.cuh);
//                     k_link_contract on the contracted forest (CC_FLAG_CONTRACT)
//   K4 k_identify     IdentifyFrequent over S seeded samples (R9)
//   K5 k_finish       ONE pass over P fusing the sampling compress (H3) with
//                     the finish scan (H5): every vertex is compressed to its
//                     root r; a marked vertex with r != L_max is queued, and
//                     k_finish_proc / k_finish_big union its list,
//                     degree-binned: warp-shared sweep / CTA per list / all
//                     CTAs per huge list; per-warp foreign-root summaries
//   K5' sv_finish     the finish as Shiloach-Vishkin (= Liu-Tarjan PRF) or
//                     Liu-Tarjan CRFA rounds (CC_FLAG_FINISH_SV / _CRFA) over the
//                     candidates' edges (k_sv_copy + k_sv_pieces for lists in
//                     4096-entry pieces; appends through WarpBuf; writeMin tested
//                     before the atomic)
//   K6 k_relabel_decide + k_relabel   H6 as a partial pass: only the tiles
//                     whose labels H5 changed (k_compress for a full pass)
//   K7 forest         Filter of Alg. 2: compact non-sentinel slots in
//                     slot order (cc_common.cuh)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "cc_common.cuh"
#include "cc_device.cuh"
#include "cc_internal.h"

namespace ccb {

struct Ctl {
    unsigned long long pend_count;
    unsigned long long cand_count;
    unsigned long long big_count;
    unsigned long long huge_count;   // lists > kHugeDeg, filled from the END of the big queue
    unsigned int lmax;
    unsigned int err;
    unsigned int skip_mid;      // set by k_probe: the round-0 chains are short
    unsigned long long rl_count;   // k_relabel_decide: dirty 512-slot chunks queued for k_relabel
};

#ifndef CC_BIG_DEG
#define CC_BIG_DEG 4096
#endif
constexpr int kBigDeg = CC_BIG_DEG; // >  : one CTA per vertex (second kernel)
constexpr int64_t kHugeDeg = 1 << 20;   // >  : every CTA takes a slice of the list

// ---------------------------------------------------------------------------
// K0: H1 + first k-out round + pending list + finish bitmap.
//
// Each warp owns a tile of 256 consecutive vertices, 8 per lane (vertex
// wbase + 32*j + lane), so every offsets/P access is a coalesced warp
// transaction and each lane keeps 8 independent first-neighbour loads in
// flight (Little's law: tens of KB per SM outstanding).  Pending links are
// appended in vertex order within a block with ONE atomicAdd per block (a
// per-warp atomic on a single address serialised the first version at L2).
// The finish bitmap has bit (u & 31) of word u >> 5 set iff deg(u) > full_deg.
#ifndef CC_SI_KV
#define CC_SI_KV 8
#endif
#ifndef CC_SI_MINB
#define CC_SI_MINB 3
#endif
constexpr int kV = CC_SI_KV;                 // vertices per lane
constexpr int kWarpTile = 32 * kV;           // 256 vertices per warp
constexpr int kBlockTile = kWarpTile * (kBlock / 32);

// Sampled neighbours j = 0 and j = 1 of a list starting at o: with WIN (adj
// 16-byte aligned, in pinned host memory) both come from ONE aligned 16-byte
// window load when they share it (3 of 4 list starts), halving the PCIe read
// requests of the zero-copy path.
template <bool WIN>
__device__ __forceinline__ uint32_t pick4(uint4 w, uint32_t r)
{
    return r == 0 ? w.x : r == 1 ? w.y : r == 2 ? w.z : w.w;
}

// VAR: 0 = afforest (positions 0..k-1), 1 = hybrid (0, then k-1 uniform picks),
// 2 = pure (k uniform picks) -- cc.h CC_VARIANT_*.
template <int VAR, bool SF, bool WIN, bool RB>
__global__ void __launch_bounds__(kBlock, CC_SI_MINB) k_sample_init(
    const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, uint32_t n, int64_t m, uint32_t k,
    uint64_t seed, uint32_t full_deg, uint32_t* __restrict__ P, uint2* __restrict__ F,
    uint2* __restrict__ pend, uint32_t* __restrict__ bm, uint2* __restrict__ rbw, Ctl* ctl, cc_counters* cnt)
{
    pdl_trigger();
    pdl_wait();
    __shared__ uint32_t s_wtot[kBlock / 32];
    __shared__ unsigned long long s_wbase[kBlock / 32];
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t wbase = (uint64_t)blockIdx.x * kBlockTile + (uint64_t)w * kWarpTile;

    int64_t o[kV];
    uint32_t d[kV];                              // list length, saturated at 2^32-1
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        const uint64_t u = wbase + 32 * j + lane;
        o[j] = ld_stream_i64(off + (u < n ? u : n));
    }
    const int64_t last = ld_stream_i64(off + (wbase + kWarpTile < n ? wbase + kWarpTile : n));
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        const int64_t nx = __shfl_down_sync(0xffffffffu, o[j], 1);
        const int64_t first_next = __shfl_sync(0xffffffffu, j + 1 < kV ? o[(j + 1) % kV] : last, 0);
        const int64_t e = lane == 31 ? (j + 1 < kV ? first_next : last) : nx;
        const uint64_t u = wbase + 32 * j + lane;
        d[j] = u < n ? (uint32_t)min(e - o[j], (int64_t)0xFFFFFFFF) : 0u;
    }
    // the first two sampled neighbours of every vertex, all loads in flight together
    uint32_t v0[kV], v1[kV];
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        const uint64_t u = wbase + 32 * j + lane;
        uint32_t i0 = 0, i1 = 1;
        if (VAR == 2 && d[j] > 0) i0 = uniform_below(mix(seed, KOUT_STREAM, u * 64 + 0), d[j]);
        if (VAR >= 1 && d[j] > 0) i1 = uniform_below(mix(seed, KOUT_STREAM, u * 64 + 1), d[j]);
        const bool need0 = d[j] > 0 && k > 0;
        const bool need1 = k > 1 && (VAR >= 1 ? d[j] > 0 : d[j] > 1);
        v0[j] = v1[j] = kSentinel;
        const int64_t b4 = o[j] & ~(int64_t)3;
        const uint32_t r = (uint32_t)(o[j] & 3);
        if (WIN && VAR != 2 && need0 && b4 + 4 <= m) {
            const uint4 wv = __ldg(reinterpret_cast<const uint4*>(adj + b4));
            v0[j] = pick4<WIN>(wv, r);
            if (need1 && r + i1 < 4) v1[j] = pick4<WIN>(wv, r + i1);
            else if (need1) v1[j] = __ldg(adj + o[j] + i1);
        } else {
            if (need0) v0[j] = __ldg(adj + o[j] + i0);
            if (need1) v1[j] = __ldg(adj + o[j] + i1);
        }
    }
    uint32_t c[kV];
    uint32_t bits = 0, rbits = 0, nwl = 0;
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        const uint64_t u = wbase + 32 * j + lane;
        uint32_t np = 0;
        if (v0[j] != kSentinel)
            np = (v0[j] > (uint32_t)u ? 1u : 0u) + (VAR >= 1 ? k : min(k, d[j])) - 1u;
        c[j] = np;
        const bool mark = u < n && d[j] > full_deg;
        nwl += mark;
        const uint32_t word = __ballot_sync(0xffffffffu, mark);
        if (lane == (unsigned)j) bits = word;
        if constexpr (RB) {             // non-isolated root of the round-0 forest F0 (contracted link)
            const uint32_t rword = __ballot_sync(0xffffffffu, u < n && d[j] > 0 && !(v0[j] < (uint32_t)u));
            if (lane == (unsigned)j) rbits = rword;
        }
    }
    if (lane < (unsigned)kV && wbase + 32 * lane < n) {
        bm[(wbase >> 5) + lane] = bits;
        if constexpr (RB) rbw[(wbase >> 5) + lane].x = rbits;
    }
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        const uint64_t u = wbase + 32 * j + lane;
        if (u < n) {
            uint32_t p = (uint32_t)u;
            if (v0[j] < (uint32_t)u) p = v0[j];        // Union(u, v0): hook singleton root u
            P[u] = p;
            // forest slots: the round-0 edge at the hooked root, else empty --
            // every slot is written here, so F needs no separate initialisation
            if (SF) F[u] = p != (uint32_t)u ? make_uint2((uint32_t)u, p) : make_uint2(kSentinel, kSentinel);
        }
    }
    // exclusive positions in vertex order: warp scans per j, then block, then one atomic
    uint32_t ex[kV];
    uint32_t run = 0;
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        uint32_t incl = c[j];
#pragma unroll
        for (int o2 = 1; o2 < 32; o2 <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o2);
            if (lane >= (unsigned)o2) incl += t;
        }
        ex[j] = run + incl - c[j];
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_wtot[w] = run;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long acc = 0;
        for (int i = 0; i < kBlock / 32; ++i) {
            s_wbase[i] = acc;
            acc += s_wtot[i];
        }
        const unsigned long long pb = acc ? atomicAdd(&ctl->pend_count, acc) : 0ull;
        for (int i = 0; i < kBlock / 32; ++i) s_wbase[i] += pb;
    }
    __syncthreads();
    const unsigned long long pbase = s_wbase[w];
    uint32_t npt = 0;
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        const uint64_t u = wbase + 32 * j + lane;
        const uint32_t np = c[j];
        npt += np;
        if (np) {
            unsigned long long pos = pbase + ex[j];
            if (v0[j] > (uint32_t)u) pend[pos++] = make_uint2((uint32_t)u, v0[j]);
            const uint32_t kk = VAR >= 1 ? k : min(k, d[j]);
            if (kk > 1) pend[pos++] = make_uint2((uint32_t)u, v1[j]);
            for (uint32_t jj = 2; jj < kk; ++jj) {        // k > 2: the rest, loaded here
                const uint32_t i = VAR >= 1 ? uniform_below(mix(seed, KOUT_STREAM, u * 64 + jj), d[j]) : jj;
                pend[pos++] = make_uint2((uint32_t)u, __ldg(adj + o[j] + i));
            }
        }
    }
    if (cnt) {
        warp_count(&cnt->pending_links, npt);
        warp_count(&cnt->worklist, nwl);
    }
}

// ---------------------------------------------------------------------------
// K0' + K1' fused (CC_FLAG_FUSED_LINK; UF-Rem-CAS + SplitAtomicOne, k <= 2).
//
// k_sample_init streams the CSR heads (HBM-bandwidth work) and k_link_refill
// then makes the random parent accesses of the links (DRAM row-activation
// bound): run back to back, neither overlaps the other.  Here one kernel does
// both per block: it samples its 2048 vertices, queues their links in SHARED
// memory (no pending list through HBM) and links them with the lane-refill
// loop, while the other resident blocks are in their streaming part.
// k_init_pf initialises P (and F) first, so any P[v] a link reads is valid; the
// round-0 hook Union(u, v0), v0 < u, is then a CAS from u to v0 (another
// block's link may already have hooked the root u: the CAS fails and (u, v0)
// is queued as an ordinary link).  Every sampled edge is unioned exactly as in
// Alg. 4; only the order of the unions differs, which does not
// change the partition (P:4259-4280 is linearizable).
// Measured (profiles/r1_fused_link_ab.txt): no overlap gain.  With P in HBM (C4)
// both halves are DRAM-bound and their DRAM times add (3.10-3.18 ms vs 2.89 ms
// split); with P in L2 (C3) it ties the split kernels; C1 gains 7 % (launches);
// a row-major grid (C2) loses the mid compress (45M vs 17M Rem steps).  Kept as
// an option, tested in the option grid.
__global__ void __launch_bounds__(kBlock) k_init_pf(uint32_t* __restrict__ P, uint32_t n, uint2* __restrict__ F)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; 4 * i < n; i += stride) {
        const uint32_t b = (uint32_t)(4 * i);
        if (b + 4 <= n && ((uintptr_t)P & 15u) == 0) {
            reinterpret_cast<uint4*>(P)[i] = make_uint4(b, b + 1, b + 2, b + 3);
        } else {
            for (uint32_t t = b; t < n && t < b + 4; ++t) P[t] = t;
        }
        if (F)
            for (uint32_t t = b; t < n && t < b + 4; ++t) F[t] = make_uint2(kSentinel, kSentinel);
    }
}

#ifndef CC_SL_MINB
#define CC_SL_MINB 3
#endif
template <int VAR, bool SF>
__global__ void __launch_bounds__(kBlock, CC_SL_MINB) k_sample_link(
    const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, uint32_t n, int64_t m, uint32_t k,
    uint64_t seed, uint32_t full_deg, uint32_t* __restrict__ P, uint2* __restrict__ F,
    uint32_t* __restrict__ bm, cc_counters* cnt)
{
    constexpr int NW = kBlock / 32;
    __shared__ uint2 s_q[2 * kBlockTile];                    // the block's links (k <= 2)
    __shared__ uint32_t s_wtot[NW], s_wbase[NW], s_total;
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t wbase = (uint64_t)blockIdx.x * kBlockTile + (uint64_t)w * kWarpTile;

    int64_t o[kV];
    uint32_t d[kV];
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        const uint64_t u = wbase + 32 * j + lane;
        o[j] = ld_stream_i64(off + (u < n ? u : n));
    }
    const int64_t last = ld_stream_i64(off + (wbase + kWarpTile < n ? wbase + kWarpTile : n));
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        const int64_t nx = __shfl_down_sync(0xffffffffu, o[j], 1);
        const int64_t first_next = __shfl_sync(0xffffffffu, j + 1 < kV ? o[(j + 1) % kV] : last, 0);
        const int64_t e = lane == 31 ? (j + 1 < kV ? first_next : last) : nx;
        const uint64_t u = wbase + 32 * j + lane;
        d[j] = u < n ? (uint32_t)min(e - o[j], (int64_t)0xFFFFFFFF) : 0u;
    }
    uint32_t v0[kV], v1[kV];
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        const uint64_t u = wbase + 32 * j + lane;
        uint32_t i0 = 0, i1 = 1;
        if (VAR == 2 && d[j] > 0) i0 = uniform_below(mix(seed, KOUT_STREAM, u * 64 + 0), d[j]);
        if (VAR >= 1 && d[j] > 0) i1 = uniform_below(mix(seed, KOUT_STREAM, u * 64 + 1), d[j]);
        const bool need0 = d[j] > 0 && k > 0;
        const bool need1 = k > 1 && (VAR >= 1 ? d[j] > 0 : d[j] > 1);
        v0[j] = need0 ? __ldg(adj + o[j] + i0) : kSentinel;
        v1[j] = need1 ? __ldg(adj + o[j] + i1) : kSentinel;
    }
    // round 0: hook the (normally still singleton) root u under v0 < u; queue the rest
    uint32_t bits = 0, nwl = 0, q0 = 0, c[kV];
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        const uint64_t u = wbase + 32 * j + lane;
        bool p0 = false;
        if (v0[j] != kSentinel) {
            if (v0[j] < (uint32_t)u) {
                if (cas(P + u, (uint32_t)u, v0[j]) == (uint32_t)u) {
                    if (SF) F[u] = make_uint2((uint32_t)u, v0[j]);
                } else {
                    p0 = true;
                }
            } else {
                p0 = v0[j] != (uint32_t)u;
            }
        }
        q0 |= (uint32_t)p0 << j;
        c[j] = (uint32_t)p0 + (v1[j] != kSentinel ? 1u : 0u);
        const bool mark = u < n && d[j] > full_deg;
        nwl += mark;
        const uint32_t word = __ballot_sync(0xffffffffu, mark);
        if (lane == (unsigned)j) bits = word;
    }
    if (lane < (unsigned)kV && wbase + 32 * lane < n) bm[(wbase >> 5) + lane] = bits;
    // queue positions: warp scans per j, then block
    uint32_t ex[kV];
    uint32_t run = 0;
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        uint32_t incl = c[j];
#pragma unroll
        for (int o2 = 1; o2 < 32; o2 <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o2);
            if (lane >= (unsigned)o2) incl += t;
        }
        ex[j] = run + incl - c[j];
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_wtot[w] = run;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < NW; ++i) {
            s_wbase[i] = acc;
            acc += s_wtot[i];
        }
        s_total = acc;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kV; ++j) {
        const uint32_t u = (uint32_t)(wbase + 32 * j + lane);
        uint32_t pos = s_wbase[w] + ex[j];
        if ((q0 >> j) & 1u) s_q[pos++] = make_uint2(u, v0[j]);
        if (v1[j] != kSentinel) s_q[pos] = make_uint2(u, v1[j]);
    }
    __syncthreads();
    const uint32_t total = s_total;
    if (cnt) {
        if (blockIdx.x == 0 && threadIdx.x == 0) cnt->fused_link = 1;
        uint32_t np = 0;
#pragma unroll
        for (int j = 0; j < kV; ++j) np += c[j];
        warp_count(&cnt->pending_links, np);
        warp_count(&cnt->worklist, nwl);
    }

    // lane-refill link loop over the block's queue (k_link_refill's step, R1/R6);
    // warp w takes the 32-entry chunks w, w + NW, ...
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t chunk = w;
    uint2 nb = make_uint2(0u, 0u);
    uint32_t npu = 0, npv = 0, navail = 0;
    auto fetch = [&]() {
        const uint32_t b0 = chunk * 32;
        navail = b0 < total ? min(32u, total - b0) : 0u;
        const bool ok = lane < navail;
        nb = ok ? s_q[b0 + lane] : make_uint2(0u, 0u);
        npu = ok ? ld_link(P + nb.x) : 0u;
        npv = ok ? ld_link(P + nb.y) : 0u;
        chunk += NW;
    };
    fetch();
    uint2 cb = nb;
    uint32_t cpu = npu, cpv = npv, cavail = navail, cpos = 0;
    if (cavail) fetch();
    bool act = false;
    uint32_t u = 0, v = 0, ru = 0, rv = 0, pu = 0, pv = 0;
    uint32_t hooked = 0, steps = 0, fails = 0;
    while (true) {
        unsigned need = __ballot_sync(0xffffffffu, !act);
        while (need && cavail) {
            const uint32_t src = cpos + __popc(need & lt_mask);
            const uint32_t sl = src & 31;
            const uint32_t xu = __shfl_sync(0xffffffffu, cb.x, sl), xv = __shfl_sync(0xffffffffu, cb.y, sl);
            const uint32_t xpu = __shfl_sync(0xffffffffu, cpu, sl), xpv = __shfl_sync(0xffffffffu, cpv, sl);
            if (!act && src < cavail && xpu != xpv) {
                act = true;
                u = ru = xu;
                v = rv = xv;
                pu = xpu;
                pv = xpv;
            }
            cpos = min(cavail, cpos + (uint32_t)__popc(need));
            if (cpos == cavail) {
                cb = nb;
                cpu = npu;
                cpv = npv;
                cavail = navail;
                cpos = 0;
                if (cavail) fetch();
            }
            need = __ballot_sync(0xffffffffu, !act);
        }
        if (!__any_sync(0xffffffffu, act)) break;
        if (act) {
            ++steps;
            if (pu < pv) {
                uint32_t t = ru; ru = rv; rv = t;
                t = pu; pu = pv; pv = t;
            }
            if (ru == pu) {
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
                const uint32_t wg = ld_link(P + pu);
                if (wg != pu) cas(P + ru, pu, wg);
                ru = pu;
                pu = wg;
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

// ---------------------------------------------------------------------------
// Kc: pointer-jumping compress.  Within this kernel no hook happens, so every
// value read is an ancestor-or-self on the path to the (fixed) root, stale or
// not; plain (L1-cacheable) loads are therefore safe and let the hot giant
// root stay in L1.  Blocks run roughly in ascending id order and P[x] < x, so
// most parents are already compressed when their children are visited.
// Each thread owns 2 x uint4 = 8 slots (2 x 16 B loads in flight per thread)
// and writes a uint4 back only if one of its slots changed.
// resident blocks per SM the streaming passes are compiled for (register caps)
#ifndef CC_COMPRESS_MINB
#define CC_COMPRESS_MINB 8
#endif
#ifndef CC_FINISH_MINB
#define CC_FINISH_MINB 8
#endif
constexpr int kCV = 8;                                   // slots per thread
constexpr int kCTile = kBlock * kCV;                     // 2048 slots per block

__device__ __forceinline__ uint32_t root_plain(const uint32_t* P, uint32_t r)
{
    uint32_t q = P[r];
    while (q != r) {
        r = q;
        q = P[r];
    }
    return r;
}

// Root walk with path halving, for passes in which no hook runs (compress, the
// finish scan): each step points x at its grandparent.  Plain walks were
// quadratic on long chains -- every thread of every resident block walking the
// same uncompressed chain (an id-ordered path: 1.6 s for 16M vertices); with
// halving the concurrent walkers shorten it for each other.  The halving store
// is a CAS on the value just read: a pass's owner thread writes the ROOT into
// its slots, and a plain halving store landing after it would replace that root
// by a mere ancestor (wrong final labels); the CAS fails instead.
__device__ __forceinline__ uint32_t root_halve(uint32_t* P, uint32_t x)
{
    uint32_t p = P[x];
    // the first steps walk without writes (normal trees are shallow after a link
    // phase that splits as it goes), halving only deeper chains
#pragma unroll 1
    for (int i = 0; i < 16 && p != x; ++i) {
        x = p;
        p = P[x];
    }
    while (p != x) {
        const uint32_t g = P[p];
        if (g == p) return p;
        atomicCAS(P + x, p, g);
        x = g;
        p = P[x];
    }
    return x;
}

// Roots of 8 slots with their first-level gathers issued together (8
// independent loads in flight instead of 8 dependent walks); deeper walks,
// rare after a compress, continue one slot at a time.  (A level-by-level
// variant that batches every level measured slower on C4: more registers
// and a serial live-mask loop for little extra parallelism.)
__device__ __forceinline__ uint32_t roots8(uint32_t* P, const uint32_t (&vv)[8], const uint32_t (&pp)[8],
                                           uint32_t (&rr)[8], uint32_t known_root = kSentinel)
{
    uint32_t q[8], gathers = 0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const bool g = !(pp[s] == vv[s] || pp[s] == known_root);
        q[s] = g ? P[pp[s]] : pp[s];
        gathers += g;
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) rr[s] = q[s] == pp[s] ? pp[s] : root_halve(P, q[s]);
    return gathers;                                      // first-level parent reads issued
}

__device__ __forceinline__ uint32_t nchanged4(uint4 a, uint4 b)
{
    return (a.x != b.x) + (a.y != b.y) + (a.z != b.z) + (a.w != b.w);
}

template <bool CNT>
__global__ void __launch_bounds__(kBlock, CC_COMPRESS_MINB) k_compress(uint32_t* P, uint32_t n, uint32_t* out,
                                                                       cc_counters* cnt, const Ctl* gate)
{
    pdl_trigger();
    pdl_wait();
    if (gate && gate->skip_mid) return;
    uint32_t writes = 0, gathers = 0;
    const uint64_t ntiles = ((uint64_t)n + kCTile - 1) / kCTile;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {    // tiles in ascending waves
        const uint64_t base = tile * kCTile;
        if (base + kCTile <= n) {
            const uint64_t i0 = base + 4 * (uint64_t)threadIdx.x, i1 = i0 + 4 * kBlock;
            const uint4 a = reinterpret_cast<const uint4*>(P)[i0 >> 2];
            const uint4 c = reinterpret_cast<const uint4*>(P)[i1 >> 2];
            const uint32_t pp[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
            uint32_t vv[8], rr[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) vv[j] = (uint32_t)((j < 4 ? i0 : i1) + (j & 3));
            const uint32_t g = roots8(P, vv, pp, rr);
            if (CNT) gathers += g;
            const uint4 r0 = make_uint4(rr[0], rr[1], rr[2], rr[3]), r1 = make_uint4(rr[4], rr[5], rr[6], rr[7]);
            const uint32_t c0 = nchanged4(r0, a), c1 = nchanged4(r1, c);
            if (CNT) writes += c0 + c1;
            if (c0) reinterpret_cast<uint4*>(P)[i0 >> 2] = r0;
            if (c1) reinterpret_cast<uint4*>(P)[i1 >> 2] = r1;
            if (out) {
                reinterpret_cast<uint4*>(out)[i0 >> 2] = r0;
                reinterpret_cast<uint4*>(out)[i1 >> 2] = r1;
            }
        } else {
            for (uint64_t v64 = base + threadIdx.x; v64 < n; v64 += kBlock) {      // ragged tail
                const uint32_t v = (uint32_t)v64;
                const uint32_t p = P[v];
                const uint32_t r = p == v ? v : root_halve(P, p);
                if (CNT) gathers += p != v;
                if (r != p) {
                    P[v] = r;
                    if (CNT) ++writes;
                }
                if (out) out[v] = r;
            }
        }
    }
    if (CNT) {
        warp_count(&cnt->h6_writes, writes);
        warp_count(&cnt->h6_gathers, gathers);
    }
}

// scalar variant for buffers that are not 16-byte aligned
__global__ void __launch_bounds__(kBlock) k_compress_scalar(uint32_t* P, uint32_t n, uint32_t* out, cc_counters* cnt,
                                                            const Ctl* gate)
{
    pdl_trigger();
    pdl_wait();
    if (gate && gate->skip_mid) return;
    const uint64_t v64 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t writes = 0;
    if (v64 < n) {
        const uint32_t v = (uint32_t)v64;
        const uint32_t p = P[v];
        const uint32_t r = p == v ? v : root_halve(P, p);
        if (r != p) { P[v] = r; writes = 1; }
        if (out) out[v] = r;
    }
    if (cnt) warp_count(&cnt->h6_writes, writes);
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static cc_status launch_compress(uint32_t* P, uint32_t n, uint32_t* out, cc_counters* cnt, cudaStream_t s,
                                 const char* what, const Ctl* gate = nullptr)
{
    // a gated (maybe skipped) compress runs as a persistent grid so that a skip
    // costs one short wave, not 65k empty blocks; otherwise one block per tile
    const uint64_t ntiles = ((uint64_t)n + kCTile - 1) / kCTile;
    const unsigned grid = (unsigned)(gate ? std::min<uint64_t>(ntiles, (uint64_t)grid_blocks(8)) : ntiles);
    if (aligned16(P) && aligned16(out) && cnt) CC_CUDA_TRY(launch_pdl(k_compress<true>, grid, kBlock, s, P, n, out, cnt, gate));
    else if (aligned16(P) && aligned16(out)) CC_CUDA_TRY(launch_pdl(k_compress<false>, grid, kBlock, s, P, n, out, nullptr, gate));
    else
        CC_CUDA_TRY(launch_pdl(k_compress_scalar, (unsigned)(((uint64_t)n + kBlock - 1) / kBlock), kBlock, s, P, n, out, cnt, gate));
    CC_LAUNCH_CHECK(what);
    return CC_OK;
}

// ---------------------------------------------------------------------------
// k_probe: is the mid compress worth a pass over P?  Walk up to kProbeDepth
// steps from 1024 seeded vertices of the round-0 forest; if at least 1/8 of
// them have not reached a root, the chains are long (ids with locality, e.g.
// the road-like grid, whose first neighbours chain up whole columns) and the
// compress runs; otherwise (random-permuted RMAT/ER) it is skipped and the CAS
// links walk the short chains themselves.  The decision stays on the device.
constexpr int kProbeDepth = 8;
constexpr uint64_t PROBE_STREAM = 18;

__global__ void __launch_bounds__(1024) k_probe(const uint32_t* P, uint32_t n, uint64_t seed, Ctl* ctl,
                                                cc_counters* cnt)
{
    pdl_trigger();
    pdl_wait();
    __shared__ uint32_t s_deep;
    if (threadIdx.x == 0) s_deep = 0;
    __syncthreads();
    uint32_t x = uniform_below(mix(seed, PROBE_STREAM, threadIdx.x), n);
    int steps = 0;
    for (uint32_t p = P[x]; p != x && steps < kProbeDepth; p = P[x], ++steps) x = p;
    const uint32_t deep = __reduce_add_sync(0xffffffffu, steps >= kProbeDepth ? 1u : 0u);
    if ((threadIdx.x & 31) == 0 && deep) atomicAdd(&s_deep, deep);
    __syncthreads();
    if (threadIdx.x == 0) {
        ctl->skip_mid = s_deep * 8 < blockDim.x ? 1u : 0u;
        if (cnt) {
            atomicAdd(reinterpret_cast<unsigned long long*>(&cnt->probe_deep), (unsigned long long)s_deep);
            if (!ctl->skip_mid) cnt->mid_compress = 1;
        }
    }
}

// ---------------------------------------------------------------------------
// K1: UF-Rem-CAS links of the pending sampled edges.  Each thread takes kLB
// links spaced one grid apart (coalesced pair loads) and issues their first
// parent reads together; most links end at that first test (equal parents),
// the rest continue in link_rem_from.  The __syncwarp re-converges the warp so
// the next group's loads are issued as whole-warp transactions again.  With
// the L1-cached Rem reads, PDL and a one-wave grid, ONE link per thread per
// iteration measured fastest (round 2; kLB 1 / 2 / 3 / 4, C4 link 1.49 / 1.56 /
// 1.57 / 1.63 ms, C3 0.18 / 0.19 / 0.20 / 0.20 ms) and faster than the lane-
// refill kernel (C4 1.68, C3 0.25 ms) except on grid-like inputs with long
// round-0 chains (C2: 0.40 vs 0.30 ms), which the probe recognises.
#ifndef CC_LINK_BATCH
#define CC_LINK_BATCH 1
#endif
constexpr int kLB = CC_LINK_BATCH;

template <int MODE, bool SF>
__global__ void __launch_bounds__(kBlock) k_link_pending(
    uint32_t* P, const uint2* __restrict__ pend, const Ctl* ctl, uint2* F, cc_counters* cnt, bool gated)
{
    pdl_trigger();
    pdl_wait();
    if (gated && !ctl->skip_mid) return;             // the device-side kernel choice picked k_link_refill
    if (cnt && blockIdx.x == 0 && threadIdx.x == 0) cnt->link_pending = 1;
    const unsigned long long total = ctl->pend_count;
    const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    Stat st;
    for (unsigned long long base = 0; base < total; base += nthreads * kLB) {
        uint2 pr[kLB];
        uint32_t pu[kLB], pv[kLB];
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
            const unsigned long long i = base + q * nthreads + tid;
            pr[q] = i < total ? pend[i] : make_uint2(0u, 0u);
        }
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
            pu[q] = ld_link(P + pr[q].x);
            pv[q] = ld_link(P + pr[q].y);
        }
        uint32_t hooked = 0;
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
            if (pu[q] == pv[q]) continue;
            if constexpr (MODE == 2) {
                if constexpr (SF) hooked += link_async(P, pr[q].x, pr[q].y, Forest{F});
                else hooked += link_async(P, pr[q].x, pr[q].y, NoForest{});
            } else {
                if constexpr (SF) hooked += link_rem_from<MODE == 1>(P, pr[q].x, pr[q].y, pu[q], pv[q], Forest{F}, cnt ? &st : nullptr);
                else hooked += link_rem_from<MODE == 1>(P, pr[q].x, pr[q].y, pu[q], pv[q], NoForest{}, cnt ? &st : nullptr);
            }
        }
        __syncwarp();
        if (cnt) warp_count(&cnt->sample_hooks, hooked);
    }
    if (cnt) {
        warp_count(&cnt->link_steps, st.steps);
        warp_count(&cnt->cas_failures, st.fails);
    }
}

// ---------------------------------------------------------------------------
// Contracted k-out link (CC_FLAG_CONTRACT; measured slower than the in-place
// link on C3/C4 -- DESIGN.md §6 -- and kept as an evaluated alternative).
//
// After round 0 the parent array is a forest F0: P[u] = v0(u) when the first
// sampled neighbour is smaller, else u.  Its roots are the isolated vertices
// and the non-isolated "local minima" (C4: 13.5M of 63M non-isolated).  Every
// remaining sampled edge (u, v) is Union(u, v), and Union(u, v) is
// Union(root_F0(u), root_F0(v)) -- same sets.  So, after one compress of F0
// (P[u] = root_F0(u), a streaming pass whose parents mostly precede their
// children), the CAS links run on a COMPACT parent array C with one slot per
// non-isolated F0 root: the link reads P[u] (coalesced) and P[v] (the one
// random HBM read of a link), maps both roots to compact ids, and the whole
// UF-Rem-CAS walk then runs in C, which (with the 8-byte rank words below)
// stays resident in the 126 MB L2 instead of walking the 512 MiB P.
//
// Compact ids are assigned in id order (the rank of r among the roots), so
// "hook the larger root under the smaller" in C is the same orientation as in
// P (reading R1) and the min-id-root invariant I1 carries over: the root of a
// sampled component is its minimum vertex, which is an F0 root (its own first
// neighbour, if smaller, would be in the component).
//
// rbw[w] (one uint2 per 32 vertices): x = bitmap of the word's non-isolated F0
// roots (written by k_sample_init), y = number of such roots in earlier words.
// cid(r) = rbw[r>>5].y + popc(rbw[r>>5].x & ((1 << (r&31)) - 1)); rid is the
// inverse map (compact -> vertex id).  Neighbours of a vertex have degree > 0
// only in a symmetric graph, hence the precondition (CC_FLAG_NO_SKIP falls back
// to the in-place link).
__device__ __forceinline__ uint32_t cid_of(uint2 w, uint32_t r)
{
    return w.y + __popc(w.x & ((1u << (r & 31)) - 1u));
}

// Forest record for C-space hooks: the hooked compact root c is the F0 root
// rid[c] in vertex space, never hooked in round 0, so its F slot is free.
struct ForestC {
    uint2* F;
    const uint32_t* rid;
    uint32_t u, v;
    __device__ __forceinline__ void record(uint32_t c, uint32_t, uint32_t) const { F[rid[c]] = make_uint2(u, v); }
};

template <int MODE, bool SF>
__global__ void __launch_bounds__(kBlock) k_link_contract(
    const uint32_t* __restrict__ P, const uint2* __restrict__ pend, const Ctl* ctl, const uint2* __restrict__ rbw,
    uint32_t* C, const uint32_t* __restrict__ rid, uint2* F, cc_counters* cnt)
{
    const unsigned long long total = ctl->pend_count;
    const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    Stat st;
    for (unsigned long long base = 0; base < total; base += nthreads * kLB) {
        uint2 pr[kLB];
        uint32_t ru[kLB], rv[kLB], cu[kLB], cv[kLB], pu[kLB], pv[kLB];
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
            const unsigned long long i = base + q * nthreads + tid;
            pr[q] = i < total ? pend[i] : make_uint2(0u, 0u);
        }
        // P is read-only in this kernel (the hooks go to C): read-only loads
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
            ru[q] = __ldg(P + pr[q].x);
            rv[q] = __ldg(P + pr[q].y);
        }
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
            if (ru[q] != rv[q]) {
                cu[q] = cid_of(__ldg(rbw + (ru[q] >> 5)), ru[q]);
                cv[q] = cid_of(__ldg(rbw + (rv[q] >> 5)), rv[q]);
            } else {
                cu[q] = cv[q] = 0u;
            }
        }
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
            pu[q] = ru[q] != rv[q] ? ld_relaxed(C + cu[q]) : 0u;
            pv[q] = ru[q] != rv[q] ? ld_relaxed(C + cv[q]) : 0u;
        }
        uint32_t hooked = 0;
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
            if (pu[q] == pv[q]) continue;
            if constexpr (MODE == 2) {
                if constexpr (SF) hooked += link_async(C, cu[q], cv[q], ForestC{F, rid, pr[q].x, pr[q].y});
                else hooked += link_async(C, cu[q], cv[q], NoForest{});
            } else {
                if constexpr (SF)
                    hooked += link_rem_from<MODE == 1>(C, cu[q], cv[q], pu[q], pv[q], ForestC{F, rid, pr[q].x, pr[q].y},
                                                       cnt ? &st : nullptr);
                else hooked += link_rem_from<MODE == 1>(C, cu[q], cv[q], pu[q], pv[q], NoForest{}, cnt ? &st : nullptr);
            }
        }
        __syncwarp();
        if (cnt) warp_count(&cnt->sample_hooks, hooked);
    }
    if (cnt) {
        warp_count(&cnt->link_steps, st.steps);
        warp_count(&cnt->cas_failures, st.fails);
    }
}

// After the links: rid[c] <- rid[root_C(c)], the vertex id of c's sampled
// component root.  Safe in place: a C root's rid slot is never rewritten (its
// root is itself) and only root slots are read through rid here.
__global__ void __launch_bounds__(kBlock) k_contract_final(const uint32_t* C, uint32_t* rid, const int64_t* Rtot)
{
    const uint64_t R = (uint64_t)*Rtot;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < R; c += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = C[c];
        if (p == (uint32_t)c) continue;
        rid[c] = rid[root_plain(C, p)];
    }
}

// The sampled label of a vertex whose F0 root (P[u] after the F0 compress) is r.
__device__ __forceinline__ uint32_t expand_root(const uint2* rbw, const uint32_t* rid, uint32_t r)
{
    const uint2 w = rbw[r >> 5];
    return (w.x >> (r & 31) & 1u) ? rid[cid_of(w, r)] : r;
}

// sampled_out debug path: P[u] <- expand(P[u]) for every u
__global__ void __launch_bounds__(kBlock) k_expand(uint32_t* P, uint32_t n, const uint2* rbw, const uint32_t* rid)
{
    const uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) P[v] = expand_root(rbw, rid, P[v]);
}

// per-block root counts of the rank words (kFTile words per block)
__global__ void __launch_bounds__(kBlock) k_rank_count(const uint2* __restrict__ rbw, uint32_t nw, uint32_t* bcnt)
{
    uint32_t tot;
    const uint64_t base = (uint64_t)blockIdx.x * kFTile + (uint64_t)threadIdx.x * kFItems;
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < kFItems; ++j)
        if (base + j < nw) c += __popc(rbw[base + j].x);
    block_excl_scan(c, &tot);
    if (threadIdx.x == 0) bcnt[blockIdx.x] = tot;
}

// per-word exclusive prefix, rid[] and C[c] = c.  The block's kFTile words are
// taken kBlock at a time (one per thread, coalesced), so each round's rid / C
// writes form one contiguous range.
__global__ void __launch_bounds__(kBlock) k_rank_fill(uint2* rbw, uint32_t nw, const unsigned long long* boff,
                                                      uint32_t* rid, uint32_t* C)
{
    uint32_t tot;
    uint32_t run = (uint32_t)boff[blockIdx.x];
    const uint64_t base = (uint64_t)blockIdx.x * kFTile;
    for (int j = 0; j < kFItems; ++j) {
        const uint64_t i = base + (uint64_t)j * kBlock + threadIdx.x;
        const uint32_t bits = i < nw ? rbw[i].x : 0u;
        uint32_t pref = run + block_excl_scan(__popc(bits), &tot);
        if (i < nw) rbw[i].y = pref;
        for (uint32_t b = bits; b; b &= b - 1) {
            rid[pref] = (uint32_t)(i * 32 + (uint32_t)(__ffs(b) - 1));
            C[pref] = pref;
            ++pref;
        }
        run += tot;
    }
}

// Grid of the static k-out link kernel.  CC_REFILL_GRID blocks per SM, 0 (default)
// = exactly one resident wave (6 blocks per SM).  With L1-cached Rem reads and PDL
// launches the one-wave grid measured fastest: C4 link 1.93 -> 1.70 ms, C3 0.285 ->
// 0.24 ms, C2 0.374 -> 0.30 ms (8 per SM = 1.33 waves had been faster with the
// round-1 L2-only reads).
#ifndef CC_REFILL_GRID
#define CC_REFILL_GRID 0
#endif
template <bool SF>
static unsigned refill_grid()
{
    return CC_REFILL_GRID ? grid_blocks(CC_REFILL_GRID) : resident_grid(k_link_refill<SF>, kBlock);
}

// ---------------------------------------------------------------------------
// K4: IdentifyFrequent: the mode of root(s_i) over S samples,
// s_i = uniform_below(mix(seed, IDENT, i), n), ties to the smaller label
// (reading R9).  One CTA: each thread finds the roots of its samples and
// counts them in a shared-memory open-addressing table (CAS on the key,
// atomicAdd on the count), then a max-reduction of (count, -label).
constexpr int kIdTable = 4096;                       // 2 * max samples (2048)

__global__ void __launch_bounds__(1024) k_identify(uint32_t* P, uint32_t n, uint64_t seed,
                                                   uint32_t samples, const uint32_t* force, Ctl* ctl,
                                                   uint32_t* lmax_out, const uint2* rbw, const uint32_t* rid)
{
    pdl_trigger();
    pdl_wait();
    __shared__ uint32_t keys[kIdTable];
    __shared__ uint32_t cnts[kIdTable];
    __shared__ unsigned long long best[32];
    const int t = threadIdx.x;
    if (force) {
        if (t == 0) {
            ctl->lmax = *force;
            if (lmax_out) *lmax_out = *force;
        }
        return;
    }
    for (int i = t; i < kIdTable; i += blockDim.x) {
        keys[i] = kSentinel;                         // labels are < n <= 0xFFFFFFFE
        cnts[i] = 0;
    }
    __syncthreads();
    for (int i = t; i < (int)samples; i += blockDim.x) {
        const uint32_t sv = uniform_below(mix(seed, IDENT_STREAM, (uint64_t)i), n);
        // no hook runs concurrently; contracted: P[sv] is sv's F0 root
        const uint32_t lab = rbw ? expand_root(rbw, rid, P[sv]) : root_halve(P, sv);
        uint32_t h = (lab * 0x9E3779B1u) >> 20;      // 12-bit multiplicative hash
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
            ctl->lmax = lm;
            if (lmax_out) *lmax_out = lm;
        }
    }
}

// ---------------------------------------------------------------------------
// K5: the finish fused with the sampling compress (H3).
//
// One coalesced pass over P (2 x uint4 per thread, like k_compress): every
// slot is compressed to its root r (H3, Def. 3.1's height-one labelling), and
// a vertex whose bitmap bit is set (its list was not wholly sampled) and whose
// root is not L_max becomes a finish candidate (reading R10: r == L_max proves
// v connected to L_max; every edge (v, y) out of a skipped v is either inside
// L_max's component or applied from y, which is then not skipped,
// P:2090-2100).  No hook runs in this kernel -- the candidates' edges are
// unioned by k_finish_proc afterwards -- so the compress is race-free, L_max
// (a root of the sampled forest) stays a root throughout, and a slot pointing
// at L_max needs no gather at all (the giant's ~46 % of the vertices on C4).
//
// Candidates are appended (warp-aggregated) to a queue that k_finish_proc
// degree-bins: lists (after the afforest-sampled prefix) of <= kSmallDeg
// entries are walked by their own lane, lists up to kBigDeg by the whole warp
// (ballot/shuffle; an edge whose endpoint already hangs directly under u's
// root is skipped without a link), longer lists are queued for k_finish_big
// (one CTA per vertex).  Keeping the edge work out of the scan keeps the scan
// a lean streaming kernel (no spills, full occupancy).
//
// Warp summaries for the partial final compress (k_relabel): after this pass
// every slot holds its sampled root, and the only labels H5 can change are
// those of slots whose root it hooks.  Each warp records, for its 256 slots,
// its "foreign" root -- a root other than the slot itself and L_max -- in one
// word: kSentinel none, r the only one, kWarpOverflow two or more distinct (ids
// are < n <= 0xFFFFFFFE, so 0xFFFFFFFE is never a root).  Warp-level only (no
// block barrier: the scan keeps fire-and-forget blocks).  Each block clears the
// hook flag of its 2048-slot tile (set by H5 when it hooks a root of the tile).
constexpr uint32_t kWarpOverflow = 0xFFFFFFFEu;
constexpr int kSumPerTile = kBlock / 32;                 // warp summaries per tile

__device__ __forceinline__ uint32_t warp_foreign_summary(const uint32_t (&rr)[kCV], uint32_t fmask)
{
    // fmask: bit s set iff slot s of this lane holds a foreign root
    const unsigned m1 = __ballot_sync(0xffffffffu, fmask != 0);
    if (!m1) return kSentinel;
    const int src = __ffs(m1) - 1;
    uint32_t x = kSentinel;                              // the lane's first foreign root (static indexing)
#pragma unroll
    for (int s = kCV - 1; s >= 0; --s)
        if (fmask >> s & 1u) x = rr[s];
    const uint32_t a = __shfl_sync(0xffffffffu, x, src);
    bool more = false;
#pragma unroll
    for (int s = 0; s < kCV; ++s) more |= (fmask >> s & 1u) && rr[s] != a;
    return __any_sync(0xffffffffu, more) ? kWarpOverflow : a;
}

// One tile of the scan, with its P words (pp) and bitmap words already loaded.
template <bool CNT, bool CONTRACT>
__device__ __forceinline__ void finish_tile(uint32_t* P, uint32_t n, uint64_t tile, bool full, uint32_t (&pp)[kCV],
                                            uint32_t w0, uint32_t w1, uint32_t lmax, uint32_t known, Ctl* ctl,
                                            uint32_t* cq,
                                            const uint2* __restrict__ rbw, const uint32_t* __restrict__ rid,
                                            uint32_t* __restrict__ wsum, uint8_t* __restrict__ td, uint32_t& writes,
                                            uint32_t& gathers)
{
    const uint64_t base = tile * kCTile;
    const uint64_t i0 = base + 4 * (uint64_t)threadIdx.x, i1 = i0 + 4 * kBlock;
    uint32_t vv[kCV], rr[kCV];
#pragma unroll
    for (int s = 0; s < kCV; ++s) vv[s] = (uint32_t)((s < 4 ? i0 : i1) + (s & 3));
    if constexpr (CONTRACT) {
        // P[v] is v's F0 root: its sampled root is one rank-word + one rid
        // lookup (L2-resident), no gather into P
        uint2 w[kCV];
#pragma unroll
        for (int s = 0; s < kCV; ++s) w[s] = (uint64_t)((s < 4 ? i0 : i1) + (s & 3)) < n ? rbw[pp[s] >> 5] : make_uint2(0u, 0u);
#pragma unroll
        for (int s = 0; s < kCV; ++s) {
            const bool cr = (w[s].x >> (pp[s] & 31)) & 1u;
            rr[s] = cr ? rid[cid_of(w[s], pp[s])] : pp[s];
            if (CNT) gathers += cr;
        }
    } else {
        const uint32_t g = roots8(P, vv, pp, rr, known);    // L_max stays a root: no hook runs here
        if (CNT) gathers += g;
    }
    if (CNT) {
#pragma unroll
        for (int s = 0; s < kCV; ++s) writes += rr[s] != pp[s];
    }
    if (full) {                                          // H3 compress writes
        if (rr[0] != pp[0] || rr[1] != pp[1] || rr[2] != pp[2] || rr[3] != pp[3])
            reinterpret_cast<uint4*>(P)[i0 >> 2] = make_uint4(rr[0], rr[1], rr[2], rr[3]);
        if (rr[4] != pp[4] || rr[5] != pp[5] || rr[6] != pp[6] || rr[7] != pp[7])
            reinterpret_cast<uint4*>(P)[i1 >> 2] = make_uint4(rr[4], rr[5], rr[6], rr[7]);
    } else {
#pragma unroll
        for (int s = 0; s < kCV; ++s)
            if (rr[s] != pp[s]) P[vv[s]] = rr[s];           // rr != pp only for in-range slots
    }
    uint32_t cm = 0, fmask = 0;                          // candidate / foreign-root slots of this thread
#pragma unroll
    for (int s = 0; s < kCV; ++s) {
        const uint64_t v64 = (s < 4 ? i0 : i1) + (s & 3);
        const uint32_t word = s < 4 ? w0 : w1;
        if (v64 < n && ((word >> (vv[s] & 31)) & 1u) && rr[s] != lmax) cm |= 1u << s;
        if (v64 < n && rr[s] != vv[s] && rr[s] != lmax) fmask |= 1u << s;
    }
    // warp summary of the foreign roots (rare outside grids)
#ifndef CC_FINISH_NOSUM
    const uint32_t ws = warp_foreign_summary(rr, fmask);
#else
    const uint32_t ws = kWarpOverflow;
#endif
    if ((threadIdx.x & 31) == 0) wsum[tile * kSumPerTile + (threadIdx.x >> 5)] = ws;
    if (threadIdx.x == 0) td[tile] = 0;
    if (__any_sync(0xffffffffu, cm != 0)) {
        const unsigned long long pos = warp_append(&ctl->cand_count, __popc(cm));
        uint32_t k2 = 0;
#pragma unroll
        for (int s = 0; s < kCV; ++s)
            if (cm >> s & 1u) cq[pos + k2++] = vv[s];
    }
}

__device__ __forceinline__ void finish_load(const uint32_t* P, const uint32_t* __restrict__ bm, uint32_t n,
                                            uint64_t tile, bool full, uint32_t (&pp)[kCV], uint32_t& w0, uint32_t& w1)
{
    const uint64_t base = tile * kCTile;
    const uint64_t i0 = base + 4 * (uint64_t)threadIdx.x, i1 = i0 + 4 * kBlock;
    if (full) {
        const uint4 a = reinterpret_cast<const uint4*>(P)[i0 >> 2];
        const uint4 c = reinterpret_cast<const uint4*>(P)[i1 >> 2];
        pp[0] = a.x; pp[1] = a.y; pp[2] = a.z; pp[3] = a.w;
        pp[4] = c.x; pp[5] = c.y; pp[6] = c.z; pp[7] = c.w;
    } else {
#pragma unroll
        for (int s = 0; s < kCV; ++s) {
            const uint64_t v = (s < 4 ? i0 : i1) + (s & 3);
            pp[s] = v < n ? P[v] : (uint32_t)v;
        }
    }
    w0 = i0 < n ? bm[i0 >> 5] : 0u;
    w1 = i1 < n ? bm[i1 >> 5] : 0u;
}

// One tile per block (65,536 blocks on C4): fire-and-forget blocks, 8 resident per SM.
template <bool VEC, bool CNT, bool CONTRACT>
__global__ void __launch_bounds__(kBlock, CC_FINISH_MINB) k_finish(uint32_t* P, const uint32_t* __restrict__ bm, uint32_t n,
                                                   Ctl* ctl, bool no_skip, uint32_t* cq, cc_counters* cnt,
                                                   const uint2* __restrict__ rbw, const uint32_t* __restrict__ rid,
                                                   uint32_t* __restrict__ wsum, uint8_t* __restrict__ td)
{
    pdl_trigger();
    pdl_wait();
    const uint32_t lmax = no_skip ? kSentinel : ctl->lmax;
    // L_max is a root of the sampled forest (IdentifyFrequent walks to roots), so a slot
    // holding it needs no gather -- unless a caller forced a non-root L_max (cc_opts.
    // lmax_force): then it is no shortcut, and since the slots' roots never equal it,
    // nothing is skipped (P stays height-one after this pass, as the SV / CRFA rounds need)
    const uint32_t known = lmax < n && ld_relaxed(P + lmax) == lmax ? lmax : kSentinel;
    const uint64_t tile = blockIdx.x;
    const bool full = VEC && (tile + 1) * kCTile <= n;
    uint32_t pp[kCV], w0, w1, writes = 0, gathers = 0;
    finish_load(P, bm, n, tile, full, pp, w0, w1);
    finish_tile<CNT, CONTRACT>(P, n, tile, full, pp, w0, w1, lmax, known, ctl, cq, rbw, rid, wsum, td, writes,
                               gathers);
    if (CNT) {
        warp_count(&cnt->compress_writes, writes);
        warp_count(&cnt->finish_gathers, gathers);
    }
}

// H5 hook record: besides the forest slot (SF), flag the tile of the hooked
// root for the partial final compress -- every label H5 changes is a slot of
// that root's component (the tiles holding its other slots name it among their
// foreign roots, see k_finish).
template <class F>
struct TileMarked {
    F f;
    uint8_t* td;
    __device__ __forceinline__ void record(uint32_t r, uint32_t u, uint32_t v) const
    {
        td[r / (uint32_t)kCTile] = 1;
        f.record(r, u, v);
    }
};

// k_finish_proc: the H5 edge work of the queued candidates.  A warp takes 32
// candidates, prefix-sums their list lengths (after the afforest-sampled
// prefix) and sweeps the concatenated lists 32 edges at a time, each lane
// finding its edge's owner by a binary search over the prefix (shuffles), so
// every lane has an independent link in flight whatever the degree mix; an
// edge whose endpoint already hangs directly under the owner's root is
// skipped without a link.  Lists longer than kBigDeg go to k_finish_big.  With
// few candidates (at most half as many as warps) several warps share each
// candidate's list instead (DESIGN.md §6 item 20).
template <int MODE, bool SF>
__global__ void __launch_bounds__(kBlock) k_finish_proc(
    const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, uint32_t* P,
    const uint32_t* __restrict__ cq, Ctl* ctl, uint32_t skip_prefix, uint32_t* big, unsigned long long big_cap,
    uint2* F, cc_counters* cnt, uint8_t* td)
{
    pdl_trigger();
    pdl_wait();
    const unsigned long long total = ctl->cand_count;
    const unsigned lane = threadIdx.x & 31;
    const unsigned long long warp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
#ifndef CC_FINISH_PROC_NOSPLIT
    if (total > 0 && 2 * total <= nwarps) {
        // Few candidates (the sampled regime: C4 253, C3 40): G >= 2 warps per candidate,
        // warp g of a candidate's group takes the list's 32-edge sweeps g, g + G, ... -- one
        // warp walking a list of hundreds of entries sweep after sweep was the kernel's
        // critical path (ncu on C3: SMs active 7 % of its 21.7 us)
        const unsigned long long G = nwarps / total;
        const unsigned long long c = warp / G, g = warp % G;
        if (c >= total) return;
        const uint32_t u = cq[c];
        int64_t b = off[u];
        const int64_t e = off[u + 1];
        b += min((int64_t)skip_prefix, e - b);
        const int64_t d = e - b;
        const bool isbig = d > kBigDeg;
        if (g == 0) {
            if (cnt && lane == 0) {
                atomicAdd((unsigned long long*)&cnt->finish_vertices, 1ull);
                atomicAdd((unsigned long long*)&cnt->finish_edges, (unsigned long long)d);
                if (isbig) atomicAdd((unsigned long long*)&cnt->big_vertices, 1ull);
            }
            if (isbig && lane == 0) {                    // the long lists keep their own kernel
                if (d > kHugeDeg) big[big_cap - 1 - atomicAdd(&ctl->huge_count, 1ull)] = u;
                else big[atomicAdd(&ctl->big_count, 1ull)] = u;
            }
        }
        if (isbig || d <= 0) return;
        const uint32_t ru = ld_relaxed(P + u);
        uint32_t hooks = 0;
        for (int64_t t = (int64_t)(g * 32 + lane); t < d; t += (int64_t)G * 32) {
            const uint32_t v = adj[b + t];
            const uint32_t pv = ld_link(P + v);
            if (pv == ru) continue;
            if constexpr (MODE == 2) {
                if constexpr (SF) hooks += link_async(P, u, v, TileMarked<Forest>{Forest{F}, td});
                else hooks += link_async(P, u, v, TileMarked<NoForest>{NoForest{}, td});
            } else {
                if constexpr (SF) hooks += link_rem_from<MODE == 1>(P, u, v, ru, pv, TileMarked<Forest>{Forest{F}, td});
                else hooks += link_rem_from<MODE == 1>(P, u, v, ru, pv, TileMarked<NoForest>{NoForest{}, td});
            }
        }
        if (cnt) warp_count(&cnt->finish_hooks, hooks);
        return;
    }
#endif
    // candidates per warp: 32 when there is plenty of work, fewer when the queue
    // is short so that every warp gets some (short queues are latency-bound)
    const unsigned cpw = (unsigned)max(1ull, min(32ull, (total + nwarps - 1) / nwarps));
    for (unsigned long long base = warp * cpw; base < total; base += nwarps * cpw) {
        const unsigned long long i = base + lane;
        const bool cand = lane < cpw && i < total;
        const uint32_t u = cand ? cq[i] : 0u;
        int64_t b = 0, e = 0;
        if (cand) {
            b = off[u];
            e = off[u + 1];
            b += min((int64_t)skip_prefix, e - b);     // afforest: the first k edges were unioned
        }
        const int64_t d = e - b;
        const bool isbig = d > kBigDeg;
        // u's parent: the root k_finish compressed u to (or a newer ancestor) --
        // as good as a full FIND for the "v already under u's root" early exit
        const uint32_t ru = cand && !isbig && d > 0 ? ld_relaxed(P + u) : 0u;
        if (cnt) {
            warp_count(&cnt->finish_vertices, cand ? 1u : 0u);
            warp_count(&cnt->finish_edges, cand ? (uint32_t)min(d, (int64_t)0xFFFFFFFF) : 0u);
            warp_count(&cnt->big_vertices, isbig ? 1u : 0u);
        }
        const bool ishuge = isbig && d > kHugeDeg;
        const unsigned long long bpos = warp_append(&ctl->big_count, isbig && !ishuge ? 1u : 0u);
        const unsigned long long hpos = warp_append(&ctl->huge_count, ishuge ? 1u : 0u);
        if (isbig && !ishuge) big[bpos] = u;
        if (ishuge) big[big_cap - 1 - hpos] = u;
        const uint32_t dd = isbig ? 0u : (uint32_t)d;   // <= kBigDeg
        uint32_t incl = dd;                             // inclusive prefix of list lengths
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (unsigned)o) incl += t;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - dd;
        uint32_t hooks = 0;
        for (uint32_t t0 = 0; t0 < tot; t0 += 32) {
            const uint32_t t = t0 + lane;
            // owner = the last lane whose exclusive prefix is <= t
            int lo = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t pe = __shfl_sync(0xffffffffu, excl, lo + step);
                if (pe <= t) lo += step;
            }
            const uint32_t ou = __shfl_sync(0xffffffffu, u, lo);
            const uint32_t orr = __shfl_sync(0xffffffffu, ru, lo);
            const int64_t ob = __shfl_sync(0xffffffffu, b, lo);
            const uint32_t oex = __shfl_sync(0xffffffffu, excl, lo);
            if (t < tot) {
                const uint32_t v = adj[ob + (t - oex)];
                const uint32_t pv = ld_link(P + v);
                if (pv != orr) {                            // enter the Rem loop with both reads done
                    if constexpr (MODE == 2) {
                        if constexpr (SF) hooks += link_async(P, ou, v, TileMarked<Forest>{Forest{F}, td});
                        else hooks += link_async(P, ou, v, TileMarked<NoForest>{NoForest{}, td});
                    } else {
                        if constexpr (SF)
                            hooks += link_rem_from<MODE == 1>(P, ou, v, orr, pv, TileMarked<Forest>{Forest{F}, td});
                        else hooks += link_rem_from<MODE == 1>(P, ou, v, orr, pv, TileMarked<NoForest>{NoForest{}, td});
                    }
                }
            }
            __syncwarp();
        }
        if (cnt) warp_count(&cnt->finish_hooks, hooks);
    }
}

// The long lists (> kBigDeg entries): one CTA per list (grid-strided over the
// queue); a list longer than kHugeDeg is instead shared by every CTA (each CTA
// walks the queue and takes a grid-strided slice of each huge list), so one hub
// of millions of entries does not serialise on one CTA.
template <int MODE, bool SF>
__global__ void __launch_bounds__(512) k_finish_big(const int64_t* __restrict__ off,
                                                    const uint32_t* __restrict__ adj, uint32_t* P,
                                                    const uint32_t* __restrict__ big, unsigned long long big_cap,
                                                    const Ctl* ctl, uint32_t skip_prefix, uint2* F, cc_counters* cnt,
                                                    uint8_t* td)
{
    pdl_trigger();
    pdl_wait();
    __shared__ uint32_t s_ru;
    const unsigned long long nbig = ctl->big_count, nhuge = ctl->huge_count;
    uint32_t hooks = 0;
    for (int pass = 0; pass < 2; ++pass) {
        // pass 0: the big lists, one CTA each; pass 1: the huge lists (queue tail), all CTAs
        const unsigned long long i0 = pass == 0 ? blockIdx.x : big_cap - nhuge;
        const unsigned long long i1 = pass == 0 ? nbig : big_cap;
        const unsigned long long di = pass == 0 ? gridDim.x : 1;
        for (unsigned long long i = i0; i < i1; i += di) {
            const uint32_t u = big[i];
            int64_t b = off[u];
            const int64_t e = off[u + 1];
            b += min((int64_t)skip_prefix, e - b);
            __syncthreads();
            if (threadIdx.x == 0) s_ru = find_naive(P, u);
            __syncthreads();
            const uint32_t ru = s_ru;
            const int64_t x0 = b + (pass == 1 ? (int64_t)blockIdx.x * blockDim.x : 0) + threadIdx.x;
            const int64_t step = pass == 1 ? (int64_t)gridDim.x * blockDim.x : (int64_t)blockDim.x;
            for (int64_t x = x0; x < e; x += step) {
                const uint32_t v = adj[x];
                if (ld_link(P + v) == ru) continue;          // equal: v already in u's set (R5)
                if constexpr (SF) hooks += link<MODE>(P, u, v, TileMarked<Forest>{Forest{F}, td});
                else hooks += link<MODE>(P, u, v, TileMarked<NoForest>{NoForest{}, td});
            }
        }
    }
    if (cnt) warp_count(&cnt->finish_hooks, hooks);
}

// ---------------------------------------------------------------------------
// K6': the final compress (H6) as a PARTIAL pass.  After k_finish every slot
// holds its sampled root, and H5 changes the label of exactly the slots whose
// root it hooked: the slots of a tile whose hook flag H5 set (the hooked root
// itself lies there) and of every tile that lists a hooked root among its
// foreign roots -- or, if L_max itself was hooked, every slot of its component
// (then every tile is re-resolved).  A tile with two distinct foreign
// roots in one of its 256-slot warp summaries is always re-resolved.  Each warp
// owns a run of consecutive tiles: one lane per tile decides (flag, 32 bytes of
// warp summaries, a P[r] == r test per named root),
// then the whole warp re-resolves each dirty tile (coalesced 16-byte loads,
// first-level parents batched as in k_compress, writes only changed slots).
// The result equals the full compress: every other slot already holds its
// final root (the canonical min-id label, reading R13).
// Re-resolve slots [base, base + 4 * 32 * Q) (Q uint4 per lane) of a tile-aligned chunk.
template <bool CNT, int Q>
__device__ __forceinline__ void relabel_span(uint32_t* P, uint32_t n, uint64_t base, bool vec, uint32_t known,
                                             uint32_t& writes, uint32_t& gathers)
{
    const unsigned lane = threadIdx.x & 31;
    const uint64_t span = 128ull * Q;
    if (vec && base + span <= n) {
#pragma unroll 1
        for (int j = 0; j < Q; j += 4) {
            uint4 q[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) q[h] = reinterpret_cast<const uint4*>(P)[base / 4 + lane + 32 * (j + h)];
#pragma unroll
            for (int h = 0; h < 4; h += 2) {
                const uint64_t i0 = base + 4 * (lane + 32 * (uint64_t)(j + h)), i1 = i0 + 128;
                const uint32_t pp[8] = {q[h].x, q[h].y, q[h].z, q[h].w, q[h + 1].x, q[h + 1].y, q[h + 1].z, q[h + 1].w};
                uint32_t vv[8], rr[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) vv[k] = (uint32_t)((k < 4 ? i0 : i1) + (k & 3));
                const uint32_t g = roots8(P, vv, pp, rr, known);
                const uint4 r0 = make_uint4(rr[0], rr[1], rr[2], rr[3]);
                const uint4 r1 = make_uint4(rr[4], rr[5], rr[6], rr[7]);
                const uint32_t c0 = nchanged4(r0, q[h]), c1 = nchanged4(r1, q[h + 1]);
                if (c0) reinterpret_cast<uint4*>(P)[i0 >> 2] = r0;
                if (c1) reinterpret_cast<uint4*>(P)[i1 >> 2] = r1;
                if (CNT) {
                    gathers += g;
                    writes += c0 + c1;
                }
            }
        }
    } else {
        const uint64_t end = (base + span < n ? base + span : (uint64_t)n);
        for (uint64_t v64 = base + lane; v64 < end; v64 += 32) {
            const uint32_t v = (uint32_t)v64;
            const uint32_t p = P[v];
            const bool g = !(p == v || p == known);
            const uint32_t r = g ? root_halve(P, p) : p;
            if (r != p) P[v] = r;
            if (CNT) {
                gathers += g;
                writes += r != p;
            }
        }
    }
}

constexpr int kRlChunk = 512;                            // slots per queued relabel chunk
constexpr int kRlPerTile = kCTile / kRlChunk;

// Two kernels (the kernel boundary is the barrier; PDL overlaps the launch):
// k_relabel_decide -- each warp decides its run of tiles (hook flag, 32 bytes of warp
// summaries, a P[r] == r test per named root) and queues the dirty ones as 512-slot
// chunks (in the candidate queue, free after H5); k_relabel -- every warp takes queued
// chunks, so a few hundred dirty tiles are spread over all warps instead of being
// walked by the few warps that own them.  If L_max was hooked, the decide kernel
// queues nothing and k_relabel re-resolves every chunk grid-strided.
template <bool CNT>
__global__ void __launch_bounds__(kBlock) k_relabel_decide(const uint32_t* P, uint32_t n, Ctl* ctl, bool no_skip,
                                                           const uint32_t* __restrict__ wsum,
                                                           const uint8_t* __restrict__ td, uint32_t* queue,
                                                           cc_counters* cnt)
{
    pdl_trigger();
    pdl_wait();
    const unsigned lane = threadIdx.x & 31;
    uint32_t lm = no_skip ? kSentinel : ctl->lmax;
    if (lm >= n) lm = kSentinel;                                      // a forced out-of-range L_max skips nothing
    // L_max no longer a root: H5 hooked it, or a forced L_max was never one -- in
    // both cases slots holding it are not final, so every tile is re-resolved
    if (lm != kSentinel && P[lm] != lm) return;                       // no hook runs in H6: plain loads
    const uint64_t ntiles = ((uint64_t)n + kCTile - 1) / kCTile;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t tpw = (ntiles + nwarps - 1) / nwarps < 32 ? (ntiles + nwarps - 1) / nwarps : (uint64_t)32;
    uint32_t tiles = 0;
    for (uint64_t t0 = warp * tpw; t0 < ntiles; t0 += nwarps * tpw) {
        const uint64_t t = t0 + lane;
        bool dirty = false;
        if (lane < tpw && t < ntiles) {
            if (td[t]) {
                dirty = true;
            } else {
                // the tile's kSumPerTile warp summaries (32 contiguous bytes)
                const uint4* w4 = reinterpret_cast<const uint4*>(wsum + t * kSumPerTile);
                const uint4 q0 = w4[0], q1 = w4[1];
                const uint32_t r8[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    dirty |= r8[c] == kWarpOverflow || (r8[c] != kSentinel && P[r8[c]] != r8[c]);
            }
        }
        if (CNT) tiles += dirty;
        const unsigned long long pos = warp_append(&ctl->rl_count, dirty ? (uint32_t)kRlPerTile : 0u);
        if (dirty)
            for (int c = 0; c < kRlPerTile; ++c) queue[pos + c] = (uint32_t)(t * kRlPerTile + c);
    }
    if (CNT) warp_count(&cnt->h6_tiles, tiles);
}

template <bool CNT>
__global__ void __launch_bounds__(kBlock) k_relabel(uint32_t* P, uint32_t n, const Ctl* ctl, bool no_skip,
                                                    const uint32_t* __restrict__ queue, cc_counters* cnt)
{
    pdl_trigger();
    pdl_wait();
    uint32_t lm = no_skip ? kSentinel : ctl->lmax;
    if (lm >= n) lm = kSentinel;
    const bool lmax_hooked = lm != kSentinel && P[lm] != lm;
    const uint32_t known = lmax_hooked ? kSentinel : lm;
    const uint64_t ntiles = ((uint64_t)n + kCTile - 1) / kCTile;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const bool vec = ((uintptr_t)P & 15u) == 0;
    uint32_t writes = 0, gathers = 0;
    if (lmax_hooked) {
        for (uint64_t c = warp; c < ntiles * kRlPerTile; c += nwarps)
            relabel_span<CNT, kRlChunk / 128>(P, n, c * kRlChunk, vec, known, writes, gathers);
        if (CNT && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt->h6_tiles),
                                                                  (unsigned long long)ntiles);
    } else {
        const unsigned long long total = ctl->rl_count;
        for (unsigned long long idx = warp; idx < total; idx += nwarps)
            relabel_span<CNT, kRlChunk / 128>(P, n, (uint64_t)queue[idx] * kRlChunk, vec, known, writes, gathers);
    }
    if (CNT) {
        warp_count(&cnt->h6_writes, writes);
        warp_count(&cnt->h6_gathers, gathers);
    }
}

// ---------------------------------------------------------------------------
// NEXT-3: Shiloach-Vishkin as the finish method (Alg. shiloach_vishkin,
// P:4282-4308; SV hooks only roots, so it composes with sampling
// and the L_max skip).  The finish candidates' edges (after the
// sampled prefix) are materialised once; then each round hooks, for every edge
// whose endpoints' labels differ, the larger label h -- if h was a root at the
// start of the round (prev_labels[h] == h, kept as a bitmap) -- under the
// smaller one with writeMin (atomicMin), then fully shortcuts.
// Rounds repeat until no edge hooks.  The host reads a flag after each round
// (one synchronisation per round), so this finish is an option, not the
// default.  In SF mode a second pass per round records, for every hooked
// root h, an edge whose writeMin value won (P[h] == l after the round).
__global__ void __launch_bounds__(kBlock) k_sv_degree(const int64_t* __restrict__ off, const uint32_t* __restrict__ cq,
                                                      const Ctl* ctl, uint32_t skip_prefix, uint32_t* deg)
{
    const unsigned long long total = ctl->cand_count;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const uint32_t u = cq[i];
        const int64_t d = off[u + 1] - off[u] - (int64_t)skip_prefix;
        deg[i] = d > 0 ? (uint32_t)min(d, (int64_t)0xFFFFFFFF) : 0u;
    }
}

// per-block sums of deg[] (kFTile entries per block, 64-bit)
__global__ void __launch_bounds__(kBlock) k_sv_blocksum(const uint32_t* deg, unsigned long long total,
                                                        unsigned long long* bsum)
{
    const uint64_t base = (uint64_t)blockIdx.x * kFTile + (uint64_t)threadIdx.x * kFItems;
    unsigned long long c = 0;
#pragma unroll
    for (int j = 0; j < kFItems; ++j)
        if (base + j < total) c += deg[base + j];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __shared__ unsigned long long ws[kBlock / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < kBlock / 32; ++i) t += ws[i];
        bsum[blockIdx.x] = t;
    }
}

// single thread: exclusive scan of the block sums (few thousand entries)
__global__ void k_sv_scan(unsigned long long* bsum, unsigned long long nb, unsigned long long* total_edges)
{
    unsigned long long acc = 0;
    for (unsigned long long i = 0; i < nb; ++i) {
        const unsigned long long t = bsum[i];
        bsum[i] = acc;
        acc += t;
    }
    *total_edges = acc;
}

// Each candidate's start in the flat edge list (exclusive prefix of deg[]: the
// block sums of k_sv_blocksum, scanned, plus a block-level scan).
__global__ void __launch_bounds__(kBlock) k_sv_starts(const uint32_t* __restrict__ deg,
                                                      const unsigned long long* __restrict__ bsum,
                                                      unsigned long long total, unsigned long long* __restrict__ start)
{
    const unsigned lane = threadIdx.x & 31;
    const uint64_t i = (uint64_t)blockIdx.x * kFTile + (uint64_t)threadIdx.x * kFItems;
    unsigned long long c = 0, pos[kFItems];
#pragma unroll
    for (int j = 0; j < kFItems; ++j) {
        pos[j] = c;
        c += (i + j < total) ? deg[i + j] : 0u;
    }
    unsigned long long incl = c;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += t;
    }
    __shared__ unsigned long long ws[kBlock / 32];
    if (lane == 31) ws[threadIdx.x >> 5] = incl;
    __syncthreads();
    unsigned long long wbase = 0;
    for (unsigned w = 0; w < (threadIdx.x >> 5); ++w) wbase += ws[w];
    const unsigned long long tbase = bsum[blockIdx.x] + wbase + incl - c;
#pragma unroll
    for (int j = 0; j < kFItems; ++j)
        if (i + j < total) start[i + j] = tbase + pos[j];
}

// Edge-parallel copy of the candidates' lists: a warp takes 32 candidates and
// sweeps their concatenated lists 32 entries at a time (each lane finds its
// entry's owner by a binary search over the warp's exclusive prefix).  A list
// longer than kSvPiece entries contributes only its first piece there; its other
// pieces are queued (candidate, piece) and copied by k_sv_pieces, one warp per
// piece, so a hub's million-entry list is spread over many warps instead of
// serialising one (C4 at k = 0: 1.7M-entry hubs, 75 ms in one warp's loop).
// FILTER (every marked vertex is a candidate: no skip, or no sampling): an edge
// between two candidates is materialised from both ends, so keep (u, v) only
// when u < v or v is not a candidate -- half the edges, appended in any order.
constexpr int kSvBuf = 384;                 // WarpBuf entries per warp (3 KB of uint2)
constexpr uint32_t kSvPiece = 4096;         // entries per piece of a long list
#ifndef CC_SV_R
#define CC_SV_R 4
#endif
constexpr int kSvR = CC_SV_R;               // entries per lane per sweep of k_sv_copy

template <bool FILTER>
struct SvCopy {
    const uint32_t* adj;
    uint2* edges;
    const uint32_t* bm;
    uint32_t lmax;
    unsigned long long* kept;
    __device__ __forceinline__ bool keep_edge(uint32_t u, uint32_t v) const
    {
        const bool cand_v = ((bm[v >> 5] >> (v & 31)) & 1u) && v != lmax;
        return u < v || !cand_v;
    }
};

template <bool FILTER>
__global__ void __launch_bounds__(kBlock) k_sv_copy(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                    const uint32_t* __restrict__ cq, const uint32_t* __restrict__ deg,
                                                    const unsigned long long* __restrict__ start,
                                                    unsigned long long total, uint32_t skip_prefix, uint2* edges,
                                                    const uint32_t* __restrict__ bm, const Ctl* ctl, bool no_skip,
                                                    unsigned long long* kept, uint2* pieces, unsigned long long* npieces)
{
    const uint32_t lmax = no_skip ? kSentinel : ctl->lmax;
    const unsigned lane = threadIdx.x & 31;
    const unsigned long long warp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    __shared__ uint2 s_buf[FILTER ? kBlock / 32 : 1][FILTER ? kSvBuf : 1];
    WarpBuf<uint2, kSvBuf> wb{s_buf[FILTER ? threadIdx.x >> 5 : 0], 0u};
    const SvCopy<FILTER> sc{adj, edges, bm, lmax, kept};
    for (unsigned long long base = warp * 32; base < total; base += nwarps * 32) {
        const unsigned long long i = base + lane;
        const bool ok = i < total;
        const uint32_t u = ok ? cq[i] : 0u;
        const uint32_t dfull = ok ? deg[i] : 0u;
        const uint64_t d = min(dfull, kSvPiece);            // the first piece here, the rest queued
        const int64_t b = ok ? off[u] + (int64_t)skip_prefix : 0;
        const unsigned long long st = ok && !FILTER ? start[i] : 0ull;
        {
            const uint32_t np = dfull > kSvPiece ? (dfull - 1) / kSvPiece : 0u;   // pieces 1 .. np
            const unsigned long long pos = warp_append(npieces, np);
            for (uint32_t q = 0; q < np; ++q) pieces[pos + q] = make_uint2((uint32_t)i, (uint32_t)(i >> 32) | ((q + 1) << 8));
        }
        uint64_t incl = d;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (unsigned)o) incl += t;
        }
        const uint64_t tot = __shfl_sync(0xffffffffu, incl, 31);
        const uint64_t excl = incl - d;
        // kSvR entries per lane per sweep, their owner searches first and their loads together
        for (uint64_t t0 = 0; t0 < tot; t0 += 32 * kSvR) {
            uint32_t ou[kSvR], v[kSvR];
            int64_t src[kSvR];
            unsigned long long dst[kSvR];
#pragma unroll
            for (int r = 0; r < kSvR; ++r) {
                const uint64_t t = t0 + (uint64_t)r * 32 + lane;
                int lo = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const uint64_t pe = __shfl_sync(0xffffffffu, excl, lo + step);
                    if (pe <= t) lo += step;
                }
                ou[r] = __shfl_sync(0xffffffffu, u, lo);
                const int64_t ob = __shfl_sync(0xffffffffu, b, lo);
                const uint64_t oex = __shfl_sync(0xffffffffu, excl, lo);
                const unsigned long long ost = __shfl_sync(0xffffffffu, st, lo);
                src[r] = ob + (int64_t)(t - oex);
                dst[r] = ost + (t - oex);
            }
#pragma unroll
            for (int r = 0; r < kSvR; ++r) v[r] = t0 + (uint64_t)r * 32 + lane < tot ? adj[src[r]] : 0u;
#pragma unroll
            for (int r = 0; r < kSvR; ++r) {
                const bool in = t0 + (uint64_t)r * 32 + lane < tot;
                if constexpr (FILTER) {
                    wb.put(in && sc.keep_edge(ou[r], v[r]), make_uint2(ou[r], v[r]), kept, edges);
                } else {
                    (void)dst;
                    if (in) edges[dst[r]] = make_uint2(ou[r], v[r]);
                }
            }
        }
    }
    if constexpr (FILTER) wb.flush(kept, edges);
}

// The queued pieces of the long lists: one warp per piece (kSvPiece entries), 8
// entries per lane per sweep with their loads issued together.  A piece word is
// (candidate index low 32 bits, high 8 bits of it | piece number << 8).
template <bool FILTER>
__global__ void __launch_bounds__(kBlock) k_sv_pieces(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                      const uint32_t* __restrict__ cq, const uint32_t* __restrict__ deg,
                                                      const unsigned long long* __restrict__ start,
                                                      uint32_t skip_prefix, uint2* edges, const uint32_t* __restrict__ bm,
                                                      const Ctl* ctl, bool no_skip, unsigned long long* kept,
                                                      const uint2* __restrict__ pieces,
                                                      const unsigned long long* __restrict__ npieces)
{
    const uint32_t lmax = no_skip ? kSentinel : ctl->lmax;
    const unsigned lane = threadIdx.x & 31;
    const unsigned long long warp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    __shared__ uint2 s_buf[FILTER ? kBlock / 32 : 1][FILTER ? kSvBuf : 1];
    WarpBuf<uint2, kSvBuf> wb{s_buf[FILTER ? threadIdx.x >> 5 : 0], 0u};
    const SvCopy<FILTER> sc{adj, edges, bm, lmax, kept};
    const unsigned long long np = *npieces;
    constexpr int R = 8;
    for (unsigned long long pc = warp; pc < np; pc += nwarps) {
        const uint2 pw = pieces[pc];
        const unsigned long long i = (unsigned long long)pw.x | ((unsigned long long)(pw.y & 0xFFu) << 32);
        const uint32_t q = pw.y >> 8;
        const uint32_t u = cq[i];
        const uint64_t p0 = (uint64_t)q * kSvPiece;
        const uint64_t len = min((uint64_t)deg[i] - p0, (uint64_t)kSvPiece);
        const int64_t b = off[u] + (int64_t)skip_prefix + (int64_t)p0;
        const unsigned long long st = FILTER ? 0ull : start[i] + p0;
        for (uint64_t t0 = 0; t0 < len; t0 += 32 * R) {
            uint32_t v[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint64_t t = t0 + (uint64_t)r * 32 + lane;
                v[r] = t < len ? adj[b + (int64_t)t] : 0u;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint64_t t = t0 + (uint64_t)r * 32 + lane;
                if constexpr (FILTER) {
                    const bool keep = t < len && sc.keep_edge(u, v[r]);
                    wb.put(keep, make_uint2(u, v[r]), kept, edges);
                } else {
                    if (t < len) edges[st + t] = make_uint2(u, v[r]);
                }
            }
        }
    }
    if constexpr (FILTER) wb.flush(kept, edges);
}

__global__ void __launch_bounds__(kBlock) k_sv_rootbits(const uint32_t* P, uint32_t n, uint32_t* bits)
{
    const uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool root = v < n && P[v] == (uint32_t)v;
    const uint32_t w = __ballot_sync(0xffffffffu, root);
    if ((threadIdx.x & 31) == 0 && v < n) bits[v >> 5] = w;
}

// the label of x at the start of the round: x itself if x was a root then,
// else its parent (non-root slots are not written during a round)
__device__ __forceinline__ uint32_t sv_label(const uint32_t* P, const uint32_t* bits, uint32_t x)
{
    return ((bits[x >> 5] >> (x & 31)) & 1u) ? x : P[x];
}

__global__ void __launch_bounds__(kBlock) k_sv_hook(uint32_t* P, const uint2* __restrict__ edges,
                                                    unsigned long long ne, const uint32_t* __restrict__ bits,
                                                    unsigned int* changed)
{
    unsigned int ch = 0;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const uint2 e = edges[i];
        const uint32_t a = sv_label(P, bits, e.x), b = sv_label(P, bits, e.y);
        if (a == b) continue;
        const uint32_t h = max(a, b), l = min(a, b);     // h is a root of the round's start (a label)
        // writeMin, tested first: P[h] only decreases, so a value read at
        // or below l (even a stale one) means the writeMin would change nothing -- which
        // spares the hot roots' slots the serialised atomics of every edge that targets
        // them (C4 k = 0, round 3: 789M atomicMin on few addresses, 567 ms)
        if (ld_link(P + h) <= l) continue;
        ch |= atomicMin(P + h, l) > l ? 1u : 0u;
    }
    if (__any_sync(0xffffffffu, ch != 0) && (threadIdx.x & 31) == 0) atomicOr(changed, 1u);
}

__global__ void __launch_bounds__(kBlock) k_sv_record(const uint32_t* P, const uint2* __restrict__ edges,
                                                      unsigned long long ne, const uint32_t* __restrict__ bits, uint2* F)
{
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const uint2 e = edges[i];
        const uint32_t a = sv_label(P, bits, e.x), b = sv_label(P, bits, e.y);
        if (a == b) continue;
        const uint32_t h = max(a, b), l = min(a, b);
        if (P[h] == l) F[h] = e;                         // this edge's writeMin won at h
    }
}

// Liu-Tarjan CRFA (the framework of P:866-905 / P:4019-4048): each round
// Connect (the endpoints of an edge are candidates for each other), RootUp (only a
// vertex that is a root at the start of the round takes a candidate), FullShortcut,
// then Alter (every edge is replaced by the labels of its endpoints; edges that
// became self-loops are dropped, so the edge list shrinks round by round).  Every
// update is a writeMin.  Edges: uint4 (a, b, u, v) = current endpoints + the input
// edge (for the forest record); without SF only (a, b) is kept.
template <bool SF>
using LtEdge = typename std::conditional<SF, uint4, uint2>::type;

template <bool SF>
__global__ void __launch_bounds__(kBlock) k_lt_init(const uint2* __restrict__ e, unsigned long long ne, LtEdge<SF>* out)
{
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const uint2 x = e[i];
        if constexpr (SF) out[i] = make_uint4(x.x, x.y, x.x, x.y);
        else out[i] = x;
    }
}

template <bool SF>
__global__ void __launch_bounds__(kBlock) k_lt_connect(uint32_t* P, const LtEdge<SF>* __restrict__ e,
                                                       const unsigned long long* ne, const uint32_t* __restrict__ bits,
                                                       unsigned int* changed)
{
    unsigned int ch = 0;
    const unsigned long long total = *ne;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const LtEdge<SF> x = e[i];
        const uint32_t h = max(x.x, x.y), l = min(x.x, x.y);
        if (h == l || !((bits[h >> 5] >> (h & 31)) & 1u)) continue;     // RootUp: h a root at round start
        if (ld_link(P + h) <= l) continue;                                // the writeMin would not change P[h]
        ch |= atomicMin(P + h, l) > l ? 1u : 0u;                          // Connect, writeMin
    }
    if (__any_sync(0xffffffffu, ch != 0) && (threadIdx.x & 31) == 0) atomicOr(changed, 1u);
}

// SF: the edge whose candidate won at h (P[h] == l after the connect phase)
__global__ void __launch_bounds__(kBlock) k_lt_record(const uint32_t* P, const uint4* __restrict__ e,
                                                      const unsigned long long* ne, const uint32_t* __restrict__ bits,
                                                      uint2* F)
{
    const unsigned long long total = *ne;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const uint4 x = e[i];
        const uint32_t h = max(x.x, x.y), l = min(x.x, x.y);
        if (h == l || !((bits[h >> 5] >> (h & 31)) & 1u)) continue;
        if (P[h] == l) F[h] = make_uint2(x.z, x.w);
    }
}

// Alter after the FullShortcut (P[x] is x's root): keep (P[a], P[b]) unless equal
template <bool SF>
__global__ void __launch_bounds__(kBlock) k_lt_alter(const uint32_t* P, const LtEdge<SF>* __restrict__ e,
                                                     const unsigned long long* ne, LtEdge<SF>* out,
                                                     unsigned long long* ne_out)
{
    const unsigned long long total = *ne;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    constexpr int CAP = SF ? kSvBuf / 2 : kSvBuf;
    __shared__ LtEdge<SF> s_buf[kBlock / 32][CAP];
    WarpBuf<LtEdge<SF>, CAP> wb{s_buf[threadIdx.x >> 5], 0u};
    for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x; base < total; base += stride) {
        const unsigned long long i = base + threadIdx.x;
        LtEdge<SF> x{};
        bool keep = false;
        if (i < total) {
            x = e[i];
            x.x = P[x.x];
            x.y = P[x.y];
            keep = x.x != x.y;
        }
        wb.put(keep, x, ne_out, out);
    }
    wb.flush(ne_out, out);
}

template <bool SF>
static cc_status sv_finish(const int64_t* off, const uint32_t* adj, uint32_t* P, uint32_t n, const uint32_t* cq,
                           Ctl* ctl, uint32_t skip_prefix, uint2* F, cc_counters* cnt, cudaStream_t s,
                           bool crfa, const uint32_t* bm, bool no_skip, bool all_marked_candidates)
{
    void* le[2] = {nullptr, nullptr};
    unsigned long long* lcnt = nullptr;
    unsigned long long cand = 0;
    CC_CUDA_TRY(cudaMemcpyAsync(&cand, &ctl->cand_count, sizeof(cand), cudaMemcpyDeviceToHost, s));
    CC_CUDA_TRY(cudaStreamSynchronize(s));
    if (cand == 0) return CC_OK;
    const unsigned long long nbk = (cand + kFTile - 1) / kFTile;
    uint32_t *deg = nullptr, *bits = nullptr;
    unsigned long long *bsum = nullptr, *tot = nullptr, *starts = nullptr, *npieces = nullptr;
    uint2* edges = nullptr;
    uint2* pieces = nullptr;              // the long lists' pieces after the first (k_sv_pieces)
    unsigned int* changed = nullptr;
    cc_status rc = CC_OK;
    auto body = [&]() -> cc_status {
        CC_CUDA_TRY(scratch_alloc((void**)&deg, sizeof(uint32_t) * cand, s));
        CC_CUDA_TRY(scratch_alloc((void**)&bsum, sizeof(unsigned long long) * nbk, s));
        CC_CUDA_TRY(scratch_alloc((void**)&tot, sizeof(unsigned long long), s));
        k_sv_degree<<<grid_blocks(8), kBlock, 0, s>>>(off, cq, ctl, skip_prefix, deg);
        CC_LAUNCH_CHECK("k_sv_degree");
        k_sv_blocksum<<<(unsigned)nbk, kBlock, 0, s>>>(deg, cand, bsum);
        CC_LAUNCH_CHECK("k_sv_blocksum");
        k_sv_scan<<<1, 1, 0, s>>>(bsum, nbk, tot);
        CC_LAUNCH_CHECK("k_sv_scan");
        unsigned long long ne = 0;
        CC_CUDA_TRY(cudaMemcpyAsync(&ne, tot, sizeof(ne), cudaMemcpyDeviceToHost, s));
        CC_CUDA_TRY(cudaStreamSynchronize(s));
        if (ne == 0) return CC_OK;
        CC_CUDA_TRY(scratch_alloc((void**)&edges, sizeof(uint2) * ne, s));
        CC_CUDA_TRY(scratch_alloc((void**)&bits, sizeof(uint32_t) * (((uint64_t)n + 31) / 32), s));
        CC_CUDA_TRY(scratch_alloc((void**)&changed, sizeof(unsigned int), s));
        CC_CUDA_TRY(scratch_alloc((void**)&pieces, sizeof(uint2) * (ne / kSvPiece + 1), s));
        CC_CUDA_TRY(scratch_alloc((void**)&npieces, sizeof(unsigned long long), s));
        CC_CUDA_TRY(cudaMemsetAsync(npieces, 0, sizeof(unsigned long long), s));
        if (all_marked_candidates) {
            CC_CUDA_TRY(cudaMemsetAsync(tot, 0, sizeof(unsigned long long), s));
            k_sv_copy<true><<<grid_blocks(8), kBlock, 0, s>>>(off, adj, cq, deg, nullptr, cand, skip_prefix, edges,
                                                                bm, ctl, no_skip, tot, pieces, npieces);
            CC_LAUNCH_CHECK("k_sv_copy");
            k_sv_pieces<true><<<grid_blocks(8), kBlock, 0, s>>>(off, adj, cq, deg, nullptr, skip_prefix, edges, bm, ctl,
                                                                  no_skip, tot, pieces, npieces);
            CC_LAUNCH_CHECK("k_sv_pieces");
            CC_CUDA_TRY(cudaMemcpyAsync(&ne, tot, sizeof(ne), cudaMemcpyDeviceToHost, s));
            CC_CUDA_TRY(cudaStreamSynchronize(s));
            if (ne == 0) return CC_OK;
        } else {
            CC_CUDA_TRY(scratch_alloc((void**)&starts, sizeof(unsigned long long) * cand, s));
            k_sv_starts<<<(unsigned)nbk, kBlock, 0, s>>>(deg, bsum, cand, starts);
            CC_LAUNCH_CHECK("k_sv_starts");
            k_sv_copy<false><<<grid_blocks(8), kBlock, 0, s>>>(off, adj, cq, deg, starts, cand, skip_prefix, edges,
                                                                 nullptr, ctl, no_skip, nullptr, pieces, npieces);
            CC_LAUNCH_CHECK("k_sv_copy");
            k_sv_pieces<false><<<grid_blocks(8), kBlock, 0, s>>>(off, adj, cq, deg, starts, skip_prefix, edges, nullptr,
                                                                   ctl, no_skip, nullptr, pieces, npieces);
            CC_LAUNCH_CHECK("k_sv_pieces");
        }
        const unsigned nbv = (unsigned)(((uint64_t)n + kBlock - 1) / kBlock);
        if (crfa) {
            // Liu-Tarjan CRFA: rounds until Alter leaves no edge
            CC_CUDA_TRY(scratch_alloc((void**)&le[1], sizeof(LtEdge<SF>) * ne, s));
            CC_CUDA_TRY(scratch_alloc((void**)&lcnt, 2 * sizeof(unsigned long long), s));
            if constexpr (SF) {
                CC_CUDA_TRY(scratch_alloc((void**)&le[0], sizeof(LtEdge<SF>) * ne, s));
                k_lt_init<SF><<<grid_blocks(8), kBlock, 0, s>>>(edges, ne, (LtEdge<SF>*)le[0]);
                CC_LAUNCH_CHECK("k_lt_init");
            } else {                          // (a, b) = (u, v): the materialised list is round 1's
                le[0] = edges;
                edges = nullptr;
            }
            CC_CUDA_TRY(cudaMemcpyAsync(lcnt, &ne, sizeof(ne), cudaMemcpyHostToDevice, s));
            for (uint64_t round = 1;; ++round) {
                const int a = (round - 1) & 1;
                k_sv_rootbits<<<nbv, kBlock, 0, s>>>(P, n, bits);
                CC_LAUNCH_CHECK("k_sv_rootbits(LT)");
                CC_CUDA_TRY(cudaMemsetAsync(changed, 0, sizeof(unsigned int), s));
                k_lt_connect<SF><<<grid_blocks(8), kBlock, 0, s>>>(P, (const LtEdge<SF>*)le[a], lcnt + a, bits, changed);
                CC_LAUNCH_CHECK("k_lt_connect");
                if constexpr (SF) {
                    k_lt_record<<<grid_blocks(8), kBlock, 0, s>>>(P, (const uint4*)le[a], lcnt + a, bits, F);
                    CC_LAUNCH_CHECK("k_lt_record");
                }
                cc_status r = launch_compress(P, n, nullptr, nullptr, s, "k_compress(LT FullShortcut)");
                if (r) return r;
                CC_CUDA_TRY(cudaMemsetAsync(lcnt + (a ^ 1), 0, sizeof(unsigned long long), s));
                k_lt_alter<SF><<<grid_blocks(8), kBlock, 0, s>>>(P, (const LtEdge<SF>*)le[a], lcnt + a, (LtEdge<SF>*)le[a ^ 1],
                                                          lcnt + (a ^ 1));
                CC_LAUNCH_CHECK("k_lt_alter");
                unsigned long long left = 0;
                CC_CUDA_TRY(cudaMemcpyAsync(&left, lcnt + (a ^ 1), sizeof(left), cudaMemcpyDeviceToHost, s));
                CC_CUDA_TRY(cudaStreamSynchronize(s));
                if (cnt) CC_CUDA_TRY(cudaMemcpyAsync(&cnt->sv_rounds, &round, sizeof(round), cudaMemcpyHostToDevice, s));
                if (!left) break;
            }
            CC_CUDA_TRY(cudaStreamSynchronize(s));
            return CC_OK;
        }
        for (uint64_t round = 1;; ++round) {
            k_sv_rootbits<<<nbv, kBlock, 0, s>>>(P, n, bits);        // prev_labels[h] == h
            CC_LAUNCH_CHECK("k_sv_rootbits");
            CC_CUDA_TRY(cudaMemsetAsync(changed, 0, sizeof(unsigned int), s));
            k_sv_hook<<<grid_blocks(8), kBlock, 0, s>>>(P, edges, ne, bits, changed);
            CC_LAUNCH_CHECK("k_sv_hook");
            if (SF) {
                k_sv_record<<<grid_blocks(8), kBlock, 0, s>>>(P, edges, ne, bits, F);
                CC_LAUNCH_CHECK("k_sv_record");
            }
            unsigned int h_changed = 0;
            CC_CUDA_TRY(cudaMemcpyAsync(&h_changed, changed, sizeof(h_changed), cudaMemcpyDeviceToHost, s));
            CC_CUDA_TRY(cudaStreamSynchronize(s));
            if (cnt) CC_CUDA_TRY(cudaMemcpyAsync(&cnt->sv_rounds, &round, sizeof(round), cudaMemcpyHostToDevice, s));
            if (!h_changed) break;
            cc_status r = launch_compress(P, n, nullptr, nullptr, s, "k_compress(SV shortcut)");   // FullShortcut
            if (r) return r;
        }
        CC_CUDA_TRY(cudaStreamSynchronize(s));
        return CC_OK;
    };
    rc = body();
    scratch_free(deg, s);
    scratch_free(bsum, s);
    scratch_free(tot, s);
    scratch_free(starts, s);
    scratch_free(edges, s);
    scratch_free(pieces, s);
    scratch_free(npieces, s);
    scratch_free(bits, s);
    scratch_free(changed, s);
    scratch_free(le[0], s);
    scratch_free(le[1], s);
    scratch_free(lcnt, s);
    return rc;
}

// ---------------------------------------------------------------------------
// K2: CSR validation (CC_FLAG_VALIDATE)
__global__ void k_validate(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, unsigned int* err)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += stride) {
        const int64_t o = off[i];
        if (i == 0 && o != 0) atomicOr(err, 1u);
        if (i == n && o != m) atomicOr(err, 2u);
        if (i < n && off[i + 1] < o) atomicOr(err, 4u);
    }
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (uint64_t)m; i += stride)
        if (adj[i] >= n) atomicOr(err, 8u);
}

cc_status validate_csr(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, cudaStream_t s)
{
    unsigned int* err = nullptr;
    CC_CUDA_TRY(scratch_alloc((void**)&err, sizeof(unsigned int), s));
    CC_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
    k_validate<<<grid_blocks(8), kBlock, 0, s>>>(off, adj, n, m, err);
    CC_LAUNCH_CHECK("k_validate");
    unsigned int h = 0;
    CC_CUDA_TRY(cudaMemcpyAsync(&h, err, sizeof(h), cudaMemcpyDeviceToHost, s));
    CC_CUDA_TRY(cudaStreamSynchronize(s));
    scratch_free(err, s);
    if (h) {
        set_error("CSR validation failed (mask " + std::to_string(h) +
                  "): 1=off[0]!=0 2=off[n]!=m 4=offsets decrease 8=adj id >= n");
        return CC_EINVAL;
    }
    return CC_OK;
}

// ---------------------------------------------------------------------------
template <int MODE, bool SF, int VAR>
static cc_status run(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, uint32_t* P,
                     uint32_t* edges, int64_t* num_edges, uint32_t* labels_out, bool want_labels, const cc_opts& o,
                     cudaStream_t s)
{
    const uint32_t k = o.kout_k;
    const bool degskip = !(o.flags & CC_FLAG_NO_DEGSKIP);
    // the list prefix known to be unioned by the sampling: afforest its first k
    // entries, hybrid its first, pure none; a list no longer than it needs no finish
    const uint32_t skip_prefix = VAR == 0 ? k : VAR == 1 ? std::min<uint32_t>(k, 1u) : 0u;
    const uint32_t full_deg = degskip ? skip_prefix : 0u;
    const bool no_skip = (o.flags & CC_FLAG_NO_SKIP) != 0;
    // contracted k-out link (opt-in; needs the symmetric-graph precondition of the skip)
    const bool contract = k > 0 && !no_skip && (o.flags & CC_FLAG_CONTRACT);
    // sampling and link in one kernel (UF-Rem-CAS + SplitAtomicOne, k <= 2, in-place)
    const bool fused = MODE == 0 && k > 0 && k <= 2 && !contract && (o.flags & CC_FLAG_FUSED_LINK);
    const uint32_t nw = (uint32_t)(((uint64_t)n + 31) / 32);
    const uint32_t nrb = (uint32_t)(((uint64_t)nw + kFTile - 1) / kFTile);

    // afforest: at most sum_u min(k, deg u) <= m pending edges; hybrid/pure: k per non-isolated vertex
    const uint64_t pend_cap = std::max<uint64_t>(
        1, VAR >= 1 ? (uint64_t)k * std::min<uint64_t>(n, (uint64_t)m) : std::min<uint64_t>((uint64_t)n * k, (uint64_t)m));
    const uint64_t big_cap = std::max<uint64_t>(1, std::min<uint64_t>(n, (uint64_t)m / kBigDeg + 1));
    const uint64_t bm_words = ((uint64_t)n + 31) / 32;
    const uint32_t nfb = (uint32_t)(((uint64_t)n + kFTile - 1) / kFTile);
    const uint64_t ntile = ((uint64_t)n + kCTile - 1) / kCTile;     // k_finish blocks = H6 tiles
    const bool sv = (o.flags & (CC_FLAG_FINISH_SV | CC_FLAG_FINISH_CRFA)) != 0;

    Ctl* ctl = nullptr;
    uint32_t* bm = nullptr;
    uint32_t* cq = nullptr;
    uint2* pend = nullptr;
    uint32_t* big = nullptr;
    uint32_t* wsum = nullptr;             // k_finish warp summaries + H5 tile hook flags (partial H6)
    uint8_t* td = nullptr;
    uint2* F = nullptr;
    uint32_t* fcnt = nullptr;
    unsigned long long* foff = nullptr;
    uint2* rbw = nullptr;                 // contracted link: rank words, compact parents, compact -> id
    uint32_t* Cc = nullptr;
    uint32_t* rid = nullptr;
    uint32_t* rcnt = nullptr;
    unsigned long long* roff = nullptr;
    int64_t* Rtot = nullptr;
    cudaEvent_t ev[5] = {};
    cc_status rc = CC_OK;

    auto cleanup = [&]() {
        scratch_free(ctl, s);
        scratch_free(bm, s);
        scratch_free(cq, s);
        scratch_free(pend, s);
        scratch_free(big, s);
        scratch_free(wsum, s);
        scratch_free(td, s);
        scratch_free(F, s);
        scratch_free(fcnt, s);
        scratch_free(foff, s);
        scratch_free(rbw, s);
        scratch_free(Cc, s);
        scratch_free(rid, s);
        scratch_free(rcnt, s);
        scratch_free(roff, s);
        scratch_free(Rtot, s);
    };
    auto body = [&]() -> cc_status {
        CC_CUDA_TRY(scratch_alloc((void**)&ctl, sizeof(Ctl), s));
        CC_CUDA_TRY(scratch_alloc((void**)&bm, sizeof(uint32_t) * bm_words, s));
        // the candidate queue; reused by k_relabel_decide for its chunk queue (kRlPerTile per tile)
        CC_CUDA_TRY(scratch_alloc((void**)&cq, sizeof(uint32_t) * std::max<size_t>(n, kRlPerTile * ntile), s));
        if (k > 0 && !fused) CC_CUDA_TRY(scratch_alloc((void**)&pend, sizeof(uint2) * pend_cap, s));
        CC_CUDA_TRY(scratch_alloc((void**)&big, sizeof(uint32_t) * big_cap, s));
        CC_CUDA_TRY(scratch_alloc((void**)&wsum, sizeof(uint32_t) * kSumPerTile * ntile, s));
        CC_CUDA_TRY(scratch_alloc((void**)&td, ntile, s));
        if (SF) {
            CC_CUDA_TRY(scratch_alloc((void**)&F, sizeof(uint2) * (size_t)n, s));
            CC_CUDA_TRY(scratch_alloc((void**)&fcnt, sizeof(uint32_t) * nfb, s));
            CC_CUDA_TRY(scratch_alloc((void**)&foff, sizeof(unsigned long long) * nfb, s));
            // (F is initialised by k_sample_init, which writes every slot)
        }
        if (contract) {
            // R <= number of non-isolated vertices <= min(n, m); sized for the worst case
            const size_t rcap = std::max<size_t>(1, std::min<uint64_t>(n, (uint64_t)m));
            CC_CUDA_TRY(scratch_alloc((void**)&rbw, sizeof(uint2) * nw, s));
            CC_CUDA_TRY(scratch_alloc((void**)&Cc, sizeof(uint32_t) * rcap, s));
            CC_CUDA_TRY(scratch_alloc((void**)&rid, sizeof(uint32_t) * rcap, s));
            CC_CUDA_TRY(scratch_alloc((void**)&rcnt, sizeof(uint32_t) * nrb, s));
            CC_CUDA_TRY(scratch_alloc((void**)&roff, sizeof(unsigned long long) * nrb, s));
            CC_CUDA_TRY(scratch_alloc((void**)&Rtot, sizeof(int64_t), s));
        }
        CC_CUDA_TRY(cudaMemsetAsync(ctl, 0, sizeof(Ctl), s));
        if (o.timings)
            for (auto& e : ev) CC_CUDA_TRY(cudaEventCreate(&e));
        if (o.timings) CC_CUDA_TRY(cudaEventRecord(ev[0], s));
        auto mark = [&](int i) -> cudaError_t {
            return o.marks ? cudaEventRecord((cudaEvent_t)o.marks[i], s) : cudaSuccess;
        };
        CC_CUDA_TRY(mark(CC_MARK_START));
        bool probed = false;                  // k_probe ran: ctl->skip_mid holds its verdict
        // H1 + H2 (first round) + finish bitmap
        const uint32_t nblk0 = (uint32_t)(((uint64_t)n + kBlockTile - 1) / kBlockTile);
        // 16-byte list-head windows pay off when adj is read over PCIe (pinned host,
        // zero-copy); from HBM two 4-byte loads of the same sector are cheaper
        const bool win = aligned16(adj) && mem_kind(adj, nullptr) == MEM_PINNED;
        if (fused) {
            k_init_pf<<<grid_blocks(16), kBlock, 0, s>>>(P, n, SF ? F : nullptr);
            CC_LAUNCH_CHECK("k_init_pf");
            k_sample_link<VAR, SF><<<nblk0, kBlock, 0, s>>>(off, adj, n, m, k, o.seed, full_deg, P, F, bm,
                                                            o.counters);
            CC_LAUNCH_CHECK("k_sample_link");
        } else if (contract && win)
            CC_CUDA_TRY(launch_pdl(k_sample_init<VAR, SF, true, true>, nblk0, kBlock, s, off, adj, n, m, k, o.seed, full_deg, P, F,
                                                                          pend, bm, rbw, ctl, o.counters));
        else if (contract)
            CC_CUDA_TRY(launch_pdl(k_sample_init<VAR, SF, false, true>, nblk0, kBlock, s, off, adj, n, m, k, o.seed, full_deg, P, F,
                                                                           pend, bm, rbw, ctl, o.counters));
        else if (win)
            CC_CUDA_TRY(launch_pdl(k_sample_init<VAR, SF, true, false>, nblk0, kBlock, s, off, adj, n, m, k, o.seed, full_deg, P, F,
                                                                           pend, bm, nullptr, ctl, o.counters));
        else
            CC_CUDA_TRY(launch_pdl(k_sample_init<VAR, SF, false, false>, nblk0, kBlock, s, off, adj, n, m, k, o.seed, full_deg, P, F,
                                                                            pend, bm, nullptr, ctl, o.counters));
        if (!fused) CC_LAUNCH_CHECK("k_sample_init");
        CC_CUDA_TRY(mark(CC_MARK_INIT));
        if (contract) {
            // rank words -> compact ids (rid, C[c] = c), then P[u] = root_F0(u)
            k_rank_count<<<nrb, kBlock, 0, s>>>(rbw, nw, rcnt);
            CC_LAUNCH_CHECK("k_rank_count");
            k_forest_scan<<<1, kBlock, 0, s>>>(rcnt, nrb, roff, Rtot);
            CC_LAUNCH_CHECK("k_forest_scan(rank)");
            k_rank_fill<<<nrb, kBlock, 0, s>>>(rbw, nw, roff, rid, Cc);
            CC_LAUNCH_CHECK("k_rank_fill");
            if (o.counters)
                CC_CUDA_TRY(cudaMemcpyAsync(&o.counters->contract_roots, Rtot, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
            cc_status r = launch_compress(P, n, nullptr, nullptr, s, "k_compress(F0)");
            if (r) return r;
        } else if (k > 0 && !fused) {
            // shorten the first-round chains before the CAS links when they are long
            // (grid-like inputs); k_probe decides on the device unless a flag forces it --
            // and its verdict also picks the link kernel below
            const bool force = (o.flags & CC_FLAG_MIDCOMPRESS) != 0;
            if (!force) {
                CC_CUDA_TRY(launch_pdl(k_probe, 1, 1024, s, P, n, o.seed, ctl, o.counters));
                CC_LAUNCH_CHECK("k_probe");
                probed = true;
            }
            if (!(o.flags & CC_FLAG_NO_MIDCOMPRESS)) {
                cc_status r = launch_compress(P, n, nullptr, nullptr, s, "k_compress(mid)", force ? nullptr : ctl);
                if (r) return r;
            }
        }
        CC_CUDA_TRY(mark(CC_MARK_MIDCOMPRESS));
        // H2: the remaining sampled edges
        if (fused) {
        } else if (contract) {
            k_link_contract<MODE, SF><<<resident_grid(k_link_contract<MODE, SF>, kBlock), kBlock, 0, s>>>(P, pend, ctl, rbw, Cc, rid, F, o.counters);
            CC_LAUNCH_CHECK("k_link_contract");
            k_contract_final<<<grid_blocks(8), kBlock, 0, s>>>(Cc, rid, Rtot);
            CC_LAUNCH_CHECK("k_contract_final");
        } else if (k > 0 && MODE == 0 && !(o.flags & (CC_FLAG_NO_REFILL | CC_FLAG_LINK_REFILL)) && probed) {
            // device-side choice (no host sync): short round-0 chains (k_probe: skip_mid)
            // -> k_link_pending (2 links per thread, first parents batched); long chains
            // (grid-like inputs) -> the lane-refill kernel; the other one exits at once
            CC_CUDA_TRY(launch_pdl(k_link_pending<MODE, SF>, resident_grid(k_link_pending<MODE, SF>, kBlock), kBlock, s,
                                   P, pend, ctl, F, o.counters, true));
            CC_LAUNCH_CHECK("k_link_pending");
            CC_CUDA_TRY(launch_pdl(k_link_refill<SF>, refill_grid<SF>(), kBlock, s, P, pend, &ctl->pend_count, 0, F,
                                   o.counters, &ctl->skip_mid));
            CC_LAUNCH_CHECK("k_link_refill");
        } else if (k > 0 && MODE == 0 && !(o.flags & CC_FLAG_NO_REFILL)) {
            CC_CUDA_TRY(launch_pdl(k_link_refill<SF>, refill_grid<SF>(), kBlock, s, P, pend, &ctl->pend_count, 0, F,
                                   o.counters, (const unsigned int*)nullptr));
            CC_LAUNCH_CHECK("k_link_refill");
        } else if (k > 0) {
            CC_CUDA_TRY(launch_pdl(k_link_pending<MODE, SF>, resident_grid(k_link_pending<MODE, SF>, kBlock), kBlock, s,
                                   P, pend, ctl, F, o.counters, false));
            CC_LAUNCH_CHECK("k_link_pending");
        }
        CC_CUDA_TRY(mark(CC_MARK_LINK));
        // H3 as its own pass only when the caller asks for the sampled labels
        // (otherwise it is fused into k_finish)
        if (o.sampled_out) {
            if (contract) {
                k_expand<<<(unsigned)(((uint64_t)n + kBlock - 1) / kBlock), kBlock, 0, s>>>(P, n, rbw, rid);
                CC_LAUNCH_CHECK("k_expand");
            } else {
                cc_status r = launch_compress(P, n, nullptr, nullptr, s, "k_compress(H3)");
                if (r) return r;
            }
            CC_CUDA_TRY(cudaMemcpyAsync(o.sampled_out, P, sizeof(uint32_t) * (size_t)n, cudaMemcpyDeviceToDevice, s));
        }
        CC_CUDA_TRY(mark(CC_MARK_SAMPLED));
        if (o.timings) CC_CUDA_TRY(cudaEventRecord(ev[1], s));
        // H4 (roots of the sampled forest; identical before or after H3)
        CC_CUDA_TRY(launch_pdl(k_identify, 1, 1024, s, P, n, o.seed, o.samples, o.lmax_force, ctl, o.lmax_out, rbw, rid));
        CC_LAUNCH_CHECK("k_identify");
        CC_CUDA_TRY(mark(CC_MARK_IDENTIFY));
        if (o.timings) CC_CUDA_TRY(cudaEventRecord(ev[2], s));
        // H3 + H5
        {
            const unsigned nb = (unsigned)ntile;
            if (contract && aligned16(P) && o.counters)
                CC_CUDA_TRY(launch_pdl(k_finish<true, true, true>, nb, kBlock, s, P, bm, n, ctl, no_skip, cq, o.counters, rbw, rid, wsum, td));
            else if (contract && aligned16(P))
                CC_CUDA_TRY(launch_pdl(k_finish<true, false, true>, nb, kBlock, s, P, bm, n, ctl, no_skip, cq, nullptr, rbw, rid, wsum, td));
            else if (contract)
                CC_CUDA_TRY(launch_pdl(k_finish<false, true, true>, nb, kBlock, s, P, bm, n, ctl, no_skip, cq, o.counters, rbw, rid, wsum, td));
            else if (aligned16(P) && o.counters)
                CC_CUDA_TRY(launch_pdl(k_finish<true, true, false>, nb, kBlock, s, P, bm, n, ctl, no_skip, cq, o.counters, nullptr, nullptr, wsum, td));
            else if (aligned16(P))
                CC_CUDA_TRY(launch_pdl(k_finish<true, false, false>, nb, kBlock, s, P, bm, n, ctl, no_skip, cq, nullptr, nullptr, nullptr, wsum, td));
            else
                CC_CUDA_TRY(launch_pdl(k_finish<false, true, false>, nb, kBlock, s, P, bm, n, ctl, no_skip, cq, o.counters, nullptr, nullptr, wsum, td));
            CC_LAUNCH_CHECK("k_finish");
        }
        CC_CUDA_TRY(mark(CC_MARK_FINISH));
        if (sv) {
            // every marked vertex is a finish candidate when the skip is off or nothing was
            // sampled (P is the identity, so only L_max itself is skipped)
            cc_status r = sv_finish<SF>(off, adj, P, n, cq, ctl, skip_prefix, F, o.counters, s,
                                        (o.flags & CC_FLAG_FINISH_CRFA) != 0, bm, no_skip, no_skip || k == 0);
            if (r) return r;
        } else {
            CC_CUDA_TRY(launch_pdl(k_finish_proc<MODE, SF>, resident_grid(k_finish_proc<MODE, SF>, kBlock), kBlock, s, 
                off, adj, P, cq, ctl, skip_prefix, big, big_cap, F, o.counters, td));
            CC_LAUNCH_CHECK("k_finish_proc");
            CC_CUDA_TRY(launch_pdl(k_finish_big<MODE, SF>, resident_grid(k_finish_big<MODE, SF>, 512), 512, s, 
                off, adj, P, big, big_cap, ctl, skip_prefix, F, o.counters, td));
            CC_LAUNCH_CHECK("k_finish_big");
        }
        CC_CUDA_TRY(mark(CC_MARK_FINISH_BIG));
        if (o.timings) CC_CUDA_TRY(cudaEventRecord(ev[3], s));
        // H6: the partial pass when the labels are P itself (k_relabel: only the tiles
        // whose labels H5 changed), nothing when no labels are wanted (a spanning
        // forest without labels), the full pass when they go to another buffer or
        // after an SV / CRFA finish (whose rounds do not keep the tile summaries)
        if (labels_out || sv) {
            cc_status r = launch_compress(P, n, labels_out, o.counters, s, "k_compress(H6)");
            if (r) return r;
        } else if (want_labels) {
            if (o.counters) {
                CC_CUDA_TRY(launch_pdl(k_relabel_decide<true>, resident_grid(k_relabel_decide<true>, kBlock), kBlock, s,
                                       P, n, ctl, no_skip, wsum, td, cq, o.counters));
                CC_LAUNCH_CHECK("k_relabel_decide");
                CC_CUDA_TRY(launch_pdl(k_relabel<true>, resident_grid(k_relabel<true>, kBlock), kBlock, s, P, n, ctl,
                                       no_skip, cq, o.counters));
            } else {
                CC_CUDA_TRY(launch_pdl(k_relabel_decide<false>, resident_grid(k_relabel_decide<false>, kBlock), kBlock,
                                       s, P, n, ctl, no_skip, wsum, td, cq, (cc_counters*)nullptr));
                CC_LAUNCH_CHECK("k_relabel_decide");
                CC_CUDA_TRY(launch_pdl(k_relabel<false>, resident_grid(k_relabel<false>, kBlock), kBlock, s, P, n, ctl,
                                       no_skip, cq, (cc_counters*)nullptr));
            }
            CC_LAUNCH_CHECK("k_relabel(H6)");
        }
        CC_CUDA_TRY(mark(CC_MARK_COMPRESS));
        // H7
        if (SF) {
            // one-pass Filter: status words (foff) and the ticket (fcnt[0]) start at zero
            CC_CUDA_TRY(cudaMemsetAsync(foff, 0, sizeof(unsigned long long) * nfb, s));
            CC_CUDA_TRY(cudaMemsetAsync(fcnt, 0, sizeof(uint32_t), s));
            CC_CUDA_TRY(launch_pdl(k_forest_filter, nfb, kBlock, s, F, n, nfb, foff, fcnt, edges, num_edges, nullptr, nullptr));
            CC_LAUNCH_CHECK("k_forest_filter");
        }
        CC_CUDA_TRY(mark(CC_MARK_FOREST));
        if (o.timings) {
            CC_CUDA_TRY(cudaEventRecord(ev[4], s));
            CC_CUDA_TRY(cudaEventSynchronize(ev[4]));
            float t[4];
            for (int i = 0; i < 4; ++i) CC_CUDA_TRY(cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]));
            o.timings->sample_ms = t[0];
            o.timings->identify_ms = t[1];
            o.timings->finish_ms = t[2];
            o.timings->compress_ms = t[3];
            CC_CUDA_TRY(cudaEventElapsedTime(&o.timings->total_ms, ev[0], ev[4]));
        }
        return CC_OK;
    };
    rc = body();
    cleanup();
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    return rc;
}

template <bool SF, int VAR>
static cc_status dispatch_mode(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, uint32_t* P,
                               uint32_t* edges, int64_t* num_edges, uint32_t* labels_out, bool want, const cc_opts& o,
                               cudaStream_t s)
{
    if (o.flags & CC_FLAG_UF_ASYNC) return run<2, SF, VAR>(off, adj, n, m, P, edges, num_edges, labels_out, want, o, s);
    if (o.flags & CC_FLAG_HALVE) return run<1, SF, VAR>(off, adj, n, m, P, edges, num_edges, labels_out, want, o, s);
    return run<0, SF, VAR>(off, adj, n, m, P, edges, num_edges, labels_out, want, o, s);
}

template <bool SF>
static cc_status dispatch_variant(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, uint32_t* P,
                                  uint32_t* edges, int64_t* num_edges, uint32_t* labels_out, bool want,
                                  const cc_opts& o, cudaStream_t s)
{
    if (o.kout_variant == CC_VARIANT_HYBRID)
        return dispatch_mode<SF, 1>(off, adj, n, m, P, edges, num_edges, labels_out, want, o, s);
    if (o.kout_variant == CC_VARIANT_PURE)
        return dispatch_mode<SF, 2>(off, adj, n, m, P, edges, num_edges, labels_out, want, o, s);
    return dispatch_mode<SF, 0>(off, adj, n, m, P, edges, num_edges, labels_out, want, o, s);
}

cc_status static_pipeline(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, uint32_t* P,
                          uint32_t* labels_out, uint32_t* edges, int64_t* num_edges, bool sf, const cc_opts& o,
                          cudaStream_t s)
{
    // P: the parent array (device memory; the caller's labels buffer for an
    // in-place cc_labels).  NULL: library scratch.  labels_out: where H6 writes
    // the labels when that is not P itself (NULL: nowhere).
    uint32_t* scratch = nullptr;
    const bool want = P != nullptr || labels_out != nullptr;   // else: a forest without labels, no H6
    if (!P) {
        CC_CUDA_TRY(scratch_alloc((void**)&scratch, sizeof(uint32_t) * (size_t)n, s));
        P = scratch;
    }
    uint32_t* out = labels_out == P ? nullptr : labels_out;
    const cc_status rc = sf ? dispatch_variant<true>(off, adj, n, m, P, edges, num_edges, out, want, o, s)
                            : dispatch_variant<false>(off, adj, n, m, P, edges, num_edges, out, want, o, s);
    scratch_free(scratch, s);
    return rc;
}

}  // namespace ccb
