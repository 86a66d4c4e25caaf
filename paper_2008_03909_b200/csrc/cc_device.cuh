// cc_device.cuh -- device primitives of the union-find hot path (sm_100a).
//
// B4 of DESIGN.md: relaxed device-scope parent loads, CAS, the UF-Rem-CAS
// link with SplitAtomicOne / HalveAtomicOne, UF-Async, FindNaive.  Citations
// P:n are PAPER.md lines; Rn are DESIGN.md readings.
//
// Memory model.  L1 is not coherent across SMs.  Reads whose freshness a
// decision depends on (a find's root test, the wait-free query's re-check) are
// ld.relaxed.gpu (served by L2, never by a stale L1 line); the paper marks
// these reads with an asterisk (reading R5).  The UF-Rem-CAS
// loop itself tolerates stale parents and reads through L1 (ld_link below).  Correctness
// rests on two invariants:
//   (I1) P[x] <= x at all times, with equality exactly at roots: a hook writes
//        pv < pu = ru, a split writes a grandparent w <= parent.  So every
//        root is the minimum of its tree and the trees stay acyclic.
//   (I2) a slot never increases, so there is no ABA: a stale (larger) value
//        only makes a CAS fail or a walk take an extra step.
#pragma once
#include <cstdint>

namespace ccb {

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p)
{
    uint32_t v;
#ifdef CC_LD_CG
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
#else
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
#endif
    return v;
}

// Parent reads inside the UF-Rem-CAS loop (link_rem_from and the lane-refill
// kernel): L1-ALLOCATING loads (ld.global.ca), so the hot slots every walk ends
// at (the big trees' roots) are served by each SM's L1 instead of one L2 slice
// (measured: C3 link 0.35 -> 0.28 ms, C1 -20 %, C4 -5 %).  The Rem loop is
// correct with stale values (reading R5): a value a slot ever held is
// in the slot's set, so "equal parents" still proves one set; a stale root claim
// is validated by the hook CAS, whose returned value is fresh; a split writes
// w <= pu < ru (I1), which cannot be a descendant of ru (every descendant is
// larger), and w is in ru's set; a hook writes pv < ru into a root ru, and the
// root is its tree's minimum (I1), so pv is not in ru's tree.  L1 is invalidated
// at every kernel launch, so staleness never crosses a kernel boundary.
// CC_LINK_LD_RELAXED restores device-scope relaxed loads (the round-1 reading).
__device__ __forceinline__ uint32_t ld_link(const uint32_t* p)
{
#ifndef CC_LINK_LD_RELAXED
    uint32_t v;
    asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
#else
    return ld_relaxed(p);
#endif
}

// Programmatic dependent launch: let the next kernel of the stream be scheduled
// now (pdl_trigger), and wait until the previous one has completed and its
// writes are visible (pdl_wait).  No-ops for kernels launched without PDL.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint32_t cas(uint32_t* p, uint32_t expect, uint32_t desired)
{
    return atomicCAS(p, expect, desired);
}

// Streaming loads that should not pollute L1 (read once).
__device__ __forceinline__ int64_t ld_stream_i64(const int64_t* p)
{
    int64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.s64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// FindNaive: walk to the root without writes.
__device__ __forceinline__ uint32_t find_naive(const uint32_t* P, uint32_t x)
{
    uint32_t p = ld_relaxed(P + x);
    while (p != x) {
        x = p;
        p = ld_relaxed(P + x);
    }
    return x;
}

// FindAtomicSplit (reading R4): CAS each node to its grandparent
// and advance one step; returns the root.
__device__ __forceinline__ uint32_t find_split(uint32_t* P, uint32_t u)
{
    uint32_t v = ld_relaxed(P + u);
    uint32_t w = ld_relaxed(P + v);
    while (v != w) {
        cas(P + u, v, w);
        u = v;
        v = w;
        w = ld_relaxed(P + v);
    }
    return v;
}

// Path halving without atomics, for phases in which no hook runs (the query
// phase of a type (3) batch): each step stores the grandparent (an ancestor)
// into the node; loads are device-scope so a root is never judged from a
// stale L1 line.
__device__ __forceinline__ uint32_t find_halve_quiet(uint32_t* P, uint32_t x)
{
    uint32_t p = ld_relaxed(P + x);
    while (p != x) {
        const uint32_t g = ld_relaxed(P + p);
        if (g == p) return p;
        P[x] = g;
        x = g;
        p = ld_relaxed(P + x);
    }
    return x;
}

// The same walk entered with p = a value P[x] held after the last hook of x's tree
// was ordered before this call (a read of x's slot taken earlier, then refreshed by the
// caller when it claimed x a root): p is x or an ancestor, so the walk below -- whose
// root tests all read L2 -- returns x's current root.
__device__ __forceinline__ uint32_t find_halve_quiet_from(uint32_t* P, uint32_t x, uint32_t p)
{
    while (p != x) {
        const uint32_t g = ld_relaxed(P + p);
        if (g == p) return p;
        P[x] = g;
        x = g;
        p = ld_relaxed(P + x);
    }
    return x;
}

struct NoForest {
    __device__ __forceinline__ void record(uint32_t, uint32_t, uint32_t) const {}
};

// Spanning-forest record: the edge whose CAS hooked root r is
// stored at slot r.  Each root is hooked at most once (it never becomes a root
// again, I2), so a plain store suffices.
struct Forest {
    uint2* F;
    __device__ __forceinline__ void record(uint32_t r, uint32_t u, uint32_t v) const
    {
        F[r] = make_uint2(u, v);
    }
};

// UF-Rem-CAS union (Alg. UF-Rem-CAS) with SplitAtomicOne
// or HalveAtomicOne as the splice step, FindNaive
// as the compress option.  Orientation (readings R1, R6): in each iteration
// pu = P[ru], pv = P[rv]; equal parents => same tree; otherwise orient so that
// pu > pv; if ru is a root, hook it under the snapshot pv by CAS, else take one
// split/halve step on ru.  Returns true iff this call hooked a root.
// Optional per-thread statistics of the loop (diagnostic counters only).
struct NoStat {
    __device__ __forceinline__ void step() {}
    __device__ __forceinline__ void casfail() {}
};
struct Stat {
    uint32_t steps = 0, fails = 0;
    __device__ __forceinline__ void step() { ++steps; }
    __device__ __forceinline__ void casfail() { ++fails; }
};

// link_rem_from: the same loop entered with the first two parent reads
// (pu = P[u], pv = P[v]) already done by the caller (batched loads).
template <bool HALVE, class Rec, class St = NoStat>
__device__ __forceinline__ bool link_rem_from(uint32_t* P, uint32_t u, uint32_t v, uint32_t pu, uint32_t pv,
                                              const Rec& rec, St* st = nullptr)
{
    uint32_t ru = u, rv = v;
    while (true) {
        if (pu == pv) return false;
        if (st) st->step();                          // an iteration that makes a memory access
        if (pu < pv) {
            uint32_t t = ru; ru = rv; rv = t;
            t = pu; pu = pv; pv = t;
        }
        if (ru == pu) {                              // ru is a root: hook it (pv < ru)
            const uint32_t old = cas(P + ru, ru, pv);
            if (old == ru) {
                rec.record(ru, u, v);
                return true;
            }
            if (st) st->casfail();
            pu = old;                                // lost a race: the CAS returned ru's new parent
            pv = ld_link(P + rv);
            continue;
        }
        uint32_t w = ld_link(P + pu);                // one splice step on ru
        if (w != pu) cas(P + ru, pu, w);
        // SplitAtomicOne continues from pu, whose parent w was just read: reuse
        // it (and the snapshot pv) instead of re-reading -- each is a value the
        // slot held during this call, which is all the loop needs (I1, I2).
#ifdef CC_LINK_NO_REUSE
        ru = HALVE ? w : pu;
        pu = ld_relaxed(P + ru);
        pv = ld_relaxed(P + rv);
#else
        if (HALVE) {
            ru = w;
            pu = ld_relaxed(P + ru);
        } else {
            ru = pu;
            pu = w;
        }
#endif
    }
}

template <bool HALVE, class Rec>
__device__ __forceinline__ bool link_rem(uint32_t* P, uint32_t u, uint32_t v, const Rec& rec)
{
    return link_rem_from<HALVE>(P, u, v, ld_relaxed(P + u), ld_relaxed(P + v), rec);
}

// UF-Async union (reading R2: the CAS targets the root slot).
template <class Rec>
__device__ __forceinline__ bool link_async(uint32_t* P, uint32_t u, uint32_t v, const Rec& rec)
{
    uint32_t ru = find_naive(P, u), rv = find_naive(P, v);
    while (ru != rv) {
        if (ru < rv) { uint32_t t = ru; ru = rv; rv = t; }
        if (cas(P + ru, ru, rv) == ru) {
            rec.record(ru, u, v);
            return true;
        }
        ru = find_naive(P, ru);                      // roots only move up: restart from them
        rv = find_naive(P, rv);
    }
    return false;
}

template <int MODE, class Rec>
__device__ __forceinline__ bool link(uint32_t* P, uint32_t u, uint32_t v, const Rec& rec)
{
    if constexpr (MODE == 0) return link_rem<false>(P, u, v, rec);
    else if constexpr (MODE == 1) return link_rem<true>(P, u, v, rec);
    else return link_async(P, u, v, rec);
}

// Counter-based generator for the method's own draws (hybrid picks, the
// IdentifyFrequent samples): mix(s,t,i) = splitmix64(s*GOLD + t*2^40 + i).
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t mix(uint64_t seed, uint64_t stream, uint64_t i)
{
    return splitmix64(seed * 0x9E3779B97F4A7C15ull + (stream << 40) + i);
}

__host__ __device__ __forceinline__ uint32_t uniform_below(uint64_t r, uint64_t bound)
{
    return (uint32_t)(((r & 0xFFFFFFFFull) * bound) >> 32);
}

constexpr uint64_t KOUT_STREAM = 16;
constexpr uint64_t IDENT_STREAM = 17;

}  // namespace ccb
