// cc_static.cu -- static connectivity / spanning forest pipeline (H1-H7).
//
// Alg. 1 / Alg. 2 on one B200, stream-ordered with
// no host synchronisation: L_max and every queue length stay in device memory.
//
//   K0 sample_init   H1 P[v] = v fused with the first k-out round: each vertex
//                    u with first neighbour v0 < u sets P[u] = v0 by a plain
//                    store (u is still a singleton root and only u writes
//                    slot u in this kernel, so this IS Union(u, v0) of
//                    Alg. 4 P:3952 with the min orientation of R1).  All other
//                    sampled edges (v0 > u, j = 1..k-1) go to a pending list;
//                    vertices whose list was not fully sampled go to the
//                    finish worklist (degree skip).
//   Kc compress      pointer-jumping compress ("fully compress"; H3/H6)
//   K1 link_pending  UF-Rem-CAS links of the pending sampled edges (H2)
//   K4 identify      IdentifyFrequent over S seeded samples (R9)
//   K5 finish        Union over the lists of worklist vertices whose sampled
//                    label != L_max, degree-binned
//                    thread / warp / CTA-per-vertex
//   K7 forest        Filter of Alg. 2: compact non-sentinel slots in
//                    slot order
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "cc_device.cuh"
#include "cc_internal.h"

namespace ccb {

struct Ctl {
    unsigned long long pend_count;
    unsigned long long wl_count;
    unsigned long long big_count;
    unsigned int lmax;
    unsigned int err;
};

constexpr uint32_t kSentinel = 0xFFFFFFFFu;
constexpr int kSmallDeg = 8;      // <= : one lane walks the list
constexpr int kBigDeg = 4096;     // >  : one CTA per vertex (second kernel)

// Exclusive warp prefix of c and one atomicAdd per warp; every lane must call.
__device__ __forceinline__ unsigned long long warp_append(unsigned long long* counter, uint32_t c)
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

__device__ __forceinline__ void warp_count(uint64_t* ctr, uint32_t c)
{
    if (!ctr) return;
    uint32_t s = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(reinterpret_cast<unsigned long long*>(ctr), (unsigned long long)s);
}

// ---------------------------------------------------------------------------
// K0: H1 + first k-out round + pending list + finish worklist.
template <bool HYBRID, bool SF>
__global__ void __launch_bounds__(kBlock) k_sample_init(
    const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, uint32_t n, uint32_t k,
    uint64_t seed, uint32_t full_deg, uint32_t* __restrict__ P, uint2* __restrict__ F,
    uint2* __restrict__ pend, uint32_t* __restrict__ wl, Ctl* ctl, cc_counters* cnt)
{
    const uint64_t u64 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = u64 < n;
    const uint32_t u = (uint32_t)u64;
    int64_t b = 0, e = 0;
    if (valid) {
        b = ld_stream_i64(off + u);
        e = ld_stream_i64(off + u + 1);
    }
    const int64_t d = e - b;
    uint32_t p = u;
    uint32_t v0 = 0;
    uint32_t npend = 0;
    if (valid && d > 0 && k > 0) {
        v0 = ld_stream_u32(adj + b);
        if (v0 < u) {
            p = v0;                                    // Union(u, v0): hook singleton root u
            if (SF) F[u] = make_uint2(u, v0);          // forest edge at the hooked root
        } else if (v0 > u) {
            npend = 1;
        }
        const int64_t kk = HYBRID ? (int64_t)k : min((int64_t)k, d);
        npend += (uint32_t)(kk - 1);
    }
    if (valid) P[u] = p;
    // pending sampled edges
    unsigned long long pos = warp_append(&ctl->pend_count, npend);
    if (npend) {
        if (v0 > u) pend[pos++] = make_uint2(u, v0);
        const int64_t kk = HYBRID ? (int64_t)k : min((int64_t)k, d);
        for (int64_t j = 1; j < kk; ++j) {
            int64_t i = HYBRID ? (int64_t)uniform_below(mix(seed, KOUT_STREAM, (uint64_t)u * 64 + j), (uint64_t)d)
                               : j;
            pend[pos++] = make_uint2(u, ld_stream_u32(adj + b + i));
        }
    }
    // finish worklist: lists not wholly unioned by the sampling
    const uint32_t inwl = (valid && d > (int64_t)full_deg) ? 1u : 0u;
    unsigned long long wpos = warp_append(&ctl->wl_count, inwl);
    if (inwl) wl[wpos] = u;
    if (cnt) warp_count(&cnt->pending_links, npend);
}

// ---------------------------------------------------------------------------
// Kc: pointer-jumping compress.  Within this kernel no hook happens, so every
// value read is an ancestor-or-self on the path to the (fixed) root, stale or
// not; plain (L1-cacheable) loads are therefore safe and let the hot giant
// root stay in L1.  Blocks run roughly in ascending id order and P[x] < x, so
// most parents are already compressed when their children are visited.
__global__ void __launch_bounds__(kBlock) k_compress(uint32_t* P, uint32_t n, uint32_t* out)
{
    const uint64_t v64 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v64 >= n) return;
    const uint32_t v = (uint32_t)v64;
    const uint32_t p = P[v];
    uint32_t r = p;
    if (p != v) {
        uint32_t q = P[r];
        while (q != r) {
            r = q;
            q = P[r];
        }
        if (r != p) P[v] = r;
    }
    if (out) out[v] = r;
}

// ---------------------------------------------------------------------------
// K1: UF-Rem-CAS links of the pending sampled edges.
template <int MODE, bool SF>
__global__ void __launch_bounds__(kBlock) k_link_pending(
    uint32_t* P, const uint2* __restrict__ pend, const Ctl* ctl, uint2* F, cc_counters* cnt)
{
    const unsigned long long total = ctl->pend_count;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x;
    for (; base < total; base += stride) {
        const unsigned long long i = base + threadIdx.x;
        uint32_t hooked = 0;
        if (i < total) {
            const uint2 pr = pend[i];
            if constexpr (SF) hooked = link<MODE>(P, pr.x, pr.y, Forest{F});
            else hooked = link<MODE>(P, pr.x, pr.y, NoForest{});
        }
        if (cnt) warp_count(&cnt->hooks, hooked);
    }
}

// ---------------------------------------------------------------------------
// K4: IdentifyFrequent: mode of P[s_i], s_i = uniform_below(mix(seed,
// IDENT, i), n), ties to the smaller label (reading R9).  One CTA of 1024
// threads; a bitonic sort in shared memory, then a max-reduction of
// (run length, -label).
__global__ void __launch_bounds__(1024) k_identify(const uint32_t* P, uint32_t n, uint64_t seed,
                                                   uint32_t samples, const uint32_t* force, Ctl* ctl,
                                                   uint32_t* lmax_out)
{
    constexpr int S = 4096;
    __shared__ uint32_t a[S];
    __shared__ unsigned long long best[32];
    const int t = threadIdx.x;
    if (force) {
        if (t == 0) {
            ctl->lmax = *force;
            if (lmax_out) *lmax_out = *force;
        }
        return;
    }
    int size = 1;
    while (size < (int)samples) size <<= 1;
    for (int i = t; i < size; i += blockDim.x) {
        uint32_t lab = kSentinel;
        if (i < (int)samples) {
            uint32_t s = uniform_below(mix(seed, IDENT_STREAM, (uint64_t)i), n);
            uint32_t r = s, q = P[r];
            while (q != r) { r = q; q = P[r]; }
            lab = r;
        }
        a[i] = lab;
    }
    __syncthreads();
    for (int kk = 2; kk <= size; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int i = t; i < size; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    uint32_t x = a[i], y = a[ixj];
                    bool up = (i & kk) == 0;
                    if ((x > y) == up) { a[i] = y; a[ixj] = x; }
                }
            }
            __syncthreads();
        }
    }
    unsigned long long key = 0;
    for (int i = t; i < (int)samples; i += blockDim.x) {
        if (i == 0 || a[i] != a[i - 1]) {
            int j = i + 1;
            while (j < (int)samples && a[j] == a[i]) ++j;
            unsigned long long kk2 = ((unsigned long long)(j - i) << 32) | (unsigned long long)(kSentinel - a[i]);
            key = key > kk2 ? key : kk2;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
        key = key > y ? key : y;
    }
    if ((t & 31) == 0) best[t >> 5] = key;
    __syncthreads();
    if (t < 32) {
        key = t < (int)(blockDim.x >> 5) ? best[t] : 0;
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
            key = key > y ? key : y;
        }
        if (t == 0) {
            uint32_t lm = kSentinel - (uint32_t)(key & 0xFFFFFFFFull);
            ctl->lmax = lm;
            if (lmax_out) *lmax_out = lm;
        }
    }
}

// ---------------------------------------------------------------------------
// K5: finish.  Each warp takes 32 worklist entries; a lane keeps
// its vertex if the vertex's sampled label is not L_max.  Short lists (after
// dropping the afforest-sampled prefix) are walked by their own lane, medium
// lists by the whole warp (ballot/shuffle; an edge whose endpoint already sits
// directly under u's root is skipped without a link), long lists are queued
// for k_finish_big (one CTA per vertex).
template <int MODE, bool SF>
__global__ void __launch_bounds__(kBlock) k_finish(
    const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, uint32_t* P,
    const uint32_t* __restrict__ wl, Ctl* ctl, uint32_t skip_prefix, bool no_skip, uint32_t* big,
    uint2* F, cc_counters* cnt)
{
    const unsigned long long total = ctl->wl_count;
    const uint32_t lmax = no_skip ? kSentinel : ctl->lmax;
    const unsigned lane = threadIdx.x & 31;
    const unsigned long long warp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    for (unsigned long long base = warp * 32; base < total; base += nwarps * 32) {
        const unsigned long long i = base + lane;
        uint32_t u = 0;
        bool proc = false;
        if (i < total) {
            u = wl[i];
            proc = ld_relaxed(P + u) != lmax;
        }
        int64_t b = 0, e = 0;
        if (proc) {
            b = off[u];
            e = off[u + 1];
            b += min((int64_t)skip_prefix, e - b);     // afforest: first k edges already unioned
        }
        const int64_t d = e - b;
        const bool small = proc && d <= kSmallDeg;
        const bool medium = proc && d > kSmallDeg && d <= kBigDeg;
        const bool isbig = proc && d > kBigDeg;
        if (cnt) {
            warp_count(&cnt->finish_vertices, proc ? 1u : 0u);
            warp_count(&cnt->finish_offsets, proc ? 1u : 0u);
            warp_count(&cnt->finish_edges, proc ? (uint32_t)min(d, (int64_t)0xFFFFFFFF) : 0u);
            warp_count(&cnt->big_vertices, isbig ? 1u : 0u);
        }
        unsigned long long bpos = warp_append(&ctl->big_count, isbig ? 1u : 0u);
        if (isbig) big[bpos] = u;
        uint32_t hooks = 0;
        if (small) {
            for (int64_t x = b; x < e; ++x) {
                const uint32_t v = adj[x];
                if constexpr (SF) hooks += link<MODE>(P, u, v, Forest{F});
                else hooks += link<MODE>(P, u, v, NoForest{});
            }
        }
        unsigned mm = __ballot_sync(0xffffffffu, medium);
        while (mm) {
            const int src = __ffs(mm) - 1;
            mm &= mm - 1;
            const uint32_t mu = __shfl_sync(0xffffffffu, u, src);
            const int64_t mb = __shfl_sync(0xffffffffu, b, src);
            const int64_t me = __shfl_sync(0xffffffffu, e, src);
            uint32_t ru = 0;
            if (lane == 0) ru = find_naive(P, mu);
            ru = __shfl_sync(0xffffffffu, ru, 0);
            for (int64_t x = mb + lane; x < me; x += 32) {
                const uint32_t v = adj[x];
                if (ld_relaxed(P + v) == ru) continue;  // v hangs directly under u's root
                if constexpr (SF) hooks += link<MODE>(P, mu, v, Forest{F});
                else hooks += link<MODE>(P, mu, v, NoForest{});
            }
        }
        if (cnt) warp_count(&cnt->hooks, hooks);
    }
}

template <int MODE, bool SF>
__global__ void __launch_bounds__(512) k_finish_big(const int64_t* __restrict__ off,
                                                    const uint32_t* __restrict__ adj, uint32_t* P,
                                                    const uint32_t* __restrict__ big, const Ctl* ctl,
                                                    uint32_t skip_prefix, uint2* F, cc_counters* cnt)
{
    __shared__ uint32_t s_ru;
    const unsigned long long total = ctl->big_count;
    for (unsigned long long i = blockIdx.x; i < total; i += gridDim.x) {
        const uint32_t u = big[i];
        int64_t b = off[u];
        const int64_t e = off[u + 1];
        b += min((int64_t)skip_prefix, e - b);
        __syncthreads();
        if (threadIdx.x == 0) s_ru = find_naive(P, u);
        __syncthreads();
        const uint32_t ru = s_ru;
        uint32_t hooks = 0;
        for (int64_t x = b + threadIdx.x; x < e; x += blockDim.x) {
            const uint32_t v = adj[x];
            if (ld_relaxed(P + v) == ru) continue;
            if constexpr (SF) hooks += link<MODE>(P, u, v, Forest{F});
            else hooks += link<MODE>(P, u, v, NoForest{});
        }
        if (cnt) warp_count(&cnt->hooks, hooks);
    }
}

// ---------------------------------------------------------------------------
// K7: Filter -- stable compaction of the non-sentinel forest slots.
constexpr int kFItems = 16;                  // slots per thread
constexpr int kFTile = kBlock * kFItems;     // slots per block

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* total)
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

__global__ void __launch_bounds__(kBlock) k_forest_count(const uint2* F, uint32_t n, uint32_t* block_cnt)
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
__global__ void __launch_bounds__(kBlock) k_forest_scan(const uint32_t* block_cnt, uint32_t nb,
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

__global__ void __launch_bounds__(kBlock) k_forest_write(const uint2* F, uint32_t n,
                                                         const unsigned long long* block_off,
                                                         uint32_t* edges)
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
            ++o;
        }
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
    k_validate<<<num_sms() * 8, kBlock, 0, s>>>(off, adj, n, m, err);
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
template <int MODE, bool SF, bool HYBRID>
static cc_status run(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, uint32_t* P,
                     uint32_t* edges, int64_t* num_edges, uint32_t* labels_out, const cc_opts& o,
                     cudaStream_t s)
{
    const uint32_t k = o.kout_k;
    const bool afforest = !HYBRID;
    const bool degskip = !(o.flags & CC_FLAG_NO_DEGSKIP);
    // a list of length <= full_deg was wholly unioned by the sampling
    const uint32_t full_deg = !degskip ? 0u : (afforest ? k : std::min<uint32_t>(k, 1u));
    const uint32_t skip_prefix = afforest ? k : std::min<uint32_t>(k, 1u);
    const bool no_skip = (o.flags & CC_FLAG_NO_SKIP) != 0;
    const int sms = num_sms();

    // afforest: at most sum_u min(k, deg u) <= m pending edges; hybrid: k per non-isolated vertex
    const uint64_t pend_cap = std::max<uint64_t>(
        1, HYBRID ? (uint64_t)k * std::min<uint64_t>(n, (uint64_t)m) : std::min<uint64_t>((uint64_t)n * k, (uint64_t)m));
    const uint64_t big_cap = std::max<uint64_t>(1, std::min<uint64_t>(n, (uint64_t)m / kBigDeg + 1));
    const uint32_t nfb = (uint32_t)(((uint64_t)n + kFTile - 1) / kFTile);

    Ctl* ctl = nullptr;
    uint32_t* wl = nullptr;
    uint2* pend = nullptr;
    uint32_t* big = nullptr;
    uint2* F = nullptr;
    uint32_t* fcnt = nullptr;
    unsigned long long* foff = nullptr;
    cudaEvent_t ev[5] = {};
    cc_status rc = CC_OK;

    auto cleanup = [&]() {
        scratch_free(ctl, s);
        scratch_free(wl, s);
        scratch_free(pend, s);
        scratch_free(big, s);
        scratch_free(F, s);
        scratch_free(fcnt, s);
        scratch_free(foff, s);
    };
    auto body = [&]() -> cc_status {
        CC_CUDA_TRY(scratch_alloc((void**)&ctl, sizeof(Ctl), s));
        CC_CUDA_TRY(scratch_alloc((void**)&wl, sizeof(uint32_t) * (size_t)n, s));
        if (k > 0) CC_CUDA_TRY(scratch_alloc((void**)&pend, sizeof(uint2) * pend_cap, s));
        CC_CUDA_TRY(scratch_alloc((void**)&big, sizeof(uint32_t) * big_cap, s));
        if (SF) {
            CC_CUDA_TRY(scratch_alloc((void**)&F, sizeof(uint2) * (size_t)n, s));
            CC_CUDA_TRY(scratch_alloc((void**)&fcnt, sizeof(uint32_t) * nfb, s));
            CC_CUDA_TRY(scratch_alloc((void**)&foff, sizeof(unsigned long long) * nfb, s));
            CC_CUDA_TRY(cudaMemsetAsync(F, 0xFF, sizeof(uint2) * (size_t)n, s));
        }
        CC_CUDA_TRY(cudaMemsetAsync(ctl, 0, sizeof(Ctl), s));
        if (o.timings)
            for (auto& e : ev) CC_CUDA_TRY(cudaEventCreate(&e));
        if (o.timings) CC_CUDA_TRY(cudaEventRecord(ev[0], s));

        const uint32_t nblk = (uint32_t)(((uint64_t)n + kBlock - 1) / kBlock);
        // H1 + H2 (first round)
        k_sample_init<HYBRID, SF><<<nblk, kBlock, 0, s>>>(off, adj, n, k, o.seed, full_deg, P, F, pend, wl, ctl,
                                                          o.counters);
        CC_LAUNCH_CHECK("k_sample_init");
        if (k > 0) {
            if (!(o.flags & CC_FLAG_NO_MIDCOMPRESS)) {
                k_compress<<<nblk, kBlock, 0, s>>>(P, n, nullptr);
                CC_LAUNCH_CHECK("k_compress(mid)");
            }
            k_link_pending<MODE, SF><<<sms * 8, kBlock, 0, s>>>(P, pend, ctl, F, o.counters);
            CC_LAUNCH_CHECK("k_link_pending");
            k_compress<<<nblk, kBlock, 0, s>>>(P, n, nullptr);     // H3: height-one (Def. 3.1)
            CC_LAUNCH_CHECK("k_compress(H3)");
        }
        if (o.sampled_out)
            CC_CUDA_TRY(cudaMemcpyAsync(o.sampled_out, P, sizeof(uint32_t) * (size_t)n, cudaMemcpyDeviceToDevice, s));
        if (o.timings) CC_CUDA_TRY(cudaEventRecord(ev[1], s));
        // H4
        k_identify<<<1, 1024, 0, s>>>(P, n, o.seed, o.samples, o.lmax_force, ctl, o.lmax_out);
        CC_LAUNCH_CHECK("k_identify");
        if (o.timings) CC_CUDA_TRY(cudaEventRecord(ev[2], s));
        // H5
        k_finish<MODE, SF><<<sms * 16, kBlock, 0, s>>>(off, adj, P, wl, ctl, skip_prefix, no_skip, big, F,
                                                       o.counters);
        CC_LAUNCH_CHECK("k_finish");
        k_finish_big<MODE, SF><<<sms * 2, 512, 0, s>>>(off, adj, P, big, ctl, skip_prefix, F, o.counters);
        CC_LAUNCH_CHECK("k_finish_big");
        if (o.timings) CC_CUDA_TRY(cudaEventRecord(ev[3], s));
        // H6
        k_compress<<<nblk, kBlock, 0, s>>>(P, n, labels_out);
        CC_LAUNCH_CHECK("k_compress(H6)");
        // H7
        if (SF) {
            k_forest_count<<<nfb, kBlock, 0, s>>>(F, n, fcnt);
            CC_LAUNCH_CHECK("k_forest_count");
            k_forest_scan<<<1, kBlock, 0, s>>>(fcnt, nfb, foff, num_edges);
            CC_LAUNCH_CHECK("k_forest_scan");
            k_forest_write<<<nfb, kBlock, 0, s>>>(F, n, foff, edges);
            CC_LAUNCH_CHECK("k_forest_write");
        }
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

template <bool SF, bool HYBRID>
static cc_status dispatch_mode(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, uint32_t* P,
                               uint32_t* edges, int64_t* num_edges, uint32_t* labels_out, const cc_opts& o,
                               cudaStream_t s)
{
    if (o.flags & CC_FLAG_UF_ASYNC) return run<2, SF, HYBRID>(off, adj, n, m, P, edges, num_edges, labels_out, o, s);
    if (o.flags & CC_FLAG_HALVE) return run<1, SF, HYBRID>(off, adj, n, m, P, edges, num_edges, labels_out, o, s);
    return run<0, SF, HYBRID>(off, adj, n, m, P, edges, num_edges, labels_out, o, s);
}

cc_status static_pipeline(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, uint32_t* labels,
                          uint32_t* edges, int64_t* num_edges, bool sf, const cc_opts& o, cudaStream_t s)
{
    // cc_labels: labels is the parent array (in place).  cc_spanning_forest:
    // a scratch parent array; labels (optional) receives the final compress.
    uint32_t* P = labels;
    uint32_t* out = nullptr;
    if (sf && !labels) CC_CUDA_TRY(scratch_alloc((void**)&P, sizeof(uint32_t) * (size_t)n, s));
    const bool hybrid = o.kout_variant == CC_VARIANT_HYBRID;
    cc_status rc;
    if (sf) {
        rc = hybrid ? dispatch_mode<true, true>(off, adj, n, m, P, edges, num_edges, out, o, s)
                    : dispatch_mode<true, false>(off, adj, n, m, P, edges, num_edges, out, o, s);
        if (!labels) scratch_free(P, s);
    } else {
        rc = hybrid ? dispatch_mode<false, true>(off, adj, n, m, P, edges, num_edges, out, o, s)
                    : dispatch_mode<false, false>(off, adj, n, m, P, edges, num_edges, out, o, s);
    }
    return rc;
}

}  // namespace ccb
