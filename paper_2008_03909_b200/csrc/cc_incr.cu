// cc_incr.cu -- batch-incremental connectivity (H8, H9).
//
// Alg. 3 with UF-Rem-CAS + SplitAtomicOne on a
// persistent parent array P owned by the handle.  Each batch is processed in
// the phase-concurrent order of type (3): one kernel applies all
// inserts (each Insert(u,v) is a Union), the kernel boundary is the barrier,
// then one kernel answers all IsConnected(a,b) queries as Find(a) == Find(b)
// (reading R15).  Answers are therefore deterministic and bit-exact with the
// sequential oracle.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "cc_device.cuh"
#include "cc_internal.h"

struct cc_incr {
    uint32_t n;
    uint32_t flags;
    uint32_t* P;
    int device;
    cudaStream_t last;
};

namespace ccb {

__global__ void __launch_bounds__(kBlock) k_iota(uint32_t* P, uint32_t n)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) P[i] = (uint32_t)i;
}

// 128-thread blocks: the batch's inserts spread over more, shorter blocks, so the
// kernel's tail (the last blocks' longest Rem walks) is shorter (C5: 34.1 -> 34.7 G
// ops/s; 64 threads 34.3; one resident grid-strided wave 31.0)
constexpr int kInsBlock = 128;
constexpr int kQryBlock = 256;               // 128 / 64: within noise (C5 34.7 G ops/s)

template <int MODE>
__global__ void __launch_bounds__(kInsBlock) k_insert(uint32_t* P, const uint2* __restrict__ ins, int64_t n_ins,
                                                   bool pre)
{
    pdl_trigger();                                // the next batch's kernel may be scheduled now
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
#ifndef CC_INCR_NOPREFETCH
    if (MODE == 0 && pre) {
        // Before the wait (while the previous batch's query kernel drains): the pair and its
        // two first parent reads.  They may be stale w.r.t. that kernel's halving stores, which
        // the Rem loop tolerates (R5: every value a slot held is an ancestor in its set; the
        // hook CAS validates a root claim), so a block resident early starts its walk at once.
        // `pre` is set only where the pairs are known to be in place (insert_query).
        uint2 e = make_uint2(0u, 0u);
        uint32_t pu = 0, pv = 0;
        if (i < n_ins) {
            e = ins[i];
            pu = ld_relaxed(P + e.x);
            pv = ld_relaxed(P + e.y);
        }
        pdl_wait();                               // ... the hooks start after the previous kernel
        if (i < n_ins) link_rem_from<false>(P, e.x, e.y, pu, pv, NoForest{});
        return;
    }
#endif
    pdl_wait();                                   // ... and this one starts after the previous kernel
    if (i >= n_ins) return;
    const uint2 e = ins[i];
    link<MODE>(P, e.x, e.y, NoForest{});
}

// Queries run after the insert kernel: no hook can happen concurrently, so
// roots are fixed and FindNaive needs no L2-forced loads; with SPLIT the finds
// also shorten paths (FindAtomicSplit) for later batches.
// FIND: 0 = path halving without atomics (default: no hook runs in the query
// phase, so pointing a node at its grandparent is a plain store of an ancestor;
// it keeps adversarial chains -- a path inserted in id order -- from costing
// O(length) per query: 29 s -> 4 ms for 2^20 queries on a 2^24 path), 1 =
// FindAtomicSplit, 2 = FindNaive.
template <int FIND>
__device__ __forceinline__ uint32_t query_find(uint32_t* P, uint32_t x)
{
    if constexpr (FIND == 1) return find_split(P, x);
    else if constexpr (FIND == 2) return find_naive(P, x);
    else return find_halve_quiet(P, x);
}

template <int FIND>
__global__ void __launch_bounds__(kQryBlock) k_query(uint32_t* P, const uint2* __restrict__ q, int64_t n_q,
                                                  uint8_t* __restrict__ ans, bool pre)
{
    pdl_trigger();                                // the next batch's kernel may be scheduled now
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
#ifndef CC_INCR_NOPREFETCH
    if (FIND == 0 && pre) {
        // Before the wait (while this batch's insert kernel drains): the pair and the two first
        // parent reads.  A stale value is an ancestor of the vertex (hooks and splits only move
        // a slot up its tree), so the walk may start there; only a stale ROOT claim (the vertex
        // itself) is re-read after the wait, and every root test below reads L2 after the wait.
        // `pre` is set only where the pairs are known to be in place (insert_query).
        uint2 e = make_uint2(0u, 0u);
        uint32_t pa = 0, pb = 0;
        if (i < n_q) {
            e = q[i];
            pa = ld_relaxed(P + e.x);
            pb = ld_relaxed(P + e.y);
        }
        pdl_wait();                               // ... the answers read the state after all inserts
        if (i >= n_q) return;
        if (pa == e.x) pa = ld_relaxed(P + e.x);
        if (pb == e.y) pb = ld_relaxed(P + e.y);
        ans[i] = find_halve_quiet_from(P, e.x, pa) == find_halve_quiet_from(P, e.y, pb) ? 1 : 0;
        return;
    }
#endif
    pdl_wait();                                   // ... and this one starts after the previous kernel
    if (i >= n_q) return;
    const uint2 e = q[i];
    const uint32_t ra = query_find<FIND>(P, e.x);
    const uint32_t rb = query_find<FIND>(P, e.y);
    ans[i] = ra == rb ? 1 : 0;
}

// Wait-free type (1) batch (Theorem P:2663-2682): inserts and
// queries of the batch in ONE kernel, interleaved over the threads so that
// they really overlap.  A query is linearizable against the concurrent
// unions: it finds ra, then rb; if they differ and ra is STILL a root after
// rb was found, a and b were in different trees at the moment rb was read
// (ra was a root throughout), so "0" is correct at that point; otherwise it
// retries.  All parent reads are device-scope relaxed loads (reading R5).
template <int MODE>
__global__ void __launch_bounds__(kBlock) k_mixed(uint32_t* P, const uint2* __restrict__ ins, int64_t n_ins,
                                                  const uint2* __restrict__ q, int64_t n_q, uint8_t* __restrict__ ans)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t both = 2 * min(n_ins, n_q);
    bool is_ins;
    int64_t i;
    if (t < both) {                      // alternate insert / query while both remain
        is_ins = (t & 1) == 0;
        i = t >> 1;
    } else {
        i = both / 2 + (t - both);
        is_ins = n_ins > n_q;
        if (i >= (is_ins ? n_ins : n_q)) return;
    }
    if (is_ins) {
        const uint2 e = ins[i];
        link<MODE>(P, e.x, e.y, NoForest{});
        return;
    }
    const uint2 e = q[i];
    while (true) {
        // FindAtomicSplit (safe next to concurrent hooks): each returned value was a root
        // when it was read, which is all the linearization argument needs, and chains stay short
        const uint32_t ra = find_split(P, e.x);
        const uint32_t rb = find_split(P, e.y);
        if (ra == rb) { ans[i] = 1; return; }
        if (ld_relaxed(P + ra) == ra) { ans[i] = 0; return; }
    }
}

// Small batches (the latency regime of the paper's Table 5, batch 10..1000):
// ONE CTA applies all inserts, passes a block barrier -- the type (3)
// insert/query barrier, P:986-993 -- and answers all queries: one launch
// instead of two.  The hooks are device-scope CAS and the query reads are
// relaxed device-scope loads, so the barrier also orders their visibility.
constexpr int64_t kSmallBatch = 256;      // one cc_incr_batch call: above this, two PDL kernels
constexpr int64_t kSmallBatches = 8192;   // cc_incr_batches: every batch up to this -> one CTA walks them all

template <int MODE, int FIND>
__global__ void __launch_bounds__(1024) k_small_batch(uint32_t* P, const uint2* __restrict__ ins, int64_t n_ins,
                                                      const uint2* __restrict__ q, int64_t n_q,
                                                      uint8_t* __restrict__ ans)
{
    pdl_trigger();                                // the next batch's kernel may be scheduled now
    pdl_wait();                                   // ... and this one starts after the previous kernel
    for (int64_t i = threadIdx.x; i < n_ins; i += blockDim.x) {
        const uint2 e = ins[i];
        link<MODE>(P, e.x, e.y, NoForest{});
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n_q; i += blockDim.x) {
        const uint2 e = q[i];
        const uint32_t ra = query_find<FIND>(P, e.x);
        const uint32_t rb = query_find<FIND>(P, e.y);
        ans[i] = ra == rb ? 1 : 0;
    }
}

// The multi-batch form of k_small_batch: one CTA walks the whole batch sequence.
template <int MODE, int FIND>
__global__ void __launch_bounds__(1024) k_small_batches(uint32_t* P, const uint2* __restrict__ ins,
                                                        const uint2* __restrict__ q, uint8_t* __restrict__ ans,
                                                        const int64_t* __restrict__ oi, const int64_t* __restrict__ oq,
                                                        int64_t nb)
{
    for (int64_t b = 0; b < nb; ++b) {
        for (int64_t i = oi[b] + threadIdx.x; i < oi[b + 1]; i += blockDim.x) {
            const uint2 e = ins[i];
            link<MODE>(P, e.x, e.y, NoForest{});
        }
        __syncthreads();                         // the batch's insert/query barrier
        for (int64_t i = oq[b] + threadIdx.x; i < oq[b + 1]; i += blockDim.x) {
            const uint2 e = q[i];
            const uint32_t ra = query_find<FIND>(P, e.x);
            const uint32_t rb = query_find<FIND>(P, e.y);
            ans[i] = ra == rb ? 1 : 0;
        }
        __syncthreads();                         // batch b+1 starts after batch b's queries
    }
}

__global__ void k_check_ids(const uint32_t* ids, int64_t count, uint32_t n, unsigned int* err)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
        if (ids[i] >= n) atomicOr(err, 1u);
}

// labels[v] = root(v); P itself is compressed too (no hook runs concurrently).
__global__ void __launch_bounds__(kBlock) k_labels(uint32_t* P, uint32_t n, uint32_t* out)
{
    const uint64_t v64 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v64 >= n) return;
    const uint32_t v = (uint32_t)v64;
    const uint32_t p = P[v];
    uint32_t r = p;
    if (p != v) {
        uint32_t q = P[r];
        while (q != r) { r = q; q = P[r]; }
        if (r != p) P[v] = r;
    }
    out[v] = r;
}

static unsigned nblocks(int64_t count) { return (unsigned)((count + kBlock - 1) / kBlock); }

// pdl: launch the batch's first kernel with PDL (false: a full dependency on the stream's
// previous work).  pre: the kernels may read their pairs (and first parents) BEFORE their PDL
// wait -- only when the pairs were written before the start of a full-dependency kernel that
// precedes them in this stream (cc_incr_batches: its first kernel is launched without PDL), so
// that the pre-wait reads see them.
static cc_status insert_query(cc_incr* h, const uint32_t* ins, int64_t n_ins, const uint32_t* qs, int64_t n_q,
                              uint8_t* ans, cudaStream_t s, bool pdl = true, bool pre = false)
{
    if (h->flags & CC_FLAG_VALIDATE) {
        unsigned int* err = nullptr;
        CC_CUDA_TRY(scratch_alloc((void**)&err, sizeof(unsigned int), s));
        CC_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
        if (n_ins) {
            k_check_ids<<<grid_blocks(4), kBlock, 0, s>>>(ins, 2 * n_ins, h->n, err);
            CC_LAUNCH_CHECK("k_check_ids");
        }
        if (n_q) {
            k_check_ids<<<grid_blocks(4), kBlock, 0, s>>>(qs, 2 * n_q, h->n, err);
            CC_LAUNCH_CHECK("k_check_ids");
        }
        unsigned int e = 0;
        CC_CUDA_TRY(cudaMemcpyAsync(&e, err, sizeof(e), cudaMemcpyDeviceToHost, s));
        CC_CUDA_TRY(cudaStreamSynchronize(s));
        scratch_free(err, s);
        if (e) {
            set_error("cc_incr_batch: vertex id >= n");
            return CC_EINVAL;
        }
    }
    if (n_ins + n_q <= kSmallBatch && !(h->flags & CC_FLAG_WAIT_FREE)) {
        const uint2* e = reinterpret_cast<const uint2*>(ins);
        const uint2* q = reinterpret_cast<const uint2*>(qs);
        const int find = (h->flags & CC_FLAG_FIND_SPLIT) ? 1 : (h->flags & CC_FLAG_FIND_NAIVE) ? 2 : 0;
        // one warp per 32 operations, up to 1024 threads: a 10-op batch is one warp
        const int64_t mx = std::max(n_ins, n_q);
        const unsigned thr = (unsigned)std::min<int64_t>(1024, std::max<int64_t>(32, (mx + 31) / 32 * 32));
        const int mode = (h->flags & CC_FLAG_UF_ASYNC) ? 2 : (h->flags & CC_FLAG_HALVE) ? 1 : 0;
        void (*kern)(uint32_t*, const uint2*, int64_t, const uint2*, int64_t, uint8_t*) =
            mode == 2 ? (find == 1 ? k_small_batch<2, 1> : find == 2 ? k_small_batch<2, 2> : k_small_batch<2, 0>)
            : mode == 1 ? (find == 1 ? k_small_batch<1, 1> : find == 2 ? k_small_batch<1, 2> : k_small_batch<1, 0>)
                        : (find == 1 ? k_small_batch<0, 1> : find == 2 ? k_small_batch<0, 2> : k_small_batch<0, 0>);
        CC_CUDA_TRY(launch_pdl_if(pdl, kern, 1, thr, s, h->P, e, n_ins, q, n_q, ans));
        CC_LAUNCH_CHECK("k_small_batch");
        return CC_OK;
    }
    if ((h->flags & CC_FLAG_WAIT_FREE) && n_ins > 0 && n_q > 0) {
        const uint2* e = reinterpret_cast<const uint2*>(ins);
        const uint2* q = reinterpret_cast<const uint2*>(qs);
        const unsigned nb = nblocks(n_ins + n_q);
        if (h->flags & CC_FLAG_UF_ASYNC) k_mixed<2><<<nb, kBlock, 0, s>>>(h->P, e, n_ins, q, n_q, ans);
        else if (h->flags & CC_FLAG_HALVE) k_mixed<1><<<nb, kBlock, 0, s>>>(h->P, e, n_ins, q, n_q, ans);
        else k_mixed<0><<<nb, kBlock, 0, s>>>(h->P, e, n_ins, q, n_q, ans);
        CC_LAUNCH_CHECK("k_mixed");
        return CC_OK;
    }
    if (n_ins > 0) {
        const uint2* e = reinterpret_cast<const uint2*>(ins);
        cudaError_t le;
        const unsigned nbi = (unsigned)((n_ins + kInsBlock - 1) / kInsBlock);
        if (h->flags & CC_FLAG_UF_ASYNC) le = launch_pdl_if(pdl, k_insert<2>, nbi, kInsBlock, s, h->P, e, n_ins, pre);
        else if (h->flags & CC_FLAG_HALVE) le = launch_pdl_if(pdl, k_insert<1>, nbi, kInsBlock, s, h->P, e, n_ins, pre);
        // one link per thread: measured faster on C5 than the static path's lane-refill
        // kernel (28.0 vs 26.1 G ops/s) and than 2 or 4 links per thread with their
        // first parent reads batched (26.3 / 24.4 vs 28.4 G ops/s: a quarter of the
        // threads, each walking its links one after another)
        else le = launch_pdl_if(pdl, k_insert<0>, nbi, kInsBlock, s, h->P, e, n_ins, pre);
        CC_CUDA_TRY(le);
        CC_LAUNCH_CHECK("k_insert");
    }
    // ---- kernel boundary: the insert/query barrier of type (3) ----
    if (n_q > 0) {
        const uint2* q = reinterpret_cast<const uint2*>(qs);
        cudaError_t le;
        const unsigned nbq = (unsigned)((n_q + kQryBlock - 1) / kQryBlock);
        if (h->flags & CC_FLAG_FIND_SPLIT) le = launch_pdl_if(pdl || n_ins > 0, k_query<1>, nbq, kQryBlock, s, h->P, q, n_q, ans, pre);
        else if (h->flags & CC_FLAG_FIND_NAIVE) le = launch_pdl_if(pdl || n_ins > 0, k_query<2>, nbq, kQryBlock, s, h->P, q, n_q, ans, pre);
        else le = launch_pdl_if(pdl || n_ins > 0, k_query<0>, nbq, kQryBlock, s, h->P, q, n_q, ans, pre);
        CC_CUDA_TRY(le);
        CC_LAUNCH_CHECK("k_query");
    }
    return CC_OK;
}

}  // namespace ccb

using namespace ccb;

extern "C" {

cc_status cc_incr_create(uint32_t n, const cc_opts* opts, void* stream, cc_incr** out)
{
    if (!out) { set_error("out is NULL"); return CC_EINVAL; }
    *out = nullptr;
    if (n > 0xFFFFFFFEu) { set_error("n > 0xFFFFFFFE"); return CC_ERANGE; }
    cudaStream_t s = (cudaStream_t)stream;
    cc_incr* h = new (std::nothrow) cc_incr{};
    if (!h) return CC_ENOMEM;
    h->n = n;
    h->flags = opts ? opts->flags : 0u;
    h->last = s;
    cudaGetDevice(&h->device);
    cudaError_t e = cudaMalloc((void**)&h->P, sizeof(uint32_t) * std::max<size_t>(n, 1));
    if (e != cudaSuccess) {
        delete h;
        return cuda_fail(e, "cc_incr_create: cudaMalloc");
    }
    if (n) {
        k_iota<<<nblocks(n), kBlock, 0, s>>>(h->P, n);
        count_launch();
        e = cudaGetLastError();
        if (e != cudaSuccess) {
            cudaFree(h->P);
            delete h;
            return cuda_fail(e, "k_iota");
        }
    }
    *out = h;
    return CC_OK;
}

cc_status cc_incr_batch(cc_incr* h, const uint32_t* inserts, int64_t n_ins, const uint32_t* queries, int64_t n_q,
                        uint8_t* answers, void* stream)
{
    if (!h) { set_error("handle is NULL"); return CC_EINVAL; }
    if (n_ins < 0 || n_q < 0) { set_error("negative count"); return CC_EINVAL; }
    if ((n_ins && !inserts) || (n_q && (!queries || !answers))) { set_error("NULL array"); return CC_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    if (h->n == 0) {
        if (n_ins || n_q) { set_error("ids >= n = 0"); return CC_EINVAL; }
        return CC_OK;
    }
    // device and pinned host arrays are used in place (pinned: zero-copy through
    // UVA); pageable host arrays are staged
    void *a_ins, *a_q, *a_ans;
    const MemKind k_ins = n_ins ? mem_kind(inserts, &a_ins) : MEM_DEVICE;
    const MemKind k_q = n_q ? mem_kind(queries, &a_q) : MEM_DEVICE;
    const MemKind k_ans = n_q ? mem_kind(answers, &a_ans) : MEM_DEVICE;
    if (!n_ins) a_ins = (void*)inserts;
    if (!n_q) a_q = (void*)queries, a_ans = (void*)answers;
    if (k_ins == MEM_DEVICE && k_q == MEM_DEVICE && k_ans == MEM_DEVICE)
        return insert_query(h, inserts, n_ins, queries, n_q, answers, s);
    std::vector<void*> bufs;
    auto release = [&]() { for (void* b : bufs) scratch_free(b, s); };
    const uint32_t* d_ins = (const uint32_t*)a_ins;
    const uint32_t* d_q = (const uint32_t*)a_q;
    uint8_t* d_ans = (uint8_t*)a_ans;
    auto stage_in = [&](const void* host, size_t bytes, void** dev_out) -> cudaError_t {
        cudaError_t e = scratch_alloc(dev_out, bytes, s);
        if (e != cudaSuccess) return e;
        bufs.push_back(*dev_out);
        return host ? cudaMemcpyAsync(*dev_out, host, bytes, cudaMemcpyHostToDevice, s) : cudaSuccess;
    };
    cudaError_t e = cudaSuccess;
    if (k_ins == MEM_PAGEABLE) e = stage_in(inserts, 8 * (size_t)n_ins, (void**)&d_ins);
    if (e == cudaSuccess && k_q == MEM_PAGEABLE) e = stage_in(queries, 8 * (size_t)n_q, (void**)&d_q);
    if (e == cudaSuccess && k_ans == MEM_PAGEABLE) e = stage_in(nullptr, (size_t)n_q, (void**)&d_ans);
    if (e != cudaSuccess) { release(); return cuda_fail(e, "cc_incr_batch: staging"); }
    cc_status rc = insert_query(h, d_ins, n_ins, d_q, n_q, d_ans, s);
    if (rc == CC_OK && k_ans == MEM_PAGEABLE) {
        e = cudaMemcpyAsync(answers, d_ans, (size_t)n_q, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) rc = cuda_fail(e, "cc_incr_batch: answers");
    }
    if (rc == CC_OK) {
        e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) rc = cuda_fail(e, "cc_incr_batch: sync");
    }
    release();
    return rc;
}

}  // extern "C"

namespace ccb {
// Double-buffered staging of pinned host batches (see cc_incr_batches).  The copy
// stream waits for the compute stream to release a buffer (event `freed`), the
// compute stream waits for its copy (event `ready`); only inserts / queries that
// live in pinned host memory are staged.
cc_status pipelined_batches(cc_incr* h, int64_t nb, const std::vector<int64_t>& oi, const std::vector<int64_t>& oq,
                            const int64_t* ins_counts, const int64_t* q_counts, const uint32_t* ins, bool stage_i,
                            const uint32_t* qs, bool stage_q, uint8_t* ans, cudaStream_t s)
{
    int64_t mi = 0, mq = 0;
    for (int64_t b = 0; b < nb; ++b) {
        mi = std::max(mi, ins_counts[b]);
        mq = std::max(mq, q_counts[b]);
    }
    uint32_t* buf_i[2] = {nullptr, nullptr};
    uint32_t* buf_q[2] = {nullptr, nullptr};
    cudaStream_t cs = nullptr;
    cudaEvent_t ready[2] = {}, freed[2] = {};
    cc_status rc = CC_OK;
    auto body = [&]() -> cc_status {
        CC_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k) {
            if (stage_i && mi) CC_CUDA_TRY(scratch_alloc((void**)&buf_i[k], 8 * (size_t)mi, s));
            if (stage_q && mq) CC_CUDA_TRY(scratch_alloc((void**)&buf_q[k], 8 * (size_t)mq, s));
            CC_CUDA_TRY(cudaEventCreateWithFlags(&ready[k], cudaEventDisableTiming));
            CC_CUDA_TRY(cudaEventCreateWithFlags(&freed[k], cudaEventDisableTiming));
            CC_CUDA_TRY(cudaEventRecord(freed[k], s));   // buffers start free (after their allocation)
        }
        bool launched = false;
        for (int64_t b = 0; b < nb; ++b) {
            const int k = (int)(b & 1);
            const uint32_t* pi = ins + 2 * oi[b];
            const uint32_t* pq = qs + 2 * oq[b];
            CC_CUDA_TRY(cudaStreamWaitEvent(cs, freed[k], 0));
            if (stage_i && ins_counts[b]) {
                CC_CUDA_TRY(cudaMemcpyAsync(buf_i[k], pi, 8 * (size_t)ins_counts[b], cudaMemcpyHostToDevice, cs));
                pi = buf_i[k];
            }
            if (stage_q && q_counts[b]) {
                CC_CUDA_TRY(cudaMemcpyAsync(buf_q[k], pq, 8 * (size_t)q_counts[b], cudaMemcpyHostToDevice, cs));
                pq = buf_q[k];
            }
            CC_CUDA_TRY(cudaEventRecord(ready[k], cs));
            CC_CUDA_TRY(cudaStreamWaitEvent(s, ready[k], 0));
            // PDL (and the pre-wait reads it enables) once a non-empty batch has launched a kernel
            cc_status r = insert_query(h, pi, ins_counts[b], pq, q_counts[b], ans + oq[b], s, launched, true);
            launched |= ins_counts[b] + q_counts[b] > 0;
            if (r) return r;
            CC_CUDA_TRY(cudaEventRecord(freed[k], s));
        }
        return CC_OK;
    };
    rc = body();
    // the staging buffers are stream-ordered on s (freed after the last kernel that reads
    // them); the copy stream is idle once s has passed the last `ready` it waited on
    for (int k = 0; k < 2; ++k) {
        scratch_free(buf_i[k], s);
        scratch_free(buf_q[k], s);
    }
    cudaStreamSynchronize(s);
    for (int k = 0; k < 2; ++k) {
        if (ready[k]) cudaEventDestroy(ready[k]);
        if (freed[k]) cudaEventDestroy(freed[k]);
    }
    if (cs) cudaStreamDestroy(cs);
    return rc;
}
}  // namespace ccb

extern "C" {

cc_status cc_incr_batches(cc_incr* h, int64_t nb, const int64_t* ins_counts, const uint32_t* inserts,
                          const int64_t* q_counts, const uint32_t* queries, uint8_t* answers, void* stream)
{
    if (!h) { set_error("handle is NULL"); return CC_EINVAL; }
    if (nb < 0 || (nb > 0 && (!ins_counts || !q_counts))) { set_error("bad batch counts"); return CC_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    std::vector<int64_t> oi(nb + 1, 0), oq(nb + 1, 0);
    int64_t maxops = 0;
    for (int64_t b = 0; b < nb; ++b) {
        if (ins_counts[b] < 0 || q_counts[b] < 0) { set_error("negative count"); return CC_EINVAL; }
        oi[b + 1] = oi[b] + ins_counts[b];
        oq[b + 1] = oq[b] + q_counts[b];
        maxops = std::max(maxops, ins_counts[b] + q_counts[b]);
    }
    const int64_t tot_i = oi[nb], tot_q = oq[nb];
    if ((tot_i && !inserts) || (tot_q && (!queries || !answers))) { set_error("NULL array"); return CC_EINVAL; }
    if (h->n == 0) {
        if (tot_i || tot_q) { set_error("ids >= n = 0"); return CC_EINVAL; }
        return CC_OK;
    }
    void *a_ins = (void*)inserts, *a_q = (void*)queries, *a_ans = (void*)answers;
    const MemKind k_ins = tot_i ? mem_kind(inserts, &a_ins) : MEM_DEVICE;
    const MemKind k_q = tot_q ? mem_kind(queries, &a_q) : MEM_DEVICE;
    const MemKind k_ans = tot_q ? mem_kind(answers, &a_ans) : MEM_DEVICE;
    if (k_ins == MEM_PAGEABLE || k_q == MEM_PAGEABLE || k_ans == MEM_PAGEABLE) {
        // pageable host arrays: fall back to one staged cc_incr_batch per batch
        for (int64_t b = 0; b < nb; ++b) {
            const cc_status rc = cc_incr_batch(h, inserts + 2 * oi[b], ins_counts[b], queries + 2 * oq[b], q_counts[b],
                                               answers + oq[b], stream);
            if (rc) return rc;
        }
        return CC_OK;
    }
    const uint32_t* d_ins = (const uint32_t*)a_ins;
    const uint32_t* d_q = (const uint32_t*)a_q;
    uint8_t* d_ans = (uint8_t*)a_ans;
    if (h->flags & CC_FLAG_VALIDATE) {
        unsigned int* err = nullptr;
        CC_CUDA_TRY(scratch_alloc((void**)&err, sizeof(unsigned int), s));
        CC_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
        if (tot_i) { k_check_ids<<<grid_blocks(4), kBlock, 0, s>>>(d_ins, 2 * tot_i, h->n, err); CC_LAUNCH_CHECK("k_check_ids"); }
        if (tot_q) { k_check_ids<<<grid_blocks(4), kBlock, 0, s>>>(d_q, 2 * tot_q, h->n, err); CC_LAUNCH_CHECK("k_check_ids"); }
        unsigned int e = 0;
        CC_CUDA_TRY(cudaMemcpyAsync(&e, err, sizeof(e), cudaMemcpyDeviceToHost, s));
        CC_CUDA_TRY(cudaStreamSynchronize(s));
        scratch_free(err, s);
        if (e) { set_error("cc_incr_batches: vertex id >= n"); return CC_EINVAL; }
    }
    const bool host = k_ins != MEM_DEVICE || k_q != MEM_DEVICE || k_ans != MEM_DEVICE;
    if (maxops <= kSmallBatches && !(h->flags & CC_FLAG_WAIT_FREE)) {
        int64_t* d_off = nullptr;
        CC_CUDA_TRY(scratch_alloc((void**)&d_off, sizeof(int64_t) * 2 * (size_t)(nb + 1), s));
        std::vector<int64_t> both(oi);
        both.insert(both.end(), oq.begin(), oq.end());
        CC_CUDA_TRY(cudaMemcpyAsync(d_off, both.data(), sizeof(int64_t) * both.size(), cudaMemcpyHostToDevice, s));
        const uint2* e = reinterpret_cast<const uint2*>(d_ins);
        const uint2* q = reinterpret_cast<const uint2*>(d_q);
        const int find = (h->flags & CC_FLAG_FIND_SPLIT) ? 1 : (h->flags & CC_FLAG_FIND_NAIVE) ? 2 : 0;
        const int64_t* po = d_off;
        const int64_t* pq = d_off + nb + 1;
        if (h->flags & CC_FLAG_UF_ASYNC) {
            if (find == 1) k_small_batches<2, 1><<<1, 1024, 0, s>>>(h->P, e, q, d_ans, po, pq, nb);
            else if (find == 2) k_small_batches<2, 2><<<1, 1024, 0, s>>>(h->P, e, q, d_ans, po, pq, nb);
            else k_small_batches<2, 0><<<1, 1024, 0, s>>>(h->P, e, q, d_ans, po, pq, nb);
        } else if (h->flags & CC_FLAG_HALVE) {
            if (find == 1) k_small_batches<1, 1><<<1, 1024, 0, s>>>(h->P, e, q, d_ans, po, pq, nb);
            else if (find == 2) k_small_batches<1, 2><<<1, 1024, 0, s>>>(h->P, e, q, d_ans, po, pq, nb);
            else k_small_batches<1, 0><<<1, 1024, 0, s>>>(h->P, e, q, d_ans, po, pq, nb);
        } else {
            if (find == 1) k_small_batches<0, 1><<<1, 1024, 0, s>>>(h->P, e, q, d_ans, po, pq, nb);
            else if (find == 2) k_small_batches<0, 2><<<1, 1024, 0, s>>>(h->P, e, q, d_ans, po, pq, nb);
            else k_small_batches<0, 0><<<1, 1024, 0, s>>>(h->P, e, q, d_ans, po, pq, nb);
        }
        CC_LAUNCH_CHECK("k_small_batches");
        // the host vector `both` must outlive the async copy: synchronise before returning
        CC_CUDA_TRY(cudaStreamSynchronize(s));
        scratch_free(d_off, s);
        return CC_OK;
    }
    const uint32_t saved = h->flags;
    h->flags &= ~CC_FLAG_VALIDATE;                       // ids already checked above
    cc_status rc = CC_OK;
    if ((k_ins == MEM_PINNED || k_q == MEM_PINNED) && nb > 1) {
        // Pinned host batches: DMA each batch's pairs into one of two device staging
        // buffers on a copy stream while the previous batch computes (double buffering);
        // read in place over PCIe by the kernels instead, every batch waited for its own
        // pairs (C5: 40 GB/s effective).  Answers are still written to the host in place.
        rc = pipelined_batches(h, nb, oi, oq, ins_counts, q_counts, d_ins, k_ins == MEM_PINNED, d_q,
                               k_q == MEM_PINNED, d_ans, s);
    } else {
        // the first non-empty batch's first kernel is an ordinary launch (all earlier work of the
        // stream, which wrote the pairs, complete and visible); PDL and pre-wait reads after it
        bool launched = false;
        for (int64_t b = 0; b < nb && rc == CC_OK; ++b) {
            rc = insert_query(h, d_ins + 2 * oi[b], ins_counts[b], d_q + 2 * oq[b], q_counts[b], d_ans + oq[b], s,
                              launched, true);
            launched |= ins_counts[b] + q_counts[b] > 0;
        }
    }
    h->flags = saved;
    if (rc == CC_OK && host) CC_CUDA_TRY(cudaStreamSynchronize(s));
    return rc;
}

cc_status cc_incr_labels(cc_incr* h, uint32_t* labels, void* stream)
{
    if (!h) { set_error("handle is NULL"); return CC_EINVAL; }
    if (h->n == 0) return CC_OK;
    if (!labels) { set_error("labels is NULL"); return CC_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    h->last = s;
    void* a_lab;
    const MemKind kl = mem_kind(labels, &a_lab);
    uint32_t* d = (uint32_t*)a_lab;
    if (kl == MEM_PAGEABLE) CC_CUDA_TRY(scratch_alloc((void**)&d, sizeof(uint32_t) * h->n, s));
    k_labels<<<nblocks(h->n), kBlock, 0, s>>>(h->P, h->n, d);
    CC_LAUNCH_CHECK("k_labels");
    if (kl == MEM_PAGEABLE) {
        CC_CUDA_TRY(cudaMemcpyAsync(labels, d, sizeof(uint32_t) * h->n, cudaMemcpyDeviceToHost, s));
        scratch_free(d, s);
    }
    if (kl != MEM_DEVICE) CC_CUDA_TRY(cudaStreamSynchronize(s));
    return CC_OK;
}

void cc_incr_destroy(cc_incr* h)
{
    if (!h) return;
    cudaStreamSynchronize(h->last);
    cudaFree(h->P);
    delete h;
}

uint32_t cc_incr_num_vertices(const cc_incr* h) { return h ? h->n : 0u; }

}  // extern "C"
