// cc_abi.cu -- the extern "C" boundary of libcc.so (include/cc.h).
//
// Argument checks, host-buffer staging, error mapping.  The compute is in
// cc_static.cu (cc_labels, cc_spanning_forest) and cc_incr.cu (cc_incr_*).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>
#include <string>

#include "cc_internal.h"

namespace ccb {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_err;

void set_error(const std::string& msg) { t_err = msg; }

cc_status cuda_fail(cudaError_t e, const char* where)
{
    t_err = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    if (e == cudaErrorMemoryAllocation) return CC_ENOMEM;
    return CC_ECUDA;
}

int num_sms()
{
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

// Test hook (cc_bench_set_grid): when non-zero, every grid-strided
// ("persistent") kernel launches exactly this many blocks instead of a
// multiple of the SM count.  Results must not depend on it.
std::atomic<unsigned> g_grid_override{0};

unsigned grid_blocks(unsigned per_sm)
{
    const unsigned o = g_grid_override.load(std::memory_order_relaxed);
    return o ? o : (unsigned)num_sms() * per_sm;
}

unsigned resident_blocks(const void* kernel, int block)
{
    const unsigned o = g_grid_override.load(std::memory_order_relaxed);
    if (o) return o;
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, int>, int>> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const std::pair<const void*, int> key{kernel, block * 64 + dev};
    {
        std::lock_guard<std::mutex> g(mu);
        for (auto& e : cache)
            if (e.first == key) return (unsigned)e.second;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
    }
    const int g = per_sm * num_sms();
    std::lock_guard<std::mutex> lk(mu);
    cache.push_back({key, g});
    return (unsigned)g;
}

bool is_device_ptr(const void* p)
{
    if (!p) return true;                   // NULL: nothing to stage
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

MemKind mem_kind(const void* p, void** dev_alias)
{
    if (dev_alias) *dev_alias = const_cast<void*>(p);
    if (!p) return MEM_DEVICE;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return MEM_PAGEABLE;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return MEM_DEVICE;
    if (a.type == cudaMemoryTypeHost && a.devicePointer) {
        if (dev_alias) *dev_alias = a.devicePointer;
        return MEM_PINNED;
    }
    return MEM_PAGEABLE;
}

static void init_pool_once()
{
    static std::once_flag flag[64];
    int dev = 0;
    cudaGetDevice(&dev);
    std::call_once(flag[dev & 63], [dev]() {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;          // keep freed scratch cached across calls
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
}

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s)
{
    init_pool_once();
    return cudaMallocAsync(p, std::max<size_t>(bytes, 16), s);
}

void scratch_free(void* p, cudaStream_t s)
{
    if (p) cudaFreeAsync(p, s);
}

// ---- host staging -----------------------------------------------------------
struct Stage {
    cudaStream_t s;
    std::vector<void*> bufs;
    ~Stage()
    {
        for (void* b : bufs) scratch_free(b, s);
    }
    template <class T>
    cudaError_t in(const T* host, size_t count, T** dev)
    {
        void* d = nullptr;
        cudaError_t e = scratch_alloc(&d, sizeof(T) * std::max<size_t>(count, 1), s);
        if (e != cudaSuccess) return e;
        bufs.push_back(d);
        *dev = (T*)d;
        if (host && count) return cudaMemcpyAsync(d, host, sizeof(T) * count, cudaMemcpyHostToDevice, s);
        return cudaSuccess;
    }
};

static cc_opts resolve(const cc_opts* o)
{
    cc_opts r;
    cc_opts_default(&r);
    if (o) r = *o;
    if (r.samples == 0) r.samples = 1024;
    return r;
}

static cc_status check_graph_args(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m,
                                  const cc_opts& o)
{
    if (n > 0xFFFFFFFEu) { set_error("n > 0xFFFFFFFE"); return CC_ERANGE; }
    if (m < 0) { set_error("m < 0"); return CC_EINVAL; }
    if (o.kout_k > 64) { set_error("kout_k > 64"); return CC_ERANGE; }
    if (o.kout_variant > CC_VARIANT_PURE) { set_error("unknown kout_variant"); return CC_EINVAL; }
    if (o.samples > 2048) { set_error("samples > 2048"); return CC_ERANGE; }
    if (n > 0 && !off) { set_error("offsets is NULL"); return CC_EINVAL; }
    if (m > 0 && !adj) { set_error("adj is NULL"); return CC_EINVAL; }
    return CC_OK;
}

}  // namespace ccb

using namespace ccb;

extern "C" {

void cc_opts_default(cc_opts* o)
{
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->kout_k = 2;
    o->kout_variant = CC_VARIANT_AFFOREST;
    o->seed = 0;
    o->samples = 1024;
    o->flags = 0;
}

const char* cc_status_str(cc_status s)
{
    switch (s) {
    case CC_OK: return "CC_OK";
    case CC_EINVAL: return "CC_EINVAL";
    case CC_ERANGE: return "CC_ERANGE";
    case CC_ENOMEM: return "CC_ENOMEM";
    case CC_ECUDA: return "CC_ECUDA";
    default: return "CC_UNKNOWN";
    }
}

const char* cc_last_error(void) { return t_err.c_str(); }

const char* cc_version(void) { return "cc-b200 0.1 (sm_100a)"; }

size_t cc_workspace_bytes(uint32_t n, int64_t m, uint32_t kout_k, int op)
{
    const size_t N = n, M = m < 0 ? 0 : (size_t)m, K = kout_k;
    const size_t nw = (N + 31) / 32, ntile = (N + 2047) / 2048, nfb = (N + 4095) / 4096;
    if (op == 2) return 64 + 4 * N;                             // the handle's parent array + flags
    if (op == 3) {
        // cc_amsf (an ESTIMATE: the bucket count depends on eps and the weight range; sized for
        // eps = 0.25-like counts): P, weight range x2, activation bucket, order, 2 carry lists,
        // index ids (4 B each), forest slots (8 B) + weights (4 B), long-list pieces, the bucket
        // index (<= 4 B per entry + per-list starts, 128 buckets), bucket starts; plus the
        // staging of pageable host inputs
        return 64 + 4 * N * 8 + 12 * N + 8 * (M / 2048 + std::min<size_t>(N, M / 2048 + 1) + 1) + 4 * M +
               4 * 129 * (M / 257 + 1) + 16 * (M / 257 + 1) + 8 * 4096 + (8 * (N + 1) + 8 * M + 12 * N + 24);
    }
    // cc_labels / cc_spanning_forest: an UPPER BOUND, the sum over every flag combination's
    // allocations (cc_static.cu run(), cc_abi.cu staging):
    size_t b = 64                                   // control block
               + 4 * nw                             // finish bitmap
               + 4 * std::max(N, 4 * ntile)         // finish candidate queue (= relabel chunk queue)
               + 8 * K * std::min(N, M)             // pending sampled links
               + 4 * std::min(N, M / 4096 + 1)      // big-list queue
               + 33 * ntile                         // warp summaries (8 x 4 B) + hook flag per tile
               + 4 * N                              // parent array when labels are not device memory
               + 8 * (N + 1) + 4 * M + 4 * N        // staging of pageable offsets / adjacency / labels
               + 8 * nw + 8 * std::min(N, M) + 12 * (nw / 4096 + 1) + 8     // CC_FLAG_CONTRACT
               + 12 * N + 8 * (N / 4096 + 1) + 8 + 8 * M + 4 * nw + 4       // FINISH_SV / CRFA edge list
               + 8 * (M / 4096 + 1) + 8                                     // ... and its long-list pieces
               + 2 * (op == 1 ? 16 : 8) * M + 16;                           // CRFA's two edge buffers
    if (op == 1) b += 8 * N + 12 * nfb             // forest slots + Filter status words
                      + 8 * N + 8;                  // staging of pageable edges / num_edges
    return b;
}

// Array arguments: device memory is used in place; pinned host memory is used
// in place too (zero-copy through UVA: the kernels read only the offsets, the
// sampled list heads and the finish candidates' lists, and H6 writes the
// labels straight into it); pageable host memory is staged through scratch.
cc_status cc_labels(const int64_t* offsets, const uint32_t* adj, uint32_t n, int64_t m, uint32_t* labels,
                    const cc_opts* opts, void* stream)
{
    const cc_opts o = resolve(opts);
    cc_status rc = check_graph_args(offsets, adj, n, m, o);
    if (rc) return rc;
    if (n == 0) return CC_OK;
    if (!labels) { set_error("labels is NULL"); return CC_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    void *a_off, *a_adj, *a_lab;
    const MemKind k_off = mem_kind(offsets, &a_off), k_adj = mem_kind(adj, &a_adj), k_lab = mem_kind(labels, &a_lab);
    Stage st{s, {}};
    const int64_t* d_off = (const int64_t*)a_off;
    const uint32_t* d_adj = (const uint32_t*)a_adj;
    if (k_off == MEM_PAGEABLE) CC_CUDA_TRY(st.in(offsets, (size_t)n + 1, (int64_t**)&d_off));
    if (k_adj == MEM_PAGEABLE) CC_CUDA_TRY(st.in(adj, (size_t)m, (uint32_t**)&d_adj));
    if (o.flags & CC_FLAG_VALIDATE) {
        rc = validate_csr(d_off, d_adj, n, m, s);
        if (rc) return rc;
    }
    // the parent array must be device memory: the caller's labels if they are, else scratch
    uint32_t* P = k_lab == MEM_DEVICE ? labels : nullptr;
    uint32_t* out = k_lab == MEM_DEVICE ? labels : (k_lab == MEM_PINNED ? (uint32_t*)a_lab : nullptr);
    uint32_t* staged = nullptr;
    if (k_lab == MEM_PAGEABLE) {
        CC_CUDA_TRY(st.in((const uint32_t*)nullptr, (size_t)n, &staged));
        out = staged;
    }
    rc = static_pipeline(d_off, d_adj, n, m, P, out, nullptr, nullptr, false, o, s);
    if (rc) return rc;
    if (staged) CC_CUDA_TRY(cudaMemcpyAsync(labels, staged, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, s));
    if (k_off != MEM_DEVICE || k_adj != MEM_DEVICE || k_lab != MEM_DEVICE) CC_CUDA_TRY(cudaStreamSynchronize(s));
    return CC_OK;
}

cc_status cc_spanning_forest(const int64_t* offsets, const uint32_t* adj, uint32_t n, int64_t m, uint32_t* edges,
                             int64_t* num_edges, uint32_t* labels, const cc_opts* opts, void* stream)
{
    const cc_opts o = resolve(opts);
    cc_status rc = check_graph_args(offsets, adj, n, m, o);
    if (rc) return rc;
    if (!num_edges) { set_error("num_edges is NULL"); return CC_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    void *a_off, *a_adj, *a_edges, *a_ne, *a_lab;
    const MemKind k_ne = mem_kind(num_edges, &a_ne);
    if (n == 0) {
        if (k_ne == MEM_DEVICE) CC_CUDA_TRY(cudaMemsetAsync(num_edges, 0, sizeof(int64_t), s));
        else *num_edges = 0;
        return CC_OK;
    }
    if (!edges) { set_error("edges is NULL"); return CC_EINVAL; }
    const MemKind k_off = mem_kind(offsets, &a_off), k_adj = mem_kind(adj, &a_adj);
    const MemKind k_edges = mem_kind(edges, &a_edges), k_lab = mem_kind(labels, &a_lab);
    Stage st{s, {}};
    const int64_t* d_off = (const int64_t*)a_off;
    const uint32_t* d_adj = (const uint32_t*)a_adj;
    uint32_t* d_edges = (uint32_t*)a_edges;
    int64_t* d_ne = (int64_t*)a_ne;
    if (k_off == MEM_PAGEABLE) CC_CUDA_TRY(st.in(offsets, (size_t)n + 1, (int64_t**)&d_off));
    if (k_adj == MEM_PAGEABLE) CC_CUDA_TRY(st.in(adj, (size_t)m, (uint32_t**)&d_adj));
    if (k_edges == MEM_PAGEABLE) CC_CUDA_TRY(st.in((const uint32_t*)nullptr, 2 * (size_t)n, &d_edges));
    if (k_ne == MEM_PAGEABLE) CC_CUDA_TRY(st.in((const int64_t*)nullptr, 1, &d_ne));
    if (o.flags & CC_FLAG_VALIDATE) {
        rc = validate_csr(d_off, d_adj, n, m, s);
        if (rc) return rc;
    }
    uint32_t* P = (labels && k_lab == MEM_DEVICE) ? labels : nullptr;
    uint32_t* out = labels ? (k_lab == MEM_PAGEABLE ? nullptr : (uint32_t*)a_lab) : nullptr;
    uint32_t* staged = nullptr;
    if (labels && k_lab == MEM_PAGEABLE) {
        CC_CUDA_TRY(st.in((const uint32_t*)nullptr, (size_t)n, &staged));
        out = staged;
    }
    rc = static_pipeline(d_off, d_adj, n, m, P, out, d_edges, d_ne, true, o, s);
    if (rc) return rc;
    const bool host = k_off != MEM_DEVICE || k_adj != MEM_DEVICE || k_edges != MEM_DEVICE || k_ne != MEM_DEVICE ||
                      (labels && k_lab != MEM_DEVICE);
    if (k_edges == MEM_PAGEABLE || k_ne == MEM_PAGEABLE) {
        int64_t ne = 0;
        CC_CUDA_TRY(cudaMemcpyAsync(&ne, d_ne, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CC_CUDA_TRY(cudaStreamSynchronize(s));
        if (k_ne == MEM_PAGEABLE) *num_edges = ne;
        if (k_edges == MEM_PAGEABLE)
            CC_CUDA_TRY(cudaMemcpyAsync(edges, d_edges, sizeof(uint32_t) * 2 * (size_t)ne, cudaMemcpyDeviceToHost, s));
    }
    if (staged) CC_CUDA_TRY(cudaMemcpyAsync(labels, staged, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, s));
    if (host) CC_CUDA_TRY(cudaStreamSynchronize(s));
    return CC_OK;
}

// AMSF-NF-S (include/cc.h).  Host arrays (pinned or pageable) are staged
// through device scratch -- the bucket rounds read every list many times, so
// zero-copy would cross PCIe once per round -- and the outputs copied back.
cc_status cc_amsf(const int64_t* offsets, const uint32_t* adj, const float* w, uint32_t n, int64_t m, double eps,
                  uint32_t* edges, float* edge_w, int64_t* num_edges, double* total, const cc_opts* opts,
                  void* stream)
{
    const cc_opts o = resolve(opts);
    cc_status rc = check_graph_args(offsets, adj, n, m, o);
    if (rc) return rc;
    if (!(eps > 0.0) || !(eps < 1e300)) { set_error("cc_amsf: eps must be > 0 and finite"); return CC_EINVAL; }
    if (!num_edges) { set_error("num_edges is NULL"); return CC_EINVAL; }
    if (n > 0 && !edges) { set_error("edges is NULL"); return CC_EINVAL; }
    if (m > 0 && !w) { set_error("w is NULL"); return CC_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    auto dev = [](const void* p) { return !p || mem_kind(p, nullptr) == MEM_DEVICE; };
    const bool host = !dev(offsets) || !dev(adj) || !dev(w) || !dev(edges) || !dev(edge_w) || !dev(num_edges) ||
                      !dev(total);
    Stage st{s, {}};
    const int64_t* d_off = offsets;
    const uint32_t* d_adj = adj;
    const float* d_w = w;
    uint32_t* d_edges = edges;
    float* d_ew = edge_w;
    int64_t* d_ne = num_edges;
    double* d_tot = total;
    if (!dev(offsets)) CC_CUDA_TRY(st.in(offsets, (size_t)n + 1, (int64_t**)&d_off));
    if (!dev(adj)) CC_CUDA_TRY(st.in(adj, (size_t)m, (uint32_t**)&d_adj));
    if (!dev(w)) CC_CUDA_TRY(st.in(w, (size_t)m, (float**)&d_w));
    if (!dev(edges)) CC_CUDA_TRY(st.in((const uint32_t*)nullptr, 2 * (size_t)std::max<uint32_t>(n, 1), &d_edges));
    if (!dev(edge_w)) CC_CUDA_TRY(st.in((const float*)nullptr, (size_t)std::max<uint32_t>(n, 1), &d_ew));
    if (!dev(num_edges)) CC_CUDA_TRY(st.in((const int64_t*)nullptr, 1, &d_ne));
    if (!dev(total)) CC_CUDA_TRY(st.in((const double*)nullptr, 1, &d_tot));
    if (n == 0) {
        CC_CUDA_TRY(cudaMemsetAsync(d_ne, 0, sizeof(int64_t), s));
        if (d_tot) CC_CUDA_TRY(cudaMemsetAsync(d_tot, 0, sizeof(double), s));
    } else {
        if (o.flags & CC_FLAG_VALIDATE) {
            rc = validate_csr(d_off, d_adj, n, m, s);
            if (rc) return rc;
        }
        rc = amsf_pipeline(d_off, d_adj, d_w, n, m, eps, d_edges, d_ew, d_ne, d_tot, o, s);
        if (rc) return rc;
    }
    if (host) {
        int64_t ne = 0;
        CC_CUDA_TRY(cudaMemcpyAsync(&ne, d_ne, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CC_CUDA_TRY(cudaStreamSynchronize(s));
        if (d_ne != num_edges) *num_edges = ne;
        if (d_edges != edges && ne)
            CC_CUDA_TRY(cudaMemcpyAsync(edges, d_edges, sizeof(uint32_t) * 2 * (size_t)ne, cudaMemcpyDeviceToHost, s));
        if (d_ew != edge_w && ne)
            CC_CUDA_TRY(cudaMemcpyAsync(edge_w, d_ew, sizeof(float) * (size_t)ne, cudaMemcpyDeviceToHost, s));
        if (d_tot != total) CC_CUDA_TRY(cudaMemcpyAsync(total, d_tot, sizeof(double), cudaMemcpyDeviceToHost, s));
        CC_CUDA_TRY(cudaStreamSynchronize(s));
    }
    return CC_OK;
}

}  // extern "C"
