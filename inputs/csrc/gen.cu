// gen.cu -- seeded CUDA generator of the BASELINE.json inputs (inputs/libccgen.so).
//
// NOT part of the method: this builds the synthetic graphs/streams that stand
// in for the paper's datasets, bit-identical to inputs/gen.py (numpy) for the
// same seed (tests/test_gpu_gen.py checks byte equality).  Every draw is
//     mix(seed, stream, i) = splitmix64(seed*GOLD + stream*2^40 + i)  (mod 2^64)
// so the output is independent of the launch configuration.
//
// CSR build: emit both directions of every non-self-loop pair as 64-bit keys
// (u << vb) | v, bucket by the top bits of u (each bucket < 2^31 keys), radix
// sort each bucket (CUB), drop duplicates (CUB), then derive offsets from the
// sorted unique keys.  The caller allocates the final offsets/adj buffers
// after gen_csr_begin() reports n and m.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

namespace {

constexpr uint64_t GOLD = 0x9E3779B97F4A7C15ull;
constexpr uint64_t ER_STREAM = 1, GRID_STREAM = 2, RMAT_STREAM = 3, PERM_STREAM = 4, QUERY_STREAM = 5,
                   WEIGHT_STREAM = 6;
constexpr uint32_t RMAT_T1 = 2448131358u, RMAT_T2 = 3264175144u, RMAT_T3 = 4080218931u;

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x)
{
    uint64_t z = x + GOLD;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t mix(uint64_t seed, uint64_t stream, uint64_t i)
{
    return splitmix64(seed * GOLD + (stream << 40) + i);
}

__host__ __device__ __forceinline__ uint64_t scale_u32(uint64_t x32, uint64_t bound) { return (x32 * bound) >> 32; }

struct Perm {
    uint64_t k[3], c[3], mask;
    uint32_t h;
    __host__ __device__ uint64_t operator()(uint64_t x) const
    {
        for (int i = 0; i < 3; ++i) {
            x ^= x >> h;
            x = (x * k[i] + c[i]) & mask;
        }
        return x;
    }
};

Perm make_perm(uint64_t seed, int s)
{
    Perm p;
    p.mask = (s >= 64) ? ~0ull : ((1ull << s) - 1);
    for (int i = 0; i < 3; ++i) {
        p.k[i] = (mix(seed, PERM_STREAM, i) | 1ull) & p.mask;
        p.c[i] = mix(seed, PERM_STREAM, 3 + i) & p.mask;
    }
    p.h = (uint32_t)((s + 1) / 2);
    return p;
}

__device__ __forceinline__ void rmat_draw_t(uint64_t seed, int s, uint64_t i, uint32_t t1, uint32_t t2, uint32_t t3,
                                            uint64_t* pu, uint64_t* pv)
{
    const uint64_t L = (uint64_t)((s + 1) / 2);
    uint64_t u = 0, v = 0, r = 0;
    for (int l = 0; l < s; ++l) {
        uint32_t x;
        if ((l & 1) == 0) {
            r = mix(seed, RMAT_STREAM, i * L + (uint64_t)(l / 2));
            x = (uint32_t)(r & 0xFFFFFFFFull);
        } else {
            x = (uint32_t)(r >> 32);
        }
        const uint64_t bit = 1ull << (s - 1 - l);
        if (x >= t2) u |= bit;
        if ((x >= t1 && x < t2) || x >= t3) v |= bit;
    }
    *pu = u;
    *pv = v;
}

__device__ __forceinline__ void rmat_draw(uint64_t seed, int s, uint64_t i, uint64_t* pu, uint64_t* pv)
{
    const uint64_t L = (uint64_t)((s + 1) / 2);
    uint64_t u = 0, v = 0, r = 0;
    for (int l = 0; l < s; ++l) {
        uint32_t x;
        if ((l & 1) == 0) {
            r = mix(seed, RMAT_STREAM, i * L + (uint64_t)(l / 2));
            x = (uint32_t)(r & 0xFFFFFFFFull);
        } else {
            x = (uint32_t)(r >> 32);
        }
        const uint64_t bit = 1ull << (s - 1 - l);
        if (x >= RMAT_T2) u |= bit;
        if ((x >= RMAT_T1 && x < RMAT_T2) || x >= RMAT_T3) v |= bit;
    }
    *pu = u;
    *pv = v;
}

enum Kind { KIND_ER = 0, KIND_GRID = 1, KIND_RMAT = 2 };

struct Spec {
    int kind;
    uint64_t seed;
    uint64_t count;     // number of draws / candidates
    uint32_t n;
    // er
    uint64_t n0;
    // grid
    uint64_t rows, cols, p32;
    // rmat
    int scale;
    int permuted;
    Perm perm;
};

// pair (u, v) of draw i; returns false if the draw produces no edge
__device__ __forceinline__ bool draw_pair(const Spec& sp, uint64_t i, uint64_t* u, uint64_t* v)
{
    if (sp.kind == KIND_ER) {
        const uint64_t r = mix(sp.seed, ER_STREAM, i);
        *u = scale_u32(r & 0xFFFFFFFFull, sp.n0);
        *v = scale_u32(r >> 32, sp.n0);
        return *u != *v;
    }
    if (sp.kind == KIND_GRID) {
        if ((mix(sp.seed, GRID_STREAM, i) & 0xFFFFFFFFull) >= sp.p32) return false;
        const uint64_t nh = sp.rows * (sp.cols - 1);
        if (i < nh) {
            const uint64_t r = i / (sp.cols - 1), c = i % (sp.cols - 1);
            *u = r * sp.cols + c;
            *v = *u + 1;
        } else {
            *u = i - nh;
            *v = *u + sp.cols;
        }
        return true;
    }
    rmat_draw(sp.seed, sp.scale, i, u, v);
    if (sp.permuted) {
        *u = sp.perm(*u);
        *v = sp.perm(*v);
    }
    return *u != *v;
}

__global__ void k_count(Spec sp, int vb, int bshift, unsigned long long* bcount)
{
    __shared__ unsigned int sh[1024];
    const int nb = 1 << (vb - bshift);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < sp.count; i += stride) {
        uint64_t u, v;
        if (!draw_pair(sp, i, &u, &v)) continue;
        atomicAdd(&sh[u >> bshift], 1u);
        atomicAdd(&sh[v >> bshift], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
        if (sh[i]) atomicAdd(&bcount[i], (unsigned long long)sh[i]);
}

__global__ void k_scatter(Spec sp, int vb, int bshift, unsigned long long* cursor, uint64_t* keys)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < sp.count; i += stride) {
        uint64_t u, v;
        if (!draw_pair(sp, i, &u, &v)) continue;
        unsigned long long p = atomicAdd(&cursor[u >> bshift], 1ull);
        keys[p] = (u << vb) | v;
        p = atomicAdd(&cursor[v >> bshift], 1ull);
        keys[p] = (v << vb) | u;
    }
}

__global__ void k_offsets(const uint64_t* keys, uint64_t m, int vb, uint32_t n, int64_t* off)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= m; i += stride) {
        // vertices w in (u_{i-1}, u_i] start at i; u_{-1} = -1, u_m = n
        const int64_t ui = i < m ? (int64_t)(keys[i] >> vb) : (int64_t)n;
        const int64_t up = i > 0 ? (int64_t)(keys[i - 1] >> vb) : -1;
        for (int64_t w = up + 1; w <= ui; ++w) off[w] = (int64_t)i;
    }
}

__global__ void k_adj(const uint64_t* keys, uint64_t m, uint64_t vmask, uint32_t* adj)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride)
        adj[i] = (uint32_t)(keys[i] & vmask);
}

__global__ void k_incr(uint64_t seed, int s, Perm perm, uint64_t first, uint64_t n_ins, uint64_t qfirst,
                       uint64_t n_q, uint32_t* ins, uint32_t* qs)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t n = 1ull << s;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_ins + n_q; i += stride) {
        if (i < n_ins) {
            uint64_t u, v;
            rmat_draw(seed, s, first + i, &u, &v);
            ins[2 * i] = (uint32_t)perm(u);
            ins[2 * i + 1] = (uint32_t)perm(v);
        } else {
            const uint64_t j = i - n_ins;
            const uint64_t r = mix(seed, QUERY_STREAM, qfirst + j);
            qs[2 * j] = (uint32_t)scale_u32(r & 0xFFFFFFFFull, n);
            qs[2 * j + 1] = (uint32_t)scale_u32(r >> 32, n);
        }
    }
}

// RMAT draws first .. first+count-1 on 2^s vertices with the thresholds
// t1 = a, t2 = a+b, t3 = a+b+c (fixed point, x 2^32), optionally permuted
__global__ void k_rmat_stream(uint64_t seed, int s, Perm perm, int permuted, uint32_t t1, uint32_t t2, uint32_t t3,
                              uint64_t first, uint64_t count, uint32_t* out)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        uint64_t u, v;
        rmat_draw_t(seed, s, first + i, t1, t2, t3, &u, &v);
        out[2 * i] = (uint32_t)(permuted ? perm(u) : u);
        out[2 * i + 1] = (uint32_t)(permuted ? perm(v) : v);
    }
}

struct State {
    uint64_t* keys = nullptr;
    uint64_t m = 0;
    uint32_t n = 0;
    int vb = 0;
};

constexpr int LN_TERMS = 10;
constexpr double LN2 = 0.6931471805599453;

__device__ __forceinline__ double atanh2(double t)
{
    const double t2 = __dmul_rn(t, t);
    double p = __ddiv_rn(1.0, (double)(2 * LN_TERMS + 1));
    for (int k = LN_TERMS - 1; k >= 0; --k) {
        p = __dmul_rn(p, t2);
        p = __dadd_rn(p, __ddiv_rn(1.0, (double)(2 * k + 1)));
    }
    return __dmul_rn(__dmul_rn(2.0, t), p);
}

__device__ __forceinline__ double neg_ln_fixed(double x)
{
    if (x < 0.5) {
        const uint64_t bits = (uint64_t)__double_as_longlong(x);
        const int64_t e = (int64_t)((bits >> 52) & 0x7FF) - 1023;
        const double mm = __longlong_as_double((long long)((bits & 0x000FFFFFFFFFFFFFull) | (1023ull << 52)));
        const double t = __ddiv_rn(__dsub_rn(mm, 1.0), __dadd_rn(mm, 1.0));
        return -__dadd_rn(__dmul_rn((double)e, LN2), atanh2(t));
    }
    const double d = __dsub_rn(1.0, x);
    return atanh2(__ddiv_rn(d, __dsub_rn(2.0, d)));
}

__global__ void k_weights(const int64_t* off, const uint32_t* adj, uint32_t n, uint64_t m, uint64_t seed, float* w)
{
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = n;                              // src: largest u with off[u] <= e
        while (hi - lo > 1) {
            const uint32_t mid = lo + (hi - lo) / 2;
            if ((uint64_t)off[mid] <= e) lo = mid; else hi = mid;
        }
        const uint64_t a = lo, b = adj[e];
        const uint64_t key = ((a < b ? a : b) << 32) | (a < b ? b : a);
        const uint64_t k = mix(seed, WEIGHT_STREAM, key) >> 12;
        const double u = __dmul_rn(__dadd_rn((double)k, 0.5), 0x1p-52);
        w[e] = __double2float_rn(neg_ln_fixed(u));
    }
}

int bits_for(uint64_t n)
{
    int b = 1;
    while ((1ull << b) < n) ++b;
    return b;
}

int grid_blocks()
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms * 8;
}

#define TRY(x)                                                                            \
    do {                                                                                  \
        cudaError_t _e = (x);                                                             \
        if (_e != cudaSuccess) {                                                          \
            fprintf(stderr, "gen: %s failed: %s\n", #x, cudaGetErrorString(_e));         \
            return -4;                                                                    \
        }                                                                                 \
    } while (0)

}  // namespace

extern "C" {

// kind 0 = ER(p0 = n0, p1 = pairs, p2 = isolated), 1 = grid(p0 = rows, p1 = cols, p2 = p32),
// 2 = rmat(p0 = scale, p1 = edge_factor, p2 = permuted).  Returns 0 and n, m.
int gen_csr_begin(int kind, uint64_t seed, uint64_t p0, uint64_t p1, uint64_t p2, uint32_t* n_out, int64_t* m_out,
                  void** state_out)
{
    Spec sp{};
    sp.kind = kind;
    sp.seed = seed;
    if (kind == KIND_ER) {
        sp.n0 = p0;
        sp.count = p1;
        sp.n = (uint32_t)(p0 + p2);
    } else if (kind == KIND_GRID) {
        sp.rows = p0;
        sp.cols = p1;
        sp.p32 = p2;
        sp.count = p0 * (p1 - 1) + (p0 - 1) * p1;
        sp.n = (uint32_t)(p0 * p1);
    } else if (kind == KIND_RMAT) {
        sp.scale = (int)p0;
        sp.count = p1 << p0;
        sp.permuted = (int)p2;
        sp.perm = make_perm(seed, sp.scale);
        sp.n = (uint32_t)(1ull << p0);
    } else {
        return -1;
    }
    const int vb = bits_for(sp.n);
    int bbits = 0;                                      // buckets = 2^bbits <= 1024, each ~< 2^30 keys
    while (bbits < 10 && bbits < vb && ((2 * sp.count) >> bbits) > (1ull << 29)) ++bbits;
    const int bshift = vb - bbits;
    const int nb = 1 << bbits;
    cudaStream_t s = 0;
    unsigned long long* bcount = nullptr;
    TRY(cudaMalloc(&bcount, sizeof(unsigned long long) * 2 * nb));
    TRY(cudaMemset(bcount, 0, sizeof(unsigned long long) * 2 * nb));
    k_count<<<grid_blocks(), 256, 0, s>>>(sp, vb, bshift, bcount);
    TRY(cudaGetLastError());
    std::vector<unsigned long long> cnt(nb), start(nb + 1, 0);
    TRY(cudaMemcpy(cnt.data(), bcount, sizeof(unsigned long long) * nb, cudaMemcpyDeviceToHost));
    for (int b = 0; b < nb; ++b) {
        start[b + 1] = start[b] + cnt[b];
        if (cnt[b] >= (1ull << 31)) {
            fprintf(stderr, "gen: bucket %d too large (%llu)\n", b, cnt[b]);
            return -2;
        }
    }
    const uint64_t K = start[nb];
    uint64_t maxb = 1;
    for (int b = 0; b < nb; ++b) maxb = cnt[b] > maxb ? cnt[b] : maxb;
    State* st = new State;
    st->n = sp.n;
    st->vb = vb;
    TRY(cudaMalloc(&st->keys, sizeof(uint64_t) * (K ? K : 1)));
    TRY(cudaMemcpy(bcount + nb, start.data(), sizeof(unsigned long long) * nb, cudaMemcpyHostToDevice));
    k_scatter<<<grid_blocks(), 256, 0, s>>>(sp, vb, bshift, bcount + nb, st->keys);
    TRY(cudaGetLastError());
    // per-bucket sort + unique, compacting into the front of keys
    uint64_t* alt = nullptr;
    int* d_nsel = nullptr;
    TRY(cudaMalloc(&alt, sizeof(uint64_t) * maxb));
    TRY(cudaMalloc(&d_nsel, sizeof(int)));
    size_t tmp_bytes = 0, tb2 = 0;
    {
        cub::DoubleBuffer<uint64_t> db(st->keys, alt);
        cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, db, (int)maxb, 0, 2 * vb, s);
        cub::DeviceSelect::Unique(nullptr, tb2, st->keys, alt, d_nsel, (int)maxb, s);
        if (tb2 > tmp_bytes) tmp_bytes = tb2;
    }
    void* tmp = nullptr;
    TRY(cudaMalloc(&tmp, tmp_bytes ? tmp_bytes : 1));
    uint64_t out = 0;
    for (int b = 0; b < nb; ++b) {
        const int c = (int)cnt[b];
        if (c == 0) continue;
        uint64_t* seg = st->keys + start[b];
        cub::DoubleBuffer<uint64_t> db(seg, alt);
        size_t tbytes = tmp_bytes;
        TRY(cub::DeviceRadixSort::SortKeys(tmp, tbytes, db, c, 0, 2 * vb, s));
        uint64_t* src = db.Current();
        tbytes = tmp_bytes;
        int nsel = 0;
        // the unique run goes to keys[out .. out+nsel); out <= start[b], so it only
        // overwrites compacted earlier output's tail or this bucket's dead input
        if (src == alt) {
            TRY(cub::DeviceSelect::Unique(tmp, tbytes, alt, st->keys + out, d_nsel, c, s));
            TRY(cudaMemcpy(&nsel, d_nsel, sizeof(int), cudaMemcpyDeviceToHost));
        } else {
            TRY(cub::DeviceSelect::Unique(tmp, tbytes, seg, alt, d_nsel, c, s));
            TRY(cudaMemcpy(&nsel, d_nsel, sizeof(int), cudaMemcpyDeviceToHost));
            TRY(cudaMemcpy(st->keys + out, alt, sizeof(uint64_t) * nsel, cudaMemcpyDeviceToDevice));
        }
        out += (uint64_t)nsel;
    }
    cudaFree(tmp);
    cudaFree(alt);
    cudaFree(d_nsel);
    cudaFree(bcount);
    st->m = out;
    *n_out = sp.n;
    *m_out = (int64_t)out;
    *state_out = st;
    return 0;
}

// Write offsets (n+1 int64) and adj (m uint32) into caller buffers; frees the state.
int gen_csr_finish(void* state, int64_t* off, uint32_t* adj)
{
    State* st = (State*)state;
    const uint64_t vmask = (1ull << st->vb) - 1;
    k_offsets<<<grid_blocks(), 256>>>(st->keys, st->m, st->vb, st->n, off);
    TRY(cudaGetLastError());
    if (st->m) {
        k_adj<<<grid_blocks(), 256>>>(st->keys, st->m, vmask, adj);
        TRY(cudaGetLastError());
    }
    TRY(cudaDeviceSynchronize());
    cudaFree(st->keys);
    delete st;
    return 0;
}

void gen_csr_abort(void* state)
{
    State* st = (State*)state;
    if (!st) return;
    cudaFree(st->keys);
    delete st;
}

// C5 batch b: n_ins RMAT-s inserts (draws b*n_ins ..) and n_q uniform query pairs (draws b*n_q ..).
int gen_incr_batch(uint64_t seed, int s, uint64_t b, uint64_t n_ins, uint64_t n_q, uint32_t* ins, uint32_t* qs,
                   void* stream)
{
    Perm perm = make_perm(seed, s);
    k_incr<<<grid_blocks(), 256, 0, (cudaStream_t)stream>>>(seed, s, perm, b * n_ins, n_ins, b * n_q, n_q, ins, qs);
    TRY(cudaGetLastError());
    return 0;
}

// RMAT pair stream with explicit (a, b, c) thresholds (inputs/gen.py rmat_pairs)
int gen_rmat_stream(uint64_t seed, int s, uint64_t first, uint64_t count, uint32_t t1, uint32_t t2, uint32_t t3,
                    int permuted, uint32_t* out, void* stream)
{
    Perm perm = make_perm(seed, s);
    k_rmat_stream<<<grid_blocks(), 256, 0, (cudaStream_t)stream>>>(seed, s, perm, permuted, t1, t2, t3, first, count,
                                                                   out);
    TRY(cudaGetLastError());
    return 0;
}

// Exp(1) edge weights (inputs/gen.py exp_weights): w(u,v) = -ln(U),
// U = (k + 1/2) 2^-52, k = mix(seed, WEIGHT, min(u,v) 2^32 + max(u,v)) >> 12,
// with gen.py's fixed-order log (explicit _rn intrinsics: no FMA contraction),
// so the float32 bytes are identical.
int gen_exp_weights(const int64_t* off, const uint32_t* adj, uint32_t n, int64_t m, uint64_t seed, float* w,
                    void* stream)
{
    if (m <= 0) return 0;
    k_weights<<<grid_blocks(), 256, 0, (cudaStream_t)stream>>>(off, adj, n, (uint64_t)m, seed, w);
    TRY(cudaGetLastError());
    return 0;
}

}  // extern "C"
