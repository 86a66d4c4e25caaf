/*
 * cc_bench.h -- measurement-floor kernels exported by libcc.so (K10).
 *
 * The paper's Table 8 compares connectivity against two
 * primitives that bound any algorithm touching every edge: MapEdges (a
 * constant per edge, i.e. a sequential read of the adjacency) and GatherEdges
 * (one indirect read x[v] per edge, "a practical lower bound").
 * These are the B200 versions, run on the same device CSR as cc_labels.
 * All pointers are DEVICE pointers; calls are asynchronous on `stream`.
 * Return CC_OK, CC_EINVAL (null pointer with n > 0) or CC_ECUDA.
 */
#ifndef CC_B200_CC_BENCH_H
#define CC_B200_CC_BENCH_H

#include <stdint.h>

#include "cc.h"

#ifdef __cplusplus
extern "C" {
#endif

/* MapEdges: out[u] = sum over e in [off[u], off[u+1]) of 1,
 * computed by actually reading every adj entry (adj[e] < 0xFFFFFFFF counts 1).
 * Both edge kernels read m = offsets[n] back to the host first (one sync) and
 * zero `out`; the sweep itself is edge-balanced (4096 entries per warp). */
cc_status cc_bench_map_edges(const int64_t* offsets, const uint32_t* adj, uint32_t n,
                             uint32_t* out, void* stream);

/* GatherEdges: out[u] = sum over v in N(u) of x[v]  (mod 2^32). */
cc_status cc_bench_gather_edges(const int64_t* offsets, const uint32_t* adj, uint32_t n,
                                const uint32_t* x, uint32_t* out, void* stream);

/* count uniformly random 4-byte loads from x[0..len): the random-sector ceiling.
 * Load i reads x[(lo32(splitmix64(seed + i)) * len) >> 32]; *out = sum mod 2^32. */
cc_status cc_bench_random_gather(const uint32_t* x, uint64_t len, uint64_t count, uint64_t seed,
                                 uint32_t* out, void* stream);

/* dst[i] = src[i] for i < words (uint32): the streaming copy ceiling. */
cc_status cc_bench_copy(const uint32_t* src, uint32_t* dst, uint64_t words, void* stream);

/* Set the device-wide cudaLimitMaxL2FetchGranularity (bytes, 0..128) of the
 * current context; returns the previous value in *prev (may be NULL).  A
 * measurement knob for the random-access kernels (32 B = one sector). */
cc_status cc_bench_set_l2_fetch(int bytes, int* prev);

/* Cumulative number of kernels libcc.so has launched in this process
 * (bench evidence for "gpu_launches"; host-side counter, no GPU access). */
uint64_t cc_bench_launch_count(void);

/* Test hook: launch every grid-strided ("persistent") kernel of libcc.so with
 * exactly `blocks` blocks (0 = the default multiple of the SM count); returns
 * the previous setting.  Process-wide, not thread-safe against concurrent
 * calls.  Results never depend on it (repeats with random launch
 * configurations); the tile-per-block streaming kernels keep their grids. */
unsigned cc_bench_set_grid(unsigned blocks);

#ifdef __cplusplus
}
#endif
#endif /* CC_B200_CC_BENCH_H */
