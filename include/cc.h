/*
 * cc.h -- C ABI of the B200 connectivity hot path (ConnectIt, arXiv 2008.03909).
 *
 * libcc.so (paper_2008_03909_b200/libcc.so) exports exactly the functions
 * declared here and in cc_bench.h.  Every signature uses plain pointers and
 * sizes; there are no torch types.  Citations "P:n" are PAPER.md lines.
 *
 * Problem statement: given an undirected graph G = (V, E) with
 * n = |V|, compute a connectivity labeling C with C(u) = C(v) iff u and v are
 * in the same connected component, and a spanning forest with one tree per
 * component.  Batch-incremental connectivity: process batches of
 * Insert(u,v) and IsConnected(u,v) operations one batch after another.
 *
 * ---- Graph layout (all calls) ----------------------------------------------
 *   offsets  int64_t[n+1], offsets[0] = 0, offsets[n] = m, non-decreasing.
 *   adj      uint32_t[m]; the neighbours of v are adj[offsets[v] .. offsets[v+1]).
 *   m counts DIRECTED adjacency entries (each undirected edge twice).
 *   The graph must be SYMMETRIC (u in N(v) iff v in N(u)) for the giant-
 *   component skip to be correct (Thm. A.1); pass
 *   CC_FLAG_NO_SKIP otherwise -- the result is then the CC of the underlying
 *   undirected graph.  Self-loops and duplicate entries are tolerated.
 *   Neighbour order only changes which "first k" edges are sampled, never the
 *   labels.  Ids are uint32 < n; n <= 0xFFFFFFFE (0xFFFFFFFF is the sentinel).
 *
 * ---- Memory, streams, ownership -----------------------------------------------
 *   Array arguments may be DEVICE pointers (cudaMalloc / torch tensors) or
 *   HOST pointers (pinned or pageable).  With device pointers every call is
 *   stream-ordered and asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *   default stream) and performs no host synchronisation.  If ANY array
 *   argument of a call is a host pointer, the call stages the host arrays
 *   through library-owned device memory (host->device copies, compute,
 *   device->host copies) and returns only after the results are in the host
 *   buffers (it synchronises `stream`).
 *   The caller owns every input and output buffer and must keep them alive
 *   until the stream has passed the call.  The library owns only cc_incr
 *   handles and transient scratch, allocated with cudaMallocAsync on `stream`
 *   and freed on the same stream before the call returns.
 *
 * ---- Errors --------------------------------------------------------------------
 *   Host-side argument checks run first and return before any launch:
 *   CC_EINVAL (null pointer with n > 0, m < 0, bad opts), CC_ERANGE
 *   (n > 0xFFFFFFFE, kout_k > 64).  n = 0 returns CC_OK with no work.
 *   Malformed CSR (offsets not monotone, adj[i] >= n) is undefined behaviour
 *   unless CC_FLAG_VALIDATE is set: then a validation kernel runs first (one
 *   stream synchronisation) and CC_EINVAL is returned with outputs untouched.
 *   CUDA failures return CC_ECUDA; cc_last_error() returns a thread-local
 *   detail string.  On any error a cc_incr handle keeps its pre-call state.
 */
#ifndef CC_B200_CC_H
#define CC_B200_CC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int cc_status;
#define CC_OK       0
#define CC_EINVAL  (-1)
#define CC_ERANGE  (-2)
#define CC_ENOMEM  (-3)
#define CC_ECUDA   (-4)

/* k-out edge choice (Alg. 4; variants P:3589-3599).
 * AFFOREST: adjacency positions 0..k-1 ("first k neighbours", the north_star).
 * HYBRID:   position 0 plus k-1 positions uniform with replacement (the
 *           paper's default);
 * PURE:     k positions uniform with replacement (Holm et al.).
 * Random draw j of vertex u is position ((lo32(mix(seed,16,u*64+j)) * deg(u)) >> 32)
 * with mix(s,t,i) = splitmix64(s*0x9E3779B97F4A7C15 + t*2^40 + i).          */
#define CC_VARIANT_AFFOREST 0u
#define CC_VARIANT_HYBRID   1u
#define CC_VARIANT_PURE     2u

#define CC_FLAG_NO_SKIP     (1u << 0)  /* finish every vertex (no L_max skip)          */
#define CC_FLAG_VALIDATE    (1u << 1)  /* check the CSR first (synchronises)                     */
#define CC_FLAG_UF_ASYNC    (1u << 2)  /* UF-Async link rule instead of UF-Rem-CAS */
#define CC_FLAG_HALVE       (1u << 3)  /* HalveAtomicOne instead of SplitAtomicOne */
#define CC_FLAG_FIND_SPLIT  (1u << 4)  /* incremental queries use FindAtomicSplit  */
#define CC_FLAG_FIND_NAIVE  (1u << 15) /* incremental queries use FindNaive; default:
                                          path halving with plain stores (no hook runs in
                                          the query phase)                                 */
#define CC_FLAG_NO_DEGSKIP  (1u << 5)  /* also finish vertices whose whole list was sampled      */
#define CC_FLAG_NO_MIDCOMPRESS (1u << 6) /* never run the compress between k-out rounds        */
#define CC_FLAG_MIDCOMPRESS (1u << 7)  /* always run it (default: a 1024-sample probe of the
                                          round-0 chain depth decides, on the device)        */
#define CC_FLAG_FINISH_SV   (1u << 9)  /* finish with Shiloach-Vishkin rounds (writeMin root
                                          hooking + full shortcut) instead of
                                          UF-Rem-CAS; one host sync per round (NEXT-3)      */
#define CC_FLAG_CONTRACT    (1u << 10) /* run the k-out CAS links on the forest contracted by
                                          the first k-out round: a compact parent array
                                          with one slot per non-isolated F0 root (see
                                          cc_labels); ignored with CC_FLAG_NO_SKIP.
                                          Measured slower than the default in place link
                                          on C3/C4                               */
#define CC_FLAG_NO_REFILL   (1u << 11) /* k-out links: always k_link_pending (links per thread
                                          with their first parent reads batched)           */
#define CC_FLAG_LINK_REFILL (1u << 18) /* k-out links: always the lane-refill kernel.  Default
                                          (neither flag): the round-0 chain probe picks on the
                                          device -- short chains k_link_pending, long chains
                                          (grid-like ids) lane refill                        */
#define CC_FLAG_FUSED_LINK  (1u << 16) /* run k-out sampling and its CAS links in one kernel
                                          (links queued in shared memory, P initialised first);
                                          UF-Rem-CAS + SplitAtomicOne with k <= 2 only, else
                                          ignored.  Measured, not the default     */
#define CC_FLAG_FINISH_CRFA (1u << 13) /* finish with the Liu-Tarjan CRFA rounds (Connect,
                                          RootUp, FullShortcut, Alter)
                                          instead of UF-Rem-CAS; one host sync per round.
                                          (CC_FLAG_FINISH_SV is the root-based PRF instance:
                                          ParentConnect + RootUp + FullShortcut)             */
#define CC_FLAG_AMSF_NO_INDEX (1u << 14) /* cc_amsf: scan the whole list of a long (> 2048
                                          entries) list every active round instead of only
                                          its current bucket's entries (hub bucket index)   */
#define CC_FLAG_AMSF_PLAIN  (1u << 12) /* cc_amsf: inspect every edge of every non-skipped
                                          vertex in every round, as AMSF-NF-S is stated
                                          (P:1819-1822), instead of consulting the per-
                                          vertex [min, max] weight index first          */
#define CC_FLAG_WAIT_FREE   (1u << 8)  /* cc_incr: the wait-free type (1) setting (P:973-977,
                                          P:2663-2682): a batch's inserts and queries run
                                          concurrently in ONE kernel.  Answers are then
                                          linearizable, not bit-exact: 1 implies connected
                                          after this batch's inserts, 0 implies not
                                          connected before them               */

/* Per-phase device times, filled when cc_opts.timings != NULL (the call then
 * synchronises `stream` before returning).  Bench/diagnostics only.          */
typedef struct {
    float sample_ms;     /* H1 init + H2 k-out link + H3 sampling compress        */
    float identify_ms;   /* H4 IdentifyFrequent                                    */
    float finish_ms;     /* H5 finish link with the L_max skip                     */
    float compress_ms;   /* H6 final compress (+ H7 forest compaction in SF mode)  */
    float total_ms;
} cc_timings;

/* Work counters, accumulated (atomicAdd) into a DEVICE struct when
 * cc_opts.counters != NULL.  Bench/diagnostics only.                         */
typedef struct {
    uint64_t pending_links;    /* H2 links left to the CAS kernel (k_link_pending)    */
    uint64_t worklist;         /* vertices marked for the finish (list not all sampled)*/
    uint64_t finish_vertices;  /* marked vertices with root != L_max, lists traversed */
    uint64_t finish_edges;     /* adjacency entries traversed by the finish          */
    uint64_t sample_hooks;     /* successful root hooks in k_link_pending (H2)       */
    uint64_t finish_hooks;     /* successful root hooks in the finish (H5)           */
    uint64_t big_vertices;     /* finish vertices sent to the CTA-per-vertex queue   */
    uint64_t compress_writes;  /* slots rewritten by the fused H3 compress (k_finish)*/
    uint64_t link_steps;       /* Rem-loop iterations of k_link_pending's walked links*/
    uint64_t cas_failures;     /* hook CAS that lost a race in k_link_pending        */
    uint64_t probe_deep;       /* probe samples whose round-0 chain exceeded 8 steps */
    uint64_t finish_gathers;   /* first-level parent reads of k_finish (P[P[v]])      */
    uint64_t h6_writes;        /* label slots rewritten by the final compress (H6)   */
    uint64_t h6_gathers;       /* first-level parent reads of the final compress     */
    uint64_t sv_rounds;        /* rounds of the Shiloach-Vishkin finish (FINISH_SV)  */
    uint64_t contract_roots;   /* slots of the contracted parent array (non-isolated
                                  roots of the first k-out round's forest F0)        */
    uint64_t amsf_rounds;      /* cc_amsf: weight buckets processed                    */
    uint64_t amsf_visits;      /* cc_amsf: active-vertex visits over all rounds        */
    uint64_t amsf_edges;       /* cc_amsf: adjacency weights inspected over all rounds */
    uint64_t amsf_hooks;       /* cc_amsf: successful root hooks (= forest edges)      */
    uint64_t amsf_rebuilds;    /* cc_amsf: rounds whose L_max left the skipped component*/
    uint64_t fused_link;       /* 1 if the k-out links ran inside k_sample_link         */
    uint64_t amsf_links;       /* cc_amsf: in-bucket edges linked (diagnostics build only)*/
    uint64_t h6_tiles;         /* tiles of kCTile = 2048 slots the partial final compress
                                  re-resolved (dirty: a root they hold or name was
                                  hooked by H5, L_max was hooked, or two distinct foreign
                                  roots in one of its 256-slot warp summaries)               */
    uint64_t link_pending;     /* 1 if the k-out links ran in k_link_pending (0: lane refill,
                                  the contracted or the fused link)                        */
    uint64_t mid_compress;     /* 1 if the chain probe ran the compress between the k-out
                                  rounds (also 0 when a flag forced or forbade it)          */
} cc_counters;

typedef struct {
    uint32_t kout_k;           /* sampled edges per vertex; default 2; 0 = no sampling */
    uint32_t kout_variant;     /* CC_VARIANT_*; default AFFOREST                       */
    uint64_t seed;             /* hybrid picks + IdentifyFrequent draws; default 0     */
    uint32_t samples;          /* IdentifyFrequent sample count; default 1024 (1..2048)*/
    uint32_t flags;            /* CC_FLAG_*                                            */
    /* test/bench hooks; NULL in production (no extra traffic, no syncs):          */
    uint32_t*       sampled_out; /* DEVICE, n: copy of P after H3 (sampled labels)    */
    uint32_t*       lmax_out;    /* DEVICE scalar: the L_max used                     */
    const uint32_t* lmax_force;  /* DEVICE scalar or NULL: overrides H4;
                                    0xFFFFFFFF = skip nothing                          */
    cc_counters*    counters;    /* DEVICE                                             */
    cc_timings*     timings;     /* HOST                                               */
    void**          marks;       /* HOST array of CC_NUM_MARKS cudaEvent_t created by
                                    the caller, or NULL: recorded on `stream` at the
                                    kernel boundaries below, no synchronisation       */
} cc_opts;

/* Kernel-boundary marks of cc_labels / cc_spanning_forest (cc_opts.marks[i] is
 * recorded after the named step; a skipped step records a zero-length span).  */
#define CC_MARK_START       0   /* before the first kernel                        */
#define CC_MARK_INIT        1   /* k_sample_init: H1 + first k-out round          */
#define CC_MARK_MIDCOMPRESS 2   /* compress between k-out rounds                  */
#define CC_MARK_LINK        3   /* k_link_pending: remaining k-out links (H2)     */
#define CC_MARK_SAMPLED     4   /* separate H3 compress, only with sampled_out    */
#define CC_MARK_IDENTIFY    5   /* IdentifyFrequent (H4)                          */
#define CC_MARK_FINISH      6   /* k_finish: H3 compress fused with the H5 scan   */
#define CC_MARK_FINISH_BIG  7   /* k_finish_proc + k_finish_big: H5 edge work     */
#define CC_MARK_COMPRESS    8   /* final compress (H6)                            */
#define CC_MARK_FOREST      9   /* forest filter (H7; zero-length in cc_labels)   */
#define CC_NUM_MARKS       10

/* Fill *o with the defaults above. */
void cc_opts_default(cc_opts* o);

/* Connectivity, Alg. 1 with k-out sampling (Alg. 4), IdentifyFrequent
 * and the UF-Rem-CAS finish, then the final
 * compress.  labels (out, n) is also the parent array, used in place:
 * on return labels[v] = minimum vertex id of v's component (canonical).
 * The first k-out round hooks every vertex under its first sampled neighbour
 * when that is smaller (a forest F0); the remaining sampled edges are then
 * unioned in place on labels (default), or, with CC_FLAG_CONTRACT, with the
 * same UF-Rem-CAS rule on a compact parent array with one slot per
 * non-isolated F0 root, numbered in id order (so the min-id orientation is
 * kept); the latter needs the symmetric-graph precondition above.  The scan
 * of the finish leaves every slot at its sampled root, so the final compress
 * re-resolves only the 2048-slot tiles whose labels the finish's hooks changed
 * (all of them if L_max itself was hooked); with labels in a host buffer, or
 * after an SV / CRFA finish, it is a full pass.  Every kernel is a
 * programmatic dependent launch; with device buffers the call never
 * synchronises, so it can be captured into a CUDA graph. */
cc_status cc_labels(const int64_t* offsets, const uint32_t* adj, uint32_t n, int64_t m,
                    uint32_t* labels, const cc_opts* opts, void* stream);

/* Spanning forest, Alg. 2 with the k-out forest rule
 * and the root-based finish.  edges (out, capacity 2*n uint32):
 * pairs (u, v) -- each an input edge with v in N(u) -- packed in ascending order
 * of the hooked root's id (the Filter of P:2415 keeps array order).
 * num_edges (out, one int64, same memory kind as edges) = n - #components.
 * labels (out, n) may be NULL; if given it receives the canonical labels. */
cc_status cc_spanning_forest(const int64_t* offsets, const uint32_t* adj, uint32_t n, int64_t m,
                             uint32_t* edges, int64_t* num_edges, uint32_t* labels,
                             const cc_opts* opts, void* stream);

/* Approximate minimum spanning forest, AMSF-NF-S (Sec. 5.1):
 * W(F_OPT) <= W(F) <= (1+eps) W(F_OPT).  The folklore algorithm:
 * W_min = min w(e) over every adjacency entry, self-loops included; bucket i holds the edges with b_i <= w < b_(i+1), b_0 =
 * W_min, b_(i+1) = b_i * (1+eps) in fp64 (reading R25); buckets are
 * processed from light to heavy, each one's edges unioned with UF-Rem-CAS +
 * SplitAtomicOne on one persistent parent array, recording the
 * edge at the hooked root as in cc_spanning_forest.  NF: the CSR
 * is never mutated.  S: each round samples L_max (IdentifyFrequent
 * on the current labeling) and skips the vertices of its component; CC_FLAG_NO_SKIP
 * turns that off.  Unless CC_FLAG_AMSF_PLAIN is set, a vertex is visited only in
 * the rounds between the buckets of its lightest and heaviest edge.
 *   w         float32[m], aligned with adj; strictly positive, finite, and
 *             symmetric (w(u,v) == w(v,u)) -- the skip relies on it.
 *   eps       > 0 (the paper uses 0.25).
 *   edges     (out, capacity 2*n uint32): forest pairs (u, v), input edges.
 *   edge_w    (out, capacity n float, may be NULL): their weights.
 *   num_edges (out, one int64) = n - #components.
 *   total     (out, one double, may be NULL): sum of the forest weights (fp64).
 * Arrays may be device memory, or host memory (pinned or pageable), which is
 * staged through device scratch (the outputs are copied back and the call
 * returns after they landed).  The call synchronises `stream` once, to read
 * W_min / W_max and size the buckets.
 * Errors: CC_EINVAL for eps <= 0 or a non-positive / non-finite weight
 * (checked on the device; outputs untouched). */
cc_status cc_amsf(const int64_t* offsets, const uint32_t* adj, const float* w, uint32_t n, int64_t m, double eps,
                  uint32_t* edges, float* edge_w, int64_t* num_edges, double* total, const cc_opts* opts,
                  void* stream);

/* Batch-incremental connectivity, Alg. 3, UF-Rem-CAS +
 * SplitAtomicOne on a persistent parent array owned by the
 * handle.  Phase-concurrent order (type (3)): all inserts of a
 * batch, then a device-wide barrier, then all queries -- so a query sees the
 * inserts of every earlier batch AND of its own batch. */
typedef struct cc_incr cc_incr;

/* Create a handle over n vertices with no edges (P[v] = v).  opts may be NULL;
 * only opts->flags (CC_FLAG_HALVE, CC_FLAG_UF_ASYNC, CC_FLAG_FIND_SPLIT,
 * CC_FLAG_VALIDATE, CC_FLAG_WAIT_FREE) is used.  *out receives the handle (host pointer). */
cc_status cc_incr_create(uint32_t n, const cc_opts* opts, void* stream, cc_incr** out);

/* inserts: 2*n_ins uint32, (u, v) interleaved; queries: 2*n_q uint32;
 * answers (out): n_q uint8, answers[j] = 1 iff queries[j] endpoints are
 * connected after all prior batches and this batch's inserts.  Self-loop and
 * duplicate inserts are legal no-ops.  With CC_FLAG_VALIDATE on the handle,
 * out-of-range ids return CC_EINVAL before any insert is applied. */
cc_status cc_incr_batch(cc_incr* h, const uint32_t* inserts, int64_t n_ins,
                        const uint32_t* queries, int64_t n_q, uint8_t* answers, void* stream);

/* Process nb batches in order in ONE call -- exactly what nb cc_incr_batch calls
 * would compute (batch b's queries see the inserts of batches 0..b).  The
 * batches' pairs are concatenated in `inserts` / `queries` and their answers in
 * `answers`; ins_counts / q_counts are HOST int64 arrays of nb counts.  When
 * every batch has at most 8192 operations the whole sequence runs in one
 * single-CTA kernel with a block barrier between each insert and query phase
 * (the paper's small-batch regime, Table 5); otherwise one launch
 * pair per batch.  Arrays may be device, pinned host or pageable host memory:
 * pinned host inserts / queries of larger batches are copied into two device
 * staging buffers by DMA on an internal copy stream, batch b+1 while batch b
 * computes (scratch: 2 x 8 B per pair of the largest batch); pinned answers
 * are written in place; pageable arrays are staged batch by batch.  A call
 * with host arrays returns after the work is complete.  Stream order: the
 * call's first kernel is an ordinary launch (it starts after all earlier work
 * of `stream` has completed), every later one a programmatic dependent launch
 * that reads its batch's pairs and first parent slots BEFORE waiting for the
 * previous kernel (DESIGN.md §6 item 21) -- so all batches' pairs must be in
 * place when the call is made (written by earlier work of `stream`, or by the
 * host), not by work enqueued on another stream afterwards.  Errors as
 * cc_incr_batch (with CC_FLAG_VALIDATE, all ids are checked first). */
cc_status cc_incr_batches(cc_incr* h, int64_t nb, const int64_t* ins_counts, const uint32_t* inserts,
                          const int64_t* q_counts, const uint32_t* queries, uint8_t* answers, void* stream);

/* labels (out, n): canonical labels (min id per component) of the current state. */
cc_status cc_incr_labels(cc_incr* h, uint32_t* labels, void* stream);

/* Synchronises the handle's last stream, then frees it.  NULL is a no-op. */
void cc_incr_destroy(cc_incr* h);

/* Number of vertices of a handle (0 for NULL). */
uint32_t cc_incr_num_vertices(const cc_incr* h);

/* Human-readable name of a status; thread-local detail of the last failure. */
const char* cc_status_str(cc_status s);
const char* cc_last_error(void);

/* Transient device scratch a call allocates (informational; no GPU access).
 * op 0 = cc_labels, 1 = cc_spanning_forest: an upper bound -- the sum of every
 * allocation any flag combination makes (pending links, queues, bitmaps, tile
 * summaries, the parent array and staging buffers used with host arguments,
 * the contracted-link arrays, the SV / CRFA edge lists; forest slots for op 1).
 * op 2 = cc_incr_create: the handle's parent array.  op 3 = cc_amsf: an
 * ESTIMATE sized for eps = 0.25-like bucket counts. */
size_t cc_workspace_bytes(uint32_t n, int64_t m, uint32_t kout_k, int op);

/* Library version string. */
const char* cc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CC_B200_CC_H */
