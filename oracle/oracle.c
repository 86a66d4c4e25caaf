/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, sequential CPU oracle
 * for the ConnectIt connectivity hot path (arXiv 2008.03909).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product library
 * (paper_2008_03909_b200/libcc.so) never links, includes or calls it, and this
 * file includes nothing from the product (no shared headers, helpers or
 * constants).  It is single threaded, uses no atomics and no GPU.
 *
 * What it computes are the paper's PLAIN DEFINITIONS, not the paper's fast
 * algorithm (the method reaches these exactly, so the definition is the oracle):
 *
 *   oracle_cc_bfs    connectivity labeling, PAPER.md P:382-388 (Sec. 2,
 *                    "Graph Connectivity and Related Problems": C(u)=C(v) iff
 *                    u and v are in the same connected component), made
 *                    canonical as lab[v] = min vertex id of v's component
 *                    (north_star; reading R13).  Breadth-first search
 *                    (P:399-402 defines BFS) from every unvisited vertex in
 *                    increasing id order; the first vertex scanned in a
 *                    component is its minimum.
 *   oracle_cc_dsu    the same labeling by an independent route: a sequential
 *                    union-find (P:406-420 defines MakeSet/Union/Find) with
 *                    union by size and path halving, then min id per root.
 *   oracle_forest_check
 *                    spanning-forest validity, P:394-396 ("one tree for each
 *                    connected component ... containing all vertices of that
 *                    component") and Alg. 2: |F| = n - c, every
 *                    pair is an input edge, and F is acyclic.  Several forests
 *                    are correct, so the oracle checks instead of computing.
 *   oracle_incr_run  batch-incremental connectivity, Sec. 3.5 P:955-958 and
 *                    the correctness definition, with the reading
 *                    that a query sees every insert of its own batch (type (3)
 *                    phase-concurrent order; reading R15):
 *                    per batch, apply all inserts to a sequential union-find,
 *                    then answer every query as find(a) == find(b).
 *   oracle_kruskal   exact minimum spanning forest (the reference point of the
 *                    AMSF definition: W(F_OPT) of "any spanning
 *                    forest of G of minimum weight"): Kruskal's algorithm --
 *                    every undirected edge once, sorted by (w, u, v), added
 *                    unless it closes a cycle (sequential union-find).
 *   oracle_amsf      the folklore AMSF algorithm, step by step in the paper's
 *                    order: W_min = min w(e); bucket i holds the
 *                    edges with W_min(1+eps)^i <= w < W_min(1+eps)^(i+1)
 *                    (boundaries b_0 = W_min, b_(i+1) = b_i * (1+eps) in fp64,
 *                    DESIGN.md reading R25); buckets from light to heavy; in
 *                    each bucket drop the edges whose endpoints are already
 *                    connected ("self-loops" of the labeling C) and add the
 *                    rest to a spanning forest F_i, updating C; F = U F_i.
 *                    The edges of a bucket are taken in CSR order (u < v).
 *
 * Pins (tests/test_oracle.py): exhaustive brute-force reachability for every
 * labelled graph on n <= 5 vertices, Warshall closure on random graphs up to
 * n = 64, closed forms (cliques, paths, star, full grid, edgeless, the paper's
 * counter-example graph P:2199-2200), scipy's connected_components partition,
 * and BFS-vs-DSU agreement.
 *
 * Conventions: offsets are int64 with off[0] = 0 and off[n] = m, adjacency is
 * uint32; vertex ids are uint32 < n.  Return 0 on success, a negative value on
 * malformed input or allocation failure.
 */
#include <float.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define UNSET 0xFFFFFFFFu

/* ---- connectivity labeling by BFS ------------------ */
int oracle_cc_bfs(uint32_t n, const int64_t* off, const uint32_t* adj, uint32_t* lab)
{
    if (n == 0) return 0;
    uint32_t* q = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    if (!q) return -3;
    for (uint32_t v = 0; v < n; ++v) lab[v] = UNSET;
    for (uint32_t s = 0; s < n; ++s) {
        if (lab[s] != UNSET) continue;
        /* s is the smallest id not yet reached: the minimum of its component */
        uint32_t head = 0, tail = 0;
        lab[s] = s;
        q[tail++] = s;
        while (head < tail) {
            uint32_t x = q[head++];
            for (int64_t e = off[x]; e < off[x + 1]; ++e) {
                uint32_t y = adj[e];
                if (y >= n) { free(q); return -1; }
                if (lab[y] == UNSET) { lab[y] = s; q[tail++] = y; }
            }
        }
    }
    free(q);
    return 0;
}

/* ---- the same labeling through a sequential union-find -------- */
static uint32_t dsu_find(uint32_t* parent, uint32_t x)
{
    while (parent[x] != x) {            /* path halving */
        parent[x] = parent[parent[x]];
        x = parent[x];
    }
    return x;
}

static void dsu_union(uint32_t* parent, uint32_t* size, uint32_t a, uint32_t b)
{
    a = dsu_find(parent, a);
    b = dsu_find(parent, b);
    if (a == b) return;
    if (size[a] < size[b]) { uint32_t t = a; a = b; b = t; }
    parent[b] = a;                      /* union by size */
    size[a] += size[b];
}

int oracle_cc_dsu(uint32_t n, const int64_t* off, const uint32_t* adj, uint32_t* lab)
{
    if (n == 0) return 0;
    uint32_t* parent = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    uint32_t* size = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    if (!parent || !size) { free(parent); free(size); return -3; }
    for (uint32_t v = 0; v < n; ++v) { parent[v] = v; size[v] = 1; }
    for (uint32_t x = 0; x < n; ++x)
        for (int64_t e = off[x]; e < off[x + 1]; ++e) {
            if (adj[e] >= n) { free(parent); free(size); return -1; }
            dsu_union(parent, size, x, adj[e]);
        }
    /* the canonical label is the minimum member id of each set */
    uint32_t* mn = size;                /* reuse: min id per root */
    for (uint32_t v = 0; v < n; ++v) mn[v] = UNSET;
    for (uint32_t v = 0; v < n; ++v) {
        uint32_t r = dsu_find(parent, v);
        if (v < mn[r]) mn[r] = v;
    }
    for (uint32_t v = 0; v < n; ++v) lab[v] = mn[dsu_find(parent, v)];
    free(parent);
    free(size);
    return 0;
}

/* ---- spanning forest validity (Alg. 2) ------------- */
/* Returns 0 if F (nf pairs, interleaved u,v) is a spanning forest of the CSR
 * graph whose component count is c; otherwise a positive code, and *bad is set
 * to the offending pair index (or -1):
 *   1  |F| != n - c
 *   2  an endpoint is >= n
 *   3  a self-loop pair (u == v)
 *   4  (u,v) is not an input edge (v not in the sorted list adj[off[u]..off[u+1]))
 *   5  the pair closes a cycle (u and v were already joined by earlier pairs)
 * Checks (2)-(5) with (1) imply F spans every component: an acyclic subgraph
 * of G with n - c edges has exactly c trees, each inside one component.      */
static int in_list(const uint32_t* a, int64_t lo, int64_t hi, uint32_t key)
{
    /* adjacency lists are sorted ascending (the input contract); binary search */
    int64_t l = lo, h = hi;
    while (l < h) {
        int64_t mid = l + (h - l) / 2;
        if (a[mid] < key) l = mid + 1; else h = mid;
    }
    return l < hi && a[l] == key;
}

int oracle_forest_check(uint32_t n, const int64_t* off, const uint32_t* adj, uint64_t c,
                        const uint32_t* F, int64_t nf, int64_t* bad)
{
    *bad = -1;
    if ((uint64_t)nf + c != (uint64_t)n) return 1;
    if (n == 0) return 0;
    uint32_t* parent = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    uint32_t* size = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    if (!parent || !size) { free(parent); free(size); return -3; }
    for (uint32_t v = 0; v < n; ++v) { parent[v] = v; size[v] = 1; }
    int rc = 0;
    for (int64_t i = 0; i < nf; ++i) {
        uint32_t u = F[2 * i], v = F[2 * i + 1];
        if (u >= n || v >= n) { rc = 2; *bad = i; break; }
        if (u == v) { rc = 3; *bad = i; break; }
        if (!in_list(adj, off[u], off[u + 1], v)) { rc = 4; *bad = i; break; }
        if (dsu_find(parent, u) == dsu_find(parent, v)) { rc = 5; *bad = i; break; }
        dsu_union(parent, size, u, v);
    }
    free(parent);
    free(size);
    return rc;
}

/* ---- batch-incremental connectivity --- */
/* nb batches; batch b has ins_cnt[b] inserts (pairs, concatenated in `ins`) and
 * q_cnt[b] queries (pairs, concatenated in `q`).  Writes one uint8 answer per
 * query (concatenated in `ans`): 1 iff the pair is connected by the inserts of
 * batches 0..b (its own batch included).  If final_lab is non-NULL it receives
 * the canonical labels (min id per component) after the last batch.          */
int oracle_incr_run(uint32_t n, int64_t nb, const int64_t* ins_cnt, const uint32_t* ins,
                    const int64_t* q_cnt, const uint32_t* q, uint8_t* ans, uint32_t* final_lab)
{
    if (n == 0) return 0;
    uint32_t* parent = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    uint32_t* size = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    if (!parent || !size) { free(parent); free(size); return -3; }
    for (uint32_t v = 0; v < n; ++v) { parent[v] = v; size[v] = 1; }
    int64_t pi = 0, pq = 0;
    for (int64_t b = 0; b < nb; ++b) {
        for (int64_t i = 0; i < ins_cnt[b]; ++i, ++pi) {
            uint32_t u = ins[2 * pi], v = ins[2 * pi + 1];
            if (u >= n || v >= n) { free(parent); free(size); return -1; }
            dsu_union(parent, size, u, v);
        }
        for (int64_t j = 0; j < q_cnt[b]; ++j, ++pq) {
            uint32_t a = q[2 * pq], c = q[2 * pq + 1];
            if (a >= n || c >= n) { free(parent); free(size); return -1; }
            ans[pq] = dsu_find(parent, a) == dsu_find(parent, c) ? 1 : 0;
        }
    }
    if (final_lab) {
        uint32_t* mn = size;
        for (uint32_t v = 0; v < n; ++v) mn[v] = UNSET;
        for (uint32_t v = 0; v < n; ++v) {
            uint32_t r = dsu_find(parent, v);
            if (v < mn[r]) mn[r] = v;
        }
        for (uint32_t v = 0; v < n; ++v) final_lab[v] = mn[dsu_find(parent, v)];
    }
    free(parent);
    free(size);
    return 0;
}

/* ---- exact minimum spanning forest: Kruskal ------------------ */
typedef struct { float w; uint32_t u, v; } wedge;

static int wedge_cmp(const void* a, const void* b)
{
    const wedge* x = (const wedge*)a;
    const wedge* y = (const wedge*)b;
    if (x->w != y->w) return x->w < y->w ? -1 : 1;
    if (x->u != y->u) return x->u < y->u ? -1 : 1;
    if (x->v != y->v) return x->v < y->v ? -1 : 1;
    return 0;
}

/* Undirected edges of a symmetric CSR (u < v), with the weight stored at u's
 * entry.  Returns the count, or -1 on a bad id / allocation failure. */
static int64_t collect_edges(uint32_t n, const int64_t* off, const uint32_t* adj, const float* w, wedge** out)
{
    int64_t ne = 0;
    for (uint32_t u = 0; u < n; ++u)
        for (int64_t e = off[u]; e < off[u + 1]; ++e) {
            if (adj[e] >= n) return -1;
            if (adj[e] > u) ++ne;
        }
    wedge* E = (wedge*)malloc((size_t)(ne ? ne : 1) * sizeof(wedge));
    if (!E) return -1;
    int64_t k = 0;
    for (uint32_t u = 0; u < n; ++u)
        for (int64_t e = off[u]; e < off[u + 1]; ++e)
            if (adj[e] > u) { E[k].w = w[e]; E[k].u = u; E[k].v = adj[e]; ++k; }
    *out = E;
    return ne;
}

/* F (out, 2*(n-1) uint32) receives the forest pairs in the order they were
 * added, Fw (out, n-1) their weights; *nf the count, *total the weight sum
 * accumulated in fp64 in that order. */
int oracle_kruskal(uint32_t n, const int64_t* off, const uint32_t* adj, const float* w, double* total,
                   uint32_t* F, float* Fw, int64_t* nf)
{
    *total = 0.0;
    *nf = 0;
    if (n == 0) return 0;
    wedge* E = NULL;
    int64_t ne = collect_edges(n, off, adj, w, &E);
    if (ne < 0) return -1;
    qsort(E, (size_t)ne, sizeof(wedge), wedge_cmp);
    uint32_t* parent = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    uint32_t* size = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    if (!parent || !size) { free(parent); free(size); free(E); return -3; }
    for (uint32_t v = 0; v < n; ++v) { parent[v] = v; size[v] = 1; }
    for (int64_t i = 0; i < ne; ++i) {
        if (dsu_find(parent, E[i].u) == dsu_find(parent, E[i].v)) continue;
        dsu_union(parent, size, E[i].u, E[i].v);
        F[2 * *nf] = E[i].u;
        F[2 * *nf + 1] = E[i].v;
        Fw[*nf] = E[i].w;
        *total += (double)E[i].w;
        ++*nf;
    }
    free(parent);
    free(size);
    free(E);
    return 0;
}

/* ---- AMSF, the folklore algorithm of P:1797-1812 --------------------------- */
/* F / Fw / *nf / *total as oracle_kruskal; Fb (out, n-1 int32) the bucket
 * index of each forest edge; *nbuckets the number of buckets up to W_max.
 * Returns -2 for a non-positive weight or eps. */
int oracle_amsf(uint32_t n, const int64_t* off, const uint32_t* adj, const float* w, double eps, double* total,
                uint32_t* F, float* Fw, int32_t* Fb, int64_t* nf, int64_t* nbuckets)
{
    *total = 0.0;
    *nf = 0;
    *nbuckets = 0;
    if (!(eps > 0.0)) return -2;
    if (n == 0) return 0;
    wedge* E = NULL;
    int64_t ne = collect_edges(n, off, adj, w, &E);
    if (ne < 0) return -1;
    if (ne == 0) { free(E); return 0; }
    /* W_min and the boundaries b_i = W_min (1+eps)^i (reading R25).  W_min / W_max
     * range over every adjacency entry as given, self-loops included (a self-loop never
     * joins the forest, but it is an element of the input edge set; reading R25) */
    const int64_t m_all = off[n];
    float wmin = w[0], wmax = w[0];
    for (int64_t i = 0; i < m_all; ++i) {
        if (!(w[i] > 0.0f) || !(w[i] <= FLT_MAX)) { free(E); return -2; }
        if (w[i] < wmin) wmin = w[i];
        if (w[i] > wmax) wmax = w[i];
    }
    const double g = 1.0 + eps;
    int64_t nb = 1;
    double bi = (double)wmin;
    while (bi * g <= (double)wmax) { bi = bi * g; ++nb; }      /* b_(nb-1) <= W_max < b_nb */
    double* b = (double*)malloc((size_t)(nb + 1) * sizeof(double));
    int32_t* bucket = (int32_t*)malloc((size_t)ne * sizeof(int32_t));
    uint32_t* parent = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    uint32_t* size = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    if (!b || !bucket || !parent || !size) { free(b); free(bucket); free(parent); free(size); free(E); return -3; }
    b[0] = (double)wmin;
    for (int64_t i = 1; i <= nb; ++i) b[i] = b[i - 1] * g;
    /* bucket of each edge: the i with b_i <= w < b_(i+1) (binary search) */
    for (int64_t e = 0; e < ne; ++e) {
        const double x = (double)E[e].w;
        int64_t lo = 0, hi = nb;                                  /* b_lo <= x < b_hi */
        while (hi - lo > 1) {
            int64_t mid = lo + (hi - lo) / 2;
            if (b[mid] <= x) lo = mid; else hi = mid;
        }
        bucket[e] = (int32_t)lo;
    }
    /* the edges of each bucket, in CSR order (u < v): a stable counting sort by bucket */
    int64_t* first = (int64_t*)calloc((size_t)nb + 1, sizeof(int64_t));
    int64_t* idx = (int64_t*)malloc((size_t)ne * sizeof(int64_t));
    if (!first || !idx) {
        free(first); free(idx); free(b); free(bucket); free(parent); free(size); free(E);
        return -3;
    }
    for (int64_t e = 0; e < ne; ++e) ++first[bucket[e] + 1];
    for (int64_t i = 0; i < nb; ++i) first[i + 1] += first[i];
    for (int64_t e = 0; e < ne; ++e) idx[first[bucket[e]]++] = e;          /* first[i] -> end of bucket i */
    for (uint32_t v = 0; v < n; ++v) { parent[v] = v; size[v] = 1; }
    /* buckets from light to heavy */
    int64_t k = 0;
    for (int64_t i = 0; i < nb; ++i)
        for (; k < first[i]; ++k) {
            const int64_t e = idx[k];
            if (dsu_find(parent, E[e].u) == dsu_find(parent, E[e].v)) continue;   /* a self-loop of C */
            dsu_union(parent, size, E[e].u, E[e].v);
            F[2 * *nf] = E[e].u;
            F[2 * *nf + 1] = E[e].v;
            Fw[*nf] = E[e].w;
            Fb[*nf] = (int32_t)i;
            *total += (double)E[e].w;
            ++*nf;
        }
    *nbuckets = nb;
    free(first);
    free(idx);
    free(b);
    free(bucket);
    free(parent);
    free(size);
    free(E);
    return 0;
}
