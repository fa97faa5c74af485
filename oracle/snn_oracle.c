/*
 * snn_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain CPU fp64 brute-force oracle for the
 * SNN hot path (arXiv 2212.07679).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code, header,
 * table or constant with the CUDA library in paper_2212_07679_b200/.
 *
 * What it computes is the plain DEFINITION of the fixed-radius near-neighbour problem,
 * not SNN: "retrieve all data points p_i satisfying ||p_i - q|| <= R" (PAPER.md:141,
 * §3.2), which SNN returns exactly ("guaranteed to return all data points within the
 * search radius"; identical sets across methods).
 *
 * Squared distance = eq:ip1 (§4):  s = sum_k (p_k - q_k)^2, evaluated
 * left to right in IEEE fp64, one rounding per operation, NO fused multiply-add
 * (compile with -ffp-contract=off -fno-fast-math; SSE2 doubles on x86-64).
 * Membership: s <= R*R (inclusive boundary, PAPER.md:141 and Alg. 2 l.6 PAPER.md:298;
 * DESIGN.md reading C1), R*R rounded once in fp64.
 *
 * DBSCAN (§6.4) with the readings of DESIGN.md (C18): neighbourhoods
 * are closed eps-balls including the point itself; core iff count >= min_pts; clusters
 * are connected components of core points under eps-adjacency; a non-core point with a
 * core neighbour joins the first cluster that reaches it in the ascending-id scan with FIFO
 * expansion (= the smallest cluster number among its core neighbours); others are noise
 * (-1); clusters are numbered 0..K-1 in increasing order of their smallest core id.
 *
 * Parallelism: OpenMP over independent queries only; the per-pair operation sequence is
 * the one above regardless of thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* eq:ip1, left to right, no FMA. */
static double sqdist(const double *p, const double *q, int32_t d) {
    double s = 0.0;
    for (int32_t k = 0; k < d; ++k) {
        double t = p[k] - q[k];
        double t2 = t * t;
        s = s + t2;
    }
    return s;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* Squared distance of one pair, exposed so tests can pin the operation order. */
double oracle_sqdist(const double *p, const double *q, int32_t d) { return sqdist(p, q, d); }

/*
 * counts[j] = #{ i : s(p_i, q_j) <= limit },  limit = (R*R) * (1 + band_rel).
 * band_rel >= 0 widens the reported set by the tolerance band of the acceptance rule
 * (BASELINE.json north_star: pairs within 1e-5*R^2 of R^2 are tolerated); the caller
 * separates hits (s <= R*R) from band pairs using the returned s.
 */
int oracle_radius_count(const double *P, int64_t n, const double *Q, int64_t m, int32_t d,
                        double R, double band_rel, int64_t *counts) {
    if (n < 0 || m < 0 || d < 1 || R < 0.0) return 1;
    const double R2 = R * R;
    const double limit = R2 * (1.0 + band_rel);
    int64_t j;
#pragma omp parallel for schedule(dynamic, 4)
    for (j = 0; j < m; ++j) {
        const double *q = Q + j * (int64_t)d;
        int64_t c = 0;
        for (int64_t i = 0; i < n; ++i)
            if (sqdist(P + i * (int64_t)d, q, d) <= limit) ++c;
        counts[j] = c;
    }
    return 0;
}

/* Fill CSR rows (ids ascending) with the ids and fp64 squared distances. */
int oracle_radius_fill(const double *P, int64_t n, const double *Q, int64_t m, int32_t d,
                       double R, double band_rel, const int64_t *offsets, int32_t *idx,
                       double *s_out) {
    if (n < 0 || m < 0 || d < 1 || R < 0.0) return 1;
    const double R2 = R * R;
    const double limit = R2 * (1.0 + band_rel);
    int64_t j;
#pragma omp parallel for schedule(dynamic, 4)
    for (j = 0; j < m; ++j) {
        const double *q = Q + j * (int64_t)d;
        int64_t o = offsets[j];
        for (int64_t i = 0; i < n; ++i) {
            double s = sqdist(P + i * (int64_t)d, q, d);
            if (s <= limit) { idx[o] = (int32_t)i; s_out[o] = s; ++o; }
        }
    }
    return 0;
}

/*
 * DBSCAN by brute force (O(n^2) distance evaluations per pass), written as the textbook
 * algorithm the paper plugs SNN into (scikit-learn's DBSCAN, §6.4) with
 * the scan order fixed (reading C18): points are visited in
 * ascending original id; an unlabelled core point seeds a new cluster K, which is expanded
 * through a FIFO queue; every point in the eps-ball of an expanded core point that has no
 * label yet joins cluster K, and is itself expanded if it is core.  A border point (non-core
 * with a core neighbour) therefore belongs to the FIRST cluster that reaches it, clusters are
 * numbered 0..K-1 in creation order (= increasing smallest core id), and points reached by no
 * cluster are noise (-1).  labels: n int32.  counts (nullable): n int64 neighbourhood sizes
 * (self included).  Returns K (>= 0) or -1 on bad arguments / allocation failure.
 */
int64_t oracle_dbscan(const double *P, int64_t n, int32_t d, double eps, int32_t min_pts,
                      int32_t *labels, int64_t *counts) {
    if (n < 0 || d < 1 || eps < 0.0 || min_pts < 1) return -1;
    const double E2 = eps * eps;
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    char *core = (char *)malloc((size_t)(n > 0 ? n : 1));
    int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!cnt || !core || !queue) { free(cnt); free(core); free(queue); return -1; }

    int64_t i;
#pragma omp parallel for schedule(dynamic, 16)
    for (i = 0; i < n; ++i) {
        int64_t c = 0;
        for (int64_t j = 0; j < n; ++j)
            if (sqdist(P + j * (int64_t)d, P + i * (int64_t)d, d) <= E2) ++c;
        cnt[i] = c;
    }
    for (i = 0; i < n; ++i) { core[i] = cnt[i] >= min_pts; labels[i] = -1; }

    /* seeds in ascending id order, FIFO expansion from core points only */
    int32_t K = 0;
    for (i = 0; i < n; ++i) {
        if (!core[i] || labels[i] != -1) continue;
        int64_t head = 0, tail = 0;
        labels[i] = K;
        queue[tail++] = i;
        while (head < tail) {
            int64_t u = queue[head++];
            const double *pu = P + u * (int64_t)d;
            for (int64_t v = 0; v < n; ++v) {
                if (labels[v] != -1) continue;
                if (sqdist(P + v * (int64_t)d, pu, d) <= E2) {
                    labels[v] = K;
                    if (core[v]) queue[tail++] = v;
                }
            }
        }
        ++K;
    }
    if (counts) memcpy(counts, cnt, sizeof(int64_t) * (size_t)n);
    free(cnt); free(core); free(queue);
    return K;
}

/*
 * Per-point DBSCAN facts for SAMPLED points of a large instance (checked one by one):
 * for each sampled id s: count (self incl.), and the smallest-id core neighbour given a
 * core flag array (from the system under test or from counts computed here).
 */
int oracle_neighbour_counts(const double *P, int64_t n, int32_t d, double eps,
                            const int64_t *ids, int64_t k, int64_t *counts) {
    if (n < 0 || d < 1 || eps < 0.0) return 1;
    const double E2 = eps * eps;
    int64_t t;
#pragma omp parallel for schedule(dynamic, 1)
    for (t = 0; t < k; ++t) {
        const double *q = P + ids[t] * (int64_t)d;
        int64_t c = 0;
        for (int64_t j = 0; j < n; ++j)
            if (sqdist(P + j * (int64_t)d, q, d) <= E2) ++c;
        counts[t] = c;
    }
    return 0;
}

/* ==========================================================================================
 * Grid-bucketed exact variants for d <= 3 (test infrastructure for FULL-SIZE parity:
 * SURVEY.md §8(d) "an exact grid-pruned variant for d <= 3 keeps the same per-pair
 * arithmetic, so its results are identical").  They return exactly what the brute-force
 * functions above return -- the pair test is the same sqdist() against the same limit --
 * but only evaluate pairs whose grid cells are adjacent.  Why no hit is skipped:
 *
 *   cell side h = max(sqrt(limit) * (1 + 1e-6), ext / 2^20) > 0, ext = largest coordinate
 *   range, cell_k(x) = floor(fl(fl(x_k - lo_k) / h)).  If s(p, q) <= limit then, with exact
 *   arithmetic, |p_k - q_k| <= ||p - q|| <= sqrt(s (1 + 2^-50)) < sqrt(limit)(1 + 1e-15).
 *   The two roundings change each quotient by at most 2^-52 * ext / h <= 2^-32 (ext/h <= 2^20),
 *   so the computed quotients differ by less than (1 + 1e-15)/(1 + 1e-6) + 2^-31 < 1 and
 *   their floors by at most 1: q lies in one of the 3^d cells around p.
 *
 * (h grows when the data's extent is large relative to R; a larger cell only adds pairs.)
 * Tested against the brute force above in tests/test_oracle.py (random, lattice points on
 * cell boundaries, duplicates, R = 0).
 * ========================================================================================== */
typedef struct {
    int32_t d;
    double lo[3], h;
    int64_t dim[3];          /* cells per axis */
    int64_t *key;            /* sorted cell keys of P (n) */
    int64_t *ord;            /* P ids in cell order (n) */
    int64_t n;
} grid_t;

static int64_t cell_of(const grid_t *g, const double *x, int32_t k) {
    double c = floor((x[k] - g->lo[k]) / g->h);
    if (c < 0.0) c = 0.0;                        /* queries outside P's box: clamp (safe: */
    if (c > (double)(g->dim[k] - 1)) c = (double)(g->dim[k] - 1);   /* clamped cells only merge) */
    return (int64_t)c;
}

static int64_t key_of(const grid_t *g, const int64_t *c) {
    int64_t key = 0;
    for (int32_t k = 0; k < g->d; ++k) key = key * g->dim[k] + c[k];
    return key;
}

static const int64_t *g_sort_key;
static int cmp_key(const void *a, const void *b) {
    int64_t ka = g_sort_key[*(const int64_t *)a], kb = g_sort_key[*(const int64_t *)b];
    if (ka != kb) return ka < kb ? -1 : 1;
    int64_t ia = *(const int64_t *)a, ib = *(const int64_t *)b;
    return ia < ib ? -1 : (ia > ib);
}

/* Build the grid over P (n x d, d <= 3) and the query set Q for search limit `limit`.
 * Returns 0, or 1 on bad input (d > 3, non-finite coordinates, allocation). */
static int grid_build(grid_t *g, const double *P, int64_t n, const double *Q, int64_t m,
                      int32_t d, double limit) {
    if (d < 1 || d > 3 || n < 0 || m < 0 || !(limit >= 0.0)) return 1;
    memset(g, 0, sizeof(*g));
    g->d = d; g->n = n;
    double hi[3];
    for (int32_t k = 0; k < d; ++k) { g->lo[k] = INFINITY; hi[k] = -INFINITY; }
    for (int pass = 0; pass < 2; ++pass) {
        const double *A = pass ? Q : P;
        int64_t cnt = pass ? m : n;
        for (int64_t i = 0; i < cnt; ++i)
            for (int32_t k = 0; k < d; ++k) {
                double v = A[i * (int64_t)d + k];
                if (!isfinite(v)) return 1;
                if (v < g->lo[k]) g->lo[k] = v;
                if (v > hi[k]) hi[k] = v;
            }
    }
    double ext = 0.0;
    for (int32_t k = 0; k < d; ++k) {
        if (!(g->lo[k] <= hi[k])) { g->lo[k] = 0.0; hi[k] = 0.0; }
        if (hi[k] - g->lo[k] > ext) ext = hi[k] - g->lo[k];
    }
    double h = sqrt(limit) * (1.0 + 1e-6);
    if (h < ext / 1048576.0) h = ext / 1048576.0;
    if (!(h > 0.0)) h = 1.0;                     /* all points identical and R = 0 */
    g->h = h;
    for (int32_t k = 0; k < d; ++k) g->dim[k] = (int64_t)floor((hi[k] - g->lo[k]) / h) + 1;
    g->key = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    g->ord = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *pk = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!g->key || !g->ord || !pk) { free(g->key); free(g->ord); free(pk); return 1; }
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < n; ++i) {
        int64_t c[3];
        for (int32_t k = 0; k < d; ++k) c[k] = cell_of(g, P + i * (int64_t)d, k);
        pk[i] = key_of(g, c);
        g->ord[i] = i;
    }
    g_sort_key = pk;
    qsort(g->ord, (size_t)n, sizeof(int64_t), cmp_key);
    for (i = 0; i < n; ++i) g->key[i] = pk[g->ord[i]];
    free(pk);
    return 0;
}

static void grid_free(grid_t *g) { free(g->key); free(g->ord); }

/* first position in the sorted key array with key >= k */
static int64_t lower(const grid_t *g, int64_t k) {
    int64_t a = 0, b = g->n;
    while (a < b) { int64_t mid = a + (b - a) / 2; if (g->key[mid] < k) a = mid + 1; else b = mid; }
    return a;
}

/* Visit every P id in the 3^d cells around query point q (any order); calls back with
 * the id.  Returns the number of ids visited. */
typedef void (*visit_fn)(void *ctx, int64_t i);
static void grid_visit(const grid_t *g, const double *q, visit_fn fn, void *ctx) {
    int64_t c[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int32_t k = 0; k < g->d; ++k) {
        int64_t ck = cell_of(g, q, k);
        lo[k] = ck > 0 ? ck - 1 : 0;
        hi[k] = ck + 1 < g->dim[k] ? ck + 1 : g->dim[k] - 1;
    }
    /* the last axis is contiguous in key space: one range per (c0, c1) */
    int32_t L = g->d - 1;
    for (c[0] = lo[0]; c[0] <= (L > 0 ? hi[0] : lo[0]); ++c[0])
        for (c[1] = lo[1]; c[1] <= (L > 1 ? hi[1] : lo[1]); ++c[1]) {
            int64_t cc[3] = {c[0], c[1], 0};
            cc[L] = lo[L];
            int64_t a = lower(g, key_of(g, cc));
            cc[L] = hi[L];
            int64_t b = lower(g, key_of(g, cc) + 1);
            for (int64_t t = a; t < b; ++t) fn(ctx, g->ord[t]);
        }
}

typedef struct {
    const double *P, *q;
    int32_t d;
    double limit;
    int64_t c;          /* count */
    int32_t *idx;       /* fill: ids */
    double *s;          /* fill: squared distances */
} rq_ctx;

static void rq_count(void *v, int64_t i) {
    rq_ctx *x = (rq_ctx *)v;
    if (sqdist(x->P + i * (int64_t)x->d, x->q, x->d) <= x->limit) ++x->c;
}
static void rq_fill(void *v, int64_t i) {
    rq_ctx *x = (rq_ctx *)v;
    double s = sqdist(x->P + i * (int64_t)x->d, x->q, x->d);
    if (s <= x->limit) { x->idx[x->c] = (int32_t)i; x->s[x->c] = s; ++x->c; }
}

/* ascending ids within a row (the brute force's order), s permuted along */
static void sort_row(int32_t *idx, double *s, int64_t k) {
    for (int64_t a = 1; a < k; ++a) {           /* insertion sort: rows are short */
        int32_t ia = idx[a]; double sa = s[a]; int64_t b = a;
        while (b > 0 && idx[b - 1] > ia) { idx[b] = idx[b - 1]; s[b] = s[b - 1]; --b; }
        idx[b] = ia; s[b] = sa;
    }
}

/* Same contract as oracle_radius_count / oracle_radius_fill (d <= 3). */
int oracle_grid_radius_count(const double *P, int64_t n, const double *Q, int64_t m, int32_t d,
                             double R, double band_rel, int64_t *counts) {
    if (R < 0.0) return 1;
    const double R2 = R * R, limit = R2 * (1.0 + band_rel);
    grid_t g;
    if (grid_build(&g, P, n, Q, m, d, limit)) return 1;
    int64_t j;
#pragma omp parallel for schedule(dynamic, 64)
    for (j = 0; j < m; ++j) {
        rq_ctx x = {P, Q + j * (int64_t)d, d, limit, 0, NULL, NULL};
        grid_visit(&g, x.q, rq_count, &x);
        counts[j] = x.c;
    }
    grid_free(&g);
    return 0;
}

int oracle_grid_radius_fill(const double *P, int64_t n, const double *Q, int64_t m, int32_t d,
                            double R, double band_rel, const int64_t *offsets, int32_t *idx,
                            double *s_out) {
    if (R < 0.0) return 1;
    const double R2 = R * R, limit = R2 * (1.0 + band_rel);
    grid_t g;
    if (grid_build(&g, P, n, Q, m, d, limit)) return 1;
    int64_t j;
#pragma omp parallel for schedule(dynamic, 64)
    for (j = 0; j < m; ++j) {
        rq_ctx x = {P, Q + j * (int64_t)d, d, limit, 0, idx + offsets[j], s_out + offsets[j]};
        grid_visit(&g, x.q, rq_fill, &x);
        sort_row(x.idx, x.s, x.c);
    }
    grid_free(&g);
    return 0;
}

/* ---- grid DBSCAN (d <= 3): same result as oracle_dbscan, by components ----------------
 * counts over the grid; clusters = connected components of the core graph by union-find
 * (union of core i with every core neighbour j > i); canonical numbering by increasing
 * smallest core id (= the FIFO scan's creation order); a border point takes the smallest
 * cluster number among its core neighbours (= the first cluster that reaches it in the
 * FIFO scan, since cluster c is expanded completely before cluster c+1 starts). */
static int64_t uf_find(int64_t *par, int64_t x) {
    while (par[x] != x) { par[x] = par[par[x]]; x = par[x]; }
    return x;
}

typedef struct {
    const double *P, *q;
    int32_t d;
    double E2;
    int64_t self, c;
    const char *core;
    int64_t *par;
    const int32_t *lab;
    int32_t best;
} db_ctx;

static void db_count(void *v, int64_t i) {
    db_ctx *x = (db_ctx *)v;
    if (sqdist(x->P + i * (int64_t)x->d, x->q, x->d) <= x->E2) ++x->c;
}
static void db_union(void *v, int64_t j) {
    db_ctx *x = (db_ctx *)v;
    if (j <= x->self || !x->core[j]) return;
    int64_t a = uf_find(x->par, x->self), b = uf_find(x->par, j);
    if (a == b) return;                                  /* already joined: union is a no-op */
    if (sqdist(x->P + j * (int64_t)x->d, x->q, x->d) <= x->E2) {
        if (a < b) x->par[b] = a; else x->par[a] = b;
    }
}
static void db_border(void *v, int64_t j) {
    db_ctx *x = (db_ctx *)v;
    if (!x->core[j] || x->lab[j] >= x->best) return;
    if (sqdist(x->P + j * (int64_t)x->d, x->q, x->d) <= x->E2) x->best = x->lab[j];
}

int64_t oracle_grid_dbscan(const double *P, int64_t n, int32_t d, double eps, int32_t min_pts,
                           int32_t *labels, int64_t *counts) {
    if (n < 0 || d < 1 || d > 3 || eps < 0.0 || min_pts < 1) return -1;
    const double E2 = eps * eps;
    grid_t g;
    if (grid_build(&g, P, n, P, 0, d, E2)) return -1;
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *par = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    char *core = (char *)malloc((size_t)(n > 0 ? n : 1));
    int32_t *rootlab = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (!cnt || !par || !core || !rootlab) {
        free(cnt); free(par); free(core); free(rootlab); grid_free(&g); return -1;
    }
    int64_t i;
#pragma omp parallel for schedule(dynamic, 256)
    for (i = 0; i < n; ++i) {
        db_ctx x = {P, P + i * (int64_t)d, d, E2, i, 0, NULL, NULL, NULL, 0};
        grid_visit(&g, x.q, db_count, &x);
        cnt[i] = x.c;
    }
    for (i = 0; i < n; ++i) { core[i] = cnt[i] >= min_pts; par[i] = i; labels[i] = -1; rootlab[i] = -1; }
    for (i = 0; i < n; ++i) {                            /* sequential union-find */
        if (!core[i]) continue;
        db_ctx x = {P, P + i * (int64_t)d, d, E2, i, 0, core, par, NULL, 0};
        grid_visit(&g, x.q, db_union, &x);
    }
    int32_t K = 0;
    for (i = 0; i < n; ++i) {                            /* numbering by smallest core id */
        if (!core[i]) continue;
        int64_t r = uf_find(par, i);
        if (rootlab[r] < 0) rootlab[r] = K++;
        labels[i] = rootlab[r];
    }
#pragma omp parallel for schedule(dynamic, 256)
    for (i = 0; i < n; ++i) {
        if (core[i]) continue;
        db_ctx x = {P, P + i * (int64_t)d, d, E2, i, 0, core, NULL, labels, 0x7fffffff};
        grid_visit(&g, x.q, db_border, &x);
        if (x.best != 0x7fffffff) labels[i] = x.best;
    }
    if (counts) memcpy(counts, cnt, sizeof(int64_t) * (size_t)n);
    free(cnt); free(par); free(core); free(rootlab); grid_free(&g);
    return K;
}
