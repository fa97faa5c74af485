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
 * core neighbour joins the cluster of its smallest-id core neighbour; others are noise
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
 * DBSCAN by brute force (O(n^2) distance evaluations per pass).  labels: n int32.
 * counts (nullable): n int64 neighbourhood sizes (self included).  Returns K (>= 0) or
 * -1 on bad arguments / allocation failure.
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

    /* connected components of the core graph, seeds in ascending id order (BFS) */
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
                if (!core[v] || labels[v] != -1) continue;
                if (sqdist(P + v * (int64_t)d, pu, d) <= E2) { labels[v] = K; queue[tail++] = v; }
            }
        }
        ++K;
    }
    /* border points: cluster of the smallest-id core neighbour */
#pragma omp parallel for schedule(dynamic, 16)
    for (i = 0; i < n; ++i) {
        if (core[i]) continue;
        const double *pi = P + i * (int64_t)d;
        for (int64_t j = 0; j < n; ++j) {
            if (!core[j]) continue;
            if (sqdist(P + j * (int64_t)d, pi, d) <= E2) { labels[i] = labels[j]; break; }
        }
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
