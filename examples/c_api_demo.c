/* Plain-C use of the boundary (include/snn.h): build an index over host points, run a
 * self radius query, copy the CSR back, run DBSCAN.  Host pointers are staged by the
 * library; no CUDA runtime calls are needed here.
 *   gcc -std=c99 -I include examples/c_api_demo.c -L paper_2212_07679_b200/lib -lsnn \
 *       -Wl,-rpath,$PWD/paper_2212_07679_b200/lib -o /tmp/c_api_demo
 * Prints "n m nnz clusters" and exits 0 on success. */
#include <stdio.h>
#include <stdlib.h>

#include "snn.h"

#define CHECK(call)                                                         \
    do {                                                                    \
        snn_status st_ = (call);                                            \
        if (st_ != SNN_OK) {                                                \
            fprintf(stderr, "%s failed: %s\n", #call, snn_last_error());    \
            return 1;                                                       \
        }                                                                   \
    } while (0)

int main(void) {
    const int64_t n = 4096;
    const int32_t d = 2;
    float *X = (float *)malloc(sizeof(float) * n * d);
    unsigned s = 12345u;
    for (int64_t i = 0; i < n * d; ++i) {   /* LCG points in [0, 1)^2 */
        s = s * 1664525u + 1013904223u;
        X[i] = (float)(s >> 8) / 16777216.0f;
    }
    snn_index idx = NULL;
    CHECK(snn_build(X, n, d, SNN_F32, NULL, &idx));
    snn_result r = NULL;
    CHECK(snn_query_self(idx, 0.02, NULL, &r));
    snn_csr csr;
    CHECK(snn_result_csr(r, &csr));
    int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (csr.m + 1));
    int32_t *ind = (int32_t *)malloc(sizeof(int32_t) * (csr.nnz > 0 ? csr.nnz : 1));
    float *dist = (float *)malloc(sizeof(float) * (csr.nnz > 0 ? csr.nnz : 1));
    CHECK(snn_result_copy(r, off, ind, dist, NULL));
    /* every point is its own neighbour at distance 0 */
    for (int64_t i = 0; i < n; ++i) {
        int self = 0;
        for (int64_t k = off[i]; k < off[i + 1]; ++k) self |= (ind[k] == (int32_t)i && dist[k] == 0.0f);
        if (!self) { fprintf(stderr, "row %lld misses itself\n", (long long)i); return 1; }
    }
    int32_t *labels = (int32_t *)malloc(sizeof(int32_t) * n);
    int32_t k = 0;
    CHECK(snn_dbscan(idx, 0.02, 4, labels, &k, NULL));
    printf("%lld %lld %lld %d\n", (long long)n, (long long)csr.m, (long long)csr.nnz, k);
    snn_result_free(r);
    snn_free(idx);
    free(X); free(off); free(ind); free(dist); free(labels);
    return 0;
}
