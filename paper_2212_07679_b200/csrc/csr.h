// csr.h -- K11 for the pair-list (tensor-core) paths: rechecked pairs -> CSR (csr.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace snn {
// largest row the fused row sort handles (bigger rows: global radix path)
int csr_row_sort_cap();
// row_count[qperm[pq[k]]] += flag[k] (row_count zeroed); *maxrow = max row (zeroed)
void launch_pairs_row_count(const uint32_t *flag, const int32_t *pq, const int32_t *qperm, int64_t P, int64_t m,
                            int32_t *row_count, int32_t *maxrow, cudaStream_t s);
// scatter hits to their rows (cursor zeroed, tmp: nnz u64) and sort every row by sorted
// index position; out_idx = perm[position], out_dist = the recheck's distance
void launch_pairs_to_rows(const uint32_t *flag, const int32_t *pq, const int32_t *pj, const float *dist,
                          const int32_t *qperm, int64_t P, int64_t m, const int64_t *offsets, int32_t *cursor,
                          uint64_t *tmp, const int32_t *perm, int32_t max_row, int32_t *out_idx, float *out_dist,
                          cudaStream_t s);
}  // namespace snn
