// index.h -- the opaque handle types of include/snn.h and small runtime helpers shared
// by api.cu and dbscan.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/snn.h"
#include "internal.h"

namespace snn {
snn_status fail(snn_status st, const std::string &msg);
// kernel-time profiler families (snn_profile_*)
enum Fam { F_BUILD = 0, F_COUNT = 1, F_WRITE = 2, F_QUERY = 3, F_DBSCAN = 4, F_UNION = 5, F_N = 6 };
int prof_begin(int fam, cudaStream_t s);                 // -1 when profiling is off
void prof_end(int tok, cudaStream_t s, double units);
snn_status cuda_fail(cudaError_t e, const char *where);
bool is_device_ptr(const void *p);

// Stream-ordered workspace: every allocation is freed on the same stream at scope exit.
struct Workspace {
    cudaStream_t s;
    std::vector<void *> ptrs;
    explicit Workspace(cudaStream_t st) : s(st) {}
    ~Workspace() {
        for (void *p : ptrs) cudaFreeAsync(p, s);
    }
    template <typename T>
    cudaError_t alloc(T **out, size_t count) {
        void *p = nullptr;
        size_t bytes = count * sizeof(T);
        if (bytes == 0) bytes = 16;
        cudaError_t e = cudaMallocAsync(&p, bytes, s);
        if (e == cudaSuccess) ptrs.push_back(p);
        *out = static_cast<T *>(p);
        return e;
    }
    void free_all() {
        for (void *p : ptrs) cudaFreeAsync(p, s);
        ptrs.clear();
    }
    void release(void *p) {   // hand ownership to the caller
        std::vector<void *> keep;
        for (void *q : ptrs) if (q != p) keep.push_back(q);
        ptrs.swap(keep);
    }
};
}  // namespace snn

struct snn_index_s {
    int64_t n = 0, n_pad = 0;
    int d = 0, ld = 0;
    snn_dtype dt = SNN_F32;
    void *Xs = nullptr;        // n_pad x ld, original coordinates in key order
    float *keys = nullptr;     // n sorted keys
    int32_t *perm = nullptr;   // n: sorted position -> original id
    float *xbar = nullptr;     // n_pad half squared norms (centered)
    double *mu_d = nullptr;
    float *mu_f = nullptr;
    double *v_d = nullptr;
    float *v_f = nullptr;
    double *stats = nullptr;   // ST_COUNT doubles
    double *G = nullptr;       // d x d Gram of the centred build data (spectrum diagnostics)
    double h_stats[snn::ST_COUNT] = {};
    int sm_count = 148;
    int tc = 0;                // tensor-core (tcgen05) query path enabled
    int tc_f16 = 0;            // operands FP16 (kind::f16, scaled by 2^xexp) instead of TF32
    int xexp = 0;              // FP16 operand scale exponent of the index copy
    int kpad = 0;              // K padded to 64 (FP16) / 32 (TF32)
    void *Xt = nullptr;        // n x kpad centred tensor-core operand copy (FP16 or TF32)
    int metric = 0;            // snn_metric (COSINE / ANGULAR: rows normalized at build; MIPS: d = input d + 1)
    int d_in = 0;              // input dimension (d - 1 for MIPS)
    void *Xo = nullptr;        // MANHATTAN / MIPS: input rows, original order (post-filter)
    double xi2 = 0.0;          // MIPS: max_i ||p_i||^2
    float *Xf = nullptr;       // low-d fp32: expanded-form filter rows (AoSoA4, d+1 floats)
    double xf_c1h = 1.0;       // c1h the filter rows were built with
    std::vector<void *> owned;
};

struct snn_result_s {
    int64_t m = 0, nnz = 0;
    cudaEvent_t copy_done = nullptr;   // snn_result_copy_async: frees wait for this event
    int64_t *offsets = nullptr;
    int32_t *indices = nullptr;
    float *distances = nullptr;
};


namespace snn {
bool dbscan_simt_filter();   // option simt_filter (api.cu)
int dbscan_union_load();     // option union_load (api.cu)
int dbscan_count_warp();     // option count_warp (api.cu)
int dbscan_union_snap();     // option union_snap (api.cu)
bool dbscan_union_phased();  // option union_phased (api.cu)
bool dbscan_union_behind();  // option union_behind (api.cu)
int dbscan_union_chunk();    // option union_chunk (api.cu)
int dbscan_block();          // option dbscan_block (api.cu)
int dbscan_union_seed();     // option union_seed (api.cu): seed scan steps of 32 positions (0 = off)
bool dbscan_union_stats();   // option union_stats (api.cu)
void dbscan_set_union_stats(const unsigned long long *v);   // [path, hits, links] of the last union pass
// metric adapters (metric.cu): exact row normalization (flag = 1 on a zero row), radius
// mapping and in-place distance conversion
void launch_normalize_rows(const void *X, bool f64, int64_t n, int d, void *out, int *zero_flag, cudaStream_t s);
double metric_radius(int metric, double r);
void launch_metric_distances(int metric, float *dist, int64_t nnz, cudaStream_t s);
void launch_sq_norms(const void *X, bool f64, int64_t n, int d, double *nrm2, unsigned long long *max_bits,
                     cudaStream_t s);
void launch_mips_rows(const void *X, bool f64, int64_t n, int d, const double *nrm2,
                      const unsigned long long *xi2_bits, void *out, cudaStream_t s);
void launch_csr_filter(int metric, bool f64, const int64_t *off, int64_t m, const int32_t *ind, const void *Xo,
                       const void *Qo, int d, double thr, uint8_t *keep, float *val, int32_t *rowcnt, cudaStream_t s);
void launch_csr_compact(const int64_t *off, int64_t m, const int32_t *ind, const uint8_t *keep, const float *val,
                        const int64_t *noff, int32_t *nind, float *ndist, cudaStream_t s);
snn_status dbscan_from_csr(const int64_t *off, const int32_t *nidx, int64_t n, int32_t min_pts, int32_t *labels,
                           int32_t *n_clusters, cudaStream_t s);
snn_status dbscan_impl(snn_index idx, double eps, int32_t min_pts, int32_t *labels,
                       int32_t *n_clusters, cudaStream_t s);
}
