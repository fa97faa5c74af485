// api.cu -- the C ABI (include/snn.h) and the host runtime around the kernels: argument
// validation, device / memory-pool setup, stream-ordered workspaces, the launch
// sequences of Algorithm 1 (build) and Algorithm 2 (query), and result ownership.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/snn.h"
#include "common.cuh"
#include "internal.h"
#include "query.h"
#include "tc.h"
#include "csr.h"
#include "index.h"

namespace snn {

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct Options {
    int force_generic = 0;
    int query_block = 256;
    int chunk = 2048;
    int power_iters = 1000;
    int cap = 64;
    int32_t ovf_rec_cap = 1 << 20;
    int variant = 1;
    int scan2q = 0;      // fp32 low-d scan with the expanded filter, two queries per thread: 0 = auto (d >= 2), 1 = on, -1 = off
    int chunk2q = 640;   // candidates per work item of that scan (128-thread CTAs: smaller chunks keep 7 CTAs per SM)
    int tc = 1;          // use the tcgen05 path for d >= tc_min_d
    int tc_min_d = 32;
    int tc_tiles = 8;    // 256-candidate tiles per work item on the tensor-core path
    int tc_diag = 0;     // diagnostics only (results invalid): 1 = no epilogue work, 2 = no MMA, 3 = no MMA and no hit path, 4 = no hit path
    int tc_f16 = 1;      // tensor-core operands FP16 (scaled) instead of TF32
    int tc_ares = 1;     // K9: query tile resident per work item when K is one block
    int tc_group = 128;  // query blocks per raster group (upper bound; L2 budget decides)
    int tc_wait_hint = 0;   // K9 mbarrier waits: suspend-time hint in ns (0 = probe loop)
    int tc_warp_arrive = 1;   // K9 epilogue: one mbarrier arrive per warp (-1: per thread)
    int tc_gram_min_d = 32;    // Gram matrix on the tensor cores for d >= this
    int symmetric = 1;   // low-d self-queries: each unordered pair evaluated once
    int stage_rows = 0;  // low-d: 1 = assemble rows in key order, then move each row whole (0: direct final rows)
    int balanced_compact = 1;   // low-d compaction: one slot record per thread (CTA scans)
    int window_all = 0;  // ablation "brute force 2": windows = all points
    // low-d fp32 expanded-form SIMT pre-filter: 0 = default (radius queries on: faster on
    // c2; DBSCAN passes off: dense hits make it slower on c5), 1 = on everywhere, -1 = off
    int simt_filter = 0;
    int lowd_tc = 0;     // low-d (fp32, d <= 8) radius queries through the tensor-core filter (option; FFMA default)
    int lowd_tc_tiles = 8;     // 256-candidate tiles per work item (low-d tensor-core path)
    int lowd_tc_group = 8;     // query blocks per raster group (low-d tensor-core path)
    int union_load = 1;        // DBSCAN union pass: parent pre-check load (0 volatile, 1 relaxed.gpu, 2 ld.cg)
    int count_warp = 1;        // DBSCAN core counts: warp per point, outward scan (-1: CTA per block)
    int union_snap = 1;        // DBSCAN union pass (fp32, d <= 8): staged parent snapshot pre-check (-1: window_lowd)
    int union_behind = 1;      // DBSCAN union pass (union_snap): candidates behind the block (pairs j < i)
    int dbscan_block = 256;    // DBSCAN: queries per block (windows, union and border passes)
    int union_seed = 8;        // DBSCAN union pass (union_snap, behind): seed pass uniting each core point with its nearest core neighbour behind (steps of 32 positions; 0 = off)
    int union_chunk = 512;     // DBSCAN union pass (union_snap): candidates per work item
    int union_phased = 0;      // DBSCAN union pass (union_snap): chunk k of every block in launch k (near pairs first)
    int union_stats = 0;       // DBSCAN union pass: count pairs sent to the union path (diagnostics)
    int finalize_order = 1;    // staged rows: rows_finalize walks rows in original-id order (sequential CSR writes)
    int lkey = 1;              // symmetric direct rows: mirrored entries gathered in key order (-1: at the CSR rows)
    int finalize_pipe = 1;     // symmetric direct rows: 32 rows per warp, software-pipelined (-1: warp per row)
    int gram_rows = 65536;     // tensor-core Gram of a large build: rows sampled (stride) down to ~this many
    int64_t gram_min_elems = int64_t(1) << 27;   // ... when n*d is at least this
};
// Options are per calling thread (snn_set_option changes only the calling thread's calls;
// every thread starts from the defaults above), so concurrent callers cannot switch each
// other's paths.  The last-query diagnostics are per thread for the same reason.
static thread_local int64_t g_last_ovf = 0, g_last_lost = 0;
static thread_local Options g_opt;

static thread_local std::string t_err;

// ------------------------------------------------------------------ kernel-time profiler
static const char *kFamNames[F_N] = {"build", "window_count", "window_write", "query", "dbscan", "dbscan_union"};
struct ProfRec {
    int fam;
    cudaEvent_t a, b;
    double units;
};
struct Profiler {
    std::mutex mu;
    bool on = false;
    std::vector<ProfRec> pending;
    double ms[F_N] = {}, units[F_N] = {};
    uint64_t launches[F_N] = {};
};
static Profiler g_prof;

int prof_begin(int fam, cudaStream_t s) {
    if (!g_prof.on) return -1;
    ProfRec r{fam, nullptr, nullptr, 0.0};
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    cudaEventRecord(r.a, s);
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.pending.push_back(r);
    return (int)g_prof.pending.size() - 1;
}
void prof_end(int tok, cudaStream_t s, double units) {
    if (tok < 0 || !g_prof.on) return;
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (tok >= (int)g_prof.pending.size()) return;
    g_prof.pending[tok].units = units;
    cudaEventRecord(g_prof.pending[tok].b, s);
}
static void prof_drain() {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (auto &r : g_prof.pending) {
        float ms = 0.f;
        cudaEventSynchronize(r.b);
        if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
            g_prof.ms[r.fam] += ms;
            g_prof.units[r.fam] += r.units;
            g_prof.launches[r.fam] += 1;
        }
        cudaGetLastError();
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_prof.pending.clear();
}

bool dbscan_simt_filter() { return g_opt.simt_filter > 0; }
int dbscan_count_warp() { return g_opt.count_warp; }
int dbscan_union_load() { return g_opt.union_load; }
int dbscan_union_snap() { return g_opt.union_snap; }
bool dbscan_union_phased() { return g_opt.union_phased > 0; }
bool dbscan_union_behind() { return g_opt.union_behind > 0; }
int dbscan_union_chunk() { return g_opt.union_chunk; }
int dbscan_block() { return g_opt.dbscan_block; }
int dbscan_union_seed() { return g_opt.union_seed; }
static thread_local int64_t g_last_union[3] = {0, 0, 0};
bool dbscan_union_stats() { return g_opt.union_stats > 0; }
void dbscan_set_union_stats(const unsigned long long *v) {
    for (int i = 0; i < 3; ++i) g_last_union[i] = (int64_t)v[i];
}

snn_status fail(snn_status st, const std::string &msg) {
    t_err = msg;
    return st;
}

snn_status cuda_fail(cudaError_t e, const char *where) {
    cudaGetLastError();   // clear sticky-free errors
    if (e == cudaErrorMemoryAllocation) return fail(SNN_ERR_OUT_OF_MEMORY, std::string(where) + ": out of device memory");
    return fail(SNN_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr, where)                                      \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return cuda_fail(_e, where);  \
    } while (0)

struct DeviceInfo {
    int ok = -1;   // -1 unknown, 0 unsupported, 1 ok
    int sm_count = 148;
};
static std::mutex g_dev_mu;
static DeviceInfo g_dev[64];

snn_status device_check(int *sm_count) {
    int dev = 0;
    CK(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= 64) return fail(SNN_ERR_UNSUPPORTED, "device ordinal out of range");
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DeviceInfo &di = g_dev[dev];
    if (di.ok < 0) {
        int major = 0, minor = 0, sms = 0;
        CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev), "attr");
        CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev), "attr");
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
        di.ok = (major == 10 && minor == 0) ? 1 : 0;
        di.sm_count = sms;
        if (di.ok) {   // keep freed stream-ordered memory in the pool (no per-call cudaMalloc)
            cudaMemPool_t pool;
            CK(cudaDeviceGetDefaultMemPool(&pool, dev), "mempool");
            uint64_t thr = UINT64_MAX;
            CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr), "mempool");
        }
    }
    if (!di.ok) return fail(SNN_ERR_UNSUPPORTED, "this library is built for sm_100a (B200) only");
    *sm_count = di.sm_count;
    return SNN_OK;
}

bool is_device_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// small pinned host staging for scalar read-backs
struct Pinned {
    void *p = nullptr;
    Pinned() { cudaMallocHost(&p, 4096); }
    ~Pinned() { if (p) cudaFreeHost(p); }
};
static thread_local Pinned t_pinned;

// row stride of the sorted copy: 0 = AoSoA4 layout (low-d kernels), else padded row-major
int generic_stride(int d) { return d == 1 ? 1 : d == 2 ? 2 : (int)round_up(d, 4); }
int row_stride(int d) {
    if (lowd_supported(d) && !g_opt.force_generic) return 0;
    return generic_stride(d);
}
int64_t row_elems(int d, int ld) { return ld ? ld : d; }

}  // namespace snn

using namespace snn;

// FP16 tensor-core operands: scale 2^e with bound * 2^e in [2^14, 2^15) (no overflow; the
// subnormal range only adds the absolute error term of the margin).  false if the bound
// needs |e| > 60 (the TF32 / generic paths are used instead).
static bool f16_exponent(double bound, int *e) {
    if (!(bound > 0.0)) { *e = 0; return true; }
    if (!std::isfinite(bound)) return false;
    const int ex = 14 - ilogb(bound);
    if (ex < -60 || ex > 60) return false;
    *e = ex;
    return bound * ldexp(1.0, ex) < 32768.0;
}

// Query sharding across GPUs: set for the duration of one
// snn_query_*_part call on this thread, read by every query path after its K7 windows.
struct PartSpec { int part = 0, nparts = 1; };
static thread_local PartSpec t_part;
struct PartGuard {
    PartGuard(int p, int n) { t_part.part = p; t_part.nparts = n; }
    ~PartGuard() { t_part = PartSpec(); }
};
static cudaError_t apply_part(Workspace &ws, cudaStream_t s, int64_t *blk_lo, int64_t *blk_hi, int64_t *nitems,
                              int64_t nblocks) {
    if (t_part.nparts <= 1 || nblocks == 0) return cudaSuccess;
    int64_t *tmp = nullptr;
    uint8_t *st = nullptr;
    cudaError_t e = ws.alloc(&tmp, (size_t)(2 * nblocks + 1));
    if (e == cudaSuccess) e = ws.alloc(&st, scan_temp_bytes(nblocks) + 4096);
    if (e != cudaSuccess) return e;
    launch_restrict_part(blk_lo, blk_hi, nitems, nblocks, t_part.part, t_part.nparts, tmp, st, s);
    return cudaGetLastError();
}

static void free_index(snn_index idx) {
    if (!idx) return;
    for (void *p : idx->owned) cudaFreeAsync(p, 0);
    delete idx;
}

// Padding rows [n, n_pad) as the build writes them: NaN coordinates (zero stride padding),
// NaN half norms, filter rows x_c = 0 with xbar' = +inf (build.cu gather_*, query.cu
// filter_rows_kernel).
template <typename T>
__global__ void restore_sentinels(T *Xs, int ld, int D, int64_t n, int64_t n_pad, float *xbar, float *Xf) {
    for (int64_t t = threadIdx.x; t < (n_pad - n) * (ld ? ld : D); t += blockDim.x) {
        const int64_t i = n + t / (ld ? ld : D);
        const int k = (int)(t % (ld ? ld : D));
        if (ld) Xs[i * ld + k] = k < D ? (T)NAN : (T)0;
        else Xs[(i >> 2) * 4 * D + 4 * k + (i & 3)] = (T)NAN;
    }
    for (int64_t i = n + threadIdx.x; i < n_pad; i += blockDim.x) {
        xbar[i] = NAN;
        if (Xf) {
            float *o = Xf + (i >> 2) * 4 * (D + 1) + (i & 3);
            for (int k = 0; k < D; ++k) o[4 * k] = 0.f;
            o[4 * D] = INFINITY;
        }
    }
}

extern "C" {

snn_status snn_profile_enable(int on) {
    prof_drain();
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = on != 0;
    for (int f = 0; f < F_N; ++f) { g_prof.ms[f] = 0; g_prof.units[f] = 0; g_prof.launches[f] = 0; }
    return SNN_OK;
}

snn_status snn_profile_read(const char *family, double *ms, uint64_t *launches, double *units) {
    if (!family) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL family");
    prof_drain();
    if (strcmp(family, "overflow") == 0) {   // hit-slot overflows of the last low-d query
        if (ms) *ms = 0.0;
        if (launches) *launches = 0;
        if (units) *units = (double)g_last_ovf;
        return SNN_OK;
    }
    if (strcmp(family, "lost") == 0) {   // items re-run by the fix pass in the last query
        if (ms) *ms = 0.0;
        if (launches) *launches = 0;
        if (units) *units = (double)g_last_lost;
        return SNN_OK;
    }
    for (int f = 0; f < F_N; ++f) {
        if (strcmp(family, kFamNames[f]) == 0) {
            if (ms) *ms = g_prof.ms[f];
            if (launches) *launches = g_prof.launches[f];
            if (units) *units = g_prof.units[f];
            return SNN_OK;
        }
    }
    return fail(SNN_ERR_INVALID_ARGUMENT, std::string("unknown profile family ") + family);
}

const char *snn_last_error(void) { return t_err.c_str(); }
uint64_t snn_launch_count(void) { return g_launches.load(); }

snn_status snn_get_option(const char *key, int64_t *value) {
    if (!key || !value) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL argument");
    static const struct { const char *name; int Options::*field; } kInt[] = {
        {"force_generic", &Options::force_generic}, {"query_block", &Options::query_block},
        {"chunk", &Options::chunk}, {"power_iters", &Options::power_iters}, {"cap", &Options::cap},
        {"variant", &Options::variant}, {"scan2q", &Options::scan2q}, {"chunk2q", &Options::chunk2q}, {"tc", &Options::tc}, {"tc_min_d", &Options::tc_min_d},
        {"tc_tiles", &Options::tc_tiles}, {"tc_diag", &Options::tc_diag}, {"tc_f16", &Options::tc_f16},
        {"tc_ares", &Options::tc_ares}, {"tc_group", &Options::tc_group},
        {"tc_wait_hint", &Options::tc_wait_hint}, {"tc_warp_arrive", &Options::tc_warp_arrive},
        {"tc_gram_min_d", &Options::tc_gram_min_d}, {"symmetric", &Options::symmetric},
        {"stage_rows", &Options::stage_rows}, {"balanced_compact", &Options::balanced_compact},
        {"window_all", &Options::window_all}, {"simt_filter", &Options::simt_filter},
        {"lowd_tc", &Options::lowd_tc}, {"lowd_tc_tiles", &Options::lowd_tc_tiles},
        {"lowd_tc_group", &Options::lowd_tc_group}, {"union_load", &Options::union_load},
        {"finalize_order", &Options::finalize_order}, {"finalize_pipe", &Options::finalize_pipe}, {"lkey", &Options::lkey},
        {"gram_rows", &Options::gram_rows},
        {"count_warp", &Options::count_warp}, {"union_snap", &Options::union_snap},
        {"union_stats", &Options::union_stats}, {"union_phased", &Options::union_phased},
        {"union_behind", &Options::union_behind}, {"union_chunk", &Options::union_chunk},
        {"dbscan_block", &Options::dbscan_block}, {"union_seed", &Options::union_seed}};
    for (const auto &o : kInt)
        if (strcmp(key, o.name) == 0) { *value = g_opt.*(o.field); return SNN_OK; }
    if (strcmp(key, "ovf_records") == 0) { *value = g_opt.ovf_rec_cap; return SNN_OK; }
    if (strcmp(key, "gram_min_elems") == 0) { *value = g_opt.gram_min_elems; return SNN_OK; }
    // read-only diagnostics of this thread's last DBSCAN union pass (option union_stats)
    if (strcmp(key, "last_union_path") == 0) { *value = g_last_union[0]; return SNN_OK; }
    if (strcmp(key, "last_union_hits") == 0) { *value = g_last_union[1]; return SNN_OK; }
    if (strcmp(key, "last_union_links") == 0) { *value = g_last_union[2]; return SNN_OK; }
    return fail(SNN_ERR_INVALID_ARGUMENT, std::string("unknown option ") + key);
}

snn_status snn_set_option(const char *key, int64_t value) {
    if (!key) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL option key");
    std::string k(key);
    if (k == "force_generic") { g_opt.force_generic = value ? 1 : 0; return SNN_OK; }
    if (k == "query_block") {
        if (value == 0) value = 256;
        if (value < 32 || value > 256 || value % 32) return fail(SNN_ERR_INVALID_ARGUMENT, "query_block must be 32..256, multiple of 32");
        g_opt.query_block = (int)value;
        return SNN_OK;
    }
    if (k == "chunk") {
        if (value == 0) value = 2048;
        if (value < 64 || value > 8192 || value % 64) return fail(SNN_ERR_INVALID_ARGUMENT, "chunk must be 64..8192, multiple of 64");
        g_opt.chunk = (int)value;
        return SNN_OK;
    }
    if (k == "cap") {
        if (value == 0) value = 64;
        if (value < 1 || value > 1024) return fail(SNN_ERR_INVALID_ARGUMENT, "cap must be 1..1024");
        g_opt.cap = (int)value;
        return SNN_OK;
    }
    if (k == "tc") { g_opt.tc = value == 0 ? 1 : (value > 0 ? 1 : 0); if (value < 0) g_opt.tc = 0; return SNN_OK; }
    if (k == "tc_min_d") {
        if (value == 0) value = 32;
        if (value < 9 || value > 65536) return fail(SNN_ERR_INVALID_ARGUMENT, "tc_min_d must be 9..65536");
        g_opt.tc_min_d = (int)value;
        return SNN_OK;
    }
    if (k == "tc_tiles") {
        if (value == 0) value = 8;
        if (value < 1 || value > 64) return fail(SNN_ERR_INVALID_ARGUMENT, "tc_tiles must be 1..64");
        g_opt.tc_tiles = (int)value;
        return SNN_OK;
    }
    if (k == "tc_diag") {   // performance diagnostics only: results are NOT valid
        if (value < 0 || value > 4) return fail(SNN_ERR_INVALID_ARGUMENT, "tc_diag must be 0..4");
        g_opt.tc_diag = (int)value;
        return SNN_OK;
    }
    if (k == "tc_gram_min_d") {
        if (value == 0) value = 32;
        if (value < 1) return fail(SNN_ERR_INVALID_ARGUMENT, "tc_gram_min_d must be >= 1");
        g_opt.tc_gram_min_d = (int)value;
        return SNN_OK;
    }
    if (k == "symmetric") { g_opt.symmetric = value < 0 ? 0 : 1; return SNN_OK; }
    if (k == "stage_rows") { g_opt.stage_rows = value > 0 ? 1 : 0; return SNN_OK; }   // 0: default (direct)
    if (k == "balanced_compact") { g_opt.balanced_compact = value < 0 ? 0 : 1; return SNN_OK; }
    if (k == "window_all") { g_opt.window_all = value > 0 ? 1 : 0; return SNN_OK; }
    if (k == "simt_filter") { g_opt.simt_filter = value > 0 ? 1 : (value < 0 ? -1 : 0); return SNN_OK; }
    if (k == "lowd_tc") { g_opt.lowd_tc = value > 0 ? 1 : 0; return SNN_OK; }   // 0: default (off)
    if (k == "lowd_tc_tiles") {
        if (value == 0) value = 8;
        if (value < 1 || value > 64) return fail(SNN_ERR_INVALID_ARGUMENT, "lowd_tc_tiles must be 1..64");
        g_opt.lowd_tc_tiles = (int)value;
        return SNN_OK;
    }
    if (k == "lowd_tc_group") {
        if (value == 0) value = 8;
        if (value < 1 || value > 1 << 20) return fail(SNN_ERR_INVALID_ARGUMENT, "lowd_tc_group must be >= 1");
        g_opt.lowd_tc_group = (int)value;
        return SNN_OK;
    }
    if (k == "tc_ares") { g_opt.tc_ares = value < 0 ? 0 : 1; return SNN_OK; }
    if (k == "gram_rows") { g_opt.gram_rows = value == 0 ? 65536 : (value < 0 ? 0 : (int)value); return SNN_OK; }
    if (k == "gram_min_elems") { g_opt.gram_min_elems = value == 0 ? (int64_t(1) << 27) : value; return SNN_OK; }
    if (k == "finalize_order") { g_opt.finalize_order = value < 0 ? 0 : 1; return SNN_OK; }
    if (k == "finalize_pipe") { g_opt.finalize_pipe = value < 0 ? 0 : 1; return SNN_OK; }
    if (k == "lkey") { g_opt.lkey = value < 0 ? 0 : 1; return SNN_OK; }
    if (k == "count_warp") { g_opt.count_warp = value < 0 ? 0 : 1; return SNN_OK; }
    if (k == "union_snap") {   // 0: default; -1 off; 2: register-capped variant; 3, 4: diagnostics (labels invalid)
        if (value < -1 || value > 4) return fail(SNN_ERR_INVALID_ARGUMENT, "union_snap must be -1..4");
        g_opt.union_snap = value < 0 ? 0 : (value == 0 ? 1 : (int)value);
        return SNN_OK;
    }
    if (k == "union_phased") { g_opt.union_phased = value > 0 ? 1 : 0; return SNN_OK; }   // 0: default (off)
    if (k == "dbscan_block") {
        if (value == 0) value = 256;
        if (value < 32 || value > 256 || value % 32) return fail(SNN_ERR_INVALID_ARGUMENT, "dbscan_block must be 32..256, multiple of 32");
        g_opt.dbscan_block = (int)value;
        return SNN_OK;
    }
    if (k == "union_seed") {   // 0: default (8 steps); -1 off; else steps of 32 positions
        if (value > 1 << 20) return fail(SNN_ERR_INVALID_ARGUMENT, "union_seed must be <= 2^20");
        g_opt.union_seed = value < 0 ? 0 : (value == 0 ? 8 : (int)value);
        return SNN_OK;
    }
    if (k == "union_chunk") {
        if (value == 0) value = 512;
        if (value < 64 || value > 8192 || value % 64) return fail(SNN_ERR_INVALID_ARGUMENT, "union_chunk must be 64..8192, multiple of 64");
        g_opt.union_chunk = (int)value;
        return SNN_OK;
    }
    if (k == "union_behind") { g_opt.union_behind = value < 0 ? 0 : 1; return SNN_OK; }
    if (k == "union_stats") { g_opt.union_stats = value > 0 ? 1 : 0; return SNN_OK; }
    if (k == "union_load") {
        if (value < -1 || value > 2) return fail(SNN_ERR_INVALID_ARGUMENT, "union_load must be -1..2");
        g_opt.union_load = value == -1 ? 0 : (value == 0 ? 1 : (int)value);   // 0: the default (relaxed)
        return SNN_OK;
    }
    if (k == "tc_warp_arrive") { g_opt.tc_warp_arrive = value < 0 ? 0 : 1; return SNN_OK; }
    if (k == "tc_wait_hint") {
        if (value < 0 || value > 1000000) return fail(SNN_ERR_INVALID_ARGUMENT, "tc_wait_hint must be 0..1e6 ns");
        g_opt.tc_wait_hint = (int)value;
        return SNN_OK;
    }
    if (k == "tc_f16") { g_opt.tc_f16 = value < 0 ? 0 : 1; return SNN_OK; }
    if (k == "tc_group") {
        if (value == 0) value = 128;
        if (value < 1 || value > 1 << 20) return fail(SNN_ERR_INVALID_ARGUMENT, "tc_group must be >= 1");
        g_opt.tc_group = (int)value;
        return SNN_OK;
    }
    if (k == "scan2q") { g_opt.scan2q = value > 0 ? 1 : value < 0 ? -1 : 0; return SNN_OK; }
    if (k == "chunk2q") {
        if (value == 0) value = 640;
        if (value < 64 || value > 8192 || value % 64) return fail(SNN_ERR_INVALID_ARGUMENT, "chunk2q must be 64..8192, multiple of 64");
        g_opt.chunk2q = (int)value;
        return SNN_OK;
    }
    if (k == "variant") {
        if (value == 0) value = 1;
        if (value < 1 || value > 2) return fail(SNN_ERR_INVALID_ARGUMENT, "variant must be 1 or 2");
        g_opt.variant = (int)value;
        return SNN_OK;
    }
    if (k == "ovf_records") {
        if (value == 0) value = 1 << 20;
        if (value < 1 || value > (int64_t(1) << 30)) return fail(SNN_ERR_INVALID_ARGUMENT, "ovf_records must be 1..2^30");
        g_opt.ovf_rec_cap = (int32_t)value;
        return SNN_OK;
    }
    if (k == "power_iters") {
        if (value == 0) value = 1000;
        if (value < 1 || value > 1000000) return fail(SNN_ERR_INVALID_ARGUMENT, "power_iters must be >= 1");
        g_opt.power_iters = (int)value;
        return SNN_OK;
    }
    return fail(SNN_ERR_INVALID_ARGUMENT, "unknown option " + k);
}

static snn_status build_impl(const void *X, int64_t n, int32_t d, snn_dtype dt, void *stream, snn_index *out) {
    if (!out) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL output handle");
    *out = nullptr;
    if (n == 0) return fail(SNN_ERR_EMPTY, "empty dataset");
    if (!X || n < 0 || d < 1 || (dt != SNN_F32 && dt != SNN_F64))
        return fail(SNN_ERR_INVALID_ARGUMENT, "invalid argument to snn_build");
    if (n >= (int64_t(1) << 30)) return fail(SNN_ERR_UNSUPPORTED, "n >= 2^30 is not supported");
    int sms = 0;
    snn_status st = device_check(&sms);
    if (st != SNN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool f64 = dt == SNN_F64;
    const size_t es = f64 ? 8 : 4;

    snn_index idx = new snn_index_s();
    idx->n = n; idx->d = d; idx->d_in = d; idx->dt = dt; idx->sm_count = sms;
    idx->ld = row_stride(d);
    idx->n_pad = round_up(n, 4);
    Workspace ws(s);
    auto own = [&](auto **p, size_t count) -> cudaError_t {
        cudaError_t e = ws.alloc(p, count);
        if (e == cudaSuccess) { ws.release(*p); idx->owned.push_back(*p); }
        return e;
    };
#define CKI(expr, where)                                                   \
    do {                                                                   \
        cudaError_t _e = (expr);                                           \
        if (_e != cudaSuccess) { free_index(idx); return cuda_fail(_e, where); } \
    } while (0)
    uint8_t *xs_bytes = nullptr;
    CKI(own(&xs_bytes, (size_t)idx->n_pad * row_elems(d, idx->ld) * es), "alloc Xs");
    idx->Xs = xs_bytes;
    CKI(own(&idx->keys, (size_t)n), "alloc keys");
    CKI(own(&idx->perm, (size_t)n), "alloc perm");
    CKI(own(&idx->xbar, (size_t)idx->n_pad + 256), "alloc xbar");   // +256: tile-wide bulk copies
    CKI(own(&idx->mu_d, (size_t)d), "alloc");
    CKI(own(&idx->mu_f, (size_t)d), "alloc");
    CKI(own(&idx->v_d, (size_t)d), "alloc");
    CKI(own(&idx->v_f, (size_t)d), "alloc");
    CKI(own(&idx->stats, (size_t)ST_COUNT + 2), "alloc");

    const void *Xd = X;
    if (!is_device_ptr(X)) {   // host input: stage (end-to-end path)
        uint8_t *tmp = nullptr;
        CKI(ws.alloc(&tmp, (size_t)n * d * es), "alloc staging");
        CKI(cudaMemcpyAsync(tmp, X, (size_t)n * d * es, cudaMemcpyHostToDevice, s), "H2D X");
        Xd = tmp;
    }
    double *sums = nullptr, *G = nullptr;
    uint32_t *maxabs = nullptr;
    int *flag = nullptr;
    float *keys_raw = nullptr;
    uint8_t *sort_tmp = nullptr;
    CKI(ws.alloc(&sums, (size_t)d), "alloc");
    CKI(ws.alloc(&maxabs, (size_t)d), "alloc");
    CKI(ws.alloc(&flag, 1), "alloc");
    CKI(own(&G, (size_t)d * d), "alloc Gram");   // kept: snn_index_sigma
    idx->G = G;
    CKI(ws.alloc(&keys_raw, (size_t)n), "alloc");
    CKI(ws.alloc(&sort_tmp, radix_sort_temp_bytes(n)), "alloc sort");
    CKI(cudaMemsetAsync(sums, 0, d * 8, s), "memset");
    CKI(cudaMemsetAsync(maxabs, 0, d * 4, s), "memset");
    CKI(cudaMemsetAsync(flag, 0, 4, s), "memset");
    CKI(cudaMemsetAsync(G, 0, (size_t)d * d * 8, s), "memset");
    CKI(cudaMemsetAsync(idx->stats, 0, (ST_COUNT + 2) * 8, s), "memset");

    const int ptok = prof_begin(F_BUILD, s);
    launch_colstats(Xd, f64, n, d, sums, maxabs, flag, s);                        // K1
    launch_finalize_mean(sums, n, d, idx->mu_d, idx->mu_f, s);
    bool gram_done = false;
    double gstride = 1.0;
    if (d >= g_opt.tc_gram_min_d && !g_opt.force_generic) {                       // K2a (tcgen05)
        // v1 only steers pruning (any unit vector keeps the results exact), so a
        // large build takes the Gram matrix over every st-th row (~gram_rows rows): the
        // direction of a strided sample of the data; snn_index_sigma recomputes the full one
        int64_t st = 1;
        if (g_opt.gram_rows > 0 && n > 2 * (int64_t)g_opt.gram_rows && (double)n * d >= (double)g_opt.gram_min_elems)
            st = ceil_div(n, (int64_t)g_opt.gram_rows);
        const int64_t ns = ceil_div(n, st);
        uint8_t *gsc = nullptr;
        CKI(ws.alloc(&gsc, gram_tc_scratch_bytes(ns, d)), "alloc Gram scratch");
        gram_done = launch_gram_tc(Xd, f64, ns, d, st * d, maxabs, 0.0, idx->mu_f, G, gsc, sms, s);
        if (gram_done && st > 1) {
            launch_scale_f64(G, (int64_t)d * d, (double)n / (double)ns, s);   // unbiased for the full data
            gstride = (double)st;
        }
    }
    if (!gram_done) launch_gram(Xd, f64, n, d, idx->mu_f, G, s);                  // K2a (SIMT)
    launch_set_f64(idx->stats + ST_GSTRIDE, gstride, s);
    double *pscratch = nullptr;
    CKI(ws.alloc(&pscratch, power_scratch_doubles(d, sms)), "alloc");
    launch_power_iteration(G, d, g_opt.power_iters, 1e-7, maxabs, idx->mu_d, idx->mu_f,
                           idx->v_d, idx->v_f, idx->stats, pscratch, s);            // K2b
    launch_keys(Xd, f64, n, d, idx->mu_d, idx->mu_f, idx->v_d, idx->v_f, keys_raw, s);  // K3
    radix_sort_pairs(keys_raw, nullptr, idx->keys, reinterpret_cast<uint32_t *>(idx->perm), n,
                     sort_tmp, s);                                                 // K4
    // tensor-core indexes gather after the stats sync (the FP16 scale needs max|x_c|), fused
    // with the operand copy; all others here
    const bool tc_cand = idx->ld != 0 && g_opt.tc && !g_opt.force_generic && d >= g_opt.tc_min_d;
    if (!tc_cand)
        launch_gather(Xd, f64, n, d, idx->ld, idx->n_pad, reinterpret_cast<const uint32_t *>(idx->perm),
                      idx->mu_d, idx->Xs, idx->xbar, s);                           // K5
    CKI(cudaGetLastError(), "launch");
    double *hs = static_cast<double *>(t_pinned.p);
    {
        ReadbackBatch rb;
        rb.add(hs, idx->stats, ST_COUNT * 8);
        rb.add(hs + ST_COUNT, flag, 4);
        CKI(small_readback_batch(rb, s), "D2H stats");
    }
    CKI(cudaStreamSynchronize(s), "build");
    memcpy(idx->h_stats, hs, sizeof(idx->h_stats));
    int nonfinite = *reinterpret_cast<int *>(hs + ST_COUNT);
    if (nonfinite) {
        free_index(idx);
        return fail(SNN_ERR_NONFINITE, "X contains NaN or Inf");
    }
    if (idx->ld == 0 && !f64) {   // low-d fp32: expanded-form filter rows (scan variant 3)
        double c1h = 1.0, r2h = 0.0;
        simt_filter_consts(d, 1.0, &c1h, &r2h);
        CKI(own(&idx->Xf, (size_t)idx->n_pad * (d + 1)), "alloc filter rows");
        idx->xf_c1h = c1h;
        launch_filter_rows(static_cast<const float *>(idx->Xs), d, n, idx->n_pad, idx->mu_f, c1h, idx->Xf, s);
    }
    if (tc_cand) {   // K5 + K5': sorted copy and tensor-core operand copy
        idx->tc = 1;
        int e = 0;
        idx->tc_f16 = g_opt.tc_f16 && f16_exponent(idx->h_stats[ST_XCMAX], &e);
        idx->xexp = e;
        idx->kpad = tc_kpad(d, idx->tc_f16);
        if (idx->tc_f16) {   // one pass over X writes both copies and the half norms
            uint16_t *xt = nullptr;
            CKI(own(&xt, (size_t)n * idx->kpad), "alloc FP16 copy");
            idx->Xt = xt;
            launch_gather_xs_f16(Xd, f64, n, idx->n_pad, d, idx->ld, reinterpret_cast<const uint32_t *>(idx->perm),
                                 idx->mu_f, ldexpf(1.0f, e), idx->Xs, idx->Xt, idx->xbar, s);
        } else {
            launch_gather(Xd, f64, n, d, idx->ld, idx->n_pad, reinterpret_cast<const uint32_t *>(idx->perm),
                          idx->mu_d, idx->Xs, idx->xbar, s);                       // K5
            float *xt = nullptr;
            CKI(own(&xt, (size_t)n * idx->kpad), "alloc TF32 copy");
            idx->Xt = xt;
            launch_gather_tf32(Xd, f64, n, d, reinterpret_cast<const uint32_t *>(idx->perm), idx->mu_f,
                               xt, idx->xbar, s);
        }
        CKI(cudaGetLastError(), "launch");
    }
    prof_end(ptok, s, (double)n);
    *out = idx;
    return SNN_OK;
#undef CKI
}

void snn_free(snn_index idx) { free_index(idx); }

snn_status snn_pool_reserve(uint64_t bytes, void *stream) {
    int sms = 0;
    snn_status st = device_check(&sms);   // also keeps freed memory in the pool (release threshold)
    if (st != SNN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    void *p = nullptr;
    CK(cudaMallocAsync(&p, (size_t)bytes, s), "pool reserve");
    CK(cudaFreeAsync(p, s), "pool reserve");
    CK(cudaStreamSynchronize(s), "pool reserve");
    return SNN_OK;
}

void snn_free_async(snn_index idx, void *stream) {
    if (!idx) return;
    for (void *p : idx->owned) cudaFreeAsync(p, static_cast<cudaStream_t>(stream));
    delete idx;
}

static void thresholds(double R2, int d, float *T_in, float *T_out) {
    const double u32 = ldexp(1.0, -24), u64 = ldexp(1.0, -53);
    const double g32 = (d + 2) * u32 / (1.0 - (d + 2) * u32);
    const double g64 = (d + 2) * u64 / (1.0 - (d + 2) * u64);
    const double eta = (2.0 * d + 2.0) * ldexp(1.0, -149);
    const double tin = R2 * (1.0 - g32) / (1.0 + g64) * (1.0 - 1e-12) - eta;
    const double tout = R2 * (1.0 + g32) / (1.0 - g64) * (1.0 + 1e-12) + eta;
    float fi = (float)tin;
    if ((double)fi > tin) fi = nextafterf(fi, -INFINITY);
    float fo = (float)tout;
    if ((double)fo < tout) fo = nextafterf(fo, INFINITY);
    *T_in = fi;
    *T_out = fo;
}

static snn_status make_empty_result(int64_t m, cudaStream_t s, snn_result *out) {
    snn_result r = new snn_result_s();
    r->m = m;
    void *p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, (size_t)(m + 1) * 8, s);
    if (e != cudaSuccess) { delete r; return cuda_fail(e, "alloc offsets"); }
    r->offsets = static_cast<int64_t *>(p);
    cudaMemsetAsync(r->offsets, 0, (size_t)(m + 1) * 8, s);
    cudaMallocAsync(&p, 16, s); r->indices = static_cast<int32_t *>(p);
    cudaMallocAsync(&p, 16, s); r->distances = static_cast<float *>(p);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { snn_result_free(r); return cuda_fail(e, "query"); }
    *out = r;
    return SNN_OK;
}

// Tensor-core query path (d >= tc_min_d): K7 windows (128-query blocks) -> K9 tcgen05
// candidate filter -> K10 exact fp64 recheck -> hits sorted (index position, then original
// query id) with two stable radix passes -> CSR.
// K11 for the pair-list paths: rechecked pairs (flag = hit, dist) -> CSR in original query
// order, rows by ascending sorted-index position (csr.cu); rows above the fused sort's
// capacity fall back to two stable global radix passes.
static snn_status pairs_to_csr(Workspace &ws, cudaStream_t s, int64_t m, int64_t P, const int32_t *pq,
                               const int32_t *pj, const uint32_t *flag, const float *dist, const int32_t *qperm,
                               const int32_t *perm, snn_result *out) {
    int32_t *row_count, *maxrow;
    uint8_t *scan_tmp;
    CK(ws.alloc(&row_count, (size_t)m), "alloc");
    CK(ws.alloc(&maxrow, 1), "alloc");
    CK(ws.alloc(&scan_tmp, scan_temp_bytes(m > 0 ? m : 1) + 4096), "alloc");
    CK(cudaMemsetAsync(row_count, 0, (size_t)m * 4, s), "memset");
    CK(cudaMemsetAsync(maxrow, 0, 4, s), "memset");
    snn_result r = new snn_result_s();
    r->m = m;
    auto bail = [&](cudaError_t e, const char *where) { snn_result_free(r); return cuda_fail(e, where); };
    void *p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, (size_t)(m + 1) * 8, s);
    if (e != cudaSuccess) return bail(e, "alloc offsets");
    r->offsets = static_cast<int64_t *>(p);
    launch_pairs_row_count(flag, pq, qperm, P, m, row_count, maxrow, s);
    exclusive_scan_i32_to_i64(row_count, r->offsets, m, scan_tmp, s);
    int64_t *hp = static_cast<int64_t *>(t_pinned.p);
    {
        ReadbackBatch rb;
        rb.add(hp, r->offsets + m, 8);
        rb.add(hp + 1, maxrow, 4);
        if ((e = small_readback_batch(rb, s)) != cudaSuccess) return bail(e, "D2H");
    }
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return bail(e, "recheck");
    const int64_t H = hp[0];
    const int32_t mr = *reinterpret_cast<int32_t *>(hp + 1);
    r->nnz = H;
    if ((e = cudaMallocAsync(&p, (size_t)(H > 0 ? H : 1) * 4, s)) != cudaSuccess) return bail(e, "alloc indices");
    r->indices = static_cast<int32_t *>(p);
    if ((e = cudaMallocAsync(&p, (size_t)(H > 0 ? H : 1) * 4, s)) != cudaSuccess) return bail(e, "alloc distances");
    r->distances = static_cast<float *>(p);
    if (mr <= csr_row_sort_cap()) {
        int32_t *cursor;
        uint64_t *tmp;
        if ((e = ws.alloc(&cursor, (size_t)m)) != cudaSuccess) return bail(e, "alloc");
        if ((e = ws.alloc(&tmp, (size_t)(H > 0 ? H : 1))) != cudaSuccess) return bail(e, "alloc");
        cudaMemsetAsync(cursor, 0, (size_t)m * 4, s);
        launch_pairs_to_rows(flag, pq, pj, dist, qperm, P, m, r->offsets, cursor, tmp, perm, mr, r->indices,
                             r->distances, s);
    } else {   // a row larger than the fused sort's capacity: stable global radix passes
        uint32_t *hq, *hj, *order1, *k2, *order2, *sk;
        float *hd;
        int64_t *pos;
        uint8_t *scan2, *sort_tmp;
        int32_t *rc2;
        if ((e = ws.alloc(&pos, (size_t)P + 1)) != cudaSuccess) return bail(e, "alloc");
        if ((e = ws.alloc(&scan2, scan_temp_bytes(P > 0 ? P : 1))) != cudaSuccess) return bail(e, "alloc");
        if ((e = ws.alloc(&rc2, (size_t)m)) != cudaSuccess) return bail(e, "alloc");
        cudaMemsetAsync(rc2, 0, (size_t)m * 4, s);
        exclusive_scan_i32_to_i64(reinterpret_cast<const int32_t *>(flag), pos, P, scan2, s);
        if ((e = ws.alloc(&hq, (size_t)H)) != cudaSuccess || (e = ws.alloc(&hj, (size_t)H)) != cudaSuccess ||
            (e = ws.alloc(&hd, (size_t)H)) != cudaSuccess || (e = ws.alloc(&order1, (size_t)H)) != cudaSuccess ||
            (e = ws.alloc(&k2, (size_t)H)) != cudaSuccess || (e = ws.alloc(&order2, (size_t)H)) != cudaSuccess ||
            (e = ws.alloc(&sk, (size_t)H)) != cudaSuccess ||
            (e = ws.alloc(&sort_tmp, radix_sort_temp_bytes(H > 0 ? H : 1))) != cudaSuccess)
            return bail(e, "alloc");
        launch_tc_scatter(flag, pos, pq, pj, dist, qperm, P, hq, hj, hd, rc2, s);
        radix_sort_u32_pairs(hj, nullptr, sk, order1, H, sort_tmp, s);
        launch_gather_u32(hq, order1, H, k2, s);
        radix_sort_u32_pairs(k2, order1, sk, order2, H, sort_tmp, s);
        launch_tc_write(order2, hj, hd, perm, H, r->indices, r->distances, s);
    }
    *out = r;
    return SNN_OK;
}

// Returns SNN_ERR_UNSUPPORTED (no error message set) when the queries' magnitude does not
// fit the index's FP16 operand scaling; the caller then uses the generic exact path.
static snn_status query_tc(snn_index idx, Workspace &ws, cudaStream_t s, int sms, int64_t m, double R,
                           const void *Qs, const float *qkeys, const int32_t *qperm, const double *eq,
                           const void *Qd, const int *qflag, snn_result *out) {
    const bool f64 = idx->dt == SNN_F64;
    const bool f16 = idx->tc_f16 != 0;
    const int D = idx->d, TM = tc_tile_rows(), TN = tc_tile_cols();
    const int chunk = TN * g_opt.tc_tiles;
    const int64_t nblocks = ceil_div(m, TM);
    // grouped raster (tc.cu): G query blocks share each candidate chunk while it is in L2;
    // their operand tiles (G x 128 x kpad) are budgeted at 48 MB of the 126 MB L2
    const double a_bytes = (double)TM * idx->kpad * (f16 ? 2 : 4);
    int64_t G = (int64_t)(48e6 / a_bytes);
    if (G > g_opt.tc_group) G = g_opt.tc_group;
    if (G > nblocks) G = nblocks;
    if (G < 1) G = 1;
    const int64_t ngroups = ceil_div(nblocks, G);
    int64_t *grp_lo, *grp_items, *grp_start;
    int64_t *blk_lo, *blk_hi, *nitems, *item_start;
    unsigned long long *pcount, *wpairs;
    uint8_t *scan_tmp;
    CK(ws.alloc(&blk_lo, (size_t)nblocks), "alloc");
    CK(ws.alloc(&blk_hi, (size_t)nblocks), "alloc");
    CK(ws.alloc(&nitems, (size_t)nblocks), "alloc");
    CK(ws.alloc(&item_start, (size_t)nblocks + 1), "alloc");
    CK(ws.alloc(&pcount, 1), "alloc");
    CK(ws.alloc(&wpairs, 1), "alloc");
    CK(cudaMemsetAsync(pcount, 0, 8, s), "memset");
    CK(cudaMemsetAsync(wpairs, 0, 8, s), "memset");
    WindowSpec w;
    w.qkeys = qkeys; w.m = m; w.B = TM; w.keys = idx->keys; w.n = idx->n; w.n_pad = idx->n_pad;
    w.R = R;
    w.wnorm = idx->stats + (f64 ? ST_WNORM_D : ST_WNORM_F);
    w.ex = idx->stats + (f64 ? ST_EX_D : ST_EX_F);
    w.eq = eq;
    w.chunk = chunk;
    w.all = g_opt.window_all;
    w.blk_lo = blk_lo; w.blk_hi = blk_hi; w.nitems = nitems; w.pairs = wpairs;
    launch_block_windows(w, s);                                                    // K7
    CK(apply_part(ws, s, blk_lo, blk_hi, nitems, nblocks), "query part");
    CK(ws.alloc(&scan_tmp, scan_temp_bytes(m > nblocks ? m : nblocks) + 4096), "alloc");
    CK(ws.alloc(&grp_lo, (size_t)ngroups), "alloc");
    CK(ws.alloc(&grp_items, (size_t)ngroups), "alloc");
    CK(ws.alloc(&grp_start, (size_t)ngroups + 1), "alloc");
    launch_tc_group_items(blk_lo, blk_hi, nblocks, (int)G, chunk, grp_lo, grp_items, s);
    exclusive_scan_i64(grp_items, grp_start, ngroups, scan_tmp, s);
    int64_t *hp = static_cast<int64_t *>(t_pinned.p);
    {
        ReadbackBatch rb;
        rb.add(hp, grp_start + ngroups, 8);
        rb.add(hp + 1, qflag, 4);
        rb.add(hp + 2, wpairs, 8);
        if (Qd) rb.add(hp + 3, eq + 1, 8);
        CK(small_readback_batch(rb, s), "D2H windows");
    }
    CK(cudaStreamSynchronize(s), "query windows");
    const int64_t total_items = hp[0];
    if (*reinterpret_cast<int *>(hp + 1)) return fail(SNN_ERR_NONFINITE, "Q contains NaN or Inf");
    const double pairs_eval = (double)*reinterpret_cast<unsigned long long *>(hp + 2);
    // tensor-core operand A: the index copy itself (self-query) or the queries' copy
    const void *Qt = idx->Xt;
    const float *qbar = idx->xbar;
    int qexp = idx->xexp;
    if (Qd) {
        const double qbound = *reinterpret_cast<double *>(hp + 3);
        if (f16 && (!f16_exponent(qbound, &qexp) || qexp + idx->xexp < -120 || qexp + idx->xexp > 120))
            return SNN_ERR_UNSUPPORTED;
        float *qb = nullptr;
        CK(ws.alloc(&qb, (size_t)m), "alloc");
        if (f16) {
            uint16_t *qt = nullptr;
            CK(ws.alloc(&qt, (size_t)m * idx->kpad), "alloc");
            launch_gather_f16(Qd, f64, m, D, reinterpret_cast<const uint32_t *>(qperm), idx->mu_f,
                              ldexpf(1.0f, qexp), qt, qb, s);
            Qt = qt;
        } else {
            float *qt = nullptr;
            CK(ws.alloc(&qt, (size_t)m * idx->kpad), "alloc");
            launch_gather_tf32(Qd, f64, m, D, reinterpret_cast<const uint32_t *>(qperm), idx->mu_f, qt, qb, s);
            Qt = qt;
        }
        qbar = qb;
    }

    // separable margin (reading C20): operand rounding u (FP16 round-to-nearest
    // 2^-11, TF32 treated as truncated 2^-10) plus fp32 centring, accumulation bound
    // (d+2) 2^-22, fp32 evaluation slack; FP16 subnormals add an absolute error eta per
    // scaled coordinate (2^-25 / scale), bounded via ||x|| <= 1/2 + xbar.
    const double u = (f16 ? ldexp(1.0, -11) : ldexp(1.0, -10)) + ldexp(1.0, -24);
    const double gacc = (D + 2) * ldexp(1.0, -22);
    const double ga = 2 * u + u * u + gacc * (1 + u) * (1 + u);
    double c1 = (2 * ga + ldexp(1.0, -21) + 8 * ldexp(1.0, -24)) * 1.01;
    double c0 = 1e-30;
    if (f16) {
        const double ex = ldexp(1.0, -25 - idx->xexp), eqt = ldexp(1.0, -25 - qexp);
        const double em = ex > eqt ? ex : eqt;
        c1 += 2.0 * sqrt((double)D) * em * (1 + u) * 1.01;
        c0 += (2.0 * sqrt((double)D) * em * (1 + u) + 2.0 * D * ex * eqt) * 1.01;
    }
    TcArgs t{};
    t.xbar = idx->xbar; t.qbar = qbar; t.n = idx->n; t.m = m;
    t.kpad = idx->kpad; t.kblocks = idx->kpad / (f16 ? 64 : 32);
    t.blk_lo = blk_lo; t.blk_hi = blk_hi;
    t.grp_lo = grp_lo; t.grp_start = grp_start; t.ngroups = ngroups; t.group = (int)G;
    t.nblocks = nblocks; t.total_items = total_items; t.chunk = chunk;
    t.sc = f16 ? ldexpf(1.0f, idx->xexp + qexp) : 1.0f;
    t.diag = g_opt.tc_diag;
    t.ares = g_opt.tc_ares;
    t.wait_hint = (uint32_t)g_opt.tc_wait_hint;
    t.warp_arrive = g_opt.tc_warp_arrive;
    {
        const double c1h = 1.0 - c1 / 2;
        const double r2h = (R * R * (1.0 + 1e-12) * (1.0 + ldexp(1.0, -20)) + c0) / 2;
        float f1 = (float)c1h;
        if ((double)f1 > c1h) f1 = nextafterf(f1, -INFINITY);
        float f2 = (float)r2h;
        if ((double)f2 < r2h) f2 = nextafterf(f2, INFINITY);
        t.c1h = f1; t.r2h = f2;
    }
    int64_t cap = g_opt.ovf_rec_cap > 0 ? (int64_t)64 * m : 0;
    if (cap < (int64_t(1) << 22)) cap = int64_t(1) << 22;
    int32_t *pq = nullptr, *pj = nullptr;
    int64_t np = 0, used_cap = 0;
    for (int attempt = 0; attempt < 3; ++attempt) {
        CK(ws.alloc(&pq, (size_t)cap), "alloc pairs");
        CK(ws.alloc(&pj, (size_t)cap), "alloc pairs");
        used_cap = cap;
        t.pair_q = pq; t.pair_j = pj; t.pair_count = pcount; t.pair_cap = cap;
        CK(cudaMemsetAsync(pcount, 0, 8, s), "memset");
        const int ctok = prof_begin(F_COUNT, s);
        if (!launch_tc_window(Qt, idx->Xt, f16, t, sms, s)) return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");   // K9
        prof_end(ctok, s, pairs_eval);
        CK(small_readback(hp, pcount, 8, s), "D2H pair count");
        CK(cudaStreamSynchronize(s), "tc filter");
        np = (int64_t)*reinterpret_cast<unsigned long long *>(hp);
        if (np <= used_cap) break;
        // re-run with room for the count plus every warp's partially used block
        cap = np + (int64_t)sms * tc_claim_slack();
    }
    // the claim count is deterministic (items map statically to CTAs), so the first re-run
    // fits; never read past the buffers if it did not
    if (np > used_cap) return fail(SNN_ERR_OUT_OF_MEMORY, "tensor-core pair list still overflowed after re-runs");
    const int64_t P = np;
    const int wtok = prof_begin(F_WRITE, s);
    uint32_t *flag;
    float *dist;
    CK(ws.alloc(&flag, (size_t)P), "alloc");
    CK(ws.alloc(&dist, (size_t)P), "alloc");
    const int ld = idx->ld;
    launch_recheck(idx->Xs, Qs, f64, ld, D, pq, pj, P, R * R, flag, dist, s);            // K10
    snn_result r = nullptr;
    snn_status st = pairs_to_csr(ws, s, m, P, pq, pj, flag, dist, qperm, idx->perm, &r);   // K11
    if (st != SNN_OK) return st;
    const int64_t H = r->nnz;
    prof_end(wtok, s, (double)H);
    g_last_ovf = P - H;   // pair-list slots that are not hits (rejected candidates + unused slots)
    g_last_lost = 0;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { snn_result_free(r); return cuda_fail(e, "query"); }
    *out = r;
    return SNN_OK;
}

// Low-d tensor-core query path (fp32 data, d <= 8, AoSoA4 copies): K7 windows (128-query
// blocks, 64-aligned), grouped raster work list -> tcgen05 split-FP16 filter fused with
// the exact decision (tc_lowd.cu) -> per-row totals -> CSR compaction in key order.
// Returns SNN_ERR_UNSUPPORTED (no message) when the folded terms do not fit FP16 (huge R
// relative to the data) -- the FFMA path is used then.
static snn_status query_tcl(snn_index idx, Workspace &ws, cudaStream_t s, int sms, int64_t m, double R,
                            const void *Qs, const float *qkeys, const int32_t *qperm, const double *eq, bool self,
                            const int *qflag, snn_result *out) {
    const int D = idx->d;
    const int TM = 128, TN = 256, kc = tcl_kc(D);
    const int chunk = TN * (g_opt.lowd_tc_tiles < 8 ? g_opt.lowd_tc_tiles : 8);   // <= 64 chunks of 32 per item
    const int64_t nblocks = ceil_div(m, TM);
    int64_t G = g_opt.lowd_tc_group;
    if (G > nblocks) G = nblocks;
    if (G < 1) G = 1;
    int64_t *blk_lo, *blk_hi, *nitems, *bcount, *bstart;
    unsigned long long *wpairs;
    uint8_t *scan_tmp;
    CK(ws.alloc(&blk_lo, (size_t)nblocks), "alloc");
    CK(ws.alloc(&blk_hi, (size_t)nblocks), "alloc");
    CK(ws.alloc(&nitems, (size_t)nblocks), "alloc");
    CK(ws.alloc(&bcount, (size_t)nblocks), "alloc");
    CK(ws.alloc(&bstart, (size_t)nblocks + 1), "alloc");
    CK(ws.alloc(&wpairs, 1), "alloc");
    CK(ws.alloc(&scan_tmp, scan_temp_bytes((nblocks > m ? nblocks : m) + 1) + 4096), "alloc");
    CK(cudaMemsetAsync(wpairs, 0, 8, s), "memset");
    WindowSpec w;
    const int64_t n64 = round_up(idx->n, 64);   // 64-aligned windows
    w.qkeys = qkeys; w.m = m; w.B = TM; w.keys = idx->keys; w.n = idx->n; w.n_pad = n64;
    w.align = 64;
    w.R = R;
    w.wnorm = idx->stats + ST_WNORM_F;
    w.ex = idx->stats + ST_EX_F;
    w.eq = eq;
    w.chunk = chunk;
    w.all = g_opt.window_all;
    w.blk_lo = blk_lo; w.blk_hi = blk_hi; w.nitems = nitems; w.pairs = wpairs;
    launch_block_windows(w, s);                                                    // K7
    CK(apply_part(ws, s, blk_lo, blk_hi, nitems, nblocks), "query part");
    launch_tcl_items(blk_lo, blk_hi, nblocks, (int)G, chunk, bcount, s);
    exclusive_scan_i64(bcount, bstart, nblocks, scan_tmp, s);
    int64_t *hp = static_cast<int64_t *>(t_pinned.p);
    {
        ReadbackBatch rb;
        rb.add(hp, bstart + nblocks, 8);
        rb.add(hp + 1, qflag, 4);
        rb.add(hp + 2, wpairs, 8);
        if (!self) rb.add(hp + 3, eq + 1, 8);
        CK(small_readback_batch(rb, s), "D2H windows");
    }
    CK(cudaStreamSynchronize(s), "query windows");
    const int64_t total_items = hp[0];
    if (*reinterpret_cast<int *>(hp + 1)) return fail(SNN_ERR_NONFINITE, "Q contains NaN or Inf");
    const double pairs_eval = (double)*reinterpret_cast<unsigned long long *>(hp + 2);
    const double xb = idx->h_stats[ST_XCMAX];
    const double qb = self ? xb : *reinterpret_cast<double *>(hp + 3);
    const double bound = xb > qb ? xb : qb;
    int e = 0;
    if (bound > 0.0) {
        if (!std::isfinite(bound)) return SNN_ERR_UNSUPPORTED;
        e = 11 - ilogb(bound);   // |x * 2^e| < 2^12 for every centred coordinate
        if (e < -40 || e > 40) return SNN_ERR_UNSUPPORTED;
    }
    // Rigorous margin (reading C20, low-d form): E <= (c1/2)(xbar + qbar) + c0/2
    // bounds the error of the folded left side; see tc_lowd.cu for the operand layout.
    const double u24 = ldexp(1.0, -24), u22 = ldexp(1.0, -22) * 1.0001;
    const double us = u24 * 1.0001 + u22;                 // centring + two-half split
    const double eta = ldexp(1.0, -25 - e);               // FP16 subnormal, per coordinate
    const double eta2 = ldexp(1.0, -25 + 15 - 2 * e);     // FP16 subnormal of the folded scalars
    const double gacc = (3.0 * D + 4 + 2) * ldexp(1.0, -22);
    const double r2 = R * R * (1.0 + 1e-12) * (1.0 + ldexp(1.0, -20));
    const double sd = sqrt((double)D);
    const double c1 = 2.0 * 1.05 * (2 * us + us * us + u22 + 2 * u24 + u22 + 2.002 * gacc + eta * sd * (1 + us));
    const double c0 = 2.0 * 1.05 * (eta * sd * (1 + us) + D * eta * eta + 2 * eta2 + (u22 + gacc) * (r2 / 2 * 1.01 + 1e-300));
    const double c1h = 1.0 - c1 / 2;
    const double r2h = (r2 + c0) / 2;
    const double s2 = ldexp(1.0, 2 * e - 15);
    const double hmax = 0.5 * D * bound * bound * 1.001;
    if (hmax * s2 >= 60000.0 || (hmax + r2h) * s2 >= 60000.0) return SNN_ERR_UNSUPPORTED;

    // operands (query side first for self: one pass builds both)
    uint16_t *cand = nullptr, *qry = nullptr;
    CK(ws.alloc(&cand, (size_t)n64 * kc), "alloc");
    CK(ws.alloc(&qry, (size_t)m * kc), "alloc");
    const float *Xs = static_cast<const float *>(idx->Xs), *Qf = static_cast<const float *>(Qs);
    if (self) {
        launch_tcl_operands(Xs, D, idx->n, n64, idx->mu_f, e, c1h, r2h, cand, qry, s);
    } else {
        launch_tcl_operands(Xs, D, idx->n, n64, idx->mu_f, e, c1h, r2h, cand, nullptr, s);
        launch_tcl_operands(Qf, D, m, m, idx->mu_f, e, c1h, r2h, nullptr, qry, s);
    }
    // work list + record storage
    int4 *desc;
    int32_t *bitems, *pre, *row_count;
    uint32_t *ecnt;
    unsigned long long *eoff, *pool_count;
    uint16_t *pool;
    const int64_t nent = total_items * TM;
    const int64_t pool_cap = 48 * m + (int64_t(1) << 20);
    CK(ws.alloc(&desc, (size_t)(total_items > 0 ? total_items : 1)), "alloc");
    CK(ws.alloc(&bitems, (size_t)(total_items > 0 ? total_items : 1)), "alloc");
    CK(ws.alloc(&ecnt, (size_t)(nent > 0 ? nent : 1)), "alloc");
    CK(ws.alloc(&eoff, (size_t)(nent > 0 ? nent : 1)), "alloc");
    CK(ws.alloc(&pool, (size_t)pool_cap), "alloc");
    CK(ws.alloc(&pool_count, 1), "alloc");
    CK(cudaMemsetAsync(pool_count, 0, 8, s), "memset");
    CK(ws.alloc(&pre, (size_t)(nent > 0 ? nent : 1)), "alloc");
    CK(ws.alloc(&row_count, (size_t)m), "alloc");
    launch_tcl_fill_items(blk_lo, blk_hi, nblocks, (int)G, chunk, bstart, desc, bitems, s);
    TclArgs t{};
    t.n = idx->n; t.m = m; t.n_pad = idx->n_pad; t.m_pad = self ? idx->n_pad : round_up(m, 4);
    t.desc = desc; t.total_items = total_items;
    t.Xs = Xs; t.Qs = Qf;
    thresholds(R * R, D, &t.T_in, &t.T_out);
    t.R2 = R * R;
    t.ecnt = ecnt; t.eoff = eoff; t.pool = pool; t.pool_count = pool_count; t.pool_cap = pool_cap;
    const int ctok = prof_begin(F_COUNT, s);
    if (!launch_tcl_window(qry, cand, D, n64, t, sms, s)) return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    prof_end(ctok, s, pairs_eval);

    const int wtok = prof_begin(F_WRITE, s);
    TclPost pp{};
    pp.n = idx->n; pp.m = m; pp.Xs = Xs; pp.Qs = Qf; pp.perm = idx->perm; pp.qperm = qperm;
    pp.T_in = t.T_in; pp.T_out = t.T_out; pp.R2 = t.R2;
    launch_tcl_row_totals(pp, bstart, bitems, ecnt, pre, row_count, s);
    snn_result r = new snn_result_s();
    r->m = m;
    void *pm = nullptr;
    cudaError_t ce = cudaMallocAsync(&pm, (size_t)(m + 1) * 8, s);
    if (ce != cudaSuccess) { delete r; return cuda_fail(ce, "alloc offsets"); }
    r->offsets = static_cast<int64_t *>(pm);
    exclusive_scan_i32_to_i64(row_count, r->offsets, m, scan_tmp, s);
    if ((ce = small_readback(hp, r->offsets + m, 8, s)) != cudaSuccess ||
        (ce = cudaStreamSynchronize(s)) != cudaSuccess) { snn_result_free(r); return cuda_fail(ce, "exact"); }
    const int64_t H = hp[0];
    r->nnz = H;
    if ((ce = cudaMallocAsync(&pm, (size_t)(H > 0 ? H : 1) * 4, s)) != cudaSuccess) { snn_result_free(r); return cuda_fail(ce, "alloc"); }
    r->indices = static_cast<int32_t *>(pm);
    if ((ce = cudaMallocAsync(&pm, (size_t)(H > 0 ? H : 1) * 4, s)) != cudaSuccess) { snn_result_free(r); return cuda_fail(ce, "alloc"); }
    r->distances = static_cast<float *>(pm);
    int64_t *ovf = nullptr;
    unsigned long long *novf = nullptr;
    if ((ce = ws.alloc(&ovf, (size_t)(nent > 0 ? nent : 1))) != cudaSuccess ||
        (ce = ws.alloc(&novf, 1)) != cudaSuccess) { snn_result_free(r); return cuda_fail(ce, "alloc"); }
    cudaMemsetAsync(novf, 0, 8, s);
    launch_tcl_compact(pp, D, nent, desc, ecnt, eoff, pool, pre, r->offsets, r->indices, r->distances, ovf, novf, s);   // K11
    prof_end(wtok, s, (double)H);
    g_last_ovf = 0;
    g_last_lost = 0;
    ce = cudaGetLastError();
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) { snn_result_free(r); return cuda_fail(ce, "query"); }
    *out = r;
    return SNN_OK;
}

static snn_status query_impl(snn_index idx, const void *Q, int64_t m, int32_t d, snn_dtype dt,
                             double R, void *stream, snn_result *out, bool allow_sym = true) {
    if (!out) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL output handle");
    *out = nullptr;
    if (!idx) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL index");
    if (m < 0 || !(R >= 0.0) || !isfinite(R)) return fail(SNN_ERR_INVALID_ARGUMENT, "negative or non-finite radius / m < 0");
    const bool self = (Q == nullptr);
    if (!self && (d != idx->d || dt != idx->dt)) return fail(SNN_ERR_DIM_MISMATCH, "query dimension / dtype differs from the index");
    if (m >= (int64_t(1) << 31)) return fail(SNN_ERR_UNSUPPORTED, "m >= 2^31");
    int sms = 0;
    snn_status st = device_check(&sms);
    if (st != SNN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (m == 0) return make_empty_result(0, s, out);

    const bool f64 = idx->dt == SNN_F64;
    const size_t es = f64 ? 8 : 4;
    const int D = idx->d, ld = idx->ld;
    const int qtok = prof_begin(F_QUERY, s);
    Workspace ws(s);
    const void *Qs = idx->Xs;
    const float *qkeys = idx->keys;
    const int32_t *qperm = idx->perm;
    const double *eq = idx->stats + ST_EX_F;
    int *qflag = nullptr;
    unsigned long long *pairs = nullptr;
    const void *Qd = nullptr;   // raw device queries (tensor-core operand gather)
    CK(ws.alloc(&qflag, 2), "alloc");
    CK(ws.alloc(&pairs, 1), "alloc");
    CK(cudaMemsetAsync(qflag, 0, 8, s), "memset");
    CK(cudaMemsetAsync(pairs, 0, 8, s), "memset");
    if (!self) {
        const void *Qdev = Q;
        if (!is_device_ptr(Q)) {
            uint8_t *tmp = nullptr;
            CK(ws.alloc(&tmp, (size_t)m * D * es), "alloc staging");
            CK(cudaMemcpyAsync(tmp, Q, (size_t)m * D * es, cudaMemcpyHostToDevice, s), "H2D Q");
            Qdev = tmp;
        }
        double *qsums = nullptr, *eqd = nullptr;
        uint32_t *qmax = nullptr;
        float *qk_raw = nullptr, *qk = nullptr;
        int32_t *qp = nullptr;
        uint8_t *qs = nullptr, *sort_tmp = nullptr;
        CK(ws.alloc(&qsums, (size_t)D), "alloc");
        CK(ws.alloc(&qmax, (size_t)D), "alloc");
        CK(ws.alloc(&eqd, 2), "alloc");
        CK(ws.alloc(&qk_raw, (size_t)m), "alloc");
        CK(ws.alloc(&qk, (size_t)m), "alloc");
        CK(ws.alloc(&qp, (size_t)m), "alloc");
        CK(ws.alloc(&qs, (size_t)round_up(m, 4) * row_elems(D, ld) * es), "alloc");
        CK(ws.alloc(&sort_tmp, radix_sort_temp_bytes(m)), "alloc");
        CK(cudaMemsetAsync(qsums, 0, D * 8, s), "memset");
        CK(cudaMemsetAsync(qmax, 0, D * 4, s), "memset");
        // K6 query prep: finiteness + max |q| (E_q), keys (Alg. 2 l.2-3), sort, gather
        launch_colstats(Qdev, f64, m, D, qsums, qmax, qflag, s);
        launch_query_key_err(D, f64, qmax, idx->mu_d, idx->mu_f, idx->v_d, idx->v_f, eqd, s);
        launch_keys(Qdev, f64, m, D, idx->mu_d, idx->mu_f, idx->v_d, idx->v_f, qk_raw, s);
        radix_sort_pairs(qk_raw, nullptr, qk, reinterpret_cast<uint32_t *>(qp), m, sort_tmp, s);
        launch_gather(Qdev, f64, m, D, ld, round_up(m, 4), reinterpret_cast<const uint32_t *>(qp), idx->mu_d, qs, nullptr, s);
        Qs = qs; qkeys = qk; qperm = qp; eq = eqd;
        Qd = Qdev;
    }
    if (ld == 0 && !f64 && g_opt.lowd_tc && !g_opt.force_generic && tcl_supported(D)) {
        snn_status r = query_tcl(idx, ws, s, sms, m, R, Qs, qkeys, qperm, eq, self, qflag, out);
        if (r != SNN_ERR_UNSUPPORTED) {
            prof_end(qtok, s, (double)m);
            return r;
        }   // folded terms outside the FP16 range: FFMA path below
    }
    if (idx->tc) {
        snn_status r = query_tc(idx, ws, s, sms, m, R, Qs, qkeys, qperm, eq, Qd, qflag, out);
        if (r != SNN_ERR_UNSUPPORTED) {
            prof_end(qtok, s, (double)m);
            return r;
        }   // query magnitudes outside the FP16 operand range: generic exact path below
    }
    const bool generic = ld != 0;
    const int B = generic ? 64 : g_opt.query_block;
    // K8 with two queries per thread (fp32 radius queries with the expanded-form filter;
    // measured faster for every d = 2..8, scripts/sweep_2q_d.py -- DESIGN.md section 6): smaller work items
    const bool scan2q = !generic && !f64 && idx->Xf && g_opt.simt_filter >= 0 && B == 256 &&
                        (g_opt.scan2q > 0 || (g_opt.scan2q == 0 && D >= 2));
    const int chunk = generic ? 1024 : scan2q ? g_opt.chunk2q : g_opt.chunk;
    const int64_t nblocks = ceil_div(m, B);
    int64_t *blk_lo = nullptr, *blk_hi = nullptr, *nitems = nullptr, *item_start = nullptr;
    uint8_t *scan_tmp = nullptr;
    CK(ws.alloc(&blk_lo, (size_t)nblocks), "alloc");
    CK(ws.alloc(&blk_hi, (size_t)nblocks), "alloc");
    CK(ws.alloc(&nitems, (size_t)nblocks), "alloc");
    CK(ws.alloc(&item_start, (size_t)nblocks + 1), "alloc");
    CK(ws.alloc(&scan_tmp, scan_temp_bytes(m > nblocks ? m : nblocks)), "alloc");
    WindowSpec w;
    w.qkeys = qkeys; w.m = m; w.B = B; w.keys = idx->keys; w.n = idx->n; w.n_pad = idx->n_pad;
    w.R = R;
    w.wnorm = idx->stats + (f64 ? ST_WNORM_D : ST_WNORM_F);
    w.ex = idx->stats + (f64 ? ST_EX_D : ST_EX_F);
    w.eq = eq;
    w.chunk = chunk;
    w.all = g_opt.window_all;
    w.blk_lo = blk_lo; w.blk_hi = blk_hi; w.nitems = nitems; w.pairs = pairs;
    launch_block_windows(w, s);                                                    // K7
    // symmetric self-query: every unordered pair once -- block b scans only candidates
    // from its own first position on (j > i); mirrored hits fill the L part of row j
    const bool sym = self && !generic && allow_sym && g_opt.symmetric && !g_opt.window_all;
    int64_t *own_dev = nullptr;   // partitioned symmetric self-query: this part's row range
    if (sym && t_part.nparts > 1) {
        int64_t *tmp = nullptr;
        uint8_t *stp = nullptr;
        CK(ws.alloc(&tmp, (size_t)(2 * nblocks + 4)), "alloc");
        CK(ws.alloc(&stp, scan_temp_bytes(nblocks) + 4096), "alloc");
        CK(ws.alloc(&own_dev, 2), "alloc");
        launch_restrict_part_sym(blk_lo, blk_hi, nitems, nblocks, B, m, t_part.part, t_part.nparts, tmp, stp, own_dev, s);
    } else {
        CK(apply_part(ws, s, blk_lo, blk_hi, nitems, nblocks), "query part");
    }
    int64_t *blk_lo_s = blk_lo;
    if (sym) {
        CK(ws.alloc(&blk_lo_s, (size_t)nblocks), "alloc");
        CK(cudaMemsetAsync(pairs, 0, 8, s), "memset");   // evaluated pairs = the clipped windows
        launch_truncate_windows(blk_lo, blk_hi, nblocks, B, chunk, blk_lo_s, nitems, m, idx->n, pairs, s);
    }
    exclusive_scan_i64(nitems, item_start, nblocks, scan_tmp, s);
    int64_t *hp = static_cast<int64_t *>(t_pinned.p);
    {
        ReadbackBatch rb;
        rb.add(hp, item_start + nblocks, 8);
        rb.add(hp + 1, qflag, 4);
        rb.add(hp + 2, pairs, 8);
        if (own_dev) rb.add(hp + 3, own_dev, 16);
        CK(small_readback_batch(rb, s), "D2H windows");
    }
    CK(cudaStreamSynchronize(s), "query windows");
    const int64_t total_items = hp[0];
    const double pairs_eval = (double)*reinterpret_cast<unsigned long long *>(hp + 2);
    const int64_t own_lo = own_dev ? hp[3] : 0, own_hi = own_dev ? hp[4] : INT64_MAX;
    if (*reinterpret_cast<int *>(hp + 1)) return fail(SNN_ERR_NONFINITE, "Q contains NaN or Inf");

    int32_t *cnt = nullptr, *pre = nullptr, *row_count = nullptr, *ovf = nullptr;
    uint16_t *slots = nullptr;
    OvfRec *ovf_rec = nullptr;
    const int cap = g_opt.cap;
    const int32_t ovf_rec_cap = g_opt.ovf_rec_cap;
    CK(ws.alloc(&cnt, (size_t)total_items * B), "alloc counts");
    CK(ws.alloc(&row_count, (size_t)m), "alloc");
    if (!generic) {
        CK(ws.alloc(&pre, (size_t)total_items * B), "alloc prefixes");
        CK(ws.alloc(&slots, (size_t)total_items * B * cap), "alloc hit slots");
        CK(ws.alloc(&ovf, (size_t)total_items + 2), "alloc");
        CK(cudaMemsetAsync(ovf + total_items, 0, 8, s), "memset");
        CK(ws.alloc(&ovf_rec, (size_t)ovf_rec_cap), "alloc overflow records");
    } else {
        pre = cnt;   // the generic write pass only needs the prefixes
    }
    snn_result r = new snn_result_s();
    r->m = m;
    auto bail = [&](cudaError_t e, const char *where) { snn_result_free(r); return cuda_fail(e, where); };
#define CKR(expr, where)                          \
    do {                                          \
        cudaError_t _e = (expr);                  \
        if (_e != cudaSuccess) return bail(_e, where); \
    } while (0)
    {
        void *p = nullptr;
        cudaError_t e = cudaMallocAsync(&p, (size_t)(m + 1) * 8, s);
        if (e != cudaSuccess) return bail(e, "alloc offsets");
        r->offsets = static_cast<int64_t *>(p);
    }
    PassArgs a{};
    a.Xs = idx->Xs; a.Qs = Qs; a.ld = ld; a.d = D; a.f64 = f64; a.m = m;
    a.perm = idx->perm; a.qperm = qperm;
    a.blk_lo = blk_lo_s; a.blk_hi = blk_hi; a.item_start = item_start;
    if (total_items > 0 && total_items < (int64_t(1) << 31)) {
        int32_t *ib = nullptr;
        CKR(ws.alloc(&ib, (size_t)total_items), "alloc item blocks");
        launch_item_blocks(item_start, nblocks, ib, s);
        a.item_block = ib;
    }
    a.nblocks = nblocks; a.total_items = total_items;
    a.B = B; a.chunk = chunk;
    a.R2 = R * R;
    a.n_index = idx->n;
    a.own_lo = own_lo; a.own_hi = own_hi;
    int32_t *maxl = nullptr;
    const bool stage = !generic && g_opt.stage_rows;
    int32_t *srow = nullptr;
    int64_t *soff = nullptr;
    if (stage) {
        CKR(ws.alloc(&srow, (size_t)m), "alloc");
        CKR(ws.alloc(&soff, (size_t)m + 1), "alloc");
    }
    if (sym) {
        a.sym = 1;
        CKR(ws.alloc(&a.lcnt, (size_t)m), "alloc");
        CKR(ws.alloc(&a.lpos, (size_t)m), "alloc");
        CKR(ws.alloc(&maxl, 1), "alloc");
        CKR(cudaMemsetAsync(a.lcnt, 0, (size_t)m * 4, s), "memset");
        CKR(cudaMemsetAsync(maxl, 0, 4, s), "memset");
    }
    thresholds(a.R2, D, &a.T_in, &a.T_out);
    a.cnt = cnt; a.pre = pre; a.slots = slots; a.cap = cap;
    // balanced compaction: measured faster for symmetric self-queries (1.22 -> 1.09 ms on
    // config 2), slower for two-sided ones (0.92 -> 1.04 ms)
    if (!generic && sym && g_opt.balanced_compact && B == 256) {   // record counts per entry
        CKR(ws.alloc(&a.nrec, (size_t)total_items * B), "alloc record counts");
    }
    a.ovf_items = ovf; a.ovf_count = ovf ? ovf + total_items : nullptr; a.n_ovf = 0;
    a.ovf_rec = ovf_rec; a.ovf_rec_count = ovf ? ovf + total_items + 1 : nullptr;
    a.ovf_rec_cap = ovf_rec_cap; a.n_ovf_rec = 0;
    a.offsets = r->offsets; a.out_idx = nullptr; a.out_dist = nullptr;
    a.sm_count = sms;
    a.variant = g_opt.variant;
    a.scan2q = scan2q ? 1 : 0;
    a.fpipe = g_opt.finalize_pipe;
    if (!generic && !f64 && idx->Xf && g_opt.simt_filter >= 0) {
        double c1h = 1.0, r2h = 0.0;
        simt_filter_consts(D, R, &c1h, &r2h);
        a.Xf = idx->Xf; a.c1h = idx->xf_c1h; a.r2h = r2h; a.mu_f = idx->mu_f;
    }
    if (total_items == 0) {
        if (sym) launch_row_totals_sym(cnt, pre, item_start, m, B, qperm, a.lcnt, row_count, maxl, srow, own_lo, own_hi, s);
        else cudaMemsetAsync(row_count, 0, (size_t)m * 4, s);
        if (srow) cudaMemsetAsync(srow, 0, (size_t)m * 4, s);
    } else {
        const int ctok = prof_begin(F_COUNT, s);
        if (generic) launch_generic_pass(false, a, s);                           // K8 count
        else launch_lowd_scan(a, s);                                             // K8 scan
        prof_end(ctok, s, pairs_eval);
        if (sym) launch_row_totals_sym(cnt, pre, item_start, m, B, qperm, a.lcnt, row_count, maxl, srow, own_lo, own_hi, s);
        else launch_row_totals(cnt, pre, item_start, m, B, qperm, row_count, srow, s);  // K11
    }
    exclusive_scan_i32_to_i64(row_count, r->offsets, m, scan_tmp, s);
    if (stage) {
        exclusive_scan_i32_to_i64(srow, soff, m, scan_tmp, s);   // key-order row starts
        a.soff = soff;
    }
    {
        ReadbackBatch rb;
        rb.add(hp, r->offsets + m, 8);
        if (a.ovf_count) rb.add(hp + 1, a.ovf_count, 8);
        if (maxl) rb.add(hp + 2, maxl, 4);
        cudaError_t e = small_readback_batch(rb, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return bail(e, "query count");
    }
    r->nnz = hp[0];
    const int32_t max_l = sym ? *reinterpret_cast<int32_t *>(hp + 2) : 0;
    if (sym && max_l > 16384) {   // a huge mirrored row: redo unsymmetric
        snn_result_free(r);
        prof_end(qtok, s, 0.0);
        ws.free_all();   // the slots and counts of this attempt: do not hold them across the re-run
        return query_impl(idx, Q, m, d, dt, R, stream, out, false);
    }
    a.n_ovf = a.ovf_count ? reinterpret_cast<int32_t *>(hp + 1)[0] : 0;
    a.n_ovf_rec = a.ovf_count ? reinterpret_cast<int32_t *>(hp + 1)[1] : 0;
    {
        void *p = nullptr;
        cudaError_t e = cudaMallocAsync(&p, (size_t)(r->nnz > 0 ? r->nnz : 1) * 4, s);
        if (e != cudaSuccess) return bail(e, "alloc indices");
        r->indices = static_cast<int32_t *>(p);
        e = cudaMallocAsync(&p, (size_t)(r->nnz > 0 ? r->nnz : 1) * 4, s);
        if (e != cudaSuccess) return bail(e, "alloc distances");
        r->distances = static_cast<float *>(p);
    }
    a.out_idx = r->indices; a.out_dist = r->distances;
    if (stage) {   // the compaction and fix passes assemble rows in key order here
        CKR(ws.alloc(&a.stage, (size_t)(r->nnz > 0 ? r->nnz : 1)), "alloc staged rows");
        if (g_opt.finalize_order) {   // finalize walks the rows in original-id order
            int32_t *qinv = nullptr;
            CKR(ws.alloc(&qinv, (size_t)m), "alloc inverse permutation");
            launch_invert_perm(qperm, m, qinv, s);
            a.qinv = qinv;
        }
    }
    if (sym) {
        CKR(ws.alloc(&a.tmpL, (size_t)(r->nnz > 0 ? r->nnz : 1)), "alloc mirrored entries");
        if (!stage && g_opt.lkey) {   // L segments in key order (sum of lcnt <= nnz)
            int64_t *loff = nullptr;
            CKR(ws.alloc(&loff, (size_t)m + 1), "alloc mirrored-entry offsets");
            exclusive_scan_i32_to_i64(a.lcnt, loff, m, scan_tmp, s);
            a.loff = loff;
        }
        launch_sym_lpos_init(a, s);
    }
    if (r->nnz > 0) {
        const int wtok = prof_begin(F_WRITE, s);
        if (generic) {
            launch_generic_pass(true, a, s);                                     // K8 write
        } else {
            launch_lowd_compact(a, s);                                           // K11 compact
            launch_lowd_fix(a, s);                                               // overflow fix
            launch_rows_finalize(a, max_l, s);                                   // rows -> CSR
        }
        prof_end(wtok, s, generic ? pairs_eval : (double)r->nnz);
    }
    g_last_ovf = a.n_ovf_rec;
    g_last_lost = a.n_ovf;
    prof_end(qtok, s, (double)m);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return bail(e, "launch");
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return bail(e, "query");
    *out = r;
    return SNN_OK;
#undef CKR
}

snn_status snn_build(const void *X, int64_t n, int32_t d, snn_dtype dt, void *stream, snn_index *out) {
    return build_impl(X, n, d, dt, stream, out);
}

// Metric adapters: COSINE / ANGULAR run the exact Euclidean machinery
// on rows normalized by launch_normalize_rows, with the radius mapped by metric_radius.
static snn_status normalized_copy(const void *X, int64_t n, int32_t d, snn_dtype dt, cudaStream_t s,
                                  Workspace &ws, const void **Xn) {
    const size_t es = dt == SNN_F64 ? 8 : 4;
    const void *Xd = X;
    if (!is_device_ptr(X)) {
        uint8_t *tmp = nullptr;
        CK(ws.alloc(&tmp, (size_t)n * d * es), "alloc staging");
        CK(cudaMemcpyAsync(tmp, X, (size_t)n * d * es, cudaMemcpyHostToDevice, s), "H2D");
        Xd = tmp;
    }
    uint8_t *u = nullptr;
    int *flag = nullptr;
    CK(ws.alloc(&u, (size_t)n * d * es), "alloc normalized rows");
    CK(ws.alloc(&flag, 1), "alloc");
    CK(cudaMemsetAsync(flag, 0, 4, s), "memset");
    launch_normalize_rows(Xd, dt == SNN_F64, n, d, u, flag, s);
    int h = 0;
    CK(cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, s), "D2H flag");
    CK(cudaStreamSynchronize(s), "normalize");
    if (h) return fail(SNN_ERR_INVALID_ARGUMENT, "zero row: cosine / angular distance undefined");
    *Xn = u;
    return SNN_OK;
}

static bool metric_radius_ok(double r) { return r >= 0.0 && isfinite(r); }

// device copy of n x d rows (host input staged); owned by ws
static snn_status device_rows(const void *X, int64_t n, int32_t d, size_t es, cudaStream_t s, Workspace &ws,
                              const void **Xd) {
    if (is_device_ptr(X)) { *Xd = X; return SNN_OK; }
    uint8_t *tmp = nullptr;
    CK(ws.alloc(&tmp, (size_t)n * d * es), "alloc staging");
    CK(cudaMemcpyAsync(tmp, X, (size_t)n * d * es, cudaMemcpyHostToDevice, s), "H2D");
    *Xd = tmp;
    return SNN_OK;
}

// MANHATTAN: index of the input rows; MIPS: index of p~ = [sqrt(xi^2 - |p|^2), p]
// (PAPER.md:73-76).  Both keep the input rows (original order) for the exact post-filter.
static snn_status build_filtered(const void *X, int64_t n, int32_t d, snn_dtype dt, int32_t metric, void *stream,
                                 snn_index *out) {
    if (!out) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL output handle");
    *out = nullptr;
    if (n == 0) return fail(SNN_ERR_EMPTY, "empty dataset");
    if (!X || n < 0 || d < 1 || (dt != SNN_F32 && dt != SNN_F64))
        return fail(SNN_ERR_INVALID_ARGUMENT, "invalid argument to snn_build_metric");
    if (n >= (int64_t(1) << 30)) return fail(SNN_ERR_UNSUPPORTED, "n >= 2^30 is not supported");
    int sms = 0;
    snn_status st = device_check(&sms);
    if (st != SNN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t es = dt == SNN_F64 ? 8 : 4;
    Workspace ws(s);
    const void *Xd = nullptr;
    if ((st = device_rows(X, n, d, es, s, ws, &Xd)) != SNN_OK) return st;
    void *Xo = nullptr;
    CK(cudaMallocAsync(&Xo, (size_t)n * d * es, s), "alloc Xo");
    cudaError_t e = cudaMemcpyAsync(Xo, Xd, (size_t)n * d * es, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) { cudaFreeAsync(Xo, s); return cuda_fail(e, "copy Xo"); }
    double xi2 = 0.0;
    if (metric == SNN_METRIC_MIPS) {
        double *nrm2 = nullptr;
        unsigned long long *mx = nullptr;
        uint8_t *Xt = nullptr;
        if (ws.alloc(&nrm2, (size_t)n) != cudaSuccess || ws.alloc(&mx, 1) != cudaSuccess ||
            ws.alloc(&Xt, (size_t)n * (d + 1) * es) != cudaSuccess) {
            cudaFreeAsync(Xo, s);
            return fail(SNN_ERR_OUT_OF_MEMORY, "alloc MIPS rows");
        }
        cudaMemsetAsync(mx, 0, 8, s);
        launch_sq_norms(Xd, dt == SNN_F64, n, d, nrm2, mx, s);
        launch_mips_rows(Xd, dt == SNN_F64, n, d, nrm2, mx, Xt, s);
        unsigned long long h = 0;
        cudaMemcpyAsync(&h, mx, 8, cudaMemcpyDeviceToHost, s);
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) { cudaFreeAsync(Xo, s); return cuda_fail(e, "MIPS rows"); }
        memcpy(&xi2, &h, 8);
        st = build_impl(Xt, n, d + 1, dt, stream, out);
    } else {
        st = build_impl(Xd, n, d, dt, stream, out);
    }
    if (st != SNN_OK) { cudaFreeAsync(Xo, s); return st; }
    (*out)->metric = metric;
    (*out)->d_in = d;
    (*out)->Xo = Xo;
    (*out)->owned.push_back(Xo);
    (*out)->xi2 = xi2;
    return SNN_OK;
}

// MANHATTAN / MIPS query: Euclidean candidate superset, then the exact post-filter
static snn_status filtered_query(snn_index idx, const void *Q, int64_t m, double r, void *stream, snn_result *out) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool f64 = idx->dt == SNN_F64;
    const size_t es = f64 ? 8 : 4;
    const int d = idx->d_in;
    Workspace ws(s);
    snn_status st;
    const void *Qo = idx->Xo;   // self query: the index's own input rows
    if (Q && (st = device_rows(Q, m, d, es, s, ws, &Qo)) != SNN_OK) return st;
    snn_result cand = nullptr;
    double thr = r;
    if (idx->metric == SNN_METRIC_MANHATTAN) {   // ||.||_2 <= ||.||_1: the L2 ball of radius r covers the L1 ball
        st = Q ? query_impl(idx, Qo, m, d, idx->dt, r, stream, &cand) : query_impl(idx, nullptr, m, d, idx->dt, r, stream, &cand);
    } else {   // p^T q >= tau  =>  ||p~ - q~||^2 = |p~|^2 + |q|^2 - 2 p^T q <= xi^2 (1 + 2^-20) + |q|^2 - 2 tau
        double *nrm2 = nullptr;
        unsigned long long *mx = nullptr;
        uint8_t *Qt = nullptr;
        CK(ws.alloc(&nrm2, (size_t)m), "alloc");
        CK(ws.alloc(&mx, 1), "alloc");
        CK(ws.alloc(&Qt, (size_t)m * (d + 1) * es), "alloc");
        CK(cudaMemsetAsync(mx, 0, 8, s), "memset");
        launch_sq_norms(Qo, f64, m, d, nrm2, mx, s);
        launch_mips_rows(Qo, f64, m, d, nrm2, nullptr, Qt, s);
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, mx, 8, cudaMemcpyDeviceToHost, s), "D2H");
        CK(cudaStreamSynchronize(s), "MIPS queries");
        double q2;
        memcpy(&q2, &h, 8);
        // slack 4e-6 relative covers the rounded first coordinate (<= 2^-20 of xi^2) and the
        // fp64 rounding of the search's squared distances
        const double R2 = (idx->xi2 + q2) * (1.0 + 4e-6) - 2.0 * r + 8e-6 * fabs(r);
        const double Re = R2 > 0.0 ? sqrt(R2) : 0.0;
        st = query_impl(idx, Qt, m, d + 1, idx->dt, Re, stream, &cand);
    }
    if (st != SNN_OK) return st;
    const int64_t nnz = cand->nnz;
    uint8_t *keep = nullptr;
    float *val = nullptr;
    int32_t *rowcnt = nullptr;
    void *temp = nullptr;
    snn_result r2 = new snn_result_s();
    r2->m = m;
    auto bail = [&](cudaError_t e, const char *w) { snn_result_free(cand); snn_result_free(r2); return cuda_fail(e, w); };
    cudaError_t e;
    if ((e = ws.alloc(&keep, (size_t)nnz)) != cudaSuccess) return bail(e, "alloc");
    if ((e = ws.alloc(&val, (size_t)nnz)) != cudaSuccess) return bail(e, "alloc");
    if ((e = ws.alloc(&rowcnt, (size_t)m + 1)) != cudaSuccess) return bail(e, "alloc");
    if ((e = ws.alloc((uint8_t **)&temp, scan_temp_bytes(m + 1))) != cudaSuccess) return bail(e, "alloc");
    void *p = nullptr;
    if ((e = cudaMallocAsync(&p, (size_t)(m + 1) * 8, s)) != cudaSuccess) return bail(e, "alloc offsets");
    r2->offsets = static_cast<int64_t *>(p);
    launch_csr_filter(idx->metric, f64, cand->offsets, m, cand->indices, idx->Xo, Qo, d, thr, keep, val, rowcnt, s);
    exclusive_scan_i32_to_i64(rowcnt, r2->offsets, m, temp, s);   // offsets[0..m], offsets[m] = total
    int64_t tot = 0;
    if ((e = cudaMemcpyAsync(&tot, r2->offsets + m, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return bail(e, "D2H");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return bail(e, "filter");
    r2->nnz = tot;
    if ((e = cudaMallocAsync(&p, (size_t)(tot > 0 ? tot : 1) * 4, s)) != cudaSuccess) return bail(e, "alloc");
    r2->indices = static_cast<int32_t *>(p);
    if ((e = cudaMallocAsync(&p, (size_t)(tot > 0 ? tot : 1) * 4, s)) != cudaSuccess) return bail(e, "alloc");
    r2->distances = static_cast<float *>(p);
    launch_csr_compact(cand->offsets, m, cand->indices, keep, val, r2->offsets, r2->indices, r2->distances, s);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return bail(e, "compact");
    snn_result_free(cand);
    *out = r2;
    return SNN_OK;
}

snn_status snn_build_metric(const void *X, int64_t n, int32_t d, snn_dtype dt, int32_t metric, void *stream,
                            snn_index *out) {
    if (metric < SNN_METRIC_EUCLIDEAN || metric > SNN_METRIC_MIPS) {
        if (out) *out = nullptr;
        return fail(SNN_ERR_INVALID_ARGUMENT, "unknown metric");
    }
    if (metric == SNN_METRIC_EUCLIDEAN) return build_impl(X, n, d, dt, stream, out);
    if (metric == SNN_METRIC_MANHATTAN || metric == SNN_METRIC_MIPS) return build_filtered(X, n, d, dt, metric, stream, out);
    if (!out) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL output handle");
    *out = nullptr;
    if (n == 0) return fail(SNN_ERR_EMPTY, "empty dataset");
    if (!X || n < 0 || d < 1 || (dt != SNN_F32 && dt != SNN_F64))
        return fail(SNN_ERR_INVALID_ARGUMENT, "invalid argument to snn_build_metric");
    if (n >= (int64_t(1) << 30)) return fail(SNN_ERR_UNSUPPORTED, "n >= 2^30 is not supported");
    int sms = 0;
    snn_status st = device_check(&sms);
    if (st != SNN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Workspace ws(s);
    const void *Xn = nullptr;
    if ((st = normalized_copy(X, n, d, dt, s, ws, &Xn)) != SNN_OK) return st;
    if ((st = build_impl(Xn, n, d, dt, stream, out)) != SNN_OK) return st;
    (*out)->metric = metric;
    (*out)->d_in = d;
    return SNN_OK;
}

static snn_status metric_query(snn_index idx, const void *Q, int64_t m, int32_t d, snn_dtype dt, double r,
                               void *stream, snn_result *out) {
    if (!out) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL output handle");
    *out = nullptr;
    const bool mips = idx->metric == SNN_METRIC_MIPS;
    if (m < 0 || !(mips ? isfinite(r) : metric_radius_ok(r)))
        return fail(SNN_ERR_INVALID_ARGUMENT, "negative or non-finite radius / m < 0");
    if (Q && m > 0 && (d != idx->d_in || dt != idx->dt))
        return fail(SNN_ERR_DIM_MISMATCH, "query dimension / dtype differs from the index");
    if (idx->metric == SNN_METRIC_MANHATTAN || mips) {
        int sms = 0;
        snn_status st0 = device_check(&sms);
        if (st0 != SNN_OK) return st0;
        if (m == 0) return make_empty_result(0, static_cast<cudaStream_t>(stream), out);
        return filtered_query(idx, Q, m, r, stream, out);
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const double Re = metric_radius(idx->metric, r);
    snn_status st;
    Workspace ws(s);
    if (Q && m > 0) {
        if (d != idx->d || dt != idx->dt) return fail(SNN_ERR_DIM_MISMATCH, "query dimension / dtype differs from the index");
        const void *Qn = nullptr;
        int sms = 0;
        if ((st = device_check(&sms)) != SNN_OK) return st;
        if ((st = normalized_copy(Q, m, d, dt, s, ws, &Qn)) != SNN_OK) return st;
        st = query_impl(idx, Qn, m, d, dt, Re, stream, out);
    } else {
        st = query_impl(idx, Q, m, d, dt, Re, stream, out);
    }
    if (st != SNN_OK) return st;
    launch_metric_distances(idx->metric, (*out)->distances, (*out)->nnz, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { snn_result_free(*out); *out = nullptr; return cuda_fail(e, "metric distances"); }
    return SNN_OK;
}

// ------------------------------------------------------------------ streaming append (f4)
// PAPER.md:33 ("online streaming"): mu and v1 stay frozen -- the window bound of eq:lower
// holds for any fixed unit vector and centring -- the new rows get keys
// under the frozen (mu, v1), and the key order is rebuilt by one stable sort of [old rows in
// key order ; new rows] (old rows first, so equal keys stay ordered by original id).  The
// key error bounds and the FP16 operand scale are recomputed for the grown data; every
// per-row array (Xs, xbar, filter rows, tensor-core copy, kept input rows) is regathered.
static void swap_owned(snn_index idx, void *old_p, void *new_p, cudaStream_t s) {
    for (auto &p : idx->owned)
        if (p == old_p) { p = new_p; if (old_p) cudaFreeAsync(old_p, s); return; }
    idx->owned.push_back(new_p);
}

snn_status snn_append(snn_index idx, const void *Y, int64_t k, int32_t d, snn_dtype dt, void *stream) {
    if (!idx) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL index");
    if (k < 0 || (k > 0 && !Y)) return fail(SNN_ERR_INVALID_ARGUMENT, "k < 0 or NULL rows");
    if (idx->metric == SNN_METRIC_MIPS) return fail(SNN_ERR_UNSUPPORTED, "append to a MIPS index (xi would change)");
    if (d != idx->d_in || dt != idx->dt) return fail(SNN_ERR_DIM_MISMATCH, "row dimension / dtype differs from the index");
    if (k == 0) return SNN_OK;
    const int64_t n0 = idx->n, n1 = n0 + k;
    if (n1 >= (int64_t(1) << 30)) return fail(SNN_ERR_UNSUPPORTED, "n >= 2^30 is not supported");
    int sms = 0;
    snn_status st = device_check(&sms);
    if (st != SNN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool f64 = idx->dt == SNN_F64;
    const size_t es = f64 ? 8 : 4;
    const int D = idx->d, ld = idx->ld;
    const int64_t np1 = round_up(n1, 4);
    Workspace ws(s);
    const void *Yin = nullptr, *Yd = nullptr;
    if ((st = device_rows(Y, k, d, es, s, ws, &Yin)) != SNN_OK) return st;
    Yd = Yin;
    if (idx->metric == SNN_METRIC_COSINE || idx->metric == SNN_METRIC_ANGULAR)
        if ((st = normalized_copy(Yin, k, d, dt, s, ws, &Yd)) != SNN_OK) return st;
    uint8_t *S = nullptr, *sort_tmp = nullptr;
    double *sums = nullptr;
    uint32_t *maxabs = nullptr, *src = nullptr;
    int *flag = nullptr;
    float *keys_raw = nullptr;
    CK(ws.alloc(&S, (size_t)n1 * D * es), "alloc rows");
    CK(ws.alloc(&sums, (size_t)D), "alloc");
    CK(ws.alloc(&maxabs, (size_t)D), "alloc");
    CK(ws.alloc(&flag, 1), "alloc");
    CK(ws.alloc(&keys_raw, (size_t)n1), "alloc");
    CK(ws.alloc(&src, (size_t)n1), "alloc");
    CK(ws.alloc(&sort_tmp, radix_sort_temp_bytes(n1)), "alloc sort");
    CK(cudaMemsetAsync(sums, 0, (size_t)D * 8, s), "memset");
    CK(cudaMemsetAsync(maxabs, 0, (size_t)D * 4, s), "memset");
    CK(cudaMemsetAsync(flag, 0, 4, s), "memset");
    launch_unpack_rows(idx->Xs, f64, n0, D, ld, S, s);
    CK(cudaMemcpyAsync(S + (size_t)n0 * D * es, Yd, (size_t)k * D * es, cudaMemcpyDeviceToDevice, s), "copy rows");
    launch_colstats(S, f64, n1, D, sums, maxabs, flag, s);
    int hflag = 0;
    CK(cudaMemcpyAsync(&hflag, flag, 4, cudaMemcpyDeviceToHost, s), "D2H");
    CK(cudaStreamSynchronize(s), "append");
    if (hflag) return fail(SNN_ERR_NONFINITE, "appended rows contain NaN or Inf");   // index unchanged

    float *keys1 = nullptr, *xbar1 = nullptr, *Xf1 = nullptr;
    int32_t *perm1 = nullptr;
    void *Xs1 = nullptr, *Xt1 = nullptr, *Xo1 = nullptr;
    std::vector<void *> fresh;
    auto grab = [&](void **p, size_t bytes) {
        cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 16, s);
        if (e == cudaSuccess) fresh.push_back(*p);
        return e;
    };
    auto bail = [&](cudaError_t e, const char *w) {
        for (void *p : fresh) cudaFreeAsync(p, s);
        return cuda_fail(e, w);
    };
    cudaError_t e;
    if ((e = grab((void **)&keys1, (size_t)n1 * 4)) != cudaSuccess) return bail(e, "alloc keys");
    if ((e = grab((void **)&perm1, (size_t)n1 * 4)) != cudaSuccess) return bail(e, "alloc perm");
    if ((e = grab((void **)&xbar1, (size_t)(np1 + 256) * 4)) != cudaSuccess) return bail(e, "alloc xbar");
    if ((e = grab(&Xs1, (size_t)np1 * row_elems(D, ld) * es)) != cudaSuccess) return bail(e, "alloc Xs");
    launch_keys(S, f64, n1, D, idx->mu_d, idx->mu_f, idx->v_d, idx->v_f, keys_raw, s);          // K3
    radix_sort_pairs(keys_raw, nullptr, keys1, src, n1, sort_tmp, s);                            // K4
    launch_append_perm(src, n0, n1, idx->perm, perm1, s);
    launch_gather(S, f64, n1, D, ld, np1, src, idx->mu_d, Xs1, xbar1, s);                        // K5
    // grown-data key bounds into a fresh stats block: committed with the other arrays below,
    // so a failure leaves the index exactly as it was
    double *stats1 = nullptr;
    if ((e = grab((void **)&stats1, (size_t)(ST_COUNT + 2) * 8)) != cudaSuccess) return bail(e, "alloc stats");
    if ((e = cudaMemcpyAsync(stats1, idx->stats, (size_t)(ST_COUNT + 2) * 8, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return bail(e, "copy stats");
    launch_key_bounds(D, maxabs, idx->mu_d, idx->mu_f, idx->v_d, idx->v_f, stats1, s);
    double *hs = static_cast<double *>(t_pinned.p);
    double h_stats1[ST_COUNT];
    if ((e = small_readback(hs, stats1, ST_COUNT * 8, s)) != cudaSuccess) return bail(e, "D2H");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return bail(e, "append");
    memcpy(h_stats1, hs, sizeof(h_stats1));
    if (idx->Xf) {
        if ((e = grab((void **)&Xf1, (size_t)np1 * (D + 1) * 4)) != cudaSuccess) return bail(e, "alloc filter rows");
        launch_filter_rows(static_cast<const float *>(Xs1), D, n1, np1, idx->mu_f, idx->xf_c1h, Xf1, s);
    }
    int tc_f16 = idx->tc_f16, xexp = idx->xexp, kpad = idx->kpad;
    if (idx->tc) {
        int ex = 0;
        tc_f16 = idx->tc_f16 && f16_exponent(h_stats1[ST_XCMAX], &ex);
        xexp = ex;
        kpad = tc_kpad(D, tc_f16);
        if ((e = grab(&Xt1, (size_t)n1 * kpad * (tc_f16 ? 2 : 4))) != cudaSuccess) return bail(e, "alloc operand copy");
        if (tc_f16)
            launch_gather_f16(S, f64, n1, D, src, idx->mu_f, ldexpf(1.0f, ex), Xt1, xbar1, s);
        else
            launch_gather_tf32(S, f64, n1, D, src, idx->mu_f, static_cast<float *>(Xt1), xbar1, s);
    }
    if (idx->Xo) {   // MANHATTAN: input rows in original order
        if ((e = grab(&Xo1, (size_t)n1 * d * es)) != cudaSuccess) return bail(e, "alloc rows");
        cudaMemcpyAsync(Xo1, idx->Xo, (size_t)n0 * d * es, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(static_cast<uint8_t *>(Xo1) + (size_t)n0 * d * es, Yin, (size_t)k * d * es,
                        cudaMemcpyDeviceToDevice, s);
    }
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(s)) != cudaSuccess) return bail(e, "append");
    swap_owned(idx, idx->stats, stats1, s); idx->stats = stats1;
    memcpy(idx->h_stats, h_stats1, sizeof(idx->h_stats));
    swap_owned(idx, idx->keys, keys1, s); idx->keys = keys1;
    swap_owned(idx, idx->perm, perm1, s); idx->perm = perm1;
    swap_owned(idx, idx->xbar, xbar1, s); idx->xbar = xbar1;
    swap_owned(idx, idx->Xs, Xs1, s); idx->Xs = Xs1;
    if (Xf1) { swap_owned(idx, idx->Xf, Xf1, s); idx->Xf = Xf1; }
    if (Xt1) { swap_owned(idx, idx->Xt, Xt1, s); idx->Xt = Xt1; }
    if (Xo1) { swap_owned(idx, idx->Xo, Xo1, s); idx->Xo = Xo1; }
    idx->tc_f16 = tc_f16; idx->xexp = xexp; idx->kpad = kpad;
    idx->n = n1; idx->n_pad = np1;
    return SNN_OK;
}

// ------------------------------------------------------------------ save / load (f4)
// File: "SNNG", u32 version 1, 23 int64 header words, then the device arrays in a fixed
// order (all little endian, host byte order of x86-64 / aarch64).  Loading validates the
// header, the file length and the index invariants (keys sorted and finite, perm a
// permutation) before touching the device; the loaded index answers queries bit-identically.
namespace {
constexpr uint32_t kVersion = 1;
constexpr int kHdr = 15 + ST_COUNT;

struct Section { void **dev; size_t bytes; };

std::vector<Section> sections(snn_index idx, bool has_xf, bool has_xo) {
    const size_t es = idx->dt == SNN_F64 ? 8 : 4;
    const int64_t n = idx->n, np = idx->n_pad;
    const int D = idx->d;
    std::vector<Section> v = {
        {(void **)&idx->mu_d, (size_t)D * 8}, {(void **)&idx->mu_f, (size_t)D * 4},
        {(void **)&idx->v_d, (size_t)D * 8},  {(void **)&idx->v_f, (size_t)D * 4},
        {(void **)&idx->stats, (size_t)(ST_COUNT + 2) * 8},
        {(void **)&idx->G, (size_t)D * D * 8},
        {(void **)&idx->keys, (size_t)n * 4}, {(void **)&idx->perm, (size_t)n * 4},
        {(void **)&idx->xbar, (size_t)(np + 256) * 4},
        {(void **)&idx->Xs, (size_t)np * row_elems(D, idx->ld) * es}};
    if (has_xf) v.push_back({(void **)&idx->Xf, (size_t)np * (D + 1) * 4});
    if (idx->tc) v.push_back({(void **)&idx->Xt, (size_t)n * idx->kpad * (idx->tc_f16 ? 2 : 4)});
    if (has_xo) v.push_back({(void **)&idx->Xo, (size_t)n * idx->d_in * es});
    return v;
}

int64_t dbits(double x) { int64_t b; memcpy(&b, &x, 8); return b; }
double bitsd(int64_t b) { double x; memcpy(&x, &b, 8); return x; }
}  // namespace

snn_status snn_save(snn_index idx, const char *path, void *stream) {
    if (!idx || !path) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int64_t h[kHdr] = {idx->n, idx->n_pad, idx->d, idx->ld, (int64_t)idx->dt, idx->metric, idx->d_in, idx->tc,
                       idx->tc_f16, idx->xexp, idx->kpad, idx->Xf != nullptr, idx->Xo != nullptr,
                       dbits(idx->xi2), dbits(idx->xf_c1h)};
    for (int i = 0; i < ST_COUNT; ++i) h[15 + i] = dbits(idx->h_stats[i]);
    FILE *f = fopen(path, "wb");
    if (!f) return fail(SNN_ERR_INVALID_ARGUMENT, std::string("cannot open for writing: ") + path);
    bool ok = fwrite("SNNG", 1, 4, f) == 4 && fwrite(&kVersion, 4, 1, f) == 1 && fwrite(h, 8, kHdr, f) == (size_t)kHdr;
    std::vector<uint8_t> buf;
    for (const Section &sec : sections(idx, idx->Xf != nullptr, idx->Xo != nullptr)) {
        if (!ok) break;
        buf.resize(sec.bytes);
        cudaError_t e = cudaMemcpyAsync(buf.data(), *sec.dev, sec.bytes, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) { fclose(f); return cuda_fail(e, "save"); }
        ok = fwrite(buf.data(), 1, sec.bytes, f) == sec.bytes;
    }
    if (fclose(f) != 0) ok = false;
    return ok ? SNN_OK : fail(SNN_ERR_INVALID_ARGUMENT, std::string("write failed: ") + path);
}

snn_status snn_load(const char *path, void *stream, snn_index *out) {
    if (!path || !out) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL argument");
    *out = nullptr;
    FILE *f = fopen(path, "rb");
    if (!f) return fail(SNN_ERR_INVALID_ARGUMENT, std::string("cannot open: ") + path);
    std::vector<uint8_t> file;
    {
        uint8_t tmp[1 << 16];
        size_t r;
        while ((r = fread(tmp, 1, sizeof(tmp), f)) > 0) file.insert(file.end(), tmp, tmp + r);
        fclose(f);
    }
    const size_t head = 8 + 8 * (size_t)kHdr;
    if (file.size() < 8 || memcmp(file.data(), "SNNG", 4) != 0) return fail(SNN_ERR_INVALID_ARGUMENT, "bad magic");
    uint32_t ver;
    memcpy(&ver, file.data() + 4, 4);
    if (ver != kVersion) return fail(SNN_ERR_INVALID_ARGUMENT, "unsupported version");
    if (file.size() < head) return fail(SNN_ERR_INVALID_ARGUMENT, "truncated");
    int64_t h[kHdr];
    memcpy(h, file.data() + 8, 8 * (size_t)kHdr);
    snn_index_s tmpl;
    tmpl.n = h[0]; tmpl.n_pad = h[1]; tmpl.d = (int)h[2]; tmpl.ld = (int)h[3]; tmpl.dt = (snn_dtype)h[4];
    tmpl.metric = (int)h[5]; tmpl.d_in = (int)h[6]; tmpl.tc = (int)h[7]; tmpl.tc_f16 = (int)h[8];
    tmpl.xexp = (int)h[9]; tmpl.kpad = (int)h[10];
    const bool has_xf = h[11] != 0, has_xo = h[12] != 0;
    tmpl.xi2 = bitsd(h[13]); tmpl.xf_c1h = bitsd(h[14]);
    for (int i = 0; i < ST_COUNT; ++i) tmpl.h_stats[i] = bitsd(h[15 + i]);
    const int64_t n = tmpl.n;
    const int D = tmpl.d;
    const bool hdr_ok =
        n >= 1 && n < (int64_t(1) << 30) && tmpl.n_pad == round_up(n, 4) && D >= 1 && h[2] < (1 << 24) &&
        (h[4] == SNN_F32 || h[4] == SNN_F64) && h[5] >= SNN_METRIC_EUCLIDEAN && h[5] <= SNN_METRIC_MIPS &&
        tmpl.d_in == (tmpl.metric == SNN_METRIC_MIPS ? D - 1 : D) &&
        // the layouts build produces (the float4 / bulk loads rely on them)
        (tmpl.ld == 0 ? lowd_supported(D) : tmpl.ld == generic_stride(D)) &&
        (!tmpl.tc || (tmpl.ld != 0 && tmpl.kpad == tc_kpad(D, tmpl.tc_f16 != 0))) &&
        (!has_xf || (tmpl.ld == 0 && tmpl.dt == SNN_F32)) &&
        (has_xo == (tmpl.metric == SNN_METRIC_MANHATTAN || tmpl.metric == SNN_METRIC_MIPS));
    if (!hdr_ok) return fail(SNN_ERR_INVALID_ARGUMENT, "invalid header");
    std::vector<Section> secs = sections(&tmpl, has_xf, has_xo);
    size_t total = head;
    for (const Section &sec : secs) total += sec.bytes;
    if (file.size() < total) return fail(SNN_ERR_INVALID_ARGUMENT, "truncated");
    if (file.size() > total) return fail(SNN_ERR_INVALID_ARGUMENT, "trailing bytes");
    // invariants: keys (section 5) non-decreasing and finite, perm (section 6) a permutation
    {
        size_t off = head, off_keys = 0, off_perm = 0;
        for (const Section &sec : secs) {   // locate the keys and perm sections
            if (sec.dev == (void **)&tmpl.keys) off_keys = off;
            if (sec.dev == (void **)&tmpl.perm) off_perm = off;
            off += sec.bytes;
        }
        const float *keys = reinterpret_cast<const float *>(file.data() + off_keys);
        const int32_t *perm = reinterpret_cast<const int32_t *>(file.data() + off_perm);
        std::vector<uint8_t> seen((size_t)n, 0);
        for (int64_t i = 0; i < n; ++i) {
            float kf;
            int32_t p;
            memcpy(&kf, keys + i, 4);
            memcpy(&p, perm + i, 4);
            if (!std::isfinite(kf) || (i > 0 && !(keys[i - 1] <= kf)))
                return fail(SNN_ERR_INVALID_ARGUMENT, "invalid index: keys not sorted");
            if (p < 0 || p >= n || seen[p]) return fail(SNN_ERR_INVALID_ARGUMENT, "invalid index: perm is not a permutation");
            seen[p] = 1;
        }
    }
    int sms = 0;
    snn_status st = device_check(&sms);
    if (st != SNN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    snn_index idx = new snn_index_s();
    *idx = tmpl;
    idx->sm_count = sms;
    idx->owned.clear();
    std::vector<Section> dst = sections(idx, has_xf, has_xo);
    size_t off = head;
    for (const Section &sec : dst) {
        void *p = nullptr;
        cudaError_t e = cudaMallocAsync(&p, sec.bytes ? sec.bytes : 16, s);
        if (e != cudaSuccess) { free_index(idx); return cuda_fail(e, "alloc"); }
        idx->owned.push_back(p);
        *sec.dev = p;
        e = cudaMemcpyAsync(p, file.data() + off, sec.bytes, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) { free_index(idx); return cuda_fail(e, "H2D"); }
        off += sec.bytes;
    }
    // the padding rows [n, n_pad) are sentinels the query kernels rely on (never hits, never
    // compacted): rewrite them instead of trusting the file
    if (idx->dt == SNN_F64)
        SNN_LAUNCH(restore_sentinels<double>, 1, 128, 0, s, (double *)idx->Xs, idx->ld, D, n, idx->n_pad, idx->xbar, idx->Xf);
    else
        SNN_LAUNCH(restore_sentinels<float>, 1, 128, 0, s, (float *)idx->Xs, idx->ld, D, n, idx->n_pad, idx->xbar, idx->Xf);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);   // `file` is pageable: copies complete before return
    if (e != cudaSuccess) { free_index(idx); return cuda_fail(e, "load"); }
    *out = idx;
    return SNN_OK;
}

snn_status snn_query_radius(snn_index idx, const void *Q, int64_t m, int32_t d, snn_dtype dt,
                            double R, void *stream, snn_result *out) {
    if (idx && idx->metric != SNN_METRIC_EUCLIDEAN && Q) return metric_query(idx, Q, m, d, dt, R, stream, out);
    if (!Q && m > 0) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL query pointer");
    if (!Q) {   // m == 0 with NULL Q: still validate the header
        if (out) *out = nullptr;
        if (!idx || !out) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL argument");
        if (d != idx->d || dt != idx->dt) return fail(SNN_ERR_DIM_MISMATCH, "query dimension / dtype differs from the index");
        if (m < 0 || !(R >= 0.0) || !isfinite(R)) return fail(SNN_ERR_INVALID_ARGUMENT, "negative or non-finite radius / m < 0");
        int sms;
        snn_status st = device_check(&sms);
        if (st != SNN_OK) return st;
        return make_empty_result(0, static_cast<cudaStream_t>(stream), out);
    }
    return query_impl(idx, Q, m, d, dt, R, stream, out);
}

snn_status snn_query_self(snn_index idx, double R, void *stream, snn_result *out) {
    if (!idx) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL index");
    if (idx->metric != SNN_METRIC_EUCLIDEAN) return metric_query(idx, nullptr, idx->n, idx->d, idx->dt, R, stream, out);
    return query_impl(idx, nullptr, idx->n, idx->d, idx->dt, R, stream, out);
}

snn_status snn_query_radius_part(snn_index idx, const void *Q, int64_t m, int32_t d, snn_dtype dt, double R,
                                 int32_t part, int32_t nparts, void *stream, snn_result *out) {
    if (nparts < 1 || part < 0 || part >= nparts) {
        if (out) *out = nullptr;
        return fail(SNN_ERR_INVALID_ARGUMENT, "need 0 <= part < nparts");
    }
    PartGuard g(part, nparts);
    return snn_query_radius(idx, Q, m, d, dt, R, stream, out);
}

snn_status snn_query_self_part(snn_index idx, double R, int32_t part, int32_t nparts, void *stream,
                               snn_result *out) {
    if (nparts < 1 || part < 0 || part >= nparts) {
        if (out) *out = nullptr;
        return fail(SNN_ERR_INVALID_ARGUMENT, "need 0 <= part < nparts");
    }
    PartGuard g(part, nparts);
    return snn_query_self(idx, R, stream, out);
}

snn_status snn_result_csr(snn_result r, snn_csr *view) {
    if (!r || !view) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL argument");
    view->m = r->m; view->nnz = r->nnz;
    view->offsets = r->offsets; view->indices = r->indices; view->distances = r->distances;
    return SNN_OK;
}

snn_status snn_result_copy(snn_result r, int64_t *offsets, int32_t *indices,
                           float *distances, void *stream) {
    if (!r || !offsets) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaMemcpyAsync(offsets, r->offsets, (size_t)(r->m + 1) * 8, cudaMemcpyDefault, s), "copy offsets");
    if (indices && r->nnz) CK(cudaMemcpyAsync(indices, r->indices, (size_t)r->nnz * 4, cudaMemcpyDefault, s), "copy indices");
    if (distances && r->nnz) CK(cudaMemcpyAsync(distances, r->distances, (size_t)r->nnz * 4, cudaMemcpyDefault, s), "copy distances");
    CK(cudaStreamSynchronize(s), "D2H");
    return SNN_OK;
}

snn_status snn_result_copy_async(snn_result r, int64_t *offsets, int32_t *indices, float *distances, void *stream) {
    if (!r || !offsets) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaMemcpyAsync(offsets, r->offsets, (size_t)(r->m + 1) * 8, cudaMemcpyDefault, s), "copy offsets");
    if (indices && r->nnz) CK(cudaMemcpyAsync(indices, r->indices, (size_t)r->nnz * 4, cudaMemcpyDefault, s), "copy indices");
    if (distances && r->nnz) CK(cudaMemcpyAsync(distances, r->distances, (size_t)r->nnz * 4, cudaMemcpyDefault, s), "copy distances");
    // snn_result_free waits for this event, not for the copy stream: frees ordered on the
    // copy stream would also wait for later copies queued there, and allocations that reuse
    // the memory would then serialise the next step behind them
    if (!r->copy_done) CK(cudaEventCreateWithFlags(&r->copy_done, cudaEventDisableTiming), "event");
    CK(cudaEventRecord(r->copy_done, s), "event");
    return SNN_OK;
}

void snn_result_free_async(snn_result r, void *stream) {
    if (!r) return;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (r->copy_done) {   // an asynchronous copy may still read the buffers
        cudaStreamWaitEvent(s, r->copy_done, 0);
        cudaEventDestroy(r->copy_done);
    }
    if (r->offsets) cudaFreeAsync(r->offsets, s);
    if (r->indices) cudaFreeAsync(r->indices, s);
    if (r->distances) cudaFreeAsync(r->distances, s);
    delete r;
}

void snn_result_free(snn_result r) { snn_result_free_async(r, nullptr); }

snn_status snn_index_sigma(snn_index idx, int32_t k, double *sigma, void *stream) {
    if (!idx || !sigma) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL argument");
    if (k < 1 || k > 16 || k > idx->d) return fail(SNN_ERR_INVALID_ARGUMENT, "need 1 <= k <= min(d, 16)");
    int sms = 0;
    snn_status st = device_check(&sms);
    if (st != SNN_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Workspace ws(s);
    double *scratch = nullptr, *dsig = nullptr;
    CK(ws.alloc(&scratch, (size_t)(k + 2) * idx->d), "alloc");
    CK(ws.alloc(&dsig, (size_t)k), "alloc");
    const double *G = idx->G;
    if (idx->h_stats[ST_GSTRIDE] > 1.0) {   // the build's Gram is a row sample: the full one from the index rows
        const int d = idx->d;
        double *Gf = nullptr;
        uint8_t *gsc = nullptr;
        CK(ws.alloc(&Gf, (size_t)d * d), "alloc Gram");
        CK(ws.alloc(&gsc, gram_tc_scratch_bytes(idx->n, d)), "alloc Gram scratch");
        CK(cudaMemsetAsync(Gf, 0, (size_t)d * d * 8, s), "memset");
        if (!launch_gram_tc(idx->Xs, idx->dt == SNN_F64, idx->n, d, idx->ld, nullptr, idx->h_stats[ST_XCMAX], idx->mu_f,
                            Gf, gsc, sms, s))
            return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        G = Gf;
    }
    launch_spectrum(G, idx->d, k, scratch, dsig, s);
    CK(cudaGetLastError(), "spectrum");
    CK(cudaMemcpyAsync(sigma, dsig, (size_t)k * 8, cudaMemcpyDeviceToHost, s), "D2H");
    CK(cudaStreamSynchronize(s), "spectrum");
    return SNN_OK;
}

snn_status snn_index_info(snn_index idx, snn_index_info_t *info) {
    if (!idx || !info) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL argument");
    const bool f64 = idx->dt == SNN_F64;
    info->n = idx->n; info->d = idx->d; info->dtype = idx->dt; info->ld = idx->ld;
    info->power_iters = (int32_t)idx->h_stats[ST_ITERS];
    info->sigma1 = idx->h_stats[ST_SIGMA1];
    info->key_err = idx->h_stats[f64 ? ST_EX_D : ST_EX_F];
    info->v1_norm = idx->h_stats[f64 ? ST_WNORM_D : ST_WNORM_F];
    info->mu = idx->mu_d; info->v1 = idx->v_f; info->keys = idx->keys; info->perm = idx->perm;
    info->xbar = idx->xbar; info->xs = idx->Xs;
    info->tc_operand = idx->tc ? (idx->tc_f16 ? 1 : 2) : 0;
    info->tc_kpad = idx->kpad;
    info->tc_exp = idx->xexp;
    info->metric = idx->metric;
    return SNN_OK;
}

snn_status snn_dbscan(snn_index idx, double eps, int32_t min_pts, int32_t *labels,
                      int32_t *n_clusters, void *stream) {
    if (!idx || !labels || !n_clusters) return fail(SNN_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!(eps >= 0.0) || !isfinite(eps) || min_pts < 1) return fail(SNN_ERR_INVALID_ARGUMENT, "eps must be finite >= 0, min_pts >= 1");
    int sms = 0;
    snn_status st = device_check(&sms);
    if (st != SNN_OK) return st;
    if (idx->metric == SNN_METRIC_MANHATTAN || idx->metric == SNN_METRIC_MIPS)
        return fail(SNN_ERR_UNSUPPORTED, "snn_dbscan: Euclidean, cosine and angular indexes only");
    eps = metric_radius(idx->metric, eps);   // PAPER.md:57-72 (identity for EUCLIDEAN)
    const int tok = prof_begin(F_DBSCAN, static_cast<cudaStream_t>(stream));
    if (idx->ld == 0) {   // low d: fused passes over the windows, neighbour lists never built
        st = dbscan_impl(idx, eps, min_pts, labels, n_clusters, static_cast<cudaStream_t>(stream));
    } else {              // any d: DBSCAN over the exact self-query CSR
        snn_result r = nullptr;
        st = query_impl(idx, nullptr, idx->n, idx->d, idx->dt, eps, stream, &r);
        if (st == SNN_OK) {
            st = dbscan_from_csr(r->offsets, r->indices, idx->n, min_pts, labels, n_clusters,
                                 static_cast<cudaStream_t>(stream));
            snn_result_free(r);
        }
    }
    prof_end(tok, static_cast<cudaStream_t>(stream), (double)idx->n);
    return st;
}

}  // extern "C"
