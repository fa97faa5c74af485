// dbscan.cu -- K12: DBSCAN with SNN as the neighbourhood backend.
//
// Readings (C18): closed eps-balls including the point itself; core iff
// |N_eps(i)| >= min_pts; clusters = connected components of core points under
// eps-adjacency; a non-core point with >= 1 core neighbour takes the first cluster that
// reaches it in the ascending-id scan with FIFO expansion (scikit-learn's
// order), i.e. the smallest cluster number among its core neighbours; other
// points are noise (-1); clusters are numbered 0..K-1 by increasing smallest original core
// id.  All neighbourhood tests use the exact
// windowed classification of the radius query (bit-identical to the fp64 oracle).
//
// Pipeline on the sorted index (neighbour lists are never materialised):
//   windows (K7, R = eps) -> core counts (chunks in order per block, early exit once
//   every point of the block has min_pts neighbours) -> core flags
//   -> M_UNION pass (core i, core j > i: lock-free union-find) -> flatten
//   -> per-root smallest original id -> flag + scan over original ids = canonical ranks
//   -> core labels -> M_BORDER pass (non-core points) -> labels scattered to original order.
#include <math.h>

#include "common.cuh"
#include "index.h"
#include "query.h"
#include "internal.h"

namespace snn {
namespace {

__global__ void init_core(const int32_t *count, int64_t n, int32_t min_pts, uint8_t *core,
                          int32_t *parent, int32_t *minid, int32_t *best) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        core[i] = count[i] >= min_pts;
        parent[i] = core[i] ? (int32_t)i : -1;   // -1 marks non-core points
        minid[i] = 0x7fffffff;
        best[i] = 0x7fffffff;
    }
}

__device__ __forceinline__ int32_t find_root(const int32_t *p, int32_t x) {
    int32_t px = p[x];
    while (px != x) { x = px; px = p[x]; }
    return x;
}

// flatten + smallest original id per root
// (warp-aggregated: lanes whose points share a root -- neighbours in key order usually do
// -- combine their ids first, so a big cluster's root sees one atomic per warp, not per point)
__global__ void flatten(int32_t *parent, const uint8_t *core, const int32_t *perm, int64_t n,
                        int32_t *minid) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {   // warp-uniform trips
        const int64_t i = base + threadIdx.x;
        int32_t r = -1, v = 0x7fffffff;
        if (i < n && core[i]) {
            r = find_root(parent, (int32_t)i);
            parent[i] = r;
            v = perm[i];
        }
        const unsigned peers = __match_any_sync(0xffffffffu, r);
        v = __reduce_min_sync(peers, v);
        if (r >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicMin(&minid[r], v);
    }
}

// flag[minid of each root] = 1 (original-id space), for the canonical ranking
__global__ void flag_roots(const int32_t *parent, const uint8_t *core, const int32_t *minid,
                           int64_t n, int32_t *flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (core[i] && parent[i] == i) flag[minid[i]] = 1;
}

// labels of core points (sorted order)
__global__ void core_labels(const int32_t *parent, const uint8_t *core, const int32_t *minid,
                            const int64_t *rank, int64_t n, int32_t *lab) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        lab[i] = core[i] ? (int32_t)rank[minid[parent[i]]] : -1;
}

// border points: smallest cluster number among core neighbours; scatter to original order
__global__ void final_labels(const int32_t *lab, const uint8_t *core, const int32_t *best,
                             const int32_t *perm, int64_t n, int32_t *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t l = lab[i];
        if (!core[i]) l = (best[i] != 0x7fffffff) ? best[i] : -1;
        out[perm[i]] = l;
    }
}

// non-core flags (for the compacted border query)
__global__ void noncore_flags(const uint8_t *core, int64_t n, int32_t *flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = core[i] ? 0 : 1;
}

// compacted border queries: list of non-core sorted positions, their keys and AoSoA4 rows
template <typename T>
__global__ void gather_noncore(const uint8_t *core, const int64_t *pos, int64_t n, int d, const T *Xs,
                               const float *keys, int32_t *list, float *qkeys, T *Qb) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (core[i]) continue;
        const int64_t t = pos[i];
        list[t] = (int32_t)i;
        qkeys[t] = keys[i];
        for (int k = 0; k < d; ++k) Qb[(t >> 2) * 4 * d + 4 * k + (t & 3)] = Xs[(i >> 2) * 4 * d + 4 * k + (i & 3)];
    }
}

// --- any d: DBSCAN over the exact self-query CSR (original order, original ids) -------
__device__ __forceinline__ int32_t uf_find_c(volatile int32_t *p, int32_t x) {
    int32_t cur = p[x];
    if (cur != x) {
        int32_t next, prev = x;
        while (cur > (next = p[cur])) {
            p[prev] = next;
            prev = cur;
            cur = next;
        }
    }
    return cur;
}
__device__ __forceinline__ void uf_unite_c(int32_t *p, int32_t a, int32_t b) {
    SNN_DASSERT(a >= 0 && b >= 0 && p[a] >= 0 && p[b] >= 0);
    volatile int32_t *vp = p;
    int32_t ra = uf_find_c(vp, a), rb = uf_find_c(vp, b);
    while (ra != rb) {
        if (ra < rb) { const int32_t t = ra; ra = rb; rb = t; }
        const int32_t old = atomicCAS(&p[ra], ra, rb);
        if (old == ra) break;
        ra = uf_find_c(vp, old);
        rb = uf_find_c(vp, rb);
    }
}

__global__ void csr_counts(const int64_t *off, int64_t n, int32_t *count) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        count[i] = (int32_t)min((int64_t)0x7fffffff, off[i + 1] - off[i]);
}

// warp per row: union core i with every core neighbour j > i
__global__ void csr_union(const int64_t *off, const int32_t *idx, const uint8_t *core, int64_t n, int32_t *parent) {
    const int lane = threadIdx.x % 32;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; i < n;
         i += (int64_t)gridDim.x * blockDim.x / 32) {
        if (!core[i]) continue;
        for (int64_t k = off[i] + lane; k < off[i + 1]; k += 32) {
            const int32_t j = idx[k];
            if (j > i && core[j]) uf_unite_c(parent, (int32_t)i, j);
        }
    }
}

// warp per non-core row: smallest cluster number among core neighbours
__global__ void csr_border(const int64_t *off, const int32_t *idx, const uint8_t *core, const int32_t *lab,
                           int64_t n, int32_t *best) {
    const int lane = threadIdx.x % 32;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; i < n;
         i += (int64_t)gridDim.x * blockDim.x / 32) {
        if (core[i]) continue;
        int32_t b = 0x7fffffff;
        for (int64_t k = off[i] + lane; k < off[i + 1]; k += 32) {
            const int32_t j = idx[k];
            if (core[j]) b = min(b, lab[j]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) b = min(b, __shfl_xor_sync(0xffffffffu, b, o));
        if (lane == 0) best[i] = b;
    }
}

__global__ void iota32(int32_t *p, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int32_t)i;
}

int grid_n(int64_t n) {
    int64_t g = ceil_div(n, 256);
    return (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

}  // namespace

snn_status dbscan_impl(snn_index idx, double eps, int32_t min_pts, int32_t *labels,
                       int32_t *n_clusters, cudaStream_t s) {
    const int64_t n = idx->n;
    const bool f64 = idx->dt == SNN_F64;
    const int B = dbscan_block(), chunk = 2048;   // queries per block (option dbscan_block)
    const int64_t nblocks = ceil_div(n, B);
    Workspace ws(s);
#define CKD(expr, where)                                       \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return cuda_fail(_e, where);    \
    } while (0)
    int64_t *blk_lo, *blk_hi, *nitems, *item_start, *hbuf;
    unsigned long long *pairs;
    uint8_t *scan_tmp;
    CKD(ws.alloc(&blk_lo, (size_t)nblocks), "alloc");
    CKD(ws.alloc(&blk_hi, (size_t)nblocks), "alloc");
    CKD(ws.alloc(&nitems, (size_t)nblocks), "alloc");
    CKD(ws.alloc(&item_start, (size_t)nblocks + 1), "alloc");
    CKD(ws.alloc(&pairs, 1), "alloc");
    CKD(ws.alloc(&scan_tmp, scan_temp_bytes(n > nblocks ? n : nblocks)), "alloc");
    CKD(cudaMallocHost(&hbuf, 32), "pinned");
    struct HostFree { void *p; ~HostFree() { cudaFreeHost(p); } } hf{hbuf};
    CKD(cudaMemsetAsync(pairs, 0, 8, s), "memset");
    WindowSpec w;
    w.qkeys = idx->keys; w.m = n; w.B = B; w.keys = idx->keys; w.n = n; w.n_pad = idx->n_pad;
    w.R = eps;
    w.wnorm = idx->stats + (f64 ? ST_WNORM_D : ST_WNORM_F);
    w.ex = idx->stats + (f64 ? ST_EX_D : ST_EX_F);
    w.eq = w.ex;
    w.chunk = chunk;
    w.blk_lo = blk_lo; w.blk_hi = blk_hi; w.nitems = nitems; w.pairs = pairs;
    launch_block_windows(w, s);
    exclusive_scan_i64(nitems, item_start, nblocks, scan_tmp, s);
    CKD(small_readback(hbuf, item_start + nblocks, 8, s), "D2H");
    CKD(cudaStreamSynchronize(s), "dbscan windows");
    const int64_t total_items = hbuf[0];

    int32_t *cnt, *count, *parent, *minid, *best, *flag, *lab, *out;
    int64_t *rank;
    uint8_t *core;
    CKD(ws.alloc(&cnt, (size_t)total_items * B), "alloc");
    CKD(ws.alloc(&count, (size_t)n), "alloc");
    CKD(ws.alloc(&core, (size_t)n), "alloc");
    CKD(ws.alloc(&parent, (size_t)idx->n_pad), "alloc");   // padding rows: -1 (group-wide parent loads)
    CKD(cudaMemsetAsync(parent + n, 0xff, (size_t)(idx->n_pad - n) * 4, s), "memset");
    CKD(ws.alloc(&minid, (size_t)n), "alloc");
    CKD(ws.alloc(&best, (size_t)n), "alloc");
    CKD(ws.alloc(&flag, (size_t)n), "alloc");
    CKD(ws.alloc(&rank, (size_t)n + 1), "alloc");
    CKD(ws.alloc(&lab, (size_t)n), "alloc");
    const bool dev_out = is_device_ptr(labels);
    if (dev_out) out = labels; else CKD(ws.alloc(&out, (size_t)n), "alloc");

    PassArgs a{};
    a.Xs = idx->Xs; a.Qs = idx->Xs; a.ld = 0; a.d = idx->d; a.f64 = f64; a.m = n;
    a.perm = idx->perm; a.qperm = idx->perm;
    a.blk_lo = blk_lo; a.blk_hi = blk_hi; a.item_start = item_start;
    a.nblocks = nblocks; a.total_items = total_items;
    if (total_items > 0 && total_items < (int64_t(1) << 31)) {   // item -> block table (locate)
        int32_t *ib = nullptr;
        CKD(ws.alloc(&ib, (size_t)total_items), "alloc");
        launch_item_blocks(item_start, nblocks, ib, s);
        a.item_block = ib;
    }
    a.B = B; a.chunk = chunk;
    a.R2 = eps * eps;
    {   // same rigorous fp32 thresholds as the radius query (api.cu)
        const int d = idx->d;
        const double u32 = ldexp(1.0, -24), u64 = ldexp(1.0, -53);
        const double g32 = (d + 2) * u32 / (1.0 - (d + 2) * u32);
        const double g64 = (d + 2) * u64 / (1.0 - (d + 2) * u64);
        const double eta = (2.0 * d + 2.0) * ldexp(1.0, -149);
        const double tin = a.R2 * (1.0 - g32) / (1.0 + g64) * (1.0 - 1e-12) - eta;
        const double tout = a.R2 * (1.0 + g32) / (1.0 - g64) * (1.0 + 1e-12) + eta;
        float fi = (float)tin, fo = (float)tout;
        if ((double)fi > tin) fi = nextafterf(fi, -INFINITY);
        if ((double)fo < tout) fo = nextafterf(fo, INFINITY);
        a.T_in = fi; a.T_out = fo;
    }
    a.cnt = cnt; a.pre = cnt; a.cap = 0; a.variant = 1;
    a.sm_count = idx->sm_count;
    a.core = core; a.parent = parent; a.best = best; a.min_pts = min_pts;
    a.count_warp = dbscan_count_warp();
    a.n_index = n;
    if (!f64 && idx->Xf && dbscan_simt_filter()) {   // expanded-form SIMT pre-filter (option)
        double c1h = 1.0, r2h = 0.0;
        simt_filter_consts(idx->d, eps, &c1h, &r2h);
        a.Xf = idx->Xf; a.c1h = idx->xf_c1h; a.r2h = r2h; a.mu_f = idx->mu_f;
    }

    unsigned long long *hp_pairs = reinterpret_cast<unsigned long long *>(hbuf);
    CKD(small_readback(hp_pairs, pairs, 8, s), "D2H");
    CKD(cudaStreamSynchronize(s), "dbscan pairs");
    const double pairs_eval = (double)*hp_pairs;
    const int ctok = prof_begin(F_COUNT, s);
    CKD(cudaMemsetAsync(pairs, 0, 8, s), "memset");
    launch_core_counts(a, count, pairs, s);                                 // counts (to min_pts)
    SNN_LAUNCH(init_core, grid_n(n), 256, 0, s, count, n, min_pts, core, parent, minid, best);
    {   // unions over the clipped windows (pairs j > i: block b starts at its first position;
        // or pairs j < i: block b's window ends after its last position)
        int64_t *lo2, *nit2, *st2;
        CKD(ws.alloc(&lo2, (size_t)nblocks), "alloc");
        CKD(ws.alloc(&nit2, (size_t)nblocks), "alloc");
        CKD(ws.alloc(&st2, (size_t)nblocks + 1), "alloc");
        unsigned long long *upairs;
        CKD(ws.alloc(&upairs, 1), "alloc");
        CKD(cudaMemsetAsync(upairs, 0, 8, s), "memset");
        // staged-snapshot union pass (fp32, d <= 8): candidates behind the block by default
        const bool snap = dbscan_union_snap() && !f64 && idx->d <= 8;
        const bool behind = snap && dbscan_union_behind();
        const int uchunk = snap ? dbscan_union_chunk() : chunk;   // candidates per union work item
        if (behind)   // lo2 holds the clipped window ends
            launch_truncate_windows_behind(blk_lo, blk_hi, nblocks, B, uchunk, lo2, nit2, n, n, upairs, s);
        else
            launch_truncate_windows(blk_lo, blk_hi, nblocks, B, uchunk, lo2, nit2, n, n, upairs, s);
        exclusive_scan_i64(nit2, st2, nblocks, scan_tmp, s);
        CKD(small_readback(hbuf, st2 + nblocks, 8, s), "D2H");
        CKD(small_readback(hbuf + 2, pairs, 8, s), "D2H");
        CKD(small_readback(hbuf + 3, upairs, 8, s), "D2H");
        unsigned long long *umax = nullptr;   // most chunks of one block (phased union order)
        CKD(ws.alloc(&umax, 1), "alloc");
        CKD(cudaMemsetAsync(umax, 0, 8, s), "memset");
        launch_max_i64(nit2, nblocks, umax, s);
        CKD(small_readback(hbuf + 1, umax, 8, s), "D2H");
        CKD(cudaStreamSynchronize(s), "dbscan union windows");
        prof_end(ctok, s, (double)*reinterpret_cast<unsigned long long *>(hbuf + 2));   // pairs evaluated
        PassArgs au = a;
        au.uload = dbscan_union_load();
        if (behind) au.blk_hi = lo2; else au.blk_lo = lo2;
        au.chunk = uchunk;
        au.item_start = st2; au.total_items = hbuf[0];
        au.item_block = nullptr;
        if (au.total_items > 0 && au.total_items < (int64_t(1) << 31)) {
            int32_t *ib2 = nullptr;
            CKD(ws.alloc(&ib2, (size_t)au.total_items), "alloc");
            launch_item_blocks(st2, nblocks, ib2, s);
            au.item_block = ib2;
        }
        const int utok = prof_begin(F_UNION, s);
        if (behind && dbscan_union_seed() > 0) launch_union_seed(a, dbscan_union_seed(), s);   // a: the full windows
        unsigned long long *ustats = nullptr;
        if (dbscan_union_stats()) {
            CKD(ws.alloc(&ustats, 3), "alloc");
            CKD(cudaMemsetAsync(ustats, 0, 24, s), "memset");
        }
        if (!(snap && launch_union_snap(au, dbscan_union_snap(), nit2, dbscan_union_phased() ? hbuf[1] : 0,
                                        behind ? 1 : 0, ustats, s)))      // unions
            launch_lowd_mode(3, au, s);
        prof_end(utok, s, (double)*reinterpret_cast<unsigned long long *>(hbuf + 3));
        if (ustats) {
            unsigned long long hs[3];
            CKD(cudaMemcpyAsync(hs, ustats, 24, cudaMemcpyDeviceToHost, s), "D2H");
            CKD(cudaStreamSynchronize(s), "union stats");
            dbscan_set_union_stats(hs);
        }
    }
    SNN_LAUNCH(flatten, grid_n(n), 256, 0, s, parent, core, idx->perm, n, minid);
    CKD(cudaMemsetAsync(flag, 0, (size_t)n * 4, s), "memset");
    SNN_LAUNCH(flag_roots, grid_n(n), 256, 0, s, parent, core, minid, n, flag);
    exclusive_scan_i32_to_i64(flag, rank, n, scan_tmp, s);                  // canonical ranks
    SNN_LAUNCH(core_labels, grid_n(n), 256, 0, s, parent, core, minid, rank, n, lab);
    {   // border points: a radius query of the compacted non-core points only
        int64_t *npos;
        CKD(ws.alloc(&npos, (size_t)n + 1), "alloc");
        SNN_LAUNCH(noncore_flags, grid_n(n), 256, 0, s, core, n, flag);
        exclusive_scan_i32_to_i64(flag, npos, n, scan_tmp, s);
        CKD(small_readback(hbuf, npos + n, 8, s), "D2H");
        CKD(cudaStreamSynchronize(s), "dbscan non-core");
        const int64_t nb = hbuf[0];
        if (nb > 0) {
            const size_t es = f64 ? 8 : 4;
            int32_t *list;
            float *qk;
            uint8_t *qb;
            int64_t *lo3, *hi3, *nit3, *st3;
            const int64_t nb3 = ceil_div(nb, B);
            CKD(ws.alloc(&list, (size_t)nb), "alloc");
            CKD(ws.alloc(&qk, (size_t)nb), "alloc");
            CKD(ws.alloc(&qb, (size_t)round_up(nb, 4) * idx->d * es), "alloc");
            CKD(ws.alloc(&lo3, (size_t)nb3), "alloc");
            CKD(ws.alloc(&hi3, (size_t)nb3), "alloc");
            CKD(ws.alloc(&nit3, (size_t)nb3), "alloc");
            CKD(ws.alloc(&st3, (size_t)nb3 + 1), "alloc");
            if (f64) SNN_LAUNCH(gather_noncore<double>, grid_n(n), 256, 0, s, core, npos, n, idx->d,
                                (const double *)idx->Xs, idx->keys, list, qk, (double *)qb);
            else SNN_LAUNCH(gather_noncore<float>, grid_n(n), 256, 0, s, core, npos, n, idx->d,
                            (const float *)idx->Xs, idx->keys, list, qk, (float *)qb);
            WindowSpec w3 = w;
            w3.qkeys = qk; w3.m = nb;
            w3.blk_lo = lo3; w3.blk_hi = hi3; w3.nitems = nit3; w3.pairs = pairs;
            launch_block_windows(w3, s);
            exclusive_scan_i64(nit3, st3, nb3, scan_tmp, s);
            CKD(small_readback(hbuf, st3 + nb3, 8, s), "D2H");
            CKD(cudaStreamSynchronize(s), "dbscan border windows");
            PassArgs ab = a;
            ab.Qs = qb; ab.m = nb; ab.qperm = list;
            ab.blk_lo = lo3; ab.blk_hi = hi3; ab.item_start = st3;
            ab.nblocks = nb3; ab.total_items = hbuf[0];
            ab.item_block = nullptr;   // its own work list: binary-search locate
            ab.cnt = nullptr; ab.pre = nullptr;
            ab.blab = lab;
            launch_lowd_mode(4, ab, s);                                      // border points
        }
    }
    SNN_LAUNCH(final_labels, grid_n(n), 256, 0, s, lab, core, best, idx->perm, n, out);
    if (!dev_out) CKD(cudaMemcpyAsync(labels, out, (size_t)n * 4, cudaMemcpyDeviceToHost, s), "D2H labels");
    CKD(small_readback(hbuf + 1, rank + n, 8, s), "D2H K");
    CKD(cudaGetLastError(), "launch");
    CKD(cudaStreamSynchronize(s), "dbscan");
    *n_clusters = (int32_t)hbuf[1];
    return SNN_OK;
#undef CKD
}

// DBSCAN for any d from the exact self-query CSR (rows and ids in original order): same
// semantics and canonical numbering as the low-d pipeline (reading C18).
snn_status dbscan_from_csr(const int64_t *off, const int32_t *nidx, int64_t n, int32_t min_pts, int32_t *labels,
                           int32_t *n_clusters, cudaStream_t s) {
    Workspace ws(s);
#define CKD(expr, where)                                       \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return cuda_fail(_e, where);    \
    } while (0)
    int32_t *count, *parent, *minid, *best, *flag, *lab, *out, *iota;
    int64_t *rank, *hbuf;
    uint8_t *core, *scan_tmp;
    CKD(ws.alloc(&count, (size_t)n), "alloc");
    CKD(ws.alloc(&core, (size_t)n), "alloc");
    CKD(ws.alloc(&parent, (size_t)n), "alloc");
    CKD(ws.alloc(&minid, (size_t)n), "alloc");
    CKD(ws.alloc(&best, (size_t)n), "alloc");
    CKD(ws.alloc(&flag, (size_t)n), "alloc");
    CKD(ws.alloc(&rank, (size_t)n + 1), "alloc");
    CKD(ws.alloc(&lab, (size_t)n), "alloc");
    CKD(ws.alloc(&iota, (size_t)n), "alloc");
    CKD(ws.alloc(&scan_tmp, scan_temp_bytes(n)), "alloc");
    CKD(cudaMallocHost(&hbuf, 32), "pinned");
    struct HostFree { void *p; ~HostFree() { cudaFreeHost(p); } } hf{hbuf};
    const bool dev_out = is_device_ptr(labels);
    if (dev_out) out = labels; else CKD(ws.alloc(&out, (size_t)n), "alloc");
    const int g = grid_n(n), gw = grid_n(n * 32);
    SNN_LAUNCH(iota32, g, 256, 0, s, iota, n);
    SNN_LAUNCH(csr_counts, g, 256, 0, s, off, n, count);
    SNN_LAUNCH(init_core, g, 256, 0, s, count, n, min_pts, core, parent, minid, best);
    SNN_LAUNCH(csr_union, gw, 256, 0, s, off, nidx, core, n, parent);
    SNN_LAUNCH(flatten, g, 256, 0, s, parent, core, iota, n, minid);
    CKD(cudaMemsetAsync(flag, 0, (size_t)n * 4, s), "memset");
    SNN_LAUNCH(flag_roots, g, 256, 0, s, parent, core, minid, n, flag);
    exclusive_scan_i32_to_i64(flag, rank, n, scan_tmp, s);
    SNN_LAUNCH(core_labels, g, 256, 0, s, parent, core, minid, rank, n, lab);
    SNN_LAUNCH(csr_border, gw, 256, 0, s, off, nidx, core, lab, n, best);
    SNN_LAUNCH(final_labels, g, 256, 0, s, lab, core, best, iota, n, out);
    if (!dev_out) CKD(cudaMemcpyAsync(labels, out, (size_t)n * 4, cudaMemcpyDeviceToHost, s), "D2H labels");
    CKD(small_readback(hbuf, rank + n, 8, s), "D2H K");
    CKD(cudaGetLastError(), "launch");
    CKD(cudaStreamSynchronize(s), "dbscan");
    *n_clusters = (int32_t)hbuf[0];
    return SNN_OK;
#undef CKD
}

}  // namespace snn
