// query.cu -- query-side kernels of Algorithm 2 "SNN Query".
//
//  K7  block_windows : for each block of B consecutive key-sorted queries, the union of
//                      their candidate ranges J (Alg. 2 l.4; eq:lower PAPER.md:142-153;
//                      one range per batch as in PAPER.md:218-219), found by binary
//                      search on the sorted keys, padded by the rigorous key error bounds
//                      (reading C8) and split into fixed-size work items.
//  K8  window passes : for every (query block, candidate chunk) item, the exact radius
//                      test of Alg. 2 l.5-6 over X(J,:):
//                        - fp32 data: the direct form eq:ip1 in fp32 on
//                          the ORIGINAL coordinates (reading C7), classified against
//                          rigorous thresholds from the paper's own bound gamma_{d+2}
//                          (reading C4): sure-in / sure-out / ambiguous;
//                          ambiguous pairs are re-evaluated in fp64 with the oracle's exact
//                          operation sequence (no FMA), so membership is bit-identical;
//                        - fp64 data: the oracle's fp64 sequence directly.
//                      Low d (<= 8, AoSoA4 rows): ONE scan pass counts and records hits
//                      (chunk-local indices, up to `cap` per (item, query)); a compaction
//                      kernel writes the CSR (original id, (float)sqrt(fp64 s)); a fix pass
//                      recomputes only the rare overflowed (item, query) entries.
//                      Generic d: count pass + recomputing write pass.
//  Candidate rows of a chunk are contiguous ("memory efficient to access
//  X(J,:)") and are staged into shared memory by the TMA bulk-copy engine
//  (cp.async.bulk + mbarrier), double-buffered across the persistent item loop.
#include <math.h>

#include "common.cuh"
#include "query.h"
#include "internal.h"

namespace snn {
namespace {

// ---------------------------------------------------------------------------- K7
// one CSR entry: into the staging buffer (one 8-byte store) or the final arrays
__device__ __forceinline__ void put_entry(const PassArgs &a, int64_t pos, int32_t id, float dist) {
    SNN_DASSERT(pos >= 0 && pos < a.offsets[a.m]);
    if (a.stage) {
        a.stage[pos] = ((unsigned long long)__float_as_uint(dist) << 32) | (uint32_t)id;
    } else {
        a.out_idx[pos] = id;
        a.out_dist[pos] = dist;
    }
}

// where row sp is assembled: its key-order start (staged rows) or its final CSR row
__device__ __forceinline__ int64_t row_base(const PassArgs &a, int64_t sp) {
    return a.soff ? a.soff[sp] : a.offsets[a.qperm[sp]];
}

__device__ __forceinline__ int64_t lower_bound_f(const float *a, int64_t n, float x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int64_t upper_bound_f(const float *a, int64_t n, float x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void block_windows(WindowSpec w) {
    const int64_t nb = ceil_div(w.m, w.B);
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int64_t s0 = b * w.B;
    const int64_t s1 = min(w.m, s0 + w.B) - 1;
    // R' = ||w|| R (1 + 1e-9) + E_x + E_q, rounded up to fp32 (reading C8)
    const double rp = w.R * (*w.wnorm) * (1.0 + 1e-9) + (*w.ex) + (*w.eq) + 1e-30;
    const float rpf = __double2float_ru(rp);
    const float lo_key = __fsub_rd(w.qkeys[s0], rpf);
    const float hi_key = __fadd_ru(w.qkeys[s1], rpf);
    int64_t lo = lower_bound_f(w.keys, w.n, lo_key);
    int64_t hi = upper_bound_f(w.keys, w.n, hi_key);
    if (w.all) { lo = 0; hi = w.n; }   // ablation: no pruning
    const int64_t al = w.align > 4 ? w.align : 4;   // >= 4: 16-byte aligned bulk copies
    lo -= lo % al;
    hi = min(round_up(hi, al), w.n_pad);
    w.blk_lo[b] = lo;
    w.blk_hi[b] = hi;
    w.nitems[b] = hi > lo ? ceil_div(hi - lo, w.chunk) : 0;
    const int64_t valid_hi = min(hi, w.n);
    if (valid_hi > lo)
        atomicAdd(w.pairs, (unsigned long long)((valid_hi - lo) * (s1 - s0 + 1)));
}

// ---------------------------------------------------------------------------- common
__device__ __forceinline__ void locate(const PassArgs &a, int64_t item, int64_t &b, int64_t &c0,
                                       int64_t &c1) {
    if (a.item_block) {   // one load instead of a dependent binary search
        b = a.item_block[item];
    } else {
        int64_t lo = 0, hi = a.nblocks;   // largest b with item_start[b] <= item
        while (hi - lo > 1) {
            int64_t mid = (lo + hi) >> 1;
            if (a.item_start[mid] <= item) lo = mid; else hi = mid;
        }
        b = lo;
    }
    c0 = a.blk_lo[b] + (item - a.item_start[b]) * a.chunk;
    c1 = min(c0 + a.chunk, a.blk_hi[b]);
    SNN_DASSERT(b >= 0 && b < a.nblocks && c0 >= 0 && (c0 & 3) == 0 && c0 < c1);
}

// ---------------------------------------------------------------------------- K8 low d
// One thread per query (registers); candidates in the AoSoA4 layout are broadcast from
// shared memory 4 at a time: coordinate k of candidates 4g..4g+3 is one float4.  The
// fp32 direct form is evaluated with packed f32x2 instructions (two candidates per
// instruction; FADD2 takes the query coordinate as a scalar broadcast operand), then one
// min-test per 4 candidates sends the rare near/inside pairs to the classification path.
__device__ __forceinline__ uint64_t f2pack(float x, float y) {
    float2 v = make_float2(x, y);
    return *reinterpret_cast<uint64_t *>(&v);
}
__device__ __forceinline__ float2 f2unpack(uint64_t u) { return *reinterpret_cast<float2 *>(&u); }
__device__ __forceinline__ uint64_t f2add(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t f2mul(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Per-4-candidate hit mask -> output.  MODE 0 records (g << 4 | mask) in the entry's
// slot list, or, once `cap` slots are used, appends (entry, hits-before, record) to the
// global overflow list; MODE 1 (fix) writes the CSR entries directly.
// 16-byte shared-memory load from a 32-bit shared address (keeps the address arithmetic
// out of the hot loop)
__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

__device__ __forceinline__ float lane4(const float4 &v, int i) {   // i is unrolled (static)
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// Hit masks -> output.  MODE 0 records (g << 4 | mask) in the entry's slot list, or, once
// `cap` slots are used, appends (entry, hits-before, record) to the global overflow list;
// MODE 1 (fix) writes the CSR entries directly.
template <typename T, int D, int MODE, bool SYM = false>
struct Emitter {
    const PassArgs &a;
    uint16_t *slot;
    int64_t e, c0, pos;
    int64_t sp = 0;
    int32_t c = 0, rec = 0;
    bool lost = false;
    // symmetric self-query: keep candidates j > sp of group g, count their mirrored hits
    __device__ __forceinline__ uint32_t symf(int g, uint32_t mask) const {
        if (!SYM || !mask) return mask;
        const int64_t jb = c0 + 4 * g;
        if (jb + 3 <= sp) return 0;
        if (jb <= sp) mask &= ~((2u << (sp - jb)) - 1u);
        uint32_t mm = mask;
        while (mm) {
            const int i = __ffs(mm) - 1;
            mm &= mm - 1;
            if (jb + i < a.own_hi) atomicAdd(&a.lcnt[jb + i], 1);   // rows of later parts: theirs
        }
        return mask;
    }
    __device__ __forceinline__ void record(int g, uint32_t mask) {   // MODE 0
        mask = symf(g, mask);
        if (!mask) return;
        const uint32_t v = ((uint32_t)g << 4) | mask;
        if (rec < a.cap) {
            slot[(size_t)rec * a.B] = (uint16_t)v;
        } else {
            const int32_t k = atomicAdd(a.ovf_rec_count, 1);
            if (k < a.ovf_rec_cap) a.ovf_rec[k] = OvfRec{(int32_t)e, c, v};
            else lost = true;
        }
        ++rec;
        c += __popc(mask);
    }
    __device__ __forceinline__ void write(int64_t j, double s) {      // MODE 1
        if (SYM && j <= sp) return;
        const float dd = (float)sqrt(s);
        if (sp >= a.own_lo) put_entry(a, pos, a.perm[j], dd);   // ghost queries: mirrors only
        ++pos;
        ++c;
        if (SYM && j < a.own_hi) {   // mirrored entry into row j's L segment
            const unsigned long long k = atomicAdd(&a.lpos[j], 1ull);
            SNN_DASSERT(k < (unsigned long long)a.offsets[a.m]);
            a.tmpL[k] = ((unsigned long long)sp << 32) | __float_as_uint(dd);
        }
    }
};

// Classify the 4 fp32 d^2 of group g (candidates of xv): sure-in (<= T_in), ambiguous
// (<= T_out: decided by the oracle-order fp64 sequence), else out.
template <typename E, int D, int MODE>
__device__ __forceinline__ void classify4(E &em, int g, const float4 (&xv)[D], float d0, float d1,
                                          float d2, float d3, float T_in, float T_out, double R2,
                                          const float (&q)[D]) {
    const float dv[4] = {d0, d1, d2, d3};
    uint32_t m_in = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (dv[i] <= T_out) {
            bool hit = dv[i] <= T_in;
            double s = 0.0;
            if (MODE == 1 || !hit) {
                float x[D];
#pragma unroll
                for (int k = 0; k < D; ++k) x[k] = lane4(xv[k], i);
                s = sqdist_exact(x, q, D);
                if (!hit) hit = s <= R2;
            }
            if (hit) {
                if (MODE == 0) m_in |= 1u << i;
                else em.write(em.c0 + g * 4 + i, s);
            }
        }
    }
    if (MODE == 0 && m_in) em.record(g, m_in);
}

__device__ __forceinline__ uint32_t mask4(float d0, float d1, float d2, float d3, float T) {
    return (uint32_t)(d0 <= T) | ((uint32_t)(d1 <= T) << 1) | ((uint32_t)(d2 <= T) << 2) |
           ((uint32_t)(d3 <= T) << 3);
}

// near-boundary candidates of a group (bits of amb): the oracle-order fp64 sequence decides
template <int D>
__device__ __forceinline__ uint32_t resolve4(uint32_t amb, const float4 (&xv)[D], const float (&q)[D],
                                             double R2) {
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (amb & (1u << i)) {
            float x[D];
#pragma unroll
            for (int k = 0; k < D; ++k) x[k] = lane4(xv[k], i);
            if (sqdist_exact(x, q, D) <= R2) m |= 1u << i;
        }
    }
    return m;
}

// packed fp32 direct form for the 4 candidates of one group: (lo, hi) = d^2 of (0,1), (2,3)
template <int D>
__device__ __forceinline__ void group_d2(const float4 (&xv)[D], const uint64_t (&nq)[D],
                                         uint64_t &lo, uint64_t &hi) {
    uint64_t t = f2add(f2pack(xv[0].x, xv[0].y), nq[0]);
    lo = f2mul(t, t);
    t = f2add(f2pack(xv[0].z, xv[0].w), nq[0]);
    hi = f2mul(t, t);
#pragma unroll
    for (int k = 1; k < D; ++k) {
        t = f2add(f2pack(xv[k].x, xv[k].y), nq[k]);
        lo = f2fma(t, t, lo);
        t = f2add(f2pack(xv[k].z, xv[k].w), nq[k]);
        hi = f2fma(t, t, hi);
    }
}

// MODE 0 = scan (count + record hits); MODE 1 = fix (recompute entries flagged lost and
// write them straight into the CSR).
// Kernel modes of the windowed pass (same exact classification in every mode):
//   M_SCAN   count + record hits (radius query, CSR path)
//   M_FIX    recompute entries whose records were lost; write CSR directly
//   M_COUNT  DBSCAN: |N_eps(i)| (self included)
//   M_UNION  DBSCAN: union core i with every core neighbour j > i (sorted positions)
//   M_BORDER DBSCAN: for non-core i, the smallest cluster number among core neighbours
enum { M_SCAN = 0, M_FIX = 1, M_COUNT = 2, M_UNION = 3, M_BORDER = 4 };

__device__ __forceinline__ int32_t ld_relaxed_gpu(const int32_t *p) {
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// Lock-free union-find over sorted positions (parent[x] <= x: every link goes from the
// larger root to the smaller, so chains decrease and path halving is race-benign).
__device__ __forceinline__ int32_t uf_rep(volatile int32_t *p, int32_t x) {
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
// the same union, returning the root of the joined component as seen when it finished
__device__ __forceinline__ int32_t uf_unite_root(int32_t *p, int32_t a, int32_t b) {
    volatile int32_t *vp = p;
    int32_t ra = uf_rep(vp, a), rb = uf_rep(vp, b);
    while (ra != rb) {
        if (ra < rb) { const int32_t t = ra; ra = rb; rb = t; }
        const int32_t old = atomicCAS(&p[ra], ra, rb);
        if (old == ra) return rb;
        ra = uf_rep(vp, old);
        rb = uf_rep(vp, rb);
    }
    return ra;
}
__device__ __forceinline__ void uf_unite(int32_t *p, int32_t a, int32_t b) {
    SNN_DASSERT(a >= 0 && b >= 0 && p[a] >= 0 && p[b] >= 0);   // both core points
    volatile int32_t *vp = p;
    int32_t ra = uf_rep(vp, a), rb = uf_rep(vp, b);
    while (ra != rb) {
        if (ra < rb) { const int32_t t = ra; ra = rb; rb = t; }
        const int32_t old = atomicCAS(&p[ra], ra, rb);
        if (old == ra) break;
        ra = uf_rep(vp, old);
        rb = uf_rep(vp, rb);
    }
}

template <typename T, int D, int MODE, int G, bool SYM = false>
__global__ void __launch_bounds__(256) window_lowd(PassArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr bool CONV = MODE == M_SCAN && (G == 1 || G == 3) && sizeof(T) == 4;   // DBSCAN modes: measured slower
    // warp-cooperative drain of the deferred hits (CONV): per warp up to 128 records, their
    // results, and the 32 queries' coordinates
    __shared__ uint32_t s_drec[CONV && G == 3 ? 8 * 128 : 1];
    __shared__ uint8_t s_dres[CONV && G == 3 ? 8 * 128 : 1];
    __shared__ float s_dq[CONV && G == 3 ? 8 * 32 * D : 1];
    const int tid = threadIdx.x;
    const T *Xs = static_cast<const T *>(a.Xs);
    const T *Qs = static_cast<const T *>(a.Qs);
    // G == 3: only the expanded-form filter rows (AoSoA4, D+1 floats per row) are staged;
    // the exact classification of the few groups that pass reads the rows from global memory
    constexpr int FW = G == 3 ? D + 1 : 0;
    const size_t orig_bytes = G == 3 ? 0 : (size_t)a.chunk * D * sizeof(T);
    const size_t buf_bytes = orig_bytes + (size_t)a.chunk * FW * 4;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 2 * buf_bytes);
    const int64_t n_work = MODE == M_FIX ? a.n_ovf : a.total_items;
    auto item_of = [&](int64_t w) -> int64_t { return MODE == M_FIX ? (int64_t)a.ovf_items[w] : w; };
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t item, int sidx) {
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const uint32_t bytes = G == 3 ? 0u : (uint32_t)((c1 - c0) * D * sizeof(T));
        const uint32_t fbytes = (uint32_t)((c1 - c0) * FW * 4);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bar[sidx], bytes + fbytes);
        if (G != 3) bulk_g2s(smem + sidx * buf_bytes, Xs + c0 * D, bytes, &bar[sidx]);
        if (FW) bulk_g2s(smem + sidx * buf_bytes + orig_bytes, a.Xf + c0 * FW, fbytes, &bar[sidx]);
    };
    uint32_t phase[2] = {0u, 0u};
    int64_t w = blockIdx.x;
    if (tid == 0 && w < n_work) issue(item_of(w), 0);
    const float T_in = a.T_in, T_out = a.T_out;
    const double R2 = a.R2;
    for (int it = 0; w < n_work; w += gridDim.x, ++it) {
        const int sidx = it & 1;
        const int64_t item = item_of(w);
        const int64_t wn = w + gridDim.x;
        if (tid == 0 && wn < n_work) issue(item_of(wn), sidx ^ 1);
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const int64_t sp = b * a.B + tid;
        bool active = sp < a.m;
        const int64_t e = item * a.B + tid;
        T q[D];
        // slot records item-major, record-major, thread-minor: record r of entry (item, t)
        // at slots[(item * cap + r) * B + t] (coalesced across the CTA's threads)
        Emitter<T, D, MODE, SYM> em{a, a.slots + (size_t)item * a.B * a.cap + tid, e, c0, 0};
        em.sp = sp;
        if (MODE == M_FIX) {
            active = active && a.cnt[e] < 0;   // lost-entry flag (sign bit)
            if (active) em.pos = row_base(a, sp) + a.pre[e];
        }
        if (MODE == M_UNION) active = active && a.core[sp] && c1 - 1 > sp;   // pairs j > i only
        // M_BORDER over a compacted query list: qperm maps to the index position
        const int64_t bpos = (MODE == M_BORDER && a.qperm) ? (active ? (int64_t)a.qperm[sp] : 0) : sp;
        if (MODE == M_BORDER) active = active && !a.core[bpos];
        int32_t best = 0x7fffffff;   // M_BORDER: smallest cluster number of a core neighbour
        int32_t uroot = -1;          // M_UNION: cached union-find root of this query
        if (MODE == M_UNION && active) uroot = uf_rep(a.parent, (int32_t)sp);
#pragma unroll
        for (int k = 0; k < D; ++k) q[k] = active ? Qs[(sp >> 2) * 4 * D + k * 4 + (sp & 3)] : (T)0;
        // the deferred-hit scan loop (fp32, G == 1) runs warp-converged: lanes without a
        // query take a NaN query (every comparison false, no hits)
        if (CONV && !active) {
#pragma unroll
            for (int k = 0; k < D; ++k) q[k] = (T)NAN;
        }
        mbar_wait(&bar[sidx], phase[sidx]);
        phase[sidx] ^= 1u;
        if (CONV ? __any_sync(0xffffffffu, active) : active) {   // CONV: whole warps
            const int ngroups = (int)((c1 - c0) >> 2);
            if constexpr (sizeof(T) == 4) {
                const float4 *g4 = G == 3 ? reinterpret_cast<const float4 *>(Xs) + (c0 >> 2) * D
                                          : reinterpret_cast<const float4 *>(smem + sidx * buf_bytes);
                uint64_t nq[D];
#pragma unroll
                for (int k = 0; k < D; ++k) nq[k] = f2pack(-q[k], -q[k]);
                // expanded-form filter operands of this query: centred coordinates and the
                // rigorous threshold thr = r2h - qbar c1h (fp64, rounded up)
                uint64_t nqc[FW > 0 ? D : 1];
                float thr = 0.f;
                if constexpr (G == 3) {
                    double qb = 0.0;
#pragma unroll
                    for (int k = 0; k < D; ++k) {
                        const float qc = (float)((double)q[k] - (double)a.mu_f[k]);
                        qb += (double)qc * (double)qc;
                        nqc[k] = f2pack(-qc, -qc);
                    }
                    thr = __double2float_ru(a.r2h - 0.5 * qb * a.c1h);
                }
                int g = 0;
                if (MODE != M_FIX) {
                    // straight-line hit path (taken by ~1 lane of a warp at a time): 4-bit
                    // masks, slot pointer precomputed; ambiguous pairs and slot overflow
                    // are rare out-of-line cases
                    uint16_t *const slotp = em.slot;
                    const int cap = a.cap;
                    auto emit0 = [&](int gg, uint32_t m) {
                        if (MODE == M_SCAN) {
                            if constexpr (SYM) {
                                m = em.symf(gg, m);
                                if (!m) return;
                            }
                            const uint32_t v = ((uint32_t)gg << 4) | m;
                            if (em.rec < cap) {
                                slotp[(size_t)em.rec * a.B] = (uint16_t)v;
                            } else {
                                const int32_t k = atomicAdd(a.ovf_rec_count, 1);
                                if (k < a.ovf_rec_cap) a.ovf_rec[k] = OvfRec{(int32_t)e, em.c, v};
                                else em.lost = true;
                            }
                            ++em.rec;
                        } else if (MODE == M_UNION) {
                            while (m) {
                                const int i = __ffs(m) - 1;
                                m &= m - 1;
                                const int64_t j = c0 + gg * 4 + i;
                                if (j > sp) {   // parent < 0: not core; == root: already joined
                                    // any value parent[j] ever held is a safe filter: links only
                                    // merge components, so pj == uroot means j is already joined
                                    const int32_t pj = a.uload == 0 ? reinterpret_cast<volatile int32_t *>(a.parent)[j]
                                                     : a.uload == 1 ? ld_relaxed_gpu(a.parent + j)
                                                                    : __ldcg(a.parent + j);
                                    if (pj >= 0 && pj != uroot) {
                                        uf_unite(a.parent, (int32_t)sp, (int32_t)j);
                                        uroot = uf_rep(a.parent, (int32_t)sp);
                                    }
                                }
                            }
                        } else if (MODE == M_BORDER) {
                            while (m) {
                                const int i = __ffs(m) - 1;
                                m &= m - 1;
                                const int64_t j = c0 + gg * 4 + i;
                                if (a.core[j]) best = min(best, a.blab[j]);
                            }
                        }
                        em.c += __popc(m);
                    };
                    // G == 3: expanded form eq:ip2 as a cheap conservative filter (PAPER.md:211-216,
                    // margin of reading C20 for fp32 FFMA chains), acc = xbar' - x_c.q_c per
                    // candidate, 2 FFMA2 per coordinate and 4 candidates; candidates go to the
                    // exact direct-form classification below (identical decisions)
                    if constexpr (G == 3 && !CONV) {
                        const float4 *f4 = reinterpret_cast<const float4 *>(smem + sidx * buf_bytes + orig_bytes);
                        for (; g + 1 < ngroups; g += 2) {
                            float4 fa[D + 1], fb[D + 1];
#pragma unroll
                            for (int k = 0; k <= D; ++k) { fa[k] = f4[g * (D + 1) + k]; fb[k] = f4[(g + 1) * (D + 1) + k]; }
                            uint64_t la = f2pack(fa[D].x, fa[D].y), ha = f2pack(fa[D].z, fa[D].w);
                            uint64_t lb = f2pack(fb[D].x, fb[D].y), hb = f2pack(fb[D].z, fb[D].w);
#pragma unroll
                            for (int k = 0; k < D; ++k) {
                                la = f2fma(f2pack(fa[k].x, fa[k].y), nqc[k], la);
                                ha = f2fma(f2pack(fa[k].z, fa[k].w), nqc[k], ha);
                                lb = f2fma(f2pack(fb[k].x, fb[k].y), nqc[k], lb);
                                hb = f2fma(f2pack(fb[k].z, fb[k].w), nqc[k], hb);
                            }
                            const float2 ea = f2unpack(la), eb = f2unpack(ha), ec = f2unpack(lb), ed = f2unpack(hb);
                            const float mnf = fminf(fminf(fminf(ea.x, ea.y), fminf(eb.x, eb.y)),
                                                    fminf(fminf(ec.x, ec.y), fminf(ed.x, ed.y)));
                            if (mnf <= thr) {
                                float4 xa[D], xb[D];
#pragma unroll
                                for (int k = 0; k < D; ++k) { xa[k] = g4[g * D + k]; xb[k] = g4[(g + 1) * D + k]; }
                                uint64_t pla, pha, plb, phb;
                                group_d2<D>(xa, nq, pla, pha);
                                group_d2<D>(xb, nq, plb, phb);
                                const float2 pa = f2unpack(pla), qa = f2unpack(pha), pb = f2unpack(plb), qb = f2unpack(phb);
                                uint32_t ia = mask4(pa.x, pa.y, qa.x, qa.y, T_in);
                                uint32_t ib = mask4(pb.x, pb.y, qb.x, qb.y, T_in);
                                const uint32_t oa = mask4(pa.x, pa.y, qa.x, qa.y, T_out);
                                const uint32_t ob = mask4(pb.x, pb.y, qb.x, qb.y, T_out);
                                if ((ia ^ oa) | (ib ^ ob)) {
                                    ia |= resolve4<D>(oa & ~ia, xa, q, R2);
                                    ib |= resolve4<D>(ob & ~ib, xb, q, R2);
                                }
                                if (ia) emit0(g, ia);
                                if (ib) emit0(g + 1, ib);
                            }
                        }
                    }
                    for (; G == 2 && g + 1 < ngroups; g += 2) {
                        float4 xa[D], xb[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) { xa[k] = g4[g * D + k]; xb[k] = g4[(g + 1) * D + k]; }
                        uint64_t la, ha, lb, hb;
                        group_d2<D>(xa, nq, la, ha);
                        group_d2<D>(xb, nq, lb, hb);
                        const float2 pa = f2unpack(la), qa = f2unpack(ha), pb = f2unpack(lb), qb = f2unpack(hb);
                        const float mn = fminf(fminf(fminf(pa.x, pa.y), fminf(qa.x, qa.y)),
                                               fminf(fminf(pb.x, pb.y), fminf(qb.x, qb.y)));
                        if (mn <= T_out) {
                            uint32_t ia = mask4(pa.x, pa.y, qa.x, qa.y, T_in);
                            uint32_t ib = mask4(pb.x, pb.y, qb.x, qb.y, T_in);
                            const uint32_t oa = mask4(pa.x, pa.y, qa.x, qa.y, T_out);
                            const uint32_t ob = mask4(pb.x, pb.y, qb.x, qb.y, T_out);
                            if ((ia ^ oa) | (ib ^ ob)) {
                                ia |= resolve4<D>(oa & ~ia, xa, q, R2);
                                ib |= resolve4<D>(ob & ~ib, xb, q, R2);
                            }
                            if (ia) emit0(g, ia);
                            if (ib) emit0(g + 1, ib);
                        }
                    }
                    // G == 1: the hit path is deferred.  A candidate group with a pair <= T_out
                    // only pushes (g << 4 | T_out mask) into a 4-record per-lane FIFO (64-bit
                    // register); when any lane's FIFO is full the whole warp drains its FIFOs
                    // together (recomputing the group's d^2 from shared memory, exact
                    // classification, emission), so the expensive path runs convergently
                    // instead of once per hitting lane.  Records keep their g order.
                    // records: index of a GS-group step (g / GS) whose 4 GS pairs have a d^2 <= T_out
                    constexpr int GS = 2;   // 4 measured slower (more records, costlier drains)
                    static_assert(GS == 2, "the step loop below is written for 2 groups");
                    uint64_t pend = 0;
                    int npend = 0;
                    // Drain (called warp-converged).  G3: warp-cooperative -- the warp's records are
                    // listed in shared memory and classified one per lane (owner's query from
                    // shared memory), then every owner emits its records' results in record order
                    // (measured 2.38 -> 2.29 ms on config 2; for G1, whose rows sit in shared
                    // memory, the scattered per-lane groups cost bank conflicts: per-lane drain).
                    auto drain = [&]() {
                        if constexpr (CONV && G == 1) {   // G1 (rows in shared memory): per lane
                            const int rmax = __reduce_max_sync(0xffffffffu, npend);
#pragma unroll 1
                            for (int r = 0; r < rmax; ++r) {
                                if (r < npend) {
                                    const int g0 = GS * (int)((uint32_t)(pend >> (16 * (npend - 1 - r))) & 0xffffu);
#pragma unroll
                                    for (int h = 0; h < GS; ++h) {
                                        const int gg = g0 + h;
                                        if (gg < ngroups) {
                                            float4 xa[D];
#pragma unroll
                                            for (int k = 0; k < D; ++k) xa[k] = g4[gg * D + k];
                                            uint64_t la, ha;
                                            group_d2<D>(xa, nq, la, ha);
                                            const float2 pa = f2unpack(la), qa = f2unpack(ha);
                                            const uint32_t oa = mask4(pa.x, pa.y, qa.x, qa.y, T_out);
                                            if (oa) {
                                                uint32_t ia = mask4(pa.x, pa.y, qa.x, qa.y, T_in);
                                                if (ia ^ oa) ia |= resolve4<D>(oa & ~ia, xa, q, R2);
                                                if (ia) emit0(gg, ia);
                                            }
                                        }
                                    }
                                }
                            }
                        } else if constexpr (CONV) {   // G3 (rows from global memory): one record per lane
                            const int lane = tid & 31, wq = tid >> 5;
                            int incl = npend;
#pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                                if (lane >= o) incl += v;
                            }
                            const int excl = incl - npend;
                            const int total = __shfl_sync(0xffffffffu, incl, 31);
                            uint32_t *drec = s_drec + wq * 128;
                            uint8_t *dres = s_dres + wq * 128;
                            float *dq = s_dq + wq * 32 * D;
                            for (int r = 0; r < npend; ++r)
                                drec[excl + r] = ((uint32_t)lane << 16) | ((uint32_t)(pend >> (16 * (npend - 1 - r))) & 0xffffu);
#pragma unroll
                            for (int k = 0; k < D; ++k) dq[lane * D + k] = (float)q[k];
                            __syncwarp();
                            for (int t = lane; t < total; t += 32) {
                                const uint32_t e = drec[t];
                                const int o = (int)(e >> 16);
                                const int g0 = GS * (int)(e & 0xffffu);
                                float qo[D];
                                uint64_t nqo[D];
#pragma unroll
                                for (int k = 0; k < D; ++k) {
                                    qo[k] = dq[o * D + k];
                                    nqo[k] = f2pack(-qo[k], -qo[k]);
                                }
                                uint32_t res = 0;
#pragma unroll
                                for (int h = 0; h < GS; ++h) {
                                    const int gg = g0 + h;
                                    if (gg < ngroups) {
                                        float4 xa[D];
#pragma unroll
                                        for (int k = 0; k < D; ++k) xa[k] = g4[gg * D + k];
                                        uint64_t la, ha;
                                        group_d2<D>(xa, nqo, la, ha);
                                        const float2 pa = f2unpack(la), qa = f2unpack(ha);
                                        const uint32_t oa = mask4(pa.x, pa.y, qa.x, qa.y, T_out);
                                        if (oa) {
                                            uint32_t ia = mask4(pa.x, pa.y, qa.x, qa.y, T_in);
                                            if (ia ^ oa) ia |= resolve4<D>(oa & ~ia, xa, qo, R2);
                                            res |= ia << (4 * h);
                                        }
                                    }
                                }
                                dres[t] = (uint8_t)res;
                            }
                            __syncwarp();
                            for (int r = 0; r < npend; ++r) {
                                const uint32_t res = dres[excl + r];
                                if (res) {
                                    const int g0 = GS * (int)((uint32_t)(pend >> (16 * (npend - 1 - r))) & 0xffffu);
                                    if (res & 15u) emit0(g0, res & 15u);
                                    if (res >> 4) emit0(g0 + 1, res >> 4);
                                }
                            }
                            __syncwarp();
                        }
                        pend = 0;
                        npend = 0;
                    };
                    constexpr bool LAZY = CONV;
                    const float t_out = T_out;
                    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(g4);
                    uint32_t ga = sbase;
                    for (; LAZY && G == 1 && g + 1 < ngroups; g += 2, ga += 32u * D) {   // 2 groups (8 pairs) per step
                        float4 xa[D], xb[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) { xa[k] = lds128(ga + 16u * k); xb[k] = lds128(ga + 16u * (D + k)); }
                        uint64_t la, ha, lb, hb;
                        group_d2<D>(xa, nq, la, ha);
                        group_d2<D>(xb, nq, lb, hb);
                        const float2 pa = f2unpack(la), qa = f2unpack(ha), pb = f2unpack(lb), qb = f2unpack(hb);
                        const float mn = fminf(fminf(fminf(pa.x, pa.y), fminf(qa.x, qa.y)),
                                               fminf(fminf(pb.x, pb.y), fminf(qb.x, qb.y)));
                        if (mn <= t_out) {
                            pend = (pend << 16) | (uint32_t)(g >> 1);   // FIFO: newest record in the low bits
                            ++npend;
                        }
                        if (__any_sync(0xffffffffu, npend >= 4)) drain();   // FIFO holds 4
                    }
                    // G == 3: the expanded form eq:ip2 as a conservative filter
                    // over the staged rows, acc = xbar' - x_c.q_c (one FFMA2 per coordinate and
                    // 2 candidates) against the rigorous threshold thr (margin of reading C20);
                    // the drain classifies the passing steps exactly in the direct form
                    if constexpr (LAZY && G == 3) {
                        uint32_t fa_addr = (uint32_t)__cvta_generic_to_shared(smem + sidx * buf_bytes + orig_bytes);
                        for (; g + 1 < ngroups; g += 2, fa_addr += 32u * (D + 1)) {
                            float4 fa[D + 1], fb[D + 1];
#pragma unroll
                            for (int k = 0; k <= D; ++k) {
                                fa[k] = lds128(fa_addr + 16u * k);
                                fb[k] = lds128(fa_addr + 16u * (D + 1 + k));
                            }
                            uint64_t la = f2pack(fa[D].x, fa[D].y), ha = f2pack(fa[D].z, fa[D].w);
                            uint64_t lb = f2pack(fb[D].x, fb[D].y), hb = f2pack(fb[D].z, fb[D].w);
#pragma unroll
                            for (int k = 0; k < D; ++k) {
                                la = f2fma(f2pack(fa[k].x, fa[k].y), nqc[k], la);
                                ha = f2fma(f2pack(fa[k].z, fa[k].w), nqc[k], ha);
                                lb = f2fma(f2pack(fb[k].x, fb[k].y), nqc[k], lb);
                                hb = f2fma(f2pack(fb[k].z, fb[k].w), nqc[k], hb);
                            }
                            const float2 ea = f2unpack(la), eb = f2unpack(ha), ec = f2unpack(lb), ed = f2unpack(hb);
                            // 8-way min as 3-input mins (FMNMX3): 4 instructions
                            const float m1 = fminf(fminf(ea.x, ea.y), eb.x), m2 = fminf(fminf(eb.y, ec.x), ec.y);
                            const float m3 = fminf(fminf(ed.x, ed.y), m1);
                            const float mnf = fminf(m2, m3);
                            if (mnf <= thr) {
                                pend = (pend << 16) | (uint32_t)(g >> 1);   // FIFO: newest record in the low bits
                                ++npend;
                            }
                            if (__any_sync(0xffffffffu, npend >= 4)) drain();
                        }
                    }
                    if (LAZY && g < ngroups) {   // tail groups (fewer than GS): one record
                        float mn = INFINITY;
                        for (int gg = g; gg < ngroups; ++gg) {
                            float4 xa[D];
#pragma unroll
                            for (int k = 0; k < D; ++k) xa[k] = g4[gg * D + k];
                            uint64_t la, ha;
                            group_d2<D>(xa, nq, la, ha);
                            const float2 pa = f2unpack(la), qa = f2unpack(ha);
                            mn = fminf(mn, fminf(fminf(pa.x, pa.y), fminf(qa.x, qa.y)));
                        }
                        const bool flag = mn <= t_out;
                        if (__any_sync(0xffffffffu, flag && npend == 4)) drain();   // drains run converged
                        if (flag) {
                            pend = (pend << 16) | (uint32_t)(g / GS);
                            ++npend;
                        }
                        g = ngroups;
                    }
                    if (LAZY) drain();
                    for (; g < ngroups; ++g) {
                        float4 xa[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) xa[k] = g4[g * D + k];
                        uint64_t la, ha;
                        group_d2<D>(xa, nq, la, ha);
                        const float2 pa = f2unpack(la), qa = f2unpack(ha);
                        if (fminf(fminf(pa.x, pa.y), fminf(qa.x, qa.y)) <= T_out) {
                            uint32_t ia = mask4(pa.x, pa.y, qa.x, qa.y, T_in);
                            const uint32_t oa = mask4(pa.x, pa.y, qa.x, qa.y, T_out);
                            if (ia ^ oa) ia |= resolve4<D>(oa & ~ia, xa, q, R2);
                            if (ia) emit0(g, ia);
                        }
                    }
                } else {   // M_FIX: per-candidate classification, direct CSR writes
                    for (; g < ngroups; ++g) {
                        float4 xa[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) xa[k] = g4[g * D + k];
                        uint64_t la, ha;
                        group_d2<D>(xa, nq, la, ha);
                        const float2 pa = f2unpack(la), qa = f2unpack(ha);
                        if (fminf(fminf(pa.x, pa.y), fminf(qa.x, qa.y)) <= T_out)
                            classify4<decltype(em), D, MODE>(em, g, xa, pa.x, pa.y, qa.x, qa.y, T_in, T_out, R2, q);
                    }
                }
            } else {   // fp64 data: the oracle's sequence directly
                const T *gb = reinterpret_cast<const T *>(smem + sidx * buf_bytes);
                for (int g = 0; g < ngroups; ++g) {
                    uint32_t m = 0;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        double s = 0.0;
#pragma unroll
                        for (int k = 0; k < D; ++k) {
                            double t = __dsub_rn(gb[g * 4 * D + k * 4 + i], q[k]);
                            s = __dadd_rn(s, __dmul_rn(t, t));
                        }
                        if (s <= R2) {
                            if (MODE == M_FIX) em.write(c0 + g * 4 + i, s);
                            else m |= 1u << i;
                        }
                    }
                    if (MODE != M_FIX && m) {
                        if (MODE == M_SCAN) {
                            em.record(g, m);
                        } else if (MODE == M_COUNT) {
                            em.c += __popc(m);
                        } else {
                            while (m) {
                                const int i = __ffs(m) - 1;
                                m &= m - 1;
                                const int64_t j = c0 + g * 4 + i;
                                if (MODE == M_UNION && j > sp && a.parent[j] >= 0 && a.parent[j] != uroot) {
                                    uf_unite(a.parent, (int32_t)sp, (int32_t)j);
                                    uroot = uf_rep(a.parent, (int32_t)sp);
                                }
                                if (MODE == M_BORDER && a.core[j]) best = min(best, a.blab[j]);
                            }
                        }
                    }
                }
            }
        }
        if (MODE == M_SCAN) {
            const bool lost = active && em.lost;
            if (tid < a.B) a.cnt[e] = em.c | (lost ? (int32_t)0x80000000 : 0);
            if (a.nrec && tid < a.B) a.nrec[e] = (uint16_t)(em.rec < a.cap ? em.rec : a.cap);
            if (__syncthreads_or(lost) && tid == 0) a.ovf_items[atomicAdd(a.ovf_count, 1)] = (int32_t)item;
        } else {
            if (MODE == M_COUNT) a.cnt[e] = em.c;
            if (MODE == M_BORDER && active && best != 0x7fffffff) atomicMin(&a.best[bpos], best);
            __syncthreads();
        }
    }
}

// K8 scan, two queries per thread (fp32 radius queries with the expanded-form filter,
// B = 256 queries per block on 128 threads: thread t owns queries t and t + 128).  Every
// staged filter row is read once for both queries, so the shared-memory loads and the loop
// bookkeeping per pair halve.  Same filter, same deferred FIFO records per query, same
// warp-cooperative exact drain and the same hit records / counts as window_lowd<G3>.
#ifdef K2Q_MINB
#define K2Q_BOUNDS __launch_bounds__(128, K2Q_MINB)
#else
#define K2Q_BOUNDS __launch_bounds__(128)
#endif
template <int D, bool SYM>
__global__ void K2Q_BOUNDS window_lowd_2q(PassArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int FW = D + 1, NW = 4, GS = 2;
    __shared__ uint16_t s_drec[NW * 256];   // (owner << 10) | step: chunk <= 8192 candidates = 1024 steps
    __shared__ uint32_t s_own[NW * 64 * 2];  // per owner: (first record | records so far << 16), hits so far (bit 31: lost)
    __shared__ uint8_t s_dres[NW * 256];
    __shared__ float s_q[NW * 64 * D];   // per warp: owner o = 2 * lane + s
    // per-query FIFO of deferred records (step indices), 4 slots: slot r of query (s, tid) at
    // s_fifo[(r * 2 + s) * 128 + tid]; a push is one predicated 16-bit store + pointer bump
    __shared__ uint16_t s_fifo[4 * 2 * 128];
    constexpr int FSTR = 2 * 128;   // slot stride (elements)
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    const float *Xs = static_cast<const float *>(a.Xs);
    const float *Qs = static_cast<const float *>(a.Qs);
    const size_t buf_bytes = (size_t)a.chunk * FW * 4;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 2 * buf_bytes);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t item, int sidx) {
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const uint32_t fbytes = (uint32_t)((c1 - c0) * FW * 4);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bar[sidx], fbytes);
        bulk_g2s(smem + sidx * buf_bytes, a.Xf + c0 * FW, fbytes, &bar[sidx]);
    };
    uint32_t phase[2] = {0u, 0u};
    int64_t w = blockIdx.x;
    if (tid == 0 && w < a.total_items) issue(w, 0);
    const float T_in = a.T_in, T_out = a.T_out;
    const double R2 = a.R2;
    const int cap = a.cap;
    float *dq = s_q + wq * 64 * D;
    for (int it = 0; w < a.total_items; w += gridDim.x, ++it) {
        const int sidx = it & 1;
        const int64_t wn = w + gridDim.x;
        if (tid == 0 && wn < a.total_items) issue(wn, sidx ^ 1);
        const int64_t item = w;
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        // per-query state (s = 0, 1: queries tid, tid + 128 of the block)
        int64_t sp[2], e[2];
        bool active[2];
        uint64_t nqc[2][D];
        float thr[2];
        // 32-bit shared addresses (bytes): query s pushes at fp[s], full at flim + 256 * s
        const uint16_t *const fbase = s_fifo + tid;
        const uint32_t fb = (uint32_t)__cvta_generic_to_shared(s_fifo + tid);
        uint32_t fp[2] = {fb, fb + 256u};
        const uint32_t flim = fb + 4u * 2u * FSTR;
        auto push = [&](int s, uint32_t v) {
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(fp[s]), "h"((uint16_t)v) : "memory");
            fp[s] += 2u * FSTR;
        };
        int32_t cnt[2] = {0, 0}, rec[2] = {0, 0};
        bool lost[2] = {false, false};
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int qi = tid + 128 * s;
            sp[s] = b * a.B + qi;
            e[s] = item * a.B + qi;
            active[s] = sp[s] < a.m;
            double qb = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const float qk = active[s] ? Qs[(sp[s] >> 2) * 4 * D + k * 4 + (sp[s] & 3)] : NAN;   // NaN: no hits
                dq[(2 * lane + s) * D + k] = qk;
                const float qc = (float)((double)qk - (double)a.mu_f[k]);
                qb += (double)qc * (double)qc;
                nqc[s][k] = f2pack(-qc, -qc);
            }
            thr[s] = __double2float_ru(a.r2h - 0.5 * qb * a.c1h);
            // pin thr to a register: ptxas otherwise rematerialises the fp64 sequence above
            // inside the step loop (12 fp64 instructions per step in SASS); a shuffle from the
            // own lane is not rematerialisable
            thr[s] = __shfl_sync(0xffffffffu, thr[s], lane);
        }
        __syncwarp();
        mbar_wait(&bar[sidx], phase[sidx]);
        phase[sidx] ^= 1u;
        const int ngroups = (int)((c1 - c0) >> 2);
        const float4 *g4 = reinterpret_cast<const float4 *>(Xs) + (c0 >> 2) * D;   // exact rows (global)
        // Warp-cooperative drain, lane-parallel throughout: (1) every owner lists its pending
        // records and its entry's running counts in shared memory; (2) one record per lane is
        // classified exactly in the direct form from the global rows (symmetric self-query:
        // only j > i kept, mirrored hits counted); (3) the same lane writes the record's slot
        // entries -- its slot index is the owner's count plus the entries of the owner's
        // earlier records in this drain (at most 3, read back from the result list), so slot
        // order stays record order; (4) owners add up their records' entries and hits.
        uint16_t *const slot_item = a.slots + (size_t)item * cap * a.B;
        auto drain = [&]() {
            const int npend[2] = {(int)((fp[0] - fb) / (2u * FSTR)), (int)((fp[1] - fb - 256u) / (2u * FSTR))};
            const int mine = npend[0] + npend[1];
            int incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const int excl = incl - mine;
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            uint16_t *drec = s_drec + wq * 256;
            uint8_t *dres = s_dres + wq * 256;
            uint32_t *own = s_own + wq * 128;
            int pos = excl;
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                own[2 * (2 * lane + s)] = (uint32_t)pos | ((uint32_t)rec[s] << 16);
                own[2 * (2 * lane + s) + 1] = (uint32_t)cnt[s];
                for (int r = 0; r < npend[s]; ++r)
                    drec[pos++] = (uint16_t)(((uint32_t)(2 * lane + s) << 10) | fbase[128 * s + FSTR * r]);
            }
            __syncwarp();
            for (int t = lane; t < total; t += 32) {
                const uint32_t ev = drec[t];
                const int o = (int)(ev >> 10);
                const int g0 = GS * (int)(ev & 0x3ffu);
                float qo[D];
                uint64_t nqo[D];
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    qo[k] = dq[o * D + k];
                    nqo[k] = f2pack(-qo[k], -qo[k]);
                }
                uint32_t res = 0;
#pragma unroll
                for (int h = 0; h < GS; ++h) {
                    const int gg = g0 + h;
                    if (gg < ngroups) {
                        float4 xa[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) xa[k] = g4[gg * D + k];
                        uint64_t la, ha;
                        group_d2<D>(xa, nqo, la, ha);
                        const float2 pa = f2unpack(la), qa = f2unpack(ha);
                        const uint32_t oa = mask4(pa.x, pa.y, qa.x, qa.y, T_out);
                        if (oa) {
                            uint32_t ia = mask4(pa.x, pa.y, qa.x, qa.y, T_in);
                            if (ia ^ oa) ia |= resolve4<D>(oa & ~ia, xa, qo, R2);
                            if constexpr (SYM) {   // keep j > sp of the owner, count the mirrored hits
                                const int64_t spo = b * a.B + 32 * wq + (o >> 1) + 128 * (o & 1);
                                const int64_t jb = c0 + 4 * gg;
                                if (jb + 3 <= spo) ia = 0;
                                else if (jb <= spo) ia &= ~((2u << (spo - jb)) - 1u);
                                uint32_t mm = ia;
                                while (mm) {
                                    const int i = __ffs(mm) - 1;
                                    mm &= mm - 1;
                                    if (jb + i < a.own_hi) atomicAdd(&a.lcnt[jb + i], 1);   // rows of later parts: theirs
                                }
                            }
                            res |= ia << (4 * h);
                        }
                    }
                }
                dres[t] = (uint8_t)res;
            }
            __syncwarp();
            for (int t = lane; t < total; t += 32) {
                uint32_t res = dres[t];
                if (res) {
                    const uint32_t ev = drec[t];
                    const int o = (int)(ev >> 10);
                    const int g0 = GS * (int)(ev & 0x3ffu);
                    const uint32_t w0 = own[2 * o];
                    int idx = (int)(w0 >> 16);                          // entries before this record
                    int hits = (int)(own[2 * o + 1] & 0x7fffffffu);     // hits before this record
                    for (int u = (int)(w0 & 0xffffu); u < t; ++u) {
                        const uint32_t x = dres[u];
                        idx += ((x & 15u) != 0) + ((x >> 4) != 0);
                        hits += __popc(x);
                    }
                    const int qi = 32 * wq + (o >> 1) + 128 * (o & 1);
#pragma unroll
                    for (int h = 0; h < GS; ++h) {
                        const uint32_t m = (res >> (4 * h)) & 15u;
                        if (m) {
                            const uint32_t v = ((uint32_t)(g0 + h) << 4) | m;
                            if (idx < cap) {
                                slot_item[(uint32_t)idx * (uint32_t)a.B + qi] = (uint16_t)v;
                            } else {
                                const int32_t kk = atomicAdd(a.ovf_rec_count, 1);
                                if (kk < a.ovf_rec_cap) a.ovf_rec[kk] = OvfRec{(int32_t)(item * a.B + qi), hits, v};
                                else atomicOr(&own[2 * o + 1], 0x80000000u);
                            }
                            ++idx;
                            hits += __popc(m);
                        }
                    }
                }
            }
            __syncwarp();
            pos = excl;
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                for (int r = 0; r < npend[s]; ++r, ++pos) {
                    const uint32_t x = dres[pos];
                    rec[s] += ((x & 15u) != 0) + ((x >> 4) != 0);
                    cnt[s] += __popc(x);
                }
                if (own[2 * (2 * lane + s) + 1] >> 31) lost[s] = true;
                fp[s] = fb + 256u * s;
            }
            __syncwarp();
        };
        int g = 0;
        uint32_t fa_addr = (uint32_t)__cvta_generic_to_shared(smem + sidx * buf_bytes);
        for (; g + 1 < ngroups; g += 2, fa_addr += 32u * FW) {
            float4 fa[FW], fb[FW];
#pragma unroll
            for (int k = 0; k < FW; ++k) {
                fa[k] = lds128(fa_addr + 16u * k);
                fb[k] = lds128(fa_addr + 16u * (FW + k));
            }
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                uint64_t la = f2pack(fa[D].x, fa[D].y), ha = f2pack(fa[D].z, fa[D].w);
                uint64_t lb = f2pack(fb[D].x, fb[D].y), hb = f2pack(fb[D].z, fb[D].w);
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    la = f2fma(f2pack(fa[k].x, fa[k].y), nqc[s][k], la);
                    ha = f2fma(f2pack(fa[k].z, fa[k].w), nqc[s][k], ha);
                    lb = f2fma(f2pack(fb[k].x, fb[k].y), nqc[s][k], lb);
                    hb = f2fma(f2pack(fb[k].z, fb[k].w), nqc[s][k], hb);
                }
                const float2 ea = f2unpack(la), eb = f2unpack(ha), ec = f2unpack(lb), ed = f2unpack(hb);
                const float m1 = fminf(fminf(ea.x, ea.y), eb.x), m2 = fminf(fminf(eb.y, ec.x), ec.y);
                const float m3 = fminf(fminf(ed.x, ed.y), m1);
                if (fminf(m2, m3) <= thr[s]) push(s, (uint32_t)g >> 1);
            }
            if (__any_sync(0xffffffffu, (fp[0] >= flim) | (fp[1] >= flim + 256u))) drain();
        }
        if (g < ngroups) {   // tail group (odd count): direct form from the global rows, one record
            float4 xa[D];
#pragma unroll
            for (int k = 0; k < D; ++k) xa[k] = g4[g * D + k];
            bool flag[2];
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                uint64_t nq[D];
#pragma unroll
                for (int k = 0; k < D; ++k) nq[k] = f2pack(-dq[(2 * lane + s) * D + k], -dq[(2 * lane + s) * D + k]);
                uint64_t la, ha;
                group_d2<D>(xa, nq, la, ha);
                const float2 pa = f2unpack(la), qa = f2unpack(ha);
                flag[s] = fminf(fminf(pa.x, pa.y), fminf(qa.x, qa.y)) <= T_out;
            }
            if (__any_sync(0xffffffffu, (flag[0] && fp[0] >= flim) | (flag[1] && fp[1] >= flim + 256u))) drain();
#pragma unroll
            for (int s = 0; s < 2; ++s)
                if (flag[s]) push(s, (uint32_t)(g / GS));
        }
        drain();
        bool anylost = false;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const bool ls = active[s] && lost[s];
            anylost |= ls;
            a.cnt[e[s]] = cnt[s] | (ls ? (int32_t)0x80000000 : 0);
            if (a.nrec) a.nrec[e[s]] = (uint16_t)(rec[s] < cap ? rec[s] : cap);
        }
        if (__syncthreads_or(anylost) && tid == 0) a.ovf_items[atomicAdd(a.ovf_count, 1)] = (int32_t)item;
    }
}

// Compaction of the recorded hits into the CSR: original ids via pi and distances as
// (float)sqrt of the oracle-order fp64 squared distance.  One CTA per item; one thread
// per (item, query) entry expands its slot records (the first `cap` records).
template <typename T, int D>
__device__ __forceinline__ void expand_record(const PassArgs &a, int64_t c0, uint32_t v,
                                                   const T (&q)[D], int64_t &pos, int64_t sp) {
    const T *Xs = static_cast<const T *>(a.Xs);
    const int64_t g = c0 / 4 + (v >> 4);
    uint32_t mask = v & 15u;
    while (mask) {
        const int i = __ffs(mask) - 1;
        mask &= mask - 1;
        T x[D];
#pragma unroll
        for (int k = 0; k < D; ++k) x[k] = Xs[g * 4 * D + k * 4 + i];
        const float dd = (float)sqrt(sqdist_exact(x, q, D));
        SNN_DASSERT(a.n_index <= 0 || g * 4 + i < a.n_index);
        if (sp >= a.own_lo) put_entry(a, pos, a.perm[g * 4 + i], dd);   // ghost queries: mirrors only
        ++pos;
        if (a.sym && g * 4 + i < a.own_hi) {
            const unsigned long long k = atomicAdd(&a.lpos[g * 4 + i], 1ull);
            SNN_DASSERT(k < (unsigned long long)a.offsets[a.m]);
            a.tmpL[k] = ((unsigned long long)sp << 32) | __float_as_uint(dd);
        }
    }
}

template <typename T, int D>
__global__ void __launch_bounds__(256) compact_lowd(PassArgs a) {
    const T *Qs = static_cast<const T *>(a.Qs);
    for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const int64_t sp = b * a.B + threadIdx.x;
        if (sp >= a.m) continue;
        const int64_t e = item * a.B + threadIdx.x;
        const int32_t cv = a.cnt[e];
        if (cv <= 0) continue;   // no hits, or lost entry (sign bit): the fix pass writes it
        int64_t pos = row_base(a, sp) + a.pre[e];
        const int64_t end = pos + cv;
        T q[D];
#pragma unroll
        for (int k = 0; k < D; ++k) q[k] = Qs[(sp >> 2) * 4 * D + k * 4 + (sp & 3)];
        const uint16_t *slot = a.slots + (size_t)item * a.B * a.cap + threadIdx.x;
        uint32_t v = slot[0];
        for (int r = 0; r < a.cap && pos < end; ++r) {
            const uint32_t nv = (r + 1 < a.cap) ? slot[(size_t)(r + 1) * a.B] : 0u;   // prefetch
            expand_record<T, D>(a, c0, v, q, pos, sp);
            v = nv;
        }
    }
}

// Balanced compaction: the CTA lists its item's slot records (entries in order, records in
// order) and gives one record per thread, so an entry with many hits no longer holds the
// whole CTA; a record's place in its row is its entry's row base plus the prefix sum of
// the hit counts of the entry's earlier records (CTA scans).
template <typename T, int D>
__global__ void __launch_bounds__(256) compact_lowd_bal(PassArgs a) {
    __shared__ int32_t s_rstart[257];
    __shared__ int64_t s_base[256];
    __shared__ int32_t s_hbase[256];
    __shared__ T s_q[256 * D];
    __shared__ int32_t s_wsum[8];
    const T *Qs = static_cast<const T *>(a.Qs);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    auto block_excl = [&](int v, int &total) {   // exclusive block scan (256 threads)
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_wsum[wid] = incl;
        __syncthreads();
        int before = 0;
        total = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const int x = s_wsum[w];
            before += w < wid ? x : 0;
            total += x;
        }
        __syncthreads();
        return before + incl - v;
    };
    for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const int64_t sp = b * a.B + tid;
        const int64_t e = item * a.B + tid;
        int nr = 0;
        if (sp < a.m) {
            const int32_t cv = a.cnt[e];
            if (cv > 0) {   // cv < 0: lost entry (the fix pass writes it)
                nr = a.nrec[e];
                s_base[tid] = row_base(a, sp) + a.pre[e];
#pragma unroll
                for (int k = 0; k < D; ++k) s_q[tid * D + k] = Qs[(sp >> 2) * 4 * D + k * 4 + (sp & 3)];
            }
        }
        int R = 0;
        const int rs = block_excl(nr, R);
        s_rstart[tid] = rs;
        if (tid == 0) s_rstart[256] = R;
        __syncthreads();
        int carry = 0;
        for (int k0 = 0; k0 < R; k0 += 256) {
            const int k = k0 + tid;
            int owner = 0, r = 0;
            uint32_t v = 0;
            if (k < R) {   // owner = last entry with rstart <= k
                int lo = 0, hi = 256;
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_rstart[mid] <= k) lo = mid; else hi = mid;
                }
                owner = lo;
                r = k - s_rstart[owner];
                v = a.slots[((size_t)item * a.cap + r) * a.B + owner];
            }
            const int h = k < R ? __popc(v & 15u) : 0;
            int hsum = 0;
            const int hex = block_excl(h, hsum) + carry;
            if (k < R && r == 0) s_hbase[owner] = hex;
            __syncthreads();
            if (k < R) {
                int64_t pos = s_base[owner] + (hex - s_hbase[owner]);
                T q[D];
#pragma unroll
                for (int kk = 0; kk < D; ++kk) q[kk] = s_q[owner * D + kk];
                expand_record<T, D>(a, c0, v, q, pos, b * a.B + owner);
            }
            carry += hsum;
            __syncthreads();
        }
    }
}

// Records beyond `cap` (global overflow list): one thread per record.
template <typename T, int D>
__global__ void __launch_bounds__(256) compact_overflow(PassArgs a, int64_t n_rec) {
    const T *Qs = static_cast<const T *>(a.Qs);
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_rec;
         k += (int64_t)gridDim.x * blockDim.x) {
        const OvfRec r = a.ovf_rec[k];
        if (a.cnt[r.e] < 0) continue;   // lost entry: rewritten by the fix pass
        const int64_t item = r.e / a.B, t = r.e % a.B;
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const int64_t sp = b * a.B + t;
        int64_t pos = row_base(a, sp) + a.pre[r.e] + r.before;
        T q[D];
#pragma unroll
        for (int kk = 0; kk < D; ++kk) q[kk] = Qs[(sp >> 2) * 4 * D + kk * 4 + (sp & 3)];
        expand_record<T, D>(a, c0, r.v, q, pos, sp);
    }
}

// ---------------------------------------------------------------------------- K8 generic d
// 64 queries x 64 candidates per tile, 256 threads, 4x4 pairs per thread, K staged in
// shared memory in slices of 16 dimensions.  Same classification as the low-d kernel.
constexpr int kGB = 64, kKT = 16;

template <typename T, bool WRITE>
__global__ void __launch_bounds__(256) window_generic(PassArgs a) {
    __shared__ __align__(16) T Qt[kKT][kGB + 4];
    __shared__ __align__(16) T Ct[kKT][kGB + 4];
    __shared__ int32_t s_cnt[kGB];
    __shared__ int64_t s_base[kGB];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const T *Xs = static_cast<const T *>(a.Xs);
    const T *Qs = static_cast<const T *>(a.Qs);
    const int ld = a.ld;
    for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const int64_t sp0 = b * kGB;
        if (tid < kGB) {
            s_cnt[tid] = 0;
            if (WRITE && sp0 + tid < a.m)
                s_base[tid] = a.offsets[a.qperm[sp0 + tid]] + a.pre[item * kGB + tid];
        }
        __syncthreads();
        for (int64_t cb = c0; cb < c1; cb += kGB) {
            T acc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = (T)0;
            for (int k0 = 0; k0 < ld; k0 += kKT) {
                for (int e = tid; e < kGB * kKT; e += 256) {
                    const int r = e / kKT, kk = e % kKT, k = k0 + kk;
                    const int64_t qrow = sp0 + r, crow = cb + r;
                    Qt[kk][r] = (qrow < a.m && k < ld) ? Qs[qrow * ld + k] : (T)0;
                    Ct[kk][r] = (crow < c1 && k < ld) ? Xs[crow * ld + k] : (T)0;
                }
                __syncthreads();
#pragma unroll
                for (int kk = 0; kk < kKT; ++kk) {
                    T qa[4], xb[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) { qa[i] = Qt[kk][ty * 4 + i]; xb[i] = Ct[kk][tx * 4 + i]; }
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            if constexpr (sizeof(T) == 4) {
                                float t = xb[j] - qa[i];
                                acc[i][j] = fmaf(t, t, acc[i][j]);
                            } else {
                                double t = __dsub_rn(xb[j], qa[i]);
                                acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(t, t));
                            }
                        }
                }
                __syncthreads();
            }
            // classify the 16 pairs
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int qi = ty * 4 + i;
                const int64_t sp = sp0 + qi;
                bool hit[4];
                double sv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t cj = cb + tx * 4 + j;
                    hit[j] = false;
                    sv[j] = 0.0;
                    if (sp < a.m && cj < c1) {
                        if constexpr (sizeof(T) == 4) {
                            const float d2 = acc[i][j];
                            if (d2 <= a.T_out) {
                                hit[j] = d2 <= a.T_in;
                                if (WRITE || !hit[j]) {
                                    sv[j] = sqdist_exact(Xs + cj * ld, Qs + sp * ld, a.d);
                                    if (!hit[j]) hit[j] = sv[j] <= a.R2;
                                }
                            }
                        } else {
                            sv[j] = acc[i][j];
                            hit[j] = sv[j] <= a.R2;
                        }
                    }
                }
                int h = (int)hit[0] + (int)hit[1] + (int)hit[2] + (int)hit[3];
                if (!WRITE) {
#pragma unroll
                    for (int o = 8; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o, 16);
                    if (tx == 0) s_cnt[qi] += h;
                } else {
                    int inc = h;
#pragma unroll
                    for (int o = 1; o < 16; o <<= 1) {
                        int y = __shfl_up_sync(0xffffffffu, inc, o, 16);
                        if (tx >= o) inc += y;
                    }
                    const int64_t base = (sp < a.m) ? s_base[qi] : 0;
                    __syncwarp();
                    int64_t p = base + inc - h;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (hit[j]) {
                            a.out_idx[p] = a.perm[cb + tx * 4 + j];
                            a.out_dist[p] = (float)sqrt(sv[j]);
                            ++p;
                        }
                    }
                    if (tx == 15 && sp < a.m) s_base[qi] = base + inc;
                    __syncwarp();
                }
            }
        }
        __syncthreads();
        if (!WRITE && tid < kGB) a.cnt[item * kGB + tid] = s_cnt[tid];
        __syncthreads();
    }
}

__global__ void row_totals(const int32_t *cnt, int32_t *pre, const int64_t *item_start, int64_t m,
                           int B, const int32_t *qperm, int32_t *row_count, int32_t *srow) {
    const int64_t sp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sp >= m) return;
    const int64_t b = sp / B, t = sp % B;
    int32_t run = 0;
    for (int64_t item = item_start[b]; item < item_start[b + 1]; ++item) {
        int32_t c = cnt[item * B + t] & 0x7fffffff;   // bit 31 = hit-slot overflow flag
        pre[item * B + t] = run;
        run += c;
    }
    row_count[qperm ? qperm[sp] : sp] = run;
    if (srow) srow[sp] = run;
}

__global__ void row_totals_sym(const int32_t *cnt, int32_t *pre, const int64_t *item_start, int64_t m, int B,
                               const int32_t *qperm, const int32_t *lcnt, int32_t *row_count, int32_t *maxl,
                               int32_t *srow, int64_t own_lo, int64_t own_hi) {
    const int64_t sp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sp >= m) return;
    if (sp < own_lo || sp >= own_hi) {   // another part's row (partitioned self-query)
        row_count[qperm[sp]] = 0;
        if (srow) srow[sp] = 0;
        return;
    }
    const int64_t b = sp / B, t = sp % B;
    const int32_t l = lcnt[sp];
    int32_t run = l + 1;   // L segment, then the point itself
    for (int64_t item = item_start[b]; item < item_start[b + 1]; ++item) {
        int32_t c = cnt[item * B + t] & 0x7fffffff;
        pre[item * B + t] = run;
        run += c;
    }
    row_count[qperm[sp]] = run;
    if (srow) srow[sp] = run;
    atomicMax(maxl, l);
}

// L segments: warp per row, bitonic sort of (position << 32 | distance bits) in registers
// (<= 32) or shared memory (<= 512); the CTA variant takes rows up to 16384.
constexpr int kLWarp = 512, kLBlock = 16384;
__device__ __forceinline__ void lemit(const PassArgs &a, unsigned long long v, int64_t pos) {
    SNN_DASSERT(pos >= 0 && pos < a.offsets[a.m] && (int64_t)(v >> 32) < a.m);
    a.out_idx[pos] = a.perm[(uint32_t)(v >> 32)];
    a.out_dist[pos] = __uint_as_float((uint32_t)v);
}
// Warp per row.  Symmetric self-query: the row's L segment (mirrored entries, arrival order)
// is sorted by position -- rank sort in registers (<= 32 entries; positions are unique), a
// shared-memory bitonic sort (<= 512; longer rows: rows_lsort_block) -- and written with
// the self entry.  Staged rows: the rest of the row is copied from the key-order staging
// buffer to the row's original-id position.
__global__ void __launch_bounds__(256) rows_finalize_warp(PassArgs a) {
    __shared__ unsigned long long sbuf[8][kLWarp];
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    unsigned long long *buf = sbuf[w];
    // staged rows with the inverse permutation: warps walk the OUTPUT rows in original-id
    // order, so consecutive warps write consecutive CSR memory (whole sectors; random row
    // writes leave partial sectors that HBM's ECC turns into read-modify-writes)
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < a.m;
         r += (int64_t)gridDim.x * blockDim.x / 32) {
        const int64_t sp = a.qinv ? (int64_t)a.qinv[r] : r;
        if (sp < a.own_lo || sp >= a.own_hi) continue;   // another part's (empty) row
        const int cnt = a.sym ? a.lcnt[sp] : 0;
        const int64_t src = a.soff ? a.soff[sp] : (int64_t)a.lpos[sp] - cnt;   // L cursor advanced by cnt
        const int64_t dst = a.soff ? a.offsets[a.qinv ? r : a.qperm[sp]] : (a.loff ? row_base(a, sp) : src);
        if (a.soff) {   // U part (after L and self) or the whole row
            const int64_t k0 = a.sym ? cnt + 1 : 0, len = a.soff[sp + 1] - src;
            SNN_DASSERT(src >= 0 && src + len <= a.offsets[a.m] && dst + len <= a.offsets[a.m]);
            for (int64_t k = k0 + lane; k < len; k += 32) {
                const unsigned long long v = a.stage[src + k];
                a.out_idx[dst + k] = (int32_t)(uint32_t)v;
                a.out_dist[dst + k] = __uint_as_float((uint32_t)(v >> 32));
            }
        }
        if (!a.sym) continue;
        if (lane == 0) { a.out_idx[dst + cnt] = a.perm[sp]; a.out_dist[dst + cnt] = 0.f; }   // the point itself
        if (cnt == 0 || cnt > kLWarp) continue;
        if (cnt <= 32) {   // rank sort: positions are unique within a row
            const unsigned long long v = lane < cnt ? a.tmpL[src + lane] : ~0ull;
            const uint32_t key = (uint32_t)(v >> 32);   // lanes >= cnt: ~0, never "<"
            int rank = 0;
            for (int j = 0; j < cnt; j += 4) {
                rank += __shfl_sync(0xffffffffu, key, j) < key;
                rank += __shfl_sync(0xffffffffu, key, j + 1) < key;
                rank += __shfl_sync(0xffffffffu, key, j + 2) < key;
                rank += __shfl_sync(0xffffffffu, key, j + 3) < key;
            }
            if (lane < cnt) lemit(a, v, dst + rank);
            continue;
        }
        if (cnt <= 64) {   // two entries per lane, rank sort in registers
            const unsigned long long v0 = a.tmpL[src + lane];
            const unsigned long long v1 = lane + 32 < cnt ? a.tmpL[src + lane + 32] : ~0ull;
            const uint32_t k0 = (uint32_t)(v0 >> 32), k1 = (uint32_t)(v1 >> 32);
            int r0 = 0, r1 = 0;
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
                const uint32_t kj = __shfl_sync(0xffffffffu, k0, j);
                r0 += kj < k0;
                r1 += kj < k1;
            }
            for (int j = 0; j < cnt - 32; j += 2) {
                const uint32_t kj = __shfl_sync(0xffffffffu, k1, j);
                const uint32_t kk = __shfl_sync(0xffffffffu, k1, j + 1);
                r0 += (kj < k0) + (kk < k0);
                r1 += (kj < k1) + (kk < k1);
            }
            lemit(a, v0, dst + r0);
            if (lane + 32 < cnt) lemit(a, v1, dst + r1);
            continue;
        }
        int S = 64;
        while (S < cnt) S <<= 1;
        for (int i = lane; i < S; i += 32) buf[i] = i < cnt ? a.tmpL[src + i] : ~0ull;
        __syncwarp();
        for (int k = 2; k <= S; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int t = lane; t < S / 2; t += 32) {   // one compare-exchange pair per thread
                    const int i = 2 * t - (t & (j - 1)), p = i + j;
                    const unsigned long long x = buf[i], y = buf[p];
                    if ((x > y) == ((i & k) == 0)) { buf[i] = y; buf[p] = x; }
                }
                __syncwarp();
            }
        }
        for (int i = lane; i < cnt; i += 32) lemit(a, buf[i], dst + i);
        __syncwarp();
    }
}
// Symmetric self-query with direct rows (no staging): warp per 32 consecutive key
// positions.  The lanes load the 32 rows' L counts, cursors and self ids together
// (coalesced), then the warp walks the rows software-pipelined: row k+1's L segment is
// loaded while row k is ranked, and row k's output stores wait one row for their perm[]
// load, so the per-row chain of dependent global loads (count -> segment -> perm ->
// store) overlaps across rows instead of serialising (rows_finalize_warp: one row per warp).
// Rows with more than 64 L entries take the shared-memory bitonic sort of
// rows_finalize_warp (<= 512) or rows_lsort_block (more).
__global__ void __launch_bounds__(256) rows_finalize_pipe(PassArgs a) {
    __shared__ unsigned long long sbuf[8][kLWarp];
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    unsigned long long *buf = sbuf[w];
    const int64_t nw = (int64_t)gridDim.x * 8;
    for (int64_t r0 = ((int64_t)blockIdx.x * 8 + w) * 32; r0 < a.m; r0 += nw * 32) {
        const int64_t spl = r0 + lane;
        const bool own = spl < a.m && spl >= a.own_lo && spl < a.own_hi;
        const int cl = own ? a.lcnt[spl] : 0;
        const int64_t bl = own ? (int64_t)a.lpos[spl] - cl : 0;   // L cursor advanced by cl
        const int64_t dl = own && a.loff ? row_base(a, spl) : bl;   // row start in the CSR
        if (own) {   // the point itself, after its L segment
            SNN_DASSERT(dl + cl < a.offsets[a.m]);
            a.out_idx[dl + cl] = a.perm[spl];
            a.out_dist[dl + cl] = 0.f;
        }
        auto load = [&](int k, unsigned long long &v0, unsigned long long &v1) {
            const int c = __shfl_sync(0xffffffffu, cl, k);
            const int64_t b = __shfl_sync(0xffffffffu, bl, k);
            v0 = (c <= 64 && lane < c) ? a.tmpL[b + lane] : ~0ull;
            v1 = (c <= 64 && lane + 32 < c) ? a.tmpL[b + lane + 32] : ~0ull;
        };
        unsigned long long v0, v1;
        load(0, v0, v1);
        // pending stores of the previous row: id (perm[] load in flight), distance, position
        int32_t pid0 = 0, pid1 = 0;
        float pd0 = 0.f, pd1 = 0.f;
        int64_t pp0 = -1, pp1 = -1;
        for (int k = 0; k < 32; ++k) {
            const int c = __shfl_sync(0xffffffffu, cl, k);
            const int64_t b = __shfl_sync(0xffffffffu, bl, k);    // L segment (tmpL)
            const int64_t o = __shfl_sync(0xffffffffu, dl, k);    // row start (CSR)
            unsigned long long n0 = ~0ull, n1 = ~0ull;
            if (k + 1 < 32) load(k + 1, n0, n1);   // prefetch the next row's segment
            int64_t q0 = -1, q1 = -1;
            int32_t id0 = 0, id1 = 0;
            if (c > 0 && c <= 32) {   // rank sort: positions are unique within a row
                const uint32_t k0 = (uint32_t)(v0 >> 32);
                int r0 = 0;
                for (int j = 0; j < c; j += 4) {   // lanes >= c hold ~0: never "<"
                    r0 += __shfl_sync(0xffffffffu, k0, j) < k0;
                    r0 += __shfl_sync(0xffffffffu, k0, j + 1) < k0;
                    r0 += __shfl_sync(0xffffffffu, k0, j + 2) < k0;
                    r0 += __shfl_sync(0xffffffffu, k0, j + 3) < k0;
                }
                if (lane < c) { q0 = o + r0; id0 = a.perm[k0]; }
            } else if (c > 32 && c <= 64) {
                const uint32_t k0 = (uint32_t)(v0 >> 32), k1 = (uint32_t)(v1 >> 32);
                int r0 = 0, r1 = 0;
                const int c32 = c < 32 ? c : 32;
                for (int j = 0; j < c32; ++j) {
                    const uint32_t kj = __shfl_sync(0xffffffffu, k0, j);
                    r0 += kj < k0;
                    r1 += kj < k1;
                }
                for (int j = 0; j < c - 32; ++j) {
                    const uint32_t kj = __shfl_sync(0xffffffffu, k1, j);
                    r0 += kj < k0;
                    r1 += kj < k1;
                }
                if (lane < c) { q0 = o + r0; id0 = a.perm[k0]; }
                if (lane + 32 < c) { q1 = o + r1; id1 = a.perm[k1]; }
            } else if (c > 64 && c <= kLWarp) {   // shared-memory bitonic sort
                int S = 128;
                while (S < c) S <<= 1;
                for (int i = lane; i < S; i += 32) buf[i] = i < c ? a.tmpL[b + i] : ~0ull;
                __syncwarp();
                for (int kk = 2; kk <= S; kk <<= 1) {
                    for (int j = kk >> 1; j > 0; j >>= 1) {
                        for (int t = lane; t < S / 2; t += 32) {
                            const int i = 2 * t - (t & (j - 1)), p = i + j;
                            const unsigned long long x = buf[i], y = buf[p];
                            if ((x > y) == ((i & kk) == 0)) { buf[i] = y; buf[p] = x; }
                        }
                        __syncwarp();
                    }
                }
                for (int i = lane; i < c; i += 32) lemit(a, buf[i], o + i);
                __syncwarp();
            }
            if (pp0 >= 0) { a.out_idx[pp0] = pid0; a.out_dist[pp0] = pd0; }
            if (pp1 >= 0) { a.out_idx[pp1] = pid1; a.out_dist[pp1] = pd1; }
            SNN_DASSERT(q0 < 0 || q0 < a.offsets[a.m]);
            SNN_DASSERT(q1 < 0 || q1 < a.offsets[a.m]);
            pp0 = q0; pid0 = id0; pd0 = __uint_as_float((uint32_t)v0);
            pp1 = q1; pid1 = id1; pd1 = __uint_as_float((uint32_t)v1);
            v0 = n0;
            v1 = n1;
        }
        if (pp0 >= 0) { a.out_idx[pp0] = pid0; a.out_dist[pp0] = pd0; }
        if (pp1 >= 0) { a.out_idx[pp1] = pid1; a.out_dist[pp1] = pd1; }
    }
}

__global__ void __launch_bounds__(1024) rows_lsort_block(PassArgs a) {
    extern __shared__ unsigned long long lbuf[];
    for (int64_t sp = blockIdx.x; sp < a.m; sp += gridDim.x) {
        const int cnt = a.lcnt[sp];
        if (cnt <= kLWarp || cnt > kLBlock) continue;
        const int64_t o0 = a.soff ? a.soff[sp] : (int64_t)a.lpos[sp] - cnt;
        const int64_t dst = a.soff ? a.offsets[a.qperm[sp]] : (a.loff ? row_base(a, sp) : o0);
        int S = 1024;
        while (S < cnt) S <<= 1;
        for (int i = threadIdx.x; i < S; i += blockDim.x) lbuf[i] = i < cnt ? a.tmpL[o0 + i] : ~0ull;
        __syncthreads();
        for (int k = 2; k <= S; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int t = threadIdx.x; t < S / 2; t += blockDim.x) {   // one compare-exchange pair per thread
                    const int i = 2 * t - (t & (j - 1)), p = i + j;
                    const unsigned long long x = lbuf[i], y = lbuf[p];
                    if ((x > y) == ((i & k) == 0)) { lbuf[i] = y; lbuf[p] = x; }
                }
                __syncthreads();
            }
        }
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) lemit(a, lbuf[i], dst + i);
        __syncthreads();
    }
}

template <typename K>
int persistent_grid(K kernel, int threads, size_t smem, int64_t items, int sm_count) {
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    if (occ < 1) occ = 1;
    int64_t g = (int64_t)sm_count * occ;
    if (items < g) g = items;
    return (int)(g < 1 ? 1 : g);
}

template <typename T, int D, int MODE>
void run_lowd(const PassArgs &a, cudaStream_t s) {
    // G == 3 (expanded-form filter, option simt_filter) stages only the filter rows
    const bool exp = sizeof(T) == 4 && MODE != M_FIX && a.Xf != nullptr &&
                     (size_t)2 * a.chunk * (D + 1) * 4 + 16 <= 200 * 1024;
    const size_t smem = (size_t)2 * a.chunk * (exp ? (D + 1) * 4 : D * sizeof(T)) + 16;
    constexpr bool SYMOK = MODE == M_SCAN || MODE == M_FIX;   // symmetric self-query variants
    auto k = exp ? window_lowd<T, D, MODE, 3>
                 : (a.variant == 1 ? window_lowd<T, D, MODE, 1> : window_lowd<T, D, MODE, 2>);
    if (SYMOK && a.sym) k = exp ? window_lowd<T, D, MODE, 3, SYMOK> : window_lowd<T, D, MODE, 1, SYMOK>;
    if constexpr (MODE == M_SCAN && sizeof(T) == 4) {
        if (exp && a.scan2q && a.B == 256) {   // two queries per thread (128-thread CTAs)
            auto k2 = a.sym ? window_lowd_2q<D, true> : window_lowd_2q<D, false>;
            cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            const int g2 = persistent_grid(k2, 128, smem, a.total_items, a.sm_count);
            SNN_LAUNCH(k2, g2, 128, smem, s, a);
            return;
        }
    }
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t work = MODE == M_FIX ? a.n_ovf : a.total_items;
    int g = persistent_grid(k, a.B, smem, work, a.sm_count);
    SNN_LAUNCH(k, g, a.B, smem, s, a);
}

template <typename T>
void run_generic(bool write, const PassArgs &a, cudaStream_t s) {
    if (write) {
        auto k = window_generic<T, true>;
        int g = persistent_grid(k, 256, 0, a.total_items, a.sm_count);
        SNN_LAUNCH(k, g, 256, 0, s, a);
    } else {
        auto k = window_generic<T, false>;
        int g = persistent_grid(k, 256, 0, a.total_items, a.sm_count);
        SNN_LAUNCH(k, g, 256, 0, s, a);
    }
}

}  // namespace

bool lowd_supported(int d) { return d >= 1 && d <= 8; }

namespace {
// multi-GPU query sharding: work of a query block = its window length
__global__ void part_len_kernel(const int64_t *lo, const int64_t *hi, int64_t nb, int64_t *len) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
        len[b] = hi[b] - lo[b];
}
// block b belongs to the part whose share of the total work contains the block's midpoint
// (contiguous, work-balanced ranges of key-sorted query blocks); other blocks get an empty
// window, so every path (low d, generic, tensor core) skips them and their rows are empty
__device__ __forceinline__ int part_owner(const int64_t *lo, const int64_t *hi, const int64_t *pre, int64_t nb,
                                          int64_t b, int nparts) {
    const double total = (double)pre[nb];
    int owner;
    if (total > 0) owner = (int)(((double)pre[b] + 0.5 * (double)(hi[b] - lo[b])) / total * nparts);
    else owner = (int)(b * nparts / nb);
    return owner >= nparts ? nparts - 1 : owner;
}
__global__ void restrict_part_kernel(int64_t *lo, int64_t *hi, int64_t *nitems, const int64_t *pre, int64_t nb,
                                     int part, int nparts) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        const int owner = part_owner(lo, hi, pre, nb, b, nparts);
        if (owner != part) {
            hi[b] = lo[b];
            if (nitems) nitems[b] = 0;
        }
    }
}
}  // namespace

// Symmetric self-query split (each unordered pair once): part p owns the
// rows of its blocks [b0, b1) (key positions [b0 B, b1 B)).  Its own blocks scan their
// windows as usual (pairs j > i); blocks before b0 whose windows reach b0 B are GHOST
// blocks, clipped to candidates j >= b0 B: their hits only supply the mirrored L entries of
// this part's rows (the owning part of those queries evaluates the same pairs for its U
// rows).  own[0..1] = the part's row range in key positions.
__global__ void part_range_kernel(const int64_t *lo, const int64_t *hi, const int64_t *pre, int64_t nb, int part,
                                  int nparts, unsigned long long *own_blocks) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
        if (part_owner(lo, hi, pre, nb, b, nparts) == part) {
            atomicMin(&own_blocks[0], (unsigned long long)b);
            atomicMax(&own_blocks[1], (unsigned long long)(b + 1));
        }
}
__global__ void part_range_init_kernel(unsigned long long *own_blocks, int64_t nb) {
    own_blocks[0] = (unsigned long long)nb;
    own_blocks[1] = 0ull;
}
__global__ void restrict_part_sym_kernel(int64_t *lo, int64_t *hi, int64_t *nitems, int64_t nb, int B, int64_t m,
                                         const unsigned long long *own_blocks, int64_t *own) {
    const int64_t b0 = (int64_t)own_blocks[0], b1 = (int64_t)own_blocks[1];
    const int64_t p0 = b0 * B;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        if (b >= b0 && b < b1) continue;                         // own block
        if (b < b0 && hi[b] > p0) lo[b] = lo[b] > p0 ? lo[b] : p0;   // ghost block (p0 is 4-aligned)
        else hi[b] = lo[b];                                      // another part's block
        if (nitems) nitems[b] = 0;                               // recomputed by the j > i clip
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        own[0] = b1 > b0 ? p0 : 0;
        own[1] = b1 > b0 ? min(b1 * (int64_t)B, m) : 0;
    }
}

void launch_restrict_part_sym(int64_t *blk_lo, int64_t *blk_hi, int64_t *nitems, int64_t nblocks, int B, int64_t m,
                              int part, int nparts, int64_t *tmp, void *scan_tmp, int64_t *own, cudaStream_t s) {
    if (nblocks == 0 || nparts <= 1) return;
    int64_t g = ceil_div(nblocks, 256);
    if (g > 148 * 16) g = 148 * 16;
    unsigned long long *ob = reinterpret_cast<unsigned long long *>(tmp + 2 * nblocks + 1);
    SNN_LAUNCH(part_range_init_kernel, 1, 1, 0, s, ob, nblocks);
    SNN_LAUNCH(part_len_kernel, (int)g, 256, 0, s, blk_lo, blk_hi, nblocks, tmp);
    exclusive_scan_i64(tmp, tmp + nblocks, nblocks, scan_tmp, s);
    SNN_LAUNCH(part_range_kernel, (int)g, 256, 0, s, blk_lo, blk_hi, tmp + nblocks, nblocks, part, nparts, ob);
    SNN_LAUNCH(restrict_part_sym_kernel, (int)g, 256, 0, s, blk_lo, blk_hi, nitems, nblocks, B, m, ob, own);
}

void launch_restrict_part(int64_t *blk_lo, int64_t *blk_hi, int64_t *nitems, int64_t nblocks, int part, int nparts,
                          int64_t *tmp, void *scan_tmp, cudaStream_t s) {
    if (nblocks == 0 || nparts <= 1) return;
    int64_t g = ceil_div(nblocks, 256);
    if (g > 148 * 16) g = 148 * 16;
    SNN_LAUNCH(part_len_kernel, (int)g, 256, 0, s, blk_lo, blk_hi, nblocks, tmp);
    exclusive_scan_i64(tmp, tmp + nblocks, nblocks, scan_tmp, s);
    SNN_LAUNCH(restrict_part_kernel, (int)g, 256, 0, s, blk_lo, blk_hi, nitems, tmp + nblocks, nblocks, part, nparts);
}

namespace {
__global__ void item_blocks_kernel(const int64_t *item_start, int64_t nblocks, int32_t *item_block) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += (int64_t)gridDim.x * blockDim.x)
        for (int64_t it = item_start[b]; it < item_start[b + 1]; ++it) item_block[it] = (int32_t)b;
}
}  // namespace

void launch_item_blocks(const int64_t *item_start, int64_t nblocks, int32_t *item_block, cudaStream_t s) {
    if (nblocks == 0) return;
    int64_t g = ceil_div(nblocks, 256);
    if (g > 148 * 16) g = 148 * 16;
    SNN_LAUNCH(item_blocks_kernel, (int)g, 256, 0, s, item_start, nblocks, item_block);
}

void launch_block_windows(const WindowSpec &w, cudaStream_t s) {
    const int64_t nb = ceil_div(w.m, w.B);
    if (nb == 0) return;
    SNN_LAUNCH(block_windows, (int)ceil_div(nb, 256), 256, 0, s, w);
}

#define SNN_LOWD_DISPATCH(FN)                                                          \
    switch (a.d) {                                                                     \
        case 1: if (a.f64) FN(double, 1); else FN(float, 1); return;                   \
        case 2: if (a.f64) FN(double, 2); else FN(float, 2); return;                   \
        case 3: if (a.f64) FN(double, 3); else FN(float, 3); return;                   \
        case 4: if (a.f64) FN(double, 4); else FN(float, 4); return;                   \
        case 5: if (a.f64) FN(double, 5); else FN(float, 5); return;                   \
        case 6: if (a.f64) FN(double, 6); else FN(float, 6); return;                   \
        case 7: if (a.f64) FN(double, 7); else FN(float, 7); return;                   \
        case 8: if (a.f64) FN(double, 8); else FN(float, 8); return;                   \
        default: return;                                                               \
    }

void launch_lowd_scan(const PassArgs &a, cudaStream_t s) {
    if (a.total_items == 0) return;
#define FN(T, D) run_lowd<T, D, 0>(a, s)
    SNN_LOWD_DISPATCH(FN)
#undef FN
}

void launch_lowd_fix(const PassArgs &a, cudaStream_t s) {
    if (a.n_ovf == 0) return;
#define FN(T, D) run_lowd<T, D, 1>(a, s)
    SNN_LOWD_DISPATCH(FN)
#undef FN
}

void launch_lowd_mode(int mode, const PassArgs &a, cudaStream_t s) {
    if (a.total_items == 0) return;
    switch (mode) {
#define FN(T, D) run_lowd<T, D, M_COUNT>(a, s)
        case M_COUNT: SNN_LOWD_DISPATCH(FN) break;
#undef FN
#define FN(T, D) run_lowd<T, D, M_UNION>(a, s)
        case M_UNION: SNN_LOWD_DISPATCH(FN) break;
#undef FN
#define FN(T, D) run_lowd<T, D, M_BORDER>(a, s)
        case M_BORDER: SNN_LOWD_DISPATCH(FN) break;
#undef FN
        default: break;
    }
}

void launch_lowd_compact(const PassArgs &a, cudaStream_t s) {
    if (a.total_items == 0) return;
    const int g = (int)(a.total_items < 148 * 32 ? a.total_items : 148 * 32);
    const int64_t n_rec = a.n_ovf_rec < a.ovf_rec_cap ? a.n_ovf_rec : a.ovf_rec_cap;
    const int go = (int)(ceil_div(n_rec, 256) < 148 * 8 ? ceil_div(n_rec, 256) : 148 * 8);
#define FN(T, D)                                                                         \
    do {                                                                                 \
        if (a.nrec && a.B == 256) SNN_LAUNCH((compact_lowd_bal<T, D>), g, 256, 0, s, a); \
        else SNN_LAUNCH((compact_lowd<T, D>), g, a.B, 0, s, a);                          \
        if (n_rec > 0) SNN_LAUNCH((compact_overflow<T, D>), go, 256, 0, s, a, n_rec);    \
    } while (0)
    SNN_LOWD_DISPATCH(FN)
#undef FN
}

void launch_generic_pass(bool write, const PassArgs &a, cudaStream_t s) {
    if (a.total_items == 0) return;
    if (a.f64) run_generic<double>(write, a, s); else run_generic<float>(write, a, s);
}

void launch_row_totals_sym(const int32_t *cnt, int32_t *pre, const int64_t *item_start, int64_t m, int B,
                           const int32_t *qperm, const int32_t *lcnt, int32_t *row_count, int32_t *maxl,
                           int32_t *srow, int64_t own_lo, int64_t own_hi, cudaStream_t s) {
    if (m == 0) return;
    SNN_LAUNCH(row_totals_sym, (int)ceil_div(m, 256), 256, 0, s, cnt, pre, item_start, m, B, qperm, lcnt, row_count,
               maxl, srow, own_lo, own_hi);
}

__global__ void sym_lpos_init(PassArgs a) {
    for (int64_t sp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; sp < a.m; sp += (int64_t)gridDim.x * blockDim.x)
        a.lpos[sp] = (unsigned long long)(a.loff ? a.loff[sp] : row_base(a, sp));
}

void launch_sym_lpos_init(const PassArgs &a, cudaStream_t s) {
    if (a.m == 0) return;
    int64_t g = ceil_div(a.m, 256);
    if (g > 148 * 16) g = 148 * 16;
    SNN_LAUNCH(sym_lpos_init, (int)g, 256, 0, s, a);
}

__global__ void invert_perm_kernel(const int32_t *perm, int64_t m, int32_t *inv) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        inv[perm[i]] = (int32_t)i;
}

void launch_invert_perm(const int32_t *perm, int64_t m, int32_t *inv, cudaStream_t s) {
    if (m == 0) return;
    int64_t g = ceil_div(m, 256);
    if (g > 148 * 16) g = 148 * 16;
    SNN_LAUNCH(invert_perm_kernel, (int)g, 256, 0, s, perm, m, inv);
}

void launch_rows_finalize(const PassArgs &a, int32_t max_l, cudaStream_t s) {
    if (a.m == 0 || (!a.sym && !a.soff)) return;
    int64_t g = ceil_div(a.m * 32, 256);
    if (g > 148 * 16) g = 148 * 16;
    if (a.sym && !a.soff && a.fpipe) {   // direct rows: 32 rows per warp, pipelined
        g = ceil_div(a.m, 256);   // 8 warps x 32 rows per CTA
        if (g > 148 * 8) g = 148 * 8;
        SNN_LAUNCH(rows_finalize_pipe, (int)g, 256, 0, s, a);
    } else {
        SNN_LAUNCH(rows_finalize_warp, (int)g, 256, 0, s, a);
    }
    if (!a.sym || max_l <= kLWarp) return;
    const size_t smem = (size_t)kLBlock * 8;
    cudaFuncSetAttribute(rows_lsort_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    SNN_LAUNCH(rows_lsort_block, 148 * 2, 1024, smem, s, a);
}

void launch_row_totals(const int32_t *cnt, int32_t *pre, const int64_t *item_start, int64_t m,
                       int B, const int32_t *qperm, int32_t *row_count, int32_t *srow, cudaStream_t s) {
    if (m == 0) return;
    SNN_LAUNCH(row_totals, (int)ceil_div(m, 256), 256, 0, s, cnt, pre, item_start, m, B, qperm, row_count, srow);
}

namespace {
// Expanded-form filter rows (G == 3 scan variant): AoSoA4 with D+1 floats per row,
// x_c = fl32(x - mu_f) and xbar' = fl32(c1h * 0.5 * ||x_c||^2) (fp64 sum); padding rows
// [n, n_pad) get x_c = 0, xbar' = +inf (never candidates).
template <int D>
__global__ void __launch_bounds__(256) filter_rows_kernel(const float *__restrict__ Xs, int64_t n, int64_t n_pad,
                                                          const float *__restrict__ mu_f, double c1h, float *Xf) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += (int64_t)gridDim.x * blockDim.x) {
        float c[D];
        double hb = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            c[k] = i < n ? (float)((double)Xs[(i >> 2) * 4 * D + 4 * k + (i & 3)] - (double)mu_f[k]) : 0.f;
            hb += (double)c[k] * (double)c[k];
        }
        float *o = Xf + (i >> 2) * 4 * (D + 1) + (i & 3);
#pragma unroll
        for (int k = 0; k < D; ++k) o[4 * k] = c[k];
        o[4 * D] = i < n ? (float)(0.5 * hb * c1h) : INFINITY;
    }
}
}  // namespace

void launch_filter_rows(const float *Xs, int d, int64_t n, int64_t n_pad, const float *mu_f, double c1h, float *Xf,
                        cudaStream_t s) {
    int64_t g = ceil_div(n_pad, 256);
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
#define CASE(D) case D: SNN_LAUNCH(filter_rows_kernel<D>, (int)g, 256, 0, s, Xs, n, n_pad, mu_f, c1h, Xf); break;
    switch (d) { CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) default: break; }
#undef CASE
}

void simt_filter_consts(int d, double R, double *c1h, double *r2h) {
    // |acc - (xbar c1h - x.q)| <= (c1/2)(xbar + qbar) + c0/2 for acc = fl(xbar' - sum x_c q_c)
    // (FFMA chain): xbar' rounding 3u, centring of x and q 2u, chain d * 2.02 u, qbar 2.02 u
    const double u = ldexp(1.0, -24);
    const double c1 = 2.0 * 1.05 * u * (3.0 + 2.01 + 2.02 * d + 2.02);
    const double c0 = 2.0 * 1.05 * (2.0 * d + 6.0) * ldexp(1.0, -149);
    *c1h = 1.0 - c1 / 2;
    *r2h = (R * R * (1.0 + 1e-12) * (1.0 + ldexp(1.0, -20)) + c0) / 2;
}

namespace {
// DBSCAN union pass: only pairs j > i are united, so block b's window starts at its own
// first position (rounded down to 4).
__global__ void truncate_windows_kernel(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int B,
                                        int chunk, int64_t *lo2, int64_t *nitems2, int64_t m, int64_t n,
                                        unsigned long long *pairs) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblocks) return;
    const int64_t lo = max(blk_lo[b], (b * B) & ~(int64_t)3), hi = blk_hi[b];
    lo2[b] = lo;
    nitems2[b] = hi > lo ? ceil_div(hi - lo, chunk) : 0;
    const int64_t vh = min(hi, n), nq = min((int64_t)B, m - b * B);   // candidate pairs evaluated
    if (pairs && vh > lo && nq > 0) atomicAdd(pairs, (unsigned long long)((vh - lo) * nq));
}
}  // namespace

namespace {
// DBSCAN union pass, candidates behind: block b's window ends after its own last position
// (rounded up to 4; pairs j < i only)
__global__ void truncate_windows_behind_kernel(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int B,
                                               int chunk, int64_t *hi2, int64_t *nitems2, int64_t m, int64_t n,
                                               unsigned long long *pairs) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblocks) return;
    const int64_t last = min(m, (b + 1) * B);   // one past the block's last position
    const int64_t lo = blk_lo[b], hi = min(blk_hi[b], round_up(last, 4));
    hi2[b] = hi;
    nitems2[b] = hi > lo ? ceil_div(hi - lo, chunk) : 0;
    const int64_t vh = min(hi, n), nq = min((int64_t)B, m - b * B);
    if (pairs && vh > lo && nq > 0) atomicAdd(pairs, (unsigned long long)((vh - lo) * nq));
}
}  // namespace

void launch_truncate_windows_behind(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int B, int chunk,
                                    int64_t *hi2, int64_t *nitems2, int64_t m, int64_t n, unsigned long long *pairs,
                                    cudaStream_t s) {
    if (nblocks == 0) return;
    SNN_LAUNCH(truncate_windows_behind_kernel, (int)ceil_div(nblocks, 256), 256, 0, s, blk_lo, blk_hi, nblocks, B,
               chunk, hi2, nitems2, m, n, pairs);
}

void launch_truncate_windows(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int B, int chunk,
                             int64_t *lo2, int64_t *nitems2, int64_t m, int64_t n, unsigned long long *pairs,
                             cudaStream_t s) {
    if (nblocks == 0) return;
    SNN_LAUNCH(truncate_windows_kernel, (int)ceil_div(nblocks, 256), 256, 0, s, blk_lo, blk_hi, nblocks, B, chunk,
               lo2, nitems2, m, n, pairs);
}

namespace {
// DBSCAN core flags need |N_eps(i)| only up to min_pts.  One CTA per query block walks
// the block's candidate chunks in order (TMA double buffer) and stops as soon as every
// query of the block has min_pts hits (config 5: the first chunk usually suffices);
// same exact classification as the radius query.  count = min(|N_eps|, >= min_pts).
template <typename T, int D>
__global__ void __launch_bounds__(256) core_count_kernel(PassArgs a, int32_t *count, unsigned long long *evaluated) {
    extern __shared__ __align__(128) uint8_t smem[];
    // the block's still-undecided queries, packed into the lowest threads after every chunk
    // (so warps whose queries all reached min_pts stop working, not just idle lanes)
    __shared__ T s_q[256 * D];
    __shared__ int32_t s_c[256];
    __shared__ int16_t s_id[256];
    __shared__ int32_t s_wsum[8];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const T *Xs = static_cast<const T *>(a.Xs);
    const size_t buf_bytes = (size_t)a.chunk * D * sizeof(T);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 2 * buf_bytes);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t item, int sidx) {
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const uint32_t bytes = (uint32_t)((c1 - c0) * D * sizeof(T));
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bar[sidx], bytes);
        bulk_g2s(smem + sidx * buf_bytes, Xs + c0 * D, bytes, &bar[sidx]);
    };
    uint32_t phase[2] = {0u, 0u};
    const float T_in = a.T_in, T_out = a.T_out;
    const double R2 = a.R2;
    const int32_t mp = a.min_pts;
    unsigned long long ev = 0;   // candidate pairs this thread evaluated (roofline accounting)
    for (int64_t b = blockIdx.x; b < a.nblocks; b += gridDim.x) {
        const int64_t sp0 = b * a.B;
        const int nqb = (int)min((int64_t)a.B, a.m - sp0);
        if (tid < nqb) {
            const int64_t sp = sp0 + tid;
            s_id[tid] = (int16_t)tid;
            s_c[tid] = 0;
#pragma unroll
            for (int k = 0; k < D; ++k) s_q[tid * D + k] = Xs[(sp >> 2) * 4 * D + k * 4 + (sp & 3)];
        }
        int n_und = nqb;
        const int64_t i0 = a.item_start[b], i1 = a.item_start[b + 1];
        // visit the block's own chunk first, then alternate outwards: the nearest keys
        // decide most points within the first chunks (early exit below)
        const int64_t nit = i1 - i0;
        const int64_t kd = nit > 0 ? min(max((sp0 - a.blk_lo[b]) / a.chunk, (int64_t)0), nit - 1) : 0;
        const int64_t up = nit - 1 - kd, mn = min(up, kd);
        auto order = [&](int64_t k) -> int64_t {
            if (k <= 2 * mn) return i0 + kd + ((k & 1) ? (k + 1) / 2 : -(k / 2));
            const int64_t r = k - 2 * mn;
            return i0 + (up > kd ? kd + mn + r : kd - mn - r);
        };
        __syncthreads();
        if (tid == 0 && nit > 0) issue(order(0), 0);
        for (int64_t k = 0; k < nit; ++k) {
            const int64_t item = order(k);
            const int sidx = (int)(k & 1);
            if (tid == 0 && k + 1 < nit) issue(order(k + 1), sidx ^ 1);
            int64_t bb, c0, c1;
            locate(a, item, bb, c0, c1);
            const bool mine = tid < n_und;
            T q[D];
            int32_t c = 0;
            int16_t id = 0;
            if (mine) {
                id = s_id[tid];
                c = s_c[tid];
#pragma unroll
                for (int kk = 0; kk < D; ++kk) q[kk] = s_q[tid * D + kk];
            }
            mbar_wait(&bar[sidx], phase[sidx]);
            phase[sidx] ^= 1u;
            if (mine) {
                const int ngroups = (int)((c1 - c0) >> 2);
                if constexpr (sizeof(T) == 4) {
                    const float4 *g4 = reinterpret_cast<const float4 *>(smem + sidx * buf_bytes);
                    uint64_t nq[D];
#pragma unroll
                    for (int kk = 0; kk < D; ++kk) nq[kk] = f2pack(-q[kk], -q[kk]);
                    int g = 0;
                    for (; g < ngroups && c < mp; ++g) {
                        float4 xa[D];
#pragma unroll
                        for (int kk = 0; kk < D; ++kk) xa[kk] = g4[g * D + kk];
                        uint64_t la, ha;
                        group_d2<D>(xa, nq, la, ha);
                        const float2 pa = f2unpack(la), qa = f2unpack(ha);
                        if (fminf(fminf(pa.x, pa.y), fminf(qa.x, qa.y)) <= T_out) {
                            uint32_t ia = mask4(pa.x, pa.y, qa.x, qa.y, T_in);
                            const uint32_t oa = mask4(pa.x, pa.y, qa.x, qa.y, T_out);
                            if (ia ^ oa) ia |= resolve4<D>(oa & ~ia, xa, q, R2);
                            c += __popc(ia);
                        }
                    }
                    ev += 4ull * g;
                } else {
                    const T *gb = reinterpret_cast<const T *>(smem + sidx * buf_bytes);
                    int g = 0;
                    for (; g < ngroups && c < mp; ++g) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            double s2 = 0.0;
#pragma unroll
                            for (int kk = 0; kk < D; ++kk) {
                                const double t = __dsub_rn(gb[g * 4 * D + kk * 4 + i], q[kk]);
                                s2 = __dadd_rn(s2, __dmul_rn(t, t));
                            }
                            c += s2 <= R2;
                        }
                    }
                    ev += 4ull * g;
                }
            }
            // decided queries write their count; the undecided ones are packed to the front
            const bool und = mine && c < mp;
            if (mine && !und) count[sp0 + id] = c;
            const unsigned bal = __ballot_sync(0xffffffffu, und);
            if (lane == 0) s_wsum[wid] = __popc(bal);
            __syncthreads();   // also: every thread has read its old list entry
            int pos = __popc(bal & ((1u << lane) - 1)), total = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const int v = s_wsum[w];
                pos += w < wid ? v : 0;
                total += v;
            }
            if (und) {
                s_id[pos] = id;
                s_c[pos] = c;
#pragma unroll
                for (int kk = 0; kk < D; ++kk) s_q[pos * D + kk] = q[kk];
            }
            n_und = total;
            __syncthreads();
            if (n_und == 0) {                 // every query of the block is decided
                if (k + 1 < nit) {            // drain the prefetched chunk
                    const int ns = sidx ^ 1;
                    mbar_wait(&bar[ns], phase[ns]);
                    phase[ns] ^= 1u;
                }
                break;
            }
        }
        if (tid < n_und) count[sp0 + s_id[tid]] = s_c[tid];   // never reached min_pts
        __syncthreads();
    }
    if (evaluated) {
        ev = warp_sum(ev);
        if ((threadIdx.x & 31) == 0 && ev) atomicAdd(evaluated, ev);
    }
}

// DBSCAN core counts, one warp per point: the warp scans its block's window OUTWARD from
// the point's own sorted position (the nearest keys first), 32 candidates on each side per
// step, and stops as soon as min_pts neighbours (self included) are found -- warp-uniform
// early exit, no per-lane divergence and no CTA barrier (core_count_kernel's per-chunk
// barrier held 77% of its stall samples on config 5).  Same exact classification (rigorous
// fp32 direct-form thresholds, oracle-order fp64 in between).  count = |N_eps| if below
// min_pts, else some value >= min_pts.
template <typename T, int D>
__global__ void __launch_bounds__(256) core_count_warp_kernel(PassArgs a, int32_t *count,
                                                              unsigned long long *evaluated) {
    const T *Xs = static_cast<const T *>(a.Xs);
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const float T_in = a.T_in, T_out = a.T_out;
    const double R2 = a.R2;
    const int32_t mp = a.min_pts;
    unsigned long long ev = 0;
    auto row = [&](int64_t j, T (&x)[D]) {
#pragma unroll
        for (int k = 0; k < D; ++k) x[k] = Xs[(j >> 2) * 4 * D + k * 4 + (j & 3)];
    };
    auto hit = [&](const T (&x)[D], const T (&q)[D]) -> bool {
        if constexpr (sizeof(T) == 4) {
            float d2 = 0.f;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const float t = x[k] - q[k];
                d2 = fmaf(t, t, d2);
            }
            if (d2 <= T_in) return true;
            if (d2 > T_out) return false;
        }
        return sqdist_exact(x, q, D) <= R2;
    };
    for (int64_t sp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sp < a.m; sp += nw) {
        const int64_t b = sp / a.B;
        const int64_t lo = a.blk_lo[b], hi = min(a.blk_hi[b], a.n_index);
        T q[D];
        row(sp, q);
        int32_t c = 1;   // the point itself
        for (int64_t off = 1;; off += 32) {
            const int64_t jr = sp + off + lane, jl = sp - off - lane;
            const bool vr = jr < hi, vl = jl >= lo;
            if (!__any_sync(0xffffffffu, vr || vl)) break;
            int h = 0;
            if (vr) { T x[D]; row(jr, x); h += hit(x, q); }
            if (vl) { T x[D]; row(jl, x); h += hit(x, q); }
            ev += (unsigned long long)(vr + vl);
            c += __reduce_add_sync(0xffffffffu, h);
            if (c >= mp) break;
        }
        if (lane == 0) count[sp] = c;
    }
    if (evaluated) {
        ev = warp_sum(ev);
        if (lane == 0 && ev) atomicAdd(evaluated, ev);
    }
}

// DBSCAN union seed (before the union pass): one warp per core point scans behind its own
// key position (pairs j < i, the nearest positions first, 32 per step) and unites it with
// the first core neighbour found within max_steps x 32 positions (same exact test as the counts).  The seeded forest joins
// most points to their component before the union pass, whose work items of one query block
// then start from settled roots instead of singletons.  Stops at the block's window start.
template <typename T, int D>
__global__ void __launch_bounds__(256) union_seed_kernel(PassArgs a, int max_steps) {
    const T *Xs = static_cast<const T *>(a.Xs);
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const float T_in = a.T_in, T_out = a.T_out;
    const double R2 = a.R2;
    auto row = [&](int64_t j, T (&x)[D]) {
#pragma unroll
        for (int k = 0; k < D; ++k) x[k] = Xs[(j >> 2) * 4 * D + k * 4 + (j & 3)];
    };
    for (int64_t sp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sp < a.m; sp += nw) {
        if (!a.core[sp]) continue;   // warp-uniform
        const int64_t lo = a.blk_lo[sp / a.B];
        T q[D];
        row(sp, q);
        for (int64_t off = 1; off <= 32 * max_steps; off += 32) {
            const int64_t j = sp - off - lane;
            if (!__any_sync(0xffffffffu, j >= lo)) break;
            bool h = false;
            if (j >= lo && a.core[j]) {
                T x[D];
                row(j, x);
                if constexpr (sizeof(T) == 4) {
                    float d2 = 0.f;
#pragma unroll
                    for (int k = 0; k < D; ++k) {
                        const float t = x[k] - q[k];
                        d2 = fmaf(t, t, d2);
                    }
                    h = d2 <= T_in || (d2 <= T_out && sqdist_exact(x, q, D) <= R2);
                } else {
                    h = sqdist_exact(x, q, D) <= R2;
                }
            }
            const uint32_t hb = __ballot_sync(0xffffffffu, h);
            if (hb) {
                if (lane == __ffs(hb) - 1) uf_unite(a.parent, (int32_t)sp, (int32_t)j);
                break;
            }
        }
    }
}

template <typename T, int D>
void run_core_count(const PassArgs &a, int32_t *count, unsigned long long *evaluated, cudaStream_t s) {
    const size_t smem = (size_t)2 * a.chunk * D * sizeof(T) + 16;
    auto k = core_count_kernel<T, D>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int g = persistent_grid(k, a.B, smem, a.nblocks, a.sm_count);
    SNN_LAUNCH(k, g, a.B, smem, s, a, count, evaluated);
}
}  // namespace

void launch_union_seed(const PassArgs &a, int max_steps, cudaStream_t s) {
    if (a.nblocks == 0) return;
#define FN(T, D) SNN_LAUNCH((union_seed_kernel<T, D>), a.sm_count * 8, 256, 0, s, a, max_steps)
    SNN_LOWD_DISPATCH(FN)
#undef FN
}

void launch_core_counts(const PassArgs &a, int32_t *count, unsigned long long *evaluated, cudaStream_t s) {
    if (a.nblocks == 0) return;
    if (a.count_warp) {
#define FN(T, D) SNN_LAUNCH((core_count_warp_kernel<T, D>), a.sm_count * 8, 256, 0, s, a, count, evaluated)
        SNN_LOWD_DISPATCH(FN)
#undef FN
    }
#define FN(T, D) run_core_count<T, D>(a, count, evaluated, s)
    SNN_LOWD_DISPATCH(FN)
#undef FN
}

}  // namespace snn

namespace snn {
namespace {
// K12 union pass with a staged parent snapshot (fp32 AoSoA4 rows, d <= 8).  For every
// (query block, candidate chunk) item the TMA stages the chunk's rows AND its slice of
// the union-find parents parent[c0, c1) (sorted positions, so the slice is contiguous).
// The staged parents are turned into the candidates' current roots (one find each,
// compressing parent[j] to the root in global memory), and a candidate pair reaches the
// divergent union path only if it may be a neighbour (fp32 d^2 <= T_out) AND its staged
// root is a core point's root different from the query's cached root: any ancestor of j
// ever found stays an ancestor (links only merge components), so equality proves the
// pair already joined and the exact test is not needed.  The predicated pre-check runs warp-converged; the rare remaining pairs
// get the exact classification (same rigorous thresholds, oracle-order fp64 in between),
// a fresh parent[j] check and, if that differs too, the lock-free union; the root joined
// is written back into the snapshot.
// ustats (nullable): [0] pairs sent to the union path, [1] exact hits among them,
// [2] unions attempted (fresh parent differed from the cached root).
template <int D, int MINB, int DIAG = 0>
__global__ void __launch_bounds__(256, MINB) union_snap_kernel(PassArgs a, const int64_t *nit, int pass_k,
                                                              int behind, unsigned long long *ustats) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x;
    const float *Xs = static_cast<const float *>(a.Xs);
    const size_t rows_bytes = (size_t)a.chunk * D * 4;
    const size_t buf_bytes = rows_bytes + (size_t)a.chunk * 4;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 2 * buf_bytes);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t item, int sidx) {
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const uint32_t nb = (uint32_t)((c1 - c0) * D * 4), pb = (uint32_t)((c1 - c0) * 4);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bar[sidx], nb + pb);
        bulk_g2s(smem + sidx * buf_bytes, Xs + c0 * D, nb, &bar[sidx]);
        bulk_g2s(smem + sidx * buf_bytes + rows_bytes, a.parent + c0, pb, &bar[sidx]);
    };
    uint32_t phase[2] = {0u, 0u};
    unsigned long long st_path = 0, st_hit = 0, st_link = 0;
    // pass_k >= 0: chunk pass_k of every query block (work index = block); else every item
    const int64_t n_work = pass_k >= 0 ? a.nblocks : a.total_items;
    auto item_of = [&](int64_t w) -> int64_t {
        if (pass_k < 0) return w;
        return nit[w] > pass_k ? a.item_start[w] + pass_k : -1;
    };
    int64_t w = blockIdx.x;
    if (tid == 0 && w < n_work && item_of(w) >= 0) issue(item_of(w), 0);
    const float T_in = a.T_in, T_out = a.T_out;
    const double R2 = a.R2;
    for (int it = 0; w < n_work; w += gridDim.x, ++it) {
        const int sidx = it & 1;
        const int64_t wn = w + gridDim.x;
        if (tid == 0 && wn < n_work && item_of(wn) >= 0) issue(item_of(wn), sidx ^ 1);
        const int64_t item = item_of(w);
        if (item < 0) continue;   // CTA-uniform: nothing staged for this work index
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const int64_t sp = b * a.B + tid;
        // pairs j > i only (candidates ahead), or j < i only (behind: windows end at the block)
        const bool active = sp < a.m && a.core[sp] && (behind ? c0 < sp : c1 - 1 > sp);
        int32_t uroot = active ? uf_rep(a.parent, (int32_t)sp) : -1;
        float q[D];
#pragma unroll
        for (int k = 0; k < D; ++k) q[k] = active ? Xs[(sp >> 2) * 4 * D + k * 4 + (sp & 3)] : NAN;   // NaN: no hits
        mbar_wait(&bar[sidx], phase[sidx]);
        phase[sidx] ^= 1u;
        int32_t *spar = reinterpret_cast<int32_t *>(smem + sidx * buf_bytes + rows_bytes);
        // staged parents -> current roots (path compressed in global memory too: writing an
        // ancestor into parent[j] of a non-root j is race-benign, links CAS only on roots)
        // Non-core candidates (parent -1) get NaN coordinates in the staged rows: no pair
        // with them passes the distance test, so the hot loop needs no core check.
        float *srows = reinterpret_cast<float *>(smem + sidx * buf_bytes);
        for (int t = tid; t < (int)(c1 - c0); t += blockDim.x) {
            const int32_t p = spar[t];
            if (p >= 0) {
                const int32_t r = DIAG == 1 ? p : uf_rep(a.parent, p);
                if (r != p) {
                    spar[t] = r;
                    a.parent[c0 + t] = r;
                }
            } else {
#pragma unroll
                for (int k = 0; k < D; ++k) srows[(t >> 2) * 4 * D + k * 4 + (t & 3)] = NAN;
            }
        }
        __syncthreads();
        if (__any_sync(0xffffffffu, active)) {
            uint64_t nq[D];
#pragma unroll
            for (int k = 0; k < D; ++k) nq[k] = f2pack(-q[k], -q[k]);
            const int ngroups = (int)((c1 - c0) >> 2);
            uint32_t ra = smem_u32(smem + sidx * buf_bytes);
            uint32_t pa = ra + (uint32_t)rows_bytes;
            // the few pairs the snapshot cannot settle: exact test, then the fresh parent[j]
            // (one relaxed load) against the cached root, union only if they differ; the
            // root joined is written back into the snapshot
            auto settle = [&](int g, const float4 (&xv)[D], const float2 dl, const float2 dh, uint32_t nb) {
                const float dv[4] = {dl.x, dl.y, dh.x, dh.y};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int64_t j = c0 + 4 * g + i;
                    if (!(nb & (1u << i)) || (behind ? j >= sp : j <= sp)) continue;
                    ++st_path;
                    bool hit = dv[i] <= T_in;
                    if (!hit) {
                        float x[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) x[k] = lane4(xv[k], i);
                        hit = sqdist_exact(x, q, D) <= R2;
                    }
                    if (!hit) continue;
                    ++st_hit;
                    const int32_t pj = ld_relaxed_gpu(a.parent + j);
                    if (pj != uroot) {
                        uroot = uf_unite_root(a.parent, uroot, pj);   // ancestors of sp and j
                        ++st_link;
                        // parent[j] -> the joined root (the smallest position of the component,
                        // so <= j; j is no root unless it is that root: race-benign)
                        if (uroot != pj) a.parent[j] = uroot;
                    }
                    spar[4 * g + i] = uroot;   // an ancestor of j now: a better filter for the CTA
                }
            };
            // need bits of one group: may be a neighbour (non-core rows are NaN) and the
            // staged root differs from the cached one
            auto need4 = [&](const float2 dl, const float2 dh, const float4 pf) -> uint32_t {
                return (uint32_t)(dl.x <= T_out && __float_as_int(pf.x) != uroot) |
                       ((uint32_t)(dl.y <= T_out && __float_as_int(pf.y) != uroot) << 1) |
                       ((uint32_t)(dh.x <= T_out && __float_as_int(pf.z) != uroot) << 2) |
                       ((uint32_t)(dh.y <= T_out && __float_as_int(pf.w) != uroot) << 3);
            };
            int g = 0;
            for (; g + 1 < ngroups; g += 2, ra += 32u * D, pa += 32u) {   // 2 groups per step
                float4 xa[D], xb[D];
#pragma unroll
                for (int k = 0; k < D; ++k) { xa[k] = lds128(ra + 16u * k); xb[k] = lds128(ra + 16u * (D + k)); }
                const float4 pfa = lds128(pa), pfb = lds128(pa + 16u);
                uint64_t la, ha, lb, hb;
                group_d2<D>(xa, nq, la, ha);
                group_d2<D>(xb, nq, lb, hb);
                const float2 dla = f2unpack(la), dha = f2unpack(ha), dlb = f2unpack(lb), dhb = f2unpack(hb);
                const uint32_t na = need4(dla, dha, pfa), nb = need4(dlb, dhb, pfb);
                if (DIAG) {   // diagnostics (labels invalid): count the pairs, skip the unions
                    st_hit += __popc(na) + __popc(nb);
                } else if (na | nb) {
                    if (na) settle(g, xa, dla, dha, na);
                    if (nb) settle(g + 1, xb, dlb, dhb, nb);
                }
            }
            if (g < ngroups) {
                float4 xa[D];
#pragma unroll
                for (int k = 0; k < D; ++k) xa[k] = lds128(ra + 16u * k);
                const float4 pfa = lds128(pa);
                uint64_t la, ha;
                group_d2<D>(xa, nq, la, ha);
                const float2 dla = f2unpack(la), dha = f2unpack(ha);
                const uint32_t na = need4(dla, dha, pfa);
                if (!DIAG && na) settle(g, xa, dla, dha, na);
            }
        }
        __syncthreads();
    }
    if (ustats) {
        if (DIAG) st_path = 1;
        st_path = warp_sum(st_path);
        st_hit = warp_sum(st_hit);
        st_link = warp_sum(st_link);
        if ((tid & 31) == 0 && st_path) {
            atomicAdd(&ustats[0], st_path);
            atomicAdd(&ustats[1], st_hit);
            atomicAdd(&ustats[2], st_link);
        }
    }
}
}  // namespace

bool launch_union_snap(const PassArgs &a, int variant, const int64_t *nit, int64_t phases, int behind,
                       unsigned long long *ustats, cudaStream_t s) {
    if (a.f64 || a.d < 1 || a.d > 8) return false;
    if (a.total_items == 0) return true;
    const size_t smem = (size_t)2 * a.chunk * (a.d + 1) * 4 + 16;
    switch (a.d) {
#define CASE(D)                                                                                    \
    case D: {                                                                                      \
        auto k = variant == 2 ? union_snap_kernel<D, 1> : variant == 3 ? union_snap_kernel<D, 4, 1>  \
               : variant == 4 ? union_snap_kernel<D, 4, 2> : union_snap_kernel<D, 4>;              \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);           \
        if (phases > 0 && nit) {                                                                   \
            const int g = persistent_grid(k, a.B, smem, a.nblocks, a.sm_count);                   \
            for (int64_t ph = 0; ph < phases; ++ph) SNN_LAUNCH(k, g, a.B, smem, s, a, nit, (int)ph, behind, ustats); \
        } else {                                                                                   \
            const int g = persistent_grid(k, a.B, smem, a.total_items, a.sm_count);               \
            SNN_LAUNCH(k, g, a.B, smem, s, a, nit, -1, behind, ustats);                            \
        }                                                                                          \
        break;                                                                                     \
    }
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
        default: break;
    }
    return true;
}

namespace {
__global__ void max_i64_kernel(const int64_t *v, int64_t n, unsigned long long *out) {
    int64_t m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, v[i]);
    m = max(m, (int64_t)__reduce_max_sync(0xffffffffu, (unsigned)m));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, (unsigned long long)m);
}
}  // namespace

void launch_max_i64(const int64_t *v, int64_t n, unsigned long long *out, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t gb = ceil_div(n, 256);
    const int g = (int)(gb < 148 * 4 ? gb : 148 * 4);
    SNN_LAUNCH(max_i64_kernel, g, 256, 0, s, v, n, out);
}

}  // namespace snn
