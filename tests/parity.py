"""Parity helpers: compare a GPU CSR result with the oracle's CSR.

Acceptance rule (BASELINE.json north_star): per query, the oracle's strict set
(s <= R^2 (1 - 1e-5)) must be contained in the GPU set, which must be contained in the
oracle's hits plus the tolerance band (R^2 < s <= R^2 (1 + 1e-5)); distances within 1e-5
relative.  The design target is stronger and is asserted too:
GPU set == oracle hits (s <= R*R) exactly and distance == float32(sqrt(s)) bit for bit.
"""
import numpy as np


def _pairs(offsets, indices):
    offsets = np.asarray(offsets, dtype=np.int64)
    m = len(offsets) - 1
    rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(offsets))
    return rows, np.asarray(indices, dtype=np.int64)


def compare(gpu, ora, rows_subset=None, exact=True):
    """gpu: CSR (host numpy) over all queries; ora: oracle.radius_query dict computed on
    queries ``rows_subset`` (or all queries if None).  Returns a stats dict; raises
    AssertionError on any violation."""
    g_off = np.asarray(gpu.offsets)
    g_idx = np.asarray(gpu.indices)
    g_dist = np.asarray(gpu.distances)
    if rows_subset is None:
        rows_subset = np.arange(len(g_off) - 1)
    rows_subset = np.asarray(rows_subset, dtype=np.int64)
    # GPU pairs restricted to the subset, re-indexed 0..k-1
    cnt = np.diff(g_off)[rows_subset]
    sel = np.concatenate([np.arange(g_off[r], g_off[r + 1]) for r in rows_subset]) \
        if len(rows_subset) else np.zeros(0, dtype=np.int64)
    sel = sel.astype(np.int64)
    g_rows = np.repeat(np.arange(len(rows_subset), dtype=np.int64), cnt)
    g_ids = g_idx[sel].astype(np.int64)
    g_d = g_dist[sel]
    o_rows, o_ids = _pairs(ora["offsets"], ora["indices"])
    s = np.asarray(ora["s"])
    R2 = ora["R2"]
    n_key = int(max(g_ids.max(initial=0), o_ids.max(initial=0))) + 1
    gk = g_rows * n_key + g_ids
    ok = o_rows * n_key + o_ids
    assert len(np.unique(gk)) == len(gk), "duplicate ids within a GPU row"
    strict = s <= R2 * (1 - 1e-5)
    hits = s <= R2
    # containment: strict subset of gpu; gpu subset of (hits or band) = all oracle pairs
    assert np.isin(ok[strict], gk).all(), "GPU missed a strict neighbour"
    in_ora = np.isin(gk, ok)
    assert in_ora.all(), f"GPU returned {int((~in_ora).sum())} pairs outside R(1+1e-5)"
    # distances for common pairs
    order_o = np.argsort(ok)
    pos = np.searchsorted(ok[order_o], gk)
    s_g = s[order_o][pos]
    d_ref = np.sqrt(s_g)
    rel = np.abs(g_d.astype(np.float64) - d_ref) / np.maximum(d_ref, 1e-300)
    assert np.all((rel <= 1e-5) | (d_ref == 0) & (g_d == 0)), "distance tolerance violated"
    stats = {"pairs": int(len(gk)), "oracle_hits": int(hits.sum()),
             "band": int((~strict).sum()), "max_rel_dist_err": float(rel.max(initial=0))}
    if exact:
        assert len(gk) == int(hits.sum()) and np.isin(ok[hits], gk).all(), \
            "membership is not bit-identical to the fp64 oracle"
        assert np.array_equal(g_d, np.sqrt(s_g).astype(np.float32)), \
            "distances not bit-identical to float32(sqrt(fp64 s))"
    return stats
