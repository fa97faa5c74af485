"""TEST INFRASTRUCTURE -- CPU fp64 oracle for the SNN hot path (arXiv 2212.07679).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_2212_07679_b200``) never imports it and shares no code with it.

Contents (each function cites the passage it follows):

* ``radius_query``      brute-force fixed-radius search = the problem's definition
                        (§3.2; exactness claim PAPER.md:31),
                        fp64 eq:ip1, in C (``snn_oracle.c``).
* ``radius_query(grid=True)``  the same result for d <= 3 from grid-pruned pairs (same
                        per-pair test; full-size parity digests of configs 2 and 5).
* ``dbscan``            DBSCAN with DESIGN.md reading C18: ascending-id
                        scan with FIFO expansion over brute-force neighbourhoods; ``grid=True``
                        computes the same labels by components for d <= 3.
* ``neighbour_counts``  eps-neighbourhood sizes of sampled points (DBSCAN's core test).
* ``column_mean``, ``center``, ``principal_direction``, ``scores``, ``sort_index``,
  ``half_norms``, ``build_index``   Algorithm 1 "SNN Index" step by
                        step in fp64 numpy, the SVD of eq:svd via LAPACK.
* ``candidate_range``, ``alg2_query``   Algorithm 2 "SNN Query", the
                        Cauchy-Schwarz window of eq:lower.
* ``normalize_rows``, ``metric_radius``, ``metric_distance``, ``metric_radius_query``,
  ``cosine_distance``, ``angular_distance``   cosine / angular distance through the
                        Euclidean search on normalized rows (DESIGN.md
                        reading C21); the direct definitions pin the reduction.
* ``manhattan_query``, ``inner_product_query``, ``mips_transform``   Manhattan radius
                        search and inner-product threshold search (MIPS
                        transform), brute force by definition (reading C22).

Parity pins live in ``tests/test_oracle.py`` (hand examples, closed forms, library
cross-checks, invariants).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "snn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
          "-std=c11", "-Wall"]

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle C library in-tree (gcc; no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        lib.oracle_radius_count.argtypes = [P, i64, P, i64, i32, f64, f64, P]
        lib.oracle_radius_count.restype = ctypes.c_int
        lib.oracle_radius_fill.argtypes = [P, i64, P, i64, i32, f64, f64, P, P, P]
        lib.oracle_radius_fill.restype = ctypes.c_int
        lib.oracle_dbscan.argtypes = [P, i64, i32, f64, i32, P, P]
        lib.oracle_dbscan.restype = ctypes.c_int64
        lib.oracle_neighbour_counts.argtypes = [P, i64, i32, f64, P, i64, P]
        lib.oracle_neighbour_counts.restype = ctypes.c_int
        lib.oracle_grid_radius_count.argtypes = [P, i64, P, i64, i32, f64, f64, P]
        lib.oracle_grid_radius_count.restype = ctypes.c_int
        lib.oracle_grid_radius_fill.argtypes = [P, i64, P, i64, i32, f64, f64, P, P, P]
        lib.oracle_grid_radius_fill.restype = ctypes.c_int
        lib.oracle_grid_dbscan.argtypes = [P, i64, i32, f64, i32, P, P]
        lib.oracle_grid_dbscan.restype = ctypes.c_int64
        lib.oracle_sqdist.argtypes = [P, P, i32]
        lib.oracle_sqdist.restype = ctypes.c_double
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(t: int) -> None:
    _load().oracle_set_num_threads(int(t))


def _f64(a) -> np.ndarray:
    """fp32 / fp64 inputs widened EXACTLY to fp64 (reading C5)."""
    a = np.asarray(a)
    if a.ndim == 1:
        a = a[:, None]
    return np.ascontiguousarray(a, dtype=np.float64)


def sqdist(p, q) -> float:
    """eq:ip1 for one pair, left to right, no FMA."""
    p, q = _f64(np.ravel(p))[:, 0], _f64(np.ravel(q))[:, 0]
    return float(_load().oracle_sqdist(p.ctypes.data, q.ctypes.data, int(p.shape[0])))


# ----------------------------------------------------------------- radius query
def radius_query(P, Q, R: float, band_rel: float = 1e-5, grid: bool = False) -> dict:
    """Brute force: all (j, i) with s(p_i, q_j) <= (R*R)(1+band_rel).

    ``grid=True`` (d <= 3 only) evaluates only the pairs in adjacent grid cells of side
    >= R(1+1e-6) (``oracle_grid_radius_*`` in ``snn_oracle.c``, with the argument why no hit
    is skipped); the per-pair test is the same, so the result is identical (pinned against
    the brute force in ``tests/test_oracle.py``).  Used for full-size d <= 3 parity.

    Returns CSR over queries (row j = query j, ids ascending): ``offsets`` (m+1 int64),
    ``indices`` (int32 original ids), ``s`` (fp64 squared distance), plus ``R2`` = R*R.
    Hits are ``s <= R2``; pairs with R2 < s <= R2(1+band_rel) form the
    tolerance band of BASELINE.json's acceptance rule.
    """
    if R < 0 or not np.isfinite(R):
        raise ValueError("negative or non-finite radius")
    P, Q = _f64(P), _f64(Q)
    n, d = P.shape
    m = Q.shape[0]
    if Q.shape[1] != d:
        raise ValueError("dimension mismatch")
    lib = _load()
    if grid and d > 3:
        raise ValueError("grid oracle is for d <= 3")
    count_fn = lib.oracle_grid_radius_count if grid else lib.oracle_radius_count
    fill_fn = lib.oracle_grid_radius_fill if grid else lib.oracle_radius_fill
    counts = np.zeros(m, dtype=np.int64)
    if count_fn(P.ctypes.data, n, Q.ctypes.data, m, d, float(R), float(band_rel), counts.ctypes.data):
        raise ValueError("oracle_radius_count failed")
    offsets = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    nnz = int(offsets[-1])
    idx = np.empty(max(nnz, 1), dtype=np.int32)
    s = np.empty(max(nnz, 1), dtype=np.float64)
    if fill_fn(P.ctypes.data, n, Q.ctypes.data, m, d, float(R), float(band_rel),
               offsets.ctypes.data, idx.ctypes.data, s.ctypes.data):
        raise ValueError("oracle_radius_fill failed")
    return {"offsets": offsets, "indices": idx[:nnz], "s": s[:nnz], "R2": float(R) * float(R)}


def neighbour_counts(P, eps: float, ids) -> np.ndarray:
    """|{j : s(p_j, p_i) <= eps^2}| (self included) for the sampled ids, one by one: the
    eps-neighbourhood size DBSCAN's core test uses (reading C18), eq:ip1
    in fp64 against every point."""
    P = _f64(P)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.zeros(ids.shape[0], dtype=np.int64)
    _load().oracle_neighbour_counts(P.ctypes.data, P.shape[0], P.shape[1], float(eps),
                                    ids.ctypes.data, ids.shape[0], out.ctypes.data)
    return out


def dbscan(P, eps: float, min_pts: int, grid: bool = False):
    """DBSCAN with DESIGN.md reading C18: the textbook scan in ascending
    id with FIFO expansion, brute-force neighbourhoods (``oracle_dbscan``).

    ``grid=True`` (d <= 3): the same labels computed as connected components of the core
    graph over grid-pruned pairs (``oracle_grid_dbscan``; border point -> smallest cluster
    number among its core neighbours = the first cluster the FIFO scan reaches it with);
    pinned against the brute force in ``tests/test_oracle.py``.  Used for full-size C5.

    Returns (labels int32[n], K, counts int64[n]).
    """
    P = _f64(P)
    n, d = P.shape
    if grid and d > 3:
        raise ValueError("grid oracle is for d <= 3")
    labels = np.empty(n, dtype=np.int32)
    counts = np.empty(n, dtype=np.int64)
    fn = _load().oracle_grid_dbscan if grid else _load().oracle_dbscan
    K = fn(P.ctypes.data, n, d, float(eps), int(min_pts), labels.ctypes.data, counts.ctypes.data)
    if K < 0:
        raise ValueError("oracle_dbscan failed")
    return labels, int(K), counts


# ----------------------------------------------------------------- Algorithm 1
def column_mean(P) -> np.ndarray:
    """Alg. 1 l.2: mu = mean({p_j}), fp64."""
    P = _f64(P)
    if P.shape[0] == 0:
        raise ValueError("empty dataset")
    return P.sum(axis=0) / P.shape[0]


def center(P, mu) -> np.ndarray:
    """Alg. 1 l.3: x_i = p_i - mu."""
    return _f64(P) - np.asarray(mu, dtype=np.float64)[None, :]


def principal_direction(Xc):
    """Alg. 1 l.4, eq:svd: thin SVD X = U S V^T, keep v1.

    Sign (reading C9): the entry of largest magnitude is made positive (ties:
    lowest index).  All-zero data: v1 = e_1, singular values 0.  Returns (v1, sigma).
    """
    Xc = _f64(Xc)
    n, d = Xc.shape
    if n == 0:
        raise ValueError("empty dataset")
    S = np.linalg.svd(Xc, compute_uv=False)
    if not np.any(S > 0):
        v1 = np.zeros(d)
        v1[0] = 1.0
        return v1, np.zeros(min(n, d))
    _, S, Vt = np.linalg.svd(Xc, full_matrices=False)
    v1 = Vt[0].copy()
    k = int(np.argmax(np.abs(v1)))
    if v1[k] < 0:
        v1 = -v1
    return v1, S


def scores(Xc, v1) -> np.ndarray:
    """Alg. 1 l.5: alpha_i = x_i^T v1."""
    return _f64(Xc) @ np.asarray(v1, dtype=np.float64)


def sort_index(alpha) -> np.ndarray:
    """Alg. 1 l.6: order by alpha; ties by original id (stable, reading C10)."""
    return np.argsort(np.asarray(alpha), kind="stable")


def half_norms(Xc) -> np.ndarray:
    """Alg. 1 l.7: xbar_i = (x_i^T x_i)/2."""
    Xc = _f64(Xc)
    return 0.5 * np.einsum("ij,ij->i", Xc, Xc)


def build_index(P) -> dict:
    """Algorithm 1, fp64. Returns mu, X (sorted, centered), v1,
    alpha (sorted), xbar, perm (pi: sorted position -> original id), sigma."""
    mu = column_mean(P)
    Xc = center(P, mu)
    v1, sigma = principal_direction(Xc)
    alpha = scores(Xc, v1)
    perm = sort_index(alpha)
    Xs = Xc[perm]
    return {"mu": mu, "X": Xs, "v1": v1, "alpha": alpha[perm], "xbar": half_norms(Xs),
            "perm": perm, "sigma": sigma}


# ----------------------------------------------------------------- Algorithm 2
def candidate_range(alpha_sorted, alpha_q: float, R: float):
    """Alg. 2 l.4: J = {j : |alpha_j - alpha_q| <= R}
    as the half-open sorted-position range [lo, hi) found by binary search."""
    if R < 0:
        raise ValueError("negative radius")
    a = np.asarray(alpha_sorted, dtype=np.float64)
    lo = int(np.searchsorted(a, alpha_q - R, side="left"))
    hi = int(np.searchsorted(a, alpha_q + R, side="right"))
    return lo, max(lo, hi)


def alg2_query(index: dict, P, q, R: float) -> np.ndarray:
    """Algorithm 2 for one query: x_q = q - mu (l.2), alpha_q (l.3),
    window J (l.4), then the radius test over X(J,:) (l.5-6).  The test is evaluated with
    eq:ip1 on the original coordinates in fp64 (readings C3, C7) so the result
    is comparable with ``radius_query``.  Returns ascending original ids."""
    q = np.asarray(q, dtype=np.float64)
    xq = q - index["mu"]
    aq = float(xq @ index["v1"])
    lo, hi = candidate_range(index["alpha"], aq, R)
    P = _f64(P)
    ids = index["perm"][lo:hi]
    R2 = float(R) * float(R)
    out = [int(i) for i in ids if sqdist(P[i], q) <= R2]
    return np.array(sorted(out), dtype=np.int64)


# ----------------------------------------------------------------- metrics
METRICS = {"euclidean": 0, "cosine": 1, "angular": 2}


def cosine_distance(p, q) -> float:
    """Definition: cdist(p, q) = 1 - p.q / (||p|| ||q||), fp64."""
    p, q = np.asarray(p, dtype=np.float64), np.asarray(q, dtype=np.float64)
    return float(1.0 - (p @ q) / (np.linalg.norm(p) * np.linalg.norm(q)))


def angular_distance(p, q) -> float:
    """Definition: theta(p, q) = arccos(p.q / (||p|| ||q||)), fp64."""
    p, q = np.asarray(p, dtype=np.float64), np.asarray(q, dtype=np.float64)
    c = (p @ q) / (np.linalg.norm(p) * np.linalg.norm(q))
    return float(np.arccos(np.clip(c, -1.0, 1.0)))


def normalize_rows(P) -> np.ndarray:
    """u_i = p_i / ||p_i|| with DESIGN.md reading C21's rule: fp64 sum of
    squares left to right, correctly rounded sqrt and division, rounded to the input
    dtype.  A zero row raises ValueError."""
    P = np.asarray(P)
    dt = P.dtype if P.dtype in (np.float32, np.float64) else np.float64
    X = P.astype(np.float64)
    s = np.zeros(X.shape[0], dtype=np.float64)
    for k in range(X.shape[1]):            # left to right over the coordinates
        s = s + X[:, k] * X[:, k]
    if np.any(s <= 0.0):
        raise ValueError("zero row")
    return (X / np.sqrt(s)[:, None]).astype(dt)


def metric_radius(metric: str, r: float) -> float:
    """Euclidean radius on unit vectors equivalent to metric radius r: 2 cdist = ||u-v||^2
     -> sqrt(2 r); theta <= alpha iff ||u-v||^2 <= 2 - 2 cos(alpha)
     -> sqrt(2 - 2 cos alpha), every pair (3.0) for alpha >= pi."""
    import math
    if metric == "cosine":
        return math.sqrt(2.0 * r)
    if metric == "angular":
        return 3.0 if r >= math.pi else math.sqrt(2.0 - 2.0 * math.cos(r))
    return float(r)


def metric_distance(metric: str, e) -> np.ndarray:
    """Metric value of a returned float32 Euclidean distance e on unit vectors:
    cdist = e^2 / 2, theta = 2 asin(e / 2) (chord length), fp64 then
    float32."""
    e = np.asarray(e, dtype=np.float64)
    if metric == "cosine":
        return (0.5 * e * e).astype(np.float32)
    if metric == "angular":
        return (2.0 * np.arcsin(np.minimum(1.0, 0.5 * e))).astype(np.float32)
    return e.astype(np.float32)


def metric_radius_query(P, Q, r: float, metric: str) -> dict:
    """Fixed-radius search under ``metric``: ``radius_query`` on the
    normalized rows with the mapped radius; adds ``dist`` = the metric value of every hit's
    float32 Euclidean distance (``metric_distance``)."""
    U, V = normalize_rows(P), normalize_rows(Q)
    out = radius_query(U, V, metric_radius(metric, r), band_rel=0.0)
    out["dist"] = metric_distance(metric, np.sqrt(out["s"]).astype(np.float32))
    out["U"], out["V"] = U, V
    return out


def manhattan_query(P, Q, R: float) -> dict:
    """Brute force ||p_i - q_j||_1 <= R: fp64 sum of |p_k - q_k| left to
    right (reading C22).  CSR over queries, ids ascending, ``dist`` = float32(L1)."""
    P, Q = _f64(P), _f64(Q)
    offs, ids, vals = [0], [], []
    for q in Q:
        v = np.zeros(P.shape[0])
        for k in range(P.shape[1]):
            v = v + np.abs(P[:, k] - q[k])
        hit = np.nonzero(v <= R)[0]
        ids.append(hit)
        vals.append(v[hit])
        offs.append(offs[-1] + len(hit))
    return {"offsets": np.array(offs, dtype=np.int64),
            "indices": np.concatenate(ids).astype(np.int32) if ids else np.zeros(0, np.int32),
            "dist": np.concatenate(vals).astype(np.float32) if vals else np.zeros(0, np.float32)}


def inner_product_query(P, Q, tau: float) -> dict:
    """Brute force p_i^T q_j >= tau (the fixed-threshold form of PAPER.md:73-78's maximum
    inner product similarity, reading C22): fp64 sum of p_k q_k left to right, no FMA.
    CSR over queries, ids ascending, ``dist`` = float32(p^T q)."""
    P, Q = _f64(P), _f64(Q)
    offs, ids, vals = [0], [], []
    for q in Q:
        v = np.zeros(P.shape[0])
        for k in range(P.shape[1]):
            v = v + P[:, k] * q[k]
        hit = np.nonzero(v >= tau)[0]
        ids.append(hit)
        vals.append(v[hit])
        offs.append(offs[-1] + len(hit))
    return {"offsets": np.array(offs, dtype=np.int64),
            "indices": np.concatenate(ids).astype(np.int32) if ids else np.zeros(0, np.int32),
            "dist": np.concatenate(vals).astype(np.float32) if vals else np.zeros(0, np.float32)}


def mips_transform(P, Q):
    """p~_i = [sqrt(xi^2 - |p_i|^2), p_i], xi = max_i |p_i|, q~ = [0, q] (fp64)."""
    P, Q = _f64(P), _f64(Q)
    n2 = (P * P).sum(axis=1)
    xi2 = n2.max()
    Pt = np.concatenate([np.sqrt(np.maximum(0.0, xi2 - n2))[:, None], P], axis=1)
    Qt = np.concatenate([np.zeros((Q.shape[0], 1)), Q], axis=1)
    return Pt, Qt, float(xi2)
