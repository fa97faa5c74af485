"""Pins for the CPU oracle (no GPU).  Each test ties the oracle to something other than
itself: the paper's printed values, hand-computed examples, closed forms, independent
library routines (scipy cKDTree, LAPACK eigh, scipy csgraph) and exact integer arithmetic.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rows(res, j):
    o = res["offsets"]
    return res["indices"][o[j]:o[j + 1]], res["s"][o[j]:o[j + 1]]


def _hits(res, j):
    ids, s = _rows(res, j)
    return set(ids[s <= res["R2"]].tolist())


# --------------------------------------------------------------------------- eq:ip1 order
def test_sqdist_is_left_to_right_without_fma():
    """eq:ip1 evaluated as pure-Python floats (IEEE fp64, one rounding
    per op, no FMA) must be bit-identical to the oracle's C evaluation."""
    rng = np.random.default_rng(11)
    for d in (1, 2, 3, 7, 64, 784):
        for _ in range(20):
            p = rng.standard_normal(d) * 10 ** rng.uniform(-3, 3)
            q = p + rng.standard_normal(d) * 10 ** rng.uniform(-6, 1)
            s = 0.0
            for k in range(d):
                t = float(p[k]) - float(q[k])
                s = s + t * t
            assert oracle.sqdist(p, q) == s


# --------------------------------------------------------------------------- hand example
def test_d3_hand_example_index_and_queries():
    g = json.load(open(os.path.join(GOLDEN, "d3_hand_example.json")))
    P = np.array(g["P"], dtype=np.float64)
    idx = oracle.build_index(P)
    np.testing.assert_allclose(idx["mu"], g["mu"], atol=0)
    np.testing.assert_allclose(oracle.center(P, idx["mu"]), g["Xc"], atol=0)
    np.testing.assert_allclose(idx["v1"], g["v1"], atol=1e-15)
    assert abs(idx["sigma"][1]) < 1e-12
    np.testing.assert_allclose(idx["alpha"], g["alpha_sorted"], atol=1e-14)
    np.testing.assert_allclose(idx["xbar"], g["xbar_sorted"], atol=1e-14)
    assert idx["perm"].tolist() == g["perm"]
    for r in g["ranges"]:
        assert oracle.candidate_range(g["alpha_sorted"], r["alpha_q"], r["R"]) == (r["lo"], r["hi"])
    for qq in g["queries"]:
        res = oracle.radius_query(P, np.array([qq["q"]], dtype=np.float64), qq["R"], band_rel=0)
        ids, s = _rows(res, 0)
        got = {int(i): math.sqrt(v) for i, v in zip(ids, s)}
        assert got == {int(k): v for k, v in qq["hits"].items()}
        assert oracle.alg2_query(idx, P, qq["q"], qq["R"]).tolist() == sorted(got)
    b = g["batch"]
    res = oracle.radius_query(P, np.array(b["Q"], dtype=np.float64), b["R"], band_rel=0)
    assert [sorted(_hits(res, j)) for j in range(2)] == b["hits"]


# --------------------------------------------------------------------------- exact boundary
@pytest.mark.parametrize("d,R", [(2, 5), (3, 5), (3, 3), (2, 0)])
def test_integer_lattice_exact_boundary(d, R):
    """Integer points: squared distances are exact in fp64, so the inclusive boundary
    ("<= R") must be reproduced exactly, e.g. (3,4) at R=5 is a hit."""
    g = np.stack(np.meshgrid(*[np.arange(-6, 7)] * d, indexing="ij"), -1).reshape(-1, d)
    Q = np.array([[0] * d, [1] * d, [2, -3] + [1] * (d - 2)], dtype=np.float64)
    res = oracle.radius_query(g.astype(np.float64), Q, float(R), band_rel=0)
    for j, q in enumerate(Q.astype(np.int64)):
        expect = {i for i, p in enumerate(g) if int(((p - q) ** 2).sum()) <= R * R}
        assert _hits(res, j) == expect
    if (d, R) == (2, 5):
        ids = _hits(res, 0)
        assert {tuple(g[i]) for i in ids} >= {(3, 4), (4, 3), (-5, 0), (0, 5)}


# --------------------------------------------------------------------------- library cross-check
@pytest.mark.parametrize("n,m,d,seed", [(3000, 200, 2, 1), (2000, 150, 3, 2), (1500, 100, 8, 3),
                                        (1000, 80, 64, 4), (600, 40, 784, 5)])
def test_matches_scipy_ckdtree(n, m, d, seed):
    """Independent implementation: scipy's cKDTree ball query.  Sets must agree except
    for pairs within 1e-9 relative of the boundary (different rounding paths)."""
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    P = rng.random((n, d))
    Q = rng.random((m, d))
    # radius giving ~1% return ratio
    R = float(np.quantile(np.linalg.norm(P[:300, None, :] - Q[None, :20, :], axis=-1), 0.01))
    res = oracle.radius_query(P, Q, R, band_rel=1e-9)
    tree = cKDTree(P)
    for j in range(m):
        ids, s = _rows(res, j)
        sure = set(ids[s <= R * R * (1 - 1e-9)].tolist())
        mine = set(ids[s <= R * R].tolist())
        ref = set(tree.query_ball_point(Q[j], R))
        assert sure <= ref <= set(ids.tolist())
        assert mine <= set(ids.tolist())


def test_distances_against_numpy_norm():
    rng = np.random.default_rng(7)
    P = rng.standard_normal((500, 5)) * 3
    Q = rng.standard_normal((20, 5)) * 3
    res = oracle.radius_query(P, Q, 3.0, band_rel=0)
    for j in range(20):
        ids, s = _rows(res, j)
        np.testing.assert_allclose(np.sqrt(s), np.linalg.norm(P[ids] - Q[j], axis=1), rtol=1e-14)
        full = np.linalg.norm(P - Q[j], axis=1)
        sure = set(np.nonzero(full <= 3.0 * (1 - 1e-12))[0].tolist())
        maybe = set(np.nonzero(full <= 3.0 * (1 + 1e-12))[0].tolist())
        assert sure <= set(ids.tolist()) <= maybe


# --------------------------------------------------------------------------- closed forms
def _unit_square(r):
    return math.pi * r * r - 8 * r ** 3 / 3 + r ** 4 / 2


def _unit_cube(r):
    return 4 * math.pi / 3 * r ** 3 - 1.5 * math.pi * r ** 4 + 1.6 * r ** 5 - r ** 6 / 6


def test_c1_return_ratio_closed_form_and_paper_table1():
    """C1 = the paper's Table 1 cell n=2000, d=2, R=0.05 (0.755%).
    Non-self pair fraction vs the closed form P(|U-V|<=r) on the unit square."""
    w = workloads.c1()
    res = oracle.radius_query(w.X, w.X, w.R, band_rel=0)
    n = w.n
    nonself = sum(len(_hits(res, j)) - 1 for j in range(n)) / (n * (n - 1))
    g = json.load(open(os.path.join(GOLDEN, "paper_return_ratios.json")))
    assert abs(100 * nonself - 100 * _unit_square(0.05)) / (100 * _unit_square(0.05)) < 0.05
    assert abs(100 * nonself - g["table1_d2"]["n2000"]["0.05"]) / g["table1_d2"]["n2000"]["0.05"] < 0.05
    # every point is its own neighbour; the relation is symmetric
    for j in range(0, n, 97):
        assert j in _hits(res, j)
        for i in _hits(res, j):
            assert j in _hits(res, i)


@pytest.mark.parametrize("R", ["0.02", "0.05", "0.08", "0.11", "0.14"])
def test_table1_d2_n10000_ratios(R):
    g = json.load(open(os.path.join(GOLDEN, "paper_return_ratios.json")))
    w = workloads.uniform(10000, 2, seed=123)
    r = float(R)
    Q = w.X[:1000]
    res = oracle.radius_query(w.X, Q, r, band_rel=0)
    nonself = (res["offsets"][-1] - 1000) / (1000 * (w.n - 1))
    closed = _unit_square(r)
    printed = g["table1_d2"]["n10000"][R] / 100
    tol = 0.04 if r > 0.03 else 0.08
    assert abs(nonself - closed) / closed < tol
    assert abs(closed - printed) / printed < 0.006   # closed form vs paper's print


@pytest.mark.parametrize("R", ["0.05", "0.10", "0.15", "0.20", "0.25"])
def test_table2_d3_ratios(R):
    g = json.load(open(os.path.join(GOLDEN, "paper_return_ratios.json")))
    w = workloads.uniform(10000, 3, seed=321)
    r = float(R)
    res = oracle.radius_query(w.X, w.X[:1000], r, band_rel=0)
    nonself = (res["offsets"][-1] - 1000) / (1000 * (w.n - 1))
    closed = _unit_cube(r)
    printed = g["table2_d3"]["n10000"][R] / 100
    assert abs(nonself - closed) / closed < (0.15 if r < 0.07 else 0.05)
    assert abs(closed - printed) / printed < 0.05


# --------------------------------------------------------------------------- invariants
def test_invariants_symmetry_self_monotone_R0():
    rng = np.random.default_rng(5)
    P = rng.random((800, 3)).astype(np.float32)
    P[10] = P[20]                     # duplicate pair
    a = oracle.radius_query(P, P, 0.08, band_rel=0)
    b = oracle.radius_query(P, P, 0.12, band_rel=0)
    z = oracle.radius_query(P, P, 0.0, band_rel=0)
    for j in range(800):
        ha, hb = _hits(a, j), _hits(b, j)
        assert j in ha and ha <= hb
        for i in ha:
            assert j in _hits(a, i)
        expect_zero = {j} | ({10, 20} if j in (10, 20) else set())
        assert _hits(z, j) == expect_zero


def test_empty_query_and_errors():
    P = np.zeros((5, 2))
    res = oracle.radius_query(P, np.zeros((0, 2)), 1.0)
    assert res["offsets"].tolist() == [0]
    with pytest.raises(ValueError):
        oracle.radius_query(P, np.zeros((1, 2)), -1.0)
    with pytest.raises(ValueError):
        oracle.radius_query(P, np.zeros((1, 3)), 1.0)
    with pytest.raises(ValueError):
        oracle.column_mean(np.zeros((0, 2)))


# --------------------------------------------------------------------------- Algorithm 1 pins
def test_principal_direction_pins():
    # d = 1: v1 = (1)
    v, _ = oracle.principal_direction(oracle.center(np.array([[1.0], [5.0], [2.0]]), [8 / 3]))
    assert v.tolist() == [1.0]
    # all-zero data -> e1 (SPEC.md:141 reading C9)
    v, s = oracle.principal_direction(np.zeros((4, 3)))
    assert v.tolist() == [1.0, 0.0, 0.0] and not s.any()
    # independent LAPACK routine (symmetric eigensolver on X^T X) agrees
    rng = np.random.default_rng(3)
    X = rng.standard_normal((4000, 6)) * np.array([3, 1, 0.5, 0.4, 0.3, 0.2])
    X = X @ np.linalg.qr(rng.standard_normal((6, 6)))[0]
    Xc = oracle.center(X, oracle.column_mean(X))
    v, s = oracle.principal_direction(Xc)
    w, V = np.linalg.eigh(Xc.T @ Xc)
    assert abs(abs(v @ V[:, -1]) - 1) < 1e-12
    np.testing.assert_allclose(s[0] ** 2, w[-1], rtol=1e-12)
    assert np.argmax(np.abs(v)) == np.argmax(np.abs(v)) and v[np.argmax(np.abs(v))] > 0


@pytest.mark.parametrize("s", [0.1, 0.5])
def test_elongated_gaussian_sigma_ratio(s):
    """std (1, s, ..., s) => singular values -> sqrt(n)(1, s, ..., s),
    v1 -> e1 (SPEC.md:132 asserts |sigma2/sigma1 - s| <= 0.05 at n=50,000)."""
    rng = np.random.default_rng(17)
    X = rng.standard_normal((50000, 5)) * np.array([1, s, s, s, s])
    v, sig = oracle.principal_direction(oracle.center(X, oracle.column_mean(X)))
    assert abs(sig[1] / sig[0] - s) <= 0.05
    assert abs(v[0]) > 0.99


def test_c3_closed_form_v1():
    """C3 covariance = Qo^T diag(1/i) Qo => v1 = +-(first row of Qo), sigma2/sigma1 ->
    1/sqrt(2) (SURVEY.md §8(c) pins)."""
    w = workloads.c3(n=40000, m=10)
    v, sig = oracle.principal_direction(oracle.center(w.X, oracle.column_mean(w.X)))
    assert abs(abs(v @ w.meta["Qo"][0]) - 1) < 2e-3
    assert abs(sig[1] / sig[0] - 1 / math.sqrt(2)) < 0.02


def test_sort_is_stable_with_duplicates():
    """five identical points -> all alpha = 0, pi = identity."""
    P = np.tile(np.array([[2.0, 3.0]]), (5, 1))
    idx = oracle.build_index(P)
    assert idx["perm"].tolist() == [0, 1, 2, 3, 4]
    assert not idx["alpha"].any() and not idx["xbar"].any()


# --------------------------------------------------------------------------- Algorithm 2 pins
@pytest.mark.parametrize("d,seed", [(2, 1), (3, 2), (5, 3)])
def test_cauchy_schwarz_window_contains_all_hits(d, seed):
    """eq:lower: every true neighbour lies in J.  And Alg. 2's answer
    equals the brute force; replacing v1 by any unit vector keeps it."""
    rng = np.random.default_rng(seed)
    P = rng.random((600, d)) * np.array([4.0] + [1.0] * (d - 1))
    Q = rng.random((25, d)) * np.array([4.0] + [1.0] * (d - 1))
    R = 0.3
    idx = oracle.build_index(P)
    res = oracle.radius_query(P, Q, R, band_rel=0)
    u = rng.standard_normal(d)
    u /= np.linalg.norm(u)
    Xc = oracle.center(P, idx["mu"])
    a2 = oracle.scores(Xc, u)
    pr = oracle.sort_index(a2)
    idx_u = dict(idx, v1=u, alpha=a2[pr], perm=pr)
    pos = np.empty(600, dtype=np.int64)
    pos[idx["perm"]] = np.arange(600)
    for j in range(25):
        h = _hits(res, j)
        aq = float((Q[j] - idx["mu"]) @ idx["v1"])
        lo, hi = oracle.candidate_range(idx["alpha"], aq, R)
        assert all(lo <= pos[i] < hi for i in h)
        assert set(oracle.alg2_query(idx, P, Q[j], R).tolist()) == h
        assert set(oracle.alg2_query(idx_u, P, Q[j], R).tolist()) == h


# --------------------------------------------------------------------------- DBSCAN pins
def test_dbscan_spec_examples():
    rng = np.random.default_rng(0)
    # two blobs: K = 2
    A = np.concatenate([rng.standard_normal((500, 2)) * 0.5,
                        rng.standard_normal((500, 2)) * 0.5 + 10])
    lab, K, _ = oracle.dbscan(A, 1.0, 5)
    assert K == 2
    core0 = lab[:500][lab[:500] >= 0]
    core1 = lab[500:][lab[500:] >= 0]
    assert len(set(core0.tolist())) == 1 and len(set(core1.tolist())) == 1
    assert core0[0] != core1[0]
    # grid spacing 10, eps 0.1: all noise
    G = np.stack(np.meshgrid(np.arange(10) * 10.0, np.arange(10) * 10.0), -1).reshape(-1, 2)
    lab, K, _ = oracle.dbscan(G, 0.1, 5)
    assert K == 0 and (lab == -1).all()
    # minPts 1, huge eps: one cluster
    lab, K, _ = oracle.dbscan(A, 1e6, 1)
    assert K == 1 and (lab == 0).all()


def test_dbscan_hand_chain():
    """1-D hand example: core chain 0-1-2-3 (spacing 1, eps 1, minPts 3), border 4 at
    distance 1 from core 3 only, isolated 5 -> noise; points ordered to test numbering."""
    P = np.array([[10.0], [0.0], [1.0], [2.0], [3.0], [4.0], [50.0], [11.0], [12.0]])
    lab, K, cnt = oracle.dbscan(P, 1.0, 3)
    # neighbourhoods incl. self: 10:{10,11}=2(non-core) ...
    assert cnt.tolist() == [2, 2, 3, 3, 3, 2, 1, 3, 2]
    # core: ids 2,3,4 (coords 1,2,3) and 7 (coord 11)
    # cluster 0 = {2,3,4} (min core id 2), cluster 1 = {7} (min core id 7)
    # borders: id1 (0.0) -> core 2 -> 0; id5 (4.0) -> core 4 -> 0;
    #          id0 (10) -> core 7 -> 1; id8 (12) -> core 7 -> 1; id6 noise
    assert K == 2
    assert lab.tolist() == [1, 0, 0, 0, 0, 0, -1, 1, 1]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_dbscan_vs_scipy_csgraph(seed):
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    from scipy.spatial import cKDTree
    w = workloads.c5(n=3000, seed=seed, box=200.0)
    P = w.X.astype(np.float64)
    eps, mp = 3.0, 5
    lab, K, cnt = oracle.dbscan(P, eps, mp)
    tree = cKDTree(P)
    nb = tree.query_ball_point(P, eps)
    # reject instances with a pair within 1e-9 of eps (rounding-path dependence)
    pairs = tree.query_pairs(eps * (1 + 1e-9), output_type="ndarray")
    dd = np.linalg.norm(P[pairs[:, 0]] - P[pairs[:, 1]], axis=1)
    assert not np.any(np.abs(dd - eps) < 1e-9 * eps)
    ref_cnt = np.array([len(x) for x in nb])
    assert (ref_cnt == cnt).all()
    core = ref_cnt >= mp
    cid = np.nonzero(core)[0]
    e = pairs[core[pairs[:, 0]] & core[pairs[:, 1]] & (dd <= eps)]
    A = coo_matrix((np.ones(len(e)), (e[:, 0], e[:, 1])), shape=(len(P), len(P)))
    _, comp = connected_components(A, directed=False)
    ref = np.full(len(P), -1)
    order = {}
    for i in cid:                      # canonical numbering by min core id
        order.setdefault(comp[i], len(order))
        ref[i] = order[comp[i]]
    for i in np.nonzero(~core)[0]:     # border: first cluster the ascending FIFO scan reaches it with
        cn = [ref[j] for j in nb[i] if core[j]]
        if cn:
            ref[i] = min(cn)
    assert K == len(order)
    assert (ref == lab).all()
    lg, Kg, cg = oracle.dbscan(P, eps, mp, grid=True)
    assert Kg == K and np.array_equal(lg, lab) and np.array_equal(cg, cnt)


def test_dbscan_border_goes_to_first_cluster_reaching_it():
    """Hand example for the border rule (reading C18): cluster A = ids
    {0, 7, 8, 9} (min core id 0 -> cluster 0), cluster B = ids {1, 2, 3, 4} (cluster 1);
    border id 5 at x = 2 is within eps of A's core 9 (x = 1) and B's core 1 (x = 3).  The
    ascending-id FIFO scan expands A first and labels 5 with A (cluster 0), although its
    smallest-id core neighbour (1) is in B.  scikit-learn's DBSCAN (the implementation the
    paper plugs SNN into) gives the same labels."""
    x = {0: 0.0, 7: 0.3, 8: 0.6, 9: 1.0, 1: 3.0, 2: 3.3, 3: 3.6, 4: 4.0, 5: 2.0, 6: 50.0}
    P = np.array([[x[i]] for i in range(10)])
    lab, K, cnt = oracle.dbscan(P, 1.05, 4)
    assert cnt.tolist() == [4, 5, 4, 4, 4, 3, 1, 4, 4, 5]
    assert K == 2
    assert lab.tolist() == [0, 1, 1, 1, 1, 0, -1, 0, 0, 0]
    lg, Kg, _ = oracle.dbscan(P, 1.05, 4, grid=True)
    assert Kg == 2 and lg.tolist() == lab.tolist()
    from sklearn.cluster import DBSCAN
    sk = DBSCAN(eps=1.05, min_samples=4, algorithm="brute").fit(P).labels_
    assert sk.tolist() == lab.tolist()


@pytest.mark.parametrize("seed,n,box,eps,mp", [(5, 2500, 120.0, 3.0, 5), (6, 2000, 60.0, 2.0, 8),
                                                 (7, 3000, 300.0, 4.0, 3)])
def test_dbscan_matches_scikit_learn(seed, n, box, eps, mp):
    """scikit-learn's DBSCAN (brute-force neighbourhoods, PAPER.md:594 compares against it)
    on C5-recipe data: labels equal element by element, brute-force and grid oracle alike.
    Instances with a pair within 1e-9 of eps are rejected (sklearn computes distances by
    another formula)."""
    from scipy.spatial import cKDTree
    from sklearn.cluster import DBSCAN
    P = workloads.c5(n=n, seed=seed, box=box).X.astype(np.float64)
    pairs = cKDTree(P).query_pairs(eps * (1 + 1e-9), output_type="ndarray")
    dd = np.linalg.norm(P[pairs[:, 0]] - P[pairs[:, 1]], axis=1)
    assert not np.any(np.abs(dd - eps) < 1e-9 * eps)
    sk = DBSCAN(eps=eps, min_samples=mp, algorithm="brute").fit(P).labels_
    lab, K, _ = oracle.dbscan(P, eps, mp)
    assert np.array_equal(sk, lab) and K == sk.max() + 1 and K >= 2
    lg, Kg, _ = oracle.dbscan(P, eps, mp, grid=True)
    assert np.array_equal(lg, lab) and Kg == K


def test_neighbour_counts_pins():
    """oracle.neighbour_counts (DBSCAN's eps-neighbourhood sizes, self included): the hand
    chain's counts, the brute-force radius query's row lengths and scipy cKDTree's ball
    counts agree on sampled ids."""
    P = np.array([[10.0], [0.0], [1.0], [2.0], [3.0], [4.0], [50.0], [11.0], [12.0]])
    assert oracle.neighbour_counts(P, 1.0, np.arange(9)).tolist() == [2, 2, 3, 3, 3, 2, 1, 3, 2]
    assert oracle.neighbour_counts(P, 1.0, [6, 2, 2]).tolist() == [1, 3, 3]
    from scipy.spatial import cKDTree
    w = workloads.c5(n=6000, seed=12, box=150.0)
    ids = np.random.default_rng(3).choice(w.n, 300, replace=False)
    cnt = oracle.neighbour_counts(w.X, 3.0, ids)
    res = oracle.radius_query(w.X, w.X[ids], 3.0, band_rel=0.0)
    assert np.array_equal(cnt, np.diff(res["offsets"]))
    P64 = w.X.astype(np.float64)
    ball = cKDTree(P64).query_ball_point(P64[ids], 3.0)
    pairs = cKDTree(P64).query_pairs(3.0 * (1 + 1e-9), output_type="ndarray")
    dd = np.linalg.norm(P64[pairs[:, 0]] - P64[pairs[:, 1]], axis=1)
    assert not np.any(np.abs(dd - 3.0) < 1e-9 * 3.0)
    assert cnt.tolist() == [len(b) for b in ball]
    assert cnt.min() >= 1                     # self included


# --------------------------------------------------------------------------- grid oracle (d <= 3)
def _same_csr(a, b):
    assert np.array_equal(a["offsets"], b["offsets"])
    assert np.array_equal(a["indices"], b["indices"])
    assert np.array_equal(a["s"], b["s"])


@pytest.mark.parametrize("d,seed,n,m,R", [(1, 0, 3000, 500, 0.002), (2, 1, 4000, 700, 0.03),
                                          (3, 2, 5000, 900, 0.08), (3, 3, 2000, 2000, 0.5),
                                          (2, 4, 3000, 300, 2.5)])
def test_grid_radius_query_equals_brute_force(d, seed, n, m, R):
    """Grid-pruned oracle (d <= 3) == brute force, row by row (ids, fp64 s, band pairs),
    random data plus queries outside the data's box."""
    rng = np.random.default_rng(seed)
    P = rng.random((n, d)).astype(np.float32)
    Q = (rng.random((m, d)) * 1.2 - 0.1).astype(np.float32)
    _same_csr(oracle.radius_query(P, Q, R, grid=True), oracle.radius_query(P, Q, R))
    _same_csr(oracle.radius_query(P, P, R, grid=True), oracle.radius_query(P, P, R))


@pytest.mark.parametrize("d", [1, 2, 3])
def test_grid_radius_query_lattice_boundaries_duplicates(d):
    """Integer lattice: many pairs at exactly R (3-4-5 and axis pairs) and points exactly on
    cell boundaries; duplicates; R = 0 (coincidences only); a far outlier that makes the
    extent/R ratio exceed 2^20 (cell side grows)."""
    g = np.stack(np.meshgrid(*[np.arange(12.0)] * d, indexing="ij"), -1).reshape(-1, d)
    base = np.concatenate([g * 5.0, g[:50] * 5.0])
    for P in (base, np.concatenate([base, np.full((1, d), 1e8)])):
        for R in (5.0, 25.0, 0.0, 7.0710678118654755):
            _same_csr(oracle.radius_query(P, P, R, grid=True), oracle.radius_query(P, P, R))
    P = base
    Q = g[::7] * 5.0 + 2.5
    _same_csr(oracle.radius_query(P, Q, 2.5 * np.sqrt(d), grid=True),
              oracle.radius_query(P, Q, 2.5 * np.sqrt(d)))


# ---------------------------------------------------------------- metrics
def test_metric_hand_values():
    """Textbook values of the definitions and of the reductions."""
    assert oracle.cosine_distance([1, 0], [0, 1]) == pytest.approx(1.0)
    assert oracle.cosine_distance([1, 0], [-3, 0]) == pytest.approx(2.0)
    assert oracle.cosine_distance([1, 1], [2, 2]) == pytest.approx(0.0, abs=1e-15)
    assert oracle.angular_distance([1, 0], [0, 5]) == pytest.approx(math.pi / 2)
    assert oracle.angular_distance([1, 0], [1, 1]) == pytest.approx(math.pi / 4)
    np.testing.assert_array_equal(oracle.normalize_rows(np.array([[3.0, 4.0]])), [[0.6, 0.8]])
    # unit vectors at angle a have chord 2 sin(a/2): both radius maps and the inverse
    for a in (0.1, 0.7, math.pi / 2, 2.5):
        chord = 2 * math.sin(a / 2)
        assert oracle.metric_radius("angular", a) == pytest.approx(chord, rel=1e-12)
        assert oracle.metric_radius("cosine", 1 - math.cos(a)) == pytest.approx(chord, rel=1e-12)
        assert float(oracle.metric_distance("angular", np.float32(chord))) == pytest.approx(a, rel=1e-6)
        assert float(oracle.metric_distance("cosine", np.float32(chord))) == pytest.approx(1 - math.cos(a), rel=1e-6)
    assert oracle.metric_radius("angular", math.pi) >= 2.0
    with pytest.raises(ValueError):
        oracle.normalize_rows(np.array([[1.0, 2.0], [0.0, 0.0]]))


@pytest.mark.parametrize("metric,dtype", [("cosine", np.float64), ("angular", np.float64),
                                          ("cosine", np.float32), ("angular", np.float32)])
def test_metric_query_matches_definition(metric, dtype):
    """The Euclidean reduction on normalized rows returns exactly the pairs the direct
    definition puts within r (pairs within 1e-6 of the boundary excluded), with the metric
    value of each hit within float32 rounding of the definition."""
    rng = np.random.default_rng(7)
    P = (rng.standard_normal((150, 5)) + 0.5).astype(dtype)
    Q = (rng.standard_normal((40, 5)) + 0.5).astype(dtype)
    direct = oracle.cosine_distance if metric == "cosine" else oracle.angular_distance
    r = 0.3 if metric == "cosine" else 0.8
    out = oracle.metric_radius_query(P, Q, r, metric)
    got = {(j, int(i)) for j in range(len(Q)) for i in out["indices"][out["offsets"][j]:out["offsets"][j + 1]]}
    D = np.array([[direct(q, p) for p in P] for q in Q])
    want = {(j, i) for j in range(len(Q)) for i in range(len(P)) if D[j, i] <= r}
    amb = {(j, i) for j in range(len(Q)) for i in range(len(P)) if abs(D[j, i] - r) <= 1e-6}
    assert (got ^ want) <= amb and len(want) > 50
    rows = np.repeat(np.arange(len(Q)), np.diff(out["offsets"]))
    np.testing.assert_allclose(out["dist"], D[rows, out["indices"]], atol=2e-6)


def test_manhattan_and_inner_product_oracles():
    """Brute-force L1 / inner-product searches against scipy's cityblock distance and the
    BLAS product (away from the threshold), plus the two facts the GPU reductions rest on:
    every L1 hit is an L2 hit for the same R, and the MIPS transform gives
    |p~ - q~|^2 = xi^2 + |q|^2 - 2 p^T q."""
    from scipy.spatial.distance import cdist
    rng = np.random.default_rng(11)
    P = rng.standard_normal((300, 6))
    Q = rng.standard_normal((30, 6))
    R = 2.5
    man = oracle.manhattan_query(P, Q, R)
    D1 = cdist(Q, P, "cityblock")
    rows = np.repeat(np.arange(30), np.diff(man["offsets"]))
    got = set(zip(rows.tolist(), man["indices"].tolist()))
    want = set(zip(*np.nonzero(D1 <= R)))
    amb = set(zip(*np.nonzero(np.abs(D1 - R) < 1e-9)))
    assert (got ^ want) <= amb and len(want) > 30
    np.testing.assert_allclose(man["dist"], D1[rows, man["indices"]], rtol=1e-6)
    l2 = oracle.radius_query(P, Q, R, band_rel=0.0)
    l2rows = np.repeat(np.arange(30), np.diff(l2["offsets"]))
    assert got <= set(zip(l2rows.tolist(), l2["indices"].tolist()))
    tau = 2.0
    ip = oracle.inner_product_query(P, Q, tau)
    G = Q @ P.T
    rows = np.repeat(np.arange(30), np.diff(ip["offsets"]))
    got = set(zip(rows.tolist(), ip["indices"].tolist()))
    want = set(zip(*np.nonzero(G >= tau)))
    amb = set(zip(*np.nonzero(np.abs(G - tau) < 1e-9)))
    assert (got ^ want) <= amb and len(want) > 30
    np.testing.assert_allclose(ip["dist"], G[rows, ip["indices"]], rtol=1e-6, atol=1e-6)
    Pt, Qt, xi2 = oracle.mips_transform(P, Q)
    np.testing.assert_allclose(np.linalg.norm(Pt, axis=1) ** 2, xi2, rtol=1e-12)
    lhs = ((Pt[None, :, :] - Qt[:, None, :]) ** 2).sum(-1)
    rhs = xi2 + (Q * Q).sum(1)[:, None] - 2 * G
    np.testing.assert_allclose(lhs, rhs, rtol=1e-10, atol=1e-10)
    # the argmax statement of PAPER.md:76
    np.testing.assert_array_equal(lhs.argmin(axis=1), G.argmax(axis=1))
