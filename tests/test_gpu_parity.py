"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by
element on the same seeded inputs.  All tests need an sm_100 device."""
import numpy as np
import pytest

import oracle
import workloads
from tests.parity import compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def snn():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_07679_b200 import build_lib
    build_lib.build()
    import paper_2212_07679_b200 as p
    p.load_library()
    return p


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(snn, X, Q, R, host=False):
    idx = snn.Index(X if host else _dev(X))
    try:
        if Q is None:
            return idx.query_self(R)
        return idx.query(Q if host else _dev(Q), R)
    finally:
        idx.free()


# --------------------------------------------------------------------------- small random
CASES = [
    # (n, m, d, dtype, R-quantile, seed)
    (1000, 300, 1, np.float32, 0.01, 1),
    (3001, 517, 2, np.float32, 0.01, 2),
    (4099, 1000, 3, np.float32, 0.005, 3),
    (2500, 333, 4, np.float32, 0.02, 4),
    (1777, 250, 5, np.float32, 0.02, 5),
    (1500, 200, 8, np.float32, 0.05, 6),
    (1200, 130, 9, np.float32, 0.05, 7),
    (1100, 129, 16, np.float32, 0.05, 8),
    (900, 100, 17, np.float32, 0.05, 9),
    (700, 77, 64, np.float32, 0.05, 10),
    (500, 65, 100, np.float32, 0.05, 11),
    (300, 40, 784, np.float32, 0.05, 12),
    (2000, 300, 2, np.float64, 0.01, 13),
    (1500, 200, 3, np.float64, 0.01, 14),
    (600, 70, 33, np.float64, 0.05, 15),
]


@pytest.mark.parametrize("n,m,d,dt,qr,seed", CASES)
def test_random_parity(snn, n, m, d, dt, qr, seed):
    rng = np.random.default_rng(seed)
    X = (rng.standard_normal((n, d)) * rng.uniform(0.5, 3, d)).astype(dt)
    Q = (rng.standard_normal((m, d)) * rng.uniform(0.5, 3, d)).astype(dt)
    R = float(np.quantile(np.linalg.norm(X[:200, None, :].astype(np.float64) - Q[None, :50, :], axis=-1), qr))
    gpu = run(snn, X, Q, R)
    ora = oracle.radius_query(X, Q, R)
    compare(gpu, ora)


@pytest.mark.parametrize("d,dt", [(2, np.float32), (3, np.float32), (3, np.float64), (20, np.float32)])
def test_self_query_parity_and_invariants(snn, d, dt):
    rng = np.random.default_rng(100 + d)
    X = (rng.random((5000, d)) * 10).astype(dt)
    X[17] = X[4000]            # exact duplicate
    R = 0.9 if d <= 3 else 6.0
    gpu = run(snn, X, None, R)
    ora = oracle.radius_query(X, X, R)
    compare(gpu, ora)
    off = gpu.offsets
    for j in range(0, 5000, 37):
        ids = set(gpu.indices[off[j]:off[j + 1]].tolist())
        assert j in ids                                   # every point is its own neighbour
        for i in list(ids)[:10]:
            assert j in set(gpu.indices[off[i]:off[i + 1]].tolist())   # symmetry
    assert 4000 in set(gpu.indices[off[17]:off[18]].tolist())


def test_host_pointer_inputs_match_device(snn):
    rng = np.random.default_rng(3)
    X = rng.random((3000, 3)).astype(np.float32)
    Q = rng.random((400, 3)).astype(np.float32)
    a = run(snn, X, Q, 0.07, host=False)
    b = run(snn, X, Q, 0.07, host=True)
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.distances, b.distances)


# --------------------------------------------------------------------------- adversarial
def test_exact_boundary_integer_lattice(snn):
    """Pairs at exactly d = R (3-4-5 triangles) are hits; fp32-exact inputs."""
    g = np.stack(np.meshgrid(np.arange(-8, 9), np.arange(-8, 9), np.arange(-2, 3), indexing="ij"), -1)
    X = g.reshape(-1, 3).astype(np.float32)
    for R in (5.0, 3.0, np.sqrt(2.0), 0.0):
        gpu = run(snn, X, X[::7], float(R))
        ora = oracle.radius_query(X, X[::7], float(R))
        compare(gpu, ora)


def test_far_from_origin_cancellation(snn):
    """Coordinates ~1e4 with R ~ 1e-2: large |x|, tiny distances (centering and the
    expanded form would lose everything; the direct form + recheck stays exact)."""
    rng = np.random.default_rng(9)
    X = (1e4 + rng.random((20000, 3)) * 0.5).astype(np.float32)
    Q = X[rng.integers(0, 20000, 500)] + rng.standard_normal((500, 3)).astype(np.float32) * 1e-3
    gpu = run(snn, X, Q.astype(np.float32), 0.02)
    ora = oracle.radius_query(X, Q.astype(np.float32), 0.02)
    st = compare(gpu, ora)
    assert st["oracle_hits"] > 0


def test_near_boundary_pairs_fp32(snn):
    """Queries placed at distance R(1 +- k 2^-24) from data points."""
    rng = np.random.default_rng(21)
    X = rng.random((4000, 3)).astype(np.float32) * 4
    R = 0.25
    u = rng.standard_normal((3000, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    k = rng.integers(-8, 9, 3000)[:, None]
    base = X[rng.integers(0, 4000, 3000)].astype(np.float64)
    Q = (base + u * R * (1 + k * 2.0 ** -24)).astype(np.float32)
    gpu = run(snn, X, Q, R)
    ora = oracle.radius_query(X, Q, R)
    compare(gpu, ora)


# --------------------------------------------------------------------------- edge cases
def test_edge_cases(snn):
    import paper_2212_07679_b200 as p
    # n = 1
    X = np.array([[1.0, 2.0]], dtype=np.float32)
    r = run(snn, X, None, 0.0)
    assert r.offsets.tolist() == [0, 1] and r.indices.tolist() == [0]
    # all identical points: every pair at distance 0
    X = np.ones((300, 4), dtype=np.float32)
    r = run(snn, X, None, 0.0)
    assert r.nnz == 300 * 300 and not r.distances.any()
    # collinear data (sigma2 = 0): every candidate on the line within R is a hit
    t = np.linspace(0, 10, 2001)
    X = np.stack([t, 2 * t, -t], 1).astype(np.float32)
    compare(run(snn, X, None, 0.05), oracle.radius_query(X, X, 0.05))
    # m = 0
    idx = p.Index(_dev(np.random.rand(10, 3).astype(np.float32)))
    r = idx.query(_dev(np.zeros((0, 3), dtype=np.float32)), 1.0)
    assert r.offsets.tolist() == [0]
    # errors
    with pytest.raises(p.SnnError) as e:
        idx.query(_dev(np.zeros((2, 4), dtype=np.float32)), 1.0)
    assert e.value.name == "SNN_ERR_DIM_MISMATCH"
    with pytest.raises(p.SnnError) as e:
        idx.query(_dev(np.zeros((2, 3), dtype=np.float32)), -1.0)
    assert e.value.name == "SNN_ERR_INVALID_ARGUMENT"
    bad = np.zeros((2, 3), dtype=np.float32)
    bad[1, 2] = np.nan
    with pytest.raises(p.SnnError) as e:
        idx.query(_dev(bad), 1.0)
    assert e.value.name == "SNN_ERR_NONFINITE"
    idx.free()
    with pytest.raises(p.SnnError) as e:
        p.Index(_dev(np.zeros((0, 3), dtype=np.float32)))
    assert e.value.name == "SNN_ERR_EMPTY"
    Xb = np.zeros((5, 3), dtype=np.float32)
    Xb[2, 0] = np.inf
    with pytest.raises(p.SnnError) as e:
        p.Index(_dev(Xb))
    assert e.value.name == "SNN_ERR_NONFINITE"


def test_options_do_not_change_results(snn):
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(31)
    X = rng.random((6000, 3)).astype(np.float32)
    Q = rng.random((700, 3)).astype(np.float32)
    ref = run(snn, X, Q, 0.06)
    ora = oracle.radius_query(X, Q, 0.06)
    try:
        settings = [[("force_generic", 1)], [("chunk", 64)], [("query_block", 32)],
                    [("power_iters", 1)], [("cap", 1)], [("cap", 3)],
                    [("cap", 1), ("ovf_records", 5)], [("cap", 2), ("ovf_records", 1), ("chunk", 128)]]
        for setting in settings:
            for key, val in setting:
                p.snn_set_option(key, val)
            r = run(snn, X, Q, 0.06)
            compare(r, ora)
            for key, _ in setting:
                p.snn_set_option(key, 0)
    finally:
        for key in ("force_generic", "chunk", "query_block", "power_iters", "cap", "ovf_records"):
            p.snn_set_option(key, 0)
    assert ref.nnz == r.nnz


# --------------------------------------------------------------------------- index build
def test_index_build_parity(snn):
    """Alg. 1 outputs: mean, v1, keys within the rigorous bound, stable sort, gather, xbar."""
    import paper_2212_07679_b200 as p
    for d, n in ((3, 50000), (2, 7777), (64, 20000), (13, 3000), (300, 20000), (784, 5000)):
        w = workloads.c2(n=n) if d == 3 else None
        # spectrum with a clear top gap (d >= 128: 1/sqrt(i) decay, lambda1/lambda2 = 2)
        scale = np.linspace(3, 0.5, d) if d < 128 else 3.0 / np.sqrt(np.arange(1, d + 1))
        X = w.X if w else np.random.default_rng(d).standard_normal((n, d)).astype(np.float32) * \
            scale.astype(np.float32)
        idx = p.Index(_dev(X))
        arr = idx.arrays()
        info = arr["info"]
        mu, v1, keys, perm, xbar, xs = (arr[k].cpu().numpy() for k in ("mu", "v1", "keys", "perm", "xbar", "xs"))
        assert np.array_equal(xs[:, :d], X[perm])        # gather is a bitwise permutation
        assert not xs[:, d:].any()
        ref = oracle.build_index(X)
        np.testing.assert_allclose(mu, ref["mu"], rtol=1e-12, atol=1e-12)
        assert abs(float(v1.astype(np.float64) @ ref["v1"])) > 1 - 1e-5
        assert abs(np.linalg.norm(v1.astype(np.float64)) - 1) < 1e-6
        # sort: the permutation is the stable argsort of the GPU keys
        assert np.array_equal(np.sort(perm), np.arange(n))
        assert np.all(np.diff(keys) >= 0)
        # keys: exact projection with the stored fp32 v1 and mu, within E_x
        exact = (X[perm].astype(np.float64) - mu.astype(np.float32).astype(np.float64)) @ v1.astype(np.float64)
        assert np.max(np.abs(exact - keys)) <= info["key_err"]
        unsorted = np.empty(n, dtype=np.float32)
        unsorted[perm] = keys
        assert np.array_equal(np.argsort(unsorted, kind="stable"), perm)
        Xc = X[perm].astype(np.float64) - ref["mu"]
        np.testing.assert_allclose(xbar, 0.5 * np.einsum("ij,ij->i", Xc, Xc), rtol=1e-6)
        idx.free()


def test_gram_tensor_core_matches_simt(snn):
    """K2a on tcgen05 (FP16 hi/lo split, d >= 128) vs the SIMT fp32-product Gram: same v1
    to ~fp32 accuracy, identical radius results."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(8)
    d = 260
    X = (rng.standard_normal((9000, d)) * (2.0 / np.sqrt(np.arange(1, d + 1))) + 5.0).astype(np.float32)
    out = {}
    try:
        for thr in (128, 100000):
            p.snn_set_option("tc_gram_min_d", thr)
            idx = p.Index(_dev(X))
            out[thr] = idx.arrays()["v1"].cpu().numpy().astype(np.float64)
            idx.free()
    finally:
        p.snn_set_option("tc_gram_min_d", 0)
    assert abs(out[128] @ out[100000]) > 1 - 1e-8
    ref = oracle.build_index(X)["v1"]
    assert abs(out[128] @ ref) > 1 - 1e-8


def test_sort_ties_and_signed_zero(snn):
    """Many equal keys (incl. -0.0 vs +0.0) must keep ascending original id."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(5)
    n = 20000
    X = np.zeros((n, 1), dtype=np.float32)
    X[:, 0] = rng.integers(-3, 4, n).astype(np.float32)
    idx = p.Index(_dev(X))
    perm = idx.arrays()["perm"].cpu().numpy()
    assert np.array_equal(perm, np.argsort(X[:, 0], kind="stable"))
    r = idx.query_self(0.0)
    compare(r, oracle.radius_query(X, X, 0.0))
    idx.free()


# --------------------------------------------------------------------------- configs
def test_c1_full(snn):
    w = workloads.c1()
    gpu = run(snn, w.X, None, w.R)
    st = compare(gpu, oracle.radius_query(w.X, w.X, w.R))
    assert 15 < st["oracle_hits"] / w.n < 17.5


@pytest.mark.parametrize("name,kw", [("c2", dict(n=60000)), ("c3", dict(n=20000, m=2000)),
                                     ("c4", dict(n=6000, m=300)), ("c5", dict(n=40000))])
def test_scaled_configs_full_parity(snn, name, kw):
    """Same recipes at sizes the oracle finishes in seconds (several tiles + ragged tails)."""
    w = workloads.CONFIGS[name](**kw)
    R = w.R if w.R is not None else {"c2": 0.5866, "c3": 1.8134, "c4": 5.948}[name]
    gpu = run(snn, w.X, w.Q, R)
    compare(gpu, oracle.radius_query(w.X, w.queries, R))


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_full_size_sampled_parity(snn, name):
    """BASELINE.json sizes, default launch configuration; oracle on sampled queries."""
    w = workloads.CONFIGS[name]()
    gpu = run(snn, w.X, w.Q, w.R)
    rng = np.random.default_rng(0)
    k = {"c2": 400, "c3": 300, "c4": 40}[name]
    rows = np.sort(rng.choice(w.m, k, replace=False))
    ora = oracle.radius_query(w.X, w.queries[rows], w.R)
    st = compare(gpu, ora, rows_subset=rows)
    assert st["oracle_hits"] > 0
    # whole-result properties at full size
    assert gpu.offsets[0] == 0 and np.all(np.diff(gpu.offsets) >= 0)
    if w.Q is None:
        assert np.all(np.diff(gpu.offsets) >= 1)      # self-membership


# --------------------------------------------------------------------------- DBSCAN (a12)
def _gpu_dbscan(snn, X, eps, mp):
    idx = snn.Index(_dev(X))
    try:
        return idx.dbscan(eps, mp)
    finally:
        idx.free()


def test_dbscan_spec_examples_gpu(snn):
    rng = np.random.default_rng(0)
    A = np.concatenate([rng.standard_normal((500, 2)) * 0.5,
                        rng.standard_normal((500, 2)) * 0.5 + 10]).astype(np.float32)
    lab, K = _gpu_dbscan(snn, A, 1.0, 5)
    ref, Kr, _ = oracle.dbscan(A, 1.0, 5)
    assert K == Kr == 2 and np.array_equal(lab, ref)
    G = np.stack(np.meshgrid(np.arange(10) * 10.0, np.arange(10) * 10.0), -1).reshape(-1, 2).astype(np.float32)
    lab, K = _gpu_dbscan(snn, G, 0.1, 5)
    assert K == 0 and (lab == -1).all()
    lab, K = _gpu_dbscan(snn, A, 1e6, 1)
    assert K == 1 and (lab == 0).all()


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_dbscan_border_rule_gpu(snn, dt):
    """Border point within eps of cores of two clusters: it joins the first cluster the
    ascending-id FIFO scan reaches it with (cluster 0), not the cluster of its smallest-id
    core neighbour (tests/test_oracle.py hand example); both the d <= 8 pipeline and the
    CSR pipeline (d = 9: same points padded with zero coordinates)."""
    x = {0: 0.0, 7: 0.3, 8: 0.6, 9: 1.0, 1: 3.0, 2: 3.3, 3: 3.6, 4: 4.0, 5: 2.0, 6: 50.0}
    P = np.array([[x[i], 0.0] for i in range(10)], dtype=dt)
    lab, K = _gpu_dbscan(snn, P, 1.05, 4)
    assert K == 2 and lab.tolist() == [0, 1, 1, 1, 1, 0, -1, 0, 0, 0]
    P9 = np.zeros((10, 9), dtype=dt)
    P9[:, 0] = P[:, 0]
    lab, K = _gpu_dbscan(snn, P9, 1.05, 4)
    assert K == 2 and lab.tolist() == [0, 1, 1, 1, 1, 0, -1, 0, 0, 0]


@pytest.mark.parametrize("n,seed,box,eps,mp,dt", [(20000, 4, 1000.0, 3.0, 5, np.float32),
                                                  (15000, 7, 300.0, 3.0, 5, np.float32),
                                                  (8000, 9, 200.0, 2.5, 4, np.float64),
                                                  (12000, 11, 150.0, 3.0, 10, np.float32)])
def test_dbscan_full_parity(snn, n, seed, box, eps, mp, dt):
    """C5 recipe at oracle-sized n: labels equal the oracle's exactly (canonical numbering)."""
    w = workloads.c5(n=n, seed=seed, box=box)
    X = w.X.astype(dt)
    lab, K = _gpu_dbscan(snn, X, eps, mp)
    ref, Kr, _ = oracle.dbscan(X, eps, mp)
    assert K == Kr
    assert np.array_equal(lab, ref)


@pytest.mark.parametrize("n,box,dt", [(200000, 400.0, np.float32), (60000, 500.0, np.float32),
                                      (30000, 150.0, np.float64)])
def test_dbscan_core_count_modes_identical(snn, n, box, dt):
    """Core counts by one warp per point scanning outward (default) and by one CTA per
    query block over whole chunks (count_warp = -1): identical labels, equal to the grid
    oracle's (reading C18)."""
    import paper_2212_07679_b200 as p
    X = workloads.c5(n=n, seed=31, box=box).X.astype(dt)
    ref, Kr, _ = oracle.dbscan(X, 3.0, 5, grid=True)
    lab1, K1 = _gpu_dbscan(snn, X, 3.0, 5)
    try:
        p.snn_set_option("count_warp", -1)
        lab2, K2 = _gpu_dbscan(snn, X, 3.0, 5)
    finally:
        p.snn_set_option("count_warp", 0)
    assert K1 == K2 == Kr
    assert np.array_equal(lab1, ref) and np.array_equal(lab2, ref)


@pytest.mark.parametrize("n,box,d", [(200000, 400.0, 2), (60000, 500.0, 2), (40000, 60.0, 3)])
def test_dbscan_union_variants_identical(snn, n, box, d):
    """The union pass through the staged root snapshot (default: seed pass, then candidates
    behind the block, pairs j < i), candidates ahead (j > i), the chunk-major phased order,
    other chunk sizes, no / short / unbounded seed scans and the plain window_lowd union pass: identical labels, equal to the grid
    oracle's (reading C18)."""
    import paper_2212_07679_b200 as p
    X = workloads.c5(n=n, seed=41, box=box).X
    if d == 3:
        X = np.concatenate([X, np.random.default_rng(3).uniform(0, 4, (n, 1))], axis=1)
    X = X.astype(np.float32)
    ref, Kr, _ = oracle.dbscan(X, 3.0, 5, grid=True)
    variants = [{}, {"union_behind": -1}, {"union_phased": 1}, {"union_phased": 1, "union_behind": -1},
                {"union_chunk": 2048}, {"union_chunk": 64}, {"union_snap": 2}, {"union_snap": -1},
                {"union_seed": -1}, {"union_seed": 1}, {"union_seed": 1 << 20}]
    for opts in variants:
        try:
            for k, v in opts.items():
                p.snn_set_option(k, v)
            lab, K = _gpu_dbscan(snn, X, 3.0, 5)
        finally:
            for k in opts:
                p.snn_set_option(k, 0)
        assert K == Kr, opts
        assert np.array_equal(lab, ref), opts


@pytest.mark.parametrize("d,dt", [(16, np.float32), (40, np.float32), (12, np.float64)])
def test_dbscan_high_d_parity(snn, d, dt):
    """d > 8: DBSCAN over the exact self-query CSR; labels equal the oracle's."""
    rng = np.random.default_rng(d)
    centers = rng.standard_normal((6, d)) * 6
    X = np.concatenate([centers[rng.integers(0, 6, 3000)] + rng.standard_normal((3000, d)) * 0.6,
                        rng.standard_normal((300, d)) * 8]).astype(dt)
    eps = float(np.sqrt(d) * 0.55)
    lab, K = _gpu_dbscan(snn, X, eps, 6)
    ref, Kr, _ = oracle.dbscan(X, eps, 6)
    assert K == Kr and K >= 2
    assert np.array_equal(lab, ref)


def test_dbscan_c5_full_size_sampled(snn):
    """BASELINE config 5 at full size (n = 2M): sampled points checked one by one."""
    w = workloads.c5()
    lab, K = _gpu_dbscan(snn, w.X, w.R, w.dbscan_min_pts)
    assert K >= 1 and lab.max() == K - 1 and lab.min() >= -1
    rng = np.random.default_rng(1)
    ids = rng.choice(w.n, 24, replace=False)
    cnt = oracle.neighbour_counts(w.X, w.R, ids)
    X64 = w.X.astype(np.float64)
    for i, c in zip(ids, cnt):
        s = ((X64 - X64[i]) ** 2).sum(axis=1)          # candidates only; membership via oracle
        nb = np.nonzero(s <= w.R * w.R * 1.001)[0]
        res = oracle.radius_query(w.X, w.X[i:i + 1], w.R)
        nb = np.sort(res["indices"][res["s"] <= res["R2"]])
        assert len(nb) == c
        sub = nb if len(nb) <= 24 else np.concatenate([[nb.min()], rng.choice(nb, 23, replace=False)])
        nbc = oracle.neighbour_counts(w.X, w.R, sub) >= w.dbscan_min_pts
        if c >= w.dbscan_min_pts:           # core: same cluster as its core neighbours
            assert lab[i] >= 0
            assert all(lab[j] == lab[i] for j, isc in zip(sub, nbc) if isc)
        else:
            allc = oracle.neighbour_counts(w.X, w.R, nb) >= w.dbscan_min_pts
            core_nb = nb[allc]
            expect = lab[core_nb].min() if len(core_nb) else -1   # first cluster reaching it
            assert lab[i] == expect


# --------------------------------------------------------------------------- tensor-core path (a9)
@pytest.mark.parametrize("d,self_q,opts", [(3, True, {}), (2, True, {}), (3, False, {}), (5, True, {"cap": 1}),
                                           (8, False, {"cap": 2, "ovf_records": 40}), (1, True, {}),
                                           (3, True, {"chunk": 1024}), (4, True, {"symmetric": -1})])
def test_scan2q_identical(snn, d, self_q, opts):
    """K8 scan with two queries per thread (option scan2q; default for d >= 2) vs one: bit-identical CSR, equal
    to the oracle; symmetric / two-sided self-queries, separate queries, slot overflow and
    the overflow-list limit (fix pass)."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(900 + d)
    X = (rng.random((30000, d)) * 10).astype(np.float32)
    Q = None if self_q else (rng.random((7001, d)) * 10).astype(np.float32)
    R = {1: 0.002, 2: 0.05, 3: 0.25, 4: 0.6, 5: 1.0, 8: 2.5}[d]
    outs = []
    try:
        for k, v in opts.items():
            p.snn_set_option(k, v)
        for v in (-1, 1):
            p.snn_set_option("scan2q", v)
            outs.append(run(snn, X, Q, R))
        p.snn_set_option("chunk2q", 128)   # many items per block, ragged last chunk
        outs.append(run(snn, X, Q, R))
    finally:
        for k in list(opts) + ["scan2q", "chunk2q"]:
            p.snn_set_option(k, 0)
    compare(outs[1], oracle.radius_query(X, X if self_q else Q, R))
    for f in ("offsets", "indices", "distances"):
        np.testing.assert_array_equal(np.asarray(getattr(outs[1], f)), np.asarray(getattr(outs[0], f)))
        np.testing.assert_array_equal(np.asarray(getattr(outs[2], f)), np.asarray(getattr(outs[0], f)))


def test_tc_and_generic_paths_agree_exactly(snn):
    """Same data through the tcgen05 TF32 filter and the SIMT generic kernel."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(77)
    X = (rng.standard_normal((5000, 40)) * np.linspace(2, 0.2, 40)).astype(np.float32)
    Q = (rng.standard_normal((900, 40)) * np.linspace(2, 0.2, 40)).astype(np.float32)
    R = 2.2
    a = run(snn, X, Q, R)
    try:
        p.snn_set_option("tc", -1)
        b = run(snn, X, Q, R)
    finally:
        p.snn_set_option("tc", 0)
    ora = oracle.radius_query(X, Q, R)
    compare(a, ora)
    compare(b, ora)
    assert np.array_equal(a.offsets, b.offsets)


@pytest.mark.parametrize("f16", [1, -1])
@pytest.mark.parametrize("d", [32, 48, 96])
def test_tc_clustered_far_from_origin(snn, d, f16):
    """Tight clusters far from the origin and from each other: |x - mu| >> R, so the
    expanded form cancels heavily; the margin must keep every true neighbour (FP16 and
    TF32 operands)."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(d)
    centers = rng.standard_normal((6, d)) * 50 + 300
    lab = rng.integers(0, 6, 6000)
    X = (centers[lab] + rng.standard_normal((6000, d)) * 0.05).astype(np.float32)
    R = float(0.05 * np.sqrt(2 * d))           # ~ typical within-cluster distance
    try:
        p.snn_set_option("tc_f16", f16)
        gpu = run(snn, X, X[:700], R)
    finally:
        p.snn_set_option("tc_f16", 0)
    compare(gpu, oracle.radius_query(X, X[:700], R))


@pytest.mark.parametrize("xs,qs", [(1e-25, 1e-25), (1.0, 1e25), (1e15, 1e15), (1.0, 1e-30)])
def test_tc_operand_scaling_extremes(snn, xs, qs):
    """FP16 operands are scaled by powers of two; magnitudes outside the scalable range
    (index or queries) fall back to TF32 / the generic kernel -- results stay exact."""
    rng = np.random.default_rng(11)
    X = (rng.standard_normal((3000, 40)) * xs).astype(np.float32)
    Q = (rng.standard_normal((300, 40)) * qs).astype(np.float32)
    Q[:50] = X[:50]
    R = float(np.sqrt(2 * 40) * max(xs, qs) * 0.9)
    compare(run(snn, X, Q, R), oracle.radius_query(X, Q, R))


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 8])
def test_lowd_tensor_core_vs_ffma_exact(snn, d):
    """Low-d radius query through the folded split-FP16 tcgen05 filter (K = 16 / 32) and
    through the FFMA direct-form kernel: bit-identical CSR, and equal to the oracle."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(100 + d)
    centers = rng.random((16, d)) * 50 + 1000.0           # far from the origin: cancellation
    X = (centers[rng.integers(0, 16, 12000)] + rng.standard_normal((12000, d))).astype(np.float32)
    Q = np.concatenate([X[:1500], (X[1500:2500] + rng.standard_normal((1000, d)) * 0.3).astype(np.float32)])
    R = 0.9
    ora = oracle.radius_query(X, Q, R)
    res = {}
    try:
        for tc in (1, -1):
            p.snn_set_option("lowd_tc", tc)
            res[tc] = (run(snn, X, Q, R), run(snn, X, None, R))
    finally:
        p.snn_set_option("lowd_tc", 0)
    for tc in (1, -1):
        compare(res[tc][0], ora)
    a, b = res[1][0], res[-1][0]
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.distances, b.distances)
    a, b = res[1][1], res[-1][1]
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.indices, b.indices)


@pytest.mark.parametrize("d", [1, 2, 3, 5, 8])
def test_simt_expanded_filter_vs_direct_exact(snn, d):
    """Low-d scan with the expanded-form fp32 pre-filter (eq:ip2 with the rigorous margin)
    vs the plain direct-form scan: bit-identical CSR and DBSCAN labels, equal to the oracle."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(200 + d)
    centers = rng.random((12, d)) * 40 + 3000.0            # far from the origin: cancellation
    X = (centers[rng.integers(0, 12, 15000)] + rng.standard_normal((15000, d))).astype(np.float32)
    Q = np.concatenate([X[:1000], (X[1000:2000] + rng.standard_normal((1000, d)) * 0.5).astype(np.float32)])
    R = 0.8
    res = {}
    try:
        for f in (1, -1):
            p.snn_set_option("simt_filter", f)
            idx = p.Index(_dev(X))
            lab, k = idx.dbscan(R, 4)
            res[f] = (idx.query(_dev(Q), R), idx.query_self(R), lab, k)
            idx.free()
    finally:
        p.snn_set_option("simt_filter", 0)
    compare(res[1][0], oracle.radius_query(X, Q, R))
    for i in (0, 1):
        a, b = res[1][i], res[-1][i]
        assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.indices, b.indices)
        assert np.array_equal(a.distances, b.distances)
    assert res[1][3] == res[-1][3] and np.array_equal(res[1][2], res[-1][2])


@pytest.mark.parametrize("d,dt,R", [(1, np.float32, 0.002), (2, np.float32, 0.02), (3, np.float32, 0.6),
                                    (3, np.float64, 0.6), (8, np.float32, 1.5), (2, np.float32, 0.0)])
def test_symmetric_self_query_identical(snn, d, dt, R):
    """Self-query with each unordered pair evaluated once (mirrored L rows, sorted) vs the
    two-sided scan: bit-identical CSR (key order, distances), equal to the oracle."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(300 + d)
    centers = rng.random((10, d)) * 30
    X = (centers[rng.integers(0, 10, 9000)] + rng.standard_normal((9000, d))).astype(dt)
    X[100:140] = X[0]                                     # duplicates (R = 0 hits)
    res = {}
    try:
        for f in (1, -1):
            p.snn_set_option("symmetric", f)
            res[f] = run(snn, X, None, R)
    finally:
        p.snn_set_option("symmetric", 0)
    a, b = res[1], res[-1]
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.distances, b.distances)
    compare(a, oracle.radius_query(X, X, R))


@pytest.mark.parametrize("d,n", [(3, 20000), (2, 30000), (64, 6000)])
def test_everything_is_a_neighbour(snn, d, n):
    """R larger than the data diameter: every row holds all n points (slot overflow, lost
    entries and the fix pass, the symmetric path's huge-row fallback, pair-list capacity
    retries); rows in key order, distances exact."""
    rng = np.random.default_rng(d)
    X = rng.random((n, d)).astype(np.float32)
    R = float(np.sqrt(d)) * 2.0
    res = run(snn, X, None, R)
    assert np.array_equal(np.diff(res.offsets), np.full(n, n))
    for r in (0, n // 2, n - 1):   # each row: a permutation of all points, exact distances
        ids = res.indices[res.offsets[r]:res.offsets[r + 1]]
        assert np.array_equal(np.sort(ids), np.arange(n))
        dd = np.sqrt(((X[ids].astype(np.float64) - X[r].astype(np.float64)) ** 2).sum(axis=1)).astype(np.float32)
        assert np.array_equal(res.distances[res.offsets[r]:res.offsets[r + 1]], dd)


@pytest.mark.parametrize("tiles,group", [(1, 1), (3, 2), (8, 8), (16, 64)])
def test_lowd_tensor_core_raster_options(snn, tiles, group):
    import paper_2212_07679_b200 as p
    w = workloads.c2(n=30000)
    R = workloads.load_radii()["c2"]["R"]
    ora = oracle.radius_query(w.X, w.X[:3000], R)
    try:
        p.snn_set_option("lowd_tc_tiles", tiles)
        p.snn_set_option("lowd_tc_group", group)
        compare(run(snn, w.X, w.X[:3000], R), ora)
    finally:
        p.snn_set_option("lowd_tc_tiles", 0)
        p.snn_set_option("lowd_tc_group", 0)


@pytest.mark.parametrize("d", [3, 64])
def test_window_all_ablation_identical(snn, d):
    """'Brute force 2' ablation (window = every point): identical CSR."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(d)
    X = rng.standard_normal((6000, d)).astype(np.float32)
    Q = rng.standard_normal((700, d)).astype(np.float32)
    R = float(np.sqrt(d)) * 0.6
    a = run(snn, X, Q, R)
    try:
        p.snn_set_option("window_all", 1)
        b = run(snn, X, Q, R)
    finally:
        p.snn_set_option("window_all", 0)
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.distances, b.distances)


@pytest.mark.parametrize("nbig", [300, 3000, 20000])
def test_tc_csr_row_sizes(snn, nbig):
    """Rows of every size class of the CSR row sort (registers <= 32, warp <= 512,
    CTA <= 16384, global radix fallback beyond): a dense blob plus scattered points."""
    rng = np.random.default_rng(nbig)
    d = 32
    X = np.concatenate([rng.standard_normal((nbig, d)) * 0.01,
                        rng.standard_normal((4000, d)) * 3.0]).astype(np.float32)
    Q = np.concatenate([X[:5], X[-200:], rng.standard_normal((50, d)).astype(np.float32) * 0.01])
    R = 1.0
    compare(run(snn, X, Q, R), oracle.radius_query(X, Q, R))


@pytest.mark.parametrize("group", [1, 3, 32])
def test_tc_raster_groups(snn, group):
    """Grouped raster order of the (query block, chunk) items, incl. empty items."""
    import paper_2212_07679_b200 as p
    w = workloads.c3(n=12000, m=1300)
    ora = oracle.radius_query(w.X, w.Q, 1.8134)
    try:
        p.snn_set_option("tc_group", group)
        p.snn_set_option("tc_tiles", 2)
        compare(run(snn, w.X, w.Q, 1.8134), ora)
    finally:
        p.snn_set_option("tc_group", 0)
        p.snn_set_option("tc_tiles", 0)


def test_tc_tile_edges_and_tiles_option(snn):
    """m and n not multiples of the 128 x 256 tile; several tiles-per-item settings."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(5)
    X = rng.standard_normal((4097, 64)).astype(np.float32)
    Q = rng.standard_normal((129, 64)).astype(np.float32)
    ora = oracle.radius_query(X, Q, 9.5)
    try:
        for f16 in (1, -1):
            p.snn_set_option("tc_f16", f16)
            for ares in (1, -1):
                p.snn_set_option("tc_ares", ares)
                for tiles in (1, 3, 8):
                    p.snn_set_option("tc_tiles", tiles)
                    compare(run(snn, X, Q, 9.5), ora)
    finally:
        p.snn_set_option("tc_tiles", 0)
        p.snn_set_option("tc_f16", 0)
        p.snn_set_option("tc_ares", 0)


# --------------------------------------------------------------------------- metrics (f3)
def _metric_compare(gpu, ora, metric):
    """Row sets identical (ids sorted per row) and distances equal to the oracle's metric
    value of float32(sqrt(s)): cosine bit for bit (fp64 e^2/2 on both sides), angular
    within 1 float32 ulp (device vs libm asin)."""
    g_off, o_off = np.asarray(gpu.offsets), np.asarray(ora["offsets"])
    np.testing.assert_array_equal(g_off, o_off)
    g_idx, g_d = np.asarray(gpu.indices), np.asarray(gpu.distances)
    rows = np.repeat(np.arange(len(g_off) - 1), np.diff(g_off))
    order = np.lexsort((g_idx, rows))
    np.testing.assert_array_equal(g_idx[order], ora["indices"])
    if metric == "cosine":
        np.testing.assert_array_equal(g_d[order], ora["dist"])
    else:
        np.testing.assert_array_max_ulp(g_d[order], ora["dist"], maxulp=1)


@pytest.mark.parametrize("metric", ["cosine", "angular"])
@pytest.mark.parametrize("n,m,d,dt", [(3000, 400, 3, np.float32), (2000, 300, 3, np.float64),
                                      (1500, 200, 8, np.float32), (900, 120, 64, np.float32),
                                      (600, 70, 33, np.float64)])
def test_metric_query_parity(snn, metric, n, m, d, dt):
    rng = np.random.default_rng(700 + d)
    X = (rng.standard_normal((n, d)) + 0.3).astype(dt)
    Q = (rng.standard_normal((m, d)) + 0.3).astype(dt)
    # radius at a small quantile of the metric over a sample
    U, V = oracle.normalize_rows(X[:300]).astype(np.float64), oracle.normalize_rows(Q[:40]).astype(np.float64)
    cosd = 1.0 - V @ U.T
    q = float(np.quantile(cosd, 0.02))
    r = q if metric == "cosine" else float(np.arccos(1.0 - q))
    idx = snn.Index(_dev(X), metric=metric)
    try:
        assert idx.info()["metric"] == oracle.METRICS[metric]
        gpu = idx.query(_dev(Q), r)
        ora = oracle.metric_radius_query(X, Q, r, metric)
        assert ora["offsets"][-1] > m
        _metric_compare(gpu, ora, metric)
        gpu_h = idx.query(Q, r)                  # host queries (normalized on the device)
        _metric_compare(gpu_h, ora, metric)
        gs = idx.query_self(r)
        _metric_compare(gs, oracle.metric_radius_query(X, X, r, metric), metric)
    finally:
        idx.free()


@pytest.mark.parametrize("metric,d", [("cosine", 3), ("angular", 3), ("cosine", 40)])
def test_metric_dbscan_parity(snn, metric, d):
    rng = np.random.default_rng(800 + d)
    if d <= 3:
        X = (rng.standard_normal((3000, d)) + 0.2).astype(np.float32)
        eps = 0.004 if metric == "cosine" else 0.09
    else:                                        # 10 directional clusters + 100 outliers
        C = rng.standard_normal((10, d))
        X = np.concatenate([C[rng.integers(0, 10, 2900)] + 0.3 * rng.standard_normal((2900, d)),
                            rng.standard_normal((100, d))]).astype(np.float32)
        eps = 0.1
    idx = snn.Index(_dev(X), metric=metric)
    try:
        labels, K = idx.dbscan(eps, 5)
    finally:
        idx.free()
    lab, K_o, _ = oracle.dbscan(oracle.normalize_rows(X), oracle.metric_radius(metric, eps), 5)
    assert K == K_o and K > 1
    np.testing.assert_array_equal(labels, lab)


def test_metric_errors(snn):
    X = np.ones((100, 4), dtype=np.float32)
    X[50] = 0.0
    with pytest.raises(snn.SnnError, match="INVALID_ARGUMENT"):
        snn.Index(_dev(X), metric="cosine")
    X[50] = 1.0
    idx = snn.Index(_dev(X), metric="angular")
    try:
        Q = np.zeros((3, 4), dtype=np.float32)
        with pytest.raises(snn.SnnError, match="INVALID_ARGUMENT"):
            idx.query(_dev(Q), 0.1)
        with pytest.raises(snn.SnnError, match="INVALID_ARGUMENT"):
            idx.query_self(-0.1)
        gs = idx.query_self(4.0)                  # alpha >= pi: every pair
        assert int(np.asarray(gs.offsets)[-1]) == 100 * 100
    finally:
        idx.free()
    with pytest.raises(snn.SnnError, match="INVALID_ARGUMENT"):
        snn.snn_build_metric(_dev(X), 7)


def _filtered_compare(gpu, ora):
    """Rows identical (ids sorted per row), values bit-identical (fp64 left-to-right sum on
    both sides, rounded to float32)."""
    g_off = np.asarray(gpu.offsets)
    np.testing.assert_array_equal(g_off, ora["offsets"])
    g_idx, g_d = np.asarray(gpu.indices), np.asarray(gpu.distances)
    rows = np.repeat(np.arange(len(g_off) - 1), np.diff(g_off))
    order = np.lexsort((g_idx, rows))
    np.testing.assert_array_equal(g_idx[order], ora["indices"])
    np.testing.assert_array_equal(g_d[order], ora["dist"])


@pytest.mark.parametrize("n,m,d,dt", [(3000, 300, 2, np.float32), (2000, 200, 3, np.float64),
                                      (1200, 100, 8, np.float32), (800, 80, 40, np.float32)])
def test_manhattan_parity(snn, n, m, d, dt):
    rng = np.random.default_rng(900 + d)
    X = (rng.standard_normal((n, d)) * rng.uniform(0.5, 2, d)).astype(dt)
    Q = (rng.standard_normal((m, d)) * rng.uniform(0.5, 2, d)).astype(dt)
    L1 = np.abs(X[:300, None, :].astype(np.float64) - Q[None, :30, :]).sum(-1)
    R = float(np.quantile(L1, 0.03))
    idx = snn.Index(_dev(X), metric="manhattan")
    try:
        _filtered_compare(idx.query(_dev(Q), R), oracle.manhattan_query(X, Q, R))
        _filtered_compare(idx.query(Q, R), oracle.manhattan_query(X, Q, R))
        _filtered_compare(idx.query_self(R), oracle.manhattan_query(X, X, R))
        with pytest.raises(snn.SnnError, match="UNSUPPORTED"):
            idx.dbscan(R, 5)
    finally:
        idx.free()


@pytest.mark.parametrize("n,m,d,dt", [(3000, 300, 3, np.float32), (2000, 200, 5, np.float64),
                                      (1000, 100, 64, np.float32)])
def test_inner_product_parity(snn, n, m, d, dt):
    rng = np.random.default_rng(950 + d)
    X = (rng.standard_normal((n, d)) * rng.uniform(0.2, 2, (n, 1))).astype(dt)
    Q = rng.standard_normal((m, d)).astype(dt)
    G = Q[:30].astype(np.float64) @ X[:300].T.astype(np.float64)
    tau = float(np.quantile(G, 0.97))
    idx = snn.Index(_dev(X), metric="mips")
    try:
        assert idx.info()["d"] == d + 1
        ora = oracle.inner_product_query(X, Q, tau)
        assert ora["offsets"][-1] > m
        _filtered_compare(idx.query(_dev(Q), tau), ora)
        _filtered_compare(idx.query_self(tau), oracle.inner_product_query(X, X, tau))
        # negative threshold: far more pairs, still exact
        t2 = float(np.quantile(G, 0.6))
        _filtered_compare(idx.query(_dev(Q[:20]), t2), oracle.inner_product_query(X, Q[:20], t2))
        # threshold above every product: empty
        big = float(np.abs(G).max() * 10 + 10)
        assert int(np.asarray(idx.query(_dev(Q), big).offsets)[-1]) == 0
    finally:
        idx.free()


# --------------------------------------------------------------------------- streaming append + save/load (f4)
def _csr_equal(a, b):
    np.testing.assert_array_equal(np.asarray(a.offsets), np.asarray(b.offsets))
    np.testing.assert_array_equal(np.asarray(a.indices), np.asarray(b.indices))
    np.testing.assert_array_equal(np.asarray(a.distances).view(np.uint32), np.asarray(b.distances).view(np.uint32))


def _check_key_order(idx):
    arr = idx.arrays()
    keys, perm = arr["keys"].cpu().numpy(), arr["perm"].cpu().numpy()
    assert np.all(np.diff(keys) >= 0)
    np.testing.assert_array_equal(np.sort(perm), np.arange(idx.n))
    ties = np.diff(keys) == 0
    assert np.all(np.diff(perm)[ties] > 0), "equal keys not ordered by original id"


@pytest.mark.parametrize("d,dt", [(2, np.float32), (3, np.float64), (8, np.float32), (20, np.float32),
                                  (64, np.float32), (40, np.float64), (130, np.float32)])
def test_append_parity(snn, d, dt):
    """Append in batches (mu, v1 frozen) == brute force on the grown data."""
    rng = np.random.default_rng(1000 + d)
    X0 = (rng.standard_normal((3000, d)) * rng.uniform(0.5, 2, d)).astype(dt)
    B1 = (rng.standard_normal((700, d)) * rng.uniform(0.5, 2, d) + 0.5).astype(dt)
    B2 = np.concatenate([X0[5:6], X0[:3] * 1.0001, 8 * rng.standard_normal((10, d))]).astype(dt)  # twin, near twins, outliers
    B3 = (rng.standard_normal((1, d))).astype(dt)
    Q = (rng.standard_normal((300, d)) * rng.uniform(0.5, 2, d)).astype(dt)
    R = float(np.quantile(np.linalg.norm(X0[:200, None, :].astype(np.float64) - Q[None, :40, :], axis=-1), 0.03))
    idx = snn.Index(_dev(X0))
    try:
        idx.append(_dev(B1))
        idx.append(B2)                         # host rows
        idx.append(_dev(B3))
        idx.append(_dev(B3[:0]))               # k = 0: no-op
        X = np.concatenate([X0, B1, B2, B3])
        assert idx.n == len(X)
        _check_key_order(idx)
        compare(idx.query(_dev(Q), R), oracle.radius_query(X, Q, R))
        compare(idx.query_self(R), oracle.radius_query(X, X, R))
        z = idx.query(_dev(X[[5, 3000 + 700]]), 0.0)      # the appended twin of row 5
        assert {5, 3700} <= set(np.asarray(z.indices)[: np.asarray(z.offsets)[1]].tolist())
    finally:
        idx.free()


def test_append_spec_examples(snn):
    """SPEC append_point examples: D3 + (9,12) -> alpha (-5, 0, 5, 10), new id 3 at
    sorted position 3; a duplicate is found with R = 0; a single-point index grows to n = 2."""
    idx = snn.Index(np.array([[0, 0], [3, 4], [6, 8]], dtype=np.float64))
    try:
        idx.append(np.array([[9, 12]], dtype=np.float64))
        arr = idx.arrays()
        np.testing.assert_allclose(arr["keys"].cpu().numpy(), [-5, 0, 5, 10], atol=1e-5)
        np.testing.assert_array_equal(arr["perm"].cpu().numpy(), [0, 1, 2, 3])
        idx.append(np.array([[3, 4]], dtype=np.float64))
        r = idx.query(np.array([[3, 4]], dtype=np.float64), 0.0)
        assert sorted(np.asarray(r.indices).tolist()) == [1, 4]
    finally:
        idx.free()
    one = snn.Index(np.array([[7, 7]], dtype=np.float32))
    try:
        one.append(np.array([[1, 2]], dtype=np.float32))
        assert one.n == 2
        _check_key_order(one)
        r = one.query_self(10.0)
        assert int(np.asarray(r.offsets)[-1]) == 4
    finally:
        one.free()


def test_append_metrics_and_errors(snn):
    rng = np.random.default_rng(1100)
    X0 = (rng.standard_normal((2000, 3)) + 0.3).astype(np.float32)
    B = (rng.standard_normal((500, 3)) + 0.3).astype(np.float32)
    Q = (rng.standard_normal((200, 3)) + 0.3).astype(np.float32)
    X = np.concatenate([X0, B])
    idx = snn.Index(_dev(X0), metric="cosine")
    try:
        idx.append(_dev(B))
        _metric_compare(idx.query(_dev(Q), 0.002), oracle.metric_radius_query(X, Q, 0.002, "cosine"), "cosine")
        bad = B[:2].copy()
        bad[1, 0] = np.nan
        before = idx.query(_dev(Q), 0.002)
        with pytest.raises(snn.SnnError, match="INVALID_ARGUMENT|NONFINITE"):
            idx.append(_dev(bad))
        assert idx.n == len(X)
        _csr_equal(before, idx.query(_dev(Q), 0.002))   # unchanged
        with pytest.raises(snn.SnnError, match="DIM_MISMATCH"):
            idx.append(_dev(np.ones((2, 4), dtype=np.float32)))
    finally:
        idx.free()
    man = snn.Index(_dev(X0), metric="manhattan")
    try:
        man.append(B)
        _filtered_compare(man.query(_dev(Q), 0.3), oracle.manhattan_query(X, Q, 0.3))
    finally:
        man.free()
    mips = snn.Index(_dev(X0), metric="mips")
    try:
        with pytest.raises(snn.SnnError, match="UNSUPPORTED"):
            mips.append(_dev(B))
    finally:
        mips.free()
    plain = snn.Index(_dev(X0))
    try:
        bad = B[:3].copy()
        bad[2, 1] = np.inf
        with pytest.raises(snn.SnnError, match="NONFINITE"):
            plain.append(_dev(bad))
        assert plain.n == len(X0)
    finally:
        plain.free()


@pytest.mark.parametrize("metric,d,dt", [("euclidean", 3, np.float32), ("euclidean", 2, np.float64),
                                         ("euclidean", 20, np.float32), ("euclidean", 64, np.float32),
                                         ("cosine", 3, np.float32), ("manhattan", 4, np.float32),
                                         ("mips", 8, np.float64)])
def test_save_load_roundtrip(snn, tmp_path, metric, d, dt):
    """Loaded index answers bit-identically; save -> load -> save writes identical bytes."""
    rng = np.random.default_rng(1200 + d)
    X = (rng.standard_normal((2500, d)) + 0.2).astype(dt)
    Q = (rng.standard_normal((200, d)) + 0.2).astype(dt)
    r = {"euclidean": 0.4 if d <= 3 else 4.0, "cosine": 0.002, "manhattan": 0.6, "mips": 6.0}[metric]
    a = snn.Index(_dev(X), metric=metric)
    p1, p2 = str(tmp_path / "a.snn"), str(tmp_path / "b.snn")
    try:
        a.save(p1)
        b = snn.Index.load(p1)
        try:
            assert (b.n, b.d, b.metric) == (a.n, a.d, metric)
            _csr_equal(a.query(_dev(Q), r), b.query(_dev(Q), r))
            _csr_equal(a.query_self(r), b.query_self(r))
            if metric in ("euclidean", "cosine"):
                la, ka = a.dbscan(r, 4)
                lb, kb = b.dbscan(r, 4)
                assert ka == kb
                np.testing.assert_array_equal(la, lb)
            b.save(p2)
        finally:
            b.free()
        assert open(p1, "rb").read() == open(p2, "rb").read()
    finally:
        a.free()


def test_load_rejects_broken_invariants(snn, tmp_path):
    X = np.random.default_rng(1300).standard_normal((100, 3)).astype(np.float32)
    a = snn.Index(_dev(X))
    p = str(tmp_path / "a.snn")
    try:
        a.save(p)
    finally:
        a.free()
    blob = bytearray(open(p, "rb").read())
    head = 8 + 8 * 23
    off_keys = head + 3 * 8 + 3 * 4 + 3 * 8 + 3 * 4 + 10 * 8 + 3 * 3 * 8   # mu_d mu_f v_d v_f stats G
    off_perm = off_keys + 100 * 4
    bad = bytearray(blob)
    bad[off_perm:off_perm + 4] = bad[off_perm + 4:off_perm + 8]   # duplicate id
    open(p, "wb").write(bad)
    with pytest.raises(snn.SnnError, match="permutation"):
        snn.Index.load(p)
    bad = bytearray(blob)
    bad[off_keys:off_keys + 4] = np.float32(1e30).tobytes()       # first key too large
    open(p, "wb").write(bad)
    with pytest.raises(snn.SnnError, match="sorted"):
        snn.Index.load(p)
    open(p, "wb").write(blob + b"\0")
    with pytest.raises(snn.SnnError, match="trailing"):
        snn.Index.load(p)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_load_rewrites_padding_sentinels(snn, tmp_path, dt):
    """A file whose padding rows [n, n_pad) hold finite values (here: the origin, right next
    to the queries) loads to an index that answers exactly like the saved one: snn_load
    rewrites the sentinels the kernels rely on instead of trusting the file."""
    rng = np.random.default_rng(1301)
    n, d = 4097, 2                        # n_pad = 4100: three padding rows
    X = (rng.random((n, d)) - 0.5).astype(dt)
    Q = (rng.random((50, d)) * 0.02 - 0.01).astype(dt)
    a = snn.Index(_dev(X))
    p = str(tmp_path / "a.snn")
    try:
        a.save(p)
        ref_q, ref_s = a.query(_dev(Q), 0.05), a.query_self(0.05)
    finally:
        a.free()
    blob = bytearray(open(p, "rb").read())
    es, npad = np.dtype(dt).itemsize, 4100
    xf = npad * (d + 1) * 4 if dt == np.float32 else 0        # filter rows (low-d fp32) follow Xs
    xs0 = len(blob) - xf - npad * d * es
    g = n >> 2
    for r in range(n & 3, 4):
        for k in range(d):
            o = xs0 + (g * 4 * d + 4 * k + r) * es
            blob[o:o + es] = np.zeros(1, dt).tobytes()         # finite padding coordinates
            if xf:
                o = xs0 + npad * d * es + (g * 4 * (d + 1) + 4 * k + r) * 4
                blob[o:o + 4] = np.float32(0).tobytes()
        if xf:
            o = xs0 + npad * d * es + (g * 4 * (d + 1) + 4 * d + r) * 4
            blob[o:o + 4] = np.float32(0).tobytes()            # xbar' 0 instead of +inf
    open(p, "wb").write(bytes(blob))
    b = snn.Index.load(p)
    try:
        _csr_equal(ref_q, b.query(_dev(Q), 0.05))
        _csr_equal(ref_s, b.query_self(0.05))
    finally:
        b.free()


@pytest.mark.parametrize("d", [2, 3, 6])
def test_row_staging_and_symmetry_options_identical(snn, d):
    """Direct final-row writes (default) vs key-order row staging, symmetric vs two-sided
    self-queries, expanded filter on/off, balanced vs per-entry compaction, pipelined vs
    warp-per-row L-segment finalize: bit-identical CSR, equal to the oracle."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(1400 + d)
    X = (rng.random((20000, d)) * 20).astype(np.float32)
    R = {2: 0.12, 3: 0.5, 6: 2.5}[d]
    outs = []
    try:
        for st, sy, sf, bc, fp in [(1, 1, 0, 0, 0), (-1, 1, 0, 0, 0), (1, -1, 0, 0, 0), (-1, -1, -1, 0, 0),
                                   (1, 1, -1, 0, 0), (1, 1, 0, -1, 0), (-1, 1, -1, -1, 0), (-1, 1, 0, 0, -1)]:
            p.snn_set_option("stage_rows", st)
            p.snn_set_option("symmetric", sy)
            p.snn_set_option("simt_filter", sf)
            p.snn_set_option("balanced_compact", bc)
            p.snn_set_option("finalize_pipe", fp)
            outs.append(run(snn, X, None, R))
    finally:
        for k in ("stage_rows", "symmetric", "simt_filter", "balanced_compact", "finalize_pipe"):
            p.snn_set_option(k, 0)
    compare(outs[0], oracle.radius_query(X, X, R))
    for o in outs[1:]:
        np.testing.assert_array_equal(np.asarray(o.offsets), np.asarray(outs[0].offsets))
        np.testing.assert_array_equal(np.asarray(o.indices), np.asarray(outs[0].indices))
        np.testing.assert_array_equal(np.asarray(o.distances), np.asarray(outs[0].distances))


def test_finalize_row_size_classes(snn):
    """Symmetric self-query L segments of every size class of the finalize (rank sort <= 64
    entries in the pipelined kernel, shared-memory bitonic <= 512, CTA sort beyond): dense
    blobs of 20 / 50 / 300 / 3000 points plus scattered points; the pipelined and the
    warp-per-row finalize give bit-identical CSRs, equal to the oracle."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(1451)
    parts = [rng.random((9000, 3)) * 40.0]
    for k, c in zip((20, 50, 300, 3000), ((5, 5, 5), (15, 15, 15), (25, 25, 25), (35, 35, 35))):
        parts.append(np.asarray(c) + rng.standard_normal((k, 3)) * 0.05)
    X = np.concatenate(parts).astype(np.float32)
    X = X[rng.permutation(len(X))]
    R = 0.4
    outs = []
    try:
        for fp in (0, -1):
            p.snn_set_option("finalize_pipe", fp)
            outs.append(run(snn, X, None, R))
    finally:
        p.snn_set_option("finalize_pipe", 0)
    assert np.diff(outs[0].offsets).max() >= 3000
    compare(outs[0], oracle.radius_query(X, X, R))
    for a, b in zip((outs[1].offsets, outs[1].indices, outs[1].distances),
                    (outs[0].offsets, outs[0].indices, outs[0].distances)):
        np.testing.assert_array_equal(np.asarray(a), np.asarray(b))


# --------------------------------------------------------------------------- query sharding (§8(e))
@pytest.mark.parametrize("d,dt,self_q,nparts", [(3, np.float32, True, 3), (2, np.float64, False, 4),
                                                (64, np.float32, False, 3), (20, np.float64, True, 2),
                                                (3, np.float32, False, 8)])
def test_query_parts_partition_the_result(snn, d, dt, self_q, nparts):
    """snn_query_*_part: every row is computed by exactly one part, the parts' rows equal the
    unpartitioned result (and the oracle), and the work split is balanced."""
    rng = np.random.default_rng(1500 + d)
    X = (rng.standard_normal((6000, d)) * rng.uniform(0.5, 2, d)).astype(dt)
    Q = None if self_q else (rng.standard_normal((6000, d)) * rng.uniform(0.5, 2, d)).astype(dt)
    R = float(np.quantile(np.linalg.norm(X[:300, None, :].astype(np.float64) - X[None, 300:400, :], axis=-1), 0.02))
    idx = snn.Index(_dev(X))
    try:
        full = idx.query_self(R) if self_q else idx.query(_dev(Q), R)
        parts = [idx.query_self(R, part=p, nparts=nparts) if self_q else idx.query(_dev(Q), R, part=p, nparts=nparts)
                 for p in range(nparts)]
        with pytest.raises(snn.SnnError, match="INVALID_ARGUMENT"):
            idx.query_self(R, part=nparts, nparts=nparts)
    finally:
        idx.free()
    m = len(np.asarray(full.offsets)) - 1
    lens = np.stack([np.diff(np.asarray(p.offsets)) for p in parts])
    full_len = np.diff(np.asarray(full.offsets))
    assert ((lens > 0).sum(axis=0) <= 1).all(), "a row computed by two parts"
    np.testing.assert_array_equal(lens.sum(axis=0), full_len)
    for p in parts:
        off = np.asarray(p.offsets)
        for r in np.nonzero(np.diff(off))[0]:
            np.testing.assert_array_equal(np.asarray(p.indices)[off[r]:off[r + 1]],
                                          np.asarray(full.indices)[full.offsets[r]:full.offsets[r + 1]])
            np.testing.assert_array_equal(np.asarray(p.distances)[off[r]:off[r + 1]],
                                          np.asarray(full.distances)[full.offsets[r]:full.offsets[r + 1]])
    totals = lens.sum(axis=1)
    assert totals.min() > 0 and totals.max() < 3 * totals.mean()
    compare(full, oracle.radius_query(X, X if self_q else Q, R))


@pytest.mark.parametrize("d,dt,nparts,opts", [(2, np.float32, 8, {}), (3, np.float64, 5, {}),
                                               (3, np.float32, 4, {"stage_rows": 1}),
                                               (3, np.float32, 3, {"balanced_compact": -1, "cap": 1, "ovf_records": 50}),
                                               (6, np.float32, 2, {"finalize_order": -1})])
def test_symmetric_query_parts(snn, d, dt, nparts, opts):
    """Partitioned SYMMETRIC self-queries (each unordered pair evaluated once, SURVEY.md
    §8(e)): every part owns a contiguous key range of rows; ghost blocks before it supply
    the mirrored entries of its rows.  The parts' rows are disjoint and bit-identical to the
    unpartitioned result, and together they evaluate about half the pairs of two-sided parts
    (under the staging / compaction / overflow-fix variants too)."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(1550 + d + nparts)
    n = 40000
    X = (rng.random((n, d)) * 30).astype(dt)
    R = {2: 0.15, 3: 0.6, 6: 4.0}[d]
    idx = snn.Index(_dev(X))

    def pairs_of(fn):
        p.snn_profile_enable(True)
        out = fn()
        pe = p.snn_profile_read("window_count")["units"]
        p.snn_profile_enable(False)
        return out, pe
    try:
        for k, v in opts.items():
            p.snn_set_option(k, v)
        full = idx.query_self(R)
        parts, pe_sym = [], 0.0
        for q in range(nparts):
            r, pe = pairs_of(lambda: idx.query_self(R, part=q, nparts=nparts))
            parts.append(r)
            pe_sym += pe
        p.snn_set_option("symmetric", -1)
        pe_two = sum(pairs_of(lambda: idx.query_self(R, part=q, nparts=nparts))[1] for q in range(nparts))
    finally:
        for k in list(opts) + ["symmetric"]:
            p.snn_set_option(k, 0)
        idx.free()
    lens = np.stack([np.diff(np.asarray(q.offsets)) for q in parts])
    assert ((lens > 0).sum(axis=0) == 1).all(), "every row in exactly one part (self is a neighbour)"
    np.testing.assert_array_equal(lens.sum(axis=0), np.diff(np.asarray(full.offsets)))
    for q in parts:
        off = np.asarray(q.offsets)
        rows = np.nonzero(np.diff(off))[0]
        sel = np.concatenate([np.arange(off[r], off[r + 1]) for r in rows])
        fsel = np.concatenate([np.arange(full.offsets[r], full.offsets[r + 1]) for r in rows])
        np.testing.assert_array_equal(np.asarray(q.indices)[sel], np.asarray(full.indices)[fsel])
        np.testing.assert_array_equal(np.asarray(q.distances)[sel].view(np.uint32),
                                      np.asarray(full.distances)[fsel].view(np.uint32))
    assert pe_sym < 0.65 * pe_two, (pe_sym, pe_two)
    compare(full, oracle.radius_query(X, X, R))


# --------------------------------------------------------------------------- spectrum diagnostic (a2)
@pytest.mark.parametrize("d,dt,s_ratio", [(3, np.float32, 0.1), (3, np.float64, 0.5), (20, np.float32, 0.5),
                                          (64, np.float32, None), (200, np.float32, None)])
def test_index_sigma_vs_oracle_svd(snn, d, dt, s_ratio):
    """snn_index_sigma (power iteration with deflation on the kept Gram) vs the oracle's
    SVD singular values of the centred data (eq:svd); the elongated Gaussian of PAPER.md:324
    gives sigma2/sigma1 -> s.  d = 200 exercises the tensor-core Gram."""
    rng = np.random.default_rng(1600 + d)
    n = 40000
    if s_ratio is not None:
        X = rng.standard_normal((n, d)) * np.array([1.0] + [s_ratio] * (d - 1))
    else:
        X = rng.standard_normal((n, d)) / np.sqrt(np.arange(1, d + 1))
    X = X.astype(dt)
    k = 4 if d > 3 else 2
    idx = snn.Index(_dev(X))
    try:
        sig = idx.sigma(k)
    finally:
        idx.free()
    P = X.astype(np.float64)
    _, S = oracle.principal_direction(oracle.center(P, oracle.column_mean(P)))
    tol = 2e-3 if d >= 128 else 1e-5   # FP16 hi/lo tensor-core Gram vs the fp64 SIMT Gram
    np.testing.assert_allclose(sig[:2], S[:2], rtol=tol)
    if s_ratio is not None:
        assert abs(sig[1] / sig[0] - s_ratio) < 0.05
    if d > 3:   # well separated spectrum (1/sqrt(i) scales): the deflated values match too
        np.testing.assert_allclose(sig, S[:k], rtol=max(tol, 1e-4))


@pytest.mark.parametrize("d", [64, 200])
def test_sampled_gram_build(snn, d):
    """A build whose tensor-core Gram uses a strided row sample (options gram_min_elems /
    gram_rows force it on a small instance): v1 is still close to the oracle's principal
    direction, the query results are exactly the oracle's (v1 only steers pruning,
    SPEC.md:132), and snn_index_sigma recomputes the full Gram (matches the oracle SVD)."""
    import paper_2212_07679_b200 as p
    rng = np.random.default_rng(1700 + d)
    n = 30000
    X = (rng.standard_normal((n, d)) / np.sqrt(np.arange(1, d + 1))).astype(np.float32)
    Q = (rng.standard_normal((300, d)) / np.sqrt(np.arange(1, d + 1))).astype(np.float32)
    R = 1.9 if d == 64 else 2.1
    try:
        p.snn_set_option("gram_min_elems", 1)
        p.snn_set_option("gram_rows", 2000)
        idx = snn.Index(_dev(X))
    finally:
        p.snn_set_option("gram_min_elems", 0)
        p.snn_set_option("gram_rows", 0)
    try:
        v = idx.arrays()["v1"].cpu().numpy().astype(np.float64)
        got = idx.query(_dev(Q), R)
        sig = idx.sigma(2)
    finally:
        idx.free()
    P = X.astype(np.float64)
    v1, S = oracle.principal_direction(oracle.center(P, oracle.column_mean(P)))
    assert abs(float(np.dot(v, v1))) / np.linalg.norm(v) > 0.99
    np.testing.assert_allclose(sig, S[:2], rtol=2e-3)
    compare(got, oracle.radius_query(X, Q, R))


def test_c_demo_runs(snn, tmp_path):
    """The plain-C example builds, queries (every point finds itself), copies the CSR to
    the host and runs DBSCAN through the C ABI alone."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2212_07679_b200", "lib")
    exe = tmp_path / "c_api_demo"
    subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(root, "include"),
                           os.path.join(root, "examples", "c_api_demo.c"), "-L", libdir, "-lsnn",
                           f"-Wl,-rpath,{libdir}", "-o", str(exe)])
    out = subprocess.check_output([str(exe)]).decode().split()
    n, m, nnz, k = map(int, out)
    assert n == m == 4096 and nnz > n and k >= 1


# --------------------------------------------------------------------------- concurrency
@pytest.mark.parametrize("kind", ["c2", "c3", "dbscan"])
def test_concurrent_queries_on_one_index(snn, kind):
    """Two host threads, each on its own CUDA stream, query ONE index at the same time
    (the library releases the GIL in every call); one of them runs with different
    per-thread options (two-sided scan / SIMT generic path).  Every result is bit-identical
    to the serial one."""
    import threading
    import torch
    import paper_2212_07679_b200 as p
    if kind == "c2":
        w = workloads.c2(n=200000)
        X, Q, R = w.X, None, 0.5866
    elif kind == "c3":
        w = workloads.c3(n=30000, m=3000)
        X, Q, R = w.X, w.Q, 1.8134
    else:
        w = workloads.c5(n=100000, seed=4, box=400.0)
        X, Q, R = w.X, None, 3.0
    idx = snn.Index(_dev(X))
    Qd = None if Q is None else _dev(Q)

    def once(stream):
        with torch.cuda.stream(stream):
            if kind == "dbscan":
                return idx.dbscan(R, 5, stream=stream)
            return idx.query_self(R, stream=stream) if Qd is None else idx.query(Qd, R, stream=stream)
    try:
        ref = once(torch.cuda.current_stream())
        out, errs = {}, []

        def worker(tid):
            try:
                if tid == 1:   # per-thread options: another (bit-identical) path
                    p.snn_set_option("symmetric", -1)
                    p.snn_set_option("tc", -1)
                st = torch.cuda.Stream()
                out[tid] = [once(st) for _ in range(3)]
            except Exception as e:   # pragma: no cover - reported below
                errs.append(e)
        th = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        assert p.snn_get_option("symmetric") == 1 and p.snn_get_option("tc") == 1   # main thread untouched
        for tid in range(2):
            for r in out[tid]:
                if kind == "dbscan":
                    assert r[1] == ref[1] and np.array_equal(r[0], ref[0])
                else:
                    _csr_equal(ref, r)
    finally:
        idx.free()
