"""Full-size parity on the BASELINE.json configurations: EVERY row of configs 2, 3 and 4
and EVERY label of config 5 against the fp64 oracle, through the C ABI in the launch
configuration bench.py times.

The oracle's results at these sizes (config 2: 38.7M pairs, config 4: 25 min of brute
force on 8 cores) are precomputed on the CPU container by ``scripts/make_digests.py``
(which calls only ``oracle/``) and stored as every row's hit count plus one 64-bit digest
per block of 1,024 rows (ids + float32 distance bits, ``tests/digest.py``); config 5 as one
digest per 4,096 labels plus K.  A mismatch names the rows / blocks and recomputes the
oracle for a few of them to show the difference.

The paper's exactness contract: "the set of returned points coincide" (§6.1)
and DBSCAN "returns exactly the same result" (§6.4).
"""
import json
import os

import numpy as np
import pytest

import workloads
from tests import digest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    meta = json.load(open(os.path.join(GOLDEN, f"full_{name}.json")))
    z = np.load(os.path.join(GOLDEN, f"full_{name}.npz"))
    return meta, {k: z[k] for k in z.files}


def check_inputs(w, meta):
    assert digest.sha256(w.X) == meta["sha256_X"], \
        "the seeded generator produced different input bytes on this host than on the digest host"
    if meta.get("sha256_Q"):
        assert digest.sha256(w.Q) == meta["sha256_Q"], "query generator differs on this host"


def compare_radius(gpu, w, meta, gold):
    """Returns a summary dict; raises AssertionError naming the mismatching rows/blocks."""
    counts, blocks = digest.csr_digests(gpu.offsets, gpu.indices, gpu.distances, meta["block_rows"])
    bad_rows = np.nonzero(counts != gold["counts"].astype(np.int64))[0]
    bad_blocks = np.nonzero(blocks != gold["blocks"])[0]
    if len(bad_rows) or len(bad_blocks):
        import oracle
        from tests.parity import compare
        rows = bad_rows[:3] if len(bad_rows) else np.arange(bad_blocks[0] * meta["block_rows"],
                                                            min(w.m, (bad_blocks[0] + 1) * meta["block_rows"]))[:64]
        detail = ""
        try:
            compare(gpu, oracle.radius_query(w.X, w.queries[rows], w.R), rows_subset=rows)
        except AssertionError as e:
            detail = str(e)
        raise AssertionError(f"{meta['config']}: {len(bad_rows)} rows with a different count, "
                             f"{len(bad_blocks)} of {len(blocks)} blocks with a different digest "
                             f"(first rows {bad_rows[:5].tolist()}, blocks {bad_blocks[:5].tolist()}); {detail}")
    return {"config": meta["config"], "rows": int(len(counts)), "pairs": int(counts.sum()),
            "blocks": int(len(blocks)), "oracle": meta["oracle"], "exact": True}


def compare_labels(lab, K, meta, gold):
    blocks = digest.label_digests(lab, meta["block_points"])
    bad = np.nonzero(blocks != gold["blocks"])[0]
    assert K == meta["K"], f"K = {K}, oracle {meta['K']}"
    assert len(bad) == 0, f"{len(bad)} of {len(blocks)} label blocks differ (first {bad[:5].tolist()})"
    return {"config": meta["config"], "points": int(len(lab)), "K": int(K), "blocks": int(len(blocks)),
            "n_noise": int((np.asarray(lab) == -1).sum()), "oracle": meta["oracle"], "exact": True}


def record(summary):
    out = os.environ.get("SNN_PARITY_RECORD")
    if out:
        with open(out, "a") as f:
            f.write(json.dumps(summary) + "\n")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_full_size_every_row_matches_oracle(snn, name):
    meta, gold = golden(name)
    w = workloads.CONFIGS[name]()
    check_inputs(w, meta)
    assert w.R == meta["R"]
    idx = snn.Index(_dev(w.X))
    try:
        gpu = idx.query_self(w.R) if w.Q is None else idx.query(_dev(w.Q), w.R)
    finally:
        idx.free()
    record(compare_radius(gpu, w, meta, gold))


@pytest.mark.gpu
def test_full_size_dbscan_labels_match_oracle(snn):
    meta, gold = golden("c5")
    w = workloads.c5()
    check_inputs(w, meta)
    idx = snn.Index(_dev(w.X))
    try:
        lab, K = idx.dbscan(w.R, w.dbscan_min_pts)
    finally:
        idx.free()
    assert int((lab == -1).sum()) == meta["n_noise"]
    record(compare_labels(lab, K, meta, gold))


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


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


# ------------------------------------------------------------------- CPU: the digests themselves
@pytest.mark.parametrize("name", ["c2", "c5"])
def test_golden_inputs_regenerate(name):
    """The stored digests belong to the inputs the generators produce here."""
    meta, _ = golden(name)
    w = workloads.CONFIGS[name]()
    check_inputs(w, meta)


def test_digest_detects_every_kind_of_difference():
    """csr_digests is independent of the order inside a row and changes if an id, a
    distance bit, or a row assignment changes."""
    import oracle
    rng = np.random.default_rng(5)
    X = rng.random((3000, 3)).astype(np.float32)
    res = oracle.radius_query(X, X, 0.06)
    c0, b0 = digest.oracle_csr_digests(res, 256)
    keep = res["s"] <= res["R2"]
    off = np.zeros(len(res["offsets"]), dtype=np.int64)
    rows = np.repeat(np.arange(3000), np.diff(res["offsets"]))
    np.cumsum(np.bincount(rows[keep], minlength=3000), out=off[1:])
    ids = res["indices"][keep].copy()
    dist = np.sqrt(res["s"][keep]).astype(np.float32)
    c1, b1 = digest.csr_digests(off, ids, dist, 256)
    assert np.array_equal(c0, c1) and np.array_equal(b0, b1)
    r = 17                                  # reverse one row: same digest
    a, b = off[r], off[r + 1]
    ids2, dist2 = ids.copy(), dist.copy()
    ids2[a:b], dist2[a:b] = ids[a:b][::-1], dist[a:b][::-1]
    assert np.array_equal(digest.csr_digests(off, ids2, dist2, 256)[1], b0)
    ids3 = ids.copy()
    ids3[a] += 1                            # wrong id
    assert not np.array_equal(digest.csr_digests(off, ids3, dist, 256)[1], b0)
    dist3 = dist.copy()
    dist3[a] = np.nextafter(dist3[a], np.float32(1))   # one ulp
    assert not np.array_equal(digest.csr_digests(off, ids, dist3, 256)[1], b0)
    lab = rng.integers(-1, 5, 10000)
    l2 = lab.copy()
    l2[[3, 4]] = l2[[4, 3]] if l2[3] != l2[4] else (l2[3], l2[4] + 1)
    assert not np.array_equal(digest.label_digests(lab, 4096), digest.label_digests(l2, 4096))
