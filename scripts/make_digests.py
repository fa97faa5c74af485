"""Write the full-size oracle digests the GPU parity test compares against
(tests/golden/full_<config>.{json,npz}).  Calls only ``oracle/`` (plus the seeded input
generators in ``workloads/`` and the hashing in ``tests/digest.py``); runs on the CPU
container, no GPU.

  python scripts/make_digests.py c2 c3 c4 c5

* c2 (n = m = 1M, d = 3): ``oracle.radius_query(grid=True)`` -- the grid-pruned variant
  with the brute force's per-pair test; additionally 2,000 random rows are recomputed by
  the plain brute force and must be identical.
* c3, c4: the plain brute force over every query (c4: ~25 min on 8 cores).
* c5 (n = 2M, d = 2, DBSCAN eps = 3, minPts = 5): ``oracle.dbscan(grid=True)``; the
  neighbourhood counts of 2,000 random points are recomputed by brute force
  (``oracle.neighbour_counts``) and must be identical.

Each JSON records the sha256 of the generated inputs: the GPU test first checks that the
box regenerated the same bytes.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads  # noqa: E402
from tests import digest  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def radius(name: str):
    w = workloads.CONFIGS[name]()
    t0 = time.time()
    meta = {"config": name, "n": w.n, "m": w.m, "d": w.d, "R": w.R, "R_hex": float(w.R).hex(),
            "sha256_X": digest.sha256(w.X), "sha256_Q": None if w.Q is None else digest.sha256(w.Q),
            "threads": oracle.num_threads(), "block_rows": 1024}
    Q = w.queries
    if w.d <= 3:
        res = oracle.radius_query(w.X, Q, w.R, grid=True)
        meta["oracle"] = "oracle.radius_query(grid=True) (grid-pruned, same per-pair test)"
        rng = np.random.default_rng(123)
        rows = np.sort(rng.choice(w.m, 2000, replace=False))
        bf = oracle.radius_query(w.X, Q[rows], w.R)
        for t, r in enumerate(rows):
            a, b = res["offsets"][r], res["offsets"][r + 1]
            c, e = bf["offsets"][t], bf["offsets"][t + 1]
            assert np.array_equal(res["indices"][a:b], bf["indices"][c:e])
            assert np.array_equal(res["s"][a:b], bf["s"][c:e])
        meta["brute_force_rows_checked"] = len(rows)
        counts, blocks = digest.oracle_csr_digests(res, 1024)
    else:   # plain brute force in query chunks (bounded memory)
        meta["oracle"] = "oracle.radius_query (brute force, every query)"
        cnts, rdig = [], []
        step = 1024
        for s0 in range(0, w.m, step):
            r = oracle.radius_query(w.X, Q[s0:s0 + step], w.R)
            c, b = digest.oracle_csr_digests(r, step, row0=s0)
            cnts.append(c)
            rdig.append(b)   # one block per chunk (chunk == block)
            print(f"  {name}: {min(w.m, s0 + step)}/{w.m} queries, {time.time() - t0:.0f} s", flush=True)
        counts, blocks = np.concatenate(cnts), np.concatenate(rdig)
    meta["nnz"] = int(counts.sum())
    meta["max_row"] = int(counts.max())
    meta["seconds"] = round(time.time() - t0, 1)
    meta["global_digest"] = hex(int(blocks.sum(dtype=np.uint64)))
    dt = np.uint8 if counts.max() < 256 else (np.uint16 if counts.max() < 65536 else np.int32)
    np.savez_compressed(os.path.join(GOLDEN, f"full_{name}.npz"), counts=counts.astype(dt), blocks=blocks)
    json.dump(meta, open(os.path.join(GOLDEN, f"full_{name}.json"), "w"), indent=1)
    print(json.dumps(meta))


def dbscan(name: str):
    w = workloads.CONFIGS[name]()
    t0 = time.time()
    lab, K, cnt = oracle.dbscan(w.X, w.R, w.dbscan_min_pts, grid=True)
    rng = np.random.default_rng(321)
    ids = rng.choice(w.n, 2000, replace=False)
    assert np.array_equal(oracle.neighbour_counts(w.X, w.R, ids), cnt[ids])
    blocks = digest.label_digests(lab, 4096)
    meta = {"config": name, "n": w.n, "d": w.d, "eps": w.R, "min_pts": w.dbscan_min_pts,
            "sha256_X": digest.sha256(w.X), "threads": oracle.num_threads(),
            "oracle": "oracle.dbscan(grid=True) (components over grid-pruned pairs, same per-pair test)",
            "brute_force_counts_checked": len(ids), "block_points": 4096,
            "K": K, "n_core": int((cnt >= w.dbscan_min_pts).sum()), "n_noise": int((lab == -1).sum()),
            "largest_cluster": int(np.bincount(lab[lab >= 0]).max()) if K else 0,
            "seconds": round(time.time() - t0, 1),
            "global_digest": hex(int(blocks.sum(dtype=np.uint64)))}
    np.savez_compressed(os.path.join(GOLDEN, f"full_{name}.npz"), blocks=blocks)
    json.dump(meta, open(os.path.join(GOLDEN, f"full_{name}.json"), "w"), indent=1)
    print(json.dumps(meta))


if __name__ == "__main__":
    for c in sys.argv[1:] or ["c2", "c3", "c5", "c4"]:
        (dbscan if c == "c5" else radius)(c)
