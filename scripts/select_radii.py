"""Select the radii of configs 2-4 with the CPU oracle (and nothing else) and write
workloads/radii.json.  Readings: DESIGN.md C17.

* C2: R = median over the first 1,000 points of their 32nd-smallest distance to all n
      points (self counted as the 1st) -- BASELINE.json configs[1].
* C3: R^2 = midpoint of the 100,000th and 100,001st smallest pooled squared distances of
      the first 1,000 queries to all n points (mean count ~100) -- configs[2].
* C4: same with 50,000 / 50,001 (mean count ~50) -- configs[3].

Usage: python scripts/select_radii.py [c2 c3 c4]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle      # noqa: E402
import workloads   # noqa: E402


def _query_all(X, Q, R):
    return oracle.radius_query(X, Q, R, band_rel=0.0)


def kth_smallest_per_query(X, Q, k, R0):
    R = R0
    while True:
        res = _query_all(X, Q, R)
        cnt = np.diff(res["offsets"])
        if cnt.min() >= k:
            break
        R *= 1.5
    out = np.empty(len(Q))
    o = res["offsets"]
    for j in range(len(Q)):
        out[j] = np.sort(res["s"][o[j]:o[j + 1]])[k - 1]
    return out


def pooled_kth(X, Q, k, R0):
    R = R0
    while True:
        res = _query_all(X, Q, R)
        if res["offsets"][-1] >= k + 1:
            break
        R *= 1.25
    s = np.sort(res["s"])
    return s[k - 1], s[k]


def main(which):
    out = workloads.load_radii()
    t0 = time.time()
    if "c2" in which:
        w = workloads.c2()
        s32 = kth_smallest_per_query(w.X, w.X[:1000], 32, 0.5)
        R = float(np.median(np.sqrt(s32)))
        out["c2"] = {"R": R, "rule": "median over first 1000 points of 32nd-smallest distance "
                     "(self = 1st), oracle fp64", "threads": oracle.num_threads()}
        print("c2 R =", R, time.time() - t0, flush=True)
    if "c3" in which:
        w = workloads.c3()
        a, b = pooled_kth(w.X, w.Q[:1000], 100000, 1.7)
        R = float(np.sqrt(0.5 * (a + b)))
        out["c3"] = {"R": R, "R2_lo": float(a), "R2_hi": float(b),
                     "rule": "R^2 = midpoint of 100000th/100001st pooled squared distance of "
                     "first 1000 queries, oracle fp64"}
        print("c3 R =", R, time.time() - t0, flush=True)
    if "c4" in which:
        w = workloads.c4()
        a, b = pooled_kth(w.X, w.Q[:1000], 50000, 5.8)
        R = float(np.sqrt(0.5 * (a + b)))
        out["c4"] = {"R": R, "R2_lo": float(a), "R2_hi": float(b),
                     "rule": "R^2 = midpoint of 50000th/50001st pooled squared distance of "
                     "first 1000 queries, oracle fp64"}
        print("c4 R =", R, time.time() - t0, flush=True)
    with open(workloads.RADII_PATH, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4"])
