"""GPU analogue of the paper's "brute force 2" ablation (ratios P:515):
the same kernels with the candidate window forced to every point (option window_all)
vs the SNN window.  Results are identical by construction (checked); prints timings.

  python scripts/ablation_pruning.py [c2 c3 c4]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_07679_b200 as snn  # noqa: E402
import workloads  # noqa: E402


def timed_query(idx, Q, R, reps):
    snn.snn_profile_enable(True)
    res = None
    for _ in range(reps):
        if res is not None:
            snn.snn_result_free(res)
        res = snn.snn_query_self(idx, R) if Q is None else snn.snn_query_radius(idx, Q, R)
    out = {f: snn.snn_profile_read(f) for f in ("window_count", "query")}
    snn.snn_profile_enable(False)
    csr = snn.snn_result_csr(res)
    nnz = csr["nnz"]
    snn.snn_result_free(res)
    return {k: v["ms"] / max(1, v["launches"]) for k, v in out.items()}, \
        out["window_count"]["units"] / max(1, out["window_count"]["launches"]), nnz


def arm(idx, Q, R, opts, reps):
    for k, v in opts.items():
        snn.snn_set_option(k, v)
    try:
        timed_query(idx, Q, R, 1)                      # warm: workspace pool grown, caches hot
        return timed_query(idx, Q, R, reps)
    finally:
        for k in opts:
            snn.snn_set_option(k, 0)


def main():
    """Three arms on the same index, each warmed up first:
      snn        the default query (symmetric self-query: each unordered pair once)
      snn_2sided the SNN window with every pair evaluated from both sides
      brute2     window forced to [0, n) ("brute force 2"), two-sided
    Ratios: the whole query, and the scan kernel alone (window_count), plus the pair
    counts; snn_2sided vs brute2 isolates the pruning at equal per-pair work."""
    names = sys.argv[1:] or ["c2", "c3", "c4"]
    for name in names:
        w = workloads.CONFIGS[name]()
        X = torch.from_numpy(w.X).cuda()
        Q = None if w.Q is None else torch.from_numpy(w.Q).cuda()
        idx = snn.snn_build(X)
        out = {}
        out["snn"] = arm(idx, Q, w.R, {}, 3)
        out["snn_2sided"] = arm(idx, Q, w.R, {"symmetric": -1}, 3)
        out["brute2"] = arm(idx, Q, w.R, {"window_all": 1, "cap": 8}, 2)
        snn.snn_free(idx)
        nnz = {k: v[2] for k, v in out.items()}
        assert len(set(nnz.values())) == 1, nnz
        rec = {"config": name, "nnz": nnz["snn"]}
        for k, (t, pairs, _) in out.items():
            rec[k] = {"query_ms": round(t["query"], 3), "scan_ms": round(t["window_count"], 3), "pairs": pairs,
                      "scan_pairs_per_s": pairs / (t["window_count"] * 1e-3)}
        b, s2, s1 = rec["brute2"], rec["snn_2sided"], rec["snn"]
        rec["pruning_pair_ratio"] = round(b["pairs"] / s2["pairs"], 2)
        rec["pruning_scan_speedup"] = round(b["scan_ms"] / s2["scan_ms"], 2)
        rec["pruning_query_speedup"] = round(b["query_ms"] / s2["query_ms"], 2)
        rec["default_vs_brute2_query_speedup"] = round(b["query_ms"] / s1["query_ms"], 2)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
