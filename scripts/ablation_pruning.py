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


def main():
    names = sys.argv[1:] or ["c2", "c3", "c4"]
    for name in names:
        w = workloads.CONFIGS[name]()
        X = torch.from_numpy(w.X).cuda()
        Q = None if w.Q is None else torch.from_numpy(w.Q).cuda()
        idx = snn.snn_build(X)
        timed_query(idx, Q, w.R, 1)
        t_snn, pairs_snn, nnz_snn = timed_query(idx, Q, w.R, 3)
        snn.snn_set_option("window_all", 1)
        try:
            t_bf, pairs_bf, nnz_bf = timed_query(idx, Q, w.R, 1)
        finally:
            snn.snn_set_option("window_all", 0)
        snn.snn_free(idx)
        assert nnz_snn == nnz_bf, (nnz_snn, nnz_bf)
        print(json.dumps({"config": name, "snn_query_ms": round(t_snn["query"], 3),
                          "bruteforce_query_ms": round(t_bf["query"], 3),
                          "speedup": round(t_bf["query"] / t_snn["query"], 2),
                          "pairs_snn": pairs_snn, "pairs_bruteforce": pairs_bf,
                          "pair_ratio": round(pairs_bf / max(pairs_snn, 1), 2), "nnz": nnz_snn}), flush=True)


if __name__ == "__main__":
    main()
