"""K8 one query per thread vs two (option scan2q) for d = 1..8 on a config-2-like Gaussian
mixture (1M points, 64 clusters in [0,100)^d, sigma 2, R = median 32nd-neighbour distance of
a 1,000-point sample): per-launch scan time and step time, self-query.

  python scripts/sweep_2q_d.py [n] [chunk2q ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_07679_b200 as snn  # noqa: E402


def measure(X, R, reps=4):
    snn.snn_profile_enable(True)
    nnz = 0
    for _ in range(reps):
        idx = snn.snn_build(X)
        r = snn.snn_query_self(idx, R)
        nnz = int(r.nnz) if hasattr(r, "nnz") else 0
        snn.snn_result_free(r)
        snn.snn_free(idx)
    out = {f: snn.snn_profile_read(f) for f in ("window_count", "window_write", "query")}
    snn.snn_profile_enable(False)
    return {k: round(v["ms"] / max(1, v["launches"]), 3) for k, v in out.items()}, nnz


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    chunks = [int(c) for c in sys.argv[2:]] or [640]
    for d in range(1, 9):
        rng = np.random.default_rng(100 + d)
        cen = rng.random((64, d)) * 100.0
        X = (cen[rng.integers(0, 64, n)] + rng.normal(0.0, 2.0, (n, d))).astype(np.float32)
        Xg = torch.from_numpy(X).cuda()
        s = Xg[torch.from_numpy(rng.choice(n, 1000, replace=False)).cuda()]
        dist = torch.cdist(s, Xg)                       # sample radius only (not the product path)
        R = float(dist.kthvalue(33, dim=1).values.median())
        del dist
        snn.snn_set_option("scan2q", -1)
        measure(Xg, R, 1)
        t1, nnz = measure(Xg, R)
        line = {"d": d, "n": n, "R": round(R, 4), "one_query": t1}
        for c in chunks:
            snn.snn_set_option("scan2q", 1)
            snn.snn_set_option("chunk2q", c)
            measure(Xg, R, 1)
            line[f"two_query_chunk{c}"] = measure(Xg, R)[0]
        snn.snn_set_option("scan2q", 0)
        snn.snn_set_option("chunk2q", 0)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
