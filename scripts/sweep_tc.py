"""Time the tensor-core filter pass (K9) under option variants (GPU tuning sweep).

  python scripts/sweep_tc.py c3 [key=v1,v2 ...]      e.g. tc_diag=0,1,2 tc_tiles=4,8,16
Diagnostic options (tc_diag) give invalid results; they only isolate pipeline stages.
"""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2212_07679_b200 as snn  # noqa: E402
import workloads  # noqa: E402


def measure(idx, Q, R, reps=5):
    snn.snn_profile_enable(True)
    for _ in range(reps):
        r = snn.snn_query_self(idx, R) if Q is None else snn.snn_query_radius(idx, Q, R)
        snn.snn_result_free(r)
    out = {f: snn.snn_profile_read(f) for f in ("window_count", "window_write", "query")}
    snn.snn_profile_enable(False)
    return {k: v["ms"] / max(1, v["launches"]) for k, v in out.items()}


def main():
    name = sys.argv[1]
    grid = {}
    for a in sys.argv[2:]:
        k, v = a.split("=")
        grid[k] = [int(x) for x in v.split(",")]
    w = workloads.CONFIGS[name]()
    X = torch.from_numpy(w.X).cuda()
    Q = None if w.Q is None else torch.from_numpy(w.Q).cuda()
    idx = snn.snn_build(X)
    measure(idx, Q, w.R, 2)
    keys = list(grid)
    for vals in itertools.product(*[grid[k] for k in keys]):
        for k, v in zip(keys, vals):
            snn.snn_set_option(k, v)
        t = measure(idx, Q, w.R)
        print(json.dumps({"config": name, **dict(zip(keys, vals)), **{k: round(v, 4) for k, v in t.items()}}), flush=True)
    for k in keys:
        snn.snn_set_option(k, 0)
    snn.snn_free(idx)


if __name__ == "__main__":
    main()
