"""Time the low-d scan pass under option variants on a config (GPU tuning sweep).

  python scripts/sweep_lowd.py c2 ['{"option": [values], ...}']
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


def measure(X, R, reps=5):
    snn.snn_profile_enable(True)
    for _ in range(reps):
        idx = snn.snn_build(X)
        r = snn.snn_query_self(idx, R)
        snn.snn_result_free(r)
        snn.snn_free(idx)
    out = {f: snn.snn_profile_read(f) for f in ("window_count", "window_write", "query")}
    ovf = snn.snn_profile_read("overflow")["units"]
    snn.snn_profile_enable(False)
    return {k: v["ms"] / max(1, v["launches"]) for k, v in out.items()}, ovf


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    w = workloads.CONFIGS[name]()
    X = torch.from_numpy(w.X).cuda()
    grid = {"variant": [1, 2], "chunk": [1024, 2048, 4096], "query_block": [128, 256], "cap": [32, 64]}
    if len(sys.argv) > 2:
        grid = json.loads(sys.argv[2])
    keys = list(grid)
    measure(X, w.R, 2)
    for vals in itertools.product(*[grid[k] for k in keys]):
        for k, v in zip(keys, vals):
            snn.snn_set_option(k, v)
        t, ovf = measure(X, w.R)
        print(json.dumps({**dict(zip(keys, vals)), **{k: round(v, 3) for k, v in t.items()}, "ovf": ovf}), flush=True)
    for k in keys:
        snn.snn_set_option(k, 0)


if __name__ == "__main__":
    main()
