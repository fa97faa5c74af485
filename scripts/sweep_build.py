"""Time snn_build under option variants (GPU tuning sweep).

  python scripts/sweep_build.py c3 tc_gram_min_d=32,128
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


def main():
    name = sys.argv[1]
    grid = {}
    for a in sys.argv[2:]:
        k, v = a.split("=")
        grid[k] = [int(x) for x in v.split(",")]
    w = workloads.CONFIGS[name]()
    X = torch.from_numpy(w.X).cuda()
    keys = list(grid)
    for vals in itertools.product(*[grid[k] for k in keys]):
        for k, v in zip(keys, vals):
            snn.snn_set_option(k, v)
        snn.snn_free(snn.snn_build(X))
        snn.snn_profile_enable(True)
        for _ in range(5):
            snn.snn_free(snn.snn_build(X))
        b = snn.snn_profile_read("build")
        snn.snn_profile_enable(False)
        idx = snn.snn_build(X)
        info = snn.snn_index_info(idx)
        snn.snn_free(idx)
        print(json.dumps({"config": name, **dict(zip(keys, vals)), "build_ms": round(b["ms"] / b["launches"], 4),
                          "power_iters": info["power_iters"], "sigma1": info["sigma1"]}), flush=True)
    for k in keys:
        snn.snn_set_option(k, 0)


if __name__ == "__main__":
    main()
