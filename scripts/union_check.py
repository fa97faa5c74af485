"""DBSCAN union-pass variants on config 5: identical labels + union-path counters.

  python scripts/union_check.py [variants...]   (each "key=v,key=v" option set; default union_snap=-1 union_snap=1)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_07679_b200 as snn  # noqa: E402
import workloads  # noqa: E402


def main():
    variants = sys.argv[1:] or ["union_snap=-1", "union_snap=1"]
    w = workloads.CONFIGS["c5"]()
    X = torch.from_numpy(w.X).cuda()
    idx = snn.snn_build(X)
    ref = None
    snn.snn_set_option("union_stats", 1)
    snn.snn_profile_enable(True)
    for v in variants:
        for kv in v.split(","):
            key, val = kv.split("=")
            snn.snn_set_option(key, int(val))
        lab = torch.empty(w.X.shape[0], dtype=torch.int32, device="cuda")
        for rep in range(4):
            p0 = snn.snn_profile_read("dbscan_union")["ms"]   # cumulative
            torch.cuda.synchronize()
            t = time.perf_counter()
            k = snn.snn_dbscan(idx, w.R, w.dbscan_min_pts, lab)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            pu = round(snn.snn_profile_read("dbscan_union")["ms"] - p0, 3)
        L = lab.cpu().numpy()
        for kv in v.split(","):
            snn.snn_set_option(kv.split("=")[0], 0)   # back to the default
        same = ref is None or np.array_equal(L, ref)
        if ref is None:
            ref = L
        st = [snn.snn_get_option(k) for k in ("last_union_path", "last_union_hits", "last_union_links")]
        print(f"{v:36s} clusters={k} wall={dt*1e3:.2f} ms union={pu} ms identical={same} "
              f"path/hits/links={st}", flush=True)
    snn.snn_free(idx)


if __name__ == "__main__":
    main()
