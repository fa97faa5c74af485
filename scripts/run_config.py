"""Run build + query of one BASELINE config a few times (profiling driver for ncu).

  python scripts/run_config.py [c1|c2|c3|c4] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2212_07679_b200 as snn  # noqa: E402
import workloads  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = workloads.CONFIGS[name]()
    X = torch.from_numpy(w.X).cuda()
    Q = None if w.Q is None else torch.from_numpy(w.Q).cuda()
    for _ in range(reps):
        idx = snn.snn_build(X)
        r = snn.snn_query_self(idx, w.R) if Q is None else snn.snn_query_radius(idx, Q, w.R)
        nnz = snn.snn_result_csr(r)["nnz"]
        snn.snn_result_free(r)
        snn.snn_free(idx)
    torch.cuda.synchronize()
    print(name, "nnz", nnz)


if __name__ == "__main__":
    main()
