"""Per-call index build time on config 4 (CUDA events on the stream + host wall), repeated.

  python scripts/build_var.py [config] [reps] [reserve_GB]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2212_07679_b200 as snn  # noqa: E402
import workloads  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    gb = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
    w = workloads.CONFIGS[name]()
    X = torch.from_numpy(w.X).cuda()
    if gb:
        snn.snn_pool_reserve(int(gb * 2**30))
    prev = None
    for r in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        e0.record()
        idx = snn.snn_build(X)
        e1.record()
        torch.cuda.synchronize()
        host = (time.perf_counter() - t) * 1e3
        if prev is not None:
            snn.snn_free(prev)
        prev = idx
        print(f"{name} rep {r}: build {e0.elapsed_time(e1):.3f} ms (host {host:.3f} ms)", flush=True)
    snn.snn_free(prev)


if __name__ == "__main__":
    main()
