"""Build-time variance probe (config 4): per-build CUDA-event times."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2212_07679_b200 as snn
snn.load_library()
w = workloads.c4()
X = torch.from_numpy(w.X).cuda()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
ts = []
for i in range(20):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    idx = snn.snn_build(X)
    e1.record(); e1.synchronize()
    snn.snn_free(idx)
    ts.append(e0.elapsed_time(e1))
print(" ".join(f"{t:.2f}" for t in ts))
snn.snn_profile_enable(True)
for i in range(5):
    idx = snn.snn_build(X); snn.snn_free(idx)
print(snn.snn_profile_read("build"))
