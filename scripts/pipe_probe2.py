"""Timeline probe of the pipelined end-to-end loop (config 2)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2212_07679_b200 as snn
from cuda.bindings import runtime as cudart

snn.load_library()
w = workloads.c2()
R = w.R
Xh = torch.from_numpy(w.X).pin_memory()
Xd = torch.from_numpy(w.X).cuda()
err, s2 = cudart.cudaStreamCreateWithFlags(cudart.cudaStreamNonBlocking)
cs = torch.cuda.ExternalStream(int(s2))
err, s3 = cudart.cudaStreamCreateWithFlags(cudart.cudaStreamNonBlocking)
comp = torch.cuda.ExternalStream(int(s3))

def step(X):
    idx = snn.snn_build(X, stream=comp)
    r = snn.snn_query_self(idx, R, stream=comp)
    snn.snn_free(idx)
    return r

r = step(Xh); nnz = snn.snn_result_csr(r)["nnz"]; snn.snn_result_free(r)
bufs = [tuple(torch.empty(k, dtype=t).pin_memory() for k, t in ((w.m + 1, torch.int64), (nnz, torch.int32), (nnz, torch.float32))) for _ in range(2)]
for X, label in ((Xd, "device X"), (Xh, "host X")):
    torch.cuda.synchronize()
    E = lambda: torch.cuda.Event(enable_timing=True)
    t0 = E(); t0.record(comp)
    marks = []
    pend = []
    for i in range(8):
        a = E(); a.record(comp)
        h0 = time.perf_counter()
        r = step(X)
        h1 = time.perf_counter()
        b = E(); b.record(comp)
        if len(pend) == 2:
            rr, ev = pend.pop(0); ev.synchronize(); snn.snn_result_free(rr)
        c = E(); c.record(cs)
        snn.snn_result_copy_async(r, *bufs[i % 2], stream=cs)
        d = E(); d.record(cs)
        pend.append((r, d))
        marks.append((a, b, c, d, (h1 - h0) * 1e3))
    for rr, ev in pend:
        ev.synchronize(); snn.snn_result_free(rr)
    torch.cuda.synchronize()
    print(label)
    for i, (a, b, c, d, hms) in enumerate(marks):
        print(f"step {i}: compute {t0.elapsed_time(a):8.2f} -> {t0.elapsed_time(b):8.2f}   copy {t0.elapsed_time(c):8.2f} -> {t0.elapsed_time(d):8.2f}   host call {hms:.2f} ms")
