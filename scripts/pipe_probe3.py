"""Does a big D2H copy on one stream overlap SNN build+query on another?"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2212_07679_b200 as snn
from cuda.bindings import runtime as cudart

snn.load_library()
w = workloads.c2()
R = w.R
Xd = torch.from_numpy(w.X).cuda()
err, s2 = cudart.cudaStreamCreateWithFlags(cudart.cudaStreamNonBlocking)
cs = torch.cuda.ExternalStream(int(s2))
err, s3 = cudart.cudaStreamCreateWithFlags(cudart.cudaStreamNonBlocking)
comp = torch.cuda.ExternalStream(int(s3))
src = torch.empty(318 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
dst = torch.empty_like(src, device="cpu").pin_memory()

def step():
    idx = snn.snn_build(Xd, stream=comp)
    r = snn.snn_query_self(idx, R, stream=comp)
    snn.snn_free(idx)
    snn.snn_result_free(r)

def build_only():
    idx = snn.snn_build(Xd, stream=comp)
    snn.snn_free(idx)

def mm():
    a = torch.randn(4096, 4096, device="cuda")
    with torch.cuda.stream(comp):
        for _ in range(20):
            a = a @ a
            a = a / a.norm()
    comp.synchronize()

for name, fn in (("snn step", step), ("snn build", build_only), ("matmul x20", mm)):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); alone = (time.perf_counter() - t) * 1e3
    with torch.cuda.stream(cs):
        dst.copy_(src, non_blocking=True)
    t = time.perf_counter(); fn(); busy = (time.perf_counter() - t) * 1e3
    cs.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(cs):
        dst.copy_(src, non_blocking=True)
    cs.synchronize(); copy = (time.perf_counter() - t) * 1e3
    print(f"{name}: alone {alone:.2f} ms, during a D2H copy {busy:.2f} ms (copy alone {copy:.2f} ms)")
