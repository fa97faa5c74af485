"""Probe: does the CSR copy-out overlap the next step's build + query? (config 2)"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads
import paper_2212_07679_b200 as snn
from cuda.bindings import runtime as cudart

snn.load_library()
w = workloads.c2()
R = w.R
Xh = torch.from_numpy(w.X).pin_memory()
dev = torch.device("cuda", 0)
cs = torch.cuda.Stream()
print("torch cs flags", cudart.cudaStreamGetFlags(cs.cuda_stream))
print("default stream ptr", torch.cuda.current_stream().cuda_stream)

def step():
    idx = snn.snn_build(Xh)
    r = snn.snn_query_self(idx, R)
    snn.snn_free(idx)
    return r

r = step(); nnz = snn.snn_result_csr(r)["nnz"]; snn.snn_result_free(r)
bufs = [tuple(torch.empty(k, dtype=t).pin_memory() for k, t in ((w.m + 1, torch.int64), (nnz, torch.int32), (nnz, torch.float32))) for _ in range(2)]

def timeit(fn, n=10):
    torch.cuda.synchronize(); t = time.perf_counter()
    fn(n)
    torch.cuda.synchronize(); return (time.perf_counter() - t) / n * 1e3

def compute_only(n):
    for _ in range(n):
        r = step(); snn.snn_result_free(r)

def serial(n):
    for i in range(n):
        r = step(); snn.snn_result_copy(r, *bufs[i % 2]); snn.snn_result_free(r)

r0 = step()
def copy_only(n):
    for i in range(n):
        snn.snn_result_copy_async(r0, *bufs[i % 2], stream=cs)
    cs.synchronize()

def piped(n, comp=None):
    pend = []
    for i in range(n):
        if comp is not None:
            with torch.cuda.stream(comp):
                r = step()
        else:
            r = step()
        if len(pend) == 2:
            rr, ev = pend.pop(0); ev.synchronize(); snn.snn_result_free(rr)
        snn.snn_result_copy_async(r, *bufs[i % 2], stream=cs)
        ev = torch.cuda.Event(); ev.record(cs); pend.append((r, ev))
    for rr, ev in pend:
        ev.synchronize(); snn.snn_result_free(rr)

print("compute only ms", timeit(compute_only))
print("copy only ms", timeit(copy_only))
print("serial ms", timeit(serial))
print("piped (default stream) ms", timeit(piped))
comp = torch.cuda.Stream()
print("piped (side compute stream) ms", timeit(lambda n: piped(n, comp)))
err, s2 = cudart.cudaStreamCreateWithFlags(cudart.cudaStreamNonBlocking)
cs_nb = torch.cuda.ExternalStream(int(s2))
cs = cs_nb
print("piped (nonblocking copy stream) ms", timeit(piped))
print("piped (both side) ms", timeit(lambda n: piped(n, comp)))
