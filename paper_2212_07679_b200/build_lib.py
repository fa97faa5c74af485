"""Compile the CUDA library in-tree: paper_2212_07679_b200/lib/libsnn.so (sm_100a only)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "lib")
OUT = os.path.join(OUT_DIR, "libsnn.so")
# debug build: device-side bounds checks (SNN_DASSERT, -DSNN_DEBUG); load it with
# SNN_LIB=<path> (tests/test_debug_build.py runs the small parity suite on it)
OUT_DEBUG = os.path.join(OUT_DIR, "libsnn_debug.so")
SOURCES = ["api.cu", "build.cu", "radix_sort.cu", "scan.cu", "query.cu", "dbscan.cu", "tc.cu", "tc_gram.cu", "csr.cu", "tc_lowd.cu", "metric.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _stale(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(SRC, f) for f in os.listdir(SRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "snn.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    out = OUT_DEBUG if debug else OUT
    if not force and not _stale(out):
        return out
    obj_dir = os.path.join(OUT_DIR, "debug") if debug else OUT_DIR
    os.makedirs(obj_dir, exist_ok=True)
    objs = []
    procs = []
    for f in SOURCES:
        obj = os.path.join(obj_dir, f.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *(["-DSNN_DEBUG"] if debug else []), "-c", os.path.join(SRC, f), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((subprocess.Popen(cmd), f))
        objs.append(obj)
    for p, f in procs:
        if p.wait() != 0:
            raise RuntimeError(f"nvcc failed on {f}")
    tmp = out + ".tmp"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                           "-o", tmp, "-cudart", "static", "-Xlinker", "--no-undefined"])
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv))
