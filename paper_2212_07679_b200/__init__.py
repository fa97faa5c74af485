"""paper_2212_07679_b200 -- B200-native SNN (arXiv 2212.07679) hot path.

Thin ctypes binding over the C ABI in ``include/snn.h`` (``lib/libsnn.so``, sm_100a).
Argument marshalling only: every step of index build and radius query runs in the
library's CUDA kernels.  PyTorch supplies device memory and the current stream.
There is no CPU fallback: importing works without a GPU, but every compute call needs the
compiled library and an sm_100 device and raises otherwise.

Low level (same names as the C ABI): ``snn_build``, ``snn_query_radius``,
``snn_query_self``, ``snn_result_csr``, ``snn_result_copy``, ``snn_result_free``,
``snn_dbscan``, ``snn_free``, ``snn_last_error``, ``snn_index_info``,
``snn_launch_count``, ``snn_set_option``.

High level: ``Index`` (owns an snn_index) and ``CSR`` (host or device copies).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SNN_LIB: an alternative in-tree build of the same library (A/B timing of two builds)
LIB_PATH = os.environ.get("SNN_LIB") or os.path.join(_HERE, "lib", "libsnn.so")

SNN_F32, SNN_F64 = 0, 1
STATUS = {0: "SNN_OK", 1: "SNN_ERR_INVALID_ARGUMENT", 2: "SNN_ERR_EMPTY",
          3: "SNN_ERR_NONFINITE", 4: "SNN_ERR_DIM_MISMATCH", 5: "SNN_ERR_OUT_OF_MEMORY",
          6: "SNN_ERR_CUDA", 7: "SNN_ERR_UNSUPPORTED"}

EXPORTS = ["snn_build", "snn_build_metric", "snn_append", "snn_save", "snn_load",
           "snn_query_radius_part", "snn_query_self_part", "snn_index_sigma", "snn_query_radius", "snn_query_self", "snn_result_csr",
           "snn_result_copy", "snn_result_copy_async", "snn_result_free", "snn_result_free_async", "snn_free_async", "snn_pool_reserve", "snn_dbscan", "snn_free", "snn_last_error",
           "snn_index_info", "snn_launch_count", "snn_set_option", "snn_get_option", "snn_profile_enable",
           "snn_profile_read"]


class SnnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class _CSR(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("nnz", ctypes.c_int64), ("offsets", ctypes.c_void_p),
                ("indices", ctypes.c_void_p), ("distances", ctypes.c_void_p)]


class _Info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("d", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("ld", ctypes.c_int32), ("power_iters", ctypes.c_int32),
                ("sigma1", ctypes.c_double), ("key_err", ctypes.c_double),
                ("v1_norm", ctypes.c_double), ("mu", ctypes.c_void_p), ("v1", ctypes.c_void_p),
                ("keys", ctypes.c_void_p), ("perm", ctypes.c_void_p), ("xbar", ctypes.c_void_p),
                ("xs", ctypes.c_void_p), ("tc_operand", ctypes.c_int32), ("tc_kpad", ctypes.c_int32),
                ("tc_exp", ctypes.c_int32), ("metric", ctypes.c_int32)]

# snn_metric (include/snn.h)
METRICS = {"euclidean": 0, "cosine": 1, "angular": 2, "manhattan": 3, "mips": 4}


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libsnn.so.  Raises (no fallback) if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"CUDA library missing: {path} (run __graft_entry__.build() or "
                           f"python paper_2212_07679_b200/build_lib.py)")
    lib = ctypes.CDLL(path)
    P, i64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    sig = {
        "snn_build": ([P, i64, i32, ctypes.c_int, P, ctypes.POINTER(P)], ctypes.c_int),
        "snn_build_metric": ([P, i64, i32, ctypes.c_int, i32, P, ctypes.POINTER(P)], ctypes.c_int),
        "snn_append": ([P, P, i64, i32, ctypes.c_int, P], ctypes.c_int),
        "snn_save": ([P, ctypes.c_char_p, P], ctypes.c_int),
        "snn_load": ([ctypes.c_char_p, P, ctypes.POINTER(P)], ctypes.c_int),
        "snn_query_radius": ([P, P, i64, i32, ctypes.c_int, f64, P, ctypes.POINTER(P)], ctypes.c_int),
        "snn_query_self": ([P, f64, P, ctypes.POINTER(P)], ctypes.c_int),
        "snn_query_radius_part": ([P, P, i64, i32, ctypes.c_int, f64, i32, i32, P, ctypes.POINTER(P)], ctypes.c_int),
        "snn_query_self_part": ([P, f64, i32, i32, P, ctypes.POINTER(P)], ctypes.c_int),
        "snn_result_csr": ([P, ctypes.POINTER(_CSR)], ctypes.c_int),
        "snn_result_copy": ([P, P, P, P, P], ctypes.c_int),
        "snn_result_copy_async": ([P, P, P, P, P], ctypes.c_int),
        "snn_result_free": ([P], None),
        "snn_result_free_async": ([P, P], None),
        "snn_free_async": ([P, P], None),
        "snn_pool_reserve": ([ctypes.c_uint64, P], ctypes.c_int),
        "snn_dbscan": ([P, f64, i32, P, ctypes.POINTER(i32), P], ctypes.c_int),
        "snn_free": ([P], None),
        "snn_last_error": ([], ctypes.c_char_p),
        "snn_index_info": ([P, ctypes.POINTER(_Info)], ctypes.c_int),
        "snn_index_sigma": ([P, i32, P, P], ctypes.c_int),
        "snn_launch_count": ([], ctypes.c_uint64),
        "snn_set_option": ([ctypes.c_char_p, i64], ctypes.c_int),
        "snn_get_option": ([ctypes.c_char_p, ctypes.c_void_p], ctypes.c_int),
        "snn_profile_enable": ([ctypes.c_int], ctypes.c_int),
        "snn_profile_read": ([ctypes.c_char_p, ctypes.POINTER(f64), ctypes.POINTER(ctypes.c_uint64),
                              ctypes.POINTER(f64)], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(st: int):
    if st != 0:
        raise SnnError(st, snn_last_error())


def _stream_ptr(stream=None):
    import torch
    if stream is None:
        if not torch.cuda.is_available():
            return None
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream) if hasattr(stream, "cuda_stream") else stream


def _ptr_dtype(X):
    """(pointer, n, d, dtype code, keepalive) for a torch tensor (cuda or cpu) or ndarray."""
    try:
        import torch
        is_t = isinstance(X, torch.Tensor)
    except ImportError:   # pragma: no cover
        is_t = False
    if is_t:
        if X.dim() != 2:
            raise ValueError("expected a 2-D tensor (n x d)")
        if X.dtype not in (torch.float32, torch.float64):
            raise TypeError("dtype must be float32 or float64")
        X = X.contiguous()
        code = SNN_F64 if X.dtype == torch.float64 else SNN_F32
        return ctypes.c_void_p(X.data_ptr()), X.shape[0], X.shape[1], code, X
    A = np.asarray(X)
    if A.ndim != 2:
        raise ValueError("expected a 2-D array (n x d)")
    if A.dtype not in (np.float32, np.float64):
        raise TypeError("dtype must be float32 or float64")
    A = np.ascontiguousarray(A)
    code = SNN_F64 if A.dtype == np.float64 else SNN_F32
    return ctypes.c_void_p(A.ctypes.data), A.shape[0], A.shape[1], code, A


# ------------------------------------------------------------------ C-ABI-named wrappers
def snn_last_error() -> str:
    return load_library().snn_last_error().decode()


def snn_launch_count() -> int:
    return int(load_library().snn_launch_count())


def snn_set_option(key: str, value: int) -> None:
    _check(load_library().snn_set_option(key.encode(), int(value)))


def snn_get_option(key: str) -> int:
    v = ctypes.c_int64(0)
    _check(load_library().snn_get_option(key.encode(), ctypes.addressof(v)))
    return int(v.value)


def snn_profile_enable(on: bool) -> None:
    _check(load_library().snn_profile_enable(1 if on else 0))


def snn_profile_read(family: str) -> dict:
    ms, n, u = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_double()
    _check(load_library().snn_profile_read(family.encode(), ctypes.byref(ms), ctypes.byref(n),
                                           ctypes.byref(u)))
    return {"ms": ms.value, "launches": int(n.value), "units": u.value}


def snn_build(X, stream=None):
    """Algorithm 1 -> opaque index handle (c_void_p)."""
    lib = load_library()
    p, n, d, code, _keep = _ptr_dtype(X)
    h = ctypes.c_void_p()
    _check(lib.snn_build(p, n, d, code, _stream_ptr(stream), ctypes.byref(h)))
    return h


def snn_build_metric(X, metric, stream=None):
    """snn_build for metric "euclidean" | "cosine" | "angular" (or its snn_metric code);
    cosine / angular normalize the rows on the device."""
    lib = load_library()
    code_m = METRICS[metric] if isinstance(metric, str) else int(metric)
    p, n, d, code, _keep = _ptr_dtype(X)
    h = ctypes.c_void_p()
    _check(lib.snn_build_metric(p, n, d, code, code_m, _stream_ptr(stream), ctypes.byref(h)))
    return h


def snn_query_radius(index, Q, R: float, stream=None):
    """Algorithm 2 for a batch of queries -> result handle."""
    lib = load_library()
    p, m, d, code, _keep = _ptr_dtype(Q)
    h = ctypes.c_void_p()
    _check(lib.snn_query_radius(index, p, m, d, code, float(R), _stream_ptr(stream), ctypes.byref(h)))
    return h


def snn_query_self(index, R: float, stream=None):
    lib = load_library()
    h = ctypes.c_void_p()
    _check(lib.snn_query_self(index, float(R), _stream_ptr(stream), ctypes.byref(h)))
    return h


def snn_query_radius_part(index, Q, R: float, part: int, nparts: int, stream=None):
    """This GPU's share of a sharded query: CSR over all queries, rows
    of other parts empty."""
    lib = load_library()
    p, m, d, code, _keep = _ptr_dtype(Q)
    h = ctypes.c_void_p()
    _check(lib.snn_query_radius_part(index, p, m, d, code, float(R), int(part), int(nparts),
                                     _stream_ptr(stream), ctypes.byref(h)))
    return h


def snn_query_self_part(index, R: float, part: int, nparts: int, stream=None):
    lib = load_library()
    h = ctypes.c_void_p()
    _check(lib.snn_query_self_part(index, float(R), int(part), int(nparts), _stream_ptr(stream), ctypes.byref(h)))
    return h


def snn_result_csr(result) -> dict:
    v = _CSR()
    _check(load_library().snn_result_csr(result, ctypes.byref(v)))
    return {"m": v.m, "nnz": v.nnz, "offsets": v.offsets, "indices": v.indices,
            "distances": v.distances}


def snn_result_copy(result, offsets, indices=None, distances=None, stream=None) -> None:
    """Copy into caller buffers (numpy arrays or torch tensors, host or device)."""
    def ptr(a):
        if a is None:
            return None
        if hasattr(a, "data_ptr"):
            return ctypes.c_void_p(a.data_ptr())
        return ctypes.c_void_p(a.ctypes.data)
    _check(load_library().snn_result_copy(result, ptr(offsets), ptr(indices), ptr(distances),
                                          _stream_ptr(stream)))


def snn_result_copy_async(result, offsets, indices=None, distances=None, stream=None) -> None:
    """Enqueue the copy on `stream` and return (buffers valid after the stream syncs; a
    later snn_result_free is ordered after the copy)."""
    def ptr(a):
        if a is None:
            return None
        if hasattr(a, "data_ptr"):
            return ctypes.c_void_p(a.data_ptr())
        return ctypes.c_void_p(a.ctypes.data)
    _check(load_library().snn_result_copy_async(result, ptr(offsets), ptr(indices), ptr(distances),
                                                _stream_ptr(stream)))


def snn_result_free(result) -> None:
    if result:
        load_library().snn_result_free(result)


def snn_free(index) -> None:
    if index:
        load_library().snn_free(index)


def snn_result_free_async(result, stream=None) -> None:
    if result:
        load_library().snn_result_free_async(result, _stream_ptr(stream))


def snn_pool_reserve(nbytes: int, stream=None) -> None:
    _check(load_library().snn_pool_reserve(int(nbytes), _stream_ptr(stream)))


def snn_free_async(index, stream=None) -> None:
    if index:
        load_library().snn_free_async(index, _stream_ptr(stream))


def snn_append(index, Y, stream=None) -> None:
    """Streaming append: rows Y (k x d) get ids n .. n+k-1; mu, v1 frozen."""
    p, k, d, code, _keep = _ptr_dtype(Y)
    _check(load_library().snn_append(index, p, k, d, code, _stream_ptr(stream)))


def snn_save(index, path: str, stream=None) -> None:
    _check(load_library().snn_save(index, os.fsencode(path), _stream_ptr(stream)))


def snn_load(path: str, stream=None):
    h = ctypes.c_void_p()
    _check(load_library().snn_load(os.fsencode(path), _stream_ptr(stream), ctypes.byref(h)))
    return h


def snn_index_sigma(index, k: int = 2, stream=None) -> np.ndarray:
    """The k largest singular values of the centred build data (eq:svd)."""
    out = np.zeros(int(k), dtype=np.float64)
    _check(load_library().snn_index_sigma(index, int(k), ctypes.c_void_p(out.ctypes.data), _stream_ptr(stream)))
    return out


def snn_index_info(index) -> dict:
    v = _Info()
    _check(load_library().snn_index_info(index, ctypes.byref(v)))
    return {f: getattr(v, f) for f, _ in _Info._fields_}


def snn_dbscan(index, eps: float, min_pts: int, labels, stream=None) -> int:
    """DBSCAN with the SNN backend; labels: int32 buffer (n), host or
    device, original order.  Returns the number of clusters K."""
    k = ctypes.c_int32()
    ptr = ctypes.c_void_p(labels.data_ptr() if hasattr(labels, "data_ptr") else labels.ctypes.data)
    _check(load_library().snn_dbscan(index, float(eps), int(min_pts), ptr, ctypes.byref(k),
                                     _stream_ptr(stream)))
    return int(k.value)


class _CAI:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2, "strides": None}


def device_view(ptr, shape, typestr):
    """Zero-copy torch view of library-owned device memory (typestr '<f4', '<f8', '<i4'...)."""
    import torch
    return torch.as_tensor(_CAI(ptr, shape, typestr), device="cuda")


def index_arrays(index) -> dict:
    """Copies (torch, cuda) of the Algorithm 1 outputs held by an index (diagnostics)."""
    info = snn_index_info(index)
    n, d, ld = info["n"], info["d"], info["ld"]
    xs_t = "<f8" if info["dtype"] == SNN_F64 else "<f4"
    if ld == 0:   # AoSoA4: element (i, k) at xs[(i/4)*4d + k*4 + i%4]
        n_pad = (n + 3) // 4 * 4
        xs = device_view(info["xs"], (n_pad // 4, d, 4), xs_t).permute(0, 2, 1).reshape(n_pad, d)[:n]
    else:
        xs = device_view(info["xs"], (n, ld), xs_t)
    return {"mu": device_view(info["mu"], (d,), "<f8").clone(),
            "v1": device_view(info["v1"], (d,), "<f4").clone(),
            "keys": device_view(info["keys"], (n,), "<f4").clone(),
            "perm": device_view(info["perm"], (n,), "<i4").clone(),
            "xbar": device_view(info["xbar"], (n,), "<f4").clone(),
            "xs": xs.clone(),
            "info": info}


# ------------------------------------------------------------------ convenience layer
@dataclass
class CSR:
    offsets: object     # (m+1,) int64
    indices: object     # (nnz,) int32 original ids
    distances: object   # (nnz,) float32

    @property
    def m(self):
        return len(self.offsets) - 1

    @property
    def nnz(self):
        return int(self.offsets[-1])

    def row(self, j):
        o = self.offsets
        return self.indices[int(o[j]):int(o[j + 1])], self.distances[int(o[j]):int(o[j + 1])]


def _fetch(result, device: str, stream=None) -> CSR:
    v = snn_result_csr(result)
    m, nnz = v["m"], v["nnz"]
    if device == "cpu":
        off = np.empty(m + 1, dtype=np.int64)
        idx = np.empty(nnz, dtype=np.int32)
        dist = np.empty(nnz, dtype=np.float32)
    else:
        import torch
        off = torch.empty(m + 1, dtype=torch.int64, device=device)
        idx = torch.empty(nnz, dtype=torch.int32, device=device)
        dist = torch.empty(nnz, dtype=torch.float32, device=device)
    snn_result_copy(result, off, idx if nnz else None, dist if nnz else None, stream)
    return CSR(off, idx, dist)


class Index:
    """Owns an SNN index built on the current CUDA device (Algorithm 1)."""

    def __init__(self, X, stream=None, metric: str = "euclidean", _handle=None):
        self._h = _handle if _handle is not None else snn_build_metric(X, metric, stream)
        self._sync()

    def _sync(self):
        info = snn_index_info(self._h)
        self.n, self.d = int(info["n"]), int(info["d"])
        self.dtype = "f64" if info["dtype"] == SNN_F64 else "f32"
        self.metric = {v: k for k, v in METRICS.items()}[int(info["metric"])]

    @classmethod
    def load(cls, path: str, stream=None) -> "Index":
        return cls(None, _handle=snn_load(path, stream))

    def save(self, path: str, stream=None) -> None:
        snn_save(self._h, path, stream)

    def append(self, Y, stream=None) -> None:
        snn_append(self._h, Y, stream)
        self._sync()

    def info(self) -> dict:
        return snn_index_info(self._h)

    def sigma(self, k: int = 2) -> np.ndarray:
        return snn_index_sigma(self._h, k)

    def arrays(self) -> dict:
        return index_arrays(self._h)

    def query(self, Q, R: float, device: str = "cpu", stream=None, part: int = 0, nparts: int = 1) -> CSR:
        r = (snn_query_radius(self._h, Q, R, stream) if nparts == 1
             else snn_query_radius_part(self._h, Q, R, part, nparts, stream))
        try:
            return _fetch(r, device, stream)
        finally:
            snn_result_free(r)

    def query_self(self, R: float, device: str = "cpu", stream=None, part: int = 0, nparts: int = 1) -> CSR:
        r = (snn_query_self(self._h, R, stream) if nparts == 1
             else snn_query_self_part(self._h, R, part, nparts, stream))
        try:
            return _fetch(r, device, stream)
        finally:
            snn_result_free(r)

    def dbscan(self, eps: float, min_pts: int, stream=None):
        labels = np.empty(self.n, dtype=np.int32)
        K = snn_dbscan(self._h, eps, min_pts, labels, stream)
        return labels, K

    def free(self):
        if self._h:
            snn_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
