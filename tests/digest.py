"""Order-independent digests of radius-query results and DBSCAN labelings (test
infrastructure; no arithmetic of the method).

Full-size oracle results (config 2: 38.7M pairs; config 5: 2M labels) are too large to
store, so ``scripts/make_digests.py`` stores, per configuration, every row's hit count plus
a 64-bit digest per block of rows, computed from the oracle's CSR; the GPU test computes the
same digests from the CUDA path's CSR and compares them block by block.

pair hash   h(row, id, dist) = mix64(mix64(row) ^ (id << 32 | float32 bits of dist))
row digest  sum of the pair hashes of the row (mod 2^64: independent of the order inside a row)
block       sum of the row digests of ``block`` consecutive rows
label hash  mix64(mix64(i) ^ (label + 1)), summed per block of points
mix64 = the SplitMix64 finaliser.  Distances are float32(sqrt(fp64 s)) -- the bit pattern
the exactness contract fixes.
"""
from __future__ import annotations

import hashlib

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def mix64(x: np.ndarray) -> np.ndarray:
    z = np.asarray(x, dtype=np.uint64) + _G
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _seg_sums(h: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    cs = np.zeros(len(h) + 1, dtype=np.uint64)
    np.cumsum(h, dtype=np.uint64, out=cs[1:])
    offsets = np.asarray(offsets, dtype=np.int64)
    return cs[offsets[1:]] - cs[offsets[:-1]]


def csr_digests(offsets, indices, dist_f32, block: int = 1024, row0: int = 0):
    """(counts int64[m], block digests uint64[ceil(m/block)]) of a CSR result whose
    distances are float32; its row j is query row0 + j of the whole result."""
    offsets = np.asarray(offsets, dtype=np.int64)
    m = len(offsets) - 1
    counts = np.diff(offsets)
    rows = np.repeat(np.arange(row0, row0 + m, dtype=np.uint64), counts)
    bits = np.ascontiguousarray(dist_f32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    key = (np.asarray(indices).astype(np.uint64) << np.uint64(32)) | bits
    h = mix64(mix64(rows) ^ key)
    del rows, key, bits
    row_dig = _seg_sums(h, offsets)
    boff = np.minimum(np.arange(0, m + block, block, dtype=np.int64), m)
    boff = np.unique(boff) if m else np.zeros(1, dtype=np.int64)
    return counts, _seg_sums(row_dig, boff)


def oracle_csr_digests(res: dict, block: int = 1024, row0: int = 0):
    """Digests of an oracle.radius_query result (for queries row0, row0 + 1, ...): hits
    only (s <= R*R), distance = float32(sqrt(s))."""
    keep = res["s"] <= res["R2"]
    off = np.asarray(res["offsets"], dtype=np.int64)
    rows = np.repeat(np.arange(len(off) - 1), np.diff(off))
    cnt = np.bincount(rows[keep], minlength=len(off) - 1)
    noff = np.zeros(len(off), dtype=np.int64)
    np.cumsum(cnt, out=noff[1:])
    return csr_digests(noff, res["indices"][keep], np.sqrt(res["s"][keep]).astype(np.float32), block, row0)


def label_digests(labels, block: int = 4096) -> np.ndarray:
    labels = np.asarray(labels, dtype=np.int64)
    n = len(labels)
    h = mix64(mix64(np.arange(n, dtype=np.uint64)) ^ (labels + 1).astype(np.uint64))
    boff = np.unique(np.minimum(np.arange(0, n + block, block, dtype=np.int64), n))
    return _seg_sums(h, boff)


def sha256(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
