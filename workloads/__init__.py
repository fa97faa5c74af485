"""Seeded synthetic inputs for the five BASELINE.json configs (and scaled-down variants).

This module is shared by the oracle side (tests, `bench.py --impl reference`) and the
CUDA side (tests, `bench.py`, `smoke()`).  It holds NO arithmetic of the method (no
centering, projection, sorting or distances) -- only the random draws that define the
workloads, so that both sides see bit-identical inputs.

Recipes follow SURVEY.md §8(c) reading C17 (numpy ``default_rng`` = PCG64):

* C1  n=m=2,000, d=2, fp64 i.i.d. uniform [0,1)^2, seed 0, self-query, R=0.05
      (the paper's own synthetic setup, §6.1; Table 1 cell n=2000, R=0.05,
      PAPER.md:401).
* C2  n=1,000,000, d=3, fp32 mixture of 64 isotropic Gaussians (centers U[0,100)^3,
      sigma=2, equal weights), seed 1, self-query.
* C3  n=200,000, m=20,000, d=64, fp32 N(0, diag(1/i)) rotated by a Haar orthogonal
      matrix, seed 2 (stand-in for the d~100 descriptor sets).
* C4  n=500,000, m=10,000, d=784, fp32 non-negative rank-32 factor product, rescaled to
      max 1, ~80% zeros, seed 3 (stand-in for F-MNIST's shape).
* C5  n=2,000,000, d=2, fp32: 20 Gaussian clusters (centers U[0,1000)^2, sigma U[5,20])
      + 10% uniform background, seed 4; DBSCAN eps=3, minPts=5 (stand-in for the UCI
      DBSCAN runs).

The radii of C2-C4 are NOT computed here (that needs distances, i.e. the oracle): they
are read from ``radii.json``, written by ``scripts/select_radii.py`` which calls only
``oracle/``.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
RADII_PATH = os.path.join(_HERE, "radii.json")


@dataclass
class Workload:
    name: str
    X: np.ndarray                 # n x d, row-major, float32 or float64
    Q: np.ndarray | None          # m x d queries; None => self-query (Q = X)
    R: float | None               # radius (None if not yet selected)
    dbscan_min_pts: int | None = None
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.X.shape[0])

    @property
    def d(self) -> int:
        return int(self.X.shape[1])

    @property
    def m(self) -> int:
        return self.n if self.Q is None else int(self.Q.shape[0])

    @property
    def queries(self) -> np.ndarray:
        return self.X if self.Q is None else self.Q


def load_radii() -> dict:
    if not os.path.exists(RADII_PATH):
        return {}
    with open(RADII_PATH) as f:
        return json.load(f)


def _radius(key: str):
    r = load_radii().get(key)
    return None if r is None else float(r["R"])


# ----------------------------------------------------------------------------- C1
def c1(n: int = 2000, seed: int = 0) -> Workload:
    rng = np.random.default_rng(seed)
    X = rng.random((n, 2))                                 # float64
    return Workload(f"c1_uniform2d_n{n}", np.ascontiguousarray(X), None, 0.05)


def uniform(n: int, d: int, seed: int, dtype=np.float64, R: float | None = None) -> Workload:
    """Uniform [0,1)^d, the paper's synthetic distribution."""
    rng = np.random.default_rng(seed)
    X = rng.random((n, d)).astype(dtype)
    return Workload(f"uniform_d{d}_n{n}_s{seed}", np.ascontiguousarray(X), None, R)


# ----------------------------------------------------------------------------- C2
def c2(n: int = 1_000_000, seed: int = 1, k: int = 64, sigma: float = 2.0,
       box: float = 100.0) -> Workload:
    rng = np.random.default_rng(seed)
    centers = rng.random((k, 3)) * box
    labels = rng.integers(0, k, n)
    X = centers[labels] + sigma * rng.standard_normal((n, 3))
    X = np.ascontiguousarray(X.astype(np.float32))
    key = "c2" if (n, seed, k, sigma, box) == (1_000_000, 1, 64, 2.0, 100.0) else None
    return Workload(f"c2_gmm3d_n{n}", X, None, _radius(key) if key else None,
                    meta={"k": k, "sigma": sigma, "box": box})


# ----------------------------------------------------------------------------- C3
def _haar_orthogonal(rng: np.random.Generator, d: int) -> np.ndarray:
    G = rng.standard_normal((d, d))
    Qo, Rr = np.linalg.qr(G)
    return Qo * np.sign(np.diag(Rr))[None, :]


def c3(n: int = 200_000, m: int = 20_000, seed: int = 2, d: int = 64) -> Workload:
    rng = np.random.default_rng(seed)
    Qo = _haar_orthogonal(rng, d)
    scale = (1.0 / np.sqrt(np.arange(1, d + 1, dtype=np.float64)))[None, :]
    X = (rng.standard_normal((n, d)) * scale) @ Qo
    Q = (rng.standard_normal((m, d)) * scale) @ Qo
    key = "c3" if (n, m, seed, d) == (200_000, 20_000, 2, 64) else None
    return Workload(f"c3_aniso{d}_n{n}_m{m}", np.ascontiguousarray(X.astype(np.float32)),
                    np.ascontiguousarray(Q.astype(np.float32)),
                    _radius(key) if key else None, meta={"Qo": Qo})


# ----------------------------------------------------------------------------- C4
def c4(n: int = 500_000, m: int = 10_000, seed: int = 3, d: int = 784, rank: int = 32,
       zero_frac: float = 0.8, chunk: int = 65536) -> Workload:
    """Rank-`rank` factor product, rescaled to max 1, ~`zero_frac` zeros.

    Rows are produced in chunks of `chunk` rows (A, B drawn first; then the zero mask is
    drawn chunk by chunk in row order, which is the same PCG64 stream as one big draw).
    """
    rng = np.random.default_rng(seed)
    N = n + m
    A = rng.random((N, rank))
    B = rng.random((rank, d))
    ymax = 0.0
    for s in range(0, N, chunk):
        ymax = max(ymax, float((A[s:s + chunk] @ B).max()))
    Y = np.empty((N, d), dtype=np.float32)
    for s in range(0, N, chunk):
        blk = (A[s:s + chunk] @ B) / ymax
        blk[rng.random(blk.shape) < zero_frac] = 0.0
        Y[s:s + chunk] = blk.astype(np.float32)
    key = "c4" if (n, m, seed, d, rank, zero_frac) == (500_000, 10_000, 3, 784, 32, 0.8) else None
    return Workload(f"c4_lowrank{d}_n{n}_m{m}", np.ascontiguousarray(Y[:n]),
                    np.ascontiguousarray(Y[n:]), _radius(key) if key else None)


# ----------------------------------------------------------------------------- C5
def c5(n: int = 2_000_000, seed: int = 4, k: int = 20, box: float = 1000.0,
       noise_frac: float = 0.1, eps: float = 3.0, min_pts: int = 5) -> Workload:
    rng = np.random.default_rng(seed)
    centers = rng.random((k, 2)) * box
    sig = rng.uniform(5.0, 20.0, k)
    n_bg = int(round(noise_frac * n))
    n_cl = n - n_bg
    labels = rng.integers(0, k, n_cl)
    pts = centers[labels] + sig[labels, None] * rng.standard_normal((n_cl, 2))
    bg = rng.random((n_bg, 2)) * box
    X = np.concatenate([pts, bg], axis=0)
    X = X[rng.permutation(n)]
    return Workload(f"c5_dbscan2d_n{n}", np.ascontiguousarray(X.astype(np.float32)), None,
                    eps, dbscan_min_pts=min_pts)


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
