"""Small tensor-core path check against the oracle (debug driver)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2212_07679_b200 as snn  # noqa: E402
from tests.parity import compare  # noqa: E402

for (n, m, d, seed) in [(700, 77, 64, 10), (3000, 500, 64, 1), (1000, 130, 100, 2), (600, 40, 784, 3)]:
    rng = np.random.default_rng(seed)
    X = (rng.standard_normal((n, d)) * rng.uniform(0.5, 3, d)).astype(np.float32)
    Q = (rng.standard_normal((m, d)) * rng.uniform(0.5, 3, d)).astype(np.float32)
    R = float(np.quantile(np.linalg.norm(X[:200, None, :].astype(np.float64) - Q[None, :50, :], axis=-1), 0.05))
    idx = snn.Index(torch.from_numpy(X).cuda())
    print("tc" , idx.info()["ld"], flush=True)
    res = idx.query(torch.from_numpy(Q).cuda(), R)
    ora = oracle.radius_query(X, Q, R)
    st = compare(res, ora)
    print(n, m, d, st, "rejected", snn.snn_profile_read("overflow")["units"], flush=True)
    idx.free()
print("TC OK")
