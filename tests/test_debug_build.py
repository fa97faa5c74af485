"""The debug build (lib/libsnn_debug.so, -DSNN_DEBUG: device-side bounds checks
SNN_DASSERT in the compaction, row assembly, pair lists, union-find and window locate)
runs the small parity suite cleanly -- the stand-in for compute-sanitizer, which this GPU
pool does not allow.  A failed check traps, the call returns
SNN_ERR_CUDA and the inner test fails."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_library_has_bounds_checks():
    from paper_2212_07679_b200 import build_lib
    path = build_lib.build(debug=True)
    strings = subprocess.check_output(["strings", path]).decode(errors="ignore")
    assert "SNN_DASSERT failed" in strings
    plain = subprocess.check_output(["strings", build_lib.build()]).decode(errors="ignore")
    assert "SNN_DASSERT failed" not in plain


@pytest.mark.gpu
def test_small_parity_suite_under_bounds_checks():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_07679_b200 import build_lib
    path = build_lib.build(debug=True)
    env = dict(os.environ, SNN_LIB=path)
    sel = ("random_parity or self_query_parity or scaled_configs or dbscan_full_parity or dbscan_high_d "
           "or row_staging or tc_csr_row_sizes or everything_is_a_neighbour or overflow or edge_cases "
           "or concurrent or save_load")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", sel,
                        os.path.join(ROOT, "tests", "test_gpu_parity.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "SNN_DASSERT failed" not in r.stdout + r.stderr
    assert " passed" in r.stdout, tail
