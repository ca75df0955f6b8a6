"""Runs the window and sequence parity suites against libmdhp_debug.so (-DMDHP_DEBUG: device-side
bounds asserts on marks, chunk offsets, window slots, permutation slots).  compute-sanitizer is
closed on this GPU pool, so this is the memory-safety check of the hot-path kernels."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_parity_suites_under_bounds_asserts():
    from paper_2411_10258_b200 import build
    lib = build.build(debug=True)
    env = dict(os.environ, MDHP_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_gpu_seq.py", "tests/test_gpu_dense.py",
                        "tests/test_gpu_fuzz.py", "tests/test_gpu_shard.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "passed" in r.stdout
