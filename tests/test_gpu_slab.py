"""The opt-in bucket-major slab form of the full sweeps (csrc/im_slab.cu, IM_SLAB_PASSES) against the oracle.

The knobs are read once per process, so the parity tests run in a child process with the slab path forced
on for every constant-threshold graph (IM_SLAB_MIN_M=0): registers after the first build and after blocked
rebuilds, seeds, scores and decisions are compared with the oracle exactly as in test_gpu_parity.py.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_slab_path_parity_in_child_process():
    env = dict(os.environ, IM_SLAB_PASSES="3", IM_SLAB_MIN_M="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_parity.py",
                        "tests/test_gpu_configs.py::test_c1_full_parity_live_oracle", "tests/test_gpu_configs.py::test_c3_parity"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
