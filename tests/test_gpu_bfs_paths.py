"""The seed diffusion (Alg. 1 lines 13-14) has two GPU paths: the multi-block level kernels and the
single-block small-frontier kernel (im_bfs_small.cu), with hand-overs both ways inside one BFS.
IM_SMALL_EDGES (read when the library context starts) picks the split, so each setting runs in
its own process: 0 = multi-block only, a huge value = single-block only, 64 = frequent hand-overs.
Every setting must give the oracle's seeds, sigma counts, step log and R_G(S) bit for bit."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import math, sys
import numpy as np
sys.path.insert(0, %(root)r)
from tests import brute
from tests.test_gpu_parity import compare_select
import gen, oracle
rng = np.random.default_rng(2024)
for g in range(4):
    n = int(rng.integers(300, 2500))
    off, tgt, pr = brute.random_graph(rng, n, 6 * n, [0.05, 0.1, None, 0.3][g], allow_dups=False, allow_loops=False)
    compare_select(n, off, tgt, pr, [64, 128, 256, 32][g], int(rng.integers(0, 2**32)), 12, [0.05, 0.0, 0.3, math.inf][g])
cfg = gen.CONFIGS["c1"]
n, off, tgt, pr = gen.workload(cfg)
compare_select(n, off, tgt, pr, cfg.J, cfg.salt_seed, cfg.K, cfg.t)
print("ok")
"""


@pytest.mark.parametrize("small_edges", ["0", "1000000000", "64"])
def test_select_parity_bfs_paths(small_edges):
    env = dict(os.environ, IM_SMALL_EDGES=small_edges)
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], env=env, cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]
