"""Small whole-path runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

Covers every kernel family of the library on small inputs: edge prep (constant and per-edge
thresholds, general and rows paths), first sweep + push / gather sweeps (in place and
synchronous, eps_c > 0), blocked rebuilds, estimate, lazy / full argmax, the three BFS paths,
the Monte-Carlo evaluator.  Parity is the tests' job; this only drives the kernels.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_2105_04023_b200 as im  # noqa: E402


def rand_graph(n, m, seed, wc=False, p=0.05):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    hub = rng.integers(0, n)
    src[: m // 8] = hub  # one long row (block gather, hash slices)
    order = np.argsort(src, kind="stable")
    src, dst = src[order], dst[order]
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, src + 1, 1)
    off = np.cumsum(off).astype(np.int32)
    pr = (rng.random(m).astype(np.float32) * 0.2) if wc else np.full(m, p, np.float32)
    return n, off, dst.astype(np.int32), pr


def run(n, off, tgt, pr, J, K, t, eps_c=0.0):
    im.im_set_policy(float("nan"), float("nan"), eps_c)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(J, 1)
    im.im_estimate(n)
    s, _ = im.im_select_seeds(K, t)
    im.im_evaluate(s, 7, 64)
    st = im.im_get_stats()
    print(f"n={n} m={len(tgt)} J={J} K={K} t={t} eps_c={eps_c}: seeds {list(s)[:4]} rebuilds {st['rebuilds']} "
          f"sweeps {st['total_sweeps']} bfs levels {st['bfs_levels']}", flush=True)


def main():
    cfg = gen.CONFIGS["c1"]
    n, off, tgt, pr = gen.workload(cfg)
    run(n, off, tgt, pr, cfg.J, cfg.K, cfg.t)
    run(n, off, tgt, pr, 256, 5, 0.3, eps_c=0.02)
    for seed, wc, J, p in [(1, False, 64, 0.05), (2, True, 128, 0.0), (3, False, 1024, 0.1), (4, False, 256, 0.01)]:
        g = rand_graph(4000, 40000, seed, wc=wc, p=p)
        run(*g, J, 6, 0.05)
    im.im_free()
    print("sanitize run done")


if __name__ == "__main__":
    main()
