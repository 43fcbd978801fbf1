"""Run one piece of the hot path once (for ncu / compute-sanitizer captures).

    python tools/profile_step.py --config c3 --what build      # load + first build
    python tools/profile_step.py --config c4 --what step       # load + build + estimate + select
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2105_04023_b200 as im  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--what", default="build", choices=["build", "step"])
ap.add_argument("--K", type=int)
ap.add_argument("--J", type=int, help="C5-style override of J (with --p / --t)")
ap.add_argument("--p", type=float)
ap.add_argument("--t", type=float)
a = ap.parse_args()
cfg = gen.CONFIGS[a.config]
n, off, tgt, pr = gen.workload(cfg)
if a.p is not None:
    import dataclasses

    import numpy as np

    pr = np.full(len(tgt), a.p, np.float32)
    cfg = dataclasses.replace(cfg, J=a.J or cfg.J, t=cfg.t if a.t is None else a.t)
elif a.J:
    import dataclasses

    cfg = dataclasses.replace(cfg, J=a.J)
t = time.time()
im.im_load_csr(n, off, tgt, pr)
im.im_build_sketches(cfg.J, cfg.salt_seed)
st = im.im_get_stats()
if a.what == "step":
    im.im_estimate(n)
    s, sc = im.im_select_seeds(a.K or cfg.K, cfg.t)
    st = im.im_get_stats()
print({k: st[k] for k in ("last_build_sweeps", "total_sweeps", "total_edges", "window_edges", "sweep_kernel_ms", "rebuilds",
                          "bfs_levels", "bfs_edges", "last_select_ms")}, f"{time.time() - t:.2f}s", flush=True)
im.im_free()
