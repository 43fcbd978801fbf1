"""C5 (BASELINE.json config 5): the parameter sweep on the C3 Chung-Lu graph,
J in {64..1024} x constant p in {0.005, 0.01, 0.1} x error threshold t in {0.01, 0.05, 0.3}, K = 100.
Per point: first sketch build (ms, sweeps, edge x simulation updates per second of its sweep
kernels), seed selection (ms, rebuilds, sigma of the K seeds), and the whole IM time.  One JSON line
per point on stdout, a summary table on stderr.  Device timing: the library's own CUDA-event sweep
times and host wall clock around the synchronous C-ABI calls (inputs already on the device).

    python tools/sweep_c5.py [--K 100] [--points all|corners] > profiles/rXX_c5_grid.jsonl
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import gen  # noqa: E402
import paper_2105_04023_b200 as im  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=100)
ap.add_argument("--points", default="all", choices=["all", "corners"])
a = ap.parse_args()
n, off, tgt = gen.graph("cl4m")
m = len(tgt)
grid = gen.C5_GRID
if a.points == "corners":
    grid = [g for g in grid if g[0] in (64, 1024) and g[2] in (0.01, 0.3)]
rows = []
for p in sorted({g[1] for g in grid}):
    pr = np.full(m, p, np.float32)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(max(g[0] for g in grid), 1)  # untimed: device buffers sized for the largest J
    for J, p2, t in grid:
        if p2 != p:
            continue
        t0 = time.perf_counter()
        im.im_build_sketches(J, 1)
        t1 = time.perf_counter()
        sb = im.im_get_stats()
        seeds, scores = im.im_select_seeds(a.K, t)
        t2 = time.perf_counter()
        ss = im.im_get_stats()
        r = {"J": J, "p": p, "t": t, "K": a.K, "n": n, "m": m,
             "build_ms": (t1 - t0) * 1e3, "build_sweeps": sb["last_build_sweeps"],
             "build_gedge_sims_per_s": sb["last_build_edges"] * J / max(sb["sweep_kernel_ms"], 1e-9) / 1e6,
             "select_ms": (t2 - t1) * 1e3, "rebuilds": ss["rebuilds"], "sweeps_in_select": ss["total_sweeps"],
             "bfs_levels": ss["bfs_levels"], "im_ms": (t2 - t0) * 1e3, "sigma_K": float(scores[-1]),
             "seeds_head": [int(x) for x in seeds[:3]]}
        rows.append(r)
        print(json.dumps(r), flush=True)
print(f"{'J':>5} {'p':>6} {'t':>5} {'build ms':>9} {'sweeps':>6} {'G e*s/s':>8} {'select ms':>9} {'rebuilds':>8} {'IM ms':>8} {'sigma':>10}",
      file=sys.stderr)
for r in rows:
    print(f"{r['J']:5d} {r['p']:6.3f} {r['t']:5.2f} {r['build_ms']:9.1f} {r['build_sweeps']:6d} {r['build_gedge_sims_per_s']:8.0f} "
          f"{r['select_ms']:9.1f} {r['rebuilds']:8d} {r['im_ms']:8.1f} {r['sigma_K']:10.1f}", file=sys.stderr)
im.im_free()
