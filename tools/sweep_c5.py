"""C5 (BASELINE.json config 5): the parameter sweep on the C3 Chung-Lu graph,
J in {64..1024} x constant p in {0.005, 0.01, 0.1} x error threshold t in {0.01, 0.05, 0.3}, K = 100.
Per point: first sketch build (ms, sweeps, edge x simulation updates per second of its sweep
kernels), seed selection (ms, rebuilds, sigma of the K seeds), and the whole IM time.  One JSON line
per point on stdout, a summary table on stderr.  Device timing: CUDA events on the library's stream
(torch's current stream) around the C-ABI calls (inputs already on the device), median of --reps runs
per point; nvidia-smi clocks sampled over the whole grid (bench.py's Clocks); the sweep kernels'
SURVEY 8(d) roofline fraction per point (bench.py's definition).

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
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--only", help="comma-separated J:p[:t] filters, e.g. 256:0.1,128:0.1:0.05 (A/B runs)")
a = ap.parse_args()
import statistics  # noqa: E402

import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

stream = torch.cuda.current_stream()
im.im_set_stream(stream)
peak, peak_kind, _ = bench.load_peaks()
clocks = bench.Clocks(0)
n, off, tgt = gen.graph("cl4m")
m = len(tgt)
grid = gen.C5_GRID
if a.points == "corners":
    grid = [g for g in grid if g[0] in (64, 1024) and g[2] in (0.01, 0.3)]
if a.only:
    flt = [tuple(float(x) for x in f.split(":")) for f in a.only.split(",")]
    grid = [g for g in grid if any(g[0] == f[0] and g[1] == f[1] and (len(f) < 3 or g[2] == f[2]) for f in flt)]
rows = []
for p in sorted({g[1] for g in grid}):
    pr = np.full(m, p, np.float32)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(max(g[0] for g in grid), 1)  # untimed: device buffers sized for the largest J
    for J, p2, t in grid:
        if p2 != p:
            continue
        reps = []
        for _ in range(a.reps):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            im.im_build_sketches(J, 1)
            e1.record(stream)
            sb = im.im_get_stats()
            seeds, scores = im.im_select_seeds(a.K, t)
            e2.record(stream)
            torch.cuda.synchronize()
            ss = im.im_get_stats()
            reps.append((e0.elapsed_time(e1), e1.elapsed_time(e2), sb, ss, seeds, scores))
        reps.sort(key=lambda x: x[0] + x[1])
        bms, sms, sb, ss, seeds, scores = reps[len(reps) // 2]
        # SURVEY 8(d) sweep-kernel roofline of the whole point (build + rebuilds), bench.py's definition
        edges = sb["total_edges"] + ss["total_edges"]
        full = 1 + ss["rebuilds"] + sb["gather_sweeps"] + ss["gather_sweeps"]
        alg = edges * (8.0 + J * (1.0 - (1.0 - p) ** 32)) + full * n * (8.0 + 2.0 * J) + ss["rebuilds"] * n * J / 8.0
        sweep_ms = sb["sweep_kernel_ms"] + ss["sweep_kernel_ms"]
        r = {"J": J, "p": p, "t": t, "K": a.K, "n": n, "m": m,
             "build_ms": bms, "build_sweeps": sb["last_build_sweeps"],
             "build_gedge_sims_per_s": sb["last_build_edges"] * J / max(sb["sweep_kernel_ms"], 1e-9) / 1e6,
             "select_ms": sms, "rebuilds": ss["rebuilds"], "sweeps_in_select": ss["total_sweeps"],
             "bfs_levels": ss["bfs_levels"], "im_ms": bms + sms, "sigma_K": float(scores[-1]),
             "sweep_kernel_ms": sweep_ms, "roofline_frac_8d": alg / (sweep_ms / 1e3) / 1e9 / peak if sweep_ms else None,
             "reps": a.reps, "seeds_head": [int(x) for x in seeds[:3]]}
        rows.append(r)
        print(json.dumps(r), flush=True)
clk = clocks.stop()
print(json.dumps({"clocks": clk, "peak_gbs": peak, "peak_kind": peak_kind}), flush=True)
print(f"{'J':>5} {'p':>6} {'t':>5} {'build ms':>9} {'sweeps':>6} {'G e*s/s':>8} {'select ms':>9} {'rebuilds':>8} {'IM ms':>8} {'sigma':>10} {'frac8d':>6}",
      file=sys.stderr)
for r in rows:
    print(f"{r['J']:5d} {r['p']:6.3f} {r['t']:5.2f} {r['build_ms']:9.1f} {r['build_sweeps']:6d} {r['build_gedge_sims_per_s']:8.0f} "
          f"{r['select_ms']:9.1f} {r['rebuilds']:8d} {r['im_ms']:8.1f} {r['sigma_K']:10.1f} {r['roofline_frac_8d'] or 0:6.3f}", file=sys.stderr)
print(f"clocks: {clk}", file=sys.stderr)
im.im_free()
