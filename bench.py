#!/usr/bin/env python
"""Benchmark of the hot path (one JSON line on rank 0).

A step = one pass of the whole hot path over one synthetic workload:
edge prep (im_load_csr*), sketch build (im_build_sketches), per-vertex estimate
(im_estimate*), and the K-step error-adaptive selection with its BFS diffusions and rebuilds
(im_select_seeds).

value : processed edge x simulation updates per second over the whole step
        (sum over every sweep of every build/rebuild of [enumerated edges x J] / step time),
        inputs resident in HBM when the timed region starts.
e2e   : the same metric through the C ABI with HOST (pinned) buffers: H2D of the CSR and the
        D2H of estimates and seeds inside the timed region.
roofline : the sweep kernel (dominant), algorithmic bytes / CUDA-event
        kernel time vs the measured HBM copy bandwidth of MEASURED_PEAKS.json.
cpu_baseline : the oracle (oracle/, plain single-threaded C) on a bounded sample of the same
        workload: the first Alg. 2 sweep over a vertex range, on the host.

multi-GPU (torchrun, N > 1): --mode shard (default) splits the J simulations of the one job over
        the ranks (im_build_sketches_shard + the library's NCCL communicator: reduce-
        scatter / max all-reduce / all-gather per argmax pass, sum all-reduces of score and sigma;
        strong scaling, value = all ranks' updates / max time);
        --mode replicas runs N independent copies of the job (weak scaling).

    python bench.py [--config c4] [--steps 3] [--warmup 3] [--gpus N] [--impl ours|reference] [--mode shard|replicas]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gen  # noqa: E402

METRIC = "sketch-build G edge·sims/s (processed edge x simulation updates per second, whole K-seed IM step)"
UNIT = "G edge·sims/s"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured", float(d.get("sm_max_mhz", 1965.0))
    return 6650.0, "fallback", 1965.0


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu_index: int):
        self.path = tempfile.mktemp(prefix="clocks", suffix=".csv")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline_subprocess(config, seconds=12.0):
    """The oracle leg in its own process (tools/cpu_baseline.py): this process never maps liboracle.so."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "cpu_baseline.py"), "--config", config,
                        "--seconds", str(seconds)], capture_output=True, text=True)
    if r.returncode != 0:
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": f"failed: {r.stderr[-300:]}"}
    return json.loads(r.stdout.strip().splitlines()[-1])


def run_reference(args, rank):
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import cpu_baseline  # the oracle leg (reference arm: the oracle IS the reference here)

    cfg = gen.CONFIGS[args.config]
    n, off, tgt, pr = gen.workload(cfg)
    vals = []
    for _ in range(args.warmup):
        pass  # the oracle has no warm-up effects beyond page faults handled inside its setup
    for _ in range(args.steps):
        vals.append(cpu_baseline.oracle_sample(cfg, n, off, tgt, pr, target_s=args.ref_seconds))
    v = statistics.median([x["value"] for x in vals])
    cb = dict(vals[-1])
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": statistics.median([x["seconds"] for x in vals]) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8/u32", "data": "synthetic",
            "config": config_dict(cfg, n, len(tgt), args), "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def latest_capture(config):
    """The newest committed ncu capture of the sweep kernels for this config (profiles/*_traffic_<cfg>.json,
    written by tools/ncu_summary.py traffic), by its recorded round tag, not by file name."""
    pdir = os.path.join(ROOT, "profiles")
    best = None
    if os.path.isdir(pdir):
        for f in os.listdir(pdir):
            if f.endswith(f"_traffic_{config}.json"):
                try:
                    tj = json.load(open(os.path.join(pdir, f)))
                    tj["sweep"]["dram_bytes_per_step"]
                except (ValueError, KeyError, TypeError):
                    continue  # an unusable capture is ignored
                key = (tj.get("round", f[:4]), f)
                if best is None or key > best[0]:
                    best = (key, f, tj)
    return (best[1], best[2]) if best else (None, None)


def roofline(cfg, n, m, pr, J, edges, full_sweeps, blocked_full, builder_bytes, sweep_ms, step_ms, peak, peak_kind, config):
    """SURVEY.md 8(d) algorithmic bytes of the sweep kernels (Alg. 2) per step, over their CUDA-event time:
      per enumerated edge  : 4 B target + 4 B hash (+ 4 B threshold when w varies)
                             + the live sectors of the target row, J * (1 - (1 - p)^32) B
                               (a 32-register sector is needed iff one of its 32 simulations is live;
                                WC: the mean of that over the edges);
      per vertex of a full-vertex sweep (first sweep of every build, gather sweeps):
                               8 B offsets + J B own-row read + J B row write (+ J/8 B blocked bits in rebuilds).
    edges = enumerated edges of all sweeps of the step (im_stats total_edges)."""
    rec = 8.0 + (0.0 if cfg.p is not None else 4.0)
    pe = float(cfg.p) if cfg.p is not None else None
    live = J * (1.0 - (1.0 - pe) ** 32) if pe is not None else float(J * np.mean(1.0 - (1.0 - pr.astype(np.float64)) ** 32))
    per_vertex = 8.0 + 2.0 * J
    alg = edges * (rec + live) + full_sweeps * n * per_vertex + blocked_full * n * J / 8.0
    s = sweep_ms / 1e3
    achieved = alg / s / 1e9 if s > 0 else None
    src, cap = latest_capture(config)
    traffic = cap["sweep"]["dram_bytes_per_step"] if cap else None
    roof = {"bound": "hbm", "kernel": "Simulate sweep kernels (k_init_registers, k_first*, k_sweep; all builds of the step)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak if achieved else None,
            "peak_kind": peak_kind + " (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)",
            "traffic": traffic, "traffic_unit": "bytes per step (ncu dram__bytes_read.sum + dram__bytes_write.sum, same kernels)",
            "traffic_source": ("profiles/" + src) if src else None,
            "alg_bytes_per_step": alg, "sweep_kernel_ms_per_step": sweep_ms, "sweep_share_of_step": sweep_ms / step_ms,
            "alg_def": {"formula": "edges*(rec + J*(1-(1-p)^32)) + full_sweeps*n*(8+2J) + blocked_full*n*J/8 (SURVEY.md 8(d))",
                        "edges": edges, "rec_bytes": rec, "live_sector_bytes_per_edge": live, "full_sweeps": full_sweeps,
                        "blocked_full_sweeps": blocked_full, "n": n, "J": J},
            "builder_model": {"bytes": builder_bytes, "frac": builder_bytes / s / 1e9 / peak if s > 0 else None,
                              "def": "DESIGN.md section 6: 8 B record (+4 B WC) per enumerated edge + one 32 B sector per worked "
                                     "window + rows of full sweeps"}}
    if cap:
        ms_cap = cap["sweep"].get("ms_per_step")
        roof["ncu"] = {"commit": cap.get("commit"), "dram_bytes_per_step": traffic,
                       "dram_gbs": traffic / (ms_cap / 1e3) / 1e9 if ms_cap else None,
                       "dram_frac": traffic / (ms_cap / 1e3) / 1e9 / peak if ms_cap else None,
                       "l2_hit_rate_pct": cap["sweep"].get("l2_hit_rate_pct"),
                       "sectors_per_request": cap["sweep"].get("sectors_per_request"),
                       "traffic_over_alg": traffic / alg if alg else None}
    return roof


def config_dict(cfg, n, m, args):
    return {"workload": f"{cfg.name}: {cfg.note}", "n": int(n), "m": int(m), "J": cfg.J, "K": cfg.K, "t": cfg.t,
            "p": cfg.p if cfg.p is not None else "weighted-cascade 1/indeg", "salt_seed": cfg.salt_seed,
            "parallelism": (f"simulation-sharded x{args.gpus} (" + ("library NCCL communicator" if os.environ.get('IM_BENCH_BACKEND', 'nccl') == 'nccl'
                                                                   else os.environ.get('IM_BENCH_BACKEND').upper() + " host-staged communicator") + ")"
                            if args.mode == "shard" else f"replicas x{args.gpus}")
            if args.gpus > 1 else "single-gpu",
            "l2": "inputs (CSR+hash records) larger than L2" if m * 16 > 126e6 else "L2 flushed (256 MB write) between steps"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("IM_BENCH_CONFIG", "c4"))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="shard", choices=["shard", "replicas"])
    args = ap.parse_args()
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    args.gpus = world if world > 1 else args.gpus
    if args.impl == "reference":
        return run_reference(args, rank)

    import torch

    import paper_2105_04023_b200 as im

    # IM_BENCH_BACKEND=gloo: plumbing check of the sharded path with several ranks on one GPU (the
    # ranks then only wait for each other on the host); the measured configuration is NCCL
    backend = os.environ.get("IM_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = gen.CONFIGS[args.config]
    t0 = time.time()
    n, off, tgt, pr = gen.workload(cfg)
    gen_s = time.time() - t0
    m = len(tgt)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    im.im_set_stream(stream)
    shard = dist is not None and args.mode == "shard"
    if shard:
        from paper_2105_04023_b200.shard import TorchComm, nccl_init, shard_range

        j0, j1 = shard_range(cfg.J, rank, world)
        if backend == "nccl":  # the library's own NCCL communicator: stream-ordered, no Python in the exchange
            nccl_init(im.default())
        else:  # host-staged plumbing check (several ranks may share one GPU)
            im.im_set_comm(TorchComm())
    else:
        j0, j1 = 0, cfg.J

    def build():
        im.im_build_sketches_shard(cfg.J, cfg.salt_seed, j0, j1)
    d_off = torch.from_numpy(off).to(dev)
    d_tgt = torch.from_numpy(tgt).to(dev)
    d_pr = torch.from_numpy(pr).to(dev)
    d_est = torch.empty(n, dtype=torch.float64, device=dev)
    h_off = torch.from_numpy(off).pin_memory()
    h_tgt = torch.from_numpy(tgt).pin_memory()
    h_pr = torch.from_numpy(pr).pin_memory()
    h_est = torch.empty(n, dtype=torch.float64).pin_memory()
    h_seeds = torch.empty(cfg.K, dtype=torch.int32).pin_memory()
    h_scores = torch.empty(cfg.K, dtype=torch.float64).pin_memory()
    flush = None if m * 16 > 126e6 else torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()

    phase_ms = {"load": [], "build": [], "estimate": [], "select": []}

    def step_device():
        t = time.perf_counter()
        im.im_load_csr_device(n, m, d_off, d_tgt, d_pr)
        t1 = time.perf_counter()
        build()
        sb = im.im_get_stats()
        t2 = time.perf_counter()
        im.im_estimate_device(d_est)
        t3 = time.perf_counter()
        seeds, scores = im.im_select_seeds(cfg.K, cfg.t)
        ss = im.im_get_stats()
        t4 = time.perf_counter()
        for k, a, b in (("load", t, t1), ("build", t1, t2), ("estimate", t2, t3), ("select", t3, t4)):
            phase_ms[k].append((b - a) * 1e3)
        return sb, ss, seeds, scores

    def step_e2e():
        im.lib().im_load_csr(n, h_off.data_ptr(), h_tgt.data_ptr(), h_pr.data_ptr())
        build()
        sb = im.im_get_stats()
        im.lib().im_estimate(h_est.data_ptr())
        im.im_select_seeds_into(cfg.K, cfg.t, h_seeds.numpy(), h_scores.numpy())
        ss = im.im_get_stats()
        return sb, ss

    const_w = float(h_pr[0]) if m > 1 and bool((h_pr == h_pr[0]).all()) else None  # the paper's constant-w settings

    def step_e2e_scalar():  # the same step through im_load_csr_const: one scalar w instead of the m-entry array
        im.lib().im_load_csr_const(n, h_off.data_ptr(), h_tgt.data_ptr(), const_w)
        build()
        im.lib().im_estimate(h_est.data_ptr())
        im.im_select_seeds_into(cfg.K, cfg.t, h_seeds.numpy(), h_scores.numpy())

    for _ in range(args.warmup):
        step_device()
    times, edges, wedges, sweep_ms, sweeps, launches_sweep, rebuilds, launches, algb = [], [], [], [], [], [], [], [], []
    full_sweeps, blocked_full = [], []
    first_build = {}
    clocks = Clocks(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[0]) if os.environ.get("CUDA_VISIBLE_DEVICES", "").strip().isdigit() else local)
    for i in range(args.steps):
        if flush is not None:
            flush.fill_(i & 0xFF)
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = im.im_kernel_launch_count()
        ev0.record(stream)
        sb, ss, seeds, scores = step_device()
        ev1.record(stream)
        barrier()
        launches.append(im.im_kernel_launch_count() - l0)
        times.append(ev0.elapsed_time(ev1))
        edges.append(sb["total_edges"] + ss["total_edges"])
        wedges.append(sb["window_edges"] + ss["window_edges"])
        algb.append(sb["sweep_alg_bytes"] + ss["sweep_alg_bytes"])
        sweep_ms.append(sb["sweep_kernel_ms"] + ss["sweep_kernel_ms"])
        sweeps.append(sb["total_sweeps"] + ss["total_sweeps"])
        launches_sweep.append(sb["sweep_launches"] + ss["sweep_launches"])
        rebuilds.append(ss["rebuilds"])
        # full-vertex sweeps (every row read and written): the first sweep of every build + gather sweeps
        full_sweeps.append(1 + ss["rebuilds"] + sb["gather_sweeps"] + ss["gather_sweeps"])
        blocked_full.append(ss["rebuilds"])
        first_build = {"ms": sb["last_build_ms"], "sweeps": sb["last_build_sweeps"], "edges": sb["last_build_edges"],
                       "sweep_kernel_ms": sb["sweep_kernel_ms"], "prep_ms": sb["prep_ms"]}
    clk = clocks.stop()
    # e2e through the host-pointer ABI (pinned host buffers), same metric
    e2e_times = []
    if not args.no_e2e:
        for i in range(max(1, args.steps)):
            if flush is not None:
                flush.fill_(i & 0xFF)
            barrier()
            t = time.perf_counter()
            step_e2e()
            torch.cuda.synchronize(dev)
            e2e_times.append((time.perf_counter() - t) * 1e3)
    e2e_scalar_times = []
    if not args.no_e2e and const_w is not None and dist is None:
        for i in range(max(1, args.steps)):
            if flush is not None:
                flush.fill_(i & 0xFF)
            t = time.perf_counter()
            step_e2e_scalar()
            torch.cuda.synchronize(dev)
            e2e_scalar_times.append((time.perf_counter() - t) * 1e3)
    # max over ranks
    ms = statistics.mean(times)
    if dist is not None:
        tt = torch.tensor([ms, statistics.mean(e2e_times) if e2e_times else 0.0], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, e2e_ms = float(tt[0]), (float(tt[1]) if e2e_times else None)
    else:
        e2e_ms = statistics.mean(e2e_times) if e2e_times else None
    J = cfg.J
    work = statistics.mean(edges) * (j1 - j0)  # this rank's edge x sim updates per step
    if dist is None:
        total_work = work
    elif shard:
        tw = torch.tensor([work], device=dev, dtype=torch.float64)
        dist.all_reduce(tw)
        total_work = float(tw[0])
    else:
        total_work = world * work
    value = total_work / (ms / 1e3) / 1e9
    hbm_peak, peak_kind, _ = load_peaks()
    roof = roofline(cfg, n, m, pr, j1 - j0, statistics.mean(edges), statistics.mean(full_sweeps),
                    statistics.mean(blocked_full), statistics.mean(algb), statistics.mean(sweep_ms), ms, hbm_peak, peak_kind,
                    args.config)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "u8/u32",
            "data": "synthetic", "config": config_dict(cfg, n, m, args), "clocks": clk,
            "gpu_launches": int(statistics.mean(launches)), "roofline": roof,
            "im_time_s": ms / 1e3,
            "sketch_build": {"first_build_ms": first_build.get("ms"), "first_build_sweeps": first_build.get("sweeps"),
                             "first_build_gedge_sims_per_s": first_build.get("edges", 0) * (j1 - j0) / max(first_build.get("sweep_kernel_ms", 1e-9), 1e-9) / 1e6,
                             "prep_ms": first_build.get("prep_ms"), "sweeps_per_step": statistics.mean(sweeps),
                             "sweep_launches_per_step": statistics.mean(launches_sweep), "rebuilds_per_step": statistics.mean(rebuilds)},
            "phase_ms": {k: statistics.mean(v[-args.steps:]) for k, v in phase_ms.items()}, "step_ms_all": times,
            "bfs": {"levels": ss["bfs_levels"], "edges": ss["bfs_edges"]},
            "argmax": {"full_passes": ss["argmax_full"], "lazy_passes": ss["argmax_lazy"], "sorted_rows": ss["sorted_rows"]},
            "seeds_head": [int(x) for x in seeds[:5]], "sigma_final": float(scores[-1]) if len(scores) else None,
            "gen_seconds": gen_s, "sims_per_rank": j1 - j0}
    if e2e_ms is not None:
        line["e2e"] = {"value": total_work / (e2e_ms / 1e3) / 1e9, "unit": UNIT,
                       "h2d_bytes_per_step": int((n + 1) * 4 + m * 8), "d2h_bytes_per_step": int(n * 8 + cfg.K * 12),
                       "ms_per_step": e2e_ms}
    if e2e_scalar_times:  # informational: the constant-w entry point moves m x 4 bytes less over PCIe; `e2e` above is the array call
        es = statistics.mean(e2e_scalar_times)
        line["e2e_scalar_w"] = {"value": total_work / (es / 1e3) / 1e9, "unit": UNIT, "call": "im_load_csr_const",
                                "h2d_bytes_per_step": int((n + 1) * 4 + m * 4), "d2h_bytes_per_step": int(n * 8 + cfg.K * 12),
                                "ms_per_step": es}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_subprocess(args.config)
        line["cpu_baseline"].pop("seconds", None)
    if rank == 0:
        print(json.dumps(line), flush=True)
    im.im_free()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
