"""Summarise ncu outputs into small text files for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py launches gpurun_out/launches_c3.csv  > profiles/r01_launches_c3.txt
    python tools/ncu_summary.py report   gpurun_out/sweep_c4.ncu-rep > profiles/r01_sweep_c4.txt
"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[iu] not in UNIT:
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", "")) * UNIT[r[iu]]
    tot = sum(x[1] for x in agg.values())
    print(f"# ncu launch list {path}: gpu__time_duration.sum per kernel (cold-cache, serialised; compare shares)")
    print(f"# total {tot:.2f} ms over {sum(x[0] for x in agg.values())} launches")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.3f} ms {t / tot * 100:5.1f}%  n={c:5d}  avg={t / c * 1e3:9.1f} us  {k}")


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_requests_srcunit_tex_op_atom_dot_cas.sum"]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"# ncu --set full {path}")
        for k in want:
            if k in d:
                print(f"{k:70s} {d[k]:>22s} {u.get(k, '')}")
        stalls = [(k, float(d[k])) for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                  and d[k] not in ("", "n/a")]
        stalls.sort(key=lambda x: -x[1])
        print("# top stall reasons (warps per issue)")
        for k, v in stalls[:8]:
            print(f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v:8.3f}")
        try:
            b = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            rd = float(d["dram__bytes_read.sum"].replace(",", "")) * b[u["dram__bytes_read.sum"]]
            wr = float(d["dram__bytes_write.sum"].replace(",", "")) * b[u["dram__bytes_write.sum"]]
            print(f"# traffic per launch = {(rd + wr) / 1e9:.4g} Gbyte")
        except (KeyError, ValueError):
            pass


BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
# kernels inside the sweep kernel's CUDA-event window (im_abi.cu simulate(): init + first/gather/push sweeps)
SWEEP_KERNELS = ("k_init_registers", "k_first", "k_first_big", "k_sweep")


def traffic(path, config="c4", round_tag=None, commit=None):
    """DRAM bytes per kernel from an `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
    gpu__time_duration.sum --csv` log of ONE hot-path step (tools/profile_step.py --what step); prints
    the JSON bench.py reads for roofline.traffic (the sweep kernels' bytes per step)."""
    import json
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ik, iid, im_, iv, iu = (hdr.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.defaultdict(lambda: {"launches": set(), "dram_bytes": 0.0, "ms": 0.0, "sect": 0.0, "req": 0.0,
                                           "hit_w": 0.0, "hit_ms": 0.0})
    lms = {}
    hits = []
    for r in rows[1:]:
        name = r[ik].split("(")[0].replace("void ", "").split("<")[0].replace("im::", "")
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        d = per[name]
        d["launches"].add(r[iid])
        if r[im_].startswith("dram__bytes_"):
            d["dram_bytes"] += v * BYTES[r[iu]]
        elif r[im_] == "gpu__time_duration.sum":
            d["ms"] += v * UNIT[r[iu]]
            lms[r[iid]] = v * UNIT[r[iu]]
        elif r[im_] == "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum":
            d["sect"] += v
        elif r[im_] == "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum":
            d["req"] += v
        elif r[im_] == "lts__t_sector_hit_rate.pct":
            hits.append((name, r[iid], v))
    for name, lid, v in hits:  # L2 hit rate weighted by launch duration
        per[name]["hit_w"] += v * lms.get(lid, 0.0)
        per[name]["hit_ms"] += lms.get(lid, 0.0)

    def fin(d):
        o = {"launches": len(d["launches"]), "dram_bytes": d["dram_bytes"], "ms": d["ms"]}
        if d["req"]:
            o["sectors_per_request"] = d["sect"] / d["req"]
        if d["hit_ms"]:
            o["l2_hit_rate_pct"] = d["hit_w"] / d["hit_ms"]
        return o
    out = {k: fin(d) for k, d in per.items()}
    sw = [k for k in SWEEP_KERNELS if k in out]
    sect = sum(per[k]["sect"] for k in sw)
    req = sum(per[k]["req"] for k in sw)
    hms = sum(per[k]["hit_ms"] for k in sw)
    res = {"source": path, "config": config, "round": round_tag, "commit": commit, "kernels": out,
           "sweep": {"kernels": list(SWEEP_KERNELS), "dram_bytes_per_step": sum(out[k]["dram_bytes"] for k in sw),
                     "ms_per_step": sum(out[k]["ms"] for k in sw), "launches": sum(out[k]["launches"] for k in sw),
                     "sectors_per_request": sect / req if req else None,
                     "l2_hit_rate_pct": sum(per[k]["hit_w"] for k in sw) / hms if hms else None}}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"launches": launches, "report": report, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
