"""Per-CUDA-line table of one kernel launch in an ncu report: warp instructions, average active lanes, stall samples.

    python tools/ncu_src.py rep.ncu-rep 'regex:k_first' [launch_skip] [file_substr] [min_pct]
"""
import csv
import io
import subprocess
import sys

rep, kn = sys.argv[1], sys.argv[2]
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
fsub = sys.argv[4] if len(sys.argv) > 4 else ""
minp = float(sys.argv[5]) if len(sys.argv) > 5 else 0.3
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kn, "--launch-skip", str(skip),
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
cur, hdr, recs = None, None, []
for r in csv.reader(io.StringIO(raw)):
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        try:
            ins, thr, st = float(r[7]), float(r[8]), float(r[4])
        except ValueError:
            continue
        if ins or st:
            recs.append((cur, int(r[0]), ins, thr, st, r[1].strip()[:80]))
ti = sum(x[2] for x in recs) or 1
tt = sum(x[3] for x in recs)
ts = sum(x[4] for x in recs) or 1
print(f"# {kn} skip={skip}: {ti:.4g} warp instr, avg active lanes {tt / ti:.1f}, {ts:.0f} stall samples")
for f, ln, ins, thr, st, src in recs:
    if fsub in (f or "") and (ins / ti * 100 >= minp or st / ts * 100 >= minp):
        print(f"{f}:{ln:<4d} ins {ins / ti * 100:5.1f}% lanes {thr / max(ins, 1):4.1f} stall {st / ts * 100:5.1f}%  {src}")
