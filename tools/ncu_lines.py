"""Top CUDA source lines of one kernel launch in an ncu report (instructions executed, stall samples).

    python tools/ncu_lines.py gpurun_out/x.ncu-rep 'regex:k_first' [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys

rep, kn = sys.argv[1], sys.argv[2]
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kn, "--launch-skip", str(skip),
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
cur_file, fn, hdr, recs = None, None, None, []
for r in csv.reader(io.StringIO(raw)):
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) == 2 and r[0] == "Function Name":
        fn = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:  # CUDA line rows (SASS rows have an empty line number)
        try:
            ins, st = float(r[7]), float(r[4])
        except ValueError:
            continue
        if ins or st:
            recs.append((cur_file, int(r[0]), ins, st, r[1].strip()[:90]))
ti = sum(x[2] for x in recs) or 1
ts = sum(x[3] for x in recs) or 1
print(f"# {rep} {fn} skip={skip}: {ti:.3g} warp instructions, {ts:.0f} stall samples")
for key, name in ((2, "instructions"), (3, "stall samples")):
    print(f"## top lines by {name}")
    for f, ln, ins, st, src in sorted(recs, key=lambda x: -x[key])[:top]:
        print(f"{f}:{ln:<5d} ins {ins / ti * 100:5.1f}%  stall {st / ts * 100:5.1f}%  {src}")
