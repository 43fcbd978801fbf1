import json, sys
for p in sys.argv[1:]:
    try:
        d = json.load(open(p))
    except Exception as e:
        print(p, "unreadable", e); continue
    r = d.get("roofline", {})
    print(p.split("/")[-1], "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 1), "phase",
          {k: round(v, 1) for k, v in d.get("phase_ms", {}).items()}, "sweepms", round(r.get("sweep_kernel_ms_per_step", 0), 1),
          "frac", round(r.get("frac") or 0, 3), "sb", d.get("sketch_build"), "bfs", d.get("bfs"), "argmax", d.get("argmax"),
          "e2e_ms", round(d.get("e2e", {}).get("ms_per_step", 0), 1), "launches", d.get("gpu_launches"), "clk", d.get("clocks"))
