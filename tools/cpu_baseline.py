"""cpu_baseline leg of bench.py, run in its own process so the product process never maps
liboracle.so: the oracle (oracle/, plain single-threaded C, as it stands) on a bounded sample of
the bench workload -- the first Alg. 2 sweep (synchronous, every u processed)
over a vertex range sized to ~target seconds of one host core.  Prints one JSON object.

    python tools/cpu_baseline.py --config c4 [--seconds 12]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402

UNIT = "G edge·sims/s"


def oracle_sample(cfg, n, off, tgt, pr, target_s=12.0):
    import oracle

    J = cfg.J
    u0 = n // 3  # calibrate on a small range, then size the timed sample
    e_small = 200_000 // max(1, J // 64)
    u1 = max(u0 + 1, min(int(np.searchsorted(off, off[u0] + e_small)), n))
    pe, dt, _ = oracle.first_sweep_sample(n, off, tgt, pr, J, cfg.salt_seed, u0, u1)
    want = int(max(pe, 1) / max(dt, 1e-6) * target_s)
    u2 = max(u0 + 1, min(int(np.searchsorted(off, off[u0] + want)), n))
    pe, dt, _ = oracle.first_sweep_sample(n, off, tgt, pr, J, cfg.salt_seed, u0, u2)
    return {"value": pe * J / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"oracle's first Alg. 2 sweep (synchronous, all u processed) over vertices [{u0},{u2}) = {pe} edges x "
                      f"J={J} = {pe * J:.3g} edge-sim tests, {dt:.1f} s on 1 host core (taskset pinned), gcc "
                      f"{' '.join(oracle.CFLAGS)}; separate process",
            "seconds": dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--seconds", type=float, default=12.0)
    a = ap.parse_args()
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except (AttributeError, OSError):
        pass
    cfg = gen.CONFIGS[a.config]
    n, off, tgt, pr = gen.workload(cfg)
    print(json.dumps(oracle_sample(cfg, n, off, tgt, pr, a.seconds)), flush=True)


if __name__ == "__main__":
    main()
