"""Offline golden digests for the full-size configs, written by the ORACLE ONLY.

    python tests/golden/make_oracle_digests.py c2 --select      # build + full K-step selection
    python tests/golden/make_oracle_digests.py c3               # first build only

Writes tests/golden/<cfg>_oracle.json with SHA-256 digests of the inputs and of
the oracle's outputs, so GPU parity tests at sizes the oracle cannot finish in
seconds compare against oracle results without re-running it (DESIGN.md
"Parity").  Imports only gen/ (inputs) and oracle/.
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import oracle  # noqa: E402


def sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def reach_words(vis):
    """bool/u8 [n, J] -> the C-ABI layout: n x (J/32) uint32, bit j%32 of word j/32."""
    n, J = vis.shape
    b = np.asarray(vis, dtype=bool).reshape(n, J // 32, 32)
    return (b.astype(np.uint64) << np.arange(32, dtype=np.uint64)).sum(axis=2).astype(np.uint32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--select", action="store_true")
    ap.add_argument("--J", type=int)
    ap.add_argument("--p", type=float)
    ap.add_argument("--t", type=float)
    ap.add_argument("--K", type=int)
    a = ap.parse_args()
    cfg = gen.CONFIGS[a.cfg]
    J = a.J or cfg.J
    K = a.K or cfg.K
    t = cfg.t if a.t is None else a.t
    n, off, tgt, pr = gen.workload(cfg)
    if a.p is not None:
        pr = np.full(len(tgt), a.p, np.float32)
    tag = f"{a.cfg}" + ("" if a.J is None and a.p is None else f"_J{J}_p{a.p}")
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{tag}_oracle.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out.update({"cfg": a.cfg, "n": int(n), "m": int(len(tgt)), "J": J, "salt_seed": cfg.salt_seed,
                "graph_sha256": sha(off, tgt, pr), "oracle_cflags": " ".join(oracle.CFLAGS),
                "writer": "tests/golden/make_oracle_digests.py (oracle/ only)"})
    t0 = time.time()
    M, st = oracle.simulate(n, off, tgt, pr, J, cfg.salt_seed)
    out["first_build"] = {"registers_sha256": sha(M), "sweeps": st["sweeps"], "processed_edges": st["processed_edges"],
                          "changed": st["changed"], "row_sums_sha256": sha(M.astype(np.int64).sum(axis=1)),
                          "seconds": time.time() - t0}
    rng = np.random.default_rng(123)
    us = rng.integers(0, n, 64)
    out["first_build"]["sample_rows"] = {"vertices": us.tolist(), "rows": [M[u].tolist() for u in us]}
    del M
    json.dump(out, open(path, "w"), indent=1)
    if a.select:
        t0 = time.time()
        r = oracle.select_seeds(n, off, tgt, pr, J, cfg.salt_seed, K, t, want_vis=True)
        out["select"] = {"K": K, "t": t, "seeds": [int(s) for s in r["seeds"]],
                         "sigma_counts": [int(s["sigma_count"]) for s in r["steps"]],
                         "scores_int": [int(s["score"]) for s in r["steps"]],
                         "e": [s["e"] for s in r["steps"]],
                         "rebuilt": [int(s["rebuilt"]) for s in r["steps"]],
                         "executed": [int(s["executed"]) for s in r["steps"]],
                         "reach_sha256": sha(reach_words(r["vis"])), "stats": r["stats"],
                         "seconds": time.time() - t0}
        json.dump(out, open(path, "w"), indent=1)
    print(path)


if __name__ == "__main__":
    main()
