"""Offline golden digests for the full-size configs, written by the ORACLE ONLY.

    python tests/golden/make_oracle_digests.py c2 --select      # build + full K-step selection
    python tests/golden/make_oracle_digests.py c3               # first build only
    python tests/golden/make_oracle_digests.py c4 --select --no-final   # C4: first-build + select digests
    python tests/golden/make_oracle_digests.py c5 --J 64 --p 0.005 --t 0.01 --select   # one C5 grid point

Writes tests/golden/<tag>_oracle.json with SHA-256 digests of the inputs and of
the oracle's outputs, so GPU parity tests at sizes the oracle cannot finish in
seconds compare against oracle results without re-running it (DESIGN.md
"Parity").  Imports only gen/ (inputs) and oracle/.

With ORACLE_GOLDEN=1 the oracle is the same source built with OpenMP over the
independent u-loop of a synchronous sweep (oracle/__init__.py); results are
identical to the default single-threaded build (the C2 first-build digest is
reproduced by both builds).
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

CHUNK = 1 << 20  # rows per chunk for the n x J conversions (bounded memory at C4 size)


def sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        a = np.ascontiguousarray(a)
        flat = a.reshape(-1).view(np.uint8)
        for i in range(0, len(flat), 1 << 28):
            h.update(flat[i:i + (1 << 28)])
    return h.hexdigest()


def reach_words(vis):
    """bool/u8 [n, J] -> the C-ABI layout: n x (J/32) uint32, bit j%32 of word j/32."""
    n, J = vis.shape
    out = np.empty((n, J // 32), np.uint32)
    sh = np.arange(32, dtype=np.uint32)
    for i in range(0, n, CHUNK):
        b = (np.asarray(vis[i:i + CHUNK]) != 0).reshape(-1, J // 32, 32).astype(np.uint32)
        out[i:i + CHUNK] = (b << sh).sum(axis=2, dtype=np.uint32)
    return out


def row_sums(M):
    n = M.shape[0]
    out = np.empty(n, np.int64)
    for i in range(0, n, CHUNK):
        out[i:i + CHUNK] = M[i:i + CHUNK].sum(axis=1, dtype=np.int64)
    return out


def sample_rows(M, n, seed):
    rng = np.random.default_rng(seed)
    us = rng.integers(0, n, 64)
    return {"vertices": us.tolist(), "rows": [M[u].tolist() for u in us]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--select", action="store_true")
    ap.add_argument("--no-final", action="store_true", help="skip the final-register digest (memory)")
    ap.add_argument("--J", type=int)
    ap.add_argument("--p", type=float)
    ap.add_argument("--t", type=float)
    ap.add_argument("--K", type=int)
    a = ap.parse_args()
    c5 = a.cfg == "c5"
    cfg = gen.CONFIGS["c3" if c5 else a.cfg]
    J = a.J or cfg.J
    K = a.K or (100 if c5 else cfg.K)
    t = cfg.t if a.t is None else a.t
    n, off, tgt, pr = gen.workload(cfg)
    if a.p is not None:
        pr = np.full(len(tgt), a.p, np.float32)
    if c5:
        tag = f"c5_J{J}_p{a.p}_t{t}"
    else:
        tag = f"{a.cfg}" + ("" if a.J is None and a.p is None else f"_J{J}_p{a.p}")
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{tag}_oracle.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out.update({"cfg": a.cfg, "n": int(n), "m": int(len(tgt)), "J": J, "salt_seed": cfg.salt_seed,
                "p": None if cfg.p is None and a.p is None else float(a.p if a.p is not None else cfg.p),
                "graph_sha256": sha(off, tgt, pr), "oracle_cflags": " ".join(oracle.CFLAGS),
                "omp_threads": os.environ.get("OMP_NUM_THREADS"),
                "writer": "tests/golden/make_oracle_digests.py (oracle/ only)"})
    if not a.select:
        t0 = time.time()
        M, st = oracle.simulate(n, off, tgt, pr, J, cfg.salt_seed)
        out["first_build"] = {"registers_sha256": sha(M), "sweeps": st["sweeps"],
                              "processed_edges": st["processed_edges"], "changed": st["changed"],
                              "row_sums_sha256": sha(row_sums(M)), "seconds": time.time() - t0,
                              "sample_rows": sample_rows(M, n, 123)}
        del M
        json.dump(out, open(path, "w"), indent=1)
    else:
        t0 = time.time()
        r = oracle.select_seeds(n, off, tgt, pr, J, cfg.salt_seed, K, t, want_vis=True, want_first=True,
                                want_final=not a.no_final)
        secs = time.time() - t0
        M1 = r.pop("M_first")
        fb = out.get("first_build", {})
        fb.update({"registers_sha256": sha(M1), "row_sums_sha256": sha(row_sums(M1)),
                   "sample_rows": sample_rows(M1, n, 123)})
        out["first_build"] = fb
        del M1
        sel = {"K": K, "t": t, "seeds": [int(s) for s in r["seeds"]],
               "sigma_counts": [int(s["sigma_count"]) for s in r["steps"]],
               "scores_int": [int(s["score"]) for s in r["steps"]],
               "e": [s["e"] for s in r["steps"]],
               "err_l": [s["err_l"] for s in r["steps"]],
               "err_g": [s["err_g"] for s in r["steps"]],
               "rebuilt": [int(s["rebuilt"]) for s in r["steps"]],
               "executed": [int(s["executed"]) for s in r["steps"]],
               "stats": r["stats"], "seconds": secs}
        vis = r.pop("vis")
        sel["reach_sha256"] = sha(reach_words(vis))
        del vis
        if "M_final" in r:
            Mf = r.pop("M_final")
            sel["final_registers_sha256"] = sha(Mf)
            sel["final_sample_rows"] = sample_rows(Mf, n, 321)
            del Mf
        out["select"] = sel
        json.dump(out, open(path, "w"), indent=1)
    print(path)


if __name__ == "__main__":
    main()
