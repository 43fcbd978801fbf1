"""TEST INFRASTRUCTURE ONLY: ctypes wrapper around oracle/oracle.c.

The plain single-threaded CPU oracle of arxiv 2105.04023 (see the header of
oracle.c for what each function follows and what pins it).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this module.  The product path (paper_2105_04023_b200) never does.

Compiled with `gcc -O2` (no OpenMP, no intrinsics; compiler auto-vectorisation
allowed) -- the flags are part of the reported cpu_baseline.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
# ORACLE_GOLDEN=1 (offline golden writer only, tests/golden/make_oracle_digests.py): the same
# source built with OpenMP over the independent u-loop of a synchronous sweep and -O3; IEEE double
# without contraction or fast-math, so every result is identical to the default build's.  Tests,
# smoke() and the bench's cpu_baseline always use the default single-threaded -O2 build.
_GOLDEN = os.environ.get("ORACLE_GOLDEN") == "1"
_LIB = os.path.join(_HERE, "liboracle_golden.so" if _GOLDEN else "liboracle.so")
CFLAGS = (["-O3", "-march=native", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared"] if _GOLDEN
          else ["-O2", "-fPIC", "-shared"])
PHI = 0.77351  # PAPER.md:170 (R8)
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Step(ctypes.Structure):
    _fields_ = [
        ("vertex", ctypes.c_int32), ("pad", ctypes.c_int32), ("score", ctypes.c_int64),
        ("e", ctypes.c_double), ("sigma_count", ctypes.c_int64), ("sigma", ctypes.c_double),
        ("delta", ctypes.c_double), ("err_l", ctypes.c_double), ("err_g", ctypes.c_double),
        ("rebuilt", ctypes.c_int32), ("executed", ctypes.c_int32),
    ]


class SimStats(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int32), ("processed_edges", ctypes.c_int64), ("processed_vertices", ctypes.c_int64)]


class SelectStats(ctypes.Structure):
    _fields_ = [("builds", ctypes.c_int32), ("total_sweeps", ctypes.c_int32), ("total_processed_edges", ctypes.c_int64)]


def _load():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        vp, i32, i64, u32, u64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double
        sig = {
            "or_murmur3_32": (u32, [vp, i64, u32]),
            "or_edge_hash": (u32, [i32, i32]),
            "or_mt_draws": (None, [u32, i64, vp]),
            "or_salts": (None, [u64, i32, vp, vp, vp]),
            "or_live": (ctypes.c_int, [u32, u32, ctypes.c_float]),
            "or_init_registers": (None, [i32, i32, u32, u32, vp]),
            "or_init_rows": (None, [i32, u64, i64, vp, vp]),
            "or_estimate_row": (f64, [vp, i32]),
            "or_estimate": (None, [i32, i32, vp, vp]),
            "or_simulate": (ctypes.c_int, [i32, vp, vp, vp, i32, vp, vp, vp, vp, vp, i32, f64]),
            "or_select_seeds": (ctypes.c_int, [i32, vp, vp, vp, i32, u64, i32, f64, f64, f64, vp, vp, vp, vp, vp, vp, vp]),
            "or_reach_register": (ctypes.c_int, [i32, vp, vp, vp, i32, u64, i64, vp, vp, vp]),
            "or_seed_sigma": (ctypes.c_int, [i32, vp, vp, vp, i32, u64, i32, vp, vp]),
            "or_mix64": (u64, [u64]),
            "or_mc_draw": (u32, [u64, i64, i32, i32]),
            "or_mc_influence": (ctypes.c_int, [i32, vp, vp, vp, i32, vp, u64, i64, i64, vp]),
            "or_khop_register": (ctypes.c_int, [i32, vp, vp, vp, i32, u64, i32, i64, vp, vp, vp]),
            "or_rebuilt_register": (ctypes.c_int, [i32, vp, vp, vp, i32, u64, i32, vp, i64, vp, vp, vp]),
            "or_first_sweep_sample": (i64, [i32, vp, vp, vp, i32, u64, i32, i32, vp, vp]),
            "or_seed_reach_per_sim": (ctypes.c_int, [i32, vp, vp, vp, i32, u64, i32, vp, i32, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data if a is not None else None


def _csr(offsets, targets, probs):
    return (np.ascontiguousarray(offsets, dtype=np.int32), np.ascontiguousarray(targets, dtype=np.int32),
            np.ascontiguousarray(probs, dtype=np.float32))


def murmur3_32(data: bytes, seed: int) -> int:
    buf = np.frombuffer(data, dtype=np.uint8) if data else np.zeros(1, np.uint8)
    return _load().or_murmur3_32(buf.ctypes.data, len(data), seed & 0xFFFFFFFF)


def edge_hash(u: int, v: int) -> int:
    return _load().or_edge_hash(u, v)


def mt_draws(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    _load().or_mt_draws(seed & 0xFFFFFFFF, n, out.ctypes.data)
    return out


def salts(seed: int, J: int):
    sv, sj = ctypes.c_uint32(), ctypes.c_uint32()
    X = np.empty(J, dtype=np.uint32)
    _load().or_salts(seed, J, ctypes.byref(sv), ctypes.byref(sj), X.ctypes.data)
    return sv.value, sj.value, X


def live(X_r: int, h: int, w: float) -> bool:
    return bool(_load().or_live(X_r, h, w))


def init_registers(n: int, J: int, seed: int) -> np.ndarray:
    sv, sj, _ = salts(seed, J)
    M = np.empty((n, J), dtype=np.uint8)
    _load().or_init_registers(n, J, sv, sj, M.ctypes.data)
    return M


def estimate_row(row) -> float:
    row = np.ascontiguousarray(row, dtype=np.uint8)
    return _load().or_estimate_row(row.ctypes.data, len(row))


def estimate(M: np.ndarray) -> np.ndarray:
    M = np.ascontiguousarray(M, dtype=np.uint8)
    n, J = M.shape
    out = np.empty(n, dtype=np.float64)
    _load().or_estimate(n, J, M.ctypes.data, out.ctypes.data)
    return out


def simulate(n, offsets, targets, probs, J, seed, blocked=None, M=None, eps_c=0.0):
    """Alg. 2 (synchronous sweeps) while |L|/|V| > eps_c; eps_c = 0: to the fixpoint.
    Returns (M, stats dict incl. per-sweep changed counts)."""
    offsets, targets, probs = _csr(offsets, targets, probs)
    sv, sj, X = salts(seed, J)
    if M is None:
        M = init_registers(n, J, seed)
    M = np.ascontiguousarray(M, dtype=np.uint8).copy()
    if blocked is not None:
        blocked = np.ascontiguousarray(blocked, dtype=np.uint8)
        assert blocked.shape == (n, J)
    st = SimStats()
    cap = 100000
    log = np.zeros(cap, dtype=np.int32)
    rc = _load().or_simulate(n, _p(offsets), _p(targets), _p(probs), J, _p(X), _p(blocked), _p(M), ctypes.byref(st), _p(log), cap, float(eps_c))
    if rc != 0:
        raise MemoryError(rc)
    return M, {"sweeps": st.sweeps, "processed_edges": st.processed_edges,
               "processed_vertices": st.processed_vertices, "changed": log[: min(st.sweeps, cap)].tolist()}


def select_seeds(n, offsets, targets, probs, J, seed, K, eps_l, eps_g=None, want_vis=False, want_final=False, eps_c=0.0,
                 want_first=False):
    """Alg. 1.  Returns dict(seeds, scores, steps[list of dict], stats, vis?, M_final?, M_first?)."""
    if eps_g is None:
        eps_g = eps_l
    offsets, targets, probs = _csr(offsets, targets, probs)
    seeds = np.zeros(max(K, 1), dtype=np.int32)
    scores = np.zeros(max(K, 1), dtype=np.float64)
    log = (Step * max(K, 1))()
    vis = np.zeros((n, J), dtype=np.uint8) if want_vis else None
    Mf = np.zeros((n, J), dtype=np.uint8) if want_final else None
    M1 = np.zeros((n, J), dtype=np.uint8) if want_first else None
    st = SelectStats()
    rc = _load().or_select_seeds(n, _p(offsets), _p(targets), _p(probs), J, seed, K, float(eps_l), float(eps_g), float(eps_c),
                                 _p(seeds), _p(scores), ctypes.cast(log, ctypes.c_void_p), _p(vis), _p(Mf), ctypes.byref(st),
                                 _p(M1))
    if rc != 0:
        raise MemoryError(rc)
    steps = [{f: getattr(log[k], f) for f, _ in Step._fields_ if f != "pad"} for k in range(K)]
    out = {"seeds": seeds[:K].copy(), "scores": scores[:K].copy(), "steps": steps,
           "stats": {"builds": st.builds, "total_sweeps": st.total_sweeps, "total_processed_edges": st.total_processed_edges}}
    if want_vis:
        out["vis"] = vis
    if want_final:
        out["M_final"] = Mf
    if want_first:
        out["M_first"] = M1
    return out


def reach_register(n, offsets, targets, probs, J, seed, us, js) -> np.ndarray:
    """Definition of the converged register (first build) for sampled (u, j) pairs."""
    offsets, targets, probs = _csr(offsets, targets, probs)
    us = np.ascontiguousarray(us, dtype=np.int32)
    js = np.ascontiguousarray(js, dtype=np.int32)
    out = np.empty(len(us), dtype=np.uint8)
    rc = _load().or_reach_register(n, _p(offsets), _p(targets), _p(probs), J, seed, len(us), _p(us), _p(js), _p(out))
    if rc != 0:
        raise MemoryError(rc)
    return out


def rebuilt_register(n, offsets, targets, probs, J, seed, seeds, us, js) -> np.ndarray:
    """Definition of a register after a rebuild blocked by R_G(seeds) (Alg. 1 lines 21-25, R12), for
    sampled (u, j) pairs; pairs are sorted by j internally (one R_S[j] BFS per distinct j)."""
    offsets, targets, probs = _csr(offsets, targets, probs)
    us = np.ascontiguousarray(us, dtype=np.int32)
    js = np.ascontiguousarray(js, dtype=np.int32)
    seeds = np.ascontiguousarray(seeds, dtype=np.int32)
    order = np.argsort(js, kind="stable")
    us_s, js_s = np.ascontiguousarray(us[order]), np.ascontiguousarray(js[order])
    out = np.empty(len(us), dtype=np.uint8)
    o = np.empty(len(us), dtype=np.uint8)
    rc = _load().or_rebuilt_register(n, _p(offsets), _p(targets), _p(probs), J, seed, len(seeds), _p(seeds), len(us),
                                     _p(us_s), _p(js_s), _p(o))
    if rc != 0:
        raise MemoryError(rc)
    out[order] = o
    return out


def khop_register(n, offsets, targets, probs, J, seed, hops, us, js) -> np.ndarray:
    """Definition of a first-build register after `hops` synchronous sweeps (eps_c > 0, R22)."""
    offsets, targets, probs = _csr(offsets, targets, probs)
    us = np.ascontiguousarray(us, dtype=np.int32)
    js = np.ascontiguousarray(js, dtype=np.int32)
    out = np.empty(len(us), dtype=np.uint8)
    rc = _load().or_khop_register(n, _p(offsets), _p(targets), _p(probs), J, seed, int(hops), len(us), _p(us), _p(js), _p(out))
    if rc != 0:
        raise MemoryError(rc)
    return out


def mix64(z: int) -> int:
    return int(_load().or_mix64(z & 0xFFFFFFFFFFFFFFFF))


def mc_draw(seed: int, r: int, u: int, v: int) -> int:
    """31-bit fresh draw of edge (u,v) in evaluation sample r (reading R23)."""
    return int(_load().or_mc_draw(seed & 0xFFFFFFFFFFFFFFFF, r, u, v))


def mc_influence(n, offsets, targets, probs, seeds, seed, r0, R) -> np.ndarray:
    """int64[K]: sum over samples r0..r0+R-1 of |R_{G_r}(first k+1 seeds)| with fresh randomness (R23)."""
    offsets, targets, probs = _csr(offsets, targets, probs)
    seeds = np.ascontiguousarray(seeds, dtype=np.int32)
    out = np.zeros(len(seeds), dtype=np.int64)
    rc = _load().or_mc_influence(n, _p(offsets), _p(targets), _p(probs), len(seeds), _p(seeds), seed & 0xFFFFFFFFFFFFFFFF,
                                 int(r0), int(R), _p(out))
    if rc != 0:
        raise MemoryError(rc)
    return out


def seed_sigma(n, offsets, targets, probs, J, seed, seeds) -> np.ndarray:
    """sum_j |R_{G_j}(first k+1 seeds)| for k = 0..K-1 (int64)."""
    offsets, targets, probs = _csr(offsets, targets, probs)
    seeds = np.ascontiguousarray(seeds, dtype=np.int32)
    out = np.zeros(len(seeds), dtype=np.int64)
    rc = _load().or_seed_sigma(n, _p(offsets), _p(targets), _p(probs), J, seed, len(seeds), _p(seeds), _p(out))
    if rc != 0:
        raise MemoryError(rc)
    return out


def seed_reach_per_sim(n, offsets, targets, probs, J, seed, sims, seeds) -> np.ndarray:
    """int64 [len(sims), K]: |R_{G_j}(first k+1 seeds)| for each listed simulation j."""
    offsets, targets, probs = _csr(offsets, targets, probs)
    sims = np.ascontiguousarray(sims, dtype=np.int32)
    seeds = np.ascontiguousarray(seeds, dtype=np.int32)
    out = np.zeros((len(sims), len(seeds)), dtype=np.int64)
    rc = _load().or_seed_reach_per_sim(n, _p(offsets), _p(targets), _p(probs), J, seed, len(sims), _p(sims), len(seeds),
                                       _p(seeds), _p(out))
    if rc != 0:
        raise MemoryError(rc)
    return out


def first_sweep_sample(n, offsets, targets, probs, J, seed, u_begin, u_end):
    """Untimed setup + the timed call; returns (processed_edges, seconds, new_rows)."""
    import time
    offsets, targets, probs = _csr(offsets, targets, probs)
    rows = np.unique(np.concatenate([np.arange(u_begin, u_end, dtype=np.int32),
                                     targets[offsets[u_begin]:offsets[u_end]]])).astype(np.int32)
    M = np.zeros((n, J), dtype=np.uint8)  # lazily committed pages; only `rows` are touched
    _load().or_init_rows(J, seed, len(rows), _p(rows), _p(M))
    Mnew = np.empty((u_end - u_begin, J), dtype=np.uint8)
    t0 = time.perf_counter()
    pe = _load().or_first_sweep_sample(n, _p(offsets), _p(targets), _p(probs), J, seed, u_begin, u_end, _p(M), _p(Mnew))
    dt = time.perf_counter() - t0
    return int(pe), dt, Mnew
