"""Seeded synthetic inputs for the five BASELINE.json configs (inputs only).

This module holds none of the method's arithmetic: it generates CSR graphs and
per-edge IC probabilities (constant, or weighted-cascade 1/indeg(v) per
PAPER.md:139-142).  Both the oracle (tests, bench cpu_baseline) and the CUDA
path consume its output.  The recipe is in DESIGN.md "Input recipe".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "graphgen.c")
_LIB = os.path.join(_HERE, "libgraphgen.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        vp = ctypes.c_void_p
        lib.gen_rmat.restype = vp
        lib.gen_rmat.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_uint64]
        lib.gen_chung_lu.restype = vp
        lib.gen_chung_lu.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]
        lib.gen_er.restype = vp
        lib.gen_er.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64]
        lib.gen_n.restype = ctypes.c_int64
        lib.gen_n.argtypes = [vp]
        lib.gen_m.restype = ctypes.c_int64
        lib.gen_m.argtypes = [vp]
        lib.gen_copy_csr32.restype = ctypes.c_int
        lib.gen_copy_csr32.argtypes = [vp, vp, vp]
        lib.gen_wc_probs.restype = None
        lib.gen_wc_probs.argtypes = [ctypes.c_int64, ctypes.c_int64, vp, vp]
        lib.gen_free.restype = None
        lib.gen_free.argtypes = [vp]
        lib.gen_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _take(h):
    lib = _load()
    if not h:
        raise ValueError("generator rejected its arguments")
    try:
        n, m = lib.gen_n(h), lib.gen_m(h)
        off = np.empty(n + 1, dtype=np.int32)
        tgt = np.empty(max(m, 1), dtype=np.int32)
        if lib.gen_copy_csr32(h, off.ctypes.data, tgt.ctypes.data) != 0:
            raise ValueError("graph too large for int32 CSR")
        return off, tgt[:m]
    finally:
        lib.gen_free(h)


def er(n: int, m: int, seed: int):
    """Directed G(n,m): m distinct uniform ordered pairs u != v (C1)."""
    return _take(_load().gen_er(n, m, seed))


def rmat(scale: int, edge_factor: int, a=0.57, b=0.19, c=0.19, seed: int = 0):
    """RMAT with Graph500-style seeded relabel; self loops and duplicates removed (C2, C4)."""
    return _take(_load().gen_rmat(scale, edge_factor, a, b, c, seed))


def chung_lu(n: int, draws: int, beta: float, dmax: float, seed: int):
    """Directed Chung-Lu, weights (i+i0)^(-1/(beta-1)), i0 solved for max expected degree dmax (C3)."""
    i0 = ctypes.c_double(0)
    return _take(_load().gen_chung_lu(n, draws, beta, dmax, seed, ctypes.byref(i0)))


def wc_probs(n: int, targets: np.ndarray) -> np.ndarray:
    """Weighted-cascade weights float32(1/indeg(v)) per edge."""
    targets = np.ascontiguousarray(targets, dtype=np.int32)
    p = np.empty(len(targets), dtype=np.float32)
    _load().gen_wc_probs(n, len(targets), targets.ctypes.data, p.ctypes.data)
    return p


def threads() -> int:
    return _load().gen_threads()


@dataclass
class Config:
    name: str
    graph: str
    J: int
    K: int
    t: float
    p: float | None  # constant IC probability; None => weighted cascade
    salt_seed: int = 1
    note: str = ""
    extra: dict = field(default_factory=dict)


CONFIGS = {
    "c1": Config("c1", "er", 64, 10, 0.05, 0.05, note="tiny directed ER n=1000 m=10000 seed 0"),
    "c2": Config("c2", "rmat16", 256, 50, 0.05, None, note="RMAT-16 ef16 seed 2, WC probs"),
    "c3": Config("c3", "cl4m", 256, 50, 0.05, 0.01, note="Chung-Lu n=4M 70M draws beta 2.1 dmax 50000 seed 3"),
    "c4": Config("c4", "rmat24", 512, 50, 0.05, 0.005, note="RMAT-24 ef32 seed 4"),
}
# C5: the C3 graph, J x p x t grid, K=100
C5_GRID = [(J, p, t) for J in (64, 128, 256, 512, 1024) for p in (0.005, 0.01, 0.1) for t in (0.01, 0.05, 0.3)]


def graph(name: str):
    """Return (n, offsets int32[n+1], targets int32[m]) for a named config graph."""
    if name == "er":
        off, tgt = er(1000, 10000, 0)
    elif name == "rmat16":
        off, tgt = rmat(16, 16, seed=2)
    elif name == "cl4m":
        off, tgt = chung_lu(4_000_000, 70_000_000, 2.1, 50_000.0, 3)
    elif name == "rmat24":
        off, tgt = rmat(24, 32, seed=4)
    else:
        raise KeyError(name)
    return len(off) - 1, off, tgt


def workload(cfg: Config | str):
    """(n, offsets, targets, probs float32[m]) for a config."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    n, off, tgt = graph(cfg.graph)
    if cfg.p is None:
        probs = wc_probs(n, tgt)
    else:
        probs = np.full(len(tgt), cfg.p, dtype=np.float32)
    return n, off, tgt, probs
