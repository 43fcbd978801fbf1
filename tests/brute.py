"""Independent brute-force references used to PIN the oracle on tiny inputs.

Nothing here imports oracle/ or the CUDA package.  Only library routines and
textbook definitions are used:
  * MurmurHash3 x86_32  -> sklearn.utils.murmurhash3_32
  * mt19937             -> numpy.random.RandomState raw stream
  * clz                 -> 32 - int.bit_length()
  * live test (Eq. 5)   -> the EXACT rational form  x / h_max < w  <=>  x < ceil(w * h_max)
                           (w is the float32 value, converted exactly with fractions)
  * reachability        -> transitive closure of the explicitly materialised sampled
                           subgraph by boolean matrix squaring (numpy matmul)
"""
from __future__ import annotations

import math
import struct
from fractions import Fraction

import numpy as np
from sklearn.utils import murmurhash3_32

HMAX = 2**31 - 1
PHI = 0.77351


def salts(seed: int, J: int):
    """Reading R3: mt19937(seed & 0xffffffff): seed_V, seed_J, then X_r = draw & (2^31-1)."""
    rs = np.random.RandomState(seed & 0xFFFFFFFF)
    raw = rs._bit_generator.random_raw(J + 2).astype(np.uint64)
    return int(raw[0]), int(raw[1]), (raw[2:] & np.uint64(0x7FFFFFFF)).astype(np.uint32)


def edge_hash(u: int, v: int) -> int:
    """Eq. 4 with R4: Murmur3(LE32 u || LE32 v, seed 0) mod 2^31."""
    return murmurhash3_32(struct.pack("<II", u, v), seed=0, positive=True) % (2**31)


def edge_hashes(offsets, targets) -> np.ndarray:
    n = len(offsets) - 1
    out = np.empty(len(targets), dtype=np.uint32)
    for u in range(n):
        for e in range(offsets[u], offsets[u + 1]):
            out[e] = edge_hash(u, int(targets[e]))
    return out


def threshold(w) -> int:
    """Exact integer threshold T with  x / h_max < w  <=>  x < T  for integer x."""
    wf = Fraction(float(np.float32(w)))
    return math.ceil(wf * HMAX)


def clz32(a: np.ndarray) -> np.ndarray:
    a = np.asarray(a, dtype=np.uint64)
    bl = np.zeros(a.shape, dtype=np.int64)
    for b in range(32):
        bl = np.where((a >> np.uint64(b)) != 0, b + 1, bl)
    return (32 - bl).astype(np.uint8)


def init_registers(n: int, J: int, seed: int) -> np.ndarray:
    sv, sj, _ = salts(seed, J)
    hv = murmurhash3_32(np.arange(n, dtype=np.int32), seed=sv, positive=True).astype(np.uint64)
    hj = murmurhash3_32(np.arange(J, dtype=np.int32), seed=sj, positive=True).astype(np.uint64)
    return clz32(hv[:, None] ^ hj[None, :])


def live_matrix(offsets, targets, probs, X) -> np.ndarray:
    """bool [m, J]: edge e is in sample j."""
    h = edge_hashes(offsets, targets).astype(np.int64)
    T = np.array([threshold(w) for w in probs], dtype=np.int64)
    return (X.astype(np.int64)[None, :] ^ h[:, None]) < T[:, None]


def closure(A: np.ndarray) -> np.ndarray:
    """Reflexive transitive closure of a boolean adjacency matrix."""
    n = A.shape[0]
    R = (A | np.eye(n, dtype=bool)).astype(np.float32)
    while True:
        R2 = ((R @ R) > 0).astype(np.float32)
        if np.array_equal(R2, R):
            return R.astype(bool)
        R = R2


def sample_adjacency(n, offsets, targets, L, j, blocked=None) -> np.ndarray:
    A = np.zeros((n, n), dtype=bool)
    for u in range(n):
        if blocked is not None and blocked[u, j]:
            continue  # a blocked source contributes no edge in sample j (reading R12)
        for e in range(offsets[u], offsets[u + 1]):
            if L[e, j]:
                A[u, targets[e]] = True
    return A


def registers(n, offsets, targets, probs, J, seed, blocked=None) -> np.ndarray:
    """Converged registers: M[u][j] = max over the reach set of u in G_j^S of the init register."""
    _, _, X = salts(seed, J)
    L = live_matrix(offsets, targets, probs, X)
    init = init_registers(n, J, seed).astype(np.int64)
    out = np.zeros((n, J), dtype=np.uint8)
    for j in range(J):
        R = closure(sample_adjacency(n, offsets, targets, L, j, blocked))
        out[:, j] = np.max(np.where(R, init[None, :, j], 0), axis=1)
    return out


def khop_registers(n, offsets, targets, probs, J, seed, hops, blocked=None) -> np.ndarray:
    """Registers after `hops` synchronous sweeps, in closed form: M[u][j] = max init register over
    the vertices within `hops` hops of u in the sampled subgraph G_j (hop distances from scipy)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import shortest_path

    _, _, X = salts(seed, J)
    L = live_matrix(offsets, targets, probs, X)
    init = init_registers(n, J, seed).astype(np.int64)
    out = np.zeros((n, J), dtype=np.uint8)
    for j in range(J):
        A = sample_adjacency(n, offsets, targets, L, j, blocked)
        D = shortest_path(csr_matrix(A.astype(np.float64)), unweighted=True, directed=True)
        out[:, j] = np.max(np.where(D <= hops, init[None, :, j], 0), axis=1)
    return out


def reach_masks(n, offsets, targets, probs, J, seed, seeds) -> np.ndarray:
    """bool [n, J]: v reachable from the seed set in sample j (no blocking)."""
    _, _, X = salts(seed, J)
    L = live_matrix(offsets, targets, probs, X)
    vis = np.zeros((n, J), dtype=bool)
    for j in range(J):
        R = closure(sample_adjacency(n, offsets, targets, L, j))
        vis[:, j] = R[list(seeds), :].any(axis=0)
    return vis


def estimate(row) -> float:
    """Eq. 2 closed form: 2^{mean} / phi."""
    return 2.0 ** (float(np.sum(np.asarray(row, dtype=np.int64))) / len(row)) / PHI


def random_graph(rng: np.random.Generator, n: int, m: int, p=None, allow_dups=True, allow_loops=True):
    """Tiny random CSR for tests (inputs only).  p None => random per-edge probabilities."""
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    if not allow_loops:
        keep = src != dst
        src, dst = src[keep], dst[keep]
    if not allow_dups:
        key = np.unique(src.astype(np.int64) * n + dst)
        src, dst = key // n, key % n
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    offsets = np.zeros(n + 1, dtype=np.int32)
    np.add.at(offsets, src + 1, 1)
    offsets = np.cumsum(offsets).astype(np.int32)
    targets = dst.astype(np.int32)
    if p is None:
        probs = rng.choice(np.array([0.0, 0.02, 0.1, 0.3, 0.5, 1.0], dtype=np.float32), len(targets))
        probs = np.where(rng.random(len(targets)) < 0.5, rng.random(len(targets)).astype(np.float32), probs).astype(np.float32)
    else:
        probs = np.full(len(targets), p, dtype=np.float32)
    return offsets, targets, probs


def simulate_registers(n, offsets, targets, probs, J, seed, blocked=None, eps_c=0.0) -> np.ndarray:
    """Registers after Alg. 2 with early exit eps_c (reading R22) in closed form: after s synchronous
    sweeps M = khop_registers(s); the run stops after the first s with |changed_s| / n <= eps_c
    (no sweep at all when eps_c >= 1).  eps_c = 0: the reach-max fixpoint (`registers`)."""
    if eps_c == 0.0:
        return registers(n, offsets, targets, probs, J, seed, blocked)
    prev = init_registers(n, J, seed)
    if not (1.0 > eps_c):
        return prev
    for s in range(1, n + 2):
        cur = khop_registers(n, offsets, targets, probs, J, seed, s, blocked=blocked)
        changed = int(np.any(cur != prev, axis=1).sum())
        prev = cur
        if not (changed / n > eps_c):
            return cur
    return prev


def select_seeds(n, offsets, targets, probs, J, seed, K, eps_l, eps_g, eps_c=0.0):
    """Alg. 1 restated with whole-array numpy operations and the closed forms above,
    readings R12-R21: registers = reach-max (or k-hop, eps_c > 0) on the residual samples, R_G(S) by
    transitive closure, pool = vertices not visited in every sample (empty -> lowest id not in S),
    argmax of the integer merged score with the lowest id on ties, keep iff err_l < eps_l or
    err_g < eps_g, else rebuild (not after the last pick, R18) with M_S' = 0 and varsigma = sigma.
    Returns a list of per-step dicts with the fields of the oracle's step log, plus 'ms_mattered'
    (the argmax would differ with M_S' = 0)."""
    M = simulate_registers(n, offsets, targets, probs, J, seed, eps_c=eps_c).astype(np.int64)
    MS = np.zeros(J, np.int64)
    varsigma = 0.0
    S = []
    vis = np.zeros((n, J), dtype=bool)
    steps = []
    for k in range(K):
        pool = ~vis.all(axis=1)
        score = np.maximum(M, MS[None, :]).sum(axis=1)
        if pool.any():
            s = int(np.argmax(np.where(pool, score, -1)))
            alt = int(np.argmax(np.where(pool, M.sum(axis=1), -1)))
        else:
            s = alt = min(v for v in range(n) if v not in S)
        S.append(s)
        e = 2.0 ** (float(score[s]) / J) / PHI
        vis = reach_masks(n, offsets, targets, probs, J, seed, S)
        sigma_count = int(vis.sum())
        sigma = sigma_count / J
        delta = sigma - varsigma
        err_l = abs((e - delta) / delta) if delta != 0 else math.inf
        err_g = abs((e - delta) / sigma)
        rebuild = not (err_l < eps_l or err_g < eps_g)
        executed = False
        if not rebuild:
            MS = np.maximum(MS, M[s])
        elif k < K - 1:
            M = simulate_registers(n, offsets, targets, probs, J, seed, blocked=vis, eps_c=eps_c).astype(np.int64)
            MS = np.zeros(J, np.int64)
            varsigma = sigma
            executed = True
        steps.append({"vertex": s, "score": int(score[s]), "e": e, "sigma_count": sigma_count, "sigma": sigma, "delta": delta,
                      "err_l": err_l, "err_g": err_g, "rebuilt": int(rebuild), "executed": int(executed), "ms_mattered": s != alt})
    return steps, vis, M.astype(np.uint8)
