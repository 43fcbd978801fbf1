"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names the passage it follows.  Library routines (sklearn Murmur3,
numpy mt19937), closed forms and brute force on explicitly sampled subgraphs
(tests/brute.py) are the independent references.
"""
import json
import math
import os
import struct

import numpy as np
import pytest
from sklearn.utils import murmurhash3_32

import oracle
from tests import brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- hashing (Eq. 4)
def test_murmur3_matches_library():
    """MurmurHash3 x86_32 (Eq. 4) vs sklearn.utils.murmurhash3_32."""
    rng = np.random.default_rng(0)
    assert oracle.murmur3_32(b"", 0) == 0
    for _ in range(400):
        ln = int(rng.integers(0, 18))
        data = bytes(rng.integers(0, 256, ln, dtype=np.uint8))
        seed = int(rng.integers(0, 2**32))
        assert oracle.murmur3_32(data, seed) == murmurhash3_32(data, seed=seed, positive=True)


def test_edge_hash_golden():
    """h(u,v) = Murmur3(LE32 u || LE32 v, 0) mod 2^31 (Eq. 4, reading R4)."""
    with open(os.path.join(GOLDEN, "edge_hash.json")) as f:
        g = json.load(f)
    for (u, v), h in zip(g["pairs"], g["hash"]):
        assert oracle.edge_hash(u, v) == h == brute.edge_hash(u, v)
    rng = np.random.default_rng(1)
    for _ in range(300):
        u, v = (int(x) for x in rng.integers(0, 2**31 - 1, 2))
        h = oracle.edge_hash(u, v)
        assert h == brute.edge_hash(u, v) and 0 <= h < 2**31
    assert oracle.edge_hash(1, 2) != oracle.edge_hash(2, 1)  # directed


# ---------------------------------------------------------------- mt19937 / salts
def test_mt19937_matches_numpy_and_std_check_value():
    """PAPER.md:472 names mt19937.  C++ [rand.predef]: 10000th draw of default seed 5489 = 4123659995."""
    assert int(oracle.mt_draws(5489, 10000)[-1]) == 4123659995
    for seed in (0, 1, 2, 5489, 2**32 - 1):
        ref = np.random.RandomState(seed)._bit_generator.random_raw(2000).astype(np.uint32)
        assert np.array_equal(oracle.mt_draws(seed, 2000), ref)


def test_salts_stream():
    """R2/R3: seed_V, seed_J, then X_r = draw & (2^31-1); values from the numpy stream."""
    sv, sj, X = oracle.salts(1, 1024)
    bv, bj, BX = brute.salts(1, 1024)
    assert (sv, sj) == (bv, bj) == (1791095845, 4282876139)
    assert np.array_equal(X, BX)
    assert list(X[:4]) == [946286476, 1857819720, 491263, 550290313]
    assert X.max() < 2**31
    # J-prefix property (R3): sims 0..J1-1 identical for any J >= J1
    assert np.array_equal(oracle.salts(1, 64)[2], X[:64])
    # the C-ABI seed is uint64; only its low 32 bits seed mt19937 (R3)
    assert np.array_equal(oracle.salts(1 + 2**32, 16)[2], X[:16])


# ---------------------------------------------------------------- live test (Eq. 5)
PAPER_W = [0.005, 0.01, 0.1, 0.05, 0.3, 0.5, 1.0, 0.0]


def test_live_closed_forms():
    """Eq. 5 strict '<': w = 0 never live; w = 1 live iff X xor h != h_max."""
    rng = np.random.default_rng(2)
    for _ in range(2000):
        X, h = (int(x) for x in rng.integers(0, 2**31, 2))
        assert not oracle.live(X, h, 0.0)
        assert oracle.live(X, h, 1.0) == ((X ^ h) != brute.HMAX)
    assert not oracle.live(0, brute.HMAX, 1.0)
    assert oracle.live(5, 5, 1e-30)  # P = 0 < w


def test_live_equals_exact_rational_threshold():
    """The double-precision Eq. 5 vs the exact rational x/h_max < w, at and around every threshold."""
    ws = PAPER_W + [1.0 / d for d in range(1, 400)] + list(np.random.default_rng(3).random(300))
    for w in ws:
        w32 = float(np.float32(w))
        T = brute.threshold(w32)
        for x in {0, T - 2, T - 1, T, T + 1, brute.HMAX - 1, brute.HMAX}:
            if 0 <= x <= brute.HMAX:
                assert oracle.live(x, 0, w32) == (x < T), (w32, x, T)
    # printed integer thresholds (SURVEY finding 4)
    assert [brute.threshold(w) for w in (0.005, 0.01, 0.05, 0.1, 1.0)] == [10737418, 21474836, 107374184, 214748368, 2147483647]


def test_live_rate_and_capture_probability():
    """Sampling rate within binomial 3 sigma; P(live in >= 1 of J=256 sims at w=0.005)
    = 1-(1-0.005)^256 = 0.72."""
    _, _, X = oracle.salts(1, 256)
    rng = np.random.default_rng(4)
    hs = rng.integers(0, 2**31, 4000)
    L = np.array([[oracle.live(int(x), int(h), 0.1) for x in X[:64]] for h in hs[:1500]])
    N = L.size
    assert abs(L.mean() - 0.1) < 3 * math.sqrt(0.1 * 0.9 / N)
    cap = np.array([any(oracle.live(int(x), int(h), 0.005) for x in X) for h in hs])
    p = 1 - (1 - 0.005) ** 256
    assert abs(p - 0.7229) < 1e-3
    assert abs(cap.mean() - p) < 4 * math.sqrt(p * (1 - p) / len(hs))


# ---------------------------------------------------------------- init (Alg. 1 lines 2-5)
def test_init_registers_vs_library_hash():
    """M_v[j] = clz(hash(v) xor hash(j)), R5/R6; clz via int.bit_length."""
    for seed, n, J in ((1, 1000, 64), (7, 50, 256), (2**40 + 3, 20, 32)):
        assert np.array_equal(oracle.init_registers(n, J, seed), brute.init_registers(n, J, seed))
    M = oracle.init_registers(1000, 64, 1)
    assert (M[0, 0], M[0, 1], M[1, 0], M[1, 63], M[999, 0]) == (0, 1, 3, 3, 1)
    assert M.max() <= 32


def test_init_geometric_tail():
    """P(register >= k) = 2^-k for a uniform 32-bit word."""
    M = oracle.init_registers(20000, 64, 9).astype(np.int64)
    for k in range(1, 7):
        frac = (M >= k).mean()
        assert abs(frac - 2.0**-k) < 4 * math.sqrt(2.0**-k / M.size)


# ---------------------------------------------------------------- estimate (Eq. 2)
def test_estimate_closed_forms():
    """e = 2^{mean}/phi, phi = 0.77351; SPEC.md:234-235 values."""
    assert abs(oracle.estimate_row(np.zeros(64, np.uint8)) - 1.29281) < 1e-5
    assert abs(oracle.estimate_row(np.full(256, 10, np.uint8)) - 1323.84) < 1e-2
    assert oracle.estimate_row(np.array([0, 2], np.uint8)) == 2.0 / 0.77351
    assert oracle.estimate_row(np.array([1, 2, 3, 6], np.uint8)) == 2.0**3 / 0.77351
    rng = np.random.default_rng(5)
    M = rng.integers(0, 33, (50, 96)).astype(np.uint8)
    e = oracle.estimate(M)
    for v in range(50):
        assert abs(e[v] - brute.estimate(M[v])) <= 1e-12 * e[v]


def test_estimate_bias_of_max_clz_register():
    """Statistical check of Eq. 2 with this register definition (SURVEY finding 3): for a set of
    c items, E[max clz] = sum_k 1-(1-2^-k)^c; the estimator is biased high (~1.6x at c >= 100)."""
    rng = np.random.default_rng(6)
    J = 256
    for c in (100, 1000):
        words = rng.integers(0, 2**32, (c, J), dtype=np.uint64)
        regs = brute.clz32(words).max(axis=0)
        ratio = oracle.estimate_row(regs) / c
        expect = 2 ** sum(1 - (1 - 2.0**-k) ** c for k in range(1, 33)) / 0.77351 / c
        assert 1.3 < ratio < 2.1 and abs(math.log(ratio / expect)) < 0.35


# ---------------------------------------------------------------- Simulate (Alg. 2)
def test_simulate_equals_bruteforce_reach_max():
    """SPEC.md:500 acceptance #1: >= 100 random graphs (n <= 120), eps_c = 0: every converged
    register equals the max init register over the reach set in the sampled subgraph."""
    rng = np.random.default_rng(7)
    for g in range(100):
        n = int(rng.integers(2, 120))
        m = int(rng.integers(0, 4 * n))
        J = int(rng.choice([32, 64]))
        seed = int(rng.integers(0, 2**32))
        p = None if g % 3 == 0 else float(rng.choice([0.05, 0.2, 0.5, 1.0]))
        off, tgt, pr = brute.random_graph(rng, n, m, p)
        M, st = oracle.simulate(n, off, tgt, pr, J, seed)
        assert np.array_equal(M, brute.registers(n, off, tgt, pr, J, seed)), g
        assert st["changed"][-1] == 0


def test_simulate_with_blocked_equals_bruteforce():
    """Alg. 2 line 'u not in R_S[j]', reading R12: blocked u never pulls in sim j."""
    rng = np.random.default_rng(8)
    for g in range(30):
        n = int(rng.integers(2, 80))
        off, tgt, pr = brute.random_graph(rng, n, int(rng.integers(0, 4 * n)), float(rng.choice([0.3, 1.0])))
        J = 32
        seed = int(rng.integers(0, 2**32))
        blocked = (rng.random((n, J)) < 0.3).astype(np.uint8)
        M, _ = oracle.simulate(n, off, tgt, pr, J, seed, blocked=blocked)
        assert np.array_equal(M, brute.registers(n, off, tgt, pr, J, seed, blocked=blocked.astype(bool)))


@pytest.mark.parametrize("eps_c", [0.02, 0.05, 0.15, 0.4])
def test_simulate_early_exit_equals_khop_closed_form(eps_c):
    """Alg. 2 with the early exit eps_c (reading R22, synchronous sweeps): the run
    stops after the first sweep s with |changed_s| / n <= eps_c, and the registers are then the max
    init register within s hops in each sampled subgraph (closed form via hop distances)."""
    rng = np.random.default_rng(int(eps_c * 1000))
    hit_early = 0
    for g in range(12):
        n = int(rng.integers(20, 90))
        off, tgt, pr = brute.random_graph(rng, n, int(rng.integers(n, 4 * n)), float(rng.choice([0.2, 0.5, 1.0])))
        J, seed = 32, int(rng.integers(0, 2**32))
        blocked = (rng.random((n, J)) < 0.2).astype(np.uint8) if g % 3 == 2 else None
        M, st = oracle.simulate(n, off, tgt, pr, J, seed, blocked=blocked, eps_c=eps_c)
        bl = None if blocked is None else blocked.astype(bool)
        prev = brute.init_registers(n, J, seed)
        changed = []
        for s in range(1, n + 2):
            cur = brute.khop_registers(n, off, tgt, pr, J, seed, s, blocked=bl)
            changed.append(int(np.any(cur != prev, axis=1).sum()))
            prev = cur
            if changed[-1] / n <= eps_c:
                break
        assert st["sweeps"] == s and st["changed"] == changed, (g, st, changed)
        assert np.array_equal(M, cur), g
        hit_early += changed[-1] > 0
    assert hit_early > 0  # some runs stopped before the fixpoint


def test_khop_register_vs_closed_form():
    """or_khop_register (sampled definition used at full size) vs the hop-distance closed form."""
    rng = np.random.default_rng(79)
    for g in range(6):
        n = int(rng.integers(20, 70))
        off, tgt, pr = brute.random_graph(rng, n, 3 * n, float(rng.choice([0.3, 0.7])))
        J, seed = 32, int(rng.integers(0, 2**32))
        for hops in (0, 1, 2, 4, n):
            want = brute.khop_registers(n, off, tgt, pr, J, seed, hops)
            us = np.repeat(np.arange(n), J)
            js = np.tile(np.arange(J), n)
            got = oracle.khop_register(n, off, tgt, pr, J, seed, hops, us, js).reshape(n, J)
            assert np.array_equal(got, want), (g, hops)


def test_simulate_early_exit_limits():
    """eps_c >= 1: the loop condition |V|/|V| > eps_c fails at once, registers stay at init; eps_c = 0
    is the fixpoint (the ordinary build)."""
    rng = np.random.default_rng(77)
    n = 40
    off, tgt, pr = brute.random_graph(rng, n, 120, 0.5)
    M, st = oracle.simulate(n, off, tgt, pr, 32, 3, eps_c=1.0)
    assert st["sweeps"] == 0 and np.array_equal(M, oracle.init_registers(n, 32, 3))
    M0, _ = oracle.simulate(n, off, tgt, pr, 32, 3)
    Me, _ = oracle.simulate(n, off, tgt, pr, 32, 3, eps_c=0.0)
    assert np.array_equal(M0, Me) and np.array_equal(M0, brute.registers(n, off, tgt, pr, 32, 3))


def test_select_with_early_exit_reduction():
    """K = 1, t = inf with eps_c > 0: the seed is the argmax row sum of the early-exit registers."""
    rng = np.random.default_rng(78)
    for g in range(5):
        n = int(rng.integers(30, 80))
        off, tgt, pr = brute.random_graph(rng, n, 3 * n, 0.5)
        J, seed = 32, int(rng.integers(0, 2**32))
        M, _ = oracle.simulate(n, off, tgt, pr, J, seed, eps_c=0.1)
        r = oracle.select_seeds(n, off, tgt, pr, J, seed, 1, math.inf, eps_c=0.1)
        rows = M.astype(np.int64).sum(axis=1)
        assert r["seeds"][0] == int(np.argmax(rows)) and r["steps"][0]["score"] == rows.max()


def test_simulate_special_cases():
    """No edges -> M unchanged after one sweep; path a->b->c with w = 1 -> pairwise max."""
    n, J, seed = 5, 64, 3
    M, st = oracle.simulate(n, np.zeros(n + 1, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float32), J, seed)
    assert np.array_equal(M, oracle.init_registers(n, J, seed)) and st["sweeps"] == 1
    off = np.array([0, 1, 2, 2], np.int32)
    tgt = np.array([1, 2], np.int32)
    M, _ = oracle.simulate(3, off, tgt, np.ones(2, np.float32), J, seed)
    I = oracle.init_registers(3, J, seed)
    # w = 1 is dead only when X xor h = h_max (probability 2^-31); check it is not the case here
    _, _, X = oracle.salts(seed, J)
    assert all((int(x) ^ brute.edge_hash(0, 1)) != brute.HMAX and (int(x) ^ brute.edge_hash(1, 2)) != brute.HMAX for x in X)
    assert np.array_equal(M[0], I.max(axis=0)) and np.array_equal(M[1], I[1:].max(axis=0)) and np.array_equal(M[2], I[2])


def test_fig5_shape():
    """Fig. 5 caption: edge (1,4) live in both sims, (4,3) live only in sim 2;
    4's sim-2 register rises in sweep 1, 1 re-pulls from 4 in sweep 2, then the process stops.
    Synchronous sweeps + the Gamma^-(L) frontier give changed sets {1,4}, {1}, {} (readings R10, R11).
    The toy graph's other edges and its register values are in the missing image (unpinned)."""
    J = 2
    for seed in range(1, 100000):
        sv, sj, X = brute.salts(seed, J)
        I = brute.init_registers(5, J, seed).astype(int)
        h43 = brute.edge_hash(4, 3)
        P = [(int(X[j]) ^ h43) / brute.HMAX for j in range(2)]
        if not P[1] < P[0]:
            continue
        if I[3, 1] > I[4, 1] and I[3, 1] > I[1, 1] and (I[4] > I[1]).any():
            break
    w43 = np.float32((P[0] + P[1]) / 2)
    off = np.array([0, 0, 1, 1, 1, 2], np.int32)  # vertices 0..4; 0 is isolated
    tgt = np.array([4, 3], np.int32)
    pr = np.array([1.0, w43], np.float32)
    M, st = oracle.simulate(5, off, tgt, pr, J, seed)
    assert st["changed"] == [2, 1, 0] and st["sweeps"] == 3
    assert M[4, 1] == I[3, 1] and M[4, 0] == I[4, 0] and M[1, 1] == I[3, 1]
    assert np.array_equal(M, brute.registers(5, off, tgt, pr, J, seed))


# ---------------------------------------------------------------- definitions used for sampled parity
def test_reach_register_and_seed_sigma_vs_bruteforce():
    rng = np.random.default_rng(9)
    for g in range(20):
        n = int(rng.integers(2, 100))
        off, tgt, pr = brute.random_graph(rng, n, int(rng.integers(0, 4 * n)), None)
        J, seed = 32, int(rng.integers(0, 2**32))
        R = brute.registers(n, off, tgt, pr, J, seed)
        us = rng.integers(0, n, 50)
        js = rng.integers(0, J, 50)
        assert np.array_equal(oracle.reach_register(n, off, tgt, pr, J, seed, us, js), R[us, js])
        seeds = rng.choice(n, min(n, 5), replace=False)
        cnt = oracle.seed_sigma(n, off, tgt, pr, J, seed, seeds)
        sims = rng.choice(J, 4, replace=False)
        per = oracle.seed_reach_per_sim(n, off, tgt, pr, J, seed, sims, seeds)
        for k in range(len(seeds)):
            vis = brute.reach_masks(n, off, tgt, pr, J, seed, seeds[: k + 1])
            assert cnt[k] == vis.sum()
            assert list(per[:, k]) == [int(vis[:, j].sum()) for j in sims]


# ---------------------------------------------------------------- Alg. 1
def star(n_leaves, center=0, base=0):
    """edges center -> leaves, ids base..base+n_leaves"""
    return [(base + center, base + i) for i in range(n_leaves + 1) if i != center]


def csr_from_edges(n, edges, w=1.0):
    edges = sorted(edges)
    off = np.zeros(n + 1, np.int32)
    for u, _ in edges:
        off[u + 1] += 1
    off = np.cumsum(off).astype(np.int32)
    tgt = np.array([v for _, v in edges], np.int32)
    return off, tgt, np.full(len(tgt), w, np.float32)


def test_select_star_and_two_stars():
    """SPEC.md:352 (star, K=1 -> centre) and SPEC.md:427 (two disjoint stars, K=2 -> both centres, larger first)."""
    off, tgt, pr = csr_from_edges(51, star(50))
    for t in (0.0, 0.05, math.inf):
        assert list(oracle.select_seeds(51, off, tgt, pr, 64, 1, 1, t)["seeds"]) == [0]
    edges = star(5, base=0) + star(10, base=6)  # small star centre 0 (5 leaves), big star centre 6 (10 leaves)
    off, tgt, pr = csr_from_edges(17, edges)
    for t in (0.0, 0.05, math.inf):
        r = oracle.select_seeds(17, off, tgt, pr, 256, 1, 2, t)
        assert list(r["seeds"]) == [6, 0], t
        assert list(r["scores"]) == [11.0, 17.0]


def test_select_reductions_and_variants():
    """K=1 with t=inf reduces to argmax of the first-build estimates; t=0 rebuilds at
    every step (strict '<'), t=inf never (Fig. 6 variants)."""
    rng = np.random.default_rng(10)
    for g in range(8):
        n = int(rng.integers(20, 120))
        off, tgt, pr = brute.random_graph(rng, n, 4 * n, float(rng.choice([0.1, 0.3])), allow_dups=False, allow_loops=False)
        J, seed = 64, int(rng.integers(0, 2**32))
        M, _ = oracle.simulate(n, off, tgt, pr, J, seed)
        r = oracle.select_seeds(n, off, tgt, pr, J, seed, 1, math.inf)
        rows = M.astype(np.int64).sum(axis=1)
        assert r["seeds"][0] == int(np.argmax(rows)) and r["steps"][0]["score"] == rows.max()
        K = 6
        r0 = oracle.select_seeds(n, off, tgt, pr, J, seed, K, 0.0)
        assert all(s["rebuilt"] == 1 for s in r0["steps"]) and r0["stats"]["builds"] == K
        assert [s["executed"] for s in r0["steps"]] == [1] * (K - 1) + [0]
        ri = oracle.select_seeds(n, off, tgt, pr, J, seed, K, math.inf)
        assert all(s["rebuilt"] == 0 for s in ri["steps"]) and ri["stats"]["builds"] == 1


def test_select_sigma_and_masks_vs_bruteforce():
    """R_G(S) and sigma (Alg. 1 lines 13-14) equal brute-force reach of the chosen seeds; sigma is
    non-decreasing and <= n; seeds are distinct (the keep/rebuild decisions are pinned field by field
    against the brute-force Alg. 1 in test_select_matches_bruteforce_alg1)."""
    rng = np.random.default_rng(11)
    for g in range(10):
        n = int(rng.integers(10, 90))
        off, tgt, pr = brute.random_graph(rng, n, 3 * n, None if g % 2 else 0.2)
        J, seed, K = 32, int(rng.integers(0, 2**32)), min(n, 6)
        t = float(rng.choice([0.0, 0.05, 0.3, math.inf]))
        r = oracle.select_seeds(n, off, tgt, pr, J, seed, K, t, want_vis=True)
        seeds = list(r["seeds"])
        assert len(set(seeds)) == K
        vis = brute.reach_masks(n, off, tgt, pr, J, seed, seeds)
        assert np.array_equal(r["vis"].astype(bool), vis)
        for k in range(K):
            assert r["steps"][k]["sigma_count"] == brute.reach_masks(n, off, tgt, pr, J, seed, seeds[: k + 1]).sum()
            assert r["scores"][k] == r["steps"][k]["sigma_count"] / J
        assert all(np.diff(r["scores"]) >= 0) and r["scores"][-1] <= n


def _alg1_cases():
    """>= 30 tiny graphs: the paper's (eps_l, eps_g) = (0.3, 0.01) and single
    thresholds t in {0.05, 0.3, inf}, eps_c in {0, 0.02}; p high enough that keeps and rebuilds mix."""
    rng = np.random.default_rng(1313)
    cases = []
    pols = [(0.3, 0.01), (0.05, 0.05), (0.3, 0.3), (math.inf, math.inf)]
    for g in range(32):
        n = int(rng.integers(12, 60))
        p = None if g % 4 == 3 else float(rng.choice([0.1, 0.2, 0.35]))
        off, tgt, pr = brute.random_graph(rng, n, int(rng.integers(2 * n, 4 * n)), p)
        eps_l, eps_g = pols[g % 4]
        eps_c = 0.02 if g % 8 >= 6 else 0.0
        cases.append((g, n, off, tgt, pr, 32, int(rng.integers(0, 2**32)), min(n, 7), eps_l, eps_g, eps_c))
    return cases


def test_select_matches_bruteforce_alg1():
    """Alg. 1 field by field against tests/brute.select_seeds, a whole-array restatement
    on closure-based registers and reach sets: seed, integer merged score, e, sigma count, delta,
    err_l, err_g, rebuild decision and execution at every step, the final R_G(S) and the registers
    after the last executed rebuild.  The cases must include keeps and rebuilds alternating within a
    run, and steps where M_S' (the merge of line 19) changes the argmax."""
    kinds, alternating, ms_mattered = set(), 0, 0
    for g, n, off, tgt, pr, J, seed, K, eps_l, eps_g, eps_c in _alg1_cases():
        r = oracle.select_seeds(n, off, tgt, pr, J, seed, K, eps_l, eps_g, want_vis=True, want_final=True, eps_c=eps_c)
        want, vis, Mf = brute.select_seeds(n, off, tgt, pr, J, seed, K, eps_l, eps_g, eps_c=eps_c)
        for k, (got, w) in enumerate(zip(r["steps"], want)):
            for f in ("vertex", "score", "sigma_count", "rebuilt", "executed"):
                assert got[f] == w[f], (g, k, f, got[f], w[f])
            for f in ("e", "sigma", "delta", "err_g"):
                assert got[f] == pytest.approx(w[f], rel=1e-12, abs=0), (g, k, f)
            assert (math.isinf(got["err_l"]) and math.isinf(w["err_l"])) or got["err_l"] == pytest.approx(w["err_l"], rel=1e-12)
            kinds.add(w["rebuilt"])
            ms_mattered += w["ms_mattered"] and k > 0 and not want[k - 1]["rebuilt"]
        dec = [w["rebuilt"] for w in want]
        alternating += any(a != b for a, b in zip(dec, dec[1:]))
        assert list(r["seeds"]) == [w["vertex"] for w in want]
        assert np.array_equal(r["vis"].astype(bool), vis)
        assert np.array_equal(r["M_final"], Mf), g
    assert kinds == {0, 1} and alternating >= 5 and ms_mattered >= 3, (kinds, alternating, ms_mattered)


def test_first_sweep_sample_vs_one_hop_closed_form():
    """The cpu_baseline helper (or_init_rows + or_first_sweep_sample: the first Alg. 2 sweep over a vertex
    range) equals the 1-hop closed form: max init register over u and its live
    out-neighbours in each sample (brute.khop_registers, hops = 1)."""
    rng = np.random.default_rng(1414)
    for g in range(6):
        n = int(rng.integers(20, 90))
        off, tgt, pr = brute.random_graph(rng, n, 4 * n, None if g % 2 else 0.3)
        J, seed = 64, int(rng.integers(0, 2**32))
        want = brute.khop_registers(n, off, tgt, pr, J, seed, 1)
        u0, u1 = int(rng.integers(0, n // 2)), int(rng.integers(n // 2, n + 1))
        pe, _, rows = oracle.first_sweep_sample(n, off, tgt, pr, J, seed, u0, u1)
        assert pe == off[u1] - off[u0]
        assert np.array_equal(rows, want[u0:u1]), g


def test_init_rows_vs_library_hash():
    """or_init_rows (bounded-sample init, Alg. 1 lines 2-5) writes exactly the listed rows, each equal to
    the sklearn-Murmur3 definition."""
    n, J, seed = 300, 64, 5
    rows = np.array([0, 7, 299, 150], np.int32)
    M = np.zeros((n, J), np.uint8)
    oracle._load().or_init_rows(J, seed, len(rows), rows.ctypes.data, M.ctypes.data)
    want = brute.init_registers(n, J, seed)
    assert np.array_equal(M[rows], want[rows])
    mask = np.ones(n, bool)
    mask[rows] = False
    assert not M[mask].any()


def test_rebuilt_register_definition_vs_bruteforce():
    """or_rebuilt_register (sampled definition of a rebuilt register, used at full size) vs the closure-based
    registers on the residual samples with R_S = R_G(seed prefix) blocked (Alg. 1 lines 21-25, R12)."""
    rng = np.random.default_rng(1515)
    for g in range(12):
        n = int(rng.integers(10, 90))
        off, tgt, pr = brute.random_graph(rng, n, 3 * n, None if g % 3 == 0 else float(rng.choice([0.3, 0.6])))
        J, seed = 32, int(rng.integers(0, 2**32))
        seeds = rng.choice(n, int(rng.integers(1, 4)), replace=False).astype(np.int32)
        blocked = brute.reach_masks(n, off, tgt, pr, J, seed, seeds)
        want = brute.registers(n, off, tgt, pr, J, seed, blocked=blocked)
        us = rng.integers(0, n, 200)
        js = rng.integers(0, J, 200)
        assert np.array_equal(oracle.rebuilt_register(n, off, tgt, pr, J, seed, seeds, us, js), want[us, js]), g


def test_rebuilt_registers_vs_bruteforce():
    """After a rebuild (t = 0, K = 2) the registers are the reach-max on G_j^S with S's reach blocked
    (lines 21-24), and no register exceeds its first-build value."""
    rng = np.random.default_rng(12)
    for g in range(10):
        n = int(rng.integers(10, 80))
        off, tgt, pr = brute.random_graph(rng, n, 3 * n, 0.4)
        J, seed = 32, int(rng.integers(0, 2**32))
        r = oracle.select_seeds(n, off, tgt, pr, J, seed, 2, 0.0, want_final=True)
        blocked = brute.reach_masks(n, off, tgt, pr, J, seed, r["seeds"][:1])
        assert np.array_equal(r["M_final"], brute.registers(n, off, tgt, pr, J, seed, blocked=blocked))
        M1, _ = oracle.simulate(n, off, tgt, pr, J, seed)
        assert (r["M_final"] <= M1).all()


# ---------------------------------------------------------------- Monte-Carlo evaluator (f2, R23)
def test_mix64_reference_outputs():
    """SplitMix64 (Steele et al. 2014) seeded with 0: outputs mix64(k * golden gamma), k = 1, 2, 3."""
    gamma = 0x9E3779B97F4A7C15
    want = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert [oracle.mix64(k * gamma) for k in (1, 2, 3)] == want


def test_mc_draw_uniform_and_independent():
    rng = np.random.default_rng(90)
    N = 40000
    us = rng.integers(0, 1 << 24, N)
    vs = rng.integers(0, 1 << 24, N)
    rs = rng.integers(0, 1 << 20, N)
    d = np.array([oracle.mc_draw(7, int(r), int(u), int(v)) for r, u, v in zip(rs, us, vs)], np.float64)
    assert d.max() < 2**31
    x = d / 2**31
    assert abs(x.mean() - 0.5) < 5 * math.sqrt(1 / 12 / N)
    counts = np.histogram(x, bins=16, range=(0, 1))[0]
    chi2 = ((counts - N / 16) ** 2 / (N / 16)).sum()
    assert chi2 < 60  # 15 dof, p ~ 1e-6
    d2 = np.array([oracle.mc_draw(7, int(r) + 1, int(u), int(v)) for r, u, v in zip(rs, us, vs)], np.float64) / 2**31
    assert abs(np.corrcoef(x, d2)[0, 1]) < 5 / math.sqrt(N)
    d3 = np.array([oracle.mc_draw(8, int(r), int(u), int(v)) for r, u, v in zip(rs, us, vs)], np.float64) / 2**31
    assert abs(np.corrcoef(x, d3)[0, 1]) < 5 / math.sqrt(N)


def test_mc_influence_closed_forms():
    """w = 0: only the seeds; w = 1: the full BFS reach in every sample (a draw equal to h_max, the
    only dead case, has probability 2^-31); star centre: E = 1 + L w; chain: E = sum_i w^i."""
    rng = np.random.default_rng(91)
    n = 60
    off, tgt, _ = brute.random_graph(rng, n, 150, 1.0, allow_dups=False, allow_loops=False)
    seeds = np.array([3, 17, 3 + 1, 40], np.int32)
    R = 64
    c0 = oracle.mc_influence(n, off, tgt, np.zeros(len(tgt), np.float32), seeds, 5, 0, R)
    assert list(c0) == [R * (k + 1) for k in range(4)]
    c1 = oracle.mc_influence(n, off, tgt, np.ones(len(tgt), np.float32), seeds, 5, 0, R)
    A = np.zeros((n, n), bool)
    for u in range(n):
        A[u, tgt[off[u]:off[u + 1]]] = True
    C = brute.closure(A)
    assert list(c1) == [R * int(C[seeds[: k + 1]].any(axis=0).sum()) for k in range(4)]
    L, w, R = 200, 0.1, 4000
    off_s, tgt_s, pr_s = csr_from_edges(L + 1, star(L))
    pr_s = np.full(len(tgt_s), w, np.float32)
    mean = oracle.mc_influence(L + 1, off_s, tgt_s, pr_s, [0], 11, 0, R)[0] / R
    assert abs(mean - (1 + L * w)) < 5 * math.sqrt(L * w * (1 - w) / R)
    d, w = 8, 0.7
    off_c = np.arange(d + 2, dtype=np.int32).clip(max=d)
    tgt_c = np.arange(1, d + 1, dtype=np.int32)
    mean = oracle.mc_influence(d + 1, off_c, tgt_c, np.full(d, w, np.float32), [0], 12, 0, R)[0] / R
    want = sum(w**i for i in range(d + 1))
    var = sum((2 * i + 1) * w**i for i in range(d + 1)) - want**2  # E[X^2] for X = 1 + number of live prefix edges
    assert abs(mean - want) < 5 * math.sqrt(var / R)


def test_mc_influence_sample_ranges_add_up():
    """Counter-based samples: [0, R) = [0, a) + [a, R); counts are non-decreasing in k."""
    rng = np.random.default_rng(92)
    n = 80
    off, tgt, pr = brute.random_graph(rng, n, 300, 0.3)
    seeds = np.array([1, 5, 9], np.int32)
    full = oracle.mc_influence(n, off, tgt, pr, seeds, 3, 0, 96)
    parts = oracle.mc_influence(n, off, tgt, pr, seeds, 3, 0, 40) + oracle.mc_influence(n, off, tgt, pr, seeds, 3, 40, 56)
    assert np.array_equal(full, parts) and all(np.diff(full) >= 0)
