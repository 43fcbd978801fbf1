/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  A plain, slow, single-threaded CPU
 * implementation of the error-adaptive sketch-based IM method of
 * arxiv 2105.04023, written from the paper.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  It shares no code with the CUDA path
 * (paper_2105_04023_b200/csrc) and the CUDA path never calls it.
 *
 * Every function follows the paper's definition or algorithm step by step, in
 * the paper's order and notation, with the readings of DESIGN.md "Readings"
 * (R1..R23) where the paper is silent or garbled.  No blocking, fusion or
 * reordering: registers are u8 per (vertex, simulation), blocked/visited flags
 * are one byte per (vertex, simulation), the live test is the double-precision
 * division of Eq. 5 evaluated per (edge, simulation).
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"):
 *   murmur3_32     <- sklearn.utils.murmurhash3_32 (library), SPEC ("",0)->0
 *   mt19937        <- numpy RandomState raw stream (library), C++ std check value
 *   or_salts       <- numpy RandomState stream (library)
 *   or_live        <- closed forms (w=0, w=1), binomial rate, 1-(1-w)^J
 *   or_init        <- sklearn murmur + Python bit_length (independent clz)
 *   or_simulate    <- brute force: per-simulation BFS on explicitly sampled subgraphs
 *                     (register = max init register over the reach set), Fig. 5 shape;
 *                     eps_c > 0: after s synchronous sweeps the register is the max init
 *                     register within s hops (hop distances by scipy's shortest_path), and the
 *                     run stops at the first s with |changed_s| <= eps_c * n
 *   or_estimate    <- closed forms of Eq. 2 (all-0 -> 1.29281, all-10 -> 1323.84)
 *   or_select      <- field by field (seed, score, e, sigma, delta, err_l, err_g, decisions, final
 *                     R_G(S) and registers) vs tests/brute.select_seeds, a whole-array restatement of
 *                     Alg. 1 on closure-based registers / reach sets, 32 graphs incl. (eps_l, eps_g) =
 *                     (0.3, 0.01), eps_c = 0.02, alternating keeps / rebuilds, M_S'-decided picks;
 *                     star / two-star / K=1 reductions, t=0 / t=inf variants
 *   or_init_rows, or_first_sweep_sample (cpu_baseline helpers) <- sklearn-Murmur3 init rows and the
 *                     1-hop closed form
 *   or_reach_register, or_khop_register, or_seed_sigma, or_rebuilt_register <- brute force on small graphs
 *   or_mix64       <- SplitMix64 published reference outputs (seed 0)
 *   or_mc_influence<- closed forms (w = 0, w = 1 -> BFS reach, star 1 + L w, chain sum w^i within
 *                     CLT bounds), draw uniformity / independence
 * All functions are pinned; see DESIGN.md "Parity".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* MurmurHash3 x86_32 (Appleby, public domain), restated.  Eq. 4 uses it */
/* as h(u,v) = Murmur3(u||v) mod 2^31.               */
/* ------------------------------------------------------------------ */
static uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }

uint32_t or_murmur3_32(const uint8_t *data, int64_t len, uint32_t seed) {
    const uint32_t c1 = 0xcc9e2d51u, c2 = 0x1b873593u;
    uint32_t h1 = seed;
    int64_t nblocks = len / 4;
    for (int64_t i = 0; i < nblocks; i++) {
        uint32_t k1 = (uint32_t)data[4 * i] | ((uint32_t)data[4 * i + 1] << 8) |
                      ((uint32_t)data[4 * i + 2] << 16) | ((uint32_t)data[4 * i + 3] << 24);
        k1 *= c1;
        k1 = rotl32(k1, 15);
        k1 *= c2;
        h1 ^= k1;
        h1 = rotl32(h1, 13);
        h1 = h1 * 5 + 0xe6546b64u;
    }
    const uint8_t *tail = data + nblocks * 4;
    uint32_t k1 = 0;
    switch (len & 3) {
    case 3: k1 ^= (uint32_t)tail[2] << 16; /* fallthrough */
    case 2: k1 ^= (uint32_t)tail[1] << 8;  /* fallthrough */
    case 1:
        k1 ^= tail[0];
        k1 *= c1;
        k1 = rotl32(k1, 15);
        k1 *= c2;
        h1 ^= k1;
    }
    h1 ^= (uint32_t)len;
    h1 ^= h1 >> 16;
    h1 *= 0x85ebca6bu;
    h1 ^= h1 >> 13;
    h1 *= 0xc2b2ae35u;
    h1 ^= h1 >> 16;
    return h1;
}

/* little-endian 32-bit word as 4 bytes */
static void le32(uint8_t *b, uint32_t x) {
    b[0] = (uint8_t)x; b[1] = (uint8_t)(x >> 8); b[2] = (uint8_t)(x >> 16); b[3] = (uint8_t)(x >> 24);
}

/* Eq. 4: h(u,v) = Murmur3(u || v) mod 2^31; R4: LE32 u then LE32 v, seed 0 */
uint32_t or_edge_hash(int32_t u, int32_t v) {
    uint8_t key[8];
    le32(key, (uint32_t)u);
    le32(key + 4, (uint32_t)v);
    return or_murmur3_32(key, 8, 0) % 2147483648u;
}

/* ------------------------------------------------------------------ */
/* mt19937 (Matsumoto & Nishimura), the paper's RNG; R3  */
/* ------------------------------------------------------------------ */
typedef struct { uint32_t mt[624]; int idx; } or_mt19937;

void or_mt_seed(or_mt19937 *g, uint32_t s) {
    g->mt[0] = s;
    for (int i = 1; i < 624; i++) g->mt[i] = 1812433253u * (g->mt[i - 1] ^ (g->mt[i - 1] >> 30)) + (uint32_t)i;
    g->idx = 624;
}

uint32_t or_mt_next(or_mt19937 *g) {
    if (g->idx >= 624) {
        for (int i = 0; i < 624; i++) {
            uint32_t y = (g->mt[i] & 0x80000000u) | (g->mt[(i + 1) % 624] & 0x7fffffffu);
            g->mt[i] = g->mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        g->idx = 0;
    }
    uint32_t y = g->mt[g->idx++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

/* draws n values of mt19937(seed) (for the pins) */
void or_mt_draws(uint32_t seed, int64_t n, uint32_t *out) {
    or_mt19937 g;
    or_mt_seed(&g, seed);
    for (int64_t i = 0; i < n; i++) out[i] = or_mt_next(&g);
}

/* R3: one mt19937 stream seeded with the low 32 bits of seed: seed_V, seed_J,
 * then X_r = draw & (2^31-1) for r = 0..J-1 (X_r in [0, h_max], R2) */
void or_salts(uint64_t seed, int32_t J, uint32_t *seed_v, uint32_t *seed_j, uint32_t *X) {
    or_mt19937 g;
    or_mt_seed(&g, (uint32_t)seed);
    *seed_v = or_mt_next(&g);
    *seed_j = or_mt_next(&g);
    for (int32_t r = 0; r < J; r++) X[r] = or_mt_next(&g) & 0x7fffffffu;
}

/* Eq. 5: P(u,v)_r = (X_r xor h(u,v)) / h_max; the edge is in
 * sample r iff P < w (strict).  R1: h_max = 2^31 - 1.  R7: double division. */
int or_live(uint32_t X_r, uint32_t h, float w) {
    double P = (double)(X_r ^ h) / 2147483647.0;
    return P < (double)w;
}

/* clz of a 32-bit word (number of leading zero bits), clz(0) = 32 (R6) */
static int clz32(uint32_t y) { return y ? __builtin_clz(y) : 32; }

static uint32_t hash_index(uint32_t x, uint32_t seed) {
    uint8_t key[4];
    le32(key, x);
    return or_murmur3_32(key, 4, seed);
}

/* Alg. 1 lines 2-5: M_v[j] <- clz(hash(v) xor hash(j)); R5: Murmur3 of
 * LE32 v with seed_V, of LE32 j with seed_J, j 0-based. */
void or_init_registers(int32_t n, int32_t J, uint32_t seed_v, uint32_t seed_j, uint8_t *M) {
    uint32_t *hj = (uint32_t *)malloc((size_t)J * sizeof(uint32_t));
    for (int32_t j = 0; j < J; j++) hj[j] = hash_index((uint32_t)j, seed_j);
    for (int32_t v = 0; v < n; v++) {
        uint32_t hv = hash_index((uint32_t)v, seed_v);
        for (int32_t j = 0; j < J; j++) M[(int64_t)v * J + j] = (uint8_t)clz32(hv ^ hj[j]);
    }
    free(hj);
}

/* the same definition for a list of rows only (bounded samples on large graphs) */
void or_init_rows(int32_t J, uint64_t seed, int64_t nrows, const int32_t *rows, uint8_t *M) {
    uint32_t seed_v, seed_j;
    uint32_t *X = (uint32_t *)malloc((size_t)J * sizeof(uint32_t));
    uint32_t *hj = (uint32_t *)malloc((size_t)J * sizeof(uint32_t));
    or_salts(seed, J, &seed_v, &seed_j, X);
    for (int32_t j = 0; j < J; j++) hj[j] = hash_index((uint32_t)j, seed_j);
    for (int64_t i = 0; i < nrows; i++) {
        int32_t v = rows[i];
        uint32_t hv = hash_index((uint32_t)v, seed_v);
        for (int32_t j = 0; j < J; j++) M[(int64_t)v * J + j] = (uint8_t)clz32(hv ^ hj[j]);
    }
    free(hj);
    free(X);
}

/* Eq. 2: e = 2^{M-bar} / phi, M-bar = avg_j M[j], phi = 0.77351 (R8) */
double or_estimate_row(const uint8_t *row, int32_t J) {
    int64_t sum = 0;
    for (int32_t j = 0; j < J; j++) sum += row[j];
    return pow(2.0, (double)sum / (double)J) / 0.77351;
}

void or_estimate(int32_t n, int32_t J, const uint8_t *M, double *out) {
    for (int32_t v = 0; v < n; v++) out[v] = or_estimate_row(M + (int64_t)v * J, J);
}

typedef struct {
    int32_t sweeps;           /* iterations of the while loop of Alg. 2 */
    int64_t processed_edges;  /* sum over sweeps of out-edges of processed vertices */
    int64_t processed_vertices;
} or_sim_stats;

/*
 * Alg. 2 Simulate(G, M, J, R_S) with the early-exit threshold eps_c
 * (the loop runs while |L|/|V| > eps_c; eps_c = 0 is the exact fixpoint,
 * R11) and the synchronous reading of Fig. 5: every sweep reads the
 * registers as they were when the sweep started (R22: with eps_c > 0 the result depends on
 * the schedule, and this one is the paper's figure's).
 *   L <- V; while |L| / |V| > eps_c:
 *     for u in Gamma^-(L) (R10: in-neighbours of L; the first sweep processes all of V):
 *       for e_{u,v} in A(u): for j: if P(u,v)_j < w_uv and u not in R_S[j]:
 *           M_u[j] <- max(M_u[j], M_v[j])        (R9: pull into u from out-neighbour v)
 *       if M_u changed: L' <- L' + u
 *     L <- L'
 * blocked: n*J bytes, blocked[u*J+j] != 0 iff u in R_S[j]; may be NULL (R_S = {}).
 * change_log (optional, cap entries): number of changed vertices per sweep.
 */
int or_simulate(int32_t n, const int32_t *offsets, const int32_t *targets, const float *probs, int32_t J,
                const uint32_t *X, const uint8_t *blocked, uint8_t *M, or_sim_stats *stats,
                int32_t *change_log, int32_t change_cap, double eps_c) {
    int64_t m = offsets[n];
    uint32_t *h = (uint32_t *)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
    uint8_t *Mold = (uint8_t *)malloc((size_t)n * (size_t)J);
    uint8_t *inL = (uint8_t *)malloc((size_t)n);
    uint8_t *inLnext = (uint8_t *)malloc((size_t)n);
    if (!h || !Mold || !inL || !inLnext) return -3;
    /* the edges' hash values are precomputed */
    for (int32_t u = 0; u < n; u++)
        for (int64_t e = offsets[u]; e < offsets[u + 1]; e++) h[e] = or_edge_hash(u, targets[e]);
    memset(inL, 1, (size_t)n); /* L <- V */
    int64_t Lsize = n;
    or_sim_stats st = {0, 0, 0};
    int first = 1;
    while ((double)Lsize / (double)n > eps_c) { /* Alg. 2 line 3 */
        memcpy(Mold, M, (size_t)n * (size_t)J);
        memset(inLnext, 0, (size_t)n);
        int64_t next = 0, pv = 0, pe = 0;
        /* The iterations over u are independent within a synchronous sweep (u writes only its
         * own row M_u and inLnext[u]; every read is of Mold / inL): the pragma is ignored by the
         * default single-threaded build (CFLAGS in oracle/__init__.py) and only used by the
         * offline golden writer's -fopenmp build, with identical results. */
#pragma omp parallel for schedule(dynamic, 512) reduction(+ : next, pv, pe)
        for (int32_t u = 0; u < n; u++) {
            /* u in Gamma^-(L): some out-neighbour of u is in L (every u in the first sweep) */
            int in_gamma = first;
            for (int64_t e = offsets[u]; e < offsets[u + 1] && !in_gamma; e++) in_gamma = inL[targets[e]];
            if (!in_gamma) continue;
            pv++;
            uint8_t *Mu = M + (int64_t)u * J;
            for (int64_t e = offsets[u]; e < offsets[u + 1]; e++) {
                pe++;
                const uint8_t *Mv = Mold + (int64_t)targets[e] * J;
                for (int32_t j = 0; j < J; j++) {
                    if (or_live(X[j], h[e], probs[e]) && !(blocked && blocked[(int64_t)u * J + j])) {
                        if (Mv[j] > Mu[j]) Mu[j] = Mv[j];
                    }
                }
            }
            if (memcmp(Mu, Mold + (int64_t)u * J, (size_t)J) != 0) {
                inLnext[u] = 1;
                next++;
            }
        }
        st.processed_vertices += pv;
        st.processed_edges += pe;
        if (change_log && st.sweeps < change_cap) change_log[st.sweeps] = (int32_t)next;
        st.sweeps++;
        memcpy(inL, inLnext, (size_t)n);
        Lsize = next;
        first = 0;
    }
    if (stats) *stats = st;
    free(h);
    free(Mold);
    free(inL);
    free(inLnext);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Alg. 1 greedy loop with error-adaptive rebuild    */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t vertex;     /* s */
    int32_t pad;
    int64_t score;      /* sum_j max(M_S'[j], M_s[j]) (integer numerator of the estimate, R14) */
    double e;           /* Estimate(Merge(M_S', M_s)) (line 12, R15) */
    int64_t sigma_count;/* sum_j |R_G(S)[j]|; sigma = sigma_count / J */
    double sigma, delta, err_l, err_g;
    int32_t rebuilt;    /* decision: 1 = else branch (rebuild) taken */
    int32_t executed;   /* 1 if the rebuild work was executed (R18: skipped after the last pick) */
} or_step;

/*
 * One incremental multi-simulation BFS from s over live edges, skipping (v,j)
 * already in R_G(S) (R13: same samples as the sketches; R_G(S) is closed under
 * reachability, so BFS from s restricted to unvisited pairs adds exactly
 * R_G(S+s) \ R_G(S)).  Returns the number of newly visited (v,j) pairs.
 */
static int64_t bfs_add_seed(int32_t n, const int32_t *offsets, const int32_t *targets, const float *probs,
                            const uint32_t *h, int32_t J, const uint32_t *X, int32_t s, uint8_t *vis, int32_t *queue) {
    int64_t added = 0;
    for (int32_t j = 0; j < J; j++) {
        if (vis[(int64_t)s * J + j]) continue;
        int64_t qh = 0, qt = 0;
        vis[(int64_t)s * J + j] = 1;
        added++;
        queue[qt++] = s;
        while (qh < qt) {
            int32_t u = queue[qh++];
            for (int64_t e = offsets[u]; e < offsets[u + 1]; e++) {
                int32_t v = targets[e];
                if (!vis[(int64_t)v * J + j] && or_live(X[j], h[e], probs[e])) {
                    vis[(int64_t)v * J + j] = 1;
                    added++;
                    queue[qt++] = v;
                }
            }
        }
    }
    (void)n;
    return added;
}

typedef struct {
    int32_t builds;          /* initial build + executed rebuilds */
    int32_t total_sweeps;
    int64_t total_processed_edges;
} or_select_stats;

/*
 * Alg. 1 with eps_l, eps_g (R17: the C-ABI's single threshold t sets both) and the
 * readings R12-R21.  Starts from freshly built sketches (Simulate with R_S = {}).
 * out_seeds[k], out_scores[k] = sigma after k+1 seeds (R21).  vis_out (optional,
 * n*J bytes) receives the final R_G(S).  M_final (optional) receives the registers
 * at return (after the last executed rebuild, or the first build if none ran); M_first
 * (optional) the registers of the first build (lines 2-6).
 */
int or_select_seeds(int32_t n, const int32_t *offsets, const int32_t *targets, const float *probs, int32_t J,
                    uint64_t seed, int32_t K, double eps_l, double eps_g, double eps_c, int32_t *out_seeds, double *out_scores,
                    or_step *log, uint8_t *vis_out, uint8_t *M_final, or_select_stats *sstats, uint8_t *M_first) {
    int64_t m = offsets[n];
    uint32_t seed_v, seed_j;
    uint32_t *X = (uint32_t *)malloc((size_t)J * sizeof(uint32_t));
    or_salts(seed, J, &seed_v, &seed_j, X);
    uint32_t *h = (uint32_t *)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
    for (int32_t u = 0; u < n; u++)
        for (int64_t e = offsets[u]; e < offsets[u + 1]; e++) h[e] = or_edge_hash(u, targets[e]);
    uint8_t *M = (uint8_t *)malloc((size_t)n * (size_t)J);
    uint8_t *vis = (uint8_t *)calloc((size_t)n * (size_t)J, 1);
    uint8_t *inS = (uint8_t *)calloc((size_t)n, 1);
    uint8_t *MS = (uint8_t *)calloc((size_t)J, 1);
    int32_t *queue = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!X || !h || !M || !vis || !inS || !MS || !queue) return -3;
    or_select_stats ss = {0, 0, 0};
    or_sim_stats st;

    /* lines 2-6: init + Simulate(G, M, J, {}) */
    or_init_registers(n, J, seed_v, seed_j, M);
    or_simulate(n, offsets, targets, probs, J, X, NULL, M, &st, NULL, 0, eps_c);
    ss.builds++;
    ss.total_sweeps += st.sweeps;
    ss.total_processed_edges += st.processed_edges;
    if (M_first) memcpy(M_first, M, (size_t)n * (size_t)J);
    /* lines 7-8: M_S' <- zeros(J); varsigma <- 0 */
    double varsigma = 0.0;
    int64_t sigma_count = 0;

    for (int32_t k = 0; k < K; k++) {
        /* line 10: s <- argmax_v Estimate(Merge(M_S', M_v)).  R14: Estimate is monotone in the
         * integer sum of the merged registers; ties -> lowest id; the pool excludes v whose
         * visited row is all ones (covers S); if the pool is empty, the lowest-id v not in S. */
        int32_t s = -1;
        int64_t best = -1;
        for (int32_t v = 0; v < n; v++) {
            int all = 1;
            for (int32_t j = 0; j < J && all; j++) all = vis[(int64_t)v * J + j] != 0;
            if (all) continue;
            int64_t score = 0;
            for (int32_t j = 0; j < J; j++) {
                uint8_t a = MS[j], b = M[(int64_t)v * J + j];
                score += a > b ? a : b;
            }
            if (score > best) { best = score; s = v; }
        }
        if (s < 0) {
            for (int32_t v = 0; v < n; v++)
                if (!inS[v]) { s = v; break; }
            best = 0;
            for (int32_t j = 0; j < J; j++) {
                uint8_t a = MS[j], b = M[(int64_t)s * J + j];
                best += a > b ? a : b;
            }
        }
        /* line 11: S <- S + s */
        inS[s] = 1;
        /* line 12: e <- Estimate(Merge(M_S', M_s)) (R15) */
        double e = pow(2.0, (double)best / (double)J) / 0.77351;
        /* lines 13-14: R_G(S) and the Monte-Carlo influence sigma over the same samples (R13) */
        sigma_count += bfs_add_seed(n, offsets, targets, probs, h, J, X, s, vis, queue);
        double sigma = (double)sigma_count / (double)J;
        /* lines 15-17 (R16: err_l = +inf when delta = 0) */
        double delta = sigma - varsigma;
        double err_l = delta != 0.0 ? fabs((e - delta) / delta) : INFINITY;
        double err_g = fabs((e - delta) / sigma);
        int rebuild = !(err_l < eps_l || err_g < eps_g);
        int executed = 0;
        if (!rebuild) {
            /* line 19: M_S' <- Merge(M_S', M_s) (Eq. 3) */
            for (int32_t j = 0; j < J; j++)
                if (M[(int64_t)s * J + j] > MS[j]) MS[j] = M[(int64_t)s * J + j];
        } else if (k < K - 1) {
            /* lines 21-27 (R18: skipped after the last pick, it cannot change the output) */
            or_init_registers(n, J, seed_v, seed_j, M);
            or_simulate(n, offsets, targets, probs, J, X, vis, M, &st, NULL, 0, eps_c);
            ss.builds++;
            ss.total_sweeps += st.sweeps;
            ss.total_processed_edges += st.processed_edges;
            memset(MS, 0, (size_t)J);
            varsigma = sigma;
            executed = 1;
        }
        out_seeds[k] = s;
        out_scores[k] = sigma;
        if (log) {
            or_step *L = &log[k];
            memset(L, 0, sizeof *L);
            L->vertex = s; L->score = best; L->e = e; L->sigma_count = sigma_count;
            L->sigma = sigma; L->delta = delta; L->err_l = err_l; L->err_g = err_g;
            L->rebuilt = rebuild; L->executed = executed;
        }
    }
    if (vis_out) memcpy(vis_out, vis, (size_t)n * (size_t)J);
    if (M_final) memcpy(M_final, M, (size_t)n * (size_t)J);
    if (sstats) *sstats = ss;
    free(X); free(h); free(M); free(vis); free(inS); free(MS); free(queue);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Per-sample definitions used for sampled parity at full sizes.       */
/* ------------------------------------------------------------------ */

/*
 * The plain definition of a converged register (first build, R_S = {}): the
 * FM union of the singleton sketches of every vertex reachable from u in the
 * j-th sampled subgraph G_j = {(x,y) : P(x,y)_j < w_xy}:
 *   M_u[j] = max_{w in R_{G_j}(u)} clz(hash(w) xor hash(j))   (Eq. 1 + Eq. 3)
 * Evaluated by BFS for npairs (u, j) pairs.
 */
int or_reach_register(int32_t n, const int32_t *offsets, const int32_t *targets, const float *probs, int32_t J,
                      uint64_t seed, int64_t npairs, const int32_t *us, const int32_t *js, uint8_t *out) {
    uint32_t seed_v, seed_j;
    uint32_t *X = (uint32_t *)malloc((size_t)J * sizeof(uint32_t));
    or_salts(seed, J, &seed_v, &seed_j, X);
    uint8_t *seen = (uint8_t *)calloc((size_t)n, 1);
    int32_t *queue = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!X || !seen || !queue) return -3;
    for (int64_t p = 0; p < npairs; p++) {
        int32_t u = us[p], j = js[p];
        uint32_t hj = hash_index((uint32_t)j, seed_j);
        int64_t qh = 0, qt = 0;
        int best = 0;
        seen[u] = 1;
        queue[qt++] = u;
        while (qh < qt) {
            int32_t x = queue[qh++];
            int r = clz32(hash_index((uint32_t)x, seed_v) ^ hj);
            if (r > best) best = r;
            for (int64_t e = offsets[x]; e < offsets[x + 1]; e++) {
                int32_t y = targets[e];
                if (!seen[y] && or_live(X[j], or_edge_hash(x, y), probs[e])) {
                    seen[y] = 1;
                    queue[qt++] = y;
                }
            }
        }
        for (int64_t q = 0; q < qt; q++) seen[queue[q]] = 0;
        out[p] = (uint8_t)best;
    }
    free(X); free(seen); free(queue);
    return 0;
}

/*
 * The plain definition of a register after a rebuild (Alg. 1 lines 21-25; reading
 * R12): with R_S[j] = R_{G_j}(S) for the seed prefix S = seeds[0..nseeds-1], a blocked vertex never
 * pulls, so in sample j
 *   M_u[j] = init(u, j)                                          if u in R_S[j]
 *          = max over w reachable from u in G_j^S of init(w, j)   otherwise,
 * G_j^S = {(x,y) live in sample j : x not in R_S[j]} (a blocked y is reached and keeps its init value
 * but is not expanded).  Pairs are evaluated in the given order; R_S[j] is recomputed by BFS from S
 * whenever j differs from the previous pair's (sort the pairs by j).
 */
int or_rebuilt_register(int32_t n, const int32_t *offsets, const int32_t *targets, const float *probs, int32_t J,
                        uint64_t seed, int32_t nseeds, const int32_t *seeds, int64_t npairs, const int32_t *us,
                        const int32_t *js, uint8_t *out) {
    uint32_t seed_v, seed_j;
    uint32_t *X = (uint32_t *)malloc((size_t)J * sizeof(uint32_t));
    or_salts(seed, J, &seed_v, &seed_j, X);
    uint8_t *blocked = (uint8_t *)calloc((size_t)n, 1);
    uint8_t *seen = (uint8_t *)calloc((size_t)n, 1);
    int32_t *queue = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!X || !blocked || !seen || !queue) return -3;
    int32_t cur_j = -1;
    for (int64_t p = 0; p < npairs; p++) {
        int32_t u = us[p], j = js[p];
        if (j != cur_j) {  /* R_S[j]: BFS from the seed prefix over the live edges of sample j */
            memset(blocked, 0, (size_t)n);
            int64_t qh = 0, qt = 0;
            for (int32_t k = 0; k < nseeds; k++)
                if (!blocked[seeds[k]]) { blocked[seeds[k]] = 1; queue[qt++] = seeds[k]; }
            while (qh < qt) {
                int32_t x = queue[qh++];
                for (int64_t e = offsets[x]; e < offsets[x + 1]; e++) {
                    int32_t y = targets[e];
                    if (!blocked[y] && or_live(X[j], or_edge_hash(x, y), probs[e])) { blocked[y] = 1; queue[qt++] = y; }
                }
            }
            cur_j = j;
        }
        uint32_t hj = hash_index((uint32_t)j, seed_j);
        int64_t qh = 0, qt = 0;
        int best = 0;
        seen[u] = 1;
        queue[qt++] = u;
        while (qh < qt) {
            int32_t x = queue[qh++];
            int r = clz32(hash_index((uint32_t)x, seed_v) ^ hj);
            if (r > best) best = r;
            if (blocked[x]) continue;  /* x in R_S[j] never pulls: its out-edges are not in G_j^S */
            for (int64_t e = offsets[x]; e < offsets[x + 1]; e++) {
                int32_t y = targets[e];
                if (!seen[y] && or_live(X[j], or_edge_hash(x, y), probs[e])) { seen[y] = 1; queue[qt++] = y; }
            }
        }
        for (int64_t q = 0; q < qt; q++) seen[queue[q]] = 0;
        out[p] = (uint8_t)best;
    }
    free(X); free(blocked); free(seen); free(queue);
    return 0;
}

/*
 * The plain definition of a register after `hops` synchronous sweeps of the first build (eps_c > 0,
 * reading R22): the FM union over the vertices within `hops` hops of u in G_j,
 *   M_u[j] = max_{w : dist_{G_j}(u, w) <= hops} clz(hash(w) xor hash(j)).
 * Level-synchronous BFS for npairs (u, j) pairs.
 */
int or_khop_register(int32_t n, const int32_t *offsets, const int32_t *targets, const float *probs, int32_t J,
                     uint64_t seed, int32_t hops, int64_t npairs, const int32_t *us, const int32_t *js, uint8_t *out) {
    uint32_t seed_v, seed_j;
    uint32_t *X = (uint32_t *)malloc((size_t)J * sizeof(uint32_t));
    or_salts(seed, J, &seed_v, &seed_j, X);
    uint8_t *seen = (uint8_t *)calloc((size_t)n, 1);
    int32_t *queue = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *depth = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!X || !seen || !queue || !depth) return -3;
    for (int64_t p = 0; p < npairs; p++) {
        int32_t u = us[p], j = js[p];
        uint32_t hj = hash_index((uint32_t)j, seed_j);
        int64_t qh = 0, qt = 0;
        int best = 0;
        seen[u] = 1;
        depth[u] = 0;
        queue[qt++] = u;
        while (qh < qt) {
            int32_t x = queue[qh++];
            int r = clz32(hash_index((uint32_t)x, seed_v) ^ hj);
            if (r > best) best = r;
            if (depth[x] == hops) continue;
            for (int64_t e = offsets[x]; e < offsets[x + 1]; e++) {
                int32_t y = targets[e];
                if (!seen[y] && or_live(X[j], or_edge_hash(x, y), probs[e])) {
                    seen[y] = 1;
                    depth[y] = depth[x] + 1;
                    queue[qt++] = y;
                }
            }
        }
        for (int64_t q = 0; q < qt; q++) seen[queue[q]] = 0;
        out[p] = (uint8_t)best;
    }
    free(X); free(seen); free(queue); free(depth);
    return 0;
}

/*
 * sigma for a given seed sequence (Alg. 1 lines 13-14): for every simulation j,
 * the number of vertices reachable in G_j from the first k+1 seeds, summed over j.
 * out_counts[k] = sum_j |R_{G_j}({s_0..s_k})|.  Memory O(n): one simulation at a time.
 */
int or_seed_sigma(int32_t n, const int32_t *offsets, const int32_t *targets, const float *probs, int32_t J,
                  uint64_t seed, int32_t K, const int32_t *seeds, int64_t *out_counts) {
    uint32_t seed_v, seed_j;
    uint32_t *X = (uint32_t *)malloc((size_t)J * sizeof(uint32_t));
    or_salts(seed, J, &seed_v, &seed_j, X);
    uint8_t *seen = (uint8_t *)calloc((size_t)n, 1);
    int32_t *queue = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!X || !seen || !queue) return -3;
    for (int32_t k = 0; k < K; k++) out_counts[k] = 0;
    for (int32_t j = 0; j < J; j++) {
        int64_t qt = 0, qh = 0;
        for (int32_t k = 0; k < K; k++) {
            int32_t s = seeds[k];
            if (!seen[s]) {
                seen[s] = 1;
                queue[qt++] = s;
            }
            while (qh < qt) {
                int32_t x = queue[qh++];
                for (int64_t e = offsets[x]; e < offsets[x + 1]; e++) {
                    int32_t y = targets[e];
                    if (!seen[y] && or_live(X[j], or_edge_hash(x, y), probs[e])) {
                        seen[y] = 1;
                        queue[qt++] = y;
                    }
                }
            }
            out_counts[k] += qt;
        }
        for (int64_t q = 0; q < qt; q++) seen[queue[q]] = 0;
    }
    free(X); free(seen); free(queue);
    return 0;
}

/*
 * Bounded-sample timing helper for the cpu_baseline: the first iteration of
 * Alg. 2 (all u processed, registers read as they were at the sweep start)
 * restricted to vertices [u_begin, u_end).  M must hold the initial registers
 * of those vertices and of their out-neighbours (or_init_rows).  The new rows
 * are written to Mnew ((u_end-u_begin)*J bytes).  Returns processed edges.
 */
int64_t or_first_sweep_sample(int32_t n, const int32_t *offsets, const int32_t *targets, const float *probs,
                              int32_t J, uint64_t seed, int32_t u_begin, int32_t u_end, const uint8_t *M,
                              uint8_t *Mnew) {
    uint32_t seed_v, seed_j;
    uint32_t *X = (uint32_t *)malloc((size_t)J * sizeof(uint32_t));
    or_salts(seed, J, &seed_v, &seed_j, X);
    int64_t processed = 0;
    for (int32_t u = u_begin; u < u_end; u++) {
        uint8_t *row = Mnew + (int64_t)(u - u_begin) * J;
        memcpy(row, M + (int64_t)u * J, (size_t)J);
        for (int64_t e = offsets[u]; e < offsets[u + 1]; e++) {
            uint32_t h = or_edge_hash(u, targets[e]);
            const uint8_t *Mv = M + (int64_t)targets[e] * J;
            processed++;
            for (int32_t j = 0; j < J; j++)
                if (or_live(X[j], h, probs[e]) && Mv[j] > row[j]) row[j] = Mv[j];
        }
    }
    (void)n;
    free(X);
    return processed;
}

/*
 * Per-simulation form of or_seed_sigma for a subset of simulations (sampled parity at full size):
 * out[s*K + k] = |R_{G_j}({seeds_0..seeds_k})| for j = sims[s] (Alg. 1 lines 13-14, R13).
 */
int or_seed_reach_per_sim(int32_t n, const int32_t *offsets, const int32_t *targets, const float *probs, int32_t J,
                          uint64_t seed, int32_t nsims, const int32_t *sims, int32_t K, const int32_t *seeds, int64_t *out) {
    uint32_t seed_v, seed_j;
    uint32_t *X = (uint32_t *)malloc((size_t)J * sizeof(uint32_t));
    or_salts(seed, J, &seed_v, &seed_j, X);
    uint8_t *seen = (uint8_t *)calloc((size_t)n, 1);
    int32_t *queue = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!X || !seen || !queue) return -3;
    for (int32_t si = 0; si < nsims; si++) {
        int32_t j = sims[si];
        int64_t qt = 0, qh = 0;
        for (int32_t k = 0; k < K; k++) {
            int32_t s = seeds[k];
            if (!seen[s]) {
                seen[s] = 1;
                queue[qt++] = s;
            }
            while (qh < qt) {
                int32_t x = queue[qh++];
                for (int64_t e = offsets[x]; e < offsets[x + 1]; e++) {
                    int32_t y = targets[e];
                    if (!seen[y] && or_live(X[j], or_edge_hash(x, y), probs[e])) {
                        seen[y] = 1;
                        queue[qt++] = y;
                    }
                }
            }
            out[(int64_t)si * K + k] = qt;
        }
        for (int64_t q = 0; q < qt; q++) seen[queue[q]] = 0;
    }
    free(X); free(seen); free(queue);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Independent Monte-Carlo influence evaluator.     */
/* ------------------------------------------------------------------ */

/*
 * The paper scores every seed set with an independent sample-then-diffuse oracle using fresh
 * randomness.  Reading R23: the fresh value of edge (u,v) in sample r is a
 * counter-based SplitMix64 draw (Steele, Lea, Flood 2014; restated) instead of an mt19937 stream,
 * so that any sample can be evaluated independently:
 *   z_e   = mix64(seed xor (u << 32 | v))
 *   P_r   = (mix64(z_e + (r + 1) * 0x9E3779B97F4A7C15) >> 33) / h_max        (31-bit draw)
 * and (u,v) is live in sample r iff P_r < w_uv -- the live test of Eq. 5 with the
 * draw in place of X_r xor h(u,v).
 */
uint64_t or_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint32_t or_mc_draw(uint64_t seed, int64_t r, int32_t u, int32_t v) {
    uint64_t ze = or_mix64(seed ^ (((uint64_t)(uint32_t)u << 32) | (uint64_t)(uint32_t)v));
    return (uint32_t)(or_mix64(ze + (uint64_t)(r + 1) * 0x9E3779B97F4A7C15ULL) >> 33);
}

/*
 * out_counts[k] = sum over samples r = r0 .. r0+R-1 of |R_{G_r}({seeds_0 .. seeds_k})|: the
 * influence of every prefix of the seed sequence, times R (mean = count / R).  One BFS per
 * sample and seed, incremental over k (R_G(S) is closed under reachability).
 */
int or_mc_influence(int32_t n, const int32_t *offsets, const int32_t *targets, const float *probs, int32_t K,
                    const int32_t *seeds, uint64_t seed, int64_t r0, int64_t R, int64_t *out_counts) {
    uint8_t *seen = (uint8_t *)calloc((size_t)n, 1);
    int32_t *queue = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!seen || !queue) return -3;
    for (int32_t k = 0; k < K; k++) out_counts[k] = 0;
    for (int64_t r = r0; r < r0 + R; r++) {
        int64_t qt = 0, qh = 0;
        for (int32_t k = 0; k < K; k++) {
            int32_t s = seeds[k];
            if (!seen[s]) {
                seen[s] = 1;
                queue[qt++] = s;
            }
            while (qh < qt) {
                int32_t x = queue[qh++];
                for (int64_t e = offsets[x]; e < offsets[x + 1]; e++) {
                    int32_t y = targets[e];
                    if (!seen[y] && or_live(or_mc_draw(seed, r, x, y), 0u, probs[e])) {
                        seen[y] = 1;
                        queue[qt++] = y;
                    }
                }
            }
            out_counts[k] += qt;
        }
        for (int64_t q = 0; q < qt; q++) seen[queue[q]] = 0;
    }
    free(seen); free(queue);
    return 0;
}
