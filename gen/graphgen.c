/*
 * graphgen.c -- seeded, deterministic synthetic input graphs for the five
 * BASELINE.json configs.
 *
 * This module holds INPUTS ONLY: it contains none of the method's arithmetic
 * (no Murmur3, no salts, no live test, no registers).  Both the oracle side
 * (tests/, bench.py cpu_baseline) and the CUDA side consume its CSR output.
 *
 * Randomness: a counter-based SplitMix64 mix of (seed, stream, index), so every
 * edge draw is a pure function of its index and the generator is identical for
 * any OpenMP thread count.  All graphs are directed, self-loop free and
 * deduplicated; every CSR row is sorted by target.
 *
 *   ER       : n vertices, m distinct ordered pairs u != v drawn uniformly (C1).
 *   RMAT     : 2^scale vertices, ef*2^scale draws, quadrant probs a,b,c,d (C2, C4),
 *              Graph500-style seeded vertex relabel permutation.
 *   ChungLu  : weights (i+i0)^(-1/(beta-1)), i0 solved so that the max expected
 *              degree equals dmax for `draws` draws; src and dst drawn independently
 *              from the same weights, then a seeded relabel (C3, C5).
 *   WC probs : p(u,v) = (float)(1.0 / indeg(v)) (Sec. 2.1),
 *              the weighted-cascade model's input weights.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t n, m;
    int64_t *offsets; /* n+1 */
    int32_t *targets; /* m */
} gen_graph;

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
/* counter-based draw: pure function of (seed, stream, idx) */
static inline uint64_t rng_at(uint64_t seed, uint64_t stream, uint64_t idx) {
    return mix64(mix64(seed * 0xD1B54A32D192ED03ull + stream) ^ (idx * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull));
}
/* uniform integer in [0, n) from 32 random bits (n < 2^32) */
static inline uint64_t below(uint32_t r, uint64_t n) { return ((uint64_t)r * n) >> 32; }

static void seeded_permutation(int32_t *perm, int64_t n, uint64_t seed) {
    for (int64_t i = 0; i < n; i++) perm[i] = (int32_t)i;
    for (int64_t i = n - 1; i > 0; i--) {
        uint64_t r = rng_at(seed, 99, (uint64_t)i);
        int64_t j = (int64_t)((r >> 11) % (uint64_t)(i + 1));
        int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/*
 * Edge source for the two-pass counting build.  kind 0 = RMAT, 1 = Chung-Lu.
 * Returns 0 and fills (u,v) for draw i (before self-loop/dup removal).
 */
typedef struct {
    int kind;
    uint64_t seed;
    /* rmat */
    int scale;
    double a, ab, abc;
    /* chung-lu */
    const double *cum; /* n+1 cumulative weights */
    int64_t n;
    const int32_t *perm;
} edge_src;

static inline int64_t cl_pick(const double *cum, int64_t n, double x) {
    int64_t lo = 0, hi = n; /* find largest i with cum[i] <= x, cum[0]=0 */
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (cum[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

static inline void draw_edge(const edge_src *s, uint64_t i, int32_t *pu, int32_t *pv) {
    if (s->kind == 0) {
        uint64_t u = 0, v = 0, r = 0;
        for (int l = 0; l < s->scale; l++) {
            if (!(l & 1)) r = rng_at(s->seed, 1 + (uint64_t)(l >> 1), i);
            uint32_t r32 = (l & 1) ? (uint32_t)(r >> 32) : (uint32_t)r;
            double x = (double)r32 * (1.0 / 4294967296.0);
            int q = x < s->a ? 0 : x < s->ab ? 1 : x < s->abc ? 2 : 3; /* a,b,c,d */
            u = (u << 1) | (uint64_t)(q >= 2);      /* src bit: quadrant in {c,d} */
            v = (v << 1) | (uint64_t)(q & 1);       /* dst bit: quadrant in {b,d} */
        }
        *pu = s->perm[u];
        *pv = s->perm[v];
    } else {
        double W = s->cum[s->n];
        uint64_t r1 = rng_at(s->seed, 1, i), r2 = rng_at(s->seed, 2, i);
        double x1 = (double)(r1 >> 11) * (1.0 / 9007199254740992.0) * W;
        double x2 = (double)(r2 >> 11) * (1.0 / 9007199254740992.0) * W;
        *pu = s->perm[cl_pick(s->cum, s->n, x1)];
        *pv = s->perm[cl_pick(s->cum, s->n, x2)];
    }
}

/* two-pass counting-sort CSR build from `draws` counter-based draws; dedup + no self loops */
static gen_graph *build_from_draws(const edge_src *s, int64_t n, int64_t draws) {
    int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    if (!cnt) return NULL;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < draws; i++) {
        int32_t u, v;
        draw_edge(s, (uint64_t)i, &u, &v);
        if (u != v) __atomic_fetch_add(&cnt[u], 1, __ATOMIC_RELAXED);
    }
    int64_t *off = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    off[0] = 0;
    for (int64_t i = 0; i < n; i++) off[i + 1] = off[i] + cnt[i];
    int64_t raw_m = off[n];
    int32_t *adj = (int32_t *)malloc((size_t)(raw_m ? raw_m : 1) * sizeof(int32_t));
    memcpy(cnt, off, (size_t)n * sizeof(int64_t)); /* cursors */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < draws; i++) {
        int32_t u, v;
        draw_edge(s, (uint64_t)i, &u, &v);
        if (u != v) {
            int64_t p = __atomic_fetch_add(&cnt[u], 1, __ATOMIC_RELAXED);
            adj[p] = v;
        }
    }
    /* sort + dedup each row in place; cnt[u] = deduped row length */
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t u = 0; u < n; u++) {
        int32_t *row = adj + off[u];
        int64_t d = off[u + 1] - off[u], k = 0;
        if (d > 48) qsort(row, (size_t)d, sizeof(int32_t), cmp_i32);
        else
            for (int64_t x = 1; x < d; x++) { /* insertion sort for short rows */
                int32_t key = row[x];
                int64_t y = x - 1;
                while (y >= 0 && row[y] > key) { row[y + 1] = row[y]; y--; }
                row[y + 1] = key;
            }
        for (int64_t e = 0; e < d; e++)
            if (k == 0 || row[e] != row[k - 1]) row[k++] = row[e];
        cnt[u] = k;
    }
    gen_graph *g = (gen_graph *)calloc(1, sizeof(gen_graph));
    g->n = n;
    g->offsets = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    g->offsets[0] = 0;
    for (int64_t u = 0; u < n; u++) g->offsets[u + 1] = g->offsets[u] + cnt[u];
    g->m = g->offsets[n];
    g->targets = (int32_t *)malloc((size_t)(g->m ? g->m : 1) * sizeof(int32_t));
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < n; u++)
        memcpy(g->targets + g->offsets[u], adj + off[u], (size_t)cnt[u] * sizeof(int32_t));
    free(adj);
    free(off);
    free(cnt);
    return g;
}

/* ---------------- public API ---------------- */

gen_graph *gen_rmat(int scale, int64_t edge_factor, double a, double b, double c, uint64_t seed) {
    int64_t n = (int64_t)1 << scale;
    int32_t *perm = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    seeded_permutation(perm, n, seed);
    edge_src s;
    memset(&s, 0, sizeof s);
    s.kind = 0; s.seed = seed; s.scale = scale;
    s.a = a; s.ab = a + b; s.abc = a + b + c; s.perm = perm;
    gen_graph *g = build_from_draws(&s, n, edge_factor * n);
    free(perm);
    return g;
}

/* deterministic (thread-count independent) sum of (i+i0)^-alpha */
static double cl_weight_sum(int64_t n, double i0, double alpha) {
    enum { NB = 256 };
    double part[NB];
#pragma omp parallel for schedule(static)
    for (int b = 0; b < NB; b++) {
        int64_t lo = n * b / NB, hi = n * (b + 1) / NB;
        double acc = 0;
        for (int64_t i = lo; i < hi; i++) acc += pow((double)i + i0, -alpha);
        part[b] = acc;
    }
    double W = 0;
    for (int b = 0; b < NB; b++) W += part[b];
    return W;
}

/* returns i0 actually used via *out_i0 */
gen_graph *gen_chung_lu(int64_t n, int64_t draws, double beta, double dmax, uint64_t seed, double *out_i0) {
    double alpha = 1.0 / (beta - 1.0);
    /* expected degree of vertex 0: draws * i0^-alpha / W(i0); decreasing in i0 -> bisection */
    double lo = 1e-6, hi = (double)n;
    for (int it = 0; it < 100; it++) {
        double mid = sqrt(lo * hi);
        double d0 = (double)draws * pow(mid, -alpha) / cl_weight_sum(n, mid, alpha);
        if (d0 > dmax) lo = mid; else hi = mid;
        if (hi / lo < 1 + 1e-12) break;
    }
    double i0 = sqrt(lo * hi);
    if (out_i0) *out_i0 = i0;
    double *cum = (double *)malloc(((size_t)n + 1) * sizeof(double));
    cum[0] = 0;
    for (int64_t i = 0; i < n; i++) cum[i + 1] = cum[i] + pow((double)i + i0, -alpha);
    int32_t *perm = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    seeded_permutation(perm, n, seed);
    edge_src s;
    memset(&s, 0, sizeof s);
    s.kind = 1; s.seed = seed; s.cum = cum; s.n = n; s.perm = perm;
    gen_graph *g = build_from_draws(&s, n, draws);
    free(perm);
    free(cum);
    return g;
}

/* n vertices, m distinct ordered pairs u != v, uniform (sequential rejection) */
gen_graph *gen_er(int64_t n, int64_t m, uint64_t seed) {
    if (n < 2 || m > n * (n - 1)) return NULL;
    uint64_t cap = 1;
    while (cap < (uint64_t)m * 2 + 16) cap <<= 1;
    uint64_t *set = (uint64_t *)malloc(cap * sizeof(uint64_t));
    memset(set, 0xFF, cap * sizeof(uint64_t));
    uint64_t *keys = (uint64_t *)malloc((size_t)(m ? m : 1) * sizeof(uint64_t));
    int64_t have = 0;
    for (uint64_t i = 0; have < m; i++) {
        uint64_t r = rng_at(seed, 7, i);
        uint64_t u = below((uint32_t)r, (uint64_t)n), v = below((uint32_t)(r >> 32), (uint64_t)n);
        if (u == v) continue;
        uint64_t key = (u << 32) | v, h = mix64(key) & (cap - 1);
        int dup = 0;
        while (set[h] != ~0ull) {
            if (set[h] == key) { dup = 1; break; }
            h = (h + 1) & (cap - 1);
        }
        if (dup) continue;
        set[h] = key;
        keys[have++] = key;
    }
    free(set);
    int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t e = 0; e < m; e++) cnt[keys[e] >> 32]++;
    gen_graph *g = (gen_graph *)calloc(1, sizeof(gen_graph));
    g->n = n; g->m = m;
    g->offsets = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    g->offsets[0] = 0;
    for (int64_t u = 0; u < n; u++) g->offsets[u + 1] = g->offsets[u] + cnt[u];
    g->targets = (int32_t *)malloc((size_t)(m ? m : 1) * sizeof(int32_t));
    for (int64_t u = 0; u < n; u++) cnt[u] = g->offsets[u];
    for (int64_t e = 0; e < m; e++) g->targets[cnt[keys[e] >> 32]++] = (int32_t)(keys[e] & 0xffffffffu);
    for (int64_t u = 0; u < n; u++)
        qsort(g->targets + g->offsets[u], (size_t)(g->offsets[u + 1] - g->offsets[u]), sizeof(int32_t), cmp_i32);
    free(cnt);
    free(keys);
    return g;
}

int64_t gen_n(const gen_graph *g) { return g->n; }
int64_t gen_m(const gen_graph *g) { return g->m; }

/* copy out as int32 CSR (the C-ABI layout); returns -1 if m does not fit int32 */
int gen_copy_csr32(const gen_graph *g, int32_t *offsets, int32_t *targets) {
    if (g->m > 2147483647LL) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i <= g->n; i++) offsets[i] = (int32_t)g->offsets[i];
    memcpy(targets, g->targets, (size_t)g->m * sizeof(int32_t));
    return 0;
}

/* weighted-cascade input weights p(u,v) = (float)(1.0/indeg(v)) */
void gen_wc_probs(int64_t n, int64_t m, const int32_t *targets, float *probs) {
    int64_t *indeg = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    for (int64_t e = 0; e < m; e++) indeg[targets[e]]++;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; e++) probs[e] = (float)(1.0 / (double)indeg[targets[e]]);
    free(indeg);
}

void gen_free(gen_graph *g) {
    if (!g) return;
    free(g->offsets);
    free(g->targets);
    free(g);
}

int gen_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
