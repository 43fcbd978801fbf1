// im_first.cu -- register init (Alg. 1 lines 2-5) fused with the first sweep of Alg. 2, and the
// same gather as a full in-place sweep for dense frontiers (direction-optimised Simulate).
//
// In the first sweep every vertex is live and every register still holds its init value
// M_v[j] = clz(hash(v) xor hash(j)), which is a pure function of (v, j).  So the
// first sweep is computed as a gather, one warp per vertex u over its out-edges (pull, reading R9):
// row(u) = max(init(u), max over live (u,v), u not blocked, of init(v)) -- exactly the synchronous
// first iteration -- with init(v) recomputed from the hashes instead of read from HBM.  The warp
// owns the row, so it is written once, without global atomics, together with u's exact
// per-simulation change mask (row != init) that drives the second sweep (im_sweep.cu).
// With MEM = true the same kernel is a full gather sweep reading the current registers (used when
// the next push frontier would cover nearly every edge): rows are read and written sequentially,
// only the window words of the out-neighbours are random reads; in place (Gauss-Seidel), and the
// fixpoint is unique.
//
// The working row lives in shared memory as packed 4-register words; an edge merges the live
// registers of its window word by word with a shared-memory bytewise-max CAS.
// Vertices with more than FIRST_BIG out-edges are done by a whole block (k_first_big).
#include <algorithm>

#include "im_device.cuh"
#include "im_internal.h"

namespace im {

struct FirstArgs {
    int n, J;
    uint32_t seedV;
    const int32_t* off;
    const uint2* fwd;
    const uint32_t* fwdT;
    uint32_t T0;
    const uint32_t* Xs;
    const uint16_t* s12;
    const int32_t* perm;
    uint32_t seedJ;
    uint8_t* M;
    const uint32_t* vis;
    uint32_t* cm_out;
    uint32_t* bits_out;
    IterCounters* ctr;
    const int4* big_units;  // {u, eb, ee}: rows with > FIRST_BIG out-edges in units of <= FIRST_CHUNK (k_first_big)
    int n_big;
    int vb;              // vertices per warp batch (<= 256; fewer on small graphs so every warp gets work)
    bool thread_rows;    // constant threshold, sparse windows: rows <= 32 edges are gathered one row per lane (first_thread)
    bool small_rows;     // rows <= 32 edges take the window-words-only path (false: wide windows, e.g. p = 0.1 with
                         // J >= 512, where every lane walking its own 64+-simulation window serially contends in
                         // shared memory; the whole-row path merges wide windows with lanes over words instead)
};

// hash(v) of Alg. 1 line 4, recomputed per edge (a per-build table of it read per edge measured no faster)
__device__ __forceinline__ uint32_t vhash(const FirstArgs& a, uint32_t v) { return murmur_word(v, a.seedV); }

// init registers of simulations 4w..4w+3 of a vertex with hash hv, packed
__device__ __forceinline__ uint32_t init_word(uint32_t hv, const uint32_t* sHJ, int w) {
    const uint4 h = reinterpret_cast<const uint4*>(sHJ)[w];
    return (uint32_t)__clz(hv ^ h.x) | ((uint32_t)__clz(hv ^ h.y) << 8) | ((uint32_t)__clz(hv ^ h.z) << 16) |
           ((uint32_t)__clz(hv ^ h.w) << 24);
}

// shared-memory bytewise max
__device__ __forceinline__ void smem_vmax(uint32_t* p, uint32_t val) {
    uint32_t cur = *p;
    uint32_t nw = __vmaxu4(cur, val);
    while (nw != cur) {
        uint32_t prev = atomicCAS(p, cur, nw);
        if (prev == cur) return;
        cur = prev;
        nw = __vmaxu4(cur, val);
    }
}

// byte mask of the simulations 4w..4w+3 that are live for (h, T) (Eq. 5).  No window bounds are needed: the
// salt of a simulation outside the edge's window lies in another 2^B block than h, so (X xor h) >= 2^B >= T.
__device__ __forceinline__ uint32_t live_word(const uint32_t* sX, uint32_t h, uint32_t T, int w) {
    const uint4 x = reinterpret_cast<const uint4*>(sX)[w];
    return ((x.x ^ h) < T ? 0x000000FFu : 0u) | ((x.y ^ h) < T ? 0x0000FF00u : 0u) | ((x.z ^ h) < T ? 0x00FF0000u : 0u) |
           ((x.w ^ h) < T ? 0xFF000000u : 0u);
}

// merge word w of edge (u -> v, h, T) restricted to [lo, hi) into the smem row
template <bool BLOCKED, bool MEM>
__device__ __forceinline__ void merge_word(const FirstArgs& a, const uint32_t* sX, const uint32_t* sHJ, const uint32_t* sVis,
                                           uint32_t* row, uint32_t v, uint32_t hv, uint32_t h, uint32_t T, int lo, int hi, int w,
                                           bool have_pre = false, uint32_t pre = 0u) {
    uint32_t live = live_word(sX, h, T, w);
    (void)lo;
    (void)hi;
    if (BLOCKED && live) live &= ~expand4((sVis[w >> 3] >> ((w & 7) << 2)) & 0xFu);
    if (!live) return;
    uint32_t val = MEM ? (have_pre ? pre : reinterpret_cast<const uint32_t*>(a.M)[(size_t)v * (a.J >> 2) + w]) : init_word(hv, sHJ, w);
    val &= live;
    if (__vmaxu4(row[w], val) != row[w]) smem_vmax(&row[w], val);
}

#ifndef IM_FIRST_DENSE_WIN
#define IM_FIRST_DENSE_WIN 48
#endif
// gather sweeps: windows wider than this are walked by the whole warp.  Unlike the push sweeps and BFS levels (whose
// per-lane path keeps a window's live bits in one 32-bit word, DENSE_WIN <= 32) the per-lane gather walks any width.
constexpr int FIRST_DENSE_WIN = IM_FIRST_DENSE_WIN;

// `e` is this lane's edge (or -1); the loop around it must be warp-uniform.  Windows wider than
// DENSE_WIN simulations (w close to 1) are walked by the whole warp, one word per lane.
template <bool CONST_T, bool BLOCKED, bool MEM>
__device__ __forceinline__ void gather_rec(const FirstArgs& a, const uint32_t* sX, const uint16_t* sS, const uint32_t* sHJ,
                                           const uint32_t* sVis, uint32_t* row, bool have, uint2 f, uint32_t Tin, uint32_t& wcount);

template <bool CONST_T, bool BLOCKED, bool MEM>
__device__ __forceinline__ void gather_edge(const FirstArgs& a, const uint32_t* sX, const uint16_t* sS, const uint32_t* sHJ,
                                            const uint32_t* sVis, uint32_t* row, int e, uint32_t& wcount) {
    uint2 f = make_uint2(0, 0);
    uint32_t T = 0;
    if (e >= 0) {
        f = ld_stream(&a.fwd[e]);
        T = CONST_T ? a.T0 : ld_stream(&a.fwdT[e]);
    }
    gather_rec<CONST_T, BLOCKED, MEM>(a, sX, sS, sHJ, sVis, row, e >= 0, f, T, wcount);
}

// the edge's record is already loaded (prefetched by the caller)
template <bool CONST_T, bool BLOCKED, bool MEM>
__device__ __forceinline__ void gather_rec(const FirstArgs& a, const uint32_t* sX, const uint16_t* sS, const uint32_t* sHJ,
                                           const uint32_t* sVis, uint32_t* row, bool have, uint2 f, uint32_t Tin, uint32_t& wcount) {
    const int lane = threadIdx.x & 31;
    uint32_t h = 0, T = 0, hv = 0, v = 0;
    int lo = 0, hi = 0;
    if (have) {
        T = Tin;
        h = f.y;
        v = f.x;
        if (T) {
            edge_window(h, T, sX, sS, a.J, lo, hi);
            if (lo < hi) {
                wcount++;
                if (!MEM) hv = vhash(a, v);
            }
        }
    }
    const bool dense = hi - lo > FIRST_DENSE_WIN;
    if (!dense && lo < hi)
        for (int w = lo >> 2; w <= (hi - 1) >> 2; ++w) merge_word<BLOCKED, MEM>(a, sX, sHJ, sVis, row, v, hv, h, T, lo, hi, w);
    uint32_t dmask = __ballot_sync(IM_FULL, dense);
    while (dmask) {
        int l = __ffs(dmask) - 1;
        dmask &= dmask - 1;
        uint32_t dh = __shfl_sync(IM_FULL, h, l), dT = __shfl_sync(IM_FULL, T, l), dhv = __shfl_sync(IM_FULL, hv, l);
        uint32_t dv = __shfl_sync(IM_FULL, v, l);
        int dlo = __shfl_sync(IM_FULL, lo, l), dhi = __shfl_sync(IM_FULL, hi, l);
        for (int w = (dlo >> 2) + lane; w <= (dhi - 1) >> 2; w += 32)
            merge_word<BLOCKED, MEM>(a, sX, sHJ, sVis, row, dv, dhv, dh, dT, dlo, dhi, w);
    }
}

// U edges per lane, e0 + lane + k * stride (k < U): all records are loaded, then every window and
// (MEM) the first window word of every edge, before any is merged -- the gather is bound by these
// dependent random loads, so U of them are kept in flight per lane.  Warp-uniform like gather_rec.
template <bool CONST_T, bool BLOCKED, bool MEM, int U>
__device__ __forceinline__ void gather_multi(const FirstArgs& a, const uint32_t* sX, const uint16_t* sS, const uint32_t* sHJ,
                                             const uint32_t* sVis, uint32_t* row, int e0, int ee, int stride, uint32_t& wcount) {
    const int lane = threadIdx.x & 31;
    uint2 f[U];
    uint32_t T[U];
#pragma unroll
    for (int k = 0; k < U; k++) {
        const int e = e0 + lane + k * stride;
        f[k] = make_uint2(0, 0);
        T[k] = 0u;
        if (e < ee) {
            f[k] = ld_stream(&a.fwd[e]);
            T[k] = CONST_T ? a.T0 : ld_stream(&a.fwdT[e]);
        }
    }
    int lo[U], hi[U];
    uint32_t pre[U], pre2[U], hv[U];
#pragma unroll
    for (int k = 0; k < U; k++) {
        lo[k] = hi[k] = 0;
        hv[k] = pre[k] = pre2[k] = 0u;
        if (T[k]) edge_window(f[k].y, T[k], sX, sS, a.J, lo[k], hi[k]);
        if (lo[k] < hi[k]) {
            wcount++;
            if (!MEM) hv[k] = vhash(a, f[k].x);
            else if (hi[k] - lo[k] <= FIRST_DENSE_WIN) {  // the first two window words (a 4-simulation window spans two words 3/4 of the time)
                const uint32_t* rv = reinterpret_cast<const uint32_t*>(a.M) + (size_t)f[k].x * (a.J >> 2);
                pre[k] = rv[lo[k] >> 2];
                if (((hi[k] - 1) >> 2) > (lo[k] >> 2)) pre2[k] = rv[(lo[k] >> 2) + 1];
            }
        }
    }
#pragma unroll
    for (int k = 0; k < U; k++) {
        if (lo[k] < hi[k] && hi[k] - lo[k] <= FIRST_DENSE_WIN)
            for (int w = lo[k] >> 2; w <= (hi[k] - 1) >> 2; ++w)
                merge_word<BLOCKED, MEM>(a, sX, sHJ, sVis, row, f[k].x, hv[k], f[k].y, T[k], lo[k], hi[k], w, w - (lo[k] >> 2) < 2,
                                         w == (lo[k] >> 2) ? pre[k] : pre2[k]);
        uint32_t dmask = __ballot_sync(IM_FULL, hi[k] - lo[k] > FIRST_DENSE_WIN);
        while (dmask) {
            const int l = __ffs(dmask) - 1;
            dmask &= dmask - 1;
            const uint32_t dh = __shfl_sync(IM_FULL, f[k].y, l), dT = __shfl_sync(IM_FULL, T[k], l), dhv = __shfl_sync(IM_FULL, hv[k], l);
            const uint32_t dv = __shfl_sync(IM_FULL, f[k].x, l);
            const int dlo = __shfl_sync(IM_FULL, lo[k], l), dhi = __shfl_sync(IM_FULL, hi[k], l);
            for (int w = (dlo >> 2) + lane; w <= (dhi - 1) >> 2; w += 32)
                merge_word<BLOCKED, MEM>(a, sX, sHJ, sVis, row, dv, dhv, dh, dT, dlo, dhi, w);
        }
    }
}

#ifndef FIRST_BIG_BPS
#define FIRST_BIG_BPS 4  // blocks per SM of k_first_big
#endif
constexpr int FW = 8;  // max words per lane of the warp kernel (J/4/32 <= 8)
constexpr int UW = 2;  // edges in flight per lane, rows of the warp kernel
#ifndef FIRST_UB
#define FIRST_UB 1
#endif
constexpr int UB = FIRST_UB;  // edges per lane per iteration in gather sweeps, rows of the block kernel (4 measured slower)

template <bool MEM>
__device__ __forceinline__ uint32_t start_word(const FirstArgs& a, const uint32_t* sHJ, uint32_t hu, uint32_t u, int w) {
    return MEM ? reinterpret_cast<const uint32_t*>(a.M)[(size_t)u * (a.J >> 2) + w] : init_word(hu, sHJ, w);
}

// final smem word vs its start value: write it back if it rose (the first sweep runs after
// k_init_registers wrote every row) and return the 4 change bits (one per simulation) of word w
__device__ __forceinline__ uint32_t finish_word(const FirstArgs& a, const uint32_t* row, uint32_t u, int w, uint32_t old,
                                                bool always_write) {
    uint32_t x = row[w];
    if (always_write || x != old) reinterpret_cast<uint32_t*>(a.M)[(size_t)u * (a.J >> 2) + w] = x;
    uint32_t eq = __vcmpeq4(x, old);
    return ((((~eq) & 0x01010101u) * 0x00204081u) >> 21) & 0xFu;
}


// A vertex with at most 32 out-edges: one edge per lane, and only the row words inside the edges'
// candidate windows are touched (marked in a per-warp bitmap, started from init / current values,
// merged, then compared and written back) instead of the whole J-register row.
template <bool CONST_T, bool BLOCKED, bool MEM>
__device__ __forceinline__ void first_small(const FirstArgs& a, const uint32_t* sX, const uint16_t* sS, const uint32_t* sHJ,
                                            const uint32_t* sVis, uint32_t* row, uint32_t* bm, uint32_t* scm, uint32_t u, bool have, uint2 f,
                                            uint32_t Tin, uint32_t& wcount) {
    const int lane = threadIdx.x & 31, J = a.J, W = J >> 5, NW = J >> 2, NB = (NW + 31) >> 5;
    uint32_t h = 0, T = 0, hv = 0, v = 0;
    int lo = 0, hi = 0;
    if (have && Tin) {
        T = Tin;
        h = f.y;
        v = f.x;
        edge_window(h, T, sX, sS, J, lo, hi);
        if (lo < hi) {
            wcount++;
            if (!MEM) hv = vhash(a, v);
        }
    }
    const uint32_t hu = MEM ? 0u : vhash(a, u);
    const int w0 = lo >> 2, w1 = lo < hi ? (hi - 1) >> 2 : w0 - 1;
    // MEM: the out-neighbour's first window word is loaded now, in flight with the row words below
    const uint32_t* rv = reinterpret_cast<const uint32_t*>(a.M) + (size_t)v * (J >> 2);
    const uint32_t pre = MEM && lo < hi ? rv[w0] : 0u, pre2 = MEM && w1 > w0 ? rv[w0 + 1] : 0u;
    if (lane < NB) bm[lane] = 0u;
    if (lane < W) scm[lane] = 0u;
    __syncwarp();
    for (int w = w0; w <= w1; ++w) atomicOr(&bm[w >> 5], 1u << (w & 31));
    for (int w = w0; w <= w1; ++w) row[w] = start_word<MEM>(a, sHJ, hu, u, w);  // same value from every writer
    __syncwarp();
    for (int w = w0; w <= w1; ++w) merge_word<BLOCKED, MEM>(a, sX, sHJ, sVis, row, v, hv, h, T, lo, hi, w, w - w0 < 2, w == w0 ? pre : pre2);
    __syncwarp();
    // every touched word is finished once, by the lane that clears its bitmap bit first; its change
    // nibble goes to the warp's change-mask words (word w >> 3 of the row's J/32)
    for (int w = w0; w <= w1; ++w) {
        const uint32_t bit = 1u << (w & 31);
        if (atomicAnd(&bm[w >> 5], ~bit) & bit) {
            const uint32_t nib = finish_word(a, row, u, w, start_word<MEM>(a, sHJ, hu, u, w), false);
            if (nib) atomicOr(&scm[w >> 3], nib << ((w & 7) << 2));
        }
    }
    __syncwarp();
    const uint32_t x = lane < W ? scm[lane] : 0u;
    if (x) a.cm_out[(size_t)u * W + lane] = x;  // the buffer starts zeroed
    const uint32_t chunks = __ballot_sync(IM_FULL, x != 0u);
    if (lane == 0 && chunks) a.bits_out[u] = chunks;
    __syncwarp();
}

// A row of at most 32 out-edges gathered by ONE lane (constant threshold, sparse windows): most rows of a
// skewed graph are this short (RMAT-24: 45% of the vertices have 1..32 out-edges, 10% of the edges), and a
// warp per such row leaves most lanes idle behind a fixed per-row cost.  The lane walks its row's edges and
// their window words alone and raises the registers of its own row in global memory (it is the row's only
// writer in a gather sweep), with the exact per-simulation change mask; no shared-memory row, no atomics.
template <bool BLOCKED, bool MEM>
__device__ __forceinline__ void first_thread(const FirstArgs& a, const uint32_t* sX, const uint16_t* sS, const uint32_t* sHJ,
                                             uint32_t u, int eb, int ee, uint32_t& wcount) {
    constexpr int TU = 2;  // edges per iteration: their records, then their window words of M_v / M_u, are loaded together
    const int J = a.J, W = J >> 5, NW = J >> 2;
    uint32_t* Mu = reinterpret_cast<uint32_t*>(a.M) + (size_t)u * NW;
    uint32_t* cmu = a.cm_out + (size_t)u * W;
    const uint32_t hu = MEM ? 0u : vhash(a, u);
    const uint32_t T = a.T0;
    uint32_t chunks = 0u;
    for (int e0 = eb; e0 < ee; e0 += TU) {
        uint2 f[TU];
#pragma unroll
        for (int k = 0; k < TU; k++) f[k] = e0 + k < ee ? ld_stream(&a.fwd[e0 + k]) : make_uint2(0u, 0u);
        int lo[TU], hi[TU];
        uint32_t mv[TU][2], mu[TU][2];
#pragma unroll
        for (int k = 0; k < TU; k++) {
            lo[k] = hi[k] = 0;
            mv[k][0] = mv[k][1] = mu[k][0] = mu[k][1] = 0u;
            if (e0 + k < ee) edge_window(f[k].y, T, sX, sS, J, lo[k], hi[k]);
            if (lo[k] < hi[k]) {
                wcount++;
                const int w0 = lo[k] >> 2, w1 = (hi[k] - 1) >> 2;
                if (MEM) {  // the first two window words of the out-neighbour and of the own row (possibly stale: re-read before a store)
                    const uint32_t* Mv = reinterpret_cast<const uint32_t*>(a.M) + (size_t)f[k].x * NW;
                    mv[k][0] = Mv[w0];
                    mu[k][0] = Mu[w0];
                    if (w1 > w0) {
                        mv[k][1] = Mv[w0 + 1];
                        mu[k][1] = Mu[w0 + 1];
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < TU; k++) {
            if (lo[k] >= hi[k]) continue;
            const uint32_t h = f[k].y;
            const uint32_t hv = MEM ? 0u : vhash(a, f[k].x);
            const int w0 = lo[k] >> 2, w1 = (hi[k] - 1) >> 2;
            for (int w = w0; w <= w1; ++w) {
                uint32_t live = live_word(sX, h, T, w);  // Eq. 5
                if (BLOCKED && live) live &= ~expand4((__ldg(&a.vis[(size_t)u * W + (w >> 3)]) >> ((w & 7) << 2)) & 0xFu);  // u in R_S[j] does not pull
                if (!live) continue;
                uint32_t val;
                if (MEM) {
                    const uint32_t pv = w == w0 ? mv[k][0] : mv[k][1], pu = w == w0 ? mu[k][0] : mu[k][1];
                    val = (w - w0 < 2 ? pv : reinterpret_cast<const uint32_t*>(a.M)[(size_t)f[k].x * NW + w]) & live;
                    if (w - w0 < 2 && __vmaxu4(pu, val) == pu) continue;  // registers only grow: no raise
                } else {
                    val = init_word(hv, sHJ, w) & live;
                    const uint32_t ci = init_word(hu, sHJ, w);
                    if (__vmaxu4(ci, val) == ci) continue;  // not above u's init values
                }
                const uint32_t cur = Mu[w];  // current value (an earlier edge of the row may have raised it)
                const uint32_t nw = __vmaxu4(cur, val);
                if (nw == cur) continue;
                Mu[w] = nw;
                const uint32_t eq = __vcmpeq4(nw, cur);
                const uint32_t nib = ((((~eq) & 0x01010101u) * 0x00204081u) >> 21) & 0xFu;
                cmu[w >> 3] |= nib << ((w & 7) << 2);  // the row's only writer; the buffer starts zeroed
                chunks |= 1u << (w >> 3);
            }
        }
    }
    if (chunks) a.bits_out[u] = chunks;
}

template <bool CONST_T, bool BLOCKED, bool MEM>
__global__ void __launch_bounds__(BLOCK, 5) k_first(FirstArgs a) {
    __shared__ __align__(16) uint32_t sX[1024];
    __shared__ uint16_t sS[4098];
    __shared__ __align__(16) uint32_t sHJ[1024];
    __shared__ uint32_t sRow[BLOCK / 32][256];
    __shared__ uint32_t sOldRow[BLOCK / 32][256];
    __shared__ uint32_t sVis[BLOCK / 32][32];
    __shared__ int sOff[BLOCK / 32][258];
    __shared__ uint32_t sBm[BLOCK / 32][8];
    __shared__ uint32_t sCm[BLOCK / 32][32];
    const int J = a.J, W = J >> 5, NW = J >> 2;
    for (int i = threadIdx.x; i < J; i += blockDim.x) {
        sX[i] = a.Xs[i];
        sHJ[i] = MEM ? 0u : murmur_word((uint32_t)a.perm[i], a.seedJ);
    }
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) sS[i] = a.s12[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t* row = sRow[wib];
    uint32_t* old = sOldRow[wib];
    uint32_t wcount = 0;
    int* off_w = sOff[wib];
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&a.ctr->batch, a.vb);
        base = __shfl_sync(IM_FULL, base, 0);
        if (base >= a.n) break;
        const int end = min(base + a.vb, a.n);
        for (int i = lane; i <= end - base; i += 32) off_w[i] = a.off[base + i];  // the batch's offsets, one coalesced read
        __syncwarp();
        const bool thr = CONST_T && a.thread_rows;
        if (thr) {  // rows of 1..32 out-edges, one per lane, in three degree classes (similar trip counts per warp)
            uint8_t* lst = reinterpret_cast<uint8_t*>(old);
            const int nv = end - base;
#pragma unroll 1
            for (int cls = 0; cls < 3; cls++) {
                const int dlo = cls == 0 ? 1 : cls == 1 ? 5 : 13, dhi = cls == 0 ? 4 : cls == 1 ? 12 : 32;
                int cnt = 0;
                for (int i0 = 0; i0 < nv; i0 += 32) {
                    const int i = i0 + lane;
                    const int d = i < nv ? off_w[i + 1] - off_w[i] : 0;
                    const bool in = d >= dlo && d <= dhi;
                    const uint32_t mk = __ballot_sync(IM_FULL, in);
                    if (in) lst[cnt + __popc(mk & ((1u << lane) - 1u))] = (uint8_t)i;
                    cnt += __popc(mk);
                }
                __syncwarp();
                for (int g = lane; g < cnt; g += 32) {
                    const int i = lst[g];
                    first_thread<BLOCKED, MEM>(a, sX, sS, sHJ, (uint32_t)(base + i), off_w[i], off_w[i + 1], wcount);
                }
                __syncwarp();
            }
        }
        // The rows left for the warp, in order: every row (then rows for k_first_big / empty rows are skipped
        // below), or with thread rows only those of 33..FIRST_BIG out-edges, found 32 vertices at a time by a
        // ballot (they are a few percent of a skewed graph's vertices).  The first 32 records of the next row
        // are prefetched while the current one is processed.
        const int nvb = end - base;
        int it_i = -1, it_i0 = -32;
        uint32_t it_mk = 0u;
        auto next_row = [&]() -> int {
            if (!thr) return ++it_i;
            while (!it_mk) {
                it_i0 += 32;
                if (it_i0 >= nvb) return nvb;
                const int i = it_i0 + lane;
                const int d = i < nvb ? off_w[i + 1] - off_w[i] : 0;
                it_mk = __ballot_sync(IM_FULL, d > 32 && d <= FIRST_BIG);
            }
            const int r = it_i0 + __ffs(it_mk) - 1;
            it_mk &= it_mk - 1;
            return r;
        };
        auto prefetch = [&](int i, uint2& f, uint32_t& T) {
            f = make_uint2(0, 0);
            T = 0;
            if (i >= nvb) return;
            const int eb1 = off_w[i], ee1 = off_w[i + 1];
            if (ee1 - eb1 <= FIRST_BIG && eb1 + lane < ee1) {
                f = ld_stream(&a.fwd[eb1 + lane]);
                T = CONST_T ? a.T0 : ld_stream(&a.fwdT[eb1 + lane]);
            }
        };
        uint2 nf;
        uint32_t nT;
        int cur_i = next_row();
        prefetch(cur_i, nf, nT);
        while (cur_i < nvb) {
            const int u = base + cur_i;
            const int eb = off_w[cur_i], ee = off_w[cur_i + 1];
            const uint2 cf = nf;
            const uint32_t cT = nT;
            cur_i = next_row();
            prefetch(cur_i, nf, nT);
            if (ee - eb > FIRST_BIG) continue;  // done by k_first_big
            if (ee == eb) {  // no out-edge: the row keeps its value (init rows and zeroed masks are written before)
                if (MEM) {
                    if (lane < W) a.cm_out[(size_t)u * W + lane] = 0u;
                    if (lane == 0) a.bits_out[u] = 0u;
                }
                continue;
            }
            // per-edge thresholds (weighted cascade): a row with any wide window takes the whole-row path
            const bool wide = !CONST_T && __any_sync(IM_FULL, cT && ((int64_t)a.J << thr_bits(cT)) > ((int64_t)DENSE_WIN << 31));
            if (ee - eb <= 32 && a.small_rows && !wide) {  // sparse path: touch only the window words
                if (BLOCKED && lane < W) sVis[wib][lane] = a.vis[(size_t)u * W + lane];
                __syncwarp();
                first_small<CONST_T, BLOCKED, MEM>(a, sX, sS, sHJ, sVis[wib], row, sBm[wib], sCm[wib], (uint32_t)u, eb + lane < ee, cf, cT,
                                                   wcount);
                continue;
            }
            const uint32_t hu = MEM ? 0u : vhash(a, (uint32_t)u);
            for (int w = lane; w < NW; w += 32) {
                uint32_t x = start_word<MEM>(a, sHJ, hu, (uint32_t)u, w);
                row[w] = x;
                old[w] = x;
            }
            if (BLOCKED && lane < W) sVis[wib][lane] = a.vis[(size_t)u * W + lane];
            __syncwarp();
            if (eb < ee) gather_rec<CONST_T, BLOCKED, MEM>(a, sX, sS, sHJ, sVis[wib], row, eb + lane < ee, cf, cT, wcount);
            for (int e0 = eb + 32; e0 < ee; e0 += 32 * (MEM ? UW : 1))  // from init values: ALU-bound, one edge per lane
                gather_multi<CONST_T, BLOCKED, MEM, MEM ? UW : 1>(a, sX, sS, sHJ, sVis[wib], row, e0, ee, 32, wcount);
            __syncwarp();
            uint32_t chunks = 0;
#pragma unroll
            for (int k = 0; k < FW; k++) {
                if (32 * k < NW) {  // warp-uniform
                    const int w = lane + 32 * k;
                    uint32_t nib = w < NW ? finish_word(a, row, (uint32_t)u, w, old[w], false) : 0u;
                    // change-mask word (w >> 3) = 4k + lane/8 from the nibbles of 8 consecutive lanes
                    uint32_t x = nib << ((lane & 7) << 2);
                    x |= __shfl_xor_sync(IM_FULL, x, 1);
                    x |= __shfl_xor_sync(IM_FULL, x, 2);
                    x |= __shfl_xor_sync(IM_FULL, x, 4);
                    if ((lane & 7) == 0 && w < NW) a.cm_out[(size_t)u * W + (w >> 3)] = x;
                    const uint32_t bl = __ballot_sync(IM_FULL, (lane & 7) == 0 && x != 0u);
#pragma unroll
                    for (int c = 0; c < 4; c++) chunks |= ((bl >> (8 * c)) & 1u) << (4 * k + c);
                }
            }
            if (lane == 0) a.bits_out[u] = chunks;
            __syncwarp();
        }
    }
    wcount = __reduce_add_sync(IM_FULL, wcount);
    if (lane == 0 && wcount) atomicAdd(&a.ctr->win_edges, (ull)wcount);
}

// global bytewise max of val into *p; returns the 4 change bits (one per register) this call raised
__device__ __forceinline__ uint32_t gmax4_raised(uint32_t* p, uint32_t val) {
    uint32_t cur = __ldcg(p), nw = __vmaxu4(cur, val);
    while (nw != cur) {
        const uint32_t prev = atomicCAS(p, cur, nw);
        if (prev == cur) {
            const uint32_t eq = __vcmpeq4(cur, nw);
            return ((((~eq) & 0x01010101u) * 0x00204081u) >> 21) & 0xFu;
        }
        cur = prev;
        nw = __vmaxu4(cur, val);
    }
    return 0u;
}

// Vertices with more than FIRST_BIG out-edges, in work units of <= FIRST_CHUNK edges (a 700k-edge hub of
// RMAT-24 is ~90 units instead of one block's serial tail): a block gathers its unit's edges into a
// shared-memory copy of row u started from the row's value (init or current), then max-merges the words
// it raised into the global row with a bytewise-max CAS; the change bits it raised go to u's change mask
// and chunk bits with atomicOr (the buffers start zeroed), so several units of one row compose.
template <bool CONST_T, bool BLOCKED, bool MEM>
__global__ void __launch_bounds__(BLOCK) k_first_big(FirstArgs a) {
    __shared__ __align__(16) uint32_t sX[1024];
    __shared__ uint16_t sS[4098];
    __shared__ __align__(16) uint32_t sHJ[1024];
    __shared__ uint32_t row[256];
    __shared__ uint32_t sOld[256];
    __shared__ uint32_t sVis[32];
    __shared__ uint32_t sMask[32];
    const int J = a.J, W = J >> 5, NW = J >> 2;
    for (int i = threadIdx.x; i < J; i += blockDim.x) {
        sX[i] = a.Xs[i];
        sHJ[i] = MEM ? 0u : murmur_word((uint32_t)a.perm[i], a.seedJ);
    }
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) sS[i] = a.s12[i];
    uint32_t wcount = 0;
    for (int bi = blockIdx.x; bi < a.n_big; bi += gridDim.x) {
        const int4 U = a.big_units[bi];
        const uint32_t u = (uint32_t)U.x;
        const int eb = U.y, ee = U.z;
        __syncthreads();
        const uint32_t hu = MEM ? 0u : vhash(a, u);
        for (int w = threadIdx.x; w < NW; w += blockDim.x) {
            uint32_t x = MEM ? __ldcg(reinterpret_cast<const uint32_t*>(a.M) + (size_t)u * (J >> 2) + w) : init_word(hu, sHJ, w);
            row[w] = x;
            sOld[w] = x;
        }
        if (threadIdx.x < W) {
            sMask[threadIdx.x] = 0u;
            if (BLOCKED) sVis[threadIdx.x] = a.vis[(size_t)u * W + threadIdx.x];
        }
        __syncthreads();
        for (int e0 = eb + (threadIdx.x & ~31); e0 < ee; e0 += (MEM ? UB : 1) * blockDim.x)  // warp-uniform trip count
            gather_multi<CONST_T, BLOCKED, MEM, MEM ? UB : 1>(a, sX, sS, sHJ, sVis, row, e0, ee, blockDim.x, wcount);
        __syncthreads();
        for (int w = threadIdx.x; w < NW; w += blockDim.x) {
            const uint32_t x = row[w];
            if (x != sOld[w]) {
                const uint32_t nib = gmax4_raised(reinterpret_cast<uint32_t*>(a.M) + (size_t)u * (J >> 2) + w, x);
                if (nib) atomicOr(&sMask[w >> 3], nib << ((w & 7) << 2));
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const uint32_t m = threadIdx.x < W ? sMask[threadIdx.x] : 0u;
            if (m) atomicOr(&a.cm_out[(size_t)u * W + threadIdx.x], m);
            const uint32_t chunks = __ballot_sync(IM_FULL, m != 0u);
            if (threadIdx.x == 0 && chunks) atomicOr(&a.bits_out[u], chunks);
        }
    }
    const int lane = threadIdx.x & 31;
    wcount = __reduce_add_sync(IM_FULL, wcount);
    if (lane == 0 && wcount) atomicAdd(&a.ctr->win_edges, (ull)wcount);
}

// In a gather sweep from memory (in place), the long rows go first: their vertices are the hubs most
// other rows read, so the rest of the sweep already sees their new values (Gauss-Seidel order).
template <bool C, bool B, bool MEM>
static cudaError_t first_inst(Ctx& c, const FirstArgs& a) {
    cudaError_t e;
    const int gb = a.n_big < c.num_sms * FIRST_BIG_BPS ? a.n_big : c.num_sms * FIRST_BIG_BPS;
    if (MEM && a.n_big) {
        k_first_big<C, B, MEM><<<gb, BLOCK, 0, c.stream>>>(a);
        if ((e = LAUNCHED(c))) return e;
    }
    k_first<C, B, MEM><<<c.max_blocks_first, BLOCK, 0, c.stream>>>(a);
    if ((e = LAUNCHED(c)) || a.n_big == 0 || MEM) return e;
    k_first_big<C, B, MEM><<<gb, BLOCK, 0, c.stream>>>(a);
    return LAUNCHED(c);
}

cudaError_t launch_first(Ctx& c, uint32_t* cm_out, uint32_t* bits_out, IterCounters* ctr, bool blocked, bool from_memory) {
    FirstArgs a;
    a.n = c.n;
    a.J = c.J;
    a.seedV = c.seedV;
    a.seedJ = c.seedJ;
    a.off = c.off;
    a.fwd = c.fwd;
    a.fwdT = c.fwdT;
    a.T0 = c.T0;
    a.Xs = c.Xs;
    a.s12 = c.s12;
    a.perm = c.permd;
    a.M = c.M;
    a.vis = c.vis;
    a.cm_out = cm_out;
    a.bits_out = bits_out;
    a.ctr = ctr;
    a.big_units = c.fbig;
    a.n_big = c.n_fbig;
    // nominal candidate window of a constant threshold: J * 2^B0 / 2^31 simulations
    a.small_rows = !c.constT || ((int64_t)c.J << c.B0) <= ((int64_t)DENSE_WIN << 31);
    a.thread_rows = c.constT && a.small_rows && c.thread_rows;
    {   // a dependent chain of loads per vertex: spread small graphs over every resident warp
        const int64_t warps = (int64_t)c.max_blocks_first * (BLOCK / 32);
        a.vb = (int)std::min<int64_t>(256, std::max<int64_t>(1, c.n / warps));
    }
    if (from_memory) {
        if (c.constT) return blocked ? first_inst<true, true, true>(c, a) : first_inst<true, false, true>(c, a);
        return blocked ? first_inst<false, true, true>(c, a) : first_inst<false, false, true>(c, a);
    }
    if (c.constT) return blocked ? first_inst<true, true, false>(c, a) : first_inst<true, false, false>(c, a);
    return blocked ? first_inst<false, true, false>(c, a) : first_inst<false, false, false>(c, a);
}

// work units of the rows with more than FIRST_BIG out-edges (once per graph): pass 1 counts them
// (units == nullptr), pass 2 writes {u, eb, ee} for each chunk of <= FIRST_CHUNK edges
__global__ void k_list_big_rows(int32_t n, const int32_t* __restrict__ off, int4* __restrict__ units, int* count) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += stride) {
        const int eb = off[u], ee = off[u + 1];
        if (ee - eb <= FIRST_BIG) continue;
        const int nch = (ee - eb + FIRST_CHUNK - 1) / FIRST_CHUNK;
        const int p = atomicAdd(count, nch);
        if (units)
            for (int k = 0; k < nch; k++) units[p + k] = make_int4((int)u, eb + k * FIRST_CHUNK, min(eb + (k + 1) * FIRST_CHUNK, ee), 0);
    }
}

cudaError_t launch_list_big_rows(Ctx& c, int4* units, int* count) {
    k_list_big_rows<<<grid_for(c, c.n), BLOCK, 0, c.stream>>>(c.n, c.off, units, count);
    return LAUNCHED(c);
}

int setup_first(int J, int* blocks_per_sm) {
    (void)J;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_first<true, true, false>, BLOCK, 0);
}

}  // namespace im
