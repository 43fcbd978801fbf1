// im_sweep.cu -- Simulate (Alg. 2) on sm_100a: the sweep kernel and the
// per-sweep frontier compaction.  DESIGN.md "Kernels / k_sweep".
//
// One sweep is an edge-parallel, in-place pass over the in-edges (u,v) of every vertex v whose
// registers changed in the previous sweep (all vertices in sweep 1).  For such an edge and every
// simulation j with (X_j xor h_uv) < T_uv and u not in R_S[j], M_u[j] <- max(M_u[j], M_v[j])
// (Alg. 2 'update', pull direction, reading R9).  Alg. 2 processes u in Gamma^-(L) with all its
// out-edges; the edges into unchanged vertices are no-ops (u already holds their values), so they
// are skipped, and edges whose candidate window misses every 32-simulation chunk of v that changed
// are skipped too.  The fixpoint is unique, hence equal to the oracle's synchronous schedule.
//
// Simulations are stored in ascending-salt order, so the simulations where an edge can be live
// form one contiguous window [lo, hi) (im_device.cuh).  A lane owns one edge; it touches only the
// 8-byte words of M_u / M_v inside the window and merges with a bytewise-max CAS.  Windows wider
// than DENSE_WIN simulations are walked by the whole warp.  Two edges per lane are kept in flight.
#include "im_device.cuh"
#include "im_internal.h"

namespace im {

struct SweepArgs {
    const int4* items;
    int n_items;
    IterCounters* ctr;
    const uint2* rev;
    const uint32_t* revT;
    uint32_t T0;
    const uint32_t* Xs;
    const uint16_t* s12;
    int J;
    ull* M64;
    const uint32_t* vis;
    const uint32_t* bits_in;
    uint32_t* bits_out;
};

__device__ __forceinline__ ull vmax8(ull a, ull b) {
    return (ull)__vmaxu4((uint32_t)a, (uint32_t)b) | ((ull)__vmaxu4((uint32_t)(a >> 32), (uint32_t)(b >> 32)) << 32);
}
__device__ __forceinline__ ull expand8(uint32_t b) { return (ull)expand4(b & 0xFu) | ((ull)expand4(b >> 4) << 32); }

// byte mask of the simulations of 8-byte word w that are live for (h, T) inside [lo, hi), minus blocked ones
template <bool BLOCKED>
__device__ __forceinline__ ull live8(const SweepArgs& a, const uint32_t* sX, uint32_t u, int w, uint32_t h, uint32_t T,
                                    int lo, int hi) {
    ull live = 0;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        int i = 8 * w + b;
        bool ok = (i >= lo) & (i < hi) & ((sX[i] ^ h) < T);
        live |= ok ? (0xFFull << (8 * b)) : 0ull;
    }
    if (BLOCKED && live) {
        uint32_t vb = (a.vis[(size_t)u * (a.J >> 5) + (w >> 2)] >> ((w & 3) << 3)) & 0xFFu;
        live &= ~expand8(vb);
    }
    return live;
}

// bytewise max of `cand` into *p given a first observed value; returns true if this thread raised a register
__device__ __forceinline__ bool vmax_cas8(ull* p, ull cur, ull cand) {
    ull nw = vmax8(cur, cand);
    while (nw != cur) {
        ull prev = atomicCAS(p, cur, nw);
        if (prev == cur) return true;
        cur = prev;
        nw = vmax8(cur, cand);
    }
    return false;
}

template <bool BLOCKED>
__device__ __forceinline__ uint32_t pull_word8(const SweepArgs& a, const uint32_t* sX, uint32_t u, uint32_t v, int w,
                                               uint32_t h, uint32_t T, int lo, int hi) {
    ull live = live8<BLOCKED>(a, sX, u, w, h, T, lo, hi);
    if (!live) return 0u;
    const size_t J8 = (size_t)(a.J >> 3);
    ull cand = a.M64[v * J8 + w] & live;
    if (!cand) return 0u;
    ull* p = &a.M64[u * J8 + w];
    return vmax_cas8(p, __ldcg(p), cand) ? (1u << (w >> 2)) : 0u;
}

constexpr int NS = 2;  // edges in flight per lane

template <bool CONST_T, bool BLOCKED, bool FILTER>
__global__ void __launch_bounds__(BLOCK, 4) k_sweep(SweepArgs a) {
    __shared__ uint32_t sX[1024];
    __shared__ uint16_t sS[4098];
    __shared__ int sSlot[BLOCK / 32][32];
    for (int i = threadIdx.x; i < a.J; i += blockDim.x) sX[i] = a.Xs[i];
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) sS[i] = a.s12[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int J = a.J;
    const size_t J8 = (size_t)(J >> 3);
    uint32_t wcount = 0;

    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&a.ctr->batch, 32);
        base = __shfl_sync(IM_FULL, base, 0);
        if (base >= a.n_items) break;
        int it = base + lane;
        int v = 0, eb = 0, cnt = 0;
        uint32_t vbits = IM_FULL;
        if (it < a.n_items) {
            int4 I = a.items[it];
            v = I.x;
            eb = I.y;
            cnt = I.z - I.y;
            if (FILTER) vbits = a.bits_in[v];
        }
        int incl = warp_incl_scan(cnt, lane);
        const int total = __shfl_sync(IM_FULL, incl, 31);
        const int start = incl - cnt;
        int carry = 0;
        for (int e0 = 0; e0 < total; e0 += 32 * NS) {
            uint32_t u[NS], h[NS], T[NS], vv[NS], ob[NS];
            int lo[NS], hi[NS];
            // owner item of each edge slot: the last non-empty item starting at or before it
#pragma unroll
            for (int s = 0; s < NS; s++) {
                const int w0 = e0 + 32 * s;
                int owner = carry;
                if (w0 < total) {  // warp-uniform
                    bool starts = cnt > 0 && start >= w0 && start < w0 + 32;
                    if (starts) sSlot[wib][start - w0] = lane;
                    uint32_t smask = __reduce_or_sync(IM_FULL, starts ? (1u << (start - w0)) : 0u);
                    __syncwarp();
                    uint32_t below = smask & ((2u << lane) - 1u);
                    if (below) owner = sSlot[wib][31 - __clz(below)];
                    __syncwarp();
                    carry = __shfl_sync(IM_FULL, owner, 31);
                }
                vv[s] = (uint32_t)__shfl_sync(IM_FULL, v, owner);
                int oeb = __shfl_sync(IM_FULL, eb, owner);
                int ost = __shfl_sync(IM_FULL, start, owner);
                ob[s] = __shfl_sync(IM_FULL, vbits, owner);
                int idx = w0 + lane;
                T[s] = 0u;
                u[s] = h[s] = 0u;
                if (idx < total) {
                    int e = oeb + (idx - ost);
                    uint2 r = a.rev[e];
                    u[s] = r.x;
                    h[s] = r.y;
                    T[s] = CONST_T ? a.T0 : a.revT[e];
                }
            }
            bool sparse[NS];
            ull mv[NS], mu[NS];
#pragma unroll
            for (int s = 0; s < NS; s++) {
                lo[s] = hi[s] = 0;
                if (T[s]) {
                    edge_window(h[s], T[s], sX, sS, J, lo[s], hi[s]);
                    if (FILTER && lo[s] < hi[s] && !(ob[s] & bit_range(lo[s] >> 5, (hi[s] - 1) >> 5))) hi[s] = lo[s];
                }
                sparse[s] = lo[s] < hi[s] && hi[s] - lo[s] <= DENSE_WIN;
                if (sparse[s]) {  // first word of the window: both loads in flight before any use
                    int w = lo[s] >> 3;
                    mv[s] = a.M64[vv[s] * J8 + w];
                    mu[s] = __ldcg(&a.M64[u[s] * J8 + w]);
                }
            }
            ull cand[NS], nw[NS], prev[NS];
            bool need[NS];
#pragma unroll
            for (int s = 0; s < NS; s++) {
                need[s] = false;
                if (sparse[s]) {
                    int w = lo[s] >> 3;
                    cand[s] = mv[s] & live8<BLOCKED>(a, sX, u[s], w, h[s], T[s], lo[s], hi[s]);
                    nw[s] = vmax8(mu[s], cand[s]);
                    need[s] = nw[s] != mu[s];
                }
            }
#pragma unroll
            for (int s = 0; s < NS; s++)  // both CASes issued before either result is used
                if (need[s]) prev[s] = atomicCAS(&a.M64[u[s] * J8 + (lo[s] >> 3)], mu[s], nw[s]);
            uint32_t chg[NS];
#pragma unroll
            for (int s = 0; s < NS; s++) {
                chg[s] = 0u;
                if (need[s]) {
                    int w = lo[s] >> 3;
                    bool up = prev[s] == mu[s] || vmax_cas8(&a.M64[u[s] * J8 + w], prev[s], cand[s]);
                    if (up) chg[s] = 1u << (w >> 2);
                }
                if (sparse[s])  // remaining words of a multi-word window
                    for (int w = (lo[s] >> 3) + 1; w <= (hi[s] - 1) >> 3; ++w)
                        chg[s] |= pull_word8<BLOCKED>(a, sX, u[s], vv[s], w, h[s], T[s], lo[s], hi[s]);
            }
            // wide windows (w close to 1, weighted cascade): the whole warp walks the window
#pragma unroll
            for (int s = 0; s < NS; s++) {
                uint32_t dmask = __ballot_sync(IM_FULL, hi[s] - lo[s] > DENSE_WIN);
                wcount += __popc(__ballot_sync(IM_FULL, lo[s] < hi[s]));
                while (dmask) {
                    int l = __ffs(dmask) - 1;
                    dmask &= dmask - 1;
                    uint32_t du = __shfl_sync(IM_FULL, u[s], l), dh = __shfl_sync(IM_FULL, h[s], l);
                    uint32_t dT = __shfl_sync(IM_FULL, T[s], l), dv = __shfl_sync(IM_FULL, vv[s], l);
                    int dlo = __shfl_sync(IM_FULL, lo[s], l), dhi = __shfl_sync(IM_FULL, hi[s], l);
                    uint32_t c = 0;
                    for (int w = (dlo >> 3) + lane; w <= (dhi - 1) >> 3; w += 32) c |= pull_word8<BLOCKED>(a, sX, du, dv, w, dh, dT, dlo, dhi);
                    c = __reduce_or_sync(IM_FULL, c);
                    if (lane == l) chg[s] |= c;
                }
            }
            // record which 32-simulation chunks of u rose (fire-and-forget; the compaction builds the next frontier)
#pragma unroll
            for (int s = 0; s < NS; s++)
                if (chg[s]) atomicOr(&a.bits_out[u[s]], chg[s]);
        }
    }
    if (lane == 0 && wcount) atomicAdd(&a.ctr->win_edges, (ull)wcount);
}

// Next frontier: every vertex whose change bits are set.  Its in-edges whose candidate window can
// meet a changed 32-simulation chunk are emitted as work items (<= 4 hash-sorted slices of its
// in-edge row when every edge has the same threshold, the whole row otherwise); the other bit
// buffer is cleared for the following sweep.
__global__ void k_compact(int32_t n, int J, int B, bool sorted, const uint32_t* __restrict__ Xs,
                          const uint32_t* __restrict__ bits_new, uint32_t* __restrict__ bits_clear,
                          const int32_t* __restrict__ roff, const uint2* __restrict__ rev, int4* __restrict__ items,
                          IterCounters* ctr) {
    const int lane = threadIdx.x & 31;
    const int NC = J >> 5, NQ = NC < 4 ? NC : 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        int64_t v = base + threadIdx.x;
        bool in = v < n;
        uint32_t b = in ? bits_new[v] : 0u;
        if (in && bits_clear && bits_clear[v]) bits_clear[v] = 0u;
        int eb[4], ee[4], k = 0, ns = 0, es = 0;
        if (b) {
            int rb = roff[v], re = roff[v + 1];
            if (sorted) {
                int sa[4], sb[4];
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    sa[q] = sb[q] = -1;
                    if (q < NQ) {
                        uint32_t qb = b & bit_range(q * NC / NQ, (q + 1) * NC / NQ - 1);
                        if (qb) {
                            sa[q] = 32 * (__ffs(qb) - 1);
                            sb[q] = 32 * (31 - __clz(qb)) + 31;
                        }
                    }
                }
                k = slices_for(rev, rb, re, Xs, B, sa, sb, eb, ee);
            } else if (rb < re) {
                eb[0] = rb;
                ee[0] = re;
                k = 1;
            }
#pragma unroll
            for (int i = 0; i < 4; i++)
                if (i < k) {
                    ns += (ee[i] - eb[i] + SEG - 1) / SEG;
                    es += ee[i] - eb[i];
                }
        }
        uint32_t fmask = __ballot_sync(IM_FULL, b != 0u);
        if (!fmask) continue;
        int ninc = warp_incl_scan(ns, lane);
        int ntot = __shfl_sync(IM_FULL, ninc, 31);
        long long esum = es;
#pragma unroll
        for (int o = 16; o; o >>= 1) esum += __shfl_xor_sync(IM_FULL, esum, o);
        int pos = 0;
        if (lane == 31) {
            if (ntot) pos = atomicAdd(&ctr->next_items, ntot);
            atomicAdd(&ctr->changed, __popc(fmask));
            if (esum) atomicAdd(&ctr->next_edges, (ull)esum);
        }
        pos = __shfl_sync(IM_FULL, pos, 31);
        int p = pos + ninc - ns;
#pragma unroll
        for (int i = 0; i < 4; i++)
            if (i < k)
                for (int s0 = eb[i]; s0 < ee[i]; s0 += SEG) items[p++] = make_int4((int)v, s0, min(s0 + SEG, ee[i]), 0);
    }
}

template <bool C, bool B, bool F>
static void sweep_inst(int grid, cudaStream_t s, const SweepArgs& a) {
    k_sweep<C, B, F><<<grid, BLOCK, 0, s>>>(a);
}

cudaError_t launch_sweep(Ctx& c, const int4* items, int n_items, const uint32_t* bits_in, uint32_t* bits_out,
                         IterCounters* ctr, bool blocked) {
    SweepArgs a;
    a.items = items;
    a.n_items = n_items;
    a.ctr = ctr;
    a.rev = c.rev;
    a.revT = c.revT;
    a.T0 = c.T0;
    a.Xs = c.Xs;
    a.s12 = c.s12;
    a.J = c.J;
    a.M64 = reinterpret_cast<ull*>(c.M);
    a.vis = c.vis;
    a.bits_in = bits_in;
    a.bits_out = bits_out;
    int64_t want = ((int64_t)n_items + 32 * (BLOCK / 32) - 1) / (32 * (BLOCK / 32));
    int grid = (int)(want < 1 ? 1 : (want > c.max_blocks_sweep ? c.max_blocks_sweep : want));
    const bool ct = c.constT, f = bits_in != nullptr;
    if (!f) {
        if (ct) { if (blocked) sweep_inst<true, true, false>(grid, c.stream, a); else sweep_inst<true, false, false>(grid, c.stream, a); }
        else { if (blocked) sweep_inst<false, true, false>(grid, c.stream, a); else sweep_inst<false, false, false>(grid, c.stream, a); }
    } else {
        if (ct) { if (blocked) sweep_inst<true, true, true>(grid, c.stream, a); else sweep_inst<true, false, true>(grid, c.stream, a); }
        else { if (blocked) sweep_inst<false, true, true>(grid, c.stream, a); else sweep_inst<false, false, true>(grid, c.stream, a); }
    }
    return LAUNCHED(c);
}

cudaError_t launch_compact(Ctx& c, const uint32_t* bits_new, uint32_t* bits_clear, int4* items_out, IterCounters* ctr) {
    k_compact<<<grid_for(c, c.n), BLOCK, 0, c.stream>>>(c.n, c.J, c.B0, c.sorted_h, c.Xs, bits_new, bits_clear, c.roff,
                                                        c.rev, items_out, ctr);
    return LAUNCHED(c);
}

int occupancy_sweep(int* blocks_per_sm) {
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_sweep<true, true, true>, BLOCK, 0);
}

}  // namespace im
