// im_sweep.cu -- Simulate (Alg. 2) on sm_100a: the sweep kernel and the
// per-sweep frontier compaction.  DESIGN.md §6 "k_sweep".
//
// One sweep is an edge-parallel, in-place pass over the in-edges (u,v) of every vertex v whose
// registers changed in the previous sweep (all vertices in sweep 1).  For such an edge and every
// simulation j with (X_j xor h_uv) < T_uv and u not in R_S[j], M_u[j] <- max(M_u[j], M_v[j])
// (Alg. 2 'update', pull direction, reading R9).  Alg. 2 processes u in Gamma^-(L) with all its
// out-edges; the edges into unchanged vertices are no-ops (u already holds their values) and so are
// the simulations in which v did not change, so an edge is only worked on when its candidate window
// holds a simulation in which v changed (exact per-simulation change masks).  The fixpoint is
// unique, hence equal to the oracle's synchronous schedule.
//
// Simulations are stored in ascending-salt order, so the simulations where an edge can be live
// form one contiguous window [lo, hi) (im_device.cuh).  A lane owns one edge; it touches only the
// 8-byte words of M_u / M_v inside the window and merges with a bytewise-max CAS.  Windows wider
// than DENSE_WIN simulations are walked by the whole warp.  Two edges per lane are kept in flight.
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>

#include "im_device.cuh"
#include "im_internal.h"

namespace cg = cooperative_groups;

namespace im {
#ifndef IM_NS
#define IM_NS 2
#endif
#ifndef IM_LB4
#define IM_LB4 1  // window live bits by aligned 16-byte salt words (0: one simulation at a time)
#endif
#ifndef SWEEP_MINB
#define SWEEP_MINB 4  // resident blocks per SM k_sweep is compiled for
#endif

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
    ull* M64;                // registers written (M_u, bytewise-max CAS)
    const ull* Mr64;         // registers read (M_v): == M64 (in place), or the pre-sweep copy (synchronous sweeps, R22)
    const uint32_t* vis;
    const uint32_t* cm_in;   // per-simulation change mask of the previous sweep, n x J/32 words (FILTER)
    uint32_t* cm_out;        // this sweep's per-simulation change mask
    uint32_t* bits_out;      // this sweep's per-vertex 32-simulation-chunk summary
    int ipw;                 // items per warp batch (<= 32; fewer when the sweep is small, to spread it over the SMs)
    const IterCounters* nin; // non-null: n_items = nin->next_items on the device (pipelined sweeps), ipw derived here
    int warps_max;           // resident warps of the grid (for the device-side ipw)
};

__device__ __forceinline__ ull vmax8(ull a, ull b) {
    return (ull)__vmaxu4((uint32_t)a, (uint32_t)b) | ((ull)__vmaxu4((uint32_t)(a >> 32), (uint32_t)(b >> 32)) << 32);
}
__device__ __forceinline__ ull expand8(uint32_t b) { return (ull)expand4(b & 0xFu) | ((ull)expand4(b >> 4) << 32); }
// one bit per byte that differs between a and b
__device__ __forceinline__ uint32_t diff_bits8(ull a, ull b) {
    uint32_t lo = ~__vcmpeq4((uint32_t)a, (uint32_t)b) & 0x01010101u, hi = ~__vcmpeq4((uint32_t)(a >> 32), (uint32_t)(b >> 32)) & 0x01010101u;
    return (((lo * 0x00204081u) >> 21) & 0xFu) | ((((hi * 0x00204081u) >> 21) & 0xFu) << 4);
}

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

// live8 from the window's live bits (same byte mask as live8)
template <bool BLOCKED>
__device__ __forceinline__ ull live8_bits(const SweepArgs& a, uint32_t u, int w, uint32_t lb, int lo) {
    ull live = expand8(bits_at(lb, lo, 8 * w, 8));
    if (BLOCKED && live) {
        uint32_t vb = (a.vis[(size_t)u * (a.J >> 5) + (w >> 2)] >> ((w & 3) << 3)) & 0xFFu;
        live &= ~expand8(vb);
    }
    return live;
}
// v's previous-sweep change bits over [lo, hi), aligned like window_live_bits
__device__ __forceinline__ uint32_t window_changed_bits(const uint32_t* __restrict__ cm, uint32_t v, int W, int lo, int hi) {
    const uint32_t* row = cm + (size_t)v * W;
    const int w0 = lo >> 5, w1 = (hi - 1) >> 5;
    const uint32_t m0 = __ldg(&row[w0]), m1 = w1 != w0 ? __ldg(&row[w1]) : 0u;
    const uint32_t x = (uint32_t)((((ull)m1 << 32) | m0) >> (lo & 31));
    const int len = hi - lo;
    return len >= 32 ? x : (x & ((1u << len) - 1u));
}

// bytewise max of `cand` into *p starting from an observed value `cur`; returns the bits of the
// registers this thread raised (0 if none: someone else already holds values >= cand)
__device__ __forceinline__ uint32_t vmax_cas8(ull* p, ull cur, ull cand) {
    ull nw = vmax8(cur, cand);
    while (nw != cur) {
        ull prev = atomicCAS(p, cur, nw);
        if (prev == cur) return diff_bits8(cur, nw);
        cur = prev;
        nw = vmax8(cur, cand);
    }
    return 0u;
}

// record raised registers of word w of u: per-simulation mask word + returns the chunk bit
__device__ __forceinline__ uint32_t record8(const SweepArgs& a, uint32_t u, int w, uint32_t raised) {
    if (!raised) return 0u;
    atomicOr(&a.cm_out[(size_t)u * (a.J >> 5) + (w >> 2)], raised << ((w & 3) << 3));
    return 1u << (w >> 2);
}

template <bool BLOCKED>
__device__ __forceinline__ uint32_t pull_word8_bits(const SweepArgs& a, uint32_t u, uint32_t v, int w, uint32_t lb, int lo) {
    ull live = live8_bits<BLOCKED>(a, u, w, lb, lo);
    if (!live) return 0u;
    const size_t J8 = (size_t)(a.J >> 3);
    ull cand = a.Mr64[v * J8 + w] & live;
    if (!cand) return 0u;
    ull* p = &a.M64[u * J8 + w];
    return record8(a, u, w, vmax_cas8(p, __ldcg(p), cand));
}

template <bool BLOCKED, bool FILTER = false>
__device__ __forceinline__ uint32_t pull_word8(const SweepArgs& a, const uint32_t* sX, uint32_t u, uint32_t v, int w,
                                               uint32_t h, uint32_t T, int lo, int hi) {
    ull live;
    if (FILTER) {  // only the simulations of word w in which v changed last sweep can raise M_u: test those
        uint32_t cand = (__ldg(&a.cm_in[(size_t)v * (a.J >> 5) + (w >> 2)]) >> ((w & 3) << 3)) & 0xFFu;
        live = 0;
        for (; cand; cand &= cand - 1) {
            const int b = __ffs(cand) - 1, i = 8 * w + b;
            if (i >= lo && i < hi && (sX[i] ^ h) < T) live |= 0xFFull << (8 * b);
        }
        if (BLOCKED && live) {
            const uint32_t vb = (a.vis[(size_t)u * (a.J >> 5) + (w >> 2)] >> ((w & 3) << 3)) & 0xFFu;
            live &= ~expand8(vb);
        }
    } else {
        live = live8<BLOCKED>(a, sX, u, w, h, T, lo, hi);
    }
    if (!live) return 0u;
    const size_t J8 = (size_t)(a.J >> 3);
    ull cand = a.Mr64[v * J8 + w] & live;
    if (!cand) return 0u;
    ull* p = &a.M64[u * J8 + w];
    return record8(a, u, w, vmax_cas8(p, __ldcg(p), cand));
}

// does v's previous-sweep change mask hold a simulation of [lo, hi)?
__device__ __forceinline__ bool window_changed(const uint32_t* __restrict__ cm, uint32_t v, int W, int lo, int hi) {
    const uint32_t* row = cm + (size_t)v * W;
    int w0 = lo >> 5, w1 = (hi - 1) >> 5;
    for (int w = w0; w <= w1; ++w) {
        uint32_t m = __ldg(&row[w]);
        int a = w == w0 ? (lo & 31) : 0, b = w == w1 ? ((hi - 1) & 31) : 31;
        if (m & bit_range(a, b)) return true;
    }
    return false;
}

// does v's previous-sweep change mask hold a simulation of [lo, hi) (<= DENSE_WIN wide, so at most two
// mask words) in which the edge is live?  Only those simulations can raise M_u (Alg. 2:
// a simulation in which v did not change was already pulled, a dead one is never pulled).
__device__ __forceinline__ bool live_changed(const uint32_t* __restrict__ cm, uint32_t v, int W, const uint32_t* sX, uint32_t h,
                                             uint32_t T, int lo, int hi) {
    const uint32_t* row = cm + (size_t)v * W;
    const int w0 = lo >> 5, w1 = (hi - 1) >> 5;
    const uint32_t m0 = __ldg(&row[w0]), m1 = w1 != w0 ? __ldg(&row[w1]) : 0u;
    if (!(m0 | m1)) return false;
    for (int i = lo; i < hi; ++i) {
        const uint32_t m = (i >> 5) == w0 ? m0 : m1;
        if (((m >> (i & 31)) & 1u) && (sX[i] ^ h) < T) return true;
    }
    return false;
}

constexpr int NS = IM_NS;  // edges in flight per lane

template <bool CONST_T, bool BLOCKED, bool FILTER>
__global__ void __launch_bounds__(BLOCK, SWEEP_MINB) k_sweep(SweepArgs a) {
    __shared__ __align__(16) uint32_t sX[1024];
    __shared__ uint16_t sS[4098];
    __shared__ int sSlot[BLOCK / 32][32];
    if (a.nin) {  // item count of the previous compaction, read on the device (no host round trip)
        a.n_items = a.nin->next_items;
        a.ipw = min(32, max(1, a.n_items / a.warps_max));
        // blocks past the work exit before filling shared memory (the batch cursor hands out all items anyway)
        if (a.n_items == 0 || (blockIdx.x > 0 && (int64_t)blockIdx.x * (BLOCK / 32) * a.ipw >= a.n_items)) return;
    }
    for (int i = threadIdx.x; i < a.J; i += blockDim.x) sX[i] = a.Xs[i];
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) sS[i] = a.s12[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int J = a.J, W = J >> 5;
    const size_t J8 = (size_t)(J >> 3);
    uint32_t wcount = 0;

    int base = 0, left = 0;  // 128-item grabs (4 batches of 32) keep the cursor atomic off the critical path
    for (;;) {
        if (left == 0) {
            if (lane == 0) base = atomicAdd(&a.ctr->batch, 4 * a.ipw);
            base = __shfl_sync(IM_FULL, base, 0);
            left = 4;
        } else {
            base += a.ipw;
        }
        --left;
        if (base >= a.n_items) break;
        int it = base + lane;
        int v = 0, eb = 0, cnt = 0;
        if (lane < a.ipw && it < a.n_items) {
            int4 I = ld_stream(&a.items[it]);
            v = I.x;
            eb = I.y;
            cnt = I.z - I.y;
        }
        int incl = warp_incl_scan(cnt, lane);
        const int total = __shfl_sync(IM_FULL, incl, 31);
        const int start = incl - cnt;
        int carry = 0;
        for (int e0 = 0; e0 < total; e0 += 32 * NS) {
            uint32_t u[NS], h[NS], T[NS], vv[NS];
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
                int idx = w0 + lane;
                T[s] = 0u;
                u[s] = h[s] = 0u;
                if (idx < total) {
                    int e = oeb + (idx - ost);
                    uint2 r = ld_stream(&a.rev[e]);
                    u[s] = r.x;
                    h[s] = r.y;
                    T[s] = CONST_T ? a.T0 : ld_stream(&a.revT[e]);
                }
            }
            bool sparse[NS];
            ull mv[NS], mu[NS];
            uint32_t lb[NS];  // sparse windows: live (and, filtered, changed-at-v) simulations, bit k = lo + k
#pragma unroll
            for (int s = 0; s < NS; s++) {
                lo[s] = hi[s] = 0;
                lb[s] = 0u;
                if (T[s]) {
                    edge_window(h[s], T[s], sX, sS, J, lo[s], hi[s]);
                    if (lo[s] < hi[s] && hi[s] - lo[s] <= DENSE_WIN) {
#if IM_LB4
                        lb[s] = window_live_bits4(sX, h[s], T[s], lo[s], hi[s]);
#else
                        lb[s] = window_live_bits(sX, h[s], T[s], lo[s], hi[s]);
#endif
                        if (FILTER) lb[s] &= window_changed_bits(a.cm_in, vv[s], W, lo[s], hi[s]);
                        narrow_window(lb[s], lo[s], hi[s]);  // to the live (changed-at-v) simulations; empty if none
                    } else if (FILTER && lo[s] < hi[s] && !window_changed(a.cm_in, vv[s], W, lo[s], hi[s])) {
                        hi[s] = lo[s];
                    }
                }
                sparse[s] = lo[s] < hi[s] && hi[s] - lo[s] <= DENSE_WIN;
                if (sparse[s]) {  // first word of the window: both loads in flight before any use
                    int w = lo[s] >> 3;
                    mv[s] = a.Mr64[vv[s] * J8 + w];
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
                    cand[s] = mv[s] & live8_bits<BLOCKED>(a, u[s], w, lb[s], lo[s]);
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
                    uint32_t raised = prev[s] == mu[s] ? diff_bits8(mu[s], nw[s])
                                                       : vmax_cas8(&a.M64[u[s] * J8 + w], prev[s], cand[s]);
                    chg[s] |= record8(a, u[s], w, raised);
                }
                if (sparse[s])  // remaining words of a multi-word window
                    for (int w = (lo[s] >> 3) + 1; w <= (hi[s] - 1) >> 3; ++w)
                        chg[s] |= pull_word8_bits<BLOCKED>(a, u[s], vv[s], w, lb[s], lo[s]);
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
                    for (int w = (dlo >> 3) + lane; w <= (dhi - 1) >> 3; w += 32) c |= pull_word8<BLOCKED, FILTER>(a, sX, du, dv, w, dh, dT, dlo, dhi);
                    c = __reduce_or_sync(IM_FULL, c);
                    if (lane == l) chg[s] |= c;
                }
            }
            // which 32-simulation chunks of u rose (fire-and-forget; the compaction builds the next frontier)
#pragma unroll
            for (int s = 0; s < NS; s++)
                if (chg[s]) atomicOr(&a.bits_out[u[s]], chg[s]);
        }
    }
    if (lane == 0 && wcount) atomicAdd(&a.ctr->win_edges, (ull)wcount);
}

// ------------------------------------------------------------------ frontier compaction
// Next frontier: every vertex v whose chunk bits are set.  A short in-edge row (<= SEG) is emitted
// whole (the sweep's exact filter skips edges whose window holds no changed simulation); a long
// row of a hash-sorted graph is queued for k_slices_big, which emits, per 32-simulation word of
// v's change mask, the slice of the row whose windows can meet those simulations.  The buffers
// of the sweep before are cleared here for the next sweep's writes.
__global__ void k_compact(int32_t n, int J, int slice_min, const uint32_t* __restrict__ bits_new, uint32_t* __restrict__ bits_clear,
                          uint32_t* __restrict__ cm_clear, const int32_t* __restrict__ roff, int4* __restrict__ items,
                          int32_t* __restrict__ big, IterCounters* ctr, int32_t* __restrict__ vl_out) {
    const int lane = threadIdx.x & 31, W = J >> 5;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    constexpr int CU = 8;  // vertex groups of BLOCK per block iteration, loaded up front
    for (int64_t base0 = (int64_t)blockIdx.x * blockDim.x * CU; base0 < n; base0 += stride * CU) {
      uint32_t bn[CU], bcl[CU];
      bool anyn = false;
#pragma unroll
      for (int k = 0; k < CU; k++) {
          const int64_t v = base0 + (int64_t)k * blockDim.x + threadIdx.x;
          bn[k] = v < n ? bits_new[v] : 0u;
          bcl[k] = v < n && bits_clear ? bits_clear[v] : 0u;
          anyn |= bn[k] != 0u;
      }
#pragma unroll
      for (int k = 0; k < CU; k++) {
          const int64_t v = base0 + (int64_t)k * blockDim.x + threadIdx.x;
          uint32_t bc = bcl[k];
          if (bc) {
              bits_clear[v] = 0u;
              for (; bc; bc &= bc - 1) cm_clear[(size_t)v * W + (__ffs(bc) - 1)] = 0u;
          }
      }
      if (!__syncthreads_or(anyn)) continue;
      // every group of this iteration at once: the row bounds of all changed vertices are loaded
      // together, then one block-wide reservation for the thread's items / big rows
      int rbk[CU], rdk[CU];
#pragma unroll
      for (int k = 0; k < CU; k++) {
          rbk[k] = rdk[k] = 0;
          if (bn[k]) {
              const int64_t v = base0 + (int64_t)k * blockDim.x + threadIdx.x;
              rbk[k] = roff[v];
              rdk[k] = roff[v + 1] - rbk[k];
          }
      }
      int t_items = 0, t_changed = 0, t_big = 0;
      long long t_edges = 0;
#pragma unroll
      for (int k = 0; k < CU; k++)
          if (bn[k]) {
              t_changed++;
              if (rdk[k] > slice_min) t_big++;
              else {
                  t_items += (rdk[k] + SEG - 1) / SEG;
                  t_edges += rdk[k];
              }
          }
      const int ci = warp_incl_scan(t_items, lane), cc = warp_incl_scan(t_changed, lane), cb = warp_incl_scan(t_big, lane);
      long long esum = t_edges;
#pragma unroll
      for (int o = 16; o; o >>= 1) esum += __shfl_xor_sync(IM_FULL, esum, o);
      BlockTotals wt{ci, cc, cb, (unsigned long long)esum};
      int pos, cpos, bpos;
      block_reserve<BLOCK / 32>(wt, lane, threadIdx.x >> 5, &ctr->next_items, &ctr->changed, &ctr->next_edges, &ctr->big,
                                pos, cpos, bpos);
      int p = pos + ci - t_items, bp = bpos + cb - t_big, cp = cpos + cc - t_changed;
#pragma unroll
      for (int k = 0; k < CU; k++) {
          if (!bn[k]) continue;
          const int v = (int)(base0 + (int64_t)k * blockDim.x + threadIdx.x);
          vl_out[cp++] = v;  // the changed vertices (k_sweep_small clears their masks by this list)
          const int rb = rbk[k], rd = rdk[k];
          if (rd > slice_min) {
              big[bp++] = v;
          } else {
              for (int s0 = rb; s0 < rb + rd; s0 += SEG) items[p++] = make_int4(v, s0, min(s0 + SEG, rb + rd), 0);
          }
      }
    }
}

// Bucket slices (rows with a bucket offset table, im_prep.cu): the edges of a bucket-ordered row whose
// candidate windows can hold simulation j are exactly its bucket Xs[j] >> B (Eq. 5: (X xor h) < T <= 2^B
// implies X >> B == h >> B).  A warp per long row marks the buckets of the set simulations of the row's
// mask (the change mask for a sweep, Delta for a BFS level) in a 2^KB-bit set, turns its runs of
// consecutive buckets into row slices (two table reads each) and cuts them into <= SEG items.  More
// than BSL runs, or runs covering >= 3/4 of the buckets: the whole row (the per-edge test drops the
// rest).  Items per row <= ceil(len / SEG) + BSL (buffer capacity, im_abi.cu).
__global__ void k_slices_buckets(int J, int B, int KB, const uint32_t* __restrict__ Xs, const int32_t* __restrict__ big,
                                 const uint32_t* __restrict__ mask, const int32_t* __restrict__ offs, int4* __restrict__ items,
                                 IterCounters* ctr, const int32_t* __restrict__ tidx, const int32_t* __restrict__ tab, int nbk) {
    __shared__ uint32_t sM[BLOCK / 32][32];
    __shared__ int sBs[257];  // first simulation of every bucket (the salts are sorted: the simulations of a bucket are a range)
    __shared__ int sRs[BLOCK / 32][BSL], sRe[BLOCK / 32][BSL];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, W = J >> 5;
    const int NBK = 1 << KB, NBW = (NBK + 31) >> 5;  // buckets, words of the bucket set (<= 8)
    const int nb = ctr->big;
    if ((int64_t)blockIdx.x * (BLOCK / 32) >= nb) return;  // no row for any warp of this block
    for (int b = threadIdx.x; b <= NBK; b += blockDim.x) {  // lower bound of bucket b among the sorted salts
        int lo = 0, hi = J;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((__ldg(&Xs[mid]) >> B) < (uint32_t)b) lo = mid + 1; else hi = mid;
        }
        sBs[b] = lo;
    }
    __syncthreads();
    // One row per warp and block iteration; the block's rows reserve their items with ONE global atomic (a
    // returning atomic per row on the same counter serialised ~300k rows of an early C4 sweep), the edge count
    // is added once per block at the end.
    __shared__ int sCnt[BLOCK / 32], sPos[BLOCK / 32];
    __shared__ ull sEd[BLOCK / 32];
    ull edges_acc = 0;  // thread 0
    for (int64_t base = (int64_t)blockIdx.x * (BLOCK / 32); base < nb; base += (int64_t)gridDim.x * (BLOCK / 32)) {
        const int64_t i = base + wib;
        const bool act = i < nb;
        int v = 0, rb = 0, re = 0, t = -1;
        if (act) {
            v = big[i];
            rb = offs[v];
            re = offs[v + 1];
            t = __ldg(&tidx[v]);
        }
        sM[wib][lane] = act && lane < W ? mask[(size_t)v * W + lane] : 0u;
        __syncwarp();
        // bucket lane + 32 k is marked iff the mask holds a simulation of its range (a loop over the set
        // simulations with one salt load and one shared atomic each cost up to 32 dependent trips per lane)
        uint32_t x = 0u;
        for (int k = 0; k < NBW; k++) {
            const int b = lane + 32 * k;
            bool hit = false;
            if (b < NBK) {
                const int s = sBs[b], e = sBs[b + 1];
                if (s < e) {
                    const int w0 = s >> 5, w1 = (e - 1) >> 5;
                    for (int w = w0; w <= w1 && !hit; ++w)
                        hit = (sM[wib][w] & bit_range(w == w0 ? (s & 31) : 0, w == w1 ? ((e - 1) & 31) : 31)) != 0u;
                }
            }
            const uint32_t xk = __ballot_sync(IM_FULL, hit);
            if (lane == k) x = xk;
        }
        uint32_t prev = __shfl_up_sync(IM_FULL, x, 1), next = __shfl_down_sync(IM_FULL, x, 1);
        if (lane == 0) prev = 0u;
        if (lane == 31) next = 0u;
        const uint32_t starts = x & ~((x << 1) | (prev >> 31)), ends = x & ~((x >> 1) | (next << 31));
        const int ns = __popc(starts), ne = __popc(ends);
        const int R = __reduce_add_sync(IM_FULL, ns), cov = __reduce_add_sync(IM_FULL, __popc(x));
        const bool whole = R > 0 && (t < 0 || R > BSL || 4 * cov >= 3 * (1 << KB));  // the whole row
        int b0 = 0, len = 0, nsl = 0, ninc = 0, ntot = 0;
        ull es = 0;
        if (whole) {
            ntot = (re - rb + SEG - 1) / SEG;
            es = (ull)(re - rb);
        } else if (R > 0) {
            // the k-th run starts at the k-th start bit and ends at the k-th end bit
            int sp = warp_incl_scan(ns, lane) - ns, ep = warp_incl_scan(ne, lane) - ne;
            for (uint32_t tt = starts; tt; tt &= tt - 1) sRs[wib][sp++] = 32 * lane + __ffs(tt) - 1;
            for (uint32_t tt = ends; tt; tt &= tt - 1) sRe[wib][ep++] = 32 * lane + __ffs(tt) - 1;
            __syncwarp();
            if (lane < R) {
                const int32_t* tb = tab + (int64_t)t * nbk;
                b0 = __ldg(&tb[sRs[wib][lane]]);
                len = __ldg(&tb[sRe[wib][lane] + 1]) - b0;
            }
            nsl = (len + SEG - 1) / SEG;
            ninc = warp_incl_scan(nsl, lane);
            ntot = __shfl_sync(IM_FULL, ninc, 31);
            es = (ull)__reduce_add_sync(IM_FULL, len);
        }
        if (lane == 0) {
            sCnt[wib] = ntot;
            sEd[wib] = es;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
#pragma unroll
            for (int w = 0; w < BLOCK / 32; w++) {
                sPos[w] = tot;
                tot += sCnt[w];
                edges_acc += sEd[w];
            }
            const int g0 = tot ? atomicAdd(&ctr->next_items, tot) : 0;
#pragma unroll
            for (int w = 0; w < BLOCK / 32; w++) sPos[w] += g0;
        }
        __syncthreads();
        const int pos = sPos[wib];
        if (whole) {
            for (int k = lane; k < ntot; k += 32) items[pos + k] = make_int4(v, rb + k * SEG, min(rb + (k + 1) * SEG, re), 0);
        } else if (ntot) {
            int p = pos + ninc - nsl;
            for (int s0 = b0; s0 < b0 + len; s0 += SEG) items[p++] = make_int4(v, s0, min(s0 + SEG, b0 + len), 0);
        }
    }
    if (threadIdx.x == 0 && edges_acc) atomicAdd(&ctr->next_edges, edges_acc);
}

// ------------------------------------------------------------------ small-frontier sweeps in one cluster
// The tail of a build (and most of a rebuild on small graphs) is a long run of sweeps over a few hundred
// changed vertices, where the multi-block sweep (k_sweep + k_compact + k_slices_buckets and a host round
// trip) is launch- and latency-bound.  k_sweep_small runs those sweeps inside ONE thread-block cluster
// (SS_CLUSTER blocks, one per SM): every changed vertex v of the previous sweep has its in-row walked
// (warp per vertex, lane per edge; rows longer than SS_LONG by every warp of the cluster), each edge (u, v)
// pushes the live simulations in which v changed into M_u with the byte-max CAS of k_sweep (the same exact
// filter, in place), and u is appended to the next sweep's vertex list by the lane whose chunk-bit OR
// first marked it.  Between sweeps: cluster barriers; the previous sweep's change masks are cleared by
// vertex list.  The first sweep takes the host loop's work items (k_compact's).  It stops at the
// fixpoint, or hands a frontier whose in-edges exceed max_edges back to the host loop (bits / masks of
// the last sweep left set, exactly as after a k_sweep).  Only for eps_c = 0 (in-place sweeps).
constexpr int SS_THREADS = 1024;
constexpr int SS_CLUSTER = 8;
constexpr int SS_LONG = 256;

struct SweepSmallArgs {
    int n, J;
    const int32_t* roff;
    const uint2* rev;
    const uint32_t* revT;
    uint32_t T0;
    const uint32_t* Xs;
    const uint16_t* s12;
    ull* M64;
    const uint32_t* vis;
    uint32_t* cm[2];
    uint32_t* bits[2];
    int32_t* vl[2];            // vertex lists (n entries each)
    int32_t* longv;            // long rows of a sweep (scratch)
    const int4* items0;        // the first sweep's work items (host loop's compaction) and their count
    int n_items0;
    int n_changed0;            // vertices the sweep before changed (their list is vl[0], written by k_compact)
    int s0;                    // index of the first sweep (buffer parity)
    long long max_edges;
    SweepSmallOut* out;
};

// one in-edge e of v (source u = rev[e].x): returns the chunk bits of u this edge raised
template <bool CONST_T, bool BLOCKED>
__device__ __forceinline__ uint32_t small_push(const SweepSmallArgs& a, const uint32_t* sX, const uint16_t* sS, int e, uint32_t v,
                                               const uint32_t* cm_in, uint32_t* cm_out, uint32_t& wcount) {
    const uint2 r = __ldcs(&a.rev[e]);
    const uint32_t T = CONST_T ? a.T0 : __ldcs(&a.revT[e]);
    if (!T) return 0u;
    int lo, hi;
    edge_window(r.y, T, sX, sS, a.J, lo, hi);
    if (lo >= hi) return 0u;
    const int W = a.J >> 5;
    const size_t J8 = (size_t)(a.J >> 3);
    const uint32_t u = r.x;
    uint32_t chg = 0u;
    bool worked = false;
    for (int w = lo >> 3; w <= (hi - 1) >> 3; ++w) {
        uint32_t cand = (__ldg(&cm_in[(size_t)v * W + (w >> 2)]) >> ((w & 3) << 3)) & 0xFFu;
        if (!cand) continue;
        ull live = 0;
        for (; cand; cand &= cand - 1) {
            const int b = __ffs(cand) - 1, i = 8 * w + b;
            if (i >= lo && i < hi && (sX[i] ^ r.y) < T) live |= 0xFFull << (8 * b);
        }
        if (BLOCKED && live) live &= ~expand8((a.vis[(size_t)u * W + (w >> 2)] >> ((w & 3) << 3)) & 0xFFu);
        if (!live) continue;
        worked = true;
        const ull cv = a.M64[v * J8 + w] & live;
        if (!cv) continue;
        ull* p = &a.M64[u * J8 + w];
        const uint32_t raised = vmax_cas8(p, __ldcg(p), cv);
        if (raised) {
            atomicOr(&cm_out[(size_t)u * W + (w >> 2)], raised << ((w & 3) << 3));
            chg |= 1u << (w >> 2);
        }
    }
    wcount += worked;
    return chg;
}

template <bool CONST_T, bool BLOCKED>
__global__ void __cluster_dims__(SS_CLUSTER, 1, 1) __launch_bounds__(SS_THREADS) k_sweep_small(SweepSmallArgs a) {
    __shared__ uint32_t sX[1024];
    __shared__ uint16_t sS[4098];
    __shared__ int s_next, s_nlong, s_changed;
    __shared__ unsigned long long s_edges, s_win;
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = (int)cluster.block_rank(), csize = (int)cluster.num_blocks();
    int* c_next = cluster.map_shared_rank(&s_next, 0);
    int* c_nlong = cluster.map_shared_rank(&s_nlong, 0);
    unsigned long long* c_edges = cluster.map_shared_rank(&s_edges, 0);
    unsigned long long* c_win = cluster.map_shared_rank(&s_win, 0);
    const int W = a.J >> 5, lane = threadIdx.x & 31, wib = threadIdx.x >> 5, NWARP = SS_THREADS / 32;
    const int gw = crank * NWARP + wib, GW = csize * NWARP, gt = crank * SS_THREADS + threadIdx.x, GT = csize * SS_THREADS;
    for (int i = threadIdx.x; i < a.J; i += blockDim.x) sX[i] = a.Xs[i];
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) sS[i] = a.s12[i];
    int t = a.s0, n_v = -1, sweeps = 0, lst = 0;
    long long edges_total = 0, win_total = 0, last_edges = 0;
    int last_changed = 0;
    bool bailed = false;
    __syncthreads();
    for (;;) {
        const int pi = (t - 1) & 1, ci = t & 1;  // input (previous sweep) / output parity
        const uint32_t* cm_in = a.cm[pi];
        uint32_t* cm_out = a.cm[ci];
        uint32_t* bits_out = a.bits[ci];
        int32_t* vln = a.vl[lst ^ 1];
        if (crank == 0 && threadIdx.x == 0) {
            s_next = 0;
            s_nlong = 0;
            s_edges = 0ull;
            s_win = 0ull;
        }
        cluster.sync();
        uint32_t wcount = 0;
        unsigned long long ed = 0;
        auto push_edge = [&](int e, uint32_t v) {
            const uint32_t chg = small_push<CONST_T, BLOCKED>(a, sX, sS, e, v, cm_in, cm_out, wcount);
            if (chg) {
                const uint32_t u = a.rev[e].x;
                if (atomicOr(&bits_out[u], chg) == 0u) vln[atomicAdd(c_next, 1)] = (int32_t)u;
            }
        };
        if (n_v < 0) {  // the first sweep: the host loop's work items (segments of <= SEG in-edges)
            for (int it = gw; it < a.n_items0; it += GW) {
                const int4 I = a.items0[it];
                for (int e = I.y + lane; e < I.z; e += 32) push_edge(e, (uint32_t)I.x);
                if (lane == 0) ed += (unsigned long long)(I.z - I.y);
            }
        } else {
            const int32_t* vl = a.vl[lst];
            for (int i = gw; i < n_v; i += GW) {
                const uint32_t v = (uint32_t)vl[i];
                const int eb = a.roff[v], ee = a.roff[v + 1];
                if (ee - eb > SS_LONG) {
                    if (lane == 0) a.longv[atomicAdd(c_nlong, 1)] = (int32_t)v;
                    continue;
                }
                for (int e = eb + lane; e < ee; e += 32) push_edge(e, v);
                if (lane == 0) ed += (unsigned long long)(ee - eb);
            }
            cluster.sync();
            const int nlong = *c_nlong;
            for (int li = 0; li < nlong; li++) {  // long in-rows: split over every warp of the cluster
                const uint32_t v = (uint32_t)a.longv[li];
                const int eb = a.roff[v], ee = a.roff[v + 1];
                for (int e = eb + gw * 32 + lane; e < ee; e += GW * 32) push_edge(e, v);
                if (gw == 0 && lane == 0) ed += (unsigned long long)(ee - eb);
            }
        }
        wcount = __reduce_add_sync(IM_FULL, wcount);
        if (lane == 0 && wcount) atomicAdd(c_win, (unsigned long long)wcount);
        if (ed) atomicAdd(c_edges, ed);
        cluster.sync();
        // the previous sweep's change masks / bits are consumed: clear them (by its vertex list, or by the
        // first sweep's items); its output is the sweep after next's input
        {   // by vertex list: the cluster's own list, or for the first sweep the host loop's (k_compact's; a scan of
            // all n chunk words by 8 blocks cost 0.7 ms on the 16.8M-vertex RMAT)
            const int32_t* vl = a.vl[lst];
            const int nc = n_v < 0 ? a.n_changed0 : n_v;
            for (int64_t i = gt; i < (int64_t)nc * W; i += GT) {
                const uint32_t v = (uint32_t)vl[i / W];
                a.cm[pi][(size_t)v * W + (i % W)] = 0u;
                if (i % W == 0) a.bits[pi][v] = 0u;
            }
        }
        const int nn = *c_next;
        edges_total += (long long)*c_edges;
        win_total += (long long)*c_win;
        last_changed = nn;
        sweeps++;
        t++;
        lst ^= 1;
        n_v = nn;
        // the next sweep's in-edges (for the hand-back test): sum of in-degrees of the new list
        if (crank == 0 && threadIdx.x == 0) s_edges = 0ull;
        cluster.sync();
        if (n_v == 0) break;
        unsigned long long ne = 0;
        for (int i = gt; i < n_v; i += GT) {
            const int v = a.vl[lst][i];
            ne += (unsigned long long)(a.roff[v + 1] - a.roff[v]);
        }
        if (ne) atomicAdd(c_edges, ne);
        cluster.sync();
        last_edges = (long long)*c_edges;
        cluster.sync();  // every block has read the counters before rank 0 resets them
        if (last_edges == 0) break;  // changed vertices without in-edges: the fixpoint
        if (last_edges > a.max_edges) {
            bailed = true;
            break;
        }
    }
    if (crank == 0 && threadIdx.x == 0) {
        a.out->sweeps = sweeps;
        a.out->edges = edges_total;
        a.out->win_edges = win_total;
        a.out->changed = last_changed;
        a.out->bailed = bailed ? 1 : 0;
        a.out->next_edges = last_edges;
        a.out->t_next = t;
    }
}

cudaError_t launch_sweep_small(Ctx& c, const int4* items, int n_items, int n_changed, int s0, bool blocked, long long max_edges) {
    SweepSmallArgs a;
    a.n = c.n;
    a.J = c.J;
    a.roff = c.roff;
    a.rev = c.rev;
    a.revT = c.revT;
    a.T0 = c.T0;
    a.Xs = c.Xs;
    a.s12 = c.s12;
    a.M64 = reinterpret_cast<ull*>(c.M);
    a.vis = c.vis;
    a.cm[0] = c.cm[0];
    a.cm[1] = c.cm[1];
    a.bits[0] = c.bits[0];
    a.bits[1] = c.bits[1];
    a.vl[0] = c.bvl[0];
    a.vl[1] = c.bvl[1];
    a.longv = c.big;
    a.items0 = items;
    a.n_items0 = n_items;
    a.n_changed0 = n_changed;
    a.s0 = s0;
    a.max_edges = max_edges;
    a.out = c.sso;
    if (c.constT) {
        if (blocked) k_sweep_small<true, true><<<SS_CLUSTER, SS_THREADS, 0, c.stream>>>(a);
        else k_sweep_small<true, false><<<SS_CLUSTER, SS_THREADS, 0, c.stream>>>(a);
    } else {
        if (blocked) k_sweep_small<false, true><<<SS_CLUSTER, SS_THREADS, 0, c.stream>>>(a);
        else k_sweep_small<false, false><<<SS_CLUSTER, SS_THREADS, 0, c.stream>>>(a);
    }
    return LAUNCHED(c);
}

template <bool C, bool B, bool F>
static void sweep_inst(int grid, cudaStream_t s, const SweepArgs& a) {
    k_sweep<C, B, F><<<grid, BLOCK, 0, s>>>(a);
}

cudaError_t launch_sweep(Ctx& c, const int4* items, int n_items, const uint32_t* cm_in, uint32_t* cm_out,
                         uint32_t* bits_out, IterCounters* ctr, bool blocked, const IterCounters* nin) {
    SweepArgs a;
    a.items = items;
    a.n_items = n_items;
    a.nin = nin;
    a.ctr = ctr;
    a.rev = c.rev;
    a.revT = c.revT;
    a.T0 = c.T0;
    a.Xs = c.Xs;
    a.s12 = c.s12;
    a.J = c.J;
    a.M64 = reinterpret_cast<ull*>(c.M);
    a.Mr64 = reinterpret_cast<const ull*>(c.sync_sweeps ? c.Mold : c.M);
    a.vis = c.vis;
    a.cm_in = cm_in;
    a.cm_out = cm_out;
    a.bits_out = bits_out;
    // items per warp batch: 32, or fewer so that a small sweep (long hub items) still fills the GPU
    const int64_t warps_max = (int64_t)c.max_blocks_sweep * (BLOCK / 32);
    a.warps_max = (int)warps_max;
    a.ipw = (int)std::min<int64_t>(32, std::max<int64_t>(1, n_items / warps_max));
    int64_t want = ((int64_t)n_items + (int64_t)a.ipw * (BLOCK / 32) - 1) / ((int64_t)a.ipw * (BLOCK / 32));
    int grid = nin ? c.max_blocks_sweep : (int)(want < 1 ? 1 : (want > c.max_blocks_sweep ? c.max_blocks_sweep : want));
    const bool ct = c.constT, f = cm_in != nullptr;
    if (!f) {
        if (ct) { if (blocked) sweep_inst<true, true, false>(grid, c.stream, a); else sweep_inst<true, false, false>(grid, c.stream, a); }
        else { if (blocked) sweep_inst<false, true, false>(grid, c.stream, a); else sweep_inst<false, false, false>(grid, c.stream, a); }
    } else {
        if (ct) { if (blocked) sweep_inst<true, true, true>(grid, c.stream, a); else sweep_inst<true, false, true>(grid, c.stream, a); }
        else { if (blocked) sweep_inst<false, true, true>(grid, c.stream, a); else sweep_inst<false, false, true>(grid, c.stream, a); }
    }
    return LAUNCHED(c);
}

// synchronous sweeps (R22): after a sweep, bring the read copy up to date -- copy every 32-simulation
// chunk whose change bit is set (bits_new) from M to Mold, so Mold == M again for the next sweep
__global__ void k_commit(int32_t n, int J, const uint32_t* __restrict__ bits_new, const uint4* __restrict__ M, uint4* Mold) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int C = J >> 4;  // 16-byte chunks per row
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
        for (uint32_t b = bits_new[v]; b; b &= b - 1) {
            const int w = __ffs(b) - 1;
            const int64_t i = v * C + 2 * w;
            Mold[i] = M[i];
            Mold[i + 1] = M[i + 1];
        }
    }
}

cudaError_t launch_commit(Ctx& c, const uint32_t* bits_new) {
    k_commit<<<grid_for(c, c.n), BLOCK, 0, c.stream>>>(c.n, c.J, bits_new, reinterpret_cast<const uint4*>(c.M),
                                                       reinterpret_cast<uint4*>(c.Mold));
    return LAUNCHED(c);
}

cudaError_t launch_compact(Ctx& c, const uint32_t* bits_new, uint32_t* bits_clear, const uint32_t* cm_new,
                           uint32_t* cm_clear, int4* items_out, IterCounters* ctr) {
    k_compact<<<grid_for(c, c.n), BLOCK, 0, c.stream>>>(c.n, c.J, c.sorted_h ? c.slice_min : INT_MAX, bits_new, bits_clear, cm_clear, c.roff,
                                                        items_out, c.big, ctr, c.bvl[0]);
    cudaError_t e = LAUNCHED(c);
    if (e || !c.sorted_h) return e;
    return launch_slices_big(c, c.big, cm_new, c.roff, c.rev, items_out, ctr, false);
}

cudaError_t launch_slices_big(Ctx& c, const int32_t* big, const uint32_t* mask, const int32_t* offs, const uint2* rec,
                              int4* items_out, IterCounters* ctr, bool whole_dense) {
    const bool fw = rec == c.fwd;
    (void)whole_dense;
    k_slices_buckets<<<c.num_sms * 4, BLOCK, 0, c.stream>>>(c.J, c.Bs, 31 - c.Bs, c.Xs, big, mask, offs, items_out, ctr,
                                                           fw ? c.ftidx : c.rtidx, fw ? c.ftab : c.rtab, c.nbk);
    return LAUNCHED(c);

}

int occupancy_sweep(int* blocks_per_sm) {
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_sweep<true, true, true>, BLOCK, 0);
}

}  // namespace im
