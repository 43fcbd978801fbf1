// im_kernels.cu -- sm_100a kernels of the hot path.
//
//   (edge prep and register init: im_prep.cu)                          a0, a2
//   (k_sweep / k_compact: im_sweep.cu)                                 a3+a4 Simulate sweeps (Alg. 2)
//   k_estimate                                                         a5 Eq. 2
//   k_argmax / k_seed_start / k_bfs_level / k_bfs_clear / k_error_check a6-a8 Alg. 1 loop body
//
// No tensor cores: the path is integer gather / byte-max, bound by HBM and the
// INT pipes.  All work-list kernels are persistent (grid <= resident blocks)
// and pull 32-item batches from a device cursor.

#include <algorithm>
#include <climits>

#include "im_device.cuh"
#include "im_internal.h"

namespace im {

// ============================================================ a5: Eq. 2 estimate
// A warp sums EV rows per iteration (16-byte loads, all EV rows' loads in flight before the
// reductions); lane k finishes row k, so the EV exp2 run in parallel.  Exact integer sums.
#ifndef IM_EV
#define IM_EV 4
#endif
constexpr int EV = IM_EV;
template <bool SUMS>
__global__ void k_estimate(int32_t n, int32_t J, const uint32_t* __restrict__ M32, double* __restrict__ out, int32_t* sums) {
    const int lane = threadIdx.x & 31, nch = J >> 4;
    const uint4* M16 = reinterpret_cast<const uint4*>(M32);
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * EV; v0 < n; v0 += warps * EV) {
        uint32_t s[EV];
#pragma unroll
        for (int k = 0; k < EV; k++) s[k] = 0u;
        for (int c0 = 0; c0 < nch; c0 += 32) {  // the EV rows' loads of this chunk column issued before any is summed
            const int c = c0 + lane;
            uint4 x[EV];
#pragma unroll
            for (int k = 0; k < EV; k++)
                x[k] = (c < nch && v0 + k < n) ? __ldcs(&M16[(v0 + k) * nch + c]) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int k = 0; k < EV; k++)
                s[k] += __vsadu4(x[k].x, 0u) + __vsadu4(x[k].y, 0u) + __vsadu4(x[k].z, 0u) + __vsadu4(x[k].w, 0u);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int k = 0; k < EV; k++) s[k] += __shfl_xor_sync(IM_FULL, s[k], o);
        uint32_t mine = s[0];
#pragma unroll
        for (int k = 1; k < EV; k++) mine = lane == k ? s[k] : mine;
        if (lane < EV && v0 + lane < n) {
            if (SUMS) sums[v0 + lane] = (int32_t)mine;
            else out[v0 + lane] = exp2((double)mine / (double)J) / 0.77351;
        }
    }
}

// sharded (Sec. 8(e) of SURVEY.md): Eq. 2 from the register sums allreduced over all J_total simulations
__global__ void k_estimate_fin(int32_t n, int32_t Jt, const int32_t* __restrict__ sums, double* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride)
        out[v] = exp2((double)sums[v] / (double)Jt) / 0.77351;
}

// ============================================================ a6: greedy argmax
// Alg. 1 line 10: s = argmax_v Estimate(Merge(M_S', M_v)).  Estimate is monotone in the integer
// score_v = sum_j max(M_S'[j], M_v[j]) = sum_j M_S'[j] + gain_v with gain_v = sum_j (M_v[j] - M_S'[j])^+,
// so the argmax over the pool (R14) is the argmax of gain_v, lowest id on ties via the 64-bit key
// gain<<32 | (2^32-1-v).  gain_v only shrinks while M_S' grows (between rebuilds), so an exact lazy
// argmax is used: a full pass stores every gain (an upper bound for later steps) and the list of
// vertices with stored gain >= theta (about T of them); later steps evaluate only that list, and the
// result is exact whenever its best current gain is >= theta (every vertex outside the list has
// current gain <= stored gain < theta).  Otherwise the host runs a new full pass.
// A row is read as 16-byte chunks by L lanes, 32/L vertices per warp, two groups in flight.
// 2 * sum (x - m)^+ = sum |x - m| + sum x - sum m over the 16 bytes; the |.| sums are single
// VABSDIFF4 instructions.  The caller subtracts sum m (a per-lane constant) and halves at the end.
__device__ __forceinline__ uint32_t gain16x2(uint4 x, uint4 m) {
    return __vsadu4(x.x, m.x) + __vsadu4(x.y, m.y) + __vsadu4(x.z, m.z) + __vsadu4(x.w, m.w) + __vsadu4(x.x, 0u) +
           __vsadu4(x.y, 0u) + __vsadu4(x.z, 0u) + __vsadu4(x.w, 0u);
}
__device__ __forceinline__ uint32_t sum16(uint4 m) {
    return __vsadu4(m.x, 0u) + __vsadu4(m.y, 0u) + __vsadu4(m.z, 0u) + __vsadu4(m.w, 0u);
}

constexpr int HIST_BINS = 4096;
#ifndef BFS_EP
#define BFS_EP 2  // edges in flight per lane of k_bfs_level2 (3 and 4 measured slower on C4)
#endif
#ifndef BFS_MINB
#define BFS_MINB 5  // min resident blocks per SM k_bfs_level2 is compiled for (48 registers, no spills)
#endif
constexpr int CU = 8;  // vertex groups of BLOCK per block iteration of the frontier compactions
constexpr int AG = 2;  // vertex groups in flight per warp in k_argmax
constexpr int AC = 4;  // max 16-byte chunks per lane in k_argmax (L = max(8, J/64))

// LIST = false: every vertex (full pass: stores gains + histogram); LIST = true: the vertices in list[0..*count)
// SHARD (list only): writes the packed local value gain + (in local pool) << 24 to gain_out[i] for list entry i
template <bool POOL, bool LIST, bool SHARD = false>
__global__ void __launch_bounds__(BLOCK) k_argmax(int32_t n, int32_t J, int L, int C, const uint4* __restrict__ M16,
                                                  const uint8_t* __restrict__ MS, const uint32_t* __restrict__ vis,
                                                  ull* key, int32_t* gain_out, uint32_t* hist, int shift,
                                                  const int32_t* __restrict__ list, const int* list_count) {
    __shared__ uint4 sMS[64];
    __shared__ ull sKey[BLOCK / 32];
    __shared__ uint32_t sHist[LIST ? 1 : HIST_BINS];
    const int nch = J >> 4, W = J >> 5;
    for (int i = threadIdx.x; i < nch; i += blockDim.x) sMS[i] = reinterpret_cast<const uint4*>(MS)[i];
    if (!LIST)
        for (int i = threadIdx.x; i < HIST_BINS; i += blockDim.x) sHist[i] = 0u;
    __syncthreads();
    const int nv = LIST ? *list_count : n;
    const int lane = threadIdx.x & 31, q = lane & (L - 1), sub = lane / L, VPW = 32 / L;
    uint4 ms[AC];
    uint32_t msum = 0;  // sum of this lane's M_S' bytes (only over chunks the lane actually loads)
#pragma unroll
    for (int c = 0; c < AC; c++) {
        int ci = c * L + q;  // interleaved: the L lanes of a vertex read 16*L contiguous bytes per c
        ms[c] = (c < C && ci < nch) ? sMS[ci] : make_uint4(0, 0, 0, 0);
        msum += sum16(ms[c]);
    }
    const int64_t groups = ((int64_t)nv + VPW - 1) / VPW;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    ull best = 0;
    for (int64_t g0 = gw; g0 < groups; g0 += AG * nwarps) {
        uint4 x[AG][AC];
        int64_t vv[AG];
        bool ok[AG];
#pragma unroll
        for (int u = 0; u < AG; u++) {
            int64_t idx = (g0 + u * nwarps) * VPW + sub;
            ok[u] = (g0 + u * nwarps) < groups && idx < nv;
            vv[u] = ok[u] ? (LIST ? (int64_t)list[idx] : idx) : 0;
            if (LIST && vv[u] < 0) {  // a hole of a sharded job's gathered list (padding of a shorter rank list)
                if (SHARD && q == 0) gain_out[idx] = 0;
                ok[u] = false;
                vv[u] = 0;
            }
#pragma unroll
            for (int c = 0; c < AC; c++) {
                int ci = c * L + q;
                x[u][c] = (ok[u] && c < C && ci < nch) ? __ldcs(&M16[vv[u] * nch + ci]) : make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int u = 0; u < AG; u++) {
            uint32_t gn = 0u - msum;
#pragma unroll
            for (int c = 0; c < AC; c++) gn += gain16x2(x[u][c], ms[c]);
            int full = 1;
            if (POOL && ok[u])
                for (int w = q; w < W; w += L) full &= __ldcs(&vis[vv[u] * W + w]) == IM_FULL;
            for (int o = L >> 1; o; o >>= 1) {
                gn += __shfl_xor_sync(IM_FULL, gn, o);
                if (POOL) full &= __shfl_xor_sync(IM_FULL, full, o);
            }
            gn >>= 1;
            bool inpool = ok[u] && (!POOL || !full);
            if (SHARD) {
                if (ok[u] && q == 0) gain_out[(g0 + u * nwarps) * VPW + sub] = (int32_t)(gn + (inpool ? SHARD_POOL_ONE : 0u));
                continue;
            }
            if (ok[u] && q == 0) {
                if (inpool) {
                    ull k = ((ull)gn << 32) | (ull)(0xFFFFFFFFu - (uint32_t)vv[u]);
                    best = k > best ? k : best;
                }
                if (!LIST) {
                    gain_out[vv[u]] = inpool ? (int32_t)gn : -1;
                    if (inpool) atomicAdd(&sHist[min((int)(gn >> shift), HIST_BINS - 1)], 1u);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ull ob = __shfl_xor_sync(IM_FULL, best, o);
        best = ob > best ? ob : best;
    }
    if (lane == 0) sKey[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        ull b = 0;
        for (int i = 0; i < BLOCK / 32; i++) b = sKey[i] > b ? sKey[i] : b;
        if (b) atomicMax(key, b);
    }
    if (!LIST)
        for (int i = threadIdx.x; i < HIST_BINS; i += blockDim.x)
            if (sHist[i]) atomicAdd(&hist[i], sHist[i]);
}

// theta = lower edge of the highest histogram bin at which the suffix count reaches T
__global__ void k_theta(const uint32_t* __restrict__ hist, int shift, int T, int* theta) {
    // the largest bin b >= 1 whose suffix count sum_{i >= b} hist[i] reaches T (0 if none), by one
    // warp: lane l owns bins [l * PB, (l + 1) * PB); the lane where the suffix count crosses T walks
    // its bins from the top
    constexpr int PB = HIST_BINS / 32;
    const int lane = threadIdx.x;
    long long tot = 0;
    for (int i = 0; i < PB; i++) tot += hist[lane * PB + i];
    long long suf = tot;  // sum over lanes >= this one
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_down_sync(IM_FULL, suf, o);
        if (lane + o < 32) suf += y;
    }
    const long long above = suf - tot;
    const bool mine = above < (long long)T && (long long)T <= suf;
    if (!__any_sync(IM_FULL, mine)) {
        if (lane == 0) *theta = 0;
        return;
    }
    if (mine) {
        long long acc = above;
        int b = lane * PB + PB - 1;
        for (;; --b) {
            acc += hist[b];
            if (acc >= T || b == lane * PB) break;
        }
        *theta = (b < 1 ? 0 : b) << shift;
    }
}

// Candidate list = the vertices with stored gain >= theta, in ascending vertex order (the order is
// deterministic, so every rank of a sharded job indexes the same list).  Block b owns a contiguous
// vertex range: k_list_count counts its matches, k_list_write places them after the matches of
// blocks 0..b-1 with a block-wide scan per 256-vertex tile.
__device__ __forceinline__ void list_range(int32_t n, int b, int nb, int64_t& v0, int64_t& v1) {
    const int64_t chunk = (((int64_t)n + nb - 1) / nb + BLOCK - 1) / BLOCK * BLOCK;
    v0 = min((int64_t)n, b * chunk);
    v1 = min((int64_t)n, v0 + chunk);
}

__global__ void k_list_count(int32_t n, const int32_t* __restrict__ gain, const int* theta, int* bcount) {  // gain[0..n)
    __shared__ int sW[BLOCK / 32];
    const int th = *theta;
    int64_t v0, v1;
    list_range(n, blockIdx.x, gridDim.x, v0, v1);
    int cnt = 0;
    for (int64_t v = v0 + threadIdx.x; v < v1; v += BLOCK) cnt += gain[v] >= th;
    cnt = __reduce_add_sync(IM_FULL, cnt);
    if ((threadIdx.x & 31) == 0) sW[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < BLOCK / 32; i++) t += sW[i];
        bcount[blockIdx.x] = t;
    }
}

__global__ void k_list_write(int32_t n, const int32_t* __restrict__ gain, const int* theta, const int* __restrict__ bcount,
                             int32_t* list, int* count, int64_t vbase) {  // lists vertex vbase + i for gain[i] >= theta
    __shared__ int sW[BLOCK / 32];
    __shared__ int sBase;
    const int th = *theta, lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int part = 0;
    for (int i = threadIdx.x; i < (int)blockIdx.x; i += BLOCK) part += bcount[i];
    part = __reduce_add_sync(IM_FULL, part);
    if (lane == 0) sW[wib] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < BLOCK / 32; i++) t += sW[i];
        sBase = t;
        if (blockIdx.x == gridDim.x - 1) *count = t + bcount[blockIdx.x];
    }
    __syncthreads();
    int base = sBase;
    int64_t v0, v1;
    list_range(n, blockIdx.x, gridDim.x, v0, v1);
    for (int64_t t0 = v0; t0 < v1; t0 += BLOCK) {
        const int64_t v = t0 + threadIdx.x;
        const bool take = v < v1 && gain[v] >= th;
        const uint32_t m = __ballot_sync(IM_FULL, take);
        __syncthreads();  // sW reuse
        if (lane == 0) sW[wib] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
        for (int i = 0; i < BLOCK / 32; i++) {
            before += i < wib ? sW[i] : 0;
            total += sW[i];
        }
        if (take) list[base + before + __popc(m & ((1u << lane) - 1u))] = (int32_t)(vbase + v);
        base += total;
    }
}

// sharded argmax: vals[i] = sum over ranks of (local gain + local pool flag << 24),
// after the allreduce.  A vertex is in the global pool iff some rank still has an unvisited simulation
// of it (R14); its global gain is the low 24 bits.  Writes the key (and, for the full pass, the stored
// gains and histogram) exactly as the unsharded kernels do.
__global__ void k_argmax_decode(int nv, const int32_t* __restrict__ list, const int* list_count, const int32_t* __restrict__ vals,
                                int32_t* gain_out, ull* key, uint32_t* hist, int shift, int64_t v0) {
    __shared__ ull sKey[BLOCK / 32];
    if (list) nv = *list_count;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    ull best = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
        const uint32_t x = (uint32_t)vals[i];
        const int64_t vi = list ? (int64_t)list[i] : v0 + i;  // list hole: -1, packed value 0 (not in the pool)
        const uint32_t gn = x & (SHARD_POOL_ONE - 1u), v = (uint32_t)vi;
        const bool inpool = vi >= 0 && (x >> 24) != 0u;
        if (inpool) {
            ull k = ((ull)gn << 32) | (ull)(0xFFFFFFFFu - v);
            best = k > best ? k : best;
            if (hist) atomicAdd(&hist[min((int)(gn >> shift), HIST_BINS - 1)], 1u);
        }
        if (gain_out) gain_out[i] = inpool ? (int32_t)gn : -1;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ull ob = __shfl_xor_sync(IM_FULL, best, o);
        best = ob > best ? ob : best;
    }
    if ((threadIdx.x & 31) == 0) sKey[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        ull b = 0;
        for (int i = 0; i < BLOCK / 32; i++) b = sKey[i] > b ? sKey[i] : b;
        if (b) atomicMax(key, b);
    }
}

// ============================================================ a7: seed diffusion
// Alg. 1 lines 11, 13-14: S <- S + s; R_G(S) by a multi-simulation BFS from s over live edges
// (same samples as the sketches, R13) carrying J-bit masks; visited bits only ever set.
__global__ void k_seed_start(int32_t n, int32_t J, const ull* key, const uint32_t* __restrict__ M32,
                             const uint8_t* __restrict__ MS, uint8_t* inS, uint32_t* vis, uint2* vd, uint32_t* delta0,
                             const int32_t* __restrict__ off, int4* items0, int32_t* vl0, IterCounters* ctr0,
                             ull* sigma_count, StepDev* rec) {
    const int lane = threadIdx.x, W = J >> 5, Jw = J >> 2;
    ull k = *key;
    uint32_t s = k ? (0xFFFFFFFFu - (uint32_t)k) : 0u;
    if (!k) {  // pool empty (every vertex covered in every simulation): lowest id not in S (R14)
        for (int b = 0; b < n; b += 32) {
            uint32_t z = __ballot_sync(IM_FULL, b + lane < n && !inS[b + lane]);
            if (z) {
                s = (uint32_t)(b + __ffs(z) - 1);
                break;
            }
        }
    }
    // integer numerator of Estimate(Merge(M_S', M_s)) (Alg. 1 line 12)
    uint32_t acc = 0;
    for (int w = lane; w < Jw; w += 32)
        acc += __vsadu4(__vmaxu4(M32[(size_t)s * Jw + w], reinterpret_cast<const uint32_t*>(MS)[w]), 0u);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(IM_FULL, acc, o);
    const int64_t score = acc;
    uint32_t bits = 0, any = 0;
    for (int w = lane; w < W; w += 32) {
        uint32_t d = ~vis[(size_t)s * W + w];
        vis[(size_t)s * W + w] = IM_FULL;
        vd[(size_t)s * W + w].x = IM_FULL;
        delta0[(size_t)s * W + w] = d;
        bits += __popc(d);
        any |= d;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        bits += __shfl_xor_sync(IM_FULL, bits, o);
        any |= __shfl_xor_sync(IM_FULL, any, o);
    }
    (void)off;
    (void)items0;
    if (lane == 0) {
        inS[s] = 1;
        *sigma_count += bits;
        ctr0->changed = any ? 1 : 0;
        if (any) vl0[0] = (int32_t)s;
        rec->vertex = (int32_t)s;
        rec->score = score;
    }
}

struct BfsArgs {
    const int4* items;
    int n_items;
    IterCounters* ctr_next; // zeroed before launch: batch cursor, appends, new bits
    ull* sigma_count;
    const int32_t* off;
    const uint2* fwd;
    const uint32_t* fwdT;
    uint32_t T0;
    const uint32_t* Xs;
    const uint16_t* s12;
    int J;
    uint2* vd;         // {visited R_G(S), new in this level} word pairs: the visited test and both ORs touch one sector
    const uint32_t* din;
    uint32_t* nbits;   // per vertex: which 32-simulation words got new bits in this level
    int ipw;           // items per warp batch (<= 32; fewer when the level is small, to spread it over the SMs)
    const IterCounters* nin;  // non-null: n_items = nin->next_items on the device (pipelined levels), ipw derived here
    int warps_max;
};

// Same level, reworked for memory-level parallelism (the level is bound by dependent random loads):
// the Delta rows of a warp's 32 items are staged in shared memory once (coalesced), so an edge's
// chain is record -> visited word only; edges are taken two per lane (e0, e0 + 32) and both visited
// words are loaded before either is used.  Windows wider than DENSE_WIN go through the warp path.
// live test only for the simulations of the window that are new at u (Delta_u): only those can be new at v
__device__ __forceinline__ uint32_t bfs_word_live(const uint32_t* sX, uint32_t h, uint32_t T, uint32_t cand, int w) {
    uint32_t nv = 0u;
    for (; cand; cand &= cand - 1) {
        const int k = (w << 5) + __ffs(cand) - 1;
        nv |= ((sX[k] ^ h) < T) ? (1u << (k & 31)) : 0u;
    }
    return nv;
}
__device__ __forceinline__ void bfs_sparse(const uint32_t* sX, const uint32_t* dRow, uint32_t h, uint32_t T, int lo, int hi,
                                           int& w0, uint32_t& nv0, uint32_t& nv1) {
    w0 = lo >> 5;
    const int w1 = (hi - 1) >> 5;
    const uint32_t d0 = dRow[w0] & bit_range(lo & 31, w1 != w0 ? 31 : (hi - 1) & 31);
    const uint32_t d1 = w1 != w0 ? dRow[w1] & bit_range(0, (hi - 1) & 31) : 0u;
    nv0 = bfs_word_live(sX, h, T, d0, w0);
    nv1 = bfs_word_live(sX, h, T, d1, w1);
}

// one edge (-> v) with a wide window [lo, hi): new bits = live & Delta_u & ~visited(v) per window word
__device__ __forceinline__ void bfs_dense_edge(uint2* vd, uint32_t* nbits, const uint32_t* sX, const uint32_t* dRow, uint32_t v,
                                               uint32_t h, uint32_t T, int lo, int hi, int W) {
    const int wlo = lo >> 5, whi = (hi - 1) >> 5;
    for (int wb = wlo; wb <= whi; wb += 8) {
        uint32_t nv[8], x[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const int w = wb + k;
            nv[k] = 0u;
            if (w <= whi) {
                const int i0 = max(lo, w << 5), i1 = min(hi, (w << 5) + 32);
                const uint32_t cand = dRow[w] & bit_range(i0 & 31, (i1 - 1) & 31);
                if (cand) nv[k] = bfs_word_live(sX, h, T, cand, w);
            }
        }
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = nv[k] ? __ldcg(&vd[(size_t)v * W + wb + k].x) : 0u;
        uint32_t words = 0u;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint32_t n = nv[k] & ~x[k];
            if (n) {
                atomicOr(reinterpret_cast<ull*>(&vd[(size_t)v * W + wb + k]), ((ull)n << 32) | n);
                words |= 1u << (wb + k);
            }
        }
        if (words) atomicOr(&nbits[v], words);
    }
}

template <bool CONST_T>
__global__ void __launch_bounds__(BLOCK, BFS_MINB) k_bfs_level2(BfsArgs a) {
    constexpr int EP = BFS_EP;  // edges in flight per lane
    extern __shared__ uint32_t sDyn[];
    __shared__ uint32_t sX[1024];
    __shared__ uint16_t sS[4098];
    __shared__ int sSlot[BLOCK / 32][32];
    if (a.nin) {  // the previous compaction's item count, read on the device (no host round trip)
        a.n_items = a.nin->next_items;
        a.ipw = min(32, max(1, a.n_items / a.warps_max));
        if (a.n_items == 0 || (blockIdx.x > 0 && (int64_t)blockIdx.x * (BLOCK / 32) * a.ipw >= a.n_items)) return;
    }
    for (int i = threadIdx.x; i < a.J; i += blockDim.x) sX[i] = a.Xs[i];
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) sS[i] = a.s12[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, W = a.J >> 5;
    uint32_t* sD = sDyn + (size_t)wib * 32 * W;  // Delta rows of this warp's 32 items
    int base = 0, left = 0;  // grabs of 4 batches of ipw items
    for (;;) {
        if (left == 0) {
            if (lane == 0) base = atomicAdd(&a.ctr_next->batch, 4 * a.ipw);
            base = __shfl_sync(IM_FULL, base, 0);
            left = 4;
        } else {
            base += a.ipw;
        }
        --left;
        if (base >= a.n_items) break;
        const int it = base + lane;
        int u = 0, eb = 0, cnt = 0;
        if (lane < a.ipw && it < a.n_items) {
            const int4 I = ld_stream(&a.items[it]);
            u = I.x;
            eb = I.y;
            cnt = I.z - I.y;
        }
        __syncwarp();
        const int nst = (a.ipw * W + 31) & ~31;  // only the batch's ipw rows, whole warp per iteration (the shuffle)
        for (int idx = lane; idx < nst; idx += 32) {
            const int i = min(idx / W, 31), w = idx - (idx / W) * W;
            const int ui = __shfl_sync(IM_FULL, u, i);
            if (idx < a.ipw * W) sD[idx] = base + i < a.n_items ? a.din[(size_t)ui * W + w] : 0u;
        }
        __syncwarp();
        const int incl = warp_incl_scan(cnt, lane);
        const int total = __shfl_sync(IM_FULL, incl, 31);
        const int start = incl - cnt;
        int carry = 0;
        for (int e0 = 0; e0 < total; e0 += 32 * EP) {
            int own[EP], ed[EP];
#pragma unroll
            for (int s = 0; s < EP; s++) {  // owner item of edge e0 + 32 s + lane
                const int b0 = e0 + 32 * s;
                const bool starts = cnt > 0 && start >= b0 && start < b0 + 32;
                if (starts) sSlot[wib][start - b0] = lane;
                const uint32_t smask = __reduce_or_sync(IM_FULL, starts ? (1u << (start - b0)) : 0u);
                __syncwarp();
                const uint32_t below = smask & ((2u << lane) - 1u);
                const int owner = below ? sSlot[wib][31 - __clz(below)] : carry;
                __syncwarp();
                carry = __shfl_sync(IM_FULL, owner, 31);
                const int oeb = __shfl_sync(IM_FULL, eb, owner), ost = __shfl_sync(IM_FULL, start, owner);
                own[s] = owner;
                ed[s] = b0 + lane < total ? oeb + (b0 + lane - ost) : -1;
            }
            uint2 f[EP];
            uint32_t T[EP];
#pragma unroll
            for (int s = 0; s < EP; s++) {
                f[s] = ed[s] >= 0 ? ld_stream(&a.fwd[ed[s]]) : make_uint2(0, 0);
                T[s] = ed[s] >= 0 ? (CONST_T ? a.T0 : ld_stream(&a.fwdT[ed[s]])) : 0u;
            }
            int lo[EP], hi[EP], w0[EP];
            uint32_t nv0[EP], nv1[EP], x0[EP], x1[EP];
            bool dense[EP];
#pragma unroll
            for (int s = 0; s < EP; s++) {
                lo[s] = hi[s] = 0;
                nv0[s] = nv1[s] = 0u;
                w0[s] = 0;
                if (T[s]) edge_window(f[s].y, T[s], sX, sS, a.J, lo[s], hi[s]);
                dense[s] = hi[s] - lo[s] > DENSE_WIN;
                if (!dense[s] && lo[s] < hi[s]) bfs_sparse(sX, sD + own[s] * W, f[s].y, T[s], lo[s], hi[s], w0[s], nv0[s], nv1[s]);
            }
#pragma unroll
            for (int s = 0; s < EP; s++) {  // every edge's visited words in flight
                const size_t r = (size_t)f[s].x * W + w0[s];
                x0[s] = nv0[s] ? __ldcg(&a.vd[r].x) : 0u;
                x1[s] = nv1[s] ? __ldcg(&a.vd[r + 1].x) : 0u;
            }
#pragma unroll
            for (int s = 0; s < EP; s++) {
                const size_t r = (size_t)f[s].x * W + w0[s];
                const uint32_t n0 = nv0[s] & ~x0[s], n1 = nv1[s] & ~x1[s];
                if (n0) atomicOr(reinterpret_cast<ull*>(&a.vd[r]), ((ull)n0 << 32) | n0);  // visited and Delta_out
                if (n1) atomicOr(reinterpret_cast<ull*>(&a.vd[r + 1]), ((ull)n1 << 32) | n1);
                if (n0 | n1) atomicOr(&a.nbits[f[s].x], (n0 ? 1u << w0[s] : 0u) | (n1 ? 2u << w0[s] : 0u));
            }
            // wide windows (> DENSE_WIN simulations, e.g. weighted cascade with small in-degree): each lane walks
            // its own edge's window words, 8 at a time, testing only the Delta_u simulations in them; the
            // visited words of the 8 are loaded together (independent loads in flight, not one per word)
#pragma unroll 1
            for (int s = 0; s < EP; s++) {
                if (!dense[s]) continue;
                const uint32_t* dRow = sD + own[s] * W;
                bfs_dense_edge(a.vd, a.nbits, sX, dRow, f[s].x, f[s].y, T[s], lo[s], hi[s], W);
            }
        }
    }
}

// Next BFS frontier: every vertex with new bits in this level (nbits != 0).  Counts the new
// (vertex, simulation) pairs (popcount of the OR-ed Delta words) into sigma, lists the vertex (to
// clear its Delta after the next level), emits its out-edge items (long rows of a hash-sorted
// graph go to k_slices_big) and clears nbits for the next level.
// VDM (the selection BFS): the level left its new bits in vd[].y; they move to the next level's
// Delta rows (dout), the visited words are copied to vis (R_G(S) for every other kernel) and vd[].y
// is cleared.  Otherwise (the evaluator) dout already holds them.
template <bool VDM>
__global__ void k_bfs_compact(int32_t n, int J, int slice_min, uint32_t* __restrict__ nbits, uint32_t* __restrict__ dout,
                              uint2* __restrict__ vd, uint32_t* __restrict__ vis,
                              const int32_t* __restrict__ off, int32_t* __restrict__ vl, int4* __restrict__ items,
                              int32_t* __restrict__ big, IterCounters* ctr, ull* sigma_count) {
    const int lane = threadIdx.x & 31, W = J >> 5;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    ull newbits = 0;
    // CU vertex groups per block iteration, loaded up front (independent loads in flight): a level
    // with few new vertices costs one pass over nbits, not a dependent load per 256 vertices
    for (int64_t base0 = (int64_t)blockIdx.x * blockDim.x * CU; base0 < n; base0 += stride * CU) {
      uint32_t bb[CU];
      bool anyb = false;
#pragma unroll
      for (int k = 0; k < CU; k++) {
          const int64_t v = base0 + (int64_t)k * blockDim.x + threadIdx.x;
          bb[k] = v < n ? nbits[v] : 0u;
          anyb |= bb[k] != 0u;
      }
      if (!__syncthreads_or(anyb)) continue;
      // every group of this iteration at once: new bits moved / counted and row bounds loaded for
      // all of the thread's vertices, then one block-wide reservation (frontier list, items, big rows)
      int rbk[CU], rdk[CU];
      int t_items = 0, t_changed = 0, t_big = 0;
      long long t_edges = 0;
#pragma unroll
      for (int k = 0; k < CU; k++) {
          rbk[k] = rdk[k] = 0;
          const uint32_t b = bb[k];
          if (!b) continue;
          const int64_t v = base0 + (int64_t)k * blockDim.x + threadIdx.x;
          nbits[v] = 0u;
          for (uint32_t t = b; t; t &= t - 1) {
              const size_t i = (size_t)v * W + (__ffs(t) - 1);
              if (VDM) {
                  const uint2 pr = vd[i];
                  dout[i] = pr.y;
                  vis[i] = pr.x;
                  vd[i] = make_uint2(pr.x, 0u);
                  newbits += __popc(pr.y);
              } else {
                  newbits += __popc(dout[i]);
              }
          }
          rbk[k] = off[v];
          rdk[k] = off[v + 1] - rbk[k];
      }
#pragma unroll
      for (int k = 0; k < CU; k++)
          if (bb[k]) {
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
      int p = pos + ci - t_items, cp = cpos + cc - t_changed, bp = bpos + cb - t_big;
#pragma unroll
      for (int k = 0; k < CU; k++) {
          if (!bb[k]) continue;
          const int v = (int)(base0 + (int64_t)k * blockDim.x + threadIdx.x);
          vl[cp++] = v;
          const int rb = rbk[k], rd = rdk[k];
          if (rd > slice_min) big[bp++] = v;
          else
              for (int s0 = rb; s0 < rb + rd; s0 += SEG) items[p++] = make_int4(v, s0, min(s0 + SEG, rb + rd), 0);
      }
    }
    newbits = __reduce_add_sync(IM_FULL, (uint32_t)newbits);
    if (lane == 0 && newbits) {
        atomicAdd(&ctr->new_bits, newbits);
        atomicAdd(sigma_count, newbits);
    }
}

// Work items of a BFS frontier: for every vertex v of vl, its out-edges; a long row of a
// hash-sorted graph is queued for k_slices_big (im_sweep.cu), which emits only the slices whose
// candidate windows can meet a simulation of Delta_v.
__global__ void k_bfs_items(int slice_min, const int32_t* __restrict__ vl, const int32_t* __restrict__ off,
                            int4* __restrict__ items, int32_t* __restrict__ big, IterCounters* ctr) {
    const int lane = threadIdx.x & 31;
    const int nv = ctr->changed;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < nv; base += stride) {
        int64_t i = base + threadIdx.x;
        int v = i < nv ? vl[i] : 0, rb = 0, rd = 0, ns = 0;
        bool isbig = false;
        if (i < nv) {
            rb = off[v];
            rd = off[v + 1] - rb;
            isbig = rd > slice_min;
            ns = isbig ? 0 : (rd + SEG - 1) / SEG;
        }
        uint32_t bmask = __ballot_sync(IM_FULL, isbig);
        int ninc = warp_incl_scan(ns, lane);
        long long esum = isbig ? 0 : rd;
#pragma unroll
        for (int o = 16; o; o >>= 1) esum += __shfl_xor_sync(IM_FULL, esum, o);
        BlockTotals wt{ninc, 0, __popc(bmask), (unsigned long long)esum};
        int pos, cpos, bpos;
        block_reserve<BLOCK / 32>(wt, lane, threadIdx.x >> 5, &ctr->next_items, nullptr, &ctr->next_edges, &ctr->big, pos,
                                  cpos, bpos);
        int p = pos + ninc - ns;
        for (int s0 = rb; s0 < rb + rd && ns; s0 += SEG) items[p++] = make_int4(v, s0, min(s0 + SEG, rb + rd), 0);
        if (isbig) big[bpos + __popc(bmask & ((1u << lane) - 1u))] = v;
    }
}

__global__ void k_bfs_clear(int n_v, int W, const int32_t* __restrict__ vl, uint32_t* __restrict__ delta,
                            const IterCounters* nin = nullptr) {
    if (nin) n_v = nin->changed;  // pipelined levels: the frontier size on the device
    int64_t total = (int64_t)n_v * W, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride)
        delta[(size_t)vl[i / W] * W + (i % W)] = 0u;
}

// ============================================================ a8: error check (Alg. 1 lines 12, 15-27)
// J: this rank's simulations (M_S' merge); Jt: all simulations (Eq. 2 and sigma; == J unless sharded)
__global__ void k_error_check(int32_t J, int32_t Jt, int k, int K, double eps_l, double eps_g, const uint32_t* __restrict__ M32,
                              uint8_t* MS, const IterCounters* ctr_unused, const ull* sigma_count, double* varsigma,
                              StepDev* rec) {
    (void)ctr_unused;
    const int lane = threadIdx.x, Jw = J >> 2;
    __shared__ int sRebuild;
    if (lane == 0) {
        double e = exp2((double)rec->score / (double)Jt) / 0.77351;
        ull cnt = *sigma_count;
        double sigma = (double)cnt / (double)Jt;
        double delta = sigma - *varsigma;
        double err_l = delta != 0.0 ? fabs((e - delta) / delta) : (double)INFINITY;
        double err_g = fabs((e - delta) / sigma);
        int rebuild = !(err_l < eps_l || err_g < eps_g);
        rec->e = e;
        rec->sigma_count = (int64_t)cnt;
        rec->sigma = sigma;
        rec->delta = delta;
        rec->err_l = err_l;
        rec->err_g = err_g;
        rec->rebuilt = rebuild;
        rec->executed = rebuild && k < K - 1;
        if (rebuild && k < K - 1) *varsigma = sigma;
        sRebuild = rebuild;
    }
    __syncwarp();
    const uint32_t s = (uint32_t)rec->vertex;
    uint32_t* MS32 = reinterpret_cast<uint32_t*>(MS);
    if (!sRebuild) {  // line 19: M_S' <- Merge(M_S', M_s) (Eq. 3)
        for (int w = lane; w < Jw; w += 32) MS32[w] = __vmaxu4(MS32[w], M32[(size_t)s * Jw + w]);
    } else if (k < K - 1) {  // line 26: M_S' <- zeros
        for (int w = lane; w < Jw; w += 32) MS32[w] = 0u;
    }
}

__global__ void k_gather_rows(int64_t nrows, int32_t J, const int32_t* __restrict__ rows, const uint8_t* __restrict__ M,
                              uint8_t* __restrict__ out) {
    int64_t total = nrows * J, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride)
        out[i] = M[(size_t)rows[i / J] * J + (i % J)];
}

// ============================================================ launchers


cudaError_t launch_estimate(Ctx& c, double* out) {
    k_estimate<false><<<grid_for(c, (int64_t)c.n * 32), BLOCK, 0, c.stream>>>(c.n, c.J, reinterpret_cast<const uint32_t*>(c.M), out, nullptr);
    return LAUNCHED(c);
}
cudaError_t launch_estimate_sums(Ctx& c, int32_t* sums) {
    k_estimate<true><<<grid_for(c, (int64_t)c.n * 32), BLOCK, 0, c.stream>>>(c.n, c.J, reinterpret_cast<const uint32_t*>(c.M), nullptr, sums);
    return LAUNCHED(c);
}
cudaError_t launch_estimate_fin(Ctx& c, const int32_t* sums, double* out) {
    k_estimate_fin<<<grid_for(c, c.n), BLOCK, 0, c.stream>>>(c.n, c.Jt, sums, out);
    return LAUNCHED(c);
}
// lanes per vertex and chunks per lane of the list pass: L = max(min(8, pow2 >= J/16), J/64), C <= AC
static void argmax_geometry(const Ctx& c, int& L, int& C) {
    const int nch = c.J >> 4;
    L = 1;
    while (L < 8 && L < nch) L <<= 1;
    while (L * AC < nch) L <<= 1;
    C = (nch + L - 1) / L;
}
static int hist_shift(const Ctx& c) {
    int sh = 0;
    while (((32 * c.Jt) >> sh) >= HIST_BINS) sh++;  // gains of all J_total simulations
    return sh;
}

// full pass: exact argmax into c.key (zeroed here) + stored gains + candidate list for later steps.
// Sharded: the pass leaves packed local values in c.gain; the caller allreduces them and calls
// launch_argmax_full_finish, which decodes them (k_argmax_decode) before theta / list.
cudaError_t launch_argmax_full(Ctx& c, bool pool) {
    int L, C;
    argmax_geometry(c, L, C);
    const int sh = hist_shift(c);
    cudaError_t e = cudaMemsetAsync(c.key, 0, sizeof(ull), c.stream);
    if (!e) e = cudaMemsetAsync(c.hist, 0, HIST_BINS * sizeof(uint32_t), c.stream);
    if (!e) e = cudaMemsetAsync(c.lcount, 0, 2 * sizeof(int), c.stream);
    if (e) return e;
    return launch_argmax_tma(c, pool, L, C, sh);  // TMA-bulk streaming pass (im_stream.cu)
}
cudaError_t launch_argmax_full_finish(Ctx& c, int T) {
    const int sh = hist_shift(c);
    cudaError_t e;
    k_theta<<<1, 32, 0, c.stream>>>(c.hist, sh, T, c.lcount + 1);
    if ((e = LAUNCHED(c))) return e;
    const int nb = grid_for(c, c.n);  // <= LIST_BLOCKS(c)
    k_list_count<<<nb, BLOCK, 0, c.stream>>>(c.n, c.gain, c.lcount + 1, c.bcount);
    if ((e = LAUNCHED(c))) return e;
    k_list_write<<<nb, BLOCK, 0, c.stream>>>(c.n, c.gain, c.lcount + 1, c.bcount, c.list, c.lcount, 0);
    return LAUNCHED(c);
}
// sharded full pass: after the reduce-scatter, c.gslice[i] is the summed packed value of
// vertex v0 + i; decode it into the local argmax key, the stored gains of the slice and the histogram
cudaError_t launch_argmax_slice_decode(Ctx& c, int64_t v0, int nv) {
    if (nv <= 0) return cudaSuccess;
    k_argmax_decode<<<grid_for(c, nv), BLOCK, 0, c.stream>>>(nv, nullptr, nullptr, c.gslice, c.gslice, c.key, c.hist,
                                                             hist_shift(c), v0);
    return LAUNCHED(c);
}
// theta from the summed histogram, then this rank's candidate list (its slice's vertices with gain >= theta,
// ascending) into c.llist, its length into c.lcount[0]
cudaError_t launch_argmax_slice_list(Ctx& c, int T, int64_t v0, int nv) {
    const int sh = hist_shift(c);
    k_theta<<<1, 32, 0, c.stream>>>(c.hist, sh, T, c.lcount + 1);
    cudaError_t e = LAUNCHED(c);
    if (e || nv <= 0) return e;
    const int nb = grid_for(c, nv);
    k_list_count<<<nb, BLOCK, 0, c.stream>>>(nv, c.gslice, c.lcount + 1, c.bcount);
    if ((e = LAUNCHED(c))) return e;
    k_list_write<<<nb, BLOCK, 0, c.stream>>>(nv, c.gslice, c.lcount + 1, c.bcount, c.llist, c.lcount, v0);
    return LAUNCHED(c);
}
__global__ void k_set_count(int* p, int v) { *p = v; }
cudaError_t launch_set_count(Ctx& c, int* p, int v) {
    k_set_count<<<1, 1, 0, c.stream>>>(p, v);
    return LAUNCHED(c);
}
__global__ void k_list_pad(int32_t* list, const int* count, int cap) {
    for (int i = *count + blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x) list[i] = -1;
}
cudaError_t launch_list_pad(Ctx& c, int32_t* list, const int* count, int cap) {
    k_list_pad<<<grid_for(c, cap), BLOCK, 0, c.stream>>>(list, count, cap);
    return LAUNCHED(c);
}

// lazy step: exact gains over the candidate list only; valid iff best gain >= theta (checked by the host).
// Sharded: packed local values go to c.lval; the caller allreduces them and calls launch_argmax_list_finish.
cudaError_t launch_argmax_list(Ctx& c, int list_len) {
    int L, C;
    argmax_geometry(c, L, C);
    cudaError_t e = cudaMemsetAsync(c.key, 0, sizeof(ull), c.stream);
    if (e) return e;
    int g = grid_for(c, (int64_t)list_len * L / 2);
    const uint4* M16 = reinterpret_cast<const uint4*>(c.M);
    if (c.ar)
        k_argmax<true, true, true><<<g, BLOCK, 0, c.stream>>>(c.n, c.J, L, C, M16, c.MS, c.vis, c.key, c.lval, nullptr, 0, c.list, c.lcount);
    else
        k_argmax<true, true><<<g, BLOCK, 0, c.stream>>>(c.n, c.J, L, C, M16, c.MS, c.vis, c.key, nullptr, nullptr, 0, c.list, c.lcount);
    return LAUNCHED(c);
}
cudaError_t launch_argmax_list_finish(Ctx& c, int list_len) {
    if (!c.ar) return cudaSuccess;
    k_argmax_decode<<<grid_for(c, list_len), BLOCK, 0, c.stream>>>(list_len, c.list, c.lcount, c.lval, nullptr, c.key, nullptr, 0, 0);
    return LAUNCHED(c);
}
cudaError_t launch_seed_start(Ctx& c, int k) {
    (void)k;
    k_seed_start<<<1, 32, 0, c.stream>>>(c.n, c.J, c.key, reinterpret_cast<const uint32_t*>(c.M), c.MS, c.inS, c.vis, c.vd,
                                          c.delta[0], c.off, c.bitems[0], c.bvl[0], &c.ctr[0], c.sigma_count, c.rec);
    return LAUNCHED(c);
}
cudaError_t launch_bfs_level(Ctx& c, int cur, int n_items, uint32_t tag, bool piped) {
    (void)tag;
    BfsArgs a;
    a.items = c.bitems[cur];
    a.n_items = n_items;
    a.nin = piped ? &c.ctr[cur] : nullptr;
    a.ctr_next = &c.ctr[cur ^ 1];
    a.sigma_count = c.sigma_count;
    a.off = c.off;
    a.fwd = c.fwd;
    a.fwdT = c.fwdT;
    a.T0 = c.T0;
    a.Xs = c.Xs;
    a.s12 = c.s12;
    a.J = c.J;
    a.vd = c.vd;
    a.din = c.delta[cur];
    a.nbits = c.nbits;
    // items per warp batch: 32, or fewer so that a small level still occupies every SM (each edge is a
    // chain of dependent loads, so a level is latency-bound unless many warps are in flight)
    const int64_t warps_max = (int64_t)c.max_blocks_bfs2 * (BLOCK / 32);
    a.warps_max = (int)warps_max;
    a.ipw = (int)std::min<int64_t>(32, std::max<int64_t>(1, n_items / warps_max));
    int64_t want = ((int64_t)n_items + (int64_t)a.ipw * (BLOCK / 32) - 1) / ((int64_t)a.ipw * (BLOCK / 32));
    {
        const size_t smem = (size_t)BLOCK * (c.J >> 5) * sizeof(uint32_t);
        int grid = piped ? c.max_blocks_bfs2 : (int)(want < 1 ? 1 : (want > c.max_blocks_bfs2 ? c.max_blocks_bfs2 : want));
        if (c.constT) k_bfs_level2<true><<<grid, BLOCK, smem, c.stream>>>(a);
        else k_bfs_level2<false><<<grid, BLOCK, smem, c.stream>>>(a);
    }
    cudaError_t e = LAUNCHED(c);
    if (e) return e;
    const int nxt = cur ^ 1;
    k_bfs_compact<true><<<grid_for(c, c.n), BLOCK, 0, c.stream>>>(c.n, c.J, c.sorted_h ? c.slice_min_bfs : INT_MAX, c.nbits, c.delta[nxt], c.vd, c.vis, c.off, c.bvl[nxt],
                                                            c.bitems[nxt], c.big, &c.ctr[nxt], c.sigma_count);
    if ((e = LAUNCHED(c))) return e;
    if (!c.sorted_h) return e;
    return launch_slices_big(c, c.big, c.delta[nxt], c.off, c.fwd, c.bitems[nxt], &c.ctr[nxt], true);
}
cudaError_t launch_bfs_items(Ctx& c, int buf) {
    k_bfs_items<<<c.num_sms * 4, BLOCK, 0, c.stream>>>(c.sorted_h ? c.slice_min_bfs : INT_MAX, c.bvl[buf], c.off, c.bitems[buf], c.big, &c.ctr[buf]);
    cudaError_t e = LAUNCHED(c);
    if (e || !c.sorted_h) return e;
    return launch_slices_big(c, c.big, c.delta[buf], c.off, c.fwd, c.bitems[buf], &c.ctr[buf], true);
}
// the same compaction / item / clear kernels on caller-chosen buffers, unsorted rows (evaluator, im_eval.cu)
cudaError_t launch_bfs_compact_raw(Ctx& c, int J, uint32_t* nbits, const uint32_t* dout, int32_t* vl, int4* items,
                                   IterCounters* ctr, ull* count) {
    k_bfs_compact<false><<<grid_for(c, c.n), BLOCK, 0, c.stream>>>(c.n, J, INT_MAX, nbits, const_cast<uint32_t*>(dout), nullptr, nullptr,
                                                                   c.off, vl, items, nullptr, ctr, count);
    return LAUNCHED(c);
}
cudaError_t launch_bfs_items_raw(Ctx& c, const int32_t* vl, int4* items, IterCounters* ctr) {
    k_bfs_items<<<c.num_sms * 4, BLOCK, 0, c.stream>>>(INT_MAX, vl, c.off, items, nullptr, ctr);
    return LAUNCHED(c);
}
cudaError_t launch_bfs_clear_raw(Ctx& c, int n_v, int W, const int32_t* vl, uint32_t* delta) {
    k_bfs_clear<<<grid_for(c, (int64_t)n_v * W), BLOCK, 0, c.stream>>>(n_v, W, vl, delta);
    return LAUNCHED(c);
}

cudaError_t launch_bfs_clear(Ctx& c, int cur, int n_v, bool piped) {
    int W = c.J >> 5;
    if (piped)  // the frontier size is read on the device from the counters that produced it
        k_bfs_clear<<<c.num_sms * 4, BLOCK, 0, c.stream>>>(0, W, c.bvl[cur], c.delta[cur], &c.ctr[cur]);
    else
        k_bfs_clear<<<grid_for(c, (int64_t)n_v * W), BLOCK, 0, c.stream>>>(n_v, W, c.bvl[cur], c.delta[cur]);
    return LAUNCHED(c);
}
cudaError_t launch_error_check(Ctx& c, int k, int K, double eps_l, double eps_g) {
    k_error_check<<<1, 32, 0, c.stream>>>(c.J, c.Jt, k, K, eps_l, eps_g, reinterpret_cast<const uint32_t*>(c.M), c.MS, nullptr,
                                          c.ar ? c.sigma_g : c.sigma_count, c.varsigma, c.rec);
    return LAUNCHED(c);
}
cudaError_t launch_gather_rows(Ctx& c, const int32_t* rows, int64_t nrows, uint8_t* out) {
    k_gather_rows<<<grid_for(c, nrows * c.J), BLOCK, 0, c.stream>>>(nrows, c.J, rows, c.M, out);
    return LAUNCHED(c);
}

int occupancy_bfs(int* blocks_per_sm) {  // grid cap of the evaluator's level kernel (persistent; any grid is correct)
    *blocks_per_sm = 8;
    return 0;
}
// k_bfs_level2 for this J (dynamic shared memory: the Delta rows of every warp's 32 items)
int occupancy_bfs2(int J, int* blocks_per_sm) {
    const int smem = BLOCK * (J >> 5) * (int)sizeof(uint32_t);
    cudaError_t e = cudaFuncSetAttribute(k_bfs_level2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (!e) e = cudaFuncSetAttribute(k_bfs_level2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e) return (int)e;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_bfs_level2<true>, BLOCK, smem);
}

}  // namespace im
