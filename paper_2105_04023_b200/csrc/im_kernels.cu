// im_kernels.cu -- sm_100a kernels of the hot path.
//
//   k_validate / k_const_check / k_edge_prep / k_transpose / k_items   a0 edge prep (Eq. 4-5, Sec. 3.3)
//   k_init_registers                                                   a2 register init (Alg. 1 lines 2-5)
//   k_sweep<...>                                                       a3+a4 Simulate sweeps (Alg. 2)
//   k_estimate                                                         a5 Eq. 2
//   k_argmax / k_seed_start / k_bfs_level / k_bfs_clear / k_error_check a6-a8 Alg. 1 loop body
//
// No tensor cores: the path is integer gather / byte-max, bound by HBM and the
// INT pipes.  All work-list kernels are persistent (grid <= resident blocks)
// and pull 32-item batches from a device cursor.
#include <cub/device/device_scan.cuh>

#include "im_device.cuh"
#include "im_internal.h"

namespace im {

// ============================================================ a0: edge prep
__global__ void k_validate(int32_t n, int64_t m, const int32_t* __restrict__ off, const int32_t* __restrict__ tgt,
                           const float* __restrict__ prob, int* flags) {
    int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    int f = 0;
    if (tid == 0) {
        if (off[0] != 0) f |= 1;
        if ((int64_t)off[n] != m) f |= 1;
    }
    for (int64_t i = tid; i < n; i += stride)
        if (off[i] > off[i + 1]) f |= 1;
    for (int64_t e = tid; e < m; e += stride) {
        int32_t v = tgt[e];
        if (v < 0 || v >= n) f |= 2;
        float w = prob[e];
        if (!(w >= 0.0f && w <= 1.0f)) f |= 4;  // also rejects NaN
    }
    if (f) atomicOr(flags, f);
}

__global__ void k_const_check(int64_t m, const float* __restrict__ prob, int* flag) {
    int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    uint32_t p0 = __float_as_uint(prob[0]);
    bool diff = false;
    for (int64_t e = tid; e < m; e += stride) diff |= __float_as_uint(prob[e]) != p0;
    if (__any_sync(IM_FULL, diff) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__device__ __forceinline__ int32_t edge_source(const int32_t* __restrict__ off, int32_t n, int64_t e) {
    int32_t lo = 0, hi = n - 1;  // largest u with off[u] <= e
    while (lo < hi) {
        int32_t mid = (lo + hi + 1) >> 1;
        if ((int64_t)off[mid] <= e) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// h(u,v) (Eq. 4) and T_e (Eq. 5) per forward edge; in-degree histogram for the transpose
__global__ void k_edge_prep(int32_t n, int64_t m, const int32_t* __restrict__ off, const int32_t* __restrict__ tgt,
                            const float* __restrict__ prob, uint2* __restrict__ fwd, uint32_t* __restrict__ fwdT,
                            int32_t* __restrict__ indeg) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += stride) {
        int32_t u = edge_source(off, n, e), v = tgt[e];
        fwd[e] = make_uint2((uint32_t)v, edge_hash((uint32_t)u, (uint32_t)v));
        if (fwdT) fwdT[e] = live_threshold(prob[e]);
        atomicAdd(&indeg[v], 1);
    }
}

__global__ void k_transpose(int32_t n, int64_t m, const int32_t* __restrict__ off, const uint2* __restrict__ fwd,
                            const uint32_t* __restrict__ fwdT, const int32_t* __restrict__ roff, int32_t* __restrict__ cursor,
                            uint2* __restrict__ rev, uint32_t* __restrict__ revT) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += stride) {
        int32_t u = edge_source(off, n, e);
        uint2 f = fwd[e];
        int32_t pos = roff[f.x] + atomicAdd(&cursor[f.x], 1);
        rev[pos] = make_uint2((uint32_t)u, f.y);
        if (revT) revT[pos] = fwdT[e];
    }
}

__global__ void k_nseg(int32_t n, const int32_t* __restrict__ offs, int32_t* __restrict__ nseg) {
    int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) nseg[v] = (offs[v + 1] - offs[v] + SEG - 1) / SEG;
    if (v == n) nseg[n] = 0;
}

__global__ void k_fill_items(int32_t n, const int32_t* __restrict__ offs, const int32_t* __restrict__ base,
                             int4* __restrict__ items) {
    int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    int32_t b = offs[v], e = offs[v + 1], p = base[v];
    for (int32_t s = b; s < e; s += SEG) items[p++] = make_int4(v, s, min(s + SEG, e), 0);
}

// ============================================================ a2: register init
// M_v[jj] = clz(Murmur3(v, seed_V) xor Murmur3(perm[jj], seed_J)), clz(0) = 32 (Alg. 1 lines 2-5; R5, R6)
__global__ void k_init_registers(int32_t n, int32_t J, uint32_t seedV, uint32_t seedJ, const int32_t* __restrict__ perm,
                                 uint4* __restrict__ M) {
    __shared__ uint32_t HJ[1024];
    for (int j = threadIdx.x; j < J; j += blockDim.x) HJ[j] = murmur_word((uint32_t)perm[j], seedJ);
    __syncthreads();
    const int cpr = J >> 4;  // 16-byte chunks per row
    const int64_t total = (int64_t)n * cpr, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += stride) {
        uint32_t v = (uint32_t)(idx / cpr);
        int c = (int)(idx - (int64_t)v * cpr) << 4;
        uint32_t hv = murmur_word(v, seedV);
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint32_t x = 0;
#pragma unroll
            for (int b = 0; b < 4; b++) x |= (uint32_t)__clz(hv ^ HJ[c + 4 * q + b]) << (8 * b);
            w[q] = x;
        }
        M[idx] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// ============================================================ a3/a4: Simulate sweeps
// Alg. 2 realised as an edge-parallel, in-place pass over the in-edges of
// the vertices whose registers changed in the previous sweep (all vertices in sweep 1):
// for in-edge (u,v) of such a v, every simulation j with (X_j xor h_uv) < T_uv and u not in
// R_S[j] gets M_u[j] <- max(M_u[j], M_v[j]) (line 'update', pull direction R9).  Edges of
// Gamma^-(L) into vertices outside L are skipped: pulling an unchanged row is a no-op.  The
// fixpoint is unique, so the in-place order reaches exactly the oracle's registers.
struct SweepArgs {
    const int4* items;
    int n_items;
    IterCounters* ctr_next; // zeroed before launch: batch cursor + appends for the next sweep
    const int32_t* roff;
    const uint2* rev;
    const uint32_t* revT;
    uint32_t T0;
    const uint32_t* Xs;
    const uint16_t* s12;
    int J;
    uint32_t* M32;
    const uint32_t* vis;
    const ull* chg_in;
    ull* chg_out;
    uint32_t tag_in, tag_out;
    int4* next_items;
};

template <bool BLOCKED>
__device__ __forceinline__ uint32_t pull_word(const SweepArgs& a, const uint32_t* sX, uint32_t u, uint32_t v, int w,
                                              uint32_t h, uint32_t T, int lo, int hi) {
    uint32_t live = 0;
#pragma unroll
    for (int b = 0; b < 4; b++) {
        int i = 4 * w + b;
        bool ok = (i >= lo) & (i < hi) & ((sX[i] ^ h) < T);
        live |= ok ? (0xFFu << (8 * b)) : 0u;
    }
    if (BLOCKED && live) {
        uint32_t vb = (a.vis[(size_t)u * (a.J >> 5) + (w >> 3)] >> ((w & 7) << 2)) & 0xFu;
        live &= ~expand4(vb);
    }
    if (!live) return 0u;
    const int Jw = a.J >> 2;
    uint32_t mv = __ldcg(&a.M32[(size_t)v * Jw + w]) & live;
    if (!mv) return 0u;
    return atomic_vmax4(&a.M32[(size_t)u * Jw + w], mv) ? (1u << (w >> 3)) : 0u;
}

template <bool CONST_T, bool BLOCKED, bool FILTER>
__global__ void __launch_bounds__(BLOCK) k_sweep(SweepArgs a) {
    __shared__ uint32_t sX[1024];
    __shared__ uint16_t sS[4098];
    __shared__ int sSlot[BLOCK / 32][32];
    for (int i = threadIdx.x; i < a.J; i += blockDim.x) sX[i] = a.Xs[i];
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) sS[i] = a.s12[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int J = a.J;

    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&a.ctr_next->batch, 32);
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
            if (FILTER) {
                ull w = a.chg_in[v];
                vbits = ((uint32_t)(w >> 32) == a.tag_in) ? (uint32_t)w : 0u;
                if (!vbits) cnt = 0;
            }
        }
        int incl = warp_incl_scan(cnt, lane);
        int total = __shfl_sync(IM_FULL, incl, 31);
        int start = incl - cnt;
        int carry = 0;
        for (int e0 = 0; e0 < total; e0 += 32) {
            // owner item of edge slot e0+lane: the last non-empty item starting at or before it
            bool starts = cnt > 0 && start >= e0 && start < e0 + 32;
            if (starts) sSlot[wib][start - e0] = lane;
            uint32_t smask = __reduce_or_sync(IM_FULL, starts ? (1u << (start - e0)) : 0u);
            __syncwarp();
            uint32_t below = smask & ((2u << lane) - 1u);
            int owner = below ? sSlot[wib][31 - __clz(below)] : carry;
            __syncwarp();
            carry = __shfl_sync(IM_FULL, owner, 31);
            int ov = __shfl_sync(IM_FULL, v, owner);
            int oeb = __shfl_sync(IM_FULL, eb, owner);
            int ost = __shfl_sync(IM_FULL, start, owner);
            uint32_t obits = __shfl_sync(IM_FULL, vbits, owner);
            int idx = e0 + lane;

            uint32_t u = 0, h = 0, T = 0, chg = 0;
            int lo = 0, hi = 0;
            bool dense = false;
            if (idx < total) {
                int e = oeb + (idx - ost);
                uint2 r = a.rev[e];
                u = r.x;
                h = r.y;
                T = CONST_T ? a.T0 : a.revT[e];
                if (T) {
                    edge_window(h, T, sX, sS, J, lo, hi);
                    if (FILTER && lo < hi && !(obits & bit_range(lo >> 5, (hi - 1) >> 5))) hi = lo;
                    if (hi - lo > DENSE_WIN) {
                        dense = true;
                    } else if (lo < hi) {
                        for (int w = lo >> 2; w <= (hi - 1) >> 2; ++w) chg |= pull_word<BLOCKED>(a, sX, u, (uint32_t)ov, w, h, T, lo, hi);
                    }
                }
            }
            uint32_t wmask = __ballot_sync(IM_FULL, lo < hi);
            if (lane == 0 && wmask) atomicAdd(&a.ctr_next->win_edges, (ull)__popc(wmask));
            // wide windows (e.g. w close to 1): the whole warp walks the window, one word per lane
            uint32_t dmask = __ballot_sync(IM_FULL, dense);
            while (dmask) {
                int l = __ffs(dmask) - 1;
                dmask &= dmask - 1;
                uint32_t du = __shfl_sync(IM_FULL, u, l), dh = __shfl_sync(IM_FULL, h, l), dT = __shfl_sync(IM_FULL, T, l);
                int dlo = __shfl_sync(IM_FULL, lo, l), dhi = __shfl_sync(IM_FULL, hi, l);
                uint32_t dv = (uint32_t)__shfl_sync(IM_FULL, ov, l);
                uint32_t c = 0;
                for (int w = (dlo >> 2) + lane; w <= (dhi - 1) >> 2; w += 32) c |= pull_word<BLOCKED>(a, sX, du, dv, w, dh, dT, dlo, dhi);
                c = __reduce_or_sync(IM_FULL, c);
                if (lane == l) chg |= c;
            }
            // record the change of u: chunk bits under this sweep's tag; the first recorder appends u's items
            bool first = false;
            if (chg) {
                ull* p = &a.chg_out[u];
                ull old = __ldcg(p);
                for (;;) {
                    uint32_t otag = (uint32_t)(old >> 32), ob = (uint32_t)old;
                    bool same = otag == a.tag_out;
                    uint32_t nb = same ? (ob | chg) : chg;
                    if (same && nb == ob) break;
                    ull want = ((ull)a.tag_out << 32) | nb;
                    ull prev = atomicCAS(p, old, want);
                    if (prev == old) {
                        first = !same;
                        break;
                    }
                    old = prev;
                }
            }
            int rd = 0, ns = 0;
            if (first) {
                int rb = a.roff[u];
                rd = a.roff[u + 1] - rb;
                ns = (rd + SEG - 1) / SEG;
            }
            int ninc = warp_incl_scan(ns, lane);
            int ntot = __shfl_sync(IM_FULL, ninc, 31);
            uint32_t fmask = __ballot_sync(IM_FULL, first);
            if (fmask) {
                int pos = 0;
                if (lane == 31) {
                    if (ntot) pos = atomicAdd(&a.ctr_next->next_items, ntot);
                    atomicAdd(&a.ctr_next->changed, __popc(fmask));
                }
                pos = __shfl_sync(IM_FULL, pos, 31);
                long long esum = rd;
#pragma unroll
                for (int o = 16; o; o >>= 1) esum += __shfl_xor_sync(IM_FULL, esum, o);
                if (lane == 0 && esum) atomicAdd(&a.ctr_next->next_edges, (ull)esum);
                if (ns) {
                    int rb = a.roff[u], re = rb + rd, p = pos + ninc - ns;
                    for (int s = rb; s < re; s += SEG) a.next_items[p++] = make_int4((int)u, s, min(s + SEG, re), 0);
                }
            }
        }
    }
}

// ============================================================ a5: Eq. 2 estimate
__global__ void k_estimate(int32_t n, int32_t J, const uint32_t* __restrict__ M32, double* __restrict__ out) {
    const int lane = threadIdx.x & 31, Jw = J >> 2;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
        uint32_t s = 0;
        for (int w = lane; w < Jw; w += 32) s += __vsadu4(__ldcs(&M32[v * Jw + w]), 0u);
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(IM_FULL, s, o);
        if (lane == 0) out[v] = exp2((double)s / (double)J) / 0.77351;
    }
}

// ============================================================ a6: greedy argmax
// score_v = sum_j max(M_S'[j], M_v[j]) over the pool (R14); key = score<<32 | (2^32-1-v) so the
// 64-bit max picks the lowest id among equal scores.  Also the lowest id not in S (pool-empty fallback).
template <bool POOL>
__global__ void __launch_bounds__(BLOCK) k_argmax(int32_t n, int32_t J, const uint32_t* __restrict__ M32,
                                                  const uint8_t* __restrict__ MS, const uint32_t* __restrict__ vis,
                                                  const uint8_t* __restrict__ inS, ull* key, int* first) {
    __shared__ uint32_t sMS[256];
    __shared__ ull sKey[BLOCK / 32];
    __shared__ int sFirst[BLOCK / 32];
    const int Jw = J >> 2, W = J >> 5;
    for (int i = threadIdx.x; i < Jw; i += blockDim.x) sMS[i] = reinterpret_cast<const uint32_t*>(MS)[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    ull best = 0;
    int fst = 0x7FFFFFFF;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
        bool inpool = true;
        if (POOL) {
            bool full = true;
            for (int w = lane; w < W; w += 32) full &= __ldcs(&vis[v * W + w]) == IM_FULL;
            inpool = !__all_sync(IM_FULL, full);
        }
        if (inpool) {
            uint32_t s = 0;
            for (int w = lane; w < Jw; w += 32) s += __vsadu4(__vmaxu4(__ldcs(&M32[v * Jw + w]), sMS[w]), 0u);
#pragma unroll
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(IM_FULL, s, o);
            ull k = ((ull)s << 32) | (ull)(0xFFFFFFFFu - (uint32_t)v);
            best = k > best ? k : best;
        }
        if (lane == 0 && fst == 0x7FFFFFFF && !inS[v]) fst = (int)v;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ull ob = __shfl_xor_sync(IM_FULL, best, o);
        best = ob > best ? ob : best;
    }
    fst = __reduce_min_sync(IM_FULL, fst);
    if (lane == 0) {
        sKey[threadIdx.x >> 5] = best;
        sFirst[threadIdx.x >> 5] = fst;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ull b = 0;
        int f = 0x7FFFFFFF;
        for (int i = 0; i < BLOCK / 32; i++) {
            b = sKey[i] > b ? sKey[i] : b;
            f = min(f, sFirst[i]);
        }
        if (b) atomicMax(key, b);
        if (f != 0x7FFFFFFF) atomicMin(first, f);
    }
}

// ============================================================ a7: seed diffusion
// Alg. 1 lines 11, 13-14: S <- S + s; R_G(S) by a multi-simulation BFS from s over live edges
// (same samples as the sketches, R13) carrying J-bit masks; visited bits only ever set.
__global__ void k_seed_start(int32_t J, const ull* key, const int* first, const uint32_t* __restrict__ M32,
                             const uint8_t* __restrict__ MS, uint8_t* inS, uint32_t* vis, uint32_t* delta0,
                             const int32_t* __restrict__ off, int4* items0, int32_t* vl0, IterCounters* ctr0,
                             ull* sigma_count, StepDev* rec) {
    const int lane = threadIdx.x, W = J >> 5, Jw = J >> 2;
    ull k = *key;
    uint32_t s = k ? (0xFFFFFFFFu - (uint32_t)k) : (uint32_t)*first;
    int64_t score;
    if (k) {
        score = (int64_t)(k >> 32);
    } else {  // pool empty: lowest id not in S (R14); its merged score is still reported
        uint32_t acc = 0;
        for (int w = lane; w < Jw; w += 32)
            acc += __vsadu4(__vmaxu4(M32[(size_t)s * Jw + w], reinterpret_cast<const uint32_t*>(MS)[w]), 0u);
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(IM_FULL, acc, o);
        score = acc;
    }
    uint32_t bits = 0, any = 0;
    for (int w = lane; w < W; w += 32) {
        uint32_t d = ~vis[(size_t)s * W + w];
        vis[(size_t)s * W + w] = IM_FULL;
        delta0[(size_t)s * W + w] = d;
        bits += __popc(d);
        any |= d;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        bits += __shfl_xor_sync(IM_FULL, bits, o);
        any |= __shfl_xor_sync(IM_FULL, any, o);
    }
    int b = off[s], e = off[s + 1];
    int ns = any ? (e - b + SEG - 1) / SEG : 0;
    for (int i = lane; i < ns; i += 32) items0[i] = make_int4((int)s, b + i * SEG, min(b + (i + 1) * SEG, e), 0);
    if (lane == 0) {
        inS[s] = 1;
        *sigma_count += bits;
        ctr0->next_items = ns;
        ctr0->changed = any ? 1 : 0;
        ctr0->next_edges = any ? (ull)(e - b) : 0ull;
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
    uint32_t* vis;
    const uint32_t* din;
    uint32_t* dout;
    uint32_t* btag;
    uint32_t tag;
    int4* next_items;
    int32_t* next_vl;
};

// one 32-simulation word of one edge: new = Delta_u & live & ~visited(v); returns popcount of truly new bits
__device__ __forceinline__ int bfs_word(const BfsArgs& a, const uint32_t* sX, uint32_t u, uint32_t v, int w, uint32_t h,
                                        uint32_t T, int lo, int hi) {
    const int W = a.J >> 5;
    uint32_t d = a.din[(size_t)u * W + w];
    if (!d) return 0;
    int i0 = max(lo, w << 5), i1 = min(hi, (w << 5) + 32);
    uint32_t live = 0;
    for (int i = i0; i < i1; ++i) live |= ((sX[i] ^ h) < T) ? (1u << (i & 31)) : 0u;
    uint32_t nv = d & live;
    if (!nv) return 0;
    nv &= ~__ldcg(&a.vis[(size_t)v * W + w]);
    if (!nv) return 0;
    uint32_t old = atomicOr(&a.vis[(size_t)v * W + w], nv);
    uint32_t tn = nv & ~old;
    if (!tn) return 0;
    atomicOr(&a.dout[(size_t)v * W + w], tn);
    return __popc(tn);
}

template <bool CONST_T>
__global__ void __launch_bounds__(BLOCK) k_bfs_level(BfsArgs a) {
    __shared__ uint32_t sX[1024];
    __shared__ uint16_t sS[4098];
    __shared__ int sSlot[BLOCK / 32][32];
    for (int i = threadIdx.x; i < a.J; i += blockDim.x) sX[i] = a.Xs[i];
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) sS[i] = a.s12[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t newbits = 0;
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&a.ctr_next->batch, 32);
        base = __shfl_sync(IM_FULL, base, 0);
        if (base >= a.n_items) break;
        int it = base + lane;
        int u = 0, eb = 0, cnt = 0;
        if (it < a.n_items) {
            int4 I = a.items[it];
            u = I.x;
            eb = I.y;
            cnt = I.z - I.y;
        }
        int incl = warp_incl_scan(cnt, lane);
        int total = __shfl_sync(IM_FULL, incl, 31);
        int start = incl - cnt;
        int carry = 0;
        for (int e0 = 0; e0 < total; e0 += 32) {
            bool starts = cnt > 0 && start >= e0 && start < e0 + 32;
            if (starts) sSlot[wib][start - e0] = lane;
            uint32_t smask = __reduce_or_sync(IM_FULL, starts ? (1u << (start - e0)) : 0u);
            __syncwarp();
            uint32_t below = smask & ((2u << lane) - 1u);
            int owner = below ? sSlot[wib][31 - __clz(below)] : carry;
            __syncwarp();
            carry = __shfl_sync(IM_FULL, owner, 31);
            int ou = __shfl_sync(IM_FULL, u, owner);
            int oeb = __shfl_sync(IM_FULL, eb, owner);
            int ost = __shfl_sync(IM_FULL, start, owner);
            int idx = e0 + lane;
            uint32_t v = 0, h = 0, T = 0;
            int lo = 0, hi = 0, got = 0;
            bool dense = false;
            if (idx < total) {
                int e = oeb + (idx - ost);
                uint2 f = a.fwd[e];
                v = f.x;
                h = f.y;
                T = CONST_T ? a.T0 : a.fwdT[e];
                if (T) {
                    edge_window(h, T, sX, sS, a.J, lo, hi);
                    if (hi - lo > DENSE_WIN) dense = true;
                    else if (lo < hi)
                        for (int w = lo >> 5; w <= (hi - 1) >> 5; ++w) got += bfs_word(a, sX, (uint32_t)ou, v, w, h, T, lo, hi);
                }
            }
            uint32_t dmask = __ballot_sync(IM_FULL, dense);
            while (dmask) {
                int l = __ffs(dmask) - 1;
                dmask &= dmask - 1;
                uint32_t dv = __shfl_sync(IM_FULL, v, l), dh = __shfl_sync(IM_FULL, h, l), dT = __shfl_sync(IM_FULL, T, l);
                int dlo = __shfl_sync(IM_FULL, lo, l), dhi = __shfl_sync(IM_FULL, hi, l);
                uint32_t du = (uint32_t)__shfl_sync(IM_FULL, ou, l);
                int c = 0;
                for (int w = (dlo >> 5) + lane; w <= (dhi - 1) >> 5; w += 32) c += bfs_word(a, sX, du, dv, w, dh, dT, dlo, dhi);
                c = __reduce_add_sync(IM_FULL, (uint32_t)c);
                if (lane == l) got += c;
            }
            newbits += (uint32_t)got;
            bool first = got > 0 && atomicMax(&a.btag[v], a.tag) < a.tag;
            int rd = 0, ns = 0;
            if (first) {
                rd = a.off[v + 1] - a.off[v];
                ns = (rd + SEG - 1) / SEG;
            }
            int ninc = warp_incl_scan(ns, lane);
            int ntot = __shfl_sync(IM_FULL, ninc, 31);
            uint32_t fmask = __ballot_sync(IM_FULL, first);
            if (fmask) {
                int pos = 0, vpos = 0;
                if (lane == 31) {
                    if (ntot) pos = atomicAdd(&a.ctr_next->next_items, ntot);
                    vpos = atomicAdd(&a.ctr_next->changed, __popc(fmask));
                }
                pos = __shfl_sync(IM_FULL, pos, 31);
                vpos = __shfl_sync(IM_FULL, vpos, 31);
                long long esum = rd;
#pragma unroll
                for (int o = 16; o; o >>= 1) esum += __shfl_xor_sync(IM_FULL, esum, o);
                if (lane == 0 && esum) atomicAdd(&a.ctr_next->next_edges, (ull)esum);
                if (first) {
                    a.next_vl[vpos + __popc(fmask & ((1u << lane) - 1u))] = (int32_t)v;
                    int b = a.off[v], e = b + rd, p = pos + ninc - ns;
                    for (int s = b; s < e; s += SEG) a.next_items[p++] = make_int4((int)v, s, min(s + SEG, e), 0);
                }
            }
        }
    }
    newbits = __reduce_add_sync(IM_FULL, newbits);
    if (lane == 0 && newbits) {
        atomicAdd(&a.ctr_next->new_bits, (ull)newbits);
        atomicAdd(a.sigma_count, (ull)newbits);
    }
}

__global__ void k_bfs_clear(int n_v, int W, const int32_t* __restrict__ vl, uint32_t* __restrict__ delta) {
    int64_t total = (int64_t)n_v * W, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride)
        delta[(size_t)vl[i / W] * W + (i % W)] = 0u;
}

// ============================================================ a8: error check (Alg. 1 lines 12, 15-27)
__global__ void k_error_check(int32_t J, int k, int K, double eps_l, double eps_g, const uint32_t* __restrict__ M32,
                              uint8_t* MS, const IterCounters* ctr_unused, const ull* sigma_count, double* varsigma,
                              StepDev* rec) {
    (void)ctr_unused;
    const int lane = threadIdx.x, Jw = J >> 2;
    __shared__ int sRebuild;
    if (lane == 0) {
        double e = exp2((double)rec->score / (double)J) / 0.77351;
        ull cnt = *sigma_count;
        double sigma = (double)cnt / (double)J;
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
static inline int grid_for(Ctx& c, int64_t work, int per_block = BLOCK) {
    int64_t g = (work + per_block - 1) / per_block;
    int64_t cap = (int64_t)c.num_sms * 8;
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}
#define LAUNCHED(c) ((c).launches++, cudaGetLastError())

cudaError_t launch_validate(Ctx& c, const int32_t* off, const int32_t* tgt, const float* prob, int* flags) {
    k_validate<<<grid_for(c, c.m > c.n ? c.m : c.n), BLOCK, 0, c.stream>>>(c.n, c.m, off, tgt, prob, flags);
    return LAUNCHED(c);
}
cudaError_t launch_const_check(Ctx& c, const float* prob, int* flag) {
    k_const_check<<<grid_for(c, c.m), BLOCK, 0, c.stream>>>(c.m, prob, flag);
    return LAUNCHED(c);
}
cudaError_t launch_edge_prep(Ctx& c, const int32_t* tgt, const float* prob, int32_t* indeg) {
    k_edge_prep<<<grid_for(c, c.m), BLOCK, 0, c.stream>>>(c.n, c.m, c.off, tgt, prob, c.fwd, c.fwdT, indeg);
    return LAUNCHED(c);
}
cudaError_t launch_transpose(Ctx& c, int32_t* cursor) {
    k_transpose<<<grid_for(c, c.m), BLOCK, 0, c.stream>>>(c.n, c.m, c.off, c.fwd, c.fwdT, c.roff, cursor, c.rev, c.revT);
    return LAUNCHED(c);
}
cudaError_t scan_exclusive(Ctx& c, const int32_t* in, int32_t* out, int n, void* tmp, size_t& tmp_bytes) {
    cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, n, c.stream);
    if (tmp) c.launches++;
    return e;
}
cudaError_t launch_build_items(Ctx& c, const int32_t* offs, int4* items, int32_t* nseg, void* tmp, size_t tmp_bytes) {
    // nseg has n+1 entries; base = exclusive scan written in place into nseg+? -> use the second half
    int32_t* base = nseg + (c.n + 1);
    k_nseg<<<(c.n + 1 + BLOCK - 1) / BLOCK, BLOCK, 0, c.stream>>>(c.n, offs, nseg);
    cudaError_t e = LAUNCHED(c);
    if (e) return e;
    e = scan_exclusive(c, nseg, base, c.n + 1, tmp, tmp_bytes);
    if (e) return e;
    if (items) {
        k_fill_items<<<(c.n + BLOCK - 1) / BLOCK, BLOCK, 0, c.stream>>>(c.n, offs, base, items);
        e = LAUNCHED(c);
    }
    return e;
}
cudaError_t launch_init_registers(Ctx& c) {
    int64_t chunks = (int64_t)c.n * (c.J >> 4);
    k_init_registers<<<grid_for(c, chunks), BLOCK, 0, c.stream>>>(c.n, c.J, c.seedV, c.seedJ, c.permd,
                                                                  reinterpret_cast<uint4*>(c.M));
    return LAUNCHED(c);
}

template <bool C, bool B, bool F>
static void sweep_inst(int grid, cudaStream_t s, const SweepArgs& a) {
    k_sweep<C, B, F><<<grid, BLOCK, 0, s>>>(a);
}

cudaError_t launch_sweep(Ctx& c, bool first, const int4* items, int n_items, uint32_t tag_in, uint32_t tag_out,
                         int out_buf, bool blocked) {
    SweepArgs a;
    a.items = items;
    a.n_items = n_items;
    a.ctr_next = &c.ctr[out_buf];
    a.roff = c.roff;
    a.rev = c.rev;
    a.revT = c.revT;
    a.T0 = c.T0;
    a.Xs = c.Xs;
    a.s12 = c.s12;
    a.J = c.J;
    a.M32 = reinterpret_cast<uint32_t*>(c.M);
    a.vis = c.vis;
    a.chg_in = c.chg[tag_in & 1];
    a.chg_out = c.chg[tag_out & 1];
    a.tag_in = tag_in;
    a.tag_out = tag_out;
    a.next_items = c.items[out_buf];
    int64_t want = ((int64_t)n_items + 32 * (BLOCK / 32) - 1) / (32 * (BLOCK / 32));
    int grid = (int)(want < 1 ? 1 : (want > c.max_blocks_sweep ? c.max_blocks_sweep : want));
    bool ct = c.constT;
    if (first) {
        if (ct) { if (blocked) sweep_inst<true, true, false>(grid, c.stream, a); else sweep_inst<true, false, false>(grid, c.stream, a); }
        else { if (blocked) sweep_inst<false, true, false>(grid, c.stream, a); else sweep_inst<false, false, false>(grid, c.stream, a); }
    } else {
        if (ct) { if (blocked) sweep_inst<true, true, true>(grid, c.stream, a); else sweep_inst<true, false, true>(grid, c.stream, a); }
        else { if (blocked) sweep_inst<false, true, true>(grid, c.stream, a); else sweep_inst<false, false, true>(grid, c.stream, a); }
    }
    return LAUNCHED(c);
}

cudaError_t launch_estimate(Ctx& c, double* out) {
    k_estimate<<<grid_for(c, (int64_t)c.n * 32), BLOCK, 0, c.stream>>>(c.n, c.J, reinterpret_cast<const uint32_t*>(c.M), out);
    return LAUNCHED(c);
}
cudaError_t launch_argmax(Ctx& c, bool pool) {
    int g = grid_for(c, (int64_t)c.n * 32);
    if (pool)
        k_argmax<true><<<g, BLOCK, 0, c.stream>>>(c.n, c.J, reinterpret_cast<const uint32_t*>(c.M), c.MS, c.vis, c.inS, c.key, c.first);
    else
        k_argmax<false><<<g, BLOCK, 0, c.stream>>>(c.n, c.J, reinterpret_cast<const uint32_t*>(c.M), c.MS, c.vis, c.inS, c.key, c.first);
    return LAUNCHED(c);
}
cudaError_t launch_seed_start(Ctx& c, int k) {
    (void)k;
    k_seed_start<<<1, 32, 0, c.stream>>>(c.J, c.key, c.first, reinterpret_cast<const uint32_t*>(c.M), c.MS, c.inS, c.vis,
                                          c.delta[0], c.off, c.bitems[0], c.bvl[0], &c.ctr[0], c.sigma_count, c.rec);
    return LAUNCHED(c);
}
cudaError_t launch_bfs_level(Ctx& c, int cur, int n_items, uint32_t tag) {
    BfsArgs a;
    a.items = c.bitems[cur];
    a.n_items = n_items;
    a.ctr_next = &c.ctr[cur ^ 1];
    a.sigma_count = c.sigma_count;
    a.off = c.off;
    a.fwd = c.fwd;
    a.fwdT = c.fwdT;
    a.T0 = c.T0;
    a.Xs = c.Xs;
    a.s12 = c.s12;
    a.J = c.J;
    a.vis = c.vis;
    a.din = c.delta[cur];
    a.dout = c.delta[cur ^ 1];
    a.btag = c.btag;
    a.tag = tag;
    a.next_items = c.bitems[cur ^ 1];
    a.next_vl = c.bvl[cur ^ 1];
    int64_t want = ((int64_t)n_items + 32 * (BLOCK / 32) - 1) / (32 * (BLOCK / 32));
    int grid = (int)(want < 1 ? 1 : (want > c.max_blocks_bfs ? c.max_blocks_bfs : want));
    if (c.constT) k_bfs_level<true><<<grid, BLOCK, 0, c.stream>>>(a);
    else k_bfs_level<false><<<grid, BLOCK, 0, c.stream>>>(a);
    return LAUNCHED(c);
}
cudaError_t launch_bfs_clear(Ctx& c, int cur, int n_v) {
    int W = c.J >> 5;
    k_bfs_clear<<<grid_for(c, (int64_t)n_v * W), BLOCK, 0, c.stream>>>(n_v, W, c.bvl[cur], c.delta[cur]);
    return LAUNCHED(c);
}
cudaError_t launch_error_check(Ctx& c, int k, int K, double eps_l, double eps_g) {
    k_error_check<<<1, 32, 0, c.stream>>>(c.J, k, K, eps_l, eps_g, reinterpret_cast<const uint32_t*>(c.M), c.MS, nullptr,
                                          c.sigma_count, c.varsigma, c.rec);
    return LAUNCHED(c);
}
cudaError_t launch_gather_rows(Ctx& c, const int32_t* rows, int64_t nrows, uint8_t* out) {
    k_gather_rows<<<grid_for(c, nrows * c.J), BLOCK, 0, c.stream>>>(nrows, c.J, rows, c.M, out);
    return LAUNCHED(c);
}

int occupancy_sweep(int* blocks_per_sm_sweep, int* blocks_per_sm_bfs) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm_sweep, k_sweep<true, true, true>, BLOCK, 0);
    if (e) return (int)e;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm_bfs, k_bfs_level<true>, BLOCK, 0);
}

}  // namespace im
