// im_first.cu -- register init (Alg. 1 lines 2-5) fused with the first sweep of Alg. 2.
//
// In the first sweep every vertex is live and every register still holds its init value
// M_v[j] = clz(hash(v) xor hash(j)), which is a pure function of (v, j).  So the
// first sweep is computed here as a gather, one warp per vertex u over its out-edges (pull, reading
// R9): row(u) = max(init(u), max over live (u,v), u not blocked, of init(v)) -- exactly the
// synchronous first iteration -- with init(v) recomputed from the hashes instead of read from HBM.
// The warp owns the row, so it is written once, with no atomics, together with u's exact
// per-simulation change mask (row != init) that drives the second sweep (im_sweep.cu).
// Vertices with more than FIRST_BIG out-edges are done by a whole block (k_first_big).
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
    const int32_t* big;   // vertices with > FIRST_BIG out-edges (k_first_big)
    int n_big;
};

// shared-memory working row: one u32 per simulation (native smem atomicMax).  `e` is this lane's
// edge (or -1); the loop around it must be warp-uniform.  Windows wider than DENSE_WIN simulations
// (w close to 1) are walked by the whole warp, one candidate per lane.
template <bool CONST_T, bool BLOCKED>
__device__ __forceinline__ void gather_edge(const FirstArgs& a, const uint32_t* sX, const uint16_t* sS, const uint32_t* sHJ,
                                            const uint32_t* sVis, uint32_t* row, int e, uint32_t& wcount) {
    const int lane = threadIdx.x & 31;
    uint32_t h = 0, T = 0, hv = 0;
    int lo = 0, hi = 0;
    if (e >= 0) {
        uint2 f = a.fwd[e];
        T = CONST_T ? a.T0 : a.fwdT[e];
        h = f.y;
        if (T) {
            edge_window(h, T, sX, sS, a.J, lo, hi);
            if (lo < hi) {
                wcount++;
                hv = murmur_word(f.x, a.seedV);
            }
        }
    }
    const bool dense = hi - lo > DENSE_WIN;
    if (!dense)
        for (int i = lo; i < hi; ++i) {
            if ((sX[i] ^ h) >= T) continue;
            if (BLOCKED && ((sVis[i >> 5] >> (i & 31)) & 1u)) continue;
            uint32_t val = __clz(hv ^ sHJ[i]);
            if (val > row[i]) atomicMax(&row[i], val);
        }
    uint32_t dmask = __ballot_sync(IM_FULL, dense);
    while (dmask) {
        int l = __ffs(dmask) - 1;
        dmask &= dmask - 1;
        uint32_t dh = __shfl_sync(IM_FULL, h, l), dT = __shfl_sync(IM_FULL, T, l), dhv = __shfl_sync(IM_FULL, hv, l);
        int dlo = __shfl_sync(IM_FULL, lo, l), dhi = __shfl_sync(IM_FULL, hi, l);
        for (int i = dlo + lane; i < dhi; i += 32) {
            if ((sX[i] ^ dh) >= dT) continue;
            if (BLOCKED && ((sVis[i >> 5] >> (i & 31)) & 1u)) continue;
            uint32_t val = __clz(dhv ^ sHJ[i]);
            if (val > row[i]) atomicMax(&row[i], val);
        }
    }
}

// write the row of u, its per-simulation change mask and chunk summary
__device__ __forceinline__ void write_row(const FirstArgs& a, const uint32_t* sHJ, const uint32_t* row, uint32_t hu, uint32_t u,
                                          int tid, int nthreads, uint32_t* sMask) {
    const int J = a.J;
    uint32_t* M32 = reinterpret_cast<uint32_t*>(a.M) + (size_t)u * (J >> 2);
    for (int w = tid; w < (J >> 2); w += nthreads) {
        uint32_t x = 0, ch = 0;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            uint32_t r = row[4 * w + b];
            x |= r << (8 * b);
            ch |= (r != (uint32_t)__clz(hu ^ sHJ[4 * w + b]) ? 1u : 0u) << b;
        }
        M32[w] = x;
        if (ch) atomicOr(&sMask[w >> 3], ch << ((w & 7) << 2));
    }
}

template <bool CONST_T, bool BLOCKED>
__global__ void __launch_bounds__(BLOCK) k_first(FirstArgs a) {
    __shared__ uint32_t sX[1024];
    __shared__ uint16_t sS[4098];
    __shared__ uint32_t sHJ[1024];
    extern __shared__ uint32_t sRows[];  // BLOCK/32 working rows of J u32 (dynamic: 8*J*4 bytes)
    __shared__ uint32_t sVis[BLOCK / 32][32];
    __shared__ uint32_t sMask[BLOCK / 32][32];
    const int J = a.J, W = J >> 5;
    for (int i = threadIdx.x; i < J; i += blockDim.x) {
        sX[i] = a.Xs[i];
        sHJ[i] = murmur_word((uint32_t)a.perm[i], a.seedJ);
    }
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) sS[i] = a.s12[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t* row = sRows + wib * J;
    uint32_t wcount = 0;
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&a.ctr->batch, 256);
        base = __shfl_sync(IM_FULL, base, 0);
        if (base >= a.n) break;
        const int end = min(base + 256, a.n);
        for (int u = base; u < end; ++u) {
            const int eb = a.off[u], ee = a.off[u + 1];
            if (ee - eb > FIRST_BIG) continue;  // done by k_first_big
            const uint32_t hu = murmur_word((uint32_t)u, a.seedV);
            for (int i = lane; i < J; i += 32) row[i] = __clz(hu ^ sHJ[i]);
            if (lane < W) {
                sMask[wib][lane] = 0u;
                if (BLOCKED) sVis[wib][lane] = a.vis[(size_t)u * W + lane];
            }
            __syncwarp();
            for (int e0 = eb; e0 < ee; e0 += 32)
                gather_edge<CONST_T, BLOCKED>(a, sX, sS, sHJ, sVis[wib], row, e0 + lane < ee ? e0 + lane : -1, wcount);
            __syncwarp();
            write_row(a, sHJ, row, hu, (uint32_t)u, lane, 32, sMask[wib]);
            __syncwarp();
            uint32_t m = lane < W ? sMask[wib][lane] : 0u;
            if (lane < W) a.cm_out[(size_t)u * W + lane] = m;
            uint32_t chunks = __ballot_sync(IM_FULL, m != 0u);
            if (lane == 0) a.bits_out[u] = chunks;
            __syncwarp();
        }
    }
    wcount = __reduce_add_sync(IM_FULL, wcount);
    if (lane == 0 && wcount) atomicAdd(&a.ctr->win_edges, (ull)wcount);
}

// one block per vertex with more than FIRST_BIG out-edges
template <bool CONST_T, bool BLOCKED>
__global__ void __launch_bounds__(BLOCK) k_first_big(FirstArgs a) {
    __shared__ uint32_t sX[1024];
    __shared__ uint16_t sS[4098];
    __shared__ uint32_t sHJ[1024];
    __shared__ uint32_t row[1024];
    __shared__ uint32_t sVis[32];
    __shared__ uint32_t sMask[32];
    const int J = a.J, W = J >> 5;
    for (int i = threadIdx.x; i < J; i += blockDim.x) {
        sX[i] = a.Xs[i];
        sHJ[i] = murmur_word((uint32_t)a.perm[i], a.seedJ);
    }
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) sS[i] = a.s12[i];
    uint32_t wcount = 0;
    for (int bi = blockIdx.x; bi < a.n_big; bi += gridDim.x) {
        const uint32_t u = (uint32_t)a.big[bi];
        __syncthreads();
        const uint32_t hu = murmur_word(u, a.seedV);
        for (int i = threadIdx.x; i < J; i += blockDim.x) row[i] = __clz(hu ^ sHJ[i]);
        if (threadIdx.x < W) {
            sMask[threadIdx.x] = 0u;
            if (BLOCKED) sVis[threadIdx.x] = a.vis[(size_t)u * W + threadIdx.x];
        }
        __syncthreads();
        const int eb = a.off[u], ee = a.off[u + 1];
        for (int e0 = eb + (threadIdx.x & ~31); e0 < ee; e0 += blockDim.x)  // warp-uniform trip count
            gather_edge<CONST_T, BLOCKED>(a, sX, sS, sHJ, sVis, row, e0 + (threadIdx.x & 31) < ee ? e0 + (threadIdx.x & 31) : -1, wcount);
        __syncthreads();
        write_row(a, sHJ, row, hu, u, threadIdx.x, blockDim.x, sMask);
        __syncthreads();
        if (threadIdx.x < 32) {
            uint32_t m = threadIdx.x < W ? sMask[threadIdx.x] : 0u;
            if (threadIdx.x < W) a.cm_out[(size_t)u * W + threadIdx.x] = m;
            uint32_t chunks = __ballot_sync(IM_FULL, m != 0u);
            if (threadIdx.x == 0) a.bits_out[u] = chunks;
        }
    }
    const int lane = threadIdx.x & 31;
    wcount = __reduce_add_sync(IM_FULL, wcount);
    if (lane == 0 && wcount) atomicAdd(&a.ctr->win_edges, (ull)wcount);
}

template <bool C, bool B>
static cudaError_t first_inst(Ctx& c, const FirstArgs& a) {
    k_first<C, B><<<c.max_blocks_first, BLOCK, (BLOCK / 32) * c.J * sizeof(uint32_t), c.stream>>>(a);
    cudaError_t e = LAUNCHED(c);
    if (e || a.n_big == 0) return e;
    k_first_big<C, B><<<a.n_big < c.num_sms * 4 ? a.n_big : c.num_sms * 4, BLOCK, 0, c.stream>>>(a);
    return LAUNCHED(c);
}

cudaError_t launch_first(Ctx& c, uint32_t* cm_out, uint32_t* bits_out, IterCounters* ctr, bool blocked) {
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
    a.big = c.fbig;
    a.n_big = c.n_fbig;
    if (c.constT) return blocked ? first_inst<true, true>(c, a) : first_inst<true, false>(c, a);
    return blocked ? first_inst<false, true>(c, a) : first_inst<false, false>(c, a);
}

// vertices with more than FIRST_BIG out-edges, ascending (once per graph)
__global__ void k_list_big_rows(int32_t n, const int32_t* __restrict__ off, int32_t* __restrict__ out, int* count) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += stride)
        if (off[u + 1] - off[u] > FIRST_BIG) out[atomicAdd(count, 1)] = (int32_t)u;
}

cudaError_t launch_list_big_rows(Ctx& c, int32_t* out, int* count) {
    k_list_big_rows<<<grid_for(c, c.n), BLOCK, 0, c.stream>>>(c.n, c.off, out, count);
    return LAUNCHED(c);
}

// opt in to the dynamic shared memory of the largest J (8 rows x 1024 x 4 B = 32 KB + 17 KB static)
int setup_first(int J, int* blocks_per_sm) {
    const int dyn = (BLOCK / 32) * 1024 * (int)sizeof(uint32_t);
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_first<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn))) return (int)e;
    if ((e = cudaFuncSetAttribute(k_first<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn))) return (int)e;
    if ((e = cudaFuncSetAttribute(k_first<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn))) return (int)e;
    if ((e = cudaFuncSetAttribute(k_first<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn))) return (int)e;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_first<true, true>, BLOCK,
                                                              (BLOCK / 32) * J * sizeof(uint32_t));
}

}  // namespace im
