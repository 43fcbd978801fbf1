// im_eval.cu -- independent Monte-Carlo influence evaluator (reading R23).
//
// The paper scores every seed set with a sample-then-diffuse oracle on fresh randomness
// (PAPER.md:471-472).  Here sample r of edge (u,v) is live iff draw_r(u,v) < T_uv, where
//   draw_r(u,v) = mix64(mix64(seed ^ (u << 32 | v)) + (r + 1) * 0x9E3779B97F4A7C15) >> 33
// (counter-based SplitMix64, so samples are independent and any range can be evaluated on its own)
// and T_uv is the same 31-bit integer threshold as Eq. 5 (draw / h_max < w  <=>  draw < T_uv).
// B samples at a time are carried as B-bit masks per vertex through the same multi-sample BFS
// machinery as the selection (frontier items, Delta words, k_bfs_compact); only the live test
// differs: a lane owns one edge and draws one value per sample bit of the source's Delta.
#include "im_device.cuh"
#include "im_internal.h"

namespace im {

constexpr ull MC_GAMMA = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ ull mc_mix64(ull z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

struct EvalArgs {
    const int4* items;
    int n_items;
    IterCounters* ctr_next;  // zeroed before launch: batch cursor
    const uint2* fwd;        // {target, h} (h unused here)
    const uint32_t* fwdT;    // per-edge thresholds (null when constant)
    uint32_t T0;
    int W;                   // 32-sample words per vertex in this batch
    ull seed;
    ull r0;                  // first sample of the batch
    uint32_t* vis;
    const uint32_t* din;
    uint32_t* dout;
    uint32_t* nbits;
};

// all sample bits of Delta_u (words 0..W-1) through edge (u, v)
__device__ __forceinline__ void mc_edge(const EvalArgs& a, uint32_t u, uint32_t v, uint32_t T) {
    const ull ze = mc_mix64(a.seed ^ (((ull)u << 32) | (ull)v));
    for (int w = 0; w < a.W; ++w) {
        const uint32_t d = a.din[(size_t)u * a.W + w];
        if (!d) continue;
        uint32_t live = 0;
        for (uint32_t t = d; t; t &= t - 1) {
            const int j = __ffs(t) - 1;
            const ull r = a.r0 + (ull)(32 * w + j);
            if ((uint32_t)(mc_mix64(ze + (r + 1ULL) * MC_GAMMA) >> 33) < T) live |= 1u << j;
        }
        if (!live) continue;
        const uint32_t nv = live & ~__ldcg(&a.vis[(size_t)v * a.W + w]);
        if (!nv) continue;
        atomicOr(&a.vis[(size_t)v * a.W + w], nv);
        atomicOr(&a.dout[(size_t)v * a.W + w], nv);
        atomicOr(&a.nbits[v], 1u << w);
    }
}

// one BFS level: the work items (u, edge range) of the frontier, flattened so every lane owns one edge
template <bool CONST_T>
__global__ void __launch_bounds__(BLOCK) k_mc_level(EvalArgs a) {
    __shared__ int sSlot[BLOCK / 32][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&a.ctr_next->batch, 32);
        base = __shfl_sync(IM_FULL, base, 0);
        if (base >= a.n_items) break;
        const int it = base + lane;
        int u = 0, eb = 0, cnt = 0;
        if (it < a.n_items) {
            const int4 I = a.items[it];
            u = I.x;
            eb = I.y;
            cnt = I.z - I.y;
        }
        const int incl = warp_incl_scan(cnt, lane);
        const int total = __shfl_sync(IM_FULL, incl, 31);
        const int start = incl - cnt;
        int carry = 0;
        for (int e0 = 0; e0 < total; e0 += 32) {
            const bool starts = cnt > 0 && start >= e0 && start < e0 + 32;
            if (starts) sSlot[wib][start - e0] = lane;
            const uint32_t smask = __reduce_or_sync(IM_FULL, starts ? (1u << (start - e0)) : 0u);
            __syncwarp();
            const uint32_t below = smask & ((2u << lane) - 1u);
            const int owner = below ? sSlot[wib][31 - __clz(below)] : carry;
            __syncwarp();
            carry = __shfl_sync(IM_FULL, owner, 31);
            const int ou = __shfl_sync(IM_FULL, u, owner);
            const int oeb = __shfl_sync(IM_FULL, eb, owner);
            const int ost = __shfl_sync(IM_FULL, start, owner);
            const int idx = e0 + lane;
            if (idx < total) {
                const int e = oeb + (idx - ost);
                const uint32_t T = CONST_T ? a.T0 : a.fwdT[e];
                if (T) mc_edge(a, (uint32_t)ou, a.fwd[e].x, T);
            }
        }
    }
}

// S <- S + s in every sample of the batch: Delta_s = samples where s was not yet reached
__global__ void k_mc_start(int32_t s, int W, uint32_t* vis, uint32_t* delta0, int32_t* vl0, IterCounters* ctr0, ull* count) {
    const int lane = threadIdx.x;
    uint32_t bits = 0, any = 0;
    for (int w = lane; w < W; w += 32) {
        const uint32_t d = ~vis[(size_t)s * W + w];
        vis[(size_t)s * W + w] = IM_FULL;
        delta0[(size_t)s * W + w] = d;
        bits += __popc(d);
        any |= d;
    }
    bits = __reduce_add_sync(IM_FULL, bits);
    any = __reduce_or_sync(IM_FULL, any);
    if (lane == 0) {
        *count += bits;
        ctr0->changed = any ? 1 : 0;
        if (any) vl0[0] = s;
    }
}

cudaError_t launch_mc_start(Ctx& c, int32_t s, int W, ull* count) {
    k_mc_start<<<1, 32, 0, c.stream>>>(s, W, c.ev_vis, c.ev_delta[0], c.ev_vl[0], &c.ev_ctr[0], count);
    return LAUNCHED(c);
}

cudaError_t launch_mc_level(Ctx& c, int cur, int n_items, int W, ull seed, ull r0, ull* count) {
    EvalArgs a;
    a.items = c.ev_items[cur];
    a.n_items = n_items;
    a.ctr_next = &c.ev_ctr[cur ^ 1];
    a.fwd = c.fwd;
    a.fwdT = c.fwdT;
    a.T0 = c.T0;
    a.W = W;
    a.seed = seed;
    a.r0 = r0;
    a.vis = c.ev_vis;
    a.din = c.ev_delta[cur];
    a.dout = c.ev_delta[cur ^ 1];
    a.nbits = c.ev_nbits;
    const int64_t want = ((int64_t)n_items + 32 * (BLOCK / 32) - 1) / (32 * (BLOCK / 32));
    const int grid = (int)(want < 1 ? 1 : (want > c.max_blocks_bfs ? c.max_blocks_bfs : want));
    if (c.constT) k_mc_level<true><<<grid, BLOCK, 0, c.stream>>>(a);
    else k_mc_level<false><<<grid, BLOCK, 0, c.stream>>>(a);
    cudaError_t e = LAUNCHED(c);
    if (e) return e;
    const int nxt = cur ^ 1;
    return launch_bfs_compact_raw(c, 32 * W, c.ev_nbits, c.ev_delta[nxt], c.ev_vl[nxt], c.ev_items[nxt], &c.ev_ctr[nxt], count);
}

}  // namespace im
