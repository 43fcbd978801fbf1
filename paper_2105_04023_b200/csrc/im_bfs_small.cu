// im_bfs_small.cu -- the seed diffusion (Alg. 1 lines 13-14) for small frontiers:
// all levels of a BFS whose frontier stays small run inside ONE single-block launch.
//
// After the first seed most greedy steps reach only a few hundred (vertex, simulation) pairs per
// level, and the multi-block level path (k_bfs_level2 + k_bfs_compact + k_slices_big + k_bfs_clear,
// one host round trip per level) is then dominated by launch and synchronisation latency.  This
// kernel runs as ONE thread-block cluster of SB_CLUSTER blocks (8 SMs, distributed shared memory for
// the level counters, cluster barriers between levels) and carries the same state (frontier list bvl[cur], Delta rows delta[cur], the {visited,
// new} pairs vd, R_G(S) words vis, per-vertex new-word flags nbits) through the levels with block
// barriers: a warp takes a frontier vertex u and walks its whole out-row, lane per edge; for each
// candidate word the simulations new at v are Delta_u & live & ~visited(v) (the same test and the
// same fire-and-forget ORs as k_bfs_level2); v is appended to the next frontier by the thread whose
// OR set its first new-word flag.  Between levels the new bits move to the next Delta rows and to vis
// and are counted into sigma, exactly like k_bfs_compact.  When the next frontier's out-edges exceed
// max_edges the kernel stops and leaves that frontier (list, Delta rows, counters) for the
// multi-block path, which continues from it.
#include <cooperative_groups.h>

#include "im_device.cuh"
#include "im_internal.h"

namespace cg = cooperative_groups;

namespace im {

constexpr int SB_THREADS = 1024;
constexpr int SB_CLUSTER = 8;  // blocks of the cluster (portable maximum), one per SM
constexpr int SB_LONG = 256;   // frontier rows longer than this are split over the whole cluster

struct BfsSmallArgs {
    int J;
    const int32_t* off;
    const uint2* fwd;
    const uint32_t* fwdT;
    uint32_t T0;
    const uint32_t* Xs;
    const uint16_t* s12;
    uint2* vd;
    uint32_t* vis;
    uint32_t* nbits;
    uint32_t* delta0;
    uint32_t* delta1;
    int32_t* vl0;
    int32_t* vl1;
    IterCounters* ctr;  // [2]
    ull* sigma_count;
    int cur, n_v;
    long long max_edges;
    BfsSmallOut* out;
    int32_t* longv;  // the level's long frontier rows (scratch, n entries)
};

// one out-edge e of a frontier vertex with Delta row dRow (shared): the new (v, simulation) pairs
template <bool CONST_T>
__device__ __forceinline__ void small_edge(const BfsSmallArgs& a, const uint32_t* sX, const uint16_t* sS, const uint32_t* dRow,
                                           int e, int W, int32_t* vln, int* c_next) {
                    const uint2 f = a.fwd[e];
                    const uint32_t T = CONST_T ? a.T0 : a.fwdT[e];
                    if (!T) return;
                    int lo, hi;
                    edge_window(f.y, T, sX, sS, a.J, lo, hi);
                    if (lo >= hi) return;
                    // the window's words 8 at a time: only the Delta_u simulations are tested, the visited
                    // words of the 8 are loaded together
                    const int wlo = lo >> 5, whi = (hi - 1) >> 5;
                    for (int wb = wlo; wb <= whi; wb += 8) {
                        uint32_t nv[8], x[8];
    #pragma unroll
                        for (int k = 0; k < 8; k++) {
                            const int w = wb + k;
                            nv[k] = 0u;
                            if (w <= whi) {
                                const int i0 = max(lo, w << 5), i1 = min(hi, (w << 5) + 32);
                                uint32_t cand = dRow[w] & bit_range(i0 & 31, (i1 - 1) & 31);
                                for (; cand; cand &= cand - 1) {
                                    const int q = (w << 5) + __ffs(cand) - 1;
                                    nv[k] |= ((sX[q] ^ f.y) < T) ? (1u << (q & 31)) : 0u;
                                }
                            }
                        }
    #pragma unroll
                        for (int k = 0; k < 8; k++) x[k] = nv[k] ? __ldcg(&a.vd[(size_t)f.x * W + wb + k].x) : 0u;
    #pragma unroll
                        for (int k = 0; k < 8; k++) {
                            const uint32_t n = nv[k] & ~x[k];
                            if (!n) continue;
                            atomicOr(reinterpret_cast<ull*>(&a.vd[(size_t)f.x * W + wb + k]), ((ull)n << 32) | n);
                            if (atomicOr(&a.nbits[f.x], 1u << (wb + k)) == 0u) vln[atomicAdd(c_next, 1)] = (int32_t)f.x;
                        }
                    }
}

template <bool CONST_T>
__global__ void __cluster_dims__(SB_CLUSTER, 1, 1) __launch_bounds__(SB_THREADS) k_bfs_small(BfsSmallArgs a) {
    __shared__ uint32_t sX[1024];
    __shared__ uint16_t sS[4098];
    __shared__ uint32_t sD[SB_THREADS / 32][32];  // Delta row of each warp's frontier vertex
    __shared__ int s_next, s_nlong;                 // the cluster's level counters live in rank 0's copies
    __shared__ unsigned long long s_edges, s_bits;
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = (int)cluster.block_rank(), csize = (int)cluster.num_blocks();
    int* c_next = cluster.map_shared_rank(&s_next, 0);
    int* c_nlong = cluster.map_shared_rank(&s_nlong, 0);
    unsigned long long* c_edges = cluster.map_shared_rank(&s_edges, 0);
    unsigned long long* c_bits = cluster.map_shared_rank(&s_bits, 0);
    const int W = a.J >> 5, lane = threadIdx.x & 31, wib = threadIdx.x >> 5, NWARP = SB_THREADS / 32;
    const int gw = crank * NWARP + wib, GW = csize * NWARP;               // warp index / warps in the cluster
    const int gt = crank * SB_THREADS + threadIdx.x, GT = csize * SB_THREADS;  // thread index / threads
    for (int i = threadIdx.x; i < a.J; i += blockDim.x) sX[i] = a.Xs[i];
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) sS[i] = a.s12[i];
    int cur = a.cur, n_v = a.n_v, levels = 0;
    long long edges_total = 0;
    bool bailed = false;
    __syncthreads();
    while (n_v > 0) {
        const int32_t* vl = cur ? a.vl1 : a.vl0;
        int32_t* vln = cur ? a.vl0 : a.vl1;
        uint32_t* dcur = cur ? a.delta1 : a.delta0;
        uint32_t* dnxt = cur ? a.delta0 : a.delta1;
        if (crank == 0 && threadIdx.x == 0) {
            s_next = 0;
            s_nlong = 0;
            s_edges = 0ull;
            s_bits = 0ull;
        }
        cluster.sync();
        // level: every out-edge of every frontier vertex (warp per vertex over the cluster, lane per edge)
        for (int i = gw; i < n_v; i += GW) {
            const uint32_t u = (uint32_t)vl[i];
            if (lane < W) sD[wib][lane] = dcur[(size_t)u * W + lane];
            __syncwarp();
            const int eb = a.off[u], ee = a.off[u + 1];
            const bool longrow = ee - eb > SB_LONG;
            if (longrow) {  // walked by every warp of the cluster in phase B
                if (lane == 0) a.longv[atomicAdd(c_nlong, 1)] = (int32_t)u;
                continue;
            }
            for (int e = eb + lane; e < ee; e += 32) small_edge<CONST_T>(a, sX, sS, sD[wib], e, W, vln, c_next);
            __syncwarp();
        }
        cluster.sync();
        // phase B: the long rows of the frontier (> SB_LONG out-edges, e.g. hubs), each split over every warp
        // of the cluster (32 edges per warp pass) instead of one warp walking it alone
        const int nlong = *c_nlong;
        for (int li = 0; li < nlong; li++) {
            const uint32_t u = (uint32_t)a.longv[li];
            if (lane < W) sD[wib][lane] = dcur[(size_t)u * W + lane];
            __syncwarp();
            const int eb = a.off[u], ee = a.off[u + 1];
            for (int e = eb + gw * 32 + lane; e < ee; e += GW * 32) small_edge<CONST_T>(a, sX, sS, sD[wib], e, W, vln, c_next);
            __syncwarp();
        }
        if (nlong) cluster.sync();
        // the level's frontier is consumed: clear its Delta rows (this buffer is the next level's output)
        for (int64_t i = gt; i < (int64_t)n_v * W; i += GT) dcur[(size_t)vl[i / W] * W + (i % W)] = 0u;
        const int nn = *c_next;
        // compaction: new bits -> next Delta rows, R_G(S) words and sigma; out-edges of the next frontier
        unsigned long long bits = 0ull, ed = 0ull;
        for (int i = gt; i < nn; i += GT) {
            const uint32_t v = (uint32_t)vln[i];
            uint32_t b = a.nbits[v];
            a.nbits[v] = 0u;
            for (; b; b &= b - 1) {
                const size_t r = (size_t)v * W + (__ffs(b) - 1);
                const uint2 p = a.vd[r];
                dnxt[r] = p.y;
                a.vis[r] = p.x;
                a.vd[r] = make_uint2(p.x, 0u);
                bits += __popc(p.y);
            }
            ed += (unsigned long long)(a.off[v + 1] - a.off[v]);
        }
        bits = __reduce_add_sync(IM_FULL, (uint32_t)bits);  // < 2^32 per warp (<= nn * J bits)
        if (lane == 0 && bits) atomicAdd(c_bits, bits);
        if (ed) atomicAdd(c_edges, ed);
        cluster.sync();
        const unsigned long long lev_edges = *c_edges, lev_bits = *c_bits;
        edges_total += (long long)lev_edges;  // the next level's enumerated edges
        if (crank == 0 && threadIdx.x == 0 && lev_bits) *a.sigma_count += lev_bits;
        levels++;
        cur ^= 1;
        n_v = nn;
        if (n_v > 0 && (long long)lev_edges > a.max_edges) {
            bailed = true;
            break;
        }
        cluster.sync();  // every block has read the counters before rank 0 resets them
    }
    cluster.sync();
    if (crank == 0 && threadIdx.x == 0) {
        a.out->levels = levels;
        a.out->cur = cur;
        a.out->n_v = n_v;
        a.out->bailed = bailed ? 1 : 0;
        a.out->edges = bailed ? edges_total - (long long)s_edges : edges_total;  // rank 0: its own s_edges
        IterCounters z{};
        z.changed = n_v;
        a.ctr[cur] = z;  // the multi-block path builds this frontier's items (k_bfs_items reads .changed)
    }
}

cudaError_t launch_bfs_small(Ctx& c, int cur, int n_v, long long max_edges) {
    BfsSmallArgs a;
    a.J = c.J;
    a.off = c.off;
    a.fwd = c.fwd;
    a.fwdT = c.fwdT;
    a.T0 = c.T0;
    a.Xs = c.Xs;
    a.s12 = c.s12;
    a.vd = c.vd;
    a.vis = c.vis;
    a.nbits = c.nbits;
    a.delta0 = c.delta[0];
    a.delta1 = c.delta[1];
    a.vl0 = c.bvl[0];
    a.vl1 = c.bvl[1];
    a.ctr = c.ctr;
    a.sigma_count = c.sigma_count;
    a.cur = cur;
    a.n_v = n_v;
    a.max_edges = max_edges;
    a.out = c.sbo;
    a.longv = c.big;
    if (c.constT) k_bfs_small<true><<<SB_CLUSTER, SB_THREADS, 0, c.stream>>>(a);
    else k_bfs_small<false><<<SB_CLUSTER, SB_THREADS, 0, c.stream>>>(a);
    return LAUNCHED(c);
}

}  // namespace im
