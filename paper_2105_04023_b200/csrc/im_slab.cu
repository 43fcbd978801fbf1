// im_slab.cu -- the full sweeps of a build (Alg. 2: every vertex live) in bucket-major
// ("slab") form.  DESIGN.md section 6 "slab passes".
//
// With a constant threshold T <= 2^B an edge (u,v) with hash h can only be live (Eq. 5, PAPER.md:231:
// (X_j xor h) < T) in the simulations j whose salt X_j lies in h's 2^B block.  Simulations never interact
// (Eq. 1-5 are per simulation), so the fixpoint of Alg. 2 decomposes by salt bucket: bucket b's
// simulations only ever read and write the registers of bucket b's simulations, over bucket b's edges.
// A row-major sweep touches one random 32-byte sector of an n x J byte array (8.6 GB on RMAT-24) per
// edge, from HBM.  Here the edges are grouped by bucket once per graph (im_prep.cu) and the registers of
// <= 4 simulations of one bucket are held as one packed 32-bit word per vertex -- a slab of 4n bytes
// (67 MB for 16.8M vertices), which stays in the 126 MB L2 while all SMs sweep that bucket's edges: an edge
// costs its streamed 12-byte record and two L2 hits.  A build runs, per group of <= 4 simulations,
//   init   S[u] = clz(hash(u) xor hash(j)) per simulation (Alg. 1 line 4); a simulation in which u is
//          blocked (u in R_S[j], Alg. 2) gets bit 7 set, so no later max can change it;
//   passes in place (the fixpoint is unique, R11): S[u] <- max(S[u], S[v] & live) per edge;
//   last pass also records which registers it raised (they are what the push sweeps still have to
//          propagate);
// then one transpose writes the row-major registers M, the per-simulation change masks and the chunk
// bits that the sparse push sweeps (im_sweep.cu) continue from.
//
// STATUS: opt-in (IM_SLAB_PASSES=3; default 0 = off).  Bit-exact on every parity test, but measured SLOWER than
// the row-major gather sweeps on RMAT-24: a pass over one bucket's 4M edges is three
// dependent memory phases of a bulk-synchronous grid (58-68 us against the ~25 us its L2 traffic allows),
// the slab's L2 hit rate is ~50% next to the 48 MB of records streamed per pass, and pinning it with a
// persisting-L2 window takes the carve-out away from every other kernel of the step.
#include <algorithm>

#include "im_device.cuh"
#include "im_internal.h"

namespace im {

constexpr int SLAB_MAXG = 1024;      // groups per build (J / 4 + buckets <= 256 + 256 for J <= 1024)
constexpr int SLAB_MAX_VISITS = 48;  // edge visits per pass as a multiple of m above which the slab path is not taken

// Groups of <= 4 consecutive (ascending-salt) simulations of one bucket h >> Bs.
int slab_group_count(Ctx& c) {
    c.slabG_h.clear();
    if (!c.brec || c.slab_passes <= 0 || c.boff_h.empty() || (int)c.Xs_h.size() != c.J) return 0;
    const int nb = 1 << (31 - c.Bs);
    double visits = 0.0;
    int i = 0;
    for (int b = 0; b < nb; b++) {
        int lo = i;
        while (i < c.J && (int)(c.Xs_h[i] >> c.Bs) == b) i++;
        const int mb = c.boff_h[b + 1] - c.boff_h[b];
        for (int s0 = lo; s0 < i; s0 += 4) {
            const int cnt = std::min(4, i - s0);
            c.slabG_h.push_back(make_int4(s0, cnt, b, (int)(cnt == 4 ? 0xFFFFFFFFu : ((1u << (8 * cnt)) - 1u))));
            visits += mb;
        }
    }
    if (i != c.J || (int)c.slabG_h.size() > SLAB_MAXG || visits > (double)SLAB_MAX_VISITS * (double)c.m) c.slabG_h.clear();
    return (int)c.slabG_h.size();
}

// salts and hash(j) of every group's simulations (pads: 0)
__global__ void k_slab_groups(int G, const int4* __restrict__ grp, const uint32_t* __restrict__ Xs, const int32_t* __restrict__ perm,
                              uint32_t seedJ, uint4* __restrict__ gX, uint4* __restrict__ gHJ) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    const int4 q = grp[g];
    uint32_t x[4] = {0u, 0u, 0u, 0u}, hj[4] = {0u, 0u, 0u, 0u};
    for (int k = 0; k < q.y; k++) {
        x[k] = Xs[q.x + k];
        hj[k] = murmur_word((uint32_t)perm[q.x + k], seedJ);
    }
    gX[g] = make_uint4(x[0], x[1], x[2], x[3]);
    gHJ[g] = make_uint4(hj[0], hj[1], hj[2], hj[3]);
}

// init values (Alg. 1 line 4), a thread per vertex, SIG consecutive groups per blockIdx.y (their simulations share
// one or two words of u's visited bits, so a rebuild reads each vis sector once per SIG groups); bit 7 marks a
// blocked (u, j)
constexpr int SIG = 8;
template <bool BLOCKED>
__global__ void __launch_bounds__(BLOCK) k_slab_init(int32_t n, size_t ns, int J, int G, uint32_t seedV, const int4* __restrict__ grp,
                                                    const uint4* __restrict__ gHJ, const uint32_t* __restrict__ vis,
                                                    uint32_t* __restrict__ S) {
    const int W = J >> 5, g0 = blockIdx.y * SIG, g1 = min(G, g0 + SIG);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
        const uint32_t hu = murmur_word((uint32_t)u, seedV);
        for (int g = g0; g < g1; g++) {
            const int4 q = __ldg(&grp[g]);
            const uint4 hj = __ldg(&gHJ[g]);
            uint32_t w = (uint32_t)__clz(hu ^ hj.x) | ((uint32_t)__clz(hu ^ hj.y) << 8) | ((uint32_t)__clz(hu ^ hj.z) << 16) |
                         ((uint32_t)__clz(hu ^ hj.w) << 24);
            w &= (uint32_t)q.w;
            if (BLOCKED) {
                const int w0 = q.x >> 5, w1 = (q.x + q.y - 1) >> 5;
                const ull m = (ull)vis[(size_t)u * W + w0] | ((ull)(w1 != w0 ? vis[(size_t)u * W + w1] : 0u) << 32);
                const uint32_t b = (uint32_t)(m >> (q.x & 31)) & ((1u << q.y) - 1u);
                w |= (expand4(b) & 0x80808080u);
            }
            S[(size_t)g * ns + u] = w;
        }
    }
}

// one in-place pass over the edges [e0, e1) of the group's bucket: S[u] <- max(S[u], S[v] & live)
constexpr int SU = 4;  // edges per thread per iteration (records, then the S[v] and S[u] loads in flight together)
template <bool LAST>
__global__ void __launch_bounds__(BLOCK) k_slab_pass(int e0, int e1, const uint2* __restrict__ brec, const int32_t* __restrict__ bv,
                                                    uint4 X, uint32_t T, uint32_t bmask, uint32_t* __restrict__ S,
                                                    uint32_t* __restrict__ C32) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    // warp-uniform trip count (the shuffles below need every lane); the next iteration's records are loaded
    // before this one's are worked on
    int64_t wb = (int64_t)e0 + blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    uint2 rn[SU];
    int vn[SU];
#pragma unroll
    for (int k = 0; k < SU; k++) {
        const int64_t e = wb + lane + k * stride;
        rn[k] = e < e1 ? ld_stream(&brec[e]) : make_uint2(0u, 0u);
        vn[k] = e < e1 ? ld_stream(&bv[e]) : -1;
    }
    for (; wb < e1; wb += SU * stride) {
        uint2 r[SU];
        int v[SU];
#pragma unroll
        for (int k = 0; k < SU; k++) {
            r[k] = rn[k];
            v[k] = vn[k];
        }
        uint32_t live[SU], sv[SU], su[SU];
#pragma unroll
        for (int k = 0; k < SU; k++) {
            const uint32_t h = r[k].y;
            live[k] = (((X.x ^ h) < T ? 0x000000FFu : 0u) | ((X.y ^ h) < T ? 0x0000FF00u : 0u) | ((X.z ^ h) < T ? 0x00FF0000u : 0u) |
                       ((X.w ^ h) < T ? 0xFF000000u : 0u)) & bmask;  // Eq. 5 for the group's simulations
            if (v[k] < 0) live[k] = 0u;
            sv[k] = live[k] ? __ldcg(&S[v[k]]) : 0u;
            su[k] = live[k] ? __ldcg(&S[r[k].x]) : 0u;  // lanes of one source share the sector
        }
        if (wb + SU * stride < e1) {
#pragma unroll
            for (int k = 0; k < SU; k++) {
                const int64_t e = wb + SU * stride + lane + k * stride;
                rn[k] = e < e1 ? ld_stream(&brec[e]) : make_uint2(0u, 0u);
                vn[k] = e < e1 ? ld_stream(&bv[e]) : -1;
            }
        }
        // Edges of one source are neighbours in the bucket list (it keeps the forward row order inside a partition
        // unit), and a hub has thousands per bucket: their candidates are max-reduced over the lanes holding the
        // same u first (segmented scan), and only the last lane of a run touches S[u] -- otherwise every edge of a
        // hub issues a CAS on one word and the pass serialises on that address.
#pragma unroll
        for (int k = 0; k < SU; k++) {
            sv[k] &= live[k] & 0x7F7F7F7Fu;  // a blocked v still offers its (init) value; the mark is not a value
            const uint32_t u = r[k].x;
            if (__any_sync(IM_FULL, sv[k] != 0u)) {
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(IM_FULL, sv[k], o), uy = __shfl_up_sync(IM_FULL, u, o);
                    if (lane >= o && uy == u) sv[k] = __vmaxu4(sv[k], y);
                }
                const uint32_t un = __shfl_down_sync(IM_FULL, u, 1);
                if (lane < 31 && un == u) sv[k] = 0u;  // not the last lane of its run
            }
        }
#pragma unroll
        for (int k = 0; k < SU; k++) {
            if (!sv[k]) continue;
            uint32_t cur = su[k], nw = __vmaxu4(cur, sv[k]);  // a marked (blocked) byte of S[u] is >= 0x80: never raised
            uint32_t raised = 0u;
            while (nw != cur) {
                const uint32_t prev = atomicCAS(&S[r[k].x], cur, nw);
                if (prev == cur) {
                    raised = ((((~__vcmpeq4(cur, nw)) & 0x01010101u) * 0x00204081u) >> 21) & 0xFu;
                    break;
                }
                cur = prev;
                nw = __vmaxu4(cur, sv[k]);
            }
            if (LAST && raised) atomicOr(&C32[r[k].x >> 2], raised << ((r[k].x & 3u) << 3));
        }
    }
}

// slabs -> row-major registers, per-simulation change masks and chunk bits, 32 vertices per block iteration
__global__ void __launch_bounds__(BLOCK) k_slab_finish(int32_t n, size_t ns, int J, int G, const int4* __restrict__ grp,
                                                      const uint32_t* __restrict__ S, const uint8_t* __restrict__ C,
                                                      uint8_t* __restrict__ M, uint32_t* __restrict__ cm_out,
                                                      uint32_t* __restrict__ bits_out) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int RS = J + 4, W = J >> 5;  // row stride in bytes: lanes (vertices) of a warp hit different banks
    uint8_t* rows = sm;
    uint32_t* cmt = reinterpret_cast<uint32_t*>(sm + (size_t)32 * RS);  // [32][W + 1]
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, NWP = blockDim.x >> 5;
    const int ntiles = (n + 31) >> 5;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int u0 = tile << 5, u = u0 + lane;
        for (int i = threadIdx.x; i < 32 * (W + 1); i += blockDim.x) cmt[i] = 0u;
        __syncthreads();
        constexpr int FB = 8;  // groups per warp iteration: their slab words and change bytes are loaded together
        for (int g0 = wib * FB; g0 < G; g0 += NWP * FB) {
            uint32_t wv[FB], cv[FB];
#pragma unroll
            for (int i = 0; i < FB; i++) {
                const int g = g0 + i;
                wv[i] = cv[i] = 0u;
                if (g < G && u < n) {
                    wv[i] = __ldcs(&S[(size_t)g * ns + u]) & 0x7F7F7F7Fu;
                    cv[i] = __ldcs(&C[(size_t)g * ns + u]);
                }
            }
#pragma unroll
            for (int i = 0; i < FB; i++) {
                const int g = g0 + i;
                if (g >= G) break;
                const int4 q = __ldg(&grp[g]);
                for (int k = 0; k < q.y; k++) rows[(size_t)lane * RS + q.x + k] = (uint8_t)(wv[i] >> (8 * k));
                if (cv[i]) {
                    const int w0 = q.x >> 5, sh = q.x & 31;
                    atomicOr(&cmt[lane * (W + 1) + w0], cv[i] << sh);
                    if (sh + q.y > 32) atomicOr(&cmt[lane * (W + 1) + w0 + 1], cv[i] >> (32 - sh));
                }
            }
        }
        __syncthreads();
        for (int r = wib; r < 32; r += NWP) {
            if (u0 + r >= n) break;
            const uint32_t* src = reinterpret_cast<const uint32_t*>(rows + (size_t)r * RS);
            uint32_t* dst = reinterpret_cast<uint32_t*>(M + (size_t)(u0 + r) * J);
            for (int w = lane; w < (J >> 2); w += 32) dst[w] = src[w];
            const uint32_t x = lane < W ? cmt[r * (W + 1) + lane] : 0u;
            if (lane < W) cm_out[(size_t)(u0 + r) * W + lane] = x;
            const uint32_t chunks = __ballot_sync(IM_FULL, x != 0u);
            if (lane == 0) bits_out[u0 + r] = chunks;
        }
        __syncthreads();
    }
}

cudaError_t launch_slab_build(Ctx& c, bool blocked, int passes, uint32_t* cm_out, uint32_t* bits_out) {
    cudaError_t e;
    const int G = (int)c.slabG_h.size();
    const int n = c.n;
    const size_t ns = slab_stride(n);
    if ((e = cudaMemcpyAsync(c.slabG, c.slabG_h.data(), (size_t)G * sizeof(int4), cudaMemcpyHostToDevice, c.stream))) return e;
    k_slab_groups<<<(G + 127) / 128, 128, 0, c.stream>>>(G, c.slabG, c.Xs, c.permd, c.seedJ, c.slabX, c.slabHJ);
    if ((e = LAUNCHED(c))) return e;
    std::vector<uint4> hX(G);
    if ((e = cudaMemcpyAsync(hX.data(), c.slabX, (size_t)G * sizeof(uint4), cudaMemcpyDeviceToHost, c.stream))) return e;
    const dim3 gi((unsigned)std::min<int64_t>(((int64_t)n + BLOCK * 4 - 1) / (BLOCK * 4), c.num_sms * 2), (unsigned)((G + SIG - 1) / SIG));
    if (blocked) k_slab_init<true><<<gi, BLOCK, 0, c.stream>>>(n, ns, c.J, G, c.seedV, c.slabG, c.slabHJ, c.vis, c.slabS);
    else k_slab_init<false><<<gi, BLOCK, 0, c.stream>>>(n, ns, c.J, G, c.seedV, c.slabG, c.slabHJ, c.vis, c.slabS);
    if ((e = LAUNCHED(c))) return e;
    if ((e = cudaMemsetAsync(c.slabC, 0, (size_t)G * ns, c.stream))) return e;
    if ((e = cudaStreamSynchronize(c.stream))) return e;  // hX
    const int grid = c.num_sms * 8;
    for (int g = 0; g < G; g++) {
        const int4 q = c.slabG_h[g];
        const int e0 = c.boff_h[q.z], e1 = c.boff_h[q.z + 1];
        if (e0 == e1) continue;
        uint32_t* S = c.slabS + (size_t)g * ns;
        uint32_t* C32 = reinterpret_cast<uint32_t*>(c.slabC + (size_t)g * ns);
        const int gg = (int)std::min<int64_t>(grid, ((int64_t)(e1 - e0) + BLOCK * SU - 1) / (BLOCK * SU));
        for (int p = 0; p < passes; p++) {
            if (p + 1 < passes) k_slab_pass<false><<<gg, BLOCK, 0, c.stream>>>(e0, e1, c.brec, c.bv, hX[g], c.T0, (uint32_t)q.w, S, C32);
            else k_slab_pass<true><<<gg, BLOCK, 0, c.stream>>>(e0, e1, c.brec, c.bv, hX[g], c.T0, (uint32_t)q.w, S, C32);
            if ((e = LAUNCHED(c))) return e;
        }
    }
    const size_t smem = (size_t)32 * (c.J + 4) + (size_t)32 * (c.J / 32 + 1) * sizeof(uint32_t);
    static bool attr = false;
    if (!attr) {
        if ((e = cudaFuncSetAttribute(k_slab_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024))) return e;
        attr = true;
    }
    k_slab_finish<<<c.num_sms * 4, BLOCK, smem, c.stream>>>(n, ns, c.J, G, c.slabG, c.slabS, c.slabC, c.M, cm_out, bits_out);
    return LAUNCHED(c);
}

}  // namespace im
