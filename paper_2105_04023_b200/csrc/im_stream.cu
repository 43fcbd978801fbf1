// im_stream.cu -- the full argmax pass (Alg. 1 line 10) as a TMA-bulk streaming
// kernel: every greedy step that cannot use the lazy candidate list reads all n*J registers and
// n*J/8 visited bits once, so the pass is a pure HBM stream.  Tiles of consecutive vertex rows are
// moved into shared memory by cp.async.bulk (the 1-D TMA path) through a 3-stage mbarrier ring
// issued by one thread; the 8 warps compute gains from shared memory.  Same arithmetic and outputs
// as k_argmax<POOL, false> (im_kernels.cu): stored gains, gain histogram, exact argmax key.
#include "im_device.cuh"
#include "im_internal.h"

namespace im {

constexpr int TS = 3;                 // pipeline stages
constexpr int TILE_M = 24576;         // register bytes per tile (TV ~ TILE_M / J vertices; 2 blocks per SM fit)
constexpr int HBINS = 4096;           // == HIST_BINS (im_kernels.cu)
constexpr int TC = 8;                 // max 16-byte chunks per lane (J <= 1024, L = 8)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    long long spins = 0;
    while (!mbar_try_wait(bar, parity))
        if (++spins > (1LL << 32)) __trap();  // fail loudly instead of hanging
}

__device__ __forceinline__ uint32_t gain16x2_s(uint4 x, uint4 m) {
    return __vsadu4(x.x, m.x) + __vsadu4(x.y, m.y) + __vsadu4(x.z, m.z) + __vsadu4(x.w, m.w) + __vsadu4(x.x, 0u) +
           __vsadu4(x.y, 0u) + __vsadu4(x.z, 0u) + __vsadu4(x.w, 0u);
}

// rows of tile t: vertices [t*TV, min(n, (t+1)*TV)); M and vis carry 64 KB of padding so the last
// tile may read past row n; TV is a multiple of 8 * (vertices per warp), so every bulk copy is a
// whole multiple of 16 bytes at a 16-byte aligned address and the per-warp loop is uniform
// SHARD: this rank holds only its simulations; gain_out[v] = local gain + (not fully visited) << 24
// for every v (the allreduce SUM over ranks then k_argmax_decode give the global gains / pool)
template <bool POOL, bool SHARD>
__global__ void __launch_bounds__(BLOCK) k_argmax_tma(int32_t n, int32_t J, int L, int C, const uint8_t* __restrict__ M,
                                                      const uint8_t* __restrict__ MS, const uint32_t* __restrict__ vis,
                                                      ull* key, int32_t* gain_out, uint32_t* hist, int shift, int TV) {
    extern __shared__ __align__(128) uint8_t dyn[];
    __shared__ __align__(8) uint64_t full[TS];
    __shared__ uint4 sMS[64];
    __shared__ ull sKey[BLOCK / 32];
    __shared__ uint32_t sHist[HBINS];
    const int nch = J >> 4, W = J >> 5;
    const uint32_t mbytes = (uint32_t)(TV * J), vbytes = (uint32_t)(TV * W * 4);
    const uint32_t stage_bytes = (mbytes + (POOL ? vbytes : 0u) + 127u) & ~127u;
    const int ntiles = (n + TV - 1) / TV;
    for (int i = threadIdx.x; i < nch; i += blockDim.x) sMS[i] = reinterpret_cast<const uint4*>(MS)[i];
    for (int i = threadIdx.x; i < HBINS; i += blockDim.x) sHist[i] = 0u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < TS; s++) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int t, int s) {  // thread 0 only
        uint8_t* dst = dyn + (size_t)s * stage_bytes;
        const size_t v0 = (size_t)t * TV;
        mbar_expect_tx(&full[s], mbytes + (POOL ? vbytes : 0u));
        bulk_g2s(dst, M + v0 * J, mbytes, &full[s]);
        if (POOL) bulk_g2s(dst + mbytes, vis + v0 * W, vbytes, &full[s]);
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < TS; s++) {
            int t = blockIdx.x + s * gridDim.x;
            if (t < ntiles) issue(t, s);
        }
    // L lanes per vertex (<= 8), chunk c of lane q = 16-byte chunk c*L + q of the row: the L lanes of a
    // vertex read one contiguous 16*L-byte run per c (conflict-free), C <= TC chunks per lane
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, q = lane & (L - 1), sub = lane / L, VPW = 32 / L;
    uint4 ms[TC];
    uint32_t msum = 0;
#pragma unroll
    for (int c = 0; c < TC; c++) {
        const int ci = c * L + q;
        ms[c] = (c < C && ci < nch) ? sMS[ci] : make_uint4(0, 0, 0, 0);
        msum += __vsadu4(ms[c].x, 0u) + __vsadu4(ms[c].y, 0u) + __vsadu4(ms[c].z, 0u) + __vsadu4(ms[c].w, 0u);
    }
    ull best = 0;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int s = it % TS;
        mbar_wait(&full[s], (uint32_t)((it / TS) & 1));
        const uint8_t* tileM = dyn + (size_t)s * stage_bytes;
        const uint32_t* tileV = reinterpret_cast<const uint32_t*>(tileM + mbytes);
        const int v0 = t * TV;
        for (int r = wib * VPW + sub; r < TV; r += (BLOCK / 32) * VPW) {  // uniform per warp: TV is a multiple of VPW*8
            const int v = v0 + r;
            const bool ok = v < n;
            uint32_t gn = 0;
#pragma unroll
            for (int c = 0; c < TC; c++) {
                const int ci = c * L + q;
                if (c < C && ci < nch) gn += gain16x2_s(reinterpret_cast<const uint4*>(tileM + (size_t)r * J)[ci], ms[c]);
            }
            gn -= msum;
            int fullrow = 1;
            if (POOL)
                for (int w = q; w < W; w += L) fullrow &= tileV[r * W + w] == IM_FULL;
            for (int o = L >> 1; o; o >>= 1) {
                gn += __shfl_xor_sync(IM_FULL, gn, o);
                if (POOL) fullrow &= __shfl_xor_sync(IM_FULL, fullrow, o);
            }
            gn >>= 1;
            const bool inpool = ok && (!POOL || !fullrow);
            if (SHARD) {
                if (ok && q == 0) gain_out[v] = (int32_t)(gn + (inpool ? SHARD_POOL_ONE : 0u));
                continue;
            }
            if (ok && q == 0) {
                if (inpool) {
                    ull k = ((ull)gn << 32) | (ull)(0xFFFFFFFFu - (uint32_t)v);
                    best = k > best ? k : best;
                    atomicAdd(&sHist[min((int)(gn >> shift), HBINS - 1)], 1u);
                }
                gain_out[v] = inpool ? (int32_t)gn : -1;
            }
        }
        __syncthreads();  // stage s fully consumed
        if (threadIdx.x == 0) {
            int tn = t + TS * gridDim.x;
            if (tn < ntiles) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(tn, s);
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ull ob = __shfl_xor_sync(IM_FULL, best, o);
        best = ob > best ? ob : best;
    }
    if (lane == 0) sKey[wib] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        ull b = 0;
        for (int i = 0; i < BLOCK / 32; i++) b = sKey[i] > b ? sKey[i] : b;
        if (b) atomicMax(key, b);
    }
    for (int i = threadIdx.x; i < HBINS; i += blockDim.x)
        if (sHist[i]) atomicAdd(&hist[i], sHist[i]);
}

// a multiple of the vertices per warp (uniform warp loop) and of 16 (16-byte aligned bulk copies of
// the TV*J register bytes and TV*J/8 visited bytes)
static int tma_tv(int J, int L) {
    const int vpw = 32 / L, step = vpw > 16 ? vpw : 16;
    int tv = (TILE_M / J) / step * step;
    return tv < step ? step : tv;
}
// lanes per vertex and chunks per lane of the TMA pass: L = min(8, pow2 >= J/16), C = ceil(J/16 / L)
static void tma_geometry(int J, int& L, int& C) {
    const int nch = J >> 4;
    L = 1;
    while (L < 8 && L < nch) L <<= 1;
    C = (nch + L - 1) / L;
}

static size_t tma_smem(int J, int TV, bool pool) {
    const int W = J >> 5;
    const size_t stage = ((size_t)TV * J + (pool ? (size_t)TV * W * 4 : 0) + 127) & ~(size_t)127;
    return TS * stage + 128;
}

int setup_argmax_tma() {
    const int dyn = 3 * (TILE_M + 4096 + 128) + 128;  // >= tma_smem for every J
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_argmax_tma<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn))) return (int)e;
    if ((e = cudaFuncSetAttribute(k_argmax_tma<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn))) return (int)e;
    if ((e = cudaFuncSetAttribute(k_argmax_tma<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn))) return (int)e;
    return (int)cudaFuncSetAttribute(k_argmax_tma<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
}

cudaError_t launch_argmax_tma(Ctx& c, bool pool, int L, int C, int shift) {
    tma_geometry(c.J, L, C);
    const int TV = tma_tv(c.J, L), ntiles = (c.n + TV - 1) / TV;
    const int grid = ntiles < c.num_sms * 2 ? ntiles : c.num_sms * 2;
    const size_t smem = tma_smem(c.J, TV, pool);
    const bool sh = c.ar;
    auto kf = pool ? (sh ? k_argmax_tma<true, true> : k_argmax_tma<true, false>)
                   : (sh ? k_argmax_tma<false, true> : k_argmax_tma<false, false>);
    kf<<<grid, BLOCK, smem, c.stream>>>(c.n, c.J, L, C, c.M, c.MS, c.vis, c.key, c.gain, c.hist, shift, TV);
    return LAUNCHED(c);
}

}  // namespace im
