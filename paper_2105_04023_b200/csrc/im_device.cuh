// im_device.cuh -- device-side helpers of the sm_100a hot path.
// Written from the paper and DESIGN.md; shares no code with oracle/.
#pragma once
#include <cstdint>

#define IM_FULL 0xFFFFFFFFu

namespace im {

// ---------------------------------------------------------------- Murmur3 x86_32
// Eq. 4 hashes the 8-byte key LE32(u) || LE32(v) with seed 0
// (reading R4); Alg. 1 line 4 hashes LE32(v) / LE32(j) with seed_V / seed_J (R5).
// A little-endian 4-byte block read as a word is the value itself, so the block
// loop is unrolled for the two fixed key lengths.
__device__ __forceinline__ uint32_t mm_block(uint32_t h, uint32_t k) {
    k *= 0xcc9e2d51u;
    k = __funnelshift_l(k, k, 15);
    k *= 0x1b873593u;
    h ^= k;
    h = __funnelshift_l(h, h, 13);
    return h * 5u + 0xe6546b64u;
}
__device__ __forceinline__ uint32_t mm_fmix(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}
__device__ __forceinline__ uint32_t murmur_word(uint32_t x, uint32_t seed) { return mm_fmix(mm_block(seed, x) ^ 4u); }
__device__ __forceinline__ uint32_t edge_hash(uint32_t u, uint32_t v) {
    return mm_fmix(mm_block(mm_block(0u, u), v) ^ 8u) & 0x7FFFFFFFu;  // mod 2^31
}

// ---------------------------------------------------------------- Eq. 5 as an integer test
// live(e, j) <=> (X_j xor h_e) / h_max < w_e (double, strict; R1, R7)
//             <=> (X_j xor h_e) < T_e,  T_e = min{x : x / h_max >= w_e}  (division is monotone).
// T_e is computed exactly in double from ceil(w*h_max) and corrected by stepping.
__host__ __device__ inline uint32_t live_threshold(float wf) {
    const double hm = 2147483647.0, w = (double)wf;
    if (!(w > 0.0)) return 0u;
    double c = ceil(w * hm);
    int64_t t = (int64_t)(c > hm ? hm : c);
    while (t > 0 && (double)(t - 1) / hm >= w) --t;
    while (t < 2147483647LL && (double)t / hm < w) ++t;
    return (uint32_t)t;
}

// ---------------------------------------------------------------- sorted-salt windows
// Simulations are stored internally in ascending-salt order.
// For T <= 2^B, (X xor h) < T implies (X >> B) == (h >> B), so the candidate
// simulations of an edge are the contiguous index range of salts in
// [ (h>>B)<<B, ((h>>B)+1)<<B ).  lower_bound over the sorted salts uses a
// 4097-entry table of the first index per 2^19-wide salt bucket.
__device__ __forceinline__ int salt_lb(uint32_t key, const uint32_t* __restrict__ sX, const uint16_t* __restrict__ s12, int J) {
    uint32_t b = key >> 19;  // key <= 2^31 -> b <= 4096
    int i = s12[b];
    if (key & 0x7FFFFu) {
        int e = s12[b + 1];
        while (i < e && sX[i] < key) ++i;
    }
    (void)J;
    return i;
}
__device__ __forceinline__ int thr_bits(uint32_t T) { return T <= 1u ? 0 : 32 - __clz(T - 1u); }
__device__ __forceinline__ void edge_window(uint32_t h, uint32_t T, const uint32_t* sX, const uint16_t* s12, int J,
                                            int& lo, int& hi) {
    int B = thr_bits(T);
    uint32_t klo = (h >> B) << B;
    uint32_t khi = klo + (1u << B);
    lo = salt_lb(klo, sX, s12, J);
    hi = salt_lb(khi, sX, s12, J);
}

// live bits of a sparse window (<= 32 simulations): bit k <=> simulation lo + k is live (Eq. 5)
__device__ __forceinline__ uint32_t window_live_bits(const uint32_t* sX, uint32_t h, uint32_t T, int lo, int hi) {
    uint32_t lb = 0u;
    for (int i = lo; i < hi; ++i) lb |= ((sX[i] ^ h) < T) ? (1u << (i - lo)) : 0u;
    return lb;
}
// the 4 live bits of the aligned simulations 4w .. 4w+3.  No window bounds are needed: the salt of a simulation
// outside the edge's window lies in another 2^B block than h, so (X xor h) >= 2^B >= T.  sX is 16-byte aligned.
__device__ __forceinline__ uint32_t live_nibble(const uint32_t* sX, uint32_t h, uint32_t T, int w) {
    const uint4 x = reinterpret_cast<const uint4*>(sX)[w];
    return ((x.x ^ h) < T ? 1u : 0u) | ((x.y ^ h) < T ? 2u : 0u) | ((x.z ^ h) < T ? 4u : 0u) | ((x.w ^ h) < T ? 8u : 0u);
}
// window_live_bits by aligned 4-simulation words: the first two words (a nominal window of a few simulations)
// in straight-line code with both salt loads in flight, the rest of a long window in a loop.  sX is 16-byte aligned.
__device__ __forceinline__ uint32_t window_live_bits4(const uint32_t* sX, uint32_t h, uint32_t T, int lo, int hi) {
    const int w0 = lo >> 2, w1 = (hi - 1) >> 2, r = lo & 3;
    const uint32_t n0 = live_nibble(sX, h, T, w0);
    const uint32_t n1 = w1 > w0 ? live_nibble(sX, h, T, w0 + 1) : 0u;
    uint32_t lb = (n0 | (n1 << 4)) >> r;
    for (int w = w0 + 2; w <= w1; ++w) lb |= live_nibble(sX, h, T, w) << (4 * (w - w0) - r);
    return lb;
}
// narrow [lo, hi) to its first and last set bit of lb (lb re-based to the new lo); empty if lb == 0
__device__ __forceinline__ void narrow_window(uint32_t& lb, int& lo, int& hi) {
    if (!lb) {
        hi = lo;
        return;
    }
    const int l0 = lo;
    lo = l0 + __ffs(lb) - 1;
    hi = l0 + 32 - __clz(lb);
    lb >>= lo - l0;
}
// the n bits of lb (re-based at lo) that cover simulations s0 .. s0 + n - 1
__device__ __forceinline__ uint32_t bits_at(uint32_t lb, int lo, int s0, int n) {
    const int sh = s0 - lo;
    return (sh >= 0 ? (sh >= 32 ? 0u : lb >> sh) : (-sh >= 32 ? 0u : lb << -sh)) & ((1u << n) - 1u);
}

// Streamed edge records / thresholds / work items are read once per sweep or level: load them with the
// evict-first hint so they do not push the reused register rows (hub rows) out of L2 (IM_STREAM_REC=0: plain)
#ifndef IM_STREAM_REC
#define IM_STREAM_REC 1
#endif
template <class T>
__device__ __forceinline__ T ld_stream(const T* p) {
#if IM_STREAM_REC
    return __ldcs(p);
#else
    return *p;
#endif
}

// byte mask from 4 bits: bit b -> byte b = 0xFF
__device__ __forceinline__ uint32_t expand4(uint32_t b) { return ((b * 0x00204081u) & 0x01010101u) * 0xFFu; }

// bits c0..c1 (inclusive), 0 <= c0 <= c1 <= 31
__device__ __forceinline__ uint32_t bit_range(int c0, int c1) {
    uint32_t hi = (c1 >= 31) ? IM_FULL : ((1u << (c1 + 1)) - 1u);
    return hi & ~((1u << c0) - 1u);
}

// Eq. 3 on one 4-register word of a row in global memory: *p = max_bytewise(*p, val).
// Registers only grow, so a stale `cur` is a lower bound and the CAS loop corrects it.
// Returns true iff some register of *p increased.
__device__ __forceinline__ bool atomic_vmax4(uint32_t* p, uint32_t val) {
    uint32_t cur = __ldcg(p);
    uint32_t nw = __vmaxu4(cur, val);
    while (nw != cur) {
        uint32_t prev = atomicCAS(p, cur, nw);
        if (prev == cur) return true;
        cur = prev;
        nw = __vmaxu4(cur, val);
    }
    return false;
}

__device__ __forceinline__ int warp_incl_scan(int x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(IM_FULL, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

}  // namespace im

namespace im {
// Block-aggregated reservation on the per-iteration counters (one atomic per counter per block
// iteration instead of one per warp).  Every thread of the block calls it; lane 31 of each warp
// passes its warp's totals.  Returns the warp's base for items / changed / big.
struct BlockTotals {
    int items, changed, big;
    unsigned long long edges;
};
template <int NW>
__device__ __forceinline__ void block_reserve(BlockTotals wt, int lane, int wib, int* c_items, int* c_changed,
                                              unsigned long long* c_edges, int* c_big, int& b_items, int& b_changed,
                                              int& b_big) {
    __shared__ BlockTotals sT[NW];
    __shared__ int sB[NW][3];
    if (lane == 31) sT[wib] = wt;
    __syncthreads();
    if (threadIdx.x < 4) {
        const int t = threadIdx.x;
        unsigned long long acc = 0;
        for (int w = 0; w < NW; w++) {
            unsigned long long x = t == 0 ? sT[w].items : t == 1 ? sT[w].changed : t == 2 ? sT[w].big : sT[w].edges;
            if (t < 3) sB[w][t] = (int)acc;
            acc += x;
        }
        if (acc) {
            if (t == 3) {
                if (c_edges) atomicAdd(c_edges, acc);
            } else {
                int* cp = t == 0 ? c_items : t == 1 ? c_changed : c_big;
                int g0 = cp ? atomicAdd(cp, (int)acc) : 0;
                for (int w = 0; w < NW; w++) sB[w][t] += g0;
            }
        }
    }
    __syncthreads();
    b_items = sB[wib][0];
    b_changed = sB[wib][1];
    b_big = sB[wib][2];
    __syncthreads();
}
}  // namespace im

