// im_prep.cu -- a0 edge preparation (Eq. 4-5, Sec. 3.3) and a2 register init (Alg. 1 lines 2-5).
//
// Edge prep, once per graph:
//   validate the CSR; detect a constant w; per edge h(u,v) = Murmur3(u||v) mod 2^31 and the exact
//   integer threshold T_e (im_device.cuh); build the forward rows {v, h} and the reverse rows {u, h}
//   (grouped by target) used by the sweeps.  With a constant threshold T (2^(B-1) < T <= 2^B) every
//   row is additionally ordered by h >> B, so the slice of a row whose candidate windows meet a
//   given simulation range is contiguous (im_device.cuh "hash-sorted adjacency ranges").  Both
//   orders come from one LSD radix sort of the composite key (row << (31-B)) | (h >> B); the row
//   part keeps CSR rows contiguous, so the sort doubles as the transpose.  Per-edge thresholds
//   (weighted cascade) keep the input row order and use an atomic-cursor transpose.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "im_device.cuh"
#include "im_internal.h"

namespace im {

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

// source vertex of every edge: the start position of each non-empty row gets its id, then a max-scan
__global__ void k_row_markers(int32_t n, const int32_t* __restrict__ off, int32_t* __restrict__ mark) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += stride)
        if (off[u] < off[u + 1]) mark[off[u]] = (int32_t)u;
}

struct MaxOp {
    __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

// forward records (+ composite sort keys when SORTED); in-degree histogram
template <typename K, bool SORTED>
__global__ void k_edge_prep(int64_t m, const int32_t* __restrict__ src, const int32_t* __restrict__ tgt,
                            const float* __restrict__ prob, int B, int KB, K* __restrict__ keys, uint2* __restrict__ rec,
                            uint32_t* __restrict__ recT, int32_t* __restrict__ indeg) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += stride) {
        uint32_t u = (uint32_t)src[e], v = (uint32_t)tgt[e];
        uint32_t h = edge_hash(u, v);
        rec[e] = make_uint2(v, h);
        if (SORTED) keys[e] = ((K)u << KB) | (K)(h >> B);
        else recT[e] = live_threshold(prob[e]);
        atomicAdd(&indeg[v], 1);
    }
}

// reverse records {u, h} keyed by (v << KB) | (h >> B); fwd is already row-ordered, so src[e] is its row
template <typename K>
__global__ void k_rev_keys(int64_t m, const int32_t* __restrict__ src, const uint2* __restrict__ fwd, int B, int KB,
                           K* __restrict__ keys, uint2* __restrict__ rec) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += stride) {
        uint2 f = fwd[e];
        keys[e] = ((K)f.x << KB) | (K)(f.y >> B);
        rec[e] = make_uint2((uint32_t)src[e], f.y);
    }
}

// per-edge thresholds: atomic-cursor transpose (row order inside reverse rows is immaterial)
__global__ void k_transpose(int64_t m, const int32_t* __restrict__ src, const uint2* __restrict__ fwd,
                            const uint32_t* __restrict__ fwdT, const int32_t* __restrict__ roff, int32_t* __restrict__ cursor,
                            uint2* __restrict__ rev, uint32_t* __restrict__ revT) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += stride) {
        uint2 f = fwd[e];
        int32_t pos = roff[f.x] + atomicAdd(&cursor[f.x], 1);
        rev[pos] = make_uint2((uint32_t)src[e], f.y);
        revT[pos] = fwdT[e];
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

// ------------------------------------------------------------------ bucket-ordered rows (constant T)
// With one threshold T (2^(B-1) < T <= 2^B) a row only has to be grouped by bucket b = h >> B
// (KB = 31 - B bits); the order inside a bucket is immaterial (every consumer takes the slice of
// a bucket range, im_device.cuh "hash-sorted adjacency ranges").  For KB <= 8 the forward rows
// are ordered in place by a row-local counting sort instead of a full-width radix sort of m keys:
//   k_rows       forward row u: h = Murmur3(u||v) mod 2^31 (Eq. 4), records {v, h} written in
//                bucket order; at the edge's input position, the reverse sort key (v << KB) | b
//                and payload {u, h} (coalesced; the radix sort of these is the transpose)
//   radix sort   reverse records grouped by v, bucket-ordered inside (one LSD sort)
//   k_row_bounds reverse offsets from the sorted keys (no in-degree atomics)
// Rows of at most 32 edges are ranked inside one warp by a radix ballot; rows up to PREP_BIG by a
// warp with a shared-memory histogram; longer rows by a whole block (k_rows_big).
constexpr int PREP_BIG = 2048;
constexpr int PREP_KB_MAX = 8;

__global__ void k_list_long(int32_t n, const int32_t* __restrict__ off, int32_t* __restrict__ lf, int* count) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += stride)
        if (off[u + 1] - off[u] > PREP_BIG) lf[atomicAdd(count, 1)] = (int32_t)u;
}

template <typename K>
struct RowSortArgs {
    int32_t n;
    int B, KB;
    const int32_t* off;     // forward row offsets
    const int32_t* tgt;     // input targets (CSR order)
    uint2* out;             // bucket-ordered forward records {v, h}
    K* rkey;                // reverse sort keys (v << KB) | b, input order
    uint2* rval;            // reverse payload {u, h}, input order
    const int32_t* lst;     // k_rows_big: rows longer than PREP_BIG
    const int* lcount;
    int* batch;             // dynamic row-batch cursor (zeroed)
    const int32_t* tidx;    // bucket offset table of each row (-1: none), tables tab[rows x nbk]
    int32_t* tab;
    int nbk;
};

// the bucket offsets of a row with a table: hist holds the exclusive scan of its bucket counts
template <typename K>
__device__ __forceinline__ void write_row_table(const RowSortArgs<K>& a, uint32_t u, int eb, int ee, const int* hist, int NB,
                                                int tid, int nthreads) {
    const int t = a.tidx ? a.tidx[u] : -1;
    if (t < 0) return;
    int32_t* tb = a.tab + (int64_t)t * a.nbk;
    for (int kb = tid; kb <= NB; kb += nthreads) tb[kb] = kb < NB ? eb + hist[kb] : ee;
}

// record {v, h(u,v)} of input edge e of row u (+ its reverse key and payload on the first visit)
template <typename K>
__device__ __forceinline__ uint2 row_rec(const RowSortArgs<K>& a, int64_t e, uint32_t u, bool first) {
    const uint32_t v = (uint32_t)a.tgt[e];
    const uint32_t h = edge_hash(u, v);
    if (first) {
        a.rkey[e] = ((K)v << a.KB) | (K)(h >> a.B);
        a.rval[e] = make_uint2(u, h);
    }
    return make_uint2(v, h);
}

// rank of this lane's key among the lanes of `act` (keys < mine, then equal keys of lower lanes)
__device__ __forceinline__ int ballot_rank(uint32_t b, int KB, uint32_t act, int lane) {
    uint32_t eq = act;
    int less = 0;
    for (int k = KB - 1; k >= 0; --k) {
        const uint32_t bit = (b >> k) & 1u;
        const uint32_t bk = __ballot_sync(IM_FULL, bit);
        if (bit) {
            less += __popc(eq & ~bk);
            eq &= bk;
        } else {
            eq &= ~bk;
        }
    }
    return less + __popc(eq & ((1u << lane) - 1u));
}

// exclusive scan of NB <= 256 shared counters by one warp (lane owns NB/32 consecutive bins)
__device__ __forceinline__ void warp_scan_bins(int* hist, int NB, int lane) {
    const int per = (NB + 31) >> 5;
    int loc[8], s = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
        loc[q] = q < per && lane * per + q < NB ? hist[lane * per + q] : 0;
        s += loc[q];
    }
    int run = warp_incl_scan(s, lane) - s;
#pragma unroll
    for (int q = 0; q < 8; q++)
        if (q < per && lane * per + q < NB) {
            hist[lane * per + q] = run;
            run += loc[q];
        }
}

template <typename K>
__global__ void __launch_bounds__(BLOCK) k_rows(RowSortArgs<K> a) {
    __shared__ int sH[BLOCK / 32][1 << PREP_KB_MAX];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int* hist = sH[wib];
    const int NB = 1 << a.KB;
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(a.batch, 63);
        base = __shfl_sync(IM_FULL, base, 0);
        if (base >= a.n) break;
        const int end = min(base + 63, a.n);  // 63 rows: their 64 offsets fit two lane registers
        const int myoff = base + lane <= end ? a.off[base + lane] : 0;
        const int myoff2 = base + 32 + lane <= end ? a.off[base + 32 + lane] : 0;
        for (int u = base; u < end; ++u) {
            const int i = u - base;
            const int eb = i < 32 ? __shfl_sync(IM_FULL, myoff, i) : __shfl_sync(IM_FULL, myoff2, i - 32);
            const int ee = i + 1 < 32 ? __shfl_sync(IM_FULL, myoff, i + 1) : __shfl_sync(IM_FULL, myoff2, i + 1 - 32);
            const int d = ee - eb;
            if (d == 0 || d > PREP_BIG) continue;  // warp-uniform
            if (d <= 32) {
                const bool have = lane < d;
                uint2 r = make_uint2(0, 0);
                if (have) r = row_rec(a, eb + lane, (uint32_t)u, true);
                const int pos = ballot_rank(r.y >> a.B, a.KB, (d == 32 ? IM_FULL : (1u << d) - 1u), lane);
                if (have) a.out[eb + pos] = r;
                continue;
            }
            for (int q = lane; q < NB; q += 32) hist[q] = 0;
            __syncwarp();
            for (int e0 = eb; e0 < ee; e0 += 32) {  // pass 1: bucket counts
                const bool have = e0 + lane < ee;
                uint32_t b = 0xFFFFFFFFu;
                if (have) b = row_rec(a, e0 + lane, (uint32_t)u, true).y >> a.B;
                const uint32_t peers = __match_any_sync(IM_FULL, b);
                if (have && lane == __ffs(peers) - 1) hist[b] += __popc(peers);
                __syncwarp();
            }
            warp_scan_bins(hist, NB, lane);
            __syncwarp();
            write_row_table(a, (uint32_t)u, eb, ee, hist, NB, lane, 32);
            for (int e0 = eb; e0 < ee; e0 += 32) {  // pass 2: place (stable)
                const bool have = e0 + lane < ee;
                uint2 r = make_uint2(0, 0);
                uint32_t b = 0xFFFFFFFFu;
                if (have) {
                    r = row_rec(a, e0 + lane, (uint32_t)u, false);
                    b = r.y >> a.B;
                }
                const uint32_t peers = __match_any_sync(IM_FULL, b);
                if (have) a.out[eb + hist[b] + __popc(peers & ((1u << lane) - 1u))] = r;
                __syncwarp();
                if (have && lane == __ffs(peers) - 1) hist[b] += __popc(peers);
                __syncwarp();
            }
        }
    }
}

// rows longer than PREP_BIG: one block per row, shared-memory histogram, atomic placement
template <typename K>
__global__ void __launch_bounds__(BLOCK) k_rows_big(RowSortArgs<K> a) {
    __shared__ int hist[1 << PREP_KB_MAX];
    const int NB = 1 << a.KB;
    const int cnt = *a.lcount;
    for (int bi = blockIdx.x; bi < cnt; bi += gridDim.x) {
        const uint32_t u = (uint32_t)a.lst[bi];
        const int eb = a.off[u], ee = a.off[u + 1];
        __syncthreads();
        for (int i = threadIdx.x; i < NB; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int e0 = eb; e0 < ee; e0 += blockDim.x) {  // block-uniform trip count
            const bool have = e0 + (int)threadIdx.x < ee;
            uint32_t b = 0xFFFFFFFFu;
            if (have) b = row_rec(a, e0 + threadIdx.x, u, true).y >> a.B;
            const uint32_t peers = __match_any_sync(IM_FULL, b);
            if (have && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[b], __popc(peers));
        }
        __syncthreads();
        if (threadIdx.x < 32) warp_scan_bins(hist, NB, threadIdx.x);
        __syncthreads();
        write_row_table(a, u, eb, ee, hist, NB, threadIdx.x, blockDim.x);
        __syncthreads();  // the table is read from hist before the placement below advances it
        for (int e0 = eb; e0 < ee; e0 += blockDim.x) {
            const bool have = e0 + (int)threadIdx.x < ee;
            uint2 r = make_uint2(0, 0);
            uint32_t b = 0xFFFFFFFFu;
            if (have) {
                r = row_rec(a, e0 + threadIdx.x, u, false);
                b = r.y >> a.B;
            }
            const uint32_t peers = __match_any_sync(IM_FULL, b);
            const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
            int p = 0;
            if (have && lane == leader) p = atomicAdd(&hist[b], __popc(peers));
            p = __shfl_sync(IM_FULL, p, leader);
            if (have) a.out[eb + p + __popc(peers & ((1u << lane) - 1u))] = r;
        }
    }
}

// reverse offsets from the sorted keys (row = key >> KB): roff[v] = first position with row >= v
template <typename K>
__global__ void k_row_bounds(int64_t m, int32_t n, const K* __restrict__ keys, int KB, int32_t* __restrict__ roff) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= m; i += stride) {
        const int64_t r = i < m ? (int64_t)(keys[i] >> KB) : (int64_t)n;
        const int64_t p = i > 0 ? (int64_t)(keys[i - 1] >> KB) : -1;
        for (int64_t v = p + 1; v <= r; ++v) roff[v] = (int32_t)i;
    }
}

// reverse-row bucket tables from the sorted keys (row = key >> KB, bucket = low KB bits): position i
// starts buckets (previous bucket of its row, bucket(i)]; the row's last position ends the rest
template <typename K>
__global__ void k_rev_tabs(int64_t m, const K* __restrict__ keys, int KB, const int32_t* __restrict__ tidx, int nbk,
                           int32_t* __restrict__ tab) {
    const K mask = ((K)1 << KB) - 1;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
        const K k = keys[i];
        const int64_t r = (int64_t)(k >> KB);
        const int t = tidx[r];
        if (t < 0) continue;
        int32_t* tb = tab + (int64_t)t * nbk;
        const int b = (int)(k & mask);
        const int pb = (i > 0 && (int64_t)(keys[i - 1] >> KB) == r) ? (int)(keys[i - 1] & mask) : -1;
        for (int kb = pb + 1; kb <= b; ++kb) tb[kb] = (int32_t)i;
        if (i + 1 == m || (int64_t)(keys[i + 1] >> KB) != r)
            for (int kb = b + 1; kb < nbk; ++kb) tb[kb] = (int32_t)(i + 1);
    }
}

// ------------------------------------------------------------------ bucket offset tables of long rows
// For a bucket-ordered row longer than TAB_MIN, tab[kb] = first position whose bucket h >> B is
// >= kb (kb = 0 .. 2^KB; the row end if none): the hash slices of k_slices_big (im_sweep.cu) are
// then two table reads instead of two binary searches over the row.
__global__ void k_tab_index(int32_t n, const int32_t* __restrict__ offs, int32_t* __restrict__ tidx, int32_t* __restrict__ rows,
                            int* count) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
        int t = -1;
        if (offs[v + 1] - offs[v] > TAB_MIN) {
            t = atomicAdd(count, 1);
            rows[t] = (int32_t)v;
        }
        tidx[v] = t;
    }
}

// rows longer than TAB_MIN get a table: index per vertex, count read back, tables allocated
static cudaError_t setup_tables(Ctx& c, const int32_t* offs, int32_t* tidx, int32_t*& tab, int* d_count) {
    cudaError_t e;
    if ((e = cudaMemsetAsync(d_count, 0, sizeof(int), c.stream))) return e;
    k_tab_index<<<grid_for(c, c.n), BLOCK, 0, c.stream>>>(c.n, offs, tidx, c.t_tabrows, d_count);
    if ((e = LAUNCHED(c))) return e;
    int h = 0;
    if ((e = cudaMemcpyAsync(c.hpin, d_count, sizeof(int), cudaMemcpyDeviceToHost, c.stream))) return e;
    if ((e = cudaStreamSynchronize(c.stream))) return e;
    h = *(int*)c.hpin;
    return h ? c.alloc_i32(tab, (size_t)h * c.nbk) : cudaSuccess;
}

// ------------------------------------------------------------------ a2: register init
// M_v[jj] = clz(Murmur3(v, seed_V) xor Murmur3(perm[jj], seed_J)), clz(0) = 32 (Alg. 1 lines 2-5; R5, R6).
// One thread per 16 bytes (16 simulations) of a row: one Murmur3 per thread, one 16-byte store.
// hash(j) is kept in shared memory transposed by word (HJ4T[q][c] = sims 16c+4q .. 16c+4q+3) so the
// 16-byte shared loads of consecutive lanes are conflict-free.
__global__ void k_init_registers(int32_t n, int32_t J, uint32_t seedV, uint32_t seedJ, const int32_t* __restrict__ perm,
                                 uint4* __restrict__ M16) {
    __shared__ uint4 HJ4T[256];
    const int cpr = J >> 4;  // 16-byte chunks per row
    for (int c = threadIdx.x; c < cpr; c += blockDim.x)
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int j0 = 16 * c + 4 * q;
            HJ4T[q * cpr + c] = make_uint4(murmur_word((uint32_t)perm[j0], seedJ), murmur_word((uint32_t)perm[j0 + 1], seedJ),
                                           murmur_word((uint32_t)perm[j0 + 2], seedJ), murmur_word((uint32_t)perm[j0 + 3], seedJ));
        }
    __syncthreads();
    // a warp per row (no 64-bit division per chunk), lanes over the row's 16-byte chunks
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < n; row += nwarps)
      for (int c = lane; c < cpr; c += 32) {
        const uint32_t v = (uint32_t)row;
        const int64_t idx = row * cpr + c;
        const uint32_t hv = murmur_word(v, seedV);
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const uint4 h = HJ4T[q * cpr + c];
            w[q] = (uint32_t)__clz(hv ^ h.x) | ((uint32_t)__clz(hv ^ h.y) << 8) | ((uint32_t)__clz(hv ^ h.z) << 16) |
                   ((uint32_t)__clz(hv ^ h.w) << 24);
        }
        M16[idx] = make_uint4(w[0], w[1], w[2], w[3]);
      }
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_validate(Ctx& c, const int32_t* off, const int32_t* tgt, const float* prob, int* flags) {
    k_validate<<<grid_for(c, c.m > c.n ? c.m : c.n), BLOCK, 0, c.stream>>>(c.n, c.m, off, tgt, prob, flags);
    return LAUNCHED(c);
}
cudaError_t launch_const_check(Ctx& c, const float* prob, int* flag) {
    k_const_check<<<grid_for(c, c.m), BLOCK, 0, c.stream>>>(c.m, prob, flag);
    return LAUNCHED(c);
}
cudaError_t scan_exclusive(Ctx& c, const int32_t* in, int32_t* out, int n, void* tmp, size_t& tmp_bytes) {
    cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, n, c.stream);
    if (tmp) c.launches++;
    return e;
}
cudaError_t launch_build_items(Ctx& c, const int32_t* offs, int4* items, int32_t* nseg, void* tmp, size_t tmp_bytes) {
    int32_t* base = nseg + (c.n + 1);  // nseg holds 2(n+1) entries: counts, then their exclusive scan
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

// bits of the composite key (row << KB) | (h >> B): rows need bits(n-1), the bucket 31-B bits
void prep_key_bits(const Ctx& c, int& KB, int& end_bit, bool& wide) {
    KB = 31 - c.B0;
    int nb = 0;
    while (nb < 31 && ((int64_t)1 << nb) < (int64_t)c.n) nb++;
    end_bit = nb + KB;
    wide = end_bit > 32;
}

// the row-local bucket ordering applies (constant threshold, at most 2^PREP_KB_MAX buckets)
bool rows_path(const Ctx& c) { return c.sorted_h && 31 - c.B0 <= PREP_KB_MAX; }

template <typename K>
static cudaError_t prep_rows(Ctx& c, const int32_t* tgt, void** scr, size_t tb, int KB, int end_bit) {
    cudaError_t e;
    const int n = c.n;
    int32_t* lf = (int32_t*)scr[0];
    int* cnt = (int*)(lf + n);  // [0] long-row count, [1] batch cursor, [2] table count
    if ((e = cudaMemsetAsync(cnt, 0, 2 * sizeof(int), c.stream))) return e;
    k_list_long<<<grid_for(c, n), BLOCK, 0, c.stream>>>(n, c.off, lf, cnt);
    if ((e = LAUNCHED(c))) return e;
    RowSortArgs<K> a{};
    a.n = n;
    a.B = c.B0;
    a.KB = KB;
    a.off = c.off;
    a.tgt = tgt;
    a.out = c.fwd;
    a.rkey = (K*)scr[1];
    a.rval = (uint2*)scr[3];
    a.lst = lf;
    a.lcount = cnt;
    a.batch = cnt + 1;
    if (c.nbk) {  // forward bucket tables, written by the row sort itself
        if ((e = setup_tables(c, c.off, c.ftidx, c.ftab, cnt + 2))) return e;
        a.tidx = c.ftidx;
        a.tab = c.ftab;
        a.nbk = c.nbk;
    }
    k_rows<K><<<c.num_sms * 8, BLOCK, 0, c.stream>>>(a);
    if ((e = LAUNCHED(c))) return e;
    k_rows_big<K><<<c.num_sms * 4, BLOCK, 0, c.stream>>>(a);
    if ((e = LAUNCHED(c))) return e;
    e = cub::DeviceRadixSort::SortPairs(scr[4], tb, (K*)scr[1], (K*)scr[2], (uint2*)scr[3], c.rev, (int)c.m, 0, end_bit, c.stream);
    c.launches += (end_bit + 7) / 8 + 1;
    if (e) return e;
    k_row_bounds<K><<<grid_for(c, c.m + 1), BLOCK, 0, c.stream>>>(c.m, n, (const K*)scr[2], KB, c.roff);
    if ((e = LAUNCHED(c)) || !c.nbk) return e;
    if ((e = setup_tables(c, c.roff, c.rtidx, c.rtab, cnt + 2))) return e;  // reverse bucket tables
    k_rev_tabs<K><<<grid_for(c, c.m), BLOCK, 0, c.stream>>>(c.m, (const K*)scr[2], KB, c.rtidx, c.nbk, c.rtab);
    return LAUNCHED(c);
}

// scratch sizes (bytes) the edge prep needs: [0] src, [1] mark/keys0, [2] keys1, [3] vals, [4] cub temp
cudaError_t prep_scratch_sizes(Ctx& c, size_t* sz) {
    const size_t m = (size_t)(c.m ? c.m : 1);
    int KB, end_bit;
    bool wide;
    prep_key_bits(c, KB, end_bit, wide);
    const size_t ks = wide ? 8 : 4;
    sz[0] = rows_path(c) ? ((size_t)c.n + 8) * 4 : m * 4;  // long-row list + counters, or the edge sources
    sz[1] = m * (c.sorted_h ? ks : 4);
    sz[2] = c.sorted_h ? m * ks : 4;
    sz[3] = c.sorted_h ? m * 8 : 8;
    size_t t1 = 0, t2 = 0;
    cudaError_t e = cub::DeviceScan::InclusiveScan(nullptr, t1, (int32_t*)nullptr, (int32_t*)nullptr, MaxOp(), (int)m, c.stream);
    if (e) return e;
    if (c.sorted_h) {
        if (wide)
            e = cub::DeviceRadixSort::SortPairs(nullptr, t2, (ull*)nullptr, (ull*)nullptr, (uint2*)nullptr, (uint2*)nullptr,
                                                (int)m, 0, end_bit, c.stream);
        else
            e = cub::DeviceRadixSort::SortPairs(nullptr, t2, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint2*)nullptr,
                                                (uint2*)nullptr, (int)m, 0, end_bit, c.stream);
    }
    if (e) return e;
    size_t t3 = 0;
    e = cub::DeviceScan::ExclusiveSum(nullptr, t3, (int32_t*)nullptr, (int32_t*)nullptr, c.n + 1, c.stream);
    size_t t = t1 > t2 ? t1 : t2;
    sz[4] = (t > t3 ? t : t3) + 256;
    return e;
}

template <typename K>
static cudaError_t prep_sorted(Ctx& c, const int32_t* src, const int32_t* tgt, const float* prob, int32_t* indeg,
                               void** scr, size_t temp_bytes, int KB, int end_bit) {
    K* k0 = (K*)scr[1];
    K* k1 = (K*)scr[2];
    uint2* vals = (uint2*)scr[3];
    cudaError_t e;
    // forward: (u << KB | h >> B) -> rows stay in place, ordered by bucket inside
    k_edge_prep<K, true><<<grid_for(c, c.m), BLOCK, 0, c.stream>>>(c.m, src, tgt, prob, c.B0, KB, k0, vals, nullptr, indeg);
    if ((e = LAUNCHED(c))) return e;
    e = cub::DeviceRadixSort::SortPairs(scr[4], temp_bytes, k0, k1, vals, c.fwd, (int)c.m, 0, end_bit, c.stream);
    c.launches += (end_bit + 7) / 8 + 1;
    if (e) return e;
    // reverse: (v << KB | h >> B) with payload {u, h}: the sort is the transpose
    k_rev_keys<K><<<grid_for(c, c.m), BLOCK, 0, c.stream>>>(c.m, src, c.fwd, c.B0, KB, k0, vals);
    if ((e = LAUNCHED(c))) return e;
    e = cub::DeviceRadixSort::SortPairs(scr[4], temp_bytes, k0, k1, vals, c.rev, (int)c.m, 0, end_bit, c.stream);
    c.launches += (end_bit + 7) / 8 + 1;
    return e;
}

// the whole edge prep after validation: fills c.fwd (+fwdT), c.roff, c.rev (+revT)
cudaError_t prep_edges(Ctx& c, const int32_t* tgt, const float* prob, int32_t* indeg, int32_t* scan_tmp_i,
                       void** scr, const size_t* sz) {
    cudaError_t e;
    const int64_t m = c.m;
    int32_t* src = (int32_t*)scr[0];
    int32_t* mark = (int32_t*)scr[1];
    size_t tb = sz[4];
    (void)scan_tmp_i;
    if ((e = cudaMemsetAsync(indeg, 0, ((size_t)c.n + 1) * sizeof(int32_t), c.stream))) return e;
    if (rows_path(c) && c.m > 0) {
        int KB, end_bit;
        bool wide;
        prep_key_bits(c, KB, end_bit, wide);
        return wide ? prep_rows<ull>(c, tgt, scr, tb, KB, end_bit) : prep_rows<uint32_t>(c, tgt, scr, tb, KB, end_bit);
    }
    if (m > 0) {
        if ((e = cudaMemsetAsync(mark, 0, (size_t)m * sizeof(int32_t), c.stream))) return e;
        k_row_markers<<<grid_for(c, c.n), BLOCK, 0, c.stream>>>(c.n, c.off, mark);
        if ((e = LAUNCHED(c))) return e;
        if ((e = cub::DeviceScan::InclusiveScan(scr[4], tb, mark, src, MaxOp(), (int)m, c.stream))) return e;
        c.launches += 2;
    }
    if (c.sorted_h) {
        int KB, end_bit;
        bool wide;
        prep_key_bits(c, KB, end_bit, wide);
        e = wide ? prep_sorted<ull>(c, src, tgt, prob, indeg, scr, tb, KB, end_bit)
                 : prep_sorted<uint32_t>(c, src, tgt, prob, indeg, scr, tb, KB, end_bit);
        if (e) return e;
        size_t t2 = tb;
        return scan_exclusive(c, indeg, c.roff, c.n + 1, scr[4], t2);
    }
    if (m > 0) {
        k_edge_prep<uint32_t, false><<<grid_for(c, m), BLOCK, 0, c.stream>>>(m, src, tgt, prob, 0, 0, nullptr, c.fwd, c.fwdT, indeg);
        if ((e = LAUNCHED(c))) return e;
    }
    size_t t2 = tb;
    if ((e = scan_exclusive(c, indeg, c.roff, c.n + 1, scr[4], t2))) return e;
    if (m > 0) {
        if ((e = cudaMemsetAsync(indeg, 0, ((size_t)c.n + 1) * sizeof(int32_t), c.stream))) return e;
        k_transpose<<<grid_for(c, m), BLOCK, 0, c.stream>>>(m, src, c.fwd, c.fwdT, c.roff, indeg, c.rev, c.revT);
        e = LAUNCHED(c);
    }
    return e;
}

}  // namespace im
