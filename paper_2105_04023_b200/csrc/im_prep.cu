// im_prep.cu -- a0 edge preparation (Eq. 4-5, Sec. 3.3) and a2 register init (Alg. 1 lines 2-5).
//
// Edge prep, once per graph, all hand-written (no library sort or scan):
//   validate the CSR; detect a constant w; per edge h(u,v) = Murmur3(u||v) mod 2^31 and the exact
//   integer threshold T_e (im_device.cuh); build the forward rows {v, h} and the reverse rows {u, h}
//   (grouped by target) used by the sweeps.
//   Reverse offsets: in-degree histogram + exclusive scan (k_scan_*).  The transpose is an atomic-cursor
//   scatter: edge (u,v) goes to roff[v] + (a per-target cursor); the order inside a reverse row is
//   immaterial except for bucket slicing (below).
//   With a constant threshold T (2^(B-1) < T <= 2^B) every row longer than TAB_MIN is additionally
//   ordered by the bucket h >> Bs (Bs = max(B, 23): at most 2^8 buckets; a simulation j can only be
//   live on edges of bucket X_j >> Bs) and gets a bucket offset table, so the slice of a long row whose
//   candidate windows meet a set of simulations is a few table reads (k_slices_buckets, im_sweep.cu).
//   Forward rows are bucket-ordered in place by a row-local counting sort (k_rows / k_rows_big, which
//   also scatter the reverse records); long reverse rows by a block-local counting sort (k_rev_rows).
//   Per-edge thresholds (weighted cascade) keep the input row order.
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

// source vertex of every edge (per-edge-threshold path): a warp per row writes its id
__global__ void k_src(int32_t n, const int32_t* __restrict__ off, int32_t* __restrict__ src) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < n; u += nwarps)
        for (int e = off[u] + lane; e < off[u + 1]; e += 32) src[e] = (int32_t)u;
}

// in-degree histogram (reverse row lengths); equal targets of a warp are aggregated first
__global__ void k_indeg(int64_t m, const int32_t* __restrict__ tgt, int32_t* __restrict__ indeg) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < m; base += stride) {
        const int64_t e = base + threadIdx.x;
        const int v = e < m ? tgt[e] : -1;
        const uint32_t peers = __match_any_sync(IM_FULL, v);
        if (v >= 0 && lane == __ffs(peers) - 1) atomicAdd(&indeg[v], __popc(peers));
    }
}

// ---------------------------------------------------------------- exclusive scan of int32 (3 passes)
// tile = SCAN_T = BLOCK * 16 values: per-tile sums, a one-block scan of the tile sums, per-tile scan
// with the tile's offset.  Sums fit int32 (CSR offsets, segment counts <= m < 2^31).
constexpr int SCAN_PER = 16, SCAN_T = BLOCK * SCAN_PER;

__device__ __forceinline__ int block_excl_scan(int x, int* sW, int* total) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int incl = warp_incl_scan(x, lane);
    if (lane == 31) sW[wib] = incl;
    __syncthreads();
    if (wib == 0) {
        const int w = lane < BLOCK / 32 ? sW[lane] : 0;
        const int wi = warp_incl_scan(w, lane);
        if (lane < BLOCK / 32) sW[lane] = wi - w;
        if (lane == BLOCK / 32 - 1) *total = wi;
    }
    __syncthreads();
    const int r = sW[wib] + incl - x;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(BLOCK) k_scan_reduce(int n, const int32_t* __restrict__ in, int32_t* __restrict__ part) {
    __shared__ int sW[BLOCK / 32];
    __shared__ int tot;
    const int64_t b0 = (int64_t)blockIdx.x * SCAN_T;
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER; k++) {
        const int64_t i = b0 + (int64_t)k * BLOCK + threadIdx.x;
        s += i < n ? in[i] : 0;
    }
    block_excl_scan(s, sW, &tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(BLOCK) k_scan_top(int nt, int32_t* __restrict__ part) {
    __shared__ int sW[BLOCK / 32];
    __shared__ int tot;
    int carry = 0;
    for (int b = 0; b < nt; b += BLOCK) {
        const int i = b + threadIdx.x;
        const int x = i < nt ? part[i] : 0;
        const int ex = block_excl_scan(x, sW, &tot);
        if (i < nt) part[i] = carry + ex;
        carry += tot;
    }
}

__global__ void __launch_bounds__(BLOCK) k_scan_down(int n, const int32_t* __restrict__ in, const int32_t* __restrict__ part,
                                                     int32_t* __restrict__ out) {
    __shared__ int sW[BLOCK / 32];
    __shared__ int tot;
    const int64_t b0 = (int64_t)blockIdx.x * SCAN_T + (int64_t)threadIdx.x * SCAN_PER;  // thread-contiguous
    int v[SCAN_PER], s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER; k++) {
        v[k] = b0 + k < n ? in[b0 + k] : 0;
        s += v[k];
    }
    int run = part[blockIdx.x] + block_excl_scan(s, sW, &tot);
#pragma unroll
    for (int k = 0; k < SCAN_PER; k++)
        if (b0 + k < n) {
            out[b0 + k] = run;
            run += v[k];
        }
}

// forward records and per-edge thresholds (weighted cascade path); in-degree histogram
__global__ void k_edge_prep(int64_t m, const int32_t* __restrict__ src, const int32_t* __restrict__ tgt,
                            const float* __restrict__ prob, uint2* __restrict__ rec, uint32_t* __restrict__ recT,
                            int32_t* __restrict__ indeg) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += stride) {
        uint32_t u = (uint32_t)src[e], v = (uint32_t)tgt[e];
        uint32_t h = edge_hash(u, v);
        rec[e] = make_uint2(v, h);
        recT[e] = live_threshold(prob[e]);
        atomicAdd(&indeg[v], 1);
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
// With one threshold T a row only has to be grouped by bucket b = h >> Bs (KB = 31 - Bs <= 8 bits);
// the order inside a bucket is immaterial (every consumer takes the slice of a bucket range).
//   k_rows       forward row u: h = Murmur3(u||v) mod 2^31 (Eq. 4), records {v, h} written in bucket
//                order by a row-local counting sort
//   k_scatter    every edge to its reverse row (atomic cursor), straight into `rev` for a short reverse
//                row, into `rtmp` for a long one
//   k_rev_rows   long reverse rows: block-local counting sort rtmp -> rev, bucket table
// Rows of at most 32 edges are ranked inside one warp by a radix ballot; rows up to PREP_BIG by a
// warp with a shared-memory histogram; longer rows by a whole block (k_rows_big).
constexpr int PREP_BIG = 2048;
constexpr int PREP_KB_MAX = 8;

__global__ void k_list_long(int32_t n, const int32_t* __restrict__ off, int32_t* __restrict__ lf, int* count) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += stride)
        if (off[u + 1] - off[u] > PREP_BIG) lf[atomicAdd(count, 1)] = (int32_t)u;
}

struct RowSortArgs {
    int32_t n;
    int B, KB;              // bucket = h >> B (B = Bs), 2^KB buckets
    const int32_t* off;     // forward row offsets
    const int32_t* tgt;     // input targets (CSR order)
    uint2* out;             // bucket-ordered forward records {v, h}
    const int32_t* roff;    // reverse row offsets
    int32_t* cursor;        // per-target scatter cursor (zeroed)
    uint2* rev;             // reverse records {u, h}: short reverse rows final
    uint2* rtmp;            // long reverse rows (> TAB_MIN), unordered, sorted by k_rev_rows
    const int32_t* lst;     // k_rows_big: rows longer than PREP_BIG
    const int* lcount;
    int* batch;             // dynamic row-batch cursor (zeroed)
    const int32_t* tidx;    // bucket offset table of each forward row (-1: none), tables tab[rows x nbk]
    int32_t* tab;
    int nbk;
};

// the bucket offsets of a row with a table: hist holds the exclusive scan of its bucket counts
__device__ __forceinline__ void write_row_table(const int32_t* tidx, int32_t* tab, int nbk, uint32_t u, int eb, int ee,
                                                const int* hist, int NB, int tid, int nthreads) {
    const int t = tidx ? tidx[u] : -1;
    if (t < 0) return;
    int32_t* tb = tab + (int64_t)t * nbk;
    for (int kb = tid; kb <= NB; kb += nthreads) tb[kb] = kb < NB ? eb + hist[kb] : ee;
}

// record {v, h(u,v)} of input edge e of row u
__device__ __forceinline__ uint2 row_rec(const RowSortArgs& a, int64_t e, uint32_t u, bool first) {
    (void)first;
    const uint32_t v = (uint32_t)a.tgt[e];
    return make_uint2(v, edge_hash(u, v));
}

// the transpose: edge (u -> v, h) of forward position e goes to its reverse row at roff[v] + a per-target
// cursor, straight into `rev` for a short reverse row, into `rtmp` for a long one (bucket-sorted after).
// SU edges per thread: their loads, then their cursor atomics, then their stores, all in flight together.
constexpr int SU = 4;
__global__ void __launch_bounds__(BLOCK) k_scatter(int64_t m, const int32_t* __restrict__ src, const uint2* __restrict__ fwd,
                                                   const int32_t* __restrict__ roff, int32_t* __restrict__ cursor,
                                                   uint2* __restrict__ rev, uint2* __restrict__ rtmp) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * SU;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * SU + threadIdx.x; base < m; base += stride) {
        uint2 f[SU];
        int32_t u[SU], rb[SU], re[SU], p[SU];
#pragma unroll
        for (int k = 0; k < SU; k++) {
            const int64_t e = base + (int64_t)k * blockDim.x;
            f[k] = e < m ? fwd[e] : make_uint2(0, 0);
            u[k] = e < m ? src[e] : -1;
        }
#pragma unroll
        for (int k = 0; k < SU; k++) {
            rb[k] = u[k] >= 0 ? __ldg(&roff[f[k].x]) : 0;
            re[k] = u[k] >= 0 ? __ldg(&roff[f[k].x + 1]) : 0;
        }
#pragma unroll
        for (int k = 0; k < SU; k++) p[k] = u[k] >= 0 ? atomicAdd(&cursor[f[k].x], 1) : 0;
#pragma unroll
        for (int k = 0; k < SU; k++)
            if (u[k] >= 0) (re[k] - rb[k] > TAB_MIN ? rtmp : rev)[rb[k] + p[k]] = make_uint2((uint32_t)u[k], f[k].y);
    }
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

__global__ void __launch_bounds__(BLOCK) k_rows(RowSortArgs a) {
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
            for (int e0 = eb; e0 < ee; e0 += 32) {  // pass 1: bucket counts (+ the reverse scatter)
                const bool have = e0 + lane < ee;
                uint32_t b = 0xFFFFFFFFu;
                if (have) b = row_rec(a, e0 + lane, (uint32_t)u, true).y >> a.B;
                const uint32_t peers = __match_any_sync(IM_FULL, b);
                if (have && lane == __ffs(peers) - 1) hist[b] += __popc(peers);
                __syncwarp();
            }
            warp_scan_bins(hist, NB, lane);
            __syncwarp();
            write_row_table(a.tidx, a.tab, a.nbk, (uint32_t)u, eb, ee, hist, NB, lane, 32);
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

// counting sort of one row [eb, ee) by bucket (y >> B) into `out` by a whole block, with the row's bucket
// table; rec(e, first) yields the record of position e (called twice per position: first = true once);
// hist: 2^KB shared counters
template <typename Rec>
__device__ __forceinline__ void block_row_sort(Rec rec, uint2* out, int eb, int ee, int B, int NB, int* hist,
                                               const int32_t* tidx, int32_t* tab, int nbk, uint32_t row) {
    __syncthreads();
    for (int i = threadIdx.x; i < NB; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int e0 = eb; e0 < ee; e0 += blockDim.x) {  // block-uniform trip count
        const bool have = e0 + (int)threadIdx.x < ee;
        const uint32_t b = have ? rec(e0 + threadIdx.x, true).y >> B : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(IM_FULL, b);
        if (have && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[b], __popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < 32) warp_scan_bins(hist, NB, threadIdx.x);
    __syncthreads();
    write_row_table(tidx, tab, nbk, row, eb, ee, hist, NB, threadIdx.x, blockDim.x);
    __syncthreads();  // the table is read from hist before the placement below advances it
    for (int e0 = eb; e0 < ee; e0 += blockDim.x) {
        const bool have = e0 + (int)threadIdx.x < ee;
        const uint2 r = have ? rec(e0 + threadIdx.x, false) : make_uint2(0, 0);
        const uint32_t b = have ? r.y >> B : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(IM_FULL, b);
        const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
        int p = 0;
        if (have && lane == leader) p = atomicAdd(&hist[b], __popc(peers));
        p = __shfl_sync(IM_FULL, p, leader);
        if (have) out[eb + p + __popc(peers & ((1u << lane) - 1u))] = r;
    }
}

// forward rows longer than PREP_BIG: one block per row (records recomputed in the placement pass)
__global__ void __launch_bounds__(BLOCK) k_rows_big(RowSortArgs a) {
    __shared__ int hist[1 << PREP_KB_MAX];
    const int cnt = *a.lcount;
    for (int bi = blockIdx.x; bi < cnt; bi += gridDim.x) {
        const uint32_t u = (uint32_t)a.lst[bi];
        block_row_sort([&](int64_t e, bool first) { return row_rec(a, e, u, first); }, a.out, a.off[u], a.off[u + 1], a.B,
                       1 << a.KB, hist, a.tidx, a.tab, a.nbk, u);
    }
}

// long reverse rows (> TAB_MIN, listed by k_tab_index): block-local counting sort rtmp -> rev + table
__global__ void __launch_bounds__(BLOCK) k_rev_rows(int nrows, const int32_t* __restrict__ rows, const int32_t* __restrict__ roff,
                                                    const uint2* __restrict__ rtmp, uint2* __restrict__ rev, int B, int KB,
                                                    const int32_t* __restrict__ tidx, int32_t* __restrict__ tab, int nbk) {
    __shared__ int hist[1 << PREP_KB_MAX];
    for (int t = blockIdx.x; t < nrows; t += gridDim.x) {
        const uint32_t v = (uint32_t)rows[t];
        block_row_sort([&](int64_t e, bool) { return rtmp[e]; }, rev, roff[v], roff[v + 1], B, 1 << KB, hist, tidx, tab, nbk, v);
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
static cudaError_t setup_tables(Ctx& c, const int32_t* offs, int32_t* tidx, int32_t*& tab, int* d_count, int* count = nullptr) {
    cudaError_t e;
    if ((e = cudaMemsetAsync(d_count, 0, sizeof(int), c.stream))) return e;
    k_tab_index<<<grid_for(c, c.n), BLOCK, 0, c.stream>>>(c.n, offs, tidx, c.t_tabrows, d_count);
    if ((e = LAUNCHED(c))) return e;
    int h = 0;
    if ((e = cudaMemcpyAsync(c.hpin, d_count, sizeof(int), cudaMemcpyDeviceToHost, c.stream))) return e;
    if ((e = cudaStreamSynchronize(c.stream))) return e;
    h = *(int*)c.hpin;
    if (count) *count = h;
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
// exclusive sum of n int32 (tmp == nullptr: tmp_bytes <- the scratch it needs, like the call below)
cudaError_t scan_exclusive(Ctx& c, const int32_t* in, int32_t* out, int n, void* tmp, size_t& tmp_bytes) {
    const int nt = (n + SCAN_T - 1) / SCAN_T;
    if (!tmp) {
        tmp_bytes = ((size_t)nt + 1) * sizeof(int32_t);
        return cudaSuccess;
    }
    if (n <= 0) return cudaSuccess;
    int32_t* part = (int32_t*)tmp;
    k_scan_reduce<<<nt, BLOCK, 0, c.stream>>>(n, in, part);
    cudaError_t e = LAUNCHED(c);
    if (e) return e;
    k_scan_top<<<1, BLOCK, 0, c.stream>>>(nt, part);
    if ((e = LAUNCHED(c))) return e;
    k_scan_down<<<nt, BLOCK, 0, c.stream>>>(n, in, part, out);
    return LAUNCHED(c);
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

// the row-local bucket ordering applies (constant threshold): every row longer than TAB_MIN is grouped by
// bucket h >> Bs (<= 2^PREP_KB_MAX buckets) and gets a bucket table
bool rows_path(const Ctx& c) { return c.sorted_h; }
int sort_shift(int B0) { return B0 > 31 - PREP_KB_MAX ? B0 : 31 - PREP_KB_MAX; }

// constant threshold: in-degrees + scan (roff), forward row sort + reverse scatter (k_rows, k_rows_big),
// long reverse rows sorted (k_rev_rows); bucket tables of the long rows in both directions
static cudaError_t prep_rows(Ctx& c, const int32_t* tgt, int32_t* indeg, void** scr, size_t tb) {
    cudaError_t e;
    const int n = c.n;
    const int B = c.Bs, KB = 31 - c.Bs;
    int32_t* lf = (int32_t*)scr[0];
    int* cnt = (int*)(lf + n);  // [0] long-row count, [1] batch cursor, [2] table count
    int32_t* cursor = (int32_t*)scr[1];
    uint2* rtmp = (uint2*)scr[2];
    k_indeg<<<grid_for(c, c.m), BLOCK, 0, c.stream>>>(c.m, tgt, indeg);
    if ((e = LAUNCHED(c))) return e;
    size_t t2 = tb;
    if ((e = scan_exclusive(c, indeg, c.roff, n + 1, scr[4], t2))) return e;
    if ((e = cudaMemsetAsync(cursor, 0, (size_t)n * sizeof(int32_t), c.stream))) return e;
    if ((e = cudaMemsetAsync(cnt, 0, 2 * sizeof(int), c.stream))) return e;
    k_list_long<<<grid_for(c, n), BLOCK, 0, c.stream>>>(n, c.off, lf, cnt);
    if ((e = LAUNCHED(c))) return e;
    RowSortArgs a{};
    a.n = n;
    a.B = B;
    a.KB = KB;
    a.off = c.off;
    a.tgt = tgt;
    a.out = c.fwd;
    a.roff = c.roff;
    a.cursor = cursor;
    a.rev = c.rev;
    a.rtmp = rtmp;
    a.lst = lf;
    a.lcount = cnt;
    a.batch = cnt + 1;
    if ((e = setup_tables(c, c.off, c.ftidx, c.ftab, cnt + 2))) return e;  // forward tables, written by the row sort
    a.tidx = c.ftidx;
    a.tab = c.ftab;
    a.nbk = c.nbk;
    k_rows<<<c.num_sms * 8, BLOCK, 0, c.stream>>>(a);
    if ((e = LAUNCHED(c))) return e;
    k_rows_big<<<c.num_sms * 4, BLOCK, 0, c.stream>>>(a);
    if ((e = LAUNCHED(c))) return e;
    int32_t* src = (int32_t*)scr[3];
    k_src<<<grid_for(c, (int64_t)n * 32), BLOCK, 0, c.stream>>>(n, c.off, src);
    if ((e = LAUNCHED(c))) return e;
    k_scatter<<<grid_for(c, (c.m + SU - 1) / SU), BLOCK, 0, c.stream>>>(c.m, src, c.fwd, c.roff, cursor, c.rev, rtmp);
    if ((e = LAUNCHED(c))) return e;
    int h = 0;  // reverse tables: count of long reverse rows (their list in c.t_tabrows)
    if ((e = setup_tables(c, c.roff, c.rtidx, c.rtab, cnt + 2, &h))) return e;
    if (h == 0) return cudaSuccess;
    k_rev_rows<<<c.num_sms * 8, BLOCK, 0, c.stream>>>(h, c.t_tabrows, c.roff, rtmp, c.rev, B, KB, c.rtidx, c.rtab, c.nbk);
    return LAUNCHED(c);
}

// scratch sizes (bytes) the edge prep needs: [0] long-row list + counters or the edge sources, [1] scatter
// cursors, [2] long reverse rows before their sort, [3] unused, [4] scan temp
cudaError_t prep_scratch_sizes(Ctx& c, size_t* sz) {
    const size_t m = (size_t)(c.m ? c.m : 1);
    sz[0] = rows_path(c) ? ((size_t)c.n + 8) * 4 : m * 4;
    sz[1] = ((size_t)c.n + 1) * 4;
    sz[2] = rows_path(c) ? m * 8 : 8;
    sz[3] = rows_path(c) ? m * 4 : 8;  // edge sources of the scatter
    size_t t = 0;
    cudaError_t e = scan_exclusive(c, nullptr, nullptr, c.n + 1, nullptr, t);
    sz[4] = t + 256;
    return e;
}

// the whole edge prep after validation: fills c.fwd (+fwdT), c.roff, c.rev (+revT), bucket tables
cudaError_t prep_edges(Ctx& c, const int32_t* tgt, const float* prob, int32_t* indeg, int32_t* scan_tmp_i,
                       void** scr, const size_t* sz) {
    cudaError_t e;
    const int64_t m = c.m;
    size_t tb = sz[4];
    (void)scan_tmp_i;
    if ((e = cudaMemsetAsync(indeg, 0, ((size_t)c.n + 1) * sizeof(int32_t), c.stream))) return e;
    if (rows_path(c) && c.m > 0) return prep_rows(c, tgt, indeg, scr, tb);
    // per-edge thresholds (weighted cascade): input row order, atomic-cursor transpose
    int32_t* src = (int32_t*)scr[0];
    if (m > 0) {
        k_src<<<grid_for(c, (int64_t)c.n * 32), BLOCK, 0, c.stream>>>(c.n, c.off, src);
        if ((e = LAUNCHED(c))) return e;
        k_edge_prep<<<grid_for(c, m), BLOCK, 0, c.stream>>>(m, src, tgt, prob, c.fwd, c.fwdT, indeg);
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
