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
#include <algorithm>

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
        if (prob) {  // null: one scalar probability, checked on the host (im_load_csr_const)
            float w = prob[e];
            if (!(w >= 0.0f && w <= 1.0f)) f |= 4;  // also rejects NaN
        }
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

constexpr int HCH = 16384;  // rows longer than this ("huge": RMAT hubs reach ~700k) are bucket-sorted by several blocks

// rows with PREP_BIG < length <= HCH into lf (count[0]); longer ones into huge (hcount[0])
__global__ void k_list_long(int32_t n, const int32_t* __restrict__ off, int32_t* __restrict__ lf, int* count,
                            int32_t* __restrict__ huge, int* hcount) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += stride) {
        const int d = off[u + 1] - off[u];
        if (d > HCH) huge[atomicAdd(hcount, 1)] = (int32_t)u;
        else if (d > PREP_BIG) lf[atomicAdd(count, 1)] = (int32_t)u;
    }
}

// the huge rows of a list of rows (rows[0..*nrows))
__global__ void k_list_huge(const int32_t* __restrict__ rows, const int* nrows, const int32_t* __restrict__ off,
                            int32_t* __restrict__ huge, int* hcount) {
    const int nr = *nrows;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += gridDim.x * blockDim.x) {
        const int v = rows[i];
        if (off[v + 1] - off[v] > HCH) huge[atomicAdd(hcount, 1)] = v;
    }
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

// ---------------------------------------------------------------- the transpose
// Reverse row v occupies [roff[v], roff[v+1]).  The forward edges are first grouped by v's high bits in
// L <= 2 radix partition passes of 256 digits each (MSD: digit = (v >> shift) & 255, pass k refines the
// 256^k segments of pass k-1), which leaves every block of 2^LB consecutive vertices (LB <= 12) in one
// contiguous segment; k_place then places each such partition's records into their reverse rows with
// per-vertex counters in shared memory.  A partition pass works on units of <= PT records of one
// segment: k_pcount counts digits per segment (shared histogram, one global add per digit and unit),
// k_pscan turns the counts into the sub-segment offsets, k_pscatter ranks a unit's records by digit in
// shared memory, reserves each digit's run with one global atomic, stages the unit sorted by digit in
// shared memory and writes every run contiguously (coalesced).  The order inside a reverse row is
// immaterial except for the bucket order of long rows (k_rev_rows).
#ifndef PREP_PT
#define PREP_PT 3072
#endif
#ifndef PSCAT_BPS
#define PSCAT_BPS 8
#endif
constexpr int PT = PREP_PT;    // records per partition-pass unit (staged in dynamic shared memory: 3072 x 9 B)
constexpr size_t PSCAT_SMEM = (size_t)PT * (sizeof(uint2) + 1);
constexpr size_t BSCAT_SMEM = (size_t)PT * (sizeof(uint2) + sizeof(int) + 1);  // k_bscatter stages {u, h}, v and the digit
constexpr int PCH = 16384;  // staged records per k_place work unit
constexpr int NPMAX = 4096; // vertices per k_place partition (shared counters)
constexpr int PSEG_MAX = 65536;  // segments after two passes (256^2)

// segment of unit un: last s with ustart[s] <= un (binary search over nseg + 1 unit starts)
__device__ __forceinline__ int unit_segment(const int32_t* __restrict__ ustart, int nseg, int un) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ustart[mid] <= un) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// unit starts of a pass over nseg segments [soff[s], soff[s+1]) in units of <= chunk records (one block)
__global__ void __launch_bounds__(BLOCK) k_seg_units(int nseg, const int32_t* __restrict__ soff, int chunk,
                                                     int32_t* __restrict__ ustart) {
    __shared__ int sW[BLOCK / 32];
    __shared__ int tot;
    int carry = 0;
    for (int b = 0; b < nseg; b += BLOCK) {
        const int sg = b + threadIdx.x;
        const int x = sg < nseg ? (soff[sg + 1] - soff[sg] + chunk - 1) / chunk : 0;
        const int ex = block_excl_scan(x, sW, &tot);
        if (sg < nseg) ustart[sg] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) ustart[nseg] = carry;
}

// the record {u, v} of position e of a pass: pass 0 reads the input edges (src, tgt), later passes the
// previous pass's output.  The passes carry 8 bytes per edge; the edge hash is recomputed once, by k_place
// (carrying {u, h} + v moved 12 bytes per edge and pass).
struct PartIn {
    const int32_t* src;  // pass 0: source vertex per input position, else null
    const int32_t* tgt;  // pass 0: targets
    const uint2* rec;    // later passes: {u, v}
    __device__ __forceinline__ int32_t tv(int e) const { return src ? tgt[e] : (int32_t)rec[e].y; }
    __device__ __forceinline__ uint2 uv(int e) const { return src ? make_uint2((uint32_t)src[e], (uint32_t)tgt[e]) : rec[e]; }
};

__global__ void __launch_bounds__(BLOCK) k_pcount(PartIn in, int nseg, const int32_t* __restrict__ soff,
                                                  const int32_t* __restrict__ ustart, int shift, int32_t* __restrict__ counts) {
    __shared__ int hist[256];
    __shared__ int sseg;
    const int nunits = ustart[nseg];
    for (int un = blockIdx.x; un < nunits; un += gridDim.x) {
        __syncthreads();
        if (threadIdx.x == 0) sseg = unit_segment(ustart, nseg, un);
        hist[threadIdx.x] = 0;  // BLOCK == 256
        __syncthreads();
        const int sg = sseg, e0 = soff[sg] + (un - ustart[sg]) * PT, e1 = min(soff[sg + 1], e0 + PT);
#pragma unroll 4
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&hist[(in.tv(e) >> shift) & 255], 1);
        __syncthreads();
        if (hist[threadIdx.x]) atomicAdd(&counts[(size_t)sg * 256 + threadIdx.x], hist[threadIdx.x]);
    }
}

// per segment: sub-segment offsets (next pass's segment table, nseg * 256 + 1 entries) and cursors
__global__ void __launch_bounds__(BLOCK) k_pscan(int nseg, const int32_t* __restrict__ soff, const int32_t* __restrict__ counts,
                                                 int32_t* __restrict__ nsoff, int32_t* __restrict__ cursor) {
    __shared__ int sW[BLOCK / 32];
    __shared__ int tot;
    for (int sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
        const int c = counts[(size_t)sg * 256 + threadIdx.x];
        const int o = soff[sg] + block_excl_scan(c, sW, &tot);
        nsoff[(size_t)sg * 256 + threadIdx.x] = o;
        cursor[(size_t)sg * 256 + threadIdx.x] = o;
        if (sg == nseg - 1 && threadIdx.x == 0) nsoff[(size_t)nseg * 256] = soff[nseg];
    }
}

__global__ void __launch_bounds__(BLOCK) k_pscatter(PartIn in, int nseg, const int32_t* __restrict__ soff,
                                                    const int32_t* __restrict__ ustart, int shift, int32_t* __restrict__ cursor,
                                                    uint2* __restrict__ orec) {
    __shared__ int hist[256], loff[256], gbase[256];
    extern __shared__ __align__(16) unsigned char dyn[];
    uint2* srec = reinterpret_cast<uint2*>(dyn);
    unsigned char* sdig = dyn + PT * sizeof(uint2);
    __shared__ int sW[BLOCK / 32];
    __shared__ int tot, sseg;
    const int nunits = ustart[nseg];
    for (int un = blockIdx.x; un < nunits; un += gridDim.x) {
        __syncthreads();
        if (threadIdx.x == 0) sseg = unit_segment(ustart, nseg, un);
        hist[threadIdx.x] = 0;
        __syncthreads();
        const int sg = sseg, e0 = soff[sg] + (un - ustart[sg]) * PT, e1 = min(soff[sg + 1], e0 + PT);
        constexpr int PU = PT / BLOCK;  // records per thread, all loads in flight together
        uint2 rr[PU];
        bool hv[PU];
#pragma unroll
        for (int k = 0; k < PU; k++) {
            const int e = e0 + k * BLOCK + threadIdx.x;
            hv[k] = e < e1;
            rr[k] = hv[k] ? in.uv(e) : make_uint2(0, 0);
        }
#pragma unroll
        for (int k = 0; k < PU; k++)
            if (hv[k]) atomicAdd(&hist[(rr[k].y >> shift) & 255], 1);
        __syncthreads();
        const int c = hist[threadIdx.x];
        loff[threadIdx.x] = block_excl_scan(c, sW, &tot);  // contains the barriers
        gbase[threadIdx.x] = c ? atomicAdd(&cursor[(size_t)sg * 256 + threadIdx.x], c) : 0;
        hist[threadIdx.x] = loff[threadIdx.x];  // now the local placement cursor
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PU; k++) {  // stage the unit sorted by digit
            if (!hv[k]) continue;
            const int d = (rr[k].y >> shift) & 255;
            const int q = atomicAdd(&hist[d], 1);
            srec[q] = rr[k];
            sdig[q] = (unsigned char)d;
        }
        __syncthreads();
        for (int q = threadIdx.x; q < e1 - e0; q += blockDim.x) {  // each digit's run is contiguous here and there
            const int d = sdig[q];
            orec[gbase[d] + (q - loff[d])] = srec[q];
        }
    }
}

// in-degrees from the partitioned records: a unit of <= PCH records of one 2^LB-vertex partition is counted per
// target in shared memory and added with one global atomic per distinct target (a histogram of the unpartitioned
// targets costs one returning atomic per warp-distinct target, 4.3 ms on the 520M-edge RMAT)
__global__ void __launch_bounds__(BLOCK) k_part_indeg(int LB, int NP, const int32_t* __restrict__ soff,
                                                      const int32_t* __restrict__ ustart, PartIn in, int32_t* __restrict__ indeg);

// ---------------------------------------------------------------- bucket-major edge list (im_slab.cu)
// All edges grouped by the salt bucket h >> Bs of their hash (<= 256 buckets): an edge can only be live in the
// simulations whose salt lies in its bucket, so the full sweeps of a build decompose into one independent
// subproblem per bucket (im_slab.cu).  One counting pass and one shared-memory-staged partition pass
// (k_pscatter's scheme with the bucket as the digit): brec[pos] = {u, h}, bv[pos] = v.
__global__ void __launch_bounds__(BLOCK) k_bcount(int64_t m, const uint2* __restrict__ fwd, int Bs, int32_t* __restrict__ counts) {
    __shared__ int hist[256];
    hist[threadIdx.x] = 0;  // BLOCK == 256
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) atomicAdd(&hist[fwd[e].y >> Bs], 1);
    __syncthreads();
    if (hist[threadIdx.x]) atomicAdd(&counts[threadIdx.x], hist[threadIdx.x]);
}

__global__ void __launch_bounds__(BLOCK) k_bscatter(int64_t m, const int32_t* __restrict__ src, const uint2* __restrict__ fwd, int Bs,
                                                    int32_t* __restrict__ cursor, uint2* __restrict__ orec, int32_t* __restrict__ ov) {
    __shared__ int hist[256], loff[256], gbase[256];
    extern __shared__ __align__(16) unsigned char dyn[];
    uint2* srec = reinterpret_cast<uint2*>(dyn);
    int* sv = reinterpret_cast<int*>(dyn + PT * sizeof(uint2));
    unsigned char* sdig = dyn + PT * (sizeof(uint2) + sizeof(int));
    __shared__ int sW[BLOCK / 32];
    __shared__ int tot;
    const int64_t nunits = (m + PT - 1) / PT;
    for (int64_t un = blockIdx.x; un < nunits; un += gridDim.x) {
        __syncthreads();
        hist[threadIdx.x] = 0;
        __syncthreads();
        const int64_t e0 = un * PT, e1 = min(m, e0 + (int64_t)PT);
        constexpr int PU = PT / BLOCK;
        uint2 ff[PU];
        int uu[PU];
#pragma unroll
        for (int k = 0; k < PU; k++) {
            const int64_t e = e0 + k * BLOCK + threadIdx.x;
            ff[k] = e < e1 ? fwd[e] : make_uint2(0u, 0u);
            uu[k] = e < e1 ? src[e] : -1;
        }
#pragma unroll
        for (int k = 0; k < PU; k++)
            if (uu[k] >= 0) atomicAdd(&hist[ff[k].y >> Bs], 1);
        __syncthreads();
        const int c = hist[threadIdx.x];
        loff[threadIdx.x] = block_excl_scan(c, sW, &tot);
        gbase[threadIdx.x] = c ? atomicAdd(&cursor[threadIdx.x], c) : 0;
        hist[threadIdx.x] = loff[threadIdx.x];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PU; k++) {
            if (uu[k] < 0) continue;
            const int d = ff[k].y >> Bs;
            const int q = atomicAdd(&hist[d], 1);
            srec[q] = make_uint2((uint32_t)uu[k], ff[k].y);
            sv[q] = (int)ff[k].x;
            sdig[q] = (unsigned char)d;
        }
        __syncthreads();
        for (int q = threadIdx.x; q < (int)(e1 - e0); q += blockDim.x) {
            const int d = sdig[q];
            const int pos = gbase[d] + (q - loff[d]);
            orec[pos] = srec[q];
            ov[pos] = sv[q];
        }
    }
}

// boff_h[0 .. nb] (host) and c.brec / c.bv (device) from the finished forward records and their sources
static cudaError_t bucket_partition(Ctx& c, const int32_t* src, int32_t* cnt256) {
    cudaError_t e;
    const int nb = 1 << (31 - c.Bs);
    if ((e = cudaMemsetAsync(cnt256, 0, 256 * sizeof(int32_t), c.stream))) return e;
    k_bcount<<<c.num_sms * 8, BLOCK, 0, c.stream>>>(c.m, c.fwd, c.Bs, cnt256);
    if ((e = LAUNCHED(c))) return e;
    int32_t hc[256];
    if ((e = cudaMemcpyAsync(hc, cnt256, sizeof hc, cudaMemcpyDeviceToHost, c.stream))) return e;
    if ((e = cudaStreamSynchronize(c.stream))) return e;
    c.boff_h.assign(nb + 1, 0);
    int32_t cur[256] = {};
    for (int b = 0; b < nb; b++) {
        cur[b] = c.boff_h[b];
        c.boff_h[b + 1] = c.boff_h[b] + hc[b];
    }
    if ((e = cudaMemcpyAsync(cnt256, cur, sizeof cur, cudaMemcpyHostToDevice, c.stream))) return e;
    static bool attr = false;
    if (!attr) {
        if ((e = cudaFuncSetAttribute(k_bscatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BSCAT_SMEM))) return e;
        attr = true;
    }
    k_bscatter<<<c.num_sms * 5, BLOCK, BSCAT_SMEM, c.stream>>>(c.m, src, c.fwd, c.Bs, cnt256, c.brec, c.bv);
    if ((e = LAUNCHED(c))) return e;
    return cudaStreamSynchronize(c.stream);  // cur is read by the copy above
}

// unit starts of k_place: partition p = vertices [p << LB, (p+1) << LB) covers [roff[p << LB], roff[...])
__global__ void __launch_bounds__(BLOCK) k_seg_units_roff(int n, int LB, int NP, const int32_t* __restrict__ roff, int chunk,
                                                          int32_t* __restrict__ ustart) {
    __shared__ int sW[BLOCK / 32];
    __shared__ int tot;
    int carry = 0;
    for (int b = 0; b < NP; b += BLOCK) {
        const int p = b + threadIdx.x;
        int x = 0;
        if (p < NP) {
            const int64_t v0 = (int64_t)p << LB, v1 = min((int64_t)n, (int64_t)(p + 1) << LB);
            x = (roff[v1] - roff[v0] + chunk - 1) / chunk;
        }
        const int ex = block_excl_scan(x, sW, &tot);
        if (p < NP) ustart[p] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) ustart[NP] = carry;
}

// a work unit = <= PCH staged records of one partition (their positions are the partition's range of the
// reverse order): count them per target in shared memory, reserve each target's run with one global atomic
// per distinct target, write each record to its reverse row (short rows straight into rev, long rows into
// ltmp for k_rev_rows)
__global__ void __launch_bounds__(BLOCK) k_place(int n, int LB, int NP, const int32_t* __restrict__ ustart,
                                                 const int32_t* __restrict__ roff, int32_t* __restrict__ cursor, PartIn in,
                                                 uint2* __restrict__ rev, uint2* __restrict__ ltmp) {
    __shared__ int cnt[NPMAX];
    __shared__ unsigned char lng[NPMAX];  // the target's reverse row is long (sorted later from ltmp)
    __shared__ int sp;
    const int nunits = ustart[NP];
    const int V = 1 << LB;
    for (int un = blockIdx.x; un < nunits; un += gridDim.x) {
        __syncthreads();
        if (threadIdx.x == 0) sp = unit_segment(ustart, NP, un);  // the partition owning unit un
        for (int i = threadIdx.x; i < V; i += blockDim.x) cnt[i] = 0;
        __syncthreads();
        const int p = sp;
        const int64_t vb = (int64_t)p << LB;
        const int rb = roff[vb], re = roff[min((int64_t)n, vb + V)];
        const int e0 = rb + (un - ustart[p]) * PCH, e1 = min(re, e0 + PCH);
#pragma unroll 4
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&cnt[in.tv(e) - vb], 1);
        __syncthreads();
        for (int i = threadIdx.x; i < V; i += blockDim.x) {  // this unit's run of target vb + i
            const int c = cnt[i];
            if (c) {
                const int r0 = roff[vb + i];
                lng[i] = roff[vb + i + 1] - r0 > TAB_MIN;
                cnt[i] = r0 + atomicAdd(&cursor[vb + i], c);
            }
        }
        __syncthreads();
#pragma unroll 4
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
            const uint2 r = in.uv(e);
            const int i = (int)r.y - (int)vb;
            const int pos = atomicAdd(&cnt[i], 1);
            (lng[i] ? ltmp : rev)[pos] = make_uint2(r.x, edge_hash(r.x, r.y));
        }
    }
}

__global__ void __launch_bounds__(BLOCK) k_part_indeg(int LB, int NP, const int32_t* __restrict__ soff,
                                                      const int32_t* __restrict__ ustart, PartIn in, int32_t* __restrict__ indeg) {
    __shared__ int cnt[NPMAX];
    __shared__ int sp;
    const int nunits = ustart[NP];
    const int V = 1 << LB;
    for (int un = blockIdx.x; un < nunits; un += gridDim.x) {
        __syncthreads();
        if (threadIdx.x == 0) sp = unit_segment(ustart, NP, un);
        for (int i = threadIdx.x; i < V; i += blockDim.x) cnt[i] = 0;
        __syncthreads();
        const int p = sp;
        const int64_t vb = (int64_t)p << LB;
        const int e0 = soff[p] + (un - ustart[p]) * PCH, e1 = min(soff[p + 1], e0 + PCH);
#pragma unroll 4
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&cnt[in.tv(e) - vb], 1);
        __syncthreads();
        for (int i = threadIdx.x; i < V; i += blockDim.x)
            if (cnt[i]) atomicAdd(&indeg[vb + i], cnt[i]);
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
            // pass 1: bucket counts.  Plain shared-memory atomics: ranking equal buckets with match.any cost more
            // than the few-way conflicts it avoided (3.6 -> 2.4 ms on the 520M-edge RMAT)
            for (int e = eb + lane; e < ee; e += 32) atomicAdd(&hist[row_rec(a, e, (uint32_t)u, true).y >> a.B], 1);
            __syncwarp();
            warp_scan_bins(hist, NB, lane);
            __syncwarp();
            write_row_table(a.tidx, a.tab, a.nbk, (uint32_t)u, eb, ee, hist, NB, lane, 32);
            __syncwarp();  // the table is read from hist before the placement advances it
            for (int e = eb + lane; e < ee; e += 32) {  // pass 2: place (the order inside a bucket is immaterial)
                const uint2 r = row_rec(a, e, (uint32_t)u, false);
                a.out[eb + atomicAdd(&hist[r.y >> a.B], 1)] = r;
            }
            __syncwarp();  // before the next row zeroes hist
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
#pragma unroll 4
    for (int e = eb + threadIdx.x; e < ee; e += blockDim.x) atomicAdd(&hist[rec(e, true).y >> B], 1);
    __syncthreads();
    if (threadIdx.x < 32) warp_scan_bins(hist, NB, threadIdx.x);
    __syncthreads();
    write_row_table(tidx, tab, nbk, row, eb, ee, hist, NB, threadIdx.x, blockDim.x);
    __syncthreads();  // the table is read from hist before the placement below advances it
#pragma unroll 4
    for (int e = eb + threadIdx.x; e < ee; e += blockDim.x) {  // the order inside a bucket is immaterial
        const uint2 r = rec(e, false);
        out[eb + atomicAdd(&hist[r.y >> B], 1)] = r;
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
        if (roff[v + 1] - roff[v] > HCH) continue;  // huge: k_huge_*
        block_row_sort([&](int64_t e, bool) { return rtmp[e]; }, rev, roff[v], roff[v + 1], B, 1 << KB, hist, tidx, tab, nbk, v);
    }
}

// Huge rows (> HCH entries), bucket-sorted by units of <= HCH entries on several blocks: k_huge_count adds
// each unit's bucket counts to the row's 256 counters, k_huge_scan turns them into the row's bucket
// table and placement cursors, k_huge_place reserves each unit's run per bucket with one global atomic
// and writes its records there (inside the row's region of the output: L2-resident writes).
struct HugeSort {
    const int32_t* huge;   // huge rows
    const int* nhuge;      // their count (device)
    const int32_t* offs;   // row offsets
    const int32_t* ustart; // unit starts per huge row (k_huge_units)
    const int32_t* tgt;    // forward rows: records {tgt[e], h(u, tgt[e])} (Eq. 4); null: in[e]
    const uint2* in;
    uint2* out;
    int B, KB;
    int32_t* cnt;          // 256 counters per huge row (zeroed), then cursors
    const int32_t* tidx;
    int32_t* tab;
    int nbk;
};

__device__ __forceinline__ uint2 huge_rec(const HugeSort& a, int e, uint32_t u) {
    if (!a.tgt) return a.in[e];
    const uint32_t v = (uint32_t)a.tgt[e];
    return make_uint2(v, edge_hash(u, v));
}

__global__ void __launch_bounds__(BLOCK) k_huge_units(HugeSort a) {
    __shared__ int sW[BLOCK / 32];
    __shared__ int tot;
    const int nh = *a.nhuge;
    int carry = 0;
    for (int b = 0; b < nh; b += BLOCK) {
        const int r = b + threadIdx.x;
        int x = 0;
        if (r < nh) {
            const int u = a.huge[r];
            x = (a.offs[u + 1] - a.offs[u] + HCH - 1) / HCH;
        }
        const int ex = block_excl_scan(x, sW, &tot);
        if (r < nh) const_cast<int32_t*>(a.ustart)[r] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) const_cast<int32_t*>(a.ustart)[nh] = carry;
}

template <bool PLACE>
__global__ void __launch_bounds__(BLOCK) k_huge_pass(HugeSort a) {
    __shared__ int hist[256];
    __shared__ int sr;
    const int nh = *a.nhuge;
    if (nh == 0) return;
    const int nunits = a.ustart[nh];
    for (int un = blockIdx.x; un < nunits; un += gridDim.x) {
        __syncthreads();
        if (threadIdx.x == 0) sr = unit_segment(a.ustart, nh, un);
        hist[threadIdx.x] = 0;
        __syncthreads();
        const int r = sr;
        const uint32_t u = (uint32_t)a.huge[r];
        const int e0 = a.offs[u] + (un - a.ustart[r]) * HCH, e1 = min(a.offs[u + 1], e0 + HCH);
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&hist[huge_rec(a, e, u).y >> a.B], 1);
        __syncthreads();
        const int c = hist[threadIdx.x];
        if (!PLACE) {
            if (c) atomicAdd(&a.cnt[(size_t)r * 256 + threadIdx.x], c);
            continue;
        }
        hist[threadIdx.x] = c ? atomicAdd(&a.cnt[(size_t)r * 256 + threadIdx.x], c) : 0;  // this unit's run per bucket
        __syncthreads();
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
            const uint2 rec = huge_rec(a, e, u);
            a.out[atomicAdd(&hist[rec.y >> a.B], 1)] = rec;
        }
    }
}

// per huge row: bucket table and placement cursors from the counts
__global__ void __launch_bounds__(BLOCK) k_huge_scan(HugeSort a) {
    __shared__ int sW[BLOCK / 32];
    __shared__ int tot;
    const int nh = *a.nhuge, NB = 1 << a.KB;
    for (int r = blockIdx.x; r < nh; r += gridDim.x) {
        const int u = a.huge[r];
        const int c = threadIdx.x < NB ? a.cnt[(size_t)r * 256 + threadIdx.x] : 0;
        const int o = a.offs[u] + block_excl_scan(c, sW, &tot);
        a.cnt[(size_t)r * 256 + threadIdx.x] = o;
        const int t = a.tidx[u];
        if (t >= 0) {
            int32_t* tb = a.tab + (int64_t)t * a.nbk;
            if (threadIdx.x < NB) tb[threadIdx.x] = o;
            if (threadIdx.x == 0) tb[NB] = a.offs[u + 1];
        }
    }
}

static cudaError_t huge_sort(Ctx& c, HugeSort& a, int32_t* ustart, int max_huge) {
    cudaError_t e;
    a.ustart = ustart;
    if ((e = cudaMemsetAsync(a.cnt, 0, (size_t)max_huge * 256 * sizeof(int32_t), c.stream))) return e;
    k_huge_units<<<1, BLOCK, 0, c.stream>>>(a);
    if ((e = LAUNCHED(c))) return e;
    k_huge_pass<false><<<c.num_sms * 4, BLOCK, 0, c.stream>>>(a);
    if ((e = LAUNCHED(c))) return e;
    k_huge_scan<<<c.num_sms * 4, BLOCK, 0, c.stream>>>(a);
    if ((e = LAUNCHED(c))) return e;
    k_huge_pass<true><<<c.num_sms * 4, BLOCK, 0, c.stream>>>(a);
    return LAUNCHED(c);
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
    if ((e = cudaMemsetAsync(cursor, 0, (size_t)n * sizeof(int32_t), c.stream))) return e;
    // huge rows: lists (forward, reverse), their counters and unit starts
    const int max_huge = (int)(c.m / HCH + 2);
    int32_t* hz = (int32_t*)scr[8];
    int* hcnt = hz;                               // [0] forward huge count, [1] reverse huge count
    int32_t* fhuge = hz + 8;
    int32_t* rhuge = fhuge + max_huge;
    int32_t* hustart = rhuge + max_huge;          // max_huge + 1
    int32_t* hcounters = hustart + max_huge + 8;  // max_huge x 256
    if ((e = cudaMemsetAsync(hcnt, 0, 8 * sizeof(int), c.stream))) return e;
    if ((e = cudaMemsetAsync(cnt, 0, 2 * sizeof(int), c.stream))) return e;
    k_list_long<<<grid_for(c, n), BLOCK, 0, c.stream>>>(n, c.off, lf, cnt, fhuge, hcnt);
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
    {
        HugeSort hs{fhuge, hcnt, c.off, nullptr, tgt, nullptr, c.fwd, B, KB, hcounters, c.ftidx, c.ftab, c.nbk};
        if ((e = huge_sort(c, hs, hustart, max_huge))) return e;
    }
    // the transpose: L radix partition passes over 8-bit digits of v, then k_place per 2^LB-vertex partition
    int NB = 1;
    while (NB < 31 && ((int64_t)1 << NB) < (int64_t)n) NB++;
    const int L = NB <= 12 ? 0 : (NB - 12 + 7) / 8, LB = NB - 8 * L;
    const int NP = (int)(((int64_t)n + (1 << LB) - 1) >> LB);
    int32_t* src = (int32_t*)scr[3];
    uint2* recA = (uint2*)scr[5];
    uint2* recB = rtmp;
    int32_t* seg = (int32_t*)scr[7];                 // segment offsets of the current pass (<= 65536 + 1)
    int32_t* nseg_off = seg + (PSEG_MAX + 1);        // of the next pass
    int32_t* cnt2 = nseg_off + (PSEG_MAX + 1);       // digit counts / cursors per (segment, digit)
    int32_t* ustart = cnt2 + PSEG_MAX;               // unit starts (<= PSEG_MAX + 1, or NP + 1 for k_place)
    k_src<<<grid_for(c, (int64_t)n * 32), BLOCK, 0, c.stream>>>(n, c.off, src);
    if ((e = LAUNCHED(c))) return e;
    if (c.brec && (e = bucket_partition(c, src, cnt2))) return e;  // before the passes below reuse src
    {
        const int32_t zm[2] = {0, (int32_t)c.m};
        if ((e = cudaMemcpyAsync(seg, zm, sizeof zm, cudaMemcpyHostToDevice, c.stream))) return e;
        if ((e = cudaStreamSynchronize(c.stream))) return e;  // zm goes out of scope
    }
    PartIn in{src, tgt, nullptr};
    const uint2* rec_final = nullptr;
    int nseg = 1;
    for (int k = 0; k < L; k++) {
        const int shift = NB - 8 * (k + 1);
        uint2* orec = (k & 1) ? recB : recA;
        k_seg_units<<<1, BLOCK, 0, c.stream>>>(nseg, seg, PT, ustart);
        if ((e = LAUNCHED(c))) return e;
        if ((e = cudaMemsetAsync(cnt2, 0, (size_t)nseg * 256 * sizeof(int32_t), c.stream))) return e;
        const int grid = c.num_sms * 8;
        k_pcount<<<grid, BLOCK, 0, c.stream>>>(in, nseg, seg, ustart, shift, cnt2);
        if ((e = LAUNCHED(c))) return e;
        k_pscan<<<std::min(nseg, c.num_sms * 8), BLOCK, 0, c.stream>>>(nseg, seg, cnt2, nseg_off, cnt2);
        if ((e = LAUNCHED(c))) return e;
        static bool attr = false;
        if (!attr) {
            if ((e = cudaFuncSetAttribute(k_pscatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PSCAT_SMEM))) return e;
            attr = true;
        }
        k_pscatter<<<c.num_sms * PSCAT_BPS, BLOCK, PSCAT_SMEM, c.stream>>>(in, nseg, seg, ustart, shift, cnt2, orec);
        if ((e = LAUNCHED(c))) return e;
        std::swap(seg, nseg_off);
        nseg *= 256;
        in = PartIn{nullptr, nullptr, orec};
        rec_final = orec;
    }
    // long reverse rows land in a buffer the passes no longer need (not the one k_place reads)
    if (L >= 1 && rec_final == recB) rtmp = recA;
    // in-degrees and reverse offsets from the partitioned records (segment p of the last pass = partition p)
    k_seg_units<<<1, BLOCK, 0, c.stream>>>(NP, seg, PCH, ustart);
    if ((e = LAUNCHED(c))) return e;
    k_part_indeg<<<c.num_sms * 8, BLOCK, 0, c.stream>>>(LB, NP, seg, ustart, in, indeg);
    if ((e = LAUNCHED(c))) return e;
    size_t t2 = tb;
    if ((e = scan_exclusive(c, indeg, c.roff, n + 1, scr[4], t2))) return e;
    k_seg_units_roff<<<1, BLOCK, 0, c.stream>>>(n, LB, NP, c.roff, PCH, ustart);
    if ((e = LAUNCHED(c))) return e;
    k_place<<<c.num_sms * 8, BLOCK, 0, c.stream>>>(n, LB, NP, ustart, c.roff, cursor, in, c.rev, rtmp);
    if ((e = LAUNCHED(c))) return e;
    int h = 0;  // reverse tables: count of long reverse rows (their list in c.t_tabrows)
    if ((e = setup_tables(c, c.roff, c.rtidx, c.rtab, cnt + 2, &h))) return e;
    if (h == 0) return cudaSuccess;
    k_rev_rows<<<c.num_sms * 8, BLOCK, 0, c.stream>>>(h, c.t_tabrows, c.roff, rtmp, c.rev, B, KB, c.rtidx, c.rtab, c.nbk);
    if ((e = LAUNCHED(c))) return e;
    if ((e = cudaMemcpyAsync(cnt + 2, &h, sizeof(int), cudaMemcpyHostToDevice, c.stream))) return e;
    k_list_huge<<<grid_for(c, h), BLOCK, 0, c.stream>>>(c.t_tabrows, cnt + 2, c.roff, rhuge, hcnt + 1);
    if ((e = LAUNCHED(c))) return e;
    HugeSort hs{rhuge, hcnt + 1, c.roff, nullptr, nullptr, rtmp, c.rev, B, KB, hcounters, c.rtidx, c.rtab, c.nbk};
    if ((e = huge_sort(c, hs, hustart, max_huge))) return e;
    return cudaStreamSynchronize(c.stream);  // &h is read by the copy above
}

// scratch sizes (bytes) the edge prep needs: [0] long-row list + counters or the edge sources, [1] scatter
// cursors, [2] long reverse rows before their sort, [3] unused, [4] scan temp
cudaError_t prep_scratch_sizes(Ctx& c, size_t* sz) {
    const size_t m = (size_t)(c.m ? c.m : 1);
    sz[0] = rows_path(c) ? ((size_t)c.n + 8) * 4 : m * 4;
    sz[1] = ((size_t)c.n + 1) * 4;
    sz[2] = rows_path(c) ? m * 8 : 8;
    sz[3] = rows_path(c) ? m * 4 : 8;  // edge sources of the transpose
    sz[5] = rows_path(c) ? m * 8 : 8;  // partition-pass records {u, v}
    sz[6] = 8;  // unused
    sz[7] = (4 * (size_t)PSEG_MAX + 8) * 4;  // segment tables, digit counts, unit starts of the transpose
    sz[8] = ((size_t)(m / HCH + 2) * 259 + 32) * 4;  // huge-row lists, unit starts, counters
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
