// im_abi.cu -- the C ABI of include/im.h: validation, device state, and the host
// control loops of Alg. 1 / Alg. 2 (sweep-to-fixpoint, greedy K loop).  Every step of
// the method runs in the kernels of im_kernels.cu; the host only sequences launches
// and reads back iteration counters (a few bytes per sweep / BFS level / greedy step).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <unordered_map>
#include <vector>

#include "im_device.cuh"
#include "im_internal.h"

namespace im {
}

using namespace im;

namespace {

Ctx g;
thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                                            \
    do {                                                                                                    \
        cudaError_t e_ = (call);                                                                            \
        if (e_ != cudaSuccess) {                                                                            \
            if (e_ == cudaErrorMemoryAllocation) { cudaGetLastError(); return fail(IM_ENOMEM, "%s: %s", #call, cudaGetErrorString(e_)); } \
            return fail(IM_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));    \
        }                                                                                                   \
    } while (0)

#define TRY(x)                 \
    do {                       \
        int r_ = (x);          \
        if (r_) return r_;     \
    } while (0)

// Device buffers are capacity-managed: a buffer is only reallocated when a call needs more
// bytes than it holds, so repeated loads / builds of the same workload never hit cudaMalloc /
// cudaFree.  Keys are the addresses of the Ctx pointer members.  im_free() releases all.
std::unordered_map<void*, size_t> g_cap;

template <class T>
void dfree(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
    g_cap.erase((void*)&p);
}

template <class T>
int dalloc(T*& p, size_t count, bool* fresh = nullptr) {
    size_t bytes = (count ? count : 1) * sizeof(T);
    auto it = g_cap.find((void*)&p);
    if (p && it != g_cap.end() && it->second >= bytes) {
        if (fresh) *fresh = false;
        return 0;
    }
    dfree(p);
    cudaError_t e = cudaMalloc((void**)&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        return fail(IM_ENOMEM, "cudaMalloc of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    }
    g_cap[(void*)&p] = bytes;
    if (fresh) *fresh = true;
    return 0;
}

cudaError_t tab_alloc(int32_t*& p, size_t count) { return dalloc(p, count) ? cudaErrorMemoryAllocation : cudaSuccess; }

using clk = std::chrono::steady_clock;
double ms_since(clk::time_point t0) { return std::chrono::duration<double, std::milli>(clk::now() - t0).count(); }

int ensure_device() {
    if (g.dev >= 0) return 0;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(IM_ECUDA, "no CUDA device: %s", cudaGetErrorString(e));
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, dev));
    if (p.major != 10 || p.minor != 0)
        return fail(IM_ECUDA, "this library is built for sm_100a (B200); device %d is sm_%d%d (%s)", dev, p.major, p.minor, p.name);
    g.dev = dev;
    g.num_sms = p.multiProcessorCount;
    int bs = 0, bb = 0;
    CK((cudaError_t)occupancy_sweep(&bs));
    CK((cudaError_t)occupancy_bfs(&bb));
    CK((cudaError_t)setup_argmax_tma());

    g.max_blocks_sweep = std::max(1, bs) * g.num_sms;
    g.max_blocks_bfs = std::max(1, bb) * g.num_sms;
    g.trace = getenv("IM_TRACE") != nullptr;
    if (const char* pf = getenv("IM_PULL_FRAC")) g.pull_frac = atof(pf);
    if (const char* pw = getenv("IM_PULL_FRAC_WIDE")) g.pull_frac_wide = atof(pw);
    if (const char* tr = getenv("IM_THREAD_ROWS")) g.thread_rows = atoi(tr) != 0;
    if (const char* sp = getenv("IM_SLAB_PASSES")) g.slab_passes = atoi(sp);
    if (const char* sm = getenv("IM_SLAB_MIN_M")) g.slab_min_m = atoll(sm);
    if (const char* lm = getenv("IM_LIST_MAX")) g.list_max = atoll(lm);
    if (const char* sm = getenv("IM_SLICE_MIN")) g.slice_min = atoi(sm);
    if (const char* sb = getenv("IM_SLICE_MIN_BFS")) g.slice_min_bfs = atoi(sb);
    if (const char* se = getenv("IM_SMALL_EDGES")) g.small_edges = atoll(se);
    if (const char* ss = getenv("IM_SMALL_SWEEP")) g.small_sweep_edges = atoll(ss);
    if (!g.own_stream) CK(cudaStreamCreateWithFlags(&g.own_stream, cudaStreamNonBlocking));
    if (!g.stream) g.stream = g.own_stream;
    if (!g.hpin) CK(cudaMallocHost(&g.hpin, 4096));
    if (!g.ev[0]) {
        CK(cudaEventCreate(&g.ev[0]));
        CK(cudaEventCreate(&g.ev[1]));
        for (int i = 0; i < 2; i++)
            for (int k = 0; k < 3; k++) CK(cudaEventCreate(&g.pev[i][k]));
    }
    if (const char* pp = getenv("IM_PIPELINE")) g.pipeline = atoi(pp) != 0;
    return 0;
}

void reset_sketch_state() {
    g.J = g.Jt = g.j0 = 0;
    g.built = g.fresh = g.any_blocked = false;
    g.perm.clear();
}

// forget the loaded graph (device buffers are kept for reuse; im_free releases them)
void reset_graph_state() {
    reset_sketch_state();
    g.loaded = false;
    g.n = 0;
    g.m = 0;
    g.steps.clear();
    g.st = im_stats{};
}

void release_all() {
    dfree(g.Xs); dfree(g.s12); dfree(g.permd); dfree(g.M); dfree(g.vis); dfree(g.vd);
    for (int i = 0; i < 2; i++) { dfree(g.items[i]); dfree(g.bits[i]); dfree(g.cm[i]); dfree(g.delta[i]); dfree(g.bitems[i]); dfree(g.bvl[i]); }
    dfree(g.inS); dfree(g.MS); dfree(g.btag); dfree(g.nbits); dfree(g.gain); dfree(g.big); dfree(g.list); dfree(g.lcount); dfree(g.hist);
    dfree(g.off); dfree(g.fwd); dfree(g.fwdT); dfree(g.roff); dfree(g.rev); dfree(g.revT); dfree(g.ritems); dfree(g.fbig);
    dfree(g.brec); dfree(g.bv); dfree(g.slabS); dfree(g.slabC); dfree(g.slabX); dfree(g.slabHJ); dfree(g.slabG);
    dfree(g.ftidx); dfree(g.rtidx); dfree(g.ftab); dfree(g.rtab); dfree(g.t_tabrows);
    dfree(g.ctr); dfree(g.rec); dfree(g.sbo); dfree(g.sso); dfree(g.varsigma); dfree(g.key); dfree(g.first); dfree(g.sigma_count);
    dfree(g.lval); dfree(g.sigma_g); dfree(g.bcount); dfree(g.Mold); dfree(g.gslice); dfree(g.llist); dfree(g.lcnt_all);
    dfree(g.ev_vis); dfree(g.ev_nbits); dfree(g.ev_ctr); dfree(g.ev_count);
    for (int i = 0; i < 2; i++) { dfree(g.ev_delta[i]); dfree(g.ev_items[i]); dfree(g.ev_vl[i]); }
    dfree(g.t_flags); dfree(g.t_indeg); dfree(g.t_nseg); dfree(g.t_scan); dfree(g.t_off); dfree(g.t_tgt); dfree(g.t_prob);
    dfree(g.t_est); dfree(g.t_rows); dfree(g.t_rowsout);
    for (int i = 0; i < 9; i++) dfree(g.t_prep[i]);
    reset_graph_state();
}

int sync() {
    CK(cudaStreamSynchronize(g.stream));
    return 0;
}

// Simulation sharding: the collectives of the installed communicator.  A host-staged
// communicator (stream_ordered = 0) gets a drained stream and returns with the result in place; NCCL
// (stream_ordered = 1) is enqueued on the library's stream.  No-ops when unsharded.
int coll_pre() {
    if (!g.comm.stream_ordered) TRY(sync());
    return 0;
}
int c_allreduce(void* buf, int64_t count, int32_t dtype, int32_t op) {
    if (!g.ar) return 0;
    TRY(coll_pre());
    int r = g.comm.allreduce(buf, count, dtype, op, (void*)g.stream, g.comm.user);
    if (r) return fail(IM_ECOMM, "allreduce (%s) of %lld elements failed (%d)", op == IM_OP_MAX ? "max" : "sum", (long long)count, r);
    return 0;
}
int c_reduce_scatter(const void* send, void* recv, int64_t recvcount, int32_t dtype) {
    TRY(coll_pre());
    int r = g.comm.reduce_scatter(send, recv, recvcount, dtype, (void*)g.stream, g.comm.user);
    if (r) return fail(IM_ECOMM, "reduce-scatter of %lld elements per rank failed (%d)", (long long)recvcount, r);
    return 0;
}
int c_allgather(const void* send, void* recv, int64_t sendcount, int32_t dtype) {
    TRY(coll_pre());
    int r = g.comm.allgather(send, recv, sendcount, dtype, (void*)g.stream, g.comm.user);
    if (r) return fail(IM_ECOMM, "allgather of %lld elements per rank failed (%d)", (long long)sendcount, r);
    return 0;
}
int allreduce(void* buf, int64_t count, int32_t dtype) { return c_allreduce(buf, count, dtype, IM_OP_SUM); }

void comm_release() {
    if (g.nccl) nccl_release(g.nccl);
    g.nccl = nullptr;
    g.comm = im_comm{};
    g.ar = false;
}

// read `bytes` of device memory to the pinned scratch (synchronous)
int readback(const void* dptr, size_t bytes, void* host) {
    CK(cudaMemcpyAsync(g.hpin, dptr, bytes, cudaMemcpyDeviceToHost, g.stream));
    TRY(sync());
    memcpy(host, g.hpin, bytes);
    return 0;
}

// ----------------------------------------------------------- a0: load + edge prep
// d_prob == nullptr: every edge has probability w_const (im_load_csr_const; m > 1, so the rows path never reads d_prob)
int load_common(int32_t n, int64_t m, const int32_t* d_off_src, const int32_t* d_tgt, const float* d_prob, float w_const = 0.0f) {
    auto t0 = clk::now();
    int64_t launches0 = g.launches;
    // offsets: own copy
    TRY(dalloc(g.off, (size_t)n + 1));
    CK(cudaMemcpyAsync(g.off, d_off_src, ((size_t)n + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, g.stream));
    int*& dflags = g.t_flags;
    TRY(dalloc(dflags, 4));
    CK(cudaMemsetAsync(dflags, 0, 4 * sizeof(int), g.stream));
    CK(launch_validate(g, g.off, d_tgt, d_prob, dflags));
    if (m > 0 && d_prob) CK(launch_const_check(g, d_prob, dflags + 1));
    int hf[4];
    TRY(readback(dflags, sizeof hf, hf));
    if (hf[0]) {
        return fail(IM_EINVAL, "invalid graph:%s%s%s", (hf[0] & 1) ? " offsets (offsets[0]!=0, decreasing, or offsets[n]!=m)" : "",
                    (hf[0] & 2) ? " targets out of [0,n)" : "", (hf[0] & 4) ? " probabilities not finite in [0,1]" : "");
    }
    // one scalar threshold only with m > 1 (the bucket-ordered rows path); a single edge takes the per-edge path, which
    // keeps its threshold next to the record (it wrote through the unallocated threshold array before: fixed, tested)
    g.constT = (m == 0) || (hf[1] == 0 && m > 1);
    g.T0 = 0;
    if (g.constT && m > 0) {
        float w0 = w_const;
        if (d_prob) TRY(readback(d_prob, sizeof(float), &w0));
        g.T0 = live_threshold(w0);
    }
    // constant threshold: rows ordered by h >> B0 (im_prep.cu)
    g.B0 = g.T0 <= 1u ? 0 : 32 - __builtin_clz(g.T0 - 1u);
    g.Bs = sort_shift(g.B0);
    g.sorted_h = g.constT && m > 1;
    // forward records {target, h}, thresholds, reverse records {source, h}
    TRY(dalloc(g.fwd, (size_t)m));
    TRY(dalloc(g.rev, (size_t)m));
    if (!g.constT) {
        TRY(dalloc(g.fwdT, (size_t)m));
        TRY(dalloc(g.revT, (size_t)m));
    }
    TRY(dalloc(g.roff, (size_t)n + 1));
    int32_t*& indeg = g.t_indeg;
    TRY(dalloc(indeg, 2 * ((size_t)n + 1)));
    size_t sz[9];
    CK(prep_scratch_sizes(g, sz));
    void* scr[9];
    for (int i = 0; i < 9; i++) {
        TRY(dalloc(g.t_prep[i], sz[i]));
        scr[i] = g.t_prep[i];
    }
    // bucket offset tables of the long rows (hash slices without binary searches), written by the prep
    g.nbk = 0;
    if (rows_path(g) && m > 0) {
        g.nbk = (1 << (31 - g.Bs)) + 1;
        TRY(dalloc(g.ftidx, (size_t)n));
        TRY(dalloc(g.rtidx, (size_t)n));
        TRY(dalloc(g.t_tabrows, (size_t)n));
        g.alloc_i32 = tab_alloc;
    }
    // bucket-major edge list for the slab form of the full sweeps (im_slab.cu): large constant-threshold graphs
    if (rows_path(g) && g.T0 > 0 && g.slab_passes > 0 && m >= g.slab_min_m) {
        TRY(dalloc(g.brec, (size_t)m));
        TRY(dalloc(g.bv, (size_t)m));
    } else {
        dfree(g.brec);
        dfree(g.bv);
    }
    g.boff_h.clear();
    CK(prep_edges(g, d_tgt, d_prob, indeg, nullptr, scr, sz));
    // work items: reverse segments of every vertex (sweep 1), forward item capacity (BFS)
    size_t tmp_bytes = 0;
    CK(scan_exclusive(g, indeg, g.roff, n + 1, nullptr, tmp_bytes));
    tmp_bytes += 256;
    char*& tmp = g.t_scan;
    TRY(dalloc(tmp, tmp_bytes));
    int32_t*& nseg = g.t_nseg;
    TRY(dalloc(nseg, 2 * ((size_t)n + 1)));
    CK(launch_build_items(g, g.roff, nullptr, nseg, tmp, tmp_bytes));
    int32_t total[2];
    TRY(readback(nseg + (n + 1) + n, sizeof(int32_t), &total[0]));
    g.n_ritems = total[0];
    TRY(dalloc(g.ritems, (size_t)g.n_ritems));
    CK(launch_build_items(g, g.roff, g.ritems, nseg, tmp, tmp_bytes));
    CK(launch_build_items(g, g.off, nullptr, nseg, tmp, tmp_bytes));
    TRY(readback(nseg + (n + 1) + n, sizeof(int32_t), &total[1]));
    g.n_fitems_cap = total[1];
    // rows gathered by a whole block in the first sweep
    CK(cudaMemsetAsync(g.t_flags + 2, 0, sizeof(int), g.stream));
    CK(launch_list_big_rows(g, nullptr, g.t_flags + 2));
    TRY(readback(g.t_flags + 2, sizeof(int), &g.n_fbig));
    TRY(dalloc(g.fbig, (size_t)g.n_fbig));
    CK(cudaMemsetAsync(g.t_flags + 2, 0, sizeof(int), g.stream));
    CK(launch_list_big_rows(g, g.fbig, g.t_flags + 2));
    TRY(sync());
    // small per-graph state
    TRY(dalloc(g.ctr, 2));
    TRY(dalloc(g.rec, 1));
    TRY(dalloc(g.sbo, 1));
    TRY(dalloc(g.sso, 1));
    TRY(dalloc(g.varsigma, 1));
    TRY(dalloc(g.key, 1));
    TRY(dalloc(g.first, 1));
    TRY(dalloc(g.sigma_count, 1));
    TRY(dalloc(g.sigma_g, 1));
    g.loaded = true;
    g.st = im_stats{};
    g.st.n = n;
    g.st.m = m;
    g.st.const_threshold = g.constT ? 1 : 0;
    g.st.threshold = g.T0;
    g.st.prep_ms = ms_since(t0);
    g.st.kernel_launches = g.launches - launches0;
    return 0;
}

int check_csr_args(int32_t n, int64_t m) {
    if (n < 1 || n > (1 << 28)) return fail(IM_EINVAL, "n must be in [1, 2^28] (got %d)", n);
    if (m < 0 || m > 2147483647LL) return fail(IM_EINVAL, "m must be in [0, 2^31-1] (got %lld)", (long long)m);
    return 0;
}

// ----------------------------------------------------------- a1-a4: build
int alloc_sketch_state(int32_t J) {
    size_t n = (size_t)g.n, W = (size_t)J / 32;
    bool fr = false;
    if (g.J != J) g.sweep_dirty = true;  // change-mask rows have J/32 words
    int bf = 0;
    CK((cudaError_t)setup_first(J, &bf));
    g.max_blocks_first = std::max(1, bf) * g.num_sms;
    int b2 = 0;
    CK((cudaError_t)occupancy_bfs2(J, &b2));
    g.max_blocks_bfs2 = std::max(1, b2) * g.num_sms;
    TRY(dalloc(g.Xs, (size_t)J));
    TRY(dalloc(g.s12, 4097));
    TRY(dalloc(g.permd, (size_t)J));
    TRY(dalloc(g.M, n * (size_t)J + 65536));  // + tail padding read by the TMA argmax tiles
    TRY(dalloc(g.vis, n * W + 16384));
    TRY(dalloc(g.vd, n * W));
    // slices add <= MAX_SLICES partial segments per vertex (word slices), or <= BSL per long row (bucket
    // slices; long rows <= m / TAB_MIN)
    const size_t slack = std::max<size_t>((size_t)(MAX_SLICES + 1) * n, (size_t)BSL * ((size_t)g.m / TAB_MIN + 1));
    for (int i = 0; i < 2; i++) {
        TRY(dalloc(g.items[i], (size_t)g.n_ritems + slack + 1));
        // a completed build leaves the change buffers zero; fresh ones are cleared by simulate()
        TRY(dalloc(g.bits[i], n, &fr));
        if (fr) g.sweep_dirty = true;
        TRY(dalloc(g.cm[i], n * W, &fr));
        if (fr) g.sweep_dirty = true;
        TRY(dalloc(g.delta[i], n * W, &fr));
        if (fr || g.J != J) CK(cudaMemsetAsync(g.delta[i], 0, n * W * sizeof(uint32_t), g.stream));
        TRY(dalloc(g.bitems[i], (size_t)g.n_fitems_cap + slack + 1));
        TRY(dalloc(g.bvl[i], n));
    }
    TRY(dalloc(g.inS, n));
    TRY(dalloc(g.MS, (size_t)J));
    TRY(dalloc(g.big, n));
    // sharded: the reduce-scatter needs nranks * S packed values (S = ceil(n / nranks)), and the gathered
    // candidate list holds nranks lists of <= S entries
    const int64_t nr = g.ar ? g.comm.nranks : 1, S = ((int64_t)n + nr - 1) / nr;
    TRY(dalloc(g.gain, (size_t)(nr * S)));
    TRY(dalloc(g.list, (size_t)(nr * S)));
    TRY(dalloc(g.lval, (size_t)(nr * S)));
    if (g.ar) {
        TRY(dalloc(g.gslice, (size_t)S));
        TRY(dalloc(g.llist, (size_t)S));
        TRY(dalloc(g.lcnt_all, (size_t)nr));
        CK(cudaMemsetAsync(g.gain, 0, (size_t)(nr * S) * sizeof(int32_t), g.stream));  // the pad beyond n stays 0
    }
    g.S = S;
    TRY(dalloc(g.lcount, 2));
    TRY(dalloc(g.bcount, (size_t)g.num_sms * 8));
    TRY(dalloc(g.hist, 4096));
    TRY(dalloc(g.nbits, n, &fr));  // zero between levels (consumed by k_bfs_compact)
    if (fr) CK(cudaMemsetAsync(g.nbits, 0, n * sizeof(uint32_t), g.stream));
    g.J = J;
    return 0;
}

// Alg. 1 salts (R2, R3): mt19937(low 32 bits of seed): seed_V, seed_J, X_j = draw & (2^31-1) for
// j < Jt; this context holds simulations [j0, j0 + J) of them (all of them unless sharded).
// Internally simulations are ordered by ascending salt.
int setup_salts(int32_t Jt, int32_t j0, int32_t J, uint64_t seed) {
    std::mt19937 gen((uint32_t)seed);
    g.seedV = gen();
    g.seedJ = gen();
    std::vector<uint32_t> X(J);
    for (int j = 0; j < j0 + J; j++) {
        uint32_t x = gen() & 0x7FFFFFFFu;
        if (j >= j0) X[j - j0] = x;
    }
    g.perm.resize(J);
    for (int j = 0; j < J; j++) g.perm[j] = j;
    std::stable_sort(g.perm.begin(), g.perm.end(), [&](int a, int b) { return X[a] < X[b]; });
    std::vector<uint32_t> Xs(J);
    for (int i = 0; i < J; i++) Xs[i] = X[g.perm[i]];
    std::vector<uint16_t> s12(4097);
    for (uint32_t b = 0, i = 0; b <= 4096; b++) {
        while ((int)i < J && (Xs[i] >> 19) < b) i++;
        s12[b] = (uint16_t)i;
    }
    g.Xs_h = Xs;
    CK(cudaMemcpyAsync(g.Xs, Xs.data(), J * sizeof(uint32_t), cudaMemcpyHostToDevice, g.stream));
    CK(cudaMemcpyAsync(g.s12, s12.data(), 4097 * sizeof(uint16_t), cudaMemcpyHostToDevice, g.stream));
    std::vector<int32_t> gj(J);
    for (int i = 0; i < J; i++) gj[i] = g.perm[i] + j0;
    CK(cudaMemcpyAsync(g.permd, gj.data(), J * sizeof(int32_t), cudaMemcpyHostToDevice, g.stream));
    TRY(sync());  // host vectors go out of scope
    g.seed = seed;
    g.Jt = Jt;
    g.j0 = j0;
    return 0;
}

// Alg. 1 lines 2-5 / 21-25 + Alg. 2 (eps_c = 0: to the fixpoint).  blocked: R_S = current visited bits.
// Sweep s consumes the items of the vertices changed in sweep s-1 (all in-edge segments for s = 1),
// filters by their chunk-change bits bits[(s-1)&1], records its own changes in bits[s&1]; the
// compaction then emits the next items and clears bits[(s-1)&1] for sweep s+1.
// eps_c > 0 (R22): synchronous sweeps -- the first sweep gathers from init values (already
// synchronous), later push sweeps read M_v from the pre-sweep copy Mold and k_commit refreshes it;
// the loop stops once a sweep changed <= eps_c * n vertices (Alg. 2 line 3).
int simulate(bool blocked) {
    auto t0 = clk::now();
    const size_t W = (size_t)g.J / 32;
    const double eps_c = g.eps_c;
    // Wide candidate windows (p = 0.1: J/8 simulations per edge): a pushed edge walks its window with a chain of
    // dependent loads per 8-byte word and costs ~2x a gathered one (C3 graph, J = 1024: 61M pushed edges 38 ms,
    // all 68M gathered 23 ms), so the gather is kept until the frontier's in-edges fall below 0.3 m (0.15 / 0.3 / 0.5 / 0.97: 118.7 / 118.9 / 123.8 / 142.9 ms of sweep kernels)
    const bool wide_windows = g.constT && ((int64_t)g.J << g.B0) > ((int64_t)DENSE_WIN << 31);
    const double pull_frac = wide_windows ? std::min(g.pull_frac, g.pull_frac_wide) : g.pull_frac;
    g.sync_sweeps = eps_c > 0.0;
    if (g.sync_sweeps) TRY(dalloc(g.Mold, (size_t)g.n * g.J));
    g.built_eps_c = eps_c;
    if (!(1.0 > eps_c)) {  // |V|/|V| > eps_c fails: no sweep, registers stay at their init values
        CK(launch_init_registers(g));
        TRY(sync());
        g.st.builds++;
        g.st.last_build_sweeps = 0;
        g.st.last_build_edges = 0;
        g.st.last_build_ms = ms_since(t0);
        g.built = true;
        g.fresh = !blocked;
        return 0;
    }
    if (g.sweep_dirty)
        for (int i = 0; i < 2; i++) {
            CK(cudaMemsetAsync(g.bits[i], 0, (size_t)g.n * sizeof(uint32_t), g.stream));
            CK(cudaMemsetAsync(g.cm[i], 0, (size_t)g.n * W * sizeof(uint32_t), g.stream));
        }
    g.sweep_dirty = true;  // until this build completes
    int sweeps = 0;
    int64_t edges = 0, wedges = 0, launches = 0;
    float kms = 0.f;
    int64_t edges_in = g.m;
    double alg = 0.0;
    int ngather = 0;
    bool dirty = true;  // the last sweep left change bits set (early exit, or changed vertices without in-edges)
    const int4* items = g.ritems;
    int n_items = g.n_ritems;
    edges = g.m;
    // Pipelining (eps_c = 0): once the frontier is sparse, sweep s is enqueued with its item count read on
    // the device from sweep s-1's compaction, and the host reads sweep s-1's counters (copied to pinned
    // memory) while sweep s runs; the stop test is one sweep late, and the extra sweep it then enqueued has
    // no items (a no-op).  Sweeps stay in stream order, so the registers are those of the host-driven loop.
    IterCounters* hpc = reinterpret_cast<IterCounters*>(static_cast<char*>(g.hpin) + 1024);  // 2 pinned slots
    bool piped = false;
    bool gathers[2] = {false, false};
    int last_done = 0;  // the last sweep whose counters were accounted
    // the bookkeeping of a finished sweep; returns false when the loop must stop after it
    auto account = [&](int s, const IterCounters& hc, bool gather, float t) {
        kms += t;
        sweeps++;
        launches++;
        wedges += (int64_t)hc.win_edges;
        {   // algorithmic bytes (DESIGN.md section 6 builder model): records + one 32-B sector per worked window
            const double nJ = (double)g.n * g.J, rec = 8.0 + (g.constT ? 0.0 : 4.0);
            const double cmb = (double)g.n * ((double)g.J / 8.0 + 4.0);  // change mask + chunk word per vertex
            if (s == 1) alg += rec * (double)g.m + nJ + cmb;                // + every row written once
            else if (gather) alg += rec * (double)g.m + 2.0 * nJ + cmb + 32.0 * (double)hc.win_edges;
            else alg += rec * (double)edges_in + 32.0 * (double)hc.win_edges;
            if (gather) ngather++;
        }
        if (g.trace)
            fprintf(stderr, "[im] sweep %d %s%s items %d edges %lld window_edges %llu -> changed %d next_items %d next_edges %llu big %d  %.3f ms\n",
                    s, s == 1 ? "init+gather" : gather ? "gather" : "push", piped ? " (piped)" : "", n_items,
                    (long long)(s == 1 || gather ? g.m : (int64_t)edges_in), hc.win_edges, hc.changed, hc.next_items, hc.next_edges,
                    hc.big, t);
        edges_in = (int64_t)hc.next_edges;
        dirty = hc.changed > 0;  // this sweep's change bits stay set until the next sweep consumes them
        if (!((double)hc.changed / (double)g.n > eps_c)) return false;  // Alg. 2 line 3 (eps_c = 0: nothing changed)
        if (hc.next_items == 0) return false;                            // changed vertices without in-edges
        n_items = hc.next_items;
        edges += (double)hc.next_edges > pull_frac * (double)g.m ? g.m : (int64_t)hc.next_edges;
        return true;
    };
    // k_sweep_small for the rest of the build once the frontier (after sweep s, counters hc) is small:
    // returns 0 = not taken, 1 = the build is done, 2 = continue the host loop at sweep s + 1, < 0 = error
    auto run_small = [&](int& s, const IterCounters& hc) -> int {
        const int sl = s & 1;
        if (g.sync_sweeps || g.small_sweep_edges <= 0 || (long long)hc.next_edges > g.small_sweep_edges) return 0;
        CK(cudaEventRecord(g.pev[sl][0], g.stream));
        CK(launch_sweep_small(g, g.items[sl], hc.next_items, hc.changed, s + 1, blocked, g.small_sweep_edges));
        CK(cudaEventRecord(g.pev[sl][1], g.stream));
        SweepSmallOut so;
        TRY(readback(g.sso, sizeof so, &so));
        float ts;
        CK(cudaEventElapsedTime(&ts, g.pev[sl][0], g.pev[sl][1]));
        kms += ts;
        sweeps += so.sweeps;
        launches++;
        wedges += so.win_edges;
        edges += so.edges - (int64_t)hc.next_edges;  // account() already counted the first one's in-edges
        alg += (8.0 + (g.constT ? 0.0 : 4.0)) * (double)so.edges + 32.0 * (double)so.win_edges;
        if (g.trace)
            fprintf(stderr, "[im] sweeps %d..%d in one cluster launch: %lld edges, %lld window_edges -> %s, %.3f ms\n", s + 1,
                    so.t_next - 1, so.edges, so.win_edges, so.bailed ? "frontier handed back" : "fixpoint", ts);
        if (!so.bailed) {
            dirty = false;
            return 1;
        }
        // hand back: compact the last cluster sweep's changes (its input masks were cleared in the kernel)
        const int tl = so.t_next - 1, tb = tl & 1;
        CK(cudaMemsetAsync(&g.ctr[tb], 0, sizeof(IterCounters), g.stream));
        CK(launch_compact(g, g.bits[tb], g.bits[tb ^ 1], g.cm[tb], g.cm[tb ^ 1], g.items[tb], &g.ctr[tb]));
        IterCounters hc2;
        TRY(readback(&g.ctr[tb], sizeof hc2, &hc2));
        if (hc2.next_items == 0) {
            dirty = hc2.changed > 0;
            return 1;
        }
        n_items = hc2.next_items;
        edges_in = (int64_t)hc2.next_edges;
        edges += (int64_t)hc2.next_edges;
        items = g.items[tb];
        s = tl;
        last_done = s;
        return 2;
    };
    // slab form of the first full sweeps: large constant-threshold graphs, eps_c = 0 (any schedule reaches the fixpoint)
    int slab_G = g.sync_sweeps ? 0 : slab_group_count(g);
    if (slab_G > 0) {
        const size_t ns = slab_stride(g.n);
        TRY(dalloc(g.slabS, (size_t)slab_G * ns));
        TRY(dalloc(g.slabC, (size_t)slab_G * ns));
        TRY(dalloc(g.slabX, (size_t)slab_G));
        TRY(dalloc(g.slabHJ, (size_t)slab_G));
        TRY(dalloc(g.slabG, (size_t)slab_G));
    }
    for (int s = 1;; s++) {
        const int sl = s & 1;
        IterCounters* ctr = &g.ctr[sl];
        CK(cudaMemsetAsync(ctr, 0, sizeof(IterCounters), g.stream));
        CK(cudaEventRecord(g.pev[sl][0], g.stream));
        // direction-optimised: a frontier whose in-edges cover most of the graph is swept by a full
        // in-place gather (every row owned by one warp, no atomics); sparse frontiers are pushed
        const bool gather = !piped && s > 1 && !g.sync_sweeps && (double)edges_in > pull_frac * (double)g.m;
        gathers[sl] = gather;
        if (s == 1 && slab_G > 0) {  // init + the first full sweeps in bucket-major slabs (im_slab.cu)
            CK(launch_slab_build(g, blocked, g.slab_passes, g.cm[1], g.bits[1]));
        } else if (s == 1) {  // streaming register init, then the first sweep as a gather from init values
            CK(launch_init_registers(g));
            CK(cudaMemsetAsync(g.cm[1], 0, (size_t)g.n * W * sizeof(uint32_t), g.stream));
            CK(cudaMemsetAsync(g.bits[1], 0, (size_t)g.n * sizeof(uint32_t), g.stream));
            CK(launch_first(g, g.cm[1], g.bits[1], ctr, blocked, false));
        }
        else if (gather)
            CK(launch_first(g, g.cm[sl], g.bits[sl], ctr, blocked, true));
        else
            CK(launch_sweep(g, items, n_items, g.cm[(s - 1) & 1], g.cm[sl], g.bits[sl], ctr, blocked, piped ? &g.ctr[(s - 1) & 1] : nullptr));
        CK(cudaEventRecord(g.pev[sl][1], g.stream));
        CK(launch_compact(g, g.bits[sl], g.bits[(s - 1) & 1], g.cm[sl], g.cm[(s - 1) & 1], g.items[sl], ctr));
        if (g.sync_sweeps) {  // Mold <- M (all rows after the first sweep, changed chunks after later ones)
            if (s == 1) CK(cudaMemcpyAsync(g.Mold, g.M, (size_t)g.n * g.J, cudaMemcpyDeviceToDevice, g.stream));
            else CK(launch_commit(g, g.bits[sl]));
        }
        items = g.items[sl];
        if (!piped) {
            IterCounters hc;
            CK(cudaMemcpyAsync(&hpc[sl], ctr, sizeof(IterCounters), cudaMemcpyDeviceToHost, g.stream));
            CK(cudaEventRecord(g.pev[sl][2], g.stream));
            CK(cudaEventSynchronize(g.pev[sl][2]));
            hc = hpc[sl];
            float t;
            CK(cudaEventElapsedTime(&t, g.pev[sl][0], g.pev[sl][1]));
            const bool go = account(s, hc, gather, t);
            if (s == 1 && slab_G > 0) {  // the slab build ran slab_passes full sweeps, not one
                sweeps += g.slab_passes - 1;
                edges += (int64_t)(g.slab_passes - 1) * g.m;
            }
            if (!go) break;
            last_done = s;
            {
                const int r = run_small(s, hc);
                if (r < 0) return r;
                if (r == 1) break;
                if (r == 2) continue;
            }
            // enter the pipelined mode once the next frontier is clearly sparse (no gather sweep any more)
            piped = g.pipeline && !g.sync_sweeps && s >= 2 && (double)hc.next_edges < 0.25 * pull_frac * (double)g.m;
            continue;
        }
        CK(cudaMemcpyAsync(&hpc[sl], ctr, sizeof(IterCounters), cudaMemcpyDeviceToHost, g.stream));
        CK(cudaEventRecord(g.pev[sl][2], g.stream));
        // the previous sweep's counters (its copy was enqueued one iteration ago), unless already accounted
        const int ps = (s - 1) & 1;
        if (s - 1 > last_done) {
            CK(cudaEventSynchronize(g.pev[ps][2]));
            float t;
            CK(cudaEventElapsedTime(&t, g.pev[ps][0], g.pev[ps][1]));
            if (!account(s - 1, hpc[ps], gathers[ps], t)) {  // sweep s was enqueued with no items: a no-op
                CK(cudaEventSynchronize(g.pev[sl][2]));
                dirty = true;  // conservative: the no-op's compaction cleared sweep s-1's bits; a fresh build re-zeroes
                break;
            }
            last_done = s - 1;
            if (!g.sync_sweeps && g.small_sweep_edges > 0 && (long long)hpc[ps].next_edges <= g.small_sweep_edges) {
                // sweep s (already enqueued) has a small frontier: finish it on the host side, then the cluster
                CK(cudaEventSynchronize(g.pev[sl][2]));
                const IterCounters hs = hpc[sl];
                float ts;
                CK(cudaEventElapsedTime(&ts, g.pev[sl][0], g.pev[sl][1]));
                if (!account(s, hs, false, ts)) break;
                last_done = s;
                piped = false;
                const int r = run_small(s, hs);
                if (r < 0) return r;
                if (r == 1) break;
                continue;  // r == 0 cannot happen here (the frontier only shrinks below the test above); r == 2
            }
        }
    }
    g.sweep_dirty = dirty;  // a last sweep without changes leaves every change buffer zero
    g.st.builds++;
    g.st.last_build_sweeps = sweeps;
    g.st.last_build_edges = edges;
    g.st.total_sweeps += sweeps;
    g.st.total_edges += edges;
    g.st.sweep_kernel_ms += kms;
    g.st.sweep_launches += launches;
    g.st.window_edges += wedges;
    g.st.sweep_alg_bytes += alg;
    g.st.gather_sweeps += ngather;
    g.st.last_build_ms = ms_since(t0);
    g.built = true;
    g.fresh = !blocked;
    return 0;
}

int build_fresh() {
    CK(cudaMemsetAsync(g.vis, 0, (size_t)g.n * (g.J / 32) * sizeof(uint32_t), g.stream));
    CK(cudaMemsetAsync(g.vd, 0, (size_t)g.n * (g.J / 32) * sizeof(uint2), g.stream));
    g.any_blocked = false;
    return simulate(false);
}

}  // namespace

// =========================================================== C ABI
extern "C" {

int32_t im_version(void) { return 103; }

const char* im_last_error(void) { return g_err.c_str(); }

int64_t im_kernel_launch_count(void) { return g.launches; }

int im_set_stream(void* s) {
    TRY(ensure_device());
    // NULL is CUDA's stream 0 (the legacy default stream, which torch's default stream wraps), so
    // work is ordered after the caller's kernels on it; until the first call: the library's stream
    g.stream = s ? (cudaStream_t)s : cudaStreamLegacy;
    return 0;
}

void im_free(void) {
    if (g.dev >= 0) cudaStreamSynchronize(g.stream);
    release_all();
    comm_release();
}

int im_load_csr(int32_t n, const int32_t* offsets, const int32_t* targets, const float* probs) {
    TRY(ensure_device());
    if (n < 1) return fail(IM_EINVAL, "n must be >= 1 (got %d)", n);  // before offsets[n] is read
    if (!offsets || (!targets && offsets[n] > 0) || (!probs && offsets[n] > 0))
        return fail(IM_EINVAL, "null pointer argument");
    TRY(check_csr_args(n, offsets[n]));
    if (offsets[0] != 0) return fail(IM_EINVAL, "offsets[0] must be 0");
    int64_t m = offsets[n];
    reset_graph_state();
    int32_t*& d_off = g.t_off;
    int32_t*& d_tgt = g.t_tgt;
    float*& d_prob = g.t_prob;
    TRY(dalloc(d_off, (size_t)n + 1));
    TRY(dalloc(d_tgt, (size_t)m));
    TRY(dalloc(d_prob, (size_t)m));
    CK(cudaMemcpyAsync(d_off, offsets, ((size_t)n + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, g.stream));
    if (m) {
        CK(cudaMemcpyAsync(d_tgt, targets, (size_t)m * sizeof(int32_t), cudaMemcpyHostToDevice, g.stream));
        CK(cudaMemcpyAsync(d_prob, probs, (size_t)m * sizeof(float), cudaMemcpyHostToDevice, g.stream));
    }
    g.n = n;
    g.m = m;
    int r = load_common(n, m, d_off, d_tgt, d_prob);
    if (r) reset_graph_state();
    return r;
}

int im_load_csr_device(int32_t n, int64_t m, const int32_t* d_offsets, const int32_t* d_targets, const float* d_probs) {
    TRY(ensure_device());
    if (!d_offsets || (m > 0 && (!d_targets || !d_probs))) return fail(IM_EINVAL, "null pointer argument");
    TRY(check_csr_args(n, m));
    reset_graph_state();
    g.n = n;
    g.m = m;
    int r = load_common(n, m, d_offsets, d_targets, d_probs);
    if (r) reset_graph_state();
    return r;
}

int im_load_csr_const(int32_t n, const int32_t* offsets, const int32_t* targets, float w) {
    TRY(ensure_device());
    if (n < 1) return fail(IM_EINVAL, "n must be >= 1 (got %d)", n);  // before offsets[n] is read
    if (!offsets || (!targets && offsets[n] > 0)) return fail(IM_EINVAL, "null pointer argument");
    if (!(w >= 0.0f && w <= 1.0f)) return fail(IM_EINVAL, "invalid graph: probabilities not finite in [0,1]");
    TRY(check_csr_args(n, offsets[n]));
    if (offsets[0] != 0) return fail(IM_EINVAL, "offsets[0] must be 0");
    const int64_t m = offsets[n];
    if (m <= 1) {  // no bucket-ordered rows below two edges: the array path
        const float p1 = w;
        return im_load_csr(n, offsets, targets, &p1);
    }
    reset_graph_state();
    int32_t*& d_off = g.t_off;
    int32_t*& d_tgt = g.t_tgt;
    TRY(dalloc(d_off, (size_t)n + 1));
    TRY(dalloc(d_tgt, (size_t)m));
    CK(cudaMemcpyAsync(d_off, offsets, ((size_t)n + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, g.stream));
    CK(cudaMemcpyAsync(d_tgt, targets, (size_t)m * sizeof(int32_t), cudaMemcpyHostToDevice, g.stream));
    g.n = n;
    g.m = m;
    int r = load_common(n, m, d_off, d_tgt, nullptr, w);
    if (r) reset_graph_state();
    return r;
}

int im_load_csr_const_device(int32_t n, int64_t m, const int32_t* d_offsets, const int32_t* d_targets, float w) {
    TRY(ensure_device());
    if (!d_offsets || (m > 0 && !d_targets)) return fail(IM_EINVAL, "null pointer argument");
    if (!(w >= 0.0f && w <= 1.0f)) return fail(IM_EINVAL, "invalid graph: probabilities not finite in [0,1]");
    TRY(check_csr_args(n, m));
    reset_graph_state();
    g.n = n;
    g.m = m;
    int r;
    if (m <= 1) {  // the array path (a one-entry device array)
        float*& d_prob = g.t_prob;
        TRY(dalloc(d_prob, (size_t)1));
        CK(cudaMemcpyAsync(d_prob, &w, sizeof(float), cudaMemcpyHostToDevice, g.stream));
        TRY(sync());
        r = load_common(n, m, d_offsets, d_targets, d_prob);
    } else {
        r = load_common(n, m, d_offsets, d_targets, nullptr, w);
    }
    if (r) reset_graph_state();
    return r;
}

int im_build_sketches_shard(int32_t J_total, uint64_t seed, int32_t j0, int32_t j1) {
    if (!g.loaded) return fail(IM_ESTATE, "im_build_sketches: no graph loaded");
    if (J_total < 32 || J_total > IM_MAX_J_TOTAL || J_total % 32)
        return fail(IM_EINVAL, "J_total must be a multiple of 32 in [32, %d] (got %d)", IM_MAX_J_TOTAL, J_total);
    if (j0 < 0 || j1 > J_total || j0 >= j1) return fail(IM_EINVAL, "shard [%d, %d) not inside [0, %d)", j0, j1, J_total);
    const int32_t J = j1 - j0;
    if (J < 32 || J > 1024 || J % 32) return fail(IM_EINVAL, "shard size j1 - j0 must be a multiple of 32 in [32, 1024] (got %d)", J);
    g.st.total_sweeps = 0;
    g.st.total_edges = 0;
    g.st.sweep_kernel_ms = 0;
    g.st.sweep_launches = 0;
    g.st.window_edges = 0;
    g.st.sweep_alg_bytes = 0;
    g.st.gather_sweeps = 0;
    int64_t l0 = g.launches;
    TRY(alloc_sketch_state(J));
    TRY(setup_salts(J_total, j0, J, seed));
    TRY(build_fresh());
    g.st.J = J;
    g.st.J_total = J_total;
    g.st.j0 = j0;
    g.st.kernel_launches = g.launches - l0;
    return 0;
}

int im_build_sketches(int32_t J, uint64_t seed) {
    if (J < 32 || J > 1024 || J % 32) return fail(IM_EINVAL, "J must be a multiple of 32 in [32, 1024] (got %d)", J);
    return im_build_sketches_shard(J, seed, 0, J);
}

int im_set_comm(const im_comm* comm) {
    if (comm) {
        if (comm->nranks < 1 || comm->nranks >= 256 || comm->rank < 0 || comm->rank >= comm->nranks)
            return fail(IM_EINVAL, "communicator: need 1 <= nranks < 256 and 0 <= rank < nranks (got rank %d of %d)", comm->rank,
                        comm->nranks);
        if (!comm->allreduce || !comm->reduce_scatter || !comm->allgather) return fail(IM_EINVAL, "communicator: null collective");
    }
    if (g.dev >= 0) TRY(sync());
    comm_release();
    if (comm) {
        g.comm = *comm;
        g.ar = true;
    }
    g.S = 0;  // argmax buffers are re-sized for the new rank count by the next build
    return 0;
}

int im_comm_nccl_unique_id(void* out_id128) {
    if (!out_id128) return fail(IM_EINVAL, "null output");
    char err[256];
    if (nccl_unique_id(out_id128, err, sizeof err)) return fail(IM_ECOMM, "%s", err);
    return 0;
}

int im_comm_nccl_init(const void* id128, int32_t rank, int32_t nranks) {
    TRY(ensure_device());
    if (!id128) return fail(IM_EINVAL, "null unique id");
    if (nranks < 1 || nranks >= 256 || rank < 0 || rank >= nranks)
        return fail(IM_EINVAL, "need 1 <= nranks < 256 and 0 <= rank < nranks (got rank %d of %d)", rank, nranks);
    TRY(sync());
    comm_release();
    im_comm c;
    void* st = nullptr;
    char err[256];
    if (nccl_init(id128, rank, nranks, &c, &st, err, sizeof err)) return fail(IM_ECOMM, "%s", err);
    g.comm = c;
    g.nccl = st;
    g.ar = true;
    g.S = 0;
    return 0;
}

static int shard_check(const char* what) {
    if (g.J != g.Jt && !g.ar) return fail(IM_ESTATE, "%s: sharded sketches (%d of %d simulations) need a communicator (im_set_comm)", what, g.J, g.Jt);
    if (g.ar && g.S != ((int64_t)g.n + g.comm.nranks - 1) / g.comm.nranks)
        return fail(IM_ESTATE, "%s: the communicator changed after the build; rebuild the sketches", what);
    return 0;
}

// Eq. 2 into device memory; sharded: register sums of this rank, allreduced, then Eq. 2 over J_total
static int estimate_into(double* d) {
    TRY(shard_check("im_estimate"));
    if (!g.ar) {
        CK(launch_estimate(g, d));
        return 0;
    }
    CK(launch_estimate_sums(g, g.gain));
    TRY(allreduce(g.gain, g.n, IM_DTYPE_I32));
    CK(launch_estimate_fin(g, g.gain, d));
    return 0;
}

int im_estimate_device(double* d_out) {
    if (!g.built) return fail(IM_ESTATE, "im_estimate: sketches not built");
    if (!d_out) return fail(IM_EINVAL, "null output");
    TRY(estimate_into(d_out));
    return sync();
}

int im_estimate(double* out) {
    if (!g.built) return fail(IM_ESTATE, "im_estimate: sketches not built");
    if (!out) return fail(IM_EINVAL, "null output");
    double*& d = g.t_est;
    TRY(dalloc(d, (size_t)g.n));
    TRY(estimate_into(d));
    CK(cudaMemcpyAsync(out, d, (size_t)g.n * sizeof(double), cudaMemcpyDeviceToHost, g.stream));
    return sync();
}

int im_select_seeds_ex(int32_t K, double eps_l, double eps_g, int32_t* out_seeds, double* out_scores) {
    if (!g.built) return fail(IM_ESTATE, "im_select_seeds: sketches not built");
    if (K < 0 || K > g.n) return fail(IM_EINVAL, "K must be in [0, n] (got %d, n = %d)", K, g.n);
    if (std::isnan(eps_l) || std::isnan(eps_g) || eps_l < 0 || eps_g < 0) return fail(IM_EINVAL, "thresholds must be >= 0 and not NaN");
    if (K > 0 && (!out_seeds || !out_scores)) return fail(IM_EINVAL, "null output");
    TRY(shard_check("im_select_seeds"));
    auto t0 = clk::now();
    int64_t l0 = g.launches;
    g.st.total_sweeps = 0;
    g.st.total_edges = 0;
    g.st.sweep_kernel_ms = 0;
    g.st.sweep_launches = 0;
    g.st.window_edges = 0;
    g.st.sweep_alg_bytes = 0;
    g.st.gather_sweeps = 0;
    g.st.rebuilds = 0;
    g.st.bfs_levels = 0;
    g.st.bfs_edges = 0;
    g.st_argmax_full = g.st_argmax_list = 0;
    g.steps.clear();
    if (K == 0) return 0;
    // start from S = {}, varsigma = 0, M_S' = 0 and freshly built sketches (under the current eps_c)
    if (!g.fresh || g.built_eps_c != g.eps_c) TRY(build_fresh());
    const size_t n = (size_t)g.n, W = (size_t)g.J / 32;
    CK(cudaMemsetAsync(g.vis, 0, n * W * sizeof(uint32_t), g.stream));
    CK(cudaMemsetAsync(g.vd, 0, n * W * sizeof(uint2), g.stream));
    CK(cudaMemsetAsync(g.inS, 0, n, g.stream));
    CK(cudaMemsetAsync(g.MS, 0, (size_t)g.J, g.stream));
    CK(cudaMemsetAsync(g.varsigma, 0, sizeof(double), g.stream));
    CK(cudaMemsetAsync(g.sigma_count, 0, sizeof(ull), g.stream));
    std::vector<int32_t> seeds(K);
    std::vector<double> scores(K);
    bool pool_check = false, need_full = true;
    const int T = (int)std::min<int64_t>(g.n, std::max<int64_t>(1024, std::min<int64_t>(g.list_max, g.n / 64)));
    int list_len = 0, theta = 0;
    for (int k = 0; k < K; k++) {
        // line 10: argmax over the pool (exact lazy evaluation, im_kernels.cu "a6")
        if (!need_full) {
            CK(launch_argmax_list(g, list_len));
            if (g.ar) {  // sharded: sum the packed local values of the list, then decode (im_kernels.cu)
                TRY(c_allreduce(g.lval, list_len, IM_DTYPE_I32, IM_OP_SUM));
                CK(launch_argmax_list_finish(g, list_len));
            }
            ull hk;
            TRY(readback(g.key, sizeof hk, &hk));
            if (hk == 0 || (int64_t)(hk >> 32) < theta) need_full = true;
            if (g.trace && need_full)
                fprintf(stderr, "[im] argmax k=%d lazy list %d: best gain %lld < theta %d -> full pass\n", k, list_len,
                        hk ? (long long)(hk >> 32) : -1LL, theta);
            g.st_argmax_list++;
        }
        if (need_full) {
            CK(launch_argmax_full(g, pool_check));
            if (!g.ar) {
                CK(launch_argmax_full_finish(g, T));
                int lc[2];
                TRY(readback(g.lcount, sizeof lc, lc));
                list_len = lc[0];
                theta = lc[1];
            } else {  // reduce-scatter, local argmax over the slice, max of the keys, lists gathered
                const int r = g.comm.rank, N = g.comm.nranks;
                const int64_t v0 = (int64_t)r * g.S;
                const int nv = (int)std::max<int64_t>(0, std::min<int64_t>(g.S, (int64_t)g.n - v0));
                TRY(c_reduce_scatter(g.gain, g.gslice, g.S, IM_DTYPE_I32));
                CK(launch_argmax_slice_decode(g, v0, nv));
                TRY(c_allreduce(g.key, 1, IM_DTYPE_I64, IM_OP_MAX));
                TRY(c_allreduce(g.hist, 4096, IM_DTYPE_I32, IM_OP_SUM));
                CK(launch_argmax_slice_list(g, T, v0, nv));
                TRY(c_allgather(g.lcount, g.lcnt_all, 1, IM_DTYPE_I32));
                std::vector<int32_t> cnt(N);
                TRY(readback(g.lcnt_all, N * sizeof(int32_t), cnt.data()));
                int th;
                TRY(readback(g.lcount + 1, sizeof th, &th));
                const int maxc = std::max(1, *std::max_element(cnt.begin(), cnt.end()));
                CK(launch_list_pad(g, g.llist, g.lcount, maxc));
                TRY(c_allgather(g.llist, g.list, maxc, IM_DTYPE_I32));
                list_len = N * maxc;  // with holes (-1) after each shorter rank list
                CK(launch_set_count(g, g.lcount, list_len));
                theta = th;
            }
            need_full = false;
            g.st_argmax_full++;
        }
        // lines 11, 13-14: S <- S + s, BFS for R_G(S), sigma
        CK(cudaMemsetAsync(&g.ctr[0], 0, sizeof(IterCounters), g.stream));
        CK(launch_seed_start(g, k));
        TRY(allreduce(&g.rec->score, 1, IM_DTYPE_I64));  // sharded: score summed over all simulations
        CK(launch_bfs_items(g, 0));
        IterCounters hc;
        TRY(readback(&g.ctr[0], sizeof hc, &hc));
        int cur = 0;
        while (hc.next_items > 0) {
            if ((long long)hc.next_edges <= g.small_edges) {  // small frontier: the next levels in one launch
                g.st.bfs_edges += (int64_t)hc.next_edges;
                CK(launch_bfs_small(g, cur, hc.changed, g.small_edges));
                BfsSmallOut so;
                TRY(readback(g.sbo, sizeof so, &so));
                g.st.bfs_levels += so.levels;
                g.st.bfs_edges += so.edges;
                cur = so.cur;
                if (g.trace)
                    fprintf(stderr, "[im] bfs k=%d single-block: %d levels, %lld edges -> %s frontier %d\n", k, so.levels, so.edges,
                            so.bailed ? "large" : "empty", so.n_v);
                hc = IterCounters{};
                if (!so.bailed) break;
                CK(launch_bfs_items(g, cur));  // continue on the multi-block path from the frontier it left
                TRY(readback(&g.ctr[cur], sizeof hc, &hc));
                continue;
            }
            int n_items = hc.next_items, n_v = hc.changed;
            g.st.bfs_edges += (int64_t)hc.next_edges;
            uint32_t tag = ++g.bt;
            CK(cudaMemsetAsync(&g.ctr[cur ^ 1], 0, sizeof(IterCounters), g.stream));
            CK(launch_bfs_level(g, cur, n_items, tag));
            CK(launch_bfs_clear(g, cur, n_v));
            TRY(readback(&g.ctr[cur ^ 1], sizeof hc, &hc));
            if (g.trace)
                fprintf(stderr, "[im] bfs k=%d level items %d frontier %d -> frontier %d next_items %d next_edges %llu big %d new_bits %llu\n",
                        k, n_items, n_v, hc.changed, hc.next_items, hc.next_edges, hc.big, hc.new_bits);
            cur ^= 1;
            g.st.bfs_levels++;
            if (!g.pipeline || (long long)hc.next_edges <= 4 * g.small_edges) continue;
            // Pipelined levels (large frontiers): level L is enqueued with its item count / frontier size read
            // on the device, then level L-1's counters (copied to pinned memory) are read while L runs; the
            // stop / small-frontier test is one level late, the level it then enqueued has no items if the
            // BFS was over (a no-op).  Levels stay in stream order: the visited bits are those of the
            // host-driven loop.
            IterCounters* hpc = reinterpret_cast<IterCounters*>(static_cast<char*>(g.hpin) + 1024);
            bool over = false;
            int level_done = 0;  // levels whose counters were read (the first piped one has none yet)
            for (int L = 0;; L++) {
                const int nx = cur ^ 1;
                CK(cudaMemsetAsync(&g.ctr[nx], 0, sizeof(IterCounters), g.stream));
                CK(launch_bfs_level(g, cur, 0, ++g.bt, true));
                CK(launch_bfs_clear(g, cur, 0, true));
                CK(cudaMemcpyAsync(&hpc[nx], &g.ctr[nx], sizeof(IterCounters), cudaMemcpyDeviceToHost, g.stream));
                CK(cudaEventRecord(g.pev[nx][2], g.stream));
                cur = nx;
                if (L == 0) {
                    g.st.bfs_edges += (int64_t)hc.next_edges;  // its input, read by the host loop
                    continue;
                }
                CK(cudaEventSynchronize(g.pev[cur ^ 1][2]));  // the level before the one just enqueued
                const IterCounters pc = hpc[cur ^ 1];
                level_done = L;
                g.st.bfs_levels++;
                if (pc.next_items == 0) {  // the level just enqueued had no items; its clear ran on the frontier
                    CK(cudaEventSynchronize(g.pev[cur][2]));
                    over = true;
                    break;
                }
                g.st.bfs_edges += (int64_t)pc.next_edges;
                if ((long long)pc.next_edges <= g.small_edges) break;  // back to the host loop (small path)
            }
            (void)level_done;
            if (over) {
                hc = IterCounters{};
                break;
            }
            CK(cudaEventSynchronize(g.pev[cur][2]));  // the last enqueued level's counters
            hc = hpc[cur];
            g.st.bfs_levels++;
        }
        if (hc.changed > 0) CK(launch_bfs_clear(g, cur, hc.changed));  // frontier without work items
        pool_check = true;
        g.any_blocked = true;
        // lines 12, 15-27: error test, M_S' merge or rebuild decision (sharded: on the summed sigma count,
        // so every rank takes the same decision)
        if (g.ar) {
            CK(cudaMemcpyAsync(g.sigma_g, g.sigma_count, sizeof(ull), cudaMemcpyDeviceToDevice, g.stream));
            TRY(allreduce(g.sigma_g, 1, IM_DTYPE_I64));
        }
        CK(launch_error_check(g, k, K, eps_l, eps_g));
        StepDev rec;
        TRY(readback(g.rec, sizeof rec, &rec));
        im_step s;
        static_assert(sizeof(im_step) == sizeof(StepDev), "im_step layout");
        memcpy(&s, &rec, sizeof s);
        g.steps.push_back(s);
        seeds[k] = rec.vertex;
        scores[k] = rec.sigma;
        if (rec.executed) {  // lines 21-25: rebuild on the residual graph, R_S = R_G(S)
            TRY(simulate(true));
            g.st.rebuilds++;
            need_full = true;
        }
    }
    memcpy(out_seeds, seeds.data(), K * sizeof(int32_t));
    memcpy(out_scores, scores.data(), K * sizeof(double));
    g.st.last_select_ms = ms_since(t0);
    g.st.kernel_launches = g.launches - l0;
    return 0;
}

int im_select_seeds(int32_t K, double err_threshold, int32_t* out_seeds, double* out_scores) {
    const double l = std::isnan(g.pol_l) ? err_threshold : g.pol_l, gg = std::isnan(g.pol_g) ? err_threshold : g.pol_g;
    return im_select_seeds_ex(K, l, gg, out_seeds, out_scores);
}

int im_set_policy(double eps_l, double eps_g, double eps_c) {
    if ((!std::isnan(eps_l) && eps_l < 0) || (!std::isnan(eps_g) && eps_g < 0))
        return fail(IM_EINVAL, "eps_l / eps_g must be >= 0 or NaN (got %g, %g)", eps_l, eps_g);
    if (std::isnan(eps_c) || eps_c < 0 || eps_c > 1) return fail(IM_EINVAL, "eps_c must be in [0, 1] (got %g)", eps_c);
    g.pol_l = eps_l;
    g.pol_g = eps_g;
    g.eps_c = eps_c;
    return 0;
}

static void unpermute_rows(const uint8_t* in, uint8_t* out, int64_t nrows) {
    const int J = g.J;
    for (int64_t r = 0; r < nrows; r++)
        for (int jj = 0; jj < J; jj++) out[r * J + g.perm[jj]] = in[r * J + jj];
}

int im_get_register_rows(int64_t nrows, const int32_t* rows, uint8_t* out) {
    if (!g.built) return fail(IM_ESTATE, "registers not built");
    if (nrows < 0 || (nrows > 0 && (!rows || !out))) return fail(IM_EINVAL, "bad arguments");
    for (int64_t i = 0; i < nrows; i++)
        if (rows[i] < 0 || rows[i] >= g.n) return fail(IM_EINVAL, "row %lld out of range", (long long)i);
    if (nrows == 0) return 0;
    int32_t*& drows = g.t_rows;
    uint8_t*& dout = g.t_rowsout;
    TRY(dalloc(drows, (size_t)nrows));
    TRY(dalloc(dout, (size_t)nrows * g.J));
    CK(cudaMemcpyAsync(drows, rows, nrows * sizeof(int32_t), cudaMemcpyHostToDevice, g.stream));
    CK(launch_gather_rows(g, drows, nrows, dout));
    std::vector<uint8_t> tmp((size_t)nrows * g.J);
    CK(cudaMemcpyAsync(tmp.data(), dout, tmp.size(), cudaMemcpyDeviceToHost, g.stream));
    TRY(sync());
    unpermute_rows(tmp.data(), out, nrows);
    return 0;
}

int im_get_registers(uint8_t* out) {
    if (!g.built) return fail(IM_ESTATE, "registers not built");
    if (!out) return fail(IM_EINVAL, "null output");
    std::vector<uint8_t> tmp((size_t)g.n * g.J);
    CK(cudaMemcpyAsync(tmp.data(), g.M, tmp.size(), cudaMemcpyDeviceToHost, g.stream));
    TRY(sync());
    unpermute_rows(tmp.data(), out, g.n);
    return 0;
}

int im_get_reach(uint32_t* out) {
    if (!g.built) return fail(IM_ESTATE, "sketches not built");
    if (!out) return fail(IM_EINVAL, "null output");
    const size_t W = (size_t)g.J / 32, n = (size_t)g.n;
    std::vector<uint32_t> tmp(n * W);
    CK(cudaMemcpyAsync(tmp.data(), g.vis, tmp.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, g.stream));
    TRY(sync());
    for (size_t v = 0; v < n; v++) {
        uint32_t* o = out + v * W;
        for (size_t w = 0; w < W; w++) o[w] = 0;
        for (int jj = 0; jj < g.J; jj++)
            if (tmp[v * W + (jj >> 5)] >> (jj & 31) & 1u) {
                int j = g.perm[jj];
                o[j >> 5] |= 1u << (j & 31);
            }
    }
    return 0;
}

int im_evaluate(int32_t K, const int32_t* seeds, uint64_t seed, int64_t r0, int64_t R, int64_t* out_counts) {
    if (!g.loaded) return fail(IM_ESTATE, "im_evaluate: no graph loaded");
    if (K < 0 || K > g.n) return fail(IM_EINVAL, "K must be in [0, n] (got %d)", K);
    if (r0 < 0 || R < 32 || R % 32) return fail(IM_EINVAL, "r0 >= 0 and R a positive multiple of 32 required (got %lld, %lld)",
                                               (long long)r0, (long long)R);
    if (K > 0 && (!seeds || !out_counts)) return fail(IM_EINVAL, "null pointer argument");
    for (int k = 0; k < K; k++)
        if (seeds[k] < 0 || seeds[k] >= g.n) return fail(IM_EINVAL, "seed %d out of range", k);
    if (K == 0) return 0;
    const int64_t l0 = g.launches;
    const int B = (int)std::min<int64_t>(R, 512), Wb = B / 32;
    const size_t n = (size_t)g.n;
    bool fr = false;
    TRY(dalloc(g.ev_vis, n * Wb));
    for (int i = 0; i < 2; i++) {
        TRY(dalloc(g.ev_delta[i], n * Wb, &fr));
        if (fr) CK(cudaMemsetAsync(g.ev_delta[i], 0, n * Wb * sizeof(uint32_t), g.stream));
        TRY(dalloc(g.ev_items[i], (size_t)g.n_fitems_cap + 1));
        TRY(dalloc(g.ev_vl[i], n));
    }
    TRY(dalloc(g.ev_ctr, 2));
    TRY(dalloc(g.ev_count, 1));
    TRY(dalloc(g.ev_nbits, n, &fr));
    if (fr) CK(cudaMemsetAsync(g.ev_nbits, 0, n * sizeof(uint32_t), g.stream));
    std::vector<int64_t> acc(K, 0);
    for (int64_t b0 = r0; b0 < r0 + R; b0 += B) {
        const int Bb = (int)std::min<int64_t>(B, r0 + R - b0), W = Bb / 32;
        CK(cudaMemsetAsync(g.ev_vis, 0, n * W * sizeof(uint32_t), g.stream));
        CK(cudaMemsetAsync(g.ev_count, 0, sizeof(ull), g.stream));
        for (int k = 0; k < K; k++) {
            CK(cudaMemsetAsync(&g.ev_ctr[0], 0, sizeof(IterCounters), g.stream));
            CK(launch_mc_start(g, seeds[k], W, g.ev_count));
            CK(launch_bfs_items_raw(g, g.ev_vl[0], g.ev_items[0], &g.ev_ctr[0]));
            IterCounters hc;
            TRY(readback(&g.ev_ctr[0], sizeof hc, &hc));
            int cur = 0;
            while (hc.next_items > 0) {
                const int n_items = hc.next_items, n_v = hc.changed;
                CK(cudaMemsetAsync(&g.ev_ctr[cur ^ 1], 0, sizeof(IterCounters), g.stream));
                CK(launch_mc_level(g, cur, n_items, W, seed, (ull)b0, g.ev_count));
                CK(launch_bfs_clear_raw(g, n_v, W, g.ev_vl[cur], g.ev_delta[cur]));
                TRY(readback(&g.ev_ctr[cur ^ 1], sizeof hc, &hc));
                cur ^= 1;
            }
            if (hc.changed > 0) CK(launch_bfs_clear_raw(g, hc.changed, W, g.ev_vl[cur], g.ev_delta[cur]));
            ull cnt;
            TRY(readback(g.ev_count, sizeof cnt, &cnt));
            acc[k] += (int64_t)cnt;  // cumulative over the prefix within this batch
        }
    }
    memcpy(out_counts, acc.data(), K * sizeof(int64_t));
    g.st.kernel_launches = g.launches - l0;
    return 0;
}

int im_get_step_log(im_step* out, int32_t cap) {
    if (cap < 0 || (cap > 0 && !out)) return fail(IM_EINVAL, "bad arguments");
    int k = (int)std::min<size_t>((size_t)cap, g.steps.size());
    if (k) memcpy(out, g.steps.data(), k * sizeof(im_step));
    return k;
}

int im_get_stats(im_stats* out) {
    if (!out) return fail(IM_EINVAL, "null output");
    *out = g.st;
    out->argmax_full = g.st_argmax_full;
    out->argmax_lazy = g.st_argmax_list;
    out->sorted_rows = g.sorted_h ? 1 : 0;
    out->n = g.n;
    out->J = g.J;
    out->m = g.m;
    out->eps_c = g.built ? g.built_eps_c : g.eps_c;
    return 0;
}

}  // extern "C"
