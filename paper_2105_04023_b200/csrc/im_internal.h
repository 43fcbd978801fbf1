// im_internal.h -- library-private state and kernel launchers (host side).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/im.h"

namespace im {

typedef unsigned long long ull;

constexpr int SEG = 256;        // max edges per work item (a segment of one vertex's edge list)
constexpr int TAB_MIN = SEG;  // rows longer than this get a bucket offset table (rows path)
constexpr int MAX_SLICES = 8; // hash slices per long row (more non-zero mask words: the whole row)
constexpr int BSL = 32;       // bucket slices per long row with a bucket table (k_slices_buckets)
#ifndef IM_DENSE_WIN
#define IM_DENSE_WIN 32
#endif
constexpr int DENSE_WIN = IM_DENSE_WIN;   // windows wider than this many simulations take the warp-cooperative path
constexpr int BLOCK = 256;      // threads per block of the persistent work-list kernels
#ifndef IM_FIRST_BIG
#define IM_FIRST_BIG 2048
#endif
constexpr int FIRST_BIG = IM_FIRST_BIG; // first sweep: rows with more out-edges are gathered by whole blocks
constexpr int FIRST_CHUNK = 8192;       // edges per work unit of such a row (k_first_big)
constexpr uint32_t SHARD_POOL_ONE = 1u << 24;  // sharded argmax: gain + (in local pool) << 24, summed over ranks

// device-side counters of one sweep / BFS level (one 32-byte D2H per iteration)
struct IterCounters {
    int next_items;     // work items appended for the next iteration
    int changed;        // vertices that changed (first change per iteration)
    ull next_edges;     // edges covered by the appended items
    int batch;          // dynamic batch cursor of the persistent kernel
    int big;            // long rows queued for per-word slicing (k_slices_big)
    ull new_bits;       // BFS: newly visited (vertex, simulation) pairs
    ull win_edges;      // sweep: edges with a non-empty candidate window (after the change filter)
};

// result of a single-block small-frontier BFS run (im_bfs_small.cu)
struct BfsSmallOut {
    int levels;      // levels run
    int cur;         // frontier buffer holding the frontier left (bailed) / the last one
    int n_v;         // its vertices (0: the BFS is complete)
    int bailed;      // 1: stopped because the next frontier's out-edges exceed max_edges
    long long edges; // edges enumerated by the levels run, after the entry frontier's
};

// result of a one-cluster small-frontier sweep run (im_sweep.cu k_sweep_small)
struct SweepSmallOut {
    int sweeps;            // sweeps run
    int changed;           // vertices changed by the last one
    int bailed;            // 1: the next frontier's in-edges exceed max_edges (the host loop continues)
    int t_next;            // index of the next sweep (buffer parity)
    long long edges;       // in-edges enumerated by the sweeps run
    long long win_edges;   // of which with a worked window
    long long next_edges;  // in-edges of the frontier left (bailed)
};

struct StepDev {  // mirrors im_step
    int32_t vertex, pad;
    int64_t score;
    double e;
    int64_t sigma_count;
    double sigma, delta, err_l, err_g;
    int32_t rebuilt, executed;
};

struct Ctx {
    int dev = -1, num_sms = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    // graph (Sec. 3.3 CSR) + edge prep (Eq. 4-5)
    bool loaded = false;
    int32_t n = 0;
    int64_t m = 0;
    int32_t* off = nullptr;     // n+1 forward offsets
    uint2* fwd = nullptr;       // m {target, h}
    uint32_t* fwdT = nullptr;   // m per-edge thresholds (null when constant)
    int32_t* roff = nullptr;    // n+1 reverse offsets
    uint2* rev = nullptr;       // m {source, h} grouped by target
    uint32_t* revT = nullptr;
    bool constT = true;
    uint32_t T0 = 0;
    int B0 = 0;                 // thr_bits(T0): candidate windows are salt blocks of 2^B0
    int Bs = 0;                 // bucket shift of the row order / bucket tables: max(B0, 23), <= 2^8 buckets
    bool sorted_h = false;      // adjacency rows sorted by h (constant threshold only)
    int4* ritems = nullptr;     // all reverse segments {v, eb, ee, 0}
    int nbk = 0;                // bucket offset tables: 2^KB + 1 entries per long row (0: none, binary search)
    int32_t* ftidx = nullptr;   // per vertex: its forward row's table, -1 if none
    int32_t* rtidx = nullptr;
    int32_t* ftab = nullptr;    // forward tables [rows x nbk]
    int32_t* rtab = nullptr;
    int32_t* t_tabrows = nullptr;
    cudaError_t (*alloc_i32)(int32_t*&, size_t) = nullptr;  // device allocation with capacity reuse (im_abi.cu)
    int32_t n_ritems = 0;
    int32_t n_fitems_cap = 0;   // sum_v ceil(outdeg/SEG)
    // bucket-major edge list and slabs of the full sweeps (im_slab.cu)
    uint2* brec = nullptr;      // m {source u, h} grouped by bucket h >> Bs (null: no slab path for this graph)
    int32_t* bv = nullptr;      // m targets v, same order
    std::vector<int32_t> boff_h;  // bucket offsets [2^(31-Bs) + 1] (host)
    uint32_t* slabS = nullptr;  // G x n packed registers (4 simulations of one bucket per word)
    uint8_t* slabC = nullptr;   // G x n change nibbles of the last slab pass
    uint4* slabX = nullptr;     // [G] salts of the group's simulations
    uint4* slabHJ = nullptr;    // [G] hash(j) of the group's simulations
    int4* slabG = nullptr;      // [G] {first simulation s0, count, bucket, byte mask}
    std::vector<int4> slabG_h;
    std::vector<uint32_t> Xs_h; // sorted salts (host copy)
    int slab_passes = 0;        // in-place full passes per build in slab form (IM_SLAB_PASSES; 0 = off, the default: measured slower)
    int64_t slab_min_m = 8 << 20;  // graphs with fewer edges keep the row-major full sweeps (IM_SLAB_MIN_M)
    int4* fbig = nullptr;       // work units {u, eb, ee} of the rows with > FIRST_BIG out-edges (<= FIRST_CHUNK edges each)
    int32_t n_fbig = 0;
    // sketches
    int32_t J = 0;              // simulations held here (this rank's shard)
    int32_t Jt = 0, j0 = 0;     // all simulations of the job / global index of the first one held here
    uint64_t seed = 0;
    uint32_t seedV = 0, seedJ = 0;
    std::vector<int32_t> perm;  // internal (ascending salt) index -> local simulation column j - j0
    uint32_t* Xs = nullptr;     // sorted salts [J]
    uint16_t* s12 = nullptr;    // [4097]
    int32_t* permd = nullptr;   // [J] internal index -> global simulation j (hash input of Eq. 1)
    uint8_t* M = nullptr;       // n*J registers, row-major, internal simulation order
    uint8_t* Mold = nullptr;    // pre-sweep copy read by synchronous sweeps (eps_c > 0, R22), n*J
    bool sync_sweeps = false;   // the running Simulate uses synchronous sweeps
    // policy (im_set_policy): NaN eps_l / eps_g = the threshold of the select call
    double pol_l = __builtin_nan(""), pol_g = __builtin_nan(""), eps_c = 0.0;
    double built_eps_c = 0.0;   // eps_c of the sketches currently held
    uint32_t* vis = nullptr;    // n*(J/32) R_G(S) bits, internal order
    uint2* vd = nullptr;        // BFS-internal {visited, new in this level} pairs, n*(J/32); .x == vis between levels
    bool built = false, fresh = false, any_blocked = false;
    // sweep buffers
    int4* items[2] = {nullptr, nullptr};
    uint32_t* bits[2] = {nullptr, nullptr};  // per-vertex 32-simulation-chunk change bits, ping-pong
    uint32_t* cm[2] = {nullptr, nullptr};    // per-(vertex, simulation) change masks, n x J/32 words, ping-pong
    int32_t* big = nullptr;                  // long rows awaiting slicing
    bool sweep_dirty = true;   // change buffers may hold stale bits (fresh / aborted build)
    bool trace = false;        // IM_TRACE: per-sweep / per-level lines on stderr
    bool pipeline = true;      // IM_PIPELINE=0 disables: sparse sweeps are enqueued before the previous one's counters are read
    cudaEvent_t pev[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};  // per slot: sweep start / end, counters copied
    int slice_min = SEG;       // sweeps: in-rows longer than this are enumerated by hash slices (IM_SLICE_MIN)
    int slice_min_bfs = SEG;   // BFS levels: out-rows longer than this are enumerated by hash slices (IM_SLICE_MIN_BFS)
    int64_t list_max = 65536;  // cap of the lazy argmax candidate list length (IM_LIST_MAX)
    bool thread_rows = true;   // first / gather sweeps: rows <= 32 out-edges one per lane (IM_THREAD_ROWS=0: warp per row)
    double pull_frac_wide = 0.3;  // the same threshold when the candidate windows are wide (> DENSE_WIN simulations; IM_PULL_FRAC_WIDE)
    double pull_frac = 0.97;   // gather sweep when the push frontier's in-edges exceed this share of m (IM_PULL_FRAC)
    IterCounters* ctr = nullptr;   // [2]
    // selection buffers
    uint8_t* inS = nullptr;
    uint8_t* MS = nullptr;
    uint32_t* delta[2] = {nullptr, nullptr};
    int4* bitems[2] = {nullptr, nullptr};
    int32_t* bvl[2] = {nullptr, nullptr};
    uint32_t* btag = nullptr;
    uint32_t bt = 0;
    uint32_t* nbits = nullptr;   // BFS: per-vertex words with new bits in the current level
    StepDev* rec = nullptr;
    BfsSmallOut* sbo = nullptr;
    SweepSmallOut* sso = nullptr;
    long long small_sweep_edges = 32768;  // sweep frontiers with at most this many in-edges: one-cluster sweeps (IM_SMALL_SWEEP; 0 = off)
    long long small_edges = 32768;  // frontiers with at most this many out-edges: one-cluster BFS (IM_SMALL_EDGES; 0 = off)
    double* varsigma = nullptr;
    ull* key = nullptr;
    int* first = nullptr;
    int32_t* gain = nullptr;     // stored gains of the last full argmax pass (-1: not in the pool)
    int32_t* list = nullptr;     // candidate list of the lazy argmax
    int* lcount = nullptr;       // [0] list length, [1] theta
    int* bcount = nullptr;       // per-block match counts of the ordered list build [num_sms * 8]
    uint32_t* hist = nullptr;    // gain histogram of the full pass
    ull* sigma_count = nullptr;
    // simulation sharding: the communicator (im_set_comm / im_comm_nccl_init)
    im_comm comm{};
    bool ar = false;             // a communicator is installed (sharded exchanges on)
    void* nccl = nullptr;        // the library's own NCCL communicator state (im_comm.cu), or null
    int64_t S = 0;               // vertex slice per rank of the reduce-scatter: ceil(n / nranks)
    int32_t* gslice = nullptr;   // this rank's slice of the summed packed argmax values / stored gains [S]
    int32_t* llist = nullptr;    // this rank's candidate list (its slice's vertices with gain >= theta) [S]
    int32_t* lcnt_all = nullptr; // candidate-list lengths of every rank [nranks]
    int32_t* lval = nullptr;     // packed local values of the lazy-list argmax [list capacity]
    ull* sigma_g = nullptr;      // sigma count summed over ranks
    // Monte-Carlo evaluator (im_eval.cu): B-sample masks, frontier buffers
    uint32_t* ev_vis = nullptr;
    uint32_t* ev_delta[2] = {nullptr, nullptr};
    int4* ev_items[2] = {nullptr, nullptr};
    int32_t* ev_vl[2] = {nullptr, nullptr};
    IterCounters* ev_ctr = nullptr;  // [2]
    uint32_t* ev_nbits = nullptr;
    ull* ev_count = nullptr;
    // reused temporaries (edge prep, host-pointer loads, diagnostics)
    int* t_flags = nullptr;
    int32_t* t_indeg = nullptr;
    int32_t* t_nseg = nullptr;
    char* t_scan = nullptr;
    int32_t* t_off = nullptr;
    int32_t* t_tgt = nullptr;
    float* t_prob = nullptr;
    double* t_est = nullptr;
    int32_t* t_rows = nullptr;
    char* t_prep[9] = {};  // edge-prep scratch (im_prep.cu)
    uint8_t* t_rowsout = nullptr;
    // host pinned scratch
    void* hpin = nullptr;
    // bookkeeping
    im_stats st{};
    std::vector<im_step> steps;
    int64_t launches = 0;
    int st_argmax_full = 0, st_argmax_list = 0;
    int max_blocks_sweep = 0, max_blocks_bfs = 0, max_blocks_first = 0, max_blocks_bfs2 = 0;
    cudaEvent_t ev[2] = {nullptr, nullptr};
};

// grid for a grid-stride kernel over `work` threads, capped at 8 resident blocks per SM
inline int grid_for(Ctx& c, int64_t work, int per_block = BLOCK) {
    int64_t g = (work + per_block - 1) / per_block;
    int64_t cap = (int64_t)c.num_sms * 8;
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}
#define LAUNCHED(c) ((c).launches++, cudaGetLastError())

// ---- launchers (im_kernels.cu, im_sweep.cu); all enqueue on c.stream, return cudaError_t ----
cudaError_t launch_compact(Ctx& c, const uint32_t* bits_new, uint32_t* bits_clear, const uint32_t* cm_new,
                           uint32_t* cm_clear, int4* items_out, IterCounters* ctr);
int occupancy_sweep(int* blocks_per_sm);
int occupancy_bfs(int* blocks_per_sm);
int occupancy_bfs2(int J, int* blocks_per_sm);
int setup_first(int J, int* blocks_per_sm);  // smem opt-in + occupancy of the first-sweep kernel for this J
// register init + first sweep (gather, im_first.cu): writes every row, its change mask and chunk bits
cudaError_t launch_first(Ctx& c, uint32_t* cm_out, uint32_t* bits_out, IterCounters* ctr, bool blocked, bool from_memory);
cudaError_t launch_list_big_rows(Ctx& c, int4* units, int* count);  // units == nullptr: count only
// slab form of the first `passes` full sweeps of a build (im_slab.cu): group table for the current salts,
// then init + passes + transpose into M / cm_out / bits_out
inline size_t slab_stride(int32_t n) { return ((size_t)n + 31) & ~(size_t)31; }  // entries per group slab
int slab_group_count(Ctx& c);  // fills c.slabG_h; number of groups, or 0 when the slab path does not apply
cudaError_t launch_slab_build(Ctx& c, bool blocked, int passes, uint32_t* cm_out, uint32_t* bits_out);
bool rows_path(const Ctx& c);  // constant threshold: long rows bucket-ordered (h >> Bs), bucket tables
int sort_shift(int B0);        // Bs for a threshold's B0

cudaError_t launch_validate(Ctx& c, const int32_t* off, const int32_t* tgt, const float* prob, int* flags);
cudaError_t launch_const_check(Ctx& c, const float* prob, int* flag);
cudaError_t prep_scratch_sizes(Ctx& c, size_t* sz);  // 9 sizes (bytes) for prep_edges scratch
cudaError_t prep_edges(Ctx& c, const int32_t* tgt, const float* prob, int32_t* indeg, int32_t* unused, void** scr,
                       const size_t* sz);
cudaError_t launch_build_items(Ctx& c, const int32_t* offs, int4* items, int32_t* nseg_scratch, void* tmp, size_t tmp_bytes);
cudaError_t scan_exclusive(Ctx& c, const int32_t* in, int32_t* out, int n, void* tmp, size_t& tmp_bytes);
cudaError_t launch_salt_tables(Ctx& c);
cudaError_t launch_init_registers(Ctx& c);
// one sweep over `items`; cm_in: per-simulation change mask of the previous sweep (null: no filter,
// sweep 1); cm_out / bits_out: this sweep's change mask and chunk summary; counters in *ctr (zeroed)
// nin non-null: the item count is read on the device from nin->next_items (n_items ignored)
cudaError_t launch_sweep(Ctx& c, const int4* items, int n_items, const uint32_t* cm_in, uint32_t* cm_out,
                         uint32_t* bits_out, IterCounters* ctr, bool blocked, const IterCounters* nin = nullptr);
cudaError_t launch_commit(Ctx& c, const uint32_t* bits_new);
// the remaining sweeps of a build from the work items of sweep s0 - 1's compaction, in one cluster launch
cudaError_t launch_sweep_small(Ctx& c, const int4* items, int n_items, int n_changed, int s0, bool blocked, long long max_edges);
cudaError_t launch_slices_big(Ctx& c, const int32_t* big, const uint32_t* mask, const int32_t* offs, const uint2* rec,
                              int4* items_out, IterCounters* ctr, bool whole_dense);
cudaError_t launch_estimate(Ctx& c, double* out);
cudaError_t launch_estimate_sums(Ctx& c, int32_t* sums);
cudaError_t launch_estimate_fin(Ctx& c, const int32_t* sums, double* out);
cudaError_t launch_argmax_full(Ctx& c, bool pool);
cudaError_t launch_argmax_full_finish(Ctx& c, int T);
// sharded full pass after the reduce-scatter: decode this rank's slice (key, stored gains, histogram)
cudaError_t launch_argmax_slice_decode(Ctx& c, int64_t v0, int nv);
// sharded: theta from the (summed) histogram, this rank's slice list into c.llist, its length into c.lcount[0]
cudaError_t launch_argmax_slice_list(Ctx& c, int T, int64_t v0, int nv);
cudaError_t launch_list_pad(Ctx& c, int32_t* list, const int* count, int cap);  // list[count..cap) = -1
cudaError_t launch_set_count(Ctx& c, int* p, int v);  // *p = v on the stream
cudaError_t launch_argmax_list_finish(Ctx& c, int list_len);
cudaError_t launch_argmax_tma(Ctx& c, bool pool, int L, int C, int shift);
int setup_argmax_tma();
cudaError_t launch_argmax_list(Ctx& c, int list_len);
cudaError_t launch_seed_start(Ctx& c, int k);
// one BFS level from frontier buffer cur (items, Delta) into cur^1, plus the compaction that builds
// the next frontier's vertex list / items and adds the level's new bits to sigma
// piped: the item count / frontier size are read on the device from c.ctr[cur] (no host round trip)
cudaError_t launch_bfs_level(Ctx& c, int cur, int n_items, uint32_t tag, bool piped = false);
cudaError_t launch_bfs_clear(Ctx& c, int cur, int n_v, bool piped = false);
// the rest of a BFS from frontier buffer cur (n_v vertices) in one single-block launch (result in c.sbo)
cudaError_t launch_bfs_small(Ctx& c, int cur, int n_v, long long max_edges);
cudaError_t launch_bfs_items(Ctx& c, int buf);
cudaError_t launch_error_check(Ctx& c, int k, int K, double eps_l, double eps_g);
cudaError_t launch_bfs_compact_raw(Ctx& c, int J, uint32_t* nbits, const uint32_t* dout, int32_t* vl, int4* items,
                                   IterCounters* ctr, ull* count);
cudaError_t launch_bfs_items_raw(Ctx& c, const int32_t* vl, int4* items, IterCounters* ctr);
cudaError_t launch_bfs_clear_raw(Ctx& c, int n_v, int W, const int32_t* vl, uint32_t* delta);
// Monte-Carlo evaluator (im_eval.cu)
cudaError_t launch_mc_start(Ctx& c, int32_t s, int W, ull* count);
cudaError_t launch_mc_level(Ctx& c, int cur, int n_items, int W, ull seed, ull r0, ull* count);
cudaError_t launch_gather_rows(Ctx& c, const int32_t* rows, int64_t nrows, uint8_t* out);

// the library's own NCCL communicator (im_comm.cu); 0 on success, else -1 with a message in err
int nccl_unique_id(void* out128, char* err, size_t errn);
int nccl_init(const void* id128, int rank, int nranks, im_comm* comm, void** state, char* err, size_t errn);
void nccl_release(void* state);

}  // namespace im
