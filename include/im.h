/*
 * im.h -- C ABI of the B200-native (sm_100a) hot path of
 *   "Fast and Error-Adaptive Influence Maximization based on Count-Distinct
 *    Sketches" (arxiv 2105.04023; PAPER.md).
 *
 * Problem: find K seed vertices maximising the expected
 * number of vertices influenced under the Independent Cascade model.  Method:
 * hash-based fused sampling (Eq. 4-5), one 8-bit
 * Flajolet-Martin register per (vertex, simulation) (Eq. 1-3),
 * Simulate to the fixpoint (Alg. 2), greedy selection with
 * error-adaptive rebuilds (Alg. 1).  Readings of the paper
 * (R1..R21) are listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Return 0 on success, a negative IM_E* code on error; im_last_error() then
 *    returns a message.  On error, caller-owned outputs are left untouched.
 *  - Calls are synchronous: outputs are on the host when the call returns.
 *  - One global context, not thread-safe.  The library owns all device state
 *    from im_load_csr* until im_free() or the next im_load_csr*.
 *  - Host pointers are caller-owned and only read/written during the call.
 *  - All work runs on one CUDA stream (im_set_stream; before it: a library stream)
 *    on the current CUDA device, which must be sm_100 (B200); otherwise IM_ECUDA.
 *    There is no CPU fallback.
 */
#ifndef IM_H
#define IM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IM_OK 0
#define IM_EINVAL (-1) /* argument or graph validation failed */
#define IM_ESTATE (-2) /* wrong call order (e.g. im_estimate before im_build_sketches) */
#define IM_ENOMEM (-3) /* device or host allocation failed */
#define IM_ECUDA (-4)  /* CUDA error, or no sm_100 device */
#define IM_ECOMM (-5)  /* a collective of the communicator (im_set_comm / im_comm_nccl_init) failed */

#define IM_DTYPE_I32 0 /* allreduce element types */
#define IM_DTYPE_I64 1
#define IM_MAX_J_TOTAL 65536 /* simulations of one (possibly sharded) job */

/* One greedy step of Alg. 1. */
typedef struct {
    int32_t vertex;      /* s chosen at this step */
    int32_t pad;
    int64_t score;       /* sum_j max(M_S'[j], M_s[j]): integer numerator of Estimate(Merge(M_S', M_s)) */
    double e;            /* 2^(score/J) / 0.77351 (Eq. 2, line 12) */
    int64_t sigma_count; /* sum_j |R_G(S)[j]| after adding s */
    double sigma;        /* sigma_count / J (line 14) */
    double delta;        /* sigma - varsigma (line 15) */
    double err_l;        /* |(e - delta) / delta|, +inf when delta == 0 (line 16) */
    double err_g;        /* |(e - delta) / sigma| (line 17) */
    int32_t rebuilt;     /* 1: the else branch (rebuild) was decided (line 18 test false) */
    int32_t executed;    /* 1: the rebuild was executed (skipped after the last pick, reading R18) */
} im_step;

typedef struct {
    int32_t n;
    int32_t J;                 /* 0 before im_build_sketches */
    int64_t m;
    int32_t const_threshold;   /* 1 if every edge has the same w (one scalar integer threshold) */
    uint32_t threshold;        /* that threshold T: live iff (X_j xor h) < T (exactly Eq. 5 in double) */
    int32_t builds;            /* Simulate runs since load (first build + executed rebuilds) */
    int32_t last_build_sweeps; /* sweeps of the most recent Simulate */
    int64_t last_build_edges;  /* edges enumerated by the most recent Simulate */
    int64_t total_sweeps;      /* since the last im_select_seeds / im_build_sketches call began */
    int64_t total_edges;       /* edges enumerated by all sweeps in the same window */
    int32_t rebuilds;          /* rebuilds executed by the last im_select_seeds */
    int32_t bfs_levels;        /* BFS levels run by the last im_select_seeds */
    int64_t bfs_edges;         /* out-edges enumerated by those BFS levels */
    double prep_ms;            /* im_load_csr*: device edge prep (hash, threshold, transpose) */
    double last_build_ms;      /* most recent Simulate incl. register init */
    double last_select_ms;     /* last im_select_seeds, wall time inside the call */
    double sweep_kernel_ms;    /* summed sweep-kernel time in the window (CUDA events) */
    int64_t sweep_launches;    /* sweep kernel launches in the window */
    int64_t window_edges;      /* enumerated edges whose candidate window was non-empty after the change filter */
    int64_t kernel_launches;   /* all kernel launches in the window */
    int32_t argmax_full;       /* full argmax passes in the last selection (exact lazy argmax) */
    int32_t argmax_lazy;       /* candidate-list argmax evaluations in the last selection */
    int32_t sorted_rows;       /* 1 if adjacency rows are sorted by edge hash (constant threshold) */
    int32_t gather_sweeps;     /* sweeps in the window run as full gathers (direction-optimised) */
    double sweep_alg_bytes;    /* algorithmic bytes of all sweeps in the window */
    int32_t J_total;           /* simulations of the whole job (== J unless sharded) */
    int32_t j0;                /* global index of this context's first simulation (0 unless sharded) */
    double eps_c;              /* early-exit threshold the current sketches were built with (im_set_policy) */
} im_stats;

/*
 * Load a directed graph in CSR form and run the one-off edge preparation:
 *   h(u,v) = Murmur3_x86_32(LE32 u || LE32 v, seed 0) mod 2^31   (Eq. 4; R4)
 *   per-edge integer threshold T_e with  (X xor h)/h_max < w  <=>  (X xor h) < T_e  (Eq. 5; R1, R7)
 *   and the transpose (in-edges) used by the sweeps.
 * n        : number of vertices, n >= 1.
 * offsets  : HOST int32[n+1], offsets[0] = 0, non-decreasing; m = offsets[n].
 * targets  : HOST int32[m], out-neighbours, each in [0, n).  Self loops and
 *            duplicate edges are allowed and result-neutral (R19).
 * probs    : HOST float32[m], IC probability w_uv of each edge, finite, in [0, 1].
 * Resets all state.  IM_EINVAL on validation failure, IM_ENOMEM, IM_ECUDA.
 */
int im_load_csr(int32_t n, const int32_t *offsets, const int32_t *targets, const float *probs);

/* Same, with DEVICE pointers (already resident in HBM; read during the call only). m must equal offsets[n]. */
int im_load_csr_device(int32_t n, int64_t m, const int32_t *d_offsets, const int32_t *d_targets, const float *d_probs);

/*
 * The same load for the paper's constant-probability settings (w = 0.005 / 0.01 / 0.1 on every edge,
 * PAPER.md:457-462): one scalar w instead of an m-entry array, so the host-pointer call moves 4 bytes
 * per edge less over PCIe.  Results are identical to im_load_csr with probs[e] = w for every e.
 * w : finite, in [0, 1]; IM_EINVAL otherwise.  Other arguments, ownership and errors as im_load_csr.
 */
int im_load_csr_const(int32_t n, const int32_t *offsets, const int32_t *targets, float w);

/* Same, with DEVICE offsets / targets. */
int im_load_csr_const_device(int32_t n, int64_t m, const int32_t *d_offsets, const int32_t *d_targets, float w);

/*
 * Alg. 1 lines 2-6: salts from mt19937(low 32 bits of seed)
 * (R2, R3), registers M_v[j] = clz(Murmur3(v, seed_V) xor Murmur3(j, seed_J))
 * (R5, R6), then Simulate to the fixpoint with R_S = {} (eps_c = 0, R10, R11).
 * J       : number of simulations, a multiple of 32 in [32, 1024].
 * Requires a loaded graph (IM_ESTATE otherwise).
 */
int im_build_sketches(int32_t J, uint64_t seed);

/*
 * Simulation sharding.  The J simulations of
 * Alg. 1 are independent samples (simulation j only reads salt
 * X_j and the hash of j), so a job of J_total simulations can be split over ranks (one
 * process and one GPU each), rank r holding simulations [j0, j1).  Every rank loads the
 * same graph, installs a communicator (im_comm_nccl_init, or im_set_comm), then calls
 * im_build_sketches_shard with its range; im_estimate and im_select_seeds* are then
 * collective calls that every rank must make with the same arguments, and all ranks
 * return the same seeds, scores, step log and estimates as one unsharded context with
 * J = J_total would.  Per-rank outputs (im_get_registers / rows / reach) cover the
 * rank's own simulations, columns j - j0.  Builds and BFS never communicate.
 *
 * Exchanged per greedy step (Alg. 1 line 10, 12, 14):
 *   full argmax pass : reduce-scatter (SUM) of the packed per-vertex values
 *                      gain_local + (not fully visited locally) << 24 (n int32, each rank
 *                      receives its vertex slice of ceil(n / nranks)); a local argmax over
 *                      the slice; an all-reduce (MAX) of the 64-bit key (gain << 32 | ~v); an
 *                      all-reduce (SUM) of the gain histogram (4096 int32); all-gathers of the
 *                      candidate-list lengths (1 int32) and lists (<= slice int32 each)
 *   lazy argmax pass : all-reduce (SUM) of the packed values of the candidate list
 *   chosen vertex    : all-reduce (SUM) of its integer score (1 int64)
 *   sigma            : all-reduce (SUM) of the visited count (1 int64)
 * im_estimate exchanges the n int32 register sums (all-reduce SUM).
 *
 * J_total  : multiple of 32 in [32, IM_MAX_J_TOTAL]; salts X_0..X_{J_total-1} are drawn
 *            as in im_build_sketches(J_total, seed) and this context keeps [j0, j1).
 * j0, j1   : 0 <= j0 < j1 <= J_total, j1 - j0 a multiple of 32 in [32, 1024].
 * im_build_sketches(J, seed) == im_build_sketches_shard(J, seed, 0, J).
 */
int im_build_sketches_shard(int32_t J_total, uint64_t seed, int32_t j0, int32_t j1);

#define IM_OP_SUM 0 /* collective reduction operators */
#define IM_OP_MAX 1

/*
 * Communicator of a sharded job: three collectives on DEVICE buffers of the library's device.
 *   allreduce(buf, count, dtype, op)      in place, op IM_OP_SUM / IM_OP_MAX
 *   reduce_scatter(send, recv, recvcount, dtype)   SUM; send holds nranks * recvcount elements,
 *                                         rank r receives elements [r * recvcount, (r+1) * recvcount)
 *   allgather(send, recv, sendcount, dtype)        recv[r * sendcount + i] = send of rank r [i]
 * dtype: IM_DTYPE_I32 / IM_DTYPE_I64.  stream: the library's cudaStream_t.  Each returns 0 on
 * success (non-zero -> IM_ECOMM).  stream_ordered = 1: the operation is enqueued on `stream`
 * (NCCL semantics); 0: the library synchronises its stream first and the call returns with the
 * result in place (host-staged transports, e.g. gloo).  1 <= nranks < 256 (the packed argmax value
 * counts in-pool ranks in 8 bits), 0 <= rank < nranks.  The struct is copied.
 */
typedef struct {
    int32_t rank, nranks;
    int32_t stream_ordered;
    int32_t pad;
    int (*allreduce)(void *buf, int64_t count, int32_t dtype, int32_t op, void *stream, void *user);
    int (*reduce_scatter)(const void *send, void *recv, int64_t recvcount, int32_t dtype, void *stream, void *user);
    int (*allgather)(const void *send, void *recv, int64_t sendcount, int32_t dtype, void *stream, void *user);
    void *user;
} im_comm;

/* Install a caller-implemented communicator (copied); NULL removes it (unsharded behaviour).  A sharded
 * context must have one installed during im_estimate / im_select_seeds*.  IM_EINVAL on bad fields. */
int im_set_comm(const im_comm *comm);

/*
 * The library's own NCCL communicator (NCCL over NVLink / NVSwitch; libnccl.so.2 is loaded at the first
 * call, no build-time dependency).  im_comm_nccl_unique_id writes the 128-byte ncclUniqueId (rank 0
 * calls it and shares the bytes with the other ranks, e.g. over torch.distributed); every rank then
 * calls im_comm_nccl_init with the same id on its own device.  The collectives are enqueued on the
 * library's stream (stream_ordered), with no host round trip and no Python in the exchange.
 * IM_ECOMM when NCCL is unavailable or fails; im_set_comm(NULL) / im_free release it.
 */
int im_comm_nccl_unique_id(void *out_id128);
int im_comm_nccl_init(const void *id128, int32_t rank, int32_t nranks);

/* e_v = 2^{mean_j M_v[j]} / 0.77351 for every vertex (Eq. 2, R8).  out: HOST double[n]. */
int im_estimate(double *out);
/* Same into DEVICE memory: d_out double[n]. */
int im_estimate_device(double *d_out);

/*
 * Alg. 1 lines 7-30 with eps_l = eps_g = err_threshold (R17): K greedy steps,
 * each an argmax of Estimate(Merge(M_S', M_v)) (lowest id on ties, R14), a
 * multi-simulation BFS for R_G(S) and sigma over the same samples (R13), the
 * error test and either M_S' merge or a rebuild on the residual graph.
 * Always starts from S = {}, varsigma = 0, M_S' = 0 and freshly built sketches.
 * K                : 0 <= K <= n (K = 0 writes nothing).
 * err_threshold    : >= 0, not NaN; +inf = never rebuild; 0 = always rebuild.
 * out_seeds        : HOST int32[K]; out_scores: HOST double[K], sigma after k+1 seeds (R21).
 */
int im_select_seeds(int32_t K, double err_threshold, int32_t *out_seeds, double *out_scores);
/* Same with separate local / global thresholds. */
int im_select_seeds_ex(int32_t K, double eps_l, double eps_g, int32_t *out_seeds, double *out_scores);

/*
 * Selection policy.  Persists across calls and loads; the default
 * (NaN, NaN, 0) is the behaviour described above.
 * eps_l, eps_g : local / global error thresholds of the keep test (Alg. 1 line 18, PAPER.md:288-290,
 *                413) used by im_select_seeds instead of its err_threshold; NaN = use err_threshold.
 *                Must be >= 0 or NaN.  im_select_seeds_ex always uses its own arguments.
 * eps_c        : early-exit threshold of Simulate (Alg. 2 line 3): sweeps run while
 *                |L|/|V| > eps_c, L = vertices changed by the last sweep.  0 = to the fixpoint
 *                (reading R11).  eps_c > 0 switches to synchronous sweeps (every sweep reads the
 *                registers as they were when it started, Fig. 5, reading R22; +n*J bytes of device
 *                memory) so the early-exit state is well defined; it applies to im_build_sketches*
 *                and to every rebuild, and im_select_seeds* rebuilds first when the held sketches
 *                were built with another eps_c.  In [0, 1]; 1 runs no sweep (registers = init).
 * IM_EINVAL on out-of-range values (policy unchanged).
 */
int im_set_policy(double eps_l, double eps_g, double eps_c);

/*
 * Independent Monte-Carlo influence of a seed sequence: the paper scores every
 * method with a sample-then-diffuse oracle on fresh randomness.  Sample r of
 * edge (u,v) is live iff its counter-based SplitMix64 draw (reading R23) / h_max < w_uv,
 * independent of the sketch salts; samples r0 .. r0+R-1 are evaluated (any range: ranks can split
 * the samples and add the counts).
 * K          : 0 <= K <= n; seeds: HOST int32[K] in [0, n) (repeats allowed).
 * seed       : evaluation seed (use one unrelated to the sketch seed).
 * r0, R      : r0 >= 0; R a positive multiple of 32 (run in batches of up to 512 samples).
 * out_counts : HOST int64[K]; out_counts[k] = sum_r |R_{G_r}({seeds_0..seeds_k})|; the expected
 *              influence estimate of the first k+1 seeds is out_counts[k] / R.
 * Needs a loaded graph only (no sketches).  IM_EINVAL / IM_ESTATE / IM_ENOMEM / IM_ECUDA.
 */
int im_evaluate(int32_t K, const int32_t *seeds, uint64_t seed, int64_t r0, int64_t R, int64_t *out_counts);

/* ---- test / diagnostic extras ---- */
/* registers after the most recent Simulate, HOST uint8[n*J] row-major, simulation order j = 0..J-1 */
int im_get_registers(uint8_t *out);
/* the same for nrows listed vertices: out uint8[nrows*J] */
int im_get_register_rows(int64_t nrows, const int32_t *rows, uint8_t *out);
/* R_G(S) after the last selection: HOST uint32[n*(J/32)], bit j%32 of word j/32 of row v */
int im_get_reach(uint32_t *out);
/* step log of the last selection: HOST im_step[cap]; returns the number of steps written (>= 0) */
int im_get_step_log(im_step *out, int32_t cap);
int im_get_stats(im_stats *out);
/* run all device work on this cudaStream_t from now on.  NULL = CUDA's stream 0 (the legacy default
 * stream; torch's default stream has handle 0), so the library's work is ordered after the caller's
 * kernels on it.  Before the first call the library uses a stream of its own. */
int im_set_stream(void *cuda_stream);
/* number of kernel launches issued by the library since load (diagnostic) */
int64_t im_kernel_launch_count(void);
void im_free(void);
const char *im_last_error(void);
/* ABI version (major*100 + minor): 101 adds sharding (im_build_sketches_shard), 102 im_set_policy,
 * 103 replaces the allreduce hook by the communicator (im_set_comm, im_comm_nccl_*) */
int32_t im_version(void);

#ifdef __cplusplus
}
#endif
#endif /* IM_H */
