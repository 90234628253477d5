/*
 * gcp.h -- C ABI of the B200-native stochastic GCP-Adam hot path
 * (arXiv 2605.20353, "parallel GCP-Adam / GCP-FedAdam"; /root/reference/PAPER.md
 * is cited as P:line with the section / equation / algorithm named).
 *
 * One gcp_ctx per rank == per GPU.  Implemented by libgcp.so
 * (the .cu sources under paper_2605_20353_b200/csrc/, sm_100a only).  No torch types cross this
 * boundary: host pointers are plain C arrays, the CUDA stream is an opaque
 * cudaStream_t, the NCCL unique id is 128 opaque bytes.
 *
 * Conventions that hold for every entry point:
 *  - Returns gcp_status; no C++ exception crosses the ABI.  On error
 *    gcp_last_error() returns a thread-local message.
 *  - Argument errors (GCP_E_ARG / GCP_E_RANGE / GCP_E_DUP / GCP_E_NO_*) are
 *    detected before any state changes (no partial mutation) -- except the
 *    data errors gcp_tensor_create finds while ingesting (duplicates,
 *    out-of-block coordinates, non-finite values), which leave the context
 *    without a tensor (the previous one is freed first).
 *  - CUDA and NCCL failures, and a zero sample hitting the rejection cap, are
 *    sticky: the context enters an error state and every later call returns
 *    GCP_E_STATE (gcp_destroy still works).  A rejection-cap or CUDA fault in
 *    an asynchronous kernel is reported by the next call that synchronises.
 *  - Host pointers are borrowed for the duration of the call and copied; the
 *    library never keeps one.  All device memory (COO records, hash set,
 *    factors, gradients, moments, checkpoints, partials) is owned by the
 *    context and freed by gcp_destroy.
 *  - Calls enqueue on the context stream and return without blocking, except:
 *    getters (*_get, *_export, gcp_tensor_info, gcp_tensor_contains),
 *    gcp_loss_estimate, gcp_loss_grad with a non-NULL sampled_loss_out,
 *    gcp_tensor_create, gcp_fit*, and every error path.
 *  - Coordinates are 0-based GLOBAL indices; the paper's 1-based ranges
 *     are shifted.
 */
#ifndef GCP_H
#define GCP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef struct gcp_ctx gcp_ctx;

typedef enum {
    GCP_OK = 0,
    GCP_E_ARG = 1,          /* bad argument, non-finite value, p+q = 0, ... */
    GCP_E_RANGE = 2,        /* coordinate outside dims / outside this rank's block; bad mode k */
    GCP_E_DUP = 3,          /* duplicate coordinates in the input tensor */
    GCP_E_NO_NONZEROS = 4,  /* global N = 0 but nonzero samples requested */
    GCP_E_NO_ZEROS = 5,     /* global M = N but (stratified) zero samples requested */
    GCP_E_REJECT_CAP = 6,   /* a zero slot was rejected 1000 times (reading R5) */
    GCP_E_STATE = 7,        /* call order violated, or the context is in a sticky error state */
    GCP_E_OOM = 8,          /* device allocation failed */
    GCP_E_CUDA = 9,         /* CUDA runtime error (sticky) */
    GCP_E_NCCL = 10         /* NCCL error (sticky) */
} gcp_status;

/* Loss f(x, m) and its lower bound l (reading R3; P:282-284 leaves f open). */
typedef enum {
    GCP_LOSS_GAUSSIAN = 0,        /* (x-m)^2,                 l = -inf */
    GCP_LOSS_POISSON = 1,         /* m - x log(m + 1e-10),    l = 0    */
    GCP_LOSS_BERNOULLI_LOGIT = 2  /* log(1+e^m) - x m,        l = -inf */
} gcp_loss;

/* Sampling scheme (P:513-537 stratified; P:561-573 semi-stratified). */
typedef enum { GCP_STRATIFIED = 0, GCP_SEMI_STRATIFIED = 1 } gcp_strategy;

/* Zero-candidate membership structure: a hash set of block keys
 * (O(1) probe, the default) or the sorted key array searched in O(log N)
 * (row f4; about 2.6x less memory). */
typedef enum { GCP_MEMBER_HASH = 0, GCP_MEMBER_SORTED = 1 } gcp_membership;

/* Arithmetic type of factors, gradients, moments (reading R10). */
typedef enum { GCP_FP32 = 0, GCP_FP64 = 1 } gcp_precision;

/* Multi-GPU scheme (P:642-749 sync, Alg. 2; P:435-450 LocalSGD, Alg. 3;
 * P:790-824 FedAdam, Alg. 4). */
typedef enum {
    GCP_DIST_SYNC = 0,            /* "all-reduce" factor layout: block rows replicated per slice group */
    GCP_DIST_ASYNC_AVG = 1,       /* LocalSGD averaging every tau iterations (Alg. 3) */
    GCP_DIST_ASYNC_FEDADAM = 2,   /* FedAdam server step every tau iterations (Alg. 4) */
    GCP_DIST_SYNC_TWO_SIDED = 3   /* "two-sided" layout: rows partitioned, per-iteration import/export;
                                     gcp_model_get, gcp_model_set and gcp_loss_estimate are collective in this
                                     mode (every rank calls them in the same order).  Within one
                                     NVLink domain of <= 8 ranks the gradient kernel reaches the owners' rows by
                                     peer access (environment GCP_TWOSIDED_NVL=1: import/export kernels over
                                     NVLink windows; =0: NCCL send/recv) */
} gcp_dist_mode;

/* Alg. 1 hyper-parameters.  lower: NaN selects the loss default. */
typedef struct { double rate, beta1, beta2, eps, lower; } gcp_adam_params;

/* gcp_fit parameters.  Sample counts are GLOBAL totals per iteration, split
 * over ranks by reading R13.  tau (iterations, reading R18) and meta_rate are
 * used by the async modes only.  Defaults (Table 2): rate 1e-3,
 * decay 0.1, beta (0.9, 0.999), eps 1e-8; epochs of 100 iterations
 * (P:868-869); 3 failures. */
typedef struct {
    int epochs, iters_per_epoch, max_fails;
    double decay;
    int64_t s_nz, s_z;          /* gradient samples per iteration (p, q) */
    int64_t f_nz, f_z;          /* loss-estimate samples (fixed set, reading R19) */
    gcp_strategy strategy;
    gcp_loss loss;
    uint64_t seed;              /* gradient-sample seed */
    uint64_t fseed;             /* f-sample seed */
    gcp_adam_params adam;
    int64_t tau;
    double meta_rate;
} gcp_fit_params;

/* Called once per epoch by gcp_fit (trace CSV epoch,iter,est_loss,rate,elapsed_s). */
typedef void (*gcp_trace_fn)(void* user, int epoch, int64_t iter, double est_loss,
                             double rate, double elapsed_s);

/* ---- context ------------------------------------------------------------ */

/* Create a context on CUDA device `cuda_device`, enqueueing on `cuda_stream`
 * (a cudaStream_t; NULL = the legacy default stream).  prec selects fp32 or
 * fp64 arithmetic for every later call.  *out is NULL on failure. */
gcp_status gcp_create(gcp_ctx** out, int cuda_device, void* cuda_stream, gcp_precision prec);

/* Free all device memory and NCCL communicators of the context. NULL is a no-op. */
void gcp_destroy(gcp_ctx* ctx);

/* Thread-local message describing the last error of this thread ("" if none). */
const char* gcp_last_error(void);

/* ---- distribution (§3.2) ------------------------------------- */

/* Medium-grained grid: over all ordered d-tuples (N_1..N_d) with
 * prod N_k = P, minimise the replicated factor storage sum_k I_k * P/N_k; ties
 * go to the lexicographically smallest tuple (reading R14).  grid_out: d ints.
 * lo_out/hi_out (nullable): P*d int64 block bounds [lo, hi) per rank, rank
 * row-major with b_1 slowest, c_k = ceil(I_k/N_k).  Pure host function. */
gcp_status gcp_grid_plan(int P, int d, const int64_t* dims, int* grid_out,
                         int64_t* lo_out, int64_t* hi_out);

/* Write a fresh 128-byte ncclUniqueId into out128 (rank 0 calls this and
 * broadcasts the bytes, e.g. with torch.distributed). */
gcp_status gcp_nccl_unique_id(void* out128);

/* Join an nranks-rank job as `rank` (one rank per GPU).  grid: d
 * ints with product nranks, or NULL = gcp_grid_plan's argmin, resolved at
 * gcp_tensor_create.  Creates the world communicator now and one slice
 * communicator per mode (ranks sharing b_k) at gcp_tensor_create.
 * nranks == 1 is allowed and needs no id (id may be NULL).  Must precede
 * gcp_tensor_create.  Collective over all ranks. */
gcp_status gcp_dist_init(gcp_ctx* ctx, int nranks, int rank, const void* nccl_unique_id,
                         const int* grid, int d, gcp_dist_mode mode);

/* Async schemes: averaging / server-step period tau (iterations, reading R18)
 * and the server Adam parameters of Alg. 4 (rate = meta-rate; NULL keeps the
 * client parameters).  gcp_fit_begin sets these from gcp_fit_params. */
gcp_status gcp_dist_set_async(gcp_ctx* ctx, int64_t tau, const gcp_adam_params* server);

/* ---- tensor (row a0) -------------------------------- */

/* Ingest this rank's nonzeros: 2 <= d <= 6 modes of global sizes dims[d] (each in
 * [1, 2^32-1]); subs = nnz*d int64 GLOBAL coordinates, row-major; vals = nnz
 * doubles (finite; 0.0 allowed, reading R26).  Both borrowed for the call:
 * host memory (pageable or pinned) or device memory of this context's GPU
 * (copied in chunks with cudaMemcpyDefault, i.e. any UVA pointer).
 * For nranks > 1 every nonzero must lie in this rank's block.  The device sorts
 * the nonzeros lexicographically (i_1 most significant, reading R15), rejects
 * duplicates, and builds the hash set of block-linearised keys (u64, or u128
 * when the block has >= 2^64 entries).  Replaces any previous tensor and drops
 * the model (both freed before the ingest; on failure the context has no
 * tensor).  GCP_E_ARG if prod I_k does not fit in 128 bits.
 * Blocks; collective for nranks > 1 (global N and M checks). */
gcp_status gcp_tensor_create(gcp_ctx* ctx, int d, const int64_t* dims, int64_t nnz,
                             const int64_t* subs, const double* vals);

/* Select the zero-test structure the NEXT gcp_tensor_create builds (default
 * GCP_MEMBER_HASH).  Sampling results are identical for both (membership is a
 * pure set predicate).  No device work. */
gcp_status gcp_set_membership(gcp_ctx* ctx, gcp_membership m);

/* Local block summary: nnz_local, block bounds lo/hi (d each, nullable),
 * M_local = prod (hi_k - lo_k) as double, global N.  Blocks. */
gcp_status gcp_tensor_info(gcp_ctx* ctx, int64_t* nnz_local, int64_t* lo, int64_t* hi,
                           double* M_local, int64_t* nnz_global);

/* Test helper: canonical (sorted) nonzeros [first, first+count) as global
 * coordinates (count*d int64) and values (count doubles).  Blocks. */
gcp_status gcp_tensor_export_sorted(gcp_ctx* ctx, int64_t first, int64_t count,
                                    int64_t* subs_out, double* vals_out);

/* Test helper: membership of n global coordinate tuples (n*d int64, must be in
 * the block) in the device hash set; out[n] = 0/1.  Blocks. */
gcp_status gcp_tensor_contains(gcp_ctx* ctx, int64_t n, const int64_t* coords, int8_t* out);

/* ---- model (Eq. CP, P:257-263 with lambda) -------------------------- */

/* Allocate rank-R factors (1 <= R <= 128 in fp32, 64 in fp64; rows padded to
 * a multiple of 4 columns) for this rank's block rows, moments B = C = 0 and
 * the gradient G = 0 (one contiguous array each), lambda = 1, and
 * fill A^(k) ~ U[0,1) by Philox (reading R12; identical on every rank and for
 * every grid).  Resets the Adam step t and the iteration counter to 0.
 * Sync nranks > 1 with the fused NVLink exchange: A, G and a second G live in
 * NCCL symmetric windows; on replacement, up to min(4 GiB, 1/32 of device
 * memory) of the previous model's registered windows stay allocated (outside
 * the allocation pool) for a next model of the same padded size, until that
 * model or gcp_destroy. */
gcp_status gcp_model_init(gcp_ctx* ctx, int R, uint64_t seed);

/* Overwrite factor k's block rows (host, (hi_k-lo_k) x R doubles, row-major;
 * rounded to the context precision) and, if lambda != NULL, lambda[R]. */
gcp_status gcp_model_set(gcp_ctx* ctx, int k, const double* rows, const double* lambda);

/* Read factor k's block rows into rows_out ((hi_k-lo_k) x R doubles). Blocks. */
gcp_status gcp_model_get(gcp_ctx* ctx, int k, double* rows_out);

/* ---- sampling and gradient (rows a1-a5) -------------------------- */

/* Bind the sampler: strategy, GLOBAL per-iteration counts s_nz (p) and s_z
 * (q), seed.  No device work.  Errors: s_nz, s_z < 0 or both 0 (E_ARG); global
 * N = 0 with s_nz > 0 (E_NO_NONZEROS); global M = N with stratified s_z > 0
 * (E_NO_ZEROS). */
gcp_status gcp_sample(gcp_ctx* ctx, gcp_strategy strategy, int64_t s_nz, int64_t s_z, uint64_t seed);

/* Test helper: the entries of Y~ the current iteration would draw for
 * stratum 0 (nonzero) or 1 (zero), local slots [first, first+count):
 * subs_out count*d global coords, j_out canonical nonzero index (-1 for
 * zeros), w_out fp64 weight (N_w/p_w or (M_w-N_w)/q_w), attempts_out.  All
 * outputs nullable except subs_out.  Blocks. */
gcp_status gcp_sample_export(gcp_ctx* ctx, int stratum, int64_t first, int64_t count,
                             int64_t* subs_out, int64_t* j_out, double* w_out,
                             int32_t* attempts_out);

/* Fused Sampling-MTTKRP: for every local sample slot draw the
 * index (Philox, iteration counter = current it), fetch the record or probe
 * and reject (stratified) the zero candidate, evaluate m, y = w df/dm, and
 * scatter-add y lambda_r prod_{j!=k} a_j[r] into G^(k) for every k.  G is the
 * gradient of the SUM objective.  Adds into G (zeroed by Adam).  If
 * sampled_loss_out != NULL, also returns sum_s w f(x, m) over this rank's
 * samples (blocks).  Requires model + sampler. */
gcp_status gcp_loss_grad(gcp_ctx* ctx, gcp_loss loss, double* sampled_loss_out);

/* Read G^(k)'s block rows ((hi_k-lo_k) x R doubles).  With nranks > 1 in sync
 * mode this is the LOCAL (pre-exchange) gradient.  In the two-sided layout with
 * peer access every rank adds into the owner's rows, so the rows this rank owns
 * hold the slice group's summed gradient once every member's gcp_loss_grad has
 * completed (the caller's barrier); other rows read as zero.  Blocks. */
gcp_status gcp_grad_get(gcp_ctx* ctx, int k, double* out);

/* ---- Adam (rows a6-a8; Alg. 1, Alg. 2-3) -------------------------- */

/* t += 1; sync nranks > 1: reduce-scatter G^(k) over each slice group
 * (Alg. 2 "Allreduce(G)", sum, reading R21); Alg. 1 on the owned rows with
 * eps inside the sqrt (reading R8) and the comparison clamp (R9); G <- 0;
 * all-gather the updated rows.  Async modes: Alg. 1 on the local replica only.
 * (In async modes gcp_loss_grad first runs the averaging of Alg. 3 or the
 * server step of Alg. 4 when the 1-based iteration number it+1 is divisible
 * by tau.)  Increments the iteration counter it.  Requires a
 * gradient. */
gcp_status gcp_adam_step(gcp_ctx* ctx, const gcp_adam_params* p);

/* ---- loss estimate (row a9) --------------------------------------------- */

/* Stratified estimate sum over ranks of (N_w/f_nz,w) sum f(x,m) +
 * ((M_w-N_w)/f_z,w) sum f(0,m) over the f-sample set of `seed` (reading R19;
 * Philox kinds 2/3, it = 0xFFFFFFFF).  Deterministic fp64 reduction.  Blocks;
 * collective for nranks > 1. */
gcp_status gcp_loss_estimate(gcp_ctx* ctx, gcp_loss loss, int64_t f_nz, int64_t f_z,
                             uint64_t seed, double* out);

/* ---- fit (epoch loop with annealing, reading R20) ------------------------ */

/* gcp_fit = gcp_fit_begin + gcp_fit_epoch until done.  begin: binds the
 * sampler, evaluates F^_0 on the current model, checkpoints (A, B, C, t).
 * epoch: iters_per_epoch x [gradient, exchange, Adam], then F^_e; accept
 * (checkpoint) if F^_e < best, else restore, rate *= decay, fails += 1;
 * *done_out = 1 when fails reached max_fails or the epoch budget is spent.
 * On a non-legacy stream the epoch's iterations are captured once per
 * schedule and replayed as one CUDA graph (not while profiling, for the
 * NCCL send/recv two-sided path or FedAdam; environment GCP_GRAPHS=0 disables it); results
 * are the same either way.  All three block; collective for nranks > 1. */
gcp_status gcp_fit_begin(gcp_ctx* ctx, const gcp_fit_params* p, double* initial_est);
gcp_status gcp_fit_epoch(gcp_ctx* ctx, double* est_out, int* accepted_out, int* done_out);
gcp_status gcp_fit(gcp_ctx* ctx, const gcp_fit_params* p, gcp_trace_fn trace, void* user,
                   double* final_est_loss);

/* ---- instrumentation ----------------------------------------------------- */

/* Layout choices the context made (all nullable; 0 without a model / tensor):
 * A/G rows interleaved in one 128-B line (factors spill L2), gradient slots
 * visited in mode-1 order (mode-1 rows spill L2 and the iteration's order array
 * fits L2; kernels.cu), L2 Bloom filter
 * in front of the zero test.  For tests and benchmarks.  Does not block. */
gcp_status gcp_layout(gcp_ctx* ctx, int* ag_interleaved, int* slot_order, int* filter);

/* Test helper for the index map of reading R11 at N >= 2^32: the
 * canonical nonzero index j of nonzero slots [first, first+count) (first+count
 * <= 2^32) of iteration word `it`, rank word `rank`, kind 0, computed by the
 * device draw path of the sample kernels with a pretend local nonzero count N
 * (every draw reads record 0, so no tensor of N nonzeros is needed; needs a
 * tensor with >= 1 nonzero).  j_out: count int64 (host).  Blocks. */
gcp_status gcp_debug_nonzero_j(gcp_ctx* ctx, uint64_t seed, uint32_t rank, uint32_t it, int64_t N,
                               int64_t first, int64_t count, int64_t* j_out);

/* Test helper for reading R11's generator: for n inputs ctr_key[6i..6i+5] =
 * (c0, c1, c2, c3, k0, k1), out[8i..8i+3] = the sampler's device
 * Philox4x32-10 and out[8i+4..8i+7] = curand's curand_Philox4x32_10 on the
 * same counter and key (host arrays).  Blocks. */
gcp_status gcp_debug_philox(gcp_ctx* ctx, int64_t n, const uint32_t* ctr_key, uint32_t* out);

/* Counters: it (Philox iteration word), t (Adam steps), kernel launches made
 * by this library since creation (all nullable).  Does not block. */
gcp_status gcp_counters(gcp_ctx* ctx, uint32_t* it, int64_t* t, int64_t* launches);

/* Which sync exchange the model runs (a6-a8), for
 * benchmarks and tests; both nullable, set after gcp_model_init:
 *   *fused_out    = 1 when reduce-scatter + Adam + all-gather is the single
 *                   NVLink kernel over symmetric windows (else NCCL calls);
 *   *multimem_out = 1 when that kernel sums and broadcasts the modes whose
 *                   slice group spans all ranks through NVLS multicast
 *                   (reduction inside the NVSwitch; fp32 only; environment
 *                   GCP_MULTIMEM=1 forces it, 0 disables it, default from
 *                   8 ranks up).
 * Does not block. */
gcp_status gcp_dist_features(gcp_ctx* ctx, int* fused_out, int* multimem_out);

/* Enable (1) / disable (0) CUDA-event timing of every library kernel launch on
 * the context stream (the events bracket each launch; adds no sync). */
gcp_status gcp_profile_enable(gcp_ctx* ctx, int on);

/* Accumulated device time (ms) and launch count of kernel class `which`
 * (0 fused gradient K2, 1 Adam K3, 2 loss estimate, 3 collectives,
 * 4 other); pending events are resolved (blocks).  reset != 0 zeroes it. */
gcp_status gcp_profile_get(gcp_ctx* ctx, int which, double* ms, int64_t* launches, int reset);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* GCP_H */
