// gcp_internal.h -- context layout and host helpers shared by the csrc/*.cu
// translation units of libgcp.so.  Not part of the ABI (see include/gcp.h).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/gcp.h"

// Bounds-checked build (python paper_2605_20353_b200/build.py --variant bounds
// -DGCP_BOUNDS_CHECK; loaded with GCP_LIB=libgcp_bounds.so): device indices of
// the hot path are checked and the first violations printed as "GCP-BOUNDS".
// compute-sanitizer is closed on this GPU pool, so this is the memory-safety
// check (tools/sanitize_c1.py, profiles/r02_bounds.sh).
#ifdef GCP_BOUNDS_CHECK
#define GCP_CHECK(cond, what, x, y)                                                                  \
    do {                                                                                           \
        if (!(cond)) printf("GCP-BOUNDS %s: %lld %lld\n", what, (long long)(x), (long long)(y));   \
    } while (0)
#else
#define GCP_CHECK(cond, what, x, y) \
    do {                            \
    } while (0)
#endif

namespace gcp {

constexpr int kMaxModes = 8;          // array capacity
constexpr int kMaxD = 6;              // d <= 6 on the device path (record = value + d coords <= 32 B)
constexpr int kRejectCap = 1000;      // reading R5
#ifndef GCP_BLOCK
#define GCP_BLOCK 256
#endif
#ifndef GCP_MINB
#define GCP_MINB 2
#endif
#ifndef GCP_RBREG
#define GCP_RBREG 10
#endif
#ifndef GCP_SMALL_MINB
#define GCP_SMALL_MINB 3
#endif
#ifndef GCP_SMALL_RBREG
#define GCP_SMALL_RBREG 8
#endif
#ifndef GCP_PEER_MINB
#define GCP_PEER_MINB 0   // > 0: the peer-access K2's own CTAs/SM and row budget (GCP_PEER_RBREG)
#endif
#ifndef GCP_PEER_RBREG
#define GCP_PEER_RBREG 8
#endif
constexpr int kBlock = GCP_BLOCK;          // threads per CTA of the sample kernels
constexpr int kSampleMinBlocks = GCP_MINB; // resident CTAs per SM the register budget must allow
constexpr int kRowRegBudget = GCP_RBREG;   // 16-B row vectors per lane kept in flight per batch
constexpr int kSmallMinBlocks = GCP_SMALL_MINB;   // the same two for small row footprints (D * NV <= 3)
constexpr int kSmallRowRegBudget = GCP_SMALL_RBREG;
constexpr double kHashLoad = 0.5;     // target hash-set load factor

enum Kind : uint32_t { KIND_GRAD_NZ = 0, KIND_GRAD_Z = 1, KIND_F_NZ = 2, KIND_F_Z = 3, KIND_INIT = 4 };
enum Prof { PROF_GRAD = 0, PROF_ADAM = 1, PROF_LOSS = 2, PROF_COMM = 3, PROF_OTHER = 4, PROF_N = 5 };

// Everything the sample kernels (K2 gradient / loss mode, export) need.
struct SampleArgs {
    const uint32_t* rec;      // AoS records: [value (1 or 2 words)][d local coords u32][pad]
    int rec_words;            // stride in 32-bit words (4 or 8)
    int val_words;            // 1 (fp32) or 2 (fp64)
    int64_t N;                // local nonzeros
    const uint64_t* hash;     // open-addressing set (u64 keys, or u128 as lo,hi pairs)
    uint64_t hash_mask;       // slots - 1 (power of two)
    int key128;               // 1: 128-bit keys
    uint32_t bdim[kMaxModes]; // block extent per mode (hi_k - lo_k)
    int64_t p, q;             // local nonzero / zero slots in this launch
    uint64_t seed;
    uint32_t rank, it, kind_nz, kind_z;
    int stratified;           // 0: semi-stratified (no membership test)
    int member_sorted;        // 1: binary search of `keys` instead of the hash set (row f4)
    const uint64_t* keys;     // sorted block keys (u64, or (lo,hi) pairs for u128)
    unsigned long long* err_slot;  // min zero slot that hit the rejection cap (ULLONG_MAX = none)
    const uint32_t* it_dev;   // non-null inside a captured epoch graph: it = *it_dev + it (offset)
    const uint64_t* filter;   // blocked Bloom filter of the block's keys (4 u64 per 32-B sector), or null
    uint64_t filter_mask;     // sectors - 1 (power of two)
    const uint32_t* order;    // gradient launches: slot processing order (null = slot order), see slot_order
    int l2_first;             // 1: record and hash-bucket reads (used once) carry an L2 evict_first policy
};

// Epoch-graph replay state: the values of rate, t and it at the start of the
// replay, uploaded once per replay.  Each captured kernel carries its own
// iteration offset as a launch argument (t = t0 + off, it = it0 + off), so no
// kernel has to advance a device counter.
struct DevStep {
    double rate, beta1, beta2;
    long long t;
    uint32_t it, pad;
};

struct ModelArgs {
    const void* A;            // factor array (T), mode-major, rows padded to R_pad
    void* G;                  // gradient array, same layout
    const void* lambda;       // R_pad values (T), zero padded
    int64_t off[kMaxModes];   // element offset of mode k's first row in the A (and G) buffer
    int R_pad;
    int row_stride;           // elements between consecutive rows (R_pad, or 2 R_pad when A/G interleave)
    // two-sided over NVLink, peer access (twosided_nvl.cu): rows of mode k are
    // owned by slice member r / shard[k] (LSA rank mem[k][.]); K2 gathers them
    // from the owner's A window and scatter-adds into the owner's G window.
    // peerA == null: every row is local.
    const void* const* peerA; // [LSA ranks] window bases of A
    void* const* peerG;       // [LSA ranks] window bases of the current G parity
    int64_t shard[kMaxModes];
    int nmem[kMaxModes];
    int mem[kMaxModes][8];
};

// The slot-order histogram pass of the NEXT iteration, carried by the gradient
// K2 of this one (kernels.cu, launch_slot_order): n = 0 means none.
struct OrdHistArgs {
    SampleArgs sa;            // the next iteration's sampler arguments
    const uint16_t* lut;      // per-tensor lookup: bucket of nonzero index j = lut[j >> lut_shift]
    int lut_shift;
    uint32_t* keys;           // (tile << bits) | bucket per slot (out)
    int tile_shift;           // slots per tile = 2^tile_shift (tiles order independently)
    uint32_t* ranks;          // rank of the slot inside its bucket (out)
    uint32_t* totals;         // bucket totals (global atomicAdd)
    int bits;                 // log2 bucket count
    int64_t n;                // slots (p + q)
};

// The scatter pass of the next iteration's slot order, carried by the Adam
// launch of this one: order[cursor[key] + rank] = slot.  n = 0 means none.
struct OrdScatterArgs {
    const uint32_t* keys;
    const uint32_t* ranks;
    const uint32_t* cursor;
    uint32_t* order;
    int64_t n;
    int ratio;                // one slot per `ratio` Adam vectors of a thread
};

struct Segment {              // contiguous ranges of the coefficient arrays (Adam)
    int64_t start[2 * kMaxModes];
    int64_t len[2 * kMaxModes];
    int n;
};

}  // namespace gcp

struct gcp_ctx {
    int dev = 0;
    cudaStream_t stream = nullptr;
    gcp_precision prec = GCP_FP32;
    int sm_count = 148;
    int64_t l2_bytes = 126 << 20;
    int tsize = 4;                      // sizeof(T)
    // ---- error state
    gcp_status sticky = GCP_OK;
    // ---- distribution
    int P = 1, rank = 0;
    gcp_dist_mode mode = GCP_DIST_SYNC;
    int grid[gcp::kMaxModes] = {0};
    bool grid_given = false;
    bool dist_ready = false;
    ncclComm_t world = nullptr;
    ncclComm_t slice[gcp::kMaxModes] = {nullptr};
    int slice_size[gcp::kMaxModes] = {0}, slice_rank[gcp::kMaxModes] = {0};
    int slice_d = 0, slice_grid[gcp::kMaxModes] = {0};   // geometry the slice comms were split for
    bool ar_mode[gcp::kMaxModes] = {false};   // sync exchange of mode k: all-reduce (else RS/AG)
    // fused NVLink exchange (fused.cu): symmetric windows + device communicator
    bool fused = false, devcomm_ready = false;
    bool multimem = false;                        // NVLS multicast usable on the LSA team
    int fused_ctas = 0;                           // max grid of the fused exchange (one LSA barrier each)
    int fused_grid = 0;                           // grid of the last launch
    void* ftrace = nullptr;                       // GCP_FUSED_TRACE diagnostics
    double ftrace_acc[16] = {0};
    int64_t ftrace_n = 0;
    ncclDevComm devcomm{};
    ncclWindow_t winA = nullptr, winG[2] = {nullptr, nullptr};
    void* d_G2 = nullptr;                         // second G buffer (iteration parity)
    void* d_bm = nullptr;                         // two-sided over NVLink: touched-row bits (2 parities)
    ncclWindow_t winBM = nullptr;
    bool tsn_peer = false;                        // two-sided over NVLink by peer access (no import / export)
    bool tsn_dirty = false;                       // peer access: local A / G written outside the step kernel (barrier owed)
    void** d_peer_bases = nullptr;                // [3][8]: LSA bases of A, G, G2 of every rank
    // windows of the previous model kept registered for the next one of the same
    // size (a replace-ingest job skips the collective deregister / register)
    void* fcache_buf[3] = {nullptr, nullptr, nullptr};
    ncclWindow_t fcache_win[3] = {nullptr, nullptr, nullptr};
    size_t fcache_bytes = 0;
    size_t fwin_bytes = 0;                        // size of each live window
    bool closing = false;                         // gcp_destroy: free everything
    void* twosided = nullptr;                     // row f3 scratch (twosided.cu)
    int fmem[gcp::kMaxModes][8] = {{0}}, fnmem[gcp::kMaxModes] = {0};
    int64_t tau = 0;
    gcp_adam_params server{};
    bool server_set = false;
    // ---- tensor
    bool have_tensor = false;
    int d = 0;
    int64_t dims[gcp::kMaxModes] = {0}, lo[gcp::kMaxModes] = {0}, hi[gcp::kMaxModes] = {0};
    int64_t N = 0, N_global = 0;
    unsigned __int128 M = 0;            // local block entries
    bool any_zero_global = true;        // some rank has M_w > N_w
    uint32_t* d_rec = nullptr;
    int rec_words = 4, val_words = 1;
    uint64_t* d_hash = nullptr;
    uint64_t hash_slots = 0;
    int key128 = 0;
    gcp_membership member = GCP_MEMBER_HASH;   // zero-test structure built at ingest
    uint64_t* d_keys = nullptr;                // sorted keys (GCP_MEMBER_SORTED)
    uint64_t* d_filter = nullptr;              // L2-resident negative test in front of the zero test
    cudaMemPool_t scratch_pool = nullptr;      // ingest scratch (ingest.cu)
    uint64_t filter_sectors = 0;
    bool lean_ingest = false;                  // the last ingest took the lean (key, value) sort path
    // ---- model
    bool have_model = false;
    int R = 0, R_pad = 0;
    int64_t rows[gcp::kMaxModes] = {0};     // allocated rows per mode (>= block rows, multiple of slice size)
    int64_t off[gcp::kMaxModes] = {0};      // element offsets
    int64_t n_coef = 0;                     // logical coefficients (B, C layout)
    int l2_first = 0;                       // K2's record / bucket reads carry an L2 evict_first policy
    bool ag_interleaved = false;            // A and G rows interleaved in one buffer (d_G = d_A + R_pad)
    int ag_stride = 0;                      // elements between consecutive A (or G) rows
    void *d_A = nullptr, *d_G = nullptr, *d_B = nullptr, *d_C = nullptr, *d_lambda = nullptr;
    void *d_Ack = nullptr, *d_Bck = nullptr, *d_Cck = nullptr;   // fit checkpoint
    void *d_U = nullptr, *d_Bs = nullptr, *d_Cs = nullptr;       // FedAdam server copy + state
    int64_t t = 0, t_ck = 0, ts = 0, ts_ck = 0;
    uint32_t it = 0;
    bool have_grad = false;
    int last_loss = 0;
    // ---- sampler binding
    bool bound = false;
    gcp_strategy strategy = GCP_STRATIFIED;
    int64_t s_nz = 0, s_z = 0, p_w = 0, q_w = 0;
    uint64_t seed = 0;
    // ---- scratch
    double* d_partials = nullptr;       // per-CTA fp64 partial sums
    int partials_cap = 0;
    double* h_scalar = nullptr;         // pinned
    unsigned long long* d_err = nullptr;
    unsigned long long* h_err = nullptr;  // pinned
    int grad_blocks = 0;                // persistent grid of the sample kernels
    // ---- epoch graph (gcp_fit_epoch): captured once per (fit, phase) key, replayed
    gcp::DevStep* d_step = nullptr;     // device step state read by K2 / Adam during replay
    gcp::DevStep* h_step = nullptr;     // pinned staging for the per-replay upload
    bool capturing = false;
    // slot ordering (kernels.cu launch_slot_order): the gradient K2 visits its slots
    // grouped by mode-1 position; one allocation (d_ord_buf) sized for ord_cap slots
    void* d_ord_buf = nullptr;
    int64_t* d_ord_T = nullptr;         // per-tensor bucket -> first record table (2^bits + 1)
    uint16_t* d_ord_lut = nullptr;      // per-tensor nonzero index -> bucket lookup (kernels.cu)
    int ord_lut_shift = 0;
    uint32_t* d_ord_cnt = nullptr;      // bucket totals, cursors
    uint32_t* d_ord = nullptr;          // visiting order (slot ids)
    uint32_t* d_ord_key = nullptr;      // (tile, bucket) per slot
    int ord_tile_shift = 62, ord_ntiles = 1;   // slot tiles ordered independently (large p + q)
    uint32_t* d_ord_rank = nullptr;     // rank of the slot inside its bucket
    int64_t ord_cap = 0;
    int ord_bits = 15;                  // log2 of the bucket count (GCP_ORD_BITS)
    int ord_stage = 0;                  // slot order of iteration ord_stage_it prepared by earlier launches:
    uint32_t ord_stage_it = 0;          // 1 histogram (in K2), 2 scan + scatter too (in Adam), 0 nothing
    int slot_order = 0;                 // decided in gcp_model_init (GCP_SLOT_ORDER overrides)
    bool slot_order_forced = false;     // GCP_SLOT_ORDER=1: also when the order array does not fit L2
    cudaGraphExec_t graph_exec = nullptr;
    double graph_key[8] = {0};
    double graph_seen[8] = {0};         // key of the last eager epoch: capture on the second sighting
    bool graph_seen_valid = false;
    int64_t graph_launches = 0;         // library launches recorded in the graph
    uint32_t graph_it0 = 0;             // it / t at the start of the capture: launch offsets are relative
    int64_t graph_t0 = 0;
    // ---- fit state
    bool fit_active = false;
    gcp_fit_params fp{};
    double best = 0, rate = 0;
    int fails = 0, epoch = 0;
    // ---- instrumentation
    int64_t launches = 0;
    bool prof_on = false;
    struct PendingEv { cudaEvent_t a, b; int which; };
    std::vector<PendingEv> pending;
    std::vector<cudaEvent_t> ev_pool;
    double prof_ms[gcp::PROF_N] = {0};
    int64_t prof_n[gcp::PROF_N] = {0};
};

namespace gcp {

// Alg. 2 schemes (one model, per-iteration exchange) vs Alg. 3 / 4 (replicas)
inline bool sync_family(const gcp_ctx* c) {
    return c->mode == GCP_DIST_SYNC || c->mode == GCP_DIST_SYNC_TWO_SIDED;
}
inline bool async_family(const gcp_ctx* c) {
    return c->mode == GCP_DIST_ASYNC_AVG || c->mode == GCP_DIST_ASYNC_FEDADAM;
}
inline bool two_sided(const gcp_ctx* c) { return c->P > 1 && c->mode == GCP_DIST_SYNC_TWO_SIDED; }

// thread-local error message + status helpers (api.cu)
gcp_status set_error(gcp_status st, const std::string& msg);
gcp_status cuda_fail(gcp_ctx* c, cudaError_t e, const char* what);
gcp_status nccl_fail(gcp_ctx* c, ncclResult_t r, const char* what);

// launch bracketing for the profiler and the launch counter
void prof_begin(gcp_ctx* c, int which, cudaEvent_t* ev);
void prof_end(gcp_ctx* c, int which, cudaEvent_t ev);

// kernels.cu launchers (enqueue on c->stream; return cudaGetLastError())
cudaError_t launch_sample_kernel(gcp_ctx* c, const SampleArgs& s, const ModelArgs& m, int loss,
                                 int loss_mode, int semi_nz, double w_nz, double w_z, int with_loss,
                                 double* partials, int nblocks,
                                 const OrdHistArgs* oh = nullptr);   // next iteration's slot histogram
size_t slot_order_bytes(int64_t cap);
cudaError_t slot_order_init(gcp_ctx* c, void* buf, int64_t cap);   // carve buffers, build the per-tensor table
cudaError_t launch_slot_order(gcp_ctx* c, const SampleArgs& s, const uint32_t** order_out, int stage);
bool ord_hist_args(gcp_ctx* c, const SampleArgs& next, OrdHistArgs* oh);
bool ord_scatter_args(gcp_ctx* c, int64_t n, OrdScatterArgs* os, int64_t adam_vecs);   // + launches the scan
cudaError_t launch_reduce_partials(gcp_ctx* c, const double* partials, int n, double* out);
cudaError_t launch_export(gcp_ctx* c, const SampleArgs& s, int stratum, int64_t first, int64_t count,
                          const int64_t* lo, int64_t* subs, int64_t* j, int32_t* att);
cudaError_t launch_adam(gcp_ctx* c, const Segment& seg, void* A, void* G, void* B, void* C,
                        double rate, double beta1, double beta2, double eps, double lower,
                        int64_t t, int zero_g, int row_stride = 0,    // row_stride 0: contiguous A/G
                        const DevStep* step = nullptr,                // step: t = step->t + t (offset), rate
                        const OrdScatterArgs* os = nullptr);          // fused next-iteration slot scatter
cudaError_t launch_init(gcp_ctx* c, uint64_t seed, const int64_t* goff);
cudaError_t launch_scale(gcp_ctx* c, void* x, int64_t n, double s);
cudaError_t launch_sub(gcp_ctx* c, const void* a, const void* b, void* out, int64_t n);
cudaError_t launch_rows_in(gcp_ctx* c, const double* src, void* dst, int64_t b);    // packed rows -> layout
cudaError_t launch_rows_out(gcp_ctx* c, const void* src, double* dst, int64_t b);   // layout -> packed rows
int sample_kernel_blocks(gcp_ctx* c);
cudaError_t launch_debug_philox(gcp_ctx* c, int64_t n, const uint32_t* in, uint32_t* out);

// ingest.cu
gcp_status ingest(gcp_ctx* c, const gcp_ctx* geom, int64_t nnz, const int64_t* subs, const double* vals);
cudaError_t launch_contains(gcp_ctx* c, int64_t n, const int64_t* coords_dev, int8_t* out_dev);

// dist.cu
gcp_status dist_make_slices(gcp_ctx* c);
gcp_status dist_sync_exchange_pre(gcp_ctx* c);     // reduce-scatter G
gcp_status dist_sync_exchange_post(gcp_ctx* c);    // all-gather A
gcp_status dist_async_sync(gcp_ctx* c);            // Alg. 3 averaging / Alg. 4 server step
gcp_status dist_allreduce_scalar(gcp_ctx* c, double* dev_scalar);
gcp_status dist_allreduce_i64_host(gcp_ctx* c, int64_t* v, int n);

// twosided.cu (row f3)
gcp_status twosided_import(gcp_ctx* c, const SampleArgs& sa);
gcp_status twosided_export(gcp_ctx* c);
void twosided_free(gcp_ctx* c);

// fused.cu
bool fused_possible(gcp_ctx* c);
bool fused_use_multimem(const gcp_ctx* c);   // NVLS multicast for full-team modes
gcp_status fused_alloc(gcp_ctx* c, size_t bytes);   // A, G, G2 as symmetric windows (collective)
void fused_free(gcp_ctx* c);
void fused_cache_release(gcp_ctx* c);   // collective: deregister the kept windows
gcp_status fused_exchange(gcp_ctx* c, const gcp_adam_params* p, double lower);
gcp_status tsn_alloc_bitmap(gcp_ctx* c);          // two-sided over NVLink: the bit window (collective)

// twosided_nvl.cu (row f3 driven by the device over the symmetric windows)
bool tsn_possible(gcp_ctx* c);
size_t tsn_bitmap_bytes(const gcp_ctx* c);
gcp_status tsn_import(gcp_ctx* c, const SampleArgs& sa);
gcp_status tsn_export(gcp_ctx* c, const gcp_adam_params* p, double lower);
gcp_status tsn_peer_setup(gcp_ctx* c);                          // the LSA base table (after fused_alloc)
gcp_status tsn_peer_step(gcp_ctx* c, const gcp_adam_params* p, double lower);   // barrier + Adam + barrier
bool tsn_peer_wanted(const gcp_ctx* c);                         // peer access (default up to 8 ranks)
gcp_status tsn_peer_sync(gcp_ctx* c);                           // LSA barrier if tsn_dirty (before peers read / add)

}  // namespace gcp

namespace gcp {
// Device allocations come from the device's stream-ordered memory pool (its
// release threshold is raised at gcp_create), so the multi-GB ingest scratch
// and model buffers of repeated jobs reuse mapped memory instead of paying
// cudaMalloc / cudaFree page mapping every time.
template <typename P>
inline cudaError_t gmalloc(gcp_ctx* c, P** p, size_t bytes) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), bytes, c->stream);
    if (e == cudaErrorMemoryAllocation && c->scratch_pool) {
        // the ingest scratch pool keeps its memory mapped between ingests: give it back and retry
        cudaGetLastError();
        cudaStreamSynchronize(c->stream);
        cudaMemPoolTrimTo(c->scratch_pool, 0);
        e = cudaMallocAsync(reinterpret_cast<void**>(p), bytes, c->stream);
    }
    return e;
}
inline cudaError_t gfree(gcp_ctx* c, void* p) { return p ? cudaFreeAsync(p, c->stream) : cudaSuccess; }
}  // namespace gcp
