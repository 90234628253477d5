// api.cu -- the C ABI of include/gcp.h: argument validation, the context state
// machine, and the host side of the hot path (which kernel runs when, with
// which weights and counters).  All arithmetic runs in the kernels of
// kernels.cuh; this file only orchestrates.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "gcp_internal.h"

using namespace gcp;

namespace gcp {

static thread_local std::string g_err;

gcp_status set_error(gcp_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

gcp_status cuda_fail(gcp_ctx* c, cudaError_t e, const char* what) {
    if (c) c->sticky = GCP_E_CUDA;
    return set_error(GCP_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

gcp_status nccl_fail(gcp_ctx* c, ncclResult_t r, const char* what) {
    if (c) c->sticky = GCP_E_NCCL;
    return set_error(GCP_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

static cudaEvent_t ev_get(gcp_ctx* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void prof_begin(gcp_ctx* c, int which, cudaEvent_t* ev) {
    (void)which;
    c->launches++;
    *ev = nullptr;
    if (!c->prof_on) return;
    *ev = ev_get(c);
    cudaEventRecord(*ev, c->stream);
}

void prof_end(gcp_ctx* c, int which, cudaEvent_t ev) {
    if (!c->prof_on || !ev) return;
    cudaEvent_t b = ev_get(c);
    cudaEventRecord(b, c->stream);
    c->pending.push_back({ev, b, which});
}

static void prof_resolve(gcp_ctx* c) {
    for (auto& p : c->pending) {
        cudaEventSynchronize(p.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.a, p.b);
        c->prof_ms[p.which] += ms;
        c->prof_n[p.which] += 1;
        c->ev_pool.push_back(p.a);
        c->ev_pool.push_back(p.b);
    }
    c->pending.clear();
}

}  // namespace gcp

// ---------------------------------------------------------------- helpers
namespace {

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

#define ENTER(c)                                                                     \
    if (!(c)) return set_error(GCP_E_ARG, "null context");                          \
    if ((c)->sticky != GCP_OK)                                                       \
        return set_error(GCP_E_STATE, "context is in a sticky error state (" +      \
                                          std::to_string((int)(c)->sticky) + ")");  \
    DevGuard guard_((c)->dev)

#define CUDA_TRY(c, x, what)                                   \
    do {                                                       \
        cudaError_t e_ = (x);                                  \
        if (e_ != cudaSuccess) return cuda_fail((c), e_, what); \
    } while (0)

#define ST_TRY(x)                      \
    do {                               \
        gcp_status s_ = (x);           \
        if (s_ != GCP_OK) return s_;   \
    } while (0)

int64_t alloc_count(int64_t total, int P, int w) { return total / P + (w < total % P ? 1 : 0); }

double u128_to_double(unsigned __int128 v) { return (double)v; }

double loss_lower(int loss) { return loss == GCP_LOSS_POISSON ? 0.0 : -INFINITY; }

// The captured epoch graph bakes in buffer pointers, sample counts and the
// iteration schedule: any change to them drops it (rebuilt on the next epoch).
void graph_drop(gcp_ctx* c) {
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    c->graph_exec = nullptr;
}

void free_model(gcp_ctx* c) {
    graph_drop(c);
    fused_free(c);                             // symmetric A / G windows (collective)
    if (c->ag_interleaved) c->d_G = nullptr;   // a view into d_A
    c->ag_interleaved = false;
    gfree(c, c->d_peer_bases);
    c->d_peer_bases = nullptr;
    c->tsn_peer = false;
    void** bufs[] = {&c->d_A, &c->d_G, &c->d_B, &c->d_C, &c->d_lambda, &c->d_Ack, &c->d_Bck, &c->d_Cck,
                     &c->d_U,  &c->d_Bs, &c->d_Cs};
    for (void** b : bufs) {
        gfree(c, *b);
        *b = nullptr;
    }
    c->have_model = false;
    c->have_grad = false;
    c->fit_active = false;
}

// Local sample counts for a GLOBAL total under the empty-strata rule
// (SURVEY C4): a rank without nonzeros (zeros) draws none of that stratum.
void local_counts(const gcp_ctx* c, int64_t s_nz, int64_t s_z, int64_t* p_w, int64_t* q_w) {
    *p_w = c->N > 0 ? alloc_count(s_nz, c->P, c->rank) : 0;
    *q_w = c->M > (unsigned __int128)c->N ? alloc_count(s_z, c->P, c->rank) : 0;
}

double weight_nz(const gcp_ctx* c, int64_t p_w) { return p_w > 0 ? (double)c->N / (double)p_w : 0.0; }
double weight_z(const gcp_ctx* c, int64_t q_w) {
    return q_w > 0 ? u128_to_double(c->M - (unsigned __int128)c->N) / (double)q_w : 0.0;
}

SampleArgs sample_args(const gcp_ctx* c, int64_t p, int64_t q, uint64_t seed, uint32_t it, uint32_t kind_nz,
                       uint32_t kind_z, int stratified) {
    SampleArgs s;
    s.rec = c->d_rec;
    s.rec_words = c->rec_words;
    s.val_words = c->val_words;
    s.N = c->N;
    s.hash = c->d_hash;
    s.hash_mask = c->hash_slots - 1;
    s.filter = c->filter_sectors ? c->d_filter : nullptr;
    s.filter_mask = c->filter_sectors ? c->filter_sectors - 1 : 0;
    s.key128 = c->key128;
    for (int k = 0; k < kMaxModes; ++k) s.bdim[k] = k < c->d ? (uint32_t)(c->hi[k] - c->lo[k]) : 1u;
    s.p = p;
    s.q = q;
    s.seed = seed;
    s.rank = (uint32_t)c->rank;
    s.it = it;
    s.kind_nz = kind_nz;
    s.kind_z = kind_z;
    s.stratified = stratified;
    s.member_sorted = c->member == GCP_MEMBER_SORTED;
    s.keys = c->d_keys;
    s.err_slot = c->d_err;
    s.it_dev = nullptr;
    s.order = nullptr;
    s.l2_first = c->l2_first;
    if (c->capturing) {   // epoch graph: this launch's iteration relative to the replay's first
        s.it_dev = &c->d_step->it;
        s.it = it - c->graph_it0;
    }
    return s;
}

// the G buffer the current iteration accumulates into (parity-double-buffered
// under the fused exchange, fused.cu)
void* cur_G(const gcp_ctx* c) { return (c->fused && (c->it & 1)) ? c->d_G2 : c->d_G; }

ModelArgs model_args(const gcp_ctx* c) {
    ModelArgs m;
    m.A = c->d_A;
    m.G = cur_G(c);
    m.lambda = c->d_lambda;
    const int64_t mult = c->ag_stride / c->R_pad;   // 1, or 2 when A/G rows interleave
    for (int k = 0; k < kMaxModes; ++k) m.off[k] = k < c->d ? c->off[k] * mult : 0;
    m.R_pad = c->R_pad;
    m.row_stride = c->ag_stride;
    m.peerA = nullptr;
    m.peerG = nullptr;
    for (int k = 0; k < kMaxModes; ++k) {
        m.shard[k] = 1;
        m.nmem[k] = 1;
        for (int j = 0; j < 8; ++j) m.mem[k][j] = 0;
    }
    if (c->tsn_peer) {
        m.peerA = const_cast<const void* const*>(c->d_peer_bases);
        m.peerG = c->d_peer_bases + ((c->it & 1) ? 16 : 8);
        for (int k = 0; k < c->d; ++k) {
            m.shard[k] = c->rows[k] / c->slice_size[k];
            m.nmem[k] = c->fnmem[k];
            for (int j = 0; j < c->fnmem[k]; ++j) m.mem[k][j] = c->fmem[k][j];
        }
    }
    return m;
}

// the slot-order buffers (their table T is per tensor: dropped with the tensor)
void ord_free(gcp_ctx* c) {
    graph_drop(c);
    c->ord_stage = 0;
    gfree(c, c->d_ord_buf);
    c->d_ord_buf = nullptr;
    c->d_ord_T = nullptr;
    c->d_ord_lut = nullptr;
    c->d_ord_cnt = nullptr;
    c->d_ord = nullptr;
    c->d_ord_key = nullptr;
    c->d_ord_rank = nullptr;
    c->ord_cap = 0;
}

gcp_status ensure_partials(gcp_ctx* c, int n) {
    if (n <= c->partials_cap) return GCP_OK;
    gfree(c, c->d_partials);
    c->d_partials = nullptr;
    CUDA_TRY(c, gmalloc(c, &c->d_partials, sizeof(double) * (n + 1)), "partials");
    c->partials_cap = n;
    return GCP_OK;
}

// Check the rejection-cap flag after a synchronisation point.
gcp_status check_err(gcp_ctx* c, const char* what) {
    CUDA_TRY(c, cudaMemcpyAsync(c->h_err, c->d_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream),
             what);
    CUDA_TRY(c, cudaStreamSynchronize(c->stream), what);
    if (*c->h_err != ULLONG_MAX) {
        c->sticky = GCP_E_REJECT_CAP;
        return set_error(GCP_E_REJECT_CAP, std::string(what) + ": rank " + std::to_string(c->rank) +
                                               " zero slot " + std::to_string(*c->h_err) +
                                               " rejected 1000 times (reading R5)");
    }
    return GCP_OK;
}

// Run the sample kernel in loss mode over a stratified sample set and return the
// local sum sum_s w f into *out_dev (device double).
gcp_status run_loss_kernel(gcp_ctx* c, int loss, int64_t p, int64_t q, uint64_t seed, uint32_t it,
                           uint32_t kind_nz, uint32_t kind_z, int stratified, int semi_nz, int prof_which,
                           int loss_mode, double* out_dev) {
    const int nb = c->grad_blocks;
    ST_TRY(ensure_partials(c, nb));
    const SampleArgs s = sample_args(c, p, q, seed, it, kind_nz, kind_z, stratified);
    const ModelArgs m = model_args(c);
    cudaEvent_t ev;
    prof_begin(c, prof_which, &ev);
    CUDA_TRY(c, launch_sample_kernel(c, s, m, loss, loss_mode, semi_nz, weight_nz(c, p), weight_z(c, q), 1,
                                     c->d_partials, nb),
             "sample kernel");
    prof_end(c, prof_which, ev);
    prof_begin(c, PROF_OTHER, &ev);
    CUDA_TRY(c, launch_reduce_partials(c, c->d_partials, nb, out_dev), "reduce partials");
    prof_end(c, PROF_OTHER, ev);
    return GCP_OK;
}

size_t tsz(const gcp_ctx* c) { return c->prec == GCP_FP32 ? 4 : 8; }

// element offset of mode k's first row in the A (or G) buffer
int64_t phys_off(const gcp_ctx* c, int k) { return c->off[k] * (c->ag_stride / c->R_pad); }

// elements of the A allocation (twice n_coef when G rows are interleaved into it)
size_t a_elems(const gcp_ctx* c) { return (size_t)c->n_coef * (c->ag_interleaved ? 2 : 1); }

gcp_status checkpoint_save(gcp_ctx* c) {
    const size_t bytes = (size_t)c->n_coef * tsz(c);
    const size_t abytes = a_elems(c) * tsz(c);   // A (with interleaved G rows, which are zero here)
    if (!c->d_Ack) {
        CUDA_TRY(c, gmalloc(c, &c->d_Ack, abytes), "checkpoint alloc");
        CUDA_TRY(c, gmalloc(c, &c->d_Bck, bytes), "checkpoint alloc");
        CUDA_TRY(c, gmalloc(c, &c->d_Cck, bytes), "checkpoint alloc");
    }
    CUDA_TRY(c, cudaMemcpyAsync(c->d_Ack, c->d_A, abytes, cudaMemcpyDeviceToDevice, c->stream), "checkpoint");
    CUDA_TRY(c, cudaMemcpyAsync(c->d_Bck, c->d_B, bytes, cudaMemcpyDeviceToDevice, c->stream), "checkpoint");
    CUDA_TRY(c, cudaMemcpyAsync(c->d_Cck, c->d_C, bytes, cudaMemcpyDeviceToDevice, c->stream), "checkpoint");
    c->t_ck = c->t;
    c->ts_ck = c->ts;
    return GCP_OK;
}

gcp_status checkpoint_restore(gcp_ctx* c) {
    const size_t bytes = (size_t)c->n_coef * tsz(c);
    const size_t abytes = a_elems(c) * tsz(c);
    CUDA_TRY(c, cudaMemcpyAsync(c->d_A, c->d_Ack, abytes, cudaMemcpyDeviceToDevice, c->stream), "restore");
    CUDA_TRY(c, cudaMemcpyAsync(c->d_B, c->d_Bck, bytes, cudaMemcpyDeviceToDevice, c->stream), "restore");
    CUDA_TRY(c, cudaMemcpyAsync(c->d_C, c->d_Cck, bytes, cudaMemcpyDeviceToDevice, c->stream), "restore");
    if (!c->ag_interleaved) CUDA_TRY(c, cudaMemsetAsync(c->d_G, 0, bytes, c->stream), "restore");
    if (c->fused) CUDA_TRY(c, cudaMemsetAsync(c->d_G2, 0, bytes, c->stream), "restore");
    if (c->d_bm) CUDA_TRY(c, cudaMemsetAsync(c->d_bm, 0, tsn_bitmap_bytes(c), c->stream), "restore");
    c->tsn_dirty = true;
    c->t = c->t_ck;
    c->ts = c->ts_ck;
    return GCP_OK;
}

// FedAdam server copy U <- current model, server moments zeroed (start of a fit).
gcp_status server_reset(gcp_ctx* c) {
    if (c->mode != GCP_DIST_ASYNC_FEDADAM) return GCP_OK;
    const size_t bytes = (size_t)c->n_coef * tsz(c);
    if (!c->d_U) {
        CUDA_TRY(c, gmalloc(c, &c->d_U, bytes), "server alloc");
        CUDA_TRY(c, gmalloc(c, &c->d_Bs, bytes), "server alloc");
        CUDA_TRY(c, gmalloc(c, &c->d_Cs, bytes), "server alloc");
    }
    CUDA_TRY(c, cudaMemcpyAsync(c->d_U, c->d_A, bytes, cudaMemcpyDeviceToDevice, c->stream), "server reset");
    CUDA_TRY(c, cudaMemsetAsync(c->d_Bs, 0, bytes, c->stream), "server reset");
    CUDA_TRY(c, cudaMemsetAsync(c->d_Cs, 0, bytes, c->stream), "server reset");
    c->ts = 0;
    return GCP_OK;
}

bool valid_loss(int loss) { return loss >= 0 && loss <= 2; }

}  // namespace

// NVTX ranges around the ABI's phases (no-ops unless a profiler is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// ================================================================ ABI
extern "C" {

const char* gcp_last_error(void) { return g_err.c_str(); }

gcp_status gcp_create(gcp_ctx** out, int cuda_device, void* cuda_stream, gcp_precision prec) {
    if (!out) return set_error(GCP_E_ARG, "gcp_create: out is NULL");
    *out = nullptr;
    if (prec != GCP_FP32 && prec != GCP_FP64) return set_error(GCP_E_ARG, "gcp_create: bad precision");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) return set_error(GCP_E_CUDA, "gcp_create: no CUDA device");
    if (cuda_device < 0 || cuda_device >= ndev) return set_error(GCP_E_ARG, "gcp_create: bad device");
    DevGuard g(cuda_device);
    int major = 0, sms = 0, l2 = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, cuda_device) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device) != cudaSuccess ||
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, cuda_device) != cudaSuccess)
        return set_error(GCP_E_CUDA, "gcp_create: cudaDeviceGetAttribute failed");
    if (major != 10) return set_error(GCP_E_CUDA, "gcp_create: libgcp is built for sm_100a (B200) only");
    {
        // stream-ordered pool keeps freed memory mapped for the next job (gmalloc)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, cuda_device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    gcp_ctx* c = new gcp_ctx();
    c->dev = cuda_device;
    c->stream = (cudaStream_t)cuda_stream;
    c->prec = prec;
    c->tsize = prec == GCP_FP32 ? 4 : 8;
    c->sm_count = sms;
    c->l2_bytes = l2;
    if (cudaMallocHost(&c->h_scalar, 64) != cudaSuccess || cudaMallocHost(&c->h_err, 64) != cudaSuccess ||
        gmalloc(c, &c->d_err, 64) != cudaSuccess) {
        gcp_destroy(c);
        return set_error(GCP_E_OOM, "gcp_create: allocation failed");
    }
    cudaMemsetAsync(c->d_err, 0xFF, sizeof(unsigned long long), c->stream);
    cudaStreamSynchronize(c->stream);
    *out = c;
    return GCP_OK;
}

void gcp_destroy(gcp_ctx* c) {
    if (!c) return;
    DevGuard g(c->dev);
    cudaStreamSynchronize(c->stream);
    c->closing = true;
    free_model(c);
    fused_cache_release(c);
    ord_free(c);
    gfree(c, c->d_rec);
    gfree(c, c->d_hash);
    gfree(c, c->d_keys);
    gfree(c, c->d_filter);
    gfree(c, c->d_partials);
    gfree(c, c->d_err);
    gfree(c, c->d_step);
    if (c->h_step) cudaFreeHost(c->h_step);
    if (c->h_scalar) cudaFreeHost(c->h_scalar);
    if (c->h_err) cudaFreeHost(c->h_err);
    for (auto& p : c->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (int k = 0; k < kMaxModes; ++k)
        if (c->slice[k]) ncclCommDestroy(c->slice[k]);
    twosided_free(c);
    if (c->scratch_pool) {
        cudaStreamSynchronize(c->stream);
        cudaMemPoolDestroy(c->scratch_pool);
    }
    if (c->devcomm_ready) ncclDevCommDestroy(c->world, &c->devcomm);
    if (c->world) ncclCommDestroy(c->world);
    delete c;
}

gcp_status gcp_dist_set_async(gcp_ctx* c, int64_t tau, const gcp_adam_params* server) {
    ENTER(c);
    if (tau < 0) return set_error(GCP_E_ARG, "gcp_dist_set_async: tau < 0");
    c->tau = tau;
    if (server) {
        c->server = *server;
        c->server_set = true;
    }
    graph_drop(c);
    return GCP_OK;
}

gcp_status gcp_set_membership(gcp_ctx* c, gcp_membership m) {
    ENTER(c);
    if (m != GCP_MEMBER_HASH && m != GCP_MEMBER_SORTED) return set_error(GCP_E_ARG, "gcp_set_membership: bad value");
    c->member = m;
    graph_drop(c);
    return GCP_OK;
}

gcp_status gcp_tensor_create(gcp_ctx* c, int d, const int64_t* dims, int64_t nnz, const int64_t* subs,
                             const double* vals) {
    ENTER(c);
    NvtxRange nvtx_("gcp_tensor_create");
    if (d < 2 || d > kMaxD) return set_error(GCP_E_ARG, "gcp_tensor_create: need 2 <= d <= 6");
    if (!dims || nnz < 0 || (nnz > 0 && (!subs || !vals)))
        return set_error(GCP_E_ARG, "gcp_tensor_create: bad pointers / nnz");
    for (int k = 0; k < d; ++k)
        if (dims[k] < 1 || dims[k] > 0xFFFFFFFFLL)
            return set_error(GCP_E_ARG, "gcp_tensor_create: each I_k must be in [1, 2^32-1]");
    if (c->P > 1 && !c->dist_ready) return set_error(GCP_E_STATE, "gcp_tensor_create: gcp_dist_init first");
    // stage the geometry
    gcp_ctx* g = new gcp_ctx();
    g->d = d;
    int grid[kMaxModes];
    if (c->P > 1) {
        if (c->grid_given) {
            int64_t prod = 1;
            for (int k = 0; k < d; ++k) prod *= c->grid[k];
            if (prod != c->P) {
                delete g;
                return set_error(GCP_E_ARG, "gcp_tensor_create: grid product != nranks");
            }
            for (int k = 0; k < d; ++k) grid[k] = c->grid[k];
        } else {
            gcp_status s = gcp_grid_plan(c->P, d, dims, grid, nullptr, nullptr);
            if (s != GCP_OK) { delete g; return s; }
        }
    } else {
        for (int k = 0; k < d; ++k) grid[k] = 1;
    }
    {
        // rank coordinates (row-major, b_1 slowest) and ceil-based block bounds (reading R14)
        int rem = c->rank;
        int b[kMaxModes];
        for (int k = d - 1; k >= 0; --k) {
            b[k] = rem % grid[k];
            rem /= grid[k];
        }
        // M = prod I_k must be representable in u128 (SPEC S:26 errors on an
        // overflowing M_tot); the block's M is at most that
        unsigned __int128 Mg = 1;
        for (int k = 0; k < d; ++k) {
            if (Mg > (~(unsigned __int128)0) / (unsigned __int128)dims[k]) {
                delete g;
                return set_error(GCP_E_ARG, "gcp_tensor_create: prod I_k overflows 128 bits");
            }
            Mg *= (unsigned __int128)dims[k];
        }
        g->M = 1;
        for (int k = 0; k < d; ++k) {
            const int64_t ck = (dims[k] + grid[k] - 1) / grid[k];
            g->dims[k] = dims[k];
            g->lo[k] = std::min<int64_t>(b[k] * ck, dims[k]);
            g->hi[k] = std::min<int64_t>((b[k] + 1) * ck, dims[k]);
            g->M *= (unsigned __int128)(g->hi[k] - g->lo[k]);
        }
    }
    // Replace: drop the previous model and tensor before the ingest, so its
    // scratch reuses their memory (the pool keeps it mapped) instead of growing
    // past them.  A failed ingest leaves the context without a tensor.
    free_model(c);
    ord_free(c);
    gfree(c, c->d_rec);
    gfree(c, c->d_hash);
    gfree(c, c->d_keys);
    gfree(c, c->d_filter);
    c->d_rec = nullptr;
    c->d_hash = nullptr;
    c->d_keys = nullptr;
    c->d_filter = nullptr;
    c->filter_sectors = 0;
    c->have_tensor = false;
    c->bound = false;
    gcp_status st = ingest(c, g, nnz, subs, vals);
    if (st != GCP_OK) {
        delete g;
        return st;
    }
    c->d = d;
    for (int k = 0; k < kMaxModes; ++k) {
        c->dims[k] = k < d ? g->dims[k] : 0;
        c->lo[k] = k < d ? g->lo[k] : 0;
        c->hi[k] = k < d ? g->hi[k] : 0;
        c->grid[k] = k < d ? grid[k] : 0;
    }
    c->M = g->M;
    c->N = nnz;
    delete g;
    c->bound = false;
    // global N and "some rank has zeros"
    int64_t agg[2] = {nnz, c->M > (unsigned __int128)nnz ? 1 : 0};
    if (c->P > 1) {
        ST_TRY(dist_make_slices(c));
        ST_TRY(dist_allreduce_i64_host(c, agg, 2));
    } else {
        for (int k = 0; k < kMaxModes; ++k) {
            c->slice_size[k] = 1;
            c->slice_rank[k] = 0;
        }
    }
    c->N_global = agg[0];
    c->any_zero_global = agg[1] > 0;
    c->have_tensor = true;
    return GCP_OK;
}

gcp_status gcp_tensor_info(gcp_ctx* c, int64_t* nnz_local, int64_t* lo, int64_t* hi, double* M_local,
                           int64_t* nnz_global) {
    ENTER(c);
    if (!c->have_tensor) return set_error(GCP_E_STATE, "no tensor");
    if (nnz_local) *nnz_local = c->N;
    for (int k = 0; k < c->d; ++k) {
        if (lo) lo[k] = c->lo[k];
        if (hi) hi[k] = c->hi[k];
    }
    if (M_local) *M_local = u128_to_double(c->M);
    if (nnz_global) *nnz_global = c->N_global;
    return GCP_OK;
}

gcp_status gcp_tensor_export_sorted(gcp_ctx* c, int64_t first, int64_t count, int64_t* subs_out,
                                    double* vals_out) {
    ENTER(c);
    if (!c->have_tensor) return set_error(GCP_E_STATE, "no tensor");
    if (first < 0 || count < 0 || first + count > c->N) return set_error(GCP_E_RANGE, "export_sorted: range");
    if (count == 0) return GCP_OK;
    std::vector<uint32_t> rec((size_t)count * c->rec_words);
    CUDA_TRY(c, cudaMemcpyAsync(rec.data(), c->d_rec + first * c->rec_words, rec.size() * 4,
                                cudaMemcpyDeviceToHost, c->stream),
             "export_sorted");
    CUDA_TRY(c, cudaStreamSynchronize(c->stream), "export_sorted");
    for (int64_t n = 0; n < count; ++n) {
        const uint32_t* r = &rec[(size_t)n * c->rec_words];
        if (vals_out) {
            if (c->val_words == 1) {
                float f;
                memcpy(&f, r, 4);
                vals_out[n] = f;
            } else {
                memcpy(&vals_out[n], r, 8);
            }
        }
        if (subs_out)
            for (int k = 0; k < c->d; ++k) subs_out[n * c->d + k] = c->lo[k] + (int64_t)r[c->val_words + k];
    }
    return GCP_OK;
}

gcp_status gcp_tensor_contains(gcp_ctx* c, int64_t n, const int64_t* coords, int8_t* out) {
    ENTER(c);
    if (!c->have_tensor) return set_error(GCP_E_STATE, "no tensor");
    if (n < 0 || (n > 0 && (!coords || !out))) return set_error(GCP_E_ARG, "contains: args");
    for (int64_t x = 0; x < n; ++x)
        for (int k = 0; k < c->d; ++k)
            if (coords[x * c->d + k] < c->lo[k] || coords[x * c->d + k] >= c->hi[k])
                return set_error(GCP_E_RANGE, "contains: coordinate outside block");
    if (n == 0) return GCP_OK;
    int64_t* dc = nullptr;
    int8_t* dout = nullptr;
    CUDA_TRY(c, gmalloc(c, &dc, sizeof(int64_t) * n * c->d), "contains");
    CUDA_TRY(c, gmalloc(c, &dout, n), "contains");
    CUDA_TRY(c, cudaMemcpyAsync(dc, coords, sizeof(int64_t) * n * c->d, cudaMemcpyHostToDevice, c->stream), "contains");
    cudaEvent_t ev;
    prof_begin(c, PROF_OTHER, &ev);
    CUDA_TRY(c, launch_contains(c, n, dc, dout), "contains");
    prof_end(c, PROF_OTHER, ev);
    CUDA_TRY(c, cudaMemcpyAsync(out, dout, n, cudaMemcpyDeviceToHost, c->stream), "contains");
    CUDA_TRY(c, cudaStreamSynchronize(c->stream), "contains");
    gfree(c, dc);
    gfree(c, dout);
    return GCP_OK;
}

gcp_status gcp_model_init(gcp_ctx* c, int R, uint64_t seed) {
    ENTER(c);
    if (!c->have_tensor) return set_error(GCP_E_STATE, "gcp_model_init: no tensor");
    const int rmax = c->prec == GCP_FP32 ? 128 : 64;
    if (R < 1 || R > rmax) return set_error(GCP_E_ARG, "gcp_model_init: need 1 <= R <= 128 (fp32) / 64 (fp64)");
    free_model(c);
    c->R = R;
    c->R_pad = (R + 3) / 4 * 4;
    int64_t off = 0;
    for (int k = 0; k < c->d; ++k) {
        const int64_t b = c->hi[k] - c->lo[k];
        const bool sy = c->P > 1 && sync_family(c);
        const int64_t g = sy ? c->slice_size[k] : 1;
        // sync P > 1: every rank uses the same padded layout (ceil block size,
        // multiple of the slice size), so the A / G windows are symmetric and
        // shards (owned rows) are whole rows of equal size
        const int64_t cb = sy ? (c->dims[k] + c->grid[k] - 1) / c->grid[k] : b;
        c->rows[k] = (cb + g - 1) / g * g;
        c->off[k] = off;
        off += c->rows[k] * c->R_pad;
    }
    c->n_coef = off;
    {
        // sync exchange per mode: all-reduce below 16 MB of block rows, else RS/AG
        const char* env = getenv("GCP_SYNC_EXCHANGE");
        const std::string pol = env ? env : "auto";
        for (int k = 0; k < kMaxModes; ++k) {
            const double mb = k < c->d ? (double)c->rows[k] * c->R_pad * tsz(c) / 1048576.0 : 0;
            c->ar_mode[k] = !two_sided(c) && (pol == "ar" || (pol == "auto" && mb <= 16.0));
        }
    }
    {
        // A/G row interleaving: with one rank in sync mode and a row pair that
        // tiles a 128-B line (R_pad*sizeof(T) in {16, 32, 64}), row i of A^(k)
        // and of G^(k) share one line, so K2's scatter-add hits the line its
        // gather just filled (DRAM traffic per sampled row: 1 fill + 1 write-back
        // instead of 2 fills + 1 write-back).  GCP_AG_INTERLEAVE=0/1 overrides.
        // Only when A + G spill out of L2: with L2-resident factors (c2) the
        // gathers and scatter-adds sharing lines contend in the L2 slices and
        // K2 is ~20% slower; for DRAM-resident factors (c4) it is ~20% faster.
        const size_t rb = (size_t)c->R_pad * tsz(c);
        const bool spills = 2.0 * (double)c->n_coef * (double)tsz(c) > 0.5 * (double)c->l2_bytes;
        bool il = c->P == 1 && c->mode == GCP_DIST_SYNC && (rb == 16 || rb == 32 || rb == 64) && spills;
        const char* env = getenv("GCP_AG_INTERLEAVE");
        if (env) il = atoi(env) != 0 && c->P == 1 && c->mode == GCP_DIST_SYNC;
        c->ag_interleaved = il;
        // the records and hash buckets K2 reads once per sample take an L2
        // evict_first policy when the factors spill out of L2, so they do not
        // displace reused factor rows (c4 K2 2.665 -> 2.62 ms; with L2-resident
        // factors it costs c2 ~1%, profiles/r02l_*); GCP_L2_HINT=0/1 overrides
        const char* hv = getenv("GCP_L2_HINT");
        c->l2_first = hv ? atoi(hv) != 0 : spills;
        c->ag_stride = il ? 2 * c->R_pad : c->R_pad;
        // slot ordering by mode-1 position: pays when mode 1's A and G rows
        // themselves spill out of L2 (c4, c5); GCP_SLOT_ORDER=0/1 overrides
        // (and, decided per iteration in gcp_loss_grad, when the order array of
        // the iteration's slots fits L2: c5's 2e8 slots ordered cost more than
        // they saved, profiles/r02_summary.md)
        const char* oenv = getenv("GCP_SLOT_ORDER");
        const bool m1_spills = 2.0 * (double)c->rows[0] * (double)rb > 0.25 * (double)c->l2_bytes;
        c->slot_order = oenv ? atoi(oenv) != 0 : m1_spills;
        c->slot_order_forced = oenv && atoi(oenv) != 0;
    }
    const size_t bytes = (size_t)std::max<int64_t>(c->n_coef, 4) * tsz(c);
    // sync: the fused NVLink exchange; two-sided: the device-driven import /
    // export (twosided_nvl.cu); both keep A, G, G2 in symmetric NVLink windows
    const bool use_fused = fused_possible(c) || tsn_possible(c);
    if (use_fused) ST_TRY(fused_alloc(c, bytes));
    c->tsn_peer = false;
    if (use_fused && two_sided(c)) {
        if (tsn_peer_wanted(c)) ST_TRY(tsn_peer_setup(c));   // K2 reaches the owners' rows directly
        else ST_TRY(tsn_alloc_bitmap(c));
    }
    {
        void** bufs[] = {&c->d_A, &c->d_B, &c->d_C};
        for (void** b : bufs) {
            if (use_fused && b == &c->d_A) continue;
            cudaError_t e = gmalloc(c, b, b == &c->d_A && c->ag_interleaved ? 2 * bytes : bytes);
            if (e != cudaSuccess) {
                cudaGetLastError();
                free_model(c);
                return set_error(GCP_E_OOM, "gcp_model_init: out of device memory");
            }
        }
        if (c->ag_interleaved) {
            c->d_G = (char*)c->d_A + (size_t)c->R_pad * tsz(c);   // view: G rows interleaved with A rows
        } else if (use_fused) {
            CUDA_TRY(c, cudaMemsetAsync(c->d_G2, 0, bytes, c->stream), "model init");
        } else {
            cudaError_t e = gmalloc(c, &c->d_G, bytes);
            if (e != cudaSuccess) {
                cudaGetLastError();
                free_model(c);
                return set_error(GCP_E_OOM, "gcp_model_init: out of device memory");
            }
        }
    }
    CUDA_TRY(c, gmalloc(c, &c->d_lambda, (size_t)c->R_pad * tsz(c)), "model lambda");
    CUDA_TRY(c, cudaMemsetAsync(c->ag_interleaved ? c->d_A : c->d_G, 0, c->ag_interleaved ? 2 * bytes : bytes,
                                c->stream),
             "model init");
    CUDA_TRY(c, cudaMemsetAsync(c->d_B, 0, bytes, c->stream), "model init");
    CUDA_TRY(c, cudaMemsetAsync(c->d_C, 0, bytes, c->stream), "model init");
    {
        std::vector<double> lam64(c->R_pad, 0.0);
        std::vector<float> lam32(c->R_pad, 0.0f);
        for (int r = 0; r < R; ++r) lam64[r] = lam32[r] = 1.0;
        const void* src = c->prec == GCP_FP32 ? (const void*)lam32.data() : (const void*)lam64.data();
        CUDA_TRY(c, cudaMemcpyAsync(c->d_lambda, src, (size_t)c->R_pad * tsz(c), cudaMemcpyHostToDevice, c->stream),
                 "lambda");
        int64_t goff[kMaxModes] = {0};
        int64_t acc = 0;
        for (int k = 0; k < c->d; ++k) {
            goff[k] = acc;
            acc += c->dims[k] * R;
        }
        cudaEvent_t ev;
        prof_begin(c, PROF_OTHER, &ev);
        CUDA_TRY(c, launch_init(c, seed, goff), "factor init");
        prof_end(c, PROF_OTHER, ev);
        CUDA_TRY(c, cudaStreamSynchronize(c->stream), "model init");
    }
    c->t = 0;
    c->ts = 0;
    c->it = 0;
    c->ord_stage = 0;
    c->grad_blocks = sample_kernel_blocks(c);
    ST_TRY(ensure_partials(c, c->grad_blocks));
    c->have_model = true;
    c->have_grad = false;
    c->tsn_dirty = true;      // peer access: a barrier before any member reads these rows
    return server_reset(c);   // FedAdam: U <- M0 (Alg. 4)
}

gcp_status gcp_model_set(gcp_ctx* c, int k, const double* rows, const double* lambda) {
    ENTER(c);
    if (!c->have_model) return set_error(GCP_E_STATE, "gcp_model_set: no model");
    if (k < 0 || k >= c->d) return set_error(GCP_E_RANGE, "gcp_model_set: mode out of range");
    if (!rows) return set_error(GCP_E_ARG, "gcp_model_set: rows NULL");
    const int64_t b = c->hi[k] - c->lo[k];
    // H2D of the packed fp64 rows, then widen / narrow and pad on the device
    double* d_rows = nullptr;
    CUDA_TRY(c, gmalloc(c, &d_rows, (size_t)std::max<int64_t>(b, 1) * c->R * 8), "model_set");
    CUDA_TRY(c, cudaMemcpyAsync(d_rows, rows, (size_t)b * c->R * 8, cudaMemcpyHostToDevice, c->stream), "model_set");
    CUDA_TRY(c, launch_rows_in(c, d_rows, (char*)c->d_A + (size_t)phys_off(c, k) * tsz(c), b), "model_set");
    gfree(c, d_rows);
    CUDA_TRY(c, cudaStreamSynchronize(c->stream), "model_set");
    if (lambda) {
        std::vector<double> l64(c->R_pad, 0.0);
        std::vector<float> l32(c->R_pad, 0.f);
        for (int r = 0; r < c->R; ++r) {
            l64[r] = lambda[r];
            l32[r] = (float)lambda[r];
        }
        const void* src = c->prec == GCP_FP32 ? (const void*)l32.data() : (const void*)l64.data();
        CUDA_TRY(c, cudaMemcpyAsync(c->d_lambda, src, (size_t)c->R_pad * tsz(c), cudaMemcpyHostToDevice, c->stream),
                 "model_set lambda");
        CUDA_TRY(c, cudaStreamSynchronize(c->stream), "model_set");
    }
    c->tsn_dirty = true;
    return server_reset(c);   // FedAdam: the server copy starts from the model as set
}

// rows of A or G (row stride ag_stride) of mode k's block as packed fp64 rows (b x R) in host memory
static gcp_status read_rows(gcp_ctx* c, const void* base, int k, double* out, const char* what) {
    const int64_t b = c->hi[k] - c->lo[k];
    // pack and widen to fp64 on the device, then one contiguous D2H into the caller's rows
    double* d_rows = nullptr;
    CUDA_TRY(c, gmalloc(c, &d_rows, (size_t)std::max<int64_t>(b, 1) * c->R * 8), what);
    CUDA_TRY(c, launch_rows_out(c, (const char*)base + (size_t)phys_off(c, k) * tsz(c), d_rows, b), what);
    CUDA_TRY(c, cudaMemcpyAsync(out, d_rows, (size_t)b * c->R * 8, cudaMemcpyDeviceToHost, c->stream), what);
    gfree(c, d_rows);
    CUDA_TRY(c, cudaStreamSynchronize(c->stream), what);
    return GCP_OK;
}

gcp_status gcp_model_get(gcp_ctx* c, int k, double* rows_out) {
    ENTER(c);
    if (!c->have_model) return set_error(GCP_E_STATE, "gcp_model_get: no model");
    if (k < 0 || k >= c->d) return set_error(GCP_E_RANGE, "gcp_model_get: mode out of range");
    if (!rows_out) return set_error(GCP_E_ARG, "gcp_model_get: NULL");
    if (two_sided(c)) ST_TRY(dist_sync_exchange_post(c));   // all-gather the owned rows (collective)
    return read_rows(c, c->d_A, k, rows_out, "model_get");
}

gcp_status gcp_grad_get(gcp_ctx* c, int k, double* out) {
    ENTER(c);
    if (!c->have_model) return set_error(GCP_E_STATE, "gcp_grad_get: no model");
    if (k < 0 || k >= c->d) return set_error(GCP_E_RANGE, "gcp_grad_get: mode out of range");
    if (!out) return set_error(GCP_E_ARG, "gcp_grad_get: NULL");
    ST_TRY(check_err(c, "gcp_grad_get"));
    return read_rows(c, cur_G(c), k, out, "grad_get");
}

gcp_status gcp_sample(gcp_ctx* c, gcp_strategy strategy, int64_t s_nz, int64_t s_z, uint64_t seed) {
    ENTER(c);
    if (!c->have_tensor) return set_error(GCP_E_STATE, "gcp_sample: no tensor");
    if (strategy != GCP_STRATIFIED && strategy != GCP_SEMI_STRATIFIED)
        return set_error(GCP_E_ARG, "gcp_sample: bad strategy");
    if (s_nz < 0 || s_z < 0 || s_nz + s_z == 0) return set_error(GCP_E_ARG, "gcp_sample: need p, q >= 0, p + q > 0");
    if (s_nz > 0 && c->N_global == 0) return set_error(GCP_E_NO_NONZEROS, "gcp_sample: tensor has no nonzeros");
    if (s_z > 0 && strategy == GCP_STRATIFIED && !c->any_zero_global)
        return set_error(GCP_E_NO_ZEROS, "gcp_sample: tensor has no zeros");
    int64_t p_w, q_w;
    local_counts(c, s_nz, s_z, &p_w, &q_w);
    if (p_w >= (int64_t)1 << 32 || q_w >= (int64_t)1 << 32)
        return set_error(GCP_E_ARG, "gcp_sample: >= 2^32 slots per rank");
    c->strategy = strategy;
    c->s_nz = s_nz;
    c->s_z = s_z;
    c->p_w = p_w;
    c->q_w = q_w;
    c->seed = seed;
    c->bound = true;
    c->ord_stage = 0;
    graph_drop(c);
    return GCP_OK;
}

gcp_status gcp_sample_export(gcp_ctx* c, int stratum, int64_t first, int64_t count, int64_t* subs_out,
                             int64_t* j_out, double* w_out, int32_t* attempts_out) {
    ENTER(c);
    if (!c->bound) return set_error(GCP_E_STATE, "gcp_sample_export: call gcp_sample first");
    if (stratum != 0 && stratum != 1) return set_error(GCP_E_ARG, "gcp_sample_export: stratum must be 0 or 1");
    const int64_t n = stratum == 0 ? c->p_w : c->q_w;
    if (first < 0 || count < 0 || first + count > n) return set_error(GCP_E_RANGE, "gcp_sample_export: slot range");
    if (!subs_out) return set_error(GCP_E_ARG, "gcp_sample_export: subs_out NULL");
    if (count == 0) return GCP_OK;
    const int stratified = c->strategy == GCP_STRATIFIED;
    const SampleArgs s = sample_args(c, c->p_w, c->q_w, c->seed, c->it, KIND_GRAD_NZ, KIND_GRAD_Z, stratified);
    int64_t *d_subs = nullptr, *d_j = nullptr, *d_lo = nullptr;
    int32_t* d_att = nullptr;
    CUDA_TRY(c, gmalloc(c, &d_subs, sizeof(int64_t) * count * c->d), "export");
    CUDA_TRY(c, gmalloc(c, &d_j, sizeof(int64_t) * count), "export");
    CUDA_TRY(c, gmalloc(c, &d_att, sizeof(int32_t) * count), "export");
    CUDA_TRY(c, gmalloc(c, &d_lo, sizeof(int64_t) * kMaxModes), "export");
    CUDA_TRY(c, cudaMemcpyAsync(d_lo, c->lo, sizeof(int64_t) * kMaxModes, cudaMemcpyHostToDevice, c->stream), "export");
    cudaEvent_t ev;
    prof_begin(c, PROF_OTHER, &ev);
    CUDA_TRY(c, launch_export(c, s, stratum, (stratum == 0 ? 0 : c->p_w) + first, count, d_lo, d_subs, d_j, d_att),
             "export");
    prof_end(c, PROF_OTHER, ev);
    CUDA_TRY(c, cudaMemcpyAsync(subs_out, d_subs, sizeof(int64_t) * count * c->d, cudaMemcpyDeviceToHost, c->stream),
             "export");
    if (j_out) CUDA_TRY(c, cudaMemcpyAsync(j_out, d_j, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, c->stream), "export");
    if (attempts_out)
        CUDA_TRY(c, cudaMemcpyAsync(attempts_out, d_att, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, c->stream),
                 "export");
    CUDA_TRY(c, cudaStreamSynchronize(c->stream), "export");
    gfree(c, d_subs);
    gfree(c, d_j);
    gfree(c, d_att);
    gfree(c, d_lo);
    if (w_out) {
        const double w = stratum == 0 ? weight_nz(c, c->p_w) : weight_z(c, c->q_w);
        for (int64_t i = 0; i < count; ++i) w_out[i] = w;
    }
    return check_err(c, "gcp_sample_export");
}

gcp_status gcp_loss_grad(gcp_ctx* c, gcp_loss loss, double* sampled_loss_out) {
    ENTER(c);
    NvtxRange nvtx_("gcp_loss_grad");
    if (!c->have_model || !c->bound) return set_error(GCP_E_STATE, "gcp_loss_grad: need model and gcp_sample");
    if (!valid_loss(loss)) return set_error(GCP_E_ARG, "gcp_loss_grad: bad loss");
    // async schemes: averaging / server step before this iteration's sampling (Alg. 3-4)
    if (async_family(c) && c->tau > 0 && ((int64_t)c->it + 1) % c->tau == 0 && !c->have_grad)
        ST_TRY(dist_async_sync(c));
    c->last_loss = loss;
    const int stratified = c->strategy == GCP_STRATIFIED;
    const SampleArgs s = sample_args(c, c->p_w, c->q_w, c->seed, c->it, KIND_GRAD_NZ, KIND_GRAD_Z, stratified);
    // two-sided layout (row f3): touch pass + import of the rows owned elsewhere
    if (two_sided(c) && !c->have_grad && !c->tsn_peer) ST_TRY(c->fused ? tsn_import(c, s) : twosided_import(c, s));
    ST_TRY(tsn_peer_sync(c));
    const ModelArgs m = model_args(c);
    const int with_loss = sampled_loss_out != nullptr;
    cudaEvent_t ev;
    SampleArgs so = s;
    // slot ids are u32: beyond 2^32 slots per rank K2 runs in slot order
    const int64_t n_slots = c->p_w + c->q_w;
    const bool order_fits = c->slot_order_forced || (double)n_slots * 4.0 <= 0.8 * (double)c->l2_bytes;
    if (c->slot_order && n_slots < ((int64_t)1 << 32) && order_fits) {
        // group this iteration's slots by mode-1 position (same sample set, other
        // visiting order), so the K2 gathers / scatter-adds of one mode-1 row meet
        // in L2 (kernels.cu launch_slot_order: hand-written histogram / scan / scatter)
        if (n_slots > c->ord_cap && !c->capturing) {
            ord_free(c);
            // a visiting-order optimisation only: without the memory for it, K2
            // runs in slot order
            if (gmalloc(c, &c->d_ord_buf, slot_order_bytes(n_slots)) != cudaSuccess) {
                cudaGetLastError();
                c->d_ord_buf = nullptr;
                c->slot_order = 0;
            } else {
                CUDA_TRY(c, slot_order_init(c, c->d_ord_buf, n_slots), "slot order");
                c->ord_cap = n_slots;
            }
        }
        if (c->slot_order && n_slots <= c->ord_cap) {
            // the previous iteration's K2 / Adam may have prepared this order
            const int stage = c->ord_stage_it == c->it ? c->ord_stage : 0;
            if (stage < 2) {
                prof_begin(c, PROF_OTHER, &ev);
                CUDA_TRY(c, launch_slot_order(c, s, &so.order, stage), "slot order");
                prof_end(c, PROF_OTHER, ev);
            } else {
                so.order = c->d_ord;
            }
        }
    }
    c->ord_stage = 0;
    // the gradient K2 carries the next iteration's slot histogram
    OrdHistArgs oh;
    bool carry = false;
    if (so.order) {
        const SampleArgs nx = sample_args(c, c->p_w, c->q_w, c->seed, c->it + 1, KIND_GRAD_NZ, KIND_GRAD_Z, stratified);
        carry = ord_hist_args(c, nx, &oh);
    }
    prof_begin(c, PROF_GRAD, &ev);
    CUDA_TRY(c, launch_sample_kernel(c, so, m, loss, 0, !stratified, weight_nz(c, c->p_w), weight_z(c, c->q_w),
                                     with_loss, c->d_partials, c->grad_blocks, carry ? &oh : nullptr),
             "gcp_loss_grad");
    prof_end(c, PROF_GRAD, ev);
    if (carry) {
        c->ord_stage = 1;
        c->ord_stage_it = c->it + 1;
    }
    c->have_grad = true;
    if (with_loss) {
        prof_begin(c, PROF_OTHER, &ev);
        CUDA_TRY(c, launch_reduce_partials(c, c->d_partials, c->grad_blocks, (double*)c->d_partials + c->partials_cap),
                 "reduce");
        prof_end(c, PROF_OTHER, ev);
        CUDA_TRY(c, cudaMemcpyAsync(c->h_scalar, (double*)c->d_partials + c->partials_cap, 8, cudaMemcpyDeviceToHost,
                                    c->stream),
                 "gcp_loss_grad");
        ST_TRY(check_err(c, "gcp_loss_grad"));
        *sampled_loss_out = *c->h_scalar;
    }
    return GCP_OK;
}

gcp_status gcp_adam_step(gcp_ctx* c, const gcp_adam_params* p) {
    ENTER(c);
    NvtxRange nvtx_("gcp_adam_step");
    if (!p) return set_error(GCP_E_ARG, "gcp_adam_step: NULL params");
    if (!c->have_grad) return set_error(GCP_E_STATE, "gcp_adam_step: no gradient (call gcp_loss_grad)");
    if (!(p->beta1 >= 0 && p->beta1 < 1 && p->beta2 >= 0 && p->beta2 < 1 && p->eps > 0 && p->rate >= 0))
        return set_error(GCP_E_ARG, "gcp_adam_step: need 0 <= beta < 1, eps > 0, rate >= 0");
    const double lower = std::isnan(p->lower) ? loss_lower(c->last_loss) : p->lower;
    c->t += 1;
    if (c->fused) {   // sync P > 1: reduce-scatter + Adam + all-gather in one NVLink kernel;
                      // two-sided: export of the touched rows + Adam on the owned rows
        ST_TRY(!two_sided(c) ? fused_exchange(c, p, lower) : c->tsn_peer ? tsn_peer_step(c, p, lower)
                                                                         : tsn_export(c, p, lower));
        c->it += 1;
        c->have_grad = false;
        return GCP_OK;
    }
    Segment seg;
    seg.n = 0;
    const bool sharded = c->P > 1 && sync_family(c);
    if (two_sided(c)) {
        // row f3: imported rows' G back to their owners; Adam on the owned rows only
        ST_TRY(twosided_export(c));
        for (int k = 0; k < c->d; ++k) {
            const int64_t shard = c->rows[k] / c->slice_size[k];
            seg.start[seg.n] = c->off[k] + (int64_t)c->slice_rank[k] * shard * c->R_pad;
            seg.len[seg.n] = shard * c->R_pad;
            seg.n++;
        }
    } else if (sharded) {
        ST_TRY(dist_sync_exchange_pre(c));
        for (int k = 0; k < c->d; ++k) {
            if (c->ar_mode[k] || c->slice_size[k] <= 1) {   // replicated rows, all-reduced G
                seg.start[seg.n] = c->off[k];
                seg.len[seg.n] = c->rows[k] * c->R_pad;
            } else {                                         // owned shard of reduce-scattered G
                const int64_t shard = c->rows[k] / c->slice_size[k];
                seg.start[seg.n] = c->off[k] + (int64_t)c->slice_rank[k] * shard * c->R_pad;
                seg.len[seg.n] = shard * c->R_pad;
            }
            seg.n++;
        }
    } else {
        seg.start[0] = 0;
        seg.len[0] = c->n_coef;
        seg.n = 1;
    }
    // the next iteration's slot-order scan (launched here) and scatter (carried
    // by this memory-bound Adam launch), when its histogram is ready
    OrdScatterArgs os;
    bool carry = false;
    cudaEvent_t ev;
    if (c->ord_stage == 1 && c->ord_stage_it == c->it + 1) {
        int64_t vecs = 0;
        for (int i = 0; i < seg.n; ++i) vecs += seg.len[i] / (c->prec == GCP_FP32 ? 4 : 2);
        prof_begin(c, PROF_OTHER, &ev);
        carry = ord_scatter_args(c, c->p_w + c->q_w, &os, vecs);
        prof_end(c, PROF_OTHER, ev);
    }
    prof_begin(c, PROF_ADAM, &ev);
    CUDA_TRY(c, launch_adam(c, seg, c->d_A, c->d_G, c->d_B, c->d_C, p->rate, p->beta1, p->beta2, p->eps, lower,
                            c->capturing ? c->t - c->graph_t0 : c->t, sharded ? 0 : 1, c->ag_stride,
                            c->capturing ? c->d_step : nullptr, carry ? &os : nullptr),
             "gcp_adam_step");
    prof_end(c, PROF_ADAM, ev);
    if (carry) c->ord_stage = 2;
    if (sharded) {
        CUDA_TRY(c, cudaMemsetAsync(c->d_G, 0, (size_t)c->n_coef * tsz(c), c->stream), "adam G reset");
        if (!two_sided(c)) ST_TRY(dist_sync_exchange_post(c));   // two-sided: rows stay partitioned
    }
    c->it += 1;
    c->have_grad = false;
    return GCP_OK;
}

gcp_status gcp_loss_estimate(gcp_ctx* c, gcp_loss loss, int64_t f_nz, int64_t f_z, uint64_t seed, double* out) {
    ENTER(c);
    NvtxRange nvtx_("gcp_loss_estimate");
    if (!c->have_model) return set_error(GCP_E_STATE, "gcp_loss_estimate: no model");
    if (!valid_loss(loss)) return set_error(GCP_E_ARG, "gcp_loss_estimate: bad loss");
    if (!out || f_nz < 0 || f_z < 0 || f_nz + f_z == 0) return set_error(GCP_E_ARG, "gcp_loss_estimate: args");
    if (f_nz > 0 && c->N_global == 0) return set_error(GCP_E_NO_NONZEROS, "gcp_loss_estimate: no nonzeros");
    if (f_z > 0 && !c->any_zero_global) return set_error(GCP_E_NO_ZEROS, "gcp_loss_estimate: no zeros");
    int64_t p, q;
    local_counts(c, f_nz, f_z, &p, &q);
    double* dout = (double*)c->d_partials + c->partials_cap;
    // f-samples read any block row: refresh them (peer access reads the owners' rows)
    if (two_sided(c) && !c->tsn_peer) ST_TRY(dist_sync_exchange_post(c));
    ST_TRY(tsn_peer_sync(c));
    ST_TRY(run_loss_kernel(c, loss, p, q, seed, 0xFFFFFFFFu, KIND_F_NZ, KIND_F_Z, 1, 0, PROF_LOSS, 1, dout));
    if (c->P > 1) ST_TRY(dist_allreduce_scalar(c, dout));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_scalar, dout, 8, cudaMemcpyDeviceToHost, c->stream), "loss_estimate");
    ST_TRY(check_err(c, "gcp_loss_estimate"));
    *out = *c->h_scalar;
    return GCP_OK;
}

gcp_status gcp_fit_begin(gcp_ctx* c, const gcp_fit_params* p, double* initial_est) {
    ENTER(c);
    NvtxRange nvtx_("gcp_fit_begin");
    if (!p) return set_error(GCP_E_ARG, "gcp_fit_begin: NULL params");
    if (!c->have_model) return set_error(GCP_E_STATE, "gcp_fit_begin: no model");
    if (p->epochs < 0 || p->iters_per_epoch < 1 || p->max_fails < 1 || !(p->decay >= 0) || !valid_loss(p->loss))
        return set_error(GCP_E_ARG, "gcp_fit_begin: bad epoch parameters");
    if (async_family(c) && p->tau < 1) return set_error(GCP_E_ARG, "gcp_fit_begin: async needs tau >= 1");
    ST_TRY(gcp_sample(c, p->strategy, p->s_nz, p->s_z, p->seed));
    c->fp = *p;
    c->rate = p->adam.rate;
    c->fails = 0;
    c->epoch = 0;
    c->last_loss = p->loss;
    if (async_family(c)) {
        c->tau = p->tau;
        if (!c->server_set) {
            c->server = p->adam;
            c->server.rate = p->meta_rate > 0 ? p->meta_rate : p->adam.rate;
        }
    }
    ST_TRY(server_reset(c));
    double est;
    ST_TRY(gcp_loss_estimate(c, p->loss, p->f_nz, p->f_z, p->fseed, &est));
    c->best = est;
    ST_TRY(checkpoint_save(c));
    c->fit_active = true;
    if (initial_est) *initial_est = est;
    return GCP_OK;
}

// An epoch's iterations (K2 + Adam / exchange) are one CUDA graph:
// captured once per schedule, replayed with the step state (t0, it0, rate)
// uploaded to device memory; each captured launch adds its own offset, so the
// replay needs no host work per iteration.  Not used on
// the legacy stream (uncapturable), while profiling (per-kernel events), for
// the NCCL two-sided layout (host-sized transfers; the device-driven one over
// NVLink windows replays) or FedAdam (host server clock).
static bool graph_ok(const gcp_ctx* c) {
    const char* env = getenv("GCP_GRAPHS");
    if (env && atoi(env) == 0) return false;
    return c->stream != nullptr && !c->prof_on && (!two_sided(c) || c->fused) && c->mode != GCP_DIST_ASYNC_FEDADAM;
}

static gcp_status epoch_graph(gcp_ctx* c, gcp_loss loss, const gcp_adam_params& ap, int iters) {
    if (!c->d_step) {
        CUDA_TRY(c, gmalloc(c, &c->d_step, sizeof(DevStep)), "step state");
        CUDA_TRY(c, cudaMallocHost(&c->h_step, sizeof(DevStep)), "step state");
    }
    const double lower = std::isnan(ap.lower) ? loss_lower(loss) : ap.lower;
    const int64_t period = 2 * std::max<int64_t>(c->tau, 1);   // G parity and the async schedule
    const double key[8] = {(double)iters, (double)((int64_t)c->it % period), ap.beta1, ap.beta2, ap.eps, lower,
                           (double)loss, (double)c->fused};
    const uint32_t it0 = c->it;
    const int64_t t0 = c->t;
    ST_TRY(tsn_peer_sync(c));   // outside the graph: owed after a restore
    if (!c->graph_exec || memcmp(key, c->graph_key, sizeof(key)) != 0) {
        graph_drop(c);
        // a schedule seen once runs eagerly (a one-epoch job would pay the
        // capture and instantiation for nothing); the second sighting captures
        if (!c->graph_seen_valid || memcmp(key, c->graph_seen, sizeof(key)) != 0) {
            memcpy(c->graph_seen, key, sizeof(key));
            c->graph_seen_valid = true;
            for (int i = 0; i < iters; ++i) {
                ST_TRY(gcp_loss_grad(c, loss, nullptr));
                ST_TRY(gcp_adam_step(c, &ap));
            }
            return GCP_OK;
        }
        const int64_t l0 = c->launches;
        c->graph_it0 = it0;
        c->graph_t0 = t0;
        CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "graph capture");
        c->capturing = true;
        gcp_status st = GCP_OK;
        for (int i = 0; i < iters && st == GCP_OK; ++i) {
            st = gcp_loss_grad(c, loss, nullptr);
            if (st == GCP_OK) st = gcp_adam_step(c, &ap);
        }
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        c->capturing = false;
        c->graph_launches = c->launches - l0;
        c->launches = l0;
        c->it = it0;
        c->t = t0;
        c->have_grad = false;
        if (st != GCP_OK || e != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            if (st != GCP_OK) return st;
            return cuda_fail(c, e, "graph capture");
        }
        const cudaError_t ei = cudaGraphInstantiate(&c->graph_exec, g, 0);
        cudaGraphDestroy(g);
        if (ei != cudaSuccess) {
            c->graph_exec = nullptr;
            return cuda_fail(c, ei, "graph instantiate");
        }
        memcpy(c->graph_key, key, sizeof(key));
    }
    DevStep* h = c->h_step;
    h->rate = ap.rate;
    h->beta1 = ap.beta1;
    h->beta2 = ap.beta2;
    h->t = t0;
    h->it = it0;
    h->pad = 0;
    CUDA_TRY(c, cudaMemcpyAsync(c->d_step, h, sizeof(DevStep), cudaMemcpyHostToDevice, c->stream), "step state");
    CUDA_TRY(c, cudaGraphLaunch(c->graph_exec, c->stream), "graph launch");
    c->it = it0 + (uint32_t)iters;
    c->t = t0 + iters;
    c->launches += c->graph_launches;
    c->have_grad = false;
    return GCP_OK;
}

gcp_status gcp_fit_epoch(gcp_ctx* c, double* est_out, int* accepted_out, int* done_out) {
    ENTER(c);
    NvtxRange nvtx_("gcp_fit_epoch");
    if (!c->fit_active) return set_error(GCP_E_STATE, "gcp_fit_epoch: call gcp_fit_begin first");
    const gcp_fit_params& p = c->fp;
    if (c->epoch >= p.epochs || c->fails >= p.max_fails) {
        if (done_out) *done_out = 1;
        return GCP_OK;
    }
    gcp_adam_params ap = p.adam;
    ap.rate = c->rate;
    if (graph_ok(c))
        ST_TRY(epoch_graph(c, p.loss, ap, p.iters_per_epoch));
    else
        for (int i = 0; i < p.iters_per_epoch; ++i) {
            ST_TRY(gcp_loss_grad(c, p.loss, nullptr));
            ST_TRY(gcp_adam_step(c, &ap));
        }
    double est;
    ST_TRY(gcp_loss_estimate(c, p.loss, p.f_nz, p.f_z, p.fseed, &est));
    int accepted = est < c->best;
    if (accepted) {
        c->best = est;
        ST_TRY(checkpoint_save(c));
    } else {
        ST_TRY(checkpoint_restore(c));
        c->rate *= p.decay;
        c->fails += 1;
    }
    c->epoch += 1;
    if (est_out) *est_out = est;
    if (accepted_out) *accepted_out = accepted;
    if (done_out) *done_out = (c->epoch >= p.epochs || c->fails >= p.max_fails) ? 1 : 0;
    return GCP_OK;
}

gcp_status gcp_fit(gcp_ctx* c, const gcp_fit_params* p, gcp_trace_fn trace, void* user, double* final_est_loss) {
    ENTER(c);
    const auto t0 = std::chrono::steady_clock::now();
    double est;
    ST_TRY(gcp_fit_begin(c, p, &est));
    int done = p->epochs == 0;
    while (!done) {
        int acc;
        ST_TRY(gcp_fit_epoch(c, &est, &acc, &done));
        if (trace) {
            const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            trace(user, c->epoch, (int64_t)c->it, est, c->rate, el);
        }
    }
    if (final_est_loss) *final_est_loss = c->best;
    c->fit_active = false;
    return GCP_OK;
}

gcp_status gcp_dist_features(gcp_ctx* c, int* fused_out, int* multimem_out) {
    ENTER(c);
    if (fused_out) *fused_out = c->fused ? 1 : 0;
    int mm = 0;
    for (int k = 0; k < c->d; ++k) mm |= fused_use_multimem(c) && c->fnmem[k] == c->P;
    if (multimem_out) *multimem_out = mm;
    return GCP_OK;
}

gcp_status gcp_layout(gcp_ctx* c, int* ag_interleaved, int* slot_order, int* filter) {
    ENTER(c);
    if (ag_interleaved) *ag_interleaved = c->have_model && c->ag_interleaved ? 1 : 0;
    const bool order_fits = c->slot_order_forced || !c->bound ||
                            (double)(c->p_w + c->q_w) * 4.0 <= 0.8 * (double)c->l2_bytes;
    if (slot_order) *slot_order = c->have_model && c->slot_order && order_fits ? 1 : 0;
    if (filter) *filter = c->have_tensor && c->filter_sectors ? 1 : 0;
    return GCP_OK;
}

gcp_status gcp_debug_nonzero_j(gcp_ctx* c, uint64_t seed, uint32_t rank, uint32_t it, int64_t N, int64_t first,
                               int64_t count, int64_t* j_out) {
    ENTER(c);
    if (!c->have_tensor || c->N < 1) return set_error(GCP_E_STATE, "gcp_debug_nonzero_j: need a tensor with nonzeros");
    if (N < 1 || first < 0 || count < 0 || first + count > ((int64_t)1 << 32) || !j_out)
        return set_error(GCP_E_ARG, "gcp_debug_nonzero_j: args");
    if (count == 0) return GCP_OK;
    // the device draw path (issue_sample + resolve_sample) with a pretend nonzero
    // count N; a record stride of 0 points every draw at record 0, so no tensor
    // of N nonzeros is needed
    SampleArgs s = sample_args(c, first + count, 0, seed, it, KIND_GRAD_NZ, KIND_GRAD_Z, 1);
    s.rank = rank;
    s.N = N;
    s.rec_words = 0;
    int64_t *d_subs = nullptr, *d_j = nullptr, *d_lo = nullptr;
    CUDA_TRY(c, gmalloc(c, &d_subs, sizeof(int64_t) * count * c->d), "debug_j");
    CUDA_TRY(c, gmalloc(c, &d_j, sizeof(int64_t) * count), "debug_j");
    CUDA_TRY(c, gmalloc(c, &d_lo, sizeof(int64_t) * kMaxModes), "debug_j");
    CUDA_TRY(c, cudaMemsetAsync(d_lo, 0, sizeof(int64_t) * kMaxModes, c->stream), "debug_j");
    CUDA_TRY(c, launch_export(c, s, 0, first, count, d_lo, d_subs, d_j, nullptr), "debug_j");
    CUDA_TRY(c, cudaMemcpyAsync(j_out, d_j, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, c->stream), "debug_j");
    CUDA_TRY(c, cudaStreamSynchronize(c->stream), "debug_j");
    gfree(c, d_subs);
    gfree(c, d_j);
    gfree(c, d_lo);
    return GCP_OK;
}

gcp_status gcp_debug_philox(gcp_ctx* c, int64_t n, const uint32_t* ctr_key, uint32_t* out) {
    ENTER(c);
    if (n < 0 || (n > 0 && (!ctr_key || !out))) return set_error(GCP_E_ARG, "gcp_debug_philox: args");
    if (n == 0) return GCP_OK;
    uint32_t *d_in = nullptr, *d_out = nullptr;
    CUDA_TRY(c, gmalloc(c, &d_in, (size_t)n * 6 * 4), "debug_philox");
    CUDA_TRY(c, gmalloc(c, &d_out, (size_t)n * 8 * 4), "debug_philox");
    CUDA_TRY(c, cudaMemcpyAsync(d_in, ctr_key, (size_t)n * 6 * 4, cudaMemcpyHostToDevice, c->stream), "debug_philox");
    CUDA_TRY(c, launch_debug_philox(c, n, d_in, d_out), "debug_philox");
    CUDA_TRY(c, cudaMemcpyAsync(out, d_out, (size_t)n * 8 * 4, cudaMemcpyDeviceToHost, c->stream), "debug_philox");
    CUDA_TRY(c, cudaStreamSynchronize(c->stream), "debug_philox");
    gfree(c, d_in);
    gfree(c, d_out);
    return GCP_OK;
}

gcp_status gcp_counters(gcp_ctx* c, uint32_t* it, int64_t* t, int64_t* launches) {
    if (!c) return set_error(GCP_E_ARG, "null context");
    if (it) *it = c->it;
    if (t) *t = c->t;
    if (launches) *launches = c->launches;
    return GCP_OK;
}

gcp_status gcp_profile_enable(gcp_ctx* c, int on) {
    ENTER(c);
    c->prof_on = on != 0;
    return GCP_OK;
}

gcp_status gcp_profile_get(gcp_ctx* c, int which, double* ms, int64_t* launches, int reset) {
    ENTER(c);
    if (which < 0 || which >= PROF_N) return set_error(GCP_E_ARG, "gcp_profile_get: bad kernel class");
    prof_resolve(c);
    if (ms) *ms = c->prof_ms[which];
    if (launches) *launches = c->prof_n[which];
    if (reset) {
        c->prof_ms[which] = 0;
        c->prof_n[which] = 0;
    }
    return GCP_OK;
}

gcp_status gcp_grid_plan(int P, int d, const int64_t* dims, int* grid_out, int64_t* lo_out, int64_t* hi_out) {
    if (P < 1 || d < 1 || d > kMaxModes || !dims || !grid_out) return set_error(GCP_E_ARG, "gcp_grid_plan: args");
    for (int k = 0; k < d; ++k)
        if (dims[k] < 1) return set_error(GCP_E_ARG, "gcp_grid_plan: dims");
    // enumerate ordered divisor tuples in lexicographic order; strict < keeps the first minimum
    int cur[kMaxModes];
    double best = INFINITY;
    std::vector<int> divs;
    for (int n = 1; n <= P; ++n)
        if (P % n == 0) divs.push_back(n);
    std::vector<int> idx(d, 0);
    for (;;) {
        int64_t prod = 1;
        for (int k = 0; k < d; ++k) prod *= divs[idx[k]];
        if (prod == P) {
            double obj = 0;
            for (int k = 0; k < d; ++k) obj += (double)dims[k] * (double)(P / divs[idx[k]]);
            if (obj < best) {
                best = obj;
                for (int k = 0; k < d; ++k) cur[k] = divs[idx[k]];
            }
        }
        int k = d - 1;
        while (k >= 0 && ++idx[k] == (int)divs.size()) idx[k--] = 0;
        if (k < 0) break;
    }
    for (int k = 0; k < d; ++k) grid_out[k] = cur[k];
    if (lo_out || hi_out) {
        for (int w = 0; w < P; ++w) {
            int rem = w, b[kMaxModes];
            for (int k = d - 1; k >= 0; --k) {
                b[k] = rem % cur[k];
                rem /= cur[k];
            }
            for (int k = 0; k < d; ++k) {
                const int64_t ck = (dims[k] + cur[k] - 1) / cur[k];
                if (lo_out) lo_out[w * d + k] = std::min<int64_t>(b[k] * ck, dims[k]);
                if (hi_out) hi_out[w * d + k] = std::min<int64_t>((b[k] + 1) * ck, dims[k]);
            }
        }
    }
    return GCP_OK;
}

}  // extern "C"
