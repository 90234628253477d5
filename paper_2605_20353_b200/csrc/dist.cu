// dist.cu -- rows a6 / a8 for nranks > 1: NCCL over NVLink/NVSwitch.
//
// Sync (Alg. 2): per iteration and mode k, the G^(k)
// block rows are reduce-scattered over the mode-k slice communicator (ranks
// sharing grid coordinate b_k), Adam runs on the owned 1/g_k shard
// (moments sharded too, so the paper's "limited parallelism in ... Adam"
// of the all-reduce layout, is removed), and the updated rows are
// all-gathered.  Mathematically this is Allreduce(G) + replicated Adam.
// Async (Alg. 3, reading R16): every tau iterations each A^(k)
// block is all-reduced over its slice group and scaled by 1/g_k.
// FedAdam (Alg. 4, reading R17): D = U - M, all-reduce (sum), server
// Adam on U, M <- U.
#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

#include "gcp_internal.h"

using namespace gcp;

namespace gcp {

#define NCCL_TRY(c, x, what)                                  \
    do {                                                      \
        ncclResult_t r_ = (x);                                \
        if (r_ != ncclSuccess) return nccl_fail((c), r_, what); \
    } while (0)

static ncclDataType_t dtype(const gcp_ctx* c) { return c->prec == GCP_FP32 ? ncclFloat32 : ncclFloat64; }
static size_t tsz(const gcp_ctx* c) { return c->prec == GCP_FP32 ? 4 : 8; }

gcp_status dist_make_slices(gcp_ctx* c) {
    // the split depends only on the grid (every rank computes the same one), so a
    // replace-ingest with the same grid keeps its communicators: ncclCommSplit is
    // a collective costing ~0.1-1 s per mode
    bool same = c->slice_d == c->d;
    for (int k = 0; same && k < c->d; ++k) same = c->slice_grid[k] == c->grid[k] && c->slice[k] != nullptr;
    if (same) return GCP_OK;
    c->slice_d = 0;
    int b[kMaxModes];
    int rem = c->rank;
    for (int k = c->d - 1; k >= 0; --k) {
        b[k] = rem % c->grid[k];
        rem /= c->grid[k];
    }
    for (int k = 0; k < kMaxModes; ++k) {
        if (c->slice[k]) {
            ncclCommDestroy(c->slice[k]);
            c->slice[k] = nullptr;
        }
        c->slice_size[k] = 1;
        c->slice_rank[k] = 0;
    }
    for (int k = 0; k < c->d; ++k) {
        NCCL_TRY(c, ncclCommSplit(c->world, b[k], c->rank, &c->slice[k], nullptr), "ncclCommSplit");
        int n = 0, r = 0;
        NCCL_TRY(c, ncclCommCount(c->slice[k], &n), "ncclCommCount");
        NCCL_TRY(c, ncclCommUserRank(c->slice[k], &r), "ncclCommUserRank");
        c->slice_size[k] = n;
        c->slice_rank[k] = r;
    }
    for (int k = 0; k < c->d; ++k) c->slice_grid[k] = c->grid[k];
    c->slice_d = c->d;
    return GCP_OK;
}

gcp_status dist_sync_exchange_pre(gcp_ctx* c) {
    // Per mode: small blocks are all-reduced (one latency-bound call, Adam then
    // runs on the replicated rows); large blocks are reduce-scattered so Adam
    // and its moments are sharded over the slice group (c->ar_mode, model_init).
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    NCCL_TRY(c, ncclGroupStart(), "ncclGroupStart");
    for (int k = 0; k < c->d; ++k) {
        if (c->slice_size[k] <= 1) continue;
        char* base = (char*)c->d_G + (size_t)c->off[k] * tsz(c);
        if (c->ar_mode[k]) {
            NCCL_TRY(c, ncclAllReduce(base, base, (size_t)c->rows[k] * c->R_pad, dtype(c), ncclSum, c->slice[k],
                                      c->stream),
                     "ncclAllReduce(G)");
            continue;
        }
        const size_t shard = (size_t)(c->rows[k] / c->slice_size[k]) * c->R_pad;
        NCCL_TRY(c, ncclReduceScatter(base, base + (size_t)c->slice_rank[k] * shard * tsz(c), shard, dtype(c), ncclSum,
                                      c->slice[k], c->stream),
                 "ncclReduceScatter(G)");
    }
    NCCL_TRY(c, ncclGroupEnd(), "ncclGroupEnd");
    prof_end(c, PROF_COMM, ev);
    return GCP_OK;
}

gcp_status dist_sync_exchange_post(gcp_ctx* c) {
    bool any = false;
    for (int k = 0; k < c->d; ++k) any |= c->slice_size[k] > 1 && !c->ar_mode[k];
    if (!any) return GCP_OK;
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    NCCL_TRY(c, ncclGroupStart(), "ncclGroupStart");
    for (int k = 0; k < c->d; ++k) {
        if (c->slice_size[k] <= 1 || c->ar_mode[k]) continue;
        const size_t shard = (size_t)(c->rows[k] / c->slice_size[k]) * c->R_pad;
        char* base = (char*)c->d_A + (size_t)c->off[k] * tsz(c);
        NCCL_TRY(c, ncclAllGather(base + (size_t)c->slice_rank[k] * shard * tsz(c), base, shard, dtype(c), c->slice[k],
                                  c->stream),
                 "ncclAllGather(A)");
    }
    NCCL_TRY(c, ncclGroupEnd(), "ncclGroupEnd");
    prof_end(c, PROF_COMM, ev);
    return GCP_OK;
}

// Sum each mode's block over its slice group (in place); no-op for groups of 1.
static gcp_status slice_allreduce(gcp_ctx* c, void* arr) {
    if (c->P <= 1) return GCP_OK;
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    NCCL_TRY(c, ncclGroupStart(), "ncclGroupStart");
    for (int k = 0; k < c->d; ++k) {
        if (c->slice_size[k] <= 1) continue;
        char* base = (char*)arr + (size_t)c->off[k] * tsz(c);
        const size_t n = (size_t)c->rows[k] * c->R_pad;
        NCCL_TRY(c, ncclAllReduce(base, base, n, dtype(c), ncclSum, c->slice[k], c->stream), "ncclAllReduce");
    }
    NCCL_TRY(c, ncclGroupEnd(), "ncclGroupEnd");
    prof_end(c, PROF_COMM, ev);
    return GCP_OK;
}

gcp_status dist_async_sync(gcp_ctx* c) {
    if (c->mode == GCP_DIST_ASYNC_AVG) {
        // Alg. 3 lines 2-4: Allreduce(M); M <- M / g_k (reading R16)
        if (c->P <= 1) return GCP_OK;
        gcp_status s = slice_allreduce(c, c->d_A);
        if (s != GCP_OK) return s;
        for (int k = 0; k < c->d; ++k) {
            if (c->slice_size[k] <= 1) continue;
            cudaEvent_t ev;
            prof_begin(c, PROF_OTHER, &ev);
            cudaError_t e = launch_scale(c, (char*)c->d_A + (size_t)c->off[k] * tsz(c), c->rows[k] * c->R_pad,
                                         1.0 / c->slice_size[k]);
            prof_end(c, PROF_OTHER, ev);
            if (e != cudaSuccess) return cuda_fail(c, e, "async average");
        }
        return GCP_OK;
    }
    // Alg. 4 lines 3-6: D = U - M; AllReduce(D); U.update(D) (server Adam); M <- U
    const size_t bytes = (size_t)c->n_coef * tsz(c);
    cudaEvent_t ev;
    prof_begin(c, PROF_OTHER, &ev);
    cudaError_t e = launch_sub(c, c->d_U, c->d_A, c->d_G, c->n_coef);   // G is zero here: use it for D
    prof_end(c, PROF_OTHER, ev);
    if (e != cudaSuccess) return cuda_fail(c, e, "fedadam D");
    gcp_status s = slice_allreduce(c, c->d_G);
    if (s != GCP_OK) return s;
    c->ts += 1;
    Segment seg;
    seg.n = 1;
    seg.start[0] = 0;
    seg.len[0] = c->n_coef;
    const double lower = std::isnan(c->server.lower) ? (c->last_loss == GCP_LOSS_POISSON ? 0.0 : -INFINITY)
                                                      : c->server.lower;
    prof_begin(c, PROF_ADAM, &ev);
    e = launch_adam(c, seg, c->d_U, c->d_G, c->d_Bs, c->d_Cs, c->server.rate, c->server.beta1, c->server.beta2,
                    c->server.eps, lower, c->ts, 1);
    prof_end(c, PROF_ADAM, ev);
    if (e != cudaSuccess) return cuda_fail(c, e, "fedadam server step");
    e = cudaMemcpyAsync(c->d_A, c->d_U, bytes, cudaMemcpyDeviceToDevice, c->stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "fedadam M <- U");
    return GCP_OK;
}

gcp_status dist_allreduce_scalar(gcp_ctx* c, double* dev_scalar) {
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    NCCL_TRY(c, ncclAllReduce(dev_scalar, dev_scalar, 1, ncclFloat64, ncclSum, c->world, c->stream), "ncclAllReduce");
    prof_end(c, PROF_COMM, ev);
    return GCP_OK;
}

gcp_status dist_allreduce_i64_host(gcp_ctx* c, int64_t* v, int n) {
    int64_t* d = nullptr;
    cudaError_t e = gmalloc(c, &d, sizeof(int64_t) * n);
    if (e != cudaSuccess) return cuda_fail(c, e, "allreduce scratch");
    cudaMemcpyAsync(d, v, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->stream);
    ncclResult_t r = ncclAllReduce(d, d, n, ncclInt64, ncclSum, c->world, c->stream);
    if (r != ncclSuccess) {
        gfree(c, d);
        return nccl_fail(c, r, "ncclAllReduce(int64)");
    }
    cudaMemcpyAsync(v, d, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->stream);
    e = cudaStreamSynchronize(c->stream);
    gfree(c, d);
    if (e != cudaSuccess) return cuda_fail(c, e, "allreduce i64");
    return GCP_OK;
}

}  // namespace gcp

extern "C" {

gcp_status gcp_nccl_unique_id(void* out128) {
    if (!out128) return set_error(GCP_E_ARG, "gcp_nccl_unique_id: NULL");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return set_error(GCP_E_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out128, &id, 128);
    return GCP_OK;
}

gcp_status gcp_dist_init(gcp_ctx* c, int nranks, int rank, const void* id, const int* grid, int d,
                         gcp_dist_mode mode) {
    if (!c) return set_error(GCP_E_ARG, "null context");
    if (c->sticky != GCP_OK) return set_error(GCP_E_STATE, "sticky error");
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(GCP_E_ARG, "gcp_dist_init: rank / nranks");
    if (mode != GCP_DIST_SYNC && mode != GCP_DIST_ASYNC_AVG && mode != GCP_DIST_ASYNC_FEDADAM &&
        mode != GCP_DIST_SYNC_TWO_SIDED)
        return set_error(GCP_E_ARG, "gcp_dist_init: mode");
    if (c->have_tensor) return set_error(GCP_E_STATE, "gcp_dist_init: must precede gcp_tensor_create");
    if (grid) {
        if (d < 2 || d > kMaxModes) return set_error(GCP_E_ARG, "gcp_dist_init: d");
        int64_t prod = 1;
        for (int k = 0; k < d; ++k) {
            if (grid[k] < 1) return set_error(GCP_E_ARG, "gcp_dist_init: grid");
            prod *= grid[k];
        }
        if (prod != nranks) return set_error(GCP_E_ARG, "gcp_dist_init: grid product != nranks");
        for (int k = 0; k < d; ++k) c->grid[k] = grid[k];
        c->grid_given = true;
    }
    int prev;
    cudaGetDevice(&prev);
    cudaSetDevice(c->dev);
    if (nranks > 1) {
        if (!id) return set_error(GCP_E_ARG, "gcp_dist_init: need the NCCL unique id");
        ncclUniqueId uid;
        memcpy(&uid, id, 128);
        ncclResult_t r = ncclCommInitRank(&c->world, nranks, uid, rank);
        if (r != ncclSuccess) {
            cudaSetDevice(prev);
            return nccl_fail(c, r, "ncclCommInitRank");
        }
    }
    cudaSetDevice(prev);
    c->P = nranks;
    c->rank = rank;
    c->mode = mode;
    c->dist_ready = true;
    return GCP_OK;
}

}  // extern "C"
