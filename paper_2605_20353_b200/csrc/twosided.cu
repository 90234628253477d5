// twosided.cu -- row f3: the paper's "two-sided" factor distribution
// (§3.2).  The factor rows of each mode-k block are partitioned
// over the g_k ranks of the slice group (rank with slice index s owns rows
// [s*sh, (s+1)*sh) of the padded block, sh = rows_k / g_k); nothing is
// replicated.  Per iteration, because the sampled indices decide which rows
// are needed, the path is non-fused across ranks:
//
//   1. touch pass: draw this iteration's samples (same Philox stream as K2)
//      and mark the block rows they touch, per mode;
//   2. setup: the touched rows owned by other slice members, grouped by
//      owner; counts all-gathered over the slice communicator;
//   3. import: row ids to the owners, rows back (grouped ncclSend/ncclRecv,
//      the MPI_Alltoall of P:731-733), scattered into the local block copy;
//   4. K2 (unchanged: fused sampling-MTTKRP into the local block G);
//   5. export: the G rows of the imported rows back to their owners, which
//      add them into their own G rows;
//   6. Adam (Alg. 1) on the owned rows only; G <- 0.
//
// Mathematically identical to Alg. 2 (sum of block gradients, then Adam):
// parity against the oracle's P-rank simulation.
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <string>
#include <vector>

#include "device.cuh"
#include "gcp_internal.h"

namespace gcp {

struct TwoSidedState {
    uint32_t* bitmap[kMaxModes] = {nullptr};   // touched block rows (1 bit per row)
    int64_t bm_words[kMaxModes] = {0};
    uint8_t* flags = nullptr;                  // scratch: needed-row flags
    int64_t flags_cap = 0;
    int32_t* need[kMaxModes] = {nullptr};      // touched rows owned elsewhere, ascending
    int64_t need_cap[kMaxModes] = {0};
    int32_t* req[kMaxModes] = {nullptr};       // rows requested from me, by requester
    int64_t req_cap[kMaxModes] = {0};
    int64_t* d_counts = nullptr;               // [d][8] my per-owner counts, then [d][8*8] gathered matrix
    int64_t* h_counts = nullptr;               // pinned mirror
    int64_t nneed[kMaxModes][8] = {{0}};       // my requests to owner o
    int64_t nreq[kMaxModes][8] = {{0}};        // requests of member p to me
    void* sbuf = nullptr;
    void* rbuf = nullptr;
    size_t sbuf_cap = 0, rbuf_cap = 0;
    void* cub_tmp = nullptr;
    size_t cub_cap = 0;
    int64_t* d_nsel = nullptr;
};

struct TouchArgs {
    uint32_t* bm[kMaxModes];
};

template <typename T, int D>
__global__ void k_touch(const SampleArgs sa, const TouchArgs ta) {
    const int64_t total = sa.p + sa.q;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < total; s += (int64_t)gridDim.x * blockDim.x) {
        const Sample<T, D> smp = draw_sample<T, D>(sa, s);
#pragma unroll
        for (int k = 0; k < D; ++k) atomicOr(ta.bm[k] + (smp.c[k] >> 5), 1u << (smp.c[k] & 31));
    }
}

// flag = touched && not owned by me
__global__ void k_need_flags(const uint32_t* __restrict__ bm, int64_t nrows, int64_t own_lo, int64_t own_hi,
                             uint8_t* __restrict__ flags) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x)
        flags[r] = ((bm[r >> 5] >> (r & 31)) & 1u) && (r < own_lo || r >= own_hi);
}

// per-owner counts of an ascending row list: owner o holds rows [o*sh, (o+1)*sh)
__global__ void k_owner_counts(const int32_t* __restrict__ rows, const int64_t* __restrict__ n, int64_t sh, int g,
                               int64_t* __restrict__ out) {
    const int o = threadIdx.x;
    if (o >= g) return;
    auto lb = [&](int64_t v) {
        int64_t a = 0, b = *n;
        while (a < b) {
            const int64_t m = (a + b) / 2;
            if (rows[m] < v) a = m + 1;
            else b = m;
        }
        return a;
    };
    out[o] = lb((int64_t)(o + 1) * sh) - lb((int64_t)o * sh);
}

template <typename T>
__global__ void k_gather_rows(const int32_t* __restrict__ rows, int64_t n, const T* __restrict__ src, int64_t off,
                              int R_pad, T* __restrict__ out) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n * R_pad; x += (int64_t)gridDim.x * blockDim.x)
        out[x] = src[off + (int64_t)rows[x / R_pad] * R_pad + x % R_pad];
}

template <typename T>
__global__ void k_scatter_rows(const int32_t* __restrict__ rows, int64_t n, const T* __restrict__ in, int64_t off,
                               int R_pad, T* __restrict__ dst, int add) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n * R_pad; x += (int64_t)gridDim.x * blockDim.x) {
        T* p = dst + off + (int64_t)rows[x / R_pad] * R_pad + x % R_pad;
        if (add) *p += in[x];
        else *p = in[x];
    }
}

#define TS_CUDA(c, x, what)                                          \
    do {                                                             \
        cudaError_t e_ = (x);                                        \
        if (e_ != cudaSuccess) return cuda_fail((c), e_, what);      \
    } while (0)
#define TS_NCCL(c, x, what)                                          \
    do {                                                             \
        ncclResult_t r_ = (x);                                       \
        if (r_ != ncclSuccess) return nccl_fail((c), r_, what);      \
    } while (0)

static size_t tsz(const gcp_ctx* c) { return c->prec == GCP_FP32 ? 4 : 8; }
static ncclDataType_t dtype(const gcp_ctx* c) { return c->prec == GCP_FP32 ? ncclFloat32 : ncclFloat64; }
static int grid_for(const gcp_ctx* c, int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8));
}

template <typename P>
static gcp_status grow(gcp_ctx* c, P** p, int64_t* cap, int64_t n, size_t elem) {
    if (n <= *cap) return GCP_OK;
    gfree(c, *p);
    *p = nullptr;
    const int64_t want = std::max<int64_t>(n, *cap * 2);
    TS_CUDA(c, gmalloc(c, p, (size_t)want * elem), "two-sided scratch");
    *cap = want;
    return GCP_OK;
}
static gcp_status grow_b(gcp_ctx* c, void** p, size_t* cap, size_t bytes) {
    if (bytes <= *cap) return GCP_OK;
    gfree(c, *p);
    *p = nullptr;
    const size_t want = std::max(bytes, *cap * 2);
    TS_CUDA(c, gmalloc(c, p, want), "two-sided buffer");
    *cap = want;
    return GCP_OK;
}

void twosided_free(gcp_ctx* c) {
    TwoSidedState* s = static_cast<TwoSidedState*>(c->twosided);
    if (!s) return;
    for (int k = 0; k < kMaxModes; ++k) {
        gfree(c, s->bitmap[k]);
        gfree(c, s->need[k]);
        gfree(c, s->req[k]);
    }
    gfree(c, s->flags);
    gfree(c, s->d_counts);
    if (s->h_counts) cudaFreeHost(s->h_counts);
    gfree(c, s->sbuf);
    gfree(c, s->rbuf);
    gfree(c, s->cub_tmp);
    gfree(c, s->d_nsel);
    delete s;
    c->twosided = nullptr;
}

static gcp_status state(gcp_ctx* c, TwoSidedState** out) {
    if (!c->twosided) {
        TwoSidedState* s = new TwoSidedState();
        c->twosided = s;
        TS_CUDA(c, gmalloc(c, &s->d_counts, sizeof(int64_t) * kMaxModes * (8 + 64)), "two-sided counts");
        TS_CUDA(c, cudaMallocHost(&s->h_counts, sizeof(int64_t) * kMaxModes * (8 + 64)), "two-sided counts");
        TS_CUDA(c, gmalloc(c, &s->d_nsel, sizeof(int64_t) * kMaxModes), "two-sided counts");
    }
    *out = static_cast<TwoSidedState*>(c->twosided);
    return GCP_OK;
}

// Steps 1-3: touch pass, setup, import.  `sa` are this iteration's sampler args.
gcp_status twosided_import(gcp_ctx* c, const SampleArgs& sa) {
    TwoSidedState* s;
    gcp_status st = state(c, &s);
    if (st != GCP_OK) return st;
    cudaStream_t strm = c->stream;
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    // 1. touch pass
    TouchArgs ta{};
    for (int k = 0; k < c->d; ++k) {
        const int64_t words = (c->rows[k] + 31) / 32;
        st = grow(c, &s->bitmap[k], &s->bm_words[k], words, sizeof(uint32_t));
        if (st != GCP_OK) return st;
        TS_CUDA(c, cudaMemsetAsync(s->bitmap[k], 0, (size_t)words * 4, strm), "touch reset");
        ta.bm[k] = s->bitmap[k];
    }
    const int nb = c->sm_count * 8;
    const bool f32 = c->prec == GCP_FP32;
    switch (c->d) {
    case 2: f32 ? k_touch<float, 2><<<nb, 256, 0, strm>>>(sa, ta) : k_touch<double, 2><<<nb, 256, 0, strm>>>(sa, ta); break;
    case 3: f32 ? k_touch<float, 3><<<nb, 256, 0, strm>>>(sa, ta) : k_touch<double, 3><<<nb, 256, 0, strm>>>(sa, ta); break;
    case 4: f32 ? k_touch<float, 4><<<nb, 256, 0, strm>>>(sa, ta) : k_touch<double, 4><<<nb, 256, 0, strm>>>(sa, ta); break;
    case 5: f32 ? k_touch<float, 5><<<nb, 256, 0, strm>>>(sa, ta) : k_touch<double, 5><<<nb, 256, 0, strm>>>(sa, ta); break;
    default: f32 ? k_touch<float, 6><<<nb, 256, 0, strm>>>(sa, ta) : k_touch<double, 6><<<nb, 256, 0, strm>>>(sa, ta); break;
    }
    TS_CUDA(c, cudaGetLastError(), "touch pass");
    // 2. needed rows per mode, grouped by owner (ascending rows = owner order)
    for (int k = 0; k < c->d; ++k) {
        const int g = c->slice_size[k];
        if (g <= 1) continue;
        const int64_t sh = c->rows[k] / g;
        const int64_t nrows = c->rows[k];
        st = grow(c, &s->flags, &s->flags_cap, nrows, 1);
        if (st != GCP_OK) return st;
        st = grow(c, &s->need[k], &s->need_cap[k], nrows, sizeof(int32_t));
        if (st != GCP_OK) return st;
        k_need_flags<<<grid_for(c, nrows), 256, 0, strm>>>(s->bitmap[k], nrows, c->slice_rank[k] * sh,
                                                           (c->slice_rank[k] + 1) * sh, s->flags);
        TS_CUDA(c, cudaGetLastError(), "need flags");
        cub::CountingInputIterator<int32_t> it(0);
        size_t tb = 0;
        TS_CUDA(c, cub::DeviceSelect::Flagged(nullptr, tb, it, s->flags, s->need[k], s->d_nsel + k, nrows, strm),
                "select");
        st = grow_b(c, &s->cub_tmp, &s->cub_cap, tb);
        if (st != GCP_OK) return st;
        TS_CUDA(c, cub::DeviceSelect::Flagged(s->cub_tmp, tb, it, s->flags, s->need[k], s->d_nsel + k, nrows, strm),
                "select");
        k_owner_counts<<<1, 32, 0, strm>>>(s->need[k], s->d_nsel + k, sh, g, s->d_counts + k * 8);
        TS_CUDA(c, cudaGetLastError(), "owner counts");
    }
    // counts matrix of every slice group: all-gather each member's per-owner counts
    TS_NCCL(c, ncclGroupStart(), "group");
    for (int k = 0; k < c->d; ++k) {
        const int g = c->slice_size[k];
        if (g <= 1) continue;
        TS_NCCL(c, ncclAllGather(s->d_counts + k * 8, s->d_counts + kMaxModes * 8 + k * 64, 8, ncclInt64, c->slice[k],
                                 strm),
                "counts all-gather");
    }
    TS_NCCL(c, ncclGroupEnd(), "group");
    TS_CUDA(c, cudaMemcpyAsync(s->h_counts, s->d_counts, sizeof(int64_t) * kMaxModes * (8 + 64), cudaMemcpyDeviceToHost,
                               strm),
            "counts D2H");
    TS_CUDA(c, cudaStreamSynchronize(strm), "two-sided setup");
    int64_t total_req = 0, total_need = 0;
    for (int k = 0; k < c->d; ++k) {
        const int g = c->slice_size[k];
        for (int o = 0; o < 8; ++o) s->nneed[k][o] = s->nreq[k][o] = 0;
        if (g <= 1) continue;
        const int me = c->slice_rank[k];
        int64_t rk = 0;
        for (int o = 0; o < g; ++o) {
            s->nneed[k][o] = s->h_counts[k * 8 + o];
            s->nreq[k][o] = s->h_counts[kMaxModes * 8 + k * 64 + o * 8 + me];   // member o's requests to me
            rk += s->nreq[k][o];
            total_need += s->nneed[k][o];
        }
        total_req += rk;
        st = grow(c, &s->req[k], &s->req_cap[k], std::max<int64_t>(rk, 1), sizeof(int32_t));
        if (st != GCP_OK) return st;
    }
    // 3a. row ids to the owners
    TS_NCCL(c, ncclGroupStart(), "group");
    for (int k = 0; k < c->d; ++k) {
        const int g = c->slice_size[k];
        if (g <= 1) continue;
        const int me = c->slice_rank[k];
        int64_t so = 0, ro = 0;
        for (int o = 0; o < g; ++o) {
            if (o != me && s->nneed[k][o] > 0)
                TS_NCCL(c, ncclSend(s->need[k] + so, s->nneed[k][o], ncclInt32, o, c->slice[k], strm), "send ids");
            so += s->nneed[k][o];
            if (o != me && s->nreq[k][o] > 0)
                TS_NCCL(c, ncclRecv(s->req[k] + ro, s->nreq[k][o], ncclInt32, o, c->slice[k], strm), "recv ids");
            ro += s->nreq[k][o];
        }
    }
    TS_NCCL(c, ncclGroupEnd(), "group");
    // 3b. owners gather the requested rows, requesters receive them
    const size_t rowb = (size_t)c->R_pad * tsz(c);
    st = grow_b(c, &s->sbuf, &s->sbuf_cap, std::max<int64_t>(total_req, 1) * rowb);
    if (st != GCP_OK) return st;
    st = grow_b(c, &s->rbuf, &s->rbuf_cap, std::max<int64_t>(total_need, 1) * rowb);
    if (st != GCP_OK) return st;
    {
        size_t sofs = 0;
        for (int k = 0; k < c->d; ++k) {
            if (c->slice_size[k] <= 1) continue;
            int64_t rk = 0;
            for (int o = 0; o < c->slice_size[k]; ++o) rk += s->nreq[k][o];
            if (rk > 0) {
                if (f32)
                    k_gather_rows<float><<<grid_for(c, rk * c->R_pad), 256, 0, strm>>>(
                        s->req[k], rk, (const float*)c->d_A, c->off[k], c->R_pad, (float*)((char*)s->sbuf + sofs));
                else
                    k_gather_rows<double><<<grid_for(c, rk * c->R_pad), 256, 0, strm>>>(
                        s->req[k], rk, (const double*)c->d_A, c->off[k], c->R_pad, (double*)((char*)s->sbuf + sofs));
                TS_CUDA(c, cudaGetLastError(), "gather rows");
            }
            sofs += (size_t)rk * rowb;
        }
    }
    TS_NCCL(c, ncclGroupStart(), "group");
    {
        size_t sofs = 0, rofs = 0;
        for (int k = 0; k < c->d; ++k) {
            const int g = c->slice_size[k];
            if (g <= 1) continue;
            const int me = c->slice_rank[k];
            for (int o = 0; o < g; ++o) {
                if (o != me && s->nreq[k][o] > 0)
                    TS_NCCL(c, ncclSend((char*)s->sbuf + sofs, s->nreq[k][o] * c->R_pad, dtype(c), o, c->slice[k], strm),
                            "send rows");
                sofs += (size_t)s->nreq[k][o] * rowb;
                if (o != me && s->nneed[k][o] > 0)
                    TS_NCCL(c, ncclRecv((char*)s->rbuf + rofs, s->nneed[k][o] * c->R_pad, dtype(c), o, c->slice[k], strm),
                            "recv rows");
                rofs += (size_t)s->nneed[k][o] * rowb;
            }
        }
    }
    TS_NCCL(c, ncclGroupEnd(), "group");
    // 3c. imported rows into the local block copy
    {
        size_t rofs = 0;
        for (int k = 0; k < c->d; ++k) {
            if (c->slice_size[k] <= 1) continue;
            int64_t nk = 0;
            for (int o = 0; o < c->slice_size[k]; ++o) nk += s->nneed[k][o];
            if (nk > 0) {
                if (f32)
                    k_scatter_rows<float><<<grid_for(c, nk * c->R_pad), 256, 0, strm>>>(
                        s->need[k], nk, (const float*)((char*)s->rbuf + rofs), c->off[k], c->R_pad, (float*)c->d_A, 0);
                else
                    k_scatter_rows<double><<<grid_for(c, nk * c->R_pad), 256, 0, strm>>>(
                        s->need[k], nk, (const double*)((char*)s->rbuf + rofs), c->off[k], c->R_pad, (double*)c->d_A, 0);
                TS_CUDA(c, cudaGetLastError(), "scatter rows");
            }
            rofs += (size_t)nk * rowb;
        }
    }
    prof_end(c, PROF_COMM, ev);
    return GCP_OK;
}

// Step 5: export the G rows of the imported rows to their owners.
gcp_status twosided_export(gcp_ctx* c) {
    TwoSidedState* s = static_cast<TwoSidedState*>(c->twosided);
    if (!s) return GCP_OK;
    cudaStream_t strm = c->stream;
    const bool f32 = c->prec == GCP_FP32;
    const size_t rowb = (size_t)c->R_pad * tsz(c);
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    {   // requesters pack the G rows they computed for other owners (same order as their requests)
        size_t ofs = 0;
        for (int k = 0; k < c->d; ++k) {
            if (c->slice_size[k] <= 1) continue;
            int64_t nk = 0;
            for (int o = 0; o < c->slice_size[k]; ++o) nk += s->nneed[k][o];
            if (nk > 0) {
                if (f32)
                    k_gather_rows<float><<<grid_for(c, nk * c->R_pad), 256, 0, strm>>>(
                        s->need[k], nk, (const float*)c->d_G, c->off[k], c->R_pad, (float*)((char*)s->rbuf + ofs));
                else
                    k_gather_rows<double><<<grid_for(c, nk * c->R_pad), 256, 0, strm>>>(
                        s->need[k], nk, (const double*)c->d_G, c->off[k], c->R_pad, (double*)((char*)s->rbuf + ofs));
                TS_CUDA(c, cudaGetLastError(), "pack G rows");
            }
            ofs += (size_t)nk * rowb;
        }
    }
    TS_NCCL(c, ncclGroupStart(), "group");
    {
        size_t sofs = 0, rofs = 0;
        for (int k = 0; k < c->d; ++k) {
            const int g = c->slice_size[k];
            if (g <= 1) continue;
            const int me = c->slice_rank[k];
            for (int o = 0; o < g; ++o) {
                if (o != me && s->nneed[k][o] > 0)
                    TS_NCCL(c, ncclSend((char*)s->rbuf + rofs, s->nneed[k][o] * c->R_pad, dtype(c), o, c->slice[k], strm),
                            "send G rows");
                rofs += (size_t)s->nneed[k][o] * rowb;
                if (o != me && s->nreq[k][o] > 0)
                    TS_NCCL(c, ncclRecv((char*)s->sbuf + sofs, s->nreq[k][o] * c->R_pad, dtype(c), o, c->slice[k], strm),
                            "recv G rows");
                sofs += (size_t)s->nreq[k][o] * rowb;
            }
        }
    }
    TS_NCCL(c, ncclGroupEnd(), "group");
    {   // owners add each requester's rows into their own G rows (per requester: rows unique)
        size_t sofs = 0;
        for (int k = 0; k < c->d; ++k) {
            const int g = c->slice_size[k];
            if (g <= 1) continue;
            int64_t rofs_rows = 0;
            for (int o = 0; o < g; ++o) {
                const int64_t n = s->nreq[k][o];
                if (n > 0) {
                    if (f32)
                        k_scatter_rows<float><<<grid_for(c, n * c->R_pad), 256, 0, strm>>>(
                            s->req[k] + rofs_rows, n, (const float*)((char*)s->sbuf + sofs), c->off[k], c->R_pad,
                            (float*)c->d_G, 1);
                    else
                        k_scatter_rows<double><<<grid_for(c, n * c->R_pad), 256, 0, strm>>>(
                            s->req[k] + rofs_rows, n, (const double*)((char*)s->sbuf + sofs), c->off[k], c->R_pad,
                            (double*)c->d_G, 1);
                    TS_CUDA(c, cudaGetLastError(), "add G rows");
                }
                rofs_rows += n;
                sofs += (size_t)n * rowb;
            }
        }
    }
    prof_end(c, PROF_COMM, ev);
    return GCP_OK;
}

}  // namespace gcp
