// fused.cu -- rows a6 + a7 + a8 (sync, nranks > 1) as ONE kernel over NVLink
// peer memory.  Alg. 2 sums G over ranks and updates M; with the
// medium-grained grid the sum for mode k runs over the mode-k slice group
// (P:683-688).  Here every rank owns 1/g_k of its mode-k block rows:
// between two LSA barriers the kernel loads those rows of G^(k) from every
// slice member's symmetric window (the reduce-scatter), applies Alg. 1 Adam to
// them with rank-local sharded moments, and stores the updated rows
// into every member's A^(k) window (the all-gather).  No NCCL collective, no
// separate Adam launch.  NCCL 2.28 device API (symmetric windows, LSA barrier).
//
// G is double-buffered by iteration parity: the K2 of iteration t accumulates
// into G[t%2]; the exchange of iteration t reads G[t%2] from the members and
// zeroes the local G[(t+1)%2], which every member finished reading in the
// exchange of t-1 (all ranks passed this kernel's first barrier, so all their
// previous exchanges are complete).
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cmath>
#include <string>

#include "gcp_internal.h"

namespace gcp {

constexpr int kFusedCTAs = 256;   // CTAs of the fused exchange == LSA barriers requested

struct FusedArgs {
    int d, R_pad;
    int64_t off[kMaxModes];           // element offset of mode k (identical on every rank)
    int64_t shard_start[kMaxModes];   // first block row of my shard
    int64_t vec_begin[kMaxModes + 1]; // prefix over modes of my shard's 16-B vectors
    int nmem[kMaxModes];
    int mem[kMaxModes][8];            // LSA ranks of the mode-k slice members (incl. me)
    int64_t zero_vecs;                // 16-B vectors of the local G buffer to zero
};

template <typename T> struct FVec;
template <> struct FVec<float> { using type = float4; static constexpr int n = 4; };
template <> struct FVec<double> { using type = double2; static constexpr int n = 2; };

template <typename T>
__global__ void __launch_bounds__(256) k_fused_exchange(ncclDevComm comm, ncclWindow_t winA, ncclWindow_t winG,
                                                        T* __restrict__ gzero, T* __restrict__ B,
                                                        T* __restrict__ C, const FusedArgs fa, T rate, T b1, T b2,
                                                        T eps, T bc1, T bc2, T lower, const DevStep* step,
                                                        long long t_off) {
    using V = typename FVec<T>::type;
    constexpr int VE = FVec<T>::n;
    if (step) {   // graph replay: t = t0 + offset, bias corrections in fp64 from it
        const double t = (double)(step->t + t_off);
        rate = (T)step->rate;
        bc1 = (T)(1.0 / (1.0 - pow(step->beta1, t)));
        bc2 = (T)(1.0 / (1.0 - pow(step->beta2, t)));
    }
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamLsa(comm), comm.lsaBarrier, blockIdx.x);
    // every rank's K2 of this iteration is complete (stream order before arrive)
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    {
        V z;
        T* zp = reinterpret_cast<T*>(&z);
#pragma unroll
        for (int q = 0; q < VE; ++q) zp[q] = T(0);
        for (int64_t x = tid; x < fa.zero_vecs; x += nt) reinterpret_cast<V*>(gzero)[x] = z;
    }
    const int vpr = fa.R_pad / VE;
    for (int64_t v = tid; v < fa.vec_begin[fa.d]; v += nt) {
        int k = 0;
        while (v >= fa.vec_begin[k + 1]) ++k;
        const int64_t lv = v - fa.vec_begin[k];
        const int64_t e = fa.off[k] + (fa.shard_start[k] + lv / vpr) * fa.R_pad + (lv % vpr) * VE;
        const size_t ob = (size_t)e * sizeof(T);
        // reduce-scatter: this shard vector of G^(k) summed over the slice group
        // (all member loads issued before the adds: up to 8 NVLink loads in flight)
        const int nm = fa.nmem[k];
        V h[8];
#pragma unroll
        for (int m = 0; m < 8; ++m)
            if (m < nm) h[m] = *reinterpret_cast<const V*>(ncclGetLsaPointer(winG, ob, fa.mem[k][m]));
        V g = h[0];
        T* gp = reinterpret_cast<T*>(&g);
#pragma unroll
        for (int m = 1; m < 8; ++m) {
            if (m >= nm) break;
            const T* hp = reinterpret_cast<const T*>(&h[m]);
#pragma unroll
            for (int q = 0; q < VE; ++q) gp[q] += hp[q];
        }
        // Alg. 1 on the owned rows (moments B, C are rank-local shards)
        V a = *reinterpret_cast<const V*>(ncclGetLocalPointer(winA, ob));
        V bb = *reinterpret_cast<const V*>(B + e);
        V cc = *reinterpret_cast<const V*>(C + e);
        T* ap = reinterpret_cast<T*>(&a);
        T* bp = reinterpret_cast<T*>(&bb);
        T* cp = reinterpret_cast<T*>(&cc);
#pragma unroll
        for (int q = 0; q < VE; ++q) {
            const T gv = gp[q];
            bp[q] = b1 * bp[q] + (T(1) - b1) * gv;
            cp[q] = b2 * cp[q] + (T(1) - b2) * gv * gv;
            const T av = ap[q] - rate * ((bp[q] * bc1) / sqrt(cp[q] * bc2 + eps));
            ap[q] = (av < lower) ? lower : av;
        }
        *reinterpret_cast<V*>(B + e) = bb;
        *reinterpret_cast<V*>(C + e) = cc;
        // all-gather: the updated rows into every member's A^(k)
        for (int m = 0; m < fa.nmem[k]; ++m) *reinterpret_cast<V*>(ncclGetLsaPointer(winA, ob, fa.mem[k][m])) = a;
    }
    // all updated rows visible on every member before any next K2
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

#define NCCL_TRY_F(c, x, what)                                      \
    do {                                                            \
        ncclResult_t r_ = (x);                                      \
        if (r_ != ncclSuccess) return nccl_fail((c), r_, what);     \
    } while (0)

static size_t round_win(size_t b) {
    const size_t g = (size_t)2 << 20;   // symmetric windows: whole 2-MB granules
    return (b + g - 1) / g * g;
}

bool fused_possible(gcp_ctx* c) {
    if (c->P <= 1 || c->mode != GCP_DIST_SYNC) return false;
    const char* env = getenv("GCP_SYNC_EXCHANGE");
    if (env && std::string(env) != "fused") return false;
    for (int k = 0; k < c->d; ++k)
        if (c->slice_size[k] > 8) return false;
    const ncclTeam_t lsa = ncclTeamLsa(c->world);
    return lsa.nRanks == c->P;
}

// Symmetric A and G[2] windows on the world communicator (collective).
gcp_status fused_alloc(gcp_ctx* c, size_t bytes) {
    const size_t wb = round_win(bytes);
    void** bufs[3] = {&c->d_A, &c->d_G, &c->d_G2};
    ncclWindow_t* wins[3] = {&c->winA, &c->winG[0], &c->winG[1]};
    for (int i = 0; i < 3; ++i) {
        NCCL_TRY_F(c, ncclMemAlloc(bufs[i], wb), "ncclMemAlloc");
        NCCL_TRY_F(c, ncclCommWindowRegister(c->world, *bufs[i], wb, wins[i], NCCL_WIN_COLL_SYMMETRIC),
                   "ncclCommWindowRegister");
    }
    if (!c->devcomm_ready) {
        ncclDevCommRequirements reqs;
        memset(&reqs, 0, sizeof(reqs));
        reqs.lsaBarrierCount = kFusedCTAs;
        NCCL_TRY_F(c, ncclDevCommCreate(c->world, &reqs, &c->devcomm), "ncclDevCommCreate");
        c->devcomm_ready = true;
    }
    // slice members of every mode as LSA ranks, in world-rank order (== slice_rank order)
    int b[kMaxModes];
    int rem = c->rank;
    for (int k = c->d - 1; k >= 0; --k) {
        b[k] = rem % c->grid[k];
        rem /= c->grid[k];
    }
    const ncclTeam_t world = ncclTeamWorld(c->world);
    for (int k = 0; k < c->d; ++k) {
        int n = 0;
        for (int w = 0; w < c->P; ++w) {
            int r = w, bw = 0;
            for (int j = c->d - 1; j >= 0; --j) {
                if (j == k) bw = r % c->grid[j];
                r /= c->grid[j];
            }
            if (bw == b[k]) c->fmem[k][n++] = ncclTeamRankToLsa(c->world, world, w);
        }
        c->fnmem[k] = n;
    }
    c->fused = true;
    return GCP_OK;
}

void fused_free(gcp_ctx* c) {
    if (!c->fused) return;
    void** bufs[3] = {&c->d_A, &c->d_G, &c->d_G2};
    ncclWindow_t* wins[3] = {&c->winA, &c->winG[0], &c->winG[1]};
    cudaStreamSynchronize(c->stream);
    for (int i = 0; i < 3; ++i) {
        if (*wins[i]) ncclCommWindowDeregister(c->world, *wins[i]);
        if (*bufs[i]) ncclMemFree(*bufs[i]);
        *wins[i] = nullptr;
        *bufs[i] = nullptr;
    }
    c->fused = false;
}

gcp_status fused_exchange(gcp_ctx* c, const gcp_adam_params* p, double lower) {
    FusedArgs fa;
    memset(&fa, 0, sizeof(fa));
    fa.d = c->d;
    fa.R_pad = c->R_pad;
    const int VE = c->prec == GCP_FP32 ? 4 : 2;
    int64_t acc = 0;
    for (int k = 0; k < c->d; ++k) {
        const int64_t shard = c->rows[k] / c->slice_size[k];
        fa.off[k] = c->off[k];
        fa.shard_start[k] = (int64_t)c->slice_rank[k] * shard;
        fa.vec_begin[k] = acc;
        acc += shard * (c->R_pad / VE);
        fa.nmem[k] = c->fnmem[k];
        for (int m = 0; m < c->fnmem[k]; ++m) fa.mem[k][m] = c->fmem[k][m];
    }
    fa.vec_begin[c->d] = acc;
    fa.zero_vecs = c->n_coef / VE;
    const int cur = (int)(c->it & 1);
    void* gnext = cur ? c->d_G : c->d_G2;
    const double bc1 = 1.0 / (1.0 - pow(p->beta1, (double)c->t));
    const double bc2 = 1.0 / (1.0 - pow(p->beta2, (double)c->t));
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    if (c->prec == GCP_FP32)
        k_fused_exchange<float><<<kFusedCTAs, 256, 0, c->stream>>>(
            c->devcomm, c->winA, c->winG[cur], (float*)gnext, (float*)c->d_B, (float*)c->d_C, fa, (float)p->rate,
            (float)p->beta1, (float)p->beta2, (float)p->eps, (float)bc1, (float)bc2, (float)lower,
            c->capturing ? c->d_step : nullptr, (long long)(c->t - c->graph_t0));
    else
        k_fused_exchange<double><<<kFusedCTAs, 256, 0, c->stream>>>(
            c->devcomm, c->winA, c->winG[cur], (double*)gnext, (double*)c->d_B, (double*)c->d_C, fa, p->rate,
            p->beta1, p->beta2, p->eps, bc1, bc2, lower, c->capturing ? c->d_step : nullptr,
            (long long)(c->t - c->graph_t0));
    prof_end(c, PROF_COMM, ev);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "fused exchange");
    return GCP_OK;
}

}  // namespace gcp
