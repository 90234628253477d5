// twosided_nvl.cu -- row f3 (the paper's two-sided factor distribution,
// P:715-743, §3.2) driven entirely by the device over NVLink symmetric memory.
// The factor rows of each mode-k block are partitioned over the g_k ranks of
// the slice group (slice rank s owns rows [s*sh, (s+1)*sh), sh = rows_k/g_k);
// nothing is replicated or all-reduced.  A, G (two parities) and a touched-row
// bitmap (two parities) live in NCCL symmetric windows, so a rank reads a
// peer's rows and bits with plain loads through its LSA pointer:
//
//   touch   (k_tsn_touch)   draw this iteration's samples (the Philox stream of
//                           K2) and set the bit of every block row they touch
//   import  (k_tsn_import)  LSA barrier (every owner finished the previous
//                           Adam); every touched row owned elsewhere is loaded
//                           from its owner's A window into the local copy
//   K2                      unchanged: fused sampling-MTTKRP into the local G
//   export  (k_tsn_export)  LSA barrier (every rank's K2 done); the owner of a
//                           row sums its own G row and the G rows of exactly
//                           the members whose bitmap marks the row (the
//                           paper's export of partial rows to their owner,
//                           pulled by the owner), runs Alg. 1 on its rows, and
//                           zeroes the previous parity's G rows (a memset after
//                           it clears the previous parity's bits)
//
// The per-iteration request lists, counts exchange, host synchronisation and
// grouped send/recv of the NCCL two-sided path (twosided.cu) disappear: only
// touched rows cross NVLink, and the epoch replays as a CUDA graph.  Bit
// parities: iteration t touches / accumulates into parity t%2; the export of t
// clears parity (t+1)%2, which every member finished reading in the export of
// t-1 (all passed this kernel's barrier).  Mathematically Alg. 2 (sum of the
// block gradients, then Adam): same parity tests as the all-reduce layout.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "device.cuh"
#include "gcp_internal.h"

namespace gcp {

struct TsnArgs {
    int d, R_pad;
    int64_t off[kMaxModes];        // element offset of mode k in A / G (identical on every rank)
    int64_t rows[kMaxModes];       // padded block rows of mode k
    int64_t bm_off[kMaxModes];     // word offset of mode k's bitmap inside one parity
    int64_t bm_words;              // words of one parity (all modes)
    int64_t shard[kMaxModes];      // sh = rows / g
    int me[kMaxModes];             // my slice rank
    int nmem[kMaxModes];
    int mem[kMaxModes][8];         // LSA ranks of the slice members in slice-rank order
};

template <typename T, int D>
__global__ void k_tsn_touch(const SampleArgs sa, uint32_t* __restrict__ bm, TsnArgs ta) {
    const int64_t total = sa.p + sa.q;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < total; s += (int64_t)gridDim.x * blockDim.x) {
        const Sample<T, D> smp = draw_sample<T, D>(sa, s);
#pragma unroll
        for (int k = 0; k < D; ++k)
            if (ta.nmem[k] > 1) atomicOr(bm + ta.bm_off[k] + (smp.c[k] >> 5), 1u << (smp.c[k] & 31));
    }
}

template <typename T> struct TVec;
template <> struct TVec<float> { using type = float4; static constexpr int n = 4; };
template <> struct TVec<double> { using type = double2; static constexpr int n = 2; };

// every touched row owned by another member: its owner's A row into the local copy
template <typename T>
__global__ void __launch_bounds__(256) k_tsn_import(ncclDevComm comm, ncclWindow_t winA, ncclWindow_t winBM,
                                                    int cur, const TsnArgs ta) {
    using V = typename TVec<T>::type;
    constexpr int VE = TVec<T>::n;
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamLsa(comm), comm.lsaBarrier, blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);   // owners' previous Adam is complete everywhere
    const uint32_t* bm = static_cast<const uint32_t*>(ncclGetLocalPointer(winBM, 0)) + (int64_t)cur * ta.bm_words;
    T* A = static_cast<T*>(ncclGetLocalPointer(winA, 0));
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    const int vpr = ta.R_pad / VE;   // 16-B vectors per row
    // a half-warp per 32-row bitmap word (coalesced word loads; only touched
    // rows owned elsewhere cost a remote load): each set, foreign bit's row is
    // copied by the half-warp's lanes, all its vectors in flight at once
    const int hl = threadIdx.x & 15;
    const int64_t half = tid >> 4, nhalf = nt >> 4;
    for (int k = 0; k < ta.d; ++k) {
        if (ta.nmem[k] <= 1) continue;
        const int64_t nw = (ta.rows[k] + 31) >> 5;
        const int64_t own0 = (int64_t)ta.me[k] * ta.shard[k], own1 = own0 + ta.shard[k];
        for (int64_t w = half; w < nw; w += nhalf) {
            uint32_t bits = bm[ta.bm_off[k] + w];
            // drop my own rows
            const int64_t rb = w << 5;
            for (int i = 0; i < 32 && bits; ++i)
                if (rb + i >= own0 && rb + i < own1) bits &= ~(1u << i);
            while (bits) {
                const int i = __ffs(bits) - 1;
                bits &= bits - 1;
                const int64_t r = rb + i;
                const int owner = (int)(r / ta.shard[k]);
                for (int v = hl; v < vpr; v += 16) {
                    const size_t e = (size_t)(ta.off[k] + r * ta.R_pad) + (size_t)v * VE;
                    *reinterpret_cast<V*>(A + e) =
                        *static_cast<const V*>(ncclGetLsaPointer(winA, e * sizeof(T), ta.mem[k][owner]));
                }
            }
        }
    }
}

// owned rows: G summed over the members that touched them, Alg. 1, then the
// previous parity's G rows and bits cleared
template <typename T>
__global__ void __launch_bounds__(256) k_tsn_export(ncclDevComm comm, ncclWindow_t winA, ncclWindow_t winG,
                                                    ncclWindow_t winGprev, ncclWindow_t winBM, int cur,
                                                    T* __restrict__ B, T* __restrict__ C, const TsnArgs ta, T rate,
                                                    T b1, T b2, T eps, T bc1, T bc2, T lower, const DevStep* step,
                                                    long long t_off) {
    using V = typename TVec<T>::type;
    constexpr int VE = TVec<T>::n;
    if (step) {   // graph replay: t = t0 + offset, bias corrections in fp64 from it
        const double t = (double)(step->t + t_off);
        rate = (T)step->rate;
        bc1 = (T)(1.0 / (1.0 - pow(step->beta1, t)));
        bc2 = (T)(1.0 / (1.0 - pow(step->beta2, t)));
    }
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamLsa(comm), comm.lsaBarrier, blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);   // every member's K2 of this iteration is complete
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    const int vpr = ta.R_pad / VE;
    T* A = static_cast<T*>(ncclGetLocalPointer(winA, 0));
    // clear the previous parity: my G rows marked by my previous bits, then the bits
    {
        const uint32_t* pbm =
            static_cast<const uint32_t*>(ncclGetLocalPointer(winBM, 0)) + (int64_t)(cur ^ 1) * ta.bm_words;
        T* Gp = static_cast<T*>(ncclGetLocalPointer(winGprev, 0));
        V z;
        T* zp = reinterpret_cast<T*>(&z);
#pragma unroll
        for (int q = 0; q < VE; ++q) zp[q] = T(0);
        for (int k = 0; k < ta.d; ++k) {
            if (ta.nmem[k] <= 1) {   // no slice group, no bits: the mode's G rows are cleared whole
                const int64_t nv = ta.rows[k] * vpr;
                for (int64_t v = tid; v < nv; v += nt) *reinterpret_cast<V*>(Gp + ta.off[k] + v * VE) = z;
                continue;
            }
            // a half-warp per bitmap word: the previous iteration's touched rows only
            const int hl = threadIdx.x & 15;
            const int64_t nw = (ta.rows[k] + 31) >> 5;
            for (int64_t w = tid >> 4; w < nw; w += nt >> 4) {
                uint32_t bits = pbm[ta.bm_off[k] + w];
                while (bits) {
                    const int i = __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int64_t r = (w << 5) + i;
                    for (int v = hl; v < vpr; v += 16)
                        *reinterpret_cast<V*>(Gp + ta.off[k] + r * ta.R_pad + v * VE) = z;
                }
            }
        }
        // (the bits themselves are cleared by a memset after this kernel: other
        // CTAs of this launch may still be reading them here)
    }
    // owned rows, a warp per 32-row bitmap word: lanes < g load the members'
    // words of this iteration (one remote load each, in parallel), the warp
    // shares them by shuffles, then walks the word's rows x vectors issuing every
    // needed peer G load of a vector before summing (two NVLink round trips per
    // word instead of one per member and vector)
    const int lane = threadIdx.x & 31;
    const int64_t warp = tid >> 5, nwarp = nt >> 5;
    for (int k = 0; k < ta.d; ++k) {
        const int64_t r0 = (int64_t)ta.me[k] * ta.shard[k], r1 = r0 + ta.shard[k];
        const int nm = ta.nmem[k];
        const int64_t w0 = r0 >> 5, w1 = (r1 + 31) >> 5;
        for (int64_t w = w0 + warp; w < w1; w += nwarp) {
            uint32_t mine = 0u;
            if (lane < nm && lane != ta.me[k] && nm > 1)
                mine = *static_cast<const uint32_t*>(ncclGetLsaPointer(
                    winBM, ((size_t)cur * ta.bm_words + ta.bm_off[k] + w) * sizeof(uint32_t), ta.mem[k][lane]));
            uint32_t bits[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) bits[m] = __shfl_sync(0xffffffffu, mine, m);
            const int items = 32 * vpr;
            for (int it = lane; it < items; it += 32) {
                const int64_t r = (w << 5) + it / vpr;
                if (r < r0 || r >= r1) continue;
                const int64_t e = ta.off[k] + r * ta.R_pad + (it % vpr) * VE;
                const size_t ob = (size_t)e * sizeof(T);
                V g = *static_cast<const V*>(ncclGetLocalPointer(winG, ob));
                V h[8];
#pragma unroll
                for (int m = 0; m < 8; ++m)
                    if (m < nm && ((bits[m] >> (r & 31)) & 1u))
                        h[m] = *static_cast<const V*>(ncclGetLsaPointer(winG, ob, ta.mem[k][m]));
                V a = *reinterpret_cast<const V*>(A + e);
                V bb = *reinterpret_cast<const V*>(B + e);
                V cc = *reinterpret_cast<const V*>(C + e);
                T* gp = reinterpret_cast<T*>(&g);
#pragma unroll
                for (int m = 0; m < 8; ++m)
                    if (m < nm && ((bits[m] >> (r & 31)) & 1u)) {
                        const T* hp = reinterpret_cast<const T*>(&h[m]);
#pragma unroll
                        for (int q = 0; q < VE; ++q) gp[q] += hp[q];
                    }
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
                *reinterpret_cast<V*>(A + e) = a;
                *reinterpret_cast<V*>(B + e) = bb;
                *reinterpret_cast<V*>(C + e) = cc;
            }
        }
    }
}

#define TSN_CUDA(c, x, what)                                    \
    do {                                                        \
        cudaError_t e_ = (x);                                   \
        if (e_ != cudaSuccess) return cuda_fail((c), e_, what); \
    } while (0)

bool tsn_possible(gcp_ctx* c) {
    if (c->P <= 1 || c->mode != GCP_DIST_SYNC_TWO_SIDED) return false;
    const char* env = getenv("GCP_TWOSIDED_NVL");
    if (env && std::string(env) == "0") return false;
    for (int k = 0; k < c->d; ++k)
        if (c->slice_size[k] > 8) return false;
    const ncclTeam_t lsa = ncclTeamLsa(c->world);
    return lsa.nRanks == c->P;
}

static TsnArgs tsn_args(const gcp_ctx* c) {
    TsnArgs ta;
    memset(&ta, 0, sizeof(ta));
    ta.d = c->d;
    ta.R_pad = c->R_pad;
    int64_t w = 0;
    for (int k = 0; k < c->d; ++k) {
        ta.off[k] = c->off[k];
        ta.rows[k] = c->rows[k];
        ta.bm_off[k] = w;
        w += (c->rows[k] + 31) / 32;
        ta.shard[k] = c->rows[k] / c->slice_size[k];
        ta.me[k] = c->slice_rank[k];
        ta.nmem[k] = c->fnmem[k];
        for (int m = 0; m < c->fnmem[k]; ++m) ta.mem[k][m] = c->fmem[k][m];
    }
    ta.bm_words = w;
    return ta;
}

size_t tsn_bitmap_bytes(const gcp_ctx* c) {
    int64_t w = 0;
    for (int k = 0; k < c->d; ++k) w += (c->rows[k] + 31) / 32;
    return (size_t)(2 * w) * sizeof(uint32_t);
}

// touch pass + import, before the iteration's K2 (gcp_loss_grad)
gcp_status tsn_import(gcp_ctx* c, const SampleArgs& sa) {
    const TsnArgs ta = tsn_args(c);
    const int cur = (int)(c->it & 1);
    uint32_t* bm = static_cast<uint32_t*>(c->d_bm) + (int64_t)cur * ta.bm_words;
    const int nb = c->sm_count * 8;
    const bool f32 = c->prec == GCP_FP32;
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    switch (c->d) {
    case 2: f32 ? k_tsn_touch<float, 2><<<nb, 256, 0, c->stream>>>(sa, bm, ta) : k_tsn_touch<double, 2><<<nb, 256, 0, c->stream>>>(sa, bm, ta); break;
    case 3: f32 ? k_tsn_touch<float, 3><<<nb, 256, 0, c->stream>>>(sa, bm, ta) : k_tsn_touch<double, 3><<<nb, 256, 0, c->stream>>>(sa, bm, ta); break;
    case 4: f32 ? k_tsn_touch<float, 4><<<nb, 256, 0, c->stream>>>(sa, bm, ta) : k_tsn_touch<double, 4><<<nb, 256, 0, c->stream>>>(sa, bm, ta); break;
    case 5: f32 ? k_tsn_touch<float, 5><<<nb, 256, 0, c->stream>>>(sa, bm, ta) : k_tsn_touch<double, 5><<<nb, 256, 0, c->stream>>>(sa, bm, ta); break;
    default: f32 ? k_tsn_touch<float, 6><<<nb, 256, 0, c->stream>>>(sa, bm, ta) : k_tsn_touch<double, 6><<<nb, 256, 0, c->stream>>>(sa, bm, ta); break;
    }
    TSN_CUDA(c, cudaGetLastError(), "two-sided touch");
    if (f32)
        k_tsn_import<float><<<c->fused_ctas, 256, 0, c->stream>>>(c->devcomm, c->winA, c->winBM, cur, ta);
    else
        k_tsn_import<double><<<c->fused_ctas, 256, 0, c->stream>>>(c->devcomm, c->winA, c->winBM, cur, ta);
    TSN_CUDA(c, cudaGetLastError(), "two-sided import");
    c->launches += 2;
    prof_end(c, PROF_COMM, ev);
    return GCP_OK;
}

// export + Adam on the owned rows (gcp_adam_step)
gcp_status tsn_export(gcp_ctx* c, const gcp_adam_params* p, double lower) {
    const TsnArgs ta = tsn_args(c);
    const int cur = (int)(c->it & 1);
    const double bc1 = 1.0 / (1.0 - pow(p->beta1, (double)c->t));
    const double bc2 = 1.0 / (1.0 - pow(p->beta2, (double)c->t));
    const DevStep* step = c->capturing ? c->d_step : nullptr;
    const long long toff = (long long)(c->t - c->graph_t0);
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    if (c->prec == GCP_FP32)
        k_tsn_export<float><<<c->fused_ctas, 256, 0, c->stream>>>(
            c->devcomm, c->winA, c->winG[cur], c->winG[cur ^ 1], c->winBM, cur, (float*)c->d_B, (float*)c->d_C, ta,
            (float)p->rate, (float)p->beta1, (float)p->beta2, (float)p->eps, (float)bc1, (float)bc2, (float)lower,
            step, toff);
    else
        k_tsn_export<double><<<c->fused_ctas, 256, 0, c->stream>>>(
            c->devcomm, c->winA, c->winG[cur], c->winG[cur ^ 1], c->winBM, cur, (double*)c->d_B, (double*)c->d_C, ta,
            p->rate, p->beta1, p->beta2, p->eps, bc1, bc2, lower, step, toff);
    TSN_CUDA(c, cudaGetLastError(), "two-sided export");
    // the previous parity's bits: every member read them in the previous export
    // (all passed this export's barrier), the next touch pass writes them
    TSN_CUDA(c, cudaMemsetAsync(static_cast<uint32_t*>(c->d_bm) + (int64_t)(cur ^ 1) * ta.bm_words, 0,
                                (size_t)ta.bm_words * sizeof(uint32_t), c->stream),
             "two-sided bits");
    c->launches += 1;
    prof_end(c, PROF_COMM, ev);
    return GCP_OK;
}

}  // namespace gcp
