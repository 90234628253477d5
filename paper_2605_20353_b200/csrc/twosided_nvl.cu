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
//   export  (k_tsn_pull)    LSA barrier (every rank's K2 done); the owner of a
//                           row adds to its own G row the G rows of exactly
//                           the members whose bitmap marks the row (the
//                           paper's export of partial rows to their owner,
//                           pulled by the owner) and zeroes the previous
//                           parity's G rows; then k_adam (Alg. 1) on the owned
//                           rows and a memset of the previous parity's bits
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
            if (ta.nmem[k] > 1) {
                GCP_CHECK(smp.c[k] < ta.rows[k], "touched row", smp.c[k], ta.rows[k]);
                atomicOr(bm + ta.bm_off[k] + (smp.c[k] >> 5), 1u << (smp.c[k] & 31));
            }
    }
}

template <typename T> struct TVec;
template <> struct TVec<float> { using type = float4; static constexpr int n = 4; };
template <> struct TVec<double> { using type = double2; static constexpr int n = 2; };

// every touched row owned by another member: its owner's A row into the local
// copy.  A thread per 16-B vector of the non-owned rows, four in flight (the
// bitmap words are L1 hits shared by the warp; only touched rows cost a remote load).
template <typename T>
__global__ void __launch_bounds__(512) k_tsn_import(ncclDevComm comm, ncclWindow_t winA, ncclWindow_t winBM,
                                                    int cur, const TsnArgs ta) {
    using V = typename TVec<T>::type;
    constexpr int VE = TVec<T>::n;
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamLsa(comm), comm.lsaBarrier, blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);   // owners' previous Adam is complete everywhere
    const uint32_t* bm = static_cast<const uint32_t*>(ncclGetLocalPointer(winBM, 0)) + (int64_t)cur * ta.bm_words;
    T* A = static_cast<T*>(ncclGetLocalPointer(winA, 0));
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    const int vpr = ta.R_pad / VE;   // 16-B vectors per row
    for (int k = 0; k < ta.d; ++k) {
        if (ta.nmem[k] <= 1) continue;
        const int64_t own0 = (int64_t)ta.me[k] * ta.shard[k];
        const int64_t nv = (ta.rows[k] - ta.shard[k]) * vpr;   // vectors of the rows owned elsewhere
        for (int64_t v0 = tid; v0 < nv; v0 += 4 * nt) {
            V val[4];
            int64_t ev[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t v = v0 + u * nt;
                ev[u] = -1;
                if (v >= nv) continue;
                int64_t r = v / vpr;
                if (r >= own0) r += ta.shard[k];   // skip my own shard
                GCP_CHECK(r < ta.rows[k] && r / ta.shard[k] < ta.nmem[k], "import row", r, ta.rows[k]);
                if (!((bm[ta.bm_off[k] + (r >> 5)] >> (r & 31)) & 1u)) continue;
                ev[u] = ta.off[k] + r * ta.R_pad + (v % vpr) * VE;
                val[u] = *static_cast<const V*>(
                    ncclGetLsaPointer(winA, (size_t)ev[u] * sizeof(T), ta.mem[k][(int)(r / ta.shard[k])]));
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (ev[u] >= 0) *reinterpret_cast<V*>(A + ev[u]) = val[u];
        }
    }
}

// The owner's side of the export: after the barrier (every member's K2 of this
// iteration is complete) each owned row's G gets the G rows of exactly the
// members whose bitmap marks it (a thread per 16-B vector, the members' bit
// words and rows for four vectors in flight), and the previous parity's G rows
// are cleared (a thread per bit word).  Adam on the owned rows follows as the
// ordinary k_adam launch (tsn_export).
template <typename T>
__global__ void __launch_bounds__(512) k_tsn_pull(ncclDevComm comm, ncclWindow_t winG, ncclWindow_t winGprev,
                                                  ncclWindow_t winBM, int cur, const TsnArgs ta) {
    using V = typename TVec<T>::type;
    constexpr int VE = TVec<T>::n;
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamLsa(comm), comm.lsaBarrier, blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    const int vpr = ta.R_pad / VE;
    V z;
    T* zp = reinterpret_cast<T*>(&z);
#pragma unroll
    for (int q = 0; q < VE; ++q) zp[q] = T(0);
    // clear the previous parity: my G rows marked by my previous bits (modes
    // without a slice group keep no bits: cleared whole).  The bits themselves
    // are cleared by a memset after this kernel (other CTAs may still read them).
    {
        const uint32_t* pbm =
            static_cast<const uint32_t*>(ncclGetLocalPointer(winBM, 0)) + (int64_t)(cur ^ 1) * ta.bm_words;
        T* Gp = static_cast<T*>(ncclGetLocalPointer(winGprev, 0));
        for (int k = 0; k < ta.d; ++k) {
            if (ta.nmem[k] <= 1) {
                const int64_t nv = ta.rows[k] * vpr;
                for (int64_t v = tid; v < nv; v += nt) *reinterpret_cast<V*>(Gp + ta.off[k] + v * VE) = z;
                continue;
            }
            const int64_t nw = (ta.rows[k] + 31) >> 5;
            for (int64_t w = tid; w < nw; w += nt) {
                uint32_t bits = pbm[ta.bm_off[k] + w];
                while (bits) {
                    const int i = __ffs(bits) - 1;
                    bits &= bits - 1;
                    T* row = Gp + ta.off[k] + ((w << 5) + i) * ta.R_pad;
                    for (int v = 0; v < vpr; ++v) *reinterpret_cast<V*>(row + v * VE) = z;
                }
            }
        }
    }
    T* G = static_cast<T*>(ncclGetLocalPointer(winG, 0));
    for (int k = 0; k < ta.d; ++k) {
        const int nm = ta.nmem[k];
        if (nm <= 1) continue;
        const int64_t r0 = (int64_t)ta.me[k] * ta.shard[k];
        const int64_t nv = ta.shard[k] * vpr;
        for (int64_t v0 = tid; v0 < nv; v0 += 4 * nt) {
            uint32_t bits[4][8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t v = v0 + u * nt;
                const int64_t r = r0 + (v < nv ? v / vpr : 0);
                const size_t wb = ((size_t)cur * ta.bm_words + ta.bm_off[k] + (r >> 5)) * sizeof(uint32_t);
#pragma unroll
                for (int m = 0; m < 8; ++m)
                    bits[u][m] = (v < nv && m < nm && m != ta.me[k])
                                     ? *static_cast<const uint32_t*>(ncclGetLsaPointer(winBM, wb, ta.mem[k][m]))
                                     : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t v = v0 + u * nt;
                if (v >= nv) continue;
                const int64_t r = r0 + v / vpr;
                const int64_t e = ta.off[k] + r * ta.R_pad + (v % vpr) * VE;
                V h[8];
                bool any = false;
#pragma unroll
                for (int m = 0; m < 8; ++m)
                    if ((bits[u][m] >> (r & 31)) & 1u) {
                        h[m] = *static_cast<const V*>(ncclGetLsaPointer(winG, (size_t)e * sizeof(T), ta.mem[k][m]));
                        any = true;
                    }
                if (!any) continue;
                V g = *reinterpret_cast<const V*>(G + e);
                T* gp = reinterpret_cast<T*>(&g);
#pragma unroll
                for (int m = 0; m < 8; ++m)
                    if ((bits[u][m] >> (r & 31)) & 1u) {
                        const T* hp = reinterpret_cast<const T*>(&h[m]);
#pragma unroll
                        for (int q = 0; q < VE; ++q) gp[q] += hp[q];
                    }
                *reinterpret_cast<V*>(G + e) = g;
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

// export + Adam on the owned rows (gcp_adam_step): the pull kernel, Alg. 1 on
// the owned shards of the current G (k_adam; G is cleared a parity later), the
// previous parity's bits cleared
gcp_status tsn_export(gcp_ctx* c, const gcp_adam_params* p, double lower) {
    const TsnArgs ta = tsn_args(c);
    const int cur = (int)(c->it & 1);
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    if (c->prec == GCP_FP32)
        k_tsn_pull<float><<<c->fused_ctas, 512, 0, c->stream>>>(c->devcomm, c->winG[cur], c->winG[cur ^ 1], c->winBM,
                                                                cur, ta);
    else
        k_tsn_pull<double><<<c->fused_ctas, 512, 0, c->stream>>>(c->devcomm, c->winG[cur], c->winG[cur ^ 1],
                                                                 c->winBM, cur, ta);
    TSN_CUDA(c, cudaGetLastError(), "two-sided export");
    c->launches += 1;
    prof_end(c, PROF_COMM, ev);
    Segment seg;
    seg.n = 0;
    for (int k = 0; k < c->d; ++k) {
        seg.start[seg.n] = c->off[k] + (int64_t)c->slice_rank[k] * (c->rows[k] / c->slice_size[k]) * c->R_pad;
        seg.len[seg.n] = (c->rows[k] / c->slice_size[k]) * c->R_pad;
        seg.n++;
    }
    prof_begin(c, PROF_ADAM, &ev);
    TSN_CUDA(c, launch_adam(c, seg, c->d_A, cur ? c->d_G2 : c->d_G, c->d_B, c->d_C, p->rate, p->beta1, p->beta2,
                            p->eps, lower, c->capturing ? c->t - c->graph_t0 : c->t, 0, c->R_pad,
                            c->capturing ? c->d_step : nullptr),
             "two-sided adam");
    c->launches += 1;
    prof_end(c, PROF_ADAM, ev);
    // the previous parity's bits: every member read them in the previous export
    // (all passed this export's barrier), the next touch pass writes them
    TSN_CUDA(c, cudaMemsetAsync(static_cast<uint32_t*>(c->d_bm) + (int64_t)(cur ^ 1) * ta.bm_words, 0,
                                (size_t)ta.bm_words * sizeof(uint32_t), c->stream),
             "two-sided bits");
    return GCP_OK;
}

}  // namespace gcp

namespace gcp {

// ---- two-sided by peer access (default; GCP_TWOSIDED_NVL=peer) ------------
// K2 itself reaches every row owned elsewhere: it gathers the row from the
// owner's A window and scatter-adds its contribution into the owner's G
// window (red.global.add over NVLink), so only the touched rows cross the link
// -- the paper's import and export, fused into the sampling kernel -- and no
// touch pass, bitmap or copy is needed.  The step kernel then has every owner
// update its rows between two LSA barriers.
// The default two-sided implementation (up to 8 ranks): in the regime where
// the two-sided layout beats the all-reduce at all -- few samples per
// iteration against the replicated rows -- peer access is the faster one (c4
// at 4 GPUs, 1e6 samples: 47.6 ms per epoch against 98.6 for the
// import/export kernels and 95.3 for the fused all-reduce; at 1e7 / 1e8 the
// all-reduce wins over both, profiles/r02m_*).  GCP_TWOSIDED_NVL=1 selects the
// import / export kernels, =0 the NCCL send/recv path (twosided.cu).
bool tsn_peer_wanted(const gcp_ctx* c) {
    const char* env = getenv("GCP_TWOSIDED_NVL");
    if (env) return std::string(env) == "peer";
    return c->P <= 8;
}

__global__ void k_tsn_bases(ncclDevComm comm, ncclWindow_t winA, ncclWindow_t winG0, ncclWindow_t winG1, int P,
                            void** out) {
    const int r = threadIdx.x;
    if (r >= P) return;
    out[r] = ncclGetLsaPointer(winA, 0, r);
    out[8 + r] = ncclGetLsaPointer(winG0, 0, r);
    out[16 + r] = ncclGetLsaPointer(winG1, 0, r);
}

gcp_status tsn_peer_setup(gcp_ctx* c) {
    if (c->P > 8) return set_error(GCP_E_ARG, "two-sided peer access: at most 8 ranks");
    TSN_CUDA(c, gmalloc(c, &c->d_peer_bases, 24 * sizeof(void*)), "peer bases");
    TSN_CUDA(c, cudaMemsetAsync(c->d_peer_bases, 0, 24 * sizeof(void*), c->stream), "peer bases");
    k_tsn_bases<<<1, 32, 0, c->stream>>>(c->devcomm, c->winA, c->winG[0], c->winG[1], c->P, c->d_peer_bases);
    TSN_CUDA(c, cudaGetLastError(), "peer bases");
    c->launches++;
    c->tsn_peer = true;
    c->tsn_dirty = true;
    return GCP_OK;
}

// Peer access makes every member's K2 read the owners' A rows and add into
// their G rows, so a rank's own writes outside the step kernel (model init /
// set, checkpoint restore: A and G rewritten on its stream) must be complete
// on every rank before any member's next K2 -- one LSA barrier, owed from the
// write to the next gradient or loss-estimate launch.
__global__ void k_tsn_barrier(ncclDevComm comm) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamLsa(comm), comm.lsaBarrier, blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

gcp_status tsn_peer_sync(gcp_ctx* c) {
    if (!c->tsn_peer || !c->tsn_dirty) return GCP_OK;
    k_tsn_barrier<<<1, 128, 0, c->stream>>>(c->devcomm);
    TSN_CUDA(c, cudaGetLastError(), "two-sided peer barrier");
    c->launches++;
    c->tsn_dirty = false;
    return GCP_OK;
}

// barrier (every member's K2 -- and so every red.add into my G rows -- is
// complete); Alg. 1 on my owned rows of the current G, and the same rows of the
// other G parity cleared in the same pass (no member adds into it before the
// next barrier; rows owned elsewhere are never written here); barrier (every
// owner's rows are updated before any next K2 gathers them)
template <typename T>
__global__ void __launch_bounds__(512) k_tsn_peer_step(ncclDevComm comm, T* __restrict__ A, const T* __restrict__ G,
                                                       T* __restrict__ Gnext, int64_t n_coef, T* __restrict__ B,
                                                       T* __restrict__ C, const TsnArgs ta, T rate, T b1, T b2,
                                                       T eps, T bc1, T bc2, T lower, const DevStep* step,
                                                       long long t_off) {
    using V = typename TVec<T>::type;
    constexpr int VE = TVec<T>::n;
    if (step) {
        const double t = (double)(step->t + t_off);
        rate = (T)step->rate;
        bc1 = (T)(1.0 / (1.0 - pow(step->beta1, t)));
        bc2 = (T)(1.0 / (1.0 - pow(step->beta2, t)));
    }
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamLsa(comm), comm.lsaBarrier, blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    V z;
    T* zp = reinterpret_cast<T*>(&z);
#pragma unroll
    for (int q = 0; q < VE; ++q) zp[q] = T(0);
    (void)n_coef;
    for (int k = 0; k < ta.d; ++k) {
        const int64_t e0 = ta.off[k] + (int64_t)ta.me[k] * ta.shard[k] * ta.R_pad;
        const int64_t nv = ta.shard[k] * ta.R_pad / VE;
        for (int64_t v = tid; v < nv; v += nt) {
            const int64_t e = e0 + v * VE;
            V g = *reinterpret_cast<const V*>(G + e);
            V a = *reinterpret_cast<const V*>(A + e);
            V bb = *reinterpret_cast<const V*>(B + e);
            V cc = *reinterpret_cast<const V*>(C + e);
            const T* gp = reinterpret_cast<const T*>(&g);
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
            // the other parity's G: only owned rows ever receive red.adds
            // (every member adds into the owner's window), so only they are cleared
            *reinterpret_cast<V*>(Gnext + e) = z;
        }
    }
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

gcp_status tsn_peer_step(gcp_ctx* c, const gcp_adam_params* p, double lower) {
    const TsnArgs ta = tsn_args(c);
    const int cur = (int)(c->it & 1);
    void* G = cur ? c->d_G2 : c->d_G;
    void* Gn = cur ? c->d_G : c->d_G2;
    const double bc1 = 1.0 / (1.0 - pow(p->beta1, (double)c->t));
    const double bc2 = 1.0 / (1.0 - pow(p->beta2, (double)c->t));
    const DevStep* step = c->capturing ? c->d_step : nullptr;
    const long long toff = (long long)(c->t - c->graph_t0);
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    if (c->prec == GCP_FP32)
        k_tsn_peer_step<float><<<c->fused_ctas, 512, 0, c->stream>>>(
            c->devcomm, (float*)c->d_A, (const float*)G, (float*)Gn, c->n_coef, (float*)c->d_B, (float*)c->d_C, ta,
            (float)p->rate, (float)p->beta1, (float)p->beta2, (float)p->eps, (float)bc1, (float)bc2, (float)lower,
            step, toff);
    else
        k_tsn_peer_step<double><<<c->fused_ctas, 512, 0, c->stream>>>(
            c->devcomm, (double*)c->d_A, (const double*)G, (double*)Gn, c->n_coef, (double*)c->d_B, (double*)c->d_C,
            ta, p->rate, p->beta1, p->beta2, p->eps, bc1, bc2, lower, step, toff);
    TSN_CUDA(c, cudaGetLastError(), "two-sided peer step");
    c->launches += 1;
    prof_end(c, PROF_COMM, ev);
    return GCP_OK;
}

}  // namespace gcp
