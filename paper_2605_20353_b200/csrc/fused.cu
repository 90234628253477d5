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

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "gcp_internal.h"

namespace gcp {

constexpr int kFusedCTAsPerSM = 1;   // CTAs of the fused exchange per SM (== LSA barriers requested / SMs);
                                     // more CTAs only lengthen the barriers (profiles/r01_summary.md)

struct FusedArgs {
    int d, R_pad;
    int64_t off[kMaxModes];           // element offset of mode k (identical on every rank)
    int64_t shard_start[kMaxModes];   // first block row of my shard
    int64_t vec_begin[kMaxModes + 1]; // prefix over modes of my shard's 16-B vectors
    int nmem[kMaxModes];
    int mem[kMaxModes][8];            // LSA ranks of the mode-k slice members (incl. me)
    int mm[kMaxModes];                // 1: mode k's slice group is the whole LSA team -> NVLS multimem
    int mm_any;
    int64_t zero_vecs;                // 16-B vectors of the local G buffer to zero
    unsigned long long* trace;        // diagnostics (GCP_FUSED_TRACE=1): per-CTA %globaltimer stamps
};

constexpr int kTraceStamps = 4 + kMaxModes;   // start, barrier 1, zeroing, each mode, barrier 2

__device__ __forceinline__ void fstamp(const FusedArgs& fa, int i) {
    if (fa.trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        fa.trace[(size_t)blockIdx.x * kTraceStamps + i] = t;
    }
}

// NVLink SHARP (NVLS) through the NVSwitch multicast object of the windows:
// one load returns the sum over every rank's copy (reduction in the switch),
// one store writes every rank's copy.
__device__ __forceinline__ float4 mm_ld_reduce(const float* p) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ void mm_st(float* p, float4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

template <typename T> struct FVec;
template <> struct FVec<float> { using type = float4; static constexpr int n = 4; };
template <> struct FVec<double> { using type = double2; static constexpr int n = 2; };

// The owned shard of one mode: reduce-scatter of G over the slice members,
// Alg. 1 with the rank-local moments, all-gather of the new rows.  U vectors
// per thread per step, every load of the step issued before any arithmetic
// (bytes in flight over NVLink); MM: one multimem load / store per vector
// (NVLS), else up to MAXM unicast peer loads and nm peer stores per vector.
template <typename T, int U, int MAXM, bool MM>
__device__ __forceinline__ void exchange_rows(const ncclDevComm& comm, ncclWindow_t winA, ncclWindow_t winG,
                                              T* __restrict__ B, T* __restrict__ C, int64_t e0, int64_t nv,
                                              const int* mem, int nm, T rate, T b1, T b2, T eps, T bc1, T bc2,
                                              T lower, int64_t tid, int64_t nt) {
    using V = typename FVec<T>::type;
    constexpr int VE = FVec<T>::n;
    for (int64_t v0 = tid; v0 < nv; v0 += nt * U) {
        V g[U], a[U], bb[U], cc[U];
        V h[U][MAXM];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + (int64_t)u * nt;
            if (v >= nv) continue;
            const int64_t e = e0 + v * VE;
            const size_t ob = (size_t)e * sizeof(T);
            if constexpr (MM) {
                const float4 r = mm_ld_reduce(static_cast<const float*>(ncclGetLsaMultimemPointer(winG, ob, comm)));
                g[u] = *reinterpret_cast<const V*>(&r);
            } else {
#pragma unroll
                for (int m = 0; m < MAXM; ++m)
                    if (m < nm) h[u][m] = *reinterpret_cast<const V*>(ncclGetLsaPointer(winG, ob, mem[m]));
            }
            a[u] = *reinterpret_cast<const V*>(ncclGetLocalPointer(winA, ob));
            bb[u] = *reinterpret_cast<const V*>(B + e);
            cc[u] = *reinterpret_cast<const V*>(C + e);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + (int64_t)u * nt;
            if (v >= nv) continue;
            const int64_t e = e0 + v * VE;
            const size_t ob = (size_t)e * sizeof(T);
            if constexpr (!MM) {
                g[u] = h[u][0];
                T* gp = reinterpret_cast<T*>(&g[u]);
#pragma unroll
                for (int m = 1; m < MAXM; ++m) {
                    if (m >= nm) break;
                    const T* hp = reinterpret_cast<const T*>(&h[u][m]);
#pragma unroll
                    for (int q = 0; q < VE; ++q) gp[q] += hp[q];
                }
            }
            const T* gp = reinterpret_cast<const T*>(&g[u]);
            T* ap = reinterpret_cast<T*>(&a[u]);
            T* bp = reinterpret_cast<T*>(&bb[u]);
            T* cp = reinterpret_cast<T*>(&cc[u]);
#pragma unroll
            for (int q = 0; q < VE; ++q) {
                const T gv = gp[q];
                bp[q] = b1 * bp[q] + (T(1) - b1) * gv;
                cp[q] = b2 * cp[q] + (T(1) - b2) * gv * gv;
                const T av = ap[q] - rate * ((bp[q] * bc1) / sqrt(cp[q] * bc2 + eps));
                ap[q] = (av < lower) ? lower : av;
            }
            *reinterpret_cast<V*>(B + e) = bb[u];
            *reinterpret_cast<V*>(C + e) = cc[u];
            if constexpr (MM) {
                mm_st(static_cast<float*>(ncclGetLsaMultimemPointer(winA, ob, comm)),
                      *reinterpret_cast<const float4*>(&a[u]));
            } else {
                for (int m = 0; m < nm; ++m) *reinterpret_cast<V*>(ncclGetLsaPointer(winA, ob, mem[m])) = a[u];
            }
        }
    }
}

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
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamLsa(comm), comm.lsaBarrier, blockIdx.x,
                                           fa.mm_any != 0, comm.lsaMultimem);
    fstamp(fa, 0);
    // every rank's K2 of this iteration is complete (stream order before arrive)
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    fstamp(fa, 1);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    {
        V z;
        T* zp = reinterpret_cast<T*>(&z);
#pragma unroll
        for (int q = 0; q < VE; ++q) zp[q] = T(0);
        for (int64_t x = tid; x < fa.zero_vecs; x += nt) reinterpret_cast<V*>(gzero)[x] = z;
    }
    fstamp(fa, 2);
    for (int k = 0; k < fa.d; ++k) {
        const int64_t nv = fa.vec_begin[k + 1] - fa.vec_begin[k];
        const int64_t e0 = fa.off[k] + fa.shard_start[k] * fa.R_pad;   // first owned element of mode k
        const int nm = fa.nmem[k];
        bool done = false;
        if constexpr (sizeof(T) == 4) {
            if (fa.mm[k]) {
                exchange_rows<T, 4, 1, true>(comm, winA, winG, B, C, e0, nv, fa.mem[k], nm, rate, b1, b2, eps, bc1,
                                             bc2, lower, tid, nt);
                done = true;
            }
        }
        if (!done) {
            if (nm <= 2)
                exchange_rows<T, 4, 2, false>(comm, winA, winG, B, C, e0, nv, fa.mem[k], nm, rate, b1, b2, eps, bc1,
                                              bc2, lower, tid, nt);
            else
                exchange_rows<T, 1, 8, false>(comm, winA, winG, B, C, e0, nv, fa.mem[k], nm, rate, b1, b2, eps, bc1,
                                              bc2, lower, tid, nt);
        }
        fstamp(fa, 3 + k);
    }
    // all updated rows visible on every member before any next K2
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    fstamp(fa, 3 + kMaxModes);
}

#define NCCL_TRY_F(c, x, what)                                      \
    do {                                                            \
        ncclResult_t r_ = (x);                                      \
        if (r_ != ncclSuccess) return nccl_fail((c), r_, what);     \
    } while (0)

static constexpr size_t kFusedCacheMax = (size_t)4 << 30;   // 4 GiB of kept windows at most

static size_t round_win(size_t b) {
    const size_t g = (size_t)2 << 20;   // symmetric windows: whole 2-MB granules
    return (b + g - 1) / g * g;
}

// NVLS for the modes whose slice group is the whole team: GCP_MULTIMEM=1 forces
// it, 0 disables it, unset = from 8 ranks up.  On 4 B200s unicast NVLink loads
// and stores beat multimem.ld_reduce / multimem.st by ~20% (tools/nvlsbench.cu,
// profiles/r01_summary.md); multicast only cuts the incoming bytes of the
// reduce-scatter from (g-1)/g to 1/g of the block, which pays for larger g.
bool fused_use_multimem(const gcp_ctx* c) {
    if (!c->fused || !c->multimem || c->prec != GCP_FP32 || c->P < 2) return false;
    const char* env = getenv("GCP_MULTIMEM");
    if (env && std::string(env) == "1") return true;
    if (env && std::string(env) == "0") return false;
    return c->P >= 8;
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

// Device communicator (LSA barriers, NVLS multicast when available), then the
// symmetric A and G[2] windows on the world communicator (collective).
gcp_status fused_alloc(gcp_ctx* c, size_t bytes) {
    const size_t wb = round_win(bytes);
    void** bufs[3] = {&c->d_A, &c->d_G, &c->d_G2};
    ncclWindow_t* wins[3] = {&c->winA, &c->winG[0], &c->winG[1]};
    if (!c->devcomm_ready) {
        ncclDevCommRequirements reqs;
        memset(&reqs, 0, sizeof(reqs));
        // every CTA must be co-resident (the LSA barrier pairs CTA i of every
        // rank): clamp the grid to the occupancy of both instantiations
        const char* cenv = getenv("GCP_FUSED_CTAS_PER_SM");
        int per_sm = cenv && atoi(cenv) > 0 ? atoi(cenv) : kFusedCTAsPerSM;
        int occ_f = 0, occ_d = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, k_fused_exchange<float>, 256, 0) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_d, k_fused_exchange<double>, 256, 0) != cudaSuccess)
            return set_error(GCP_E_CUDA, "fused exchange: occupancy query failed");
        per_sm = std::max(1, std::min(per_sm, std::min(occ_f, occ_d)));
        c->fused_ctas = c->sm_count * per_sm;
        reqs.lsaBarrierCount = c->fused_ctas;
        // NVLS multicast on the LSA team when the switch supports it (else unicast loads / stores)
        const char* mmenv = getenv("GCP_MULTIMEM");
        reqs.lsaMultimem = !(mmenv && std::string(mmenv) == "0");
        ncclResult_t r = ncclDevCommCreate(c->world, &reqs, &c->devcomm);
        if (r != ncclSuccess && reqs.lsaMultimem) {
            reqs.lsaMultimem = false;
            r = ncclDevCommCreate(c->world, &reqs, &c->devcomm);
        }
        NCCL_TRY_F(c, r, "ncclDevCommCreate");
        c->devcomm_ready = true;
        c->multimem = reqs.lsaMultimem && c->devcomm.lsaMultimem.mcBasePtr != nullptr;
    }
    c->fwin_bytes = wb;
    // every rank pads to the same window size, so all take the same branch here
    if (c->fcache_bytes == wb) {
        for (int i = 0; i < 3; ++i) {
            *bufs[i] = c->fcache_buf[i];
            *wins[i] = c->fcache_win[i];
            c->fcache_buf[i] = nullptr;
            c->fcache_win[i] = nullptr;
        }
        c->fcache_bytes = 0;
    } else {
        fused_cache_release(c);
        for (int i = 0; i < 3; ++i) {
            NCCL_TRY_F(c, ncclMemAlloc(bufs[i], wb), "ncclMemAlloc");
            NCCL_TRY_F(c, ncclCommWindowRegister(c->world, *bufs[i], wb, wins[i], NCCL_WIN_COLL_SYMMETRIC),
                       "ncclCommWindowRegister");
        }
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

// Two-sided over NVLink (twosided_nvl.cu): the touched-row bits of both
// parities in a symmetric window of their own, zeroed.
gcp_status tsn_alloc_bitmap(gcp_ctx* c) {
    const size_t wb = round_win(std::max<size_t>(tsn_bitmap_bytes(c), 64));
    NCCL_TRY_F(c, ncclMemAlloc(&c->d_bm, wb), "ncclMemAlloc");
    NCCL_TRY_F(c, ncclCommWindowRegister(c->world, c->d_bm, wb, &c->winBM, NCCL_WIN_COLL_SYMMETRIC),
               "ncclCommWindowRegister");
    if (cudaMemsetAsync(c->d_bm, 0, wb, c->stream) != cudaSuccess)
        return set_error(GCP_E_CUDA, "two-sided bits: memset failed");
    return GCP_OK;
}

static void fused_trace_print(gcp_ctx* c);

void fused_free(gcp_ctx* c) {
    if (!c->fused) return;
    if (c->winBM) {
        cudaStreamSynchronize(c->stream);
        ncclCommWindowDeregister(c->world, c->winBM);
        ncclMemFree(c->d_bm);
        c->winBM = nullptr;
        c->d_bm = nullptr;
    }
    fused_trace_print(c);
    if (c->ftrace) gfree(c, c->ftrace);
    c->ftrace = nullptr;
    c->ftrace_n = 0;
    for (double& x : c->ftrace_acc) x = 0.0;
    void** bufs[3] = {&c->d_A, &c->d_G, &c->d_G2};
    ncclWindow_t* wins[3] = {&c->winA, &c->winG[0], &c->winG[1]};
    cudaStreamSynchronize(c->stream);
    fused_cache_release(c);
    // keep up to min(kFusedCacheMax, 1/32 of device memory) of registered
    // windows for the next model of the same size (replace-ingest jobs skip the
    // collective deregister / register).  The decision must agree on every rank
    // (deregistration is collective): it depends only on the symmetric window
    // size and the device's total memory, never on its free memory.  The kept
    // windows live outside the allocation pool until the next model of the same
    // size or gcp_destroy (include/gcp.h, gcp_model_init).
    const size_t wb = c->fwin_bytes;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t cap = std::min(kFusedCacheMax, tot / 32);
    const bool keep = !c->closing && 3 * wb <= cap && *wins[0] && *wins[1] && *wins[2];
    for (int i = 0; i < 3; ++i) {
        if (keep) {
            c->fcache_buf[i] = *bufs[i];
            c->fcache_win[i] = *wins[i];
        } else {
            if (*wins[i]) ncclCommWindowDeregister(c->world, *wins[i]);
            if (*bufs[i]) ncclMemFree(*bufs[i]);
        }
        *wins[i] = nullptr;
        *bufs[i] = nullptr;
    }
    c->fcache_bytes = keep ? wb : 0;
    c->fused = false;
}

void fused_cache_release(gcp_ctx* c) {
    for (int i = 0; i < 3; ++i) {
        if (c->fcache_win[i]) ncclCommWindowDeregister(c->world, c->fcache_win[i]);
        if (c->fcache_buf[i]) ncclMemFree(c->fcache_buf[i]);
        c->fcache_win[i] = nullptr;
        c->fcache_buf[i] = nullptr;
    }
    c->fcache_bytes = 0;
}

#define CUDA_TRY_F(c, x, what)                                  \
    do {                                                        \
        cudaError_t e_ = (x);                                   \
        if (e_ != cudaSuccess) return cuda_fail((c), e_, what); \
    } while (0)

// Diagnostics: GCP_FUSED_TRACE=1 stamps %globaltimer per CTA at each phase of
// the fused exchange and syncs after every launch (never inside a graph);
// fused_free prints the mean phase ends (max over CTAs, relative to the
// earliest CTA start) to stderr.
static bool fused_trace_on() {
    const char* env = getenv("GCP_FUSED_TRACE");
    return env && std::string(env) == "1";
}

static void fused_trace_collect(gcp_ctx* c) {
    std::vector<unsigned long long> h((size_t)kTraceStamps * c->fused_ctas);
    if (cudaMemcpyAsync(h.data(), c->ftrace, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost, c->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess)
        return;
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < c->fused_grid; ++b) t0 = std::min(t0, h[(size_t)b * kTraceStamps]);
    for (int i = 1; i < kTraceStamps; ++i) {
        unsigned long long mx = 0;
        for (int b = 0; b < c->fused_grid; ++b) mx = std::max(mx, h[(size_t)b * kTraceStamps + i]);
        c->ftrace_acc[i] += mx > t0 ? (double)(mx - t0) * 1e-3 : 0.0;
    }
    c->ftrace_n += 1;
}

static void fused_trace_print(gcp_ctx* c) {
    if (!c->ftrace_n) return;
    fprintf(stderr, "[gcp rank %d] fused exchange trace, us after the first CTA start (mean of %lld): "
                    "barrier1 %.1f zero %.1f", c->rank, (long long)c->ftrace_n, c->ftrace_acc[1] / c->ftrace_n,
            c->ftrace_acc[2] / c->ftrace_n);
    for (int k = 0; k < c->d; ++k) fprintf(stderr, " mode%d %.1f", k, c->ftrace_acc[3 + k] / c->ftrace_n);
    fprintf(stderr, " barrier2 %.1f\n", c->ftrace_acc[3 + kMaxModes] / c->ftrace_n);
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
        fa.mm[k] = fused_use_multimem(c) && c->fnmem[k] == c->P;
        fa.mm_any |= fa.mm[k];
    }
    fa.vec_begin[c->d] = acc;
    fa.zero_vecs = c->n_coef / VE;
    // grid: one CTA per SM.  Fewer CTAs for the small c2 exchange (32-64 of
    // 148) measured within run-to-run noise (profiles/fused_grid_r01.sh).
    // Must be identical on every rank: the barrier pairs CTA i across ranks.
    // GCP_FUSED_GRID overrides (experiments).
    int grid = c->fused_ctas;
    const char* genv = getenv("GCP_FUSED_GRID");
    if (genv && atoi(genv) > 0) grid = std::min(c->fused_ctas, atoi(genv));
    c->fused_grid = grid;
    fa.trace = nullptr;
    if (!c->capturing && fused_trace_on()) {
        if (!c->ftrace) {
            const size_t b = sizeof(unsigned long long) * kTraceStamps * c->fused_ctas;
            CUDA_TRY_F(c, gmalloc(c, &c->ftrace, b), "trace alloc");
            CUDA_TRY_F(c, cudaMemsetAsync(c->ftrace, 0, b, c->stream), "trace alloc");
        }
        fa.trace = (unsigned long long*)c->ftrace;
    }
    const int cur = (int)(c->it & 1);
    void* gnext = cur ? c->d_G : c->d_G2;
    const double bc1 = 1.0 / (1.0 - pow(p->beta1, (double)c->t));
    const double bc2 = 1.0 / (1.0 - pow(p->beta2, (double)c->t));
    cudaEvent_t ev;
    prof_begin(c, PROF_COMM, &ev);
    if (c->prec == GCP_FP32)
        k_fused_exchange<float><<<grid, 256, 0, c->stream>>>(
            c->devcomm, c->winA, c->winG[cur], (float*)gnext, (float*)c->d_B, (float*)c->d_C, fa, (float)p->rate,
            (float)p->beta1, (float)p->beta2, (float)p->eps, (float)bc1, (float)bc2, (float)lower,
            c->capturing ? c->d_step : nullptr, (long long)(c->t - c->graph_t0));
    else
        k_fused_exchange<double><<<grid, 256, 0, c->stream>>>(
            c->devcomm, c->winA, c->winG[cur], (double*)gnext, (double*)c->d_B, (double*)c->d_C, fa, p->rate,
            p->beta1, p->beta2, p->eps, bc1, bc2, lower, c->capturing ? c->d_step : nullptr,
            (long long)(c->t - c->graph_t0));
    prof_end(c, PROF_COMM, ev);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "fused exchange");
    if (fa.trace) fused_trace_collect(c);
    return GCP_OK;
}

}  // namespace gcp
