// kernels.cuh -- the device kernels of the hot path, templated on the
// arithmetic type T (float / double), the number of modes D, and the lane
// geometry of a sample (GL lanes x NV 16-byte vectors cover one factor row).
//
//   k_sample  (K2)  rows a1-a5 fused: Philox draw -> record fetch or hash probe
//                   -> gather d rows -> m -> y = w df/dm -> per-mode scatter-add.
//                   loss_mode = 1 turns it into the f-sample loss estimate (a9):
//                   same draw and gather, accumulates w f(x, m), no scatter.
//   k_export        test-only: the same draws, written out as indices.
//   k_adam    (K3)  Alg. 1 over contiguous segments, G reset fused (a7).
//   k_init    (K0)  Philox U[0,1) factor initialisation (reading R12).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"

namespace gcp {

template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };

template <typename T> struct KParams {
    OrdHistArgs oh;   // gradient launches: the next iteration's slot histogram (oh.n = 0: none)
    int loss;
    int loss_mode;    // 1: loss estimate only (no scatter)
    int semi_nz;      // 1: semi-stratified nonzero value w (f'(x,m) - f'(0,m))
    int with_loss;    // accumulate sum w f(x, m)
    T w_nz, w_z;
    double* partials; // per-CTA fp64 partial of sum w f
};

__device__ __forceinline__ void red_add_v(float* p, const float (&v)[4]) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3])
                 : "memory");
}
__device__ __forceinline__ void red_add_v(double* p, const double (&v)[2]) {
    atomicAdd(p, v[0]);
    atomicAdd(p + 1, v[1]);
}

template <typename T, int N>
__device__ __forceinline__ void ldg_vec(T (&dst)[N], const T* src);
template <>
__device__ __forceinline__ void ldg_vec<float, 4>(float (&dst)[4], const float* src) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(src));
    dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
}
template <>
__device__ __forceinline__ void ldg_vec<double, 2>(double (&dst)[2], const double* src) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(src));
    dst[0] = v.x; dst[1] = v.y;
}

// Slot-order bucket of slot s (kernels.cu, launch_slot_order): nonzero slot ->
// the bucket of the mode-1 row of record j = mulhi(W0, N), looked up in a
// per-tensor table over the top bits of j (exact up to the records straddling a
// lookup cell, which only moves a slot to a neighbouring bucket); zero slot ->
// floor(c_1 B / I_1) of its attempt-0 candidate c_1 = mulhi(W0, I_1).
__device__ __forceinline__ uint32_t ord_bucket(const SampleArgs& a, const uint16_t* __restrict__ lut, int lut_shift,
                                               int bits, int64_t s, uint32_t it, uint64_t inv) {
    const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
    if (s < a.p) {
        const U64x2 w = philox((uint32_t)s, a.rank, a.kind_nz << 28, it, k0, k1);
        const uint64_t j = range_map(w.w0, (uint64_t)a.N);
        GCP_CHECK(j < (uint64_t)a.N, "nonzero index for the bucket lookup", j, a.N);
        return __ldg(lut + (j >> lut_shift));
    }
    const U64x2 w = philox((uint32_t)(s - a.p), a.rank, a.kind_z << 28, it, k0, k1);
    const uint64_t c1 = range_map(w.w0, a.bdim[0]);
    uint64_t q = __umul64hi(c1 << bits, inv);   // floor or floor - 1 (c_1 B < 2^47)
    if ((q + 1) * a.bdim[0] <= (c1 << bits)) ++q;
    return (uint32_t)q;
}

// bucket of slot s and its rank inside the bucket (arrival order of a global
// atomicAdd: the scatter then needs no reservation pass)
__device__ __forceinline__ void ord_hist_slot(const OrdHistArgs& oh, int64_t s, uint32_t it, uint64_t inv) {
    const uint32_t b = ((uint32_t)(s >> oh.tile_shift) << oh.bits) | ord_bucket(oh.sa, oh.lut, oh.lut_shift, oh.bits, s, it, inv);
    GCP_CHECK((b & ((1u << oh.bits) - 1)) < (1u << oh.bits) && s < oh.n, "histogram slot", s, b);
    oh.keys[s] = b;
    oh.ranks[s] = atomicAdd(oh.totals + b, 1u);
}

// One warp takes 32 consecutive slots: each lane draws one sample (index work
// is per thread, so Philox and the probe run once per sample), then the warp
// processes the 32 samples in GL rounds of 32/GL samples, a sample per group of
// GL lanes, each lane owning NV 16-byte vectors of every factor row.  Rounds are
// handled RB at a time with all their row loads issued before any arithmetic.
// Register budget per instantiation: small fp32 row footprints (D*NV <= 3:
// c2, c4, c5) run at kSmallMinBlocks = 3 CTAs/SM (80 regs) with two rounds of
// row loads in flight -- more loads in flight per warp beat a fourth CTA when
// rows come from DRAM (c4 K2 2.61 -> 2.48 ms, c2 1.205 -> 1.192 ms against 4
// CTAs x one round; 2 CTAs x 2 or 4 rounds were slower, profiles/r02q_*);
// small fp64 footprints (the parity mode) 3 CTAs/SM with one round (their
// doubles need the registers); larger ones run at kSampleMinBlocks with kRowRegBudget row
// vectors in flight (B200 K2 tuning, profiles/r01_summary.md).
template <typename T, int D, int NV, int VAR = 0> struct SampleGeom {
    static constexpr bool small = D * NV <= 3;
    static constexpr bool f32 = sizeof(T) == 4;
    // the peer-access variant's remote rows (NVLink latency) may want more in flight
    static constexpr bool peer = VAR == 1 && GCP_PEER_MINB > 0;
    static constexpr int minb = peer ? GCP_PEER_MINB : small ? (f32 ? kSmallMinBlocks : 3) : kSampleMinBlocks;
    static constexpr int rowregs = peer ? GCP_PEER_RBREG : small ? (f32 ? kSmallRowRegBudget : 4) : kRowRegBudget;
    static constexpr int rbcap = peer ? 4 : small ? 2 : 4;   // rounds per load batch at most
};

// position s of the visiting order -> slot (identity unless a slot order is given)
__device__ __forceinline__ int64_t slot_at(const SampleArgs& a, int64_t s, int64_t total) {
    if (!(a.order && s < total)) return s;
    const int64_t v = (int64_t)__ldg(a.order + s);
    GCP_CHECK(v < total, "order entry >= p + q", v, total);
    return v;
}

// K2 variants, one instantiation each so the default carries neither branch:
// kVarPlain; kVarPeer -- rows owned by other ranks are gathered from / added into
// their A / G windows over NVLink (two-sided by peer access); kVarWagg -- same-row
// scatter-adds of a round aggregated in registers (GCP_WAGG=1)
enum { kVarPlain = 0, kVarPeer = 1, kVarWagg = 2 };

template <typename T, int D, int GL, int NV, int VAR = kVarPlain>
__global__ void __launch_bounds__(kBlock, SampleGeom<T, D, NV, VAR>::minb) k_sample(const SampleArgs sa, const ModelArgs ma,
                                                   const KParams<T> kp) {
    constexpr int VE = Vec16<T>::n;
    constexpr int SPR = 32 / GL;                 // samples per round
    // rounds per load batch: bounded so the row registers (RB*D*NV*16 B) fit the
    // budget (a power of two, so it divides GL)
    constexpr int RB_REG = SampleGeom<T, D, NV, VAR>::rowregs / (D * NV);
    constexpr int RB_CAP = GL < SampleGeom<T, D, NV, VAR>::rbcap ? GL : SampleGeom<T, D, NV, VAR>::rbcap;
    constexpr int RB = RB_REG >= 4 && RB_CAP >= 4 ? 4 : (RB_REG >= 2 && RB_CAP >= 2 ? 2 : 1);
    const int lane = threadIdx.x & 31;
    const int grp = lane / GL, gl = lane % GL;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t total = sa.p + sa.q;
    const int64_t nchunks = (total + 31) >> 5;
    const T* __restrict__ A = static_cast<const T*>(ma.A);
    T* __restrict__ G = static_cast<T*>(ma.G);
    const int R_pad = ma.R_pad;

    // this lane's slice of lambda (zero beyond R)
    T lam[NV][VE];
    bool vok[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const int col = (gl + v * GL) * VE;
        vok[v] = col < R_pad;
        if (vok[v]) ldg_vec<T, VE>(lam[v], static_cast<const T*>(ma.lambda) + col);
        else {
#pragma unroll
            for (int e = 0; e < VE; ++e) lam[v][e] = T(0);
        }
    }

    double lacc = 0.0;
    const uint32_t hit = kp.oh.n ? iter_word(kp.oh.sa) : 0u;
    const uint64_t hinv = kp.oh.n && kp.oh.sa.bdim[0] > 1 ? (~0ull) / kp.oh.sa.bdim[0] : 0ull;
    // software pipeline: the next chunk's record / first-bucket loads are in
    // flight while this chunk's rows are gathered and scattered
    Pending<D> nxt = issue_sample<T, D>(sa, slot_at(sa, (warp0 << 5) + lane, total));
    for (int64_t chunk = warp0; chunk < nchunks; chunk += nwarps) {
        const int64_t s = (chunk << 5) + lane;
        const bool valid = s < total;
        const Pending<D> cur = nxt;
        nxt = issue_sample<T, D>(sa, slot_at(sa, ((chunk + nwarps) << 5) + lane, total));
        Sample<T, D> smp;
        if (valid) smp = resolve_sample<T, D>(sa, cur);
        else {
#pragma unroll
            for (int k = 0; k < D; ++k) smp.c[k] = 0;
            smp.x = T(0); smp.nz = false;
        }
        const T wv = smp.nz ? kp.w_nz : kp.w_z;
        const int flags = (valid ? 1 : 0) | (smp.nz ? 2 : 0);
        if (kp.oh.n) {   // next iteration's histogram: slot s (natural order), ALU work under this chunk's loads
            if (s < kp.oh.n) ord_hist_slot(kp.oh, s, hit, hinv);
        }

#pragma unroll
        for (int r0 = 0; r0 < GL; r0 += RB) {
            uint32_t rc[RB][D];
            T rx[RB], rw[RB];
            int rf[RB];
            T a[RB][D][NV][VE];
            // ---- phase 1: fetch this batch's samples and issue every row load
#pragma unroll
            for (int b = 0; b < RB; ++b) {
                const int src = (r0 + b) * SPR + grp;
#pragma unroll
                for (int k = 0; k < D; ++k) rc[b][k] = __shfl_sync(0xffffffffu, smp.c[k], src);
                rx[b] = __shfl_sync(0xffffffffu, smp.x, src);
                rw[b] = __shfl_sync(0xffffffffu, wv, src);
                rf[b] = __shfl_sync(0xffffffffu, flags, src);
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    GCP_CHECK(!(rf[b] & 1) || rc[b][k] < sa.bdim[k], "gather row", rc[b][k], sa.bdim[k]);
                    const T* Ak = A;
                    if (VAR == kVarPeer && ma.nmem[k] > 1)   // the owner's A window (peer access over NVLink)
                        Ak = static_cast<const T*>(ma.peerA[ma.mem[k][(int)(rc[b][k] / (uint64_t)ma.shard[k])]]);
                    const T* row = Ak + ma.off[k] + (int64_t)rc[b][k] * ma.row_stride;
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        if ((rf[b] & 1) && vok[v]) ldg_vec<T, VE>(a[b][k][v], row + (gl + v * GL) * VE);
                        else {
#pragma unroll
                            for (int e = 0; e < VE; ++e) a[b][k][v][e] = T(0);
                        }
                    }
                }
            }
            // ---- phase 2: model value, derivative, scatter
#pragma unroll
            for (int b = 0; b < RB; ++b) {
                T mpart = T(0);
#pragma unroll
                for (int v = 0; v < NV; ++v)
#pragma unroll
                    for (int e = 0; e < VE; ++e) {
                        T p = lam[v][e];
#pragma unroll
                        for (int k = 0; k < D; ++k) p *= a[b][k][v][e];
                        mpart += p;
                    }
#pragma unroll
                for (int o = GL / 2; o > 0; o >>= 1) mpart += __shfl_xor_sync(0xffffffffu, mpart, o);
                const T m = mpart;
                const bool ok = rf[b] & 1, isnz = rf[b] & 2;
                T y;
                if (kp.semi_nz && isnz) y = rw[b] * (loss_df<T>(kp.loss, rx[b], m) - loss_df<T>(kp.loss, T(0), m));
                else y = rw[b] * loss_df<T>(kp.loss, rx[b], m);
                if (kp.with_loss && ok && gl == 0) lacc += (double)(rw[b] * loss_f<T>(kp.loss, rx[b], m));
                if (!kp.loss_mode) {
#pragma unroll
                    for (int k = 0; k < D; ++k) {
                        // warp aggregation (kVarWagg, north star / P:591-598): the
                        // samples of this round that hit the same row of mode k add
                        // their contributions in registers and the lowest such group
                        // issues one red.add; cost 1 match + 1 vote when no row repeats
                        bool lead = ok, dup = false;
                        uint32_t key = ok ? rc[b][k] : 0xFFFFFFFFu;
                        if (VAR == kVarWagg) {
                            constexpr uint32_t pat = 0xFFFFFFFFu / (uint32_t)((1ull << GL) - 1);
                            const uint32_t peers = __match_any_sync(0xffffffffu, key) & (pat << gl);
                            dup = __any_sync(0xffffffffu, ok && __popc(peers) > 1);
                            lead = ok && (__ffs(peers) - 1 == lane);
                        }
                        if (!dup && !ok) continue;
                        GCP_CHECK(!ok || rc[b][k] < sa.bdim[k], "scatter row", rc[b][k], sa.bdim[k]);
                        T* Gk = G;
                        if (VAR == kVarPeer && ma.nmem[k] > 1)   // the owner's G window: red.add over NVLink
                            Gk = static_cast<T*>(ma.peerG[ma.mem[k][(int)(rc[b][k] / (uint64_t)ma.shard[k])]]);
                        T* grow = Gk + ma.off[k] + (int64_t)rc[b][k] * ma.row_stride;
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            if (!vok[v] && !dup) continue;   // (a dup round keeps every lane in the shuffles)
                            T cv[VE];
#pragma unroll
                            for (int e = 0; e < VE; ++e) {
                                T z = y * lam[v][e];
#pragma unroll
                                for (int j = 0; j < D; ++j)
                                    if (j != k) z *= a[b][j][v][e];
                                cv[e] = z;
                            }
                            if (dup) {   // rare: sum the other groups' vectors of the same row
                                T own[VE];   // shuffled from an unmodified copy (every lane accumulates into cv)
#pragma unroll
                                for (int e = 0; e < VE; ++e) own[e] = cv[e];
#pragma unroll
                                for (int j = 1; j < SPR; ++j) {
                                    const int srcl = (lane + j * GL) & 31;
                                    const uint32_t ok2 = __shfl_sync(0xffffffffu, key, srcl);
                                    T o[VE];
#pragma unroll
                                    for (int e = 0; e < VE; ++e) o[e] = __shfl_sync(0xffffffffu, own[e], srcl);
                                    if (ok2 == key)
#pragma unroll
                                        for (int e = 0; e < VE; ++e) cv[e] += o[e];
                                }
                            }
                            if (lead && vok[v]) red_add_v(grow + (gl + v * GL) * VE, cv);
                        }
                    }
                }
            }
        }
    }
    if (kp.with_loss) {
        // deterministic CTA reduction of the per-thread fp64 partials
        __shared__ double red[kBlock / 32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lacc += __shfl_xor_sync(0xffffffffu, lacc, o);
        if (lane == 0) red[threadIdx.x >> 5] = lacc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < kBlock / 32; ++w) t += red[w];
            kp.partials[blockIdx.x] = t;
        }
    }
}

template <typename T, int D>
__global__ void k_export(const SampleArgs sa, int64_t first, int64_t count, const int64_t* lo,
                         int64_t* subs, int64_t* jout, int32_t* att) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const Sample<T, D> smp = draw_sample<T, D>(sa, first + i);
#pragma unroll
    for (int k = 0; k < D; ++k) subs[i * D + k] = lo[k] + (int64_t)smp.c[k];
    if (jout) jout[i] = smp.j;
    if (att) att[i] = smp.attempts;
}

// Alg. 1 over the segments of the contiguous arrays:
// B <- b1 B + (1-b1) g; C <- b2 C + (1-b2) g^2; A <- A - rate (B bc1)/sqrt(C bc2 + eps);
// A <- (A < l) ? l : A; G <- 0 (fused reset).  bc = 1/(1-beta^t) from the host in fp64.
template <typename T>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 5 : 4) k_adam(const Segment seg, int64_t nvec_total, T* __restrict__ A,
                                              T* __restrict__ G, T* __restrict__ B, T* __restrict__ C,
                                              T rate, T b1, T b2, T eps, T bc1, T bc2, T lower,
                                              int zero_g, int R_pad, int row_stride, const DevStep* step,
                                              long long t_off, const OrdScatterArgs os) {
    using V = typename Vec16<T>::type;
    constexpr int VE = Vec16<T>::n;
    if (step) {   // graph replay: t = t0 + offset, bias corrections in fp64 from it
        const double t = (double)(step->t + t_off);
        rate = (T)step->rate;
        bc1 = (T)(1.0 / (1.0 - pow(step->beta1, t)));
        bc2 = (T)(1.0 / (1.0 - pow(step->beta2, t)));
    }
    // the next iteration's slot-order scatter (random 4-B stores into L2)
    // interleaved with this memory-bound stream, one slot per os.ratio vectors
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    int64_t hs = tid;
    int hstep = 0;
    for (int64_t i = tid; i < nvec_total; i += nt) {
        if (hs < os.n && ++hstep == os.ratio) {
            hstep = 0;
            os.order[__ldg(os.cursor + os.keys[hs]) + os.ranks[hs]] = (uint32_t)hs;
            hs += nt;
        }
        // map the virtual vector index onto its segment
        int64_t rem = i;
        int sidx = 0;
        while (sidx < seg.n - 1 && rem >= seg.len[sidx] / VE) { rem -= seg.len[sidx] / VE; ++sidx; }
        const int64_t e = seg.start[sidx] + rem * VE;                   // B, C (logical) index
        const int64_t ea = (e / R_pad) * row_stride + e % R_pad;          // A, G (row-strided) index
        V g = *reinterpret_cast<const V*>(G + ea);
        V a = *reinterpret_cast<const V*>(A + ea);
        V b = *reinterpret_cast<const V*>(B + e);
        V c = *reinterpret_cast<const V*>(C + e);
        T* gp = reinterpret_cast<T*>(&g);
        T* ap = reinterpret_cast<T*>(&a);
        T* bp = reinterpret_cast<T*>(&b);
        T* cp = reinterpret_cast<T*>(&c);
#pragma unroll
        for (int q = 0; q < VE; ++q) {
            const T gv = gp[q];
            bp[q] = b1 * bp[q] + (T(1) - b1) * gv;
            cp[q] = b2 * cp[q] + (T(1) - b2) * gv * gv;
            T av = ap[q] - rate * ((bp[q] * bc1) / sqrt(cp[q] * bc2 + eps));
            ap[q] = (av < lower) ? lower : av;
        }
        *reinterpret_cast<V*>(A + ea) = a;
        *reinterpret_cast<V*>(B + e) = b;
        *reinterpret_cast<V*>(C + e) = c;
        if (zero_g) {
            V z;
            T* zp = reinterpret_cast<T*>(&z);
#pragma unroll
            for (int q = 0; q < VE; ++q) zp[q] = T(0);
            *reinterpret_cast<V*>(G + ea) = z;
        }
    }
    for (; hs < os.n; hs += nt) os.order[__ldg(os.cursor + os.keys[hs]) + os.ranks[hs]] = (uint32_t)hs;
}

struct InitArgs {
    int d, R, R_pad, row_stride;
    int64_t rows[kMaxModes], bdim[kMaxModes], lo[kMaxModes], off[kMaxModes], goff[kMaxModes];
    int64_t n_coef;
    uint64_t seed;
};

// Factor k, local row i, column r < R: global element e = goff_k + (lo_k + i) R + r of the
// unpadded mode-major concatenation; value (W0 >> 11) 2^-53 of Philox(lo32 e, hi32 e, 4<<28, 0).
template <typename T>
__global__ void k_init(const InitArgs ia, T* __restrict__ A) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < ia.n_coef;
         x += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        while (k < ia.d - 1 && x >= ia.off[k + 1]) ++k;
        const int64_t loc = x - ia.off[k];
        const int64_t i = loc / ia.R_pad;
        const int r = (int)(loc % ia.R_pad);
        T v = T(0);
        if (r < ia.R && i < ia.bdim[k]) {
            const uint64_t e = (uint64_t)(ia.goff[k] + (ia.lo[k] + i) * ia.R + r);
            const U64x2 w = philox((uint32_t)e, (uint32_t)(e >> 32), (uint32_t)KIND_INIT << 28, 0u,
                                   (uint32_t)ia.seed, (uint32_t)(ia.seed >> 32));
            v = (T)((double)(w.w0 >> 11) * 0x1.0p-53);
        }
        A[(x / ia.R_pad) * ia.row_stride + x % ia.R_pad] = v;
    }
}

}  // namespace gcp
