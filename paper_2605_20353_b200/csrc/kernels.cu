// kernels.cu -- precision dispatch of the hot-path launchers plus the small
// helper kernels (deterministic partial-sum reduction, scale, subtract).
#include "kernels.cuh"

#include <curand_philox4x32_x.h>

#include <algorithm>
#include <string>

namespace gcp {

cudaError_t sample_kernel_f32(gcp_ctx*, const SampleArgs&, const ModelArgs&, int, int, int, double, double,
                              int, double*, int, const OrdHistArgs*);
cudaError_t sample_kernel_f64(gcp_ctx*, const SampleArgs&, const ModelArgs&, int, int, int, double, double,
                              int, double*, int, const OrdHistArgs*);
cudaError_t sample_kernel_peer_f32(gcp_ctx*, const SampleArgs&, const ModelArgs&, int, int, int, double, double,
                              int, double*, int, const OrdHistArgs*);
cudaError_t sample_kernel_peer_f64(gcp_ctx*, const SampleArgs&, const ModelArgs&, int, int, int, double, double,
                              int, double*, int, const OrdHistArgs*);
cudaError_t sample_kernel_wagg_f32(gcp_ctx*, const SampleArgs&, const ModelArgs&, int, int, int, double, double,
                              int, double*, int, const OrdHistArgs*);
cudaError_t sample_kernel_wagg_f64(gcp_ctx*, const SampleArgs&, const ModelArgs&, int, int, int, double, double,
                              int, double*, int, const OrdHistArgs*);
int sample_occupancy_f32(int, int);
int sample_occupancy_f64(int, int);
int sample_occupancy_peer_f32(int, int);
int sample_occupancy_peer_f64(int, int);
cudaError_t export_f32(gcp_ctx*, const SampleArgs&, int64_t, int64_t, const int64_t*, int64_t*, int64_t*,
                       int32_t*);
cudaError_t export_f64(gcp_ctx*, const SampleArgs&, int64_t, int64_t, const int64_t*, int64_t*, int64_t*,
                       int32_t*);
cudaError_t adam_f32(gcp_ctx*, const Segment&, void*, void*, void*, void*, double, double, double, double,
                     double, int64_t, int, int, int, const DevStep*, const OrdScatterArgs*);
cudaError_t adam_f64(gcp_ctx*, const Segment&, void*, void*, void*, void*, double, double, double, double,
                     double, int64_t, int, int, int, const DevStep*, const OrdScatterArgs*);
cudaError_t init_f32(gcp_ctx*, const InitArgs&, void*);
cudaError_t init_f64(gcp_ctx*, const InitArgs&, void*);

int sample_kernel_blocks(gcp_ctx* c) {
    // persistent grid: the resident CTAs of the variant the context launches
    const bool f32 = c->prec == GCP_FP32;
    const int occ = c->tsn_peer ? (f32 ? sample_occupancy_peer_f32(c->d, c->R_pad) : sample_occupancy_peer_f64(c->d, c->R_pad))
                                : (f32 ? sample_occupancy_f32(c->d, c->R_pad) : sample_occupancy_f64(c->d, c->R_pad));
    return c->sm_count * (occ > 0 ? occ : 1);
}

cudaError_t launch_sample_kernel(gcp_ctx* c, const SampleArgs& s, const ModelArgs& m, int loss, int loss_mode,
                                 int semi_nz, double w_nz, double w_z, int with_loss, double* partials,
                                 int nblocks, const OrdHistArgs* oh) {
    // K2 variant: rows owned elsewhere (two-sided by peer access) -> kVarPeer;
    // GCP_WAGG=1 -> warp-aggregated scatter-adds (gradient launches only)
    const char* we = getenv("GCP_WAGG");
    const int var = m.peerA ? kVarPeer : (!loss_mode && we && we[0] == '1') ? kVarWagg : kVarPlain;
    if (var == kVarPeer)
        return c->prec == GCP_FP32
                   ? sample_kernel_peer_f32(c, s, m, loss, loss_mode, semi_nz, w_nz, w_z, with_loss, partials, nblocks, oh)
                   : sample_kernel_peer_f64(c, s, m, loss, loss_mode, semi_nz, w_nz, w_z, with_loss, partials, nblocks, oh);
    if (var == kVarWagg)
        return c->prec == GCP_FP32
                   ? sample_kernel_wagg_f32(c, s, m, loss, loss_mode, semi_nz, w_nz, w_z, with_loss, partials, nblocks, oh)
                   : sample_kernel_wagg_f64(c, s, m, loss, loss_mode, semi_nz, w_nz, w_z, with_loss, partials, nblocks, oh);
    return c->prec == GCP_FP32
               ? sample_kernel_f32(c, s, m, loss, loss_mode, semi_nz, w_nz, w_z, with_loss, partials, nblocks, oh)
               : sample_kernel_f64(c, s, m, loss, loss_mode, semi_nz, w_nz, w_z, with_loss, partials, nblocks, oh);
}

cudaError_t launch_export(gcp_ctx* c, const SampleArgs& s, int stratum, int64_t first, int64_t count,
                          const int64_t* lo, int64_t* subs, int64_t* j, int32_t* att) {
    (void)stratum;
    return c->prec == GCP_FP32 ? export_f32(c, s, first, count, lo, subs, j, att)
                               : export_f64(c, s, first, count, lo, subs, j, att);
}

cudaError_t launch_adam(gcp_ctx* c, const Segment& seg, void* A, void* G, void* B, void* C, double rate,
                        double beta1, double beta2, double eps, double lower, int64_t t, int zero_g,
                        int row_stride, const DevStep* step, const OrdScatterArgs* os) {
    const int rs = row_stride > 0 ? row_stride : c->R_pad;
    return c->prec == GCP_FP32
               ? adam_f32(c, seg, A, G, B, C, rate, beta1, beta2, eps, lower, t, zero_g, c->R_pad, rs, step, os)
               : adam_f64(c, seg, A, G, B, C, rate, beta1, beta2, eps, lower, t, zero_g, c->R_pad, rs, step, os);
}

cudaError_t launch_init(gcp_ctx* c, uint64_t seed, const int64_t* goff) {
    InitArgs ia;
    ia.d = c->d; ia.R = c->R; ia.R_pad = c->R_pad; ia.row_stride = c->ag_stride; ia.n_coef = c->n_coef;
    ia.seed = seed;
    for (int k = 0; k < kMaxModes; ++k) {
        ia.rows[k] = k < c->d ? c->rows[k] : 0;
        ia.bdim[k] = k < c->d ? c->hi[k] - c->lo[k] : 0;
        ia.lo[k] = k < c->d ? c->lo[k] : 0;
        ia.off[k] = k < c->d ? c->off[k] : 0;
        ia.goff[k] = k < c->d ? goff[k] : 0;
    }
    return c->prec == GCP_FP32 ? init_f32(c, ia, c->d_A) : init_f64(c, ia, c->d_A);
}

// Slot ordering for the gradient K2 (DRAM-resident mode-1 rows: c4, c5): a
// hand-written counting sort of the iteration's slots into 2^bits buckets of
// mode-1 position (default 2^15), nonzero and zero slots interleaved (a bucket
// holds the nonzero slots whose record lies in a mode-1 row range AND the zero
// slots whose attempt-0 candidate lies in the same range, so K2 fills the A|G
// lines of a row range once per iteration, not once per stratum).  The sample
// set, and so the estimate, is unchanged; only the visiting order changes, so
// that K2's gathers and scatter-adds of one mode-1 row meet in L2 and its DRAM
// accesses walk the records and rows forward.
//   histogram      per slot: Philox word -> bucket (kernels.cuh ord_bucket) and
//                  the slot's rank inside its bucket (a global atomicAdd);
//                  carried by the previous iteration's gradient K2 (OrdHistArgs:
//                  ALU work under its memory-bound gathers), else k_ord_hist
//   k_ord_scan     one CTA: exclusive scan of the bucket totals -> cursors;
//                  totals reset for the next iteration
//   k_ord_scatter  order[cursor[bucket] + rank] = slot (GCP_ORD_FUSE=2 carries
//                  it in the previous Adam launch instead: slower, see
//                  ord_scatter_args)
// So in steady state an iteration launches the scan and the scatter.
// Order inside a bucket is the atomics' arrival order (run to run it varies),
// which only moves the fp32 atomic summation order of K2.
constexpr int kOrdMaxBits = 15;            // table / counter capacity
constexpr int kOrdThreads = 1024;
constexpr int kOrdLutBits = 20;            // nonzero-index lookup cells (u16 each: 2 MB, L2-resident)

// bucket bits (GCP_ORD_BITS, default 15), read once per context at allocation
int ord_bits_env() {
    const char* e = getenv("GCP_ORD_BITS");
    const int b = e ? atoi(e) : 15;
    return b < 10 ? 10 : (b > kOrdMaxBits ? kOrdMaxBits : b);
}

// T[b] = first canonical record whose c_1 >= ceil(b I_1 / B), b = 0..B (T[B] = N):
// records are sorted with i_1 most significant (reading R15)
__global__ void k_ord_table(const uint32_t* __restrict__ rec, int rec_words, int val_words, int64_t N, uint32_t I1,
                            int bits, int64_t* __restrict__ T) {
    const int B = 1 << bits;
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > B) return;
    const uint64_t row = ((uint64_t)b * I1 + B - 1) >> bits;
    int64_t lo = 0, hi = N;
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (rec[mid * rec_words + val_words] < row) lo = mid + 1;
        else hi = mid;
    }
    T[b] = lo;
}

// lut[x] = bucket of nonzero index j = x << shift: the largest b with T[b] <= j
__global__ void k_ord_lut(const int64_t* __restrict__ T, int bits, int shift, int64_t ncell, int64_t N,
                          uint16_t* __restrict__ lut) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < ncell; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = min(x << shift, N - 1);
        uint32_t lo = 0, hi = 1u << bits;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (T[mid] <= j) lo = mid;
            else hi = mid;
        }
        lut[x] = (uint16_t)lo;
    }
}

// Histogram pass for an iteration whose histogram no gradient K2 computed (the
// first of an epoch graph, eager calls):
// bucket and in-bucket rank of every slot, four slots per thread in flight.
__global__ void __launch_bounds__(256) k_ord_hist(const OrdHistArgs oh) {
    const uint32_t it = iter_word(oh.sa);
    const uint64_t inv = oh.sa.bdim[0] > 1 ? (~0ull) / oh.sa.bdim[0] : 0;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < oh.n; s += 4 * nt) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (s + u * nt < oh.n) ord_hist_slot(oh, s + u * nt, it, inv);
    }
}

// one CTA: exclusive scan of the bucket totals -> cursors; totals reset.  The
// totals pass through shared memory with one pad word per 32 (conflict-free
// per-thread segments).
__global__ void __launch_bounds__(kOrdThreads) k_ord_scan(uint32_t* __restrict__ totals, uint32_t* __restrict__ cursor,
                                                         int B, int tile_shift) {
    // CTA t scans tile t's buckets; tile t's slots fill order[t << tile_shift, ...)
    totals += (size_t)blockIdx.x * B;
    cursor += (size_t)blockIdx.x * B;
    const uint32_t tile_base = tile_shift < 32 ? (uint32_t)blockIdx.x << tile_shift : 0u;
    extern __shared__ __align__(16) unsigned char ord_smem[];
    uint32_t* sv = reinterpret_cast<uint32_t*>(ord_smem);   // B + B/32 words
    __shared__ uint32_t wsum[kOrdThreads / 32];
    for (int i = threadIdx.x; i < B; i += kOrdThreads) {
        sv[i + (i >> 5)] = totals[i];
        totals[i] = 0;
    }
    __syncthreads();
    const int per = B / kOrdThreads;   // B >= 2^10
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t run = 0;
    for (int i = 0; i < per; ++i) {
        const int x = t * per + i;
        run += sv[x + (x >> 5)];
    }
    uint32_t incl = run;   // inclusive warp scan of the per-thread sums
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        uint32_t x = lane < kOrdThreads / 32 ? wsum[lane] : 0, xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        if (lane < kOrdThreads / 32) wsum[lane] = xi - x;   // exclusive prefix of the warp totals
    }
    __syncthreads();
    uint32_t base = tile_base + wsum[w] + incl - run;
    for (int i = 0; i < per; ++i) {
        const int x = t * per + i;
        const uint32_t v = sv[x + (x >> 5)];
        sv[x + (x >> 5)] = base;
        base += v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < B; i += kOrdThreads) cursor[i] = sv[i + (i >> 5)];
}

// order[cursor[bucket] + rank] = slot: one pass, no atomics
__global__ void __launch_bounds__(256) k_ord_scatter(const uint32_t* __restrict__ keys,
                                                    const uint32_t* __restrict__ ranks, int64_t n,
                                                    const uint32_t* __restrict__ cursor, uint32_t* __restrict__ order) {
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += nt) {
        const uint32_t pos = __ldg(cursor + keys[s]) + ranks[s];
        GCP_CHECK(pos < (uint64_t)n, "order position >= p + q", pos, n);
        order[pos] = (uint32_t)s;
    }
}

static int64_t lut_cells(int64_t N, int* shift) {
    int sh = 0;
    while (((N - 1) >> sh) >= ((int64_t)1 << kOrdLutBits)) ++sh;
    *shift = sh;
    return ((std::max<int64_t>(N, 1) - 1) >> sh) + 1;
}

// Large p + q (c5 at one GPU: 2e8 slots, an 800-MB order array) are ordered in
// independent tiles of consecutive slots whose order regions fit L2, so the
// scatter's random stores stay in L2 (an order array spilling to DRAM turns
// every 4-B store into a sector read-modify-write); K2 then visits the tiles
// one after the other, each in mode-1 order.  GCP_ORD_TILE_MB (default 128)
// bounds a tile's order region.
static constexpr int kOrdMaxTiles = 64;
static int ord_tile_shift_for(int64_t cap) {
    const char* e = getenv("GCP_ORD_TILE_MB");
    const double mb = e && atof(e) > 0 ? atof(e) : 128.0;
    if ((double)cap * 4.0 <= mb * 1048576.0 * 1.25) return 62;   // one tile
    int sh = 10;
    while ((double)((int64_t)1 << (sh + 1)) * 4.0 <= mb * 1048576.0) ++sh;
    while (((cap + ((int64_t)1 << sh) - 1) >> sh) > kOrdMaxTiles) ++sh;
    return sh;
}

size_t slot_order_bytes(int64_t cap) {
    constexpr int B = 1 << kOrdMaxBits;
    const size_t capr = (size_t)(cap + 15) / 16 * 16;
    return capr * (3 * sizeof(uint32_t)) + 2 * (size_t)kOrdMaxTiles * B * sizeof(uint32_t) +
           (B + 2) * sizeof(int64_t) + ((size_t)1 << kOrdLutBits) * sizeof(uint16_t) + 256;
}

// Carve the order buffers out of one allocation of slot_order_bytes(cap) and
// build the per-tensor tables T and lut (once per tensor).
cudaError_t slot_order_init(gcp_ctx* c, void* buf, int64_t cap) {
    constexpr int B = 1 << kOrdMaxBits;
    const size_t capr = (size_t)(cap + 15) / 16 * 16;
    c->ord_bits = ord_bits_env();
    c->ord_tile_shift = ord_tile_shift_for(cap);
    c->ord_ntiles = c->ord_tile_shift >= 62 ? 1 : (int)((cap + ((int64_t)1 << c->ord_tile_shift) - 1) >> c->ord_tile_shift);
    char* p = static_cast<char*>(buf);
    c->d_ord_T = reinterpret_cast<int64_t*>(p);
    p += (B + 2) * sizeof(int64_t);
    c->d_ord_cnt = reinterpret_cast<uint32_t*>(p);   // counts [tiles][B], then cursors [tiles][B]
    p += 2 * (size_t)kOrdMaxTiles * B * sizeof(uint32_t);
    c->d_ord = reinterpret_cast<uint32_t*>(p);
    p += capr * sizeof(uint32_t);
    c->d_ord_rank = reinterpret_cast<uint32_t*>(p);
    p += capr * sizeof(uint32_t);
    c->d_ord_key = reinterpret_cast<uint32_t*>(p);
    p += capr * sizeof(uint32_t);
    c->d_ord_lut = reinterpret_cast<uint16_t*>(p);
    cudaError_t e = cudaMemsetAsync(c->d_ord_cnt, 0, 2 * (size_t)kOrdMaxTiles * B * sizeof(uint32_t), c->stream);
    if (e != cudaSuccess) return e;
    k_ord_table<<<((1 << c->ord_bits) + 1 + 255) / 256, 256, 0, c->stream>>>(
        c->d_rec, c->rec_words, c->val_words, c->N, (uint32_t)(c->hi[0] - c->lo[0]), c->ord_bits, c->d_ord_T);
    const int64_t ncell = lut_cells(c->N, &c->ord_lut_shift);
    k_ord_lut<<<(int)std::min<int64_t>((ncell + 255) / 256, 4096), 256, 0, c->stream>>>(
        c->d_ord_T, c->ord_bits, c->ord_lut_shift, ncell, std::max<int64_t>(c->N, 1), c->d_ord_lut);
    c->launches += 2;
    return cudaGetLastError();
}

static uint32_t* ord_cursor(gcp_ctx* c) { return c->d_ord_cnt + (size_t)kOrdMaxTiles * (1 << kOrdMaxBits); }

static OrdHistArgs make_hist_args(gcp_ctx* c, const SampleArgs& sa) {
    OrdHistArgs oh;
    oh.sa = sa;
    oh.lut = c->d_ord_lut;
    oh.lut_shift = c->ord_lut_shift;
    oh.keys = c->d_ord_key;
    oh.ranks = c->d_ord_rank;
    oh.totals = c->d_ord_cnt;
    oh.bits = c->ord_bits;
    oh.tile_shift = c->ord_tile_shift;
    oh.n = sa.p + sa.q;
    return oh;
}

static cudaError_t ord_scan(gcp_ctx* c) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_ord_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(((1 << kOrdMaxBits) + (1 << kOrdMaxBits) / 32) * 4));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int B = 1 << c->ord_bits;
    k_ord_scan<<<c->ord_ntiles, kOrdThreads, (size_t)(B + B / 32) * 4, c->stream>>>(c->d_ord_cnt, ord_cursor(c), B,
                                                                                    c->ord_tile_shift);
    c->launches++;
    return cudaGetLastError();
}

// The order of this iteration's slots, from whatever the previous launches
// prepared: stage 2 = nothing left, 1 = scan + scatter, 0 = everything.
cudaError_t launch_slot_order(gcp_ctx* c, const SampleArgs& s, const uint32_t** order_out, int stage) {
    const int64_t n = s.p + s.q;
    *order_out = c->d_ord;
    if (n == 0 || stage >= 2) return cudaSuccess;
    const int B = 1 << c->ord_bits;
    uint32_t* totals = c->d_ord_cnt;
    const int nb = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8);
    if (stage < 1) {
        // totals may hold an unconsumed histogram (a K2 prepared an iteration
        // that did not follow): start from zero
        cudaError_t e = cudaMemsetAsync(totals, 0, (size_t)c->ord_ntiles * B * sizeof(uint32_t), c->stream);
        if (e != cudaSuccess) return e;
        k_ord_hist<<<nb, 256, 0, c->stream>>>(make_hist_args(c, s));
        c->launches++;
    }
    cudaError_t e = ord_scan(c);
    if (e != cudaSuccess) return e;
    k_ord_scatter<<<nb, 256, 0, c->stream>>>(c->d_ord_key, c->d_ord_rank, n, ord_cursor(c), c->d_ord);
    c->launches++;
    return cudaGetLastError();
}

// The histogram of the next iteration for the gradient K2 to carry
// (GCP_ORD_FUSE=0 keeps every pass a launch of its own; the histogram's Philox
// and table lookups cost K2 nothing measurable on c4).
bool ord_hist_args(gcp_ctx* c, const SampleArgs& next, OrdHistArgs* oh) {
    const char* fe = getenv("GCP_ORD_FUSE");
    if ((fe && atoi(fe) == 0) || !c->d_ord) return false;
    const int64_t n = next.p + next.q;
    if (n == 0 || n > c->ord_cap) return false;
    *oh = make_hist_args(c, next);
    return true;
}

// The scan of the next iteration (launched here) and its scatter for the Adam
// launch to carry -- only with GCP_ORD_FUSE=2: the random 4-B stores slowed
// Adam's stream by more than the scatter launch costs (c4: Adam 0.70 -> 1.07 ms
// against a 0.2-ms scatter).  Writing the slot ids straight into fixed-capacity
// bucket buffers from the K2 histogram (no scatter pass at all) cost K2 the same
// 0.2 ms of random 4-B stores (profiles/r02_summary.md).
bool ord_scatter_args(gcp_ctx* c, int64_t n, OrdScatterArgs* os, int64_t adam_vecs) {
    const char* fe = getenv("GCP_ORD_FUSE");
    if (!(fe && atoi(fe) == 2)) return false;
    if (!c->d_ord || n == 0 || n > c->ord_cap) return false;
    if (ord_scan(c) != cudaSuccess) return false;
    os->keys = c->d_ord_key;
    os->ranks = c->d_ord_rank;
    os->cursor = ord_cursor(c);
    os->order = c->d_ord;
    os->n = n;
    os->ratio = (int)std::max<int64_t>(1, adam_vecs / n);
    return true;
}

// Test helper (gcp_debug_philox): the sampler's device Philox4x32-10 and curand's
// curand_Philox4x32_10 on the same (counter, key) inputs.
__global__ void k_debug_philox(int64_t n, const uint32_t* __restrict__ in, uint32_t* __restrict__ out) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t* v = in + 6 * x;
        const U64x2 w = philox(v[0], v[1], v[2], v[3], v[4], v[5]);
        const uint4 r = curand_Philox4x32_10(make_uint4(v[0], v[1], v[2], v[3]), make_uint2(v[4], v[5]));
        uint32_t* o = out + 8 * x;
        o[0] = (uint32_t)w.w0; o[1] = (uint32_t)(w.w0 >> 32); o[2] = (uint32_t)w.w1; o[3] = (uint32_t)(w.w1 >> 32);
        o[4] = r.x; o[5] = r.y; o[6] = r.z; o[7] = r.w;
    }
}

cudaError_t launch_debug_philox(gcp_ctx* c, int64_t n, const uint32_t* in, uint32_t* out) {
    if (n == 0) return cudaSuccess;
    k_debug_philox<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, c->stream>>>(n, in, out);
    c->launches++;
    return cudaGetLastError();
}

// Fixed-order sum of n fp64 partials (deterministic; one CTA).
__global__ void k_reduce_partials(const double* __restrict__ p, int n, double* out) {
    __shared__ double s[256];
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += 256) t += p[i];
    s[threadIdx.x] = t;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s[0];
}

cudaError_t launch_reduce_partials(gcp_ctx* c, const double* partials, int n, double* out) {
    k_reduce_partials<<<1, 256, 0, c->stream>>>(partials, n, out);
    return cudaGetLastError();
}

template <typename T>
__global__ void k_scale(T* x, int64_t n, T s) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] *= s;
}
template <typename T>
__global__ void k_sub(const T* a, const T* b, T* out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a[i] - b[i];
}

static int grid_for(gcp_ctx* c, int64_t n) {
    int64_t nb = (n + 255) / 256;
    const int64_t cap = (int64_t)c->sm_count * 8;
    if (nb > cap) nb = cap;
    return nb < 1 ? 1 : (int)nb;
}

cudaError_t launch_scale(gcp_ctx* c, void* x, int64_t n, double s) {
    if (n == 0) return cudaSuccess;
    if (c->prec == GCP_FP32) k_scale<float><<<grid_for(c, n), 256, 0, c->stream>>>((float*)x, n, (float)s);
    else k_scale<double><<<grid_for(c, n), 256, 0, c->stream>>>((double*)x, n, s);
    return cudaGetLastError();
}

// packed host-order rows (b x R doubles) <-> the factor layout (rows of R_pad T
// at row stride `stride`, zero padding): model_set / model_get on the device
template <typename T>
__global__ void k_rows_in(const double* __restrict__ src, T* __restrict__ dst, int64_t b, int R, int R_pad,
                          int stride) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < b * R_pad;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = x / R_pad;
        const int r = (int)(x % R_pad);
        dst[i * stride + r] = r < R ? (T)src[i * R + r] : T(0);
    }
}
template <typename T>
__global__ void k_rows_out(const T* __restrict__ src, double* __restrict__ dst, int64_t b, int R, int stride) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < b * R;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = x / R;
        dst[x] = (double)src[i * stride + (int)(x % R)];
    }
}

cudaError_t launch_rows_in(gcp_ctx* c, const double* src, void* dst, int64_t b) {
    if (b == 0) return cudaSuccess;
    const int64_t n = b * c->R_pad;
    if (c->prec == GCP_FP32)
        k_rows_in<float><<<grid_for(c, n), 256, 0, c->stream>>>(src, (float*)dst, b, c->R, c->R_pad, c->ag_stride);
    else
        k_rows_in<double><<<grid_for(c, n), 256, 0, c->stream>>>(src, (double*)dst, b, c->R, c->R_pad, c->ag_stride);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_rows_out(gcp_ctx* c, const void* src, double* dst, int64_t b) {
    if (b == 0) return cudaSuccess;
    const int64_t n = b * c->R;
    if (c->prec == GCP_FP32)
        k_rows_out<float><<<grid_for(c, n), 256, 0, c->stream>>>((const float*)src, dst, b, c->R, c->ag_stride);
    else
        k_rows_out<double><<<grid_for(c, n), 256, 0, c->stream>>>((const double*)src, dst, b, c->R, c->ag_stride);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_sub(gcp_ctx* c, const void* a, const void* b, void* out, int64_t n) {
    if (n == 0) return cudaSuccess;
    if (c->prec == GCP_FP32)
        k_sub<float><<<grid_for(c, n), 256, 0, c->stream>>>((const float*)a, (const float*)b, (float*)out, n);
    else
        k_sub<double><<<grid_for(c, n), 256, 0, c->stream>>>((const double*)a, (const double*)b, (double*)out, n);
    return cudaGetLastError();
}

}  // namespace gcp
