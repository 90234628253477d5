// kernels.cu -- precision dispatch of the hot-path launchers plus the small
// helper kernels (deterministic partial-sum reduction, scale, subtract).
#include "kernels.cuh"

#include <algorithm>
#include <string>

namespace gcp {

cudaError_t sample_kernel_f32(gcp_ctx*, const SampleArgs&, const ModelArgs&, int, int, int, double, double,
                              int, double*, int, const OrdHistArgs*);
cudaError_t sample_kernel_f64(gcp_ctx*, const SampleArgs&, const ModelArgs&, int, int, int, double, double,
                              int, double*, int, const OrdHistArgs*);
int sample_occupancy_f32(int, int);
int sample_occupancy_f64(int, int);
cudaError_t export_f32(gcp_ctx*, const SampleArgs&, int64_t, int64_t, const int64_t*, int64_t*, int64_t*,
                       int32_t*);
cudaError_t export_f64(gcp_ctx*, const SampleArgs&, int64_t, int64_t, const int64_t*, int64_t*, int64_t*,
                       int32_t*);
cudaError_t adam_f32(gcp_ctx*, const Segment&, void*, void*, void*, void*, double, double, double, double,
                     double, int64_t, int, int, int, const DevStep*);
cudaError_t adam_f64(gcp_ctx*, const Segment&, void*, void*, void*, void*, double, double, double, double,
                     double, int64_t, int, int, int, const DevStep*);
cudaError_t init_f32(gcp_ctx*, const InitArgs&, void*);
cudaError_t init_f64(gcp_ctx*, const InitArgs&, void*);

int sample_kernel_blocks(gcp_ctx* c) {
    const int occ = c->prec == GCP_FP32 ? sample_occupancy_f32(c->d, c->R_pad) : sample_occupancy_f64(c->d, c->R_pad);
    return c->sm_count * (occ > 0 ? occ : 1);
}

cudaError_t launch_sample_kernel(gcp_ctx* c, const SampleArgs& s, const ModelArgs& m, int loss, int loss_mode,
                                 int semi_nz, double w_nz, double w_z, int with_loss, double* partials,
                                 int nblocks, const OrdHistArgs* oh) {
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
                        int row_stride, const DevStep* step) {
    const int rs = row_stride > 0 ? row_stride : c->R_pad;
    return c->prec == GCP_FP32
               ? adam_f32(c, seg, A, G, B, C, rate, beta1, beta2, eps, lower, t, zero_g, c->R_pad, rs, step)
               : adam_f64(c, seg, A, G, B, C, rate, beta1, beta2, eps, lower, t, zero_g, c->R_pad, rs, step);
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

// Slot ordering for the gradient K2 (DRAM-resident mode-1 rows: c4, c5): the
// iteration's slots grouped into 2^bits buckets of mode-1 position (default
// 2^15), nonzero and zero slots interleaved (a bucket holds the nonzero slots
// whose record lies in a mode-1 row range AND the zero slots whose attempt-0
// candidate lies in the same range, so K2 fills the A|G lines of a row range
// once per iteration, not once per stratum).  The sample set, and so the
// estimate, is unchanged; only the visiting order changes, so that K2's
// gathers and scatter-adds of one mode-1 row meet in L2 and its DRAM accesses
// walk the records and rows forward.
//   histogram   per slot: Philox word -> bucket (kernels.cuh ord_bucket); the
//               slot id goes straight into the bucket's fixed-capacity buffer at
//               the rank an atomicAdd on the bucket count returns (overflow list
//               past the capacity).  Carried by the previous iteration's
//               gradient K2 (OrdHistArgs: ALU work and scattered 4-B stores
//               under its memory-bound gathers), else k_ord_hist.
//   k_ord_scan  one CTA: exclusive prefix of min(count, capacity) -> the visiting
//               order's bucket offsets; counts and the next parity's overflow
//               count reset
//   K2          position p -> bucket (binary search of the prefix, L1-resident)
//               -> slot id in the bucket buffer (kernels.cuh slot_at)
// No scatter pass: a bucket buffer is read where the histogram wrote it.  The
// buffers are double-buffered by iteration parity (K2 of t reads parity t while
// it fills parity t+1).  Order inside a bucket is the atomics' arrival order
// (run to run it varies), which only moves the fp32 atomic summation order of K2.
constexpr int kOrdMaxBits = 15;            // counter / table capacity
constexpr int kOrdThreads = 1024;
constexpr int kOrdLutBits = 20;            // nonzero-index lookup cells (u16 each: 2 MB, L2-resident)

// bucket bits (GCP_ORD_BITS, default 15), read once per context at allocation
int ord_bits_env() {
    const char* e = getenv("GCP_ORD_BITS");
    const int b = e ? atoi(e) : 15;
    return b < 10 ? 10 : (b > kOrdMaxBits ? kOrdMaxBits : b);
}

// bucket capacity 2^capbits: >= 2.5x the mean bucket load (the overflow list
// takes the rest)
static int ord_capbits_for(int64_t cap, int bits) {
    const double mean = (double)cap / (double)(1 << bits);
    int cb = 4;
    while ((double)(1 << cb) < 2.5 * mean && cb < 24) ++cb;
    return cb;
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

// Histogram for an iteration whose histogram no gradient K2 carried (the first
// of an epoch graph, eager calls): four slots per thread in flight.
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

// one CTA: prefix[b] = sum_{b' < b} min(count[b'], capacity), prefix[B] = the
// slots in buckets; counts reset, the next parity's overflow count reset.  The
// counts pass through shared memory with one pad word per 32 (conflict-free
// per-thread segments).
__global__ void __launch_bounds__(kOrdThreads) k_ord_scan(uint32_t* __restrict__ counts, uint32_t* __restrict__ prefix,
                                                         uint32_t* __restrict__ novf_next, int B, uint32_t capacity) {
    extern __shared__ __align__(16) unsigned char ord_smem[];
    uint32_t* sv = reinterpret_cast<uint32_t*>(ord_smem);   // B + B/32 words
    __shared__ uint32_t wsum[kOrdThreads / 32];
    for (int i = threadIdx.x; i < B; i += kOrdThreads) {
        sv[i + (i >> 5)] = min(counts[i], capacity);
        counts[i] = 0;
    }
    if (threadIdx.x == 0) *novf_next = 0;
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
    uint32_t base = wsum[w] + incl - run;
    for (int i = 0; i < per; ++i) {
        const int x = t * per + i;
        const uint32_t v = sv[x + (x >> 5)];
        sv[x + (x >> 5)] = base;
        base += v;
    }
    if (t == kOrdThreads - 1) prefix[B] = base;
    __syncthreads();
    for (int i = threadIdx.x; i < B; i += kOrdThreads) prefix[i] = sv[i + (i >> 5)];
}

static int64_t lut_cells(int64_t N, int* shift) {
    int sh = 0;
    while (((N - 1) >> sh) >= ((int64_t)1 << kOrdLutBits)) ++sh;
    *shift = sh;
    return ((std::max<int64_t>(N, 1) - 1) >> sh) + 1;
}

// layout of the one slot-order allocation for cap slots (and the bucket bits)
struct OrdLayout {
    size_t T, lut, cnt, bkt[2], ovf[2], total;
};
static OrdLayout ord_layout(int64_t cap, int bits) {
    constexpr int B = 1 << kOrdMaxBits;
    const int cb = ord_capbits_for(cap, bits);
    const size_t capr = (size_t)(cap + 15) / 16 * 16;
    const size_t bk = ((size_t)1 << bits) << cb;
    OrdLayout L;
    size_t o = 0;
    L.T = o;   o += (size_t)(B + 2) * sizeof(int64_t);
    L.lut = o; o += ((size_t)1 << kOrdLutBits) * sizeof(uint16_t);
    L.cnt = o; o += (size_t)(2 * B + 16) * sizeof(uint32_t);   // counts, prefix (B + 1), overflow counts
    for (int i = 0; i < 2; ++i) { L.bkt[i] = o; o += bk * sizeof(uint32_t); }
    for (int i = 0; i < 2; ++i) { L.ovf[i] = o; o += capr * sizeof(uint32_t); }
    L.total = o + 256;
    return L;
}

size_t slot_order_bytes(int64_t cap) { return ord_layout(cap, ord_bits_env()).total; }

// Carve the order buffers out of one allocation of slot_order_bytes(cap) and
// build the per-tensor tables T and lut (once per tensor).
cudaError_t slot_order_init(gcp_ctx* c, void* buf, int64_t cap) {
    constexpr int B = 1 << kOrdMaxBits;
    c->ord_bits = ord_bits_env();
    c->ord_capbits = ord_capbits_for(cap, c->ord_bits);
    const OrdLayout L = ord_layout(cap, c->ord_bits);
    char* p = static_cast<char*>(buf);
    c->d_ord_T = reinterpret_cast<int64_t*>(p + L.T);
    c->d_ord_lut = reinterpret_cast<uint16_t*>(p + L.lut);
    c->d_ord_cnt = reinterpret_cast<uint32_t*>(p + L.cnt);
    for (int i = 0; i < 2; ++i) {
        c->d_ord_bkt[i] = reinterpret_cast<uint32_t*>(p + L.bkt[i]);
        c->d_ord_ovf[i] = reinterpret_cast<uint32_t*>(p + L.ovf[i]);
    }
    cudaError_t e = cudaMemsetAsync(c->d_ord_cnt, 0, (size_t)(2 * B + 16) * sizeof(uint32_t), c->stream);
    if (e != cudaSuccess) return e;
    k_ord_table<<<((1 << c->ord_bits) + 1 + 255) / 256, 256, 0, c->stream>>>(
        c->d_rec, c->rec_words, c->val_words, c->N, (uint32_t)(c->hi[0] - c->lo[0]), c->ord_bits, c->d_ord_T);
    const int64_t ncell = lut_cells(c->N, &c->ord_lut_shift);
    k_ord_lut<<<(int)std::min<int64_t>((ncell + 255) / 256, 4096), 256, 0, c->stream>>>(
        c->d_ord_T, c->ord_bits, c->ord_lut_shift, ncell, std::max<int64_t>(c->N, 1), c->d_ord_lut);
    c->launches += 2;
    return cudaGetLastError();
}

static uint32_t* ord_prefix(gcp_ctx* c) { return c->d_ord_cnt + (1 << kOrdMaxBits); }
static uint32_t* ord_novf(gcp_ctx* c, int par) { return c->d_ord_cnt + 2 * (1 << kOrdMaxBits) + 4 + par; }

static OrdHistArgs make_hist_args(gcp_ctx* c, const SampleArgs& sa, int par) {
    OrdHistArgs oh;
    oh.sa = sa;
    oh.lut = c->d_ord_lut;
    oh.lut_shift = c->ord_lut_shift;
    oh.bits = c->ord_bits;
    oh.capbits = c->ord_capbits;
    oh.counts = c->d_ord_cnt;
    oh.buf = c->d_ord_bkt[par];
    oh.ovf = c->d_ord_ovf[par];
    oh.novf = ord_novf(c, par);
    oh.n = sa.p + sa.q;
    return oh;
}

// The visiting order of this iteration (parity it & 1): its histogram unless
// the previous gradient K2 carried it, then the scan; sets s->ord_*.
cudaError_t launch_slot_order(gcp_ctx* c, SampleArgs* s, bool hist_done) {
    const int64_t n = s->p + s->q;
    const int par = (int)(c->it & 1);
    const int B = 1 << c->ord_bits;
    s->ord_buf = c->d_ord_bkt[par];
    s->ord_prefix = ord_prefix(c);
    s->ord_ovf = c->d_ord_ovf[par];
    s->ord_bits = c->ord_bits;
    s->ord_capbits = c->ord_capbits;
    if (n == 0) return cudaSuccess;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_ord_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(((1 << kOrdMaxBits) + (1 << kOrdMaxBits) / 32) * 4));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (!hist_done) {
        // counts may hold an unconsumed histogram (a K2 prepared an iteration
        // that did not follow): start from zero
        cudaError_t e = cudaMemsetAsync(c->d_ord_cnt, 0, (size_t)B * sizeof(uint32_t), c->stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(ord_novf(c, par), 0, sizeof(uint32_t), c->stream);
        if (e != cudaSuccess) return e;
        const int nb = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8);
        k_ord_hist<<<nb, 256, 0, c->stream>>>(make_hist_args(c, *s, par));
        c->launches++;
    }
    k_ord_scan<<<1, kOrdThreads, (size_t)(B + B / 32) * 4, c->stream>>>(c->d_ord_cnt, ord_prefix(c),
                                                                        ord_novf(c, par ^ 1), B,
                                                                        1u << c->ord_capbits);
    c->launches++;
    return cudaGetLastError();
}

// The histogram of the next iteration (parity (it + 1) & 1) for the gradient
// K2 to carry (GCP_ORD_FUSE=0 keeps it a launch of its own).
bool ord_hist_args(gcp_ctx* c, const SampleArgs& next, OrdHistArgs* oh) {
    const char* fe = getenv("GCP_ORD_FUSE");
    if ((fe && atoi(fe) == 0) || !c->d_ord_buf) return false;
    const int64_t n = next.p + next.q;
    if (n == 0 || n > c->ord_cap) return false;
    *oh = make_hist_args(c, next, (int)((c->it + 1) & 1));
    return true;
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
