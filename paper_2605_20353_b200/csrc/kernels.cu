// kernels.cu -- precision dispatch of the hot-path launchers plus the small
// helper kernels (deterministic partial-sum reduction, scale, subtract).
#include "kernels.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <string>

namespace gcp {

cudaError_t sample_kernel_f32(gcp_ctx*, const SampleArgs&, const ModelArgs&, int, int, int, double, double,
                              int, double*, int);
cudaError_t sample_kernel_f64(gcp_ctx*, const SampleArgs&, const ModelArgs&, int, int, int, double, double,
                              int, double*, int);
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
                                 int nblocks) {
    return c->prec == GCP_FP32
               ? sample_kernel_f32(c, s, m, loss, loss_mode, semi_nz, w_nz, w_z, with_loss, partials, nblocks)
               : sample_kernel_f64(c, s, m, loss, loss_mode, semi_nz, w_nz, w_z, with_loss, partials, nblocks);
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

// Slot ordering for the gradient K2: a counting sort of the slots into
// 2*kOrdB mode-1 position buckets -- nonzero slots by j (records are sorted
// with i_1 most significant, so j order is i_1 order), zero slots by c_1 of the
// attempt-0 candidate, each taken from the top bits of the Philox word
// issue_sample scales into j or c_1 (device.cuh).  Order inside a bucket is arbitrary.
// The sample set, and so the estimate, is unchanged; only the visiting order
// changes, so that K2's gathers and scatter-adds of one mode-1 row meet in L2.
// Three launches: per-CTA bucket histograms (shared-memory atomics), one
// exclusive scan of the bucket-major [bucket][CTA] counts, and the scatter of
// slot ids to their positions (each CTA re-draws the keys of its slot range).
constexpr int kOrdBits = 12;
constexpr int kOrdB = 1 << kOrdBits;
constexpr int kOrdNB = 2 * kOrdB;
constexpr int kOrdThreads = 512;

__device__ __forceinline__ uint32_t slot_bucket(const SampleArgs& a, int64_t s) {
    const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
    // j = mulhi(W, N) and c_1 = mulhi(W, I_1) are monotone in the Philox word W,
    // so its top bits order the slots by j (nonzero) or c_1 (zero) -- no division
    if (s < a.p) {
        const U64x2 w = philox((uint32_t)s, a.rank, a.kind_nz << 28, iter_word(a), k0, k1);
        return (uint32_t)(w.w0 >> (64 - kOrdBits));
    }
    const U64x2 w = philox((uint32_t)(s - a.p), a.rank, a.kind_z << 28, iter_word(a), k0, k1);
    return (uint32_t)kOrdB + (uint32_t)(w.w0 >> (64 - kOrdBits));
}

// radix variant (the default): 16-bit keys, the top 15 bits of W and the
// stratum bit, sorted as (key, slot) pairs by cub (2 passes of 8 bits)
__global__ void k_slot_keys16(const SampleArgs a, uint32_t* __restrict__ keys, uint32_t* __restrict__ slots) {
    const int64_t total = a.p + a.q;
    const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < total;
         s += (int64_t)gridDim.x * blockDim.x) {
        const bool nz = s < a.p;
        const U64x2 w = philox((uint32_t)(nz ? s : s - a.p), a.rank, (nz ? a.kind_nz : a.kind_z) << 28, iter_word(a),
                               k0, k1);
        keys[s] = ((uint32_t)(w.w0 >> 49) << 1) | (nz ? 0u : 1u);
        slots[s] = (uint32_t)s;
    }
}

__global__ void __launch_bounds__(kOrdThreads) k_slot_hist(const SampleArgs a, int64_t per,
                                                            uint32_t* __restrict__ counts) {
    __shared__ uint32_t h[kOrdNB];
    for (int b = threadIdx.x; b < kOrdNB; b += kOrdThreads) h[b] = 0;
    __syncthreads();
    const int64_t s0 = (int64_t)blockIdx.x * per, s1 = min(s0 + per, a.p + a.q);
    for (int64_t s = s0 + threadIdx.x; s < s1; s += kOrdThreads) atomicAdd(&h[slot_bucket(a, s)], 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < kOrdNB; b += kOrdThreads) counts[(size_t)b * gridDim.x + blockIdx.x] = h[b];
}

__global__ void __launch_bounds__(kOrdThreads) k_slot_scatter(const SampleArgs a, int64_t per,
                                                               const uint32_t* __restrict__ offs,
                                                               uint32_t* __restrict__ order) {
    __shared__ uint32_t h[kOrdNB];
    for (int b = threadIdx.x; b < kOrdNB; b += kOrdThreads) h[b] = offs[(size_t)b * gridDim.x + blockIdx.x];
    __syncthreads();
    const int64_t s0 = (int64_t)blockIdx.x * per, s1 = min(s0 + per, a.p + a.q);
    for (int64_t s = s0 + threadIdx.x; s < s1; s += kOrdThreads)
        order[atomicAdd(&h[slot_bucket(a, s)], 1u)] = (uint32_t)s;
}

static int ord_ctas(const gcp_ctx* c) { return c->sm_count * 2; }

// the radix order (16-bit keys) is finer than the counting sort's 2 x 4096
// buckets: on c4 K2 2.85 vs 3.17 ms for 0.47 vs 0.29 ms of ordering, 2.48 vs
// 2.39 epochs/s (profiles/r01_slotorder_*.json); GCP_SLOT_SORT=count selects the other
static bool ord_radix() {
    const char* e = getenv("GCP_SLOT_SORT");
    return !(e && std::string(e) == "count");
}

size_t slot_order_words(const gcp_ctx* c, int64_t cap) {
    return ord_radix() ? 4 * (size_t)cap : 2 * (size_t)kOrdNB * ord_ctas(c) + (size_t)cap;
}

static cudaError_t slot_order_radix(gcp_ctx* c, const SampleArgs& s, uint32_t* buf, int64_t cap, void* tmp,
                                    size_t* tmp_bytes, const uint32_t** order_out) {
    cub::DoubleBuffer<uint32_t> keys(buf, buf ? buf + cap : nullptr);
    cub::DoubleBuffer<uint32_t> vals(buf ? buf + 2 * cap : nullptr, buf ? buf + 3 * cap : nullptr);
    if (!tmp) return cub::DeviceRadixSort::SortPairs(nullptr, *tmp_bytes, keys, vals, (int)cap, 0, 16, c->stream);
    const int64_t n = s.p + s.q;
    const int nb = (int)std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), (int64_t)c->sm_count * 8);
    k_slot_keys16<<<nb, 256, 0, c->stream>>>(s, keys.Current(), vals.Current());
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    c->launches++;
    e = cub::DeviceRadixSort::SortPairs(tmp, *tmp_bytes, keys, vals, (int)n, 0, 16, c->stream);
    if (e != cudaSuccess) return e;
    *order_out = vals.Current();
    return cudaSuccess;
}

// buf: slot_order_words(c, cap) u32 (counts, offsets, order); tmp == nullptr
// queries the scan's *tmp_bytes
cudaError_t launch_slot_order(gcp_ctx* c, const SampleArgs& s, uint32_t* buf, int64_t cap, void* tmp,
                              size_t* tmp_bytes, const uint32_t** order_out) {
    if (ord_radix()) return slot_order_radix(c, s, buf, cap, tmp, tmp_bytes, order_out);
    const int nc = ord_ctas(c);
    const int nbins = kOrdNB * nc;
    uint32_t* counts = buf;
    uint32_t* offs = buf ? buf + nbins : nullptr;
    uint32_t* order = buf ? buf + 2 * (size_t)nbins : nullptr;
    if (!tmp) return cub::DeviceScan::ExclusiveSum(nullptr, *tmp_bytes, counts, offs, nbins, c->stream);
    const int64_t n = s.p + s.q;
    if (n > cap) return cudaErrorInvalidValue;
    const int64_t per = (n + nc - 1) / nc;
    k_slot_hist<<<nc, kOrdThreads, 0, c->stream>>>(s, per, counts);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = cub::DeviceScan::ExclusiveSum(tmp, *tmp_bytes, counts, offs, nbins, c->stream);
    if (e != cudaSuccess) return e;
    k_slot_scatter<<<nc, kOrdThreads, 0, c->stream>>>(s, per, offs, order);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    c->launches += 2;
    *order_out = order;
    return cudaSuccess;
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
