// kernels.cu -- precision dispatch of the hot-path launchers plus the small
// helper kernels (deterministic partial-sum reduction, scale, subtract).
#include "kernels.cuh"

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

// Slot ordering for the gradient K2 (DRAM-resident mode-1 rows: c4, c5): a
// hand-written counting sort of the iteration's slots into kOrdB buckets of
// mode-1 position, nonzero and zero slots interleaved (a bucket holds the
// nonzero slots whose record lies in a mode-1 row range AND the zero slots
// whose attempt-0 candidate lies in the same range, so K2 fills the A|G lines
// of a row range once per iteration, not once per stratum).  The sample set,
// and so the estimate, is unchanged; only the visiting order changes, so that
// K2's gathers and scatter-adds of one mode-1 row meet in L2.
//   k_ord_hist     Philox word -> bucket (nonzero: j = mulhi(W, N), then the
//                  bucket whose record range [T[b], T[b+1]) holds j, by binary
//                  search of the per-tensor table T in shared memory; zero:
//                  c_1 = mulhi(W, I_1), bucket floor(c_1 B / I_1)); u16 key per
//                  slot; shared-memory histogram; one global atomicAdd per
//                  (CTA, bucket)
//   k_ord_scan     one CTA: exclusive scan of the bucket totals -> cursors;
//                  totals reset for the next iteration
//   k_ord_scatter  per CTA: histogram of its keys again, one atomicAdd per
//                  (CTA, bucket) reserves its run, slot ids scattered into it
// Order inside a bucket is arbitrary (and run to run: CTAs reserve in arrival
// order), which only moves the fp32 atomic summation order.
constexpr int kOrdBits = 12;
constexpr int kOrdB = 1 << kOrdBits;
constexpr int kOrdThreads = 1024;
constexpr size_t kOrdSmem = kOrdB * sizeof(uint32_t) + (kOrdB + 1) * sizeof(int64_t);

// T[b] = first canonical record whose c_1 >= ceil(b I_1 / B), b = 0..B (T[B] = N):
// records are sorted with i_1 most significant (reading R15)
__global__ void k_ord_table(const uint32_t* __restrict__ rec, int rec_words, int val_words, int64_t N, uint32_t I1,
                            int64_t* __restrict__ T) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > kOrdB) return;
    const uint64_t row = ((uint64_t)b * I1 + kOrdB - 1) >> kOrdBits;
    int64_t lo = 0, hi = N;
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (rec[mid * rec_words + val_words] < row) lo = mid + 1;
        else hi = mid;
    }
    T[b] = lo;
}

__global__ void __launch_bounds__(kOrdThreads) k_ord_hist(const SampleArgs a, const int64_t* __restrict__ T,
                                                         int64_t per, uint16_t* __restrict__ keys,
                                                         uint32_t* __restrict__ totals) {
    extern __shared__ __align__(16) unsigned char ord_smem[];
    int64_t* sT = reinterpret_cast<int64_t*>(ord_smem);
    uint32_t* h = reinterpret_cast<uint32_t*>(sT + kOrdB + 1);
    for (int b = threadIdx.x; b < kOrdB; b += kOrdThreads) h[b] = 0;
    for (int b = threadIdx.x; b <= kOrdB; b += kOrdThreads) sT[b] = T[b];
    __syncthreads();
    const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
    const uint32_t it = iter_word(a);
    const int64_t s0 = (int64_t)blockIdx.x * per, s1 = min(s0 + per, a.p + a.q);
    for (int64_t s = s0 + threadIdx.x; s < s1; s += kOrdThreads) {
        uint32_t b;
        if (s < a.p) {
            const U64x2 w = philox((uint32_t)s, a.rank, a.kind_nz << 28, it, k0, k1);
            const int64_t j = (int64_t)range_map(w.w0, (uint64_t)a.N);
            uint32_t lo = 0, hi = kOrdB;          // largest b with T[b] <= j (T[0] = 0 <= j < T[B] = N)
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (sT[mid] <= j) lo = mid;
                else hi = mid;
            }
            b = lo;
        } else {
            const U64x2 w = philox((uint32_t)(s - a.p), a.rank, a.kind_z << 28, it, k0, k1);
            const uint64_t c1 = range_map(w.w0, a.bdim[0]);
            b = (uint32_t)((c1 << kOrdBits) / a.bdim[0]);
        }
        keys[s] = (uint16_t)b;
        atomicAdd(&h[b], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kOrdB; b += kOrdThreads)
        if (h[b]) atomicAdd(&totals[b], h[b]);
}

__global__ void __launch_bounds__(kOrdThreads) k_ord_scan(uint32_t* __restrict__ totals, uint32_t* __restrict__ cursor) {
    constexpr int PER = kOrdB / kOrdThreads;
    __shared__ uint32_t wsum[kOrdThreads / 32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t v[PER], run = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        v[i] = totals[t * PER + i];
        totals[t * PER + i] = 0;
        run += v[i];
    }
    uint32_t incl = run;   // inclusive warp scan of the per-thread sums
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
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
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        cursor[t * PER + i] = base;
        base += v[i];
    }
}

__global__ void __launch_bounds__(kOrdThreads) k_ord_scatter(const uint16_t* __restrict__ keys, int64_t n,
                                                            int64_t per, uint32_t* __restrict__ cursor,
                                                            uint32_t* __restrict__ order) {
    __shared__ uint32_t h[kOrdB];
    for (int b = threadIdx.x; b < kOrdB; b += kOrdThreads) h[b] = 0;
    __syncthreads();
    const int64_t s0 = (int64_t)blockIdx.x * per, s1 = min(s0 + per, n);
    for (int64_t s = s0 + threadIdx.x; s < s1; s += kOrdThreads) atomicAdd(&h[keys[s]], 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < kOrdB; b += kOrdThreads)
        if (h[b]) h[b] = atomicAdd(&cursor[b], h[b]);   // this CTA's run of bucket b
    __syncthreads();
    for (int64_t s = s0 + threadIdx.x; s < s1; s += kOrdThreads) order[atomicAdd(&h[keys[s]], 1u)] = (uint32_t)s;
}

size_t slot_order_bytes(int64_t cap) {
    return (size_t)cap * (sizeof(uint32_t) + sizeof(uint16_t)) + 2 * kOrdB * sizeof(uint32_t) +
           (kOrdB + 1) * sizeof(int64_t) + 64;
}

// Carve the order buffers out of one allocation of slot_order_bytes(cap) and
// build the per-tensor table T (once per tensor).
cudaError_t slot_order_init(gcp_ctx* c, void* buf, int64_t cap) {
    char* p = static_cast<char*>(buf);
    c->d_ord_T = reinterpret_cast<int64_t*>(p);
    p += (kOrdB + 1) * sizeof(int64_t);
    c->d_ord_cnt = reinterpret_cast<uint32_t*>(p);
    p += 2 * kOrdB * sizeof(uint32_t);
    c->d_ord = reinterpret_cast<uint32_t*>(p);
    p += (size_t)cap * sizeof(uint32_t);
    c->d_ord_key = reinterpret_cast<uint16_t*>(p);
    cudaError_t e = cudaMemsetAsync(c->d_ord_cnt, 0, 2 * kOrdB * sizeof(uint32_t), c->stream);
    if (e != cudaSuccess) return e;
    k_ord_table<<<(kOrdB + 1 + 255) / 256, 256, 0, c->stream>>>(c->d_rec, c->rec_words, c->val_words, c->N,
                                                                (uint32_t)(c->hi[0] - c->lo[0]), c->d_ord_T);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_slot_order(gcp_ctx* c, const SampleArgs& s, const uint32_t** order_out) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_ord_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOrdSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int64_t n = s.p + s.q;
    if (n == 0) {
        *order_out = c->d_ord;
        return cudaSuccess;
    }
    const int nc = c->sm_count;
    const int64_t per = (n + nc - 1) / nc;
    uint32_t* totals = c->d_ord_cnt;
    uint32_t* cursor = c->d_ord_cnt + kOrdB;
    k_ord_hist<<<nc, kOrdThreads, kOrdSmem, c->stream>>>(s, c->d_ord_T, per, c->d_ord_key, totals);
    k_ord_scan<<<1, kOrdThreads, 0, c->stream>>>(totals, cursor);
    k_ord_scatter<<<nc, kOrdThreads, 0, c->stream>>>(c->d_ord_key, n, per, cursor, c->d_ord);
    c->launches += 3;
    *order_out = c->d_ord;
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
