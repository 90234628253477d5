// kernels.cu -- precision dispatch of the hot-path launchers plus the small
// helper kernels (deterministic partial-sum reduction, scale, subtract).
#include "kernels.cuh"

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
