// dispatch.cuh -- host-side template dispatch of k_sample / k_export / k_adam /
// k_init for one arithmetic type T.  Included by kernels_f32.cu and kernels_f64.cu
// (one translation unit per T so the two instantiation sets compile in parallel).
#pragma once

#include "kernels.cuh"

namespace gcp {

template <typename T, int D, int GL, int NV, int VAR>
static cudaError_t run_sample(gcp_ctx* c, const SampleArgs& s, const ModelArgs& m, const KParams<T>& kp,
                              int nblocks) {
    k_sample<T, D, GL, NV, VAR><<<nblocks, kBlock, 0, c->stream>>>(s, m, kp);
    return cudaGetLastError();
}

template <typename T, int D, int GL, int NV, int VAR = kVarPlain>
static int occ_sample() {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sample<T, D, GL, NV, VAR>, kBlock, 0);
    return nb;
}

// (GL, NV) from the number of 16-byte vectors per row
template <typename T, int D, typename F>
static auto geom_switch(int nvec, F&& f) {
    if (nvec <= 1) return f.template operator()<T, D, 1, 1>();
    if (nvec <= 2) return f.template operator()<T, D, 2, 1>();
    if (nvec <= 4) return f.template operator()<T, D, 4, 1>();
    if (nvec <= 8) return f.template operator()<T, D, 8, 1>();
    if (nvec <= 16) return f.template operator()<T, D, 8, 2>();
    return f.template operator()<T, D, 8, 4>();
}

template <typename T, typename F>
static auto mode_switch(int d, int nvec, F&& f) {
    switch (d) {
    case 2: return geom_switch<T, 2>(nvec, f);
    case 3: return geom_switch<T, 3>(nvec, f);
    case 4: return geom_switch<T, 4>(nvec, f);
    case 5: return geom_switch<T, 5>(nvec, f);
    default: return geom_switch<T, 6>(nvec, f);
    }
}

template <int VAR>
struct SampleLaunch {
    gcp_ctx* c; const SampleArgs* s; const ModelArgs* m; const void* kp; int nblocks;
    template <typename T, int D, int GL, int NV> cudaError_t operator()() const {
        return run_sample<T, D, GL, NV, VAR>(c, *s, *m, *static_cast<const KParams<T>*>(kp), nblocks);
    }
};
template <int VAR = kVarPlain>
struct SampleOcc {
    template <typename T, int D, int GL, int NV> int operator()() const { return occ_sample<T, D, GL, NV, VAR>(); }
};

// one K2 launch of variant VAR (kernels_f32.cu / kernels_f64.cu instantiate the
// plain kernel, kernels_var.cu the peer-access and warp-aggregated ones)
template <typename T, int VAR>
cudaError_t sample_kernel_T(gcp_ctx* c, const SampleArgs& s, const ModelArgs& m, int loss, int loss_mode,
                            int semi_nz, double w_nz, double w_z, int with_loss, double* partials,
                            int nblocks, const OrdHistArgs* oh) {
    KParams<T> kp;
    if (oh) kp.oh = *oh;
    else memset(&kp.oh, 0, sizeof(kp.oh));
    kp.loss = loss; kp.loss_mode = loss_mode; kp.semi_nz = semi_nz; kp.with_loss = with_loss;
    kp.w_nz = (T)w_nz; kp.w_z = (T)w_z; kp.partials = partials;
    const int nvec = m.R_pad / Vec16<T>::n;
    return mode_switch<T>(c->d, nvec, SampleLaunch<VAR>{c, &s, &m, &kp, nblocks});
}

template <typename T, int VAR = kVarPlain>
int sample_occupancy_T(int d, int R_pad) {
    return mode_switch<T>(d, R_pad / Vec16<T>::n, SampleOcc<VAR>{});
}

template <typename T>
cudaError_t export_T(gcp_ctx* c, const SampleArgs& s, int64_t first, int64_t count, const int64_t* lo,
                     int64_t* subs, int64_t* j, int32_t* att) {
    const int nb = (int)((count + 255) / 256);
    if (count == 0) return cudaSuccess;
    switch (c->d) {
    case 2: k_export<T, 2><<<nb, 256, 0, c->stream>>>(s, first, count, lo, subs, j, att); break;
    case 3: k_export<T, 3><<<nb, 256, 0, c->stream>>>(s, first, count, lo, subs, j, att); break;
    case 4: k_export<T, 4><<<nb, 256, 0, c->stream>>>(s, first, count, lo, subs, j, att); break;
    case 5: k_export<T, 5><<<nb, 256, 0, c->stream>>>(s, first, count, lo, subs, j, att); break;
    default: k_export<T, 6><<<nb, 256, 0, c->stream>>>(s, first, count, lo, subs, j, att); break;
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t adam_T(gcp_ctx* c, const Segment& seg, void* A, void* G, void* B, void* C, double rate,
                   double beta1, double beta2, double eps, double lower, int64_t t, int zero_g, int R_pad,
                   int row_stride, const DevStep* step, const OrdScatterArgs* os) {
    const double bc1 = 1.0 / (1.0 - pow(beta1, (double)t));
    const double bc2 = 1.0 / (1.0 - pow(beta2, (double)t));
    int64_t nvec = 0;
    for (int i = 0; i < seg.n; ++i) nvec += seg.len[i] / Vec16<T>::n;
    OrdScatterArgs nos;
    memset(&nos, 0, sizeof(nos));
    if (nvec == 0 && !(os && os->n)) return cudaSuccess;
    int64_t nb = (std::max<int64_t>(nvec, 1) + 255) / 256;
    const int64_t cap = (int64_t)c->sm_count * 8;
    if (nb > cap) nb = cap;
    k_adam<T><<<(int)nb, 256, 0, c->stream>>>(seg, nvec, (T*)A, (T*)G, (T*)B, (T*)C, (T)rate, (T)beta1,
                                              (T)beta2, (T)eps, (T)bc1, (T)bc2, (T)lower, zero_g, R_pad, row_stride, step,
                                              (long long)t, os ? *os : nos);
    return cudaGetLastError();
}

template <typename T>
cudaError_t init_T(gcp_ctx* c, const InitArgs& ia, void* A) {
    int64_t nb = (ia.n_coef + 255) / 256;
    const int64_t cap = (int64_t)c->sm_count * 8;
    if (nb > cap) nb = cap;
    if (nb < 1) nb = 1;
    k_init<T><<<(int)nb, 256, 0, c->stream>>>(ia, (T*)A);
    return cudaGetLastError();
}

}  // namespace gcp
