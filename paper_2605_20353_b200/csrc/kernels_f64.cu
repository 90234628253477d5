// kernels_f64.cu -- instantiation of the hot-path kernels for T = double.
#include "dispatch.cuh"

namespace gcp {
cudaError_t sample_kernel_f64(gcp_ctx* c, const SampleArgs& s, const ModelArgs& m, int loss, int loss_mode,
                            int semi_nz, double w_nz, double w_z, int with_loss, double* partials, int nb,
                            const OrdHistArgs* oh) {
    return sample_kernel_T<double, kVarPlain>(c, s, m, loss, loss_mode, semi_nz, w_nz, w_z, with_loss, partials, nb, oh);
}
int sample_occupancy_f64(int d, int R_pad) { return sample_occupancy_T<double>(d, R_pad); }
cudaError_t export_f64(gcp_ctx* c, const SampleArgs& s, int64_t first, int64_t count, const int64_t* lo,
                     int64_t* subs, int64_t* j, int32_t* att) {
    return export_T<double>(c, s, first, count, lo, subs, j, att);
}
cudaError_t adam_f64(gcp_ctx* c, const Segment& seg, void* A, void* G, void* B, void* C, double rate,
                   double b1, double b2, double eps, double lower, int64_t t, int zero_g, int R_pad,
                   int row_stride, const DevStep* step, const OrdScatterArgs* os) {
    return adam_T<double>(c, seg, A, G, B, C, rate, b1, b2, eps, lower, t, zero_g, R_pad, row_stride, step, os);
}
cudaError_t init_f64(gcp_ctx* c, const InitArgs& ia, void* A) { return init_T<double>(c, ia, A); }
}  // namespace gcp
