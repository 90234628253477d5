// kernels_peer_f32.cu -- instantiation of the K2 peer-access (two-sided over NVLink) variant (kernels.cuh)
// for T = float; one translation unit per (variant, type) so they compile in
// parallel with the plain kernels (kernels_f32.cu / kernels_f64.cu).
#include "dispatch.cuh"

namespace gcp {
cudaError_t sample_kernel_peer_f32(gcp_ctx* c, const SampleArgs& s, const ModelArgs& m, int loss, int loss_mode,
                                  int semi_nz, double w_nz, double w_z, int with_loss, double* partials, int nb,
                                  const OrdHistArgs* oh) {
    return sample_kernel_T<float, kVarPeer>(c, s, m, loss, loss_mode, semi_nz, w_nz, w_z, with_loss, partials, nb, oh);
}
int sample_occupancy_peer_f32(int d, int R_pad) { return sample_occupancy_T<float, kVarPeer>(d, R_pad); }
}  // namespace gcp
