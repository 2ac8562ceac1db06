// The Gauss-Newton Hessian matvec on device (proj/include/vreg/optim.hpp:115-137,
// HessianAdjoint::Transpose with the gradient cache on):
//
//   inc state   : nt fused gather steps (linearity: I[m~] - dt/2 I[u] = I[w])
//   transpose   : nt scatter sweeps psi_{t-1} = I^T psi_t
//   regulariser : R2C(vt) -> beta |k|^2 / N -> C2R   (cuFFT, timed as fft)
//   assembly    : out = sum_{t=nt..0} w_t psi_t grad m_t + beta A vt, one pass
//
// 2 nt + 2 of our kernels + 2 batched cuFFT calls per matvec.
#include "common.cuh"

namespace vb {

struct SpecDesc;
void sl_inc_state(vreg_ctx ctx, const Slab& s, const float* disp3, int flags, int degree,
                  const float* grads, const float* vt3, float* mt_all, float* psi_out);
void sl_transpose_sweeps(vreg_ctx ctx, const Slab& s, const float* disp3, int flags, int degree,
                         float* psi);
void sl_assemble(vreg_ctx ctx, const Slab& s, int descending, const float* sl, const float* grads,
                 const float* reg, float* out3);
void spectral_regop(vreg_ctx ctx, const Slab& s, const float* v3, double beta, bool unit_zero,
                    bool inverse, float* out3);

void gn_matvec(vreg_ctx ctx, const Slab& s, const float* disp3, int flags, int degree,
               const float* grads, double beta, const float* vt3, float* out3) {
  const size_t N = s.local();
  float* psi = static_cast<float*>(workspace(ctx, "mv_psi", size_t(s.nt + 1) * N * sizeof(float)));
  float* reg = static_cast<float*>(workspace(ctx, "mv_reg", 3 * N * sizeof(float)));
  spectral_regop(ctx, s, vt3, beta, false, false, reg);
  sl_inc_state(ctx, s, disp3, flags, degree, grads, vt3, nullptr, psi + size_t(s.nt) * N);
  sl_transpose_sweeps(ctx, s, disp3, flags, degree, psi);
  sl_assemble(ctx, s, 1, psi, grads, reg, out3);
}

}  // namespace vb

using namespace vb;

extern "C" int vreg_gn_matvec(vreg_ctx ctx, const vreg_grid* g, const float* disp3, int identity,
                              int degree, const float* grads, double beta, const float* vt3,
                              float* out3) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    gn_matvec(ctx, s, disp3, identity, degree, grads, beta, vt3, out3);
  });
}
