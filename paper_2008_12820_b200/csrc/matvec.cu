// The Gauss-Newton Hessian matvec on device (proj/include/vreg/optim.hpp:115-137,
// HessianAdjoint::Transpose with the gradient cache on):
//
//   pre-pass    : w_0 and u_t = vt . grad m_t for all t (k_inc_u)
//   inc state   : nt fused gather steps (linearity: I[m~] - dt/2 I[u] = I[w]),
//                 the TMA-fed pipeline of sl_pipe.cuh
//   transpose   : nt scatter sweeps psi_{t-1} = I^T psi_t (sl_tile.cuh)
//   regulariser : beta (D_3 + D_2 + D_1) vt as three separable 1-D spectral
//                 passes (spec_axis.cu, H1; x1 pass over the slab transpose on
//                 several GPUs), else R2C -> symbol -> C2R through cuFFT
//                 (H2 or axis sizes the in-register FFT lacks); timed as fft
//   assembly    : out = sum_{t=nt..0} w_t psi_t grad m_t + beta A vt, one pass
//
// 2 nt + 5 of our kernels per matvec on one GPU, no host synchronisation.
#include <cstdlib>
#include "common.cuh"

namespace vb {

struct SpecDesc;
void sl_inc_state(vreg_ctx ctx, const Slab& s, const float* disp3, int flags, int degree,
                  const float* grads, const float* vt3, float* mt_all, float* psi_out,
                  float* zero_slices);
void sl_transpose_sweeps(vreg_ctx ctx, const Slab& s, const float* disp3, int flags, int degree,
                         float* psi, bool prezeroed);
float* sl_matvec_psi(vreg_ctx ctx, const Slab& s, const float* disp3, int flags, int degree);
void sl_assemble(vreg_ctx ctx, const Slab& s, int descending, const float* sl, const float* grads,
                 const float* reg, float* out3);
void spectral_regop(vreg_ctx ctx, const Slab& s, const float* v3, double beta, bool unit_zero,
                    bool inverse, float* out3);

namespace {
// Temporarily route the context's stream/communicator to the side branch.
struct SideRoute {
  vreg_ctx ctx;
  cudaStream_t main;
  ncclComm_t comm;
  explicit SideRoute(vreg_ctx c) : ctx(c), main(c->stream), comm(c->comm) {
    c->stream = c->side;
    if (c->fft_comm) c->comm = c->fft_comm;
  }
  ~SideRoute() {
    ctx->stream = main;
    ctx->comm = comm;
  }
};
}  // namespace

// The regulariser branch (separable passes, plus the slab transposes on
// several GPUs) is independent of the transport sweeps until the final
// assembly, so it runs on a side stream (own NCCL communicator) beside them.
void gn_matvec(vreg_ctx ctx, const Slab& s, const float* disp3, int flags, int degree,
               const float* grads, double beta, const float* vt3, float* out3) {
  const size_t N = s.local();
  float* psi = sl_matvec_psi(ctx, s, disp3, flags, degree);
  float* reg = static_cast<float*>(workspace(ctx, "mv_reg", 3 * N * sizeof(float)));
  // Where the regulariser branch runs: 0 serial on the main stream, 1 on the
  // side stream beside the inc-state steps, 2 beside the transpose sweeps.
  // The persistent step sweeps hold every SM, so a branch beside them only
  // delays their CTAs (steps 296 vs 197 us at 256^3); beside the transpose
  // sweeps (many short CTAs) it overlaps: 2.715 (2) vs 2.764 (1) vs 2.789 ms
  // (0) on one GPU. On several GPUs the sweeps carry the boundary bands and
  // reverse exchanges: mode 1 is faster at 256^3 per GPU (3.40 vs 3.65 ms,
  // p = 2), mode 2 from 512^3 per GPU on (25.32 vs 25.67 ms at p = 2, 26.24
  // vs 26.42 ms at p = 4). VREG_MATVEC_OVERLAP overrides,
  // VREG_SERIAL_MATVEC=1 forces 0.
  static const int env_mode = [] {
    const char* e = std::getenv("VREG_SERIAL_MATVEC");
    if (e && e[0] == '1') return 0;
    const char* o = std::getenv("VREG_MATVEC_OVERLAP");
    return o ? std::atoi(o) : -1;
  }();
  const int mode =
      env_mode >= 0 ? env_mode : (ctx->nranks > 1 && N < (size_t(1) << 26) ? 1 : 2);
  auto side_regop = [&] {
    VB_CUDA(cudaEventRecord(ctx->ev_fork, ctx->stream));
    VB_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    SideRoute route(ctx);
    spectral_regop(ctx, s, vt3, beta, false, false, reg);
    VB_CUDA(cudaEventRecord(ctx->ev_join, ctx->side));
  };
  if (mode == 0) spectral_regop(ctx, s, vt3, beta, false, false, reg);
  if (mode == 1) side_regop();
  // on one GPU the inc-state steps also zero psi's slices 0..nt-1, the
  // transpose sweeps' accumulation targets (2.662 vs 2.727 ms at 256^3);
  // on several GPUs the per-sweep memsets stay (the zeroing steps measured
  // 2-5% slower at 512^3 per GPU, neutral at 256^3)
  const bool prezero = ctx->nranks == 1;
  sl_inc_state(ctx, s, disp3, flags, degree, grads, vt3, nullptr, psi + size_t(s.nt) * N,
               prezero ? psi : nullptr);
  if (mode == 2) side_regop();
  sl_transpose_sweeps(ctx, s, disp3, flags, degree, psi, prezero);
  if (mode != 0) VB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
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
