// Device-resident Gauss-Newton-Krylov registration on the B200 backend.
//
// The reference drives its solve from templated host code over field
// objects (proj/include/vreg/{transport,pcg,precond,optim}.hpp). Here the
// inner loops live on the device:
//
//  * Transport       -- one linearisation (velocity): lazy characteristics,
//                       the state series and its gradient cache as flat
//                       device buffers feeding the fused kernels;
//  * DevicePrecond   -- InvA / InvH0 / 2LInvH0 as stream-ordered device
//                       operators; the H0 inner solves are Krylov solves
//                       (csrc/krylov.cu), recorded as nested conditional
//                       graph nodes when the outer PCG body is captured, and
//                       a stand-alone apply replays a cached graph;
//  * Newton          -- one Gauss-Newton level: the PCG solve of H dv = -g is
//                       a single conditional-WHILE graph launch with fp64
//                       iterates, followed by the Armijo backtracking on the
//                       objective;
//  * run_registration -- the beta continuation.
//
// Decisions (stopping rules, forcing term, line-search acceptance, the InvA
// switch, the beta schedule) are the reference's, so runs follow the same
// iteration counts; logical kernel counters are derived from the iteration
// counts the device reports, identical to the reference's increments.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <optional>
#include <vector>

#include "common.cuh"
#include "krylov.hpp"
#include "vreg_b200/cuda_engine.hpp"
#include "vreg_b200/records.hpp"

namespace vreg_b200 {

// Contiguous device buffer of n fp32 values (time series, gradient caches).
class DBuffer {
 public:
  DBuffer() = default;
  DBuffer(std::shared_ptr<Device> dev, size_t n) : dev_(std::move(dev)), n_(n) {
    void* p = nullptr;
    check(vreg_alloc(dev_->ctx(), n * sizeof(float), &p));
    auto d = dev_;
    buf_ = std::shared_ptr<float>(static_cast<float*>(p), [d](float* q) { vreg_free(d->ctx(), q); });
  }
  float* data() { return buf_.get(); }
  const float* data() const { return buf_.get(); }
  size_t size() const { return n_; }
  bool empty() const { return !buf_; }

 private:
  std::shared_ptr<Device> dev_;
  std::shared_ptr<float> buf_;
  size_t n_ = 0;
};

inline vb::Slab slab_for(vreg_ctx ctx, const Grid3& g) {
  const vreg_grid vg = to_vg(g);
  return vb::slab_of(ctx, &vg);
}

// ---- transport state of one velocity (transport.hpp:17-228 semantics) ------

class Transport {
 public:
  Transport(CudaEngine& eng, DVField v, int degree)
      : eng_(&eng), vel_(std::move(v)), degree_(degree) {}

  CudaEngine& engine() { return *eng_; }
  const DVField& velocity() const { return vel_; }
  int degree() const { return degree_; }
  size_t points() const { return size_t(vel_.local_points()); }

  const CudaEngine::Char& forward() {
    if (!fwd_) fwd_ = eng_->make_characteristics(vel_, degree_);
    return *fwd_;
  }
  const CudaEngine::Char& backward() {  // characteristics of -v
    if (!bwd_) {
      DVField neg = eng_->make_vfield();
      axpy(Real(-1), vel_, neg);
      bwd_ = eng_->make_characteristics(neg, degree_);
    }
    return *bwd_;
  }

  // m(., t), t = 0..nt
  void solve_state(const DField& m0) {
    auto& c = eng_->counters();
    c.sl_state++;
    const int nt = eng_->grid().nt;
    const size_t N = points();
    m_ = DBuffer(eng_->device(), size_t(nt + 1) * N);
    check(vreg_memcpy_d2d(eng_->ctx(), m_.data(), m0.data(), N * sizeof(float)));
    const auto& ch = forward();
    const vreg_grid g = eng_->vg();
    check(vreg_solve_state(eng_->ctx(), &g, ch.dep.data(), ch.flags, degree_, m_.data()));
    c.ip_eval += std::uint64_t(nt);
    grads_ = DBuffer();
  }
  const float* state(int t) const { return m_.data() + size_t(t) * points(); }
  DField state_field(int t) const {
    DField f = eng_->make_field();
    check(vreg_memcpy_d2d(eng_->ctx(), f.data(), state(t), points() * sizeof(float)));
    return f;
  }

  // grad m(., t) for all t, contiguous (the gradient cache)
  const float* gradients() {
    if (grads_.empty()) {
      const int nt = eng_->grid().nt;
      const size_t N = points();
      grads_ = DBuffer(eng_->device(), size_t(nt + 1) * 3 * N);
      const vreg_grid g = eng_->vg();
      for (int t = 0; t <= nt; ++t) {
        eng_->counters().fd_gradient++;
        check(vreg_fd_grad(eng_->ctx(), &g, state(t), grads_.data() + size_t(t) * 3 * N));
      }
    }
    return grads_.data();
  }

  // adjoint source factor q = (1 + dt/2 D(dep_bwd)) / (1 - dt/2 D)
  const DField& source_factor() {
    if (!q_) {
      const auto& b = backward();
      DField q = eng_->make_field();
      auto& c = eng_->counters();
      c.fd_divergence++;
      c.ip_eval++;
      const vreg_grid g = eng_->vg();
      check(vreg_adjoint_source_factor(eng_->ctx(), &g, vel_.data(), b.dep.data(), b.flags,
                                       degree_, q.data()));
      q_ = std::move(q);
    }
    return *q_;
  }

  // lambda_t backward from lambda_nt = fin
  DBuffer adjoint(const DField& fin) {
    const int nt = eng_->grid().nt;
    const size_t N = points();
    const DField& q = source_factor();
    const auto& b = backward();
    DBuffer lam(eng_->device(), size_t(nt + 1) * N);
    check(vreg_memcpy_d2d(eng_->ctx(), lam.data() + size_t(nt) * N, fin.data(), N * sizeof(float)));
    const vreg_grid g = eng_->vg();
    check(vreg_adjoint_sweep(eng_->ctx(), &g, b.dep.data(), b.flags, degree_, q.data(), lam.data()));
    eng_->counters().ip_eval += std::uint64_t(nt);
    return lam;
  }

  DVField lambda_grad_m(const DBuffer& lam) {
    const float* gr = gradients();
    DVField out = eng_->make_vfield();
    const vreg_grid g = eng_->vg();
    check(vreg_integrate_lambda_grad_m(eng_->ctx(), &g, lam.data(), gr, out.data()));
    return out;
  }

 private:
  CudaEngine* eng_;
  DVField vel_;
  int degree_;
  std::optional<CudaEngine::Char> fwd_, bwd_;
  std::optional<DField> q_;
  DBuffer m_, grads_;
};

// J = 1/2 ||m(.,1) - m1||^2 + beta/2 |v|_H1^2 + gamma/2 ||div v||^2; fills tr's state
inline ObjectiveValue objective(CudaEngine& eng, Transport& tr, const DField& m0, const DField& m1,
                                Real beta, const RegistrationConfig& cfg) {
  tr.solve_state(m0);
  DField resid = eng.make_field();
  sub(tr.state_field(eng.grid().nt), m1, resid);
  ObjectiveValue J;
  J.mismatch = Real(0.5) * eng.inner(resid, resid);
  J.regularization = beta / 2 * eng.seminorm(tr.velocity());
  if (cfg.gamma_div > 0) {
    DField dv = eng.fd_div(tr.velocity());
    J.div_penalty = cfg.gamma_div / 2 * eng.inner(dv, dv);
  }
  J.total = J.mismatch + J.regularization + J.div_penalty;
  return J;
}

// g = beta A v + int lambda grad m dt (lambda_1 = m1 - m(.,1)) [- gamma grad div v]
inline DVField gradient(CudaEngine& eng, Transport& tr, const DField& m1, Real beta,
                        const RegistrationConfig& cfg) {
  DField fin = eng.make_field();
  sub(m1, tr.state_field(eng.grid().nt), fin);
  eng.counters().sl_adjoint++;
  DVField g = tr.lambda_grad_m(tr.adjoint(fin));
  axpy(Real(1), eng.regop(tr.velocity(), beta, false), g);
  if (cfg.gamma_div > 0) axpy(-cfg.gamma_div, eng.fd_grad(eng.fd_div(tr.velocity())), g);
  if (cfg.project_divfree) g = eng.leray(g);
  return g;
}

// Logical counters of one GN matvec (the reference's increments).
inline void count_matvecs(KernelCounters& c, const RegistrationConfig& cfg, int nt,
                          std::uint64_t n) {
  c.sl_inc_state += n;
  c.sl_inc_adjoint += n;
  c.ip_eval += 2 * std::uint64_t(nt) * n;
  if (cfg.hessian_adjoint == HessianAdjoint::Transpose) {
    c.ip_scatter += std::uint64_t(nt) * n;
    c.fft_forward += 3 * n;
    c.fft_inverse += 3 * n;
  } else {  // SL adjoint: + nt interpolations, regop FFTs
    c.ip_eval += std::uint64_t(nt) * n;
    c.fft_forward += 3 * n;
    c.fft_inverse += 3 * n;
  }
  if (cfg.gamma_div > 0) {
    c.fd_divergence += n;
    c.fd_gradient += n;
  }
}

// H vt as a stream-ordered device operation (no host synchronisation), for
// the Krylov solver. Transpose adjoint without div penalty: the fused
// pipeline on the caller's buffers; other variants build on the engine ops.
inline void matvec_into(CudaEngine& eng, Transport& tr, Real beta, const RegistrationConfig& cfg,
                        const float* vt3, float* out3) {
  const vreg_grid g = eng.vg();
  const auto& ch = tr.forward();
  const float* gr = tr.gradients();
  const size_t bytes = 3 * tr.points() * sizeof(float);
  if (cfg.hessian_adjoint == HessianAdjoint::Transpose && cfg.gamma_div == 0) {
    check(vreg_gn_matvec(eng.ctx(), &g, ch.dep.data(), ch.flags, tr.degree(), gr, beta, vt3, out3));
    return;
  }
  DVField vt = eng.make_vfield();
  check(vreg_memcpy_d2d(eng.ctx(), vt.data(), vt3, bytes));
  const KernelCounters keep = eng.counters();  // the caller counts matvecs
  DVField h;
  if (cfg.hessian_adjoint == HessianAdjoint::Transpose) {
    h = eng.make_vfield();
    check(vreg_gn_matvec(eng.ctx(), &g, ch.dep.data(), ch.flags, tr.degree(), gr, beta,
                         vt.data(), h.data()));
  } else {
    DField fin = eng.make_field();
    check(vreg_inc_state(eng.ctx(), &g, ch.dep.data(), ch.flags, tr.degree(), gr, vt.data(),
                         nullptr, fin.data()));
    scale(fin, Real(-1));
    h = tr.lambda_grad_m(tr.adjoint(fin));
    axpy(Real(1), eng.regop(vt, beta, false), h);
  }
  if (cfg.gamma_div > 0) axpy(-cfg.gamma_div, eng.fd_grad(eng.fd_div(vt)), h);
  eng.counters() = keep;
  check(vreg_memcpy_d2d(eng.ctx(), out3, h.data(), bytes));
}

// ---- preconditioners (precond.hpp:56-173 semantics) -------------------------

struct PrecondTally {
  std::uint64_t inva = 0, h0 = 0, inner = 0;
  bool capped = false;
};

class DevicePrecond {
 public:
  DevicePrecond(CudaEngine& eng, PrecondKind kind, Real beta, Real eps_h0, int inner_cap)
      : eng_(&eng), kind_(kind), beta_(beta), beta_pc_(std::max(beta, h0_beta_floor)),
        eps_h0_(eps_h0), cap_(inner_cap) {
    if (kind_ != PrecondKind::InvA && (eps_h0 <= 0 || eps_h0 >= 1))
      throw parameter_error("eps_h0 must lie in (0,1)");
    if (kind_ == PrecondKind::TwoLevelInvH0) coarse_.emplace(eng.make_coarse());
    if (kind_ != PrecondKind::InvA) {
      void* p = nullptr;
      check(vreg_alloc(eng.ctx(), 2 * sizeof(unsigned long long), &p));
      acc_ = static_cast<unsigned long long*>(p);
      VB_CUDA(cudaMemsetAsync(acc_, 0, 2 * sizeof(unsigned long long), eng.ctx()->stream));
    }
  }
  ~DevicePrecond() {
    if (graph_) cudaGraphExecDestroy(graph_);
    if (cstream_) cudaStreamDestroy(cstream_);
    if (acc_) vreg_free(eng_->ctx(), acc_);
  }
  DevicePrecond(const DevicePrecond&) = delete;
  DevicePrecond& operator=(const DevicePrecond&) = delete;

  PrecondKind kind() const { return kind_; }
  Real beta_pc() const { return kind_ == PrecondKind::InvA ? Real(0) : beta_pc_; }

  // grad of the deformed template (and its restriction for 2LInvH0)
  void refresh(const DField& deformed_template) {
    if (kind_ == PrecondKind::InvA) return;
    gm_.emplace(eng_->fd_grad(deformed_template));
    if (kind_ == PrecondKind::TwoLevelInvH0) gm_c_.emplace(eng_->restrict_to_coarse(*gm_));
    eng_->counters().pc_refresh++;
    drop_graph();
  }

  // z = M r, stream-ordered (recorded when the stream is being captured)
  void apply(const float* r, float* z, Real eps_k) {
    vreg_ctx ctx = eng_->ctx();
    if (kind_ == PrecondKind::InvA) {
      const vreg_grid g = eng_->vg();
      check(vreg_inv_regop(ctx, &g, r, beta_, z));
      return;
    }
    if (!gm_) throw numerical_error("preconditioner not refreshed");
    const Real tol = eps_h0_ * eps_k;
    if (kind_ == PrecondKind::InvH0) {
      // s0 = InvA_pc r, then PCG on H0 s = r with InvA_pc (precond.hpp:104-131)
      const vreg_grid g = eng_->vg();
      check(vreg_inv_regop(ctx, &g, r, beta_pc_, z));
      if (split_h0())
        inner(*eng_, *gm_).solve_h0(gm_->data(), op_inv(*eng_), r, z, tol, cap_, acc_);
      else
        inner(*eng_, *gm_).solve(op_h0(*eng_, *gm_), op_inv(*eng_), r, z, tol, cap_, true, acc_);
      return;
    }
    // two-level: restrictions of r and InvA_pc r from one forward transform,
    // the coarse H0 solve, prolongation + high pass with one inverse
    CudaEngine& ce = *coarse_;
    if (!rc_) {
      rc_.emplace(ce.make_vfield());
      sc_.emplace(ce.make_vfield());
    }
    const vreg_grid g = eng_->vg();
    std::optional<vb::Timed> phase;
    phase.emplace(ctx, -1, "pc_2l_begin");
    if (eng_->workers() == 1) {
      // the split inner solve starts from s_c0 alone (r0 = -G s_c0)
      check(vreg_two_level_begin(ctx, &g, r, beta_pc_, split_h0() ? nullptr : rc_->data(),
                                 sc_->data()));
    } else {
      // slab-distributed: restrict(InvA_f r) = InvA_c restrict(r) mode by
      // mode, so high_pass(InvA_f r) = InvA_f r - prolong(s_c0) with the
      // coarse start s_c0 = InvA_c r_c, and the apply is
      // InvA_f r + prolong(s_c - s_c0): one fine restriction and one
      // prolongation instead of three and two (precond.hpp:133-162)
      if (!tmp_) {
        tmp_.emplace(eng_->make_vfield());
        sc0_.emplace(ce.make_vfield());
      }
      const vreg_grid gc = ce.vg();
      check(vreg_inv_regop(ctx, &g, r, beta_pc_, tmp_->data()));
      check(vreg_restrict(ctx, &g, 3, r, rc_->data()));
      check(vreg_inv_regop(ctx, &gc, rc_->data(), beta_pc_, sc_->data()));
      check(vreg_copy(ctx, &gc, 3, sc_->data(), sc0_->data()));
    }
    phase.emplace(ctx, -1, "pc_2l_inner");
    if (split_h0())
      inner(ce, *gm_c_).solve_h0(gm_c_->data(), op_inv(ce), rc_->data(), sc_->data(), tol, cap_,
                                 acc_);
    else
      inner(ce, *gm_c_).solve(op_h0(ce, *gm_c_), op_inv(ce), rc_->data(), sc_->data(), tol,
                              cap_, true, acc_);
    phase.emplace(ctx, -1, "pc_2l_end");
    if (eng_->workers() == 1) {
      check(vreg_two_level_end(ctx, &g, sc_->data(), z));
    } else {
      const vreg_grid gc = ce.vg();
      check(vreg_axpy(ctx, &gc, 3, -1.0, sc0_->data(), sc_->data()));
      check(vreg_prolong(ctx, &g, 3, sc_->data(), z));
      check(vreg_axpy(ctx, &g, 3, 1.0, tmp_->data(), z));
    }
  }

  // One stand-alone apply (not inside a captured solve): the whole apply is
  // a cached graph per (refresh, eps_k), replayed on fixed buffers.
  void apply_once(const float* r, float* z, Real eps_k) {
    if (kind_ == PrecondKind::InvA || !graph_ok() || eng_->workers() > 1) {
      apply(r, z, eps_k);
      return;
    }
    vreg_ctx ctx = eng_->ctx();
    const size_t bytes = 3 * slab_for(ctx, eng_->grid()).local() * sizeof(float);
    if (!gin_) {
      gin_.emplace(eng_->make_vfield());
      gout_.emplace(eng_->make_vfield());
    }
    check(vreg_memcpy_d2d(ctx, gin_->data(), r, bytes));
    if (!graph_ || graph_eps_ != eps_k) {
      drop_graph();
      apply(gin_->data(), gout_->data(), eps_k);  // warm: plans, workspaces
      // captured on a private stream (the context's stream may be the legacy
      // default stream, which cannot be captured); launched on the context's
      cudaStream_t st = ctx->stream;
      if (!cstream_) VB_CUDA(cudaStreamCreateWithFlags(&cstream_, cudaStreamNonBlocking));
      VB_CUDA(cudaStreamSynchronize(st));
      cudaGraph_t gr;
      VB_CUDA(cudaStreamBeginCapture(cstream_, cudaStreamCaptureModeRelaxed));
      ctx->stream = cstream_;
      try {
        apply(gin_->data(), gout_->data(), eps_k);
      } catch (...) {
        ctx->stream = st;
        cudaStreamEndCapture(cstream_, &gr);
        throw;
      }
      ctx->stream = st;
      VB_CUDA(cudaStreamEndCapture(cstream_, &gr));
      VB_CUDA(cudaGraphInstantiate(&graph_, gr, 0));
      cudaGraphDestroy(gr);
      graph_eps_ = eps_k;
      // the warm apply above counts as an application: undo its tally
      take_device();
    }
    VB_CUDA(cudaGraphLaunch(graph_, ctx->stream));
    check(vreg_memcpy_d2d(ctx, z, gout_->data(), bytes));
  }

  // Logical counters of `apps` applications whose inner solves ran `inner`
  // iterations in total (the reference's increments, precond.hpp:30-162).
  void count(std::uint64_t apps, std::uint64_t inner_its, PrecondTally& t) {
    KernelCounters& c = eng_->counters();
    if (kind_ == PrecondKind::InvA) {
      c.pc_inva_apply += apps;
      c.fft_forward += 3 * apps;
      c.fft_inverse += 3 * apps;
      t.inva += apps;
      return;
    }
    c.pc_h0_apply += apps;
    c.pc_h0_inner_solves += apps;
    c.pc_h0_inner_iters += inner_its;
    t.h0 += apps;
    t.inner += inner_its;
    // each inner solve: one H0 apply for r = b - H0 s0 plus one per
    // iteration, one InvA_pc per iteration (applied at the top of each)
    const std::uint64_t h0s = apps + inner_its, invs = inner_its;
    if (kind_ == PrecondKind::InvH0) {
      const std::uint64_t N = std::uint64_t(eng_->grid().points());
      c.fft_forward += 3 * (apps + h0s + invs);
      c.fft_inverse += 3 * (apps + h0s + invs);
      c.h0_inner_work_fine += N * h0s;
      return;
    }
    const std::uint64_t Nc = std::uint64_t(eng_->grid().coarse().points());
    // fine: InvA r, two restrictions' forward transforms; high pass, prolongation's inverse
    c.fft_forward += apps * (3 + 6 + 3);
    c.fft_inverse += apps * (3 + 3 + 3);
    c.fft_inverse_coarse += apps * 6;
    c.fft_forward_coarse += apps * 3;
    c.fft_forward_coarse += 3 * (h0s + invs);
    c.fft_inverse_coarse += 3 * (h0s + invs);
    c.h0_inner_work_coarse += Nc * h0s;
  }

  // inner iterations / capped flag accumulated on the device since the last call
  std::pair<std::uint64_t, bool> take_device() {
    if (!acc_) return {0, false};
    unsigned long long h[2] = {0, 0};
    vreg_ctx ctx = eng_->ctx();
    VB_CUDA(cudaMemcpyAsync(h, acc_, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
    VB_CUDA(cudaMemsetAsync(acc_, 0, sizeof(h), ctx->stream));
    return {h[0], h[1] != 0};
  }

 private:
  // the inner H0 solves run split (one spectral solve per iteration,
  // Krylov::solve_h0); VREG_H0_SPLIT=0 applies H0 and InvA as two operators
  static bool split_h0() {
    static const bool on = [] {
      const char* e = std::getenv("VREG_H0_SPLIT");
      return !(e && e[0] == '0');
    }();
    return on;
  }
  static bool graph_ok() {
    const char* e = std::getenv("VREG_PCG_GRAPH");
    return !(e && e[0] == '0');
  }
  void drop_graph() {
    if (graph_) cudaGraphExecDestroy(graph_);
    graph_ = nullptr;
  }
  vb::Krylov& inner(CudaEngine& e, const DVField&) {
    auto& k = e.is_coarse() ? kc_ : kf_;
    // fp32 iterates: the inner tolerance is eps_h0 eps_k (~1e-4)
    if (!k) k = std::make_unique<vb::Krylov>(e.ctx(), slab_for(e.ctx(), e.grid()), false);
    return *k;
  }
  vb::KrylovOp op_h0(CudaEngine& e, const DVField& gm) {
    const vreg_grid g = e.vg();
    const float* gmp = gm.data();
    vreg_ctx ctx = e.ctx();
    const double b = beta_pc_;
    return [=](const float* in, float* out) { check(vreg_h0_matvec(ctx, &g, in, gmp, b, out)); };
  }
  vb::KrylovOp op_inv(CudaEngine& e) {
    const vreg_grid g = e.vg();
    vreg_ctx ctx = e.ctx();
    const double b = beta_pc_;
    return [=](const float* in, float* out) { check(vreg_inv_regop(ctx, &g, in, b, out)); };
  }

  CudaEngine* eng_;
  std::optional<CudaEngine> coarse_;
  PrecondKind kind_;
  Real beta_, beta_pc_, eps_h0_;
  int cap_;
  std::optional<DVField> gm_, gm_c_, rc_, sc_, sc0_, tmp_, gin_, gout_;
  std::unique_ptr<vb::Krylov> kf_, kc_;
  unsigned long long* acc_ = nullptr;
  cudaGraphExec_t graph_ = nullptr;
  cudaStream_t cstream_ = nullptr;  // capture stream of the cached apply graph
  Real graph_eps_ = -1;
};

// ---- the outer PCG: H dv = -g ----------------------------------------------

struct PcgOutcome {
  vb::KrylovStats stats;
  PrecondTally tally;
  double t_pc = 0, t_hess = 0;
};

class OuterPcg {
 public:
  OuterPcg(CudaEngine& eng) : eng_(&eng) {}
  PcgOutcome solve(Transport& tr, DevicePrecond& pc, Real beta, const RegistrationConfig& cfg,
                   const DVField& g, Real eps_k, DVField& dv) {
    if (!kr_ || kr_->fp64() != cfg.pcg_fp64)
      kr_ = std::make_unique<vb::Krylov>(eng_->ctx(), slab_for(eng_->ctx(), eng_->grid()),
                                         cfg.pcg_fp64);
    DVField rhs = eng_->make_vfield();
    axpy(Real(-1), g, rhs);
    const bool fixed = cfg.fixed();
    const double tol = fixed ? 0.0 : double(eps_k);
    const int max_it = fixed ? cfg.fixed_pcg : cfg.max_pcg;
    // phase split: CUDA events around the operator and the preconditioner
    // on their eager (uncaptured) passes give the device-time ratio the
    // solve's wall time is divided by
    vreg_ctx ctx = eng_->ctx();
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pc, ev_h;
    auto timed = [&](std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& evs, auto&& f) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      VB_CUDA(cudaStreamIsCapturing(ctx->stream, &cs));
      if (cs != cudaStreamCaptureStatusNone) return f();
      cudaEvent_t a, b;
      VB_CUDA(cudaEventCreate(&a));
      VB_CUDA(cudaEventCreate(&b));
      VB_CUDA(cudaEventRecord(a, ctx->stream));
      f();
      VB_CUDA(cudaEventRecord(b, ctx->stream));
      evs.emplace_back(a, b);
    };
    vb::KrylovOp A = [&](const float* in, float* out) {
      timed(ev_h, [&] { matvec_into(*eng_, tr, beta, cfg, in, out); });
    };
    vb::KrylovOp M = [&](const float* in, float* out) {
      timed(ev_pc, [&] { pc.apply(in, out, eps_k); });
    };
    pc.take_device();
    const auto t0 = std::chrono::steady_clock::now();
    PcgOutcome o;
    // the fused matvec is capture-safe (no host synchronisation, no
    // allocation); the op-by-op variants run the loop eagerly
    const bool graph = cfg.hessian_adjoint == HessianAdjoint::Transpose && cfg.gamma_div == 0;
    o.stats = kr_->solve(A, M, rhs.data(), dv.data(), tol, max_it, false, nullptr, graph);
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const auto inner = pc.take_device();
    const std::uint64_t apps = std::uint64_t(o.stats.iters);
    count_matvecs(eng_->counters(), cfg, eng_->grid().nt, apps);
    pc.count(apps, inner.first, o.tally);
    o.tally.capped = inner.second;
    auto sum = [](std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& evs) {
      double t = 0;
      for (auto& e : evs) {
        float ms = 0;
        VB_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
        t += ms;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
      }
      return t;
    };
    const double d_pc = sum(ev_pc), d_h = sum(ev_h);
    o.t_pc = d_pc + d_h > 0 ? wall * d_pc / (d_pc + d_h) : 0;
    o.t_hess = wall - o.t_pc;
    return o;
  }

 private:
  CudaEngine* eng_;
  std::unique_ptr<vb::Krylov> kr_;
};

// ---- one Gauss-Newton level and the continuation ---------------------------

class Registration {
 public:
  Registration(CudaEngine& eng, const DField& m0, const DField& m1, const RegistrationConfig& cfg)
      : eng_(eng), m0_(m0), m1_(m1), cfg_(cfg), pcg_(eng) {}

  // Levels of the continuation: beta_start / 10^k while above beta_target
  // (relative tolerance 1e-12), then beta_target (optim.hpp:290-303).
  std::vector<Real> levels() const {
    std::vector<Real> out;
    if (cfg_.continuation && cfg_.beta_target < cfg_.beta_start) {
      Real b = cfg_.beta_start;
      while (b > cfg_.beta_target * Real(1 + 1e-12)) {
        out.push_back(b);
        b /= 10;
      }
    }
    out.push_back(cfg_.beta_target);
    return out;
  }

  PrecondKind precond_at(Real beta) const {
    const bool force_inva =
        cfg_.continuation && cfg_.precond != PrecondKind::InvA && beta > inva_switch_beta;
    return force_inva ? PrecondKind::InvA : cfg_.precond;
  }

  SolverReport run(DVField* v_out) {
    cfg_.validate();
    if (cfg_.nt != eng_.grid().nt) throw config_error("config nt differs from the engine grid nt");
    SolverReport rep;
    rep.grid = eng_.grid();
    rep.nt = eng_.grid().nt;
    rep.p = eng_.workers();
    {
      PhaseClock total(eng_, &rep.phases.total);
      DField d0 = eng_.make_field();
      sub(m0_, m1_, d0);
      const Real dist0 = eng_.norm2(d0);
      rep.initial_mismatch = Real(0.5) * dist0 * dist0;
      v_ = eng_.make_vfield();
      for (Real beta : levels()) {
        rep.levels.push_back(level(beta, precond_at(beta), rep));
        if (rep.levels.back().line_search_failed) break;
      }
      rep.final_mismatch = rep.levels.back().final_mismatch;
      rep.final_g_rel = rep.levels.back().final_g_rel;
      rep.mism_rel = dist0 > 0 ? std::sqrt(Real(2) * rep.final_mismatch) / dist0 : Real(0);
    }
    if (v_out) *v_out = v_;
    rep.counters = eng_.counters();
    rep.comm = eng_.comm();
    rep.kernels = eng_.kernel_timers();
    return rep;
  }

 private:
  // host wall clock around device work, synchronised at the end
  struct PhaseClock {
    PhaseClock(CudaEngine& e, double* acc) : eng(e), t(acc) {}
    ~PhaseClock() { vreg_ctx_synchronize(eng.ctx()); }
    CudaEngine& eng;
    ScopedTimer t;
  };

  struct Iterate {  // linearisation point of the current Newton iterate
    std::unique_ptr<Transport> flow;
    ObjectiveValue J;
  };

  Iterate evaluate(DVField v, Real beta, SolverReport& rep) {
    Iterate it;
    it.flow = std::make_unique<Transport>(eng_, std::move(v), cfg_.interp_degree);
    PhaseClock t(eng_, &rep.phases.obj);
    it.J = objective(eng_, *it.flow, m0_, m1_, beta, cfg_);
    return it;
  }

  DVField grad(Iterate& it, Real beta, SolverReport& rep) {
    PhaseClock t(eng_, &rep.phases.grad);
    return gradient(eng_, *it.flow, m1_, beta, cfg_);
  }

  // Armijo backtracking from v along dv (sufficient decrease c alpha <g, dv>;
  // a fixed-iteration run takes the full step). Returns the accepted iterate.
  std::optional<Iterate> line_search(const Iterate& cur, const DVField& dv, Real gdv, Real beta,
                                     GnIterRecord& rec, LevelRecord& lev, SolverReport& rep) {
    const bool fixed = cfg_.fixed();
    const int budget = fixed ? 1 : cfg_.armijo_max_trials;
    rec.line_search_trials = cfg_.armijo_max_trials;
    rec.alpha = 0;
    if (!(gdv < 0 || fixed)) return std::nullopt;
    Real alpha = 1;
    for (int trial = 1; trial <= budget; ++trial, alpha *= cfg_.armijo_shrink) {
      DVField v_try = v_;
      axpy(alpha, dv, v_try);
      Iterate cand = evaluate(std::move(v_try), beta, rep);
      lev.line_search_states++;
      if (fixed || cand.J.total <= cur.J.total + cfg_.armijo_c * alpha * gdv) {
        rec.line_search_trials = trial;
        rec.alpha = alpha;
        return cand;
      }
    }
    return std::nullopt;
  }

  LevelRecord level(Real beta, PrecondKind pc_kind, SolverReport& rep) {
    LevelRecord lev;
    lev.beta = beta;
    lev.pc_name = precond_name(pc_kind);
    lev.pc_switched_from_config = pc_kind != cfg_.precond;
    Iterate cur = evaluate(v_, beta, rep);
    lev.initial_mismatch = cur.J.mismatch;
    DVField g = grad(cur, beta, rep);
    const Real g0 = eng_.norm2(g);
    Real g_norm = g0;
    DevicePrecond pc(eng_, pc_kind, beta, cfg_.eps_h0, cfg_.h0_inner_cap);
    const int cap = cfg_.fixed() ? cfg_.fixed_gn : cfg_.max_gn;
    for (int k = 0;; ++k) {
      const Real g_rel = g0 > 0 ? g_norm / g0 : Real(0);
      lev.final_g_rel = g_rel;
      if (!cfg_.fixed() && (g0 == 0 || g_rel <= cfg_.eps_newton)) {
        lev.converged = true;
        break;
      }
      if (k >= cap) {
        if (!cfg_.fixed()) rep.flagged = true;
        break;
      }
      GnIterRecord rec;
      rec.g_norm = g_norm;
      rec.g_rel = g_rel;
      rec.eps_k = std::min(std::sqrt(g_rel), Real(0.5));  // forcing term
      {
        PhaseClock t(eng_, &rep.phases.pc);
        pc.refresh(cur.flow->state_field(eng_.grid().nt));
      }
      if (pc_kind != PrecondKind::InvA) lev.refresh_count++;
      DVField dv = eng_.make_vfield();
      PcgOutcome o = pcg_.solve(*cur.flow, pc, beta, cfg_, g, rec.eps_k, dv);
      rep.phases.pc += o.t_pc;
      rep.phases.hess += o.t_hess;
      if (o.stats.negative_curvature)
        throw numerical_error("PCG detected negative curvature in the Gauss-Newton Hessian");
      rec.pcg_iters = o.stats.iters;
      rec.pcg_relres = o.stats.history;
      rec.beta_pc = pc.beta_pc();
      rec.h0_inner_iters = o.tally.inner;
      lev.pcg_total += o.stats.iters;
      lev.pc_inva_apps += o.tally.inva;
      lev.pc_h0_apps += o.tally.h0;
      lev.h0_inner_total += o.tally.inner;
      if (o.tally.capped) {
        lev.inner_capped = true;
        rep.flagged = true;
      }
      if (cfg_.project_divfree) dv = eng_.leray(dv);
      const Real gdv = eng_.inner(g, dv);
      std::optional<Iterate> next = line_search(cur, dv, gdv, beta, rec, lev, rep);
      if (!next) {
        lev.line_search_failed = true;
        rep.flagged = true;
        lev.iters.push_back(std::move(rec));
        break;
      }
      axpy(rec.alpha, dv, v_);
      cur = std::move(*next);
      g = grad(cur, beta, rep);
      g_norm = eng_.norm2(g);
      rec.objective = cur.J.total;
      rec.mismatch = cur.J.mismatch;
      lev.iters.push_back(std::move(rec));
    }
    lev.gn_iters = int(lev.iters.size());
    lev.final_mismatch = cur.J.mismatch;
    lev.final_objective = cur.J.total;
    return lev;
  }

  CudaEngine& eng_;
  const DField& m0_;
  const DField& m1_;
  RegistrationConfig cfg_;
  OuterPcg pcg_;
  DVField v_;
};

}  // namespace vreg_b200
