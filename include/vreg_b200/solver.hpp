// Host drivers of the Gauss-Newton-Krylov solver on the B200 backend:
// transport solves, reduced gradient, GN Hessian matvec, PCG, the InvA /
// InvH0 / 2LInvH0 preconditioners and the GN loop with Armijo line search
// and beta continuation. Same algorithms, defaults, stopping rules and
// logical kernel counters as the reference
// (proj/include/vreg/{transport,pcg,precond,optim}.hpp), driving the fused
// device pipelines of libvreg_b200.so instead of op-by-op field code.
#pragma once

#include <algorithm>
#include <cmath>
#include <functional>
#include <optional>
#include <string>
#include <vector>

#include "vreg_b200/cuda_engine.hpp"

namespace vreg_b200 {

enum class PrecondKind { InvA, InvH0, TwoLevelInvH0 };      // precond.hpp:12
enum class HessianAdjoint { Transpose, SemiLagrangian };  // optim.hpp:11-14

inline std::string precond_name(PrecondKind k) {
  return k == PrecondKind::InvA ? "inva" : (k == PrecondKind::InvH0 ? "invh0" : "2linvh0");
}

inline constexpr Real h0_beta_floor = Real(5e-2);     // precond.hpp:24
inline constexpr Real inva_switch_beta = Real(5e-1);  // precond.hpp:25

// optim.hpp:16-55
struct RegistrationConfig {
  Real beta_target = Real(5e-4);
  Real beta_start = Real(1);
  bool continuation = true;
  Real gamma_div = 0;
  bool project_divfree = false;
  Real eps_newton = Real(5e-2);
  Real eps_h0 = Real(1e-3);
  int max_gn = 50;
  int max_pcg = 500;
  PrecondKind precond = PrecondKind::TwoLevelInvH0;
  int interp_degree = 3;
  bool cache_state_gradient = true;
  int fixed_gn = 0;
  int fixed_pcg = 0;
  HessianAdjoint hessian_adjoint = HessianAdjoint::Transpose;
  int nt = 4;
  Real armijo_c = Real(1e-4);
  Real armijo_shrink = Real(0.5);
  int armijo_max_trials = 10;
  int h0_inner_cap = 100;

  void validate() const {
    if (beta_target <= 0 || beta_start <= 0) throw parameter_error("beta must be > 0");
    if (eps_newton <= 0 || eps_newton >= 1) throw parameter_error("eps_newton must lie in (0,1)");
    if (precond != PrecondKind::InvA && (eps_h0 <= 0 || eps_h0 >= 1))
      throw parameter_error("eps_h0 must lie in (0,1)");
    if (gamma_div < 0) throw parameter_error("gamma_div must be >= 0");
    if (interp_degree != 1 && interp_degree != 3)
      throw parameter_error("interp_degree must be 1 or 3");
    if (nt < 1) throw parameter_error("nt must be >= 1");
    if (max_gn < 1 || max_pcg < 1) throw parameter_error("iteration caps must be >= 1");
    if ((fixed_gn > 0) != (fixed_pcg > 0))
      throw parameter_error("fixed_gn and fixed_pcg go together");
  }
};

struct ObjectiveValue {
  Real total = 0, mismatch = 0, regularization = 0, div_penalty = 0;
};

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

// Per-velocity transport state (Flow + StateCache, transport.hpp:17-87):
// lazy forward/backward characteristics, the state series m(t) and the
// cached gradients grad m(t), t = 0..nt, stored contiguously for the fused
// kernels.
class Transport {
 public:
  Transport(CudaEngine& eng, DVField v, int degree)
      : eng_(&eng), vel_(std::move(v)), degree_(degree) {}

  CudaEngine& engine() { return *eng_; }
  const DVField& velocity() const { return vel_; }
  int degree() const { return degree_; }

  const CudaEngine::Char& forward() {
    if (!fwd_) fwd_ = eng_->make_characteristics(vel_, degree_);
    return *fwd_;
  }
  const CudaEngine::Char& backward() {
    if (!bwd_) {
      DVField neg = eng_->make_vfield();
      axpy(Real(-1), vel_, neg);
      bwd_ = eng_->make_characteristics(neg, degree_);
    }
    return *bwd_;
  }

  // m(.,t), t = 0..nt (transport.hpp:90-102)
  void solve_state(const DField& m0) {
    auto& c = eng_->counters();
    c.sl_state++;
    const int nt = eng_->grid().nt;
    const size_t N = m0.local_points();
    m_ = DBuffer(eng_->device(), size_t(nt + 1) * N);
    check(vreg_memcpy_d2d(eng_->ctx(), m_.data(), m0.data(), N * sizeof(float)));
    const auto& ch = forward();
    const vreg_grid g = eng_->vg();
    check(vreg_solve_state(eng_->ctx(), &g, ch.dep.data(), ch.flags, degree_, m_.data()));
    c.ip_eval += std::uint64_t(nt);  // one interp_at per step (transport.hpp:99-100)
    grads_ = DBuffer();
  }
  const float* state(int t) const { return m_.data() + size_t(t) * slab_points(); }
  DField state_field(int t) const {
    DField f = eng_->make_field();
    check(vreg_memcpy_d2d(eng_->ctx(), f.data(), state(t), slab_points() * sizeof(float)));
    return f;
  }

  // grad m(.,t) for all t (StateCache::ensure_gradients, transport.hpp:82-86)
  const float* gradients() {
    if (grads_.empty()) {
      const int nt = eng_->grid().nt;
      const size_t N = slab_points();
      grads_ = DBuffer(eng_->device(), size_t(nt + 1) * 3 * N);
      const vreg_grid g = eng_->vg();
      for (int t = 0; t <= nt; ++t) {
        eng_->counters().fd_gradient++;
        check(vreg_fd_grad(eng_->ctx(), &g, state(t), grads_.data() + size_t(t) * 3 * N));
      }
    }
    return grads_.data();
  }

  // q = (1 + dt/2 D(dep_bwd)) / (1 - dt/2 D) (transport.hpp:49-64)
  const DField& adjoint_source_factor() {
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

  // lambda_t = I_bwd[lambda_{t+1}] .* q, lambda_nt = fin (transport.hpp:106-121)
  DBuffer adjoint_sweep(const DField& fin) {
    const int nt = eng_->grid().nt;
    const size_t N = slab_points();
    const DField& q = adjoint_source_factor();
    const auto& b = backward();
    DBuffer lam(eng_->device(), size_t(nt + 1) * N);
    check(vreg_memcpy_d2d(eng_->ctx(), lam.data() + size_t(nt) * N, fin.data(), N * sizeof(float)));
    const vreg_grid g = eng_->vg();
    check(vreg_adjoint_sweep(eng_->ctx(), &g, b.dep.data(), b.flags, degree_, q.data(), lam.data()));
    eng_->counters().ip_eval += std::uint64_t(nt);
    return lam;
  }

  // sum_t w_t lambda_t grad m_t (transport.hpp:184-201)
  DVField integrate_lambda_grad_m(const DBuffer& lam) {
    const float* gr = gradients();
    DVField out = eng_->make_vfield();
    const vreg_grid g = eng_->vg();
    check(vreg_integrate_lambda_grad_m(eng_->ctx(), &g, lam.data(), gr, out.data()));
    return out;
  }

  size_t slab_points() const {
    return size_t(vel_.local_points());
  }

 private:
  CudaEngine* eng_;
  DVField vel_;
  int degree_;
  std::optional<CudaEngine::Char> fwd_, bwd_;
  std::optional<DField> q_;
  DBuffer m_, grads_;
};

// J = 1/2 ||m(.,1) - m1||^2 + beta/2 |v|_H1^2 + gamma/2 ||div v||^2
// (optim.hpp:66-87); fills the transport state.
inline ObjectiveValue evaluate_objective(CudaEngine& eng, Transport& tr, const DField& m0,
                                         const DField& m1, Real beta,
                                         const RegistrationConfig& cfg) {
  tr.solve_state(m0);
  DField mt = tr.state_field(eng.grid().nt);
  DField resid = eng.make_field();
  sub(mt, m1, resid);
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

// beta A v + int lambda grad m dt, lambda_1 = m1 - m(.,1) (optim.hpp:89-111)
inline DVField evaluate_gradient(CudaEngine& eng, Transport& tr, const DField& m1, Real beta,
                                 const RegistrationConfig& cfg) {
  DField fin = eng.make_field();
  sub(m1, tr.state_field(eng.grid().nt), fin);
  eng.counters().sl_adjoint++;
  DBuffer lam = tr.adjoint_sweep(fin);
  DVField g = tr.integrate_lambda_grad_m(lam);
  DVField reg = eng.regop(tr.velocity(), beta, false);
  axpy(Real(1), reg, g);
  if (cfg.gamma_div > 0) {
    DField dv = eng.fd_div(tr.velocity());
    DVField gd = eng.fd_grad(dv);
    axpy(-cfg.gamma_div, gd, g);
  }
  if (cfg.project_divfree) g = eng.leray(g);
  return g;
}

// GN matvec beta A vt + int lambda~ grad m dt (optim.hpp:113-137). The
// Transpose adjoint runs as one fused device pipeline (vreg_gn_matvec).
inline DVField hessian_matvec(CudaEngine& eng, Transport& tr, const DVField& vt, Real beta,
                              const RegistrationConfig& cfg) {
  auto& c = eng.counters();
  const int nt = eng.grid().nt;
  const vreg_grid g = eng.vg();
  const auto& ch = tr.forward();
  const float* gr = tr.gradients();
  c.sl_inc_state++;
  c.sl_inc_adjoint++;
  c.ip_eval += 2 * std::uint64_t(nt);
  DVField h = eng.make_vfield();
  if (cfg.hessian_adjoint == HessianAdjoint::Transpose) {
    c.ip_scatter += std::uint64_t(nt);
    c.fft_forward += 3;
    c.fft_inverse += 3;
    check(vreg_gn_matvec(eng.ctx(), &g, ch.dep.data(), ch.flags, tr.degree(), gr, beta, vt.data(),
                         h.data()));
  } else {
    DField fin = eng.make_field();
    check(vreg_inc_state(eng.ctx(), &g, ch.dep.data(), ch.flags, tr.degree(), gr, vt.data(),
                         nullptr, fin.data()));
    scale(fin, Real(-1));
    DBuffer lam = tr.adjoint_sweep(fin);
    h = tr.integrate_lambda_grad_m(lam);
    DVField reg = eng.regop(vt, beta, false);
    axpy(Real(1), reg, h);
  }
  if (cfg.gamma_div > 0) {
    DField dv = eng.fd_div(vt);
    DVField gd = eng.fd_grad(dv);
    axpy(-cfg.gamma_div, gd, h);
  }
  return h;
}

// ---- PCG (pcg.hpp:11-94) ----------------------------------------------------

struct PcgOptions {
  Real tol = Real(1e-6);
  int max_iters = 500;
  bool x_is_zero = true;
  bool record_history = true;
};

struct PcgResult {
  int iters = 0;
  Real rel_res = 1;
  bool converged = false;
  bool negative_curvature = false;
  std::vector<Real> history;
};

inline PcgResult pcg(CudaEngine& eng, const std::function<DVField(const DVField&)>& apply_h,
                     const std::function<DVField(const DVField&)>& apply_p, const DVField& b,
                     DVField& x, const PcgOptions& opt) {
  PcgResult res;
  DVField r = b;
  if (!opt.x_is_zero) {
    DVField hx = apply_h(x);
    axpy(Real(-1), hx, r);
  }
  const Real r0n = eng.norm2(r);
  if (r0n == Real(0)) {
    res.converged = true;
    res.rel_res = 0;
    if (opt.record_history) res.history.push_back(0);
    return res;
  }
  DVField z = apply_p(r);
  DVField p = z;
  Real rho = eng.inner(r, z);
  if (opt.record_history) res.history.push_back(1);
  for (int it = 1; it <= opt.max_iters; ++it) {
    DVField q = apply_h(p);
    const Real pq = eng.inner(p, q);
    if (pq <= Real(0)) {
      res.negative_curvature = true;
      return res;
    }
    const Real alpha = rho / pq;
    axpy(alpha, p, x);
    axpy(-alpha, q, r);
    const Real rn = eng.norm2(r);
    res.iters = it;
    res.rel_res = rn / r0n;
    if (opt.record_history) res.history.push_back(res.rel_res);
    if (res.rel_res <= opt.tol) {
      res.converged = true;
      return res;
    }
    if (it == opt.max_iters) break;
    z = apply_p(r);
    const Real rho_new = eng.inner(r, z);
    const Real beta = rho_new / rho;
    rho = rho_new;
    const vreg_grid g = eng.vg();
    check(vreg_aypx(eng.ctx(), &g, 3, beta, z.data(), p.data()));  // p = beta p + z
  }
  return res;
}

// ---- preconditioners (precond.hpp:27-173) ----------------------------------

// H0 s = beta_pc A s + grad_mref (grad_mref . s), unit zero mode (precond.hpp:30-42)
inline DVField h0_matvec(CudaEngine& eng, const DVField& s, const DVField& grad_mref, Real beta_pc) {
  auto& c = eng.counters();
  (eng.is_coarse() ? c.fft_forward_coarse : c.fft_forward) += 3;
  (eng.is_coarse() ? c.fft_inverse_coarse : c.fft_inverse) += 3;
  (eng.is_coarse() ? c.h0_inner_work_coarse : c.h0_inner_work_fine) +=
      std::uint64_t(eng.grid().points());
  DVField out = eng.make_vfield();
  const vreg_grid g = eng.vg();
  check(vreg_h0_matvec(eng.ctx(), &g, s.data(), grad_mref.data(), beta_pc, out.data()));
  return out;
}

struct PrecondStats {
  std::uint64_t inva_applications = 0, h0_applications = 0, inner_iterations = 0;
  Real beta_pc = 0;
  bool inner_capped = false;
};

class Preconditioner {
 public:
  Preconditioner(CudaEngine& eng, PrecondKind kind, Real beta, Real eps_h0, int inner_cap = 100)
      : eng_(&eng), kind_(kind), beta_(beta), beta_pc_(std::max(beta, h0_beta_floor)),
        eps_h0_(eps_h0), inner_cap_(inner_cap) {
    if (kind_ == PrecondKind::TwoLevelInvH0) coarse_.emplace(eng.make_coarse());
    if (kind_ != PrecondKind::InvA && (eps_h0 <= 0 || eps_h0 >= 1))
      throw parameter_error("eps_h0 must lie in (0,1)");
  }
  PrecondKind kind() const { return kind_; }
  Real beta_pc() const { return beta_pc_; }

  void refresh(const DField& deformed_template) {
    if (kind_ == PrecondKind::InvA) return;
    grad_mref_ = eng_->fd_grad(deformed_template);
    if (kind_ == PrecondKind::TwoLevelInvH0) grad_mref_coarse_ = eng_->restrict_to_coarse(*grad_mref_);
    eng_->counters().pc_refresh++;
  }
  void set_reference_gradient(DVField g) {
    grad_mref_ = std::move(g);
    if (kind_ == PrecondKind::TwoLevelInvH0) grad_mref_coarse_ = eng_->restrict_to_coarse(*grad_mref_);
  }

  DVField apply(const DVField& r, Real eps_k, PrecondStats& stats) {
    if (kind_ == PrecondKind::InvA) {
      eng_->counters().pc_inva_apply++;
      stats.inva_applications++;
      return eng_->inv_regop(r, beta_);
    }
    if (!grad_mref_) throw numerical_error("preconditioner not refreshed");
    eng_->counters().pc_h0_apply++;
    eng_->counters().pc_h0_inner_solves++;
    stats.h0_applications++;
    stats.beta_pc = beta_pc_;
    PcgOptions opt;
    opt.tol = eps_h0_ * eps_k;
    opt.max_iters = inner_cap_;
    opt.x_is_zero = false;
    opt.record_history = false;
    if (kind_ == PrecondKind::InvH0) {
      DVField s = eng_->inv_regop(r, beta_pc_);
      auto res = pcg(
          *eng_, [&](const DVField& x) { return h0_matvec(*eng_, x, *grad_mref_, beta_pc_); },
          [&](const DVField& x) { return eng_->inv_regop(x, beta_pc_); }, r, s, opt);
      account(res, stats);
      return s;
    }
    CudaEngine& ce = *coarse_;
    auto inner = [&](const DVField& r_c, DVField& s_c) {
      auto res = pcg(
          ce, [&](const DVField& x) { return h0_matvec(ce, x, *grad_mref_coarse_, beta_pc_); },
          [&](const DVField& x) { return ce.inv_regop(x, beta_pc_); }, r_c, s_c, opt);
      account(res, stats);
    };
    if (eng_->two_level_fused()) {  // one fine forward + one fine inverse transform
      auto rs = eng_->two_level_begin(r, beta_pc_);
      inner(rs.first, rs.second);
      return eng_->two_level_end(rs.second);
    }
    DVField s_f = eng_->inv_regop(r, beta_pc_);
    DVField r_c = eng_->restrict_to_coarse(r);
    DVField s_c = eng_->restrict_to_coarse(s_f);
    inner(r_c, s_c);
    DVField out = eng_->prolong_to_fine(s_c);
    DVField hp = eng_->high_pass_field(s_f);
    axpy(Real(1), hp, out);
    return out;
  }

 private:
  void account(const PcgResult& res, PrecondStats& stats) {
    eng_->counters().pc_h0_inner_iters += std::uint64_t(res.iters);
    stats.inner_iterations += std::uint64_t(res.iters);
    if (!res.converged) stats.inner_capped = true;
  }

  CudaEngine* eng_;
  std::optional<CudaEngine> coarse_;
  PrecondKind kind_;
  Real beta_, beta_pc_, eps_h0_;
  int inner_cap_;
  std::optional<DVField> grad_mref_, grad_mref_coarse_;
};

// ---- Gauss-Newton (optim.hpp:141-359) ---------------------------------------

struct GnIterRecord {
  Real objective = 0, mismatch = 0, g_norm = 0, g_rel = 0, eps_k = 0, alpha = 0;
  int pcg_iters = 0, line_search_trials = 0;
  Real beta_pc = 0;
  std::uint64_t h0_inner_iters = 0;
  std::vector<Real> pcg_relres;
};

struct LevelRecord {
  Real beta = 0;
  std::string pc_name;
  bool pc_switched_from_config = false;
  int gn_iters = 0, pcg_total = 0;
  Real initial_mismatch = 0, final_mismatch = 0, final_g_rel = 0, final_objective = 0;
  bool converged = false, line_search_failed = false, inner_capped = false;
  std::uint64_t refresh_count = 0, pc_inva_apps = 0, pc_h0_apps = 0, h0_inner_total = 0;
  int line_search_states = 0;
  std::vector<GnIterRecord> iters;
};

struct SolverReport {
  Grid3 grid;
  int p = 1, nt = 1;
  std::vector<LevelRecord> levels;
  KernelCounters counters;
  CommCounters comm;
  PhaseTimers phases;
  KernelTimers kernels;
  Real initial_mismatch = 0, final_mismatch = 0, mism_rel = 0, final_g_rel = 0;
  bool flagged = false;
  int total_gn() const {
    int s = 0;
    for (const auto& l : levels) s += l.gn_iters;
    return s;
  }
  int total_pcg() const {
    int s = 0;
    for (const auto& l : levels) s += l.pcg_total;
    return s;
  }
};

// phase timers are host wall clock around device work: synchronise on exit
struct PhaseTimer {
  PhaseTimer(CudaEngine& e, double* acc) : eng(e), t(acc) {}
  ~PhaseTimer() { vreg_ctx_synchronize(eng.ctx()); }
  CudaEngine& eng;
  ScopedTimer t;
};

inline LevelRecord gauss_newton_level(CudaEngine& eng, const DField& m0, const DField& m1, Real beta,
                                      PrecondKind pc_kind, const RegistrationConfig& cfg,
                                      DVField& v, SolverReport& rep) {
  const bool fixed = cfg.fixed_gn > 0;
  LevelRecord lev;
  lev.beta = beta;
  lev.pc_name = precond_name(pc_kind);
  lev.pc_switched_from_config = pc_kind != cfg.precond;

  auto flow = std::make_unique<Transport>(eng, v, cfg.interp_degree);
  ObjectiveValue J;
  {
    PhaseTimer t(eng, &rep.phases.obj);
    J = evaluate_objective(eng, *flow, m0, m1, beta, cfg);
  }
  lev.initial_mismatch = J.mismatch;
  DVField g;
  {
    PhaseTimer t(eng, &rep.phases.grad);
    g = evaluate_gradient(eng, *flow, m1, beta, cfg);
  }
  const Real g0 = eng.norm2(g);
  Preconditioner prec(eng, pc_kind, beta, cfg.eps_h0, cfg.h0_inner_cap);

  Real g_norm = g0;
  for (int k = 0;; ++k) {
    const Real g_rel = g0 > 0 ? g_norm / g0 : Real(0);
    lev.final_g_rel = g_rel;
    if (!fixed && (g0 == Real(0) || g_rel <= cfg.eps_newton)) {
      lev.converged = true;
      break;
    }
    if (fixed ? k >= cfg.fixed_gn : k >= cfg.max_gn) {
      if (!fixed) rep.flagged = true;
      break;
    }
    GnIterRecord rec;
    rec.g_norm = g_norm;
    rec.g_rel = g_rel;
    rec.eps_k = std::min(std::sqrt(g_rel), Real(0.5));
    {
      PhaseTimer t(eng, &rep.phases.pc);
      prec.refresh(flow->state_field(eng.grid().nt));
    }
    if (pc_kind != PrecondKind::InvA) lev.refresh_count++;

    PrecondStats pstats;
    DVField rhs = eng.make_vfield();
    axpy(Real(-1), g, rhs);
    DVField dv = eng.make_vfield();
    PcgOptions opt;
    opt.tol = fixed ? Real(0) : rec.eps_k;
    opt.max_iters = fixed ? cfg.fixed_pcg : cfg.max_pcg;
    opt.x_is_zero = true;
    auto pres = pcg(
        eng,
        [&](const DVField& s) {
          PhaseTimer t(eng, &rep.phases.hess);
          return hessian_matvec(eng, *flow, s, beta, cfg);
        },
        [&](const DVField& r) {
          PhaseTimer t(eng, &rep.phases.pc);
          return prec.apply(r, rec.eps_k, pstats);
        },
        rhs, dv, opt);
    if (pres.negative_curvature)
      throw numerical_error("PCG detected negative curvature in the Gauss-Newton Hessian");
    rec.pcg_iters = pres.iters;
    rec.pcg_relres = std::move(pres.history);
    rec.beta_pc = pstats.beta_pc;
    rec.h0_inner_iters = pstats.inner_iterations;
    lev.pcg_total += pres.iters;
    lev.pc_inva_apps += pstats.inva_applications;
    lev.pc_h0_apps += pstats.h0_applications;
    lev.h0_inner_total += pstats.inner_iterations;
    if (pstats.inner_capped) {
      lev.inner_capped = true;
      rep.flagged = true;
    }
    if (cfg.project_divfree) dv = eng.leray(dv);

    const Real gdv = eng.inner(g, dv);
    bool accepted = false;
    Real alpha = 1;
    std::unique_ptr<Transport> trial;
    ObjectiveValue Jt;
    int trials = 0;
    if (gdv < 0 || fixed) {
      const int max_trials = fixed ? 1 : cfg.armijo_max_trials;
      for (trials = 1; trials <= max_trials; ++trials) {
        DVField v_try = v;
        axpy(alpha, dv, v_try);
        auto f_try = std::make_unique<Transport>(eng, std::move(v_try), cfg.interp_degree);
        {
          PhaseTimer t(eng, &rep.phases.obj);
          Jt = evaluate_objective(eng, *f_try, m0, m1, beta, cfg);
        }
        lev.line_search_states++;
        if (fixed || Jt.total <= J.total + cfg.armijo_c * alpha * gdv) {
          accepted = true;
          trial = std::move(f_try);
          break;
        }
        alpha *= cfg.armijo_shrink;
      }
    }
    rec.line_search_trials = accepted ? trials : cfg.armijo_max_trials;
    rec.alpha = accepted ? alpha : Real(0);
    if (!accepted) {
      lev.line_search_failed = true;
      rep.flagged = true;
      lev.iters.push_back(std::move(rec));
      break;
    }
    axpy(alpha, dv, v);
    flow = std::move(trial);
    J = Jt;
    {
      PhaseTimer t(eng, &rep.phases.grad);
      g = evaluate_gradient(eng, *flow, m1, beta, cfg);
    }
    g_norm = eng.norm2(g);
    rec.objective = J.total;
    rec.mismatch = J.mismatch;
    lev.iters.push_back(std::move(rec));
  }
  lev.gn_iters = int(lev.iters.size());
  lev.final_mismatch = J.mismatch;
  lev.final_objective = J.total;
  return lev;
}

// geometric x10 from beta_start, last level clamped to beta_target (optim.hpp:290-303)
inline std::vector<Real> beta_schedule(const RegistrationConfig& cfg) {
  std::vector<Real> levels;
  if (!cfg.continuation || cfg.beta_target >= cfg.beta_start) {
    levels.push_back(cfg.beta_target);
    return levels;
  }
  for (Real b = cfg.beta_start; b > cfg.beta_target * Real(1 + 1e-12); b /= 10) levels.push_back(b);
  levels.push_back(cfg.beta_target);
  return levels;
}

// optim.hpp:305-347
inline SolverReport register_images(CudaEngine& eng, const DField& m0, const DField& m1,
                                    const RegistrationConfig& cfg, DVField* v_out = nullptr) {
  cfg.validate();
  if (cfg.nt != eng.grid().nt) throw config_error("config nt differs from the engine grid nt");
  SolverReport rep;
  rep.grid = eng.grid();
  rep.nt = eng.grid().nt;
  rep.p = eng.workers();
  {
    PhaseTimer t_total(eng, &rep.phases.total);
    DField d0 = eng.make_field();
    sub(m0, m1, d0);
    const Real dist0 = eng.norm2(d0);
    rep.initial_mismatch = Real(0.5) * dist0 * dist0;
    DVField v = eng.make_vfield();
    for (Real beta : beta_schedule(cfg)) {
      PrecondKind pc = cfg.precond;
      if (cfg.continuation && cfg.precond != PrecondKind::InvA && beta > inva_switch_beta)
        pc = PrecondKind::InvA;
      rep.levels.push_back(gauss_newton_level(eng, m0, m1, beta, pc, cfg, v, rep));
      if (rep.levels.back().line_search_failed) break;
    }
    rep.final_mismatch = rep.levels.back().final_mismatch;
    rep.final_g_rel = rep.levels.back().final_g_rel;
    rep.mism_rel = dist0 > 0 ? std::sqrt(Real(2) * rep.final_mismatch) / dist0 : Real(0);
    if (v_out) *v_out = std::move(v);
  }
  rep.counters = eng.counters();
  rep.comm = eng.comm();
  rep.kernels = eng.kernel_timers();
  return rep;
}

}  // namespace vreg_b200
