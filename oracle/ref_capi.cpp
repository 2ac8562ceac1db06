// C ABI over the UNMODIFIED reference library (oracle/_ref/libvreg_ref.so).
//
// TEST INFRASTRUCTURE ONLY: built by oracle/Makefile from the reference
// sources where they lie (/root/reference/proj/src/*.cpp, never copied) plus
// the FFTW3 shim. Used by tests/ as the differential oracle, by
// tests/golden/make_golden.py to generate committed fixtures, and by
// bench.py's cpu_baseline / --impl reference legs (kind "reference"). The
// product never links or loads it.
//
// Every entry point is a thin call into the reference's own public API; the
// cited lines are the functions exercised.
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>

#include "vreg/cost_model.hpp"
#include "vreg/optim.hpp"
#include "vreg/syn.hpp"

using namespace vreg;

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const parameter_error*>(&e)) return 2;
  if (dynamic_cast<const numerical_error*>(&e)) return 3;
  if (dynamic_cast<const io_error*>(&e)) return 4;
  if (dynamic_cast<const input_error*>(&e)) return 5;
  if (dynamic_cast<const dimension_error*>(&e)) return 6;
  if (dynamic_cast<const config_error*>(&e)) return 7;
  return 9;
}

#define GUARD(...)                  \
  try {                             \
    __VA_ARGS__;                           \
    return 0;                       \
  } catch (const std::exception& e) { \
    return status_of(e);            \
  }

ScalarField load(const Grid3& g, const double* p) {
  ScalarField f(g);
  std::memcpy(f.data(), p, sizeof(double) * size_t(g.points()));
  return f;
}

VectorField loadv(const Grid3& g, const double* p) {
  VectorField v(g);
  const size_t n = size_t(g.points());
  for (int c = 0; c < 3; ++c)
    std::memcpy(v.comp(c).data(), p + c * n, sizeof(double) * n);
  return v;
}

void store(const ScalarField& f, double* p) {
  std::memcpy(p, f.data(), sizeof(double) * f.v.size());
}

void storev(const VectorField& v, double* p) {
  const size_t n = v.c1.v.size();
  for (int c = 0; c < 3; ++c)
    std::memcpy(p + c * n, v.comp(c).data(), sizeof(double) * n);
}

// Grid without the n >= 8 floor, so coarse grids of the reference's own
// tests (e.g. 6 x 6 x 10) can be addressed; sizes must still be even.
Grid3 grid(int n1, int n2, int n3, int nt) { return Grid3{n1, n2, n3, nt}; }

}  // namespace

// Mirrors RegistrationConfig (proj/include/vreg/optim.hpp:16-37).
struct vref_config {
  double beta_target, beta_start;
  int continuation;
  double gamma_div;
  int project_divfree;
  double eps_newton, eps_h0;
  int max_gn, max_pcg;
  int precond;  // 0 InvA, 1 InvH0, 2 TwoLevelInvH0 (PrecondKind, precond.hpp:12)
  int interp_degree;
  int cache_state_gradient;
  int fixed_gn, fixed_pcg;
  int hessian_adjoint;  // 0 Transpose, 1 SemiLagrangian (optim.hpp:11-14)
  int nt;
  double armijo_c, armijo_shrink;
  int armijo_max_trials, h0_inner_cap;
};

namespace {

RegistrationConfig to_cfg(const vref_config* c) {
  RegistrationConfig r;
  r.beta_target = c->beta_target;
  r.beta_start = c->beta_start;
  r.continuation = c->continuation != 0;
  r.gamma_div = c->gamma_div;
  r.project_divfree = c->project_divfree != 0;
  r.eps_newton = c->eps_newton;
  r.eps_h0 = c->eps_h0;
  r.max_gn = c->max_gn;
  r.max_pcg = c->max_pcg;
  r.precond = PrecondKind(c->precond);
  r.interp_degree = c->interp_degree;
  r.cache_state_gradient = c->cache_state_gradient != 0;
  r.fixed_gn = c->fixed_gn;
  r.fixed_pcg = c->fixed_pcg;
  r.hessian_adjoint = HessianAdjoint(c->hessian_adjoint);
  r.nt = c->nt;
  r.armijo_c = c->armijo_c;
  r.armijo_shrink = c->armijo_shrink;
  r.armijo_max_trials = c->armijo_max_trials;
  r.h0_inner_cap = c->h0_inner_cap;
  return r;
}

void dump_counters(const KernelCounters& k, uint64_t* o) {
  const uint64_t v[] = {k.fft_forward,        k.fft_inverse,
                        k.fft_forward_coarse, k.fft_inverse_coarse,
                        k.fd_gradient,        k.fd_divergence,
                        k.ip_eval,            k.ip_scatter,
                        k.characteristics,    k.characteristics_identity,
                        k.sl_state,           k.sl_adjoint,
                        k.sl_inc_state,       k.sl_inc_adjoint,
                        k.pc_inva_apply,      k.pc_h0_apply,
                        k.pc_h0_inner_iters,  k.pc_h0_inner_solves,
                        k.pc_refresh,         k.h0_inner_work_fine,
                        k.h0_inner_work_coarse};
  std::memcpy(o, v, sizeof(v));
}

// A fixed linearisation point: Flow + StateCache after objective + gradient,
// exactly the state gauss_newton_level holds when it enters PCG
// (optim.hpp:155-168).
struct Session {
  SerialEngine eng;
  RegistrationConfig cfg;
  double beta;
  ScalarField m0, m1;
  std::unique_ptr<Flow<SerialEngine>> flow;
  StateCache<SerialEngine> sc;
  ObjectiveValue J;
  VectorField g;
  std::unique_ptr<Preconditioner<SerialEngine>> prec;
};

}  // namespace

extern "C" {

const char* vref_last_error() { return g_err.c_str(); }

int vref_num_counters() { return 21; }

// syn_template / syn_velocity / syn_reference (proj/src/syn.cpp:9-49).
int vref_syn(int n1, int n2, int n3, int nt, int degree, double* m0,
             double* v3, double* m1) {
  GUARD({
    Grid3 g = Grid3::make(n1, n2, n3, nt);
    if (m0) store(syn_template(g), m0);
    if (v3) storev(syn_velocity(g), v3);
    if (m1) store(syn_reference(g, degree), m1);
  })
}

// SerialEngine::make_characteristics (engine.hpp:111-155); departure points
// interleaved xyz in radians, as QueryPoints stores them (interp.hpp:13-24).
int vref_characteristics(int n1, int n2, int n3, int nt, const double* v3,
                         int degree, double* xyz, int* identity) {
  GUARD({
    Grid3 g = Grid3::make(n1, n2, n3, nt);
    auto ch = compute_characteristics(loadv(g, v3), degree);
    std::memcpy(xyz, ch.dep.xyz.data(), sizeof(double) * ch.dep.xyz.size());
    if (identity) *identity = ch.identity ? 1 : 0;
  })
}

// interpolate / interpolate_core (interp.cpp:70-90).
int vref_interp(int n1, int n2, int n3, const double* f, const double* xyz,
                int64_t m, int degree, double* out) {
  GUARD({
    Grid3 g = grid(n1, n2, n3, 1);
    QueryPoints q(g, m);
    std::memcpy(q.xyz.data(), xyz, sizeof(double) * size_t(3 * m));
    auto vals = interpolate(load(g, f), q, degree);
    std::memcpy(out, vals.data(), sizeof(double) * vals.size());
  })
}

// scatter_transpose_add (interp.cpp:92-108); acc is accumulated into.
int vref_scatter(int n1, int n2, int n3, const double* xyz, const double* z,
                 int64_t m, int degree, double* acc) {
  GUARD({
    Grid3 g = grid(n1, n2, n3, 1);
    ScalarField a = load(g, acc);
    scatter_transpose_add(a, xyz, z, m, degree);
    store(a, acc);
  })
}

// FdOps::gradient / divergence (fd.cpp:150-179).
int vref_fd_grad(int n1, int n2, int n3, const double* f, double* out3) {
  GUARD({ storev(fd_gradient(load(grid(n1, n2, n3, 1), f)), out3); })
}
int vref_fd_div(int n1, int n2, int n3, const double* v3, double* out) {
  GUARD({ store(fd_divergence(loadv(grid(n1, n2, n3, 1), v3)), out); })
}
int vref_fd8_weights(double* w9) {
  GUARD({
    auto w = central_difference_weights(fd_half_width, 1);
    for (int i = 0; i < 9; ++i) w9[i] = w[size_t(i)];
  })
}

// SpectralOps (spectral.cpp:48-288) through the thread-local convenience API.
int vref_regop(int n1, int n2, int n3, const double* v3, double beta,
               int unit_zero, double* out3) {
  GUARD({ storev(apply_regop(loadv(grid(n1, n2, n3, 1), v3), beta, unit_zero != 0), out3); })
}
int vref_inv_regop(int n1, int n2, int n3, const double* v3, double beta,
                   double* out3) {
  GUARD({ storev(apply_inv_regop(loadv(grid(n1, n2, n3, 1), v3), beta), out3); })
}
int vref_seminorm(int n1, int n2, int n3, const double* v3, double* out) {
  GUARD({ *out = h1_seminorm(loadv(grid(n1, n2, n3, 1), v3)); })
}
int vref_leray(int n1, int n2, int n3, const double* v3, double* out3) {
  GUARD({ storev(leray_project(loadv(grid(n1, n2, n3, 1), v3)), out3); })
}
int vref_restrict(int n1, int n2, int n3, const double* f, double* outc) {
  GUARD({ store(restrict_field(load(grid(n1, n2, n3, 1), f)), outc); })
}
int vref_prolong(int n1, int n2, int n3, const double* fc, double* outf) {
  GUARD({
    Grid3 gf = grid(n1, n2, n3, 1);
    store(prolong_field(load(grid(n1 / 2, n2 / 2, n3 / 2, 1), fc), gf), outf);
  })
}
int vref_high_pass(int n1, int n2, int n3, const double* f, double* out) {
  GUARD({ store(high_pass(load(grid(n1, n2, n3, 1), f)), out); })
}
// Half-space spectrum, interleaved (re, im), n1 x n2 x (n3/2+1) (fft.hpp:16-46).
int vref_fft_forward(int n1, int n2, int n3, const double* f, double* out) {
  GUARD({
    SpectralField F = fft_forward(load(grid(n1, n2, n3, 1), f));
    std::memcpy(out, F.c.data(), sizeof(double) * 2 * F.c.size());
  })
}
int vref_inner(int n1, int n2, int n3, const double* a, const double* b,
               double* out) {
  GUARD({
    Grid3 g = grid(n1, n2, n3, 1);
    *out = inner(load(g, a), load(g, b));
  })
}

// ---- linearisation sessions (the PCG-time state of gauss_newton_level) ----

void* vref_session_create(int n1, int n2, int n3, const vref_config* c,
                          double beta, const double* m0, const double* m1,
                          const double* v3) {
  try {
    auto s = std::make_unique<Session>();
    s->cfg = to_cfg(c);
    Grid3 g = Grid3::make(n1, n2, n3, s->cfg.nt);
    s->eng = SerialEngine::create(g);
    s->beta = beta;
    s->m0 = load(g, m0);
    s->m1 = load(g, m1);
    s->flow = std::make_unique<Flow<SerialEngine>>(s->eng, loadv(g, v3),
                                                   s->cfg.interp_degree);
    s->J = detail::evaluate_objective_with(s->eng, *s->flow, s->sc, s->m0,
                                           s->m1, beta, s->cfg);
    s->g = detail::evaluate_gradient_with(s->eng, *s->flow, s->sc, s->m1,
                                          beta, s->cfg);
    return s.release();
  } catch (const std::exception& e) {
    status_of(e);
    return nullptr;
  }
}

void vref_session_destroy(void* h) { delete static_cast<Session*>(h); }

// J.total, J.mismatch, J.regularization, J.div_penalty (optim.hpp:57-87).
int vref_session_objective(void* h, double* J4) {
  auto* s = static_cast<Session*>(h);
  J4[0] = s->J.total;
  J4[1] = s->J.mismatch;
  J4[2] = s->J.regularization;
  J4[3] = s->J.div_penalty;
  return 0;
}

int vref_session_gradient(void* h, double* g3) {
  storev(static_cast<Session*>(h)->g, g3);
  return 0;
}

// m(.,t) for t = 0..nt (sc.m, transport.hpp:90-102).
int vref_session_state(void* h, double* m) {
  auto* s = static_cast<Session*>(h);
  const size_t n = s->m0.v.size();
  for (size_t t = 0; t < s->sc.m.size(); ++t)
    std::memcpy(m + t * n, s->sc.m[t].data(), sizeof(double) * n);
  return 0;
}

int vref_session_chars(void* h, double* fwd_xyz, double* bwd_xyz) {
  auto* s = static_cast<Session*>(h);
  GUARD({
    if (fwd_xyz) {
      const auto& f = s->flow->forward();
      std::memcpy(fwd_xyz, f.dep.xyz.data(), sizeof(double) * f.dep.xyz.size());
    }
    if (bwd_xyz) {
      const auto& b = s->flow->backward();
      std::memcpy(bwd_xyz, b.dep.xyz.data(), sizeof(double) * b.dep.xyz.size());
    }
  })
}

// detail::hessian_matvec_with (optim.hpp:115-137).
int vref_session_matvec(void* h, const double* vt3, double* out3) {
  auto* s = static_cast<Session*>(h);
  GUARD({
    Grid3 g = s->eng.grid();
    storev(detail::hessian_matvec_with(s->eng, *s->flow, s->sc, loadv(g, vt3),
                                       s->beta, s->cfg),
           out3);
  })
}

// solve_inc_state (transport.hpp:145-181): m~(.,t), t = 0..nt.
int vref_session_inc_state(void* h, const double* vt3, double* mt) {
  auto* s = static_cast<Session*>(h);
  GUARD({
    Grid3 g = s->eng.grid();
    auto r = solve_inc_state(*s->flow, loadv(g, vt3), s->sc);
    const size_t n = size_t(g.points());
    for (size_t t = 0; t < r.size(); ++t)
      std::memcpy(mt + t * n, r[t].data(), sizeof(double) * n);
  })
}

// adjoint_transpose_assemble (transport.hpp:207-228) with final condition fin.
int vref_session_transpose_assemble(void* h, const double* fin, double* out3) {
  auto* s = static_cast<Session*>(h);
  GUARD({
    Grid3 g = s->eng.grid();
    storev(adjoint_transpose_assemble(*s->flow, s->sc, load(g, fin)), out3);
  })
}

// Preconditioner<E>::refresh + apply (precond.hpp:80-162), refreshed from the
// deformed template m(.,1) as gauss_newton_level does (optim.hpp:191).
int vref_session_precond(void* h, int kind, const double* r3, double eps_k,
                         double* out3, uint64_t* stats4) {
  auto* s = static_cast<Session*>(h);
  GUARD({
    Grid3 g = s->eng.grid();
    if (!s->prec || int(s->prec->kind()) != kind) {
      s->prec = std::make_unique<Preconditioner<SerialEngine>>(
          s->eng, PrecondKind(kind), s->beta, s->cfg.eps_h0,
          s->cfg.h0_inner_cap);
      s->prec->refresh(s->sc.m.back());
    }
    PrecondStats st;
    storev(s->prec->apply(loadv(g, r3), eps_k, st), out3);
    if (stats4) {
      stats4[0] = st.inva_applications;
      stats4[1] = st.h0_applications;
      stats4[2] = st.inner_iterations;
      stats4[3] = st.inner_capped ? 1 : 0;
    }
  })
}

int vref_session_counters(void* h, uint64_t* out) {
  dump_counters(static_cast<Session*>(h)->eng.counters(), out);
  return 0;
}

int vref_session_timers(void* h, double* out3) {
  auto& k = static_cast<Session*>(h)->eng.kernel_timers();
  out3[0] = k.fft;
  out3[1] = k.fd;
  out3[2] = k.sl;
  return 0;
}

// register_images (optim.hpp:308-347). rep[]: initial_mismatch,
// final_mismatch, mism_rel, final_g_rel, total_gn, total_pcg, flagged,
// phases pc/obj/grad/hess/total, kernels fft/fd/sl, cost-model match.
int vref_register(int n1, int n2, int n3, const vref_config* c,
                  const double* m0, const double* m1, double* v_out3,
                  double* rep, uint64_t* counters) {
  GUARD({
    RegistrationConfig cfg = to_cfg(c);
    Grid3 g = Grid3::make(n1, n2, n3, cfg.nt);
    SerialEngine eng = SerialEngine::create(g);
    VectorField v;
    SolverReport r = register_images(eng, load(g, m0), load(g, m1), cfg, &v);
    if (v_out3) storev(v, v_out3);
    if (rep) {
      rep[0] = r.initial_mismatch;
      rep[1] = r.final_mismatch;
      rep[2] = r.mism_rel;
      rep[3] = r.final_g_rel;
      rep[4] = r.total_gn();
      rep[5] = r.total_pcg();
      rep[6] = r.flagged ? 1 : 0;
      rep[7] = r.phases.pc;
      rep[8] = r.phases.obj;
      rep[9] = r.phases.grad;
      rep[10] = r.phases.hess;
      rep[11] = r.phases.total;
      rep[12] = r.kernels.fft;
      rep[13] = r.kernels.fd;
      rep[14] = r.kernels.sl;
      rep[15] = estimate_cost(r, cfg).matches(r.counters) ? 1 : 0;
    }
    if (counters) dump_counters(r.counters, counters);
  })
}

// register_images (optim.hpp:308-347) with the per-level / per-GN-iteration
// records of its SolverReport (report.hpp:12-78): level rows of 8 doubles
// (beta, pc is inva, switched, gn_iters, pcg_total, final_mismatch,
// final_g_rel, converged) and GN rows of 8 (level, objective, mismatch,
// g_rel, eps_k, alpha, pcg_iters, h0_inner_iters). Capacities in rows;
// counts returned.
int vref_register_levels(int n1, int n2, int n3, const vref_config* c, const double* m0,
                         const double* m1, double* v_out3, double* lev, int lev_cap,
                         int* nlev, double* its, int its_cap, int* nits) {
  GUARD({
    RegistrationConfig cfg = to_cfg(c);
    Grid3 g = Grid3::make(n1, n2, n3, cfg.nt);
    SerialEngine eng = SerialEngine::create(g);
    VectorField v;
    SolverReport r = register_images(eng, load(g, m0), load(g, m1), cfg, &v);
    if (v_out3) storev(v, v_out3);
    int L = 0, I = 0;
    for (const LevelRecord& l : r.levels) {
      if (L < lev_cap) {
        double* o = lev + 8 * L;
        o[0] = l.beta;
        o[1] = l.pc_name == "inva" ? 1.0 : 0.0;
        o[2] = l.pc_switched_from_config ? 1.0 : 0.0;
        o[3] = l.gn_iters;
        o[4] = l.pcg_total;
        o[5] = l.final_mismatch;
        o[6] = l.final_g_rel;
        o[7] = l.converged ? 1.0 : 0.0;
      }
      for (const GnIterRecord& it : l.iters) {
        if (I < its_cap) {
          double* o = its + 8 * I;
          o[0] = L;
          o[1] = it.objective;
          o[2] = it.mismatch;
          o[3] = it.g_rel;
          o[4] = it.eps_k;
          o[5] = it.alpha;
          o[6] = it.pcg_iters;
          o[7] = double(it.h0_inner_iters);
        }
        ++I;
      }
      ++L;
    }
    *nlev = L;
    *nits = I;
  })
}

// PCG relative-residual histories of the last register_levels-style run:
// (level, gn index, pcg iteration, rel. residual) rows, as render_residuals_csv.
int vref_register_residuals(int n1, int n2, int n3, const vref_config* c, const double* m0,
                            const double* m1, double* rows4, int cap, int* nrows) {
  GUARD({
    RegistrationConfig cfg = to_cfg(c);
    Grid3 g = Grid3::make(n1, n2, n3, cfg.nt);
    SerialEngine eng = SerialEngine::create(g);
    SolverReport r = register_images(eng, load(g, m0), load(g, m1), cfg, nullptr);
    int n = 0;
    for (size_t li = 0; li < r.levels.size(); ++li)
      for (size_t k = 0; k < r.levels[li].iters.size(); ++k) {
        const auto& h = r.levels[li].iters[k].pcg_relres;
        for (size_t j = 0; j < h.size(); ++j) {
          if (n < cap) {
            rows4[4 * n] = double(li);
            rows4[4 * n + 1] = double(k + 1);
            rows4[4 * n + 2] = double(j);
            rows4[4 * n + 3] = h[j];
          }
          ++n;
        }
      }
    *nrows = n;
  })
}

}  // extern "C"
