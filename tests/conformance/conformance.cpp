// Drop-in conformance: the reference's OWN templates, instantiated with
// vreg_b200::CudaEngine in place of vreg::SerialEngine, against the serial
// run of the same templates.
//
//   vreg::solve_state / evaluate_objective_with   (transport.hpp, optim.hpp)
//   vreg::detail::hessian_matvec_with              (optim.hpp:115-137)
//   vreg::pcg                                      (pcg.hpp:30-94)
//   vreg::Preconditioner<E> (InvA, 2LInvH0)        (precond.hpp:56-173)
//
// Built by tests/conformance/Makefile against /root/reference/proj/include
// (read in place) + oracle/_ref/libvreg_ref.a + libvreg_b200.so. Prints one
// line per check "name rel_err" and exits non-zero if any exceeds 1e-4.
#define VREG_B200_WITH_REFERENCE
#include <cstdio>
#include <vector>

#include "vreg/optim.hpp"
#include "vreg/syn.hpp"
#include "vreg_b200/cuda_engine.hpp"

using namespace vreg;
using CE = vreg_b200::CudaEngine;

static double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / den);
}

static std::vector<double> flat(const VectorField& v) {
  std::vector<double> o;
  for (int c = 0; c < 3; ++c) o.insert(o.end(), v.comp(c).v.begin(), v.comp(c).v.end());
  return o;
}
static std::vector<double> flat(const ScalarField& f) { return f.v; }

int main() {
  const int n = 32, nt = 4;
  const Real beta = 1e-3;
  Grid3 g = Grid3::make(n, n, n, nt);
  RegistrationConfig cfg;
  cfg.continuation = false;
  cfg.beta_target = beta;

  ScalarField m0 = syn_template(g), m1 = syn_reference(g, 3);
  VectorField v = syn_velocity(g);
  scale(v, Real(0.5));

  // serial reference run of the templates
  SerialEngine se = SerialEngine::create(g);
  Flow<SerialEngine> fs(se, v, 3);
  StateCache<SerialEngine> ss;
  ObjectiveValue Js = detail::evaluate_objective_with(se, fs, ss, m0, m1, beta, cfg);
  VectorField grad = detail::evaluate_gradient_with(se, fs, ss, m1, beta, cfg);
  VectorField vt = grad;
  scale(vt, Real(-1));
  VectorField Hs = detail::hessian_matvec_with(se, fs, ss, vt, beta, cfg);

  // the same templates on the B200 backend
  CE ce = CE::create(g);
  Flow<CE> fc(ce, ce.from_global_v(v), 3);
  StateCache<CE> sc;
  ObjectiveValue Jc = detail::evaluate_objective_with(ce, fc, sc, ce.from_global(m0),
                                                      ce.from_global(m1), beta, cfg);
  CE::VField vtc = ce.from_global_v(vt);
  CE::VField Hc = detail::hessian_matvec_with(ce, fc, sc, vtc, beta, cfg);

  int bad = 0;
  auto report = [&](const char* name, double e) {
    std::printf("%s %.3e\n", name, e);
    if (!(e <= 1e-4)) ++bad;
  };
  report("objective", std::abs(Jc.total / Js.total - 1));
  report("mismatch", std::abs(Jc.mismatch / Js.mismatch - 1));
  report("hessian_matvec", rel(Hc.to_host(), flat(Hs)));
  // engine.hpp:63-66 round trip: from_global / to_global(_v)
  report("to_global", rel(flat(ce.to_global(ce.from_global(m0))), flat(m0)));
  report("to_global_v", rel(flat(ce.to_global_v(Hc)), Hc.to_host()));

  // pcg on the GN Hessian with the InvA preconditioner, 5 iterations
  PcgOptions opt;
  opt.tol = 0;
  opt.max_iters = 5;
  VectorField xs(g);
  VectorField rhs = grad;
  scale(rhs, Real(-1));
  pcg(se, [&](const VectorField& s) { return detail::hessian_matvec_with(se, fs, ss, s, beta, cfg); },
      [&](const VectorField& r) { return se.inv_regop(r, beta); }, rhs, xs, opt);
  CE::VField xc = ce.make_vfield();
  CE::VField rhsc = ce.from_global_v(rhs);
  pcg(ce, [&](const CE::VField& s) { return detail::hessian_matvec_with(ce, fc, sc, s, beta, cfg); },
      [&](const CE::VField& r) { return ce.inv_regop(r, beta); }, rhsc, xc, opt);
  report("pcg_5_inva", rel(xc.to_host(), flat(xs)));

  // two-level preconditioner apply (reference gradient installed directly)
  VectorField gm = fd_gradient(m1);
  Preconditioner<SerialEngine> ps(se, PrecondKind::TwoLevelInvH0, beta, cfg.eps_h0);
  ps.set_reference_gradient(gm);
  Preconditioner<CE> pc(ce, PrecondKind::TwoLevelInvH0, beta, cfg.eps_h0);
  pc.set_reference_gradient(ce.from_global_v(gm));
  PrecondStats st1, st2;
  VectorField zs = ps.apply(rhs, 0.5, st1);
  CE::VField zc = pc.apply(rhsc, 0.5, st2);
  report("precond_2linvh0", rel(zc.to_host(), flat(zs)));
  std::printf("inner_iters serial %llu device %llu\n", (unsigned long long)st1.inner_iterations,
              (unsigned long long)st2.inner_iterations);

  // identical logical counters on both backends for the matvec
  std::printf("counters ip_eval serial %llu device %llu, ip_scatter %llu %llu\n",
              (unsigned long long)se.counters().ip_eval, (unsigned long long)ce.counters().ip_eval,
              (unsigned long long)se.counters().ip_scatter,
              (unsigned long long)ce.counters().ip_scatter);
  return bad ? 1 : 0;
}
