// Public schema of the B200 Gauss-Newton-Krylov solver: the run
// configuration and the report records. Field names, defaults and the
// validation rules are the reference's interface (RegistrationConfig,
// proj/include/vreg/optim.hpp:16-55; GnIterRecord / LevelRecord /
// SolverReport, proj/include/vreg/report.hpp:12-78), so reports and configs
// round-trip between the two. The solver itself is device-resident
// (paper_2008_12820_b200/csrc/host/gnk.hpp over csrc/krylov.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "vreg_b200/types.hpp"

namespace vreg_b200 {

enum class PrecondKind { InvA, InvH0, TwoLevelInvH0 };      // precond.hpp:12
enum class HessianAdjoint { Transpose, SemiLagrangian };  // optim.hpp:11-14

inline std::string precond_name(PrecondKind k) {
  switch (k) {
    case PrecondKind::InvA: return "inva";
    case PrecondKind::InvH0: return "invh0";
    default: return "2linvh0";
  }
}

// beta floor of the H0 solves and the continuation's InvA threshold
// (precond.hpp:22-25)
inline constexpr Real h0_beta_floor = Real(5e-2);
inline constexpr Real inva_switch_beta = Real(5e-1);

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
  // B200 extension: PCG iterates in fp64 (x, r, p) around the fp32 operator
  // (SURVEY §7 hard part 3); off = fp32 vectors rounded every update
  bool pcg_fp64 = true;
  // B200 extension: regularisation order, 1 = H1 (the reference), 2 = H2
  // (beta/2 |Delta v|^2, symbol |k|^4)
  int reg_order = 1;

  bool fixed() const { return fixed_gn > 0; }

  void validate() const {
    auto need = [](bool ok, const char* what) {
      if (!ok) throw parameter_error(what);
    };
    need(beta_target > 0 && beta_start > 0, "beta must be > 0");
    need(eps_newton > 0 && eps_newton < 1, "eps_newton must lie in (0,1)");
    need(precond == PrecondKind::InvA || (eps_h0 > 0 && eps_h0 < 1),
         "eps_h0 must lie in (0,1)");
    need(gamma_div >= 0, "gamma_div must be >= 0");
    // 1 trilinear, 3 cubic Lagrange (reference); 4 cubic B-spline (B200)
    need(interp_degree == 1 || interp_degree == 3 || interp_degree == 4,
         "interp_degree must be 1, 3 or 4");
    need(nt >= 1, "nt must be >= 1");
    need(max_gn >= 1 && max_pcg >= 1, "iteration caps must be >= 1");
    need((fixed_gn > 0) == (fixed_pcg > 0), "fixed_gn and fixed_pcg go together");
    need(reg_order == 1 || reg_order == 2, "reg_order must be 1 (H1) or 2 (H2)");
  }
};

struct ObjectiveValue {
  Real total = 0, mismatch = 0, regularization = 0, div_penalty = 0;
};

struct GnIterRecord {
  Real objective = 0, mismatch = 0, g_norm = 0, g_rel = 0, eps_k = 0, alpha = 0;
  int pcg_iters = 0, line_search_trials = 0;
  Real beta_pc = 0;  // 0 when the spectral preconditioner is active
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

}  // namespace vreg_b200
