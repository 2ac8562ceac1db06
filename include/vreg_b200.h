/* vreg_b200.h -- solver-level C ABI of libvreg_b200.so: the Gauss-Newton
 * hot path behind a handle, for FFI callers (Python ctypes, bench, tests).
 *
 * Each entry point is the device counterpart of one reference call path
 * (paths under /root/reference/proj):
 *   vreg_solver_linearize  -> gauss_newton_level's setup: Flow + StateCache,
 *                             evaluate_objective_with / evaluate_gradient_with
 *                             (include/vreg/optim.hpp:155-168, 68-111)
 *   vreg_solver_matvec     -> detail::hessian_matvec_with (optim.hpp:115-137)
 *   vreg_solver_precond    -> Preconditioner<E>::refresh + apply
 *                             (include/vreg/precond.hpp:80-162)
 *   vreg_solver_register   -> register_images (optim.hpp:308-347)
 * Field pointers are DEVICE pointers (this rank's x1 slab, fp32, vector
 * fields as 3 consecutive components) unless the name says _host. Status
 * codes as in vreg_cuda.h.
 */
#ifndef VREG_B200_H
#define VREG_B200_H
#include <stdint.h>

#include "vreg_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* RegistrationConfig (optim.hpp:16-37); precond 0 InvA, 1 InvH0,
 * 2 TwoLevelInvH0; hessian_adjoint 0 Transpose, 1 SemiLagrangian. */
typedef struct {
  double beta_target, beta_start;
  int continuation;
  double gamma_div;
  int project_divfree;
  double eps_newton, eps_h0;
  int max_gn, max_pcg;
  int precond;
  int interp_degree;
  int cache_state_gradient;
  int fixed_gn, fixed_pcg;
  int hessian_adjoint;
  int nt;
  double armijo_c, armijo_shrink;
  int armijo_max_trials, h0_inner_cap;
  int pcg_fp64;  /* B200: PCG iterates in fp64 around the fp32 operator (default 1) */
  int reg_order; /* B200: 1 = H1 (reference, default), 2 = H2 (symbol |k|^4) */
} vreg_config;

typedef struct vreg_solver_s* vreg_solver;

void vreg_config_default(vreg_config* cfg);
int vreg_solver_create(vreg_ctx ctx, const vreg_grid* g, const vreg_config* cfg, vreg_solver* out);
int vreg_solver_destroy(vreg_solver s);
/* template m0 / reference m1 (device, local slab) */
int vreg_solver_set_images(vreg_solver s, const float* m0, const float* m1);
/* SYN pair built on device: m0 = syn_template, m1 = state of syn_velocity
 * at t = 1 (proj/src/syn.cpp:46-49) */
int vreg_solver_syn_images(vreg_solver s);
int vreg_solver_images(vreg_solver s, float* m0, float* m1);
/* linearisation point v (device vector field) at regularisation beta */
int vreg_solver_linearize(vreg_solver s, const float* v3, double beta);
int vreg_solver_objective(vreg_solver s, double J4[4]);
int vreg_solver_gradient(vreg_solver s, float* g3);
int vreg_solver_matvec(vreg_solver s, const float* vt3, float* out3);
/* the same matvec on HOST buffers (H2D + matvec + D2H) */
int vreg_solver_matvec_host(vreg_solver s, const float* vt3_host, float* out3_host);

/* Pipelined host-buffer matvec: enqueue H2D of vt3_host, the fused matvec
 * and D2H into out3_host, and return. Two device slots and two copy streams
 * (H2D, D2H) let call k's upload, call k-1's matvec and call k-2's download
 * overlap. Both host buffers must be pinned and stay untouched until
 * vreg_solver_wait returns. Same result as vreg_solver_matvec_host. */
int vreg_solver_matvec_host_async(vreg_solver s, const float* vt3_host, float* out3_host);
/* Block until every enqueued host-buffer matvec has landed in host memory. */
int vreg_solver_wait(vreg_solver s);
/* stats4: inva applications, h0 applications, inner iterations, capped */
int vreg_solver_precond(vreg_solver s, int kind, const float* r3, double eps_k, float* out3,
                        uint64_t stats4[4]);
/* full solve from v = 0; rep16: initial_mismatch, final_mismatch, mism_rel,
 * final_g_rel, total_gn, total_pcg, flagged, phases pc/obj/grad/hess/total,
 * kernels fft/fd/sl, levels. counters21 in KernelCounters order. */
int vreg_solver_register(vreg_solver s, float* v_out3, double rep16[16], uint64_t counters21[21]);
/* Text of the last vreg_solver_register report (include/vreg_b200/report.hpp):
 * which 0 = render_report (deterministic, no timings), 1 = render_timings,
 * 2 = render_residuals_csv (reference report.hpp:79-84). Copies at most cap-1
 * bytes + NUL into buf; *len = full length. */
int vreg_solver_report_text(vreg_solver s, int which, char* buf, size_t cap, size_t* len);

/* VolumeFile "VRG1", host buffers: kind 0 = f32, 1 = f64;
 * ncomp 1 or 3; data = components concatenated, row-major. Bad magic or a
 * payload length that disagrees with the header -> VREG_EIO. */
int vreg_volume_save(const char* path, int n1, int n2, int n3, int kind, int ncomp,
                     const void* data);
int vreg_volume_header(const char* path, int hdr5[5]); /* n1, n2, n3, kind, ncomp */
int vreg_volume_load(const char* path, void* data, size_t cap_bytes);

int vreg_solver_counters(vreg_solver s, uint64_t counters21[21]);
int vreg_solver_reset_counters(vreg_solver s);

#ifdef __cplusplus
}
#endif
#endif
