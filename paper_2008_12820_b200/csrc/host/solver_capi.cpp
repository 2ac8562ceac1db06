// Solver-level C ABI (include/vreg_b200.h) over the device-resident
// Gauss-Newton-Krylov layer (csrc/host/gnk.hpp). Exceptions never cross the
// ABI: they map back to the status codes of vreg_cuda.h.
#include <cuda_runtime.h>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>

#include "vreg_b200.h"
#include "gnk.hpp"
#include "vreg_b200/report.hpp"

namespace vb {
void set_last_error(const std::string& m);
}

using namespace vreg_b200;

struct vreg_solver_s {
  std::shared_ptr<Device> dev;
  CudaEngine eng;
  RegistrationConfig cfg;
  DField m0, m1;
  std::unique_ptr<Transport> lin;
  ObjectiveValue J;
  std::optional<DVField> grad;
  Real beta = 0;
  std::unique_ptr<DevicePrecond> prec;
  std::optional<DVField> io_in, io_out;  // device staging of the host-buffer matvec
  std::optional<SolverReport> last;      // of the last vreg_solver_register
  // pipelined host-buffer matvec: two slots, upload / download streams
  std::optional<DVField> pin[2], pout[2];
  cudaStream_t up = nullptr, down = nullptr;
  cudaEvent_t ev_up[2] = {}, ev_mv[2] = {}, ev_down[2] = {};
  bool slot_used[2] = {false, false};
  std::uint64_t pk = 0;
  ~vreg_solver_s() {
    if (up) {
      cudaStreamSynchronize(up);
      cudaStreamSynchronize(down);
      cudaStreamDestroy(up);
      cudaStreamDestroy(down);
      for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(ev_up[i]);
        cudaEventDestroy(ev_mv[i]);
        cudaEventDestroy(ev_down[i]);
      }
    }
  }
};

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return VREG_OK;
  } catch (const parameter_error& e) {
    vb::set_last_error(e.what());
    return VREG_EPARAM;
  } catch (const numerical_error& e) {
    vb::set_last_error(e.what());
    return VREG_ENUMERICAL;
  } catch (const io_error& e) {
    vb::set_last_error(e.what());
    return VREG_EIO;
  } catch (const input_error& e) {
    vb::set_last_error(e.what());
    return VREG_EINPUT;
  } catch (const dimension_error& e) {
    vb::set_last_error(e.what());
    return VREG_EDIM;
  } catch (const config_error& e) {
    vb::set_last_error(e.what());
    return VREG_ECONFIG;
  } catch (const std::exception& e) {
    vb::set_last_error(e.what());
    return VREG_ECUDA;
  }
}

RegistrationConfig from_c(const vreg_config* c) {
  RegistrationConfig r;
  if (!c) return r;
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
  r.pcg_fp64 = c->pcg_fp64 != 0;
  r.reg_order = c->reg_order;
  return r;
}

void dump_counters(const KernelCounters& k, uint64_t* o) {
  const uint64_t v[] = {k.fft_forward, k.fft_inverse, k.fft_forward_coarse, k.fft_inverse_coarse,
                        k.fd_gradient, k.fd_divergence, k.ip_eval, k.ip_scatter,
                        k.characteristics, k.characteristics_identity, k.sl_state, k.sl_adjoint,
                        k.sl_inc_state, k.sl_inc_adjoint, k.pc_inva_apply, k.pc_h0_apply,
                        k.pc_h0_inner_iters, k.pc_h0_inner_solves, k.pc_refresh,
                        k.h0_inner_work_fine, k.h0_inner_work_coarse};
  std::memcpy(o, v, sizeof(v));
}

void require_lin(const vreg_solver_s* s) {
  if (!s->lin) throw config_error("solver not linearised (call vreg_solver_linearize)");
}

// The context's regularisation order follows the solver's config for the
// duration of a call (the context may serve several solvers).
struct OrderScope {
  vreg_ctx ctx;
  OrderScope(const vreg_solver_s* s) : ctx(s->eng.ctx()) { check(vreg_ctx_set_reg_order(ctx, s->cfg.reg_order)); }
  ~OrderScope() { vreg_ctx_set_reg_order(ctx, 1); }
};

}  // namespace

extern "C" {

void vreg_config_default(vreg_config* c) {
  RegistrationConfig r;
  c->beta_target = r.beta_target;
  c->beta_start = r.beta_start;
  c->continuation = r.continuation;
  c->gamma_div = r.gamma_div;
  c->project_divfree = r.project_divfree;
  c->eps_newton = r.eps_newton;
  c->eps_h0 = r.eps_h0;
  c->max_gn = r.max_gn;
  c->max_pcg = r.max_pcg;
  c->precond = int(r.precond);
  c->interp_degree = r.interp_degree;
  c->cache_state_gradient = r.cache_state_gradient;
  c->fixed_gn = r.fixed_gn;
  c->fixed_pcg = r.fixed_pcg;
  c->hessian_adjoint = int(r.hessian_adjoint);
  c->nt = r.nt;
  c->armijo_c = r.armijo_c;
  c->armijo_shrink = r.armijo_shrink;
  c->armijo_max_trials = r.armijo_max_trials;
  c->h0_inner_cap = r.h0_inner_cap;
  c->pcg_fp64 = r.pcg_fp64;
  c->reg_order = r.reg_order;
}

int vreg_solver_create(vreg_ctx ctx, const vreg_grid* g, const vreg_config* cfg,
                       vreg_solver* out) {
  return guarded([&] {
    if (!ctx || !g || !out) throw parameter_error("null argument");
    auto s = std::make_unique<vreg_solver_s>();
    s->cfg = from_c(cfg);
    s->cfg.validate();
    s->dev = Device::adopt(ctx);
    Grid3 grid = Grid3::make(g->n1, g->n2, g->n3, s->cfg.nt);
    s->eng = CudaEngine::create(grid, s->dev);
    s->m0 = s->eng.make_field();
    s->m1 = s->eng.make_field();
    // working set of a solve, twice the paper's estimate (74 + nt) N mu0 / p
    // (SPEC.md:384-386), reserved in the pool up front
    const double n_local = double(g->n1) * g->n2 * g->n3 / double(s->eng.workers());
    check(vreg_ctx_reserve(ctx, size_t(2.0 * (74 + s->cfg.nt) * n_local * sizeof(float))));
    *out = s.release();
  });
}

int vreg_solver_destroy(vreg_solver s) {
  return guarded([&] { delete s; });
}

int vreg_solver_set_images(vreg_solver s, const float* m0, const float* m1) {
  return guarded([&] {
    const size_t bytes = s->m0.local_points() * sizeof(float);
    check(vreg_memcpy_d2d(s->eng.ctx(), s->m0.data(), m0, bytes));
    check(vreg_memcpy_d2d(s->eng.ctx(), s->m1.data(), m1, bytes));
  });
}

int vreg_solver_syn_images(vreg_solver s) {
  return guarded([&] {
    CudaEngine& e = s->eng;
    const vreg_grid g = e.vg();
    check(vreg_syn_template(e.ctx(), &g, s->m0.data()));
    DVField v = e.make_vfield();
    check(vreg_syn_velocity(e.ctx(), &g, v.data()));
    // syn_reference: solve_state(syn_velocity, syn_template)(., 1) on a
    // private engine state so the solver's counters stay clean
    CudaEngine aux = CudaEngine::create(e.grid(), s->dev);
    Transport tr(aux, v, s->cfg.interp_degree);
    tr.solve_state(s->m0);
    const size_t N = s->m0.local_points();
    check(vreg_memcpy_d2d(e.ctx(), s->m1.data(), tr.state(e.grid().nt), N * sizeof(float)));
  });
}

int vreg_solver_images(vreg_solver s, float* m0, float* m1) {
  return guarded([&] {
    const size_t bytes = s->m0.local_points() * sizeof(float);
    if (m0) check(vreg_memcpy_d2d(s->eng.ctx(), m0, s->m0.data(), bytes));
    if (m1) check(vreg_memcpy_d2d(s->eng.ctx(), m1, s->m1.data(), bytes));
  });
}

int vreg_solver_linearize(vreg_solver s, const float* v3, double beta) {
  return guarded([&] {
    OrderScope order(s);
    if (beta <= 0) throw parameter_error("beta must be > 0");
    CudaEngine& e = s->eng;
    DVField v = e.make_vfield();
    check(vreg_memcpy_d2d(e.ctx(), v.data(), v3, 3 * v.local_points() * sizeof(float)));
    s->beta = beta;
    s->lin = std::make_unique<Transport>(e, std::move(v), s->cfg.interp_degree);
    s->J = objective(e, *s->lin, s->m0, s->m1, beta, s->cfg);
    s->grad = gradient(e, *s->lin, s->m1, beta, s->cfg);
    s->lin->gradients();  // state-gradient cache for the matvecs
    s->prec.reset();
  });
}

int vreg_solver_objective(vreg_solver s, double J4[4]) {
  return guarded([&] {
    require_lin(s);
    J4[0] = s->J.total;
    J4[1] = s->J.mismatch;
    J4[2] = s->J.regularization;
    J4[3] = s->J.div_penalty;
  });
}

int vreg_solver_gradient(vreg_solver s, float* g3) {
  return guarded([&] {
    require_lin(s);
    check(vreg_memcpy_d2d(s->eng.ctx(), g3, s->grad->data(),
                          3 * s->grad->local_points() * sizeof(float)));
  });
}

namespace {

// The hot path proper: Transpose adjoint, no div penalty -> the fused device
// pipeline straight on the caller's buffers (no field copies).
bool direct_matvec(vreg_solver s, const float* vt3, float* out3) {
  const RegistrationConfig& c = s->cfg;
  if (c.hessian_adjoint != HessianAdjoint::Transpose || c.gamma_div > 0) return false;
  CudaEngine& e = s->eng;
  const auto& ch = s->lin->forward();
  const float* gr = s->lin->gradients();
  count_matvecs(e.counters(), c, e.grid().nt, 1);
  const vreg_grid g = e.vg();
  check(vreg_gn_matvec(e.ctx(), &g, ch.dep.data(), ch.flags, s->lin->degree(), gr, s->beta, vt3,
                       out3));
  return true;
}

}  // namespace

int vreg_solver_matvec(vreg_solver s, const float* vt3, float* out3) {
  return guarded([&] {
    OrderScope order(s);
    require_lin(s);
    if (direct_matvec(s, vt3, out3)) return;
    CudaEngine& e = s->eng;
    count_matvecs(e.counters(), s->cfg, e.grid().nt, 1);
    matvec_into(e, *s->lin, s->beta, s->cfg, vt3, out3);
  });
}

int vreg_solver_matvec_host(vreg_solver s, const float* vt3_host, float* out3_host) {
  return guarded([&] {
    OrderScope order(s);
    require_lin(s);
    CudaEngine& e = s->eng;
    if (!s->io_in) {
      s->io_in.emplace(e.make_vfield());
      s->io_out.emplace(e.make_vfield());
    }
    const size_t bytes = 3 * s->io_in->local_points() * sizeof(float);
    check(vreg_memcpy_h2d(e.ctx(), s->io_in->data(), vt3_host, bytes));
    if (!direct_matvec(s, s->io_in->data(), s->io_out->data())) {
      count_matvecs(e.counters(), s->cfg, e.grid().nt, 1);
      matvec_into(e, *s->lin, s->beta, s->cfg, s->io_in->data(), s->io_out->data());
    }
    check(vreg_memcpy_d2h(e.ctx(), out3_host, s->io_out->data(), bytes));
  });
}

namespace {
void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}
}  // namespace

int vreg_solver_matvec_host_async(vreg_solver s, const float* vt3_host, float* out3_host) {
  return guarded([&] {
    OrderScope order(s);
    require_lin(s);
    CudaEngine& e = s->eng;
    void* mv = nullptr;
    check(vreg_ctx_get_stream(e.ctx(), &mv));
    cudaStream_t st = static_cast<cudaStream_t>(mv);
    if (!s->up) {
      cuda_check(cudaStreamCreateWithFlags(&s->up, cudaStreamNonBlocking));
      cuda_check(cudaStreamCreateWithFlags(&s->down, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        cuda_check(cudaEventCreateWithFlags(&s->ev_up[i], cudaEventDisableTiming));
        cuda_check(cudaEventCreateWithFlags(&s->ev_mv[i], cudaEventDisableTiming));
        cuda_check(cudaEventCreateWithFlags(&s->ev_down[i], cudaEventDisableTiming));
        s->pin[i].emplace(e.make_vfield());
        s->pout[i].emplace(e.make_vfield());
      }
      cuda_check(cudaStreamSynchronize(st));  // slots allocated on the matvec stream
    }
    const int k = int(s->pk & 1);
    const size_t bytes = 3 * s->pin[k]->local_points() * sizeof(float);
    // upload into slot k once call k-2's matvec has consumed it
    if (s->slot_used[k]) cuda_check(cudaStreamWaitEvent(s->up, s->ev_mv[k], 0));
    cuda_check(cudaMemcpyAsync(s->pin[k]->data(), vt3_host, bytes, cudaMemcpyHostToDevice, s->up));
    cuda_check(cudaEventRecord(s->ev_up[k], s->up));
    // matvec once the upload landed and call k-2's download freed the output
    cuda_check(cudaStreamWaitEvent(st, s->ev_up[k], 0));
    if (s->slot_used[k]) cuda_check(cudaStreamWaitEvent(st, s->ev_down[k], 0));
    if (!direct_matvec(s, s->pin[k]->data(), s->pout[k]->data())) {
      count_matvecs(e.counters(), s->cfg, e.grid().nt, 1);
      matvec_into(e, *s->lin, s->beta, s->cfg, s->pin[k]->data(), s->pout[k]->data());
    }
    cuda_check(cudaEventRecord(s->ev_mv[k], st));
    cuda_check(cudaStreamWaitEvent(s->down, s->ev_mv[k], 0));
    cuda_check(cudaMemcpyAsync(out3_host, s->pout[k]->data(), bytes, cudaMemcpyDeviceToHost,
                               s->down));
    cuda_check(cudaEventRecord(s->ev_down[k], s->down));
    s->slot_used[k] = true;
    ++s->pk;
  });
}

int vreg_solver_wait(vreg_solver s) {
  return guarded([&] {
    if (!s->up) return;
    cuda_check(cudaStreamSynchronize(s->up));
    cuda_check(cudaStreamSynchronize(s->down));
  });
}

int vreg_solver_precond(vreg_solver s, int kind, const float* r3, double eps_k, float* out3,
                        uint64_t stats4[4]) {
  return guarded([&] {
    OrderScope order(s);
    require_lin(s);
    CudaEngine& e = s->eng;
    if (kind < 0 || kind > 2) throw parameter_error("preconditioner kind must be 0, 1 or 2");
    if (!s->prec || int(s->prec->kind()) != kind) {
      s->prec = std::make_unique<DevicePrecond>(e, PrecondKind(kind), s->beta, s->cfg.eps_h0,
                                                s->cfg.h0_inner_cap);
      s->prec->refresh(s->lin->state_field(e.grid().nt));
    }
    s->prec->take_device();
    s->prec->apply_once(r3, out3, eps_k);
    const auto inner = s->prec->take_device();
    PrecondTally t;
    s->prec->count(1, inner.first, t);
    if (stats4) {
      stats4[0] = t.inva;
      stats4[1] = t.h0;
      stats4[2] = t.inner;
      stats4[3] = inner.second ? 1 : 0;
    }
  });
}

int vreg_solver_register(vreg_solver s, float* v_out3, double rep16[16], uint64_t counters21[21]) {
  return guarded([&] {
    OrderScope order(s);
    CudaEngine& e = s->eng;
    DVField v;
    SolverReport r = Registration(e, s->m0, s->m1, s->cfg).run(&v);
    s->last = r;
    if (v_out3)
      check(vreg_memcpy_d2d(e.ctx(), v_out3, v.data(), 3 * v.local_points() * sizeof(float)));
    if (rep16) {
      rep16[0] = r.initial_mismatch;
      rep16[1] = r.final_mismatch;
      rep16[2] = r.mism_rel;
      rep16[3] = r.final_g_rel;
      rep16[4] = r.total_gn();
      rep16[5] = r.total_pcg();
      rep16[6] = r.flagged ? 1 : 0;
      rep16[7] = r.phases.pc;
      rep16[8] = r.phases.obj;
      rep16[9] = r.phases.grad;
      rep16[10] = r.phases.hess;
      rep16[11] = r.phases.total;
      rep16[12] = r.kernels.fft;
      rep16[13] = r.kernels.fd;
      rep16[14] = r.kernels.sl;
      rep16[15] = double(r.levels.size());
    }
    if (counters21) dump_counters(r.counters, counters21);
  });
}

int vreg_solver_report_text(vreg_solver s, int which, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    if (!s->last) throw config_error("no registration report yet (call vreg_solver_register)");
    const std::string t = which == 0   ? render_report(*s->last)
                          : which == 1 ? render_timings(*s->last)
                          : which == 2 ? render_residuals_csv(*s->last)
                                       : throw parameter_error("report kind must be 0, 1 or 2");
    if (len) *len = t.size();
    if (buf && cap) {
      const size_t n = t.size() < cap - 1 ? t.size() : cap - 1;
      std::memcpy(buf, t.data(), n);
      buf[n] = 0;
    }
  });
}

int vreg_volume_save(const char* path, int n1, int n2, int n3, int kind, int ncomp,
                     const void* data) {
  return guarded([&] {
    Volume v;
    v.n1 = n1;
    v.n2 = n2;
    v.n3 = n3;
    v.kind = kind;
    v.ncomp = ncomp;
    if ((kind != 0 && kind != 1) || (ncomp != 1 && ncomp != 3) || n1 <= 0 || n2 <= 0 || n3 <= 0)
      throw parameter_error("volume: bad header fields");
    const auto* p = static_cast<const unsigned char*>(data);
    v.payload.assign(p, p + v.expected_bytes());
    save_volume(path, v);
  });
}

int vreg_volume_header(const char* path, int hdr5[5]) {
  return guarded([&] {
    const Volume v = load_volume(path);
    hdr5[0] = v.n1;
    hdr5[1] = v.n2;
    hdr5[2] = v.n3;
    hdr5[3] = v.kind;
    hdr5[4] = v.ncomp;
  });
}

int vreg_volume_load(const char* path, void* data, size_t cap_bytes) {
  return guarded([&] {
    const Volume v = load_volume(path);
    if (cap_bytes < v.payload.size()) throw parameter_error("volume: destination too small");
    std::memcpy(data, v.payload.data(), v.payload.size());
  });
}

int vreg_solver_counters(vreg_solver s, uint64_t counters21[21]) {
  return guarded([&] { dump_counters(s->eng.counters(), counters21); });
}

int vreg_solver_reset_counters(vreg_solver s) {
  return guarded([&] { s->eng.counters() = KernelCounters{}; });
}

}  // extern "C"
