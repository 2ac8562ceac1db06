// CudaEngine: the B200 backend of the reference's engine concept
// (proj/include/vreg/engine.hpp:24-183), member for member, over the C ABI
// of include/vreg_cuda.h. Device fields (fp32, x1-slab per rank) have the
// value semantics of ScalarField / VectorField (copies are device copies),
// and the free functions the reference templates call on E::Field /
// E::VField (field.hpp:67-141) are provided by ADL.
//
// Header-only; link libvreg_b200.so.
#pragma once

#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "vreg_b200/types.hpp"
#include "vreg_cuda.h"

namespace vreg_b200 {

// Map a C-ABI status to the reference's exception types (types.hpp:19-41).
inline void check(int st) {
  if (st == VREG_OK) return;
  const std::string m = vreg_last_error();
  switch (st) {
    case VREG_EPARAM: throw parameter_error(m);
    case VREG_ENUMERICAL: throw numerical_error(m);
    case VREG_EIO: throw io_error(m);
    case VREG_EINPUT: throw input_error(m);
    case VREG_EDIM: throw dimension_error(m);
    case VREG_ECONFIG: throw config_error(m);
    default: throw std::runtime_error("vreg_b200 device error: " + m);
  }
}

// One GPU context (stream, FFT plans, NCCL communicator); shared by every
// field and engine (fine and coarse) of a rank.
class Device {
 public:
  explicit Device(int device = 0) { check(vreg_ctx_create(device, &ctx_)); }
  Device(int device, int rank, int nranks, const void* nccl_uid128) {
    check(vreg_ctx_create_dist(device, rank, nranks, nccl_uid128, &ctx_));
  }
  // adopt an existing context (not destroyed here)
  static std::shared_ptr<Device> adopt(vreg_ctx c) {
    auto d = std::shared_ptr<Device>(new Device(AdoptTag{}));
    d->ctx_ = c;
    d->owns_ = false;
    return d;
  }
  ~Device() {
    if (owns_ && ctx_) vreg_ctx_destroy(ctx_);
  }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  vreg_ctx ctx() const { return ctx_; }
  int rank() const {
    int r = 0, p = 1;
    vreg_ctx_rank(ctx_, &r, &p);
    return r;
  }
  int workers() const {
    int r = 0, p = 1;
    vreg_ctx_rank(ctx_, &r, &p);
    return p;
  }

 private:
  struct AdoptTag {};
  explicit Device(AdoptTag) {}
  vreg_ctx ctx_ = nullptr;
  bool owns_ = true;
};

inline vreg_grid to_vg(const Grid3& g) { return vreg_grid{g.n1, g.n2, g.n3, g.nt}; }

// Device field with NC components (1: scalar, 3: vector, SoA in one
// allocation) holding this rank's x1 slab.
template <int NC>
class DeviceField {
 public:
  // Host view `.v` of this rank's slab: the reference's templates touch
  // Field::v directly in one place (Flow::adjoint_source_factor,
  // transport.hpp:56-60). The first host access downloads the slab; the next
  // device access uploads it back if it was written. Device kernels never go
  // through it.
  class HostMirror {
   public:
    size_t size() const { return owner_->n_ * NC; }
    Real& operator[](size_t i) {
      owner_->pull();
      owner_->host_dirty_ = true;
      return host_[i];
    }

   private:
    friend class DeviceField;
    DeviceField* owner_ = nullptr;
    std::vector<Real> host_;
  };

  Grid3 grid;
  HostMirror v;

  DeviceField() { v.owner_ = this; }
  DeviceField(std::shared_ptr<Device> dev, const Grid3& g) : grid(g), dev_(std::move(dev)) {
    v.owner_ = this;
    const vreg_grid vg = to_vg(g);
    int n1l = 0, off = 0;
    check(vreg_slab(dev_->ctx(), &vg, &n1l, &off));
    n_ = size_t(n1l) * size_t(g.n2) * size_t(g.n3);
    void* p = nullptr;
    check(vreg_alloc(dev_->ctx(), NC * n_ * sizeof(float), &p));
    auto d = dev_;
    buf_ = std::shared_ptr<float>(static_cast<float*>(p), [d](float* q) { vreg_free(d->ctx(), q); });
    check(vreg_fill(dev_->ctx(), &vg, NC, buf_.get(), 0.0));  // ScalarField(g) zero-fills
  }
  DeviceField(const DeviceField& o) : grid(o.grid), dev_(o.dev_), n_(o.n_) {
    v.owner_ = this;
    if (!o.buf_) return;
    DeviceField t(o.dev_, o.grid);
    check(vreg_memcpy_d2d(dev_->ctx(), t.data(), o.data(), NC * n_ * sizeof(float)));
    buf_ = std::move(t.buf_);
  }
  DeviceField& operator=(const DeviceField& o) {
    if (this != &o) {
      DeviceField t(o);
      *this = std::move(t);
    }
    return *this;
  }
  DeviceField(DeviceField&& o) noexcept { *this = std::move(o); }
  DeviceField& operator=(DeviceField&& o) noexcept {
    grid = o.grid;
    dev_ = std::move(o.dev_);
    buf_ = std::move(o.buf_);
    n_ = o.n_;
    v.host_ = std::move(o.v.host_);
    host_valid_ = o.host_valid_;
    host_dirty_ = o.host_dirty_;
    v.owner_ = this;
    o.host_valid_ = o.host_dirty_ = false;
    return *this;
  }

  float* data() {
    push();
    host_valid_ = false;  // the device copy may change
    return buf_.get();
  }
  const float* data() const {
    const_cast<DeviceField*>(this)->push();
    return buf_.get();
  }
  float* comp(int c) { return data() + size_t(c) * n_; }
  const float* comp(int c) const { return data() + size_t(c) * n_; }
  size_t local_points() const { return n_; }
  index_t size() const { return index_t(n_); }
  bool empty() const { return !buf_; }
  vreg_ctx ctx() const { return dev_->ctx(); }
  vreg_grid vg() const { return to_vg(grid); }
  const std::shared_ptr<Device>& device() const { return dev_; }

  // host copies of the GLOBAL field (slab gather over ranks), double
  std::vector<double> to_host() const {
    const size_t N = size_t(grid.points());
    std::vector<float> tmp(NC * N);
    const vreg_grid g = vg();
    check(vreg_to_global(ctx(), &g, NC, data(), tmp.data()));
    return std::vector<double>(tmp.begin(), tmp.end());
  }
  void from_host(const double* global) {
    const size_t N = size_t(grid.points());
    std::vector<float> tmp(global, global + NC * N);
    const vreg_grid g = vg();
    check(vreg_from_global(ctx(), &g, NC, tmp.data(), data()));
  }

 private:
  void pull() {
    if (host_valid_) return;
    std::vector<float> tmp(NC * n_);
    check(vreg_memcpy_d2h(dev_->ctx(), tmp.data(), buf_.get(), NC * n_ * sizeof(float)));
    v.host_.assign(tmp.begin(), tmp.end());
    host_valid_ = true;
  }
  void push() {
    if (!host_dirty_) return;
    std::vector<float> tmp(v.host_.begin(), v.host_.end());
    check(vreg_memcpy_h2d(dev_->ctx(), buf_.get(), tmp.data(), NC * n_ * sizeof(float)));
    host_dirty_ = false;
  }

  std::shared_ptr<Device> dev_;
  std::shared_ptr<float> buf_;
  size_t n_ = 0;
  bool host_valid_ = false;
  bool host_dirty_ = false;
};

using DField = DeviceField<1>;
using DVField = DeviceField<3>;

// ---- free functions on device fields (field.hpp:67-188; ADL) ---------------

template <int NC>
inline void check_same_grid(const DeviceField<NC>& a, const DeviceField<NC>& b) {
  if (!a.grid.same_space(b.grid)) throw dimension_error("field grid mismatch");
}
template <int NC>
inline void fill(DeviceField<NC>& f, Real value) {
  const vreg_grid g = f.vg();
  check(vreg_fill(f.ctx(), &g, NC, f.data(), value));
}
template <int NC>
inline void axpy(Real a, const DeviceField<NC>& x, DeviceField<NC>& y) {
  check_same_grid(x, y);
  const vreg_grid g = x.vg();
  check(vreg_axpy(x.ctx(), &g, NC, a, x.data(), y.data()));
}
template <int NC>
inline void scale(DeviceField<NC>& f, Real a) {
  const vreg_grid g = f.vg();
  check(vreg_scale(f.ctx(), &g, NC, f.data(), a));
}
// out = a - b
template <int NC>
inline void sub(const DeviceField<NC>& a, const DeviceField<NC>& b, DeviceField<NC>& out) {
  check_same_grid(a, b);
  if (out.empty() || !out.grid.same_space(a.grid)) out = DeviceField<NC>(a.device(), a.grid);
  const vreg_grid g = a.vg();
  check(vreg_sub(a.ctx(), &g, NC, a.data(), b.data(), out.data()));
}
inline void hadamard(const DField& a, const DField& b, DField& out) {
  check_same_grid(a, b);
  if (out.empty() || !out.grid.same_space(a.grid)) out = DField(a.device(), a.grid);
  const vreg_grid g = a.vg();
  check(vreg_hadamard(a.ctx(), &g, a.data(), b.data(), out.data()));
}
inline void pointwise_dot(const DVField& v, const DVField& w, DField& out) {
  check_same_grid(v, w);
  if (out.empty() || !out.grid.same_space(v.grid)) out = DField(v.device(), v.grid);
  const vreg_grid g = v.vg();
  check(vreg_pointwise_dot(v.ctx(), &g, v.data(), w.data(), out.data()));
}
inline void axpy_scaled_vector(Real a, const DField& s, const DVField& w, DVField& out) {
  if (!s.grid.same_space(w.grid) || !w.grid.same_space(out.grid))
    throw dimension_error("field grid mismatch");
  const vreg_grid g = s.vg();
  check(vreg_axpy_scaled_vector(s.ctx(), &g, a, s.data(), w.data(), out.data()));
}
template <int NC>
inline Real inner(const DeviceField<NC>& a, const DeviceField<NC>& b) {
  check_same_grid(a, b);
  double r = 0;
  const vreg_grid g = a.vg();
  check(vreg_inner(a.ctx(), &g, NC, a.data(), b.data(), &r));
  return r;
}
template <int NC>
inline Real norm2(const DeviceField<NC>& a) {
  return std::sqrt(inner(a, a));
}
template <int NC>
inline Real max_abs(const DeviceField<NC>& a) {
  double r = 0;
  const vreg_grid g = a.vg();
  check(vreg_max_abs(a.ctx(), &g, NC, a.data(), &r));
  return r;
}

// ---- engine state (engine.hpp:14-19) ---------------------------------------

struct EngineState {
  std::shared_ptr<Device> dev;
  KernelCounters counters;
  KernelTimers kernel_timers;
  CommCounters comm;
};

class CudaEngine {
 public:
  using Field = DField;
  using VField = DVField;

  // Departure points of one step of the backward characteristics, stored as
  // grid-unit displacements (+ identity / ghost-width flags).
  struct Char {
    DVField dep;
    int flags = 0;
    bool identity = false;
  };

  CudaEngine() = default;
  CudaEngine(const Grid3& g, std::shared_ptr<EngineState> st, bool coarse = false)
      : grid_(g), state_(std::move(st)), coarse_(coarse) {}

  static CudaEngine create(const Grid3& g, int device = 0) {
    auto st = std::make_shared<EngineState>();
    st->dev = std::make_shared<Device>(device);
    return CudaEngine(g, st);
  }
  static CudaEngine create(const Grid3& g, std::shared_ptr<Device> dev) {
    auto st = std::make_shared<EngineState>();
    st->dev = std::move(dev);
    return CudaEngine(g, st);
  }

  const Grid3& grid() const { return grid_; }
  int workers() const { return state_->dev->workers(); }
  int rank() const { return state_->dev->rank(); }
  bool is_coarse() const { return coarse_; }
  KernelCounters& counters() { return state_->counters; }
  const KernelCounters& counters() const { return state_->counters; }
  KernelTimers& kernel_timers() {
    double t[8];
    check(vreg_ctx_timers(ctx(), t));
    KernelTimers& k = state_->kernel_timers;
    k.fft = t[0]; k.fd = t[1]; k.sl = t[2]; k.ghost_comm = t[3]; k.interp_comm = t[4];
    k.scatter_comm = t[5]; k.scatter_buffer = t[6]; k.transpose_comm = t[7];
    return k;
  }
  CommCounters& comm() {
    uint64_t c[9];
    check(vreg_ctx_comm(ctx(), c));
    CommCounters& m = state_->comm;
    m.ghost_fd_bytes = c[0]; m.ghost_interp_bytes = c[1]; m.scatter_points_bytes = c[2];
    m.interp_values_bytes = c[3]; m.fft_transpose_bytes = c[4]; m.spectral_gather_bytes = c[5];
    m.reduce_bytes = c[6]; m.p2p_messages = c[7]; m.alltoall_collectives = c[8];
    return m;
  }
  CudaEngine make_coarse() const { return CudaEngine(grid_.coarse(), state_, true); }
  vreg_ctx ctx() const { return state_->dev->ctx(); }
  const std::shared_ptr<Device>& device() const { return state_->dev; }
  vreg_grid vg() const { return to_vg(grid_); }

  // ---- field management ----
  Field make_field() const { return DField(state_->dev, grid_); }
  VField make_vfield() const { return DVField(state_->dev, grid_); }

  // Host <-> engine fields; any host type with `grid` and `v` (the
  // reference's ScalarField / VectorField, engine.hpp:63-66).
  template <class HostScalar>
  Field from_global(const HostScalar& f) const {
    Field out = make_field();
    out.from_host(f.v.data());
    return out;
  }
  // Engine fields -> host fields of the whole grid (slab gather over the
  // ranks), engine.hpp:64,66. HostScalar / HostVector are any types with a
  // Grid3 constructor and `v` / comp(c).v storage (the reference's
  // ScalarField / VectorField).
  template <class HostScalar>
  HostScalar to_global(const Field& f) const {
    HostScalar out(grid_);
    const std::vector<double> h = f.to_host();
    for (size_t i = 0; i < h.size(); ++i) out.v[i] = h[i];
    return out;
  }
  template <class HostVector>
  HostVector to_global_v(const VField& f) const {
    HostVector out(grid_);
    const std::vector<double> h = f.to_host();
    const size_t N = size_t(grid_.points());
    for (int c = 0; c < 3; ++c)
      for (size_t i = 0; i < N; ++i) out.comp(c).v[i] = h[size_t(c) * N + i];
    return out;
  }
#ifdef VREG_B200_WITH_REFERENCE
  vreg::ScalarField to_global(const Field& f) const { return to_global<vreg::ScalarField>(f); }
  vreg::VectorField to_global_v(const VField& f) const {
    return to_global_v<vreg::VectorField>(f);
  }
#endif
  template <class HostVector>
  VField from_global_v(const HostVector& v) const {
    const size_t N = size_t(grid_.points());
    std::vector<double> tmp(3 * N);
    for (int c = 0; c < 3; ++c) std::memcpy(tmp.data() + c * N, v.comp(c).v.data(), N * sizeof(double));
    VField out = make_vfield();
    out.from_host(tmp.data());
    return out;
  }

  // ---- pointwise / reductions ----
  Real inner(const Field& a, const Field& b) const { return vreg_b200::inner(a, b); }
  Real inner(const VField& a, const VField& b) const { return vreg_b200::inner(a, b); }
  Real norm2(const Field& f) const { return vreg_b200::norm2(f); }
  Real norm2(const VField& f) const { return vreg_b200::norm2(f); }
  Real max_abs_field(const Field& f) const { return vreg_b200::max_abs(f); }
  Real max_abs_vfield(const VField& f) const { return vreg_b200::max_abs(f); }

  // ---- kernels (counters as SerialEngine / FdOps / SpectralOps) ----
  VField fd_grad(const Field& f) const {
    state_->counters.fd_gradient++;
    VField out = make_vfield();
    const vreg_grid g = vg();
    check(vreg_fd_grad(ctx(), &g, f.data(), out.data()));
    return out;
  }
  Field fd_div(const VField& v) const {
    state_->counters.fd_divergence++;
    Field out = make_field();
    const vreg_grid g = vg();
    check(vreg_fd_div(ctx(), &g, v.data(), out.data()));
    return out;
  }
  VField regop(const VField& v, Real beta, bool unit_zero_mode) const {
    if (beta <= Real(0)) throw parameter_error("regularization beta must be > 0");
    count_fft(3, 3);
    VField out = make_vfield();
    const vreg_grid g = vg();
    check(vreg_regop(ctx(), &g, v.data(), beta, unit_zero_mode ? 1 : 0, out.data()));
    return out;
  }
  VField inv_regop(const VField& v, Real beta) const {
    if (beta <= Real(0)) throw parameter_error("regularization beta must be > 0");
    count_fft(3, 3);
    VField out = make_vfield();
    const vreg_grid g = vg();
    check(vreg_inv_regop(ctx(), &g, v.data(), beta, out.data()));
    return out;
  }
  Real seminorm(const VField& v) const {
    count_fft(3, 0);
    double r = 0;
    const vreg_grid g = vg();
    check(vreg_seminorm(ctx(), &g, v.data(), &r));
    return r;
  }
  VField leray(const VField& v) const {
    count_fft(3, 3);
    VField out = make_vfield();
    const vreg_grid g = vg();
    check(vreg_leray(ctx(), &g, v.data(), out.data()));
    return out;
  }
  Field restrict_to_coarse(const Field& f) const { return restrict_impl<1>(f); }
  VField restrict_to_coarse(const VField& v) const { return restrict_impl<3>(v); }
  Field prolong_to_fine(const Field& f) const { return prolong_impl<1>(f); }
  VField prolong_to_fine(const VField& v) const { return prolong_impl<3>(v); }
  Field high_pass_field(const Field& f) const { return high_pass_impl<1>(f); }
  VField high_pass_field(const VField& v) const { return high_pass_impl<3>(v); }

  // Fused fine-grid steps of the two-level preconditioner on one rank
  // (precond.hpp:143-160): begin returns (restrict(r), restrict(InvA r)) from
  // one forward transform, end returns prolong(s_c) + high_pass(InvA r) with
  // one inverse. Logical counters as InvA + two restrictions / prolongation
  // + high pass, so the cost model is unchanged.
  bool two_level_fused() const {
    const char* e = std::getenv("VREG_TWO_LEVEL_UNFUSED");
    return workers() == 1 && !coarse_ && !(e && e[0] == '1');
  }
  std::pair<VField, VField> two_level_begin(const VField& r, Real beta_pc) const {
    if (beta_pc <= Real(0)) throw parameter_error("regularization beta must be > 0");
    count_fft(3, 3);
    auto& c = state_->counters;
    c.fft_forward += 6;
    c.fft_inverse_coarse += 6;
    VField rc(state_->dev, grid_.coarse()), sc(state_->dev, grid_.coarse());
    const vreg_grid g = vg();
    check(vreg_two_level_begin(ctx(), &g, r.data(), beta_pc, rc.data(), sc.data()));
    return {std::move(rc), std::move(sc)};
  }
  VField two_level_end(const VField& s_c) const {
    auto& c = state_->counters;
    c.fft_forward_coarse += 3;
    c.fft_inverse += 3;
    count_fft(3, 3);
    VField out = make_vfield();
    const vreg_grid g = vg();
    check(vreg_two_level_end(ctx(), &g, s_c.data(), out.data()));
    return out;
  }

  // ---- semi-Lagrangian support (engine.hpp:108-169) ----
  Char make_characteristics(const VField& v, int degree) const {
    state_->counters.characteristics++;
    Char ch;
    ch.dep = make_vfield();
    const vreg_grid g = vg();
    check(vreg_characteristics(ctx(), &g, v.data(), degree, ch.dep.data(), &ch.flags));
    ch.identity = (ch.flags & 1) != 0;
    if (ch.identity)
      state_->counters.characteristics_identity++;
    else
      state_->counters.ip_eval += 3;  // the RK2 midpoint interpolations of v
    return ch;
  }
  Field interp_at(const Field& f, const Char& ch, int degree) const {
    state_->counters.ip_eval++;
    Field out = make_field();
    const vreg_grid g = vg();
    check(vreg_interp(ctx(), &g, f.data(), ch.dep.data(), ch.flags, degree, out.data()));
    return out;
  }
  Field scatter_at(const Field& z, const Char& ch, int degree) const {
    state_->counters.ip_scatter++;
    Field out = make_field();
    const vreg_grid g = vg();
    check(vreg_scatter(ctx(), &g, z.data(), ch.dep.data(), ch.flags, degree, out.data()));
    return out;
  }

 private:
  void count_fft(int fwd, int inv) const {
    auto& c = state_->counters;
    (coarse_ ? c.fft_forward_coarse : c.fft_forward) += std::uint64_t(fwd);
    (coarse_ ? c.fft_inverse_coarse : c.fft_inverse) += std::uint64_t(inv);
  }
  template <int NC>
  DeviceField<NC> restrict_impl(const DeviceField<NC>& f) const {
    auto& c = state_->counters;
    c.fft_forward += NC;         // fine forward (spectral.cpp:246)
    c.fft_inverse_coarse += NC;  // coarse inverse (spectral.cpp:249-250)
    DeviceField<NC> out(state_->dev, f.grid.coarse());
    const vreg_grid g = f.vg();
    check(vreg_restrict(ctx(), &g, NC, f.data(), out.data()));
    return out;
  }
  template <int NC>
  DeviceField<NC> prolong_impl(const DeviceField<NC>& fc) const {
    auto& c = state_->counters;
    c.fft_forward_coarse += NC;  // spectral.cpp:255-256
    c.fft_inverse += NC;         // spectral.cpp:259
    DeviceField<NC> out(state_->dev, grid_);
    const vreg_grid g = vg();
    check(vreg_prolong(ctx(), &g, NC, fc.data(), out.data()));
    return out;
  }
  template <int NC>
  DeviceField<NC> high_pass_impl(const DeviceField<NC>& f) const {
    count_fft(NC, NC);
    DeviceField<NC> out(state_->dev, f.grid);
    const vreg_grid g = f.vg();
    check(vreg_high_pass(ctx(), &g, NC, f.data(), out.data()));
    return out;
  }

  Grid3 grid_;
  std::shared_ptr<EngineState> state_;
  bool coarse_ = false;
};

}  // namespace vreg_b200
