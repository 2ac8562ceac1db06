// Scalar types, grid, error taxonomy and instrumentation records of the
// B200 backend.
//
// Two modes:
//  * standalone (default): definitions with the same names, members and
//    semantics as the reference's proj/include/vreg/{types,grid,counters}.hpp;
//  * drop-in (define VREG_B200_WITH_REFERENCE and put the reference's
//    proj/include on the include path): the reference's own types are used,
//    so CudaEngine plugs into vreg::register_images & co. unchanged.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>

#ifdef VREG_B200_WITH_REFERENCE
#include "vreg/counters.hpp"
#include "vreg/grid.hpp"
#include "vreg/types.hpp"
namespace vreg_b200 {
using vreg::CommCounters;
using vreg::config_error;
using vreg::dimension_error;
using vreg::Grid3;
using vreg::index_t;
using vreg::input_error;
using vreg::io_error;
using vreg::KernelCounters;
using vreg::KernelTimers;
using vreg::numerical_error;
using vreg::parameter_error;
using vreg::PhaseTimers;
using vreg::Real;
using vreg::ScopedTimer;
inline constexpr double two_pi = vreg::two_pi;
}  // namespace vreg_b200
#else
namespace vreg_b200 {

using Real = double;  // host scalars (beta, inner products); fields are fp32 on device
using index_t = std::int64_t;
inline constexpr double two_pi = 6.283185307179586476925286766559;

// Error types (types.hpp:17-41): config/dimension/parameter -> exit 2,
// numerical -> 3, io -> 4.
struct dimension_error : std::runtime_error {
  explicit dimension_error(const std::string& m) : std::runtime_error(m) {}
};
struct parameter_error : std::runtime_error {
  explicit parameter_error(const std::string& m) : std::runtime_error(m) {}
};
struct config_error : std::runtime_error {
  explicit config_error(const std::string& m) : std::runtime_error(m) {}
};
struct numerical_error : std::runtime_error {
  explicit numerical_error(const std::string& m) : std::runtime_error(m) {}
};
struct io_error : std::runtime_error {
  explicit io_error(const std::string& m) : std::runtime_error(m) {}
};
struct input_error : std::runtime_error {
  explicit input_error(const std::string& m) : std::runtime_error(m) {}
};

// Periodic grid on [0, 2pi)^3, nt time steps on [0, 1] (grid.hpp:13-64).
struct Grid3 {
  int n1 = 0, n2 = 0, n3 = 0;
  int nt = 1;

  static Grid3 make(int n1, int n2, int n3, int nt = 1) {
    if (n1 < 8 || n2 < 8 || n3 < 8) throw dimension_error("grid sizes must be >= 8");
    if (n1 % 2 || n2 % 2 || n3 % 2) throw dimension_error("grid sizes must be even");
    if (nt < 1) throw parameter_error("nt must be >= 1");
    return Grid3{n1, n2, n3, nt};
  }
  static Grid3 cube(int n, int nt = 1) { return make(n, n, n, nt); }
  int n(int axis) const { return axis == 0 ? n1 : (axis == 1 ? n2 : n3); }
  Real h(int axis) const { return Real(two_pi) / Real(n(axis)); }
  Real dt() const { return Real(1) / Real(nt); }
  index_t points() const { return index_t(n1) * index_t(n2) * index_t(n3); }
  Real cell_volume() const { return h(0) * h(1) * h(2); }
  index_t index(int i, int j, int k) const { return (index_t(i) * n2 + j) * n3 + k; }
  Grid3 coarse() const {
    if (n1 % 2 || n2 % 2 || n3 % 2) throw dimension_error("grid not refinable");
    if (n1 < 8 || n2 < 8 || n3 < 8) throw dimension_error("grid too small to restrict");
    return Grid3{n1 / 2, n2 / 2, n3 / 2, nt};
  }
  bool same_space(const Grid3& o) const { return n1 == o.n1 && n2 == o.n2 && n3 == o.n3; }
  bool operator==(const Grid3& o) const { return same_space(o) && nt == o.nt; }
};

// Logical per-operation counters, independent of the GPU count
// (counters.hpp:11-45); the engine increments them exactly like
// SerialEngine so the Eq. 8 cost model still matches.
struct KernelCounters {
  std::uint64_t fft_forward = 0, fft_inverse = 0, fft_forward_coarse = 0, fft_inverse_coarse = 0;
  std::uint64_t fd_gradient = 0, fd_divergence = 0;
  std::uint64_t ip_eval = 0, ip_scatter = 0;
  std::uint64_t characteristics = 0, characteristics_identity = 0;
  std::uint64_t sl_state = 0, sl_adjoint = 0, sl_inc_state = 0, sl_inc_adjoint = 0;
  std::uint64_t pc_inva_apply = 0, pc_h0_apply = 0, pc_h0_inner_iters = 0, pc_h0_inner_solves = 0,
                pc_refresh = 0;
  std::uint64_t h0_inner_work_fine = 0, h0_inner_work_coarse = 0;
  std::uint64_t fft(bool coarse) const {
    return coarse ? fft_forward_coarse + fft_inverse_coarse : fft_forward + fft_inverse;
  }
};

// Bytes moved between GPUs per category (counters.hpp:49-59).
struct CommCounters {
  std::uint64_t ghost_fd_bytes = 0, ghost_interp_bytes = 0, scatter_points_bytes = 0,
                interp_values_bytes = 0, fft_transpose_bytes = 0, spectral_gather_bytes = 0,
                reduce_bytes = 0, p2p_messages = 0, alltoall_collectives = 0;
};

struct PhaseTimers {
  double pc = 0, obj = 0, grad = 0, hess = 0, total = 0;
};

// Kernel timers (counters.hpp:69-78), measured on the device with CUDA events.
struct KernelTimers {
  double fft = 0, fd = 0, sl = 0, ghost_comm = 0, interp_comm = 0, scatter_comm = 0,
         scatter_buffer = 0, transpose_comm = 0;
};

class ScopedTimer {
 public:
  explicit ScopedTimer(double* acc) : acc_(acc), start_(std::chrono::steady_clock::now()) {}
  ~ScopedTimer() {
    if (acc_)
      *acc_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - start_).count();
  }
  ScopedTimer(const ScopedTimer&) = delete;
  ScopedTimer& operator=(const ScopedTimer&) = delete;

 private:
  double* acc_;
  std::chrono::steady_clock::time_point start_;
};

}  // namespace vreg_b200
#endif
