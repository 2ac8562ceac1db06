// Report rendering and volume files for the B200 solver.
//
// The reference declares render_report / render_timings /
// render_residuals_csv (proj/include/vreg/report.hpp:79-84) without defining
// them, and specifies the VolumeFile format "VRG1". These
// are the definitions for vreg_b200::SolverReport (records.hpp):
//   * render_report: deterministic structured text, no timings, so serial
//     reruns are byte-identical;
//   * render_timings: the wall-clock section (phase and kernel timers);
//   * render_residuals_csv: per-iteration PCG relative residuals;
//   * save_volume / load_volume: "VRG1", u32 LE n1 n2 n3, u8 scalar kind
//     (0 f32, 1 f64), u8 components (1 or 3), components concatenated,
//     row-major little-endian; corrupted magic/length -> io_error.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "vreg_b200/records.hpp"

namespace vreg_b200 {

namespace detail {
inline std::string num(double x) {
  char b[40];
  std::snprintf(b, sizeof b, "%.10e", x);
  return b;
}
}  // namespace detail

inline std::string render_report(const SolverReport& r) {
  using detail::num;
  std::ostringstream o;
  o << "vreg_b200 report\n";
  o << "grid " << r.grid.n1 << " " << r.grid.n2 << " " << r.grid.n3 << " nt " << r.nt << " p "
    << r.p << "\n";
  o << "initial_mismatch " << num(r.initial_mismatch) << "\n";
  for (size_t li = 0; li < r.levels.size(); ++li) {
    const LevelRecord& l = r.levels[li];
    o << "level " << li << " beta " << num(l.beta) << " pc " << l.pc_name << " switched "
      << (l.pc_switched_from_config ? 1 : 0) << " gn " << l.gn_iters << " pcg " << l.pcg_total
      << " converged " << (l.converged ? 1 : 0) << " line_search_failed "
      << (l.line_search_failed ? 1 : 0) << " inner_capped " << (l.inner_capped ? 1 : 0) << "\n";
    o << "  mismatch " << num(l.initial_mismatch) << " -> " << num(l.final_mismatch)
      << " g_rel " << num(l.final_g_rel) << " objective " << num(l.final_objective) << "\n";
    o << "  refresh " << l.refresh_count << " pc_inva_apps " << l.pc_inva_apps << " pc_h0_apps "
      << l.pc_h0_apps << " h0_inner_total " << l.h0_inner_total << " line_search_states "
      << l.line_search_states << "\n";
    for (size_t k = 0; k < l.iters.size(); ++k) {
      const GnIterRecord& it = l.iters[k];
      o << "  gn " << k + 1 << " J " << num(it.objective) << " mismatch " << num(it.mismatch)
        << " g " << num(it.g_norm) << " g_rel " << num(it.g_rel) << " eps_k " << num(it.eps_k)
        << " alpha " << num(it.alpha) << " pcg " << it.pcg_iters << " ls " << it.line_search_trials
        << " beta_pc " << num(it.beta_pc) << " h0_inner " << it.h0_inner_iters << "\n";
    }
  }
  const KernelCounters& c = r.counters;
  o << "counters fft_forward " << c.fft_forward << " fft_inverse " << c.fft_inverse
    << " fft_forward_coarse " << c.fft_forward_coarse << " fft_inverse_coarse "
    << c.fft_inverse_coarse << " fd_gradient " << c.fd_gradient << " fd_divergence "
    << c.fd_divergence << " ip_eval " << c.ip_eval << " ip_scatter " << c.ip_scatter
    << " characteristics " << c.characteristics << " sl_state " << c.sl_state << " sl_adjoint "
    << c.sl_adjoint << " sl_inc_state " << c.sl_inc_state << " sl_inc_adjoint "
    << c.sl_inc_adjoint << " pc_inva_apply " << c.pc_inva_apply << " pc_h0_apply "
    << c.pc_h0_apply << " pc_h0_inner_iters " << c.pc_h0_inner_iters << "\n";
  o << "final mismatch " << num(r.final_mismatch) << " mism_rel " << num(r.mism_rel) << " g_rel "
    << num(r.final_g_rel) << " gn " << r.total_gn() << " pcg " << r.total_pcg() << " flagged "
    << (r.flagged ? 1 : 0) << "\n";
  return o.str();
}

inline std::string render_timings(const SolverReport& r) {
  std::ostringstream o;
  char b[256];
  std::snprintf(b, sizeof b, "phases_s total %.6f pc %.6f obj %.6f grad %.6f hess %.6f\n",
                r.phases.total, r.phases.pc, r.phases.obj, r.phases.grad, r.phases.hess);
  o << b;
  const KernelTimers& k = r.kernels;
  std::snprintf(b, sizeof b,
                "kernels_s fft %.6f fd %.6f sl %.6f ghost_comm %.6f interp_comm %.6f "
                "scatter_comm %.6f scatter_buffer %.6f transpose_comm %.6f\n",
                k.fft, k.fd, k.sl, k.ghost_comm, k.interp_comm, k.scatter_comm, k.scatter_buffer,
                k.transpose_comm);
  o << b;
  return o.str();
}

inline std::string render_residuals_csv(const SolverReport& r) {
  std::ostringstream o;
  o << "level,beta,gn_iter,pcg_iter,rel_residual\n";  // pcg_iter 0: initial residual
  for (size_t li = 0; li < r.levels.size(); ++li)
    for (size_t k = 0; k < r.levels[li].iters.size(); ++k) {
      const auto& h = r.levels[li].iters[k].pcg_relres;
      for (size_t j = 0; j < h.size(); ++j)
        o << li << "," << detail::num(r.levels[li].beta) << "," << k + 1 << "," << j << ","
          << detail::num(h[j]) << "\n";
    }
  return o.str();
}

// ---- VolumeFile "VRG1" ------------------------------------------------------

struct Volume {
  int n1 = 0, n2 = 0, n3 = 0;
  int kind = 0;   // 0 = f32, 1 = f64
  int ncomp = 1;  // 1 or 3
  std::vector<unsigned char> payload;  // components concatenated, little-endian
  size_t scalar_bytes() const { return kind == 0 ? 4 : 8; }
  size_t expected_bytes() const {
    return size_t(ncomp) * size_t(n1) * size_t(n2) * size_t(n3) * scalar_bytes();
  }
};

namespace detail {
inline void put_u32(std::string& s, std::uint32_t v) {
  for (int i = 0; i < 4; ++i) s.push_back(char((v >> (8 * i)) & 0xff));
}
inline std::uint32_t get_u32(const unsigned char* p) {
  return std::uint32_t(p[0]) | std::uint32_t(p[1]) << 8 | std::uint32_t(p[2]) << 16 |
         std::uint32_t(p[3]) << 24;
}
}  // namespace detail

inline void save_volume(const std::string& path, const Volume& v) {
  if ((v.kind != 0 && v.kind != 1) || (v.ncomp != 1 && v.ncomp != 3) || v.n1 <= 0 || v.n2 <= 0 ||
      v.n3 <= 0)
    throw parameter_error("volume: bad header fields");
  if (v.payload.size() != v.expected_bytes()) throw parameter_error("volume: payload size");
  std::string h = "VRG1";
  detail::put_u32(h, std::uint32_t(v.n1));
  detail::put_u32(h, std::uint32_t(v.n2));
  detail::put_u32(h, std::uint32_t(v.n3));
  h.push_back(char(v.kind));
  h.push_back(char(v.ncomp));
  std::ofstream f(path, std::ios::binary);
  if (!f) throw io_error("volume: cannot open " + path + " for writing");
  f.write(h.data(), std::streamsize(h.size()));
  f.write(reinterpret_cast<const char*>(v.payload.data()), std::streamsize(v.payload.size()));
  if (!f) throw io_error("volume: write failed: " + path);
}

inline Volume load_volume(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw io_error("volume: cannot open " + path);
  std::vector<unsigned char> all((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  if (all.size() < 18 || std::memcmp(all.data(), "VRG1", 4) != 0)
    throw io_error("volume: bad magic in " + path);
  Volume v;
  v.n1 = int(detail::get_u32(&all[4]));
  v.n2 = int(detail::get_u32(&all[8]));
  v.n3 = int(detail::get_u32(&all[12]));
  v.kind = all[16];
  v.ncomp = all[17];
  if ((v.kind != 0 && v.kind != 1) || (v.ncomp != 1 && v.ncomp != 3) || v.n1 <= 0 || v.n2 <= 0 ||
      v.n3 <= 0)
    throw io_error("volume: bad header in " + path);
  if (all.size() - 18 != v.expected_bytes())
    throw io_error("volume: payload length does not match the header in " + path);
  v.payload.assign(all.begin() + 18, all.end());
  return v;
}

}  // namespace vreg_b200
