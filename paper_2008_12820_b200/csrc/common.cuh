// Shared internals of libvreg_b200.so: the per-GPU context (EngineState
// analogue, proj/include/vreg/engine.hpp:14-19), error plumbing for the C
// ABI, launch helpers, workspace cache and CUDA-event kernel timers.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "vreg_cuda.h"

namespace vb {

// ---- errors ---------------------------------------------------------------

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& m);

template <class F>
inline int guard(F&& f) {
  try {
    f();
    return VREG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return VREG_ECUDA;
  }
}

#define VB_CUDA(call)                                                       \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess)                                                  \
      throw ::vb::Error(VREG_ECUDA, std::string(#call ": ") +               \
                                        cudaGetErrorString(e_));            \
  } while (0)

#define VB_CUFFT(call)                                                      \
  do {                                                                      \
    cufftResult r_ = (call);                                                \
    if (r_ != CUFFT_SUCCESS)                                                \
      throw ::vb::Error(VREG_ECUDA, std::string(#call ": cufft error ") +   \
                                        std::to_string(int(r_)));           \
  } while (0)

#define VB_NCCL(call)                                                       \
  do {                                                                      \
    ncclResult_t r_ = (call);                                               \
    if (r_ != ncclSuccess)                                                  \
      throw ::vb::Error(VREG_ECUDA, std::string(#call ": ") +               \
                                        ncclGetErrorString(r_));            \
  } while (0)

inline void require(bool ok, int code, const char* msg) {
  if (!ok) throw Error(code, msg);
}

// ---- timers ---------------------------------------------------------------

enum TimerCat {
  T_FFT = 0,
  T_FD,
  T_SL,
  T_GHOST,
  T_INTERP_COMM,
  T_SCATTER_COMM,
  T_SCATTER_BUF,
  T_TRANSPOSE,
  T_COUNT
};

enum CommCat {
  C_GHOST_FD = 0,
  C_GHOST_INTERP,
  C_SCATTER_POINTS,
  C_INTERP_VALUES,
  C_FFT_TRANSPOSE,
  C_SPECTRAL_GATHER,
  C_REDUCE,
  C_P2P_MSGS,
  C_ALLTOALL,
  C_COUNT
};

// ---- FFT plans ------------------------------------------------------------

struct FftPlans {
  cufftHandle r2c = 0, c2r = 0;
  size_t work = 0;
  cudaStream_t stream = nullptr;  // stream the plans are bound to
};

// ---- context --------------------------------------------------------------

}  // namespace vb

struct vreg_ctx_s {
  int device = 0;
  int rank = 0;
  int nranks = 1;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  ncclComm_t comm = nullptr;
  // side stream + dedicated communicator for the regulariser branch of the
  // matvec (FFTs and their all-to-alls overlap the SL sweeps)
  cudaStream_t side = nullptr;
  ncclComm_t fft_comm = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // halo exchanges of the distributed SL sweeps run here, overlapping the
  // interior tiles (high priority so NCCL's CTAs are scheduled promptly)
  // transpose sweeps in exact fixed point (bitwise reproducible, independent
  // of the GPU count) instead of fp32 L2 reductions (VREG_DETERMINISTIC=1)
  bool deterministic = false;
  // regularisation order of the spectral operators: 1 = H1 (symbol |k|^2,
  // the reference's spectral.cpp:61-63), 2 = H2 (|k|^4, B200 extension)
  int reg_order = 1;
  double tl_beta = 0;  // beta_pc of the last two-level begin (read by its end)
  bool pipe_dynamic = false;  // next gather-pipe launches take tiles from a ticket counter
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_c0 = nullptr, ev_c1 = nullptr;
  // regulariser x2-slab transposes by copy engine into the peers' buffers
  // (CUDA IPC over NVLink, spec_axis.cu): local send/recv buffers, the peers'
  // receive buffers, a barrier word
  float* xbuf[2] = {nullptr, nullptr};
  std::vector<float*> peer_recv;
  size_t xbytes = 0;
  int* xflag = nullptr;

  // FFT plans keyed by (n1, n2, n3, batch); one shared work area
  std::map<std::tuple<int, int, int, int>, vb::FftPlans> plans;
  void* fft_work = nullptr;
  size_t fft_work_size = 0;

  // named workspace buffers (reused across calls)
  std::map<std::string, std::pair<void*, size_t>> ws;

  // per-characteristics tile box tables (sl_tile.cuh), small LRU
  struct TileTable {
    const float* disp;
    int n1, n2, n3, n1l, deg;
    int* table;
    uint64_t used;
    int smem_words;  // largest box in words: the launches' dynamic smem
  };
  std::vector<TileTable> tile_tables;
  uint64_t tile_clock = 0;
  uint64_t tiles_built = 0, tiles_misfit = 0;  // boxes over the smem budget

  // reduction scratch
  double* h_pinned = nullptr;  // host staging
  size_t h_pinned_cap = 0;

  // timers
  bool timers_on = false;
  struct Pending {
    int cat;
    const char* name;
    cudaEvent_t a, b;
  };
  std::map<std::string, std::pair<uint64_t, double>> kstats;  // per named kernel
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  double timer_acc[vb::T_COUNT] = {0};
  uint64_t comm_bytes[vb::C_COUNT] = {0};
  uint64_t launches = 0;
};

namespace vb {

// Slab geometry of grid g on this context.
struct Slab {
  int n1, n2, n3, nt;
  int n1l, off;
  size_t plane() const { return size_t(n2) * size_t(n3); }
  size_t local() const { return size_t(n1l) * plane(); }
  size_t global() const { return size_t(n1) * plane(); }
  double h(int a) const;
  double dt() const { return 1.0 / double(nt); }
};

Slab slab_of(vreg_ctx ctx, const vreg_grid* g);

void* workspace(vreg_ctx ctx, const std::string& name, size_t bytes);
void resolve_timers(vreg_ctx ctx);
double* pinned(vreg_ctx ctx, size_t n);

FftPlans& fft_plans(vreg_ctx ctx, int n1, int n2, int n3, int batch);

class Timed {
 public:
  Timed(vreg_ctx ctx, int cat, const char* name = nullptr);
  ~Timed();
  Timed(const Timed&) = delete;
  Timed& operator=(const Timed&) = delete;

 private:
  vreg_ctx ctx_;
  int cat_;
  const char* name_;
  cudaEvent_t a_ = nullptr;
};

inline void count_launch(vreg_ctx ctx, uint64_t n = 1) { ctx->launches += n; }

// Opt a kernel in to `bytes` of dynamic shared memory on the current device
// (function attributes are per device: once per (device, kernel), thread-safe).
void smem_optin(const void* kernel, int bytes);

inline void check_launch() { VB_CUDA(cudaGetLastError()); }

// Division by a runtime-invariant divisor as a multiply-high and shift
// (round-up reciprocal, exact for dividends < 2^31): the flat spectral
// kernels split element indices with it instead of 32-bit IDIV sequences.
struct FastDiv {
  unsigned d = 1, m = 0;
  int sh = 0;
  FastDiv() = default;
  explicit FastDiv(unsigned dv) : d(dv) {
    if (d <= 1) return;
    int l = 0;
    while ((1u << l) < d) ++l;  // ceil log2 d
    const int p = 31 + l;
    m = unsigned(((1ull << p) + d - 1) / d);
    sh = p - 32;
  }
#ifdef __CUDACC__
  __device__ __forceinline__ unsigned div(unsigned n) const {
    return d == 1 ? n : (__umulhi(n, m) >> sh);
  }
  __device__ __forceinline__ unsigned divmod(unsigned n, unsigned& r) const {
    const unsigned q = div(n);
    r = n - q * d;
    return q;
  }
#endif
};

inline unsigned blocks_for(size_t n, unsigned threads, unsigned cap = 148u * 32u) {
  size_t b = (n + threads - 1) / threads;
  if (b > cap) b = cap;
  if (b == 0) b = 1;
  return unsigned(b);
}

// Plane-folded fp64 reduction (pointwise.cu): inner product (is_max false,
// times the cell volume) or max |a| (is_max true) over ncomp components.
double reduce(vreg_ctx ctx, const Slab& s, int ncomp, const float* a, const float* b,
              bool is_max);

// ---- x1 halos (dist.cu) ----------------------------------------------------
// Ghost planes of a slab-distributed field: lo = the G planes below the slab
// (owned by lower ranks), hi = the G planes above it (periodic ring).
struct Ghosts {
  const float* lo = nullptr;
  const float* hi = nullptr;
  int G = 0;
};
struct GhostAcc {
  float* lo = nullptr;
  float* hi = nullptr;
  int G = 0;
};
// Exchange G boundary planes of f with the ring neighbours (ncclSend/Recv).
Ghosts halo_exchange(vreg_ctx ctx, const Slab& s, const float* f, int G,
                     const char* slot, int timer_cat, int comm_cat);
// Zeroed ghost accumulators for a transpose (scatter) sweep.
GhostAcc ghost_accumulators(vreg_ctx ctx, const Slab& s, int G, const char* slot);
// Reverse halo: ship the ghost accumulators to their owners and add them
// into the owners' boundary planes of out.

// Reverse halo add in two halves so the exchange can run on another stream:
// send the ghost accumulators / receive the neighbours' (top, bot), then add.
struct RevHalo {
  float* top = nullptr;
  float* bot = nullptr;
  int G = 0;
};
RevHalo halo_reverse_send(vreg_ctx ctx, const Slab& s, const GhostAcc& acc, const char* slot);
void halo_reverse_finish(vreg_ctx ctx, const Slab& s, const RevHalo& r, float* out,
                         bool as_int = false);
void halo_reverse_add(vreg_ctx ctx, const Slab& s, const GhostAcc& acc, float* out,
                      const char* slot, bool as_int = false);
// Ghost width for a semi-Lagrangian sweep: floor(max|disp1|) + degree-dependent
// stencil reach; checked against the slab width.
int sl_ghost_width(vreg_ctx ctx, const Slab& s, const float* disp1, int degree);
// All-gather of per-plane fp64 partials in global plane order.
void allgather_partials(vreg_ctx ctx, const Slab& s, const double* d_local, double* d_global,
                        size_t per_plane);

}  // namespace vb
