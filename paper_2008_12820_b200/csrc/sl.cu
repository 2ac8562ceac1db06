// Semi-Lagrangian kernels: RK2 characteristics (engine.hpp:111-155), gather
// interpolation (interp.cpp:70-115), its exact transpose (interp.cpp:92-123)
// and the fused transport steps of the state / adjoint / incremental solves
// (transport.hpp:49-228).
//
// Thread mapping: CTA = 32 x3-columns x 8 x2-rows of one x1 plane, so a
// warp's 32 departure points are contiguous nodes with near-identical
// displacements and their 4x4x4 stencils overlap in L1.
#include "common.cuh"
#include "sl_common.cuh"

namespace vb {

namespace {

constexpr int BX = 32, BY = 8;

inline dim3 sl_grid(const Slab& s) {
  return dim3(unsigned((s.n3 + BX - 1) / BX), unsigned((s.n2 + BY - 1) / BY), unsigned(s.n1l));
}

inline Geo geo_of(const Slab& s) {
  Geo g;
  g.n1 = s.n1;
  g.n1l = s.n1l;
  g.n2 = s.n2;
  g.n3 = s.n3;
  g.plane = s.plane();
  g.N = s.local();
  return g;
}

#define SL_INDEX                                           \
  const int k = blockIdx.x * BX + threadIdx.x;             \
  const int j = blockIdx.y * BY + threadIdx.y;             \
  const int i = blockIdx.z;                                \
  if (k >= g.n3 || j >= g.n2) return;                      \
  const size_t p = (size_t(i) * g.n2 + j) * g.n3 + k;

template <int DEG, bool DIST>
__global__ void __launch_bounds__(BX* BY) k_interp(Geo g, SrcField<DIST> src,
                                                   const float* __restrict__ D,
                                                   float* __restrict__ out) {
  SL_INDEX
  Stencil<DEG> st;
  st.template build<DIST>(g, i, j, k, D[p], D[g.N + p], D[2 * g.N + p]);
  out[p] = st.gather(g, src);
}

// out = I[f] .* q (adjoint sweep step: interp then hadamard, transport.hpp:115-117)
template <int DEG, bool DIST>
__global__ void __launch_bounds__(BX* BY) k_interp_mul(Geo g, SrcField<DIST> src,
                                                       const float* __restrict__ D,
                                                       const float* __restrict__ q,
                                                       float* __restrict__ out) {
  SL_INDEX
  Stencil<DEG> st;
  st.template build<DIST>(g, i, j, k, D[p], D[g.N + p], D[2 * g.N + p]);
  out[p] = st.gather(g, src) * q[p];
}

template <int DEG, bool DIST>
__global__ void __launch_bounds__(BX* BY) k_scatter(Geo g, DstField<DIST> dst,
                                                    const float* __restrict__ D,
                                                    const float* __restrict__ z) {
  SL_INDEX
  const float zp = z[p];
  if (zp == 0.0f) return;  // contributes nothing
  Stencil<DEG> st;
  st.template build<DIST>(g, i, j, k, D[p], D[g.N + p], D[2 * g.N + p]);
  st.scatter(g, dst, zp);
}

// RK2: mid = -dt/h v (grid units); vs = I[v](mid); D = -(dt/2)/h (v + vs).
template <int DEG, bool DIST>
__global__ void __launch_bounds__(BX* BY) k_characteristics(
    Geo g, SrcField<DIST> v1, SrcField<DIST> v2, SrcField<DIST> v3,
    const float* __restrict__ v, float m1, float m2, float m3, float c1, float c2, float c3,
    float* __restrict__ D) {
  SL_INDEX
  const float a = v[p], b = v[g.N + p], c = v[2 * g.N + p];
  Stencil<DEG> st;
  st.template build<DIST>(g, i, j, k, m1 * a, m2 * b, m3 * c);
  const float va = st.gather(g, v1);
  const float vb = st.gather(g, v2);
  const float vc = st.gather(g, v3);
  D[p] = c1 * (a + va);
  D[g.N + p] = c2 * (b + vb);
  D[2 * g.N + p] = c3 * (c + vc);
}

// One fused incremental-state step (transport.hpp:164-179), using linearity
// of I: w_t = m~_t - dt/2 u_t, I[m~_t] - dt/2 I[u_t] = I[w_t]:
//   G = I[w_t], u = vt . grad m_{t+1}, m~_{t+1} = G - dt/2 u,
//   w_{t+1} = m~_{t+1} - dt/2 u   (or psi_nt = -m~_nt on the last step).
template <int DEG, bool DIST>
__global__ void __launch_bounds__(BX* BY) k_inc_step(Geo g, SrcField<DIST> wsrc,
                                                     const float* __restrict__ D, int ident,
                                                     const float* __restrict__ vt,
                                                     const float* __restrict__ gr, float half,
                                                     int last, float* __restrict__ w_next,
                                                     float* __restrict__ mt_out) {
  SL_INDEX
  float G;
  if (ident) {
    G = wsrc.f[p];
  } else {
    Stencil<DEG> st;
    st.template build<DIST>(g, i, j, k, D[p], D[g.N + p], D[2 * g.N + p]);
    G = st.gather(g, wsrc);
  }
  const float u = vt[p] * gr[p] + vt[g.N + p] * gr[g.N + p] + vt[2 * g.N + p] * gr[2 * g.N + p];
  const float m = G - half * u;
  if (mt_out) mt_out[p] = m;
  w_next[p] = last ? -m : m - half * u;
}

// w0 = -dt/2 (vt . grad m_0)
__global__ void k_inc_init(size_t n, const float* __restrict__ vt, const float* __restrict__ gr,
                           float half, float* __restrict__ w0) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n; p += stride) {
    const float u = vt[p] * gr[p] + vt[n + p] * gr[n + p] + vt[2 * n + p] * gr[2 * n + p];
    w0[p] = -half * u;
  }
}

// out_c = sum_t w_t s_t grad_{t,c} (+ reg_c), t running nt..0 (descending,
// transport.hpp:217-224 then optim.hpp:130) or 0..nt (ascending,
// transport.hpp:191-199).
__global__ void k_assemble(size_t n, int nt, float dt, int descending,
                           const float* __restrict__ s, const float* __restrict__ grads,
                           const float* __restrict__ reg, float* __restrict__ out) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n; p += stride) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
    for (int q = 0; q <= nt; ++q) {
      const int t = descending ? nt - q : q;
      const float w = (t == 0 || t == nt) ? dt * 0.5f : dt;
      const float ws = w * s[size_t(t) * n + p];
      const float* gt = grads + size_t(t) * 3 * n;
      a0 += ws * gt[p];
      a1 += ws * gt[n + p];
      a2 += ws * gt[2 * n + p];
    }
    if (reg) {
      a0 += reg[p];
      a1 += reg[n + p];
      a2 += reg[2 * n + p];
    }
    out[p] = a0;
    out[n + p] = a1;
    out[2 * n + p] = a2;
  }
}

// q = (1 + dt/2 I_bwd[d]) / (1 - dt/2 d) (transport.hpp:55-60)
template <int DEG, bool DIST>
__global__ void __launch_bounds__(BX* BY) k_source_factor(Geo g, SrcField<DIST> dsrc,
                                                          const float* __restrict__ D,
                                                          int ident, float half,
                                                          float* __restrict__ q) {
  SL_INDEX
  float dd;
  if (ident) {
    dd = dsrc.f[p];
  } else {
    Stencil<DEG> st;
    st.template build<DIST>(g, i, j, k, D[p], D[g.N + p], D[2 * g.N + p]);
    dd = st.gather(g, dsrc);
  }
  q[p] = (1.0f + half * dd) / (1.0f - half * dsrc.f[p]);
}

template <bool DIST>
SrcField<DIST> src_of(const float* f, const Ghosts& gh) {
  SrcField<DIST> s;
  s.f = f;
  s.lo = gh.lo;
  s.hi = gh.hi;
  s.G = gh.G;
  return s;
}

template <bool DIST>
DstField<DIST> dst_of(float* f, const GhostAcc& gh) {
  DstField<DIST> s;
  s.f = f;
  s.lo = gh.lo;
  s.hi = gh.hi;
  s.G = gh.G;
  return s;
}

inline void check_degree(int degree) {
  require(degree == 1 || degree == 3, VREG_EPARAM, "interpolation degree must be 1 or 3");
}

// Dispatch a kernel template over (degree, dist).
#define SL_DISPATCH(degree, dist, LAUNCH)                 \
  do {                                                    \
    if (degree == 3) {                                    \
      if (dist) {                                         \
        constexpr int DEG = 3;                            \
        constexpr bool DIST = true;                       \
        LAUNCH;                                           \
      } else {                                            \
        constexpr int DEG = 3;                            \
        constexpr bool DIST = false;                      \
        LAUNCH;                                           \
      }                                                   \
    } else {                                              \
      if (dist) {                                         \
        constexpr int DEG = 1;                            \
        constexpr bool DIST = true;                       \
        LAUNCH;                                           \
      } else {                                            \
        constexpr int DEG = 1;                            \
        constexpr bool DIST = false;                      \
        LAUNCH;                                           \
      }                                                   \
    }                                                     \
    count_launch(ctx);                                    \
    check_launch();                                       \
  } while (0)

struct CharsInfo {
  bool identity;
  int G;  // x1 ghost width for multi-rank sweeps
};

inline CharsInfo chars_info(vreg_ctx ctx, const Slab& s, const float* disp3, int flags,
                            int degree) {
  CharsInfo ci;
  ci.identity = (flags & 1) != 0;
  ci.G = 0;
  if (ctx->nranks > 1 && !ci.identity) {
    ci.G = (flags >> 8) - 1;
    if (ci.G < 0) ci.G = sl_ghost_width(ctx, s, disp3, degree);
  }
  return ci;
}

// out = I[f] at disp (optionally .* q)
void interp_sweep(vreg_ctx ctx, const Slab& s, const float* f, const float* disp3,
                  const CharsInfo& ci, int degree, const float* q, float* out) {
  if (ci.identity) {
    if (q) {
      VB_CUDA(cudaMemcpyAsync(out, f, s.local() * sizeof(float), cudaMemcpyDeviceToDevice,
                              ctx->stream));
      vreg_grid gg{s.n1, s.n2, s.n3, s.nt};
      int st = vreg_hadamard(ctx, &gg, out, q, out);
      require(st == VREG_OK, st, "hadamard failed");
    } else if (out != f) {
      VB_CUDA(cudaMemcpyAsync(out, f, s.local() * sizeof(float), cudaMemcpyDeviceToDevice,
                              ctx->stream));
    }
    return;
  }
  const bool dist = ctx->nranks > 1;
  Ghosts gh;
  if (dist) gh = halo_exchange(ctx, s, f, ci.G, "sl_ghost", T_INTERP_COMM, C_GHOST_INTERP);
  Timed t(ctx, T_SL, "sl_interp");
  const Geo g = geo_of(s);
  const dim3 grid = sl_grid(s), block(BX, BY);
  if (q)
    SL_DISPATCH(degree, dist,
                (k_interp_mul<DEG, DIST><<<grid, block, 0, ctx->stream>>>(
                    g, src_of<DIST>(f, gh), disp3, q, out)));
  else
    SL_DISPATCH(degree, dist,
                (k_interp<DEG, DIST><<<grid, block, 0, ctx->stream>>>(g, src_of<DIST>(f, gh),
                                                                      disp3, out)));
}

// out = I^T z (out is overwritten)
void scatter_sweep(vreg_ctx ctx, const Slab& s, const float* z, const float* disp3,
                   const CharsInfo& ci, int degree, float* out) {
  if (ci.identity) {
    if (out != z)
      VB_CUDA(cudaMemcpyAsync(out, z, s.local() * sizeof(float), cudaMemcpyDeviceToDevice,
                              ctx->stream));
    return;
  }
  require(out != z, VREG_EPARAM, "scatter cannot run in place");
  const bool dist = ctx->nranks > 1;
  GhostAcc acc;
  if (dist) acc = ghost_accumulators(ctx, s, ci.G, "sl_gacc");
  {
    Timed t(ctx, T_SL, "sl_scatter_sweep");
    VB_CUDA(cudaMemsetAsync(out, 0, s.local() * sizeof(float), ctx->stream));
    const Geo g = geo_of(s);
    const dim3 grid = sl_grid(s), block(BX, BY);
    SL_DISPATCH(degree, dist,
                (k_scatter<DEG, DIST><<<grid, block, 0, ctx->stream>>>(
                    g, dst_of<DIST>(out, acc), disp3, z)));
  }
  if (dist) halo_reverse_add(ctx, s, acc, out, "sl_gacc");
}

}  // namespace

// Shared with matvec.cu / precond paths.
void sl_interp(vreg_ctx ctx, const Slab& s, const float* f, const float* disp3, int flags,
               int degree, const float* q, float* out) {
  check_degree(degree);
  interp_sweep(ctx, s, f, disp3, chars_info(ctx, s, disp3, flags, degree), degree, q, out);
}

void sl_scatter(vreg_ctx ctx, const Slab& s, const float* z, const float* disp3, int flags,
                int degree, float* out) {
  check_degree(degree);
  scatter_sweep(ctx, s, z, disp3, chars_info(ctx, s, disp3, flags, degree), degree, out);
}

void sl_inc_state(vreg_ctx ctx, const Slab& s, const float* disp3, int flags, int degree,
                  const float* grads, const float* vt3, float* mt_all, float* psi_out) {
  check_degree(degree);
  const CharsInfo ci = chars_info(ctx, s, disp3, flags, degree);
  const size_t N = s.local();
  const int nt = s.nt;
  const float half = float(0.5 * s.dt());
  float* w = static_cast<float*>(workspace(ctx, "inc_w", 2 * N * sizeof(float)));
  {
    Timed t(ctx, T_SL, "sl_inc_init");
    k_inc_init<<<blocks_for(N, 256), 256, 0, ctx->stream>>>(N, vt3, grads, half, w);
    count_launch(ctx);
    check_launch();
  }
  if (mt_all) VB_CUDA(cudaMemsetAsync(mt_all, 0, N * sizeof(float), ctx->stream));
  const bool dist = ctx->nranks > 1 && !ci.identity;
  const Geo g = geo_of(s);
  const dim3 grid = sl_grid(s), block(BX, BY);
  for (int t = 0; t < nt; ++t) {
    const float* wt = w + size_t(t & 1) * N;
    const bool last = t == nt - 1;
    float* wn = last ? psi_out : w + size_t((t + 1) & 1) * N;
    float* mo = mt_all ? mt_all + size_t(t + 1) * N : nullptr;
    Ghosts gh;
    if (dist) gh = halo_exchange(ctx, s, wt, ci.G, "sl_ghost", T_INTERP_COMM, C_GHOST_INTERP);
    Timed tm(ctx, T_SL, "sl_inc_step");
    SL_DISPATCH(degree, dist,
                (k_inc_step<DEG, DIST><<<grid, block, 0, ctx->stream>>>(
                    g, src_of<DIST>(wt, gh), disp3, ci.identity ? 1 : 0, vt3,
                    grads + size_t(t + 1) * 3 * N, half, last ? 1 : 0, wn, mo)));
  }
}

// psi[t-1] = I^T psi[t] for t = nt..1; psi holds nt+1 slices, psi[nt] set.
void sl_transpose_sweeps(vreg_ctx ctx, const Slab& s, const float* disp3, int flags,
                         int degree, float* psi) {
  check_degree(degree);
  const CharsInfo ci = chars_info(ctx, s, disp3, flags, degree);
  const size_t N = s.local();
  for (int t = s.nt; t > 0; --t)
    scatter_sweep(ctx, s, psi + size_t(t) * N, disp3, ci, degree, psi + size_t(t - 1) * N);
}

void sl_assemble(vreg_ctx ctx, const Slab& s, int descending, const float* sl,
                 const float* grads, const float* reg, float* out3) {
  Timed t(ctx, T_SL, "sl_assemble");
  const size_t N = s.local();
  k_assemble<<<blocks_for(N, 256), 256, 0, ctx->stream>>>(N, s.nt, float(s.dt()), descending,
                                                            sl, grads, reg, out3);
  count_launch(ctx);
  check_launch();
}

int sl_characteristics(vreg_ctx ctx, const Slab& s, const float* v3, int degree,
                       float* disp3) {
  check_degree(degree);
  const size_t N = s.local();
  const double vmax = reduce(ctx, s, 3, v3, v3, true);
  if (vmax == 0.0) {
    VB_CUDA(cudaMemsetAsync(disp3, 0, 3 * N * sizeof(float), ctx->stream));
    return 1;
  }
  const bool dist = ctx->nranks > 1;
  const double dt = s.dt();
  Ghosts g1, g2, g3;
  if (dist) {
    // ghost width from the midpoint displacement bound dt max|v1| / h1
    const double vmax1 = reduce(ctx, s, 1, v3, v3, true);
    int G = int(std::floor(dt * vmax1 / s.h(0))) + (degree == 3 ? 3 : 2);
    require(G <= s.n1l, VREG_ECONFIG,
            "displacement exceeds the slab width (halo would span several ranks)");
    g1 = halo_exchange(ctx, s, v3, G, "chars_g1", T_INTERP_COMM, C_GHOST_INTERP);
    g2 = halo_exchange(ctx, s, v3 + N, G, "chars_g2", T_INTERP_COMM, C_GHOST_INTERP);
    g3 = halo_exchange(ctx, s, v3 + 2 * N, G, "chars_g3", T_INTERP_COMM, C_GHOST_INTERP);
  }
  Timed t(ctx, T_SL, "sl_characteristics");
  const Geo g = geo_of(s);
  const dim3 grid = sl_grid(s), block(BX, BY);
  const float m1 = float(-dt / s.h(0)), m2 = float(-dt / s.h(1)), m3 = float(-dt / s.h(2));
  const float c1 = float(-0.5 * dt / s.h(0)), c2 = float(-0.5 * dt / s.h(1)),
              c3 = float(-0.5 * dt / s.h(2));
  SL_DISPATCH(degree, dist,
              (k_characteristics<DEG, DIST><<<grid, block, 0, ctx->stream>>>(
                  g, src_of<DIST>(v3, g1), src_of<DIST>(v3 + N, g2),
                  src_of<DIST>(v3 + 2 * N, g3), v3, m1, m2, m3, c1, c2, c3, disp3)));
  return 0;
}

void sl_source_factor(vreg_ctx ctx, const Slab& s, const float* d, const float* disp_bwd3,
                      int flags, int degree, float* q) {
  check_degree(degree);
  const CharsInfo ci = chars_info(ctx, s, disp_bwd3, flags, degree);
  const bool dist = ctx->nranks > 1 && !ci.identity;
  Ghosts gh;
  if (dist) gh = halo_exchange(ctx, s, d, ci.G, "sl_ghost", T_INTERP_COMM, C_GHOST_INTERP);
  Timed t(ctx, T_SL);
  const Geo g = geo_of(s);
  const dim3 grid = sl_grid(s), block(BX, BY);
  const float half = float(0.5 * s.dt());
  SL_DISPATCH(degree, dist,
              (k_source_factor<DEG, DIST><<<grid, block, 0, ctx->stream>>>(
                  g, src_of<DIST>(d, gh), disp_bwd3, ci.identity ? 1 : 0, half, q)));
}

}  // namespace vb

using namespace vb;

extern "C" {

int vreg_characteristics(vreg_ctx ctx, const vreg_grid* g, const float* v3, int degree,
                         float* disp3, int* identity) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    int ident = sl_characteristics(ctx, s, v3, degree, disp3);
    int flags = ident;
    if (ctx->nranks > 1 && !ident) flags |= (sl_ghost_width(ctx, s, disp3, degree) + 1) << 8;
    if (identity) *identity = flags;
  });
}

int vreg_interp(vreg_ctx ctx, const vreg_grid* g, const float* f, const float* disp3,
                int identity, int degree, float* out) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    sl_interp(ctx, s, f, disp3, identity, degree, nullptr, out);
  });
}

int vreg_scatter(vreg_ctx ctx, const vreg_grid* g, const float* z, const float* disp3,
                 int identity, int degree, float* out) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    sl_scatter(ctx, s, z, disp3, identity, degree, out);
  });
}

int vreg_solve_state(vreg_ctx ctx, const vreg_grid* g, const float* disp3, int identity,
                     int degree, float* m) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    for (int t = 0; t < s.nt; ++t)
      sl_interp(ctx, s, m + size_t(t) * s.local(), disp3, identity, degree, nullptr,
                m + size_t(t + 1) * s.local());
  });
}

int vreg_inc_state(vreg_ctx ctx, const vreg_grid* g, const float* disp3, int identity,
                   int degree, const float* grads, const float* vt3, float* mt_all,
                   float* mt_final) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    const size_t N = s.local();
    float* psi = static_cast<float*>(workspace(ctx, "inc_psi", N * sizeof(float)));
    sl_inc_state(ctx, s, disp3, identity, degree, grads, vt3, mt_all, psi);
    if (mt_final) {  // psi_nt = -m~_nt
      VB_CUDA(cudaMemcpyAsync(mt_final, psi, N * sizeof(float), cudaMemcpyDeviceToDevice,
                              ctx->stream));
      int st = vreg_scale(ctx, g, 1, mt_final, -1.0);
      require(st == VREG_OK, st, "scale failed");
    }
  });
}

int vreg_transpose_assemble(vreg_ctx ctx, const vreg_grid* g, const float* disp3, int identity,
                            int degree, const float* grads, const float* fin, float* out3) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    const size_t N = s.local();
    float* psi = static_cast<float*>(
        workspace(ctx, "mv_psi", size_t(s.nt + 1) * N * sizeof(float)));
    VB_CUDA(cudaMemcpyAsync(psi + size_t(s.nt) * N, fin, N * sizeof(float),
                            cudaMemcpyDeviceToDevice, ctx->stream));
    sl_transpose_sweeps(ctx, s, disp3, identity, degree, psi);
    sl_assemble(ctx, s, 1, psi, grads, nullptr, out3);
  });
}

int vreg_adjoint_source_factor(vreg_ctx ctx, const vreg_grid* g, const float* v3,
                               const float* disp_bwd3, int identity_bwd, int degree,
                               float* q) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    float* d = static_cast<float*>(workspace(ctx, "asf_div", s.local() * sizeof(float)));
    int st = vreg_fd_div(ctx, g, v3, d);
    require(st == VREG_OK, st, vreg_last_error());
    const double dmax = reduce(ctx, s, 1, d, d, true);
    require(!(0.5 * s.dt() * dmax >= 0.99), VREG_ENUMERICAL,
            "divergence too large for the time step");
    sl_source_factor(ctx, s, d, disp_bwd3, identity_bwd, degree, q);
  });
}

int vreg_adjoint_sweep(vreg_ctx ctx, const vreg_grid* g, const float* disp_bwd3,
                       int identity_bwd, int degree, const float* q, float* lam) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    const size_t N = s.local();
    for (int t = s.nt - 1; t >= 0; --t)
      sl_interp(ctx, s, lam + size_t(t + 1) * N, disp_bwd3, identity_bwd, degree, q,
                lam + size_t(t) * N);
  });
}

int vreg_integrate_lambda_grad_m(vreg_ctx ctx, const vreg_grid* g, const float* lam,
                                 const float* grads, float* out3) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    sl_assemble(ctx, s, 0, lam, grads, nullptr, out3);
  });
}

}  // extern "C"
