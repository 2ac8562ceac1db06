// 8th-order periodic finite differences (proj/src/fd.cpp:7-179).
//
// All three axes use the paired antisymmetric form sum_j c_j (f_{+j} - f_{-j})
// (fd.cpp:60-78; the reference uses it on x1 and an unpaired 9-tap sum with
// a ~3e-16 centre weight on x2/x3, fd.cpp:80-125 -- identical to fp64
// round-off). Weights are the closed-form values of the
// reference's Fornberg recursion (fd.cpp:7-48), rounded once to fp32.
//
// Tiling: see the x1-marching kernels below (register window along x1,
// double-buffered shared tile with the x2/x3 halo of 4).
#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace vb {

namespace {

constexpr int TX = 32, H = 4;

// Paired 8th-order first-derivative weights c_j, j = 1..4, unit spacing: the
// antisymmetric half of the 9-point Fornberg stencil the reference builds in
// fd.cpp:7-48 (4/5, -1/5, 4/105, -1/280), rounded once to fp32.
struct FdW {
  float c[4];
};

FdW fd_weights() {
  return FdW{{float(4.0 / 5.0), float(-1.0 / 5.0), float(4.0 / 105.0), float(-1.0 / 280.0)}};
}

struct FdGeo {
  int n1, n1l, n2, n3;
  size_t plane;
};

template <bool DIST>
__device__ __forceinline__ const float* fd_plane(const float* f, const float* lo, const float* hi,
                                                 int p, const FdGeo& g) {
  if constexpr (DIST) {
    if (p < 0) return lo + size_t(p + H) * g.plane;
    if (p >= g.n1l) return hi + size_t(p - g.n1l) * g.plane;
    return f + size_t(p) * g.plane;
  } else {
    p = p < 0 ? p + g.n1 : (p >= g.n1 ? p - g.n1 : p);
    return f + size_t(p) * g.plane;
  }
}

// ---- x1-marching kernels ----------------------------------------------------
// A CTA owns a 32 (x3) x 8 (x2) column of the slab and marches FD_CH planes
// along x1: each thread keeps its column's 9-plane window in registers (the
// x1 stencil; the plane two steps ahead is already in flight), and the
// current plane's tile + x2/x3 halo sits in a 3-deep ring of shared tiles
// filled by 16-byte cp.async two planes ahead, so the loop never waits on a
// fresh global load. Each input element is read from HBM about once; no
// integer division is left in the loop. Same paired sums in the same order as
// the per-plane formulation: bitwise identical results.
constexpr int FD_RING = 3;  // shared tiles in flight
constexpr int TW = TX + 2 * H;

__device__ __forceinline__ int wrap_fd(int x, int n) { return x < 0 ? x + n : (x >= n ? x - n : x); }
// halo-tile wrap: axes shorter than the tile extent (n3 < TW columns,
// n2 < TY + 2H rows) wrap more than once, so those grids take a true modulo
__device__ __forceinline__ int wrap_col(int x, int n) {
  return n >= TW ? wrap_fd(x, n) : ((x % n) + n) % n;
}
template <int TY>
__device__ __forceinline__ int wrap_row(int x, int n) {
  return n >= TY + 2 * H ? wrap_fd(x, n) : ((x % n) + n) % n;
}

__device__ __forceinline__ void fd_cp16(float* smem, const float* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void fd_cp4(float* smem, const float* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void fd_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void fd_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Issue the tile + halo of plane P (rows j0-H .. j0+TY+H-1, columns k0-H ..
// k0+TX+H-1, periodic) into t: 16-byte chunks when n3 % 4 == 0.
template <int TY>
__device__ __forceinline__ void stage_async(float (*t)[TW], const float* P, int j0, int k0,
                                            const FdGeo& g) {
  const int tid = threadIdx.y * TX + threadIdx.x;
  if ((g.n3 & 3) == 0) {
    constexpr int CH = TW / 4;  // 10 chunks per row
    for (int c = tid; c < (TY + 2 * H) * CH; c += TX * TY) {
      const int y = c / CH, x4 = c - y * CH;
      const float* R = P + size_t(wrap_row<TY>(j0 + y - H, g.n2)) * g.n3;
      fd_cp16(&t[y][4 * x4], R + wrap_col(k0 - H + 4 * x4, g.n3));
    }
  } else {
    for (int c = tid; c < (TY + 2 * H) * TW; c += TX * TY) {
      const int y = c / TW, x = c - y * TW;
      const float* R = P + size_t(wrap_row<TY>(j0 + y - H, g.n2)) * g.n3;
      fd_cp4(&t[y][x], R + wrap_col(k0 - H + x, g.n3));
    }
  }
}

template <bool DIST, bool DIV, int TY, int FD_CH>
__global__ void __launch_bounds__(TX* TY) k_fd_m(FdGeo g, const float* __restrict__ f,
                                                 const float* __restrict__ lo,
                                                 const float* __restrict__ hi, FdW w, float h1,
                                                 float h2, float h3, float* __restrict__ out) {
  // grad: f scalar; ring holds f. div: f = v (3 comps): the window follows v1,
  // the rings hold v2 (x2 derivative) and v3 (x3 derivative).
  constexpr int NR = DIV ? 2 : 1;
  __shared__ __align__(16) float t[NR][FD_RING][TY + 2 * H][TW];
  const size_t N = size_t(g.n1l) * g.plane;
  const int k0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int i0 = blockIdx.z * FD_CH, i1 = min(i0 + FD_CH, g.n1l);
  const int k = k0 + threadIdx.x, j = j0 + threadIdx.y;
  const bool valid = k < g.n3 && j < g.n2;
  const size_t off = valid ? size_t(j) * g.n3 + k : 0;
  auto ring_src = [&](int r, int i) -> const float* {
    if constexpr (DIV)
      return f + size_t(r + 1) * N + size_t(i) * g.plane;
    else
      return fd_plane<DIST>(f, lo, hi, i, g);
  };
  // prologue: planes i0, i0+1 in flight
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    if (i0 + d < i1)
#pragma unroll
      for (int r = 0; r < NR; ++r) stage_async<TY>(t[r][d], ring_src(r, i0 + d), j0, k0, g);
    fd_commit();
  }
  float win[2 * H + 1];
#pragma unroll
  for (int q = 0; q <= 2 * H; ++q)
    win[q] = valid ? __ldg(fd_plane<DIST>(f, lo, hi, i0 - H + q, g) + off) : 0.f;
  float nxt = (valid && i0 + 1 < i1) ? __ldg(fd_plane<DIST>(f, lo, hi, i0 + H + 1, g) + off) : 0.f;
  for (int i = i0; i < i1; ++i) {
    const int b = (i - i0) % FD_RING;
    fd_wait<1>();     // plane i landed (i+1 may still be in flight)
    __syncthreads();  // ... for every thread; ring slot (i+2) % 3 is free
    if (i + 2 < i1)
#pragma unroll
      for (int r = 0; r < NR; ++r)
        stage_async<TY>(t[r][(i + 2 - i0) % FD_RING], ring_src(r, i + 2), j0, k0, g);
    fd_commit();
    const float nxt2 =
        (valid && i + 2 < i1) ? __ldg(fd_plane<DIST>(f, lo, hi, i + H + 2, g) + off) : 0.f;
    if (valid) {
      const int x = threadIdx.x + H, y = threadIdx.y + H;
      float a3 = 0.f, a2 = 0.f, a1 = 0.f;
#pragma unroll
      for (int q = 1; q <= 4; ++q) {
        a3 += w.c[q - 1] * (t[NR - 1][b][y][x + q] - t[NR - 1][b][y][x - q]);
        a2 += w.c[q - 1] * (t[0][b][y + q][x] - t[0][b][y - q][x]);
      }
#pragma unroll
      for (int q = 1; q <= 4; ++q) a1 += w.c[q - 1] * (win[H + q] - win[H - q]);
      const size_t p = size_t(i) * g.plane + off;
      if constexpr (DIV) {
        float o = a1 * h1;  // out = d1 v1; += d2 v2; += d3 v3 (fd.cpp:171-177)
        o += a2 * h2;
        o += a3 * h3;
        out[p] = o;
      } else {
        out[p] = a1 * h1;
        out[N + p] = a2 * h2;
        out[2 * N + p] = a3 * h3;
      }
    }
#pragma unroll
    for (int q = 0; q < 2 * H; ++q) win[q] = win[q + 1];
    win[2 * H] = nxt;
    nxt = nxt2;
  }
  fd_wait<0>();
}

// Launch k_fd_m: 32 x 8 columns, 16 planes per CTA (measured best of
// 4/8/16 rows x 16/32/64 planes at 256^3).
template <bool DIST, bool DIV>
void launch_fd(vreg_ctx ctx, const Slab& s, const FdGeo& g, const float* f, const float* lo,
               const float* hi, float h1, float h2, float h3, float* out) {
  constexpr int ty = 8, ch = 16;
  const dim3 grid((s.n3 + TX - 1) / TX, (s.n2 + ty - 1) / ty, (s.n1l + ch - 1) / ch),
      block(TX, ty);
  k_fd_m<DIST, DIV, ty, ch><<<grid, block, 0, ctx->stream>>>(g, f, lo, hi, fd_weights(), h1, h2,
                                                             h3, out);
}

FdGeo fd_geo(const Slab& s) {
  FdGeo g;
  g.n1 = s.n1;
  g.n1l = s.n1l;
  g.n2 = s.n2;
  g.n3 = s.n3;
  g.plane = s.plane();
  return g;
}

void check_fd(const Slab& s) {
  require(s.n1 >= 9 && s.n2 >= 9 && s.n3 >= 9, VREG_EDIM, "fd kernels need grid sizes >= 9");
}

}  // namespace

}  // namespace vb

using namespace vb;

extern "C" {

int vreg_fd_grad(vreg_ctx ctx, const vreg_grid* gr, const float* f, float* out3) {
  return guard([&] {
    Slab s = slab_of(ctx, gr);
    check_fd(s);
    const bool dist = ctx->nranks > 1;
    Ghosts gh;
    if (dist) {
      require(s.n1l >= H, VREG_ECONFIG, "slab width below the FD ghost width 4");
      gh = halo_exchange(ctx, s, f, H, "fd_ghost", T_GHOST, C_GHOST_FD);
    }
    Timed t(ctx, T_FD, "fd_grad");
    const FdGeo g = fd_geo(s);
    const float h1 = float(1.0 / s.h(0)), h2 = float(1.0 / s.h(1)), h3 = float(1.0 / s.h(2));
    if (dist)
      launch_fd<true, false>(ctx, s, g, f, gh.lo, gh.hi, h1, h2, h3, out3);
    else
      launch_fd<false, false>(ctx, s, g, f, nullptr, nullptr, h1, h2, h3, out3);
    count_launch(ctx);
    check_launch();
  });
}

int vreg_fd_div(vreg_ctx ctx, const vreg_grid* gr, const float* v3, float* out) {
  return guard([&] {
    Slab s = slab_of(ctx, gr);
    check_fd(s);
    const bool dist = ctx->nranks > 1;
    Ghosts gh;
    if (dist) {
      require(s.n1l >= H, VREG_ECONFIG, "slab width below the FD ghost width 4");
      gh = halo_exchange(ctx, s, v3, H, "fd_ghost", T_GHOST, C_GHOST_FD);
    }
    Timed t(ctx, T_FD, "fd_div");
    const FdGeo g = fd_geo(s);
    const float h1 = float(1.0 / s.h(0)), h2 = float(1.0 / s.h(1)), h3 = float(1.0 / s.h(2));
    if (dist)
      launch_fd<true, true>(ctx, s, g, v3, gh.lo, gh.hi, h1, h2, h3, out);
    else
      launch_fd<false, true>(ctx, s, g, v3, nullptr, nullptr, h1, h2, h3, out);
    count_launch(ctx);
    check_launch();
  });
}

}  // extern "C"
