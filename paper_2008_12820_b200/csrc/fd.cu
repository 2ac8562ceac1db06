// 8th-order periodic finite differences (proj/src/fd.cpp:7-179).
//
// All three axes use the paired antisymmetric form sum_j c_j (f_{+j} - f_{-j})
// (fd.cpp:60-78; the reference uses it on x1 and an unpaired 9-tap sum with
// a ~3e-16 centre weight on x2/x3, fd.cpp:80-125 -- identical to fp64
// round-off). Weights come from the same Fornberg
// recursion (fd.cpp:7-48), evaluated in fp64 and rounded once.
//
// Tiling: a CTA owns a 32 (x3) x 8 (x2) tile of one x1 plane and stages the
// tile plus its x2/x3 halo of 4 in shared memory; x1 neighbours stream from
// L2 (each plane is re-read by the 8 CTAs that need it, so HBM sees ~1x).
#include <cmath>
#include <vector>

#include "common.cuh"

namespace vb {

namespace {

constexpr int TX = 32, TY = 8, H = 4;

std::vector<double> fornberg(int half_width, int deriv) {
  const int n = 2 * half_width;
  const int m = deriv;
  std::vector<double> x(size_t(n) + 1);
  for (int i = 0; i <= n; ++i) x[size_t(i)] = double(i - half_width);
  std::vector<std::vector<double>> c(size_t(n) + 1, std::vector<double>(size_t(m) + 1, 0.0));
  double c1 = 1.0, c4 = x[0];
  c[0][0] = 1.0;
  for (int i = 1; i <= n; ++i) {
    const int mn = i < m ? i : m;
    double c2 = 1.0;
    const double c5 = c4;
    c4 = x[size_t(i)];
    for (int j = 0; j <= i - 1; ++j) {
      const double c3 = x[size_t(i)] - x[size_t(j)];
      c2 *= c3;
      if (j == i - 1) {
        for (int k = mn; k >= 1; --k)
          c[size_t(i)][size_t(k)] =
              c1 * (k * c[size_t(i) - 1][size_t(k) - 1] - c5 * c[size_t(i) - 1][size_t(k)]) / c2;
        c[size_t(i)][0] = -c1 * c5 * c[size_t(i) - 1][0] / c2;
      }
      for (int k = mn; k >= 1; --k)
        c[size_t(j)][size_t(k)] =
            (c4 * c[size_t(j)][size_t(k)] - k * c[size_t(j)][size_t(k) - 1]) / c3;
      c[size_t(j)][0] = c4 * c[size_t(j)][0] / c3;
    }
    c1 = c2;
  }
  std::vector<double> out(size_t(n) + 1);
  for (int i = 0; i <= n; ++i) out[size_t(i)] = c[size_t(i)][size_t(m)];
  return out;
}

struct FdW {
  float c[4];  // c_j for j = 1..4, unit spacing
};

FdW fd_weights() {
  static const FdW w = [] {
    auto d = fornberg(4, 1);
    FdW r;
    for (int j = 1; j <= 4; ++j) r.c[j - 1] = float(d[size_t(4 + j)]);
    return r;
  }();
  return w;
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

// Stage tile (TY+2H) x (TX+2H) of plane P into smem with x2/x3 wrap.
__device__ __forceinline__ void stage_tile(float (*t)[TX + 2 * H], const float* P, int j0, int k0,
                                           const FdGeo& g) {
  for (int y = threadIdx.y; y < TY + 2 * H; y += TY) {
    int jj = (j0 + y - H) % g.n2;
    jj = jj < 0 ? jj + g.n2 : jj;
    const float* R = P + size_t(jj) * g.n3;
    for (int x = threadIdx.x; x < TX + 2 * H; x += TX) {
      int kk = (k0 + x - H) % g.n3;
      kk = kk < 0 ? kk + g.n3 : kk;
      t[y][x] = __ldg(R + kk);
    }
  }
}

template <bool DIST>
__global__ void __launch_bounds__(TX* TY) k_fd_grad(FdGeo g, const float* __restrict__ f,
                                                    const float* __restrict__ lo,
                                                    const float* __restrict__ hi, FdW w,
                                                    float h1, float h2, float h3,
                                                    float* __restrict__ out) {
  __shared__ float t[TY + 2 * H][TX + 2 * H];
  const int k0 = blockIdx.x * TX, j0 = blockIdx.y * TY, i = blockIdx.z;
  stage_tile(t, fd_plane<DIST>(f, lo, hi, i, g), j0, k0, g);
  __syncthreads();
  const int k = k0 + threadIdx.x, j = j0 + threadIdx.y;
  if (k >= g.n3 || j >= g.n2) return;
  const int x = threadIdx.x + H, y = threadIdx.y + H;
  float a3 = 0.f, a2 = 0.f, a1 = 0.f;
#pragma unroll
  for (int q = 1; q <= 4; ++q) {
    a3 += w.c[q - 1] * (t[y][x + q] - t[y][x - q]);
    a2 += w.c[q - 1] * (t[y + q][x] - t[y - q][x]);
  }
  const size_t off = size_t(j) * g.n3 + k;
#pragma unroll
  for (int q = 1; q <= 4; ++q)
    a1 += w.c[q - 1] * (__ldg(fd_plane<DIST>(f, lo, hi, i + q, g) + off) -
                        __ldg(fd_plane<DIST>(f, lo, hi, i - q, g) + off));
  const size_t N = size_t(g.n1l) * g.plane;
  const size_t p = size_t(i) * g.plane + off;
  out[p] = a1 * h1;
  out[N + p] = a2 * h2;
  out[2 * N + p] = a3 * h3;
}

template <bool DIST>
__global__ void __launch_bounds__(TX* TY) k_fd_div(FdGeo g, const float* __restrict__ v,
                                                   const float* __restrict__ lo,
                                                   const float* __restrict__ hi, FdW w,
                                                   float h1, float h2, float h3,
                                                   float* __restrict__ out) {
  __shared__ float t2[TY + 2 * H][TX + 2 * H];
  __shared__ float t3[TY + 2 * H][TX + 2 * H];
  const size_t N = size_t(g.n1l) * g.plane;
  const int k0 = blockIdx.x * TX, j0 = blockIdx.y * TY, i = blockIdx.z;
  stage_tile(t2, v + N + size_t(i) * g.plane, j0, k0, g);
  stage_tile(t3, v + 2 * N + size_t(i) * g.plane, j0, k0, g);
  __syncthreads();
  const int k = k0 + threadIdx.x, j = j0 + threadIdx.y;
  if (k >= g.n3 || j >= g.n2) return;
  const int x = threadIdx.x + H, y = threadIdx.y + H;
  float a3 = 0.f, a2 = 0.f, a1 = 0.f;
#pragma unroll
  for (int q = 1; q <= 4; ++q) {
    a3 += w.c[q - 1] * (t3[y][x + q] - t3[y][x - q]);
    a2 += w.c[q - 1] * (t2[y + q][x] - t2[y - q][x]);
  }
  const size_t off = size_t(j) * g.n3 + k;
#pragma unroll
  for (int q = 1; q <= 4; ++q)
    a1 += w.c[q - 1] * (__ldg(fd_plane<DIST>(v, lo, hi, i + q, g) + off) -
                        __ldg(fd_plane<DIST>(v, lo, hi, i - q, g) + off));
  // out = d1 v1; out += d2 v2; out += d3 v3 (fd.cpp:171-177)
  float o = a1 * h1;
  o += a2 * h2;
  o += a3 * h3;
  out[size_t(i) * g.plane + off] = o;
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
    const dim3 grid((s.n3 + TX - 1) / TX, (s.n2 + TY - 1) / TY, s.n1l), block(TX, TY);
    const float h1 = float(1.0 / s.h(0)), h2 = float(1.0 / s.h(1)), h3 = float(1.0 / s.h(2));
    if (dist)
      k_fd_grad<true><<<grid, block, 0, ctx->stream>>>(g, f, gh.lo, gh.hi, fd_weights(), h1, h2,
                                                       h3, out3);
    else
      k_fd_grad<false><<<grid, block, 0, ctx->stream>>>(g, f, nullptr, nullptr, fd_weights(), h1,
                                                        h2, h3, out3);
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
    const dim3 grid((s.n3 + TX - 1) / TX, (s.n2 + TY - 1) / TY, s.n1l), block(TX, TY);
    const float h1 = float(1.0 / s.h(0)), h2 = float(1.0 / s.h(1)), h3 = float(1.0 / s.h(2));
    if (dist)
      k_fd_div<true><<<grid, block, 0, ctx->stream>>>(g, v3, gh.lo, gh.hi, fd_weights(), h1, h2,
                                                      h3, out);
    else
      k_fd_div<false><<<grid, block, 0, ctx->stream>>>(g, v3, nullptr, nullptr, fd_weights(), h1,
                                                       h2, h3, out);
    count_launch(ctx);
    check_launch();
  });
}

}  // extern "C"
