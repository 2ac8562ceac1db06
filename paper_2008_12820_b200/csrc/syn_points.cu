// Synthetic inputs on device (proj/src/syn.cpp:9-44; the CPU
// cannot build them at >= 512^3) and point-query interpolation at arbitrary
// coordinates in radians (interpolate / scatter_transpose_add,
// proj/src/interp.cpp:9-108), used for the reference's interpolation
// known-answer tests (proj/tests/test_interp.cpp).
#include <cmath>

#include "common.cuh"
#include "sl_common.cuh"

namespace vb {

void bspline_prefilter(vreg_ctx ctx, const Slab& s, int ncomp, const float* in, float* out);

namespace {

__global__ void k_syn_template(int n1l, int off, int n2, int n3, double h1, double h2, double h3,
                               float* __restrict__ m0) {
  const size_t N = size_t(n1l) * n2 * n3;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x; p < N; p += stride) {
    const int k = int(p % n3), j = int((p / n3) % n2), i = int(p / (size_t(n3) * n2)) + off;
    const double s1 = sin(i * h1), s2 = sin(j * h2), s3 = sin(k * h3);
    m0[p] = float((s1 * s1 + s2 * s2 + s3 * s3) / 3.0);
  }
}

__global__ void k_syn_velocity(int n1l, int off, int n2, int n3, double h1, double h2, double h3,
                               float* __restrict__ v) {
  const size_t N = size_t(n1l) * n2 * n3;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x; p < N; p += stride) {
    const int k = int(p % n3), j = int((p / n3) % n2), i = int(p / (size_t(n3) * n2)) + off;
    const double x1 = i * h1, x2 = j * h2, x3 = k * h3;
    v[p] = float(sin(x3) * cos(x2) * sin(x2));
    v[N + p] = float(sin(x1) * cos(x3) * sin(x3));
    v[2 * N + p] = float(sin(x2) * cos(x1) * sin(x1));
  }
}

// fp64 axis split with the reference's wrap + snap (interp.cpp:9-24)
__device__ __forceinline__ void axis_split64(double x, double h, int n, int& base, float& s) {
  double u = x / h;
  u -= floor(u / double(n)) * double(n);
  if (u < 0.0) u = 0.0;
  if (u >= double(n)) u -= double(n);
  const double fl = floor(u);
  double sd = u - fl;
  base = int(fl);
  if (sd < 1e-12) {
    sd = 0.0;
  } else if (sd > 1.0 - 1e-12) {
    sd = 0.0;
    if (++base == n) base = 0;
  }
  if (base >= n) base -= n;
  s = float(sd);
}

template <int DEG>
__device__ __forceinline__ void point_stencil(const Geo& g, const double* xyz, double h1, double h2,
                                              double h3, Stencil<DEG>& st) {
  int b1, b2, b3;
  float s1, s2, s3;
  axis_split64(xyz[0], h1, g.n1, b1, s1);
  axis_split64(xyz[1], h2, g.n2, b2, s2);
  axis_split64(xyz[2], h3, g.n3, b3, s3);
  lagrange_weights<DEG>(s1, st.w1);
  lagrange_weights<DEG>(s2, st.w2);
  lagrange_weights<DEG>(s3, st.w3);
  constexpr int O0 = Basis<DEG>::O0;
#pragma unroll
  for (int o = 0; o < Basis<DEG>::NN; ++o) {
    st.p1[o] = wrap1(b1 + O0 + o, g.n1);
    st.r2[o] = wrap1(b2 + O0 + o, g.n2) * g.n3;
    st.c3[o] = wrap1(b3 + O0 + o, g.n3);
  }
}

__global__ void k_nan_check(int64_t m, const double* __restrict__ xyz, int* flag) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < 3 * m;
       q += int64_t(gridDim.x) * blockDim.x)
    if (isnan(xyz[q])) atomicOr(flag, 1);
}

template <int DEG>
__global__ void k_interp_points(Geo g, const float* __restrict__ f, const double* __restrict__ xyz,
                                int64_t m, double h1, double h2, double h3,
                                float* __restrict__ out) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < m;
       q += int64_t(gridDim.x) * blockDim.x) {
    Stencil<DEG> st;
    point_stencil<DEG>(g, xyz + 3 * q, h1, h2, h3, st);
    SrcField<false> src{f, nullptr, nullptr, 0};
    out[q] = st.gather(g, src);
  }
}

template <int DEG>
__global__ void k_scatter_points(Geo g, float* __restrict__ acc, const double* __restrict__ xyz,
                                 const float* __restrict__ z, int64_t m, double h1, double h2,
                                 double h3) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < m;
       q += int64_t(gridDim.x) * blockDim.x) {
    Stencil<DEG> st;
    point_stencil<DEG>(g, xyz + 3 * q, h1, h2, h3, st);
    DstField<false> dst{acc, nullptr, nullptr, 0};
    st.scatter(g, dst, z[q]);
  }
}

Geo point_geo(const Slab& s) {
  Geo g;
  g.n1 = s.n1;
  g.n1l = s.n1l;
  g.n2 = s.n2;
  g.n3 = s.n3;
  g.plane = s.plane();
  g.N = s.local();
  return g;
}

void check_points(vreg_ctx ctx, const double* xyz, int64_t m, int degree) {
  require(degree == 1 || degree == 3 || degree == VREG_INTERP_BSPLINE3, VREG_EPARAM,
          "interpolation degree must be 1, 3 or 4 (cubic B-spline)");
  require(ctx->nranks == 1, VREG_ECONFIG, "point queries are single-rank");
  int* flag = static_cast<int*>(workspace(ctx, "nan_flag", sizeof(int)));
  VB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  if (m > 0) {
    k_nan_check<<<blocks_for(size_t(3 * m), 256), 256, 0, ctx->stream>>>(m, xyz, flag);
    count_launch(ctx);
    check_launch();
  }
  int h = 0;
  VB_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  VB_CUDA(cudaStreamSynchronize(ctx->stream));
  require(h == 0, VREG_EINPUT, "NaN query coordinate");
}

}  // namespace

}  // namespace vb

using namespace vb;

extern "C" {

int vreg_syn_template(vreg_ctx ctx, const vreg_grid* g, float* m0) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    k_syn_template<<<blocks_for(s.local(), 256), 256, 0, ctx->stream>>>(
        s.n1l, s.off, s.n2, s.n3, s.h(0), s.h(1), s.h(2), m0);
    count_launch(ctx);
    check_launch();
  });
}

int vreg_syn_velocity(vreg_ctx ctx, const vreg_grid* g, float* v3) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    k_syn_velocity<<<blocks_for(s.local(), 256), 256, 0, ctx->stream>>>(
        s.n1l, s.off, s.n2, s.n3, s.h(0), s.h(1), s.h(2), v3);
    count_launch(ctx);
    check_launch();
  });
}

int vreg_interp_points(vreg_ctx ctx, const vreg_grid* gr, const float* f, const double* xyz,
                       int64_t m, int degree, float* out) {
  return guard([&] {
    Slab s = slab_of(ctx, gr);
    check_points(ctx, xyz, m, degree);
    if (m == 0) return;
    const Geo g = point_geo(s);
    if (degree == VREG_INTERP_BSPLINE3) {  // evaluate the B-spline coefficients
      float* c = static_cast<float*>(workspace(ctx, "bs_points", s.local() * sizeof(float)));
      bspline_prefilter(ctx, s, 1, f, c);
      k_interp_points<4><<<blocks_for(size_t(m), 256), 256, 0, ctx->stream>>>(
          g, c, xyz, m, s.h(0), s.h(1), s.h(2), out);
    } else if (degree == 3)
      k_interp_points<3><<<blocks_for(size_t(m), 256), 256, 0, ctx->stream>>>(
          g, f, xyz, m, s.h(0), s.h(1), s.h(2), out);
    else
      k_interp_points<1><<<blocks_for(size_t(m), 256), 256, 0, ctx->stream>>>(
          g, f, xyz, m, s.h(0), s.h(1), s.h(2), out);
    count_launch(ctx);
    check_launch();
  });
}

int vreg_scatter_points(vreg_ctx ctx, const vreg_grid* gr, const double* xyz, const float* z,
                        int64_t m, int degree, float* acc) {
  return guard([&] {
    Slab s = slab_of(ctx, gr);
    check_points(ctx, xyz, m, degree);
    if (m == 0) return;
    const Geo g = point_geo(s);
    if (degree == VREG_INTERP_BSPLINE3) {  // acc += P B^T z (P the symmetric prefilter)
      float* t = static_cast<float*>(workspace(ctx, "bs_points", s.local() * sizeof(float)));
      VB_CUDA(cudaMemsetAsync(t, 0, s.local() * sizeof(float), ctx->stream));
      k_scatter_points<4><<<blocks_for(size_t(m), 256), 256, 0, ctx->stream>>>(
          g, t, xyz, z, m, s.h(0), s.h(1), s.h(2));
      count_launch(ctx);
      check_launch();
      bspline_prefilter(ctx, s, 1, t, t);
      vreg_grid gg{s.n1, s.n2, s.n3, s.nt};
      const int st = vreg_axpy(ctx, &gg, 1, 1.0, t, acc);
      require(st == VREG_OK, st, "axpy failed");
      return;
    }
    if (degree == 3)
      k_scatter_points<3><<<blocks_for(size_t(m), 256), 256, 0, ctx->stream>>>(
          g, acc, xyz, z, m, s.h(0), s.h(1), s.h(2));
    else
      k_scatter_points<1><<<blocks_for(size_t(m), 256), 256, 0, ctx->stream>>>(
          g, acc, xyz, z, m, s.h(0), s.h(1), s.h(2));
    count_launch(ctx);
    check_launch();
  });
}

}  // extern "C"
