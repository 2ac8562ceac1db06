// Pointwise field arithmetic and plane-folded fp64 reductions
// (proj/include/vreg/field.hpp:67-188). Streaming kernels: 128-bit
// vectorised grid-stride loops sized to the SM count.
#include <cmath>

#include "common.cuh"

namespace vb {

namespace {

constexpr unsigned kThreads = 256;

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <class Op>
__global__ void k_map1(size_t n4, size_t n, float* __restrict__ y, Op op) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  float4* y4 = reinterpret_cast<float4*>(y);
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 v = y4[i];
    v.x = op(v.x); v.y = op(v.y); v.z = op(v.z); v.w = op(v.w);
    y4[i] = v;
  }
  for (size_t i = 4 * n4 + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = op(y[i]);
}

template <class Op>
__global__ void k_map2(size_t n4, size_t n, const float* __restrict__ x, float* __restrict__ y,
                       Op op) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4* y4 = reinterpret_cast<float4*>(y);
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 a = x4[i];
    float4 b = y4[i];
    b.x = op(a.x, b.x); b.y = op(a.y, b.y); b.z = op(a.z, b.z); b.w = op(a.w, b.w);
    y4[i] = b;
  }
  for (size_t i = 4 * n4 + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = op(x[i], y[i]);
}

template <class Op>
__global__ void k_map3(size_t n4, size_t n, const float* __restrict__ a,
                       const float* __restrict__ b, float* __restrict__ out, Op op) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  float4* o4 = reinterpret_cast<float4*>(out);
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 x = a4[i], y = b4[i];
    o4[i] = make_float4(op(x.x, y.x), op(x.y, y.y), op(x.z, y.z), op(x.w, y.w));
  }
  for (size_t i = 4 * n4 + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = op(a[i], b[i]);
}

// out = v1 w1 + v2 w2 + v3 w3 (field.hpp:118-127, same association)
__global__ void k_dot3(size_t n, const float* __restrict__ v, const float* __restrict__ w,
                       float* __restrict__ out) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = v[i] * w[i] + v[n + i] * w[n + i] + v[2 * n + i] * w[2 * n + i];
}

// out_c += a * s * w_c (field.hpp:130-141)
__global__ void k_axpy_sv(size_t n, float a, const float* __restrict__ s,
                          const float* __restrict__ w, float* __restrict__ out) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float as = a * s[i];
    out[i] += as * w[i];
    out[n + i] += as * w[n + i];
    out[2 * n + i] += as * w[2 * n + i];
  }
}

// Per-(component, plane, chunk) fp64 partial sums; fixed association so the
// result depends only on the plane's data (p-independent).
template <bool kMax>
__global__ void k_plane_partials(const float* __restrict__ a, const float* __restrict__ b,
                                 size_t plane, int chunks, size_t chunk_len,
                                 double* __restrict__ partials) {
  const size_t blk = blockIdx.x;  // (plane_index * chunks + chunk) over all comps
  const size_t pl = blk / chunks;
  const size_t ch = blk % chunks;
  const size_t beg = pl * plane + ch * chunk_len;
  size_t end = beg + chunk_len;
  if (end > (pl + 1) * plane) end = (pl + 1) * plane;
  double acc = 0.0;
  if (((beg | end) & 3) == 0 && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0) {
    // 16-byte lanes (uniform per block): same element set, 4x fewer loads
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    for (size_t i = beg / 4 + threadIdx.x; i < end / 4; i += blockDim.x) {
      const float4 x = a4[i];
      if (kMax) {
        acc = fmax(fmax(fmax(fmax(acc, fabs(double(x.x))), fabs(double(x.y))), fabs(double(x.z))),
                   fabs(double(x.w)));
      } else {
        const float4 y = b4[i];
        acc += double(x.x) * double(y.x);
        acc += double(x.y) * double(y.y);
        acc += double(x.z) * double(y.z);
        acc += double(x.w) * double(y.w);
      }
    }
  } else {
    for (size_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
      if (kMax) {
        acc = fmax(acc, fabs(double(a[i])));
      } else {
        acc += double(a[i]) * double(b[i]);
      }
    }
  }
  __shared__ double sh[kThreads];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (unsigned s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      sh[threadIdx.x] = kMax ? fmax(sh[threadIdx.x], sh[threadIdx.x + s])
                             : sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blk] = sh[0];
}

void map_fill(vreg_ctx ctx, size_t n, float* x, float v) {
  auto op = [v] __device__(float) { return v; };
  if (aligned16(x)) {
    k_map1<<<blocks_for(n / 4, kThreads), kThreads, 0, ctx->stream>>>(n / 4, n, x, op);
  } else {
    k_map1<<<blocks_for(n, kThreads), kThreads, 0, ctx->stream>>>(0, n, x, op);
  }
  count_launch(ctx);
  check_launch();
}

}  // namespace

int chunks_per_plane(const Slab& s) {
  const size_t chunk = 8192;
  return int((s.plane() + chunk - 1) / chunk);
}

void plane_partials(vreg_ctx ctx, const Slab& s, int ncomp, const float* a, const float* b,
                    bool is_max, double* d_partials, int chunks) {
  const size_t chunk_len = (s.plane() + chunks - 1) / chunks;
  const unsigned blocks = unsigned(size_t(ncomp) * s.n1l * chunks);
  if (is_max)
    k_plane_partials<true><<<blocks, kThreads, 0, ctx->stream>>>(a, b, s.plane(), chunks,
                                                                 chunk_len, d_partials);
  else
    k_plane_partials<false><<<blocks, kThreads, 0, ctx->stream>>>(a, b, s.plane(), chunks,
                                                                  chunk_len, d_partials);
  count_launch(ctx);
  check_launch();
}

// Fold partials of ncomp components: per component, planes in global order,
// each plane's chunks in order (field.hpp:150-175).
double fold_partials(vreg_ctx ctx, const Slab& s, const double* d_local, int chunks, int ncomp,
                     bool is_max) {
  const size_t per_comp_local = size_t(s.n1l) * chunks;
  const size_t per_comp_global = size_t(s.n1) * chunks;
  const double* src = d_local;
  if (ctx->nranks > 1) {
    double* g = static_cast<double*>(
        workspace(ctx, "red_global", sizeof(double) * per_comp_global * ncomp));
    for (int c = 0; c < ncomp; ++c)
      allgather_partials(ctx, s, d_local + c * per_comp_local, g + c * per_comp_global,
                         size_t(chunks));
    src = g;
  }
  double* h = pinned(ctx, per_comp_global * ncomp);
  VB_CUDA(cudaMemcpyAsync(h, src, sizeof(double) * per_comp_global * ncomp,
                          cudaMemcpyDeviceToHost, ctx->stream));
  VB_CUDA(cudaStreamSynchronize(ctx->stream));
  double total = 0.0;
  for (int c = 0; c < ncomp; ++c) {
    double comp = 0.0;
    for (int i = 0; i < s.n1; ++i) {
      double pl = 0.0;
      for (int k = 0; k < chunks; ++k) {
        const double v = h[size_t(c) * per_comp_global + size_t(i) * chunks + k];
        pl = is_max ? std::fmax(pl, v) : pl + v;
      }
      comp = is_max ? std::fmax(comp, pl) : comp + pl;
    }
    if (is_max)
      total = std::fmax(total, comp);
    else
      total += comp * (s.h(0) * s.h(1) * s.h(2));
  }
  return total;
}

double reduce(vreg_ctx ctx, const Slab& s, int ncomp, const float* a, const float* b,
              bool is_max) {
  const int chunks = chunks_per_plane(s);
  double* d = static_cast<double*>(
      workspace(ctx, "red_local", sizeof(double) * size_t(ncomp) * s.n1l * chunks));
  plane_partials(ctx, s, ncomp, a, b, is_max, d, chunks);
  return fold_partials(ctx, s, d, chunks, ncomp, is_max);
}

}  // namespace vb

using namespace vb;

extern "C" {

int vreg_fill(vreg_ctx ctx, const vreg_grid* g, int ncomp, float* x, double value) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    const size_t n = size_t(ncomp) * s.local();
    if (value == 0.0) {
      VB_CUDA(cudaMemsetAsync(x, 0, n * sizeof(float), ctx->stream));
    } else {
      map_fill(ctx, n, x, float(value));
    }
  });
}

int vreg_copy(vreg_ctx ctx, const vreg_grid* g, int ncomp, const float* x, float* y) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    VB_CUDA(cudaMemcpyAsync(y, x, size_t(ncomp) * s.local() * sizeof(float),
                            cudaMemcpyDeviceToDevice, ctx->stream));
  });
}

#define VB_MAP2(x, y, n, OP)                                                          \
  do {                                                                                \
    auto op_ = OP;                                                                    \
    if (aligned16(x) && aligned16(y))                                                 \
      k_map2<<<blocks_for((n) / 4, kThreads), kThreads, 0, ctx->stream>>>((n) / 4, n, \
                                                                          x, y, op_); \
    else                                                                              \
      k_map2<<<blocks_for(n, kThreads), kThreads, 0, ctx->stream>>>(0, n, x, y, op_); \
    count_launch(ctx);                                                                \
    check_launch();                                                                   \
  } while (0)

int vreg_axpy(vreg_ctx ctx, const vreg_grid* g, int ncomp, double a, const float* x, float* y) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    const size_t n = size_t(ncomp) * s.local();
    const float af = float(a);
    VB_MAP2(x, y, n, [af] __device__(float xv, float yv) { return yv + af * xv; });
  });
}

int vreg_aypx(vreg_ctx ctx, const vreg_grid* g, int ncomp, double a, const float* x, float* y) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    const size_t n = size_t(ncomp) * s.local();
    const float af = float(a);
    // scale(p, beta) then axpy(1, z, p) (pcg.hpp:90-91), same rounding order
    VB_MAP2(x, y, n, [af] __device__(float xv, float yv) { return yv * af + xv; });
  });
}

int vreg_scale(vreg_ctx ctx, const vreg_grid* g, int ncomp, float* x, double a) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    const size_t n = size_t(ncomp) * s.local();
    const float af = float(a);
    auto op = [af] __device__(float v) { return v * af; };
    if (aligned16(x))
      k_map1<<<blocks_for(n / 4, kThreads), kThreads, 0, ctx->stream>>>(n / 4, n, x, op);
    else
      k_map1<<<blocks_for(n, kThreads), kThreads, 0, ctx->stream>>>(0, n, x, op);
    count_launch(ctx);
    check_launch();
  });
}

int vreg_sub(vreg_ctx ctx, const vreg_grid* g, int ncomp, const float* a, const float* b,
             float* out) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    const size_t n = size_t(ncomp) * s.local();
    auto op = [] __device__(float x, float y) { return x + (-1.0f) * y; };
    if (aligned16(a) && aligned16(b) && aligned16(out))
      k_map3<<<blocks_for(n / 4, kThreads), kThreads, 0, ctx->stream>>>(n / 4, n, a, b, out, op);
    else
      k_map3<<<blocks_for(n, kThreads), kThreads, 0, ctx->stream>>>(0, n, a, b, out, op);
    count_launch(ctx);
    check_launch();
  });
}

int vreg_hadamard(vreg_ctx ctx, const vreg_grid* g, const float* a, const float* b, float* out) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    const size_t n = s.local();
    auto op = [] __device__(float x, float y) { return x * y; };
    if (aligned16(a) && aligned16(b) && aligned16(out))
      k_map3<<<blocks_for(n / 4, kThreads), kThreads, 0, ctx->stream>>>(n / 4, n, a, b, out, op);
    else
      k_map3<<<blocks_for(n, kThreads), kThreads, 0, ctx->stream>>>(0, n, a, b, out, op);
    count_launch(ctx);
    check_launch();
  });
}

int vreg_pointwise_dot(vreg_ctx ctx, const vreg_grid* g, const float* v3, const float* w3,
                       float* out) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    k_dot3<<<blocks_for(s.local(), kThreads), kThreads, 0, ctx->stream>>>(s.local(), v3, w3, out);
    count_launch(ctx);
    check_launch();
  });
}

int vreg_axpy_scaled_vector(vreg_ctx ctx, const vreg_grid* g, double a, const float* sf,
                            const float* w3, float* out3) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    k_axpy_sv<<<blocks_for(s.local(), kThreads), kThreads, 0, ctx->stream>>>(
        s.local(), float(a), sf, w3, out3);
    count_launch(ctx);
    check_launch();
  });
}

int vreg_inner(vreg_ctx ctx, const vreg_grid* g, int ncomp, const float* a, const float* b,
               double* out) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    *out = reduce(ctx, s, ncomp, a, b, false);
  });
}

int vreg_max_abs(vreg_ctx ctx, const vreg_grid* g, int ncomp, const float* x, double* out) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    *out = reduce(ctx, s, ncomp, x, x, true);
  });
}

}  // extern "C"
