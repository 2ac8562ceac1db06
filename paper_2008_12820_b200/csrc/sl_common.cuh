// Device-side semi-Lagrangian building blocks: per-axis split of a departure
// displacement, Lagrange weights, slab-aware field accessors and the
// tensor-product gather/scatter with the reference's accumulation order
// (proj/src/interp.cpp:9-68, proj/include/vreg/interp.hpp:47-61).
//
// Characteristics are stored as displacements d (grid units) of the
// departure point from its node, so the stencil base is node + floor(d)
// and the fraction d - floor(d) is exact in fp32 (no absolute-coordinate
// rounding, which would cost ~1e-4 grid units at 1024^3 in fp32).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace vb {

struct Geo {
  int n1;   // global planes (wrap modulus on one rank)
  int n1l;  // local planes
  int n2, n3;
  size_t plane;  // n2 * n3
  size_t N;      // local points
};

// One fixed-point contribution into an int32 accumulator field. Packed mode
// (n3 % 4 == 0): adjacent cells (2m, 2m+1) share one 64-bit word updated as
// lo + 2^32 hi -- exact in int64, decoded per pair once every cell's total
// fits int32 -- so the tile flush needs half the atomics. Every writer of a
// field must use the same mode.
__device__ __forceinline__ void fixed_add(int* p, int v, bool packed) {
  if (packed) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    unsigned long long* q = reinterpret_cast<unsigned long long*>(a & ~uintptr_t(7));
    const long long w = (a & 4) ? (static_cast<long long>(v) << 32) : static_cast<long long>(v);
    atomicAdd(q, static_cast<unsigned long long>(w));
  } else {
    atomicAdd(p, v);
  }
}
__device__ __forceinline__ bool fixed_packed(const Geo& g) { return (g.n3 & 3) == 0; }

// base = q + floor(d), s = d - floor(d) in [0, 1]. s rounds to 1 only for
// tiny negative d; the cubic / linear weights at s = 1 are exactly
// (0, 0, 1, 0) / (0, 1), i.e. the node value, so no snap branch is needed
// (and k_tile_boxes' reach, floor(d), stays the same).
__device__ __forceinline__ void split_axis(float d, int q, int& base, float& s) {
  const float fd = floorf(d);
  s = d - fd;
  base = q + int(fd);
}

__device__ __forceinline__ int wrap_mod(int b, int n) {
  b %= n;
  return b < 0 ? b + n : b;
}

__device__ __forceinline__ int wrap1(int b, int n) {
  return b < 0 ? b + n : (b >= n ? b - n : b);
}

// Interpolation bases, by template DEG: 1 linear, 3 cubic Lagrange (the
// reference's two, interp.cpp:26-35), 4 cubic B-spline (B200 extension named
// by the north star; evaluated on prefiltered coefficients, spline.cu).
// Both cubic bases use the 4 nodes {-1, 0, 1, 2} around floor(x).
template <int DEG>
struct Basis {
  static constexpr int NN = DEG == 1 ? 2 : 4;    // taps per axis
  static constexpr int O0 = DEG == 1 ? 0 : -1;   // offset of the first tap
};

template <int DEG>
__device__ __forceinline__ void lagrange_weights(float s, float* w) {
  if constexpr (DEG == 4) {
    // cubic B-spline: ((1-s)^3, 3s^3 - 6s^2 + 4, -3s^3 + 3s^2 + 3s + 1, s^3) / 6
    const float ms = 1.0f - s, s2 = s * s, s3 = s2 * s;
    w[0] = ms * ms * ms * (1.0f / 6.0f);
    w[1] = __fmaf_rn(3.0f, s3, __fmaf_rn(-6.0f, s2, 4.0f)) * (1.0f / 6.0f);
    w[2] = __fmaf_rn(-3.0f, s3, __fmaf_rn(3.0f, s2, __fmaf_rn(3.0f, s, 1.0f))) * (1.0f / 6.0f);
    w[3] = s3 * (1.0f / 6.0f);
  } else if constexpr (DEG == 3) {
    // factored: q = -s (1-s) / 6, r = (s+1)(2-s) / 2; w = (q (2-s), r (1-s), r s, q (s+1))
    const float ms = 1.0f - s, sp = s + 1.0f, ns2 = 2.0f - s;
    const float q = __fmul_rn(__fmul_rn(s, ms), -1.0f / 6.0f);
    const float r = __fmul_rn(__fmul_rn(sp, ns2), 0.5f);
    w[0] = __fmul_rn(q, ns2);
    w[1] = __fmul_rn(r, ms);
    w[2] = __fmul_rn(r, s);
    w[3] = __fmul_rn(q, sp);
  } else {
    w[0] = 1.0f - s;
    w[1] = s;
  }
}

// Read-only field with optional x1 ghosts (DIST) or periodic x1 wrap.
template <bool DIST>
struct SrcField {
  const float* f;
  const float* lo;
  const float* hi;
  int G;
  __device__ __forceinline__ const float* plane_ptr(int p, const Geo& g) const {
    if constexpr (DIST) {
      if (p < 0) return lo + size_t(p + G) * g.plane;
      if (p >= g.n1l) return hi + size_t(p - g.n1l) * g.plane;
      return f + size_t(p) * g.plane;
    } else {
      return f + size_t(wrap1(p, g.n1)) * g.plane;
    }
  }
};

// Accumulation target with optional x1 ghost accumulators.
template <bool DIST>
struct DstField {
  float* f;
  float* lo;
  float* hi;
  int G;
  __device__ __forceinline__ float* plane_ptr(int p, const Geo& g) const {
    if constexpr (DIST) {
      if (p < 0) return lo + size_t(p + G) * g.plane;
      if (p >= g.n1l) return hi + size_t(p - g.n1l) * g.plane;
      return f + size_t(p) * g.plane;
    } else {
      return f + size_t(wrap1(p, g.n1)) * g.plane;
    }
  }
};

// Stencil of one departure point: plane index per x1 tap (unwrapped for
// DIST, wrapped otherwise), row offsets along x2, columns along x3.
template <int DEG>
struct Stencil {
  static constexpr int NN = Basis<DEG>::NN;
  static constexpr int O0 = Basis<DEG>::O0;
  int p1[NN];
  int r2[NN];
  int c3[NN];
  float w1[NN], w2[NN], w3[NN];

  template <bool DIST>
  __device__ __forceinline__ void build(const Geo& g, int i, int j, int k, float d1, float d2,
                                        float d3) {
    int b1, b2, b3;
    float s1, s2, s3;
    split_axis(d1, i, b1, s1);
    split_axis(d2, j, b2, s2);
    split_axis(d3, k, b3, s3);
    if constexpr (!DIST) b1 = wrap_mod(b1, g.n1);
    b2 = wrap_mod(b2, g.n2);
    b3 = wrap_mod(b3, g.n3);
    lagrange_weights<DEG>(s1, w1);
    lagrange_weights<DEG>(s2, w2);
    lagrange_weights<DEG>(s3, w3);
#pragma unroll
    for (int o = 0; o < NN; ++o) {
      p1[o] = b1 + O0 + o;
      r2[o] = wrap1(b2 + O0 + o, g.n2) * g.n3;
      c3[o] = wrap1(b3 + O0 + o, g.n3);
    }
  }

  // acc1 = sum_a w1 (sum_b w2 (sum_c w3 f)) (interp.hpp:47-61)
  template <bool DIST>
  __device__ __forceinline__ float gather(const Geo& g, const SrcField<DIST>& src) const {
    float acc1 = 0.0f;
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      const float* P = src.plane_ptr(p1[a], g);
      float acc2 = 0.0f;
#pragma unroll
      for (int b = 0; b < NN; ++b) {
        const float* R = P + r2[b];
        float acc3 = 0.0f;
#pragma unroll
        for (int c = 0; c < NN; ++c) acc3 += w3[c] * __ldg(R + c3[c]);
        acc2 += w2[b] * acc3;
      }
      acc1 += w1[a] * acc2;
    }
    return acc1;
  }

  // acc[node] += w1 w2 w3 z (interp.cpp:92-108)
  template <bool DIST>
  __device__ __forceinline__ void scatter(const Geo& g, const DstField<DIST>& dst,
                                          float z) const {
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      float* P = dst.plane_ptr(p1[a], g);
      const float za = w1[a] * z;
#pragma unroll
      for (int b = 0; b < NN; ++b) {
        float* R = P + r2[b];
        const float zab = za * w2[b];
#pragma unroll
        for (int c = 0; c < NN; ++c) atomicAdd(R + c3[c], zab * w3[c]);
      }
    }
  }

  // Fixed-point variant: dst holds int32 at scale S (zS = z S); each
  // contribution rounded as the tile path does (DFMA against 1.5 * 2^52).
  template <bool DIST>
  __device__ __forceinline__ void scatter_fixed(const Geo& g, const DstField<DIST>& dst,
                                                float zS) const {
    constexpr double MAGIC = 6755399441055744.0;
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      int* P = reinterpret_cast<int*>(dst.plane_ptr(p1[a], g));
      const float za = w1[a] * zS;
#pragma unroll
      for (int b = 0; b < NN; ++b) {
        int* R = P + r2[b];
        const double zab = double(za * w2[b]);
#pragma unroll
        for (int c = 0; c < NN; ++c)
          fixed_add(R + c3[c], __double2loint(fma(zab, double(w3[c]), MAGIC)), fixed_packed(g));
      }
    }
  }
};

// Global fixed-point scale of a transpose sweep: S = 2^(26 - e) with
// max|z| < 2^e, from the max's float bits (device memory, uniform).
__device__ __forceinline__ float fixed_scale(unsigned zmax_bits, float* inv) {
  int e = 0;
  frexpf(__uint_as_float(zmax_bits), &e);
  *inv = ldexpf(1.0f, e - 26);
  return ldexpf(1.0f, 26 - e);
}

}  // namespace vb
