// Register-blocked semi-Lagrangian gather/scatter: one thread owns a QUAD of
// 4 consecutive x3 nodes of one (x1, x2) row.
//
// Why: a cubic sweep touches 64 taps per point. Neighbouring x3 points have
// near-identical displacements, so their stencils overlap: when the integer
// offsets of the 4 points differ by at most one per axis (the common case
// for smooth velocities), all 4 stencils fit in a (NN+1) x (NN+1) x (NN+4)
// box of rows x columns, each row an 8-column frame:
//   gather : 2-3 aligned 128-bit loads per frame row instead of 16 scalar
//            loads;
//   scatter: the contributions of the 4 points to a row are pre-summed in
//            registers and pushed with 2-3 REDG.E.ADD.F32x4 (vector L2
//            reductions) instead of 16 scalar REDs. Shared-memory fp32
//            atomics are a CAS loop on sm_100a, so the reduction stays in
//            registers + L2.
// The row count (NN or NN+1 per axis) is warp-uniform so the whole warp runs
// one code path; points whose weight row falls outside their own stencil
// get an exact zero weight, so the per-point accumulation order is the
// reference's a -> b -> c (interp.hpp:47-61) with zero terms interleaved.
// Frames crossing the periodic x3 edge use scalar wrapped I/O; only quads
// with an offset spread > 1 take the per-point fallback.
#pragma once

#include "sl_common.cuh"

namespace vb {

template <int DEG>
struct Quad {
  static constexpr int NN = DEG + 1;
  static constexpr int O0 = DEG == 3 ? -1 : 0;
  static constexpr int F = NN + 4;  // frame columns
  float w1[4][NN], w2[4][NN], w3[4][NN];
  int o1[4], o2[4], o3[4];
  float h1[4], h2[4], h3[4];  // 1.0f when the point's offset is the quad min + 1
  int m1, m2, m3;             // quad minimum offsets
  bool fast;                  // all spreads <= 1
  bool s1, s2;                // x1 / x2 spread present

  __device__ __forceinline__ void build(const float4& d1, const float4& d2, const float4& d3) {
    const float a1[4] = {d1.x, d1.y, d1.z, d1.w};
    const float a2[4] = {d2.x, d2.y, d2.z, d2.w};
    const float a3[4] = {d3.x, d3.y, d3.z, d3.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float t1, t2, t3;
      split_axis(a1[q], 0, o1[q], t1);
      split_axis(a2[q], 0, o2[q], t2);
      split_axis(a3[q], 0, o3[q], t3);
      lagrange_weights<DEG>(t1, w1[q]);
      lagrange_weights<DEG>(t2, w2[q]);
      lagrange_weights<DEG>(t3, w3[q]);
    }
    m1 = min(min(o1[0], o1[1]), min(o1[2], o1[3]));
    m2 = min(min(o2[0], o2[1]), min(o2[2], o2[3]));
    m3 = min(min(o3[0], o3[1]), min(o3[2], o3[3]));
    const int M1 = max(max(o1[0], o1[1]), max(o1[2], o1[3]));
    const int M2 = max(max(o2[0], o2[1]), max(o2[2], o2[3]));
    const int M3 = max(max(o3[0], o3[1]), max(o3[2], o3[3]));
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      h1[q] = float(o1[q] - m1);
      h2[q] = float(o2[q] - m2);
      h3[q] = float(o3[q] - m3);
    }
    fast = (M1 - m1 <= 1) & (M2 - m2 <= 1) & (M3 - m3 <= 1);
    s1 = M1 != m1;
    s2 = M2 != m2;
  }

  // weight of relative row r (0..NN) for a point with shift h on that axis
  __device__ __forceinline__ static float rw(const float* w, float h, int r) {
    const float lo = r < NN ? w[r < NN ? r : 0] : 0.0f;
    const float hi = r >= 1 ? w[r >= 1 ? r - 1 : 0] : 0.0f;
    return h != 0.0f ? hi : lo;
  }
};

// ---- aligned frame I/O --------------------------------------------------

template <int OFF, int F>
__device__ __forceinline__ void load_frame_off(const float* base, float* v) {
  constexpr int NG = (OFF + F + 3) / 4;
  float t[4 * NG];
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(base) + gi);
    t[4 * gi] = x.x;
    t[4 * gi + 1] = x.y;
    t[4 * gi + 2] = x.z;
    t[4 * gi + 3] = x.w;
  }
#pragma unroll
  for (int e = 0; e < F; ++e) v[e] = t[OFF + e];
}

template <int F>
__device__ __forceinline__ void load_frame(const float* row, int cbase, int n3, float* v) {
  if (cbase >= 0 && cbase + F <= n3) {
    const int off = cbase & 3;
    const float* base = row + (cbase - off);
    switch (off) {
      case 0: load_frame_off<0, F>(base, v); break;
      case 1: load_frame_off<1, F>(base, v); break;
      case 2: load_frame_off<2, F>(base, v); break;
      default: load_frame_off<3, F>(base, v); break;
    }
  } else {
#pragma unroll
    for (int e = 0; e < F; ++e) v[e] = __ldg(row + wrap_mod(cbase + e, n3));
  }
}

template <int OFF, int F>
__device__ __forceinline__ void red_frame_off(float* base, const float* v) {
  constexpr int NG = (OFF + F + 3) / 4;
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    float t[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = 4 * gi + e - OFF;
      t[e] = (idx >= 0 && idx < F) ? v[idx] : 0.0f;
    }
    atomicAdd(reinterpret_cast<float4*>(base) + gi, make_float4(t[0], t[1], t[2], t[3]));
  }
}

template <int F>
__device__ __forceinline__ void red_frame(float* row, int cbase, int n3, const float* v) {
  if (cbase >= 0 && cbase + F <= n3) {
    const int off = cbase & 3;
    float* base = row + (cbase - off);
    switch (off) {
      case 0: red_frame_off<0, F>(base, v); break;
      case 1: red_frame_off<1, F>(base, v); break;
      case 2: red_frame_off<2, F>(base, v); break;
      default: red_frame_off<3, F>(base, v); break;
    }
  } else {
#pragma unroll
    for (int e = 0; e < F; ++e)
      if (v[e] != 0.0f) atomicAdd(row + wrap_mod(cbase + e, n3), v[e]);
  }
}

// warp-uniform row counts per axis: NN, or NN+1 when any quad of the warp
// straddles an integer offset on that axis
template <int DEG>
__device__ __forceinline__ void quad_rows(const Quad<DEG>& Q, int& na, int& nb) {
  constexpr int NN = Quad<DEG>::NN;
  na = NN + (__any_sync(__activemask(), Q.s1) ? 1 : 0);
  nb = NN + (__any_sync(__activemask(), Q.s2) ? 1 : 0);
}

// ---- quad gather: out[q] = I[f](point q), q = 0..3 ------------------------

template <int DEG, bool DIST>
__device__ __forceinline__ void quad_gather(const Geo& g, const SrcField<DIST>& src,
                                            const Quad<DEG>& Q, int i, int j, int k0,
                                            float* out) {
  constexpr int NN = Quad<DEG>::NN, O0 = Quad<DEG>::O0, F = Quad<DEG>::F;
  const bool all_fast = __all_sync(__activemask(), Q.fast);
  if (all_fast) {
    int na, nb;
    quad_rows(Q, na, nb);
    int p1 = i + Q.m1 + O0;
    if constexpr (!DIST) p1 = wrap_mod(p1, g.n1);
    const int r0 = wrap_mod(j + Q.m2 + O0, g.n2);
    const int cbase = k0 + Q.m3 + O0;
    float acc1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int a = 0; a < NN + 1; ++a) {
      if (a >= na) break;
      const float* P = src.plane_ptr(p1 + a, g);
      float acc2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int b = 0; b < NN + 1; ++b) {
        if (b >= nb) break;
        const float* R = P + size_t(wrap1(r0 + b, g.n2)) * g.n3;
        float v[F];
        load_frame<F>(R, cbase, g.n3, v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float acc3 = 0.f;
#pragma unroll
          for (int c = 0; c < NN; ++c) {
            const float x = Q.h3[q] != 0.0f ? v[q + c + 1] : v[q + c];
            acc3 += Q.w3[q][c] * x;
          }
          acc2[q] += Quad<DEG>::rw(Q.w2[q], Q.h2[q], b) * acc3;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) acc1[q] += Quad<DEG>::rw(Q.w1[q], Q.h1[q], a) * acc2[q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = acc1[q];
    return;
  }
  // rare: a quad of the warp has an offset spread > 1 -> per-point stencils
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float acc1 = 0.f;
    int p1 = i + Q.o1[q] + O0;
    if constexpr (!DIST) p1 = wrap_mod(p1, g.n1);
    const int b2 = wrap_mod(j + Q.o2[q], g.n2), b3 = wrap_mod(k0 + q + Q.o3[q], g.n3);
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      const float* P = src.plane_ptr(p1 + a, g);
      float acc2 = 0.f;
#pragma unroll
      for (int b = 0; b < NN; ++b) {
        const float* R = P + size_t(wrap1(b2 + O0 + b, g.n2)) * g.n3;
        float acc3 = 0.f;
#pragma unroll
        for (int c = 0; c < NN; ++c) acc3 += Q.w3[q][c] * __ldg(R + wrap1(b3 + O0 + c, g.n3));
        acc2 += Q.w2[q][b] * acc3;
      }
      acc1 += Q.w1[q][a] * acc2;
    }
    out[q] = acc1;
  }
}

// ---- quad scatter: acc[stencil(q)] += w z[q] -------------------------------

template <int DEG, bool DIST>
__device__ __forceinline__ void quad_scatter(const Geo& g, const DstField<DIST>& dst,
                                             const Quad<DEG>& Q, int i, int j, int k0,
                                             const float* z) {
  constexpr int NN = Quad<DEG>::NN, O0 = Quad<DEG>::O0, F = Quad<DEG>::F;
  const bool all_fast = __all_sync(__activemask(), Q.fast);
  if (all_fast) {
    int na, nb;
    quad_rows(Q, na, nb);
    int p1 = i + Q.m1 + O0;
    if constexpr (!DIST) p1 = wrap_mod(p1, g.n1);
    const int r0 = wrap_mod(j + Q.m2 + O0, g.n2);
    const int cbase = k0 + Q.m3 + O0;
#pragma unroll
    for (int a = 0; a < NN + 1; ++a) {
      if (a >= na) break;
      float* P = dst.plane_ptr(p1 + a, g);
      float za[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) za[q] = Quad<DEG>::rw(Q.w1[q], Q.h1[q], a) * z[q];
#pragma unroll
      for (int b = 0; b < NN + 1; ++b) {
        if (b >= nb) break;
        float* R = P + size_t(wrap1(r0 + b, g.n2)) * g.n3;
        float v[F];
#pragma unroll
        for (int e = 0; e < F; ++e) v[e] = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float zab = za[q] * Quad<DEG>::rw(Q.w2[q], Q.h2[q], b);
          const float hi = Q.h3[q], lo = 1.0f - hi;
#pragma unroll
          for (int c = 0; c < NN; ++c) {
            const float t = zab * Q.w3[q][c];
            v[q + c] += lo * t;
            v[q + c + 1] += hi * t;
          }
        }
        red_frame<F>(R, cbase, g.n3, v);
      }
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int p1 = i + Q.o1[q] + O0;
    if constexpr (!DIST) p1 = wrap_mod(p1, g.n1);
    const int b2 = wrap_mod(j + Q.o2[q], g.n2), b3 = wrap_mod(k0 + q + Q.o3[q], g.n3);
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      float* P = dst.plane_ptr(p1 + a, g);
      const float za = Q.w1[q][a] * z[q];
#pragma unroll
      for (int b = 0; b < NN; ++b) {
        float* R = P + size_t(wrap1(b2 + O0 + b, g.n2)) * g.n3;
        const float zab = za * Q.w2[q][b];
#pragma unroll
        for (int c = 0; c < NN; ++c) atomicAdd(R + wrap1(b3 + O0 + c, g.n3), zab * Q.w3[q][c]);
      }
    }
  }
}

}  // namespace vb
