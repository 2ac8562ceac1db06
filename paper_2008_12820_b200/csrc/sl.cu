// Semi-Lagrangian kernels: RK2 characteristics (engine.hpp:111-155), gather
// interpolation (interp.cpp:70-115), its exact transpose (interp.cpp:92-123)
// and the fused transport steps of the state / adjoint / incremental solves
// (transport.hpp:49-228).
//
// Thread mapping: CTA = 32 x3-columns x 8 x2-rows of one x1 plane, so a
// warp's 32 departure points are contiguous nodes with near-identical
// displacements and their 4x4x4 stencils overlap in L1.
#include <cstdlib>
#include <set>

#include "common.cuh"
#include "sl_common.cuh"
#include "sl_tile.cuh"
#include "sl_pipe.cuh"

#include <cudaTypedefs.h>

namespace vb {

void bspline_prefilter(vreg_ctx ctx, const Slab& s, int ncomp, const float* in, float* out);

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

// One streaming pass for the whole incremental-state solve:
// w0 = -dt/2 (vt . grad m_0) and u_t = vt . grad m_t, t = 1..nt (u holds nt
// slices), so each fused step then loads one float instead of six.
__global__ void k_inc_u(size_t n4, int nt, const float4* __restrict__ vt,
                        const float4* __restrict__ gr, float half, float4* __restrict__ w0,
                        float4* __restrict__ u) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n4; p += stride) {
    const float4 a = vt[p], b = vt[n4 + p], c = vt[2 * n4 + p];
    for (int t = 0; t <= nt; ++t) {
      const float4* g = gr + size_t(t) * 3 * n4;
      const float4 x = g[p], y = g[n4 + p], z = g[2 * n4 + p];
      float4 r;
      r.x = a.x * x.x + b.x * y.x + c.x * z.x;
      r.y = a.y * x.y + b.y * y.y + c.y * z.y;
      r.z = a.z * x.z + b.z * y.z + c.z * z.z;
      r.w = a.w * x.w + b.w * y.w + c.w * z.w;
      if (t == 0)
        w0[p] = make_float4(-half * r.x, -half * r.y, -half * r.z, -half * r.w);
      else
        u[size_t(t - 1) * n4 + p] = r;
    }
  }
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

// k_assemble on float4 lanes (n % 4 == 0): the same per-element operations
// in the same order, 16-byte loads/stores.
__global__ void k_assemble4(size_t n4, int nt, float dt, int descending,
                            const float4* __restrict__ s, const float4* __restrict__ grads,
                            const float4* __restrict__ reg, float4* __restrict__ out) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n4; p += stride) {
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, a2 = a0;
    for (int q = 0; q <= nt; ++q) {
      const int t = descending ? nt - q : q;
      const float w = (t == 0 || t == nt) ? dt * 0.5f : dt;
      const float4 sv = s[size_t(t) * n4 + p];
      const float4* gt = grads + size_t(t) * 3 * n4;
      const float4 g0 = gt[p], g1 = gt[n4 + p], g2 = gt[2 * n4 + p];
      const float4 ws = make_float4(w * sv.x, w * sv.y, w * sv.z, w * sv.w);
      a0.x += ws.x * g0.x; a0.y += ws.y * g0.y; a0.z += ws.z * g0.z; a0.w += ws.w * g0.w;
      a1.x += ws.x * g1.x; a1.y += ws.y * g1.y; a1.z += ws.z * g1.z; a1.w += ws.w * g1.w;
      a2.x += ws.x * g2.x; a2.y += ws.y * g2.y; a2.z += ws.z * g2.z; a2.w += ws.w * g2.w;
    }
    if (reg) {
      const float4 r0 = reg[p], r1 = reg[n4 + p], r2 = reg[2 * n4 + p];
      a0.x += r0.x; a0.y += r0.y; a0.z += r0.z; a0.w += r0.w;
      a1.x += r1.x; a1.y += r1.y; a1.z += r1.z; a1.w += r1.w;
      a2.x += r2.x; a2.y += r2.y; a2.z += r2.z; a2.w += r2.w;
    }
    out[p] = a0;
    out[n4 + p] = a1;
    out[2 * n4 + p] = a2;
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

// ---- tile-staged variants (sl_tile.cuh) -----------------------------------

constexpr int kTileCap = BOX_CAP;

template <int DEG, bool DIST>
__device__ __forceinline__ float tile_gather(const Geo& g, const SrcField<DIST>& src,
                                             const TileBox& b, bool fits, const float* fbox,
                                             const float* __restrict__ D, int i, int j, int k,
                                             size_t p) {
  const float d1 = D[p], d2 = D[g.N + p], d3 = D[2 * g.N + p];
  if (fits) {
    BoxStencil<DEG> bs;
    if (bs.build(b, i, j, k, d1, d2, d3)) return bs.gather(b, fbox);
  }
  return point_gather<DEG, DIST>(g, src, i, j, k, d1, d2, d3);
}

// Point `it` of this thread in the tile (warp w: rows it*8 + w; lanes: x3).
#define TILE_PT(it)                                                          \
  const int row_##it = (it) * (TILE_THREADS / 32) + (threadIdx.x >> 5);      \
  const int i = layer * TT1 + row_##it / TT2;                                \
  const int j = blockIdx.y * TT2 + row_##it % TT2;                           \
  const int k = blockIdx.x * TT3 + (threadIdx.x & 31);                       \
  const bool ok = i < g.n1l && j < g.n2 && k < g.n3;                         \
  const size_t p = ok ? (size_t(i) * g.n2 + j) * g.n3 + k : 0;

// Gather kernels: issue the box as cp.async, prefetch the 8 points'
// displacements meanwhile, then serve all taps from smem.
template <int DEG, bool DIST, int MODE>  // MODE 0: interp(*q), 1: inc-state step,
                                         // 2: inc-state step on precomputed u, 3: source factor
__global__ void __launch_bounds__(TILE_THREADS, TILE_MIN_BLOCKS) k_gather_tile(
    Geo g, SrcField<DIST> src, const int* __restrict__ boxes, const float* __restrict__ D,
    const float* __restrict__ qf, float* __restrict__ out, const float* __restrict__ vt,
    const float* __restrict__ gr, float half, int last, float* __restrict__ mt_out, TileZ zm) {
  extern __shared__ __align__(16) float fbox[];
  __shared__ const float* rows[BOX_ROWS_MAX];
  const int layer = tile_layer(zm);
  const TileBox b = load_tile_box(boxes, tile_index_at(layer, int(gridDim.y)));
  const bool fits = b.ext[0] > 0;
  if (fits) {  // uniform per CTA
    if (box_vec(g)) {
      box_rows<DIST>(g, src, b, rows);
      __syncthreads();
    }
#ifndef VB_DIAG_NOBOX  // timing diagnostics only (wrong results): no box staging
    load_box(g, src, b, fbox, rows);
#endif
  }
  // prefetch the points' displacements (and, MODE 2, the precomputed
  // u = vt . grad m_{t+1} passed in qf) while the box streams in
  float d1[TILE_PPT], d2[TILE_PPT], d3[TILE_PPT], uu[TILE_PPT];
#pragma unroll
  for (int it = 0; it < TILE_PPT; ++it) {
    TILE_PT(it)
    d1[it] = ok ? D[p] : 0.f;
    d2[it] = ok ? D[g.N + p] : 0.f;
    d3[it] = ok ? D[2 * g.N + p] : 0.f;
    if constexpr (MODE == 2) uu[it] = ok ? qf[p] : 0.f;
  }
  cp_async_wait_all();
  __syncthreads();
#pragma unroll
  for (int it = 0; it < TILE_PPT; ++it) {
    TILE_PT(it)
    if (!ok) continue;
    float G;
    BoxStencil<DEG> bs;
    if (fits && bs.build(b, i, j, k, d1[it], d2[it], d3[it]))
#ifndef VB_DIAG_NOTAPS  // timing diagnostics only (wrong results): no tap contraction
      G = bs.gather(b, fbox);
#else
      G = bs.w1[0] + bs.w2[1] + bs.w3[2] + float(bs.base);
#endif
    else
      G = point_gather<DEG, DIST>(g, src, i, j, k, d1[it], d2[it], d3[it]);
    if constexpr (MODE == 0) {
      out[p] = qf ? G * qf[p] : G;
    } else if constexpr (MODE == 3) {  // adjoint source factor (transport.hpp:55-60)
      out[p] = (1.0f + half * G) / (1.0f - half * qf[p]);
    } else {
      float u;
      if constexpr (MODE == 2)
        u = uu[it];
      else
        u = vt[p] * gr[p] + vt[g.N + p] * gr[g.N + p] + vt[2 * g.N + p] * gr[2 * g.N + p];
      const float m = G - half * u;
      if (mt_out) mt_out[p] = m;
      out[p] = last ? -m : m - half * u;
    }
  }
}

// Tile-staged RK2 characteristics (engine.hpp:111-155). v changes with
// every call, so each CTA derives its box from its own points' midpoint
// displacements mid = -dt/h v (block min/max of the floors, as k_tile_boxes)
// and then serves the three velocity components from one shared box in
// turn: D_c = -(dt/2)/h_c (v_c + I[v_c](mid)). Tiles whose box exceeds the
// budget take the per-point global path.
template <int DEG, bool DIST>
__global__ void __launch_bounds__(TILE_THREADS, DIST ? 2 : TILE_MIN_BLOCKS) k_chars_tile(
    Geo g, SrcField<DIST> s1, SrcField<DIST> s2, SrcField<DIST> s3, const float* __restrict__ v,
    float m1, float m2, float m3, float c1, float c2, float c3, int box_cap_words,
    float* __restrict__ D) {
  constexpr int NN = Basis<DEG>::NN, O0 = Basis<DEG>::O0;
  extern __shared__ __align__(16) float fbox[];
  __shared__ const float* rows[BOX_ROWS_MAX];
  __shared__ int smn[3], smx[3];
  __shared__ TileBox sb;
  const int layer = blockIdx.z;
  if (threadIdx.x < 3) {
    smn[threadIdx.x] = 1 << 30;
    smx[threadIdx.x] = -(1 << 30);
  }
  float va[TILE_PPT], vb[TILE_PPT], vc[TILE_PPT];
  int mn[3] = {1 << 30, 1 << 30, 1 << 30}, mx[3] = {-(1 << 30), -(1 << 30), -(1 << 30)};
#pragma unroll
  for (int it = 0; it < TILE_PPT; ++it) {
    TILE_PT(it)
    va[it] = ok ? v[p] : 0.f;
    vb[it] = ok ? v[g.N + p] : 0.f;
    vc[it] = ok ? v[2 * g.N + p] : 0.f;
    if (ok) {
      const int f[3] = {int(floorf(m1 * va[it])), int(floorf(m2 * vb[it])),
                        int(floorf(m3 * vc[it]))};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        mn[a] = min(mn[a], f[a]);
        mx[a] = max(mx[a], f[a]);
      }
    }
  }
  __syncthreads();  // smn/smx initialised
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    mn[a] = __reduce_min_sync(0xffffffffu, mn[a]);
    mx[a] = __reduce_max_sync(0xffffffffu, mx[a]);
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(&smn[a], mn[a]);
      atomicMax(&smx[a], mx[a]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // box of the tile (k_tile_boxes rules)
    const int t[3] = {layer * TT1, int(blockIdx.y) * TT2, int(blockIdx.x) * TT3};
    const int T[3] = {min(TT1, g.n1l - t[0]), min(TT2, g.n2 - t[1]), min(TT3, g.n3 - t[2])};
    TileBox bx;
    for (int a = 0; a < 3; ++a) {
      bx.lo[a] = t[a] + smn[a] + O0;
      bx.ext[a] = T[a] - 1 + (smx[a] - smn[a]) + NN;
    }
    if ((g.n3 & 3) == 0) {
      const int sh = bx.lo[2] & 3;
      bx.lo[2] -= sh;
      bx.ext[2] = (bx.ext[2] + sh + 3) & ~3;
    }
    const int n[3] = {g.n1, g.n2, g.n3};
    bool fits = smn[0] <= smx[0] && bx.ext[2] <= BOX_PITCH &&
                bx.ext[0] * bx.ext[1] * BOX_PITCH <= box_cap_words;
    for (int a = 0; a < 3; ++a)
      fits = fits && bx.ext[a] <= n[a] && bx.lo[a] >= -n[a] && bx.lo[a] + bx.ext[a] <= 2 * n[a];
    if (!fits) bx.ext[0] = -1;
    sb = bx;
  }
  __syncthreads();
  const TileBox b = sb;
  const bool fits = b.ext[0] > 0;
  const float cc[3] = {c1, c2, c3};
#pragma unroll
  for (int comp = 0; comp < 3; ++comp) {
    const SrcField<DIST>& src = comp == 0 ? s1 : (comp == 1 ? s2 : s3);
    if (fits) {
      if (comp > 0) __syncthreads();  // previous component's gathers done
      if (box_vec(g)) {
        box_rows<DIST>(g, src, b, rows);
        __syncthreads();
      }
      load_box(g, src, b, fbox, rows);
      cp_async_wait_all();
      __syncthreads();
    }
#pragma unroll
    for (int it = 0; it < TILE_PPT; ++it) {
      TILE_PT(it)
      if (!ok) continue;
      const float d1 = m1 * va[it], d2 = m2 * vb[it], d3 = m3 * vc[it];
      float vs;
      BoxStencil<DEG> bs;
      if (fits && bs.build(b, i, j, k, d1, d2, d3))
        vs = bs.gather(b, fbox);
      else
        vs = point_gather<DEG, DIST>(g, src, i, j, k, d1, d2, d3);
      const float own = comp == 0 ? va[it] : (comp == 1 ? vb[it] : vc[it]);
      D[size_t(comp) * g.N + p] = cc[comp] * (own + vs);
    }
  }
}

// Default transpose sweep: per-tile power-of-two scale S = 2^(26-e_tile)
// in the shared int32 box (exact to 2^-27 max|z_tile| per contribution; a
// cell holds 32 max|z| -- the cubic weights' absolute sum under the
// compression the adjoint factor allows stays below ~14 max|z|),
// flushed with float4 REDs. The L2 adds of overlapping tiles land in any
// order, so the last bits can differ between runs (VREG_DETERMINISTIC=1 /
// vreg_ctx_set_deterministic selects the fixed-point variant below).
// (two CTAs per SM at 96 registers, leaving room for the regulariser's CTAs
// beside it, measured 299 vs 265 us per sweep: three CTAs per SM stay; the
// multi-rank variant runs spill-free at two, within 1% of three CTAs at 80
// registers with spills around the fallback calls, p = 2)
template <int DEG, bool DIST>
__global__ void __launch_bounds__(TILE_THREADS, DIST ? 2 : TILE_MIN_BLOCKS) k_scatter_tile_fp(Geo g, DstField<DIST> dst,
                                                                  const int* __restrict__ boxes,
                                                                  const float* __restrict__ D,
                                                                  const float* __restrict__ z,
                                                                  TileZ lay) {
  extern __shared__ __align__(16) int ibox[];
  __shared__ unsigned s_zmax;
  __shared__ float* rows[BOX_ROWS_MAX];
  const int layer = tile_layer(lay);
  const TileBox b = load_tile_box(boxes, tile_index_at(layer, int(gridDim.y)));
  const bool fits = b.ext[0] > 0;
  if (threadIdx.x == 0) s_zmax = 0u;
  if (fits) {
    if (box_vec(g)) box_rows<DIST>(g, dst, b, rows);  // read after the barriers below
    const int words = b.ext[0] * b.ext[1] * BOX_PITCH;
    int4* ib4 = reinterpret_cast<int4*>(ibox);  // words % 64 == 0
    for (int c = threadIdx.x; c < words / 4; c += TILE_THREADS) ib4[c] = make_int4(0, 0, 0, 0);
  }
  float zv[TILE_PPT], d1[TILE_PPT], d2[TILE_PPT], d3[TILE_PPT];
  unsigned zb = 0u;
#pragma unroll
  for (int it = 0; it < TILE_PPT; ++it) {
    TILE_PT(it)
    zv[it] = ok ? z[p] : 0.f;
    const float az = fabsf(zv[it]);
    zb = max(zb, az != az ? 0x7fc00000u : __float_as_uint(az));  // NaN sorts above Inf
    d1[it] = ok ? D[p] : 0.f;
    d2[it] = ok ? D[g.N + p] : 0.f;
    d3[it] = ok ? D[2 * g.N + p] : 0.f;
  }
  zb = __reduce_max_sync(0xffffffffu, zb);
  __syncthreads();  // s_zmax initialised, box zeroed
  if ((threadIdx.x & 31) == 0) atomicMax(&s_zmax, zb);
  __syncthreads();
  const float zm = __uint_as_float(s_zmax);
  if (zm == 0.0f) return;  // whole tile contributes nothing
  // non-finite z: fp32 atomics for the whole tile, so NaN / Inf reach the
  // output as in the reference's fp32 scatter (a fixed-point box cannot hold them)
  const bool boxed = fits && zm <= 3.4028235e38f;
  int e = 0;
  if (boxed) frexpf(zm, &e);  // max |z| < 2^e
  e = max(e, -99);            // scale stays a finite float for tiny tiles
  const float S = ldexpf(1.0f, 26 - e), invS = ldexpf(1.0f, e - 26);
#pragma unroll
  for (int it = 0; it < TILE_PPT; ++it) {
    TILE_PT(it)
    if (!ok || zv[it] == 0.0f) continue;
    BoxStencil<DEG> bs;
    if (boxed && bs.build(b, i, j, k, d1[it], d2[it], d3[it]))
      bs.scatter(b, ibox, zv[it] * S);
    else
      point_scatter<DEG, DIST>(g, dst, i, j, k, d1[it], d2[it], d3[it], zv[it]);
  }
  if (boxed) {
    __syncthreads();
    flush_box(g, dst, b, ibox, invS, rows);
  }
}

// Transpose sweep into an int32 accumulator field at the sweep's global
// fixed-point scale S = 2^(26 - e), max|z| < 2^e (zmax_bits: device, the max
// over all ranks). Every contribution is rounded once (DFMA), tiles add
// integers (shared then global atomics), so the result is exact in its
// quantisation and independent of tile / rank order: bitwise reproducible.
// A cell holds up to 32 max|z|; each contribution is exact to 2^-27 max|z|.
template <int DEG, bool DIST>
__global__ void __launch_bounds__(TILE_THREADS, TILE_MIN_BLOCKS) k_scatter_tile(Geo g, DstField<DIST> dst,
                                                                  const int* __restrict__ boxes,
                                                                  const float* __restrict__ D,
                                                                  const float* __restrict__ z,
                                                                  const unsigned* __restrict__ zmax_bits,
                                                                  TileZ lay) {
  extern __shared__ __align__(16) int ibox[];
  __shared__ float* rows[BOX_ROWS_MAX];
  const unsigned zmb = __ldg(zmax_bits);
  if (zmb == 0u) return;  // z == 0 everywhere: the (zeroed) output stays 0
  const int layer = tile_layer(lay);
  const TileBox b = load_tile_box(boxes, tile_index_at(layer, int(gridDim.y)));
  const bool fits = b.ext[0] > 0;
  if (fits) {
    if (box_vec(g)) box_rows<DIST>(g, dst, b, rows);  // read after the barriers below
    const int words = b.ext[0] * b.ext[1] * BOX_PITCH;
    int4* ib4 = reinterpret_cast<int4*>(ibox);  // words % 64 == 0
    for (int c = threadIdx.x; c < words / 4; c += TILE_THREADS) ib4[c] = make_int4(0, 0, 0, 0);
  }
  float zv[TILE_PPT], d1[TILE_PPT], d2[TILE_PPT], d3[TILE_PPT];
#pragma unroll
  for (int it = 0; it < TILE_PPT; ++it) {
    TILE_PT(it)
    zv[it] = ok ? z[p] : 0.f;
    d1[it] = ok ? D[p] : 0.f;
    d2[it] = ok ? D[g.N + p] : 0.f;
    d3[it] = ok ? D[2 * g.N + p] : 0.f;
  }
  float invS;
  const float S = fixed_scale(zmb, &invS);
  __syncthreads();  // box zeroed, row table written
#pragma unroll
  for (int it = 0; it < TILE_PPT; ++it) {
    TILE_PT(it)
    if (!ok || zv[it] == 0.0f) continue;
    BoxStencil<DEG> bs;
    if (fits && bs.build(b, i, j, k, d1[it], d2[it], d3[it]))
      bs.scatter(b, ibox, zv[it] * S);
    else
      point_scatter_fixed<DEG, DIST>(g, dst, i, j, k, d1[it], d2[it], d3[it], zv[it] * S);
  }
  if (fits) {
    __syncthreads();
    flush_box_fixed(g, dst, b, ibox, rows);
  }
}

// block max -> one atomic per CTA (blockDim.x == 256)
__device__ __forceinline__ void block_max_atomic(unsigned m, unsigned* out) {
  __shared__ unsigned sm[8];
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < 8 ? sm[threadIdx.x] : 0u;
    m = __reduce_max_sync(0xffffffffu, m);
    if (threadIdx.x == 0 && m) atomicMax(out, m);
  }
}

// max |x| over n floats as float bits (non-negative floats order as uints)
__global__ void k_maxabs_bits(size_t n, const float* __restrict__ x, unsigned* __restrict__ out) {
  unsigned m = 0u;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    m = max(m, __float_as_uint(fabsf(x[i])));
  block_max_atomic(m, out);
}

// packed pairs (n % 4 == 0): two int64 words = four cells per thread-iteration
__global__ void k_fixed_finish(size_t n4, const longlong2* __restrict__ I,
                               const unsigned* __restrict__ zmax_bits, float4* __restrict__ out,
                               unsigned* __restrict__ next_max) {
  float inv;
  fixed_scale(__ldg(zmax_bits), &inv);
  unsigned m = 0u;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const longlong2 v = I[i];
    const int a = int(v.x), c = int(v.y);  // low halves, sign-extended
    const int b = int((v.x - a) >> 32), d = int((v.y - c) >> 32);
    const float4 f = make_float4(float(a) * inv, float(b) * inv, float(c) * inv, float(d) * inv);
    out[i] = f;
    m = max(max(max(m, __float_as_uint(fabsf(f.x))), __float_as_uint(fabsf(f.y))),
            max(__float_as_uint(fabsf(f.z)), __float_as_uint(fabsf(f.w))));
  }
  if (next_max) block_max_atomic(m, next_max);
}

__global__ void k_fixed_finish1(size_t n, const int* __restrict__ I,
                                const unsigned* __restrict__ zmax_bits, float* __restrict__ out,
                                unsigned* __restrict__ next_max) {
  float inv;
  fixed_scale(__ldg(zmax_bits), &inv);
  unsigned m = 0u;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    out[i] = float(I[i]) * inv;
    m = max(m, __float_as_uint(fabsf(out[i])));
  }
  if (next_max) block_max_atomic(m, next_max);
}


inline dim3 tile_grid(const Slab& s) {
  return dim3(unsigned((s.n3 + TT3 - 1) / TT3), unsigned((s.n2 + TT2 - 1) / TT2),
              unsigned((s.n1l + TT1 - 1) / TT1));
}

constexpr TileZ kAllLayers{0, 1 << 30, 0};

inline dim3 tile_grid_nz(const Slab& s, int nz) {
  dim3 g = tile_grid(s);
  g.z = unsigned(nz);
  return g;
}

// x1 tile layers of a slab whose stencils stay clear of the ghost planes for
// ghost width G (floor(max|d1|) + 3): layer z reaches planes
// [4z - G + 1, 4z + G + 2], so zb = ceil((G + 3) / 4) boundary layers per side.
struct LayerSplit {
  bool on = false;
  int zb = 0, ntz = 0;
};
inline LayerSplit layer_split(const Slab& s, int G) {
  LayerSplit l;
  l.ntz = (s.n1l + TT1 - 1) / TT1;
  l.zb = (G + 3 + TT1 - 1) / TT1;
  static const bool overlap = [] {
    const char* e = std::getenv("VREG_HALO_OVERLAP");
    return !(e && e[0] == '0');
  }();
  l.on = overlap && 2 * l.zb < l.ntz;
  return l;
}

struct OnStream {  // issue on another stream for the scope (NCCL + its timers)
  vreg_ctx c;
  cudaStream_t prev;
  OnStream(vreg_ctx c_, cudaStream_t st) : c(c_), prev(c_->stream) { c->stream = st; }
  ~OnStream() { c->stream = prev; }
};

// Tile gather on several ranks: the halo exchange of f runs on the comm
// stream while the interior layers (no ghost reads) run; the two boundary
// bands follow once the ghosts have landed. launch(TileZ, nz) issues the
// tile kernel on ctx->stream.
template <class Launch>
void gather_tiles(vreg_ctx ctx, const Slab& s, const float* f, int G, bool dist, Ghosts& gh,
                  Launch launch) {
  const LayerSplit ls = layer_split(s, dist ? G : 0);
  if (!dist) {
    launch(kAllLayers, ls.ntz);
    return;
  }
  if (!ls.on) {
    gh = halo_exchange(ctx, s, f, G, "sl_ghost", T_INTERP_COMM, C_GHOST_INTERP);
    launch(kAllLayers, ls.ntz);
    return;
  }
  // the halo exchange and then the boundary layers run on the comm stream,
  // next to the interior sweep: the boundary sweep (dynamically scheduled)
  // starts on the SMs the interior leaves free and fills the ones its CTAs
  // release, instead of running alone after it
  VB_CUDA(cudaEventRecord(ctx->ev_c0, ctx->stream));
  VB_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_c0, 0));
  {
    OnStream os(ctx, ctx->comm_stream);
    gh = halo_exchange(ctx, s, f, G, "sl_ghost", T_INTERP_COMM, C_GHOST_INTERP);
    Timed tb(ctx, -1, "sl_gather_boundary");
    ctx->pipe_dynamic = true;
    try {
      launch(TileZ{0, ls.zb, ls.ntz - ls.zb}, 2 * ls.zb);
    } catch (...) {
      ctx->pipe_dynamic = false;
      throw;
    }
    ctx->pipe_dynamic = false;
  }
  VB_CUDA(cudaEventRecord(ctx->ev_c1, ctx->comm_stream));
  {
    Timed ti(ctx, -1, "sl_gather_interior");
    launch(TileZ{ls.zb, 1 << 30, 0}, ls.ntz - 2 * ls.zb);
  }
  Timed tw(ctx, -1, "sl_gather_boundary_wait");
  VB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_c1, 0));
}

// Tile scatter on several ranks: the boundary bands (the only tiles that
// write ghost accumulators) go first, their reverse exchange overlaps the
// interior layers, and the received planes are added at the end.
template <class Launch>
void scatter_tiles(vreg_ctx ctx, const Slab& s, const GhostAcc& acc, float* out, bool dist,
                   Launch launch, bool as_int = false) {
  const LayerSplit ls = layer_split(s, dist ? acc.G : 0);
  if (!dist) {
    launch(kAllLayers, ls.ntz);
    return;
  }
  if (!ls.on) {
    launch(kAllLayers, ls.ntz);
    halo_reverse_add(ctx, s, acc, out, "sl_gacc", as_int);
    return;
  }
  // boundary bands and their reverse exchange on the (high-priority) comm
  // stream, beside the interior sweep: both only add into out (atomics), and
  // the boundary's last partial wave no longer runs alone
  VB_CUDA(cudaEventRecord(ctx->ev_c0, ctx->stream));
  VB_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_c0, 0));
  RevHalo r;
  {
    OnStream os(ctx, ctx->comm_stream);
    {
      Timed tb(ctx, -1, "sl_scatter_boundary");
      launch(TileZ{0, ls.zb, ls.ntz - ls.zb}, 2 * ls.zb);
    }
    r = halo_reverse_send(ctx, s, acc, "sl_gacc");
    VB_CUDA(cudaEventRecord(ctx->ev_c1, ctx->stream));
  }
  {
    Timed ti(ctx, -1, "sl_scatter_interior");
    launch(TileZ{ls.zb, 1 << 30, 0}, ls.ntz - 2 * ls.zb);
  }
  VB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_c1, 0));
  halo_reverse_finish(ctx, s, r, out, as_int);
}

// Box table of the characteristics disp3 (cached per pointer/grid/degree;
// `refresh` recomputes after the characteristics were rewritten). A stale
// table only costs speed: points outside their box take the global path.
struct TileLaunch {
  const int* boxes;
  size_t smem;  // dynamic shared memory bytes: the largest box of the table
};

TileLaunch tile_table(vreg_ctx ctx, const Slab& s, const float* disp3, int degree, bool refresh) {
  const Geo g = geo_of(s);
  const dim3 grid = tile_grid(s);
  const size_t ntiles = size_t(grid.x) * grid.y * grid.z;
  // returns the largest box (words); one small D2H per characteristics
  auto build = [&](int* table) -> int {
    int* mw = table + 6 * ntiles;  // [0] largest box words, [1] misfit tiles
    VB_CUDA(cudaMemsetAsync(mw, 0, 2 * sizeof(int), ctx->stream));
    if (degree != 1)  // both cubic bases reach nodes -1..2
      k_tile_boxes<3><<<grid, TILE_THREADS, 0, ctx->stream>>>(g, disp3, table, mw);
    else
      k_tile_boxes<1><<<grid, TILE_THREADS, 0, ctx->stream>>>(g, disp3, table, mw);
    count_launch(ctx);
    check_launch();
    int h[2] = {0, 0};
    VB_CUDA(cudaMemcpyAsync(h, mw, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->tiles_built += ntiles;
    ctx->tiles_misfit += uint64_t(h[1]);
    return h[0] > 0 ? h[0] : BOX_PITCH;
  };
  for (auto& t : ctx->tile_tables) {
    if (t.disp == disp3 && t.n1 == s.n1 && t.n2 == s.n2 && t.n3 == s.n3 && t.n1l == s.n1l &&
        t.deg == degree) {
      if (refresh) t.smem_words = build(t.table);
      t.used = ++ctx->tile_clock;
      return {t.table, size_t(t.smem_words) * sizeof(float)};
    }
  }
  if (ctx->tile_tables.size() >= 16) {
    auto lru = ctx->tile_tables.begin();
    for (auto it = ctx->tile_tables.begin(); it != ctx->tile_tables.end(); ++it)
      if (it->used < lru->used) lru = it;
    VB_CUDA(cudaFreeAsync(lru->table, ctx->stream));
    ctx->tile_tables.erase(lru);
  }
  int* table = nullptr;
  VB_CUDA(cudaMallocAsync(&table, (6 * ntiles + 2) * sizeof(int), ctx->stream));
  const int words = build(table);
  ctx->tile_tables.push_back(
      {disp3, s.n1, s.n2, s.n3, s.n1l, degree, table, ++ctx->tile_clock, words});
  return {table, size_t(words) * sizeof(float)};
}

constexpr size_t kTileSmem = kTileCap * sizeof(float);

// Opt a tile kernel in to kTileSmem of dynamic shared memory (once).
template <class Kern>
inline Kern tile_kernel(Kern k) {
  smem_optin(reinterpret_cast<const void*>(k), int(kTileSmem));
  return k;
}

// ---- TMA pipeline (sl_pipe.cuh) host side ----------------------------------

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    VB_CUDA(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000,
                                             cudaEnableDefault, &q));
    require(q == cudaDriverEntryPointSuccess && f, VREG_ECUDA,
            "cuTensorMapEncodeTiled is not available");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// 3-D tensor map over `depth` stacked (n2 x n3) fp32 planes, boxes of one
// tile (TT3 x TT2 x TT1); out-of-range boxes zero-fill (masked points).
CUtensorMap tmap_planes(const float* base, const Slab& s, int depth) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {cuuint64_t(s.n3), cuuint64_t(s.n2), cuuint64_t(depth)};
  const cuuint64_t strides[2] = {cuuint64_t(s.n3) * 4u, cuuint64_t(s.n2) * cuuint64_t(s.n3) * 4u};
  const cuuint32_t box[3] = {cuuint32_t(TT3), cuuint32_t(TT2), cuuint32_t(TT1)};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = tmap_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                                    const_cast<float*>(base), dims, strides, box, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, VREG_ECUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

int sm_count(vreg_ctx ctx) {
  static int n = [&] {
    int v = 0;
    VB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, ctx->device));
    return v;
  }();
  return n;
}

// The pipeline needs 16-byte rows and whole-tile tensor boxes; other grids
// and misaligned streams take the cp.async tile kernels (VREG_SL_PIPE=0
// forces them, for A/B measurements).
inline bool use_pipe(const Slab& s, std::initializer_list<const void*> ptrs) {
  static const bool on = [] {
    const char* e = std::getenv("VREG_SL_PIPE");
    return !(e && e[0] == '0');
  }();
  if (!on || s.n3 % 4 != 0 || s.n3 < TT3 || s.n2 < TT2 || s.n1l < TT1) return false;
  for (const void* q : ptrs)
    if (q && (reinterpret_cast<uintptr_t>(q) & 15u)) return false;
  return true;
}

inline PipeTiles pipe_tiles(const Slab& s, int nz) {
  PipeTiles t;
  t.tx = (s.n3 + TT3 - 1) / TT3;
  t.ty = (s.n2 + TT2 - 1) / TT2;
  t.n = nz * t.tx * t.ty;
  return t;
}

// Tile ticket counters of the pipeline launches ({next ticket, CTAs done},
// zero between launches: the last CTA of a launch rewinds its pair). A ring
// of pairs, so launches in flight on different streams never share one.
constexpr int kSchedSlots = 64;
int* pipe_sched(vreg_ctx ctx) {
  const bool fresh = ctx->ws.find("pipe_sched") == ctx->ws.end();
  int* base = static_cast<int*>(workspace(ctx, "pipe_sched", 2 * kSchedSlots * sizeof(int)));
  if (fresh) VB_CUDA(cudaMemsetAsync(base, 0, 2 * kSchedSlots * sizeof(int), ctx->stream));
  static thread_local unsigned slot = 0;
  return base + 2 * (slot++ % kSchedSlots);
}

template <class Kern>
inline Kern pipe_kernel(Kern k) {
  smem_optin(reinterpret_cast<const void*>(k), int(PIPE_SMEM));
  return k;
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
  require(degree == 1 || degree == 3 || degree == VREG_INTERP_BSPLINE3, VREG_EPARAM,
          "interpolation degree must be 1, 3 or 4 (cubic B-spline)");
}

// Source of a gather: the field itself, or for the cubic B-spline its
// prefiltered coefficients (in the workspace `slot`).
inline const float* gather_source(vreg_ctx ctx, const Slab& s, int degree, const float* f,
                                  const char* slot) {
  if (degree != VREG_INTERP_BSPLINE3) return f;
  float* c = static_cast<float*>(workspace(ctx, slot, s.local() * sizeof(float)));
  bspline_prefilter(ctx, s, 1, f, c);
  return c;
}

// Dispatch a kernel template over (degree, dist).
#define SL_DISPATCH(degree, dist, LAUNCH)                 \
  do {                                                    \
    if (degree == VREG_INTERP_BSPLINE3) {                 \
      if (dist) {                                         \
        constexpr int DEG = 4;                            \
        constexpr bool DIST = true;                       \
        LAUNCH;                                           \
      } else {                                            \
        constexpr int DEG = 4;                            \
        constexpr bool DIST = false;                      \
        LAUNCH;                                           \
      }                                                   \
    } else if (degree == 3) {                             \
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

// One gather sweep launch through the TMA pipeline (nz tile layers of zm).
template <int MODE>
void gather_pipe(vreg_ctx ctx, const Slab& s, int degree, bool dist, const float* f,
                 const Ghosts& gh, const int* boxes, const float* disp3, const float* aux,
                 float* out, float half, int last, float* mt_out, TileZ zm, int nz,
                 float* zero_out = nullptr) {
  const Geo g = geo_of(s);
  const CUtensorMap tmD = tmap_planes(disp3, s, 3 * s.n1l);
  const CUtensorMap tmA = aux ? tmap_planes(aux, s, s.n1l) : tmD;
  const PipeTiles pt = pipe_tiles(s, nz);
  // One persistent CTA per SM holds its SM for the whole sweep, so on
  // several GPUs a few SMs stay free for the NCCL kernels of the halo
  // exchanges that overlap the interior layers (VREG_PIPE_RESERVE SMs)
  static const int reserve = [] {
    const char* e = std::getenv("VREG_PIPE_RESERVE");
    return e ? std::max(0, std::atoi(e)) : 8;
  }();
  const int ctas = ctx->nranks > 1 ? std::max(1, sm_count(ctx) - reserve) : sm_count(ctx);
  const unsigned grid = unsigned(std::min(pt.n, ctas));
  int* sched = ctx->pipe_dynamic ? pipe_sched(ctx) : nullptr;
  SL_DISPATCH(degree, dist,
              (pipe_kernel(k_gather_pipe<DEG, DIST, MODE>)<<<grid, PIPE_THREADS, PIPE_SMEM,
                                                             ctx->stream>>>(
                  g, src_of<DIST>(f, gh), boxes, tmD, tmA, aux ? 1 : 0, out, half, last, mt_out,
                  zm, pt, sched, zero_out)));
}

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
  f = gather_source(ctx, s, degree, f, "bs_coef");
  Timed t(ctx, T_SL, "sl_interp");
  const Geo g = geo_of(s);
  const TileLaunch tl = tile_table(ctx, s, disp3, degree, false);
  const bool pipe = use_pipe(s, {f, disp3, q, out});
  gather_tiles(ctx, s, f, ci.G, dist, gh, [&](TileZ zm, int nz) {
    if (pipe) {
      gather_pipe<0>(ctx, s, degree, dist, f, gh, tl.boxes, disp3, q, out, 0.f, 0, nullptr, zm,
                     nz);
      return;
    }
    SL_DISPATCH(degree, dist,
                (tile_kernel(k_gather_tile<DEG, DIST, 0>)<<<tile_grid_nz(s, nz), TILE_THREADS,
                                                             tl.smem, ctx->stream>>>(
                    g, src_of<DIST>(f, gh), tl.boxes, disp3, q, out, nullptr, nullptr, 0.f, 0,
                    nullptr, zm)));
  });
}

// out = I^T z (out is overwritten). Default: per-tile fixed point flushed
// with fp32 L2 reductions (k_scatter_tile_fp). Deterministic mode: one
// global fixed-point scale (k_scatter_tile); zmax = device max|z| bits of
// this sweep's input (computed here when null), next_max (optional)
// receives max|out| bits for a following sweep.
void scatter_sweep(vreg_ctx ctx, const Slab& s, const float* z, const float* disp3,
                   const CharsInfo& ci, int degree, float* out, unsigned* zmax = nullptr,
                   unsigned* next_max = nullptr, bool prezeroed = false) {
  const size_t N = s.local();
  if (ci.identity) {
    if (out != z)
      VB_CUDA(cudaMemcpyAsync(out, z, N * sizeof(float), cudaMemcpyDeviceToDevice,
                              ctx->stream));
    if (next_max) {
      k_maxabs_bits<<<blocks_for(N, 256), 256, 0, ctx->stream>>>(N, out, next_max);
      count_launch(ctx);
      check_launch();
    }
    return;
  }
  require(out != z, VREG_EPARAM, "scatter cannot run in place");
  const bool dist = ctx->nranks > 1;
  GhostAcc acc;
  if (dist) acc = ghost_accumulators(ctx, s, ci.G, "sl_gacc");
  Timed t(ctx, T_SL, "sl_scatter_sweep");
  const Geo g = geo_of(s);
  if (!ctx->deterministic) {
    if (!prezeroed) VB_CUDA(cudaMemsetAsync(out, 0, N * sizeof(float), ctx->stream));
    const TileLaunch tl = tile_table(ctx, s, disp3, degree, false);
    scatter_tiles(ctx, s, acc, out, dist, [&](TileZ zm, int nz) {
      SL_DISPATCH(degree, dist,
                  (tile_kernel(k_scatter_tile_fp<DEG, DIST>)<<<tile_grid_nz(s, nz), TILE_THREADS,
                                                               tl.smem, ctx->stream>>>(
                      g, dst_of<DIST>(out, acc), tl.boxes, disp3, z, zm)));
    });
    // B-spline: I = B P (P the symmetric prefilter), so I^T = P B^T
    if (degree == VREG_INTERP_BSPLINE3) bspline_prefilter(ctx, s, 1, out, out);
    return;
  }
  if (!zmax) {
    zmax = static_cast<unsigned*>(workspace(ctx, "sc_zmax", 64));
    VB_CUDA(cudaMemsetAsync(zmax, 0, sizeof(unsigned), ctx->stream));
    k_maxabs_bits<<<blocks_for(N, 256), 256, 0, ctx->stream>>>(N, z, zmax);
    count_launch(ctx);
    check_launch();
  }
  if (dist)  // one scale on every rank
    VB_NCCL(ncclAllReduce(zmax, zmax, 1, ncclUint32, ncclMax, ctx->comm, ctx->stream));
  float* I = static_cast<float*>(workspace(ctx, "sc_fixed", N * sizeof(float)));  // int32
  VB_CUDA(cudaMemsetAsync(I, 0, N * sizeof(float), ctx->stream));
  const TileLaunch tl = tile_table(ctx, s, disp3, degree, false);
  scatter_tiles(
      ctx, s, acc, I, dist,
      [&](TileZ zm, int nz) {
        SL_DISPATCH(degree, dist,
                    (tile_kernel(k_scatter_tile<DEG, DIST>)<<<tile_grid_nz(s, nz), TILE_THREADS,
                                                              tl.smem, ctx->stream>>>(
                        g, dst_of<DIST>(I, acc), tl.boxes, disp3, z, zmax, zm)));
      },
      true);
  if (s.n3 % 4 == 0) {  // packed pairs (fixed_add)
    k_fixed_finish<<<blocks_for(N / 4, 256), 256, 0, ctx->stream>>>(
        N / 4, reinterpret_cast<const longlong2*>(I), zmax, reinterpret_cast<float4*>(out),
        next_max);
  } else {
    k_fixed_finish1<<<blocks_for(N, 256), 256, 0, ctx->stream>>>(
        N, reinterpret_cast<const int*>(I), zmax, out, next_max);
  }
  count_launch(ctx);
  check_launch();
  if (degree == VREG_INTERP_BSPLINE3) bspline_prefilter(ctx, s, 1, out, out);
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
                  const float* grads, const float* vt3, float* mt_all, float* psi_out,
                  float* zero_slices) {
  check_degree(degree);
  const CharsInfo ci = chars_info(ctx, s, disp3, flags, degree);
  const size_t N = s.local();
  const int nt = s.nt;
  const float half = float(0.5 * s.dt());
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  // all u_t in one streaming pass; the steps then read one float each
  // (forming u_{t+1} = vt . grad m_{t+1} inside the pipeline steps instead --
  // six more loads per point next to the taps -- cost 78 us per step against
  // the 145 us the pre-pass saved)
  const bool fused_u = !ci.identity && N % 4 == 0 && al16(vt3) && al16(grads);
  float* w = static_cast<float*>(workspace(ctx, "inc_w", 2 * N * sizeof(float)));
  float* u = fused_u ? static_cast<float*>(workspace(ctx, "inc_u", size_t(nt) * N * sizeof(float)))
                     : nullptr;
  {
    Timed t(ctx, T_SL, "sl_inc_init");
    if (fused_u)
      k_inc_u<<<blocks_for(N / 4, 256), 256, 0, ctx->stream>>>(
          N / 4, nt, reinterpret_cast<const float4*>(vt3), reinterpret_cast<const float4*>(grads),
          half, reinterpret_cast<float4*>(w), reinterpret_cast<float4*>(u));
    else
      k_inc_init<<<blocks_for(N, 256), 256, 0, ctx->stream>>>(N, vt3, grads, half, w);
    count_launch(ctx);
    check_launch();
  }
  if (mt_all) VB_CUDA(cudaMemsetAsync(mt_all, 0, N * sizeof(float), ctx->stream));
  // zero_slices (the transpose sweeps' outputs, nt slices): the pipeline
  // steps store the zeros next to their outputs (an HBM write in LSU-bound
  // sweeps instead of a memset per transpose sweep); other paths memset here
  if (zero_slices && !(fused_u && use_pipe(s, {w, w + N, disp3, u, psi_out, mt_all}))) {
    VB_CUDA(cudaMemsetAsync(zero_slices, 0, size_t(nt) * N * sizeof(float), ctx->stream));
    zero_slices = nullptr;
  }
  const bool dist = ctx->nranks > 1 && !ci.identity;
  const Geo g = geo_of(s);
  const dim3 grid = sl_grid(s), block(BX, BY);
  for (int t = 0; t < nt; ++t) {
    const float* wt = w + size_t(t & 1) * N;
    const bool last = t == nt - 1;
    float* wn = last ? psi_out : w + size_t((t + 1) & 1) * N;
    float* mo = mt_all ? mt_all + size_t(t + 1) * N : nullptr;
    Ghosts gh;
    // B-spline: the step gathers the coefficients of w_t
    const float* src = ci.identity ? wt : gather_source(ctx, s, degree, wt, "bs_w");
    Timed tm(ctx, T_SL, "sl_inc_step");
    if (ci.identity) {  // identity characteristics: pointwise step
      SL_DISPATCH(degree, dist,
                  (k_inc_step<DEG, DIST><<<grid, block, 0, ctx->stream>>>(
                      g, src_of<DIST>(wt, gh), disp3, 1, vt3, grads + size_t(t + 1) * 3 * N,
                      half, last ? 1 : 0, wn, mo)));
    } else if (fused_u) {
      const TileLaunch tl = tile_table(ctx, s, disp3, degree, false);
      const float* ut = u + size_t(t) * N;
      const bool pipe = use_pipe(s, {src, disp3, ut, wn, mo});
      float* zo = zero_slices ? zero_slices + size_t(t) * N : nullptr;
      if (zo && !pipe) VB_CUDA(cudaMemsetAsync(zo, 0, N * sizeof(float), ctx->stream));
      gather_tiles(ctx, s, src, ci.G, dist, gh, [&](TileZ zm, int nz) {
        if (pipe) {
          gather_pipe<2>(ctx, s, degree, dist, src, gh, tl.boxes, disp3, ut, wn, half,
                         last ? 1 : 0, mo, zm, nz, zo);
          return;
        }
        SL_DISPATCH(degree, dist,
                    (tile_kernel(k_gather_tile<DEG, DIST, 2>)<<<tile_grid_nz(s, nz), TILE_THREADS,
                                                                 tl.smem, ctx->stream>>>(
                        g, src_of<DIST>(src, gh), tl.boxes, disp3, u + size_t(t) * N, wn, nullptr,
                        nullptr, half, last ? 1 : 0, mo, zm)));
      });
    } else {
      const TileLaunch tl = tile_table(ctx, s, disp3, degree, false);
      gather_tiles(ctx, s, src, ci.G, dist, gh, [&](TileZ zm, int nz) {
        SL_DISPATCH(degree, dist,
                    (tile_kernel(k_gather_tile<DEG, DIST, 1>)<<<tile_grid_nz(s, nz), TILE_THREADS,
                                                                 tl.smem, ctx->stream>>>(
                        g, src_of<DIST>(src, gh), tl.boxes, disp3, nullptr, wn, vt3,
                        grads + size_t(t + 1) * 3 * N, half, last ? 1 : 0, mo, zm)));
      });
    }
  }
}

// psi[t-1] = I^T psi[t] for t = nt..1; psi holds nt+1 slices, psi[nt] set.
void sl_transpose_sweeps(vreg_ctx ctx, const Slab& s, const float* disp3, int flags,
                         int degree, float* psi, bool prezeroed) {
  check_degree(degree);
  const CharsInfo ci = chars_info(ctx, s, disp3, flags, degree);
  const size_t N = s.local();
  // max|psi_t| bits per slice: each sweep's finish hands the next its scale
  unsigned* mx = nullptr;
  // (the B-spline prefilter after each sweep changes max|psi|: those sweeps
  // measure their own input)
  if (ctx->deterministic && !ci.identity && degree != VREG_INTERP_BSPLINE3) {
    mx = static_cast<unsigned*>(workspace(ctx, "sc_chain", size_t(s.nt + 1) * sizeof(unsigned)));
    VB_CUDA(cudaMemsetAsync(mx, 0, size_t(s.nt + 1) * sizeof(unsigned), ctx->stream));
    k_maxabs_bits<<<blocks_for(N, 256), 256, 0, ctx->stream>>>(N, psi + size_t(s.nt) * N,
                                                               mx + s.nt);
    count_launch(ctx);
    check_launch();
  }
  for (int t = s.nt; t > 0; --t)
    scatter_sweep(ctx, s, psi + size_t(t) * N, disp3, ci, degree, psi + size_t(t - 1) * N,
                  mx ? mx + t : nullptr, mx && t > 1 ? mx + t - 1 : nullptr, prezeroed);
}

// psi buffer ((nt+1) slices) of a GN matvec
float* sl_matvec_psi(vreg_ctx ctx, const Slab& s, const float* disp3, int flags, int degree) {
  (void)disp3;
  (void)flags;
  (void)degree;
  return static_cast<float*>(
      workspace(ctx, "mv_psi", size_t(s.nt + 1) * s.local() * sizeof(float)));
}

void sl_assemble(vreg_ctx ctx, const Slab& s, int descending, const float* sl,
                 const float* grads, const float* reg, float* out3) {
  Timed t(ctx, T_SL, "sl_assemble");
  const size_t N = s.local();
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  if (N % 4 == 0 && al16(sl) && al16(grads) && (!reg || al16(reg)) && al16(out3))
    k_assemble4<<<blocks_for(N / 4, 256), 256, 0, ctx->stream>>>(
        N / 4, s.nt, float(s.dt()), descending, reinterpret_cast<const float4*>(sl),
        reinterpret_cast<const float4*>(grads), reinterpret_cast<const float4*>(reg),
        reinterpret_cast<float4*>(out3));
  else
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
  // midpoint samples come from v itself or, for the B-spline, its coefficients
  const float* vs = v3;
  if (degree == VREG_INTERP_BSPLINE3) {
    float* c = static_cast<float*>(workspace(ctx, "bs_v", 3 * N * sizeof(float)));
    bspline_prefilter(ctx, s, 3, v3, c);
    vs = c;
  }
  Ghosts g1, g2, g3;
  if (dist) {
    // ghost width from the midpoint displacement bound dt max|v1| / h1
    const double vmax1 = reduce(ctx, s, 1, v3, v3, true);
    int G = int(std::floor(dt * vmax1 / s.h(0))) + (degree != 1 ? 3 : 2);
    require(G <= 2 * s.n1, VREG_ECONFIG, "displacement exceeds twice the domain");
    g1 = halo_exchange(ctx, s, vs, G, "chars_g1", T_INTERP_COMM, C_GHOST_INTERP);
    g2 = halo_exchange(ctx, s, vs + N, G, "chars_g2", T_INTERP_COMM, C_GHOST_INTERP);
    g3 = halo_exchange(ctx, s, vs + 2 * N, G, "chars_g3", T_INTERP_COMM, C_GHOST_INTERP);
  }
  Timed t(ctx, T_SL, "sl_characteristics");
  const Geo g = geo_of(s);
  const float m1 = float(-dt / s.h(0)), m2 = float(-dt / s.h(1)), m3 = float(-dt / s.h(2));
  const float c1 = float(-0.5 * dt / s.h(0)), c2 = float(-0.5 * dt / s.h(1)),
              c3 = float(-0.5 * dt / s.h(2));
  // box bound from max|v| (the midpoint floors spread by <= 2 floor(dt vmax / h) + 1)
  int ext[3];
  const int T[3] = {TT1, TT2, TT3};
  for (int a = 0; a < 3; ++a)
    ext[a] = T[a] + (degree != 1 ? 3 : 1) + 2 * int(std::floor(dt * vmax / s.h(a))) + 2;
  ext[2] = ((ext[2] + 3 + 3) / 4) * 4;
  const int words = std::min(BOX_CAP, ext[0] * ext[1] * BOX_PITCH);
  const size_t smem = size_t(words) * sizeof(float);
  SL_DISPATCH(degree, dist,
              (tile_kernel(k_chars_tile<DEG, DIST>)<<<tile_grid(s), TILE_THREADS, smem,
                                                      ctx->stream>>>(
                  g, src_of<DIST>(vs, g1), src_of<DIST>(vs + N, g2),
                  src_of<DIST>(vs + 2 * N, g3), v3, m1, m2, m3, c1, c2, c3, words, disp3)));
  return 0;
}

void sl_source_factor(vreg_ctx ctx, const Slab& s, const float* d, const float* disp_bwd3,
                      int flags, int degree, float* q) {
  check_degree(degree);
  const CharsInfo ci = chars_info(ctx, s, disp_bwd3, flags, degree);
  const bool dist = ctx->nranks > 1 && !ci.identity;
  // gathered field: d, or its B-spline coefficients; the own term uses d
  const float* dsrc = ci.identity ? d : gather_source(ctx, s, degree, d, "bs_coef");
  Ghosts gh;
  if (dist) gh = halo_exchange(ctx, s, dsrc, ci.G, "sl_ghost", T_INTERP_COMM, C_GHOST_INTERP);
  Timed t(ctx, T_SL);
  const Geo g = geo_of(s);
  const dim3 grid = sl_grid(s), block(BX, BY);
  const float half = float(0.5 * s.dt());
  if (!ci.identity) {
    const TileLaunch tl = tile_table(ctx, s, disp_bwd3, degree, false);
    if (use_pipe(s, {dsrc, d, disp_bwd3, q})) {
      gather_pipe<3>(ctx, s, degree, dist, dsrc, gh, tl.boxes, disp_bwd3, d, q, half, 0,
                     nullptr, kAllLayers, (s.n1l + TT1 - 1) / TT1);
      return;
    }
    SL_DISPATCH(degree, dist,
                (tile_kernel(k_gather_tile<DEG, DIST, 3>)<<<tile_grid(s), TILE_THREADS, tl.smem,
                                                             ctx->stream>>>(
                    g, src_of<DIST>(dsrc, gh), tl.boxes, disp_bwd3, d, q, nullptr, nullptr, half,
                    0, nullptr, kAllLayers)));
    return;
  }
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
    if (!ident) tile_table(ctx, s, disp3, degree, true);
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
    sl_inc_state(ctx, s, disp3, identity, degree, grads, vt3, mt_all, psi, nullptr);
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
    sl_transpose_sweeps(ctx, s, disp3, identity, degree, psi, false);
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
