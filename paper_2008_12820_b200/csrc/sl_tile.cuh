// Tile-staged semi-Lagrangian sweeps (the hot kernels of the GN matvec).
//
// A CTA owns a 4 x 16 x 32 (x1, x2, x3) tile of departure points. Each tile
// has a BOX of grid cells its stencils touch,
//   box_a = [tile_a + min_a + O0, tile_a + T_a - 1 + max_a + O0 + NN - 1],
// min/max over the tile of floor(disp_a). Boxes depend only on the
// characteristics, so they are computed once per characteristics
// (k_tile_boxes) and cached; ~2.8 cells per point for smooth flows.
//
// gather : the source box is loaded once (coalesced rows, periodic wrap /
//          x1 ghost planes applied on load) into shared memory and every
//          point's 64 taps are served from smem.
// scatter: contributions accumulate in a shared-memory box in 32-bit fixed
//          point (native ATOMS.ADD; fp32 smem atomics are a CAS loop on
//          sm_100a, ~4x slower, tools/smem_atomic_bench.cu) with a per-tile
//          power-of-two scale S = 2^(26-e), max|z_tile| < 2^e, so each
//          contribution is exact to 2^-27 max|z| and a cell absorbs 32
//          max|z| without overflow; tiles with non-finite z use fp32
//          global atomics (NaN / Inf propagate). Each contribution is rounded by one
//          DFMA against 1.5 * 2^52 (F2I is quarter-rate XU and was the
//          binding pipe). The box is flushed once with float4 REDs:
//          ~3 L2 reductions per point instead of 64 (the L2 RED path is
//          payload-bound at ~6.4 TB/s, tools/red_bench.cu).
// Smem rows have a pitch of 64 words, so lanes of a warp (32 consecutive x3
// points) whose x1/x2 offsets differ by one row/plane still hit distinct
// banks. Tiles whose box exceeds the smem budget, and single points outside
// a (stale) cached box, take the per-point global-memory path.
#pragma once

#include "sl_common.cuh"

namespace vb {

#ifndef VB_TT1
#define VB_TT1 4
#define VB_TT2 16
#define VB_TILE_THREADS 256
#endif
constexpr int TT1 = VB_TT1, TT2 = VB_TT2, TT3 = 32;
constexpr int TILE_THREADS = VB_TILE_THREADS;
constexpr int TILE_POINTS = TT1 * TT2 * TT3;
constexpr int TILE_PPT = TILE_POINTS / TILE_THREADS;  // points per thread (8)
constexpr int BOX_PITCH = 64;                          // smem row pitch (words)
#ifndef TILE_MIN_BLOCKS
#define TILE_MIN_BLOCKS 3  // CTAs per SM the register budget is sized for
#endif
constexpr int BOX_CAP = 18432;                         // smem words per CTA (72 KB: 3 CTAs/SM)

// Cached per-tile box: lo1, lo2, lo3, e1, e2, e3 (e1 = 0: empty, e1 < 0: no fit)
struct TileBox {
  int lo[3];
  int ext[3];
};

__device__ __forceinline__ TileBox load_tile_box(const int* __restrict__ table, int tile) {
  TileBox b;
  const int* t = table + 6 * size_t(tile);
  b.lo[0] = __ldg(t);
  b.lo[1] = __ldg(t + 1);
  b.lo[2] = __ldg(t + 2);
  b.ext[0] = __ldg(t + 3);
  b.ext[1] = __ldg(t + 4);
  b.ext[2] = __ldg(t + 5);
  return b;
}

__device__ __forceinline__ int tile_index() {
  return (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
}

// x1 tile-layer range of a launch: layer = z < zs ? z0 + z : z1 + (z - zs).
// Full launches use {0, INT_MAX, 0}; on several ranks the interior layers
// (boxes clear of the ghost planes) and the two boundary bands are launched
// separately so the halo exchange overlaps the interior tiles.
struct TileZ {
  int z0, zs, z1;
};
__device__ __forceinline__ int tile_layer(const TileZ& m) {
  const int z = int(blockIdx.z);
  return z < m.zs ? m.z0 + z : m.z1 + (z - m.zs);
}
__device__ __forceinline__ int tile_index_at(int layer, int ntile_y) {
  return (layer * ntile_y + int(blockIdx.y)) * int(gridDim.x) + int(blockIdx.x);
}

// Point (i, j, k) of iteration `it` of this thread: warp w covers rows
// (x1, x2) = (it*8 + w) / TT2, % TT2 and its lanes the 32 x3 columns.
#define TILE_POINT_LOOP(g)                                                     \
  const int t1 = blockIdx.z * TT1, t2 = blockIdx.y * TT2, t3 = blockIdx.x * TT3; \
  const int k = t3 + (threadIdx.x & 31);                                       \
  _Pragma("unroll 1") for (int it = 0; it < TILE_PPT; ++it) {                  \
    const int row = it * (TILE_THREADS / 32) + (threadIdx.x >> 5);             \
    const int i = t1 + row / TT2, j = t2 + row % TT2;                          \
    if (i >= (g).n1l || j >= (g).n2 || k >= (g).n3) continue;                  \
    const size_t p = (size_t(i) * (g).n2 + j) * (g).n3 + k;

#define TILE_POINT_LOOP_END }

// ---- box computation (one CTA per tile) ------------------------------------

template <int DEG>
__global__ void __launch_bounds__(TILE_THREADS) k_tile_boxes(Geo g, const float* __restrict__ D,
                                                             int* __restrict__ table,
                                                             int* __restrict__ max_words) {
  constexpr int NN = Basis<DEG>::NN, O0 = Basis<DEG>::O0;
  __shared__ int smn[3], smx[3];
  if (threadIdx.x < 3) {
    smn[threadIdx.x] = 1 << 30;
    smx[threadIdx.x] = -(1 << 30);
  }
  __syncthreads();
  int mn[3] = {1 << 30, 1 << 30, 1 << 30}, mx[3] = {-(1 << 30), -(1 << 30), -(1 << 30)};
  TILE_POINT_LOOP(g)
  const int f[3] = {int(floorf(D[p])), int(floorf(D[g.N + p])), int(floorf(D[2 * g.N + p]))};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    mn[a] = min(mn[a], f[a]);
    mx[a] = max(mx[a], f[a]);
  }
  TILE_POINT_LOOP_END
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
  if (threadIdx.x == 0) {
    const int t[3] = {int(blockIdx.z) * TT1, int(blockIdx.y) * TT2, int(blockIdx.x) * TT3};
    const int T[3] = {min(TT1, g.n1l - t[0]), min(TT2, g.n2 - t[1]), min(TT3, g.n3 - t[2])};
    int* out = table + 6 * size_t(tile_index());
    int e[3];
    for (int a = 0; a < 3; ++a) {
      out[a] = t[a] + smn[a] + O0;
      e[a] = T[a] - 1 + (smx[a] - smn[a]) + NN;
    }
    if ((g.n3 & 3) == 0) {  // 16-byte rows: x3 origin and extent 4-aligned
      const int sh = out[2] & 3;
      out[2] -= sh;
      e[2] = (e[2] + sh + 3) & ~3;
    }
    // single-period wrap on load/flush needs every box coordinate in [-n, 2n)
    const int n[3] = {g.n1, g.n2, g.n3};
    bool fits = e[2] <= BOX_PITCH && e[0] * e[1] * BOX_PITCH <= BOX_CAP;
    for (int a = 0; a < 3; ++a) fits = fits && e[a] <= n[a] && out[a] >= -n[a] && out[a] + e[a] <= 2 * n[a];
    out[3] = fits ? e[0] : -1;
    if (fits && max_words) atomicMax(max_words, e[0] * e[1] * BOX_PITCH);
    if (!fits && max_words) atomicAdd(max_words + 1, 1);  // misfit tiles
    out[4] = e[1];
    out[5] = e[2];
  }
}

// ---- smem box I/O ----------------------------------------------------------
// Warps walk box rows (u1 outer, u2 strided by warp), lanes the columns. Box
// coordinates stay within one period of the grid (ext < n), so periodic wrap
// is a single conditional add/subtract -- no integer division anywhere.

__device__ __forceinline__ int wrap_once(int x, int n) {
  return x < 0 ? x + n : (x >= n ? x - n : x);
}

__device__ __forceinline__ void cp_async4(float* smem, const float* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Issue the box load as cp.async (LDGSTS: no register staging); the caller
// overlaps its own global loads and then calls cp_async_wait_all() +
// __syncthreads().
__device__ __forceinline__ void cp_async16(float* smem, const float* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// Rows of 16-byte chunks (n3 % 4 == 0: boxes are 4-aligned in x3, see
// k_tile_boxes): a half-warp per box row, 16 rows per CTA pass. The global
// start of every box row (x1 wrap or ghost plane, x2 wrap) is resolved once
// per tile into a shared row table, so the copy loops are one table load, an
// add and the 16-byte transfer per row.
constexpr int BOX_ROWS_MAX = BOX_CAP / BOX_PITCH;

__device__ __forceinline__ bool box_vec(const Geo& g) { return (g.n3 & 3) == 0; }

template <bool DIST, class Field, class T>
__device__ __forceinline__ void box_rows(const Geo& g, const Field& f, const TileBox& b, T** rows) {
  const int nr = b.ext[0] * b.ext[1];
  for (int r = threadIdx.x; r < nr; r += TILE_THREADS) {
    const int u1 = r / b.ext[1], u2 = r - u1 * b.ext[1];
    int p1 = b.lo[0] + u1;
    if constexpr (!DIST) p1 = wrap_once(p1, g.n1);
    rows[r] = f.plane_ptr(p1, g) + size_t(wrap_once(b.lo[1] + u2, g.n2)) * g.n3;
  }
}

// box_vec(g): `rows` must be filled (box_rows + __syncthreads) before the call
template <bool DIST>
__device__ __forceinline__ void load_box(const Geo& g, const SrcField<DIST>& src,
                                         const TileBox& b, float* sbox,
                                         const float* const* rows) {
  if (box_vec(g)) {
    const int q = threadIdx.x & 15;
    if (4 * q < b.ext[2]) {
      const int c = wrap_once(b.lo[2] + 4 * q, g.n3);
      const int nr = b.ext[0] * b.ext[1];
      for (int r = threadIdx.x >> 4; r < nr; r += TILE_THREADS / 16)
        cp_async16(sbox + r * BOX_PITCH + 4 * q, rows[r] + c);
    }
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c0 = wrap_once(b.lo[2] + lane, g.n3);
  int c1 = wrap_once(b.lo[2] + lane + 32, g.n3);
  for (int u1 = 0; u1 < b.ext[0]; ++u1) {
    int p1 = b.lo[0] + u1;
    if constexpr (!DIST) p1 = wrap_once(p1, g.n1);
    const float* P = src.plane_ptr(p1, g);
    float* SP = sbox + u1 * b.ext[1] * BOX_PITCH;
    for (int u2 = warp; u2 < b.ext[1]; u2 += TILE_THREADS / 32) {
      const float* R = P + size_t(wrap_once(b.lo[1] + u2, g.n2)) * g.n3;
      float* S = SP + u2 * BOX_PITCH;
      if (lane < b.ext[2]) cp_async4(S + lane, R + c0);
      if (lane + 32 < b.ext[2]) cp_async4(S + lane + 32, R + c1);
    }
  }
}

template <bool DIST>
__device__ __forceinline__ void flush_box(const Geo& g, const DstField<DIST>& dst,
                                          const TileBox& b, const int* sbox, float invS,
                                          float* const* rows) {
  if (box_vec(g)) {
    const int q = threadIdx.x & 15;
    if (4 * q < b.ext[2]) {
      const int c = wrap_once(b.lo[2] + 4 * q, g.n3);
      const int nr = b.ext[0] * b.ext[1];
      for (int r = threadIdx.x >> 4; r < nr; r += TILE_THREADS / 16) {
        const int4 v = *reinterpret_cast<const int4*>(sbox + r * BOX_PITCH + 4 * q);
        if ((v.x | v.y | v.z | v.w) != 0)
          atomicAdd(reinterpret_cast<float4*>(rows[r] + c),
                    make_float4(float(v.x) * invS, float(v.y) * invS, float(v.z) * invS,
                                float(v.w) * invS));
      }
    }
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c0 = wrap_once(b.lo[2] + lane, g.n3);
  int c1 = wrap_once(b.lo[2] + lane + 32, g.n3);
  for (int u1 = 0; u1 < b.ext[0]; ++u1) {
    int p1 = b.lo[0] + u1;
    if constexpr (!DIST) p1 = wrap_once(p1, g.n1);
    float* P = dst.plane_ptr(p1, g);
    const int* SP = sbox + u1 * b.ext[1] * BOX_PITCH;
    for (int u2 = warp; u2 < b.ext[1]; u2 += TILE_THREADS / 32) {
      float* R = P + size_t(wrap_once(b.lo[1] + u2, g.n2)) * g.n3;
      const int* S = SP + u2 * BOX_PITCH;
      if (lane < b.ext[2]) {
        const int v = S[lane];
        if (v != 0) atomicAdd(R + c0, float(v) * invS);
      }
      if (lane + 32 < b.ext[2]) {
        const int v = S[lane + 32];
        if (v != 0) atomicAdd(R + c1, float(v) * invS);
      }
    }
  }
}

// Integer flush: the box (int32 at the sweep's global scale) is added into
// the int32 accumulator field with integer atomics -- exact, so the result
// does not depend on the order tiles (or ranks) arrive in.
template <bool DIST>
__device__ __forceinline__ void flush_box_fixed(const Geo& g, const DstField<DIST>& dst,
                                                const TileBox& b, const int* sbox,
                                                float* const* rows) {
  if (box_vec(g)) {
    const int q = threadIdx.x & 15;
    if (4 * q < b.ext[2]) {
      const int c = wrap_once(b.lo[2] + 4 * q, g.n3);
      const int nr = b.ext[0] * b.ext[1];
      for (int r = threadIdx.x >> 4; r < nr; r += TILE_THREADS / 16) {
        const int4 v = *reinterpret_cast<const int4*>(sbox + r * BOX_PITCH + 4 * q);
        // two adjacent cells per 64-bit atomic: lo + 2^32 hi is exact in
        // int64 and decodes uniquely while each cell's total fits int32
        unsigned long long* R = reinterpret_cast<unsigned long long*>(rows[r] + c);
        if (v.x | v.y)
          atomicAdd(R, (unsigned long long)((long long)v.x + ((long long)v.y << 32)));
        if (v.z | v.w)
          atomicAdd(R + 1, (unsigned long long)((long long)v.z + ((long long)v.w << 32)));
      }
    }
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c0 = wrap_once(b.lo[2] + lane, g.n3);
  int c1 = wrap_once(b.lo[2] + lane + 32, g.n3);
  for (int u1 = 0; u1 < b.ext[0]; ++u1) {
    int p1 = b.lo[0] + u1;
    if constexpr (!DIST) p1 = wrap_once(p1, g.n1);
    int* P = reinterpret_cast<int*>(dst.plane_ptr(p1, g));
    const int* SP = sbox + u1 * b.ext[1] * BOX_PITCH;
    for (int u2 = warp; u2 < b.ext[1]; u2 += TILE_THREADS / 32) {
      int* R = P + size_t(wrap_once(b.lo[1] + u2, g.n2)) * g.n3;
      const int* S = SP + u2 * BOX_PITCH;
      if (lane < b.ext[2] && S[lane]) fixed_add(R + c0, S[lane], fixed_packed(g));
      if (lane + 32 < b.ext[2] && S[lane + 32]) fixed_add(R + c1, S[lane + 32], fixed_packed(g));
    }
  }
}

// ---- per-point stencil in box coordinates ---------------------------------

template <int DEG>
struct BoxStencil {
  static constexpr int NN = Basis<DEG>::NN, O0 = Basis<DEG>::O0;
  int base;  // smem word index of tap (0,0,0)
  float w1[NN], w2[NN], w3[NN];

  // false if the stencil leaves the box (stale cache) -> caller falls back
  __device__ __forceinline__ bool build(const TileBox& b, int i, int j, int k, float d1, float d2,
                                        float d3) {
    int b1, b2, b3;
    float s1, s2, s3;
    split_axis(d1, i, b1, s1);
    split_axis(d2, j, b2, s2);
    split_axis(d3, k, b3, s3);
    const int r1 = b1 + O0 - b.lo[0], r2 = b2 + O0 - b.lo[1], r3 = b3 + O0 - b.lo[2];
    const bool in = (unsigned)r1 <= unsigned(b.ext[0] - NN) &&
                    (unsigned)r2 <= unsigned(b.ext[1] - NN) &&
                    (unsigned)r3 <= unsigned(b.ext[2] - NN);
    lagrange_weights<DEG>(s1, w1);
    lagrange_weights<DEG>(s2, w2);
    lagrange_weights<DEG>(s3, w3);
    base = (r1 * b.ext[1] + r2) * BOX_PITCH + r3;
    return in;
  }

  __device__ __forceinline__ float gather(const TileBox& b, const float* sbox) const {
    const int e23 = b.ext[1] * BOX_PITCH;
    if constexpr (NN == 4) {
      // packed fp32x2 (FFMA2): tap pairs (c0,c1), (c2,c3) of each row with
      // the outer-product weights w2[bb] w3[c]; planes folded with w1.
      const float2 w3a = make_float2(w3[0], w3[1]), w3b = make_float2(w3[2], w3[3]);
      float2 w23[NN][2];
#pragma unroll
      for (int bb = 0; bb < NN; ++bb) {
        const float2 wb = make_float2(w2[bb], w2[bb]);
        w23[bb][0] = __fmul2_rn(wb, w3a);
        w23[bb][1] = __fmul2_rn(wb, w3b);
      }
      float2 F = make_float2(0.f, 0.f);
#pragma unroll
      for (int a = 0; a < NN; ++a) {
        const float* P = sbox + base + a * e23;
        float2 acc = __fmul2_rn(w23[0][0], make_float2(P[0], P[1]));
        acc = __ffma2_rn(w23[0][1], make_float2(P[2], P[3]), acc);
#pragma unroll
        for (int bb = 1; bb < NN; ++bb) {
          const float* R = P + bb * BOX_PITCH;
          acc = __ffma2_rn(w23[bb][0], make_float2(R[0], R[1]), acc);
          acc = __ffma2_rn(w23[bb][1], make_float2(R[2], R[3]), acc);
        }
        F = __ffma2_rn(make_float2(w1[a], w1[a]), acc, F);
      }
      return F.x + F.y;
    }
    float acc1 = 0.f;
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      float acc2 = 0.f;
#pragma unroll
      for (int bb = 0; bb < NN; ++bb) {
        const float* R = sbox + base + a * e23 + bb * BOX_PITCH;
        float acc3 = 0.f;
#pragma unroll
        for (int c = 0; c < NN; ++c) acc3 += w3[c] * R[c];
        acc2 += w2[bb] * acc3;
      }
      acc1 += w1[a] * acc2;
    }
    return acc1;
  }

  // Fixed-point contributions round(zS w1 w2 w3). The final product and its
  // rounding run as one DFMA against 1.5 * 2^52 (the low word of the sum is
  // the rounded integer, two's complement, for |x| < 2^51): F2I sits on the
  // quarter-rate XU pipe and bound this kernel, DFMA is half-rate FP64.
  __device__ __forceinline__ void scatter(const TileBox& b, int* sbox, float zS) const {
    const int e23 = b.ext[1] * BOX_PITCH;
    constexpr double MAGIC = 6755399441055744.0;  // 1.5 * 2^52
    double w3d[NN];
#pragma unroll
    for (int c = 0; c < NN; ++c) w3d[c] = double(w3[c]);
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      const float za = w1[a] * zS;
#pragma unroll
      for (int bb = 0; bb < NN; ++bb) {
        int* R = sbox + base + a * e23 + bb * BOX_PITCH;
        const double zab = double(za * w2[bb]);
#pragma unroll
        for (int c = 0; c < NN; ++c) atomicAdd(R + c, __double2loint(fma(zab, w3d[c], MAGIC)));
      }
    }
  }
};

// ---- per-point global fallbacks (rare; kept out of line) -------------------

template <int DEG, bool DIST>
__device__ __noinline__ float point_gather(const Geo& g, const SrcField<DIST> src, int i, int j,
                                           int k, float d1, float d2, float d3) {
  Stencil<DEG> st;
  st.template build<DIST>(g, i, j, k, d1, d2, d3);
  return st.gather(g, src);
}

template <int DEG, bool DIST>
__device__ __noinline__ void point_scatter_fixed(const Geo& g, const DstField<DIST> dst, int i,
                                                 int j, int k, float d1, float d2, float d3,
                                                 float zS) {
  Stencil<DEG> st;
  st.template build<DIST>(g, i, j, k, d1, d2, d3);
  st.scatter_fixed(g, dst, zS);
}

template <int DEG, bool DIST>
__device__ __noinline__ void point_scatter(const Geo& g, const DstField<DIST> dst, int i, int j,
                                           int k, float d1, float d2, float d3, float z) {
  Stencil<DEG> st;
  st.template build<DIST>(g, i, j, k, d1, d2, d3);
  st.scatter(g, dst, z);
}

}  // namespace vb
