// Persistent, warp-specialised SL gather sweeps fed by the Tensor Memory
// Accelerator (the gather of interp.cpp:70-108, fused into the transport
// steps of transport.hpp). The transpose sweeps stay on the 3-CTA/SM tile
// kernels of sl_tile.cuh: a pipelined variant (accumulate in the consumer
// warps, flush by the producer group) measured 332 us against 267 us at
// 256^3 -- one CTA per SM serialises the atomic and flush phases that three
// independent CTAs overlap.
//
// One CTA per SM walks the 4 x 16 x 32 departure-point tiles of a launch
// (tile = blockIdx.x + n * gridDim.x, x3 fastest, so co-resident CTAs work on
// neighbouring tiles and their box halos meet in L2) through a ring of
// PIPE_STAGES shared-memory stages:
//
//   producer       (4 warps) wait `empty[s]`, then for the next tile
//                  * cp.async.bulk.tensor (UTMALDG): the tile's 3 displacement
//                    components and its per-point stream (u_t / q / z) as
//                    32 x 16 x 4 boxes of 3-D tensor maps,
//                  * 16-byte cp.async (LDGSTS): the source box (the cells the
//                    tile's stencils reach, k_tile_boxes), periodic wrap and
//                    multi-rank ghost planes resolved per chunk; completion
//                    through cp.async.mbarrier.arrive.noinc on `full[s]`.
//                    (Per-row cp.async.bulk copies were measured 2x slower:
//                    ~150 160-byte bulk requests per tile serialise in the
//                    TMA unit; tensor boxes cannot wrap periodically.)
//   16 consumer    wait `full[s]`, contract the taps from shared memory and
//   warps          write their outputs, then release the stage (`empty[s]`).
//
// The consumers never touch global memory for inputs, so box staging, the
// displacement stream and the previous tile's taps overlap.
#pragma once

#include <cuda.h>

#include "sl_tile.cuh"

namespace vb {

constexpr int PIPE_CONS_WARPS = 16;
constexpr int PIPE_CONS = PIPE_CONS_WARPS * 32;     // consumer threads
constexpr int PIPE_PROD_WARPS = 4;                   // producer warps (one per SM sub-partition)
constexpr int PIPE_PROD = PIPE_PROD_WARPS * 32;
constexpr int PIPE_THREADS = PIPE_CONS + PIPE_PROD;
constexpr int PIPE_STAGES = 2;
constexpr int PIPE_PPT = TILE_POINTS / PIPE_CONS;    // points per consumer thread (4)
// Box rows sit at a pitch of 64 words (and planes at e2 * 64): lanes whose
// stencils start on different rows or planes then differ only in their x3
// offset, so they keep hitting distinct banks (a 48-word pitch doubled the
// shared-memory wavefronts through bank conflicts, ncu).
constexpr int PIPE_P3 = 64;                          // box row pitch in smem (words)
constexpr int PIPE_BOX_WORDS = 19456;                // box capacity per stage (304 rows)
constexpr int PIPE_BOX_ROWS = PIPE_BOX_WORDS / PIPE_P3;
constexpr int PIPE_AUX_OFF = 3 * TILE_POINTS;        // stage layout (words): D | aux | box
constexpr int PIPE_BOX_OFF = 4 * TILE_POINTS;
constexpr int PIPE_STAGE_WORDS = PIPE_BOX_OFF + PIPE_BOX_WORDS;
constexpr size_t PIPE_SMEM = size_t(PIPE_STAGES) * PIPE_STAGE_WORDS * sizeof(float) + 128;
static_assert(PIPE_PPT == 4, "four points per consumer thread");

// per-stage tile descriptor written by the producer (box ext[0] < 0: no box)
struct PipeHdr {
  int lo[3], ext[3], t[3], pad;
};

// ---- mbarrier / TMA primitives ----------------------------------------------

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
// 3-D tensor tile (x3, x2, plane) -> smem, completing on bar
__device__ __forceinline__ void tma_tile3(float* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar))
      : "memory");
}
// Tiles of one launch: nz x1 layers (TileZ mapping) x ty x tx.
struct PipeTiles {
  int tx, ty, n;
  __device__ __forceinline__ void coords(int tile, const TileZ& zm, int& layer, int& y,
                                         int& x) const {
    x = tile % tx;
    const int r = tile / tx;
    y = r % ty;
    const int z = r / ty;
    layer = z < zm.zs ? zm.z0 + z : zm.z1 + (z - zm.zs);
  }
};

// Producer group (PIPE_PROD threads): stage one tile -- D and the optional
// point stream by TMA (thread 0), the source box by 16-byte LDGSTS. The
// global start of every box row (x1 wrap or multi-rank ghost plane, x2
// wrap) is resolved once into a row table; then 16 threads per row issue
// its chunks (x3 wrap per chunk; lo3 and e3 are multiples of 4 when
// n3 % 4 == 0, k_tile_boxes), so each instruction moves whole lines.
// Completion: thread 0's expect_tx arrival (TMA bytes) plus one
// cp.async.mbarrier.arrive.noinc per producer thread.
template <bool DIST, class Field, class RowT>
__device__ __forceinline__ void pipe_produce(const Geo& g, const Field& src, const int* boxes,
                                             const CUtensorMap* tmD, const CUtensorMap* tmA,
                                             bool load_box, const PipeTiles& pt, const TileZ& zm,
                                             int tile, float* st, PipeHdr* hdr, RowT** rows,
                                             uint64_t* full) {
  const int t = threadIdx.x - PIPE_CONS;
  int layer, y, x;
  pt.coords(tile, zm, layer, y, x);
  const TileBox b = load_tile_box(boxes, (layer * pt.ty + y) * pt.tx + x);
  const bool fits =
      load_box && b.ext[0] > 0 && b.ext[2] <= PIPE_P3 && b.ext[0] * b.ext[1] <= PIPE_BOX_ROWS;
  if (t == 0) {
    PipeHdr h;
    for (int a = 0; a < 3; ++a) {
      h.lo[a] = b.lo[a];
      h.ext[a] = b.ext[a];
    }
    if (!fits) h.ext[0] = -1;
    h.t[0] = layer * TT1;
    h.t[1] = y * TT2;
    h.t[2] = x * TT3;
    h.pad = 0;
    *hdr = h;
    mbar_expect_tx(full, 3u * TILE_POINTS * 4u + (tmA ? TILE_POINTS * 4u : 0u));
#pragma unroll
    for (int c = 0; c < 3; ++c)
      tma_tile3(st + c * TILE_POINTS, tmD, x * TT3, y * TT2, c * g.n1l + layer * TT1, full);
    if (tmA) tma_tile3(st + PIPE_AUX_OFF, tmA, x * TT3, y * TT2, layer * TT1, full);
  }
  const int nr = fits ? b.ext[0] * b.ext[1] : 0;
  for (int r = t; r < nr; r += PIPE_PROD) {
    const int u1 = r / b.ext[1], u2 = r - u1 * b.ext[1];
    int p1 = b.lo[0] + u1;
    if constexpr (!DIST) p1 = wrap_once(p1, g.n1);
    rows[r] = src.plane_ptr(p1, g) + size_t(wrap_once(b.lo[1] + u2, g.n2)) * g.n3;
  }
  // producer group only; every tile, so no thread rewrites a stage's row
  // table while another still issues that stage's previous tile
  asm volatile("bar.sync 1, %0;" ::"n"(PIPE_PROD) : "memory");
  if (fits) {
    const int q = t & 15;
    if (4 * q < b.ext[2]) {
      float* sb = st + PIPE_BOX_OFF + 4 * q;
      const int col = wrap_once(b.lo[2] + 4 * q, g.n3);
      for (int r = t >> 4; r < nr; r += PIPE_PROD / 16) cp_async16(sb + r * PIPE_P3, rows[r] + col);
    }
  }
  // arrives once this thread's box chunks have landed
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(full))
               : "memory");
}

// ---- per-point stencil in pipe-box coordinates (row pitch PIPE_P3) ----------

template <int DEG>
struct PipeStencil {
  static constexpr int NN = Basis<DEG>::NN, O0 = Basis<DEG>::O0;
  int base;
  float w1[NN], w2[NN], w3[NN];

  // b: box origin (lo), e: extents; false if the stencil leaves the box
  __device__ __forceinline__ bool build(const PipeHdr& h, int i, int j, int k, float d1, float d2,
                                        float d3) {
    int b1, b2, b3;
    float s1, s2, s3;
    split_axis(d1, i, b1, s1);
    split_axis(d2, j, b2, s2);
    split_axis(d3, k, b3, s3);
    const int r1 = b1 + O0 - h.lo[0], r2 = b2 + O0 - h.lo[1], r3 = b3 + O0 - h.lo[2];
    const bool in = (unsigned)r1 <= unsigned(h.ext[0] - NN) &&
                    (unsigned)r2 <= unsigned(h.ext[1] - NN) &&
                    (unsigned)r3 <= unsigned(h.ext[2] - NN);
    lagrange_weights<DEG>(s1, w1);
    lagrange_weights<DEG>(s2, w2);
    lagrange_weights<DEG>(s3, w3);
    base = (r1 * h.ext[1] + r2) * PIPE_P3 + r3;
    return in;
  }

  __device__ __forceinline__ float gather(int e2, const float* sbox) const {
    const int e23 = e2 * PIPE_P3;
    if constexpr (NN == 4) {
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
          const float* R = P + bb * PIPE_P3;
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
        const float* R = sbox + base + a * e23 + bb * PIPE_P3;
        float acc3 = 0.f;
#pragma unroll
        for (int c = 0; c < NN; ++c) acc3 += w3[c] * R[c];
        acc2 += w2[bb] * acc3;
      }
      acc1 += w1[a] * acc2;
    }
    return acc1;
  }
};

// ---- the gather sweep -------------------------------------------------------
// MODE 0: out = I[f] (.* aux when has_aux); MODE 2: inc-state step on the
// precomputed u_{t+1} (aux): m = I[w_t] - dt/2 u, out = last ? -m : m - dt/2 u
// (mt_out = m optional); MODE 3: adjoint source factor, src = aux = d:
// out = (1 + dt/2 I[d]) / (1 - dt/2 d) (transport.hpp:55-60).
template <int DEG, bool DIST, int MODE>
__global__ void __launch_bounds__(PIPE_THREADS, 1)
    k_gather_pipe(Geo g, SrcField<DIST> src, const int* __restrict__ boxes,
                  const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmA,
                  int has_aux, float* __restrict__ out, float half, int last,
                  float* __restrict__ mt_out, TileZ zm, PipeTiles pt, int* __restrict__ sched,
                  float* __restrict__ zero_out) {
  extern __shared__ __align__(128) float pipe_raw[];
  __shared__ int next_tile;
  __shared__ __align__(8) uint64_t full[PIPE_STAGES], empty[PIPE_STAGES];
  __shared__ PipeHdr hdr[PIPE_STAGES];
  __shared__ const float* rows[PIPE_STAGES][PIPE_BOX_ROWS];
  // 128-byte aligned stage base; pointer arithmetic on the __shared__ array
  // keeps the accesses in the shared window (LDS, 32-bit addresses)
  float* smem = pipe_raw + ((128u - (smem_addr(pipe_raw) & 127u)) & 127u) / 4u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < PIPE_STAGES; ++s) {
      mbar_init(&full[s], 1 + PIPE_PROD);  // expect_tx + one cp.async arrival per producer
      mbar_init(&empty[s], PIPE_CONS_WARPS);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp >= PIPE_CONS_WARPS) {  // ---- producer group
    // static round robin, or (sched != nullptr) tiles taken from a global
    // ticket counter, so CTAs that start late -- their SMs still busy with
    // another kernel -- take fewer tiles instead of delaying the sweep (the
    // multi-rank boundary layers, launched while the interior sweep drains)
    const int t = threadIdx.x - PIPE_CONS;
    for (int it = 0;; ++it) {
      const int s = it % PIPE_STAGES;
      mbar_wait(&empty[s], ((it / PIPE_STAGES) & 1) ^ 1);
      int tile;
      if (sched) {
        if (t == 0) next_tile = atomicAdd(&sched[0], 1);
        asm volatile("bar.sync 1, %0;" ::"n"(PIPE_PROD) : "memory");
        tile = next_tile;
      } else {
        tile = int(blockIdx.x) + it * int(gridDim.x);
      }
      if (tile >= pt.n) {  // sentinel stage: the consumers stop on it
        if (t == 0) {
          hdr[s].t[0] = -1;
          mbar_expect_tx(&full[s], 0u);
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                         smem_addr(&full[s]))
                     : "memory");
        // the last CTA out rewinds the counter for the next launch
        if (sched && t == 0) {
          __threadfence();
          if (atomicAdd(&sched[1], 1) == int(gridDim.x) - 1) {
            atomicExch(&sched[0], 0);
            atomicExch(&sched[1], 0);
          }
        }
        return;
      }
      pipe_produce<DIST>(g, src, boxes, &tmD, has_aux ? &tmA : nullptr, true, pt, zm, tile,
                         smem + s * PIPE_STAGE_WORDS, &hdr[s], rows[s], &full[s]);
    }
  }
  // ---- consumers: thread = points (g1 + q1, g2 + q2, lane), q1, q2 in {0, 1}
  const int g1 = 2 * (warp >> 3), g2 = 2 * (warp & 7);
  for (int it = 0;; ++it) {
    const int s = it % PIPE_STAGES;
    mbar_wait(&full[s], (it / PIPE_STAGES) & 1);
    const PipeHdr h = hdr[s];
    if (h.t[0] < 0) break;
    const float* st = smem + s * PIPE_STAGE_WORDS;
    const bool fits = h.ext[0] > 0;
    const int k = h.t[2] + lane;
#pragma unroll
    for (int q = 0; q < PIPE_PPT; ++q) {
      const int a1 = g1 + (q >> 1), a2 = g2 + (q & 1);
      const int i = h.t[0] + a1, j = h.t[1] + a2;
      if (i >= g.n1l || j >= g.n2 || k >= g.n3) continue;
      const int idx = (a1 * TT2 + a2) * TT3 + lane;
      const float d1 = st[idx], d2 = st[TILE_POINTS + idx], d3 = st[2 * TILE_POINTS + idx];
      float G;
      PipeStencil<DEG> ps;
      if (fits && ps.build(h, i, j, k, d1, d2, d3))
        G = ps.gather(h.ext[1], st + PIPE_BOX_OFF);
      else
        G = point_gather<DEG, DIST>(g, src, i, j, k, d1, d2, d3);
      const size_t p = (size_t(i) * g.n2 + j) * g.n3 + k;
      if constexpr (MODE == 0) {
        out[p] = has_aux ? G * st[PIPE_AUX_OFF + idx] : G;
      } else if constexpr (MODE == 3) {
        out[p] = (1.0f + half * G) / (1.0f - half * st[PIPE_AUX_OFF + idx]);
      } else {
        const float u = st[PIPE_AUX_OFF + idx];
        const float m = G - half * u;
        if (mt_out) mt_out[p] = m;
        out[p] = last ? -m : m - half * u;
        if (zero_out) zero_out[p] = 0.0f;  // a transpose sweep's output, pre-zeroed here
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

}  // namespace vb
