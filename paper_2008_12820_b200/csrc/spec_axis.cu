// Separable H1 regulariser: beta (-Lap) v = beta (D_1 + D_2 + D_3) v with
// D_a = F_a^-1 diag(k_a^2) F_a the 1-D spectral second derivative along x_a.
//
// The reference applies beta |k|^2 through a 3-D r2c -> symbol -> c2r
// (spectral.cpp:48-70). The 3-D DFT is separable and |k|^2 = k1^2 + k2^2 +
// k3^2 (every k_a^2 is real and even, Nyquist included), so the same
// operator is three 1-D passes, each one read of v and one read-modify-write
// of the output (32 B per voxel and component) instead of the six cuFFT
// passes plus the symbol pass (~56 B/voxel/comp) of the 3-D route.
//
// Pass layout: a CTA owns 32 real pencils of length N along the pass axis
// (x3 pass: 32 consecutive rows; x2 / x1 passes: 32 consecutive x3 columns,
// 128-byte coalesced rows). Real pencils are paired into 16 complex pencils
// (D_a is real, so D_a (x + i y) = D_a x + i D_a y). Each complex pencil is
// transformed by a four-step FFT N = 16 * R2 held in registers: R2-point
// DFTs over n2, twiddle W_N^{n1 k2}, one shared-memory transpose, 16-point
// DFTs over n1; the symbol is applied in registers and the inverse runs the
// same steps backwards, so the pencil crosses shared memory twice.
#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"

namespace vb {

namespace {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmul_conj(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

// exp(SIGN * 2 pi i m / 32), m in [0, 16): compile-time index after unrolling
template <int SIGN>
__device__ __forceinline__ float2 unit32(int m) {
  constexpr float C[16] = {1.000000000e+00f,  9.807852804e-01f,  9.238795325e-01f,
                           8.314696123e-01f,  7.071067812e-01f,  5.555702330e-01f,
                           3.826834324e-01f,  1.950903220e-01f,  0.0f,
                           -1.950903220e-01f, -3.826834324e-01f, -5.555702330e-01f,
                           -7.071067812e-01f, -8.314696123e-01f, -9.238795325e-01f,
                           -9.807852804e-01f};
  constexpr float S[16] = {0.0f,             1.950903220e-01f, 3.826834324e-01f,
                           5.555702330e-01f, 7.071067812e-01f, 8.314696123e-01f,
                           9.238795325e-01f, 9.807852804e-01f, 1.000000000e+00f,
                           9.807852804e-01f, 9.238795325e-01f, 8.314696123e-01f,
                           7.071067812e-01f, 5.555702330e-01f, 3.826834324e-01f,
                           1.950903220e-01f};
  return make_float2(C[m], SIGN * S[m]);
}

template <int R>
__host__ __device__ constexpr int bit_reverse(int i) {
  int r = 0;
  for (int b = 1; b < R; b <<= 1) {
    r = (r << 1) | (i & 1);
    i >>= 1;
  }
  return r;
}

template <int R, int LEN, int SIGN>
__device__ __forceinline__ void dit_stages(float2 (&b)[R]) {
  if constexpr (LEN <= R) {
#pragma unroll
    for (int i = 0; i < R; i += LEN) {
#pragma unroll
      for (int j = 0; j < LEN / 2; ++j) {
        float2 t = b[i + j + LEN / 2];
        if (j != 0) t = cmul(t, unit32<SIGN>(j * (32 / LEN)));
        const float2 u = b[i + j];
        b[i + j] = make_float2(u.x + t.x, u.y + t.y);
        b[i + j + LEN / 2] = make_float2(u.x - t.x, u.y - t.y);
      }
    }
    dit_stages<R, LEN * 2, SIGN>(b);
  }
}

// In-register DFT of size R (power of two, <= 32), natural order in and out;
// SIGN -1 forward, +1 inverse (unnormalised).
template <int R, int SIGN>
__device__ __forceinline__ void dft(float2 (&a)[R]) {
  if constexpr (R > 1) {
    float2 b[R];
#pragma unroll
    for (int i = 0; i < R; ++i) b[bit_reverse<R>(i)] = a[i];
    dit_stages<R, 2, SIGN>(b);
#pragma unroll
    for (int i = 0; i < R; ++i) a[i] = b[i];
  }
}

constexpr int AX_THREADS = 256;

// Pencil decomposition N = T1 * R2: T1 threads per complex pencil, NP
// complex (2 NP real) pencils per CTA; 1024-point pencils use 32 threads so
// a thread still holds 32 values.
template <int N>
struct AxisShape {
  static constexpr int T1 = N <= 512 ? 16 : 32;
  static constexpr int NP = AX_THREADS / T1;
};

// out (+)= coef * D_ax v over all 3 components. coef = beta / N (1-D
// inverse normalisation folded in); tw[m] = exp(-2 pi i m / N). CTAs walk
// the (component, tile) list with a grid stride: one tile each when the grid
// covers the list, a persistent sweep when the grid is capped (the matvec's
// side stream, so the sweep shares the SMs with the SL kernels).
template <int N, int AX>
__global__ void __launch_bounds__(AX_THREADS, N <= 256 ? 3 : 2) k_axis_d2(int n1l, int n2, int n3,
                                                         int tiles,
                                                         const float* __restrict__ v,
                                                         float* __restrict__ out,
                                                         const float2* __restrict__ tw,
                                                         float coef, int accumulate,
                                                         const double* __restrict__ bias_sums,
                                                         double bias_scale) {
  constexpr int T1 = AxisShape<N>::T1, NP = AxisShape<N>::NP, WQ = 2 * NP;
  constexpr int R2 = N / T1;
  constexpr int SK = T1 + 1, SP = R2 * SK + 1;  // odd float2 pitches: conflict-free
  extern __shared__ float2 S[];  // NP * SP
  const size_t nloc = size_t(n1l) * n2 * n3;
  for (int t = blockIdx.x; t < 3 * tiles; t += gridDim.x) {
  const int comp = t / tiles, tile = t - comp * tiles;
  const float* vc = v + size_t(comp) * nloc;
  float* oc = out + size_t(comp) * nloc;
  // unit null-mode symbol: + beta * mean(v_c) on the writing (first) pass
  const float bias = bias_sums ? float(bias_scale * bias_sums[comp]) : 0.0f;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  (void)w;
  (void)l;
  // x3 pass: T1 lanes run along a row (n1 fastest); x2/x1 passes: along the
  // NP column pairs of a row segment (p fastest)
  const int n1 = AX == 3 ? int(threadIdx.x) % T1 : int(threadIdx.x) / NP;
  const int p = AX == 3 ? int(threadIdx.x) / T1 : int(threadIdx.x) % NP;
  size_t base, js, qs;
  if constexpr (AX == 3) {
    base = size_t(tile) * WQ * n3;
    js = 1;
    qs = size_t(n3);
  } else {
    const int nb = n3 / WQ;
    const int r = tile / nb, xb = tile - r * nb;
    base = (AX == 2 ? size_t(r) * n2 * n3 : size_t(r) * n3) + size_t(xb) * WQ;
    js = AX == 2 ? size_t(n3) : size_t(n2) * n3;
    qs = 1;
  }
  const size_t off = base + size_t(2 * p) * qs + size_t(n1) * js;

  if (accumulate) {  // pull the output rows towards L2 while v streams in
#pragma unroll
    for (int m = 0; m < R2; ++m) {
      const float* q = oc + off + size_t(T1 * m) * js;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
      if constexpr (AX == 3) asm volatile("prefetch.global.L2 [%0];" ::"l"(q + qs));
    }
  }
  float2 a[R2];
#pragma unroll
  for (int m = 0; m < R2; ++m) {
    const float* q = vc + off + size_t(T1 * m) * js;
    if constexpr (AX == 3)
      a[m] = make_float2(__ldg(q), __ldg(q + qs));
    else
      a[m] = __ldg(reinterpret_cast<const float2*>(q));
  }
  dft<R2, -1>(a);
  float2* Sp = S + p * SP;
#pragma unroll
  for (int k2 = 0; k2 < R2; ++k2) {
    if (k2 != 0 && n1 != 0) a[k2] = cmul(a[k2], __ldg(tw + n1 * k2));
    Sp[k2 * SK + n1] = a[k2];
  }
  __syncthreads();
  for (int k2 = n1; k2 < R2; k2 += T1) {  // T1-point DFTs over n1, symbol, inverse
    float2 b[T1];
#pragma unroll
    for (int j = 0; j < T1; ++j) b[j] = Sp[k2 * SK + j];
    dft<T1, -1>(b);
#pragma unroll
    for (int k1 = 0; k1 < T1; ++k1) {
      const int f = k2 + R2 * k1;
      const float fs = float(f <= N / 2 ? f : f - N);
      const float m = coef * fs * fs;
      b[k1].x *= m;
      b[k1].y *= m;
    }
    dft<T1, 1>(b);
#pragma unroll
    for (int j = 0; j < T1; ++j) Sp[k2 * SK + j] = b[j];
  }
  __syncthreads();
#pragma unroll
  for (int k2 = 0; k2 < R2; ++k2) {
    a[k2] = Sp[k2 * SK + n1];
    if (k2 != 0 && n1 != 0) a[k2] = cmul_conj(a[k2], __ldg(tw + n1 * k2));
  }
  dft<R2, 1>(a);
#pragma unroll
  for (int m = 0; m < R2; ++m) {
    float* q = oc + off + size_t(T1 * m) * js;
    if constexpr (AX == 3) {
      if (accumulate) {
        q[0] += a[m].x;
        q[qs] += a[m].y;
      } else {
        q[0] = a[m].x + bias;
        q[qs] = a[m].y + bias;
      }
    } else {
      float2* q2 = reinterpret_cast<float2*>(q);
      if (accumulate) {
        const float2 o = *q2;
        *q2 = make_float2(o.x + a[m].x, o.y + a[m].y);
      } else {
        *q2 = make_float2(a[m].x + bias, a[m].y + bias);
      }
    }
  }
  __syncthreads();  // S is reused by the next tile
  }
}

bool axis_size_ok(int n) { return n >= 32 && n <= 1024 && (n & (n - 1)) == 0; }

const float2* twiddles(vreg_ctx ctx, int n) {
  const std::string name = "axis_tw_" + std::to_string(n);
  if (ctx->ws.count(name)) return static_cast<const float2*>(ctx->ws[name].first);
  float2* d = static_cast<float2*>(workspace(ctx, name, size_t(n) * sizeof(float2)));
  std::vector<float2> h(n);
  const double two_pi = 6.283185307179586476925286766559;
  for (int m = 0; m < n; ++m)
    h[m] = make_float2(float(std::cos(two_pi * m / n)), float(-std::sin(two_pi * m / n)));
  // stream-ordered: the pool may hand back memory pending kernels still use
  VB_CUDA(cudaMemcpyAsync(d, h.data(), size_t(n) * sizeof(float2), cudaMemcpyHostToDevice,
                          ctx->stream));
  VB_CUDA(cudaStreamSynchronize(ctx->stream));  // once per size; h dies here
  return d;
}

// Geometry of the array a pass runs over: n1l planes of n2 x n3 (on p > 1
// the x1 pass runs on the x2-slab transpose: all n1 planes of n2/p rows).
struct AxisGeom {
  int n1l, n2, n3;
};

template <int AX>
void launch_axis(vreg_ctx ctx, const AxisGeom& s, int n, const float* v3, float* out3,
                 double beta, int accumulate, int ctas_per_sm,
                 const double* bias_sums = nullptr, double bias_scale = 0.0) {
  const int wq = n <= 512 ? 32 : 16;  // 2 * AxisShape<n>::NP
  const int tiles = AX == 3 ? int(size_t(s.n1l) * s.n2 / wq)
                            : (AX == 2 ? s.n1l : s.n2) * (s.n3 / wq);
  static const char* names[4] = {"", "spec_axis1", "spec_axis2", "spec_axis3"};
  Timed timer(ctx, T_FFT, names[AX]);
  int grid = 3 * tiles;
  if (ctas_per_sm > 0) {
    int dev = 0, sms = 0;
    VB_CUDA(cudaGetDevice(&dev));
    VB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = std::min(grid, sms * ctas_per_sm);
  }
  const float2* tw = twiddles(ctx, n);
  const float coef = float(beta / double(n));
#define VB_AXIS_CASE(NN)                                                                   \
  case NN: {                                                                               \
    const size_t smem = size_t(AxisShape<NN>::NP) *                                        \
                        ((NN / AxisShape<NN>::T1) * (AxisShape<NN>::T1 + 1) + 1) * sizeof(float2); \
    smem_optin(reinterpret_cast<const void*>(k_axis_d2<NN, AX>), int(smem));           \
    k_axis_d2<NN, AX><<<grid, AX_THREADS, smem, ctx->stream>>>(s.n1l, s.n2, s.n3, tiles, v3, \
                                                               out3, tw, coef, accumulate, \
                                                               bias_sums, bias_scale);     \
    break;                                                                                 \
  }
  switch (n) {
    VB_AXIS_CASE(32)
    VB_AXIS_CASE(64)
    VB_AXIS_CASE(128)
    VB_AXIS_CASE(256)
    VB_AXIS_CASE(512)
    VB_AXIS_CASE(1024)
    default:
      require(false, VREG_EDIM, "axis transform size");
  }
#undef VB_AXIS_CASE
  count_launch(ctx);
  check_launch();
}

// x1-slab [c][i1l][j][k] -> blocks [c][q][i1l][j_l][k] (j = q n2l + j_l)
__global__ void k_axis_pack(int p, int n1l, int n2l, int n3, const float4* __restrict__ in,
                            float4* __restrict__ out) {
  const int n34 = n3 / 4;
  const size_t per = size_t(n1l) * p * n2l * n34;  // float4 per component
  const size_t total = 3 * per;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += size_t(gridDim.x) * blockDim.x) {
    const int c = int(e / per);
    size_t r = e - size_t(c) * per;
    const int k4 = int(r % n34);
    r /= n34;
    const int j = int(r % (size_t(p) * n2l));
    const int i = int(r / (size_t(p) * n2l));
    const int q = j / n2l, jl = j - q * n2l;
    out[((((size_t(c) * p + q) * n1l + i) * n2l + jl) * n34) + k4] = in[e];
  }
}

// out3[c][i1l][j][k] += blocks[c][q][i1l][j_l][k]
__global__ void k_axis_unpack_add(int p, int n1l, int n2l, int n3, const float4* __restrict__ in,
                                  float4* __restrict__ out) {
  const int n34 = n3 / 4;
  const size_t per = size_t(n1l) * p * n2l * n34;
  const size_t total = 3 * per;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += size_t(gridDim.x) * blockDim.x) {
    const int c = int(e / per);
    size_t r = e - size_t(c) * per;
    const int k4 = int(r % n34);
    r /= n34;
    const int j = int(r % (size_t(p) * n2l));
    const int i = int(r / (size_t(p) * n2l));
    const int q = j / n2l, jl = j - q * n2l;
    const float4 a = in[((((size_t(c) * p + q) * n1l + i) * n2l + jl) * n34) + k4];
    float4 o = out[e];
    o.x += a.x;
    o.y += a.y;
    o.z += a.z;
    o.w += a.w;
    out[e] = o;
  }
}

// Transpose buffers. Peer path: cudaMalloc'd send/recv buffers whose
// receive side is opened by every peer through CUDA IPC (handles all-gathered
// over NCCL; collective, every rank arrives with the same size).
bool axis_buffers(vreg_ctx ctx, size_t bytes, float** a, float** b) {
  static const bool peer = [] {
    const char* e = std::getenv("VREG_PEER_TRANSPOSE");
    return !(e && e[0] == '0');
  }();
  if (!peer) {
    *a = static_cast<float*>(workspace(ctx, "axis_a", bytes));
    *b = static_cast<float*>(workspace(ctx, "axis_b", bytes));
    return false;
  }
  if (ctx->xbytes < bytes) {
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (float* q : ctx->peer_recv)
      if (q) VB_CUDA(cudaIpcCloseMemHandle(q));
    ctx->peer_recv.clear();
    for (int i = 0; i < 2; ++i)
      if (ctx->xbuf[i]) VB_CUDA(cudaFree(ctx->xbuf[i]));
    for (int i = 0; i < 2; ++i) VB_CUDA(cudaMalloc(&ctx->xbuf[i], bytes));
    if (!ctx->xflag) VB_CUDA(cudaMalloc(&ctx->xflag, 64 * sizeof(int)));
    const int p = ctx->nranks;
    cudaIpcMemHandle_t h;
    VB_CUDA(cudaIpcGetMemHandle(&h, ctx->xbuf[1]));
    char* dh = nullptr;
    VB_CUDA(cudaMalloc(&dh, size_t(p + 1) * sizeof(h)));
    VB_CUDA(cudaMemcpyAsync(dh + size_t(p) * sizeof(h), &h, sizeof(h), cudaMemcpyHostToDevice,
                            ctx->stream));
    VB_NCCL(ncclAllGather(dh + size_t(p) * sizeof(h), dh, sizeof(h), ncclChar, ctx->comm,
                          ctx->stream));
    std::vector<cudaIpcMemHandle_t> all(p);
    VB_CUDA(cudaMemcpyAsync(all.data(), dh, size_t(p) * sizeof(h), cudaMemcpyDeviceToHost,
                            ctx->stream));
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
    VB_CUDA(cudaFree(dh));
    ctx->peer_recv.assign(p, nullptr);
    for (int q = 0; q < p; ++q) {
      if (q == ctx->rank) continue;
      void* ptr = nullptr;
      VB_CUDA(cudaIpcOpenMemHandle(&ptr, all[q], cudaIpcMemLazyEnablePeerAccess));
      ctx->peer_recv[q] = static_cast<float*>(ptr);
    }
    ctx->xbytes = bytes;
  }
  *a = ctx->xbuf[0];
  *b = ctx->xbuf[1];
  return true;
}

// Stream-ordered barrier across ranks (a 1-int all-reduce): on return every
// rank's earlier work on its stream is complete.
void axis_barrier(vreg_ctx ctx) {
  VB_NCCL(ncclAllReduce(ctx->xflag, ctx->xflag + 32, 1, ncclInt, ncclSum, ctx->comm,
                        ctx->stream));
}

// All-to-all of [c][q] blocks of `blk` floats, one per component: block
// (c, q) of `send` goes to rank q and lands at block (c, me) of its `recv`.
// Peer path: the copy engines write straight into the peers' receive buffers
// over NVLink (no SM time taken from the SL sweeps), bracketed by barriers
// (peers done reading the previous contents / all blocks landed).
void axis_alltoall(vreg_ctx ctx, const float* send, float* recv, size_t blk, bool peer) {
  const int p = ctx->nranks, me = ctx->rank;
  if (peer) {
    axis_barrier(ctx);
    for (int k = 1; k < p; ++k) {
      const int q = (me + k) % p;  // stagger the targets
      for (int c = 0; c < 3; ++c)
        VB_CUDA(cudaMemcpyAsync(ctx->peer_recv[q] + (size_t(c) * p + me) * blk,
                                send + (size_t(c) * p + q) * blk, blk * sizeof(float),
                                cudaMemcpyDeviceToDevice, ctx->stream));
    }
  } else {
    VB_NCCL(ncclGroupStart());
    for (int q = 0; q < p; ++q) {
      if (q == me) continue;
      for (int c = 0; c < 3; ++c) {
        VB_NCCL(ncclSend(send + (size_t(c) * p + q) * blk, blk, ncclFloat, q, ctx->comm,
                         ctx->stream));
        VB_NCCL(ncclRecv(recv + (size_t(c) * p + q) * blk, blk, ncclFloat, q, ctx->comm,
                         ctx->stream));
      }
    }
    VB_NCCL(ncclGroupEnd());
  }
  for (int c = 0; c < 3; ++c)
    VB_CUDA(cudaMemcpyAsync(recv + (size_t(c) * p + me) * blk, send + (size_t(c) * p + me) * blk,
                            blk * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
  if (peer) axis_barrier(ctx);
  ctx->comm_bytes[C_FFT_TRANSPOSE] += uint64_t(p - 1) * 3 * blk * sizeof(float);
  ctx->comm_bytes[C_ALLTOALL] += 1;
}

// x1 pass on p > 1: transpose the three components to x2 slabs (one grouped
// exchange of real data), run the pass over all n1 planes there, transpose
// back and add. Same per-pencil arithmetic and the same accumulation order
// (D3, + D2, + D1) as one GPU, so the result is independent of p.
void dist_axis1(vreg_ctx ctx, const Slab& s, const float* v3, float* out3, double beta,
                int cap) {
  const int p = ctx->nranks, n1l = s.n1l, n2l = s.n2 / p, n3 = s.n3;
  const size_t blk = size_t(n1l) * n2l * n3;  // floats per (peer, component)
  const size_t all = 3 * size_t(p) * blk;
  float *a, *b;
  const bool ce = axis_buffers(ctx, all * sizeof(float), &a, &b);
  const unsigned g4 = unsigned(blocks_for(all / 4, 256));
  k_axis_pack<<<g4, 256, 0, ctx->stream>>>(p, n1l, n2l, n3, reinterpret_cast<const float4*>(v3),
                                           reinterpret_cast<float4*>(a));
  count_launch(ctx);
  check_launch();
  {  // b[c] = component c on the x2 slab, [i1 = q n1l + i1l][j_l][k]
    Timed t(ctx, T_TRANSPOSE);
    axis_alltoall(ctx, a, b, blk, ce);
  }
  launch_axis<1>(ctx, AxisGeom{s.n1, n2l, n3}, s.n1, b, a, beta, 0, cap);
  {
    Timed t(ctx, T_TRANSPOSE);
    axis_alltoall(ctx, a, b, blk, ce);
  }
  k_axis_unpack_add<<<g4, 256, 0, ctx->stream>>>(p, n1l, n2l, n3,
                                                 reinterpret_cast<const float4*>(b),
                                                 reinterpret_cast<float4*>(out3));
  count_launch(ctx);
  check_launch();
}

// Per-component sums of v (the k = 0 mode), deterministic: fixed block
// partials, then one ordered fold per component.
constexpr int SUM_BLOCKS = 296;
__global__ void k_comp_partials(size_t n, const float* __restrict__ v, double* __restrict__ part) {
  const int c = blockIdx.y;
  const float* vc = v + size_t(c) * n;
  double acc = 0.0;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    acc += double(vc[i]);
  __shared__ double sh[256];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (int(threadIdx.x) < st) sh[threadIdx.x] += sh[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[c * SUM_BLOCKS + blockIdx.x] = sh[0];
}
__global__ void k_comp_fold(const double* __restrict__ part, double* __restrict__ sums) {
  const int c = threadIdx.x >> 5, l = threadIdx.x & 31;  // warp c folds component c
  double acc = 0.0;
  for (int b = l; b < SUM_BLOCKS; b += 32) acc += part[c * SUM_BLOCKS + b];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if (l == 0) sums[c] = acc;
}

}  // namespace

// out3 = beta (-Lap) v3 via three 1-D spectral passes; false if the grid is
// outside the fast path (non power-of-two or > 512 sizes, x2 not divisible
// by the rank count).
bool regop_separable(vreg_ctx ctx, const Slab& s, const float* v3, double beta, float* out3,
                     bool unit_zero) {
  if (!axis_size_ok(s.n1) || !axis_size_ok(s.n2) || !axis_size_ok(s.n3)) return false;
  if (ctx->nranks > 1 && s.n2 % ctx->nranks != 0) return false;
  static const bool off = [] {
    const char* e = std::getenv("VREG_REGOP_3D");
    return e && e[0] == '1';
  }();
  if (off) return false;
  const int cap = 0;  // one tile per CTA (a persistent cap measured slower)
  const AxisGeom loc{s.n1l, s.n2, s.n3};
  const double* sums = nullptr;
  if (unit_zero) {  // symbol beta at k = 0: + beta * mean(v_c) (spectral.cpp:48-70)
    double* part = static_cast<double*>(workspace(ctx, "axis_part", 3 * SUM_BLOCKS * sizeof(double)));
    double* sm = static_cast<double*>(workspace(ctx, "axis_sums", 4 * sizeof(double)));
    k_comp_partials<<<dim3(SUM_BLOCKS, 3), 256, 0, ctx->stream>>>(s.local(), v3, part);
    k_comp_fold<<<1, 96, 0, ctx->stream>>>(part, sm);
    count_launch(ctx, 2);
    check_launch();
    if (ctx->nranks > 1)
      VB_NCCL(ncclAllReduce(sm, sm, 3, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    sums = sm;
  }
  launch_axis<3>(ctx, loc, s.n3, v3, out3, beta, 0, cap, sums,
                 beta / double(s.global()));
  launch_axis<2>(ctx, loc, s.n2, v3, out3, beta, 1, cap);
  if (ctx->nranks == 1)
    launch_axis<1>(ctx, loc, s.n1, v3, out3, beta, 1, cap);
  else
    dist_axis1(ctx, s, v3, out3, beta, cap);
  return true;
}

}  // namespace vb
