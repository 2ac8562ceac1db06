// Device-resident preconditioned CG (krylov.hpp). pcg.hpp:30-94 is the
// algorithm; the layout of the work is the GPU's: fused fp64 vector updates
// with per-plane partial inner products, device folds that run the CG
// recurrences, and a conditional-WHILE CUDA graph for the iteration loop.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "krylov.hpp"

namespace vb {

namespace {

constexpr int KT = 256;  // threads of the partial-sum kernels

// One CTA per (component, local plane, chunk); returns the CTA's fp64 sum of
// f(i) over its chunk (thread 0 holds it).
template <class F>
__device__ __forceinline__ double chunk_sum(size_t plane, int n1l, int chunks, F f) {
  const int cta = blockIdx.x;
  const int ch = cta % chunks, rest = cta / chunks, pl = rest % n1l, c = rest / n1l;
  const size_t len = (plane + chunks - 1) / chunks;
  const size_t b0 = size_t(ch) * len, b1 = min(plane, b0 + len);
  const size_t base = (size_t(c) * n1l + pl) * plane;
  double acc = 0.0;
  for (size_t q = b0 + threadIdx.x; q < b1; q += KT) acc += f(base + q);
  __shared__ double sm[KT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < KT / 32 ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  }
  return acc;
}

struct Geo3 {
  size_t plane;
  int n1l, chunks;
};

// Iterates of type T: double (the reference's Real) or float (fp32 storage;
// the operator's fp32 copies then alias the iterates themselves).

// r = b - (x0 ? q : 0), r32 = r, x = x0 ? x32 : 0; partial r.r
template <class T>
__global__ void __launch_bounds__(KT) k_init(Geo3 g, const float* __restrict__ b,
                                             const float* __restrict__ q,
                                             const float* __restrict__ x32, T* x, T* r,
                                             float* r32, double* __restrict__ part) {
  const bool copy = static_cast<void*>(r32) != static_cast<void*>(r);
  const double s = chunk_sum(g.plane, g.n1l, g.chunks, [&](size_t i) {
    const T ri = T(double(b[i]) - (q ? double(q[i]) : 0.0));
    r[i] = ri;
    if (copy) r32[i] = float(ri);
    x[i] = x32 ? T(x32[i]) : T(0);
    return double(ri) * double(ri);
  });
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// partial a.b (a an iterate, b fp32)
template <class T>
__global__ void __launch_bounds__(KT) k_dot(Geo3 g, const T* __restrict__ a,
                                            const float* __restrict__ b,
                                            double* __restrict__ part) {
  const double s = chunk_sum(g.plane, g.n1l, g.chunks,
                             [&](size_t i) { return double(a[i]) * double(b[i]); });
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// p = z + beta p (p = z on the first iteration), p32 = p
template <class T>
__global__ void k_dir(size_t n, const KrylovState* __restrict__ st, const float* __restrict__ z,
                      T* p, float* p32) {
  if (st->pad) return;
  const bool copy = static_cast<void*>(p32) != static_cast<void*>(p);
  const bool first = st->it == 0;
  const double beta = st->beta;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const T v = T(first ? double(z[i]) : double(z[i]) + beta * double(p[i]));
    p[i] = v;
    if (copy) p32[i] = float(v);
  }
}

// x += alpha p, r -= alpha q, r32 = r (skipped after negative curvature); partial r.r
template <class T>
__global__ void __launch_bounds__(KT) k_step(Geo3 g, const KrylovState* __restrict__ st,
                                             const T* __restrict__ p,
                                             const float* __restrict__ q, T* __restrict__ x,
                                             T* r, float* r32, double* __restrict__ part) {
  if (st->negcurv || st->pad) {
    if (threadIdx.x == 0) part[blockIdx.x] = 0.0;
    return;
  }
  const bool copy = static_cast<void*>(r32) != static_cast<void*>(r);
  const double a = st->alpha;
  const double s = chunk_sum(g.plane, g.n1l, g.chunks, [&](size_t i) {
    x[i] = T(double(x[i]) + a * double(p[i]));
    const T ri = T(double(r[i]) - a * double(q[i]));
    r[i] = ri;
    if (copy) r32[i] = float(ri);
    return double(ri) * double(ri);
  });
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

template <class T>
__global__ void k_to_f32(size_t n, const T* __restrict__ x, float* __restrict__ y) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = float(x[i]);
}

// ---- H0 solves with the operator split H0 = B + G, M B = I ---------------
// (precond.hpp:31-42: B = beta_pc A with the unit zero mode, G s = g (g . s);
// the preconditioner M = B^-1 is InvA at the same beta). With y = B p kept by
// the recurrence y = r + beta y (B z = r) and z updated as z -= alpha (p +
// M G p), an iteration needs one spectral solve instead of two.

// One CTA per (local plane, chunk) over all three components; fills the
// three per-component partials of f(c, point) (layout [c][plane][chunk]).
template <class F>
__device__ __forceinline__ void chunk_sum3(size_t plane, int n1l, int chunks, size_t N,
                                           double* __restrict__ part, F f) {
  const int cta = blockIdx.x;
  const int ch = cta % chunks, pl = cta / chunks;
  const size_t len = (plane + chunks - 1) / chunks;
  const size_t b0 = size_t(ch) * len, b1 = min(plane, b0 + len);
  const size_t base = size_t(pl) * plane;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (size_t q = b0 + threadIdx.x; q < b1; q += KT) {
    double v[3];
    f(base + q, v);
    a0 += v[0];
    a1 += v[1];
    a2 += v[2];
  }
  __shared__ double sm[3][KT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_down_sync(0xffffffffu, a0, o);
    a1 += __shfl_down_sync(0xffffffffu, a1, o);
    a2 += __shfl_down_sync(0xffffffffu, a2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sm[0][threadIdx.x >> 5] = a0;
    sm[1][threadIdx.x >> 5] = a1;
    sm[2][threadIdx.x >> 5] = a2;
  }
  __syncthreads();
  if (threadIdx.x < 96) {
    const int c = threadIdx.x >> 5, l = threadIdx.x & 31;
    double a = l < KT / 32 ? sm[c][l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if (l == 0) part[(size_t(c) * n1l + pl) * chunks + ch] = a;
  }
}

// r = b - B x0 - G x0 = -g (g . x0) (B x0 = b: x0 = M b), x = x0; partial r.r
__global__ void __launch_bounds__(KT) k_h0_init(Geo3 g, size_t N, const float* __restrict__ gm,
                                                const float* __restrict__ x0, float* __restrict__ x,
                                                float* __restrict__ r, double* __restrict__ part) {
  chunk_sum3(g.plane, g.n1l, g.chunks, N, part, [&](size_t i, double* v) {
    const float g1 = gm[i], g2 = gm[N + i], g3 = gm[2 * N + i];
    const float a = x0[i], b = x0[N + i], c = x0[2 * N + i];
    const float d = g1 * a + g2 * b + g3 * c;
    const float r1 = -(d * g1), r2 = -(d * g2), r3 = -(d * g3);
    x[i] = a;
    x[N + i] = b;
    x[2 * N + i] = c;
    r[i] = r1;
    r[N + i] = r2;
    r[2 * N + i] = r3;
    v[0] = double(r1) * r1;
    v[1] = double(r2) * r2;
    v[2] = double(r3) * r3;
  });
}

// p = z + beta p, y = r + beta y (p = z, y = r on the first iteration)
// (a fused variant with the q pass below measured slower: fewer, longer
// CTAs keep fewer bytes in flight)
__global__ void k_h0_dir(size_t n, const KrylovState* __restrict__ st, const float* __restrict__ z,
                         const float* __restrict__ r, float* __restrict__ p, float* __restrict__ y) {
  if (st->pad) return;
  const bool first = st->it == 0;
  const double beta = st->beta;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    p[i] = first ? z[i] : float(double(z[i]) + beta * double(p[i]));
    y[i] = first ? r[i] : float(double(r[i]) + beta * double(y[i]));
  }
}

// gp = g (g . p), q = y + gp; partial p.q
__global__ void __launch_bounds__(KT) k_h0_q(Geo3 g, size_t N, const KrylovState* __restrict__ st,
                                             const float* __restrict__ gm,
                                             const float* __restrict__ p,
                                             const float* __restrict__ y, float* __restrict__ gp,
                                             float* __restrict__ q, double* __restrict__ part) {
  if (st->pad) {
    if (threadIdx.x < 3)
      part[(size_t(threadIdx.x) * g.n1l + blockIdx.x / g.chunks) * g.chunks +
           blockIdx.x % g.chunks] = 0.0;
    return;
  }
  chunk_sum3(g.plane, g.n1l, g.chunks, N, part, [&](size_t i, double* v) {
    const float g1 = gm[i], g2 = gm[N + i], g3 = gm[2 * N + i];
    const float p1 = p[i], p2 = p[N + i], p3 = p[2 * N + i];
    const float d = g1 * p1 + g2 * p2 + g3 * p3;
    const float a1 = d * g1, a2 = d * g2, a3 = d * g3;
    const float q1 = y[i] + a1, q2 = y[N + i] + a2, q3 = y[2 * N + i] + a3;
    gp[i] = a1;
    gp[N + i] = a2;
    gp[2 * N + i] = a3;
    q[i] = q1;
    q[N + i] = q2;
    q[2 * N + i] = q3;
    v[0] = double(p1) * q1;
    v[1] = double(p2) * q2;
    v[2] = double(p3) * q3;
  });
}

// x += alpha p, r -= alpha q, z -= alpha (p + M G p); partials r.r (part)
// and r.z (part + np, the next iteration's rho)
__global__ void __launch_bounds__(KT) k_h0_step(Geo3 g, size_t np, const KrylovState* __restrict__ st,
                                                const float* __restrict__ p,
                                                const float* __restrict__ q,
                                                const float* __restrict__ mg, float* __restrict__ x,
                                                float* __restrict__ r, float* __restrict__ z,
                                                double* __restrict__ part) {
  if (st->negcurv || st->pad) {
    if (threadIdx.x == 0) part[blockIdx.x] = part[np + blockIdx.x] = 0.0;
    return;
  }
  const double a = st->alpha;
  const int cta = blockIdx.x;
  const int ch = cta % g.chunks, rest = cta / g.chunks, pl = rest % g.n1l, c = rest / g.n1l;
  const size_t len = (g.plane + g.chunks - 1) / g.chunks;
  const size_t b0 = size_t(ch) * len, b1 = min(g.plane, b0 + len);
  const size_t base = (size_t(c) * g.n1l + pl) * g.plane;
  double srr = 0.0, srz = 0.0;
  for (size_t k = b0 + threadIdx.x; k < b1; k += KT) {
    const size_t i = base + k;
    const double pi = p[i];
    x[i] = float(double(x[i]) + a * pi);
    const float ri = float(double(r[i]) - a * double(q[i]));
    const float zi = float(double(z[i]) - a * (pi + double(mg[i])));
    r[i] = ri;
    z[i] = zi;
    srr += double(ri) * ri;
    srz += double(ri) * zi;
  }
  __shared__ double sm[2][KT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    srr += __shfl_down_sync(0xffffffffu, srr, o);
    srz += __shfl_down_sync(0xffffffffu, srz, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sm[0][threadIdx.x >> 5] = srr;
    sm[1][threadIdx.x >> 5] = srz;
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    double v = l < KT / 32 ? sm[w][l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (l == 0) part[size_t(w) * np + blockIdx.x] = v;
  }
}

enum FoldMode { F_R0 = 0, F_RZ, F_PQ, F_RR, F_R0Z, F_RRZ };

// Sum of one partial array [rank][comp][plane][chunk] (rank blocks rs
// doubles apart): per component over the global planes (field.hpp:150-175 up
// to association), components summed after scaling by h^3. Every thread
// calls it; thread 0 gets the total.
__device__ double fold_total(const double* __restrict__ part, size_t rs, int nranks, int n1l,
                             int chunks, double h3, double* plsum, double* comp) {
  const int n1 = n1l * nranks;
  for (int e = threadIdx.x; e < 3 * n1; e += KT) {
    const int c = e / n1, gp = e - c * n1, rk = gp / n1l, pl = gp - rk * n1l;
    const double* src = part + size_t(rk) * rs + (size_t(c) * n1l + pl) * chunks;
    double s = 0.0;
    for (int k = 0; k < chunks; ++k) s += src[k];
    plsum[e] = s;
  }
  __syncthreads();
  // per component: lane l folds the global planes [l B, (l + 1) B) in order,
  // then a fixed shuffle tree -- an association independent of the rank
  // count (planes are in global order), so p GPUs give bitwise the same sums
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (w < 3) {
    const int B = (n1 + 31) / 32;
    double a = 0.0;
    for (int i = l * B; i < min(n1, (l + 1) * B); ++i) a += plsum[w * n1 + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if (l == 0) comp[w] = a;
  }
  __syncthreads();
  double total = 0.0;
  for (int c = 0; c < 3; ++c) total += comp[c] * h3;
  __syncthreads();  // plsum / comp reusable
  return total;
}

// Fold the partials and apply the CG recurrence of `mode`. F_R0Z / F_RRZ
// (split H0 solves) fold a second array (r.z) after the first, np doubles
// on. Single CTA; ends by setting the loop condition (cond != 0).
__global__ void __launch_bounds__(KT) k_fold(int mode, int nranks, int n1l, int chunks,
                                             double h3, const double* __restrict__ part,
                                             size_t rs, size_t np, KrylovState* __restrict__ st,
                                             double* __restrict__ hist,
                                             unsigned long long cond) {
  __shared__ double plsum[3 * 1024];  // per (comp, global plane) sums (n1 <= 1024)
  __shared__ double comp[3];
  const double total = fold_total(part, rs, nranks, n1l, chunks, h3, plsum, comp);
  const bool two = mode == F_R0Z || mode == F_RRZ;
  const double total2 = two ? fold_total(part + np, rs, nranks, n1l, chunks, h3, plsum, comp) : 0.0;
  if (threadIdx.x != 0) return;
  if (mode == F_R0Z) mode = F_R0;
  KrylovState& S = *st;
  // a body entered after the solve stopped (the WHILE condition is checked
  // before each body) leaves the state alone: pad marks such a pass
  if (mode == F_RZ) S.pad = S.stop;
  if (mode != F_R0 && S.pad) {
    if (cond && (mode == F_RR || mode == F_RRZ))
      cudaGraphSetConditional(cudaGraphConditionalHandle(cond), 0u);
    return;
  }
  switch (mode) {
    case F_R0:
      S.rr = total;
      S.r0n = sqrt(total);
      S.it = 0;
      S.conv = 0;
      S.negcurv = 0;
      S.stop = 0;
      S.pad = 0;
      hist[0] = S.r0n == 0.0 ? 0.0 : 1.0;
      if (S.r0n == 0.0) {
        S.conv = 1;
        S.stop = 1;
      } else if (S.max_it <= 0) {
        S.stop = 1;
      }
      break;
    case F_RZ:
      S.beta = S.it == 0 ? 0.0 : total / S.rho;
      S.rho = total;
      break;
    case F_PQ:
      S.pq = total;
      if (total <= 0.0) {  // negative curvature: stop before the step
        S.negcurv = 1;
        S.stop = 1;
        S.alpha = 0.0;
      } else {
        S.alpha = S.rho / total;
      }
      break;
    default:  // F_RR, F_RRZ
      if (!S.negcurv) {
        S.rr = total;
        S.it += 1;
        const double rel = sqrt(total) / S.r0n;
        hist[S.it] = rel;
        if (rel <= S.tol) {
          S.conv = 1;
          S.stop = 1;
        } else if (S.it >= S.max_it) {
          S.stop = 1;
        }
      }
      break;
  }
  if (two && !S.stop) {  // rho = r.z of the new residual (beta for the next direction)
    S.beta = S.it == 0 ? 0.0 : total2 / S.rho;
    S.rho = total2;
  }
  if (two) S.pad = S.stop;
  if (cond && (mode == F_R0 || mode == F_RR || mode == F_RRZ))
    cudaGraphSetConditional(cudaGraphConditionalHandle(cond), S.stop ? 0u : 1u);
}

__global__ void k_set_state(KrylovState* st, double tol, int max_it) {
  st->tol = tol;
  st->max_it = max_it;
}

// acc[0] += iterations, acc[1] |= not converged
__global__ void k_accumulate(const KrylovState* st, unsigned long long* acc) {
  acc[0] += static_cast<unsigned long long>(st->it);
  if (!st->conv) acc[1] = 1ull;
}

inline void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(VREG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

Krylov::Krylov(vreg_ctx ctx, const Slab& s, bool fp64) : ctx_(ctx), s_(s), fp64_(fp64) {
  // 2048-element chunks (8 per thread): enough CTAs that the streaming
  // update kernels keep their loads in flight (8192 left them latency-bound)
  chunks_ = int((s.plane() + 2047) / 2048);
  n3_ = 3 * s.local();
  require(s.n1 <= 1024, VREG_ECONFIG, "Krylov fold supports n1 <= 1024");
  const size_t es = fp64 ? sizeof(double) : sizeof(float);
  cuda_ok(cudaMallocAsync(&x_, n3_ * es, ctx->stream), "krylov alloc");
  cuda_ok(cudaMallocAsync(&r_, n3_ * es, ctx->stream), "krylov alloc");
  cuda_ok(cudaMallocAsync(&p_, n3_ * es, ctx->stream), "krylov alloc");
  cuda_ok(cudaMallocAsync(&z32_, n3_ * sizeof(float), ctx->stream), "krylov alloc");
  cuda_ok(cudaMallocAsync(&q32_, n3_ * sizeof(float), ctx->stream), "krylov alloc");
  if (fp64) {  // fp32 copies for the operator; fp32 iterates are their own copies
    cuda_ok(cudaMallocAsync(&p32_, n3_ * sizeof(float), ctx->stream), "krylov alloc");
    cuda_ok(cudaMallocAsync(&r32_, n3_ * sizeof(float), ctx->stream), "krylov alloc");
  } else {
    p32_ = static_cast<float*>(p_);
    r32_ = static_cast<float*>(r_);
  }
  const size_t np = size_t(3) * s.n1l * chunks_;  // two arrays: r.r and r.z (split H0)
  cuda_ok(cudaMallocAsync(&part_, 2 * np * sizeof(double), ctx->stream), "krylov alloc");
  if (ctx->nranks > 1)
    cuda_ok(cudaMallocAsync(&part_all_, 2 * np * ctx->nranks * sizeof(double), ctx->stream),
            "krylov alloc");
  cuda_ok(cudaMallocAsync(&st_, sizeof(KrylovState), ctx->stream), "krylov alloc");
  cuda_ok(cudaMemsetAsync(st_, 0, sizeof(KrylovState), ctx->stream), "krylov memset");
  cuda_ok(cudaMallocHost(&h_st_, sizeof(KrylovState)), "krylov pinned");
  cuda_ok(cudaStreamCreateWithFlags(&cap_stream_, cudaStreamNonBlocking), "krylov stream");
}

Krylov::~Krylov() {
  cudaStreamSynchronize(ctx_->stream);
  if (!fp64_) p32_ = r32_ = nullptr;  // aliases of p_ and r_
  for (void* q : {x_, r_, p_, static_cast<void*>(z32_), static_cast<void*>(q32_),
                  static_cast<void*>(p32_), static_cast<void*>(r32_), static_cast<void*>(part_),
                  static_cast<void*>(part_all_), static_cast<void*>(st_),
                  static_cast<void*>(hist_), static_cast<void*>(y_), static_cast<void*>(gp_),
                  static_cast<void*>(mg_)})
    if (q) cudaFree(q);
  if (h_st_) cudaFreeHost(h_st_);
  if (cap_stream_) cudaStreamDestroy(cap_stream_);
}

void Krylov::issue_fold(int mode, unsigned long long cond) {
  const size_t np = size_t(3) * s_.n1l * chunks_;
  const size_t cnt = (mode == F_R0Z || mode == F_RRZ) ? 2 * np : np;  // r.z follows r.r
  const double* src = part_;
  size_t rs = cnt;
  if (ctx_->nranks > 1) {
    VB_NCCL(ncclAllGather(part_, part_all_, cnt, ncclDouble, ctx_->comm, ctx_->stream));
    ctx_->comm_bytes[C_REDUCE] += cnt * sizeof(double) * (ctx_->nranks - 1);
    src = part_all_;
  }
  const double h3 = s_.h(0) * s_.h(1) * s_.h(2);
  k_fold<<<1, KT, 0, ctx_->stream>>>(mode, ctx_->nranks, s_.n1l, chunks_, h3, src, rs, np, st_,
                                      hist_, cond);
  count_launch(ctx_);
  check_launch();
}

void Krylov::issue_init(const KrylovOp& A, const float* b, const float* x, bool x0, double tol,
                        int max_it) {
  k_set_state<<<1, 1, 0, ctx_->stream>>>(st_, tol, max_it);
  if (h0g_) {  // split H0 solve: r0 = -G x0, z0 = M r0 (x0 = M b)
    const Geo3 g{s_.plane(), s_.n1l, chunks_};
    k_h0_init<<<unsigned(s_.n1l * chunks_), KT, 0, ctx_->stream>>>(
        g, s_.local(), h0g_, x, static_cast<float*>(x_), static_cast<float*>(r_), part_);
    count_launch(ctx_, 2);
    check_launch();
    (*h0m_)(r32_, z32_);
    dot(r_, z32_, part_ + size_t(3) * s_.n1l * chunks_);  // rho_0 = r0.z0
    return;
  }
  if (x0) A(x, q32_);  // r = b - A x0 (precond.hpp:141 inner solves, x_is_zero = false)
  const Geo3 g{s_.plane(), s_.n1l, chunks_};
  const unsigned nb = unsigned(3 * s_.n1l * chunks_);
  const float* qq = x0 ? q32_ : nullptr;
  const float* xx = x0 ? x : nullptr;
  if (fp64_)
    k_init<double><<<nb, KT, 0, ctx_->stream>>>(g, b, qq, xx, static_cast<double*>(x_),
                                                static_cast<double*>(r_), r32_, part_);
  else
    k_init<float><<<nb, KT, 0, ctx_->stream>>>(g, b, qq, xx, static_cast<float*>(x_),
                                               static_cast<float*>(r_), r32_, part_);
  count_launch(ctx_, 2);
  check_launch();
}

void Krylov::issue_body(const KrylovOp& A, const KrylovOp& M, unsigned long long cond) {
  const Geo3 g{s_.plane(), s_.n1l, chunks_};
  const unsigned nb = unsigned(3 * s_.n1l * chunks_);
  if (h0g_) {  // split H0 iteration: z and y = B p are kept by recurrences
    const size_t np = size_t(3) * s_.n1l * chunks_;
    float* p = static_cast<float*>(p_);
    k_h0_dir<<<blocks_for(n3_, 256), 256, 0, ctx_->stream>>>(
        n3_, st_, z32_, static_cast<const float*>(r_), p, y_);
    k_h0_q<<<unsigned(s_.n1l * chunks_), KT, 0, ctx_->stream>>>(g, s_.local(), st_, h0g_, p, y_,
                                                                 gp_, q32_, part_);
    count_launch(ctx_, 2);
    check_launch();
    issue_fold(F_PQ, 0);
    M(gp_, mg_);
    k_h0_step<<<nb, KT, 0, ctx_->stream>>>(g, np, st_, static_cast<const float*>(p_), q32_, mg_,
                                           static_cast<float*>(x_), static_cast<float*>(r_),
                                           z32_, part_);
    count_launch(ctx_);
    check_launch();
    issue_fold(F_RRZ, cond);
    return;
  }
  M(r32_, z32_);
  dot(r_, z32_);
  issue_fold(F_RZ, 0);
  if (fp64_)
    k_dir<double><<<blocks_for(n3_, 256), 256, 0, ctx_->stream>>>(
        n3_, st_, z32_, static_cast<double*>(p_), p32_);
  else
    k_dir<float><<<blocks_for(n3_, 256), 256, 0, ctx_->stream>>>(
        n3_, st_, z32_, static_cast<float*>(p_), p32_);
  count_launch(ctx_);
  A(p32_, q32_);
  dot(p_, q32_);
  issue_fold(F_PQ, 0);
  if (fp64_)
    k_step<double><<<nb, KT, 0, ctx_->stream>>>(g, st_, static_cast<const double*>(p_), q32_,
                                                static_cast<double*>(x_),
                                                static_cast<double*>(r_), r32_, part_);
  else
    k_step<float><<<nb, KT, 0, ctx_->stream>>>(g, st_, static_cast<const float*>(p_), q32_,
                                               static_cast<float*>(x_), static_cast<float*>(r_),
                                               r32_, part_);
  count_launch(ctx_);
  check_launch();
  issue_fold(F_RR, cond);
}

// per-plane partials of <a, b32> (a an iterate)
void Krylov::dot(const void* a, const float* b32, double* dst) {
  const Geo3 g{s_.plane(), s_.n1l, chunks_};
  const unsigned nb = unsigned(3 * s_.n1l * chunks_);
  if (!dst) dst = part_;
  if (fp64_)
    k_dot<double><<<nb, KT, 0, ctx_->stream>>>(g, static_cast<const double*>(a), b32, dst);
  else
    k_dot<float><<<nb, KT, 0, ctx_->stream>>>(g, static_cast<const float*>(a), b32, dst);
  count_launch(ctx_);
}

void Krylov::issue_finish(float* x, unsigned long long* acc) {
  if (fp64_) {
    k_to_f32<double><<<blocks_for(n3_, 256), 256, 0, ctx_->stream>>>(
        n3_, static_cast<const double*>(x_), x);
    count_launch(ctx_);
  } else {
    VB_CUDA(cudaMemcpyAsync(x, x_, n3_ * sizeof(float), cudaMemcpyDeviceToDevice, ctx_->stream));
  }
  if (acc) {
    k_accumulate<<<1, 1, 0, ctx_->stream>>>(st_, acc);
    count_launch(ctx_);
  }
  check_launch();
}

// Record the WHILE loop over the body. nested: into the graph the context's
// stream is capturing -- the init fold (recorded here, upstream of the
// conditional node) seeds the loop condition; otherwise into a fresh graph
// that is launched here (the caller checked that the solve has not stopped).
void Krylov::capture_loop(const KrylovOp& A, const KrylovOp& M, bool nested) {
  cudaStream_t st = ctx_->stream;
  static const bool dbg = std::getenv("VREG_DEBUG_CAPTURE") != nullptr;
  auto status = [&](const char* where) {
    if (!dbg) return;
    cudaStreamCaptureStatus a = cudaStreamCaptureStatusNone, b = a;
    cudaStreamIsCapturing(st, &a);
    cudaStreamIsCapturing(cap_stream_, &b);
    std::fprintf(stderr, "[krylov] %s nested=%d st=%p(%d) cap=%p(%d)\n", where, int(nested),
                 (void*)st, int(a), (void*)cap_stream_, int(b));
  };
  status("enter");
  cudaGraph_t graph = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaStreamCaptureStatus cs;
  if (nested)
    cuda_ok(cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &ndeps), "capture info");
  else
    cuda_ok(cudaGraphCreate(&graph, 0), "graph create");
  cudaGraphConditionalHandle h;
  cuda_ok(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault),
          "conditional handle");
  if (nested) {
    issue_fold(h0g_ ? F_R0Z : F_R0, static_cast<unsigned long long>(h));
    cuda_ok(cudaStreamGetCaptureInfo(st, &cs, nullptr, &graph, &deps, &ndeps), "capture info");
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  cuda_ok(cudaGraphAddNode(&node, graph, deps, ndeps, &cp), "conditional node");
  if (nested)
    cuda_ok(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies),
            "capture dependencies");
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  // the body is captured on a private stream; the library issues on
  // ctx->stream, so route it there for the duration
  cuda_ok(cudaStreamBeginCaptureToGraph(cap_stream_, body, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeRelaxed),
          "begin capture");
  ctx_->stream = cap_stream_;
  try {
    issue_body(A, M, static_cast<unsigned long long>(h));
  } catch (...) {
    ctx_->stream = st;
    cudaGraph_t dummy;
    cudaStreamEndCapture(cap_stream_, &dummy);
    throw;
  }
  ctx_->stream = st;
  status("before end");
  cuda_ok(cudaStreamEndCapture(cap_stream_, &body), "end capture");
  status("after end");
  if (!nested) {
    cudaGraphExec_t ex;
    cuda_ok(cudaGraphInstantiate(&ex, graph, 0), "graph instantiate");
    cuda_ok(cudaGraphLaunch(ex, st), "graph launch");
    cuda_ok(cudaStreamSynchronize(st), "graph sync");
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(graph);
  }
}

KrylovStats Krylov::read_stats() {
  KrylovStats r;
  cuda_ok(cudaMemcpyAsync(h_st_, st_, sizeof(KrylovState), cudaMemcpyDeviceToHost, ctx_->stream),
          "state d2h");
  cuda_ok(cudaStreamSynchronize(ctx_->stream), "state sync");
  const KrylovState& S = *h_st_;
  r.iters = S.it;
  r.converged = S.conv != 0;
  r.negative_curvature = S.negcurv != 0;
  r.history.resize(size_t(S.it) + 1);
  cuda_ok(cudaMemcpy(r.history.data(), hist_, r.history.size() * sizeof(double),
                     cudaMemcpyDeviceToHost),
          "history d2h");
  r.rel_res = S.r0n == 0.0 ? 0.0 : (S.it ? r.history.back() : 1.0);
  return r;
}

KrylovStats Krylov::solve(const KrylovOp& A, const KrylovOp& M, const float* b, float* x,
                          double tol, int max_it, bool x0, unsigned long long* acc, bool graph) {
  // graphs on one GPU; on several the loop runs eagerly (one 64-byte state
  // read per iteration) unless VREG_PCG_GRAPH=1 -- NCCL collectives of two
  // communicators (halo/fold and the regulariser's transposes) inside one
  // captured body are not ordered across ranks
  static const int graphs_env = [] {
    const char* e = std::getenv("VREG_PCG_GRAPH");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  graph = graph && (graphs_env == 1 || (graphs_env == -1 && ctx_->nranks == 1));
  if (max_it + 1 > hist_cap_) {
    if (hist_) cuda_ok(cudaFreeAsync(hist_, ctx_->stream), "history free");
    hist_cap_ = max_it + 1;
    cuda_ok(cudaMallocAsync(&hist_, size_t(hist_cap_) * sizeof(double), ctx_->stream),
            "history alloc");
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cuda_ok(cudaStreamIsCapturing(ctx_->stream, &cs), "capture status");
  issue_init(A, b, x, x0, tol, max_it);
  if (cs == cudaStreamCaptureStatusActive) {
    capture_loop(A, M, true);  // records the init fold and the loop
    issue_finish(x, acc);
    return KrylovStats{};
  }
  issue_fold(h0g_ ? F_R0Z : F_R0, 0);
  // first iteration eagerly: allocates the operator's workspaces and plans
  // outside any capture, and solves that stop at once skip the graph
  cuda_ok(cudaMemcpyAsync(h_st_, st_, sizeof(KrylovState), cudaMemcpyDeviceToHost, ctx_->stream),
          "state d2h");
  cuda_ok(cudaStreamSynchronize(ctx_->stream), "state sync");
  // the first iterations run eagerly with one 64-byte state read each:
  // capturing and instantiating the loop graph costs more than the host
  // round trips of a short solve (the registration's outer solves take 1-8
  // iterations; measured at 256^3: 0.34 s eager vs 0.35-0.42 s always-graph).
  // Longer solves switch to the conditional graph.
  static const int eager = [] {
    const char* e = std::getenv("VREG_PCG_EAGER");
    return e ? std::atoi(e) : 8;
  }();
  for (int k = 1; !h_st_->stop; ++k) {
    issue_body(A, M, 0);
    cuda_ok(cudaMemcpyAsync(h_st_, st_, sizeof(KrylovState), cudaMemcpyDeviceToHost,
                            ctx_->stream),
            "state d2h");
    cuda_ok(cudaStreamSynchronize(ctx_->stream), "state sync");
    if (!h_st_->stop && graph && k >= eager) {
      capture_loop(A, M, false);
      break;
    }
  }
  issue_finish(x, acc);
  return read_stats();
}

KrylovStats Krylov::solve_h0(const float* gm, const KrylovOp& M, const float* b, float* x,
                             double tol, int max_it, unsigned long long* acc, bool graph) {
  require(!fp64_, VREG_ECONFIG, "split H0 solves use fp32 iterates");
  if (!y_) {
    cuda_ok(cudaMallocAsync(&y_, n3_ * sizeof(float), ctx_->stream), "krylov alloc");
    cuda_ok(cudaMallocAsync(&gp_, n3_ * sizeof(float), ctx_->stream), "krylov alloc");
    cuda_ok(cudaMallocAsync(&mg_, n3_ * sizeof(float), ctx_->stream), "krylov alloc");
  }
  (void)b;  // enters only through x0 = M b
  h0g_ = gm;
  h0m_ = &M;
  struct Reset {
    Krylov* k;
    ~Reset() {
      k->h0g_ = nullptr;
      k->h0m_ = nullptr;
    }
  } reset{this};
  static const KrylovOp none = [](const float*, float*) {};
  return solve(none, M, b, x, tol, max_it, true, acc, graph);
}

}  // namespace vb
