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

int chunks_per_plane(const Slab& s);

namespace {

constexpr int KT = 256;  // threads of the partial-sum kernels

// One CTA per (component, local plane, chunk); returns the CTA's fp64 sum of
// f(i) over its chunk (thread 0 holds it).
__device__ __forceinline__ double rnd(double v, bool f32) { return f32 ? double(float(v)) : v; }

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

// r = b - (x0 ? q : 0), r32 = r, x = x0 ? x32 : 0; partial r.r
__global__ void __launch_bounds__(KT) k_init(Geo3 g, bool f32, const float* __restrict__ b,
                                             const float* __restrict__ q,
                                             const float* __restrict__ x32, double* __restrict__ x,
                                             double* __restrict__ r, float* __restrict__ r32,
                                             double* __restrict__ part) {
  const double s = chunk_sum(g.plane, g.n1l, g.chunks, [&](size_t i) {
    const double ri = rnd(double(b[i]) - (q ? double(q[i]) : 0.0), f32);
    r[i] = ri;
    r32[i] = float(ri);
    x[i] = x32 ? double(x32[i]) : 0.0;
    return ri * ri;
  });
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// partial a.b (a fp64, b fp32)
__global__ void __launch_bounds__(KT) k_dot(Geo3 g, const double* __restrict__ a,
                                            const float* __restrict__ b,
                                            double* __restrict__ part) {
  const double s =
      chunk_sum(g.plane, g.n1l, g.chunks, [&](size_t i) { return a[i] * double(b[i]); });
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// p = z + beta p (p = z on the first iteration), p32 = p
__global__ void k_dir(size_t n, const KrylovState* __restrict__ st, const float* __restrict__ z,
                      double* __restrict__ p, float* __restrict__ p32) {
  if (st->pad) return;
  const bool f32 = st->round32 != 0;
  const bool first = st->it == 0;
  const double beta = st->beta;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = rnd(first ? double(z[i]) : double(z[i]) + beta * p[i], f32);
    p[i] = v;
    p32[i] = float(v);
  }
}

// x += alpha p, r -= alpha q, r32 = r (skipped after negative curvature); partial r.r
__global__ void __launch_bounds__(KT) k_step(Geo3 g, const KrylovState* __restrict__ st,
                                             const double* __restrict__ p,
                                             const float* __restrict__ q, double* __restrict__ x,
                                             double* __restrict__ r, float* __restrict__ r32,
                                             double* __restrict__ part) {
  if (st->negcurv || st->pad) {
    if (threadIdx.x == 0) part[blockIdx.x] = 0.0;
    return;
  }
  const double a = st->alpha;
  const bool f32 = st->round32 != 0;
  const double s = chunk_sum(g.plane, g.n1l, g.chunks, [&](size_t i) {
    x[i] = rnd(x[i] + a * p[i], f32);
    const double ri = rnd(r[i] - a * double(q[i]), f32);
    r[i] = ri;
    r32[i] = float(ri);
    return ri * ri;
  });
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_to_f32(size_t n, const double* __restrict__ x, float* __restrict__ y) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = float(x[i]);
}

enum FoldMode { F_R0 = 0, F_RZ, F_PQ, F_RR };

// Fold the partials [rank][comp][plane][chunk] in the reference association
// (per component: planes in global order, chunks in order; components summed
// after scaling by h^3, field.hpp:150-175) and apply the CG recurrence of
// `mode`. Single CTA; ends by setting the loop condition (cond != 0).
__global__ void __launch_bounds__(KT) k_fold(int mode, int nranks, int n1l, int chunks,
                                             double h3, const double* __restrict__ part,
                                             KrylovState* __restrict__ st,
                                             double* __restrict__ hist,
                                             unsigned long long cond) {
  __shared__ double plsum[3 * 1024];  // per (comp, global plane) sums (n1 <= 1024)
  const int n1 = n1l * nranks;
  for (int e = threadIdx.x; e < 3 * n1; e += KT) {
    const int c = e / n1, gp = e - c * n1, rk = gp / n1l, pl = gp - rk * n1l;
    const double* src = part + ((size_t(rk) * 3 + c) * n1l + pl) * chunks;
    double s = 0.0;
    for (int k = 0; k < chunks; ++k) s += src[k];
    plsum[e] = s;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double total = 0.0;
  for (int c = 0; c < 3; ++c) {
    double comp = 0.0;
    for (int i = 0; i < n1; ++i) comp += plsum[c * n1 + i];
    total += comp * h3;
  }
  KrylovState& S = *st;
  // a body entered after the solve stopped (the WHILE condition is checked
  // before each body) leaves the state alone: pad marks such a pass
  if (mode == F_RZ) S.pad = S.stop;
  if (mode != F_R0 && S.pad) {
    if (cond && mode == F_RR) cudaGraphSetConditional(cudaGraphConditionalHandle(cond), 0u);
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
    default:  // F_RR
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
  if (cond && (mode == F_R0 || mode == F_RR))
    cudaGraphSetConditional(cudaGraphConditionalHandle(cond), S.stop ? 0u : 1u);
}

__global__ void k_set_state(KrylovState* st, double tol, int max_it, int round32) {
  st->tol = tol;
  st->max_it = max_it;
  st->round32 = round32;
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

Krylov::Krylov(vreg_ctx ctx, const Slab& s) : ctx_(ctx), s_(s) {
  chunks_ = chunks_per_plane(s);
  n3_ = 3 * s.local();
  require(s.n1 <= 1024, VREG_ECONFIG, "Krylov fold supports n1 <= 1024");
  cuda_ok(cudaMallocAsync(&x_, n3_ * sizeof(double), ctx->stream), "krylov alloc");
  cuda_ok(cudaMallocAsync(&r_, n3_ * sizeof(double), ctx->stream), "krylov alloc");
  cuda_ok(cudaMallocAsync(&p_, n3_ * sizeof(double), ctx->stream), "krylov alloc");
  cuda_ok(cudaMallocAsync(&z32_, n3_ * sizeof(float), ctx->stream), "krylov alloc");
  cuda_ok(cudaMallocAsync(&q32_, n3_ * sizeof(float), ctx->stream), "krylov alloc");
  cuda_ok(cudaMallocAsync(&p32_, n3_ * sizeof(float), ctx->stream), "krylov alloc");
  cuda_ok(cudaMallocAsync(&r32_, n3_ * sizeof(float), ctx->stream), "krylov alloc");
  const size_t np = size_t(3) * s.n1l * chunks_;
  cuda_ok(cudaMallocAsync(&part_, np * sizeof(double), ctx->stream), "krylov alloc");
  if (ctx->nranks > 1)
    cuda_ok(cudaMallocAsync(&part_all_, np * ctx->nranks * sizeof(double), ctx->stream),
            "krylov alloc");
  cuda_ok(cudaMallocAsync(&st_, sizeof(KrylovState), ctx->stream), "krylov alloc");
  cuda_ok(cudaMemsetAsync(st_, 0, sizeof(KrylovState), ctx->stream), "krylov memset");
  cuda_ok(cudaMallocHost(&h_st_, sizeof(KrylovState)), "krylov pinned");
  cuda_ok(cudaStreamCreateWithFlags(&cap_stream_, cudaStreamNonBlocking), "krylov stream");
}

Krylov::~Krylov() {
  cudaStreamSynchronize(ctx_->stream);
  for (void* q : {static_cast<void*>(x_), static_cast<void*>(r_), static_cast<void*>(p_),
                  static_cast<void*>(z32_), static_cast<void*>(q32_), static_cast<void*>(p32_),
                  static_cast<void*>(r32_), static_cast<void*>(part_),
                  static_cast<void*>(part_all_), static_cast<void*>(st_),
                  static_cast<void*>(hist_)})
    if (q) cudaFree(q);
  if (h_st_) cudaFreeHost(h_st_);
  if (cap_stream_) cudaStreamDestroy(cap_stream_);
}

void Krylov::issue_fold(int mode, unsigned long long cond) {
  const double* src = part_;
  if (ctx_->nranks > 1) {
    VB_NCCL(ncclAllGather(part_, part_all_, size_t(3) * s_.n1l * chunks_, ncclDouble, ctx_->comm,
                          ctx_->stream));
    ctx_->comm_bytes[C_REDUCE] += size_t(3) * s_.n1l * chunks_ * sizeof(double) * (ctx_->nranks - 1);
    src = part_all_;
  }
  const double h3 = s_.h(0) * s_.h(1) * s_.h(2);
  k_fold<<<1, KT, 0, ctx_->stream>>>(mode, ctx_->nranks, s_.n1l, chunks_, h3, src, st_, hist_,
                                      cond);
  count_launch(ctx_);
  check_launch();
}

void Krylov::issue_init(const KrylovOp& A, const float* b, const float* x, bool x0, double tol,
                        int max_it) {
  k_set_state<<<1, 1, 0, ctx_->stream>>>(st_, tol, max_it, fp32_ ? 1 : 0);
  if (x0) A(x, q32_);  // r = b - A x0 (precond.hpp:141 inner solves, x_is_zero = false)
  const Geo3 g{s_.plane(), s_.n1l, chunks_};
  const unsigned nb = unsigned(3 * s_.n1l * chunks_);
  k_init<<<nb, KT, 0, ctx_->stream>>>(g, fp32_, b, x0 ? q32_ : nullptr, x0 ? x : nullptr, x_, r_, r32_,
                                       part_);
  count_launch(ctx_, 2);
  check_launch();
}

void Krylov::issue_body(const KrylovOp& A, const KrylovOp& M, unsigned long long cond) {
  const Geo3 g{s_.plane(), s_.n1l, chunks_};
  const unsigned nb = unsigned(3 * s_.n1l * chunks_);
  M(r32_, z32_);
  k_dot<<<nb, KT, 0, ctx_->stream>>>(g, r_, z32_, part_);
  count_launch(ctx_);
  issue_fold(F_RZ, 0);
  k_dir<<<blocks_for(n3_, 256), 256, 0, ctx_->stream>>>(n3_, st_, z32_, p_, p32_);
  count_launch(ctx_);
  A(p32_, q32_);
  k_dot<<<nb, KT, 0, ctx_->stream>>>(g, p_, q32_, part_);
  count_launch(ctx_);
  issue_fold(F_PQ, 0);
  k_step<<<nb, KT, 0, ctx_->stream>>>(g, st_, p_, q32_, x_, r_, r32_, part_);
  count_launch(ctx_);
  check_launch();
  issue_fold(F_RR, cond);
}

void Krylov::issue_finish(float* x, unsigned long long* acc) {
  k_to_f32<<<blocks_for(n3_, 256), 256, 0, ctx_->stream>>>(n3_, x_, x);
  count_launch(ctx_);
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
    issue_fold(F_R0, static_cast<unsigned long long>(h));
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
  static const bool graphs_on = [] {
    const char* e = std::getenv("VREG_PCG_GRAPH");
    return !(e && e[0] == '0');
  }();
  graph = graph && graphs_on;
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
  issue_fold(F_R0, 0);
  // first iteration eagerly: allocates the operator's workspaces and plans
  // outside any capture, and solves that stop at once skip the graph
  cuda_ok(cudaMemcpyAsync(h_st_, st_, sizeof(KrylovState), cudaMemcpyDeviceToHost, ctx_->stream),
          "state d2h");
  cuda_ok(cudaStreamSynchronize(ctx_->stream), "state sync");
  while (!h_st_->stop) {
    issue_body(A, M, 0);
    cuda_ok(cudaMemcpyAsync(h_st_, st_, sizeof(KrylovState), cudaMemcpyDeviceToHost,
                            ctx_->stream),
            "state d2h");
    cuda_ok(cudaStreamSynchronize(ctx_->stream), "state sync");
    if (!h_st_->stop && graph) {
      capture_loop(A, M, false);
      break;
    }
  }
  issue_finish(x, acc);
  return read_stats();
}

}  // namespace vb
