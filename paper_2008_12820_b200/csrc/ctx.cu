// Context lifecycle, pooled memory, workspace cache, FFT plan cache, kernel
// timers and slab distribution (EngineState analogue, engine.hpp:14-19;
// FftPlanCache, fft.cpp:66-72; from_global/to_global, engine.hpp:63-66).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <iterator>
#include <map>
#include <mutex>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace vb {

void smem_optin(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  VB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{dev, kernel}];
  if (have >= bytes) return;
  VB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

namespace {
thread_local std::string g_last_error;
std::mutex g_plan_mutex;  // plan creation is serialised (fft.hpp:81-83)
}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }

double Slab::h(int a) const {
  const int n = a == 0 ? n1 : (a == 1 ? n2 : n3);
  return 6.283185307179586476925286766559 / double(n);
}

Slab slab_of(vreg_ctx ctx, const vreg_grid* g) {
  require(g != nullptr, VREG_EPARAM, "null grid");
  require(g->n1 >= 2 && g->n2 >= 2 && g->n3 >= 2, VREG_EDIM, "grid sizes must be >= 2");
  require(g->n1 % 2 == 0 && g->n2 % 2 == 0 && g->n3 % 2 == 0, VREG_EDIM,
          "grid sizes must be even");
  require(g->n1 % ctx->nranks == 0, VREG_ECONFIG,
          "slab layout infeasible: n1 must be divisible by the rank count");
  Slab s;
  s.n1 = g->n1;
  s.n2 = g->n2;
  s.n3 = g->n3;
  s.nt = g->nt < 1 ? 1 : g->nt;
  s.n1l = g->n1 / ctx->nranks;
  s.off = ctx->rank * s.n1l;
  return s;
}

void* workspace(vreg_ctx ctx, const std::string& name, size_t bytes) {
  auto it = ctx->ws.find(name);
  if (it != ctx->ws.end()) {
    if (it->second.second >= bytes) return it->second.first;
    VB_CUDA(cudaFreeAsync(it->second.first, ctx->stream));
    ctx->ws.erase(it);
  }
  void* p = nullptr;
  VB_CUDA(cudaMallocAsync(&p, bytes ? bytes : 16, ctx->stream));
  ctx->ws[name] = {p, bytes};
  return p;
}

double* pinned(vreg_ctx ctx, size_t n) {
  if (n > ctx->h_pinned_cap) {
    if (ctx->h_pinned) VB_CUDA(cudaFreeHost(ctx->h_pinned));
    size_t cap = n < 4096 ? 4096 : n;
    VB_CUDA(cudaMallocHost(&ctx->h_pinned, cap * sizeof(double)));
    ctx->h_pinned_cap = cap;
  }
  return ctx->h_pinned;
}

FftPlans& fft_plans(vreg_ctx ctx, int n1, int n2, int n3, int batch) {
  auto key = std::make_tuple(n1, n2, n3, batch);
  auto it = ctx->plans.find(key);
  if (it != ctx->plans.end()) {
    // plans follow the context's current stream (side-stream branches,
    // graph-capture streams of the Krylov solver)
    if (it->second.stream != ctx->stream) {
      VB_CUFFT(cufftSetStream(it->second.r2c, ctx->stream));
      VB_CUFFT(cufftSetStream(it->second.c2r, ctx->stream));
      it->second.stream = ctx->stream;
    }
    return it->second;
  }
  std::lock_guard<std::mutex> lock(g_plan_mutex);
  FftPlans p;
  int n[3] = {n1, n2, n3};
  const long long N = (long long)n1 * n2 * n3;
  const long long NC = (long long)n1 * n2 * (n3 / 2 + 1);
  size_t w1 = 0, w2 = 0;
  VB_CUFFT(cufftCreate(&p.r2c));
  VB_CUFFT(cufftCreate(&p.c2r));
  VB_CUFFT(cufftSetAutoAllocation(p.r2c, 0));
  VB_CUFFT(cufftSetAutoAllocation(p.c2r, 0));
  VB_CUFFT(cufftMakePlanMany(p.r2c, 3, n, nullptr, 1, int(N), nullptr, 1, int(NC),
                             CUFFT_R2C, batch, &w1));
  VB_CUFFT(cufftMakePlanMany(p.c2r, 3, n, nullptr, 1, int(NC), nullptr, 1, int(N),
                             CUFFT_C2R, batch, &w2));
  p.work = w1 > w2 ? w1 : w2;
  if (p.work > ctx->fft_work_size) {
    if (ctx->fft_work) VB_CUDA(cudaFreeAsync(ctx->fft_work, ctx->stream));
    VB_CUDA(cudaMallocAsync(&ctx->fft_work, p.work, ctx->stream));
    ctx->fft_work_size = p.work;
    for (auto& kv : ctx->plans) {
      VB_CUFFT(cufftSetWorkArea(kv.second.r2c, ctx->fft_work));
      VB_CUFFT(cufftSetWorkArea(kv.second.c2r, ctx->fft_work));
    }
  }
  VB_CUFFT(cufftSetWorkArea(p.r2c, ctx->fft_work));
  VB_CUFFT(cufftSetWorkArea(p.c2r, ctx->fft_work));
  VB_CUFFT(cufftSetStream(p.r2c, ctx->stream));
  VB_CUFFT(cufftSetStream(p.c2r, ctx->stream));
  p.stream = ctx->stream;
  return ctx->plans.emplace(key, p).first->second;
}

namespace {
const char* const kCatNames[T_COUNT] = {"fft",          "fd",           "sl",
                                        "ghost_comm",   "interp_comm",  "scatter_comm",
                                        "scatter_buffer", "transpose_comm"};
}  // namespace

// Every timed kernel group is also an NVTX range (ranges per
// engine call next to the CUDA-event timers), visible to nsys / ncu --nvtx.
Timed::Timed(vreg_ctx ctx, int cat, const char* name) : ctx_(ctx), cat_(cat), name_(name) {
  nvtxRangePushA(name ? name : (cat >= 0 && cat < T_COUNT ? kCatNames[cat] : "vreg"));
  if (!ctx_->timers_on) return;
  // scopes recorded into a CUDA graph (stream capture) are not timed: their
  // events would never complete on their own
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(ctx_->stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
    return;
  if (ctx_->event_pool.empty()) {
    cudaEvent_t e;
    VB_CUDA(cudaEventCreate(&e));
    ctx_->event_pool.push_back(e);
  }
  a_ = ctx_->event_pool.back();
  ctx_->event_pool.pop_back();
  VB_CUDA(cudaEventRecord(a_, ctx_->stream));
}

Timed::~Timed() {
  nvtxRangePop();
  if (!a_) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(ctx_->stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    ctx_->event_pool.push_back(a_);  // began outside the capture: drop the sample
    return;
  }
  cudaEvent_t b;
  if (ctx_->event_pool.empty()) {
    if (cudaEventCreate(&b) != cudaSuccess) return;
  } else {
    b = ctx_->event_pool.back();
    ctx_->event_pool.pop_back();
  }
  cudaEventRecord(b, ctx_->stream);
  ctx_->pending.push_back({cat_, name_, a_, b});
}

void resolve_timers(vreg_ctx ctx) {
  VB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (auto& p : ctx->pending) {
    float ms = 0.f;
    VB_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    if (p.cat >= 0) ctx->timer_acc[p.cat] += double(ms) * 1e-3;  // cat < 0: named only
    if (p.name) {
      auto& st = ctx->kstats[p.name];
      st.first += 1;
      st.second += double(ms) * 1e-3;
    }
    ctx->event_pool.push_back(p.a);
    ctx->event_pool.push_back(p.b);
  }
  ctx->pending.clear();
}

}  // namespace vb

using namespace vb;

extern "C" {

const char* vreg_last_error(void) { return g_last_error.c_str(); }

int vreg_status_exit_code(int status) {
  switch (status) {
    case VREG_OK: return 0;
    case VREG_EPARAM:
    case VREG_EDIM:
    case VREG_ECONFIG:
    case VREG_EINPUT: return 2;
    case VREG_ENUMERICAL: return 3;
    case VREG_EIO: return 4;
    default: return 1;
  }
}

static void init_ctx(vreg_ctx c, int device) {
  {
    const char* e = std::getenv("VREG_DETERMINISTIC");
    c->deterministic = e && e[0] == '1';
  }
  c->device = device;
  VB_CUDA(cudaSetDevice(device));
  VB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->own_stream = true;
  VB_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  {
    int lo = 0, hi = 0;
    VB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    VB_CUDA(cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi));
    VB_CUDA(cudaEventCreateWithFlags(&c->ev_c0, cudaEventDisableTiming));
    VB_CUDA(cudaEventCreateWithFlags(&c->ev_c1, cudaEventDisableTiming));
  }
  VB_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  VB_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  cudaMemPool_t pool;
  VB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thresh = UINT64_MAX;  // keep freed blocks cached in the pool
  VB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
}

int vreg_ctx_create(int device, vreg_ctx* out) {
  return guard([&] {
    require(out != nullptr, VREG_EPARAM, "null out");
    auto c = std::make_unique<vreg_ctx_s>();
    init_ctx(c.get(), device);
    *out = c.release();
  });
}

int vreg_nccl_unique_id(void* uid128) {
  return guard([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    VB_NCCL(ncclGetUniqueId(&id));
    std::memcpy(uid128, &id, sizeof(id));
  });
}

int vreg_ctx_create_dist(int device, int rank, int nranks, const void* uid128,
                         vreg_ctx* out) {
  return guard([&] {
    require(out != nullptr && uid128 != nullptr, VREG_EPARAM, "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, VREG_EPARAM, "bad rank");
    auto c = std::make_unique<vreg_ctx_s>();
    init_ctx(c.get(), device);
    c->rank = rank;
    c->nranks = nranks;
    if (nranks > 1) {
      ncclUniqueId id;
      std::memcpy(&id, uid128, sizeof(id));
      VB_NCCL(ncclCommInitRank(&c->comm, nranks, id, rank));
      VB_NCCL(ncclCommSplit(c->comm, 0, rank, &c->fft_comm, nullptr));
    }
    *out = c.release();
  });
}

int vreg_ctx_destroy(vreg_ctx ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->side);
    cudaStreamSynchronize(ctx->comm_stream);
    for (auto& kv : ctx->plans) {
      cufftDestroy(kv.second.r2c);
      cufftDestroy(kv.second.c2r);
    }
    for (auto& kv : ctx->ws) cudaFree(kv.second.first);
    for (auto& t : ctx->tile_tables) cudaFree(t.table);
    if (ctx->fft_work) cudaFree(ctx->fft_work);
    if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
    for (auto& p : ctx->pending) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    cudaStreamSynchronize(ctx->side);
    for (float* q : ctx->peer_recv)
      if (q) cudaIpcCloseMemHandle(q);
    for (int i = 0; i < 2; ++i)
      if (ctx->xbuf[i]) cudaFree(ctx->xbuf[i]);
    if (ctx->xflag) cudaFree(ctx->xflag);
    if (ctx->fft_comm) ncclCommDestroy(ctx->fft_comm);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    cudaStreamDestroy(ctx->side);
    cudaStreamDestroy(ctx->comm_stream);
    cudaEventDestroy(ctx->ev_c0);
    cudaEventDestroy(ctx->ev_c1);
    cudaEventDestroy(ctx->ev_fork);
    cudaEventDestroy(ctx->ev_join);
    delete ctx;
  });
}

int vreg_ctx_rank(vreg_ctx ctx, int* rank, int* nranks) {
  if (rank) *rank = ctx->rank;
  if (nranks) *nranks = ctx->nranks;
  return VREG_OK;
}

int vreg_ctx_reserve(vreg_ctx ctx, size_t bytes) {
  return guard([&] {
    // grow the stream-ordered pool once (its release threshold keeps the
    // pages): mapping fresh device memory inside a solve costs ~0.1 s per
    // few GB and showed up as random per-phase spikes in the registration
    size_t free_b = 0, total_b = 0;
    VB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    bytes = std::min(bytes, free_b / 2);
    if (bytes == 0) return;
    void* p = nullptr;
    VB_CUDA(cudaMallocAsync(&p, bytes, ctx->stream));
    VB_CUDA(cudaFreeAsync(p, ctx->stream));
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int vreg_ctx_set_deterministic(vreg_ctx ctx, int on) {
  return guard([&] { ctx->deterministic = on != 0; });
}

int vreg_ctx_set_reg_order(vreg_ctx ctx, int order) {
  return guard([&] {
    require(order == 1 || order == 2, VREG_EPARAM, "regularization order must be 1 (H1) or 2 (H2)");
    ctx->reg_order = order;
  });
}

int vreg_ctx_get_stream(vreg_ctx ctx, void** s) {
  return guard([&] {
    require(s != nullptr, VREG_EPARAM, "null argument");
    *s = ctx->stream;
  });
}

int vreg_ctx_set_stream(vreg_ctx ctx, void* s) {
  return guard([&] {
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->own_stream) VB_CUDA(cudaStreamDestroy(ctx->stream));
    ctx->stream = static_cast<cudaStream_t>(s);
    ctx->own_stream = false;
    for (auto& kv : ctx->plans) {
      VB_CUFFT(cufftSetStream(kv.second.r2c, ctx->stream));
      VB_CUFFT(cufftSetStream(kv.second.c2r, ctx->stream));
      kv.second.stream = ctx->stream;
    }
  });
}

void* vreg_ctx_stream(vreg_ctx ctx) { return ctx->stream; }

int vreg_ctx_synchronize(vreg_ctx ctx) {
  return guard([&] { VB_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int vreg_slab(vreg_ctx ctx, const vreg_grid* g, int* n1_local, int* offset) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    if (n1_local) *n1_local = s.n1l;
    if (offset) *offset = s.off;
  });
}

int vreg_ctx_enable_timers(vreg_ctx ctx, int on) {
  ctx->timers_on = on != 0;
  return VREG_OK;
}

int vreg_ctx_timers(vreg_ctx ctx, double out8[8]) {
  return guard([&] {
    resolve_timers(ctx);
    for (int i = 0; i < T_COUNT; ++i) out8[i] = ctx->timer_acc[i];
  });
}

int vreg_ctx_kernel_stats(vreg_ctx ctx, int idx, char* name64, uint64_t* count,
                          double* seconds) {
  return guard([&] {
    resolve_timers(ctx);
    require(idx >= 0 && size_t(idx) < ctx->kstats.size(), VREG_EPARAM, "no such kernel stat");
    auto it = ctx->kstats.begin();
    std::advance(it, idx);
    std::snprintf(name64, 64, "%s", it->first.c_str());
    *count = it->second.first;
    *seconds = it->second.second;
  });
}

int vreg_ctx_reset_kernel_stats(vreg_ctx ctx) {
  return guard([&] {
    resolve_timers(ctx);
    ctx->kstats.clear();
  });
}

int vreg_ctx_comm(vreg_ctx ctx, uint64_t out9[9]) {
  for (int i = 0; i < C_COUNT; ++i) out9[i] = ctx->comm_bytes[i];
  return VREG_OK;
}

int vreg_ctx_launches(vreg_ctx ctx, uint64_t* out) {
  *out = ctx->launches;
  return VREG_OK;
}

int vreg_ctx_tile_stats(vreg_ctx ctx, uint64_t* tiles, uint64_t* misfit) {
  if (tiles) *tiles = ctx->tiles_built;
  if (misfit) *misfit = ctx->tiles_misfit;
  return VREG_OK;
}

int vreg_alloc(vreg_ctx ctx, size_t bytes, void** out) {
  return guard([&] {
    VB_CUDA(cudaMallocAsync(out, bytes ? bytes : 16, ctx->stream));
  });
}

int vreg_free(vreg_ctx ctx, void* p) {
  return guard([&] {
    if (p) VB_CUDA(cudaFreeAsync(p, ctx->stream));
  });
}

int vreg_memcpy_d2d(vreg_ctx ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    VB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  });
}

int vreg_memcpy_h2d(vreg_ctx ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    VB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int vreg_memcpy_d2h(vreg_ctx ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    VB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int vreg_from_global(vreg_ctx ctx, const vreg_grid* g, int ncomp, const float* host_global,
                     float* dev_local) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    for (int c = 0; c < ncomp; ++c)
      VB_CUDA(cudaMemcpyAsync(dev_local + c * s.local(),
                              host_global + c * s.global() + size_t(s.off) * s.plane(),
                              s.local() * sizeof(float), cudaMemcpyHostToDevice,
                              ctx->stream));
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int vreg_to_global(vreg_ctx ctx, const vreg_grid* g, int ncomp, const float* dev_local,
                   float* host_global) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    if (ctx->nranks == 1) {
      VB_CUDA(cudaMemcpyAsync(host_global, dev_local, ncomp * s.local() * sizeof(float),
                              cudaMemcpyDeviceToHost, ctx->stream));
      VB_CUDA(cudaStreamSynchronize(ctx->stream));
      return;
    }
    // all-gather the slabs (every rank receives the global field)
    float* buf = static_cast<float*>(workspace(ctx, "to_global", s.global() * sizeof(float)));
    for (int c = 0; c < ncomp; ++c) {
      VB_NCCL(ncclAllGather(dev_local + c * s.local(), buf, s.local(), ncclFloat, ctx->comm,
                            ctx->stream));
      VB_CUDA(cudaMemcpyAsync(host_global + c * s.global(), buf, s.global() * sizeof(float),
                              cudaMemcpyDeviceToHost, ctx->stream));
    }
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
