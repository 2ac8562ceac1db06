// Fused multi-GPU SL sweeps over NVLink peer memory.
//
// The inc-state gathers read their x1 ghost planes straight out of the ring
// neighbours' buffers (P2P loads inside the tile kernels: SrcField's ghost
// pointers point into the neighbour's last / first planes), and the
// transpose sweeps' boundary tiles flush their ghost-plane contributions
// straight into the neighbours' outputs (remote float REDs): no halo copy,
// no reverse exchange, no add pass. Ordering between the GPUs is a handful
// of release/acquire flag words in each GPU's IPC-mapped arena:
//   READY  neighbour's w_t is complete          (before reading its planes)
//   DONE   neighbour finished reading my w slot (before overwriting it)
//   ZEROED neighbour's output slice is zeroed   (before adding into it)
//   ADDED  neighbour's remote adds have landed  (before using my slice)
// Sequence numbers follow the program order every rank executes, waits are
// spin loops with a 10 s timeout (__trap) so a broken peer cannot hang the GPU.
#include <cstdlib>

#include "common.cuh"

namespace vb {

namespace {

constexpr size_t kFlagBytes = 4096;  // flags[type][side], side 0: from prev, 1: from next

__global__ void k_p2p_signal(unsigned long long* prev_flags, unsigned long long* next_flags,
                             int type, unsigned long long seq) {
  __threadfence_system();  // the stream's earlier writes (local and remote) first
  // I am my prev's "next" (side 1) and my next's "prev" (side 0)
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(prev_flags + 2 * type + 1), "l"(seq)
               : "memory");
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(next_flags + 2 * type + 0), "l"(seq)
               : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_p2p_wait(const unsigned long long* my_flags, int type, unsigned long long seq) {
  const unsigned long long t0 = now_ns();
  while (ld_acquire(my_flags + 2 * type) < seq || ld_acquire(my_flags + 2 * type + 1) < seq) {
    __nanosleep(200);
    if (now_ns() - t0 > 10000000000ull) __trap();  // peer never arrived: fail, do not hang
  }
  __threadfence_system();
}

}  // namespace

bool p2p_enabled(vreg_ctx ctx) {
  static const bool on = [] {
    const char* e = std::getenv("VREG_P2P_SL");
    return e && e[0] == '1';
  }();
  return on && ctx->nranks > 1;
}

char* p2p_data(vreg_ctx ctx, size_t bytes) {
  const size_t need = kFlagBytes + ((bytes + 255) / 256) * 256;
  if (ctx->parena_bytes >= need) return ctx->parena + kFlagBytes;
  // collective: every rank reaches here with the same size in the same order
  VB_CUDA(cudaStreamSynchronize(ctx->stream));
  VB_CUDA(cudaDeviceSynchronize());
  if (ctx->parena_prev) VB_CUDA(cudaIpcCloseMemHandle(ctx->parena_prev));
  if (ctx->parena_next && ctx->parena_next != ctx->parena_prev)
    VB_CUDA(cudaIpcCloseMemHandle(ctx->parena_next));
  if (ctx->parena) VB_CUDA(cudaFree(ctx->parena));
  ctx->parena_prev = ctx->parena_next = nullptr;
  VB_CUDA(cudaMalloc(&ctx->parena, need));
  VB_CUDA(cudaMemset(ctx->parena, 0, kFlagBytes));
  ctx->parena_bytes = need;
  ctx->pseq = 0;
  ctx->pdone = 0;
  const int p = ctx->nranks;
  cudaIpcMemHandle_t h;
  VB_CUDA(cudaIpcGetMemHandle(&h, ctx->parena));
  char* dh = nullptr;
  VB_CUDA(cudaMalloc(&dh, size_t(p + 1) * sizeof(h)));
  VB_CUDA(cudaMemcpy(dh + size_t(p) * sizeof(h), &h, sizeof(h), cudaMemcpyHostToDevice));
  VB_NCCL(ncclAllGather(dh + size_t(p) * sizeof(h), dh, sizeof(h), ncclChar, ctx->comm,
                        ctx->stream));
  std::vector<cudaIpcMemHandle_t> all(p);
  VB_CUDA(cudaMemcpyAsync(all.data(), dh, size_t(p) * sizeof(h), cudaMemcpyDeviceToHost,
                          ctx->stream));
  VB_CUDA(cudaStreamSynchronize(ctx->stream));
  VB_CUDA(cudaFree(dh));
  const int prev = (ctx->rank - 1 + p) % p, next = (ctx->rank + 1) % p;
  void* ptr = nullptr;
  VB_CUDA(cudaIpcOpenMemHandle(&ptr, all[prev], cudaIpcMemLazyEnablePeerAccess));
  ctx->parena_prev = static_cast<char*>(ptr);
  if (next == prev) {
    ctx->parena_next = ctx->parena_prev;
  } else {
    VB_CUDA(cudaIpcOpenMemHandle(&ptr, all[next], cudaIpcMemLazyEnablePeerAccess));
    ctx->parena_next = static_cast<char*>(ptr);
  }
  // all arenas (and their zeroed flags) exist before anyone signals
  int* scratch = reinterpret_cast<int*>(ctx->parena + kFlagBytes / 2);
  VB_NCCL(ncclAllReduce(scratch, scratch, 1, ncclInt, ncclSum, ctx->comm, ctx->stream));
  VB_CUDA(cudaStreamSynchronize(ctx->stream));
  return ctx->parena + kFlagBytes;
}

const char* p2p_peer(vreg_ctx ctx, const void* local, bool next) {
  const size_t off = static_cast<const char*>(local) - ctx->parena;
  return (next ? ctx->parena_next : ctx->parena_prev) + off;
}

uint64_t p2p_seq(vreg_ctx ctx) { return ++ctx->pseq; }

void p2p_signal(vreg_ctx ctx, int type, uint64_t seq) {
  k_p2p_signal<<<1, 1, 0, ctx->stream>>>(
      reinterpret_cast<unsigned long long*>(ctx->parena_prev),
      reinterpret_cast<unsigned long long*>(ctx->parena_next), type, seq);
  count_launch(ctx);
  check_launch();
}

void p2p_wait(vreg_ctx ctx, int type, uint64_t seq) {
  k_p2p_wait<<<1, 1, 0, ctx->stream>>>(reinterpret_cast<const unsigned long long*>(ctx->parena),
                                       type, seq);
  count_launch(ctx);
  check_launch();
}

}  // namespace vb
