// Slab-decomposed runtime over NCCL (§3):
//  - x1 halo exchange for FD (4 planes) and SL sweeps (dynamic width from the
//    exact max displacement, "computed, not estimated"), ring
//    neighbours via grouped ncclSend/ncclRecv;
//  - reverse halo add for the transpose (scatter) sweeps;
//  - slab 3-D FFT: one batched 2-D R2C over all local x2-x3 planes of all
//    components, written directly in k2-major order, ONE grouped all-to-all
//    to x2 slabs, unpack, batched 1-D C2C along x1; inverse in
//    reverse order;
//  - all-gather of per-plane fp64 reduction partials (p-independent folds).
#include <cmath>

#include "common.cuh"

namespace vb {

namespace {

__global__ void k_add_planes(size_t n, const float* __restrict__ src, float* __restrict__ dst) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] += src[i];
}

// fixed-point accumulators (int32, or packed int64 pairs when n3 % 4 == 0,
// see fixed_add) stored in the float buffers
__global__ void k_add_planes_int(size_t n, const int* __restrict__ src, int* __restrict__ dst) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] += src[i];
}
__global__ void k_add_planes_i64(size_t n2, const long long* __restrict__ src,
                                 long long* __restrict__ dst) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += stride)
    dst[i] += src[i];
}

// received [q][k2l][c*n1l + il][h]  ->  F[c][q*n1l + il][k2l][h]
__global__ void k_unpack(int p, int ncomp, int n1l, int n2l, int h, const float2* __restrict__ in,
                         float2* __restrict__ out) {
  const size_t nc = size_t(p) * n1l * n2l * h;
  const size_t total = nc * ncomp;
  const int B = ncomp * n1l;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int c = int(e / nc);
    size_t r = e - size_t(c) * nc;
    const int k3 = int(r % h);
    r /= h;
    const int k2l = int(r % n2l);
    const int k1 = int(r / n2l);
    const int q = k1 / n1l, il = k1 % n1l;
    out[e] = in[((size_t(q) * n2l + k2l) * B + c * n1l + il) * h + k3];
  }
}

// F[c][q*n1l + il][k2l][h]  ->  send [q][k2l][c*n1l + il][h]
__global__ void k_pack(int p, int ncomp, int n1l, int n2l, int h, const float2* __restrict__ in,
                       float2* __restrict__ out) {
  const size_t nc = size_t(p) * n1l * n2l * h;
  const size_t total = nc * ncomp;
  const int B = ncomp * n1l;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    // e indexes the OUTPUT [q][k2l][b][k3]
    const int k3 = int(e % h);
    size_t r = e / h;
    const int b = int(r % B);
    r /= B;
    const int k2l = int(r % n2l);
    const int q = int(r / n2l);
    const int c = b / n1l, il = b % n1l;
    out[e] = in[size_t(c) * nc + ((size_t(q) * n1l + il) * n2l + k2l) * h + k3];
  }
}

struct DistPlans {
  cufftHandle r2c2d = 0, c2r2d = 0, c2c1d = 0;
};

std::map<std::tuple<vreg_ctx, int, int, int, int>, DistPlans>& dist_plan_map() {
  static std::map<std::tuple<vreg_ctx, int, int, int, int>, DistPlans> m;
  return m;
}

DistPlans& dist_plans(vreg_ctx ctx, const Slab& s, int ncomp) {
  auto key = std::make_tuple(ctx, s.n1, s.n2, s.n3, ncomp);
  auto& m = dist_plan_map();
  auto it = m.find(key);
  if (it != m.end()) return it->second;
  const int p = ctx->nranks, n1l = s.n1l, n2l = s.n2 / p, h = s.n3 / 2 + 1;
  const int B = ncomp * n1l;
  DistPlans d;
  int n2d[2] = {s.n2, s.n3};
  int real_embed[2] = {s.n2, s.n3};
  int cplx_embed[2] = {s.n2, B * h};
  VB_CUFFT(cufftPlanMany(&d.r2c2d, 2, n2d, real_embed, 1, s.n2 * s.n3, cplx_embed, 1, h,
                         CUFFT_R2C, B));
  VB_CUFFT(cufftPlanMany(&d.c2r2d, 2, n2d, cplx_embed, 1, h, real_embed, 1, s.n2 * s.n3,
                         CUFFT_C2R, B));
  int n1d[1] = {s.n1};
  int e1[1] = {s.n1};
  VB_CUFFT(cufftPlanMany(&d.c2c1d, 1, n1d, e1, n2l * h, 1, e1, n2l * h, 1, CUFFT_C2C, n2l * h));
  return m.emplace(key, d).first->second;
}

void alltoall_chunks(vreg_ctx ctx, const float2* send, float2* recv, size_t chunk_elems) {
  const int p = ctx->nranks;
  VB_NCCL(ncclGroupStart());
  for (int q = 0; q < p; ++q) {
    if (q == ctx->rank) continue;
    VB_NCCL(ncclSend(send + size_t(q) * chunk_elems, 2 * chunk_elems, ncclFloat, q, ctx->comm,
                     ctx->stream));
    VB_NCCL(ncclRecv(recv + size_t(q) * chunk_elems, 2 * chunk_elems, ncclFloat, q, ctx->comm,
                     ctx->stream));
  }
  VB_NCCL(ncclGroupEnd());
  VB_CUDA(cudaMemcpyAsync(recv + size_t(ctx->rank) * chunk_elems,
                          send + size_t(ctx->rank) * chunk_elems, chunk_elems * sizeof(float2),
                          cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->comm_bytes[C_FFT_TRANSPOSE] += uint64_t(p - 1) * chunk_elems * sizeof(float2);
  ctx->comm_bytes[C_ALLTOALL] += 1;
}

}  // namespace

Ghosts halo_exchange(vreg_ctx ctx, const Slab& s, const float* f, int G, const char* slot,
                     int timer_cat, int comm_cat) {
  require(G >= 1 && G <= s.n1l, VREG_ECONFIG,
          "ghost width exceeds the slab width (reduce ranks or time step)");
  const size_t gp = size_t(G) * s.plane();
  std::string base(slot);
  float* lo = static_cast<float*>(workspace(ctx, base + "_lo", gp * sizeof(float)));
  float* hi = static_cast<float*>(workspace(ctx, base + "_hi", gp * sizeof(float)));
  Timed t(ctx, timer_cat);
  const int p = ctx->nranks;
  const int prev = (ctx->rank - 1 + p) % p, next = (ctx->rank + 1) % p;
  const float* first = f;
  const float* last = f + size_t(s.n1l - G) * s.plane();
  VB_NCCL(ncclGroupStart());
  // order per peer: the message that lands in the peer's lo goes first
  VB_NCCL(ncclSend(last, gp, ncclFloat, next, ctx->comm, ctx->stream));
  VB_NCCL(ncclSend(first, gp, ncclFloat, prev, ctx->comm, ctx->stream));
  VB_NCCL(ncclRecv(lo, gp, ncclFloat, prev, ctx->comm, ctx->stream));
  VB_NCCL(ncclRecv(hi, gp, ncclFloat, next, ctx->comm, ctx->stream));
  VB_NCCL(ncclGroupEnd());
  ctx->comm_bytes[comm_cat] += 2 * gp * sizeof(float);
  ctx->comm_bytes[C_P2P_MSGS] += 2;
  Ghosts g;
  g.lo = lo;
  g.hi = hi;
  g.G = G;
  return g;
}

GhostAcc ghost_accumulators(vreg_ctx ctx, const Slab& s, int G, const char* slot) {
  require(G >= 1 && G <= s.n1l, VREG_ECONFIG,
          "ghost width exceeds the slab width (reduce ranks or time step)");
  const size_t gp = size_t(G) * s.plane();
  std::string base(slot);
  float* lo = static_cast<float*>(workspace(ctx, base + "_lo", gp * sizeof(float)));
  float* hi = static_cast<float*>(workspace(ctx, base + "_hi", gp * sizeof(float)));
  {
    Timed t(ctx, T_SCATTER_BUF);
    VB_CUDA(cudaMemsetAsync(lo, 0, gp * sizeof(float), ctx->stream));
    VB_CUDA(cudaMemsetAsync(hi, 0, gp * sizeof(float), ctx->stream));
  }
  GhostAcc a;
  a.lo = lo;
  a.hi = hi;
  a.G = G;
  return a;
}

RevHalo halo_reverse_send(vreg_ctx ctx, const Slab& s, const GhostAcc& acc, const char* slot) {
  const size_t gp = size_t(acc.G) * s.plane();
  std::string base(slot);
  RevHalo r;
  r.top = static_cast<float*>(workspace(ctx, base + "_rtop", gp * sizeof(float)));
  r.bot = static_cast<float*>(workspace(ctx, base + "_rbot", gp * sizeof(float)));
  r.G = acc.G;
  const int p = ctx->nranks;
  const int prev = (ctx->rank - 1 + p) % p, next = (ctx->rank + 1) % p;
  Timed t(ctx, T_SCATTER_COMM);
  VB_NCCL(ncclGroupStart());
  VB_NCCL(ncclSend(acc.lo, gp, ncclFloat, prev, ctx->comm, ctx->stream));
  VB_NCCL(ncclSend(acc.hi, gp, ncclFloat, next, ctx->comm, ctx->stream));
  VB_NCCL(ncclRecv(r.top, gp, ncclFloat, next, ctx->comm, ctx->stream));
  VB_NCCL(ncclRecv(r.bot, gp, ncclFloat, prev, ctx->comm, ctx->stream));
  VB_NCCL(ncclGroupEnd());
  ctx->comm_bytes[C_SCATTER_POINTS] += 2 * gp * sizeof(float);
  ctx->comm_bytes[C_P2P_MSGS] += 2;
  return r;
}

void halo_reverse_finish(vreg_ctx ctx, const Slab& s, const RevHalo& r, float* out,
                         bool as_int) {
  const size_t gp = size_t(r.G) * s.plane();
  Timed t(ctx, T_SCATTER_BUF);
  if (as_int && s.n3 % 4 == 0) {  // packed pairs
    k_add_planes_i64<<<blocks_for(gp / 2, 256), 256, 0, ctx->stream>>>(
        gp / 2, reinterpret_cast<const long long*>(r.top),
        reinterpret_cast<long long*>(out + size_t(s.n1l - r.G) * s.plane()));
    k_add_planes_i64<<<blocks_for(gp / 2, 256), 256, 0, ctx->stream>>>(
        gp / 2, reinterpret_cast<const long long*>(r.bot), reinterpret_cast<long long*>(out));
    count_launch(ctx, 2);
    check_launch();
    return;
  }
  if (as_int) {
    k_add_planes_int<<<blocks_for(gp, 256), 256, 0, ctx->stream>>>(
        gp, reinterpret_cast<const int*>(r.top),
        reinterpret_cast<int*>(out + size_t(s.n1l - r.G) * s.plane()));
    k_add_planes_int<<<blocks_for(gp, 256), 256, 0, ctx->stream>>>(
        gp, reinterpret_cast<const int*>(r.bot), reinterpret_cast<int*>(out));
    count_launch(ctx, 2);
    check_launch();
    return;
  }
  k_add_planes<<<blocks_for(gp, 256), 256, 0, ctx->stream>>>(
      gp, r.top, out + size_t(s.n1l - r.G) * s.plane());
  k_add_planes<<<blocks_for(gp, 256), 256, 0, ctx->stream>>>(gp, r.bot, out);
  count_launch(ctx, 2);
  check_launch();
}

void halo_reverse_add(vreg_ctx ctx, const Slab& s, const GhostAcc& acc, float* out,
                      const char* slot, bool as_int) {
  halo_reverse_finish(ctx, s, halo_reverse_send(ctx, s, acc, slot), out, as_int);
}

int sl_ghost_width(vreg_ctx ctx, const Slab& s, const float* disp1, int degree) {
  const double m = reduce(ctx, s, 1, disp1, disp1, true);
  const int G = int(std::floor(m)) + (degree == 3 ? 3 : 2);
  require(G <= s.n1l, VREG_ECONFIG,
          "departure points beyond the neighbouring slab (displacement > slab width)");
  return G;
}

void allgather_partials(vreg_ctx ctx, const Slab& s, const double* d_local, double* d_global,
                        size_t per_plane) {
  Timed t(ctx, T_GHOST);
  VB_NCCL(ncclAllGather(d_local, d_global, size_t(s.n1l) * per_plane, ncclDouble, ctx->comm,
                        ctx->stream));
  ctx->comm_bytes[C_REDUCE] += size_t(s.n1l) * per_plane * sizeof(double) * (ctx->nranks - 1);
}

void dist_fft_forward(vreg_ctx ctx, const Slab& s, int ncomp, const float* f, float2* F) {
  const int p = ctx->nranks;
  require(s.n2 % p == 0, VREG_ECONFIG, "slab FFT needs n2 divisible by the rank count");
  const int n1l = s.n1l, n2l = s.n2 / p, h = s.n3 / 2 + 1;
  const size_t nc = size_t(s.n1) * n2l * h;  // local spectral elements per component
  DistPlans& d = dist_plans(ctx, s, ncomp);
  float2* a = static_cast<float2*>(workspace(ctx, "dfft_a", ncomp * nc * sizeof(float2)));
  float2* b = static_cast<float2*>(workspace(ctx, "dfft_b", ncomp * nc * sizeof(float2)));
  VB_CUFFT(cufftSetStream(d.r2c2d, ctx->stream));
  VB_CUFFT(cufftExecR2C(d.r2c2d, const_cast<float*>(f), reinterpret_cast<cufftComplex*>(a)));
  {
    Timed t(ctx, T_TRANSPOSE);
    alltoall_chunks(ctx, a, b, size_t(n2l) * ncomp * n1l * h);
  }
  k_unpack<<<blocks_for(ncomp * nc, 256), 256, 0, ctx->stream>>>(p, ncomp, n1l, n2l, h, b, F);
  count_launch(ctx);
  check_launch();
  VB_CUFFT(cufftSetStream(d.c2c1d, ctx->stream));
  for (int c = 0; c < ncomp; ++c) {
    float2* Fc = F + size_t(c) * nc;
    VB_CUFFT(cufftExecC2C(d.c2c1d, reinterpret_cast<cufftComplex*>(Fc),
                          reinterpret_cast<cufftComplex*>(Fc), CUFFT_FORWARD));
  }
}

void dist_fft_inverse(vreg_ctx ctx, const Slab& s, int ncomp, float2* F, float* f) {
  const int p = ctx->nranks;
  require(s.n2 % p == 0, VREG_ECONFIG, "slab FFT needs n2 divisible by the rank count");
  const int n1l = s.n1l, n2l = s.n2 / p, h = s.n3 / 2 + 1;
  const size_t nc = size_t(s.n1) * n2l * h;
  DistPlans& d = dist_plans(ctx, s, ncomp);
  float2* a = static_cast<float2*>(workspace(ctx, "dfft_a", ncomp * nc * sizeof(float2)));
  float2* b = static_cast<float2*>(workspace(ctx, "dfft_b", ncomp * nc * sizeof(float2)));
  VB_CUFFT(cufftSetStream(d.c2c1d, ctx->stream));
  for (int c = 0; c < ncomp; ++c) {
    float2* Fc = F + size_t(c) * nc;
    VB_CUFFT(cufftExecC2C(d.c2c1d, reinterpret_cast<cufftComplex*>(Fc),
                          reinterpret_cast<cufftComplex*>(Fc), CUFFT_INVERSE));
  }
  k_pack<<<blocks_for(ncomp * nc, 256), 256, 0, ctx->stream>>>(p, ncomp, n1l, n2l, h, F, a);
  count_launch(ctx);
  check_launch();
  {
    Timed t(ctx, T_TRANSPOSE);
    alltoall_chunks(ctx, a, b, size_t(n2l) * ncomp * n1l * h);
  }
  VB_CUFFT(cufftSetStream(d.c2r2d, ctx->stream));
  VB_CUFFT(cufftExecC2R(d.c2r2d, reinterpret_cast<cufftComplex*>(b), f));
}

}  // namespace vb
