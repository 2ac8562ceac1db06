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
#include <algorithm>
#include <cmath>
#include <vector>

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

// Halo chunks for a ghost width G that may exceed the slab width n1l (wide
// halos: large displacements or many ranks). Chunk d = 1..D, D = ceil(G/n1l),
// comes from the rank at ring distance d and has c_d = min(n1l, G - (d-1) n1l)
// planes: the owner's last c_d planes land in lo at plane G - (d-1) n1l - c_d,
// its first c_d planes in hi at plane (d-1) n1l. D = 1 is the plain
// neighbour halo. Per peer pair, messages are issued in d order with the
// lo-bound one first on both sides, which is what NCCL's in-order matching
// of same-peer send/recv needs (at p = 2, or d >= p, peers repeat).
struct HaloChunk {
  int d, c;
  size_t lo_plane, hi_plane;
};
std::vector<HaloChunk> halo_chunks(int n1l, int G) {
  std::vector<HaloChunk> v;
  for (int d = 1; (d - 1) * n1l < G; ++d) {
    const int c = std::min(n1l, G - (d - 1) * n1l);
    v.push_back({d, c, size_t(G - (d - 1) * n1l - c), size_t(d - 1) * n1l});
  }
  return v;
}

namespace {
// ncclSend/ncclRecv pair, or a device copy when the peer is this rank
void xfer(vreg_ctx ctx, const float* src, float* dst, size_t n, int to, int from) {
  if (to == ctx->rank) {
    VB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  VB_NCCL(ncclSend(src, n, ncclFloat, to, ctx->comm, ctx->stream));
  VB_NCCL(ncclRecv(dst, n, ncclFloat, from, ctx->comm, ctx->stream));
}
}  // namespace

Ghosts halo_exchange(vreg_ctx ctx, const Slab& s, const float* f, int G, const char* slot,
                     int timer_cat, int comm_cat) {
  require(G >= 1, VREG_ECONFIG, "ghost width must be positive");
  const size_t gp = size_t(G) * s.plane(), pl = s.plane();
  std::string base(slot);
  float* lo = static_cast<float*>(workspace(ctx, base + "_lo", gp * sizeof(float)));
  float* hi = static_cast<float*>(workspace(ctx, base + "_hi", gp * sizeof(float)));
  Timed t(ctx, timer_cat);
  const int p = ctx->nranks, r = ctx->rank;
  const auto chunks = halo_chunks(s.n1l, G);
  VB_NCCL(ncclGroupStart());
  for (const HaloChunk& h : chunks) {
    const int fwd = (r + h.d) % p, bwd = ((r - h.d) % p + p) % p;
    const size_t n = size_t(h.c) * pl;
    // my last c planes -> lo of rank r+d; lo chunk from rank r-d
    xfer(ctx, f + size_t(s.n1l - h.c) * pl, lo + h.lo_plane * pl, n, fwd, bwd);
    // my first c planes -> hi of rank r-d; hi chunk from rank r+d
    xfer(ctx, f, hi + h.hi_plane * pl, n, bwd, fwd);
  }
  VB_NCCL(ncclGroupEnd());
  ctx->comm_bytes[comm_cat] += 2 * gp * sizeof(float);
  ctx->comm_bytes[C_P2P_MSGS] += 2 * chunks.size();
  Ghosts g;
  g.lo = lo;
  g.hi = hi;
  g.G = G;
  return g;
}

GhostAcc ghost_accumulators(vreg_ctx ctx, const Slab& s, int G, const char* slot) {
  require(G >= 1, VREG_ECONFIG, "ghost width must be positive");
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

// Reverse halo: ghost accumulator chunks go back to their owners; the
// received chunks keep the senders' offsets (top mirrors lo, bot mirrors hi).
RevHalo halo_reverse_send(vreg_ctx ctx, const Slab& s, const GhostAcc& acc, const char* slot) {
  const size_t gp = size_t(acc.G) * s.plane(), pl = s.plane();
  std::string base(slot);
  RevHalo r;
  r.top = static_cast<float*>(workspace(ctx, base + "_rtop", gp * sizeof(float)));
  r.bot = static_cast<float*>(workspace(ctx, base + "_rbot", gp * sizeof(float)));
  r.G = acc.G;
  const int p = ctx->nranks, me = ctx->rank;
  const auto chunks = halo_chunks(s.n1l, acc.G);
  Timed t(ctx, T_SCATTER_COMM);
  VB_NCCL(ncclGroupStart());
  for (const HaloChunk& h : chunks) {
    const int fwd = (me + h.d) % p, bwd = ((me - h.d) % p + p) % p;
    const size_t n = size_t(h.c) * pl;
    // lo chunk -> its owner r-d; the owner-side copy arrives from r+d into top
    xfer(ctx, acc.lo + h.lo_plane * pl, r.top + h.lo_plane * pl, n, bwd, fwd);
    // hi chunk -> its owner r+d; from r-d into bot
    xfer(ctx, acc.hi + h.hi_plane * pl, r.bot + h.hi_plane * pl, n, fwd, bwd);
  }
  VB_NCCL(ncclGroupEnd());
  ctx->comm_bytes[C_SCATTER_POINTS] += 2 * gp * sizeof(float);
  ctx->comm_bytes[C_P2P_MSGS] += 2 * chunks.size();
  return r;
}

void halo_reverse_finish(vreg_ctx ctx, const Slab& s, const RevHalo& r, float* out,
                         bool as_int) {
  const size_t pl = s.plane();
  Timed t(ctx, T_SCATTER_BUF);
  // chunk d adds into my last c planes (top) and my first c planes (bot);
  // chunks overlap when G > n1l, so the adds stay stream-ordered
  for (const HaloChunk& h : halo_chunks(s.n1l, r.G)) {
    const size_t n = size_t(h.c) * pl;
    const float* top = r.top + h.lo_plane * pl;
    const float* bot = r.bot + h.hi_plane * pl;
    float* otop = out + size_t(s.n1l - h.c) * pl;
    if (as_int && s.n3 % 4 == 0) {  // packed pairs
      k_add_planes_i64<<<blocks_for(n / 2, 256), 256, 0, ctx->stream>>>(
          n / 2, reinterpret_cast<const long long*>(top), reinterpret_cast<long long*>(otop));
      k_add_planes_i64<<<blocks_for(n / 2, 256), 256, 0, ctx->stream>>>(
          n / 2, reinterpret_cast<const long long*>(bot), reinterpret_cast<long long*>(out));
    } else if (as_int) {
      k_add_planes_int<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(
          n, reinterpret_cast<const int*>(top), reinterpret_cast<int*>(otop));
      k_add_planes_int<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(
          n, reinterpret_cast<const int*>(bot), reinterpret_cast<int*>(out));
    } else {
      k_add_planes<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(n, top, otop);
      k_add_planes<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(n, bot, out);
    }
    count_launch(ctx, 2);
    check_launch();
  }
}

void halo_reverse_add(vreg_ctx ctx, const Slab& s, const GhostAcc& acc, float* out,
                      const char* slot, bool as_int) {
  halo_reverse_finish(ctx, s, halo_reverse_send(ctx, s, acc, slot), out, as_int);
}

int sl_ghost_width(vreg_ctx ctx, const Slab& s, const float* disp1, int degree) {
  const double m = reduce(ctx, s, 1, disp1, disp1, true);
  const int G = int(std::floor(m)) + (degree != 1 ? 3 : 2);
  // wider than the slab: multi-rank (wide) halos, see halo_chunks
  require(G <= 2 * s.n1, VREG_ECONFIG, "displacement exceeds twice the domain");
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

extern "C" int vreg_halo_chunks(int n1l, int G, int cap, int* d, int* c, long long* lo,
                                long long* hi) {
  if (n1l < 1 || G < 1 || cap < 0) return -1;
  const auto v = vb::halo_chunks(n1l, G);
  for (size_t i = 0; i < v.size() && int(i) < cap; ++i) {
    d[i] = v[i].d;
    c[i] = v[i].c;
    lo[i] = (long long)v[i].lo_plane;
    hi[i] = (long long)v[i].hi_plane;
  }
  return int(v.size());
}
