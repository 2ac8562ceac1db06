// Slab-decomposed restriction / prolongation / high pass (spectral.cpp:149-288)
// for the two-level preconditioner on several GPUs.
//
// The reference's partner sums are separable, R = R1 (x) R2 (x) R3 (likewise
// P), and the Hermitian mirror needed on the coarse Nyquist lines of axis 3
// is local to each real x2-x3 plane (G[k2, n3-k3] = conj G[-k2, k3]). So:
//   restrict: 2-D R2C per fine x1 plane -> R2 R3 on the plane spectrum ->
//             all-to-all to coarse-k2 slabs -> 1-D FFT along x1 (fine) -> R1
//             -> inverse 1-D FFT (coarse) -> all-to-all back to coarse x1
//             slabs -> 2-D C2R per coarse plane;
//   prolong : the reverse with P1, P2 P3;
//   high_pass(f) = f - prolong(restrict(f)) (the identity the reference's
//             tests pin, test_spectral.cpp:242-247).
// Scale: unnormalised transforms throughout, one 1/Nf (restrict) or 1/Nc
// (prolong) applied with R1 / P1.
#include "common.cuh"

namespace vb {

namespace {

__device__ __forceinline__ int pm(int a, int n) {
  a %= n;
  return a < 0 ? a + n : a;
}

// plane half spectrum value at (k2, k3) for any k3 in [0, n3): mirror when k3 > n3/2
__device__ __forceinline__ float2 plane_full(const float2* G, int n2, int n3, int k2, int k3) {
  const int h = n3 / 2 + 1;
  if (k3 <= n3 / 2) return G[size_t(k2) * h + k3];
  float2 v = G[size_t((n2 - k2) % n2) * h + (n3 - k3)];
  v.y = -v.y;
  return v;
}

// R2 R3: fine plane spectra [b][n2][hf] -> coarse [b][nc2][hc] (partner sums)
__global__ void k_r23(int B, int n2, int n3, const float2* __restrict__ G, float2* __restrict__ C) {
  const int nc2 = n2 / 2, nc3 = n3 / 2, hf = n3 / 2 + 1, hc = nc3 / 2 + 1;
  const size_t total = size_t(B) * nc2 * hc;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int k3 = int(e % hc);
    const int k2 = int((e / hc) % nc2);
    const int b = int(e / (size_t(hc) * nc2));
    const int nu2 = k2 <= nc2 / 2 ? k2 : k2 - nc2;
    int p2[2] = {nu2, 0}, p3[2] = {k3, 0}, c2 = 1, c3 = 1;
    if (abs(nu2) == nc2 / 2) { p2[0] = nc2 / 2; p2[1] = -nc2 / 2; c2 = 2; }
    if (k3 == nc3 / 2) { p3[0] = nc3 / 2; p3[1] = -nc3 / 2; c3 = 2; }
    const float2* Gb = G + size_t(b) * n2 * hf;
    float ax = 0.f, ay = 0.f;
    for (int i = 0; i < c2; ++i)
      for (int q = 0; q < c3; ++q) {
        const float2 v = plane_full(Gb, n2, n3, pm(p2[i], n2), pm(p3[q], n3));
        ax += v.x;
        ay += v.y;
      }
    C[e] = make_float2(ax, ay);
  }
}

// P2 P3: coarse plane spectra [b][nc2][hc] -> fine [b][n2][hf] (split, zero fill)
__global__ void k_p23(int B, int n2, int n3, const float2* __restrict__ C, float2* __restrict__ G) {
  const int nc2 = n2 / 2, nc3 = n3 / 2, hf = n3 / 2 + 1, hc = nc3 / 2 + 1;
  const size_t total = size_t(B) * n2 * hf;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int f3 = int(e % hf);
    const int f2 = int((e / hf) % n2);
    const int b = int(e / (size_t(hf) * n2));
    const int nu2 = f2 <= n2 / 2 ? f2 : f2 - n2;
    float2 out = make_float2(0.f, 0.f);
    if (abs(nu2) <= nc2 / 2 && f3 <= nc3 / 2) {
      const float w = 1.0f / float((abs(nu2) == nc2 / 2 ? 2 : 1) * (f3 == nc3 / 2 ? 2 : 1));
      const float2 v = C[(size_t(b) * nc2 + pm(nu2, nc2)) * hc + f3];
      out = make_float2(v.x * w, v.y * w);
    }
    G[e] = out;
  }
}

// R1 along the (fine) k1 axis of [c][n1][K][h] -> [c][nc1][K][h], times scale
__global__ void k_r1(int ncomp, int n1, int K, float scale, const float2* __restrict__ F,
                     float2* __restrict__ Fc) {
  const int nc1 = n1 / 2;
  const size_t per_c = size_t(nc1) * K;
  const size_t total = per_c * ncomp;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int c = int(e / per_c);
    const size_t r = e % per_c;
    const int k1 = int(r / K);
    const size_t rest = r % K;
    const int nu1 = k1 <= nc1 / 2 ? k1 : k1 - nc1;
    const float2* Fb = F + size_t(c) * n1 * K;
    float2 v = Fb[size_t(pm(nu1, n1)) * K + rest];
    if (abs(nu1) == nc1 / 2) {
      const float2 w = Fb[size_t(pm(-nu1, n1)) * K + rest];
      v.x += w.x;
      v.y += w.y;
    }
    Fc[e] = make_float2(v.x * scale, v.y * scale);
  }
}

// P1 along k1: [c][nc1][K][h] -> [c][n1][K][h] (split Nyquist, zero fill), times scale
__global__ void k_p1(int ncomp, int n1, int K, float scale, const float2* __restrict__ Fc,
                     float2* __restrict__ F) {
  const int nc1 = n1 / 2;
  const size_t per_c = size_t(n1) * K;
  const size_t total = per_c * ncomp;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int c = int(e / per_c);
    const size_t r = e % per_c;
    const int f1 = int(r / K);
    const size_t rest = r % K;
    const int nu1 = f1 <= n1 / 2 ? f1 : f1 - n1;
    float2 out = make_float2(0.f, 0.f);
    if (abs(nu1) <= nc1 / 2) {
      const float w = scale / (abs(nu1) == nc1 / 2 ? 2.0f : 1.0f);
      const float2 v = Fc[size_t(c) * nc1 * K + size_t(pm(nu1, nc1)) * K + rest];
      out = make_float2(v.x * w, v.y * w);
    }
    F[e] = out;
  }
}

// [b][K2][h] (b = c*L + l, K2 = p*K2l) -> send [q][c][l][K2l][h]
__global__ void k_pack_k2(int ncomp, int L, int p, int K2l, int h, const float2* __restrict__ in,
                          float2* __restrict__ out) {
  const size_t total = size_t(ncomp) * L * p * K2l * h;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int k3 = int(e % h);
    size_t r = e / h;
    const int k2l = int(r % K2l);
    r /= K2l;
    const int l = int(r % L);
    r /= L;
    const int c = int(r % ncomp);
    const int q = int(r / ncomp);
    out[e] = in[((size_t(c) * L + l) * (size_t(p) * K2l) + size_t(q) * K2l + k2l) * h + k3];
  }
}

// received [q][c][l][K2l][h] -> [c][q*L + l][K2l][h]
__global__ void k_unpack_k2(int ncomp, int L, int p, int K2l, int h, const float2* __restrict__ in,
                            float2* __restrict__ out) {
  const size_t total = size_t(ncomp) * p * L * K2l * h;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    // e indexes the OUTPUT [c][x1 = q*L + l][k2l][k3]
    const int k3 = int(e % h);
    size_t r = e / h;
    const int k2l = int(r % K2l);
    r /= K2l;
    const int x1 = int(r % (size_t(p) * L));
    const int c = int(r / (size_t(p) * L));
    const int q = x1 / L, l = x1 % L;
    out[e] = in[((((size_t(q) * ncomp + c) * L + l) * K2l + k2l) * h) + k3];
  }
}

// [c][q*L + l][K2l][h] -> send [q][c][l][K2l][h]   (inverse of k_unpack_k2)
__global__ void k_pack_x1(int ncomp, int L, int p, int K2l, int h, const float2* __restrict__ in,
                          float2* __restrict__ out) {
  const size_t total = size_t(ncomp) * p * L * K2l * h;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    // e indexes the OUTPUT [q][c][l][k2l][k3]
    const int k3 = int(e % h);
    size_t r = e / h;
    const int k2l = int(r % K2l);
    r /= K2l;
    const int l = int(r % L);
    r /= L;
    const int c = int(r % ncomp);
    const int q = int(r / ncomp);
    out[e] = in[((size_t(c) * p * L + size_t(q) * L + l) * K2l + k2l) * h + k3];
  }
}

// received [q][c][l][K2l][h] (q = k2 owner) -> [c*L + l][q*K2l + k2l][h]
__global__ void k_unpack_x1(int ncomp, int L, int p, int K2l, int h, const float2* __restrict__ in,
                            float2* __restrict__ out) {
  const size_t total = size_t(ncomp) * L * p * K2l * h;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    // e indexes the OUTPUT [b = c*L + l][k2 = q*K2l + k2l][k3]
    const int k3 = int(e % h);
    size_t r = e / h;
    const int k2 = int(r % (size_t(p) * K2l));
    const int b = int(r / (size_t(p) * K2l));
    const int q = k2 / K2l, k2l = k2 % K2l;
    const int c = b / L, l = b % L;
    out[e] = in[((((size_t(q) * ncomp + c) * L + l) * K2l + k2l) * h) + k3];
  }
}

struct Plans2 {
  cufftHandle r2c = 0, c2r = 0;
};

// batched 2-D R2C / C2R over B planes of n2 x n3, standard [b][k2][k3] layout
Plans2& plane_plans(vreg_ctx ctx, int n2, int n3, int B) {
  static std::map<std::tuple<vreg_ctx, int, int, int>, Plans2> m;
  auto key = std::make_tuple(ctx, n2, n3, B);
  auto it = m.find(key);
  if (it != m.end()) return it->second;
  Plans2 p;
  int n[2] = {n2, n3};
  VB_CUFFT(cufftPlanMany(&p.r2c, 2, n, nullptr, 1, n2 * n3, nullptr, 1, n2 * (n3 / 2 + 1),
                         CUFFT_R2C, B));
  VB_CUFFT(cufftPlanMany(&p.c2r, 2, n, nullptr, 1, n2 * (n3 / 2 + 1), nullptr, 1, n2 * n3,
                         CUFFT_C2R, B));
  return m.emplace(key, p).first->second;
}

// 1-D C2C along the slowest axis of [n1][K]: stride K, batch K (per component)
cufftHandle axis_plan(vreg_ctx ctx, int n1, int K) {
  static std::map<std::tuple<vreg_ctx, int, int>, cufftHandle> m;
  auto key = std::make_tuple(ctx, n1, K);
  auto it = m.find(key);
  if (it != m.end()) return it->second;
  cufftHandle h;
  int n[1] = {n1};
  VB_CUFFT(cufftPlanMany(&h, 1, n, n, K, 1, n, K, 1, CUFFT_C2C, K));
  return m.emplace(key, h).first->second;
}

void alltoall_equal(vreg_ctx ctx, const float2* send, float2* recv, size_t chunk) {
  const int p = ctx->nranks;
  Timed t(ctx, T_TRANSPOSE);
  VB_NCCL(ncclGroupStart());
  for (int q = 0; q < p; ++q) {
    if (q == ctx->rank) continue;
    VB_NCCL(ncclSend(send + size_t(q) * chunk, 2 * chunk, ncclFloat, q, ctx->comm, ctx->stream));
    VB_NCCL(ncclRecv(recv + size_t(q) * chunk, 2 * chunk, ncclFloat, q, ctx->comm, ctx->stream));
  }
  VB_NCCL(ncclGroupEnd());
  VB_CUDA(cudaMemcpyAsync(recv + size_t(ctx->rank) * chunk, send + size_t(ctx->rank) * chunk,
                          chunk * sizeof(float2), cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->comm_bytes[C_SPECTRAL_GATHER] += uint64_t(p - 1) * chunk * sizeof(float2);
  ctx->comm_bytes[C_ALLTOALL] += 1;
}

template <class K, class... A>
void launch(vreg_ctx ctx, size_t n, K k, A... a) {
  k<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(a...);
  count_launch(ctx);
  check_launch();
}

float2* buf(vreg_ctx ctx, const char* name, size_t n) {
  return static_cast<float2*>(workspace(ctx, name, n * sizeof(float2)));
}

}  // namespace

// fine slab (n1l planes of n2 x n3) -> coarse slab (n1l/2 planes of n2/2 x n3/2)
void dist_restrict(vreg_ctx ctx, const Slab& s, int ncomp, const float* f, float* outc) {
  const int p = ctx->nranks;
  const int n1 = s.n1, n2 = s.n2, n3 = s.n3, nc1 = n1 / 2, nc2 = n2 / 2, nc3 = n3 / 2;
  require(nc1 % p == 0 && nc2 % p == 0, VREG_ECONFIG,
          "restrict: coarse n1 and n2 must be divisible by the rank count");
  const int L = s.n1l, Lc = nc1 / p, K2l = nc2 / p, hf = n3 / 2 + 1, hc = nc3 / 2 + 1;
  Timed t(ctx, T_FFT, "dist_restrict");
  // 1. 2-D R2C of every fine plane, R2 R3 on the plane spectra
  const int B = ncomp * L;
  float2* G = buf(ctx, "rs_G", size_t(B) * n2 * hf);
  Plans2& pf = plane_plans(ctx, n2, n3, B);
  VB_CUFFT(cufftSetStream(pf.r2c, ctx->stream));
  VB_CUFFT(cufftExecR2C(pf.r2c, const_cast<float*>(f), reinterpret_cast<cufftComplex*>(G)));
  float2* C = buf(ctx, "rs_C", size_t(B) * nc2 * hc);
  launch(ctx, size_t(B) * nc2 * hc, k_r23, B, n2, n3, (const float2*)G, C);
  // 2. to coarse-k2 slabs: [c][x1 fine][K2l][hc]
  float2* S = buf(ctx, "rs_S", size_t(B) * nc2 * hc);
  launch(ctx, size_t(B) * nc2 * hc, k_pack_k2, ncomp, L, p, K2l, hc, (const float2*)C, S);
  float2* R = buf(ctx, "rs_R", size_t(B) * nc2 * hc);
  alltoall_equal(ctx, S, R, size_t(ncomp) * L * K2l * hc);
  float2* X = buf(ctx, "rs_X", size_t(ncomp) * n1 * K2l * hc);
  launch(ctx, size_t(ncomp) * n1 * K2l * hc, k_unpack_k2, ncomp, L, p, K2l, hc, (const float2*)R, X);
  // 3. x1 DFT (fine), R1 (+ 1/Nf), inverse x1 DFT (coarse)
  const int K = K2l * hc;
  cufftHandle af = axis_plan(ctx, n1, K), ac = axis_plan(ctx, nc1, K);
  VB_CUFFT(cufftSetStream(af, ctx->stream));
  VB_CUFFT(cufftSetStream(ac, ctx->stream));
  for (int c = 0; c < ncomp; ++c)
    VB_CUFFT(cufftExecC2C(af, reinterpret_cast<cufftComplex*>(X + size_t(c) * n1 * K),
                          reinterpret_cast<cufftComplex*>(X + size_t(c) * n1 * K), CUFFT_FORWARD));
  float2* Y = buf(ctx, "rs_Y", size_t(ncomp) * nc1 * K);
  launch(ctx, size_t(ncomp) * nc1 * K, k_r1, ncomp, n1, K, float(1.0 / double(s.global())),
         (const float2*)X, Y);
  for (int c = 0; c < ncomp; ++c)
    VB_CUFFT(cufftExecC2C(ac, reinterpret_cast<cufftComplex*>(Y + size_t(c) * nc1 * K),
                          reinterpret_cast<cufftComplex*>(Y + size_t(c) * nc1 * K), CUFFT_INVERSE));
  // 4. back to coarse x1 slabs [c*Lc + l][nc2][hc], 2-D C2R per coarse plane
  float2* S2 = buf(ctx, "rs_S", size_t(ncomp) * nc1 * K);
  launch(ctx, size_t(ncomp) * nc1 * K, k_pack_x1, ncomp, Lc, p, K2l, hc, (const float2*)Y, S2);
  float2* R2 = buf(ctx, "rs_R", size_t(ncomp) * nc1 * K);
  alltoall_equal(ctx, S2, R2, size_t(ncomp) * Lc * K2l * hc);
  float2* Gc = buf(ctx, "rs_C", size_t(ncomp) * Lc * nc2 * hc);
  launch(ctx, size_t(ncomp) * Lc * nc2 * hc, k_unpack_x1, ncomp, Lc, p, K2l, hc, (const float2*)R2,
         Gc);
  Plans2& pc = plane_plans(ctx, nc2, nc3, ncomp * Lc);
  VB_CUFFT(cufftSetStream(pc.c2r, ctx->stream));
  VB_CUFFT(cufftExecC2R(pc.c2r, reinterpret_cast<cufftComplex*>(Gc), outc));
}

// coarse slab -> fine slab
void dist_prolong(vreg_ctx ctx, const Slab& s, int ncomp, const float* fc, float* outf) {
  const int p = ctx->nranks;
  const int n1 = s.n1, n2 = s.n2, n3 = s.n3, nc1 = n1 / 2, nc2 = n2 / 2, nc3 = n3 / 2;
  require(nc1 % p == 0 && nc2 % p == 0, VREG_ECONFIG,
          "prolong: coarse n1 and n2 must be divisible by the rank count");
  const int L = s.n1l, Lc = nc1 / p, K2l = nc2 / p, hf = n3 / 2 + 1, hc = nc3 / 2 + 1;
  const int K = K2l * hc;
  Timed t(ctx, T_FFT, "dist_prolong");
  // 1. 2-D R2C per coarse plane
  const int Bc = ncomp * Lc;
  float2* Gc = buf(ctx, "pl_Gc", size_t(Bc) * nc2 * hc);
  Plans2& pc = plane_plans(ctx, nc2, nc3, Bc);
  VB_CUFFT(cufftSetStream(pc.r2c, ctx->stream));
  VB_CUFFT(cufftExecR2C(pc.r2c, const_cast<float*>(fc), reinterpret_cast<cufftComplex*>(Gc)));
  // 2. to coarse-k2 slabs [c][x1c][K2l][hc], x1 DFT (coarse), P1 (+1/Nc), inverse x1 DFT (fine)
  float2* S = buf(ctx, "pl_S", size_t(Bc) * nc2 * hc);
  launch(ctx, size_t(Bc) * nc2 * hc, k_pack_k2, ncomp, Lc, p, K2l, hc, (const float2*)Gc, S);
  float2* R = buf(ctx, "pl_R", size_t(Bc) * nc2 * hc);
  alltoall_equal(ctx, S, R, size_t(ncomp) * Lc * K);
  float2* Y = buf(ctx, "pl_Y", size_t(ncomp) * nc1 * K);
  launch(ctx, size_t(ncomp) * nc1 * K, k_unpack_k2, ncomp, Lc, p, K2l, hc, (const float2*)R, Y);
  cufftHandle ac = axis_plan(ctx, nc1, K), af = axis_plan(ctx, n1, K);
  VB_CUFFT(cufftSetStream(ac, ctx->stream));
  VB_CUFFT(cufftSetStream(af, ctx->stream));
  for (int c = 0; c < ncomp; ++c)
    VB_CUFFT(cufftExecC2C(ac, reinterpret_cast<cufftComplex*>(Y + size_t(c) * nc1 * K),
                          reinterpret_cast<cufftComplex*>(Y + size_t(c) * nc1 * K), CUFFT_FORWARD));
  Slab sc = s;
  sc.n1 = nc1;
  sc.n2 = nc2;
  sc.n3 = nc3;
  float2* X = buf(ctx, "pl_X", size_t(ncomp) * n1 * K);
  launch(ctx, size_t(ncomp) * n1 * K, k_p1, ncomp, n1, K, float(1.0 / double(sc.global())),
         (const float2*)Y, X);
  for (int c = 0; c < ncomp; ++c)
    VB_CUFFT(cufftExecC2C(af, reinterpret_cast<cufftComplex*>(X + size_t(c) * n1 * K),
                          reinterpret_cast<cufftComplex*>(X + size_t(c) * n1 * K), CUFFT_INVERSE));
  // 3. back to fine x1 slabs [c*L + l][nc2][hc], P2 P3, 2-D C2R per fine plane
  const int B = ncomp * L;
  float2* S2 = buf(ctx, "pl_S", size_t(ncomp) * n1 * K);
  launch(ctx, size_t(ncomp) * n1 * K, k_pack_x1, ncomp, L, p, K2l, hc, (const float2*)X, S2);
  float2* R2 = buf(ctx, "pl_R", size_t(ncomp) * n1 * K);
  alltoall_equal(ctx, S2, R2, size_t(ncomp) * L * K);
  float2* C = buf(ctx, "pl_C", size_t(B) * nc2 * hc);
  launch(ctx, size_t(B) * nc2 * hc, k_unpack_x1, ncomp, L, p, K2l, hc, (const float2*)R2, C);
  float2* G = buf(ctx, "pl_G", size_t(B) * n2 * hf);
  launch(ctx, size_t(B) * n2 * hf, k_p23, B, n2, n3, (const float2*)C, G);
  Plans2& pf = plane_plans(ctx, n2, n3, B);
  VB_CUFFT(cufftSetStream(pf.c2r, ctx->stream));
  VB_CUFFT(cufftExecC2R(pf.c2r, reinterpret_cast<cufftComplex*>(G), outf));
}

}  // namespace vb
