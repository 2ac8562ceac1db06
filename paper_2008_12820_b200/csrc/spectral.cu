// Pointwise spectral operators on cuFFT half spectra (proj/src/spectral.cpp).
//
// One fused pass per operator over all components of the half spectrum
// n1 x n2 x (n3/2+1): the symbol, the 1/N inverse normalisation
// (fft.cpp:56-64) and any cross-component coupling (Leray) are applied in a
// single read+write of the spectrum. Forward R2C / inverse C2R are batched
// over the 3 components (one plan each, shared work area) and timed as
// "fft" (counters.hpp:69-78).
//
// Spectral element addressing is written against a slab descriptor
// (k1 all, k2 in [k2off, k2off + n2l), k3 half) so the same symbol kernels
// run on the x2-slab layout of the distributed transform (dist.cu).
#include <cmath>

#include "common.cuh"

namespace vb {

struct SpecDesc {
  int n1, n2, n3, h;  // h = n3/2 + 1
  int n2l, k2off;     // local k2 range
  size_t nc;          // local complex elements per component
};

// 32-bit index arithmetic: a GPU's spectra stay below 2^31 elements, and
// 64-bit div/mod (~100 instructions each) dominated these streaming passes.
__device__ __forceinline__ void spec_index(const SpecDesc& d, unsigned e, int& k1, int& k2, int& k3) {
  k3 = int(e % unsigned(d.h));
  const unsigned r = e / unsigned(d.h);
  k2 = int(r % unsigned(d.n2l)) + d.k2off;
  k1 = int(r / unsigned(d.n2l));
}

// Flat element e of ncomp stacked half spectra [c][k1][k2][k3 < h]: the
// component and wavenumbers by multiply-high divisions (FastDiv).
struct Idx3 {
  FastDiv h, n2, nc;
  Idx3(unsigned hh, unsigned nn2, size_t ncc) : h(hh), n2(nn2), nc(unsigned(ncc)) {}
  __device__ __forceinline__ int split(unsigned e, int& k1, int& k2, int& k3) const {
    unsigned r, k3u, k2u;
    const unsigned c = nc.divmod(e, r);
    const unsigned q = h.divmod(r, k3u);
    k1 = int(n2.divmod(q, k2u));
    k2 = int(k2u);
    k3 = int(k3u);
    return int(c);
  }
};

__device__ __forceinline__ float sfreq(int k, int n) { return float(k <= n / 2 ? k : k - n); }

namespace {

constexpr unsigned kT = 256;

// F *= scale * sym(k), sym = beta |k|^2 (zero mode: unit or 0) [regop] or
// 1 / (beta |k|^2) (zero mode 1/beta) [inv_regop] (spectral.cpp:48-93);
// order 2: |k|^4 (H2).
__global__ void k_symbol(SpecDesc d, Idx3 ix, int ncomp, float2* __restrict__ F, float beta,
                         int inverse, int unit_zero, float scale, int order) {
  // flat over every (component, k1, local k2, k3) element: one row of
  // n3/2 + 1 per CTA left most threads idle on the odd tail element
  const unsigned total = unsigned(ncomp) * unsigned(d.n1) * unsigned(d.n2l) * unsigned(d.h);
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    int k1, k2l, k3;
    ix.split(e, k1, k2l, k3);
    const float f1 = sfreq(k1, d.n1), f2 = sfreq(k2l + d.k2off, d.n2), f3 = float(k3);
    float sym = f1 * f1 + f2 * f2 + f3 * f3;
    if (order == 2) sym *= sym;  // H2: |k|^4
    float m;
    if (inverse) {
      if (sym == 0.0f) sym = 1.0f;
      m = scale / (beta * sym);
    } else {
      if (sym == 0.0f) sym = unit_zero ? 1.0f : 0.0f;
      m = scale * (beta * sym);
    }
    float2 v = F[e];
    v.x *= m;
    v.y *= m;
    F[e] = v;
  }
}

// Cubic B-spline prefilter: F *= scale / (b(k1) b(k2) b(k3)), b(k) =
// (2 + cos(2 pi k / n)) / 3 -- the spectrum of the periodic B-spline
// coefficients that interpolate the field at the nodes (b is the symbol of
// the node samples 1/6, 2/3, 1/6 of the cubic B-spline).
__global__ void k_bspline_prefilter(SpecDesc d, int ncomp, float2* __restrict__ F, float scale) {
  const int k2l = blockIdx.x, c = blockIdx.y / d.n1, k1 = blockIdx.y - c * d.n1;
  const float b12 = ((2.0f + cospif(2.0f * float(k1) / float(d.n1))) / 3.0f) *
                    ((2.0f + cospif(2.0f * float(k2l + d.k2off) / float(d.n2))) / 3.0f);
  float2* R = F + size_t(c) * d.nc + (size_t(k1) * d.n2l + k2l) * d.h;
  for (int k3 = threadIdx.x; k3 < d.h; k3 += blockDim.x) {
    const float b = b12 * ((2.0f + cospif(2.0f * float(k3) / float(d.n3))) / 3.0f);
    const float m = scale / b;
    float2 v = R[k3];
    v.x *= m;
    v.y *= m;
    R[k3] = v;
  }
}

// Leray: F_c -= f_c (f . F)/|k|^2, zero mode untouched (spectral.cpp:120-147).
__global__ void k_leray(SpecDesc d, float2* __restrict__ F, float scale) {
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < unsigned(d.nc); e += stride) {
    int k1, k2, k3;
    spec_index(d, e, k1, k2, k3);
    const float f1 = sfreq(k1, d.n1), f2 = sfreq(k2, d.n2), f3 = float(k3);
    const float ksq = f1 * f1 + f2 * f2 + f3 * f3;
    float2 a = F[e], b = F[d.nc + e], c = F[2 * d.nc + e];
    if (ksq != 0.0f) {
      const float kvx = (f1 * a.x + f2 * b.x + f3 * c.x) / ksq;
      const float kvy = (f1 * a.y + f2 * b.y + f3 * c.y) / ksq;
      a.x -= f1 * kvx; a.y -= f1 * kvy;
      b.x -= f2 * kvx; b.y -= f2 * kvy;
      c.x -= f3 * kvx; c.y -= f3 * kvy;
    }
    a.x *= scale; a.y *= scale; b.x *= scale; b.y *= scale; c.x *= scale; c.y *= scale;
    F[e] = a;
    F[d.nc + e] = b;
    F[2 * d.nc + e] = c;
  }
}

// Per-(component, k2-row) fp64 partial of sum w3 |k|^2 |F|^2 over k3, k1
// (spectral.cpp:95-118: k2-major fold).
__global__ void k_seminorm_rows(SpecDesc d, const float2* __restrict__ F, double* __restrict__ rows,
                                int order) {
  const int c = blockIdx.y;
  const int k2l = blockIdx.x;
  const int k2 = k2l + d.k2off;
  const float f2 = sfreq(k2, d.n2);
  const float2* Fc = F + size_t(c) * d.nc;
  double acc = 0.0;
  const int cnt = d.n1 * d.h;
  for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
    const int k1 = t / d.h, k3 = t % d.h;
    const float f1 = sfreq(k1, d.n1);
    const double w3 = (k3 == 0 || 2 * k3 == d.n3) ? 1.0 : 2.0;
    double sym = double(f1) * f1 + double(f2) * f2 + double(k3) * k3;
    if (order == 2) sym *= sym;
    const float2 v = Fc[(size_t(k1) * d.n2l + k2l) * d.h + k3];
    acc += w3 * sym * (double(v.x) * v.x + double(v.y) * v.y);
  }
  __shared__ double sh[kT];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (unsigned s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) rows[size_t(c) * d.n2l + k2l] = sh[0];
}

// Full-space lookup of a half spectrum (fft.hpp:35-43).
__device__ __forceinline__ float2 full_at(const float2* F, int n1, int n2, int n3, int k1, int k2,
                                          int k3) {
  const int h = n3 / 2 + 1;
  if (k3 <= n3 / 2) return F[(size_t(k1) * n2 + k2) * h + k3];
  const int m1 = (n1 - k1) % n1, m2 = (n2 - k2) % n2, m3 = n3 - k3;
  float2 v = F[(size_t(m1) * n2 + m2) * h + m3];
  v.y = -v.y;
  return v;
}

__device__ __forceinline__ int pmod(int a, int n) {
  a %= n;
  return a < 0 ? a + n : a;
}

// Coarse half spectrum from the fine one: partner sums on the coarse
// Nyquist lines, times scale (spectral.cpp:149-174).
__global__ void k_restrict(Idx3 ix, int nf1, int nf2, int nf3, int nc1, int nc2, int nc3, int ncomp,
                           const float2* __restrict__ Ff, float2* __restrict__ Fc, float scale) {
  const int hc = nc3 / 2 + 1, hf = nf3 / 2 + 1;
  const size_t ncc = size_t(nc1) * nc2 * hc, ncf = size_t(nf1) * nf2 * hf;
  const unsigned total = unsigned(ncc) * unsigned(ncomp);
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    int k1, k2, k3;
    const int c = ix.split(e, k1, k2, k3);
    const int nu1 = k1 <= nc1 / 2 ? k1 : k1 - nc1;
    const int nu2 = k2 <= nc2 / 2 ? k2 : k2 - nc2;
    const int nu3 = k3;
    int p1[2] = {nu1, 0}, p2[2] = {nu2, 0}, p3[2] = {nu3, 0};
    int c1 = 1, c2 = 1, c3 = 1;
    if (abs(nu1) == nc1 / 2) { p1[0] = nc1 / 2; p1[1] = -nc1 / 2; c1 = 2; }
    if (abs(nu2) == nc2 / 2) { p2[0] = nc2 / 2; p2[1] = -nc2 / 2; c2 = 2; }
    if (abs(nu3) == nc3 / 2) { p3[0] = nc3 / 2; p3[1] = -nc3 / 2; c3 = 2; }
    const float2* F = Ff + size_t(c) * ncf;
    float ax = 0.f, ay = 0.f;
    for (int a = 0; a < c1; ++a)
      for (int b = 0; b < c2; ++b)
        for (int q = 0; q < c3; ++q) {
          const float2 v = full_at(F, nf1, nf2, nf3, pmod(p1[a], nf1), pmod(p2[b], nf2),
                                   pmod(p3[q], nf3));
          ax += v.x;
          ay += v.y;
        }
    Fc[e] = make_float2(ax * scale, ay * scale);
  }
}

// Inverse regularisation symbol 1 / (beta |k|^2) (|k|^4 for H2), zero mode
// 1 / beta (spectral.cpp:72-93); even in every wavenumber.
__device__ __forceinline__ float inv_symbol(int nu1, int nu2, int nu3, float beta, int order) {
  float sym = float(nu1) * nu1 + float(nu2) * nu2 + float(nu3) * nu3;
  if (order == 2) sym *= sym;
  if (sym == 0.0f) sym = 1.0f;
  return 1.0f / (beta * sym);
}

// Both restrictions of the two-level apply from one pass over the fine
// spectrum: Fr = restrict(F) and Fs = restrict(InvA F). Restriction only
// pairs alias partners of equal |k| (the coarse Nyquist lines), so
// restrict(InvA F) = InvA_c restrict(F) mode by mode.
__global__ void k_restrict_pair(Idx3 ix, int nf1, int nf2, int nf3, int nc1, int nc2, int nc3,
                                const float2* __restrict__ Ff, float2* __restrict__ Fr,
                                float2* __restrict__ Fs, float scale, float beta, int order) {
  const int hc = nc3 / 2 + 1, hf = nf3 / 2 + 1;
  const size_t ncc = size_t(nc1) * nc2 * hc, ncf = size_t(nf1) * nf2 * hf;
  const unsigned total = 3u * unsigned(ncc);
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    int k1, k2, k3;
    const int c = ix.split(e, k1, k2, k3);
    const int nu1 = k1 <= nc1 / 2 ? k1 : k1 - nc1;
    const int nu2 = k2 <= nc2 / 2 ? k2 : k2 - nc2;
    const int nu3 = k3;
    int p1[2] = {nu1, 0}, p2[2] = {nu2, 0}, p3[2] = {nu3, 0};
    int c1 = 1, c2 = 1, c3 = 1;
    if (abs(nu1) == nc1 / 2) { p1[0] = nc1 / 2; p1[1] = -nc1 / 2; c1 = 2; }
    if (abs(nu2) == nc2 / 2) { p2[0] = nc2 / 2; p2[1] = -nc2 / 2; c2 = 2; }
    if (abs(nu3) == nc3 / 2) { p3[0] = nc3 / 2; p3[1] = -nc3 / 2; c3 = 2; }
    const float2* F = Ff + size_t(c) * ncf;
    float ax = 0.f, ay = 0.f;
    for (int a = 0; a < c1; ++a)
      for (int b = 0; b < c2; ++b)
        for (int q = 0; q < c3; ++q) {
          const float2 v = full_at(F, nf1, nf2, nf3, pmod(p1[a], nf1), pmod(p2[b], nf2),
                                   pmod(p3[q], nf3));
          ax += v.x;
          ay += v.y;
        }
    const float m = inv_symbol(nu1, nu2, nu3, beta, order);
    if (Fr) Fr[e] = make_float2(ax * scale, ay * scale);
    Fs[e] = make_float2(ax * scale * m, ay * scale * m);
  }
}

// Fine half spectrum from the coarse one: coarse modes split evenly over
// their fine partners, zero outside the band (spectral.cpp:176-203).
__device__ __forceinline__ float2 prolong_elem(int nf1, int nf2, int nc1, int nc2, int nc3,
                                               const float2* __restrict__ Fc, int f1, int f2,
                                               int f3, float scale) {
  const int hc = nc3 / 2 + 1;
  const int nu1 = f1 <= nf1 / 2 ? f1 : f1 - nf1;
  const int nu2 = f2 <= nf2 / 2 ? f2 : f2 - nf2;
  if (abs(nu1) <= nc1 / 2 && abs(nu2) <= nc2 / 2 && f3 <= nc3 / 2) {
    const int cnt = (abs(nu1) == nc1 / 2 ? 2 : 1) * (abs(nu2) == nc2 / 2 ? 2 : 1) *
                    (f3 == nc3 / 2 ? 2 : 1);
    const float2 v = Fc[(size_t(pmod(nu1, nc1)) * nc2 + pmod(nu2, nc2)) * hc + f3];
    const float m = scale / float(cnt);
    return make_float2(v.x * m, v.y * m);
  }
  return make_float2(0.f, 0.f);
}

__global__ void k_prolong(Idx3 ix, int nf1, int nf2, int nf3, int nc1, int nc2, int nc3, int ncomp,
                          const float2* __restrict__ Fc, float2* __restrict__ Ff, float scale) {
  const int hc = nc3 / 2 + 1, hf = nf3 / 2 + 1;
  const size_t ncc = size_t(nc1) * nc2 * hc, ncf = size_t(nf1) * nf2 * hf;
  const unsigned total = unsigned(ncf) * unsigned(ncomp);
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    int f1, f2, f3;
    const int c = ix.split(e, f1, f2, f3);
    Ff[e] = prolong_elem(nf1, nf2, nc1, nc2, nc3, Fc + size_t(c) * ncc, f1, f2, f3, scale);
  }
}

// High pass with the alias-pair remainder on the coarse Nyquist lines
// (spectral.cpp:205-240); out of place (reads the original spectrum).
__device__ __forceinline__ float2 high_pass_elem(int n1, int n2, int n3,
                                                 const float2* __restrict__ F, int k1, int k2,
                                                 int k3, float scale) {
  const int h = n3 / 2 + 1;
  const int b1 = n1 / 4, b2 = n2 / 4, b3 = n3 / 4;
  const int nu1 = k1 <= n1 / 2 ? k1 : k1 - n1;
  const int nu2 = k2 <= n2 / 2 ? k2 : k2 - n2;
  float2 v = F[(size_t(k1) * n2 + k2) * h + k3];
  if (!(abs(nu1) > b1 || abs(nu2) > b2 || k3 > b3)) {
    const bool y1 = abs(nu1) == b1, y2 = abs(nu2) == b2, y3 = k3 == b3;
    if (!y1 && !y2 && !y3) {
      v = make_float2(0.f, 0.f);
    } else {
      float ax = 0.f, ay = 0.f;
      int cnt = 0;
      for (int s1 = 0; s1 < (y1 ? 2 : 1); ++s1)
        for (int s2 = 0; s2 < (y2 ? 2 : 1); ++s2)
          for (int s3 = 0; s3 < (y3 ? 2 : 1); ++s3) {
            const int m1 = y1 ? (s1 ? n1 - b1 : b1) : k1;
            const int m2 = y2 ? (s2 ? n2 - b2 : b2) : k2;
            const int m3 = y3 ? (s3 ? n3 - b3 : b3) : k3;
            const float2 w = full_at(F, n1, n2, n3, m1, m2, m3);
            ax += w.x;
            ay += w.y;
            ++cnt;
          }
      v.x -= ax / float(cnt);
      v.y -= ay / float(cnt);
    }
  }
  return make_float2(v.x * scale, v.y * scale);
}

__global__ void k_high_pass(Idx3 ix, int n1, int n2, int n3, int ncomp, const float2* __restrict__ Fin,
                            float2* __restrict__ Fout, float scale) {
  const int h = n3 / 2 + 1;
  const size_t nc = size_t(n1) * n2 * h;
  const unsigned total = unsigned(nc) * unsigned(ncomp);
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    int k1, k2, k3;
    const int c = ix.split(e, k1, k2, k3);
    Fout[e] = high_pass_elem(n1, n2, n3, Fin + size_t(c) * nc, k1, k2, k3, scale);
  }
}

// Fused end of the two-level apply: G = prolong(Fc) + high_pass(Ff) on the
// fine half spectrum, flat over the elements (a CTA per n3/2 + 1 row left
// most threads idle on the odd tail: 170 us -> memory speed at 256^3).
// One warp per (component, k1, k2) row of the fine half spectrum: the row's
// band test, coarse row and partial |k|^2 are computed once, lanes walk k3
// in batches of four chunks whose loads are issued together (one load in
// flight per warp left the pass latency-bound; a flat four-per-thread
// mapping measured 147 vs 138 us). Elements on the coarse Nyquist lines
// (alias-partner sums) take the element functions; the arithmetic is the
// same everywhere.
__global__ void k_prolong_plus_hp(int nf1, int nf2, int nf3, int nc1, int nc2, int nc3,
                                  const float2* __restrict__ Fc, const float2* __restrict__ Ff,
                                  float2* __restrict__ G, float scale_p, float scale_h,
                                  float beta, int order) {
  const int hf = nf3 / 2 + 1, hc = nc3 / 2 + 1;
  const size_t ncf = size_t(nf1) * nf2 * hf, ncc = size_t(nc1) * nc2 * hc;
  const int b1 = nc1 / 2, b2 = nc2 / 2, b3 = nc3 / 2;  // coarse Nyquist = n / 4
  const int lane = threadIdx.x & 31;
  const int rows = 3 * nf1 * nf2;
  const int wstride = gridDim.x * (blockDim.x >> 5);
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += wstride) {
    const int c = row / (nf1 * nf2), k12 = row - c * nf1 * nf2;
    const int k1 = k12 / nf2, k2 = k12 - k1 * nf2;
    const int nu1 = k1 <= nf1 / 2 ? k1 : k1 - nf1, nu2 = k2 <= nf2 / 2 ? k2 : k2 - nf2;
    const int a1 = abs(nu1), a2 = abs(nu2);
    const bool band = a1 <= b1 && a2 <= b2;
    const bool nyq = a1 == b1 || a2 == b2;
    const float s12 = float(nu1) * nu1 + float(nu2) * nu2;
    const float2* F = Ff + size_t(c) * ncf;
    const float2* Fr = F + size_t(k12) * hf;
    float2* Gr = G + size_t(c) * ncf + size_t(k12) * hf;
    const float2* Cr =
        band ? Fc + size_t(c) * ncc + (size_t(nu1 < 0 ? nu1 + nc1 : nu1) * nc2 +
                                       (nu2 < 0 ? nu2 + nc2 : nu2)) * hc
             : nullptr;
    for (int base = 0; base < hf; base += 128) {
      float2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k3 = base + 32 * u + lane;
        v[u] = make_float2(0.f, 0.f);
        if (k3 < hf) v[u] = (!band || k3 > b3) ? Fr[k3] : ((!nyq && k3 != b3) ? Cr[k3] : v[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k3 = base + 32 * u + lane;
        if (k3 >= hf) continue;
        float sym = s12 + float(k3) * k3;
        if (order == 2) sym *= sym;
        if (sym == 0.0f) sym = 1.0f;
        const float hs = __fdividef(scale_h, beta * sym);  // approximate reciprocal (2 ulp)
        float2 out;
        if (!band || k3 > b3) {  // outside the coarse band: high pass keeps InvA F
          out = make_float2(0.0f + v[u].x * hs, 0.0f + v[u].y * hs);
        } else if (!nyq && k3 != b3) {  // band interior: the prolongation alone
          out = make_float2(v[u].x * scale_p + 0.0f, v[u].y * scale_p + 0.0f);
        } else {  // coarse Nyquist lines: partner sums
          const float2 a = prolong_elem(nf1, nf2, nc1, nc2, nc3, Fc + size_t(c) * ncc, k1, k2,
                                        k3, scale_p);
          const float2 b = high_pass_elem(nf1, nf2, nf3, F, k1, k2, k3, hs);
          out = make_float2(a.x + b.x, a.y + b.y);
        }
        Gr[k3] = out;
      }
    }
  }
}

// out_c += g_c (g . s) (precond.hpp:36-37)
__global__ void k_h0_pointwise(size_t n, const float* __restrict__ s, const float* __restrict__ g,
                               float* __restrict__ out) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n; p += stride) {
    const float g1 = g[p], g2 = g[n + p], g3 = g[2 * n + p];
    const float dot = g1 * s[p] + g2 * s[n + p] + g3 * s[2 * n + p];
    out[p] += dot * g1;
    out[n + p] += dot * g2;
    out[2 * n + p] += dot * g3;
  }
}

}  // namespace

// ---- transform plumbing (single rank: cuFFT 3-D; multi-rank: dist.cu) ----

SpecDesc spec_desc(vreg_ctx ctx, const Slab& s) {
  SpecDesc d;
  d.n1 = s.n1;
  d.n2 = s.n2;
  d.n3 = s.n3;
  d.h = s.n3 / 2 + 1;
  d.n2l = s.n2 / ctx->nranks;
  d.k2off = ctx->rank * d.n2l;
  d.nc = size_t(s.n1) * d.n2l * d.h;
  require(3 * d.nc < (size_t(1) << 31), VREG_EDIM, "spectrum too large for 32-bit indexing");
  return d;
}

void dist_fft_forward(vreg_ctx ctx, const Slab& s, int ncomp, const float* f, float2* F);
void dist_fft_inverse(vreg_ctx ctx, const Slab& s, int ncomp, float2* F, float* f);
void dist_restrict(vreg_ctx ctx, const Slab& s, int ncomp, const float* f, float* outc);
void dist_prolong(vreg_ctx ctx, const Slab& s, int ncomp, const float* fc, float* outf);

float2* spec_buffer(vreg_ctx ctx, const SpecDesc& d, int ncomp, const char* name) {
  return static_cast<float2*>(workspace(ctx, name, d.nc * size_t(ncomp) * sizeof(float2)));
}

void fft_forward(vreg_ctx ctx, const Slab& s, int ncomp, const float* f, float2* F) {
  Timed t(ctx, T_FFT, "fft_r2c");
  if (ctx->nranks > 1) {
    dist_fft_forward(ctx, s, ncomp, f, F);
    return;
  }
  FftPlans& p = fft_plans(ctx, s.n1, s.n2, s.n3, ncomp);
  VB_CUFFT(cufftSetStream(p.r2c, ctx->stream));  // main or side stream (matvec overlap)
  VB_CUFFT(cufftExecR2C(p.r2c, const_cast<float*>(f), reinterpret_cast<cufftComplex*>(F)));
}

void fft_inverse(vreg_ctx ctx, const Slab& s, int ncomp, float2* F, float* f) {
  Timed t(ctx, T_FFT, "fft_c2r");
  if (ctx->nranks > 1) {
    dist_fft_inverse(ctx, s, ncomp, F, f);
    return;
  }
  FftPlans& p = fft_plans(ctx, s.n1, s.n2, s.n3, ncomp);
  VB_CUFFT(cufftSetStream(p.c2r, ctx->stream));
  VB_CUFFT(cufftExecC2R(p.c2r, reinterpret_cast<cufftComplex*>(F), f));
}

void apply_symbol(vreg_ctx ctx, const SpecDesc& d, int ncomp, float2* F, double beta, bool inverse,
                  bool unit_zero, double scale) {
  Timed t(ctx, T_FFT, "spec_symbol");
  k_symbol<<<blocks_for(size_t(ncomp) * d.nc, 256), 256, 0, ctx->stream>>>(
      d, Idx3(unsigned(d.h), unsigned(d.n2l), d.nc), ncomp, F, float(beta), inverse ? 1 : 0, unit_zero ? 1 : 0, float(scale), ctx->reg_order);
  count_launch(ctx);
  check_launch();
}

bool regop_separable(vreg_ctx ctx, const Slab& s, const float* v3, double beta, float* out3,
                     bool unit_zero);

// out3 = beta A v3 (or its inverse); used by the fused matvec too. The
// forward operator is separable (|k|^2 = k1^2 + k2^2 + k3^2; a unit null-mode
// symbol is + beta mean(v)) and runs as three 1-D spectral passes
// (spec_axis.cu) where the grid allows; the inverse stays on cuFFT.
void spectral_regop(vreg_ctx ctx, const Slab& s, const float* v3, double beta, bool unit_zero,
                    bool inverse, float* out3) {
  require(beta > 0.0, VREG_EPARAM, "regularization beta must be > 0");
  // H2 (|k|^4) takes the 3-D transform with the order-2 symbol: composing
  // two separable H1 sweeps would amplify the fp32 transform noise of the
  // first by the second's |k|^2 (measured ~1e-5 relative on single modes)
  if (!inverse && ctx->reg_order == 1 && regop_separable(ctx, s, v3, beta, out3, unit_zero))
    return;
  // (InvA as 2-D plane transforms around one fused x1 FFT/symbol/IFFT pencil
  // pass: 86 vs 91 us per 128^3 apply, but its 226 MB plane workspace at
  // 256^3 slowed the registration's gradient phase by 10 ms; not kept)
  const SpecDesc d = spec_desc(ctx, s);
  float2* F = spec_buffer(ctx, d, 3, "spec3");
  fft_forward(ctx, s, 3, v3, F);
  apply_symbol(ctx, d, 3, F, beta, inverse, unit_zero, 1.0 / double(s.global()));
  fft_inverse(ctx, s, 3, F, out3);
}

// Cubic B-spline coefficients of ncomp fields (in == out allowed).
void bspline_prefilter(vreg_ctx ctx, const Slab& s, int ncomp, const float* in, float* out) {
  const SpecDesc d = spec_desc(ctx, s);
  float2* F = spec_buffer(ctx, d, ncomp, ncomp == 3 ? "spec3" : "spec1");
  fft_forward(ctx, s, ncomp, in, F);
  Timed t(ctx, T_FFT, "spec_bspline");
  k_bspline_prefilter<<<dim3(unsigned(d.n2l), unsigned(ncomp * d.n1)), 128, 0, ctx->stream>>>(
      d, ncomp, F, float(1.0 / double(s.global())));
  count_launch(ctx);
  check_launch();
  fft_inverse(ctx, s, ncomp, F, out);
}

void h0_pointwise(vreg_ctx ctx, const Slab& s, const float* s3, const float* g3, float* out3) {
  k_h0_pointwise<<<blocks_for(s.local(), kT), kT, 0, ctx->stream>>>(s.local(), s3, g3, out3);
  count_launch(ctx);
  check_launch();
}

}  // namespace vb

using namespace vb;

extern "C" {

int vreg_regop(vreg_ctx ctx, const vreg_grid* g, const float* v3, double beta, int unit_zero,
               float* out3) {
  return guard([&] { spectral_regop(ctx, slab_of(ctx, g), v3, beta, unit_zero != 0, false, out3); });
}

int vreg_inv_regop(vreg_ctx ctx, const vreg_grid* g, const float* v3, double beta, float* out3) {
  return guard([&] { spectral_regop(ctx, slab_of(ctx, g), v3, beta, true, true, out3); });
}

int vreg_seminorm(vreg_ctx ctx, const vreg_grid* g, const float* v3, double* out) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    const SpecDesc d = spec_desc(ctx, s);
    float2* F = spec_buffer(ctx, d, 3, "spec3");
    fft_forward(ctx, s, 3, v3, F);
    double* rows = static_cast<double*>(workspace(ctx, "semi_rows", sizeof(double) * 3 * s.n2));
    k_seminorm_rows<<<dim3(d.n2l, 3), kT, 0, ctx->stream>>>(d, F, rows, ctx->reg_order);
    count_launch(ctx);
    check_launch();
    const double* src = rows;
    if (ctx->nranks > 1) {
      double* gl = static_cast<double*>(workspace(ctx, "semi_rows_g", sizeof(double) * 3 * s.n2));
      for (int c = 0; c < 3; ++c) {
        Slab rs = s;  // rows are distributed over k2 like planes over x1
        rs.n1 = s.n2;
        rs.n1l = d.n2l;
        allgather_partials(ctx, rs, rows + size_t(c) * d.n2l, gl + size_t(c) * s.n2, 1);
      }
      src = gl;
    }
    double* h = pinned(ctx, size_t(3) * s.n2);
    VB_CUDA(cudaMemcpyAsync(h, src, sizeof(double) * 3 * s.n2, cudaMemcpyDeviceToHost,
                            ctx->stream));
    VB_CUDA(cudaStreamSynchronize(ctx->stream));
    double total = 0.0;
    for (int c = 0; c < 3; ++c)
      for (int k2 = 0; k2 < s.n2; ++k2) total += h[size_t(c) * s.n2 + k2];
    const double two_pi = 6.283185307179586476925286766559;
    const double N = double(s.global());
    *out = total * (two_pi * two_pi * two_pi) / (N * N);
  });
}

int vreg_leray(vreg_ctx ctx, const vreg_grid* g, const float* v3, float* out3) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    const SpecDesc d = spec_desc(ctx, s);
    float2* F = spec_buffer(ctx, d, 3, "spec3");
    fft_forward(ctx, s, 3, v3, F);
    k_leray<<<blocks_for(d.nc, kT), kT, 0, ctx->stream>>>(d, F, float(1.0 / double(s.global())));
    count_launch(ctx);
    check_launch();
    fft_inverse(ctx, s, 3, F, out3);
  });
}

int vreg_restrict(vreg_ctx ctx, const vreg_grid* g, int ncomp, const float* f, float* outc) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    if (ctx->nranks > 1) {
      dist_restrict(ctx, s, ncomp, f, outc);
      return;
    }
    vreg_grid gc{s.n1 / 2, s.n2 / 2, s.n3 / 2, s.nt};
    Slab sc = slab_of(ctx, &gc);
    const SpecDesc df = spec_desc(ctx, s), dc = spec_desc(ctx, sc);
    float2* Ff = spec_buffer(ctx, df, ncomp, "spec_f");
    float2* Fc = spec_buffer(ctx, dc, ncomp, "spec_c");
    fft_forward(ctx, s, ncomp, f, Ff);
    // (Nc/Nf) partner sum, then the coarse inverse's 1/Nc: net 1/Nf
    k_restrict<<<blocks_for(dc.nc * ncomp, kT), kT, 0, ctx->stream>>>(
        Idx3(unsigned(dc.h), unsigned(sc.n2), dc.nc), s.n1, s.n2, s.n3, sc.n1, sc.n2, sc.n3, ncomp, Ff, Fc, float(1.0 / double(s.global())));
    count_launch(ctx);
    check_launch();
    fft_inverse(ctx, sc, ncomp, Fc, outc);
  });
}

int vreg_prolong(vreg_ctx ctx, const vreg_grid* g, int ncomp, const float* fc, float* outf) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    if (ctx->nranks > 1) {
      dist_prolong(ctx, s, ncomp, fc, outf);
      return;
    }
    vreg_grid gc{s.n1 / 2, s.n2 / 2, s.n3 / 2, s.nt};
    Slab sc = slab_of(ctx, &gc);
    const SpecDesc df = spec_desc(ctx, s), dc = spec_desc(ctx, sc);
    float2* Ff = spec_buffer(ctx, df, ncomp, "spec_f");
    float2* Fc = spec_buffer(ctx, dc, ncomp, "spec_c");
    fft_forward(ctx, sc, ncomp, fc, Fc);
    // (Nf/Nc)/nsplit, then the fine inverse's 1/Nf: net 1/(Nc nsplit)
    k_prolong<<<blocks_for(df.nc * ncomp, kT), kT, 0, ctx->stream>>>(
        Idx3(unsigned(df.h), unsigned(s.n2), df.nc), s.n1, s.n2, s.n3, sc.n1, sc.n2, sc.n3, ncomp, Fc, Ff, float(1.0 / double(sc.global())));
    count_launch(ctx);
    check_launch();
    fft_inverse(ctx, s, ncomp, Ff, outf);
  });
}

int vreg_high_pass(vreg_ctx ctx, const vreg_grid* g, int ncomp, const float* f, float* out) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    if (ctx->nranks > 1) {
      // high_pass(f) = f - prolong(restrict(f)) (test_spectral.cpp:242-247)
      float* fc = static_cast<float*>(
          workspace(ctx, "hp_coarse", size_t(ncomp) * s.local() / 8 * sizeof(float)));
      dist_restrict(ctx, s, ncomp, f, fc);
      dist_prolong(ctx, s, ncomp, fc, out);
      int st = vreg_sub(ctx, g, ncomp, f, out, out);
      require(st == VREG_OK, st, vreg_last_error());
      return;
    }
    const SpecDesc d = spec_desc(ctx, s);
    float2* F = spec_buffer(ctx, d, ncomp, "spec_f");
    float2* G = spec_buffer(ctx, d, ncomp, "spec_f2");
    fft_forward(ctx, s, ncomp, f, F);
    k_high_pass<<<blocks_for(d.nc * ncomp, kT), kT, 0, ctx->stream>>>(
        Idx3(unsigned(d.h), unsigned(s.n2), d.nc), s.n1, s.n2, s.n3, ncomp, F, G, float(1.0 / double(s.global())));
    count_launch(ctx);
    check_launch();
    fft_inverse(ctx, s, ncomp, G, out);
  });
}

int vreg_h0_matvec(vreg_ctx ctx, const vreg_grid* g, const float* s3, const float* gm3,
                   double beta_pc, float* out3) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    spectral_regop(ctx, s, s3, beta_pc, true, false, out3);
    h0_pointwise(ctx, s, s3, gm3, out3);
  });
}

int vreg_fft_forward(vreg_ctx ctx, const vreg_grid* g, const float* f, float* out_c) {
  return guard([&] {
    Slab s = slab_of(ctx, g);
    require(ctx->nranks == 1, VREG_ECONFIG, "fft_forward test hook is single-rank");
    fft_forward(ctx, s, 1, f, reinterpret_cast<float2*>(out_c));
  });
}

// Fused fine-grid work of the two-level preconditioner (precond.hpp:143-160)
// on one rank: one forward transform of r and one inverse for the result.
//   begin: F = R2C(r); one restriction pass gives restrict(F) and
//          restrict(InvA F) = InvA_c restrict(F); rc, sc = C2R_c of both.
//          F is kept for the end.
//   end:   out = C2R(prolong(R2C_c(sc)) + high_pass(InvA F)), the symbol
//          applied inside the high pass.
int vreg_two_level_begin(vreg_ctx ctx, const vreg_grid* g, const float* r3, double beta_pc,
                         float* rc3, float* sc3) {
  return guard([&] {
    require(ctx->nranks == 1, VREG_ECONFIG, "fused two-level apply is single-rank");
    require(beta_pc > 0.0, VREG_EPARAM, "regularization beta must be > 0");
    Slab s = slab_of(ctx, g);
    vreg_grid gc{s.n1 / 2, s.n2 / 2, s.n3 / 2, s.nt};
    Slab sc = slab_of(ctx, &gc);
    const SpecDesc df = spec_desc(ctx, s), dc = spec_desc(ctx, sc);
    float2* F = spec_buffer(ctx, df, 3, "tl_F");
    float2* Fc = rc3 ? spec_buffer(ctx, dc, 3, "tl_Fc") : nullptr;
    float2* Fs = spec_buffer(ctx, dc, 3, "tl_Fs");
    fft_forward(ctx, s, 3, r3, F);
    const float rs = float(1.0 / double(s.global()));
    k_restrict_pair<<<blocks_for(dc.nc * 3, kT), kT, 0, ctx->stream>>>(
        Idx3(unsigned(dc.h), unsigned(sc.n2), dc.nc), s.n1, s.n2, s.n3, sc.n1, sc.n2, sc.n3, F,
        Fc, Fs, rs, float(beta_pc), ctx->reg_order);
    count_launch(ctx);
    check_launch();
    if (rc3) fft_inverse(ctx, sc, 3, Fc, rc3);
    fft_inverse(ctx, sc, 3, Fs, sc3);
    ctx->tl_beta = beta_pc;  // F stays the spectrum of r; the end applies InvA to it
  });
}

int vreg_two_level_end(vreg_ctx ctx, const vreg_grid* g, const float* sc3, float* out3) {
  return guard([&] {
    require(ctx->nranks == 1, VREG_ECONFIG, "fused two-level apply is single-rank");
    Slab s = slab_of(ctx, g);
    vreg_grid gc{s.n1 / 2, s.n2 / 2, s.n3 / 2, s.nt};
    Slab sc = slab_of(ctx, &gc);
    const SpecDesc df = spec_desc(ctx, s), dc = spec_desc(ctx, sc);
    float2* F = spec_buffer(ctx, df, 3, "tl_F");
    float2* Fc = spec_buffer(ctx, dc, 3, "tl_Fc");
    float2* G = spec_buffer(ctx, df, 3, "tl_G");
    fft_forward(ctx, sc, 3, sc3, Fc);
    // (fusing this pass with the x1 pass of the inverse -- plane C2R after
    // one pencil kernel -- measured slower: 1.94 vs 1.88 ms per apply, the
    // pencil kernel's strided k1 reads at 224 us)
    k_prolong_plus_hp<<<blocks_for(size_t(3) * s.n1 * s.n2, kT / 32), kT, 0, ctx->stream>>>(
        s.n1, s.n2, s.n3, sc.n1, sc.n2, sc.n3, Fc, F, G, float(1.0 / double(sc.global())),
        float(1.0 / double(s.global())), float(ctx->tl_beta), ctx->reg_order);
    count_launch(ctx);
    check_launch();
    fft_inverse(ctx, s, 3, G, out3);
  });
}

}  // extern "C"
