/* CPU implementation of the FFTW3-API subset in fftw3.h.
 *
 * TEST INFRASTRUCTURE ONLY (oracle/ build of the reference, never linked into
 * the product). Stands in for the absent FFTW3 so the reference's FftPlan
 * (proj/src/fft.cpp:24-64) builds unmodified. Pinned by the reference's own
 * spectral tests (proj/tests/test_spectral.cpp:49-83: DC-only, single mode,
 * round trip 1e-12, Parseval 1e-12), which oracle/Makefile runs.
 *
 * Algorithm: recursive mixed-radix decimation-in-time Cooley-Tukey with
 * specialised radix-2/4 butterflies and a generic radix-p butterfly, one
 * precomputed twiddle table per length. 3-D r2c = two real x3-lines packed
 * into one complex FFT, then complex FFTs along x2 and x1 on the half space.
 * c2r is the exact reverse and drops the imaginary part of the k3 = 0 and
 * k3 = n3/2 entries (FFTW's c2r convention for the self-conjugate planes).
 */
#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double re, im;
} cpx;

typedef struct {
  int n;
  int fac[64]; /* (p, m) pairs, p*m = length at that level */
  cpx* tw;     /* exp(-2 pi i k / n), k = 0..n-1 */
  cpx* tmp;    /* line buffers */
  cpx* tmp2;
  cpx* scr;    /* radix-p scratch */
} fft1d;

struct shim_plan_s {
  int kind; /* 0 = r2c, 1 = c2r */
  int single;
  int n0, n1, n2;
  void* in;
  void* out;
  fft1d *f0, *f1, *f2;
  cpx* work; /* n0*n1*(n2/2+1) */
};

static void factorize(int n, int* fac) {
  int p = 4, k = 0;
  double fl = floor(sqrt((double)n));
  do {
    while (n % p) {
      switch (p) {
        case 4: p = 2; break;
        case 2: p = 3; break;
        default: p += 2; break;
      }
      if (p > fl) p = n;
    }
    n /= p;
    fac[k++] = p;
    fac[k++] = n;
  } while (n > 1);
}

static fft1d* fft1d_new(int n) {
  fft1d* f = (fft1d*)calloc(1, sizeof(fft1d));
  f->n = n;
  factorize(n, f->fac);
  f->tw = (cpx*)malloc(sizeof(cpx) * (size_t)n);
  for (int k = 0; k < n; ++k) {
    const double a = -2.0 * M_PI * (double)k / (double)n;
    f->tw[k].re = cos(a);
    f->tw[k].im = sin(a);
  }
  f->tmp = (cpx*)malloc(sizeof(cpx) * (size_t)n);
  f->tmp2 = (cpx*)malloc(sizeof(cpx) * (size_t)n);
  f->scr = (cpx*)malloc(sizeof(cpx) * (size_t)n);
  return f;
}

static void fft1d_free(fft1d* f) {
  if (!f) return;
  free(f->tw);
  free(f->tmp);
  free(f->tmp2);
  free(f->scr);
  free(f);
}

static inline cpx cmul(cpx a, cpx b) {
  cpx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}

static inline cpx twid(const fft1d* f, size_t k, int sign) {
  cpx w = f->tw[k];
  if (sign > 0) w.im = -w.im;
  return w;
}

static void butterfly(cpx* out, size_t fstride, const fft1d* f, int m, int p,
                      int sign) {
  const int N = f->n;
  if (p == 2) {
    for (int u = 0; u < m; ++u) {
      cpx t = cmul(out[u + m], twid(f, (size_t)u * fstride, sign));
      out[u + m].re = out[u].re - t.re;
      out[u + m].im = out[u].im - t.im;
      out[u].re += t.re;
      out[u].im += t.im;
    }
    return;
  }
  if (p == 4) {
    const double s = (double)sign; /* W4 = exp(sign * i pi/2) = sign * i */
    for (int u = 0; u < m; ++u) {
      cpx y0 = out[u];
      cpx y1 = cmul(out[u + m], twid(f, (size_t)u * fstride, sign));
      cpx y2 = cmul(out[u + 2 * m], twid(f, (size_t)2 * u * fstride, sign));
      cpx y3 = cmul(out[u + 3 * m], twid(f, (size_t)3 * u * fstride, sign));
      cpx a = {y0.re + y2.re, y0.im + y2.im};
      cpx b = {y0.re - y2.re, y0.im - y2.im};
      cpx c = {y1.re + y3.re, y1.im + y3.im};
      cpx d = {y1.re - y3.re, y1.im - y3.im};
      /* i*s*d */
      cpx isd = {-s * d.im, s * d.re};
      out[u].re = a.re + c.re;
      out[u].im = a.im + c.im;
      out[u + 2 * m].re = a.re - c.re;
      out[u + 2 * m].im = a.im - c.im;
      out[u + m].re = b.re + isd.re;
      out[u + m].im = b.im + isd.im;
      out[u + 3 * m].re = b.re - isd.re;
      out[u + 3 * m].im = b.im - isd.im;
    }
    return;
  }
  cpx* t = f->scr;
  const size_t np = (size_t)(N / p);
  for (int u = 0; u < m; ++u) {
    for (int q = 0; q < p; ++q)
      t[q] = cmul(out[u + q * m], twid(f, ((size_t)q * u * fstride) % N, sign));
    for (int s = 0; s < p; ++s) {
      cpx acc = {0.0, 0.0};
      for (int q = 0; q < p; ++q) {
        cpx w = twid(f, (size_t)((q * s) % p) * np, sign);
        cpx v = cmul(t[q], w);
        acc.re += v.re;
        acc.im += v.im;
      }
      out[u + s * m] = acc;
    }
  }
}

static void work(cpx* out, const cpx* in, size_t fstride, const int* fac,
                 const fft1d* f, int sign) {
  const int p = fac[0], m = fac[1];
  if (m == 1) {
    for (int k = 0; k < p; ++k) out[k] = in[(size_t)k * fstride];
  } else {
    for (int q = 0; q < p; ++q)
      work(out + (size_t)q * m, in + (size_t)q * fstride, fstride * (size_t)p,
           fac + 2, f, sign);
  }
  butterfly(out, fstride, f, m, p, sign);
}

/* in-place transform of a strided line through the plan's buffers */
static void fft_line(fft1d* f, cpx* base, size_t stride, int sign) {
  const int n = f->n;
  for (int k = 0; k < n; ++k) f->tmp[k] = base[(size_t)k * stride];
  work(f->tmp2, f->tmp, 1, f->fac, f, sign);
  for (int k = 0; k < n; ++k) base[(size_t)k * stride] = f->tmp2[k];
}

static void axes01(struct shim_plan_s* p, int sign) {
  const int n0 = p->n0, n1 = p->n1, h = p->n2 / 2 + 1;
  cpx* C = p->work;
  for (int i = 0; i < n0; ++i)
    for (int k = 0; k < h; ++k)
      fft_line(p->f1, C + (size_t)i * n1 * h + k, (size_t)h, sign);
  for (int j = 0; j < n1; ++j)
    for (int k = 0; k < h; ++k)
      fft_line(p->f0, C + (size_t)j * h + k, (size_t)n1 * h, sign);
}

static double rd(const struct shim_plan_s* p, size_t i) {
  return p->single ? (double)((const float*)p->in)[i] : ((const double*)p->in)[i];
}

static void exec_r2c(struct shim_plan_s* p) {
  const int n2 = p->n2, h = n2 / 2 + 1;
  const size_t lines = (size_t)p->n0 * p->n1;
  fft1d* f = p->f2;
  for (size_t L = 0; L < lines; L += 2) {
    const int has_b = L + 1 < lines;
    for (int x = 0; x < n2; ++x) {
      f->tmp[x].re = rd(p, L * n2 + x);
      f->tmp[x].im = has_b ? rd(p, (L + 1) * n2 + x) : 0.0;
    }
    work(f->tmp2, f->tmp, 1, f->fac, f, -1);
    const cpx* Z = f->tmp2;
    for (int k = 0; k < h; ++k) {
      const cpx zk = Z[k];
      const cpx zc = Z[(n2 - k) % n2];
      /* A = (Z_k + conj Z_-k)/2 ; B = -i (Z_k - conj Z_-k)/2 */
      cpx A = {0.5 * (zk.re + zc.re), 0.5 * (zk.im - zc.im)};
      cpx B = {0.5 * (zk.im + zc.im), -0.5 * (zk.re - zc.re)};
      p->work[L * h + k] = A;
      if (has_b) p->work[(L + 1) * h + k] = B;
    }
  }
  axes01(p, -1);
  const size_t nc = lines * (size_t)h;
  if (p->single) {
    float* o = (float*)p->out;
    for (size_t i = 0; i < nc; ++i) {
      o[2 * i] = (float)p->work[i].re;
      o[2 * i + 1] = (float)p->work[i].im;
    }
  } else {
    memcpy(p->out, p->work, sizeof(cpx) * nc);
  }
}

static void exec_c2r(struct shim_plan_s* p) {
  const int n2 = p->n2, h = n2 / 2 + 1;
  const size_t lines = (size_t)p->n0 * p->n1;
  const size_t nc = lines * (size_t)h;
  if (p->single) {
    const float* in = (const float*)p->in;
    for (size_t i = 0; i < nc; ++i) {
      p->work[i].re = in[2 * i];
      p->work[i].im = in[2 * i + 1];
    }
  } else {
    memcpy(p->work, p->in, sizeof(cpx) * nc);
  }
  axes01(p, +1);
  fft1d* f = p->f2;
  for (size_t L = 0; L < lines; L += 2) {
    const int has_b = L + 1 < lines;
    const cpx* A = p->work + L * h;
    const cpx* B = has_b ? p->work + (L + 1) * h : NULL;
    for (int k = 0; k < n2; ++k) {
      cpx a, b = {0.0, 0.0};
      if (k < h) {
        a = A[k];
        if (B) b = B[k];
        if (k == 0 || 2 * k == n2) {
          a.im = 0.0;
          b.im = 0.0;
        }
      } else {
        a = A[n2 - k];
        a.im = -a.im;
        if (B) {
          b = B[n2 - k];
          b.im = -b.im;
        }
      }
      /* z = a + i b */
      f->tmp[k].re = a.re - b.im;
      f->tmp[k].im = a.im + b.re;
    }
    work(f->tmp2, f->tmp, 1, f->fac, f, +1);
    for (int x = 0; x < n2; ++x) {
      if (p->single) {
        float* o = (float*)p->out;
        o[L * n2 + x] = (float)f->tmp2[x].re;
        if (has_b) o[(L + 1) * n2 + x] = (float)f->tmp2[x].im;
      } else {
        double* o = (double*)p->out;
        o[L * n2 + x] = f->tmp2[x].re;
        if (has_b) o[(L + 1) * n2 + x] = f->tmp2[x].im;
      }
    }
  }
}

static struct shim_plan_s* mk(int kind, int single, int n0, int n1, int n2,
                              void* in, void* out) {
  if (n0 < 1 || n1 < 1 || n2 < 2) return NULL;
  struct shim_plan_s* p = (struct shim_plan_s*)calloc(1, sizeof(*p));
  p->kind = kind;
  p->single = single;
  p->n0 = n0;
  p->n1 = n1;
  p->n2 = n2;
  p->in = in;
  p->out = out;
  p->f0 = fft1d_new(n0);
  p->f1 = fft1d_new(n1);
  p->f2 = fft1d_new(n2);
  p->work = (cpx*)malloc(sizeof(cpx) * (size_t)n0 * n1 * (size_t)(n2 / 2 + 1));
  return p;
}

static void destroy(struct shim_plan_s* p) {
  if (!p) return;
  fft1d_free(p->f0);
  fft1d_free(p->f1);
  fft1d_free(p->f2);
  free(p->work);
  free(p);
}

static void execute(struct shim_plan_s* p) {
  if (p->kind == 0)
    exec_r2c(p);
  else
    exec_c2r(p);
}

void* fftw_malloc(size_t n) { return malloc(n ? n : 1); }
void fftw_free(void* p) { free(p); }
fftw_plan fftw_plan_dft_r2c_3d(int n0, int n1, int n2, double* in,
                               fftw_complex* out, unsigned flags) {
  (void)flags;
  return mk(0, 0, n0, n1, n2, in, out);
}
fftw_plan fftw_plan_dft_c2r_3d(int n0, int n1, int n2, fftw_complex* in,
                               double* out, unsigned flags) {
  (void)flags;
  return mk(1, 0, n0, n1, n2, in, out);
}
void fftw_execute(const fftw_plan p) { execute(p); }
void fftw_destroy_plan(fftw_plan p) { destroy(p); }

void* fftwf_malloc(size_t n) { return malloc(n ? n : 1); }
void fftwf_free(void* p) { free(p); }
fftwf_plan fftwf_plan_dft_r2c_3d(int n0, int n1, int n2, float* in,
                                 fftwf_complex* out, unsigned flags) {
  (void)flags;
  return mk(0, 1, n0, n1, n2, in, out);
}
fftwf_plan fftwf_plan_dft_c2r_3d(int n0, int n1, int n2, fftwf_complex* in,
                                 float* out, unsigned flags) {
  (void)flags;
  return mk(1, 1, n0, n1, n2, in, out);
}
void fftwf_execute(const fftwf_plan p) { execute(p); }
void fftwf_destroy_plan(fftwf_plan p) { destroy(p); }
