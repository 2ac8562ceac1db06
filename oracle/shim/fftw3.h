/* FFTW3-API subset used by the reference's FftPlan (proj/src/fft.cpp:3-64).
 *
 * TEST INFRASTRUCTURE ONLY. FFTW3 is not installed in this image (SURVEY.md
 * §8c item 1; the reference pins no version, proj/CMakeLists.txt:14-15). This
 * header declares exactly the calls the reference makes -- malloc/free,
 * plan_dft_r2c_3d / plan_dft_c2r_3d with FFTW_ESTIMATE, execute, destroy_plan,
 * in double and float flavours -- with FFTW's published semantics:
 * forward transform unnormalised with sign -1, r2c output is the half-space
 * n0 x n1 x (n2/2+1), c2r is the unnormalised inverse (sign +1) that ignores
 * the imaginary parts of the self-conjugate k2 = 0 and k2 = n2/2 planes.
 * Implementation: fftw_shim.c (own code, mixed-radix Cooley-Tukey).
 */
#ifndef VREG_ORACLE_FFTW3_SHIM_H
#define VREG_ORACLE_FFTW3_SHIM_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef float fftwf_complex[2];
typedef struct shim_plan_s* fftw_plan;
typedef struct shim_plan_s* fftwf_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_MEASURE (0U)

void* fftw_malloc(size_t n);
void fftw_free(void* p);
fftw_plan fftw_plan_dft_r2c_3d(int n0, int n1, int n2, double* in,
                               fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r_3d(int n0, int n1, int n2, fftw_complex* in,
                               double* out, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

void* fftwf_malloc(size_t n);
void fftwf_free(void* p);
fftwf_plan fftwf_plan_dft_r2c_3d(int n0, int n1, int n2, float* in,
                                 fftwf_complex* out, unsigned flags);
fftwf_plan fftwf_plan_dft_c2r_3d(int n0, int n1, int n2, fftwf_complex* in,
                                 float* out, unsigned flags);
void fftwf_execute(const fftwf_plan p);
void fftwf_destroy_plan(fftwf_plan p);

#ifdef __cplusplus
}
#endif
#endif
