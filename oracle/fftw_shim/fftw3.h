/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
 *
 * Minimal FFTW3-API shim so the unmodified reference core (`/root/reference/proj/core`)
 * compiles and runs in this image, which has no libfftw3.  It declares exactly the entry
 * points the reference calls (`proj/core/src/fft.cpp:23-63`):
 *   fftw{,f}_malloc / _free / _plan_dft_r2c_2d / _plan_dft_1d / _execute / _destroy_plan
 * The arithmetic lives in fftw_shim.cpp (mixed-radix Cooley-Tukey + Bluestein), which is
 * an independent implementation of the published DFT definitions FFTW computes:
 *   forward  X[k] = sum_n x[n] exp(-2 pi i n k / n)   (FFTW_FORWARD  = -1)
 *   backward X[k] = sum_n x[n] exp(+2 pi i n k / n)   (FFTW_BACKWARD = +1)
 * both unnormalised; r2c_2d(n0 = rows, n1 = cols) writes the n0 x (n1/2+1) half plane.
 */
#ifndef DDM_ORACLE_FFTW_SHIM_H
#define DDM_ORACLE_FFTW_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

typedef double fftw_complex[2];
typedef float fftwf_complex[2];

typedef struct ddm_shim_plan_d* fftw_plan;
typedef struct ddm_shim_plan_f* fftwf_plan;

void* fftw_malloc(size_t n);
void fftw_free(void* p);
fftw_plan fftw_plan_dft_r2c_2d(int n0, int n1, double* in, fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

void* fftwf_malloc(size_t n);
void fftwf_free(void* p);
fftwf_plan fftwf_plan_dft_r2c_2d(int n0, int n1, float* in, fftwf_complex* out, unsigned flags);
fftwf_plan fftwf_plan_dft_1d(int n, fftwf_complex* in, fftwf_complex* out, int sign,
                             unsigned flags);
void fftwf_execute(const fftwf_plan p);
void fftwf_destroy_plan(fftwf_plan p);

#ifdef __cplusplus
}
#endif

#endif
