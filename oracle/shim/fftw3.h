/* ORACLE TEST INFRASTRUCTURE — not product code.
 *
 * From-scratch subset of the fftw3.h API used by the reference's fft.cpp
 * (/root/reference/proj/src/fft.cpp:3,28-35,48-49,57-58): complex-to-complex
 * 1-D plans, unnormalised, exact length n (mixed radix for 7-smooth factors,
 * Bluestein otherwise). FFTW itself is absent from this image; see
 * SURVEY.md §8(c). The transform is exact up to fp64 round-off.
 */
#pragma once

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct shim_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif
