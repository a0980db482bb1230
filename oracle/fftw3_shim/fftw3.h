/*
 * FFTW3-API shim (fp64) — TEST INFRASTRUCTURE ONLY.
 *
 * The reference (`/root/reference/proj`) links FFTW3, which is not vendored and not
 * installed in this image. This header declares exactly the FFTW
 * symbols the reference's `core/fft.hpp` uses (fft.hpp:30-42,53,60,78-90,99,106) so
 * that the UNMODIFIED reference headers compile into the oracle (`oracle/_ref`).
 * Semantics follow FFTW's documented contract: unnormalized transforms, forward sign
 * -1, r2c/c2r over the last (contiguous) axis half spectrum, plans bound to the
 * arrays given at plan time. The implementation is an in-repo mixed-radix Stockham
 * FFT (`fftw_shim.cpp`), not FFTW. Never linked into the product.
 */
#ifndef USTFWI_ORACLE_FFTW3_SHIM_H
#define USTFWI_ORACLE_FFTW3_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_DESTROY_INPUT (1U << 0)
#define FFTW_PRESERVE_INPUT (1U << 4)
#define FFTW_ESTIMATE (1U << 6)

void* fftw_malloc(size_t n);
void fftw_free(void* p);
fftw_plan fftw_plan_dft_r2c(int rank, const int* n, double* in, fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r(int rank, const int* n, fftw_complex* in, double* out, unsigned flags);
fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
